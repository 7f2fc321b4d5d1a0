// facade_forward_io — runs fusim::fused_forward (the B200 façade) on cases read
// from stdin and writes the outputs to stdout, so tests/test_facade_cpp.py can
// compare them BIT FOR BIT with the reference's own outputs (tests/golden/).
// Input per case (little-endian): int32 d, k, J, ranks[J], nseq, seq_job[nseq],
// seq_len[nseq]; then float64 W0[d*k], A_all, B_all, X_all.  Output per case:
// float64 out[S * max_len * d].  With --bf16 the cases run through
// fusim::b200::fused_forward_bf16 (the tcgen05 path behind the same signature).
#include <cstdint>
#include <cstdio>
#include <map>
#include <vector>

#include <cstring>

#include "fusim/b200.hpp"
#include "fusim/lora.hpp"

using namespace fusim;

template <class T>
static bool rd(T* p, size_t n) { return std::fread(p, sizeof(T), n, stdin) == n; }

int main(int argc, char** argv) {
    const bool bf16 = argc > 1 && std::strcmp(argv[1], "--bf16") == 0;
    int32_t ncases = 0;
    if (!rd(&ncases, 1)) return 2;
    for (int c = 0; c < ncases; ++c) {
        int32_t d, k, J;
        rd(&d, 1); rd(&k, 1); rd(&J, 1);
        std::vector<int32_t> ranks(J);
        rd(ranks.data(), J);
        int32_t nseq;
        rd(&nseq, 1);
        std::vector<int32_t> sj(nseq), sl(nseq);
        rd(sj.data(), nseq); rd(sl.data(), nseq);
        Matrix W0(d, k);
        rd(W0.data.data(), W0.data.size());
        std::map<std::string, AdapterWeights> adapters;
        std::vector<AdapterWeights> ads(J);
        for (int j = 0; j < J; ++j) { ads[j].A = Matrix(ranks[j], k); rd(ads[j].A.data.data(), ads[j].A.data.size()); }
        for (int j = 0; j < J; ++j) { ads[j].B = Matrix(d, ranks[j]); rd(ads[j].B.data.data(), ads[j].B.data.size()); }
        for (int j = 0; j < J; ++j) {
            ads[j].job_id = "j" + std::to_string(j);
            ads[j].rank = ranks[j];
            adapters[ads[j].job_id] = ads[j];
        }
        std::vector<JobBatch> batches;
        for (int s = 0; s < nseq; ++s) {
            const std::string id = "j" + std::to_string(sj[s]);
            if (batches.empty() || batches.back().job_id != id) batches.push_back(JobBatch{id, {}});
            Matrix x(sl[s], k);
            rd(x.data.data(), x.data.size());
            batches.back().sequences.push_back(std::move(x));
        }
        const auto fb = fuse(batches);
        const auto outs = bf16 ? b200::fused_forward_bf16(W0, adapters, fb) : fused_forward(W0, adapters, fb);
        for (const auto& o : outs) std::fwrite(o.data.data(), sizeof(double), o.data.size(), stdout);
    }
    return 0;
}
