// ref_shim_memory.cpp — extern "C" access to the reference's memory-model fit
// (/root/reference/proj/src/memory_model.cpp, compiled in place by oracle/Makefile).
// TEST INFRASTRUCTURE: used to check that the B200 memory probes
// (tools/memory_probe.py) feed the reference's own Eq. 6 fit.
#include <string>
#include <vector>

#include "fusim/errors.hpp"
#include "fusim/memory_model.hpp"

extern "C" int ref_fit_memory_model(int n, const int* bs, const int* seq, const double* mem, int nonneg,
                                    double* out /* beta0, beta1, beta2, rmse */) {
    try {
        std::vector<fusim::MemSample> s(n);
        for (int i = 0; i < n; ++i) s[i] = fusim::MemSample{bs[i], seq[i], mem[i]};
        const fusim::MemoryModel m = fusim::fit_memory_model(
            s, nonneg ? fusim::FitConstraint::NonNegative : fusim::FitConstraint::Unconstrained);
        out[0] = m.beta0;
        out[1] = m.beta1;
        out[2] = m.beta2;
        out[3] = m.rmse;
        return 0;
    } catch (const fusim::FitError&) {
        return 8;
    } catch (const std::exception&) {
        return 9;
    }
}
