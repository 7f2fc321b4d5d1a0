// executor_loop — a run_simulation-shaped loop (sim.cpp:163-191) driven through
// the B200 façade's real executor (fusim::b200::FusedIterationExecutor): every
// fused iteration runs on the GPU and its IterationDone{ξ, ξ_p, jobs_in_batch}
// is charged with the MEASURED device time.  Prints one JSON line per event
// (losses also as float32 bit patterns) and a final line with the
// IterationTimeModel fitted from the measured iterations, so
// tests/test_gpu_cpp_executor.py can compare the trace with the Python
// executor's (paper_2312_02515_b200/executor.py) on the same workload.
//
//   executor_loop <padded 0|1> <strategy fifo|priority|minpad>
//
// The workload (6 jobs, TINY layer) is the one EXECUTOR_WORKLOAD in the test.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "fusim/b200.hpp"

using namespace fusim;

int main(int argc, char** argv) {
    const bool padded = argc > 1 && std::string(argv[1]) == "1";
    const std::string strat = argc > 2 ? argv[2] : "minpad";
    const b200::Strategy strategy = strat == "fifo" ? b200::Strategy::Fifo
                                    : strat == "priority" ? b200::Strategy::Priority
                                                          : b200::Strategy::MinPad;
    const int prio[6] = {1, 2, 1, 3, 1, 2};
    const double submit[6] = {0.0, 0.0, 1.0, 1.0, 2.0, 2.0};
    const int bs[6] = {2, 3, 2, 2, 4, 2};
    const int rank[6] = {8, 16, 32, 8, 16, 64};
    const float lr[6] = {1e-3f, 2e-3f, 5e-4f, 1e-3f, 3e-3f, 1e-3f};
    const int iters[6] = {5, 7, 4, 6, 8, 5};
    std::vector<b200::ExecutorJob> jobs;
    for (int i = 0; i < 6; ++i) {
        b200::ExecutorJob j;
        j.spec.id = "job" + std::to_string(i);
        j.spec.priority = prio[i];
        j.spec.submit_time = submit[i];
        j.spec.batch_size = bs[i];
        j.spec.lora_rank = rank[i];
        j.spec.true_iterations = iters[i];
        for (int t = 0; t < 6; ++t) j.spec.dataset.items.push_back(DataItem{(17 * (i + 1) * (t + 3)) % 190 + 8});
        j.scale = 2.0f;
        j.lr = lr[i];
        jobs.push_back(std::move(j));
    }
    try {
        b200::FusedIterationExecutor ex(0, b200::llama_layer(256, 688), jobs, 3, strategy, padded, 7);
        const long launches0 = ex.layer().launches();
        const auto events = ex.run();
        for (const auto& e : events) {
            std::printf("{\"total_tokens\": %ld, \"padding_tokens\": %ld, \"effective_tokens\": %ld, \"rows\": %ld, "
                        "\"jobs_in_batch\": %d, \"duration_s\": %.9g, \"time\": %.9g, \"routing\": [",
                        e.total_tokens, e.padding_tokens, e.effective_tokens, e.rows, e.jobs_in_batch, e.duration_s,
                        e.time);
            for (std::size_t i = 0; i < e.routing.size(); ++i)
                std::printf("%s\"%s\"", i ? ", " : "", e.routing[i].c_str());
            std::printf("], \"loss_bits\": {");
            bool first = true;
            for (const auto& kv : e.losses) {
                std::uint32_t u;
                std::memcpy(&u, &kv.second, 4);
                std::printf("%s\"%s\": %u", first ? "" : ", ", kv.first.c_str(), u);
                first = false;
            }
            std::printf("}}\n");
        }
        const b200::IterationTimeModel fit = b200::fit_iteration_time(events);
        std::printf("{\"fit\": {\"base\": %.9g, \"per_token\": %.9g, \"per_launch\": %.9g}, \"launches\": %ld, "
                    "\"clock\": %.9g}\n",
                    fit.base, fit.per_token, fit.per_launch, ex.layer().launches() - launches0, ex.clock());
    } catch (const std::exception& e) {
        std::fprintf(stderr, "executor_loop: %s\n", e.what());
        return 1;
    }
    return 0;
}
