// ref_shim_scheduler.cpp — extern "C" access to the reference's admission
// decision, schedule() (/root/reference/proj/src/scheduler.cpp:74-170, compiled
// in place by oracle/Makefile).  TEST INFRASTRUCTURE: the checker of the
// executor's memory-budget admission (paper_2312_02515_b200/executor.py).
#include <exception>
#include <string>
#include <vector>

#include "fusim/scheduler.hpp"

// Job i: ids[i], priority[i], submit[i], batch_size[i], its dataset item lengths
// (counts[i] of them, flattened in `lengths`), cursor[i], static memory_gb[i].
// strategy: 0 M1 fifo, 1 M2 priority, 2 M3 minpad.  has_model: use beta[0..2]
// (rmse irrelevant).  out_idx receives the selected job indices in admission
// order, *out_n their count, *est_gb the decision's estimated memory.
extern "C" int ref_schedule(int n, const char* const* ids, const int* priority, const double* submit,
                            const int* batch_size, const int* counts, const int* lengths, const long* cursor,
                            const double* memory_gb, int strategy, int has_model, const double* beta,
                            double budget_gb, double floor_gb, int max_concurrent, int* out_idx, int* out_n,
                            double* est_gb) {
    try {
        std::vector<fusim::JobState> states;
        states.reserve(n);
        int off = 0;
        for (int i = 0; i < n; ++i) {
            fusim::JobSpec s;
            s.id = ids[i];
            s.priority = priority[i];
            s.submit_time = submit[i];
            s.batch_size = batch_size[i];
            s.memory_gb = memory_gb[i];
            for (int t = 0; t < counts[i]; ++t) s.dataset.items.push_back(fusim::DataItem{lengths[off + t]});
            off += counts[i];
            states.emplace_back(s);
            states.back().cursor = static_cast<std::size_t>(cursor[i]);
        }
        std::vector<const fusim::JobState*> queue;
        for (const auto& js : states) queue.push_back(&js);
        fusim::SchedulerConfig cfg;
        cfg.strategy = strategy == 0 ? fusim::Strategy::FifoM1
                     : strategy == 1 ? fusim::Strategy::PriorityM2
                                     : fusim::Strategy::MinPadM3;
        cfg.memory_budget_gb = budget_gb;
        cfg.memory_floor_gb = floor_gb;
        cfg.max_concurrent = max_concurrent;
        fusim::MemoryModel model;
        if (has_model) {
            model.beta0 = beta[0];
            model.beta1 = beta[1];
            model.beta2 = beta[2];
        }
        const auto d = fusim::schedule(queue, cfg, has_model ? &model : nullptr, nullptr);
        int k = 0;
        for (const auto& id : d.selected)
            for (int i = 0; i < n; ++i)
                if (states[i].spec.id == id) out_idx[k++] = i;
        *out_n = k;
        *est_gb = d.estimated_memory_gb;
        return 0;
    } catch (const std::exception&) {
        return 9;
    }
}
