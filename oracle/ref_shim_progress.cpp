// ref_shim_progress.cpp — extern "C" access to the reference's early-stop rule
// (/root/reference/proj/src/progress.cpp:90-124, compiled in place by
// oracle/Makefile).  TEST INFRASTRUCTURE: pins the executor's restatement
// (paper_2312_02515_b200/executor.py detect_stop) on random loss/accuracy streams.
#include <exception>
#include <vector>

#include "fusim/progress.hpp"

// Returns 1 and fills (iteration, cause) when a stop fires, 0 when none, 9 on error.
// cause: 0 NaNLoss, 1 AccuracyDecline, 2 Completed.
extern "C" int ref_detect_stop(int nl, const double* losses, int na, const double* accs, int patience,
                               int* iteration, int* cause) {
    try {
        std::vector<double> l(losses, losses + nl), a(accs, accs + na);
        fusim::StopPolicy pol;
        pol.patience = patience;
        const auto ev = fusim::detect_stop("job", l, a, pol);
        if (!ev) return 0;
        *iteration = ev->iteration;
        *cause = ev->cause == fusim::StopCause::NaNLoss ? 0 : ev->cause == fusim::StopCause::AccuracyDecline ? 1 : 2;
        return 1;
    } catch (const std::exception&) {
        return 9;
    }
}
