// fusim/b200.hpp — B200 extensions of the fusim façade (libfusim_b200.so).
//
// The reference's C++ API (fusim/lora.hpp, batch_select.hpp, workload.hpp) is
// reproduced unchanged by the other façade headers.  This header adds what a
// reference user needs to move the hot path itself onto the B200:
//
//  (1) fused_forward_bf16 — the reference's fused_forward signature
//      (/root/reference/proj/include/fusim/lora.hpp:93-95) on the bf16 tcgen05
//      path: fp64 -> bf16 marshalling, one mlora_linear_fwd, the same
//      vector<Matrix> out (pad rows zero) and the same exceptions, raised
//      before any device work.
//  (2) FusedLayer — one transformer layer's LoRA'd projections for J jobs on
//      one GPU; step() is ONE C-ABI call (mlora_layer_step_timed): fwd + loss +
//      bwd + per-job AdamW, returning the per-job losses and the measured
//      device time.
//  (3) FusedIterationExecutor — the runtime counterpart of the simulator's
//      fused iteration (/root/reference/proj/src/sim.cpp:163-191): peek every
//      live job's next batch (JobState::next_candidate_batch, workload.cpp:50-60),
//      select (select_fifo / _priority / _minpad, batch_select.cpp:56-128),
//      account ξ / ξ_p (fused_shape, lora.cpp:72-85), fuse the rows on the
//      device (fuse, lora.cpp:114-158), run the step, commit the items
//      (workload.cpp:62-66) and emit IterationDone{ξ, ξ_p, jobs_in_batch}
//      (sim.cpp:185-191) charged with the MEASURED device time instead of
//      IterationTimeModel's analytic base + per_token·ξ + per_launch·launches
//      (sim.cpp:177-179).
//  (4) fit_iteration_time — least-squares IterationTimeModel{base, per_token,
//      per_launch = 0} from measured iterations: a drop-in value for the
//      reference's SimConfig::iter_time (sim.hpp:15-19), so the unmodified
//      simulator charges B200-measured time.
//
// Synthetic weights and per-job datasets are initialised with the library's
// counter-based fill (mlora_fill_uniform, seeds from mix_seed), exactly as the
// Python host does (paper_2312_02515_b200/layer.py, executor.py), so the two
// hosts run bit-identical iterations.
#pragma once

#include <cstdint>
#include <initializer_list>
#include <map>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include "fusim/batch_select.hpp"
#include "fusim/lora.hpp"
#include "fusim/workload.hpp"

struct mlora_ctx;

namespace fusim::b200 {

/// 64-bit FNV-1a over the parts (the per-tensor seed of the synthetic fills);
/// identical to paper_2312_02515_b200.fused.mix_seed.
std::uint64_t mix_seed(std::initializer_list<std::int64_t> parts);

/// (1) fusim::fused_forward on the bf16 tcgen05 path (bf16 operands, fp32
/// accumulation: rel-L2 <= 1e-2 against the fp64 reference).  Preconditions and
/// exceptions as lora.cpp:160-167 (ShapeError on W0.cols != fb.dim, RoutingError
/// for an unknown job, before any device work).  d and k are zero-padded to
/// multiples of 8 (TMA row pitch) on the way in and cropped on the way out.
std::vector<Matrix> fused_forward_bf16(const Matrix& W0,
                                       const std::map<std::string, AdapterWeights>& adapters,
                                       const FusedBatch& fb);

/// One LoRA'd projection of a layer: Y = X W0^T + s (X A^T) B^T, W0 d x k.
/// src: "x" (the layer input) or the name of the projection whose Y feeds it;
/// src_col0 > 0 or a wider source reads a column slice of that Y.
struct Projection {
    std::string name;
    int d = 0;
    int k = 0;
    std::string src = "x";
    int src_col0 = 0;
};

/// LLaMA-style layer (q, k, v, o, gate, up, down); o <- v, down <- up (the
/// bench's step semantics).
std::vector<Projection> llama_layer(int hidden, int ffn);

struct TrainJob {
    int rank = 16;
    float scale = 2.0f;
    float lr = 1e-4f;
};

/// (2) One layer's fused multi-LoRA training state for J jobs on one GPU.
class FusedLayer {
public:
    FusedLayer(int device, std::vector<Projection> shapes, std::vector<TrainJob> jobs, long capacity,
               std::uint64_t seed);
    ~FusedLayer();
    FusedLayer(const FusedLayer&) = delete;
    FusedLayer& operator=(const FusedLayer&) = delete;

    int num_jobs() const;
    long capacity() const;
    int input_width() const;
    mlora_ctx* context() const;
    long launches() const;  // kernels launched through the context so far

    /// Segment layout of the next fused batch (J + 1 offsets; stream-ordered).
    void set_layout(const std::vector<long>& seg);

    struct StepResult {
        double device_ms = 0.0;
        std::vector<float> loss;  // per job; 0 for jobs not in the batch
    };
    /// One fused iteration on device bf16 rows x input_width(): fwd, loss,
    /// guard, bwd, AdamW (jobs with active[j] == false untouched).
    StepResult step(const void* x_device, const std::vector<bool>& active);

    struct Impl;

private:
    std::unique_ptr<Impl> impl_;
};

enum class Strategy { Fifo, Priority, MinPad };

/// A job as the executor runs it: the reference's JobSpec (id, priority,
/// submit_time, dataset item lengths, batch_size, lora_rank, true_iterations)
/// plus its LoRA scale and learning rate.
struct ExecutorJob {
    JobSpec spec;
    float scale = 2.0f;
    float lr = 1e-4f;
};

/// sim.hpp TraceEvent{IterationDone}, with the measured duration and losses.
struct IterationDone {
    double time = 0.0;        // executor clock: sum of measured iteration times (s)
    double duration_s = 0.0;  // measured device time of this iteration
    long total_tokens = 0;    // ξ   (reference accounting, fused_shape)
    long padding_tokens = 0;  // ξ_p
    long effective_tokens = 0;
    long rows = 0;            // rows the kernels processed (packed: = effective)
    int jobs_in_batch = 0;
    std::vector<std::string> routing;       // job ids, selection (urgency) order
    std::map<std::string, float> losses;    // per job in the batch
};

/// (3) The real executor behind the fused iteration (see header comment).
class FusedIterationExecutor {
public:
    FusedIterationExecutor(int device, std::vector<Projection> shapes, std::vector<ExecutorJob> jobs,
                           int max_concurrent, Strategy strategy, bool padded, std::uint64_t seed);
    ~FusedIterationExecutor();
    FusedIterationExecutor(const FusedIterationExecutor&) = delete;
    FusedIterationExecutor& operator=(const FusedIterationExecutor&) = delete;

    /// One fused iteration; nullopt when every job has finished.
    std::optional<IterationDone> step();
    /// Iterate until every job finished (or max_iterations > 0 reached).
    std::vector<IterationDone> run(int max_iterations = -1);

    const std::vector<JobState>& jobs() const;
    double clock() const;
    FusedLayer& layer();

    struct Impl;

private:
    std::unique_ptr<Impl> impl_;
};

/// sim.hpp:15-19, field for field.
struct IterationTimeModel {
    double base = 0.0;
    double per_token = 0.001;
    double per_launch = 0.0;
};

/// (4) Least squares duration ≈ base + per_token · ξ over measured iterations
/// (per_launch = 0: the fused step's launch count does not depend on the job
/// count).  ConfigError-free: with fewer than two distinct ξ, per_token = 0.
IterationTimeModel fit_iteration_time(const std::vector<IterationDone>& events);

}  // namespace fusim::b200
