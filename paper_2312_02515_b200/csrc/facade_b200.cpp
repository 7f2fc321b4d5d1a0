// facade_b200.cpp — fusim::b200 (include/fusim/b200.hpp): the bf16 tcgen05
// fused_forward behind the reference signature, the one-call fused layer step,
// and the executor behind the simulator's fused iteration
// (/root/reference/proj/src/sim.cpp:163-191).  Everything device-side goes
// through the C ABI (include/mlora.h); this file links no CUDA runtime.
#include "fusim/b200.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <set>

#include "mlora.h"

namespace fusim {
namespace detail {
mlora_ctx* facade_ctx();  // facade_lora.cpp
}  // namespace detail

namespace b200 {
namespace {

[[noreturn]] void raise(mlora_status st, const std::string& what, const mlora_ctx* ctx) {
    const std::string msg = what + ": " + mlora_last_error(ctx);
    switch (st) {
        case MLORA_USAGE: throw UsageError(msg);
        case MLORA_SHAPE: throw ShapeError(msg);
        case MLORA_ROUTING: throw RoutingError(msg);
        case MLORA_NUMERIC: throw NumericError(msg);
        case MLORA_STATE: throw StateError(msg);
        default: throw DeviceError(msg);
    }
}

void ok(mlora_status st, const char* what, const mlora_ctx* ctx) {
    if (st != MLORA_OK) raise(st, what, ctx);
}

// float -> bf16, round to nearest even (NaN stays NaN)
std::uint16_t to_bf16(float f) {
    std::uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return static_cast<std::uint16_t>((u >> 16) | 0x40);
    u += 0x7fffu + ((u >> 16) & 1u);
    return static_cast<std::uint16_t>(u >> 16);
}

float from_bf16(std::uint16_t h) {
    const std::uint32_t u = static_cast<std::uint32_t>(h) << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

long roundup8(long v) { return (v + 7) / 8 * 8; }

// Device allocations of one owner, freed together (RAII).
class Arena {
public:
    explicit Arena(mlora_ctx* ctx) : ctx_(ctx) {}
    ~Arena() {
        for (void* p : ptrs_) mlora_free(ctx_, p);
    }
    Arena(const Arena&) = delete;
    Arena& operator=(const Arena&) = delete;
    void* alloc(std::size_t bytes, bool zero = false) {
        void* p = nullptr;
        ok(mlora_malloc(ctx_, bytes, &p), "mlora_malloc", ctx_);
        ptrs_.push_back(p);
        if (zero) ok(mlora_memset(ctx_, p, 0, bytes, nullptr), "mlora_memset", ctx_);
        return p;
    }
    template <typename T>
    T* upload(const std::vector<T>& host) {
        void* p = alloc(host.size() * sizeof(T));
        ok(mlora_memcpy(ctx_, p, host.data(), host.size() * sizeof(T), 0, nullptr), "mlora_memcpy H2D", ctx_);
        return static_cast<T*>(p);
    }

private:
    mlora_ctx* ctx_;
    std::vector<void*> ptrs_;
};

void fill(void* dst, long n, int dtype, std::uint64_t seed, double half_width) {
    const float hw = static_cast<float>(half_width);
    ok(mlora_fill_uniform(dst, n, dtype, seed, -hw, hw, nullptr), "mlora_fill_uniform", nullptr);
}

}  // namespace

std::uint64_t mix_seed(std::initializer_list<std::int64_t> parts) {
    std::uint64_t h = 0xCBF29CE484222325ull;
    for (std::int64_t v : parts) h = (h ^ static_cast<std::uint64_t>(v)) * 0x100000001B3ull;
    return h;
}

// ------------------------------------------------------------------ (1) fused_forward_bf16
std::vector<Matrix> fused_forward_bf16(const Matrix& W0, const std::map<std::string, AdapterWeights>& adapters,
                                       const FusedBatch& fb) {
    // preconditions exactly as fusim::fused_forward (lora.cpp:163-167), before any device work
    if (W0.cols != fb.dim) throw ShapeError("fused_forward: W0 column dim does not match batch dim");
    for (const auto& job : fb.routing)
        if (adapters.find(job) == adapters.end()) throw RoutingError("fused_forward: no adapter for job " + job);
    const int d = W0.rows, k = W0.cols;
    for (const auto& job : fb.routing) adapters.at(job).validate(d, k);
    const long L = fb.max_len, S = fb.num_sequences;
    std::vector<Matrix> outs;
    outs.reserve(static_cast<std::size_t>(S));
    if (S * L == 0 || d == 0 || k == 0) {
        for (long s = 0; s < S; ++s) outs.emplace_back(static_cast<int>(L), d);
        return outs;
    }
    mlora_ctx* ctx = detail::facade_ctx();
    const long dp = roundup8(d), kp = roundup8(k);
    // one plan "job" per run of consecutive sequences routed to the same adapter
    // (the kernels need each adapter's rows contiguous); at most 128 per launch
    std::vector<std::pair<long, long>> runs;  // [s0, s1)
    for (long s0 = 0; s0 < S;) {
        long s1 = s0 + 1;
        while (s1 < S && fb.routing[s1] == fb.routing[s0]) ++s1;
        runs.emplace_back(s0, s1);
        s0 = s1;
    }
    Arena keep(ctx);
    std::vector<std::uint16_t> w16(static_cast<std::size_t>(dp * kp), 0);
    for (int i = 0; i < d; ++i)
        for (int c = 0; c < k; ++c) w16[i * kp + c] = to_bf16(static_cast<float>(W0.at(i, c)));
    const void* dW = keep.upload(w16);
    std::vector<std::uint16_t> yh;
    for (std::size_t r0 = 0; r0 < runs.size(); r0 += 128) {
        const std::size_t r1 = std::min(runs.size(), r0 + 128);
        const int J = static_cast<int>(r1 - r0);
        const long s_begin = runs[r0].first, s_end = runs[r1 - 1].second;
        const long rows = (s_end - s_begin) * L;
        Arena a(ctx);
        std::vector<std::int64_t> seg(J + 1, 0);
        std::vector<std::int32_t> ranks(J);
        std::vector<float> scales(J, 1.0f);  // the reference has no scale
        std::vector<const float*> Ap(J), Bp(J);
        for (int j = 0; j < J; ++j) {
            const auto& run = runs[r0 + j];
            seg[j + 1] = seg[j] + (run.second - run.first) * L;
            const AdapterWeights& ad = adapters.at(fb.routing[run.first]);
            ranks[j] = ad.rank;
            std::vector<float> A(static_cast<std::size_t>(ad.rank * kp), 0.f), B(static_cast<std::size_t>(dp * ad.rank), 0.f);
            for (int i = 0; i < ad.rank; ++i)
                for (int c = 0; c < k; ++c) A[i * kp + c] = static_cast<float>(ad.A.at(i, c));
            for (int i = 0; i < d; ++i)
                for (int c = 0; c < ad.rank; ++c) B[i * ad.rank + c] = static_cast<float>(ad.B.at(i, c));
            Ap[j] = a.upload(A);
            Bp[j] = a.upload(B);
        }
        mlora_plan* plan = nullptr;
        ok(mlora_plan_create(ctx, J, seg.data(), ranks.data(), scales.data(), nullptr, &plan), "mlora_plan_create",
           ctx);
        struct PlanGuard {
            mlora_plan* p;
            ~PlanGuard() { mlora_plan_destroy(p); }
        } pg{plan};
        const int R = mlora_plan_rank_padded(plan);
        void* A16 = a.alloc(static_cast<std::size_t>(R) * kp * 2);
        void* B16 = a.alloc(static_cast<std::size_t>(dp) * R * 2);
        ok(mlora_pack_adapters(ctx, plan, static_cast<int>(dp), static_cast<int>(kp), Ap.data(), Bp.data(), nullptr,
                               nullptr, A16, B16, nullptr),
           "mlora_pack_adapters", ctx);
        std::vector<std::uint16_t> x16(static_cast<std::size_t>(rows * kp), 0);
        for (long r = 0; r < rows; ++r) {
            const double* src = fb.data.data() + static_cast<std::size_t>((s_begin * L + r) * k);
            for (int c = 0; c < k; ++c) x16[r * kp + c] = to_bf16(static_cast<float>(src[c]));
        }
        const void* dX = a.upload(x16);
        void* dY = a.alloc(static_cast<std::size_t>(rows) * dp * 2);
        void* dH = a.alloc(static_cast<std::size_t>(rows) * R * 2);
        ok(mlora_linear_fwd(ctx, plan, static_cast<int>(dp), static_cast<int>(kp), dX, dW, A16, B16, dY, dH, nullptr),
           "mlora_linear_fwd", ctx);
        yh.assign(static_cast<std::size_t>(rows * dp), 0);
        ok(mlora_memcpy(ctx, yh.data(), dY, yh.size() * 2, 1, nullptr), "mlora_memcpy D2H", ctx);
        for (long s = s_begin; s < s_end; ++s) {
            Matrix o(static_cast<int>(L), d);
            for (long t = 0; t < L; ++t) {
                const bool real = fb.mask[static_cast<std::size_t>(s * L + t)] != 0;
                for (int c = 0; c < d; ++c)
                    o.at(static_cast<int>(t), c) =
                        real ? static_cast<double>(from_bf16(yh[((s - s_begin) * L + t) * dp + c])) : 0.0;
            }
            outs.push_back(std::move(o));
        }
    }
    return outs;
}

// ------------------------------------------------------------------ layer shapes
std::vector<Projection> llama_layer(int hidden, int ffn) {
    return {{"q", hidden, hidden, "x", 0},  {"k", hidden, hidden, "x", 0},  {"v", hidden, hidden, "x", 0},
            {"o", hidden, hidden, "v", 0},  {"gate", ffn, hidden, "x", 0},  {"up", ffn, hidden, "x", 0},
            {"down", hidden, ffn, "up", 0}};
}

// ------------------------------------------------------------------ (2) FusedLayer
struct FusedLayer::Impl {
    mlora_ctx* ctx = nullptr;
    mlora_plan* plan = nullptr;
    mlora_layer* layer = nullptr;
    std::unique_ptr<Arena> mem;
    std::vector<Projection> shapes;
    std::vector<TrainJob> jobs;
    long capacity = 0;
    int input_width = 0;
    std::vector<int> step_count;
    std::vector<float> lr;
    float* loss = nullptr;

    ~Impl() {
        if (layer) mlora_layer_destroy(layer);
        mem.reset();
        if (plan) mlora_plan_destroy(plan);
        if (ctx) mlora_ctx_destroy(ctx);
    }
};

FusedLayer::FusedLayer(int device, std::vector<Projection> shapes, std::vector<TrainJob> jobs, long capacity,
                       std::uint64_t seed)
    : impl_(std::make_unique<Impl>()) {
    Impl& m = *impl_;
    if (shapes.empty() || jobs.empty()) throw UsageError("FusedLayer: need at least one projection and one job");
    if (capacity < 1) throw UsageError("FusedLayer: capacity must be >= 1");
    ok(mlora_ctx_create(device, &m.ctx), "mlora_ctx_create", nullptr);
    m.mem = std::make_unique<Arena>(m.ctx);
    m.shapes = std::move(shapes);
    m.jobs = std::move(jobs);
    m.capacity = capacity;
    const int J = static_cast<int>(m.jobs.size());
    m.step_count.assign(J, 0);
    std::vector<std::int64_t> seg(J + 1, 0);
    seg[J] = capacity;  // placeholder layout; set_layout installs the real one
    std::vector<std::int32_t> ranks(J);
    std::vector<float> scales(J);
    for (int j = 0; j < J; ++j) {
        ranks[j] = m.jobs[j].rank;
        scales[j] = m.jobs[j].scale;
        m.lr.push_back(m.jobs[j].lr);
    }
    ok(mlora_plan_create(m.ctx, J, seg.data(), ranks.data(), scales.data(), nullptr, &m.plan), "mlora_plan_create",
       m.ctx);
    const long R = mlora_plan_rank_padded(m.plan);
    const int n = static_cast<int>(m.shapes.size());
    std::vector<mlora_layer_proj> desc(n);
    Arena tmp(m.ctx);
    for (int pi = 0; pi < n; ++pi) {
        const Projection& p = m.shapes[pi];
        const long d = p.d, k = p.k;
        mlora_layer_proj& q = desc[pi];
        std::memset(&q, 0, sizeof(q));
        q.d = p.d;
        q.k = p.k;
        q.src = -1;
        q.src_col0 = p.src_col0;
        if (p.src != "x") {
            auto it = std::find_if(m.shapes.begin(), m.shapes.end(), [&](const Projection& s) { return s.name == p.src; });
            if (it == m.shapes.end()) throw UsageError("FusedLayer: unknown source " + p.src + " of " + p.name);
            q.src = static_cast<int>(it - m.shapes.begin());
            if (it->d != p.k || p.src_col0 != 0)
                q.in_scratch = m.mem->alloc(static_cast<std::size_t>(capacity) * k * 2);
        } else if (m.input_width == 0) {
            m.input_width = p.k;
        }
        // the synthetic initialisation of paper_2312_02515_b200/layer.py, tensor for tensor
        void* W0 = m.mem->alloc(static_cast<std::size_t>(d) * k * 2);
        fill(W0, d * k, 1, mix_seed({static_cast<std::int64_t>(seed), 0, pi}), std::pow(static_cast<double>(k), -0.5));
        q.W0 = W0;
        std::vector<const float*> Ap(J), Bp(J);
        for (int j = 0; j < J; ++j) {
            const long r = m.jobs[j].rank;
            float* A = static_cast<float*>(tmp.alloc(static_cast<std::size_t>(r) * k * 4));
            float* B = static_cast<float*>(tmp.alloc(static_cast<std::size_t>(d) * r * 4));
            fill(A, r * k, 0, mix_seed({static_cast<std::int64_t>(seed), 1, pi, j}), std::pow(static_cast<double>(k), -0.5));
            fill(B, d * r, 0, mix_seed({static_cast<std::int64_t>(seed), 2, pi, j}), std::pow(static_cast<double>(r), -0.5));
            Ap[j] = A;
            Bp[j] = B;
        }
        q.A = static_cast<float*>(m.mem->alloc(static_cast<std::size_t>(R) * k * 4));
        q.B = static_cast<float*>(m.mem->alloc(static_cast<std::size_t>(d) * R * 4));
        q.A_bf16 = m.mem->alloc(static_cast<std::size_t>(R) * k * 2);
        q.B_bf16 = m.mem->alloc(static_cast<std::size_t>(d) * R * 2);
        ok(mlora_pack_adapters(m.ctx, m.plan, p.d, p.k, Ap.data(), Bp.data(), q.A, q.B, q.A_bf16, q.B_bf16, nullptr),
           "mlora_pack_adapters", m.ctx);
        q.mA = static_cast<float*>(m.mem->alloc(static_cast<std::size_t>(R) * k * 4, true));
        q.vA = static_cast<float*>(m.mem->alloc(static_cast<std::size_t>(R) * k * 4, true));
        q.mB = static_cast<float*>(m.mem->alloc(static_cast<std::size_t>(d) * R * 4, true));
        q.vB = static_cast<float*>(m.mem->alloc(static_cast<std::size_t>(d) * R * 4, true));
        q.dA = static_cast<float*>(m.mem->alloc(static_cast<std::size_t>(R) * k * 4, true));
        q.dB = static_cast<float*>(m.mem->alloc(static_cast<std::size_t>(d) * R * 4, true));
        q.Y = m.mem->alloc(static_cast<std::size_t>(capacity) * d * 2);
        q.H = m.mem->alloc(static_cast<std::size_t>(capacity) * R * 2);
        q.G = m.mem->alloc(static_cast<std::size_t>(capacity) * R * 2);
        q.dX = m.mem->alloc(static_cast<std::size_t>(capacity) * k * 2);
        q.row_sq = static_cast<float*>(
            m.mem->alloc(static_cast<std::size_t>(mlora_rowsq_blocks(p.d)) * capacity * 4));
    }
    ok(mlora_stream_sync(m.ctx, nullptr), "initialisation", m.ctx);  // temporaries freed at scope exit
    if (m.input_width == 0) throw UsageError("FusedLayer: no projection reads the layer input x");
    m.loss = static_cast<float*>(m.mem->alloc(static_cast<std::size_t>(J) * 4, true));
    ok(mlora_layer_create(m.ctx, m.plan, n, desc.data(), capacity, &m.layer), "mlora_layer_create", m.ctx);
}

FusedLayer::~FusedLayer() = default;

int FusedLayer::num_jobs() const { return static_cast<int>(impl_->jobs.size()); }
long FusedLayer::capacity() const { return impl_->capacity; }
int FusedLayer::input_width() const { return impl_->input_width; }
mlora_ctx* FusedLayer::context() const { return impl_->ctx; }
long FusedLayer::launches() const { return static_cast<long>(mlora_ctx_launch_count(impl_->ctx)); }

void FusedLayer::set_layout(const std::vector<long>& seg) {
    if (seg.size() != impl_->jobs.size() + 1) throw UsageError("set_layout: need num_jobs + 1 offsets");
    if (seg.back() < 1 || seg.back() > impl_->capacity) throw UsageError("set_layout: rows outside [1, capacity]");
    std::vector<std::int64_t> s(seg.begin(), seg.end());
    ok(mlora_plan_update(impl_->plan, s.data(), nullptr), "mlora_plan_update", impl_->ctx);
}

FusedLayer::StepResult FusedLayer::step(const void* x_device, const std::vector<bool>& active) {
    Impl& m = *impl_;
    const int J = static_cast<int>(m.jobs.size());
    if (static_cast<int>(active.size()) != J) throw UsageError("step: need one active flag per job");
    std::vector<std::int32_t> steps(J);
    for (int j = 0; j < J; ++j) {
        if (active[j]) ++m.step_count[j];
        steps[j] = active[j] ? m.step_count[j] : 0;
    }
    StepResult r;
    r.loss.assign(J, 0.f);
    ok(mlora_layer_step_timed(m.layer, const_cast<void*>(x_device), m.lr.data(), steps.data(), nullptr, m.loss,
                              r.loss.data(), &r.device_ms, nullptr),
       "mlora_layer_step", m.ctx);
    return r;
}

// ------------------------------------------------------------------ (3) FusedIterationExecutor
struct FusedIterationExecutor::Impl {
    std::unique_ptr<FusedLayer> layer;
    std::vector<JobState> states;
    std::vector<ExecutorJob> cfg;
    int M = 1;
    Strategy strategy = Strategy::MinPad;
    bool padded = false;
    double clock = 0.0;
    int k_in = 0;
    std::unique_ptr<Arena> mem;
    std::vector<std::vector<void*>> data;  // per job, per dataset item: bf16 [len, k_in]
    void* x = nullptr;
    std::uint8_t* mask = nullptr;
};

FusedIterationExecutor::FusedIterationExecutor(int device, std::vector<Projection> shapes, std::vector<ExecutorJob> jobs,
                                               int max_concurrent, Strategy strategy, bool padded, std::uint64_t seed)
    : impl_(std::make_unique<Impl>()) {
    Impl& m = *impl_;
    if (jobs.empty()) throw UsageError("executor: no jobs");
    if (max_concurrent < 1) throw UsageError("executor: max_concurrent must be >= 1");
    int max_len = 0, max_bs = 0;
    std::vector<TrainJob> train;
    for (const auto& j : jobs) {
        j.spec.validate();
        max_len = std::max(max_len, j.spec.dataset.max_length());
        max_bs = std::max(max_bs, j.spec.batch_size);
        train.push_back(TrainJob{j.spec.lora_rank, j.scale, j.lr});
    }
    const long capacity = static_cast<long>(max_concurrent) * max_bs * max_len;
    m.layer = std::make_unique<FusedLayer>(device, std::move(shapes), std::move(train), capacity, seed);
    m.cfg = std::move(jobs);
    for (const auto& j : m.cfg) m.states.emplace_back(j.spec);
    m.M = max_concurrent;
    m.strategy = strategy;
    m.padded = padded;
    m.k_in = m.layer->input_width();
    mlora_ctx* ctx = m.layer->context();
    m.mem = std::make_unique<Arena>(ctx);
    // each job's dataset, resident in HBM (executor.py: fill seed mix_seed(seed, 3, i, item))
    for (std::size_t i = 0; i < m.cfg.size(); ++i) {
        std::vector<void*> items;
        const auto& ds = m.cfg[i].spec.dataset.items;
        for (std::size_t it = 0; it < ds.size(); ++it) {
            const long n = static_cast<long>(ds[it].length) * m.k_in;
            void* p = m.mem->alloc(static_cast<std::size_t>(n) * 2);
            fill(p, n, 1, mix_seed({static_cast<std::int64_t>(seed), 3, static_cast<std::int64_t>(i),
                                    static_cast<std::int64_t>(it)}),
                 1.0);
            items.push_back(p);
        }
        m.data.push_back(std::move(items));
    }
    m.x = m.mem->alloc(static_cast<std::size_t>(capacity) * m.k_in * 2);
    m.mask = static_cast<std::uint8_t*>(m.mem->alloc(static_cast<std::size_t>(capacity)));
    ok(mlora_stream_sync(ctx, nullptr), "executor initialisation", ctx);
}

FusedIterationExecutor::~FusedIterationExecutor() = default;

const std::vector<JobState>& FusedIterationExecutor::jobs() const { return impl_->states; }
double FusedIterationExecutor::clock() const { return impl_->clock; }
FusedLayer& FusedIterationExecutor::layer() { return *impl_->layer; }

std::optional<IterationDone> FusedIterationExecutor::step() {
    Impl& m = *impl_;
    std::vector<int> live;
    for (int i = 0; i < static_cast<int>(m.states.size()); ++i)
        if (!m.states[i].finished()) live.push_back(i);
    if (live.empty()) return std::nullopt;
    // the scheduler's view: each live job's next candidate batch (workload.cpp:50-60)
    std::vector<BatchCandidate> cands;
    for (std::size_t pos = 0; pos < live.size(); ++pos) {
        const JobState& js = m.states[live[pos]];
        BatchCandidate c;
        c.job_id = js.spec.id;
        for (const DataItem& item : js.next_candidate_batch()) c.item_lengths.push_back(item.length);
        c.priority = js.spec.priority;
        c.submit_time = js.spec.submit_time;
        cands.push_back(std::move(c));
    }
    const SelectionResult sel = m.strategy == Strategy::Fifo       ? select_fifo(cands, m.M)
                                : m.strategy == Strategy::Priority ? select_priority(cands, m.M)
                                                                   : select_minpad(cands, m.M);
    std::vector<int> chosen;  // job indices, urgency (routing) order
    for (const auto& id : sel.chosen)
        for (int i : live)
            if (m.states[i].spec.id == id) chosen.push_back(i);
    std::vector<int> in_batch = chosen;  // row order: job-index order (each job's rows contiguous)
    std::sort(in_batch.begin(), in_batch.end());
    std::vector<std::vector<int>> lengths;
    for (int j : in_batch) {
        std::vector<int> ls;
        for (const DataItem& item : m.states[j].next_candidate_batch()) ls.push_back(item.length);
        lengths.push_back(std::move(ls));
    }
    const FusedShape shape = fused_shape(lengths);  // ξ, ξ_p (lora.cpp:72-85)
    const int J = static_cast<int>(m.states.size());
    std::vector<long> seg(J + 1, 0);
    std::vector<bool> active(J, false);
    std::vector<const void*> srcs;
    std::vector<std::int32_t> lens;
    long effective = 0;
    {
        std::size_t b = 0;
        for (int j = 0; j < J; ++j) {
            seg[j + 1] = seg[j];
            if (b < in_batch.size() && in_batch[b] == j) {
                active[j] = true;
                const std::size_t n = m.cfg[j].spec.dataset.items.size();
                const std::size_t pos = m.states[j].cursor % n;
                for (std::size_t t = 0; t < lengths[b].size(); ++t) {
                    seg[j + 1] += m.padded ? shape.max_len : lengths[b][t];
                    srcs.push_back(m.data[j][pos + t]);
                    lens.push_back(lengths[b][t]);
                    effective += lengths[b][t];
                }
                ++b;
            }
        }
    }
    mlora_ctx* ctx = m.layer->context();
    // the measured iteration: layout upload + device fuse (lora.cpp:114-158) + the fused step
    ok(mlora_ctx_timer_start(ctx, nullptr), "timer", ctx);
    m.layer->set_layout(seg);
    ok(mlora_fuse_rows(ctx, static_cast<int>(srcs.size()), srcs.data(), nullptr, lens.data(), m.k_in,
                       m.padded ? 1 : 0, m.x, m.mask, nullptr, nullptr),
       "mlora_fuse_rows", ctx);
    const FusedLayer::StepResult r = m.layer->step(m.x, active);
    double ms = 0.0;
    ok(mlora_ctx_timer_stop(ctx, nullptr, &ms), "timer", ctx);
    IterationDone ev;
    ev.duration_s = ms / 1e3;
    m.clock += ev.duration_s;
    ev.time = m.clock;
    ev.total_tokens = shape.total_tokens;
    ev.padding_tokens = shape.padding_tokens;
    ev.effective_tokens = effective;
    ev.rows = seg[J];
    ev.jobs_in_batch = static_cast<int>(chosen.size());
    for (int j : chosen) {
        ev.routing.push_back(m.states[j].spec.id);
        ev.losses[m.states[j].spec.id] = r.loss[j];
    }
    // commit (workload.cpp:62-66) and the iteration bound (sim.cpp:193-208)
    for (std::size_t b = 0; b < in_batch.size(); ++b) {
        JobState& js = m.states[in_batch[b]];
        js.commit_batch(lengths[b].size());
        if (js.status == JobStatus::Pending) {
            js.status = JobStatus::Running;
            js.start_time = m.clock - ev.duration_s;
        }
        ++js.iterations_done;
        if (js.iterations_done >= js.spec.true_iterations) {
            js.status = JobStatus::Completed;
            js.finish_time = m.clock;
        }
    }
    return ev;
}

std::vector<IterationDone> FusedIterationExecutor::run(int max_iterations) {
    std::vector<IterationDone> out;
    while (max_iterations < 0 || static_cast<int>(out.size()) < max_iterations) {
        auto ev = step();
        if (!ev) break;
        out.push_back(std::move(*ev));
    }
    return out;
}

// ------------------------------------------------------------------ (4) calibration
IterationTimeModel fit_iteration_time(const std::vector<IterationDone>& events) {
    IterationTimeModel m;
    m.per_launch = 0.0;
    if (events.empty()) {
        m.base = 0.0;
        m.per_token = 0.0;
        return m;
    }
    double sx = 0, sy = 0, sxx = 0, sxy = 0;
    const double n = static_cast<double>(events.size());
    for (const auto& e : events) {
        const double x = static_cast<double>(e.total_tokens), y = e.duration_s;
        sx += x;
        sy += y;
        sxx += x * x;
        sxy += x * y;
    }
    const double var = sxx - sx * sx / n;
    if (var <= 0.0) {
        m.per_token = 0.0;
        m.base = sy / n;
        return m;
    }
    m.per_token = (sxy - sx * sy / n) / var;
    m.base = (sy - m.per_token * sx) / n;
    if (m.per_token < 0.0) {  // time does not grow with ξ here: a flat model
        m.per_token = 0.0;
        m.base = sy / n;
    } else if (m.base < 0.0) {  // through the origin
        m.base = 0.0;
        m.per_token = sxy / sxx;
    }
    return m;
}

}  // namespace b200
}  // namespace fusim
