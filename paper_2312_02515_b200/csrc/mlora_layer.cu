// mlora_layer.cu — the one-call fused layer step (include/mlora.h, "one fused
// layer step"): the trainer hook that the reference simulator's fused iteration
// (/root/reference/proj/src/sim.cpp:163-191) charges analytically.  Host
// orchestration only — every kernel is launched through the C ABI entry points
// of mlora_capi.cu — plus the device-memory helpers and the deterministic
// uniform fill used to build identical synthetic weights / data from any host
// language.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/mlora.h"

namespace mlora_internal {
mlora_status set_error(mlora_ctx* ctx, mlora_status st, const std::string& msg);  // mlora_capi.cu
int ctx_device(const mlora_ctx* ctx);
}  // namespace mlora_internal
void mlora_count_free_launch();  // mlora_decoder.cu

namespace {

using mlora_internal::set_error;

constexpr int kMaxLayerProj = 16;

struct DevGuard {
    int prev = -1;
    explicit DevGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DevGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

// splitmix64 of (seed, index): a counter-based generator, so the value of
// element i depends on nothing but (seed, i).
__device__ __forceinline__ float uniform01(unsigned long long seed, unsigned long long i) {
    unsigned long long z = seed * 0x9E3779B97F4A7C15ull + i + 0x632BE59BD9B4E019ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    return static_cast<float>(z >> 40) * (1.0f / 16777216.0f);  // 24 random bits -> [0, 1)
}

__global__ void fill_uniform_kernel(void* __restrict__ dst, long long n, int dtype, unsigned long long seed,
                                    float lo, float span) {
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const float v = lo + span * uniform01(seed, static_cast<unsigned long long>(i));
        if (dtype == 0)
            static_cast<float*>(dst)[i] = v;
        else
            static_cast<__nv_bfloat16*>(dst)[i] = __float2bfloat16_rn(v);
    }
}

}  // namespace

struct mlora_layer {
    mlora_ctx* ctx = nullptr;
    mlora_plan* plan = nullptr;
    int n = 0;
    long long capacity = 0;
    std::vector<mlora_layer_proj> proj;
    std::vector<std::vector<int>> waves;  // forward dependency waves (projection indices)
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
};

namespace mlora {
mlora_status layer_loss_guard(mlora_ctx* ctx, const mlora_plan* plan, const float* const* row_sq, const int32_t* d,
                              int32_t num_rowsq, float* loss, void* const* tensors, const int32_t* cols,
                              int32_t num_tensors, cudaStream_t s);  // mlora_capi.cu
}

namespace {

mlora_status forward_backward(mlora_layer* L, void* x, float* loss, cudaStream_t s) {
    mlora_ctx* ctx = L->ctx;
    const mlora_plan* plan = L->plan;
    const long long rows = mlora_plan_rows(plan);
    if (rows < 1 || rows > L->capacity)
        return set_error(ctx, MLORA_USAGE, "layer step: plan rows " + std::to_string(rows) + " outside [1, capacity " +
                                               std::to_string(L->capacity) + "]");
    if (!x || !loss) return set_error(ctx, MLORA_USAGE, "layer step: null x or loss");
    const int n = L->n;
    const int R = mlora_plan_rank_padded(plan);
    std::vector<const void*> in(n, nullptr);
    mlora_status st;
    // ---- forward, in dependency waves
    for (const auto& wave : L->waves) {
        const int nw = static_cast<int>(wave.size());
        std::vector<int32_t> width(nw);
        std::vector<const void*> ins(nw), ad(nw);
        std::vector<void*> outs(nw);
        for (int w = 0; w < nw; ++w) {
            const int i = wave[w];
            const mlora_layer_proj& p = L->proj[i];
            if (p.src < 0) {
                in[i] = x;
            } else if (p.in_scratch) {  // column slice of a wider source -> contiguous copy
                const mlora_layer_proj& q = L->proj[p.src];
                if (cudaMemcpy2DAsync(p.in_scratch, static_cast<size_t>(p.k) * 2,
                                      static_cast<const char*>(q.Y) + static_cast<size_t>(p.src_col0) * 2,
                                      static_cast<size_t>(q.d) * 2, static_cast<size_t>(p.k) * 2, rows,
                                      cudaMemcpyDeviceToDevice, s) != cudaSuccess)
                    return set_error(ctx, MLORA_CUDA, "layer step: input slice copy failed");
                in[i] = p.in_scratch;
            } else {
                in[i] = L->proj[p.src].Y;
            }
            width[w] = p.k;
            ins[w] = in[i];
            ad[w] = p.A_bf16;
            outs[w] = p.H;
        }
        if ((st = mlora_down_group(ctx, plan, nw, 0, width.data(), ins.data(), ad.data(), outs.data(), s)) != MLORA_OK)
            return st;
        for (int i : wave) {
            const mlora_layer_proj& p = L->proj[i];
            if ((st = mlora_base_fwd(ctx, plan, p.d, p.k, in[i], p.W0, p.H, p.B_bf16, p.Y, p.row_sq, s)) != MLORA_OK)
                return st;
        }
    }
    // ---- per-job loss from the forward epilogues' row sums (no re-read of Y)
    std::vector<const float*> rsq(n);
    std::vector<int32_t> dd(n), kk(n);
    for (int i = 0; i < n; ++i) {
        rsq[i] = L->proj[i].row_sq;
        dd[i] = L->proj[i].d;
        kk[i] = L->proj[i].k;
    }
    // ---- non-finite guard over every tensor the backward reads (deduplicated), fused
    // with the per-job loss reduction: a job whose loss is not finite has its rows of
    // these tensors zeroed before any backward kernel reads them
    std::vector<void*> gt;
    std::vector<int32_t> gc;
    auto guard = [&](const void* t, int cols) {
        if (std::find(gt.begin(), gt.end(), t) != gt.end()) return;
        gt.push_back(const_cast<void*>(t));
        gc.push_back(cols);
    };
    for (int i = 0; i < n; ++i) {
        guard(L->proj[i].Y, L->proj[i].d);
        guard(L->proj[i].H, R);
        guard(in[i], L->proj[i].k);
    }
    const int nt0 = static_cast<int>(std::min<size_t>(32, gt.size()));
    if ((st = mlora::layer_loss_guard(ctx, plan, rsq.data(), dd.data(), n, loss, gt.data(), gc.data(), nt0, s)) !=
        MLORA_OK)
        return st;
    for (size_t t0 = 32; t0 < gt.size(); t0 += 32) {
        const int nt = static_cast<int>(std::min<size_t>(32, gt.size() - t0));
        if ((st = mlora_zero_nonfinite_rows(ctx, plan, loss, gt.data() + t0, gc.data() + t0, nt, s)) != MLORA_OK)
            return st;
    }
    // ---- backward: dL/dY_p = Y_p
    std::vector<const void*> ys(n), bs(n), hs(n), gs(n);
    std::vector<void*> gout(n);
    std::vector<float*> das(n), dbs(n);
    for (int i = 0; i < n; ++i) {
        const mlora_layer_proj& p = L->proj[i];
        ys[i] = p.Y;
        bs[i] = p.B_bf16;
        hs[i] = p.H;
        gs[i] = p.G;
        gout[i] = p.G;
        das[i] = p.dA;
        dbs[i] = p.dB;
    }
    if ((st = mlora_down_group(ctx, plan, n, 1, dd.data(), ys.data(), bs.data(), gout.data(), s)) != MLORA_OK)
        return st;
    for (int i = n - 1; i >= 0; --i) {
        const mlora_layer_proj& p = L->proj[i];
        if (!p.dX) continue;
        if ((st = mlora_base_dx(ctx, plan, p.d, p.k, p.Y, p.W0, p.G, p.A_bf16, p.dX, s)) != MLORA_OK) return st;
    }
    return mlora_grad_group(ctx, plan, n, dd.data(), kk.data(), in.data(), ys.data(), hs.data(), gs.data(),
                            das.data(), dbs.data(), s);
}

mlora_status adam(mlora_layer* L, const float* lr, const int32_t* step, const mlora_adam_hparams* hp,
                  const float* loss, cudaStream_t s) {
    if (!lr || !step) return set_error(L->ctx, MLORA_USAGE, "layer step: null lr or step");
    const mlora_adam_hparams h = hp ? *hp : mlora_adam_hparams{0.9f, 0.999f, 1e-8f, 0.0f};
    const int R = mlora_plan_rank_padded(L->plan);
    std::vector<mlora_adam_group> g;
    g.reserve(2 * L->n);
    for (const mlora_layer_proj& p : L->proj) {
        g.push_back(mlora_adam_group{p.A, p.dA, p.mA, p.vA, p.A_bf16, R, p.k, 0, 0});
        g.push_back(mlora_adam_group{p.B, p.dB, p.mB, p.vB, p.B_bf16, p.d, R, 1, 0});
    }
    return mlora_adam_step_ex(L->ctx, L->plan, g.data(), static_cast<int32_t>(g.size()), lr, step, h.beta1, h.beta2,
                              h.eps, h.weight_decay, loss, s);
}

}  // namespace

extern "C" {

mlora_status mlora_layer_create(mlora_ctx* ctx, mlora_plan* plan, int32_t n, const mlora_layer_proj* proj,
                                int64_t capacity, mlora_layer** out) {
    if (!ctx || !plan || !proj || !out) return set_error(ctx, MLORA_USAGE, "layer: null argument");
    *out = nullptr;
    if (n < 1 || n > kMaxLayerProj)
        return set_error(ctx, MLORA_USAGE, "layer: 1 to " + std::to_string(kMaxLayerProj) + " projections");
    if (capacity < 1) return set_error(ctx, MLORA_USAGE, "layer: capacity must be >= 1");
    for (int i = 0; i < n; ++i) {
        const mlora_layer_proj& p = proj[i];
        if (p.d <= 0 || p.k <= 0 || p.d % 8 || p.k % 8)
            return set_error(ctx, MLORA_SHAPE, "layer: projection " + std::to_string(i) +
                                                   ": d and k must be positive multiples of 8");
        if (!p.W0 || !p.A || !p.B || !p.mA || !p.vA || !p.mB || !p.vB || !p.A_bf16 || !p.B_bf16 || !p.dA || !p.dB ||
            !p.Y || !p.H || !p.G || !p.row_sq)
            return set_error(ctx, MLORA_USAGE, "layer: projection " + std::to_string(i) + ": null tensor");
        if (p.src >= n || p.src == i || p.src < -1)
            return set_error(ctx, MLORA_USAGE, "layer: projection " + std::to_string(i) + ": bad source index");
        if (p.src >= 0) {
            const mlora_layer_proj& q = proj[p.src];
            if (p.src_col0 < 0 || p.src_col0 % 8 || p.src_col0 + p.k > q.d)
                return set_error(ctx, MLORA_SHAPE, "layer: projection " + std::to_string(i) +
                                                       ": input slice outside its source");
            if ((p.src_col0 != 0 || q.d != p.k) && !p.in_scratch)
                return set_error(ctx, MLORA_USAGE, "layer: projection " + std::to_string(i) +
                                                       ": a column-slice input needs in_scratch");
        }
    }
    // dependency waves (Kahn): wave w = projections whose source is in an earlier wave
    std::vector<int> level(n, -1);
    std::vector<std::vector<int>> waves;
    int placed = 0;
    while (placed < n) {
        std::vector<int> wave;
        for (int i = 0; i < n; ++i)
            if (level[i] < 0 && (proj[i].src < 0 || level[proj[i].src] >= 0)) wave.push_back(i);
        if (wave.empty()) return set_error(ctx, MLORA_USAGE, "layer: projection inputs form a cycle");
        for (int i : wave) level[i] = static_cast<int>(waves.size());
        placed += static_cast<int>(wave.size());
        waves.push_back(std::move(wave));
    }
    auto* L = new mlora_layer();
    L->ctx = ctx;
    L->plan = plan;
    L->n = n;
    L->capacity = capacity;
    L->proj.assign(proj, proj + n);
    L->waves = std::move(waves);
    *out = L;
    return MLORA_OK;
}

mlora_status mlora_layer_destroy(mlora_layer* layer) {
    if (!layer) return MLORA_OK;
    {
        DevGuard g(mlora_internal::ctx_device(layer->ctx));
        if (layer->ev0) cudaEventDestroy(layer->ev0);
        if (layer->ev1) cudaEventDestroy(layer->ev1);
    }
    delete layer;
    return MLORA_OK;
}

mlora_status mlora_layer_forward_backward(mlora_layer* layer, void* x, float* loss, void* stream) {
    if (!layer) return set_error(nullptr, MLORA_USAGE, "null layer");
    DevGuard g(mlora_internal::ctx_device(layer->ctx));
    return forward_backward(layer, x, loss, static_cast<cudaStream_t>(stream));
}

mlora_status mlora_layer_step(mlora_layer* layer, void* x, const float* lr, const int32_t* step,
                              const mlora_adam_hparams* hp, float* loss, void* stream) {
    if (!layer) return set_error(nullptr, MLORA_USAGE, "null layer");
    DevGuard g(mlora_internal::ctx_device(layer->ctx));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    mlora_status st = forward_backward(layer, x, loss, s);
    if (st != MLORA_OK) return st;
    return adam(layer, lr, step, hp, loss, s);
}

mlora_status mlora_layer_step_timed(mlora_layer* layer, void* x, const float* lr, const int32_t* step,
                                    const mlora_adam_hparams* hp, float* loss, float* loss_host,
                                    double* device_ms, void* stream) {
    if (!layer || !loss_host || !device_ms) return set_error(layer ? layer->ctx : nullptr, MLORA_USAGE,
                                                             "layer step: null argument");
    mlora_ctx* ctx = layer->ctx;
    DevGuard g(mlora_internal::ctx_device(ctx));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (!layer->ev0 && (cudaEventCreate(&layer->ev0) != cudaSuccess || cudaEventCreate(&layer->ev1) != cudaSuccess))
        return set_error(ctx, MLORA_CUDA, "layer step: cudaEventCreate failed");
    if (cudaEventRecord(layer->ev0, s) != cudaSuccess) return set_error(ctx, MLORA_CUDA, "cudaEventRecord failed");
    mlora_status st = forward_backward(layer, x, loss, s);
    if (st == MLORA_OK) st = adam(layer, lr, step, hp, loss, s);
    if (st != MLORA_OK) return st;
    if (cudaEventRecord(layer->ev1, s) != cudaSuccess) return set_error(ctx, MLORA_CUDA, "cudaEventRecord failed");
    const int32_t jobs = mlora_plan_num_jobs(layer->plan);
    if (cudaMemcpyAsync(loss_host, loss, sizeof(float) * jobs, cudaMemcpyDeviceToHost, s) != cudaSuccess)
        return set_error(ctx, MLORA_CUDA, "layer step: loss copy failed");
    if (cudaEventSynchronize(layer->ev1) != cudaSuccess || cudaStreamSynchronize(s) != cudaSuccess)
        return set_error(ctx, MLORA_CUDA, std::string("layer step: ") + cudaGetErrorString(cudaGetLastError()));
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, layer->ev0, layer->ev1) != cudaSuccess)
        return set_error(ctx, MLORA_CUDA, "cudaEventElapsedTime failed");
    *device_ms = ms;
    return MLORA_OK;
}

// ---------------------------------------------------------------- memory helpers
mlora_status mlora_malloc(mlora_ctx* ctx, size_t bytes, void** out) {
    if (!ctx || !out) return set_error(ctx, MLORA_USAGE, "malloc: null argument");
    DevGuard g(mlora_internal::ctx_device(ctx));
    *out = nullptr;
    if (bytes == 0) return MLORA_OK;
    const cudaError_t e = cudaMalloc(out, bytes);
    if (e != cudaSuccess) return set_error(ctx, MLORA_CUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    return MLORA_OK;
}

mlora_status mlora_free(mlora_ctx* ctx, void* ptr) {
    if (!ctx) return set_error(nullptr, MLORA_USAGE, "free: null context");
    if (!ptr) return MLORA_OK;
    DevGuard g(mlora_internal::ctx_device(ctx));
    const cudaError_t e = cudaFree(ptr);
    if (e != cudaSuccess) return set_error(ctx, MLORA_CUDA, std::string("cudaFree: ") + cudaGetErrorString(e));
    return MLORA_OK;
}

mlora_status mlora_memcpy(mlora_ctx* ctx, void* dst, const void* src, size_t bytes, int32_t kind, void* stream) {
    if (!ctx || (bytes && (!dst || !src))) return set_error(ctx, MLORA_USAGE, "memcpy: null argument");
    if (kind < 0 || kind > 2) return set_error(ctx, MLORA_USAGE, "memcpy: bad kind");
    if (!bytes) return MLORA_OK;
    DevGuard g(mlora_internal::ctx_device(ctx));
    const cudaMemcpyKind k[3] = {cudaMemcpyHostToDevice, cudaMemcpyDeviceToHost, cudaMemcpyDeviceToDevice};
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaMemcpyAsync(dst, src, bytes, k[kind], s);
    if (e == cudaSuccess && kind != 2) e = cudaStreamSynchronize(s);  // host buffers may be pageable
    if (e != cudaSuccess) return set_error(ctx, MLORA_CUDA, std::string("cudaMemcpy: ") + cudaGetErrorString(e));
    return MLORA_OK;
}

mlora_status mlora_memset(mlora_ctx* ctx, void* dst, int32_t value, size_t bytes, void* stream) {
    if (!ctx || (bytes && !dst)) return set_error(ctx, MLORA_USAGE, "memset: null argument");
    if (!bytes) return MLORA_OK;
    DevGuard g(mlora_internal::ctx_device(ctx));
    const cudaError_t e = cudaMemsetAsync(dst, value, bytes, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return set_error(ctx, MLORA_CUDA, std::string("cudaMemset: ") + cudaGetErrorString(e));
    return MLORA_OK;
}

mlora_status mlora_stream_sync(mlora_ctx* ctx, void* stream) {
    if (!ctx) return set_error(nullptr, MLORA_USAGE, "sync: null context");
    DevGuard g(mlora_internal::ctx_device(ctx));
    const cudaError_t e = cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return set_error(ctx, MLORA_CUDA, std::string("stream sync: ") + cudaGetErrorString(e));
    return MLORA_OK;
}

mlora_status mlora_mem_info(mlora_ctx* ctx, size_t* free_bytes, size_t* total_bytes) {
    if (!ctx || !free_bytes || !total_bytes) return set_error(ctx, MLORA_USAGE, "mem_info: null argument");
    DevGuard g(mlora_internal::ctx_device(ctx));
    const cudaError_t e = cudaMemGetInfo(free_bytes, total_bytes);
    if (e != cudaSuccess) return set_error(ctx, MLORA_CUDA, std::string("cudaMemGetInfo: ") + cudaGetErrorString(e));
    return MLORA_OK;
}

mlora_status mlora_fill_uniform(void* dst, int64_t n, int32_t dtype, uint64_t seed, float lo, float hi,
                                void* stream) {
    if (n < 0 || (n > 0 && !dst)) return set_error(nullptr, MLORA_USAGE, "fill: null argument");
    if (dtype != 0 && dtype != 1) return set_error(nullptr, MLORA_USAGE, "fill: dtype must be 0 (fp32) or 1 (bf16)");
    if (!(lo <= hi)) return set_error(nullptr, MLORA_USAGE, "fill: need lo <= hi");
    if (n == 0) return MLORA_OK;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long long blocks = std::min<long long>((n + 255) / 256, 8LL * sms);
    fill_uniform_kernel<<<static_cast<unsigned>(blocks), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        dst, n, dtype, seed, lo, hi - lo);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(nullptr, MLORA_CUDA, std::string("fill: ") + cudaGetErrorString(e));
    mlora_count_free_launch();
    return MLORA_OK;
}

}  // extern "C"
