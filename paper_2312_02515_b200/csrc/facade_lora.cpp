// facade_lora.cpp — fusim::lora API (include/fusim/lora.hpp) over the C ABI.
//
// Reference counterpart: /root/reference/proj/src/lora.cpp.  Preconditions are
// checked on the host exactly where the reference checks them and raise the
// same exception types; the arithmetic runs on the device (mlora_f64_gemm /
// mlora_f64_add) with the reference's per-element operation order.
#include "fusim/lora.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>

#include "mlora.h"

namespace fusim {
namespace {

void check_status(mlora_status st, const char* what) {
    switch (st) {
        case MLORA_OK: return;
        case MLORA_USAGE: throw UsageError(what);
        case MLORA_SHAPE: throw ShapeError(what);
        case MLORA_ROUTING: throw RoutingError(what);
        case MLORA_NUMERIC: throw NumericError(what);
        case MLORA_STATE: throw StateError(what);
        default: throw DeviceError(std::string(what) + ": " + mlora_last_error(nullptr));
    }
}

}  // namespace

namespace detail {
// The façade's device context (GPU 0, created on first use).  The façade links
// no CUDA runtime of its own: every allocation, copy and sync goes through
// libmlora.so (mlora_malloc / mlora_memcpy / mlora_stream_sync), so a process
// using both holds ONE runtime instance and one error state.
mlora_ctx* facade_ctx() {
    static std::once_flag once;
    static mlora_ctx* ctx = nullptr;
    static mlora_status st = MLORA_OK;
    std::call_once(once, [] { st = mlora_ctx_create(0, &ctx); });
    if (st != MLORA_OK || !ctx) throw DeviceError(std::string("mlora_ctx_create: ") + mlora_last_error(nullptr));
    return ctx;
}
}  // namespace detail

namespace {

// A device fp64 buffer (RAII); the façade's only allocation is per call.
class DevBuf {
public:
    explicit DevBuf(std::size_t n) : n_(n) {
        if (n_ == 0) return;
        if (mlora_malloc(detail::facade_ctx(), n_ * sizeof(double), &p_) != MLORA_OK)
            throw DeviceError(std::string("mlora_malloc: ") + mlora_last_error(detail::facade_ctx()));
    }
    DevBuf(const double* host, std::size_t n) : DevBuf(n) { upload(host, n, 0); }
    ~DevBuf() {
        if (p_) mlora_free(detail::facade_ctx(), p_);
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    double* get() const { return static_cast<double*>(p_); }
    void upload(const double* host, std::size_t n, std::size_t off) {
        if (n == 0) return;
        if (mlora_memcpy(detail::facade_ctx(), get() + off, host, n * sizeof(double), 0, nullptr) != MLORA_OK)
            throw DeviceError(std::string("H2D copy: ") + mlora_last_error(detail::facade_ctx()));
    }
    void download(double* host, std::size_t n, std::size_t off) const {
        if (n == 0) return;
        if (mlora_memcpy(detail::facade_ctx(), host, get() + off, n * sizeof(double), 1, nullptr) != MLORA_OK)
            throw DeviceError(std::string("D2H copy: ") + mlora_last_error(detail::facade_ctx()));
    }

private:
    void* p_ = nullptr;
    std::size_t n_ = 0;
};

// C = op(A) op(B) on device buffers.
void gemm(long M, long N, long K, const double* A, long lda, bool tA, const double* B, long ldb, bool tB,
          double* C, long ldc) {
    check_status(mlora_f64_gemm(M, N, K, A, lda, tA ? 1 : 0, B, ldb, tB ? 1 : 0, C, ldc, nullptr),
                 "mlora_f64_gemm");
}

void sync() {
    if (mlora_stream_sync(detail::facade_ctx(), nullptr) != MLORA_OK)
        throw DeviceError(std::string("device execution: ") + mlora_last_error(detail::facade_ctx()));
}

}  // namespace

// ------------------------------------------------------------------ Matrix
Matrix::Matrix(int r, int c) : rows(r), cols(c), data(static_cast<std::size_t>(r) * c, 0.0) {}

Matrix Matrix::identity(int n) {
    Matrix m(n, n);
    for (int i = 0; i < n; ++i) m.at(i, i) = 1.0;
    return m;
}

bool Matrix::all_finite() const {
    for (double v : data)
        if (!std::isfinite(v)) return false;
    return true;
}

Matrix matmul(const Matrix& a, const Matrix& b) {
    if (a.cols != b.rows)
        throw ShapeError("matmul: " + std::to_string(a.rows) + "x" + std::to_string(a.cols) + " * " +
                         std::to_string(b.rows) + "x" + std::to_string(b.cols));
    Matrix c(a.rows, b.cols);
    if (c.data.empty()) return c;
    DevBuf da(a.data.data(), a.data.size()), db(b.data.data(), b.data.size()), dc(c.data.size());
    gemm(a.rows, b.cols, a.cols, da.get(), a.cols, false, db.get(), b.cols, false, dc.get(), b.cols);
    sync();
    dc.download(c.data.data(), c.data.size(), 0);
    return c;
}

Matrix add(const Matrix& a, const Matrix& b) {
    if (a.rows != b.rows || a.cols != b.cols) throw ShapeError("add: incompatible shapes");
    Matrix c = a;
    for (std::size_t i = 0; i < c.data.size(); ++i) c.data[i] += b.data[i];
    return c;
}

Matrix transpose(const Matrix& a) {
    Matrix t(a.cols, a.rows);
    for (int i = 0; i < a.rows; ++i)
        for (int j = 0; j < a.cols; ++j) t.at(j, i) = a.at(i, j);
    return t;
}

double max_rel_diff(const Matrix& a, const Matrix& b) {
    if (a.rows != b.rows || a.cols != b.cols) throw ShapeError("max_rel_diff: incompatible shapes");
    double worst = 0.0;
    for (std::size_t i = 0; i < a.data.size(); ++i) {
        const double scale = std::max({std::fabs(a.data[i]), std::fabs(b.data[i]), 1.0});
        worst = std::max(worst, std::fabs(a.data[i] - b.data[i]) / scale);
    }
    return worst;
}

// ------------------------------------------------------------------ adapters / accounting
void AdapterWeights::validate(int d, int k) const {
    if (rank < 1) throw UsageError("adapter rank must be >= 1");
    if (rank > std::min(d, k)) throw UsageError("adapter rank exceeds min(d, k)");
    if (A.rows != rank || A.cols != k) throw ShapeError("adapter A must be rank x k");
    if (B.rows != d || B.cols != rank) throw ShapeError("adapter B must be d x rank");
}

double FusedShape::padding_ratio() const {
    return total_tokens == 0 ? 0.0 : static_cast<double>(padding_tokens) / static_cast<double>(total_tokens);
}

FusedShape fused_shape(const std::vector<std::vector<int>>& per_group_lengths) {
    std::vector<int32_t> flat;
    for (const auto& g : per_group_lengths) flat.insert(flat.end(), g.begin(), g.end());
    mlora_fused_shape s{};
    check_status(mlora_fused_shape_of(flat.data(), static_cast<int64_t>(flat.size()), &s), "fused_shape");
    FusedShape out;
    out.max_len = s.max_len;
    out.sequences = s.sequences;
    out.total_tokens = s.total_tokens;
    out.padding_tokens = s.padding_tokens;
    return out;
}

double FusedBatch::padding_ratio() const {
    return total_tokens == 0 ? 0.0 : static_cast<double>(padding_tokens) / static_cast<double>(total_tokens);
}

int FusedBatch::real_length(int seq) const {
    const auto* m = mask.data() + static_cast<std::size_t>(seq) * max_len;
    return static_cast<int>(std::count(m, m + max_len, std::uint8_t{1}));
}

Matrix FusedBatch::sequence(int seq) const {
    Matrix m(max_len, dim);
    const std::size_t off = static_cast<std::size_t>(seq) * max_len * dim;
    std::copy_n(data.begin() + static_cast<std::ptrdiff_t>(off), m.data.size(), m.data.begin());
    return m;
}

FusedBatch fuse(const std::vector<JobBatch>& batches) {
    if (batches.empty()) throw UsageError("fuse: empty batch list");
    int dim = -1;
    std::vector<std::vector<int>> lengths;
    lengths.reserve(batches.size());
    for (const auto& b : batches) {
        std::vector<int> ls;
        for (const auto& s : b.sequences) {
            if (dim < 0) dim = s.cols;
            if (s.cols != dim) throw ShapeError("fuse: embedding dims differ across sequences");
            if (s.rows < 1) throw UsageError("fuse: empty sequence");
            ls.push_back(s.rows);
        }
        lengths.push_back(std::move(ls));
    }
    const FusedShape shape = fused_shape(lengths);
    if (shape.sequences == 0) throw UsageError("fuse: no sequences");

    FusedBatch fb;
    fb.num_sequences = static_cast<int>(shape.sequences);
    fb.max_len = shape.max_len;
    fb.dim = dim;
    fb.total_tokens = shape.total_tokens;
    fb.padding_tokens = shape.padding_tokens;
    fb.data.assign(static_cast<std::size_t>(fb.num_sequences) * fb.max_len * dim, 0.0);
    fb.mask.assign(static_cast<std::size_t>(fb.num_sequences) * fb.max_len, 0);
    std::size_t row = 0;
    for (const auto& b : batches) {
        for (const auto& s : b.sequences) {
            fb.routing.push_back(b.job_id);
            std::fill_n(fb.mask.begin() + static_cast<std::ptrdiff_t>(row), s.rows, std::uint8_t{1});
            std::copy(s.data.begin(), s.data.end(), fb.data.begin() + static_cast<std::ptrdiff_t>(row * dim));
            row += fb.max_len;
        }
    }
    return fb;
}

// ------------------------------------------------------------------ compute (device)
Matrix lora_forward(const Matrix& W0, const AdapterWeights& adapter, const Matrix& x) {
    const int d = W0.rows, k = W0.cols;
    adapter.validate(d, k);
    if (x.rows != k) throw ShapeError("lora_forward: x must be k x m");
    if (!W0.all_finite() || !x.all_finite() || !adapter.A.all_finite() || !adapter.B.all_finite())
        throw NumericError("lora_forward: non-finite input");
    const int m = x.cols, r = adapter.rank;
    Matrix h(d, m);
    if (h.data.empty()) return h;
    DevBuf dW(W0.data.data(), W0.data.size()), dx(x.data.data(), x.data.size()),
        dA(adapter.A.data.data(), adapter.A.data.size()), dB(adapter.B.data.data(), adapter.B.data.size()),
        base(static_cast<std::size_t>(d) * m), ax(static_cast<std::size_t>(r) * m),
        low(static_cast<std::size_t>(d) * m);
    gemm(d, m, k, dW.get(), k, false, dx.get(), m, false, base.get(), m);   // W0 x
    gemm(r, m, k, dA.get(), k, false, dx.get(), m, false, ax.get(), m);     // A x
    gemm(d, m, r, dB.get(), r, false, ax.get(), m, false, low.get(), m);    // B (A x)
    check_status(mlora_f64_add(static_cast<int64_t>(h.data.size()), base.get(), low.get(), base.get(), nullptr),
                 "mlora_f64_add");
    sync();
    base.download(h.data.data(), h.data.size(), 0);
    return h;
}

std::vector<Matrix> fused_forward(const Matrix& W0, const std::map<std::string, AdapterWeights>& adapters,
                                  const FusedBatch& fb) {
    if (W0.cols != fb.dim) throw ShapeError("fused_forward: W0 column dim does not match batch dim");
    for (const auto& job : fb.routing)
        if (adapters.find(job) == adapters.end())
            throw RoutingError("fused_forward: no adapter for job " + job);
    const int d = W0.rows, k = W0.cols;
    for (const auto& job : fb.routing) adapters.at(job).validate(d, k);

    const long L = fb.max_len, S = fb.num_sequences;
    const long rows = S * L;
    std::vector<Matrix> outs;
    outs.reserve(static_cast<std::size_t>(S));
    if (rows == 0 || d == 0) {
        for (long s = 0; s < S; ++s) outs.emplace_back(static_cast<int>(L), d);
        return outs;
    }
    DevBuf dX(fb.data.data(), fb.data.size()), dW(W0.data.data(), W0.data.size()),
        dY(static_cast<std::size_t>(rows) * d);
    // one base pass over every fused row: Y = X W0^T (W0 read transposed in place)
    gemm(rows, d, k, dX.get(), k, false, dW.get(), k, true, dY.get(), d);
    // one low-rank pass per run of consecutive sequences of the same job
    long s0 = 0;
    while (s0 < S) {
        long s1 = s0 + 1;
        while (s1 < S && fb.routing[s1] == fb.routing[s0]) ++s1;
        const AdapterWeights& ad = adapters.at(fb.routing[s0]);
        const long n = (s1 - s0) * L, r = ad.rank;
        DevBuf dA(ad.A.data.data(), ad.A.data.size()), dB(ad.B.data.data(), ad.B.data.size()),
            t(static_cast<std::size_t>(n) * r), low(static_cast<std::size_t>(n) * d);
        const double* xrun = dX.get() + s0 * L * k;
        double* yrun = dY.get() + s0 * L * d;
        gemm(n, r, k, xrun, k, false, dA.get(), k, true, t.get(), r);      // X A^T
        gemm(n, d, r, t.get(), r, false, dB.get(), r, true, low.get(), d); // (X A^T) B^T
        check_status(mlora_f64_add(n * d, yrun, low.get(), yrun, nullptr), "mlora_f64_add");
        sync();  // the run's temporaries are freed at scope exit
        s0 = s1;
    }
    sync();
    for (long s = 0; s < S; ++s) {
        Matrix o(static_cast<int>(L), d);
        dY.download(o.data.data(), o.data.size(), static_cast<std::size_t>(s * L * d));
        outs.push_back(std::move(o));
    }
    return outs;
}

LaunchCount count_launches(int num_jobs, LaunchMode mode) {
    int64_t small = 0, large = 0;
    check_status(mlora_count_launches(num_jobs, mode == LaunchMode::PerJob ? 0 : 1, &small, &large),
                 "count_launches: need at least one job");
    LaunchCount c;
    c.small_launches = small;
    c.large_launches = large;
    return c;
}

}  // namespace fusim
