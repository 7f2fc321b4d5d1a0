// mlora_f64.cu — the fp64 device path behind the reference-typed C++ façade.
//
// fusim::Matrix is fp64 (/root/reference/proj/include/fusim/lora.hpp:13-27), so
// the façade's fused_forward / lora_forward / matmul run here, on the GPU, with
// the reference's exact per-element operation sequence:
//   c = 0; for k = 0..K-1 in order: if (a_ik != 0) c = c + a_ik * b_kj
// (lora.cpp:25-32: i-k-j loop with the a_ik == 0 skip, no FMA contraction —
// x86-64 g++ -O3 without -mfma rounds the product and the sum separately).
// Every output element is owned by one thread that walks k in ascending order,
// so results are bit-identical to the reference regardless of tiling.
// This is a compatibility path (correct fp64 semantics for the reference API),
// not the throughput path — that is the bf16 tcgen05 engine in mlora_gemm.cuh.
#include <cuda_runtime.h>

#include <string>

#include "../../include/mlora.h"

namespace {

constexpr int kT = 32;   // output tile (kT x kT) per 256-thread block, 4 outputs per thread
constexpr int kKT = 16;  // k-slab staged in shared memory

// C[M,N] = op(A)[M,K] * op(B)[K,N];  op(A)(i,k) = transA ? A[k*lda+i] : A[i*lda+k]
__global__ void f64_gemm_seq_kernel(int M, int N, int K, const double* __restrict__ A, long long lda,
                                    int transA, const double* __restrict__ B, long long ldb, int transB,
                                    double* __restrict__ C, long long ldc) {
    __shared__ double sA[kT][kKT + 1];
    __shared__ double sB[kKT][kT + 1];
    const int tx = threadIdx.x % kT;          // column within tile
    const int ty = threadIdx.x / kT;          // 0..7, rows ty + 8*u
    const int i0 = blockIdx.y * kT, j0 = blockIdx.x * kT;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int k0 = 0; k0 < K; k0 += kKT) {
        for (int e = threadIdx.x; e < kT * kKT; e += blockDim.x) {
            const int r = e / kKT, kk = e % kKT;
            const int i = i0 + r, k = k0 + kk;
            sA[r][kk] = (i < M && k < K) ? (transA ? A[(long long)k * lda + i] : A[(long long)i * lda + k]) : 0.0;
            const int kb = e / kT, cb = e % kT;
            const int j = j0 + cb, k2 = k0 + kb;
            sB[kb][cb] = (j < N && k2 < K) ? (transB ? B[(long long)j * ldb + k2] : B[(long long)k2 * ldb + j]) : 0.0;
        }
        __syncthreads();
        const int kend = min(kKT, K - k0);
        for (int kk = 0; kk < kend; ++kk) {
            const double b = sB[kk][tx];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const double a = sA[ty + 8 * u][kk];
                if (a != 0.0) acc[u] = __dadd_rn(acc[u], __dmul_rn(a, b));
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int i = i0 + ty + 8 * u, j = j0 + tx;
        if (i < M && j < N) C[(long long)i * ldc + j] = acc[u];
    }
}

__global__ void f64_add_kernel(long long n, const double* __restrict__ a, const double* __restrict__ b,
                               double* __restrict__ c) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        c[i] = __dadd_rn(a[i], b[i]);
}

}  // namespace

extern "C" {

mlora_status mlora_f64_gemm(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, int32_t transA,
                            const double* B, int64_t ldb, int32_t transB, double* C, int64_t ldc, void* stream) {
    if (M < 0 || N < 0 || K < 0) return MLORA_SHAPE;
    if (M == 0 || N == 0) return MLORA_OK;
    if (!A || !B || !C) return MLORA_USAGE;
    if (M > (1LL << 31) / kT || N > (1LL << 31) / kT) return MLORA_USAGE;
    dim3 grid(static_cast<unsigned>((N + kT - 1) / kT), static_cast<unsigned>((M + kT - 1) / kT));
    f64_gemm_seq_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<int>(M), static_cast<int>(N), static_cast<int>(K), A, lda, transA, B, ldb, transB, C, ldc);
    return cudaGetLastError() == cudaSuccess ? MLORA_OK : MLORA_CUDA;
}

mlora_status mlora_f64_add(int64_t n, const double* a, const double* b, double* c, void* stream) {
    if (n < 0) return MLORA_SHAPE;
    if (n == 0) return MLORA_OK;
    if (!a || !b || !c) return MLORA_USAGE;
    const long long blocks = (n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096;
    f64_add_kernel<<<static_cast<unsigned>(blocks), 256, 0, static_cast<cudaStream_t>(stream)>>>(n, a, b, c);
    return cudaGetLastError() == cudaSuccess ? MLORA_OK : MLORA_CUDA;
}

}  // extern "C"
