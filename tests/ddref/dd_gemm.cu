// Double-double reference GEMM for the full-matrix accuracy sweep (test
// infrastructure, not the product: only tests/accuracy_full.py loads it).
//
// The reference measures max_rel_err against exact_gemm_oracle, a correctly
// rounded exact dot product per entry (proj/src/oracle.cpp:276-301,
// max_rel_err :321-335).  On the CPU that costs hours at n = 8192; here every
// entry is computed with the compensated dot product Dot2 (Ogita, Rump,
// Oishi 2005): TwoProd by FMA, TwoSum of the running sum, the two error terms
// summed in a second double.  The pair (hi, lo) = (s, c) approximates the
// exact value with error <= gamma_n^2 sum|a_l b_l| (~8e-25 sum|a b| at
// n = 8192), far below every error it is used to measure; tests/accuracy_full.py
// pins it against the reference's exact oracle on sampled entries.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a --fmad=false (no FMA
// contraction may touch TwoSum) -shared.  FP64 CUDA-core arithmetic: 10 flops
// per multiply-add, 64 x 64 outputs per 256-thread CTA, 4 x 4 per thread.
#include <cuda_runtime.h>
#include <cstdint>

namespace {

constexpr int kT = 64, kK = 16;

__global__ void __launch_bounds__(256) dd_gemm_kernel(const double* __restrict__ A, const double* __restrict__ B,
                                                      double* __restrict__ hi, double* __restrict__ lo, int m, int n,
                                                      int p) {
  __shared__ __align__(16) double As[kK][kT];
  __shared__ __align__(16) double Bs[kK][kT];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int row0 = blockIdx.y * kT, col0 = blockIdx.x * kT;
  double s[4][4], c[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) s[i][j] = 0.0, c[i][j] = 0.0;
  for (int k0 = 0; k0 < n; k0 += kK) {
    // A tile 64 x 16 (transposed into As), B tile 16 x 64: 4 elements per thread each
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = tid + 256 * u;
      const int ar = e / kK, ak = e % kK;
      const int gr = row0 + ar, gk = k0 + ak;
      As[ak][ar] = (gr < m && gk < n) ? A[static_cast<int64_t>(gr) * n + gk] : 0.0;
      const int bk = e / kT, bc = e % kT;
      const int gk2 = k0 + bk, gc = col0 + bc;
      Bs[bk][bc] = (gk2 < n && gc < p) ? B[static_cast<int64_t>(gk2) * p + gc] : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < kK; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i], b[i] = Bs[kk][tx * 4 + i];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const double pr = __dmul_rn(a[i], b[j]);
          const double pe = __fma_rn(a[i], b[j], -pr);  // TwoProd: a b = pr + pe exactly
          const double t = __dadd_rn(s[i][j], pr);     // TwoSum(s, pr) = t + q exactly
          const double z = __dsub_rn(t, s[i][j]);
          const double q = __dadd_rn(__dsub_rn(s[i][j], __dsub_rn(t, z)), __dsub_rn(pr, z));
          s[i][j] = t;
          c[i][j] = __dadd_rn(c[i][j], __dadd_rn(q, pe));
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = row0 + ty * 4 + i, col = col0 + tx * 4 + j;
      if (r < m && col < p) {
        // FastTwoSum-normalised pair: h = fl(s + c), l = c - (h - s)
        const double h = __dadd_rn(s[i][j], c[i][j]);
        hi[static_cast<int64_t>(r) * p + col] = h;
        lo[static_cast<int64_t>(r) * p + col] = __dsub_rn(c[i][j], __dsub_rn(h, s[i][j]));
      }
    }
}

}  // namespace

extern "C" int dd_gemm(const double* A, const double* B, double* hi, double* lo, int64_t m, int64_t n, int64_t p,
                       void* stream) {
  if (m < 1 || n < 1 || p < 1 || m > (1 << 30) || p > (1 << 30) || n > (1 << 30)) return 1;
  dim3 grid(static_cast<unsigned>((p + kT - 1) / kT), static_cast<unsigned>((m + kT - 1) / kT));
  dd_gemm_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(A, B, hi, lo, static_cast<int>(m),
                                                                      static_cast<int>(n), static_cast<int>(p));
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
