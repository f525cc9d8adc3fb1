// K1 variants for the comparison methods of the paper:
//
//   ozIMMU     = BitMask split            + per-product FP64 accumulation
//   ozIMMU_EF  = BitMask split            + group-wise accumulation
//   ozIMMU_RN  = RoundNearestPerSlice     + per-product FP64 accumulation
//   (ozIMMU_H  = RoundNearestConstShift   + group-wise: slicer.cuh)
//   -- config_for, proj/src/scheme.cpp:137-159.
//
// Same output layout as slicer.cuh (int8 planes [k][line][lds], K-major).
#pragma once

#include <cstdint>

#include "fp64_exact.cuh"
#include "slicer.cuh"

namespace ozb {

// ---------------------------------------------------------------- bitmask
// bitmask_rows (proj/src/split.cpp:56-104) for 16 elements of one line with
// row exponent p = ufp_exponent(rm) (INT32_MIN: zero line, slices stay 0):
// slice s holds the s-th beta-bit field of |a| on the row grid, with a's sign.
__device__ __forceinline__ void emit16_bitmask(const double (&w)[16], int p, int beta, int k,
                                               int8_t* dst, int64_t plane) {
  const uint64_t mask = (1ull << beta) - 1;
  for (int s = 1; s <= k; ++s) {
    uint32_t packed[4] = {0u, 0u, 0u, 0u};
    if (p != INT32_MIN) {
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        // decompose (include/ozmm/ufp.hpp:61-80)
        const uint64_t bits = static_cast<uint64_t>(__double_as_longlong(w[e]));
        const int biased = static_cast<int>((bits >> 52) & 0x7FF);
        const uint64_t frac = bits & 0x000FFFFFFFFFFFFFull;
        const uint64_t asig = biased == 0 ? frac : (frac | (1ull << 52));
        const int exp = biased == 0 ? -1074 : biased - 1075;
        uint32_t q = 0;
        if (asig != 0) {
          const int t = exp - p - 1 + s * beta;  // split.cpp:76
          uint64_t chunk = 0;
          if (t >= beta) chunk = 0;
          else if (t >= 0) chunk = (asig << t) & mask;
          else if (-t <= 63) chunk = (asig >> -t) & mask;
          const int v = (bits >> 63) ? -static_cast<int>(chunk) : static_cast<int>(chunk);
          q = static_cast<uint32_t>(v) & 0xFFu;
        }
        packed[e >> 2] |= q << (8 * (e & 3));
      }
    }
    *reinterpret_cast<uint4*>(dst + static_cast<int64_t>(s - 1) * plane) =
        make_uint4(packed[0], packed[1], packed[2], packed[3]);
  }
}

// Row exponent of bitmask_rows: p = ufp_exponent(rm), underflow flag only
// (split.cpp:65-69; the bitmask splitter has no range error).
__device__ __forceinline__ int bitmask_pe(double rm, bool* under) {
  if (rm == 0.0) return INT32_MIN;
  const int p = ufp_exponent(rm);
  if (p < -1000) *under = true;
  return p;
}

// Cluster-split rows (like slice_rows_cluster_kernel) for BitMask.
template <bool kVec>
__global__ void __launch_bounds__(1024) slice_rows_bitmask_kernel(
    const double* __restrict__ X, int64_t ld, int64_t rows, int64_t len, int64_t lds, int k,
    int beta, int8_t* __restrict__ S, int64_t plane, double* __restrict__ shift,
    int* __restrict__ flags) {
  __shared__ double red[32];
  __shared__ double cmax[8];
  uint32_t crank, csize;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(csize));
  const int64_t row = blockIdx.x / csize;
  const double* x = X + row * ld;
  int8_t* out = S + row * lds;
  const int64_t base0 = 16 * (static_cast<int64_t>(crank) * blockDim.x + threadIdx.x);
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  double w[16];
  load16(x, base0, len, kVec, w);
  double rm = 0.0;
#pragma unroll
  for (int e = 0; e < 16; ++e) rm = fmax(rm, fabs(w[e]));
  rm = block_max(rm, red);
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
  if (threadIdx.x < csize) {
    uint32_t local = static_cast<uint32_t>(__cvta_generic_to_shared(&cmax[crank]));
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(threadIdx.x));
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(remote), "d"(rm) : "memory");
  }
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  for (uint32_t c = 0; c < csize; ++c) rm = fmax(rm, cmax[c]);
  bool under = false;
  const int p = bitmask_pe(rm, &under);
  if (crank == 0 && threadIdx.x == 0) {
    shift[row] = p == INT32_MIN ? 0.0 : pow2(p);
    report_flags(flags, under, false);
  }
  if (base0 < lds) emit16_bitmask(w, p, beta, k, out + base0, plane);
}

// Column mode for BitMask (after colmax_kernel): same tiling as slice_cols_kernel.
__global__ void __launch_bounds__(256) slice_cols_bitmask_kernel(
    const double* __restrict__ X, int64_t ld, int64_t len, int64_t cols, int64_t lds, int k,
    int beta, const unsigned long long* __restrict__ colmax, int8_t* __restrict__ S,
    int64_t plane, double* __restrict__ shift, int* __restrict__ flags) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t col = static_cast<int64_t>(blockIdx.x) * 32 + warp * 4 + (lane & 3);
  const int64_t base = static_cast<int64_t>(blockIdx.y) * 128 + 16 * (lane >> 2);
  if (col >= cols || base >= lds) return;
  const double rm = __longlong_as_double(static_cast<long long>(colmax[col]));
  bool under = false;
  const int p = bitmask_pe(rm, &under);
  if (blockIdx.y == 0 && (lane >> 2) == 0) {
    shift[col] = p == INT32_MIN ? 0.0 : pow2(p);
    report_flags(flags, under, false);
  }
  double w[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) w[e] = base + e < len ? __ldg(X + (base + e) * ld + col) : 0.0;
  emit16_bitmask(w, p, beta, k, S + col * lds + base, plane);
}

// ------------------------------------------------- round-nearest per slice
// round_nearest_rows (proj/src/split.cpp:132-149): for s = 0..k-1 the grid
// is re-derived from the CURRENT residual's row max (rn_unit, :121-130);
// a row whose residual vanished keeps zero slices and zero units (break, :141).
// Rows are cluster-split and held in registers; one cluster max per slice.
template <bool kVec>
__global__ void __launch_bounds__(1024) slice_rows_rnps_kernel(
    const double* __restrict__ X, int64_t ld, int64_t rows, int64_t len, int64_t lds, int k,
    int beta, int8_t* __restrict__ S, int64_t plane, double* __restrict__ units,
    int* __restrict__ flags) {
  __shared__ double red[32];
  __shared__ double cmax[2][8];  // double-buffered cluster exchange (one per slice)
  uint32_t crank, csize;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(csize));
  const int64_t row = blockIdx.x / csize;
  const double* x = X + row * ld;
  int8_t* out = S + row * lds;
  const int64_t base0 = 16 * (static_cast<int64_t>(crank) * blockDim.x + threadIdx.x);
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  double w[16];
  load16(x, base0, len, kVec, w);
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
  bool under = false, range = false, done = false;
  for (int s = 0; s < k; ++s) {
    double rm = 0.0;
    if (!done) {
#pragma unroll
      for (int e = 0; e < 16; ++e) rm = fmax(rm, fabs(w[e]));
      rm = block_max(rm, red);
      __syncthreads();  // red[] is reused by the next slice
      if (threadIdx.x < csize) {
        uint32_t local = static_cast<uint32_t>(__cvta_generic_to_shared(&cmax[s & 1][crank]));
        uint32_t remote;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(threadIdx.x));
        asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(remote), "d"(rm) : "memory");
      }
      asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
      asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
      for (uint32_t c = 0; c < csize; ++c) rm = fmax(rm, cmax[s & 1][c]);
      if (rm == 0.0) done = true;  // remaining slices and units stay zero
    }
    uint32_t packed[4] = {0u, 0u, 0u, 0u};
    double unit = 0.0;
    if (!done) {
      // rn_unit: pe = ufp_exponent(rm); bump if rm >= (2 - 2^-beta) 2^pe
      const int pe = line_pe(rm, beta, &under, &range);  // returns pe + bump
      const int ue = pe + 1 - beta;
      unit = pow2(ue);
      if (unit != 0.0) {
        const double sigma = __dmul_rn(kSigmaScale, unit);
        const long long sbits = __double_as_longlong(sigma);
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const double t = __dadd_rn(w[e], sigma);
          const double xx = __dadd_rn(t, -sigma);
          const uint32_t q = static_cast<uint32_t>(__double_as_longlong(t) - sbits);
          w[e] = __dadd_rn(w[e], -xx);
          packed[e >> 2] |= (q & 0xFFu) << (8 * (e & 3));
        }
      } else {
#pragma unroll
        for (int e = 0; e < 16; ++e) w[e] = __dadd_rn(w[e], -w[e]);
      }
    }
    if (crank == 0 && threadIdx.x == 0) units[static_cast<int64_t>(s) * rows + row] = unit;
    if (base0 < lds)
      *reinterpret_cast<uint4*>(out + base0 + static_cast<int64_t>(s) * plane) =
          make_uint4(packed[0], packed[1], packed[2], packed[3]);
  }
  if (crank == 0 && threadIdx.x == 0) report_flags(flags, under, range);
}

// FP64 transpose (rows x cols, row stride ld) -> (cols x rows, dense): used to
// give the per-slice RN splitter contiguous lines for column-wise splits.
__global__ void __launch_bounds__(256) transpose_f64_kernel(const double* __restrict__ X,
                                                            int64_t ld, int64_t rows,
                                                            int64_t cols,
                                                            double* __restrict__ Y) {
  __shared__ double tile[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * 32, c0 = static_cast<int64_t>(blockIdx.x) * 32;
  for (int j = ty; j < 32; j += 8)
    if (r0 + j < rows && c0 + tx < cols) tile[j][tx] = X[(r0 + j) * ld + c0 + tx];
  __syncthreads();
  for (int j = ty; j < 32; j += 8)
    if (c0 + j < cols && r0 + tx < rows) Y[(c0 + j) * rows + r0 + tx] = tile[tx][j];
}

// Residual of a split, the reference's SplitMatrix::residual (split.cpp:49,
// dumped by dump_split, :269): w = x, then for s = 1..k the exact w -= slice_s
// unit_s of the strategy's extraction.  Every step is exact in all three
// splitters (the slice is w's rounded or truncated digit on the unit grid), so
// the FP64 recurrence reproduces the reference bit for bit; the sign-of-zero
// cases follow the reference's control flow:
//   * RN (const shift, per slice): a unit that underflowed to 0 extracts x = w,
//     so w becomes +0 unless it already was a zero;
//   * bitmask: a zero element, or a unit below 2^-1074 (no bits there), leaves
//     the skeleton's +0 / w unchanged;
//   * a zero line (shift 0) keeps the skeleton's +0 for the const-shift
//     splitters, while the per-slice splitter stores w (x itself) there.
// X: the op(X) lines as in the splitters (row_mode: line i = X[i][0..n), else
// X[0..n)[i]); sh: const shift [lines] (strategy 0, 1) or units [k][lines] (2).
// R: [lines][n].
__global__ void split_residual_kernel(const double* __restrict__ X, int64_t ldx, int row_mode, int64_t lines,
                                      int64_t n, int k, int beta, int strategy, const int8_t* __restrict__ S,
                                      int64_t lds, int64_t plane, const double* __restrict__ sh,
                                      double* __restrict__ R) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= lines * n) return;
  const int64_t line = idx / n, j = idx % n;
  const double x = row_mode ? X[line * ldx + j] : X[j * ldx + line];
  double w = x;
  if (strategy != 2 && sh[line] == 0.0) {
    w = 0.0;  // zero line: the const-shift splitters skip it (residual stays +0)
  } else if (strategy == 1 && x == 0.0) {
    w = 0.0;  // bitmask: zero elements are skipped
  } else {
    for (int s = 1; s <= k; ++s) {
      const double unit = strategy == 2 ? sh[static_cast<int64_t>(s - 1) * lines + line]
                                        : __dmul_rn(sh[line], pow2(1 - beta * s));
      if (unit == 0.0) {
        if (strategy != 1 && w != 0.0) w = 0.0;
        continue;
      }
      const int8_t v = S[static_cast<int64_t>(s - 1) * plane + line * lds + j];
      w = __dsub_rn(w, __dmul_rn(static_cast<double>(v), unit));
    }
  }
  R[line * n + j] = w;
}

}  // namespace ozb
