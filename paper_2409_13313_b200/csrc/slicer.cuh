// K1 -- the slicing kernels (ozIMMU_H round-to-nearest, constant shift).
//
// Restates rn_const_shift_rows (proj/src/split.cpp:151-173) with rn_unit
// (:121-130) and extract_row (:109-117) on the GPU, bit-exactly:
//   per line (row of op(A) / column of op(B)):  rm = max |x|,
//     pe0 = ufp_exponent(rm), bump = rm >= (2-2^-beta) 2^pe0, PE = pe0+bump,
//     shift = 2^PE, unit_s = 2^(PE+1-beta*s);
//   per element, s = 1..k:  sigma = 0.75*2^53*unit_s,
//     x = (w + sigma) - sigma, slice_s = int8(x / unit_s), w -= x.
//
// Output layout (the GEMM's K-major operand layout): slices[s][line][0..lds),
// one int8 plane of `lines x lds` bytes per slice, where lds = round_up(n, 16)
// so every line starts 16-byte aligned for TMA; bytes [n, lds) are written as
// zeros.  The shift vector is written as doubles (const_shift, split.hpp:37).
//
// Offset-binary planes (`lsum != nullptr`, the fused GEMM's operand format):
// byte = slice + o_s with the even offsets o_1 = 2^beta and o_s = max(2,
// 2^(beta-1)) for s >= 2 (slice_offset), so every byte is an unsigned value in
// [0, 255] (|slice_1| <= 2^beta - 1 by rn_unit's bump rule, |slice_s| <=
// 2^(beta-1) after round-to-nearest); padding bytes stay 0.  lsum[s * lsum_plane + line * lsum_lstride] (zeroed by
// the caller) receives the line's sum of the SIGNED slice values (mod 2^32), from which the GEMM removes
// the offsets' contribution exactly (ozimmu_gemm_pair.cuh).  The signed planes
// (lsum == nullptr) are the reference's SplitMatrix slices, bit for bit.
//
// Two access patterns, both one coalesced read of the FP64 input plus one
// 16-byte-vector write per slice:
//   * slice_rows_kernel: lines are contiguous rows (A, or B when transb='T').
//     One CTA per line, 16 consecutive elements per thread held in registers:
//     the row max is a warp-shuffle + smem reduction, then the same registers
//     are sliced -- the row is read from HBM once (rows up to 16384).
//   * colmax_kernel + slice_cols_kernel: lines are strided columns (B, or A
//     when transa='T').  Pass 1 reduces column maxima (warp-coalesced rows,
//     smem tree + atomicMax on the IEEE bit pattern, which orders like the
//     value for |x|).  Pass 2 reads 32-column x 128-row tiles coalesced and
//     writes each column's 16-byte slice runs: the transposed K-major planes.
#pragma once

#include <cstdint>

#include "fp64_exact.cuh"
#include "ptx.cuh"

namespace ozb {

constexpr double kSigmaScale = 6755399441055744.0;  // 0.75 * 2^53 (split.cpp:16)
constexpr int kMaxSlices = 32;  // = kMaxK of the GEMM (line-sum scratch in shared memory)

// flags[0] |= underflow (pe < -1000), flags[1] |= range (pe > 920).
__device__ __forceinline__ void report_flags(int* flags, bool under, bool range) {
  if (under) atomicOr(flags + 0, 1);
  if (range) atomicOr(flags + 1, 1);
}

// Slice 16 consecutive elements of one line (w[] is updated in place) and
// store the k 16-byte runs.  PE == INT32_MIN marks a zero line.
//
// Per element and slice: t = w + sigma, x = t - sigma, w -= x (three RN adds,
// exactly extract_row's (w+sigma)-sigma and w -= x).  sigma = 1.5 * 2^52 *
// unit is built from its bits (its low word is 0) and |x| < 2^51 * unit puts
// t in sigma's binade [2^52 unit, 2^53 unit), whose ulp is unit, so the low
// word of bits(t) is the slice integer x / unit in two's complement -- no
// subtract, division or float->int conversion.  Valid for every unit >=
// 2^-1074 (sigma is then normal); unit == 0 (underflowed grid) is handled
// separately.
//
// Offset mode (lsum != nullptr): sigma is replaced by sigma' = sigma + o_s unit
// (bits(sigma) + o_s: same binade).  Adding an exact multiple of the ulp
// commutes with round-to-nearest inside a binade, and because o_s is EVEN the
// ties-to-even choice is the same too, so t' = RN(w + sigma') = t + o_s unit
// and x = t' - sigma' = t - sigma bit for bit; the low byte of bits(t') is the
// offset-binary byte slice + o_s with no further instruction.  Padding elements
// (the `nvalid`.. 15 tail of a line) are masked to byte 0.  The per-slice sums
// of the SIGNED values (sum of the bytes minus o_s per valid element) are
// reduced over the lanes that share the line (kLaneGroup: 32 = the whole warp
// is one line, 8 = lanes l, l^4, l^8, .. of slice_cols_kernel) and added into
// lsum[s-1][0] by the group's first lane.  Every lane of the warp must call it
// (nvalid = 0 and store = false for lanes without data).
template <int kLaneGroup = 32>
__device__ __forceinline__ void emit16(double (&w)[16], int PE, int beta, int k,
                                       int8_t* dst, int64_t plane, int nvalid = 16,
                                       bool store = true, int* lsum = nullptr,
                                       int64_t lsum_plane = 0) {
  // Loop invariants (the slicer is issue-bound: ncu 73 % of issue slots, with the
  // FP64 pipe the next limit): the padding mask, both offsets and their share of
  // the line sums, the unit exponent (stepped by -beta), the store pointer (stepped
  // by plane) and the shared-memory address of the line sums (lsum always points
  // into shared memory; red.shared avoids the generic atomic's warp aggregation).
  const bool partial = lsum != nullptr && nvalid < 16;
  uint32_t keep[4] = {~0u, ~0u, ~0u, ~0u};
  if (partial) {
#pragma unroll
    for (int e = 0; e < 16; ++e)
      if (e >= nvalid) keep[e >> 2] &= ~(0xFFu << (8 * (e & 3)));
  }
  uint32_t o1 = lsum == nullptr ? 0u : slice_offset(1, beta);  // 0: signed planes
  uint32_t os = lsum == nullptr ? 0u : slice_offset(2, beta);
  uint32_t nv = static_cast<uint32_t>(nvalid);
  uint32_t part = partial ? 1u : 0u, st = store ? 1u : 0u;
  uint32_t lead = kLaneGroup == 32 ? ((threadIdx.x & 31) == 0 ? 1u : 0u)
                                   : ((threadIdx.x & 31) < 32 / kLaneGroup ? 1u : 0u);
  // opaque to the optimiser: kept in registers, not re-derived inside the slice loop
  asm volatile("" : "+r"(o1), "+r"(os), "+r"(nv), "+r"(part), "+r"(st), "+r"(lead));
  const bool zero_line = PE == INT32_MIN;
  uint32_t ls_addr = lsum == nullptr ? 0u : static_cast<uint32_t>(__cvta_generic_to_shared(lsum));
  const uint32_t ls_step = static_cast<uint32_t>(lsum_plane) * 4u;
  int ue = PE + 1 - beta;  // exponent of unit_s
  int8_t* out = dst;
  for (int s = 1; s <= k; ++s, ue -= beta, out += plane, ls_addr += ls_step) {
    const uint32_t off = s == 1 ? o1 : os;
    const uint32_t off4 = off * 0x01010101u;
    uint32_t packed[4] = {off4, off4, off4, off4};  // zero line / underflowed grid: slice 0
    int qsum = 0;  // signed slice sum of this lane's elements (offset mode)
    if (!zero_line && ue >= -1074) {
      // sigma' = (1.5 * 2^52 + off) * 2^ue: exponent field ue + 1075, mantissa 0x8000000000000 + off
      const double sig = __hiloint2double(((ue + 1075) << 20) | 0x00080000, static_cast<int>(off));
      uint32_t q[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const double t = __dadd_rn(w[e], sig);
        const double x = __dadd_rn(t, -sig);
        q[e] = static_cast<uint32_t>(__double2loint(t));
        w[e] = __dadd_rn(w[e], -x);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t lo = __byte_perm(q[4 * i], q[4 * i + 1], 0x0040);
        const uint32_t hi = __byte_perm(q[4 * i + 2], q[4 * i + 3], 0x0040);
        packed[i] = __byte_perm(lo, hi, 0x5410);
      }
      if (lsum != nullptr) {
        if (part) {  // padding bytes stay 0
#pragma unroll
          for (int i = 0; i < 4; ++i) packed[i] &= keep[i];
        }
        uint32_t bsum = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) bsum = __dp4a(packed[i], 0x01010101u, bsum);
        qsum = static_cast<int>(bsum - off * nv);
      }
    } else {
      if (!zero_line) {
        // unit underflowed to 0: the reference computes x = w, int8(w/0) = 0
        // (cvttsd2si of +-inf/NaN), w -= x -> 0.
#pragma unroll
        for (int e = 0; e < 16; ++e) w[e] = __dadd_rn(w[e], -w[e]);
      }
      if (part) {
#pragma unroll
        for (int i = 0; i < 4; ++i) packed[i] &= keep[i];
      }
    }
    if (lsum != nullptr) {
      bool add;
      if constexpr (kLaneGroup == 32) {
        qsum = __reduce_add_sync(0xffffffffu, qsum);
        add = lead && qsum != 0;
      } else {
#pragma unroll
        for (int o = 32 / kLaneGroup; o < 32; o <<= 1) qsum += __shfl_xor_sync(0xffffffffu, qsum, o);
        add = lead && st && qsum != 0;
      }
      if (add) asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(ls_addr), "r"(qsum) : "memory");
    }
    if (st)
      *reinterpret_cast<uint4*>(out) = make_uint4(packed[0], packed[1], packed[2], packed[3]);
  }
}

// Number of valid elements in a 16-element run with `rest` elements left in the line.
__device__ __forceinline__ int valid16(int64_t rest) {
  return rest <= 0 ? 0 : (rest >= 16 ? 16 : static_cast<int>(rest));
}

__device__ __forceinline__ void load16(const double* x, int64_t base, int64_t len, bool vec,
                                       double (&w)[16]) {
  if (vec && base + 16 <= len) {
#pragma unroll
    for (int e = 0; e < 16; e += 2) {
      const double2 v = __ldg(reinterpret_cast<const double2*>(x + base + e));
      w[e] = v.x;
      w[e + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int e = 0; e < 16; ++e) w[e] = base + e < len ? __ldg(x + base + e) : 0.0;
  }
}

// Block-wide max of non-negative doubles (blockDim.x multiple of 32, <= 1024).
__device__ __forceinline__ double block_max(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  const int nw = blockDim.x >> 5;
  v = lane < nw ? red[lane] : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// One CTA per row.  X: rows x len (row stride ld doubles).  When the padded
// row fits 16 elements per thread (lds <= 16 * blockDim.x) the row is read
// from HBM exactly once and kept in registers between the max reduction and
// the slicing; longer rows take a second (L2-resident) pass.
template <bool kVec>
__global__ void __launch_bounds__(1024) slice_rows_kernel(const double* __restrict__ X, int64_t ld,
                                                          int64_t rows, int64_t len, int64_t lds,
                                                          int k, int beta,
                                                          int8_t* __restrict__ S, int64_t plane,
                                                          double* __restrict__ shift,
                                                          int* __restrict__ flags,
                                                          int* __restrict__ lsum, int64_t lsum_plane, int64_t lsum_lstride) {
  __shared__ double red[32];
  __shared__ int lsum_s[kMaxSlices];  // offset mode: the row's per-slice sums
  if (threadIdx.x < kMaxSlices) lsum_s[threadIdx.x] = 0;  // ordered by block_max's barrier
  const int64_t row = blockIdx.x;
  const double* x = X + row * ld;
  int8_t* out = S + row * lds;
  const int64_t step = 16 * static_cast<int64_t>(blockDim.x);
  const int64_t base0 = 16 * static_cast<int64_t>(threadIdx.x);
  double w[16];
  double rm = 0.0;
  if (lds <= step) {
    load16(x, base0, len, kVec, w);
#pragma unroll
    for (int e = 0; e < 16; ++e) rm = fmax(rm, fabs(w[e]));
  } else {
    for (int64_t base = base0; base < len; base += step) {
      load16(x, base, len, kVec, w);
#pragma unroll
      for (int e = 0; e < 16; ++e) rm = fmax(rm, fabs(w[e]));
    }
  }
  rm = block_max(rm, red);
  bool under = false, range = false;
  const int PE = line_pe(rm, beta, &under, &range);
  if (threadIdx.x == 0) {
    shift[row] = PE == INT32_MIN ? 0.0 : pow2(PE);
    report_flags(flags, under, range);
  }
  int* ls = lsum ? lsum_s : nullptr;
  auto nval = [&](int64_t base) { return valid16(len - base); };
  if (lds <= step) {
    if (ls)  // every lane takes part in the line-sum reduction
      emit16(w, PE, beta, k, out + base0, plane, nval(base0), base0 < lds, ls, 1);
    else if (base0 < lds)
      emit16(w, PE, beta, k, out + base0, plane);
  } else {
    for (int64_t it = 0; it * step < lds; ++it) {  // same trip count in every thread
      const int64_t base = base0 + it * step;
      load16(x, base, len, kVec, w);
      if (ls)
        emit16(w, PE, beta, k, out + base, plane, nval(base), base < lds, ls, 1);
      else if (base < lds)
        emit16(w, PE, beta, k, out + base, plane);
    }
  }
  if (lsum) {  // one CTA owns the row: plain stores
    __syncthreads();
    if (threadIdx.x < k) lsum[threadIdx.x * lsum_plane + row * lsum_lstride] = lsum_s[threadIdx.x];
  }
}

// Cluster variant: a row is split over the `csize` CTAs of a thread-block
// cluster (16 elements per thread, whole row in registers); the CTA maxima
// are exchanged through distributed shared memory.  Small CTAs let several
// rows share an SM, so one row's loads overlap another row's slicing.
template <bool kVec>
__global__ void __launch_bounds__(512) slice_rows_cluster_kernel(
    const double* __restrict__ X, int64_t ld, int64_t rows, int64_t len, int64_t lds, int k,
    int beta, int8_t* __restrict__ S, int64_t plane, double* __restrict__ shift,
    int* __restrict__ flags, int* __restrict__ lsum, int64_t lsum_plane, int64_t lsum_lstride) {
  __shared__ double red[32];
  __shared__ double cmax[8];  // one slot per CTA of the cluster
  __shared__ int lsum_s[kMaxSlices];  // offset mode: this CTA's part of the row sums
  if (threadIdx.x < kMaxSlices) lsum_s[threadIdx.x] = 0;  // ordered by block_max's barrier
  uint32_t crank, csize;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(csize));
  const int64_t row = blockIdx.x / csize;
  const double* x = X + row * ld;
  int8_t* out = S + row * lds;
  const int64_t base0 = 16 * (static_cast<int64_t>(crank) * blockDim.x + threadIdx.x);
  // every CTA of the cluster must be running before its shared memory is written
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  double w[16];
  load16(x, base0, len, kVec, w);
  double rm = 0.0;
#pragma unroll
  for (int e = 0; e < 16; ++e) rm = fmax(rm, fabs(w[e]));
  rm = block_max(rm, red);
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
  if (threadIdx.x < csize) {  // publish this CTA's max into every CTA's slot crank
    uint32_t local = static_cast<uint32_t>(__cvta_generic_to_shared(&cmax[crank]));
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(threadIdx.x));
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(remote), "d"(rm) : "memory");
  }
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  for (uint32_t c = 0; c < csize; ++c) rm = fmax(rm, cmax[c]);
  bool under = false, range = false;
  const int PE = line_pe(rm, beta, &under, &range);
  if (crank == 0 && threadIdx.x == 0) {
    shift[row] = PE == INT32_MIN ? 0.0 : pow2(PE);
    report_flags(flags, under, range);
  }
  if (lsum) {
    emit16(w, PE, beta, k, out + base0, plane, valid16(len - base0), base0 < lds, lsum_s, 1);
    __syncthreads();
    if (threadIdx.x < k && lsum_s[threadIdx.x] != 0)
      atomicAdd(lsum + threadIdx.x * lsum_plane + row * lsum_lstride, lsum_s[threadIdx.x]);
  } else if (base0 < lds) {
    emit16(w, PE, beta, k, out + base0, plane);
  }
}

// Column maxima of |X| for X: len x cols (row stride ld).  colmax holds the
// IEEE bit pattern of the max (must be zeroed first).  Block 32 x 8 threads.
__global__ void __launch_bounds__(256) colmax_kernel(const double* __restrict__ X, int64_t ld,
                                                     int64_t len, int64_t cols, int64_t rows_per_block,
                                                     unsigned long long* __restrict__ colmax) {
  __shared__ double red[8][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t col = static_cast<int64_t>(blockIdx.x) * 32 + tx;
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * rows_per_block;
  const int64_t r1 = min(len, r0 + rows_per_block);
  double m = 0.0;
  if (col < cols) {
    int64_t r = r0 + ty;
    for (; r + 56 < r1; r += 64) {  // 8 independent loads in flight per thread
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldg(X + (r + 8 * u) * ld + col);
#pragma unroll
      for (int u = 0; u < 8; ++u) m = fmax(m, fabs(v[u]));
    }
    for (; r < r1; r += 8) m = fmax(m, fabs(__ldg(X + r * ld + col)));
  }
  red[ty][tx] = m;
  __syncthreads();
  if (ty == 0) {
#pragma unroll
    for (int q = 1; q < 8; ++q) m = fmax(m, red[q][tx]);
    if (col < cols && m != 0.0)
      atomicMax(colmax + col, static_cast<unsigned long long>(__double_as_longlong(m)));
  }
}

// Slices of the columns of X (len x cols, row stride ld) written as the rows
// of the transposed planes S[s][col][0..lds).  A CTA of 8 warps covers 32
// columns x 128 rows; lane l of warp w owns column 4w + (l & 3) and the 16
// rows 16*(l >> 2) .. +16.  Each warp load then touches 8 fully used 32-byte
// sectors (4 adjacent columns x 8 rows) and, per slice, each column's 8
// chunks form one contiguous 128-byte line of the output plane.
//
// slice_cols_tile: the work of one CTA (tile bx of 32 columns, tile by of
// tiles_per_cta x 128 rows).
__device__ __forceinline__ void slice_cols_tile(const double* __restrict__ X, int64_t ld, int64_t len,
                                                int64_t cols, int64_t lds, int k, int beta,
                                                const unsigned long long* colmax, int8_t* __restrict__ S,
                                                int64_t plane, double* __restrict__ shift, int* __restrict__ flags,
                                                int* __restrict__ lsum, int64_t lsum_plane, int64_t lsum_lstride,
                                                int tiles_per_cta, int64_t bx, int64_t by, int (*lsum_s)[32]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t col = bx * 32 + warp * 4 + (lane & 3);
  auto cmax = [&](int64_t c) { return __longlong_as_double(static_cast<long long>(colmax[c])); };
  if (lsum == nullptr) {  // signed planes: one 128-row tile per CTA
    const int64_t base = by * 128 + 16 * (lane >> 2);
    if (col >= cols || base >= lds) return;
    const double rm = cmax(col);
    bool under = false, range = false;
    const int PE = line_pe(rm, beta, &under, &range);
    if (by == 0 && (lane >> 2) == 0) {
      shift[col] = PE == INT32_MIN ? 0.0 : pow2(PE);
      report_flags(flags, under, range);
    }
    double w[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) w[e] = base + e < len ? __ldg(X + (base + e) * ld + col) : 0.0;
    emit16(w, PE, beta, k, S + col * lds + base, plane);
    return;
  }
  // offset planes: `tiles_per_cta` 128-row tiles per CTA; the column sums
  // collect in shared memory and leave with one atomic per column and slice
  for (int i = threadIdx.x; i < kMaxSlices * 32; i += blockDim.x) lsum_s[i / 32][i % 32] = 0;
  __syncthreads();
  const double rm = col < cols ? cmax(col) : 0.0;
  bool under = false, range = false;
  const int PE = line_pe(rm, beta, &under, &range);
  if (col < cols && by == 0 && (lane >> 2) == 0) {
    shift[col] = PE == INT32_MIN ? 0.0 : pow2(PE);
    report_flags(flags, under, range);
  }
  for (int it = 0; it < tiles_per_cta; ++it) {  // uniform trip count: every lane reduces
    const int64_t base = (by * tiles_per_cta + it) * 128 + 16 * (lane >> 2);
    const bool valid = col < cols && base < lds;
    double w[16];
#pragma unroll
    for (int e = 0; e < 16; ++e)
      w[e] = valid && base + e < len ? __ldg(X + (base + e) * ld + col) : 0.0;
    emit16<8>(w, PE, beta, k, S + col * lds + base, plane, valid ? valid16(len - base) : 0, valid,
              &lsum_s[0][warp * 4 + (lane & 3)], 32);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < k * 32; i += blockDim.x) {
    const int64_t c = bx * 32 + (i % 32);
    if (c < cols && lsum_s[i / 32][i % 32] != 0)
      atomicAdd(lsum + (i / 32) * lsum_plane + c * lsum_lstride, lsum_s[i / 32][i % 32]);
  }
}

__global__ void __launch_bounds__(256) slice_cols_kernel(const double* __restrict__ X, int64_t ld,
                                                         int64_t len, int64_t cols, int64_t lds,
                                                         int k, int beta,
                                                         const unsigned long long* __restrict__ colmax,
                                                         int8_t* __restrict__ S, int64_t plane,
                                                         double* __restrict__ shift,
                                                         int* __restrict__ flags,
                                                         int* __restrict__ lsum, int64_t lsum_plane,
                                                         int64_t lsum_lstride, int tiles_per_cta) {
  __shared__ int lsum_s[kMaxSlices][32];
  slice_cols_tile(X, ld, len, cols, lds, k, beta, colmax, S, plane, shift, flags, lsum, lsum_plane,
                         lsum_lstride, tiles_per_cta, blockIdx.x, blockIdx.y, lsum_s);
}

// One-pass column split (K1 for columns of op(B), op(B) read from HBM ONCE).
// A thread-block cluster of up to 16 CTAs owns a strip of 8 columns over the
// whole column length: CTA r holds rows [r R, (r+1) R) of the strip in shared
// memory (R = 512 kU), brought in by 2-D TMA boxes of 256 rows x 8 columns
// (64 B per row, zero-filled past the matrix).  Pass 1 over shared memory takes
// the column maxima (lane shuffles, the 8 warps through shared memory, then the
// cluster's CTAs through distributed shared memory: every CTA stores its 8
// maxima into slot r of every CTA, double-buffered by strip parity, one cluster
// barrier per strip).  Pass 2 slices each thread's kU units of 16 rows x 1
// column straight out of shared memory with emit16.  Nothing is held in
// registers across the cluster barrier, so several CTAs share an SM and one's
// barrier and TMA latency hide behind another's slicing.  Columns longer than
// 16 x 1536 rows take the two-pass path (colmax_kernel + slice_cols_kernel).
constexpr int kOPCols = 8, kOPThreads = 256, kOPBox = 256;
template <int kU>
__global__ void __launch_bounds__(kOPThreads, 3) slice_cols_onepass_kernel(
    const __grid_constant__ CUtensorMap map_x, int64_t len, int64_t cols, int64_t lds, int k, int beta,
    int8_t* __restrict__ S, int64_t plane, double* __restrict__ shift, int* __restrict__ flags,
    int* __restrict__ lsum, int64_t lsum_plane, int64_t lsum_lstride) {
  constexpr int kR = 512 * kU;                            // rows per CTA
  constexpr uint32_t kBufBytes = kR * kOPCols * 8;        // this CTA's part of a strip
  extern __shared__ __align__(1024) uint8_t op_smem[];
  double* buf = reinterpret_cast<double*>(op_smem);       // [kR][8]
  uint64_t* full = reinterpret_cast<uint64_t*>(op_smem + kBufBytes);
  double* cmax = reinterpret_cast<double*>(full + 2);     // [2][16][8]: per parity, source CTA, column
  double* red = cmax + 2 * 16 * kOPCols;                  // [8 warps][8]
  int* lsum_s = reinterpret_cast<int*>(red + 8 * kOPCols);  // [kMaxSlices][8]
  const uint32_t crank = ptx::cluster_ctarank();
  uint32_t csize;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(csize));
  const int64_t ncl = gridDim.x / csize, cl = blockIdx.x / csize;
  const int64_t nstrips = (cols + kOPCols - 1) / kOPCols;
  const int64_t row0 = static_cast<int64_t>(crank) * kR;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = threadIdx.x & (kOPCols - 1);  // this thread's column in the strip
  if (threadIdx.x == 0) {
    ptx::tma_prefetch_desc(&map_x);
    ptx::mbar_init(full, 1);
    ptx::fence_barrier_init();
  }
  for (int i = threadIdx.x; i < kMaxSlices * kOPCols; i += kOPThreads) lsum_s[i] = 0;
  ptx::cluster_sync();  // barrier init visible; every CTA of the cluster is running (DSMEM)
  auto issue = [&](int64_t q) {
    ptx::mbar_arrive_expect_tx(full, kBufBytes);
    for (int j = 0; j < kR / kOPBox; ++j)
      ptx::tma_load_2d(buf + j * kOPBox * kOPCols, &map_x, full, static_cast<int32_t>(q * kOPCols),
                       static_cast<int32_t>(row0 + j * kOPBox));
  };
  if (threadIdx.x == 0 && cl < nstrips) issue(cl);
  int it = 0;
  for (int64_t q = cl; q < nstrips; q += ncl, ++it) {
    const int par = it & 1;
    const int64_t col = q * kOPCols + c;
    ptx::mbar_wait(full, it & 1);
    // pass 1: column maxima, read as 16-byte column pairs -- a warp reads 512
    // contiguous bytes per instruction (8 rows x 4 pairs), conflict-free
    {
      const int pr = lane & 3;  // column pair 2pr, 2pr + 1
      double m0 = 0.0, m1 = 0.0;
      const double2* b2 = reinterpret_cast<const double2*>(buf);
#pragma unroll 8
      for (int row = warp * 8 + (lane >> 2); row < kR; row += kOPThreads / 4) {
        const double2 v = b2[row * (kOPCols / 2) + pr];
        m0 = fmax(m0, fabs(v.x));
        m1 = fmax(m1, fabs(v.y));
      }
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        m0 = fmax(m0, __shfl_xor_sync(0xffffffffu, m0, o));
        m1 = fmax(m1, __shfl_xor_sync(0xffffffffu, m1, o));
      }
      if (lane < 4) {
        red[warp * kOPCols + 2 * pr] = m0;
        red[warp * kOPCols + 2 * pr + 1] = m1;
      }
    }
    __syncthreads();
    if (threadIdx.x < kOPCols) {
      double v = 0.0;
#pragma unroll
      for (int r = 0; r < kOPThreads / 32; ++r) v = fmax(v, red[r * kOPCols + threadIdx.x]);
      red[threadIdx.x] = v;  // row 0 of red: this CTA's maxima
    }
    __syncthreads();
    if (threadIdx.x < kOPCols * csize) {  // this CTA's maxima into slot crank of every CTA
      const int cc = threadIdx.x % kOPCols, dst = threadIdx.x / kOPCols;
      const uint32_t remote = ptx::mapa_shared(&cmax[(par * 16 + crank) * kOPCols + cc], dst);
      asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(remote), "d"(red[cc]) : "memory");
    }
    ptx::cluster_sync();
    double rm = 0.0;
    for (uint32_t r = 0; r < csize; ++r) rm = fmax(rm, cmax[(par * 16 + r) * kOPCols + c]);
    bool under = false, range = false;
    const int PE = line_pe(rm, beta, &under, &range);
    if (crank == 0 && threadIdx.x < kOPCols && col < cols) {
      shift[col] = PE == INT32_MIN ? 0.0 : pow2(PE);
      report_flags(flags, under, range);
    }
    // pass 2: slices
#pragma unroll 1
    for (int u = 0; u < kU; ++u) {
      const int chunk = (threadIdx.x + kOPThreads * u) >> 3;
      const int64_t base = row0 + chunk * 16;
      const bool valid = col < cols && base < lds;
      // the 4 lanes of a column sit on rows 16 apart (same banks): odd chunks read
      // their row pairs swapped so a warp load spans all 32 banks (2 wavefronts)
      double w[16];
      const bool odd = chunk & 1;
#pragma unroll
      for (int e = 0; e < 16; e += 2) {
        const double x0 = buf[(chunk * 16 + e + (odd ? 1 : 0)) * kOPCols + c];
        const double x1 = buf[(chunk * 16 + e + (odd ? 0 : 1)) * kOPCols + c];
        w[e] = odd ? x1 : x0;
        w[e + 1] = odd ? x0 : x1;
      }
      if (lsum)  // every lane takes part in the column-sum reduction (4 lanes per column)
        emit16<4>(w, PE, beta, k, S + col * lds + base, plane, valid ? valid16(len - base) : 0, valid,
                  lsum_s + c, kOPCols);
      else if (valid)
        emit16<4>(w, PE, beta, k, S + col * lds + base, plane);
    }
    __syncthreads();  // the strip buffer is free: fetch the next one while the sums leave
    if (threadIdx.x == 0 && q + ncl < nstrips) issue(q + ncl);
    if (lsum) {
      for (int i = threadIdx.x; i < k * kOPCols; i += kOPThreads) {
        const int64_t cg = q * kOPCols + (i % kOPCols);
        const int v = lsum_s[i];
        if (cg < cols && v != 0) atomicAdd(lsum + (i / kOPCols) * lsum_plane + cg * lsum_lstride, v);
        lsum_s[i] = 0;
      }
      __syncthreads();
    }
  }
  ptx::cluster_sync();  // no CTA leaves while a peer may still address its shared memory
}

}  // namespace ozb
