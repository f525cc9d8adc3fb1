// Bit-exact FP64 helpers shared by the slicer and the GEMM epilogue.
//
// Every rounded FP64 operation on the ozIMMU_H path is written with an
// explicit _rn intrinsic so nvcc can neither contract a*b+c into an FMA nor
// reorder: this is the GPU form of the reference's -ffp-contract=off rule
// (proj/src/CMakeLists.txt:18-20).
#pragma once

#include <cstdint>

namespace ozb {

// 2^e as a double, exactly as std::ldexp(1.0, e) rounds it: normal for
// e >= -1022, subnormal down to 2^-1074, 0 below (2^-1075 is a tie that rounds
// to even = 0), +inf above 1023.
// Slice offsets of the offset-binary planes: o_1 = 2^beta, o_s = max(2, 2^(beta-1))
// for s >= 2 -- both EVEN, see emit16 -- so every byte slice + o_s lies in
// [0, 255]: slice 1 + o_1 in [1, 2^(beta+1) - 1] (|slice_1| <= 2^beta - 1 by
// rn_unit's bump rule), slice s + o_s in [0, 2^beta] (|slice_s| <= 2^(beta-1)
// after round-to-nearest).
__host__ __device__ __forceinline__ uint32_t slice_offset(int s, int beta) {
  return s == 1 ? (1u << beta) : (beta >= 2 ? 1u << (beta - 1) : 2u);
}

__host__ __device__ __forceinline__ double pow2(int e) {
  uint64_t bits;
  if (e >= -1022) {
    if (e > 1023) bits = 0x7FF0000000000000ull;
    else bits = static_cast<uint64_t>(e + 1023) << 52;
  } else if (e >= -1074) {
    bits = 1ull << (e + 1074);
  } else {
    bits = 0;
  }
#ifdef __CUDA_ARCH__
  return __longlong_as_double(static_cast<long long>(bits));
#else
  double d;
  __builtin_memcpy(&d, &bits, 8);
  return d;
#endif
}

// ufp_exponent (proj/include/ozmm/ufp.hpp:35-41): e with 2^e <= |c| < 2^(e+1),
// subnormals via the position of the top set bit.  c must be finite, nonzero.
__device__ __forceinline__ int ufp_exponent(double c) {
  const uint64_t b = static_cast<uint64_t>(__double_as_longlong(c)) & 0x7FFFFFFFFFFFFFFFull;
  const int biased = static_cast<int>(b >> 52);
  if (biased > 0) return biased - 1023;
  return (63 - __clzll(static_cast<long long>(b))) - 1074;
}

// Per-line splitting parameters of rn_const_shift_rows / rn_unit
// (proj/src/split.cpp:121-130, :158-166) for line max `rm`:
//   pe0 = ufp_exponent(rm); bump if rm >= (2 - 2^-beta) * 2^pe0;
//   PE = pe0 + bump; const_shift = 2^PE; unit_s = 2^(PE + 1 - beta*s).
// Returns PE, or INT32_MIN for a zero line.  *range set when pe0 > 920,
// *under when pe0 < -1000.
__device__ __forceinline__ int line_pe(double rm, int beta, bool* under, bool* range) {
  if (rm == 0.0) return INT32_MIN;
  const int pe0 = ufp_exponent(rm);
  if (pe0 < -1000) *under = true;
  if (pe0 > 920) *range = true;
  const double threshold = __dmul_rn(2.0 - pow2(-beta), pow2(pe0));  // == ldexp(2-2^-b, pe0)
  return pe0 + (rm >= threshold ? 1 : 0);
}

}  // namespace ozb
