// Host-side input generator: the reference's phi test matrices, shardable.
//
// Restates gen_phi_matrix (proj/src/generate.cpp:11-29) with counter_hash /
// uniform_open (proj/include/ozmm/generate.hpp:11-21): entry idx = i*cols + j
// of the GLOBAL rows x cols matrix is (U - 0.5) * exp(phi * N), U and N drawn
// from counters 3*idx, 3*idx+1, 3*idx+2.  Because every entry depends only on
// its own counter, any block of the matrix can be generated on any rank --
// bench.py and the multi-GPU path use this to build each rank's shard.
// Compiled by g++ with -ffp-contract=off and linked against the same libm as
// the reference, so values are bit-identical to the reference generator
// (checked by tests/test_host_logic.py against the reference build).
// Not on the hot path: inputs are made on the host, as the reference does.
#include <cmath>
#include <cstdint>

#include "../../include/ozmm_b200.h"

extern "C" {

uint64_t ozmm_counter_hash(uint64_t seed, uint64_t ctr) {
  uint64_t z = seed + ctr * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

int ozmm_gen_phi_block(int64_t rows, int64_t cols, double phi, uint64_t seed, int64_t row0,
                       int64_t nrows, int64_t col0, int64_t ncols, double* out, int64_t ldo) {
  if (rows < 1 || cols < 1) return OZMM_ERR_ARG;
  if (!(phi >= 0)) return OZMM_ERR_ARG;
  if (row0 < 0 || col0 < 0 || nrows < 0 || ncols < 0 || row0 + nrows > rows ||
      col0 + ncols > cols || ldo < ncols)
    return OZMM_ERR_ARG;
  const double pi = 3.141592653589793;  // std::numbers::pi
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < nrows; ++i) {
    for (int64_t j = 0; j < ncols; ++j) {
      const uint64_t idx = static_cast<uint64_t>((row0 + i) * cols + (col0 + j));
      const uint64_t ctr = idx * 3;
      const double u = static_cast<double>((ozmm_counter_hash(seed, ctr) >> 11) | 1ull) * 0x1p-53;
      const double u1 =
          static_cast<double>((ozmm_counter_hash(seed, ctr + 1) >> 11) | 1ull) * 0x1p-53;
      const double u2 =
          static_cast<double>((ozmm_counter_hash(seed, ctr + 2) >> 11) | 1ull) * 0x1p-53;
      const double normal = std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * pi * u2);
      out[i * ldo + j] = (u - 0.5) * std::exp(phi * normal);
    }
  }
  return OZMM_OK;
}

}  // extern "C"
