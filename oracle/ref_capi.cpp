// extern "C" wrapper over the UNMODIFIED reference library -- TEST
// INFRASTRUCTURE ONLY (parity checker + CPU baseline arm of bench.py).
//
// Built by oracle/Makefile from the sources under /root/reference/proj/src
// (compiled in place, never copied) into oracle/_ref/libozmm_ref.so.  Every
// function forwards to the reference's own public API:
//   ozaki_gemm_ex       proj/include/ozmm/scheme.hpp:96-98  (scheme.cpp:274-291)
//   config_for          proj/src/scheme.cpp:137-159
//   split_rn_const_shift proj/src/split.cpp:233-237
//   i8_gemm_accumulate  proj/src/int_gemm.cpp:248-251
//   compute_beta/compute_r/op_counts_with_r  split.cpp:211, int_gemm.cpp:253, scheme.cpp:176
//   gen_phi_matrix      proj/src/generate.cpp:11-29
//   exact_gemm_oracle / fp64_gemm_reference / max_rel_err  proj/src/oracle.cpp:276-335
// Exceptions never cross this boundary: they become status codes plus a
// thread-local message, mirroring the GPU library's error convention.
#include "ozmm/analysis.hpp"
#include "ozmm/generate.hpp"
#include "ozmm/int_gemm.hpp"
#include "ozmm/oracle.hpp"
#include "ozmm/parallel.hpp"
#include "ozmm/scheme.hpp"
#include "ozmm/split.hpp"

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>

using namespace ozmm;

namespace {

thread_local std::string g_err;

enum : int {
  kOk = 0,
  kErrArg = 1,      // std::invalid_argument (shapes, k, n range)
  kErrConfig = 2,   // ConfigError
  kErrRange = 3,    // std::overflow_error (row magnitude >= 2^921)
  kErrOverflow = 4, // OverflowError (INT32 chunk overflow in Checked mode)
  kErrOther = 9,
};

template <class F>
int guard(F&& f) {
  try {
    f();
    return kOk;
  } catch (const OverflowError& e) {
    g_err = e.what();
    return kErrOverflow;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return kErrConfig;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return kErrArg;
  } catch (const std::overflow_error& e) {
    g_err = e.what();
    return kErrRange;
  } catch (const std::exception& e) {
    g_err = e.what();
    return kErrOther;
  }
}

MatrixF64 load(const double* p, std::int64_t r, std::int64_t c) {
  MatrixF64 m(r, c);
  std::memcpy(m.data(), p, sizeof(double) * r * c);
  return m;
}

Method method_of(int code) {
  switch (code) {
    case 0: return Method::ozIMMU;
    case 1: return Method::ozIMMU_RN;
    case 2: return Method::ozIMMU_EF;
    default: return Method::ozIMMU_H;
  }
}

}  // namespace

extern "C" {

const char* ozref_last_error() { return g_err.c_str(); }

void ozref_set_threads(int n) { set_thread_count(n); }
int ozref_thread_count() { return thread_count(); }

int ozref_compute_beta(std::int64_t n, int* out) {
  return guard([&] { *out = compute_beta(n); });
}

int ozref_compute_r(std::int64_t n, int beta, std::int64_t* out) {
  return guard([&] { *out = compute_r(n, beta); });
}

// counts = {int8_gemms, fp64_flushes, r, w}
int ozref_op_counts_with_r(int k, std::int64_t r, int accumulation, std::int64_t* counts) {
  return guard([&] {
    const OpCounts c = op_counts_with_r(k, r, static_cast<Accumulation>(accumulation));
    counts[0] = c.int8_gemms;
    counts[1] = c.fp64_flushes;
    counts[2] = c.r;
    counts[3] = c.w;
  });
}

std::uint64_t ozref_counter_hash(std::uint64_t seed, std::uint64_t ctr) {
  return counter_hash(seed, ctr);
}

int ozref_gen_phi_matrix(std::int64_t m, std::int64_t n, double phi, std::uint64_t seed,
                         double* out) {
  return guard([&] {
    const MatrixF64 a = gen_phi_matrix(m, n, phi, seed);
    std::memcpy(out, a.data(), sizeof(double) * m * n);
  });
}

// out = ozaki_gemm_ex(alpha, A(m x n), B(n x p), beta, C(m x p), cfg).
// counts = {int8_gemms, fp64_flushes, r, w}; timings = {split_a, split_b,
// int_gemm, accum_fp64, copy} seconds.  Either may be null.
int ozref_gemm(int method, int k, int force_beta, std::int64_t force_r, int overflow_mode,
               double alpha, const double* a, std::int64_t m, std::int64_t n,
               const double* b, std::int64_t p, double beta, const double* c,
               double* out, std::int64_t* counts, double* timings) {
  return guard([&] {
    SchemeConfig cfg = config_for(method_of(method), k);
    cfg.force_beta = force_beta;
    cfg.force_r = force_r;
    cfg.overflow = overflow_mode ? OverflowMode::Wrapping : OverflowMode::Checked;
    const MatrixF64 A = load(a, m, n), B = load(b, n, p), C = load(c, m, p);
    const OzakiResult res = ozaki_gemm_ex(alpha, A, B, beta, C, cfg);
    std::memcpy(out, res.d.data(), sizeof(double) * m * p);
    if (counts) {
      counts[0] = res.counts.int8_gemms;
      counts[1] = res.counts.fp64_flushes;
      counts[2] = res.counts.r;
      counts[3] = res.counts.w;
    }
    if (timings) {
      timings[0] = res.timings.split_a;
      timings[1] = res.timings.split_b;
      timings[2] = res.timings.int_gemm;
      timings[3] = res.timings.accum_fp64;
      timings[4] = res.timings.copy;
    }
  });
}

// RN constant-shift split of a rows x cols matrix.  side 0 = Left (row-wise
// scaling), 1 = Right (column-wise).  slices: k x rows x cols int8 in the
// matrix's own row-major layout; shift: rows (Left) or cols (Right) doubles.
int ozref_split_rn_const_shift(const double* a, std::int64_t rows, std::int64_t cols, int k,
                               int side, int force_beta, std::int8_t* slices, double* shift,
                               double* residual, int* beta_out, int* underflow) {
  return guard([&] {
    const MatrixF64 A = load(a, rows, cols);
    const SplitMatrix s =
        split_rn_const_shift(A, k, side ? Side::Right : Side::Left, force_beta);
    for (int t = 0; t < k; ++t)
      std::memcpy(slices + static_cast<std::int64_t>(t) * rows * cols, s.slices[t].data(),
                  static_cast<std::size_t>(rows * cols));
    std::memcpy(shift, s.const_shift.data(), sizeof(double) * s.const_shift.size());
    if (residual) std::memcpy(residual, s.residual.data(), sizeof(double) * rows * cols);
    if (beta_out) *beta_out = s.beta;
    if (underflow) *underflow = s.underflow_flagged ? 1 : 0;
  });
}

// Any splitting strategy: 0 = RN const shift, 1 = bitmask, 2 = RN per slice
// (split.cpp:223-237).  out: const shift [rows or cols] (0, 1) or per-slice
// units [k][rows or cols] (2); residual (nullable): rows x cols.
int ozref_split_any(int strategy, const double* a, std::int64_t rows, std::int64_t cols, int k,
                    int side, int force_beta, std::int8_t* slices, double* out, double* residual) {
  return guard([&] {
    const MatrixF64 A = load(a, rows, cols);
    const Side sd = side ? Side::Right : Side::Left;
    const SplitMatrix s = strategy == 1   ? split_bitmask(A, k, sd, force_beta)
                          : strategy == 2 ? split_round_nearest(A, k, sd, force_beta)
                                          : split_rn_const_shift(A, k, sd, force_beta);
    for (int t = 0; t < k; ++t)
      std::memcpy(slices + static_cast<std::int64_t>(t) * rows * cols, s.slices[t].data(),
                  static_cast<std::size_t>(rows * cols));
    if (strategy == 2) {
      const std::int64_t lines = side ? cols : rows;
      for (int t = 0; t < k; ++t)
        std::memcpy(out + t * lines, s.slice_units[t].data(), sizeof(double) * lines);
    } else {
      std::memcpy(out, s.const_shift.data(), sizeof(double) * s.const_shift.size());
    }
    // SplitMatrix::residual in the matrix's own layout (dump_split, split.cpp:269)
    if (residual) std::memcpy(residual, s.residual.data(), sizeof(double) * rows * cols);
  });
}

// The INT32 chunk sums of the ozIMMU_H group-wise schedule, in flush order,
// produced by the reference's own splitter and i8_gemm_accumulate following
// the loop of groupwise_impl (scheme.cpp:81-101).  acc_out receives w
// matrices m x p; chunk_g/chunk_s0/chunk_s1 (length w) describe each chunk.
int ozref_groupwise_chunks(const double* a, std::int64_t m, std::int64_t n, const double* b,
                           std::int64_t p, int k, int force_beta, std::int64_t force_r,
                           std::int32_t* acc_out, int* chunk_g, int* chunk_s0,
                           int* chunk_s1, std::int64_t* w_out) {
  return guard([&] {
    const MatrixF64 A = load(a, m, n), B = load(b, n, p);
    const SplitMatrix sa = split_rn_const_shift(A, k, Side::Left, force_beta);
    const SplitMatrix sb = split_rn_const_shift(B, k, Side::Right, force_beta);
    const std::int64_t r = force_r ? force_r : compute_r(n, sa.beta);
    std::int64_t w = 0;
    for (int g = 2; g <= k + 1; ++g) {
      MatrixI32 acc = MatrixI32::Zero(m, p);
      std::int64_t q = 0;
      int s0 = 1;
      for (int s = 1; s <= g - 1; ++s) {
        ++q;
        acc = i8_gemm_accumulate(acc, sa.slices[s - 1], sb.slices[g - s - 1],
                                 OverflowMode::Checked);
        const bool group_done = s == g - 1;
        if (q == r || group_done) {
          std::memcpy(acc_out + w * m * p, acc.data(), sizeof(std::int32_t) * m * p);
          chunk_g[w] = g;
          chunk_s0[w] = s0;
          chunk_s1[w] = s;
          ++w;
          q = 0;
          s0 = s + 1;
          if (!group_done) acc.setZero();
        }
      }
    }
    *w_out = w;
  });
}

// total_bound (analysis.cpp:73-100) of ozaki_mm(A, B, config_for(method, k))
// with |A||B| from exact_gemm_oracle(|A|, |B|), as verify_bounds does
// (harness.cpp:156-157).  out: m x p elementwise bound.
int ozref_total_bound(int method, int k, int force_beta, std::int64_t force_r, const double* a,
                      std::int64_t m, std::int64_t n, const double* b, std::int64_t p,
                      double* out) {
  return guard([&] {
    SchemeConfig cfg = config_for(method_of(method), k);
    cfg.force_beta = force_beta;
    cfg.force_r = force_r;
    const MatrixF64 A = load(a, m, n), B = load(b, n, p);
    const MatrixF64 absAB = exact_gemm_oracle(A.cwiseAbs(), B.cwiseAbs());
    const ErrorBundle eb = total_bound(A, B, cfg, absAB);
    std::memcpy(out, eb.total_bound.data(), sizeof(double) * m * p);
  });
}

int ozref_exact_gemm(const double* a, std::int64_t m, std::int64_t n, const double* b,
                     std::int64_t p, double* out) {
  return guard([&] {
    const MatrixF64 r = exact_gemm_oracle(load(a, m, n), load(b, n, p));
    std::memcpy(out, r.data(), sizeof(double) * m * p);
  });
}

int ozref_fp64_gemm(const double* a, std::int64_t m, std::int64_t n, const double* b,
                    std::int64_t p, double* out) {
  return guard([&] {
    const MatrixF64 r = fp64_gemm_reference(load(a, m, n), load(b, n, p));
    std::memcpy(out, r.data(), sizeof(double) * m * p);
  });
}

int ozref_max_rel_err(const double* t, const double* r, std::int64_t m, std::int64_t p,
                      double* out) {
  return guard([&] { *out = max_rel_err(load(t, m, p), load(r, m, p)); });
}

}  // extern "C"
