// ozmm::gpu -- header-only C++ adapter with the REFERENCE's operator API over
// the B200 C ABI (include/ozmm_b200.h).
//
// Drop-in for (proj/include/ozmm/scheme.hpp):
//   MatrixF64   ozaki_gemm   (double alpha, const MatrixF64& a, const MatrixF64& b,
//                             double beta, const MatrixF64& c, const SchemeConfig& cfg);  :92-95
//   OzakiResult ozaki_gemm_ex(...same...);                                                :96-98
//   OzakiResult ozaki_mm     (const MatrixF64& a, const MatrixF64& b, const SchemeConfig&); :89-90
// and for the splitters (proj/include/ozmm/split.hpp:61-74), filling the
// reference's SplitMatrix (or any type with its members):
//   split<SplitMatrix>(a, k, side, strategy [, forced_beta])  -- split_bitmask /
//   split_round_nearest / split_rn_const_shift, slices + shifts (or per-slice
//   units) + residual + underflow flag, computed on the GPU (ozmm_split_host)
// for every valid SchemeConfig: the (strategy, accumulation) pair selects the
// GPU method -- ozIMMU_H (the hot path), ozIMMU, ozIMMU_RN, ozIMMU_EF and the two
// other valid pairs -- and overflow / force_beta / force_r are honoured
// (scheme.hpp:24-31, scheme.cpp:137-174).
//
// Templated over the matrix type: anything row-major with rows(), cols(),
// data() and a (rows, cols) constructor -- the reference's
// ozmm::DenseMatrix<double> (Eigen RowMajor, types.hpp:13-16) included -- so
// the reference CLI/harness can switch by changing a namespace.  Same
// semantics as the reference: inputs are const, a NEW matrix is returned
// (scheme.cpp:281, :289), errors are thrown as the reference's exception
// types (std::invalid_argument, a ConfigError-compatible invalid_argument,
// std::overflow_error for rows >= 2^921, an OverflowError runtime_error for an
// INT32 chunk overflow in OverflowMode::Checked, int_gemm.hpp:15-26).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/ozmm_b200.h"

namespace ozmm {
namespace gpu {

struct ConfigError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
// INT32 chunk overflow in OverflowMode::Checked (int_gemm.hpp:15-26)
struct OverflowError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct OpCounts {
  std::int64_t int8_gemms = 0, fp64_flushes = 0, r = 0, w = 0;
};
struct PhaseTimings {
  double split_a = 0, split_b = 0, int_gemm = 0, accum_fp64 = 0, copy = 0;
};
template <class Mat>
struct OzakiResultT {
  Mat d;
  OpCounts counts;
  PhaseTimings timings;
};

// The reference SchemeConfig (scheme.hpp:24-31) as the C ABI's options.
struct GpuConfig {
  int k = 8;
  int method = OZMM_METHOD_OZIMMU_H;
  int overflow_wrap = 0;  // OverflowMode::Checked (the reference's default)
  int force_beta = 0;
  std::int64_t force_r = 0;
};

// (SliceStrategy, Accumulation) -> OZMM_METHOD_*.  Enum orders of the reference:
// SliceStrategy {BitMask, RoundNearestPerSlice, RoundNearestConstShift}
// (split.hpp:11-15), Accumulation {PerProduct, Groupwise, GroupwiseSimple}
// (scheme.hpp:13-17).  The one invalid pair -- per-slice RN with group-wise
// accumulation -- is the reference's ConfigError (validate_config, scheme.cpp:164-168).
inline int method_code(int strategy, int accumulation) {
  switch (strategy * 3 + accumulation) {
    case 2 * 3 + 1: return OZMM_METHOD_OZIMMU_H;
    case 0 * 3 + 0: return OZMM_METHOD_OZIMMU;
    case 1 * 3 + 0: return OZMM_METHOD_OZIMMU_RN;
    case 0 * 3 + 1: return OZMM_METHOD_OZIMMU_EF;
    case 2 * 3 + 0: return OZMM_METHOD_RN_CONST_PER_PRODUCT;
    case 2 * 3 + 2: return OZMM_METHOD_OZIMMU_H_SIMPLE;
    case 0 * 3 + 2: return OZMM_METHOD_OZIMMU_EF_SIMPLE;
    case 1 * 3 + 1:
    case 1 * 3 + 2:
      throw ConfigError(
          "per-slice round-to-nearest shifts are only valid with per-product accumulation");
    default: throw ConfigError("unknown slice strategy / accumulation");
  }
}

// Accept the reference's SchemeConfig (k, strategy, accumulation, overflow,
// force_beta, force_r; enum class members).
template <class Cfg>
GpuConfig to_gpu_config(const Cfg& cfg) {
  GpuConfig g;
  g.k = cfg.k;
  g.method = method_code(static_cast<int>(cfg.strategy), static_cast<int>(cfg.accumulation));
  g.overflow_wrap = static_cast<int>(cfg.overflow);  // OverflowMode {Checked, Wrapping}
  g.force_beta = cfg.force_beta;
  g.force_r = static_cast<std::int64_t>(cfg.force_r);
  return g;
}
inline GpuConfig to_gpu_config(const GpuConfig& cfg) { return cfg; }

// One handle per host thread, created on first use (device 0 or OZMM_DEVICE).
inline ozmm_handle_t thread_handle() {
  thread_local struct Owner {
    ozmm_handle_t h = nullptr;
    ~Owner() {
      if (h) ozmm_destroy(h);
    }
  } owner;
  if (!owner.h) {
    int dev = 0;
    if (const char* s = std::getenv("OZMM_DEVICE")) dev = std::atoi(s);
    if (int rc = ozmm_create(&owner.h, dev))
      throw std::runtime_error(std::string("ozmm_create: ") + ozmm_last_error(nullptr) + " (" +
                               ozmm_status_string(rc) + ")");
  }
  return owner.h;
}

inline void throw_status(int rc, ozmm_handle_t h) {
  const std::string msg = ozmm_last_error(h);
  switch (rc) {
    case OZMM_OK: return;
    case OZMM_ERR_ARG: throw std::invalid_argument(msg);
    case OZMM_ERR_CONFIG: throw ConfigError(msg);
    case OZMM_ERR_RANGE: throw std::overflow_error(msg);
    case OZMM_ERR_OVERFLOW: throw OverflowError(msg);
    default: throw std::runtime_error(msg + " (" + ozmm_status_string(rc) + ")");
  }
}

template <class Mat, class Cfg>
OzakiResultT<Mat> ozaki_gemm_ex(double alpha, const Mat& a, const Mat& b, double beta,
                                const Mat& c, const Cfg& cfg_in) {
  const GpuConfig cfg = to_gpu_config(cfg_in);
  if (a.cols() != b.rows()) throw std::invalid_argument("ozaki_mm: inner dimensions differ");
  if (c.rows() != a.rows() || c.cols() != b.cols())
    throw std::invalid_argument("ozaki_gemm: C shape mismatch");
  if (cfg.k < 1) throw ConfigError("k must be >= 1");
  const std::int64_t m = a.rows(), n = a.cols(), p = b.cols();
  Mat out(c.rows(), c.cols());  // the new result matrix: C is only read (scheme.cpp:281, :289)
  ozmm_options_t opt{};
  opt.method = cfg.method;
  opt.overflow_wrap = cfg.overflow_wrap;
  opt.force_beta = cfg.force_beta;
  opt.force_r = cfg.force_r;
  opt.timings = 1;
  ozmm_counts_t cnt{};
  ozmm_timings_t tim{};
  ozmm_handle_t h = thread_handle();
  throw_status(ozmm_dgemm_host_out(h, 'N', 'N', m, n, p, alpha, a.data(), n, b.data(), p, beta,
                                   c.data(), p, out.data(), p, cfg.k, &opt, &cnt, &tim),
               h);
  OzakiResultT<Mat> res{std::move(out), {}, {}};
  res.counts = {cnt.int8_gemms, cnt.fp64_flushes, cnt.r, cnt.w};
  res.timings = {tim.split_a, tim.split_b, tim.int_gemm, tim.accum_fp64, tim.copy};
  return res;
}

template <class Mat, class Cfg>
Mat ozaki_gemm(double alpha, const Mat& a, const Mat& b, double beta, const Mat& c,
               const Cfg& cfg) {
  return ozaki_gemm_ex(alpha, a, b, beta, c, cfg).d;
}

template <class Mat, class Cfg>
OzakiResultT<Mat> ozaki_mm(const Mat& a, const Mat& b, const Cfg& cfg) {
  Mat zero(a.rows(), b.cols());
  std::fill(zero.data(), zero.data() + a.rows() * b.cols(), 0.0);
  return ozaki_gemm_ex(1.0, a, b, 0.0, zero, cfg);
}

// The reference's splitters on the GPU (split.hpp:61-74): Split is the caller's
// SplitMatrix type (split.hpp:31-50); side / strategy are its Side {Left, Right}
// and SliceStrategy {BitMask, RoundNearestPerSlice, RoundNearestConstShift}.
// Fills side, k, beta, strategy, slices (the matrix's own layout), const_shift
// (const-shift strategies) or slice_units (per-slice RN), residual and
// underflow_flagged exactly as the reference's split_any does (split.cpp:182-198).
template <class Split, class Mat, class SideT, class StrategyT>
Split split(const Mat& a, int k, SideT side, StrategyT strategy, int forced_beta = 0) {
  if (k < 1) throw std::invalid_argument("split: k must be >= 1");
  const int sd = static_cast<int>(side), st = static_cast<int>(strategy);
  const int code = st == 0 ? OZMM_SPLIT_BITMASK : (st == 1 ? OZMM_SPLIT_RN_PER_SLICE : OZMM_SPLIT_RN_CONST_SHIFT);
  const std::int64_t rows = a.rows(), cols = a.cols();
  const std::int64_t lines = sd == 0 ? rows : cols, n = sd == 0 ? cols : rows;
  std::vector<std::int8_t> sl(static_cast<size_t>(k * lines * n));
  std::vector<double> out(static_cast<size_t>(st == 1 ? k * lines : lines));
  std::vector<double> res(static_cast<size_t>(lines * n));
  ozmm_handle_t h = thread_handle();
  int pending_under = 0;
  ozmm_sync_status(h, &pending_under);  // start from clear flags (this call's underflow only)
  throw_status(ozmm_split_host(h, sd == 0 ? 'L' : 'R', 'N', lines, n, a.data(), cols, k, forced_beta, code,
                               sl.data(), out.data(), res.data()),
               h);
  int under = 0;
  throw_status(ozmm_sync_status(h, &under), h);
  int beta = forced_beta;
  if (!beta) throw_status(ozmm_compute_beta(n, &beta), nullptr);
  Split s;
  s.side = side;
  s.k = k;
  s.beta = beta;
  s.strategy = strategy;
  using MatI8 = typename decltype(s.slices)::value_type;
  using Vec = decltype(s.const_shift);
  // line-major [lines][n] -> the matrix's own rows x cols (Right: transposed back)
  auto at = [&](std::int64_t i, std::int64_t j) { return sd == 0 ? i * n + j : j * n + i; };
  for (int t = 0; t < k; ++t) {
    MatI8 m(rows, cols);
    const std::int8_t* src = sl.data() + static_cast<size_t>(t) * lines * n;
    for (std::int64_t i = 0; i < rows; ++i)
      for (std::int64_t j = 0; j < cols; ++j) m.data()[i * cols + j] = src[at(i, j)];
    s.slices.push_back(std::move(m));
  }
  if (st == 1) {
    for (int t = 0; t < k; ++t) {
      Vec v(lines);
      for (std::int64_t i = 0; i < lines; ++i) v.data()[i] = out[t * lines + i];
      s.slice_units.push_back(std::move(v));
    }
  } else {
    Vec v(lines);
    for (std::int64_t i = 0; i < lines; ++i) v.data()[i] = out[i];
    s.const_shift = std::move(v);
  }
  decltype(s.residual) r(rows, cols);
  for (std::int64_t i = 0; i < rows; ++i)
    for (std::int64_t j = 0; j < cols; ++j) r.data()[i * cols + j] = res[at(i, j)];
  s.residual = std::move(r);
  s.underflow_flagged = under != 0;
  return s;
}

}  // namespace gpu
}  // namespace ozmm
