// Drop-in demonstration (TEST INFRASTRUCTURE): the same call site with the
// reference's ozmm::ozaki_gemm_ex (CPU, from oracle/_ref/libozmm_ref.so -- the
// unmodified reference sources) and ozmm::gpu::ozaki_gemm_ex (B200, through
// the C ABI).  Built by tests/test_dropin_cpp.py against the reference headers
// and the Eigen shim; prints "MATCH <n>" when every entry is bitwise equal.
//
//   dropin_demo <m> <n> <p> <k> <phi> [method] [--closed-forms-only]
//   method: ozIMMU_H (default) | ozIMMU | ozIMMU_RN | ozIMMU_EF -- the
//   reference's config_for preset, passed unchanged to both calls; or
//   "overflow <force_r>": ozIMMU_H with force_r on INT32-overflowing inputs:
//   Wrapping bit-identical on both sides, Checked throws on the GPU side
//   (prints "OVERFLOW-OK");
//   "split": the reference's split_bitmask / split_round_nearest /
//   split_rn_const_shift of A (Left) and B (Right) against ozmm::gpu::split
//   into the reference's own SplitMatrix type (prints "SPLIT-OK").
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "ozmm/generate.hpp"
#include "ozmm/scheme.hpp"
#include "ozmm/split.hpp"
#include "ozmm_gpu.hpp"

// bitwise equality of two reference SplitMatrix objects
static bool same_split(const ozmm::SplitMatrix& x, const ozmm::SplitMatrix& y) {
  auto eq = [](const void* a, const void* b, size_t bytes) { return std::memcmp(a, b, bytes) == 0; };
  if (x.side != y.side || x.k != y.k || x.beta != y.beta || x.strategy != y.strategy ||
      x.underflow_flagged != y.underflow_flagged || x.slices.size() != y.slices.size() ||
      x.slice_units.size() != y.slice_units.size() || x.const_shift.size() != y.const_shift.size())
    return false;
  const size_t cells = static_cast<size_t>(x.residual.rows() * x.residual.cols());
  for (size_t t = 0; t < x.slices.size(); ++t)
    if (!eq(x.slices[t].data(), y.slices[t].data(), cells)) return false;
  for (size_t t = 0; t < x.slice_units.size(); ++t)
    if (!eq(x.slice_units[t].data(), y.slice_units[t].data(), sizeof(double) * x.slice_units[t].size()))
      return false;
  return eq(x.const_shift.data(), y.const_shift.data(), sizeof(double) * x.const_shift.size()) &&
         eq(x.residual.data(), y.residual.data(), sizeof(double) * cells);
}

int main(int argc, char** argv) {
  if (argc < 6) return 2;
  const long m = std::atol(argv[1]), n = std::atol(argv[2]), p = std::atol(argv[3]);
  const int k = std::atoi(argv[4]);
  const double phi = std::atof(argv[5]);
  // closed forms agree (no GPU needed)
  int beta = 0;
  std::int64_t r = 0;
  ozmm_compute_beta(n, &beta);
  ozmm_compute_r(n, beta, &r);
  if (beta != ozmm::compute_beta(n) || r != ozmm::compute_r(n, beta)) {
    std::printf("CLOSED-FORM MISMATCH\n");
    return 1;
  }
  if (argc > 6 && std::strcmp(argv[argc - 1], "--closed-forms-only") == 0) {
    std::printf("CLOSED-FORMS OK beta=%d r=%lld\n", beta, static_cast<long long>(r));
    return 0;
  }
  const ozmm::MatrixF64 A = ozmm::gen_phi_matrix(m, n, phi, ozmm::counter_hash(1, 1));
  const ozmm::MatrixF64 B = ozmm::gen_phi_matrix(n, p, phi, ozmm::counter_hash(1, 2));
  const ozmm::MatrixF64 C = ozmm::gen_phi_matrix(m, p, phi, ozmm::counter_hash(1, 3));
  const char* method = argc > 6 ? argv[6] : "ozIMMU_H";
  if (std::strcmp(method, "overflow") == 0) {
    // constant operands whose slices are all positive (127, 63, 63, ...): every
    // product of a group adds up, so long chunks (forced r) leave INT32 once n is
    // large (n = 65536, k = 14, force_r = 14)
    const double v = (127.0 + 63.0 / 127.0) / 64.0;
    ozmm::MatrixF64 Ac(m, n), Bc(n, p), Cc(m, p);
    for (long i = 0; i < m * n; ++i) Ac.data()[i] = v;
    for (long i = 0; i < n * p; ++i) Bc.data()[i] = v;
    for (long i = 0; i < m * p; ++i) Cc.data()[i] = 0.0;
    ozmm::SchemeConfig cfg = ozmm::config_for(ozmm::Method::ozIMMU_H, k);
    cfg.force_r = argc > 7 ? std::atol(argv[7]) : 14;
    // Wrapping: both sides wrap mod 2^32 -- bit-identical results
    cfg.overflow = ozmm::OverflowMode::Wrapping;
    const ozmm::OzakiResult ref = ozmm::ozaki_gemm_ex(1.0, Ac, Bc, 0.0, Cc, cfg);
    const auto gpu = ozmm::gpu::ozaki_gemm_ex(1.0, Ac, Bc, 0.0, Cc, cfg);
    const bool same = std::memcmp(ref.d.data(), gpu.d.data(), sizeof(double) * m * p) == 0;
    // Checked: the GPU adapter throws the OverflowError type.  (The reference's
    // own Checked throw leaves an OpenMP parallel region -- gemm_wide,
    // int_gemm.cpp:40-52 -- which terminates the process, so it is not called.)
    cfg.overflow = ozmm::OverflowMode::Checked;
    bool threw = false;
    try {
      (void)ozmm::gpu::ozaki_gemm_ex(1.0, Ac, Bc, 0.0, Cc, cfg);
    } catch (const ozmm::gpu::OverflowError& e) {
      threw = true;
      std::printf("gpu Checked: %s\n", e.what());
    }
    std::printf("%s wrapping-match=%d checked-threw=%d\n", same && threw ? "OVERFLOW-OK" : "OVERFLOW-BAD",
                same, threw);
    return same && threw ? 0 : 1;
  }
  if (std::strcmp(method, "split") == 0) {
    bool ok = true;
    for (auto st : {ozmm::SliceStrategy::BitMask, ozmm::SliceStrategy::RoundNearestPerSlice,
                    ozmm::SliceStrategy::RoundNearestConstShift}) {
      auto ref_split = [&](const ozmm::MatrixF64& x, ozmm::Side sd) {
        return st == ozmm::SliceStrategy::BitMask ? ozmm::split_bitmask(x, k, sd)
               : st == ozmm::SliceStrategy::RoundNearestPerSlice ? ozmm::split_round_nearest(x, k, sd)
                                                                  : ozmm::split_rn_const_shift(x, k, sd);
      };
      const bool a_ok = same_split(ref_split(A, ozmm::Side::Left),
                                   ozmm::gpu::split<ozmm::SplitMatrix>(A, k, ozmm::Side::Left, st));
      const bool b_ok = same_split(ref_split(B, ozmm::Side::Right),
                                   ozmm::gpu::split<ozmm::SplitMatrix>(B, k, ozmm::Side::Right, st));
      std::printf("strategy %s: A %s B %s\n", ozmm::to_string(st), a_ok ? "same" : "DIFFERS", b_ok ? "same" : "DIFFERS");
      ok = ok && a_ok && b_ok;
    }
    std::printf("%s\n", ok ? "SPLIT-OK" : "SPLIT-BAD");
    return ok ? 0 : 1;
  }
  const ozmm::SchemeConfig cfg = ozmm::config_for(ozmm::method_from_string(method), k);
  const ozmm::OzakiResult ref = ozmm::ozaki_gemm_ex(1.5, A, B, 0.5, C, cfg);       // reference
  const auto gpu = ozmm::gpu::ozaki_gemm_ex(1.5, A, B, 0.5, C, cfg);               // B200
  long same = 0;
  for (long i = 0; i < m * p; ++i)
    same += std::memcmp(ref.d.data() + i, gpu.d.data() + i, sizeof(double)) == 0;
  std::printf("%s %ld of %ld; counts ref(%lld,%lld) gpu(%lld,%lld); gpu int_gemm %.6f s\n",
              same == m * p ? "MATCH" : "MISMATCH", same, m * p,
              static_cast<long long>(ref.counts.int8_gemms),
              static_cast<long long>(ref.counts.fp64_flushes),
              static_cast<long long>(gpu.counts.int8_gemms),
              static_cast<long long>(gpu.counts.fp64_flushes), gpu.timings.int_gemm);
  return same == m * p ? 0 : 1;
}
