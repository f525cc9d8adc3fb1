// ozmm_b200_cli -- the reference CLI's `gemm` and `counts` subcommands
// (proj/tools/ozmm_cli.cpp:57-108, :171-186) over the B200 C ABI, reading and
// writing the reference's OZMM matrix files (proj/src/io.cpp:16-89).
//
//   ozmm_b200_cli gemm A.ozmm B.ozmm [C.ozmm] --out D.ozmm [--alpha a] [--beta b]
//                 [--k 8] [--method ozIMMU_H] [--overflow-mode checked|wrapping]
//                 [--force-beta b] [--force-r r] [--dump-splits PREFIX]
//                 [--transa] [--transb] [--device d]
//   ozmm_b200_cli counts --n N --k K --method M [--force-beta b] [--force-r r]
//
// Exit codes as the reference: 0 ok, 2 format / configuration / argument
// errors, 1 anything else (ozmm_cli.cpp:279-304).  `gemm` prints one JSON
// line with the reference's keys (:92-106); timings are CUDA-event phases.
// --transa/--transb are the DGEMM-style extension: op(X) = X^T of the stored
// matrix.  --overflow-mode as the reference (checked: an INT32 chunk overflow,
// reachable only with --force-r / --force-beta, is an error and D is not
// written; wrapping: sums mod 2^32).  --dump-splits writes the split of op(A)
// (Left) and op(B) (Right) with the method's strategy as the reference's
// dump_split does (split.cpp:254-270): PREFIX.{a,b}.slice<s>.ozmm (int8),
// PREFIX.{a,b}.shift.ozmm (1 x lines) or .shift<s>.ozmm (per-slice units) and
// PREFIX.{a,b}.residual.ozmm, computed on the GPU (ozmm_split_host).
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/ozmm_b200.h"

namespace {

struct FormatError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ---------------------------------------------------------------- OZMM IO
// Layout (io.cpp:16-18, :56-89): "OZMM", version 1, element kind (0 = F64),
// 6 zero bytes, u64 LE rows, u64 LE cols, row-major little-endian payload.
struct Matrix {
  uint64_t rows = 0, cols = 0;
  std::vector<double> data;
};

uint64_t get_u64(const unsigned char* p) {
  uint64_t v = 0;
  for (int i = 0; i < 8; ++i) v |= static_cast<uint64_t>(p[i]) << (8 * i);
  return v;
}

void put_u64(unsigned char* p, uint64_t v) {
  for (int i = 0; i < 8; ++i) p[i] = static_cast<unsigned char>(v >> (8 * i));
}

Matrix load_f64(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw FormatError(path + ": cannot open");
  unsigned char h[28];
  in.read(reinterpret_cast<char*>(h), sizeof h);
  if (!in) throw FormatError(path + ": truncated header");
  if (std::memcmp(h, "OZMM", 4) != 0) throw FormatError(path + ": bad magic, not an OZMM file");
  if (h[4] != 1) throw FormatError(path + ": unsupported format version " + std::to_string(h[4]));
  if (h[5] > 3) throw FormatError(path + ": unknown element kind");
  for (int i = 6; i < 12; ++i)
    if (h[i] != 0) throw FormatError(path + ": nonzero reserved bytes");
  if (h[5] != 0) throw FormatError(path + ": element kind mismatch");
  Matrix m;
  m.rows = get_u64(h + 12);
  m.cols = get_u64(h + 20);
  if (m.rows < 1 || m.cols < 1) throw FormatError(path + ": empty shape");
  if (m.rows > (1ull << 32) || m.cols > (1ull << 32)) throw FormatError(path + ": implausible shape");
  m.data.resize(m.rows * m.cols);
  in.read(reinterpret_cast<char*>(m.data.data()),
          static_cast<std::streamsize>(sizeof(double) * m.data.size()));
  if (!in) throw FormatError(path + ": truncated payload");
  char extra;
  if (in.read(&extra, 1)) throw FormatError(path + ": trailing bytes");
  return m;
}

// element kind 0 = F64, 1 = I8 (io.hpp:17)
void save_raw(const std::string& path, uint64_t rows, uint64_t cols, int kind, const void* data, size_t bytes) {
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) throw FormatError(path + ": cannot open for writing");
  unsigned char h[28] = {'O', 'Z', 'M', 'M', 1, static_cast<unsigned char>(kind)};
  put_u64(h + 12, rows);
  put_u64(h + 20, cols);
  out.write(reinterpret_cast<const char*>(h), sizeof h);
  out.write(static_cast<const char*>(data), static_cast<std::streamsize>(bytes));
  if (!out) throw FormatError(path + ": write failed");
}

void save_f64(const std::string& path, const Matrix& m) {
  save_raw(path, m.rows, m.cols, 0, m.data.data(), sizeof(double) * m.data.size());
}

// ---------------------------------------------------------------- args
struct Args {
  std::vector<std::string> pos;
  std::string out, method = "ozIMMU_H", overflow = "checked", dump_prefix;
  double alpha = 1.0, beta = 0.0;
  int k = 8, force_beta = 0, device = 0;
  int64_t force_r = 0, n = -1;
  bool transa = false, transb = false, have_k = false, have_method = false;
};

Args parse(int argc, char** argv, int first) {
  Args a;
  for (int i = first; i < argc; ++i) {
    const std::string s = argv[i];
    auto val = [&]() -> std::string {
      if (i + 1 >= argc) throw UsageError(s + ": missing value");
      return argv[++i];
    };
    auto num = [&](const std::string& v) {
      char* end = nullptr;
      const double d = std::strtod(v.c_str(), &end);
      if (end == v.c_str() || *end) throw UsageError(s + ": not a number: " + v);
      return d;
    };
    if (s == "--out") a.out = val();
    else if (s == "--alpha") a.alpha = num(val());
    else if (s == "--beta") a.beta = num(val());
    else if (s == "--k") a.k = static_cast<int>(num(val())), a.have_k = true;
    else if (s == "--method") a.method = val(), a.have_method = true;
    else if (s == "--overflow-mode") a.overflow = val();
    else if (s == "--dump-splits") a.dump_prefix = val();
    else if (s == "--force-beta") a.force_beta = static_cast<int>(num(val()));
    else if (s == "--force-r") a.force_r = static_cast<int64_t>(num(val()));
    else if (s == "--device") a.device = static_cast<int>(num(val()));
    else if (s == "--n") a.n = static_cast<int64_t>(num(val()));
    else if (s == "--transa") a.transa = true;
    else if (s == "--transb") a.transb = true;
    else if (s.rfind("--", 0) == 0) throw UsageError("unknown option " + s);
    else a.pos.push_back(s);
  }
  return a;
}

int method_code(const std::string& m) {  // method_from_string, scheme.cpp:129-135
  if (m == "ozIMMU_H") return OZMM_METHOD_OZIMMU_H;
  if (m == "ozIMMU") return OZMM_METHOD_OZIMMU;
  if (m == "ozIMMU_RN") return OZMM_METHOD_OZIMMU_RN;
  if (m == "ozIMMU_EF") return OZMM_METHOD_OZIMMU_EF;
  throw ConfigError("unknown method: " + m);
}

std::string fmt(double v) {
  char buf[40];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

void check(int rc, ozmm_handle_t h) {
  if (rc == OZMM_OK) return;
  const std::string msg = ozmm_last_error(h);
  if (rc == OZMM_ERR_ARG) throw UsageError(msg);
  if (rc == OZMM_ERR_CONFIG) throw ConfigError(msg);
  throw std::runtime_error(msg + " (" + ozmm_status_string(rc) + ")");
}

// ---------------------------------------------------------------- dump
// split strategy of a method (config_for, scheme.cpp:137-159): 0 RN const shift,
// 1 bitmask, 2 RN per slice
int method_strategy(int code) {
  if (code == OZMM_METHOD_OZIMMU || code == OZMM_METHOD_OZIMMU_EF) return OZMM_SPLIT_BITMASK;
  if (code == OZMM_METHOD_OZIMMU_RN) return OZMM_SPLIT_RN_PER_SLICE;
  return OZMM_SPLIT_RN_CONST_SHIFT;
}

// dump_split (split.cpp:254-270) of op(X) split on `side`: lines x n line-major
// results from the GPU, written in op(X)'s own layout (Right: transposed back).
void dump_split(ozmm_handle_t h, const std::string& prefix, char side, bool trans, const Matrix& X, int64_t lines,
                int64_t n, int k, int force_beta, int strategy) {
  std::vector<int8_t> sl(static_cast<size_t>(k) * lines * n);
  std::vector<double> out(static_cast<size_t>(strategy == OZMM_SPLIT_RN_PER_SLICE ? k * lines : lines));
  std::vector<double> res(static_cast<size_t>(lines * n));
  // op(X) lines: Left = rows of op(X), Right = columns of op(X)
  const char tr = trans ? 'T' : 'N';
  check(ozmm_split_host(h, side, tr, lines, n, X.data.data(), static_cast<int64_t>(X.cols), k, force_beta, strategy,
                        sl.data(), out.data(), res.data()),
        h);
  const bool right = side == 'R';
  const uint64_t R = right ? n : lines, Cc = right ? lines : n;  // op(X) shape
  std::vector<int8_t> tile(R * Cc);
  for (int s = 0; s < k; ++s) {
    const int8_t* p = sl.data() + static_cast<size_t>(s) * lines * n;
    for (int64_t i = 0; i < lines; ++i)
      for (int64_t j = 0; j < n; ++j) tile[right ? j * lines + i : i * n + j] = p[i * n + j];
    save_raw(prefix + ".slice" + std::to_string(s + 1) + ".ozmm", R, Cc, 1, tile.data(), tile.size());
  }
  if (strategy == OZMM_SPLIT_RN_PER_SLICE) {
    for (int s = 0; s < k; ++s)
      save_raw(prefix + ".shift" + std::to_string(s + 1) + ".ozmm", 1, lines, 0, out.data() + s * lines,
               sizeof(double) * lines);
  } else {
    save_raw(prefix + ".shift.ozmm", 1, lines, 0, out.data(), sizeof(double) * lines);
  }
  std::vector<double> rt(R * Cc);
  for (int64_t i = 0; i < lines; ++i)
    for (int64_t j = 0; j < n; ++j) rt[right ? j * lines + i : i * n + j] = res[i * n + j];
  save_raw(prefix + ".residual.ozmm", R, Cc, 0, rt.data(), sizeof(double) * rt.size());
}

// ---------------------------------------------------------------- gemm
int run_gemm(const Args& a) {
  if (a.pos.size() < 2 || a.pos.size() > 3) throw UsageError("gemm: expected A B [C]");
  if (a.out.empty()) throw UsageError("gemm: --out is required");
  const int code = method_code(a.method);
  const Matrix A = load_f64(a.pos[0]), B = load_f64(a.pos[1]);
  const int64_t m = a.transa ? A.cols : A.rows, n = a.transa ? A.rows : A.cols;
  const int64_t nb = a.transb ? B.cols : B.rows, p = a.transb ? B.rows : B.cols;
  if (n != nb) throw UsageError("ozaki_mm: inner dimensions differ");
  Matrix C;
  if (a.pos.size() == 3) {
    C = load_f64(a.pos[2]);
    if (static_cast<int64_t>(C.rows) != m || static_cast<int64_t>(C.cols) != p)
      throw UsageError("ozaki_gemm: C shape mismatch");
  } else {  // C defaults to zeros (ozmm_cli.cpp:63-65)
    C.rows = m;
    C.cols = p;
    C.data.assign(m * p, 0.0);
  }
  ozmm_handle_t h = nullptr;
  if (int rc = ozmm_create(&h, a.device)) {
    throw std::runtime_error(std::string("ozmm_create: ") + ozmm_last_error(nullptr) + " (" +
                             ozmm_status_string(rc) + ")");
  }
  if (a.overflow != "checked" && a.overflow != "wrapping") {
    ozmm_destroy(h);
    throw ConfigError("--overflow-mode must be 'checked' or 'wrapping'");
  }
  if (!a.dump_prefix.empty()) {  // before the GEMM, as the reference CLI does (ozmm_cli.cpp:73-86)
    try {
      dump_split(h, a.dump_prefix + ".a", 'L', a.transa, A, m, n, a.k, a.force_beta, method_strategy(code));
      dump_split(h, a.dump_prefix + ".b", 'R', a.transb, B, p, n, a.k, a.force_beta, method_strategy(code));
    } catch (...) {
      ozmm_destroy(h);
      throw;
    }
  }
  ozmm_options_t opt{};
  opt.force_beta = a.force_beta;
  opt.force_r = a.force_r;
  opt.overflow_wrap = a.overflow == "wrapping" ? 1 : 0;
  opt.timings = 1;
  opt.method = code;
  ozmm_counts_t cnt{};
  ozmm_timings_t tim{};
  const int rc = ozmm_dgemm_host(h, a.transa ? 'T' : 'N', a.transb ? 'T' : 'N', m, n, p, a.alpha,
                                 A.data.data(), static_cast<int64_t>(A.cols), B.data.data(),
                                 static_cast<int64_t>(B.cols), a.beta, C.data.data(), p, a.k, &opt,
                                 &cnt, &tim);
  try {
    check(rc, h);
  } catch (...) {
    ozmm_destroy(h);
    throw;
  }
  ozmm_destroy(h);
  save_f64(a.out, C);
  std::printf(
      "{\"cmd\":\"gemm\",\"m\":%lld,\"n\":%lld,\"p\":%lld,\"k\":%d,\"method\":\"%s\","
      "\"alpha\":%s,\"beta\":%s,\"int8_gemms\":%lld,\"fp64_flushes\":%lld,\"r\":%lld,"
      "\"w\":%lld,\"out\":\"%s\",\"t_split_a\":%s,\"t_split_b\":%s,\"t_int_gemm\":%s,"
      "\"t_accum\":%s,\"t_copy\":%s,\"device\":\"B200 (sm_100a)\"}\n",
      static_cast<long long>(m), static_cast<long long>(n), static_cast<long long>(p), a.k,
      a.method.c_str(), fmt(a.alpha).c_str(), fmt(a.beta).c_str(),
      static_cast<long long>(cnt.int8_gemms), static_cast<long long>(cnt.fp64_flushes),
      static_cast<long long>(cnt.r), static_cast<long long>(cnt.w), a.out.c_str(),
      fmt(tim.split_a).c_str(), fmt(tim.split_b).c_str(), fmt(tim.int_gemm).c_str(),
      fmt(tim.accum_fp64).c_str(), fmt(tim.copy).c_str());
  return 0;
}

// ---------------------------------------------------------------- counts
// counts_report (proj/src/harness.cpp:121-135) printed as ozmm_cli.cpp:175-185.
int run_counts(const Args& a) {
  if (a.n < 0 || !a.have_k || !a.have_method) throw UsageError("counts: --n, --k and --method are required");
  const int code = method_code(a.method);
  int beta = a.force_beta;
  if (!beta && ozmm_compute_beta(a.n, &beta) != OZMM_OK) throw UsageError(ozmm_last_error(nullptr));
  int64_t r = a.force_r;
  if (!r && ozmm_compute_r(a.n, beta, &r) != OZMM_OK) throw UsageError(ozmm_last_error(nullptr));
  ozmm_counts_t c{};
  if (ozmm_op_counts(a.k, r, &c) != OZMM_OK) throw ConfigError(ozmm_last_error(nullptr));
  const bool per_product = code == OZMM_METHOD_OZIMMU || code == OZMM_METHOD_OZIMMU_RN;
  const int64_t flushes = per_product ? c.int8_gemms : c.w;
  // kprime_max (analysis.cpp:57-63)
  int kpm = 1;
  if (beta >= 3) {
    int fl = 0;
    for (uint64_t v = static_cast<uint64_t>(a.n); v > 1; v >>= 1) ++fl;
    kpm = std::max(1, (51 - fl) / beta - 1);
  }
  std::printf("n            %lld\nk            %d\nmethod       %s\nbeta         %d\n"
              "r            %lld\nw            %lld\nkprime_max   %d\nint8_gemms   %lld\n"
              "fp64_flushes %lld\nflush_ratio  %lld/%lld = %g\n",
              static_cast<long long>(a.n), a.k, a.method.c_str(), beta,
              static_cast<long long>(r), static_cast<long long>(c.w), kpm,
              static_cast<long long>(c.int8_gemms), static_cast<long long>(flushes),
              static_cast<long long>(flushes), static_cast<long long>(c.int8_gemms),
              static_cast<double>(flushes) / static_cast<double>(c.int8_gemms));
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s gemm|counts ...\n", argv[0]);
    return 2;
  }
  const std::string cmd = argv[1];
  try {
    const Args a = parse(argc, argv, 2);
    if (cmd == "gemm") return run_gemm(a);
    if (cmd == "counts") return run_counts(a);
    std::fprintf(stderr, "error: unknown subcommand %s\n", cmd.c_str());
    return 2;
  } catch (const FormatError& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  } catch (const ConfigError& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  } catch (const UsageError& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
