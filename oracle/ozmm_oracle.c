/* Plain-C restatement of the reference ozIMMU_H path -- TEST INFRASTRUCTURE.
 *
 * CPU oracle ("port").  Not part of the product: the CUDA library never links
 * or calls it.  Compiled with -ffp-contract=off like the reference
 * (proj/src/CMakeLists.txt:18-20) so every FP64 operation rounds exactly once
 * in the order written.  Each function cites the reference file:line it
 * restates (paths relative to /root/reference/proj).
 */
#include "ozmm_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { OK = 0, ERR_ARG = 1, ERR_CONFIG = 2, ERR_RANGE = 3, ERR_OVERFLOW = 4, ERR_OTHER = 9 };

static _Thread_local char g_err[256];

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

const char* ozport_last_error(void) { return g_err; }

static int g_threads = 0;
void ozport_set_threads(int n) { g_threads = n > 0 ? n : 0; }
int ozport_thread_count(void) {
#ifdef _OPENMP
  return g_threads > 0 ? g_threads : omp_get_max_threads();
#else
  return 1;
#endif
}
#define NT ozport_thread_count()

/* ---------------------------------------------------------------- bit tools */

static uint64_t bits_of(double x) {
  uint64_t u;
  memcpy(&u, &x, 8);
  return u;
}

static int bit_width_u64(uint64_t v) { return v ? 64 - __builtin_clzll(v) : 0; }

/* ceil(log2 n) via bit width: split.cpp:20-22, int_gemm.cpp:255. */
static int ceil_log2(int64_t n) { return n <= 1 ? 0 : bit_width_u64((uint64_t)n - 1); }

/* ufp_exponent: include/ozmm/ufp.hpp:35-41 (exponent field; subnormals via
 * the position of the top set fraction bit). */
static int ufp_exponent(double c) {
  const uint64_t b = bits_of(c) & ~0x8000000000000000ull;
  const int biased = (int)(b >> 52);
  if (biased > 0) return biased - 1023;
  return (63 - __builtin_clzll(b)) - 1074;
}

/* static_cast<std::int8_t>(double) as compiled by g++ on x86-64: cvttsd2si to
 * int32 (non-finite / out-of-range -> 0x80000000), then the low byte.  The
 * reference relies on it in extract_row (split.cpp:114); in range it is plain
 * truncation toward zero. */
static int8_t x86_cast_i8(double q) {
  int32_t v;
  if (!(q > -2147483649.0 && q < 2147483648.0)) v = INT32_MIN;
  else v = (int32_t)q;
  return (int8_t)(uint8_t)(uint32_t)v;
}

/* --------------------------------------------------------- closed forms */

/* compute_beta: split.cpp:211-216. */
int ozport_compute_beta(int64_t n, int* out) {
  if (n < 1) return fail(ERR_ARG, "compute_beta: n must be >= 1");
  if (n > ((int64_t)1 << 29)) return fail(ERR_ARG, "compute_beta: n > 2^29 unsupported");
  const int b = (31 - ceil_log2(n)) / 2;
  *out = b < 7 ? b : 7;
  return OK;
}

/* compute_r: int_gemm.cpp:253-258. */
int ozport_compute_r(int64_t n, int beta, int64_t* out) {
  if (n < 1 || beta < 1) return fail(ERR_ARG, "compute_r: bad arguments");
  const int e = 31 - 2 * beta - ceil_log2(n);
  *out = e <= 0 ? 1 : ((int64_t)1 << e);
  return OK;
}

/* flush_count_w: scheme.cpp:109-115 (exact: ceil(k/r)*floor((k-1)/r) even). */
static int64_t flush_count_w(int k, int64_t r) {
  const int64_t q = (k + r - 1) / r;
  const int64_t f = (k - 1) / r;
  return q * k - (q * f / 2) * r;
}

/* op_counts_with_r: scheme.cpp:176-184; int8_gemm_count :105-107.
 * accumulation: 0 PerProduct, 1 Groupwise, 2 GroupwiseSimple. */
int ozport_op_counts_with_r(int k, int64_t r, int accumulation, int64_t* c) {
  if (k < 1 || r < 1) return fail(ERR_CONFIG, "op_counts: bad arguments");
  c[0] = (int64_t)k * (k + 1) / 2;
  c[2] = r;
  c[3] = flush_count_w(k, r);
  c[1] = accumulation == 0 ? c[0] : c[3];
  return OK;
}

/* ---------------------------------------------------------- generator */

/* counter_hash: include/ozmm/generate.hpp:11-17 (SplitMix64 finalizer). */
uint64_t ozport_counter_hash(uint64_t seed, uint64_t ctr) {
  uint64_t z = seed + ctr * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* uniform_open: generate.hpp:19-21 (odd 53-bit numerator / 2^53). */
static double uniform_open(uint64_t h) { return (double)((h >> 11) | 1ull) * 0x1p-53; }

/* gen_phi_matrix: generate.cpp:11-29 ((U-0.5)*exp(phi*N), Box-Muller). */
int ozport_gen_phi_matrix(int64_t m, int64_t n, double phi, uint64_t seed, double* out) {
  if (m < 1 || n < 1) return fail(ERR_ARG, "gen_phi_matrix: empty shape");
  if (!(phi >= 0)) return fail(ERR_ARG, "gen_phi_matrix: phi must be >= 0");
  const int64_t total = m * n;
  const double pi = 3.141592653589793; /* std::numbers::pi */
#pragma omp parallel for schedule(static) num_threads(NT)
  for (int64_t idx = 0; idx < total; ++idx) {
    const uint64_t ctr = (uint64_t)idx * 3;
    const double u = uniform_open(ozport_counter_hash(seed, ctr));
    const double u1 = uniform_open(ozport_counter_hash(seed, ctr + 1));
    const double u2 = uniform_open(ozport_counter_hash(seed, ctr + 2));
    const double normal = sqrt(-2.0 * log(u1)) * cos(2.0 * pi * u2);
    out[idx] = (u - 0.5) * exp(phi * normal);
  }
  return OK;
}

/* ---------------------------------------------------------- splitter */

#define K_SIGMA_SCALE 6755399441055744.0 /* 0.75 * 2^53: split.cpp:16 */
#define K_UNDERFLOW_EXP (-1000)          /* split.cpp:17 */
#define K_OVERFLOW_EXP 920               /* split.cpp:18 */

/* One line (row of A, or column of B) of rn_const_shift_rows:
 * split.cpp:151-173 with rn_unit :121-130 and extract_row :109-117.
 * v: line values at stride `st`; slices written at the same offsets into each
 * of the k planes (plane stride `plane`); shift -> *shift_out. */
static int split_line(const double* v, int64_t len, int64_t st, int k, int beta,
                      int8_t* sl, int64_t plane, double* shift_out, double* res, double* w,
                      int* flagged) {
  double rm = 0.0;
  for (int64_t j = 0; j < len; ++j) {
    const double a = fabs(v[j * st]);
    if (j == 0 || a > rm) rm = a; /* maxCoeff of cwiseAbs */
  }
  if (rm == 0.0) { /* :159 zero line: shift 0, slices stay 0, residual stays 0 */
    *shift_out = 0.0;
    if (res)
      for (int64_t j = 0; j < len; ++j) res[j * st] = 0.0;
    return OK;
  }
  /* rn_unit :121-130 */
  const int pe0 = ufp_exponent(rm);
  if (pe0 < K_UNDERFLOW_EXP) *flagged = 1;
  if (pe0 > K_OVERFLOW_EXP) return ERR_RANGE;
  const double threshold = ldexp(2.0 - ldexp(1.0, -beta), pe0);
  const int up = rm >= threshold;
  const double u1 = ldexp(1.0, pe0 + 1 - beta + up);
  const int pe = pe0 + up; /* :162 */
  *shift_out = ldexp(1.0, pe);
  for (int64_t j = 0; j < len; ++j) w[j] = v[j * st];
  for (int s = 1; s <= k; ++s) {
    const double unit = s == 1 ? u1 : ldexp(1.0, pe + 1 - beta * s); /* :166 */
    int any = 0;
    for (int64_t j = 0; j < len; ++j) any |= w[j] != 0.0; /* :167 */
    if (!any) continue;
    const double sigma = K_SIGMA_SCALE * unit; /* extract_row :111-116 */
    int8_t* out = sl + (int64_t)(s - 1) * plane;
    for (int64_t j = 0; j < len; ++j) {
      const double x = (w[j] + sigma) - sigma;
      out[j * st] = x86_cast_i8(x / unit);
      w[j] -= x;
    }
  }
  if (res)
    for (int64_t j = 0; j < len; ++j) res[j * st] = w[j];
  return OK;
}

/* split_rn_const_shift: split.cpp:233-237 via split_any :182-198.  side 0 =
 * Left (rows of a, inner dimension = cols), 1 = Right (columns of a, inner
 * dimension = rows; the reference transposes in and out, :194-197, which is
 * the same per-column arithmetic).  slices: k planes in a's row-major layout. */
int ozport_split_rn_const_shift(const double* a, int64_t rows, int64_t cols, int k, int side,
                                int force_beta, int8_t* slices, double* shift, double* residual,
                                int* beta_out, int* underflow) {
  if (rows < 1 || cols < 1) return fail(ERR_ARG, "split: empty matrix");
  if (k < 1) return fail(ERR_ARG, "split: k must be >= 1");
  int beta;
  if (force_beta != 0) { /* resolve_beta :24-31 */
    if (force_beta < 1 || force_beta > 7)
      return fail(ERR_ARG, "split: forced beta outside 1..7");
    beta = force_beta;
  } else {
    const int rc = ozport_compute_beta(side == 0 ? cols : rows, &beta);
    if (rc) return rc;
  }
  const int64_t plane = rows * cols;
  memset(slices, 0, (size_t)(plane * k));
  const int64_t lines = side == 0 ? rows : cols;
  const int64_t len = side == 0 ? cols : rows;
  const int64_t st = side == 0 ? 1 : cols;
  int flagged = 0, range = 0;
#pragma omp parallel num_threads(NT) reduction(| : flagged, range)
  {
    double* w = (double*)malloc(sizeof(double) * (size_t)len);
#pragma omp for schedule(static)
    for (int64_t i = 0; i < lines; ++i) {
      const int64_t base = side == 0 ? i * cols : i;
      if (split_line(a + base, len, st, k, beta, slices + base, plane, shift + i,
                     residual ? residual + base : NULL, w, &flagged) != OK)
        range = 1;
    }
    free(w);
  }
  if (range) return fail(ERR_RANGE, "split: row magnitude too large for shift extraction");
  if (beta_out) *beta_out = beta;
  if (underflow) *underflow = flagged;
  return OK;
}

/* --------------------------------------------------- INT8 unit + scheme */

/* acc64 += A_s * B_t exactly (the INT8-unit contract of i8_gemm_accumulate,
 * int_gemm.cpp:206-251): A_s m x n, B_t n x p, both row-major int8.  Per
 * product the sum fits int32 (n * 127^2 < 2^31 for n <= 2^17); larger n is
 * summed in int64 directly. */
static void i8_product_add(const int8_t* as, const int8_t* bt, int64_t m, int64_t n, int64_t p,
                           int64_t* acc64) {
  const int narrow = n * 127 * 127 <= INT32_MAX;
#pragma omp parallel num_threads(NT)
  {
    int32_t* row32 = (int32_t*)malloc(sizeof(int32_t) * (size_t)p);
    int64_t* row64 = (int64_t*)malloc(sizeof(int64_t) * (size_t)p);
#pragma omp for schedule(static)
    for (int64_t i = 0; i < m; ++i) {
      const int8_t* ar = as + i * n;
      int64_t* out = acc64 + i * p;
      if (narrow) {
        memset(row32, 0, sizeof(int32_t) * (size_t)p);
        for (int64_t l = 0; l < n; ++l) {
          const int32_t av = ar[l];
          if (!av) continue;
          const int8_t* br = bt + l * p;
          for (int64_t j = 0; j < p; ++j) row32[j] += av * (int32_t)br[j];
        }
        for (int64_t j = 0; j < p; ++j) out[j] += row32[j];
      } else {
        memset(row64, 0, sizeof(int64_t) * (size_t)p);
        for (int64_t l = 0; l < n; ++l) {
          const int64_t av = ar[l];
          if (!av) continue;
          const int8_t* br = bt + l * p;
          for (int64_t j = 0; j < p; ++j) row64[j] += av * (int64_t)br[j];
        }
        for (int64_t j = 0; j < p; ++j) out[j] += row64[j];
      }
    }
    free(row32);
    free(row64);
  }
}

/* Checked/Wrapping handling of the running INT32 sum after each product
 * (int_gemm.cpp:49-53 applied to the full running sum, i.e. cin + a*b). */
static int settle(int64_t* acc64, int64_t mp, int wrapping) {
  for (int64_t e = 0; e < mp; ++e) {
    const int64_t s = acc64[e];
    if (s < INT32_MIN || s > INT32_MAX) {
      if (!wrapping) return ERR_OVERFLOW;
      acc64[e] = (int32_t)(uint32_t)(uint64_t)s;
    }
  }
  return OK;
}

/* flush_scaled: scheme.cpp:29-41 with rowu = scaled_shift(mu, 2 - beta*g)
 * (:51-55, :93).  c += (ru * double(acc)) * cv, rows with ru == 0 skipped. */
static void flush_scaled(double* c, const int64_t* acc64, const double* mu, const double* nu,
                         int64_t m, int64_t p, int exp2) {
#pragma omp parallel for schedule(static) num_threads(NT)
  for (int64_t i = 0; i < m; ++i) {
    const double ru = ldexp(mu[i], exp2);
    if (ru == 0.0) continue;
    double* crow = c + i * p;
    const int64_t* prow = acc64 + i * p;
    for (int64_t j = 0; j < p; ++j) crow[j] += ru * (double)(int32_t)prow[j] * nu[j];
  }
}

typedef struct {
  int8_t *sa, *sb;
  double *mu, *nu;
  int beta;
} SplitPair;

static int split_pair(const double* a, int64_t m, int64_t n, const double* b, int64_t p, int k,
                      int force_beta, SplitPair* sp) {
  sp->sa = (int8_t*)malloc((size_t)(k * m * n));
  sp->sb = (int8_t*)malloc((size_t)(k * n * p));
  sp->mu = (double*)malloc(sizeof(double) * (size_t)m);
  sp->nu = (double*)malloc(sizeof(double) * (size_t)p);
  int beta_b;
  int rc = ozport_split_rn_const_shift(a, m, n, k, 0, force_beta, sp->sa, sp->mu, NULL,
                                       &sp->beta, NULL);
  if (!rc)
    rc = ozport_split_rn_const_shift(b, n, p, k, 1, force_beta, sp->sb, sp->nu, NULL, &beta_b,
                                     NULL);
  return rc;
}

static void free_pair(SplitPair* sp) {
  free(sp->sa);
  free(sp->sb);
  free(sp->mu);
  free(sp->nu);
}

/* groupwise_impl: scheme.cpp:65-103.  For g = 2..k+1 accumulate A_s B_{g-s}
 * for s = 1..g-1, flushing when q == r or the group ends (:91).  When
 * chunks != NULL the INT32 chunk sums are also recorded in flush order. */
static int groupwise(const SplitPair* sp, int64_t m, int64_t n, int64_t p, int k, int64_t r,
                     int wrapping, double* d, int32_t* acc_out, int* cg, int* cs0, int* cs1,
                     int64_t* w_out, int64_t* gemms) {
  const int64_t mp = m * p;
  int64_t* acc64 = (int64_t*)calloc((size_t)mp, sizeof(int64_t));
  int64_t w = 0;
  int rc = OK;
  if (d) memset(d, 0, sizeof(double) * (size_t)mp); /* MatrixF64::Zero :78 */
  for (int g = 2; g <= k + 1 && rc == OK; ++g) {
    memset(acc64, 0, sizeof(int64_t) * (size_t)mp);
    int64_t q = 0;
    int s0 = 1;
    for (int s = 1; s <= g - 1; ++s) {
      ++q;
      i8_product_add(sp->sa + (int64_t)(s - 1) * m * n, sp->sb + (int64_t)(g - s - 1) * n * p,
                     m, n, p, acc64);
      if (gemms) ++*gemms;
      if ((rc = settle(acc64, mp, wrapping)) != OK) break;
      const int group_done = s == g - 1;
      if (q == r || group_done) {
        if (d) flush_scaled(d, acc64, sp->mu, sp->nu, m, p, 2 - sp->beta * g);
        if (acc_out) {
          int32_t* dst = acc_out + w * mp;
          for (int64_t e = 0; e < mp; ++e) dst[e] = (int32_t)acc64[e];
          cg[w] = g;
          cs0[w] = s0;
          cs1[w] = s;
        }
        ++w;
        q = 0;
        s0 = s + 1;
        if (!group_done) memset(acc64, 0, sizeof(int64_t) * (size_t)mp);
      }
    }
  }
  free(acc64);
  if (w_out) *w_out = w;
  if (rc == ERR_OVERFLOW) return fail(ERR_OVERFLOW, "i8_gemm: INT32 overflow");
  return rc;
}

/* ozaki_gemm_ex for the ozIMMU_H preset: scheme.cpp:274-291 over ozaki_mm
 * :228-272 (validate_config :161-174, config_for :137-159). */
int ozport_gemm(int method, int k, int force_beta, int64_t force_r, int overflow_mode,
                double alpha, const double* a, int64_t m, int64_t n, const double* b,
                int64_t p, double beta, const double* c, double* out, int64_t* counts,
                double* timings) {
  if (method != 3) return fail(ERR_CONFIG, "port oracle restates ozIMMU_H only");
  if (k < 1) return fail(ERR_CONFIG, "k must be >= 1");
  if (m < 1 || n < 1 || p < 1) return fail(ERR_ARG, "split: empty matrix");
  if (force_r < 0) return fail(ERR_CONFIG, "force_r must be >= 1");
  int bchk;
  if (!force_beta) {
    const int rc = ozport_compute_beta(n, &bchk);
    if (rc) return rc;
  }
  SplitPair sp;
  int rc = split_pair(a, m, n, b, p, k, force_beta, &sp);
  if (rc) {
    free_pair(&sp);
    return rc;
  }
  int64_t r = force_r;
  if (!r) ozport_compute_r(n, sp.beta, &r);
  double* d = (double*)malloc(sizeof(double) * (size_t)(m * p));
  int64_t w = 0, gemms = 0;
  rc = groupwise(&sp, m, n, p, k, r, overflow_mode, d, NULL, NULL, NULL, NULL, &w, &gemms);
  if (rc == OK) {
    const int64_t total = m * p;
#pragma omp parallel for schedule(static) num_threads(NT)
    for (int64_t idx = 0; idx < total; ++idx) out[idx] = alpha * d[idx] + beta * c[idx];
    if (counts) {
      counts[0] = gemms;
      counts[1] = w;
      counts[2] = r;
      counts[3] = flush_count_w(k, r);
    }
    if (timings) memset(timings, 0, sizeof(double) * 5);
  }
  free(d);
  free_pair(&sp);
  return rc;
}

int ozport_groupwise_chunks(const double* a, int64_t m, int64_t n, const double* b, int64_t p,
                            int k, int force_beta, int64_t force_r, int32_t* acc_out,
                            int* chunk_g, int* chunk_s0, int* chunk_s1, int64_t* w_out) {
  if (k < 1) return fail(ERR_CONFIG, "k must be >= 1");
  SplitPair sp;
  int rc = split_pair(a, m, n, b, p, k, force_beta, &sp);
  if (!rc) {
    int64_t r = force_r;
    if (!r) ozport_compute_r(n, sp.beta, &r);
    rc = groupwise(&sp, m, n, p, k, r, 0, NULL, acc_out, chunk_g, chunk_s0, chunk_s1, w_out,
                   NULL);
  }
  free_pair(&sp);
  return rc;
}

/* ------------------------------------------------------ accuracy tools */

/* Correctly rounded dot products: restates exact_gemm_oracle
 * (oracle.cpp:276-300) using its exact wide-accumulator route (DigitWindow
 * :99-159: signed base-2^32 digits, one normalisation) for every entry, and
 * round_magnitude (:56-90, RNE with the subnormal floor at 2^-1074). */
typedef struct {
  int64_t* dig;
  int cap;
} Digits;

static int exact_dot(const double* a, const double* b, int64_t n, int64_t bstride, Digits* dw,
                     double* out) {
  int emin = 1 << 30, emax = -(1 << 30);
  for (int64_t l = 0; l < n; ++l) {
    const double x = a[l], y = b[l * bstride];
    if (x == 0.0 || y == 0.0) continue;
    int ex, ey;
    frexp(x, &ex);
    frexp(y, &ey);
    const int e = (ex - 53) + (ey - 53);
    if (e < emin) emin = e;
    if (e > emax) emax = e;
  }
  if (emax < emin) {
    *out = 0.0;
    return OK;
  }
  const int base = (int)floor(emin / 32.0) * 32;
  const int nd = (emax + 106 + 2 + bit_width_u64((uint64_t)n) - base) / 32 + 2;
  if (nd > dw->cap) {
    dw->dig = (int64_t*)realloc(dw->dig, sizeof(int64_t) * (size_t)nd);
    dw->cap = nd;
  }
  int64_t* dig = dw->dig;
  memset(dig, 0, sizeof(int64_t) * (size_t)nd);
  for (int64_t l = 0; l < n; ++l) {
    const double x = a[l], y = b[l * bstride];
    if (x == 0.0 || y == 0.0) continue;
    int ex, ey;
    const double fx = frexp(x, &ex), fy = frexp(y, &ey);
    const int64_t sx = (int64_t)ldexp(fx, 53), sy = (int64_t)ldexp(fy, 53);
    const int e = (ex - 53) + (ey - 53);
    __int128 prod = (__int128)sx * sy;
    const int neg = prod < 0;
    unsigned __int128 mag = neg ? (unsigned __int128)(-prod) : (unsigned __int128)prod;
    const int off = e - base, d0 = off >> 5, sh = off & 31;
    uint64_t carry = 0;
    for (int t = 0; t < 5; ++t) {
      const uint64_t g = t < 4 ? (uint64_t)((mag >> (32 * t)) & 0xFFFFFFFFu) : 0;
      const uint64_t cur = (g << sh) | carry;
      carry = cur >> 32;
      const int64_t piece = (int64_t)(cur & 0xFFFFFFFFu);
      dig[d0 + t] += neg ? -piece : piece;
    }
  }
  /* normalise to canonical digits + sign */
  int64_t carry = 0;
  for (int t = 0; t < nd; ++t) {
    const int64_t s = dig[t] + carry;
    dig[t] = s & 0xFFFFFFFF;
    carry = s >> 32;
  }
  const int negative = carry < 0;
  if (negative) {
    int64_t borrow = 1;
    for (int t = 0; t < nd; ++t) {
      const int64_t s = (~dig[t] & 0xFFFFFFFF) + borrow;
      dig[t] = s & 0xFFFFFFFF;
      borrow = s >> 32;
    }
  }
  int msb = -1;
  for (int t = nd - 1; t >= 0; --t)
    if (dig[t]) {
      msb = 32 * t + bit_width_u64((uint64_t)dig[t]) - 1;
      break;
    }
  if (msb < 0) {
    *out = 0.0;
    return OK;
  }
#define BIT(pos) ((pos) < 0 ? 0 : (int)((dig[(pos) >> 5] >> ((pos)&31)) & 1))
  const int value_exp = base + msb;
  int round_exp = value_exp - 52 > -1074 ? value_exp - 52 : -1074;
  const int pp = round_exp - base;
  double mag;
  if (pp <= 0) {
    uint64_t v = 0;
    for (int q = msb; q >= 0; --q) v = (v << 1) | (uint64_t)BIT(q);
    mag = ldexp((double)v, base);
  } else {
    uint64_t mant = 0;
    for (int q = msb; q >= pp; --q) mant = (mant << 1) | (uint64_t)BIT(q);
    const int guard = BIT(pp - 1);
    int sticky = 0;
    for (int q = pp - 2; q >= 0 && !sticky; --q) sticky = BIT(q);
    if (guard && (sticky || (mant & 1))) {
      ++mant;
      if (mant == (1ull << 53)) {
        mant = 1ull << 52;
        ++round_exp;
      }
    }
    if (round_exp > 1023 - 52) return ERR_RANGE;
    mag = ldexp((double)mant, round_exp);
  }
#undef BIT
  if (isinf(mag)) return ERR_RANGE;
  *out = negative ? -mag : mag;
  return OK;
}

int ozport_exact_gemm(const double* a, int64_t m, int64_t n, const double* b, int64_t p,
                      double* out) {
  int bad = 0;
#pragma omp parallel num_threads(NT) reduction(| : bad)
  {
    Digits dw = {NULL, 0};
#pragma omp for schedule(dynamic, 1)
    for (int64_t i = 0; i < m; ++i)
      for (int64_t j = 0; j < p; ++j)
        if (exact_dot(a + i * n, b + j, n, p, &dw, out + i * p + j) != OK) bad = 1;
    free(dw.dig);
  }
  if (bad) return fail(ERR_RANGE, "exact_gemm_oracle: FP64 overflow");
  return OK;
}

/* fp64_gemm_reference: oracle.cpp:302-319 (ascending inner index, no FMA). */
int ozport_fp64_gemm(const double* a, int64_t m, int64_t n, const double* b, int64_t p,
                     double* out) {
#pragma omp parallel for schedule(static) num_threads(NT)
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < p; ++j) {
      double s = 0.0;
      for (int64_t l = 0; l < n; ++l) s += a[i * n + l] * b[l * p + j];
      out[i * p + j] = s;
    }
  return OK;
}

/* max_rel_err: oracle.cpp:321-335. */
int ozport_max_rel_err(const double* t, const double* r, int64_t m, int64_t p, double* out) {
  const int64_t total = m * p;
  double rmax = 0.0;
  for (int64_t e = 0; e < total; ++e) {
    const double v = fabs(r[e]);
    if (e == 0 || v > rmax) rmax = v;
  }
  if (rmax == 0.0) return fail(ERR_ARG, "max_rel_err: all-zero reference");
  double worst = 0.0;
  for (int64_t e = 0; e < total; ++e) {
    const double rv = r[e];
    const double err = rv != 0.0 ? fabs(t[e] - rv) / fabs(rv) : fabs(t[e]) / rmax;
    if (worst < err) worst = err; /* std::max(worst, e) */
  }
  *out = worst;
  return OK;
}
