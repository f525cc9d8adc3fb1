/* ozmm_b200 -- B200-native (sm_100a) ozIMMU_H emulated DGEMM: the C ABI.
 *
 * This is the drop-in boundary for the reference's hot path, the ozIMMU_H
 * preset of the Ozaki-scheme GEMM in /root/reference/proj:
 *
 *   MatrixF64   ozaki_gemm   (alpha, A, B, beta, C, cfg)   include/ozmm/scheme.hpp:92-95
 *   OzakiResult ozaki_gemm_ex(alpha, A, B, beta, C, cfg)   include/ozmm/scheme.hpp:96-98
 *   OzakiResult ozaki_mm     (A, B, cfg)                   include/ozmm/scheme.hpp:89-90
 *   cfg = config_for(Method::ozIMMU_H, k)                  src/scheme.cpp:137-159
 *
 * Everything here is plain C: pointers, sizes, status codes.  No exception,
 * no C++ or torch type crosses it.  The C++ adapter with the reference's own
 * signature (ozmm::gpu::ozaki_gemm_ex over any row-major matrix type) is the
 * header-only paper_2409_13313_b200/cpp/ozmm_gpu.hpp; the Python mirror is
 * paper_2409_13313_b200/ozmm.py.  INTEGRATION.md shows the bindings.
 *
 * Conventions (matching the reference):
 *   - ROW-MAJOR storage, like the reference's Eigen RowMajor DenseMatrix
 *     (include/ozmm/types.hpp:13-16).  op(A) is m x n, op(B) is n x p, C is
 *     m x p; n is the INNER dimension (the paper's naming).
 *     ld* is the row stride in elements.  transa = 'T' means A is stored
 *     n x m and op(A) = A^T (same for transb).  Column-major BLAS callers
 *     swap operands: C^T = op(B)^T op(A)^T (bit-identical: transpose symmetry,
 *     SURVEY.md Appendix A.5).
 *   - Result: C <- fl(fl(alpha * D) + fl(beta * C)) elementwise
 *     (src/scheme.cpp:286-287).  As in the reference, fl(beta*C) is ALWAYS
 *     formed, also for beta == 0 (so C must hold finite values; a NaN/inf in
 *     C propagates even when beta == 0, exactly like the reference).
 *   - The reference returns a NEW matrix and never modifies C; here C is
 *     overwritten in place (BLAS style).  The adapters restore the copy-out.
 *   - Device pointers, stream-ordered on the handle's stream.  The _host
 *     variant takes host pointers and is synchronous.
 *   - Inputs must be finite.  Rows/columns whose max magnitude is >= 2^921
 *     make the reference throw std::overflow_error (src/split.cpp:124-125):
 *     here OZMM_ERR_RANGE.  Row scales below 2^-1000 set the underflow flag
 *     (SplitMatrix::underflow_flagged, split.hpp:40).
 */
#ifndef OZMM_B200_H
#define OZMM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OZMM_B200_VERSION 1

/* Status codes.  The reference's exception types map as:
 *   std::invalid_argument (shapes, k, n range; scheme.cpp:230-231, :278,
 *                          split.cpp:34-36, :212-214)   -> OZMM_ERR_ARG
 *   ConfigError (scheme.hpp:20-22, scheme.cpp:162)      -> OZMM_ERR_CONFIG
 *   std::overflow_error (row max >= 2^921, split.cpp:124-125) -> OZMM_ERR_RANGE
 *   OverflowError (INT32 chunk overflow in OverflowMode::Checked,
 *                  int_gemm.hpp:13-26, int_gemm.cpp:37-59; unreachable with
 *                  the derived beta and r, reachable through force_beta /
 *                  force_r)                              -> OZMM_ERR_OVERFLOW
 *                  (ozmm_options_t.overflow_wrap = 1 selects Wrapping, which
 *                  is what the tensor core does: sums mod 2^32). */
typedef enum {
  OZMM_OK = 0,
  OZMM_ERR_ARG = 1,
  OZMM_ERR_CONFIG = 2,
  OZMM_ERR_RANGE = 3,
  OZMM_ERR_OVERFLOW = 4,
  OZMM_ERR_CUDA = 5,
  OZMM_ERR_NCCL = 6,
  OZMM_ERR_UNSUPPORTED = 7,
  OZMM_ERR_INTERNAL = 9
} ozmm_status_t;

typedef struct ozmm_handle_s* ozmm_handle_t;

/* Runtime-tallied operation counts; same fields as OpCounts (scheme.hpp:45-50). */
typedef struct {
  int64_t int8_gemms;   /* slice products issued: k(k+1)/2 */
  int64_t fp64_flushes; /* FP64 folds per element: w */
  int64_t r;            /* max products per INT32 chunk (compute_r) */
  int64_t w;            /* closed-form flush count (flush_count_w) */
} ozmm_counts_t;

/* Phase timings in seconds (CUDA events on the handle's stream); same fields
 * as PhaseTimings (scheme.hpp:52-58).  The INT8 GEMMs, the FP64 accumulation
 * and the alpha/beta epilogue are ONE fused kernel here: its time is reported
 * in int_gemm, and accum_fp64 = copy = 0. */
typedef struct {
  double split_a;
  double split_b;
  double int_gemm;
  double accum_fp64;
  double copy;
} ozmm_timings_t;

/* Options of ozmm_dgemm_ex; zero-initialise for the defaults.  force_beta /
 * force_r mirror the test-only SchemeConfig overrides (scheme.hpp:29-30). */
typedef struct {
  int force_beta;          /* 0: derive beta from n (compute_beta) */
  int64_t force_r;         /* 0: derive r from (n, beta) (compute_r) */
  int timings;             /* nonzero: fill ozmm_timings_t (adds event records) */
  int sync_check;          /* nonzero: synchronise after slicing and return
                              OZMM_ERR_RANGE before the GEMM, like the reference's
                              throw; otherwise the range flag is deferred to
                              ozmm_sync_status() */
  int32_t* chunk_dump;     /* nullable device buffer [w][m][p]: the INT32 chunk
                              sums in flush order (debug / parity) */
  int tile_n;              /* 0 = auto; 32/64/128: single-CTA kernel with that many
                              output columns per CTA (forces cta_pair = 1) */
  int cta_pair;            /* 0 = auto (CTA-pair kernel, M = 256 x N = 128 per 2-CTA
                              cluster), 1 = single-CTA kernel, 2 = CTA-pair kernel,
                              3 = experimental 4-CTA cluster sharing B by TMA multicast */
  int method;              /* OZMM_METHOD_*: 0 = ozIMMU_H (the hot path, default) */
  int signed_slices;       /* 0 = auto: when the CTA-pair kernel runs ozIMMU_H, the
                              internal slice planes are offset-binary (slice + o_s
                              as u8, u8 x u8 MMAs, offsets removed exactly in the
                              epilogue; same results, less tensor-core power);
                              1 = keep the reference's signed int8 planes */
  int c_write_only;        /* slice-level GEMMs only: C is output only (not read).
                              Valid only with beta == 0, alpha > 0 and a C free of
                              inf/NaN, where fl(alpha*d) + fl(beta*c) = fl(alpha*d)
                              bit for bit (alpha <= 0 could need the sign of a zero
                              from fl(beta*c)); ozmm_gemm_slices* reject it otherwise */
  int overflow_wrap;       /* OverflowMode (int_gemm.hpp:13).  0 = Checked, the
                              reference's default (SchemeConfig, scheme.hpp:28): when
                              force_beta / force_r make an INT32 chunk overflow
                              possible, the running chunk sums are verified exactly
                              (int64, after every product, in the reference's order,
                              int_gemm.cpp:37-59) before C is written, and a sum
                              outside INT32 returns OZMM_ERR_OVERFLOW with C
                              untouched.  1 = Wrapping (sums mod 2^32, the tensor
                              core's own behaviour; no verification). */
  int kpair;               /* tuning, same results: 0 = auto, 1 = off, 2 = on --
                              thin passes of the CTA-pair kernel in K-block pairs */
  int stages;              /* tuning, same results: 0 = auto, else the A-ring depth
                              of the CTA-pair kernel (clamped to what fits, >= 2) */
  int host_panels;         /* tuning, same results (ozmm_dgemm_host): 0 = auto (16)
                              row panels of op(A) / column panels of op(B) */
  int col_split;           /* tuning, same results: column splits of op(B) (op(A)
                              when transa).  0 = auto: the one-pass kernel
                              (slice_cols_onepass_kernel, op(B) read from HBM once)
                              in ozmm_dgemm_host, whose panel splits hide under
                              PCIe; the faster two-pass colmax + slice_cols path
                              in ozmm_dgemm[_ex].  1 = two-pass, 2 = one-pass
                              (columns up to 24576 long; longer ones two-pass) */
  int host_staging;        /* ozmm_dgemm_host, same results: 0 = auto -- pageable
                              (unregistered) A / B / C go through rings of pinned
                              slots filled by a team of host threads, pinned ones
                              are copied directly; 1 = off (the driver copies
                              pageable memory itself, single-threaded);
                              2 = stage every buffer (tests) */
  int host_threads;        /* ozmm_dgemm_host staging team size; 0 = auto
                              (the hardware threads, at most 16; each
                              holds four pinned slots of up to 2 MB per
                              direction, sized by the operands) */
} ozmm_options_t;

/* Scheme presets (config_for, scheme.cpp:137-159) plus the two other valid
 * (strategy, accumulation) pairs.  ozIMMU_H is the hot path; the others are
 * the paper's comparison methods. */
enum {
  OZMM_METHOD_OZIMMU_H = 0,            /* RN const shift + group-wise */
  OZMM_METHOD_OZIMMU = 1,              /* bitmask + per-product FP64 accumulation */
  OZMM_METHOD_OZIMMU_RN = 2,           /* RN per slice + per-product */
  OZMM_METHOD_OZIMMU_EF = 3,           /* bitmask + group-wise */
  OZMM_METHOD_RN_CONST_PER_PRODUCT = 4,/* RN const shift + per-product */
  OZMM_METHOD_OZIMMU_H_SIMPLE = 5,     /* RN const shift + GroupwiseSimple (needs r >= k) */
  OZMM_METHOD_OZIMMU_EF_SIMPLE = 6     /* bitmask + GroupwiseSimple (needs r >= k) */
};

/* Splitting strategies of ozmm_split_ex (SliceStrategy, split.hpp:11-15). */
enum { OZMM_SPLIT_RN_CONST_SHIFT = 0, OZMM_SPLIT_BITMASK = 1, OZMM_SPLIT_RN_PER_SLICE = 2 };

/* ---- handle ------------------------------------------------------------- */
int ozmm_create(ozmm_handle_t* handle, int device);
int ozmm_destroy(ozmm_handle_t handle);
/* stream: a cudaStream_t (NULL = legacy default stream). */
int ozmm_set_stream(ozmm_handle_t handle, void* stream);
int ozmm_get_stream(ozmm_handle_t handle, void** stream);
/* Message of the last failing call on this handle (or thread, when handle is NULL). */
const char* ozmm_last_error(ozmm_handle_t handle);
const char* ozmm_status_string(int status);
/* Waits for the handle's stream; returns OZMM_ERR_RANGE if any split since the
 * last query saw a line max >= 2^921 and that error was not already returned
 * by the call that raised it, and sets *underflow (nullable) when a line scale
 * fell below 2^-1000.  Clears both flags.  Every ozmm_dgemm_ex / _host call
 * reports its own range error only (sync_check / host entry): a pending flag
 * of an earlier stream-ordered call is kept for this query, never attributed
 * to a later call. */
int ozmm_sync_status(ozmm_handle_t handle, int* underflow);
/* Bytes of device workspace the handle currently owns (grown lazily). */
size_t ozmm_workspace_bytes(ozmm_handle_t handle);

/* ---- closed forms (host only, no device work) ---------------------------- */
int ozmm_compute_beta(int64_t n, int* beta);              /* split.cpp:211-216 */
int ozmm_compute_r(int64_t n, int beta, int64_t* r);      /* int_gemm.cpp:253-258 */
/* counts for (k, r): int8_gemms = k(k+1)/2, w = flush_count_w (scheme.cpp:105-115,
 * :176-184); accumulation = 1 (Groupwise) for ozIMMU_H. */
int ozmm_op_counts(int k, int64_t r, ozmm_counts_t* counts);

/* ---- the emulated DGEMM --------------------------------------------------- */
int ozmm_dgemm(ozmm_handle_t h, char transa, char transb, int64_t m, int64_t n, int64_t p,
               double alpha, const double* A, int64_t lda, const double* B, int64_t ldb,
               double beta, double* C, int64_t ldc, int k);

int ozmm_dgemm_ex(ozmm_handle_t h, char transa, char transb, int64_t m, int64_t n, int64_t p,
                  double alpha, const double* A, int64_t lda, const double* B, int64_t ldb,
                  double beta, double* C, int64_t ldc, int k, const ozmm_options_t* opt,
                  ozmm_counts_t* counts, ozmm_timings_t* timings);

/* Host-pointer variant (what the reference API takes, scheme.hpp:96-98): A, B
 * (and C when beta != 0) stream to the device in panels while the GPU splits
 * and multiplies, finished strips of the result stream back; C is overwritten
 * in place.  Synchronous.  Range errors are returned directly (sync_check is
 * implied) and leave C untouched.  Host buffers may be pinned (copied by the
 * DMA engines) or pageable (staged through pinned slots by a team of host
 * threads: ozmm_options_t.host_staging / host_threads). */
int ozmm_dgemm_host(ozmm_handle_t h, char transa, char transb, int64_t m, int64_t n, int64_t p,
                    double alpha, const double* A, int64_t lda, const double* B, int64_t ldb,
                    double beta, double* C, int64_t ldc, int k, const ozmm_options_t* opt,
                    ozmm_counts_t* counts, ozmm_timings_t* timings);

/* The same with a separate result D (m x p, row stride ldd): C is only read, as
 * the reference's ozaki_gemm_ex returns a NEW matrix and leaves C const
 * (scheme.cpp:281, :289) -- the C++ / Python drop-ins use it instead of copying
 * C first.  D may equal C (then it is ozmm_dgemm_host) but may not otherwise
 * overlap it (OZMM_ERR_ARG).  On any error D's contents are unspecified and C
 * is untouched. */
int ozmm_dgemm_host_out(ozmm_handle_t h, char transa, char transb, int64_t m, int64_t n,
                        int64_t p, double alpha, const double* A, int64_t lda, const double* B,
                        int64_t ldb, double beta, const double* C, int64_t ldc, double* D,
                        int64_t ldd, int k, const ozmm_options_t* opt, ozmm_counts_t* counts,
                        ozmm_timings_t* timings);

/* ---- the two halves, for sharded (multi-GPU) callers and parity tests ---- */
/* Row stride of a slice plane for inner dimension n: round_up(n, 16). */
int64_t ozmm_slice_ld(int64_t n);

/* K1: RN constant-shift split of `lines` lines of length n (split.cpp:151-198).
 *   side 'L': lines are the rows of op(X) where op(X) is lines x n
 *             (trans 'N': X stored lines x n; 'T': X stored n x lines).
 *   side 'R': lines are the columns of op(X) where op(X) is n x lines
 *             (trans 'N': X stored n x lines; 'T': X stored lines x n).
 * slices: device [k][lines][lds] int8 (lds = ozmm_slice_ld(n) unless larger);
 * shift: device [lines] doubles (const_shift).  beta: 0 = compute_beta(n). */
int ozmm_split(ozmm_handle_t h, char side, char trans, int64_t lines, int64_t n,
               const double* X, int64_t ldx, int k, int beta, int8_t* slices, int64_t lds,
               double* shift);

/* ozmm_split for any strategy.  out: the const shift [lines] for
 * OZMM_SPLIT_RN_CONST_SHIFT / OZMM_SPLIT_BITMASK, the per-slice units
 * [k][lines] for OZMM_SPLIT_RN_PER_SLICE (slice_units, split.hpp:38). */
int ozmm_split_ex(ozmm_handle_t h, char side, char trans, int64_t lines, int64_t n,
                  const double* X, int64_t ldx, int k, int beta, int strategy, int8_t* slices,
                  int64_t lds, double* out);

/* Host-memory split with its residual: the reference's SplitMatrix as
 * dump_split / `ozmm gemm --dump-splits` write it (split.cpp:254-270,
 * tools/ozmm_cli.cpp:73-86).  X (host) is split by side/trans/strategy as in
 * ozmm_split_ex on the GPU; results (host), line-major (transpose them for the
 * reference's Right-side layout): slices [k][lines][n] int8, out = the const
 * shift [lines] or per-slice units [k][lines], residual [lines][n] (nullable) --
 * what is left of each element after the k slices.  Range errors return
 * OZMM_ERR_RANGE like the reference's throw. */
int ozmm_split_host(ozmm_handle_t h, char side, char trans, int64_t lines, int64_t n,
                    const double* X, int64_t ldx, int k, int beta, int strategy, int8_t* slices,
                    double* out, double* residual);

/* K2+K3 over already-split operands: C <- alpha * D + beta * C with D the
 * group-wise ozIMMU_H accumulation of A slices [k][m][lds_a] / mu [m] and
 * B slices [k][p][lds_b] / nu [p] (B stored transposed: row j = column j of
 * op(B)).  n is the inner dimension the slices were cut for; beta_bits the
 * slice width used; r = 0 derives compute_r(n, beta_bits). */
int ozmm_gemm_slices(ozmm_handle_t h, int64_t m, int64_t n, int64_t p, int k, int beta_bits,
                     int64_t r, const int8_t* As, int64_t lds_a, const double* mu,
                     const int8_t* Bs, int64_t lds_b, const double* nu, double alpha,
                     double beta, double* C, int64_t ldc, const ozmm_options_t* opt);

/* ozmm_gemm_slices with explicit slice-plane strides (elements between slice s
 * and s+1): plane_a >= m*lds_a, plane_b >= p*lds_b.  Lets a caller run the
 * GEMM on a row range of a taller A panel / a column range of a wider B panel
 * in place (the 2-D grid's per-strip launches, grid2d.py). */
int ozmm_gemm_slices_strided(ozmm_handle_t h, int64_t m, int64_t n, int64_t p, int k,
                             int beta_bits, int64_t r, const int8_t* As, int64_t lds_a,
                             int64_t plane_a, const double* mu, const int8_t* Bs, int64_t lds_b,
                             int64_t plane_b, const double* nu, double alpha, double beta,
                             double* C, int64_t ldc, const ozmm_options_t* opt);

/* Offset-binary halves (the fused GEMM's fast operand format, see
 * ozmm_options_t.signed_slices).  ozmm_split_offset writes byte = slice + o_s
 * (even offsets o_1 = 2^beta, o_s = max(2, 2^(beta-1)) for s >= 2; padding
 * bytes 0) and the
 * line sums of the SIGNED slices (mod 2^32) at
 *   lsum[s * lsum_plane + line * lsum_lstride],  s = 0..k-1
 * -- [k][lines] (lsum_lstride = 1, lsum_plane >= lines) or [lines][k]
 * (lsum_plane = 1, lsum_lstride >= k); it zeroes them first.
 * ozmm_gemm_slices_offset consumes such planes with their line sums (row sums
 * of A lsa, column sums of B lsb, same indexing) and returns exactly what
 * ozmm_gemm_slices_strided returns for the signed planes. */
int ozmm_split_offset(ozmm_handle_t h, char side, char trans, int64_t lines, int64_t n,
                      const double* X, int64_t ldx, int k, int beta, int8_t* slices, int64_t lds,
                      double* shift, int32_t* lsum, int64_t lsum_plane, int64_t lsum_lstride);
/* ozmm_split_offset into planes `plane` bytes apart (plane >= lines * lds):
 * a range of lines of a larger slice array, e.g. one row panel of A split as
 * soon as it lands (grid2d.Grid2DGemm.step with per-panel ready events). */
int ozmm_split_offset_strided(ozmm_handle_t h, char side, char trans, int64_t lines, int64_t n,
                              const double* X, int64_t ldx, int k, int beta, int8_t* slices,
                              int64_t lds, int64_t plane, double* shift, int32_t* lsum,
                              int64_t lsum_plane, int64_t lsum_lstride);
int ozmm_gemm_slices_offset(ozmm_handle_t h, int64_t m, int64_t n, int64_t p, int k,
                            int beta_bits, int64_t r, const int8_t* As, int64_t lds_a,
                            int64_t plane_a, const double* mu, const int32_t* lsa,
                            int64_t lsa_plane, int64_t lsa_lstride, const int8_t* Bs,
                            int64_t lds_b, int64_t plane_b, const double* nu, const int32_t* lsb,
                            int64_t lsb_plane, int64_t lsb_lstride, double alpha, double beta,
                            double* C, int64_t ldc, const ozmm_options_t* opt);

/* ---- 2-D grid over several GPUs (SURVEY.md 8b "multi-GPU", 8e) -----------
 * One process and one handle per GPU.  The ranks form a Pr x Pc grid
 * (ozmm_grid_shape: 1x1, 2x1, 2x2, 2x4, ...); rank (gr, gc) = (rank / Pc,
 * rank % Pc) owns C block (gr, gc) of (m/Pr) x (p/Pc) and passes
 *   A: its m/(Pr*Pc) rows of op(A), rows [gr*m/Pr + gc*m/(Pr*Pc), +m/(Pr*Pc))
 *      -- (m/(Pr*Pc)) x n, or its transpose when transa;
 *   B: its p/(Pr*Pc) columns of op(B), columns [gc*p/Pc + gr*p/(Pr*Pc), ...)
 *      -- n x (p/(Pr*Pc)), or its transpose when transb;
 *   C: its C block (ldc >= p/Pc), overwritten with alpha*D + beta*C.
 * ozmm_dgemm_2d splits the rank's lines, all-gathers the INT8 slice planes,
 * shifts and line sums inside the row group (A) and the column group (B) --
 * broadcasts only -- and runs the fused GEMM on the block in three strips.
 * The result is bit-identical to ozmm_dgemm on the whole matrices.  After the
 * splits the range flags are max-reduced over the whole grid (two tiny
 * gathers, row group then column group, and one host synchronisation): if any
 * rank saw a line max >= 2^921, EVERY rank returns OZMM_ERR_RANGE before any
 * strip writes C -- the reference's throw-before-write (split.cpp:124-125).
 * The rest is stream-ordered on the handle's stream.
 * The all-gather is NCCL (every rank passes the same 128-byte id from
 * ozmm_nccl_unique_id on one rank; libnccl.so.2 is loaded on first use) or,
 * when `hook` is non-NULL, the caller's: hook(ctx, group, send, recv, bytes,
 * stream) gathers `bytes` from each member of group 0 (this grid row, member
 * index gc) or group 1 (this grid column, index gr) into recv, rank-major,
 * ordered on `stream` (a cudaStream_t); send == recv + index * bytes.
 * Returns 0 on success. */
typedef struct ozmm_grid* ozmm_grid_t;
typedef int (*ozmm_allgather_fn)(void* ctx, int group, const void* send, void* recv,
                                 int64_t bytes, void* stream);
int ozmm_grid_shape(int world, int* pr, int* pc);
int ozmm_nccl_unique_id(void* id128);
int ozmm_grid_create(ozmm_handle_t h, int device, int world, int rank, const void* nccl_id,
                     ozmm_allgather_fn hook, void* hook_ctx, ozmm_grid_t* grid);
int ozmm_grid_destroy(ozmm_grid_t grid);
int ozmm_grid_coords(ozmm_grid_t grid, int* pr, int* pc, int* gr, int* gc);
const char* ozmm_grid_last_error(void);
int ozmm_dgemm_2d(ozmm_grid_t grid, char transa, char transb, int64_t m, int64_t n, int64_t p,
                  double alpha, const double* A, int64_t lda, const double* B, int64_t ldb,
                  double beta, double* C, int64_t ldc, int k);

/* ---- introspection (host only; used by tests/test_host_logic.py) ---------- */
/* The GEMM's host schedule for (k, r) and a kernel choice (cta_pair/tile_n as
 * in ozmm_options_t): one row of 8 ints per slice product, in issue order:
 * {batch, pass, chunk (flush order), g, s, t, first-product-of-chunk, in-pass-range}.
 * info[7] = {products, chunks (= w), batches, passes, stages, a_slots, b_slots}. */
int ozmm_debug_schedule(int k, int64_t r, int cta_pair, int tile_n, int* rows, int cap,
                        int* info);

/* ---- input generator (host, OpenMP) --------------------------------------- */
/* The reference's phi test matrices (src/generate.cpp:11-29,
 * include/ozmm/generate.hpp:11-21): entry (i, j) of the GLOBAL rows x cols
 * matrix is (U - 0.5) * exp(phi * N) drawn from counter index (i*cols + j)*3.
 * Writes the block [row0, row0+nrows) x [col0, col0+ncols) into out (row
 * stride ldo), so any shard of a matrix can be generated independently. */
int ozmm_gen_phi_block(int64_t rows, int64_t cols, double phi, uint64_t seed, int64_t row0,
                       int64_t nrows, int64_t col0, int64_t ncols, double* out, int64_t ldo);
uint64_t ozmm_counter_hash(uint64_t seed, uint64_t ctr);

#ifdef __cplusplus
}
#endif
#endif /* OZMM_B200_H */
