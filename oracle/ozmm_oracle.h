/* Plain-C restatement of the reference ozIMMU_H path -- TEST INFRASTRUCTURE.
 *
 * This is the "port" CPU oracle.  It is a checker: only tests/, the graft
 * smoke() and bench.py's CPU-baseline leg may load it.  It is pinned against
 * the unmodified reference library (oracle/_ref/libozmm_ref.so) and against
 * the committed golden fixtures (tests/golden) by tests/test_oracle.py.
 *
 * Every entry point mirrors an ozref_* entry of oracle/ref_capi.cpp with the
 * same arguments, so tests can run the two side by side.  Status codes:
 * 0 ok, 1 argument error, 2 config error, 3 range (row max >= 2^921 or FP64
 * overflow in the exact oracle), 4 INT32 overflow in Checked mode.
 */
#ifndef OZMM_ORACLE_H
#define OZMM_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* ozport_last_error(void);
void ozport_set_threads(int n);
int ozport_thread_count(void);

int ozport_compute_beta(int64_t n, int* out);
int ozport_compute_r(int64_t n, int beta, int64_t* out);
int ozport_op_counts_with_r(int k, int64_t r, int accumulation, int64_t* counts);

uint64_t ozport_counter_hash(uint64_t seed, uint64_t ctr);
int ozport_gen_phi_matrix(int64_t m, int64_t n, double phi, uint64_t seed, double* out);

int ozport_gemm(int method, int k, int force_beta, int64_t force_r, int overflow_mode,
                double alpha, const double* a, int64_t m, int64_t n, const double* b,
                int64_t p, double beta, const double* c, double* out, int64_t* counts,
                double* timings);
int ozport_split_rn_const_shift(const double* a, int64_t rows, int64_t cols, int k, int side,
                                int force_beta, int8_t* slices, double* shift, double* residual,
                                int* beta_out, int* underflow);
int ozport_groupwise_chunks(const double* a, int64_t m, int64_t n, const double* b, int64_t p,
                            int k, int force_beta, int64_t force_r, int32_t* acc_out,
                            int* chunk_g, int* chunk_s0, int* chunk_s1, int64_t* w_out);

int ozport_exact_gemm(const double* a, int64_t m, int64_t n, const double* b, int64_t p,
                      double* out);
int ozport_fp64_gemm(const double* a, int64_t m, int64_t n, const double* b, int64_t p,
                     double* out);
int ozport_max_rel_err(const double* t, const double* r, int64_t m, int64_t p, double* out);

#ifdef __cplusplus
}
#endif
#endif
