// Host side of the C ABI (include/ozmm_b200.h): handle + workspace, the
// ozIMMU_H orchestration (split op(A) rows, split op(B) columns, fused GEMM),
// TMA descriptor encoding and the launch configuration.
//
// Mirrors ozaki_gemm_ex / ozaki_mm (proj/src/scheme.cpp:228-291) for the
// ozIMMU_H preset (config_for, :153-156): RoundNearestConstShift splits of A
// (Left) and B (Right) with beta = compute_beta(n), then group-wise
// accumulation with r = compute_r(n, beta), then the alpha/beta epilogue.
// There is no CPU fallback: every numeric step runs in the kernels below.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <atomic>
#include <memory>
#include <chrono>
#include <thread>
#include <utility>
#include <vector>

#include "../../include/ozmm_b200.h"
#include "ozimmu_gemm.cuh"
#include "ozimmu_gemm_pair.cuh"
#include "host_stage.hpp"
#include "schedule.hpp"
#include "slicer.cuh"
#include "slicer_methods.cuh"

// Environment overrides (tuning sweeps, timing probes, per-tile traces) exist
// only in the diagnostic build (-DOZMM_DIAG: `python -m
// paper_2409_13313_b200.build --diag`).  The release library reads no
// environment variable at all -- the macro drops the names at preprocessing --
// so no stray variable can change a launch, let alone a result.  Tuning that
// keeps results identical is reachable in release through ozmm_options_t.
#ifdef OZMM_DIAG
#define OZMM_ENV(name) std::getenv(name)
#else
#define OZMM_ENV(name) (static_cast<const char*>(nullptr))
#endif

// SM ids the park scratch covers (the kernel traps beyond it); B200 has 148 SMs
constexpr int kParkSmIds = 256;

namespace {

thread_local std::string g_thread_err;

// Device flags of a handle: [0] underflow, [1] range -- raised by the splits of
// the CURRENT call; [2] / [3] the same, pending from earlier stream-ordered
// calls that did not report them (folded in at the start of every GEMM entry,
// returned by ozmm_sync_status).
constexpr int kNumFlags = 4;
__global__ void fold_flags_kernel(int* f) {
  f[2] |= f[0];
  f[3] |= f[1];
  f[0] = 0;
  f[1] = 0;
}

// Splitting strategy (SliceStrategy, split.hpp:11-15) and FP64 flush scaling of
// the fused GEMM (GemmParams::scale_mode).
enum Strategy { kRNConstShift = 0, kBitMask = 1, kRNPerSlice = 2 };
struct FlushCfg {
  int scale_mode = 0;
  const double* units_a = nullptr;
  const double* units_b = nullptr;
  bool per_product = false;  // chunks of one product (accumulate_per_product)
  // offset-binary slice planes (CTA-pair kernel only): signed line sums [k][plane]
  const int32_t* lsa = nullptr;
  const int32_t* lsb = nullptr;
  int64_t lsa_plane = 0, lsb_plane = 0, lsa_lstride = 1, lsb_lstride = 1;
  int64_t n = 0;
  // tuning (same results): kpair 0 auto (on) / 1 off / 2 on, stages 0 auto
  int kpair = 0, stages = 0;
  bool biased() const { return lsa != nullptr; }
};

// method code of ozmm_options_t -> (strategy, per-product accumulation)
struct MethodCfg {
  Strategy strategy;
  bool per_product;
  bool simple;  // GroupwiseSimple: requires r >= k
};
bool method_cfg(int method, MethodCfg* out) {
  switch (method) {
    case OZMM_METHOD_OZIMMU_H: *out = {kRNConstShift, false, false}; return true;
    case OZMM_METHOD_OZIMMU: *out = {kBitMask, true, false}; return true;
    case OZMM_METHOD_OZIMMU_RN: *out = {kRNPerSlice, true, false}; return true;
    case OZMM_METHOD_OZIMMU_EF: *out = {kBitMask, false, false}; return true;
    case OZMM_METHOD_RN_CONST_PER_PRODUCT: *out = {kRNConstShift, true, false}; return true;
    case OZMM_METHOD_OZIMMU_H_SIMPLE: *out = {kRNConstShift, false, true}; return true;
    case OZMM_METHOD_OZIMMU_EF_SIMPLE: *out = {kBitMask, false, true}; return true;
    default: return false;
  }
}

struct Handle {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  // workspace (grown lazily, owned)
  int8_t* slices_a = nullptr;
  size_t slices_a_bytes = 0;
  int8_t* slices_b = nullptr;
  size_t slices_b_bytes = 0;
  double* mu = nullptr;
  size_t mu_n = 0;
  double* nu = nullptr;
  size_t nu_n = 0;
  unsigned long long* colmax = nullptr;
  size_t colmax_n = 0;
  int* flags = nullptr;  // [kNumFlags]: see fold_flags_kernel
  double* units_a = nullptr;  // per-slice units (RN per slice) [k][m] / [k][p]
  size_t units_a_n = 0;
  double* units_b = nullptr;
  size_t units_b_n = 0;
  int32_t* lsa = nullptr;  // offset-binary planes: signed line sums [k][m] / [k][p]
  size_t lsa_n = 0;
  int32_t* lsb = nullptr;
  size_t lsb_n = 0;
  int32_t* park = nullptr;  // CTA-pair kernel: parked INT32 chunk tiles, per SM id
  size_t park_n = 0;
  double* tscratch = nullptr;  // transposed operand for per-slice RN column splits
  size_t tscratch_n = 0;
  // device staging for the host-pointer entry (grown lazily, reused)
  double* host_a = nullptr;
  size_t host_a_n = 0;
  double* host_b = nullptr;
  size_t host_b_n = 0;
  double* host_c = nullptr;
  size_t host_c_n = 0;
  double* host_o = nullptr;  // GEMM output for the host entry (the input C stays intact)
  size_t host_o_n = 0;
  cudaStream_t s_in = nullptr, s_out = nullptr;  // copy streams of the host entry
  cudaStream_t s_split = nullptr;                 // host entry: panel splits (high priority)
  cudaStream_t s_gemm[2] = {nullptr, nullptr};    // host entry: strip GEMMs
  cudaStream_t s_aux = nullptr;                   // device entry: B's column maxima
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int* hflags = nullptr;                          // pinned copy of flags (host entry gate)
  bool one_pass_cols = false;  // this call's column splits: one-pass kernel (ozmm_options_t.col_split)
  // host entry, pageable caller buffers: pinned slot rings + the copy team (host_stage.hpp)
  std::unique_ptr<ozb::WorkerPool> pool;
  ozb::HostStager stage_in, stage_out;
  cudaEvent_t ev[5] = {};
  bool gemm_attr_set[3] = {false, false, false};
  bool pair_attr_set[2] = {false, false};
  int num_sms = 148;
  size_t smem_optin = 232448;
};

// Scoped choice of the column-split kernel for one call (restored on return).
struct ColSplitScope {
  Handle* h;
  bool saved;
  ColSplitScope(Handle* hh, bool one_pass);
  ~ColSplitScope();
};

int set_err(Handle* h, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (h) h->err = buf;
  g_thread_err = buf;
  return code;
}

#define CUDA_TRY(h, call)                                                               \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return set_err(h, OZMM_ERR_CUDA, "%s failed: %s (%s:%d)", #call,                  \
                     cudaGetErrorString(e_), __FILE__, __LINE__);                       \
  } while (0)

template <class T>
int ensure(Handle* h, T** ptr, size_t* have, size_t want) {
  if (*have >= want && *ptr) return OZMM_OK;
  if (*ptr) {
    cudaFree(*ptr);
    *ptr = nullptr;
    *have = 0;
  }
  CUDA_TRY(h, cudaMalloc(reinterpret_cast<void**>(ptr), std::max<size_t>(want, 256) * sizeof(T)));
  *have = std::max<size_t>(want, 256);
  return OZMM_OK;
}

ColSplitScope::ColSplitScope(Handle* hh, bool one_pass) : h(hh), saved(hh->one_pass_cols) {
  hh->one_pass_cols = one_pass;
}
ColSplitScope::~ColSplitScope() { h->one_pass_cols = saved; }

// ---- TMA descriptor encoding through the driver entry point (no -lcuda) ----
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

// 3-D int8 map over slice planes [k][lines][lds]: box = 32 B of K x rows x 1 slice,
// 32-byte swizzle (matches the UMMA descriptors built in the kernel).
int make_slice_map(Handle* h, CUtensorMap* map, const int8_t* base, int64_t lds, int64_t lines,
                   int64_t plane, int k, uint32_t box_rows, uint32_t box_k = ozb::kBK,
                   CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_32B) {
  EncodeFn fn = encode_fn();
  if (!fn) return set_err(h, OZMM_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(lds), static_cast<cuuint64_t>(lines),
                              static_cast<cuuint64_t>(k)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(lds),
                                 static_cast<cuuint64_t>(plane)};
  const cuuint32_t box[3] = {box_k, box_rows, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(base), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_err(h, OZMM_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", r);
  return OZMM_OK;
}

bool is_trans(char t) { return t == 'T' || t == 't' || t == 'C' || t == 'c'; }
bool valid_trans(char t) { return is_trans(t) || t == 'N' || t == 'n'; }

// ---- K1 launch ----------------------------------------------------------------
// Lines of op(X): row mode when the line is contiguous in memory.
// lsum != nullptr: offset-binary planes + signed line sums lsum[s][line] (plane
// stride lsum_plane; zeroed by the caller), the fused pair GEMM's operand format.
// Column maxima of the `lines` columns of X (n x lines) into h->colmax.
int launch_colmax(Handle* h, int64_t lines, int64_t n, const double* X, int64_t ldx) {
  if (int rc = ensure(h, &h->colmax, &h->colmax_n, static_cast<size_t>(lines))) return rc;
  CUDA_TRY(h, cudaMemsetAsync(h->colmax, 0, sizeof(unsigned long long) * lines, h->stream));
  const int64_t rows_per_block = 512;
  const dim3 g1(static_cast<unsigned>((lines + 31) / 32),
                static_cast<unsigned>((n + rows_per_block - 1) / rows_per_block));
  ozb::colmax_kernel<<<g1, 256, 0, h->stream>>>(X, ldx, n, lines, rows_per_block, h->colmax);
  CUDA_TRY(h, cudaGetLastError());
  return OZMM_OK;
}

// One-pass column split (slice_cols_onepass_kernel): columns of up to
// 16 x 2048 rows, X 16-byte aligned with an even ld (TMA).  cols_onepass_units
// returns the kernel's rows-per-CTA factor kU, or 0 when the shape does not
// qualify and the two-pass path runs.
int cols_onepass_units(const Handle* h, int64_t n, const double* X, int64_t ldx) {
  bool on = h->one_pass_cols;
  if (const char* e = OZMM_ENV("OZMM_COLS_TWO_PASS")) on = std::atoi(e) == 0;
  if (!on) return 0;
  if (reinterpret_cast<uintptr_t>(X) % 16 != 0 || ldx % 2 != 0 || ldx > (int64_t(1) << 36) / 8) return 0;
  // the fewest rows per CTA the 16-CTA limit allows: 1024 rows (kU = 2) beat 1536 and
  // 2048 at C3 (1.53 / 1.66 / 2.16 ms) and C2 (profiles/r2/cols_onepass_v4.txt)
  int kU = n <= 512 ? 1 : (n <= 16 * 1024 ? 2 : (n <= 16 * 1536 ? 3 : (n <= 16 * 2048 ? 4 : 0)));
  if (const char* e = OZMM_ENV("OZMM_COLS_UNITS")) kU = std::max(1, std::min(4, std::atoi(e)));
  if (kU == 0 || (n + 512 * kU - 1) / (512 * kU) > 16) return 0;
  return kU;
}

int launch_cols_onepass(Handle* h, int kU, int64_t lines, int64_t n, const double* X, int64_t ldx, int k,
                        int beta, int8_t* S, int64_t lds, int64_t plane, double* shift, int* lsum,
                        int64_t lsum_plane, int64_t lsum_lstride) {
  const int cs = static_cast<int>((n + 512 * kU - 1) / (512 * kU));
  EncodeFn fn = encode_fn();
  if (!fn) return set_err(h, OZMM_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  CUtensorMap map;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(lines), static_cast<cuuint64_t>(n)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ldx) * 8};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(ozb::kOPCols), static_cast<cuuint32_t>(ozb::kOPBox)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(X), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_err(h, OZMM_ERR_CUDA, "cuTensorMapEncodeTiled (columns) failed (%d)", r);
  const size_t smem = size_t(512) * kU * ozb::kOPCols * 8 + 16 + (2 * 16 + 8) * ozb::kOPCols * 8 +
                      ozb::kMaxSlices * ozb::kOPCols * 4;
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(ozb::kOPThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = h->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  auto go = [&](auto kern) -> int {
    CUDA_TRY(h, cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    CUDA_TRY(h, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    // as many clusters as fit at once (strips are dealt round-robin), at most one per strip
    cfg.gridDim = dim3(static_cast<unsigned>(cs));
    int nclusters = 0;
    CUDA_TRY(h, cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg));
    const int64_t nstrips = (lines + ozb::kOPCols - 1) / ozb::kOPCols;
    nclusters = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(nstrips, std::max(1, nclusters))));
    cfg.gridDim = dim3(static_cast<unsigned>(nclusters * cs));
    CUDA_TRY(h, cudaLaunchKernelEx(&cfg, kern, map, n, lines, lds, k, beta, S, plane, shift, h->flags, lsum,
                                   lsum_plane, lsum_lstride));
    return OZMM_OK;
  };
  if (kU == 1) return go(ozb::slice_cols_onepass_kernel<1>);
  if (kU == 2) return go(ozb::slice_cols_onepass_kernel<2>);
  if (kU == 3) return go(ozb::slice_cols_onepass_kernel<3>);
  return go(ozb::slice_cols_onepass_kernel<4>);
}

// colmax_ready: column mode only, h->colmax already holds this X's maxima.
int launch_split(Handle* h, bool row_mode, int64_t lines, int64_t n, const double* X, int64_t ldx,
                 int k, int beta, int8_t* S, int64_t lds, int64_t plane, double* shift,
                 int* lsum = nullptr, int64_t lsum_plane = 0, int64_t lsum_lstride = 1,
                 bool colmax_ready = false) {
  if (row_mode) {
    const bool vec = (reinterpret_cast<uintptr_t>(X) % 16 == 0) && (ldx % 2 == 0);
    // Whole row in registers, 16 elements per thread, split over a cluster of up
    // to 8 CTAs (smallest CTAs first: more rows in flight per SM); longer rows
    // use one 1024-thread CTA with a second pass.
    const int64_t chunks = (lds + 15) / 16;  // 16-element chunks per row
    int csize = 0, cthreads = 128;
    {
      int t0 = 128;
      if (const char* e = OZMM_ENV("OZMM_ROW_CTA")) t0 = std::atoi(e);
      for (int t : {t0, 256, 512}) {
        const int64_t c = (chunks + t - 1) / t;
        if (c <= 8) {
          csize = static_cast<int>(c);
          cthreads = t;
          break;
        }
      }
    }
    if (csize >= 2) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(static_cast<unsigned>(lines * csize));
      cfg.blockDim = dim3(static_cast<unsigned>(cthreads));
      cfg.stream = h->stream;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = csize;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      if (vec)
        CUDA_TRY(h, cudaLaunchKernelEx(&cfg, ozb::slice_rows_cluster_kernel<true>, X, ldx, lines, n,
                                       lds, k, beta, S, plane, shift, h->flags, lsum, lsum_plane, lsum_lstride));
      else
        CUDA_TRY(h, cudaLaunchKernelEx(&cfg, ozb::slice_rows_cluster_kernel<false>, X, ldx, lines,
                                       n, lds, k, beta, S, plane, shift, h->flags, lsum,
                                       lsum_plane, lsum_lstride));
    } else {
      const int64_t want = (chunks + 31) / 32 * 32;
      const int threads = static_cast<int>(std::min<int64_t>(1024, std::max<int64_t>(32, want)));
      const dim3 grid(static_cast<unsigned>(lines));
      if (vec)
        ozb::slice_rows_kernel<true><<<grid, threads, 0, h->stream>>>(X, ldx, lines, n, lds, k,
                                                                      beta, S, plane, shift,
                                                                      h->flags, lsum, lsum_plane, lsum_lstride);
      else
        ozb::slice_rows_kernel<false><<<grid, threads, 0, h->stream>>>(X, ldx, lines, n, lds, k,
                                                                       beta, S, plane, shift,
                                                                       h->flags, lsum, lsum_plane, lsum_lstride);
    }
  } else {
    if (!colmax_ready) {
      if (const int kU = cols_onepass_units(h, n, X, ldx))
        return launch_cols_onepass(h, kU, lines, n, X, ldx, k, beta, S, lds, plane, shift, lsum, lsum_plane,
                                   lsum_lstride);
      if (int rc = launch_colmax(h, lines, n, X, ldx)) return rc;
    }
    // offset planes: 8 row tiles per CTA (column sums leave with one atomic per
    // column, slice and CTA); signed planes: one tile per CTA
    const int tpc = lsum ? 8 : 1;
    const dim3 g2(static_cast<unsigned>((lines + 31) / 32),
                  static_cast<unsigned>((lds + 128 * tpc - 1) / (128 * tpc)));
    ozb::slice_cols_kernel<<<g2, 256, 0, h->stream>>>(X, ldx, n, lines, lds, k, beta, h->colmax,
                                                       S, plane, shift, h->flags, lsum, lsum_plane,
                                                       lsum_lstride, tpc);
  }
  CUDA_TRY(h, cudaGetLastError());
  return OZMM_OK;
}

// Cluster split of a row over up to 8 CTAs of 256/512 threads (16 elements per
// thread, whole row in registers).  Returns false when the row is too long.
bool cluster_rows_config(int64_t lds, int* csize, int* threads) {
  const int64_t chunks = (lds + 15) / 16;
  for (int t : {256, 512, 1024}) {
    const int64_t c = (chunks + t - 1) / t;
    if (c <= 8) {
      *csize = static_cast<int>(c);
      *threads = t;
      return true;
    }
  }
  return false;
}

template <class Kern, class... Args>
int launch_cluster_rows(Handle* h, Kern kern, int64_t lines, int csize, int threads,
                        Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(lines * csize));
  cfg.blockDim = dim3(static_cast<unsigned>(threads));
  cfg.stream = h->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = csize;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CUDA_TRY(h, cudaLaunchKernelEx(&cfg, kern, args...));
  return OZMM_OK;
}

// K1 for any strategy.  out = const shift [lines] (RN const shift, bitmask) or
// per-slice units [k][lines] (RN per slice).
int launch_split_m(Handle* h, Strategy st, bool row_mode, int64_t lines, int64_t n,
                   const double* X, int64_t ldx, int k, int beta, int8_t* S, int64_t lds,
                   int64_t plane, double* out) {
  if (st == kRNConstShift)
    return launch_split(h, row_mode, lines, n, X, ldx, k, beta, S, lds, plane, out);
  if (st == kRNPerSlice && !row_mode) {
    // per-slice grids need several reductions per line: transpose to contiguous lines
    if (int rc = ensure(h, &h->tscratch, &h->tscratch_n, static_cast<size_t>(lines) * n)) return rc;
    const dim3 g(static_cast<unsigned>((lines + 31) / 32), static_cast<unsigned>((n + 31) / 32));
    ozb::transpose_f64_kernel<<<g, 256, 0, h->stream>>>(X, ldx, n, lines, h->tscratch);
    CUDA_TRY(h, cudaGetLastError());
    X = h->tscratch;
    ldx = n;
    row_mode = true;
  }
  const bool vec = (reinterpret_cast<uintptr_t>(X) % 16 == 0) && (ldx % 2 == 0);
  if (row_mode) {
    int csize, threads;
    if (!cluster_rows_config(lds, &csize, &threads))
      return set_err(h, OZMM_ERR_UNSUPPORTED, "inner dimension too long for this splitter");
    if (st == kBitMask)
      return vec ? launch_cluster_rows(h, ozb::slice_rows_bitmask_kernel<true>, lines, csize,
                                       threads, X, ldx, lines, n, lds, k, beta, S, plane, out,
                                       h->flags)
                 : launch_cluster_rows(h, ozb::slice_rows_bitmask_kernel<false>, lines, csize,
                                       threads, X, ldx, lines, n, lds, k, beta, S, plane, out,
                                       h->flags);
    return vec ? launch_cluster_rows(h, ozb::slice_rows_rnps_kernel<true>, lines, csize, threads,
                                     X, ldx, lines, n, lds, k, beta, S, plane, out, h->flags)
               : launch_cluster_rows(h, ozb::slice_rows_rnps_kernel<false>, lines, csize,
                                     threads, X, ldx, lines, n, lds, k, beta, S, plane, out,
                                     h->flags);
  }
  // bitmask, column lines
  if (int rc = ensure(h, &h->colmax, &h->colmax_n, static_cast<size_t>(lines))) return rc;
  CUDA_TRY(h, cudaMemsetAsync(h->colmax, 0, sizeof(unsigned long long) * lines, h->stream));
  const int64_t rows_per_block = 512;
  const dim3 g1(static_cast<unsigned>((lines + 31) / 32),
                static_cast<unsigned>((n + rows_per_block - 1) / rows_per_block));
  ozb::colmax_kernel<<<g1, 256, 0, h->stream>>>(X, ldx, n, lines, rows_per_block, h->colmax);
  const dim3 g2(static_cast<unsigned>((lines + 31) / 32), static_cast<unsigned>((lds + 127) / 128));
  ozb::slice_cols_bitmask_kernel<<<g2, 256, 0, h->stream>>>(X, ldx, n, lines, lds, k, beta,
                                                             h->colmax, S, plane, out, h->flags);
  CUDA_TRY(h, cudaGetLastError());
  return OZMM_OK;
}

// ---- K2+K3 launch -------------------------------------------------------------
constexpr size_t kSmemReserve = 2048;  // barriers, tmem slot, alignment slack (+ nu cache)

// Fills the kernel parameter block from the host schedule.
void fill_params(ozb::GemmParams& P, const ozb::Schedule& S, int64_t m, int64_t p, int64_t lds_a,
                 int64_t lds_b, int tiles_m, int tiles_n, int beta_bits, int stages, double alpha,
                 double beta, const double* mu, const double* nu, const double* Cin, double* Cout,
                 int64_t ldc, int32_t* dump, const FlushCfg& fl) {
  std::memset(&P, 0, sizeof P);
  P.scale_mode = fl.scale_mode;
  P.bias = fl.biased() ? 1 : 0;
  P.n_inner = fl.n;
  P.lsa = fl.lsa;
  P.lsb = fl.lsb;
  P.lsa_plane = fl.lsa_plane;
  P.lsb_plane = fl.lsb_plane;
  P.lsa_lstride = fl.lsa_lstride;
  P.lsb_lstride = fl.lsb_lstride;
  P.units_a = fl.units_a;
  P.units_b = fl.units_b;
  P.m = static_cast<int>(m);
  P.p = static_cast<int>(p);
  P.n_kb = static_cast<int>((std::max(lds_a, lds_b) + ozb::kBK - 1) / ozb::kBK);
  P.tiles_m = tiles_m;
  P.tiles_n = tiles_n;
  P.group_m = 2;  // tile-row group of the raster (measured sweep, tools/l2_sweep.sh)
  if (const char* g = OZMM_ENV("OZMM_GROUP_M")) P.group_m = std::max(1, std::atoi(g));
  P.hint_a = 2;  // A panels are reused by every column tile of the group: keep them in L2
  P.hint_b = 0;
  if (const char* g = OZMM_ENV("OZMM_HINT_A")) P.hint_a = std::atoi(g);
  if (const char* g = OZMM_ENV("OZMM_HINT_B")) P.hint_b = std::atoi(g);
#ifdef OZMM_DIAG
  if (const char* g = OZMM_ENV("OZMM_DUP_MMA")) P.dup_mma = std::atoi(g);  // timing probe: wrong results
#endif
  // CTA-pair kernel: A groups issued two per barrier round (one wait burst, one
  // MMA burst, one release burst): C3 +9-12 %, C5 k=12 +7.5 %, C4 +2 % against one
  // group per round; three per round starve the producer (tools/gpairs_probe*.sh)
  P.group_pairs = 2;
  if (const char* g = OZMM_ENV("OZMM_GROUP_PAIRS")) P.group_pairs = std::atoi(g);
#ifdef OZMM_DIAG
  // timing probe: flips instruction-descriptor bits (wrong results)
  if (const char* g = OZMM_ENV("OZMM_IDESC_XOR")) P.idesc_xor = static_cast<uint32_t>(std::strtoul(g, nullptr, 0));
#endif
  P.ksnake = 1;
  if (const char* g = OZMM_ENV("OZMM_KSNAKE")) P.ksnake = std::atoi(g);
  P.nbatch = static_cast<int>(S.batches.size());
  P.npass = static_cast<int>(S.passes.size());
  P.beta = beta_bits;
  P.stages = stages;
  // a round waits for group_pairs A stages at once: never more than the ring holds
  P.group_pairs = std::max(1, std::min(P.group_pairs, stages));
  P.a_slots = S.a_slots;
  P.b_slots = S.b_slots;
  P.n_chunks = static_cast<int>(S.chunks.size());
  P.alpha = alpha;
  P.beta_c = beta;
  P.mu = mu;
  P.nu = nu;
  P.c_in = Cin;
  P.c_out = Cout;
  P.ldc = ldc;
  P.dump = dump;
  static_assert(ozb::kFlushTmem == ozb::kActFlush && ozb::kPark == ozb::kActPark &&
                    ozb::kFlushParked == ozb::kActUnpark,
                "schedule.hpp FlushKind and the kernel's action codes must agree");
  for (size_t b = 0; b < S.batches.size(); ++b) {
    const ozb::Batch& B = S.batches[b];
    P.b_c0[b] = static_cast<uint16_t>(B.c0);
    P.b_nc[b] = static_cast<uint16_t>(B.nc);
    P.b_pass0[b] = static_cast<uint16_t>(B.pass0);
    P.b_pass1[b] = static_cast<uint16_t>(B.pass1);
    for (int ci = 0; ci < B.nc && ci < 4; ++ci) P.b_cid[b * 4 + ci] = static_cast<uint16_t>(B.cids[ci]);
    P.b_act0[b] = static_cast<uint16_t>(B.act0);
    P.b_act1[b] = static_cast<uint16_t>(B.act1);
  }
  for (size_t a = 0; a < S.acts.size(); ++a) {
    const ozb::FlushAct& x = S.acts[a];
    P.act[a] = static_cast<uint32_t>(x.c) | (static_cast<uint32_t>(x.kind) << 10) |
               (static_cast<uint32_t>(std::max(0, x.ci)) << 12) | (static_cast<uint32_t>(std::max(0, x.slot)) << 16);
  }
  P.park_slots = S.park_slots;
  for (size_t q = 0; q < S.passes.size(); ++q) {
    P.p_alo[q] = static_cast<uint8_t>(S.passes[q].alo);
    P.p_ahi[q] = static_cast<uint8_t>(S.passes[q].ahi);
    P.p_blo[q] = static_cast<uint8_t>(S.passes[q].blo);
    P.p_bhi[q] = static_cast<uint8_t>(S.passes[q].bhi);
    P.p_p0[q] = static_cast<uint16_t>(S.passes[q].p0);
    P.p_p1[q] = static_cast<uint16_t>(S.passes[q].p1);
  }
  for (size_t i = 0; i < S.products.size(); ++i) {
    P.pr_ci[i] = static_cast<uint8_t>(S.products[i].ci | (S.products[i].first ? 0x80 : 0));
    P.pr_s[i] = static_cast<uint8_t>(S.products[i].s);
    P.pr_t[i] = static_cast<uint8_t>(S.products[i].t);
  }
  for (size_t c = 0; c < S.chunks.size(); ++c) {
    P.c_g[c] = static_cast<uint8_t>(S.chunks[c].g);
    P.c_s[c] = static_cast<uint8_t>(S.chunks[c].s0);
    P.c_e[c] = static_cast<uint8_t>(S.chunks[c].s1);
  }
  for (size_t q = 0; q < S.passes.size(); ++q) {
    P.p_g0[q] = static_cast<uint16_t>(S.passes[q].g0);
    P.p_g1[q] = static_cast<uint16_t>(S.passes[q].g1);
  }
#ifdef OZMM_DIAG
  // timing experiment only (results are wrong): OZMM_ONLY_BATCH=b runs batch b alone
  if (const char* e = OZMM_ENV("OZMM_ONLY_BATCH")) {
    const int b = std::atoi(e);
    if (b >= 0 && b < P.nbatch) {
      const int q0 = P.b_pass0[b], q1 = P.b_pass1[b];
      for (int q = q0; q < q1; ++q) {
        P.p_alo[q - q0] = P.p_alo[q], P.p_ahi[q - q0] = P.p_ahi[q];
        P.p_blo[q - q0] = P.p_blo[q], P.p_bhi[q - q0] = P.p_bhi[q];
        P.p_p0[q - q0] = P.p_p0[q], P.p_p1[q - q0] = P.p_p1[q];
        P.p_g0[q - q0] = P.p_g0[q], P.p_g1[q - q0] = P.p_g1[q];
      }
      P.b_c0[0] = P.b_c0[b], P.b_nc[0] = P.b_nc[b];
      P.b_pass0[0] = 0, P.b_pass1[0] = static_cast<uint16_t>(q1 - q0);
      // its chunks flushed straight from TMEM
      for (int ci = 0; ci < P.b_nc[b]; ++ci) {
        P.b_cid[ci] = P.b_cid[b * 4 + ci];
        P.act[ci] = static_cast<uint32_t>(P.b_cid[ci]) | (ozb::kActFlush << 10) | (static_cast<uint32_t>(ci) << 12);
      }
      P.b_act0[0] = 0, P.b_act1[0] = P.b_nc[b];
      P.park_slots = 0;
      P.nbatch = 1, P.npass = q1 - q0;
    }
  }
#endif
  for (size_t g = 0; g < S.agroups.size(); ++g) {
    P.ag_s[g] = static_cast<uint8_t>(S.agroups[g].s);
    P.ag_p0[g] = static_cast<uint16_t>(S.agroups[g].p0);
    P.ag_p1[g] = static_cast<uint16_t>(S.agroups[g].p1);
  }
}

bool schedule_fits(const ozb::Schedule& S) {
  return S.batches.size() <= static_cast<size_t>(ozb::kMaxBatches) &&
         S.acts.size() <= static_cast<size_t>(ozb::kMaxActs) && S.park_slots <= ozb::kMaxPark &&
         S.passes.size() <= static_cast<size_t>(ozb::kMaxPasses) &&
         S.products.size() <= static_cast<size_t>(ozb::kMaxProducts) &&
         S.chunks.size() <= static_cast<size_t>(ozb::kMaxChunks) &&
         S.agroups.size() <= static_cast<size_t>(ozb::kMaxAGroups);
}

// Single-CTA kernel: 128 x kBN tile per CTA.
template <int kBN>
int launch_gemm_bn(Handle* h, int64_t m, int64_t n, int64_t p, int k, int beta_bits, int64_t r,
                   const int8_t* As, int64_t lds_a, int64_t plane_a, const double* mu, const int8_t* Bs,
                   int64_t lds_b, int64_t plane_b, const double* nu, double alpha, double beta, const double* Cin,
                   double* Cout, int64_t ldc, int32_t* dump, const FlushCfg& fl) {
  using Cfg = ozb::GemmCfg<kBN>;
  const size_t budget = h->smem_optin - kSmemReserve - kBN * sizeof(double);
  const int64_t max_stage = static_cast<int64_t>(budget / 3);
  auto slot_bytes = [](int a, int b) {
    return static_cast<int64_t>(a) * Cfg::kATile + static_cast<int64_t>(b) * Cfg::kBTile;
  };
  const ozb::Schedule S =
      ozb::make_schedule(k, fl.per_product ? 1 : r, Cfg::kNAcc, max_stage, slot_bytes);
  if (!schedule_fits(S))
    return set_err(h, OZMM_ERR_UNSUPPORTED, "schedule too large (k=%d, r=%lld)", k,
                   static_cast<long long>(r));
  const size_t stage_bytes = slot_bytes(S.a_slots, S.b_slots);
  const int stages = static_cast<int>(std::min<size_t>(8, budget / stage_bytes));
  if (stages < 2)
    return set_err(h, OZMM_ERR_UNSUPPORTED, "pipeline stage (%zu B) exceeds smem budget",
                   stage_bytes);
  ozb::GemmParams P;  // ~3 KB, passed by value as __grid_constant__
  const int tiles_m = static_cast<int>((m + ozb::kBM - 1) / ozb::kBM);
  const int tiles_n = static_cast<int>((p + kBN - 1) / kBN);
  fill_params(P, S, m, p, lds_a, lds_b, tiles_m, tiles_n, beta_bits, stages, alpha, beta, mu, nu,
              Cin, Cout, ldc, dump, fl);
  CUtensorMap map_a, map_b;
  if (int rc = make_slice_map(h, &map_a, As, lds_a, m, plane_a, k, ozb::kBM)) return rc;
  if (int rc = make_slice_map(h, &map_b, Bs, lds_b, p, plane_b, k, kBN)) return rc;
  const size_t smem = stages * stage_bytes + kSmemReserve + kBN * sizeof(double);
  const int bn_idx = kBN == 32 ? 0 : (kBN == 64 ? 1 : 2);
  if (!h->gemm_attr_set[bn_idx]) {
    CUDA_TRY(h, cudaFuncSetAttribute(ozb::ozimmu_gemm_kernel<kBN>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(h->smem_optin)));
    h->gemm_attr_set[bn_idx] = true;
  }
  const dim3 grid(static_cast<unsigned>(tiles_m * tiles_n));
  ozb::ozimmu_gemm_kernel<kBN><<<grid, ozb::kGemmThreads, smem, h->stream>>>(map_a, map_b, P);
  CUDA_TRY(h, cudaGetLastError());
  return OZMM_OK;
}

// CTA-pair kernel: 256 x kBN tile per 2-CTA cluster (cta_group::2).
template <int kBN, int kPairs>
int launch_gemm_pair(Handle* h, int64_t m, int64_t n, int64_t p, int k, int beta_bits, int64_t r,
                     const int8_t* As, int64_t lds_a, int64_t plane_a, const double* mu, const int8_t* Bs,
                     int64_t lds_b, int64_t plane_b, const double* nu, double alpha, double beta,
                     const double* Cin, double* Cout, int64_t ldc, int32_t* dump,
                     const FlushCfg& fl) {
  using Cfg = ozb::PairCfg<kBN, kPairs>;
  // passes are limited by the resident B slices per K block (A slices stream)
  auto slot_bytes = [](int, int b) { return static_cast<int64_t>(b) * Cfg::kBTile; };
  ozb::PassCost cm;
  cm.a_tile /= kPairs;  // the 4-CTA variant multicasts A: each CTA fills half
  if (const char* e = OZMM_ENV("OZMM_SCHED_BATCH")) cm.batch = std::atof(e);
  if (const char* e = OZMM_ENV("OZMM_SCHED_FILL"))  // scale of the fill terms
    cm.a_tile *= std::atof(e), cm.b_tile *= std::atof(e);
  if (const char* e = OZMM_ENV("OZMM_SCHED")) cm.greedy = std::string(e) == "greedy";
  // A groups alternate large and small when every batch is a single pass (k <= 8:
  // all B slices resident), so that the two-group issue rounds are even (8+1,
  // 7+2, ... products): C3 +3-4 % (profiles/r1/aorder_g2.txt).  Multi-window
  // schedules (k >= 9) keep the sorted order (C5 k=12: -1.7 % interleaved).
  // B slices resident per K block (the window of a pass); OZMM_BWIN (diag) probes
  // wider windows at the cost of A-ring depth
  int bwin = Cfg::kMaxBSlots;
  if (const char* e = OZMM_ENV("OZMM_BWIN")) bwin = std::max(1, std::min(12, std::atoi(e)));
  cm.interleave = k <= bwin;
  if (const char* e = OZMM_ENV("OZMM_AORDER")) cm.interleave = std::string(e) == "interleave";
  // ... and no two consecutive products into one accumulator (C3 +1 %)
  cm.avoid_raw = cm.interleave;
  if (const char* e = OZMM_ENV("OZMM_AVOID_RAW")) cm.avoid_raw = std::atoi(e) != 0;
  const int64_t r_eff = fl.per_product ? 1 : r;
  ozb::Schedule S = ozb::make_schedule(k, r_eff, Cfg::kNAcc, static_cast<int64_t>(bwin) * Cfg::kBTile,
                                       slot_bytes, bwin, cm);
  // Chunks batched by shared A slices instead of in flush order, the ones ahead
  // of their turn parked by the epilogue (schedule.hpp make_schedule_free): taken
  // whenever the model says cheaper -- small r (C4: 26 -> 12 A loads per K block,
  // +58 %) and the r = 8 schedules with split groups (C5 k = 10 / 12 / 14: +4 /
  // +15 / +12 %; profiles/r2/park_schedules.txt).  Results are unchanged: the
  // INT32 sums are exact and the FP64 flushes keep their order.
  {
    int free_mode = -1;  // -1 auto, 0 off, 1 on when it fits
    if (const char* e = OZMM_ENV("OZMM_SCHED_FREE")) free_mode = std::atoi(e);
    if (free_mode != 0) {
      ozb::Schedule F = ozb::make_schedule_free(k, r_eff, Cfg::kNAcc, static_cast<int64_t>(bwin) * Cfg::kBTile,
                                                slot_bytes, bwin, cm);
      if (F.park_slots > 0 && schedule_fits(F) &&
          (free_mode == 1 || ozb::schedule_cost(F, cm) < 0.995 * ozb::schedule_cost(S, cm)))
        S = std::move(F);
    }
  }
  // OZMM_SCHED_SETS (diag): explicit batches as chunk ids in execution order,
  // "0.1.2/3.4.5/6.7.8.9" -- chunks ahead of their turn are parked as usual
  if (const char* e = OZMM_ENV("OZMM_SCHED_SETS")) {
    std::vector<std::vector<int>> sets(1);
    int v = -1;
    for (const char* c = e;; ++c) {
      if (*c >= '0' && *c <= '9') {
        v = (v < 0 ? 0 : 10 * v) + (*c - '0');
        continue;
      }
      if (v >= 0) sets.back().push_back(v), v = -1;
      if (*c == '/') sets.emplace_back();
      if (*c == '\0') break;
    }
    ozb::Schedule X;
    X.chunks = ozb::make_chunks(k, r_eff);
    std::vector<int> seen(X.chunks.size(), 0);
    bool ok = true;
    for (const auto& s : sets) {
      ok = ok && !s.empty() && static_cast<int>(s.size()) <= Cfg::kNAcc;
      for (int c : s) ok = ok && c < static_cast<int>(seen.size()) && !seen[c]++;
    }
    for (int x : seen) ok = ok && x == 1;
    if (!ok) return set_err(h, OZMM_ERR_ARG, "OZMM_SCHED_SETS: not a partition of the %d chunks",
                            static_cast<int>(X.chunks.size()));
    ozb::detail::build_batches(X, sets, slot_bytes, static_cast<int64_t>(bwin) * Cfg::kBTile, bwin, cm);
    S = std::move(X);
  }
  if (!schedule_fits(S))
    return set_err(h, OZMM_ERR_UNSUPPORTED, "schedule too large (k=%d, r=%lld)", k,
                   static_cast<long long>(r));
  // K-pair decision (the kernel re-derives it per pass from P.kpair and the B
  // buffer size): thin passes in K-block pairs (runs of 8 MMAs per accumulator):
  // +4 % at C5 (k = 12), +1 % at C4, C2 +2 %.  Round 1 measured -3 % at the
  // two-batch C3 (profiles/r1/kpair_ab.txt) and kept it off there; after the
  // round-2 epilogue and the K-snake pass order it is +0.4..+3.5 % at C3 (two boxes,
  // profiles/r2/kpair_c3.txt), so it is on everywhere.
  int kpair = 1;
  if (fl.kpair) kpair = fl.kpair == 2 ? 1 : 0;
  if (const char* g = OZMM_ENV("OZMM_KPAIR")) kpair = std::atoi(g);
  const int n_kb = static_cast<int>((std::max(lds_a, lds_b) + ozb::kKB - 1) / ozb::kKB);
  // B buffers sized for the widest pass (two K blocks of a K-pair pass)
  int b_slots = 1;
  for (const auto& q : S.passes) {
    const int nbw = q.bhi - q.blo + 1;
    const bool pair_kb = kPairs == 1 && kpair && 2 * nbw <= bwin && n_kb % 2 == 0;
    b_slots = std::max(b_slots, pair_kb ? 2 * nbw : nbw);
  }
  const size_t fixed = Cfg::smem_bytes(b_slots, 0);
  // A-ring depth.  When each A tile feeds >= 2.5 products on average (tensor-bound
  // schedules, e.g. C3), 5 stages, not the 6 that fit.  With one A group per
  // barrier round, a deeper ring let each CTA pair run further ahead along K:
  // the tiles of a wave drifted apart and stopped sharing slice tiles in L2 (C3,
  // 6 vs 4 stages: 233 vs 148 GB of DRAM reads, clock 1.43 vs 1.55 GHz; 4 was
  // best, tools/stage_ncu.sh).  With two groups per round (P.group_pairs) a
  // round holds two slots, and 5 stages beat 4 by 2 % (DRAM 86 GB).  Schedules
  // with few products per A tile (C4: r = 2, 1.4 per tile) are L2-throughput
  // bound and keep 6.
  int64_t a_loads = 0;
  for (const auto& q : S.passes) a_loads += q.g1 - q.g0;
  const bool dense = a_loads > 0 && 2 * static_cast<int64_t>(S.products.size()) >= 5 * a_loads;
  const size_t fit = std::min<size_t>(Cfg::kMaxStages, (h->smem_optin - fixed) / Cfg::kATile);
  int stages = static_cast<int>(std::min<size_t>(dense ? 5 : 6, fit));
  if (fl.stages) stages = static_cast<int>(std::min<size_t>(fit, std::max(2, fl.stages)));
  if (const char* e = OZMM_ENV("OZMM_STAGES"))
    stages = static_cast<int>(std::min<size_t>(fit, std::max(2, std::atoi(e))));
  if (stages < 2)
    return set_err(h, OZMM_ERR_UNSUPPORTED, "A ring does not fit shared memory");
  // the C pass stages the FP64 tile in the operand pools: grow the B buffers if
  // a small schedule leaves the pools short of it
  while (Cfg::smem_bytes(b_slots, stages) - Cfg::smem_bytes(0, 0) < Cfg::kStageBytes) ++b_slots;
  if (Cfg::smem_bytes(b_slots, stages) > h->smem_optin)
    return set_err(h, OZMM_ERR_UNSUPPORTED, "operand pools do not fit shared memory");
  ozb::GemmParams P;
  const int tiles_m = static_cast<int>((m + 2 * ozb::kBM - 1) / (2 * ozb::kBM));
  const int tiles_n = static_cast<int>((p + kPairs * kBN - 1) / (kPairs * kBN));
  fill_params(P, S, m, p, lds_a, lds_b, tiles_m, tiles_n, beta_bits, stages, alpha, beta, mu, nu,
              Cin, Cout, ldc, dump, fl);
  P.n_kb = n_kb;
  P.kpair = kpair;
  P.b_buf_slots = b_slots;
  if (S.park_slots > 0) {
    // kMaxPark slots per SM id (the kernel indexes by %smid; one CTA per SM, below):
    // a fixed stride, so concurrent launches on the handle's streams that park
    // different numbers of chunks never share a region
    const size_t want = static_cast<size_t>(kParkSmIds) * ozb::kMaxPark * ozb::kBM * kBN;
    if (int rc = ensure(h, &h->park, &h->park_n, want)) return rc;
    P.park = h->park;
  }
  for (const auto& ps : S.passes)
    for (int i = ps.p0; i < ps.p1; ++i) {
      const auto& pr = S.products[i];
      P.pr_info[i] = static_cast<uint32_t>(((pr.t - ps.blo) * Cfg::kBTile) >> 4) |
                     (static_cast<uint32_t>(pr.ci) << 16) | (pr.first ? 1u << 24 : 0u);
    }
  // raster: tensor-bound schedules visit 4 pair-row-blocks per group (a wave of
  // 74 tiles then spans ~4 x 18 tiles and re-reads less of B from DRAM: C3 DRAM
  // 135 -> 82 GB, +3 %; tools/group_ncu.sh); L2-bound ones (C4) keep 2
  if (!OZMM_ENV("OZMM_GROUP_M")) P.group_m = dense ? 4 : 2;
  CUtensorMap map_a, map_b;
  if (int rc = make_slice_map(h, &map_a, As, lds_a, m, plane_a, k, Cfg::kAPart, ozb::kKB,
                              CU_TENSOR_MAP_SWIZZLE_128B))
    return rc;
  if (int rc = make_slice_map(h, &map_b, Bs, lds_b, p, plane_b, k, Cfg::kBHalf, ozb::kKB,
                              CU_TENSOR_MAP_SWIZZLE_128B))
    return rc;
  if (fl.biased() && (fl.per_product || fl.scale_mode != 0))
    return set_err(h, OZMM_ERR_UNSUPPORTED, "offset-binary slices need the CTA-pair ozIMMU_H kernel");
  size_t smem = Cfg::smem_bytes(b_slots, stages);
  // parked chunks live in per-SM scratch: never two CTAs on one SM
  if (S.park_slots > 0) smem = std::max(smem, static_cast<size_t>(h->smem_optin / 2 + 1024));
  if (!h->pair_attr_set[kPairs - 1]) {
    CUDA_TRY(h, cudaFuncSetAttribute(ozb::ozimmu_gemm_pair_kernel<kBN, kPairs>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(h->smem_optin)));
    h->pair_attr_set[kPairs - 1] = true;
  }
  const dim3 grid(static_cast<unsigned>(Cfg::kCluster * tiles_m * tiles_n));
  // OZMM_TILE_TRACE=1 (diagnostics): per-CTA globaltimer stamps, summarised on stderr
  const bool ttrace = OZMM_ENV("OZMM_TILE_TRACE") != nullptr;
  uint64_t* tbuf = nullptr;
  constexpr int kTS = ozb::kTraceSlots;
  if (ttrace) {
    CUDA_TRY(h, cudaMalloc(&tbuf, sizeof(uint64_t) * kTS * grid.x));
    CUDA_TRY(h, cudaMemsetAsync(tbuf, 0, sizeof(uint64_t) * kTS * grid.x, h->stream));
    P.tile_trace = tbuf;
  }
  ozb::ozimmu_gemm_pair_kernel<kBN, kPairs>
      <<<grid, ozb::kPairThreads, smem, h->stream>>>(map_a, map_b, P);
  CUDA_TRY(h, cudaGetLastError());
  if (ttrace) {
    std::vector<uint64_t> t(kTS * static_cast<size_t>(grid.x));
    CUDA_TRY(h, cudaMemcpyAsync(t.data(), tbuf, t.size() * 8, cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    cudaFree(tbuf);
    // mean interval between consecutive stamps over leader CTAs (us), plus the
    // MMA thread's / producer's wait shares and the epilogue drain times
    double sum[8] = {}, tot = 0, w[16] = {}, drain0 = 0, drainl = 0, mma0 = 0;
    int cnt = 0;
    uint64_t t_min = ~0ull, t_max = 0;
    for (unsigned c = 0; c < grid.x; c += Cfg::kCluster) {
      const uint64_t* r = t.data() + kTS * c;
      if (!r[0] || !r[7]) continue;
      ++cnt;
      t_min = std::min(t_min, r[0]);
      t_max = std::max(t_max, r[7]);
      uint64_t prev = r[0];
      for (int i = 1; i < 8; ++i)
        if (r[i]) {
          sum[i] += static_cast<double>(r[i] - prev) * 1e-3;
          prev = r[i];
        }
      tot += static_cast<double>(r[7] - r[0]) * 1e-3;
      for (int i = 8; i < 16; ++i) w[i] += static_cast<double>(r[i]);
      if (r[12] && r[2]) mma0 += static_cast<double>(r[12] - r[2]) * 1e-3;
      const uint64_t d0 = P.nbatch > 1 ? r[3] : r[5];
      if (r[12] && d0 > r[12]) drain0 += static_cast<double>(d0 - r[12]) * 1e-3;
      if (r[13] && r[5] > r[13]) drainl += static_cast<double>(r[5] - r[13]) * 1e-3;
    }
    const double n = cnt ? cnt : 1, mt = w[11] > 0 ? w[11] : 1;
    std::fprintf(stderr,
                 "[ozmm tile trace] %d tiles, launch span %.2f ms, mean tile %.1f us: prologue %.1f | to 1st MMA %.1f |"
                 " batch0 %.1f | to next MMA %.1f | rest %.1f | C write %.1f | teardown %.1f\n"
                 "[ozmm tile trace] batch0 MMAs %.1f us, drain %.1f us; last drain %.1f us | MMA thread "
                 "%.0f clk/tile: waits A %.1f%% B %.1f%% TMEM %.1f%% | producer waits A-slot %.1f%% B-slot %.1f%%\n",
                 cnt, (t_max - t_min) * 1e-6, tot / n, sum[1] / n, sum[2] / n, sum[3] / n, sum[4] / n,
                 sum[5] / n, sum[6] / n, sum[7] / n, mma0 / n, drain0 / n, drainl / n, w[11] / n,
                 100 * w[8] / mt, 100 * w[9] / mt, 100 * w[10] / mt, 100 * w[14] / mt, 100 * w[15] / mt);
  }
  return OZMM_OK;
}

// The kernel launch_gemm picks for these options is a CTA-pair one (<128, 1>
// or the 4-CTA <128, 2>), which can run on offset-binary planes.
bool pair_kernel_selected(const ozmm_options_t* opt) {
  const int tile_n = opt ? opt->tile_n : 0;
  const int pair = opt ? opt->cta_pair : 0;
  return pair == 2 || pair == 3 || (pair == 0 && tile_n == 0);
}

// Offset-binary planes for the ozIMMU_H hot path unless the caller asks for
// the signed ones (options / OZMM_SIGNED=1) or another kernel runs.
bool use_offset_planes(const ozmm_options_t* opt, const MethodCfg& mc) {
  if (opt && opt->signed_slices) return false;
  if (const char* e = OZMM_ENV("OZMM_SIGNED"))
    if (std::atoi(e) != 0) return false;
  return mc.strategy == kRNConstShift && !mc.per_product && pair_kernel_selected(opt);
}

int launch_gemm(Handle* h, int64_t m, int64_t n, int64_t p, int k, int beta_bits, int64_t r,
                const int8_t* As, int64_t lds_a, int64_t plane_a, const double* mu, const int8_t* Bs,
                int64_t lds_b, int64_t plane_b, const double* nu, double alpha, double beta, const double* Cin, double* Cout,
                int64_t ldc, const ozmm_options_t* opt, const FlushCfg& fl_in = FlushCfg{}) {
  int32_t* dump = opt ? opt->chunk_dump : nullptr;
  FlushCfg fl = fl_in;
  if (opt) {
    if (opt->kpair < 0 || opt->kpair > 2 || opt->stages < 0)
      return set_err(h, OZMM_ERR_ARG, "options: kpair must be 0..2 and stages >= 0");
    fl.kpair = opt->kpair;
    fl.stages = opt->stages;
  }
  if (fl.biased() && !pair_kernel_selected(opt))
    return set_err(h, OZMM_ERR_UNSUPPORTED, "offset-binary slices need the CTA-pair kernel");
  const int tile_n = opt ? opt->tile_n : 0;
  const int pair = opt ? opt->cta_pair : 0;
  if (pair == 3 || (pair == 0 && tile_n == 0 && OZMM_ENV("OZMM_QUAD")))
    return launch_gemm_pair<128, 2>(h, m, n, p, k, beta_bits, r, As, lds_a, plane_a, mu, Bs, lds_b,
                                    plane_b, nu, alpha, beta, Cin, Cout, ldc, dump, fl);
  if (pair == 2 || (pair == 0 && tile_n == 0))
    return launch_gemm_pair<128, 1>(h, m, n, p, k, beta_bits, r, As, lds_a, plane_a, mu, Bs, lds_b, plane_b, nu, alpha,
                                 beta, Cin, Cout, ldc, dump, fl);
  switch (tile_n ? tile_n : 64) {
    case 32:
      return launch_gemm_bn<32>(h, m, n, p, k, beta_bits, r, As, lds_a, plane_a, mu, Bs, lds_b, plane_b, nu, alpha,
                                beta, Cin, Cout, ldc, dump, fl);
    case 64:
      return launch_gemm_bn<64>(h, m, n, p, k, beta_bits, r, As, lds_a, plane_a, mu, Bs, lds_b, plane_b, nu, alpha,
                                beta, Cin, Cout, ldc, dump, fl);
    case 128:
      return launch_gemm_bn<128>(h, m, n, p, k, beta_bits, r, As, lds_a, plane_a, mu, Bs, lds_b, plane_b, nu,
                                 alpha, beta, Cin, Cout, ldc, dump, fl);
    default:
      return set_err(h, OZMM_ERR_ARG, "tile_n must be 32, 64 or 128 (got %d)", tile_n);
  }
}

// ---- OverflowMode::Checked ------------------------------------------------------
// The reference checks every running INT32 chunk sum after each slice product in
// int64 and throws OverflowError outside INT32 (gemm_wide, int_gemm.cpp:37-59; the
// INT32 fast path runs only when no entry can leave the range, :213-219).  The
// tensor core wraps, so the GPU verifies instead -- but only where an overflow is
// possible at all, i.e. where a chunk's bound n * sum max|A_s| max|B_t| exceeds
// INT32_MAX.  With the derived beta and r that never happens (r n 2^(2 beta) <=
// 2^31 and max|slice| <= 2^beta - 1, int_gemm.cpp:24-25); force_beta / force_r can.
//
// max |slice s| (1-based): RN constant shift 2^beta - 1 for s = 1 (the bump rule,
// split.cpp:126-129) and 2^(beta-1) after it (round to nearest); bitmask fields
// and per-slice RN 2^beta - 1 (split.cpp:60, :121-130).
int64_t slice_max(Strategy st, int beta, int s) {
  if (st == kRNConstShift && s >= 2) return int64_t(1) << (beta - 1);
  return (int64_t(1) << beta) - 1;
}

// 0: no overflow possible; 1: possible, verifiable per product; -1: a single
// product may already leave INT32 (its wrapped value cannot be verified).
int overflow_possible(Strategy st, bool per_product, int k, int64_t r, int beta, int64_t n) {
  const int64_t lim = INT32_MAX;
  int verdict = 0;
  for (const ozb::Chunk& c : ozb::make_chunks(k, per_product ? 1 : r)) {
    int64_t sum = 0;
    for (int s0 = c.s0; s0 <= c.s1; ++s0) {
      const int64_t one = slice_max(st, beta, s0) * slice_max(st, beta, c.g - s0);
      if (n > lim / one) return -1;  // n * one > INT32_MAX
      sum += one;
    }
    if (sum > lim / n) verdict = 1;
  }
  return verdict;
}

// Exact INT32 range check of the running chunk sums.  prod [P][m][p]: the exact
// per-product sums A_s B_t in flush order (a chunk schedule with r = 1); the
// chunks of the real r are replayed over them (scheme.cpp:81-101).  first: the
// earliest (product, entry) that leaves INT32 as product << 40 | entry.
__global__ void checked_overflow_kernel(const int32_t* __restrict__ prod, int64_t mp, int k,
                                        int64_t r, unsigned long long* first) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < mp;
       e += int64_t(gridDim.x) * blockDim.x) {
    int64_t q = 0;
    for (int g = 2; g <= k + 1; ++g) {
      int64_t acc = 0, cnt = 0;
      for (int s = 1; s <= g - 1; ++s, ++q) {
        acc += prod[q * mp + e];
        if (acc < INT32_MIN || acc > INT32_MAX) {
          atomicMin(first, (static_cast<unsigned long long>(q) << 40) | static_cast<unsigned long long>(e));
          return;
        }
        if (++cnt == r || s == g - 1) acc = 0, cnt = 0;
      }
    }
  }
}

int check_range_sync(Handle* h) {
  int f[2] = {0, 0};
  CUDA_TRY(h, cudaMemcpyAsync(f, h->flags, sizeof f, cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  if (f[1]) {
    CUDA_TRY(h, cudaMemsetAsync(h->flags + 1, 0, sizeof(int), h->stream));
    return set_err(h, OZMM_ERR_RANGE, "split: row magnitude too large for shift extraction");
  }
  return OZMM_OK;
}

int gemm_slices_checked(Handle* h, int64_t m, int64_t n, int64_t p, int k, int beta_bits,
                        int64_t r, const int8_t* As, int64_t lds_a, int64_t plane_a,
                        const double* mu, const int8_t* Bs, int64_t lds_b, int64_t plane_b,
                        const double* nu, double alpha, double beta, double* C, int64_t ldc,
                        const ozmm_options_t* opt, const FlushCfg& fl);

// OverflowMode::Checked verification of one call's split operands (see
// overflow_possible): the per-product sums (the fused kernel's chunk dump with r
// = 1, into scratch), then the running sums of the real chunks.  Synchronous;
// returns OZMM_ERR_OVERFLOW with the reference's message, before C is written.
int verify_no_overflow(Handle* h, int64_t m, int64_t n, int64_t p, int k, int beta_bits, int64_t r,
                       const int8_t* As, int64_t lds, const double* mu, const int8_t* Bs,
                       const double* nu, const ozmm_options_t* opt, const FlushCfg& fl) {
  if (int rc = check_range_sync(h)) return rc;  // the split throws first (split.cpp:124)
  const int64_t np = int64_t(k) * (k + 1) / 2, mp = m * p;
  int32_t* prod = nullptr;
  double* scratch = nullptr;
  unsigned long long* first = nullptr;
  auto release = [&] {
    cudaFree(prod);
    cudaFree(scratch);
    cudaFree(first);
  };
  if (cudaMalloc(&prod, sizeof(int32_t) * np * mp) != cudaSuccess ||
      cudaMalloc(&scratch, sizeof(double) * mp) != cudaSuccess ||
      cudaMalloc(&first, sizeof(unsigned long long)) != cudaSuccess) {
    release();
    cudaGetLastError();
    return set_err(h, OZMM_ERR_CUDA, "Checked overflow verification: out of device memory "
                   "(%lld x %lld x %lld INT32 sums); use overflow_wrap", static_cast<long long>(np),
                   static_cast<long long>(m), static_cast<long long>(p));
  }
  ozmm_options_t o = opt ? *opt : ozmm_options_t{};
  o.chunk_dump = prod;
  int rc = launch_gemm(h, m, n, p, k, beta_bits, 1, As, lds, m * lds, mu, Bs, lds, p * lds, nu,
                       1.0, 0.0, nullptr, scratch, p, &o, fl);
  unsigned long long hit = ~0ull;
  if (rc == OZMM_OK) {
    cudaMemsetAsync(first, 0xFF, sizeof hit, h->stream);
    const int64_t blocks = std::min<int64_t>((mp + 255) / 256, int64_t(h->num_sms) * 8);
    checked_overflow_kernel<<<static_cast<unsigned>(blocks), 256, 0, h->stream>>>(prod, mp, k, r, first);
    cudaMemcpyAsync(&hit, first, sizeof hit, cudaMemcpyDeviceToHost, h->stream);
    const cudaError_t e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) rc = set_err(h, OZMM_ERR_CUDA, "overflow check: %s", cudaGetErrorString(e));
  }
  if (rc == OZMM_OK && hit != ~0ull) {
    const int64_t q = static_cast<int64_t>(hit >> 40), e = static_cast<int64_t>(hit & ((1ull << 40) - 1));
    std::vector<int32_t> v(static_cast<size_t>(np));
    cudaMemcpy2D(v.data(), sizeof(int32_t), prod + e, sizeof(int32_t) * mp, sizeof(int32_t), np,
                 cudaMemcpyDeviceToHost);
    // replay the entry's chunks up to product q for the exact value
    int64_t qq = 0, val = 0;
    for (int g = 2; g <= k + 1 && qq <= q; ++g) {
      int64_t acc = 0, cnt = 0;
      for (int s0 = 1; s0 <= g - 1 && qq <= q; ++s0, ++qq) {
        acc += v[qq];
        val = acc;
        if (++cnt == r || s0 == g - 1) acc = 0, cnt = 0;
      }
    }
    rc = set_err(h, OZMM_ERR_OVERFLOW, "i8_gemm: INT32 overflow at (%lld, %lld), exact value %lld",
                 static_cast<long long>(e / p), static_cast<long long>(e % p), static_cast<long long>(val));
  }
  release();
  return rc;
}

}  // namespace

// =============================================================================
extern "C" {

int ozmm_create(ozmm_handle_t* out, int device) {
  if (!out) return set_err(nullptr, OZMM_ERR_ARG, "null handle pointer");
  Handle* h = new Handle();
  h->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) {
    delete h;
    return set_err(nullptr, OZMM_ERR_CUDA, "cudaSetDevice(%d): %s", device, cudaGetErrorString(e));
  }
  int major = 0, minor = 0, sms = 0, optin = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  if (major != 10 || minor != 0) {
    delete h;
    return set_err(nullptr, OZMM_ERR_UNSUPPORTED,
                   "device %d is sm_%d%d; this library is built for sm_100a (B200) only", device,
                   major, minor);
  }
  h->num_sms = sms;
  h->smem_optin = static_cast<size_t>(optin);
  if (cudaMalloc(&h->flags, kNumFlags * sizeof(int)) != cudaSuccess ||
      cudaMemset(h->flags, 0, kNumFlags * sizeof(int)) != cudaSuccess) {
    delete h;
    return set_err(nullptr, OZMM_ERR_CUDA, "flag allocation failed");
  }
  for (auto& ev : h->ev) cudaEventCreate(&ev);
  *out = reinterpret_cast<ozmm_handle_t>(h);
  return OZMM_OK;
}

int ozmm_destroy(ozmm_handle_t handle) {
  Handle* h = reinterpret_cast<Handle*>(handle);
  if (!h) return OZMM_OK;
  cudaSetDevice(h->device);
  cudaFree(h->slices_a);
  cudaFree(h->slices_b);
  cudaFree(h->mu);
  cudaFree(h->nu);
  cudaFree(h->colmax);
  cudaFree(h->flags);
  cudaFree(h->units_a);
  cudaFree(h->units_b);
  cudaFree(h->tscratch);
  cudaFree(h->lsa);
  cudaFree(h->lsb);
  cudaFree(h->park);
  cudaFree(h->host_a);
  cudaFree(h->host_b);
  cudaFree(h->host_c);
  cudaFree(h->host_o);
  if (h->s_in) cudaStreamDestroy(h->s_in);
  if (h->s_out) cudaStreamDestroy(h->s_out);
  if (h->s_split) cudaStreamDestroy(h->s_split);
  for (auto sg : h->s_gemm)
    if (sg) cudaStreamDestroy(sg);
  if (h->s_aux) cudaStreamDestroy(h->s_aux);
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_join) cudaEventDestroy(h->ev_join);
  if (h->hflags) cudaFreeHost(h->hflags);
  for (auto& ev : h->ev) cudaEventDestroy(ev);
  h->stage_in.release();
  h->stage_out.release();
  delete h;
  return OZMM_OK;
}

int ozmm_set_stream(ozmm_handle_t handle, void* stream) {
  Handle* h = reinterpret_cast<Handle*>(handle);
  if (!h) return set_err(nullptr, OZMM_ERR_ARG, "null handle");
  h->stream = static_cast<cudaStream_t>(stream);
  return OZMM_OK;
}

int ozmm_get_stream(ozmm_handle_t handle, void** stream) {
  Handle* h = reinterpret_cast<Handle*>(handle);
  if (!h || !stream) return set_err(h, OZMM_ERR_ARG, "null handle or output");
  *stream = h->stream;
  return OZMM_OK;
}

const char* ozmm_last_error(ozmm_handle_t handle) {
  Handle* h = reinterpret_cast<Handle*>(handle);
  return h ? h->err.c_str() : g_thread_err.c_str();
}

const char* ozmm_status_string(int s) {
  switch (s) {
    case OZMM_OK: return "ok";
    case OZMM_ERR_ARG: return "invalid argument";
    case OZMM_ERR_CONFIG: return "configuration error";
    case OZMM_ERR_RANGE: return "row magnitude too large for shift extraction";
    case OZMM_ERR_CUDA: return "CUDA error";
    case OZMM_ERR_NCCL: return "NCCL error";
    case OZMM_ERR_UNSUPPORTED: return "unsupported";
    default: return "internal error";
  }
}

// Library-internal (hidden, not part of the ABI): the 2-D grid entry
// (ozmm_grid.cpp) starts each call with clear flags and reads this call's range
// flag on the device for its grid-wide max.
__attribute__((visibility("hidden"))) int* ozmm_internal_range_flag(ozmm_handle_t handle) {
  return reinterpret_cast<Handle*>(handle)->flags + 1;
}
__attribute__((visibility("hidden"))) int ozmm_internal_fold_flags(ozmm_handle_t handle) {
  Handle* h = reinterpret_cast<Handle*>(handle);
  fold_flags_kernel<<<1, 1, 0, h->stream>>>(h->flags);
  CUDA_TRY(h, cudaGetLastError());
  return OZMM_OK;
}

int ozmm_sync_status(ozmm_handle_t handle, int* underflow) {
  Handle* h = reinterpret_cast<Handle*>(handle);
  if (!h) return set_err(nullptr, OZMM_ERR_ARG, "null handle");
  int f[kNumFlags] = {};
  CUDA_TRY(h, cudaSetDevice(h->device));
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  CUDA_TRY(h, cudaMemcpy(f, h->flags, sizeof f, cudaMemcpyDeviceToHost));
  CUDA_TRY(h, cudaMemset(h->flags, 0, sizeof f));
  if (underflow) *underflow = f[0] | f[2];
  if (f[1] | f[3]) return set_err(h, OZMM_ERR_RANGE, "split: row magnitude too large for shift extraction");
  return OZMM_OK;
}

size_t ozmm_workspace_bytes(ozmm_handle_t handle) {
  Handle* h = reinterpret_cast<Handle*>(handle);
  if (!h) return 0;
  return h->slices_a_bytes + h->slices_b_bytes +
         8 * (h->mu_n + h->nu_n + h->colmax_n + h->host_a_n + h->host_b_n + h->host_c_n);
}

int ozmm_compute_beta(int64_t n, int* beta) {
  if (!beta) return set_err(nullptr, OZMM_ERR_ARG, "null output");
  if (n < 1) return set_err(nullptr, OZMM_ERR_ARG, "compute_beta: n must be >= 1");
  if (n > (int64_t(1) << 29)) return set_err(nullptr, OZMM_ERR_ARG, "compute_beta: n > 2^29 unsupported");
  *beta = ozb::compute_beta_host(n);
  return OZMM_OK;
}

int ozmm_compute_r(int64_t n, int beta, int64_t* r) {
  if (!r) return set_err(nullptr, OZMM_ERR_ARG, "null output");
  if (n < 1 || beta < 1) return set_err(nullptr, OZMM_ERR_ARG, "compute_r: bad arguments");
  *r = ozb::compute_r_host(n, beta);
  return OZMM_OK;
}

int ozmm_op_counts(int k, int64_t r, ozmm_counts_t* c) {
  if (!c) return set_err(nullptr, OZMM_ERR_ARG, "null output");
  if (k < 1 || r < 1) return set_err(nullptr, OZMM_ERR_CONFIG, "op_counts: bad arguments");
  c->int8_gemms = static_cast<int64_t>(k) * (k + 1) / 2;
  c->r = r;
  c->w = ozb::flush_count_w_host(k, r);
  c->fp64_flushes = c->w;
  return OZMM_OK;
}

int64_t ozmm_slice_ld(int64_t n) { return (n + 15) / 16 * 16; }

int ozmm_debug_schedule(int k, int64_t r, int cta_pair, int tile_n, int* rows, int cap,
                        int* info) {
  if (k < 1 || k > ozb::kMaxK || r < 1 || !rows || !info)
    return set_err(nullptr, OZMM_ERR_ARG, "debug_schedule: bad arguments");
  int n_acc, a_tile, b_tile, bn;
  if (cta_pair == 2 || (cta_pair == 0 && tile_n == 0)) {
    bn = 128;
    n_acc = ozb::PairCfg<128, 1>::kNAcc;
    a_tile = ozb::PairCfg<128, 1>::kATile;
    b_tile = ozb::PairCfg<128, 1>::kBTile;  // per CTA, 128-byte K block
  } else {
    bn = tile_n ? tile_n : 64;
    if (bn != 32 && bn != 64 && bn != 128) return set_err(nullptr, OZMM_ERR_ARG, "tile_n");
    n_acc = 512 / bn;
    a_tile = ozb::kBM * ozb::kBK;
    b_tile = bn * ozb::kBK;
  }
  const size_t budget = 232448 - kSmemReserve - bn * sizeof(double);
  const bool pair_kernel = cta_pair == 2 || (cta_pair == 0 && tile_n == 0);
  auto slot_bytes = [&](int a, int b) {
    return (pair_kernel ? 0 : static_cast<int64_t>(a) * a_tile) + static_cast<int64_t>(b) * b_tile;
  };
  const int64_t max_stage = pair_kernel
                                ? static_cast<int64_t>(ozb::PairCfg<128, 1>::kMaxBSlots) * b_tile
                                : static_cast<int64_t>(budget / 3);
  const ozb::Schedule S = ozb::make_schedule(k, r, n_acc, max_stage, slot_bytes,
                                             pair_kernel ? ozb::PairCfg<128, 1>::kMaxBSlots : 0);
  const int np = static_cast<int>(S.products.size());
  if (np > cap) return set_err(nullptr, OZMM_ERR_ARG, "debug_schedule: cap too small");
  for (int q = 0; q < static_cast<int>(S.passes.size()); ++q) {
    const ozb::Pass& ps = S.passes[q];
    for (int i = ps.p0; i < ps.p1; ++i) {
      const ozb::Product& pr = S.products[i];
      const ozb::Batch& b = S.batches[ps.batch];
      const ozb::Chunk& c = S.chunks[b.cids[pr.ci]];
      int* row = rows + 8 * i;
      row[0] = ps.batch;
      row[1] = q;
      row[2] = b.cids[pr.ci];  // global chunk index (flush order)
      row[3] = c.g;
      row[4] = pr.s;
      row[5] = pr.t;
      row[6] = pr.first ? 1 : 0;
      row[7] = (pr.s >= ps.alo && pr.s <= ps.ahi && pr.t >= ps.blo && pr.t <= ps.bhi) ? 1 : 0;
    }
  }
  const size_t stage_bytes =
      pair_kernel ? static_cast<size_t>(a_tile) : static_cast<size_t>(slot_bytes(S.a_slots, S.b_slots));
  const size_t fixed = pair_kernel ? ozb::kBBufs * ozb::PairCfg<128, 1>::kMaxBSlots * b_tile : 0;
  info[0] = np;
  info[1] = static_cast<int>(S.chunks.size());
  info[2] = static_cast<int>(S.batches.size());
  info[3] = static_cast<int>(S.passes.size());
  info[4] = static_cast<int>(std::min<size_t>(8, (budget - fixed) / stage_bytes));  // stages
  info[5] = S.a_slots;
  info[6] = S.b_slots;
  return OZMM_OK;
}

int ozmm_split(ozmm_handle_t handle, char side, char trans, int64_t lines, int64_t n,
               const double* X, int64_t ldx, int k, int beta, int8_t* slices, int64_t lds,
               double* shift) {
  Handle* h = reinterpret_cast<Handle*>(handle);
  if (!h) return set_err(nullptr, OZMM_ERR_ARG, "null handle");
  if (side != 'L' && side != 'R') return set_err(h, OZMM_ERR_ARG, "side must be 'L' or 'R'");
  if (!valid_trans(trans)) return set_err(h, OZMM_ERR_ARG, "trans must be 'N' or 'T'");
  if (lines < 1 || n < 1) return set_err(h, OZMM_ERR_ARG, "split: empty matrix");
  if (k < 1 || k > ozb::kMaxK) return set_err(h, OZMM_ERR_ARG, "split: k must be in 1..%d", ozb::kMaxK);
  if (lds < ozmm_slice_ld(n) || lds % 16) return set_err(h, OZMM_ERR_ARG, "split: lds too small or not a multiple of 16");
  if (beta == 0) {
    beta = ozb::compute_beta_host(n);
    if (beta < 0) return set_err(h, OZMM_ERR_ARG, "compute_beta: n out of range");
  } else if (beta < 1 || beta > 7) {
    return set_err(h, OZMM_ERR_ARG, "split: forced beta outside 1..7");
  }
  // Left/'N' and Right/'T' have contiguous lines; the others are strided.
  const bool row_mode = (side == 'L') != is_trans(trans);
  const int64_t need_ld = row_mode ? n : lines;
  if (ldx < need_ld) return set_err(h, OZMM_ERR_ARG, "split: leading dimension too small");
  CUDA_TRY(h, cudaSetDevice(h->device));
  return launch_split(h, row_mode, lines, n, X, ldx, k, beta, slices, lds, lines * lds, shift);
}

int ozmm_split_offset(ozmm_handle_t handle, char side, char trans, int64_t lines, int64_t n,
                      const double* X, int64_t ldx, int k, int beta, int8_t* slices, int64_t lds,
                      double* shift, int32_t* lsum, int64_t lsum_plane, int64_t lsum_lstride) {
  return ozmm_split_offset_strided(handle, side, trans, lines, n, X, ldx, k, beta, slices, lds,
                                   lines * lds, shift, lsum, lsum_plane, lsum_lstride);
}

int ozmm_split_offset_strided(ozmm_handle_t handle, char side, char trans, int64_t lines,
                              int64_t n, const double* X, int64_t ldx, int k, int beta,
                              int8_t* slices, int64_t lds, int64_t plane, double* shift,
                              int32_t* lsum, int64_t lsum_plane, int64_t lsum_lstride) {
  Handle* h = reinterpret_cast<Handle*>(handle);
  if (!h) return set_err(nullptr, OZMM_ERR_ARG, "null handle");
  if (side != 'L' && side != 'R') return set_err(h, OZMM_ERR_ARG, "side must be 'L' or 'R'");
  if (!valid_trans(trans)) return set_err(h, OZMM_ERR_ARG, "trans must be 'N' or 'T'");
  if (lines < 1 || n < 1) return set_err(h, OZMM_ERR_ARG, "split: empty matrix");
  if (k < 1 || k > ozb::kMaxK) return set_err(h, OZMM_ERR_ARG, "split: k must be in 1..%d", ozb::kMaxK);
  if (lds < ozmm_slice_ld(n) || lds % 16) return set_err(h, OZMM_ERR_ARG, "split: lds too small or not a multiple of 16");
  if (!lsum || lsum_plane < 1 || lsum_lstride < 1 ||
      !((lsum_lstride == 1 && lsum_plane >= lines) || (lsum_plane == 1 && lsum_lstride >= k)))
    return set_err(h, OZMM_ERR_ARG, "split: line sums need [k][>=lines] or [lines][>=k] strides");
  if (beta == 0) {
    beta = ozb::compute_beta_host(n);
    if (beta < 0) return set_err(h, OZMM_ERR_ARG, "compute_beta: n out of range");
  } else if (beta < 1 || beta > 7) {
    return set_err(h, OZMM_ERR_ARG, "split: forced beta outside 1..7");
  }
  if (plane < lines * lds) return set_err(h, OZMM_ERR_ARG, "split: plane stride below lines * lds");
  const bool row_mode = (side == 'L') != is_trans(trans);
  if (ldx < (row_mode ? n : lines)) return set_err(h, OZMM_ERR_ARG, "split: leading dimension too small");
  CUDA_TRY(h, cudaSetDevice(h->device));
  if (lsum_lstride == 1)
    CUDA_TRY(h, cudaMemset2DAsync(lsum, sizeof(int32_t) * lsum_plane, 0, sizeof(int32_t) * lines, k,
                                  h->stream));
  else
    CUDA_TRY(h, cudaMemset2DAsync(lsum, sizeof(int32_t) * lsum_lstride, 0, sizeof(int32_t) * k, lines,
                                  h->stream));
  return launch_split(h, row_mode, lines, n, X, ldx, k, beta, slices, lds, plane, shift,
                      lsum, lsum_plane, lsum_lstride);
}

int ozmm_gemm_slices_offset(ozmm_handle_t handle, int64_t m, int64_t n, int64_t p, int k,
                            int beta_bits, int64_t r, const int8_t* As, int64_t lds_a,
                            int64_t plane_a, const double* mu, const int32_t* lsa,
                            int64_t lsa_plane, int64_t lsa_lstride, const int8_t* Bs, int64_t lds_b,
                            int64_t plane_b, const double* nu, const int32_t* lsb,
                            int64_t lsb_plane, int64_t lsb_lstride, double alpha, double beta,
                            double* C, int64_t ldc, const ozmm_options_t* opt) {
  Handle* h = reinterpret_cast<Handle*>(handle);
  if (!h) return set_err(nullptr, OZMM_ERR_ARG, "null handle");
  if (!lsa || !lsb || lsa_plane < 1 || lsb_plane < 1 || lsa_lstride < 1 || lsb_lstride < 1)
    return set_err(h, OZMM_ERR_ARG, "line sums missing or bad strides");
  if (!pair_kernel_selected(opt))
    return set_err(h, OZMM_ERR_UNSUPPORTED, "offset-binary slices need the CTA-pair kernel");
  FlushCfg fl;
  fl.lsa = lsa;
  fl.lsb = lsb;
  fl.lsa_plane = lsa_plane;
  fl.lsb_plane = lsb_plane;
  fl.lsa_lstride = lsa_lstride;
  fl.lsb_lstride = lsb_lstride;
  fl.n = n;
  return gemm_slices_checked(h, m, n, p, k, beta_bits, r, As, lds_a, plane_a, mu, Bs, lds_b,
                             plane_b, nu, alpha, beta, C, ldc, opt, fl);
}

int ozmm_split_ex(ozmm_handle_t handle, char side, char trans, int64_t lines, int64_t n,
                  const double* X, int64_t ldx, int k, int beta, int strategy, int8_t* slices,
                  int64_t lds, double* out) {
  Handle* h = reinterpret_cast<Handle*>(handle);
  if (!h) return set_err(nullptr, OZMM_ERR_ARG, "null handle");
  if (strategy < 0 || strategy > 2) return set_err(h, OZMM_ERR_ARG, "unknown split strategy");
  if (side != 'L' && side != 'R') return set_err(h, OZMM_ERR_ARG, "side must be 'L' or 'R'");
  if (!valid_trans(trans)) return set_err(h, OZMM_ERR_ARG, "trans must be 'N' or 'T'");
  if (lines < 1 || n < 1) return set_err(h, OZMM_ERR_ARG, "split: empty matrix");
  if (k < 1 || k > ozb::kMaxK) return set_err(h, OZMM_ERR_ARG, "split: k must be in 1..%d", ozb::kMaxK);
  if (lds < ozmm_slice_ld(n) || lds % 16) return set_err(h, OZMM_ERR_ARG, "split: lds too small or not a multiple of 16");
  if (beta == 0) {
    beta = ozb::compute_beta_host(n);
    if (beta < 0) return set_err(h, OZMM_ERR_ARG, "compute_beta: n out of range");
  } else if (beta < 1 || beta > 7) {
    return set_err(h, OZMM_ERR_ARG, "split: forced beta outside 1..7");
  }
  const bool row_mode = (side == 'L') != is_trans(trans);
  if (ldx < (row_mode ? n : lines)) return set_err(h, OZMM_ERR_ARG, "split: leading dimension too small");
  CUDA_TRY(h, cudaSetDevice(h->device));
  if (strategy == 2)  // per-slice units start at zero (rows that vanish keep 0)
    CUDA_TRY(h, cudaMemsetAsync(out, 0, sizeof(double) * k * lines, h->stream));
  return launch_split_m(h, static_cast<Strategy>(strategy == 0 ? kRNConstShift
                                                 : strategy == 1 ? kBitMask : kRNPerSlice),
                        row_mode, lines, n, X, ldx, k, beta, slices, lds, lines * lds, out);
}

int ozmm_split_host(ozmm_handle_t handle, char side, char trans, int64_t lines, int64_t n, const double* X,
                    int64_t ldx, int k, int beta, int strategy, int8_t* slices, double* out, double* residual) {
  // Host-memory split with its residual (the reference's SplitMatrix as
  // dump_split writes it, split.cpp:254-270): X is uploaded, split on the GPU by
  // ozmm_split_ex, the residual recurrence runs on the GPU
  // (split_residual_kernel), and the results come back line-major.
  Handle* h = reinterpret_cast<Handle*>(handle);
  if (!h) return set_err(nullptr, OZMM_ERR_ARG, "null handle");
  if (!X || !slices || !out) return set_err(h, OZMM_ERR_ARG, "null pointer");
  if (side != 'L' && side != 'R') return set_err(h, OZMM_ERR_ARG, "side must be 'L' or 'R'");
  if (!valid_trans(trans)) return set_err(h, OZMM_ERR_ARG, "trans must be 'N' or 'T'");
  if (lines < 1 || n < 1) return set_err(h, OZMM_ERR_ARG, "split: empty matrix");
  // checked before the workspace is sized from them (ozmm_split_ex repeats it)
  if (strategy < 0 || strategy > 2) return set_err(h, OZMM_ERR_ARG, "unknown split strategy");
  if (k < 1 || k > ozb::kMaxK) return set_err(h, OZMM_ERR_ARG, "split: k must be in 1..%d", ozb::kMaxK);
  const bool row_mode = (side == 'L') != is_trans(trans);
  const int64_t rows = row_mode ? lines : n, cols = row_mode ? n : lines;  // X as stored
  if (ldx < cols) return set_err(h, OZMM_ERR_ARG, "split: leading dimension too small");
  if (beta == 0) {
    beta = ozb::compute_beta_host(n);
    if (beta < 0) return set_err(h, OZMM_ERR_ARG, "compute_beta: n out of range");
  }
  CUDA_TRY(h, cudaSetDevice(h->device));
  const int64_t lds = ozmm_slice_ld(n);
  const size_t nout = static_cast<size_t>(strategy == 2 ? k * lines : lines);
  double *dX = nullptr, *dOut = nullptr, *dR = nullptr;
  int8_t* dS = nullptr;
  int rc = OZMM_OK;
  auto cu = [&](cudaError_t e, const char* what) {
    if (e != cudaSuccess && rc == OZMM_OK) rc = set_err(h, OZMM_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
    return rc == OZMM_OK;
  };
  if (cu(cudaMalloc(&dX, sizeof(double) * rows * cols), "cudaMalloc") &&
      cu(cudaMalloc(&dS, static_cast<size_t>(k) * lines * lds), "cudaMalloc") &&
      cu(cudaMalloc(&dOut, sizeof(double) * nout), "cudaMalloc") &&
      cu(cudaMalloc(&dR, sizeof(double) * lines * n), "cudaMalloc") &&
      cu(cudaMemcpy2DAsync(dX, sizeof(double) * cols, X, sizeof(double) * ldx, sizeof(double) * cols, rows,
                           cudaMemcpyHostToDevice, h->stream), "H2D")) {
    fold_flags_kernel<<<1, 1, 0, h->stream>>>(h->flags);  // this call's range flag starts clear
    rc = ozmm_split_ex(handle, side, trans, lines, n, dX, cols, k, beta, strategy, dS, lds, dOut);
    if (rc == OZMM_OK) rc = check_range_sync(h);  // the reference throws from the split
    if (rc == OZMM_OK) {
      const int64_t total = lines * n;
      ozb::split_residual_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, h->stream>>>(
          dX, cols, row_mode ? 1 : 0, lines, n, k, beta, strategy, dS, lds, lines * lds, dOut, dR);
      cu(cudaGetLastError(), "residual kernel") &&
          cu(cudaMemcpy2DAsync(slices, n, dS, lds, n, static_cast<size_t>(k) * lines, cudaMemcpyDeviceToHost,
                               h->stream), "D2H") &&
          cu(cudaMemcpyAsync(out, dOut, sizeof(double) * nout, cudaMemcpyDeviceToHost, h->stream), "D2H") &&
          (!residual || cu(cudaMemcpyAsync(residual, dR, sizeof(double) * lines * n, cudaMemcpyDeviceToHost,
                                           h->stream), "D2H")) &&
          cu(cudaStreamSynchronize(h->stream), "sync");
    }
  }
  cudaFree(dX);
  cudaFree(dS);
  cudaFree(dOut);
  cudaFree(dR);
  return rc;
}

int ozmm_gemm_slices(ozmm_handle_t handle, int64_t m, int64_t n, int64_t p, int k, int beta_bits,
                     int64_t r, const int8_t* As, int64_t lds_a, const double* mu, const int8_t* Bs,
                     int64_t lds_b, const double* nu, double alpha, double beta, double* C,
                     int64_t ldc, const ozmm_options_t* opt) {
  return ozmm_gemm_slices_strided(handle, m, n, p, k, beta_bits, r, As, lds_a, m * lds_a, mu, Bs,
                                  lds_b, p * lds_b, nu, alpha, beta, C, ldc, opt);
}

int ozmm_gemm_slices_strided(ozmm_handle_t handle, int64_t m, int64_t n, int64_t p, int k,
                             int beta_bits, int64_t r, const int8_t* As, int64_t lds_a,
                             int64_t plane_a, const double* mu, const int8_t* Bs, int64_t lds_b,
                             int64_t plane_b, const double* nu, double alpha, double beta,
                             double* C, int64_t ldc, const ozmm_options_t* opt) {
  Handle* h = reinterpret_cast<Handle*>(handle);
  if (!h) return set_err(nullptr, OZMM_ERR_ARG, "null handle");
  return gemm_slices_checked(h, m, n, p, k, beta_bits, r, As, lds_a, plane_a, mu, Bs, lds_b,
                             plane_b, nu, alpha, beta, C, ldc, opt, FlushCfg{});
}

}  // extern "C"

namespace {
// argument checks shared by the two slice-level GEMM entries
int gemm_slices_checked(Handle* h, int64_t m, int64_t n, int64_t p, int k, int beta_bits,
                        int64_t r, const int8_t* As, int64_t lds_a, int64_t plane_a,
                        const double* mu, const int8_t* Bs, int64_t lds_b, int64_t plane_b,
                        const double* nu, double alpha, double beta, double* C, int64_t ldc,
                        const ozmm_options_t* opt, const FlushCfg& fl) {
  if (m < 1 || n < 1 || p < 1) return set_err(h, OZMM_ERR_ARG, "empty shape");
  if (m > INT32_MAX || p > INT32_MAX) return set_err(h, OZMM_ERR_ARG, "m, p must fit int32");
  if (k < 1 || k > ozb::kMaxK) return set_err(h, OZMM_ERR_CONFIG, "k must be in 1..%d", ozb::kMaxK);
  if (beta_bits < 1 || beta_bits > 7) return set_err(h, OZMM_ERR_ARG, "beta_bits outside 1..7");
  if (ldc < p) return set_err(h, OZMM_ERR_ARG, "ldc < p");
  if (lds_a % 16 || lds_b % 16 || lds_a < n || lds_b < n)
    return set_err(h, OZMM_ERR_ARG, "slice strides must be multiples of 16 and >= n");
  if (plane_a < m * lds_a || plane_b < p * lds_b || plane_a % 16 || plane_b % 16)
    return set_err(h, OZMM_ERR_ARG, "slice plane strides must be multiples of 16 and cover the plane");
  if (r == 0) r = ozb::compute_r_host(n, beta_bits);
  if (r < 1) return set_err(h, OZMM_ERR_CONFIG, "force_r must be >= 1");
  CUDA_TRY(h, cudaSetDevice(h->device));
  const bool write_only = opt && opt->c_write_only;
  // fl(alpha*d) + fl(beta*c) == fl(alpha*d) bit for bit needs beta == 0 AND alpha
  // > 0: with alpha <= 0, alpha*d may be -0 and the sign of the zero would come
  // from fl(beta*c) (-0 + +0 = +0)
  if (write_only && !(beta == 0.0 && alpha > 0.0))
    return set_err(h, OZMM_ERR_ARG, "c_write_only needs beta == 0 and alpha > 0");
  return launch_gemm(h, m, n, p, k, beta_bits, r, As, lds_a, plane_a, mu, Bs, lds_b, plane_b, nu,
                     alpha, beta, write_only ? nullptr : C, C, ldc, opt, fl);
}
// the pipelined host entry behind ozmm_dgemm_host / ozmm_dgemm_host_out
int dgemm_host_impl(Handle* h, char transa, char transb, int64_t m, int64_t n, int64_t p, double alpha,
                    const double* A, int64_t lda, const double* B, int64_t ldb, double beta,
                    const double* C, int64_t ldc, double* Cout, int64_t ldo, int k,
                    const ozmm_options_t* opt, ozmm_counts_t* counts, ozmm_timings_t* timings);
}  // namespace

extern "C" {

int ozmm_dgemm_ex(ozmm_handle_t handle, char transa, char transb, int64_t m, int64_t n, int64_t p,
                  double alpha, const double* A, int64_t lda, const double* B, int64_t ldb,
                  double beta, double* C, int64_t ldc, int k, const ozmm_options_t* opt,
                  ozmm_counts_t* counts, ozmm_timings_t* timings) {
  Handle* h = reinterpret_cast<Handle*>(handle);
  if (!h) return set_err(nullptr, OZMM_ERR_ARG, "null handle");
  if (!valid_trans(transa) || !valid_trans(transb))
    return set_err(h, OZMM_ERR_ARG, "trans must be 'N' or 'T'");
  // validate_config (scheme.cpp:161-174) then the split argument checks (split.cpp:33-37)
  if (k < 1) return set_err(h, OZMM_ERR_CONFIG, "k must be >= 1");
  if (k > ozb::kMaxK) return set_err(h, OZMM_ERR_UNSUPPORTED, "k > %d not supported on the GPU path", ozb::kMaxK);
  if (m < 1 || n < 1 || p < 1) return set_err(h, OZMM_ERR_ARG, "split: empty matrix");
  if (m > INT32_MAX || p > INT32_MAX) return set_err(h, OZMM_ERR_ARG, "m, p must fit int32");
  if (opt && (opt->col_split < 0 || opt->col_split > 2)) return set_err(h, OZMM_ERR_ARG, "options: col_split must be 0..2");
  // device entry: the two-pass column split unless asked (it is on the critical path)
  ColSplitScope col_scope(h, opt && opt->col_split == 2);
  const int fb = opt ? opt->force_beta : 0;
  int beta_bits;
  if (fb) {
    if (fb < 1 || fb > 7) return set_err(h, OZMM_ERR_ARG, "split: forced beta outside 1..7");
    beta_bits = fb;
  } else {
    beta_bits = ozb::compute_beta_host(n);
    if (beta_bits < 0) return set_err(h, OZMM_ERR_ARG, "compute_beta: n > 2^29 unsupported");
  }
  const int64_t fr = opt ? opt->force_r : 0;
  if (fr < 0) return set_err(h, OZMM_ERR_CONFIG, "force_r must be >= 1");
  const int64_t r = fr ? fr : ozb::compute_r_host(n, beta_bits);
  MethodCfg mc;
  if (!method_cfg(opt ? opt->method : 0, &mc)) return set_err(h, OZMM_ERR_CONFIG, "unknown method");
  if (mc.simple && r < k)  // validate_config, scheme.cpp:169-173
    return set_err(h, OZMM_ERR_CONFIG, "simple group-wise accumulation requires r >= k");
  const int64_t lda_need = is_trans(transa) ? m : n, ldb_need = is_trans(transb) ? n : p;
  if (lda < lda_need || ldb < ldb_need || ldc < p)
    return set_err(h, OZMM_ERR_ARG, "leading dimension too small");
  // OverflowMode::Checked: only forced beta / r can make an INT32 overflow possible
  const int ovf = (opt && opt->overflow_wrap) || !(fb || fr)
                      ? 0 : overflow_possible(mc.strategy, mc.per_product, k, r, beta_bits, n);
  if (ovf < 0)
    return set_err(h, OZMM_ERR_UNSUPPORTED, "Checked overflow mode: a single slice product may leave "
                   "INT32 for this forced beta and n (its wrapped sum cannot be verified); use "
                   "overflow_wrap");
  if (ovf > 0 && mc.per_product)  // per-product chunks are single products: in range
    return set_err(h, OZMM_ERR_INTERNAL, "overflow bound inconsistent");

  CUDA_TRY(h, cudaSetDevice(h->device));
  const int64_t lds = ozmm_slice_ld(n);
  if (int rc = ensure(h, &h->slices_a, &h->slices_a_bytes, static_cast<size_t>(k) * m * lds)) return rc;
  if (int rc = ensure(h, &h->slices_b, &h->slices_b_bytes, static_cast<size_t>(k) * p * lds)) return rc;
  if (int rc = ensure(h, &h->mu, &h->mu_n, static_cast<size_t>(m))) return rc;
  if (int rc = ensure(h, &h->nu, &h->nu_n, static_cast<size_t>(p))) return rc;
  // this call's flags start clear; earlier unreported ones stay pending
  fold_flags_kernel<<<1, 1, 0, h->stream>>>(h->flags);
  CUDA_TRY(h, cudaGetLastError());

  const bool want_t = (opt && opt->timings) || timings;
  if (want_t) CUDA_TRY(h, cudaEventRecord(h->ev[0], h->stream));
  FlushCfg fl;
  fl.per_product = mc.per_product;
  fl.scale_mode = !mc.per_product ? 0 : (mc.strategy == kRNPerSlice ? 2 : 1);
  double* out_a = h->mu;
  double* out_b = h->nu;
  if (mc.strategy == kRNPerSlice) {
    if (int rc = ensure(h, &h->units_a, &h->units_a_n, static_cast<size_t>(k) * m)) return rc;
    if (int rc = ensure(h, &h->units_b, &h->units_b_n, static_cast<size_t>(k) * p)) return rc;
    CUDA_TRY(h, cudaMemsetAsync(h->units_a, 0, sizeof(double) * k * m, h->stream));
    CUDA_TRY(h, cudaMemsetAsync(h->units_b, 0, sizeof(double) * k * p, h->stream));
    fl.units_a = out_a = h->units_a;
    fl.units_b = out_b = h->units_b;
  }
  const bool offset = use_offset_planes(opt, mc);
  if (offset) {
    if (int rc = ensure(h, &h->lsa, &h->lsa_n, static_cast<size_t>(k) * m)) return rc;
    if (int rc = ensure(h, &h->lsb, &h->lsb_n, static_cast<size_t>(k) * p)) return rc;
    CUDA_TRY(h, cudaMemsetAsync(h->lsa, 0, sizeof(int32_t) * k * m, h->stream));
    CUDA_TRY(h, cudaMemsetAsync(h->lsb, 0, sizeof(int32_t) * k * p, h->stream));
    fl.lsa = h->lsa;
    fl.lsb = h->lsb;
    fl.lsa_plane = m;
    fl.lsb_plane = p;
    fl.n = n;
  }
  // B's column maxima (an HBM-bound pass) run on a side stream beside A's row
  // split (issue-bound) when A is split by rows and B by columns
  // OZMM_SPLIT_OVERLAP: 2 (default) B's whole column split on the side stream,
  // 1 only its column maxima, 0 none (A/B switch)
  static const int split_overlap = [] {
    const char* e = OZMM_ENV("OZMM_SPLIT_OVERLAP");
    return e ? std::atoi(e) : 2;
  }();
  const bool overlap_colmax = offset && !is_trans(transa) && !is_trans(transb) && split_overlap > 0;
  const bool overlap_bsplit = overlap_colmax && split_overlap > 1;
  if (overlap_colmax) {
    if (!h->s_aux) CUDA_TRY(h, cudaStreamCreateWithFlags(&h->s_aux, cudaStreamNonBlocking));
    if (!h->ev_fork) CUDA_TRY(h, cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
    if (!h->ev_join) CUDA_TRY(h, cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
    cudaStream_t user = h->stream;
    CUDA_TRY(h, cudaEventRecord(h->ev_fork, user));
    CUDA_TRY(h, cudaStreamWaitEvent(h->s_aux, h->ev_fork, 0));
    h->stream = h->s_aux;
    // one-pass column split: no separate maxima pass
    const bool one_pass = overlap_bsplit && cols_onepass_units(h, n, B, ldb) != 0;
    int rc = one_pass ? OZMM_OK : launch_colmax(h, p, n, B, ldb);
    if (!rc && overlap_bsplit)  // split B (Right, columns) -- scheme.cpp:251
      rc = launch_split(h, false, p, n, B, ldb, k, beta_bits, h->slices_b, lds, p * lds, out_b,
                        h->lsb, p, 1, !one_pass);
    h->stream = user;
    if (rc) return rc;
    CUDA_TRY(h, cudaEventRecord(h->ev_join, h->s_aux));
  }
  // split A (Left, rows of op(A)) -- split.cpp:233 via scheme.cpp:248
  if (offset) {
    if (int rc = launch_split(h, !is_trans(transa), m, n, A, lda, k, beta_bits, h->slices_a, lds,
                              m * lds, out_a, h->lsa, m))
      return rc;
  } else if (int rc = launch_split_m(h, mc.strategy, !is_trans(transa), m, n, A, lda, k, beta_bits,
                                     h->slices_a, lds, m * lds, out_a)) {
    return rc;
  }
  if (want_t) CUDA_TRY(h, cudaEventRecord(h->ev[1], h->stream));
  // split B (Right, columns of op(B)) -- scheme.cpp:251
  if (offset) {
    if (overlap_colmax) CUDA_TRY(h, cudaStreamWaitEvent(h->stream, h->ev_join, 0));
    if (!overlap_bsplit)
      if (int rc = launch_split(h, is_trans(transb), p, n, B, ldb, k, beta_bits, h->slices_b,
                                lds, p * lds, out_b, h->lsb, p, 1, overlap_colmax))
        return rc;
  } else if (int rc = launch_split_m(h, mc.strategy, is_trans(transb), p, n, B, ldb, k, beta_bits,
                                     h->slices_b, lds, p * lds, out_b)) {
    return rc;
  }
  if (want_t) CUDA_TRY(h, cudaEventRecord(h->ev[2], h->stream));
  if (opt && opt->sync_check)
    if (int rc = check_range_sync(h)) return rc;
  if (ovf > 0)
    if (int rc = verify_no_overflow(h, m, n, p, k, beta_bits, r, h->slices_a, lds, h->mu,
                                    h->slices_b, h->nu, opt, fl))
      return rc;
  // fused group-wise accumulation + epilogue -- scheme.cpp:261-263, :286-287
  if (int rc = launch_gemm(h, m, n, p, k, beta_bits, r, h->slices_a, lds, m * lds, h->mu,
                           h->slices_b, lds, p * lds,
                           h->nu, alpha, beta, C, C, ldc, opt, fl))
    return rc;
  if (want_t) CUDA_TRY(h, cudaEventRecord(h->ev[3], h->stream));
  if (counts) {
    counts->int8_gemms = static_cast<int64_t>(k) * (k + 1) / 2;
    counts->r = r;
    counts->w = ozb::flush_count_w_host(k, r);
    counts->fp64_flushes =
        mc.per_product ? counts->int8_gemms : static_cast<int64_t>(ozb::make_chunks(k, r).size());
  }
  if (timings) {
    CUDA_TRY(h, cudaEventSynchronize(h->ev[3]));
    float t01, t12, t23;
    cudaEventElapsedTime(&t01, h->ev[0], h->ev[1]);
    cudaEventElapsedTime(&t12, h->ev[1], h->ev[2]);
    cudaEventElapsedTime(&t23, h->ev[2], h->ev[3]);
    timings->split_a = t01 * 1e-3;
    timings->split_b = t12 * 1e-3;
    timings->int_gemm = t23 * 1e-3;
    timings->accum_fp64 = 0.0;
    timings->copy = 0.0;
  }
  return OZMM_OK;
}

int ozmm_dgemm(ozmm_handle_t h, char transa, char transb, int64_t m, int64_t n, int64_t p,
               double alpha, const double* A, int64_t lda, const double* B, int64_t ldb,
               double beta, double* C, int64_t ldc, int k) {
  return ozmm_dgemm_ex(h, transa, transb, m, n, p, alpha, A, lda, B, ldb, beta, C, ldc, k, nullptr,
                       nullptr, nullptr);
}

// Host entry for the comparison methods: copy in, ozmm_dgemm_ex, copy out
// (only ozIMMU_H, the hot path, gets the pipelined host entry below).
int dgemm_host_simple(Handle* h, char transa, char transb, int64_t m, int64_t n, int64_t p,
                      double alpha, const double* A, int64_t lda, const double* B, int64_t ldb,
                      double beta, const double* C, int64_t ldc, double* Cout, int64_t ldo, int k,
                      const ozmm_options_t* opt, ozmm_counts_t* counts, ozmm_timings_t* timings) {
  const bool ta = is_trans(transa), tb = is_trans(transb);
  const int64_t arows = ta ? n : m, brows = tb ? p : n, acols = ta ? m : n, bcols = tb ? n : p;
  if (lda < acols || ldb < bcols || ldc < p || ldo < p)
    return set_err(h, OZMM_ERR_ARG, "leading dimension too small");
  CUDA_TRY(h, cudaSetDevice(h->device));
  if (int rc = ensure(h, &h->host_a, &h->host_a_n, static_cast<size_t>(arows) * acols)) return rc;
  if (int rc = ensure(h, &h->host_b, &h->host_b_n, static_cast<size_t>(brows) * bcols)) return rc;
  if (int rc = ensure(h, &h->host_c, &h->host_c_n, static_cast<size_t>(m) * p)) return rc;
  const size_t D = sizeof(double);
  CUDA_TRY(h, cudaMemcpy2DAsync(h->host_a, D * acols, A, D * lda, D * acols, arows,
                                cudaMemcpyHostToDevice, h->stream));
  CUDA_TRY(h, cudaMemcpy2DAsync(h->host_b, D * bcols, B, D * ldb, D * bcols, brows,
                                cudaMemcpyHostToDevice, h->stream));
  CUDA_TRY(h, cudaMemcpy2DAsync(h->host_c, D * p, C, D * ldc, D * p, m, cudaMemcpyHostToDevice,
                                h->stream));
  ozmm_options_t o = opt ? *opt : ozmm_options_t{};
  o.sync_check = 1;
  if (int rc = ozmm_dgemm_ex(reinterpret_cast<ozmm_handle_t>(h), transa, transb, m, n, p, alpha,
                             h->host_a, acols, h->host_b, bcols, beta, h->host_c, p, k, &o,
                             counts, timings))
    return rc;
  CUDA_TRY(h, cudaMemcpy2DAsync(Cout, D * ldo, h->host_c, D * p, D * p, m, cudaMemcpyDeviceToHost,
                                h->stream));
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  return OZMM_OK;
}

int ozmm_dgemm_host(ozmm_handle_t handle, char transa, char transb, int64_t m, int64_t n,
                    int64_t p, double alpha, const double* A, int64_t lda, const double* B,
                    int64_t ldb, double beta, double* C, int64_t ldc, int k,
                    const ozmm_options_t* opt, ozmm_counts_t* counts, ozmm_timings_t* timings) {
  Handle* h = reinterpret_cast<Handle*>(handle);
  if (!h) return set_err(nullptr, OZMM_ERR_ARG, "null handle");
  return dgemm_host_impl(h, transa, transb, m, n, p, alpha, A, lda, B, ldb, beta, C, ldc, C, ldc, k, opt,
                         counts, timings);
}

int ozmm_dgemm_host_out(ozmm_handle_t handle, char transa, char transb, int64_t m, int64_t n,
                        int64_t p, double alpha, const double* A, int64_t lda, const double* B,
                        int64_t ldb, double beta, const double* C, int64_t ldc, double* D,
                        int64_t ldd, int k, const ozmm_options_t* opt, ozmm_counts_t* counts,
                        ozmm_timings_t* timings) {
  // The reference's ozaki_gemm_ex leaves C alone and returns a new matrix
  // (scheme.cpp:281, :289): with a separate destination no copy of C is needed.
  Handle* h = reinterpret_cast<Handle*>(handle);
  if (!h) return set_err(nullptr, OZMM_ERR_ARG, "null handle");
  if (!C || !D) return set_err(h, OZMM_ERR_ARG, "null pointer");
  if (D != C) {
    // the destination may not overlap C (or A / B): the result is written while C is still read
    const char* c0 = reinterpret_cast<const char*>(C);
    const char* c1 = reinterpret_cast<const char*>(C + (m - 1) * ldc + p);
    const char* d0 = reinterpret_cast<const char*>(D);
    const char* d1 = reinterpret_cast<const char*>(D + (m - 1) * ldd + p);
    if (m >= 1 && p >= 1 && d0 < c1 && c0 < d1) return set_err(h, OZMM_ERR_ARG, "D overlaps C (pass D == C for in place)");
  }
  return dgemm_host_impl(h, transa, transb, m, n, p, alpha, A, lda, B, ldb, beta, C, ldc, D, ldd, k, opt,
                         counts, timings);
}

}  // extern "C"

namespace {
int dgemm_host_impl(Handle* h, char transa, char transb, int64_t m, int64_t n, int64_t p, double alpha,
                    const double* A, int64_t lda, const double* B, int64_t ldb, double beta,
                    const double* C, int64_t ldc, double* Cout, int64_t ldo, int k,
                    const ozmm_options_t* opt, ozmm_counts_t* counts, ozmm_timings_t* timings) {

  // Pipelined host entry (the reference's calling convention: host matrices in,
  // C overwritten).  op(A) is cut into row panels A_s and op(B) into column
  // panels B_s (about 16 of each), sent over PCIe in the order A_0 B_0 A_1 B_1
  // ... .  When A_s lands, the row strip (A_s x B_0..B_{s-1}) of C becomes
  // computable; when B_s lands, the column strip (A_0..A_s x B_s).  Each strip
  // is one fused-GEMM launch (two GEMM streams, so a small strip's tail overlaps
  // the next one), the panel splits run on a high-priority stream, and finished
  // strips go back on the D2H stream.  The GEMM therefore starts after 2/16 of
  // an operand has crossed PCIe instead of after all of B.
  //
  // C input.  fl(beta*c) is always formed (scheme.cpp:287).  For beta = +-0 and
  // alpha > 0 it cannot change a finite entry: D is never -0 (it starts at +0 and
  // only exact cancellation gives zero, which rounds to +0), so fl(alpha*d) is
  // never -0 and fl(alpha*d) + (+-0) = fl(alpha*d).  In that mode C is NOT
  // copied to the device: host threads scan it for non-finite entries while the
  // GPU works, and those entries are recomputed on the host afterwards as
  // fl(fl(alpha*d) + fl(beta*c)) -- the reference's own expression.  Otherwise
  // C strips are copied in just ahead of their GEMM.
  //
  // Errors.  A range error (row max >= 2^921, split.cpp:124-125) is only known
  // once every panel is split; the reference throws without touching C.  With C
  // on the device the original is copied back on error; in the no-C mode the
  // D2H copies are not issued until the last split has run and the flags are
  // clear, so C is never written on error.
  //
  // Output.  The result goes to Cout (ldo): C itself for ozmm_dgemm_host, a
  // separate matrix for ozmm_dgemm_host_out, which then never writes C.
  if (!valid_trans(transa) || !valid_trans(transb))
    return set_err(h, OZMM_ERR_ARG, "trans must be 'N' or 'T'");
  if (k < 1) return set_err(h, OZMM_ERR_CONFIG, "k must be >= 1");
  if (k > ozb::kMaxK) return set_err(h, OZMM_ERR_UNSUPPORTED, "k > %d not supported on the GPU path", ozb::kMaxK);
  if (m < 1 || n < 1 || p < 1) return set_err(h, OZMM_ERR_ARG, "split: empty matrix");
  if (m > INT32_MAX || p > INT32_MAX) return set_err(h, OZMM_ERR_ARG, "m, p must fit int32");
  // comparison methods, and calls that need the Checked-overflow verification
  // (forced beta / r), take the plain copy-in / ozmm_dgemm_ex / copy-out route
  if ((opt && opt->method != OZMM_METHOD_OZIMMU_H) ||
      (opt && !opt->overflow_wrap && (opt->force_beta || opt->force_r)))
    return dgemm_host_simple(h, transa, transb, m, n, p, alpha, A, lda, B, ldb, beta, C, ldc, Cout, ldo, k,
                             opt, counts, timings);
  const bool ta = is_trans(transa), tb = is_trans(transb);
  const int64_t acols = ta ? m : n, bcols = tb ? n : p;
  if (lda < acols || ldb < bcols || ldc < p || ldo < p)
    return set_err(h, OZMM_ERR_ARG, "leading dimension too small");
  if (opt && (opt->col_split < 0 || opt->col_split > 2)) return set_err(h, OZMM_ERR_ARG, "options: col_split must be 0..2");
  // host entry: the one-pass column split by default -- the panel splits run under the
  // PCIe transfers, so the kernel's extra time is hidden and B crosses HBM once
  ColSplitScope col_scope(h, !(opt && opt->col_split == 1));
  const int fb = opt ? opt->force_beta : 0;
  int beta_bits;
  if (fb) {
    if (fb < 1 || fb > 7) return set_err(h, OZMM_ERR_ARG, "split: forced beta outside 1..7");
    beta_bits = fb;
  } else {
    beta_bits = ozb::compute_beta_host(n);
    if (beta_bits < 0) return set_err(h, OZMM_ERR_ARG, "compute_beta: n > 2^29 unsupported");
  }
  const int64_t fr = opt ? opt->force_r : 0;
  if (fr < 0) return set_err(h, OZMM_ERR_CONFIG, "force_r must be >= 1");
  const int64_t r = fr ? fr : ozb::compute_r_host(n, beta_bits);
  const bool no_c = beta == 0.0 && alpha > 0.0 && !(opt && opt->chunk_dump);

  // panels: ~16 per operand, A panels in whole CTA-pair tile rows (256), B panels
  // in whole tile columns (128)
  int64_t npanels = 16;
  if (opt && opt->host_panels < 0) return set_err(h, OZMM_ERR_ARG, "options: host_panels must be >= 0");
  if (opt && opt->host_panels) npanels = opt->host_panels;
  if (const char* e = OZMM_ENV("OZMM_HOST_PANELS")) npanels = std::max(1, std::atoi(e));
  auto round_up = [](int64_t x, int64_t q) { return (x + q - 1) / q * q; };
  int64_t pa = round_up((m + npanels - 1) / npanels, 256), pb = round_up((p + npanels - 1) / npanels, 128);
  if (pa >= m) pa = m;
  if (pb >= p) pb = p;
  const int ra = static_cast<int>((m + pa - 1) / pa), rb = static_cast<int>((p + pb - 1) / pb);
  const int steps = std::max(ra, rb);

  CUDA_TRY(h, cudaSetDevice(h->device));
  const int64_t lds = ozmm_slice_ld(n);
  if (int rc = ensure(h, &h->host_a, &h->host_a_n, static_cast<size_t>(m) * n)) return rc;
  if (int rc = ensure(h, &h->host_b, &h->host_b_n, static_cast<size_t>(n) * p)) return rc;
  if (!no_c)
    if (int rc = ensure(h, &h->host_c, &h->host_c_n, static_cast<size_t>(m) * p)) return rc;
  if (int rc = ensure(h, &h->host_o, &h->host_o_n, static_cast<size_t>(m) * p)) return rc;
  if (int rc = ensure(h, &h->slices_a, &h->slices_a_bytes, static_cast<size_t>(k) * m * lds)) return rc;
  if (int rc = ensure(h, &h->slices_b, &h->slices_b_bytes, static_cast<size_t>(k) * p * lds)) return rc;
  if (int rc = ensure(h, &h->mu, &h->mu_n, static_cast<size_t>(m))) return rc;
  if (int rc = ensure(h, &h->nu, &h->nu_n, static_cast<size_t>(p))) return rc;
  // column-line splits reuse h->colmax: size it once so no launch reallocates it
  if (int rc = ensure(h, &h->colmax, &h->colmax_n, static_cast<size_t>(std::max(pa, pb)))) return rc;
  if (!h->s_in) CUDA_TRY(h, cudaStreamCreateWithFlags(&h->s_in, cudaStreamNonBlocking));
  if (!h->s_out) CUDA_TRY(h, cudaStreamCreateWithFlags(&h->s_out, cudaStreamNonBlocking));
  if (!h->s_split) {
    int lo = 0, hi = 0;
    CUDA_TRY(h, cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CUDA_TRY(h, cudaStreamCreateWithPriority(&h->s_split, cudaStreamNonBlocking, hi));
  }
  for (auto& sg : h->s_gemm)
    if (!sg) CUDA_TRY(h, cudaStreamCreateWithFlags(&sg, cudaStreamNonBlocking));
  if (!h->hflags) CUDA_TRY(h, cudaMallocHost(reinterpret_cast<void**>(&h->hflags), 2 * sizeof(int)));
  double *dA = h->host_a, *dB = h->host_b, *dC = h->host_c, *dO = h->host_o;
  const size_t D = sizeof(double);
  // Pageable caller buffers (numpy, Eigen, std::vector) cross PCIe through rings
  // of pinned slots filled by a team of host threads (host_stage.hpp); pinned
  // ones are copied directly by the DMA engines.
  const int hs_mode = opt ? opt->host_staging : 0;
  if (hs_mode < 0 || hs_mode > 2 || (opt && opt->host_threads < 0))
    return set_err(h, OZMM_ERR_ARG, "options: host_staging must be 0..2 and host_threads >= 0");
  auto staged = [&](const void* ptr) { return hs_mode == 2 || (hs_mode == 0 && ozb::host_pageable(ptr)); };
  // pg_c: the result's destination; pg_ci: C when it is uploaded (beta != 0)
  const bool pg_a = staged(A), pg_b = staged(B), pg_c = staged(Cout), pg_ci = Cout == C ? pg_c : staged(C);
  if (pg_a || pg_b || pg_c || pg_ci) {
    // default team: every hardware thread, at most 16 (16-core box, C3 call: 8 threads
    // 157-162 ms, 12 155-159 ms, 16 147-150 ms; profiles/r2/stage_sweep3.txt)
    int nt = opt && opt->host_threads
                 ? opt->host_threads
                 : static_cast<int>(std::min(16u, std::max(1u, std::thread::hardware_concurrency())));
    if (const char* e = OZMM_ENV("OZMM_STAGE_THREADS")) nt = std::max(1, std::atoi(e));
    if (!h->pool || h->pool->size() != nt) {
      h->stage_in.release();  // slots are per team thread
      h->stage_out.release();
      h->pool.reset(new ozb::WorkerPool(nt));
    }
    // four slots per team thread and direction: 2 MB for large operands (16 threads:
    // 256 MB pinned in all), smaller for small ones (a power of two >= 256 KB, about a
    // quarter of a thread's share of the largest staged matrix); grown when a later
    // call is larger.  C3 pageable call, 16 threads: 2 MB x 4 146-148 ms, 4 MB x 2
    // 143-157, 8 MB x 2 153-170, 1 MB x 8 151-152 (profiles/r2/stage_sweep4.txt)
    const size_t big = D * static_cast<size_t>(std::max({pg_a ? m * n : 0, pg_b ? n * p : 0, pg_c || pg_ci ? m * p : 0}));
    size_t slot = size_t(256) << 10;
    while (slot < (size_t(2) << 20) && slot * 4 * nt < big) slot <<= 1;
    int nslots = 4;
    if (const char* e = OZMM_ENV("OZMM_STAGE_SLOT_MB")) slot = size_t(std::max(1, std::atoi(e))) << 20;
    if (const char* e = OZMM_ENV("OZMM_STAGE_SLOTS")) nslots = std::max(2, std::atoi(e));
    for (ozb::HostStager* st : {&h->stage_in, &h->stage_out}) {
      if (st->ready() && st->slot_bytes() < slot) st->release();
      CUDA_TRY(h, st->init(slot, nslots, h->pool.get()));
    }
  }

  // Panel arrival order over PCIe: A_s then B_s per step, except that the last
  // step sends B first, so the final strip is a row strip -- full-width host
  // rows, whose D2H is the tail of the call (a narrow column strip's D2H runs
  // at ~31 GB/s while the GEMM is busy, full rows at ~52+).
  struct Arrival {
    bool is_a;
    int idx;
  };
  std::vector<Arrival> order;
  for (int s = 0; s < steps; ++s) {
    if (s == steps - 1 && s < ra && s < rb) {
      order.push_back({false, s});
      order.push_back({true, s});
      continue;
    }
    if (s < ra) order.push_back({true, s});
    if (s < rb) order.push_back({false, s});
  }
  // strips in issue order: each arrival makes one block of C computable, A_s x
  // (the B panels so far) or (the A panels so far) x B_s; it waits on the split
  // of that arrival (the split stream is in order, so that covers every panel)
  struct Strip {
    int64_t r0, rows, c0, cols;
    bool trig_a;
    int trig;
  };
  std::vector<Strip> strips;
  std::vector<int> strip_of(order.size(), -1);
  {
    int64_t na_arr = 0, nb_arr = 0;
    for (size_t o = 0; o < order.size(); ++o) {
      const int i = order[o].idx;
      if (order[o].is_a) {
        if (nb_arr > 0) {
          strip_of[o] = static_cast<int>(strips.size());
          strips.push_back({i * pa, std::min(pa, m - i * pa), 0, std::min<int64_t>(p, nb_arr * pb), true, i});
        }
        ++na_arr;
      } else {
        if (na_arr > 0) {
          strip_of[o] = static_cast<int>(strips.size());
          strips.push_back({0, std::min<int64_t>(m, na_arr * pa), i * pb, std::min(pb, p - i * pb), false, i});
        }
        ++nb_arr;
      }
    }
  }
  const int ns = static_cast<int>(strips.size());
  // events: A/B copied [ra + rb], A/B split [ra + rb], C strip copied [ns], GEMM done [ns], start, splits done
  std::vector<cudaEvent_t> ev(2 * (ra + rb) + 2 * ns + 2);
  // OZMM_TRACE=1: timed events and a per-panel / per-strip timeline on stderr
  const bool trace = OZMM_ENV("OZMM_TRACE") != nullptr;
  const auto t_entry = std::chrono::steady_clock::now();
  for (auto& e : ev) CUDA_TRY(h, cudaEventCreateWithFlags(&e, trace ? 0 : cudaEventDisableTiming));
  std::vector<cudaEvent_t> evGs(trace ? ns : 0), evO(trace ? ns : 0);
  for (auto& e : evGs) CUDA_TRY(h, cudaEventCreate(&e));
  for (auto& e : evO) CUDA_TRY(h, cudaEventCreate(&e));
  cudaEvent_t* evA = ev.data();
  cudaEvent_t* evB = evA + ra;
  cudaEvent_t* evSA = evB + rb;
  cudaEvent_t* evSB = evSA + ra;
  cudaEvent_t* evC = evSB + rb;
  cudaEvent_t* evG = evC + ns;
  cudaEvent_t evStart = evG[ns], evSplit = evG[ns + 1];
  cudaStream_t user = h->stream;
  int rc = OZMM_OK;
  auto cu = [&](cudaError_t e, const char* what) {
    if (e != cudaSuccess && rc == OZMM_OK)
      rc = set_err(h, OZMM_ERR_CUDA, "%s failed: %s", what, cudaGetErrorString(e));
    return e == cudaSuccess;
  };
  // 2-D copies between the caller's buffers and the device: direct for pinned
  // memory, through the slot rings for pageable memory (the staged calls return
  // once the host side is done: they pace the issue loop below)
  // With A and B both staged (no_c mode), the staging copy also screens every
  // element for the range error (host_stage.hpp copy_screen), so no scanner has
  // to re-read them; with C staged too, the old C entries are checked for inf /
  // NaN as the result overwrites them (copy_patch) instead of by a separate scan.
  // staged C of a beta = 0 call: the non-finite-C patch rides on the copy-out (C
  // scanned up front by scanner threads instead: 150-160 vs 146-151 ms at C3,
  // profiles/r2/cscan_rejected.txt)
  const bool patch_c = no_c && pg_c;
  const bool screen_ab = no_c && pg_a && pg_b;
  std::atomic<uint64_t> big_ab{0};
  auto h2d = [&](bool pg, void* dst, size_t dp, const void* src, size_t sp, size_t w, size_t rows,
                 const char* what, bool screen = false) {
    return cu(pg ? h->stage_in.h2d(dst, dp, src, sp, w, rows, h->s_in, screen ? &big_ab : nullptr)
                 : cudaMemcpy2DAsync(dst, dp, src, sp, w, rows, cudaMemcpyHostToDevice, h->s_in), what);
  };
  // cin / cp: the caller's C at the same block (read by the fused non-finite-C patch)
  auto d2h = [&](void* dst, size_t dp, const void* src, size_t sp, size_t w, size_t rows, const void* cin,
                 size_t cp, const char* what) {
    return cu(pg_c ? h->stage_out.d2h(dst, dp, src, sp, w, rows, h->s_out, patch_c ? &beta : nullptr, cin, cp)
                   : cudaMemcpy2DAsync(dst, dp, src, sp, w, rows, cudaMemcpyDeviceToHost, h->s_out), what);
  };

  // Host scans (no-C mode), concurrent with the GPU:
  //  1. C for non-finite entries (patched on the host afterwards, see below);
  //  2. then the A and B panels of the LAST steps, backwards, for any element
  //     with |x| >= 2^921 (exponent field >= 1944, incl. inf / NaN).  A line
  //     max >= 2^921 is the only range error (split.cpp:124-125), so a clean
  //     scan of a panel proves its split cannot raise the range flag.  The D2H
  //     gate then opens as soon as the GPU has split every earlier step with
  //     clean flags -- the GPU-split prefix meets the host-scanned suffix at
  //     ~55 ms at C3 instead of the last split at ~81 ms.
  std::vector<std::thread> scanners;
  std::vector<std::vector<std::pair<int64_t, double>>> bad;  // (index, original c)
  std::atomic<int> c_scans_left{0}, next_tail{steps - 1}, tail_hit{0}, stop_tail{0};
  std::unique_ptr<std::atomic<int>[]> tail_done(new std::atomic<int>[steps]);
  for (int s0 = 0; s0 < steps; ++s0) tail_done[s0] = 0;
  auto any_big = [](const double* x, int64_t rows, int64_t cols, int64_t ld) {
    constexpr uint64_t kExp = 0x7FF0000000000000ull, kBias = uint64_t(2048 - 1944) << 52;
    uint64_t any = 0;
    for (int64_t i = 0; i < rows; ++i) {
      const uint64_t* row = reinterpret_cast<const uint64_t*>(x + i * ld);
      for (int64_t j = 0; j < cols; ++j) any |= (row[j] & kExp) + kBias;  // bit 63: exp >= 1944
    }
    return (any >> 63) != 0;
  };
  auto scan_step = [&](int st) {  // A panel st and B panel st of op(A) / op(B)
    bool big = false;
    if (st < ra) {
      const int64_t r0 = st * pa, rows = std::min(pa, m - r0);
      big = ta ? any_big(A + r0, n, rows, lda) : any_big(A + r0 * lda, rows, n, lda);
    }
    if (!big && st < rb) {
      const int64_t c0 = st * pb, cols = std::min(pb, p - c0);
      big = tb ? any_big(B + c0 * ldb, cols, n, ldb) : any_big(B + c0, n, cols, ldb);
    }
    return big;
  };
  if (no_c && (!patch_c || !screen_ab)) {
    int64_t want = 8;
    if (const char* e = OZMM_ENV("OZMM_SCAN_THREADS")) want = std::max(1, std::atoi(e));
    const int nt = static_cast<int>(std::max<int64_t>(
        1, std::min<int64_t>({want, static_cast<int64_t>(std::thread::hardware_concurrency()), (m * p) >> 20})));
    bad.resize(nt);
    c_scans_left = patch_c ? 0 : nt;
    for (int t = 0; t < nt; ++t)
      scanners.emplace_back([&, t, nt] {
        const int64_t i0 = patch_c ? 0 : m * t / nt, i1 = patch_c ? 0 : m * (t + 1) / nt;
        constexpr uint64_t kExp = 0x7FF0000000000000ull, kOne = 0x0010000000000000ull;
        for (int64_t i = i0; i < i1; ++i) {
          const uint64_t* row = reinterpret_cast<const uint64_t*>(C + i * ldc);
          // (x & kExp) + kOne carries into bit 63 exactly when the exponent field is
          // all ones (inf / NaN): and + add + or per element, which vectorises
          uint64_t any = 0;
          for (int64_t j = 0; j < p; ++j) any |= (row[j] & kExp) + kOne;
          if (any >> 63)
            for (int64_t j = 0; j < p; ++j)
              if ((row[j] & 0x7FF0000000000000ull) == 0x7FF0000000000000ull)
                bad[t].push_back({i * ldo + j, C[i * ldc + j]});  // (index into Cout, old c)
        }
        if (!patch_c) --c_scans_left;
        if (screen_ab) return;  // the staging copies screen A and B
        // tail scan: claim steps from the last one backwards until the gate opens
        while (!stop_tail.load() && !tail_hit.load()) {
          const int st = next_tail.fetch_sub(1);
          if (st < 0) break;
          if (scan_step(st)) tail_hit = 1;
          tail_done[st] = 1;
        }
      });
  }

  // offset-binary slice planes (the fused pair kernel's operand format)
  MethodCfg mch;
  method_cfg(OZMM_METHOD_OZIMMU_H, &mch);
  const bool offset = use_offset_planes(opt, mch);
  FlushCfg fl;
  if (offset && rc == OZMM_OK) {
    if ((rc = ensure(h, &h->lsa, &h->lsa_n, static_cast<size_t>(k) * m)) == OZMM_OK &&
        (rc = ensure(h, &h->lsb, &h->lsb_n, static_cast<size_t>(k) * p)) == OZMM_OK) {
      cu(cudaMemsetAsync(h->lsa, 0, sizeof(int32_t) * k * m, user), "memset");
      cu(cudaMemsetAsync(h->lsb, 0, sizeof(int32_t) * k * p, user), "memset");
    }
    fl.lsa_plane = m;
    fl.lsb_plane = p;
    fl.n = n;
  }
  // this call's flags start clear (earlier unreported ones stay pending); every
  // stream starts after earlier work on the handle's stream
  fold_flags_kernel<<<1, 1, 0, user>>>(h->flags);
  cu(cudaGetLastError(), "fold flags");
  cu(cudaEventRecord(evStart, user), "event");
  for (cudaStream_t s : {h->s_in, h->s_out, h->s_split, h->s_gemm[0], h->s_gemm[1]})
    cu(cudaStreamWaitEvent(s, evStart, 0), "wait");

  // One issue loop over the panel arrivals: the panel's H2D copy (each followed by
  // the C block its strip reads), its split on the high-priority split stream,
  // then the strip of C it completes on one of the two GEMM streams (the split
  // stream is in order, so the strip's split event covers every panel it reads).
  // Staged copies block here while the host team fills the slots; everything
  // else is asynchronous.
  auto copy_c = [&](int q) {
    const Strip& t = strips[q];
    h2d(pg_ci, dC + t.r0 * p + t.c0, D * p, C + t.r0 * ldc + t.c0, D * ldc, D * t.cols, t.rows, "H2D C");
    cu(cudaEventRecord(evC[q], h->s_in), "event");
  };
  for (size_t o = 0; o < order.size() && rc == OZMM_OK; ++o) {
    const int s0 = order[o].idx;
    if (order[o].is_a) {
      const int64_t r0 = s0 * pa, rows = std::min(pa, m - r0);
      if (ta)  // op(A) rows r0.. = columns r0.. of the stored n x m A
        h2d(pg_a, dA + r0, D * m, A + r0, D * lda, D * rows, n, "H2D A", screen_ab);
      else
        h2d(pg_a, dA + r0 * n, D * n, A + r0 * lda, D * lda, D * n, rows, "H2D A", screen_ab);
      cu(cudaEventRecord(evA[s0], h->s_in), "event");
    } else {
      const int64_t c0 = s0 * pb, cols = std::min(pb, p - c0);
      if (tb)  // op(B) columns c0.. = rows c0.. of the stored p x n B
        h2d(pg_b, dB + c0 * n, D * n, B + c0 * ldb, D * ldb, D * n, cols, "H2D B", screen_ab);
      else
        h2d(pg_b, dB + c0, D * p, B + c0, D * ldb, D * cols, n, "H2D B", screen_ab);
      cu(cudaEventRecord(evB[s0], h->s_in), "event");
    }
    const int q = strip_of[o];
    if (!no_c && q >= 0) copy_c(q);
    // split (high-priority stream), as soon as the panel lands
    h->stream = h->s_split;
    if (order[o].is_a) {
      const int64_t r0 = s0 * pa, rows = std::min(pa, m - r0);
      cu(cudaStreamWaitEvent(h->s_split, evA[s0], 0), "wait");
      if (rc == OZMM_OK)
        rc = launch_split(h, !ta, rows, n, ta ? dA + r0 : dA + r0 * n, ta ? m : n, k, beta_bits,
                          h->slices_a + r0 * lds, lds, m * lds, h->mu + r0,
                          offset ? h->lsa + r0 : nullptr, m);
      cu(cudaEventRecord(evSA[s0], h->s_split), "event");
    } else {
      const int64_t c0 = s0 * pb, cols = std::min(pb, p - c0);
      cu(cudaStreamWaitEvent(h->s_split, evB[s0], 0), "wait");
      if (rc == OZMM_OK)
        rc = launch_split(h, tb, cols, n, tb ? dB + c0 * n : dB + c0, tb ? n : p, k, beta_bits,
                          h->slices_b + c0 * lds, lds, p * lds, h->nu + c0,
                          offset ? h->lsb + c0 : nullptr, p);
      cu(cudaEventRecord(evSB[s0], h->s_split), "event");
    }
    if (q < 0 || rc != OZMM_OK) continue;
    // the strip of C this arrival completes
    const Strip& t = strips[q];
    cudaStream_t sg = h->s_gemm[q & 1];
    cu(cudaStreamWaitEvent(sg, t.trig_a ? evSA[t.trig] : evSB[t.trig], 0), "wait");
    if (!no_c) cu(cudaStreamWaitEvent(sg, evC[q], 0), "wait");
    h->stream = sg;
    if (trace) cu(cudaEventRecord(evGs[q], sg), "event");
    if (offset) {
      fl.lsa = h->lsa + t.r0;
      fl.lsb = h->lsb + t.c0;
    }
    if (rc == OZMM_OK)
      rc = launch_gemm(h, t.rows, n, t.cols, k, beta_bits, r, h->slices_a + t.r0 * lds, lds, m * lds,
                       h->mu + t.r0, h->slices_b + t.c0 * lds, lds, p * lds, h->nu + t.c0, alpha, beta,
                       no_c ? nullptr : dC + t.r0 * p + t.c0, dO + t.r0 * p + t.c0, p, opt, fl);
    cu(cudaEventRecord(evG[q], sg), "event");
  }
  cu(cudaEventRecord(evSplit, h->s_split), "event");
  h->stream = user;
  auto copy_out = [&](int q) {
    const Strip& t = strips[q];
    cu(cudaStreamWaitEvent(h->s_out, evG[q], 0), "wait");
    d2h(Cout + t.r0 * ldo + t.c0, D * ldo, dO + t.r0 * p + t.c0, D * p, D * t.cols, t.rows,
        C + t.r0 * ldc + t.c0, D * ldc, "D2H C");
    if (trace) cu(cudaEventRecord(evO[q], h->s_out), "event");
  };
  bool range_err = false;
  if (!no_c) {
    for (int q = 0; q < ns && rc == OZMM_OK; ++q) copy_out(q);
  } else {
    // every c read before any D2H writes C
    while (c_scans_left.load() > 0) std::this_thread::sleep_for(std::chrono::microseconds(100));
    if (trace)
      std::fprintf(stderr, "[ozmm trace] host C scan done %.2f ms after entry\n",
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_entry)
                       .count());
    // gate: open when the GPU has split steps [0, s) and the host has scanned
    // steps [s, steps) clean; otherwise (a big element on the host side, or a
    // device error) after every split, as before
    bool early = false;
    // staged A and B: every panel has been screened on its way in (the issue loop
    // above returned), so a clean screen opens the gate at once
    if (screen_ab && rc == OZMM_OK) {
      early = (big_ab.load() >> 63) == 0;
      if (!early) tail_hit = 1;  // the device flags decide, after every split
    }
    for (; !screen_ab;) {
      if (tail_hit.load() || rc != OZMM_OK) break;
      int gd = 0;
      while (gd < steps && (gd >= ra || cudaEventQuery(evSA[gd]) == cudaSuccess) &&
             (gd >= rb || cudaEventQuery(evSB[gd]) == cudaSuccess))
        ++gd;
      int hs = steps;
      while (hs > 0 && tail_done[hs - 1].load()) --hs;
      if (gd == steps) break;  // every split already done: the plain gate below
      if (gd >= hs && !tail_hit.load()) {
        early = true;
        break;
      }
      std::this_thread::sleep_for(std::chrono::microseconds(200));
    }
    stop_tail = 1;
    if (!early) cu(cudaEventSynchronize(evSplit), "sync");
    // the flags of the splits that have run (all of them on the plain path)
    cu(cudaMemcpyAsync(h->hflags, h->flags, 2 * sizeof(int), cudaMemcpyDeviceToHost, h->s_out), "flags");
    cu(cudaStreamSynchronize(h->s_out), "sync");
    range_err = rc == OZMM_OK && h->hflags[1] != 0;
    if (trace)
      std::fprintf(stderr, "[ozmm trace] D2H gate open %.2f ms after entry (%s)\n",
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_entry)
                       .count(), early ? "early: host-scanned tail" : "after the last split");
    // The strips already finished by now form (typically) the square
    // [0, X) x [0, Y): it goes back as ONE copy with X-wide host rows -- host
    // writes in narrow 8 KB row pieces drop to ~31 GB/s while the GEMM runs,
    // full rows keep ~52-57 GB/s (tools/d2h_2d.py).  The rest goes per strip.
    int q0 = 0;
    if (rc == OZMM_OK && !range_err) {
      int qd = 0;
      while (qd < ns && cudaEventQuery(evG[qd]) == cudaSuccess) ++qd;
      for (; qd > 1; --qd) {
        int64_t R = 0, Cc = 0, area = 0;
        for (int q = 0; q < qd; ++q) {
          R = std::max(R, strips[q].r0 + strips[q].rows);
          Cc = std::max(Cc, strips[q].c0 + strips[q].cols);
          area += strips[q].rows * strips[q].cols;
        }
        if (area == R * Cc) {
          for (int q = 0; q < qd; ++q) cu(cudaStreamWaitEvent(h->s_out, evG[q], 0), "wait");
          d2h(Cout, D * ldo, dO, D * p, D * Cc, R, C, D * ldc, "D2H C");
          if (trace)
            for (int q = 0; q < qd; ++q) cu(cudaEventRecord(evO[q], h->s_out), "event");
          q0 = qd;
          break;
        }
      }
    }
    for (int q = q0; q < ns && rc == OZMM_OK && !range_err; ++q) copy_out(q);
  }
  for (auto& th : scanners)
    if (th.joinable()) th.join();
  for (cudaStream_t s : {h->s_in, h->s_split, h->s_gemm[0], h->s_gemm[1], h->s_out})
    cu(cudaStreamSynchronize(s), "sync");
  if (rc == OZMM_OK && no_c && !range_err) {
    // early gate: the host scan proved the later panels clean; confirm on the device
    int f[2] = {0, 0};
    cu(cudaMemcpy(f, h->flags, sizeof f, cudaMemcpyDeviceToHost), "flags");
    if (f[1]) {
      const int zero = 0;
      cu(cudaMemcpy(h->flags + 1, &zero, sizeof(int), cudaMemcpyHostToDevice), "flags");
      rc = set_err(h, OZMM_ERR_CUDA, "internal: range flag raised on a host-scanned panel");
    }
  }
  if (rc == OZMM_OK && !no_c) {
    int f[2] = {0, 0};
    cu(cudaMemcpy(f, h->flags, sizeof f, cudaMemcpyDeviceToHost), "flags");
    if (f[1]) {  // restore the caller's C (in place), then report like the reference's throw
      range_err = true;
      if (Cout == C) cu(cudaMemcpy2D(Cout, D * ldo, dC, D * p, D * p, m, cudaMemcpyDeviceToHost), "restore C");
    }
  }
  if (range_err) {
    const int zero = 0;
    cu(cudaMemcpy(h->flags + 1, &zero, sizeof(int), cudaMemcpyHostToDevice), "flags");
    if (rc == OZMM_OK) rc = set_err(h, OZMM_ERR_RANGE, "split: row magnitude too large for shift extraction");
  }
  if (rc == OZMM_OK && no_c) {
    // non-finite c: the reference's fl(fl(alpha*d) + fl(beta*c)) on the host
    // (the device wrote fl(alpha*d) there)
    for (const auto& v : bad)
      for (const auto& [idx, c] : v) {
        const double z = beta * c;
        Cout[idx] = Cout[idx] + z;
      }
  }
  if (trace && rc == OZMM_OK) {
    auto ms = [&](cudaEvent_t e) {
      float t = -1.f;
      cudaEventElapsedTime(&t, evStart, e);
      return t;
    };
    for (int s = 0; s < steps; ++s)
      std::fprintf(stderr, "[ozmm trace] step %2d  A copied %7.2f split %7.2f | B copied %7.2f split %7.2f\n",
                   s, s < ra ? ms(evA[s]) : -1.f, s < ra ? ms(evSA[s]) : -1.f,
                   s < rb ? ms(evB[s]) : -1.f, s < rb ? ms(evSB[s]) : -1.f);
    for (int q = 0; q < ns; ++q)
      std::fprintf(stderr, "[ozmm trace] strip %2d %s %6lld x %6lld  gemm %7.2f -> %7.2f  d2h done %7.2f\n", q,
                   strips[q].trig_a ? "row" : "col", static_cast<long long>(strips[q].rows),
                   static_cast<long long>(strips[q].cols), ms(evGs[q]), ms(evG[q]), ms(evO[q]));
  }
  for (auto& e : evGs) cudaEventDestroy(e);
  for (auto& e : evO) cudaEventDestroy(e);
  for (auto& e : ev) cudaEventDestroy(e);
  if (rc == OZMM_OK && counts) {
    counts->int8_gemms = static_cast<int64_t>(k) * (k + 1) / 2;
    counts->r = r;
    counts->w = ozb::flush_count_w_host(k, r);
    counts->fp64_flushes = static_cast<int64_t>(ozb::make_chunks(k, r).size());
  }
  if (rc == OZMM_OK && timings) *timings = ozmm_timings_t{};  // phases overlap: not separable
  return rc;
}

}  // namespace
