// ozmm_dgemm_2d: the 2-D grid partition of the emulated DGEMM as a native entry
// (SURVEY.md section 8b "multi-GPU" row, 8e).  One process (and one ozmm handle)
// per GPU; ranks form a Pr x Pc grid and rank (gr, gc) = (rank / Pc, rank % Pc)
// owns the C block (gr, gc).  Same partition and bit-identical results as the
// Python orchestration in paper_2409_13313_b200/grid2d.py (Grid2DGemm.step):
//   1. split the rank's m/(Pr*Pc) full rows of op(A) and p/(Pr*Pc) full columns
//      of op(B) straight into their slot of the row / column panel
//      (ozmm_split_offset_strided; row maxima are local, split.cpp:157-171);
//   2. all-gather the offset-binary slice planes, the shifts and the line sums:
//      A inside the row group (the Pc ranks of grid row gr), B inside the
//      column group (the Pr ranks of grid column gc).  In place, broadcast
//      only -- no reductions;
//   3. three strip launches of the fused GEMM on the C block: G1 own rows x
//      own columns on a side stream (no communication), G2 own rows x the
//      other columns after B's gather, G3 the other rows after A's gather.
//
// The all-gather is either NCCL (communicators from ncclCommInitRank +
// ncclCommSplit; libnccl is dlopen'ed on first use, so the library itself does
// not depend on it) or a caller-supplied hook (ozmm_allgather_fn), which is how
// the single-GPU tests emulate W ranks.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "../../include/ozmm_b200.h"

// library-internal helpers of ozmm_capi.cu (hidden; see there)
extern "C" int* ozmm_internal_range_flag(ozmm_handle_t h);
extern "C" int ozmm_internal_fold_flags(ozmm_handle_t h);

namespace {

// ---- NCCL, resolved at run time ------------------------------------------
struct Nccl {
  bool ok = false;
  std::string why;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_split)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    // torch's bundled libnccl is already loaded in a torch process: same soname
    void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) {
      n.why = std::string("dlopen libnccl.so.2: ") + dlerror();
      return;
    }
    auto sym = [&](const char* name) { return dlsym(lib, name); };
    n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(sym("ncclGetUniqueId"));
    n.comm_init_rank = reinterpret_cast<decltype(n.comm_init_rank)>(sym("ncclCommInitRank"));
    n.comm_split = reinterpret_cast<decltype(n.comm_split)>(sym("ncclCommSplit"));
    n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(sym("ncclCommDestroy"));
    n.all_gather = reinterpret_cast<decltype(n.all_gather)>(sym("ncclAllGather"));
    n.group_start = reinterpret_cast<decltype(n.group_start)>(sym("ncclGroupStart"));
    n.group_end = reinterpret_cast<decltype(n.group_end)>(sym("ncclGroupEnd"));
    n.error_string = reinterpret_cast<decltype(n.error_string)>(sym("ncclGetErrorString"));
    n.ok = n.get_unique_id && n.comm_init_rank && n.comm_split && n.comm_destroy &&
           n.all_gather && n.group_start && n.group_end && n.error_string;
    if (!n.ok) n.why = "libnccl.so.2 lacks ncclCommSplit (needs NCCL >= 2.18)";
  });
  return n;
}

thread_local std::string g_grid_err;

int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_grid_err = buf;
  return code;
}

#define GRID_CUDA(call)                                                               \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess) return fail(OZMM_ERR_CUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)

#define GRID_OZ(call)                                                                 \
  do {                                                                                \
    int rc_ = (call);                                                                 \
    if (rc_ != OZMM_OK) return fail(rc_, "%s: %s", #call, ozmm_last_error(g->h));     \
  } while (0)

}  // namespace

struct ozmm_grid {
  ozmm_handle_t h = nullptr;
  int device = 0, world = 1, rank = 0, pr = 1, pc = 1, gr = 0, gc = 0;
  // collective: hook or NCCL
  ozmm_allgather_fn hook = nullptr;
  void* hook_ctx = nullptr;
  ncclComm_t world_comm = nullptr, row_comm = nullptr, col_comm = nullptr;
  cudaStream_t s_side = nullptr, s_comm = nullptr;
  cudaEvent_t ev_split = nullptr, ev_b = nullptr, ev_a = nullptr, ev_side = nullptr;
  // panels (device): slices [k][lines][lds] int8, shifts [lines] f64, sums [lines][k] i32
  int8_t* a_pan = nullptr;
  int8_t* b_pan = nullptr;
  double* mu = nullptr;
  double* nu = nullptr;
  int32_t* lsa = nullptr;
  int32_t* lsb = nullptr;
  int* gflag = nullptr;  // [pr][pc] range flags of the grid (grid-wide max)
  size_t a_bytes = 0, b_bytes = 0, mu_n = 0, nu_n = 0, lsa_n = 0, lsb_n = 0, gflag_n = 0;
};

namespace {

template <class T>
int grow(T** p, size_t* have, size_t need) {
  if (*have >= need) return OZMM_OK;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *have = 0;
  GRID_CUDA(cudaMalloc(reinterpret_cast<void**>(p), need * sizeof(T)));
  *have = need;
  return OZMM_OK;
}

// all-gather `bytes` per member of `group` (0 row, 1 column) in place: this
// rank's part already sits at recv + index * bytes
int gather(ozmm_grid* g, int group, void* recv, int64_t bytes) {
  const int members = group == 0 ? g->pc : g->pr;
  if (members == 1) return OZMM_OK;
  const int index = group == 0 ? g->gc : g->gr;
  void* send = static_cast<int8_t*>(recv) + index * bytes;
  if (g->hook) {
    int rc = g->hook(g->hook_ctx, group, send, recv, bytes, g->s_comm);
    return rc == 0 ? OZMM_OK : fail(OZMM_ERR_NCCL, "all-gather hook returned %d", rc);
  }
  Nccl& n = nccl();
  ncclResult_t r = n.all_gather(send, recv, static_cast<size_t>(bytes), ncclInt8,
                                group == 0 ? g->row_comm : g->col_comm, g->s_comm);
  return r == ncclSuccess ? OZMM_OK : fail(OZMM_ERR_NCCL, "ncclAllGather: %s", n.error_string(r));
}

int gather_group(ozmm_grid* g, int group, const std::vector<std::pair<void*, int64_t>>& bufs) {
  const bool use_nccl = !g->hook && (group == 0 ? g->pc : g->pr) > 1;
  if (use_nccl) nccl().group_start();
  int rc = OZMM_OK;
  for (auto& b : bufs)
    if ((rc = gather(g, group, b.first, b.second))) break;
  if (use_nccl) {
    ncclResult_t r = nccl().group_end();
    if (rc == OZMM_OK && r != ncclSuccess)
      rc = fail(OZMM_ERR_NCCL, "ncclGroupEnd: %s", nccl().error_string(r));
  }
  return rc;
}

// [0, total) minus [own0, own0 + own)
std::vector<std::pair<int64_t, int64_t>> others(int64_t total, int64_t own0, int64_t own) {
  std::vector<std::pair<int64_t, int64_t>> v;
  if (own0 > 0) v.push_back({0, own0});
  if (own0 + own < total) v.push_back({own0 + own, total});
  return v;
}

}  // namespace

extern "C" {

int ozmm_grid_shape(int world, int* pr, int* pc) {
  if (world < 1 || !pr || !pc) return fail(OZMM_ERR_ARG, "world must be >= 1");
  int r = 1;
  if (world == 2) {
    r = 2;  // 2x1: each rank slices half the rows, keeps all columns (grid2d.grid_shape)
  } else {
    while ((r + 1) * (r + 1) <= world) ++r;
    while (world % r) --r;
  }
  *pr = r;
  *pc = world / r;
  return OZMM_OK;
}

const char* ozmm_grid_last_error(void) { return g_grid_err.c_str(); }

int ozmm_nccl_unique_id(void* id128) {
  if (!id128) return fail(OZMM_ERR_ARG, "null id buffer");
  Nccl& n = nccl();
  if (!n.ok) return fail(OZMM_ERR_NCCL, "%s", n.why.c_str());
  ncclUniqueId id;
  ncclResult_t r = n.get_unique_id(&id);
  if (r != ncclSuccess) return fail(OZMM_ERR_NCCL, "ncclGetUniqueId: %s", n.error_string(r));
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(id128, &id, sizeof(id));
  return OZMM_OK;
}

int ozmm_grid_create(ozmm_handle_t h, int device, int world, int rank, const void* nccl_id,
                     ozmm_allgather_fn hook, void* hook_ctx, ozmm_grid_t* out) {
  if (!h || !out) return fail(OZMM_ERR_ARG, "null handle or output");
  if (world < 1 || rank < 0 || rank >= world) return fail(OZMM_ERR_ARG, "rank outside [0, world)");
  if (world > 1 && !hook && !nccl_id)
    return fail(OZMM_ERR_ARG, "world > 1 needs an NCCL id or an all-gather hook");
  auto* g = new ozmm_grid();
  g->h = h;
  g->device = device;
  g->world = world;
  g->rank = rank;
  ozmm_grid_shape(world, &g->pr, &g->pc);
  g->gr = rank / g->pc;
  g->gc = rank % g->pc;
  g->hook = hook;
  g->hook_ctx = hook_ctx;
  auto bail = [&](int rc) {
    ozmm_grid_destroy(g);
    return rc;
  };
  if (cudaSetDevice(device) != cudaSuccess) return bail(fail(OZMM_ERR_CUDA, "cudaSetDevice"));
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  if (cudaStreamCreateWithFlags(&g->s_side, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithPriority(&g->s_comm, cudaStreamNonBlocking, hi) != cudaSuccess)
    return bail(fail(OZMM_ERR_CUDA, "stream creation failed"));
  for (cudaEvent_t* e : {&g->ev_split, &g->ev_b, &g->ev_a, &g->ev_side})
    if (cudaEventCreateWithFlags(e, cudaEventDisableTiming) != cudaSuccess)
      return bail(fail(OZMM_ERR_CUDA, "event creation failed"));
  if (!hook && nccl_id) {
    Nccl& n = nccl();
    if (!n.ok) return bail(fail(OZMM_ERR_NCCL, "%s", n.why.c_str()));
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof(id));
    ncclResult_t r = n.comm_init_rank(&g->world_comm, world, id, rank);
    if (r == ncclSuccess) r = n.comm_split(g->world_comm, g->gr, g->gc, &g->row_comm, nullptr);
    if (r == ncclSuccess) r = n.comm_split(g->world_comm, g->gc, g->gr, &g->col_comm, nullptr);
    if (r != ncclSuccess) return bail(fail(OZMM_ERR_NCCL, "NCCL init: %s", n.error_string(r)));
  }
  *out = g;
  return OZMM_OK;
}

int ozmm_grid_destroy(ozmm_grid_t g) {
  if (!g) return OZMM_OK;
  cudaSetDevice(g->device);
  if (g->s_side) cudaStreamSynchronize(g->s_side);
  if (g->s_comm) cudaStreamSynchronize(g->s_comm);
  Nccl& n = nccl();
  for (ncclComm_t c : {g->row_comm, g->col_comm, g->world_comm})
    if (c && n.ok) n.comm_destroy(c);
  for (void* p : {static_cast<void*>(g->a_pan), static_cast<void*>(g->b_pan),
                  static_cast<void*>(g->mu), static_cast<void*>(g->nu),
                  static_cast<void*>(g->lsa), static_cast<void*>(g->lsb),
                  static_cast<void*>(g->gflag)})
    if (p) cudaFree(p);
  for (cudaEvent_t e : {g->ev_split, g->ev_b, g->ev_a, g->ev_side})
    if (e) cudaEventDestroy(e);
  if (g->s_side) cudaStreamDestroy(g->s_side);
  if (g->s_comm) cudaStreamDestroy(g->s_comm);
  delete g;
  return OZMM_OK;
}

int ozmm_grid_coords(ozmm_grid_t g, int* pr, int* pc, int* gr, int* gc) {
  if (!g) return fail(OZMM_ERR_ARG, "null grid");
  if (pr) *pr = g->pr;
  if (pc) *pc = g->pc;
  if (gr) *gr = g->gr;
  if (gc) *gc = g->gc;
  return OZMM_OK;
}

int ozmm_dgemm_2d(ozmm_grid_t g, char transa, char transb, int64_t m, int64_t n, int64_t p,
                  double alpha, const double* A, int64_t lda, const double* B, int64_t ldb,
                  double beta, double* C, int64_t ldc, int k) {
  if (!g) return fail(OZMM_ERR_ARG, "null grid");
  const int64_t cells = static_cast<int64_t>(g->pr) * g->pc;
  if (m < 1 || n < 1 || p < 1) return fail(OZMM_ERR_ARG, "empty shape");
  if (m % cells || p % cells)
    return fail(OZMM_ERR_ARG, "m=%lld and p=%lld must be divisible by Pr*Pc=%lld",
                static_cast<long long>(m), static_cast<long long>(p), static_cast<long long>(cells));
  if (k < 1 || k > 32) return fail(OZMM_ERR_CONFIG, "k must be in 1..32");
  const int64_t mr = m / g->pr, pcols = p / g->pc;  // C block
  const int64_t ms = mr / g->pc, ps = pcols / g->pr;  // lines this rank slices
  if (ldc < pcols) return fail(OZMM_ERR_ARG, "ldc below the C block's %lld columns",
                               static_cast<long long>(pcols));
  int beta_bits = 0;
  if (ozmm_compute_beta(n, &beta_bits) != OZMM_OK) return fail(OZMM_ERR_ARG, "n out of range");
  const int64_t lds = ozmm_slice_ld(n);
  const int64_t plane_a = mr * lds, plane_b = pcols * lds;
  if (int rc = grow(&g->a_pan, &g->a_bytes, static_cast<size_t>(k * plane_a))) return rc;
  if (int rc = grow(&g->b_pan, &g->b_bytes, static_cast<size_t>(k * plane_b))) return rc;
  if (int rc = grow(&g->mu, &g->mu_n, static_cast<size_t>(mr))) return rc;
  if (int rc = grow(&g->nu, &g->nu_n, static_cast<size_t>(pcols))) return rc;
  if (int rc = grow(&g->lsa, &g->lsa_n, static_cast<size_t>(mr * k))) return rc;
  if (int rc = grow(&g->lsb, &g->lsb_n, static_cast<size_t>(pcols * k))) return rc;
  if (int rc = grow(&g->gflag, &g->gflag_n, static_cast<size_t>(g->pr) * g->pc)) return rc;
  GRID_CUDA(cudaSetDevice(g->device));
  cudaStream_t main_s = nullptr;
  {
    void* s = nullptr;
    GRID_OZ(ozmm_get_stream(g->h, &s));
    main_s = static_cast<cudaStream_t>(s);
  }
  const int64_t r0 = g->gc * ms, c0 = g->gr * ps;  // own rows / columns in the C block

  // 1. split into this rank's slot of the panels (handle stream); this call's
  // range flag starts clear
  GRID_OZ(ozmm_internal_fold_flags(g->h));
  GRID_OZ(ozmm_split_offset_strided(g->h, 'L', transa, ms, n, A, lda, k, beta_bits,
                                    g->a_pan + r0 * lds, lds, plane_a, g->mu + r0,
                                    g->lsa + r0 * k, 1, k));
  GRID_OZ(ozmm_split_offset_strided(g->h, 'R', transb, ps, n, B, ldb, k, beta_bits,
                                    g->b_pan + c0 * lds, lds, plane_b, g->nu + c0,
                                    g->lsb + c0 * k, 1, k));
  // this rank's range flag into its cell of the [pr][pc] grid matrix
  int* cell = g->gflag + g->gr * g->pc + g->gc;
  GRID_CUDA(cudaMemcpyAsync(cell, ozmm_internal_range_flag(g->h), sizeof(int),
                            cudaMemcpyDeviceToDevice, main_s));
  GRID_CUDA(cudaEventRecord(g->ev_split, main_s));

  // 2. grid-wide range check before anything writes C (the reference throws
  // from the split, split.cpp:124-125): gather the flags along the grid row,
  // then the rows along the grid column, and read the whole matrix -- every
  // rank sees the same flags and returns the same status
  GRID_CUDA(cudaStreamWaitEvent(g->s_comm, g->ev_split, 0));
  if (int rc = gather_group(g, 0, {{g->gflag + g->gr * g->pc, static_cast<int64_t>(sizeof(int))}}))
    return rc;
  if (int rc = gather_group(g, 1, {{g->gflag, static_cast<int64_t>(sizeof(int)) * g->pc}})) return rc;
  {
    std::vector<int> flags(static_cast<size_t>(g->pr) * g->pc, 0);
    GRID_CUDA(cudaMemcpyAsync(flags.data(), g->gflag, sizeof(int) * flags.size(),
                              cudaMemcpyDeviceToHost, g->s_comm));
    GRID_CUDA(cudaStreamSynchronize(g->s_comm));
    for (size_t i = 0; i < flags.size(); ++i)
      if (flags[i]) {
        GRID_CUDA(cudaMemsetAsync(ozmm_internal_range_flag(g->h), 0, sizeof(int), main_s));
        GRID_CUDA(cudaStreamSynchronize(main_s));
        return fail(OZMM_ERR_RANGE, "split: row magnitude too large for shift extraction "
                    "(grid rank %zu)", i);
      }
  }

  // 3. gathers on the comm stream: B (unblocks G2) first, then A
  {
    std::vector<std::pair<void*, int64_t>> bb, ab;
    for (int s = 0; s < k; ++s) bb.push_back({g->b_pan + s * plane_b, ps * lds});
    bb.push_back({g->nu, ps * 8});
    bb.push_back({g->lsb, ps * k * 4});
    for (int s = 0; s < k; ++s) ab.push_back({g->a_pan + s * plane_a, ms * lds});
    ab.push_back({g->mu, ms * 8});
    ab.push_back({g->lsa, ms * k * 4});
    if (int rc = gather_group(g, 1, bb)) return rc;
    GRID_CUDA(cudaEventRecord(g->ev_b, g->s_comm));
    if (int rc = gather_group(g, 0, ab)) return rc;
    GRID_CUDA(cudaEventRecord(g->ev_a, g->s_comm));
  }

  // 4. strips
  auto strip = [&](int64_t row0, int64_t rows, int64_t col0, int64_t cols) {
    return ozmm_gemm_slices_offset(g->h, rows, n, cols, k, beta_bits, 0, g->a_pan + row0 * lds,
                                   lds, plane_a, g->mu + row0, g->lsa + row0 * k, 1, k,
                                   g->b_pan + col0 * lds, lds, plane_b, g->nu + col0,
                                   g->lsb + col0 * k, 1, k, alpha, beta, C + row0 * ldc + col0,
                                   ldc, nullptr);
  };
  // G1 on the side stream: needs no communication
  GRID_CUDA(cudaStreamWaitEvent(g->s_side, g->ev_split, 0));
  GRID_OZ(ozmm_set_stream(g->h, g->s_side));
  int rc = strip(r0, ms, c0, ps);
  ozmm_set_stream(g->h, main_s);
  if (rc) return fail(rc, "G1: %s", ozmm_last_error(g->h));
  GRID_CUDA(cudaEventRecord(g->ev_side, g->s_side));
  // G2 after B's gather, G3 after A's
  GRID_CUDA(cudaStreamWaitEvent(main_s, g->ev_b, 0));
  for (auto& c : others(pcols, c0, ps)) GRID_OZ(strip(r0, ms, c.first, c.second - c.first));
  GRID_CUDA(cudaStreamWaitEvent(main_s, g->ev_a, 0));
  for (auto& r : others(mr, r0, ms)) GRID_OZ(strip(r.first, r.second - r.first, 0, pcols));
  GRID_CUDA(cudaStreamWaitEvent(main_s, g->ev_side, 0));
  return OZMM_OK;
}

}  // extern "C"
