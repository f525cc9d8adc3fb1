// K2+K3 -- the fused ozIMMU_H GEMM: tcgen05 kind::i8 anti-diagonal group
// accumulation in TMEM + exact FP64 flush + alpha/beta epilogue.
//
// What it computes (per output tile, bit-identical to the reference):
//   D = 0                                                     scheme.cpp:78
//   for each chunk c in flush order (g ascending, then chunk):
//       acc_c = sum_{s in chunk c} A_s * B_{g-s}   (exact INT32)  scheme.cpp:84-90
//       D    += (mu_i * 2^(2-beta*g) * acc_c) * nu_j  (2 exact muls, 1 RN add)
//                                                             scheme.cpp:29-41, :93-94
//   C_out = fl(fl(alpha*D) + fl(beta*C_in))                     scheme.cpp:286-287
// where chunks split each anti-diagonal group g every r products (:91).
//
// B200 mapping.  One CTA owns a 128 x BN tile of C.  The chunks are processed
// in "batches" of at most kNAcc chunks; every chunk of a batch owns its own
// INT32 accumulator of BN TMEM columns (kNAcc * BN <= 512).  The K loop runs
// OUTERMOST inside a batch: each pipeline stage holds, for one 32-byte K step,
// every A slice and every B slice the batch needs, and the single MMA thread
// issues all of the batch's slice products on that stage into their chunk
// accumulators.  So each loaded slice tile is reused by every product that
// needs it (A_1 by k products, ...): ~(k+1)/2 x fewer bytes per MMA than
// streaming one product at a time.  D never exists in memory: after the last
// K step of a batch the epilogue warps read the batch's accumulators out of
// TMEM (tcgen05.ld) in flush order and fold them into FP64 D held in
// registers; after the last batch they apply alpha/beta and store C.
//
// Warp roles (320 threads): warp 0 = TMA producer, warp 1 = TMEM allocator +
// MMA issuer, warps 2..9 = epilogue (warp w reads TMEM lanes 32*(w%4).. and
// the column half (w-2)/4 of the tile).
#pragma once

#include <cstdint>
#include <cuda.h>

#include "fp64_exact.cuh"
#include "ptx.cuh"

namespace ozb {

constexpr int kBM = 128;         // UMMA M (cta_group::1), TMEM lanes
constexpr int kBK = 32;          // bytes of K per pipeline stage = one MMA (kind::i8, K=32)
// Slice counts up to 32 (the FP64 floor is reached by k ~ 13-14; the reference
// only requires k >= 1).  The schedule tables below travel as kernel parameters
// (about 16 KB of the 32 KB parameter space).
constexpr int kMaxK = 32;
constexpr int kMaxChunks = 528;    // >= k(k+1)/2 for k <= kMaxK (r = 1)
constexpr int kMaxProducts = 528;  // k(k+1)/2 for k <= kMaxK
constexpr int kMaxBatches = 192;
constexpr int kMaxPasses = 384;
// CTA-pair epilogue actions (schedule.hpp FlushAct): flush accumulator, park
// accumulator, flush a parked chunk; at most 2 per chunk, at most kMaxPark slots
constexpr int kActFlush = 0, kActPark = 1, kActUnpark = 2;
constexpr int kMaxActs = 2 * kMaxChunks;
constexpr int kMaxPark = 16;
constexpr int kMaxAGroups = 528;
constexpr int kGemmThreads = 320;
constexpr int kEpiWarps = 8;

struct GemmParams {
  int m, p;            // output shape
  int n_kb;            // number of 32-byte K steps (ceil(lds / 32))
  int tiles_m, tiles_n;
  int group_m;         // raster: tiles of this many row-blocks are visited together
  int nbatch, npass;
  int beta;            // slice width (bits)
  int stages;          // smem pipeline depth
  int a_slots, b_slots;  // slice tiles per stage (max over passes)
  int n_chunks;
  uint32_t idesc_xor;  // diagnostic build only (OZMM_IDESC_XOR): flips instruction-descriptor bits
  int dup_mma;         // diagnostic build only (OZMM_DUP_MMA): repeat each product's MMAs (timing only)
  uint64_t* tile_trace;  // optional [tiles][8] globaltimer stamps of each leader CTA (OZMM_TILE_TRACE)
  int group_pairs;     // CTA-pair kernel: issue A groups two at a time (OZMM_GROUP_PAIRS)
  int kpair;           // CTA-pair kernel: thin passes take K blocks in pairs (OZMM_KPAIR)
  // Offset-binary operands (CTA-pair kernel only; slicer.cuh): the slice planes
  // hold slice + o_s (o_1 = 2^beta, o_s = max(2, 2^(beta-1)), slice_offset) as u8 and the MMAs run
  // u8 x u8.  For a chunk c the accumulator then holds, mod 2^32,
  //   acc_c + sum_{(s,t) in c} [ o_t lsa[s][i] + o_s lsb[t][j] + o_s o_t n ]
  // and the epilogue subtracts that exactly (lsa / lsb = signed line sums).
  int bias;
  int64_t n_inner;
  const int32_t* lsa;  // row sums of the signed A slices: lsa[(s-1)*lsa_plane + i*lsa_lstride]
  const int32_t* lsb;  // column sums of the signed B slices (same indexing)
  int64_t lsa_plane, lsb_plane, lsa_lstride, lsb_lstride;
  int hint_a, hint_b;  // L2 policies of the A / B slice loads (0 normal, 1 evict_first, 2 evict_last)
  // FP64 flush scaling (scheme.cpp:29-41 with the caller's unit vectors):
  //   0 group-wise        ru = mu_i 2^(2-beta g),   cv = nu_j                (:93-94)
  //   1 per-product const ru = mu_i 2^(1-beta s),   cv = nu_j 2^(1-beta t)   (:205, units_of)
  //   2 per-product units ru = units_a[s-1][i],     cv = units_b[t-1][j]     (RN per slice)
  int scale_mode;
  const double* units_a;  // [k][m] per-slice row units (scale_mode 2)
  const double* units_b;  // [k][p] per-slice column units (scale_mode 2)
  double alpha, beta_c;
  const double* mu;    // [m] row shifts of op(A)
  const double* nu;    // [p] column shifts of op(B)
  // [m x ldc] (read: fl(beta*c) is always formed, as the reference does).  nullptr
  // only from the host entry's beta = 0, alpha > 0 mode, where fl(alpha*d) + fl(0*c)
  // equals fl(alpha*d) for every finite c (d is never -0) and the host patches the
  // non-finite c entries afterwards.
  const double* c_in;
  double* c_out;
  int64_t ldc;
  int32_t* dump;       // optional [n_chunks][m][p] INT32 chunk sums (parity/debug)
  // per batch: first chunk, chunk count, pass range [pass0, pass1)
  uint16_t b_c0[kMaxBatches], b_nc[kMaxBatches], b_pass0[kMaxBatches], b_pass1[kMaxBatches];
  // per pass: A slice range, B slice range (1-based, inclusive), product range
  uint8_t p_alo[kMaxPasses], p_ahi[kMaxPasses], p_blo[kMaxPasses], p_bhi[kMaxPasses];
  uint16_t p_p0[kMaxPasses], p_p1[kMaxPasses];
  // per product: accumulator slot | first-product flag (bit 7), A slice, B slice
  uint8_t pr_ci[kMaxProducts], pr_s[kMaxProducts], pr_t[kMaxProducts];
  // CTA-pair kernel, per product: B tile offset within its pass's B buffer in
  // smem-descriptor units (bytes >> 4) | accumulator << 16 | first << 24
  uint32_t pr_info[kMaxProducts];
  // per chunk in flush order: group g and first A slice s0
  uint8_t c_g[kMaxChunks];
  uint8_t c_s[kMaxChunks];
  uint8_t c_e[kMaxChunks];  // last A slice of chunk c (products s = c_s .. c_e, t = g - s)
  // CTA-pair kernel: per pass the A-slice groups [p_g0, p_g1); per group the
  // A slice and its product range (products are sorted by A slice in a pass)
  uint16_t p_g0[kMaxPasses], p_g1[kMaxPasses];
  uint8_t ag_s[kMaxAGroups];
  uint16_t ag_p0[kMaxAGroups], ag_p1[kMaxAGroups];
  int b_buf_slots;     // CTA-pair kernel: B slice tiles per B buffer (sized per launch)
  // CTA-pair kernel: odd passes sweep the K blocks in reverse, so each pass starts on
  // the K blocks the previous one loaded last (still in L2); the INT32 sums are
  // order-free, so results are unchanged
  int ksnake;
  // CTA-pair kernel: per batch its chunk ids (accumulator ci holds b_cid[b * 4 + ci])
  // and its epilogue actions act[b_act0[b] .. b_act1[b]) (schedule.hpp FlushAct:
  // chunk id | kind << 10 | accumulator << 12 | park slot << 16); park: per-SM
  // scratch of park_slots INT32 128 x 128 tiles per CTA, or null when nothing is parked
  uint16_t b_cid[kMaxBatches * 4];
  uint16_t b_act0[kMaxBatches], b_act1[kMaxBatches];
  uint32_t act[kMaxActs];
  int32_t* park;
  int park_slots;
};

template <int kBN>
struct GemmCfg {
  static constexpr int kNAcc = 512 / kBN;               // accumulators per batch
  static constexpr uint32_t kATile = kBM * kBK;         // bytes per A slice tile
  static constexpr uint32_t kBTile = kBN * kBK;         // bytes per B slice tile
  static constexpr uint32_t kIdesc = ptx::idesc_i8(kBM, kBN);
};

// Row factor of chunk c's flush for row `row` (mu = the row's shift).
__device__ __forceinline__ double flush_row_scale(const GemmParams& P, int c, int row,
                                                  double mu) {
  if (P.scale_mode == 0) return __dmul_rn(mu, pow2(2 - P.beta * P.c_g[c]));  // ldexp(mu, 2-beta g)
  if (P.scale_mode == 1) return __dmul_rn(mu, pow2(1 - P.beta * P.c_s[c]));  // unit(s-1, i)
  return row < P.m ? P.units_a[static_cast<int64_t>(P.c_s[c] - 1) * P.m + row] : 0.0;
}

// Column factor of chunk c's flush for column `col` (nu = the column's shift).
__device__ __forceinline__ double flush_col_scale(const GemmParams& P, int c, int col,
                                                  double nu) {
  if (P.scale_mode == 0) return nu;
  const int t = P.c_g[c] - P.c_s[c];
  if (P.scale_mode == 1) return __dmul_rn(nu, pow2(1 - P.beta * t));  // unit(t-1, j)
  return col < P.p ? P.units_b[static_cast<int64_t>(t - 1) * P.p + col] : 0.0;
}

// Dynamic smem: [stages x (a_slots*ATile + b_slots*BTile)] tiles (1024-aligned)
// then barriers and the nu cache.
template <int kBN>
__global__ void __launch_bounds__(kGemmThreads, 1)
    ozimmu_gemm_kernel(const __grid_constant__ CUtensorMap map_a,
                       const __grid_constant__ CUtensorMap map_b,
                       const __grid_constant__ GemmParams P) {
  using Cfg = GemmCfg<kBN>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t a_bytes = P.a_slots * Cfg::kATile;
  const uint32_t stage_bytes = a_bytes + P.b_slots * Cfg::kBTile;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + P.stages * stage_bytes);
  uint64_t* empty = full + P.stages;
  uint64_t* tmem_full = empty + P.stages;
  uint64_t* tmem_empty = tmem_full + 1;
  uint32_t* tmem_base_smem = reinterpret_cast<uint32_t*>(tmem_empty + 1);
  double* nu_s = reinterpret_cast<double*>(tmem_base_smem + 4);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  // grouped raster over tiles
  const int bid = blockIdx.x;
  const int per_group = P.group_m * P.tiles_n;
  const int first_m = (bid / per_group) * P.group_m;
  const int gm = min(P.group_m, P.tiles_m - first_m);
  const int tm = first_m + (bid % per_group) % gm;
  const int tn = (bid % per_group) / gm;

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&map_a);
    ptx::tma_prefetch_desc(&map_b);
    for (int s = 0; s < P.stages; ++s) {
      ptx::mbar_init(full + s, 1);
      ptx::mbar_init(empty + s, 1);
    }
    ptx::mbar_init(tmem_full, 1);
    ptx::mbar_init(tmem_empty, kEpiWarps);
    ptx::fence_barrier_init();
  }
  if (warp == 1) ptx::tmem_alloc<512>(tmem_base_smem);
  for (int j = threadIdx.x; j < kBN; j += blockDim.x) {
    const int col = tn * kBN + j;
    nu_s[j] = col < P.p ? P.nu[col] : 0.0;
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_base_smem;

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer
    if (ptx::elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int q = 0; q < P.npass; ++q) {
        const int alo = P.p_alo[q], ahi = P.p_ahi[q], blo = P.p_blo[q], bhi = P.p_bhi[q];
        const uint32_t tx = (ahi - alo + 1) * Cfg::kATile + (bhi - blo + 1) * Cfg::kBTile;
        for (int kb = 0; kb < P.n_kb; ++kb) {
          ptx::mbar_wait(empty + stage, phase ^ 1);
          uint8_t* st = smem + stage * stage_bytes;
          ptx::mbar_arrive_expect_tx(full + stage, tx);
          for (int s = alo; s <= ahi; ++s)
            ptx::tma_load_3d(st + (s - alo) * Cfg::kATile, &map_a, full + stage, kb * kBK,
                             tm * kBM, s - 1);
          for (int t = blo; t <= bhi; ++t)
            ptx::tma_load_3d(st + a_bytes + (t - blo) * Cfg::kBTile, &map_b, full + stage,
                             kb * kBK, tn * kBN, t - 1);
          if (++stage == P.stages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------- MMA issuer
    int stage = 0;
    uint32_t phase = 0;
    for (int b = 0; b < P.nbatch; ++b) {
      ptx::mbar_wait(tmem_empty, (b & 1) ^ 1);
      ptx::tc_fence_after();
      for (int q = P.b_pass0[b]; q < P.b_pass1[b]; ++q) {
        const int alo = P.p_alo[q], blo = P.p_blo[q], p0 = P.p_p0[q], p1 = P.p_p1[q];
        for (int kb = 0; kb < P.n_kb; ++kb) {
          ptx::mbar_wait(full + stage, phase);
          ptx::tc_fence_after();
          if (ptx::elect_one()) {
            const uint32_t sa = ptx::smem_u32(smem + stage * stage_bytes);
            const uint32_t sb = sa + a_bytes;
            for (int pr = p0; pr < p1; ++pr) {
              const uint32_t ci = P.pr_ci[pr];
              const uint64_t adesc =
                  ptx::smem_desc(sa + (P.pr_s[pr] - alo) * Cfg::kATile, 256, 6);
              const uint64_t bdesc =
                  ptx::smem_desc(sb + (P.pr_t[pr] - blo) * Cfg::kBTile, 256, 6);
              const uint32_t acc = (kb > 0 || !(ci & 0x80u)) ? 1u : 0u;
              ptx::mma_i8(tmem_base + (ci & 0x7Fu) * kBN, adesc, bdesc, Cfg::kIdesc, acc);
            }
            ptx::mma_commit(empty + stage);  // frees the smem stage when these MMAs finish
          }
          __syncwarp();
          if (++stage == P.stages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      if (ptx::elect_one()) ptx::mma_commit(tmem_full);  // batch accumulators complete
      __syncwarp();
    }
  } else {
    // --------------------------------------------------------- epilogue
    const int ew = warp - 2;             // 0..7
    const int quarter = warp & 3;        // TMEM lane quarter this warp may access
    const int half = ew >> 2;            // column half of the tile
    constexpr int kHalf = kBN / 2;
    constexpr int kLd = kHalf < 32 ? kHalf : 32;  // tcgen05.ld width
    const int row = tm * kBM + quarter * 32 + lane;
    const int col0 = tn * kBN + half * kHalf;
    const bool row_ok = row < P.m;
    const double mu = row_ok ? P.mu[row] : 0.0;
    double d[kHalf];
#pragma unroll
    for (int j = 0; j < kHalf; ++j) d[j] = 0.0;

    for (int b = 0; b < P.nbatch; ++b) {
      ptx::mbar_wait(tmem_full, b & 1);
      ptx::tc_fence_after();
      const int c0 = P.b_c0[b], nc = P.b_nc[b];
      for (int ci = 0; ci < nc; ++ci) {
        const int c = c0 + ci;
        const double ru = flush_row_scale(P, c, row, mu);
#pragma unroll
        for (int cc = 0; cc < kHalf; cc += kLd) {
          uint32_t v[kLd];
          ptx::tmem_ld_32x32b<kLd>(
              tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + ci * kBN + half * kHalf + cc,
              v);
          ptx::tmem_ld_wait();
          if (P.dump != nullptr && row_ok) {
            int32_t* dst = P.dump + (static_cast<int64_t>(c) * P.m + row) * P.p;
#pragma unroll
            for (int j = 0; j < kLd; ++j)
              if (col0 + cc + j < P.p) dst[col0 + cc + j] = static_cast<int32_t>(v[j]);
          }
#pragma unroll
          for (int j = 0; j < kLd; ++j) {
            const double cv = flush_col_scale(P, c, col0 + cc + j, nu_s[half * kHalf + cc + j]);
            const double t = __dmul_rn(__dmul_rn(ru, static_cast<double>(static_cast<int32_t>(v[j]))), cv);
            d[cc + j] = __dadd_rn(d[cc + j], t);
          }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(tmem_empty);
    }

    if (row_ok) {
      const double* cin = P.c_in ? P.c_in + static_cast<int64_t>(row) * P.ldc : nullptr;
      double* cout = P.c_out + static_cast<int64_t>(row) * P.ldc;
#pragma unroll
      for (int j = 0; j < kHalf; ++j) {
        const int col = col0 + j;
        if (col < P.p)
          cout[col] = __dadd_rn(__dmul_rn(P.alpha, d[j]), cin ? __dmul_rn(P.beta_c, cin[col]) : 0.0);
      }
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem_base);
  }
}

}  // namespace ozb
