// K2+K3, CTA-pair variant: the fused ozIMMU_H GEMM computed by a 2-CTA
// cluster with tcgen05 cta_group::2 (UMMA M = 256, N = kBN).
//
// Why a pair: with M = 128 x N = 64 per CTA the tensor core's shared-memory
// operand fetch (A 128x32 B + B 64x32 B per 32-cycle MMA) saturates before the
// INT8 datapath (ncu: sm__pipe_tc_cycles_active 83 % at 45 % tensor
// utilisation, profiles/r1/gemm_v1_bn64_*).  In a CTA pair each SM owns 128
// rows of the output but the B operand is split N/2 + N/2 across the two SMs:
// per SM 4 KB + kBN*16 B of operand reads per kBN/2-cycle MMA.
//
// Pipeline (per CTA; K advances in 128-byte blocks, 128-byte swizzle):
//   * B buffers (2): for the current K block every B slice of the pass
//     (kBN/2 rows x 128 B each), resident while all of the block's MMAs run;
//   * A ring (P.stages, 5 for tensor-bound schedules): one A slice tile
//     (128 rows x 128 B) per stage, streamed in pass order; the MMA thread
//     takes the A groups two per barrier round (P.group_pairs) and issues every
//     product that uses them (4 MMAs of K = 32 each) into its chunk
//     accumulator, then releases both stages together.
//   * Operands are offset-binary u8 planes by default (P.bias): the epilogue
//     removes the offsets' contribution exactly, see GemmParams.
// One TMA box per 128-byte row keeps the TMA request count 4x below a
// 32-byte-row design (ncu: l1tex2xbar request cycles were 87 % busy there).
//
// Roles per CTA (384 threads): warp 0 = TMA producer (both CTAs load their own
// A rows and their half of the B rows; bytes are counted on the LEADER's
// barriers), warp 1 = TMEM allocator (both) + MMA issuer (leader only),
// warps 4..11 = epilogue (each CTA drains its own TMEM: its 128 rows x kBN
// columns, 64 columns per warp).  Commits multicast to both CTAs' barriers;
// both CTAs' epilogues release the accumulators on the leader's tmem_empty.
#pragma once

#include "ozimmu_gemm.cuh"

namespace ozb {

constexpr int kPairThreads = 384;
constexpr int kPairEpiWarps = 8;  // per CTA
constexpr int kKB = 128;          // bytes of K per block (= one 128B swizzle row)
constexpr int kBBufs = 2;
// Shared-memory header in front of the operand pools (byte offsets): barriers,
// TMEM slot, the tile's column shifts nu, their exponents for the fast flush, and
// the per-column offset corrections of a batch.
constexpr int kHdrTmem = 512, kHdrNu = 1024, kHdrEc = 2048, kHdrCcol = 3072;
constexpr int kPairHdr = 5120;
// diagnostics (OZMM_TILE_TRACE, -DOZMM_DIAG builds): per-CTA stamps 0..7 (globaltimer,
// see below) and wait accounting in SM clocks: 8 MMA thread on A tiles, 9 on B
// tiles, 10 on TMEM (epilogue drain), 11 MMA thread total; 12/13 globaltimer when
// the epilogue sees batch 0 / the last batch complete; 14/15 producer on free A / B
// slots
constexpr int kTraceSlots = 16;
#ifdef OZMM_DIAG
#define OZMM_TWAIT(slot, call)                    \
  do {                                            \
    const long long tw0_ = trace ? clock64() : 0; \
    call;                                         \
    if (trace) tw_[slot] += clock64() - tw0_;     \
  } while (0)
#else
#define OZMM_TWAIT(slot, call) call
#endif
// timing probe (diag builds, OZMM_DUP_MMA=-1): skip the MMAs, keep loads and commits
#ifdef OZMM_DIAG
#define OZMM_MMA_ON (P.dup_mma >= 0)
#else
#define OZMM_MMA_ON true
#endif
template <int kBN, int kPairs = 1>
struct PairCfg {
  static constexpr int kNAcc = 512 / kBN;
  static constexpr int kCluster = 2 * kPairs;             // CTAs per cluster
  static constexpr int kAPart = kBM / kPairs;             // A rows each CTA loads (multicast)
  static constexpr int kBHalf = kBN / 2;                  // B rows loaded per CTA
  static constexpr uint32_t kATile = kBM * kKB;           // 16 KB
  static constexpr uint32_t kBTile = kBHalf * kKB;        // bytes per CTA per B slice
  static constexpr int kMaxBSlots = 8;                    // B slices resident per K block
  static constexpr uint32_t kIdesc = ptx::idesc_i8(2 * kBM, kBN);
  static constexpr int kMaxStages = (512 - 16 - 8 * 2 * kBBufs) / 16;  // barrier header room
  // host: dynamic shared memory for B buffers of b_slots tiles and `stages` A stages
  static constexpr size_t smem_bytes(int b_slots, int stages) {
    return 1024 + kPairHdr + size_t(kBBufs) * b_slots * kBTile + size_t(stages) * kATile;
  }
  // the C pass stages the 128 x kBN FP64 tile (rows padded by one double) in the pools
  static constexpr size_t kStageBytes = size_t(kBM) * (kBN + 1) * 8;
};

// kPairs = 2: a 4-CTA cluster of two CTA pairs side by side along N that share
// the A tiles (same 256 rows): each CTA loads half of its 128-row A tile and
// TMA-multicasts it to the same-half CTA of the other pair, halving A's L2->SM
// traffic (A is 2/3 of it).  An A stage is released by both pairs' MMAs, so the
// pairs are coupled through the A ring only; B stays per pair.  A 4-CTA cluster
// can only use 132 of the 148 SMs, which costs more than the L2 traffic saves
// (profiles/r1/quad_ab.txt): this variant is off by default.
template <int kBN, int kPairs>
__global__ void __cluster_dims__(2 * kPairs, 1, 1) __launch_bounds__(kPairThreads, 1)
    ozimmu_gemm_pair_kernel(const __grid_constant__ CUtensorMap map_a,
                            const __grid_constant__ CUtensorMap map_b,
                            const __grid_constant__ GemmParams P) {
  using Cfg = PairCfg<kBN, kPairs>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-aligned (128-byte swizzle atoms); pointer arithmetic on smem_raw keeps
  // the shared state space visible to the compiler (LDS/STS, not generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  const int n_a = P.stages;  // A ring depth
  const uint32_t b_buf = static_cast<uint32_t>(P.b_buf_slots) * Cfg::kBTile;  // one B buffer
  uint64_t* b_full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* b_empty = b_full + kBBufs;
  uint64_t* a_full = b_empty + kBBufs;
  uint64_t* a_empty = a_full + n_a;
  uint64_t* tmem_full = a_empty + n_a;
  uint64_t* tmem_empty = tmem_full + 1;
  uint32_t* tmem_base_smem = reinterpret_cast<uint32_t*>(smem + kHdrTmem);
  double* nu_s = reinterpret_cast<double*>(smem + kHdrNu);
  int32_t* ec20 = reinterpret_cast<int32_t*>(smem + kHdrEc);  // exponent of nu_j << 20
  // offset mode: the batch's per-column corrections [kNAcc][kBN] (int32)
  uint32_t* ccol = reinterpret_cast<uint32_t*>(smem + kHdrCcol);
  uint8_t* bbuf = smem + kPairHdr;
  uint8_t* aring = bbuf + kBBufs * b_buf;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // diagnostics: stamps 0 start, 1 prologue done, 2 first MMA issued, 3 batch 0
  // drained, 4 second batch's first MMA, 5 last batch drained, 6 C written, 7 end
  uint64_t* trace = P.tile_trace ? P.tile_trace + static_cast<int64_t>(blockIdx.x) * kTraceSlots : nullptr;
  if (trace && threadIdx.x == 0) trace[0] = ptx::globaltimer();
  const uint32_t rank = ptx::cluster_ctarank();
  const uint32_t lead_rank = rank & ~1u;      // leader of this CTA's pair
  const uint32_t pp = rank >> 1;              // pair index in the cluster
  const bool leader = rank == lead_rank;
  const uint16_t pair_mask = static_cast<uint16_t>(0x3u << (2 * pp));
  const uint16_t all_mask = static_cast<uint16_t>((1u << Cfg::kCluster) - 1);

  // grouped raster over cluster tiles (256 rows x kPairs*kBN columns)
  const int bid = blockIdx.x / Cfg::kCluster;
  const int per_group = P.group_m * P.tiles_n;
  const int first_m = (bid / per_group) * P.group_m;
  const int gm = min(P.group_m, P.tiles_m - first_m);
  const int tm = first_m + (bid % per_group) % gm;  // pair row-block (256 rows)
  const int tn = (bid % per_group) / gm;
  const int row_base = tm * 2 * kBM + static_cast<int>(rank & 1u) * kBM;
  const int col_tile = tn * kPairs + static_cast<int>(pp);  // this pair's kBN-column tile
  const int n_kb = P.n_kb;  // 128-byte K blocks

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&map_a);
    ptx::tma_prefetch_desc(&map_b);
    for (int s = 0; s < kBBufs; ++s) {
      ptx::mbar_init(b_full + s, 1);
      ptx::mbar_init(b_empty + s, 1);
    }
    for (int s = 0; s < n_a; ++s) {
      ptx::mbar_init(a_full + s, 1);
      ptx::mbar_init(a_empty + s, kPairs);  // released by every pair that reads it
    }
    ptx::mbar_init(tmem_full, 1);
    ptx::mbar_init(tmem_empty, 2 * kPairEpiWarps);
    ptx::fence_barrier_init();
  }
  if (warp == 1) ptx::tmem_alloc_pair<512>(tmem_base_smem);
  for (int j = threadIdx.x; j < kBN; j += blockDim.x) {
    const int col = col_tile * kBN + j;
    const double nu = col < P.p ? P.nu[col] : 0.0;
    nu_s[j] = nu;
    // unbiased exponent << 20 (the high word's exponent field) for the fast flush
    ec20[j] = static_cast<int32_t>(((__double2hiint(nu) >> 20) & 0x7FF) - 1023) * (1 << 20);
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();  // barrier inits + TMEM address visible cluster-wide
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_base_smem;
  if (trace && threadIdx.x == 0) trace[1] = ptx::globaltimer();

  // registers: the producer / MMA warpgroup needs few, the epilogue holds a 64-column
  // FP64 row of D plus 32 of a chunk's INT32 sums per thread (no spills at 216)
  if (warp < 4) {
    ptx::setmaxnreg_dec<72>();
    if (warp == 0) {
      // ------------------------------------------------------ TMA producer
      if (ptx::elect_one()) {
        long long tw_[16] = {};
        (void)tw_;
        int bi = 0, ai = 0;
        uint32_t bph = 0, aph = 0;
        const int b_row = col_tile * kBN + static_cast<int>(rank & 1u) * Cfg::kBHalf;
        const int a_row = row_base + static_cast<int>(pp) * Cfg::kAPart;
        const uint16_t a_mask = static_cast<uint16_t>(kPairs == 1 ? 0 : (0x5u << (rank & 1u)));
        const uint64_t pol_a = ptx::l2_policy(P.hint_a), pol_b = ptx::l2_policy(P.hint_b);
        for (int q = 0; q < P.npass; ++q) {
          const int blo = P.p_blo[q], bhi = P.p_bhi[q], g0 = P.p_g0[q], g1 = P.p_g1[q];
          const uint32_t btx = 2u * (bhi - blo + 1) * Cfg::kBTile;
          const int nbw = bhi - blo + 1;
          // K block of loop step kb (the MMA side only needs the step: integer sums)
          const bool rev = P.ksnake && (q & 1);
          if (kPairs == 1 && P.kpair && 2 * nbw <= P.b_buf_slots && n_kb % 2 == 0) {
            // K-pair pass: one B buffer holds K blocks kb and kb+1; each A group loads
            // both of its K blocks into consecutive ring slots
            for (int kb = 0; kb < n_kb; kb += 2) {
              const int kc = rev ? n_kb - 2 - kb : kb;  // first K block of the pair
              OZMM_TWAIT(15, ptx::mbar_wait(b_empty + bi, bph ^ 1));
              const uint32_t fb = ptx::mapa_shared(b_full + bi, lead_rank);
              if (leader) ptx::mbar_arrive_expect_tx(b_full + bi, 2u * btx);
              uint8_t* dst = bbuf + bi * b_buf;
              for (int h = 0; h < 2; ++h)
                for (int t = blo; t <= bhi; ++t)
                  ptx::tma_load_3d_pair_hint(dst + (h * nbw + t - blo) * Cfg::kBTile, &map_b, fb,
                                             (kc + h) * kKB, b_row, t - 1, pol_b);
              if (++bi == kBBufs) {
                bi = 0;
                bph ^= 1;
              }
              for (int g = g0; g < g1; ++g)
                for (int h = 0; h < 2; ++h) {
                  OZMM_TWAIT(14, ptx::mbar_wait(a_empty + ai, aph ^ 1));
                  const uint32_t fa = ptx::mapa_shared(a_full + ai, lead_rank);
                  if (leader) ptx::mbar_arrive_expect_tx(a_full + ai, 2u * Cfg::kATile);
                  ptx::tma_load_3d_pair_hint(aring + ai * Cfg::kATile, &map_a, fa, (kc + h) * kKB,
                                             a_row, P.ag_s[g] - 1, pol_a);
                  if (++ai == n_a) {
                    ai = 0;
                    aph ^= 1;
                  }
                }
            }
            continue;
          }
          for (int kb = 0; kb < n_kb; ++kb) {
            const int kc = rev ? n_kb - 1 - kb : kb;
            OZMM_TWAIT(15, ptx::mbar_wait(b_empty + bi, bph ^ 1));
            {
              const uint32_t fb = ptx::mapa_shared(b_full + bi, lead_rank);
              if (leader) ptx::mbar_arrive_expect_tx(b_full + bi, btx);
              uint8_t* dst = bbuf + bi * b_buf;
              for (int t = blo; t <= bhi; ++t)
                ptx::tma_load_3d_pair_hint(dst + (t - blo) * Cfg::kBTile, &map_b, fb, kc * kKB,
                                           b_row, t - 1, pol_b);
            }
            if (++bi == kBBufs) {
              bi = 0;
              bph ^= 1;
            }
            for (int g = g0; g < g1; ++g) {
              OZMM_TWAIT(14, ptx::mbar_wait(a_empty + ai, aph ^ 1));
              const uint32_t fa = ptx::mapa_shared(a_full + ai, lead_rank);
              if (leader) ptx::mbar_arrive_expect_tx(a_full + ai, 2u * Cfg::kATile);
              if constexpr (kPairs == 1)
                ptx::tma_load_3d_pair_hint(aring + ai * Cfg::kATile, &map_a, fa, kc * kKB, a_row,
                                           P.ag_s[g] - 1, pol_a);
              else
                ptx::tma_load_3d_pair_mc(aring + ai * Cfg::kATile + pp * Cfg::kAPart * kKB, &map_a,
                                         a_full + ai, kc * kKB, a_row, P.ag_s[g] - 1, a_mask, pol_a);
              if (++ai == n_a) {
                ai = 0;
                aph ^= 1;
              }
            }
          }
        }
#ifdef OZMM_DIAG
        if (trace && leader) trace[14] = tw_[14], trace[15] = tw_[15];
#endif
      }
    } else if (warp == 1) {
      // ------------------------------------------- MMA issuer (leader CTA)
      // u8 x u8 for offset-binary planes (instruction-descriptor bits 7 / 10)
#ifdef OZMM_DIAG
      const uint32_t idesc = (P.bias ? (Cfg::kIdesc & ~((1u << 7) | (1u << 10))) : Cfg::kIdesc) ^ P.idesc_xor;
#else
      const uint32_t idesc = P.bias ? (Cfg::kIdesc & ~((1u << 7) | (1u << 10))) : Cfg::kIdesc;
#endif
      if (leader) {
        long long tw_[16] = {};
        (void)tw_;
#ifdef OZMM_DIAG
        const long long t_mma0 = clock64();
#endif
        int bi = 0, ai = 0;
        uint32_t bph = 0, aph = 0;
        for (int b = 0; b < P.nbatch; ++b) {
          OZMM_TWAIT(10, ptx::mbar_wait(tmem_empty, (b & 1) ^ 1));
          ptx::tc_fence_after();
          for (int q = P.b_pass0[b]; q < P.b_pass1[b]; ++q) {
            const int blo = P.p_blo[q], g0 = P.p_g0[q], g1 = P.p_g1[q];
            const int nbw = P.p_bhi[q] - blo + 1;
            if (kPairs == 1 && P.kpair && 2 * nbw <= P.b_buf_slots && n_kb % 2 == 0) {
              // K-pair pass: each product's MMAs for K blocks kb and kb+1 back to
              // back -- runs of 8 MMAs on one accumulator instead of 4
              for (int kb = 0; kb < n_kb; kb += 2) {
                OZMM_TWAIT(9, ptx::mbar_wait(b_full + bi, bph));
                ptx::tc_fence_after();
                if (trace && kb == 0 && q == P.b_pass0[b] && b < 2 && lane == 0) trace[2 + 2 * b] = ptx::globaltimer();
                const uint64_t bdesc0 = ptx::smem_desc(ptx::smem_u32(bbuf + bi * b_buf), 1024, 2);
                const uint32_t bstep = (nbw * Cfg::kBTile) >> 4;  // K block kb+1's tiles
                for (int g = g0; g < g1; ++g) {
                  const int s1 = ai + 1 == n_a ? 0 : ai + 1;
                  const uint32_t ph1 = ai + 1 == n_a ? aph ^ 1 : aph;
                  OZMM_TWAIT(8, ptx::mbar_wait(a_full + ai, aph));
                  OZMM_TWAIT(8, ptx::mbar_wait(a_full + s1, ph1));
                  ptx::tc_fence_after();
                  if (ptx::elect_one()) {
                    const uint64_t ad0 = ptx::smem_desc(ptx::smem_u32(aring + ai * Cfg::kATile), 1024, 2);
                    const uint64_t ad1 = ptx::smem_desc(ptx::smem_u32(aring + s1 * Cfg::kATile), 1024, 2);
                    for (int pr = P.ag_p0[g]; pr < P.ag_p1[g]; ++pr) {
                      const uint32_t info = P.pr_info[pr];
                      const uint64_t bdesc = bdesc0 + (info & 0xFFFFu);
                      const uint32_t d = tmem_base + ((info >> 16) & 0x7Fu) * kBN;
                      const bool first = kb == 0 && (info >> 24);
#pragma unroll
                      for (int j = 0; j < kKB / kBK; ++j)
                        if (OZMM_MMA_ON) ptx::mma_i8_pair(d, ad0 + 2 * j, bdesc + 2 * j, idesc,
                                         (first && j == 0) ? 0u : 1u);
#pragma unroll
                      for (int j = 0; j < kKB / kBK; ++j)
                        if (OZMM_MMA_ON) ptx::mma_i8_pair(d, ad1 + 2 * j, bdesc + bstep + 2 * j, idesc, 1u);
                    }
                    ptx::mma_commit_pair(a_empty + ai, all_mask);
                    ptx::mma_commit_pair(a_empty + s1, all_mask);
                  }
                  __syncwarp();
                  for (int h = 0; h < 2; ++h)
                    if (++ai == n_a) {
                      ai = 0;
                      aph ^= 1;
                    }
                }
                if (ptx::elect_one()) ptx::mma_commit_pair(b_empty + bi, pair_mask);
                __syncwarp();
                if (++bi == kBBufs) {
                  bi = 0;
                  bph ^= 1;
                }
              }
              continue;
            }
            for (int kb = 0; kb < n_kb; ++kb) {
              OZMM_TWAIT(9, ptx::mbar_wait(b_full + bi, bph));
              ptx::tc_fence_after();
              if (trace && kb == 0 && q == P.b_pass0[b] && b < 2 && lane == 0) trace[2 + 2 * b] = ptx::globaltimer();
              const uint32_t sb = ptx::smem_u32(bbuf + bi * b_buf);
              const uint64_t bdesc0 = ptx::smem_desc(sb, 1024, 2);
              for (int g = g0; g < g1; ++g) {
                if (P.group_pairs > 1 && g + 1 < g1) {
                  // up to group_pairs A stages per barrier round: wait for all, issue
                  // their MMAs in one burst, release all (fewer issue-stream breaks)
                  const int ng = min(P.group_pairs, g1 - g);
                  {
                    int sl = ai;
                    uint32_t ph = aph;
                    for (int h2 = 0; h2 < ng; ++h2) {
                      OZMM_TWAIT(8, ptx::mbar_wait(a_full + sl, ph));
                      if (++sl == n_a) sl = 0, ph ^= 1;
                    }
                  }
                  ptx::tc_fence_after();
                  if (ptx::elect_one()) {
                    int sl = ai;
                    for (int h2 = 0; h2 < ng; ++h2) {
                      const int gg = g + h2;
                      const uint64_t adesc = ptx::smem_desc(ptx::smem_u32(aring + sl * Cfg::kATile), 1024, 2);
                      for (int pr = P.ag_p0[gg]; pr < P.ag_p1[gg]; ++pr) {
                        // one 32-bit word per product (host-packed): B tile offset in
                        // descriptor units | accumulator << 16 | first << 24 -- the
                        // issuing thread was the bottleneck of thin batches
                        const uint32_t info = P.pr_info[pr];
                        const uint64_t bdesc = bdesc0 + (info & 0xFFFFu);
                        const uint32_t d = tmem_base + ((info >> 16) & 0x7Fu) * kBN;
                        const bool first = kb == 0 && (info >> 24);
#pragma unroll
                        for (int j = 0; j < kKB / kBK; ++j)
                          if (OZMM_MMA_ON) ptx::mma_i8_pair(d, adesc + 2 * j, bdesc + 2 * j, idesc,
                                           (first && j == 0) ? 0u : 1u);
                      }
                      if (++sl == n_a) sl = 0;
                    }
                    sl = ai;
                    for (int h2 = 0; h2 < ng; ++h2) {
                      ptx::mma_commit_pair(a_empty + sl, all_mask);
                      if (++sl == n_a) sl = 0;
                    }
                  }
                  __syncwarp();
                  g += ng - 1;
                  for (int h2 = 0; h2 < ng; ++h2)
                    if (++ai == n_a) {
                      ai = 0;
                      aph ^= 1;
                    }
                  continue;
                }
                OZMM_TWAIT(8, ptx::mbar_wait(a_full + ai, aph));
                ptx::tc_fence_after();
                if (ptx::elect_one()) {
                  const uint64_t adesc = ptx::smem_desc(ptx::smem_u32(aring + ai * Cfg::kATile), 1024, 2);
                  for (int pr = P.ag_p0[g]; pr < P.ag_p1[g]; ++pr) {
                    const uint32_t info = P.pr_info[pr];
                    const uint64_t bdesc = bdesc0 + (info & 0xFFFFu);
                    const uint32_t d = tmem_base + ((info >> 16) & 0x7Fu) * kBN;
                    const bool first = kb == 0 && (info >> 24);
#pragma unroll
                    for (int j = 0; j < kKB / kBK; ++j)  // K = 32 per MMA: +32 B = +2 in desc.lo
                      if (OZMM_MMA_ON) ptx::mma_i8_pair(d, adesc + 2 * j, bdesc + 2 * j, idesc,
                                       (first && j == 0) ? 0u : 1u);
#ifdef OZMM_DIAG
                    for (int x = 0; x < P.dup_mma; ++x)  // timing experiment only (wrong results)
                      for (int j = 0; j < kKB / kBK; ++j)
                        if (OZMM_MMA_ON) ptx::mma_i8_pair(d, adesc + 2 * j, bdesc + 2 * j, idesc, 1u);
#endif
                  }
                  ptx::mma_commit_pair(a_empty + ai, all_mask);  // A stage free (all sharers)
                }
                __syncwarp();
                if (++ai == n_a) {
                  ai = 0;
                  aph ^= 1;
                }
              }
              if (ptx::elect_one()) ptx::mma_commit_pair(b_empty + bi, pair_mask);
              __syncwarp();
              if (++bi == kBBufs) {
                bi = 0;
                bph ^= 1;
              }
            }
          }
          if (ptx::elect_one()) ptx::mma_commit_pair(tmem_full, pair_mask);
          __syncwarp();
        }
#ifdef OZMM_DIAG
        if (trace && lane == 0) {
          trace[8] = tw_[8], trace[9] = tw_[9], trace[10] = tw_[10];
          trace[11] = clock64() - t_mma0;
        }
#endif
      }
    }
  } else {
    ptx::setmaxnreg_inc<216>();
    // --------------------------------------------------------- epilogue
    const int quarter = warp & 3;          // TMEM lane quarter
    const int cslice = (warp - 4) >> 2;    // 0/1: which column half
    constexpr int kCols = kBN / 2;         // columns per epilogue warp
    constexpr int kLd = 16;
    const int row = row_base + quarter * 32 + lane;
    const int col0 = col_tile * kBN + cslice * kCols;
    const bool row_ok = row < P.m;
    const double mu = row_ok ? P.mu[row] : 0.0;
    const uint32_t empty_leader = ptx::mapa_shared(tmem_empty, lead_rank);
    double d[kCols];
#pragma unroll
    for (int j = 0; j < kCols; ++j) d[j] = 0.0;
    // fast-flush preconditions (see the chunk loop): group-wise scaling, mu a normal
    // power of two (or 0: a zero row), and this warp's column shifts normal powers of
    // two (or 0), with their exponent range [ec_lo, ec_hi] -- warp-uniform
    const uint32_t mu_hi = static_cast<uint32_t>(__double2hiint(mu));
    const int mu_e = static_cast<int>((mu_hi >> 20) & 0x7FF) - 1023;
    bool fast_ok = P.scale_mode == 0 &&
                   (mu == 0.0 || (mu_e > -1023 && (mu_hi & 0xFFFFF) == 0 && __double2loint(mu) == 0));
    int ec_lo = 4096, ec_hi = -4096;
    for (int j = 0; j < kCols; ++j) {
      const double nu = nu_s[cslice * kCols + j];
      if (nu == 0.0) continue;
      const uint32_t hi = static_cast<uint32_t>(__double2hiint(nu));
      const int e = static_cast<int>((hi >> 20) & 0x7FF) - 1023;
      if (e == -1023 || (hi & 0xFFFFF) != 0 || __double2loint(nu) != 0) fast_ok = false;
      ec_lo = min(ec_lo, e);
      ec_hi = max(ec_hi, e);
    }

    const uint32_t o1 = slice_offset(1, P.beta), os = slice_offset(2, P.beta);  // slice offsets
    // C is read once, after the last MMA: pull this CTA's 128 rows x kBN columns
    // into L2 now, while the MMAs run, so that the final pass waits on L2 rather
    // than HBM (it was 31 us per tile, profiles/r1/tile_trace.txt)
    if (P.c_in != nullptr) {
      constexpr int kLines = kBN * 8 / 128;  // 128-byte lines per row
      for (int i = threadIdx.x - 4 * 32; i < kBM * kLines; i += kPairEpiWarps * 32) {
        const int r = row_base + i / kLines, c = col_tile * kBN + (i % kLines) * 16;
        if (r < P.m && c < P.p)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(P.c_in + static_cast<int64_t>(r) * P.ldc + c));
      }
    }
    // parked chunks (schedule.hpp FlushAct): this CTA's scratch, one SM per CTA
    // (the host enables parking only when the shared memory admits one CTA per SM);
    // layout [slot][column/4][row] of uint4, so a warp's 32 rows are contiguous
    uint4* park = nullptr;
    if (P.park != nullptr) {
      uint32_t smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      if (smid >= 256u) __trap();  // the host sizes the scratch for 256 SM ids (kParkSmIds)
      park = reinterpret_cast<uint4*>(P.park) + static_cast<int64_t>(smid) * kMaxPark * (kBM * kBN / 4);
    }
    const int prow = quarter * 32 + lane;  // this thread's row of the CTA's tile
    for (int b = 0; b < P.nbatch; ++b) {
      const int nc = P.b_nc[b];
      const uint16_t* cid = P.b_cid + b * Cfg::kNAcc;
      if (P.bias) {
        // per-column part of the batch's offset corrections, while its MMAs run:
        // ccol[ci][j] = sum_{(s,t) in chunk} o_s lsb[t][col] + o_s o_t n
        asm volatile("bar.sync 1, %0;" ::"r"(kPairEpiWarps * 32) : "memory");  // previous batch done
        for (int idx = threadIdx.x - 4 * 32; idx < nc * kBN; idx += kPairEpiWarps * 32) {
          const int ci = idx / kBN, j = idx % kBN, c = cid[ci], g = P.c_g[c];
          const int col = col_tile * kBN + j;
          uint32_t acc = 0;
          for (int s = P.c_s[c]; s <= P.c_e[c]; ++s) {
            const int t = g - s;
            const uint32_t oa = s == 1 ? o1 : os, ob = t == 1 ? o1 : os;
            const uint32_t ls = col < P.p ? static_cast<uint32_t>(P.lsb[(t - 1) * P.lsb_plane + col * P.lsb_lstride]) : 0u;
            acc += oa * ls + oa * ob * static_cast<uint32_t>(P.n_inner);
          }
          ccol[ci * kBN + j] = acc;
        }
        asm volatile("bar.sync 1, %0;" ::"r"(kPairEpiWarps * 32) : "memory");
      }
      // per-row part of the offset corrections, sum_{(s,t) in chunk} o_t lsa[s][row],
      // loaded before the wait so the drain does not start with global loads
      uint32_t rrow[Cfg::kNAcc];
#pragma unroll
      for (int ci = 0; ci < Cfg::kNAcc; ++ci) {
        rrow[ci] = 0;
        if (P.bias && row_ok && ci < nc) {
          const int c = cid[ci];
          for (int s = P.c_s[c]; s <= P.c_e[c]; ++s) {
            const int t = P.c_g[c] - s;
            rrow[ci] += (t == 1 ? o1 : os) * static_cast<uint32_t>(P.lsa[(s - 1) * P.lsa_plane + row * P.lsa_lstride]);
          }
        }
      }
      ptx::mbar_wait(tmem_full, b & 1);
      ptx::tc_fence_after();
      if (trace && warp == 4 && lane == 0 && (b == 0 || b == P.nbatch - 1))
        trace[b == 0 ? 12 : 13] = ptx::globaltimer();
#pragma unroll 1
      for (int a = P.b_act0[b]; a < P.b_act1[b]; ++a) {
        // action word: chunk id | kind << 10 | accumulator << 12 | park slot << 16
        const uint32_t act = P.act[a];
        const int c = static_cast<int>(act & 0x3FFu), kind = static_cast<int>((act >> 10) & 3u);
        const int ci = static_cast<int>((act >> 12) & 3u), slot = static_cast<int>(act >> 16);
        const bool from_park = kind == kActUnpark;
        uint32_t rr = 0;
        if (!from_park) {
          rr = rrow[0];
#pragma unroll
          for (int x = 1; x < Cfg::kNAcc; ++x)
            if (ci == x) rr = rrow[x];
        }
        const uint32_t* cc_s = ccol + (from_park ? 0 : ci) * kBN + cslice * kCols;
        const bool corr = P.bias && !from_park;  // parked values are already corrected
        const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + (from_park ? 0 : ci) * kBN +
                               cslice * kCols;
        uint4* pk = park ? park + static_cast<int64_t>(slot) * (kBM * kBN / 4) + (cslice * kCols / 4) * kBM + prow
                         : nullptr;
        if (kind == kActPark) {
          // exact INT32 chunk sums (offset terms removed) to the park slot
#pragma unroll
          for (int cc = 0; cc < kCols; cc += 2 * kLd) {
            uint32_t v0[kLd], v1[kLd];
            ptx::tmem_ld_32x32b<kLd>(taddr + cc, v0);
            ptx::tmem_ld_32x32b<kLd>(taddr + cc + kLd, v1);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int q = 0; q < 2 * kLd; q += 4) {
              uint32_t w[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int j = q + u;
                w[u] = (j < kLd ? v0[j] : v1[j - kLd]) - (corr ? rr + cc_s[cc + j] : 0u);
              }
              pk[((cc + q) / 4) * kBM] = make_uint4(w[0], w[1], w[2], w[3]);
            }
          }
          continue;
        }
        // 32 INT32 sums of this thread's row at columns cc.. (TMEM or park slot)
        auto load32 = [&](int cc, uint32_t (&v0)[kLd], uint32_t (&v1)[kLd]) {
          if (from_park) {
#pragma unroll
            for (int q = 0; q < 2 * kLd; q += 4) {
              const uint4 x = pk[((cc + q) / 4) * kBM];
              uint32_t* dst = q < kLd ? v0 + q : v1 + (q - kLd);
              dst[0] = x.x, dst[1] = x.y, dst[2] = x.z, dst[3] = x.w;
            }
          } else {
            ptx::tmem_ld_32x32b<kLd>(taddr + cc, v0);
            ptx::tmem_ld_32x32b<kLd>(taddr + cc + kLd, v1);
            ptx::tmem_ld_wait();
          }
        };
        // Fast flush (group-wise scaling): ru = mu 2^(2 - beta g) and cv = nu_j are
        // powers of two, so t = fl(fl(ru acc) cv) = acc 2^(Er + Ec) exactly whenever
        // both products stay normal -- the reference's two rounded multiplies are
        // then exact.  acc -> double by the 2^52 + 2^31 bias (one exact subtract),
        // the scale by an add to the exponent field; acc = 0 (also every entry of a
        // zero row or column) contributes +0, which leaves D unchanged (D is never -0).
        const int er = mu_e + 2 - P.beta * P.c_g[c];
        // warp-uniform: tcgen05.ld is .sync.aligned (a row outside the range sends
        // its whole warp down the exact path)
        const bool fast = __all_sync(0xffffffffu, fast_ok && P.dump == nullptr &&
                                                      (mu == 0.0 || (er >= -1022 && er <= 992 && er + ec_lo >= -1022 &&
                                                                     er + ec_hi <= 992)));
        if (fast) {
          const int er20 = er * (1 << 20);
          const uint32_t cc_addr = ptx::smem_u32(cc_s), ec_addr = ptx::smem_u32(ec20 + cslice * kCols);
          // 32 columns per TMEM round trip (two x16 loads, one wait)
#pragma unroll
          for (int cc = 0; cc < kCols; cc += 2 * kLd) {
            uint32_t v0[kLd], v1[kLd];
            load32(cc, v0, v1);
#pragma unroll
            for (int q = 0; q < 2 * kLd; q += 4) {
              const uint4 e4 = ptx::lds_u32x4(ec_addr + 4 * (cc + q));
              const uint4 c4 = corr ? ptx::lds_u32x4(cc_addr + 4 * (cc + q)) : make_uint4(0, 0, 0, 0);
              const uint32_t esh[4] = {e4.x, e4.y, e4.z, e4.w}, cor[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int j = q + u;
                const uint32_t a = (j < kLd ? v0[j] : v1[j - kLd]) - rr - cor[u];  // exact INT32 chunk sum
                const double ad = __dsub_rn(__hiloint2double(0x43300000, static_cast<int>(a ^ 0x80000000u)),
                                            4503601774854144.0);  // == (double)(int32)a, exactly
                const int hi = a != 0u ? __double2hiint(ad) + er20 + static_cast<int>(esh[u]) : 0;
                d[cc + j] = __dadd_rn(d[cc + j], __hiloint2double(hi, __double2loint(ad)));
              }
            }
          }
        } else {
          const double ru = flush_row_scale(P, c, row, mu);
#pragma unroll
          for (int cc = 0; cc < kCols; cc += 2 * kLd) {
            uint32_t v0[kLd], v1[kLd];
            load32(cc, v0, v1);
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              uint32_t* v = hh ? v1 : v0;
              const int c1 = cc + hh * kLd;
              if (corr) {
#pragma unroll
                for (int j = 0; j < kLd; ++j) v[j] -= rr + cc_s[c1 + j];
              }
              if (P.dump != nullptr && row_ok) {
                int32_t* dst = P.dump + (static_cast<int64_t>(c) * P.m + row) * P.p;
#pragma unroll
                for (int j = 0; j < kLd; ++j)
                  if (col0 + c1 + j < P.p) dst[col0 + c1 + j] = static_cast<int32_t>(v[j]);
              }
#pragma unroll
              for (int j = 0; j < kLd; ++j) {
                const double cv = flush_col_scale(P, c, col0 + c1 + j, nu_s[cslice * kCols + c1 + j]);
                const double t =
                    __dmul_rn(__dmul_rn(ru, static_cast<double>(static_cast<int32_t>(v[j]))), cv);
                d[c1 + j] = __dadd_rn(d[c1 + j], t);
              }
            }
          }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive_cluster(empty_leader);
      if (trace && warp == 4 && lane == 0 && (b == 0 || b == P.nbatch - 1))
        trace[b == 0 && P.nbatch > 1 ? 3 : 5] = ptx::globaltimer();
    }

    // C = fl(fl(alpha*D) + fl(beta*C)).  Each thread holds one row of D, so storing
    // (and reading C) straight from registers makes every warp access touch 32
    // rows 128 KB apart: 32 L1 wavefronts per instruction, ~70 us per tile at C3
    // (a fixed cost independent of n, tools/fixed_cost_probe.sh).  D is staged
    // in the operand pool instead -- free now: the tile's last MMA has completed
    // -- and C is read and written row by row with consecutive lanes on
    // consecutive columns.
    constexpr int kStageLd = kBN + 1;  // doubles; the pad spreads a row-per-lane write over banks
    double* stage = reinterpret_cast<double*>(bbuf);  // host sizes the pools >= Cfg::kStageBytes
    const int lrow = quarter * 32 + lane;
#pragma unroll
    for (int j = 0; j < kCols; ++j) stage[lrow * kStageLd + cslice * kCols + j] = d[j];
    asm volatile("bar.sync 1, %0;" ::"r"(kPairEpiWarps * 32) : "memory");
    const int ew = warp - 4;
    const int crow0 = row_base;  // this CTA's first row
    // 4 rows per warp per round, all their C loads issued before any store: C is
    // read and written in place, so a load after a store to the same array
    // would wait for it (the single-row loop ran at ~13 GB/s per SM)
    constexpr int kU = kBN / 32;
    for (int r0 = ew; r0 < kBM; r0 += 4 * kPairEpiWarps) {
      double cv[4][kU];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int grow = crow0 + r0 + i * kPairEpiWarps;
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int col = col_tile * kBN + lane + 32 * u;
          cv[i][u] = (P.c_in && grow < P.m && col < P.p)
                         ? P.c_in[static_cast<int64_t>(grow) * P.ldc + col] : 0.0;
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int rr = r0 + i * kPairEpiWarps, grow = crow0 + rr;
        if (grow >= P.m) continue;
        double* cout = P.c_out + static_cast<int64_t>(grow) * P.ldc;
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int cc = lane + 32 * u, col = col_tile * kBN + cc;
          if (col < P.p)
            cout[col] = __dadd_rn(__dmul_rn(P.alpha, stage[rr * kStageLd + cc]),
                                  P.c_in ? __dmul_rn(P.beta_c, cv[i][u]) : 0.0);
        }
      }
    }
    if (trace && warp == 4 && lane == 0) trace[6] = ptx::globaltimer();
  }

  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_pair<512>(tmem_base);
  }
  if (trace && threadIdx.x == 0) trace[7] = ptx::globaltimer();
}

}  // namespace ozb
