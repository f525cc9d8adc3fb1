// K2+K3, CTA-pair variant: the same fused ozIMMU_H GEMM as ozimmu_gemm.cuh,
// computed by a 2-CTA cluster with tcgen05 cta_group::2 (UMMA M = 256).
//
// Why: with M = 128 x N = 64 per CTA the tensor core's shared-memory operand
// fetch (A 128x32 B + B 64x32 B per 32-cycle MMA) saturates before the INT8
// datapath (ncu: sm__pipe_tc_cycles_active 83 % at 45 % tensor utilisation,
// profiles/r1/gemm_v1_bn64_*).  In a CTA pair each SM still owns 128 rows of
// the output, but the B operand is split N/2 + N/2 across the two SMs and a
// 256 x kBN x 32 MMA takes kBN/2 cycles: per SM 4 KB + kBN*16 B of operand
// reads per kBN/2 cycles (96 B/cycle at kBN = 128 instead of 192).
//
// Roles per CTA (384 threads): warp 0 = TMA producer (both CTAs load their own
// A rows and their half of the B rows; the bytes are counted on the LEADER's
// full barrier), warp 1 = TMEM allocator (both) + MMA issuer (leader only),
// warps 4..11 = epilogue (each CTA drains its own TMEM: its 128 rows x kBN
// columns, 64 columns per warp).  Commits multicast to both CTAs' barriers;
// the epilogues of both CTAs release the accumulators on the leader's
// tmem_empty barrier.
#pragma once

#include "ozimmu_gemm.cuh"

namespace ozb {

constexpr int kPairThreads = 384;
constexpr int kPairEpiWarps = 8;  // per CTA

template <int kBN>
struct PairCfg {
  static constexpr int kNAcc = 512 / kBN;
  static constexpr int kBHalf = kBN / 2;                  // B rows loaded per CTA
  static constexpr uint32_t kATile = kBM * kBK;           // 4 KB
  static constexpr uint32_t kBTile = kBHalf * kBK;        // bytes per CTA per B slice
  static constexpr uint32_t kIdesc = ptx::idesc_i8(2 * kBM, kBN);
};

template <int kBN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kPairThreads, 1)
    ozimmu_gemm_pair_kernel(const __grid_constant__ CUtensorMap map_a,
                            const __grid_constant__ CUtensorMap map_b,
                            const __grid_constant__ GemmParams P) {
  using Cfg = PairCfg<kBN>;
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
  const uint32_t rank = ptx::cluster_ctarank();
  const bool leader = rank == 0;

  // grouped raster over pair tiles (256 rows x kBN columns)
  const int bid = blockIdx.x >> 1;
  const int per_group = P.group_m * P.tiles_n;
  const int first_m = (bid / per_group) * P.group_m;
  const int gm = min(P.group_m, P.tiles_m - first_m);
  const int tm = first_m + (bid % per_group) % gm;  // pair row-block (256 rows)
  const int tn = (bid % per_group) / gm;
  const int row_base = tm * 2 * kBM + static_cast<int>(rank) * kBM;

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&map_a);
    ptx::tma_prefetch_desc(&map_b);
    for (int s = 0; s < P.stages; ++s) {
      ptx::mbar_init(full + s, 1);
      ptx::mbar_init(empty + s, 1);
    }
    ptx::mbar_init(tmem_full, 1);
    ptx::mbar_init(tmem_empty, 2 * kPairEpiWarps);
    ptx::fence_barrier_init();
  }
  if (warp == 1) ptx::tmem_alloc_pair<512>(tmem_base_smem);
  for (int j = threadIdx.x; j < kBN; j += blockDim.x) {
    const int col = tn * kBN + j;
    nu_s[j] = col < P.p ? P.nu[col] : 0.0;
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();  // barrier inits + TMEM address visible cluster-wide
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_base_smem;

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer
    if (ptx::elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int q = 0; q < P.npass; ++q) {
        const int alo = P.p_alo[q], ahi = P.p_ahi[q], blo = P.p_blo[q], bhi = P.p_bhi[q];
        const uint32_t tx =
            2u * ((ahi - alo + 1) * Cfg::kATile + (bhi - blo + 1) * Cfg::kBTile);
        for (int kb = 0; kb < P.n_kb; ++kb) {
          ptx::mbar_wait(empty + stage, phase ^ 1);
          uint8_t* st = smem + stage * stage_bytes;
          const uint32_t fb = ptx::mapa_shared(full + stage, 0);
          if (leader) ptx::mbar_arrive_expect_tx(full + stage, tx);
          for (int s = alo; s <= ahi; ++s)
            ptx::tma_load_3d_pair(st + (s - alo) * Cfg::kATile, &map_a, fb, kb * kBK, row_base,
                                  s - 1);
          for (int t = blo; t <= bhi; ++t)
            ptx::tma_load_3d_pair(st + a_bytes + (t - blo) * Cfg::kBTile, &map_b, fb, kb * kBK,
                                  tn * kBN + static_cast<int>(rank) * Cfg::kBHalf, t - 1);
          if (++stage == P.stages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------- MMA issuer (leader CTA)
    if (leader) {
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
                ptx::mma_i8_pair(tmem_base + (ci & 0x7Fu) * kBN, adesc, bdesc, Cfg::kIdesc, acc);
              }
              ptx::mma_commit_pair(empty + stage, 0x3);  // free this stage in both CTAs
            }
            __syncwarp();
            if (++stage == P.stages) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
        if (ptx::elect_one()) ptx::mma_commit_pair(tmem_full, 0x3);
        __syncwarp();
      }
    }
  } else if (warp >= 4) {
    // --------------------------------------------------------- epilogue
    const int quarter = warp & 3;          // TMEM lane quarter
    const int cslice = (warp - 4) >> 2;    // 0/1: which 64-column half
    constexpr int kCols = kBN / 2;         // columns per epilogue warp
    constexpr int kLd = 16;
    const int row = row_base + quarter * 32 + lane;
    const int col0 = tn * kBN + cslice * kCols;
    const bool row_ok = row < P.m;
    const double mu = row_ok ? P.mu[row] : 0.0;
    const uint32_t empty_leader = ptx::mapa_shared(tmem_empty, 0);
    double d[kCols];
#pragma unroll
    for (int j = 0; j < kCols; ++j) d[j] = 0.0;

    for (int b = 0; b < P.nbatch; ++b) {
      ptx::mbar_wait(tmem_full, b & 1);
      ptx::tc_fence_after();
      const int c0 = P.b_c0[b], nc = P.b_nc[b];
      for (int ci = 0; ci < nc; ++ci) {
        const int c = c0 + ci;
        const double ru = __dmul_rn(mu, pow2(2 - P.beta * P.c_g[c]));  // ldexp(mu, 2-beta*g)
#pragma unroll
        for (int cc = 0; cc < kCols; cc += kLd) {
          uint32_t v[kLd];
          ptx::tmem_ld_32x32b<kLd>(tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) +
                                       ci * kBN + cslice * kCols + cc,
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
            const double t =
                __dmul_rn(__dmul_rn(ru, static_cast<double>(static_cast<int32_t>(v[j]))),
                          nu_s[cslice * kCols + cc + j]);
            d[cc + j] = __dadd_rn(d[cc + j], t);
          }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive_cluster(empty_leader);
    }

    if (row_ok) {
      const double* cin = P.c_in + static_cast<int64_t>(row) * P.ldc;
      double* cout = P.c_out + static_cast<int64_t>(row) * P.ldc;
#pragma unroll
      for (int j = 0; j < kCols; ++j) {
        const int col = col0 + j;
        if (col < P.p)
          cout[col] = __dadd_rn(__dmul_rn(P.alpha, d[j]), __dmul_rn(P.beta_c, cin[col]));
      }
    }
  }

  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_pair<512>(tmem_base);
  }
}

}  // namespace ozb
