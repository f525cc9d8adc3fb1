// Micro-benchmark of the CTA-pair tcgen05 kind::i8 issue loop (round-2 probe).
//
// One 2-CTA cluster per SM pair (grid 148), operands static in shared memory
// (no TMA), the leader's MMA thread issues R rounds of P products x 4 MMAs
// (M = 256, N = 128, K = 32 each; 64 cycles per MMA at the tcgen05 floor).
// Variants (argv): per-round tcgen05.commit (to a ring of barriers, like the
// A-stage releases of ozimmu_gemm_pair_kernel), per-round mbarrier wait on an
// already-completed barrier, accumulator rotation over 1..8 slots, MMAs per
// accumulator visit.  Prints cycles per MMA (clock64 on the issuing SM).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_2409_13313_b200/csrc tools/mma_bench.cu -o /tmp/mma_bench -lcuda
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>

#include "ptx.cuh"

using namespace ozb;

struct BP {
  int rounds, prods, commit, wait, nacc, run, fill, nbars, bn, mode;
  int copy_kb;        // > 0: warp 2 streams bulk copies of copy_kb KB global -> smem meanwhile
  int copy_sleep_ns;  // pause between copies (rate control)
  const uint8_t* src; // copy source (L2-resident buffer)
  uint32_t info[64];  // per product: B tile offset (desc units) | acc << 16 (mode 1, like pr_info)
};

constexpr int kATile = 128 * 128;  // 16 KB
constexpr int kBTile = 64 * 128;   // 8 KB per CTA

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    mma_bench(BP P, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* aring = smem;                 // 5 A tiles
  uint8_t* bbuf = smem + 5 * kATile;     // 8 B tiles
  uint8_t* cbuf = bbuf + 8 * kBTile;    // 2 x 16 KB copy targets
  uint64_t* bars = reinterpret_cast<uint64_t*>(cbuf + 2 * 16384);  // [0..15] commit ring, 16 ready, 17 final, 18/19 copy
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 20);
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = ptx::cluster_ctarank();
  const bool leader = rank == 0;
  // operand bytes: 0 = zeros, 1 = pseudo-random u8
  for (int i = threadIdx.x; i < (5 * kATile + 8 * kBTile) / 4; i += blockDim.x) {
    uint32_t v = 0;
    if (P.fill) {
      uint32_t x = i * 2654435761u + rank * 97u;
      x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
      v = x;
    }
    reinterpret_cast<uint32_t*>(smem)[i] = v;
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < 20; ++i) ptx::mbar_init(bars + i, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 1) ptx::tmem_alloc_pair<512>(tslot);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem = *tslot;
  if (threadIdx.x == 0) ptx::mbar_arrive(bars + 16);  // "ready" barrier: phase 0 complete
  __syncthreads();
  if (warp == 1 && leader) {
    const uint32_t idesc = ptx::idesc_i8(256, P.bn) & ~((1u << 7) | (1u << 10));  // u8 x u8
    const uint64_t bd0 = ptx::smem_desc(ptx::smem_u32(bbuf), 1024, 2);
    const int per_acc_cols = P.bn;
    unsigned long long t0 = clock64();
    for (int r = 0; r < P.rounds; ++r) {
      if (P.wait) ptx::mbar_wait(bars + 16, 0);
      ptx::tc_fence_after();
      if (P.mode >= 2 && ptx::elect_one()) {
        // compile-time schedule: 8 products, 4 accumulators, 4 MMAs each
        const uint64_t ad = ptx::smem_desc(ptx::smem_u32(aring + (r % 5) * kATile), 1024, 2);
#pragma unroll
        for (int p = 0; p < 8; ++p) {
          // mode 2: new accumulator and new B tile per product; 3: same accumulator,
          // new B; 4: new accumulator, same B
          const uint32_t d = tmem + (P.mode == 3 ? 0 : (p & 3) * 128);
          const uint64_t bd = bd0 + (P.mode == 4 ? 0 : ((p & 7) * kBTile >> 4));
#pragma unroll
          for (int j = 0; j < 4; ++j) ptx::mma_i8_pair(d, ad + 2 * j, bd + 2 * j, idesc, 1u);
        }
        if (P.commit) ptx::mma_commit_pair(bars + (r % 5), 0x3);
      } else if (P.mode == 1 && ptx::elect_one()) {
        // runtime schedule from the parameter space, decoded like the pair kernel
        const uint64_t ad = ptx::smem_desc(ptx::smem_u32(aring + (r % 5) * kATile), 1024, 2);
        for (int p = 0; p < P.prods; ++p) {
          const uint32_t info = P.info[p];
          const uint64_t bd = bd0 + (info & 0xFFFFu);
          const uint32_t d = tmem + ((info >> 16) & 0x7Fu) * 128;
#pragma unroll
          for (int j = 0; j < 4; ++j) ptx::mma_i8_pair(d, ad + 2 * j, bd + 2 * j, idesc, 1u);
        }
        if (P.commit) ptx::mma_commit_pair(bars + (r % 5), 0x3);
      } else if (P.mode == 0 && ptx::elect_one()) {
        const uint64_t ad = ptx::smem_desc(ptx::smem_u32(aring + (r % 5) * kATile), 1024, 2);
        for (int p = 0; p < P.prods; ++p) {
          const uint32_t d = tmem + (p % P.nacc) * per_acc_cols;
          const uint64_t bd = bd0 + ((p % 8) * kBTile >> 4);
          for (int j = 0; j < P.run; ++j)
            ptx::mma_i8_pair(d, ad + 2 * (j & 3), bd + 2 * (j & 3), idesc, (r | p | j) ? 1u : 0u);
        }
        if (P.commit)
          for (int c = 0; c < P.commit; ++c) ptx::mma_commit_pair(bars + ((r * P.commit + c) % P.nbars), 0x3);
      }
      __syncwarp();
    }
    if (ptx::elect_one()) ptx::mma_commit_pair(bars + 17, 0x3);
    __syncwarp();
    ptx::mbar_wait(bars + 17, 0);
    unsigned long long t1 = clock64();
    if (threadIdx.x == 32) out[blockIdx.x / 2] = t1 - t0;
  } else if (warp == 1) {
    ptx::mbar_wait(bars + 17, 0);  // the peer's copy of the final commit
  } else if (warp == 2 && P.copy_kb > 0 && ptx::elect_one()) {
    // concurrent smem fill traffic: bulk copies until the MMA side is done
    const uint32_t bytes = P.copy_kb * 1024u;
    unsigned long long t0 = clock64(), moved = 0;
    for (int i = 0; !ptx::mbar_try_wait(bars + 17, 0); ++i) {
      uint64_t* bar = bars + 18 + (i & 1);
      if (i >= 2) ptx::mbar_wait(bar, ((i >> 1) - 1) & 1);
      ptx::mbar_arrive_expect_tx(bar, bytes);
      const uint8_t* src = P.src + (static_cast<uint64_t>(blockIdx.x * 7 + i) % 64) * 65536;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(ptx::smem_u32(cbuf + (i & 1) * 16384)), "l"(src), "r"(bytes), "r"(ptx::smem_u32(bar)) : "memory");
      moved += bytes;
      if (P.copy_sleep_ns) __nanosleep(P.copy_sleep_ns);
    }
    unsigned long long t1 = clock64();
    out[1024 + blockIdx.x] = (moved << 20) / (t1 - t0 + 1);  // bytes/clk << 20
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_pair<512>(tmem);
  }
}

int main(int argc, char** argv) {
  BP P{2000, 4, 1, 1, 4, 4, 1, 5, 128, 0, 0, 0, nullptr, {}};
  if (argc > 1) P.rounds = atoi(argv[1]);
  if (argc > 2) P.prods = atoi(argv[2]);
  if (argc > 3) P.commit = atoi(argv[3]);
  if (argc > 4) P.wait = atoi(argv[4]);
  if (argc > 5) P.nacc = atoi(argv[5]);
  if (argc > 6) P.run = atoi(argv[6]);
  if (argc > 7) P.fill = atoi(argv[7]);
  if (argc > 8) P.nbars = atoi(argv[8]);
  if (argc > 9) P.bn = atoi(argv[9]);
  int grid = argc > 10 ? atoi(argv[10]) : 148;
  if (argc > 11) P.mode = atoi(argv[11]);
  if (argc > 12) P.copy_kb = atoi(argv[12]);
  if (argc > 13) P.copy_sleep_ns = atoi(argv[13]);
  uint8_t* src;
  cudaMalloc(&src, 64 << 20);
  cudaMemset(src, 0x5a, 64 << 20);
  P.src = src;
  if (P.mode >= 2) P.prods = 8, P.run = 4, P.nacc = 4;
  for (int p = 0; p < 64; ++p) P.info[p] = ((p % 8) * kBTile >> 4) | ((p % P.nacc) << 16);
  const size_t smem = 5 * kATile + 8 * kBTile + 2 * 16384 + 1024 + 256;
  cudaFuncSetAttribute(mma_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  unsigned long long* d;
  cudaMalloc(&d, sizeof(unsigned long long) * 2048);
  cudaMemset(d, 0, sizeof(unsigned long long) * 2048);
  mma_bench<<<grid, 128, smem>>>(P, d);  // warm-up
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mma_bench<<<grid, 128, smem>>>(P, d);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  if (err != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(err));
    return 1;
  }
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  std::vector<unsigned long long> h(grid / 2);
  cudaMemcpy(h.data(), d, sizeof(unsigned long long) * grid / 2, cudaMemcpyDeviceToHost);
  std::sort(h.begin(), h.end());
  std::vector<unsigned long long> hc(grid);
  cudaMemcpy(hc.data(), d + 1024, sizeof(unsigned long long) * grid, cudaMemcpyDeviceToHost);
  double cbw = 0;
  for (auto x : hc) cbw += x / double(1 << 20);
  cbw /= grid;
  const double mmas = double(P.rounds) * P.prods * P.run;
  const double floor_cyc = 256.0 * P.bn / 512.0;  // max(M,128)*N/(256*2)
  printf("mode=%d rounds=%d prods=%d commit=%d wait=%d nacc=%d run=%d fill=%d nbars=%d N=%d grid=%d: "
         "cyc/MMA med %.1f (min %.1f max %.1f) floor %.0f -> eff %.3f | %.3f ms, %.0f TOPS | copy %dKB: %.1f B/clk/SM\n",
         P.mode, P.rounds, P.prods, P.commit, P.wait, P.nacc, P.run, P.fill, P.nbars, P.bn, grid,
         h[h.size() / 2] / mmas, h[0] / mmas, h.back() / mmas, floor_cyc,
         floor_cyc / (h[h.size() / 2] / mmas), ms,
         mmas * (grid / 2) * 256.0 * P.bn * 32 * 2 / (ms * 1e-3) / 1e12, P.copy_kb, cbw);
  return 0;
}
