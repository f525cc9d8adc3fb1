// Host-side schedule of the ozIMMU_H group-wise accumulation.
//
// 1. Chunks (the reference's flushes, in flush order): for g = 2..k+1 the
//    products s = 1..g-1 (A_s * B_{g-s}) are cut every r products
//    (groupwise_impl, proj/src/scheme.cpp:81-101; flush when q == r or the
//    group ends, :91).  There are w = flush_count_w(k, r) chunks (:109-115).
// 2. Batches: consecutive chunks whose INT32 accumulators are live in TMEM
//    at the same time (n_acc = 512 / tile_n columns each).
// 3. Passes: a batch's products are issued over one or more full sweeps of
//    the inner dimension; each pass loads a contiguous range of A slices and
//    of B slices per K step, sized so a pipeline stage fits the shared-memory
//    budget with >= 3 stages where possible.
//
// The schedule is pure integer bookkeeping; tests/test_host_logic.py checks it
// (through ozmm_debug_schedule) against the reference's chunk boundaries.
#pragma once

#include <algorithm>
#include <cstdint>
#include <vector>

namespace ozb {

struct Chunk {
  int g, s0, s1;  // group and inclusive A-slice range
};

struct Product {
  int ci;     // accumulator slot inside the batch
  int s, t;   // A slice, B slice (1-based), s + t = g
  bool first; // first product issued into this accumulator in the batch
};

struct Pass {
  int batch;
  int alo, ahi, blo, bhi;
  int p0, p1;  // product range [p0, p1)
  int g0, g1;  // A-slice group range [g0, g1) (products sorted by A slice)
};

// Products of one pass that share an A slice (the CTA-pair kernel streams A
// slices one at a time and issues each group when its A tile lands).
struct AGroup {
  int s;
  int p0, p1;
};

struct Batch {
  int c0, nc;        // chunk range
  int pass0, pass1;  // pass range [pass0, pass1)
};

struct Schedule {
  std::vector<Chunk> chunks;
  std::vector<Batch> batches;
  std::vector<Pass> passes;
  std::vector<Product> products;
  std::vector<AGroup> agroups;
  int a_slots = 0, b_slots = 0;  // max slice tiles per stage over passes
};

// ceil(log2 n) via bit width (split.cpp:20-22).
inline int ceil_log2_i64(int64_t n) {
  if (n <= 1) return 0;
  uint64_t v = static_cast<uint64_t>(n) - 1;
  int w = 0;
  while (v) {
    ++w;
    v >>= 1;
  }
  return w;
}

// compute_beta (split.cpp:211-216); returns -1 outside 1..2^29.
inline int compute_beta_host(int64_t n) {
  if (n < 1 || n > (int64_t(1) << 29)) return -1;
  return std::min(7, (31 - ceil_log2_i64(n)) / 2);
}

// compute_r (int_gemm.cpp:253-258); returns -1 on bad arguments.
inline int64_t compute_r_host(int64_t n, int beta) {
  if (n < 1 || beta < 1) return -1;
  const int e = 31 - 2 * beta - ceil_log2_i64(n);
  return e <= 0 ? 1 : (int64_t(1) << e);
}

// flush_count_w (scheme.cpp:109-115).
inline int64_t flush_count_w_host(int k, int64_t r) {
  const int64_t q = (k + r - 1) / r;
  const int64_t f = (k - 1) / r;
  return q * k - (q * f / 2) * r;
}

inline std::vector<Chunk> make_chunks(int k, int64_t r) {
  std::vector<Chunk> out;
  for (int g = 2; g <= k + 1; ++g) {
    int64_t q = 0;
    int s0 = 1;
    for (int s = 1; s <= g - 1; ++s) {
      ++q;
      if (q == r || s == g - 1) {
        out.push_back({g, s0, s});
        q = 0;
        s0 = s + 1;
      }
    }
  }
  return out;
}

// stage_slot_bytes(a, b) must be <= max_stage_bytes for every pass (a single
// product always fits: 1 A tile + 1 B tile).
//
// b_windows > 0 (the CTA-pair kernel, whose A slices stream through a ring and
// only the B slices of a K block are resident): a batch's products are split
// into passes by windows of at most b_windows consecutive B slices, so every
// pass issues all products of its B window and each streamed A tile feeds as
// many products as possible.  Otherwise passes are cut greedily in flush order
// under stage_slot_bytes (the single-CTA kernels stage every slice of a pass).
template <class SlotBytes>
inline Schedule make_schedule(int k, int64_t r, int n_acc, int64_t max_stage_bytes,
                              SlotBytes stage_slot_bytes, int b_windows = 0) {
  Schedule S;
  S.chunks = make_chunks(k, r);
  const int w = static_cast<int>(S.chunks.size());
  for (int c0 = 0; c0 < w; c0 += n_acc) {
    Batch b;
    b.c0 = c0;
    b.nc = std::min(n_acc, w - c0);
    b.pass0 = static_cast<int>(S.passes.size());
    // products of the batch in flush order
    std::vector<Product> prods;
    for (int ci = 0; ci < b.nc; ++ci) {
      const Chunk& c = S.chunks[c0 + ci];
      for (int s = c.s0; s <= c.s1; ++s) prods.push_back({ci, s, c.g - s, false});
    }
    std::vector<bool> seen(b.nc, false);
    if (b_windows > 0) {
      std::stable_sort(prods.begin(), prods.end(),
                       [](const Product& x, const Product& y) { return x.t < y.t; });
    }
    size_t i = 0;
    while (i < prods.size()) {
      Pass ps;
      ps.batch = static_cast<int>(S.batches.size());
      ps.alo = ps.ahi = prods[i].s;
      ps.blo = ps.bhi = prods[i].t;
      size_t j = i;
      while (j < prods.size()) {
        const int alo = std::min(ps.alo, prods[j].s), ahi = std::max(ps.ahi, prods[j].s);
        const int blo = std::min(ps.blo, prods[j].t), bhi = std::max(ps.bhi, prods[j].t);
        if (b_windows > 0) {
          if (bhi - blo + 1 > b_windows) break;
        } else if (j > i && stage_slot_bytes(ahi - alo + 1, bhi - blo + 1) > max_stage_bytes) {
          break;
        }
        ps.alo = alo, ps.ahi = ahi, ps.blo = blo, ps.bhi = bhi;
        ++j;
      }
      // issue order inside the pass: by A slice (integer sums are order-free)
      std::vector<Product> pass_prods(prods.begin() + i, prods.begin() + j);
      std::stable_sort(pass_prods.begin(), pass_prods.end(),
                       [](const Product& x, const Product& y) { return x.s < y.s; });
      ps.p0 = static_cast<int>(S.products.size());
      ps.g0 = static_cast<int>(S.agroups.size());
      for (Product pr : pass_prods) {
        pr.first = !seen[pr.ci];
        seen[pr.ci] = true;
        if (S.agroups.size() == static_cast<size_t>(ps.g0) || S.agroups.back().s != pr.s)
          S.agroups.push_back({pr.s, static_cast<int>(S.products.size()), 0});
        S.products.push_back(pr);
        S.agroups.back().p1 = static_cast<int>(S.products.size());
      }
      ps.p1 = static_cast<int>(S.products.size());
      ps.g1 = static_cast<int>(S.agroups.size());
      S.a_slots = std::max(S.a_slots, ps.ahi - ps.alo + 1);
      S.b_slots = std::max(S.b_slots, ps.bhi - ps.blo + 1);
      S.passes.push_back(ps);
      i = j;
    }
    b.pass1 = static_cast<int>(S.passes.size());
    S.batches.push_back(b);
  }
  return S;
}

}  // namespace ozb
