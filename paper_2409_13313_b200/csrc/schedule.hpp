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
#include <utility>
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
  int c0, nc;        // chunk range (consecutive batches; c0 = cids[0] otherwise)
  int pass0, pass1;  // pass range [pass0, pass1)
  std::vector<int> cids;  // the batch's chunks (global ids); accumulator ci holds cids[ci]
  int act0 = 0, act1 = 0;  // its epilogue actions [act0, act1)
};

// Epilogue action after a batch's MMAs (CTA-pair kernel).  The FP64 flushes must
// run in the reference's chunk order (scheme.cpp:91-94); a batch may hold chunks
// whose turn has not come yet: they are PARKED (exact INT32 tile, corrections
// applied, into per-CTA scratch) and flushed from there later.
enum FlushKind { kFlushTmem = 0, kPark = 1, kFlushParked = 2 };
struct FlushAct {
  int kind;
  int c;     // global chunk id
  int ci;    // accumulator (kFlushTmem, kPark)
  int slot;  // park slot (kPark, kFlushParked)
};

struct Schedule {
  std::vector<Chunk> chunks;
  std::vector<Batch> batches;
  std::vector<Pass> passes;
  std::vector<Product> products;
  std::vector<AGroup> agroups;
  std::vector<FlushAct> acts;
  int a_slots = 0, b_slots = 0;  // max slice tiles per stage over passes
  int park_slots = 0;            // park slots the schedule needs (0: chunks consecutive)
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

// Per-K-block cost model of one pass of the CTA-pair kernel, in SM clocks:
// the tensor core needs `prod` per product (4 MMAs of K = 32), and the pass's
// slice tiles must be filled from L2 (`a_tile` / `b_tile` per distinct A / B
// slice).  A pass runs at the slower of the two.  Fitted on B200 (C3 vs C4,
// profiles/r1/configs.csv): an SM fills about 48 B/clk while the GEMM runs.
struct PassCost {
  double prod = 256.0;    // 4 x (M=256, N=128, K=32) MMAs per CTA pair at 8192 MAC/clk/SM
  double a_tile = 341.0;  // 16 KB A tile per CTA
  double b_tile = 171.0;  // 8 KB B tile per CTA
  double batch = 24.0;    // per-batch drain/refill, amortised per K block
  bool greedy = false;    // n_acc chunks per batch, B windows cut every b_windows slices
  bool interleave = false; // A groups in large/small alternation (see make_schedule)
  bool avoid_raw = false;  // no back-to-back products into one accumulator
};

namespace detail {

// Products of a batch (chunks [c0, c0 + nc)) in flush order.
inline std::vector<Product> batch_products(const std::vector<Chunk>& chunks, int c0, int nc) {
  std::vector<Product> prods;
  for (int ci = 0; ci < nc; ++ci) {
    const Chunk& c = chunks[c0 + ci];
    for (int s = c.s0; s <= c.s1; ++s) prods.push_back({ci, s, c.g - s, false});
  }
  return prods;
}

// Products of a batch given by its chunk ids (accumulator ci = position in ids).
inline std::vector<Product> batch_products_ids(const std::vector<Chunk>& chunks, const std::vector<int>& ids) {
  std::vector<Product> prods;
  for (int ci = 0; ci < static_cast<int>(ids.size()); ++ci) {
    const Chunk& c = chunks[ids[ci]];
    for (int s = c.s0; s <= c.s1; ++s) prods.push_back({ci, s, c.g - s, false});
  }
  return prods;
}

inline double pass_cost(const std::vector<Product>& prods, int u, int v, const PassCost& cm) {
  int np = 0, tlo = 1 << 20, thi = -1;
  uint64_t amask[4] = {0, 0, 0, 0};
  for (const Product& p : prods)
    if (p.t >= u && p.t <= v) {
      ++np;
      tlo = std::min(tlo, p.t);
      thi = std::max(thi, p.t);
      amask[p.s >> 6] |= uint64_t(1) << (p.s & 63);
    }
  if (np == 0) return 0.0;
  int na = 0;
  for (uint64_t m : amask) na += __builtin_popcountll(m);
  return std::max(cm.prod * np, cm.a_tile * na + cm.b_tile * (thi - tlo + 1));
}

// Best split of the batch's B-slice range into windows of <= b_windows slices:
// returns the window boundaries [u, v] and the cost.
inline double best_windows(const std::vector<Product>& prods, int b_windows, const PassCost& cm,
                           std::vector<std::pair<int, int>>* out) {
  int blo = 1 << 20, bhi = -1;
  for (const Product& p : prods) blo = std::min(blo, p.t), bhi = std::max(bhi, p.t);
  const int nb = bhi - blo + 1;
  std::vector<double> best(nb + 1, 1e300);
  std::vector<int> from(nb + 1, 0);
  best[0] = 0.0;
  for (int e = 1; e <= nb; ++e)
    for (int b = std::max(0, e - b_windows); b < e; ++b) {
      const double c = best[b] + pass_cost(prods, blo + b, blo + e - 1, cm);
      if (c < best[e] - 1e-9) best[e] = c, from[e] = b;
    }
  if (out) {
    out->clear();
    for (int e = nb; e > 0; e = from[e]) out->push_back({blo + from[e], blo + e - 1});
    std::reverse(out->begin(), out->end());
  }
  return best[nb];
}

}  // namespace detail


namespace detail {

// Batches from chunk-id sets (in execution order): passes, products, A groups,
// and the epilogue actions (flush in chunk order, park what runs ahead).
template <class SlotBytes>
inline void build_batches(Schedule& S, const std::vector<std::vector<int>>& sets, SlotBytes stage_slot_bytes,
                          int64_t max_stage_bytes, int b_windows, const PassCost& cm) {
  const int w = static_cast<int>(S.chunks.size());
  std::vector<char> done(w, 0);
  std::vector<int> park_of(w, -1);
  std::vector<char> slot_busy;
  int next = 0;
  for (const std::vector<int>& ids : sets) {
    Batch b;
    b.cids = ids;
    b.c0 = ids[0];
    b.nc = static_cast<int>(ids.size());
    b.pass0 = static_cast<int>(S.passes.size());
    const std::vector<Product> prods = batch_products_ids(S.chunks, ids);
    std::vector<bool> seen(b.nc, false);
    // the passes, as product subsets
    std::vector<std::vector<Product>> pass_sets;
    if (b_windows > 0) {
      std::vector<std::pair<int, int>> wins;
      if (cm.greedy) {
        int blo = 1 << 20, bhi = -1;
        for (const Product& p : prods) blo = std::min(blo, p.t), bhi = std::max(bhi, p.t);
        for (int u = blo; u <= bhi; u += b_windows) wins.push_back({u, std::min(bhi, u + b_windows - 1)});
      } else {
        detail::best_windows(prods, b_windows, cm, &wins);
      }
      for (const auto& [u, v] : wins) {
        std::vector<Product> ps;
        for (const Product& p : prods)
          if (p.t >= u && p.t <= v) ps.push_back(p);
        if (!ps.empty()) pass_sets.push_back(std::move(ps));
      }
    } else {
      size_t i = 0;
      while (i < prods.size()) {
        int alo = prods[i].s, ahi = alo, blo = prods[i].t, bhi = blo;
        size_t j = i + 1;
        while (j < prods.size()) {
          const int a0 = std::min(alo, prods[j].s), a1 = std::max(ahi, prods[j].s);
          const int b0 = std::min(blo, prods[j].t), b1 = std::max(bhi, prods[j].t);
          if (stage_slot_bytes(a1 - a0 + 1, b1 - b0 + 1) > max_stage_bytes) break;
          alo = a0, ahi = a1, blo = b0, bhi = b1;
          ++j;
        }
        pass_sets.emplace_back(prods.begin() + i, prods.begin() + j);
        i = j;
      }
    }
    for (auto& pass_prods : pass_sets) {
      Pass ps;
      ps.batch = static_cast<int>(S.batches.size());
      ps.alo = ps.ahi = pass_prods[0].s;
      ps.blo = ps.bhi = pass_prods[0].t;
      for (const Product& p : pass_prods) {
        ps.alo = std::min(ps.alo, p.s), ps.ahi = std::max(ps.ahi, p.s);
        ps.blo = std::min(ps.blo, p.t), ps.bhi = std::max(ps.bhi, p.t);
      }
      // issue order inside the pass: grouped by A slice (integer sums are
      // order-free), slices ascending.  Optionally (PassCost::interleave) the
      // groups alternate large and small (8, 1, 7, 2, ...) so the A ring's lead
      // time never drops to a run of one-product stages: measured at C3 it keeps
      // the tensor pipe busier (87.2 vs 85.5 %) but lets the tiles of a wave
      // drift apart, DRAM reads rise 90 -> 162 GB and the capped clock falls --
      // net 4 % slower, so it is off (tools/aorder_ab.sh).
      std::stable_sort(pass_prods.begin(), pass_prods.end(),
                       [](const Product& x, const Product& y) { return x.s < y.s; });
      if (b_windows > 0 && (cm.interleave || cm.avoid_raw)) {
        std::vector<std::vector<Product>> groups;
        for (const Product& p : pass_prods) {
          if (groups.empty() || groups.back()[0].s != p.s) groups.emplace_back();
          groups.back().push_back(p);
        }
        if (cm.interleave) {
          std::stable_sort(groups.begin(), groups.end(),
                           [](const auto& x, const auto& y) { return x.size() > y.size(); });
          std::vector<std::vector<Product>> il;
          for (size_t lo = 0, hi = groups.size(); lo < hi;) {
            il.push_back(groups[lo++]);
            if (lo < hi) il.push_back(groups[--hi]);
          }
          groups.swap(il);
        }
        if (cm.avoid_raw) {
          // no two consecutive products into the same accumulator, also across the
          // wrap to the next K block: rotate a group whose first product would
          // follow one into the same chunk
          for (int sweep = 0; sweep < 2; ++sweep)
            for (size_t i = 0; i < groups.size(); ++i) {
              const auto& prev = groups[(i + groups.size() - 1) % groups.size()];
              auto& gr = groups[i];
              if (groups.size() < 2 && gr.size() < 2) break;
              for (size_t rot = 0; rot < gr.size() && gr[0].ci == prev.back().ci; ++rot)
                std::rotate(gr.begin(), gr.begin() + 1, gr.end());
            }
        }
        pass_prods.clear();
        for (const auto& gr : groups)
          for (const Product& p : gr) pass_prods.push_back(p);
      }
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
    }
    b.pass1 = static_cast<int>(S.passes.size());
    // epilogue actions: flush every chunk whose turn has come (this batch's from
    // TMEM, earlier ones from their park slot), park the rest of this batch
    b.act0 = static_cast<int>(S.acts.size());
    for (int c : ids) done[c] = 1;
    while (next < w && done[next]) {
      int ci = -1;
      for (int x = 0; x < b.nc; ++x)
        if (ids[x] == next) ci = x;
      if (ci >= 0) {
        S.acts.push_back({kFlushTmem, next, ci, -1});
      } else {
        S.acts.push_back({kFlushParked, next, -1, park_of[next]});
        slot_busy[park_of[next]] = 0;
      }
      ++next;
    }
    for (int x = 0; x < b.nc; ++x) {
      const int c = ids[x];
      if (c < next) continue;
      int sl = 0;
      while (sl < static_cast<int>(slot_busy.size()) && slot_busy[sl]) ++sl;
      if (sl == static_cast<int>(slot_busy.size())) slot_busy.push_back(0);
      slot_busy[sl] = 1;
      park_of[c] = sl;
      S.acts.push_back({kPark, c, x, sl});
    }
    S.park_slots = std::max(S.park_slots, static_cast<int>(slot_busy.size()));
    b.act1 = static_cast<int>(S.acts.size());
    S.batches.push_back(b);
  }
}

}  // namespace detail

// stage_slot_bytes(a, b) must be <= max_stage_bytes for every pass (a single
// product always fits: 1 A tile + 1 B tile).
//
// b_windows > 0 (the CTA-pair kernel, whose A slices stream through a ring and
// only the B slices of a K block are resident): batches are cut by dynamic
// programming over the chunk sequence (consecutive chunks, at most n_acc per
// batch, minimising the PassCost model), and each batch's products are split
// into passes by windows of at most b_windows consecutive B slices (again the
// cheapest split), so every streamed A tile feeds as many products as possible
// and no batch degenerates into a fill-bound sweep.  Otherwise batches take
// n_acc chunks in turn and passes are cut greedily in flush order under
// stage_slot_bytes (the single-CTA kernels stage every slice of a pass).
template <class SlotBytes>
inline Schedule make_schedule(int k, int64_t r, int n_acc, int64_t max_stage_bytes,
                              SlotBytes stage_slot_bytes, int b_windows = 0,
                              const PassCost& cm = PassCost{}) {
  Schedule S;
  S.chunks = make_chunks(k, r);
  const int w = static_cast<int>(S.chunks.size());
  // batch boundaries
  std::vector<int> starts;
  if (b_windows > 0 && !cm.greedy) {
    std::vector<double> best(w + 1, 1e300);
    std::vector<int> from(w + 1, 0);
    best[0] = 0.0;
    for (int e = 1; e <= w; ++e)
      for (int b = std::max(0, e - n_acc); b < e; ++b) {
        const auto prods = detail::batch_products(S.chunks, b, e - b);
        const double c = best[b] + cm.batch + detail::best_windows(prods, b_windows, cm, nullptr);
        if (c < best[e] - 1e-9) best[e] = c, from[e] = b;
      }
    for (int e = w; e > 0; e = from[e]) starts.push_back(from[e]);
    std::reverse(starts.begin(), starts.end());
  } else {
    for (int c0 = 0; c0 < w; c0 += n_acc) starts.push_back(c0);
  }
  std::vector<std::vector<int>> sets;
  for (size_t bi = 0; bi < starts.size(); ++bi) {
    const int c0 = starts[bi], c1 = bi + 1 < starts.size() ? starts[bi + 1] : w;
    std::vector<int> ids;
    for (int c = c0; c < c1; ++c) ids.push_back(c);
    sets.push_back(std::move(ids));
  }
  detail::build_batches(S, sets, stage_slot_bytes, max_stage_bytes, b_windows, cm);
  return S;
}

// Modelled cost of a CTA-pair schedule per K block (PassCost units).
inline double schedule_cost(const Schedule& S, const PassCost& cm) {
  double c = 0.0;
  for (const Batch& b : S.batches) {
    c += cm.batch;
    for (int q = b.pass0; q < b.pass1; ++q) {
      const Pass& p = S.passes[q];
      c += std::max(cm.prod * (p.p1 - p.p0), cm.a_tile * (p.g1 - p.g0) + cm.b_tile * (p.bhi - p.blo + 1));
    }
  }
  return c;
}

// CTA-pair schedule over chunks taken in (first A slice, group) order instead of
// flush order.  With small r (C4: r = 2, 20 chunks of <= 2 products) consecutive
// chunks in flush order are the pieces of ONE group -- disjoint A and B slices,
// one product per slice tile -- while chunks at the same position of consecutive
// groups share their A slices and all but one B slice.  Batches are cut by the
// same dynamic programming over this order; chunks computed ahead of their turn
// are parked by the epilogue (Schedule::acts) so the FP64 flushes still run in
// the reference's order (scheme.cpp:91-94).
template <class SlotBytes>
inline Schedule make_schedule_free(int k, int64_t r, int n_acc, int64_t max_stage_bytes,
                                   SlotBytes stage_slot_bytes, int b_windows, const PassCost& cm) {
  Schedule S;
  S.chunks = make_chunks(k, r);
  const int w = static_cast<int>(S.chunks.size());
  std::vector<int> order(w);
  for (int c = 0; c < w; ++c) order[c] = c;
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) {
    return S.chunks[x].s0 != S.chunks[y].s0 ? S.chunks[x].s0 < S.chunks[y].s0 : S.chunks[x].g < S.chunks[y].g;
  });
  std::vector<double> best(w + 1, 1e300);
  std::vector<int> from(w + 1, 0);
  best[0] = 0.0;
  for (int e = 1; e <= w; ++e)
    for (int b = std::max(0, e - n_acc); b < e; ++b) {
      const std::vector<int> ids(order.begin() + b, order.begin() + e);
      const auto prods = detail::batch_products_ids(S.chunks, ids);
      const double c = best[b] + cm.batch + detail::best_windows(prods, b_windows, cm, nullptr);
      if (c < best[e] - 1e-9) best[e] = c, from[e] = b;
    }
  std::vector<std::vector<int>> sets;
  for (int e = w; e > 0; e = from[e]) sets.emplace_back(order.begin() + from[e], order.begin() + e);
  std::reverse(sets.begin(), sets.end());
  detail::build_batches(S, sets, stage_slot_bytes, max_stage_bytes, b_windows, cm);
  return S;
}

}  // namespace ozb
