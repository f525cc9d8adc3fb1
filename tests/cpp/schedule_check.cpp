// Host check of the CTA-pair schedules (csrc/schedule.hpp), standard and
// free (chunks batched by shared A slices, early ones parked):
//  * every product (s, t) with s + t = g of every chunk appears exactly once,
//    in a batch holding its chunk, inside its pass's slice windows;
//  * the epilogue actions flush every chunk exactly once, in chunk order (the
//    reference's flush order, scheme.cpp:91-94), a parked chunk from the slot it
//    was parked in, and no slot holds two chunks at once;
//  * batches hold at most n_acc chunks, B windows at most 8 slices.
// (Free schedules that need more than kMaxPark = 16 park slots are valid but
// never selected by the host.)
// Prints the modelled cost of both schedules and the park slots for the
// BASELINE configs' (k, r).  CPU only.
#include <cstdio>
#include <cstdlib>
#include <map>
#include <vector>

#include "../../paper_2409_13313_b200/csrc/schedule.hpp"

static int check(const ozb::Schedule& S, int k, long r, const char* what) {
  auto fail = [&](const char* msg) {
    std::printf("FAIL %s k=%d r=%ld: %s\n", what, k, r, msg);
    return 1;
  };
  const int w = static_cast<int>(S.chunks.size());
  std::map<std::pair<int, int>, int> seen;  // (s, t) -> count
  for (size_t bi = 0; bi < S.batches.size(); ++bi) {
    const ozb::Batch& b = S.batches[bi];
    if (b.nc < 1 || b.nc > 4 || static_cast<int>(b.cids.size()) != b.nc) return fail("batch size");
    for (int q = b.pass0; q < b.pass1; ++q) {
      const ozb::Pass& p = S.passes[q];
      if (p.bhi - p.blo + 1 > 8) return fail("B window > 8");
      for (int i = p.p0; i < p.p1; ++i) {
        const ozb::Product& pr = S.products[i];
        if (pr.ci < 0 || pr.ci >= b.nc) return fail("accumulator index");
        const ozb::Chunk& c = S.chunks[b.cids[pr.ci]];
        if (pr.s < c.s0 || pr.s > c.s1 || pr.s + pr.t != c.g) return fail("product outside its chunk");
        if (pr.s < p.alo || pr.s > p.ahi || pr.t < p.blo || pr.t > p.bhi) return fail("product outside its pass");
        ++seen[{pr.s, pr.t}];
      }
    }
  }
  for (int g = 2; g <= k + 1; ++g)
    for (int s = 1; s < g; ++s)
      if (seen[{s, g - s}] != 1) return fail("product missing or repeated");
  if (static_cast<int>(seen.size()) != k * (k + 1) / 2) return fail("extra products");
  int next = 0;
  std::vector<int> slot_of(w, -1), slot_chunk(64, -1);
  std::vector<char> done(w, 0);
  for (size_t bi = 0; bi < S.batches.size(); ++bi) {
    const ozb::Batch& b = S.batches[bi];
    for (int c : b.cids) done[c] = 1;
    for (int a = b.act0; a < b.act1; ++a) {
      const ozb::FlushAct& x = S.acts[a];
      if (x.kind == ozb::kPark) {
        if (x.slot < 0 || x.slot >= S.park_slots || slot_chunk[x.slot] != -1) return fail("park slot busy");
        if (b.cids[x.ci] != x.c) return fail("park of a chunk not in the accumulator");
        slot_chunk[x.slot] = x.c, slot_of[x.c] = x.slot;
      } else {
        if (x.c != next) return fail("flush out of order");
        if (!done[x.c]) return fail("flush before the chunk ran");
        if (x.kind == ozb::kFlushTmem) {
          if (b.cids[x.ci] != x.c) return fail("flush of a chunk not in the accumulator");
        } else {
          if (slot_of[x.c] != x.slot || slot_chunk[x.slot] != x.c) return fail("unpark from the wrong slot");
          slot_chunk[x.slot] = -1;
        }
        ++next;
      }
    }
  }
  if (next != w) return fail("not every chunk flushed");
  return 0;  // (schedules needing more than kMaxPark = 16 slots are not selected)
}

int main() {
  ozb::PassCost cm;
  auto sb = [](int, int b) { return static_cast<long>(b) * 8192; };
  int nfree = 0;
  for (int k = 1; k <= 16; ++k)
    for (long r : {1L, 2L, 3L, 4L, 8L, 16L, 128L}) {
      cm.interleave = cm.avoid_raw = k <= 8;
      const ozb::Schedule S = ozb::make_schedule(k, r, 4, 8L * 8192, sb, 8, cm);
      const ozb::Schedule F = ozb::make_schedule_free(k, r, 4, 8L * 8192, sb, 8, cm);
      if (check(S, k, r, "standard") || check(F, k, r, "free")) return 1;
      if (S.park_slots != 0) {
        std::printf("FAIL standard schedule parks (k=%d r=%ld)\n", k, r);
        return 1;
      }
      if (F.park_slots > 0 && F.park_slots <= 16 && ozb::schedule_cost(F, cm) < 0.995 * ozb::schedule_cost(S, cm))
        ++nfree;
    }
  const int cfg[][2] = {{8, 2}, {8, 8}, {9, 8}, {10, 8}, {12, 8}, {14, 8}, {8, 16}, {14, 16}};
  for (const auto& kr : cfg) {
    cm.interleave = cm.avoid_raw = kr[0] <= 8;
    const ozb::Schedule S = ozb::make_schedule(kr[0], kr[1], 4, 8L * 8192, sb, 8, cm);
    const ozb::Schedule F = ozb::make_schedule_free(kr[0], kr[1], 4, 8L * 8192, sb, 8, cm);
    std::printf("k=%2d r=%3d: standard %zu batches cost %.0f | free %zu batches cost %.0f, %d park slots\n", kr[0],
                kr[1], S.batches.size(), ozb::schedule_cost(S, cm), F.batches.size(), ozb::schedule_cost(F, cm),
                F.park_slots);
  }
  std::printf("SCHEDULE-OK (%d of 112 (k, r) take the free schedule)\n", nfree);
  return 0;
}
