// Stress test of the host entry's copy team (csrc/host_stage.hpp WorkerPool):
// many back-to-back jobs of varying size on a team of threads; every index of
// every job must run exactly once, on the job's own function (a worker that
// wakes late must not run an old job's function on a new job's indices).
// CPU only (no CUDA call is made).
#include <atomic>
#include <cstdio>
#include <vector>

#include "../../paper_2409_13313_b200/csrc/host_stage.hpp"

int main(int argc, char** argv) {
  const int jobs = argc > 1 ? std::atoi(argv[1]) : 20000;
  for (int team : {2, 5, 16}) {
    ozb::WorkerPool pool(team);
    std::vector<std::atomic<int>> hits(64);
    for (int j = 0; j < jobs; ++j) {
      const int n = 1 + (j * 7919) % 40;
      for (int i = 0; i < 64; ++i) hits[i].store(0);
      const int tag = j;
      std::atomic<int> wrong{0};
      pool.run(n, [&, tag](int i) {
        if (tag != j) wrong.fetch_add(1);
        hits[i].fetch_add(1);
      });
      for (int i = 0; i < 64; ++i)
        if (hits[i].load() != (i < n ? 1 : 0) || wrong.load()) {
          std::printf("FAIL team=%d job=%d n=%d index=%d hits=%d wrong=%d\n", team, j, n, i, hits[i].load(),
                      wrong.load());
          return 1;
        }
    }
  }
  std::printf("POOL-OK %d jobs x 3 teams\n", jobs);
  return 0;
}
