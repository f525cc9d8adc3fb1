// Stress test of the host entry's copy team (csrc/host_stage.hpp WorkerPool):
// many back-to-back jobs of varying size on a team of threads; every index of
// every job must run exactly once, on the job's own function (a worker that
// wakes late must not run an old job's function on a new job's indices).
// Also the staging copy loops (copy_screen / copy_patch / copy_stream) against
// plain scalar loops over misaligned starts and odd lengths.
// CPU only (no CUDA call is made).
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <vector>

#include "../../paper_2409_13313_b200/csrc/host_stage.hpp"

static bool same_bits(const double* a, const double* b, size_t n) { return std::memcmp(a, b, 8 * n) == 0; }

static int check_copies() {
  std::vector<double> src(1031), dst(1040), c(1040), want(1040);
  for (size_t i = 0; i < src.size(); ++i) src[i] = std::ldexp(1.0 + 0.37 * i, static_cast<int>(i % 90) - 45) * (i & 1 ? -1 : 1);
  for (size_t off : {0, 1}) {
    for (size_t n : {0, 1, 2, 3, 4, 5, 7, 8, 9, 63, 64, 65, 1000}) {
      // copy_stream: plain copy
      std::fill(dst.begin(), dst.end(), -7.0);
      ozb::copy_stream(dst.data() + off, src.data(), n);
      if (!same_bits(dst.data() + off, src.data(), n) || dst[off + n] != -7.0 || (off && dst[0] != -7.0)) {
        std::printf("FAIL copy_stream off=%zu n=%zu\n", off, n);
        return 1;
      }
      // copy_screen: copy + big-element flag (exponent field >= 1944)
      std::vector<double> s2(src.begin(), src.begin() + std::max<size_t>(n, 1));
      for (int big = 0; big < 2; ++big) {
        if (big && n) s2[n / 2] = std::ldexp(1.0, 950);
        std::fill(dst.begin(), dst.end(), -7.0);
        const uint64_t acc = ozb::copy_screen(dst.data() + off, s2.data(), n);
        if (!same_bits(dst.data() + off, s2.data(), n) || dst[off + n] != -7.0 || ((acc >> 63) != 0) != (big && n)) {
          std::printf("FAIL copy_screen off=%zu n=%zu big=%d\n", off, n, big);
          return 1;
        }
      }
      // copy_patch: c <- res, plus fl(beta * c_old) where c_old is inf / NaN
      for (size_t i = 0; i < n; ++i) c[off + i] = (i % 5 == 3) ? std::numeric_limits<double>::infinity()
                                                 : (i % 7 == 6) ? std::nan("") : 1.5 * i;
      for (size_t i = 0; i < n; ++i) {
        const double co = c[off + i];
        want[i] = std::isfinite(co) ? src[i] : src[i] + 0.5 * co;
      }
      // separate destination first (c is the old C), then in place
      std::fill(dst.begin(), dst.end(), -7.0);
      ozb::copy_patch(dst.data() + off, src.data(), c.data() + off, n, 0.5);
      ozb::copy_patch(c.data() + off, src.data(), c.data() + off, n, 0.5);
      for (size_t i = 0; i < n; ++i) {
        for (const double* got : {dst.data() + off, c.data() + off}) {
          const bool ok = std::isnan(want[i]) ? std::isnan(got[i]) : std::memcmp(&want[i], &got[i], 8) == 0;
          if (!ok) {
            std::printf("FAIL copy_patch off=%zu n=%zu i=%zu\n", off, n, i);
            return 1;
          }
        }
      }
      if (dst[off + n] != -7.0) {
        std::printf("FAIL copy_patch wrote past n (off=%zu n=%zu)\n", off, n);
        return 1;
      }
    }
  }
  std::printf("COPY-OK\n");
  return 0;
}

int main(int argc, char** argv) {
  if (check_copies()) return 1;
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
