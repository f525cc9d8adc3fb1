// Microbenchmark of the host entry's pinned staging (csrc/host_stage.hpp):
// pageable <-> device throughput through the slot rings, per team size and slot
// size, against the driver's own pageable copies and pinned DMA.
//   nvcc -O3 -std=c++17 -Xcompiler -fopenmp -o tools/stage_bench tools/stage_bench.cu
//   tools/stage_bench [GB=2]
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_2409_13313_b200/csrc/host_stage.hpp"

using clk = std::chrono::steady_clock;
static double secs(clk::time_point a) { return std::chrono::duration<double>(clk::now() - a).count(); }

int main(int argc, char** argv) {
  const size_t bytes = size_t((argc > 1 ? atof(argv[1]) : 2.0) * (1 << 30));
  const size_t width = 16384 * 8, rows = bytes / width;  // C3-like rows of 128 KB
  std::vector<char> host(rows * width);
  std::memset(host.data(), 1, host.size());
  void* dev = nullptr;
  cudaMalloc(&dev, rows * width);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  void* pin = nullptr;
  cudaHostAlloc(&pin, rows * width, 0);
  std::memset(pin, 1, rows * width);
  const double gb = rows * width / 1e9;
  for (int rep = 0; rep < 2; ++rep) {
    auto t = clk::now();
    cudaMemcpyAsync(dev, pin, rows * width, cudaMemcpyHostToDevice, s);
    cudaStreamSynchronize(s);
    printf("pinned DMA H2D        %6.1f GB/s\n", gb / secs(t));
    t = clk::now();
    cudaMemcpyAsync(pin, dev, rows * width, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    printf("pinned DMA D2H        %6.1f GB/s\n", gb / secs(t));
    t = clk::now();
    cudaMemcpy2DAsync(pin, width, dev, width, 8192, rows, cudaMemcpyDeviceToHost, s);  // 8 KB row pieces
    cudaStreamSynchronize(s);
    printf("pinned DMA D2H 8KB rows %4.1f GB/s\n", rows * 8192 / 1e9 / secs(t));
    t = clk::now();
    cudaMemcpyAsync(dev, host.data(), rows * width, cudaMemcpyHostToDevice, s);
    cudaStreamSynchronize(s);
    printf("driver pageable H2D   %6.1f GB/s\n", gb / secs(t));
    t = clk::now();
    cudaMemcpyAsync(host.data(), dev, rows * width, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    printf("driver pageable D2H   %6.1f GB/s\n", gb / secs(t));
  }
  for (int nt : {4, 8, 12, 16})
    for (int mb : {4, 8, 16}) {
      ozb::WorkerPool pool(nt);
      ozb::HostStager in, out;
      in.init(size_t(mb) << 20, 2, &pool);
      out.init(size_t(mb) << 20, 2, &pool);
      std::atomic<uint64_t> scr{0};
      double beta = 0.0;
      for (int rep = 0; rep < 2; ++rep) {
        auto t = clk::now();
        in.h2d(dev, width, host.data(), width, width, rows, s);
        cudaStreamSynchronize(s);
        const double h = gb / secs(t);
        t = clk::now();
        in.h2d(dev, width, host.data(), width, width, rows, s, &scr);
        cudaStreamSynchronize(s);
        const double hs = gb / secs(t);
        t = clk::now();
        out.d2h(host.data(), width, dev, width, width, rows, s);
        const double d = gb / secs(t);
        t = clk::now();
        out.d2h(host.data(), width, dev, width, width, rows, s, &beta);
        const double dp = gb / secs(t);
        t = clk::now();
        out.d2h(host.data(), width, dev, width, 8192, rows, s, &beta);
        const double dn = rows * 8192 / 1e9 / secs(t);
        if (rep)
          printf("team %2d slot %2d MB: H2D %5.1f  H2D+screen %5.1f  D2H %5.1f  D2H+patch %5.1f  D2H+patch 8KB rows %5.1f GB/s\n",
                 nt, mb, h, hs, d, dp, dn);
      }
    }
  return 0;
}
