// Pinned staging of PAGEABLE host buffers for the host entry (ozmm_dgemm_host).
//
// The reference's callers hand over ordinary heap memory (Eigen matrices,
// numpy arrays).  cudaMemcpyAsync from pageable memory is carried out by the
// driver through its own small bounce buffer, one thread, synchronously: at
// C3 the drop-in ran at 545 ms per call against 117 ms with pinned buffers
// (BENCH r2 e2e_pageable).  Registering the caller's 6.4 GB per call
// (cudaHostRegister) costs more than the copy itself.  Instead the host entry
// streams each panel through a ring of pinned slots:
//
//   H2D  slot j:  wait until slot j's previous DMA has drained (its event),
//                 copy the block's rows into it with the worker pool (host
//                 memcpy at DRAM speed, several threads), enqueue the DMA
//                 slot -> device on the copy stream, record the slot's event.
//                 The DMA of block j overlaps the host copy of block j+1.
//   D2H  the DMAs of up to `nslots` blocks are enqueued ahead; block j is
//                 copied out of its slot by the pool as soon as its event
//                 fires, then the slot takes block j + nslots.
//
// Pure plumbing: bytes are copied, never interpreted, so results are the
// same as with direct copies (tests/test_gpu_semantics.py checks pinned,
// pageable-staged and driver-copied calls bit for bit).
#pragma once

#include <cuda_runtime.h>
#if defined(__SSE2__)
#include <emmintrin.h>
#endif

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace ozb {

// Exponent-field screen for the range error (split.cpp:124-125): a line max >=
// 2^921 is the only one, so a block whose elements all have an exponent field
// < 1944 cannot raise it.  (x & kExp) + kBigBias carries into bit 63 exactly
// when the field is >= 1944 (inf / NaN included).
constexpr uint64_t kExpMask = 0x7FF0000000000000ull, kBigBias = uint64_t(2048 - 1944) << 52;

// dst <- src (n doubles) and the OR of the screen above, bit 63 = "big element".
// Streaming stores (the slot is read next by the DMA engine, not by this core);
// the caller fences (sfence) before the DMA is enqueued.
inline uint64_t copy_screen(double* dst, const double* src, size_t n) {
  uint64_t acc = 0;
  size_t i = 0;
  auto one = [&](size_t j) {
    uint64_t b;
    std::memcpy(&b, src + j, 8);
    acc |= (b & kExpMask) + kBigBias;
    dst[j] = src[j];
  };
#if defined(__SSE2__)
  if (reinterpret_cast<uintptr_t>(dst) & 15) one(i++);
  __m128i va = _mm_setzero_si128();
  const __m128i ke = _mm_set1_epi64x(static_cast<long long>(kExpMask)),
                kb = _mm_set1_epi64x(static_cast<long long>(kBigBias));
  for (; i + 4 <= n; i += 4) {
    const __m128i v0 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i));
    const __m128i v1 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 2));
    va = _mm_or_si128(va, _mm_add_epi64(_mm_and_si128(v0, ke), kb));
    va = _mm_or_si128(va, _mm_add_epi64(_mm_and_si128(v1, ke), kb));
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i), v0);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 2), v1);
  }
  alignas(16) uint64_t lanes[2];
  _mm_store_si128(reinterpret_cast<__m128i*>(lanes), va);
  acc |= lanes[0] | lanes[1];
#endif
  for (; i < n; ++i) one(i);
  return acc;
}

// C <- result (n doubles), where the device wrote fl(alpha d) for beta = 0 and
// C was never uploaded: an old C entry that is inf / NaN still enters the
// reference's fl(fl(alpha d) + fl(beta c)) (scheme.cpp:287), so it is applied
// here, reading each old entry just before it is overwritten.
inline void copy_patch(double* c, const double* res, size_t n, double beta) {
  for (size_t i = 0; i < n; ++i) {
    double v = res[i];
    uint64_t b;
    std::memcpy(&b, c + i, 8);
    if ((b & kExpMask) == kExpMask) {
      const double z = beta * c[i];
      v = v + z;
    }
    c[i] = v;
  }
}

// Fixed team of worker threads; run(n, fn) executes fn(0..n-1) on the team
// plus the calling thread and returns when every index is done.
class WorkerPool {
 public:
  explicit WorkerPool(int nthreads) {
    for (int t = 1; t < nthreads; ++t) workers_.emplace_back([this] { loop(); });
  }
  ~WorkerPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      quit_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& w : workers_) w.join();
  }
  int size() const { return static_cast<int>(workers_.size()) + 1; }

  void run(int n, const std::function<void(int)>& fn) {
    if (n <= 0) return;
    if (workers_.empty() || n == 1) {
      for (int i = 0; i < n; ++i) fn(i);
      return;
    }
    {
      std::lock_guard<std::mutex> lk(mu_);
      fn_ = &fn;
      n_ = n;
      next_.store(0);
      left_.store(n);
      ++gen_;
    }
    cv_.notify_all();
    work();
    while (left_.load(std::memory_order_acquire) > 0) std::this_thread::yield();
    std::lock_guard<std::mutex> lk(mu_);
    fn_ = nullptr;
  }

 private:
  void work() {
    for (;;) {
      const int i = next_.fetch_add(1);
      if (i >= n_) return;
      (*fn_)(i);
      left_.fetch_sub(1, std::memory_order_release);
    }
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        if (quit_) return;
        if (fn_ == nullptr) continue;
      }
      work();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_;
  std::condition_variable cv_;
  uint64_t gen_ = 0;
  bool quit_ = false;
  const std::function<void(int)>* fn_ = nullptr;
  int n_ = 0;
  std::atomic<int> next_{0}, left_{0};
};

// A ring of pinned slots for one copy direction.
class HostStager {
 public:
  ~HostStager() { release(); }

  cudaError_t init(size_t slot_bytes, int nslots, WorkerPool* pool) {
    if (!slot_.empty()) return cudaSuccess;
    pool_ = pool;
    slot_bytes_ = slot_bytes;
    for (int i = 0; i < nslots; ++i) {
      void* p = nullptr;
      cudaError_t e = cudaHostAlloc(&p, slot_bytes, cudaHostAllocDefault);
      if (e != cudaSuccess) {
        release();
        return e;
      }
      slot_.push_back(static_cast<uint8_t*>(p));
      cudaEvent_t ev;
      e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
      if (e != cudaSuccess) {
        release();
        return e;
      }
      ev_.push_back(ev);
    }
    return cudaSuccess;
  }
  bool ready() const { return !slot_.empty(); }
  void release() {
    for (auto e : ev_) cudaEventDestroy(e);
    for (auto p : slot_) cudaFreeHost(p);
    ev_.clear();
    slot_.clear();
  }

  // dst (device, dpitch) <- src (pageable host, spitch): height rows of width bytes.
  // Returns when every byte has left src (the last DMAs may still be in flight on s).
  // screen != nullptr (double elements): every element is also screened for the
  // range error on its way through (copy_screen), bit 63 of *screen = found.
  cudaError_t h2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height,
                  cudaStream_t s, std::atomic<uint64_t>* screen = nullptr) {
    return for_blocks(width, height, [&](size_t r0, size_t nr, size_t c0, size_t nc) -> cudaError_t {
      const int j = next_;
      next_ = (next_ + 1) % static_cast<int>(slot_.size());
      cudaError_t e = cudaEventSynchronize(ev_[j]);  // the slot's previous DMA has drained
      if (e != cudaSuccess) return e;
      uint8_t* sl = slot_[j];
      const uint8_t* sp = static_cast<const uint8_t*>(src) + r0 * spitch + c0;
      if (screen)
        copy_rows(sl, nc, sp, spitch, nc, nr, [&](uint8_t* d, const uint8_t* x, size_t bytes) {
          const uint64_t a = copy_screen(reinterpret_cast<double*>(d), reinterpret_cast<const double*>(x), bytes / 8);
          if (a >> 63) screen->fetch_or(a);
        });
      else
        copy_rows(sl, nc, sp, spitch, nc, nr);
      e = cudaMemcpy2DAsync(static_cast<uint8_t*>(dst) + r0 * dpitch + c0, dpitch, sl, nc, nc, nr,
                            cudaMemcpyHostToDevice, s);
      if (e != cudaSuccess) return e;
      return cudaEventRecord(ev_[j], s);
    });
  }

  // dst (pageable host, dpitch) <- src (device, spitch), after the work already
  // enqueued on s.  Returns when every byte has landed in dst.
  // patch_beta != nullptr (double elements, C of a beta = 0 call that was not
  // uploaded): copy_patch instead of a plain copy.
  cudaError_t d2h(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height,
                  cudaStream_t s, const double* patch_beta = nullptr) {
    struct Blk {
      size_t r0, nr, c0, nc;
    };
    std::vector<Blk> blks;
    for_blocks(width, height, [&](size_t r0, size_t nr, size_t c0, size_t nc) -> cudaError_t {
      blks.push_back({r0, nr, c0, nc});
      return cudaSuccess;
    });
    const int ns = static_cast<int>(slot_.size());
    auto issue = [&](size_t b) -> cudaError_t {
      const Blk& k = blks[b];
      const int j = static_cast<int>(b % ns);
      cudaError_t e = cudaMemcpy2DAsync(slot_[j], k.nc, static_cast<const uint8_t*>(src) + k.r0 * spitch + k.c0,
                                        spitch, k.nc, k.nr, cudaMemcpyDeviceToHost, s);
      if (e != cudaSuccess) return e;
      return cudaEventRecord(ev_[j], s);
    };
    for (size_t b = 0; b < blks.size() && b < static_cast<size_t>(ns); ++b)
      if (cudaError_t e = issue(b)) return e;
    for (size_t b = 0; b < blks.size(); ++b) {
      const int j = static_cast<int>(b % ns);
      if (cudaError_t e = cudaEventSynchronize(ev_[j])) return e;
      const Blk& k = blks[b];
      uint8_t* d = static_cast<uint8_t*>(dst) + k.r0 * dpitch + k.c0;
      if (patch_beta) {
        const double pb = *patch_beta;
        copy_rows(d, dpitch, slot_[j], k.nc, k.nc, k.nr, [pb](uint8_t* o, const uint8_t* x, size_t bytes) {
          copy_patch(reinterpret_cast<double*>(o), reinterpret_cast<const double*>(x), bytes / 8, pb);
        });
      } else {
        copy_rows(d, dpitch, slot_[j], k.nc, k.nc, k.nr);
      }
      if (b + ns < blks.size())
        if (cudaError_t e = issue(b + ns)) return e;
    }
    next_ = 0;
    return cudaSuccess;
  }

 private:
  // Cuts a height x width-byte region into blocks that fit one slot: whole rows
  // when a row fits, else one row in slot-sized pieces.
  template <class F>
  cudaError_t for_blocks(size_t width, size_t height, F&& f) {
    if (width == 0 || height == 0) return cudaSuccess;
    if (width <= slot_bytes_) {
      const size_t rows = std::max<size_t>(1, slot_bytes_ / width);
      for (size_t r0 = 0; r0 < height; r0 += rows)
        if (cudaError_t e = f(r0, std::min(rows, height - r0), size_t(0), width)) return e;
    } else {
      for (size_t r0 = 0; r0 < height; ++r0)
        for (size_t c0 = 0; c0 < width; c0 += slot_bytes_)
          if (cudaError_t e = f(r0, size_t(1), c0, std::min(slot_bytes_, width - c0))) return e;
    }
    return cudaSuccess;
  }
  // rows x width bytes, split over the pool in pieces of >= 1 MB; `op(dst, src,
  // bytes)` copies one contiguous run (memcpy by default)
  template <class Op>
  void copy_rows(uint8_t* dst, size_t dpitch, const uint8_t* src, size_t spitch, size_t width, size_t rows,
                 Op op) {
    const size_t total = width * rows;
    const int parts = static_cast<int>(std::max<size_t>(
        1, std::min<size_t>(static_cast<size_t>(2 * pool_->size()), total >> 20)));
    if (rows >= static_cast<size_t>(parts)) {
      pool_->run(parts, [&](int t) {
        const size_t i0 = rows * t / parts, i1 = rows * (t + 1) / parts;
        if (dpitch == width && spitch == width) {
          op(dst + i0 * width, src + i0 * width, (i1 - i0) * width);
        } else {
          for (size_t i = i0; i < i1; ++i) op(dst + i * dpitch, src + i * spitch, width);
        }
        fence();
      });
    } else {  // few wide rows: split each row's bytes (8-byte aligned pieces)
      pool_->run(parts, [&](int t) {
        const size_t b0 = (width * t / parts) & ~size_t(63), b1 = t + 1 == parts ? width : (width * (t + 1) / parts) & ~size_t(63);
        for (size_t i = 0; i < rows; ++i) op(dst + i * dpitch + b0, src + i * spitch + b0, b1 - b0);
        fence();
      });
    }
  }
  void copy_rows(uint8_t* dst, size_t dpitch, const uint8_t* src, size_t spitch, size_t width, size_t rows) {
    copy_rows(dst, dpitch, src, spitch, width, rows,
              [](uint8_t* d, const uint8_t* x, size_t bytes) { std::memcpy(d, x, bytes); });
  }
  // streaming stores are weakly ordered: drain them before the DMA may read the slot
  static void fence() {
#if defined(__SSE2__)
    _mm_sfence();
#endif
  }

  WorkerPool* pool_ = nullptr;
  size_t slot_bytes_ = 0;
  std::vector<uint8_t*> slot_;
  std::vector<cudaEvent_t> ev_;
  int next_ = 0;
};

// true when p is ordinary (pageable) host memory; pinned / registered / managed
// memory and device pointers are copied directly
inline bool host_pageable(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    (void)cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

}  // namespace ozb
