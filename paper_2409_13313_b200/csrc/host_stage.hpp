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
//   H2D  each team thread takes every T-th block: it waits until its slot's
//        previous DMA has drained (the slot's event), copies the block's rows
//        into the slot (host memcpy at DRAM speed), enqueues the DMA slot ->
//        device on the copy stream and records the slot's event.  With two
//        slots per thread, a thread's DMA overlaps its next copy.
//   D2H  each thread DMAs its next blocks into its slots ahead and copies each
//        out as soon as its event fires.
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
  if ((reinterpret_cast<uintptr_t>(dst) & 15) && n > 0) one(i++);
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

// dst <- result (n doubles), where the device wrote fl(alpha d) for beta = 0 and
// C was never uploaded: an old C entry (cin, the caller's C -- dst itself for an
// in-place call) that is inf / NaN still enters the reference's
// fl(fl(alpha d) + fl(beta c)) (scheme.cpp:287), so it is applied here, each old
// entry read before its position of dst is written.
inline void copy_patch(double* dst, const double* res, const double* cin, size_t n, double beta) {
  auto one = [&](size_t i) {
    double v = res[i];
    uint64_t b;
    std::memcpy(&b, cin + i, 8);
    if ((b & kExpMask) == kExpMask) {
      const double z = beta * cin[i];
      v = v + z;
    }
    dst[i] = v;
  };
  size_t i = 0;
#if defined(__SSE2__)
  // 4 entries per step: the exponent test on the high dwords (one compare + one
  // movemask); a group with an inf / NaN entry takes the scalar path
  const __m128i ke = _mm_set1_epi32(0x7FF00000);
  for (; i + 4 <= n; i += 4) {
    const __m128i c0 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(cin + i));
    const __m128i c1 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(cin + i + 2));
    const __m128i e0 = _mm_cmpeq_epi32(_mm_and_si128(c0, ke), ke);
    const __m128i e1 = _mm_cmpeq_epi32(_mm_and_si128(c1, ke), ke);
    if ((_mm_movemask_epi8(_mm_or_si128(e0, e1)) & 0xF0F0) != 0) {
      for (size_t j = i; j < i + 4; ++j) one(j);
      continue;
    }
    _mm_storeu_si128(reinterpret_cast<__m128i*>(dst + i), _mm_loadu_si128(reinterpret_cast<const __m128i*>(res + i)));
    _mm_storeu_si128(reinterpret_cast<__m128i*>(dst + i + 2),
                     _mm_loadu_si128(reinterpret_cast<const __m128i*>(res + i + 2)));
  }
#endif
  for (; i < n; ++i) one(i);
}

// dst <- src (n doubles) with streaming stores: the destination (the caller's C)
// is not read back here, so its lines need not be fetched or kept in cache.
inline void copy_stream(double* dst, const double* src, size_t n) {
  size_t i = 0;
#if defined(__SSE2__)
  if (reinterpret_cast<uintptr_t>(dst) & 15) {
    if (n == 0) return;
    dst[0] = src[0];
    i = 1;
  }
  for (; i + 4 <= n; i += 4) {
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i), _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i)));
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 2),
                     _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 2)));
  }
  _mm_sfence();
#endif
  for (; i < n; ++i) dst[i] = src[i];
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
    work(&fn, n);
    while (left_.load(std::memory_order_acquire) > 0) std::this_thread::yield();
    {
      std::lock_guard<std::mutex> lk(mu_);
      fn_ = nullptr;  // no worker joins this job from here on
    }
    // workers that joined may still be leaving work(): the next job may not reset
    // the shared counters under them
    while (active_.load(std::memory_order_acquire) > 0) std::this_thread::yield();
  }

 private:
  void work(const std::function<void(int)>* fn, int n) {
    for (;;) {
      const int i = next_.fetch_add(1);
      if (i >= n) return;
      (*fn)(i);
      left_.fetch_sub(1, std::memory_order_release);
    }
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(int)>* fn = nullptr;
      int n = 0;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        if (quit_) return;
        if (fn_ == nullptr) continue;  // that job is already over
        fn = fn_;
        n = n_;
        active_.fetch_add(1, std::memory_order_relaxed);
      }
      work(fn, n);
      active_.fetch_sub(1, std::memory_order_release);
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_;
  std::condition_variable cv_;
  uint64_t gen_ = 0;
  bool quit_ = false;
  const std::function<void(int)>* fn_ = nullptr;
  int n_ = 0;
  std::atomic<int> next_{0}, left_{0}, active_{0};
};

// Pinned slots for one copy direction, two per team thread.  A region is cut
// into blocks that fit one slot, dealt round-robin to the team; each thread
// streams ITS blocks through ITS two slots (double buffering), so threads never
// wait for each other per block -- a shared ring with a team barrier per block
// ran at 35-45 GB/s (profiles/r2/stage_bench.txt), the barrier and wake-up cost
// rivalling a block's copy.  All DMAs go to one stream, enqueued from several
// threads (the CUDA runtime serialises the calls); each slot's event guards its
// reuse.
class HostStager {
 public:
  ~HostStager() { release(); }

  cudaError_t init(size_t slot_bytes, int nslots_per_thread, WorkerPool* pool) {
    if (!slot_.empty()) return cudaSuccess;
    pool_ = pool;
    slot_bytes_ = slot_bytes;
    per_thread_ = std::max(2, nslots_per_thread);
    const int n = per_thread_ * pool->size();
    for (int i = 0; i < n; ++i) {
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
  size_t slot_bytes() const { return slot_bytes_; }
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
    const std::vector<Blk> blks = blocks(width, height);
    const int nt = std::min<int>(pool_->size(), static_cast<int>(blks.size()));
    std::atomic<int> err{0};
    pool_->run(nt, [&](int t) {
      int use = 0;
      for (size_t b = t; b < blks.size() && err.load() == 0; b += nt) {
        const Blk& k = blks[b];
        const int j = t * per_thread_ + use;
        use = (use + 1) % per_thread_;
        cudaError_t e = cudaEventSynchronize(ev_[j]);  // the slot's previous DMA has drained
        uint8_t* sl = slot_[j];
        const uint8_t* sp = static_cast<const uint8_t*>(src) + k.r0 * spitch + k.c0;
        if (e == cudaSuccess) {
          uint64_t acc = 0;
          for (size_t r = 0; r < k.nr; ++r) {
            if (screen)
              acc |= copy_screen(reinterpret_cast<double*>(sl + r * k.nc),
                                 reinterpret_cast<const double*>(sp + r * spitch), k.nc / 8);
            else
              std::memcpy(sl + r * k.nc, sp + r * spitch, k.nc);
          }
          fence();
          if (screen && (acc >> 63)) screen->fetch_or(acc);
          e = cudaMemcpy2DAsync(static_cast<uint8_t*>(dst) + k.r0 * dpitch + k.c0, dpitch, sl, k.nc, k.nc, k.nr,
                                cudaMemcpyHostToDevice, s);
        }
        if (e == cudaSuccess) e = cudaEventRecord(ev_[j], s);
        if (e != cudaSuccess) err = static_cast<int>(e);
      }
    });
    return static_cast<cudaError_t>(err.load());
  }

  // dst (pageable host, dpitch) <- src (device, spitch), after the work already
  // enqueued on s.  Returns when every byte has landed in dst.
  // patch_beta != nullptr (double elements, C of a beta = 0 call that was not
  // uploaded): copy_patch against the caller's C at cin (cpitch; dst itself for an
  // in-place call) instead of a plain copy.
  cudaError_t d2h(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height,
                  cudaStream_t s, const double* patch_beta = nullptr, const void* cin = nullptr,
                  size_t cpitch = 0) {
    if (cin == nullptr) cin = dst, cpitch = dpitch;
    const std::vector<Blk> blks = blocks(width, height);
    const int nt = std::min<int>(pool_->size(), static_cast<int>(blks.size()));
    std::atomic<int> err{0};
    pool_->run(nt, [&](int t) {
      // this thread's blocks b = t, t + nt, ...: DMA up to per_thread_ of them
      // ahead into its own slots, copy each out as its event fires
      std::vector<size_t> mine;
      for (size_t b = t; b < blks.size(); b += nt) mine.push_back(b);
      auto issue = [&](size_t i) -> cudaError_t {
        const Blk& k = blks[mine[i]];
        const int j = t * per_thread_ + static_cast<int>(i % per_thread_);
        cudaError_t e = cudaMemcpy2DAsync(slot_[j], k.nc, static_cast<const uint8_t*>(src) + k.r0 * spitch + k.c0,
                                          spitch, k.nc, k.nr, cudaMemcpyDeviceToHost, s);
        return e == cudaSuccess ? cudaEventRecord(ev_[j], s) : e;
      };
      cudaError_t e = cudaSuccess;
      for (size_t i = 0; i < mine.size() && i < static_cast<size_t>(per_thread_) && e == cudaSuccess; ++i) e = issue(i);
      for (size_t i = 0; i < mine.size() && e == cudaSuccess; ++i) {
        const int j = t * per_thread_ + static_cast<int>(i % per_thread_);
        e = cudaEventSynchronize(ev_[j]);
        if (e != cudaSuccess) break;
        const Blk& k = blks[mine[i]];
        uint8_t* d = static_cast<uint8_t*>(dst) + k.r0 * dpitch + k.c0;
        const uint8_t* ci = static_cast<const uint8_t*>(cin) + k.r0 * cpitch + k.c0;
        for (size_t r = 0; r < k.nr; ++r) {
          if (patch_beta)
            copy_patch(reinterpret_cast<double*>(d + r * dpitch),
                       reinterpret_cast<const double*>(slot_[j] + r * k.nc),
                       reinterpret_cast<const double*>(ci + r * cpitch), k.nc / 8, *patch_beta);
          else if (k.nc % 8 == 0)  // streaming stores: 150-157 vs 159-180 ms with plain ones
            copy_stream(reinterpret_cast<double*>(d + r * dpitch),
                        reinterpret_cast<const double*>(slot_[j] + r * k.nc), k.nc / 8);
          else
            std::memcpy(d + r * dpitch, slot_[j] + r * k.nc, k.nc);
        }
        if (i + per_thread_ < mine.size()) e = issue(i + per_thread_);
      }
      if (e != cudaSuccess) err = static_cast<int>(e);
    });
    return static_cast<cudaError_t>(err.load());
  }

 private:
  struct Blk {
    size_t r0, nr, c0, nc;
  };
  // Cuts a height x width-byte region into blocks that fit one slot: whole rows
  // when a row fits, else one row in slot-sized pieces (multiples of 64 bytes).
  std::vector<Blk> blocks(size_t width, size_t height) const {
    std::vector<Blk> out;
    if (width == 0 || height == 0) return out;
    if (width <= slot_bytes_) {
      const size_t rows = std::max<size_t>(1, slot_bytes_ / width);
      for (size_t r0 = 0; r0 < height; r0 += rows) out.push_back({r0, std::min(rows, height - r0), 0, width});
    } else {
      const size_t piece = slot_bytes_ & ~size_t(63);
      for (size_t r0 = 0; r0 < height; ++r0)
        for (size_t c0 = 0; c0 < width; c0 += piece) out.push_back({r0, 1, c0, std::min(piece, width - c0)});
    }
    return out;
  }
  // streaming stores are weakly ordered: drain them before the DMA may read the slot
  static void fence() {
#if defined(__SSE2__)
    _mm_sfence();
#endif
  }

  WorkerPool* pool_ = nullptr;
  size_t slot_bytes_ = 0;
  int per_thread_ = 2;
  std::vector<uint8_t*> slot_;
  std::vector<cudaEvent_t> ev_;
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
