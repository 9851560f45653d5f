// hostio.cu -- host <-> device transfer pipeline for the reference-facing
// entry points (the reference's arrays are pageable numpy buffers:
// int64 row offsets / column indices, float64 values, sparse.py:59-71).
//
// A cudaMemcpy from pageable memory runs at a fraction of PCIe speed (the
// driver stages it through a small bounce buffer on one thread).  Here a
// persistent pool of host threads converts each chunk of the caller's array
// straight into a ring of pinned staging slots -- narrowing int64 column
// indices / row offsets to the device's int32 on the way, so only 12 bytes
// per nonzero cross PCIe instead of 16 -- and each full slot is sent with
// cudaMemcpyAsync on the caller's stream while the threads fill the next
// slot.  Downloads run the same ring backwards.  Everything is stream-
// ordered: the calls return once the last chunk is enqueued (uploads) or
// landed in the caller's buffer (downloads).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/pipecg_b200.h"
#include "internal.h"

namespace pcg {
namespace {

// ---------------------------------------------------------------------------
// persistent fork-join pool: run(n_parts, fn) calls fn(part) for every part
// on the workers and the calling thread, returns when all are done
// ---------------------------------------------------------------------------
class Pool {
 public:
  static Pool& get() {
    static Pool p;
    return p;
  }
  int size() const { return (int)workers_.size() + 1; }
  void run(int parts, const std::function<void(int)>& fn) {
    std::unique_lock<std::mutex> lk(mu_);
    fn_ = &fn;
    parts_ = parts;
    next_.store(0);
    pending_ = (int)workers_.size();
    ++gen_;
    cv_.notify_all();
    lk.unlock();
    work();
    lk.lock();
    done_cv_.wait(lk, [&] { return pending_ == 0; });
    fn_ = nullptr;
  }

 private:
  Pool() {
    unsigned hw = std::thread::hardware_concurrency();
    int n = (int)std::min(std::max(hw, 2u), 32u) - 1;
    if (const char* e = getenv("PIPECG_B200_HOST_THREADS")) n = std::max(atoi(e), 1) - 1;
    for (int i = 0; i < n; ++i) workers_.emplace_back([this] { loop(); });
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  void work() {
    for (int p; (p = next_.fetch_add(1)) < parts_;) (*fn_)(p);
  }
  void loop() {
    unsigned long long seen = 0;
    for (;;) {
      std::unique_lock<std::mutex> lk(mu_);
      cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
      if (stop_) return;
      seen = gen_;
      lk.unlock();
      work();
      lk.lock();
      if (--pending_ == 0) done_cv_.notify_all();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* fn_ = nullptr;
  std::atomic<int> next_{0};
  int parts_ = 0, pending_ = 0;
  unsigned long long gen_ = 0;
  bool stop_ = false;
};

// ---------------------------------------------------------------------------
// pinned staging ring (allocated once per process, per device)
// ---------------------------------------------------------------------------
// ring geometry: kSlots slots of slot_bytes (env PIPECG_B200_H2D_SLOT_MB to
// experiment); small slots let the host conversion of chunk k+1 overlap the
// DMA of chunk k even for arrays of a few tens of MB
constexpr int kSlots = 8;

struct Ring {
  char* slot[kSlots] = {};
  cudaEvent_t ev[kSlots] = {};
  size_t slot_bytes = 8u << 20;
  int device = -1;
  std::mutex mu;  // one transfer at a time per process
  int init() {
    int dev = 0;
    cudaGetDevice(&dev);
    if (device == dev) return PCG_OK;
    release();
    if (const char* e = getenv("PIPECG_B200_H2D_SLOT_MB"))
      slot_bytes = (size_t)std::max(1, atoi(e)) << 20;
    for (int s = 0; s < kSlots; ++s) {
      if (cudaHostAlloc(reinterpret_cast<void**>(&slot[s]), slot_bytes, cudaHostAllocPortable) !=
          cudaSuccess)
        return set_error(PCG_ENOMEM, "hostio: pinned staging allocation failed");
      if (cudaEventCreateWithFlags(&ev[s], cudaEventDisableTiming) != cudaSuccess)
        return set_error(PCG_ENOMEM, "hostio: event creation failed");
    }
    device = dev;
    return PCG_OK;
  }
  void release() {
    for (int s = 0; s < kSlots; ++s) {
      if (ev[s]) cudaEventDestroy(ev[s]);
      if (slot[s]) cudaFreeHost(slot[s]);
      ev[s] = nullptr;
      slot[s] = nullptr;
    }
    device = -1;
  }
};

Ring& ring() {
  static Ring r;
  return r;
}

// convert n elements src -> dst (host), in parallel parts; returns true on
// an int64 -> int32 overflow
bool convert(void* dst, const void* src, int64_t n, int kind) {
  Pool& pool = Pool::get();
  const int parts = std::min<int64_t>(pool.size() * 2, std::max<int64_t>(1, n / 16384));
  std::atomic<bool> ovf{false};
  pool.run(parts, [&](int p) {
    const int64_t lo = n * p / parts, hi = n * (p + 1) / parts;
    if (kind == PCG_H2D_I64_TO_I32) {
      const int64_t* s = static_cast<const int64_t*>(src);
      int32_t* d = static_cast<int32_t*>(dst);
      bool bad = false;
      for (int64_t i = lo; i < hi; ++i) {
        const int64_t v = s[i];
        bad |= v < INT32_MIN || v > INT32_MAX;
        d[i] = (int32_t)v;
      }
      if (bad) ovf.store(true);
    } else {
      const size_t es = 8;
      std::memcpy(static_cast<char*>(dst) + lo * es, static_cast<const char*>(src) + lo * es,
                  (hi - lo) * es);
    }
  });
  return ovf.load();
}

}  // namespace

thread_local cudaStream_t t_alloc_stream = nullptr;

AllocStream::AllocStream(cudaStream_t st) : prev(t_alloc_stream) { t_alloc_stream = st; }
AllocStream::~AllocStream() { t_alloc_stream = prev; }

cudaError_t pool_malloc_bytes(void** p, size_t bytes) {
  if (!t_alloc_stream) return cudaMalloc(p, bytes);
  return cudaMallocAsync(p, bytes, t_alloc_stream);
}

void pool_free(void* p) {
  if (!p) return;
  if (t_alloc_stream) cudaFreeAsync(p, t_alloc_stream);
  else cudaFree(p);
}

void pool_init() {
  int dev = 0;
  cudaGetDevice(&dev);
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess) return;
  unsigned long long keep = 2ULL << 30;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  // No hidden cross-stream waits: by default cudaMallocAsync may hand out a
  // block another stream freed with cudaFreeAsync and make the allocating
  // stream WAIT for that stream up to the free.  With several solvers of
  // one process (virtual ranks) such a wait could land behind a peer's spin
  // on this rank's arrival.  Blocks whose free has completed are still
  // reused (opportunistic reuse needs no new dependency).
  int no = 0;
  cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowInternalDependencies, &no);
}

}  // namespace pcg

using namespace pcg;

extern "C" int pipecg_b200_h2d_multi(int n_arrays, void* const* dst_dev,
                                     const void* const* src_host, const int64_t* count,
                                     const int* kind, void* stream) {
  if (n_arrays < 0 || (n_arrays > 0 && (!dst_dev || !src_host || !count || !kind)))
    return set_error(PCG_EINVAL, "h2d: bad arguments");
  for (int a = 0; a < n_arrays; ++a)
    if (count[a] < 0 || (count[a] > 0 && (!dst_dev[a] || !src_host[a])) ||
        (kind[a] != PCG_H2D_COPY64 && kind[a] != PCG_H2D_I64_TO_I32))
      return set_error(PCG_EINVAL, "h2d: bad arguments");
  Ring& R = ring();
  std::lock_guard<std::mutex> lk(R.mu);
  int rc = R.init();
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  // chunks of the arrays taken round-robin: a narrowing chunk is host-bound
  // (~57 GB/s of source) and a copy chunk PCIe-bound (~50 GB/s), so
  // alternating them keeps the host threads and the copy engine busy at
  // the same time instead of one after the other
  std::vector<int64_t> off(n_arrays, 0);
  bool overflow = false;
  int k = 0;
  for (bool more = true; more;) {
    more = false;
    for (int a = 0; a < n_arrays; ++a) {
      if (off[a] >= count[a]) continue;
      const size_t out_es = kind[a] == PCG_H2D_I64_TO_I32 ? 4 : 8;
      const int64_t per_slot = (int64_t)(R.slot_bytes / out_es);
      const int64_t n = std::min(per_slot, count[a] - off[a]);
      const int s = k++ % kSlots;
      cudaError_t e = cudaEventSynchronize(R.ev[s]);  // slot's previous copy has left
      if (e != cudaSuccess) return cuda_status(e, "h2d slot wait");
      overflow |= convert(R.slot[s], static_cast<const char*>(src_host[a]) + off[a] * 8, n, kind[a]);
      e = cudaMemcpyAsync(static_cast<char*>(dst_dev[a]) + off[a] * out_es, R.slot[s], n * out_es,
                          cudaMemcpyHostToDevice, st);
      if (e != cudaSuccess) return cuda_status(e, "h2d copy");
      cudaEventRecord(R.ev[s], st);
      off[a] += n;
      more |= off[a] < count[a];
    }
  }
  return overflow ? set_error(PCG_ERANGE, "h2d: index outside int32 range") : PCG_OK;
}

extern "C" int pipecg_b200_h2d(void* dst_dev, const void* src_host, int64_t count, int kind,
                               void* stream) {
  return pipecg_b200_h2d_multi(1, &dst_dev, &src_host, &count, &kind, stream);
}

extern "C" int pipecg_b200_host_prefault(void* host, int64_t bytes) {
  if (bytes < 0 || (bytes > 0 && !host)) return set_error(PCG_EINVAL, "host_prefault: bad arguments");
  if (bytes == 0) return PCG_OK;
  Ring& R = ring();
  std::lock_guard<std::mutex> lk(R.mu);  // the pool serves one transfer at a time
  Pool& pool = Pool::get();
  constexpr int64_t kPage = 4096;
  const int64_t pages = (bytes + kPage - 1) / kPage;
  const int parts = (int)std::min<int64_t>(pool.size() * 4, std::max<int64_t>(1, pages / 64));
  char* base = static_cast<char*>(host);
  pool.run(parts, [&](int p) {
    const int64_t lo = pages * p / parts, hi = pages * (p + 1) / parts;
    for (int64_t g = lo; g < hi; ++g) reinterpret_cast<volatile char*>(base)[g * kPage] = 0;
  });
  return PCG_OK;
}

extern "C" int pipecg_b200_d2h(void* dst_host, const void* src_dev, int64_t bytes, void* stream) {
  if (bytes < 0 || (bytes > 0 && (!dst_host || !src_dev)) || bytes % 8)
    return set_error(PCG_EINVAL, "d2h: bad arguments");
  if (bytes == 0) return PCG_OK;
  Ring& R = ring();
  std::lock_guard<std::mutex> lk(R.mu);
  int rc = R.init();
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const char* src = static_cast<const char*>(src_dev);
  char* dst = static_cast<char*>(dst_host);
  const int64_t n_chunks = (bytes + R.slot_bytes - 1) / R.slot_bytes;
  // keep up to kSlots chunks in flight; drain each into the caller's buffer
  for (int64_t c = 0; c < n_chunks + kSlots; ++c) {
    if (c < n_chunks) {
      const int s = (int)(c % kSlots);
      const int64_t off = c * (int64_t)R.slot_bytes;
      const int64_t nb = std::min<int64_t>(R.slot_bytes, bytes - off);
      cudaError_t e = cudaEventSynchronize(R.ev[s]);
      if (e != cudaSuccess) return cuda_status(e, "d2h slot wait");
      e = cudaMemcpyAsync(R.slot[s], src + off, nb, cudaMemcpyDeviceToHost, st);
      if (e != cudaSuccess) return cuda_status(e, "d2h copy");
      cudaEventRecord(R.ev[s], st);
    }
    const int64_t d = c - (kSlots - 1);  // chunk to drain now
    if (d >= 0 && d < n_chunks) {
      const int s = (int)(d % kSlots);
      const int64_t off = d * (int64_t)R.slot_bytes;
      const int64_t nb = std::min<int64_t>(R.slot_bytes, bytes - off);
      cudaError_t e = cudaEventSynchronize(R.ev[s]);
      if (e != cudaSuccess) return cuda_status(e, "d2h wait");
      convert(dst + off, R.slot[s], nb / 8, PCG_H2D_COPY64);
    }
  }
  return PCG_OK;
}
