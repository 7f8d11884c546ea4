// Host -> device upload of caller-owned (pageable) host buffers for the
// drop-in entry points: fit_variogram((coords, values)) and
// fill_missing(VolumeGrid(numpy grid)) receive numpy arrays (kriging.py:264,
// :458), which the CUDA driver copies from pageable memory at ~11 GB/s
// (measured on a C4 sub-part: 68 MB grid in 5.8 ms).  Here the bytes go
// through a ring of page-locked staging chunks: host threads copy chunk i + 1
// into its staging buffer while the DMA engine moves chunk i, so the upload
// runs at the smaller of the threads' memcpy rate and the PCIe rate.
//
// Ordering: each chunk's DMA is enqueued on the caller's stream after its
// staging copy; a staging buffer is reused only after the event recorded
// behind its previous DMA has completed.  The call returns once every chunk
// is staged and enqueued, so the caller may reuse or free `src` immediately;
// consumers of `dst` on the same stream see the data in stream order.
#include <cuda_runtime.h>

#include <algorithm>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include <string>

#include "volkrig_b200.h"

namespace vk {
int comm_set_err(int status, const std::string& msg);   // vk_api.cu: the ABI's last-error slot
namespace {

int set_err(int code, const std::string& msg) { return comm_set_err(code, msg); }

#define VK_CUDA(call)                                                             \
  do {                                                                            \
    cudaError_t e_ = (call);                                                      \
    if (e_ != cudaSuccess)                                                        \
      return set_err(VK_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

constexpr size_t CHUNK = (size_t)4 << 20;   // staging chunk
constexpr int NBUF = 4;                      // chunks in flight

// fixed pool of memcpy workers: job() copies [lo, hi) of the current chunk
class CopyPool {
 public:
  explicit CopyPool(int n) {
    for (int i = 0; i < n; ++i) th_.emplace_back([this, i] { loop(i); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> l(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  int size() const { return (int)th_.size() + 1; }
  // copies n bytes src -> dst with the workers plus the calling thread
  void copy(char* dst, const char* src, size_t n) {
    const int parts = size();
    const size_t step = ((n + parts - 1) / parts + 63) & ~(size_t)63;
    {
      std::lock_guard<std::mutex> l(mu_);
      dst_ = dst;
      src_ = src;
      n_ = n;
      step_ = step;
      pending_ = (int)th_.size();
      ++gen_;
    }
    cv_.notify_all();
    slice(0);
    std::unique_lock<std::mutex> l(mu_);
    done_.wait(l, [this] { return pending_ == 0; });
  }

 private:
  void slice(int i) {
    const size_t lo = std::min(n_, (size_t)i * step_), hi = std::min(n_, lo + step_);
    if (hi > lo) std::memcpy(dst_ + lo, src_ + lo, hi - lo);
  }
  void loop(int i) {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> l(mu_);
        cv_.wait(l, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_) return;
      }
      slice(i + 1);
      {
        std::lock_guard<std::mutex> l(mu_);
        if (--pending_ == 0) done_.notify_one();
      }
    }
  }
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_, done_;
  uint64_t gen_ = 0;
  bool stop_ = false;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t n_ = 0, step_ = 0;
  int pending_ = 0;
};

struct Stager {
  std::mutex mu;                       // one upload at a time
  char* buf[NBUF] = {};
  cudaEvent_t ev[NBUF] = {};
  int device = -1;
  CopyPool* pool = nullptr;
  uint64_t next = 0;
};

Stager& stager() {
  static Stager s;
  return s;
}

int host_threads() {
  if (const char* e = std::getenv("VK_UPLOAD_THREADS")) return std::max(1, std::atoi(e));
  const int hw = (int)std::max(1u, std::thread::hardware_concurrency());
  return std::min(8, hw);
}

}  // namespace
}  // namespace vk

using namespace vk;

extern "C" int vk_copy_h2d(void* dst, const void* src, int64_t bytes, void* stream) {
  if (bytes < 0 || (bytes > 0 && (!dst || !src))) return set_err(VK_E_INVALID_ARGUMENT, "null argument");
  if (bytes == 0) return VK_OK;
  cudaStream_t st = (cudaStream_t)stream;
  Stager& s = stager();
  std::lock_guard<std::mutex> lock(s.mu);
  int dev = 0;
  VK_CUDA(cudaGetDevice(&dev));
  if (s.device != dev) {                 // staging belongs to one device context
    for (int i = 0; i < NBUF; ++i) {
      if (s.ev[i]) { cudaEventSynchronize(s.ev[i]); cudaEventDestroy(s.ev[i]); s.ev[i] = nullptr; }
      if (s.buf[i]) { cudaFreeHost(s.buf[i]); s.buf[i] = nullptr; }
    }
    for (int i = 0; i < NBUF; ++i) {
      VK_CUDA(cudaHostAlloc((void**)&s.buf[i], CHUNK, cudaHostAllocPortable));
      VK_CUDA(cudaEventCreateWithFlags(&s.ev[i], cudaEventDisableTiming));
    }
    s.device = dev;
  }
  if (!s.pool) s.pool = new CopyPool(host_threads() - 1);   // lives for the process
  // small uploads: one pageable copy is cheaper than the staging hand-off
  if (bytes < (int64_t)(1 << 20)) {
    VK_CUDA(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyHostToDevice, st));
    return VK_OK;
  }
  const char* in = static_cast<const char*>(src);
  char* out = static_cast<char*>(dst);
  for (int64_t off = 0; off < bytes; off += (int64_t)CHUNK) {
    const int b = (int)(s.next++ % NBUF);
    const size_t n = (size_t)std::min<int64_t>((int64_t)CHUNK, bytes - off);
    VK_CUDA(cudaEventSynchronize(s.ev[b]));          // previous DMA from this buffer done
    s.pool->copy(s.buf[b], in + off, n);
    VK_CUDA(cudaMemcpyAsync(out + off, s.buf[b], n, cudaMemcpyHostToDevice, st));
    VK_CUDA(cudaEventRecord(s.ev[b], st));
  }
  return VK_OK;
}
