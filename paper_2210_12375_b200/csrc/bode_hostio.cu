// bode_hostio.cu -- pinned staging arena and parallel host copies for
// bode_solve_host (see bode_hostio.cuh).
#include <algorithm>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include "bode_hostio.cuh"

namespace bode {
namespace hostio {

bool is_pinned(const void* p) {
  if (!p) return false;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();  // clear the sticky-free error of an unknown pointer
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

namespace {

// A fixed team of worker threads; par_copy splits one copy into `workers+1`
// slices (the caller copies one itself) and waits for all of them.
class Team {
 public:
  Team() {
    int n = (int)std::thread::hardware_concurrency();
    if (const char* e = std::getenv("BODE_COPY_THREADS")) n = std::atoi(e);
    n = std::max(1, std::min(n, 16));
    for (int i = 0; i + 1 < n; i++) th_.emplace_back([this, i] { loop(i); });
  }
  ~Team() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  void copy(void* dst, const void* src, size_t bytes) {
    const int parts = (int)th_.size() + 1;
    const size_t kMin = 1 << 20;  // below ~1 MiB a single memcpy wins
    if (parts == 1 || bytes < 2 * kMin) {
      std::memcpy(dst, src, bytes);
      return;
    }
    std::lock_guard<std::mutex> serial(call_);  // one parallel copy at a time
    const size_t slice = ((bytes + parts - 1) / parts + 4095) & ~(size_t)4095;
    {
      std::lock_guard<std::mutex> g(m_);
      dst_ = (char*)dst;
      src_ = (const char*)src;
      bytes_ = bytes;
      slice_ = slice;
      pending_ = (int)th_.size();
      gen_++;
    }
    cv_.notify_all();
    const size_t lo = (size_t)(parts - 1) * slice;  // the caller takes the last slice
    if (lo < bytes) std::memcpy((char*)dst + lo, (const char*)src + lo, bytes - lo);
    std::unique_lock<std::mutex> g(m_);
    done_.wait(g, [this] { return pending_ == 0; });
  }

 private:
  void loop(int i) {
    uint64_t seen = 0;
    for (;;) {
      char* d;
      const char* s;
      size_t b, sl;
      {
        std::unique_lock<std::mutex> g(m_);
        cv_.wait(g, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        d = dst_;
        s = src_;
        b = bytes_;
        sl = slice_;
      }
      const size_t lo = (size_t)i * sl;
      if (lo < b) std::memcpy(d + lo, s + lo, std::min(sl, b - lo));
      {
        std::lock_guard<std::mutex> g(m_);
        if (--pending_ == 0) done_.notify_one();
      }
    }
  }
  std::vector<std::thread> th_;
  std::mutex m_, call_;
  std::condition_variable cv_, done_;
  bool stop_ = false;
  uint64_t gen_ = 0;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t bytes_ = 0, slice_ = 0;
  int pending_ = 0;
};

Team& team() {
  static Team* t = new Team();  // leaked on purpose: no join at static destruction
  return *t;
}

}  // namespace

void par_copy(void* dst, const void* src, size_t bytes) {
  if (bytes) team().copy(dst, src, bytes);
}

cudaError_t Arena::reserve(size_t bytes) {
  if (bytes <= cap) return cudaSuccess;
  if (p) cudaFreeHost(p);
  p = nullptr;
  cap = 0;
  const size_t want = std::max(bytes, (size_t)64 << 20);
  cudaError_t e = cudaHostAlloc((void**)&p, want, cudaHostAllocPortable);
  if (e != cudaSuccess) {
    p = nullptr;
    return e;
  }
  cap = want;
  return cudaSuccess;
}

Arena& arena() {
  static Arena* a = new Arena();
  return *a;
}

}  // namespace hostio
}  // namespace bode
