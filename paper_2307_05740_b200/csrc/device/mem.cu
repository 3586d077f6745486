// Device memory for CSF layouts, plans and their decompositions.
//
// Every device allocation of the engine comes from a caching allocator: each
// block is its own cudaMalloc allocation, and a freed block goes to a
// per-device free list (ordered by size) instead of back to the driver, so a
// plan (or CSF) destroyed and rebuilt — the end-to-end loop of a solver that
// re-plans each sweep — reuses blocks instead of paying cudaMalloc / cudaFree
// page mapping and the implicit device synchronisation every time (measured:
// 5-110 ms of the TTMc-4 / MTTKRP-4 plan builds without caching).
//
// Why not a cudaMemPool (rounds 1-2 used one with an unbounded release
// threshold): once the pool held the freed blocks of a smaller tensor's plans
// it satisfied a larger tensor's requests by re-mapping those fragments, and
// every kernel that streams or gathers from such memory ran slower for the
// rest of the process — TTMc-3 212 -> 322 us after an MTTKRP-3 plan loop in
// the same process (same items, same 24 resident warps per SM, per-item times
// 180 -> 242 us median; plain cudaMalloc blocks: 206 us). A block here is
// always one contiguous driver allocation, reused whole.
//
// Stream order: dfree(p, s) makes the block reusable by work enqueued on `s`
// after the call; a request on another stream first makes that stream wait
// on an event recorded on `s` (lazily, at reuse). Blocks freed by their owner
// after a synchronisation (kStreamIdle, the default) need no ordering. Requests are rounded to
// 512 B (small) or 2 MB (large) and served by the smallest cached block that
// wastes at most a quarter. On an out-of-memory cudaMalloc the cache is
// returned to the driver and the request retried. spttn_release_cached()
// returns the cache to the driver.
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>
#include <algorithm>

#include "internal.cuh"
#include "../../../include/spttn_b200.h"

namespace spttn_dev {

namespace {

constexpr int kMaxDevices = 64;

struct FreeBlock {
  void* ptr;
  cudaStream_t stream;  // reusable in stream order on this stream
};

struct DevCache {
  std::multimap<size_t, FreeBlock> free_by_size;
  std::unordered_map<void*, size_t> live;  // block size of every allocation handed out
};

std::mutex g_mem_mu;
DevCache g_cache[kMaxDevices];

bool no_cache() {
  static const bool off = std::getenv("SPTTN_POOL") && std::atoi(std::getenv("SPTTN_POOL")) == 0;
  return off;
}

size_t round_size(size_t bytes) {
  if (bytes == 0) bytes = 1;
  const size_t g = bytes <= (size_t{1} << 20) ? 512 : (size_t{2} << 20);
  return (bytes + g - 1) / g * g;
}

// caller holds g_mem_mu and has synchronised the device
void drop_cached(DevCache& c) {
  for (auto& kv : c.free_by_size) cudaFree(kv.second.ptr);
  c.free_by_size.clear();
}

}  // namespace

void dmalloc_raw(void** p, size_t bytes, cudaStream_t s) {
  int dev = 0;
  SPTTN_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDevices) throw Status(SPTTN_ECUDA, "device ordinal out of range");
  const size_t want = round_size(bytes);
  if (!no_cache()) {
    FreeBlock hit{nullptr, nullptr};
    size_t hit_size = 0;
    {
      std::lock_guard<std::mutex> lock(g_mem_mu);
      DevCache& c = g_cache[dev];
      const size_t cap = want + want / 4;
      // smallest fitting block; among equal sizes prefer one freed on this stream
      auto it = c.free_by_size.lower_bound(want);
      auto pick = c.free_by_size.end();
      for (auto j = it; j != c.free_by_size.end() && j->first <= cap; ++j) {
        if (pick == c.free_by_size.end()) pick = j;
        if (j->second.stream == s || j->second.stream == kStreamIdle) { pick = j; break; }
        if (j->first != it->first) break;  // only scan the smallest size for a same-stream block
      }
      if (pick != c.free_by_size.end()) {
        hit = pick->second;
        hit_size = pick->first;
        c.free_by_size.erase(pick);
        c.live[hit.ptr] = hit_size;
      }
    }
    if (hit.ptr) {
      if (hit.stream != s && hit.stream != kStreamIdle) {  // order after the old stream's work
        cudaEvent_t ev = nullptr;
        bool ok = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) == cudaSuccess &&
                  cudaEventRecord(ev, hit.stream) == cudaSuccess &&
                  cudaStreamWaitEvent(s, ev, 0) == cudaSuccess;
        if (ev) cudaEventDestroy(ev);
        if (!ok) {  // e.g. the freeing stream no longer exists
          cudaGetLastError();
          cudaDeviceSynchronize();
        }
      }
      *p = hit.ptr;
      return;
    }
  }
  cudaError_t e = cudaMalloc(p, want);
  if (e == cudaErrorMemoryAllocation && !no_cache()) {  // give the cache back and retry
    cudaGetLastError();
    cudaDeviceSynchronize();
    {
      std::lock_guard<std::mutex> lock(g_mem_mu);
      drop_cached(g_cache[dev]);
    }
    e = cudaMalloc(p, want);
  }
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    throw Status(SPTTN_ENOMEM, "device allocation of " + std::to_string(bytes) + " bytes failed");
  }
  if (e != cudaSuccess)
    throw Status(SPTTN_ECUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  // kernels rely on cudaMalloc alignment (LDG.256 factor rows, int4 headers)
  if (reinterpret_cast<uintptr_t>(*p) % 256 != 0)
    throw Status(SPTTN_ECUDA, "device allocation is not 256-byte aligned");
  if (!no_cache()) {
    std::lock_guard<std::mutex> lock(g_mem_mu);
    g_cache[dev].live[*p] = want;
  }
}

void dfree(void* p, cudaStream_t s) {
  if (!p) return;
  if (no_cache()) {
    cudaFree(p);
    return;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) dev = 0;
  std::lock_guard<std::mutex> lock(g_mem_mu);
  // blocks are freed on the device they were allocated on (plans and CSF
  // layouts set their device first); look there, then everywhere
  for (int k = -1; k < kMaxDevices; ++k) {
    DevCache& c = g_cache[k < 0 ? dev : k];
    auto it = c.live.find(p);
    if (it == c.live.end()) continue;
    c.free_by_size.emplace(it->second, FreeBlock{p, s});
    c.live.erase(it);
    return;
  }
  cudaFree(p);  // not one of ours (cannot happen through dmalloc)
}

namespace {
std::mutex g_pin_mu;
std::vector<void*> g_pin_free[40];
unsigned char* g_pin_cur = nullptr;
size_t g_pin_left = 0;

int pin_class(size_t bytes) {
  int c = 8;  // 256 B minimum
  while ((size_t{1} << c) < bytes) ++c;
  return c;
}
}  // namespace

void* pinned_alloc(size_t bytes) {
  const int c = pin_class(bytes);
  const size_t sz = size_t{1} << c;
  std::lock_guard<std::mutex> lock(g_pin_mu);
  if (!g_pin_free[c].empty()) {
    void* p = g_pin_free[c].back();
    g_pin_free[c].pop_back();
    return p;
  }
  if (g_pin_left < sz) {
    const size_t slab = std::max<size_t>(sz, size_t{8} << 20);
    void* p = nullptr;
    SPTTN_CUDA(cudaHostAlloc(&p, slab, cudaHostAllocPortable));
    g_pin_cur = static_cast<unsigned char*>(p);  // the old slab's tail is dropped
    g_pin_left = slab;
  }
  void* p = g_pin_cur;
  g_pin_cur += sz;
  g_pin_left -= sz;
  return p;
}

void pinned_free(void* p, size_t bytes) {
  if (!p) return;
  std::lock_guard<std::mutex> lock(g_pin_mu);
  g_pin_free[pin_class(bytes)].push_back(p);
}

void release_cached() {
  int cur = 0;
  cudaGetDevice(&cur);
  for (int d = 0; d < kMaxDevices; ++d) {
    {
      std::lock_guard<std::mutex> lock(g_mem_mu);
      if (g_cache[d].free_by_size.empty()) continue;
    }
    cudaSetDevice(d);
    cudaDeviceSynchronize();  // cached blocks may still be in use in stream order
    std::lock_guard<std::mutex> lock(g_mem_mu);
    drop_cached(g_cache[d]);
  }
  cudaSetDevice(cur);
}

}  // namespace spttn_dev
