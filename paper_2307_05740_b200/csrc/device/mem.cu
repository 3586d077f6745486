// Device memory for CSF layouts, plans and their decompositions.
//
// Every device allocation of the engine comes from one stream-ordered memory
// pool per device whose release threshold is unbounded: a plan (or CSF)
// destroyed and rebuilt — the end-to-end loop of a solver that re-plans each
// sweep — reuses the pool's mapped pages instead of paying cudaMalloc /
// cudaFree page mapping and the implicit device synchronisation every time
// (measured: 5-110 ms of the TTMc-4 / MTTKRP-4 plan builds before the pool).
// spttn_release_cached() trims the pools back to the driver.
#include <mutex>
#include <string>
#include <vector>
#include <algorithm>

#include "internal.cuh"
#include "../../../include/spttn_b200.h"

namespace spttn_dev {

namespace {

constexpr int kMaxDevices = 64;
std::mutex g_pool_mu;
cudaMemPool_t g_pool[kMaxDevices] = {};

cudaMemPool_t pool_for(int dev) {
  std::lock_guard<std::mutex> lock(g_pool_mu);
  if (dev < 0 || dev >= kMaxDevices) throw Status(SPTTN_ECUDA, "device ordinal out of range");
  if (!g_pool[dev]) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t p = nullptr;
    SPTTN_CUDA(cudaMemPoolCreate(&p, &props));
    uint64_t keep = ~uint64_t{0};
    SPTTN_CUDA(cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &keep));
    g_pool[dev] = p;
  }
  return g_pool[dev];
}

}  // namespace

void dmalloc_raw(void** p, size_t bytes, cudaStream_t s) {
  int dev = 0;
  SPTTN_CUDA(cudaGetDevice(&dev));
  const cudaError_t e = cudaMallocFromPoolAsync(p, bytes ? bytes : 1, pool_for(dev), s);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    throw Status(SPTTN_ENOMEM, "device allocation of " + std::to_string(bytes) + " bytes failed");
  }
  if (e != cudaSuccess)
    throw Status(SPTTN_ECUDA, std::string("cudaMallocFromPoolAsync: ") + cudaGetErrorString(e));
  // kernels rely on cudaMalloc-like alignment (LDG.256 factor rows, int4 headers)
  if (reinterpret_cast<uintptr_t>(*p) % 256 != 0)
    throw Status(SPTTN_ECUDA, "pool allocation is not 256-byte aligned");
}

void dfree(void* p, cudaStream_t s) {
  if (p) cudaFreeAsync(p, s);
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
  std::lock_guard<std::mutex> lock(g_pool_mu);
  for (int d = 0; d < kMaxDevices; ++d)
    if (g_pool[d]) cudaMemPoolTrimTo(g_pool[d], 0);
}

}  // namespace spttn_dev
