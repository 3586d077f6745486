// Shared device helpers for the sm_100a SpTTN kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

#include <stdexcept>
#include <string>

namespace spttn_dev {

// Status exception used inside the C-ABI implementation; converted to a
// status code + message at the extern "C" boundary (capi.cu).
struct Status : std::runtime_error {
  int code;
  Status(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define SPTTN_CUDA(call)                                                                 \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      throw ::spttn_dev::Status(4, std::string(#call ": ") + cudaGetErrorString(e_));    \
  } while (0)

constexpr int kWarp = 32;

// Device bounds checks of the bounds-checked build (make debug ->
// lib/debug/libspttn_b200.so, loaded with SPTTN_DEBUG_BOUNDS=1): every factor
// row a kernel gathers, every staged-window index and every output row is
// checked; a violation prints the site and traps the kernel. compute-sanitizer
// is closed on this GPU pool, so this build is the memory-safety check the
// tests run (tests/test_gpu_bounds.py). The product library compiles them out.
#ifdef SPTTN_DEBUG_BOUNDS
#define SPTTN_DCHECK(cond)                                                          \
  do {                                                                              \
    if (!(cond)) {                                                                  \
      printf("SPTTN_DCHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond);          \
      __trap();                                                                     \
    }                                                                               \
  } while (0)
#else
#define SPTTN_DCHECK(cond) \
  do {                     \
  } while (0)
#endif

__device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

__device__ __forceinline__ double4 ld256(const double* p) {
  double4 v;
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
               : "l"(p));
  return v;
}

// Predicated 256-bit load without a branch: the load is issued (or not) in
// straight-line code, so several gathers stay in flight together; inactive
// lanes / iterations read as zero.
// Predicated 256-bit load into existing registers: when pred is false the
// destination keeps its value (no zero fill, no select) — row reuse.
__device__ __forceinline__ void ld256_keep(double4& v, const double* p, bool pred) {
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.b32 q, %5, 0;\n"
      " @q ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];\n}\n"
      : "+d"(v.x), "+d"(v.y), "+d"(v.z), "+d"(v.w)
      : "l"(p), "r"(static_cast<int>(pred)));
}

__device__ __forceinline__ double4 ld256_if(const double* p, bool pred) {
  double4 v;
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.b32 q, %5, 0;\n"
      " mov.b64 %0, 0;\n mov.b64 %1, 0;\n mov.b64 %2, 0;\n mov.b64 %3, 0;\n"
      " @q ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];\n}\n"
      : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
      : "l"(p), "r"(static_cast<int>(pred)));
  return v;
}

__device__ __forceinline__ double2 ld128_if(const double* p, bool pred) {
  double2 v;
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.b32 q, %3, 0;\n mov.b64 %0, 0;\n mov.b64 %1, 0;\n"
      " @q ld.global.nc.v2.f64 {%0,%1}, [%2];\n}\n"
      : "=d"(v.x), "=d"(v.y)
      : "l"(p), "r"(static_cast<int>(pred)));
  return v;
}

__device__ __forceinline__ double2 ld128(const double* p) {
  double2 v;
  asm volatile("ld.global.nc.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

// Ampere-style asynchronous global->shared copies (SASS LDGSTS): the CSF
// streams of a work window are staged into shared memory one window ahead.
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
}
// 16-byte copy through L2 only (does not allocate in L1); bytes beyond
// `src_bytes` are zero-filled.
__device__ __forceinline__ void cp_async16_cg(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(src_bytes)
               : "memory");
}
// 16-byte copy that may allocate in L1 (reused factor rows)
__device__ __forceinline__ void cp_async16_ca(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// TMA bulk copies (cp.async.bulk, SASS UBLKCP) completing on an mbarrier:
// one elected lane stages a whole contiguous stream window into shared
// memory with one instruction per array instead of one LDGSTS per lane and
// element (the per-element form costs ~1 L1 data-pipe wavefront per thread).
__device__ __forceinline__ void mbar_init(uint64_t* m, int count) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(m));
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* m, unsigned bytes) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(m));
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes)
               : "memory");
}
// bytes and both addresses must be multiples of 16
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* m) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(m));
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
      "l"(src), "r"(bytes), "r"(b)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, unsigned parity) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(m));
  asm volatile(
      "{\n .reg .pred p;\n W%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W%=;\n}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
// order this thread's earlier generic-proxy shared-memory accesses before
// later async-proxy (bulk copy) writes to the same buffer
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Warp-collective forms of the TMA issue helpers : every lane
// calls them with the same (shuffle-broadcast, hence provably warp-uniform)
// operands and one elected lane issues, so the operands live in uniform
// registers — the lane-0-only form made the compiler wrap every bulk copy in
// a divergent-operand loop (~240 instructions per staged window).
__device__ __forceinline__ void expect_tx_elect(uint64_t* m, unsigned bytes) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(m));
  asm volatile(
      "{\n .reg .pred p;\n elect.sync _|p, 0xffffffff;\n"
      " @p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n}\n" ::"r"(a),
      "r"(bytes)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s_elect(void* dst, const void* src, unsigned bytes,
                                               uint64_t* m) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(m));
  asm volatile(
      "{\n .reg .pred p;\n elect.sync _|p, 0xffffffff;\n"
      " @p cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n}\n" ::"r"(d),
      "l"(src), "r"(bytes), "r"(b)
      : "memory");
}
__device__ __forceinline__ long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return static_cast<long long>(t);
}
__device__ __forceinline__ int smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return static_cast<int>(r);
}

__device__ __forceinline__ int32_t uni(int32_t v) { return __shfl_sync(0xffffffffu, v, 0); }

__device__ __forceinline__ int ldg_i32(const int32_t* p) { return __ldg(p); }
__device__ __forceinline__ double ldg_f64(const double* p) { return __ldg(p); }

// fp64 tensor-core MMA (SASS: DMMA.8x8x4). Fragment layout, lane L:
//   A (8x4, row-major):  a = A[L/4][L%4]
//   B (4x8, col-major):  b = B[L%4][L/4]
//   C/D (8x8):           d0 = D[L/4][2(L%4)], d1 = D[L/4][2(L%4)+1]
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Row slice of 4 consecutive doubles starting at column c of a row of
// length R; columns >= R read as zero. VEC requires R % 4 == 0 and a
// 32-byte aligned base (checked on the host).
template <bool VEC>
__device__ __forceinline__ double4 row4(const double* row, int c, int R) {
  if (VEC) {
    if (c < R) return ld256(row + c);
    return make_double4(0, 0, 0, 0);
  } else {
    double4 v;
    v.x = c + 0 < R ? __ldg(row + c + 0) : 0.0;
    v.y = c + 1 < R ? __ldg(row + c + 1) : 0.0;
    v.z = c + 2 < R ? __ldg(row + c + 2) : 0.0;
    v.w = c + 3 < R ? __ldg(row + c + 3) : 0.0;
    return v;
  }
}

template <bool VEC>
__device__ __forceinline__ double2 row2(const double* row, int c, int R) {
  if (VEC) {
    if (c < R) return ld128(row + c);
    return make_double2(0, 0);
  } else {
    double2 v;
    v.x = c + 0 < R ? __ldg(row + c + 0) : 0.0;
    v.y = c + 1 < R ? __ldg(row + c + 1) : 0.0;
    return v;
  }
}

// Two consecutive columns c, c+1 of a row of length n (zero beyond n). VEC
// requires n even and a 16-byte aligned base.
template <bool VEC>
__device__ __forceinline__ double2 pair2(const double* row, int c, int n) {
  if (VEC) return c < n ? ld128(row + c) : make_double2(0, 0);
  double2 v;
  v.x = c < n ? __ldg(row + c) : 0.0;
  v.y = c + 1 < n ? __ldg(row + c + 1) : 0.0;
  return v;
}

__device__ __forceinline__ void fma4(double4& acc, double s, const double4& v) {
  acc.x = fma(s, v.x, acc.x);
  acc.y = fma(s, v.y, acc.y);
  acc.z = fma(s, v.z, acc.z);
  acc.w = fma(s, v.w, acc.w);
}

__device__ __forceinline__ void fma4v(double4& acc, const double4& a, const double4& b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.y = fma(a.y, b.y, acc.y);
  acc.z = fma(a.z, b.z, acc.z);
  acc.w = fma(a.w, b.w, acc.w);
}

__device__ __forceinline__ void store4(double* row, int c, int R, const double4& v) {
  if (c + 0 < R) row[c + 0] = v.x;
  if (c + 1 < R) row[c + 1] = v.y;
  if (c + 2 < R) row[c + 2] = v.z;
  if (c + 3 < R) row[c + 3] = v.w;
}


// Programmatic dependent launch (sm_90+): a grid launched with launch_pdl may
// start while the previous kernel in the stream drains; grid_dependency_wait()
// blocks until that kernel has completed and its memory operations are
// visible.
__device__ __forceinline__ void grid_dependency_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
// lets the next grid's CTAs be scheduled once every CTA of this grid has
// started (they still wait for its completion in grid_dependency_wait)
__device__ __forceinline__ void grid_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), unsigned grid, unsigned block, cudaStream_t s,
                       Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

}  // namespace spttn_dev
