// Microbenchmark: 128-byte row gathers with cp.async.bulk (TMA bulk copy,
// SASS UBLKCP) into shared memory, one row per lane per instruction,
// completion on an mbarrier per stage; compared by bench with LDG gathers
// (tools/gather_probe.cu). Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bulk_probe tools/bulk_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void mbar_init(unsigned long long* m, int count) {
  unsigned a = (unsigned)__cvta_generic_to_shared(m);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count));
}
__device__ __forceinline__ void mbar_expect(unsigned long long* m, int bytes) {
  unsigned a = (unsigned)__cvta_generic_to_shared(m);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, int bytes, unsigned long long* m) {
  unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  unsigned b = (unsigned)__cvta_generic_to_shared(m);
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(d), "l"(src), "r"(bytes), "r"(b) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* m, int phase) {
  unsigned a = (unsigned)__cvta_generic_to_shared(m);
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n"
      ::"r"(a), "r"(phase) : "memory");
}

template <int STAGES>
__global__ void k_bulk(const double* __restrict__ table, int rows, int iters, double* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  double* buf = reinterpret_cast<double*>(smem) + (size_t)warp * STAGES * 32 * 16;
  unsigned long long* bars =
      reinterpret_cast<unsigned long long*>(smem + (size_t)nw * STAGES * 32 * 128) + warp * STAGES;
  if (lane == 0)
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  unsigned x = 12345u + blockIdx.x * 977u + warp * 131u + lane * 7u;
  double acc = 0;
  auto issue = [&](int s) {
    x = x * 1664525u + 1013904223u;
    const int r = (x >> 8) % rows;
    if (lane == 0) mbar_expect(&bars[s], 32 * 128);
    __syncwarp();
    bulk_copy(buf + (s * 32 + lane) * 16, table + (size_t)r * 16, 128, &bars[s]);
  };
  for (int s = 0; s < STAGES; ++s) issue(s);
  for (int it = 0; it < iters; ++it) {
    const int s = it % STAGES;
    mbar_wait(&bars[s], (it / STAGES) & 1);
    // consume: 8 lanes per row, 16 B each (LDS.128), 4 rows per instruction
    for (int q = 0; q < 8; ++q) {
      const double2 v = reinterpret_cast<const double2*>(buf + (s * 32 + q * 4 + (lane >> 3)) * 16)[lane & 7];
      acc += v.x + v.y;
    }
    __syncwarp();
    if (it + STAGES < iters) issue(s);
  }
  if (acc == 1234.5) out[0] = acc;
}

template <int STAGES>
void run(const double* table, int rows, double* out, int sms, int warps) {
  const int iters = 2048, threads = 32 * warps, blocks = sms * 2;
  const size_t smem = (size_t)warps * STAGES * 32 * 128 + warps * STAGES * 8;
  cudaFuncSetAttribute(k_bulk<STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_bulk<STAGES><<<blocks, threads, smem>>>(table, rows, iters, out);
  cudaEventRecord(a);
  k_bulk<STAGES><<<blocks, threads, smem>>>(table, rows, iters, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double bytes = double(blocks) * warps * iters * 32 * 128;
  printf("bulk stages %d warps/blk %2d rows %5d : %8.2f TB/s  %.1f rows/clk/SM  (%s)\n", STAGES,
         warps, rows, bytes / (ms * 1e-3) / 1e12, bytes / 128 / (ms * 1e-3) / sms / 1.9e9,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *table, *out;
  cudaMalloc(&table, (1 << 16) * 16 * sizeof(double));
  cudaMemset(table, 0, (1 << 16) * 16 * sizeof(double));
  cudaMalloc(&out, 8);
  for (int rows : {1024, 20000}) {
    run<2>(table, rows, out, sms, 8);
    run<4>(table, rows, out, sms, 8);
    run<4>(table, rows, out, sms, 4);
    run<8>(table, rows, out, sms, 4);
  }
  return 0;
}
