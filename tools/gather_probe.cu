// Microbenchmark: throughput of factor-row gathers on B200 for different
// load widths and sources (L1-resident global table vs shared memory).
// Each warp repeatedly gathers random rows of a ROWS x 16-double table;
// WIDTH = bytes per lane per load (8, 16, 32); rows are 128 B, so
// 128/WIDTH lanes share a row and 32*WIDTH/128 rows are read per instruction.
// Build: make probes (-> tools/gather_probe)
#include <cstdio>
#include <cuda_runtime.h>

template <int WIDTH, bool SMEM, bool FRAG = false>
__global__ void k_gather(const double* __restrict__ table, int rows, int iters, double* out, int active) {
  extern __shared__ double sh[];
  const int lane = threadIdx.x & 31;
  constexpr int LPR = 128 / WIDTH;      // lanes per row
  // FRAG: DMMA fragment order — row = lane % 4, 8-byte column = lane / 4
  const int slot = FRAG ? (lane & 3) : lane / LPR;
  const int col = FRAG ? (lane >> 2) : (lane % LPR) * (WIDTH / 8);
  if (SMEM) {
    for (int i = threadIdx.x; i < rows * 16; i += blockDim.x) sh[i] = table[i];
    __syncthreads();
  }
  unsigned x = 12345u + blockIdx.x * 977u + (threadIdx.x >> 5) * 131u + slot * 7u;
  double acc = 0;
  constexpr int U = 8;  // independent loads in flight per warp
  for (int it = 0; it < iters; it += U) {
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      x = x * 1664525u + 1013904223u;
      const int r = (x >> 8) % rows;
      const double* p = (SMEM ? sh : table) + r * 16 + col;
      v[u] = 0;
      if (slot < active) {
        if (WIDTH == 8) {
          v[u] = SMEM ? p[0] : __ldg(p);
        } else if (WIDTH == 16) {
          double2 w;
          if (SMEM) w = *reinterpret_cast<const double2*>(p);
          else asm volatile("ld.global.nc.v2.f64 {%0,%1}, [%2];" : "=d"(w.x), "=d"(w.y) : "l"(p));
          v[u] = w.x + w.y;
        } else {
          double4 w;
          if (SMEM) w = *reinterpret_cast<const double4*>(p);
          else asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                            : "=d"(w.x), "=d"(w.y), "=d"(w.z), "=d"(w.w) : "l"(p));
          v[u] = w.x + w.y + w.z + w.w;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u];
  }
  if (acc == 1234.5) out[0] = acc;
}

template <int WIDTH, bool SMEM, bool FRAG = false>
void run(const double* table, int rows, double* out, int sms, int active = 32) {
  const int iters = 4096, threads = 256, blocks = sms * 4;
  const size_t smem = SMEM ? rows * 16 * sizeof(double) : 0;
  if (SMEM) cudaFuncSetAttribute(k_gather<WIDTH, SMEM, FRAG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_gather<WIDTH, SMEM, FRAG><<<blocks, threads, smem>>>(table, rows, iters, out, active);
  cudaEventRecord(a);
  k_gather<WIDTH, SMEM, FRAG><<<blocks, threads, smem>>>(table, rows, iters, out, active);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const int lpr = FRAG ? 8 : 128 / WIDTH; const int act = active < 32 / lpr ? active : 32 / lpr;
  const double bytes = double(blocks) * threads / 32 * act * lpr * iters * WIDTH;
  printf("%s width %2d B/lane %-6s rows %5d active-rows %2d : %8.2f TB/s  (%.1f B/clk/SM @1.9GHz)  err=%s\n",
         FRAG ? "frag" : "rows", WIDTH,
         SMEM ? "smem" : "global", rows, act, bytes / (ms * 1e-3) / 1e12,
         bytes / (ms * 1e-3) / sms / 1.9e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *table, *out;
  const int maxrows = 1 << 16;
  cudaMalloc(&table, maxrows * 16 * sizeof(double));
  cudaMemset(table, 0, maxrows * 16 * sizeof(double));
  cudaMalloc(&out, 8);
  for (int rows : {1024, 20000}) {
    run<8, false, true>(table, rows, out, sms);
    run<8, true, true>(table, rows < 1024 ? rows : 512, out, sms);
  }
  for (int rows : {256, 1024, 20000}) {
    run<8, false>(table, rows, out, sms);
    run<16, false>(table, rows, out, sms);
    run<32, false>(table, rows, out, sms);
  }
  for (int rows : {256, 512}) {
    run<8, true>(table, rows, out, sms);
    run<16, true>(table, rows, out, sms);
    run<32, true>(table, rows, out, sms);
  }
  for (int rows : {1024, 20000})
    for (int act : {1, 2, 4, 8}) {
      run<16, false>(table, rows, out, sms, act);
      run<32, false>(table, rows, out, sms, act);
    }
  return 0;
}
