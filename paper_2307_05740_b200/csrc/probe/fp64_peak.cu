// FP64 throughput probe (roofline denominator). MEASURED_PEAKS.json carries
// only HBM copy bandwidth and bf16 GEMM throughput; the north-star roofline
// for this fp64 path needs the fp64 peaks of the same box, so bench.py
// measures them here: DMMA.8x8x4 (fp64 tensor pipe, what the TTMc kernels
// use) and DFMA (fp64 FMA pipe, what MTTKRP / TTTP use).
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

constexpr int kChains = 8;

__global__ void k_dmma(int iters, double* sink) {
  double d[kChains][2];
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
  for (int c = 0; c < kChains; ++c) d[c][0] = d[c][1] = c * 1e-3;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(d[c][0]), "+d"(d[c][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += d[c][0] + d[c][1];
  if (s == 12345.678) sink[0] = s;
}

__global__ void k_dfma(int iters, double* sink) {
  double d[kChains];
  const double a = 1.0 + threadIdx.x * 1e-12, b = 1e-12;
#pragma unroll
  for (int c = 0; c < kChains; ++c) d[c] = c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) d[c] = fma(d[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += d[c];
  if (s == 12345.678) sink[0] = s;
}

}  // namespace

extern "C" {

// Returns achieved TFLOP/s (2 flops per FMA) of the chosen pipe
// (0 = DMMA, 1 = DFMA), best of `reps` timed launches; <0 on error.
double spttn_probe_fp64_tflops(int pipe, int reps) {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* sink = nullptr;
  cudaMalloc(&sink, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
  const int threads = 256;
  const int blocks = sms * 8;
  double best = 0;
  for (int r = 0; r < reps + 1; ++r) {
    cudaEventRecord(e0);
    if (pipe == 0)
      k_dmma<<<blocks, threads>>>(iters, sink);
    else
      k_dfma<<<blocks, threads>>>(iters, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double warps = static_cast<double>(blocks) * threads / 32;
    const double flops = pipe == 0 ? warps * iters * kChains * (8.0 * 8 * 4 * 2)
                                   : warps * 32 * iters * kChains * 2.0;
    if (r > 0) best = best > flops / (ms * 1e-3) ? best : flops / (ms * 1e-3);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  if (cudaGetLastError() != cudaSuccess) return -2;
  return best / 1e12;
}

}  // extern "C"
