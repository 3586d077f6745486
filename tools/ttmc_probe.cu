// Synthetic upper bound for the TTMc-3 packed kernel: per "group" each warp
// issues NV packed 256-bit gathers of Zipf(1.1)-distributed rows of a
// 20000 x 16 fp64 table (V) plus one packed gather of sequential rows (U),
// then 4 xor-16 shuffles and 8 DMMA — no CSF stream, no slice logic.
// Measures how long 627k groups take on the whole GPU.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ttmc_probe tools/ttmc_probe.cu
#include <cmath>
#include <cstdio>
#include <cuda_runtime.h>
#include <vector>

__device__ __forceinline__ double4 ld256(const double* p) {
  double4 v;
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int NV>
__global__ void __launch_bounds__(256, 3) k(const double* V, const double* U, const int* zipf,
                                           int nz, int groups_per_warp, double* out) {
  const int lane = threadIdx.x & 31;
  const int slot = (lane >> 4) * 4 + (lane & 3), c4 = (lane >> 2) & 3, ch = lane >> 4;
  const int w = (blockIdx.x * 256 + threadIdx.x) >> 5;
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  unsigned x = 7919u * w + 13u * slot;
  int ju = (w * 97) % 20000;
  for (int g = 0; g < groups_per_warp; ++g) {
    int kk[NV];
#pragma unroll
    for (int it = 0; it < NV; ++it) {
      x = x * 1664525u + 1013904223u;
      kk[it] = zipf[(x >> 8) % nz];
    }
    const double4 ur = ld256(U + (size_t)((ju + slot) % 20000) * 16 + 4 * c4);
    ju = (ju + 8) % 20000;
    double4 xv = make_double4(0, 0, 0, 0);
#pragma unroll
    for (int it = 0; it < NV; ++it) {
      const double4 v = ld256(V + (size_t)kk[it] * 16 + 4 * c4);
      xv.x += v.x; xv.y += v.y; xv.z += v.z; xv.w += v.w;
    }
    const double r0 = __shfl_xor_sync(~0u, ch ? xv.x : xv.z, 16);
    const double r1 = __shfl_xor_sync(~0u, ch ? xv.y : xv.w, 16);
    const double s0 = __shfl_xor_sync(~0u, ch ? ur.x : ur.z, 16);
    const double s1 = __shfl_xor_sync(~0u, ch ? ur.y : ur.w, 16);
    dmma(acc[0], acc[1], ur.x, xv.x);
    dmma(acc[2], acc[3], ur.y, xv.y);
    dmma(acc[4], acc[5], s0, r0);
    dmma(acc[6], acc[7], s1, r1);
    dmma(acc[0], acc[1], ur.z, xv.z);
    dmma(acc[2], acc[3], ur.w, xv.w);
    dmma(acc[4], acc[5], s0, r1);
    dmma(acc[6], acc[7], s1, r0);
  }
  double s = 0;
  for (int e = 0; e < 8; ++e) s += acc[e];
  if (s == 1234.5) out[0] = s;
}

int main(int argc, char** argv) {
  const bool uniform = argc > 1;
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  // Zipf(1.1) sample table over 20000 ranks mapped through a permutation
  const int nz = 1 << 20, K = 20000;
  std::vector<double> cdf(K);
  double acc = 0;
  for (int r = 0; r < K; ++r) cdf[r] = (acc += std::pow(r + 1.0, -1.1));
  std::vector<int> perm(K), z(nz);
  for (int i = 0; i < K; ++i) perm[i] = (int)((i * 7919LL) % K);
  unsigned long long st = 88172645463325252ull;
  for (int i = 0; i < nz; ++i) {
    st ^= st << 13; st ^= st >> 7; st ^= st << 17;
    const double u = (st >> 11) * 0x1.0p-53 * acc;
    int lo = 0, hi = K - 1;
    while (lo < hi) { int m = (lo + hi) / 2; if (cdf[m] < u) lo = m + 1; else hi = m; }
    z[i] = uniform ? (int)((st >> 20) % K) : perm[lo];
  }
  double *V, *U, *out;
  int* dz;
  cudaMalloc(&V, (size_t)K * 16 * 8);
  cudaMalloc(&U, (size_t)K * 16 * 8);
  cudaMemset(V, 0, (size_t)K * 16 * 8);
  cudaMemset(U, 0, (size_t)K * 16 * 8);
  cudaMalloc(&out, 8);
  cudaMalloc(&dz, nz * 4);
  cudaMemcpy(dz, z.data(), nz * 4, cudaMemcpyHostToDevice);
  const int total_groups = 627716;
  for (int warps_per_sm : {16, 24}) {
    const int blocks = sms * warps_per_sm / 8;
    const int gpw = (total_groups + blocks * 8 - 1) / (blocks * 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    k<2><<<blocks, 256>>>(V, U, dz, nz, gpw, out);
    cudaEventRecord(a);
    k<2><<<blocks, 256>>>(V, U, dz, nz, gpw, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("NV=2 warps/SM %d: %.1f us for %d groups (%s)\n", warps_per_sm, ms * 1e3, blocks * 8 * gpw,
           cudaGetErrorString(cudaGetLastError()));
    k<3><<<blocks, 256>>>(V, U, dz, nz, gpw, out);
    cudaEventRecord(a);
    k<3><<<blocks, 256>>>(V, U, dz, nz, gpw, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("NV=3 warps/SM %d: %.1f us\n", warps_per_sm, ms * 1e3);
  }
  return 0;
}
