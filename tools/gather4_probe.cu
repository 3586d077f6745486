// Microbenchmark: factor-row gathers with the Blackwell TMA gather4 mode
// (cp.async.bulk.tensor.2d ... tile::gather4, SASS UTMALDG.2D.GATHER4): one
// instruction brings 4 arbitrary rows of a 2D fp64 tensor map into shared
// memory, completing on an mbarrier. Measures rows per clock per SM for
// random rows of a 20000 x 16 (and 1024 x 16) table, with and without
// consuming the rows (LDS) — compared with LDG gathers (tools/gather_probe.cu).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gather4_probe tools/gather4_probe.cu
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>

__device__ __forceinline__ void mbar_init(unsigned long long* m, int count) {
  unsigned a = (unsigned)__cvta_generic_to_shared(m);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count));
}
__device__ __forceinline__ void mbar_expect(unsigned long long* m, int bytes) {
  unsigned a = (unsigned)__cvta_generic_to_shared(m);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* m, int phase) {
  unsigned a = (unsigned)__cvta_generic_to_shared(m);
  asm volatile(
      "{\n .reg .pred p;\n W%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W%=;\n}\n"
      ::"r"(a), "r"(phase) : "memory");
}
__device__ __forceinline__ void gather4(void* dst, const CUtensorMap* map, int col, int r0, int r1,
                                        int r2, int r3, unsigned long long* m) {
  unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  unsigned b = (unsigned)__cvta_generic_to_shared(m);
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
      ::"r"(d), "l"(map), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(b)
      : "memory");
}

// each warp: ISSUERS lanes each issue one gather4 (4 rows) per stage into a
// ring of STAGES stages of (ISSUERS*4) rows x 128 B
template <int STAGES, int ISSUERS, bool CONSUME>
__global__ void k_g4(const __grid_constant__ CUtensorMap map, int rows, int iters, double* out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  constexpr int kRowsPerStage = ISSUERS * 4;
  constexpr int kStageBytes = kRowsPerStage * 128;
  double* buf = reinterpret_cast<double*>(smem) + (size_t)warp * STAGES * kRowsPerStage * 16;
  unsigned long long* bars =
      reinterpret_cast<unsigned long long*>(smem + (size_t)nw * STAGES * kStageBytes) + warp * STAGES;
  if (lane == 0)
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  unsigned x = 12345u + blockIdx.x * 977u + warp * 131u + lane * 7u;
  double acc = 0;
  auto issue = [&](int s) {
    if (lane == 0) mbar_expect(&bars[s], kStageBytes);
    __syncwarp();
    if (lane < ISSUERS) {
      int r[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        x = x * 1664525u + 1013904223u;
        r[q] = (x >> 8) % rows;
      }
      gather4(buf + ((size_t)s * kRowsPerStage + lane * 4) * 16, &map, 0, r[0], r[1], r[2], r[3],
              &bars[s]);
    }
  };
  for (int s = 0; s < STAGES; ++s) issue(s);
  for (int it = 0; it < iters; ++it) {
    const int s = it % STAGES;
    mbar_wait(&bars[s], (it / STAGES) & 1);
    if (CONSUME) {
      // 4 lanes per 128-byte row, 32 bytes each: kRowsPerStage/8 LDS.256-equivalents
      for (int q = 0; q < kRowsPerStage / 8; ++q) {
        const double2 v = reinterpret_cast<const double2*>(
            buf + ((size_t)s * kRowsPerStage + q * 8 + (lane >> 2)) * 16)[(lane & 3) * 2];
        acc += v.x + v.y;
      }
    }
    __syncwarp();
    if (it + STAGES < iters) issue(s);
  }
  if (acc == 1234.5) out[0] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);

template <int STAGES, int ISSUERS, bool CONSUME>
void run(EncodeFn enc, double* table, int rows, double* out, int sms, int warps) {
  CUtensorMap map;
  cuuint64_t gdim[2] = {16, (cuuint64_t)rows};
  cuuint64_t gstride[1] = {16 * sizeof(double)};
  cuuint32_t box[2] = {16, 1};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, table, gdim, gstride, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("encode failed %d\n", (int)r);
    return;
  }
  const int iters = 1024, threads = 32 * warps, blocks = sms * 2;
  const size_t smem = (size_t)warps * STAGES * ISSUERS * 4 * 128 + warps * STAGES * 8;
  cudaFuncSetAttribute(k_g4<STAGES, ISSUERS, CONSUME>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_g4<STAGES, ISSUERS, CONSUME><<<blocks, threads, smem>>>(map, rows, iters, out);
  cudaEventRecord(a);
  k_g4<STAGES, ISSUERS, CONSUME><<<blocks, threads, smem>>>(map, rows, iters, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double nrows = double(blocks) * warps * iters * ISSUERS * 4;
  printf("gather4 stages %d issuers %2d warps %2d consume %d rows %5d : %7.2f TB/s  %.2f rows/clk/SM (%s)\n",
         STAGES, ISSUERS, warps, CONSUME, rows, nrows * 128 / (ms * 1e-3) / 1e12,
         nrows / (ms * 1e-3) / sms / 1.9e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  if (!enc) {
    printf("no cuTensorMapEncodeTiled\n");
    return 1;
  }
  double *table, *out;
  cudaMalloc(&table, (size_t)(1 << 16) * 16 * sizeof(double));
  cudaMemset(table, 0, (size_t)(1 << 16) * 16 * sizeof(double));
  cudaMalloc(&out, 8);
  for (int rows : {1024, 20000}) {
    run<2, 8, false>(enc, table, rows, out, sms, 8);
    run<4, 8, false>(enc, table, rows, out, sms, 8);
    run<2, 32, false>(enc, table, rows, out, sms, 4);
    run<4, 8, true>(enc, table, rows, out, sms, 8);
    run<2, 32, true>(enc, table, rows, out, sms, 4);
  }
  return 0;
}
