// Microbenchmark: L1 shared-memory wavefronts of one LDS.128 per warp for
// explicit lane -> 16-byte-chunk address tables (the TTMc-4 V / W tile reads
// and candidate re-mappings). Run under ncu for the wavefront counts:
//   ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,
//       smsp__inst_executed_op_shared_ld.sum tools/lds_probe
// Build: make probes (-> tools/lds_probe)
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kPat = 8;
// chunk (16 bytes) index read by each lane, per pattern
__constant__ int c_chunk[kPat][32];

template <int P>
__global__ void k_lds(int iters, double* out) {
  __shared__ __align__(16) double tile[2 * 64];  // 16 chunks of 16 bytes... extended below
  __shared__ __align__(16) double big[512];
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 512; i += blockDim.x) big[i] = i;
  if (threadIdx.x < 128) tile[threadIdx.x] = threadIdx.x;
  __syncthreads();
  const int off = 2 * c_chunk[P][lane];
  double acc = 0;
  for (int it = 0; it < iters; ++it) {
    const double2 v = *reinterpret_cast<const double2*>(big + ((off + 64 * (it & 3)) & 511));
    acc += v.x * v.y;
  }
  if (acc == 1234.5) out[0] = acc;
}

int main() {
  int h_chunk[kPat][32];
  for (int L = 0; L < 32; ++L) {
    const int q = L & 3, h = L >> 2;
    const int sw = (q >> 1) & 1;
    // rows of 64 bytes (4 chunks): slot row r at chunk 4r
    h_chunk[0][L] = q * 4 + ((2 * (h & 1)) ^ sw);        // TTMc-4 V read a0 (sb = h&1)
    h_chunk[1][L] = q * 4 + ((h >> 1) ^ sw);             // TTMc-4 W read wa (tb = h>>1)
    h_chunk[2][L] = q * 4 + ((2 * (h >> 2)) ^ sw);       // V with sb = h>>2
    h_chunk[3][L] = q * 4 + ((h & 3) ^ sw);              // W with tb = h&3
    h_chunk[4][L] = (L >> 2);                            // bc4 reference: 8 chunks, 4 consecutive lanes each
    h_chunk[5][L] = (L & 7);                             // bc8 reference
    h_chunk[6][L] = q * 4 + (2 * (h & 1));               // V a0 without swizzle
    h_chunk[7][L] = (L & 3) * 4;                         // 4 rows, same chunk column: 4 distinct, period 4
  }
  cudaMemcpyToSymbol(c_chunk, h_chunk, sizeof(h_chunk));
  double* out;
  cudaMalloc(&out, 8);
  const int iters = 1 << 14;
  k_lds<0><<<148, 256>>>(iters, out);
  k_lds<1><<<148, 256>>>(iters, out);
  k_lds<2><<<148, 256>>>(iters, out);
  k_lds<3><<<148, 256>>>(iters, out);
  k_lds<4><<<148, 256>>>(iters, out);
  k_lds<5><<<148, 256>>>(iters, out);
  k_lds<6><<<148, 256>>>(iters, out);
  k_lds<7><<<148, 256>>>(iters, out);
  cudaDeviceSynchronize();
  printf("lds_probe: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
