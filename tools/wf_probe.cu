// Microbenchmark: L1 data-pipe wavefronts and throughput of the lane layouts
// the TTMc kernels can use to move 128-byte factor rows into registers —
// row-contiguous vs DMMA-fragment order, 64/128/256-bit, global vs shared,
// broadcast reads and shuffles. Run under ncu for the wavefront counts:
//   ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_lgds.sum,
//       l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed.sum,
//       gpu__time_duration.sum tools/wf_probe
// Build: make probes (-> tools/wf_probe)
#include <cstdio>
#include <cuda_runtime.h>

enum {
  G256_ROW = 0,   // LDG.256, 4 consecutive lanes per row, 8 rows
  G128_ROW = 1,   // LDG.128, 8 consecutive lanes per row, 4 rows
  G128_FRAG = 2,  // LDG.128, row = lane%4, 16-byte chunk = lane/4 (4 full rows)
  G64_FRAG = 3,   // LDG.64, row = lane%4, column = lane/4 (4 half rows)
  G64_ROW = 4,    // LDG.64, 16 consecutive lanes per row, 2 rows
  S128_ROW = 10,  // LDS.128 row order
  S128_FRAG = 11, // LDS.128 fragment order
  S64_FRAG = 12,  // LDS.64 fragment order
  S128_BC4 = 13,  // LDS.128, one row for the warp, chunk = lane/4 (4 lanes per address)
  S64_BC4 = 14,   // LDS.64, one row, column = lane/4
  S128_BC8 = 15,  // LDS.128, one row, chunk = lane%8
  SHFL = 16,      // SHFL.IDX 32-bit, arbitrary source lane
  S128_ST = 17,   // STS.128 row order (then one LDS.128 back)
  S64_ROW = 18,   // LDS.64 row order (2 rows)
  CPA16_ROW = 20, // cp.async 16 B (LDGSTS.128), 8 consecutive lanes per row, 4 rows, into smem
};

template <int PAT>
__global__ void k_probe(const double* __restrict__ table, int rows, int iters, double* out) {
  extern __shared__ double sh[];
  const int lane = threadIdx.x & 31;
  constexpr bool SMEM = PAT >= 10 && PAT < 20;
  if (SMEM) {
    for (int i = threadIdx.x; i < rows * 16; i += blockDim.x) sh[i] = table[i];
    __syncthreads();
  }
  int slot, col;
  switch (PAT) {
    case G256_ROW: slot = lane >> 2; col = 4 * (lane & 3); break;
    case G128_ROW: case S128_ROW: case S128_ST: case CPA16_ROW: slot = lane >> 3; col = 2 * (lane & 7); break;
    case G128_FRAG: case S128_FRAG: slot = lane & 3; col = 2 * (lane >> 2); break;
    case G64_FRAG: case S64_FRAG: slot = lane & 3; col = lane >> 2; break;
    case G64_ROW: case S64_ROW: slot = lane >> 4; col = lane & 15; break;
    case S128_BC4: slot = 0; col = 2 * (lane >> 2); break;
    case S64_BC4: slot = 0; col = lane >> 2; break;
    case S128_BC8: slot = 0; col = 2 * (lane & 7); break;
    default: slot = lane; col = 0; break;
  }
  unsigned x = 12345u + blockIdx.x * 977u + (threadIdx.x >> 5) * 131u + slot * 7u;
  double acc = 0;
  constexpr int U = 8;
  double* wsh = sh + (threadIdx.x >> 5) * 128;  // per-warp scratch (S128_ST, CPA16_ROW)
  for (int it = 0; it < iters; it += U) {
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      x = x * 1664525u + 1013904223u;
      const int r = (x >> 8) % rows;
      const double* p = (SMEM ? sh : table) + r * 16 + col;
      if (PAT == G256_ROW) {
        double4 w;
        asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                     : "=d"(w.x), "=d"(w.y), "=d"(w.z), "=d"(w.w) : "l"(p));
        v[u] = w.x + w.y + w.z + w.w;
      } else if (PAT == G128_ROW || PAT == G128_FRAG) {
        double2 w;
        asm volatile("ld.global.nc.v2.f64 {%0,%1}, [%2];" : "=d"(w.x), "=d"(w.y) : "l"(p));
        v[u] = w.x + w.y;
      } else if (PAT == G64_FRAG || PAT == G64_ROW) {
        v[u] = __ldg(p);
      } else if (PAT == S128_ROW || PAT == S128_FRAG || PAT == S128_BC4 || PAT == S128_BC8) {
        const double2 w = *reinterpret_cast<const double2*>(p);
        v[u] = w.x + w.y;
      } else if (PAT == S64_FRAG || PAT == S64_BC4 || PAT == S64_ROW) {
        v[u] = *p;
      } else if (PAT == SHFL) {
        v[u] = __int_as_float(__shfl_sync(0xffffffffu, __float_as_int(static_cast<float>(acc)) + u,
                                          (x >> 3) & 31));
      } else if (PAT == CPA16_ROW) {
        const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(wsh + 2 * lane + 64 * (u & 1)));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(p) : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
        if (u & 1) {
          asm volatile("cp.async.wait_group 0;" ::: "memory");
          __syncwarp();
          v[u] = wsh[2 * lane] + wsh[2 * lane + 64];
        } else {
          v[u] = 0;
        }
      } else {  // S128_ST
        *reinterpret_cast<double2*>(wsh + 2 * (lane & 31)) = make_double2(acc, u);
        __syncwarp();
        const double2 w = *reinterpret_cast<const double2*>(wsh + 2 * ((lane + u) & 31));
        __syncwarp();
        v[u] = w.x + w.y;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u];
  }
  if (acc == 1234.5) out[0] = acc;
}

template <int PAT>
void run(const char* name, const double* table, int rows, double* out, int sms) {
  const int iters = 4096, threads = 256, blocks = sms * 4;
  const size_t smem = PAT >= 20 ? 8 * 128 * sizeof(double)
                     : PAT >= 10 ? static_cast<size_t>(rows) * 16 * sizeof(double) : 0;
  if (smem) cudaFuncSetAttribute(k_probe<PAT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_probe<PAT><<<blocks, threads, smem>>>(table, rows, iters, out);
  cudaEventRecord(a);
  k_probe<PAT><<<blocks, threads, smem>>>(table, rows, iters, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double instr = double(blocks) * threads / 32 * iters;  // warp-level loads
  printf("%-10s rows %5d : %7.3f ms  %6.3f warp-loads/clk/SM @1.9GHz  err=%s\n", name, rows, ms,
         instr / (ms * 1e-3) / sms / 1.9e9, cudaGetErrorString(cudaGetLastError()));
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
    run<G256_ROW>("g256row", table, rows, out, sms);
    run<G128_ROW>("g128row", table, rows, out, sms);
    run<G128_FRAG>("g128frag", table, rows, out, sms);
    run<G64_FRAG>("g64frag", table, rows, out, sms);
    run<G64_ROW>("g64row", table, rows, out, sms);
  }
  run<CPA16_ROW>("cpa16row", table, 20000, out, sms);
  const int srows = 256;
  run<S128_ROW>("s128row", table, srows, out, sms);
  run<S128_FRAG>("s128frag", table, srows, out, sms);
  run<S64_FRAG>("s64frag", table, srows, out, sms);
  run<S128_BC4>("s128bc4", table, srows, out, sms);
  run<S64_BC4>("s64bc4", table, srows, out, sms);
  run<S128_BC8>("s128bc8", table, srows, out, sms);
  run<SHFL>("shfl", table, srows, out, sms);
  run<S128_ST>("s128st", table, srows, out, sms);
  run<S64_ROW>("s64row", table, srows, out, sms);
  return 0;
}
