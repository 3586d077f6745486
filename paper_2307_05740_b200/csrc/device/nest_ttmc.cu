// TTMc kernels on the fp64 tensor cores (mma.sync m8n8k4 f64 -> SASS DMMA).
//
// TTMc-3, reference nest ((T*V)*U) with orders (i,j,k,s)(i,j,s,r):
//   per (i,j) fiber   X[s] = sum_k t * V[k,s]            (vector-accumulate hook)
//   per (i,j) fiber   Y_i[r,s] += U[j,r] * X[s]           (rank-1 hook)
// The rank-1 updates of one root slice are a dense GEMM Y_i = U_J^T X_J whose
// K dimension runs over the slice's fibers: each warp feeds 4 fiber segments
// per step into four 8x8x4 DMMAs (16x16 tile, R,S <= 16).
//
// TTMc-4, reference nest (((T*W)*V)*U) with orders (i,j,k,l,t)(i,j,k,s,t)
// (i,j,r,s,t):
//   per (i,j,k)   X[t] = sum_l t * W[l,t]                 (vector-accumulate)
//   per (i,j,k)   Y[s,t] += V[k,s] * X[t]                 (rank-1, DFMA)
//   per (i,j)     Out_i[r,(s,t)] += U[j,r] * Y[s,t]       (loop r + axpy)
// The last stage is Out_i(R x ST) += U_J^T Y_J with K over the slice's (i,j)
// fibers: eight 8x8x4 DMMAs per 4 segments (R,S,T <= 8).
//
// Work: the warp's item is `chunk` consecutive segments (fiber pieces of at
// most seg_len leaves / children). Lane L works on K-slot q = L%4 (one
// segment) and on the column pair/index h = L/4 of the fragments. Rows and
// columns are interleaved (r = 2h+mt, s = 2(2q+e)+nt for TTMc-3) so every
// factor-row gather is one 16-byte load per lane, 8 lanes per 128-byte row.
#include "internal.cuh"

namespace spttn_dev {

namespace {

constexpr int kBlock = 256;

__device__ __forceinline__ int warp_max4(int v) {
  v = max(v, __shfl_xor_sync(0xffffffffu, v, 1));
  v = max(v, __shfl_xor_sync(0xffffffffu, v, 2));
  return v;
}

template <bool VECU, bool VECV>
__global__ void __launch_bounds__(kBlock) k_ttmc3(RootOutArgs a) {
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * kBlock + threadIdx.x) / 32;
  if (w >= a.n_items) return;  // warp-uniform
  const int lane = threadIdx.x & 31;
  const int q = lane & 3;
  const int h = lane >> 2;
  const int R = a.R, S = a.S;
  const CsfView& t = a.t;
  const double* __restrict__ U = a.f[1];
  const double* __restrict__ V = a.f[2];
  const int32_t* __restrict__ kidx = t.idx[2];
  const double* __restrict__ vals = t.vals;
  const int32_t* __restrict__ seg_begin = a.seg_begin;
  const int32_t* __restrict__ seg_node = a.seg_node;

  int64_t c = w * a.chunk;
  const int64_t cend = min64(c + a.chunk, a.n_seg);
  int32_t sl = a.item_pos[w];
  int64_t sl_end = a.slice_seg[sl + 1];
  bool head = a.slice_seg[sl] < c;
  int32_t row = t.idx[0][sl];
  bool pending = false;
  double acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.0;

  auto flush = [&](int slot) {
    double* dst = slot < 0 ? a.out + static_cast<int64_t>(row) * R * S
                           : a.part + (w * 2 + slot) * static_cast<int64_t>(R) * S;
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = 2 * h + mt;
          const int s = 2 * (2 * q + e) + nt;
          if (r < R && s < S) dst[r * S + s] = acc[(mt * 2 + nt) * 2 + e];
        }
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.0;
  };

  while (c < cend) {
    const int64_t lim = min(cend, sl_end);
    const int64_t my = c + q;
    const bool valid = my < lim;
    int32_t lb = 0, le = 0, j = 0;
    if (valid) {
      lb = __ldg(seg_begin + my);
      le = __ldg(seg_begin + my + 1);
      j = __ldg(seg_node + my);
    }
    const double2 u = valid ? row2<VECU>(U + static_cast<int64_t>(j) * R, 2 * h, R)
                            : make_double2(0, 0);
    const int n = le - lb;
    const int nmax = warp_max4(n);
    double x0 = 0.0, x1 = 0.0;
    int it = 0;
    for (; it + 2 <= nmax; it += 2) {
      int32_t k0 = 0, k1 = 0;
      double v0 = 0, v1 = 0;
      if (it < n) {
        k0 = __ldg(kidx + lb + it);
        v0 = __ldg(vals + lb + it);
      }
      if (it + 1 < n) {
        k1 = __ldg(kidx + lb + it + 1);
        v1 = __ldg(vals + lb + it + 1);
      }
      const double2 r0 = it < n ? row2<VECV>(V + static_cast<int64_t>(k0) * S, 2 * h, S)
                                : make_double2(0, 0);
      const double2 r1 = it + 1 < n ? row2<VECV>(V + static_cast<int64_t>(k1) * S, 2 * h, S)
                                    : make_double2(0, 0);
      x0 = fma(v0, r0.x, x0);
      x1 = fma(v0, r0.y, x1);
      x0 = fma(v1, r1.x, x0);
      x1 = fma(v1, r1.y, x1);
    }
    if (it < nmax && it < n) {
      const int32_t k0 = __ldg(kidx + lb + it);
      const double v0 = __ldg(vals + lb + it);
      const double2 r0 = row2<VECV>(V + static_cast<int64_t>(k0) * S, 2 * h, S);
      x0 = fma(v0, r0.x, x0);
      x1 = fma(v0, r0.y, x1);
    }
    // rank-1 updates of 4 segments: D[mt][nt] += A[mt] (8x4) * B[nt] (4x8)
    dmma_8x8x4(acc[0], acc[1], u.x, x0);
    dmma_8x8x4(acc[2], acc[3], u.x, x1);
    dmma_8x8x4(acc[4], acc[5], u.y, x0);
    dmma_8x8x4(acc[6], acc[7], u.y, x1);
    pending = true;
    c = min(c + 4, lim);
    if (c == sl_end) {
      flush(head ? 0 : -1);
      pending = false;
      head = false;
      if (c < cend) {
        ++sl;
        sl_end = a.slice_seg[sl + 1];
        row = t.idx[0][sl];
      }
    }
  }
  if (pending) flush(head ? 0 : 1);
}

template <bool VECV>
__global__ void __launch_bounds__(kBlock) k_ttmc4(RootOutArgs a) {
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * kBlock + threadIdx.x) / 32;
  if (w >= a.n_items) return;
  const int lane = threadIdx.x & 31;
  const int q = lane & 3;
  const int h = lane >> 2;
  const int R = a.R, S = a.S, T = a.T;
  const CsfView& t = a.t;
  const double* __restrict__ U = a.f[1];
  const double* __restrict__ V = a.f[2];
  const double* __restrict__ W = a.f[3];
  const int32_t* __restrict__ kidx = t.idx[2];
  const int32_t* __restrict__ lidx = t.idx[3];
  const int32_t* __restrict__ kptr = t.ptr[2];
  const double* __restrict__ vals = t.vals;
  const int64_t tile = static_cast<int64_t>(R) * S * T;

  int64_t c = w * a.chunk;
  const int64_t cend = min64(c + a.chunk, a.n_seg);
  int32_t sl = a.item_pos[w];
  int64_t sl_end = a.slice_seg[sl + 1];
  bool head = a.slice_seg[sl] < c;
  int32_t row = t.idx[0][sl];
  bool pending = false;
  double acc[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) acc[e] = 0.0;

  auto flush = [&](int slot) {
    double* dst = slot < 0 ? a.out + static_cast<int64_t>(row) * tile
                           : a.part + (w * 2 + slot) * tile;
    // tile nt = s: D[r = h][col = 2q+e] -> (r, s, t = 2q+e)
#pragma unroll
    for (int s = 0; s < 8; ++s)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int tt = 2 * q + e;
        if (h < R && s < S && tt < T) dst[(h * S + s) * T + tt] = acc[2 * s + e];
      }
#pragma unroll
    for (int e = 0; e < 16; ++e) acc[e] = 0.0;
  };

  while (c < cend) {
    const int64_t lim = min(cend, sl_end);
    const int64_t my = c + q;
    const bool valid = my < lim;
    int32_t kb = 0, ke = 0, j = 0;
    if (valid) {
      kb = __ldg(a.seg_begin + my);
      ke = __ldg(a.seg_begin + my + 1);
      j = __ldg(a.seg_node + my);
    }
    const double u = (valid && h < R) ? __ldg(U + static_cast<int64_t>(j) * R + h) : 0.0;
    int32_t lb = 0, le = 0, kend = 0, k = 0;
    if (valid) {
      lb = __ldg(kptr + kb);
      le = __ldg(kptr + ke);
      kend = __ldg(kptr + kb + 1);
      k = __ldg(kidx + kb);
    }
    int32_t kc = kb;
    const int n = le - lb;
    const int nmax = warp_max4(n);
    double Y[8];
#pragma unroll
    for (int s = 0; s < 8; ++s) Y[s] = 0.0;
    double X = 0.0;
    for (int it = 0; it < nmax; ++it) {
      if (it < n) {
        const int32_t p = lb + it;
        const int32_t l = __ldg(lidx + p);
        const double v = __ldg(vals + p);
        const double wv = h < T ? __ldg(W + static_cast<int64_t>(l) * T + h) : 0.0;
        X = fma(v, wv, X);  // X[t] += t_ijkl * W[l,t]
        if (p + 1 == kend) {
          // rank-1: Y[s,t] += V[k,s] * X[t]
          double vr[8];
          const double* vrow = V + static_cast<int64_t>(k) * S;
          if (VECV) {
            const double4 a0 = ld256(vrow);
            const double4 a1 = ld256(vrow + 4);
            vr[0] = a0.x; vr[1] = a0.y; vr[2] = a0.z; vr[3] = a0.w;
            vr[4] = a1.x; vr[5] = a1.y; vr[6] = a1.z; vr[7] = a1.w;
          } else {
#pragma unroll
            for (int s = 0; s < 8; ++s) vr[s] = s < S ? __ldg(vrow + s) : 0.0;
          }
#pragma unroll
          for (int s = 0; s < 8; ++s) Y[s] = fma(vr[s], X, Y[s]);
          X = 0.0;
          ++kc;
          if (kc < ke) {
            kend = __ldg(kptr + kc + 1);
            k = __ldg(kidx + kc);
          }
        }
      }
    }
    // Out_i[r, s, t] += U[j,r] * Y[s,t]: tile nt = s, A = U^T (8 x 4 slots)
#pragma unroll
    for (int s = 0; s < 8; ++s) dmma_8x8x4(acc[2 * s], acc[2 * s + 1], u, Y[s]);
    pending = true;
    c = min(c + 4, lim);
    if (c == sl_end) {
      flush(head ? 0 : -1);
      pending = false;
      head = false;
      if (c < cend) {
        ++sl;
        sl_end = a.slice_seg[sl + 1];
        row = t.idx[0][sl];
      }
    }
  }
  if (pending) flush(head ? 0 : 1);
}

}  // namespace

void launch_ttmc3(const RootOutArgs& a, cudaStream_t s) {
  const int64_t blocks = (a.n_items * 32 + kBlock - 1) / kBlock;
  if (blocks == 0) return;
  const bool vu = a.vec & 1, vv = a.vec & 2;
  if (vu && vv)
    k_ttmc3<true, true><<<static_cast<unsigned>(blocks), kBlock, 0, s>>>(a);
  else if (vu)
    k_ttmc3<true, false><<<static_cast<unsigned>(blocks), kBlock, 0, s>>>(a);
  else if (vv)
    k_ttmc3<false, true><<<static_cast<unsigned>(blocks), kBlock, 0, s>>>(a);
  else
    k_ttmc3<false, false><<<static_cast<unsigned>(blocks), kBlock, 0, s>>>(a);
  SPTTN_CUDA(cudaGetLastError());
}

void launch_ttmc4(const RootOutArgs& a, cudaStream_t s) {
  const int64_t blocks = (a.n_items * 32 + kBlock - 1) / kBlock;
  if (blocks == 0) return;
  if (a.vec & 2)
    k_ttmc4<true><<<static_cast<unsigned>(blocks), kBlock, 0, s>>>(a);
  else
    k_ttmc4<false><<<static_cast<unsigned>(blocks), kBlock, 0, s>>>(a);
  SPTTN_CUDA(cudaGetLastError());
}

}  // namespace spttn_dev
