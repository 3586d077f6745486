// Leaf-range "group" kernels: MTTKRP-3 and MTTKRP-4 for any rank (the packed
// kernels cover R <= 32).
//
// Each work item is a fixed range of `chunk` consecutive CSF leaves (the
// nnz-balanced partition; long fibers and slices are split across items).
// An item is owned by a group of G lanes; lane g of the group owns the 4
// consecutive rank columns [4g, 4g+4) of every factor row, so a factor-row
// gather is one 256-bit load per lane and G*32 bytes per group (coalesced).
// The per-fiber intermediates of the fused nest (X[r], Y[r], P[r]) and the
// per-slice output row live in registers.
//
// The walk follows the reference's fused nests exactly (executor.cpp:453-490
// with the hooks of :411-451):
//   MTTKRP-3  ((T*C)*B)  (i,j,k,a)(i,j,a):      X += t*C[k];  acc += X*B[j]
//   MTTKRP-4  (((T*D)*C)*B):  X += t*D[l]; Y += X*C[k]; acc += Y*B[j]
// A fiber cut by an item boundary contributes through the same products
// (linearity), and a root slice split across items is written as HEAD/TAIL
// partial rows that the fix-up kernel sums in item order: the result is
// deterministic (bit-identical across runs).
#include "internal.cuh"

namespace spttn_dev {

namespace {

constexpr int kBlock = 256;
constexpr int kBatch = 4;

// Where a finished (or interrupted) root-slice accumulator goes.
template <int G>
__device__ __forceinline__ void flush_row(const RootOutArgs& a, int64_t item, int slot, int row,
                                          int c, const double4& acc) {
  double* dst = slot < 0 ? a.out + static_cast<int64_t>(row) * a.R
                         : a.part + (item * 2 + slot) * static_cast<int64_t>(a.R);
  store4(dst, c, a.R, acc);
}

template <int G, bool VEC>
__global__ void __launch_bounds__(kBlock) k_mttkrp3(RootOutArgs a) {
  const int64_t gid = (static_cast<int64_t>(blockIdx.x) * kBlock + threadIdx.x) / G;
  if (gid >= a.n_items) return;
  const int c = (threadIdx.x & (G - 1)) * 4;
  const int R = a.R;
  const CsfView& t = a.t;
  const double* __restrict__ B = a.f[1];
  const double* __restrict__ C = a.f[2];
  const int32_t* __restrict__ kidx = t.idx[2];
  const double* __restrict__ vals = t.vals;

  int32_t p = static_cast<int32_t>(gid * a.chunk);
  const int32_t pend = static_cast<int32_t>(min64(gid * a.chunk + a.chunk, t.nlev[2]));
  int32_t p0 = a.item_pos[gid * 3 + 0];
  int32_t p1 = a.item_pos[gid * 3 + 1];
  int32_t f0end = t.ptr[0][p0 + 1];
  int32_t f1end = t.ptr[1][p1 + 1];
  bool head = t.ptr[1][t.ptr[0][p0]] < p;
  int32_t row = t.idx[0][p0];
  double4 brow = row4<VEC>(B + static_cast<int64_t>(t.idx[1][p1]) * R, c, R);
  double4 X = make_double4(0, 0, 0, 0), acc = X;

  for (; p < pend; p += kBatch) {
    int32_t kk[kBatch];
    double vv[kBatch];
    double4 cr[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u)
      if (p + u < pend) {
        kk[u] = __ldg(kidx + p + u);
        vv[u] = __ldg(vals + p + u);
      }
#pragma unroll
    for (int u = 0; u < kBatch; ++u)
      if (p + u < pend) cr[u] = row4<VEC>(C + static_cast<int64_t>(kk[u]) * R, c, R);
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const int32_t q = p + u;
      if (q >= pend) break;
      // vector-accumulate hook: X[a] += t * C[k,a]
      fma4(X, vv[u], cr[u]);
      const bool last = q + 1 == pend;
      const bool e1 = q + 1 == f1end;
      const bool e0 = e1 && (p1 + 1 == f0end);
      if (e1 || last) {  // term 2 leaf: acc[a] += X[a] * B[j,a]
        fma4v(acc, X, brow);
        X = make_double4(0, 0, 0, 0);
      }
      if (e0) {
        flush_row<G>(a, gid, head ? 0 : -1, row, c, acc);
        acc = make_double4(0, 0, 0, 0);
        head = false;
      } else if (last) {
        flush_row<G>(a, gid, head ? 0 : 1, row, c, acc);
      }
      if (!last) {
        if (e1) {
          ++p1;
          f1end = t.ptr[1][p1 + 1];
          brow = row4<VEC>(B + static_cast<int64_t>(t.idx[1][p1]) * R, c, R);
        }
        if (e0) {
          ++p0;
          f0end = t.ptr[0][p0 + 1];
          row = t.idx[0][p0];
        }
      }
    }
  }
}

template <int G, bool VEC>
__global__ void __launch_bounds__(kBlock) k_mttkrp4(RootOutArgs a) {
  const int64_t gid = (static_cast<int64_t>(blockIdx.x) * kBlock + threadIdx.x) / G;
  if (gid >= a.n_items) return;
  const int c = (threadIdx.x & (G - 1)) * 4;
  const int R = a.R;
  const CsfView& t = a.t;
  const double* __restrict__ B = a.f[1];
  const double* __restrict__ C = a.f[2];
  const double* __restrict__ D = a.f[3];
  const int32_t* __restrict__ lidx = t.idx[3];
  const double* __restrict__ vals = t.vals;

  int32_t p = static_cast<int32_t>(gid * a.chunk);
  const int32_t pend = static_cast<int32_t>(min64(gid * a.chunk + a.chunk, t.nlev[3]));
  int32_t p0 = a.item_pos[gid * 4 + 0];
  int32_t p1 = a.item_pos[gid * 4 + 1];
  int32_t p2 = a.item_pos[gid * 4 + 2];
  int32_t f0end = t.ptr[0][p0 + 1];
  int32_t f1end = t.ptr[1][p1 + 1];
  int32_t f2end = t.ptr[2][p2 + 1];
  bool head = t.ptr[2][t.ptr[1][t.ptr[0][p0]]] < p;
  int32_t row = t.idx[0][p0];
  double4 brow = row4<VEC>(B + static_cast<int64_t>(t.idx[1][p1]) * R, c, R);
  double4 crow = row4<VEC>(C + static_cast<int64_t>(t.idx[2][p2]) * R, c, R);
  double4 X = make_double4(0, 0, 0, 0), Y = X, acc = X;

  for (; p < pend; p += kBatch) {
    int32_t ll[kBatch];
    double vv[kBatch];
    double4 dr[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u)
      if (p + u < pend) {
        ll[u] = __ldg(lidx + p + u);
        vv[u] = __ldg(vals + p + u);
      }
#pragma unroll
    for (int u = 0; u < kBatch; ++u)
      if (p + u < pend) dr[u] = row4<VEC>(D + static_cast<int64_t>(ll[u]) * R, c, R);
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const int32_t q = p + u;
      if (q >= pend) break;
      fma4(X, vv[u], dr[u]);  // X[r] += t * D[l,r]
      const bool last = q + 1 == pend;
      const bool e2 = q + 1 == f2end;
      const bool e1 = e2 && (p2 + 1 == f1end);
      const bool e0 = e1 && (p1 + 1 == f0end);
      if (e2 || last) {  // Y[r] += X[r] * C[k,r]
        fma4v(Y, X, crow);
        X = make_double4(0, 0, 0, 0);
      }
      if (e1 || last) {  // acc[r] += Y[r] * B[j,r]
        fma4v(acc, Y, brow);
        Y = make_double4(0, 0, 0, 0);
      }
      if (e0) {
        flush_row<G>(a, gid, head ? 0 : -1, row, c, acc);
        acc = make_double4(0, 0, 0, 0);
        head = false;
      } else if (last) {
        flush_row<G>(a, gid, head ? 0 : 1, row, c, acc);
      }
      if (!last) {
        if (e2) {
          ++p2;
          f2end = t.ptr[2][p2 + 1];
          crow = row4<VEC>(C + static_cast<int64_t>(t.idx[2][p2]) * R, c, R);
        }
        if (e1) {
          ++p1;
          f1end = t.ptr[1][p1 + 1];
          brow = row4<VEC>(B + static_cast<int64_t>(t.idx[1][p1]) * R, c, R);
        }
        if (e0) {
          ++p0;
          f0end = t.ptr[0][p0 + 1];
          row = t.idx[0][p0];
        }
      }
    }
  }
}

template <template <int, bool> class K>
struct Dispatch;

#define SPTTN_GROUP_LAUNCH(KERNEL)                                                        \
  template <int G>                                                                        \
  void launch_##KERNEL##_g(const RootOutArgs& a, cudaStream_t s) {                        \
    const int64_t threads = a.n_items * G;                                                \
    const int64_t blocks = (threads + kBlock - 1) / kBlock;                               \
    if (blocks == 0) return;                                                              \
    if (a.vec)                                                                            \
      k_##KERNEL<G, true><<<static_cast<unsigned>(blocks), kBlock, 0, s>>>(a);            \
    else                                                                                  \
      k_##KERNEL<G, false><<<static_cast<unsigned>(blocks), kBlock, 0, s>>>(a);           \
  }                                                                                       \
  void dispatch_##KERNEL(const RootOutArgs& a, cudaStream_t s) {                          \
    switch (group_lanes_for(a.R)) {                                                       \
      case 1: launch_##KERNEL##_g<1>(a, s); break;                                        \
      case 2: launch_##KERNEL##_g<2>(a, s); break;                                        \
      case 4: launch_##KERNEL##_g<4>(a, s); break;                                        \
      case 8: launch_##KERNEL##_g<8>(a, s); break;                                        \
      case 16: launch_##KERNEL##_g<16>(a, s); break;                                      \
      default: launch_##KERNEL##_g<32>(a, s); break;                                      \
    }                                                                                     \
    SPTTN_CUDA(cudaGetLastError());                                                       \
  }

SPTTN_GROUP_LAUNCH(mttkrp3)
SPTTN_GROUP_LAUNCH(mttkrp4)

}  // namespace

int group_lanes_for(int R) {
  int g = 1;
  while (g * 4 < R) g *= 2;
  return g;
}

void launch_mttkrp3(const RootOutArgs& a, cudaStream_t s) { dispatch_mttkrp3(a, s); }
void launch_mttkrp4(const RootOutArgs& a, cudaStream_t s) { dispatch_mttkrp4(a, s); }

}  // namespace spttn_dev
