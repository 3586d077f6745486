// TTTP-3 / completion residual, leaf-parallel form.
//
// Reference nest (((A*B)*C)*T), orders (i,j,r)(i,j,k,r)(i,j,k)
// (proj/src/executor.cpp:389-409 walking the forest of loop_nest.cpp):
//   per (i,j) fiber  X[r] = A[i,r] * B[j,r]
//   per leaf         Y = sum_r X[r] * C[k,r];   S[leaf] = Y * t   (rho = t - Y)
// The output lives at each leaf's own position, so leaves are independent.
// At the BASELINE shape (5e7 leaves in 4.98e7 (i,j) fibers) fibers hold ~1
// leaf, so walking fibers buys no reuse; instead the plan expands the (i, j)
// coordinates of every leaf once (int32 per leaf, replacing the fiber level's
// idx+ptr reads) and every group of G lanes handles U leaves per step with no
// fiber logic: X[r] is recomputed per leaf with the same single rounding
// (A*B), so results equal the fiber-factored walk bit-for-bit.
//
// Lane g of a group owns the 4 rank columns [4g, 4g+4) (one 256-bit load per
// factor row). The U partial dot products of a group are combined by a
// transpose-reduction (log2 U exchange steps of halving width, then a plain
// butterfly): 2U-1 shuffles for U leaves instead of U*log2(G), after which
// lane (G/U)*q holds leaf q's sum and writes it.
#include "internal.cuh"
#include "tttp_reduce.cuh"

namespace spttn_dev {

namespace {

constexpr int kBlock = 256;

template <int G, int U, bool VEC>
__global__ void __launch_bounds__(kBlock) k_tttp3_leaf(RootOutArgs a, const int32_t* leaf_i,
                                                       const int32_t* leaf_j) {
  constexpr int kGroups = 32 / G;         // groups per warp
  constexpr int kWarpLeaves = kGroups * U;
  const int lane = threadIdx.x & 31;
  const int lg = lane & (G - 1);
  const int grp = lane / G;
  const int c = lg * 4;
  const int R = a.R;
  const double* __restrict__ A = a.f[0];
  const double* __restrict__ B = a.f[1];
  const double* __restrict__ C = a.f[2];
  const int32_t* __restrict__ kidx = a.t.idx[2];
  const double* __restrict__ vals = a.t.vals;
  const int64_t nnz = a.t.nlev[2];
  const bool residual = (a.flags & 1) != 0;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (kBlock / 32);
  const int64_t nbatch = (nnz + kWarpLeaves - 1) / kWarpLeaves;
  for (int64_t b = static_cast<int64_t>(blockIdx.x) * (kBlock / 32) + threadIdx.x / 32; b < nbatch;
       b += warps) {
    const int64_t base = b * kWarpLeaves + static_cast<int64_t>(grp) * U;
    int32_t ii[U], jj[U], kk[U];
    double tv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t p = base + u;
      const bool ok = p < nnz;
      ii[u] = ok ? __ldg(leaf_i + p) : 0;
      jj[u] = ok ? __ldg(leaf_j + p) : 0;
      kk[u] = ok ? __ldg(kidx + p) : 0;
      tv[u] = ok ? __ldg(vals + p) : 0.0;
    }
    double part[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      // (a data-dependent A[i] reuse branch serialises the gathers: measured
      // slower, so every leaf issues its three row loads back to back)
      const double4 ar = row4<VEC>(A + static_cast<int64_t>(ii[u]) * R, c, R);
      const double4 br = row4<VEC>(B + static_cast<int64_t>(jj[u]) * R, c, R);
      const double4 cr = row4<VEC>(C + static_cast<int64_t>(kk[u]) * R, c, R);
      // X[r] = A[i,r]*B[j,r] (term 1); Y += X[r]*C[k,r] (term 2)
      double y = (ar.x * br.x) * cr.x;
      y = fma(ar.y * br.y, cr.y, y);
      y = fma(ar.z * br.z, cr.z, y);
      y = fma(ar.w * br.w, cr.w, y);
      part[u] = y;
    }
    int q = 0;
    const double y = transpose_reduce<G, U>(part, lg, &q);
    if ((lg & (G / U - 1)) == 0) {
      const int64_t p = base + q;
      double t = tv[0];
#pragma unroll
      for (int u = 1; u < U; ++u) t = q == u ? tv[u] : t;
      if (p < nnz) a.out[p] = residual ? t - y : 0.0 + y * t;  // executor.cpp:402
    }
  }
}


template <int G, int U>
void launch_g(const RootOutArgs& a, const int32_t* li, const int32_t* lj, cudaStream_t s,
              int sms) {
  const int64_t nnz = a.t.nlev[2];
  if (nnz == 0) return;
  const int64_t warps_needed = (nnz + (32 / G) * U - 1) / ((32 / G) * U);
  const int64_t blocks = std::min<int64_t>((warps_needed + 7) / 8, static_cast<int64_t>(sms) * 8);
  if (a.vec)
    k_tttp3_leaf<G, U, true><<<static_cast<unsigned>(blocks), kBlock, 0, s>>>(a, li, lj);
  else
    k_tttp3_leaf<G, U, false><<<static_cast<unsigned>(blocks), kBlock, 0, s>>>(a, li, lj);
}

}  // namespace

void launch_tttp3_leaf(const RootOutArgs& a, const int32_t* leaf_i, const int32_t* leaf_j,
                       int batch, cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int G = group_lanes_for(a.R);
  const bool b4 = batch >= 4;
  const bool b8 = batch >= 8;
#define SPTTN_TTTP_G(GG)                                 \
  case GG:                                               \
    if (b8 && GG >= 8)                                   \
      launch_g<GG, (GG >= 8 ? 8 : 1)>(a, leaf_i, leaf_j, s, sms); \
    else if (b4 && GG >= 4)                              \
      launch_g<GG, (GG >= 4 ? 4 : 1)>(a, leaf_i, leaf_j, s, sms); \
    else if (GG >= 2)                                    \
      launch_g<GG, (GG >= 2 ? 2 : 1)>(a, leaf_i, leaf_j, s, sms); \
    else                                                 \
      launch_g<GG, 1>(a, leaf_i, leaf_j, s, sms);        \
    break;
  switch (G) {
    SPTTN_TTTP_G(1)
    SPTTN_TTTP_G(2)
    SPTTN_TTTP_G(4)
    SPTTN_TTTP_G(8)
    SPTTN_TTTP_G(16)
    SPTTN_TTTP_G(32)
  }
#undef SPTTN_TTTP_G
  SPTTN_CUDA(cudaGetLastError());
}

}  // namespace spttn_dev
