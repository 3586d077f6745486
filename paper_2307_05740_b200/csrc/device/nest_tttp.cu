// TTTP-3 / completion residual.
//
// Reference nest (((A*B)*C)*T), orders (i,j,r)(i,j,k,r)(i,j,k)
// (proj/src/executor.cpp:389-409 walking the forest of loop_nest.cpp):
//   per (i,j) fiber  X[r] = A[i,r] * B[j,r]
//   per leaf         Y = sum_r X[r] * C[k,r];   S[leaf] = Y * t   (rho = t - Y)
// The output lives at each leaf's own position, so leaves are independent.
// At the BASELINE shape (5e7 leaves in 4.98e7 (i,j) fibers) fibers hold ~1
// leaf, so walking fibers buys no reuse; the plan stores each leaf's {j, k}
// (one 8-byte record, replacing the fiber level's idx+ptr reads) and cuts
// every root slice into pieces of <= 64 consecutive leaves. A warp takes a
// piece: A[i] is loaded once into registers, then groups of G lanes handle
// U leaves per step with no fiber logic — X[r] is recomputed per leaf with the
// same single rounding (A*B), so results equal the fiber-factored walk's
// arithmetic per term.
//
// Lane g of a group owns the 4 rank columns [4g, 4g+4) (one 256-bit load per
// factor row). The U partial dot products of a group are combined by a
// transpose-reduction (log2 U exchange steps of halving width, then a plain
// butterfly): 2U-1 shuffles for U leaves instead of U*log2(G), after which
// lane (G/U)*q holds leaf q's sum and writes it.
#include <cub/cub.cuh>

#include "internal.cuh"
#include "tttp_reduce.cuh"

namespace spttn_dev {

namespace {

constexpr int kBlock = 256;

// A warp takes a piece of <= 64 consecutive leaves of ONE root slice
// (plan-time table {i, leaf lo, leaf hi}), so A[i] is gathered once per piece
// into registers instead of once per leaf and no per-leaf i coordinate is
// streamed. Per leaf the L1 data pipe then carries only the B[j] and C[k]
// rows (4 + 4 wavefronts at R = 64), the {j, k} / value fields and the
// transpose-reduction: ~12 instead of ~16 wavefronts for the round-1 leaf
// kernel (3.52 -> 2.75 ms at the BASELINE shape).
template <int G, int U, bool VEC>
__global__ void __launch_bounds__(kBlock) k_tttp3_piece(RootOutArgs a, const int4* pieces,
                                                        int64_t n_pieces, const int2* leaf_jk) {
  constexpr int kGroups = 32 / G;
  constexpr int kStep = kGroups * U;  // leaves per warp step
  const int lane = threadIdx.x & 31;
  const int lg = lane & (G - 1);
  const int grp = lane / G;
  const int c = lg * 4;
  const int R = a.R;
  const double* __restrict__ A = a.f[0];
  const double* __restrict__ B = a.f[1];
  const double* __restrict__ C = a.f[2];
  const double* __restrict__ vals = a.t.vals;
  const bool residual = (a.flags & 1) != 0;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (kBlock / 32);
  for (int64_t pc = static_cast<int64_t>(blockIdx.x) * (kBlock / 32) + threadIdx.x / 32;
       pc < n_pieces; pc += warps) {
    const int4 piece = __ldg(pieces + pc);  // {i, leaf lo, leaf hi, -}, warp-uniform
    SPTTN_DCHECK(piece.x >= 0 && piece.x < a.frows[0] && piece.y <= piece.z &&
                 piece.z <= a.t.nlev[2]);
    const double4 ar = row4<VEC>(A + static_cast<int64_t>(piece.x) * R, c, R);
    for (int32_t b = piece.y; b < piece.z; b += kStep) {
      const int32_t base = b + grp * U;
      int32_t jj[U], kk[U];
      double tv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const bool ok = base + u < piece.z;
        const int2 jk = ok ? __ldg(leaf_jk + base + u) : make_int2(0, 0);  // one 8-byte load
        jj[u] = jk.x;
        kk[u] = jk.y;
        SPTTN_DCHECK(jk.x >= 0 && jk.x < a.frows[1] && jk.y >= 0 && jk.y < a.frows[2]);
        tv[u] = ok ? __ldg(vals + base + u) : 0.0;
      }
      double part[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
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
        const int32_t p = base + q;
        double t = tv[0];
#pragma unroll
        for (int u = 1; u < U; ++u) t = q == u ? tv[u] : t;
        if (p < piece.z) a.out[p] = residual ? t - y : 0.0 + y * t;  // executor.cpp:402
      }
    }
  }
}

// piece table: slice s -> ceil(n_s / P) pieces {i, lo, hi}
__global__ void k_piece_counts(CsfView t, int P, int32_t* cnt) {
  const int32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= t.nlev[0]) return;
  const int32_t lo = t.ptr[1][t.ptr[0][s]], hi = t.ptr[1][t.ptr[0][s + 1]];
  cnt[s] = (hi - lo + P - 1) / P;
}

__global__ void k_piece_fill(CsfView t, int P, const int32_t* first, int4* pieces) {
  const int32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= t.nlev[0]) return;
  const int32_t lo = t.ptr[1][t.ptr[0][s]], hi = t.ptr[1][t.ptr[0][s + 1]];
  const int32_t row = t.idx[0][s];
  int32_t o = first[s];
  for (int32_t b = lo; b < hi; b += P) pieces[o++] = make_int4(row, b, min(b + P, hi), 0);
}

}  // namespace

int64_t build_tttp_pieces(const DevCsf& D, int P, int4** pieces, cudaStream_t s) {
  const int32_t n0 = static_cast<int32_t>(D.level_size[0]);
  *pieces = nullptr;
  if (n0 == 0 || D.level_size[2] == 0) return 0;
  int32_t* cnt = nullptr;
  dmalloc(&cnt, (static_cast<int64_t>(n0) + 1) * sizeof(int32_t), s);
  SPTTN_CUDA(cudaMemsetAsync(cnt + n0, 0, sizeof(int32_t), s));
  const CsfView t = D.view();
  k_piece_counts<<<(n0 + 255) / 256, 256, 0, s>>>(t, P, cnt);
  size_t bytes = 0;
  SPTTN_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, cnt, cnt, n0 + 1, s));
  void* tmp = nullptr;
  dmalloc(&tmp, std::max<size_t>(1, bytes), s);
  SPTTN_CUDA(cub::DeviceScan::ExclusiveSum(tmp, bytes, cnt, cnt, n0 + 1, s));
  dfree(tmp, s);
  int32_t n = 0;
  SPTTN_CUDA(cudaMemcpyAsync(&n, cnt + n0, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  SPTTN_CUDA(cudaStreamSynchronize(s));
  dmalloc(pieces, std::max<int64_t>(1, n) * sizeof(int4), s);
  k_piece_fill<<<(n0 + 255) / 256, 256, 0, s>>>(t, P, cnt, *pieces);
  SPTTN_CUDA(cudaGetLastError());
  dfree(cnt, s);
  return n;
}

__global__ void k_pack_jk(const int32_t* leaf_j, const int32_t* kidx, int64_t n, int2* jk) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e < n) jk[e] = make_int2(leaf_j[e], kidx[e]);
}

void pack_leaf_jk(const DevCsf& D, const int32_t* leaf_j, int2** jk, cudaStream_t s) {
  const int64_t n = D.level_size[2];
  dmalloc(jk, std::max<int64_t>(1, n) * sizeof(int2), s);
  if (n > 0) k_pack_jk<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(leaf_j, D.idx[2], n, *jk);
  SPTTN_CUDA(cudaGetLastError());
}

void launch_tttp3_pieces(const RootOutArgs& a, const int4* pieces, int64_t n_pieces,
                         const int2* leaf_jk, int batch, cudaStream_t s) {
  if (n_pieces == 0) return;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int G = group_lanes_for(a.R);
  const int64_t blocks = std::min<int64_t>((n_pieces + 7) / 8, static_cast<int64_t>(sms) * 8);
  const unsigned nb = static_cast<unsigned>(blocks);
  auto go = [&](auto kern) {
    pin_carveout(kern, 0, 0, 0);  // no shared memory: all of it to L1
    kern<<<nb, kBlock, 0, s>>>(a, pieces, n_pieces, leaf_jk);
  };
#define SPTTN_TTTP_P(GG, UU)                                                                     \
  if (a.vec) go(k_tttp3_piece<GG, UU, true>);                                                    \
  else go(k_tttp3_piece<GG, UU, false>);
  const bool b8 = batch >= 8;
  switch (G) {
    case 1: SPTTN_TTTP_P(1, 1) break;
    case 2: SPTTN_TTTP_P(2, 2) break;
    case 4: SPTTN_TTTP_P(4, 4) break;
    case 8: if (b8) { SPTTN_TTTP_P(8, 8) } else { SPTTN_TTTP_P(8, 4) } break;
    case 16: if (b8) { SPTTN_TTTP_P(16, 8) } else { SPTTN_TTTP_P(16, 4) } break;
    default: if (b8) { SPTTN_TTTP_P(32, 8) } else { SPTTN_TTTP_P(32, 4) } break;
  }
#undef SPTTN_TTTP_P
  SPTTN_CUDA(cudaGetLastError());
}

}  // namespace spttn_dev
