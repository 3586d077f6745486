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
#include <cstdlib>

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
__global__ void __launch_bounds__(kBlock, 3) k_ttmc3(RootOutArgs a) {
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

  int32_t c = static_cast<int32_t>(w * a.chunk);
  const int32_t cend = static_cast<int32_t>(min64(c + a.chunk, a.n_seg));
  const int32_t n_seg = static_cast<int32_t>(a.n_seg);
  int32_t sl = a.item_pos[w];
  int32_t sl_end = a.slice_seg[sl + 1];
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

  const int32_t nnz = t.nlev[2];
  // Software pipeline: the leaf block (<= 32 leaves) of the next group is
  // loaded while the current group's V rows are in flight.
  int32_t pf_base = -1, pf_k = 0;
  double pf_t = 0.0;
  while (c < cend) {
    // segment metadata for a window of 32 segments, one per lane
    const int32_t wb = c;
    const int32_t wend = min(wb + 32, cend);
    const int32_t sb = wb + lane <= n_seg ? __ldg(seg_begin + wb + lane) : nnz;
    const int32_t sb32 = __ldg(seg_begin + min(wb + 32, n_seg));
    const int32_t sn = wb + lane < n_seg ? __ldg(seg_node + wb + lane) : 0;
    while (c < wend) {
      const int32_t lim = min(wend, sl_end);
      const int nvalid = min(4, lim - c);
      const int r0 = c - wb;
      const int rq = r0 + q;
      const bool valid = q < nvalid;
      const int32_t L0 = __shfl_sync(0xffffffffu, sb, r0);
      const int32_t L1a = __shfl_sync(0xffffffffu, sb, min(r0 + nvalid, 31));
      const int32_t L1 = r0 + nvalid < 32 ? L1a : sb32;
      int32_t lb = __shfl_sync(0xffffffffu, sb, min(rq, 31));
      const int32_t lea = __shfl_sync(0xffffffffu, sb, min(rq + 1, 31));
      int32_t le = rq + 1 < 32 ? lea : sb32;
      int32_t j = __shfl_sync(0xffffffffu, sn, min(rq, 31));
      if (!valid) lb = le = j = 0;
      // this group's leaves [L0, L1) (at most 4 * seg_len <= 32), lane-parallel
      int32_t kreg;
      double treg;
      if (pf_base == L0) {
        kreg = pf_k;
        treg = pf_t;
      } else {
        kreg = L0 + lane < L1 ? __ldg(kidx + L0 + lane) : 0;
        treg = L0 + lane < L1 ? __ldg(vals + L0 + lane) : 0.0;
      }
      pf_base = L1;
      pf_k = L1 + lane < nnz ? __ldg(kidx + L1 + lane) : 0;
      pf_t = L1 + lane < nnz ? __ldg(vals + L1 + lane) : 0.0;
      const double2 u = valid ? row2<VECU>(U + static_cast<int64_t>(j) * R, 2 * h, R)
                              : make_double2(0, 0);
      const int n = le - lb;
      const int nmax = warp_max4(n);
      const int base = lb - L0;
      double x0 = 0.0, x1 = 0.0;
      for (int it = 0; it < nmax; it += 4) {
        int32_t kk[4];
        double tt[4];
        double2 vr[4];
#pragma unroll
        for (int u4 = 0; u4 < 4; ++u4) {
          const int src = (base + it + u4) & 31;
          kk[u4] = __shfl_sync(0xffffffffu, kreg, src);
          tt[u4] = __shfl_sync(0xffffffffu, treg, src);
        }
#pragma unroll
        for (int u4 = 0; u4 < 4; ++u4)
          vr[u4] = it + u4 < n ? row2<VECV>(V + static_cast<int64_t>(kk[u4]) * S, 2 * h, S)
                               : make_double2(0, 0);
#pragma unroll
        for (int u4 = 0; u4 < 4; ++u4) {
          const double tv = it + u4 < n ? tt[u4] : 0.0;
          x0 = fma(tv, vr[u4].x, x0);  // X[s] += t * V[k,s]
          x1 = fma(tv, vr[u4].y, x1);
        }
      }
      // rank-1 updates of 4 segments: D[mt][nt] += A[mt] (8x4) * B[nt] (4x8)
      dmma_8x8x4(acc[0], acc[1], u.x, x0);
      dmma_8x8x4(acc[2], acc[3], u.x, x1);
      dmma_8x8x4(acc[4], acc[5], u.y, x0);
      dmma_8x8x4(acc[6], acc[7], u.y, x1);
      pending = true;
      c += nvalid;
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
  }
  if (pending) flush(head ? 0 : 1);
}

// Stream-staged variant (mode 4). The warp's CSF stream — segment metadata
// and the leaves' coordinates / values — is copied into a per-warp shared
// memory ring with cp.async (LDGSTS) one 32-segment window ahead (metadata
// two windows ahead, since a window's leaf range comes from its metadata),
// so HBM latency never sits on the critical path; the only round trip left
// per 4-segment step is the factor-row gather (L1/L2 resident rows).
constexpr int kWin = 32;
constexpr int kWinLeaves = kWin * 4;  // seg_len <= 4

struct Stage3 {
  int32_t sb[3][kWin + 1];
  int32_t sn[3][kWin];
  int32_t kk[2][kWinLeaves];
  double tv[2][kWinLeaves];
};

template <bool VECU, bool VECV>
__global__ void __launch_bounds__(kBlock, 3) k_ttmc3s(RootOutArgs a) {
  __shared__ Stage3 stage[kBlock / 32];
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * kBlock + threadIdx.x) / 32;
  if (w >= a.n_items) return;  // warp-uniform
  Stage3& S = stage[threadIdx.x / 32];
  const int lane = threadIdx.x & 31;
  const int q = lane & 3;
  const int h = lane >> 2;
  const int R = a.R, S_ = a.S;
  const CsfView& t = a.t;
  const double* __restrict__ U = a.f[1];
  const double* __restrict__ V = a.f[2];
  const int32_t* __restrict__ kidx = t.idx[2];
  const double* __restrict__ vals = t.vals;
  const int32_t* __restrict__ seg_begin = a.seg_begin;
  const int32_t* __restrict__ seg_node = a.seg_node;
  const int32_t* __restrict__ slice_seg = a.slice_seg;

  const int32_t cbeg = static_cast<int32_t>(w * a.chunk);
  const int32_t cend = static_cast<int32_t>(min64(cbeg + a.chunk, a.n_seg));
  int32_t sl = a.item_pos[w];
  int32_t sl_end = slice_seg[sl + 1];
  bool head = slice_seg[sl] < cbeg;
  int32_t row = t.idx[0][sl];
  // one-slice lookahead so slice switches do not wait on global loads
  int32_t nx_end = sl + 2 <= t.nlev[0] ? __ldg(slice_seg + sl + 2) : 0;
  int32_t nx_row = sl + 1 < t.nlev[0] ? __ldg(t.idx[0] + sl + 1) : 0;
  bool pending = false;
  double acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.0;

  auto flush = [&](int slot) {
    double* dst = slot < 0 ? a.out + static_cast<int64_t>(row) * R * S_
                           : a.part + (w * 2 + slot) * static_cast<int64_t>(R) * S_;
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = 2 * h + mt;
          const int s = 2 * (2 * q + e) + nt;
          if (r < R && s < S_) dst[r * S_ + s] = acc[(mt * 2 + nt) * 2 + e];
        }
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.0;
  };
  auto issue_meta = [&](int buf, int32_t ws) {
    const int32_t nsw = min(ws + kWin, cend) - ws;
    if (lane <= nsw) cp_async4(&S.sb[buf][lane], seg_begin + ws + lane);
    if (lane == 0 && nsw == kWin) cp_async4(&S.sb[buf][kWin], seg_begin + ws + kWin);
    if (lane < nsw) cp_async4(&S.sn[buf][lane], seg_node + ws + lane);
  };
  auto issue_leaves = [&](int lbuf, int mbuf, int32_t ws) {
    const int32_t nsw = min(ws + kWin, cend) - ws;
    const int32_t L0 = S.sb[mbuf][0];
    const int32_t nl = S.sb[mbuf][nsw] - L0;
    for (int32_t i = lane; i < nl; i += 32) {
      cp_async4(&S.kk[lbuf][i], kidx + L0 + i);
      cp_async8(&S.tv[lbuf][i], vals + L0 + i);
    }
  };

  const int32_t nwin = (cend - cbeg + kWin - 1) / kWin;
  issue_meta(0, cbeg);
  cp_async_commit();
  cp_async_wait<0>();
  __syncwarp();
  issue_leaves(0, 0, cbeg);
  if (nwin > 1) issue_meta(1, cbeg + kWin);
  cp_async_commit();
  int32_t cs = cbeg;
  for (int32_t win = 0; win < nwin; ++win) {
    cp_async_wait<0>();
    __syncwarp();
    const int mb = win % 3, lbf = win & 1;
    const int32_t ws = cbeg + win * kWin;
    if (win + 1 < nwin) issue_leaves((win + 1) & 1, (win + 1) % 3, ws + kWin);
    if (win + 2 < nwin) issue_meta((win + 2) % 3, ws + 2 * kWin);
    cp_async_commit();
    const int32_t we = min(ws + kWin, cend);
    const int32_t L0 = S.sb[mb][0];
    while (cs < we) {
      const int32_t lim = min(we, sl_end);
      const int nv = min(4, lim - cs);
      const int r = cs - ws + q;
      const bool valid = q < nv;
      int32_t lb = 0, n = 0, j = 0;
      if (valid) {
        lb = S.sb[mb][r] - L0;
        n = S.sb[mb][r + 1] - S.sb[mb][r];
        j = S.sn[mb][r];
      }
      double2 vr[4];
      double tt[4];
#pragma unroll
      for (int it = 0; it < 4; ++it) {
        const int32_t k = it < n ? S.kk[lbf][lb + it] : 0;
        tt[it] = it < n ? S.tv[lbf][lb + it] : 0.0;
        vr[it] = it < n ? row2<VECV>(V + static_cast<int64_t>(k) * S_, 2 * h, S_)
                        : make_double2(0, 0);
      }
      const double2 u = valid ? row2<VECU>(U + static_cast<int64_t>(j) * R, 2 * h, R)
                              : make_double2(0, 0);
      double x0 = 0.0, x1 = 0.0;
#pragma unroll
      for (int it = 0; it < 4; ++it) {
        x0 = fma(tt[it], vr[it].x, x0);  // X[s] += t * V[k,s]
        x1 = fma(tt[it], vr[it].y, x1);
      }
      dmma_8x8x4(acc[0], acc[1], u.x, x0);
      dmma_8x8x4(acc[2], acc[3], u.x, x1);
      dmma_8x8x4(acc[4], acc[5], u.y, x0);
      dmma_8x8x4(acc[6], acc[7], u.y, x1);
      pending = true;
      cs += nv;
      if (cs == sl_end) {
        flush(head ? 0 : -1);
        pending = false;
        head = false;
        if (cs < cend) {
          ++sl;
          sl_end = nx_end;
          row = nx_row;
          nx_end = sl + 2 <= t.nlev[0] ? __ldg(slice_seg + sl + 2) : 0;
          nx_row = sl + 1 < t.nlev[0] ? __ldg(t.idx[0] + sl + 1) : 0;
        }
      }
    }
    __syncwarp();
  }
  if (pending) flush(head ? 0 : 1);
}

// Packed variant (mode 6): the warp walks length-sorted groups of 8
// equal-length segments (pack.cu), so each of a group's n V-row gathers and
// its U-row gather is a full 8-row 256-bit load with a warp-uniform trip
// count. Group headers are prefetched two groups ahead and the leaf
// coordinates of the next group one group ahead. Lane L = (q = L%4,
// c4 = (L/4)%4, ch = L/16) gathers slot 4*ch + q, columns [4*c4, 4*c4+4) of
// its rows (fragment order), one xor-16 exchange builds both K-chunks.
template <bool VECU, bool VECV>
__global__ void __launch_bounds__(kBlock, 2) k_ttmc3pk(RootOutArgs a) {
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * kBlock + threadIdx.x) / 32;
  if (w >= a.n_items) return;  // warp-uniform
  const int lane = threadIdx.x & 31;
  const int q = lane & 3;
  const int c4 = (lane >> 2) & 3;
  const int ch = lane >> 4;
  const int slot = ch * 4 + q;
  const int h = lane >> 2;
  const int R = a.R, S_ = a.S;
  const CsfView& t = a.t;
  const double* __restrict__ U = a.f[1];
  const double* __restrict__ V = a.f[2];
  const int4* __restrict__ hdr = a.grp_hdr;
  const int32_t* __restrict__ gnode = a.grp_node;
  const int32_t* __restrict__ pk = a.pk;
  const double* __restrict__ pv = a.pv;
  const int32_t* __restrict__ slice_grp = a.slice_grp;
  const int32_t ng = static_cast<int32_t>(a.n_groups);

  const int32_t cbeg = static_cast<int32_t>(w * a.chunk);
  const int32_t cend = static_cast<int32_t>(min64(cbeg + a.chunk, a.n_groups));
  int32_t sl = a.item_pos[w];
  int32_t sl_end = slice_grp[sl + 1];
  bool head = slice_grp[sl] < cbeg;
  int32_t row = t.idx[0][sl];
  int32_t nx_end = sl + 2 <= t.nlev[0] ? __ldg(slice_grp + sl + 2) : 0;
  int32_t nx_row = sl + 1 < t.nlev[0] ? __ldg(t.idx[0] + sl + 1) : 0;
  bool pending = false;
  double acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.0;

  auto flush = [&](int dslot) {
    double* dst = dslot < 0 ? a.out + static_cast<int64_t>(row) * R * S_
                            : a.part + (w * 2 + dslot) * static_cast<int64_t>(R) * S_;
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = 4 * (h & 3) + 2 * (h >> 2) + mt;
          const int n = 2 * q + e;
          const int s = 4 * (n & 3) + 2 * (n >> 2) + nt;
          if (r < R && s < S_) dst[r * S_ + s] = acc[(mt * 2 + nt) * 2 + e];
        }
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.0;
  };
  auto load_hdr = [&](int32_t g) { return g < ng ? __ldg(hdr + g) : make_int4(0, 0, 0, 0); };
  auto load_k = [&](const int4& hh, int32_t* k) {
#pragma unroll
    for (int it = 0; it < 4; ++it) k[it] = it < hh.y ? __ldg(pk + hh.x + it * kPackSlots + slot) : 0;
  };

  int4 hc = load_hdr(cbeg), hn = load_hdr(cbeg + 1);
  int32_t jc = cbeg < ng ? __ldg(gnode + static_cast<int64_t>(cbeg) * kPackSlots + slot) : 0;
  int32_t kc[4];
  load_k(hc, kc);
  for (int32_t g = cbeg; g < cend; ++g) {
    const int n = hc.y;  // warp-uniform segment length of this group
    double4 vr[4];
    double tt[4];
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      if (it < n) {
        tt[it] = __ldg(pv + hc.x + it * kPackSlots + slot);
        vr[it] = row4<VECV>(V + static_cast<int64_t>(kc[it]) * S_, 4 * c4, S_);
      } else {
        tt[it] = 0.0;
        vr[it] = make_double4(0, 0, 0, 0);
      }
    }
    const double4 ur = row4<VECU>(U + static_cast<int64_t>(jc) * R, 4 * c4, R);
    // prefetch: header two groups ahead, coordinates of the next group
    const int4 hnn = load_hdr(g + 2);
    const int32_t jn = g + 1 < ng ? __ldg(gnode + static_cast<int64_t>(g + 1) * kPackSlots + slot) : 0;
    int32_t kn[4];
    load_k(hn, kn);
    double4 x = make_double4(0, 0, 0, 0);
#pragma unroll
    for (int it = 0; it < 4; ++it) fma4(x, tt[it], vr[it]);  // X[s] += t * V[k,s]
    const double sx0 = ch == 0 ? x.z : x.x, sx1 = ch == 0 ? x.w : x.y;
    const double su0 = ch == 0 ? ur.z : ur.x, su1 = ch == 0 ? ur.w : ur.y;
    const double rx0 = __shfl_xor_sync(0xffffffffu, sx0, 16);
    const double rx1 = __shfl_xor_sync(0xffffffffu, sx1, 16);
    const double ru0 = __shfl_xor_sync(0xffffffffu, su0, 16);
    const double ru1 = __shfl_xor_sync(0xffffffffu, su1, 16);
    const double bA0 = ch == 0 ? x.x : rx0, bA1 = ch == 0 ? x.y : rx1;
    const double bB0 = ch == 0 ? rx0 : x.z, bB1 = ch == 0 ? rx1 : x.w;
    const double aA0 = ch == 0 ? ur.x : ru0, aA1 = ch == 0 ? ur.y : ru1;
    const double aB0 = ch == 0 ? ru0 : ur.z, aB1 = ch == 0 ? ru1 : ur.w;
    dmma_8x8x4(acc[0], acc[1], aA0, bA0);
    dmma_8x8x4(acc[2], acc[3], aA0, bA1);
    dmma_8x8x4(acc[4], acc[5], aA1, bA0);
    dmma_8x8x4(acc[6], acc[7], aA1, bA1);
    dmma_8x8x4(acc[0], acc[1], aB0, bB0);
    dmma_8x8x4(acc[2], acc[3], aB0, bB1);
    dmma_8x8x4(acc[4], acc[5], aB1, bB0);
    dmma_8x8x4(acc[6], acc[7], aB1, bB1);
    pending = true;
    hc = hn;
    hn = hnn;
    jc = jn;
#pragma unroll
    for (int it = 0; it < 4; ++it) kc[it] = kn[it];
    if (g + 1 == sl_end) {
      flush(head ? 0 : -1);
      pending = false;
      head = false;
      if (g + 1 < cend) {
        ++sl;
        sl_end = nx_end;
        row = nx_row;
        nx_end = sl + 2 <= t.nlev[0] ? __ldg(slice_grp + sl + 2) : 0;
        nx_row = sl + 1 < t.nlev[0] ? __ldg(t.idx[0] + sl + 1) : 0;
      }
    }
  }
  if (pending) flush(head ? 0 : 1);
}

// Packed + staged variant: packed groups (full 8-row gathers) whose stream
// (headers, slot coordinates, interleaved leaf coordinates / values) is
// copied into a per-warp shared-memory ring by cp.async kGW groups at a time,
// headers two windows ahead and leaf data one window ahead, so only the
// factor-row gathers remain on the critical path and registers hold no
// prefetch state.
constexpr int kGW = 4;                             // groups per window
constexpr int kGWLeaves = kGW * kPackSlots * 4;    // leaves per window (len <= 4)

struct StageP {
  alignas(16) int4 hdr[3][kGW];
  int32_t node[3][kGW * kPackSlots];
  int32_t kk[2][kGWLeaves];
  double tv[2][kGWLeaves];
};

template <bool VECU, bool VECV>
__global__ void __launch_bounds__(kBlock, 3) k_ttmc3ps(RootOutArgs a) {
  __shared__ StageP stage[kBlock / 32];
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * kBlock + threadIdx.x) / 32;
  if (w >= a.n_items) return;  // warp-uniform
  StageP& S = stage[threadIdx.x / 32];
  const int lane = threadIdx.x & 31;
  const int q = lane & 3;
  const int c4 = (lane >> 2) & 3;
  const int ch = lane >> 4;
  const int slot = ch * 4 + q;
  const int h = lane >> 2;
  const int R = a.R, S_ = a.S;
  const CsfView& t = a.t;
  const double* __restrict__ U = a.f[1];
  const double* __restrict__ V = a.f[2];
  const int32_t* __restrict__ slice_grp = a.slice_grp;

  const int32_t cbeg = static_cast<int32_t>(w * a.chunk);
  const int32_t cend = static_cast<int32_t>(min64(cbeg + a.chunk, a.n_groups));
  int32_t sl = a.item_pos[w];
  int32_t sl_end = slice_grp[sl + 1];
  bool head = slice_grp[sl] < cbeg;
  int32_t row = t.idx[0][sl];
  int32_t nx_end = sl + 2 <= t.nlev[0] ? __ldg(slice_grp + sl + 2) : 0;
  int32_t nx_row = sl + 1 < t.nlev[0] ? __ldg(t.idx[0] + sl + 1) : 0;
  bool pending = false;
  double acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.0;

  auto flush = [&](int dslot) {
    double* dst = dslot < 0 ? a.out + static_cast<int64_t>(row) * R * S_
                            : a.part + (w * 2 + dslot) * static_cast<int64_t>(R) * S_;
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = 4 * (h & 3) + 2 * (h >> 2) + mt;
          const int n = 2 * q + e;
          const int s = 4 * (n & 3) + 2 * (n >> 2) + nt;
          if (r < R && s < S_) dst[r * S_ + s] = acc[(mt * 2 + nt) * 2 + e];
        }
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.0;
  };
  // window w covers groups [gs, min(gs + kGW, cend))
  auto issue_meta = [&](int buf, int32_t gs) {
    const int32_t nw = min(gs + kGW, cend) - gs;
    if (lane < nw) cp_async16_cg(&S.hdr[buf][lane], a.grp_hdr + gs + lane, 16);
    for (int i = lane; i < nw * kPackSlots; i += 32)
      cp_async4(&S.node[buf][i], a.grp_node + static_cast<int64_t>(gs) * kPackSlots + i);
  };
  auto issue_leaves = [&](int lbuf, int mbuf, int32_t gs) {
    const int32_t nw = min(gs + kGW, cend) - gs;
    const int32_t L0 = S.hdr[mbuf][0].x;
    const int32_t L1 = S.hdr[mbuf][nw - 1].x + kPackSlots * S.hdr[mbuf][nw - 1].y;
    for (int32_t i = lane; i < L1 - L0; i += 32) {
      cp_async4(&S.kk[lbuf][i], a.pk + L0 + i);
      cp_async8(&S.tv[lbuf][i], a.pv + L0 + i);
    }
  };

  const int32_t nwin = (cend - cbeg + kGW - 1) / kGW;
  issue_meta(0, cbeg);
  cp_async_commit();
  cp_async_wait<0>();
  __syncwarp();
  issue_leaves(0, 0, cbeg);
  if (nwin > 1) issue_meta(1, cbeg + kGW);
  cp_async_commit();
  for (int32_t win = 0; win < nwin; ++win) {
    cp_async_wait<0>();
    __syncwarp();
    const int mb = win % 3, lbf = win & 1;
    const int32_t gs = cbeg + win * kGW;
    if (win + 1 < nwin) issue_leaves((win + 1) & 1, (win + 1) % 3, gs + kGW);
    if (win + 2 < nwin) issue_meta((win + 2) % 3, gs + 2 * kGW);
    cp_async_commit();
    const int32_t ge = min(gs + kGW, cend);
    const int32_t L0 = S.hdr[mb][0].x;
    for (int32_t g = gs; g < ge; ++g) {
      const int4 hh = S.hdr[mb][g - gs];
      const int n = hh.y;  // warp-uniform
      const int32_t lbase = hh.x - L0 + slot;
      // straight-line: read every index first, then issue all gathers
      const int32_t j = S.node[mb][(g - gs) * kPackSlots + slot];
      int32_t kk[4];
      double tt[4];
#pragma unroll
      for (int it = 0; it < 4; ++it) {
        kk[it] = S.kk[lbf][lbase + it * kPackSlots];
        tt[it] = it < n ? S.tv[lbf][lbase + it * kPackSlots] : 0.0;
      }
      const double4 ur = row4<VECU>(U + static_cast<int64_t>(j) * R, 4 * c4, R);
      double4 vr[4];
#pragma unroll
      for (int it = 0; it < 4; ++it) {
        if (VECV) {
          vr[it] = ld256_if(V + static_cast<int64_t>(kk[it]) * S_ + 4 * c4, it < n && 4 * c4 < S_);
        } else {
          vr[it] = it < n ? row4<false>(V + static_cast<int64_t>(kk[it]) * S_, 4 * c4, S_)
                          : make_double4(0, 0, 0, 0);
        }
      }
      double4 x = make_double4(0, 0, 0, 0);
#pragma unroll
      for (int it = 0; it < 4; ++it) fma4(x, tt[it], vr[it]);  // X[s] += t * V[k,s]
      const double sx0 = ch == 0 ? x.z : x.x, sx1 = ch == 0 ? x.w : x.y;
      const double su0 = ch == 0 ? ur.z : ur.x, su1 = ch == 0 ? ur.w : ur.y;
      const double rx0 = __shfl_xor_sync(0xffffffffu, sx0, 16);
      const double rx1 = __shfl_xor_sync(0xffffffffu, sx1, 16);
      const double ru0 = __shfl_xor_sync(0xffffffffu, su0, 16);
      const double ru1 = __shfl_xor_sync(0xffffffffu, su1, 16);
      const double bA0 = ch == 0 ? x.x : rx0, bA1 = ch == 0 ? x.y : rx1;
      const double bB0 = ch == 0 ? rx0 : x.z, bB1 = ch == 0 ? rx1 : x.w;
      const double aA0 = ch == 0 ? ur.x : ru0, aA1 = ch == 0 ? ur.y : ru1;
      const double aB0 = ch == 0 ? ru0 : ur.z, aB1 = ch == 0 ? ru1 : ur.w;
      dmma_8x8x4(acc[0], acc[1], aA0, bA0);
      dmma_8x8x4(acc[2], acc[3], aA0, bA1);
      dmma_8x8x4(acc[4], acc[5], aA1, bA0);
      dmma_8x8x4(acc[6], acc[7], aA1, bA1);
      dmma_8x8x4(acc[0], acc[1], aB0, bB0);
      dmma_8x8x4(acc[2], acc[3], aB0, bB1);
      dmma_8x8x4(acc[4], acc[5], aB1, bB0);
      dmma_8x8x4(acc[6], acc[7], aB1, bB1);
      pending = true;
      if (g + 1 == sl_end) {
        flush(head ? 0 : -1);
        pending = false;
        head = false;
        if (g + 1 < cend) {
          ++sl;
          sl_end = nx_end;
          row = nx_row;
          nx_end = sl + 2 <= t.nlev[0] ? __ldg(slice_grp + sl + 2) : 0;
          nx_row = sl + 1 < t.nlev[0] ? __ldg(t.idx[0] + sl + 1) : 0;
        }
      }
    }
    __syncwarp();
  }
  if (pending) flush(head ? 0 : 1);
}

// TMA-staged stream window: group headers, slot coordinates, interleaved leaf
// coordinates and values — all contiguous and 32-byte aligned in the packed
// layout — staged by lane 0 with one bulk copy per array, completing on a
// per-stage mbarrier (instead of one LDGSTS per lane and element).
struct StageT {
  alignas(16) int4 hdr[3][kGW];
  alignas(16) int32_t node[3][kGW * kPackSlots];
  alignas(16) int32_t kk[2][kGWLeaves];
  alignas(16) double tv[2][kGWLeaves];
  uint64_t mbar_meta[3];
  uint64_t mbar_leaf[2];
};

// Packed + TMA-staged + row-contiguous gathers (TTMc-3 default).
//
// The m8n8k4 fragment puts the contracted (segment) index at lane%4, so a
// gather made directly in fragment layout has 4 consecutive lanes reading 4
// different factor rows. ncu: such a 256-bit gather costs ~32 L1 data-pipe
// wavefronts (one per 32-byte piece) instead of 8 (one per 128-byte row) —
// every earlier variant sat at ~78 % of the data-pipe peak with 4x inflated
// gather wavefronts. Here lane L gathers row slot = L/4, columns 4(L%4)..+3
// (4 consecutive lanes per row), computes its X quad, and the X and U quads of
// the group are transposed into fragment layout through a per-warp shared
// tile: 16 B-aligned stores, column swizzle col ^ 4*(slot%4) ^ 2*(slot%2) so
// both the 64-bit fragment reads and the 128-bit quad stores are
// conflict-free. Tiles are double-buffered by
// group parity, so one __syncwarp per group orders stores before loads.
struct StageQ {
  alignas(16) double xs[2][kPackSlots * 16];
  alignas(16) double us[2][kPackSlots * 16];
};

constexpr size_t kPqSmem = (sizeof(StageT) + sizeof(StageQ)) * (kBlock / 32);

template <bool VECU, bool VECV>
__global__ void __launch_bounds__(kBlock, 3) k_ttmc3pq(RootOutArgs a) {
  grid_launch_dependents();
  extern __shared__ __align__(16) unsigned char pq_smem[];  // kPqSmem bytes
  StageT* stage = reinterpret_cast<StageT*>(pq_smem);
  StageQ* tiles = reinterpret_cast<StageQ*>(pq_smem + sizeof(StageT) * (kBlock / 32));
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * kBlock + threadIdx.x) / 32;
  if (w >= a.n_items) return;  // warp-uniform
  StageT& S = stage[threadIdx.x / 32];
  StageQ& Q = tiles[threadIdx.x / 32];
  const int lane = threadIdx.x & 31;
  // gather role: row slot gs, column quad gc
  const int gs = lane >> 2, gc = lane & 3;
  // fragment role: K index fq (segment within a 4-chunk), M/N index fh
  const int fq = lane & 3, fh = lane >> 2;
  const int R = a.R, S_ = a.S;
  const CsfView& t = a.t;
  const double* __restrict__ U = a.f[1];
  const double* __restrict__ V = a.f[2];
  const int32_t* __restrict__ slice_grp = a.slice_grp;

  const int32_t cbeg =
      uni(a.item_unit ? __ldg(a.item_unit + w) : static_cast<int32_t>(w * a.chunk));
  const int32_t cend = uni(a.item_unit ? __ldg(a.item_unit + w + 1)
                                       : static_cast<int32_t>(min64(cbeg + a.chunk, a.n_groups)));
  int32_t sl = a.item_pos[w];
  int32_t sl_end = slice_grp[sl + 1];
  bool head = slice_grp[sl] < cbeg;
  int32_t row = t.idx[0][sl];
  int32_t nx_end = sl + 2 <= t.nlev[0] ? __ldg(slice_grp + sl + 2) : 0;
  int32_t nx_row = sl + 1 < t.nlev[0] ? __ldg(t.idx[0] + sl + 1) : 0;
  bool pending = false;
  double acc[8];  // tile (mt, nt) element e at acc[(mt*2+nt)*2+e]
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.0;

  auto flush = [&](int dslot) {
    double* dst = dslot < 0 ? a.out + static_cast<int64_t>(row) * R * S_
                            : a.part + (w * 2 + dslot) * static_cast<int64_t>(R) * S_;
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = 8 * mt + fh;
          const int s = 8 * nt + 2 * fq + e;
          if (r < R && s < S_) dst[r * S_ + s] = acc[(mt * 2 + nt) * 2 + e];
        }
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.0;
  };
  auto issue_meta = [&](int32_t wi) {
    const int32_t g0 = cbeg + wi * kGW;
    const int32_t nw = min(g0 + kGW, cend) - g0;
    const int b = wi % 3;
    const unsigned hb = nw * sizeof(int4), nb = nw * kPackSlots * sizeof(int32_t);
    fence_proxy_async();
    expect_tx_elect(&S.mbar_meta[b], hb + nb);
    bulk_g2s_elect(&S.hdr[b][0], a.grp_hdr + g0, hb, &S.mbar_meta[b]);
    bulk_g2s_elect(&S.node[b][0], a.grp_node + static_cast<int64_t>(g0) * kPackSlots, nb, &S.mbar_meta[b]);
  };
  auto issue_leaves = [&](int32_t wi) {
    const int32_t g0 = cbeg + wi * kGW;
    const int32_t nw = min(g0 + kGW, cend) - g0;
    const int b = wi % 3, lb = wi & 1;
    mbar_wait(&S.mbar_meta[b], (wi / 3) & 1);
    const int32_t L0 = uni(S.hdr[b][0].x);
    const int32_t L1 = uni(S.hdr[b][nw - 1].x + kPackSlots * S.hdr[b][nw - 1].y);
    const unsigned n = static_cast<unsigned>(L1 - L0);
    fence_proxy_async();
    expect_tx_elect(&S.mbar_leaf[lb], n * 12u);
    bulk_g2s_elect(&S.kk[lb][0], a.pk + L0, n * 4u, &S.mbar_leaf[lb]);
    bulk_g2s_elect(&S.tv[lb][0], a.pv + L0, n * 8u, &S.mbar_leaf[lb]);
  };

  // swizzled tile: element (slot, col) at slot*16 + (col ^ 4*(slot&3) ^ 2*(slot&1))
  const int st_off = gs * 16 + ((4 * gc) ^ (4 * (gs & 3)));
  const int o_lo = st_off + 2 * (gs & 1), o_hi = st_off + 2 - 2 * (gs & 1);
  int par = 0;

  const int32_t nwin = (cend - cbeg + kGW - 1) / kGW;
  if (lane == 0) {
    for (int b = 0; b < 3; ++b) mbar_init(&S.mbar_meta[b], 1);
    for (int b = 0; b < 2; ++b) mbar_init(&S.mbar_leaf[b], 1);
    mbar_init_fence();
  }
  __syncwarp();
  if (nwin > 0) {  // warp-collective issue (elected lane), uniform operands
    issue_meta(0);
    if (nwin > 1) issue_meta(1);
    issue_leaves(0);
  }
  for (int32_t win = 0; win < nwin; ++win) {
    const int mb = win % 3, lbf = win & 1;
    if (win + 1 < nwin) issue_leaves(win + 1);
    if (win + 2 < nwin) issue_meta(win + 2);
    mbar_wait(&S.mbar_meta[mb], (win / 3) & 1);
    mbar_wait(&S.mbar_leaf[lbf], (win / 2) & 1);
    const int32_t g0 = cbeg + win * kGW;
    const int32_t ge = min(g0 + kGW, cend);
    const int32_t L0 = S.hdr[mb][0].x;
    for (int32_t g = g0; g < ge; ++g) {
      const int4 hh = S.hdr[mb][g - g0];
      const int n = hh.y;  // warp-uniform
      const int32_t lbase = hh.x - L0 + gs;
      const int32_t j = S.node[mb][(g - g0) * kPackSlots + gs];
      int32_t kk[4];
      double tt[4];
#pragma unroll
      for (int it = 0; it < 4; ++it) {
        kk[it] = it < n ? S.kk[lbf][lbase + it * kPackSlots] : 0;
        tt[it] = it < n ? S.tv[lbf][lbase + it * kPackSlots] : 0.0;
      }
      const double4 ur = row4<VECU>(U + static_cast<int64_t>(j) * R, 4 * gc, R);
      double4 vr[4];
#pragma unroll
      for (int it = 0; it < 4; ++it) {
        if (VECV) {
          vr[it] = ld256_if(V + static_cast<int64_t>(kk[it]) * S_ + 4 * gc, it < n && 4 * gc < S_);
        } else {
          vr[it] = it < n ? row4<false>(V + static_cast<int64_t>(kk[it]) * S_, 4 * gc, S_)
                          : make_double4(0, 0, 0, 0);
        }
      }
      double4 x = make_double4(0, 0, 0, 0);
#pragma unroll
      for (int it = 0; it < 4; ++it) fma4(x, tt[it], vr[it]);  // X[s] += t * V[k,s]
      // transpose X and U quads into fragment layout through the tile
      double* xs = Q.xs[par];
      double* us = Q.us[par];
      *reinterpret_cast<double2*>(xs + o_lo) = make_double2(x.x, x.y);
      *reinterpret_cast<double2*>(us + o_lo) = make_double2(ur.x, ur.y);
      *reinterpret_cast<double2*>(xs + o_hi) = make_double2(x.z, x.w);
      *reinterpret_cast<double2*>(us + o_hi) = make_double2(ur.z, ur.w);
      __syncwarp();
      double af[2][2], bf[2][2];  // [K chunk][m / n tile]
#pragma unroll
      for (int kc = 0; kc < 2; ++kc) {
        const int seg = 4 * kc + fq;
        const int sw = 4 * (seg & 3) ^ 2 * (seg & 1);
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          af[kc][mt] = us[seg * 16 + ((8 * mt + fh) ^ sw)];
          bf[kc][mt] = xs[seg * 16 + ((8 * mt + fh) ^ sw)];
        }
      }
#pragma unroll
      for (int kc = 0; kc < 2; ++kc)
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int nt = 0; nt < 2; ++nt)
            dmma_8x8x4(acc[(mt * 2 + nt) * 2], acc[(mt * 2 + nt) * 2 + 1], af[kc][mt], bf[kc][nt]);
      par ^= 1;
      pending = true;
      if (g + 1 == sl_end) {
        flush(head ? 0 : -1);
        pending = false;
        head = false;
        if (g + 1 < cend) {
          ++sl;
          sl_end = nx_end;
          row = nx_row;
          nx_end = sl + 2 <= t.nlev[0] ? __ldg(slice_grp + sl + 2) : 0;
          nx_row = sl + 1 < t.nlev[0] ? __ldg(t.idx[0] + sl + 1) : 0;
        }
      }
    }
    __syncwarp();  // stage buffers of this window are free after this point
  }
  if (pending) flush(head ? 0 : 1);
}

// TTMc-4, packed form (default). Units are (i,j) fiber pieces of <= 4 LEAVES
// (the (i,j,k) level holds ~1 leaf at the BASELINE shape, so X[t] = v*W[l,t]
// per leaf and Y[s,t] += V[k,s] * X[t] regroups the reference's per-(i,j,k)
// sums), length-sorted into groups of 8 (pack.cu) with the leaf's level-3 and
// level-2 coordinates interleaved. Lane L = (q = L%4, h = L/4) owns segments
// q and q+4 (the two DMMA K-chunks) and holds Y[seg][s = 0..7][t = h] — which
// is already the B fragment of tile s for the last stage, eight DMMA per
// K-chunk: Out_i(R x ST) += U_J^T Y_J. Gathers: the V row is read by the 8
// lanes of a slot (broadcast, 2 x 256-bit), W[l, h] per lane (8 rows per
// 64-bit instruction), all issued in straight-line code.
template <bool VECV>
__global__ void __launch_bounds__(kBlock, 2) k_ttmc4pk(RootOutArgs a) {
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * kBlock + threadIdx.x) / 32;
  if (w >= a.n_items) return;  // warp-uniform
  const int lane = threadIdx.x & 31;
  const int q = lane & 3;
  const int h = lane >> 2;
  const int R = a.R, S = a.S, T = a.T;
  const CsfView& t = a.t;
  const double* __restrict__ U = a.f[1];
  const double* __restrict__ V = a.f[2];
  const double* __restrict__ W = a.f[3];
  const int4* __restrict__ hdr = a.grp_hdr;
  const int32_t* __restrict__ gnode = a.grp_node;
  const int32_t* __restrict__ pl = a.pk;
  const int32_t* __restrict__ pkk = a.pk2;
  const double* __restrict__ pv = a.pv;
  const int32_t* __restrict__ slice_grp = a.slice_grp;
  const int64_t tile = static_cast<int64_t>(R) * S * T;

  const int32_t cbeg = static_cast<int32_t>(w * a.chunk);
  const int32_t cend = static_cast<int32_t>(min64(cbeg + a.chunk, a.n_groups));
  int32_t sl = a.item_pos[w];
  int32_t sl_end = slice_grp[sl + 1];
  bool head = slice_grp[sl] < cbeg;
  int32_t row = t.idx[0][sl];
  bool pending = false;
  double acc[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) acc[e] = 0.0;

  auto flush = [&](int dslot) {
    double* dst = dslot < 0 ? a.out + static_cast<int64_t>(row) * tile
                            : a.part + (w * 2 + dslot) * tile;
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
  auto vrow = [&](int32_t k, bool on, double* vr) {
    const double* p = V + static_cast<int64_t>(k) * S;
    if (VECV) {
      const double4 a0 = ld256_if(p, on), a1 = ld256_if(p + 4, on);
      vr[0] = a0.x; vr[1] = a0.y; vr[2] = a0.z; vr[3] = a0.w;
      vr[4] = a1.x; vr[5] = a1.y; vr[6] = a1.z; vr[7] = a1.w;
    } else {
#pragma unroll
      for (int s = 0; s < 8; ++s) vr[s] = (on && s < S) ? __ldg(p + s) : 0.0;
    }
  };

  for (int32_t g = cbeg; g < cend; ++g) {
    const int4 hh = __ldg(hdr + g);
    const int n = hh.y;  // warp-uniform leaves per segment
    const int64_t gs = static_cast<int64_t>(g) * kPackSlots;
    const int32_t jA = __ldg(gnode + gs + q), jB = __ldg(gnode + gs + 4 + q);
    const double uA = h < R ? __ldg(U + static_cast<int64_t>(jA) * R + h) : 0.0;
    const double uB = h < R ? __ldg(U + static_cast<int64_t>(jB) * R + h) : 0.0;
    double YA[8], YB[8];
#pragma unroll
    for (int s = 0; s < 8; ++s) YA[s] = YB[s] = 0.0;
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      if (it < n) {  // warp-uniform
        const int32_t eA = hh.x + it * kPackSlots + q, eB = eA + 4;
        const int32_t lA = __ldg(pl + eA), lB = __ldg(pl + eB);
        const int32_t kA = __ldg(pkk + eA), kB = __ldg(pkk + eB);
        const double vA = __ldg(pv + eA), vB = __ldg(pv + eB);
        const double wA = h < T ? __ldg(W + static_cast<int64_t>(lA) * T + h) : 0.0;
        const double wB = h < T ? __ldg(W + static_cast<int64_t>(lB) * T + h) : 0.0;
        double vrA[8], vrB[8];
        vrow(kA, true, vrA);
        vrow(kB, true, vrB);
        const double xA = vA * wA, xB = vB * wB;  // X[t] = t_ijkl * W[l,t]
#pragma unroll
        for (int s = 0; s < 8; ++s) {
          YA[s] = fma(vrA[s], xA, YA[s]);  // Y[s,t] += V[k,s] * X[t]
          YB[s] = fma(vrB[s], xB, YB[s]);
        }
      }
    }
    // Out_i[r, s, t] += U[j, r] * Y[s, t] for both K-chunks
#pragma unroll
    for (int s = 0; s < 8; ++s) dmma_8x8x4(acc[2 * s], acc[2 * s + 1], uA, YA[s]);
#pragma unroll
    for (int s = 0; s < 8; ++s) dmma_8x8x4(acc[2 * s], acc[2 * s + 1], uB, YB[s]);
    pending = true;
    if (g + 1 == sl_end) {
      flush(head ? 0 : -1);
      pending = false;
      head = false;
      if (g + 1 < cend) {
        ++sl;
        sl_end = slice_grp[sl + 1];
        row = t.idx[0][sl];
      }
    }
  }
  if (pending) flush(head ? 0 : 1);
}

// TTMc-4 packed + TMA-staged (default): k_ttmc4pk's fragment mapping and
// math, with (1) each window of kGW groups (headers, slot coordinates and the
// three interleaved leaf streams l, k, value) staged into shared memory by
// lane 0 with bulk copies two (meta) / one (leaves) windows ahead, and (2) the
// V and W rows of an iteration's 8 leaves gathered row-contiguously (4 lanes
// per 64-byte row, one 128-bit load each) into small per-warp row tiles, from
// which each lane reads its segment's V row (broadcast) and W[l, t=h].
// ncu on k_ttmc4pk: the fragment-order gathers (8 lanes broadcast-reading one
// row with 256-bit loads, W[l_q, h] with 64-bit loads) cost ~110 L1
// data-pipe wavefronts per 8-leaf iteration and bound the kernel at 84 %.
struct StageT4 {
  alignas(16) double vs[kPackSlots][10];  // this iteration's V rows (padded)
  alignas(16) double ws[kPackSlots][10];  // this iteration's W rows
  alignas(16) int4 hdr[3][kGW];
  alignas(16) int32_t node[3][kGW * kPackSlots];
  alignas(16) int32_t ll[2][kGWLeaves];
  alignas(16) int32_t kk[2][kGWLeaves];
  alignas(16) double tv[2][kGWLeaves];
  uint64_t mbar_meta[3];
  uint64_t mbar_leaf[2];
};

template <bool VECV, bool VECW, bool BLK>
__global__ void __launch_bounds__(kBlock, 2) k_ttmc4pq(RootOutArgs a) {
  grid_launch_dependents();
  __shared__ StageT4 stage[kBlock / 32];
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * kBlock + threadIdx.x) / 32;
  if (w >= a.n_items) return;  // warp-uniform
  StageT4& S = stage[threadIdx.x / 32];
  const int lane = threadIdx.x & 31;
  const int q = lane & 3;   // fragment role: segment (K) index
  const int h = lane >> 2;  //   and r / t index
  const int gs = lane >> 2, gc = lane & 3;  // gather role: row slot, column pair
  const int R = a.R, S_ = a.S, T = a.T;
  const CsfView& t = a.t;
  const double* __restrict__ U = a.f[1];
  const double* __restrict__ V = a.f[2];
  const double* __restrict__ W = a.f[3];
  const int32_t* __restrict__ slice_grp = a.slice_grp;
  const int64_t tile = static_cast<int64_t>(R) * S_ * T;

  const int32_t cbeg = uni(static_cast<int32_t>(w * a.chunk));
  const int32_t cend = uni(static_cast<int32_t>(min64(cbeg + a.chunk, a.n_groups)));
  int32_t sl = a.item_pos[w];
  int32_t sl_end = slice_grp[sl + 1];
  bool head = slice_grp[sl] < cbeg;
  int32_t row = t.idx[0][sl];
  int32_t nx_end = sl + 2 <= t.nlev[0] ? __ldg(slice_grp + sl + 2) : 0;
  int32_t nx_row = sl + 1 < t.nlev[0] ? __ldg(t.idx[0] + sl + 1) : 0;
  bool pending = false;
  double acc[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) acc[e] = 0.0;

  auto flush = [&](int dslot) {
    double* dst = dslot < 0 ? a.out + static_cast<int64_t>(row) * tile
                            : a.part + (w * 2 + dslot) * tile;
#pragma unroll
    for (int nb = 0; nb < 8; ++nb)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        // n-tile nb, n index c = 2q + e: BLK maps it to the (s, t) of the
        // 4 x 2 block lane-column c owns, otherwise to (s = nb, t = c)
        const int c = 2 * q + e;
        const int ss = BLK ? 4 * (c & 1) + (nb >> 1) : nb;
        const int tt = BLK ? 2 * (c >> 1) + (nb & 1) : c;
        if (h < R && ss < S_ && tt < T) dst[(h * S_ + ss) * T + tt] = acc[2 * nb + e];
      }
#pragma unroll
    for (int e = 0; e < 16; ++e) acc[e] = 0.0;
  };
  auto issue_meta = [&](int32_t wi) {
    const int32_t g0 = cbeg + wi * kGW;
    const int32_t nw = min(g0 + kGW, cend) - g0;
    const int b = wi % 3;
    const unsigned hb = nw * sizeof(int4), nb = nw * kPackSlots * sizeof(int32_t);
    fence_proxy_async();
    expect_tx_elect(&S.mbar_meta[b], hb + nb);
    bulk_g2s_elect(&S.hdr[b][0], a.grp_hdr + g0, hb, &S.mbar_meta[b]);
    bulk_g2s_elect(&S.node[b][0], a.grp_node + static_cast<int64_t>(g0) * kPackSlots, nb, &S.mbar_meta[b]);
  };
  auto issue_leaves = [&](int32_t wi) {
    const int32_t g0 = cbeg + wi * kGW;
    const int32_t nw = min(g0 + kGW, cend) - g0;
    const int b = wi % 3, lb = wi & 1;
    mbar_wait(&S.mbar_meta[b], (wi / 3) & 1);
    const int32_t L0 = uni(S.hdr[b][0].x);
    const int32_t L1 = uni(S.hdr[b][nw - 1].x + kPackSlots * S.hdr[b][nw - 1].y);
    const unsigned n = static_cast<unsigned>(L1 - L0);
    fence_proxy_async();
    expect_tx_elect(&S.mbar_leaf[lb], n * 16u);
    bulk_g2s_elect(&S.ll[lb][0], a.pk + L0, n * 4u, &S.mbar_leaf[lb]);
    bulk_g2s_elect(&S.kk[lb][0], a.pk2 + L0, n * 4u, &S.mbar_leaf[lb]);
    bulk_g2s_elect(&S.tv[lb][0], a.pv + L0, n * 8u, &S.mbar_leaf[lb]);
  };

  const int32_t nwin = (cend - cbeg + kGW - 1) / kGW;
  if (lane == 0) {
    for (int b = 0; b < 3; ++b) mbar_init(&S.mbar_meta[b], 1);
    for (int b = 0; b < 2; ++b) mbar_init(&S.mbar_leaf[b], 1);
    mbar_init_fence();
  }
  __syncwarp();
  if (nwin > 0) {  // warp-collective issue (elected lane), uniform operands
    issue_meta(0);
    if (nwin > 1) issue_meta(1);
    issue_leaves(0);
  }
  for (int32_t win = 0; win < nwin; ++win) {
    const int mb = win % 3, lbf = win & 1;
    if (win + 1 < nwin) issue_leaves(win + 1);
    if (win + 2 < nwin) issue_meta(win + 2);
    mbar_wait(&S.mbar_meta[mb], (win / 3) & 1);
    mbar_wait(&S.mbar_leaf[lbf], (win / 2) & 1);
    const int32_t g0 = cbeg + win * kGW;
    const int32_t ge = min(g0 + kGW, cend);
    const int32_t L0 = S.hdr[mb][0].x;
    for (int32_t g = g0; g < ge; ++g) {
      const int4 hh = S.hdr[mb][g - g0];
      const int n = hh.y;  // warp-uniform leaves per segment
      const int32_t jA = S.node[mb][(g - g0) * kPackSlots + q];
      const int32_t jB = S.node[mb][(g - g0) * kPackSlots + 4 + q];
      const double uA = h < R ? __ldg(U + static_cast<int64_t>(jA) * R + h) : 0.0;
      const double uB = h < R ? __ldg(U + static_cast<int64_t>(jB) * R + h) : 0.0;
      double YA[8], YB[8];
#pragma unroll
      for (int s = 0; s < 8; ++s) YA[s] = YB[s] = 0.0;
#pragma unroll
      for (int it = 0; it < 4; ++it) {
        if (it < n) {  // warp-uniform
          // row-contiguous gathers: lane (gs, gc) fetches columns 2gc, 2gc+1
          // of slot gs's V and W rows into the per-warp row tiles
          const int32_t eg = hh.x - L0 + it * kPackSlots + gs;
          const double2 vg = pair2<VECV>(V + static_cast<int64_t>(S.kk[lbf][eg]) * S_, 2 * gc, S_);
          const double2 wg = pair2<VECW>(W + static_cast<int64_t>(S.ll[lbf][eg]) * T, 2 * gc, T);
          // BLK: 64-byte rows, 16-byte chunk c stored at c ^ ((row >> 1) & 1)
          *reinterpret_cast<double2*>(BLK ? &S.vs[0][0] + gs * 8 + 2 * (gc ^ ((gs >> 1) & 1))
                                          : &S.vs[gs][2 * gc]) = vg;
          // BLK: W rows swizzled like V (64-byte rows; the padded 80-byte rows
          // of the other path made these stores 2-way bank conflicts)
          *reinterpret_cast<double2*>(BLK ? &S.ws[0][0] + gs * 8 + 2 * (gc ^ ((gs >> 1) & 1))
                                          : &S.ws[gs][2 * gc]) = wg;
          __syncwarp();
          const int32_t eA = hh.x - L0 + it * kPackSlots + q, eB = eA + 4;
          const double vA = S.tv[lbf][eA], vB = S.tv[lbf][eB];
          if (BLK) {
            // lane (q, h) owns Y[s = 4sb + i][t = 2tb + j] (i < 4, j < 2):
            // 4 V and 2 W values per leaf and K-chunk
            const int sb = h & 1, tb = h >> 1;
            const int sw = (q >> 1) & 1;
            const double* vsf = &S.vs[0][0];  // BLK: rows of 8 doubles
            const double2 a0 = *reinterpret_cast<const double2*>(vsf + q * 8 + 2 * ((2 * sb) ^ sw));
            const double2 a1 = *reinterpret_cast<const double2*>(vsf + q * 8 + 2 * ((2 * sb + 1) ^ sw));
            const double2 b0 = *reinterpret_cast<const double2*>(vsf + (q + 4) * 8 + 2 * ((2 * sb) ^ sw));
            const double2 b1 =
                *reinterpret_cast<const double2*>(vsf + (q + 4) * 8 + 2 * ((2 * sb + 1) ^ sw));
            const double* wsf = &S.ws[0][0];
            const double2 wa = *reinterpret_cast<const double2*>(wsf + q * 8 + 2 * (tb ^ sw));
            const double2 wb = *reinterpret_cast<const double2*>(wsf + (q + 4) * 8 + 2 * (tb ^ sw));
            __syncwarp();  // row tiles are rewritten by the next iteration
            const double va[4] = {a0.x, a0.y, a1.x, a1.y}, vb[4] = {b0.x, b0.y, b1.x, b1.y};
            const double xa[2] = {vA * wa.x, vA * wa.y}, xb[2] = {vB * wb.x, vB * wb.y};
#pragma unroll
            for (int i2 = 0; i2 < 4; ++i2)
#pragma unroll
              for (int j2 = 0; j2 < 2; ++j2) {
                YA[2 * i2 + j2] = fma(va[i2], xa[j2], YA[2 * i2 + j2]);  // Y[s,t] += V[k,s] * X[t]
                YB[2 * i2 + j2] = fma(vb[i2], xb[j2], YB[2 * i2 + j2]);
              }
          } else {
            const double wA = S.ws[q][h], wB = S.ws[q + 4][h];
            double vrA[8], vrB[8];
#pragma unroll
            for (int m = 0; m < 4; ++m) {
              const double2 a2 = *reinterpret_cast<const double2*>(&S.vs[q][2 * m]);
              const double2 b2 = *reinterpret_cast<const double2*>(&S.vs[q + 4][2 * m]);
              vrA[2 * m] = a2.x; vrA[2 * m + 1] = a2.y;
              vrB[2 * m] = b2.x; vrB[2 * m + 1] = b2.y;
            }
            __syncwarp();  // row tiles are rewritten by the next iteration
            const double xA = vA * wA, xB = vB * wB;  // X[t] = t_ijkl * W[l,t]
#pragma unroll
            for (int s = 0; s < 8; ++s) {
              YA[s] = fma(vrA[s], xA, YA[s]);  // Y[s,t] += V[k,s] * X[t]
              YB[s] = fma(vrB[s], xB, YB[s]);
            }
          }
        }
      }
      // Out_i[r, s, t] += U[j, r] * Y[s, t] for both K-chunks
#pragma unroll
      for (int s = 0; s < 8; ++s) dmma_8x8x4(acc[2 * s], acc[2 * s + 1], uA, YA[s]);
#pragma unroll
      for (int s = 0; s < 8; ++s) dmma_8x8x4(acc[2 * s], acc[2 * s + 1], uB, YB[s]);
      pending = true;
      if (g + 1 == sl_end) {
        flush(head ? 0 : -1);
        pending = false;
        head = false;
        if (g + 1 < cend) {
          ++sl;
          sl_end = nx_end;
          row = nx_row;
          nx_end = sl + 2 <= t.nlev[0] ? __ldg(slice_grp + sl + 2) : 0;
          nx_row = sl + 1 < t.nlev[0] ? __ldg(t.idx[0] + sl + 1) : 0;
        }
      }
    }
    __syncwarp();  // stage buffers of this window are free after this point
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


// TTMc-4 packed + TMA-staged, asynchronous row gathers (mode 4, default for
// R, S, T <= 8 with S = T = 8 and 16-byte aligned factors). k_ttmc4pq's
// mapping and math, but the V and W rows of a leaf step are copied into the
// row tiles by cp.async (16 bytes per lane, the same row-contiguous lanes)
// one step ahead — within a group, across groups and across staged windows —
// into double-buffered tiles. ncu on k_ttmc4pq: the hottest instructions
// were the tile stores waiting on their gathers (long-scoreboard 30 % at
// 12.8 warps per SM); here the gather of step s+1 is in flight while step s
// is computed, with no extra registers.
struct StageT4a {
  alignas(16) double vs[2][kPackSlots * 8];  // V rows (64 bytes, swizzled), double-buffered
  alignas(16) double ws[2][kPackSlots * 8];  // W rows
  alignas(16) int4 hdr[3][kGW];
  alignas(16) int32_t node[3][kGW * kPackSlots];
  alignas(16) int32_t ll[2][kGWLeaves];
  alignas(16) int32_t kk[2][kGWLeaves];
  alignas(16) double tv[2][kGWLeaves];
  uint64_t mbar_meta[3];
  uint64_t mbar_leaf[2];
};
constexpr size_t t4a_smem_bytes(int nb) { return sizeof(StageT4a) * (nb / 32); }

template <int NB, int MB>
__global__ void __launch_bounds__(NB, MB) k_ttmc4pa(RootOutArgs a) {
  grid_launch_dependents();
  extern __shared__ __align__(16) unsigned char t4a_smem[];
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * NB + threadIdx.x) / 32;
  if (w >= a.n_items) return;  // warp-uniform
  StageT4a& S = reinterpret_cast<StageT4a*>(t4a_smem)[threadIdx.x / 32];
  const int lane = threadIdx.x & 31;
  const int q = lane & 3;   // fragment role: segment (K) index
  const int h = lane >> 2;  //   and r / t index
  const int gs = lane >> 2, gc = lane & 3;  // gather role: row slot, 16-byte chunk
  const int R = a.R;
  const CsfView& t = a.t;
  const double* __restrict__ U = a.f[1];
  const double* __restrict__ V = a.f[2];
  const double* __restrict__ W = a.f[3];
  const int32_t* __restrict__ slice_grp = a.slice_grp;
  const int64_t tile = static_cast<int64_t>(R) * 64;
  const int st_off = gs * 8 + 2 * (gc ^ ((gs >> 1) & 1));  // swizzled chunk of this lane

  const int32_t cbeg =
      uni(a.item_unit ? __ldg(a.item_unit + w) : static_cast<int32_t>(w * a.chunk));
  const int32_t cend = uni(a.item_unit ? __ldg(a.item_unit + w + 1)
                                       : static_cast<int32_t>(min64(cbeg + a.chunk, a.n_groups)));
  int32_t sl = a.item_pos[w];
  int32_t sl_end = slice_grp[sl + 1];
  bool head = slice_grp[sl] < cbeg;
  int32_t row = t.idx[0][sl];
  int32_t nx_end = sl + 2 <= t.nlev[0] ? __ldg(slice_grp + sl + 2) : 0;
  int32_t nx_row = sl + 1 < t.nlev[0] ? __ldg(t.idx[0] + sl + 1) : 0;
  bool pending = false;
  double acc[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) acc[e] = 0.0;

  auto flush = [&](int dslot) {
    double* dst = dslot < 0 ? a.out + static_cast<int64_t>(row) * tile
                            : a.part + (w * 2 + dslot) * tile;
#pragma unroll
    for (int nb = 0; nb < 8; ++nb)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = 2 * q + e;
        const int ss = 4 * (c & 1) + (nb >> 1);
        const int tt = 2 * (c >> 1) + (nb & 1);
        if (h < R) dst[(h * 8 + ss) * 8 + tt] = acc[2 * nb + e];
      }
#pragma unroll
    for (int e = 0; e < 16; ++e) acc[e] = 0.0;
  };
  auto issue_meta = [&](int32_t wi) {
    const int32_t g0 = cbeg + wi * kGW;
    const int32_t nw = min(g0 + kGW, cend) - g0;
    const int b = wi % 3;
    const unsigned hb = nw * sizeof(int4), nb = nw * kPackSlots * sizeof(int32_t);
    fence_proxy_async();
    expect_tx_elect(&S.mbar_meta[b], hb + nb);
    bulk_g2s_elect(&S.hdr[b][0], a.grp_hdr + g0, hb, &S.mbar_meta[b]);
    bulk_g2s_elect(&S.node[b][0], a.grp_node + static_cast<int64_t>(g0) * kPackSlots, nb, &S.mbar_meta[b]);
  };
  auto issue_leaves = [&](int32_t wi) {
    const int32_t g0 = cbeg + wi * kGW;
    const int32_t nw = min(g0 + kGW, cend) - g0;
    const int b = wi % 3, lb = wi & 1;
    mbar_wait(&S.mbar_meta[b], (wi / 3) & 1);
    const int32_t L0 = uni(S.hdr[b][0].x);
    const int32_t L1 = uni(S.hdr[b][nw - 1].x + kPackSlots * S.hdr[b][nw - 1].y);
    const unsigned n = static_cast<unsigned>(L1 - L0);
    fence_proxy_async();
    expect_tx_elect(&S.mbar_leaf[lb], n * 16u);
    bulk_g2s_elect(&S.ll[lb][0], a.pk + L0, n * 4u, &S.mbar_leaf[lb]);
    bulk_g2s_elect(&S.kk[lb][0], a.pk2 + L0, n * 4u, &S.mbar_leaf[lb]);
    bulk_g2s_elect(&S.tv[lb][0], a.pv + L0, n * 8u, &S.mbar_leaf[lb]);
  };
  // cp.async of one leaf step's V and W rows (slot gs, chunk gc) into tile buf
  auto issue_rows = [&](int buf, int lbuf, int32_t e) {
    cp_async16_ca(&S.vs[buf][st_off], V + static_cast<int64_t>(S.kk[lbuf][e]) * 8 + 2 * gc);
    cp_async16_ca(&S.ws[buf][st_off], W + static_cast<int64_t>(S.ll[lbuf][e]) * 8 + 2 * gc);
    cp_async_commit();
  };

  const int32_t nwin = (cend - cbeg + kGW - 1) / kGW;
  if (lane == 0) {
    for (int b = 0; b < 3; ++b) mbar_init(&S.mbar_meta[b], 1);
    for (int b = 0; b < 2; ++b) mbar_init(&S.mbar_leaf[b], 1);
    mbar_init_fence();
  }
  __syncwarp();
  if (nwin > 0) {
    issue_meta(0);
    if (nwin > 1) issue_meta(1);
    issue_leaves(0);
    mbar_wait(&S.mbar_meta[0], 0);
    mbar_wait(&S.mbar_leaf[0], 0);
    issue_rows(0, 0, gs);  // first step of the item (window 0 starts at its L0)
  }
  int buf = 0;  // tile of the current step
  for (int32_t win = 0; win < nwin; ++win) {
    const int mb = win % 3, lbf = win & 1;
    if (win + 1 < nwin) issue_leaves(win + 1);
    if (win + 2 < nwin) issue_meta(win + 2);
    mbar_wait(&S.mbar_meta[mb], (win / 3) & 1);
    mbar_wait(&S.mbar_leaf[lbf], (win / 2) & 1);
    const int32_t g0 = cbeg + win * kGW;
    const int32_t ge = min(g0 + kGW, cend);
    const int32_t L0 = S.hdr[mb][0].x;
    for (int32_t g = g0; g < ge; ++g) {
      const int4 hh = S.hdr[mb][g - g0];
      const int n = hh.y;  // warp-uniform leaves per segment
      const int32_t jA = S.node[mb][(g - g0) * kPackSlots + q];
      const int32_t jB = S.node[mb][(g - g0) * kPackSlots + 4 + q];
      const double uA = h < R ? __ldg(U + static_cast<int64_t>(jA) * R + h) : 0.0;
      const double uB = h < R ? __ldg(U + static_cast<int64_t>(jB) * R + h) : 0.0;
      double YA[8], YB[8];
#pragma unroll
      for (int s = 0; s < 8; ++s) YA[s] = YB[s] = 0.0;
#pragma unroll
      for (int it = 0; it < 4; ++it) {
        if (it < n) {  // warp-uniform
          // prefetch the next leaf step (this group, the next group of the
          // window, or the first group of the next window)
          bool more = true;
          if (it + 1 < n) {
            issue_rows(buf ^ 1, lbf, hh.x - L0 + (it + 1) * kPackSlots + gs);
          } else if (g + 1 < ge) {
            issue_rows(buf ^ 1, lbf, S.hdr[mb][g + 1 - g0].x - L0 + gs);
          } else if (win + 1 < nwin) {
            const int nm = (win + 1) % 3, nl = (win + 1) & 1;
            mbar_wait(&S.mbar_meta[nm], ((win + 1) / 3) & 1);
            mbar_wait(&S.mbar_leaf[nl], ((win + 1) / 2) & 1);
            issue_rows(buf ^ 1, nl, gs);  // the next window's first group starts at its L0
          } else {
            more = false;
          }
          if (more) cp_async_wait<1>(); else cp_async_wait<0>();
          __syncwarp();
          const int32_t eA = hh.x - L0 + it * kPackSlots + q, eB = eA + 4;
          const double vA = S.tv[lbf][eA], vB = S.tv[lbf][eB];
          // lane (q, h) owns Y[s = 4sb + i][t = 2tb + j] (i < 4, j < 2)
          const int sb = h & 1, tb = h >> 1;
          const int sw = (q >> 1) & 1;
          const double* vsf = S.vs[buf];
          const double* wsf = S.ws[buf];
          const double2 a0 = *reinterpret_cast<const double2*>(vsf + q * 8 + 2 * ((2 * sb) ^ sw));
          const double2 a1 = *reinterpret_cast<const double2*>(vsf + q * 8 + 2 * ((2 * sb + 1) ^ sw));
          const double2 b0 = *reinterpret_cast<const double2*>(vsf + (q + 4) * 8 + 2 * ((2 * sb) ^ sw));
          const double2 b1 =
              *reinterpret_cast<const double2*>(vsf + (q + 4) * 8 + 2 * ((2 * sb + 1) ^ sw));
          const double2 wa = *reinterpret_cast<const double2*>(wsf + q * 8 + 2 * (tb ^ sw));
          const double2 wb = *reinterpret_cast<const double2*>(wsf + (q + 4) * 8 + 2 * (tb ^ sw));
          __syncwarp();  // this tile is refilled by the step after next
          buf ^= 1;
          const double va[4] = {a0.x, a0.y, a1.x, a1.y}, vb[4] = {b0.x, b0.y, b1.x, b1.y};
          const double xa[2] = {vA * wa.x, vA * wa.y}, xb[2] = {vB * wb.x, vB * wb.y};
#pragma unroll
          for (int i2 = 0; i2 < 4; ++i2)
#pragma unroll
            for (int j2 = 0; j2 < 2; ++j2) {
              YA[2 * i2 + j2] = fma(va[i2], xa[j2], YA[2 * i2 + j2]);  // Y[s,t] += V[k,s] * X[t]
              YB[2 * i2 + j2] = fma(vb[i2], xb[j2], YB[2 * i2 + j2]);
            }
        }
      }
      // Out_i[r, s, t] += U[j, r] * Y[s, t] for both K-chunks
#pragma unroll
      for (int s = 0; s < 8; ++s) dmma_8x8x4(acc[2 * s], acc[2 * s + 1], uA, YA[s]);
#pragma unroll
      for (int s = 0; s < 8; ++s) dmma_8x8x4(acc[2 * s], acc[2 * s + 1], uB, YB[s]);
      pending = true;
      if (g + 1 == sl_end) {
        flush(head ? 0 : -1);
        pending = false;
        head = false;
        if (g + 1 < cend) {
          ++sl;
          sl_end = nx_end;
          row = nx_row;
          nx_end = sl + 2 <= t.nlev[0] ? __ldg(slice_grp + sl + 2) : 0;
          nx_row = sl + 1 < t.nlev[0] ? __ldg(t.idx[0] + sl + 1) : 0;
        }
      }
    }
    __syncwarp();  // stage buffers of this window are free after this point
  }
  if (pending) flush(head ? 0 : 1);
}

}  // namespace

// resident warps per SM of the TTMc-3 default kernel (plan-time item sizing:
// one item per resident warp, a single wave)
int ttmc3pq_warps_per_sm() {
  int blocks = 0;
  if (cudaFuncSetAttribute(k_ttmc3pq<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(kPqSmem)) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k_ttmc3pq<true, true>, kBlock,
                                                    kPqSmem) != cudaSuccess)
    blocks = 3;
  return std::max(1, blocks) * (kBlock / 32);
}

void launch_ttmc3(const RootOutArgs& a, cudaStream_t s) {
  const int64_t blocks = (a.n_items * 32 + kBlock - 1) / kBlock;
  if (blocks == 0) return;
  const bool vu = a.vec & 1, vv = a.vec & 2;
  const int mode = a.flags >> 8;  // kernel variant chosen at plan time
  if (mode == 10) {
    const bool wu = a.vec & 4, wv = a.vec & 8;
    auto go = [&](auto kern) {
      SPTTN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(kPqSmem)));
      kern<<<static_cast<unsigned>(blocks), kBlock, kPqSmem, s>>>(a);
    };
    if (wu && wv)
      go(k_ttmc3pq<true, true>);
    else if (wu)
      go(k_ttmc3pq<true, false>);
    else if (wv)
      go(k_ttmc3pq<false, true>);
    else
      go(k_ttmc3pq<false, false>);
    SPTTN_CUDA(cudaGetLastError());
    return;
  }
  if (mode == 7) {
    const bool wu = a.vec & 4, wv = a.vec & 8;
    if (wu && wv)
      k_ttmc3ps<true, true><<<static_cast<unsigned>(blocks), kBlock, 0, s>>>(a);
    else if (wu)
      k_ttmc3ps<true, false><<<static_cast<unsigned>(blocks), kBlock, 0, s>>>(a);
    else if (wv)
      k_ttmc3ps<false, true><<<static_cast<unsigned>(blocks), kBlock, 0, s>>>(a);
    else
      k_ttmc3ps<false, false><<<static_cast<unsigned>(blocks), kBlock, 0, s>>>(a);
    SPTTN_CUDA(cudaGetLastError());
    return;
  }
  if (mode == 6) {
    const bool wu = a.vec & 4, wv = a.vec & 8;
    if (wu && wv)
      k_ttmc3pk<true, true><<<static_cast<unsigned>(blocks), kBlock, 0, s>>>(a);
    else if (wu)
      k_ttmc3pk<true, false><<<static_cast<unsigned>(blocks), kBlock, 0, s>>>(a);
    else if (wv)
      k_ttmc3pk<false, true><<<static_cast<unsigned>(blocks), kBlock, 0, s>>>(a);
    else
      k_ttmc3pk<false, false><<<static_cast<unsigned>(blocks), kBlock, 0, s>>>(a);
    SPTTN_CUDA(cudaGetLastError());
    return;
  }
  if (mode == 4) {
    if (vu && vv)
      k_ttmc3s<true, true><<<static_cast<unsigned>(blocks), kBlock, 0, s>>>(a);
    else if (vu)
      k_ttmc3s<true, false><<<static_cast<unsigned>(blocks), kBlock, 0, s>>>(a);
    else if (vv)
      k_ttmc3s<false, true><<<static_cast<unsigned>(blocks), kBlock, 0, s>>>(a);
    else
      k_ttmc3s<false, false><<<static_cast<unsigned>(blocks), kBlock, 0, s>>>(a);
    SPTTN_CUDA(cudaGetLastError());
    return;
  }
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
  const int mode = a.flags >> 8;
  if (mode == 4) {  // async row gathers (the plan checked S = T = 8, R <= 8, alignment)
    // 384 threads x 1 block per SM: up to 168 registers (163 used, no spill);
    // 256 x 2 capped them at 128 and spilled 32 B per group at the same speed
    // (404 vs 407 us at the BASELINE shape)
    constexpr int nb = 384;
    const size_t sm = t4a_smem_bytes(nb);
    SPTTN_CUDA(cudaFuncSetAttribute(k_ttmc4pa<nb, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(sm)));
    k_ttmc4pa<nb, 1><<<static_cast<unsigned>((a.n_items * 32 + nb - 1) / nb), nb, sm, s>>>(a);
  } else if (mode == 2 || mode == 3) {
    const bool vv = a.vec & 2, vw = a.vec & 4;
    const unsigned b = static_cast<unsigned>(blocks);
    if (mode == 3) {  // 4 x 2 (s, t) blocks per lane
      if (vv && vw) k_ttmc4pq<true, true, true><<<b, kBlock, 0, s>>>(a);
      else if (vv) k_ttmc4pq<true, false, true><<<b, kBlock, 0, s>>>(a);
      else if (vw) k_ttmc4pq<false, true, true><<<b, kBlock, 0, s>>>(a);
      else k_ttmc4pq<false, false, true><<<b, kBlock, 0, s>>>(a);
    } else {
      if (vv && vw) k_ttmc4pq<true, true, false><<<b, kBlock, 0, s>>>(a);
      else if (vv) k_ttmc4pq<true, false, false><<<b, kBlock, 0, s>>>(a);
      else if (vw) k_ttmc4pq<false, true, false><<<b, kBlock, 0, s>>>(a);
      else k_ttmc4pq<false, false, false><<<b, kBlock, 0, s>>>(a);
    }
  } else if (mode == 1) {
    if (a.vec & 2)
      k_ttmc4pk<true><<<static_cast<unsigned>(blocks), kBlock, 0, s>>>(a);
    else
      k_ttmc4pk<false><<<static_cast<unsigned>(blocks), kBlock, 0, s>>>(a);
  } else if (a.vec & 2) {
    k_ttmc4<true><<<static_cast<unsigned>(blocks), kBlock, 0, s>>>(a);
  } else {
    k_ttmc4<false><<<static_cast<unsigned>(blocks), kBlock, 0, s>>>(a);
  }
  SPTTN_CUDA(cudaGetLastError());
}

}  // namespace spttn_dev
