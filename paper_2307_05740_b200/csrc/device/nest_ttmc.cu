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
#include <type_traits>

#include "internal.cuh"

namespace spttn_dev {

namespace {

constexpr int kBlock = 256;


// Packed groups are consumed in windows of kGW groups staged into shared
// memory (TMA bulk copies on mbarriers, two windows of headers / slot
// coordinates and one of leaf streams ahead).
constexpr int kGW = 4;                             // groups per window
constexpr int kGWLeaves = kGW * kPackSlots * 4;    // leaves per window (len <= 4)

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

// CLK (diagnostics build, SPTTN_ITEM_CLOCKS=1): per item {start ns, end ns,
// SM, groups, leaf steps, tile flushes} for fitting the item work model
// PF: U rows of every group and V rows of single-leaf groups are copied
// into the fragment tiles by cp.async.cg (LDGSTS.BYPASS, already in the
// swizzled tile layout) one group ahead within a staged window, so the
// STS half of their register transposition disappears and the gathers
// overlap the previous group's DMMAs. Needs the pair-permuted packing
// (logical slots a, a+4 stored adjacently, so one 8-byte LDS yields the
// two rows a lane copies) and R = S = 16 (one 128-byte row = 8 chunks).
template <bool VECU, bool VECV, bool CLK = false, bool PF = false>
__global__ void __launch_bounds__(kBlock, 3) k_ttmc3pq(RootOutArgs a) {
  grid_launch_dependents();
  extern __shared__ __align__(16) unsigned char pq_smem[];  // kPqSmem bytes
  StageT* stage = reinterpret_cast<StageT*>(pq_smem);
  StageQ* tiles = reinterpret_cast<StageQ*>(pq_smem + sizeof(StageT) * (kBlock / 32));
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * kBlock + threadIdx.x) / 32;
  if (w >= a.n_items) return;  // warp-uniform
  if (CLK && (threadIdx.x & 31) == 0) a.clk[6 * w] = globaltimer_ns();
  int dbg_steps = 0, dbg_flush = 0;
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
    SPTTN_DCHECK(dslot >= 0 || (row >= 0 && row < a.frows[0]));
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const int r = 8 * mt + fh;
        const int s = 8 * nt + 2 * fq;  // the lane's two columns s, s + 1
        if (VECV && r < R && s < S_) {  // S % 4 == 0: the pair is in range, 16-byte aligned
          *reinterpret_cast<double2*>(dst + r * S_ + s) =
              make_double2(acc[(mt * 2 + nt) * 2], acc[(mt * 2 + nt) * 2 + 1]);
        } else {
#pragma unroll
          for (int e = 0; e < 2; ++e)
            if (r < R && s + e < S_) dst[r * S_ + s + e] = acc[(mt * 2 + nt) * 2 + e];
        }
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
    SPTTN_DCHECK(n <= static_cast<unsigned>(kGWLeaves));
    fence_proxy_async();
    expect_tx_elect(&S.mbar_leaf[lb], n * 12u);
    bulk_g2s_elect(&S.kk[lb][0], a.pk + L0, n * 4u, &S.mbar_leaf[lb]);
    bulk_g2s_elect(&S.tv[lb][0], a.pv + L0, n * 8u, &S.mbar_leaf[lb]);
  };

  // swizzled tile: element (slot, col) at slot*16 + (col ^ 4*(slot&3) ^ 2*(slot&1))
  const int st_off = gs * 16 + ((4 * gc) ^ (4 * (gs & 3)));
  const int o_lo = st_off + 2 * (gs & 1), o_hi = st_off + 2 - 2 * (gs & 1);
  // PF: storage position of logical slot gs in the pair-permuted packing,
  // and the cp.async role (16-byte chunk cc of rows cr, cr + 4)
  const int gpos = PF ? 2 * (gs & 3) + (gs >> 2) : gs;
  const int cr = lane >> 3, cc = lane & 7;
  const int cp_lo = cr * 16 + ((2 * cc) ^ (4 * (cr & 3)) ^ (2 * (cr & 1)));
  const int cp_hi = (cr + 4) * 16 + ((2 * cc) ^ (4 * (cr & 3)) ^ (2 * (cr & 1)));
  // cp.async of group gi's (window buffers b, lb) U rows and, if it is a
  // single-leaf group, V rows into tile tp
  auto prefetch = [&](int b, int lb, int32_t l0, int gl, int tp) {
    const int4 h2 = S.hdr[b][gl];
    const int2 nd = *reinterpret_cast<const int2*>(&S.node[b][gl * kPackSlots + 2 * cr]);
    SPTTN_DCHECK(nd.x >= 0 && nd.y >= 0 && nd.x < a.frows[1] && nd.y < a.frows[1]);
    cp_async16_cg(&Q.us[tp][cp_lo], U + static_cast<uint32_t>(nd.x) * 16u + 2 * cc, 16);
    cp_async16_cg(&Q.us[tp][cp_hi], U + static_cast<uint32_t>(nd.y) * 16u + 2 * cc, 16);
    if (h2.y == 1) {
      const int2 k2 = *reinterpret_cast<const int2*>(&S.kk[lb][h2.x - l0 + 2 * cr]);
      SPTTN_DCHECK(k2.x >= 0 && k2.y >= 0 && k2.x < a.frows[2] && k2.y < a.frows[2]);
      cp_async16_cg(&Q.xs[tp][cp_lo], V + static_cast<uint32_t>(k2.x) * 16u + 2 * cc, 16);
      cp_async16_cg(&Q.xs[tp][cp_hi], V + static_cast<uint32_t>(k2.y) * 16u + 2 * cc, 16);
    }
    cp_async_commit();
  };
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
    if (PF && g0 < ge) {
      __syncwarp();
      prefetch(mb, lbf, L0, 0, par);  // the window's first group: no earlier prefetch
    }
    for (int32_t g = g0; g < ge; ++g) {
      const int4 hh = S.hdr[mb][g - g0];
      const int n = hh.y;  // warp-uniform
      if (CLK) dbg_steps += n;
      if (PF) {
        __syncwarp();  // tile par^1 (group g-1) is read by every lane
        if (g + 1 < ge) prefetch(mb, lbf, L0, g + 1 - g0, par ^ 1);
      }
      const int32_t lbase = hh.x - L0 + gpos;
      const int32_t j = S.node[mb][(g - g0) * kPackSlots + gpos];
      SPTTN_DCHECK(j >= 0 && j < a.frows[1]);
      SPTTN_DCHECK(lbase + (n - 1) * kPackSlots < kGWLeaves);
      const double4 ur = PF ? make_double4(0, 0, 0, 0)
                            : row4<VECU>(U + static_cast<int64_t>(j) * R, 4 * gc, R);
      // X[s] += t * V[k,s] over the group's n (warp-uniform) leaf steps,
      // specialised per n: no predicated-off stream loads / gathers / FMAs
      double4 x = make_double4(0, 0, 0, 0);
      auto steps = [&](auto NS) {
        constexpr int kN = decltype(NS)::value;
        int32_t kk[kN];
        double tt[kN];
#pragma unroll
        for (int it = 0; it < kN; ++it) {
          kk[it] = S.kk[lbf][lbase + it * kPackSlots];
          tt[it] = S.tv[lbf][lbase + it * kPackSlots];
        }
        double4 vr[kN];
#pragma unroll
        for (int it = 0; it < kN; ++it) SPTTN_DCHECK(kk[it] >= 0 && kk[it] < a.frows[2]);
#pragma unroll
        for (int it = 0; it < kN; ++it) {
          if (VECV)
            vr[it] = ld256_if(V + static_cast<int64_t>(kk[it]) * S_ + 4 * gc, 4 * gc < S_);
          else
            vr[it] = row4<false>(V + static_cast<int64_t>(kk[it]) * S_, 4 * gc, S_);
        }
#pragma unroll
        for (int it = 0; it < kN; ++it) fma4(x, tt[it], vr[it]);
      };
      double* xs = Q.xs[par];
      double* us = Q.us[par];
      if (!PF || n != 1) {
        switch (n) {
          case 1: steps(std::integral_constant<int, 1>{}); break;
          case 2: steps(std::integral_constant<int, 2>{}); break;
          case 3: steps(std::integral_constant<int, 3>{}); break;
          default: steps(std::integral_constant<int, 4>{}); break;
        }
        // transpose X (and U) quads into fragment layout through the tile
        *reinterpret_cast<double2*>(xs + o_lo) = make_double2(x.x, x.y);
        *reinterpret_cast<double2*>(xs + o_hi) = make_double2(x.z, x.w);
      }
      if (!PF) {
        *reinterpret_cast<double2*>(us + o_lo) = make_double2(ur.x, ur.y);
        *reinterpret_cast<double2*>(us + o_hi) = make_double2(ur.z, ur.w);
      } else {
        if (g + 1 < ge) cp_async_wait<1>(); else cp_async_wait<0>();  // group g's copies
      }
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
      if (PF && n == 1) {  // X = t * V[k] for single-leaf segments (copied rows)
#pragma unroll
        for (int kc = 0; kc < 2; ++kc) {
          const int seg = 4 * kc + fq;  // logical slot; stored at 2(seg&3) + (seg>>2)
          const double tk = S.tv[lbf][hh.x - L0 + 2 * (seg & 3) + (seg >> 2)];
          bf[kc][0] *= tk;
          bf[kc][1] *= tk;
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
        if (CLK) ++dbg_flush;
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
  if (CLK && pending) ++dbg_flush;
  if (pending) flush(head ? 0 : 1);
  if (CLK && lane == 0) {
    a.clk[6 * w + 1] = globaltimer_ns();
    a.clk[6 * w + 2] = smid();
    a.clk[6 * w + 3] = cend - cbeg;
    a.clk[6 * w + 4] = dbg_steps;
    a.clk[6 * w + 5] = dbg_flush;
  }
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
// TTMc-4 packed + TMA-staged (general R, S, T <= 8): DMMA fragment mapping
// as described at the top of the file, with (1) each window of kGW groups (headers, slot coordinates and the
// three interleaved leaf streams l, k, value) staged into shared memory by
// lane 0 with bulk copies two (meta) / one (leaves) windows ahead, and (2) the
// V and W rows of an iteration's 8 leaves gathered row-contiguously (4 lanes
// per 64-byte row, one 128-bit load each) into small per-warp row tiles, from
// which each lane reads its segment's V row (broadcast) and W[l, t=h].
// (Gathering in fragment order instead — 8 lanes broadcast-reading one row
// with 256-bit loads, W[l_q, h] with 64-bit loads — cost ~110 L1 data-pipe
// wavefronts per 8-leaf iteration, round 1.)
struct StageT4 {
  alignas(16) double vs[kPackSlots][8];  // this iteration's V rows (swizzled)
  alignas(16) double ws[kPackSlots][8];  // this iteration's W rows
  alignas(16) int4 hdr[3][kGW];
  alignas(16) int32_t node[3][kGW * kPackSlots];
  alignas(16) int32_t ll[2][kGWLeaves];
  alignas(16) int32_t kk[2][kGWLeaves];
  alignas(16) double tv[2][kGWLeaves];
  uint64_t mbar_meta[3];
  uint64_t mbar_leaf[2];
};

template <bool VECV, bool VECW>
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
        // n-tile nb, n index c = 2q + e: the (s, t) of the 4 x 2 block
        // lane-column c owns
        const int c = 2 * q + e;
        const int ss = 4 * (c & 1) + (nb >> 1);
        const int tt = 2 * (c >> 1) + (nb & 1);
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
          // 64-byte rows, 16-byte chunk c stored at c ^ ((row >> 1) & 1)
          *reinterpret_cast<double2*>(&S.vs[0][0] + gs * 8 + 2 * (gc ^ ((gs >> 1) & 1))) = vg;
          *reinterpret_cast<double2*>(&S.ws[0][0] + gs * 8 + 2 * (gc ^ ((gs >> 1) & 1))) = wg;
          __syncwarp();
          const int32_t eA = hh.x - L0 + it * kPackSlots + q, eB = eA + 4;
          const double vA = S.tv[lbf][eA], vB = S.tv[lbf][eB];
          // lane (q, h) owns Y[s = 4sb + i][t = 2tb + j] (i < 4, j < 2):
          // 4 V and 2 W values per leaf and K-chunk
          const int sb = h & 1, tb = h >> 1;
          const int sw = (q >> 1) & 1;
          const double* vsf = &S.vs[0][0];  // rows of 8 doubles
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

// TTMc-4 packed + TMA-staged, asynchronous row gathers (mode 4, default for
// R, S, T <= 8 with S = T = 8 and 16-byte aligned factors). k_ttmc4pq's
// mapping and math, but the V and W rows of a leaf step are copied into the
// row tiles by cp.async (16 bytes per lane, the same row-contiguous lanes)
// one step ahead — within a group, across groups and across staged windows —
// into double-buffered tiles. ncu on k_ttmc4pq: the hottest instructions
// were the tile stores waiting on their gathers (long-scoreboard 30 % at
// 12.8 warps per SM); here the gather of step s+1 is in flight while step s
// is computed, with no extra registers.
// TTMc-4 staging windows (1 CTA of 12 warps per SM: room for larger windows
// than TTMc-3's 3 CTAs)
#ifndef SPTTN_GW4
#define SPTTN_GW4 12
#endif
constexpr int kGW4 = SPTTN_GW4;                      // groups per window
constexpr int kGW4Leaves = kGW4 * kPackSlots * 4;    // leaves per window (len <= 4)
struct StageT4a {
  alignas(16) double vs[2][kPackSlots * 8];  // V rows (64 bytes, swizzled), double-buffered
  alignas(16) double ws[2][kPackSlots * 8];  // W rows
  alignas(16) int4 hdr[3][kGW4];
  alignas(16) int32_t node[3][kGW4 * kPackSlots];
  alignas(16) int32_t ll[2][kGW4Leaves];
  alignas(16) int32_t kk[2][kGW4Leaves];
  alignas(16) double tv[2][kGW4Leaves];
  uint64_t mbar_meta[3];
  uint64_t mbar_leaf[2];
};
constexpr size_t t4a_smem_bytes(int nb) { return sizeof(StageT4a) * (nb / 32); }
// TTMc-4 default kernel: 384 threads x 1 CTA per SM (up to 168 registers)
constexpr int kT4Block = 384;

template <int NB, int MB, bool CLK = false>
__global__ void __launch_bounds__(NB, MB) k_ttmc4pa(RootOutArgs a) {
  grid_launch_dependents();
  extern __shared__ __align__(16) unsigned char t4a_smem[];
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * NB + threadIdx.x) / 32;
  if (w >= a.n_items) return;  // warp-uniform
  if (CLK && (threadIdx.x & 31) == 0) a.clk[6 * w] = globaltimer_ns();
  int dbg_steps = 0, dbg_flush = 0;
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
    // n-tiles 2m and 2m+1 hold the adjacent columns tt, tt + 1 of the same
    // (h, ss) row: one 16-byte store per pair
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = 2 * q + e;
        const int ss = 4 * (c & 1) + m;
        const int tt = 2 * (c >> 1);
        if (h < R)
          *reinterpret_cast<double2*>(dst + (h * 8 + ss) * 8 + tt) =
              make_double2(acc[2 * (2 * m) + e], acc[2 * (2 * m + 1) + e]);
      }
#pragma unroll
    for (int e = 0; e < 16; ++e) acc[e] = 0.0;
  };
  auto issue_meta = [&](int32_t wi) {
    const int32_t g0 = cbeg + wi * kGW4;
    const int32_t nw = min(g0 + kGW4, cend) - g0;
    const int b = wi % 3;
    const unsigned hb = nw * sizeof(int4), nb = nw * kPackSlots * sizeof(int32_t);
    fence_proxy_async();
    expect_tx_elect(&S.mbar_meta[b], hb + nb);
    bulk_g2s_elect(&S.hdr[b][0], a.grp_hdr + g0, hb, &S.mbar_meta[b]);
    bulk_g2s_elect(&S.node[b][0], a.grp_node + static_cast<int64_t>(g0) * kPackSlots, nb, &S.mbar_meta[b]);
  };
  auto issue_leaves = [&](int32_t wi) {
    const int32_t g0 = cbeg + wi * kGW4;
    const int32_t nw = min(g0 + kGW4, cend) - g0;
    const int b = wi % 3, lb = wi & 1;
    mbar_wait(&S.mbar_meta[b], (wi / 3) & 1);
    const int32_t L0 = uni(S.hdr[b][0].x);
    const int32_t L1 = uni(S.hdr[b][nw - 1].x + kPackSlots * S.hdr[b][nw - 1].y);
    const unsigned n = static_cast<unsigned>(L1 - L0);
    SPTTN_DCHECK(n <= static_cast<unsigned>(kGW4Leaves));
    fence_proxy_async();
    expect_tx_elect(&S.mbar_leaf[lb], n * 16u);
    bulk_g2s_elect(&S.ll[lb][0], a.pk + L0, n * 4u, &S.mbar_leaf[lb]);
    bulk_g2s_elect(&S.kk[lb][0], a.pk2 + L0, n * 4u, &S.mbar_leaf[lb]);
    bulk_g2s_elect(&S.tv[lb][0], a.pv + L0, n * 8u, &S.mbar_leaf[lb]);
  };
  // cp.async of one leaf step's V and W rows (slot gs, chunk gc) into tile
  // buf — .cg (L2 -> shared, no L1 allocation: LDGSTS.BYPASS): 391 vs 408 us
  // for the L1-allocating .ca at the BASELINE shape (fewer L1 wavefronts per
  // copy; the 128 KB V / W are L2-resident)
  auto issue_rows = [&](int buf, int lbuf, int32_t e) {
    SPTTN_DCHECK(e >= 0 && e < kGW4Leaves);
    SPTTN_DCHECK(S.kk[lbuf][e] >= 0 && S.kk[lbuf][e] < a.frows[2]);
    SPTTN_DCHECK(S.ll[lbuf][e] >= 0 && S.ll[lbuf][e] < a.frows[3]);
    cp_async16_cg(&S.vs[buf][st_off], V + static_cast<int64_t>(S.kk[lbuf][e]) * 8 + 2 * gc, 16);
    cp_async16_cg(&S.ws[buf][st_off], W + static_cast<int64_t>(S.ll[lbuf][e]) * 8 + 2 * gc, 16);
    cp_async_commit();
  };

  const int32_t nwin = (cend - cbeg + kGW4 - 1) / kGW4;
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
    const int32_t g0 = cbeg + win * kGW4;
    const int32_t ge = min(g0 + kGW4, cend);
    const int32_t L0 = S.hdr[mb][0].x;
    for (int32_t g = g0; g < ge; ++g) {
      const int4 hh = S.hdr[mb][g - g0];
      const int n = hh.y;  // warp-uniform leaves per segment
      if (CLK) dbg_steps += n;
      const int32_t jA = S.node[mb][(g - g0) * kPackSlots + q];
      const int32_t jB = S.node[mb][(g - g0) * kPackSlots + 4 + q];
      SPTTN_DCHECK(jA >= 0 && jA < a.frows[1] && jB >= 0 && jB < a.frows[1]);
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
        if (CLK) ++dbg_flush;
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
  if (CLK && pending) ++dbg_flush;
  if (pending) flush(head ? 0 : 1);
  if (CLK && lane == 0) {
    a.clk[6 * w + 1] = globaltimer_ns();
    a.clk[6 * w + 2] = smid();
    a.clk[6 * w + 3] = cend - cbeg;
    a.clk[6 * w + 4] = dbg_steps;
    a.clk[6 * w + 5] = dbg_flush;
  }
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

// resident warps per SM of the TTMc-4 default kernel (plan-time item sizing:
// one item per resident warp — items past a whole wave of 384-thread CTAs
// left 1/3 of the SMs idle for the last third of the kernel)
int ttmc4pa_warps_per_sm() {
  int blocks = 0;
  const size_t sm = t4a_smem_bytes(kT4Block);
  if (cudaFuncSetAttribute(k_ttmc4pa<kT4Block, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(sm)) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k_ttmc4pa<kT4Block, 1>, kT4Block, sm) !=
          cudaSuccess)
    blocks = 1;
  return std::max(1, blocks) * (kT4Block / 32);
}

void launch_ttmc3(const RootOutArgs& a, cudaStream_t s) {
  const int64_t blocks = (a.n_items * 32 + kBlock - 1) / kBlock;
  if (blocks == 0) return;
  const bool wu = a.vec & 4, wv = a.vec & 8;  // 256-bit U / V row gathers allowed
  auto go = [&](auto kern) {
    SPTTN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kPqSmem)));
    pin_carveout(kern, 3, kPqSmem);  // the items are one per resident warp at 3 CTAs per SM
    kern<<<static_cast<unsigned>(blocks), kBlock, kPqSmem, s>>>(a);
  };
  const bool pf = (a.flags >> 8) == 16;
  if (wu && wv && a.clk)
    go(pf ? k_ttmc3pq<true, true, true, true> : k_ttmc3pq<true, true, true>);
  else if (wu && wv && pf)
    go(k_ttmc3pq<true, true, false, true>);
  else if (wu && wv)
    go(k_ttmc3pq<true, true>);
  else if (wu)
    go(k_ttmc3pq<true, false>);
  else if (wv)
    go(k_ttmc3pq<false, true>);
  else
    go(k_ttmc3pq<false, false>);
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
    auto go4 = [&](auto kern, int nb) {
      const size_t sm = t4a_smem_bytes(nb);
      SPTTN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(sm)));
      pin_carveout(kern, 1, sm);
      kern<<<static_cast<unsigned>((a.n_items * 32 + nb - 1) / nb), nb, sm, s>>>(a);
    };
    if (a.clk)  // diagnostics instantiation (SPTTN_ITEM_CLOCKS=1)
      go4(k_ttmc4pa<kT4Block, 1, true>, kT4Block);
    else
      go4(k_ttmc4pa<kT4Block, 1>, kT4Block);
  } else {  // packed, 4 x 2 (s, t) blocks per lane (any R, S, T <= 8)
    const bool vv = a.vec & 2, vw = a.vec & 4;
    const unsigned b = static_cast<unsigned>(blocks);
    auto goq = [&](auto kern) {
      pin_carveout(kern, 2, 0);
      kern<<<b, kBlock, 0, s>>>(a);
    };
    if (vv && vw) goq(k_ttmc4pq<true, true>);
    else if (vv) goq(k_ttmc4pq<true, false>);
    else if (vw) goq(k_ttmc4pq<false, true>);
    else goq(k_ttmc4pq<false, false>);
  }
  SPTTN_CUDA(cudaGetLastError());
}

}  // namespace spttn_dev
