// MTTKRP-3 / MTTKRP-4, segment form (R <= 32).
//
// Reference nests (proj/src/executor.cpp:453-490, hooks :411-451):
//   MTTKRP-3 ((T*C)*B), orders (i,j,k,a)(i,j,a):
//       per (i,j)    X[a] = sum_k t * C[k,a]         (vector-accumulate hook)
//       per (i,j)    A[i,a] += X[a] * B[j,a]
//   MTTKRP-4 (((T*D)*C)*B), orders (i,j,k,l,r)(i,j,k,r)(i,j,r):
//       per (i,j,k)  X[r] = sum_l t * D[l,r]
//       per (i,j,k)  Y[r] += X[r] * C[k,r];   per (i,j)  A[i,r] += Y[r] * B[j,r]
//
// Work units are the fibers one level above the leaves ((i,j) for order 3,
// (i,j,k) for order 4) cut into segments of <= 4 leaves and packed into
// length-sorted groups (pack.cu). Each slot accumulates its slice
// contribution in registers (order 4 folds Y*B per (i,j,k) segment:
// A_i += (X*C[k])*B[j], the same sum regrouped); a finished slice is reduced
// over the slots with shuffles and written once (owner computes), and slices
// cut by item boundaries go through the deterministic HEAD/TAIL fix-up.
#include <cstdlib>
#include <type_traits>

#include "internal.cuh"

namespace spttn_dev {

namespace {

constexpr int kBlock = 256;

// Packed form (default for R <= 32): the warp walks length-sorted groups of 4
// equal-length segments (pack.cu with 4 slots: a 256-byte row needs 8 lanes
// of 32 bytes, so 4 rows fill one 256-bit warp gather). Lane L = (slot =
// L/8, column quad c = 4*(L%8)). Every gather is issued in straight-line
// code (predicated, no branches) so all of a group's rows are in flight
// together; the group's segment length n is warp-uniform.
template <int ORDER, bool VEC>
__global__ void __launch_bounds__(kBlock, 4) k_mttkrp_pk(RootOutArgs a) {
  grid_launch_dependents();
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * kBlock + threadIdx.x) / 32;
  if (w >= a.n_items) return;  // warp-uniform
  constexpr int kSlots = 4;
  const int lane = threadIdx.x & 31;
  const int slot = lane >> 3;
  const int c = (lane & 7) * 4;
  const int R = a.R;
  const CsfView& t = a.t;
  const double* __restrict__ Fleaf = a.f[ORDER - 1];
  const double* __restrict__ Funit = a.f[ORDER - 2];
  const double* __restrict__ Ftop = a.f[1];
  const int4* __restrict__ hdr = a.grp_hdr;
  const int32_t* __restrict__ gnode = a.grp_node;
  const int32_t* __restrict__ gnode1 = a.grp_node1;
  const int32_t* __restrict__ pk = a.pk;
  const double* __restrict__ pv = a.pv;
  const int32_t* __restrict__ slice_grp = a.slice_grp;

  const int32_t cbeg = static_cast<int32_t>(w * a.chunk);
  const int32_t cend = static_cast<int32_t>(min64(cbeg + a.chunk, a.n_groups));
  int32_t sl = a.item_pos[w];
  int32_t sl_end = slice_grp[sl + 1];
  bool head = slice_grp[sl] < cbeg;
  int32_t row = t.idx[0][sl];
  bool pending = false;
  double4 acc = make_double4(0, 0, 0, 0);
  const bool colok = c < R;

  auto flush = [&](int dslot) {
    double v[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      v[e] += __shfl_xor_sync(0xffffffffu, v[e], 8);
      v[e] += __shfl_xor_sync(0xffffffffu, v[e], 16);
    }
    if (slot == 0) {
      double* dst = dslot < 0 ? a.out + static_cast<int64_t>(row) * R
                              : a.part + (w * 2 + dslot) * static_cast<int64_t>(R);
      store4(dst, c, R, make_double4(v[0], v[1], v[2], v[3]));
    }
    acc = make_double4(0, 0, 0, 0);
  };
  auto rowq = [&](const double* base, int32_t r, bool pred) {
    if (VEC) return ld256_if(base + static_cast<int64_t>(r) * R + c, pred && colok);
    return pred ? row4<false>(base + static_cast<int64_t>(r) * R, c, R) : make_double4(0, 0, 0, 0);
  };

  for (int32_t g = cbeg; g < cend; ++g) {
    const int4 hh = __ldg(hdr + g);
    const int n = hh.y;  // warp-uniform
    const int64_t gs = static_cast<int64_t>(g) * kSlots + slot;
    const int32_t u = __ldg(gnode + gs);
    const int32_t j = ORDER == 4 ? __ldg(gnode1 + gs) : 0;
    int32_t kk[4];
    double tt[4];
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      const bool on = it < n;
      kk[it] = on ? __ldg(pk + hh.x + it * kSlots + slot) : 0;
      tt[it] = on ? __ldg(pv + hh.x + it * kSlots + slot) : 0.0;
    }
    const double4 ur = rowq(Funit, u, true);
    double4 tr = make_double4(0, 0, 0, 0);
    if (ORDER == 4) tr = rowq(Ftop, j, true);
    double4 rr[4];
#pragma unroll
    for (int it = 0; it < 4; ++it) rr[it] = rowq(Fleaf, kk[it], it < n);
    double4 X = make_double4(0, 0, 0, 0);
#pragma unroll
    for (int it = 0; it < 4; ++it) fma4(X, tt[it], rr[it]);  // X += t * F_leaf[k]
    if (ORDER == 3) {
      fma4v(acc, X, ur);  // A[i] += X * B[j]
    } else {
      const double4 Y = make_double4(X.x * ur.x, X.y * ur.y, X.z * ur.z, X.w * ur.w);
      fma4v(acc, Y, tr);  // A[i] += (X * C[k]) * B[j]
    }
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

// Packed + TMA-staged (default): k_mttkrp_pk's lane mapping and math, with
// each window of kMW groups — headers, slot coordinates (both levels for
// order 4) and the interleaved leaf coordinate / value streams, contiguous
// and 16-byte aligned in the packed layout — staged into shared memory by
// lane 0 with bulk copies (meta two windows ahead, leaves one), completing on
// per-stage mbarriers. k_mttkrp_pk loaded them with __ldg right before the
// gathers they feed: two dependent L2 round trips per group (ncu: long
// scoreboard 67 %, data pipe 57 %).
constexpr int kMSlots = 4;

// MW = groups per window (leaves per window: MW * kMSlots * 4, len <= 4)
template <int MW>
struct StageM {
  alignas(16) int4 hdr[3][MW];
  alignas(16) int32_t node[3][MW * kMSlots];
  alignas(16) int32_t node1[3][MW * kMSlots];
  alignas(16) int32_t kk[2][MW * kMSlots * 4];
  alignas(16) double tv[2][MW * kMSlots * 4];
  uint64_t mbar_meta[3];
  uint64_t mbar_leaf[2];
};

// RC = compile-time rank (32 at the BASELINE shapes: full 256-byte rows over
// 8 lanes, constant row strides, no column predicates) or 0 = a.R at run time
// CLK: diagnostics instantiation (SPTTN_ITEM_CLOCKS=1), per item {start ns,
// end ns, SM, groups, leaf steps, tile flushes}
template <int ORDER, bool VEC, int RC = 0, bool CLK = false, int MW = 8>
__global__ void __launch_bounds__(kBlock, 3) k_mttkrp_pq(RootOutArgs a) {
  constexpr int kMW = MW;
  constexpr int kMWLeaves = MW * kMSlots * 4;
  grid_launch_dependents();
  extern __shared__ __align__(16) unsigned char pq_smem_raw[];
  StageM<MW>* stage = reinterpret_cast<StageM<MW>*>(pq_smem_raw);
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * kBlock + threadIdx.x) / 32;
  if (w >= a.n_items) return;  // warp-uniform
  if (CLK && (threadIdx.x & 31) == 0) a.clk[6 * w] = globaltimer_ns();
  int dbg_steps = 0, dbg_flush = 0;
  StageM<MW>& S = stage[threadIdx.x / 32];
  const int lane = threadIdx.x & 31;
  const int slot = lane >> 3;
  const int c = (lane & 7) * 4;
  const int R = RC > 0 ? RC : a.R;
  const CsfView& t = a.t;
  const double* __restrict__ Fleaf = a.f[ORDER - 1];
  const double* __restrict__ Funit = a.f[ORDER - 2];
  const double* __restrict__ Ftop = a.f[1];
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
  // order 4: the B[j] row stays in registers while consecutive groups give
  // the lane's slot segments of the same (i,j) fiber (predicated-off load)
  int32_t prev_j = -1;
  double4 brow = make_double4(0, 0, 0, 0);
  double4 acc = make_double4(0, 0, 0, 0);
  const bool colok = RC > 0 ? true : c < R;

  auto flush = [&](int dslot) {
    double v[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      v[e] += __shfl_xor_sync(0xffffffffu, v[e], 8);
      v[e] += __shfl_xor_sync(0xffffffffu, v[e], 16);
    }
    if (slot == 0) {
      double* dst = dslot < 0 ? a.out + static_cast<int64_t>(row) * R
                              : a.part + (w * 2 + dslot) * static_cast<int64_t>(R);
      if (VEC && RC > 0)  // full 32-byte sectors (R = RC: every quad in range, aligned)
        *reinterpret_cast<double4*>(dst + c) = make_double4(v[0], v[1], v[2], v[3]);
      else
        store4(dst, c, R, make_double4(v[0], v[1], v[2], v[3]));
    }
    acc = make_double4(0, 0, 0, 0);
  };
  auto rowq = [&](const double* base, int32_t r, bool pred) {
    // full rows (RC > 0): every lane's quad is in range, no zero-fill / predicate
    if (VEC && RC > 0) return ld256(base + static_cast<int64_t>(r) * R + c);
    if (VEC) return ld256_if(base + static_cast<int64_t>(r) * R + c, pred && colok);
    return pred ? row4<false>(base + static_cast<int64_t>(r) * R, c, R) : make_double4(0, 0, 0, 0);
  };
  auto issue_meta = [&](int32_t wi) {
    const int32_t g0 = cbeg + wi * kMW;
    const int32_t nw = min(g0 + kMW, cend) - g0;
    const int b = wi % 3;
    const unsigned hb = nw * sizeof(int4), nb = nw * kMSlots * sizeof(int32_t);
    fence_proxy_async();
    expect_tx_elect(&S.mbar_meta[b], hb + (ORDER == 4 ? 2 : 1) * nb);
    bulk_g2s_elect(&S.hdr[b][0], a.grp_hdr + g0, hb, &S.mbar_meta[b]);
    bulk_g2s_elect(&S.node[b][0], a.grp_node + static_cast<int64_t>(g0) * kMSlots, nb, &S.mbar_meta[b]);
    if (ORDER == 4)
      bulk_g2s_elect(&S.node1[b][0], a.grp_node1 + static_cast<int64_t>(g0) * kMSlots, nb,
               &S.mbar_meta[b]);
  };
  auto issue_leaves = [&](int32_t wi) {
    const int32_t g0 = cbeg + wi * kMW;
    const int32_t nw = min(g0 + kMW, cend) - g0;
    const int b = wi % 3, lb = wi & 1;
    mbar_wait(&S.mbar_meta[b], (wi / 3) & 1);
    const int32_t L0 = uni(S.hdr[b][0].x);
    const int32_t L1 = uni(S.hdr[b][nw - 1].x + kMSlots * S.hdr[b][nw - 1].y);
    const unsigned n = static_cast<unsigned>(L1 - L0);
    SPTTN_DCHECK(n <= static_cast<unsigned>(kMWLeaves));
    fence_proxy_async();
    expect_tx_elect(&S.mbar_leaf[lb], n * 12u);
    bulk_g2s_elect(&S.kk[lb][0], a.pk + L0, n * 4u, &S.mbar_leaf[lb]);
    bulk_g2s_elect(&S.tv[lb][0], a.pv + L0, n * 8u, &S.mbar_leaf[lb]);
  };

  const int32_t nwin = (cend - cbeg + kMW - 1) / kMW;
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
    const int32_t g0 = cbeg + win * kMW;
    const int32_t ge = min(g0 + kMW, cend);
    const int32_t L0 = S.hdr[mb][0].x;
    for (int32_t g = g0; g < ge; ++g) {
      const int4 hh = S.hdr[mb][g - g0];
      const int n = hh.y;  // warp-uniform
      if (CLK) dbg_steps += n;
      const int32_t u = S.node[mb][(g - g0) * kMSlots + slot];
      const int32_t j = ORDER == 4 ? S.node1[mb][(g - g0) * kMSlots + slot] : 0;
      const int32_t lbase = hh.x - L0 + slot;
      SPTTN_DCHECK(u >= 0 && u < a.frows[ORDER - 2]);
      SPTTN_DCHECK(ORDER == 3 || (j >= 0 && j < a.frows[1]));
      SPTTN_DCHECK(lbase + (n - 1) * kMSlots < kMWLeaves);
      const double4 ur = rowq(Funit, u, true);
      double4 tr = make_double4(0, 0, 0, 0);
      if (ORDER == 4) {
        const bool fresh = j != prev_j;
        if (VEC) {  // reload only for a new fiber; otherwise the registers keep B[j]
          ld256_keep(brow, Ftop + static_cast<int64_t>(j) * R + c, fresh && colok);
        } else if (fresh) {
          brow = row4<false>(Ftop + static_cast<int64_t>(j) * R, c, R);
        }
        prev_j = j;
        tr = brow;
      }
      // X += t * F_leaf[k] over the group's n (warp-uniform) leaf steps: the
      // body is specialised per n, so no predicated-off stream loads, row
      // gathers or FMAs are issued for short segments (most have 1 leaf)
      double4 X = make_double4(0, 0, 0, 0);
      auto steps = [&](auto NS) {
        constexpr int kN = decltype(NS)::value;
        int32_t kk[kN];
        double tt[kN];
#pragma unroll
        for (int it = 0; it < kN; ++it) {
          kk[it] = S.kk[lbf][lbase + it * kMSlots];
          tt[it] = S.tv[lbf][lbase + it * kMSlots];
        }
        double4 rr[kN];
#pragma unroll
        for (int it = 0; it < kN; ++it) SPTTN_DCHECK(kk[it] >= 0 && kk[it] < a.frows[ORDER - 1]);
#pragma unroll
        for (int it = 0; it < kN; ++it) rr[it] = rowq(Fleaf, kk[it], true);
        // first step as a product (= fma with a zero addend, bit for bit)
        X = make_double4(tt[0] * rr[0].x, tt[0] * rr[0].y, tt[0] * rr[0].z, tt[0] * rr[0].w);
#pragma unroll
        for (int it = 1; it < kN; ++it) fma4(X, tt[it], rr[it]);
      };
      switch (n) {
        case 1: steps(std::integral_constant<int, 1>{}); break;
        case 2: steps(std::integral_constant<int, 2>{}); break;
        case 3: steps(std::integral_constant<int, 3>{}); break;
        default: steps(std::integral_constant<int, 4>{}); break;
      }
      if (ORDER == 3) {
        fma4v(acc, X, ur);  // A[i] += X * B[j]
      } else {
        const double4 Y = make_double4(X.x * ur.x, X.y * ur.y, X.z * ur.z, X.w * ur.w);
        fma4v(acc, Y, tr);  // A[i] += (X * C[k]) * B[j]
      }
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

void launch_mttkrp_pq(const RootOutArgs& a, int order, cudaStream_t s) {
  const int64_t blocks = (a.n_items * 32 + kBlock - 1) / kBlock;
  if (blocks == 0) return;
  const unsigned b = static_cast<unsigned>(blocks);
  auto gow = [&](auto kern, size_t sm) {  // items are sized for 3 resident CTAs per SM
    SPTTN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(sm)));
    // order 4: the largest shared-memory split (smallest L1) measured fastest
    pin_carveout(kern, 3, sm, order == 4 ? 100 : -1);
    kern<<<b, kBlock, sm, s>>>(a);
  };
  auto go = [&](auto kern) { gow(kern, sizeof(StageM<8>) * (kBlock / 32)); };
  // order 4, R = 32: windows of 16 groups (the 100 % carveout leaves room for
  // 3 x 68 KB of staging): 565 -> 553 us; SPTTN_M4_WIN=8 selects the 8-group windows
  static const int mw = std::getenv("SPTTN_M4_WIN") ? std::atoi(std::getenv("SPTTN_M4_WIN")) : 16;
  if (order == 4 && a.vec && a.R == 32 && mw == 16) {
    const size_t sm = sizeof(StageM<16>) * (kBlock / 32);
    if (a.clk) gow(k_mttkrp_pq<4, true, 32, true, 16>, sm);
    else gow(k_mttkrp_pq<4, true, 32, false, 16>, sm);
    SPTTN_CUDA(cudaGetLastError());
    return;
  }
  if (order == 3) {
    if (a.vec) go(k_mttkrp_pq<3, true>);
    else go(k_mttkrp_pq<3, false>);
  } else {
    if (a.vec && a.R == 32 && a.clk) go(k_mttkrp_pq<4, true, 32, true>);
    else if (a.vec && a.R == 32) go(k_mttkrp_pq<4, true, 32>);
    else if (a.vec) go(k_mttkrp_pq<4, true>);
    else go(k_mttkrp_pq<4, false>);
  }
  SPTTN_CUDA(cudaGetLastError());
}

void launch_mttkrp_pk(const RootOutArgs& a, cudaStream_t s) {  // order 3
  const int64_t blocks = (a.n_items * 32 + kBlock - 1) / kBlock;
  if (blocks == 0) return;
  const unsigned b = static_cast<unsigned>(blocks);
  auto go = [&](auto kern) {
    pin_carveout(kern, 4, 0);
    kern<<<b, kBlock, 0, s>>>(a);
  };
  if (a.vec) go(k_mttkrp_pk<3, true>);
  else go(k_mttkrp_pk<3, false>);
  SPTTN_CUDA(cudaGetLastError());
}

// ---- MTTKRP-3 for the non-root output modes ------------
//
// On the same (i,j,k) CSF, the other two CP-ALS products:
//   mode j  ((T*C)*A), orders e.g. (i,j,r,k)(i,j,r):
//       per (i,j)  X[r] = sum_k t * C[k,r];   B[j,r] += X[r] * A[i,r]
//   mode k  ((A*B)*T), orders e.g. (i,j,r)(i,j,r,k):
//       per (i,j)  W[r] = A[i,r] * B[j,r];    per leaf  C[k,r] += W[r] * t
// The output row is not owned by a root slice, so contributions are added
// with fp64 atomics (RED.E.ADD.F64) — the "atomics only where the output mode
// is not the root" half of the north star. The work layout is the packed
// 4-slot groups of (i,j) segments of the mode-i kernel; a group belongs to
// one root slice, whose A[i] row a warp loads once per slice. Warps stride
// over groups; no items or fix-up. Summation order varies run to run (atomic
// arrival), within the fp64 tolerance.
namespace {

template <int MODE, bool VEC>
__global__ void __launch_bounds__(kBlock, 3) k_mttkrp3_nonroot(RootOutArgs a) {
  const int lane = threadIdx.x & 31;
  const int slot = lane >> 3;
  const int c = (lane & 7) * 4;
  const int R = a.R;
  const CsfView& t = a.t;
  const double* __restrict__ A = a.f[0];
  const double* __restrict__ F = a.f[1];  // C[k] (mode j) or B[j] (mode k)
  const int4* __restrict__ hdr = a.grp_hdr;
  const int32_t* __restrict__ gnode = a.grp_node;
  const int32_t* __restrict__ pk = a.pk;
  const double* __restrict__ pv = a.pv;
  const bool colok = c < R;
  auto rowq = [&](const double* base, int32_t r, bool pred) {
    if (VEC) return ld256_if(base + static_cast<int64_t>(r) * R + c, pred && colok);
    return pred ? row4<false>(base + static_cast<int64_t>(r) * R, c, R) : make_double4(0, 0, 0, 0);
  };
  auto red4 = [&](int32_t row, const double4& v, bool on) {
    if (!on) return;
    double* dst = a.out + static_cast<int64_t>(row) * R + c;
    if (c + 0 < R) atomicAdd(dst + 0, v.x);
    if (c + 1 < R) atomicAdd(dst + 1, v.y);
    if (c + 2 < R) atomicAdd(dst + 2, v.z);
    if (c + 3 < R) atomicAdd(dst + 3, v.w);
  };
  const int64_t nw = static_cast<int64_t>(gridDim.x) * (kBlock / 32);
  int32_t cur_slice = -1;
  double4 ar = make_double4(0, 0, 0, 0);
  for (int64_t g = static_cast<int64_t>(blockIdx.x) * (kBlock / 32) + threadIdx.x / 32;
       g < a.n_groups; g += nw) {
    const int4 hh = __ldg(hdr + g);
    const int n = hh.y;  // warp-uniform
    const bool live = slot < hh.z;
    if (hh.w != cur_slice) {  // warp-uniform: A[i] once per root slice
      cur_slice = hh.w;
      ar = rowq(A, __ldg(t.idx[0] + cur_slice), true);
    }
    const int32_t j = __ldg(gnode + g * 4 + slot);
    int32_t kk[4];
    double tt[4];
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      const bool on = it < n;
      kk[it] = on ? __ldg(pk + hh.x + it * 4 + slot) : 0;
      tt[it] = on ? __ldg(pv + hh.x + it * 4 + slot) : 0.0;
    }
    if (MODE == 1) {  // B[j] += (sum_k t C[k]) * A[i]
      double4 rr[4];
#pragma unroll
      for (int it = 0; it < 4; ++it) rr[it] = rowq(F, kk[it], it < n);
      double4 X = make_double4(0, 0, 0, 0);
#pragma unroll
      for (int it = 0; it < 4; ++it) fma4(X, tt[it], rr[it]);
      red4(j, make_double4(X.x * ar.x, X.y * ar.y, X.z * ar.z, X.w * ar.w), live);
    } else {  // C[k] += (A[i] * B[j]) * t
      const double4 br = rowq(F, j, true);
      const double4 W = make_double4(ar.x * br.x, ar.y * br.y, ar.z * br.z, ar.w * br.w);
#pragma unroll
      for (int it = 0; it < 4; ++it)
        if (it < n)
          red4(kk[it], make_double4(W.x * tt[it], W.y * tt[it], W.z * tt[it], W.w * tt[it]), live);
    }
  }
}

}  // namespace

void launch_mttkrp3_nonroot(const RootOutArgs& a, int mode, cudaStream_t s) {
  if (a.n_groups == 0) return;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (a.n_groups + 7) / 8;
  const unsigned b = static_cast<unsigned>(std::min<int64_t>(want, static_cast<int64_t>(sms) * 3 * 4));
  if (mode == 1) {
    if (a.vec) k_mttkrp3_nonroot<1, true><<<b, kBlock, 0, s>>>(a);
    else k_mttkrp3_nonroot<1, false><<<b, kBlock, 0, s>>>(a);
  } else {
    if (a.vec) k_mttkrp3_nonroot<2, true><<<b, kBlock, 0, s>>>(a);
    else k_mttkrp3_nonroot<2, false><<<b, kBlock, 0, s>>>(a);
  }
  SPTTN_CUDA(cudaGetLastError());
}

}  // namespace spttn_dev
