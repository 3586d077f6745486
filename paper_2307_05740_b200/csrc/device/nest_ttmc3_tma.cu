// TTMc-3 with TMA gather4 factor-row loads (mode 11).
//
// Same nest and work layout as k_ttmc3pq (packed 8-slot groups of <= 4-leaf
// (i,j) segments, warp items of consecutive groups, HEAD/TAIL partial tiles),
// but the factor rows never pass through the LSU: every U[j] and V[k] row of
// a group is fetched by `cp.async.bulk.tensor.2d.tile::gather4` (4 rows per
// instruction, SASS UTMALDG.2D.GATHER4) into a per-warp ring of 1 KB blocks
// with the 128-byte swizzle, completing on a per-group mbarrier. The rows of
// a block are placed so that the DMMA fragments can be read straight out of
// it with conflict-free 128-bit loads:
//   block line of slot s = 2*(s%4) + s/4        (K-chunk kc = s/4, k = s%4)
//   lane (fq = L%4, fh = L/4) reads line 2*fq + kc, 16-byte chunk fh, which
//   the swizzle puts at chunk fh ^ (2*fq + kc): 8 distinct chunks per quarter
//   warp.
// Each lane thus holds columns (2fh, 2fh+1) of its segment's rows — the DMMA
// M / N tiles are taken over the interleaved columns (r = 2*row + mt,
// s = 2*col + nt) — so X = sum t * V[k] is accumulated directly in fragment
// order and no shared-memory transpose is needed. The LSU only reads each
// gathered row once from shared memory (1 wavefront per row) plus the small
// per-group value / header traffic.
#include <cuda.h>

#include "internal.cuh"

namespace spttn_dev {

namespace {

constexpr int kTgBlock = 128;   // threads per CTA (4 warps)
constexpr int kTgRing = 8;      // 1 KB row blocks per warp
constexpr int kTgSlots = 4;     // groups in flight per warp (>= 2 blocks each)
constexpr int kTgW = 4;         // groups per stream window
constexpr int kTgWin = 4;       // stream window stages (window w in stage w % kTgWin)
constexpr int kTgWLeaves = kTgW * kPackSlots * 4;

struct TgWarp {
  alignas(1024) unsigned char ring[kTgRing][1024];
  // stream windows: headers, slot coordinates, leaf coordinates and values
  alignas(16) int4 hdr[kTgWin][kTgW];
  alignas(16) int32_t node[kTgWin][kTgW * kPackSlots];
  alignas(16) int32_t kk[kTgWin][kTgWLeaves];
  alignas(16) double tv[kTgWin][kTgWLeaves];
  int32_t blk0[kTgSlots];
  uint64_t mbar_win[kTgWin];
  uint64_t mbar_grp[kTgSlots];
};
constexpr size_t kTgSmem = sizeof(TgWarp) * (kTgBlock / 32) + 1024;

__device__ __forceinline__ void gather4(void* dst, const CUtensorMap* map, int r0, int r1, int r2,
                                        int r3, uint64_t* m) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(m));
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(d),
      "l"(map), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(b)
      : "memory");
}

__device__ __forceinline__ double2 lds128(const void* p) {
  double2 v;
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(p));
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}

__global__ void __launch_bounds__(kTgBlock) k_ttmc3tg(RootOutArgs a,
                                                     const __grid_constant__ CUtensorMap mapU,
                                                     const __grid_constant__ CUtensorMap mapV) {
  extern __shared__ unsigned char tg_raw[];
  TgWarp* warps = reinterpret_cast<TgWarp*>(
      (reinterpret_cast<uintptr_t>(tg_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * kTgBlock + threadIdx.x) / 32;
  if (w >= a.n_items) return;  // warp-uniform
  TgWarp& S = warps[threadIdx.x / 32];
  const int lane = threadIdx.x & 31;
  const int fq = lane & 3, fh = lane >> 2;
  const int R = a.R, S_ = a.S;
  const CsfView& t = a.t;
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
          const int r = 2 * fh + mt;
          const int s = 2 * (2 * fq + e) + nt;
          dst[r * S_ + s] = acc[(mt * 2 + nt) * 2 + e];
        }
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.0;
  };

  const int32_t nwin = (cend - cbeg + kTgW - 1) / kTgW;
  // lane 0: stage window wi (headers, slot coordinates, leaf streams) with
  // bulk copies; its leaf range comes from two header reads
  auto load_window = [&](int32_t wi) {
    const int32_t g0 = cbeg + wi * kTgW;
    const int32_t nw = min(g0 + kTgW, cend) - g0;
    const int b = wi % kTgWin;
    const int32_t L0 = __ldg(&a.grp_hdr[g0].x);
    const int4 hl = __ldg(a.grp_hdr + g0 + nw - 1);
    const int32_t L1 = hl.x + kPackSlots * hl.y;
    const unsigned nl = static_cast<unsigned>(L1 - L0);
    const unsigned hb = nw * sizeof(int4), nb = nw * kPackSlots * sizeof(int32_t);
    fence_proxy_async();
    mbar_expect_tx(&S.mbar_win[b], hb + nb + 12u * nl);
    bulk_g2s(&S.hdr[b][0], a.grp_hdr + g0, hb, &S.mbar_win[b]);
    bulk_g2s(&S.node[b][0], a.grp_node + static_cast<int64_t>(g0) * kPackSlots, nb, &S.mbar_win[b]);
    bulk_g2s(&S.kk[b][0], a.pk + L0, 4u * nl, &S.mbar_win[b]);
    bulk_g2s(&S.tv[b][0], a.pv + L0, 8u * nl, &S.mbar_win[b]);
  };

  if (lane == 0) {
    for (int b = 0; b < kTgWin; ++b) mbar_init(&S.mbar_win[b], 1);
    for (int b = 0; b < kTgSlots; ++b) mbar_init(&S.mbar_grp[b], 1);
    mbar_init_fence();
    for (int wi = 0; wi < kTgWin && wi < nwin; ++wi) load_window(wi);
  }
  __syncwarp();

  int32_t gi = cbeg, gc = cbeg;  // next group to issue / to consume
  int32_t ring_head = 0, ring_used = 0;
  int32_t win_ready = -1;  // highest window known complete (warp-uniform)
  auto window_wait = [&](int32_t wi) {
    if (wi > win_ready) {
      mbar_wait(&S.mbar_win[wi % kTgWin], static_cast<unsigned>((wi / kTgWin) & 1));
      win_ready = wi;
    }
  };
  // lane m issues gather4 m of the group: m = 0, 1 -> U rows of slots
  // {2m, 4+2m, 2m+1, 5+2m}; m = 2 + 2*it + h -> V rows of leaf it of slots
  // {2h, 4+2h, 2h+1, 5+2h}. Block line of slot s = 2*(s%4) + s/4.
  const int m = lane;
  const int mh = m < 2 ? m : (m - 2) & 1;
  const int mit = m < 2 ? 0 : (m - 2) >> 1;
  auto issue = [&]() {
    const int32_t wi = (gi - cbeg) / kTgW;
    window_wait(wi);
    const int b = wi % kTgWin, q = (gi - cbeg) % kTgW;
    const int4 hh = S.hdr[b][q];
    const int n = hh.y;
    const int32_t lb = hh.x - S.hdr[b][0].x;
    const int slot = (gi - cbeg) % kTgSlots;
    const int b0 = ring_head;
    int rr[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int sidx = (k & 1) ? 4 + 2 * mh + (k >> 1) : 2 * mh + (k >> 1);
      rr[k] = m < 2 ? S.node[b][q * kPackSlots + sidx]
                    : (m < 2 + 2 * n ? S.kk[b][lb + 8 * mit + sidx] : 0);
    }
    if (lane == 0) {
      S.blk0[slot] = b0;
      mbar_expect_tx(&S.mbar_grp[slot], static_cast<unsigned>((2 + 2 * n) * 512));
    }
    __syncwarp();
    if (m < 2 + 2 * n) {
      fence_proxy_async();  // the ring block was last read through the generic proxy
      const int blk = m < 2 ? b0 : (b0 + 1 + mit) % kTgRing;
      gather4(&S.ring[blk][(m & 1) * 512], m < 2 ? &mapU : &mapV, rr[0], rr[1], rr[2], rr[3],
              &S.mbar_grp[slot]);
    }
    ring_head = (ring_head + 1 + n) % kTgRing;
    ring_used += 1 + n;
    ++gi;
  };

  while (gc < cend) {
    // keep the ring full (the next group's size needs its window)
    while (gi < cend && gi - gc < kTgSlots) {
      const int32_t wi = (gi - cbeg) / kTgW;
      window_wait(wi);
      const int nn = S.hdr[wi % kTgWin][(gi - cbeg) % kTgW].y;
      if (ring_used + 1 + nn > kTgRing) break;
      issue();
    }
    const int32_t wc = (gc - cbeg) / kTgW;
    const int b = wc % kTgWin, q = (gc - cbeg) % kTgW;
    const int4 hh = S.hdr[b][q];
    const int n = hh.y;
    const int32_t lb = hh.x - S.hdr[b][0].x;
    const int slot = (gc - cbeg) % kTgSlots;
    mbar_wait(&S.mbar_grp[slot], static_cast<unsigned>(((gc - cbeg) / kTgSlots) & 1));
    const int b0 = S.blk0[slot];
    double2 x[2] = {make_double2(0, 0), make_double2(0, 0)};
    double2 u[2];
#pragma unroll
    for (int kc = 0; kc < 2; ++kc) {
      const int line = 2 * fq + kc;
      const int off = line * 128 + ((fh ^ line) << 4);
      u[kc] = lds128(&S.ring[b0][off]);
#pragma unroll
      for (int it = 0; it < 4; ++it) {
        if (it < n) {
          const double tv = S.tv[b][lb + 8 * it + 4 * kc + fq];
          const double2 v = lds128(&S.ring[(b0 + 1 + it) % kTgRing][off]);
          x[kc].x = fma(tv, v.x, x[kc].x);  // X[s] += t * V[k,s]
          x[kc].y = fma(tv, v.y, x[kc].y);
        }
      }
    }
    __syncwarp();  // every lane has read the group's blocks and window entries
    ring_used -= 1 + n;
    // window wc fully consumed: refill its stage with window wc + kTgWin
    if ((q == kTgW - 1 || gc + 1 == cend) && lane == 0 && wc + kTgWin < nwin)
      load_window(wc + kTgWin);
#pragma unroll
    for (int kc = 0; kc < 2; ++kc) {
      dmma_8x8x4(acc[0], acc[1], u[kc].x, x[kc].x);  // (mt 0, nt 0)
      dmma_8x8x4(acc[2], acc[3], u[kc].x, x[kc].y);  // (mt 0, nt 1)
      dmma_8x8x4(acc[4], acc[5], u[kc].y, x[kc].x);  // (mt 1, nt 0)
      dmma_8x8x4(acc[6], acc[7], u[kc].y, x[kc].y);  // (mt 1, nt 1)
    }
    pending = true;
    if (gc + 1 == sl_end) {
      flush(head ? 0 : -1);
      pending = false;
      head = false;
      if (gc + 1 < cend) {
        ++sl;
        sl_end = nx_end;
        row = nx_row;
        nx_end = sl + 2 <= t.nlev[0] ? __ldg(slice_grp + sl + 2) : 0;
        nx_row = sl + 1 < t.nlev[0] ? __ldg(t.idx[0] + sl + 1) : 0;
      }
    }
    ++gc;
  }
  if (pending) flush(head ? 0 : 1);
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

}  // namespace

bool ttmc3_tma_supported(int R, int S) { return R == 16 && S == 16 && encode_fn() != nullptr; }

// A [rows x 16] fp64 row-major factor as a 2D tensor map for gather4: box
// 16 columns x 1 row, 128-byte swizzle.
void make_row_map(void* map, const double* base, int64_t rows) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) throw Status(4, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t gdim[2] = {16, static_cast<cuuint64_t>(rows)};
  cuuint64_t gstride[1] = {16 * sizeof(double)};
  cuuint32_t box[2] = {16, 1};
  cuuint32_t estr[2] = {1, 1};
  const CUresult r = enc(static_cast<CUtensorMap*>(map), CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
                         const_cast<double*>(base), gdim, gstride, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Status(4, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
}

void launch_ttmc3_tma(const RootOutArgs& a, const void* mapU, const void* mapV, cudaStream_t s) {
  const int64_t blocks = (a.n_items * 32 + kTgBlock - 1) / kTgBlock;
  if (blocks == 0) return;
  static bool attr = false;
  if (!attr) {
    SPTTN_CUDA(cudaFuncSetAttribute(k_ttmc3tg, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kTgSmem)));
    attr = true;
  }
  k_ttmc3tg<<<static_cast<unsigned>(blocks), kTgBlock, kTgSmem, s>>>(
      a, *static_cast<const CUtensorMap*>(mapU), *static_cast<const CUtensorMap*>(mapV));
  SPTTN_CUDA(cudaGetLastError());
}

}  // namespace spttn_dev
