// MTTKRP-3 with the leaf factor resident in shared memory (default when it
// fits).
//
// Reference nest ((T*C)*B), orders (i,j,k,a)(i,j,a) (proj/src/executor.cpp:
// 453-490, vector-accumulate hook :411-451, micro_kernels.hpp:11-16):
//     per (i,j)  X[a] = sum_k t * C[k,a];     A[i,a] += X[a] * B[j,a]
//
// k_mttkrp_pk gathers a 256-byte C[k] row per leaf and a B[j] row per fiber
// through L1 from a 512 KB working set (BASELINE: 1000 x 32 factors) that
// does not fit in L1, so most rows come from L2 and every group waits out an
// L2 round trip (ncu: latency-bound, 49 us for 0.42 GB of row reads).
//
// Here the rank columns are cut into halves of 16 (128-byte rows). The CTA
// for half h keeps C[:, 16h:16h+16] in shared memory — rows_C * 128 bytes,
// 128 KB at the BASELINE shape — loaded once per CTA with cp.async, so the
// per-leaf row read (the bulk of the traffic) is an LDS.128 by 8 lanes per
// row: a full 128-byte row per shared-memory wavefront, free of bank
// conflicts by construction (a 64-byte quarter-row layout measured 1.5
// wavefronts per row pair: two random rows share a bank line). The per-fiber
// B[j] half rows (128 bytes) are gathered from L2 one group ahead into
// registers. The CSF streams are the packed length-sorted 8-slot groups
// (pack.cu) with plan-time pre-scaled offsets (leaf coordinate -> byte
// offset of its C row in shared memory, fiber coordinate -> element offset of
// its B row), staged per warp in windows of 4 groups by TMA bulk copies on
// mbarriers (metadata two windows ahead, leaves one). Lane L = 8p + c works
// on slots 2p, 2p+1 and on columns 16h + 2c, 16h + 2c + 1.
//
// Work split without a fix-up pass: the plan cuts the group sequence into
// one range per CTA at root-slice boundaries (balanced by groups,
// `cta_grp`), so a slice never spans CTAs; the CTA's warps take equal group
// ranges. Slices interior to a warp's range are reduced over the slots
// (shuffles) and written once (owner computes); the first and last slice
// piece of every warp go to shared memory and one warp sums them in warp
// order — a fixed order, so results are bit-reproducible. Absent root rows
// are zeroed by the same kernel: one launch per execute.
#include "internal.cuh"

namespace spttn_dev {

namespace {

constexpr int kSmfWarps = 24;
constexpr int kSW = 4;                        // groups per staged window
constexpr int kSSlots = 8;                    // segments per group
constexpr int kSWLeaves = kSW * kSSlots * 4;  // leaves per window (segment length <= 4)
constexpr int kHalf = 16;                     // columns per CTA (128-byte rows)

struct StageS {
  alignas(16) int2 hdr[3][kSW + 2];           // {leaf base, slice * 8 + length}; +1 lead, +1 tail
  alignas(16) int32_t node[3][kSW * kSSlots];  // B row element offsets
  alignas(16) int32_t kk[2][kSWLeaves];        // C row byte offsets in shared memory
  alignas(16) double tv[2][kSWLeaves];
  uint64_t mbar_meta[3];
  uint64_t mbar_leaf[2];
};

__device__ __forceinline__ void mbar_inval(uint64_t* m) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(m));
  asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(a) : "memory");
}

__device__ __forceinline__ double2 lds128(unsigned addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}

struct Piece {
  double v[kHalf];
  int32_t slice;
  int32_t pad[3];
};

__global__ void __launch_bounds__(kSmfWarps * 32, 1) k_mttkrp3_smf(RootOutArgs a, SmfArgs x) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int NT = kSmfWarps * 32;
  const int tid = threadIdx.x;
  const int wid = uni(tid >> 5);
  const int lane = tid & 31;
  const int sp = lane >> 3;  // slots 2sp, 2sp+1
  const int cq = lane & 7;   // columns 2cq, 2cq+1 of the half
  const int h = blockIdx.x % x.nq;
  const int cta = blockIdx.x / x.nq;
  const int R = a.R;
  const unsigned cs = static_cast<unsigned>(__cvta_generic_to_shared(smem)) + 16u * cq;
  StageS* stages = reinterpret_cast<StageS*>(smem + static_cast<int64_t>(x.rows_c) * 128);
  StageS& S = stages[wid];
  const double* __restrict__ Bh = a.f[1] + kHalf * h + 2 * cq;

  // 1. C[:, 16h:16h+16] -> shared memory (16-byte cp.async, L2 only)
  {
    const double* C = a.f[2];
    const int32_t n16 = x.rows_c * 8;
    for (int32_t e = tid; e < n16; e += NT) {
      const double* src = C + static_cast<int64_t>(e >> 3) * R + kHalf * h + 2 * (e & 7);
      cp_async16_cg(smem + static_cast<int64_t>(e) * 16, src, 16);
    }
    cp_async_commit();
  }

  // 2. this warp's group range inside the CTA's slice-aligned range
  const int32_t G0 = __ldg(x.cta_grp + cta), G1 = __ldg(x.cta_grp + cta + 1);
  const int32_t cbeg =
      uni(G0 + static_cast<int32_t>((static_cast<int64_t>(G1 - G0) * wid) / kSmfWarps));
  const int32_t cend =
      uni(G0 + static_cast<int32_t>((static_cast<int64_t>(G1 - G0) * (wid + 1)) / kSmfWarps));

  auto issue_meta = [&](int32_t wi) {
    const int32_t g0 = cbeg + wi * kSW;
    const int32_t nw = min(g0 + kSW, cend) - g0;
    const int b = wi % 3;
    // 16-byte aligned source: start at the even group <= g0 (hdr2 is padded
    // by 2 entries, so the rounded-up tail stays inside it)
    const unsigned hb = ((static_cast<unsigned>(nw + (g0 & 1)) * 8u) + 15u) & ~15u;
    const unsigned nb = nw * kSSlots * sizeof(int32_t);
    fence_proxy_async();
    expect_tx_elect(&S.mbar_meta[b], hb + nb);
    bulk_g2s_elect(&S.hdr[b][0], x.hdr2 + (g0 & ~1), hb, &S.mbar_meta[b]);
    bulk_g2s_elect(&S.node[b][0], a.grp_node + static_cast<int64_t>(g0) * kSSlots, nb,
                   &S.mbar_meta[b]);
  };
  auto issue_leaves = [&](int32_t wi) {
    const int32_t g0 = cbeg + wi * kSW;
    const int32_t nw = min(g0 + kSW, cend) - g0;
    const int b = wi % 3, lb = wi & 1;
    mbar_wait(&S.mbar_meta[b], (wi / 3) & 1);
    const int o = g0 & 1;
    const int32_t L0 = uni(S.hdr[b][o].x);
    const int32_t L1 =
        uni(S.hdr[b][o + nw - 1].x + kSSlots * (S.hdr[b][o + nw - 1].y & 7));
    const unsigned n = static_cast<unsigned>(L1 - L0);
    SPTTN_DCHECK(n <= static_cast<unsigned>(kSWLeaves));
    fence_proxy_async();
    expect_tx_elect(&S.mbar_leaf[lb], n * 12u);
    bulk_g2s_elect(&S.kk[lb][0], a.pk + L0, n * 4u, &S.mbar_leaf[lb]);
    bulk_g2s_elect(&S.tv[lb][0], a.pv + L0, n * 8u, &S.mbar_leaf[lb]);
  };
  const int32_t nwin = (cend - cbeg + kSW - 1) / kSW;
  if (nwin > 0) {
    if (lane == 0) {
      for (int b = 0; b < 3; ++b) mbar_init(&S.mbar_meta[b], 1);
      for (int b = 0; b < 2; ++b) mbar_init(&S.mbar_leaf[b], 1);
      mbar_init_fence();
    }
    __syncwarp();
    issue_meta(0);
    if (nwin > 1) issue_meta(1);
    issue_leaves(0);
  }

  // 3. absent root rows (no nonzeros) of this half are zero
  for (int64_t e = static_cast<int64_t>(cta) * NT + tid; e < x.n_absent * (kHalf / 2);
       e += static_cast<int64_t>(x.n_cta) * NT) {
    const int32_t r = __ldg(x.absent_rows + e / (kHalf / 2));
    double* d = a.out + static_cast<int64_t>(r) * R + kHalf * h + 2 * static_cast<int>(e % (kHalf / 2));
    *reinterpret_cast<double2*>(d) = make_double2(0, 0);
  }

  // 4. the warp's groups
  int32_t cur = -1;
  bool first = true;
  double2 acc = make_double2(0, 0), fp = make_double2(0, 0);
  int32_t fslice = -1;
  auto reduce = [&]() {
    double2 v = acc;
    v.x += __shfl_xor_sync(0xffffffffu, v.x, 8);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, 8);
    v.x += __shfl_xor_sync(0xffffffffu, v.x, 16);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, 16);
    acc = make_double2(0, 0);
    return v;
  };
  auto flush = [&]() {  // slice `cur` done inside this warp's range
    const double2 v = reduce();
    if (first) {
      fp = v;
      fslice = cur;
      first = false;
    } else if (sp == 0) {
      double* d = a.out + static_cast<int64_t>(__ldg(a.t.idx[0] + cur)) * R + kHalf * h + 2 * cq;
      *reinterpret_cast<double2*>(d) = v;
    }
  };
  // B rows of the next group, gathered one group ahead
  double2 b0 = make_double2(0, 0), b1 = make_double2(0, 0);
  auto load_b = [&](int buf, int gi) {
    const int2 jj = *reinterpret_cast<const int2*>(&S.node[buf][gi * kSSlots + 2 * sp]);
    SPTTN_DCHECK(jj.x >= 0 && jj.x < a.frows[1] * a.R && jj.y >= 0 && jj.y < a.frows[1] * a.R);
    b0 = ld128(Bh + jj.x);
    b1 = ld128(Bh + jj.y);
  };

  cp_async_wait<0>();
  __syncthreads();  // C half resident

  if (nwin > 0) {
    mbar_wait(&S.mbar_meta[0], 0);
    load_b(0, 0);
  }
  for (int32_t win = 0; win < nwin; ++win) {
    const int mb = win % 3, lbf = win & 1;
    if (win + 1 < nwin) issue_leaves(win + 1);  // waits for meta(win + 1)
    if (win + 2 < nwin) issue_meta(win + 2);
    mbar_wait(&S.mbar_meta[mb], (win / 3) & 1);
    mbar_wait(&S.mbar_leaf[lbf], (win / 2) & 1);
    const int32_t g0 = cbeg + win * kSW;
    const int ng = min(g0 + kSW, cend) - g0;
    const int o = g0 & 1;
    const int32_t L0 = S.hdr[mb][o].x;
    for (int gi = 0; gi < ng; ++gi) {
      const int2 hh = S.hdr[mb][o + gi];
      const int32_t sl = hh.y >> 3;
      if (sl != cur) {  // warp-uniform
        if (cur >= 0) flush();
        cur = sl;
      }
      const double2 B0 = b0, B1 = b1;
      {
        const bool in_win = gi + 1 < ng;
        if (in_win || win + 1 < nwin) load_b(in_win ? mb : (win + 1) % 3, in_win ? gi + 1 : 0);
      }
      const int n = hh.y & 7;  // warp-uniform
      const int lb = hh.x - L0 + 2 * sp;
      double2 X0 = make_double2(0, 0), X1 = make_double2(0, 0);
      auto leaf = [&](int it) {
        SPTTN_DCHECK(lb + it * kSSlots + 1 < kSWLeaves);
        const int2 k2 = *reinterpret_cast<const int2*>(&S.kk[lbf][lb + it * kSSlots]);
        SPTTN_DCHECK(k2.x >= 0 && k2.x < x.rows_c * 128 && k2.y >= 0 && k2.y < x.rows_c * 128);
        const double2 t2 = *reinterpret_cast<const double2*>(&S.tv[lbf][lb + it * kSSlots]);
        const double2 c0 = lds128(cs + k2.x);
        const double2 c1 = lds128(cs + k2.y);
        X0.x = fma(t2.x, c0.x, X0.x);  // X += t * C[k]
        X0.y = fma(t2.x, c0.y, X0.y);
        X1.x = fma(t2.y, c1.x, X1.x);
        X1.y = fma(t2.y, c1.y, X1.y);
      };
      switch (n) {  // straight-line code per segment length
        case 1: leaf(0); break;
        case 2: leaf(0); leaf(1); break;
        case 3: leaf(0); leaf(1); leaf(2); break;
        default: leaf(0); leaf(1); leaf(2); leaf(3); break;
      }
      acc.x = fma(X0.x, B0.x, acc.x);  // A[i] += X * B[j]
      acc.y = fma(X0.y, B0.y, acc.y);
      acc.x = fma(X1.x, B1.x, acc.x);
      acc.y = fma(X1.y, B1.y, acc.y);
    }
    __syncwarp();  // this window's stage buffers are free
  }
  double2 lp = make_double2(0, 0);
  int32_t lslice = -1;
  if (cur >= 0) {
    const double2 v = reduce();
    if (first) {
      fp = v;
      fslice = cur;
    } else {
      lp = v;
      lslice = cur;
    }
  }

  // 5. first / last slice pieces of every warp, summed in warp order
  if (lane == 0 && nwin > 0) {  // stage memory (barriers included) is reused for the pieces
    for (int b = 0; b < 3; ++b) mbar_inval(&S.mbar_meta[b]);
    for (int b = 0; b < 2; ++b) mbar_inval(&S.mbar_leaf[b]);
  }
  __syncthreads();
  Piece* P = reinterpret_cast<Piece*>(stages);
  if (sp == 0) {
    P[2 * wid].v[2 * cq] = fp.x;
    P[2 * wid].v[2 * cq + 1] = fp.y;
    P[2 * wid + 1].v[2 * cq] = lp.x;
    P[2 * wid + 1].v[2 * cq + 1] = lp.y;
    if (cq == 0) {
      P[2 * wid].slice = fslice;
      P[2 * wid + 1].slice = lslice;
    }
  }
  __syncthreads();
  if (wid == 0 && lane < kHalf) {
    int32_t rs = -1;
    double run = 0.0;
    for (int p = 0; p < 2 * kSmfWarps; ++p) {
      const int32_t s = P[p].slice;
      if (s < 0) continue;
      const double v = P[p].v[lane];
      if (s != rs) {
        if (rs >= 0) a.out[static_cast<int64_t>(__ldg(a.t.idx[0] + rs)) * R + kHalf * h + lane] = run;
        rs = s;
        run = v;
      } else {
        run += v;
      }
    }
    if (rs >= 0) a.out[static_cast<int64_t>(__ldg(a.t.idx[0] + rs)) * R + kHalf * h + lane] = run;
  }
}

// plan time: header {leaf base, slice * 8 + length}; leaf coordinates -> byte
// offsets of their C rows in shared memory; fiber coordinates -> element
// offsets of their B rows
__global__ void k_smf_prep(const int4* hdr, int32_t ngroups, int2* hdr2, int32_t* gnode,
                           int32_t* pk, int64_t nleaves, int R) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e < ngroups) {
    const int4 hh = hdr[e];
    hdr2[e] = make_int2(hh.x, hh.w * 8 + hh.y);
  }
  if (e < static_cast<int64_t>(ngroups) * kSSlots) gnode[e] *= R;
  if (e < nleaves) pk[e] *= kHalf * 8;
}


// ---- MTTKRP-3 for the non-root output modes, shared-memory form ----------
//
// The other two CP-ALS products on the same (i,j,k) CSF (nest_mttkrp.cu
// k_mttkrp3_nonroot has the reference nests): mode j  B[j] += (sum_k t C[k])
// * A[i]; mode k  C[k] += (A[i] * B[j]) * t. The output row is not owned by
// a root slice, so contributions are accumulated — here into a per-CTA copy
// of the output's column quarter in shared memory (fp64 shared atomics),
// together with the gathered factor's column quarter (C for mode j, B for
// mode k), both rows * 64 bytes (64 KB each at the BASELINE shape). Each CTA
// then adds its accumulator into the zeroed global output with fp64 RED
// (rows_out * 8 per CTA instead of one global atomic per contribution:
// 2.4 M instead of 20-32 M). A[i] quarter rows come from L2 once per slice
// change. Summation order varies with atomic arrival (within tolerance).
__global__ void __launch_bounds__(kSmfWarps * 32, 1) k_mttkrp3_nr_smf(RootOutArgs a, SmfArgs x,
                                                                     int mode) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int NT = kSmfWarps * 32;
  const int tid = threadIdx.x;
  const int wid = uni(tid >> 5);
  const int lane = tid & 31;
  const int slot = lane >> 2;  // 8 slots, 4 lanes per 64-byte row
  const int cp = lane & 3;     // columns cp, cp+4 of the quarter (see add2)
  const int q = blockIdx.x % x.nq;
  const int cta = blockIdx.x / x.nq;
  const int R = a.R;
  const int col = 8 * q + cp;
  const unsigned sbase = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const unsigned cs = sbase + 8u * cp;
  const int32_t rows_in = x.rows_c, rows_out = x.rows_out;
  double* acc_sm = reinterpret_cast<double*>(smem + static_cast<int64_t>(rows_in) * 64);
  StageS* stages = reinterpret_cast<StageS*>(smem + static_cast<int64_t>(rows_in + rows_out) * 64);
  StageS& S = stages[wid];

  // 1. gathered factor quarter -> shared memory; accumulator quarter = 0
  {
    const double* F = a.f[1];  // C (mode j) or B (mode k)
    for (int32_t e = tid; e < rows_in * 4; e += NT) {
      const double* src = F + static_cast<int64_t>(e >> 2) * R + 8 * q + 2 * (e & 3);
      cp_async16_cg(smem + static_cast<int64_t>(e) * 16, src, 16);
    }
    cp_async_commit();
    for (int32_t e = tid; e < rows_out * 4; e += NT)
      reinterpret_cast<double2*>(acc_sm)[e] = make_double2(0, 0);
  }

  // 2. even group ranges (outputs are not slice-owned)
  const int64_t G = a.n_groups;
  const int32_t G0 = static_cast<int32_t>(G * cta / x.n_cta);
  const int32_t G1 = static_cast<int32_t>(G * (cta + 1) / x.n_cta);
  const int32_t cbeg =
      uni(G0 + static_cast<int32_t>((static_cast<int64_t>(G1 - G0) * wid) / kSmfWarps));
  const int32_t cend =
      uni(G0 + static_cast<int32_t>((static_cast<int64_t>(G1 - G0) * (wid + 1)) / kSmfWarps));

  auto issue_meta = [&](int32_t wi) {
    const int32_t g0 = cbeg + wi * kSW;
    const int32_t nw = min(g0 + kSW, cend) - g0;
    const int b = wi % 3;
    const unsigned hb = ((static_cast<unsigned>(nw + (g0 & 1)) * 8u) + 15u) & ~15u;
    const unsigned nb = nw * kSSlots * sizeof(int32_t);
    fence_proxy_async();
    expect_tx_elect(&S.mbar_meta[b], hb + nb);
    bulk_g2s_elect(&S.hdr[b][0], x.hdr2 + (g0 & ~1), hb, &S.mbar_meta[b]);
    bulk_g2s_elect(&S.node[b][0], a.grp_node + static_cast<int64_t>(g0) * kSSlots, nb,
                   &S.mbar_meta[b]);
  };
  auto issue_leaves = [&](int32_t wi) {
    const int32_t g0 = cbeg + wi * kSW;
    const int32_t nw = min(g0 + kSW, cend) - g0;
    const int b = wi % 3, lb = wi & 1;
    mbar_wait(&S.mbar_meta[b], (wi / 3) & 1);
    const int o = g0 & 1;
    const int32_t L0 = uni(S.hdr[b][o].x);
    const int32_t L1 =
        uni(S.hdr[b][o + nw - 1].x + kSSlots * (S.hdr[b][o + nw - 1].y & 7));
    const unsigned n = static_cast<unsigned>(L1 - L0);
    fence_proxy_async();
    expect_tx_elect(&S.mbar_leaf[lb], n * 12u);
    bulk_g2s_elect(&S.kk[lb][0], a.pk + L0, n * 4u, &S.mbar_leaf[lb]);
    bulk_g2s_elect(&S.tv[lb][0], a.pv + L0, n * 8u, &S.mbar_leaf[lb]);
  };
  const int32_t nwin = (cend - cbeg + kSW - 1) / kSW;
  if (nwin > 0) {
    if (lane == 0) {
      for (int b = 0; b < 3; ++b) mbar_init(&S.mbar_meta[b], 1);
      for (int b = 0; b < 2; ++b) mbar_init(&S.mbar_leaf[b], 1);
      mbar_init_fence();
    }
    __syncwarp();
    issue_meta(0);
    if (nwin > 1) issue_meta(1);
    issue_leaves(0);
  }
  cp_async_wait<0>();
  __syncthreads();  // factor quarter resident, accumulator zeroed

  const double* __restrict__ Aq = a.f[0] + col;
  int32_t cur = -1;
  double2 ar = make_double2(0, 0);
  // shared fp64 atomics (CAS loops) on columns cp and cp+4 of a 64-byte row:
  // the row's half picked first alternates with bit 1 of the row index, so
  // the 8 slots' rows of one instruction spread over 4 bank groups (2-way)
  // instead of 2 (4-way, with columns 2cp, 2cp+1)
  auto add2 = [&](unsigned off, double vx, double vy) {
    double* p = reinterpret_cast<double*>(smem + (off - sbase));
    const bool h = ((off - sbase) >> 7) & 1;  // (row >> 1) & 1
    atomicAdd(p + (h ? 4 : 0), h ? vy : vx);
    atomicAdd(p + (h ? 0 : 4), h ? vx : vy);
  };
  auto lds2 = [&](unsigned off) {  // columns cp, cp+4
    const double* p = reinterpret_cast<const double*>(smem + (off - sbase));
    return make_double2(p[0], p[4]);
  };
  for (int32_t win = 0; win < nwin; ++win) {
    const int mb = win % 3, lbf = win & 1;
    if (win + 1 < nwin) issue_leaves(win + 1);
    if (win + 2 < nwin) issue_meta(win + 2);
    mbar_wait(&S.mbar_meta[mb], (win / 3) & 1);
    mbar_wait(&S.mbar_leaf[lbf], (win / 2) & 1);
    const int32_t g0 = cbeg + win * kSW;
    const int ng = min(g0 + kSW, cend) - g0;
    const int o = g0 & 1;
    const int32_t L0 = S.hdr[mb][o].x;
    for (int gi = 0; gi < ng; ++gi) {
      const int2 hh = S.hdr[mb][o + gi];
      const int32_t sl = hh.y >> 3;
      if (sl != cur) {  // warp-uniform: A[i] once per root slice
        cur = sl;
        const double* arow = Aq + static_cast<int64_t>(__ldg(a.t.idx[0] + sl)) * R;
        ar = make_double2(__ldg(arow), __ldg(arow + 4));
      }
      const int n = hh.y & 7;  // warp-uniform
      const int lb = hh.x - L0 + slot;
      const unsigned nodeoff = static_cast<unsigned>(S.node[mb][gi * kSSlots + slot]);
      if (mode == 1) {  // B[j] += (sum_k t C[k]) * A[i]
        double2 X = make_double2(0, 0);
#pragma unroll
        for (int it = 0; it < 4; ++it) {
          if (it < n) {
            const unsigned kof = static_cast<unsigned>(S.kk[lbf][lb + it * kSSlots]);
            const double t = S.tv[lbf][lb + it * kSSlots];
            const double2 c = lds2(cs + kof);
            X.x = fma(t, c.x, X.x);
            X.y = fma(t, c.y, X.y);
          }
        }
        add2(cs + nodeoff, X.x * ar.x, X.y * ar.y);
      } else {  // C[k] += (A[i] * B[j]) * t
        const double2 b = lds2(cs + nodeoff);
        const double2 W = make_double2(ar.x * b.x, ar.y * b.y);
#pragma unroll
        for (int it = 0; it < 4; ++it) {
          if (it < n) {
            const unsigned kof = static_cast<unsigned>(S.kk[lbf][lb + it * kSSlots]);
            const double t = S.tv[lbf][lb + it * kSSlots];
            add2(cs + kof, W.x * t, W.y * t);
          }
        }
      }
    }
    __syncwarp();  // this window's stage buffers are free
  }

  // 3. accumulator quarter -> global output (fp64 RED, zero entries skipped)
  __syncthreads();
  for (int32_t e = tid; e < rows_out * 8; e += NT) {
    const double v = acc_sm[e];
    if (v != 0.0) atomicAdd(a.out + static_cast<int64_t>(e >> 3) * R + 8 * q + (e & 7), v);
  }
}

// plan time (non-root kernel): shared-memory byte offsets — the gathered
// factor's rows from 0, the accumulator's rows from rows_in * 64
__global__ void k_nr_prep(const int4* hdr, int32_t ngroups, int2* hdr2, int32_t* gnode,
                          int32_t* pk, int64_t nleaves, int node_base, int leaf_base) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e < ngroups) {
    const int4 hh = hdr[e];
    hdr2[e] = make_int2(hh.x, hh.w * 8 + hh.y);
  }
  if (e < static_cast<int64_t>(ngroups) * kSSlots) gnode[e] = node_base + gnode[e] * 64;
  if (e < nleaves) pk[e] = leaf_base + pk[e] * 64;
}

}  // namespace

size_t mttkrp3_smf_smem(int64_t rows_c) {
  return static_cast<size_t>(rows_c) * 128 + kSmfWarps * sizeof(StageS);
}

void mttkrp3_smf_prepare(Decomp& d, int R, cudaStream_t s) {
  dmalloc(&d.hdr2, (d.n_groups + 2) * sizeof(int2), s);
  SPTTN_CUDA(cudaMemsetAsync(d.hdr2, 0, (d.n_groups + 2) * sizeof(int2), s));
  const int64_t n = std::max<int64_t>(d.n_groups * kSSlots, d.n_packed_leaves);
  if (n > 0) {
    k_smf_prep<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(
        d.grp_hdr, static_cast<int32_t>(d.n_groups), d.hdr2, d.grp_node, d.pk, d.n_packed_leaves, R);
    SPTTN_CUDA(cudaGetLastError());
  }
}

void launch_mttkrp3_smf(const RootOutArgs& a, const SmfArgs& x, cudaStream_t s) {
  const unsigned blocks = static_cast<unsigned>(x.nq * x.n_cta);
  if (blocks == 0) return;
  const size_t sm = mttkrp3_smf_smem(x.rows_c);
  SPTTN_CUDA(cudaFuncSetAttribute(k_mttkrp3_smf, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(sm)));
  k_mttkrp3_smf<<<blocks, kSmfWarps * 32, sm, s>>>(a, x);
  SPTTN_CUDA(cudaGetLastError());
}

}  // namespace spttn_dev

namespace spttn_dev {

size_t mttkrp3_nr_smem(int64_t rows_in, int64_t rows_out) {
  return static_cast<size_t>(rows_in + rows_out) * 64 + kSmfWarps * sizeof(StageS);
}

void mttkrp3_nr_prepare(Decomp& d, int mode, int64_t rows_in, cudaStream_t s) {
  dmalloc(&d.hdr2, (d.n_groups + 2) * sizeof(int2), s);
  SPTTN_CUDA(cudaMemsetAsync(d.hdr2, 0, (d.n_groups + 2) * sizeof(int2), s));
  const int64_t n = std::max<int64_t>(d.n_groups * kSSlots, d.n_packed_leaves);
  const int acc0 = static_cast<int>(rows_in * 64);
  if (n > 0) {
    k_nr_prep<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(
        d.grp_hdr, static_cast<int32_t>(d.n_groups), d.hdr2, d.grp_node, d.pk, d.n_packed_leaves,
        mode == 1 ? acc0 : 0, mode == 1 ? 0 : acc0);
    SPTTN_CUDA(cudaGetLastError());
  }
}

void launch_mttkrp3_nr_smf(const RootOutArgs& a, const SmfArgs& x, int mode, cudaStream_t s) {
  const unsigned blocks = static_cast<unsigned>(x.nq * x.n_cta);
  if (blocks == 0 || a.n_groups == 0) return;
  const size_t sm = mttkrp3_nr_smem(x.rows_c, x.rows_out);
  SPTTN_CUDA(cudaFuncSetAttribute(k_mttkrp3_nr_smf, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(sm)));
  k_mttkrp3_nr_smf<<<blocks, kSmfWarps * 32, sm, s>>>(a, x, mode);
  SPTTN_CUDA(cudaGetLastError());
}

}  // namespace spttn_dev
