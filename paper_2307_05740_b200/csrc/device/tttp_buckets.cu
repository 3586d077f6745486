// Plan-time construction of the C-bucketed TTTP leaf layout (nest_tttp.cu
// k_tttp3_kb): leaves keyed by (i range, k bucket), stable radix sort (CSF
// order kept inside a key), every key's run padded to a multiple of 4
// leaves. The bucketed kernel lives here too: in nest_tttp.cu's translation unit
// it changed the leaf kernel's code generation (60 -> 48 registers, 3.5 ->
// 4.0 ms).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "internal.cuh"
#include "tttp_reduce.cuh"

namespace spttn_dev {

namespace {

#ifndef KB_THREADS
#define KB_THREADS 640  // 96 registers, no spills (768: spills, 512: too few warps)
#endif
constexpr int kKbThreads = KB_THREADS;

// ---- C-bucketed form (default when the buckets balance) ------------------
//
// The leaf kernel above is bound by L2 -> SM delivery of the per-leaf B[j]
// and C[k] rows (52.7 GB per launch at the BASELINE shape, ~15 TB/s). Leaves
// are independent, so they may be processed in any order: the plan groups
// them by k-bucket (kb consecutive C rows, stable, so CSF order — i, then j —
// is kept inside a bucket) and every CTA keeps its bucket's C rows in shared
// memory (loaded once, cp.async). Per leaf only B[j] still comes from L2;
// A[i] is re-read only when i changes (a bucket holds dims_i-ordered leaves,
// ~7 per i at the BASELINE shape). L2 -> SM bytes per leaf: 1024 -> ~590.
// Groups of G lanes walk contiguous, 4-aligned leaf ranges of the bucket
// (the plan pads every bucket to a multiple of 4; padding leaves carry
// position -1), loading each field of 4 leaves with one broadcast vector load.
template <int G, int U, bool VEC>
__global__ void __launch_bounds__(kKbThreads, 1) k_tttp3_kb(RootOutArgs a, TttpKbArgs x) {
  extern __shared__ __align__(128) unsigned char smem[];
  static_assert(U == 4, "vector leaf loads assume 4 leaves per step");
  const double* Cs = reinterpret_cast<const double*>(smem);
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int lg = lane & (G - 1);
  const int c = lg * 4;
  const int R = a.R;
  const int b = blockIdx.x / x.ppb, part = blockIdx.x % x.ppb;  // b = (i range, k bucket)
  const int32_t k0 = (b % x.nb) * x.kb;
  const int32_t rows = max(0, min(x.kb, x.rows_c - k0));
  {  // the bucket's C rows (contiguous in global) -> shared memory. The two
     // 16-byte halves of every odd 32-byte chunk quad are swapped so that the
     // 8 lanes of an LDS.128 phase (32-byte column chunks 8p..8p+7) hit 8
     // distinct bank groups: unswizzled, chunks c and c+4 collide (2-way)
    const double* src = a.f[2] + static_cast<int64_t>(k0) * R;
    const int32_t n16 = rows * R / 2;
    for (int32_t e = tid; e < n16; e += blockDim.x) {
      const int32_t ch = (e >> 1) % (R / 4);  // 32-byte chunk within the row
      const int32_t d = e ^ ((ch >> 2) & 1);
      cp_async16_cg(smem + static_cast<int64_t>(d) * 16, src + 2 * e, 16);
    }
    cp_async_commit();
  }
  const int sw = (lg >> 2) & 1;  // this lane's chunk has swapped halves
  // this group's 4-aligned leaf range
  const int64_t s0 = __ldg(x.bstart + b), s1 = __ldg(x.bstart + b + 1);
  const int64_t q0 = (s1 - s0) / 4;  // quads in the bucket
  const int64_t p0 = s0 + 4 * (q0 * part / x.ppb), p1 = s0 + 4 * (q0 * (part + 1) / x.ppb);
  const int ngroups = blockDim.x / G;
  const int gid = tid / G;
  const int64_t nq = (p1 - p0) / 4;
  const int64_t e0 = p0 + 4 * (nq * gid / ngroups), e1 = p0 + 4 * (nq * (gid + 1) / ngroups);
  const double* __restrict__ A = a.f[0];
  const double* __restrict__ B = a.f[1];
  const bool residual = (a.flags & 1) != 0;
  cp_async_wait<0>();
  __syncthreads();

  int32_t prev_i = -1;
  double4 prev_a = make_double4(0, 0, 0, 0);
  for (int64_t e = e0; e < e1; e += U) {
    const int4 ii = __ldg(reinterpret_cast<const int4*>(x.li + e));
    const int4 jj = __ldg(reinterpret_cast<const int4*>(x.lj + e));
    const int4 kk = __ldg(reinterpret_cast<const int4*>(x.lk + e));
    const int4 pp = __ldg(reinterpret_cast<const int4*>(x.lp + e));
    const double4 tv = ld256(x.lv + e);
    const int32_t iv[4] = {ii.x, ii.y, ii.z, ii.w};
    const int32_t jv[4] = {jj.x, jj.y, jj.z, jj.w};
    const int32_t kv[4] = {kk.x, kk.y, kk.z, kk.w};
    double part_[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      // A[i] only when i changes (predicated-off loads move no data)
      const int32_t pi = u == 0 ? prev_i : iv[u - 1];
      const bool fresh = iv[u] != pi;
      double4 ld;
      if (VEC) {
        ld = ld256_if(A + static_cast<int64_t>(iv[u]) * R + c, fresh && c < R);
      } else {
        ld = fresh ? row4<false>(A + static_cast<int64_t>(iv[u]) * R, c, R) : prev_a;
      }
      const double4 ar = fresh ? ld : prev_a;
      prev_a = ar;
      const double4 br = row4<VEC>(B + static_cast<int64_t>(jv[u]) * R, c, R);
      double4 cr = make_double4(0, 0, 0, 0);
      if (c < R) {
        const double* crow = Cs + static_cast<int64_t>(kv[u]) * R + c;
        const double2 c01 = *reinterpret_cast<const double2*>(crow + 2 * sw);
        const double2 c23 = *reinterpret_cast<const double2*>(crow + 2 - 2 * sw);
        cr = make_double4(c01.x, c01.y, c23.x, c23.y);
      }
      double y = (ar.x * br.x) * cr.x;  // X[r] = A[i,r]*B[j,r]; Y += X[r]*C[k,r]
      y = fma(ar.y * br.y, cr.y, y);
      y = fma(ar.z * br.z, cr.z, y);
      y = fma(ar.w * br.w, cr.w, y);
      part_[u] = y;
    }
    prev_i = iv[U - 1];
    int q = 0;
    const double y = transpose_reduce<G, U>(part_, lg, &q);
    if ((lg & (G / U - 1)) == 0) {
      const int32_t pos = q == 0 ? pp.x : q == 1 ? pp.y : q == 2 ? pp.z : pp.w;
      const double t = q == 0 ? tv.x : q == 1 ? tv.y : q == 2 ? tv.z : tv.w;
      if (pos >= 0) a.out[pos] = residual ? t - y : 0.0 + y * t;  // executor.cpp:402
    }
  }
}



// plan-time helpers for the bucketed layout
__global__ void k_kb_keys(const int32_t* kidx, const int32_t* leaf_i, int64_t nnz, int kb, int nb,
                          int ir, uint32_t* keys, int32_t* ids, int32_t* counts) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= nnz) return;
  const uint32_t b = static_cast<uint32_t>((leaf_i[p] / ir) * nb + kidx[p] / kb);
  keys[p] = b;
  ids[p] = static_cast<int32_t>(p);
  atomicAdd(counts + b, 1);
}

__global__ void k_kb_fill(const uint32_t* skeys, const int32_t* perm, int64_t nnz, int kb,
                          const int64_t* ustart, const int64_t* pstart, const int32_t* leaf_i,
                          const int32_t* leaf_j, const int32_t* kidx, const double* vals,
                          int32_t* li, int32_t* lj, int32_t* lk, int32_t* lp, double* lv) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= nnz) return;
  const uint32_t b = skeys[e];
  const int64_t d = pstart[b] + (e - ustart[b]);
  const int32_t p = perm[e];
  li[d] = leaf_i[p];
  lj[d] = leaf_j[p];
  lk[d] = kidx[p] % kb;
  lp[d] = p;
  lv[d] = vals[p];
}

}  // namespace

bool build_tttp_buckets(const DevCsf& csf, int R, int sms, const int32_t* leaf_i,
                        const int32_t* leaf_j, TttpKb& kbl, cudaStream_t s) {
  csf.wait_values(s);
  const int64_t nnz = csf.level_size[2];
  const int64_t rows_c = csf.dims[2];
  const int G = group_lanes_for(R);
  if (nnz == 0 || R % 4 != 0 || G < 4 || nnz >= (int64_t{1} << 31)) return false;
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const int64_t budget = std::min<int64_t>(200 * 1024, optin - 1024);
  const int64_t row_bytes = static_cast<int64_t>(R) * 8;
  const int64_t nb_min = std::max<int64_t>(1, (rows_c * row_bytes + budget - 1) / budget);
  if (nb_min > sms) return false;
  const int ppb = std::max<int>(1, static_cast<int>(sms / nb_min));
  const int nb = std::max<int>(static_cast<int>(nb_min), sms / ppb);
  const int kb = static_cast<int>((rows_c + nb - 1) / nb);
  if (kb * row_bytes > budget) return false;
  // i ranges: the scattered rho writes of the CTAs running together stay in
  // a ~24 MB output window (merged in L2 instead of partial-sector
  // read-modify-writes in HBM)
  const int64_t dims_i = csf.dims[0];
  const int64_t n_i = std::clamp<int64_t>((nnz * 8 + (24 << 20) - 1) / (24 << 20), 1,
                                          std::max<int64_t>(1, 65536 / nb));
  const int ir = static_cast<int>((dims_i + n_i - 1) / n_i);
  const int nkey = static_cast<int>(((dims_i + ir - 1) / ir) * nb);
  uint32_t *keys = nullptr, *skeys = nullptr;
  int32_t *ids = nullptr, *perm = nullptr, *counts = nullptr;
  dmalloc(&keys, nnz * sizeof(uint32_t), s);
  dmalloc(&skeys, nnz * sizeof(uint32_t), s);
  dmalloc(&ids, nnz * sizeof(int32_t), s);
  dmalloc(&perm, nnz * sizeof(int32_t), s);
  dmalloc(&counts, nkey * sizeof(int32_t), s);
  SPTTN_CUDA(cudaMemsetAsync(counts, 0, nkey * sizeof(int32_t), s));
  const unsigned nbk = static_cast<unsigned>((nnz + 255) / 256);
  k_kb_keys<<<nbk, 256, 0, s>>>(csf.idx[2], leaf_i, nnz, kb, nb, ir, keys, ids, counts);
  int bits = 1;
  while ((1 << bits) < nkey) ++bits;
  size_t tb = 0;
  void* tmp = nullptr;
  SPTTN_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, skeys, ids, perm, nnz, 0, bits, s));
  dmalloc(&tmp, tb, s);
  SPTTN_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, keys, skeys, ids, perm, nnz, 0, bits, s));
  dfree(tmp, s);
  std::vector<int32_t> cnt(nkey);
  SPTTN_CUDA(cudaMemcpyAsync(cnt.data(), counts, nkey * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  SPTTN_CUDA(cudaStreamSynchronize(s));
  int64_t widest = 0;
  std::vector<int64_t> us(nkey + 1, 0), ps(nkey + 1, 0);
  for (int b = 0; b < nkey; ++b) {
    us[b + 1] = us[b] + cnt[b];
    ps[b + 1] = ps[b] + (cnt[b] + 3) / 4 * 4;
    widest = std::max<int64_t>(widest, cnt[b]);
  }
  const bool ok = std::getenv("SPTTN_TTTP_KB_FORCE") != nullptr ||
                  widest * nkey <= nnz + nnz / 2 + 4096 * nkey;  // balanced buckets only
  if (ok) {
    const int64_t np = std::max<int64_t>(4, ps[nkey]);
    kbl.nkey = nkey;
    kbl.nb = nb;
    kbl.ppb = ppb;
    kbl.kb = kb;
    kbl.rows_c = static_cast<int32_t>(rows_c);
    int64_t* d_us = nullptr;
    dmalloc(&kbl.bstart, (nkey + 1) * sizeof(int64_t), s);
    dmalloc(&d_us, (nkey + 1) * sizeof(int64_t), s);
    dmalloc(&kbl.li, np * 4, s);
    dmalloc(&kbl.lj, np * 4, s);
    dmalloc(&kbl.lk, np * 4, s);
    dmalloc(&kbl.lp, np * 4, s);
    dmalloc(&kbl.lv, np * 8, s);
    SPTTN_CUDA(cudaMemsetAsync(kbl.li, 0, np * 4, s));
    SPTTN_CUDA(cudaMemsetAsync(kbl.lj, 0, np * 4, s));
    SPTTN_CUDA(cudaMemsetAsync(kbl.lk, 0, np * 4, s));
    SPTTN_CUDA(cudaMemsetAsync(kbl.lp, 0xff, np * 4, s));  // padding: position -1
    SPTTN_CUDA(cudaMemsetAsync(kbl.lv, 0, np * 8, s));
    SPTTN_CUDA(cudaMemcpyAsync(kbl.bstart, ps.data(), (nkey + 1) * sizeof(int64_t),
                               cudaMemcpyHostToDevice, s));
    SPTTN_CUDA(cudaMemcpyAsync(d_us, us.data(), (nkey + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    k_kb_fill<<<nbk, 256, 0, s>>>(skeys, perm, nnz, kb, d_us, kbl.bstart, leaf_i, leaf_j, csf.idx[2],
                                  csf.vals, kbl.li, kbl.lj, kbl.lk, kbl.lp, kbl.lv);
    SPTTN_CUDA(cudaGetLastError());
    SPTTN_CUDA(cudaStreamSynchronize(s));
    dfree(d_us, s);
  }
  for (void* p : {static_cast<void*>(keys), static_cast<void*>(skeys), static_cast<void*>(ids),
                  static_cast<void*>(perm), static_cast<void*>(counts)})
    dfree(p, s);
  SPTTN_CUDA(cudaStreamSynchronize(s));
  return ok;
}

void free_tttp_buckets(TttpKb& kbl) {
  for (void* p : {static_cast<void*>(kbl.bstart), static_cast<void*>(kbl.li),
                  static_cast<void*>(kbl.lj), static_cast<void*>(kbl.lk),
                  static_cast<void*>(kbl.lp), static_cast<void*>(kbl.lv)})
    dfree(p);
  kbl = TttpKb{};
}

void launch_tttp3_kb(const RootOutArgs& a, const TttpKb& kbl, cudaStream_t s) {
  if (kbl.nkey == 0) return;
  TttpKbArgs x{kbl.bstart, kbl.nb, kbl.ppb, kbl.kb, kbl.rows_c, kbl.li, kbl.lj, kbl.lk, kbl.lp, kbl.lv};
  const size_t sm = static_cast<size_t>(kbl.kb) * a.R * 8;
  const unsigned grid = static_cast<unsigned>(kbl.nkey * kbl.ppb);
  auto go = [&](auto kern) {
    SPTTN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(sm)));
    kern<<<grid, kKbThreads, sm, s>>>(a, x);
  };
  switch (group_lanes_for(a.R)) {
    case 4: a.vec ? go(k_tttp3_kb<4, 4, true>) : go(k_tttp3_kb<4, 4, false>); break;
    case 8: a.vec ? go(k_tttp3_kb<8, 4, true>) : go(k_tttp3_kb<8, 4, false>); break;
    case 16: a.vec ? go(k_tttp3_kb<16, 4, true>) : go(k_tttp3_kb<16, 4, false>); break;
    default: a.vec ? go(k_tttp3_kb<32, 4, true>) : go(k_tttp3_kb<32, 4, false>); break;
  }
  SPTTN_CUDA(cudaGetLastError());
}

}  // namespace spttn_dev
