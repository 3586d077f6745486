// Packed (length-sorted) segment layout — built once per plan.
//
// B200's L1 serves a warp-wide gather instruction at a cost set by the
// instruction, not by how many of its lanes are active (tools/gather_probe.cu:
// 1, 2, 4 or 8 rows per 256-bit instruction cost about the same), so a gather
// must carry a full set of rows. Segments (fiber pieces of <= 4 leaves) of
// one root slice are therefore regrouped by length: a *group* is `slots`
// segments of the same slice and the same length n (8 for 128-byte factor
// rows, 4 for 256-byte rows), with their leaves interleaved (leaf `it` of slot
// `s` at base + slots*it + s), so the it-th gather of a group fetches a full
// set of rows with no predicated-off lanes and the trip count n is
// warp-uniform. Summing a slice's segments in this fixed (sorted) order keeps
// results deterministic.
#include <cub/cub.cuh>

#include "internal.cuh"

namespace spttn_dev {

namespace {

unsigned nblk(int64_t n, int b) { return static_cast<unsigned>((n + b - 1) / b); }

__global__ void k_seg_keys(const int32_t* seg_begin, const int32_t* slice_seg, int32_t n0,
                           int32_t nseg, uint64_t* keys, int32_t* ids) {
  const int32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nseg) return;
  // slice of segment s: largest p with slice_seg[p] <= s
  int32_t lo = 0, hi = n0;
  while (hi - lo > 1) {
    const int32_t mid = (lo + hi) >> 1;
    if (slice_seg[mid] <= s) lo = mid; else hi = mid;
  }
  const int32_t len = seg_begin[s + 1] - seg_begin[s];
  keys[s] = (static_cast<uint64_t>(lo) << 3) | static_cast<uint64_t>(len & 7);
  ids[s] = s;
}

// run start of each sorted position (for equal keys): head flags -> max scan
__global__ void k_run_heads(const uint64_t* keys, int32_t n, int32_t* head) {
  const int32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  head[p] = (p == 0 || keys[p] != keys[p - 1]) ? p : 0;
}

// one past the last sorted position of each run, stored at the run's start
__global__ void k_run_ends(const uint64_t* keys, const int32_t* runstart, int32_t n,
                           int32_t* end_at_start) {
  const int32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  if (p == n - 1 || keys[p] != keys[p + 1]) end_at_start[runstart[p]] = p + 1;
}

__global__ void k_run_end_of(const int32_t* runstart, const int32_t* end_at_start, int32_t n,
                             int32_t* runend) {
  const int32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  runend[p] = end_at_start[runstart[p]];
}

__global__ void k_group_flags(const int32_t* runstart, int32_t n, int slots, int32_t* flag) {
  const int32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  flag[p] = ((p - runstart[p]) % slots) == 0 ? 1 : 0;
}

// per group: len, slice, nseg; gleaves = slots * len for the leaf-base scan
__global__ void k_group_headers(const uint64_t* keys, const int32_t* runstart, const int32_t* gid,
                                const int32_t* runend, int32_t n, int slots, int4* hdr,
                                int32_t* gleaves) {
  const int32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  if ((p - runstart[p]) % slots != 0) return;
  const int32_t g = gid[p] - 1;
  const int32_t len = static_cast<int32_t>(keys[p] & 7);
  const int32_t slice = static_cast<int32_t>(keys[p] >> 3);
  const int32_t nseg = min(slots, runend[p] - p);
  hdr[g] = make_int4(0, len, nseg, slice);
  gleaves[g] = slots * len;
}

__global__ void k_fill_groups(const int32_t* ids, const int32_t* runstart, const int32_t* gid,
                              const int32_t* leaf_off, const int32_t* seg_begin,
                              const int32_t* seg_node, const int32_t* seg_node1,
                              const int32_t* kidx, const int32_t* kidx2, const double* vals,
                              int32_t n, int slots, bool pair_perm, int4* hdr, int32_t* gnode,
                              int32_t* gnode1, int32_t* pk, int32_t* pk2, double* pv) {
  const int32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int32_t g = gid[p] - 1;
  const int32_t slot0 = (p - runstart[p]) % slots;
  // storage position of the slot (pair_perm: slots a and a + slots/2 adjacent)
  const int32_t slot = pair_perm ? 2 * (slot0 % (slots / 2)) + slot0 / (slots / 2) : slot0;
  const int32_t s = ids[p];
  const int32_t base = leaf_off[g];
  if (slot0 == 0) hdr[g].x = base;
  gnode[static_cast<int64_t>(g) * slots + slot] = seg_node[s];
  if (gnode1) gnode1[static_cast<int64_t>(g) * slots + slot] = seg_node1[s];
  const int32_t b = seg_begin[s], len = seg_begin[s + 1] - b;
  for (int32_t it = 0; it < len; ++it) {
    const int64_t e = base + it * slots + slot;
    pk[e] = kidx[b + it];
    if (pk2) pk2[e] = kidx2[b + it];
    pv[e] = vals[b + it];
  }
}

__global__ void k_slice_groups(const int4* hdr, int32_t ngroups, int32_t n0, int32_t* slice_grp) {
  const int32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g > ngroups) return;
  if (g == ngroups) {
    slice_grp[n0] = ngroups;
    return;
  }
  const int32_t sl = hdr[g].w;
  if (g == 0 || hdr[g - 1].w != sl) slice_grp[sl] = g;
}

template <class Op>
void scan_incl(int32_t* in, int32_t* out, int32_t n, Op op, cudaStream_t s) {
  size_t bytes = 0;
  void* tmp = nullptr;
  SPTTN_CUDA(cub::DeviceScan::InclusiveScan(nullptr, bytes, in, out, op, n, s));
  dmalloc(&tmp, bytes, s);
  SPTTN_CUDA(cub::DeviceScan::InclusiveScan(tmp, bytes, in, out, op, n, s));
  dfree(tmp, s);
}

void scan_excl_sum(int32_t* in, int32_t* out, int32_t n, cudaStream_t s) {
  size_t bytes = 0;
  void* tmp = nullptr;
  SPTTN_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, s));
  dmalloc(&tmp, bytes, s);
  SPTTN_CUDA(cub::DeviceScan::ExclusiveSum(tmp, bytes, in, out, n, s));
  dfree(tmp, s);
}

struct MaxOp {
  __device__ __forceinline__ int32_t operator()(int32_t a, int32_t b) const { return a > b ? a : b; }
};

}  // namespace

void build_packed(const DevCsf& csf, int leaf_level, Decomp& d, cudaStream_t s, int slots,
                  const int32_t* leaf_coord2, cudaEvent_t* fill_done, bool pair_perm) {
  plan_trace("pack: enter", s);
  const int32_t nseg = static_cast<int32_t>(d.n_seg);
  const int32_t n0 = static_cast<int32_t>(csf.level_size[0]);
  d.pack_slots = slots;
  if (nseg == 0) {
    d.n_groups = 0;
    dmalloc(&d.slice_grp, (static_cast<int64_t>(n0) + 1) * sizeof(int32_t), s);
    SPTTN_CUDA(cudaMemsetAsync(d.slice_grp, 0, (static_cast<int64_t>(n0) + 1) * sizeof(int32_t), s));
    return;
  }
  uint64_t *keys = nullptr, *keys2 = nullptr;
  int32_t *ids = nullptr, *ids2 = nullptr, *head = nullptr, *runstart = nullptr,
          *end_at_start = nullptr, *runend = nullptr, *flag = nullptr, *gid = nullptr;
  dmalloc(&keys, nseg * sizeof(uint64_t), s);
  dmalloc(&keys2, nseg * sizeof(uint64_t), s);
  dmalloc(&ids, nseg * sizeof(int32_t), s);
  dmalloc(&ids2, nseg * sizeof(int32_t), s);
  k_seg_keys<<<nblk(nseg, 256), 256, 0, s>>>(d.seg_begin, d.slice_seg, n0, nseg, keys, ids);
  SPTTN_CUDA(cudaGetLastError());
  int key_bits = 3;
  while (key_bits < 64 && (uint64_t{1} << (key_bits - 3)) <= static_cast<uint64_t>(n0)) ++key_bits;
  size_t bytes = 0;
  SPTTN_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys, keys2, ids, ids2, nseg, 0,
                                             key_bits, s));
  void* tmp = nullptr;
  dmalloc(&tmp, bytes, s);
  SPTTN_CUDA(cub::DeviceRadixSort::SortPairs(tmp, bytes, keys, keys2, ids, ids2, nseg, 0, key_bits,
                                             s));
  dfree(tmp, s);
  dmalloc(&head, nseg * sizeof(int32_t), s);
  dmalloc(&runstart, nseg * sizeof(int32_t), s);
  dmalloc(&end_at_start, nseg * sizeof(int32_t), s);
  dmalloc(&runend, nseg * sizeof(int32_t), s);
  dmalloc(&flag, nseg * sizeof(int32_t), s);
  dmalloc(&gid, nseg * sizeof(int32_t), s);
  k_run_heads<<<nblk(nseg, 256), 256, 0, s>>>(keys2, nseg, head);
  scan_incl(head, runstart, nseg, MaxOp{}, s);
  k_run_ends<<<nblk(nseg, 256), 256, 0, s>>>(keys2, runstart, nseg, end_at_start);
  k_run_end_of<<<nblk(nseg, 256), 256, 0, s>>>(runstart, end_at_start, nseg, runend);
  k_group_flags<<<nblk(nseg, 256), 256, 0, s>>>(runstart, nseg, slots, flag);
  scan_incl(flag, gid, nseg, cub::Sum{}, s);
  int32_t ngroups = 0;
  plan_trace("pack: sort + group ids", s);
  SPTTN_CUDA(cudaMemcpyAsync(&ngroups, gid + nseg - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  SPTTN_CUDA(cudaStreamSynchronize(s));
  d.n_groups = ngroups;
  int32_t* gleaves = nullptr;
  int32_t* leaf_off = nullptr;
  dmalloc(&d.grp_hdr, static_cast<int64_t>(ngroups) * sizeof(int4), s);
  dmalloc(&gleaves, (static_cast<int64_t>(ngroups) + 1) * sizeof(int32_t), s);
  dmalloc(&leaf_off, (static_cast<int64_t>(ngroups) + 1) * sizeof(int32_t), s);
  SPTTN_CUDA(cudaMemsetAsync(gleaves, 0, (static_cast<int64_t>(ngroups) + 1) * sizeof(int32_t), s));
  k_group_headers<<<nblk(nseg, 256), 256, 0, s>>>(keys2, runstart, gid, runend, nseg, slots,
                                                  d.grp_hdr, gleaves);
  scan_excl_sum(gleaves, leaf_off, ngroups + 1, s);
  int32_t nleaves = 0;
  SPTTN_CUDA(cudaMemcpyAsync(&nleaves, leaf_off + ngroups, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  SPTTN_CUDA(cudaStreamSynchronize(s));
  d.n_packed_leaves = nleaves;
  const int64_t nslots = static_cast<int64_t>(ngroups) * slots;
  dmalloc(&d.grp_node, nslots * sizeof(int32_t), s);
  SPTTN_CUDA(cudaMemsetAsync(d.grp_node, 0, nslots * sizeof(int32_t), s));
  if (d.seg_node1) {
    dmalloc(&d.grp_node1, nslots * sizeof(int32_t), s);
    SPTTN_CUDA(cudaMemsetAsync(d.grp_node1, 0, nslots * sizeof(int32_t), s));
  }
  // separate coordinate / value streams measured faster than 16-byte
  // {coord, coord2, value} records for TTMc-4 (750 vs 810 us)
  const int64_t nl = std::max<int64_t>(1, nleaves);
  dmalloc(&d.pk, nl * sizeof(int32_t), s);
  dmalloc(&d.pv, nl * sizeof(double), s);
  SPTTN_CUDA(cudaMemsetAsync(d.pk, 0, nl * sizeof(int32_t), s));
  SPTTN_CUDA(cudaMemsetAsync(d.pv, 0, nl * sizeof(double), s));
  if (leaf_coord2) {
    dmalloc(&d.pk2, nl * sizeof(int32_t), s);
    SPTTN_CUDA(cudaMemsetAsync(d.pk2, 0, nl * sizeof(int32_t), s));
  }
  const CsfView t = csf.view();
  // the fill needs the leaf values: on a side stream when the caller lets
  // the rest of the plan run meanwhile (values may still be on the link)
  cudaStream_t fs = s;
  if (fill_done) {
    fs = aux_stream();
    cudaEvent_t ready = nullptr;
    SPTTN_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    SPTTN_CUDA(cudaEventRecord(ready, s));
    SPTTN_CUDA(cudaStreamWaitEvent(fs, ready, 0));
    SPTTN_CUDA(cudaEventDestroy(ready));
  }
  csf.wait_values(fs);  // the structure work above overlaps an async values upload
  k_fill_groups<<<nblk(nseg, 256), 256, 0, fs>>>(ids2, runstart, gid, leaf_off, d.seg_begin,
                                                 d.seg_node, d.seg_node1, t.idx[leaf_level],
                                                 leaf_coord2, t.vals, nseg, slots, pair_perm,
                                                 d.grp_hdr,
                                                 d.grp_node, d.grp_node1, d.pk, d.pk2, d.pv);
  dmalloc(&d.slice_grp, (static_cast<int64_t>(n0) + 1) * sizeof(int32_t), s);
  k_slice_groups<<<nblk(static_cast<int64_t>(ngroups) + 1, 256), 256, 0, s>>>(d.grp_hdr, ngroups,
                                                                            n0, d.slice_grp);
  SPTTN_CUDA(cudaGetLastError());
  for (void* p : {static_cast<void*>(keys), static_cast<void*>(keys2), static_cast<void*>(ids),
                  static_cast<void*>(head), static_cast<void*>(end_at_start),
                  static_cast<void*>(runend), static_cast<void*>(flag),
                  static_cast<void*>(gleaves)})
    dfree(p, s);
  // the fill's inputs are released in its own stream order
  for (void* p : {static_cast<void*>(ids2), static_cast<void*>(runstart), static_cast<void*>(gid),
                  static_cast<void*>(leaf_off)})
    dfree(p, fs);
  if (fill_done) {
    SPTTN_CUDA(cudaEventCreateWithFlags(fill_done, cudaEventDisableTiming));
    SPTTN_CUDA(cudaEventRecord(*fill_done, fs));
  } else {
    SPTTN_CUDA(cudaStreamSynchronize(s));
  }
}

}  // namespace spttn_dev
