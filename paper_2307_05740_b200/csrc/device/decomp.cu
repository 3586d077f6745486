// Plan-time work decomposition (built once per plan on the device) and the
// deterministic fix-up epilogue for root slices split across work items.
#include <cub/cub.cuh>

#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "internal.cuh"

namespace spttn_dev {

namespace {

// Largest node n in [0, count) with ptr[n] <= key (ptr ascending).
__device__ __forceinline__ int32_t parent_of(const int32_t* ptr, int32_t count, int32_t key) {
  int32_t lo = 0, hi = count;  // invariant: ptr[lo] <= key, answer in [lo, hi)
  while (hi - lo > 1) {
    const int32_t mid = (lo + hi) >> 1;
    if (ptr[mid] <= key) lo = mid; else hi = mid;
  }
  return lo;
}

__global__ void k_leaf_items(CsfView t, int64_t chunk, int64_t n_items, int32_t* item_pos) {
  const int64_t it = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (it >= n_items) return;
  const int d = t.order;
  int32_t pos = static_cast<int32_t>(it * chunk);
  item_pos[it * d + d - 1] = pos;
  for (int l = d - 2; l >= 0; --l) {
    pos = parent_of(t.ptr[l], t.nlev[l], pos);
    item_pos[it * d + l] = pos;
  }
}

// Root slices whose leaves span more than one item.
__global__ void k_leaf_splits(CsfView t, int64_t chunk, int32_t* node, int32_t* first,
                              int32_t* last, int32_t* count, unsigned char* present) {
  const int32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= t.nlev[0]) return;
  int32_t a = s, b = s + 1;
  for (int l = 0; l + 1 < t.order; ++l) {
    a = t.ptr[l][a];
    b = t.ptr[l][b];
  }
  const int64_t f = a / chunk, g = (static_cast<int64_t>(b) - 1) / chunk;
  if (f != g) {
    const int32_t slot = atomicAdd(count, 1);
    node[slot] = s;
    first[slot] = static_cast<int32_t>(f);
    last[slot] = static_cast<int32_t>(g);
  }
  present[t.idx[0][s]] = 1;
}

__global__ void k_absent(const unsigned char* present, int64_t dim0, int32_t* rows,
                         int32_t* count) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= dim0) return;
  if (!present[i]) rows[atomicAdd(count, 1)] = static_cast<int32_t>(i);
}

// Parent coordinate broadcast one level down (child c of node n gets
// coord[n]), balanced for any fan-out: every parent with children marks its
// first child, an inclusive max-scan carries the parent id across its
// children, a gather reads the coordinate — three streaming passes, so a root
// slice with a million children costs no more than a million small fibers.
__global__ void k_mark_first_child(const int32_t* ptr, int32_t nparent, int32_t* mark) {
  const int32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= nparent) return;
  if (ptr[p] < ptr[p + 1]) mark[ptr[p]] = p;
}

__global__ void k_gather_parent(const int32_t* parent, const int32_t* coord, int64_t n,
                                int32_t* out) {
  const int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c < n) out[c] = coord[parent[c]];
}

// one thread per parent: for levels whose fan-out is ~1 (fibers of one leaf)
__global__ void k_child_coord_loop(const int32_t* ptr, const int32_t* coord, int32_t n,
                                   int32_t* child_coord) {
  const int32_t node = blockIdx.x * blockDim.x + threadIdx.x;
  if (node >= n) return;
  const int32_t v = coord[node];
  for (int32_t c = ptr[node]; c < ptr[node + 1]; ++c) child_coord[c] = v;
}

struct MaxI32 {
  __device__ __forceinline__ int32_t operator()(int32_t a, int32_t b) const { return a > b ? a : b; }
};

// Segment counts per unit node: ceil(children / seg_len).
// Child range of unit node f: its direct children, or (leaf_space) its
// leaves, found by following the child pointers down to the leaf level.
__device__ __forceinline__ void child_range(const CsfView& t, int unit_level, int32_t f,
                                            bool leaf_space, int32_t* b, int32_t* e) {
  int32_t lo = t.ptr[unit_level][f], hi = t.ptr[unit_level][f + 1];
  if (leaf_space)
    for (int l = unit_level + 1; l + 1 < t.order; ++l) {
      lo = t.ptr[l][lo];
      hi = t.ptr[l][hi];
    }
  *b = lo;
  *e = hi;
}

__global__ void k_seg_count(CsfView t, int unit_level, int seg_len, bool leaf_space,
                            int32_t* cnt) {
  const int32_t f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= t.nlev[unit_level]) return;
  int32_t b, e;
  child_range(t, unit_level, f, leaf_space, &b, &e);
  cnt[f] = (e - b + seg_len - 1) / seg_len;
}

__global__ void k_seg_fill(CsfView t, int unit_level, int seg_len, bool leaf_space,
                           const int32_t* off, const int32_t* unit_parent, int32_t* seg_begin,
                           int32_t* seg_node, int32_t* seg_node1) {
  const int32_t f = blockIdx.x * blockDim.x + threadIdx.x;
  const int32_t nf = t.nlev[unit_level];
  if (f >= nf) return;
  int32_t b, e;
  child_range(t, unit_level, f, leaf_space, &b, &e);
  const int32_t coord = t.idx[unit_level][f];
  const int32_t pc = unit_parent ? unit_parent[f] : 0;
  int32_t o = off[f];
  for (int32_t x = b; x < e; x += seg_len, ++o) {
    seg_begin[o] = x;
    seg_node[o] = coord;
    if (seg_node1) seg_node1[o] = pc;
  }
  if (f == nf - 1) seg_begin[o] = e;
}

// slice_seg[s] = first segment of root slice s: its first unit node is found
// by following the child pointers from level 0 down to unit_level.
__global__ void k_slice_seg(CsfView t, int unit_level, const int32_t* off, int32_t* slice_seg) {
  const int32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s > t.nlev[0]) return;
  int32_t node = s;
  for (int l = 0; l < unit_level; ++l) node = t.ptr[l][node];
  slice_seg[s] = off[node];
}

__global__ void k_seg_items(const int32_t* slice_seg, int32_t n0, int64_t chunk, int64_t n_items,
                            const int32_t* item_unit, int32_t* item_pos) {
  const int64_t w = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (w >= n_items) return;
  const int32_t u0 = item_unit ? item_unit[w] : static_cast<int32_t>(w * chunk);
  item_pos[w] = parent_of(slice_seg, n0, u0);
}

// item holding unit u: fixed chunks, or the last item starting at or before u
__device__ __forceinline__ int64_t item_of(int64_t u, int64_t chunk, const int32_t* item_unit,
                                           int64_t n_items) {
  if (!item_unit) return u / chunk;
  return parent_of(item_unit, static_cast<int32_t>(n_items), static_cast<int32_t>(u));
}

__global__ void k_seg_splits(CsfView t, const int32_t* slice_seg, int64_t chunk,
                             const int32_t* item_unit, int64_t n_items, int32_t* node,
                             int32_t* first, int32_t* last, int32_t* count,
                             unsigned char* present) {
  const int32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= t.nlev[0]) return;
  const int64_t f = item_of(slice_seg[s], chunk, item_unit, n_items);
  const int64_t g = item_of(static_cast<int64_t>(slice_seg[s + 1]) - 1, chunk, item_unit, n_items);
  if (f != g) {
    const int32_t slot = atomicAdd(count, 1);
    node[slot] = s;
    first[slot] = static_cast<int32_t>(f);
    last[slot] = static_cast<int32_t>(g);
  }
  present[t.idx[0][s]] = 1;
}

// per-group work of a packed group: its leaf steps plus the group overhead
// (header / slot loads, U gather, fragment transposition, 8 DMMA) in
// leaf-step units. Measured on the TTMc-3 BASELINE shape (kernel us):
// overhead 2: 295, 6: 259, 9: 252, 12: 249, 16: 249, 24: 251, equal group
// counts (infinite overhead): 256.

__global__ void k_group_work(const int4* hdr, int64_t n, int overhead, int64_t* work) {
  const int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g < n) work[g] = static_cast<int64_t>(hdr[g].y) + overhead;
}

// raw bound of item t: the first group whose inclusive work prefix (int64:
// total work reaches ~1.6 x nnz) exceeds t * total / n_items, stored as
// raw(t) - t for the max-scan that makes the bounds strictly increasing
__global__ void k_work_raw(const int64_t* cum, int64_t n, int64_t n_items, int32_t* raw_minus_t) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n_items) return;
  if (t == 0) { raw_minus_t[0] = 0; return; }
  const int64_t total = cum[n - 1];
  // total * t / n_items without overflowing int64
  const int64_t target = static_cast<int64_t>(
      (static_cast<__int128>(total) * t) / n_items);
  int64_t lo = 0, hi = n;  // first g with cum[g] > target
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (cum[mid] > target) hi = mid; else lo = mid + 1;
  }
  raw_minus_t[t] = static_cast<int32_t>(lo - t);
}

// item_unit[t] = t + max_{s<=t}(raw(s) - s), capped at n - (n_items - t):
// both sequences rise by >= 1 per item, so every item holds >= 1 group even
// when one heavy group spans several items' shares of the work
__global__ void k_work_bounds(const int32_t* scanned, int64_t n, int64_t n_items,
                              int32_t* item_unit) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t > n_items) return;
  if (t == n_items) { item_unit[t] = static_cast<int32_t>(n); return; }
  int64_t b = static_cast<int64_t>(scanned[t]) + t;
  const int64_t cap = n - (n_items - t);
  item_unit[t] = static_cast<int32_t>(b < cap ? b : cap);
}

unsigned blocks_for(int64_t n, int b) { return static_cast<unsigned>((n + b - 1) / b); }

void child_coords(const int32_t* ptr, int32_t nparent, const int32_t* coord, int64_t nchild,
                  int32_t* out, cudaStream_t s) {
  if (nchild == 0 || nparent == 0) return;
  if (nchild <= 4 * static_cast<int64_t>(nparent)) {  // small fan-out: a loop per parent
    k_child_coord_loop<<<blocks_for(nparent, 256), 256, 0, s>>>(ptr, coord, nparent, out);
    SPTTN_CUDA(cudaGetLastError());
    return;
  }
  int32_t* mark = nullptr;
  dmalloc(&mark, nchild * sizeof(int32_t), s);
  SPTTN_CUDA(cudaMemsetAsync(mark, 0, nchild * sizeof(int32_t), s));
  k_mark_first_child<<<blocks_for(nparent, 256), 256, 0, s>>>(ptr, nparent, mark);
  size_t bytes = 0;
  SPTTN_CUDA(cub::DeviceScan::InclusiveScan(nullptr, bytes, mark, mark, MaxI32{},
                                            static_cast<int>(nchild), s));
  void* tmp = nullptr;
  dmalloc(&tmp, std::max<size_t>(1, bytes), s);
  SPTTN_CUDA(cub::DeviceScan::InclusiveScan(tmp, bytes, mark, mark, MaxI32{},
                                            static_cast<int>(nchild), s));
  k_gather_parent<<<blocks_for(nchild, 256), 256, 0, s>>>(mark, coord, nchild, out);
  SPTTN_CUDA(cudaGetLastError());
  dfree(tmp, s);
  dfree(mark, s);
}

// slice_units: first work unit (segment / packed group) of every root slice,
// or nullptr when items are leaf ranges.
void find_splits_and_absent(const DevCsf& csf, Decomp& d, const int32_t* slice_units,
                            cudaStream_t s) {
  const bool segments = slice_units != nullptr;
  const CsfView t = csf.view();
  const int32_t n0 = static_cast<int32_t>(csf.level_size[0]);
  int32_t* counts = nullptr;
  unsigned char* present = nullptr;
  dmalloc(&counts, 2 * sizeof(int32_t), s);
  SPTTN_CUDA(cudaMemsetAsync(counts, 0, 2 * sizeof(int32_t), s));
  dmalloc(&present, csf.dims[0], s);
  SPTTN_CUDA(cudaMemsetAsync(present, 0, csf.dims[0], s));
  const int64_t nsplit_cap = n0 > 0 ? n0 : 1;
  dmalloc(&d.split_node, nsplit_cap * sizeof(int32_t), s);
  dmalloc(&d.split_first, nsplit_cap * sizeof(int32_t), s);
  dmalloc(&d.split_last, nsplit_cap * sizeof(int32_t), s);
  dmalloc(&d.absent_rows, csf.dims[0] * sizeof(int32_t), s);
  if (n0 > 0) {
    if (segments)
      k_seg_splits<<<blocks_for(n0, 256), 256, 0, s>>>(t, slice_units, d.chunk, d.item_unit,
                                                       d.n_items, d.split_node, d.split_first,
                                                       d.split_last, counts, present);
    else
      k_leaf_splits<<<blocks_for(n0, 256), 256, 0, s>>>(t, d.chunk, d.split_node, d.split_first,
                                                        d.split_last, counts, present);
    SPTTN_CUDA(cudaGetLastError());
  }
  k_absent<<<blocks_for(csf.dims[0], 256), 256, 0, s>>>(present, csf.dims[0], d.absent_rows,
                                                          counts + 1);
  SPTTN_CUDA(cudaGetLastError());
  int32_t h[2] = {0, 0};
  SPTTN_CUDA(cudaMemcpyAsync(h, counts, sizeof(h), cudaMemcpyDeviceToHost, s));
  SPTTN_CUDA(cudaStreamSynchronize(s));
  d.n_split = h[0];
  d.n_absent = h[1];
  build_fixup_chunks(d, t.idx[0], s);
  dfree(counts, s);
  dfree(present, s);
}

}  // namespace

void plan_trace(const char* what, cudaStream_t s) {
  static const bool on = [] {
    const char* e = std::getenv("SPTTN_PLAN_TRACE");
    return e && *e && *e != '0';
  }();
  if (!on) return;
  using clk = std::chrono::steady_clock;
  static clk::time_point last = clk::now();
  cudaStreamSynchronize(s);
  const clk::time_point now = clk::now();
  std::fprintf(stderr, "[plan] %-28s %8.3f ms\n", what,
               std::chrono::duration<double, std::milli>(now - last).count());
  last = now;
}

void build_leaf_items(const DevCsf& csf, int64_t chunk, Decomp& d, int64_t tile, cudaStream_t s) {
  const int64_t nnz = csf.level_size[csf.order - 1];
  d.chunk = chunk;
  d.tile = tile;
  d.n_items = (nnz + chunk - 1) / chunk;
  const CsfView t = csf.view();
  dmalloc(&d.item_pos, std::max<int64_t>(1, d.n_items * csf.order) * sizeof(int32_t), s);
  if (d.n_items > 0) {
    k_leaf_items<<<blocks_for(d.n_items, 256), 256, 0, s>>>(t, chunk, d.n_items, d.item_pos);
    SPTTN_CUDA(cudaGetLastError());
  }
  if (tile > 0) {  // dense root-indexed output
    dmalloc(&d.part, std::max<int64_t>(1, d.n_items * 2 * tile) * sizeof(double), s);
    find_splits_and_absent(csf, d, nullptr, s);
  }
}

void build_segments(const DevCsf& csf, int unit_level, int seg_len, int64_t chunk, Decomp& d,
                    int64_t tile, cudaStream_t s, bool make_items, bool leaf_space) {
  const CsfView t = csf.view();
  const int32_t nf = static_cast<int32_t>(csf.level_size[unit_level]);
  const int32_t n0 = static_cast<int32_t>(csf.level_size[0]);
  d.seg_len = seg_len;
  d.chunk = chunk;
  d.tile = tile;
  int32_t* off = nullptr;
  dmalloc(&off, (static_cast<int64_t>(nf) + 1) * sizeof(int32_t), s);
  SPTTN_CUDA(cudaMemsetAsync(off, 0, (static_cast<int64_t>(nf) + 1) * sizeof(int32_t), s));
  if (nf > 0) {
    k_seg_count<<<blocks_for(nf, 256), 256, 0, s>>>(t, unit_level, seg_len, leaf_space, off);
    SPTTN_CUDA(cudaGetLastError());
  }
  size_t temp_bytes = 0;
  SPTTN_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, temp_bytes, off, off, nf + 1, s));
  void* temp = nullptr;
  dmalloc(&temp, temp_bytes, s);
  SPTTN_CUDA(cub::DeviceScan::ExclusiveSum(temp, temp_bytes, off, off, nf + 1, s));
  dfree(temp, s);
  int32_t nseg = 0;
  SPTTN_CUDA(cudaMemcpyAsync(&nseg, off + nf, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  SPTTN_CUDA(cudaStreamSynchronize(s));
  d.n_seg = nseg;
  dmalloc(&d.seg_begin, (static_cast<int64_t>(nseg) + 1) * sizeof(int32_t), s);
  dmalloc(&d.seg_node, std::max<int64_t>(1, nseg) * sizeof(int32_t), s);
  dmalloc(&d.slice_seg, (static_cast<int64_t>(n0) + 1) * sizeof(int32_t), s);
  SPTTN_CUDA(cudaMemsetAsync(d.seg_begin, 0, sizeof(int32_t), s));
  int32_t* unit_parent = nullptr;  // level-1 coordinate of each unit node (unit_level 2)
  if (unit_level == 2) {
    dmalloc(&d.seg_node1, std::max<int64_t>(1, nseg) * sizeof(int32_t), s);
    dmalloc(&unit_parent, std::max<int32_t>(1, nf) * sizeof(int32_t), s);
    const int32_t n1 = static_cast<int32_t>(csf.level_size[1]);
    if (n1 > 0)
      child_coords(t.ptr[1], n1, t.idx[1], nf, unit_parent, s);
  }
  if (nf > 0) {
    k_seg_fill<<<blocks_for(nf, 256), 256, 0, s>>>(t, unit_level, seg_len, leaf_space, off,
                                                   unit_parent, d.seg_begin, d.seg_node,
                                                   d.seg_node1);
    SPTTN_CUDA(cudaGetLastError());
  }
  if (unit_parent) dfree(unit_parent, s);
  k_slice_seg<<<blocks_for(static_cast<int64_t>(n0) + 1, 256), 256, 0, s>>>(t, unit_level, off,
                                                                          d.slice_seg);
  SPTTN_CUDA(cudaGetLastError());
  dfree(off, s);
  plan_trace("build_segments", s);
  if (make_items) finish_unit_items(csf, d, d.slice_seg, d.n_seg, chunk, tile, s);
}

void finish_unit_items(const DevCsf& csf, Decomp& d, const int32_t* slice_units, int64_t n_units,
                       int64_t chunk, int64_t tile, cudaStream_t s, int group_overhead) {
  const int32_t n0 = static_cast<int32_t>(csf.level_size[0]);
  d.chunk = chunk;
  d.tile = tile;
  d.n_items = (n_units + chunk - 1) / chunk;
  if (group_overhead > 0 && d.n_items > 1) {
    // cumulative work per packed group (leaf steps + per-group overhead),
    // then item t starts at the first group whose prefix reaches t/n of it
    int64_t* cum = nullptr;
    dmalloc(&cum, n_units * sizeof(int64_t), s);
    k_group_work<<<blocks_for(n_units, 256), 256, 0, s>>>(d.grp_hdr, n_units, group_overhead, cum);
    size_t bytes = 0;
    SPTTN_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, cum, cum, n_units, s));
    void* tmp = nullptr;
    dmalloc(&tmp, std::max<size_t>(1, bytes), s);
    SPTTN_CUDA(cub::DeviceScan::InclusiveSum(tmp, bytes, cum, cum, n_units, s));
    dfree(tmp, s);
    int32_t* raw = nullptr;
    dmalloc(&raw, d.n_items * sizeof(int32_t), s);
    k_work_raw<<<blocks_for(d.n_items, 256), 256, 0, s>>>(cum, n_units, d.n_items, raw);
    SPTTN_CUDA(cudaGetLastError());
    bytes = 0;
    SPTTN_CUDA(cub::DeviceScan::InclusiveScan(nullptr, bytes, raw, raw, MaxI32{},
                                              static_cast<int>(d.n_items), s));
    dmalloc(&tmp, std::max<size_t>(1, bytes), s);
    SPTTN_CUDA(cub::DeviceScan::InclusiveScan(tmp, bytes, raw, raw, MaxI32{},
                                              static_cast<int>(d.n_items), s));
    dfree(tmp, s);
    dmalloc(&d.item_unit, (d.n_items + 1) * sizeof(int32_t), s);
    k_work_bounds<<<blocks_for(d.n_items + 1, 256), 256, 0, s>>>(raw, n_units, d.n_items,
                                                                 d.item_unit);
    SPTTN_CUDA(cudaGetLastError());
    dfree(raw, s);
    dfree(cum, s);
  }
  dmalloc(&d.item_pos, std::max<int64_t>(1, d.n_items) * sizeof(int32_t), s);
  if (d.n_items > 0) {
    k_seg_items<<<blocks_for(d.n_items, 256), 256, 0, s>>>(slice_units, n0, chunk, d.n_items,
                                                          d.item_unit, d.item_pos);
    SPTTN_CUDA(cudaGetLastError());
  }
  dmalloc(&d.part, std::max<int64_t>(1, d.n_items * 2 * tile) * sizeof(double), s);
  plan_trace("unit items", s);
  find_splits_and_absent(csf, d, slice_units, s);
  plan_trace("splits/absent/fixup chunks", s);
}

void expand_coords(const DevCsf& csf, int level, const int32_t* coords, int32_t* out,
                   cudaStream_t s) {
  const int32_t n = static_cast<int32_t>(csf.level_size[level]);
  if (n > 0) {
    child_coords(csf.ptr[level], n, coords, csf.level_size[level + 1], out, s);
    SPTTN_CUDA(cudaGetLastError());
  }
}

void build_leaf_coords(const DevCsf& csf, int32_t** leaf_i, int32_t** leaf_j, cudaStream_t s) {
  const int64_t n0 = csf.level_size[0], n1 = csf.level_size[1], nnz = csf.level_size[2];
  int32_t* fib_i = nullptr;
  dmalloc(leaf_i, std::max<int64_t>(1, nnz) * sizeof(int32_t), s);
  dmalloc(leaf_j, std::max<int64_t>(1, nnz) * sizeof(int32_t), s);
  dmalloc(&fib_i, std::max<int64_t>(1, n1) * sizeof(int32_t), s);
  child_coords(csf.ptr[0], static_cast<int32_t>(n0), csf.idx[0], n1, fib_i, s);
  child_coords(csf.ptr[1], static_cast<int32_t>(n1), csf.idx[1], nnz, *leaf_j, s);
  child_coords(csf.ptr[1], static_cast<int32_t>(n1), fib_i, nnz, *leaf_i, s);
  SPTTN_CUDA(cudaGetLastError());
  dfree(fib_i, s);
}

namespace {

// Two-level fix-up for slices spread over many items. Level 1: one block per
// chunk of <= kFixChunk consecutive items of one split slice sums their
// partial tiles (TAIL of the slice's first item, HEAD of the others) in item
// order; level 2: one block per split slice sums its chunk tiles in chunk
// order. Both orders are fixed by the plan, so results are deterministic.
// Epilogue, pass 1 — one warp per work unit. Warps [0, n_chunk) each sum one
// chunk of <= kFixChunk items of a split root slice (the first item's TAIL
// tile, the other items' HEAD tiles, in item order; lanes stride the tile
// with 256-bit loads, 8 item tiles in flight). A slice with one chunk is
// written straight to the output, otherwise the chunk sum goes to part2 for
// pass 2. Warps past n_chunk zero absent rows.
template <bool V4>
__global__ void __launch_bounds__(256) k_fix1(const int4* __restrict__ meta,
                                              const double* __restrict__ part, int64_t tile,
                                              int64_t n_chunk, double* part2,
                                              const int32_t* absent_rows, int64_t n_absent,
                                              double* out) {
  const int64_t wid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  if (wid >= n_chunk) {  // absent root rows: zero their output tiles
    grid_dependency_wait();
    const int64_t zw = nwarps - n_chunk;
    for (int64_t z = (wid - n_chunk) * 32 + lane; z < n_absent * tile; z += zw * 32)
      out[static_cast<int64_t>(absent_rows[z / tile]) * tile + z % tile] = 0.0;
    return;
  }
  // one dependent metadata load per chunk (built at plan time, so it is
  // read before waiting for the nest kernel under programmatic launch)
  const int4 m = meta[wid];
  grid_dependency_wait();
  const int32_t lo = m.x, hi = m.y, first = m.z;
  double* dst = m.w >= 0 ? out + static_cast<int64_t>(m.w) * tile : part2 + wid * tile;
  const int64_t nv = V4 ? tile / 4 : tile;
  for (int64_t e = lane; e < nv; e += 32) {
    double4 sum = make_double4(0, 0, 0, 0);
    for (int32_t it = lo; it <= hi; it += 8) {
      double4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int32_t i = it + u;
        const double* src = part + (static_cast<int64_t>(i) * 2 + (i == first ? 1 : 0)) * tile;
        if (V4)
          v[u] = i <= hi ? reinterpret_cast<const double4*>(src)[e] : make_double4(0, 0, 0, 0);
        else
          v[u] = make_double4(i <= hi ? src[e] : 0.0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (it + u <= hi) {
          sum.x += v[u].x;
          sum.y += v[u].y;
          sum.z += v[u].z;
          sum.w += v[u].w;
        }
    }
    if (V4)
      reinterpret_cast<double4*>(dst)[e] = sum;
    else
      dst[e] = sum.x;
  }
}

__global__ void k_chunk_meta(const int32_t* chunk_split, const int32_t* chunk_lo,
                             const int32_t* chunk_hi, const int32_t* split_first,
                             const int32_t* split_chunk, const int32_t* split_node,
                             const int32_t* idx0, int64_t n_chunk, int4* meta) {
  const int64_t w = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (w >= n_chunk) return;
  const int32_t sidx = chunk_split[w];
  const bool single = split_chunk[sidx + 1] - split_chunk[sidx] == 1;
  meta[w] = make_int4(chunk_lo[w], chunk_hi[w], split_first[sidx],
                      single ? idx0[split_node[sidx]] : -1);
}

// Epilogue, pass 2 — one block per slice split into several chunks (the
// heavy root slices of skewed tensors). The block's threads form G groups of
// tile/4 (or tile) threads; group g adds chunk sums c0+g, c0+g+G, ... in
// order (8 loads in flight), then the G group sums are added in group order
// through shared memory. Fixed order: deterministic.
template <bool V4>
__global__ void __launch_bounds__(256) k_fix2(const int32_t* multi, const int32_t* split_chunk,
                                              const int32_t* split_node, const int32_t* idx0,
                                              const double* part2, int64_t tile, double* out) {
  __shared__ double4 ws[256];
  const int32_t sidx = multi[blockIdx.x];
  const int32_t c0 = split_chunk[sidx], c1 = split_chunk[sidx + 1];
  const int64_t row = idx0[split_node[sidx]];
  grid_dependency_wait();
  const int64_t nv = V4 ? tile / 4 : tile;  // vector elements per tile
  // piece of the tile handled per pass: up to 256 elements, G = 256 / piece groups
  const int64_t piece = nv < 256 ? nv : 256;
  const int G = static_cast<int>(256 / piece);
  const int g = threadIdx.x / static_cast<int>(piece);
  const int64_t el = threadIdx.x % piece;
  for (int64_t p0 = 0; p0 < nv; p0 += piece) {
    const int64_t e = p0 + el;
    const bool act = g < G && e < nv;
    double4 sum = make_double4(0, 0, 0, 0);
    if (act) {
      for (int32_t c = c0 + g; c < c1; c += 8 * G) {
        double4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int32_t k = c + u * G;
          const double* src = part2 + static_cast<int64_t>(k) * tile;
          if (V4)
            v[u] = k < c1 ? reinterpret_cast<const double4*>(src)[e] : make_double4(0, 0, 0, 0);
          else
            v[u] = make_double4(k < c1 ? src[e] : 0.0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (c + u * G < c1) {
            sum.x += v[u].x;
            sum.y += v[u].y;
            sum.z += v[u].z;
            sum.w += v[u].w;
          }
      }
    }
    ws[threadIdx.x] = sum;
    __syncthreads();
    if (g == 0 && e < nv) {
      double4 t = ws[el];
      for (int k = 1; k < G; ++k) {
        const double4 o = ws[k * piece + el];
        t.x += o.x;
        t.y += o.y;
        t.z += o.z;
        t.w += o.w;
      }
      if (V4)
        reinterpret_cast<double4*>(out + row * tile)[e] = t;
      else
        out[row * tile + e] = t.x;
    }
    __syncthreads();
  }
}

// Epilogue in one launch: blocks [0, n_multi) each sum one heavy split slice
// straight from its items' partial tiles (TAIL of the first item, HEAD of the
// others; G thread groups stride the items in order, 8 loads in flight, then
// the group sums are added in group order: a fixed order, deterministic);
// the other blocks run k_fix1's warp-per-chunk pass for the single-chunk
// split slices and zero the absent rows. One launch instead of k_fix1 then
// k_fix2 — the second dependent launch cost ~4 us per step.
// 1024 threads: a heavy slice's items are strided by up to 1024 / tile-quads
// thread groups (MTTKRP-4: 128 groups over ~2500 items of its largest slice)
constexpr int kFixBlock = 1024;
template <bool V4>
__global__ void __launch_bounds__(kFixBlock) k_fix_all(const int4* __restrict__ meta,
                                                 const double* __restrict__ part, int64_t tile,
                                                 int64_t n_chunk, const int32_t* absent_rows,
                                                 int64_t n_absent, double* out,
                                                 const int32_t* multi, int64_t n_multi,
                                                 const int32_t* split_first,
                                                 const int32_t* split_last,
                                                 const int32_t* split_node, const int32_t* idx0) {
  __shared__ double4 ws[kFixBlock];
  const int64_t nv = V4 ? tile / 4 : tile;
  if (blockIdx.x < n_multi) {
    const int32_t sidx = multi[blockIdx.x];
    const int32_t first = split_first[sidx], last = split_last[sidx];
    const int64_t row = idx0[split_node[sidx]];
    grid_dependency_wait();
    const int64_t piece = nv < kFixBlock ? nv : kFixBlock;
    const int G = static_cast<int>(kFixBlock / piece);
    const int g = threadIdx.x / static_cast<int>(piece);
    const int64_t el = threadIdx.x % piece;
    for (int64_t p0 = 0; p0 < nv; p0 += piece) {
      const int64_t e = p0 + el;
      const bool act = g < G && e < nv;
      double4 sum = make_double4(0, 0, 0, 0);
      if (act) {
        for (int32_t i0 = first + g; i0 <= last; i0 += 8 * G) {
          double4 v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int32_t i = i0 + u * G;
            const double* src = part + (static_cast<int64_t>(i) * 2 + (i == first ? 1 : 0)) * tile;
            if (V4)
              v[u] = i <= last ? reinterpret_cast<const double4*>(src)[e] : make_double4(0, 0, 0, 0);
            else
              v[u] = make_double4(i <= last ? src[e] : 0.0, 0, 0, 0);
          }
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (i0 + u * G <= last) {
              sum.x += v[u].x;
              sum.y += v[u].y;
              sum.z += v[u].z;
              sum.w += v[u].w;
            }
        }
      }
      ws[threadIdx.x] = sum;
      __syncthreads();
      if (g == 0 && e < nv) {
        double4 t = ws[el];
        for (int k = 1; k < G; ++k) {
          const double4 o = ws[k * piece + el];
          t.x += o.x;
          t.y += o.y;
          t.z += o.z;
          t.w += o.w;
        }
        if (V4)
          reinterpret_cast<double4*>(out + row * tile)[e] = t;
        else
          out[row * tile + e] = t.x;
      }
      __syncthreads();
    }
    return;
  }
  const int64_t wid =
      ((static_cast<int64_t>(blockIdx.x) - n_multi) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((static_cast<int64_t>(gridDim.x) - n_multi) * blockDim.x) >> 5;
  if (wid >= n_chunk) {  // absent root rows: zero their output tiles
    grid_dependency_wait();
    const int64_t zw = nwarps - n_chunk;
    for (int64_t z = (wid - n_chunk) * 32 + lane; z < n_absent * tile; z += zw * 32)
      out[static_cast<int64_t>(absent_rows[z / tile]) * tile + z % tile] = 0.0;
    return;
  }
  const int4 m = meta[wid];
  if (m.w < 0) return;  // a chunk of a heavy slice: summed by its slice's block above
  grid_dependency_wait();
  const int32_t lo = m.x, hi = m.y, first = m.z;
  double* dst = out + static_cast<int64_t>(m.w) * tile;
  for (int64_t e = lane; e < nv; e += 32) {
    double4 sum = make_double4(0, 0, 0, 0);
    for (int32_t it = lo; it <= hi; it += 8) {
      double4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int32_t i = it + u;
        const double* src = part + (static_cast<int64_t>(i) * 2 + (i == first ? 1 : 0)) * tile;
        if (V4)
          v[u] = i <= hi ? reinterpret_cast<const double4*>(src)[e] : make_double4(0, 0, 0, 0);
        else
          v[u] = make_double4(i <= hi ? src[e] : 0.0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (it + u <= hi) {
          sum.x += v[u].x;
          sum.y += v[u].y;
          sum.z += v[u].z;
          sum.w += v[u].w;
        }
    }
    if (V4)
      reinterpret_cast<double4*>(dst)[e] = sum;
    else
      dst[e] = sum.x;
  }
}

}  // namespace

void build_fixup_chunks(Decomp& d, const int32_t* idx0, cudaStream_t s) {
  if (d.n_split == 0) return;
  std::vector<int32_t> first(d.n_split), last(d.n_split);
  SPTTN_CUDA(cudaMemcpyAsync(first.data(), d.split_first, d.n_split * sizeof(int32_t),
                             cudaMemcpyDeviceToHost, s));
  SPTTN_CUDA(cudaMemcpyAsync(last.data(), d.split_last, d.n_split * sizeof(int32_t),
                             cudaMemcpyDeviceToHost, s));
  SPTTN_CUDA(cudaStreamSynchronize(s));
  std::vector<int32_t> cs, clo, chi, sc(d.n_split + 1, 0), multi;
  for (int64_t k = 0; k < d.n_split; ++k) {
    sc[k] = static_cast<int32_t>(cs.size());
    for (int32_t lo = first[k]; lo <= last[k]; lo += kFixChunk) {
      cs.push_back(static_cast<int32_t>(k));
      clo.push_back(lo);
      chi.push_back(std::min(last[k], lo + kFixChunk - 1));
    }
    if (static_cast<int32_t>(cs.size()) - sc[k] > 1) multi.push_back(static_cast<int32_t>(k));
  }
  sc[d.n_split] = static_cast<int32_t>(cs.size());
  d.n_chunk = static_cast<int64_t>(cs.size());
  auto up = [&](int32_t** dst, const std::vector<int32_t>& v) {
    dmalloc(dst, std::max<size_t>(1, v.size()) * sizeof(int32_t), s);
    SPTTN_CUDA(cudaMemcpyAsync(*dst, v.data(), v.size() * sizeof(int32_t), cudaMemcpyHostToDevice, s));
  };
  up(&d.chunk_split, cs);
  up(&d.chunk_lo, clo);
  up(&d.chunk_hi, chi);
  up(&d.split_chunk, sc);
  up(&d.multi_split, multi);
  d.n_multi = static_cast<int64_t>(multi.size());
  dmalloc(&d.part2, std::max<int64_t>(1, d.n_chunk * d.tile) * sizeof(double), s);
  dmalloc(&d.chunk_meta, std::max<int64_t>(1, d.n_chunk) * sizeof(int4), s);
  if (d.n_chunk > 0)
    k_chunk_meta<<<blocks_for(d.n_chunk, 256), 256, 0, s>>>(d.chunk_split, d.chunk_lo, d.chunk_hi,
                                                           d.split_first, d.split_chunk,
                                                           d.split_node, idx0, d.n_chunk,
                                                           d.chunk_meta);
  SPTTN_CUDA(cudaGetLastError());
  SPTTN_CUDA(cudaStreamSynchronize(s));
}

void launch_fixup(const Decomp& d, const CsfView& t, double* out, cudaStream_t s) {
  if (d.n_split == 0 && d.n_absent == 0) return;
  const int64_t zero_warps =
      d.n_absent > 0 ? std::min<int64_t>((d.n_absent * d.tile + 31) / 32, 148 * 64) : 0;
  // programmatic dependent launch: the fix-up grids are scheduled while the
  // previous kernel drains and wait in griddepcontrol.wait for its results
  static const int sms = [] {
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  if (d.n_multi <= sms) {
    // few heavy slices (TTMc-3: split slices 2069, heavy ~tens): one launch,
    // each heavy slice summed by one 1024-thread block (step 234.5 -> 230.4
    // us for TTMc-3, 349.2 -> 345.2 us for TTMc-4)
    const unsigned blocks =
        static_cast<unsigned>(d.n_multi) + blocks_for((d.n_chunk + zero_warps) * 32, kFixBlock);
    if (d.tile % 4 == 0)
      launch_pdl(k_fix_all<true>, blocks, kFixBlock, s, d.chunk_meta, d.part, d.tile, d.n_chunk,
                 d.absent_rows, d.n_absent, out, d.multi_split, d.n_multi, d.split_first,
                 d.split_last, d.split_node, t.idx[0]);
    else
      launch_pdl(k_fix_all<false>, blocks, kFixBlock, s, d.chunk_meta, d.part, d.tile, d.n_chunk,
                 d.absent_rows, d.n_absent, out, d.multi_split, d.n_multi, d.split_first,
                 d.split_last, d.split_node, t.idx[0]);
    SPTTN_CUDA(cudaGetLastError());
    return;
  }
  // many heavy slices (MTTKRP-4 Zipf): chunk sums spread over warps, then
  // one block per heavy slice over its chunk sums (two launches)
  const unsigned blocks = blocks_for((d.n_chunk + zero_warps) * 32, 256);
  if (d.tile % 4 == 0)
    launch_pdl(k_fix1<true>, blocks, 256, s, d.chunk_meta, d.part, d.tile, d.n_chunk, d.part2,
               d.absent_rows, d.n_absent, out);
  else
    launch_pdl(k_fix1<false>, blocks, 256, s, d.chunk_meta, d.part, d.tile, d.n_chunk, d.part2,
               d.absent_rows, d.n_absent, out);
  const unsigned nb = static_cast<unsigned>(d.n_multi);
  if (d.tile % 4 == 0)
    launch_pdl(k_fix2<true>, nb, 256, s, d.multi_split, d.split_chunk, d.split_node, t.idx[0],
               d.part2, d.tile, out);
  else
    launch_pdl(k_fix2<false>, nb, 256, s, d.multi_split, d.split_chunk, d.split_node, t.idx[0],
               d.part2, d.tile, out);
  SPTTN_CUDA(cudaGetLastError());
}

void free_decomp(Decomp& d) {
  dfree(d.item_pos);
  dfree(d.part);
  dfree(d.split_node);
  dfree(d.split_first);
  dfree(d.split_last);
  dfree(d.absent_rows);
  dfree(d.seg_begin);
  dfree(d.seg_node);
  dfree(d.seg_node1);
  dfree(d.chunk_meta);
  dfree(d.chunk_split);
  dfree(d.chunk_lo);
  dfree(d.chunk_hi);
  dfree(d.split_chunk);
  dfree(d.part2);
  dfree(d.multi_split);
  dfree(d.grp_hdr);
  dfree(d.grp_node);
  dfree(d.grp_node1);
  dfree(d.pk);
  dfree(d.pk2);
  dfree(d.pv);
  dfree(d.slice_grp);
  dfree(d.slice_seg);
  dfree(d.cta_grp);
  dfree(d.item_unit);
  dfree(d.hdr2);
  d = Decomp{};
}

}  // namespace spttn_dev
