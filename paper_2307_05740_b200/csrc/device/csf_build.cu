// Device CSF construction from COO and CSF export.
//
// The reference builds the CSF on the host: CooTensor::normalize sorts the
// entries and sums duplicates (proj/src/tensor.cpp:24-35), build_csf sorts
// the rows in mode order and emits a new node at level l wherever the
// coordinate prefix [0, l] changes, with ptr[l] = the child count so far
// (tensor.cpp:41-94) — 0.42 s at 1e6 nnz, sort-dominated. Here the same tree
// is built on the GPU straight into the engine's int32 device layout:
//   1. LSD radix sort of the row permutation, one stable CUB pass per level
//      from the last level to the root (bits per pass from the mode size);
//   2. duplicate rows (all coordinates equal) summed in input order — the
//      stable sort keeps equal rows in input order, like the host restatement
//      (the reference's std::sort leaves the order of 3+ duplicates
//      unspecified; two duplicates sum identically either way);
//   3. per level: new-node flags (prefix change), node ids by an inclusive
//      scan, idx[l][node] = coordinate, ptr[l][node] = first child's id at
//      level l+1, sentinel = level l+1 node count.
#include <cub/cub.cuh>

#include "../../../include/spttn_b200.h"
#include "internal.cuh"

namespace spttn_dev {

namespace {

unsigned nb(int64_t n, int b) { return static_cast<unsigned>((n + b - 1) / b); }

__global__ void k_level_keys(const int64_t* coords, int64_t nnz, int d, int l, int64_t dim,
                             uint32_t* key, int* err) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= nnz) return;
  const int64_t c = coords[e * d + l];
  if (c < 0 || c >= dim) atomicOr(err, 1);
  key[e] = static_cast<uint32_t>(c);
}

__global__ void k_iota(int32_t* v, int64_t n) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e < n) v[e] = static_cast<int32_t>(e);
}

// per-level coordinates, SoA int32 (device)
struct Soa {
  const int32_t* c[kMaxOrder];
};

__global__ void k_aos_to_soa(const int64_t* coords, int64_t nnz, int d, Soa out) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= nnz) return;
  for (int l = 0; l < d; ++l) const_cast<int32_t*>(out.c[l])[e] = static_cast<int32_t>(coords[e * d + l]);
}

__global__ void k_gather_keys(Soa co, int l, const int32_t* perm, int64_t n, uint32_t* out) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r < n) out[r] = static_cast<uint32_t>(co.c[l][perm[r]]);
}

// parent coordinate broadcast to every child, one thread per child (binary
// search of the child's parent: balanced for any fan-out)
__global__ void k_expand_parent(const int32_t* ptr, int32_t nparent, const int32_t* pcoord,
                                int64_t nchild, int32_t* out) {
  const int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= nchild) return;
  int32_t lo = 0, hi = nparent;  // largest p with ptr[p] <= c
  while (hi - lo > 1) {
    const int32_t mid = (lo + hi) >> 1;
    if (ptr[mid] <= c) lo = mid; else hi = mid;
  }
  out[c] = pcoord[lo];
}

// run heads: row r of the sorted order starts a new distinct coordinate tuple
__global__ void k_run_heads(Soa co, int d, const int32_t* perm, int64_t n, int32_t* head) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n) return;
  int h = r == 0;
  if (!h)
    for (int l = 0; l < d; ++l) h |= co.c[l][perm[r]] != co.c[l][perm[r - 1]];
  head[r] = h;
}

// unique row u (= run id) <- first sorted row of its run; values summed over
// the run in sorted (= input) order
__global__ void k_merge_runs(const int32_t* head, const int32_t* run_id, const int32_t* perm,
                             const double* vals, int64_t n, int32_t* urow, double* uval) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n || !head[r]) return;
  double s = vals[perm[r]];
  for (int64_t q = r + 1; q < n && !head[q]; ++q) s += vals[perm[q]];
  urow[run_id[r] - 1] = perm[r];
  uval[run_id[r] - 1] = s;
}

// new node at level l for unique row u: its prefix [0, l] differs from u-1
__global__ void k_node_flags(Soa co, int l, const int32_t* urow, int64_t nu, int32_t* flag) {
  const int64_t u = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (u >= nu) return;
  int f = u == 0;
  if (!f)
    for (int m = 0; m <= l; ++m) f |= co.c[m][urow[u]] != co.c[m][urow[u - 1]];
  flag[u] = f;
}

// nid_l = inclusive scan of the level-l flags (1-based); for level l < d-1
// the first child of node nid_l[u]-1 is node nid_{l+1}[u]-1
__global__ void k_emit_level(Soa co, int l, const int32_t* urow, const int32_t* flag,
                             const int32_t* nid, const int32_t* nid_next, int64_t nu,
                             int32_t* idx, int32_t* ptr) {
  const int64_t u = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (u >= nu || !flag[u]) return;
  const int32_t node = nid[u] - 1;
  idx[node] = co.c[l][urow[u]];
  if (ptr) ptr[node] = nid_next[u] - 1;
}

__global__ void k_widen(const int32_t* src, int64_t n, int64_t* dst) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e < n) dst[e] = src[e];
}

template <class T>
T* scratch(int64_t n, cudaStream_t s) {
  T* p = nullptr;
  dmalloc(&p, static_cast<size_t>(std::max<int64_t>(1, n)) * sizeof(T), s);
  return p;
}

void scan_incl_sum(int32_t* in, int32_t* out, int64_t n, cudaStream_t s) {
  size_t bytes = 0;
  SPTTN_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, in, out, static_cast<int>(n), s));
  void* tmp = scratch<unsigned char>(static_cast<int64_t>(bytes), s);
  SPTTN_CUDA(cub::DeviceScan::InclusiveSum(tmp, bytes, in, out, static_cast<int>(n), s));
  dfree(tmp, s);
}

int bits_for(int64_t dim) {
  int b = 1;
  while (b < 32 && (int64_t{1} << b) < dim) ++b;
  return b;
}

}  // namespace

namespace {

// The build proper: device SoA coordinates (co.c[l], CSF level order) and
// values -> D (sorted rows, duplicates summed in order, levels emitted).
void build_from_soa(DevCsf& D, int d, const int64_t* dims, int64_t nnz, const Soa& co,
                    const double* vals, cudaStream_t s) {
  D.order = d;
  for (int l = 0; l < d; ++l) D.dims[l] = dims[l];
  // 1. LSD radix sort of the row permutation, last level first
  uint32_t* key = scratch<uint32_t>(nnz, s);
  uint32_t* key2 = scratch<uint32_t>(nnz, s);
  int32_t* perm = scratch<int32_t>(nnz, s);
  int32_t* perm2 = scratch<int32_t>(nnz, s);
  if (nnz > 0) k_iota<<<nb(nnz, 256), 256, 0, s>>>(perm, nnz);
  size_t tbytes = 0;
  SPTTN_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tbytes, key, key2, perm, perm2,
                                             static_cast<int>(nnz), 0, 32, s));
  void* ttmp = scratch<unsigned char>(static_cast<int64_t>(tbytes), s);
  for (int l = d - 1; l >= 0 && nnz > 0; --l) {
    k_gather_keys<<<nb(nnz, 256), 256, 0, s>>>(co, l, perm, nnz, key);
    SPTTN_CUDA(cub::DeviceRadixSort::SortPairs(ttmp, tbytes, key, key2, perm, perm2,
                                               static_cast<int>(nnz), 0, bits_for(dims[l]), s));
    std::swap(perm, perm2);
  }
  dfree(ttmp, s);
  // 2. distinct rows, duplicates summed in order
  int32_t* head = scratch<int32_t>(nnz, s);
  int32_t* run_id = scratch<int32_t>(nnz, s);
  int32_t nu = 0;
  if (nnz > 0) {
    k_run_heads<<<nb(nnz, 256), 256, 0, s>>>(co, d, perm, nnz, head);
    scan_incl_sum(head, run_id, nnz, s);
    SPTTN_CUDA(cudaMemcpyAsync(&nu, run_id + nnz - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    SPTTN_CUDA(cudaStreamSynchronize(s));
  }
  int32_t* urow = scratch<int32_t>(nu, s);
  dmalloc(&D.vals, static_cast<size_t>(std::max<int32_t>(1, nu)) * sizeof(double), s);
  if (nnz > 0)
    k_merge_runs<<<nb(nnz, 256), 256, 0, s>>>(head, run_id, perm, vals, nnz, urow, D.vals);
  // 3. levels, root first (node ids of level l+1 are needed for ptr[l])
  std::vector<int32_t*> flag(d), nid(d);
  std::vector<int32_t> count(d, 0);
  for (int l = 0; l < d; ++l) {
    flag[l] = scratch<int32_t>(nu, s);
    nid[l] = scratch<int32_t>(nu, s);
    if (nu > 0) {
      k_node_flags<<<nb(nu, 256), 256, 0, s>>>(co, l, urow, nu, flag[l]);
      scan_incl_sum(flag[l], nid[l], nu, s);
      SPTTN_CUDA(cudaMemcpyAsync(&count[l], nid[l] + nu - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    }
  }
  SPTTN_CUDA(cudaStreamSynchronize(s));
  D.bytes = static_cast<int64_t>(nu) * 8;
  for (int l = 0; l < d; ++l) {
    D.level_size[l] = count[l];
    dmalloc(&D.idx[l], static_cast<size_t>(std::max<int32_t>(1, count[l])) * sizeof(int32_t), s);
    D.bytes += static_cast<int64_t>(count[l]) * 4;
    if (l + 1 < d) {
      dmalloc(&D.ptr[l], (static_cast<size_t>(count[l]) + 1) * sizeof(int32_t), s);
      D.bytes += (static_cast<int64_t>(count[l]) + 1) * 4;
      // sentinel: the child level's node count
      SPTTN_CUDA(cudaMemcpyAsync(D.ptr[l] + count[l], &count[l + 1], sizeof(int32_t),
                                 cudaMemcpyHostToDevice, s));
    }
    if (nu > 0)
      k_emit_level<<<nb(nu, 256), 256, 0, s>>>(co, l, urow, flag[l], nid[l],
                                               l + 1 < d ? nid[l + 1] : nullptr, nu, D.idx[l],
                                               l + 1 < d ? D.ptr[l] : nullptr);
  }
  SPTTN_CUDA(cudaStreamSynchronize(s));  // the sentinel sources live on this stack
  for (int l = 0; l < d; ++l) {
    dfree(flag[l], s);
    dfree(nid[l], s);
  }
  for (void* p : {static_cast<void*>(key), static_cast<void*>(key2), static_cast<void*>(perm),
                  static_cast<void*>(perm2), static_cast<void*>(head), static_cast<void*>(run_id),
                  static_cast<void*>(urow)})
    dfree(p, s);
  SPTTN_CUDA(cudaGetLastError());
}

}  // namespace

void csf_from_coo(DevCsf& D, int d, const int64_t* dims, int64_t nnz, const int64_t* h_coords,
                  const double* h_vals, cudaStream_t s) {
  if (nnz >= INT32_MAX) throw Status(SPTTN_EINVAL, "COO exceeds the int32 device layout");
  for (int l = 0; l < d; ++l)
    if (dims[l] < 1 || dims[l] > INT32_MAX) throw Status(SPTTN_EINVAL, "mode size must be in [1, 2^31)");
  int64_t* coords = scratch<int64_t>(nnz * d, s);
  double* vals = scratch<double>(nnz, s);
  int* err = scratch<int>(1, s);
  SPTTN_CUDA(cudaMemsetAsync(err, 0, sizeof(int), s));
  if (nnz > 0) {
    SPTTN_CUDA(cudaMemcpyAsync(coords, h_coords, nnz * d * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    SPTTN_CUDA(cudaMemcpyAsync(vals, h_vals, nnz * sizeof(double), cudaMemcpyHostToDevice, s));
  }
  uint32_t* key = scratch<uint32_t>(nnz, s);
  for (int l = 0; l < d && nnz > 0; ++l)  // bounds check
    k_level_keys<<<nb(nnz, 256), 256, 0, s>>>(coords, nnz, d, l, dims[l], key, err);
  int herr = 0;
  SPTTN_CUDA(cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, s));
  SPTTN_CUDA(cudaStreamSynchronize(s));
  dfree(key, s);
  dfree(err, s);
  if (herr) {
    dfree(coords, s);
    dfree(vals, s);
    throw Status(SPTTN_EINVAL, "COO coordinate out of bounds");
  }
  Soa co{};
  std::vector<int32_t*> cols(d);
  for (int l = 0; l < d; ++l) {
    cols[l] = scratch<int32_t>(nnz, s);
    co.c[l] = cols[l];
  }
  if (nnz > 0) k_aos_to_soa<<<nb(nnz, 256), 256, 0, s>>>(coords, nnz, d, co);
  dfree(coords, s);
  build_from_soa(D, d, dims, nnz, co, vals, s);
  for (int l = 0; l < d; ++l) dfree(cols[l], s);
  dfree(vals, s);
}

void csf_permute(const DevCsf& src, const int* order, DevCsf& D, cudaStream_t s) {
  src.wait_values(s);
  const int d = src.order;
  const int64_t nnz = src.level_size[d - 1];
  // every leaf's coordinate at every level (parents broadcast downwards)
  std::vector<int32_t*> leafc(d, nullptr);
  for (int l = 0; l < d; ++l) {
    if (l == d - 1) {
      leafc[l] = src.idx[l];
      continue;
    }
    int32_t* cur = nullptr;  // coordinate of level l at the nodes of level m
    for (int m = l + 1; m < d; ++m) {
      int32_t* next = scratch<int32_t>(src.level_size[m], s);
      if (src.level_size[m] > 0)
        k_expand_parent<<<nb(src.level_size[m], 256), 256, 0, s>>>(
            src.ptr[m - 1], static_cast<int32_t>(src.level_size[m - 1]), m == l + 1 ? src.idx[l] : cur,
            src.level_size[m], next);
      if (cur) dfree(cur, s);
      cur = next;
    }
    leafc[l] = cur;
  }
  Soa co{};
  int64_t dims[kMaxOrder];
  for (int l = 0; l < d; ++l) {
    co.c[l] = leafc[order[l]];
    dims[l] = src.dims[order[l]];
  }
  build_from_soa(D, d, dims, nnz, co, src.vals, s);
  for (int l = 0; l + 1 < d; ++l) dfree(leafc[l], s);
}

void csf_download(const DevCsf& D, int64_t* const* idx, int64_t* const* ptr, double* values,
                  cudaStream_t s) {
  D.wait_values(s);
  int64_t maxn = 1;
  for (int l = 0; l < D.order; ++l) maxn = std::max(maxn, D.level_size[l] + 1);
  int64_t* wide = scratch<int64_t>(maxn, s);
  auto one = [&](const int32_t* src, int64_t n, int64_t* dst) {
    if (n == 0 || !dst) return;
    k_widen<<<nb(n, 256), 256, 0, s>>>(src, n, wide);
    SPTTN_CUDA(cudaMemcpyAsync(dst, wide, n * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    SPTTN_CUDA(cudaStreamSynchronize(s));  // `wide` is reused by the next array
  };
  for (int l = 0; l < D.order; ++l) {
    one(D.idx[l], D.level_size[l], idx ? idx[l] : nullptr);
    if (l + 1 < D.order) one(D.ptr[l], D.level_size[l] + 1, ptr ? ptr[l] : nullptr);
  }
  const int64_t nnz = D.level_size[D.order - 1];
  if (values && nnz > 0)
    SPTTN_CUDA(cudaMemcpyAsync(values, D.vals, nnz * sizeof(double), cudaMemcpyDeviceToHost, s));
  SPTTN_CUDA(cudaStreamSynchronize(s));
  dfree(wide, s);
}

}  // namespace spttn_dev
