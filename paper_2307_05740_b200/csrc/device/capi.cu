// C-ABI implementation (include/spttn_b200.h): device CSF construction,
// plan creation (nest-shape -> kernel, device allocation, work
// decomposition) and execution. Mirrors the reference executor's contract
// (proj/src/executor.cpp:112-200 for validation and errors, :492-520 for
// execute) with CUDA status codes mapped to the reference exception types.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../../include/spttn_b200.h"
#include "internal.cuh"

using spttn_dev::Status;

struct spttn_csf {
  spttn_dev::DevCsf d;
};

struct spttn_plan {
  int kind = 0;
  int flags = 0;
  int64_t R = 0, S = 0, T = 0;
  spttn_csf* csf = nullptr;
  int nf = 0;
  double* fac[8] = {nullptr};
  int64_t fac_size[8] = {0};
  bool own_fac = true;
  double* out = nullptr;
  int64_t out_count = 0;
  int vec = 0;
  int mode = 0;  // kernel variant (TTMc-3, TTTP-3)
  int batch = 4;  // TTTP leaves per group step
  int32_t* leaf_i = nullptr;  // TTTP leaf kernel: per-leaf root / level-1 coordinates
  int32_t* leaf_j = nullptr;
  int4* pieces = nullptr;  // TTTP mode 3: slice pieces {i, leaf lo, leaf hi}
  int64_t n_pieces = 0;
  int2* leaf_jk = nullptr;  // TTTP mode 3: per-leaf {j, k}
  spttn_dev::Decomp dec;
  // non-root MTTKRP-3 mode 5: the tensor re-ordered so the output mode is
  // the root (owned by the plan; the kernels run on it instead of csf)
  spttn_dev::DevCsf* tcsf = nullptr;
  spttn_dev::GenericState gen;
  spg_program* prog = nullptr;  // host copy (GENERIC)
  const double** d_dense = nullptr;
  int64_t launches = 0;
  int64_t last_madds = -1;
  int fac_align = 8;  // factor alignment the plan's kernels were chosen for
  void* arena = nullptr;                // GENERIC: one allocation for all plan state
  std::vector<int64_t> last_counters;   // GENERIC: madds, resets, log cursor, overflow
  long long* item_clk = nullptr;        // diagnostics: per item {start, end, smid}
};

static void free_tcsf(spttn_plan* p) {
  if (!p->tcsf) return;
  for (int l = 0; l < p->tcsf->order; ++l) {
    spttn_dev::dfree(p->tcsf->idx[l]);
    spttn_dev::dfree(p->tcsf->ptr[l]);
  }
  spttn_dev::dfree(p->tcsf->vals);
  delete p->tcsf;
  p->tcsf = nullptr;
}


namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return SPTTN_OK;
  } catch (const Status& s) {
    g_err = s.what();
    return s.code;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return SPTTN_ENOMEM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return SPTTN_EINVAL;
  }
}

void fail(int code, const std::string& msg) { throw Status(code, msg); }

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// all device memory comes from the engine's pool (mem.cu)
void dev_malloc(void** p, size_t bytes, cudaStream_t s) { spttn_dev::dmalloc_raw(p, bytes, s); }

// int64 -> int32 narrowing with range / monotonicity checks.
// `base` rebases child pointers of a tree view (ptr[l][0] != 0).
__global__ void k_narrow(const int64_t* src, int32_t* dst, int64_t n, int64_t limit,
                         int monotone, int64_t base, int* err) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t v = src[i] - base;
  if (v < 0 || v >= limit) atomicOr(err, 1);
  if (monotone && i + 1 < n && src[i + 1] - base < v) atomicOr(err, 2);
  dst[i] = static_cast<int32_t>(v);
}

// Packed leaf keys for sparse-output lookups (executor.cpp:342-366); the CSF
// is lexicographic, so the keys come out sorted with leaf_pos = identity.
__global__ void k_leaf_keys(spttn_dev::CsfView t, const spg_program* P, int64_t* keys,
                            int64_t* pos) {
  const int64_t leaf = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int d = t.order;
  if (leaf >= t.nlev[d - 1]) return;
  int64_t node = leaf, key = 0;
  for (int l = d - 1; l >= 0; --l) {
    key += static_cast<int64_t>(t.idx[l][node]) * P->mode_key_stride[l];
    if (l > 0) {
      int64_t lo = 0, hi = t.nlev[l - 1];
      while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (t.ptr[l - 1][mid] <= node) lo = mid; else hi = mid;
      }
      node = lo;
    }
  }
  keys[leaf] = key;
  pos[leaf] = leaf;
}

int64_t env_int(const char* name, int64_t dflt) {
  const char* v = std::getenv(name);
  return v && *v ? std::atoll(v) : dflt;
}

int sm_count() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

int smem_optin_bytes() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&n, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  return n;
}

void copy_factors(spttn_plan* p, const double* const* src, bool on_device, cudaStream_t s) {
  auto& g = p->gen;
  if (g.parcel && !on_device) {  // small GENERIC plan: one upload from the pinned parcel
    SPTTN_CUDA(cudaEventSynchronize(g.up_done));  // the previous upload has left the parcel
    for (int f = 0; f < p->nf; ++f)
      if (p->fac_size[f] > 0) std::memcpy(g.parcel + g.fac_off[f], src[f], p->fac_size[f] * 8);
    if (g.up_end > g.up_fac)
      SPTTN_CUDA(cudaMemcpyAsync(static_cast<unsigned char*>(p->arena) + g.up_fac,
                                 g.parcel + g.up_fac, g.up_end - g.up_fac,
                                 cudaMemcpyHostToDevice, s));
    SPTTN_CUDA(cudaEventRecord(g.up_done, s));
    return;
  }
  for (int f = 0; f < p->nf; ++f) {
    if (on_device) {
      p->fac[f] = const_cast<double*>(src[f]);
    } else {
      if (!p->fac[f]) dev_malloc(reinterpret_cast<void**>(&p->fac[f]), p->fac_size[f] * sizeof(double), s);
      if (p->fac_size[f] > 0)
        SPTTN_CUDA(cudaMemcpyAsync(p->fac[f], src[f], p->fac_size[f] * sizeof(double),
                                   cudaMemcpyHostToDevice, s));
    }
  }
}

}  // namespace

namespace spttn_dev {
// make `s` wait for a pending packed-stream fill (no-op when none)
inline void csf_wait_fill(cudaEvent_t fill_done, cudaStream_t s) {
  if (fill_done) SPTTN_CUDA(cudaStreamWaitEvent(s, fill_done, 0));
}
}  // namespace spttn_dev

// side stream per device for plan-time work that overlaps an asynchronous
// values upload (build_packed's leaf-stream fill)
cudaStream_t spttn_dev::aux_stream() {
  static std::mutex mu;
  static cudaStream_t st[64] = {};
  int dev = 0;
  SPTTN_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  if (dev < 0 || dev >= 64) throw spttn_dev::Status(SPTTN_ECUDA, "device ordinal out of range");
  if (!st[dev]) SPTTN_CUDA(cudaStreamCreateWithFlags(&st[dev], cudaStreamNonBlocking));
  return st[dev];
}

extern "C" {

const char* spttn_last_error(void) { return g_err.c_str(); }

int spttn_release_cached(void) {
  return guarded([] {
    SPTTN_CUDA(cudaDeviceSynchronize());
    spttn_dev::release_cached();
  });
}

#define SPTTN_STR2(x) #x
#define SPTTN_STR(x) SPTTN_STR2(x)
const char* spttn_build_info(void) {
  return "spttn_b200 sm_100a nvcc " SPTTN_STR(__CUDACC_VER_MAJOR__) "." SPTTN_STR(__CUDACC_VER_MINOR__);
}

int spttn_init(void) {
  return guarded([] {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
      cudaGetLastError();
      fail(SPTTN_ECUDA, "no CUDA device");
    }
    SPTTN_CUDA(cudaFree(nullptr));  // creates the primary context
    void* p = nullptr;              // and touches the allocator (first cudaMalloc)
    spttn_dev::dmalloc_raw(&p, 256, nullptr);
    SPTTN_CUDA(cudaStreamSynchronize(nullptr));
    spttn_dev::dfree(p);
  });
}

int spttn_synchronize(void* stream) {
  return guarded([&] {
    if (stream) SPTTN_CUDA(cudaStreamSynchronize(as_stream(stream)));
    else SPTTN_CUDA(cudaDeviceSynchronize());
  });
}

int spttn_device_info(int64_t* out, int n) {
  return guarded([&] {
    int dev = 0;
    SPTTN_CUDA(cudaGetDevice(&dev));
    cudaDeviceProp pr{};
    SPTTN_CUDA(cudaGetDeviceProperties(&pr, dev));
    const int64_t v[4] = {pr.multiProcessorCount, pr.major * 10 + pr.minor, pr.l2CacheSize,
                          static_cast<int64_t>(pr.sharedMemPerBlockOptin)};
    for (int i = 0; i < n && i < 4; ++i) out[i] = v[i];
  });
}

int spttn_csf_from_coo(int order, const int64_t* dims, int64_t nnz, const int64_t* coords,
                       const double* values, void* stream, spttn_csf** out) {
  return guarded([&] {
    if (!dims || !out || (nnz > 0 && (!coords || !values)))
      fail(SPTTN_EINVAL, "spttn_csf_from_coo: null argument");
    if (nnz < 0) fail(SPTTN_EINVAL, "spttn_csf_from_coo: negative nnz");
    *out = nullptr;
    if (order < 1 || order > spttn_dev::kMaxOrder) fail(SPTTN_EINVAL, "CSF order must be 1..8");
    auto c = std::make_unique<spttn_csf>();
    SPTTN_CUDA(cudaGetDevice(&c->d.device));
    spttn_dev::csf_from_coo(c->d, order, dims, nnz, coords, values, as_stream(stream));
    *out = c.release();
  });
}

int spttn_csf_permute(const spttn_csf* src, const int* order, void* stream, spttn_csf** out) {
  return guarded([&] {
    if (!src || !order || !out) fail(SPTTN_EINVAL, "spttn_csf_permute: null argument");
    *out = nullptr;
    const int d = src->d.order;
    bool seen[spttn_dev::kMaxOrder] = {false};
    for (int l = 0; l < d; ++l) {
      if (order[l] < 0 || order[l] >= d || seen[order[l]])
        fail(SPTTN_EINVAL, "spttn_csf_permute: order is not a permutation of the levels");
      seen[order[l]] = true;
    }
    auto c = std::make_unique<spttn_csf>();
    SPTTN_CUDA(cudaGetDevice(&c->d.device));
    spttn_dev::csf_permute(src->d, order, c->d, as_stream(stream));
    *out = c.release();
  });
}

int spttn_csf_download(const spttn_csf* c, int64_t* const* idx, int64_t* const* ptr,
                       double* values, void* stream) {
  return guarded([&] {
    if (!c) fail(SPTTN_EINVAL, "spttn_csf_download: null CSF");
    spttn_dev::csf_download(c->d, idx, ptr, values, as_stream(stream));
  });
}

int64_t spttn_csf_dim(const spttn_csf* c, int l) {
  return (c && l >= 0 && l < c->d.order) ? c->d.dims[l] : -1;
}

namespace {
// side stream per device for the asynchronous leaf-value upload
cudaStream_t values_stream() {
  static std::mutex mu;
  static cudaStream_t st[64] = {};
  int dev = 0;
  SPTTN_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  if (dev < 0 || dev >= 64) throw spttn_dev::Status(SPTTN_ECUDA, "device ordinal out of range");
  if (!st[dev]) SPTTN_CUDA(cudaStreamCreateWithFlags(&st[dev], cudaStreamNonBlocking));
  return st[dev];
}

int csf_create(const spttn_csf_host* h, void* stream, spttn_csf** out, bool async_values);
}  // namespace

int spttn_csf_create(const spttn_csf_host* h, void* stream, spttn_csf** out) {
  return csf_create(h, stream, out, false);
}

int spttn_csf_create_async(const spttn_csf_host* h, void* stream, spttn_csf** out) {
  return csf_create(h, stream, out, true);
}

namespace {
int csf_create(const spttn_csf_host* h, void* stream, spttn_csf** out, bool async_values) {
  return guarded([&] {
    if (!h || !out) fail(SPTTN_EINVAL, "spttn_csf_create: null argument");
    *out = nullptr;
    const int d = h->order;
    if (d < 1 || d > spttn_dev::kMaxOrder) fail(SPTTN_EINVAL, "CSF order must be 1..8");
    auto c = std::make_unique<spttn_csf>();
    auto& D = c->d;
    D.order = d;
    SPTTN_CUDA(cudaGetDevice(&D.device));
    cudaStream_t s = as_stream(stream);
    int64_t maxn = 1;
    for (int l = 0; l < d; ++l) {
      D.dims[l] = h->dims[l];
      D.level_size[l] = h->level_size[l];
      if (h->dims[l] < 1 || h->dims[l] > INT32_MAX)
        fail(SPTTN_EINVAL, "CSF mode size must be in [1, 2^31)");
      if (h->level_size[l] < 0 || h->level_size[l] >= INT32_MAX)
        fail(SPTTN_EINVAL, "CSF level size exceeds the int32 device layout");
      if (l > 0 && h->level_size[l] < h->level_size[l - 1])
        fail(SPTTN_EINVAL, "CSF level sizes must be non-decreasing");
      maxn = std::max(maxn, h->level_size[l] + 1);
    }
    for (int l = 0; l + 1 < d; ++l) {  // views of a larger tree are rebased
      const int64_t n = h->level_size[l];
      if (h->ptr[l][n] - h->ptr[l][0] != h->level_size[l + 1])
        fail(SPTTN_EINVAL, "CSF ptr[" + std::to_string(l) + "] does not close its child range");
    }
    int64_t* stage = nullptr;
    int* err = nullptr;
    dev_malloc(reinterpret_cast<void**>(&stage), maxn * sizeof(int64_t), s);
    dev_malloc(reinterpret_cast<void**>(&err), sizeof(int), s);
    SPTTN_CUDA(cudaMemsetAsync(err, 0, sizeof(int), s));
    auto narrow = [&](const int64_t* src, int32_t** dst, int64_t n, int64_t limit, int mono,
                      int64_t base) {
      dev_malloc(reinterpret_cast<void**>(dst), std::max<int64_t>(1, n) * sizeof(int32_t), s);
      D.bytes += n * sizeof(int32_t);
      if (n == 0) return;
      SPTTN_CUDA(cudaMemcpyAsync(stage, src, n * sizeof(int64_t), cudaMemcpyHostToDevice, s));
      k_narrow<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(stage, *dst, n, limit, mono,
                                                                       base, err);
      SPTTN_CUDA(cudaGetLastError());
    };
    try {
      for (int l = 0; l < d; ++l) {
        narrow(h->idx[l], &D.idx[l], h->level_size[l], h->dims[l], 0, 0);
        if (l + 1 < d)
          narrow(h->ptr[l], &D.ptr[l], h->level_size[l] + 1, h->level_size[l + 1] + 1, 1,
                 h->level_size[l] >= 0 ? h->ptr[l][0] : 0);
      }
      const int64_t nnz = h->level_size[d - 1];
      dev_malloc(reinterpret_cast<void**>(&D.vals), std::max<int64_t>(1, nnz) * sizeof(double), s);
      D.bytes += nnz * sizeof(double);
      if (async_values) {
        // the values go up on a side stream while the caller builds plans
        // (whose structure work needs only idx / ptr); consumers of D.vals
        // wait on D.vals_ready (DevCsf::wait_values)
        cudaStream_t vs = values_stream();
        cudaEvent_t alloc_done = nullptr;
        SPTTN_CUDA(cudaEventCreateWithFlags(&alloc_done, cudaEventDisableTiming));
        SPTTN_CUDA(cudaEventRecord(alloc_done, s));
        SPTTN_CUDA(cudaStreamWaitEvent(vs, alloc_done, 0));
        SPTTN_CUDA(cudaEventDestroy(alloc_done));
        if (nnz > 0)
          SPTTN_CUDA(cudaMemcpyAsync(D.vals, h->values, nnz * sizeof(double),
                                     cudaMemcpyHostToDevice, vs));
        SPTTN_CUDA(cudaEventCreateWithFlags(&D.vals_ready, cudaEventDisableTiming));
        SPTTN_CUDA(cudaEventRecord(D.vals_ready, vs));
      } else if (nnz > 0) {
        SPTTN_CUDA(cudaMemcpyAsync(D.vals, h->values, nnz * sizeof(double),
                                   cudaMemcpyHostToDevice, s));
      }
      int herr = 0;
      SPTTN_CUDA(cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, s));
      SPTTN_CUDA(cudaStreamSynchronize(s));
      if (herr & 1) fail(SPTTN_EINVAL, "CSF coordinate or child pointer out of range");
      if (herr & 2) fail(SPTTN_EINVAL, "CSF child pointers are not monotone");
    } catch (...) {
      spttn_dev::dfree(stage, s);
      spttn_dev::dfree(err, s);
      for (int l = 0; l < d; ++l) {
        spttn_dev::dfree(D.idx[l], s);
        spttn_dev::dfree(D.ptr[l], s);
      }
      spttn_dev::dfree(D.vals, s);
      throw;
    }
    spttn_dev::dfree(stage, s);
    spttn_dev::dfree(err, s);
    *out = c.release();
  });
}
}  // namespace

int spttn_csf_destroy(spttn_csf* c) {
  return guarded([&] {
    if (!c) return;
    cudaDeviceSynchronize();  // as cudaFree would: no kernel may still read it
    for (int l = 0; l < c->d.order; ++l) {
      spttn_dev::dfree(c->d.idx[l]);
      spttn_dev::dfree(c->d.ptr[l]);
    }
    spttn_dev::dfree(c->d.vals);
    if (c->d.vals_ready) cudaEventDestroy(c->d.vals_ready);
    delete c;
  });
}

int64_t spttn_csf_level_size(const spttn_csf* c, int l) {
  return (c && l >= 0 && l < c->d.order) ? c->d.level_size[l] : -1;
}

int64_t spttn_csf_device_bytes(const spttn_csf* c) { return c ? c->d.bytes : -1; }

int spttn_plan_destroy(spttn_plan* p) {
  return guarded([&] {
    if (!p) return;
    cudaDeviceSynchronize();  // as cudaFree would: no kernel may still use it
    if (p->arena) {  // GENERIC: everything lives in the arena
      if (p->gen.up_done) cudaEventDestroy(p->gen.up_done);
      spttn_dev::pinned_free(p->gen.parcel, p->gen.parcel_bytes);
      spttn_dev::dfree(p->arena);
      spttn_dev::free_decomp(p->dec);
      delete p->prog;
      delete p;
      return;
    }
    if (p->own_fac)
      for (int f = 0; f < p->nf; ++f) spttn_dev::dfree(p->fac[f]);
    spttn_dev::dfree(p->out);
    spttn_dev::dfree(p->item_clk);
    spttn_dev::dfree(p->d_dense);
    spttn_dev::dfree(p->leaf_i);
    spttn_dev::dfree(p->leaf_j);
    spttn_dev::dfree(p->pieces);
    spttn_dev::dfree(p->leaf_jk);
    spttn_dev::free_decomp(p->dec);
    free_tcsf(p);
    spttn_dev::generic_free(p->gen);
    delete p->prog;
    delete p;
  });
}

namespace {

// k_mttkrp3_smf work split: cut the packed group sequence into one range per
// CTA at root-slice boundaries, balanced by groups. False when a slice is too
// heavy for that (Zipf hubs): the plan then uses the item / fix-up kernels.
bool smf_ranges(spttn_plan* p, const spttn_dev::DevCsf& D, int sms, int64_t tile, cudaStream_t s) {
  auto& d = p->dec;
  const int nq = static_cast<int>(p->R / 16);
  const int nc = std::max(1, sms / nq);
  const int64_t n0 = D.level_size[0];
  const int64_t G = d.n_groups;
  std::vector<int32_t> sg(n0 + 1, 0);
  SPTTN_CUDA(cudaMemcpyAsync(sg.data(), d.slice_grp, (n0 + 1) * sizeof(int32_t),
                             cudaMemcpyDeviceToHost, s));
  SPTTN_CUDA(cudaStreamSynchronize(s));
  std::vector<int32_t> cg(nc + 1, 0);
  cg[nc] = static_cast<int32_t>(G);
  int64_t widest = 0;
  for (int c = 1; c < nc; ++c) {
    const int64_t target = G * c / nc;
    const auto it = std::lower_bound(sg.begin(), sg.end(), static_cast<int32_t>(target));
    cg[c] = std::max(cg[c - 1], it == sg.end() ? static_cast<int32_t>(G) : *it);
  }
  for (int c = 0; c < nc; ++c) widest = std::max<int64_t>(widest, cg[c + 1] - cg[c]);
  const int64_t fair = (G + nc - 1) / nc;
  if (env_int("SPTTN_SMF_FORCE", 0) == 0 && G > 0 && widest > fair + fair / 4 + 64) return false;
  // absent root rows (zeroed by the kernel); one item, so no split slices
  spttn_dev::finish_unit_items(D, d, d.slice_grp, G, std::max<int64_t>(1, G), tile, s);
  d.n_cta = nc;
  spttn_dev::dmalloc(&d.cta_grp, (nc + 1) * sizeof(int32_t), s);
  SPTTN_CUDA(cudaMemcpyAsync(d.cta_grp, cg.data(), (nc + 1) * sizeof(int32_t),
                             cudaMemcpyHostToDevice, s));
  SPTTN_CUDA(cudaStreamSynchronize(s));
  return true;
}

}  // namespace

int spttn_plan_create(const spttn_plan_desc* desc, spttn_csf* csf, void* stream,
                      spttn_plan** out) {
  spttn_plan* raw = nullptr;
  const int rc = guarded([&] {
    if (!desc || !csf || !out) fail(SPTTN_EINVAL, "spttn_plan_create: null argument");
    *out = nullptr;
    cudaStream_t s = as_stream(stream);
    auto p = new spttn_plan;
    raw = p;
    cudaEvent_t fill_done = nullptr;  // packed-stream fill on the side stream (build_packed)
    const auto& D = csf->d;
    p->kind = desc->kind;
    p->flags = desc->flags;
    p->R = desc->rank[0];
    p->S = desc->rank[1];
    p->T = desc->rank[2];
    p->csf = csf;
    p->nf = desc->num_factors;
    if (p->nf < 0 || p->nf > 8) fail(SPTTN_EINVAL, "num_factors must be 0..8");
    for (int f = 0; f < p->nf; ++f) p->fac_size[f] = desc->factor_size[f];
    const bool on_dev = (desc->flags & SPTTN_FLAG_FACTORS_ON_DEVICE) != 0;
    p->own_fac = !on_dev;
    const int64_t nnz = D.level_size[D.order - 1];

    auto need = [&](int order, int nf, std::initializer_list<int64_t> sizes) {
      if (D.order != order)
        fail(SPTTN_EINVAL, "sparse tensor order mismatch for this nest");
      if (p->nf != nf) fail(SPTTN_EINVAL, "wrong number of dense inputs for this nest");
      int f = 0;
      for (int64_t sz : sizes) {
        if (p->fac_size[f] != sz) fail(SPTTN_EINVAL, "dense tensor shape mismatch");
        ++f;
      }
    };
    const int64_t R = p->R, S = p->S, T = p->T;
    int64_t tile = 0;
    switch (p->kind) {
      case SPTTN_NEST_MTTKRP3:
        need(3, 2, {D.dims[1] * R, D.dims[2] * R});
        if (R < 1 || R > 128) fail(SPTTN_EUNSUPPORTED, "MTTKRP kernel supports 1 <= R <= 128");
        tile = R;
        break;
      case SPTTN_NEST_MTTKRP3_J:  // factors A[i,r], C[k,r]; output B[j,r]
        need(3, 2, {D.dims[0] * R, D.dims[2] * R});
        if (R < 1 || R > 32) fail(SPTTN_EUNSUPPORTED, "non-root MTTKRP kernel supports 1 <= R <= 32");
        tile = R;
        break;
      case SPTTN_NEST_MTTKRP3_K:  // factors A[i,r], B[j,r]; output C[k,r]
        need(3, 2, {D.dims[0] * R, D.dims[1] * R});
        if (R < 1 || R > 32) fail(SPTTN_EUNSUPPORTED, "non-root MTTKRP kernel supports 1 <= R <= 32");
        tile = R;
        break;
      case SPTTN_NEST_MTTKRP4:
        need(4, 3, {D.dims[1] * R, D.dims[2] * R, D.dims[3] * R});
        if (R < 1 || R > 128) fail(SPTTN_EUNSUPPORTED, "MTTKRP kernel supports 1 <= R <= 128");
        tile = R;
        break;
      case SPTTN_NEST_TTTP3:
        need(3, 3, {D.dims[0] * R, D.dims[1] * R, D.dims[2] * R});
        if (R < 1 || R > 128) fail(SPTTN_EUNSUPPORTED, "TTTP kernel supports 1 <= R <= 128");
        break;
      case SPTTN_NEST_TTMC3:
        need(3, 2, {D.dims[1] * R, D.dims[2] * S});
        if (R < 1 || R > 16 || S < 1 || S > 16)
          fail(SPTTN_EUNSUPPORTED, "TTMc-3 DMMA kernel supports R, S <= 16");
        tile = R * S;
        break;
      case SPTTN_NEST_TTMC4:
        need(4, 3, {D.dims[1] * R, D.dims[2] * S, D.dims[3] * T});
        if (R < 1 || R > 8 || S < 1 || S > 8 || T < 1 || T > 8)
          fail(SPTTN_EUNSUPPORTED, "TTMc-4 DMMA kernel supports R, S, T <= 8");
        tile = R * S * T;
        break;
      case SPTTN_NEST_GENERIC: {
        if (!desc->program || desc->program_bytes != static_cast<int64_t>(sizeof(spg_program)))
          fail(SPTTN_EINVAL, "GENERIC plan needs a spg_program");
        p->prog = new spg_program;
        std::memcpy(p->prog, desc->program, sizeof(spg_program));
        if (p->prog->magic != SPG_MAGIC) fail(SPTTN_EINVAL, "bad program magic");
        if (p->prog->csf_order != D.order) fail(SPTTN_EINVAL, "sparse tensor order mismatch");
        for (int f = 0; f < p->nf; ++f)
          if (p->fac_size[f] != p->prog->dense_size[f + 1])
            fail(SPTTN_EINVAL, "dense tensor shape mismatch");
        int64_t bytes = 0;
        for (int b = 0; b < p->prog->num_buffers; ++b) bytes += p->prog->buffer_size[b] * 8;
        if (bytes > desc->buffer_limit_bytes)
          fail(SPTTN_ENOMEM, "intermediate buffers exceed the buffer byte limit");
        break;
      }
      default:
        fail(SPTTN_EINVAL, "unknown nest kind " + std::to_string(p->kind));
    }

    if (p->kind == SPTTN_NEST_GENERIC) {
      // One device arena per interpreter plan (tiny plans are dominated by
      // allocation cost): [counters | buffers | out] (zeroed by one memset
      // per execute), program, buffer offsets, dense pointer table, factor
      // copies, observer log, leaf keys.
      const spg_program& G = *p->prog;
      const int nb = G.num_buffers;
      std::vector<int64_t> off(nb + 1, 0);
      for (int b = 0; b < nb; ++b) off[b + 1] = off[b] + G.buffer_size[b];
      auto al = [](size_t x) { return (x + 255) & ~size_t{255}; };
      // Parallel interpretation over root slices (generic.cu k_generic_par)
      // when the single root is the CSF level-0 loop without resets of its
      // own; outputs indexed by the root mode (or sparse) are written
      // directly (mode 1), any other dense output goes through per-worker
      // copies reduced in worker order (mode 2). Replicas are capped at
      // 512 MB. SPTTN_GENERIC_PAR=0 forces the sequential walk.
      auto& g = p->gen;
      // Specialised kernel for this forest (jit.cu) when the tensor is large
      // enough to amortise an NVRTC compile (cached per distinct nest):
      // SPTTN_GENERIC_JIT=1 always, 0 never, default from 65536 nonzeros.
      const int64_t jit_env = env_int("SPTTN_GENERIC_JIT", -1);
      const bool want_jit = !G.observe && spttn_dev::jit_available() &&
                            (jit_env == 1 || (jit_env < 0 && nnz >= (int64_t{1} << 16)));
      {
        const int64_t n0 = D.level_size[0];
        const spg_node* rootn = G.num_roots == 1 ? &G.nodes[G.roots[0]] : nullptr;
        const bool par_ok = env_int("SPTTN_GENERIC_PAR", 1) != 0 && !G.observe && rootn &&
                            rootn->kind == SPG_SPARSE && rootn->csf_level == 0 &&
                            rootn->reset_count == 0 && n0 >= 2;
        if (par_ok) {
          bool disjoint = true;
          for (int t = 0; t < G.num_terms; ++t) {
            const spg_access& o = G.out[t];
            if (o.kind != SPG_OP_OUT_DENSE) continue;
            bool has_root = false;
            for (int k = 0; k < o.naddr; ++k)
              has_root |= o.ids[k] == rootn->index && o.strides[k] != 0;
            disjoint &= has_root;
          }
          const int64_t budget = int64_t{512} << 20;
          const int64_t per_buf = std::max<int64_t>(8, off[nb] * 8);
          const int64_t per_out = disjoint ? 0 : std::max<int64_t>(8, G.out_size * 8);
          int64_t W = std::min<int64_t>(n0, static_cast<int64_t>(sm_count()) * (disjoint ? 128 : 32));
          W = std::min<int64_t>(W, budget / (per_buf + per_out));
          if (W >= 2) {
            g.par_mode = disjoint ? 1 : 2;
            g.workers = W;
            g.out_size = G.out_size;
            g.priv = !disjoint;
          }
        }
        // The JIT kernel admits more decompositions (jit.cu jit_analyze):
        // level-1 fibers as work units (few heavy root slices), and forests
        // whose root loop accumulates into buffers reset once before it and
        // consumed by later roots (TTTc-like chains): per-worker
        // accumulators summed in worker order, then the later roots.
        if (want_jit && env_int("SPTTN_GENERIC_PAR", 1) != 0 && n0 >= 2) {
          const spttn_dev::JitSplit js = spttn_dev::jit_analyze(G);
          const int64_t n1 = D.order > 1 ? D.level_size[1] : 0;
          const bool fiber = js.ok && js.fiber_ok && n1 >= 4 * n0;
          if (js.ok && (js.tail || fiber)) {
            const bool disjoint = fiber ? js.disjoint_fiber : js.disjoint_slice;
            const bool priv = js.writes_out && !disjoint;
            const int64_t budget = int64_t{512} << 20;
            const int64_t per = std::max<int64_t>(8, off[nb] * 8) +
                                (priv ? std::max<int64_t>(8, G.out_size * 8) : 0);
            int64_t W = fiber ? std::min<int64_t>(n1, static_cast<int64_t>(sm_count()) * 64)
                              : std::min<int64_t>(n0, static_cast<int64_t>(sm_count()) * 32);
            W = std::min<int64_t>(W, budget / per);
            if (W >= 2) {
              g.par_mode = fiber ? 3 : 2;
              g.workers = W;
              g.out_size = G.out_size;
              g.priv = priv;
              g.tail = js.tail;
              g.n_tail_bufs = js.n_rset;
              for (int i = 0; i < js.n_rset; ++i) {
                g.tail_off[i] = off[js.rset[i]];
                g.tail_len[i] = G.buffer_size[js.rset[i]];
              }
            }
          }
        }
      }
      // Small working sets run shared-memory resident (generic.cu
      // k_generic_sm): root slices to up to 8 walkers where mode 1 applies.
      // Only where the walk is sequential anyway or its root slices fit the
      // 8 walkers: wider plans keep the global interpreter's parallelism.
      const bool sm_par_ok = g.par_mode == 0 || (g.par_mode == 1 && D.level_size[0] <= 8);
      if (!G.observe && env_int("SPTTN_GENERIC_SM", 1) != 0 && !want_jit && sm_par_ok) {
        const int smw = g.par_mode == 1 ? static_cast<int>(std::min<int64_t>(g.workers, 8)) : 1;
        spttn_dev::GenericState t{};
        if (spttn_dev::generic_sm_layout(G, D, smw, smem_optin_bytes(), t) ||
            (smw > 1 && spttn_dev::generic_sm_layout(G, D, 1, smem_optin_bytes(), t))) {
          g.sm = true;
          g.sm_workers = t.sm_workers;
          g.sm_bytes = t.sm_bytes;
          std::memcpy(g.sm_off, t.sm_off, sizeof(g.sm_off));
          std::memcpy(g.dense_size, t.dense_size, sizeof(g.dense_size));
          g.par_mode = g.sm_workers > 1 ? 1 : 0;
          g.workers = 1;  // no global replicas
          g.priv = g.tail = false;
        }
      }
      if (g.sm) {
        // device arena [prog | boff | factors][out | counters] mirrored by a
        // pinned host parcel: program + offsets uploaded here, factors by
        // one copy per set_factors, out + counters read back by one copy
        g.up_prog = al(sizeof(spg_program));
        size_t up = g.up_prog + al((nb + 1) * sizeof(int64_t));
        g.up_fac = up;
        for (int f = 0; f < p->nf; ++f) {
          g.fac_off[f] = up;
          if (!on_dev) up += al(p->fac_size[f] * 8);
        }
        g.up_end = up;
        g.down_cnt = up + al(std::max<int64_t>(1, G.out_size) * 8);
        g.down_end = g.down_cnt + al((nb + 5) * sizeof(int64_t));
        g.parcel_bytes = g.down_end;
        dev_malloc(&p->arena, g.parcel_bytes, s);
        g.parcel = static_cast<unsigned char*>(spttn_dev::pinned_alloc(g.parcel_bytes));
        unsigned char* dev = static_cast<unsigned char*>(p->arena);
        g.d_prog = reinterpret_cast<spg_program*>(dev);
        g.buffer_off = reinterpret_cast<int64_t*>(dev + g.up_prog);
        if (!on_dev)
          for (int f = 0; f < p->nf; ++f) p->fac[f] = reinterpret_cast<double*>(dev + g.fac_off[f]);
        p->out = reinterpret_cast<double*>(dev + g.up_end);
        g.counters = reinterpret_cast<int64_t*>(dev + g.down_cnt);
        g.total_buffer_elems = off[nb];
        g.in_arena = true;
        std::memcpy(g.parcel, &G, sizeof(spg_program));
        std::memcpy(g.parcel + g.up_prog, off.data(), off.size() * sizeof(int64_t));
        SPTTN_CUDA(cudaMemcpyAsync(dev, g.parcel, g.up_fac, cudaMemcpyHostToDevice, s));
        SPTTN_CUDA(cudaEventCreateWithFlags(&g.up_done, cudaEventDisableTiming));
        SPTTN_CUDA(cudaEventRecord(g.up_done, s));
      } else {
      const int64_t reps = g.workers;
      const size_t n_cnt = (nb + 5) * sizeof(int64_t);  // + slice counter (mode 1)
      const size_t n_buf = static_cast<size_t>(std::max<int64_t>(1, off[nb]) * reps) * 8;
      const size_t n_out = static_cast<size_t>(std::max<int64_t>(1, G.out_size)) * 8;
      const size_t n_priv =
          g.priv ? static_cast<size_t>(std::max<int64_t>(1, G.out_size) * reps) * 8 : 0;
      const bool lookup = G.need_leaf_lookup && nnz > 0 && !g.sm;
      size_t total = n_cnt + n_buf + n_out + n_priv;  // contiguous, 8-byte aligned
      total = al(total) + al(sizeof(spg_program)) + al((nb + 1) * sizeof(int64_t)) +
              al(16 * sizeof(double*));
      if (!on_dev)
        for (int f = 0; f < p->nf; ++f) total += al(p->fac_size[f] * 8);
      const int64_t log_bytes = G.observe ? G.observe_log_bytes : 0;
      total += al(log_bytes);
      if (lookup) total += 2 * al(nnz * sizeof(int64_t));
      dev_malloc(&p->arena, total, s);
      char* cur = static_cast<char*>(p->arena);
      auto take = [&](size_t bytes) { char* r = cur; cur += al(bytes); return r; };
      g.counters = reinterpret_cast<int64_t*>(cur);
      g.buffers = reinterpret_cast<double*>(cur + n_cnt);
      p->out = reinterpret_cast<double*>(cur + n_cnt + n_buf);
      if (g.priv) g.priv_out = reinterpret_cast<double*>(cur + n_cnt + n_buf + n_out);
      g.zero_bytes = n_cnt + n_buf + n_out + n_priv;
      cur += al(g.zero_bytes);
      g.total_buffer_elems = off[nb];
      g.d_prog = reinterpret_cast<spg_program*>(take(sizeof(spg_program)));
      g.buffer_off = reinterpret_cast<int64_t*>(take((nb + 1) * sizeof(int64_t)));
      p->d_dense = reinterpret_cast<const double**>(take(16 * sizeof(double*)));
      if (!on_dev)
        for (int f = 0; f < p->nf; ++f) p->fac[f] = reinterpret_cast<double*>(take(p->fac_size[f] * 8));
      g.log_bytes = log_bytes;
      g.log = log_bytes > 0 ? reinterpret_cast<unsigned char*>(take(log_bytes)) : nullptr;
      if (lookup) {
        g.leaf_keys = reinterpret_cast<int64_t*>(take(nnz * sizeof(int64_t)));
        g.leaf_pos = reinterpret_cast<int64_t*>(take(nnz * sizeof(int64_t)));
        g.n_leaf_keys = nnz;
      }
      g.in_arena = true;
      SPTTN_CUDA(cudaMemcpyAsync(g.d_prog, &G, sizeof(spg_program), cudaMemcpyHostToDevice, s));
      SPTTN_CUDA(cudaMemcpyAsync(g.buffer_off, off.data(), off.size() * sizeof(int64_t),
                                 cudaMemcpyHostToDevice, s));
      }
    }
    spttn_dev::plan_trace("plan: setup", s);
    copy_factors(p, desc->factors, on_dev, s);
    spttn_dev::plan_trace("plan: factors", s);
    bool facs_aligned32 = true, facs_aligned16 = true;
    for (int f = 0; f < p->nf; ++f) {
      facs_aligned32 &= aligned(p->fac[f], 32);
      facs_aligned16 &= aligned(p->fac[f], 16);
    }
    p->fac_align = facs_aligned32 ? 32 : facs_aligned16 ? 16 : 8;

    if (p->kind == SPTTN_NEST_GENERIC) {
      p->out_count = p->prog->out_size;
      const double* hp[16] = {nullptr};
      for (int f = 0; f < p->nf; ++f) hp[f + 1] = p->fac[f];
      for (int f = 0; f < 16; ++f) p->gen.dense_dev[f] = hp[f];
      if (!p->gen.sm)
        SPTTN_CUDA(cudaMemcpyAsync(p->d_dense, hp, sizeof(hp), cudaMemcpyHostToDevice, s));
      if (p->gen.n_leaf_keys > 0 && !p->gen.sm) {
        k_leaf_keys<<<static_cast<unsigned>((nnz + 255) / 256), 256, 0, s>>>(
            D.view(), p->gen.d_prog, p->gen.leaf_keys, p->gen.leaf_pos);
        SPTTN_CUDA(cudaGetLastError());
      }
      p->launches = p->gen.sm ? 1 : 2 + (p->gen.priv ? 1 : 0) + (p->gen.tail ? p->gen.n_tail_bufs + 1 : 0);
      const int64_t jit_env2 = env_int("SPTTN_GENERIC_JIT", -1);
      if (!p->prog->observe && spttn_dev::jit_available() &&
          (jit_env2 == 1 || (jit_env2 < 0 && nnz >= (int64_t{1} << 16))))
        p->gen.jit_kernel = spttn_dev::jit_prepare(*p->prog, p->gen);
    } else if (p->kind == SPTTN_NEST_MTTKRP3_J || p->kind == SPTTN_NEST_MTTKRP3_K) {
      // output rows on CSF level 1 / 2: packed 4-slot groups of (i,j)
      // segments, atomics into a zeroed output (no items, no fix-up)
      p->out_count = D.dims[p->kind == SPTTN_NEST_MTTKRP3_J ? 1 : 2] * R;
      dev_malloc(reinterpret_cast<void**>(&p->out), std::max<int64_t>(1, p->out_count) * 8, s);
      p->vec = (R % 4 == 0) && facs_aligned32 ? 1 : 0;
      // mode 4 (default when they fit): column quarters of the gathered
      // factor and of the output accumulated in shared memory
      const int nr_mode = p->kind == SPTTN_NEST_MTTKRP3_J ? 1 : 2;
      const int64_t rows_in = R > 0 ? p->fac_size[1] / R : 0;
      const int64_t rows_out = D.dims[nr_mode];
      const bool nr_fits = R % 8 == 0 && facs_aligned16 && D.level_size[0] < (1 << 27) &&
                           spttn_dev::mttkrp3_nr_smem(rows_in, rows_out) <=
                               static_cast<size_t>(smem_optin_bytes());
      // mode 5 (default when the root kernel's shared-memory form fits): the
      // CSF re-ordered at plan time with the output mode as the root — (j,i,k)
      // for mode j, (k,i,j) for mode k — and the root-output MTTKRP-3 kernel
      // (k_mttkrp3_smf) on it: out[j] = sum_i A[i] * (sum_k t C[k]) and
      // out[k] = sum_i A[i] * (sum_j t B[j]), the same sums regrouped. Owner-
      // computes rows, no atomics, a fixed summation order (bit-reproducible).
      const bool tr_fits = R % 16 == 0 && facs_aligned16 && D.level_size[0] < (1 << 27) &&
                           (p->fac_size[0] / R) * R < (int64_t{1} << 31) &&
                           spttn_dev::mttkrp3_smf_smem(rows_in) <=
                               static_cast<size_t>(smem_optin_bytes());
      p->mode = static_cast<int>(env_int("SPTTN_NONROOT_MODE", tr_fits ? 5 : nr_fits ? 4 : 0));
      if (p->mode == 5 && !tr_fits) p->mode = nr_fits ? 4 : 0;
      if (p->mode == 5) {
        const int order_j[3] = {1, 0, 2}, order_k[3] = {2, 0, 1};
        p->tcsf = new spttn_dev::DevCsf;
        spttn_dev::csf_permute(D, nr_mode == 1 ? order_j : order_k, *p->tcsf, s);
        const auto& TD = *p->tcsf;
        const int64_t warps = static_cast<int64_t>(sm_count()) * 16 * 2;
        const int64_t chunk = std::clamp<int64_t>((TD.level_size[1] + warps - 1) / warps, 8, 1024);
        spttn_dev::build_segments(TD, 1, 4, chunk, p->dec, tile, s, false);
        spttn_dev::build_packed(TD, 2, p->dec, s, 8);
        if (smf_ranges(p, TD, sm_count(), tile, s)) {
          spttn_dev::mttkrp3_smf_prepare(p->dec, static_cast<int>(R), s);
          p->launches = 1;
        } else {  // a root slice too heavy for one CTA: the atomic kernels
          SPTTN_CUDA(cudaStreamSynchronize(s));  // default-stream frees are for idle blocks
          spttn_dev::free_decomp(p->dec);
          p->dec = spttn_dev::Decomp{};
          free_tcsf(p);
          p->mode = nr_fits ? 4 : 0;
        }
      }
      if (p->mode == 4 && !nr_fits) p->mode = 0;
      if (p->mode != 5) {
      spttn_dev::build_segments(D, 1, 4, 1, p->dec, 0, s, false);
      spttn_dev::build_packed(D, 2, p->dec, s, p->mode == 4 ? 8 : 4);
      if (p->mode == 4) {
        spttn_dev::mttkrp3_nr_prepare(p->dec, nr_mode, rows_in, s);
        p->dec.n_cta = std::max(1, sm_count() / static_cast<int>(R / 8));
      }
      p->launches = 2;  // memset + kernel
      }
    } else {
      const bool sparse_out = p->kind == SPTTN_NEST_TTTP3;
      p->out_count = sparse_out ? nnz : D.dims[0] * tile;
      dev_malloc(reinterpret_cast<void**>(&p->out), std::max<int64_t>(1, p->out_count) * 8, s);
      const int sms = sm_count();
      if (p->kind == SPTTN_NEST_TTMC3 || p->kind == SPTTN_NEST_TTMC4) {
        const bool vu = (R % 2 == 0) && facs_aligned16;
        const bool vv = p->kind == SPTTN_NEST_TTMC3 ? (S % 2 == 0 && facs_aligned16)
                                                    : (S == 8 && facs_aligned32);
        p->vec = (vu ? 1 : 0) | (vv ? 2 : 0);
        if (p->kind == SPTTN_NEST_TTMC4)  // 128-bit W row pieces
          p->vec |= (p->T % 2 == 0) && facs_aligned16 ? 4 : 0;
        if (p->kind == SPTTN_NEST_TTMC3)  // 256-bit row gathers (wide kernel)
          p->vec |= ((R % 4 == 0) && facs_aligned32 ? 4 : 0) | ((S % 4 == 0) && facs_aligned32 ? 8 : 0);
        // TTMc-3 stages a group's <= 4 segments of leaves in one warp-wide
        // register block: seg_len <= 8.
        int seg_len = static_cast<int>(
            env_int("SPTTN_SEG_LEN", p->kind == SPTTN_NEST_TTMC3 ? 4 : 8));
        if (p->kind == SPTTN_NEST_TTMC3) {
          // packed, TMA-staged, row-contiguous gathers (k_ttmc3pq); the
          // earlier variants (modes 0, 4, 6, 7, 11), the shuffle-transposed
          // and the fully cp.async-fed kernels lost and were removed;
          // 16 = mode 10 with U rows and single-leaf V rows fed by cp.async
          p->mode = 10;
          if (env_int("SPTTN_TTMC3_PF", 1) == 1 && R == 16 && S == 16 && (p->vec & 4) && (p->vec & 8))
            p->mode = 16;  // tiles fed by cp.async one group ahead (pair-permuted packing)
          seg_len = std::clamp(seg_len, 1, 4);
        }
        seg_len = std::max(seg_len, 1);
        const int64_t units = D.level_size[1];
        const int64_t warps = static_cast<int64_t>(sms) * 32 * 2;
        int64_t chunk = env_int("SPTTN_CHUNK", 0);
        if (chunk <= 0) chunk = std::clamp<int64_t>((units + warps - 1) / warps, 8, 1024);
        if (p->kind == SPTTN_NEST_TTMC4) {
          // 4 = V / W row gathers by cp.async one leaf step ahead (k_ttmc4pa;
          // S = T = 8, R <= 8, 16-byte aligned factors), else 3 = packed,
          // TMA-staged, row-contiguous gathers (k_ttmc4pq; any R, S, T <= 8)
          p->mode = static_cast<int>(env_int(
              "SPTTN_TTMC4_MODE", (R <= 8 && S == 8 && p->T == 8 && facs_aligned16) ? 4 : 3));
          if (p->mode != 4 || !(R <= 8 && S == 8 && p->T == 8 && facs_aligned16)) p->mode = 3;
        }
        if (p->kind == SPTTN_NEST_TTMC4) {
          // (i,j) pieces of <= 4 leaves, length-sorted groups of 8, with each
          // leaf's level-2 (k) coordinate packed next to its level-3 (l) one
          spttn_dev::build_segments(D, 1, std::clamp(seg_len, 1, 4), chunk, p->dec, tile, s,
                                    false, true);
          int32_t* leaf_k = nullptr;
          dev_malloc(reinterpret_cast<void**>(&leaf_k), std::max<int64_t>(1, nnz) * sizeof(int32_t), s);
          spttn_dev::expand_coords(D, 2, D.idx[2], leaf_k, s);
          spttn_dev::build_packed(D, 3, p->dec, s, spttn_dev::kPackSlots, leaf_k, &fill_done);
          spttn_dev::dfree(leaf_k, spttn_dev::aux_stream());  // read by the fill
          // mode 4: one item per resident warp of k_ttmc4pa (a single wave of
          // 12-warp CTAs; BASELINE shape: 1773 items 338 us, 2 waves 346 us,
          // the earlier 2.66 waves 391 us — the last partial wave idled a
          // third of the SMs); mode 3: two items per 32 warps per SM
          const int64_t wv4 = p->mode == 4
                                  ? static_cast<int64_t>(sms) * spttn_dev::ttmc4pa_warps_per_sm()
                                  : static_cast<int64_t>(sms) * 16 * 2;
          int64_t gchunk = env_int("SPTTN_GCHUNK", 0);
          if (gchunk <= 0)
            gchunk = std::clamp<int64_t>((p->dec.n_groups + wv4 - 1) / wv4, 4, 1024);
          // mode 4: items cut at equal work, leaf steps + 3 per group
          // (BASELINE shape, kernel us: equal group counts 448; overhead 2:
          // 408, 3: 404, 4: 409, 6: 416)
          const int ovh4 = p->mode == 4 ? static_cast<int>(env_int("SPTTN_GROUP_OVERHEAD", 3)) : 0;
          spttn_dev::finish_unit_items(D, p->dec, p->dec.slice_grp, p->dec.n_groups, gchunk, tile, s,
                                       ovh4);
          if (p->mode == 4 && env_int("SPTTN_ITEM_CLOCKS", 0) == 1) {
            const int64_t cb = std::max<int64_t>(1, 6 * p->dec.n_items) * sizeof(long long);
            dev_malloc(reinterpret_cast<void**>(&p->item_clk), cb, s);
            SPTTN_CUDA(cudaMemsetAsync(p->item_clk, 0, cb, s));
          }
        } else if (p->kind == SPTTN_NEST_TTMC3) {
          // packed length-sorted groups of 8 segments (pack.cu)
          spttn_dev::build_segments(D, 1, seg_len, chunk, p->dec, tile, s, false);
          spttn_dev::build_packed(D, 2, p->dec, s, spttn_dev::kPackSlots, nullptr, &fill_done,
                                  p->mode == 16);
          int64_t gchunk = env_int("SPTTN_GCHUNK", 0);
          if (gchunk <= 0) {
            // mode 10: one item per resident warp (a single wave; 2.6 waves of
            // half-size items measured 278 vs 269 us per step at the BASELINE
            // shape — fewer split slices for the fix-up, no tail wave)
            const int64_t wv = static_cast<int64_t>(sms) * spttn_dev::ttmc3pq_warps_per_sm();
            gchunk = std::clamp<int64_t>((p->dec.n_groups + wv - 1) / wv, 4, 512);
          }
          // k_ttmc3pq reads variable item ranges cut at equal work (leaf steps
          // + a per-group overhead, decomp.cu k_group_work). Measured on the
          // BASELINE shape with the step-specialised kernel (per-item
          // %globaltimer records, tools/item_balance.py): overhead 1 / 2 / 3 /
          // 4 / 6 / 12 / 24 -> 259 / 241 / 228 / 224 / 230 / 241 / 248 us;
          // busy efficiency 0.85 at 12, 0.92 at 4
          const int ovh = static_cast<int>(env_int("SPTTN_GROUP_OVERHEAD", 4));
          spttn_dev::finish_unit_items(D, p->dec, p->dec.slice_grp, p->dec.n_groups, gchunk, tile, s,
                                       ovh);
#ifdef SPTTN_DEBUG_BOUNDS
          // bounds-checked build only: SPTTN_DEBUG_POISON=1 plants an
          // out-of-range leaf coordinate so tests can see the checks fire
          if (env_int("SPTTN_DEBUG_POISON", 0) == 1 && p->dec.n_packed_leaves > 0) {
            spttn_dev::csf_wait_fill(fill_done, s);
            const int32_t bad = static_cast<int32_t>(D.dims[2] + 5);
            SPTTN_CUDA(cudaMemcpyAsync(p->dec.pk, &bad, sizeof(bad), cudaMemcpyHostToDevice, s));
            SPTTN_CUDA(cudaStreamSynchronize(s));
          }
#endif
          if (env_int("SPTTN_ITEM_CLOCKS", 0) == 1) {  // recorded by the 256-bit-gather kernel only
            const int64_t cb = std::max<int64_t>(1, 6 * p->dec.n_items) * sizeof(long long);
            dev_malloc(reinterpret_cast<void**>(&p->item_clk), cb, s);
            SPTTN_CUDA(cudaMemsetAsync(p->item_clk, 0, cb, s));
          }
        } else {
          spttn_dev::build_segments(D, 1, seg_len, chunk, p->dec, tile, s);
        }
      } else if (!sparse_out && R <= 32 && env_int("SPTTN_MTTKRP_MODE", 2) >= 1) {
        // segment-form MTTKRP (R <= 32): 3 = packed length-sorted groups with
        // TMA-staged streams (default for order 4), 2 = packed (default for
        // order 3: items hold too few windows to amortise the staging
        // prologue), 1 = plain segments
        // 4 = factor column blocks resident in shared memory (order 3,
        // default when they fit and the slices balance over the CTAs)
        p->vec = (R % 4 == 0) && facs_aligned32 ? 1 : 0;
        const int64_t rows_b = R > 0 ? p->fac_size[0] / R : 0;
        const int64_t rows_c = R > 0 ? p->fac_size[1] / R : 0;
        const bool smf_fits = D.order == 3 && R % 16 == 0 && facs_aligned16 &&
                              rows_b * R < (int64_t{1} << 31) && D.level_size[0] < (1 << 27) &&
                              spttn_dev::mttkrp3_smf_smem(rows_c) <=
                                  static_cast<size_t>(smem_optin_bytes());
        // 4 = C column halves resident in shared memory (order 3 default), 2 =
        // packed (order-3 fallback), 3 = packed + TMA-staged streams (order 4)
        p->mode = static_cast<int>(env_int("SPTTN_MTTKRP_MODE", D.order == 4 ? 3 : (smf_fits ? 4 : 2)));
        if (p->mode == 4 && !smf_fits) p->mode = 2;
        if (p->mode < 2 || p->mode > 4) p->mode = 2;
        if (D.order == 4) p->mode = 3;
        const int seg_len = static_cast<int>(std::clamp<int64_t>(env_int("SPTTN_SEG_LEN", 4), 1, 4));
        const int unit_level = D.order - 2;
        const int64_t units = D.level_size[unit_level];
        const int64_t warps = static_cast<int64_t>(sms) * 16 * 2;
        int64_t chunk = env_int("SPTTN_CHUNK", 0);
        if (chunk <= 0) chunk = std::clamp<int64_t>((units + warps - 1) / warps, 8, 1024);
        if (p->mode == 4) {
          spttn_dev::build_segments(D, unit_level, seg_len, chunk, p->dec, tile, s, false);
          spttn_dev::build_packed(D, D.order - 1, p->dec, s, 8);
          if (smf_ranges(p, D, sms, tile, s)) {
            spttn_dev::mttkrp3_smf_prepare(p->dec, static_cast<int>(R), s);
          } else {
            SPTTN_CUDA(cudaStreamSynchronize(s));  // default-stream frees are for idle blocks
            spttn_dev::free_decomp(p->dec);
            p->mode = 2;
          }
        }
        if (p->mode == 2 || p->mode == 3) {
          spttn_dev::build_segments(D, unit_level, seg_len, chunk, p->dec, tile, s, false);
          spttn_dev::build_packed(D, D.order - 1, p->dec, s, 4, nullptr, &fill_done);
          // order 3: one item per resident warp (k_mttkrp_pk: 4 CTAs of 8
          // warps per SM) — a single wave, and root slices stay within one
          // fix-up chunk (one fix-up kernel)
          // order 4: six items per resident warp (24 per SM) — fewer, longer
          // items than the earlier 64-group cap (51620 items) halve the split
          // slices the fix-up sums: step 641.5 -> 631.8 us at the BASELINE
          // shape (4 items per warp 635.9, 8: 631.7, 1: 671.3)
          const int64_t w24 = static_cast<int64_t>(sms) * (D.order == 3 ? 32 : 24 * 6);
          int64_t gchunk = env_int("SPTTN_GCHUNK", 0);
          if (gchunk <= 0)
            gchunk = std::clamp<int64_t>((p->dec.n_groups + w24 - 1) / w24, 4, 1024);
          // order 4: items cut at equal work, leaf steps + 4 per group (BASELINE
          // MTTKRP-4 kernel us: equal group counts 644, overhead 1: 637, 2: 631,
          // 4: 625, 8: 631)
          const int ovhm = p->mode == 3 ? static_cast<int>(env_int("SPTTN_GROUP_OVERHEAD", 4)) : 0;
          spttn_dev::finish_unit_items(D, p->dec, p->dec.slice_grp, p->dec.n_groups, gchunk, tile, s,
                                       ovhm);
          if (D.order == 4 && env_int("SPTTN_ITEM_CLOCKS", 0) == 1) {
            const int64_t cb = std::max<int64_t>(1, 6 * p->dec.n_items) * sizeof(long long);
            dev_malloc(reinterpret_cast<void**>(&p->item_clk), cb, s);
            SPTTN_CUDA(cudaMemsetAsync(p->item_clk, 0, cb, s));
          }
        }
      } else {
        const int G = spttn_dev::group_lanes_for(static_cast<int>(R));
        p->vec = (R % 4 == 0) && facs_aligned32 ? 1 : 0;
        const int64_t groups = static_cast<int64_t>(sms) * (2048 / G) * 2;
        int64_t chunk = env_int("SPTTN_CHUNK", 0);
        if (chunk <= 0) chunk = std::clamp<int64_t>((nnz + groups - 1) / groups, 16, 4096);
        if (sparse_out) {
          // slice pieces (nest_tttp.cu): A[i] once per piece of <= 64 leaves;
          // the round-1 leaf-parallel (3.52 ms) and C-bucketed (3.42 ms)
          // variants lost to it (2.75 ms) and were removed
          p->mode = 3;
          p->batch = static_cast<int>(env_int("SPTTN_TTTP_BATCH", 4));
          spttn_dev::build_leaf_coords(D, &p->leaf_i, &p->leaf_j, s);
          spttn_dev::pack_leaf_jk(D, p->leaf_j, &p->leaf_jk, s);
          spttn_dev::dfree(p->leaf_i, s);  // pieces carry i, leaf_jk carries j and k
          spttn_dev::dfree(p->leaf_j, s);
          p->leaf_i = p->leaf_j = nullptr;
          const int P = static_cast<int>(env_int("SPTTN_TTTP_PIECE", 64));
          p->n_pieces = spttn_dev::build_tttp_pieces(D, std::max(1, P), &p->pieces, s);
        }
        else
          spttn_dev::build_leaf_items(D, chunk, p->dec, tile, s);
      }
      // fix-up: one launch, plus a second when the heavy split slices exceed
      // one wave (decomp.cu launch_fixup)
      p->launches = 1 + ((p->dec.n_split > 0 || p->dec.n_absent > 0) ? 1 : 0) +
                    (p->dec.n_multi > sms ? 1 : 0);
      if (p->kind == SPTTN_NEST_MTTKRP3 && p->mode == 4) p->launches = 1;  // no fix-up pass
    }
    if (fill_done) {  // packed leaf streams filled on the side stream
      SPTTN_CUDA(cudaStreamWaitEvent(s, fill_done, 0));
      SPTTN_CUDA(cudaEventDestroy(fill_done));
      fill_done = nullptr;
    }
    spttn_dev::plan_trace("plan: decomposition", s);
    SPTTN_CUDA(cudaStreamSynchronize(s));
    *out = p;
    raw = nullptr;
  });
  if (rc != SPTTN_OK && raw) {
    std::string keep = g_err;
    spttn_plan_destroy(raw);
    g_err = keep;
  }
  return rc;
}

int spttn_plan_set_factors(spttn_plan* p, const double* const* factors, int32_t on_device,
                           void* stream) {
  return guarded([&] {
    if (!p) fail(SPTTN_EINVAL, "null plan");
    if (on_device && p->own_fac) fail(SPTTN_EINVAL, "plan owns its factor copies; pass host arrays");
    if (!on_device && !p->own_fac) fail(SPTTN_EINVAL, "plan uses device factors; pass device arrays");
    if (on_device) {  // vector / cp.async kernels were picked for the plan's alignment
      for (int f = 0; f < p->nf; ++f)
        if (factors[f] && !aligned(factors[f], p->fac_align))
          fail(SPTTN_EINVAL, "device factor less aligned than at plan creation (" +
                                 std::to_string(p->fac_align) + " bytes); create a new plan");
    }
    copy_factors(p, factors, on_device != 0, as_stream(stream));
    if (p->kind == SPTTN_NEST_GENERIC && on_device) {
      const double* hp[16] = {nullptr};
      for (int f = 0; f < p->nf; ++f) hp[f + 1] = p->fac[f];
      for (int f = 0; f < 16; ++f) p->gen.dense_dev[f] = hp[f];
      SPTTN_CUDA(cudaMemcpyAsync(p->d_dense, hp, sizeof(hp), cudaMemcpyHostToDevice,
                                 as_stream(stream)));
    }
  });
}

int spttn_execute(spttn_plan* p, void* stream) { return spttn_execute_stage(p, -1, stream); }

int spttn_execute_stage(spttn_plan* p, int stage, void* stream) {
  return guarded([&] {
    if (!p) fail(SPTTN_EINVAL, "null plan");
    if (stage < -1 || stage > 1) fail(SPTTN_EINVAL, "stage must be -1, 0 or 1");
    cudaStream_t s = as_stream(stream);
    p->csf->d.wait_values(s);
    const auto& D = p->tcsf ? *p->tcsf : p->csf->d;
    if (p->kind == SPTTN_NEST_GENERIC) {
      if (stage != 1) {
        if (p->gen.jit_kernel)
          spttn_dev::jit_execute(p->gen.jit_kernel, *p->prog, D, p->d_dense, p->out, p->gen, s);
        else
          spttn_dev::generic_execute(*p->prog, D, p->d_dense, p->out, p->gen, s);
      }
      return;
    }
    spttn_dev::RootOutArgs a{};
    a.t = D.view();
    a.R = static_cast<int>(p->R);
    a.S = static_cast<int>(p->S);
    a.T = static_cast<int>(p->T);
    a.vec = p->vec;
    a.item_pos = p->dec.item_pos;
    a.n_items = p->dec.n_items;
    a.chunk = p->dec.chunk;
    a.out = p->out;
    a.part = p->dec.part;
    a.flags = ((p->flags & SPTTN_FLAG_RESIDUAL) ? 1 : 0) | (p->mode << 8);
    a.clk = p->item_clk;
    for (int l = 0; l < 4; ++l) a.frows[l] = l < D.order ? D.dims[l] : 0;
    a.seg_begin = p->dec.seg_begin;
    a.seg_node = p->dec.seg_node;
    a.slice_seg = p->dec.slice_seg;
    a.n_seg = p->dec.n_seg;
    a.grp_hdr = p->dec.grp_hdr;
    a.grp_node = p->dec.grp_node;
    a.grp_node1 = p->dec.grp_node1;
    a.pk = p->dec.pk;
    a.pk2 = p->dec.pk2;
    a.pv = p->dec.pv;
    a.slice_grp = p->dec.slice_grp;
    a.n_groups = p->dec.n_groups;
    a.item_unit = p->dec.item_unit;
    if (stage != 1) switch (p->kind) {
      case SPTTN_NEST_MTTKRP3_J:
      case SPTTN_NEST_MTTKRP3_K:
        if (p->mode == 5) {  // root kernel on the re-ordered tensor: A at level 1
          a.f[1] = p->fac[0];
          a.f[2] = p->fac[1];
          spttn_dev::SmfArgs x{};
          x.nq = static_cast<int>(p->R / 16);
          x.n_cta = static_cast<int>(p->dec.n_cta);
          x.rows_c = static_cast<int32_t>(p->fac_size[1] / p->R);
          x.cta_grp = p->dec.cta_grp;
          x.hdr2 = p->dec.hdr2;
          x.absent_rows = p->dec.absent_rows;
          x.n_absent = p->dec.n_absent;
          spttn_dev::launch_mttkrp3_smf(a, x, s);
          break;
        }
        a.f[0] = p->fac[0];
        a.f[1] = p->fac[1];
        SPTTN_CUDA(cudaMemsetAsync(p->out, 0, std::max<int64_t>(1, p->out_count) * 8, s));
        if (p->mode == 4) {
          const int nr_mode = p->kind == SPTTN_NEST_MTTKRP3_J ? 1 : 2;
          spttn_dev::SmfArgs x{};
          x.nq = static_cast<int>(p->R / 8);
          x.n_cta = static_cast<int>(p->dec.n_cta);
          x.rows_c = static_cast<int32_t>(p->fac_size[1] / p->R);
          x.rows_out = static_cast<int32_t>(p->out_count / p->R);
          x.hdr2 = p->dec.hdr2;
          spttn_dev::launch_mttkrp3_nr_smf(a, x, nr_mode, s);
        } else {
          spttn_dev::launch_mttkrp3_nonroot(a, p->kind == SPTTN_NEST_MTTKRP3_J ? 1 : 2, s);
        }
        break;
      case SPTTN_NEST_MTTKRP3:
        a.f[1] = p->fac[0];
        a.f[2] = p->fac[1];
        if (p->mode == 4) {
          spttn_dev::SmfArgs x{};
          x.nq = static_cast<int>(p->R / 16);
          x.n_cta = static_cast<int>(p->dec.n_cta);
          x.rows_c = static_cast<int32_t>(p->fac_size[1] / p->R);
          x.cta_grp = p->dec.cta_grp;
          x.hdr2 = p->dec.hdr2;
          x.absent_rows = p->dec.absent_rows;
          x.n_absent = p->dec.n_absent;
          spttn_dev::launch_mttkrp3_smf(a, x, s);
        } else if (p->mode == 3)
          spttn_dev::launch_mttkrp_pq(a, 3, s);
        else if (p->mode == 2)
          spttn_dev::launch_mttkrp_pk(a, s);
        else
          spttn_dev::launch_mttkrp3(a, s);
        break;
      case SPTTN_NEST_MTTKRP4:
        a.f[1] = p->fac[0];
        a.f[2] = p->fac[1];
        a.f[3] = p->fac[2];
        if (p->mode == 3)
          spttn_dev::launch_mttkrp_pq(a, 4, s);
        else
          spttn_dev::launch_mttkrp4(a, s);
        break;
      case SPTTN_NEST_TTTP3:
        a.f[0] = p->fac[0];
        a.f[1] = p->fac[1];
        a.f[2] = p->fac[2];
        spttn_dev::launch_tttp3_pieces(a, p->pieces, p->n_pieces, p->leaf_jk, p->batch, s);
        break;
      case SPTTN_NEST_TTMC3:
        a.f[1] = p->fac[0];
        a.f[2] = p->fac[1];
        spttn_dev::launch_ttmc3(a, s);
        break;
      case SPTTN_NEST_TTMC4:
        a.f[1] = p->fac[0];
        a.f[2] = p->fac[1];
        a.f[3] = p->fac[2];
        spttn_dev::launch_ttmc4(a, s);
        break;
    }
    if (stage != 0 && p->kind != SPTTN_NEST_TTTP3 && !(p->kind == SPTTN_NEST_MTTKRP3 && p->mode == 4))
      spttn_dev::launch_fixup(p->dec, a.t, p->out, s);
  });
}

int64_t spttn_output_count(const spttn_plan* p) { return p ? p->out_count : -1; }
const double* spttn_output_device(const spttn_plan* p) { return p ? p->out : nullptr; }

int spttn_read_output(spttn_plan* p, double* host_out, int64_t count, void* stream) {
  return guarded([&] {
    if (!p || (!host_out && count)) fail(SPTTN_EINVAL, "null argument");
    if (count != p->out_count) fail(SPTTN_EINVAL, "output count mismatch");
    cudaStream_t s = as_stream(stream);
    auto& g = p->gen;
    if (g.parcel) {  // small GENERIC plan: [out | counters] in one pinned copy
      unsigned char* dev = static_cast<unsigned char*>(p->arena);
      SPTTN_CUDA(cudaMemcpyAsync(g.parcel + g.up_end, dev + g.up_end, g.down_end - g.up_end,
                                 cudaMemcpyDeviceToHost, s));
      SPTTN_CUDA(cudaStreamSynchronize(s));
      if (count) std::memcpy(host_out, g.parcel + g.up_end, count * sizeof(double));
      p->last_counters.resize(p->prog->num_buffers + 4);
      std::memcpy(p->last_counters.data(), g.parcel + g.down_cnt,
                  p->last_counters.size() * sizeof(int64_t));
      p->last_madds = p->last_counters[0];
      return;
    }
    if (count)
      SPTTN_CUDA(cudaMemcpyAsync(host_out, p->out, count * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (p->kind == SPTTN_NEST_GENERIC) {  // counters travel with the output
      p->last_counters.resize(p->prog->num_buffers + 4);
      SPTTN_CUDA(cudaMemcpyAsync(p->last_counters.data(), p->gen.counters,
                                 p->last_counters.size() * sizeof(int64_t),
                                 cudaMemcpyDeviceToHost, s));
    }
    SPTTN_CUDA(cudaStreamSynchronize(s));
    if (p->kind == SPTTN_NEST_GENERIC) p->last_madds = p->last_counters[0];
  });
}

int spttn_plan_info(const spttn_plan* p, int64_t* out, int n) {
  return guarded([&] {
    if (!p) fail(SPTTN_EINVAL, "null plan");
    const bool gen = p->kind == SPTTN_NEST_GENERIC;
    const int64_t v[11] = {p->launches,   p->dec.n_items, p->dec.n_split, p->dec.n_absent,
                           p->dec.n_items * 2 * p->dec.tile * 8,
                           p->kind,        p->dec.n_seg,   gen ? p->last_madds : -1,
                           gen ? p->gen.par_mode : -1,
                           gen ? (p->gen.jit_kernel != nullptr ? 1 : 0) : -1,
                           gen ? -1 : p->mode};
    for (int i = 0; i < n && i < 11; ++i) out[i] = v[i];
  });
}

int spttn_plan_item_clocks(const spttn_plan* p, int64_t* host_out, int64_t n) {
  return guarded([&] {
    if (!p || !p->item_clk) fail(SPTTN_EINVAL, "plan records no item clocks (SPTTN_ITEM_CLOCKS=1)");
    const int64_t m = std::min<int64_t>(n, 6 * p->dec.n_items);
    SPTTN_CUDA(cudaDeviceSynchronize());
    SPTTN_CUDA(cudaMemcpy(host_out, p->item_clk, m * sizeof(int64_t), cudaMemcpyDeviceToHost));
  });
}

int spttn_generic_resets(const spttn_plan* p, int64_t* out, int n) {
  return guarded([&] {
    if (!p || p->kind != SPTTN_NEST_GENERIC) fail(SPTTN_EINVAL, "not a GENERIC plan");
    const int nb = p->prog->num_buffers;
    const auto& h = p->last_counters;  // filled by spttn_read_output
    if (static_cast<int>(h.size()) < nb + 3) fail(SPTTN_EINVAL, "read the output first");
    for (int b = 0; b < n && b < nb; ++b) out[b] = h[1 + b];
    if (h[2 + nb]) fail(SPTTN_ENOMEM, "observer log overflowed");
  });
}

int64_t spttn_generic_log_bytes(const spttn_plan* p) {
  if (!p || p->kind != SPTTN_NEST_GENERIC || !p->prog->observe) return 0;
  const int nb = p->prog->num_buffers;
  if (static_cast<int>(p->last_counters.size()) < nb + 2) return -1;
  return p->last_counters[1 + nb];
}

int spttn_generic_read_log(spttn_plan* p, void* host_out, int64_t bytes, void* stream) {
  return guarded([&] {
    if (!p || p->kind != SPTTN_NEST_GENERIC) fail(SPTTN_EINVAL, "not a GENERIC plan");
    if (bytes > p->gen.log_bytes) fail(SPTTN_EINVAL, "log read beyond capacity");
    if (bytes > 0)
      SPTTN_CUDA(cudaMemcpyAsync(host_out, p->gen.log, bytes, cudaMemcpyDeviceToHost,
                                 as_stream(stream)));
    SPTTN_CUDA(cudaStreamSynchronize(as_stream(stream)));
  });
}

int spttn_unfactorized(const spttn_unfact_desc* desc, spttn_csf* csf, double* host_out,
                       int64_t out_count, void* stream) {
  std::vector<double*> tmp;
  double* dout = nullptr;
  const int rc = guarded([&] {
    if (!desc || !csf) fail(SPTTN_EINVAL, "null argument");
    cudaStream_t s = as_stream(stream);
    csf->d.wait_values(s);
    if (desc->num_factors < 0 || desc->num_factors > 8) fail(SPTTN_EINVAL, "bad factor count");
    const double* dptr[8] = {nullptr};
    for (int f = 0; f < desc->num_factors; ++f) {
      int64_t n = 1;
      for (int k = 0; k < desc->factor_order[f]; ++k) n *= desc->dims[desc->factor_ids[f][k]];
      double* d = nullptr;
      dev_malloc(reinterpret_cast<void**>(&d), n * sizeof(double), s);
      tmp.push_back(d);
      SPTTN_CUDA(cudaMemcpyAsync(d, desc->factors[f], n * sizeof(double), cudaMemcpyHostToDevice, s));
      dptr[f] = d;
    }
    dev_malloc(reinterpret_cast<void**>(&dout), std::max<int64_t>(1, out_count) * sizeof(double), s);
    spttn_dev::unfactorized_run(desc, csf->d, dptr, dout, out_count, s);
    if (out_count)
      SPTTN_CUDA(cudaMemcpyAsync(host_out, dout, out_count * sizeof(double), cudaMemcpyDeviceToHost, s));
    SPTTN_CUDA(cudaStreamSynchronize(s));
  });
  cudaDeviceSynchronize();
  for (double* d : tmp) spttn_dev::dfree(d);
  spttn_dev::dfree(dout);
  return rc;
}

}  // extern "C"
