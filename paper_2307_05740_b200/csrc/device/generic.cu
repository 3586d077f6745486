// GENERIC device forest interpreter and the device execute_unfactorized.
//
// The interpreter runs any admissible fused loop forest (every order the
// reference planner can emit, including sparse-output nests that iterate
// modes densely) on the GPU. It walks the serialized program exactly like the
// reference's exec_node / exec_leaf / exec_hook (proj/src/executor.cpp:
// 389-490): same loop order, same reset points, same hook arithmetic, so the
// floating-point results are bit-identical to the reference and the
// multiply-add / reset counters are counted, not estimated. It is the
// coverage path (one device thread per plan; the pinned nests have dedicated
// kernels), used for non-pinned orders and small ranks.
//
// The unfactorized oracle (executor.cpp:522-626) runs one thread per output
// entry (dense output) or per leaf (sparse output); each thread accumulates
// its entry's contributions in the reference's order, so it is deterministic
// and bit-identical as well.
#include "../../../include/spttn_b200.h"
#include "internal.cuh"

namespace spttn_dev {

namespace {

struct Interp {
  const spg_program* P;
  CsfView t;
  const double* const* dense;
  double* out;
  double* bufs;
  const int64_t* boff;
  int64_t* counters;
  unsigned char* log;
  int64_t log_cap;
  const int64_t* leaf_keys;
  const int64_t* leaf_pos;
  int64_t nkeys;
  int64_t ival[SPG_MAX_IDX];
  int64_t pos[SPG_MAX_LEVELS];
  int64_t madds;

  __device__ int64_t offset(const spg_access& a) const {
    int64_t off = 0;
    for (int k = 0; k < a.naddr; ++k) off += ival[a.ids[k]] * a.strides[k];
    return off;
  }
  __device__ double* base(const spg_access& a) const {
    switch (a.kind) {
      case SPG_OP_DENSE: return const_cast<double*>(dense[a.slot]);
      case SPG_OP_BUFFER: return bufs + boff[a.slot];
      case SPG_OP_OUT_DENSE: return out;
      default: return nullptr;
    }
  }
  __device__ double read(const spg_access& a) const {
    if (a.kind == SPG_OP_SPARSE) return t.vals[pos[t.order - 1]];
    if (a.kind == SPG_OP_OUT_SPARSE) return 0.0;
    return base(a)[offset(a)];
  }

  __device__ void leaf(int term) {
    const double v = read(P->lhs[term]) * read(P->rhs[term]);
    madds += 2;
    const spg_access& o = P->out[term];
    if (o.kind == SPG_OP_OUT_SPARSE) {
      if (P->need_leaf_lookup) {
        int64_t key = 0;
        for (int l = 0; l < t.order; ++l) key += ival[P->sparse_mode_ids[l]] * P->mode_key_stride[l];
        int64_t lo = 0, hi = nkeys;
        while (lo < hi) {
          const int64_t mid = (lo + hi) >> 1;
          if (leaf_keys[mid] < key) lo = mid + 1; else hi = mid;
        }
        // off-pattern coordinates only produce exact zeros (executor.cpp:400)
        if (lo < nkeys && leaf_keys[lo] == key) out[leaf_pos ? leaf_pos[lo] : lo] += v;
      } else {
        out[pos[t.order - 1]] += v;
      }
      return;
    }
    base(o)[offset(o)] += v;
  }

  __device__ void hook(const spg_hook& h) {
    const int term = h.term;
    for (int k = 0; k < h.nspan; ++k) ival[h.span[k]] = 0;
    const spg_access& lhs = P->lhs[term];
    const spg_access& rhs = P->rhs[term];
    const spg_access& o = P->out[term];
    double* y = base(o) + offset(o);
    if (h.kind == SPG_HOOK_VEC) {
      const spg_access& vec = h.vec_is_lhs ? lhs : rhs;
      const spg_access& sca = h.vec_is_lhs ? rhs : lhs;
      const double alpha = read(sca);
      const double* x = base(vec) + offset(vec);
      // scaled_vector_accumulate (micro_kernels.hpp:11-14)
      for (int64_t i = 0; i < h.len; ++i) y[i * h.out_inc] += alpha * x[i * h.vec_inc];
      madds += 2 * h.len;
      return;
    }
    const spg_access& xa = h.x_is_lhs ? lhs : rhs;
    const spg_access& ya = h.x_is_lhs ? rhs : lhs;
    const double* x = base(xa) + offset(xa);
    const double* yv = base(ya) + offset(ya);
    // rank1_update (micro_kernels.hpp:17-23)
    for (int64_t i = 0; i < h.m; ++i) {
      const double xi = x[i * h.x_inc];
      for (int64_t j = 0; j < h.n; ++j) y[i * h.out_row + j * h.out_col] += xi * yv[j * h.y_inc];
    }
    madds += 2 * h.m * h.n;
  }

  __device__ void resets(const spg_node& nd) {
    for (int r = 0; r < nd.reset_count; ++r) {
      const int b = P->resets[nd.reset_begin + r];
      double* buf = bufs + boff[b];
      const int64_t n = P->buffer_size[b];
      for (int64_t i = 0; i < n; ++i) buf[i] = 0.0;
      atomicAdd(reinterpret_cast<unsigned long long*>(&counters[1 + b]), 1ull);
      if (P->observe) {
        int64_t* cursor = &counters[1 + P->num_buffers];
        const int64_t need = 16 + 8 * n;
        if (*cursor + need > log_cap) {
          counters[2 + P->num_buffers] = 1;  // overflow
        } else {
          int64_t* hdr = reinterpret_cast<int64_t*>(log + *cursor);
          hdr[0] = b;
          hdr[1] = n;
          double* dst = reinterpret_cast<double*>(hdr + 2);
          for (int64_t i = 0; i < n; ++i) dst[i] = buf[i];
          *cursor += need;
        }
      }
    }
  }
};

struct Frame {
  int node;
  int child;
  int64_t it, end;
};

__device__ void set_iter(Interp& I, const spg_node& nd, int64_t it) {
  if (nd.kind == SPG_SPARSE) {
    I.pos[nd.csf_level] = it;
    I.ival[nd.index] = I.t.idx[nd.csf_level][it];
  } else {
    I.ival[nd.index] = it;
  }
}

// Walks root node `root` of the forest like exec_node; a sparse level-0 root
// may be restricted to the iteration range [rlo, rhi) (parallel mode).
__device__ void walk(Interp& I, const spg_program* P, int root, int64_t rlo, int64_t rhi) {
  Frame st[SPG_MAX_IDX + 2];
  int sp = 0;
  int pending = root;
  bool top = true;
  for (;;) {
    if (pending >= 0) {
      const spg_node& nd = P->nodes[pending];
      I.resets(nd);
      if (nd.kind == SPG_LEAF) {
        I.leaf(nd.term);
      } else if (nd.hook >= 0) {
        I.hook(P->hooks[nd.hook]);
      } else {
        int64_t lo = 0, hi = 0;
        if (nd.kind == SPG_SPARSE) {
          if (nd.csf_level == 0) {
            hi = I.t.nlev[0];
            if (top && rlo >= 0) {
              lo = rlo;
              hi = rhi;
            }
          } else {
            lo = I.t.ptr[nd.csf_level - 1][I.pos[nd.csf_level - 1]];
            hi = I.t.ptr[nd.csf_level - 1][I.pos[nd.csf_level - 1] + 1];
          }
        } else {
          hi = P->dims[nd.index];
        }
        if (lo < hi) {
          st[sp++] = Frame{pending, 0, lo, hi};
          set_iter(I, nd, lo);
        }
      }
      pending = -1;
      top = false;
    }
    if (sp == 0) break;
    Frame& f = st[sp - 1];
    const spg_node& fn = P->nodes[f.node];
    if (f.child < fn.child_count) {
      pending = P->children[fn.child_begin + f.child];
      ++f.child;
      continue;
    }
    ++f.it;
    if (f.it < f.end) {
      f.child = 0;
      set_iter(I, fn, f.it);
    } else {
      --sp;
    }
  }
}

__device__ void stage_program(const spg_program* src_prog, unsigned char* smem) {
  const int4* src = reinterpret_cast<const int4*>(src_prog);
  int4* dst = reinterpret_cast<int4*>(smem);
  for (size_t w = threadIdx.x; w < sizeof(spg_program) / sizeof(int4); w += blockDim.x)
    dst[w] = src[w];
  __syncthreads();
}

// Sequential interpreter: the program (~23 KB) is staged into shared memory by
// the whole block so the interpreting thread reads node / operand / hook
// tables at shared-memory latency instead of global-memory latency.
__global__ void __launch_bounds__(256) k_generic(Interp I) {
  extern __shared__ __align__(16) unsigned char prog_smem[];
  stage_program(I.P, prog_smem);
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  const spg_program* P = reinterpret_cast<const spg_program*>(prog_smem);
  I.P = P;
  for (int k = 0; k < SPG_MAX_IDX; ++k) I.ival[k] = 0;
  for (int k = 0; k < SPG_MAX_LEVELS; ++k) I.pos[k] = 0;
  I.madds = 0;
  for (int ri = 0; ri < P->num_roots; ++ri) walk(I, P, P->roots[ri], -1, -1);
  I.counters[0] = I.madds;
}

// Parallel interpreter over the root slices of a forest whose single root is
// the CSF level-0 loop with no resets of its own (so iterations share no
// buffer state). Every thread is a worker with private buffers.
//  mode 1 (outputs disjoint across root slices: indexed by the root mode, or
//          sparse): workers take root slices dynamically and write the output
//          directly — each slice is computed exactly as in the sequential
//          walk, so results are bit-identical to it.
//  mode 2 (dense output not indexed by the root mode, e.g. MTTKRP for mode
//          j): worker w walks the fixed root range [w*n0/W, (w+1)*n0/W) into
//          a private output copy; k_generic_reduce adds the copies in worker
//          order (deterministic; grouping differs from the sequential sum).
__global__ void __launch_bounds__(256) k_generic_par(Interp I0, int mode, int64_t workers,
                                                     int64_t buf_elems, double* priv,
                                                     int64_t out_size) {
  extern __shared__ __align__(16) unsigned char prog_smem[];
  stage_program(I0.P, prog_smem);
  const int64_t w = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (w >= workers) return;
  const spg_program* P = reinterpret_cast<const spg_program*>(prog_smem);
  Interp I = I0;
  I.P = P;
  I.bufs = I0.bufs + w * buf_elems;
  if (mode == 2) I.out = priv + w * out_size;
  for (int k = 0; k < SPG_MAX_IDX; ++k) I.ival[k] = 0;
  for (int k = 0; k < SPG_MAX_LEVELS; ++k) I.pos[k] = 0;
  I.madds = 0;
  const int root = P->roots[0];
  const int64_t n0 = I.t.nlev[0];
  if (mode == 1) {
    unsigned long long* next =
        reinterpret_cast<unsigned long long*>(&I.counters[P->num_buffers + 3]);
    for (;;) {
      const int64_t sl = static_cast<int64_t>(atomicAdd(next, 1ull));
      if (sl >= n0) break;
      walk(I, P, root, sl, sl + 1);
    }
  } else {
    const int64_t lo = w * n0 / workers, hi = (w + 1) * n0 / workers;
    if (lo < hi) walk(I, P, root, lo, hi);
  }
  atomicAdd(reinterpret_cast<unsigned long long*>(&I.counters[0]),
            static_cast<unsigned long long>(I.madds));
}

__global__ void k_generic_reduce(const double* priv, int64_t workers, int64_t out_size,
                                 double* out) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= out_size) return;
  double sum = 0.0;
  for (int64_t w = 0; w < workers; ++w) sum += priv[w * out_size + e];
  out[e] = sum;
}

// ---- small plans: the whole working set in shared memory -------------------
//
// The global-memory interpreter above is latency bound on tiny tensors (the
// regime of the reference's acceptance criterion 6: every admissible order of
// 10-100-nonzero fixtures): each buffer / output update is a store followed by
// a load of the same word, i.e. an L2 round trip per multiply-add. When the
// program, the CSF, the dense inputs, the intermediate buffers and the output
// together fit one CTA's shared memory, the CTA stages them there (all
// threads, coalesced), walks the forest out of shared memory, and writes the
// output and counters back once. Same walk, same arithmetic (no FMA
// contraction in this file): results stay bit-identical to the reference.
// Root slices go to up to 8 walkers (thread 0 of each warp) only where the
// global interpreter's mode 1 would (disjoint outputs, no root resets).

enum SmSlot {
  kSmProg = 0, kSmBoff, kSmDenseTab, kSmBufs, kSmOut, kSmCnt, kSmVals, kSmKeys,
  kSmIdx = 8,                       // + level
  kSmPtr = 8 + SPG_MAX_LEVELS,      // + level
  kSmDense = 8 + 2 * SPG_MAX_LEVELS,  // + dense slot (1..)
  kSmSlots = kSmDense + SPG_MAX_DENSE
};
static_assert(kSmSlots <= 48, "GenericState::sm_off capacity");

struct SmArgs {
  const spg_program* P;
  const int64_t* boff;
  CsfView t;
  const double* dense[SPG_MAX_DENSE];
  int64_t dense_size[SPG_MAX_DENSE];
  double* out;
  int64_t* counters;
  int64_t buf_elems;
  int32_t off[48];
  int32_t workers;
};

bool generic_sm_layout_impl(const spg_program& G, const DevCsf& csf, int workers, int64_t limit,
                            GenericState& g) {
  int64_t cur = 0;
  auto take = [&](int slot, int64_t bytes) {
    g.sm_off[slot] = static_cast<int32_t>(cur);
    cur += (bytes + 15) & ~int64_t{15};
  };
  const int nb = G.num_buffers;
  int64_t buf_elems = 0;
  for (int b = 0; b < nb; ++b) buf_elems += G.buffer_size[b];
  take(kSmProg, sizeof(spg_program));
  take(kSmBoff, (nb + 1) * 8);
  take(kSmDenseTab, SPG_MAX_DENSE * 8);
  take(kSmBufs, std::max<int64_t>(1, buf_elems) * workers * 8);
  take(kSmOut, std::max<int64_t>(1, G.out_size) * 8);
  take(kSmCnt, (nb + 4) * 8);
  const int d = csf.order;
  const int64_t nnz = d > 0 ? csf.level_size[d - 1] : 0;
  take(kSmVals, std::max<int64_t>(1, nnz) * 8);
  take(kSmKeys, G.need_leaf_lookup ? std::max<int64_t>(1, nnz) * 8 : 0);
  for (int l = 0; l < d; ++l) {
    take(kSmIdx + l, std::max<int64_t>(1, csf.level_size[l]) * 4);
    if (l + 1 < d) take(kSmPtr + l, (csf.level_size[l] + 1) * 4);
  }
  for (int f = 1; f <= G.num_dense && f < SPG_MAX_DENSE; ++f) take(kSmDense + f, G.dense_size[f] * 8);
  if (cur > limit) return false;
  g.sm_bytes = cur;
  g.sm_workers = workers;
  for (int f = 0; f < SPG_MAX_DENSE; ++f) g.dense_size[f] = (f >= 1 && f <= G.num_dense) ? G.dense_size[f] : 0;
  return true;
}

__device__ __forceinline__ void sm_copy(void* dst, const void* src, int64_t bytes) {
  // 8-byte words; every staged array is 8-byte sized except the int32 CSF
  // arrays, which are copied as int32
  const double* s = static_cast<const double*>(src);
  double* o = static_cast<double*>(dst);
  for (int64_t w = threadIdx.x; w < bytes / 8; w += blockDim.x) o[w] = s[w];
}

__device__ __forceinline__ void sm_copy32(int32_t* dst, const int32_t* src, int64_t n) {
  for (int64_t w = threadIdx.x; w < n; w += blockDim.x) dst[w] = src[w];
}

__global__ void __launch_bounds__(256) k_generic_sm(SmArgs a) {
  extern __shared__ __align__(16) unsigned char sm[];
  const spg_program* P = reinterpret_cast<const spg_program*>(sm + a.off[kSmProg]);
  {
    const int4* src = reinterpret_cast<const int4*>(a.P);
    int4* dst = reinterpret_cast<int4*>(sm + a.off[kSmProg]);
    for (int w = threadIdx.x; w < static_cast<int>(sizeof(spg_program) / sizeof(int4)); w += blockDim.x)
      dst[w] = src[w];
  }
  const int d = a.t.order;
  CsfView t{};
  t.order = d;
  for (int l = 0; l < d; ++l) {
    t.nlev[l] = a.t.nlev[l];
    int32_t* idx = reinterpret_cast<int32_t*>(sm + a.off[kSmIdx + l]);
    sm_copy32(idx, a.t.idx[l], a.t.nlev[l]);
    t.idx[l] = idx;
    if (l + 1 < d) {
      int32_t* ptr = reinterpret_cast<int32_t*>(sm + a.off[kSmPtr + l]);
      sm_copy32(ptr, a.t.ptr[l], a.t.nlev[l] + 1);
      t.ptr[l] = ptr;
    }
  }
  const int64_t nnz = d > 0 ? a.t.nlev[d - 1] : 0;
  double* vals = reinterpret_cast<double*>(sm + a.off[kSmVals]);
  sm_copy(vals, a.t.vals, nnz * 8);
  t.vals = vals;
  const double** tab = reinterpret_cast<const double**>(sm + a.off[kSmDenseTab]);
  for (int f = 1; f < SPG_MAX_DENSE; ++f) {
    if (a.dense_size[f] <= 0) continue;
    double* dst = reinterpret_cast<double*>(sm + a.off[kSmDense + f]);
    sm_copy(dst, a.dense[f], a.dense_size[f] * 8);
  }
  if (threadIdx.x < SPG_MAX_DENSE)
    tab[threadIdx.x] = a.dense_size[threadIdx.x] > 0
                           ? reinterpret_cast<const double*>(sm + a.off[kSmDense + threadIdx.x])
                           : nullptr;
  __syncthreads();  // program staged: sizes below come from it
  const int nb = P->num_buffers;
  int64_t* boff = reinterpret_cast<int64_t*>(sm + a.off[kSmBoff]);
  sm_copy(boff, a.boff, (nb + 1) * 8);
  double* bufs = reinterpret_cast<double*>(sm + a.off[kSmBufs]);
  for (int64_t w = threadIdx.x; w < a.buf_elems * a.workers; w += blockDim.x) bufs[w] = 0.0;
  double* out = reinterpret_cast<double*>(sm + a.off[kSmOut]);
  for (int64_t w = threadIdx.x; w < P->out_size; w += blockDim.x) out[w] = 0.0;
  int64_t* cnt = reinterpret_cast<int64_t*>(sm + a.off[kSmCnt]);
  for (int w = threadIdx.x; w < nb + 4; w += blockDim.x) cnt[w] = 0;
  int64_t* keys = P->need_leaf_lookup ? reinterpret_cast<int64_t*>(sm + a.off[kSmKeys]) : nullptr;
  __syncthreads();  // CSF staged: leaf keys (sorted by construction) from it
  if (keys)
    for (int64_t leaf = threadIdx.x; leaf < nnz; leaf += blockDim.x) {
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
    }
  __syncthreads();
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0 && w < a.workers) {
    Interp I{};
    I.P = P;
    I.t = t;
    I.dense = tab;
    I.out = out;
    I.bufs = bufs + w * a.buf_elems;
    I.boff = boff;
    I.counters = cnt;
    I.log = nullptr;
    I.log_cap = 0;
    I.leaf_keys = keys;
    I.leaf_pos = nullptr;
    I.nkeys = keys ? nnz : 0;
    for (int k = 0; k < SPG_MAX_IDX; ++k) I.ival[k] = 0;
    for (int k = 0; k < SPG_MAX_LEVELS; ++k) I.pos[k] = 0;
    I.madds = 0;
    if (a.workers == 1) {
      for (int ri = 0; ri < P->num_roots; ++ri) walk(I, P, P->roots[ri], -1, -1);
    } else {  // disjoint root slices, fixed round-robin assignment
      const int64_t n0 = t.nlev[0];
      for (int64_t sl = w; sl < n0; sl += a.workers) walk(I, P, P->roots[0], sl, sl + 1);
    }
    atomicAdd(reinterpret_cast<unsigned long long*>(&cnt[0]),
              static_cast<unsigned long long>(I.madds));
  }
  __syncthreads();
  for (int64_t e = threadIdx.x; e < P->out_size; e += blockDim.x) a.out[e] = out[e];
  for (int k = threadIdx.x; k < nb + 4; k += blockDim.x) a.counters[k] = cnt[k];
}

// ---- unfactorized ---------------------------------------------------------

struct Unf {
  spttn_unfact_desc d;
  CsfView t;
  const double* dense[8];
  double* out;
  int64_t out_count;
};

__device__ double unf_body(const Unf& u, const int64_t* ival, int64_t leaf) {
  double v = u.t.vals[leaf];
  for (int f = 0; f < u.d.num_factors; ++f) {
    int64_t off = 0;
    for (int k = 0; k < u.d.factor_order[f]; ++k) {
      const int id = u.d.factor_ids[f][k];
      off = off * u.d.dims[id] + ival[id];
    }
    v *= u.dense[f][off];
  }
  return v;
}

// Dense output: one thread per output entry; walks the CSF in order and the
// non-output free indices in first-appearance order.
__global__ void k_unf_dense(Unf u) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= u.out_count) return;
  int64_t ival[32];
  for (int k = 0; k < 32; ++k) ival[k] = 0;
  bool fixed[32];
  for (int k = 0; k < 32; ++k) fixed[k] = false;
  int64_t rest = e;
  for (int q = u.d.out_order - 1; q >= 0; --q) {
    const int id = u.d.out_ids[q];
    ival[id] = rest % u.d.dims[id];
    rest /= u.d.dims[id];
    fixed[id] = true;
  }
  // non-output free indices, in first-appearance order
  int loop_ids[32];
  int nloop = 0;
  int64_t loop_total = 1;
  for (int q = 0; q < u.d.num_free; ++q) {
    const int id = u.d.free_ids[q];
    if (!fixed[id]) {
      loop_ids[nloop++] = id;
      loop_total *= u.d.dims[id];
    }
  }
  const int d = u.t.order;
  // root restriction when the output carries the level-0 mode
  int64_t r_lo = 0, r_hi = u.t.nlev[0];
  int root_id = -1;
  for (int id = 0; id < u.d.num_indices; ++id)
    if (u.d.csf_level[id] == 0) root_id = id;
  if (root_id >= 0 && fixed[root_id]) {
    int64_t lo = 0, hi = u.t.nlev[0];
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (u.t.idx[0][mid] < ival[root_id]) lo = mid + 1; else hi = mid;
    }
    if (lo < u.t.nlev[0] && u.t.idx[0][lo] == ival[root_id]) {
      r_lo = lo;
      r_hi = lo + 1;
    } else {
      u.out[e] = 0.0;
      return;
    }
  }
  int lvl_id[8];
  for (int id = 0; id < u.d.num_indices; ++id)
    if (u.d.csf_level[id] >= 0) lvl_id[u.d.csf_level[id]] = id;
  double sum = 0.0;
  int64_t pos[8], hi[8];
  int lvl = 0;
  pos[0] = r_lo;
  hi[0] = r_hi;
  while (true) {
    if (pos[lvl] >= hi[lvl]) {
      if (lvl == 0) break;
      --lvl;
      ++pos[lvl];
      continue;
    }
    const int id = lvl_id[lvl];
    const int64_t coord = u.t.idx[lvl][pos[lvl]];
    if (fixed[id] && coord != ival[id]) {
      ++pos[lvl];
      continue;
    }
    ival[id] = coord;
    if (lvl + 1 < d) {
      pos[lvl + 1] = u.t.ptr[lvl][pos[lvl]];
      hi[lvl + 1] = u.t.ptr[lvl][pos[lvl] + 1];
      ++lvl;
      continue;
    }
    for (int64_t f = 0; f < loop_total; ++f) {
      int64_t r = f;
      for (int q = nloop - 1; q >= 0; --q) {
        ival[loop_ids[q]] = r % u.d.dims[loop_ids[q]];
        r /= u.d.dims[loop_ids[q]];
      }
      sum += unf_body(u, ival, pos[lvl]);
    }
    ++pos[lvl];
  }
  u.out[e] = sum;
}

// Sparse output: one thread per leaf.
__global__ void k_unf_sparse(Unf u, const int32_t* leaf_parent /* unused */) {
  const int64_t leaf = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int d = u.t.order;
  if (leaf >= u.t.nlev[d - 1]) return;
  int64_t ival[32];
  for (int k = 0; k < 32; ++k) ival[k] = 0;
  int lvl_id[8];
  for (int id = 0; id < u.d.num_indices; ++id)
    if (u.d.csf_level[id] >= 0) lvl_id[u.d.csf_level[id]] = id;
  // coordinates of the leaf: parent search level by level
  int64_t node = leaf;
  for (int l = d - 1; l >= 0; --l) {
    ival[lvl_id[l]] = u.t.idx[l][node];
    if (l > 0) {
      int64_t lo = 0, hi = u.t.nlev[l - 1];
      while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (u.t.ptr[l - 1][mid] <= node) lo = mid; else hi = mid;
      }
      node = lo;
    }
  }
  int64_t total = 1;
  for (int q = 0; q < u.d.num_free; ++q) total *= u.d.dims[u.d.free_ids[q]];
  double sum = 0.0;
  for (int64_t f = 0; f < total; ++f) {
    int64_t r = f;
    for (int q = u.d.num_free - 1; q >= 0; --q) {
      const int id = u.d.free_ids[q];
      ival[id] = r % u.d.dims[id];
      r /= u.d.dims[id];
    }
    sum += unf_body(u, ival, leaf);
  }
  u.out[leaf] = sum;
}

}  // namespace

bool generic_sm_layout(const spg_program& G, const DevCsf& csf, int workers, int64_t limit,
                       GenericState& g) {
  return generic_sm_layout_impl(G, csf, workers, limit, g);
}

void generic_execute(const spg_program& prog, const DevCsf& csf, const double* const* dense,
                     double* out, GenericState& g, cudaStream_t s) {
  if (g.sm) {
    // every input is staged by the kernel and the output / counters are
    // written in full: no memset, one launch
    SmArgs a{};
    a.P = g.d_prog;
    a.boff = g.buffer_off;
    a.t = csf.view();
    for (int f = 0; f < SPG_MAX_DENSE; ++f) {
      a.dense[f] = g.dense_dev[f];
      a.dense_size[f] = a.dense[f] ? g.dense_size[f] : 0;
    }
    a.out = out;
    a.counters = g.counters;
    a.buf_elems = g.total_buffer_elems;
    for (int k = 0; k < 48; ++k) a.off[k] = g.sm_off[k];
    a.workers = g.sm_workers;
    static int configured = -1;
    int dev = 0;
    SPTTN_CUDA(cudaGetDevice(&dev));
    if (configured != dev) {  // opt in to the large dynamic shared memory once per device
      SPTTN_CUDA(cudaFuncSetAttribute(k_generic_sm, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      227 * 1024));
      configured = dev;
    }
    k_generic_sm<<<1, 256, static_cast<size_t>(g.sm_bytes), s>>>(a);
    SPTTN_CUDA(cudaGetLastError());
    return;
  }
  // counters, buffers and output are contiguous in the plan arena
  SPTTN_CUDA(cudaMemsetAsync(g.counters, 0, g.zero_bytes, s));
  Interp I{};
  I.P = g.d_prog;
  I.t = csf.view();
  I.dense = dense;
  I.out = out;
  I.bufs = g.buffers;
  I.boff = g.buffer_off;
  I.counters = g.counters;
  I.log = g.log;
  I.log_cap = g.log_bytes;
  I.leaf_keys = g.leaf_keys;
  I.leaf_pos = g.leaf_pos;
  I.nkeys = g.n_leaf_keys;
  static_assert(sizeof(spg_program) % sizeof(int4) == 0, "program must be int4-copyable");
  static_assert(sizeof(spg_program) <= 48 * 1024, "program must fit default shared memory");
  if (g.tail || g.par_mode > 2) throw Status(SPTTN_EINVAL, "JIT-only decomposition without a JIT kernel");
  if (g.par_mode == 0) {
    k_generic<<<1, 256, sizeof(spg_program), s>>>(I);
  } else {
    const unsigned blocks = static_cast<unsigned>((g.workers + 127) / 128);
    k_generic_par<<<blocks, 128, sizeof(spg_program), s>>>(I, g.par_mode, g.workers,
                                                           g.total_buffer_elems, g.priv_out,
                                                           g.out_size);
    if (g.par_mode == 2)
      k_generic_reduce<<<static_cast<unsigned>((g.out_size + 255) / 256), 256, 0, s>>>(
          g.priv_out, g.workers, g.out_size, out);
  }
  SPTTN_CUDA(cudaGetLastError());
}

void generic_reduce(const GenericState& g, double* out, cudaStream_t s) {
  k_generic_reduce<<<static_cast<unsigned>((g.out_size + 255) / 256), 256, 0, s>>>(
      g.priv_out, g.workers, g.out_size, out);
  SPTTN_CUDA(cudaGetLastError());
}

// worker 0's copy of each accumulator = sum over workers, in worker order
__global__ void k_buffer_reduce(double* bufs, int64_t workers, int64_t stride, int64_t off,
                                int64_t n) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= n) return;
  double sum = 0.0;
  for (int64_t w = 0; w < workers; ++w) sum += bufs[w * stride + off + e];
  bufs[off + e] = sum;
}

void generic_reduce_buffers(const GenericState& g, cudaStream_t s) {
  for (int i = 0; i < g.n_tail_bufs; ++i) {
    if (g.tail_len[i] <= 0) continue;
    k_buffer_reduce<<<static_cast<unsigned>((g.tail_len[i] + 127) / 128), 128, 0, s>>>(
        g.buffers, g.workers, g.total_buffer_elems, g.tail_off[i], g.tail_len[i]);
  }
  SPTTN_CUDA(cudaGetLastError());
}

void generic_free(GenericState& g) {
  if (g.in_arena) {  // owned by the plan arena
    g = GenericState{};
    return;
  }
  dfree(g.d_prog);
  dfree(g.buffers);
  dfree(g.buffer_off);
  dfree(g.counters);
  dfree(g.log);
  dfree(g.leaf_keys);
  dfree(g.leaf_pos);
  g = GenericState{};
}

void unfactorized_run(const void* desc, const DevCsf& csf, const double* const* dense,
                      double* out, int64_t out_count, cudaStream_t s) {
  Unf u{};
  u.d = *static_cast<const spttn_unfact_desc*>(desc);
  u.t = csf.view();
  for (int f = 0; f < u.d.num_factors; ++f) u.dense[f] = dense[f];
  u.out = out;
  u.out_count = out_count;
  if (out_count == 0) return;
  const unsigned blocks = static_cast<unsigned>((out_count + 127) / 128);
  if (u.d.out_sparse)
    k_unf_sparse<<<blocks, 128, 0, s>>>(u, nullptr);
  else
    k_unf_dense<<<blocks, 128, 0, s>>>(u);
  SPTTN_CUDA(cudaGetLastError());
}

}  // namespace spttn_dev
