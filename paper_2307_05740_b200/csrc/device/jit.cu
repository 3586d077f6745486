// Fused-nest JIT: any admissible forest — TTTc chains and
// every order the planners emit that has no dedicated kernel — compiled to a
// specialised sm_100a kernel at plan time instead of being interpreted.
//
// The generator walks the same serialized program the interpreter runs
// (program.h, built by the shim from the reference's FusedLoopForest with
// prepare()'s addressing, resets and hooks, executor.cpp:191-366) and emits
// straight-line C++: one `for` per forest vertex (CSF child ranges for sparse
// vertices, [0, dim) for dense ones), buffer resets at vertex entry, the
// leaf `out[off] += lhs[off] * rhs[off]` and the two hook micro-kernels
// (micro_kernels.hpp:11-23) with every stride, dimension and buffer offset a
// literal. The arithmetic and its order are exactly the interpreter's
// (exec_node / exec_leaf / exec_hook) and, compiled without FMA contraction
// like the interpreter, its results are bit-identical to it; counters
// (multiply-adds, resets) are counted the same way. Work is distributed like the parallel interpreter (generic.cu):
// root slices to worker threads with private buffers, outputs written
// directly when root-indexed / sparse, per-worker copies reduced in worker
// order otherwise, one thread for the rest. NVRTC compiles each distinct
// source once per process (cache keyed by the source text); the CUBIN is
// loaded with cudaLibraryLoadData.
#include <nvrtc.h>

#include <mutex>
#include <sstream>
#include <string>
#include <cstdlib>
#include <cstdio>
#include <unordered_map>
#include <vector>

#include "../../../include/spttn_b200.h"
#include "internal.cuh"

namespace spttn_dev {

namespace {

struct JitArgs {
  const int32_t* idx[kMaxOrder];
  const int32_t* ptr[kMaxOrder];
  int32_t nlev[kMaxOrder];
  const double* vals;
  const double* const* dense;
  double* out;
  double* bufs;
  int64_t buf_elems;
  double* priv;
  int64_t out_size;
  int64_t workers;
  int64_t* counters;
  const int64_t* leaf_keys;
  const int64_t* leaf_pos;
  int64_t nkeys;
  int64_t phase;
};

class Gen {
 public:
  Gen(const spg_program& P, const GenericState& g) : P_(P), mode_(g.par_mode), g_(g) {}

  std::string source() {
    std::ostringstream o;
    o << "typedef long long int64_t;\ntypedef int int32_t;\n"
         "struct JitArgs { const int32_t* idx[8]; const int32_t* ptr[8]; int32_t nlev[8];\n"
         "  const double* vals; const double* const* dense; double* out; double* bufs;\n"
         "  int64_t buf_elems; double* priv; int64_t out_size; int64_t workers;\n"
         "  int64_t* counters; const int64_t* leaf_keys; const int64_t* leaf_pos; int64_t nkeys;\n"
         "  int64_t phase; };\n"
         "extern \"C\" __global__ void __launch_bounds__(128) spg_nest(JitArgs a) {\n"
         "  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;\n"
         "  if (w >= a.workers) return;\n";
    for (int l = 0; l < P_.csf_order; ++l)
      o << "  const int32_t* __restrict__ idx" << l << " = a.idx[" << l << "];\n";
    for (int l = 0; l + 1 < P_.csf_order; ++l)
      o << "  const int32_t* __restrict__ ptr" << l << " = a.ptr[" << l << "];\n";
    o << "  const double* __restrict__ vals = a.vals;\n";
    if (g_.priv && g_.tail)
      o << "  double* out = a.phase == 0 ? a.priv + w * a.out_size : a.out;\n";
    else
      o << "  double* out = " << (g_.priv ? "a.priv + w * a.out_size" : "a.out") << ";\n";
    int64_t off = 0;
    for (int b = 0; b < P_.num_buffers; ++b) {
      o << "  double* B" << b << " = a.bufs + w * a.buf_elems + " << off << "LL;\n";
      off += P_.buffer_size[b];
    }
    for (int f = 1; f <= 15; ++f)
      if (P_.dense_size[f] > 0) o << "  const double* __restrict__ D" << f << " = a.dense[" << f << "];\n";
    o << "  int64_t madds = 0;\n";
    for (int b = 0; b < P_.num_buffers; ++b) o << "  int64_t rs" << b << " = 0;\n";
    // index values and CSF positions persist across vertices, as in the
    // interpreter's ival[] / pos[]
    o << "  int64_t ";
    for (int k = 0; k < P_.num_indices; ++k) o << (k ? ", " : "") << "v" << k << " = 0";
    o << ";\n  int64_t ";
    for (int l = 0; l < P_.csf_order; ++l) o << (l ? ", " : "") << "p" << l << " = 0";
    o << ";\n";
    o << "  (void)vals; (void)out;\n";
    if (mode_ == 0) {
      for (int r = 0; r < P_.num_roots; ++r) emit_node(o, P_.roots[r], 1, false);
    } else {
      if (g_.tail) o << "  if (a.phase == 0) {\n";
      emit_parallel_root(o);
      if (g_.tail) {
        o << "  } else {\n";
        for (int r = 1; r < P_.num_roots; ++r) emit_node(o, P_.roots[r], 2, false);
        o << "  }\n";
      }
    }
    o << "  atomicAdd((unsigned long long*)&a.counters[0], (unsigned long long)madds);\n";
    for (int b = 0; b < P_.num_buffers; ++b)
      o << "  if (rs" << b << ") atomicAdd((unsigned long long*)&a.counters[" << 1 + b
        << "], (unsigned long long)rs" << b << ");\n";
    o << "}\n";
    return o.str();
  }

 private:
  const spg_program& P_;
  int mode_;
  const GenericState& g_;

  // Root 0 restricted to this worker's work units: atomically claimed root
  // slices (mode 1), a static range of slices (mode 2) or of level-1
  // fibers (mode 3, p0 follows along). Root-level resets zero each worker's
  // private accumulators; only worker 0 counts them (they happen once in
  // the sequential walk).
  void emit_parallel_root(std::ostringstream& o) {
    const spg_node& root = P_.nodes[P_.roots[0]];
    if (mode_ == 3) {
      const spg_node& l1 = P_.nodes[P_.children[root.child_begin]];
      emit_resets(o, root, 1, true);
      o << "  {\n"
           "    const int64_t n1 = a.nlev[1];\n"
           "    const int64_t flo = w * n1 / a.workers, fhi = (w + 1) * n1 / a.workers;\n"
           "    if (flo < fhi) {\n"
           "      int64_t lo = 0, hi = a.nlev[0];\n"
           "      while (hi - lo > 1) { const int64_t mid = (lo + hi) >> 1;"
           " if (ptr0[mid] <= flo) lo = mid; else hi = mid; }\n"
           "      p0 = lo;\n"
           "      v" << root.index << " = idx0[p0];\n"
           "      for (p1 = flo; p1 < fhi; ++p1) {\n"
           "        while (ptr0[p0 + 1] <= p1) { ++p0; v" << root.index << " = idx0[p0]; }\n"
           "        v" << l1.index << " = idx1[p1];\n";
      for (int c = 0; c < l1.child_count; ++c) emit_node(o, P_.children[l1.child_begin + c], 4, false);
      o << "      }\n    }\n  }\n";
      return;
    }
    if (mode_ == 1) {
      o << "  for (;;) {\n"
           "    const int64_t r = (int64_t)atomicAdd((unsigned long long*)&a.counters["
        << P_.num_buffers + 3 << "], 1ULL);\n"
           "    if (r >= a.nlev[0]) break;\n"
           "    const int64_t rlo = r, rhi = r + 1;\n";
    } else {
      o << "  {\n    const int64_t rlo = w * a.nlev[0] / a.workers, rhi = (w + 1) * a.nlev[0] / a.workers;\n";
    }
    emit_node(o, P_.roots[0], 2, true);
    o << "  }\n";
  }

  void emit_resets(std::ostringstream& o, const spg_node& nd, int d, bool once) {
    for (int r = 0; r < nd.reset_count; ++r) {
      const int b = P_.resets[nd.reset_begin + r];
      o << ind(d) << "for (int64_t e = 0; e < " << P_.buffer_size[b] << "LL; ++e) B" << b
        << "[e] = 0.0;\n"
        << ind(d) << (once ? "if (w == 0) " : "") << "++rs" << b << ";\n";
    }
  }

  static std::string ind(int d) { return std::string(2 * d, ' '); }

  std::string offset(const spg_access& a) const {
    std::ostringstream o;
    o << "(0LL";
    for (int k = 0; k < a.naddr; ++k)
      if (a.strides[k] != 0) o << " + v" << a.ids[k] << " * " << a.strides[k] << "LL";
    o << ")";
    return o.str();
  }
  std::string base(const spg_access& a) const {
    switch (a.kind) {
      case SPG_OP_DENSE: return "D" + std::to_string(a.slot);
      case SPG_OP_BUFFER: return "B" + std::to_string(a.slot);
      case SPG_OP_OUT_DENSE: return "out";
      default: return "";
    }
  }
  std::string read(const spg_access& a) const {
    if (a.kind == SPG_OP_SPARSE) return "vals[p" + std::to_string(P_.csf_order - 1) + "]";
    if (a.kind == SPG_OP_OUT_SPARSE) return "0.0";
    return base(a) + "[" + offset(a) + "]";
  }

  void emit_node(std::ostringstream& o, int v, int d, bool top) {
    const spg_node& nd = P_.nodes[v];
    emit_resets(o, nd, d, top);
    if (nd.kind == SPG_LEAF) {
      emit_leaf(o, nd.term, d);
      return;
    }
    if (nd.hook >= 0) {
      emit_hook(o, P_.hooks[nd.hook], d);
      return;
    }
    const std::string var = "v" + std::to_string(nd.index);
    if (nd.kind == SPG_SPARSE) {
      const int l = nd.csf_level;
      const std::string p = "p" + std::to_string(l);
      if (l == 0) {
        if (top)
          o << ind(d) << "for (" << p << " = rlo; " << p << " < rhi; ++" << p << ") {\n";
        else
          o << ind(d) << "for (" << p << " = 0; " << p << " < a.nlev[0]; ++" << p << ") {\n";
      } else {
        const std::string pp = "p" + std::to_string(l - 1);
        o << ind(d) << "for (" << p << " = ptr" << l - 1 << "[" << pp << "]; " << p << " < ptr"
          << l - 1 << "[" << pp << " + 1]; ++" << p << ") {\n";
      }
      o << ind(d + 1) << var << " = idx" << l << "[" << p << "];\n";
    } else {
      o << ind(d) << "for (" << var << " = 0; " << var << " < " << P_.dims[nd.index] << "LL; ++"
        << var << ") {\n";
    }
    for (int c = 0; c < nd.child_count; ++c) emit_node(o, P_.children[nd.child_begin + c], d + 1, false);
    o << ind(d) << "}\n";
  }

  void emit_leaf(std::ostringstream& o, int term, int d) {
    const spg_access& lhs = P_.lhs[term];
    const spg_access& rhs = P_.rhs[term];
    const spg_access& out = P_.out[term];
    o << ind(d) << "{\n"
      << ind(d + 1) << "const double val = " << read(lhs) << " * " << read(rhs) << ";\n"
      << ind(d + 1) << "madds += 2;\n";
    if (out.kind == SPG_OP_OUT_SPARSE) {
      if (P_.need_leaf_lookup) {
        o << ind(d + 1) << "int64_t key = 0";
        for (int l = 0; l < P_.csf_order; ++l)
          o << " + v" << P_.sparse_mode_ids[l] << " * " << P_.mode_key_stride[l] << "LL";
        o << ";\n"
          << ind(d + 1) << "int64_t lo = 0, hi = a.nkeys;\n"
          << ind(d + 1) << "while (lo < hi) { const int64_t mid = (lo + hi) >> 1;"
                           " if (a.leaf_keys[mid] < key) lo = mid + 1; else hi = mid; }\n"
          << ind(d + 1) << "if (lo < a.nkeys && a.leaf_keys[lo] == key) out[a.leaf_pos[lo]] += val;\n";
      } else {
        o << ind(d + 1) << "out[p" << P_.csf_order - 1 << "] += val;\n";
      }
    } else {
      o << ind(d + 1) << base(out) << "[" << offset(out) << "] += val;\n";
    }
    o << ind(d) << "}\n";
  }

  void emit_hook(std::ostringstream& o, const spg_hook& h, int d) {
    const spg_access& lhs = P_.lhs[h.term];
    const spg_access& rhs = P_.rhs[h.term];
    const spg_access& out = P_.out[h.term];
    o << ind(d) << "{\n";
    for (int k = 0; k < h.nspan; ++k) o << ind(d + 1) << "v" << h.span[k] << " = 0;\n";
    o << ind(d + 1) << "double* y = " << base(out) << " + " << offset(out) << ";\n";
    if (h.kind == SPG_HOOK_VEC) {
      const spg_access& vec = h.vec_is_lhs ? lhs : rhs;
      const spg_access& sca = h.vec_is_lhs ? rhs : lhs;
      o << ind(d + 1) << "const double alpha = " << read(sca) << ";\n"
        << ind(d + 1) << "const double* x = " << base(vec) << " + " << offset(vec) << ";\n"
        << ind(d + 1) << "for (int64_t i = 0; i < " << h.len << "LL; ++i) y[i * " << h.out_inc
        << "LL] += alpha * x[i * " << h.vec_inc << "LL];\n"
        << ind(d + 1) << "madds += " << 2 * h.len << "LL;\n";
    } else {
      const spg_access& xa = h.x_is_lhs ? lhs : rhs;
      const spg_access& ya = h.x_is_lhs ? rhs : lhs;
      o << ind(d + 1) << "const double* x = " << base(xa) << " + " << offset(xa) << ";\n"
        << ind(d + 1) << "const double* yv = " << base(ya) << " + " << offset(ya) << ";\n"
        << ind(d + 1) << "for (int64_t i = 0; i < " << h.m << "LL; ++i) {\n"
        << ind(d + 2) << "const double xi = x[i * " << h.x_inc << "LL];\n"
        << ind(d + 2) << "for (int64_t j = 0; j < " << h.n << "LL; ++j) y[i * " << h.out_row
        << "LL + j * " << h.out_col << "LL] += xi * yv[j * " << h.y_inc << "LL];\n"
        << ind(d + 1) << "}\n"
        << ind(d + 1) << "madds += " << 2 * h.m * h.n << "LL;\n";
    }
    o << ind(d) << "}\n";
  }
};

std::mutex g_jit_mu;
std::unordered_map<std::string, cudaKernel_t>& jit_cache() {
  static auto* c = new std::unordered_map<std::string, cudaKernel_t>;  // leaked on purpose
  return *c;
}

cudaKernel_t compile(const std::string& src) {
  std::lock_guard<std::mutex> lock(g_jit_mu);
  auto& cache = jit_cache();
  auto it = cache.find(src);
  if (it != cache.end()) return it->second;
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, src.c_str(), "spg_nest.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS)
    throw Status(SPTTN_ECUDA, "nvrtcCreateProgram failed");
  // --fmad=false: the reference's host arithmetic (separate multiply and add,
  // executor.cpp:395-404, micro_kernels.hpp:11-23) — same as generic.cu
  const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "-default-device",
                        "--fmad=false"};
  const nvrtcResult rc = nvrtcCompileProgram(prog, 4, opts);
  if (rc != NVRTC_SUCCESS) {
    size_t n = 0;
    nvrtcGetProgramLogSize(prog, &n);
    std::string log(n, '\0');
    nvrtcGetProgramLog(prog, &log[0]);
    nvrtcDestroyProgram(&prog);
    throw Status(SPTTN_ECUDA, "nest JIT compile failed: " + log.substr(0, 400));
  }
  size_t n = 0;
  nvrtcGetCUBINSize(prog, &n);
  std::string cubin(n, '\0');
  nvrtcGetCUBIN(prog, &cubin[0]);
  nvrtcDestroyProgram(&prog);
  cudaLibrary_t lib;
  SPTTN_CUDA(cudaLibraryLoadData(&lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
  cudaKernel_t k;
  SPTTN_CUDA(cudaLibraryGetKernel(&k, lib, "spg_nest"));
  cache.emplace(src, k);
  return k;
}

}  // namespace

bool jit_available() {
  int major = 0, minor = 0;
  return nvrtcVersion(&major, &minor) == NVRTC_SUCCESS;
}

void* jit_prepare(const spg_program& prog, const GenericState& g) {
  Gen gen(prog, g);
  const std::string src = gen.source();
  if (const char* d = std::getenv("SPTTN_JIT_DUMP"); d && *d && *d != '0')
    std::fprintf(stderr, "// ---- spttn JIT nest (mode %d, %lld workers) ----\n%s\n", g.par_mode,
                 static_cast<long long>(g.workers), src.c_str());
  return reinterpret_cast<void*>(compile(src));
}

void jit_execute(void* kernel, const spg_program& P, const DevCsf& csf,
                 const double* const* dense, double* out, GenericState& g, cudaStream_t s) {
  SPTTN_CUDA(cudaMemsetAsync(g.counters, 0, g.zero_bytes, s));
  JitArgs a{};
  const CsfView t = csf.view();
  for (int l = 0; l < csf.order; ++l) {
    a.idx[l] = t.idx[l];
    a.ptr[l] = t.ptr[l];
    a.nlev[l] = t.nlev[l];
  }
  a.vals = t.vals;
  a.dense = dense;
  a.out = out;
  a.bufs = g.buffers;
  a.buf_elems = g.total_buffer_elems;
  a.priv = g.priv_out;
  a.out_size = g.out_size;
  a.workers = g.par_mode == 0 ? 1 : g.workers;
  a.counters = g.counters;
  a.leaf_keys = g.leaf_keys;
  a.leaf_pos = g.leaf_pos;
  a.nkeys = g.n_leaf_keys;
  a.phase = 0;
  void* args[] = {&a};
  const unsigned blocks = static_cast<unsigned>((a.workers + 127) / 128);
  SPTTN_CUDA(cudaLaunchKernel(kernel, dim3(blocks), dim3(128), args, 0, s));
  (void)P;
  if (g.priv) generic_reduce(g, out, s);
  if (g.tail) {
    generic_reduce_buffers(g, s);
    a.phase = 1;
    a.workers = 1;
    SPTTN_CUDA(cudaLaunchKernel(kernel, dim3(1), dim3(128), args, 0, s));
  }
}

JitSplit jit_analyze(const spg_program& G) {
  JitSplit js;
  if (G.observe || G.num_roots < 1) return js;
  const spg_node& r = G.nodes[G.roots[0]];
  if (r.kind != SPG_SPARSE || r.csf_level != 0 || r.hook >= 0) return js;
  bool in_r[SPG_MAX_BUFFERS] = {};
  for (int k = 0; k < r.reset_count; ++k) {
    const int b = G.resets[r.reset_begin + k];
    if (!in_r[b] && js.n_rset < 16) js.rset[js.n_rset++] = b;
    in_r[b] = true;
  }
  const spg_node* l1 = nullptr;
  if (r.child_count == 1) {
    const spg_node& c = G.nodes[G.children[r.child_begin]];
    if (c.kind == SPG_SPARSE && c.csf_level == 1 && c.reset_count == 0 && c.hook < 0) l1 = &c;
  }
  auto term_of = [&](const spg_node& n) {
    if (n.kind == SPG_LEAF) return static_cast<int>(n.term);
    return n.hook >= 0 ? static_cast<int>(G.hooks[n.hook].term) : -1;
  };
  auto has = [](const spg_access& a, int id) {
    for (int k = 0; k < a.naddr; ++k)
      if (a.ids[k] == id && a.strides[k] != 0) return true;
    return false;
  };
  bool ok = true, ds = true, df = l1 != nullptr;
  std::vector<int> st(G.children + r.child_begin, G.children + r.child_begin + r.child_count);
  while (!st.empty()) {
    const spg_node& n = G.nodes[st.back()];
    st.pop_back();
    for (int k = 0; k < n.reset_count; ++k) ok &= !in_r[G.resets[n.reset_begin + k]];
    const int t = term_of(n);
    if (t >= 0) {
      for (const spg_access* a : {&G.lhs[t], &G.rhs[t]})
        ok &= !(a->kind == SPG_OP_BUFFER && in_r[a->slot]);
      const spg_access& o = G.out[t];
      if (o.kind == SPG_OP_OUT_DENSE || o.kind == SPG_OP_OUT_SPARSE) js.writes_out = true;
      if (o.kind == SPG_OP_OUT_DENSE) {
        ds &= has(o, r.index);
        df &= l1 && has(o, r.index) && has(o, l1->index);
      }
    }
    if (n.kind != SPG_LEAF && n.hook < 0)
      for (int c = 0; c < n.child_count; ++c) st.push_back(G.children[n.child_begin + c]);
  }
  // later roots run sequentially after the accumulators are summed: every
  // buffer they read is one of those or is reset among them
  bool reset_tail[SPG_MAX_BUFFERS] = {};
  std::vector<int> tail;
  for (int q = 1; q < G.num_roots; ++q) st.push_back(G.roots[q]);
  while (!st.empty()) {
    const spg_node& n = G.nodes[st.back()];
    st.pop_back();
    tail.push_back(static_cast<int>(&n - G.nodes));
    for (int k = 0; k < n.reset_count; ++k) reset_tail[G.resets[n.reset_begin + k]] = true;
    if (n.kind != SPG_LEAF && n.hook < 0)
      for (int c = 0; c < n.child_count; ++c) st.push_back(G.children[n.child_begin + c]);
  }
  for (int v : tail) {
    const int t = term_of(G.nodes[v]);
    if (t < 0) continue;
    for (const spg_access* a : {&G.lhs[t], &G.rhs[t]})
      ok &= !(a->kind == SPG_OP_BUFFER && !in_r[a->slot] && !reset_tail[a->slot]);
  }
  js.ok = ok;
  js.fiber_ok = l1 != nullptr;
  js.disjoint_slice = ds;
  js.disjoint_fiber = df;
  js.tail = G.num_roots > 1 || js.n_rset > 0;
  return js;
}

}  // namespace spttn_dev
