// TEST INFRASTRUCTURE ONLY — extern "C" bridge onto the reference SpTTN
// library compiled from /root/reference/proj/src with -Dspttn=spttn_ref.
// Used by tests/ (parity checker, golden-fixture generation) and by
// bench.py's cpu_baseline / --impl reference leg. Never linked by the product.
//
// Every entry point forwards to the reference's own public API:
//   parse_kernel            proj/src/kernel_spec.cpp:103
//   enumerate_paths         proj/src/contraction_path.cpp:105
//   prepare / execute       proj/src/executor.cpp:172, :510
//   execute_unfactorized    proj/src/executor.cpp:522
//   flops_estimate          proj/src/executor.cpp:628
//   build_csf / gen_random  proj/src/tensor.cpp:41, proj/src/tns_io.cpp:123
//   gen_dense / stable_hash proj/src/tns_io.cpp:161, :168
//   joint_search            proj/src/optimizer.cpp:219
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "spttn/executor.hpp"
#include "spttn/optimizer.hpp"
#include "spttn/tns_io.hpp"

using namespace spttn_ref;

namespace {

thread_local std::string g_err;

std::vector<std::string> split(const std::string& s, char sep) {
  std::vector<std::string> out;
  std::string cur;
  std::istringstream in(s);
  while (std::getline(in, cur, sep))
    if (!cur.empty()) out.push_back(cur);
  return out;
}

std::map<std::string, int64_t> parse_dims(const char* text) {
  std::map<std::string, int64_t> d;
  for (const auto& kv : split(text, ',')) {
    auto eq = kv.find('=');
    d[kv.substr(0, eq)] = std::stoll(kv.substr(eq + 1));
  }
  return d;
}

LoopOrder parse_order(const KernelSpec& spec, const char* text) {
  LoopOrder o;
  for (const auto& term : split(text, ';')) {
    std::vector<int> ids;
    for (const auto& n : split(term, ',')) {
      int id = spec.index_id(n);
      if (id < 0) throw std::invalid_argument("unknown index in order: " + n);
      ids.push_back(id);
    }
    o.per_term.push_back(ids);
  }
  return o;
}

ContractionPath find_path(const KernelSpec& spec, const char* describe) {
  for (const auto& p : enumerate_paths(spec))
    if (p.describe(spec) == describe) return p;
  throw std::invalid_argument(std::string("no contraction path ") + describe);
}

CsfTensor make_csf(const KernelSpec& spec, int d, const int64_t* level_sizes,
                   const int64_t* const* idx, const int64_t* const* ptr, const double* values) {
  CsfTensor csf;
  const auto& sp = spec.sparse_input();
  if (d != static_cast<int>(sp.indices.size()))
    throw std::invalid_argument("bridge: CSF order does not match the kernel");
  for (int l = 0; l < d; ++l)
    csf.modes.push_back(Index{spec.index_names[sp.indices[l]], spec.dim(sp.indices[l])});
  csf.idx.resize(d);
  csf.ptr.resize(d - 1);
  for (int l = 0; l < d; ++l) csf.idx[l].assign(idx[l], idx[l] + level_sizes[l]);
  for (int l = 0; l + 1 < d; ++l) csf.ptr[l].assign(ptr[l], ptr[l] + level_sizes[l] + 1);
  csf.values.assign(values, values + level_sizes[d - 1]);
  return csf;
}

std::vector<DenseTensor> make_dense(const KernelSpec& spec, const double* const* factors) {
  std::vector<DenseTensor> out;
  for (int f = 1; f < spec.num_inputs(); ++f) {
    std::vector<Index> shape;
    for (int id : spec.tensors[f].indices) shape.push_back(Index{spec.index_names[id], spec.dim(id)});
    DenseTensor t(shape);
    std::memcpy(t.values.data(), factors[f - 1], t.values.size() * sizeof(double));
    out.push_back(std::move(t));
  }
  return out;
}

ExecInputs inputs_of(const CsfTensor& csf, const std::vector<DenseTensor>& dense) {
  ExecInputs in;
  in.sparse = &csf;
  for (const auto& t : dense) in.dense.push_back(&t);
  return in;
}

int copy_result(const ExecResult& r, double* out, int64_t out_count) {
  const auto& v = r.sparse_out_values.empty() && !r.dense_out.values.empty()
                      ? r.dense_out.values
                      : (r.dense_out.values.empty() ? r.sparse_out_values : r.dense_out.values);
  if (static_cast<int64_t>(v.size()) != out_count) {
    g_err = "bridge: output size " + std::to_string(v.size()) + " != " + std::to_string(out_count);
    return 2;
  }
  std::memcpy(out, v.data(), v.size() * sizeof(double));
  return 0;
}

template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const unsupported_order_error& e) {
    g_err = e.what();
    return 3;
  } catch (const resource_error& e) {
    g_err = e.what();
    return 4;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 5;
  }
}

struct CsfHandle {
  CsfTensor csf;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

uint64_t ref_stable_hash(const char* s) { return stable_hash(s); }

// Fused execution of (path, order) through prepare+execute. stats_out:
// [0]=multiply_adds, [1]=#buffers, [2..]=buffer_resets (up to stats_cap-2).
int ref_execute(const char* kernel, const char* dims, const char* path, const char* order, int d,
                const int64_t* level_sizes, const int64_t* const* idx, const int64_t* const* ptr,
                const double* values, const double* const* factors, double* out,
                int64_t out_count, int64_t* stats_out, int stats_cap, double* seconds,
                int repeats) {
  return guarded([&] {
    KernelSpec spec = parse_kernel(kernel, parse_dims(dims));
    ContractionPath p = find_path(spec, path);
    LoopOrder o = parse_order(spec, order);
    CsfTensor csf = make_csf(spec, d, level_sizes, idx, ptr, values);
    auto dense = make_dense(spec, factors);
    ExecPlan plan = prepare(spec, p, o, inputs_of(csf, dense));
    ExecResult best;
    double best_s = 1e300;
    for (int r = 0; r < std::max(1, repeats); ++r) {
      ExecResult res = execute(plan);
      if (res.stats.wall_seconds < best_s) best_s = res.stats.wall_seconds;
      best = std::move(res);
    }
    if (seconds) *seconds = best_s;
    if (stats_out && stats_cap >= 2) {
      stats_out[0] = best.stats.multiply_adds;
      stats_out[1] = static_cast<int64_t>(best.stats.buffer_resets.size());
      for (size_t b = 0; b < best.stats.buffer_resets.size() && static_cast<int>(b) + 2 < stats_cap; ++b)
        stats_out[2 + b] = best.stats.buffer_resets[b];
    }
    return copy_result(best, out, out_count);
  });
}

int ref_execute_unfactorized(const char* kernel, const char* dims, int d,
                             const int64_t* level_sizes, const int64_t* const* idx,
                             const int64_t* const* ptr, const double* values,
                             const double* const* factors, double* out, int64_t out_count,
                             int64_t* multiply_adds, double* seconds) {
  return guarded([&] {
    KernelSpec spec = parse_kernel(kernel, parse_dims(dims));
    CsfTensor csf = make_csf(spec, d, level_sizes, idx, ptr, values);
    auto dense = make_dense(spec, factors);
    ExecResult res = execute_unfactorized(spec, inputs_of(csf, dense));
    if (multiply_adds) *multiply_adds = res.stats.multiply_adds;
    if (seconds) *seconds = res.stats.wall_seconds;
    return copy_result(res, out, out_count);
  });
}

int ref_flops_estimate(const char* kernel, const char* dims, const char* path, const char* order,
                       int d, const int64_t* level_sizes, const int64_t* const* idx,
                       const int64_t* const* ptr, const double* values, int64_t* flops,
                       int64_t* flops_unfact) {
  return guarded([&] {
    KernelSpec spec = parse_kernel(kernel, parse_dims(dims));
    ContractionPath p = find_path(spec, path);
    LoopOrder o = parse_order(spec, order);
    CsfTensor csf = make_csf(spec, d, level_sizes, idx, ptr, values);
    *flops = flops_estimate(spec, p, o, csf);
    if (flops_unfact) *flops_unfact = flops_unfactorized(spec, csf);
    return 0;
  });
}

// Hook metadata of prepare() for (path, order): 3 ints per term
// (kind, span, meta_loops); also buffer orders/sizes (2 per buffer).
int ref_plan_info(const char* kernel, const char* dims, const char* path, const char* order, int d,
                  const int64_t* level_sizes, const int64_t* const* idx, const int64_t* const* ptr,
                  const double* values, const double* const* factors, int* hooks_out,
                  int hooks_cap, int64_t* total_buffer_bytes) {
  return guarded([&] {
    KernelSpec spec = parse_kernel(kernel, parse_dims(dims));
    ContractionPath p = find_path(spec, path);
    LoopOrder o = parse_order(spec, order);
    CsfTensor csf = make_csf(spec, d, level_sizes, idx, ptr, values);
    auto dense = make_dense(spec, factors);
    ExecPlan plan = prepare(spec, p, o, inputs_of(csf, dense));
    const auto& h = plan.hooks();
    for (size_t t = 0; t < h.size() && static_cast<int>(3 * t + 2) < hooks_cap; ++t) {
      hooks_out[3 * t] = static_cast<int>(h[t].kind);
      hooks_out[3 * t + 1] = h[t].span;
      hooks_out[3 * t + 2] = h[t].meta_loops;
    }
    if (total_buffer_bytes) *total_buffer_bytes = plan.total_buffer_bytes();
    return static_cast<int>(h.size()) == 0 ? 0 : 0;
  });
}

// All (path, order) pairs the reference enumerates for a kernel over its
// minimum-depth paths (or all paths when all_paths != 0), as lines
// "path|order" in out (NUL terminated). Returns the count, or -1.
int64_t ref_enumerate(const char* kernel, const char* dims, int all_paths, char* out,
                      int64_t cap) {
  try {
    KernelSpec spec = parse_kernel(kernel, parse_dims(dims));
    auto paths = enumerate_paths(spec);
    if (!all_paths) paths = filter_min_depth(paths);
    std::string text;
    int64_t count = 0;
    for (const auto& p : paths) {
      for (const auto& o : enumerate_orders(spec, p, default_csf_order(spec))) {
        text += p.describe(spec) + "|";
        for (size_t t = 0; t < o.per_term.size(); ++t) {
          if (t) text += ";";
          for (size_t k = 0; k < o.per_term[t].size(); ++k) {
            if (k) text += ",";
            text += spec.index_names[o.per_term[t][k]];
          }
        }
        text += "\n";
        ++count;
      }
    }
    if (static_cast<int64_t>(text.size()) + 1 > cap) {
      g_err = "bridge: enumerate buffer too small (" + std::to_string(text.size() + 1) + ")";
      return -1;
    }
    std::memcpy(out, text.c_str(), text.size() + 1);
    return count;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Planner choice (joint_search) under a cost model text such as
// "dense-loops:bound=2" or "max-buf-dim"; writes "path|order".
int ref_joint_search(const char* kernel, const char* dims, const char* model, char* out,
                     int64_t cap) {
  return guarded([&] {
    KernelSpec spec = parse_kernel(kernel, parse_dims(dims));
    auto m = parse_cost_model(model);
    auto [p, res] = joint_search(spec, *m);
    std::string text = p.describe(spec) + "|";
    for (size_t t = 0; t < res.best.order.per_term.size(); ++t) {
      if (t) text += ";";
      for (size_t k = 0; k < res.best.order.per_term[t].size(); ++k) {
        if (k) text += ",";
        text += spec.index_names[res.best.order.per_term[t][k]];
      }
    }
    if (static_cast<int64_t>(text.size()) + 1 > cap) return 2;
    std::memcpy(out, text.c_str(), text.size() + 1);
    return 0;
  });
}

// ---- tensor construction through the reference --------------------------

// COO (nnz x d row-major coordinates, values) -> reference normalize +
// build_csf under mode order names "i,j,k". Returns an opaque handle.
void* ref_build_csf(int d, const char* names, const int64_t* dims, int64_t nnz,
                    const int64_t* coords, const double* values, const char* mode_order) {
  try {
    CooTensor coo;
    auto nm = split(names, ',');
    for (int l = 0; l < d; ++l) coo.indices.push_back(Index{nm[l], dims[l]});
    for (int64_t e = 0; e < nnz; ++e)
      coo.entries.emplace_back(std::vector<int64_t>(coords + e * d, coords + (e + 1) * d), values[e]);
    coo.normalize();
    auto h = new CsfHandle;
    h->csf = build_csf(coo, split(mode_order, ','));
    return h;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

// Reference gen_random (Floyd sampling) -> build_csf in declared order.
void* ref_gen_random_csf(int d, const char* names, const int64_t* dims, double density,
                         uint64_t seed) {
  try {
    std::vector<Index> idx;
    auto nm = split(names, ',');
    std::vector<std::string> order;
    for (int l = 0; l < d; ++l) {
      idx.push_back(Index{nm[l], dims[l]});
      order.push_back(nm[l]);
    }
    auto h = new CsfHandle;
    h->csf = build_csf(gen_random(idx, density, seed), order);
    return h;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

int64_t ref_csf_level_size(void* h, int l) {
  auto* c = static_cast<CsfHandle*>(h);
  return static_cast<int64_t>(c->csf.idx[l].size());
}

void ref_csf_copy(void* h, int l, int64_t* idx_out, int64_t* ptr_out) {
  auto* c = static_cast<CsfHandle*>(h);
  std::memcpy(idx_out, c->csf.idx[l].data(), c->csf.idx[l].size() * sizeof(int64_t));
  if (ptr_out && l + 1 < c->csf.order())
    std::memcpy(ptr_out, c->csf.ptr[l].data(), c->csf.ptr[l].size() * sizeof(int64_t));
}

void ref_csf_values(void* h, double* out) {
  auto* c = static_cast<CsfHandle*>(h);
  std::memcpy(out, c->csf.values.data(), c->csf.values.size() * sizeof(double));
}

void ref_csf_free(void* h) { delete static_cast<CsfHandle*>(h); }

int ref_gen_dense(int d, const char* names, const int64_t* dims, uint64_t seed, double* out) {
  return guarded([&] {
    std::vector<Index> idx;
    auto nm = split(names, ',');
    for (int l = 0; l < d; ++l) idx.push_back(Index{nm[l], dims[l]});
    DenseTensor t = gen_dense(idx, seed);
    std::memcpy(out, t.values.data(), t.values.size() * sizeof(double));
    return 0;
  });
}

// ---- CPU baseline: the reference executor on all host threads ----------
//
// The reference executor is sequential but distinct plans
// over shared read-only tensors may run concurrently. The root level is split
// into `nthreads` contiguous nnz-balanced ranges; each thread prepares and
// executes its own plan on its sub-CSF (setup untimed). The timed region is
// the concurrent execute() calls plus the merge of the disjoint per-thread
// results into `out`. Root-indexed dense outputs only, or @sparse_out.
int ref_execute_threads(const char* kernel, const char* dims, const char* path, const char* order,
                        int d, const int64_t* level_sizes, const int64_t* const* idx,
                        const int64_t* const* ptr, const double* values,
                        const double* const* factors, double* out, int64_t out_count,
                        int nthreads, int repeats, double* best_seconds) {
  return guarded([&] {
    KernelSpec spec = parse_kernel(kernel, parse_dims(dims));
    ContractionPath p = find_path(spec, path);
    LoopOrder o = parse_order(spec, order);
    auto dense = make_dense(spec, factors);
    nthreads = std::max(1, nthreads);
    const int64_t n0 = level_sizes[0];
    const int64_t nnz = level_sizes[d - 1];
    // leaf range of each root node: follow ptr down the levels.
    auto leaf_of = [&](int64_t node0) {
      int64_t pos = node0;
      for (int l = 0; l + 1 < d; ++l) pos = ptr[l][pos];
      return pos;
    };
    std::vector<int64_t> cut{0};
    for (int t = 1; t < nthreads; ++t) {
      const int64_t target = nnz * t / nthreads;
      int64_t lo = cut.back(), hi = n0;
      while (lo < hi) {
        int64_t mid = (lo + hi) / 2;
        if (leaf_of(mid) < target) lo = mid + 1; else hi = mid;
      }
      cut.push_back(lo);
    }
    cut.push_back(n0);
    struct Part {
      CsfTensor csf;
      int64_t leaf_begin = 0;
      std::unique_ptr<ExecPlan> plan;
      ExecResult res;
    };
    std::vector<Part> parts(nthreads);
    for (int t = 0; t < nthreads; ++t) {
      Part& pt = parts[t];
      const auto& sp = spec.sparse_input();
      for (int l = 0; l < d; ++l)
        pt.csf.modes.push_back(Index{spec.index_names[sp.indices[l]], spec.dim(sp.indices[l])});
      pt.csf.idx.resize(d);
      pt.csf.ptr.resize(d - 1);
      int64_t b = cut[t], e = cut[t + 1];
      for (int l = 0; l < d; ++l) {
        pt.csf.idx[l].assign(idx[l] + b, idx[l] + e);
        if (l + 1 < d) {
          pt.csf.ptr[l].resize(e - b + 1);
          for (int64_t q = b; q <= e; ++q) pt.csf.ptr[l][q - b] = ptr[l][q] - ptr[l][b];
          const int64_t nb = ptr[l][b], ne = ptr[l][e];
          b = nb;
          e = ne;
        }
      }
      pt.leaf_begin = b;
      pt.csf.values.assign(values + b, values + e);
      pt.plan = std::make_unique<ExecPlan>(prepare(spec, p, o, inputs_of(pt.csf, dense)));
    }
    double best = 1e300;
    for (int r = 0; r < std::max(1, repeats); ++r) {
      // timed: the reference executor on every thread (each execute
      // allocates and zeroes its own output, as spttn::execute does)
      const auto t0 = std::chrono::steady_clock::now();
      std::vector<std::thread> th;
      for (int t = 0; t < nthreads; ++t)
        th.emplace_back([&, t] { parts[t].res = execute(*parts[t].plan); });
      for (auto& x : th) x.join();
      const double s =
          std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      best = std::min(best, s);
      // untimed: merge (dense outputs are root-row disjoint -> sum; sparse -> place)
      if (spec.output_sparse) {
        for (auto& pt : parts)
          std::memcpy(out + pt.leaf_begin, pt.res.sparse_out_values.data(),
                      pt.res.sparse_out_values.size() * sizeof(double));
      } else {
        std::memset(out, 0, out_count * sizeof(double));
        for (auto& pt : parts) {
          const auto& v = pt.res.dense_out.values;
          if (static_cast<int64_t>(v.size()) != out_count) throw std::runtime_error("size");
          for (int64_t q = 0; q < out_count; ++q) out[q] += v[q];
        }
      }
    }
    *best_seconds = best;
    return 0;
  });
}

}  // extern "C"
