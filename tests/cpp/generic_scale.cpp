// Non-pinned nests at scale through the drop-in (the §8f-1 row): the orders
// the reference's own planners pick, and MTTKRP / TTMc for non-root output
// modes, on a 1e6-nonzero 1000^3 tensor. Runs each through spttn::prepare /
// execute (device forest interpreter, parallel over root slices) and checks
// it against the pinned kernel's result for the same product (dense outputs
// of the same spec) or against execute_unfactorized (non-root outputs),
// within the reference tolerance 1e-10 * (1 + max|ref|).
//   build/tests/generic_scale [nnz_density]
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "fixtures.hpp"
#include "spttn/cost_model.hpp"
#include "spttn/executor.hpp"
#include "spttn/optimizer.hpp"

using namespace spttn;
using namespace spttn::testing;

namespace {

double seconds_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

LoopOrder order_from(const KernelSpec& spec, const std::string& text) {
  LoopOrder o;
  std::vector<int> cur;
  std::string name;
  auto flush = [&] {
    if (!name.empty()) cur.push_back(spec.index_id(name));
    name.clear();
  };
  for (char c : text) {
    if (c == ',') {
      flush();
    } else if (c == ';') {
      flush();
      o.per_term.push_back(cur);
      cur.clear();
    } else {
      name += c;
    }
  }
  flush();
  o.per_term.push_back(cur);
  return o;
}

double max_err(const std::vector<double>& a, const std::vector<double>& b, double* scale) {
  double e = 0, m = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    e = std::max(e, std::fabs(a[i] - b[i]));
    m = std::max(m, std::fabs(b[i]));
  }
  *scale = m;
  return e;
}

int run(const char* label, const KernelSpec& spec, const Tensors& t, const std::string& path_text,
        const std::string& order_text, const std::vector<double>* want) {
  ContractionPath path = find_path(spec, path_text);
  LoopOrder order = order_from(spec, order_text);
  auto in = t.inputs();
  auto t0 = std::chrono::steady_clock::now();
  ExecPlan plan = prepare(spec, path, order, in);
  const double tp = seconds_since(t0);
  execute(plan);  // warm
  t0 = std::chrono::steady_clock::now();
  ExecResult r = execute(plan);
  const double te = seconds_since(t0);
  int bad = 0;
  double err = 0, scale = 0;
  if (want) {
    err = max_err(r.dense_out.values, *want, &scale);
    bad = err > 1e-10 * (1.0 + scale);
  }
  std::printf("%-34s %-12s %-22s prepare %8.2f ms  execute %9.2f ms  err %.2e%s\n", label,
              path_text.c_str(), order_text.c_str(), tp * 1e3, te * 1e3, err, bad ? "  MISMATCH" : "");
  return bad;
}

}  // namespace

int main(int argc, char** argv) {
  const double density = argc > 1 ? std::atof(argv[1]) : 1e-3;
  int bad = 0;
  {
    KernelSpec spec = mttkrp3(1000, 1000, 1000, 32);
    Tensors t = make_tensors(spec, random_coo(spec, density, 11));
    std::printf("MTTKRP-3 1000^3 nnz %lld\n", static_cast<long long>(t.csf.nnz()));
    // pinned (dedicated kernel) gives the reference for this path
    auto in = t.inputs();
    ExecPlan pin = prepare(spec, find_path(spec, "((T*C)*B)"), order_from(spec, "i,j,k,a;i,j,a"), in);
    const std::vector<double> want = execute(pin).dense_out.values;
    bad += run("pinned kernel", spec, t, "((T*C)*B)", "i,j,k,a;i,j,a", &want);
    bad += run("max-buf-dim planner order", spec, t, "((T*C)*B)", "i,j,a,k;i,j,a", &want);
    ExecPlan other = prepare(spec, find_path(spec, "((T*B)*C)"), order_from(spec, "i,j,k,a;i,k,a"), in);
    const std::vector<double> want2 = execute(other).dense_out.values;
    bad += run("dense-loops planner (other path)", spec, t, "((T*B)*C)", "i,j,k,a;i,k,a", &want2);
    double sc = 0;
    const double e = max_err(want2, want, &sc);
    std::printf("  paths agree: %.2e (scale %.2e)\n", e, sc);
    bad += e > 1e-10 * (1.0 + sc);
  }
  {
    // non-root outputs: MTTKRP for modes j and k on the (i,j,k) CSF; the
    // reference result is the sequential interpreter walk (bit-identical to
    // the reference executor), timed beside the parallel one
    KernelSpec s2 = parse_kernel("T[i,j,k]*A[i,a]*C[k,a]->B[j,a]",
                                 {{"i", 1000}, {"j", 1000}, {"k", 1000}, {"a", 32}});
    Tensors t2 = make_tensors(s2, random_coo(s2, density, 11));
    auto in2 = t2.inputs();
    auto seq = [&](const KernelSpec& sp, const Tensors& tt, const char* path, const char* ord) {
      setenv("SPTTN_GENERIC_PAR", "0", 1);
      auto in = tt.inputs();
      ExecPlan pl = prepare(sp, find_path(sp, path), order_from(sp, ord), in);
      unsetenv("SPTTN_GENERIC_PAR");
      auto t0 = std::chrono::steady_clock::now();
      std::vector<double> v = execute(pl).dense_out.values;
      std::printf("  sequential walk %s %s: %.1f ms\n", path, ord, seconds_since(t0) * 1e3);
      return v;
    };
    std::printf("MTTKRP-3 mode j\n");
    const std::vector<double> want = seq(s2, t2, "((T*C)*A)", "i,j,a,k;i,j,a");
    bad += run("mode j, max-buf-dim order", s2, t2, "((T*C)*A)", "i,j,a,k;i,j,a", &want);
    bad += run("mode j, dense-loops order", s2, t2, "((T*C)*A)", "i,j,k,a;i,a,j", &want);
    KernelSpec s3 = parse_kernel("T[i,j,k]*A[i,a]*B[j,a]->C[k,a]",
                                 {{"i", 1000}, {"j", 1000}, {"k", 1000}, {"a", 32}});
    Tensors t3 = make_tensors(s3, random_coo(s3, density, 11));
    std::printf("MTTKRP-3 mode k\n");
    const std::vector<double> want3 = seq(s3, t3, "((A*B)*T)", "i,j,a;i,j,a,k");
    bad += run("mode k, max-buf-dim order", s3, t3, "((A*B)*T)", "i,j,a;i,j,a,k", &want3);
    (void)in2;
  }
  {
    // TTTc-4 through the JIT-compiled nest vs the
    // interpreter, on the max-buf-dim planner's path / order
    KernelSpec spec = tttc4(60, 8);
    Tensors t = make_tensors(spec, random_coo(spec, 0.02, 31));
    std::printf("TTTc-4 60^4 R=8 nnz %lld\n", static_cast<long long>(t.csf.nnz()));
    auto in = t.inputs();
    auto model = max_buffer_dim_model();
    auto [path, result] = joint_search(spec, *model);
    auto timed = [&](const char* what, const char* jit, const char* par) {
      setenv("SPTTN_GENERIC_JIT", jit, 1);
      setenv("SPTTN_GENERIC_PAR", par, 1);
      auto t0 = std::chrono::steady_clock::now();
      ExecPlan plan = prepare(spec, path, result.best.order, in);
      const double tp = seconds_since(t0);
      unsetenv("SPTTN_GENERIC_JIT");
      unsetenv("SPTTN_GENERIC_PAR");
      execute(plan);
      t0 = std::chrono::steady_clock::now();
      ExecResult r = execute(plan);
      std::printf("  %-22s prepare %8.2f ms  execute %9.2f ms\n", what, tp * 1e3,
                  seconds_since(t0) * 1e3);
      return r.dense_out.values;
    };
    const std::vector<double> a = timed("JIT (parallel)", "1", "1"), c = timed("JIT (sequential)", "1", "0"),
                              b = timed("interpreter", "0", "1");
    double err = 0, mag = 0;
    for (size_t e = 0; e < a.size(); ++e) {
      err = std::max(err, std::abs(a[e] - b[e]));
      mag = std::max(mag, std::abs(b[e]));
    }
    std::printf("  sequential JIT bit-identical to interpreter: %s; parallel JIT max rel err %.2e\n",
                c == b ? "yes" : "NO", err / std::max(mag, 1e-300));
    bad += c != b || err > 1e-12 * mag;
  }
  std::printf("%s\n", bad ? "FAILED" : "all match");
  return bad ? 1 : 0;
}
