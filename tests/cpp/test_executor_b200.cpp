// Executor contract tests run against the B200 drop-in (spttn::prepare /
// execute defined by csrc/shim/executor_b200.cpp over the device engine).
// They restate the cases of the reference's proj/tests/test_executor.cpp
// (doctest is not available here, so a tiny CHECK harness replaces it) and
// add device-routing checks: pinned nests must run on their dedicated
// kernels, every other admissible order on the device interpreter.
// Inputs come from the reference fixtures (proj/tests/fixtures.hpp).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <set>
#include <string>

#include "fixtures.hpp"
#include "spttn/executor.hpp"
#include "spttn/optimizer.hpp"
#include "spttn_b200.h"
#include "spttn_b200_shim.hpp"

using namespace spttn;
using namespace spttn::testing;

namespace {

int g_fail = 0, g_checks = 0;
std::string g_case;

#define CHECK(cond)                                                                    \
  do {                                                                                 \
    ++g_checks;                                                                        \
    if (!(cond)) {                                                                     \
      ++g_fail;                                                                        \
      std::printf("  FAIL %s:%d [%s] %s\n", __FILE__, __LINE__, g_case.c_str(), #cond); \
    }                                                                                  \
  } while (0)

template <class E, class F>
bool throws_as(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

LoopOrder order_of(const KernelSpec& spec, const std::vector<std::vector<std::string>>& names) {
  LoopOrder o;
  for (const auto& term : names) {
    std::vector<int> ids;
    for (const auto& n : term) ids.push_back(spec.index_id(n));
    o.per_term.push_back(ids);
  }
  return o;
}

double tolerance(const ExecResult& oracle) {
  double m = 0.0;
  for (double v : oracle.dense_out.values) m = std::max(m, std::abs(v));
  for (double v : oracle.sparse_out_values) m = std::max(m, std::abs(v));
  return 1e-10 * (1.0 + m);
}

bool close(const ExecResult& got, const ExecResult& want) {
  const double tol = tolerance(want);
  if (got.dense_out.values.size() != want.dense_out.values.size()) return false;
  if (got.sparse_out_values.size() != want.sparse_out_values.size()) return false;
  for (size_t i = 0; i < got.dense_out.values.size(); ++i)
    if (std::abs(got.dense_out.values[i] - want.dense_out.values[i]) > tol) return false;
  for (size_t i = 0; i < got.sparse_out_values.size(); ++i)
    if (std::abs(got.sparse_out_values[i] - want.sparse_out_values[i]) > tol) return false;
  return true;
}

void run_case(const char* name, const std::function<void()>& body) {
  g_case = name;
  const int before = g_fail;
  try {
    body();
  } catch (const std::exception& e) {
    ++g_fail;
    std::printf("  FAIL [%s] exception: %s\n", name, e.what());
  }
  std::printf("%s %s\n", g_fail == before ? "PASS" : "FAIL", name);
}

}  // namespace

int main() {
  run_case("mttkrp on the 3-entry fixture, every order, vs direct evaluation", [] {
    KernelSpec spec = mttkrp3(2, 2, 3, 2);
    CooTensor coo = coo3(2, 2, 3);
    Tensors tensors = make_tensors(spec, coo);
    const DenseTensor& B = tensors.dense[0];
    const DenseTensor& C = tensors.dense[1];
    DenseTensor expect({{"i", 2}, {"a", 2}});
    for (const auto& e : coo.entries)
      for (int64_t a = 0; a < 2; ++a)
        expect.at({e.first[0], a}) += e.second * B.at({e.first[1], a}) * C.at({e.first[2], a});
    auto inputs = tensors.inputs();
    int pinned = 0, orders = 0, on_path = 0;
    for (const auto& path : filter_min_depth(enumerate_paths(spec)))
      for (const auto& order : enumerate_orders(spec, path, default_csf_order(spec))) {
        ExecPlan plan = prepare(spec, path, order, inputs);
        pinned += spttn_b200_plan_device_kind(plan) == SPTTN_NEST_MTTKRP3;
        on_path += path.describe(spec) == "((T*C)*B)";
        ++orders;
        ExecResult res = execute(plan);
        for (int64_t i = 0; i < 2; ++i)
          for (int64_t a = 0; a < 2; ++a)
            CHECK(std::abs(res.dense_out.at({i, a}) - expect.at({i, a})) <= 1e-12);
      }
    CHECK(pinned == on_path && on_path >= 1);  // every order on the ((T*C)*B) path
    CHECK(orders > 1);
    ExecResult oracle = execute_unfactorized(spec, inputs);
    for (int64_t i = 0; i < 2; ++i)
      for (int64_t a = 0; a < 2; ++a)
        CHECK(std::abs(oracle.dense_out.at({i, a}) - expect.at({i, a})) <= 1e-12);
  });

  run_case("unfactorized operation counts and the empty tensor", [] {
    KernelSpec spec = mttkrp3(2, 2, 3, 2);
    Tensors t = make_tensors(spec, coo3(2, 2, 3));
    auto in = t.inputs();
    CHECK(execute_unfactorized(spec, in).stats.multiply_adds == 18);
    CHECK(flops_unfactorized(spec, t.csf) == 18);
    KernelSpec tt = ttmc3(2, 2, 3, 2, 2);
    Tensors t2 = make_tensors(tt, coo3(2, 2, 3));
    auto in2 = t2.inputs();
    CHECK(execute_unfactorized(tt, in2).stats.multiply_adds == 36);
    CooTensor empty;
    empty.indices = {{"i", 2}, {"j", 2}, {"k", 3}};
    Tensors te = make_tensors(spec, empty);
    auto ine = te.inputs();
    ExecResult r = execute_unfactorized(spec, ine);
    CHECK(r.stats.multiply_adds == 0);
    for (double v : r.dense_out.values) CHECK(v == 0.0);
    ContractionPath path = find_path(spec, "((T*C)*B)");
    ExecPlan plan = prepare(spec, path, order_of(spec, {{"i", "j", "k", "a"}, {"i", "j", "a"}}), ine);
    ExecResult f = execute(plan);
    for (double v : f.dense_out.values) CHECK(v == 0.0);
  });

  run_case("tttp output shares the pattern and matches the oracle, every order", [] {
    KernelSpec spec = tttp3(4, 3, 3, 2);
    Tensors t = make_tensors(spec, random_coo(spec, 0.25, 11));
    auto in = t.inputs();
    ExecResult oracle = execute_unfactorized(spec, in);
    CHECK(oracle.sparse_out_values.size() == static_cast<size_t>(t.csf.nnz()));
    int n = 0, pinned = 0, on_path = 0;
    for (const auto& path : filter_min_depth(enumerate_paths(spec)))
      for (const auto& order : enumerate_orders(spec, path, default_csf_order(spec))) {
        ExecPlan plan = prepare(spec, path, order, in);
        pinned += spttn_b200_plan_device_kind(plan) == SPTTN_NEST_TTTP3;
        on_path += path.describe(spec) == "(((U*V)*W)*T)";
        CHECK(close(execute(plan), oracle));
        ++n;
      }
    CHECK(n > 0);
    CHECK(pinned == on_path && on_path >= 1);
  });

  run_case("an all-zero dense factor gives an exactly-zero output", [] {
    KernelSpec spec = ttmc3(3, 3, 3, 2, 2);
    Tensors t = make_tensors(spec, random_coo(spec, 0.3, 5));
    t.dense[0].values.assign(t.dense[0].values.size(), 0.0);
    auto in = t.inputs();
    auto model = max_buffer_dim_model();
    auto [path, result] = joint_search(spec, *model);
    ExecResult res = execute(*std::make_unique<ExecPlan>(prepare(spec, path, result.best.order, in)));
    for (double v : res.dense_out.values) CHECK(v == 0.0);
    // and on the pinned DMMA kernel
    ExecPlan p2 = prepare(spec, find_path(spec, "((T*V)*U)"),
                          order_of(spec, {{"i", "j", "k", "s"}, {"i", "j", "s", "r"}}), in);
    CHECK(spttn_b200_plan_device_kind(p2) == SPTTN_NEST_TTMC3);
    for (double v : execute(p2).dense_out.values) CHECK(v == 0.0);
  });

  run_case("order-4 TTMc hooks: vector / rank-1 / loop+vector, flop count", [] {
    KernelSpec spec = ttmc4(3, 2, 2, 2);
    ContractionPath path = find_path(spec, "(((T*W)*V)*U)");
    LoopOrder order = order_of(spec, {{"i", "j", "k", "l", "t"}, {"i", "j", "k", "s", "t"},
                                      {"i", "j", "r", "s", "t"}});
    Tensors t = make_tensors(spec, random_coo(spec, 0.2, 3));
    auto in = t.inputs();
    ExecPlan plan = prepare(spec, path, order, in);
    const auto& h = plan.hooks();
    CHECK(h.size() == 3);
    CHECK(h[0].kind == HookKind::VectorAccumulate && h[0].span == 1 && h[0].meta_loops == 0);
    CHECK(h[1].kind == HookKind::Rank1Update && h[1].span == 2 && h[1].meta_loops == 0);
    CHECK(h[2].kind == HookKind::VectorAccumulate && h[2].span == 2 && h[2].meta_loops == 1);
    CHECK(spttn_b200_plan_device_kind(plan) == SPTTN_NEST_TTMC4);
    ExecResult res = execute(plan);
    CHECK(close(res, execute_unfactorized(spec, in)));
    CHECK(res.stats.multiply_adds == flops_estimate(spec, path, order, t.csf));
  });

  run_case("scalar-buffer TTMc order: term 0 unhooked, same path runs on the kernel", [] {
    KernelSpec spec = ttmc3(3, 3, 3, 2, 2);
    ContractionPath path = find_path(spec, "((T*V)*U)");
    LoopOrder order = order_of(spec, {{"i", "j", "s", "k"}, {"i", "j", "s", "r"}});
    Tensors t = make_tensors(spec, random_coo(spec, 0.3, 9));
    auto in = t.inputs();
    ExecPlan plan = prepare(spec, path, order, in);
    CHECK(plan.hooks().size() == 2);
    CHECK(plan.hooks()[0].kind == HookKind::None);
    CHECK(plan.hooks()[1].kind == HookKind::VectorAccumulate);
    CHECK(spttn_b200_plan_device_kind(plan) == SPTTN_NEST_TTMC3);
    CHECK(execute(plan).stats.multiply_adds == flops_estimate(spec, path, order, t.csf));
    CHECK(close(execute(plan), execute_unfactorized(spec, in)));
  });

  run_case("a trailing dense index of size 1 degenerates to a scalar update", [] {
    KernelSpec spec = ttmc3(3, 3, 3, 2, 1);
    ContractionPath path = find_path(spec, "((T*V)*U)");
    LoopOrder order = order_of(spec, {{"i", "j", "k", "s"}, {"i", "j", "s", "r"}});
    Tensors t = make_tensors(spec, random_coo(spec, 0.4, 21));
    auto in = t.inputs();
    ExecPlan plan = prepare(spec, path, order, in);
    CHECK(close(execute(plan), execute_unfactorized(spec, in)));
  });

  run_case("oracle equivalence and flop equality over every admissible order", [] {
    for (const KernelSpec& spec : {mttkrp3(3, 3, 2, 2), ttmc3(3, 2, 3, 2, 2), tttp3(3, 2, 3, 2)}) {
      Tensors t = make_tensors(spec, random_coo(spec, 0.3, 17));
      auto in = t.inputs();
      ExecResult oracle = execute_unfactorized(spec, in);
      for (const auto& path : filter_min_depth(enumerate_paths(spec)))
        for (const auto& order : enumerate_orders(spec, path, default_csf_order(spec))) {
          ExecPlan plan = prepare(spec, path, order, in);
          ExecResult res = execute(plan);
          CHECK(close(res, oracle));
          CHECK(res.stats.multiply_adds == flops_estimate(spec, path, order, t.csf));
        }
    }
  });

  run_case("repeated execution is bit-identical (interpreter and DMMA kernel)", [] {
    KernelSpec spec = ttmc3(4, 4, 4, 3, 3);
    Tensors t = make_tensors(spec, random_coo(spec, 0.2, 31));
    auto in = t.inputs();
    auto model = dense_loop_metric(2);
    auto [path, result] = joint_search(spec, *model);
    for (const LoopOrder& order :
         {result.best.order, order_of(spec, {{"i", "j", "k", "s"}, {"i", "j", "s", "r"}})}) {
      const ContractionPath p = order == result.best.order ? path : find_path(spec, "((T*V)*U)");
      ExecPlan plan = prepare(spec, p, order, in);
      ExecResult a = execute(plan), b = execute(plan);
      CHECK(a.dense_out.values.size() == b.dense_out.values.size());
      CHECK(std::memcmp(a.dense_out.values.data(), b.dense_out.values.data(),
                        a.dense_out.values.size() * sizeof(double)) == 0);
      ExecPlan plan2 = prepare(spec, p, order, in);
      ExecResult c = execute(plan2);
      CHECK(std::memcmp(a.dense_out.values.data(), c.dense_out.values.data(),
                        a.dense_out.values.size() * sizeof(double)) == 0);
    }
  });

  run_case("pairwise flop counts follow the CSF level formulas", [] {
    KernelSpec spec = mttkrp3(8, 8, 8, 4);
    Tensors t = make_tensors(spec, random_coo(spec, 0.05, 13));
    auto in = t.inputs();
    const int64_t nnz = t.csf.nnz(), nij = nnz_at_level(t.csf, 2), A = 4;
    ContractionPath path = find_path(spec, "((T*C)*B)");
    LoopOrder order = order_of(spec, {{"i", "j", "k", "a"}, {"i", "j", "a"}});
    ExecPlan plan = prepare(spec, path, order, in);
    ExecResult res = execute(plan);
    CHECK(res.stats.multiply_adds == 2 * nnz * A + 2 * nij * A);
    CHECK(flops_estimate(spec, path, order, t.csf) == 2 * nnz * A + 2 * nij * A);
    ExecResult oracle = execute_unfactorized(spec, in);
    CHECK(oracle.stats.multiply_adds == 3 * nnz * A);
    CHECK(close(res, oracle));
    KernelSpec tt = ttmc3(8, 8, 8, 3, 2);
    Tensors t2 = make_tensors(tt, random_coo(tt, 0.05, 29));
    auto in2 = t2.inputs();
    const int64_t n2 = t2.csf.nnz(), nij2 = nnz_at_level(t2.csf, 2);
    ExecPlan tp = prepare(tt, find_path(tt, "((T*V)*U)"),
                          order_of(tt, {{"i", "j", "k", "s"}, {"i", "j", "s", "r"}}), in2);
    CHECK(execute(tp).stats.multiply_adds == 2 * n2 * 2 + 2 * nij2 * 2 * 3);
  });

  run_case("buffers are zero on every producer-subtree entry (observer via device log)", [] {
    KernelSpec spec = ttmc3(5, 4, 4, 3, 2);
    ContractionPath path = find_path(spec, "((T*V)*U)");
    LoopOrder order = order_of(spec, {{"i", "j", "k", "s"}, {"i", "j", "s", "r"}});
    Tensors t = make_tensors(spec, random_coo(spec, 0.2, 41));
    auto in = t.inputs();
    struct Obs : ExecObserver {
      int64_t entries = 0;
      bool all_zero = true;
      void on_producer_entry(int, const double* data, int64_t size) override {
        ++entries;
        for (int64_t i = 0; i < size; ++i)
          if (data[i] != 0.0) all_zero = false;
      }
    } obs;
    ExecOptions opts;
    opts.observer = &obs;
    ExecPlan plan = prepare(spec, path, order, in, opts);
    ExecResult res = execute(plan);
    CHECK(obs.all_zero);
    CHECK(obs.entries == nnz_at_level(t.csf, 2));
    CHECK(res.stats.buffer_resets.size() == 1);
    CHECK(res.stats.buffer_resets[0] == nnz_at_level(t.csf, 2));
    CHECK(close(res, execute_unfactorized(spec, in)));
    // the same counts, analytic, on the fast kernel
    ExecPlan fast = prepare(spec, path, order, in);
    CHECK(spttn_b200_plan_device_kind(fast) == SPTTN_NEST_TTMC3);
    CHECK(execute(fast).stats.buffer_resets == res.stats.buffer_resets);
  });

  run_case("prepare validates shapes, orders and buffer limits", [] {
    KernelSpec spec = ttmc3(3, 3, 3, 2, 2);
    ContractionPath path = find_path(spec, "((T*V)*U)");
    LoopOrder good = order_of(spec, {{"i", "j", "k", "s"}, {"i", "j", "s", "r"}});
    Tensors t = make_tensors(spec, random_coo(spec, 0.3, 1));
    auto in = t.inputs();
    LoopOrder bad = order_of(spec, {{"i", "k", "j", "s"}, {"i", "j", "s", "r"}});
    CHECK(throws_as<unsupported_order_error>([&] { prepare(spec, path, bad, in); }));
    CHECK(throws_as<unsupported_order_error>([&] { flops_estimate(spec, path, bad, t.csf); }));
    Tensors broken = make_tensors(spec, random_coo(spec, 0.3, 1));
    broken.dense[0] = gen_dense({{"j", 3}, {"r", 3}}, 2);
    auto bin = broken.inputs();
    CHECK(throws_as<std::invalid_argument>([&] { prepare(spec, path, good, bin); }));
    ExecInputs none;
    none.dense = in.dense;
    CHECK(throws_as<std::invalid_argument>([&] { prepare(spec, path, good, none); }));
    ExecOptions tiny;
    tiny.buffer_limit_bytes = 4;
    CHECK(throws_as<resource_error>([&] { prepare(spec, path, good, in, tiny); }));
  });

  run_case("sparse-output kernels with densely iterated modes (leaf lookup)", [] {
    KernelSpec spec = tttp3(3, 3, 2, 2);
    Tensors t = make_tensors(spec, random_coo(spec, 0.3, 23));
    auto in = t.inputs();
    ExecResult oracle = execute_unfactorized(spec, in);
    int n = 0;
    for (const auto& path : enumerate_paths(spec))
      for (const auto& order : enumerate_orders(spec, path, default_csf_order(spec))) {
        ExecPlan plan = prepare(spec, path, order, in);
        CHECK(close(execute(plan), oracle));
        ++n;
      }
    CHECK(n > 0);
  });

  run_case("non-root outputs are re-rooted on the device onto the pinned kernels", [] {
    struct Case {
      const char* kernel;
      std::map<std::string, int64_t> dims;
      const char* path;
      int kind;
    };
    const std::vector<Case> cases = {
        {"T[i,j,k]*A[i,a]*C[k,a]->B[j,a]", {{"i", 9}, {"j", 8}, {"k", 7}, {"a", 4}}, "((T*C)*A)",
         SPTTN_NEST_MTTKRP3},
        {"T[i,j,k]*U[i,r]*V[k,s]->Y[j,r,s]", {{"i", 9}, {"j", 8}, {"k", 7}, {"r", 3}, {"s", 2}},
         "((T*V)*U)", SPTTN_NEST_TTMC3},
        {"T[i,j,k]*U[i,r]*V[j,s]->Y[k,r,s]", {{"i", 9}, {"j", 8}, {"k", 7}, {"r", 3}, {"s", 2}},
         "((T*V)*U)", SPTTN_NEST_TTMC3},
        {"T[i,j,k,l]*A[i,r]*B[j,r]*C[k,r]->D[l,r]",
         {{"i", 5}, {"j", 4}, {"k", 6}, {"l", 5}, {"r", 4}}, "(((T*C)*B)*A)", SPTTN_NEST_MTTKRP4},
    };
    for (const auto& c : cases) {
      KernelSpec spec = parse_kernel(c.kernel, c.dims);
      Tensors t = make_tensors(spec, random_coo(spec, 0.2, 17));
      auto in = t.inputs();
      ExecResult oracle = execute_unfactorized(spec, in);
      int routed = 0, n = 0;
      for (const auto& path : filter_min_depth(enumerate_paths(spec))) {
        if (path.describe(spec) != c.path) continue;
        for (const auto& order : enumerate_orders(spec, path, default_csf_order(spec))) {
          ExecPlan plan = prepare(spec, path, order, in);
          routed += spttn_b200_plan_device_kind(plan) == c.kind;
          ExecResult r = execute(plan);
          CHECK(close(r, oracle));
          CHECK(r.stats.multiply_adds == flops_estimate(spec, path, order, t.csf));
          ++n;
        }
      }
      CHECK(n > 0);
      CHECK(routed == n);
    }
  });

  run_case("JIT-compiled nests: sequential JIT equals the interpreter bit for bit, parallel JIT "
           "decompositions (slices, fibers, accumulator tails) match (TTTc-4, sparse out, other paths)", [] {
    struct Case {
      KernelSpec spec;
      double density;
      int max_orders;
    };
    std::vector<Case> cases;
    cases.push_back({tttc4(5, 3), 0.3, 12});
    cases.push_back({tttc4(9, 2), 0.5, 6});
    cases.push_back({mttkrp3(12, 11, 10, 4), 0.2, 12});
    cases.push_back({tttp3(7, 6, 5, 3), 0.3, 12});
    for (auto& c : cases) {
      Tensors t = make_tensors(c.spec, random_coo(c.spec, c.density, 29));
      auto in = t.inputs();
      ExecResult oracle = execute_unfactorized(c.spec, in);
      int n = 0;
      for (const auto& path : filter_min_depth(enumerate_paths(c.spec)))
        for (const auto& order : enumerate_orders(c.spec, path, default_csf_order(c.spec))) {
          if (n >= c.max_orders) break;
          auto plan = [&](const char* jit, const char* par) {
            setenv("SPTTN_GENERIC_JIT", jit, 1);
            setenv("SPTTN_GENERIC_PAR", par, 1);
            ExecPlan p = prepare(c.spec, path, order, in);
            unsetenv("SPTTN_GENERIC_JIT");
            unsetenv("SPTTN_GENERIC_PAR");
            return p;
          };
          ExecPlan pj = plan("1", "1"), pjs = plan("1", "0"), pis = plan("0", "0"), pi = plan("0", "1");
          if (spttn_b200_plan_device_kind(pj) != SPTTN_NEST_GENERIC) continue;
          ExecResult rj = execute(pj), rjs = execute(pjs), ris = execute(pis), ri = execute(pi);
          CHECK(rjs.dense_out.values == ris.dense_out.values);
          CHECK(rjs.sparse_out_values == ris.sparse_out_values);
          for (const ExecResult* r : {&rj, &rjs, &ri}) {
            CHECK(r->stats.multiply_adds == ris.stats.multiply_adds);
            CHECK(r->stats.buffer_resets == ris.stats.buffer_resets);
            CHECK(close(*r, oracle));
          }
          ++n;
        }
      CHECK(n > 0);
    }
  });

  run_case("device build_csf equals the reference build_csf (any mode order)", [] {
    CooTensor coo;
    coo.indices = {{"i", 23}, {"j", 17}, {"k", 29}};
    uint64_t x = 88172645463325252ull;
    auto next = [&](int64_t m) {
      x ^= x << 13; x ^= x >> 7; x ^= x << 17;
      return static_cast<int64_t>(x % static_cast<uint64_t>(m));
    };
    std::set<std::vector<int64_t>> seen;  // distinct rows, then duplicate PAIRS only:
    while (coo.entries.size() < 2500) {   // (a+b == b+a; the order std::sort gives 3+
      std::vector<int64_t> c{next(23), next(17), next(29)};  // duplicates is unspecified)
      if (seen.insert(c).second) coo.entries.push_back({c, (next(2000) - 1000) / 997.0});
    }
    for (int e = 0; e < 300; ++e)
      coo.entries.push_back({coo.entries[e].first, (next(2000) - 1000) / 991.0});
    for (const auto& order : std::vector<std::vector<std::string>>{{"i", "j", "k"}, {"k", "i", "j"}}) {
      CooTensor norm = coo;
      norm.normalize();
      CsfTensor want = build_csf(norm, order);
      CsfTensor got = spttn_b200_build_csf(coo, order);
      CHECK(got.idx == want.idx);
      CHECK(got.ptr == want.ptr);
      CHECK(got.values == want.values);
      CHECK(got.modes.size() == want.modes.size() && got.modes[0].name == want.modes[0].name);
    }
    CooTensor bad = coo;
    bad.entries.push_back({{23, 0, 0}, 1.0});
    CHECK(throws_as<std::invalid_argument>([&] { spttn_b200_build_csf(bad, {"i", "j", "k"}); }));
    CHECK(throws_as<std::invalid_argument>([&] { spttn_b200_build_csf(coo, {"i", "j", "j"}); }));
  });

  run_case("pinned nests at BASELINE ranks run on their kernels and match", [] {
    struct K {
      KernelSpec spec;
      const char* path;
      std::vector<std::vector<std::string>> order;
      int kind;
      double density;
    };
    std::vector<K> ks = {
        {mttkrp3(20, 16, 24, 32), "((T*C)*B)", {{"i", "j", "k", "a"}, {"i", "j", "a"}},
         SPTTN_NEST_MTTKRP3, 0.05},
        {ttmc3(24, 24, 24, 16, 16), "((T*V)*U)", {{"i", "j", "k", "s"}, {"i", "j", "s", "r"}},
         SPTTN_NEST_TTMC3, 0.02},
        {tttp3(16, 12, 10, 64), "(((U*V)*W)*T)", {{"i", "j", "r"}, {"i", "j", "k", "r"}, {"i", "j", "k"}},
         SPTTN_NEST_TTTP3, 0.1},
        {ttmc4(7, 8, 8, 8), "(((T*W)*V)*U)",
         {{"i", "j", "k", "l", "t"}, {"i", "j", "k", "s", "t"}, {"i", "j", "r", "s", "t"}},
         SPTTN_NEST_TTMC4, 0.08},
        {parse_kernel("T[i,j,k,l]*B[j,r]*C[k,r]*D[l,r]->A[i,r]",
                      {{"i", 9}, {"j", 8}, {"k", 7}, {"l", 10}, {"r", 32}}),
         "(((T*D)*C)*B)", {{"i", "j", "k", "l", "r"}, {"i", "j", "k", "r"}, {"i", "j", "r"}},
         SPTTN_NEST_MTTKRP4, 0.05},
    };
    for (auto& k : ks) {
      Tensors t = make_tensors(k.spec, random_coo(k.spec, k.density, 77));
      auto in = t.inputs();
      ContractionPath path = find_path(k.spec, k.path);
      LoopOrder order = order_of(k.spec, k.order);
      ExecPlan plan = prepare(k.spec, path, order, in);
      CHECK(spttn_b200_plan_device_kind(plan) == k.kind);
      ExecResult res = execute(plan);
      CHECK(close(res, execute_unfactorized(k.spec, in)));
      CHECK(res.stats.multiply_adds == flops_estimate(k.spec, path, order, t.csf));
    }
  });

  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
