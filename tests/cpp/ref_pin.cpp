// Pins every device path of the drop-in to the reference executor itself
// (TEST INFRASTRUCTURE). For each fixture, every admissible loop order of
// every minimum-depth contraction path (the enumeration of the reference's
// acceptance criterion 6, proj/tests/acceptance.cpp:248-274) — or a seeded
// sample of them where the space is too large (TTTc-6: 84.7 M orders) — runs
// through spttn::prepare / spttn::execute (the drop-in: pinned sm_100a
// kernels, the device forest interpreter, the NVRTC-compiled forests) and
// through spttn_ref::prepare / execute (the reference library compiled from
// /root/reference/proj/src, renamed; ref_side.cpp). Checked per order:
//  * output: bit-identical where the device path claims it (the forest
//    interpreter walking root slices in the reference's order, decompositions
//    0 and 1), otherwise within the reference's own tolerance
//    1e-10 * (1 + max|ref|) (proj/tests/test_executor.cpp:24-29);
//  * ExecStats::multiply_adds and buffer_resets equal to the reference's;
//  * sparse-output length = nnz.
// And per fixture: the device execute_unfactorized bit-identical to
// spttn_ref::execute_unfactorized.
//
//   ref_pin [--quick]      --quick samples TTTc-4 (every 97th order)
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "fixtures.hpp"
#include "ref_side.hpp"
#include "spttn/executor.hpp"
#include "spttn/contraction_path.hpp"
#include "spttn/loop_nest.hpp"
#include "spttn_b200.h"
#include "spttn_b200_shim.hpp"

using namespace spttn;
using namespace spttn::testing;

namespace {

KernelSpec make_spec(const refpin::FixtureDesc& d) {
  const auto& s = d.shape;
  if (d.kind == "mttkrp3") return mttkrp3(s[0], s[1], s[2], s[3]);
  if (d.kind == "ttmc3") return ttmc3(s[0], s[1], s[2], s[3], s[4]);
  if (d.kind == "tttp3") return tttp3(s[0], s[1], s[2], s[3]);
  if (d.kind == "ttmc4") return ttmc4(s[0], s[1], s[2], s[3]);
  if (d.kind == "tttc4") return tttc4(s[0], s[1]);
  return tttc6(s[0], s[1]);
}

std::vector<std::vector<std::string>> names_of(const KernelSpec& spec, const LoopOrder& o) {
  std::vector<std::vector<std::string>> out;
  for (const auto& term : o.per_term) {
    std::vector<std::string> t;
    for (int id : term) t.push_back(spec.index_names[id]);
    out.push_back(t);
  }
  return out;
}

bool same_bits(const std::vector<double>& a, const std::vector<double>& b) {
  return a.size() == b.size() &&
         (a.empty() || std::memcmp(a.data(), b.data(), a.size() * sizeof(double)) == 0);
}

double max_abs(const std::vector<double>& a) {
  double m = 0;
  for (double v : a) m = std::max(m, std::abs(v));
  return m;
}

double max_delta(const std::vector<double>& a, const std::vector<double>& b) {
  if (a.size() != b.size()) return INFINITY;
  double m = 0;
  for (size_t i = 0; i < a.size(); ++i) m = std::max(m, std::abs(a[i] - b[i]));
  return m;
}

struct Tally {
  int64_t orders = 0, bit_identical = 0, exact_required = 0, failures = 0;
  int64_t by_route[8] = {0};  // pinned, interp seq, interp slices, interp ranges, jit
  double worst = 0;
};

}  // namespace

int main(int argc, char** argv) {
  const bool quick = argc > 1 && std::string(argv[1]) == "--quick";
  // acceptance fixture_set() (acceptance.cpp:83-95, coordinates seed 101 as
  // in criterion 6) + TTTc-6 (fixtures.hpp:42-47) + BASELINE-like shapes
  // through the dedicated kernels + a TTTc-4 large enough for the JIT path
  const std::vector<refpin::FixtureDesc> fx = {
      {"MTTKRP-3", "mttkrp3", {5, 4, 4, 3}, 0.15, 101},
      {"TTMc-3", "ttmc3", {5, 4, 4, 3, 2}, 0.15, 101},
      {"TTTP-3", "tttp3", {4, 4, 3, 2}, 0.2, 101},
      {"TTMc-4", "ttmc4", {3, 2, 2, 2}, 0.15, 101},
      {"TTTc-4", "tttc4", {3, 2}, 0.15, 101},
      {"TTTc-6", "tttc6", {3, 2}, 0.15, 101},
      {"MTTKRP-3 R32", "mttkrp3", {60, 50, 40, 32}, 0.05, 7},
      {"TTMc-3 R16", "ttmc3", {60, 50, 40, 16, 16}, 0.05, 8},
      {"TTTP-3 R64", "tttp3", {40, 30, 20, 64}, 0.1, 9},
      {"TTMc-4 R8", "ttmc4", {16, 8, 8, 8}, 0.05, 10},
      {"TTTc-4 N20 (JIT)", "tttc4", {20, 2}, 0.45, 11},
      {"TTTc-6 N7 (JIT)", "tttc6", {7, 2}, 0.6, 12},
  };
  // orders per fixture: 0 = all; >0 = a seeded sample of that many
  const std::vector<int64_t> sample = {0, 0, 0, 0, quick ? 20000 : 0, 3000, 48, 96, 60, 60, 6, 4};
  refpin::ref_register(fx);
  int total_fail = 0;
  const auto t_start = std::chrono::steady_clock::now();
  for (size_t f = 0; f < fx.size(); ++f) {
    const KernelSpec spec = make_spec(fx[f]);
    Tensors t = make_tensors(spec, random_coo(spec, fx[f].density, fx[f].seed));
    const auto in = t.inputs();
    Tally tl;
    // unfactorized: device vs reference, bit for bit
    {
      ExecResult u = execute_unfactorized(spec, in);
      refpin::Result ru = refpin::ref_unfactorized(static_cast<int>(f));
      const bool ok = same_bits(u.dense_out.values, ru.dense) &&
                      same_bits(u.sparse_out_values, ru.sparse) &&
                      u.stats.multiply_adds == ru.multiply_adds;
      if (!ok) {
        std::printf("  FAIL %s: execute_unfactorized differs from spttn_ref (max delta %.3g)\n",
                    fx[f].name.c_str(),
                    std::max(max_delta(u.dense_out.values, ru.dense),
                             max_delta(u.sparse_out_values, ru.sparse)));
        ++tl.failures;
      }
    }
    const std::vector<int> csf_order = default_csf_order(spec);
    // minimum-depth paths (filter_min_depth, contraction_path.cpp:117-125) by
    // their position in enumerate_paths, which the reference side shares
    const auto all_paths = enumerate_paths(spec);
    int best = max_loop_depth(all_paths[0]);
    for (const auto& p : all_paths) best = std::min(best, max_loop_depth(p));
    std::vector<int> path_ids;
    for (size_t k = 0; k < all_paths.size(); ++k)
      if (max_loop_depth(all_paths[k]) == best) path_ids.push_back(static_cast<int>(k));
    std::vector<std::pair<int, LoopOrder>> work;
    if (sample[f] == 0) {
      for (int id : path_ids)
        for_each_order(spec, all_paths[id], csf_order,
                       [&](const LoopOrder& o) { work.emplace_back(id, o); });
    } else {
      // seeded sample: a path, then one admissible order per term
      std::mt19937_64 rng(1234 + f);
      std::vector<std::vector<std::vector<std::vector<int>>>> per_path;
      for (int id : path_ids) {
        const auto& p = all_paths[id];
        std::vector<std::vector<std::vector<int>>> terms;
        for (int k = 0; k < p.num_terms(); ++k)
          terms.push_back(enumerate_term_orders(spec, p, k, csf_order));
        per_path.push_back(std::move(terms));
      }
      for (int64_t s = 0; s < sample[f]; ++s) {
        const size_t pi = rng() % path_ids.size();
        LoopOrder o;
        for (const auto& choices : per_path[pi]) o.per_term.push_back(choices[rng() % choices.size()]);
        if (!order_admissible(spec, all_paths[path_ids[pi]], o, csf_order)) continue;
        work.emplace_back(path_ids[pi], o);
      }
    }
    for (const auto& [pid, order] : work) {
      const ContractionPath& path = all_paths[pid];
      ExecPlan plan = prepare(spec, path, order, in);
      ExecResult got = execute(plan);
      refpin::Result want = refpin::ref_execute(static_cast<int>(f), pid, names_of(spec, order));
      int64_t info[10];
      // route: 0 pinned kernel, 1 + decomposition (interpreter), 5 JIT
      int route = 0;
      if (spttn_b200_plan_device_kind(plan) == SPTTN_NEST_GENERIC) {
        spttn_b200_plan_info(plan, info, 10);
        route = info[9] == 1 ? 5 : 1 + static_cast<int>(info[8]);
      }
      ++tl.by_route[route];
      ++tl.orders;
      const bool bits = same_bits(got.dense_out.values, want.dense) &&
                        same_bits(got.sparse_out_values, want.sparse);
      tl.bit_identical += bits;
      const bool exact = route == 1 || route == 2;  // walk in the reference's order
      tl.exact_required += exact;
      const double tol = 1e-10 * (1.0 + std::max(max_abs(want.dense), max_abs(want.sparse)));
      const double d = std::max(max_delta(got.dense_out.values, want.dense),
                                max_delta(got.sparse_out_values, want.sparse));
      tl.worst = std::max(tl.worst, d);
      const bool stats_ok = got.stats.multiply_adds == want.multiply_adds &&
                            got.stats.buffer_resets == want.buffer_resets;
      const bool ok = (exact ? bits : d <= tol) && stats_ok &&
                      (!spec.output_sparse ||
                       got.sparse_out_values.size() == static_cast<size_t>(t.csf.nnz()));
      if (!ok) {
        if (tl.failures < 5)
          std::printf("  FAIL %s %s route %d: bits %d delta %.3g tol %.3g madds %lld/%lld resets %s\n",
                      fx[f].name.c_str(), path.describe(spec).c_str(), route, bits, d, tol,
                      static_cast<long long>(got.stats.multiply_adds),
                      static_cast<long long>(want.multiply_adds),
                      got.stats.buffer_resets == want.buffer_resets ? "ok" : "differ");
        ++tl.failures;
      }
    }
    const double el =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
    std::printf("%-18s nnz %6lld orders %8lld (%s)  bit-identical %8lld (required %lld)  "
                "routes pinned/seq/slices/ranges/fibers/jit %lld/%lld/%lld/%lld/%lld/%lld  "
                "max|delta| %.2e  failures %lld  [%.1fs]\n",
                fx[f].name.c_str(), static_cast<long long>(t.csf.nnz()),
                static_cast<long long>(tl.orders), sample[f] ? "sampled" : "all",
                static_cast<long long>(tl.bit_identical), static_cast<long long>(tl.exact_required),
                static_cast<long long>(tl.by_route[0]), static_cast<long long>(tl.by_route[1]),
                static_cast<long long>(tl.by_route[2]), static_cast<long long>(tl.by_route[3]),
                static_cast<long long>(tl.by_route[4]), static_cast<long long>(tl.by_route[5]),
                tl.worst, static_cast<long long>(tl.failures), el);
    std::fflush(stdout);
    total_fail += tl.failures > 0;
  }
  std::printf(total_fail ? "REF PIN FAILED\n" : "REF PIN OK\n");
  return total_fail ? 1 : 0;
}
