// Per-plan overhead of the drop-in executor on tiny tensors (the regime of
// the reference's acceptance criterion 6: every admissible order of small
// fixtures). Prints the mean prepare+execute time over the first N orders of
// the TTTc-4 fixture and of the order-3 fixtures.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "fixtures.hpp"
#include "spttn/executor.hpp"

using namespace spttn;
using namespace spttn::testing;

int main(int argc, char** argv) {
  const int limit = argc > 1 ? std::atoi(argv[1]) : 200;
  const char* only = argc > 2 ? argv[2] : nullptr;  // run one fixture
  struct F {
    const char* name;
    KernelSpec spec;
    double density;
  };
  F fs[] = {{"MTTKRP-3", mttkrp3(5, 4, 4, 3), 0.15}, {"TTMc-3", ttmc3(5, 4, 4, 3, 2), 0.15},
            {"TTTP-3", tttp3(4, 4, 3, 2), 0.2}, {"TTMc-4", ttmc4(3, 2, 2, 2), 0.15},
            {"TTTc-4", tttc4(3, 2), 0.15}};
  for (auto& f : fs) {
    if (only && std::string(only) != f.name) continue;
    Tensors t = make_tensors(f.spec, random_coo(f.spec, f.density, 101));
    auto in = t.inputs();
    ExecResult oracle = execute_unfactorized(f.spec, in);
    int n = 0, bad = 0;
    double prep = 0, exec = 0;
    for (const auto& path : filter_min_depth(enumerate_paths(f.spec))) {
      for (const auto& order : enumerate_orders(f.spec, path, default_csf_order(f.spec))) {
        if (n >= limit) break;
        auto t0 = std::chrono::steady_clock::now();
        ExecPlan plan = prepare(f.spec, path, order, in);
        auto t1 = std::chrono::steady_clock::now();
        ExecResult r = execute(plan);
        auto t2 = std::chrono::steady_clock::now();
        prep += std::chrono::duration<double>(t1 - t0).count();
        exec += std::chrono::duration<double>(t2 - t1).count();
        double m = 0;
        for (size_t i = 0; i < r.dense_out.values.size(); ++i)
          m = std::max(m, std::abs(r.dense_out.values[i] - oracle.dense_out.values[i]));
        for (size_t i = 0; i < r.sparse_out_values.size(); ++i)
          m = std::max(m, std::abs(r.sparse_out_values[i] - oracle.sparse_out_values[i]));
        bad += m > 1e-10;
        ++n;
      }
    }
    std::printf("%-9s orders %5d  prepare %8.1f us  execute %8.1f us  mismatches %d\n", f.name, n,
                1e6 * prep / n, 1e6 * exec / n, bad);
  }
  return 0;
}
