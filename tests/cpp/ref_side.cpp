// Reference side of the drop-in pinning test — see ref_side.hpp. Compiled
// with -Dspttn=spttn_ref: every reference symbol used here is the renamed
// reference library (oracle/_ref), never the drop-in.
#include "ref_side.hpp"

#include <memory>
#include <stdexcept>

#include "fixtures.hpp"
#include "spttn/executor.hpp"
#include "spttn/loop_nest.hpp"

namespace refpin {
namespace {

using namespace spttn;
using namespace spttn::testing;

KernelSpec make_spec(const FixtureDesc& d) {
  const auto& s = d.shape;
  if (d.kind == "mttkrp3") return mttkrp3(s[0], s[1], s[2], s[3]);
  if (d.kind == "ttmc3") return ttmc3(s[0], s[1], s[2], s[3], s[4]);
  if (d.kind == "tttp3") return tttp3(s[0], s[1], s[2], s[3]);
  if (d.kind == "ttmc4") return ttmc4(s[0], s[1], s[2], s[3]);
  if (d.kind == "tttc4") return tttc4(s[0], s[1]);
  if (d.kind == "tttc6") return tttc6(s[0], s[1]);
  throw std::invalid_argument("unknown fixture kind " + d.kind);
}

struct Fx {
  KernelSpec spec;
  Tensors tensors;
  std::vector<ContractionPath> paths;
};

std::vector<std::unique_ptr<Fx>>& registry() {
  static std::vector<std::unique_ptr<Fx>> r;
  return r;
}

Result to_result(const ExecResult& r) {
  Result o;
  o.dense = r.dense_out.values;
  o.sparse = r.sparse_out_values;
  o.multiply_adds = r.stats.multiply_adds;
  o.buffer_resets = r.stats.buffer_resets;
  return o;
}

}  // namespace

void ref_register(const std::vector<FixtureDesc>& fixtures) {
  auto& reg = registry();
  reg.clear();
  for (const auto& d : fixtures) {
    auto fx = std::make_unique<Fx>();
    fx->spec = make_spec(d);
    fx->tensors = make_tensors(fx->spec, random_coo(fx->spec, d.density, d.seed));
    fx->paths = enumerate_paths(fx->spec);
    reg.push_back(std::move(fx));
  }
}

Result ref_execute(int f, int path, const std::vector<std::vector<std::string>>& order) {
  Fx& fx = *registry().at(static_cast<size_t>(f));
  LoopOrder o;
  for (const auto& term : order) {
    std::vector<int> ids;
    for (const auto& n : term) ids.push_back(fx.spec.index_id(n));
    o.per_term.push_back(ids);
  }
  ExecPlan plan = prepare(fx.spec, fx.paths.at(static_cast<size_t>(path)), o, fx.tensors.inputs());
  return to_result(execute(plan));
}

Result ref_unfactorized(int f) {
  Fx& fx = *registry().at(static_cast<size_t>(f));
  return to_result(execute_unfactorized(fx.spec, fx.tensors.inputs()));
}

int64_t ref_nnz(int f) { return registry().at(static_cast<size_t>(f))->tensors.csf.nnz(); }

}  // namespace refpin
