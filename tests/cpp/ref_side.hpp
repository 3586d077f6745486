// Reference side of the drop-in pinning test (TEST INFRASTRUCTURE).
//
// ref_side.cpp is compiled with -Dspttn=spttn_ref against the reference
// library built from /root/reference/proj/src by oracle/Makefile
// (oracle/_ref/libspttn_ref.a), so the reference executor and the drop-in
// (spttn::, libspttn_b200_host.so) live in one process. This header carries
// only standard-library types across that boundary.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace refpin {

struct Result {
  std::vector<double> dense;   // ExecResult::dense_out.values
  std::vector<double> sparse;  // ExecResult::sparse_out_values
  int64_t multiply_adds = 0;
  std::vector<int64_t> buffer_resets;
};

// Fixture f is rebuilt on the reference side from the same recipe the drop-in
// side uses (proj/tests/fixtures.hpp random_coo + make_tensors, seed given).
struct FixtureDesc {
  std::string name;
  std::string kind;  // mttkrp3 ttmc3 tttp3 ttmc4 tttc4 tttc6
  std::vector<int64_t> shape;
  double density;
  uint64_t seed;
};

void ref_register(const std::vector<FixtureDesc>& fixtures);
// spttn_ref::prepare + execute on enumerate_paths(spec)[path] (describe()
// strings are not unique across paths) with the given per-term orders
// (index names)
Result ref_execute(int fixture, int path,
                   const std::vector<std::vector<std::string>>& order);
Result ref_unfactorized(int fixture);
int64_t ref_nnz(int fixture);

}  // namespace refpin
