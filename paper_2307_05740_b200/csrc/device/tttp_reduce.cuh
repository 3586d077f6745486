// Transpose-reduction shared by the TTTP kernels (nest_tttp.cu,
// tttp_buckets.cu): U partial dot products spread over a group of G lanes
// are combined with 2U-1 shuffles (log2 U halving exchanges, then a plain
// butterfly), after which lane (G/U)*q holds leaf q's sum.
#pragma once

namespace spttn_dev {
namespace {

template <int G, int U>
__device__ __forceinline__ double transpose_reduce(double (&v)[U], int lane_in_group, int* leaf) {
  // halving exchanges: after them each lane holds one leaf's partial sum
  int q = 0;
  int o = G / 2;
#pragma unroll
  for (int n = U; n > 1; n >>= 1, o >>= 1) {
    const int half = n / 2;
    const bool hi = (lane_in_group & o) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const double send = hi ? v[i] : v[i + half];
      const double keep = hi ? v[i + half] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
    q = (q << 1) | (hi ? 1 : 0);
  }
  double s = v[0];
#pragma unroll
  for (; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  *leaf = q;
  return s;
}

}  // namespace
}  // namespace spttn_dev
