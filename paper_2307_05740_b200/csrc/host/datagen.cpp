// Host-side synthetic tensor generation and COO -> CSF construction.
//
// Two families of generators live here:
//  * reference-compatible ones, restated from the reference library so that
//    test fixtures reproduce the reference's own test inputs bit-for-bit:
//      gen_random  (Floyd sampling over mt19937_64)  proj/src/tns_io.cpp:123-159
//      gen_dense   (uniform(-1,1) "unit_value")      proj/src/tns_io.cpp:161-166
//      stable_hash (FNV-1a)                          proj/src/tns_io.cpp:168-175
//      bounded / unit_value                          proj/src/tns_io.cpp:108-119
//  * the BASELINE.json synthetic workloads: distinct
//    uniform-random or Zipf(s) coordinates kept in first-draw order, values
//    unit_value, factors N(0, sigma^2) by Box-Muller.
//
// The CSF produced is the reference's CsfTensor layout (int64 idx/ptr per
// level, fp64 values; proj/include/spttn/tensor.hpp:49-57, built like
// build_csf proj/src/tensor.cpp:41-94 from lexicographically sorted rows).
// Sorting uses an LSD radix sort over linearised coordinates.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_set>
#include <vector>

namespace {

thread_local std::string g_err;

uint64_t stable_hash(const char* s) {
  uint64_t h = 1469598103934665603ull;
  for (const unsigned char* p = reinterpret_cast<const unsigned char*>(s); *p; ++p) {
    h ^= *p;
    h *= 1099511628211ull;
  }
  return h;
}

uint64_t bounded(std::mt19937_64& rng, uint64_t n) {
  const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
  uint64_t x;
  do {
    x = rng();
  } while (x >= limit);
  return x % n;
}

double unit_value(std::mt19937_64& rng) {
  return 2.0 * (static_cast<double>(rng() >> 11) * 0x1.0p-53) - 1.0;
}

double uniform01(std::mt19937_64& rng) { return static_cast<double>(rng() >> 11) * 0x1.0p-53; }

struct Csf {
  int order = 0;
  int64_t dims[8] = {0};
  std::vector<int64_t> idx[8];
  std::vector<int64_t> ptr[8];
  std::vector<double> values;
};

// Stable LSD radix sort of (key, payload) pairs by key.
void radix_sort(std::vector<uint64_t>& keys, std::vector<uint64_t>& pay, int key_bits) {
  const size_t n = keys.size();
  std::vector<uint64_t> k2(n), p2(n);
  constexpr int B = 11;
  constexpr size_t NB = size_t{1} << B;
  for (int shift = 0; shift < key_bits; shift += B) {
    std::vector<size_t> cnt(NB + 1, 0);
    for (size_t i = 0; i < n; ++i) ++cnt[((keys[i] >> shift) & (NB - 1)) + 1];
    for (size_t b = 0; b < NB; ++b) cnt[b + 1] += cnt[b];
    for (size_t i = 0; i < n; ++i) {
      const size_t d = cnt[(keys[i] >> shift) & (NB - 1)]++;
      k2[d] = keys[i];
      p2[d] = pay[i];
    }
    keys.swap(k2);
    pay.swap(p2);
  }
}

int bits_for(uint64_t total) {
  int b = 1;
  while (b < 64 && (uint64_t{1} << b) < total) ++b;
  return b;
}

// Sorted, distinct linear keys + values -> CSF with root-to-leaf = declared order.
Csf* csf_from_sorted_keys(int d, const int64_t* dims, const std::vector<uint64_t>& keys,
                          const std::vector<double>& vals) {
  auto* c = new Csf;
  c->order = d;
  for (int l = 0; l < d; ++l) c->dims[l] = dims[l];
  const size_t n = keys.size();
  std::vector<int64_t> prev(d, -1), cur(d);
  c->values = vals;
  for (size_t e = 0; e < n; ++e) {
    uint64_t rest = keys[e];
    for (int l = d - 1; l >= 0; --l) {
      cur[l] = static_cast<int64_t>(rest % static_cast<uint64_t>(dims[l]));
      rest /= static_cast<uint64_t>(dims[l]);
    }
    bool changed = e == 0;
    for (int l = 0; l < d; ++l) {
      if (!changed && cur[l] != prev[l]) changed = true;
      if (changed) {
        if (l + 1 < d) c->ptr[l].push_back(static_cast<int64_t>(c->idx[l + 1].size()));
        c->idx[l].push_back(cur[l]);
      }
    }
    prev = cur;
  }
  for (int l = 0; l + 1 < d; ++l) c->ptr[l].push_back(static_cast<int64_t>(c->idx[l + 1].size()));
  return c;
}

uint64_t linear_total(int d, const int64_t* dims) {
  long double t = 1;
  uint64_t total = 1;
  for (int l = 0; l < d; ++l) {
    if (dims[l] < 1) throw std::invalid_argument("dimensions must be >= 1");
    t *= dims[l];
    total *= static_cast<uint64_t>(dims[l]);
  }
  if (t > static_cast<long double>(UINT64_MAX / 2))
    throw std::invalid_argument("linearised coordinate space exceeds 63 bits");
  return total;
}

}  // namespace

extern "C" {

const char* dg_last_error() { return g_err.c_str(); }

uint64_t dg_stable_hash(const char* s) { return stable_hash(s); }

// ---- CSF handle accessors --------------------------------------------------
int dg_csf_order(void* h) { return static_cast<Csf*>(h)->order; }
int64_t dg_csf_level_size(void* h, int l) {
  return static_cast<int64_t>(static_cast<Csf*>(h)->idx[l].size());
}
int64_t dg_csf_dim(void* h, int l) { return static_cast<Csf*>(h)->dims[l]; }
const int64_t* dg_csf_idx(void* h, int l) { return static_cast<Csf*>(h)->idx[l].data(); }
const int64_t* dg_csf_ptr(void* h, int l) { return static_cast<Csf*>(h)->ptr[l].data(); }
const double* dg_csf_values(void* h) { return static_cast<Csf*>(h)->values.data(); }
void dg_csf_free(void* h) { delete static_cast<Csf*>(h); }

// COO (nnz x d row-major) -> normalize (sort, sum duplicates; tensor.cpp:24-35)
// -> CSF in declared mode order.
void* dg_csf_from_coo(int d, const int64_t* dims, int64_t nnz, const int64_t* coords,
                      const double* values) {
  try {
    const uint64_t total = linear_total(d, dims);
    std::vector<uint64_t> keys(nnz), pay(nnz);
    for (int64_t e = 0; e < nnz; ++e) {
      uint64_t k = 0;
      for (int l = 0; l < d; ++l) {
        const int64_t c = coords[e * d + l];
        if (c < 0 || c >= dims[l]) throw std::invalid_argument("coordinate out of bounds");
        k = k * static_cast<uint64_t>(dims[l]) + static_cast<uint64_t>(c);
      }
      keys[e] = k;
      pay[e] = static_cast<uint64_t>(e);
    }
    radix_sort(keys, pay, bits_for(total));
    std::vector<uint64_t> uk;
    std::vector<double> uv;
    for (int64_t e = 0; e < nnz; ++e) {
      if (!uk.empty() && uk.back() == keys[e])
        uv.back() += values[pay[e]];
      else {
        uk.push_back(keys[e]);
        uv.push_back(values[pay[e]]);
      }
    }
    return csf_from_sorted_keys(d, dims, uk, uv);
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

// Reference-compatible gen_random (tns_io.cpp:123-159) + build_csf in the
// declared order.
void* dg_gen_random(int d, const int64_t* dims, double density, uint64_t seed) {
  try {
    if (!(density > 0.0) || density > 1.0)
      throw std::invalid_argument("gen_random: density must be in (0, 1]");
    const uint64_t total = linear_total(d, dims);
    const uint64_t count = static_cast<uint64_t>(std::ceil(density * static_cast<double>(total)));
    std::mt19937_64 rng(seed);
    std::unordered_set<uint64_t> chosen;
    chosen.reserve(count * 2);
    for (uint64_t j = total - count; j < total; ++j) {
      const uint64_t t = bounded(rng, j + 1);
      if (!chosen.insert(t).second) chosen.insert(j);
    }
    std::vector<uint64_t> cells(chosen.begin(), chosen.end());
    std::sort(cells.begin(), cells.end());
    std::vector<double> vals(cells.size());
    for (size_t e = 0; e < cells.size(); ++e) vals[e] = unit_value(rng);
    return csf_from_sorted_keys(d, dims, cells, vals);
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

// Reference-compatible gen_dense (tns_io.cpp:161-166): n values uniform(-1,1).
void dg_gen_dense(int64_t n, uint64_t seed, double* out) {
  std::mt19937_64 rng(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = unit_value(rng);
}

// N(0, sigma^2) by Box-Muller on 53-bit uniforms: each draw
// pair (u1 in (0,1], u2 in [0,1)) yields r*cos, r*sin in that order.
void dg_gen_normal(int64_t n, uint64_t seed, double sigma, double* out) {
  std::mt19937_64 rng(seed);
  const double two_pi = 6.283185307179586476925286766559;
  for (int64_t i = 0; i < n; i += 2) {
    const double u1 = (static_cast<double>(rng() >> 11) + 1.0) * 0x1.0p-53;
    const double u2 = uniform01(rng);
    const double r = std::sqrt(-2.0 * std::log(u1));
    out[i] = sigma * r * std::cos(two_pi * u2);
    if (i + 1 < n) out[i + 1] = sigma * r * std::sin(two_pi * u2);
  }
}

// BASELINE synthetic sparse tensor: draws tuples from one
// mt19937_64(seed) stream — per mode a uniform bounded() draw (zipf_s <= 0)
// or a Zipf(zipf_s) rank by inverse CDF over r^-s, r = 1..dim, mapped through
// a per-mode Fisher-Yates permutation seeded seed ^ stable_hash("perm<l>") —
// then one unit_value(); keeps the first nnz distinct tuples in draw order.
void* dg_gen_baseline(int d, const int64_t* dims, int64_t nnz, double zipf_s, uint64_t seed) {
  try {
    const uint64_t total = linear_total(d, dims);
    if (nnz < 0 || static_cast<uint64_t>(nnz) > total)
      throw std::invalid_argument("gen_baseline: nnz exceeds the coordinate space");
    std::vector<std::vector<double>> cdf(d);
    std::vector<std::vector<int64_t>> perm(d);
    if (zipf_s > 0) {
      for (int l = 0; l < d; ++l) {
        cdf[l].resize(dims[l]);
        double acc = 0;
        for (int64_t r = 0; r < dims[l]; ++r) {
          acc += std::pow(static_cast<double>(r + 1), -zipf_s);
          cdf[l][r] = acc;
        }
        perm[l].resize(dims[l]);
        for (int64_t r = 0; r < dims[l]; ++r) perm[l][r] = r;
        std::string tag = "perm" + std::to_string(l);
        std::mt19937_64 prng(seed ^ stable_hash(tag.c_str()));
        for (int64_t r = dims[l] - 1; r > 0; --r) {
          const int64_t q = static_cast<int64_t>(bounded(prng, static_cast<uint64_t>(r + 1)));
          std::swap(perm[l][r], perm[l][q]);
        }
      }
    }
    std::mt19937_64 rng(seed);
    std::vector<uint64_t> draw_key;
    std::vector<double> draw_val;
    std::vector<uint8_t> first;  // first occurrence flag per draw
    int64_t distinct = 0;
    int64_t want_draws = nnz + nnz / 8 + 1024;
    while (distinct < nnz) {
      const int64_t old = static_cast<int64_t>(draw_key.size());
      draw_key.resize(want_draws);
      draw_val.resize(want_draws);
      for (int64_t n = old; n < want_draws; ++n) {
        uint64_t k = 0;
        for (int l = 0; l < d; ++l) {
          uint64_t c;
          if (zipf_s > 0) {
            const double u = uniform01(rng) * cdf[l].back();
            const auto it = std::upper_bound(cdf[l].begin(), cdf[l].end(), u);
            int64_t rank = it - cdf[l].begin();
            if (rank >= dims[l]) rank = dims[l] - 1;
            c = static_cast<uint64_t>(perm[l][rank]);
          } else {
            c = bounded(rng, static_cast<uint64_t>(dims[l]));
          }
          k = k * static_cast<uint64_t>(dims[l]) + c;
        }
        draw_key[n] = k;
        draw_val[n] = unit_value(rng);
      }
      // distinct count: stable sort (key, draw index); first of each run wins.
      std::vector<uint64_t> keys(draw_key), pay(want_draws);
      for (int64_t n = 0; n < want_draws; ++n) pay[n] = static_cast<uint64_t>(n);
      radix_sort(keys, pay, bits_for(total));
      first.assign(want_draws, 0);
      distinct = 0;
      for (int64_t e = 0; e < want_draws; ++e)
        if (e == 0 || keys[e] != keys[e - 1]) {
          first[pay[e]] = 1;
          ++distinct;
        }
      want_draws = want_draws + (want_draws / 2) + 1024;
    }
    std::vector<uint64_t> keys, pay;
    keys.reserve(nnz);
    pay.reserve(nnz);
    for (size_t n = 0; n < first.size() && static_cast<int64_t>(keys.size()) < nnz; ++n)
      if (first[n]) {
        keys.push_back(draw_key[n]);
        pay.push_back(n);
      }
    radix_sort(keys, pay, bits_for(total));
    std::vector<double> vals(keys.size());
    for (size_t e = 0; e < keys.size(); ++e) vals[e] = draw_val[pay[e]];
    return csf_from_sorted_keys(d, dims, keys, vals);
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

// Sub-tensor made of every `stride`-th root slice starting at `offset`
// (bounded CPU-baseline samples; slices are copied whole).
void* dg_csf_root_sample(void* h, int64_t stride, int64_t offset) {
  const Csf* s = static_cast<Csf*>(h);
  auto* c = new Csf;
  c->order = s->order;
  const int d = s->order;
  for (int l = 0; l < d; ++l) c->dims[l] = s->dims[l];
  std::vector<std::pair<int64_t, int64_t>> ranges;  // per level node ranges
  for (int64_t p0 = offset; p0 < static_cast<int64_t>(s->idx[0].size()); p0 += stride)
    ranges.emplace_back(p0, p0 + 1);
  for (int l = 0; l < d; ++l) {
    std::vector<std::pair<int64_t, int64_t>> next;
    int64_t acc = 0;
    for (auto [b, e] : ranges) {
      for (int64_t p = b; p < e; ++p) {
        c->idx[l].push_back(s->idx[l][p]);
        if (l + 1 < d) {
          c->ptr[l].push_back(acc);
          acc += s->ptr[l][p + 1] - s->ptr[l][p];
        } else {
          c->values.push_back(s->values[p]);
        }
      }
      if (l + 1 < d && e > b) next.emplace_back(s->ptr[l][b], s->ptr[l][e]);
    }
    if (l + 1 < d) c->ptr[l].push_back(acc);
    ranges.swap(next);
  }
  return c;
}

}  // extern "C"
