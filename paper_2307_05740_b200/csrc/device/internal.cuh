// Internal device-side structures shared by the kernels and the C-ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <unordered_set>
#include <vector>

#include "common.cuh"
#include "program.h"

namespace spttn_dev {

constexpr int kMaxOrder = 8;

// Device CSF: SoA int32 coordinates / child pointers per level, fp64 leaf
// values (cudaMalloc: 256-B aligned, so LDG.256-friendly).
struct CsfView {
  int order;
  int32_t nlev[kMaxOrder];
  const int32_t* idx[kMaxOrder];
  const int32_t* ptr[kMaxOrder];
  const double* vals;
};

struct DevCsf {
  int order = 0;
  int device = 0;
  int64_t dims[kMaxOrder] = {0};
  int64_t level_size[kMaxOrder] = {0};
  int32_t* idx[kMaxOrder] = {nullptr};
  int32_t* ptr[kMaxOrder] = {nullptr};
  double* vals = nullptr;
  int64_t bytes = 0;
  // spttn_csf_create_async: the leaf values arrive on a side stream; every
  // consumer of `vals` orders itself after this event (wait_values)
  cudaEvent_t vals_ready = nullptr;

  void wait_values(cudaStream_t s) const {
    if (vals_ready) cudaStreamWaitEvent(s, vals_ready, 0);
  }

  CsfView view() const {
    CsfView v{};
    v.order = order;
    for (int l = 0; l < order; ++l) {
      v.nlev[l] = static_cast<int32_t>(level_size[l]);
      v.idx[l] = idx[l];
      v.ptr[l] = ptr[l];
    }
    v.vals = vals;
    return v;
  }
};

// Work decomposition shared by the root-output kernels.
//  * group kernels (MTTKRP-3/4, TTTP-3): items are fixed leaf ranges of
//    `chunk` leaves, item_pos[t*order + l] = node at level l holding the
//    item's first leaf.
//  * DMMA kernels (TTMc-3/4): items are fixed ranges of `chunk` segments
//    (a segment = a fiber piece of <= seg_len children), item_pos[t] = root
//    slice holding the item's first segment.
//  Root slices spread over several items are combined by the fix-up kernel
//  from per-item HEAD (slot 0) / TAIL (slot 1) partial tiles in item order.
struct Decomp {
  int64_t n_items = 0;
  int64_t chunk = 0;
  int32_t* item_pos = nullptr;
  double* part = nullptr;  // [n_items][2][tile]
  int64_t tile = 0;
  int64_t n_split = 0;
  int32_t* split_node = nullptr;   // root node ids
  int32_t* split_first = nullptr;  // first item touching it
  int32_t* split_last = nullptr;   // last item touching it
  int64_t n_absent = 0;
  int32_t* absent_rows = nullptr;  // root coordinates absent from the CSF
  // DMMA kernels
  int64_t n_seg = 0;
  int32_t seg_len = 0;
  int32_t* seg_begin = nullptr;    // [n_seg+1] child-node (or leaf) offsets
  int32_t* seg_node = nullptr;     // [n_seg]  coordinate of the segment's fiber
  int32_t* seg_node1 = nullptr;    // [n_seg]  level-1 coordinate (unit level 2 only)
  // two-level fix-up: chunks of <= kFixChunk items per split slice
  int64_t n_chunk = 0;
  int4* chunk_meta = nullptr;  // per chunk {lo, hi, first item, out row or -(1 + part2 slot)}
  int32_t* chunk_split = nullptr;
  int32_t* chunk_lo = nullptr;
  int32_t* chunk_hi = nullptr;
  int32_t* split_chunk = nullptr;  // [n_split+1] first chunk of each split slice
  double* part2 = nullptr;         // [n_chunk][tile]
  int64_t n_multi = 0;
  int32_t* multi_split = nullptr;  // split slices with more than one chunk (pass 2)
  // packed groups (pack.cu): header {leaf_base, len, nseg, slice} per group
  int64_t n_groups = 0;
  int64_t n_packed_leaves = 0;
  int pack_slots = 0;
  int4* grp_hdr = nullptr;
  int32_t* grp_node = nullptr;     // [n_groups][8] fiber coordinate per slot
  int32_t* grp_node1 = nullptr;    // [n_groups][8] level-1 coordinate (order 4)
  int32_t* pk = nullptr;           // interleaved leaf coordinates
  int32_t* pk2 = nullptr;          // interleaved second per-leaf coordinate (optional)
  double* pv = nullptr;            // interleaved leaf values
  int32_t* slice_grp = nullptr;    // [n0+1] first group of each slice
  int32_t* slice_seg = nullptr;    // [n0+1]   segment offset of each slice
  // variable items (finish_unit_items with unit_work): item t = units
  // [item_unit[t], item_unit[t+1]), cut at equal cumulative work
  int32_t* item_unit = nullptr;    // [n_items+1] or nullptr (fixed `chunk` items)
  // CTA-range kernels (k_mttkrp3_smf): slice-aligned group range per CTA
  int64_t n_cta = 0;
  int32_t* cta_grp = nullptr;      // [n_cta+1]
  int2* hdr2 = nullptr;            // [n_groups+2] k_mttkrp3_smf headers
};

// ---- device memory (mem.cu): caching allocator over cudaMalloc blocks ---
void dmalloc_raw(void** p, size_t bytes, cudaStream_t s);
template <class T>
inline void dmalloc(T** p, size_t bytes, cudaStream_t s) {
  dmalloc_raw(reinterpret_cast<void**>(p), bytes, s);
}
// Frees in stream order on `s`. Owners (plan / CSF destroy) synchronise first
// and free with the default kStreamIdle: the block has no pending work and may
// be reused on any stream without an ordering event.
inline const cudaStream_t kStreamIdle = reinterpret_cast<cudaStream_t>(static_cast<intptr_t>(-16));
void dfree(void* p, cudaStream_t s = kStreamIdle);
void release_cached();
// Page-locked host staging blocks (size classes over cudaHostAlloc slabs), so
// a small plan's uploads / downloads are single DMA copies without a
// pageable bounce; blocks are recycled, never returned to the driver.
void* pinned_alloc(size_t bytes);
void pinned_free(void* p, size_t bytes);

// ---- kernel launchers (nest_*.cu) --------------------------------------
struct RootOutArgs {
  CsfView t;
  const double* f[4];   // factors by CSF level 1..order-1 (f[0] unused) or by role
  int R, S, T;
  int vec;              // vector loads allowed
  const int32_t* item_pos;
  int64_t n_items;
  int64_t chunk;
  double* out;
  double* part;
  int flags;
  // DMMA kernels
  const int32_t* seg_begin;
  const int32_t* seg_node;
  const int32_t* slice_seg;
  int64_t n_seg;
  // packed groups
  const int4* grp_hdr;
  const int32_t* grp_node;
  const int32_t* grp_node1;
  const int32_t* pk;
  const int32_t* pk2;
  const double* pv;
  const int32_t* slice_grp;
  int64_t n_groups;
  const int32_t* item_unit;  // variable item boundaries (TTMc-3 default kernel) or nullptr
  long long* clk;            // per item {start ns, end ns, smid} (diagnostics) or nullptr
  int64_t frows[4];          // rows of f[l] (= CSF mode sizes; bounds-checked build)
};

void launch_mttkrp3(const RootOutArgs& a, cudaStream_t s);
void launch_mttkrp4(const RootOutArgs& a, cudaStream_t s);
// TTTP-3 slice pieces (nest_tttp.cu): {i, leaf lo, leaf hi} per piece of <= P
// leaves of one root slice; A[i] gathered once per piece.
int64_t build_tttp_pieces(const DevCsf& D, int P, int4** pieces, cudaStream_t s);
void pack_leaf_jk(const DevCsf& D, const int32_t* leaf_j, int2** jk, cudaStream_t s);
void launch_tttp3_pieces(const RootOutArgs& a, const int4* pieces, int64_t n_pieces,
                         const int2* leaf_jk, int batch, cudaStream_t s);
void launch_ttmc3(const RootOutArgs& a, cudaStream_t s);
int ttmc3pq_warps_per_sm();
int ttmc4pa_warps_per_sm();
void launch_ttmc4(const RootOutArgs& a, cudaStream_t s);
// Segment-form MTTKRP (R <= 32) on packed groups: pk = order 3 (fallback of
// the shared-memory kernel), pq = TMA-staged streams (order 4 default).
void launch_mttkrp_pk(const RootOutArgs& a, cudaStream_t s);
void launch_mttkrp_pq(const RootOutArgs& a, int order, cudaStream_t s);
// MTTKRP-3 with the leaf factor's column halves resident in shared memory
// (nest_mttkrp_smf.cu): one CTA range of packed 8-slot groups per
// slice-aligned `cta_grp` entry and column half, no fix-up pass.
struct SmfArgs {
  int nq;                   // column halves (R / 16)
  int n_cta;                // CTAs per half
  int32_t rows_c;           // gathered-factor rows held in shared memory
  int32_t rows_out;         // non-root kernel: output rows accumulated in shared memory
  const int32_t* cta_grp;   // [n_cta + 1] slice-aligned group ranges
  const int2* hdr2;         // [n_groups + 2] {leaf base, slice * 8 + length}
  const int32_t* absent_rows;
  int64_t n_absent;
};
size_t mttkrp3_smf_smem(int64_t rows_c);
// plan time: hdr2 + in-place pre-scaling of grp_node / pk (plan-owned)
void mttkrp3_smf_prepare(Decomp& d, int R, cudaStream_t s);
void launch_mttkrp3_smf(const RootOutArgs& a, const SmfArgs& x, cudaStream_t s);
// non-root MTTKRP-3 (mode 1 = j, 2 = k) with column quarters of the gathered
// factor and of the output accumulator in shared memory
size_t mttkrp3_nr_smem(int64_t rows_in, int64_t rows_out);
void mttkrp3_nr_prepare(Decomp& d, int mode, int64_t rows_in, cudaStream_t s);
void launch_mttkrp3_nr_smf(const RootOutArgs& a, const SmfArgs& x, int mode, cudaStream_t s);
// MTTKRP-3 with the output on CSF level 1 (mode 1) or 2 (mode 2): atomics.
void launch_mttkrp3_nonroot(const RootOutArgs& a, int mode, cudaStream_t s);
// Per-leaf root / level-1 coordinates of an order-3 CSF (TTTP pieces).
void build_leaf_coords(const DevCsf& csf, int32_t** leaf_i, int32_t** leaf_j, cudaStream_t s);

// group geometry used by the leaf-range kernels: lanes per group for a
// padded row width (4 doubles per lane).
int group_lanes_for(int R);

// ---- device CSF construction (csf_build.cu) -------------------------------
// COO rows (nnz x d, row-major, CSF level order) -> normalize + build_csf
// semantics straight into the int32 device layout.
void csf_from_coo(DevCsf& D, int d, const int64_t* dims, int64_t nnz, const int64_t* h_coords,
                  const double* h_vals, cudaStream_t s);
// The same tensor with its levels reordered (new level l = source level
// order[l]), built on the device from the source layout.
void csf_permute(const DevCsf& src, const int* order, DevCsf& dst, cudaStream_t s);
// int32 device layout -> the reference's int64 idx / ptr arrays + values (host).
void csf_download(const DevCsf& D, int64_t* const* idx, int64_t* const* ptr, double* values,
                  cudaStream_t s);

// ---- plan-time helpers (decomp.cu) ----------------------------------------
void build_leaf_items(const DevCsf& csf, int64_t chunk, Decomp& d, int64_t tile, cudaStream_t s);
// leaf_space: segments are cut in the unit's LEAF range (seg_begin in leaf
// offsets) instead of its direct children.
void build_segments(const DevCsf& csf, int unit_level, int seg_len, int64_t chunk, Decomp& d,
                    int64_t tile, cudaStream_t s, bool make_items = true,
                    bool leaf_space = false);
// Coordinate of each node's ancestor one level up, broadcast to the node's
// children (level `l` -> level `l+1`), into `out` (nlev[l+1] entries).
void expand_coords(const DevCsf& csf, int level, const int32_t* coords, int32_t* out,
                   cudaStream_t s);
// Items of `chunk` consecutive units (segments or packed groups) given the
// first unit of every root slice; partial tiles, split slices, absent rows.
// group_overhead > 0 (packed groups only): items cut at equal cumulative
// work (leaf steps + group_overhead per group) instead of equal group
// counts; the kernel must then read its range from d.item_unit.
void finish_unit_items(const DevCsf& csf, Decomp& d, const int32_t* slice_units, int64_t n_units,
                       int64_t chunk, int64_t tile, cudaStream_t s, int group_overhead = 0);
// Length-sorted packed groups of 8 segments (pack.cu); leaf_level = CSF level
// of the streamed coordinates.
constexpr int kPackSlots = 8;  // TTMc-3 groups (128-byte rows)
// leaf_coord2 (optional, per leaf) is packed alongside as pk2 (TTMc-4: the
// leaf's level-2 coordinate).
// fill_done != nullptr: the leaf streams (pk / pk2 / pv) and the group leaf
// bases (grp_hdr .x) are filled on a side stream that waits for the CSF
// values, so the plan's item / fix-up work on `s` overlaps an asynchronous
// values upload; *fill_done is recorded when they are complete (the caller
// makes its stream wait on it and destroys it). Group lengths / slices
// (.y / .w), slot coordinates and slice_grp are ready on `s` either way.
// pair_perm: slot s stored at position 2(s % (slots/2)) + s / (slots/2) of
// its group's slot-coordinate and leaf rows (slots a and a + slots/2 adjacent).
void build_packed(const DevCsf& csf, int leaf_level, Decomp& d, cudaStream_t s,
                  int slots = kPackSlots, const int32_t* leaf_coord2 = nullptr,
                  cudaEvent_t* fill_done = nullptr, bool pair_perm = false);
// side stream per device (plan-time work overlapping the values upload)
cudaStream_t aux_stream();
constexpr int kFixChunk = 8;  // items per pass-1 chunk (one batch of loads)
void build_fixup_chunks(Decomp& d, const int32_t* idx0, cudaStream_t s);
void launch_fixup(const Decomp& d, const CsfView& t, double* out, cudaStream_t s);
void free_decomp(Decomp& d);
// Plan-build tracing (env SPTTN_PLAN_TRACE=1): synchronises `s` and prints the
// milliseconds since the previous mark to stderr. Development aid only.
void plan_trace(const char* what, cudaStream_t s);

// ---- generic interpreter (generic.cu) -------------------------------------
struct GenericState {
  spg_program* d_prog = nullptr;
  double* buffers = nullptr;       // all buffers back to back
  int64_t* buffer_off = nullptr;   // device offsets
  int64_t* counters = nullptr;     // [0] madds, [1..] resets per buffer, [..] log cursor, error
  unsigned char* log = nullptr;
  int64_t log_bytes = 0;
  int64_t* leaf_keys = nullptr;    // sorted packed coordinates (sparse-out lookup)
  int64_t* leaf_pos = nullptr;
  int64_t n_leaf_keys = 0;
  int64_t total_buffer_elems = 0;
  size_t zero_bytes = 0;  // [counters | buffers | out | private outs] cleared by one memset
  bool in_arena = false;  // all pointers live in the plan's arena
  // parallel interpreter (generic.cu k_generic_par): 0 = sequential,
  // 1 = root slices to workers with disjoint outputs, 2 = private outputs
  int par_mode = 0;
  int64_t workers = 1;
  double* priv_out = nullptr;  // mode 2: [workers][out_size]
  int64_t out_size = 0;
  void* jit_kernel = nullptr;  // specialised kernel (jit.cu), or the interpreter
  // JIT-only extensions (jit.cu): mode 3 = level-1 fibers to workers;
  // `priv` = the root loop's dense output goes through per-worker copies;
  // `tail` = buffers the root loop accumulates across slices (reset once,
  // before it) are summed over workers in worker order, then the remaining
  // roots run on one thread (phase 1)
  bool priv = false;
  bool tail = false;
  int n_tail_bufs = 0;
  int64_t tail_off[16] = {}, tail_len[16] = {};
  // small plans (generic.cu k_generic_sm): the whole working set — program,
  // CSF, dense inputs, buffers, output, counters — staged into one CTA's
  // shared memory; `sm_workers` threads (one per warp) walk root slices
  bool sm = false;
  int sm_workers = 1;
  int64_t sm_bytes = 0;
  int32_t sm_off[48] = {};  // byte offsets, see generic.cu SmSlot
  int64_t dense_size[SPG_MAX_DENSE] = {};
  const double* dense_dev[SPG_MAX_DENSE] = {};  // device factor pointers, slot 1..
  // sm plans: pinned host parcel mirroring the device arena
  // [prog | boff | factors][out | counters]; the factor block is uploaded by
  // one copy per set_factors, [out | counters] downloaded by one copy
  unsigned char* parcel = nullptr;
  size_t parcel_bytes = 0, up_prog = 0, up_fac = 0, up_end = 0, down_cnt = 0, down_end = 0;
  size_t fac_off[8] = {};
  cudaEvent_t up_done = nullptr;  // last factor upload from the parcel
};
// Shared-memory footprint / layout of a small GENERIC plan; returns false when
// it does not fit `limit` bytes (generic.cu).
bool generic_sm_layout(const spg_program& G, const DevCsf& csf, int workers, int64_t limit,
                       GenericState& g);
// Which JIT parallel decompositions a forest admits (jit.cu).
struct JitSplit {
  bool ok = false;           // root 0 is the CSF level-0 loop, accumulators are safe
  bool fiber_ok = false;     // root 0 encloses only the level-1 loop, no resets on either
  bool writes_out = false;   // root 0 writes the output
  bool disjoint_slice = false, disjoint_fiber = false;
  bool tail = false;         // more roots, or root-level accumulators
  int n_rset = 0;
  int rset[16] = {};
};
JitSplit jit_analyze(const spg_program& prog);
// phase-1 input: per-worker accumulator copies summed into worker 0's
void generic_reduce_buffers(const GenericState& g, cudaStream_t s);
void generic_execute(const spg_program& prog, const DevCsf& csf, const double* const* dense,
                     double* out, GenericState& g, cudaStream_t s);
void generic_free(GenericState& g);
// mode 2: out = sum of the per-worker output copies, in worker order
void generic_reduce(const GenericState& g, double* out, cudaStream_t s);

// ---- fused-nest JIT (jit.cu) -----------------------------------------------
bool jit_available();
// compiles (or fetches from the process cache) the specialised kernel of a
// program for g's parallel mode; returns a cudaKernel_t
void* jit_prepare(const spg_program& prog, const GenericState& g);
void jit_execute(void* kernel, const spg_program& prog, const DevCsf& csf,
                 const double* const* dense, double* out, GenericState& g, cudaStream_t s);

struct UnfactArgs;
void unfactorized_run(const void* desc, const DevCsf& csf, const double* const* dense,
                      double* out, int64_t out_count, cudaStream_t s);

// Pins a kernel's L1 / shared-memory split to what `blocks_per_sm` resident
// CTAs need (static + dynamic + the 1 KB the hardware reserves per CTA), so
// that the residency the plan's single-wave items are sized for does not rest
// on the driver's default choice: measured on TTMc-3 (3 CTAs of 61 KB per SM),
// a preferred carveout of 50-60 % fits only 2 (320 vs 212 us), 40 % one
// (413 us), 75-100 % all three. Applied once per kernel. `fixed_pct` pins a
// measured optimum instead: MTTKRP-4 runs 8 % faster with the largest
// shared-memory split although 47 % fits its 3 CTAs (620 us at 47-85 %, 569 us
// at 90-100 %), TTTP (no shared memory) 1 % faster at 0 % than at the
// driver's default (2.72 vs 2.75 ms; 3.39 ms at 100 %).
template <class K>
inline void pin_carveout(K kern, int blocks_per_sm, size_t dyn_smem, int fixed_pct = -1) {
  if (const char* cv = std::getenv("SPTTN_CARVEOUT")) {  // tuning override, every pinned kernel
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, std::atoi(cv));
    return;
  }
  static std::mutex mu;
  static std::unordered_set<const void*> done;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!done.insert(reinterpret_cast<const void*>(kern)).second) return;
  }
  int pct = fixed_pct;
  if (pct < 0) {
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, kern) != cudaSuccess) return;
    int dev = 0, max_sm = 233472;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&max_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    const size_t need = static_cast<size_t>(blocks_per_sm) * (fa.sharedSizeBytes + dyn_smem + 1024);
    pct = static_cast<int>(std::min<size_t>(100, (need * 100 + max_sm - 1) / max_sm));
  }
  cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
}

}  // namespace spttn_dev
