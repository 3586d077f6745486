/* spttn_b200 — C-ABI of the B200-native SpTTN fused-nest execution engine.
 *
 * This is the device boundary under the reference's executor API
 * (/root/reference/proj/include/spttn/executor.hpp:80-95). The C++ shim
 * paper_2307_05740_b200/csrc/shim/executor_b200.cpp implements
 * spttn::prepare / execute / execute_unfactorized / flops_estimate /
 * flops_unfactorized with the reference's exact signatures on top of these
 * entry points; ctypes / cgo / JNI bindings can call them directly
 * (INTEGRATION.md). Plain pointers and sizes only; no C++ or torch types.
 *
 * Mapping to the reference interface it replaces:
 *   spttn_csf_create      CsfTensor handed to prepare() via ExecInputs::sparse
 *                         (executor.hpp:55-58; layout tensor.hpp:49-57)
 *   spttn_plan_create     spttn::prepare (executor.hpp:87-88, executor.cpp:172-371)
 *   spttn_execute         spttn::execute (executor.hpp:90, executor.cpp:510-520)
 *   spttn_read_output     ExecResult::dense_out / sparse_out_values (executor.hpp:60-66)
 *   spttn_unfactorized    spttn::execute_unfactorized (executor.hpp:92-94, executor.cpp:522-626)
 *   status codes          std::invalid_argument / unsupported_order_error /
 *                         resource_error (executor.hpp:18-23, executor.cpp:112-200)
 *
 * Threading: like the reference executor, one plan per host thread at a time;
 * distinct plans over one read-only spttn_csf may run concurrently on
 * different streams. All calls taking a `stream` enqueue on
 * that cudaStream_t (NULL = legacy default stream).
 */
#ifndef SPTTN_B200_H
#define SPTTN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
#define SPTTN_OK 0
#define SPTTN_EINVAL 1       /* std::invalid_argument (shapes, missing tensor) */
#define SPTTN_EUNSUPPORTED 2 /* unsupported_order_error                        */
#define SPTTN_ENOMEM 3       /* resource_error (buffer limit, device memory)   */
#define SPTTN_ECUDA 4        /* CUDA runtime / launch failure, no device       */

/* Thread-local message for the last non-OK status. */
const char* spttn_last_error(void);

/* ---- device CSF -------------------------------------------------------- */
typedef struct spttn_csf spttn_csf;

/* Host view of a CSF tree in the reference's CsfTensor layout. The arrays may
 * be a view into a larger tree — e.g. a range of root slices of a CsfTensor,
 * pointers into its arrays: ptr[l][0] need not be 0 (the device layout is
 * rebased), only ptr[l][level_size[l]] - ptr[l][0] == level_size[l+1]. */
typedef struct {
  int32_t order;              /* number of modes, 1..8                        */
  const int64_t* dims;        /* [order] mode sizes, root-to-leaf             */
  const int64_t* level_size;  /* [order] node count per level (nnz_at_level)  */
  const int64_t* const* idx;  /* [order] host arrays of level_size[l] coords  */
  const int64_t* const* ptr;  /* [order-1] host arrays of level_size[l]+1     */
  const double* values;       /* [level_size[order-1]] leaf values            */
} spttn_csf_host;

/* Copies the tree to the current device and builds the device layout
 * (SoA int32 fiber pointers / coordinates, 256-B aligned fp64 values).
 * Fails with SPTTN_EINVAL on malformed trees or coordinates beyond int32.
 * The device CSF is a SNAPSHOT of the host arrays: plans built on it (which
 * may also copy leaf values into packed streams) do not see later changes
 * to the host tensor — create a new CSF and plan for changed values (the C++
 * drop-in does this automatically at execute). */
int spttn_csf_create(const spttn_csf_host* host, void* stream, spttn_csf** out);
/* As spttn_csf_create, but the leaf values are uploaded on a side stream
 * while the call returns after the (validated) structure: plan creation,
 * whose decomposition needs only idx / ptr, overlaps the values' transfer
 * (every consumer of the values waits for it on its own stream). The caller
 * must keep host->values unchanged and allocated until the first plan
 * created on the CSF has finished spttn_plan_create (or any execute /
 * download on it has completed); with page-locked host->values the transfer
 * is a true background DMA. */
int spttn_csf_create_async(const spttn_csf_host* host, void* stream, spttn_csf** out);
int spttn_csf_destroy(spttn_csf* csf);
/* Builds the device CSF from COO on the GPU (replaces CooTensor::normalize +
 * build_csf, proj/src/tensor.cpp:24-94): coords are nnz x order int64,
 * row-major, already in CSF mode order; rows are sorted, duplicates summed in
 * input order. SPTTN_EINVAL for out-of-range coordinates. */
int spttn_csf_from_coo(int order, const int64_t* dims, int64_t nnz, const int64_t* coords,
                       const double* values, void* stream, spttn_csf** out);
/* Copies a device CSF back as the reference's CsfTensor arrays: idx[l]
 * (level_size[l] int64), ptr[l] (level_size[l]+1 int64), values. Any array
 * pointer may be NULL to skip it. */
int spttn_csf_download(const spttn_csf* csf, int64_t* const* idx, int64_t* const* ptr,
                       double* values, void* stream);
int64_t spttn_csf_dim(const spttn_csf* csf, int level);
/* The same tensor with its levels reordered on the device (new level l =
 * source level order[l]) — re-rooting a CSF so an output on a non-root mode
 * becomes root-indexed (owner computes, no atomics). */
int spttn_csf_permute(const spttn_csf* src, const int* order, void* stream, spttn_csf** out);
int64_t spttn_csf_level_size(const spttn_csf* csf, int level);
int64_t spttn_csf_device_bytes(const spttn_csf* csf);

/* ---- plans --------------------------------------------------------------- */
typedef struct spttn_plan spttn_plan;

/* Fused nest shapes with a dedicated sm_100a kernel (SURVEY.md §8a pinned
 * nests); GENERIC runs any admissible forest through the device forest
 * interpreter (program built by the shim, see spttn_program_*). */
enum {
  SPTTN_NEST_MTTKRP3 = 1, /* T[i,j,k]*B[j,r]*C[k,r]->A[i,r]  ((T*C)*B)        */
  SPTTN_NEST_TTMC3 = 2,   /* T[i,j,k]*U[j,r]*V[k,s]->Y[i,r,s] ((T*V)*U)       */
  SPTTN_NEST_TTTP3 = 3,   /* T*A[i,r]*B[j,r]*C[k,r]->S[i,j,k] (((A*B)*C)*T)   */
  SPTTN_NEST_MTTKRP4 = 4, /* T[i,j,k,l]*B*C*D->A[i,r]  (((T*D)*C)*B)          */
  SPTTN_NEST_TTMC4 = 5,   /* T[i,j,k,l]*U*V*W->Y[i,r,s,t] (((T*W)*V)*U)       */
  SPTTN_NEST_MTTKRP3_J = 6, /* T[i,j,k]*A[i,r]*C[k,r]->B[j,r] ((T*C)*A), atomics */
  SPTTN_NEST_MTTKRP3_K = 7, /* T[i,j,k]*A[i,r]*B[j,r]->C[k,r] ((A*B)*T), atomics */
  SPTTN_NEST_GENERIC = 100
};

/* TTTP: emit the completion residual rho = t - sum_r A B C instead of the
 * reference's S = t * sum_r A B C. */
#define SPTTN_FLAG_RESIDUAL 1
/* Factor pointers are device pointers that outlive the plan (not copied). */
#define SPTTN_FLAG_FACTORS_ON_DEVICE 2

typedef struct {
  int32_t kind;               /* SPTTN_NEST_*                                  */
  int32_t flags;              /* SPTTN_FLAG_*                                  */
  int64_t rank[3];            /* R, S, T (unused entries 0)                    */
  int32_t num_factors;        /* dense inputs, in kernel input order           */
  const double* factors[8];   /* factor arrays (host unless FACTORS_ON_DEVICE) */
  int64_t factor_size[8];     /* element counts                                */
  int64_t buffer_limit_bytes; /* ExecOptions::buffer_limit_bytes               */
  const void* program;        /* GENERIC: serialized forest program            */
  int64_t program_bytes;
} spttn_plan_desc;

int spttn_plan_create(const spttn_plan_desc* desc, spttn_csf* csf, void* stream,
                      spttn_plan** out);
int spttn_plan_destroy(spttn_plan* plan);

/* Replaces the factor values (same shapes), e.g. between ALS sweeps. Device
 * factors (on_device) must be at least as aligned as those the plan was
 * created with (the kernel variant depends on it): SPTTN_EINVAL otherwise. */
int spttn_plan_set_factors(spttn_plan* plan, const double* const* factors, int32_t on_device,
                           void* stream);

/* Runs the fused nest; output stays in device memory. */
int spttn_execute(spttn_plan* plan, void* stream);
/* One stage of spttn_execute, for per-kernel timing: stage 0 = the fused
 * nest kernel, stage 1 = the epilogue (split-slice fix-up, absent-row
 * zeroing); spttn_execute == stage 0 then stage 1. */
int spttn_execute_stage(spttn_plan* plan, int stage, void* stream);

int64_t spttn_output_count(const spttn_plan* plan);
const double* spttn_output_device(const spttn_plan* plan);
/* Copies the output to host memory (count must equal spttn_output_count) and
 * synchronises the stream. */
int spttn_read_output(spttn_plan* plan, double* host_out, int64_t count, void* stream);

/* Per-plan facts: [0] kernel launches per execute, [1] work items,
 * [2] split root slices, [3] absent root rows, [4] device scratch bytes,
 * [5] nest kind actually run, [6] segments (DMMA kernels),
 * [7] multiply-adds counted by the device interpreter on the last execute
 *     (GENERIC only; fast kernels report -1: use flops_estimate),
 * [8] GENERIC decomposition: 0 sequential walk, 1 root slices written
 *     directly, 2 root ranges into per-worker outputs summed in worker
 *     order, 3 level-1 fibers (JIT only); -1 for the fused kernels,
 * [9] GENERIC: 1 when the forest runs as an NVRTC-compiled kernel,
 * [10] kernel variant of the fused nests (the SPTTN_*_MODE value chosen,
 *     e.g. 5 = non-root MTTKRP-3 on the output-mode-major re-ordered
 *     tensor); -1 for GENERIC.                                           */
int spttn_plan_info(const spttn_plan* plan, int64_t* out, int n);

/* Diagnostics (kernel tuning): with SPTTN_ITEM_CLOCKS=1 set at plan
 * creation, the packed TTMc-3 kernel (its diagnostics instantiation)
 * records per work item {start ns, end ns, SM id, groups, leaf steps, tile
 * flushes} (%globaltimer, %smid) on every execute; this copies the last
 * execute's records (6 * items int64) to host memory. EINVAL when the plan
 * records none.                                                           */
int spttn_plan_item_clocks(const spttn_plan* plan, int64_t* host_out, int64_t n);

/* GENERIC only: per-buffer reset counts of the last execute (as counted on
 * the device, ExecStats::buffer_resets) and the observer log (buffer id +
 * buffer contents after each reset, in execution order) when the program
 * requested one. */
int spttn_generic_resets(const spttn_plan* plan, int64_t* out, int n);
int64_t spttn_generic_log_bytes(const spttn_plan* plan);
int spttn_generic_read_log(spttn_plan* plan, void* host_out, int64_t bytes, void* stream);

/* ---- unfactorized oracle on the device --------------------------------- */
/* execute_unfactorized for a kernel whose dense inputs are described by
 * index-role lists: see spttn_unfact_desc. Deterministic: every output entry
 * accumulates its contributions in the reference's order. */
typedef struct {
  int32_t num_indices;        /* kernel index count                            */
  int64_t dims[32];           /* per index id                                  */
  int32_t csf_level[32];      /* CSF level of a sparse index, -1 if dense      */
  int32_t num_free;           /* free dense indices, first-appearance order     */
  int32_t free_ids[32];
  int32_t num_factors;
  int32_t factor_order[8];    /* index count per dense factor                  */
  int32_t factor_ids[8][8];   /* index ids per dense factor (row-major order)  */
  const double* factors[8];   /* host arrays                                   */
  int32_t out_sparse;
  int32_t out_order;
  int32_t out_ids[8];
} spttn_unfact_desc;

int spttn_unfactorized(const spttn_unfact_desc* desc, spttn_csf* csf, double* host_out,
                       int64_t out_count, void* stream);

/* ---- device facts ------------------------------------------------------ */
/* [0] SM count, [1] compute capability major*10+minor, [2] L2 bytes,
 * [3] max shared memory per block (opt-in). */
int spttn_device_info(int64_t* out, int n);
/* Creates the CUDA context up front (the C++
 * drop-in calls it when it is loaded, so the first prepare() does not pay for
 * context creation; SPTTN_LAZY_INIT=1 skips that). SPTTN_ECUDA without a
 * device. */
int spttn_init(void);
/* Waits for all work on `stream` (NULL = the whole device); used by the
 * drop-in's phase tracing (SPTTN_SHIM_TRACE=2). */
int spttn_synchronize(void* stream);
/* Build identification string (arch, nvcc version). */
const char* spttn_build_info(void);
/* Device memory of CSF layouts and plans comes from a per-device caching
 * allocator (whole cudaMalloc blocks kept on a free list and reused in stream
 * order), so rebuilding plans is cheap. Synchronises the device and returns
 * the cached (unused) blocks to the driver.
 * Stream lifetime: the temporaries of spttn_csf_create* / spttn_plan_create
 * are freed in the order of the stream passed to them; such a block later
 * reused on another stream makes that stream wait on an event recorded on
 * the first one at reuse time. A stream given to those calls must therefore
 * outlive the engine's use, or be followed by spttn_release_cached() before
 * it is destroyed (an event record that fails on a dead stream falls back
 * to a device synchronisation). Destroy calls synchronise the device first,
 * so the blocks they release carry no stream ordering. */
int spttn_release_cached(void);

#ifdef __cplusplus
}
#endif

#endif /* SPTTN_B200_H */
