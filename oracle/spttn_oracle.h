/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference executor's
 * pinned fused nests (the parity oracle). Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it; the product never does.
 *
 * Each function walks the CSF tree exactly as the reference's recursive
 * interpreter does for that (path, order) — exec_node / exec_leaf / exec_hook
 * in /root/reference/proj/src/executor.cpp:389-490, with the micro-kernels of
 * proj/include/spttn/micro_kernels.hpp:11-23 — so every floating-point
 * operation happens in the same order and the results are bit-identical to
 * spttn::execute on the same plan (pinned by tests/test_oracle.py against the
 * compiled reference in oracle/_ref).
 *
 * CSF layout = the reference CsfTensor (proj/include/spttn/tensor.hpp:49-57):
 * idx[l] has level_size[l] int64 coordinates, ptr[l] (l < order-1) has
 * level_size[l]+1 int64 child offsets, values has level_size[order-1] doubles.
 * Dense tensors are row-major, last index fastest (tensor.hpp:17-30).
 */
#ifndef SPTTN_ORACLE_H
#define SPTTN_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int order;
  int64_t dims[8];
  int64_t level_size[8];
  const int64_t* idx[8];
  const int64_t* ptr[8];
  const double* values;
} oc_csf;

/* MTTKRP-3  T[i,j,k]*B[j,a]*C[k,a]->A[i,a], path ((T*C)*B), orders
 * (i,j,k,a)(i,j,a). out: I x R, overwritten. */
void oc_mttkrp3(const oc_csf* t, int64_t R, const double* B, const double* C, double* out);

/* MTTKRP-3 for the non-root modes:
 *   _j: T[i,j,k]*A[i,a]*C[k,a]->B[j,a], path ((T*C)*A), orders (i,j,a,k)(i,j,a)
 *   _k: T[i,j,k]*A[i,a]*B[j,a]->C[k,a], path ((A*B)*T), orders (i,j,a)(i,j,a,k)
 * out: J x R / K x R, overwritten. */
void oc_mttkrp3_j(const oc_csf* t, int64_t R, const double* A, const double* C, double* out);
void oc_mttkrp3_k(const oc_csf* t, int64_t R, const double* A, const double* B, double* out);

/* TTMc-3  T[i,j,k]*U[j,r]*V[k,s]->S[i,r,s], path ((T*V)*U), orders
 * (i,j,k,s)(i,j,s,r). out: I x R x S. */
void oc_ttmc3(const oc_csf* t, int64_t R, int64_t S, const double* U, const double* V,
              double* out);

/* TTTP-3  T[i,j,k]*U[i,r]*V[j,r]*W[k,r]->S[i,j,k] @sparse_out, path
 * (((U*V)*W)*T), orders (i,j,r)(i,j,k,r)(i,j,k). out: nnz values in CSF
 * leaf order. residual=0: S = Y*t (reference); residual=1: rho = t - Y. */
void oc_tttp3(const oc_csf* t, int64_t R, const double* U, const double* V, const double* W,
              double* out, int residual);

/* MTTKRP-4  T[i,j,k,l]*B[j,r]*C[k,r]*D[l,r]->A[i,r], path (((T*D)*C)*B),
 * orders (i,j,k,l,r)(i,j,k,r)(i,j,r). out: I x R. */
void oc_mttkrp4(const oc_csf* t, int64_t R, const double* B, const double* C, const double* D,
                double* out);

/* TTMc-4  T[i,j,k,l]*U[j,r]*V[k,s]*W[l,t]->S[i,r,s,t], path (((T*W)*V)*U),
 * orders (i,j,k,l,t)(i,j,k,s,t)(i,j,r,s,t). out: I x R x S x T. */
void oc_ttmc4(const oc_csf* t, int64_t R, int64_t S, int64_t T, const double* U, const double* V,
              const double* W, double* out);

/* The reference's execute_unfactorized (executor.cpp:522-626) for a kernel
 * whose dense factors are all matrices F_f[mode_f, rank_f] (mode_f = CSF level
 * index, rank index shared or private): the five families above. Free dense
 * indices are given in first-appearance order; nfree <= 4.
 *   factor_level[f]  CSF level of factor f's sparse index (or -1 for none)
 *   factor_free[f]   which free index (0..nfree-1) factor f carries
 *   out_free[q]      output's free indices in output order (-1 terminated)
 *   out_has_root     1 if the output's first index is CSF level 0
 * Dense output row-major [root?][out_free...]; sparse output per leaf. */
typedef struct {
  int nfactors;
  int nfree;
  int64_t free_dim[4];
  int factor_level[6];
  int factor_free[6];
  const double* factor[6];
  int out_sparse;
  int out_has_root;
  int out_nfree;
  int out_free[4];
} oc_unfact_desc;

void oc_unfactorized(const oc_csf* t, const oc_unfact_desc* d, double* out, int64_t* madds);

#ifdef __cplusplus
}
#endif

#endif
