/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference executor's
 * pinned fused nests; see spttn_oracle.h for the contract and citations. */
#include "spttn_oracle.h"

#include <stdlib.h>
#include <string.h>

/* Children of node p at level l: [ptr[l][p], ptr[l][p+1]) (tensor.hpp:49-57,
 * walked like exec_node's sparse vertex, executor.cpp:470-483). */
#define KIDS(t, l, p) (t)->ptr[l][p], (t)->ptr[l][(p) + 1]

static int64_t dense_out_size(int64_t a, int64_t b, int64_t c, int64_t d) {
  return a * b * c * d;
}

void oc_mttkrp3(const oc_csf* t, int64_t R, const double* B, const double* C, double* out) {
  const int64_t I = t->dims[0];
  memset(out, 0, sizeof(double) * dense_out_size(I, R, 1, 1));
  double* X = (double*)calloc((size_t)R, sizeof(double));
  for (int64_t p0 = 0; p0 < t->level_size[0]; ++p0) {
    const int64_t i = t->idx[0][p0];
    for (int64_t p1 = t->ptr[0][p0]; p1 < t->ptr[0][p0 + 1]; ++p1) {
      const int64_t j = t->idx[1][p1];
      /* X reset on entry of the k vertex (executor.cpp:226-242, :455-461) */
      memset(X, 0, sizeof(double) * R);
      for (int64_t p2 = t->ptr[1][p1]; p2 < t->ptr[1][p1 + 1]; ++p2) {
        const int64_t k = t->idx[2][p2];
        const double alpha = t->values[p2];
        /* vector-accumulate hook: y += alpha * x (micro_kernels.hpp:11-14) */
        for (int64_t a = 0; a < R; ++a) X[a] += alpha * C[k * R + a];
      }
      /* term 2 leaf: out += read(lhs) * read(rhs) (executor.cpp:389-409) */
      for (int64_t a = 0; a < R; ++a) out[i * R + a] += X[a] * B[j * R + a];
    }
  }
  free(X);
}

/* MTTKRP-3 for mode j: T[i,j,k]*A[i,a]*C[k,a]->B[j,a], path ((T*C)*A),
 * orders (i,j,a,k)(i,j,a) (max-buf-dim's pick): per (i,j) X[a] = sum_k t*C[k,a]
 * in CSF order (the dense a loop outside k keeps each X[a] a sum over k in
 * leaf order), then B[j,a] += X[a]*A[i,a] in (i,j) CSF order. */
void oc_mttkrp3_j(const oc_csf* t, int64_t R, const double* A, const double* C, double* out) {
  const int64_t J = t->dims[1];
  memset(out, 0, sizeof(double) * dense_out_size(J, R, 1, 1));
  double* X = (double*)calloc((size_t)R, sizeof(double));
  for (int64_t p0 = 0; p0 < t->level_size[0]; ++p0) {
    const int64_t i = t->idx[0][p0];
    for (int64_t p1 = t->ptr[0][p0]; p1 < t->ptr[0][p0 + 1]; ++p1) {
      const int64_t j = t->idx[1][p1];
      memset(X, 0, sizeof(double) * R);
      for (int64_t a = 0; a < R; ++a)
        for (int64_t p2 = t->ptr[1][p1]; p2 < t->ptr[1][p1 + 1]; ++p2)
          X[a] += t->values[p2] * C[t->idx[2][p2] * R + a];
      for (int64_t a = 0; a < R; ++a) out[j * R + a] += X[a] * A[i * R + a];
    }
  }
  free(X);
}

/* MTTKRP-3 for mode k: T[i,j,k]*A[i,a]*B[j,a]->C[k,a], path ((A*B)*T),
 * orders (i,j,a)(i,j,a,k): per (i,j) W[a] = A[i,a]*B[j,a], per leaf
 * C[k,a] += W[a]*t, contributions to each C[k,a] in (i,j) CSF order. */
void oc_mttkrp3_k(const oc_csf* t, int64_t R, const double* A, const double* B, double* out) {
  const int64_t K = t->dims[2];
  memset(out, 0, sizeof(double) * dense_out_size(K, R, 1, 1));
  double* W = (double*)calloc((size_t)R, sizeof(double));
  for (int64_t p0 = 0; p0 < t->level_size[0]; ++p0) {
    const int64_t i = t->idx[0][p0];
    for (int64_t p1 = t->ptr[0][p0]; p1 < t->ptr[0][p0 + 1]; ++p1) {
      const int64_t j = t->idx[1][p1];
      for (int64_t a = 0; a < R; ++a) W[a] = A[i * R + a] * B[j * R + a];
      for (int64_t a = 0; a < R; ++a)
        for (int64_t p2 = t->ptr[1][p1]; p2 < t->ptr[1][p1 + 1]; ++p2)
          out[t->idx[2][p2] * R + a] += W[a] * t->values[p2];
    }
  }
  free(W);
}

void oc_ttmc3(const oc_csf* t, int64_t R, int64_t S, const double* U, const double* V,
              double* out) {
  const int64_t I = t->dims[0];
  memset(out, 0, sizeof(double) * dense_out_size(I, R, S, 1));
  double* X = (double*)calloc((size_t)S, sizeof(double));
  for (int64_t p0 = 0; p0 < t->level_size[0]; ++p0) {
    const int64_t i = t->idx[0][p0];
    for (int64_t p1 = t->ptr[0][p0]; p1 < t->ptr[0][p0 + 1]; ++p1) {
      const int64_t j = t->idx[1][p1];
      memset(X, 0, sizeof(double) * S);
      for (int64_t p2 = t->ptr[1][p1]; p2 < t->ptr[1][p1 + 1]; ++p2) {
        const int64_t k = t->idx[2][p2];
        const double alpha = t->values[p2];
        for (int64_t s = 0; s < S; ++s) X[s] += alpha * V[k * S + s];
      }
      /* rank-1 hook over (s, r): A[s*row + r*col] += x_s * y_r
       * (micro_kernels.hpp:17-23), row = 1, col = S in S[i,r,s]. */
      double* o = out + i * R * S;
      for (int64_t s = 0; s < S; ++s) {
        const double xs = X[s];
        for (int64_t r = 0; r < R; ++r) o[s + r * S] += xs * U[j * R + r];
      }
    }
  }
  free(X);
}

void oc_tttp3(const oc_csf* t, int64_t R, const double* U, const double* V, const double* W,
              double* out, int residual) {
  double* X = (double*)calloc((size_t)R, sizeof(double));
  for (int64_t p0 = 0; p0 < t->level_size[0]; ++p0) {
    const int64_t i = t->idx[0][p0];
    for (int64_t p1 = t->ptr[0][p0]; p1 < t->ptr[0][p0 + 1]; ++p1) {
      const int64_t j = t->idx[1][p1];
      /* term 1 (i,j,r): X[r] = U[i,r]*V[j,r], reset on the r vertex entry */
      memset(X, 0, sizeof(double) * R);
      for (int64_t r = 0; r < R; ++r) X[r] += U[i * R + r] * V[j * R + r];
      for (int64_t p2 = t->ptr[1][p1]; p2 < t->ptr[1][p1 + 1]; ++p2) {
        const int64_t k = t->idx[2][p2];
        /* term 2 (i,j,k,r): scalar Y, reset per (i,j,k) */
        double Y = 0.0;
        for (int64_t r = 0; r < R; ++r) Y += X[r] * W[k * R + r];
        /* term 3 leaf at the leaf's own position (executor.cpp:402) */
        const double tv = t->values[p2];
        out[p2] = residual ? tv - Y : 0.0 + Y * tv;
      }
    }
  }
  free(X);
}

void oc_mttkrp4(const oc_csf* t, int64_t R, const double* B, const double* C, const double* D,
                double* out) {
  const int64_t I = t->dims[0];
  memset(out, 0, sizeof(double) * dense_out_size(I, R, 1, 1));
  double* X = (double*)calloc((size_t)R, sizeof(double));
  double* Y = (double*)calloc((size_t)R, sizeof(double));
  for (int64_t p0 = 0; p0 < t->level_size[0]; ++p0) {
    const int64_t i = t->idx[0][p0];
    for (int64_t p1 = t->ptr[0][p0]; p1 < t->ptr[0][p0 + 1]; ++p1) {
      const int64_t j = t->idx[1][p1];
      memset(Y, 0, sizeof(double) * R); /* Y reset on the k vertex entry */
      for (int64_t p2 = t->ptr[1][p1]; p2 < t->ptr[1][p1 + 1]; ++p2) {
        const int64_t k = t->idx[2][p2];
        memset(X, 0, sizeof(double) * R); /* X reset on the l vertex entry */
        for (int64_t p3 = t->ptr[2][p2]; p3 < t->ptr[2][p2 + 1]; ++p3) {
          const int64_t l = t->idx[3][p3];
          const double alpha = t->values[p3];
          for (int64_t a = 0; a < R; ++a) X[a] += alpha * D[l * R + a];
        }
        for (int64_t a = 0; a < R; ++a) Y[a] += X[a] * C[k * R + a];
      }
      for (int64_t a = 0; a < R; ++a) out[i * R + a] += Y[a] * B[j * R + a];
    }
  }
  free(X);
  free(Y);
}

void oc_ttmc4(const oc_csf* t, int64_t R, int64_t S, int64_t T, const double* U, const double* V,
              const double* W, double* out) {
  const int64_t I = t->dims[0];
  const int64_t ST = S * T;
  memset(out, 0, sizeof(double) * dense_out_size(I, R, S, T));
  double* X = (double*)calloc((size_t)T, sizeof(double));
  double* Y = (double*)calloc((size_t)ST, sizeof(double));
  for (int64_t p0 = 0; p0 < t->level_size[0]; ++p0) {
    const int64_t i = t->idx[0][p0];
    for (int64_t p1 = t->ptr[0][p0]; p1 < t->ptr[0][p0 + 1]; ++p1) {
      const int64_t j = t->idx[1][p1];
      memset(Y, 0, sizeof(double) * ST); /* Y(s,t) reset on the k vertex entry */
      for (int64_t p2 = t->ptr[1][p1]; p2 < t->ptr[1][p1 + 1]; ++p2) {
        const int64_t k = t->idx[2][p2];
        memset(X, 0, sizeof(double) * T); /* X(t) reset on the l vertex entry */
        for (int64_t p3 = t->ptr[2][p2]; p3 < t->ptr[2][p2 + 1]; ++p3) {
          const int64_t l = t->idx[3][p3];
          const double alpha = t->values[p3];
          for (int64_t c = 0; c < T; ++c) X[c] += alpha * W[l * T + c];
        }
        /* rank-1 hook over (s,t): x = V[k,:] (rhs), y = X (lhs) */
        for (int64_t s = 0; s < S; ++s) {
          const double xs = V[k * S + s];
          for (int64_t c = 0; c < T; ++c) Y[s * T + c] += xs * X[c];
        }
      }
      /* meta loop r around a flattened vector-accumulate over (s,t):
       * y += alpha * x with alpha = U[j,r], x = Y (executor.cpp:415-432) */
      double* o = out + i * R * ST;
      for (int64_t r = 0; r < R; ++r) {
        const double alpha = U[j * R + r];
        for (int64_t q = 0; q < ST; ++q) o[r * ST + q] += alpha * Y[q];
      }
    }
  }
  free(X);
  free(Y);
}

/* execute_unfactorized (executor.cpp:522-626): CSF levels outermost, free
 * dense indices inside (first-appearance order), every factor multiplied in
 * the body in kernel order. */
void oc_unfactorized(const oc_csf* t, const oc_unfact_desc* d, double* out, int64_t* madds) {
  const int order = t->order;
  const int64_t nnz = t->level_size[order - 1];
  int64_t free_total = 1;
  for (int q = 0; q < d->nfree; ++q) free_total *= d->free_dim[q];
  int64_t out_size = 0;
  if (d->out_sparse) {
    out_size = nnz;
  } else {
    out_size = d->out_has_root ? t->dims[0] : 1;
    for (int q = 0; q < d->out_nfree; ++q) out_size *= d->free_dim[d->out_free[q]];
  }
  memset(out, 0, sizeof(double) * (size_t)out_size);
  int64_t count = 0;
  int64_t pos[8] = {0};
  int64_t coord[8] = {0};
  int64_t digit[4] = {0};
  /* iterative depth-first walk over the CSF levels */
  int64_t hi[8];
  int lvl = 0;
  pos[0] = 0;
  hi[0] = t->level_size[0];
  if (hi[0] == 0) {
    if (madds) *madds = 0;
    return;
  }
  for (;;) {
    if (pos[lvl] >= hi[lvl]) {
      if (lvl == 0) break;
      --lvl;
      ++pos[lvl];
      continue;
    }
    coord[lvl] = t->idx[lvl][pos[lvl]];
    if (lvl + 1 < order) {
      pos[lvl + 1] = t->ptr[lvl][pos[lvl]];
      hi[lvl + 1] = t->ptr[lvl][pos[lvl] + 1];
      ++lvl;
      continue;
    }
    /* leaf: dense loop over the free indices, first one outermost */
    const int64_t p = pos[lvl];
    for (int64_t f = 0; f < free_total; ++f) {
      int64_t rest = f;
      for (int q = d->nfree - 1; q >= 0; --q) {
        digit[q] = rest % d->free_dim[q];
        rest /= d->free_dim[q];
      }
      double v = t->values[p];
      for (int k = 0; k < d->nfactors; ++k) {
        int64_t off = 0;
        if (d->factor_level[k] >= 0) off = coord[d->factor_level[k]];
        if (d->factor_free[k] >= 0) off = off * d->free_dim[d->factor_free[k]] + digit[d->factor_free[k]];
        v *= d->factor[k][off];
      }
      count += d->nfactors + 1;
      if (d->out_sparse) {
        out[p] += v;
      } else {
        int64_t off = d->out_has_root ? coord[0] : 0;
        for (int q = 0; q < d->out_nfree; ++q)
          off = off * d->free_dim[d->out_free[q]] + digit[d->out_free[q]];
        out[off] += v;
      }
    }
    ++pos[lvl];
  }
  if (madds) *madds = count;
}
