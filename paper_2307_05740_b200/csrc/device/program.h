/* Serialized fused-loop-forest program for the GENERIC device interpreter.
 *
 * Produced on the host by the shim's plan compiler from the reference
 * FusedLoopForest (proj/include/spttn/loop_nest.hpp:24-55) with the same
 * operand addressing, reset placement and hook classification as the
 * reference prepare() (proj/src/executor.cpp:191-366); consumed by
 * generic.cu, which walks it like exec_node / exec_leaf / exec_hook
 * (executor.cpp:389-490). Plain-old-data, fixed capacity, memcpy-able.
 */
#ifndef SPTTN_PROGRAM_H
#define SPTTN_PROGRAM_H

#include <stdint.h>

#define SPG_MAGIC 0x53505447454e3031LL /* "SPTGEN01" */
#define SPG_MAX_IDX 32
#define SPG_MAX_LEVELS 8
#define SPG_MAX_NODES 256
#define SPG_MAX_TERMS 16
#define SPG_MAX_BUFFERS 16
#define SPG_MAX_CHILDREN 512
#define SPG_MAX_RESETS 64
#define SPG_MAX_DENSE 16
#define SPG_MAX_ADDR 12

enum { SPG_LEAF = 0, SPG_SPARSE = 1, SPG_DENSE = 2 };
enum { SPG_OP_SPARSE = 0, SPG_OP_DENSE = 1, SPG_OP_BUFFER = 2, SPG_OP_OUT_DENSE = 3, SPG_OP_OUT_SPARSE = 4 };
enum { SPG_HOOK_NONE = 0, SPG_HOOK_VEC = 1, SPG_HOOK_RANK1 = 2 };

typedef struct {
  int32_t kind;      /* SPG_OP_*                                    */
  int32_t slot;      /* dense input number (1..n-1) or buffer id    */
  int32_t naddr;
  int32_t ids[SPG_MAX_ADDR];
  int64_t strides[SPG_MAX_ADDR];
} spg_access;

typedef struct {
  int32_t kind;      /* SPG_LEAF / SPG_SPARSE / SPG_DENSE           */
  int32_t index;     /* loop index id                               */
  int32_t csf_level; /* sparse vertices                             */
  int32_t term;      /* leaves                                      */
  int32_t child_begin, child_count;
  int32_t reset_begin, reset_count;
  int32_t hook;      /* index into hooks or -1                      */
} spg_node;

typedef struct {
  int32_t kind;      /* SPG_HOOK_*                                  */
  int32_t term;
  int32_t nspan;
  int32_t span[SPG_MAX_ADDR];
  int64_t len, out_inc, vec_inc;
  int32_t vec_is_lhs, x_is_lhs;
  int64_t m, n, x_inc, y_inc, out_row, out_col;
} spg_hook;

typedef struct {
  int64_t magic;
  int32_t num_indices;
  int64_t dims[SPG_MAX_IDX];
  int32_t csf_order;                   /* sparse tensor order           */
  int32_t num_nodes, num_roots, num_terms, num_buffers, num_hooks, num_dense;
  int32_t roots[SPG_MAX_NODES];
  int32_t children[SPG_MAX_CHILDREN];
  int32_t resets[SPG_MAX_RESETS];
  spg_node nodes[SPG_MAX_NODES];
  spg_access lhs[SPG_MAX_TERMS], rhs[SPG_MAX_TERMS], out[SPG_MAX_TERMS];
  spg_hook hooks[SPG_MAX_TERMS];
  int64_t buffer_size[SPG_MAX_BUFFERS];
  int64_t dense_size[SPG_MAX_DENSE];   /* element count per dense input 1..n-1 (index 0 unused) */
  int32_t out_sparse;
  int64_t out_size;
  int32_t need_leaf_lookup;            /* executor.cpp:342-366          */
  int32_t sparse_mode_ids[SPG_MAX_LEVELS];
  int64_t mode_key_stride[SPG_MAX_LEVELS];
  int32_t observe;                     /* log buffer snapshots on reset */
  int64_t observe_log_bytes;           /* capacity for the log          */
  int64_t reserved;                    /* keeps sizeof a multiple of 16 */
} spg_program;

#endif
