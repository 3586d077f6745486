"""Multi-GPU sharding of the fused nests.

The root slices of a CSF tensor are independent work units for every pinned
nest: MTTKRP / TTMc write disjoint output rows A[i,:] / Y[i,:,:] (owner
computes), and TTTP writes each leaf's own value. A job over N GPUs therefore
needs no data-path collective:

  * `partition_roots` cuts the root level into N contiguous ranges balanced by
    nnz (prefix sums over the child pointers);
  * `shard_csf` extracts one range as a standalone CSF (same mode sizes, so
    row-indexed outputs keep global row numbers);
  * factors are replicated (`broadcast_factors`, one NCCL broadcast each —
    the only exchange, and only when ranks do not generate them locally);
  * `gather_dense_rows` / `gather_sparse_leaves` assemble the full output on
    every rank when a caller needs it (all_gather of the owned rows / leaf
    ranges), replacing the paper's CTF reduction + redistribution
    (PAPER.md:1106-1115).

Outputs NOT indexed by the root mode (MTTKRP for modes j / k,
SPTTN_NEST_MTTKRP3_J / _K) are the one place the path has a real exchange:
every shard adds into every output row, so the full output is the sum of the
ranks' outputs (`reduce_dense_output`, one all_reduce — NCCL over NVLink on a
GPU job).

bench.py runs N independent full-size tensors (weak scaling, one per rank);
`--shard` runs one tensor split with these helpers (strong scaling).
"""
from __future__ import annotations

import numpy as np

from .tensor import Csf


def leaf_range_of_roots(csf: Csf, r0: int, r1: int) -> tuple[int, int]:
    a, b = r0, r1
    for l in range(csf.order - 1):
        a, b = int(csf.ptr[l][a]), int(csf.ptr[l][b])
    return a, b


def partition_roots(csf: Csf, world: int) -> list[tuple[int, int]]:
    """Contiguous root-node ranges [r0, r1) with ~nnz/world leaves each."""
    n0 = csf.level_sizes()[0]
    # leaf offset of every root node
    off = np.arange(n0 + 1, dtype=np.int64)
    for l in range(csf.order - 1):
        off = csf.ptr[l][off]
    nnz = csf.nnz
    cuts = [0]
    for r in range(1, world):
        target = nnz * r // world
        cuts.append(max(cuts[-1], int(np.searchsorted(off, target, side="left"))))
    cuts.append(n0)
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def shard_csf(csf: Csf, r0: int, r1: int) -> Csf:
    """Root nodes [r0, r1) as a standalone CSF with rebased child pointers."""
    idx, ptr = [], []
    b, e = r0, r1
    for l in range(csf.order):
        idx.append(np.ascontiguousarray(csf.idx[l][b:e]))
        if l + 1 < csf.order:
            p = csf.ptr[l][b:e + 1]
            ptr.append(np.ascontiguousarray(p - p[0]))
            b, e = int(p[0]), int(p[-1])
    return Csf(list(csf.dims), idx, ptr, np.ascontiguousarray(csf.values[b:e]), csf.names)


def owned_rows(shard: Csf) -> np.ndarray:
    """Root coordinates (output rows) a shard owns."""
    return shard.idx[0]


def broadcast_factors(factors, src: int = 0):
    """Replicate host factor arrays from `src` (torch.distributed, any backend)."""
    import torch
    import torch.distributed as dist
    out = []
    for f in factors:
        t = torch.from_numpy(np.ascontiguousarray(f)) if dist.get_rank() == src else \
            torch.empty(f.shape, dtype=torch.float64)
        dist.broadcast(t, src)
        out.append(t.numpy())
    return out


def gather_dense_rows(local_out: np.ndarray, rows: np.ndarray, tile: int, dim0: int) -> np.ndarray:
    """Assemble the full root-indexed output from every rank's owned rows."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size()
    mine = np.ascontiguousarray(local_out.reshape(dim0, tile)[rows])
    counts = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(counts, torch.tensor([len(rows)], dtype=torch.int64))
    n_max = int(max(c.item() for c in counts))
    pad_rows = torch.full((n_max,), -1, dtype=torch.int64)
    pad_rows[:len(rows)] = torch.from_numpy(rows.astype(np.int64))
    pad_vals = torch.zeros((n_max, tile), dtype=torch.float64)
    pad_vals[:len(rows)] = torch.from_numpy(mine)
    all_rows = [torch.empty_like(pad_rows) for _ in range(world)]
    all_vals = [torch.empty_like(pad_vals) for _ in range(world)]
    dist.all_gather(all_rows, pad_rows)
    dist.all_gather(all_vals, pad_vals)
    full = np.zeros((dim0, tile))
    for r, v in zip(all_rows, all_vals):
        keep = r.numpy() >= 0
        full[r.numpy()[keep]] = v.numpy()[keep]
    return full.reshape(-1)


def gather_sparse_leaves(local_out: np.ndarray, leaf_begin: int, nnz: int) -> np.ndarray:
    """Assemble per-leaf outputs (TTTP) from contiguous leaf ranges."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size()
    meta = torch.tensor([leaf_begin, len(local_out)], dtype=torch.int64)
    metas = [torch.empty_like(meta) for _ in range(world)]
    dist.all_gather(metas, meta)
    n_max = int(max(m[1].item() for m in metas))
    pad = torch.zeros(n_max, dtype=torch.float64)
    pad[:len(local_out)] = torch.from_numpy(np.ascontiguousarray(local_out))
    vals = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(vals, pad)
    full = np.zeros(nnz)
    for m, v in zip(metas, vals):
        b, n = int(m[0]), int(m[1])
        full[b:b + n] = v.numpy()[:n]
    return full


def reduce_dense_output(local_out) -> "np.ndarray":
    """Sum of every rank's full-size output (non-root output modes). Accepts a
    numpy array (host, any backend) or a torch tensor (reduced in place, e.g.
    a CUDA tensor over NCCL); returns the summed array / tensor."""
    import torch
    import torch.distributed as dist
    if isinstance(local_out, torch.Tensor):
        dist.all_reduce(local_out, op=dist.ReduceOp.SUM)
        return local_out
    t = torch.from_numpy(np.ascontiguousarray(local_out, dtype=np.float64)).clone()
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t.numpy()
