"""Multi-GPU sharding of the fused nests.

One process per GPU; the nonzeros of one CSF tensor are cut into N
contiguous pieces balanced by nnz, at FIBER granularity (the level above the
leaves: (i,j) fibers for order 3, (i,j,k) for order 4) — not at root slices,
because Zipf root slices hold up to 12 % of all nonzeros (MTTKRP-4), which at
N = 8 would leave one rank with ~2x its share. Every pinned nest is linear in
the fibers, so a shard is just a standalone CSF over its fibers (with their
ancestors; a root slice cut by a shard boundary appears in both shards):

  * `partition_fibers` / `shard_csf_fibers` — the cut and the shard CSF;
  * factors are replicated (`broadcast_factors`: one broadcast each, NCCL
    over NVLink for CUDA tensors — the only input exchange);
  * root-indexed outputs (MTTKRP A[i,:], TTMc Y[i,:,:]): each rank computes
    its shard's rows; a root row cut by a boundary is PARTIAL on every rank
    holding a piece, and `reduce_split_rows` sums those pieces in rank order
    into the lowest such rank (one all_gather of 2 rows per rank) — the
    "one partial-row reduction" that replaces the paper's CTF reduction +
    redistribution;
  * `gather_dense_rows` / `gather_sparse_leaves` assemble the full output on
    every rank when a caller needs it (all_gather of owned rows / leaf
    ranges); TTTP's per-leaf outputs need no reduction at all;
  * outputs NOT indexed by the root mode (MTTKRP for modes j / k) get every
    rank's contribution in every row: `reduce_dense_output` (one all_reduce).

Every collective takes torch tensors on the device the process group works
on: CUDA tensors for NCCL (the device output of a plan is wrapped zero-copy by
`engine.Plan.output_tensor()`), CPU tensors for gloo. Root-slice cuts
(`partition_roots`, `shard_csf`) are kept for callers that want whole slices
per rank (no reduction step).

bench.py runs N independent full-size tensors (weak scaling, one per rank);
`--shard` runs one tensor split with these helpers (strong scaling).
"""
from __future__ import annotations

import numpy as np

from .tensor import Csf


# ---- cuts --------------------------------------------------------------------

def _leaf_offsets(csf: Csf, level: int) -> np.ndarray:
    """First leaf of every node at `level` (n_level + 1 entries)."""
    off = np.arange(csf.level_sizes()[level] + 1, dtype=np.int64)
    for l in range(level, csf.order - 1):
        off = csf.ptr[l][off]
    return off


def leaf_range_of_roots(csf: Csf, r0: int, r1: int) -> tuple[int, int]:
    a, b = r0, r1
    for l in range(csf.order - 1):
        a, b = int(csf.ptr[l][a]), int(csf.ptr[l][b])
    return a, b


def fiber_level(csf: Csf) -> int:
    return max(0, csf.order - 2)


def partition_fibers(csf: Csf, world: int) -> list[tuple[int, int]]:
    """Contiguous fiber ranges [f0, f1) (nodes of level order-2) with
    ~nnz/world leaves each; a root slice may be cut."""
    lvl = fiber_level(csf)
    off = _leaf_offsets(csf, lvl)
    n = csf.level_sizes()[lvl]
    cuts = [0]
    for r in range(1, world):
        target = csf.nnz * r // world
        cuts.append(max(cuts[-1], min(n, int(np.searchsorted(off, target, side="left")))))
    cuts.append(n)
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def partition_roots(csf: Csf, world: int) -> list[tuple[int, int]]:
    """Contiguous root-node ranges [r0, r1) with ~nnz/world leaves each."""
    n0 = csf.level_sizes()[0]
    off = _leaf_offsets(csf, 0)
    cuts = [0]
    for r in range(1, world):
        target = csf.nnz * r // world
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


def shard_csf_fibers(csf: Csf, f0: int, f1: int) -> Csf:
    """Fibers [f0, f1) of the fiber level, with their leaves below and their
    ancestors above (an ancestor cut by f0 / f1 keeps only the children in
    range), as a standalone CSF in the same mode sizes."""
    d = csf.order
    lvl = fiber_level(csf)
    lo = [0] * d
    hi = [0] * d
    lo[lvl], hi[lvl] = f0, f1
    for l in range(lvl - 1, -1, -1):  # ancestors: parents of the first / last node
        if hi[l + 1] > lo[l + 1]:
            lo[l] = int(np.searchsorted(csf.ptr[l], lo[l + 1], side="right")) - 1
            hi[l] = int(np.searchsorted(csf.ptr[l], hi[l + 1] - 1, side="right"))
        else:
            lo[l] = hi[l] = 0
    for l in range(lvl, d - 1):  # descendants: contiguous child ranges
        lo[l + 1] = int(csf.ptr[l][lo[l]]) if hi[l] > lo[l] else 0
        hi[l + 1] = int(csf.ptr[l][hi[l]]) if hi[l] > lo[l] else 0
    idx, ptr = [], []
    for l in range(d):
        idx.append(np.ascontiguousarray(csf.idx[l][lo[l]:hi[l]]))
        if l + 1 < d:
            if hi[l] > lo[l]:
                p = np.clip(csf.ptr[l][lo[l]:hi[l] + 1], lo[l + 1], hi[l + 1]) - lo[l + 1]
            else:
                p = np.zeros(1, np.int64)
            ptr.append(np.ascontiguousarray(p, dtype=np.int64))
    return Csf(list(csf.dims), idx, ptr,
               np.ascontiguousarray(csf.values[lo[d - 1]:hi[d - 1]]), csf.names)


def leaf_begin_of_fibers(csf: Csf, f0: int) -> int:
    return int(_leaf_offsets(csf, fiber_level(csf))[f0])


def owned_rows(shard: Csf) -> np.ndarray:
    """Root coordinates (output rows) a root-slice shard owns."""
    return shard.idx[0]


# ---- collectives (torch tensors on the process group's device) --------------

def _dev():
    import torch
    import torch.distributed as dist
    if dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def broadcast_factors(factors, src: int = 0, device=None):
    """Replicate factor matrices from `src`. Accepts numpy arrays or torch
    tensors; returns torch tensors on `device` (default: CUDA for NCCL, CPU
    for gloo) — pass their data_ptr()s to a plan with on_device=True."""
    import torch
    import torch.distributed as dist
    dev = torch.device(device) if device is not None else _dev()
    out = []
    for f in factors:
        if dist.get_rank() == src:
            t = (f if isinstance(f, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(f)))
            t = t.to(dev, dtype=torch.float64).contiguous()
        else:
            t = torch.empty(tuple(f.shape), dtype=torch.float64, device=dev)
        dist.broadcast(t, src)
        out.append(t)
    return out


def reduce_split_rows(local_out, shard: Csf, tile: int):
    """Sum the partial rows of root slices cut by shard boundaries.

    `local_out` (torch tensor, dim0 * tile, on the group's device) holds this
    rank's shard result. Its first and last root rows may be partial; every
    rank contributes those (at most 2 rows, fixed size) to one all_gather,
    and each row held by several ranks is summed in rank order into the
    lowest of them (deterministic) and zeroed on the others. Returns the
    rows this rank owns afterwards (numpy)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size()
    rank = dist.get_rank()
    dev = local_out.device
    rows = shard.idx[0]
    y = local_out.view(-1, tile)
    ids = torch.full((2,), -1, dtype=torch.int64, device=dev)
    vals = torch.zeros((2, tile), dtype=torch.float64, device=dev)
    if len(rows):
        ids[0] = int(rows[0])
        vals[0] = y[int(rows[0])]
        if len(rows) > 1:
            ids[1] = int(rows[-1])
            vals[1] = y[int(rows[-1])]
    all_ids = [torch.empty_like(ids) for _ in range(world)]
    all_vals = [torch.empty_like(vals) for _ in range(world)]
    dist.all_gather(all_ids, ids)
    dist.all_gather(all_vals, vals)
    holders: dict[int, list[tuple[int, int]]] = {}
    host_ids = [a.cpu().numpy() for a in all_ids]
    for r in range(world):
        for s in range(2):
            i = int(host_ids[r][s])
            if i >= 0 and (r, s) not in holders.get(i, []) and \
                    not (s == 1 and host_ids[r][0] == i):
                holders.setdefault(i, []).append((r, s))
    owned = set(int(x) for x in rows)
    for i, hs in holders.items():
        if len(hs) < 2 or all(r != rank for r, _ in hs):
            continue
        first = min(r for r, _ in hs)
        if rank == first:
            acc = torch.zeros(tile, dtype=torch.float64, device=dev)
            for r, s in sorted(hs):
                acc = acc + all_vals[r][s]
            y[i] = acc
        else:
            y[i] = 0.0
            owned.discard(i)
    return np.array(sorted(owned), dtype=np.int64)


def gather_dense_rows(local_out, rows: np.ndarray, tile: int, dim0: int):
    """Assemble the full root-indexed output from every rank's owned rows
    (torch tensor in / out, on the group's device)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size()
    dev = local_out.device
    y = local_out.view(dim0, tile)
    r_t = torch.as_tensor(np.asarray(rows, dtype=np.int64), device=dev)
    n = torch.tensor([r_t.numel()], dtype=torch.int64, device=dev)
    counts = [torch.empty_like(n) for _ in range(world)]
    dist.all_gather(counts, n)
    n_max = int(max(int(c.item()) for c in counts))
    pad_rows = torch.full((n_max,), -1, dtype=torch.int64, device=dev)
    pad_vals = torch.zeros((n_max, tile), dtype=torch.float64, device=dev)
    if r_t.numel():
        pad_rows[:r_t.numel()] = r_t
        pad_vals[:r_t.numel()] = y[r_t]
    all_rows = [torch.empty_like(pad_rows) for _ in range(world)]
    all_vals = [torch.empty_like(pad_vals) for _ in range(world)]
    dist.all_gather(all_rows, pad_rows)
    dist.all_gather(all_vals, pad_vals)
    full = torch.zeros((dim0, tile), dtype=torch.float64, device=dev)
    for r, v in zip(all_rows, all_vals):
        keep = r >= 0
        full[r[keep]] = v[keep]
    return full.view(-1)


def gather_sparse_leaves(local_out, leaf_begin: int, nnz: int):
    """Assemble per-leaf outputs (TTTP) from contiguous leaf ranges."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size()
    dev = local_out.device
    meta = torch.tensor([leaf_begin, local_out.numel()], dtype=torch.int64, device=dev)
    metas = [torch.empty_like(meta) for _ in range(world)]
    dist.all_gather(metas, meta)
    n_max = int(max(int(m[1].item()) for m in metas))
    pad = torch.zeros(n_max, dtype=torch.float64, device=dev)
    pad[:local_out.numel()] = local_out
    vals = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(vals, pad)
    full = torch.zeros(nnz, dtype=torch.float64, device=dev)
    for m, v in zip(metas, vals):
        b, n = int(m[0]), int(m[1])
        full[b:b + n] = v[:n]
    return full


def reduce_dense_output(local_out):
    """Sum of every rank's full-size output (non-root output modes), in place
    on a torch tensor (CUDA over NCCL, CPU over gloo)."""
    import torch.distributed as dist
    dist.all_reduce(local_out, op=dist.ReduceOp.SUM)
    return local_out
