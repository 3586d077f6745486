"""World-size-2/3 gloo tests of the sharded (multi-GPU) path on CPU.

The nonzeros are cut at fiber granularity (distributed.partition_fibers), so
a root slice can be split across ranks; each rank's shard is computed here by
the C oracle (standing in for its device plan — tests/test_gpu_distributed.py
runs the CUDA plans), partial rows of split slices are summed in rank order
(reduce_split_rows), and the gathered output must match the whole-tensor
oracle result at the north-star bar (split rows are summed in a different
association, so not bit-for-bit; everything else is bit-identical).
"""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _skewed(key):
    """BASELINE-shaped tensor plus one giant root slice (~45 % of nnz), so a
    world-2/3 cut must split it."""
    from paper_2307_05740_b200.configs import make_workload
    from paper_2307_05740_b200.tensor import Csf
    w = make_workload(key, scale=3e-3)
    coo, vals = w.csf.to_coo()
    rng = np.random.default_rng(5)
    n_hot = int(0.8 * len(vals))
    hot = np.stack([np.full(n_hot, int(coo[0, 0]))] +
                   [rng.integers(0, d, n_hot) for d in w.dims[1:]], axis=1)
    coo = np.concatenate([coo, hot])
    vals = np.concatenate([vals, rng.uniform(-1, 1, n_hot)])
    w.csf = Csf.from_coo(list(w.dims), coo, vals)
    return w


def _worker(rank, world, port, key, skew, result_q):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle_bindings as OB
        from paper_2307_05740_b200 import distributed as D
        from paper_2307_05740_b200.configs import make_workload
        w = _skewed(key) if skew else make_workload(key, scale=3e-3)
        c = w.cfg
        factors = [t.numpy() for t in D.broadcast_factors(w.factors, src=0)]
        parts = D.partition_fibers(w.csf, world)
        f0, f1 = parts[rank]
        shard = D.shard_csf_fibers(w.csf, f0, f1)
        local = torch.from_numpy(OB.oracle_nest(c.kind, shard, factors, c.ranks,
                                                residual=c.residual))
        want = OB.oracle_nest(c.kind, w.csf, w.factors, c.ranks, residual=c.residual)
        norm = OB.oracle_abs_nest(c.kind, w.csf, w.factors, c.ranks, residual=c.residual)
        if c.kind == 3:
            full = D.gather_sparse_leaves(local, D.leaf_begin_of_fibers(w.csf, f0), w.csf.nnz)
        elif c.kind in (6, 7):  # non-root output: every shard adds into every row
            full = D.reduce_dense_output(local)
        else:
            tile = int(np.prod([r for r in c.ranks if r]))
            rows = D.reduce_split_rows(local, shard, tile)
            full = D.gather_dense_rows(local, rows, tile, w.dims[0])
        full = full.numpy()
        ok = bool(np.all(np.abs(full - want) <= 1e-10 * norm)) and \
            bool(np.all(full[norm == 0] == 0))
        result_q.put((rank, ok, shard.nnz, int(shard.idx[0][0]) if len(shard.idx[0]) else -1,
                      int(shard.idx[0][-1]) if len(shard.idx[0]) else -1))
    finally:
        dist.destroy_process_group()


def _run(key, world, skew):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, key, skew, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("key", ["mttkrp3", "ttmc3", "tttp3", "mttkrp4", "ttmc4", "mttkrp3_j",
                                 "mttkrp3_k"])
def test_sharded_equals_whole_world2(key):
    res = _run(key, 2, False)
    assert all(ok for _, ok, _, _, _ in res), res


@pytest.mark.parametrize("key", ["mttkrp3", "ttmc3", "mttkrp4", "ttmc4"])
def test_giant_slice_is_split_and_reduced_world3(key):
    """One root slice holds ~45 % of the nonzeros: the fiber cut splits it
    across ranks (same root row at a shard boundary), nnz stays balanced, and
    the partial rows are summed in rank order."""
    res = _run(key, 3, True)
    assert all(ok for _, ok, _, _, _ in res), res
    nnz = [n for _, _, n, _, _ in res]
    assert max(nnz) <= 1.05 * sum(nnz) / 3 + 64, nnz
    # a boundary row shared by consecutive ranks
    assert any(res[r][4] == res[r + 1][3] for r in range(2)), res


def test_partitions_cover_and_balance():
    sys.path.insert(0, str(ROOT))
    from paper_2307_05740_b200 import distributed as D
    from paper_2307_05740_b200.configs import make_workload
    w = make_workload("ttmc3", scale=1e-3)
    for world in (2, 4, 8):
        parts = D.partition_roots(w.csf, world)
        assert parts[0][0] == 0 and parts[-1][1] == w.csf.level_sizes()[0]
        assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
        nnz = [D.shard_csf(w.csf, a, b).nnz for a, b in parts]
        assert sum(nnz) == w.csf.nnz
        off = [D.leaf_range_of_roots(w.csf, r, r + 1) for r in range(w.csf.level_sizes()[0])]
        biggest = max(b - a for a, b in off)
        assert max(nnz) <= w.csf.nnz / world + biggest
        fparts = D.partition_fibers(w.csf, world)
        shards = [D.shard_csf_fibers(w.csf, a, b) for a, b in fparts]
        assert sum(s.nnz for s in shards) == w.csf.nnz
        # fiber cuts: within one fiber of the ideal share
        fl = D.fiber_level(w.csf)
        foff = D._leaf_offsets(w.csf, fl)
        longest = int(np.max(np.diff(foff)))
        assert max(s.nnz for s in shards) <= w.csf.nnz / world + longest
        # leaves are the original leaves, in order
        assert np.array_equal(np.concatenate([s.values for s in shards]), w.csf.values)
