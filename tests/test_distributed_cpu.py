"""World-size-2 gloo tests of the sharded (multi-GPU) path on CPU: shards of
the root level computed independently (here by the C oracle, standing in for
each rank's device plan) and gathered must equal the whole-tensor result,
for dense root-row outputs and per-leaf TTTP outputs."""
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


def _worker(rank, world, port, key, result_q):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle_bindings as OB
        from paper_2307_05740_b200 import distributed as D
        from paper_2307_05740_b200.configs import make_workload
        w = make_workload(key, scale=3e-3)
        c = w.cfg
        factors = D.broadcast_factors(w.factors, src=0)
        parts = D.partition_roots(w.csf, world)
        r0, r1 = parts[rank]
        shard = D.shard_csf(w.csf, r0, r1)
        local = OB.oracle_nest(c.kind, shard, factors, c.ranks, residual=c.residual)
        if c.kind == 3:
            lb, _ = D.leaf_range_of_roots(w.csf, r0, r1)
            full = D.gather_sparse_leaves(local, lb, w.csf.nnz)
        elif c.kind in (6, 7):  # non-root output: every shard adds into every row
            full = D.reduce_dense_output(local)
            want = OB.oracle_nest(c.kind, w.csf, w.factors, c.ranks)
            scale = OB.oracle_nest(c.kind, w.csf.abs(), [np.abs(f) for f in w.factors], c.ranks)
            ok = bool(np.all(np.abs(full - want) <= 1e-12 * scale + 1e-300))
            result_q.put((rank, ok, [p[1] - p[0] for p in parts], shard.nnz))
            return
        else:
            tile = int(np.prod([r for r in c.ranks if r]))
            full = D.gather_dense_rows(local, D.owned_rows(shard), tile, w.dims[0])
        want = OB.oracle_nest(c.kind, w.csf, w.factors, c.ranks, residual=c.residual)
        result_q.put((rank, bool(np.array_equal(full, want)),
                      [p[1] - p[0] for p in parts], shard.nnz))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("key", ["mttkrp3", "ttmc3", "tttp3", "mttkrp4", "ttmc4", "mttkrp3_j",
                                 "mttkrp3_k"])
def test_sharded_equals_whole_world2(key):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, key, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _, _ in res), res
    nnzs = [n for _, _, _, n in res]
    assert sum(nnzs) > 0


def test_partition_balances_nnz():
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
        # contiguous cuts: no shard exceeds its share by more than the largest slice
        off = [D.leaf_range_of_roots(w.csf, r, r + 1) for r in range(w.csf.level_sizes()[0])]
        biggest = max(b - a for a, b in off)
        assert max(nnz) <= w.csf.nnz / world + biggest
