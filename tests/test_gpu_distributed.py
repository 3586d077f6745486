"""Two ranks, each running the CUDA plan on its fiber shard.

Both processes share cuda:0 (the driver's GPU tier has one GPU; NCCL refuses
two ranks on one device), so the group is gloo — with CUDA tensors, i.e. the
same device-tensor code path the NCCL job takes: factors broadcast into CUDA
tensors and handed to the plan as device pointers, the plan's device output
wrapped zero-copy (Plan.output_tensor), partial rows of split root slices
reduced and the owned rows all-gathered on the device. The assembled output
must match the whole-tensor oracle at the north-star bar.
"""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

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
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle_bindings as OB
        import paper_2307_05740_b200 as P
        from paper_2307_05740_b200 import distributed as D
        from paper_2307_05740_b200.configs import make_workload
        from test_distributed_cpu import _skewed
        w = _skewed(key) if key in ("ttmc3", "mttkrp4") else make_workload(key, scale=3e-3)
        c = w.cfg
        fac = D.broadcast_factors(w.factors, src=0, device="cuda")
        assert all(t.is_cuda for t in fac)
        f0, f1 = D.partition_fibers(w.csf, world)[rank]
        shard = D.shard_csf_fibers(w.csf, f0, f1)
        dev = P.DeviceCsf(shard)
        plan = P.Plan(c.kind, dev, [t.data_ptr() for t in fac], ranks=c.ranks,
                      flags=P.FLAG_RESIDUAL if c.residual else 0, on_device=True,
                      factor_sizes=[t.numel() for t in fac])
        plan.execute()
        torch.cuda.synchronize()
        local = plan.output_tensor().clone()
        assert local.is_cuda
        if c.kind == 3:
            full = D.gather_sparse_leaves(local, D.leaf_begin_of_fibers(w.csf, f0), w.csf.nnz)
        elif c.kind in (6, 7):
            full = D.reduce_dense_output(local)
        else:
            tile = int(np.prod([r for r in c.ranks if r]))
            rows = D.reduce_split_rows(local, shard, tile)
            full = D.gather_dense_rows(local, rows, tile, w.dims[0])
        assert full.is_cuda
        full = full.cpu().numpy()
        want = OB.oracle_nest(c.kind, w.csf, w.factors, c.ranks, residual=c.residual)
        norm = OB.oracle_abs_nest(c.kind, w.csf, w.factors, c.ranks, residual=c.residual)
        ok = bool(np.all(np.abs(full - want) <= 1e-10 * norm)) and \
            bool(np.all(full[norm == 0] == 0))
        result_q.put((rank, ok, shard.nnz, plan.info()["launches"]))
        plan.close()
        dev.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("key", ["mttkrp3", "ttmc3", "tttp3", "mttkrp4", "ttmc4", "mttkrp3_j"])
def test_two_ranks_run_cuda_plans_on_fiber_shards(key):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, key, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert all(ok for _, ok, _, _ in res), res
    assert all(n > 0 for _, _, n, _ in res)
