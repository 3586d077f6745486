"""Kernel-variant sweep on one workload (development tool, not the bench).

    python tools/sweep.py ttmc3 'SPTTN_GROUP_OVERHEAD=6' 'SPTTN_GROUP_OVERHEAD=12' ...

Generates the BASELINE workload once, then for each variant (env settings
read at plan creation) times the fused-nest kernel with CUDA events, L2
flushed between launches, and checks the output against the first variant.
"""
import os
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2307_05740_b200 as P  # noqa: E402
from paper_2307_05740_b200.configs import algorithmic_flops, make_workload  # noqa: E402


def main():
    key = sys.argv[1]
    variants = sys.argv[2:] or [""]
    scale = float(os.environ.get("SWEEP_SCALE", "1"))
    w = make_workload(key, scale=scale)
    c = w.cfg
    s = torch.cuda.Stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    dev = P.DeviceCsf(w.csf, stream=s)
    tf = [torch.from_numpy(np.ascontiguousarray(f)).cuda() for f in w.factors]
    ref = None
    flops = algorithmic_flops(w)
    for v in variants:
        env = dict(kv.split("=") for kv in v.split(",") if kv)
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        plan = P.Plan(c.kind, dev, [t.data_ptr() for t in tf], ranks=c.ranks,
                      flags=P.FLAG_RESIDUAL if c.residual else 0, stream=s, on_device=True,
                      factor_sizes=[t.numel() for t in tf])
        for k, o in old.items():
            if o is None:
                os.environ.pop(k)
            else:
                os.environ[k] = o
        for _ in range(3):
            plan.execute(s)
        ts = []
        with torch.cuda.stream(s):
            for _ in range(10):
                flush.zero_()
                e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
                e0.record(s)
                plan.execute_stage(0, s)
                e1.record(s)
                plan.execute_stage(1, s)
                e2.record(s)
                ts.append((e0, e1, e2))
        whole = []
        with torch.cuda.stream(s):
            for _ in range(10):
                flush.zero_()
                e0, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(2))
                e0.record(s)
                plan.execute(s)
                e2.record(s)
                whole.append((e0, e2))
        torch.cuda.synchronize()
        step = statistics.median(a.elapsed_time(b) for a, b in whole)
        ms = [a.elapsed_time(b) for a, b, _ in ts]
        epi = statistics.median(b.elapsed_time(c) for _, b, c in ts)
        out = plan.read_output(s)
        if ref is None:
            ref = out
            err = 0.0
        else:
            err = float(np.max(np.abs(out - ref)) / max(1e-300, np.max(np.abs(ref))))
        info = plan.info()
        print(f"{key} [{v}] kernel {statistics.median(ms)*1e3:8.1f} us (min {min(ms)*1e3:.1f}) epi {epi*1e3:6.1f} us step {step*1e3:7.1f} us"
              f"  {flops/statistics.median(ms)/1e9:6.2f} TF/s  items {info['items']} "
              f"segs {info['segments']} split {info['split_slices']}  relerr {err:.2e}",
              flush=True)
        plan.close()


if __name__ == "__main__":
    main()
