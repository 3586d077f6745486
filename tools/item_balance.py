"""Load balance of the packed TTMc-3 / TTMc-4 kernels (development tool;
BALANCE_KEY=ttmc4 for TTMc-4):
    python tools/item_balance.py [env settings...]
Runs the BASELINE ttmc3 plan with SPTTN_ITEM_CLOCKS=1 (the kernel's
diagnostics instantiation) and prints the spread of per-item and per-SM busy
times from its %globaltimer records, plus a least-squares fit of item time on
the item's groups / leaf steps / tile flushes — the work model that
decomp.cu's item cut (leaf steps + overhead x groups) approximates."""
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2307_05740_b200 as P  # noqa: E402
from paper_2307_05740_b200.configs import make_workload  # noqa: E402


def main():
    os.environ["SPTTN_ITEM_CLOCKS"] = "1"
    key = os.environ.get("BALANCE_KEY", "ttmc3")  # ttmc3, ttmc4 or mttkrp4
    w = make_workload(key, scale=float(os.environ.get("SWEEP_SCALE", "1")))
    c = w.cfg
    s = torch.cuda.Stream()
    dev = P.DeviceCsf(w.csf, stream=s)
    tf = [torch.from_numpy(np.ascontiguousarray(f)).cuda() for f in w.factors]
    for v in sys.argv[1:] or [""]:
        env = dict(kv.split("=") for kv in v.split(",") if kv)
        os.environ.update(env)
        plan = P.Plan(c.kind, dev, [t.data_ptr() for t in tf], ranks=c.ranks, stream=s,
                      on_device=True, factor_sizes=[t.numel() for t in tf])
        recs = []
        for _ in range(5):
            plan.execute(s)
            torch.cuda.synchronize()
            recs.append(plan.item_clocks())
        k = recs[-1]
        t0 = k[:, 0].min()
        st, en, sm = (k[:, 0] - t0) / 1e3, (k[:, 1] - t0) / 1e3, k[:, 2]
        d = en - st
        span = en.max()
        sm_end = np.array([en[sm == i].max() for i in np.unique(sm)])
        sm_busy = np.array([d[sm == i].sum() for i in np.unique(sm)])
        q = lambda a: " ".join(f"{x:7.1f}" for x in np.percentile(a, [0, 10, 50, 90, 100]))
        print(f"[{v}] items {len(d)} span {span:.1f} us; item us p0/10/50/90/100: {q(d)}")
        print(f"   SM last end: {q(sm_end)}   SM busy sum: {q(sm_busy)}")
        print(f"   efficiency sum(d)/(span*items) = {d.sum() / (span * len(d)):.3f}")
        # work model fit over the runs (median item time per item)
        dm = np.median(np.stack([(r[:, 1] - r[:, 0]) / 1e3 for r in recs]), axis=0)
        X = np.stack([k[:, 3], k[:, 4], k[:, 5]], axis=1).astype(np.float64)
        coef, res, *_ = np.linalg.lstsq(X, dm, rcond=None)
        pred = X @ coef
        r2 = 1 - ((dm - pred) ** 2).sum() / ((dm - dm.mean()) ** 2).sum()
        print(f"   fit us = {coef[0]:.4f}*groups + {coef[1]:.4f}*steps + {coef[2]:.4f}*flushes"
              f"  (R^2 {r2:.3f}); per-group overhead in steps = {coef[0] / coef[1]:.2f},"
              f" per-flush = {coef[2] / coef[1]:.2f}")
        plan.close()
        for kk in env:
            os.environ.pop(kk)


if __name__ == "__main__":
    main()
