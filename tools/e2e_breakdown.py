"""Where does the end-to-end (host buffers -> C-ABI -> host result) time go?
Development tool: python tools/e2e_breakdown.py ttmc3"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2307_05740_b200 as P  # noqa: E402
from paper_2307_05740_b200.configs import make_workload  # noqa: E402
from paper_2307_05740_b200.tensor import Csf  # noqa: E402


def pinned(a):
    t = torch.empty(a.shape, dtype=torch.from_numpy(a[:0]).dtype, pin_memory=True)
    t.numpy()[...] = a
    return t


def main():
    key = sys.argv[1] if len(sys.argv) > 1 else "ttmc3"
    w = make_workload(key)
    c = w.cfg
    pi = [pinned(a) for a in w.csf.idx]
    pp = [pinned(a) for a in w.csf.ptr]
    pv = pinned(w.csf.values)
    pf = [pinned(np.ascontiguousarray(f)) for f in w.factors]
    host = Csf(w.csf.dims, [t.numpy() for t in pi], [t.numpy() for t in pp], pv.numpy())
    out = pinned(np.zeros(w.out_count))
    s = torch.cuda.Stream()
    for it in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dev = P.DeviceCsf(host, stream=s)
        t1 = time.perf_counter()
        plan = P.Plan(c.kind, dev, [t.numpy() for t in pf], ranks=c.ranks,
                      flags=P.FLAG_RESIDUAL if c.residual else 0, stream=s)
        t2 = time.perf_counter()
        plan.execute(s)
        s.synchronize()
        t3 = time.perf_counter()
        plan.read_output(s, out=out.numpy())
        t4 = time.perf_counter()
        plan.close()
        dev.close()
        t5 = time.perf_counter()
        print(f"{key} csf {1e3*(t1-t0):.2f} ms  plan {1e3*(t2-t1):.2f}  exec {1e3*(t3-t2):.2f}  "
              f"d2h {1e3*(t4-t3):.2f}  free {1e3*(t5-t4):.2f}  total {1e3*(t4-t0):.2f}", flush=True)


if __name__ == "__main__":
    main()
