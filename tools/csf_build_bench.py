"""Device CSF construction (spttn_csf_from_coo) vs the host build_csf
restatement (datagen, radix sort) and the reference's build_csf
(oracle/_ref, test infrastructure) on the BASELINE tensors.
Development tool:  python tools/csf_build_bench.py ttmc3 mttkrp3 ..."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import paper_2307_05740_b200 as P  # noqa: E402
from paper_2307_05740_b200.configs import make_workload  # noqa: E402
from paper_2307_05740_b200.tensor import Csf  # noqa: E402


def main():
    for key in sys.argv[1:] or ["ttmc3"]:
        w = make_workload(key)
        coo, vals = w.csf.to_coo()
        perm = np.random.default_rng(1).permutation(vals.shape[0])
        coo, vals = np.ascontiguousarray(coo[perm]), np.ascontiguousarray(vals[perm])
        pc = torch.from_numpy(coo).pin_memory()
        pv = torch.from_numpy(vals).pin_memory()
        ts = []
        for _ in range(4):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            dev = P.DeviceCsf.from_coo(w.csf.dims, pc.numpy(), pv.numpy())
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
            dev.close()
        t0 = time.perf_counter()
        Csf.from_coo(w.csf.dims, coo, vals)
        th = time.perf_counter() - t0
        tr = float("nan")
        try:
            import oracle_bindings as OB
            if OB.ref_available():
                t0 = time.perf_counter()
                OB.ref_build_csf(list(w.cfg.mode_names), list(w.csf.dims), coo, vals,
                                 list(w.cfg.mode_names))
                tr = time.perf_counter() - t0
        except Exception as e:  # noqa: BLE001
            print("reference build unavailable:", e)
        print(f"{key}: nnz {vals.shape[0]}  device (H2D from pinned + build) {1e3*min(ts[1:]):.1f} ms"
              f"  host restatement {1e3*th:.0f} ms  reference build_csf {1e3*tr:.0f} ms", flush=True)


if __name__ == "__main__":
    main()
