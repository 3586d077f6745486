"""SpTTN fused-nest benchmark on B200 (BASELINE.json metric: nnz/s + roofline).

A "step" is one execution of the pinned fused nest over the whole synthetic
tensor of a BASELINE.json config. The headline line (value / ms_per_step /
roofline / e2e / cpu_baseline) is configs[1], Order-3 TTMc (Zipf 1.1,
1e7 nnz, R=S=16); the other four configs are measured the same way and
reported under "configs" (skip with --configs ttmc3).

  value        nnz/s of the whole job, inputs resident in HBM, device-timed
               with CUDA events on the launch stream, L2 flushed (256 MB
               write) between timed steps, max over ranks.
  e2e          same metric through the C-ABI with HOST (pinned) buffers:
               CSF + factor H2D, device layout + plan build, kernels, D2H.
  roofline     dominant kernel (the fused nest kernel) against the north-star
               roof max(bytes_alg/HBM, flops_alg/FP64): "bound" names the
               larger term; fp64 peaks are measured here (DMMA / DFMA probe)
               because MEASURED_PEAKS.json has none.
  cpu_baseline the reference executor (oracle/_ref, compiled from
               /root/reference) on the same pinned nest, 1 host core, on a
               bounded root-slice sample of the same tensor.

--impl reference runs the reference's CPU implementation of the path on all
host threads (one plan per thread over nnz-balanced root-slice partitions)
on a bounded sample, printing the same JSON keys.

Multi-GPU (torchrun): each rank owns an independent tensor of the config's
size (seed + rank): no data-path collective, "scaling": "weak".
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "SpTTN nnz/s (MTTKRP, TTMc, TTTP) + % of HBM/fp64 roofline on 1 B200"
WORKLOAD = ("ttmc3: BASELINE configs[1] Order-3 TTMc 20000^3, 1e7 nnz Zipf(1.1), U,V 20000x16 "
            "N(0,1), pinned nest ((T*V)*U)")
HEADLINE = "ttmc3"
ORDER = ["mttkrp3", "ttmc3", "tttp3", "mttkrp4", "ttmc4", "mttkrp3_j", "mttkrp3_k"]
L2_FLUSH_BYTES = 256 << 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--configs", default="all", help="comma list or 'all'")
    ap.add_argument("--cpu-seconds", type=float, default=3.0,
                    help="target CPU time of one bounded reference sample")
    ap.add_argument("--dump-workload", default=None, help=argparse.SUPPRESS)
    ap.add_argument("--out", default=None, help=argparse.SUPPRESS)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-parity", action="store_true",
                    help="skip the per-config parity check against the C oracle")
    ap.add_argument("--shard", action="store_true",
                    help="N>1: split ONE tensor's fibers over the ranks (strong "
                         "scaling) instead of one independent tensor per rank (weak)")
    return ap.parse_args()


def _load_traffic():
    """Per-launch DRAM traffic of each config's dominant kernel, from the
    committed ncu --set full summaries (profiles/traffic.json)."""
    try:
        return json.loads((ROOT / "profiles" / "traffic.json").read_text())
    except (OSError, ValueError):
        return {}


TRAFFIC = _load_traffic()


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text()), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.f = None

    def __enter__(self):
        try:
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=self.f, stderr=subprocess.DEVNULL)
            # nvidia-smi needs ~0.1-0.3 s to start: wait for its first sample so
            # even short timed regions are covered (that pre-region sample is
            # dropped from the summary when later ones exist)
            t0 = time.time()
            while time.time() - t0 < 3.0 and not Path(self.f.name).read_text().strip():
                time.sleep(0.01)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.f.flush()
        rows = []
        for line in Path(self.f.name).read_text().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        if len(rows) > 1:
            rows = rows[1:]  # the first sample predates the timed region
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


def fp64_peaks():
    lib = C.CDLL(str(ROOT / "paper_2307_05740_b200" / "lib" / "libspttn_probe.so"))
    lib.spttn_probe_fp64_tflops.restype = C.c_double
    lib.spttn_probe_fp64_tflops.argtypes = [C.c_int, C.c_int]
    return {"dmma_tflops": lib.spttn_probe_fp64_tflops(0, 3),
            "dfma_tflops": lib.spttn_probe_fp64_tflops(1, 3)}


def pinned_copy(a: np.ndarray):
    import torch
    t = torch.empty(a.shape, dtype=torch.from_numpy(a[:0]).dtype, pin_memory=True)
    t.numpy()[...] = a
    return t


def device_time_config(P, w, steps, warmup, stream, flush, ev):
    """Device-timed steps of one workload. Returns per-stage mean ms and plan."""
    import torch
    c = w.cfg
    dev = P.DeviceCsf(w.csf, stream=stream)
    tfac = [torch.from_numpy(np.ascontiguousarray(f)).to("cuda") for f in w.factors]
    plan = P.Plan(c.kind, dev, [t.data_ptr() for t in tfac], ranks=c.ranks,
                  flags=P.FLAG_RESIDUAL if c.residual else 0, stream=stream, on_device=True,
                  factor_sizes=[t.numel() for t in tfac])
    for _ in range(warmup):
        plan.execute(stream)
    torch.cuda.synchronize()
    # the K timed steps: one whole execute each (nest kernel + fix-up, which
    # starts under programmatic dependent launch while the nest drains)
    whole = []
    with torch.cuda.stream(stream):
        for _ in range(steps):
            flush.zero_()  # evict L2 (256 MB write) between timed steps
            e0, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(2))
            e0.record(stream)
            plan.execute(stream)
            e2.record(stream)
            ev.append((e0, e2))
            whole.append((e0, e2))
    torch.cuda.synchronize()
    # diagnostic pass (after the timed steps): the two stages timed apart,
    # for the nest kernel's roofline (an event between them serialises the
    # fix-up launch, so these two add up to more than a step)
    main, epi = [], []
    with torch.cuda.stream(stream):
        for _ in range(steps):
            flush.zero_()
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record(stream)
            plan.execute_stage(0, stream)
            e1.record(stream)
            plan.execute_stage(1, stream)
            e2.record(stream)
            main.append((e0, e1))
            epi.append((e1, e2))
    torch.cuda.synchronize()
    m = [a.elapsed_time(b) for a, b in main]
    e = [a.elapsed_time(b) for a, b in epi]
    w_ms = [a.elapsed_time(b) for a, b in whole]
    return {"main_ms": statistics.mean(m), "epi_ms": statistics.mean(e),
            "main_ms_min": min(m), "main_ms_median": statistics.median(m),
            "main_ms_all": [round(x, 4) for x in m],
            "step_ms": statistics.mean(w_ms)}, plan, dev, tfac


def parity_check(P, w, plan, stream):
    """Checker, outside every timed region: the output of the plan just timed
    against the plain-C oracle (test infrastructure, pinned to the reference
    by tests/test_oracle.py) on the same full-size inputs. Bar: |gpu - cpu|
    <= 1e-10 * sum|contributions| per entry, entries without contributions
    exactly 0, a second execute bit-identical (owner-computes kernels)."""
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_bindings as OB
    c = w.cfg
    t0 = time.perf_counter()
    plan.execute(stream)
    got = plan.read_output(stream)
    plan.execute(stream)
    again = plan.read_output(stream)
    want = OB.oracle_nest(c.kind, w.csf, w.factors, c.ranks, residual=c.residual)
    norm = OB.oracle_abs_nest(c.kind, w.csf, w.factors, c.ranks, residual=c.residual)
    err = np.abs(got - want)
    nz = norm > 0
    rel = float((err[nz] / norm[nz]).max()) if nz.any() else 0.0
    # non-root MTTKRP-3 is owner-computes unless it fell back to the atomic kernels
    atomic = c.kind in (P.NEST_MTTKRP3_J, P.NEST_MTTKRP3_K) and plan.info()["variant"] != 5
    return {"checker": "oracle/spttn_oracle.c (pinned to the reference executor)",
            "entries": int(got.size), "max_normalised_err": rel, "tol": 1e-10,
            "outside_tol": int((err > 1e-10 * norm).sum()),
            "zero_entries": int((~nz).sum()),
            "nonzero_where_zero": int((got[~nz] != 0.0).sum()),
            "rerun_bit_identical": bool(np.array_equal(got, again)),
            "rerun_required_bit_identical": not atomic,
            "ok": bool(rel <= 1e-10 and not (got[~nz] != 0.0).any() and
                       (atomic or np.array_equal(got, again))),
            "seconds": time.perf_counter() - t0}


def e2e_config(P, w, steps, stream):
    """Through the C-ABI from pinned host buffers: H2D CSF + factors, device
    layout + plan build, fused nest, D2H of the output — every step."""
    import torch
    from paper_2307_05740_b200.tensor import Csf
    c = w.cfg
    pin_idx = [pinned_copy(a) for a in w.csf.idx]
    pin_ptr = [pinned_copy(a) for a in w.csf.ptr]
    pin_val = pinned_copy(w.csf.values)
    pin_fac = [pinned_copy(np.ascontiguousarray(f)) for f in w.factors]
    host = Csf(w.csf.dims, [t.numpy() for t in pin_idx], [t.numpy() for t in pin_ptr],
               pin_val.numpy())
    out = pinned_copy(np.zeros(w.out_count))
    h2d = sum(t.numel() * 8 for t in pin_idx + pin_ptr) + pin_val.numel() * 8 + \
        sum(t.numel() * 8 for t in pin_fac)
    d2h = w.out_count * 8
    times, parts = [], []
    for it in range(steps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        # factors first (small), then the CSF: its leaf values stream up in the
        # background (spttn_csf_create_async) while the plan's decomposition
        # runs — no plan-side copy queues behind the values on the copy engine
        with torch.cuda.stream(stream):
            dfac = [t.to("cuda", non_blocking=True) for t in pin_fac]
        dev = P.DeviceCsf(host, stream=stream, async_values=True)
        ta = time.perf_counter()
        plan = P.Plan(c.kind, dev, [t.data_ptr() for t in dfac], ranks=c.ranks,
                      flags=P.FLAG_RESIDUAL if c.residual else 0, stream=stream,
                      on_device=True, factor_sizes=[t.numel() for t in dfac])
        tb = time.perf_counter()
        plan.execute(stream)
        plan.read_output(stream, out=out.numpy())
        t1 = time.perf_counter()
        plan.close()
        dev.close()
        del dfac
        if it > 0:
            times.append(t1 - t0)
            parts.append((ta - t0, tb - ta, t1 - tb))
    brk = [statistics.mean(p[i] for p in parts) * 1e3 for i in range(3)]
    # the solver-loop case (CP-ALS / HOOI sweep): one plan reused, each step
    # uploads the step's factors from pinned memory, executes and reads the
    # output back (spttn_plan_set_factors + spttn_execute + spttn_read_output)
    dev = P.DeviceCsf(host, stream=stream)
    plan = P.Plan(c.kind, dev, [t.numpy() for t in pin_fac], ranks=c.ranks,
                  flags=P.FLAG_RESIDUAL if c.residual else 0, stream=stream)
    als = []
    fac_bytes = sum(t.numel() * 8 for t in pin_fac)
    for it in range(steps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        plan.set_factors([t.numpy() for t in pin_fac], stream)
        plan.execute(stream)
        plan.read_output(stream, out=out.numpy())
        t1 = time.perf_counter()
        if it > 0:
            als.append(t1 - t0)
    plan.close()
    dev.close()
    return {"seconds": statistics.mean(times), "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h),
            "path": "factors H2D, DeviceCsf (async values) + Plan + execute + read_output",
            "breakdown_ms": {"csf_h2d_layout": brk[0], "plan_h2d_decomp": brk[1],
                             "execute_d2h": brk[2]},
            "als_loop": {"seconds": statistics.mean(als), "h2d_bytes_per_step": int(fac_bytes),
                         "d2h_bytes_per_step": int(d2h)}}


def ref_args(w):
    c = w.cfg
    dims = dict(zip(c.mode_names, w.dims))
    rank_names = {1: ["r"], 2: ["r", "s"], 3: ["r"], 4: ["r"], 5: ["r", "s", "t"], 6: ["r"],
                  7: ["r"]}[c.kind]
    for n, r in zip(rank_names, c.ranks):
        dims[n] = r
    return c.kernel, dims, c.path, c.order_text


def _ref_run(w, sub, threads, repeats=1):
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_bindings as OB  # the reference build (test infrastructure)
    from paper_2307_05740_b200.configs import Workload
    ws = Workload(w.cfg, sub, w.factors, w.dims, sub.nnz)
    kernel, dims, path, order = ref_args(w)
    if w.cfg.residual:  # reference flow for rho: S on unit values
        sub = sub.with_values(np.ones_like(sub.values))
    if threads == 1:
        _, st = OB.ref_execute(kernel, dims, path, order, sub, w.factors, ws.out_count,
                               repeats=repeats)
        return st["seconds"]
    _, secs = OB.ref_execute_threads(kernel, dims, path, order, sub, w.factors, ws.out_count,
                                     threads, repeats=repeats)
    return secs


def csf_build_config(P, w, stream, ref_sample=1_000_000):
    """the headline tensor's CSF built on the GPU from its
    COO (shuffled rows in pinned host memory; H2D + radix-sort build, through
    spttn_csf_from_coo) vs the reference's CooTensor::normalize + build_csf
    (oracle/_ref, host) on a bounded sample of the same rows."""
    import torch
    coo, vals = w.csf.to_coo()
    perm = np.random.default_rng(1).permutation(vals.shape[0])
    pc = pinned_copy(np.ascontiguousarray(coo[perm]))
    pv = pinned_copy(np.ascontiguousarray(vals[perm]))
    ts = []
    for it in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dev = P.DeviceCsf.from_coo(w.csf.dims, pc.numpy(), pv.numpy(), stream=stream)
        torch.cuda.synchronize()
        if it:
            ts.append(time.perf_counter() - t0)
        dev.close()
    out = {"device_ms": 1e3 * min(ts), "nnz": int(vals.shape[0]),
           "device_nnz_per_s": vals.shape[0] / min(ts)}
    try:
        sys.path.insert(0, str(ROOT / "tests"))
        import oracle_bindings as OB  # the reference build (test infrastructure)
        if OB.ref_available():
            n = min(ref_sample, vals.shape[0])
            names = list(w.cfg.mode_names)
            t0 = time.perf_counter()
            OB.ref_build_csf(names, list(w.csf.dims), coo[perm][:n], vals[perm][:n], names)
            tr = time.perf_counter() - t0
            out.update({"reference_sample_nnz": int(n), "reference_s": tr,
                        "reference_nnz_per_s": n / tr, "reference_cores": 1})
    except Exception as e:  # noqa: BLE001
        out["reference"] = f"unavailable: {e}"
    return out


def cpu_sample(w, seconds, threads):
    """Every k-th root slice of the tensor, k calibrated on a ~1/64 probe so
    the reference executor needs about `seconds`."""
    n0 = w.csf.level_sizes()[0]
    # two probes (1/64 and 1/16 of the root slices) fit t = fixed + per_nnz * nnz;
    # the fixed part (the reference allocates and zeroes the whole dense
    # output every execute) does not shrink with the sample.
    pts = []
    for frac in (64, 16):
        st = max(1, min(frac, n0 // 4))  # every st-th slice ~ 1/st of the tensor
        probe = w.csf if st == 1 else w.csf.root_sample(st)
        pts.append((probe.nnz, _ref_run(w, probe, threads)))
    (n1, t1), (n2, t2) = pts
    per = max((t2 - t1) / max(1, n2 - n1), 1e-12)
    fixed = max(0.0, t1 - per * n1)
    budget = max(seconds - fixed, 0.25 * seconds)
    stride = max(1, int(np.ceil(per * w.csf.nnz / budget)))
    sub = w.csf if stride == 1 else w.csf.root_sample(stride)
    return sub, stride


def _geomean_ratios(results):
    """Geometric means over the BASELINE configs of this arm's value / e2e
    against the reference on all host threads (same run, same box)."""
    out = {}
    for k in ("value_ratio", "e2e_ratio"):
        xs = [r["vs_reference"][k] for key, r in results.items()
              if key in BASELINE_KEYS and r.get("vs_reference", {}).get(k)]
        if xs:
            out[k] = float(np.exp(np.mean(np.log(xs))))
            out["configs"] = len(xs)
    return out or None


def cpu_reference(w, seconds, threads, repeats=1, sample=None):
    sub, stride = sample if sample is not None else cpu_sample(w, seconds, threads)
    path = ref_args(w)[2]
    secs = _ref_run(w, sub, threads, repeats)
    return {"value": sub.nnz / secs, "unit": "nnz/s", "cores": threads, "kind": "reference",
            "sample": f"every {stride}th root slice of the same tensor: {sub.nnz} nnz "
                      f"({sub.level_sizes()[0]} slices), best of {repeats}, spttn_ref::execute "
                      f"on the pinned nest {path}", "seconds": secs}


BASELINE_KEYS = ["mttkrp3", "ttmc3", "tttp3", "mttkrp4", "ttmc4"]


def dump_workload(key, out_dir):
    """--dump-workload (run in a child process): generate one workload with
    the repo's generator and store its arrays, so the reference arm's own
    process maps only the reference build (oracle/_ref)."""
    from paper_2307_05740_b200.configs import make_workload
    w = make_workload(key)
    arrs = {"dims": np.asarray(w.dims, np.int64), "values": w.csf.values}
    for l, a in enumerate(w.csf.idx):
        arrs[f"idx{l}"] = a
    for l, a in enumerate(w.csf.ptr):
        arrs[f"ptr{l}"] = a
    for f, a in enumerate(w.factors):
        arrs[f"factor{f}"] = a
    np.savez(Path(out_dir) / f"{key}.npz", **arrs)


def load_workload_via_child(key):
    """The workload generated in a child process (dump_workload) and loaded
    here from .npz: no repo native library enters this process."""
    from paper_2307_05740_b200.configs import CONFIGS, Workload
    from paper_2307_05740_b200.tensor import Csf
    with tempfile.TemporaryDirectory(prefix="spttn_ref_in_") as d:
        subprocess.run([sys.executable, str(Path(__file__).resolve()), "--dump-workload", key,
                        "--out", d], check=True)
        z = np.load(Path(d) / f"{key}.npz")
        dims = [int(x) for x in z["dims"]]
        order = len(dims)
        csf = Csf(dims, [z[f"idx{l}"] for l in range(order)],
                  [z[f"ptr{l}"] for l in range(order - 1)], z["values"],
                  list(CONFIGS[key].mode_names))
        nf = len([k for k in z.files if k.startswith("factor")])
        factors = [z[f"factor{f}"] for f in range(nf)]
    return Workload(CONFIGS[key], csf, factors, tuple(dims), csf.nnz)


def run_reference_impl(args, rank, world):
    """--impl reference: the reference CPU executor (oracle/_ref, compiled
    from /root/reference) on all host threads, one plan per thread over
    nnz-balanced root-slice partitions, on a bounded sample of each BASELINE
    config; the headline fields are TTMc-3 (configs[1]), the rest under
    "configs". Inputs come from a child process (load_workload_via_child)."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    per_step = 2 * args.cpu_seconds / max(1, args.steps + args.warmup)
    results = {}
    for key in BASELINE_KEYS:
        w = load_workload_via_child(key)
        sample = cpu_sample(w, per_step, threads)
        vals = []
        res = None
        for step in range(args.warmup + args.steps):
            res = cpu_reference(w, 0, threads, sample=sample)
            if step >= args.warmup:
                vals.append(res["value"])
        results[key] = {"value": statistics.median(vals), "unit": "nnz/s",
                        "ms_per_step": res["seconds"] * 1e3, "sample": res["sample"]}
        print(f"[bench-ref] {key}: {results[key]['value']:.3e} nnz/s", file=sys.stderr, flush=True)
    h = results[HEADLINE]
    v = h["value"]
    line = {"impl": "reference", "metric": METRIC,
            "value": v, "unit": "nnz/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": h["ms_per_step"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": WORKLOAD,
                                            "l2": "n/a (host CPU)",
                                            "parallelism": f"{threads} host threads"},
            "cpu_baseline": {"value": v, "unit": "nnz/s", "cores": threads, "kind": "reference",
                             "sample": h["sample"]},
            "e2e": {"value": v, "unit": "nnz/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "configs": results}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.dump_workload:
        dump_workload(args.dump_workload, args.out)
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference_impl(args, rank, world)
        return
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2307_05740_b200 as P
    from paper_2307_05740_b200.configs import (algorithmic_bytes, algorithmic_flops, gather_bytes,
                                               make_workload)
    keys = ORDER if args.configs == "all" else args.configs.split(",")
    if HEADLINE not in keys:
        keys = [HEADLINE] + keys
    peaks, peak_src = measured_peaks()
    fp64 = fp64_peaks()
    stream = torch.cuda.Stream()
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device="cuda")
    results = {}
    head_clocks = None
    for key in keys:
        strong = args.shard and world > 1
        if strong and key.startswith("mttkrp3_"):
            continue  # non-root outputs: fiber shards would need an output all-reduce
        w = make_workload(key, seed_offset=0 if strong else rank)
        job_nnz = w.csf.nnz if strong else w.csf.nnz * world
        if strong:  # this rank's nnz-balanced fiber range (split root slices are
            # partial rows, summed by distributed.reduce_split_rows after the step)
            from paper_2307_05740_b200 import distributed as D
            f0, f1 = D.partition_fibers(w.csf, world)[rank]
            w.csf = D.shard_csf_fibers(w.csf, f0, f1)
        ev = []
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        with Clocks(local) as clk:
            t0 = time.perf_counter()
            st, plan, dev, tfac = device_time_config(P, w, args.steps, args.warmup, stream,
                                                     flush, ev)
            region = time.perf_counter() - t0
        torch.cuda.synchronize()
        step_ms = st["step_ms"]
        if world > 1:
            t = torch.tensor([step_ms], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            step_ms = float(t.item())
        info = plan.info()
        nnz = w.csf.nnz
        bytes_alg = algorithmic_bytes(w)
        flops_alg = algorithmic_flops(w)
        # single-launch plans (no fix-up): the timed steps themselves are the
        # kernel's launches, so its time is taken over the timed region; plans
        # with a fix-up pass use the stage-split diagnostic pass (an event
        # between the stages would serialise the fix-up inside the timed steps)
        single = info["launches"] == 1
        if single:
            st["main_ms"] = st["step_ms"]
        main_s = st["main_ms"] * 1e-3
        hbm = peaks["hbm_gbs"]
        fp_peak = fp64["dmma_tflops"] if w.cfg.kind in (P.NEST_TTMC3, P.NEST_TTMC4) else \
            fp64["dfma_tflops"]
        t_hbm = bytes_alg / (hbm * 1e9)
        t_fp = flops_alg / (fp_peak * 1e12)
        bound = "tensor" if t_fp >= t_hbm else "hbm"
        if bound == "hbm":
            roof = {"bound": "hbm", "achieved": bytes_alg / main_s / 1e9, "peak": hbm,
                    "unit": "GB/s"}
        else:
            roof = {"bound": "tensor", "achieved": flops_alg / main_s / 1e12, "peak": fp_peak,
                    "unit": "TFLOP/s"}
        roof["frac"] = roof["achieved"] / roof["peak"]
        roof["traffic"] = None
        tr = TRAFFIC.get(key)
        if tr:  # dram read+write bytes of one launch of this config's kernel (ncu --set full)
            roof["traffic"] = tr["traffic_bytes"]
            roof["traffic_kernel"] = tr["kernel"]
            roof["traffic_source"] = tr["source"]
        roof["peak_source"] = (f"{peak_src} MEASURED_PEAKS.json hbm_gbs" if bound == "hbm" else
                               "fp64 " + ("DMMA" if fp_peak == fp64["dmma_tflops"] else "DFMA") +
                               " probe measured by bench.py (MEASURED_PEAKS.json has no fp64)")
        roof["t_roof_us"] = max(t_hbm, t_fp) * 1e6
        roof["north_star_frac"] = max(t_hbm, t_fp) / main_s
        roof["hbm_frac"] = (bytes_alg / main_s / 1e9) / hbm
        roof["fp64_frac"] = (flops_alg / main_s / 1e12) / fp_peak
        roof["bytes_alg"] = bytes_alg
        roof["flops_alg"] = flops_alg
        roof["gather_bytes"] = gather_bytes(w)
        r = {"nnz": nnz, "level_sizes": w.csf.level_sizes(),
             "value": job_nnz / (step_ms * 1e-3), "ms_per_step": step_ms,
             "kernel_ms": st["main_ms"], "kernel_ms_min": st["main_ms_min"],
             "kernel_ms_median": st["main_ms_median"], "kernel_ms_all": st["main_ms_all"],
             "kernel_ms_source": ("timed steps (single launch per step)" if single else
                                  "stage-split diagnostic pass after the timed steps (mean)"),
             "epilogue_ms": st["epi_ms"], "launches_per_step": info["launches"],
             "items": info["items"], "split_slices": info["split_slices"],
             "region_s": region, "roofline": roof}
        if not args.no_parity:
            r["parity"] = parity_check(P, w, plan, stream)
        plan.close()
        dev.close()
        del tfac
        if args.e2e_steps > 0:
            e = e2e_config(P, w, max(1, args.e2e_steps), stream)
            secs = e["seconds"]
            if world > 1:
                t = torch.tensor([secs], device="cuda", dtype=torch.float64)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                secs = float(t.item())
            r["e2e"] = {"value": job_nnz / secs, "unit": "nnz/s",
                        "h2d_bytes_per_step": e["h2d_bytes_per_step"],
                        "d2h_bytes_per_step": e["d2h_bytes_per_step"], "ms_per_step": secs * 1e3,
                        "path": e["path"],
                        "breakdown_ms": e["breakdown_ms"],
                        "als_loop": {"value": job_nnz / e["als_loop"]["seconds"], "unit": "nnz/s",
                                     "ms_per_step": e["als_loop"]["seconds"] * 1e3,
                                     "h2d_bytes_per_step": e["als_loop"]["h2d_bytes_per_step"],
                                     "d2h_bytes_per_step": e["als_loop"]["d2h_bytes_per_step"],
                                     "what": "plan reused: set_factors (pinned H2D) + execute + "
                                             "read_output (D2H) per step"}}
        if rank == 0 and world == 1 and not args.no_cpu:
            r["cpu_baseline"] = cpu_reference(w, args.cpu_seconds, 1, repeats=3)
            # the reference arm's setting (all host threads) on a bounded
            # sample, for per-config ratios (the driver computes the headline)
            threads = os.cpu_count() or 1
            mt = cpu_reference(w, args.cpu_seconds / 2, threads, repeats=3)
            r["reference_threads"] = {"value": mt["value"], "cores": threads,
                                      "sample": mt["sample"]}
            r["vs_reference"] = {"value_ratio": r["value"] / mt["value"],
                                 "e2e_ratio": (r["e2e"]["value"] / mt["value"]) if "e2e" in r
                                 else None}
            if key == HEADLINE:
                r["csf_build"] = csf_build_config(P, w, stream)
        if key == HEADLINE:
            head_clocks = clk.summary()
        else:
            r["clocks"] = clk.summary()
        results[key] = r
        print(f"[bench] {key}: {r['value']:.3e} nnz/s kernel {st['main_ms']:.3f} ms "
              f"roof {roof['frac']:.3f} ({bound})", file=sys.stderr, flush=True)

    h = results[HEADLINE]
    line = {
        "metric": METRIC,
        "value": h["value"], "unit": "nnz/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": h["ms_per_step"], "higher_is_better": True,
        "scaling": "strong" if (args.shard and world > 1) else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD,
                   "l2": "256 MB L2 flush write between timed steps",
                   "parallelism": (f"fiber shards x{world} of one tensor"
                                   if (args.shard and world > 1) else
                                   f"weak x{world} (independent tensor per rank)")},
        "roofline": h["roofline"], "gpu_launches": h["launches_per_step"] * args.steps,
        "clocks": head_clocks, "e2e": h.get("e2e"), "cpu_baseline": h.get("cpu_baseline"),
        "fp64_peaks": fp64,
        "parity": {k: v.get("parity", {}).get("ok") for k, v in results.items()},
        "vs_reference_geomean": _geomean_ratios(results),
        "configs": {k: v for k, v in results.items()},
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
