"""GPU parity suite: the sm_100a kernels (through the C-ABI) against the oracle.

Bar (BASELINE.json north star): sparsity / index structure bit-exact, fp64
values within 1e-10 x sum|contributions| per output entry; exact zeros stay
exact; repeated execution is bit-identical (proj/tests/test_executor.cpp:
203-220).
"""
import json
import os
from pathlib import Path

import numpy as np
import pytest

import oracle_bindings as OB
from parity import assert_parity, oracle_with_norm

pytestmark = pytest.mark.gpu

GOLD = Path(__file__).resolve().parent / "golden"
MANIFEST = json.loads((GOLD / "manifest.json").read_text())
CASES = [m for m in MANIFEST if "kernel" in m]


@pytest.fixture(scope="module")
def E():
    import torch
    assert torch.cuda.is_available(), "GPU suite needs a CUDA device"
    import paper_2307_05740_b200 as P
    return P


def load_case(m):
    from paper_2307_05740_b200.tensor import Csf
    z = np.load(GOLD / f"{m['name']}.npz")
    d = len(m["sparse_dims"])
    csf = Csf(list(m["sparse_dims"]), [z[f"idx{l}"] for l in range(d)],
              [z[f"ptr{l}"] for l in range(d - 1)], z["values"])
    nf = len([k for k in z.files if k.startswith("factor")])
    return csf, [z[f"factor{f}"] for f in range(nf)], z


def run(E, kind, csf, factors, ranks, flags=0):
    dev = E.DeviceCsf(csf)
    plan = E.Plan(kind, dev, factors, ranks=ranks, flags=flags)
    plan.execute()
    out = plan.read_output()
    return out, plan, dev


@pytest.mark.parametrize("m", CASES, ids=[m["name"] for m in CASES])
def test_golden_reference_outputs(E, m):
    csf, factors, z = load_case(m)
    out, plan, _ = run(E, m["kind"], csf, factors, m["ranks"])
    _, norm = oracle_with_norm(m["kind"], csf, factors, m["ranks"])
    assert_parity(out, z["fused"], norm, m["name"])
    # second run on the same plan: bit-identical (atomic non-root kernels:
    # within tolerance — arrival order of the fp64 atomics varies)
    plan.execute()
    if m["kind"] in (6, 7):
        assert_parity(plan.read_output(), z["fused"], norm, m["name"] + " rerun")
    else:
        assert np.array_equal(plan.read_output(), out)


@pytest.mark.parametrize("m", [m for m in CASES if m["sparse_out"]],
                         ids=[m["name"] for m in CASES if m["sparse_out"]])
def test_golden_completion_residual(E, m):
    csf, factors, z = load_case(m)
    out, _, _ = run(E, m["kind"], csf, factors, m["ranks"], flags=E.FLAG_RESIDUAL)
    _, norm = oracle_with_norm(m["kind"], csf, factors, m["ranks"], residual=True)
    assert_parity(out, z["residual"], norm, m["name"] + " residual")


@pytest.mark.parametrize("chunk", ["1", "2", "3", "7", "64"])
@pytest.mark.parametrize("name", ["mttkrp3_r32", "ttmc3_r16", "tttp3_r64", "mttkrp4_r32",
                                  "ttmc4_r8"])
def test_partition_independence(E, name, chunk, monkeypatch):
    """Tiny work items force split fibers, split slices and many HEAD/TAIL
    partials; results must stay within tolerance and be deterministic."""
    m = [c for c in CASES if c["name"] == name][0]
    csf, factors, z = load_case(m)
    monkeypatch.setenv("SPTTN_CHUNK", chunk)
    monkeypatch.setenv("SPTTN_SEG_LEN", "1" if chunk in ("1", "2") else "3")
    if name == "mttkrp3_r32":  # the item / fix-up kernel (the default has no items)
        monkeypatch.setenv("SPTTN_MTTKRP_MODE", "2")
    out, plan, _ = run(E, m["kind"], csf, factors, m["ranks"])
    _, norm = oracle_with_norm(m["kind"], csf, factors, m["ranks"])
    assert_parity(out, z["fused"], norm, f"{name} chunk={chunk}")
    if m["kind"] != 3 and chunk == "1":
        assert plan.info()["split_slices"] > 0


VARIANTS = [("SPTTN_MTTKRP_MODE", m, ["mttkrp3_small", "mttkrp3_r32", "mttkrp4_small", "mttkrp4_r32"])
            for m in ("0", "2", "3", "4")] + \
    [("SPTTN_TTTP_BATCH", m, ["tttp3_small", "tttp3_r64"]) for m in ("2", "4", "8")] + \
    [("SPTTN_TTMC4_MODE", m, ["ttmc4_small", "ttmc4_r8"]) for m in ("3", "4")] + \
    [("SPTTN_NONROOT_MODE", m, ["mttkrp3j_small", "mttkrp3j_r32", "mttkrp3k_small", "mttkrp3k_r32"])
     for m in ("0", "4", "5")]


@pytest.mark.parametrize("env,mode,names", VARIANTS, ids=[f"{v[0]}={v[1]}" for v in VARIANTS])
def test_kernel_variants_agree(E, env, mode, names, monkeypatch):
    """Every kernel variant kept for A/B measurement stays within tolerance,
    on the golden fixtures and on BASELINE-shaped inputs."""
    from paper_2307_05740_b200.configs import make_workload
    monkeypatch.setenv(env, mode)
    for name in names:
        m = [c for c in CASES if c["name"] == name][0]
        csf, factors, z = load_case(m)
        out, _, _ = run(E, m["kind"], csf, factors, m["ranks"])
        _, norm = oracle_with_norm(m["kind"], csf, factors, m["ranks"])
        assert_parity(out, z["fused"], norm, f"{name} {env}={mode}")
    key = {"SPTTN_MTTKRP_MODE": "mttkrp4", "SPTTN_TTTP_BATCH": "tttp3",
           "SPTTN_TTMC4_MODE": "ttmc4", "SPTTN_NONROOT_MODE": "mttkrp3_k"}[env]
    w = make_workload(key, scale=2e-3)
    c = w.cfg
    out, _, _ = run(E, c.kind, w.csf, w.factors, c.ranks, E.FLAG_RESIDUAL if c.residual else 0)
    want, norm = oracle_with_norm(c.kind, w.csf, w.factors, c.ranks, residual=c.residual)
    assert_parity(out, want, norm, f"{key} {env}={mode}")


@pytest.mark.parametrize("key", ["mttkrp3", "ttmc3", "tttp3", "mttkrp4", "ttmc4"])
def test_baseline_shaped_reduced_scale(E, key):
    from paper_2307_05740_b200.configs import make_workload
    w = make_workload(key, scale=1e-3)
    c = w.cfg
    flags = E.FLAG_RESIDUAL if c.residual else 0
    out, _, _ = run(E, c.kind, w.csf, w.factors, c.ranks, flags)
    want, norm = oracle_with_norm(c.kind, w.csf, w.factors, c.ranks, residual=c.residual)
    assert_parity(out, want, norm, key)


def _skewed_csf(order, dims, nnz_in_one_fiber, extra, seed):
    """One giant fiber (all under root 0 / fiber 0) plus scattered extras."""
    from paper_2307_05740_b200.tensor import Csf
    rng = np.random.default_rng(seed)
    big = np.zeros((nnz_in_one_fiber, order), np.int64)
    big[:, order - 1] = np.arange(nnz_in_one_fiber) % dims[order - 1]
    if order == 4:
        big[:, 2] = np.arange(nnz_in_one_fiber) // dims[3] % dims[2]
    rest = rng.integers(0, dims, size=(extra, order))
    coords = np.concatenate([big, rest])
    vals = rng.uniform(-1, 1, coords.shape[0])
    return Csf.from_coo(list(dims), coords, vals)


@pytest.mark.parametrize("kind,ranks,order", [(1, (32, 0, 0), 3), (2, (16, 16, 0), 3),
                                              (3, (64, 0, 0), 3), (4, (32, 0, 0), 4),
                                              (5, (8, 8, 8), 4)])
def test_extreme_skew_long_fiber(E, kind, ranks, order):
    """A single fiber with ~20k leaves (MTTKRP-4's largest fiber holds 2e5;
    SURVEY.md §0.8) must be split across work items deterministically."""
    dims = (50, 40, 300, 70) if order == 4 else (50, 40, 20000)
    csf = _skewed_csf(order, dims[:order], 20000, 3000, 5)
    rng = np.random.default_rng(1)
    R, S, T = ranks
    if kind in (1, 4):
        fs = [rng.standard_normal((dims[l], R)) for l in range(1, order)]
    elif kind == 2:
        fs = [rng.standard_normal((dims[1], R)), rng.standard_normal((dims[2], S))]
    elif kind == 3:
        fs = [rng.standard_normal((dims[l], R)) for l in range(3)]
    else:
        fs = [rng.standard_normal((dims[1], R)), rng.standard_normal((dims[2], S)),
              rng.standard_normal((dims[3], T))]
    out, plan, _ = run(E, kind, csf, fs, ranks)
    want, norm = oracle_with_norm(kind, csf, fs, ranks)
    assert_parity(out, want, norm, f"skew kind={kind}")
    plan.execute()
    assert np.array_equal(plan.read_output(), out)


@pytest.mark.parametrize("kind,ranks,order", [(1, (32, 0, 0), 3), (2, (16, 16, 0), 3),
                                              (3, (64, 0, 0), 3), (4, (32, 0, 0), 4),
                                              (5, (8, 8, 8), 4)])
def test_empty_and_single_entry(E, kind, ranks, order):
    from paper_2307_05740_b200.tensor import Csf
    dims = [5, 4, 6, 3][:order]
    R, S, T = ranks
    rng = np.random.default_rng(0)
    rows = {1: [1, 2], 4: [1, 2, 3], 2: [1, 2], 3: [0, 1, 2], 5: [1, 2, 3]}[kind]
    cols = {1: [R, R], 4: [R, R, R], 2: [R, S], 3: [R, R, R], 5: [R, S, T]}[kind]
    fs = [rng.standard_normal((dims[r], c)) for r, c in zip(rows, cols)]
    empty = Csf.from_coo(dims, np.zeros((0, order), np.int64), np.zeros(0))
    out, _, _ = run(E, kind, empty, fs, ranks)
    assert np.all(out == 0.0)
    one = Csf.from_coo(dims, np.array([[d - 1 for d in dims]]), np.array([0.75]))
    out, _, _ = run(E, kind, one, fs, ranks)
    want, norm = oracle_with_norm(kind, one, fs, ranks)
    assert_parity(out, want, norm, "single entry")


@pytest.mark.parametrize("m", [CASES[1], CASES[3], CASES[7], CASES[9]],
                         ids=[CASES[i]["name"] for i in (1, 3, 7, 9)])
def test_zero_factor_gives_exact_zero(E, m):
    """proj/tests/test_executor.cpp:122-132."""
    csf, factors, _ = load_case(m)
    factors = [np.zeros_like(factors[0])] + factors[1:]
    out, _, _ = run(E, m["kind"], csf, factors, m["ranks"])
    assert np.all(out == 0.0)


def test_errors_map_to_reference_exception_types(E):
    """Shape errors -> invalid_argument, unsupported rank -> unsupported_order_error,
    malformed CSF -> invalid_argument (executor.cpp:112-140, :176-178)."""
    m = [c for c in CASES if c["name"] == "ttmc3_r16"][0]
    csf, factors, _ = load_case(m)
    dev = E.DeviceCsf(csf)
    with pytest.raises(ValueError):
        E.Plan(E.NEST_TTMC3, dev, [factors[0][:, :8], factors[1]], ranks=(16, 16))
    with pytest.raises(ValueError):
        E.Plan(E.NEST_MTTKRP4, dev, factors, ranks=(16, 0))
    big = [np.zeros((csf.dims[1], 17)), np.zeros((csf.dims[2], 16))]
    with pytest.raises(E.UnsupportedOrderError):
        E.Plan(E.NEST_TTMC3, dev, big, ranks=(17, 16))
    bad = csf.with_values(csf.values)
    bad.idx = [a.copy() for a in csf.idx]
    bad.idx[2][0] = csf.dims[2] + 5
    with pytest.raises(ValueError):
        E.DeviceCsf(bad)


def test_device_factors_and_set_factors(E):
    """Factors resident on the device (FACTORS_ON_DEVICE) and refreshed
    between executions (ALS-style), against the oracle each time."""
    import torch
    m = [c for c in CASES if c["name"] == "mttkrp3_r32"][0]
    csf, factors, _ = load_case(m)
    dev = E.DeviceCsf(csf)
    tf = [torch.from_numpy(np.ascontiguousarray(f)).cuda() for f in factors]
    plan = E.Plan(E.NEST_MTTKRP3, dev, [t.data_ptr() for t in tf], ranks=(32,),
                  on_device=True, factor_sizes=[t.numel() for t in tf])
    plan.execute()
    out = plan.read_output()
    want, norm = oracle_with_norm(1, csf, factors, (32, 0, 0))
    assert_parity(out, want, norm, "device factors")
    tf[0].mul_(-2.0)
    plan.execute()
    out2 = plan.read_output()
    want2, norm2 = oracle_with_norm(1, csf, [factors[0] * -2.0, factors[1]], (32, 0, 0))
    assert_parity(out2, want2, norm2, "updated device factors")
    hplan = E.Plan(E.NEST_MTTKRP3, dev, factors, ranks=(32,))
    hplan.set_factors([factors[0] * -2.0, factors[1]])
    hplan.execute()
    assert_parity(hplan.read_output(), want2, norm2, "set_factors")


@pytest.mark.parametrize("name", ["mttkrp3_r32", "ttmc3_r16", "tttp3_r64", "mttkrp4_r32",
                                  "ttmc4_r8"])
def test_device_factors_at_unaligned_addresses(E, name):
    """Device-resident factors that start 8 bytes past a 32-byte boundary (a
    caller's tensor view) take the scalar-load paths (no 128/256-bit
    gathers); results must not change."""
    import torch
    m = [c for c in CASES if c["name"] == name][0]
    csf, factors, _ = load_case(m)
    dev = E.DeviceCsf(csf)
    views, keep = [], []
    for f in factors:
        flat = np.ascontiguousarray(f).ravel()
        buf = torch.zeros(flat.size + 4, dtype=torch.float64, device="cuda")
        buf[1:1 + flat.size] = torch.from_numpy(flat).cuda()
        keep.append(buf)
        views.append(buf[1:1 + flat.size])
    assert all(v.data_ptr() % 32 == 8 for v in views)
    plan = E.Plan(m["kind"], dev, [v.data_ptr() for v in views], ranks=m["ranks"],
                  on_device=True, factor_sizes=[v.numel() for v in views])
    plan.execute()
    out = plan.read_output()
    want, norm = oracle_with_norm(m["kind"], csf, factors, m["ranks"])
    assert_parity(out, want, norm, name + " unaligned device factors")


def test_unit_values_tttp_equals_residual_flow(E):
    """rho = T - S(unit values): the residual flag equals the oracle flow the
    survey prescribes."""
    m = [c for c in CASES if c["name"] == "tttp3_r64"][0]
    csf, factors, z = load_case(m)
    unit = csf.with_values(np.ones_like(csf.values))
    s_unit, _, _ = run(E, 3, unit, factors, m["ranks"])
    rho, _, _ = run(E, 3, csf, factors, m["ranks"], flags=E.FLAG_RESIDUAL)
    _, norm = oracle_with_norm(3, csf, factors, m["ranks"], residual=True)
    assert_parity(rho, csf.values - s_unit, norm, "residual vs T - S(1)")


@pytest.mark.parametrize("kind", [6, 7])
@pytest.mark.parametrize("shape", ["baseline", "skew", "empty"])
def test_nonroot_mttkrp(E, kind, shape):
    """MTTKRP-3 for the non-root modes (output on CSF level 1 / 2, fp64
    atomics): BASELINE-shaped (mttkrp3 config, reduced), one 20k-leaf fiber
    (every atomic of a row contended), and an empty tensor (zero output)."""
    from paper_2307_05740_b200.configs import make_workload
    from paper_2307_05740_b200.tensor import Csf
    rng = np.random.default_rng(kind)
    R = 32
    if shape == "baseline":
        csf = make_workload("mttkrp3", scale=5e-2).csf
    elif shape == "skew":
        csf = _skewed_csf(3, (50, 40, 20000), 20000, 3000, 5)
    else:
        csf = Csf.from_coo([9, 7, 5], np.zeros((0, 3), np.int64), np.zeros(0))
    dims = csf.dims
    fs = [rng.standard_normal((dims[0], R)), rng.standard_normal((dims[2 if kind == 6 else 1], R))]
    out, plan, _ = run(E, kind, csf, fs, (R, 0, 0))
    want, norm = oracle_with_norm(kind, csf, fs, (R, 0, 0))
    assert out.shape == want.shape
    assert_parity(out, want, norm, f"nonroot kind={kind} {shape}")
    if shape == "empty":
        assert not np.any(out)
    if shape == "baseline":  # the re-ordered root kernel: owner-computes, reproducible
        assert plan.info()["variant"] == 5
        plan.execute()
        assert np.array_equal(plan.read_output(), out)


@pytest.mark.parametrize("kind", [6, 7])
@pytest.mark.parametrize("mode", ["0", "4", "5"])
def test_nonroot_variants_with_absent_rows(E, kind, mode, monkeypatch):
    """Every non-root variant on a tensor with absent output rows (mode-j /
    mode-k indices that never occur): they must come out exactly zero — the
    re-ordered variant (5) writes them from its absent-root-row list, the
    atomic ones from the zeroed output."""
    from paper_2307_05740_b200.tensor import Csf
    monkeypatch.setenv("SPTTN_NONROOT_MODE", mode)
    rng = np.random.default_rng(40 + kind)
    dims = (300, 400, 500)
    n = 60000
    co = np.stack([rng.integers(0, dims[0], n), rng.integers(0, dims[1] - 50, n),
                   rng.integers(0, dims[2] - 60, n)], 1).astype(np.int64)
    co = np.unique(co, axis=0)
    csf = Csf.from_coo(list(dims), co, rng.uniform(-1, 1, len(co)))
    R = 32
    fs = [rng.standard_normal((dims[0], R)), rng.standard_normal((dims[2 if kind == 6 else 1], R))]
    out, plan, _ = run(E, kind, csf, fs, (R, 0, 0))
    want, norm = oracle_with_norm(kind, csf, fs, (R, 0, 0))
    assert_parity(out, want, norm, f"nonroot kind={kind} mode={mode}")
    assert plan.info()["variant"] == int(mode)
    rows = out.reshape(-1, R)
    zrows = np.abs(np.asarray(norm).reshape(-1, R)).sum(1) == 0
    assert zrows.sum() >= 50 and not np.any(rows[zrows])


@pytest.mark.parametrize("order", [3, 4])
def test_device_csf_from_coo_matches_build_csf(E, order):
    """spttn_csf_from_coo (GPU normalize + build_csf) == the host restatement
    of the reference's CooTensor::normalize + build_csf (tensor.cpp:24-94),
    array for array: shuffled input rows and duplicate pairs (summed)."""
    from paper_2307_05740_b200.tensor import Csf
    rng = np.random.default_rng(order)
    dims = [37, 23, 41, 19][:order]
    n = 3000
    coords = np.stack([rng.integers(0, d, n) for d in dims], axis=1)
    coords = np.concatenate([coords, coords[:200]])  # duplicate pairs
    vals = rng.uniform(-1, 1, coords.shape[0])
    perm = rng.permutation(coords.shape[0])
    coords, vals = coords[perm], vals[perm]
    want = Csf.from_coo(dims, coords, vals)
    dev = E.DeviceCsf.from_coo(dims, coords, vals)
    got = dev.download()
    assert got.dims == want.dims
    for a, b in zip(got.idx, want.idx):
        assert np.array_equal(a, b)
    for a, b in zip(got.ptr, want.ptr):
        assert np.array_equal(a, b)
    assert np.array_equal(got.values, want.values)


def test_device_csf_from_coo_baseline_tensor_and_plan(E):
    """The TTMc-3 BASELINE tensor (Zipf, 1e7 nnz) rebuilt on the GPU from its
    shuffled COO is the same CSF, and a plan on it gives bit-identical output."""
    from paper_2307_05740_b200.configs import make_workload
    w = make_workload("ttmc3")
    coo, vals = w.csf.to_coo()
    perm = np.random.default_rng(5).permutation(vals.shape[0])
    dev = E.DeviceCsf.from_coo(w.csf.dims, coo[perm], vals[perm])
    got = dev.download()
    for a, b in zip(got.idx + got.ptr, w.csf.idx + w.csf.ptr):
        assert np.array_equal(a, b)
    assert np.array_equal(got.values, w.csf.values)
    c = w.cfg
    p1 = E.Plan(c.kind, dev, w.factors, ranks=c.ranks)
    p1.execute()
    host_dev = E.DeviceCsf(w.csf)
    p2 = E.Plan(c.kind, host_dev, w.factors, ranks=c.ranks)
    p2.execute()
    assert np.array_equal(p1.read_output(), p2.read_output())


def test_device_csf_from_coo_errors_and_empty(E):
    with pytest.raises(ValueError):  # SPTTN_EINVAL
        E.DeviceCsf.from_coo([4, 4, 4], np.array([[0, 1, 4]]), np.array([1.0]))
    dev = E.DeviceCsf.from_coo([4, 5, 6], np.zeros((0, 3), np.int64), np.zeros(0))
    got = dev.download()
    assert got.level_sizes() == [0, 0, 0]
    assert [p.tolist() for p in got.ptr] == [[0], [0]]


def test_device_csf_permute_reroots(E):
    """spttn_csf_permute: the (j, i, k) CSF of a tensor equals the host build
    of its COO in that mode order, and the re-rooted MTTKRP-3 kernel then gives
    the mode-j product (owner computes, no atomics)."""
    from paper_2307_05740_b200.configs import make_workload
    from paper_2307_05740_b200.tensor import Csf
    w = make_workload("mttkrp3", scale=2e-2)
    dev = E.DeviceCsf(w.csf)
    rr = dev.permute([1, 0, 2])
    coo, vals = w.csf.to_coo()
    want = Csf.from_coo([w.csf.dims[1], w.csf.dims[0], w.csf.dims[2]], coo[:, [1, 0, 2]], vals)
    got = rr.download()
    for a, b in zip(got.idx + got.ptr, want.idx + want.ptr):
        assert np.array_equal(a, b)
    assert np.array_equal(got.values, want.values)
    rng = np.random.default_rng(3)
    R = 32
    A = rng.standard_normal((w.csf.dims[0], R))
    Cf = rng.standard_normal((w.csf.dims[2], R))
    plan = E.Plan(E.NEST_MTTKRP3, rr, [A, Cf], ranks=(R, 0, 0))  # level-1 factor = A
    plan.execute()
    out = plan.read_output()
    ref, norm = oracle_with_norm(6, w.csf, [A, Cf], (R, 0, 0))
    assert_parity(out, ref, norm, "re-rooted mode-j MTTKRP")


def test_device_csf_permute_edge_cases(E):
    """Re-rooting an empty tensor, a 4-D tensor in every rotation, and the
    order-1 / order-2 device builds."""
    from paper_2307_05740_b200.tensor import Csf
    empty = E.DeviceCsf.from_coo([4, 5, 6], np.zeros((0, 3), np.int64), np.zeros(0))
    assert empty.permute([2, 0, 1]).download().level_sizes() == [0, 0, 0]
    rng = np.random.default_rng(11)
    dims = [7, 6, 5, 8]
    coords = np.unique(np.stack([rng.integers(0, d, 400) for d in dims], axis=1), axis=0)
    vals = rng.uniform(-1, 1, coords.shape[0])
    dev = E.DeviceCsf.from_coo(dims, coords, vals)
    for order in ([1, 0, 2, 3], [3, 2, 1, 0], [2, 3, 0, 1]):
        got = dev.permute(order).download()
        want = Csf.from_coo([dims[o] for o in order], coords[:, order], vals)
        for a, b in zip(got.idx + got.ptr, want.idx + want.ptr):
            assert np.array_equal(a, b)
        assert np.array_equal(got.values, want.values)
    for d in (1, 2):
        c = np.unique(rng.integers(0, 9, (30, d)), axis=0)
        v = rng.uniform(-1, 1, c.shape[0])
        got = E.DeviceCsf.from_coo([9] * d, c, v).download()
        want = Csf.from_coo([9] * d, c, v)
        for a, b in zip(got.idx + got.ptr, want.idx + want.ptr):
            assert np.array_equal(a, b)
        assert np.array_equal(got.values, want.values)


@pytest.mark.parametrize("R", [16, 32])
@pytest.mark.parametrize("force,skew", [(False, False), (True, True)])
def test_mttkrp3_shared_factor_kernel(E, R, force, skew, monkeypatch):
    """k_mttkrp3_smf (factor column blocks resident in shared memory, one
    launch, no fix-up): slice-aligned CTA ranges, warp-order piece merge,
    absent root rows zeroed in-kernel. `force` keeps it on a tensor with one
    heavy slice that the plan would otherwise route to the item kernels."""
    from paper_2307_05740_b200.tensor import Csf
    if force:
        monkeypatch.setenv("SPTTN_SMF_FORCE", "1")
    rng = np.random.default_rng(R)
    dims = (700, 300, 500)
    nnz = 60000
    coords = np.stack([rng.integers(0, d, nnz) for d in dims], axis=1)
    coords[:, 0] = coords[:, 0] // 2 * 2  # odd root rows absent
    if skew:
        coords[: nnz // 3, 0] = 4
    vals = rng.uniform(-1, 1, nnz)
    csf = Csf.from_coo(list(dims), coords, vals)
    fs = [rng.standard_normal((dims[1], R)), rng.standard_normal((dims[2], R))]
    out, plan, _ = run(E, 1, csf, fs, (R, 0, 0))
    assert plan.info()["launches"] == 1, plan.info()
    want, norm = oracle_with_norm(1, csf, fs, (R, 0, 0))
    assert_parity(out, want, norm, f"smf R={R} force={force}")
    assert np.all(out.reshape(dims[0], R)[1::2] == 0.0)
    plan.execute()
    assert np.array_equal(plan.read_output(), out)


@pytest.mark.parametrize("piece", ["1", "7", "64", "1000"])
def test_tttp_slice_pieces_skew_and_residual(E, piece, monkeypatch):
    """TTTP slice pieces (A[i] once per piece): a root-skewed pattern (one
    slice with a quarter of the leaves, many 1-leaf slices) at several piece
    sizes, with and without the residual flag, against the oracle;
    re-execution bit-identical."""
    from paper_2307_05740_b200.tensor import Csf
    monkeypatch.setenv("SPTTN_TTTP_PIECE", piece)
    rng = np.random.default_rng(7)
    dims = (3000, 200, 300)
    nnz = 50000
    coords = np.stack([rng.integers(0, d, nnz) for d in dims], axis=1)
    coords[: nnz // 4, 0] = 17  # one hot root slice
    vals = rng.uniform(-1, 1, nnz)
    csf = Csf.from_coo(list(dims), coords, vals)
    R = 64
    fs = [rng.standard_normal((d, R)) * 0.35 for d in dims]
    for flags, residual in ((0, False), (E.FLAG_RESIDUAL, True)):
        out, plan, _ = run(E, 3, csf, fs, (R, 0, 0), flags)
        want, norm = oracle_with_norm(3, csf, fs, (R, 0, 0), residual=residual)
        assert_parity(out, want, norm, f"tttp pieces P={piece} residual={residual}")
        plan.execute()
        assert np.array_equal(plan.read_output(), out)


def test_set_factors_rejects_less_aligned_device_factors(E):
    """Kernels are chosen for the factor alignment seen at plan creation
    (256/128-bit gathers, 16-byte cp.async of factor columns); refreshing
    device factors with a less aligned pointer is an EINVAL, not a fault."""
    import torch
    m = [c for c in CASES if c["name"] == "mttkrp3_r32"][0]
    csf, factors, _ = load_case(m)
    dev = E.DeviceCsf(csf)
    tf = [torch.from_numpy(np.ascontiguousarray(f)).cuda() for f in factors]
    plan = E.Plan(E.NEST_MTTKRP3, dev, [t.data_ptr() for t in tf], ranks=(32,),
                  on_device=True, factor_sizes=[t.numel() for t in tf])
    buf = torch.zeros(tf[0].numel() + 4, dtype=torch.float64, device="cuda")
    view = buf[1:1 + tf[0].numel()]
    with pytest.raises(ValueError):
        plan.set_factors([view.data_ptr(), tf[1].data_ptr()], on_device=True)
    plan.set_factors([t.data_ptr() for t in tf], on_device=True)
    plan.execute()
    want, norm = oracle_with_norm(1, csf, factors, (32, 0, 0))
    assert_parity(plan.read_output(), want, norm, "after rejected refresh")


@pytest.mark.parametrize("key", ["mttkrp3", "ttmc3", "tttp3", "mttkrp4", "ttmc4"])
def test_async_value_upload(E, key):
    """spttn_csf_create_async: values arrive on a side stream while the plan
    is built; every consumer orders itself after them (plan packing, execute,
    download) — same results as the synchronous upload, bit for bit."""
    import torch
    from paper_2307_05740_b200.configs import make_workload
    w = make_workload(key, scale=2e-3)
    c = w.cfg
    flags = E.FLAG_RESIDUAL if c.residual else 0
    s = torch.cuda.Stream()
    dev = E.DeviceCsf(w.csf, stream=s, async_values=True)
    plan = E.Plan(c.kind, dev, w.factors, ranks=c.ranks, flags=flags, stream=s)
    plan.execute(s)
    got = plan.read_output(s)
    back = dev.download(s)
    assert np.array_equal(back.values, w.csf.values)
    ref, _, _ = run(E, c.kind, w.csf, w.factors, c.ranks, flags)
    assert np.array_equal(got, ref)


def test_csf_view_rebased(E):
    """A root range passed as a view (ptr[l][0] != 0) downloads as the same
    tree as an explicitly rebased copy."""
    from paper_2307_05740_b200 import distributed as D
    from paper_2307_05740_b200.configs import make_workload
    w = make_workload("mttkrp4", scale=1e-3)
    n0 = w.csf.level_sizes()[0]
    r0, r1 = n0 // 3, 2 * n0 // 3
    dev = E.DeviceCsf.from_root_range(w.csf, r0, r1)
    got = dev.download()
    ref = D.shard_csf(w.csf, r0, r1)
    for a, b in zip(got.idx + got.ptr, ref.idx + ref.ptr):
        assert np.array_equal(a, b)
    assert np.array_equal(got.values, ref.values)


@pytest.mark.parametrize("m", CASES, ids=[m["name"] for m in CASES])
def test_device_unfactorized_equals_reference_golden(E, m):
    """spttn_unfactorized (the device execute_unfactorized) against the
    golden arrays the reference's own execute_unfactorized produced
    (tests/golden/make_golden.py): bit for bit."""
    csf, factors, z = load_case(m)
    dev = E.DeviceCsf(csf)
    got = E.unfactorized(m["kernel"], m["dims"], dev, factors)
    assert np.array_equal(got, z["unfactorized"]), np.abs(got - z["unfactorized"]).max()


@pytest.mark.parametrize("key", ["ttmc3", "ttmc4", "mttkrp4"])
def test_item_clock_diagnostics(E, key, monkeypatch):
    """SPTTN_ITEM_CLOCKS=1 (tuning aid): the packed TTMc-3 / TTMc-4 / MTTKRP-4
    kernels' diagnostics instantiations record one {start, end, SM, groups,
    steps, flushes} per work item, with results identical to the plain
    kernel; a plan without the records reports EINVAL."""
    from paper_2307_05740_b200.configs import make_workload
    w = make_workload(key, scale=2e-3)
    monkeypatch.setenv("SPTTN_ITEM_CLOCKS", "1")
    monkeypatch.setenv("SPTTN_GCHUNK", "4")
    out, plan, dev = run(E, w.cfg.kind, w.csf, w.factors, w.cfg.ranks)
    k = plan.item_clocks()
    assert k.shape == (plan.info()["items"], 6) and k.shape[0] > 1
    assert np.all(k[:, 1] >= k[:, 0]) and np.all(k[:, 0] > 0)
    assert np.all((k[:, 2] >= 0) & (k[:, 2] < 1024))
    assert np.all(k[:, 3] >= 1) and np.all(k[:, 4] >= k[:, 3]) and np.all(k[:, 5] >= 1)
    monkeypatch.delenv("SPTTN_ITEM_CLOCKS")
    plain = E.Plan(w.cfg.kind, dev, w.factors, ranks=w.cfg.ranks)
    plain.execute()
    assert np.array_equal(plain.read_output(), out)  # the records do not change results
    with pytest.raises(Exception):
        plain.item_clocks()
