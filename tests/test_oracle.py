"""CPU suite: the oracle is pinned before it is trusted.

* the plain-C restatement (oracle/spttn_oracle.c) reproduces the reference's
  own outputs bit-for-bit on the committed golden fixtures (generated from the
  compiled reference by tests/golden/make_golden.py);
* the host generators reproduce the reference's gen_random / gen_dense /
  build_csf (the inputs of every reference test) bit-for-bit;
* the flop formulas used for the roofline equal the reference's
  multiply-add counters.
"""
import json
from pathlib import Path

import numpy as np
import pytest

import oracle_bindings as OB
from paper_2307_05740_b200.tensor import Csf, gen_dense, stable_hash

GOLD = Path(__file__).resolve().parent / "golden"
MANIFEST = json.loads((GOLD / "manifest.json").read_text())
CASES = [m for m in MANIFEST if "kernel" in m]


def load_case(m):
    z = np.load(GOLD / f"{m['name']}.npz")
    d = len(m["sparse_dims"])
    idx = [z[f"idx{l}"] for l in range(d)]
    ptr = [z[f"ptr{l}"] for l in range(d - 1)]
    csf = Csf(list(m["sparse_dims"]), idx, ptr, z["values"])
    nf = len([k for k in z.files if k.startswith("factor")])
    factors = [z[f"factor{f}"] for f in range(nf)]
    return csf, factors, z


@pytest.mark.parametrize("m", CASES, ids=[m["name"] for m in CASES])
def test_c_oracle_bit_identical_to_reference_golden(m):
    csf, factors, z = load_case(m)
    got = OB.oracle_nest(m["kind"], csf, factors, m["ranks"])
    assert np.array_equal(got, z["fused"]), np.abs(got - z["fused"]).max()


@pytest.mark.parametrize("m", [m for m in CASES if m["sparse_out"]],
                         ids=[m["name"] for m in CASES if m["sparse_out"]])
def test_c_oracle_residual_matches_reference_unit_value_flow(m):
    csf, factors, z = load_case(m)
    got = OB.oracle_nest(m["kind"], csf, factors, m["ranks"], residual=True)
    assert np.array_equal(got, z["residual"])


@pytest.mark.parametrize("m", CASES, ids=[m["name"] for m in CASES])
def test_generators_reproduce_reference_inputs(m):
    """gen_random + build_csf and gen_dense(7 ^ stable_hash(name))
    (proj/tests/fixtures.hpp:65-95) rebuilt without the reference."""
    csf, factors, z = load_case(m)
    mine = Csf.gen_random(m["sparse_dims"], m["density"], m["seed"])
    assert mine.level_sizes() == m["level_sizes"]
    for l in range(csf.order):
        assert np.array_equal(mine.idx[l], csf.idx[l])
    for l in range(csf.order - 1):
        assert np.array_equal(mine.ptr[l], csf.ptr[l])
    assert np.array_equal(mine.values, csf.values)
    lhs = m["kernel"].split("->")[0]
    names = [t.split("[")[0] for t in lhs.split("*")][1:]
    for name, f in zip(names, factors):
        assert np.array_equal(gen_dense(f.size, 7 ^ stable_hash(name)), f.ravel())


def test_coo3_golden_csf():
    """proj/tests/test_tensor.cpp:11-21 (also pinned through the reference build_csf)."""
    g = [m for m in MANIFEST if m["name"] == "coo3_csf"][0]
    assert g["idx"] == [[0, 1], [0, 1, 0], [0, 2, 0]]
    assert g["ptr"] == [[0, 2, 3], [0, 1, 2, 3]]
    coords = np.array([[0, 0, 0], [0, 1, 2], [1, 0, 0]])
    csf = Csf.from_coo([2, 2, 3], coords, np.array([1.0, 2.0, 3.0]))
    assert [a.tolist() for a in csf.idx] == g["idx"]
    assert [a.tolist() for a in csf.ptr] == g["ptr"]
    assert csf.values.tolist() == g["values"]


def test_gen_random_count_and_determinism():
    """proj/tests/test_tns_io.cpp:65-92: ceil(0.1*512) = 52, seeded."""
    a = Csf.gen_random([8, 8, 8], 0.1, 42)
    b = Csf.gen_random([8, 8, 8], 0.1, 42)
    c = Csf.gen_random([8, 8, 8], 0.1, 43)
    assert a.nnz == 52 and c.nnz == 52
    assert np.array_equal(a.values, b.values)
    assert not np.array_equal(a.values, c.values)
    assert Csf.gen_random([4, 4], 1.0, 7).nnz == 16
    with pytest.raises(ValueError):
        Csf.gen_random([8, 8, 8], 0.0, 1)


def test_mttkrp_on_coo3_direct_evaluation():
    """proj/tests/test_executor.cpp:43-72: MTTKRP on the 3-entry fixture."""
    coords = np.array([[0, 0, 0], [0, 1, 2], [1, 0, 0]])
    vals = np.array([1.0, 2.0, 3.0])
    csf = Csf.from_coo([2, 2, 3], coords, vals)
    B = gen_dense(2 * 2, 7 ^ stable_hash("B")).reshape(2, 2)
    C = gen_dense(3 * 2, 7 ^ stable_hash("C")).reshape(3, 2)
    expect = np.zeros((2, 2))
    for (i, j, k), v in zip(coords, vals):
        expect[i] += v * B[j] * C[k]
    got = OB.oracle_nest(1, csf, [B, C], (2, 0, 0)).reshape(2, 2)
    assert np.abs(got - expect).max() <= 1e-12


def pinned_flops(kind, L, nnz, R, S, T):
    if kind in (1, 6, 7):  # MTTKRP-3, any output mode: 2·nnz·R + 2·nnz_ij·R
        return 2 * nnz * R + 2 * L[1] * R
    if kind == 2:
        return 2 * nnz * S + 2 * L[1] * R * S
    if kind == 3:
        return 2 * L[1] * R + 2 * nnz * R + 2 * nnz
    if kind == 4:
        return 2 * R * (nnz + L[2] + L[1])
    return 2 * nnz * T + 2 * L[2] * S * T + 2 * L[1] * R * S * T


@pytest.mark.parametrize("m", CASES, ids=[m["name"] for m in CASES])
def test_pinned_flop_formulas_equal_reference_counters(m):
    """SURVEY.md §8a pinned-nest formulas == spttn::execute multiply_adds
    (== flops_estimate, proj/src/executor.cpp:628-650)."""
    L = m["level_sizes"]
    R, S, T = m["ranks"]
    assert pinned_flops(m["kind"], L, L[-1], R, S, T) == m["multiply_adds"]


@pytest.mark.parametrize("m", CASES, ids=[m["name"] for m in CASES])
def test_reset_counts_are_level_counts(m):
    """Buffers reset once per entry of their producer subtree
    (proj/tests/test_executor.cpp:270-288): MTTKRP-3/TTMc-3 X per (i,j);
    TTTP X per (i,j), Y per leaf; order 4: X per (i,j,k), Y per (i,j)."""
    L = m["level_sizes"]
    R = m["ranks"][0]
    # non-root MTTKRP orders keep a scalar buffer per (i,j,a): reset L1*R times
    want = {1: [L[1]], 2: [L[1]], 3: [L[1], L[2]], 4: [L[2], L[1]], 5: [L[2], L[1]],
            6: [L[1] * R], 7: [L[1] * R]}[m["kind"]]
    assert m["buffer_resets"] == want


def test_unfactorized_counts_golden():
    """Unfactorized madds = num_inputs * nnz * prod(free dims) (executor.cpp:652-658)."""
    for m in CASES:
        dims = m["dims"]
        sp = set(m["kernel"].split("[")[1].split("]")[0].split(","))
        free = np.prod([v for k, v in dims.items() if k not in sp])
        ninputs = len(m["kernel"].split("->")[0].split("*"))
        assert m["unfactorized_multiply_adds"] == ninputs * m["level_sizes"][-1] * free


@pytest.mark.parametrize("m", CASES, ids=[m["name"] for m in CASES])
def test_fused_matches_unfactorized_within_reference_tolerance(m):
    """proj/tests/test_executor.cpp:24-39 tolerance 1e-10 (1 + max|oracle|)."""
    _, _, z = load_case(m)
    tol = 1e-10 * (1 + np.abs(z["unfactorized"]).max())
    assert np.abs(z["fused"] - z["unfactorized"]).max() <= tol


# ---- live reference (built here from /root/reference) -------------------------

ref_only = pytest.mark.skipif(not OB.ref_available(), reason="oracle/_ref not built")


@ref_only
@pytest.mark.parametrize("seed", [1, 5, 9])
def test_gen_random_matches_live_reference(seed):
    idx, ptr, vals = OB.ref_gen_random_csf(["i", "j", "k", "l"], [7, 5, 6, 4], 0.3, seed)
    mine = Csf.gen_random([7, 5, 6, 4], 0.3, seed)
    assert all(np.array_equal(a, b) for a, b in zip(idx, mine.idx))
    assert all(np.array_equal(a, b) for a, b in zip(ptr, mine.ptr))
    assert np.array_equal(vals, mine.values)


@ref_only
def test_csf_from_coo_matches_reference_build_csf_with_duplicates():
    rng = np.random.default_rng(3)
    coords = rng.integers(0, [5, 4, 6], size=(200, 3))
    vals = rng.uniform(-1, 1, 200)
    idx, ptr, rv = OB.ref_build_csf(["i", "j", "k"], [5, 4, 6], coords, vals, ["i", "j", "k"])
    mine = Csf.from_coo([5, 4, 6], coords, vals)
    assert all(np.array_equal(a, b) for a, b in zip(idx, mine.idx))
    assert all(np.array_equal(a, b) for a, b in zip(ptr, mine.ptr))
    # duplicates summed in sorted order; values agree to rounding of the sum order
    assert np.allclose(rv, mine.values, rtol=0, atol=1e-15)


@ref_only
@pytest.mark.parametrize("key", ["mttkrp3", "ttmc3", "tttp3", "mttkrp4", "ttmc4"])
def test_c_oracle_matches_live_reference_on_baseline_shaped_inputs(key):
    """BASELINE-shaped synthetic inputs (Zipf / uniform, N(0,1) factors) at
    reduced scale: C oracle == spttn_ref::execute bit-for-bit."""
    from paper_2307_05740_b200.configs import make_workload
    w = make_workload(key, scale=2e-4 if key != "tttp3" else 4e-5)
    c = w.cfg
    dims = dict(zip(c.mode_names, w.dims))
    rank_names = {"mttkrp3": ["r"], "ttmc3": ["r", "s"], "tttp3": ["r"], "mttkrp4": ["r"],
                  "ttmc4": ["r", "s", "t"]}[key]
    for n, r in zip(rank_names, c.ranks):
        dims[n] = r
    got = OB.oracle_nest(c.kind, w.csf, w.factors, c.ranks)
    ref, stats = OB.ref_execute(c.kernel, dims, c.path, c.order_text, w.csf, w.factors,
                                len(got))
    assert np.array_equal(got, ref)
    from paper_2307_05740_b200.configs import algorithmic_flops
    assert stats["multiply_adds"] == algorithmic_flops(w)
