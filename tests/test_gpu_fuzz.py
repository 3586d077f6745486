"""Seeded random sweep over the pinned kernels' supported envelope: ranks
that are not multiples of 4 or 8 (vector / fragment tails), tensor shapes
from 1 to 60 per mode, uniform or single-hot-index skew, tiny work items that
force split slices, and every kernel variant kept for A/B — each case against
the C oracle at the north-star bar, plus bit-identical re-execution for the
owner-computes kernels."""
import numpy as np
import pytest

from parity import assert_parity, oracle_with_norm

pytestmark = pytest.mark.gpu

RANKS = [1, 2, 3, 4, 5, 7, 8, 12, 16, 17, 24, 31, 32, 33, 48, 64, 100, 128]
VARIANT_ENV = {1: ("SPTTN_MTTKRP_MODE", ["0", "2", "3", "4"]),
               4: ("SPTTN_MTTKRP_MODE", ["0", "3"]),
               2: ("SPTTN_GROUP_OVERHEAD", ["0", "12"]),
               5: ("SPTTN_TTMC4_MODE", ["3", "4"]),
               3: ("SPTTN_TTTP_PIECE", ["1", "5", "64"])}


@pytest.fixture(scope="module")
def E():
    import torch
    assert torch.cuda.is_available(), "GPU suite needs a CUDA device"
    import paper_2307_05740_b200 as P
    return P


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    kind = int(rng.choice([1, 2, 3, 4, 5, 6, 7]))
    order = 4 if kind in (4, 5) else 3
    dims = [int(rng.integers(1, 61)) for _ in range(order)]
    if kind == 2:
        ranks = (int(rng.integers(1, 17)), int(rng.integers(1, 17)), 0)
    elif kind == 5:
        ranks = tuple(int(rng.integers(1, 9)) for _ in range(3))
    elif kind in (6, 7):
        ranks = (int(rng.choice([r for r in RANKS if r <= 32])), 0, 0)
    else:
        ranks = (int(rng.choice(RANKS)), 0, 0)
    cap = int(np.prod(dims))
    nnz = int(rng.integers(1, min(cap, 4000) + 1))
    if rng.random() < 0.4:  # one hot index per mode: long fibers and a heavy slice
        hot = [int(rng.integers(0, d)) for d in dims]
        coords = np.stack([np.where(rng.random(nnz) < 0.6, hot[m], rng.integers(0, dims[m], nnz))
                           for m in range(order)], axis=1)
    else:
        coords = np.stack([rng.integers(0, d, nnz) for d in dims], axis=1)
    vals = rng.uniform(-1, 1, coords.shape[0])
    R, S, T = ranks
    if kind in (1, 4):
        fs = [rng.standard_normal((dims[m], R)) for m in range(1, order)]
    elif kind == 2:
        fs = [rng.standard_normal((dims[1], R)), rng.standard_normal((dims[2], S))]
    elif kind == 3:
        fs = [rng.standard_normal((dims[m], R)) for m in range(3)]
    elif kind == 5:
        fs = [rng.standard_normal((dims[1], R)), rng.standard_normal((dims[2], S)),
              rng.standard_normal((dims[3], T))]
    else:
        other = 2 if kind == 6 else 1
        fs = [rng.standard_normal((dims[0], R)), rng.standard_normal((dims[other], R))]
    env = {}
    if kind in VARIANT_ENV and rng.random() < 0.5:
        name, modes = VARIANT_ENV[kind]
        env[name] = str(rng.choice(modes))
    if rng.random() < 0.5:
        env["SPTTN_CHUNK"] = str(int(rng.choice([1, 2, 3, 8])))
        env["SPTTN_GCHUNK"] = str(int(rng.choice([1, 2, 4])))
    residual = kind == 3 and rng.random() < 0.5
    # work-cut items (decomp.cu finish_unit_items): the per-group overhead of
    # the modes that read variable item bounds, incl. overhead 1 with tiny
    # GCHUNK, where one heavy group spans several items' shares (separate
    # stream: the original draws above stay unchanged)
    r2 = np.random.default_rng(5000 + seed)
    item_mode = {1: ("SPTTN_MTTKRP_MODE", "3"), 4: ("SPTTN_MTTKRP_MODE", "3"),
                 2: ("SPTTN_TTMC3_MODE", "10"), 5: ("SPTTN_TTMC4_MODE", "4")}  # TTMc-3: one kernel, env unused
    if kind in item_mode and (env.get(item_mode[kind][0], item_mode[kind][1]) == item_mode[kind][1]
                              or seed >= 160):
        env[item_mode[kind][0]] = item_mode[kind][1]
        env["SPTTN_GROUP_OVERHEAD"] = str(int(r2.choice([0, 1, 3, 12])))
        if seed >= 160 or r2.random() < 0.5:
            env["SPTTN_GCHUNK"] = str(int(r2.choice([1, 2, 4])))
            env["SPTTN_CHUNK"] = str(int(r2.choice([1, 2, 3])))
    return kind, dims, coords, vals, fs, ranks, env, residual


@pytest.mark.parametrize("seed", range(220))
def test_random_case_matches_oracle(E, seed, monkeypatch):
    from paper_2307_05740_b200.tensor import Csf
    kind, dims, coords, vals, fs, ranks, env, residual = _case(seed)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    csf = Csf.from_coo(dims, coords, vals)
    dev = E.DeviceCsf(csf)
    plan = E.Plan(kind, dev, fs, ranks=ranks, flags=E.FLAG_RESIDUAL if residual else 0)
    plan.execute()
    out = plan.read_output()
    want, norm = oracle_with_norm(kind, csf, fs, ranks, residual=residual)
    what = f"seed {seed} kind {kind} dims {dims} ranks {ranks} nnz {csf.nnz} env {env}"
    assert_parity(out, want, norm, what)
    plan.execute()
    again = plan.read_output()
    if kind in (6, 7):  # fp64 atomics: arrival order varies
        assert_parity(again, want, norm, what + " rerun")
    else:
        assert np.array_equal(again, out), what + ": re-execution not bit-identical"
