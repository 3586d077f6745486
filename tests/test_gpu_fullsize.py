"""Full-size parity: every BASELINE.json config (and the non-root MTTKRP-3
modes) at its exact bench shape and seed, CUDA path vs the plain-C oracle.

The oracle (oracle/spttn_oracle.c) is pinned bit-for-bit to the compiled
reference executor by tests/test_oracle.py (goldens + live reference); here
it is the checker at the sizes bench.py measures. Bar (BASELINE.json north
star): |gpu - oracle| <= 1e-10 * sum|contributions| per output entry, the
normaliser being the oracle on |T|, |factors| (+|t| for the residual);
output sparsity bit-exact (an entry with no contribution stays exactly 0);
repeated execution bit-identical (proj/tests/test_executor.cpp:203-220) for
every owner-computes kernel.

These are the paths the bench times: the heavy-slice second fix-up pass,
thousands of split slices, the Zipf giant fibers — none of which the
reduced-scale cases reach without forcing tiny items.
"""
import numpy as np
import pytest

from parity import REL_TOL, oracle_with_norm

pytestmark = pytest.mark.gpu

KEYS = ["mttkrp3", "ttmc3", "tttp3", "mttkrp4", "ttmc4", "mttkrp3_j", "mttkrp3_k"]
# every default plan is owner-computes (the non-root MTTKRP-3 modes run on
# the output-mode-major re-ordered tensor): re-executions are bit-identical
ATOMIC = set()


@pytest.fixture(scope="module")
def E():
    import torch
    assert torch.cuda.is_available(), "GPU suite needs a CUDA device"
    import paper_2307_05740_b200 as P
    return P


@pytest.mark.parametrize("key", KEYS)
def test_full_size_config_matches_oracle(E, key):
    from paper_2307_05740_b200.configs import make_workload
    w = make_workload(key)  # scale 1.0: the bench's exact tensor, seed and factors
    c = w.cfg
    assert w.csf.nnz == c.nnz
    flags = E.FLAG_RESIDUAL if c.residual else 0
    dev = E.DeviceCsf(w.csf)
    plan = E.Plan(c.kind, dev, w.factors, ranks=c.ranks, flags=flags)
    plan.execute()
    got = plan.read_output()
    want, norm = oracle_with_norm(c.kind, w.csf, w.factors, c.ranks, residual=c.residual)
    assert got.shape == want.shape
    err = np.abs(got - want)
    bad = err > REL_TOL * norm
    rel = np.where(norm > 0, err / np.where(norm > 0, norm, 1.0), 0.0)
    assert not bad.any(), (f"{key}: {int(bad.sum())} of {got.size} entries outside tolerance, "
                           f"max normalised error {rel.max():.3e}")
    zero = norm == 0
    assert np.all(got[zero] == 0.0), f"{key}: non-zero where every contribution is zero"
    print(f"{key}: nnz={w.csf.nnz} entries={got.size} max normalised err {rel.max():.3e} "
          f"exact zeros {int(zero.sum())} split_slices={plan.info()['split_slices']}")
    plan.execute()
    again = plan.read_output()
    if key in ATOMIC:
        assert np.all(np.abs(again - want) <= REL_TOL * norm), f"{key}: re-execution"
        assert np.all(again[zero] == 0.0)
    else:
        assert np.array_equal(again, got), f"{key}: re-execution is not bit-identical"
    plan.close()
    dev.close()
