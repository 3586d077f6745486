"""BASELINE.json workloads and the algorithmic byte / flop figures.

Each config is synthetic (no public dataset is involved): distinct uniform or
Zipf(1.1) coordinates kept in first-draw order from mt19937_64(seed = config
number), values uniform(-1,1), factors N(0, sigma^2) seeded
`seed ^ stable_hash(name)` (mirroring proj/tests/fixtures.hpp:92).
`scale` < 1 shrinks nnz (and dims by scale**(1/order)) for quick tests.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import engine as E
from .tensor import Csf, gen_normal, stable_hash


@dataclass(frozen=True)
class Config:
    key: str
    number: int          # 1-based position in BASELINE.json "configs"
    kind: int
    kernel: str          # reference kernel-spec text
    path: str            # pinned contraction path (reference describe())
    order_text: str      # pinned per-term loop orders
    mode_names: tuple
    dims: tuple
    nnz: int
    zipf_s: float
    ranks: tuple         # (R, S, T) as used by the nest
    factor_names: tuple  # kernel input order
    factor_rows: tuple   # CSF level of each factor's row index
    factor_rank: tuple   # which of ranks indexes each factor's columns
    sigma: float
    residual: bool = False


CONFIGS = {
    "mttkrp3": Config("mttkrp3", 1, E.NEST_MTTKRP3, "T[i,j,k]*B[j,r]*C[k,r]->A[i,r]",
                      "((T*C)*B)", "i,j,k,r;i,j,r", ("i", "j", "k"), (1000, 1000, 1000),
                      1_000_000, 0.0, (32, 0, 0), ("B", "C"), (1, 2), (0, 0), 1.0),
    "ttmc3": Config("ttmc3", 2, E.NEST_TTMC3, "T[i,j,k]*U[j,r]*V[k,s]->Y[i,r,s]",
                    "((T*V)*U)", "i,j,k,s;i,j,s,r", ("i", "j", "k"), (20000, 20000, 20000),
                    10_000_000, 1.1, (16, 16, 0), ("U", "V"), (1, 2), (0, 1), 1.0),
    "tttp3": Config("tttp3", 3, E.NEST_TTTP3, "T[i,j,k]*A[i,r]*B[j,r]*C[k,r]->S[i,j,k] @sparse_out",
                    "(((A*B)*C)*T)", "i,j,r;i,j,k,r;i,j,k", ("i", "j", "k"),
                    (100000, 50000, 20000), 50_000_000, 0.0, (64, 0, 0), ("A", "B", "C"),
                    (0, 1, 2), (0, 0, 0), math.sqrt(1.0 / 8.0), residual=True),
    "mttkrp4": Config("mttkrp4", 4, E.NEST_MTTKRP4, "T[i,j,k,l]*B[j,r]*C[k,r]*D[l,r]->A[i,r]",
                      "(((T*D)*C)*B)", "i,j,k,l,r;i,j,k,r;i,j,r", ("i", "j", "k", "l"),
                      (5000, 5000, 5000, 5000), 20_000_000, 1.1, (32, 0, 0), ("B", "C", "D"),
                      (1, 2, 3), (0, 0, 0), 1.0),
    # §8f-2: MTTKRP-3 for the non-root modes on the mttkrp3 tensor (same seed),
    # the planners' (max-buf-dim) orders; not BASELINE configs
    "mttkrp3_j": Config("mttkrp3_j", 1, E.NEST_MTTKRP3_J, "T[i,j,k]*A[i,r]*C[k,r]->B[j,r]",
                        "((T*C)*A)", "i,j,r,k;i,j,r", ("i", "j", "k"), (1000, 1000, 1000),
                        1_000_000, 0.0, (32, 0, 0), ("A", "C"), (0, 2), (0, 0), 1.0),
    "mttkrp3_k": Config("mttkrp3_k", 1, E.NEST_MTTKRP3_K, "T[i,j,k]*A[i,r]*B[j,r]->C[k,r]",
                        "((A*B)*T)", "i,j,r;i,j,r,k", ("i", "j", "k"), (1000, 1000, 1000),
                        1_000_000, 0.0, (32, 0, 0), ("A", "B"), (0, 1), (0, 0), 1.0),
    "ttmc4": Config("ttmc4", 5, E.NEST_TTMC4, "T[i,j,k,l]*U[j,r]*V[k,s]*W[l,t]->Y[i,r,s,t]",
                    "(((T*W)*V)*U)", "i,j,k,l,t;i,j,k,s,t;i,j,r,s,t", ("i", "j", "k", "l"),
                    (2000, 2000, 2000, 2000), 10_000_000, 0.0, (8, 8, 8), ("U", "V", "W"),
                    (1, 2, 3), (0, 1, 2), 1.0),
}


@dataclass
class Workload:
    cfg: Config
    csf: Csf
    factors: list          # numpy arrays, kernel input order, row-major [dim, rank]
    dims: tuple
    nnz_requested: int

    @property
    def out_count(self) -> int:
        c = self.cfg
        if c.kind == E.NEST_TTTP3:
            return self.csf.nnz
        R, S, T = c.ranks
        if c.kind in (E.NEST_MTTKRP3_J, E.NEST_MTTKRP3_K):  # output rows on level 1 / 2
            return self.dims[1 if c.kind == E.NEST_MTTKRP3_J else 2] * R
        return self.dims[0] * R * max(S, 1) * max(T, 1)


def make_workload(key: str, scale: float = 1.0, seed_offset: int = 0) -> Workload:
    cfg = CONFIGS[key]
    d = len(cfg.dims)
    if scale >= 1.0:
        dims, nnz = cfg.dims, cfg.nnz
    else:
        f = scale ** (1.0 / d)
        dims = tuple(max(4, int(round(x * f))) for x in cfg.dims)
        nnz = max(1, int(cfg.nnz * scale))
        nnz = min(nnz, int(np.prod(np.array(dims, dtype=np.float64)) // 2))
    seed = cfg.number + seed_offset
    csf = Csf.gen_baseline(list(dims), nnz, cfg.zipf_s, seed, list(cfg.mode_names))
    factors = []
    for name, lvl, rk in zip(cfg.factor_names, cfg.factor_rows, cfg.factor_rank):
        rows, cols = dims[lvl], cfg.ranks[rk]
        f = gen_normal(rows * cols, seed ^ stable_hash(name), cfg.sigma).reshape(rows, cols)
        factors.append(f)
    return Workload(cfg, csf, factors, dims, nnz)


def algorithmic_bytes(w: Workload) -> int:
    """bytes_alg: 12 per leaf (fp64 value + int32 coordinate),
    8 per non-leaf node (int32 idx + int32 ptr), each factor read once, the
    output written once (TTTP: 8 per leaf)."""
    csf = w.csf
    sizes = csf.level_sizes()
    b = 12 * csf.nnz + 8 * sum(sizes[:-1])
    b += 8 * sum(int(f.size) for f in w.factors)
    b += 8 * w.out_count
    return int(b)


def algorithmic_flops(w: Workload) -> int:
    """flops_estimate of the pinned nest (proj/src/executor.cpp:628-650),
    2 per multiply-add (SURVEY.md §8a pinned-nest table)."""
    csf = w.csf
    L = csf.level_sizes()
    R, S, T = w.cfg.ranks
    k = w.cfg.kind
    if k in (E.NEST_MTTKRP3, E.NEST_MTTKRP3_J, E.NEST_MTTKRP3_K):
        return 2 * csf.nnz * R + 2 * L[1] * R
    if k == E.NEST_TTMC3:
        return 2 * csf.nnz * S + 2 * L[1] * R * S
    if k == E.NEST_TTTP3:
        return 2 * L[1] * R + 2 * csf.nnz * R + 2 * csf.nnz
    if k == E.NEST_MTTKRP4:
        return 2 * R * (csf.nnz + L[2] + L[1])
    if k == E.NEST_TTMC4:
        return 2 * csf.nnz * T + 2 * L[2] * S * T + 2 * L[1] * R * S * T
    raise ValueError(k)


def gather_bytes(w: Workload) -> int:
    """Diagnostic: factor-row bytes gathered with no reuse (one row per leaf
    and per fiber level that reads a factor)."""
    csf = w.csf
    L = csf.level_sizes()
    R, S, T = w.cfg.ranks
    k = w.cfg.kind
    if k == E.NEST_MTTKRP3:
        return 8 * R * (csf.nnz + L[1])
    if k == E.NEST_MTTKRP3_J:  # C row per leaf, A row per slice, B row atomics per (i,j)
        return 8 * R * (csf.nnz + L[0] + L[1])
    if k == E.NEST_MTTKRP3_K:  # A row per slice, B row per (i,j), C row atomics per leaf
        return 8 * R * (L[0] + L[1] + csf.nnz)
    if k == E.NEST_TTMC3:
        return 8 * (S * csf.nnz + R * L[1])
    if k == E.NEST_TTTP3:
        return 8 * R * (csf.nnz + L[1] + L[0])
    if k == E.NEST_MTTKRP4:
        return 8 * R * (csf.nnz + L[2] + L[1])
    if k == E.NEST_TTMC4:
        return 8 * (T * csf.nnz + S * L[2] + R * L[1])
    raise ValueError(k)
