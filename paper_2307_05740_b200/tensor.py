"""Host-side sparse tensors in the reference's CsfTensor layout.

`Csf` holds exactly what `spttn::CsfTensor` holds (proj/include/spttn/
tensor.hpp:49-57): per level an int64 coordinate array `idx[l]`, for all but
the leaf level an int64 child-pointer array `ptr[l]` (nodes+1 entries), and
the fp64 leaf values. Generators come from libspttn_datagen.so:
  * `gen_random` / `gen_dense` / `stable_hash` reproduce the reference's
    seeded generators bit-for-bit (proj/src/tns_io.cpp:108-175), so the
    reference's test fixtures (proj/tests/fixtures.hpp:57-95) can be rebuilt
    without the reference;
  * `gen_baseline` / `gen_normal` build the BASELINE.json workloads
    (SURVEY.md §8d).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as N


@dataclass
class Csf:
    dims: list[int]
    idx: list[np.ndarray]
    ptr: list[np.ndarray]
    values: np.ndarray
    names: list[str] = field(default_factory=list)

    @property
    def order(self) -> int:
        return len(self.dims)

    @property
    def nnz(self) -> int:
        return int(self.values.shape[0])

    def level_sizes(self) -> list[int]:
        return [int(a.shape[0]) for a in self.idx]

    def nnz_at_level(self, k: int) -> int:
        """Node count at level k (1-based), spttn::nnz_at_level (tensor.cpp:96-100)."""
        return int(self.idx[k - 1].shape[0])

    # -- construction ------------------------------------------------------
    @staticmethod
    def _from_handle(h, names=None) -> "Csf":
        lib = N.datagen()
        if not h:
            raise ValueError(lib.dg_last_error().decode())
        try:
            d = lib.dg_csf_order(h)
            dims = [int(lib.dg_csf_dim(h, l)) for l in range(d)]
            sizes = [int(lib.dg_csf_level_size(h, l)) for l in range(d)]
            idx, ptr = [], []
            for l in range(d):
                n = sizes[l]
                a = np.ctypeslib.as_array(lib.dg_csf_idx(h, l), shape=(n,)).copy() if n else \
                    np.zeros(0, np.int64)
                idx.append(a)
                if l + 1 < d:
                    ptr.append(np.ctypeslib.as_array(lib.dg_csf_ptr(h, l), shape=(n + 1,)).copy())
            nnz = sizes[-1]
            vals = np.ctypeslib.as_array(lib.dg_csf_values(h), shape=(nnz,)).copy() if nnz else \
                np.zeros(0, np.float64)
        finally:
            lib.dg_csf_free(h)
        return Csf(dims, idx, ptr, vals, list(names or []))

    @staticmethod
    def gen_random(dims, density: float, seed: int, names=None) -> "Csf":
        """Reference gen_random (tns_io.cpp:123-159) + build_csf in declared order."""
        lib = N.datagen()
        d = (C.c_int64 * len(dims))(*dims)
        return Csf._from_handle(lib.dg_gen_random(len(dims), d, float(density), seed), names)

    @staticmethod
    def gen_baseline(dims, nnz: int, zipf_s: float, seed: int, names=None) -> "Csf":
        lib = N.datagen()
        d = (C.c_int64 * len(dims))(*dims)
        return Csf._from_handle(
            lib.dg_gen_baseline(len(dims), d, int(nnz), float(zipf_s), seed), names)

    @staticmethod
    def from_coo(dims, coords: np.ndarray, values: np.ndarray, names=None) -> "Csf":
        """normalize() + build_csf in declared order (tensor.cpp:24-94)."""
        lib = N.datagen()
        coords = np.ascontiguousarray(coords, dtype=np.int64)
        values = np.ascontiguousarray(values, dtype=np.float64)
        d = (C.c_int64 * len(dims))(*dims)
        return Csf._from_handle(
            lib.dg_csf_from_coo(len(dims), d, int(values.shape[0]),
                                coords.ctypes.data_as(N.c_i64_p),
                                values.ctypes.data_as(N.c_dbl_p)), names)

    def root_sample(self, stride: int, offset: int = 0) -> "Csf":
        """Every `stride`-th root slice, copied whole (bounded CPU samples)."""
        # rebuild through COO (keeps this file free of a second CSF writer)
        keep = np.arange(offset, self.level_sizes()[0], stride)
        coo, vals = self.to_coo()
        leaf_root = self.leaf_ancestors(0)
        mask = np.isin(leaf_root, keep)
        return Csf.from_coo(self.dims, coo[mask], vals[mask], self.names)

    def leaf_ancestors(self, level: int) -> np.ndarray:
        """Node id at `level` owning each leaf."""
        node = np.arange(self.nnz, dtype=np.int64)
        for l in range(self.order - 2, level - 1, -1):
            node = np.searchsorted(self.ptr[l], node, side="right") - 1
        return node

    def to_coo(self) -> tuple[np.ndarray, np.ndarray]:
        """csf_to_coo (tensor.cpp:102-126): leaf-order coordinates."""
        coo = np.zeros((self.nnz, self.order), dtype=np.int64)
        for l in range(self.order):
            coo[:, l] = self.idx[l][self.leaf_ancestors(l)] if self.nnz else 0
        return coo, self.values.copy()

    def abs(self) -> "Csf":
        return Csf(self.dims, self.idx, self.ptr, np.abs(self.values), self.names)

    def with_values(self, values: np.ndarray) -> "Csf":
        return Csf(self.dims, self.idx, self.ptr, np.ascontiguousarray(values, np.float64),
                   self.names)


def stable_hash(name: str) -> int:
    return int(N.datagen().dg_stable_hash(name.encode()))


def gen_dense(n: int, seed: int) -> np.ndarray:
    """Reference gen_dense (tns_io.cpp:161-166): n values uniform(-1, 1)."""
    out = np.empty(n, dtype=np.float64)
    N.datagen().dg_gen_dense(n, seed & 0xFFFFFFFFFFFFFFFF, out.ctypes.data_as(N.c_dbl_p))
    return out


def gen_normal(n: int, seed: int, sigma: float = 1.0) -> np.ndarray:
    """N(0, sigma^2) by Box-Muller."""
    out = np.empty(n, dtype=np.float64)
    N.datagen().dg_gen_normal(n, seed & 0xFFFFFFFFFFFFFFFF, float(sigma),
                              out.ctypes.data_as(N.c_dbl_p))
    return out
