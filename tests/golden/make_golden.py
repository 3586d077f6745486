"""Generates the golden parity fixtures in tests/golden/ from the REFERENCE
library itself (oracle/_ref/libspttn_ref_bridge.so, built from
/root/reference by oracle/Makefile). Run in the build container:

    python tests/golden/make_golden.py

Inputs follow the reference's own test fixtures (proj/tests/fixtures.hpp):
gen_random(density, seed) coordinates, gen_dense factors seeded
7 ^ stable_hash(name); outputs are spttn_ref::execute on the pinned nest,
spttn_ref::execute_unfactorized, the multiply-add / reset counters and hooks.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE.parents[1]))

import oracle_bindings as OB  # noqa: E402

# (name, kernel, dims, path, order, density, seed, kind, ranks, sparse-out)
CASES = [
    ("mttkrp3_small", "T[i,j,k]*B[j,a]*C[k,a]->A[i,a]", {"i": 8, "j": 8, "k": 8, "a": 4},
     "((T*C)*B)", "i,j,k,a;i,j,a", 0.05, 13, 1, (4, 0, 0), False),
    ("mttkrp3_r32", "T[i,j,k]*B[j,a]*C[k,a]->A[i,a]", {"i": 20, "j": 16, "k": 24, "a": 32},
     "((T*C)*B)", "i,j,k,a;i,j,a", 0.05, 202, 1, (32, 0, 0), False),
    ("ttmc3_small", "T[i,j,k]*U[j,r]*V[k,s]->S[i,r,s]",
     {"i": 8, "j": 8, "k": 8, "r": 3, "s": 2}, "((T*V)*U)", "i,j,k,s;i,j,s,r", 0.05, 29, 2,
     (3, 2, 0), False),
    ("ttmc3_r16", "T[i,j,k]*U[j,r]*V[k,s]->S[i,r,s]",
     {"i": 24, "j": 24, "k": 24, "r": 16, "s": 16}, "((T*V)*U)", "i,j,k,s;i,j,s,r", 0.02, 203,
     2, (16, 16, 0), False),
    ("tttp3_small", "T[i,j,k]*U[i,r]*V[j,r]*W[k,r]->S[i,j,k] @sparse_out",
     {"i": 6, "j": 5, "k": 7, "r": 3}, "(((U*V)*W)*T)", "i,j,r;i,j,k,r;i,j,k", 0.25, 11, 3,
     (3, 0, 0), True),
    ("tttp3_r64", "T[i,j,k]*U[i,r]*V[j,r]*W[k,r]->S[i,j,k] @sparse_out",
     {"i": 16, "j": 12, "k": 10, "r": 64}, "(((U*V)*W)*T)", "i,j,r;i,j,k,r;i,j,k", 0.1, 17, 3,
     (64, 0, 0), True),
    ("mttkrp4_small", "T[i,j,k,l]*B[j,r]*C[k,r]*D[l,r]->A[i,r]",
     {"i": 6, "j": 5, "k": 6, "l": 5, "r": 4}, "(((T*D)*C)*B)", "i,j,k,l,r;i,j,k,r;i,j,r", 0.1,
     41, 4, (4, 0, 0), False),
    ("mttkrp4_r32", "T[i,j,k,l]*B[j,r]*C[k,r]*D[l,r]->A[i,r]",
     {"i": 9, "j": 8, "k": 7, "l": 10, "r": 32}, "(((T*D)*C)*B)", "i,j,k,l,r;i,j,k,r;i,j,r", 0.05,
     43, 4, (32, 0, 0), False),
    ("mttkrp3j_small", "T[i,j,k]*A[i,a]*C[k,a]->B[j,a]", {"i": 8, "j": 9, "k": 7, "a": 4},
     "((T*C)*A)", "i,j,a,k;i,j,a", 0.08, 21, 6, (4, 0, 0), False),
    ("mttkrp3j_r32", "T[i,j,k]*A[i,a]*C[k,a]->B[j,a]", {"i": 20, "j": 18, "k": 16, "a": 32},
     "((T*C)*A)", "i,j,a,k;i,j,a", 0.05, 22, 6, (32, 0, 0), False),
    ("mttkrp3k_small", "T[i,j,k]*A[i,a]*B[j,a]->C[k,a]", {"i": 7, "j": 8, "k": 9, "a": 4},
     "((A*B)*T)", "i,j,a;i,j,a,k", 0.08, 23, 7, (4, 0, 0), False),
    ("mttkrp3k_r32", "T[i,j,k]*A[i,a]*B[j,a]->C[k,a]", {"i": 16, "j": 20, "k": 18, "a": 32},
     "((A*B)*T)", "i,j,a;i,j,a,k", 0.05, 24, 7, (32, 0, 0), False),
    ("ttmc4_small", "T[i,j,k,l]*U[j,r]*V[k,s]*W[l,t]->S[i,r,s,t]",
     {"i": 4, "j": 4, "k": 4, "l": 4, "r": 2, "s": 3, "t": 2}, "(((T*W)*V)*U)",
     "i,j,k,l,t;i,j,k,s,t;i,j,r,s,t", 0.2, 3, 5, (2, 3, 2), False),
    ("ttmc4_r8", "T[i,j,k,l]*U[j,r]*V[k,s]*W[l,t]->S[i,r,s,t]",
     {"i": 7, "j": 6, "k": 8, "l": 6, "r": 8, "s": 8, "t": 8}, "(((T*W)*V)*U)",
     "i,j,k,l,t;i,j,k,s,t;i,j,r,s,t", 0.08, 77, 5, (8, 8, 8), False),
]


def parse_tensors(kernel: str):
    lhs, out = kernel.split("->")
    out = out.split("@")[0].strip()
    terms = [t.strip() for t in lhs.split("*")]

    def one(t):
        name, rest = t.split("[")
        return name, rest.rstrip("]").split(",")
    return [one(t) for t in terms], one(out)


def main():
    manifest = []
    for (name, kernel, dims, path, order, density, seed, kind, ranks, sparse) in CASES:
        inputs, (oname, oids) = parse_tensors(kernel)
        sp_name, sp_ids = inputs[0]
        sdims = [dims[i] for i in sp_ids]
        idx, ptr, vals = OB.ref_gen_random_csf(sp_ids, sdims, density, seed)
        factors = []
        for fname, fids in inputs[1:]:
            fdims = [dims[i] for i in fids]
            fseed = 7 ^ OB.ref().ref_stable_hash(fname.encode())
            factors.append(OB.ref_gen_dense(fids, fdims, fseed).reshape(fdims))

        class _C:  # minimal Csf-like view for the bridge
            pass
        c = _C()
        c.order, c.dims, c.idx, c.ptr, c.values = len(sdims), sdims, idx, ptr, vals
        c.level_sizes = lambda: [len(a) for a in idx]
        c.nnz = len(vals)
        out_count = len(vals) if sparse else int(np.prod([dims[i] for i in oids]))
        fused, stats = OB.ref_execute(kernel, dims, path, order, c, factors, out_count)
        unf, unf_madds = OB.ref_unfactorized(kernel, dims, c, factors, out_count)
        arrays = {f"idx{l}": a for l, a in enumerate(idx)}
        arrays.update({f"ptr{l}": a for l, a in enumerate(ptr)})
        arrays["values"] = vals
        for f, a in enumerate(factors):
            arrays[f"factor{f}"] = a
        arrays["fused"] = fused
        arrays["unfactorized"] = unf
        if sparse:  # completion residual oracle: reference on unit values, rho = T - S
            c1 = _C()
            c1.order, c1.dims, c1.idx, c1.ptr, c1.values = c.order, c.dims, idx, ptr, np.ones_like(vals)
            c1.level_sizes, c1.nnz = c.level_sizes, c.nnz
            s_unit, _ = OB.ref_execute(kernel, dims, path, order, c1, factors, out_count)
            arrays["residual"] = vals - s_unit
        np.savez_compressed(HERE / f"{name}.npz", **arrays)
        manifest.append({"name": name, "kernel": kernel, "dims": dims, "path": path,
                         "order": order, "density": density, "seed": seed, "kind": kind,
                         "ranks": list(ranks), "sparse_out": sparse, "sparse_dims": sdims,
                         "multiply_adds": stats["multiply_adds"],
                         "buffer_resets": stats["buffer_resets"],
                         "unfactorized_multiply_adds": unf_madds,
                         "level_sizes": [len(a) for a in idx]})
        print(f"{name}: nnz={len(vals)} madds={stats['multiply_adds']}")
    # coo3 golden CSF (proj/tests/test_tensor.cpp:11-21) through the reference build_csf
    coords = np.array([[0, 0, 0], [0, 1, 2], [1, 0, 0]], np.int64)
    idx, ptr, vals = OB.ref_build_csf(["i", "j", "k"], [2, 2, 3], coords, [1.0, 2.0, 3.0],
                                      ["i", "j", "k"])
    manifest.append({"name": "coo3_csf", "idx": [a.tolist() for a in idx],
                     "ptr": [a.tolist() for a in ptr], "values": vals.tolist()})
    (HERE / "manifest.json").write_text(json.dumps(manifest, indent=1) + "\n")


if __name__ == "__main__":
    main()
