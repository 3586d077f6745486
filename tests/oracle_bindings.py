"""TEST INFRASTRUCTURE: ctypes views of the oracles (never used by the product).

  oracle/build/libspttn_oracle_c.so   plain-C restatement of the pinned nests
  oracle/_ref/libspttn_ref_bridge.so  the reference library itself (built from
                                      /root/reference by oracle/Makefile)
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
ORACLE_C = ROOT / "oracle" / "build" / "libspttn_oracle_c.so"
REF_BRIDGE = ROOT / "oracle" / "_ref" / "libspttn_ref_bridge.so"

i64p = C.POINTER(C.c_int64)
dblp = C.POINTER(C.c_double)


class OcCsf(C.Structure):
    _fields_ = [("order", C.c_int), ("dims", C.c_int64 * 8), ("level_size", C.c_int64 * 8),
                ("idx", i64p * 8), ("ptr", i64p * 8), ("values", dblp)]


class OcUnfact(C.Structure):
    _fields_ = [("nfactors", C.c_int), ("nfree", C.c_int), ("free_dim", C.c_int64 * 4),
                ("factor_level", C.c_int * 6), ("factor_free", C.c_int * 6),
                ("factor", dblp * 6), ("out_sparse", C.c_int), ("out_has_root", C.c_int),
                ("out_nfree", C.c_int), ("out_free", C.c_int * 4)]


_oc = None
_ref = None


def oracle_c():
    global _oc
    if _oc is None:
        if not ORACLE_C.exists():
            raise RuntimeError(f"{ORACLE_C} missing: run make -C oracle")
        _oc = C.CDLL(str(ORACLE_C))
    return _oc


def ref_available() -> bool:
    return REF_BRIDGE.exists()


def ref():
    global _ref
    if _ref is None:
        lib = C.CDLL(str(REF_BRIDGE))
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_stable_hash.restype = C.c_uint64
        lib.ref_stable_hash.argtypes = [C.c_char_p]
        lib.ref_build_csf.restype = C.c_void_p
        lib.ref_gen_random_csf.restype = C.c_void_p
        lib.ref_gen_random_csf.argtypes = [C.c_int, C.c_char_p, i64p, C.c_double, C.c_uint64]
        lib.ref_csf_level_size.restype = C.c_int64
        lib.ref_csf_level_size.argtypes = [C.c_void_p, C.c_int]
        lib.ref_csf_copy.argtypes = [C.c_void_p, C.c_int, i64p, i64p]
        lib.ref_csf_values.argtypes = [C.c_void_p, dblp]
        lib.ref_csf_free.argtypes = [C.c_void_p]
        lib.ref_gen_dense.argtypes = [C.c_int, C.c_char_p, i64p, C.c_uint64, dblp]
        lib.ref_enumerate.restype = C.c_int64
        _ref = lib
    return _ref


class _CsfArgs:
    """Keeps ctypes arrays alive for one call."""

    def __init__(self, csf):
        d = csf.order
        self.idx = [np.ascontiguousarray(a, np.int64) for a in csf.idx]
        self.ptr = [np.ascontiguousarray(a, np.int64) for a in csf.ptr]
        self.vals = np.ascontiguousarray(csf.values, np.float64)
        self.sizes = (C.c_int64 * d)(*csf.level_sizes())
        self.idx_p = (i64p * d)(*[a.ctypes.data_as(i64p) for a in self.idx])
        self.ptr_p = (i64p * max(1, d - 1))(*[a.ctypes.data_as(i64p) for a in self.ptr])
        self.vals_p = self.vals.ctypes.data_as(dblp)
        oc = OcCsf()
        oc.order = d
        for l in range(d):
            oc.dims[l] = csf.dims[l]
            oc.level_size[l] = csf.level_sizes()[l]
            oc.idx[l] = self.idx_p[l]
            if l + 1 < d:
                oc.ptr[l] = self.ptr_p[l]
        oc.values = self.vals_p
        self.oc = oc


def oracle_nest(kind: int, csf, factors, ranks, residual=False) -> np.ndarray:
    """The pinned nest through the plain-C oracle (bit-identical to spttn::execute)."""
    lib = oracle_c()
    a = _CsfArgs(csf)
    fs = [np.ascontiguousarray(f, np.float64).ravel() for f in factors]
    fp = [f.ctypes.data_as(dblp) for f in fs]
    R, S, T = (list(ranks) + [0, 0, 0])[:3]
    I = csf.dims[0]
    if kind == 1:
        out = np.zeros(I * R)
        lib.oc_mttkrp3(C.byref(a.oc), C.c_int64(R), fp[0], fp[1], out.ctypes.data_as(dblp))
    elif kind == 2:
        out = np.zeros(I * R * S)
        lib.oc_ttmc3(C.byref(a.oc), C.c_int64(R), C.c_int64(S), fp[0], fp[1],
                     out.ctypes.data_as(dblp))
    elif kind == 3:
        out = np.zeros(csf.nnz)
        lib.oc_tttp3(C.byref(a.oc), C.c_int64(R), fp[0], fp[1], fp[2], out.ctypes.data_as(dblp),
                     C.c_int(1 if residual else 0))
    elif kind == 4:
        out = np.zeros(I * R)
        lib.oc_mttkrp4(C.byref(a.oc), C.c_int64(R), fp[0], fp[1], fp[2], out.ctypes.data_as(dblp))
    elif kind in (6, 7):  # MTTKRP-3 non-root modes j / k
        rows = csf.dims[1] if kind == 6 else csf.dims[2]
        out = np.zeros(rows * R)
        fn = lib.oc_mttkrp3_j if kind == 6 else lib.oc_mttkrp3_k
        fn(C.byref(a.oc), C.c_int64(R), fp[0], fp[1], out.ctypes.data_as(dblp))
    elif kind == 5:
        out = np.zeros(I * R * S * T)
        lib.oc_ttmc4(C.byref(a.oc), C.c_int64(R), C.c_int64(S), C.c_int64(T), fp[0], fp[1], fp[2],
                     out.ctypes.data_as(dblp))
    else:
        raise ValueError(kind)
    return out


def oracle_abs_nest(kind, csf, factors, ranks, residual=False) -> np.ndarray:
    """Per-entry normaliser: sum of |contributions| (nest on |T|, |factors|);
    for the residual, |t| is added."""
    absf = [np.abs(f) for f in factors]
    if kind == 3 and residual:
        unit = csf.with_values(np.ones_like(csf.values))
        return oracle_nest(kind, unit, absf, ranks, residual=False) + np.abs(csf.values)
    return oracle_nest(kind, csf.abs(), absf, ranks, residual=False)


# ---- reference bridge (prepare/execute of any order) ------------------------

def _dims_text(spec_dims: dict) -> bytes:
    return ",".join(f"{k}={v}" for k, v in spec_dims.items()).encode()


def ref_execute(kernel, dims, path, order, csf, factors, out_count, repeats=1):
    lib = ref()
    a = _CsfArgs(csf)
    fs = [np.ascontiguousarray(f, np.float64).ravel() for f in factors]
    fp = (dblp * max(1, len(fs)))(*[f.ctypes.data_as(dblp) for f in fs])
    out = np.zeros(out_count)
    stats = (C.c_int64 * 18)()
    secs = C.c_double()
    rc = lib.ref_execute(kernel.encode(), _dims_text(dims), path.encode(), order.encode(),
                         C.c_int(csf.order), a.sizes, a.idx_p, a.ptr_p, a.vals_p, fp,
                         out.ctypes.data_as(dblp), C.c_int64(out_count), stats, C.c_int(18),
                         C.byref(secs), C.c_int(repeats))
    if rc != 0:
        raise RuntimeError(f"ref_execute rc={rc}: {lib.ref_last_error().decode()}")
    nb = stats[1]
    return out, {"multiply_adds": stats[0], "buffer_resets": list(stats[2:2 + nb]),
                 "seconds": secs.value}


def ref_unfactorized(kernel, dims, csf, factors, out_count):
    lib = ref()
    a = _CsfArgs(csf)
    fs = [np.ascontiguousarray(f, np.float64).ravel() for f in factors]
    fp = (dblp * max(1, len(fs)))(*[f.ctypes.data_as(dblp) for f in fs])
    out = np.zeros(out_count)
    madds = C.c_int64()
    secs = C.c_double()
    rc = lib.ref_execute_unfactorized(kernel.encode(), _dims_text(dims), C.c_int(csf.order),
                                      a.sizes, a.idx_p, a.ptr_p, a.vals_p, fp,
                                      out.ctypes.data_as(dblp), C.c_int64(out_count),
                                      C.byref(madds), C.byref(secs))
    if rc != 0:
        raise RuntimeError(f"ref_unfactorized rc={rc}: {lib.ref_last_error().decode()}")
    return out, madds.value


def ref_execute_threads(kernel, dims, path, order, csf, factors, out_count, nthreads, repeats=1):
    lib = ref()
    a = _CsfArgs(csf)
    fs = [np.ascontiguousarray(f, np.float64).ravel() for f in factors]
    fp = (dblp * max(1, len(fs)))(*[f.ctypes.data_as(dblp) for f in fs])
    out = np.zeros(out_count)
    secs = C.c_double()
    rc = lib.ref_execute_threads(kernel.encode(), _dims_text(dims), path.encode(), order.encode(),
                                 C.c_int(csf.order), a.sizes, a.idx_p, a.ptr_p, a.vals_p, fp,
                                 out.ctypes.data_as(dblp), C.c_int64(out_count), C.c_int(nthreads),
                                 C.c_int(repeats), C.byref(secs))
    if rc != 0:
        raise RuntimeError(f"ref_execute_threads rc={rc}: {lib.ref_last_error().decode()}")
    return out, secs.value


def ref_gen_random_csf(names, dims, density, seed):
    lib = ref()
    d = len(dims)
    h = lib.ref_gen_random_csf(d, ",".join(names).encode(), (C.c_int64 * d)(*dims),
                               C.c_double(density), C.c_uint64(seed))
    return _ref_csf_arrays(h, d)


def ref_build_csf(names, dims, coords, values, mode_order):
    lib = ref()
    d = len(dims)
    coords = np.ascontiguousarray(coords, np.int64)
    values = np.ascontiguousarray(values, np.float64)
    lib.ref_build_csf.argtypes = [C.c_int, C.c_char_p, i64p, C.c_int64, i64p, dblp, C.c_char_p]
    h = lib.ref_build_csf(d, ",".join(names).encode(), (C.c_int64 * d)(*dims),
                          C.c_int64(values.shape[0]), coords.ctypes.data_as(i64p),
                          values.ctypes.data_as(dblp), ",".join(mode_order).encode())
    return _ref_csf_arrays(h, d)


def _ref_csf_arrays(h, d):
    lib = ref()
    if not h:
        raise RuntimeError(lib.ref_last_error().decode())
    idx, ptr = [], []
    for l in range(d):
        n = lib.ref_csf_level_size(h, l)
        a = np.zeros(n, np.int64)
        p = np.zeros(n + 1, np.int64) if l + 1 < d else None
        lib.ref_csf_copy(h, l, a.ctypes.data_as(i64p), p.ctypes.data_as(i64p) if p is not None else None)
        idx.append(a)
        if p is not None:
            ptr.append(p)
    vals = np.zeros(len(idx[-1]))
    lib.ref_csf_values(h, vals.ctypes.data_as(dblp))
    lib.ref_csf_free(h)
    return idx, ptr, vals


def ref_gen_dense(names, dims, seed):
    lib = ref()
    d = len(dims)
    out = np.zeros(int(np.prod(dims)))
    lib.ref_gen_dense(d, ",".join(names).encode(), (C.c_int64 * d)(*dims), C.c_uint64(seed),
                      out.ctypes.data_as(dblp))
    return out


def ref_enumerate(kernel, dims, all_paths=False):
    lib = ref()
    buf = C.create_string_buffer(1 << 24)
    n = lib.ref_enumerate(kernel.encode(), _dims_text(dims), C.c_int(1 if all_paths else 0), buf,
                          C.c_int64(1 << 24))
    if n < 0:
        raise RuntimeError(lib.ref_last_error().decode())
    return [tuple(line.split("|")) for line in buf.value.decode().splitlines()]
