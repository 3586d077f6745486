"""Python bindings of the device engine (C-ABI in include/spttn_b200.h).

The C++ shim (csrc/shim/executor_b200.cpp) is the reference-facing drop-in
(`spttn::prepare` / `spttn::execute`). This module exposes the same engine to
Python for the parity tests and bench.py:

    csf_dev = DeviceCsf(csf)                       # H2D + device layout
    plan = Plan(NEST_TTMC3, csf_dev, [U, V], ranks=(R, S))
    plan.execute(stream)                           # async on `stream`
    y = plan.read_output()                         # D2H + sync

Errors raise the Python analogue of the reference's exception types
(ValueError ~ std::invalid_argument, UnsupportedOrderError,
ResourceError); CUDA failures raise RuntimeError.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .tensor import Csf

NEST_MTTKRP3 = 1
NEST_TTMC3 = 2
NEST_TTTP3 = 3
NEST_MTTKRP4 = 4
NEST_TTMC4 = 5
NEST_MTTKRP3_J = 6  # T[i,j,k]*A[i,r]*C[k,r]->B[j,r], output on CSF level 1 (atomics)
NEST_MTTKRP3_K = 7  # T[i,j,k]*A[i,r]*B[j,r]->C[k,r], output on CSF level 2 (atomics)
NEST_GENERIC = 100

FLAG_RESIDUAL = 1
FLAG_FACTORS_ON_DEVICE = 2


class UnsupportedOrderError(RuntimeError):
    pass


class ResourceError(RuntimeError):
    pass


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = N.engine().spttn_last_error().decode()
    if rc == 1:
        raise ValueError(msg)
    if rc == 2:
        raise UnsupportedOrderError(msg)
    if rc == 3:
        raise ResourceError(msg)
    raise RuntimeError(f"spttn_b200 CUDA failure: {msg}")


def _stream_ptr(stream) -> C.c_void_p:
    if stream is None:
        return C.c_void_p(0)
    if isinstance(stream, int):
        return C.c_void_p(stream)
    return C.c_void_p(int(stream.cuda_stream))


def device_info() -> dict:
    out = (C.c_int64 * 4)()
    _check(N.engine().spttn_device_info(out, 4))
    return {"sm_count": out[0], "cc": out[1], "l2_bytes": out[2], "smem_optin": out[3]}


def release_cached() -> None:
    """spttn_release_cached: return the engine's cached (unused) device blocks to the driver."""
    _check(N.engine().spttn_release_cached())


class DeviceCsf:
    """spttn_csf_create: copies a host Csf and builds the int32 device layout.
    async_values=True: spttn_csf_create_async (values uploaded in the
    background; keep csf.values alive until a plan on it has been created)."""

    def __init__(self, csf: Csf, stream=None, async_values: bool = False):
        lib = N.engine()
        self.csf = csf
        d = csf.order
        self._dims = (C.c_int64 * d)(*csf.dims)
        self._sizes = (C.c_int64 * d)(*csf.level_sizes())
        self._keep = [np.ascontiguousarray(a, np.int64) for a in csf.idx + csf.ptr]
        idx_p = (N.c_i64_p * d)(*[a.ctypes.data_as(N.c_i64_p) for a in self._keep[:d]])
        ptr_p = (N.c_i64_p * max(1, d - 1))(*[a.ctypes.data_as(N.c_i64_p) for a in self._keep[d:]])
        vals = np.ascontiguousarray(csf.values, np.float64)
        host = N.CsfHost(d, self._dims, self._sizes, idx_p, ptr_p, vals.ctypes.data_as(N.c_dbl_p))
        h = C.c_void_p()
        fn = lib.spttn_csf_create_async if async_values else lib.spttn_csf_create
        _check(fn(C.byref(host), _stream_ptr(stream), C.byref(h)))
        self.handle = h
        self._keep = [vals] if async_values else None

    @classmethod
    def from_root_range(cls, csf: Csf, r0: int, r1: int, stream=None,
                        async_values: bool = False) -> "DeviceCsf":
        """Root slices [r0, r1) of a host Csf as a device CSF, passed as a
        zero-copy view into csf's arrays (spttn_csf_host views: ptr[l][0] may
        be non-zero, the device layout is rebased). Output rows keep their
        global numbering."""
        lib = N.engine()
        d = csf.order
        lo, hi = [r0], [r1]
        for l in range(d - 1):
            lo.append(int(csf.ptr[l][lo[-1]]))
            hi.append(int(csf.ptr[l][hi[-1]]))
        arrs = [np.ascontiguousarray(a, np.int64) for a in csf.idx + csf.ptr]
        vals = np.ascontiguousarray(csf.values, np.float64)
        self = cls.__new__(cls)
        self.csf = None
        self._dims = (C.c_int64 * d)(*csf.dims)
        self._sizes = (C.c_int64 * d)(*[hi[l] - lo[l] for l in range(d)])
        idx_p = (N.c_i64_p * d)(*[C.cast(arrs[l].ctypes.data + 8 * lo[l], N.c_i64_p)
                                  for l in range(d)])
        ptr_p = (N.c_i64_p * max(1, d - 1))(*[C.cast(arrs[d + l].ctypes.data + 8 * lo[l], N.c_i64_p)
                                              for l in range(d - 1)])
        host = N.CsfHost(d, self._dims, self._sizes, idx_p, ptr_p,
                         C.cast(vals.ctypes.data + 8 * lo[d - 1], N.c_dbl_p))
        h = C.c_void_p()
        fn = lib.spttn_csf_create_async if async_values else lib.spttn_csf_create
        _check(fn(C.byref(host), _stream_ptr(stream), C.byref(h)))
        self.handle = h
        self._keep = [arrs, vals] if async_values else None
        self.leaf_range = (lo[d - 1], hi[d - 1])
        return self

    @classmethod
    def from_coo(cls, dims, coords: np.ndarray, values: np.ndarray, stream=None) -> "DeviceCsf":
        """spttn_csf_from_coo: normalize + build_csf on the GPU (rows in CSF
        mode order, nnz x order int64); the host Csf is not materialised."""
        lib = N.engine()
        coords = np.ascontiguousarray(coords, np.int64).reshape(-1, len(dims))
        values = np.ascontiguousarray(values, np.float64)
        if coords.shape[0] != values.shape[0]:
            raise ValueError("coords / values length mismatch")
        dd = (C.c_int64 * len(dims))(*dims)
        h = C.c_void_p()
        _check(lib.spttn_csf_from_coo(len(dims), dd, int(values.shape[0]),
                                      coords.ctypes.data_as(N.c_i64_p),
                                      values.ctypes.data_as(N.c_dbl_p), _stream_ptr(stream),
                                      C.byref(h)))
        self = cls.__new__(cls)
        self.csf = None
        self.handle = h
        self._keep = None
        return self

    def permute(self, order, stream=None) -> "DeviceCsf":
        """spttn_csf_permute: the same tensor with levels in `order` (new level
        l = current level order[l]), rebuilt on the device."""
        lib = N.engine()
        o = (C.c_int * len(order))(*order)
        h = C.c_void_p()
        _check(lib.spttn_csf_permute(self.handle, o, _stream_ptr(stream), C.byref(h)))
        out = DeviceCsf.__new__(DeviceCsf)
        out.csf = None
        out.handle = h
        out._keep = None
        return out

    def level_sizes(self):
        lib = N.engine()
        sizes = []
        for l in range(8):
            n = int(lib.spttn_csf_level_size(self.handle, l))
            if n < 0:
                break
            sizes.append(n)
        return sizes

    def download(self, stream=None) -> Csf:
        """spttn_csf_download: the reference's int64 CSF arrays back on the host."""
        lib = N.engine()
        sizes = self.level_sizes()
        d = len(sizes)
        dims = [int(lib.spttn_csf_dim(self.handle, l)) for l in range(d)]
        idx = [np.empty(n, np.int64) for n in sizes]
        ptr = [np.empty(sizes[l] + 1, np.int64) for l in range(d - 1)]
        vals = np.empty(sizes[-1] if sizes else 0, np.float64)
        ip = (N.c_i64_p * d)(*[a.ctypes.data_as(N.c_i64_p) for a in idx])
        pp = (N.c_i64_p * max(1, d - 1))(*[a.ctypes.data_as(N.c_i64_p) for a in ptr])
        _check(lib.spttn_csf_download(self.handle, ip, pp, vals.ctypes.data_as(N.c_dbl_p),
                                      _stream_ptr(stream)))
        return Csf(dims, idx, ptr, vals)

    def device_bytes(self) -> int:
        return int(N.engine().spttn_csf_device_bytes(self.handle))

    def close(self):
        if getattr(self, "handle", None):
            N.engine().spttn_csf_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Plan:
    """spttn_plan_create: one fused nest bound to a device CSF and factors.

    factors: numpy fp64 arrays (copied) or, with on_device=True, integer
    device pointers (e.g. torch tensor .data_ptr()) that outlive the plan.
    """

    def __init__(self, kind: int, csf: DeviceCsf, factors, ranks=(0, 0, 0), flags: int = 0,
                 stream=None, on_device: bool = False, factor_sizes=None, program=None,
                 buffer_limit_bytes: int = 1 << 30):
        lib = N.engine()
        self.csf = csf
        desc = N.PlanDesc()
        desc.kind = kind
        desc.flags = flags | (FLAG_FACTORS_ON_DEVICE if on_device else 0)
        for i, r in enumerate(list(ranks)[:3]):
            desc.rank[i] = int(r)
        desc.num_factors = len(factors)
        self._factors = []
        for f, a in enumerate(factors):
            if on_device:
                desc.factors[f] = C.cast(C.c_void_p(int(a)), N.c_dbl_p)
                desc.factor_size[f] = int(factor_sizes[f])
            else:
                arr = np.ascontiguousarray(a, np.float64).ravel()
                self._factors.append(arr)
                desc.factors[f] = arr.ctypes.data_as(N.c_dbl_p)
                desc.factor_size[f] = arr.shape[0]
        desc.buffer_limit_bytes = buffer_limit_bytes
        self._program = program
        if program is not None:
            desc.program = C.cast(C.byref(program), C.c_void_p)
            desc.program_bytes = C.sizeof(program)
        h = C.c_void_p()
        _check(lib.spttn_plan_create(C.byref(desc), csf.handle, _stream_ptr(stream), C.byref(h)))
        self.handle = h
        self._factors = None
        self.kind = kind

    @property
    def output_count(self) -> int:
        return int(N.engine().spttn_output_count(self.handle))

    @property
    def output_ptr(self) -> int:
        return int(N.engine().spttn_output_device(self.handle) or 0)

    def output_tensor(self):
        """The plan's device output as a torch CUDA tensor (zero-copy view via
        __cuda_array_interface__; valid while the plan lives), e.g. for NCCL
        collectives on it (distributed.py)."""
        import torch

        class _View:
            def __init__(self, ptr, n):
                self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8",
                                                 "data": (ptr, False), "version": 3,
                                                 "strides": None}
        n = self.output_count
        if n == 0:
            return torch.zeros(0, dtype=torch.float64, device="cuda")
        return torch.as_tensor(_View(self.output_ptr, n), device="cuda")

    def info(self) -> dict:
        out = (C.c_int64 * 11)()
        _check(N.engine().spttn_plan_info(self.handle, out, 11))
        keys = ["launches", "items", "split_slices", "absent_rows", "scratch_bytes", "kind",
                "segments", "device_madds", "generic_mode", "generic_jit", "variant"]
        return dict(zip(keys, list(out)))

    def item_clocks(self) -> np.ndarray:
        """Diagnostics: per work item [start ns, end ns, SM id, groups, leaf
        steps, tile flushes] of the last execute (plans created with
        SPTTN_ITEM_CLOCKS=1; packed TTMc-3)."""
        n = self.info()["items"]
        out = np.zeros(6 * n, np.int64)
        _check(N.engine().spttn_plan_item_clocks(self.handle, out.ctypes.data_as(N.c_i64_p), out.size))
        return out.reshape(n, 6)

    def set_factors(self, factors, stream=None, on_device=False):
        arrs = []
        ptrs = (N.c_dbl_p * 8)()
        for f, a in enumerate(factors):
            if on_device:
                ptrs[f] = C.cast(C.c_void_p(int(a)), N.c_dbl_p)
            else:
                arr = np.ascontiguousarray(a, np.float64).ravel()
                arrs.append(arr)
                ptrs[f] = arr.ctypes.data_as(N.c_dbl_p)
        _check(N.engine().spttn_plan_set_factors(self.handle, ptrs, int(on_device),
                                                 _stream_ptr(stream)))
        if not on_device:  # host copies are async: keep them alive until the stream drains
            import torch
            (torch.cuda.synchronize() if stream is None else stream.synchronize())

    def execute(self, stream=None) -> None:
        _check(N.engine().spttn_execute(self.handle, _stream_ptr(stream)))

    def execute_stage(self, stage: int, stream=None) -> None:
        """0 = fused nest kernel, 1 = epilogue (fix-up / absent rows)."""
        _check(N.engine().spttn_execute_stage(self.handle, stage, _stream_ptr(stream)))

    def read_output(self, stream=None, out: np.ndarray | None = None) -> np.ndarray:
        n = self.output_count
        if out is None:
            out = np.empty(n, dtype=np.float64)
        _check(N.engine().spttn_read_output(self.handle, out.ctypes.data_as(N.c_dbl_p), n,
                                            _stream_ptr(stream)))
        return out

    def close(self):
        if getattr(self, "handle", None):
            N.engine().spttn_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass



def _parse_kernel(text: str):
    """Index ids of a kernel-spec string the way the reference's parse_kernel
    assigns them (first appearance over the inputs, proj/src/kernel_spec.cpp:
    103-156): returns ([(name, [index names])...] inputs, output names,
    sparse_out)."""
    body = text.replace(" ", "")
    sparse_out = body.endswith("@sparse_out")
    if sparse_out:
        body = body[: -len("@sparse_out")]
    lhs, rhs = body.split("->")

    def tensor(tok):
        name, rest = tok.split("[")
        return name, [x for x in rest.rstrip("]").split(",") if x]
    return [tensor(t) for t in lhs.split("*")], tensor(rhs)[1], sparse_out


def unfactorized(kernel: str, dims: dict, csf: DeviceCsf, factors, stream=None) -> np.ndarray:
    """spttn_unfactorized: the reference's execute_unfactorized oracle nest
    (executor.cpp:522-626) on the device for a kernel-spec string, factors in
    kernel input order (host arrays, row-major). Same descriptor the C++
    drop-in builds; bit-identical to the reference."""
    lib = N.engine()
    inputs, out_idx, sparse_out = _parse_kernel(kernel)
    names = []
    for _, ix in inputs:
        for n in ix:
            if n not in names:
                names.append(n)
    d = N.UnfactDesc()
    d.num_indices = len(names)
    sparse = inputs[0][1]
    for k, n in enumerate(names):
        d.dims[k] = int(dims[n])
        d.csf_level[k] = sparse.index(n) if n in sparse else -1
    free = [n for _, ix in inputs for n in ix if n not in sparse]
    free = list(dict.fromkeys(free))  # first appearance (executor.cpp:530-537)
    d.num_free = len(free)
    for q, n in enumerate(free):
        d.free_ids[q] = names.index(n)
    d.num_factors = len(inputs) - 1
    keep = []
    for f, (_, ix) in enumerate(inputs[1:]):
        d.factor_order[f] = len(ix)
        for k, n in enumerate(ix):
            d.factor_ids[f][k] = names.index(n)
        a = np.ascontiguousarray(factors[f], np.float64).ravel()
        keep.append(a)
        d.factors[f] = a.ctypes.data_as(N.c_dbl_p)
    d.out_sparse = 1 if sparse_out else 0
    d.out_order = len(out_idx)
    for k, n in enumerate(out_idx):
        d.out_ids[k] = names.index(n)
    if sparse_out:
        count = csf.level_sizes()[-1]
    else:
        count = int(np.prod([int(dims[n]) for n in out_idx])) if out_idx else 1
    out = np.empty(count, np.float64)
    _check(lib.spttn_unfactorized(C.byref(d), csf.handle, out.ctypes.data_as(N.c_dbl_p), count,
                                  _stream_ptr(stream)))
    return out
