"""ctypes bindings for the in-tree native libraries.

libspttn_b200.so   — the CUDA engine behind the C-ABI in include/spttn_b200.h
libspttn_datagen.so — host-side synthetic tensor generators / COO->CSF

The engine library is mandatory: importing the device API when it is
missing raises immediately (there is no CPU fallback for the hot path).
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_DIR = Path(__file__).resolve().parent / "lib"

c_i64 = C.c_int64
c_i32 = C.c_int32
c_dbl_p = C.POINTER(C.c_double)
c_i64_p = C.POINTER(C.c_int64)


class CsfHost(C.Structure):
    _fields_ = [
        ("order", c_i32),
        ("dims", c_i64_p),
        ("level_size", c_i64_p),
        ("idx", C.POINTER(c_i64_p)),
        ("ptr", C.POINTER(c_i64_p)),
        ("values", c_dbl_p),
    ]


class PlanDesc(C.Structure):
    _fields_ = [
        ("kind", c_i32),
        ("flags", c_i32),
        ("rank", c_i64 * 3),
        ("num_factors", c_i32),
        ("factors", c_dbl_p * 8),
        ("factor_size", c_i64 * 8),
        ("buffer_limit_bytes", c_i64),
        ("program", C.c_void_p),
        ("program_bytes", c_i64),
    ]


class UnfactDesc(C.Structure):
    _fields_ = [
        ("num_indices", c_i32),
        ("dims", c_i64 * 32),
        ("csf_level", c_i32 * 32),
        ("num_free", c_i32),
        ("free_ids", c_i32 * 32),
        ("num_factors", c_i32),
        ("factor_order", c_i32 * 8),
        ("factor_ids", (c_i32 * 8) * 8),
        ("factors", c_dbl_p * 8),
        ("out_sparse", c_i32),
        ("out_order", c_i32),
        ("out_ids", c_i32 * 8),
    ]


# exported C-ABI symbols (include/spttn_b200.h), checked by the CPU tests
ENGINE_SYMBOLS = [
    "spttn_last_error", "spttn_csf_create", "spttn_csf_create_async", "spttn_csf_destroy", "spttn_csf_level_size",
    "spttn_csf_device_bytes", "spttn_plan_create", "spttn_plan_destroy",
    "spttn_plan_set_factors", "spttn_execute", "spttn_execute_stage", "spttn_output_count", "spttn_output_device",
    "spttn_read_output", "spttn_plan_info", "spttn_generic_resets", "spttn_generic_log_bytes",
    "spttn_generic_read_log", "spttn_unfactorized", "spttn_device_info", "spttn_build_info",
    "spttn_release_cached", "spttn_init", "spttn_synchronize", "spttn_csf_from_coo", "spttn_csf_download",
    "spttn_csf_dim", "spttn_csf_permute", "spttn_plan_item_clocks",
]

_engine = None
_datagen = None


def _load(name: str) -> C.CDLL:
    path = LIB_DIR / name
    if not path.exists():
        raise RuntimeError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the SpTTN hot path has no CPU fallback)")
    return C.CDLL(str(path), mode=C.RTLD_GLOBAL)


def engine() -> C.CDLL:
    global _engine
    if _engine is None:
        # SPTTN_DEBUG_BOUNDS=1: the bounds-checked build (device SPTTN_DCHECKs)
        lib = _load("debug/libspttn_b200.so" if os.environ.get("SPTTN_DEBUG_BOUNDS") == "1"
                    else "libspttn_b200.so")
        P = C.c_void_p
        lib.spttn_last_error.restype = C.c_char_p
        lib.spttn_build_info.restype = C.c_char_p
        lib.spttn_csf_create.argtypes = [C.POINTER(CsfHost), P, C.POINTER(P)]
        lib.spttn_csf_create_async.argtypes = [C.POINTER(CsfHost), P, C.POINTER(P)]
        lib.spttn_csf_destroy.argtypes = [P]
        lib.spttn_csf_level_size.argtypes = [P, C.c_int]
        lib.spttn_csf_level_size.restype = c_i64
        lib.spttn_csf_device_bytes.argtypes = [P]
        lib.spttn_csf_device_bytes.restype = c_i64
        lib.spttn_plan_create.argtypes = [C.POINTER(PlanDesc), P, P, C.POINTER(P)]
        lib.spttn_plan_destroy.argtypes = [P]
        lib.spttn_plan_set_factors.argtypes = [P, C.POINTER(c_dbl_p), c_i32, P]
        lib.spttn_execute.argtypes = [P, P]
        lib.spttn_execute_stage.argtypes = [P, C.c_int, P]
        lib.spttn_output_count.argtypes = [P]
        lib.spttn_output_count.restype = c_i64
        lib.spttn_output_device.argtypes = [P]
        lib.spttn_output_device.restype = C.c_void_p
        lib.spttn_read_output.argtypes = [P, c_dbl_p, c_i64, P]
        lib.spttn_plan_info.argtypes = [P, c_i64_p, C.c_int]
        lib.spttn_plan_item_clocks.argtypes = [P, c_i64_p, c_i64]
        lib.spttn_generic_resets.argtypes = [P, c_i64_p, C.c_int]
        lib.spttn_generic_log_bytes.argtypes = [P]
        lib.spttn_generic_log_bytes.restype = c_i64
        lib.spttn_generic_read_log.argtypes = [P, C.c_void_p, c_i64, P]
        lib.spttn_unfactorized.argtypes = [C.POINTER(UnfactDesc), P, c_dbl_p, c_i64, P]
        lib.spttn_device_info.argtypes = [c_i64_p, C.c_int]
        lib.spttn_synchronize.argtypes = [P]
        lib.spttn_csf_from_coo.argtypes = [C.c_int, c_i64_p, c_i64, c_i64_p, c_dbl_p, P,
                                           C.POINTER(P)]
        lib.spttn_csf_download.argtypes = [P, C.POINTER(c_i64_p), C.POINTER(c_i64_p), c_dbl_p, P]
        lib.spttn_csf_dim.argtypes = [P, C.c_int]
        lib.spttn_csf_permute.argtypes = [P, C.POINTER(C.c_int), P, C.POINTER(P)]
        lib.spttn_csf_dim.restype = c_i64
        _engine = lib
    return _engine


def datagen() -> C.CDLL:
    global _datagen
    if _datagen is None:
        lib = _load("libspttn_datagen.so")
        P = C.c_void_p
        lib.dg_last_error.restype = C.c_char_p
        lib.dg_stable_hash.argtypes = [C.c_char_p]
        lib.dg_stable_hash.restype = C.c_uint64
        lib.dg_csf_order.argtypes = [P]
        lib.dg_csf_level_size.argtypes = [P, C.c_int]
        lib.dg_csf_level_size.restype = c_i64
        lib.dg_csf_dim.argtypes = [P, C.c_int]
        lib.dg_csf_dim.restype = c_i64
        lib.dg_csf_idx.argtypes = [P, C.c_int]
        lib.dg_csf_idx.restype = c_i64_p
        lib.dg_csf_ptr.argtypes = [P, C.c_int]
        lib.dg_csf_ptr.restype = c_i64_p
        lib.dg_csf_values.argtypes = [P]
        lib.dg_csf_values.restype = c_dbl_p
        lib.dg_csf_free.argtypes = [P]
        lib.dg_csf_from_coo.argtypes = [C.c_int, c_i64_p, c_i64, c_i64_p, c_dbl_p]
        lib.dg_csf_from_coo.restype = P
        lib.dg_gen_random.argtypes = [C.c_int, c_i64_p, C.c_double, C.c_uint64]
        lib.dg_gen_random.restype = P
        lib.dg_gen_dense.argtypes = [c_i64, C.c_uint64, c_dbl_p]
        lib.dg_gen_normal.argtypes = [c_i64, C.c_uint64, C.c_double, c_dbl_p]
        lib.dg_gen_baseline.argtypes = [C.c_int, c_i64_p, c_i64, C.c_double, C.c_uint64]
        lib.dg_gen_baseline.restype = P
        lib.dg_csf_root_sample.argtypes = [P, c_i64, c_i64]
        lib.dg_csf_root_sample.restype = P
        _datagen = lib
    return _datagen


def libs_present() -> bool:
    return all((LIB_DIR / n).exists() for n in ("libspttn_b200.so", "libspttn_datagen.so"))


def engine_path() -> str:
    return os.fspath(LIB_DIR / "libspttn_b200.so")
