"""B200-native SpTTN fused-nest execution engine (arXiv 2307.05740 hot path).

Native pieces (built in-tree by __graft_entry__.build()):
  lib/libspttn_b200.so       sm_100a kernels + C-ABI (include/spttn_b200.h)
  lib/libspttn_b200_host.so  C++ drop-in for spttn::prepare / execute
  lib/libspttn_datagen.so    host generators / COO->CSF
This package is the Python view of the same engine (tests, bench.py).
"""
from .engine import (FLAG_FACTORS_ON_DEVICE, FLAG_RESIDUAL, NEST_GENERIC, NEST_MTTKRP3,
                     NEST_MTTKRP3_J, NEST_MTTKRP3_K, NEST_MTTKRP4, NEST_TTMC3, NEST_TTMC4,
                     NEST_TTTP3, DeviceCsf, Plan,
                     ResourceError, UnsupportedOrderError, device_info, release_cached,
                     unfactorized)
from .tensor import Csf, gen_dense, gen_normal, stable_hash

__all__ = [
    "Csf", "DeviceCsf", "Plan", "device_info", "release_cached", "unfactorized", "gen_dense", "gen_normal", "stable_hash",
    "NEST_MTTKRP3", "NEST_TTMC3", "NEST_TTTP3", "NEST_MTTKRP4", "NEST_TTMC4", "NEST_GENERIC",
    "NEST_MTTKRP3_J", "NEST_MTTKRP3_K",
    "FLAG_RESIDUAL", "FLAG_FACTORS_ON_DEVICE", "UnsupportedOrderError", "ResourceError",
]
