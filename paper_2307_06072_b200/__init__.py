"""B200-native (sm_100a) Ozaki-scheme complex multiple-precision GEMM (arXiv 2307.06072).

The hot path lives in libmpcgemm.so (csrc/*.cu, C ABI in include/mpcgemm.h); this package
is the thin Python binding (mpcgemm.py) and the multi-GPU driver (dist.py).
"""
from .mpcgemm import (DevCMat, DevRMat, MpcgemmError, empty_device, gemm, lib, mpcgemm_device_rule_result,
                      mpcgemm_ex, mpcgemm_host, mpcgemm_host_async, mpcgemm_host_wait,
                      mpcgemm_release, mpcgemm_rho_bounds, mpcgemm_slices_for, mpcgemm_strerror,
                      mpcgemm_version, mpcgemm_workspace_size, mpc_scalar, mpclu_factor, mpclu_solve, to_device,
                      to_host)

__all__ = ["DevCMat", "DevRMat", "MpcgemmError", "empty_device", "gemm", "lib", "mpcgemm_device_rule_result",
           "mpcgemm_ex", "mpcgemm_host",
           "mpcgemm_host_async", "mpcgemm_host_wait",
           "mpcgemm_release", "mpcgemm_rho_bounds", "mpcgemm_slices_for", "mpcgemm_strerror",
           "mpcgemm_version", "mpcgemm_workspace_size", "mpc_scalar", "mpclu_factor", "mpclu_solve", "to_device",
           "to_host"]
