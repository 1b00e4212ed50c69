"""B200-native Nievergelt slice-map solver (drop-in for the reference pint path).

Layout: csrc/ (sm_100a kernels + C ABI -> libpint_cuda.so), host/ + include/pint/ (C++ drop-in of
the reference's pint:: API -> libpint_b200.so), capi.py (ctypes binding), pint.py (Python mirror
of the reference API), dist.py (slice-block sharding over torch.distributed).
"""
from . import capi  # noqa: F401

__all__ = ["capi"]
