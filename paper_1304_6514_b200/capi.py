"""ctypes binding of libpint_cuda.so (include/pint_cuda.h).

The library is the only compute path: if it is missing or no CUDA device is present every call
raises — there is no CPU fallback. Device-pointer entry points accept torch CUDA tensors (torch
is used for device memory and streams only).
"""
from __future__ import annotations

import ctypes as C
import os
import pathlib

HERE = pathlib.Path(__file__).resolve().parent
LIB_PATH = HERE / "libpint_cuda.so"

PINT_OK = 0
PINT_E_NO_REAL_ROOT = 1
PINT_E_SINGULAR = 2
PINT_E_BAD_GRID = 3
PINT_E_NON_INTEGER_STEPS = 4
PINT_E_DUPLICATE_NODES = 5
PINT_E_RANGE_RETRY = 6
PINT_E_SERIALIZED = 7
PINT_E_INVALID = 16
PINT_E_CUDA = 17
PINT_E_NO_DEVICE = 18
PINT_E_NCCL = 19

RHS_RICCATI_BE = 0
RHS_LOGISTIC_RK4 = 1
F64, F32 = 0, 1
WEIGHTS_PRODUCT, WEIGHTS_CLOSED2 = 0, 1
SWEEP_EXACT, SWEEP_TREE = 0, 1
COMPOSE_CHAIN, COMPOSE_TREE = 0, 1
BUILD_EXACT, BUILD_FAST = 0, 1
NODES_FIRST_KIND, NODES_SECOND_KIND = 0, 1


class PintError(RuntimeError):
    """A non-OK status from libpint_cuda.so; `.code` is the PINT_E_* value."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[pint code {code}] {msg}")
        self.code = code


class Slice(C.Structure):
    _fields_ = [("t_begin", C.c_double), ("t_end", C.c_double), ("steps", C.c_int64), ("dt", C.c_double)]


class Fail(C.Structure):
    _fields_ = [("index", C.c_int64), ("code", C.c_int32), ("pad", C.c_int32), ("value", C.c_double)]


class ScalarRHS(C.Structure):
    _fields_ = [("kind", C.c_int32), ("precision", C.c_int32), ("r", C.c_double), ("K", C.c_double)]


class Report(C.Structure):
    _fields_ = [
        ("message_count", C.c_int64), ("bytes_communicated", C.c_int64),
        ("extrapolation_count", C.c_int64), ("device_ms", C.c_double), ("total_ms", C.c_double),
        ("traj_steps", C.c_int64), ("gpu_launches", C.c_int64), ("h2d_bytes", C.c_int64),
        ("d2h_bytes", C.c_int64), ("compose_ms", C.c_double),
    ]


_vp, _d, _i, _int = C.c_void_p, C.c_double, C.c_int64, C.c_int
# pint_send_fn / pint_recv_fn: int (*)(void* user, int peer, [const] void* buf, size_t bytes)
SEND_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_size_t)
RECV_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_size_t)
_SIGS = {
    "pint_version": (C.c_char_p, []),
    "pint_device_count": (_int, []),
    "pint_ctx_create": (_int, [_int, C.POINTER(_vp)]),
    "pint_ctx_destroy": (None, [_vp]),
    "pint_ctx_last_error": (C.c_char_p, [_vp]),
    "pint_ctx_sync": (_int, [_vp]),
    "pint_ctx_stream": (_vp, [_vp]),
    "pint_ctx_set_stream": (_int, [_vp, _vp]),
    "pint_ctx_launch_count": (_i, [_vp]),
    "pint_fail_read": (_int, [_vp, C.POINTER(Fail)]),
    "pint_debug_fail_inject": (_int, [_vp, _i, _vp, _vp, _vp]),
    "pint_steps_for": (_i, [_d, _d]),
    "pint_decompose": (_int, [_d, _d, _i, _d, C.POINTER(Slice)]),
    "pint_sample_nodes": (_int, [_int, _i, _d, _d, _vp]),
    "pint_affine_ldm": (_i, [_i]),
    "pint_scalar_ensemble_dev": (_int, [_vp, C.POINTER(ScalarRHS), _i, _i, _vp, _vp, _vp, _vp, _vp]),
    "pint_bary_weights_dev": (_int, [_vp, _int, _i, _vp, _vp]),
    "pint_scalar_sweep_dev": (_int, [_vp, _int, _i, _i, _vp, _i, _vp, _vp, _vp, _vp, _i, _d, _vp, _vp, _vp]),
    "pint_heat_total_steps": (_i, [C.POINTER(Slice), _i]),
    "pint_heat_coefficients": (_int, [_d, C.POINTER(Slice), _i, _vp, _vp, _vp, _vp, _vp, C.POINTER(_i)]),
    "pint_heat_records_size": (_i, [_i, _i, _i]),
    "pint_heat_factor_dev": (_int, [_vp, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "pint_heat_build_dev": (_int, [_vp, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _int]),
    "pint_heat_fast_records_size": (_i, [_i, _i, _i]),
    "pint_heat_fast_factor_dev": (_int, [_vp, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "pint_heat_fast_build_dev": (_int, [_vp, _i, _i, _i, _vp, _vp]),
    "pint_heat_integrate_dev": (_int, [_vp, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _int, _vp, _int]),
    "pint_heat_serial_begin": (_int, [_vp, _d, _d, _d, _vp]),
    "pint_heat_serial_end": (_int, [_vp, _vp]),
    "pint_heat_build_chain_dev": (_int, [_vp, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _int]),
    "pint_heat_fast_build_chain_dev": (_int, [_vp, _i, _i, _i, _vp, _vp, _vp, _vp]),
    "pint_ctx_build_chain_ms": (_int, [_vp, C.POINTER(_d), C.POINTER(_d)]),
    "pint_affine_compose_dev": (_int, [_vp, _int, _i, _i, _vp, _vp, _vp, _vp, _vp]),
    "pint_affine_pair_dev": (_int, [_vp, _i, _i, _vp, _vp, _vp]),
    "pint_lv_ensemble_dev": (_int, [_vp, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp]),
    "pint_bilinear_sweep_dev": (_int, [_vp, _i, _i, _i, _vp, _vp, _vp, _d, _d, _vp, _vp, _vp]),
    "pint_run_scalar": (_int, [_vp, C.POINTER(ScalarRHS), _d, _d, _d, _i, _d, _int, _i, _d, _d, _int, _int,
                               _vp, _vp, _vp, _vp, C.POINTER(Report), C.POINTER(Fail)]),
    "pint_run_heat": (_int, [_vp, _d, _d, _d, _i, _int, _vp, _vp, _vp, C.POINTER(Report)]),
    "pint_run_heat_ex": (_int, [_vp, _d, _d, _d, _i, _int, _int, _vp, _vp, _vp, C.POINTER(Report)]),
    "pint_parareal_scalar": (_int, [_vp, _d, _d, _d, _i, _i, _d, _d, _vp, _vp, _vp, C.POINTER(Report),
                                     C.POINTER(Fail)]),
    "pint_parareal_heat": (_int, [_vp, _d, _d, _vp, _i, _i, _d, _d, _vp, C.POINTER(Report)]),
    "pint_comm_unique_id": (_int, [_vp]),
    "pint_comm_init": (_int, [_vp, _vp, _int, _int]),
    "pint_comm_init_all": (_int, [C.POINTER(_vp), _int]),
    "pint_comm_init_callbacks": (_int, [_vp, _int, _int, SEND_FN, RECV_FN, _vp]),
    "pint_comm_rank": (_int, [_vp, C.POINTER(_int), C.POINTER(_int)]),
    "pint_comm_destroy": (_int, [_vp]),
    "pint_run_heat_sharded": (_int, [_vp, _d, _d, _d, _i, _int, _int, _vp, _vp, C.POINTER(Report)]),
    "pint_heat_maps": (_int, [_vp, _d, _d, C.POINTER(Slice), _i, _vp, _vp]),
    "pint_heat_integrate": (_int, [_vp, _d, C.POINTER(Slice), _d, _int, _i, _vp]),
    "pint_scalar_integrate": (_int, [_vp, C.POINTER(ScalarRHS), C.POINTER(Slice), _i, _vp, _vp, C.POINTER(Fail)]),
    "pint_affine_compose": (_int, [_vp, _int, _i, _i, _vp, _vp, _vp, _vp]),
    "pint_scalar_sweep": (_int, [_vp, _int, _i, _i, _vp, _i, _vp, _vp, _vp, _vp, _i, _d, _vp, _vp, _vp]),
    "pint_wave_maps": (_int, [_vp, _i, _vp, _d, C.POINTER(Slice), _i, _d, _vp, _vp]),
    "pint_wave_integrate": (_int, [_vp, _i, _vp, _d, C.POINTER(Slice), _d, _i, _vp]),
    "pint_run_wave": (_int, [_vp, _i, _vp, _d, _d, _i, _d, _int, _vp, _vp, _vp, C.POINTER(Report)]),
    "pint_bary_weights": (_int, [_vp, _int, _i, _vp, _vp]),
    "pint_probe_peak": (_int, [_vp, _int, C.POINTER(_d)]),
    "pint_probe_latency": (_int, [_vp, _vp]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load():
    """Load libpint_cuda.so (raises if it has not been built: no fallback exists)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback)")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def ptr(x) -> int | None:
    """Device/host pointer of a torch tensor or numpy array (None passes through)."""
    if x is None:
        return None
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if hasattr(x, "ctypes"):
        return x.ctypes.data
    return int(x)


class Context:
    """Owns one pint_ctx (device, stream, scratch, failure record)."""

    def __init__(self, device: int = 0, stream=None):
        self.lib = load()
        h = C.c_void_p()
        rc = self.lib.pint_ctx_create(device, C.byref(h))
        if rc != PINT_OK:
            raise PintError(rc, "pint_ctx_create failed (no CUDA device?)")
        self.h = h
        self.device = device
        if stream is not None:
            self.set_stream(stream)

    def close(self):
        if getattr(self, "h", None):
            self.lib.pint_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def check(self, rc: int):
        if rc != PINT_OK:
            raise PintError(rc, self.lib.pint_ctx_last_error(self.h).decode())

    def set_stream(self, stream):
        handle = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        self.check(self.lib.pint_ctx_set_stream(self.h, handle))

    def stream_handle(self) -> int:
        return self.lib.pint_ctx_stream(self.h)

    def sync(self):
        self.check(self.lib.pint_ctx_sync(self.h))

    def launches(self) -> int:
        return int(self.lib.pint_ctx_launch_count(self.h))

    def fail(self) -> Fail:
        f = Fail()
        self.check(self.lib.pint_fail_read(self.h, C.byref(f)))
        return f

    def call(self, name: str, *args):
        self.check(getattr(self.lib, name)(self.h, *args))


def version() -> str:
    return load().pint_version().decode()


def lib_path() -> str:
    return os.fspath(LIB_PATH)
