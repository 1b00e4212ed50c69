"""CPU-side checks of the drop-in boundary: libpint_cuda.so loads without a GPU, exports every
function include/pint_cuda.h declares, and its host-side table functions (decompose, steps_for,
sample_nodes) are bit-identical to the reference (via the pinned oracle). No compute calls."""
import pathlib
import re

import numpy as np
import pytest

import oracle as O
from paper_1304_6514_b200 import capi, pint

ROOT = pathlib.Path(__file__).resolve().parents[1]


def declared_functions():
    text = (ROOT / "include" / "pint_cuda.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pint_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = capi.load()
    names = declared_functions()
    assert len(names) >= 30
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(capi.EXPORTED)


def test_version_string():
    assert "sm_100a" in capi.version()


def test_no_device_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(capi.PintError):
        capi.Context(0)


@pytest.mark.parametrize("args", [(0.0, 0.5, 4, 0.01), (0.0, 0.5, 64, 1e-4), (0.0, 0.5, 7, 1e-3),
                                  (0.0, 10.0, 256, 10.0 / 65536), (0.0, 10.0, 4096, 10.0 / 65536)])
def test_host_decompose_is_the_reference(args):
    dec = pint.decompose(*args)
    tb, te, st, h = O.decompose(*args)
    assert np.array_equal([s.t_begin for s in dec.slices], tb)
    assert np.array_equal([s.t_end for s in dec.slices], te)
    assert np.array_equal([s.steps for s in dec.slices], st)
    assert np.array_equal([s.dt for s in dec.slices], h)


def test_host_nodes_are_the_reference(golden):
    for M in (1, 2, 5, 6, 7, 33, 64, 512):
        assert np.array_equal(pint.cheb_nodes_second_kind(M, 0.0, 2.0), golden[f"nodes2_{M}"])
        assert np.array_equal(pint.cheb_nodes(M, 0.0, 2.0), golden[f"nodes1_{M}"])


def test_host_steps_for(golden):
    for w, dt, s in zip(golden["steps_for_width"], golden["steps_for_dt"], golden["steps_for_steps"]):
        assert pint.steps_for(w, dt) == s


def test_heat_coefficient_tables_match_reference_arithmetic():
    """The per-step tables the device consumes equal the reference's in-loop values."""
    import ctypes as C
    import math

    dx, dt, T, N = 0.1, 0.005, 10.0, 4
    dec = pint.decompose(0.0, T, N, dt)
    arr = (capi.Slice * N)(*[s.c() for s in dec.slices])
    Q = sum(s.steps for s in dec.slices)
    off = np.empty(N + 1, dtype=np.int64)
    r, fa, fb = (np.empty(Q) for _ in range(3))
    sx = np.empty(9)
    n = C.c_int64()
    assert capi.load().pint_heat_coefficients(dx, arr, N, capi.ptr(off), capi.ptr(r), capi.ptr(fa),
                                              capi.ptr(fb), capi.ptr(sx), C.byref(n)) == 0
    assert n.value == 9 and off[-1] == Q
    s = dec.slices[2]
    for i in (1, 7, s.steps):
        t = s.t_begin + i * s.dt
        q = off[2] + i - 1
        assert r[q] == s.dt * O.lib().or_heat_coefficient(t) * (1.0 / (dx * dx))
        for k in range(9):
            x = (k + 1) * dx
            b = fa[q] * sx[k] + fb[q] * sx[k]
            assert b == O.lib().or_heat_forcing(x, t)


def test_affine_ldm():
    assert [capi.load().pint_affine_ldm(n) for n in (1, 3, 4, 9, 128, 512)] == [4, 4, 8, 12, 132, 516]


def test_host_pool_back_to_back_jobs_from_threads():
    """The host thread pool behind the table fills (capi.cu HostPool): many back-to-back
    parallel_for jobs, from several caller threads at once, each result identical to a serial
    reference — a worker waking late must never run a finished job's function — and a fork of
    the process runs the fill serially instead of waiting on workers it does not have. (In a child
    process: the pool's threads must not live in the pytest process, which later forks gloo ranks.)"""
    import subprocess
    import sys

    code = r"""
import ctypes as C, sys, threading
import numpy as np
sys.path.insert(0, ".")
from paper_1304_6514_b200 import capi, pint
dx, T, N = 1.0 / 129, 10.0, 512
dt = T / (N * 16)
dec = pint.decompose(0.0, T, N, dt)
arr = (capi.Slice * N)(*[s.c() for s in dec.slices])
Q = sum(s.steps for s in dec.slices)  # >= 4096 steps: the pool path
def fill():
    off = np.empty(N + 1, dtype=np.int64)
    r, fa, fb = (np.empty(Q) for _ in range(3))
    sx = np.empty(128)
    n = C.c_int64()
    assert capi.load().pint_heat_coefficients(dx, arr, N, capi.ptr(off), capi.ptr(r), capi.ptr(fa),
                                              capi.ptr(fb), capi.ptr(sx), C.byref(n)) == 0
    return r, fa, fb
ref = fill()
bad = []
def worker():
    for _ in range(60):
        if not all(np.array_equal(a, b) for a, b in zip(fill(), ref)):
            bad.append(1)
ts = [threading.Thread(target=worker) for _ in range(4)]
for t in ts: t.start()
for t in ts: t.join()
import os
pid = os.fork()  # a forked child has none of the pool's workers: it must run the fill serially
if pid == 0:
    os._exit(0 if all(np.array_equal(a, b) for a, b in zip(fill(), ref)) else 1)
_, st = os.waitpid(pid, 0)
sys.exit(1 if bad or st != 0 else 0)
"""
    root = str(__import__("pathlib").Path(__file__).resolve().parents[1])
    subprocess.run([sys.executable, "-c", code], cwd=root, check=True, timeout=300)
