"""Parareal on the device (pint_parareal_scalar / pint_parareal_heat) against the UNMODIFIED
reference's parareal_sweep (tests/golden/parareal_golden.npz, made by
tests/golden/make_parareal_golden.py from oracle/_ref/parareal_golden): every iterate
(final_per_iteration) BIT-EXACT, including acceptance criterion 2's table (N in {1..64},
k in {0, 2, 3, 5}) and the heat system of test_parareal.cpp."""
import ctypes as C
import pathlib

import numpy as np
import pytest

from paper_1304_6514_b200 import capi, pint

pytestmark = pytest.mark.gpu

Z = np.load(pathlib.Path(__file__).resolve().parent / "golden" / "parareal_golden.npz")
SCALAR = sorted({k.split("_")[0] for k in Z if k.startswith("scalar")}, key=lambda s: int(s[6:]))
HEAT = sorted({k.split("_")[0] for k in Z if k.startswith("heat")}, key=lambda s: int(s[4:]))


@pytest.fixture(scope="module")
def ctx():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a B200"
    return pint.context()


@pytest.mark.parametrize("case", SCALAR)
def test_parareal_scalar_bit_exact(ctx, case):
    N, k, dt, DT = Z[f"{case}_cfg"]
    N, k = int(N), int(k)
    fin = np.empty(k + 1)
    fine = np.empty(N)
    coarse = C.c_double()
    rep = capi.Report()
    fail = capi.Fail()
    ctx.check(ctx.lib.pint_parareal_scalar(ctx.h, 0.0, 0.5, 1.0, N, k, dt, DT, capi.ptr(fin), capi.ptr(fine),
                                           C.byref(coarse), C.byref(rep), C.byref(fail)))
    assert np.array_equal(fin, Z[f"{case}_finals"]), (case, fin - Z[f"{case}_finals"])
    assert rep.message_count == (2 * k + 1) * (N - 1)
    assert np.all(fine >= 0.0) and coarse.value >= 0.0


@pytest.mark.parametrize("case", HEAT)
def test_parareal_heat_bit_exact(ctx, case):
    dx, T, N, k, dt, DT = Z[f"{case}_cfg"]
    N, k = int(N), int(k)
    n = int(round(1.0 / dx)) - 1
    fin = np.empty((k + 1) * n)
    rep = capi.Report()
    ctx.check(ctx.lib.pint_parareal_heat(ctx.h, dx, T, None, N, k, dt, DT, capi.ptr(fin), C.byref(rep)))
    assert np.array_equal(fin.reshape(k + 1, n), Z[f"{case}_finals"]), case


def test_parareal_no_real_root_is_a_task_failure(ctx):
    """y0 large enough that a fine step has 1 - 4 dt y < 0 in slice 0: NoRealRoot, slice index 0."""
    fin = np.empty(3)
    fail = capi.Fail()
    rc = ctx.lib.pint_parareal_scalar(ctx.h, 0.0, 0.5, 3000.0, 4, 2, 1e-4, 0.1, capi.ptr(fin), None, None, None,
                                      C.byref(fail))
    assert rc == capi.PINT_E_NO_REAL_ROOT
