"""Pin the C restatement oracle (oracle/pint_oracle.c) to the UNMODIFIED reference.

Every comparison is bit-exact (np.array_equal on float64) against tests/golden/reference_golden.npz,
which tests/golden/make_golden.py produced from oracle/_ref/ref_tool (reference sources compiled
as-is). Frozen values from the reference's own unit tests are re-checked as well.
"""
import math

import numpy as np
import pytest

import oracle as O


def test_steps_for_matches_reference(golden):
    for w, dt, s in zip(golden["steps_for_width"], golden["steps_for_dt"], golden["steps_for_steps"]):
        assert O.steps_for(w, dt) == s
    # test_ode_core.cpp:25-31
    assert [O.steps_for(0.125, 0.01), O.steps_for(0.125, 1e-4), O.steps_for(0.5, 1e-4),
            O.steps_for(0.3, 0.1), O.steps_for(0.05, 0.1)] == [13, 1250, 5000, 3, 1]


@pytest.mark.parametrize("tag,args", [
    ("dec_4_001", (0.0, 0.5, 4, 0.01)),
    ("dec_64_1em4", (0.0, 0.5, 64, 1e-4)),
    ("dec_7_1em3", (0.0, 0.5, 7, 1e-3)),
    ("dec_3_1em2", (0.0, 0.5, 3, 1e-2)),
    ("dec_heat_256", (0.0, 10.0, 256, 10.0 / 65536.0)),
])
def test_decompose_bit_exact(golden, tag, args):
    tb, te, st, h = O.decompose(*args)
    assert np.array_equal(tb, golden[tag + "_t_begin"])
    assert np.array_equal(te, golden[tag + "_t_end"])
    assert np.array_equal(st, golden[tag + "_steps"])
    assert np.array_equal(h, golden[tag + "_dt"])


def test_decompose_bad_grid():
    with pytest.raises(ValueError):
        O.decompose(0.0, 0.5, 0, 0.01)


def test_riccati_step(golden):
    for y, dt, z in zip(golden["riccati_y"], golden["riccati_dt"], golden["riccati_z"]):
        rc, got = O.riccati_step(y, dt)
        assert rc == 0 and got == z
    assert O.riccati_step(1.0, 0.01)[1] == pytest.approx(1.0102051443364402, rel=1e-15)
    assert O.riccati_step(2.0, 0.25)[0] == 1  # NoRealRoot, test_ode_core.cpp:21-23


@pytest.mark.parametrize("M", [1, 2, 5, 6, 7, 33, 64, 512])
def test_nodes_and_weights(golden, M):
    assert np.array_equal(O.cheb_nodes(M, 0.0, 2.0, kind=2), golden[f"nodes2_{M}"])
    assert np.array_equal(O.cheb_nodes(M, 0.0, 2.0, kind=1), golden[f"nodes1_{M}"])
    if M > 1:
        assert np.array_equal(O.bary_weights(golden[f"nodes2_{M}"]), golden[f"weights2_{M}"])


def test_duplicate_nodes():
    with pytest.raises(ValueError):
        O.bary_weights([0.0, 1.0, 1.0])


def test_interp_eval(golden):
    x = golden["nodes2_33"]
    w = golden["weights2_33"]
    v = golden["interp33_values"]
    got = np.array([O.interp_eval(x, w, v, q) for q in golden["interp33_xi"]])
    assert np.array_equal(got, golden["interp33_out"])


SCALAR_RUNS = [
    ("sc_N4_M5_1em4", 4, 1e-4, 5, 0.0, 2.0),
    ("sc_N4_M6_1em4", 4, 1e-4, 6, 0.0, 2.0),
    ("sc_N4_M7_1em4", 4, 1e-4, 7, 0.0, 2.0),
    ("sc_N64_M6_1em4", 64, 1e-4, 6, 0.0, 2.0),
    ("sc_N8_M6_1em3", 8, 1e-3, 6, 0.0, 2.0),
    ("sc_N16_M33_1em3", 16, 1e-3, 33, 0.0, 2.0),
    ("sc_N64_M64_1em4", 64, 1e-4, 64, 0.0, 2.0),
    ("sc_extrap_N4_M5_1em3", 4, 1e-3, 5, 0.0, 0.5),
]


@pytest.mark.parametrize("tag,N,dt,M,a,b", SCALAR_RUNS)
def test_scalar_run_bit_exact(golden, tag, N, dt, M, a, b):
    tb, te, st, h = O.decompose(0.0, 0.5, N, dt)
    x = O.cheb_nodes(M, a, b)
    ends, fail, _ = O.riccati_ensemble(st, h, x)
    assert fail == -1
    assert np.array_equal(ends, golden[tag + "_endpoints"])
    w = O.bary_weights(x)
    y, lam, ext = O.scalar_sweep(x, w, ends, a, b, 1.0)
    assert np.array_equal(lam, golden[tag + "_lambdas"])
    assert y == golden[tag + "_final"][0]
    assert ext == golden[tag + "_extrapolation_count"][0]
    assert abs(y - 1.0 / (1.0 - 0.5)) == golden[tag + "_error_vs_exact"][0]


def test_scalar_M512_final(golden):
    tb, te, st, h = O.decompose(0.0, 0.5, 64, 1e-4)
    x = O.cheb_nodes(512, 0.0, 2.0)
    ends, _, _ = O.riccati_ensemble(st, h, x)
    y, _, _ = O.scalar_sweep(x, O.bary_weights(x), ends, 0.0, 2.0, 1.0)
    assert y == golden["sc_N64_M512_1em4_final"][0]


def test_frozen_unit_test_errors(golden):
    # test_nievergelt.cpp:31-45 (5e-3 relative) and SURVEY §8c full-precision probes
    assert golden["sc_N4_M5_1em4_error_vs_exact"][0] == pytest.approx(5.061e-5, rel=5e-3)
    assert golden["sc_N4_M6_1em4_error_vs_exact"][0] == pytest.approx(2.9623e-4, rel=5e-3)
    assert golden["sc_N4_M7_1em4_error_vs_exact"][0] == pytest.approx(2.783e-4, rel=5e-3)
    assert golden["sc_N4_M5_1em4_final"][0] == 2.0000506110633056
    assert golden["sc_N64_M6_1em4_final"][0] == 2.0002742994992597


def test_serial_scalar(golden):
    _, _, st, h = O.decompose(0.0, 0.5, 1, 1e-4)
    ends, fail, _ = O.riccati_ensemble(st, h, [1.0])
    assert ends[0, 0] == golden["serial_1em4_final"][0]


def test_table1_grid(golden):
    errs = np.empty((5, 5))
    for r, dt in enumerate([0.01, 0.005, 0.0025, 0.001, 0.0001]):
        _, _, st, h = O.decompose(0.0, 0.5, 4, dt)
        for c, M in enumerate([3, 4, 5, 6, 7]):
            x = O.cheb_nodes(M, 0.0, 2.0)
            ends, _, _ = O.riccati_ensemble(st, h, x)
            y, _, _ = O.scalar_sweep(x, O.bary_weights(x), ends, 0.0, 2.0, 1.0)
            errs[r, c] = abs(y - 2.0)
    assert np.array_equal(errs, golden["table1_errors"])


def test_heat9_build_and_chain(golden):
    tb, te, st, h = O.decompose(0.0, 10.0, 4, 0.005)
    Gs, cs = [], []
    for j in range(4):
        G, c = O.heat_build(0.1, tb[j], te[j], 0.005)
        Gs.append(G)
        cs.append(c)
    assert np.array_equal(np.stack(Gs), golden["heat9_G"])
    assert np.array_equal(np.stack(cs), golden["heat9_c"])
    y = O.affine_chain(np.stack(Gs), np.stack(cs), O.heat_initial(0.1))
    assert np.array_equal(y, golden["heat9_N4_final"])
    serial = O.heat_integrate(0.1, 0.0, 10.0, 0.005, O.heat_initial(0.1))
    assert np.array_equal(serial, golden["heat9_serial_final"])
    assert np.max(np.abs(serial - O.heat_exact(0.1, 10.0))) == golden["heat9_serial_error"][0]
    assert serial[4] == -0.84617156960930295  # SURVEY §8c probe
    direct = O.heat_integrate(0.1, tb[1], te[1], 0.005, golden["heat9_direct_y"])
    assert np.array_equal(direct, golden["heat9_direct_out"])


def test_heat128_slice_and_run(golden):
    dx, dt = 1.0 / 129.0, 10.0 / (16 * 32)
    tb, te, st, h = O.decompose(0.0, 10.0, 16, dt)
    G, c = O.heat_build(dx, tb[5], te[5], dt)
    assert np.array_equal(G, golden["heat128_slice5_G"])
    assert np.array_equal(c, golden["heat128_slice5_c"])
    serial = O.heat_integrate(dx, 0.0, 10.0, dt, O.heat_initial(dx))
    assert np.array_equal(serial, golden["heat128_serial_final"])


def test_linalg(golden):
    n = 12
    sub, sup = np.full(n - 1, -1.0), np.full(n - 1, -1.3)
    diag = 4.0 + 0.1 * np.arange(n)
    rhs = 1.0 / (1.0 + np.arange(n))
    assert np.array_equal(O.thomas(sub, diag, sup, rhs), golden["thomas12_x"])
    A, x = golden["linalg5_A"], golden["linalg5_x"]
    assert np.array_equal(O.matvec(A, x), golden["linalg5_Ax"])
    assert np.array_equal(O.matmul(A, A), golden["linalg5_AA"])
    with pytest.raises(ValueError):
        O.thomas([1.0], [0.0, 1.0], [1.0], [1.0, 1.0])
