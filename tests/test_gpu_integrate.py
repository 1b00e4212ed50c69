"""GPU parity of the integrate closure / run_serial path (heat.cu heat_integrate_kernel, chunked
records) against the C oracle (oracle/pint_oracle.c, pinned to the reference): bit-exact.

The reference's integrate closure is make_heat_problem's (pde_problems.cpp:86-98); run_serial
(nievergelt.cpp:126-143) is one such integration over [t0, T]. These check: many caller columns
(several warps), both forcing modes, step counts that are not multiples of the record chunk, the
full C2 serial interval (65536 steps, the length the drop-in's run_nievergelt integrates), the
guarded re-run on a subnormal range trip, and the background serial run (pint_heat_serial_begin/
_end) concurrently with a parallel run on the same context.
"""
import ctypes as C

import numpy as np
import pytest

import oracle as O
from paper_1304_6514_b200 import capi, pint

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a B200"
    return pint.context()


@pytest.mark.parametrize("n,K,steps,forcing", [(9, 1, 5, True), (128, 1, 300, True), (128, 70, 77, False),
                                               (97, 33, 41, True), (300, 5, 20, True), (512, 2, 9, False)])
def test_integrate_bit_exact(ctx, n, K, steps, forcing):
    rng = np.random.default_rng(n * 1000 + K)
    dx, dt = 1.0 / (n + 1), 2e-4
    s = pint.TimeSlice(0, 0.3, 0.3 + steps * dt, steps, dt)
    y = rng.uniform(-1, 1, (K, n))
    got = pint.heat_integrate(dx, s, y, dt, forcing)
    for k in range(K):
        want = O.heat_integrate(dx, s.t_begin, s.t_end, dt, y[k], forcing)
        assert np.array_equal(got[k], want), k


def test_integrate_chunk_boundaries(ctx):
    """n = 128: chunk = 2^21 / record_stride(128) = 4032 steps; 9000 steps cross two boundaries."""
    n, steps = 128, 9000
    dx, dt = 1.0 / (n + 1), 1e-4
    s = pint.TimeSlice(0, 0.0, steps * dt, steps, dt)
    y0 = np.asarray(pint.heat_initial(dx))
    got = pint.heat_integrate(dx, s, y0, dt, True)
    assert np.array_equal(got, O.heat_integrate(dx, s.t_begin, s.t_end, dt, y0, True))


def test_serial_c2_length_bit_exact(ctx):
    """run_serial at config 2's resolution (n = 128, 65536 steps over [0, 10])."""
    n, N, S = 128, 256, 256
    dx, dt = 1.0 / (n + 1), 10.0 / (N * S)
    prob = pint.make_heat_problem(dx, dt, 10.0)
    got = pint.run_serial(prob).final_state
    want = O.heat_integrate(dx, 0.0, 10.0, dt, prob.y0, True)
    assert np.array_equal(got, want)


def test_integrate_underflow_retries_guarded(ctx):
    """dt = 1e-9 at n = 128 drives e_k columns through the subnormal range in the first step: the
    fast division's range check trips and the guarded re-run is bit-exact."""
    n, dt = 128, 1e-9
    dx = 1.0 / (n + 1)
    s = pint.TimeSlice(0, 0.0, 6 * dt, 6, dt)
    y = np.eye(n)[:40]
    got = pint.heat_integrate(dx, s, y, dt, False)
    for k in range(40):
        want = O.heat_integrate(dx, s.t_begin, s.t_end, dt, y[k], False)
        assert np.array_equal(got[k], want), k
    assert np.count_nonzero((got != 0) & (np.abs(got) < 2.3e-308)) > 0  # subnormals really occur


def test_background_serial_with_parallel_run(ctx):
    """pint_heat_serial_begin, a full parallel run on the same context, pint_heat_serial_end: both
    results bit-exact (the serial run's failure record and stream are its own)."""
    n, N, S = 128, 64, 32
    dx, dt, T = 1.0 / (n + 1), 10.0 / (N * S), 10.0
    prob = pint.make_heat_problem(dx, dt, T)
    y0 = np.ascontiguousarray(prob.y0)
    ctx.check(ctx.lib.pint_heat_serial_begin(ctx.h, dx, dt, T, capi.ptr(y0)))
    y = np.empty(n)
    rep = capi.Report()
    ctx.check(ctx.lib.pint_run_heat(ctx.h, dx, dt, T, N, capi.COMPOSE_CHAIN, capi.ptr(y0), capi.ptr(y), None,
                                    C.byref(rep)))
    ys = np.empty(n)
    ctx.check(ctx.lib.pint_heat_serial_end(ctx.h, capi.ptr(ys)))
    assert np.array_equal(ys, O.heat_integrate(dx, 0.0, T, dt, y0, True))
    dec = pint.decompose(0.0, T, N, dt)
    G = np.empty((N, n, n))
    c = np.empty((N, n))
    for j, s in enumerate(dec.slices):
        G[j], c[j] = O.heat_build(dx, s.t_begin, s.t_end, dt)
    assert np.array_equal(y, O.affine_chain(G, c, y0))
    assert ctx.lib.pint_heat_serial_end(ctx.h, capi.ptr(ys)) == capi.PINT_E_INVALID  # nothing in flight


def test_drop_in_run_nievergelt_c2_wall(ctx):
    """The drop-in's run_nievergelt at config 2 (serial reference run included, in the background)
    is bit-exact against the reference's golden final state; its wall time is reported."""
    import pathlib
    import time

    z = np.load(pathlib.Path(__file__).resolve().parent / "golden" / "heat_finals.npz")
    n, N, S = (int(v) for v in z["c2_config"])
    dx, dt = 1.0 / (n + 1), 10.0 / (N * S)
    prob = pint.make_heat_problem(dx, dt, 10.0)
    pint.run_nievergelt(prob, N, pint.ExecConfig())  # warm
    t0 = time.perf_counter()
    r = pint.run_nievergelt(prob, N, pint.ExecConfig())
    wall = time.perf_counter() - t0
    assert np.array_equal(r.final_state, z["c2_final"])
    assert r.error_vs_serial <= 1e-10
    print(f"drop-in run_nievergelt C2 wall {wall:.3f} s (T_total {r.T_total:.4f} s)")
    assert wall < 0.8  # the reference's run_serial + T_total on 16 host cores is ~0.87 s
