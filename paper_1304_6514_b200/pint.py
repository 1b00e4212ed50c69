"""Host-side mirror of the reference's pint:: API for the slice-map path, in Python.

Same names, argument meaning and error behaviour as /root/reference/proj/include/pint/
(nievergelt.hpp:78-106, ode_core.hpp:15-63, interp.hpp:9-36, exec_harness.hpp:15-112,
pde_problems.hpp:13-25, errors.hpp:9-43), so parity tests read like the reference's own tests.
Every numerical call goes through libpint_cuda.so (capi.py); host code here only does what the
reference does on its coordinator thread besides computing: report assembly, the simulated
wire's sleeps/counters, and the modeled schedule.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import math
import time
from typing import Callable, List, Optional, Sequence, Union

import numpy as np

from . import capi

# ---- errors (errors.hpp:9-43) ------------------------------------------------------------------


class NoRealRoot(RuntimeError):
    pass


class SingularSystem(RuntimeError):
    pass


class BadGrid(RuntimeError):
    pass


class NonIntegerStepCount(RuntimeError):
    pass


class DuplicateNodes(RuntimeError):
    pass


class TaskFailure(RuntimeError):
    def __init__(self, index: int, what: str):
        super().__init__(f"task {index}: {what}")
        self.task_index = index


_CODE_TO_EXC = {
    capi.PINT_E_NO_REAL_ROOT: NoRealRoot,
    capi.PINT_E_SINGULAR: SingularSystem,
    capi.PINT_E_BAD_GRID: BadGrid,
    capi.PINT_E_NON_INTEGER_STEPS: NonIntegerStepCount,
    capi.PINT_E_DUPLICATE_NODES: DuplicateNodes,
}

_ctx: Optional[capi.Context] = None


def context() -> capi.Context:
    """The process-wide device context (cuda:0 unless set_context was called)."""
    global _ctx
    if _ctx is None:
        _ctx = capi.Context(0)
    return _ctx


def set_context(ctx: capi.Context) -> None:
    global _ctx
    _ctx = ctx


def _check(rc: int, ctx: capi.Context, fail: Optional[capi.Fail] = None):
    if rc == capi.PINT_OK:
        return
    msg = ctx.lib.pint_ctx_last_error(ctx.h).decode()
    exc = _CODE_TO_EXC.get(rc)
    if fail is not None and fail.index >= 0:  # a task failed: parallel_map's wrapping
        raise TaskFailure(int(fail.index), msg)
    if exc is not None:
        raise exc(msg)
    raise capi.PintError(rc, msg)


# ---- exec harness (exec_harness.hpp:15-45, exec_harness.cpp:7-13) -------------------------------

MEASURED, MODELED, BOTH = "measured", "modeled", "both"


@dataclasses.dataclass
class ExecConfig:
    workers: int = 1                  # the device replaces the pool; kept for report parity
    latency_per_receive: float = 0.0  # seconds slept per simulated receive
    clock: str = BOTH


class Stopwatch:
    def __init__(self):
        self.t0 = time.perf_counter()

    def seconds(self) -> float:
        return time.perf_counter() - self.t0


def inject_latency(seconds: float) -> None:
    if seconds > 0.0:
        time.sleep(seconds)


def modeled_time_nievergelt(per_slice_compute: Sequence[float], latency: float, apply_cost: float) -> float:
    if len(per_slice_compute) == 0:
        return 0.0
    n_msgs = float(len(per_slice_compute) - 1)
    return max(per_slice_compute) + n_msgs * latency + n_msgs * apply_cost


# ---- ode core (ode_core.hpp:15-63) -------------------------------------------------------------


@dataclasses.dataclass
class ScalarIVP:
    """y' = f(t, y) on [t0, T]. `kind` selects the device stepper: the reference runs backward-
    Euler Riccati whatever rhs says (nievergelt.cpp:28-35); "logistic_rk4" is an EXTENSION."""
    rhs: Optional[Callable[[float, float], float]] = None
    t0: float = 0.0
    T: float = 1.0
    y0: float = 0.0
    exact: Optional[Callable[[float], float]] = None
    kind: str = "riccati_be"
    r: float = 1.0
    K: float = 1.0
    precision: str = "f64"

    def device_rhs(self) -> capi.ScalarRHS:
        kind = {"riccati_be": capi.RHS_RICCATI_BE, "logistic_rk4": capi.RHS_LOGISTIC_RK4}[self.kind]
        return capi.ScalarRHS(kind, capi.F32 if self.precision == "f32" else capi.F64, self.r, self.K)


def make_model_problem() -> ScalarIVP:
    """y' = y^2, y(0) = 1 on [0, 0.5]; exact 1/(1 - t) (ode_core.cpp:8-16)."""
    return ScalarIVP(rhs=lambda t, y: y * y, t0=0.0, T=0.5, y0=1.0, exact=lambda t: 1.0 / (1.0 - t))


def make_logistic_problem(r: float = 1.0, K: float = 1.0, y0: float = 0.1, T: float = 10.0,
                          precision: str = "f64") -> ScalarIVP:
    """EXTENSION (config 1): y' = r y (1 - y/K), RK4; exact logistic solution."""
    def exact(t):
        e = math.exp(r * t)
        return K * y0 * e / (K + y0 * (e - 1.0))
    return ScalarIVP(rhs=lambda t, y: r * y * (1 - y / K), t0=0.0, T=T, y0=y0, exact=exact,
                     kind="logistic_rk4", r=r, K=K, precision=precision)


@dataclasses.dataclass
class TimeSlice:
    index: int = 0
    t_begin: float = 0.0
    t_end: float = 0.0
    steps: int = 1
    dt: float = 0.0

    def c(self) -> capi.Slice:
        return capi.Slice(self.t_begin, self.t_end, self.steps, self.dt)


@dataclasses.dataclass
class TimeSliceDecomposition:
    N: int = 1
    t0: float = 0.0
    T: float = 0.0
    dt_nominal: float = 0.0
    slices: List[TimeSlice] = dataclasses.field(default_factory=list)


def steps_for(width: float, dt: float) -> int:
    return int(capi.load().pint_steps_for(width, dt))


def decompose(t0: float, T: float, N: int, dt: float) -> TimeSliceDecomposition:
    if N <= 0 or not (T > t0) or not (dt > 0.0):
        raise BadGrid("decompose: need N >= 1, T > t0, dt > 0")
    arr = (capi.Slice * N)()
    rc = capi.load().pint_decompose(t0, T, N, dt, arr)
    if rc:
        raise BadGrid("decompose: need N >= 1, T > t0, dt > 0")
    return TimeSliceDecomposition(N, t0, T, dt, [TimeSlice(j, s.t_begin, s.t_end, s.steps, s.dt)
                                                 for j, s in enumerate(arr)])


def slice_table(dec: TimeSliceDecomposition):
    """(steps int64[N], dt float64[N]) — the slice assignment shipped to the device."""
    return (np.array([s.steps for s in dec.slices], dtype=np.int64),
            np.array([s.dt for s in dec.slices], dtype=np.float64))


# ---- interpolation (interp.hpp:9-36) -----------------------------------------------------------

FIRST_KIND, SECOND_KIND = "first_kind", "second_kind"


def sample_nodes(kind: str, M: int, a: float, b: float) -> np.ndarray:
    out = np.empty(M)
    rc = capi.load().pint_sample_nodes(capi.NODES_FIRST_KIND if kind == FIRST_KIND else capi.NODES_SECOND_KIND,
                                       M, a, b, capi.ptr(out))
    if rc:
        raise BadGrid("cheb_nodes: M >= 1 required")
    return out


def cheb_nodes(M: int, a: float, b: float) -> np.ndarray:
    return sample_nodes(FIRST_KIND, M, a, b)


def cheb_nodes_second_kind(M: int, a: float, b: float) -> np.ndarray:
    return sample_nodes(SECOND_KIND, M, a, b)


@dataclasses.dataclass
class InterpolantData:
    nodes: np.ndarray
    weights: np.ndarray
    values: np.ndarray
    a: float = 0.0
    b: float = 0.0


def barycentric_weights(nodes, kind: str = "product") -> np.ndarray:
    """Product-form weights on the device (interp.cpp:43-55); kind="closed2" is the EXTENSION."""
    import torch

    ctx = context()
    x = torch.as_tensor(np.ascontiguousarray(nodes, dtype=np.float64), device=f"cuda:{ctx.device}")
    w = torch.empty_like(x)
    ctx.call("pint_bary_weights_dev", capi.WEIGHTS_CLOSED2 if kind == "closed2" else capi.WEIGHTS_PRODUCT,
             len(x), capi.ptr(x), capi.ptr(w))
    ctx.sync()
    f = ctx.fail()
    if f.index >= 0:
        raise DuplicateNodes("barycentric_weights: repeated node")
    return w.cpu().numpy()


def make_interpolant(nodes, values, a: float, b: float, weights: str = "product") -> InterpolantData:
    nodes = np.ascontiguousarray(nodes, dtype=np.float64)
    return InterpolantData(nodes, barycentric_weights(nodes, weights),
                           np.ascontiguousarray(values, dtype=np.float64), a, b)


def interp_eval(f: InterpolantData, xi: float) -> float:
    """interp_eval (interp.cpp:68-80) as a one-slice device sweep."""
    y, _, _ = _scalar_sweep([f], xi)
    return y


# ---- slice maps and reports (nievergelt.hpp:17-91) ---------------------------------------------


@dataclasses.dataclass
class InitialValueSpace:
    a: float = 0.0
    b: float = 2.0
    M: int = 6
    kind: str = SECOND_KIND
    weights: str = "product"   # "closed2": EXTENSION, finite for M > 512
    sweep: str = "exact"       # "tree": EXTENSION warp-tree barycentric sums


@dataclasses.dataclass
class SliceMap:
    slice_index: int
    interpolant: InterpolantData


@dataclasses.dataclass
class AffinePropagator:
    slice_index: int
    G: np.ndarray
    c: np.ndarray


@dataclasses.dataclass
class SweepStats:
    T_comm: float = 0.0
    message_count: int = 0
    bytes_communicated: int = 0
    extrapolation_count: int = 0
    apply_cost: float = 0.0


@dataclasses.dataclass
class RunReport:
    final_state: np.ndarray = dataclasses.field(default_factory=lambda: np.empty(0))
    error_vs_exact: Optional[float] = None
    error_vs_serial: Optional[float] = None
    T_total: float = 0.0
    T_comm: float = 0.0
    modeled_time: Optional[float] = None
    message_count: int = 0
    bytes_communicated: int = 0
    per_slice_compute: List[float] = dataclasses.field(default_factory=list)
    extrapolation_count: int = 0
    method: str = ""
    N: int = 1
    M: int = 0
    k: int = 0
    dt: float = 0.0
    DT: float = 0.0
    latency: float = 0.0
    workers: int = 1
    device_ms: float = 0.0
    traj_steps: int = 0
    gpu_launches: int = 0


@dataclasses.dataclass
class LinearProblem:
    """The heat problem as both methods consume it (nievergelt.hpp:66-74). `integrate` runs on the
    device; `dx` is the device-describable spec the opaque reference closure lacks."""
    dim: int = 0
    t0: float = 0.0
    T: float = 0.0
    dt: float = 0.0
    y0: np.ndarray = dataclasses.field(default_factory=lambda: np.empty(0))
    exact_final: Optional[np.ndarray] = None
    name: str = ""
    dx: float = 0.0

    def integrate(self, s: TimeSlice, y, step_nominal: float, with_forcing: bool) -> np.ndarray:
        return heat_integrate(self.dx, s, y, step_nominal, with_forcing)


def heat_coefficient(t: float) -> float:
    return 1.0 + 0.25 * math.sin(t)


def _heat_dim(dx: float) -> int:
    inv = 1.0 / dx
    m = int(round(inv))
    if m < 2 or abs(inv - m) > 1e-9 * inv:
        raise BadGrid(f"make_heat_system: 1/dx must be an integer >= 2, got dx = {dx:f}")
    return m - 1


def heat_initial(dx: float) -> np.ndarray:
    n = _heat_dim(dx)
    return np.array([math.sin(math.pi * ((i + 1) * dx)) for i in range(n)])


def heat_exact(dx: float, t: float) -> np.ndarray:
    n = _heat_dim(dx)
    return np.array([math.cos(t) * math.sin(math.pi * ((i + 1) * dx)) for i in range(n)])


def make_heat_problem(dx: float, dt: float, T: float) -> LinearProblem:
    n = _heat_dim(dx)
    return LinearProblem(dim=n, t0=0.0, T=T, dt=dt, y0=heat_initial(dx), exact_final=heat_exact(dx, T),
                         name="heat", dx=dx)


def heat_integrate(dx: float, s: TimeSlice, y, step_nominal: float, with_forcing: bool) -> np.ndarray:
    """make_heat_problem's integrate closure (pde_problems.cpp:86-98) on the device. y may be one
    state (n,) or K states (K, n)."""
    ctx = context()
    arr = np.array(y, dtype=np.float64, copy=True, order="C")
    K = 1 if arr.ndim == 1 else arr.shape[0]
    sl = s.c()
    _check(ctx.lib.pint_heat_integrate(ctx.h, dx, C.byref(sl), step_nominal, int(with_forcing), K,
                                       capi.ptr(arr)), ctx)
    return arr


# ---- builders and sweeps (nievergelt.cpp:41-110) -----------------------------------------------


def _scalar_integrate_many(ivp: ScalarIVP, y0s, t_begin: float, t_end: float, dt: float) -> np.ndarray:
    """integrate_scalar (nievergelt.cpp:29-35) for K initial values, on the device."""
    ctx = context()
    n = steps_for(t_end - t_begin, dt)
    sl = capi.Slice(t_begin, t_end, n, (t_end - t_begin) / n)
    y0s = np.ascontiguousarray(y0s, dtype=np.float64)
    out = np.empty_like(y0s)
    fail = capi.Fail()
    rhs = ivp.device_rhs()
    rc = ctx.lib.pint_scalar_integrate(ctx.h, C.byref(rhs), C.byref(sl), len(y0s), capi.ptr(y0s),
                                       capi.ptr(out), C.byref(fail))
    _check(rc, ctx, fail if fail.index >= 0 and len(y0s) > 1 else None)
    return out


def build_scalar_slice_map(ivp: ScalarIVP, s: TimeSlice, space: InitialValueSpace, dt: float) -> SliceMap:
    nodes = sample_nodes(space.kind, space.M, space.a, space.b)
    ends = _scalar_integrate_many(ivp, nodes, s.t_begin, s.t_end, dt)
    return SliceMap(s.index, make_interpolant(nodes, ends, space.a, space.b, space.weights))


def build_affine_propagator(problem: LinearProblem, s: TimeSlice) -> AffinePropagator:
    ctx = context()
    n = problem.dim
    G = np.empty((n, n))
    c = np.empty(n)
    sl = s.c()
    _check(ctx.lib.pint_heat_maps(ctx.h, problem.dx, problem.dt, C.byref(sl), 1, capi.ptr(G), capi.ptr(c)), ctx)
    return AffinePropagator(s.index, G, c)


def build_affine_propagators(problem: LinearProblem, dec: TimeSliceDecomposition):
    """All slices in one device launch: (G[N, n, n], c[N, n])."""
    ctx = context()
    N, n = len(dec.slices), problem.dim
    arr = (capi.Slice * N)(*[s.c() for s in dec.slices])
    G = np.empty((N, n, n))
    c = np.empty((N, n))
    _check(ctx.lib.pint_heat_maps(ctx.h, problem.dx, problem.dt, arr, N, capi.ptr(G), capi.ptr(c)), ctx)
    return G, c


def _scalar_sweep(maps: Sequence[InterpolantData], y0: float, mode: str = "exact"):
    ctx = context()
    N = len(maps)
    M = len(maps[0].nodes)
    nodes = np.ascontiguousarray(np.stack([m.nodes for m in maps]), dtype=np.float64)
    weights = np.ascontiguousarray(np.stack([m.weights for m in maps]), dtype=np.float64)
    values = np.ascontiguousarray(np.stack([m.values for m in maps]), dtype=np.float64)
    a = np.array([m.a for m in maps])
    b = np.array([m.b for m in maps])
    lam = np.empty(N)
    y = C.c_double()
    ext = C.c_longlong()
    rc = ctx.lib.pint_scalar_sweep(ctx.h, capi.SWEEP_TREE if mode == "tree" else capi.SWEEP_EXACT, N, M,
                                   capi.ptr(nodes), M, capi.ptr(weights), capi.ptr(values), capi.ptr(a),
                                   capi.ptr(b), 1, y0, capi.ptr(lam), C.byref(y), C.byref(ext))
    _check(rc, ctx)
    return y.value, lam, int(ext.value)


def compose_sweep(maps, y0, latency: float, stats: SweepStats):
    """compose_sweep for SliceMap or AffinePropagator lists (nievergelt.cpp:68-110). The maps are
    applied on the device; the simulated wire (sleep + counters) stays on the host."""
    if len(maps) == 0:
        return y0
    affine = isinstance(maps[0], AffinePropagator)
    n = len(maps[0].c) if affine else 1
    for _ in range(len(maps) - 1):
        sw = Stopwatch()
        inject_latency(latency)
        stats.T_comm += sw.seconds() if latency > 0.0 else 0.0
        stats.message_count += 1
        stats.bytes_communicated += 8 * n
    sw = Stopwatch()
    if affine:
        ctx = context()
        G = np.ascontiguousarray(np.stack([m.G for m in maps]), dtype=np.float64)
        c = np.ascontiguousarray(np.stack([m.c for m in maps]), dtype=np.float64)
        y0a = np.ascontiguousarray(y0, dtype=np.float64)
        y = np.empty(n)
        _check(ctx.lib.pint_affine_compose(ctx.h, capi.COMPOSE_CHAIN, n, len(maps), capi.ptr(G), capi.ptr(c),
                                           capi.ptr(y0a), capi.ptr(y)), ctx)
        out = y
    else:
        out, _, ext = _scalar_sweep([m.interpolant for m in maps], float(y0))
        stats.extrapolation_count += ext
    stats.apply_cost = sw.seconds() / len(maps)
    return out


# ---- full runs (nievergelt.cpp:112-265) --------------------------------------------------------


def run_serial(problem: Union[ScalarIVP, LinearProblem], dt: Optional[float] = None) -> RunReport:
    r = RunReport(method="serial", N=1)
    if isinstance(problem, LinearProblem):
        r.dt = problem.dt
        n = steps_for(problem.T - problem.t0, problem.dt)
        whole = TimeSlice(0, problem.t0, problem.T, n, (problem.T - problem.t0) / n)
        sw = Stopwatch()
        r.final_state = problem.integrate(whole, problem.y0, problem.dt, True)
        r.T_total = sw.seconds()
        r.per_slice_compute = [r.T_total]
        if problem.exact_final is not None:
            r.error_vs_exact = float(np.max(np.abs(r.final_state - problem.exact_final)))
        return r
    ivp = problem
    r.dt = dt
    sw = Stopwatch()
    y = float(_scalar_integrate_many(ivp, [ivp.y0], ivp.t0, ivp.T, dt)[0])
    r.T_total = sw.seconds()
    r.final_state = np.array([y])
    r.per_slice_compute = [r.T_total]
    if ivp.exact is not None:
        r.error_vs_exact = abs(y - ivp.exact(ivp.T))
    return r


def run_nievergelt(problem: Union[ScalarIVP, LinearProblem], N: int, *args, compose: str = "chain") -> RunReport:
    """run_nievergelt(ivp, N, dt, space, exec) or run_nievergelt(problem, N, exec)."""
    if isinstance(problem, LinearProblem):
        exec_ = args[0] if args else ExecConfig()
        return _run_linear(problem, N, exec_, compose)
    dt, space = args[0], args[1]
    exec_ = args[2] if len(args) > 2 else ExecConfig()
    return _run_scalar(problem, N, dt, space, exec_)


def _run_scalar(ivp: ScalarIVP, N: int, dt: float, space: InitialValueSpace, exec_: ExecConfig) -> RunReport:
    if N <= 1:
        r = run_serial(ivp, dt)
        r.method = "nievergelt"
        r.workers = exec_.workers
        return r
    y_serial = float(_scalar_integrate_many(ivp, [ivp.y0], ivp.t0, ivp.T, dt)[0])  # outside the timer
    ctx = context()
    r = RunReport(method="nievergelt", N=N, M=space.M, dt=dt, latency=exec_.latency_per_receive,
                  workers=exec_.workers)
    total = Stopwatch()
    rhs = ivp.device_rhs()
    y = C.c_double()
    per_slice = np.zeros(N)
    rep = capi.Report()
    fail = capi.Fail()
    rc = ctx.lib.pint_run_scalar(ctx.h, C.byref(rhs), ivp.t0, ivp.T, ivp.y0, N, dt,
                                 capi.NODES_FIRST_KIND if space.kind == FIRST_KIND else capi.NODES_SECOND_KIND,
                                 space.M, space.a, space.b,
                                 capi.WEIGHTS_CLOSED2 if space.weights == "closed2" else capi.WEIGHTS_PRODUCT,
                                 capi.SWEEP_TREE if space.sweep == "tree" else capi.SWEEP_EXACT,
                                 C.byref(y), None, None, capi.ptr(per_slice), C.byref(rep), C.byref(fail))
    _check(rc, ctx, fail)
    stats = SweepStats(message_count=N - 1, bytes_communicated=8 * (N - 1),
                       extrapolation_count=int(rep.extrapolation_count), apply_cost=rep.compose_ms * 1e-3 / N)
    for _ in range(N - 1):  # the simulated wire (nievergelt.cpp:73-79)
        if exec_.latency_per_receive > 0.0:
            sw = Stopwatch()
            inject_latency(exec_.latency_per_receive)
            stats.T_comm += sw.seconds()
    r.T_total = total.seconds()
    _fill_report(r, np.array([y.value]), stats, per_slice, rep, exec_)
    if ivp.exact is not None:
        r.error_vs_exact = abs(y.value - ivp.exact(ivp.T))
    r.error_vs_serial = abs(y.value - y_serial) / max(1e-300, abs(y_serial))
    return r


def _run_linear(problem: LinearProblem, N: int, exec_: ExecConfig, compose: str) -> RunReport:
    if N <= 1:
        r = run_serial(problem)
        r.method = "nievergelt"
        r.workers = exec_.workers
        return r
    ctx = context()
    r = RunReport(method="nievergelt", N=N, dt=problem.dt, latency=exec_.latency_per_receive, workers=exec_.workers)
    n = problem.dim
    y = np.empty(n)
    y0 = np.ascontiguousarray(problem.y0, dtype=np.float64)
    per_slice = np.zeros(N)
    rep = capi.Report()
    # the serial reference run (outside T_total, nievergelt.cpp:221) in the background on the device
    serial = np.empty(n)
    _check(ctx.lib.pint_heat_serial_begin(ctx.h, problem.dx, problem.dt, problem.T, capi.ptr(y0)), ctx)
    total = Stopwatch()
    rc = ctx.lib.pint_run_heat(ctx.h, problem.dx, problem.dt, problem.T, N,
                               capi.COMPOSE_TREE if compose == "tree" else capi.COMPOSE_CHAIN,
                               capi.ptr(y0), capi.ptr(y), capi.ptr(per_slice), C.byref(rep))
    t_run = total.seconds()
    rs = ctx.lib.pint_heat_serial_end(ctx.h, capi.ptr(serial))
    _check(rc, ctx)
    _check(rs, ctx)
    stats = SweepStats(message_count=N - 1, bytes_communicated=8 * n * (N - 1), apply_cost=rep.compose_ms * 1e-3 / N)
    for _ in range(N - 1):
        if exec_.latency_per_receive > 0.0:
            sw = Stopwatch()
            inject_latency(exec_.latency_per_receive)
            stats.T_comm += sw.seconds()
    r.T_total = t_run + stats.T_comm
    _fill_report(r, y, stats, per_slice, rep, exec_)
    if problem.exact_final is not None:
        r.error_vs_exact = float(np.max(np.abs(y - problem.exact_final)))
    scale = float(np.max(np.abs(serial)))
    gap = float(np.max(np.abs(y - serial)))
    r.error_vs_serial = gap if scale == 0.0 else gap / scale
    return r


def _fill_report(r: RunReport, final, stats: SweepStats, per_slice, rep, exec_: ExecConfig):
    r.final_state = final
    r.T_comm = stats.T_comm
    r.message_count = stats.message_count
    r.bytes_communicated = stats.bytes_communicated
    r.extrapolation_count = stats.extrapolation_count
    r.per_slice_compute = list(map(float, per_slice))
    r.device_ms = rep.device_ms
    r.traj_steps = int(rep.traj_steps)
    r.gpu_launches = int(rep.gpu_launches)
    if exec_.clock != MEASURED:
        r.modeled_time = modeled_time_nievergelt(r.per_slice_compute, exec_.latency_per_receive, stats.apply_cost)
