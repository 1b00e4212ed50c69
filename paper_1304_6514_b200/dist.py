"""Slice-block sharding across GPUs — north_star subsystem (4), SURVEY.md §8e.

One process per GPU (torch.distributed, NCCL over NVLink on the box, gloo in CPU tests). Rank g
owns the contiguous slice block [floor(gN/W), floor((g+1)N/W)) of the reference decomposition
(ode_core.cpp:26-45, computed identically on every rank, so slice assignment is bit-exact), builds
those slice maps (K3), tree-composes them locally (K4) into one augmented map, and the ONE
collective is the gather of the W composed maps to rank 0 — the paper's single final
gather/compose step (§3, nievergelt.cpp:90-110 is its sequential stand-in). Rank 0 then
applies the W maps to y0 in rank order with the bit-exact chain.

This replaces the reference's simulated wire (inject_latency + counters, nievergelt.cpp:95-101):
message_count stays N-1 in the RunReport sense; the real exchange is W-1 map transfers.

Nonlinear composition (scalar C1/C5, 2-D Lotka-Volterra C3) is sequential by nature — a
composition of interpolants has no closed form — so the blocks build their slice tables in
parallel (K1, no collective) and the sweep runs in one of the two ways §8e names:
  * gather_rows: the endpoint tables of every block to rank 0 (C1/C5: 64 x 1024 doubles =
    512 KiB), which sweeps all N slices (K2) — one collective;
  * lambda_chain: the paper's hand-off of the running value (C3, whose tables
    are 448 MiB): rank g receives the value leaving block g-1, sweeps its own block, sends the
    result on — W-1 messages of 1-2 doubles.
Both give results bit-identical to the single-GPU sweep (same slices, same order).
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Tuple

import numpy as np

from . import capi, pint


def slice_block(N: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous block of slices owned by `rank` (deterministic, identical on every rank)."""
    return (rank * N) // world, ((rank + 1) * N) // world


def closure_slices(dec: pint.TimeSliceDecomposition, dt_nominal: float) -> List[capi.Slice]:
    """Slices as the heat integrate closure steps them (pde_problems.cpp:88-89)."""
    out = []
    for s in dec.slices:
        n = pint.steps_for(s.t_end - s.t_begin, dt_nominal)
        out.append(capi.Slice(s.t_begin, s.t_end, n, (s.t_end - s.t_begin) / n))
    return out


class HeatTablesHost:
    """Per-step coefficient tables for a block of slices, in pinned host memory (allocated once;
    refill() recomputes them in place, so a timed e2e loop allocates nothing)."""

    def __init__(self, dx: float, slices: List[capi.Slice]):
        import torch

        N = len(slices)
        arr = (capi.Slice * N)(*slices)
        Q = int(capi.load().pint_heat_total_steps(arr, N))
        self.N, self.Q = N, Q
        self.step_off = torch.empty(N + 1, dtype=torch.int64).pin_memory()
        self.slice_dt = torch.empty(N, dtype=torch.float64).pin_memory()
        self.r = torch.empty(Q, dtype=torch.float64).pin_memory()
        self.fa = torch.empty(Q, dtype=torch.float64).pin_memory()
        self.fb = torch.empty(Q, dtype=torch.float64).pin_memory()
        n_int = int(round(1.0 / dx)) - 1
        self._sx = torch.empty(max(n_int, 1), dtype=torch.float64).pin_memory()
        self.refill(dx, slices)

    def refill(self, dx: float, slices: List[capi.Slice]) -> None:
        """Recompute every table (glibc sin/cos on the host, the reference's arithmetic)."""
        N = len(slices)
        if N != self.N:
            raise ValueError(f"refill: {N} slices, tables hold {self.N}")
        arr = (capi.Slice * N)(*slices)
        n = C.c_int64()
        for j, s in enumerate(slices):
            self.slice_dt[j] = s.dt
        rc = capi.load().pint_heat_coefficients(dx, arr, N, self.step_off.data_ptr(), self.r.data_ptr(),
                                                self.fa.data_ptr(), self.fb.data_ptr(), self._sx.data_ptr(),
                                                C.byref(n))
        if rc != capi.PINT_OK:
            raise pint.BadGrid(f"make_heat_system: 1/dx must be an integer >= 2, got dx = {dx:f}")
        self.n = int(n.value)
        self.sx = self._sx[: self.n]

    def tensors(self):
        return [self.step_off, self.slice_dt, self.r, self.fa, self.fb, self.sx]

    def nbytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in self.tensors())


class HeatPlan:
    """Device-resident plan for slices [lo, hi) of make_heat_problem(dx, dt, T) cut into N slices."""

    def __init__(self, ctx: capi.Context, dx: float, dt: float, T: float, N: int, lo: int = 0,
                 hi: Optional[int] = None, tables: Optional[HeatTablesHost] = None, build: str = "exact"):
        import torch

        if build not in ("exact", "fast"):
            raise ValueError(f"build must be 'exact' or 'fast', got {build!r}")
        self.build = build
        self.ctx = ctx
        self.dx, self.dt, self.T, self.N_total = dx, dt, T, N
        hi = N if hi is None else hi
        self.lo, self.hi = lo, hi
        self.slices = closure_slices(pint.decompose(0.0, T, N, dt), dt)[lo:hi]
        self.host = tables or HeatTablesHost(dx, self.slices)
        self.n = self.host.n
        self.N = hi - lo
        self.Q = self.host.Q
        self.ldm = int(capi.load().pint_affine_ldm(self.n))
        dev = torch.device("cuda", ctx.device)
        self.dev = [t.to(dev) for t in self.host.tensors()]
        self.S = max(s.steps for s in self.slices)
        size = capi.load().pint_heat_fast_records_size if build == "fast" else capi.load().pint_heat_records_size
        rec_doubles = int(size(self.n, self.N, self.S))
        if rec_doubles <= 0:
            raise ValueError(f"the {build} build does not support n = {self.n}")
        self.factor = torch.empty(rec_doubles, dtype=torch.float64, device=dev)
        stride = self.n * self.ldm
        self.maps = torch.zeros(self.N * stride, dtype=torch.float64, device=dev)
        self.scratch = torch.zeros(max(1, (self.N + 1) // 2) * stride, dtype=torch.float64, device=dev)
        self.composed = torch.zeros(stride, dtype=torch.float64, device=dev)
        self.y0 = torch.as_tensor(pint.heat_initial(dx)).to(dev)
        self.y = torch.empty(self.n, dtype=torch.float64, device=dev)
        self.guarded = 0

    @property
    def traj_steps(self) -> int:
        return self.Q * (self.n + 1)

    def upload(self):
        """Host -> device copies of the tables (the e2e path); returns bytes copied."""
        for d, h in zip(self.dev, self.host.tensors()):
            d.copy_(h, non_blocking=True)
        return self.host.nbytes()

    def factor_and_build(self):
        c, P = self.ctx, capi.ptr
        step_off, slice_dt, r, fa, fb, sx = self.dev
        if self.build == "fast":
            c.call("pint_heat_fast_factor_dev", self.n, self.N, self.S, P(step_off), P(slice_dt), P(r), P(fa), P(fb),
                   P(sx), P(self.factor))
            c.call("pint_heat_fast_build_dev", self.n, self.N, self.S, P(self.factor), P(self.maps))
            return
        c.call("pint_heat_factor_dev", self.n, self.N, self.S, P(step_off), P(slice_dt), P(r), P(fa), P(fb), P(sx),
               P(self.factor))
        c.call("pint_heat_build_dev", self.n, self.N, self.S, P(step_off), P(slice_dt), P(self.factor), P(sx),
               P(self.maps), None, self.guarded)

    def verify(self) -> bool:
        """Read the failure record after a step: a tripped range check switches this plan to the
        guarded build (returns False: re-run the step); a singular pivot raises."""
        f = self.ctx.fail()
        if f.index < 0:
            return True
        if f.code == capi.PINT_E_SERIALIZED:  # the concurrent chain ran alone: the maps are complete
            self.compose_local(capi.COMPOSE_CHAIN, want_composed=False)
            self.ctx.sync()
            return self.verify()
        if f.code == capi.PINT_E_RANGE_RETRY:
            self.guarded = 1
            return False
        raise pint.SingularSystem(f"thomas_solve: zero pivot at row {int(f.value)}")

    def compose_local(self, mode: int = capi.COMPOSE_TREE, want_composed: bool = True):
        """Compose this block's maps: self.y = block map applied to y0, and (TREE with
        want_composed) the composed augmented map in self.composed — the multi-GPU path needs it;
        a single GPU only needs y, so the tree stops early and chain-applies its last few maps."""
        P = capi.ptr
        if mode == capi.COMPOSE_TREE:
            self.ctx.call("pint_affine_compose_dev", capi.COMPOSE_TREE, self.n, self.N, P(self.maps), P(self.scratch),
                          P(self.y0), P(self.y), P(self.composed) if want_composed else None)
        else:
            self.ctx.call("pint_affine_compose_dev", capi.COMPOSE_CHAIN, self.n, self.N, P(self.maps), None,
                          P(self.y0), P(self.y), None)

    def step(self, mode: int = capi.COMPOSE_TREE):
        self.factor_and_build()
        self.compose_local(mode)


def gather_maps(local, group=None, root: int = 0):
    """Gather every rank's composed augmented map to `root` (the one collective)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    bufs = [torch.empty_like(local) for _ in range(world)] if rank == root else None
    dist.gather(local, bufs, dst=root, group=group)
    return bufs


def apply_chain(ctx: capi.Context, n: int, maps_cat, y0, y):
    """Rank 0: apply the gathered block maps in rank order (bit-exact chain, K4)."""
    P = capi.ptr
    W = maps_cat.numel() // (n * int(capi.load().pint_affine_ldm(n)))
    ctx.call("pint_affine_compose_dev", capi.COMPOSE_CHAIN, n, W, P(maps_cat), None, P(y0), P(y), None)


def sharded_heat_step(plan: HeatPlan, group=None) -> None:
    """One full solve on this rank's block + the final gather/compose. Rank 0 ends with plan.y
    holding the global final state."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    mode = capi.COMPOSE_TREE if world > 1 else capi.COMPOSE_CHAIN
    for _ in range(2):  # a tripped range check switches the plan to the guarded build: re-run once
        plan.factor_and_build()
        plan.compose_local(mode, want_composed=world > 1)
        plan.ctx.sync()  # (also orders the maps before the collective on torch's stream)
        if plan.verify():
            break
    if world == 1:
        return
    maps = gather_maps(plan.composed, group)
    if dist.get_rank(group) == 0:
        cat = torch.cat(maps)
        # gather and cat ran on torch's current stream; the chain runs on the context's stream
        torch.cuda.current_stream(cat.device).synchronize()
        apply_chain(plan.ctx, plan.n, cat, plan.y0, plan.y)
        plan.ctx.sync()


# ---- the sharded run behind the C ABI (pint_run_heat_sharded) -----------------------------------

class TorchDistTransport:
    """pint_comm_init_callbacks transport over torch.distributed point-to-point (e.g. gloo): the
    library hands host buffers to these callbacks. Keep the object alive while the context uses it."""

    def __init__(self, ctx: capi.Context, group=None):
        import torch.distributed as dist

        self.ctx, self.group = ctx, group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)

        def _send(user, peer, buf, nbytes):
            try:
                import torch

                arr = np.ctypeslib.as_array(C.cast(buf, C.POINTER(C.c_uint8)), shape=(nbytes,))
                dist.send(torch.from_numpy(arr.copy()), peer, group=group)
                return 0
            except Exception:  # (reported to the library as a transport failure)
                return 1

        def _recv(user, peer, buf, nbytes):
            try:
                import torch

                t = torch.empty(nbytes, dtype=torch.uint8)
                dist.recv(t, peer, group=group)
                C.memmove(buf, t.numpy().ctypes.data, nbytes)
                return 0
            except Exception:
                return 1

        self._send, self._recv = capi.SEND_FN(_send), capi.RECV_FN(_recv)
        ctx.check(ctx.lib.pint_comm_init_callbacks(ctx.h, self.rank, self.world, self._send, self._recv, None))


def nccl_comm_init(ctx: capi.Context, group=None) -> None:
    """pint_comm_init over NCCL: rank 0 makes the unique id, torch.distributed broadcasts it."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    uid = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        ctx.check(ctx.lib.pint_comm_unique_id(capi.ptr(uid.numpy())))
    if dist.get_backend(group) == "nccl":
        u = uid.cuda()
        dist.broadcast(u, 0, group=group)
        uid = u.cpu()
    else:
        dist.broadcast(uid, 0, group=group)
    ctx.check(ctx.lib.pint_comm_init(ctx.h, capi.ptr(uid.numpy()), rank, world))


def run_heat_sharded(ctx: capi.Context, dx: float, dt: float, T: float, N: int, build: str = "exact",
                     compose: str = "chain", y0=None):
    """pint_run_heat_sharded on this rank (every rank calls it): returns (y or None, report)."""
    rank, world = C.c_int(), C.c_int()
    ctx.check(ctx.lib.pint_comm_rank(ctx.h, C.byref(rank), C.byref(world)))
    n = int(round(1.0 / dx)) - 1
    y = np.empty(n) if rank.value == 0 else None
    y0a = None if y0 is None else np.ascontiguousarray(y0, dtype=np.float64)
    rep = capi.Report()
    ctx.check(ctx.lib.pint_run_heat_sharded(ctx.h, dx, dt, T, N, capi.BUILD_FAST if build == "fast" else capi.BUILD_EXACT,
                                            capi.COMPOSE_TREE if compose == "tree" else capi.COMPOSE_CHAIN,
                                            capi.ptr(y0a), capi.ptr(y), C.byref(rep)))
    return y, rep


# ---- nonlinear composition across ranks ---------------------------------------

def block_sizes(N: int, world: int) -> List[int]:
    return [b - a for a, b in (slice_block(N, world, r) for r in range(world))]


def gather_rows(local, N: int, group=None, root: int = 0):
    """Gather every rank's contiguous block of per-slice rows (local: [rows, ...]) to `root` in
    slice order. Blocks differ by at most one slice, so each rank pads to the largest block;
    ONE gather; root trims and concatenates. Returns the [N, ...] tensor on root, None elsewhere."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    sizes = block_sizes(N, world)
    if local.shape[0] != sizes[rank]:
        raise ValueError(f"rank {rank}: {local.shape[0]} rows, block holds {sizes[rank]}")
    pad = torch.zeros((max(sizes),) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)] if rank == root else None
    dist.gather(pad, bufs, dst=root, group=group)
    if rank != root:
        return None
    return torch.cat([b[:n] for b, n in zip(bufs, sizes)])


def lambda_chain(sweep_block, lam0, group=None):
    """The paper's hand-off for nonlinear maps: rank g receives the value leaving block g-1
    (rank 0 starts from lam0), applies its own block with sweep_block(lam) -> lam, sends the
    result to g+1. The final value (leaving the last block) is broadcast to every rank."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lam = lam0.clone()
    if rank > 0:
        dist.recv(lam, src=rank - 1, group=group)
    out = sweep_block(lam).clone()
    if rank < world - 1:
        dist.send(out, dst=rank + 1, group=group)
    dist.broadcast(out, src=world - 1, group=group)
    return out


class ScalarPlan:
    """Device plan for the slice block [lo, hi) of a scalar Nievergelt run (C1/C5): the K1
    ensemble of the block's N_local x M trajectories (pint_scalar_ensemble_dev), and — on the
    rank that holds all N tables — the weights and the sweep (pint_bary_weights_dev,
    pint_scalar_sweep_dev), exactly as pint_run_scalar sequences them (capi.cu)."""

    def __init__(self, ctx: capi.Context, rhs: capi.ScalarRHS, t0: float, T: float, y0: float, N: int,
                 dt: float, M: int, a: float, b: float, node_kind: int = capi.NODES_SECOND_KIND,
                 weight_kind: int = capi.WEIGHTS_PRODUCT, sweep_mode: int = capi.SWEEP_EXACT,
                 lo: int = 0, hi: Optional[int] = None):
        import torch

        hi = N if hi is None else hi
        self.ctx, self.rhs, self.y0, self.N, self.M, self.a, self.b = ctx, rhs, y0, N, M, a, b
        self.weight_kind, self.sweep_mode, self.lo, self.hi = weight_kind, sweep_mode, lo, hi
        dec = pint.decompose(t0, T, N, dt)
        steps, dts = pint.slice_table(dec)
        dev = f"cuda:{ctx.device}"
        self.steps = torch.as_tensor(steps[lo:hi]).to(dev)
        self.dt = torch.as_tensor(dts[lo:hi]).to(dev)
        kind = pint.FIRST_KIND if node_kind == capi.NODES_FIRST_KIND else pint.SECOND_KIND
        self.nodes = torch.as_tensor(pint.sample_nodes(kind, M, a, b)).to(dev)
        self.ab = torch.tensor([a, b], dtype=torch.float64, device=dev)
        self.ends = torch.empty((hi - lo, M), dtype=torch.float64, device=dev)

    def build(self):
        """Launch the block's ensemble on the context's stream (asynchronous)."""
        P = capi.ptr
        self.ctx.call("pint_scalar_ensemble_dev", C.byref(self.rhs), self.hi - self.lo, self.M, P(self.steps),
                      P(self.dt), P(self.nodes), P(self.ends), None)

    def sweep(self, tables) -> Tuple[float, "object", int]:
        """Sweep all N slice tables ([N, M] on this device) from y0: (y, lambdas[N], extrapolations)."""
        import torch

        P = capi.ptr
        dev = tables.device
        w = torch.empty(self.M, dtype=torch.float64, device=dev)
        lam = torch.empty(self.N, dtype=torch.float64, device=dev)
        y = torch.empty(1, dtype=torch.float64, device=dev)
        ext = torch.zeros(1, dtype=torch.int64, device=dev)
        self.ctx.call("pint_bary_weights_dev", self.weight_kind, self.M, P(self.nodes), P(w))
        self.ctx.call("pint_scalar_sweep_dev", self.sweep_mode, self.N, self.M, P(self.nodes), 0, P(w),
                      P(tables), P(self.ab), P(self.ab[1:]), 0, self.y0, P(lam), P(y), P(ext))
        self.ctx.sync()
        return float(y.item()), lam, int(ext.item())


def sharded_scalar_run(plan: ScalarPlan, group=None):
    """C1/C5 on W GPUs: every rank builds its block's tables; the tables are gathered to rank 0,
    which sweeps. Returns (y, lambdas, extrapolations) on rank 0, None elsewhere."""
    import torch.distributed as dist

    plan.build()
    plan.ctx.sync()  # the tables are produced on the context's stream; the collective runs on torch's
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return plan.sweep(plan.ends)
    tables = gather_rows(plan.ends, plan.N, group)
    return plan.sweep(tables) if dist.get_rank(group) == 0 else None


class LVPlan:
    """Device plan for the slice block [lo, hi) of the 2-D Lotka-Volterra run (C3, EXTENSION):
    the block's tensor-grid RK4 tables (pint_lv_ensemble_dev) and the block's bilinear sweep
    (pint_bilinear_sweep_dev) from an incoming value."""

    def __init__(self, ctx: capi.Context, params, T: float, N: int, S: int, un, vn, lo: int = 0,
                 hi: Optional[int] = None):
        import torch

        hi = N if hi is None else hi
        self.ctx, self.N, self.lo, self.hi = ctx, N, lo, hi
        dec = pint.decompose(0.0, T, N, T / (N * S))
        steps, dts = pint.slice_table(dec)
        dev = f"cuda:{ctx.device}"
        self.steps = torch.as_tensor(steps[lo:hi]).to(dev)
        self.dt = torch.as_tensor(dts[lo:hi]).to(dev)
        self.un = torch.as_tensor(np.ascontiguousarray(un, np.float64)).to(dev)
        self.vn = torch.as_tensor(np.ascontiguousarray(vn, np.float64)).to(dev)
        self.params = np.ascontiguousarray(params, np.float64)
        self.tables = torch.empty((hi - lo) * 2 * len(un) * len(vn), dtype=torch.float64, device=dev)
        self.lam = torch.empty(2 * (hi - lo), dtype=torch.float64, device=dev)
        self.br = torch.empty(2 * (hi - lo), dtype=torch.int64, device=dev)
        self.ext = torch.zeros(1, dtype=torch.int64, device=dev)

    def build(self):
        P = capi.ptr
        self.ctx.call("pint_lv_ensemble_dev", self.hi - self.lo, len(self.un), len(self.vn), P(self.steps), P(self.dt),
                      P(self.un), P(self.vn), P(self.params), P(self.tables))

    def sweep_block(self, lam):
        """Apply this block's bilinear maps in order from lam = (u, v); returns the value leaving it."""
        P = capi.ptr
        u0, v0 = (float(x) for x in lam.cpu())
        self.ctx.call("pint_bilinear_sweep_dev", self.hi - self.lo, len(self.un), len(self.vn), P(self.un), P(self.vn),
                      P(self.tables), u0, v0, P(self.lam), P(self.br), P(self.ext))
        self.ctx.sync()
        return self.lam.view(-1, 2)[-1].clone()


def sharded_lv_run(plan: LVPlan, u0: float, v0: float, group=None):
    """C3 on W GPUs: blocks build their tables in parallel; the running value crosses the ranks
    once (lambda_chain). Returns the final (u, v) on every rank."""
    import torch
    import torch.distributed as dist

    plan.build()
    plan.ctx.sync()
    lam0 = torch.tensor([u0, v0], dtype=torch.float64, device=plan.lam.device)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return plan.sweep_block(lam0)
    return lambda_chain(plan.sweep_block, lam0, group)
