"""Slice-block sharding of the heat (affine) path across GPUs — north_star subsystem (4).

One process per GPU (torch.distributed, NCCL over NVLink on the box, gloo in CPU tests). Rank g
owns the contiguous slice block [floor(gN/W), floor((g+1)N/W)) of the reference decomposition
(ode_core.cpp:26-45, computed identically on every rank, so slice assignment is bit-exact), builds
those slice maps (K3), tree-composes them locally (K4) into one augmented map, and the ONE
collective is the gather of the W composed maps to rank 0 — the paper's single final
gather/compose step (§3, nievergelt.cpp:90-110 is its sequential stand-in). Rank 0 then
applies the W maps to y0 in rank order with the bit-exact chain.

This replaces the reference's simulated wire (inject_latency + counters, nievergelt.cpp:95-101):
message_count stays N-1 in the RunReport sense; the real exchange is W-1 map transfers.
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
    """Per-step coefficient tables for a block of slices, in pinned host memory."""

    def __init__(self, dx: float, slices: List[capi.Slice]):
        import torch

        N = len(slices)
        arr = (capi.Slice * N)(*slices)
        Q = int(capi.load().pint_heat_total_steps(arr, N))
        n = C.c_int64()
        self.N, self.Q = N, Q
        self.step_off = torch.empty(N + 1, dtype=torch.int64).pin_memory()
        self.slice_dt = torch.tensor([s.dt for s in slices], dtype=torch.float64).pin_memory()
        self.r = torch.empty(Q, dtype=torch.float64).pin_memory()
        self.fa = torch.empty(Q, dtype=torch.float64).pin_memory()
        self.fb = torch.empty(Q, dtype=torch.float64).pin_memory()
        n_int = int(round(1.0 / dx)) - 1
        self.sx = torch.empty(max(n_int, 1), dtype=torch.float64).pin_memory()
        rc = capi.load().pint_heat_coefficients(dx, arr, N, self.step_off.data_ptr(), self.r.data_ptr(),
                                                self.fa.data_ptr(), self.fb.data_ptr(), self.sx.data_ptr(),
                                                C.byref(n))
        if rc != capi.PINT_OK:
            raise pint.BadGrid(f"make_heat_system: 1/dx must be an integer >= 2, got dx = {dx:f}")
        self.n = int(n.value)
        self.sx = self.sx[: self.n]

    def tensors(self):
        return [self.step_off, self.slice_dt, self.r, self.fa, self.fb, self.sx]

    def nbytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in self.tensors())


class HeatPlan:
    """Device-resident plan for slices [lo, hi) of make_heat_problem(dx, dt, T) cut into N slices."""

    def __init__(self, ctx: capi.Context, dx: float, dt: float, T: float, N: int, lo: int = 0,
                 hi: Optional[int] = None, tables: Optional[HeatTablesHost] = None):
        import torch

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
        rec_doubles = int(capi.load().pint_heat_records_size(self.n, self.N, self.S))
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

    plan.step(capi.COMPOSE_TREE)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return
    maps = gather_maps(plan.composed, group)
    if dist.get_rank(group) == 0:
        cat = torch.cat(maps)
        apply_chain(plan.ctx, plan.n, cat, plan.y0, plan.y)

