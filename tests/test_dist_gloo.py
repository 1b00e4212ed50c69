"""Multi-process (gloo, CPU) tests of the slice-block sharding in paper_1304_6514_b200/dist.py.

On the GPU box each rank builds its block's slice maps and tree-composes them on its B200; here
the C oracle stands in for that device work so the host logic — contiguous deterministic slice
blocks, the single gather of composed block maps to rank 0, and the ordered root composition —
is exercised with real torch.distributed collectives (gloo, world sizes 2 and 3).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_1304_6514_b200 import capi
from paper_1304_6514_b200.dist import slice_block, gather_maps

DX, T, N, S = 0.1, 10.0, 12, 40


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _augmented(G, c):
    """The device layout of one map: row-major [G | c] with ldm = pint_affine_ldm(n)."""
    n = G.shape[0]
    ldm = int(capi.load().pint_affine_ldm(n))
    A = np.zeros((n, ldm))
    A[:, :n] = G
    A[:, n] = c
    return A


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dt = T / (N * S)
        tb, te, _, _ = O.decompose(0.0, T, N, dt)
        lo, hi = slice_block(N, world, rank)
        Gs, cs = zip(*[O.heat_build(DX, tb[j], te[j], dt) for j in range(lo, hi)])
        Gb, cb, _ = O.affine_tree(np.stack(Gs), np.stack(cs), np.zeros(len(cs[0])))
        local = torch.from_numpy(_augmented(Gb, cb).ravel().copy())
        maps = gather_maps(local)
        if rank == 0:
            n = Gb.shape[0]
            blocks = [m.numpy().reshape(n, -1) for m in maps]
            G = np.stack([b[:, :n] for b in blocks])
            c = np.stack([b[:, n] for b in blocks])
            out[0] = O.affine_chain(G, c, O.heat_initial(DX))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_block_gather_compose_matches_full_chain(world):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    dt = T / (N * S)
    tb, te, _, _ = O.decompose(0.0, T, N, dt)
    G, c = zip(*[O.heat_build(DX, tb[j], te[j], dt) for j in range(N)])
    want = O.affine_chain(np.stack(G), np.stack(c), O.heat_initial(DX))
    got = np.asarray(out[0])
    assert np.max(np.abs(got - want)) <= 1e-12 * np.max(np.abs(want))


@pytest.mark.parametrize("N_,W", [(256, 8), (4096, 8), (7, 3), (5, 8)])
def test_slice_blocks_partition(N_, W):
    blocks = [slice_block(N_, W, r) for r in range(W)]
    assert blocks[0][0] == 0 and blocks[-1][1] == N_
    for (a, b), (c, d) in zip(blocks, blocks[1:]):
        assert b == c and a <= b
    sizes = [b - a for a, b in blocks]
    assert max(sizes) - min(sizes) <= 1


# ---- nonlinear composition across ranks: the oracle stands in for K1/K2 --------

def _scalar_worker(rank, world, port, out, N, M):
    from paper_1304_6514_b200.dist import gather_rows

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _, _, steps, h = O.decompose(0.0, 0.5, N, 1e-4)
        nodes = O.cheb_nodes(M, 0.0, 2.0)
        lo, hi = slice_block(N, world, rank)
        ends, fail, _ = O.riccati_ensemble(steps[lo:hi], h[lo:hi], nodes)
        assert fail < 0
        tables = gather_rows(torch.from_numpy(ends.copy()), N)
        if rank == 0:
            y, lam, ext = O.scalar_sweep(nodes, O.bary_weights(nodes), tables.numpy(), 0.0, 2.0, 1.0)
            out["y"], out["lam"], out["ext"] = y, lam.tolist(), ext
        else:
            assert tables is None
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_scalar_tables_gather_then_sweep_is_bit_exact(world):
    """C1/C5 across ranks: blocks of endpoint tables gathered to rank 0 (uneven blocks padded),
    swept there: identical bits to the single-process pipeline."""
    N, M = 7, 6
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_scalar_worker, args=(world, _free_port(), out, N, M), nprocs=world, join=True)
    _, _, steps, h = O.decompose(0.0, 0.5, N, 1e-4)
    nodes = O.cheb_nodes(M, 0.0, 2.0)
    ends, _, _ = O.riccati_ensemble(steps, h, nodes)
    y, lam, ext = O.scalar_sweep(nodes, O.bary_weights(nodes), ends, 0.0, 2.0, 1.0)
    assert out["y"] == y and out["lam"] == lam.tolist() and out["ext"] == ext


LV = (1.5, 1.0, 1.0, 3.0)


def _lv_worker(rank, world, port, out, N, Mu, Mv, S):
    from paper_1304_6514_b200.dist import lambda_chain

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _, _, steps, h = O.decompose(0.0, 10.0, N, 10.0 / (N * S))
        un, vn = O.uniform_nodes(Mu, 0.1, 8.0), O.uniform_nodes(Mv, 0.1, 8.0)
        lo, hi = slice_block(N, world, rank)
        tables = O.lv_rk4_ensemble(steps[lo:hi], h[lo:hi], un, vn, LV)

        def sweep_block(lam):
            got, _, _ = O.bilinear_sweep(un, vn, tables, float(lam[0]), float(lam[1]))
            return torch.from_numpy(got[-1].copy())

        final = lambda_chain(sweep_block, torch.tensor([1.0, 1.0], dtype=torch.float64))
        out[rank] = final.tolist()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_lv_lambda_chain_is_bit_exact(world):
    """C3 across ranks: the running value crosses the ranks once (W-1 two-double messages);
    every rank ends with the single-process sweep's final value, bit for bit."""
    N, Mu, Mv, S = 8, 17, 13, 8
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_lv_worker, args=(world, _free_port(), out, N, Mu, Mv, S), nprocs=world, join=True)
    _, _, steps, h = O.decompose(0.0, 10.0, N, 10.0 / (N * S))
    un, vn = O.uniform_nodes(Mu, 0.1, 8.0), O.uniform_nodes(Mv, 0.1, 8.0)
    lam, _, _ = O.bilinear_sweep(un, vn, O.lv_rk4_ensemble(steps, h, un, vn, LV), 1.0, 1.0)
    for r in range(world):
        assert out[r] == lam[-1].tolist()
