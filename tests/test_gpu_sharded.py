"""The sharded heat run behind the C ABI (pint_run_heat_sharded, comm.cu) on the GPU box.

Only one GPU is available, so W > 1 runs W PROCESSES on the same device with the host-callback
transport over torch.distributed gloo (pint_comm_init_callbacks): every rank's kernels are real,
the exchange goes through the host, and no kernel waits on another process's kernel. Checked
against the single-GPU run and the reference: CHAIN (the state handed rank to rank) bit-identical
to pint_run_heat; TREE (block maps gathered to rank 0) within 1e-12; ragged blocks (N % W != 0)
and an empty block (N < W). The NCCL transport itself runs at W = 1 (pint_comm_init).
"""
import ctypes as C
import os
import pathlib
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = pathlib.Path(__file__).resolve().parents[1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cases, out):
    import sys

    sys.path.insert(0, str(ROOT))
    import torch.distributed as dist

    from paper_1304_6514_b200 import capi
    from paper_1304_6514_b200.dist import TorchDistTransport, run_heat_sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ctx = capi.Context(0)
    tr = TorchDistTransport(ctx)
    res = {}
    for key, (n, N, S, build, compose) in cases.items():
        dx, dt = 1.0 / (n + 1), 10.0 / (N * S)
        y, rep = run_heat_sharded(ctx, dx, dt, 10.0, N, build, compose)
        res[key] = (y, rep.message_count, rep.bytes_communicated, rep.traj_steps)
    out.put((rank, res))
    dist.barrier()
    del tr
    ctx.close()
    dist.destroy_process_group()


def _run(world, cases):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return got


def _single(n, N, S, build, compose):
    from paper_1304_6514_b200 import capi, pint

    c = pint.context()
    dx, dt = 1.0 / (n + 1), 10.0 / (N * S)
    y = np.empty(n)
    c.check(c.lib.pint_run_heat_ex(c.h, dx, dt, 10.0, N, capi.BUILD_FAST if build == "fast" else capi.BUILD_EXACT,
                                   capi.COMPOSE_TREE if compose == "tree" else capi.COMPOSE_CHAIN, None, capi.ptr(y),
                                   None, None))
    return y


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_callbacks(world):
    cases = {
        "chain_c2": (128, 256, 16, "exact", "chain"),
        "tree_c2": (128, 256, 16, "exact", "tree"),
        "chain_ragged": (300, 7, 4, "exact", "chain"),
        "tree_ragged": (300, 7, 4, "exact", "tree"),
        "chain_empty": (64, 2, 8, "exact", "chain"),
        "tree_fast": (128, 33, 8, "fast", "tree"),
    }
    got = _run(world, cases)
    for key, (n, N, S, build, compose) in cases.items():
        y = got[0][key][0]
        ref = _single(n, N, S, build, "chain")
        if compose == "chain":
            assert np.array_equal(y, ref), key
        else:
            assert np.max(np.abs(y - ref)) / np.max(np.abs(ref)) <= 1e-12, key
        # real transfers: CHAIN one state per rank, TREE one block map per rank > 0
        for r in range(world):
            msgs, nbytes = got[r][key][1], got[r][key][2]
            ldm = (n + 1 + 3) // 4 * 4
            if compose == "chain":
                assert msgs == 1 and nbytes == 8 * n, (key, r)
            else:
                assert (msgs, nbytes) == ((0, 0) if r == 0 else (1, 8 * n * ldm)), (key, r)
        assert sum(got[r][key][3] for r in range(world)) == N * S * (n + 1)


def test_sharded_c2_matches_reference_golden():
    z = np.load(ROOT / "tests" / "golden" / "heat_finals.npz")
    n, N, S = (int(v) for v in z["c2_config"])
    got = _run(2, {"c2": (n, N, S, "exact", "chain")})
    assert np.array_equal(got[0]["c2"][0], z["c2_final"])


def test_sharded_nccl_world1():
    """The NCCL transport (pint_comm_unique_id + pint_comm_init, world 1): the run is the single-GPU
    one, bit-identical."""
    from paper_1304_6514_b200 import capi

    ctx = capi.Context(0)
    uid = np.zeros(128, dtype=np.uint8)
    ctx.check(ctx.lib.pint_comm_unique_id(capi.ptr(uid)))
    ctx.check(ctx.lib.pint_comm_init(ctx.h, capi.ptr(uid), 0, 1))
    r, w = C.c_int(), C.c_int()
    ctx.check(ctx.lib.pint_comm_rank(ctx.h, C.byref(r), C.byref(w)))
    assert (r.value, w.value) == (0, 1)
    from paper_1304_6514_b200.dist import run_heat_sharded

    n, N, S = 128, 64, 8
    y, rep = run_heat_sharded(ctx, 1.0 / (n + 1), 10.0 / (N * S), 10.0, N)
    assert np.array_equal(y, _single(n, N, S, "exact", "chain"))
    assert rep.message_count == 0
    ctx.check(ctx.lib.pint_comm_destroy(ctx.h))
    ctx.close()
