"""Where the end-to-end time of pint_run_heat goes (bench config): wall vs device time, and the
host-side table computation alone.   python tools/e2e_breakdown.py [c2|c4]"""
import ctypes as C
import json
import pathlib
import sys
import time

import numpy as np

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main():
    import torch

    from paper_1304_6514_b200 import capi, pint
    from paper_1304_6514_b200.dist import HeatTablesHost, closure_slices

    ctx = capi.Context(0, stream=torch.cuda.current_stream())
    c4 = len(sys.argv) > 1 and sys.argv[1] == "c4"
    n, N, S, T = (512, 4096, 16, 10.0) if c4 else (128, 256, 256, 10.0)
    mode = capi.COMPOSE_CHAIN if c4 else capi.COMPOSE_TREE
    dx, dt = 1.0 / (n + 1), T / (N * S)
    y = np.empty(n)
    rep = capi.Report()
    rows = []
    for i in range(12):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.check(ctx.lib.pint_run_heat(ctx.h, dx, dt, T, N, mode, None, capi.ptr(y), None,
                                        C.byref(rep)))
        wall = (time.perf_counter() - t0) * 1e3
        rows.append((wall, rep.total_ms, rep.device_ms, rep.compose_ms))
    slices = closure_slices(pint.decompose(0.0, T, N, dt), dt)
    t0 = time.perf_counter()
    for _ in range(10):
        HeatTablesHost(dx, slices)
    tables_ms = (time.perf_counter() - t0) * 100
    w = np.array(rows[2:])
    print(json.dumps({"wall_ms": w[:, 0].mean(), "total_ms": w[:, 1].mean(), "device_ms": w[:, 2].mean(),
                      "compose_ms": w[:, 3].mean(), "host_tables_ms(py, incl. pinned alloc)": tables_ms}))


if __name__ == "__main__" and (len(sys.argv) == 1 or sys.argv[1] in ("c2", "c4")):
    main()


def host_tables_ms(reps: int = 20, c4: bool = False) -> float:
    """Host-only time of pint_heat_coefficients for the bench's slices (the glibc sin/cos tables)."""
    from paper_1304_6514_b200 import capi, pint
    from paper_1304_6514_b200.dist import closure_slices

    n, N, S, T = (512, 4096, 16, 10.0) if c4 else (128, 256, 256, 10.0)
    dx, dt = 1.0 / (n + 1), T / (N * S)
    sl = closure_slices(pint.decompose(0.0, T, N, dt), dt)
    arr = (capi.Slice * N)(*sl)
    Q = sum(s.steps for s in sl)
    off, r, fa, fb, sx = np.empty(N + 1, np.int64), np.empty(Q), np.empty(Q), np.empty(Q), np.empty(n)
    nn = C.c_int64()
    lib = capi.load()
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        lib.pint_heat_coefficients(dx, arr, N, capi.ptr(off), capi.ptr(r), capi.ptr(fa), capi.ptr(fb),
                                   capi.ptr(sx), C.byref(nn))
        best = min(best, time.perf_counter() - t0)
    return best * 1e3


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "--host":
    print(json.dumps({"host_tables_ms": host_tables_ms(c4="c4" in sys.argv)}))
