"""Where the end-to-end time of pint_run_heat goes (bench config): wall vs device time, and the
host-side table computation alone.   python tools/e2e_breakdown.py"""
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
    n, N, S, T = 128, 256, 256, 10.0
    dx, dt = 1.0 / (n + 1), T / (N * S)
    y = np.empty(n)
    rep = capi.Report()
    rows = []
    for i in range(12):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.check(ctx.lib.pint_run_heat(ctx.h, dx, dt, T, N, capi.COMPOSE_TREE, None, capi.ptr(y), None,
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


if __name__ == "__main__":
    main()
