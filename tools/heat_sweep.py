"""Timing sweep of the heat map build alone (CUDA events around pint_heat_build_dev).

    python tools/heat_sweep.py --cases 128:256:256 128:1:256 66:1:256 ...   (n:N:S)

Prints one JSON line per case: build ms, cycles per (row, step) of one column chain at the
measured SM clock, and the per-row chain floor (7 dependent FP64 ops) for comparison.
"""
import argparse
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--cases", nargs="+", default=["128:256:256"])
    p.add_argument("--reps", type=int, default=5)
    p.add_argument("--clock-mhz", type=float, default=1965.0)
    a = p.parse_args()
    import torch

    from paper_1304_6514_b200 import capi
    from paper_1304_6514_b200.dist import HeatPlan

    torch.cuda.set_device(0)
    ctx = capi.Context(0, stream=torch.cuda.current_stream())
    for case in a.cases:
        n, N, S = (int(v) for v in case.split(":"))
        dx, dt = 1.0 / (n + 1), 10.0 / (N * S)
        plan = HeatPlan(ctx, dx, dt, 10.0, N)
        plan.upload()
        plan.factor_and_build()
        torch.cuda.synchronize()
        c, P = ctx, capi.ptr
        times = []
        for _ in range(a.reps):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            c.call("pint_heat_build_dev", plan.n, plan.N, plan.S, P(plan.dev[0]), P(plan.dev[1]), P(plan.factor),
                   P(plan.dev[-1]), P(plan.maps), None, plan.guarded)
            e.record()
            e.synchronize()
            times.append(s.elapsed_time(e))
        ms = min(times)
        cyc = ms * 1e-3 * a.clock_mhz * 1e6 / (plan.S * plan.n)
        comp = {}
        for mode, name in ((capi.COMPOSE_CHAIN, "chain_ms"), (capi.COMPOSE_TREE, "tree_ms")):
            ts = []
            for _ in range(a.reps):
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                plan.compose_local(mode, want_composed=False)
                e.record()
                e.synchronize()
                ts.append(s.elapsed_time(e))
            comp[name] = round(min(ts), 4)
        print(json.dumps({"n": n, "N": N, "S": plan.S, "build_ms": round(ms, 4), "cycles_per_row": round(cyc, 1),
                          "chain_floor_cycles_per_row": 7 * 8.1, **comp}), flush=True)


if __name__ == "__main__":
    main()
