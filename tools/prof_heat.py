"""Profiling driver: one heat map build (+ tree compose) at a chosen size, for ncu captures.

    python tools/prof_heat.py --n 128 --N 256 --S 64 [--reps 2]
"""
import argparse
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--n", type=int, default=128)
    p.add_argument("--N", type=int, default=256)
    p.add_argument("--S", type=int, default=64)
    p.add_argument("--reps", type=int, default=2)
    a = p.parse_args()
    import torch

    from paper_1304_6514_b200 import capi
    from paper_1304_6514_b200.dist import HeatPlan

    torch.cuda.set_device(0)
    ctx = capi.Context(0, stream=torch.cuda.current_stream())
    dx, dt = 1.0 / (a.n + 1), 10.0 / (a.N * a.S)
    plan = HeatPlan(ctx, dx, dt, 10.0, a.N)
    for _ in range(a.reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        plan.step()
        e.record()
        e.synchronize()
        print(f"step {s.elapsed_time(e):.3f} ms  y[0]={plan.y[0].item():.15g}")


if __name__ == "__main__":
    main()
