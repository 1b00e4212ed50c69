"""Timing driver for the heat map builds: records + build (exact and/or fast) at a chosen size,
CUDA events on the launching stream, after warm-up. Also the ncu target for one build launch.

    python tools/prof_fast.py --n 512 --N 4096 --S 16 [--build fast|exact|both] [--reps 5]
"""
import argparse
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--n", type=int, default=512)
    p.add_argument("--N", type=int, default=4096)
    p.add_argument("--S", type=int, default=16)
    p.add_argument("--reps", type=int, default=5)
    p.add_argument("--build", default="both", choices=["fast", "exact", "both"])
    p.add_argument("--compose", action="store_true", help="also time the chain to y")
    a = p.parse_args()
    import torch

    from paper_1304_6514_b200 import capi
    from paper_1304_6514_b200.dist import HeatPlan

    torch.cuda.set_device(0)
    ctx = capi.Context(0, stream=torch.cuda.current_stream())
    dx, dt = 1.0 / (a.n + 1), 10.0 / (a.N * a.S)
    flops = a.N * a.S * ((a.n + 1) * (5 * a.n - 4) + 5 * a.n)
    builds = ["fast", "exact"] if a.build == "both" else [a.build]
    ref = None
    for b in builds:
        plan = HeatPlan(ctx, dx, dt, 10.0, a.N, build=b)
        P = capi.ptr
        step_off, slice_dt, r, fa, fb, sx = plan.dev
        for rep in range(a.reps + 1):
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            ev[0].record()
            if b == "fast":
                ctx.call("pint_heat_fast_factor_dev", plan.n, plan.N, plan.S, P(step_off), P(slice_dt), P(r), P(fa),
                         P(fb), P(sx), P(plan.factor))
                ev[1].record()
                ctx.call("pint_heat_fast_build_dev", plan.n, plan.N, plan.S, P(plan.factor), P(plan.maps))
            else:
                ctx.call("pint_heat_factor_dev", plan.n, plan.N, plan.S, P(step_off), P(slice_dt), P(r), P(fa), P(fb),
                         P(sx), P(plan.factor))
                ev[1].record()
                ctx.call("pint_heat_build_dev", plan.n, plan.N, plan.S, P(step_off), P(slice_dt), P(plan.factor),
                         P(sx), P(plan.maps), None, 0)
            ev[2].record()
            if a.compose:
                plan.compose_local(capi.COMPOSE_CHAIN, want_composed=False)
            ev[3].record()
            ev[3].synchronize()
            if rep == 0:
                continue
            rec_ms, build_ms, comp_ms = ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3])
            print(f"{b:5s} n={a.n} N={a.N} S={a.S}: records {rec_ms:.3f} ms  build {build_ms:.3f} ms "
                  f"({flops / build_ms / 1e9:.2f} TFLOP/s alg)  compose {comp_ms:.3f} ms", flush=True)
        m = plan.maps.view(plan.N, plan.n, plan.ldm)[:64, :, : plan.n + 1].cpu()
        if ref is None:
            ref = m
        else:
            d = (m - ref).abs().max().item() / ref.abs().max().item()
            print(f"max |{builds[0]} - {b}| / max|map| = {d:.3e}")


if __name__ == "__main__":
    main()
