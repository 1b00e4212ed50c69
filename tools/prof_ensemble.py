"""Ensemble-integrator (K1) throughput on device-resident inputs, for profiling and DESIGN numbers.

    python tools/prof_ensemble.py [--kind logistic|riccati] [--prec f64|f32] [--N 64] [--M 1024] [--S 977]

Prints one JSON line: kernel ms (CUDA events, best of reps), traj-steps/s, algorithmic TFLOP/s
(29 flops per logistic RK4 step, 6 per Riccati BE step counting sqrt and div as one each) and
the fraction of the measured FMA peak (tools/probe.py's kernel).
"""
import argparse
import ctypes as C
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--kind", default="logistic", choices=["logistic", "riccati"])
    p.add_argument("--prec", default="f64", choices=["f64", "f32"])
    p.add_argument("--N", type=int, default=64)
    p.add_argument("--M", type=int, default=1024)
    p.add_argument("--S", type=int, default=977)
    p.add_argument("--reps", type=int, default=5)
    a = p.parse_args()
    import numpy as np
    import torch

    from paper_1304_6514_b200 import capi, pint

    torch.cuda.set_device(0)
    stream = torch.cuda.current_stream()
    ctx = capi.Context(0, stream=stream)
    T, lo, hi = (10.0, 0.0, 1.25) if a.kind == "logistic" else (0.5, 0.0, 2.0)
    dec = pint.decompose(0.0, T, a.N, T / (a.N * a.S))
    steps, h = pint.slice_table(dec)
    nodes = pint.cheb_nodes_second_kind(a.M, lo, hi)
    dt = torch.float32 if a.prec == "f32" else torch.float64
    d_steps, d_h = torch.from_numpy(steps).cuda(), torch.from_numpy(h).cuda()
    d_nodes = torch.from_numpy(nodes).to(dt).cuda()
    d_out = torch.empty(a.N * a.M, dtype=dt, device="cuda")
    kind = capi.RHS_LOGISTIC_RK4 if a.kind == "logistic" else capi.RHS_RICCATI_BE
    rhs = capi.ScalarRHS(kind, capi.F32 if a.prec == "f32" else capi.F64, 1.0, 1.0)
    best = 1e30
    for _ in range(a.reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        ctx.call("pint_scalar_ensemble_dev", C.byref(rhs), a.N, a.M, capi.ptr(d_steps), capi.ptr(d_h),
                 capi.ptr(d_nodes), capi.ptr(d_out), None)
        e.record(stream)
        e.synchronize()
        best = min(best, s.elapsed_time(e))
    traj_steps = int(steps.sum()) * a.M
    flops = traj_steps * (29 if a.kind == "logistic" else 6)
    peak = C.c_double()
    ctx.check(ctx.lib.pint_probe_peak(ctx.h, capi.F32 if a.prec == "f32" else capi.F64, C.byref(peak)))
    tf = flops / (best * 1e-3) / 1e12
    print(json.dumps({"kind": a.kind, "prec": a.prec, "N": a.N, "M": a.M, "S": a.S, "kernel_ms": best,
                      "traj_steps_per_s": traj_steps / (best * 1e-3), "algorithmic_tflops": tf,
                      "measured_peak_tflops": peak.value, "frac_of_peak": tf / peak.value,
                      "checksum": float(d_out.double().sum().item())}))


if __name__ == "__main__":
    main()
