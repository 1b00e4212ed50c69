"""One-GPU measurements of BASELINE.json's other configs (bench.py runs configs[1] and, with
--n 512, configs[3]'s per-GPU share). One JSON line per case:

    python tools/config_bench.py [--reps 5] [--cases c1ref c1rk4 c5 c3]

c1ref  config 1 on the reference path: y' = y^2 (make_model_problem), backward-Euler Riccati,
       N = 64, M = 512, S in {79, 782}; pint_run_scalar with host buffers vs the unmodified
       reference (oracle/_ref/ref_tool bench-scalar, all host cores).
c1rk4  config 1 as BASELINE.json names it: logistic y' = y (1 - y), RK4, y0 = 0.1 on [0, 10],
       nodes second kind on [0, 1.25], N = 64, M = 1024 (closed-form weights), S = 977.
c5     config 5: the c1rk4 and c1ref problems at M*S ~ 1e5, 1e6, 1e7 trajectory-steps per slice.
c3     config 3: Lotka-Volterra (1.5, 1, 1, 3) from (1, 1) on [0, 10], 256 x 256 uniform grid on
       [0.1, 8]^2 per slice, N = 512, S in {8, 64}: tables (pint_lv_ensemble_dev) + the bilinear
       chain (pint_bilinear_sweep_dev).
Extensions (logistic, LV) have no reference implementation: their CPU figure is the oracle
port (one core) on a bounded sample of slices, scaled.
"""
import argparse
import ctypes as C
import json
import os
import pathlib
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def run_scalar(ctx, capi, kind, N, M, S, reps, closed_weights=False):
    if kind == "riccati":
        rhs = capi.ScalarRHS(capi.RHS_RICCATI_BE, capi.F64, 0.0, 0.0)
        t0, T, y0, a, b, wk = 0.0, 0.5, 1.0, 0.0, 2.0, capi.WEIGHTS_PRODUCT
    else:
        rhs = capi.ScalarRHS(capi.RHS_LOGISTIC_RK4, capi.F64, 1.0, 1.0)
        t0, T, y0, a, b, wk = 0.0, 10.0, 0.1, 0.0, 1.25, capi.WEIGHTS_CLOSED2
    if closed_weights:
        wk = capi.WEIGHTS_CLOSED2
    dt = (T - t0) / (N * S)
    y = C.c_double()
    rep, fail = capi.Report(), capi.Fail()
    walls, dev = [], []
    for i in range(reps + 2):
        t = time.perf_counter()
        ctx.check(ctx.lib.pint_run_scalar(ctx.h, C.byref(rhs), t0, T, y0, N, dt, capi.NODES_SECOND_KIND, M, a, b,
                                          wk, capi.SWEEP_EXACT, C.byref(y), None, None, None, C.byref(rep),
                                          C.byref(fail)))
        w = time.perf_counter() - t
        if i >= 2:
            walls.append(w)
            dev.append(rep.device_ms * 1e-3)
    steps = N * M * S
    return {"traj_steps": steps, "e2e_ms": 1e3 * statistics.median(walls), "device_ms": 1e3 * statistics.median(dev),
            "e2e_traj_steps_per_s": steps / statistics.median(walls),
            "device_traj_steps_per_s": steps / statistics.median(dev), "final": y.value,
            "gpu_launches": int(rep.gpu_launches), "h2d_bytes": int(rep.h2d_bytes), "d2h_bytes": int(rep.d2h_bytes)}


def ref_scalar(N, M, S):
    tool = ROOT / "oracle" / "_ref" / "ref_tool"
    if not tool.exists():
        return None
    cores = os.cpu_count() or 1
    out = subprocess.run([str(tool), "bench-scalar", "--N", str(N), "--M", str(M), "--S", str(S), "--workers",
                          str(cores), "--reps", "2"], capture_output=True, text=True, timeout=600, check=True).stdout
    r = min(json.loads(out), key=lambda x: x["seconds"])
    return {"value": r["traj_steps"] / r["seconds"], "cores": cores, "kind": "reference",
            "sample": f"full pint::run_nievergelt(make_model_problem) N={N} M={M} S={S}", "final": r["final"]}


def port_logistic(N, M, S, sample=4):
    import oracle as O
    from paper_1304_6514_b200 import pint

    dec = O.decompose(0.0, 10.0, N, 10.0 / (N * S))
    steps, h = dec[2][:sample], dec[3][:sample]
    nodes = pint.sample_nodes(pint.SECOND_KIND, M, 0.0, 1.25)
    t = time.perf_counter()
    O.logistic_rk4_ensemble(steps, h, nodes, 1.0, 1.0)
    sec = time.perf_counter() - t
    return {"value": sample * M * S / sec, "cores": 1, "kind": "port",
            "sample": f"oracle logistic_rk4_ensemble, {sample} of {N} slices x {M} ICs x {S} steps"}


def run_lv(ctx, N, Mg, S, reps):
    import torch

    from paper_1304_6514_b200.dist import LVPlan

    LV = [1.5, 1.0, 1.0, 3.0]
    un = 0.1 + ((8.0 - 0.1) * np.arange(Mg, dtype=np.float64)) / (Mg - 1)  # uniform grid on [0.1, 8]
    plan = LVPlan(ctx, LV, 10.0, N, S, un, un)
    lam0 = torch.tensor([1.0, 1.0], dtype=torch.float64)
    stream = torch.cuda.current_stream()
    devs, walls = [], []
    out = None
    for i in range(reps + 2):
        torch.cuda.synchronize()
        t = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        plan.build()
        out = plan.sweep_block(lam0)  # (syncs; the result comes back to the host)
        e1.record(stream)
        e1.synchronize()
        w = time.perf_counter() - t
        if i >= 2:
            walls.append(w)
            devs.append(e0.elapsed_time(e1) * 1e-3)
    steps = N * Mg * Mg * S
    return {"traj_steps": steps, "e2e_ms": 1e3 * statistics.median(walls), "device_ms": 1e3 * statistics.median(devs),
            "e2e_traj_steps_per_s": steps / statistics.median(walls),
            "device_traj_steps_per_s": steps / statistics.median(devs), "final": [float(x) for x in out.cpu()],
            "flops_per_traj_step": 54}


def port_lv(N, Mg, S, sample=2):
    import oracle as O

    LV = [1.5, 1.0, 1.0, 3.0]
    un = O.uniform_nodes(Mg, 0.1, 8.0)
    dec = O.decompose(0.0, 10.0, N, 10.0 / (N * S))
    t = time.perf_counter()
    O.lv_rk4_ensemble(dec[2][:sample], dec[3][:sample], un, un, LV)
    sec = time.perf_counter() - t
    return {"value": sample * Mg * Mg * S / sec, "cores": 1, "kind": "port",
            "sample": f"oracle lv_rk4_ensemble, {sample} of {N} slices x {Mg}^2 ICs x {S} steps"}


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--reps", type=int, default=5)
    p.add_argument("--cases", nargs="+", default=["c1ref", "c1rk4", "c5", "c3"])
    a = p.parse_args()
    import torch

    from paper_1304_6514_b200 import capi

    torch.cuda.set_device(0)
    ctx = capi.Context(0, stream=torch.cuda.current_stream())
    peak = C.c_double()
    ctx.check(ctx.lib.pint_probe_peak(ctx.h, capi.F64, C.byref(peak)))

    def emit(d):
        print(json.dumps(d), flush=True)

    if "c1ref" in a.cases:
        for S in (79, 782):
            r = run_scalar(ctx, capi, "riccati", 64, 512, S, a.reps)
            emit({"config": "c1 reference path (Riccati BE)", "N": 64, "M": 512, "S": S, **r,
                  "cpu_baseline": ref_scalar(64, 512, S)})
    if "c1rk4" in a.cases:
        r = run_scalar(ctx, capi, "logistic", 64, 1024, 977, a.reps)
        emit({"config": "c1 logistic RK4", "N": 64, "M": 1024, "S": 977, **r,
              "fp64_frac_of_peak_device": r["device_traj_steps_per_s"] * 29 / (peak.value * 1e12),
              "cpu_baseline": port_logistic(64, 1024, 977)})
    if "c5" in a.cases:
        for S in (98, 977, 9766):
            r = run_scalar(ctx, capi, "logistic", 64, 1024, S, a.reps)
            emit({"config": "c5 logistic RK4", "N": 64, "M": 1024, "S": S, "per_slice_traj_steps": 1024 * S, **r,
                  "fp64_frac_of_peak_device": r["device_traj_steps_per_s"] * 29 / (peak.value * 1e12),
                  "cpu_baseline": port_logistic(64, 1024, S, sample=max(1, min(8, 4000 // S)))})
        for S in (98, 977, 9766):  # (M = 1024: closed-form weights; the reference's product form overflows)
            r = run_scalar(ctx, capi, "riccati", 64, 1024, S, a.reps, closed_weights=True)
            emit({"config": "c5 Riccati BE", "N": 64, "M": 1024, "S": S, "per_slice_traj_steps": 1024 * S, **r})
    if "c3" in a.cases:
        for S in (8, 64):
            r = run_lv(ctx, 512, 256, S, a.reps)
            emit({"config": "c3 Lotka-Volterra RK4 + bilinear chain", "N": 512, "grid": "256x256", "S": S, **r,
                  "fp64_frac_of_peak_device": r["device_traj_steps_per_s"] * 54 / (peak.value * 1e12),
                  "cpu_baseline": port_lv(512, 256, S)})


if __name__ == "__main__":
    main()
