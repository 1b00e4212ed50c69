"""B200 refit of the paper's GPU cost model (cost_model.cpp:36-81).

Runs ON the GPU box from the repo root:

    python tools/cost_model_refit.py [--reps 7] [--out gpurun_out]

1. Times the scalar benchmark the fixture describes (make_model_problem, y' = y^2 on [0, 0.5],
   backward-Euler Riccati, nodes second kind on [0, 2]) end to end through pint_run_scalar with
   host buffers, at the fixture's own (dt, N, M) rows (reference data/gpu_timings.txt) plus rows
   at larger M where the per-trajectory term matters on a B200.
2. Times the reference's serial run (oracle/_ref/ref_tool bench-serial, one core) for the ratio
   column (ratio * T_total = serial CPU time, as fit_params reads it).
3. Writes the observations in the fixture's 5-column format (profiles/r01_b200_timings.txt) and
   fits them with the reference's own fit_params (ref_tool fit), next to the reference fixture's
   fit, into profiles/r01_cost_model.json.
"""
import argparse
import ctypes as C
import json
import pathlib
import statistics
import subprocess
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
TOOL = ROOT / "oracle" / "_ref" / "ref_tool"
PAPER_ROWS = [(6.103515625e-05, N, 4) for N in (32, 64, 128)] + \
             [(3.0517578125e-05, N, 5) for N in (32, 64, 128)] + \
             [(1.52587890625e-05, N, 7) for N in (32, 64, 128)]
B200_ROWS = [(dt, N, M) for dt in (6.103515625e-05, 1.52587890625e-05) for N in (32, 128) for M in (64, 512)]


def device_total_us(ctx, capi, dt, N, M, reps):
    rhs = capi.ScalarRHS(capi.RHS_RICCATI_BE, capi.F64, 0.0, 0.0)
    y, rep, fail = C.c_double(), capi.Report(), capi.Fail()
    walls = []
    for i in range(reps + 2):
        t = time.perf_counter()
        ctx.check(ctx.lib.pint_run_scalar(ctx.h, C.byref(rhs), 0.0, 0.5, 1.0, N, dt, capi.NODES_SECOND_KIND, M, 0.0,
                                          2.0, capi.WEIGHTS_PRODUCT, capi.SWEEP_EXACT, C.byref(y), None, None, None,
                                          C.byref(rep), C.byref(fail)))
        if i >= 2:
            walls.append(time.perf_counter() - t)
    return 1e6 * statistics.median(walls), y.value


def serial_us(dt):
    out = subprocess.run([str(TOOL), "bench-serial", "--dt", repr(dt), "--reps", "5"], capture_output=True,
                         text=True, check=True, timeout=300).stdout
    return 1e6 * json.loads(out)["seconds"]


def fit(path):
    out = subprocess.run([str(TOOL), "fit", str(path)], capture_output=True, text=True, check=True).stdout
    return json.loads(out)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--reps", type=int, default=7)
    p.add_argument("--out", default="profiles", help="output directory (gpurun_out on the GPU box)")
    a = p.parse_args()
    import torch

    from paper_1304_6514_b200 import capi

    torch.cuda.set_device(0)
    ctx = capi.Context(0)
    lines = ["# B200 (sm_100a) timings for the scalar benchmark, T = 0.5: pint_run_scalar end to end",
             "# (host buffers), median of the reps; ratio = reference run_serial on one host core / T_total.",
             "# Columns: dt, N (slices), M (trajectories), T_total (us), cpu/device ratio."]
    rows = []
    serial = {}
    for dt, N, M in PAPER_ROWS + B200_ROWS:
        if dt not in serial:
            serial[dt] = serial_us(dt)
        tot, y = device_total_us(ctx, capi, dt, N, M, a.reps)
        ratio = serial[dt] / tot
        rows.append({"dt": dt, "N": N, "M": M, "T_total_us": tot, "ratio": ratio, "final": y})
        lines.append(f"{dt!r}, {N}, {M}, {tot:.1f}, {ratio:.4f}")
    prof = ROOT / a.out
    prof.mkdir(exist_ok=True)
    fixture = prof / "r01_b200_timings.txt"
    fixture.write_text("\n".join(lines) + "\n")
    paper_rows = prof / "r01_b200_timings_paper_rows.txt"
    paper_rows.write_text("\n".join(lines[:3 + len(PAPER_ROWS)]) + "\n")
    ref_fixture = ROOT / "oracle" / "_ref" / "dropin" / "data" / "gpu_timings.txt"
    result = {
        "b200_fit_all_rows": fit(fixture),
        "b200_fit_paper_rows": fit(paper_rows),
        "reference_fixture_fit": fit(ref_fixture) if ref_fixture.exists() else None,
        "published": {"tau_F": 0.040, "tau_N": 0.701, "tau_K": 137.0, "tau_F_cpu": 0.051},
        "rows": rows,
        "serial_us": {repr(k): v for k, v in serial.items()},
        "units": "microseconds (tau_F per fine step per trajectory, tau_N per slice, tau_K per run)",
    }
    (prof / "r01_cost_model.json").write_text(json.dumps(result, indent=1) + "\n")
    print(json.dumps({k: result[k] for k in ("b200_fit_all_rows", "b200_fit_paper_rows", "reference_fixture_fit")}))


if __name__ == "__main__":
    main()
