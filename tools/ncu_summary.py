"""Summarise `ncu --set full` captures into profiles/ (run HERE, on the .ncu-rep files gpurun
brought back):

    python tools/ncu_summary.py gpurun_out/full.ncu-rep --round r01

Writes profiles/<round>_ncu_summary.json (key metrics + top stall reasons per kernel) and
profiles/<round>_build_traffic.json (DRAM bytes per heat_build_kernel launch, read by bench.py).
"""
import argparse
import csv
import io
import json
import pathlib
import subprocess
from collections import defaultdict

ROOT = pathlib.Path(__file__).resolve().parents[1]
METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__warps_eligible.avg.per_cycle_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "sm__cycles_active.avg", "lts__t_sector_hit_rate.pct",
]


def ncu(*args) -> str:
    return subprocess.run(["ncu", *args], capture_output=True, text=True, check=True).stdout


def main():
    p = argparse.ArgumentParser()
    p.add_argument("report")
    p.add_argument("--round", default="r01")
    p.add_argument("--name", default="", help="summary of another capture: profiles/<round>_<name>_ncu_summary.json")
    p.add_argument("--config", default="128,256,256", help="n,N,S of the capture (build traffic file)")
    a = p.parse_args()
    raw = list(csv.reader(io.StringIO(ncu("-i", a.report, "--page", "raw", "--csv"))))
    hdr, units, rows = raw[0], raw[1], raw[2:]
    col = {h: i for i, h in enumerate(hdr)}
    stall_cols = [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
    out, seen = {}, defaultdict(int)
    for r in rows:
        name = r[col["Kernel Name"]].split("(")[0].replace("void ", "").split("::")[-1]
        seen[name] += 1
        key = f"{name} #{seen[name]}"
        d = {m: f"{r[col[m]]} {units[col[m]]}".strip() for m in METRICS if m in col}
        st = {h.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(r[col[h]] or 0) for h in stall_cols}
        tot = sum(st.values()) or 1.0
        d["top_stalls_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(st.items(), key=lambda x: -x[1])[:6]}
        out[key] = d
    prof = ROOT / "profiles"
    if a.name:
        (prof / f"{a.round}_{a.name}_ncu_summary.json").write_text(json.dumps(out, indent=1) + "\n")
        print(json.dumps({k: {m: v.get(m) for m in ("gpu__time_duration.sum", "dram__bytes_read.sum")}
                          for k, v in out.items()}, indent=1))
        return
    (prof / f"{a.round}_ncu_summary.json").write_text(json.dumps(out, indent=1) + "\n")
    # the dominant launch: the basis grid (mode 0), else any build kernel
    import re
    basis = re.compile(r"heat_build_kernel<\d+, [03], 0>")  # the basis grid (modes 0 / 3), unguarded
    build = [v for k, v in out.items() if basis.match(k)] or \
        [v for k, v in out.items() if k.startswith("heat_build_kernel")]
    if build:
        b = build[0]

        def val(m):
            num, unit = b[m].split()[0], b[m].split()[-1]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            return float(num.replace(",", "")) * scale

        traffic = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
        (prof / f"{a.round}_build_traffic.json").write_text(json.dumps({
            "kernel": "heat_build_kernel (basis grid)", "dram_bytes_per_launch": int(traffic),
            "config": [int(v) for v in a.config.split(",")],
            "source": f"profiles/{a.round}_ncu_summary.json (ncu --set full, one launch, n=128 N=256 S=256)"},
            indent=1) + "\n")
    print(json.dumps({k: {m: v.get(m) for m in ("gpu__time_duration.sum", "dram__bytes_read.sum")}
                      for k, v in out.items()}, indent=1))


if __name__ == "__main__":
    main()
