"""Regenerate tests/golden/parareal_golden.npz: the UNMODIFIED reference's parareal_sweep
(parareal.cpp:47-190) final_per_iteration, from oracle/_ref/parareal_golden (the reference compiled
from its own sources by oracle/Makefile). Run here (the GPU box has no /root/reference):

    make -C oracle && python tests/golden/make_parareal_golden.py

Cases: acceptance criterion 2's table (model problem, N in {1..64}, k in {2, 3, 5}, dt = 1e-4,
DT = 0.1) plus k = 0 and the unit tests' configurations (test_parareal.cpp); the heat system of
test_parareal.cpp (dx = 0.1, T = 1, N = 4, dt = 0.01, DT = 0.05, k = 1..4) and a 128-point case.
"""
import pathlib
import subprocess
import sys

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[2]
TOOL = ROOT / "oracle" / "_ref" / "parareal_golden"
OUT = pathlib.Path(__file__).resolve().parent / "parareal_golden.npz"

SCALAR = [(N, k, 1e-4, 0.1) for N in (1, 2, 4, 8, 16, 32, 64) for k in (0, 2, 3, 5)] + [
    (4, 3, 1e-3, 0.125), (4, 0, 1e-3, 0.125), (4, 4, 0.01, 0.0625), (4, 5, 0.01, 0.0625), (2, 2, 1e-3, 0.05),
    (100, 3, 1e-4, 0.05)]
HEAT = [(0.1, 1.0, 4, k, 0.01, 0.05) for k in (1, 2, 3, 4)] + [(1.0 / 129, 0.5, 16, 3, 1e-3, 5e-3)]


def run(*args):
    out = subprocess.run([str(TOOL), *map(str, args)], check=True, capture_output=True, text=True).stdout
    rows = [l.split() for l in out.splitlines() if l and l[0].isdigit()]
    return np.array([[float(v) for v in r[1:]] for r in rows])


def main() -> int:
    if not TOOL.exists():
        print(f"missing {TOOL}; run `make -C oracle` first", file=sys.stderr)
        return 1
    z = {}
    for i, (N, k, dt, DT) in enumerate(SCALAR):
        z[f"scalar{i}_cfg"] = np.array([N, k, dt, DT])
        z[f"scalar{i}_finals"] = run("scalar", N, k, repr(dt), repr(DT))[:, 0]
    for i, (dx, T, N, k, dt, DT) in enumerate(HEAT):
        z[f"heat{i}_cfg"] = np.array([dx, T, N, k, dt, DT])
        z[f"heat{i}_finals"] = run("heat", repr(dx), repr(T), N, k, repr(dt), repr(DT))
    np.savez_compressed(OUT, **z)
    print(f"wrote {OUT}: {len(SCALAR)} scalar, {len(HEAT)} heat cases")
    return 0


if __name__ == "__main__":
    sys.exit(main())
