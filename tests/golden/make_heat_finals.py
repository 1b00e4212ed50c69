"""Regenerate tests/golden/heat_finals.npz: the UNMODIFIED reference's final states at the bench
configurations (BASELINE.json configs[1] and configs[3]), for bench.py's in-run parity check and
the full-size GPU parity tests.

    c2_final: pint::run_nievergelt(make_heat_problem(1/129, 10/(256*256), 10), N=256).final_state
    c4_final: pint::run_nievergelt(make_heat_problem(1/513, 10/(4096*16), 10), N=4096).final_state

Both come from oracle/_ref/ref_tool bench-heat --final-out (the reference compiled from its own
sources by oracle/Makefile; the tool calls only the reference's public API). Run here, in the
build container (the GPU box has no /root/reference); C4 takes about a minute on 8 host cores and
~9 GB of host memory (the reference keeps all 4096 dense 512 x 512 maps):

    make -C oracle && python tests/golden/make_heat_finals.py
"""
import pathlib
import subprocess
import sys
import tempfile

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[2]
TOOL = ROOT / "oracle" / "_ref" / "ref_tool"
OUT = pathlib.Path(__file__).resolve().parent / "heat_finals.npz"
CASES = {"c2": (128, 256, 256), "c4": (512, 4096, 16)}  # n, N slices, S steps per slice


def main() -> int:
    if not TOOL.exists():
        print(f"missing {TOOL}; run `make -C oracle` first", file=sys.stderr)
        return 1
    arrays = {}
    with tempfile.TemporaryDirectory() as tmp:
        for name, (n, N, S) in CASES.items():
            path = pathlib.Path(tmp) / f"{name}.f64"
            subprocess.run([str(TOOL), "bench-heat", "--n", str(n), "--N", str(N), "--S", str(S), "--T", "10",
                            "--final-out", str(path)], check=True)
            arrays[f"{name}_final"] = np.fromfile(path, dtype="<f8")
            arrays[f"{name}_config"] = np.array([n, N, S], dtype=np.int64)
            assert arrays[f"{name}_final"].shape == (n,)
    np.savez_compressed(OUT, **arrays)
    print(f"wrote {OUT}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
