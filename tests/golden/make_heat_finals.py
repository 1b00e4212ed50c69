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

It also stores {c2,c4}_truth: the same problem solved serially in long double
(tests/golden/heat_truth.c), the near-exact answer. The reference's own FP64 rounding puts its C4
final state ~2.6e-12 (relative, max-norm) from it (C2: ~9e-14), which bounds how closely ANY
differently-ordered FP64 computation (the tolerance build, heat_fast.cu) can match the reference.
`--truth-only` recomputes just these (seconds; keeps the reference finals).
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


def truths() -> dict:
    out = {}
    with tempfile.TemporaryDirectory() as tmp:
        exe = pathlib.Path(tmp) / "heat_truth"
        subprocess.run(["gcc", "-O2", str(pathlib.Path(__file__).resolve().parent / "heat_truth.c"), "-o", str(exe),
                        "-lm"], check=True)
        for name, (n, N, S) in CASES.items():
            txt = subprocess.run([str(exe), str(n), str(N * S)], check=True, capture_output=True, text=True).stdout
            out[f"{name}_truth"] = np.array([float(v) for v in txt.split()])
            assert out[f"{name}_truth"].shape == (n,)
    return out


def main() -> int:
    if "--truth-only" in sys.argv:
        z = dict(np.load(OUT))
        z.update(truths())
        np.savez_compressed(OUT, **z)
        print(f"updated {OUT}")
        return 0
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
    arrays.update(truths())
    np.savez_compressed(OUT, **arrays)
    print(f"wrote {OUT}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
