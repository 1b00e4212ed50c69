"""Stress the concurrent chain + build (ready counters, PDL) and the tolerance build: many
consecutive pint_run_heat calls, every final state compared bit-for-bit with the first (exact) and
with the first fast one.    python tools/stress_overlap.py [--iters 100]"""
import argparse
import pathlib
import sys

import numpy as np

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=100)
    a = ap.parse_args()
    from paper_1304_6514_b200 import capi, pint

    ctx = pint.context()
    bad = 0
    for (n, N, S) in ((512, 256, 4), (384, 333, 3), (300, 128, 2)):
        dx, dt = 1.0 / (n + 1), 1e-4
        T = N * S * dt
        ref = {}
        for it in range(a.iters):
            for mode in (capi.BUILD_EXACT, capi.BUILD_FAST):
                y = np.empty(n)
                ctx.check(ctx.lib.pint_run_heat_ex(ctx.h, dx, dt, T, N, mode, capi.COMPOSE_CHAIN, None, capi.ptr(y),
                                                   None, None))
                if mode not in ref:
                    ref[mode] = y.copy()
                elif not np.array_equal(y, ref[mode]):
                    bad += 1
                    print(f"MISMATCH n={n} it={it} mode={mode} max={np.max(np.abs(y - ref[mode]))}", flush=True)
        print(f"n={n} N={N} S={S}: {a.iters} x 2 runs, mismatches so far {bad}", flush=True)
    print("stress", "FAILED" if bad else "ok")


if __name__ == "__main__":
    main()
