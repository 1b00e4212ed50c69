"""Where the fixed per-call time of pint_run_scalar goes (the Table-3 rows, bench.py --cost-model).

    python tools/scalar_overhead.py [--trace]

Prints the median wall time of pint_run_scalar for the paper's rows and for S = 1 (no stepping),
the bare round trip of a small pinned H2D + D2H + stream sync, and with --trace the device
timeline (torch.profiler / CUPTI sees every kernel and copy in the process) of one call.
"""
import argparse
import ctypes as C
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trace", action="store_true")
    ap.add_argument("--reps", type=int, default=50)
    a = ap.parse_args()
    import torch

    from paper_1304_6514_b200 import capi

    torch.cuda.set_device(0)
    ctx = capi.Context(0)
    rhs = capi.ScalarRHS(capi.RHS_RICCATI_BE, capi.F64, 0.0, 0.0)
    y, rep, fail = C.c_double(), capi.Report(), capi.Fail()

    def call(dt, N, M, mode=capi.SWEEP_EXACT):
        ctx.check(ctx.lib.pint_run_scalar(ctx.h, C.byref(rhs), 0.0, 0.5, 1.0, N, dt, capi.NODES_SECOND_KIND, M, 0.0,
                                          2.0, capi.WEIGHTS_PRODUCT, mode, C.byref(y), None, None, None,
                                          C.byref(rep), C.byref(fail)))

    def med(f, reps):
        for _ in range(3):
            f()
        w = []
        for _ in range(reps):
            t = time.perf_counter()
            f()
            w.append(time.perf_counter() - t)
        return 1e6 * statistics.median(w)

    rows = [(0.5 / N, N, 4) for N in (32, 128)] + [(6.103515625e-05, N, 4) for N in (32, 64, 128)] + \
           [(1.52587890625e-05, N, 7) for N in (32, 64, 128)]
    for dt, N, M in rows:
        tot, dev = [], []

        def rec():
            call(dt, N, M)
            tot.append(rep.total_ms * 1e3)
            dev.append(rep.device_ms * 1e3)

        w = med(rec, a.reps)
        print(f"run_scalar dt={dt:.3g} N={N} M={M} S={round(0.5 / dt / N)}: {w:.1f} us "
              f"(inside the C call {statistics.median(tot):.1f}, device events {statistics.median(dev):.1f})")
    h = torch.empty(64, dtype=torch.float64, pin_memory=True)
    d = torch.empty(64, dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream()

    def rt():
        d.copy_(h, non_blocking=True)
        h.copy_(d, non_blocking=True)
        s.synchronize()

    print(f"bare H2D + D2H + sync: {med(rt, a.reps):.1f} us")
    if a.trace:
        from torch.profiler import ProfilerActivity, profile
        for dt, N, M in [(6.103515625e-05, 64, 4), (1.52587890625e-05, 32, 7)]:
            call(dt, N, M)
            torch.cuda.synchronize()
            with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as p:
                for _ in range(3):
                    call(dt, N, M)
                torch.cuda.synchronize()
            evs = [e for e in p.events() if e.device_type.name == "CUDA"]
            evs.sort(key=lambda e: e.time_range.start)
            t0 = evs[-1].time_range.start
            # the last call's events
            last = [e for e in evs if e.time_range.start >= evs[len(evs) * 2 // 3].time_range.start]
            t0 = last[0].time_range.start
            print(f"--- device timeline, dt={dt} N={N} M={M} (us from the first event)")
            for e in last:
                print(f"  {e.time_range.start - t0:8.1f} {e.time_range.end - e.time_range.start:8.1f}  {e.name[:70]}")


if __name__ == "__main__":
    main()
