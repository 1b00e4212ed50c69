"""Time the DMMA pair kernel (pint_affine_pair_dev: P products of augmented n x (n+1) maps) against
cuBLAS batched DGEMM (torch.bmm, same shapes) with CUDA events; also the ncu target.

    python tools/prof_pair.py [--n 512] [--P 128] [--reps 5] [--no-cublas]
"""
import argparse
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--P", type=int, default=128)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--no-cublas", action="store_true")
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--tree", type=int, default=0, help="also time the full tree over this many maps (to one map)")
    a = ap.parse_args()
    import torch

    from paper_1304_6514_b200 import capi

    torch.cuda.set_device(0)
    ctx = capi.Context(0, stream=torch.cuda.current_stream())
    n, P = a.n, a.P
    ldm = int(capi.load().pint_affine_ldm(n))
    g = torch.Generator(device="cuda").manual_seed(1)
    E = torch.randn(P, n, ldm, dtype=torch.float64, device="cuda", generator=g) / n ** 0.5
    L = torch.randn(P, n, ldm, dtype=torch.float64, device="cuda", generator=g) / n ** 0.5
    O = torch.empty_like(E)
    flops = 2.0 * P * n * n * (n + 1)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    best = 1e9
    for r in range(a.reps + 1):
        ev[0].record()
        ctx.call("pint_affine_pair_dev", n, P, capi.ptr(E), capi.ptr(L), capi.ptr(O))
        ev[1].record()
        ev[1].synchronize()
        if r:
            best = min(best, ev[0].elapsed_time(ev[1]))
    print(f"pair  n={n} P={P}: {best:.3f} ms  {flops / best / 1e9:.2f} TFLOP/s", flush=True)
    if a.check:
        ref = torch.bmm(L[:, :, :n], E[:, :, : n + 1])
        ref[:, :, n] += L[:, :, n]
        d = (O[:, :, : n + 1] - ref).abs().max().item()
        print(f"max |pair - bmm| = {d:.3e}")
    if not a.no_cublas:
        torch.backends.cuda.matmul.allow_tf32 = False
        A = L[:, :, :n].contiguous()
        B = E[:, :, : n + 1].contiguous()
        best = 1e9
        for r in range(a.reps + 1):
            ev[0].record()
            torch.bmm(A, B)
            ev[1].record()
            ev[1].synchronize()
            if r:
                best = min(best, ev[0].elapsed_time(ev[1]))
        print(f"cuBLAS bmm n={n} P={P}: {best:.3f} ms  {flops / best / 1e9:.2f} TFLOP/s", flush=True)

    if a.tree:
        N = a.tree
        maps = torch.randn(N, n, ldm, dtype=torch.float64, device="cuda", generator=g) / n ** 0.5
        scratch = torch.empty((N + 1) // 2, n, ldm, dtype=torch.float64, device="cuda")
        y0 = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
        y = torch.empty(n, dtype=torch.float64, device="cuda")
        comp = torch.empty(n, ldm, dtype=torch.float64, device="cuda")
        best = 1e9
        for r in range(a.reps + 1):
            work = maps.clone()
            ev[0].record()
            ctx.call("pint_affine_compose_dev", capi.COMPOSE_TREE, n, N, capi.ptr(work), capi.ptr(scratch),
                     capi.ptr(y0), capi.ptr(y), capi.ptr(comp))
            ev[1].record()
            ev[1].synchronize()
            if r:
                best = min(best, ev[0].elapsed_time(ev[1]))
        tf = 2.0 * (N - 1) * n * n * (n + 1)
        print(f"tree  n={n} N={N} (to one map): {best:.3f} ms  {tf / best / 1e9:.2f} TFLOP/s", flush=True)


if __name__ == "__main__":
    main()
