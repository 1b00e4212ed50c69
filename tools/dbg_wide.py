import sys, pathlib, numpy as np
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import oracle as O
from paper_1304_6514_b200 import capi, pint
from paper_1304_6514_b200.dist import HeatPlan
ctx = pint.context()
P = capi.ptr
for (n, N, S) in [(512, 600, 2), (512, 600, 16), (512, 200, 2), (512, 64, 2), (384, 100, 2), (272, 50, 2)]:
    dx, dt = 1.0 / (n + 1), 1e-4
    plan = HeatPlan(ctx, dx, dt, N * S * dt, N)
    step_off, slice_dt, r, fa, fb, sx = plan.dev
    ctx.call("pint_heat_factor_dev", n, N, plan.S, P(step_off), P(slice_dt), P(r), P(fa), P(fb), P(sx), P(plan.factor))
    res = []
    for it in range(3):
        plan.y.zero_()
        plan.maps.fill_(float('nan'))
        ctx.call("pint_heat_build_chain_dev", n, N, plan.S, P(step_off), P(slice_dt), P(plan.factor), P(sx),
                 P(plan.maps), P(plan.y0), P(plan.y), 0)
        ctx.sync()
        ok = plan.verify()
        host = plan.maps.view(N, n, plan.ldm).cpu().numpy()
        y0 = plan.y0.cpu().numpy()
        y_or = O.affine_chain(host[:, :, :n], host[:, :, n], y0)
        y = plan.y.cpu().numpy()
        res.append((ok, bool(np.array_equal(y, y_or)), float(np.max(np.abs(y - y_or))), int(np.isnan(y).sum())))
    # standalone chain (no build beside it) through compose_local
    plan.compose_local(capi.COMPOSE_CHAIN, want_composed=False); ctx.sync()
    y2 = plan.y.cpu().numpy()
    print(n, N, S, res, "standalone", bool(np.array_equal(y2, y_or)), flush=True)
