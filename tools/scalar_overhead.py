import ctypes as C, time, statistics, sys, json
sys.path.insert(0, '.')
import torch
from paper_1304_6514_b200 import capi
ctx = capi.Context(0)
rhs = capi.ScalarRHS(capi.RHS_RICCATI_BE, capi.F64, 0.0, 0.0)
y, rep, fail = C.c_double(), capi.Report(), capi.Fail()
for (dt, N, M) in [(6.103515625e-05, 32, 4), (6.103515625e-05, 128, 4), (1.52587890625e-05, 32, 512)]:
    w = []; dv = []; tt = []
    for i in range(12):
        t = time.perf_counter()
        ctx.check(ctx.lib.pint_run_scalar(ctx.h, C.byref(rhs), 0.0, 0.5, 1.0, N, dt, capi.NODES_SECOND_KIND, M, 0.0, 2.0, capi.WEIGHTS_PRODUCT, capi.SWEEP_EXACT, C.byref(y), None, None, None, C.byref(rep), C.byref(fail)))
        w.append(time.perf_counter() - t); dv.append(rep.device_ms); tt.append(rep.total_ms)
    print(json.dumps({"dt": dt, "N": N, "M": M, "wall_us": 1e6 * statistics.median(w[2:]), "device_us": 1e3 * statistics.median(dv[2:]), "total_us": 1e3 * statistics.median(tt[2:]), "launches": rep.gpu_launches}))
