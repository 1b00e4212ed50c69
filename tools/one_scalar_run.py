import ctypes as C, sys
sys.path.insert(0, '.')
from paper_1304_6514_b200 import capi
ctx = capi.Context(0)
rhs = capi.ScalarRHS(capi.RHS_RICCATI_BE, capi.F64, 0.0, 0.0)
y, rep, fail = C.c_double(), capi.Report(), capi.Fail()
for i in range(3):
    ctx.check(ctx.lib.pint_run_scalar(ctx.h, C.byref(rhs), 0.0, 0.5, 1.0, 128, 6.103515625e-05, capi.NODES_SECOND_KIND, 4, 0.0, 2.0, capi.WEIGHTS_PRODUCT, capi.SWEEP_EXACT, C.byref(y), None, None, None, C.byref(rep), C.byref(fail)))
