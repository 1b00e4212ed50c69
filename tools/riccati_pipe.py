"""One C5 Riccati run (N=64, M=1024, S=9766) for an ncu pipe-utilisation capture of the ensemble kernel."""
import ctypes as C
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
from paper_1304_6514_b200 import capi  # noqa: E402

ctx = capi.Context(0)
rhs = capi.ScalarRHS(capi.RHS_RICCATI_BE, capi.F64, 0.0, 0.0)
y, rep, fail = C.c_double(), capi.Report(), capi.Fail()
N, M, S = 64, 1024, 9766
ctx.check(ctx.lib.pint_run_scalar(ctx.h, C.byref(rhs), 0.0, 0.5, 1.0, N, 0.5 / (N * S), capi.NODES_SECOND_KIND, M, 0.0,
                                  2.0, capi.WEIGHTS_CLOSED2, capi.SWEEP_EXACT, C.byref(y), None, None, None,
                                  C.byref(rep), C.byref(fail)))
print(y.value, rep.device_ms)
