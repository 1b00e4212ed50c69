"""Print measured FP64/FP32 peaks and dependent-chain latencies of this GPU."""
import ctypes as C
import json
import pathlib
import sys

import numpy as np

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
from paper_1304_6514_b200 import capi  # noqa: E402

ctx = capi.Context(0)
p64, p32, pmma = C.c_double(), C.c_double(), C.c_double()
ctx.check(ctx.lib.pint_probe_peak(ctx.h, 2, C.byref(pmma)))  # PINT_PROBE_DMMA
ctx.check(ctx.lib.pint_probe_peak(ctx.h, capi.F64, C.byref(p64)))
ctx.check(ctx.lib.pint_probe_peak(ctx.h, capi.F32, C.byref(p32)))
lat = np.zeros(8)
ctx.check(ctx.lib.pint_probe_latency(ctx.h, capi.ptr(lat)))
print(json.dumps({"fp64_fma_tflops": p64.value, "fp32_fma_tflops": p32.value, "fp64_dmma_tflops": pmma.value,
                  "latency_cycles": dict(zip(["dfma", "dadd", "dmul", "ffma", "lds64", "heat_forward_row", "heat_back_row", "dmul_dadd_alt"], lat.tolist()))}))
