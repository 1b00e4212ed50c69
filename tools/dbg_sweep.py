import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1] / "tests"))
import numpy as np
from paper_1304_6514_b200 import capi, pint
from test_gpu_parity import run_scalar
ctx = pint.context()
N, M, dt = 64, 512, 0.5 / (64 * 79)
rc, ye, ends, le, *_ = run_scalar(ctx, pint.make_model_problem(), N, dt, M)
rc2, yt, ends2, lt, *_ = run_scalar(ctx, pint.make_model_problem(), N, dt, M, sweep=capi.SWEEP_TREE)
print(rc, rc2, ye, yt)
bad = np.nonzero(~np.isfinite(lt))[0]
print("first bad slice", bad[:5], "lam exact", le[:4], "tree", lt[:4])
j = bad[0] if len(bad) else 0
print("ends row j min/max", ends[j].min(), ends[j].max(), np.isfinite(ends[j]).all())
