"""Multi-GPU runs of the nonlinear configs, one process per GPU:

    python -m torch.distributed.run --nnodes=1 --nproc-per-node G --master-addr 127.0.0.1 \\
        --master-port 29511 tools/config_bench_dist.py [--cases c5 c3] [--steps 10 --warmup 3]

c5: config 5's strong-scaling sweep — the scalar problem at fixed N = 64 slices x M = 1024
    trajectories x S steps (M*S ~ 1e5, 1e6, 1e7 per slice), logistic RK4 (FP64). Slices shard in
    contiguous blocks (dist.ScalarPlan), the endpoint tables are gathered to rank 0 (ONE NCCL
    gather, dist.gather_rows) and rank 0 runs the ordered sweep (dist.sharded_scalar_run).
c3: config 3 — Lotka-Volterra tensor-grid tables (N = 512 slices of 256 x 256) built per block,
    the running value handed rank to rank (the paper's lambda chain, dist.sharded_lv_run).
Time = CUDA events between barriers, max over ranks (all_reduce MAX); rank 0 prints one JSON line
per case with traj-steps/s for the whole job.
"""
import argparse
import json
import os
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--cases", nargs="+", default=["c5", "c3"])
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    a = p.parse_args()
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1304_6514_b200 import capi
    from paper_1304_6514_b200.dist import LVPlan, ScalarPlan, sharded_lv_run, sharded_scalar_run, slice_block

    rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    ctx = capi.Context(local, stream=torch.cuda.current_stream())

    def timed(run):
        for _ in range(a.warmup):
            run()
        torch.cuda.synchronize()
        dist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        out = None
        for _ in range(a.steps):
            out = run()
        e.record()
        torch.cuda.synchronize()
        t = torch.tensor([s.elapsed_time(e) / a.steps], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item()), out

    if "c5" in a.cases:
        N, M = 64, 1024
        rhs = capi.ScalarRHS(capi.RHS_LOGISTIC_RK4, capi.F64, 1.0, 1.0)
        for S in (98, 977, 9766):
            lo, hi = slice_block(N, world, rank)
            plan = ScalarPlan(ctx, rhs, 0.0, 10.0, 0.1, N, 10.0 / (N * S), M, 0.0, 1.25,
                              weight_kind=capi.WEIGHTS_CLOSED2, lo=lo, hi=hi)
            ms, out = timed(lambda: sharded_scalar_run(plan))
            if rank == 0:
                y = float(out[0]) if isinstance(out, tuple) else float(out)
                print(json.dumps({"config": "c5 logistic RK4 (strong scaling)", "n_gpus": world, "N": N, "M": M,
                                  "S": S, "ms_per_solve": ms, "traj_steps_per_s": N * M * S / (ms * 1e-3),
                                  "collective": "one NCCL gather of the endpoint tables to rank 0", "final": y}),
                      flush=True)
    if "c3" in a.cases:
        N, Mg = 512, 256
        un = 0.1 + ((8.0 - 0.1) * np.arange(Mg, dtype=np.float64)) / (Mg - 1)  # uniform grid on [0.1, 8]
        for S in (8, 64):
            lo, hi = slice_block(N, world, rank)
            plan = LVPlan(ctx, [1.5, 1.0, 1.0, 3.0], 10.0, N, S, un, un, lo, hi)
            ms, out = timed(lambda: sharded_lv_run(plan, 1.0, 1.0))
            if rank == 0:
                print(json.dumps({"config": "c3 Lotka-Volterra (strong scaling: N fixed, lambda chain)", "n_gpus": world,
                                  "N": N, "grid": f"{Mg}x{Mg}", "S": S, "ms_per_solve": ms,
                                  "traj_steps_per_s": N * Mg * Mg * S / (ms * 1e-3),
                                  "collective": f"{world - 1} point-to-point hand-offs of (u, v)",
                                  "final": [float(x) for x in np.asarray(out.cpu())]}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
