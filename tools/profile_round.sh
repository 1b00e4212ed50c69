#!/bin/bash
# The round's measurement pass, run ON the GPU box from the repo root (each ncu pass only after the
# same command has exited 0 without ncu):
#   gpurun --timeout 1800 -- 'bash tools/profile_round.sh'
# then, here: python tools/ncu_summary.py gpurun_out/full.ncu-rep --round rNN
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"
python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_small.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
      python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "launches rc=$?"
python tools/prof_heat.py --n 128 --N 256 --S 256 --reps 1 > gpurun_out/prof_heat.log 2>&1 && \
  ncu --set full --import-source on --clock-control none \
      -k regex:"heat_build_kernel|heat_record_kernel|affine_pair_kernel|affine_chain" -c 8 \
      -o gpurun_out/full python tools/prof_heat.py --n 128 --N 256 --S 256 --reps 1 > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
tail -c 3000 gpurun_out/bench_full.log; tail -c 600 gpurun_out/bench_ref.log
