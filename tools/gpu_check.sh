#!/bin/bash
# One GPU pass: gpu tests, smoke, the default bench line and the reference arm.
#   gpurun --timeout 1500 -- 'bash tools/gpu_check.sh [pytest -k expr]'
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
K=${1:+-k "$1"}
timeout 900 python -m pytest tests -m gpu -x -q $K > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
tail -c 2500 gpurun_out/bench.log; echo; tail -c 800 gpurun_out/bench_ref.log
