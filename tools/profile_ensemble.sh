cd ${GRAFT_REPO_ROOT:-.}
rm -f gpurun_out/ensemble.jsonl
for S in 977 9766; do python tools/prof_ensemble.py --S $S >> gpurun_out/ensemble.jsonl; done
python tools/prof_ensemble.py --S 9766 --prec f32 >> gpurun_out/ensemble.jsonl
python tools/prof_ensemble.py --kind riccati --M 512 --S 782 >> gpurun_out/ensemble.jsonl
python tools/prof_ensemble.py --kind riccati --M 1024 --S 7813 >> gpurun_out/ensemble.jsonl
cat gpurun_out/ensemble.jsonl
ncu --set full --import-source on --clock-control none -k regex:scalar_ensemble_kernel -c 2 -o gpurun_out/ens python tools/prof_ensemble.py --S 9766 --reps 1 > gpurun_out/ncu_ens.log 2>&1; echo ncu=$?
