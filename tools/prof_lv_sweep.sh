cd paper_1304_6514_b200 && touch csrc/interp.cu && make -s NVFLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC,-ffp-contract=off,-O2 -I../include -Icsrc -DPINT_SWEEP_PROF" > /dev/null 2>&1; cd ..
python bench.py --configs c3 --config-reps 1 2>&1 | grep -v "^{" | sort | uniq -c
