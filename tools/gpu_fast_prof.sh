#!/bin/bash
# ncu capture of k_fast_scalar on C2a (args: R T [tag])
R=${1:-32}; T=${2:-256}; TAG=${3:-}
TGK_FAST_VERBOSE=1 TGK_FAST_R=$R TGK_FAST_T=$T timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fast_scalar -c 1 -o gpurun_out/fast_c2a_R${R}_T${T}${TAG} -f python tools/fast_bench.py c2a --reps 1 --modes fast > gpurun_out/ncu_fast_R${R}.log 2>&1
grep "\[fast\]" gpurun_out/ncu_fast_R${R}.log | head -2; tail -2 gpurun_out/ncu_fast_R${R}.log
