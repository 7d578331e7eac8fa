#!/bin/bash
# ncu full capture of the v4 fused kernel (C2a) + plan statistics
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
W=${W:-c2a}
for RT in ${SHAPES:-"128 128" "256 256"}; do set -- $RT
TGK_PLAN_STATS=1 TGK4_R=$1 TGK4_T=$2 timeout 300 python bench.py --workload $W --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline 2>&1 | grep plan4
done
set -- ${PROF:-128 128}
TGK4_R=$1 TGK4_T=$2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 3 -c 1 \
  -o gpurun_out/prof4_$W python bench.py --workload $W --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu4_$W.log 2>&1
