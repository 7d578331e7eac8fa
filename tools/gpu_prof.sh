#!/bin/bash
# ncu full captures of the fused kernel: default and phase-B-only (TGK_FUSED_DEBUG=2)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
W=${W:-c2a}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 3 -c 1 \
  -o gpurun_out/prof_$W python bench.py --workload $W --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_$W.log 2>&1
if [ -n "$NOA" ]; then
TGK_FUSED_DEBUG=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 3 -c 1 \
  -o gpurun_out/prof_${W}_noA python bench.py --workload $W --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_${W}_noA.log 2>&1
fi
