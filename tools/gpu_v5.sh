#!/bin/bash
# v5 fused kernel: GPU parity tests (TGK_FUSED_V=5), then device-time sweep vs v3
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TGK_FUSED_V=5 timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_v5.log 2>&1
tail -3 gpurun_out/pytest_gpu_v5.log
for w in c2a c2; do
  for cfg in "3 128" "5 64" "5 128" "5 256"; do set -- $cfg
    TGK_PLAN_STATS=1 TGK_FUSED_V=$1 TGK5_R=$2 timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/v5_${w}_$1_$2.json 2> gpurun_out/v5_${w}_$1_$2.err
    python -c "
import json; d=json.load(open('gpurun_out/v5_${w}_$1_$2.json')); print('$w v$1 R=$2', round(d['ms_per_step']*1e3,1), 'us frac', round(d['roofline']['frac'],3))" 2>/dev/null || (echo "$w v$1 $2 failed"; tail -3 gpurun_out/v5_${w}_$1_$2.err)
    grep plan5 gpurun_out/v5_${w}_$1_$2.err
  done
done
