#!/bin/bash
# v4 fused kernel: GPU parity tests, then a block-shape sweep on C2a / C2 (device time only)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
for w in c2a c2; do for RT in ${SHAPES:-"128 128" "256 128" "256 256" "512 256"}; do
  set -- $RT
  TGK4_R=$1 TGK4_T=$2 timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/v4_${w}_$1_$2.json 2> gpurun_out/v4_${w}_$1_$2.err
  python -c "
import json; d=json.load(open('gpurun_out/v4_${w}_$1_$2.json')); print('$w R=$1 T=$2', round(d['ms_per_step']*1e3,1), 'us frac', round(d['roofline']['frac'],3))" 2>/dev/null || (echo "$w $1 $2 failed"; tail -3 gpurun_out/v4_${w}_$1_$2.err)
done; done
