#!/bin/bash
# one optimisation iteration: GPU tests, traces, bench lines
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
for w in c2a c2; do for R in ${RS:-128 256}; do TGK_FUSED_R=$R timeout 300 python tools/trace_fused.py $w gpurun_out/trace_${w}_$R.bin > /dev/null 2>&1; done; done
for w in c2a c2; do for R in ${RS:-128 256}; do TGK_FUSED_R=$R timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/exp_${w}_$R.json 2>gpurun_out/exp_${w}_$R.err; done; done
for f in gpurun_out/exp_*.json; do python -c "
import json; d=json.load(open('$f')); print('$f'.split('exp_')[1][:-5].ljust(12), round(d['ms_per_step']*1e3,1), 'us', 'frac', round(d['roofline']['frac'],3))" 2>/dev/null || echo "$f failed"; done
