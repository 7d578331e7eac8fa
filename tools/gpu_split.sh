#!/bin/bash
# time split of the fused kernel: full / no phase B / no phase A math / neither, R=128 and 256
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for w in c2a c2; do for R in 128 256; do for D in 0 1 2 3; do
  TGK_FUSED_R=$R TGK_FUSED_DEBUG=$D timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/split_${w}_${R}_$D.json 2>/dev/null
done; done; done
for w in c2a c2; do for R in 128 256; do TGK_FUSED_R=$R timeout 300 python tools/trace_fused.py $w gpurun_out/trace_${w}_$R.bin > gpurun_out/trace_${w}_$R.txt 2>&1; done; done
for f in gpurun_out/split_*.json; do python -c "
import json; d=json.load(open('$f')); print('$f'.split('split_')[1][:-5].ljust(14), round(d['ms_per_step']*1e3,1), 'us', round(d['config']['fused_plan']['recompute_factor'],3), d['config']['fused_plan']['blocks'])" 2>/dev/null || echo "$f failed"; done
cat gpurun_out/trace_*.txt
