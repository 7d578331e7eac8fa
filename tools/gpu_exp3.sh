#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
L=paper_2602_05052_b200/lib
run() { name=$1; shift; env "$@" timeout 600 python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline $EXTRA > gpurun_out/exp_$name.json 2> gpurun_out/exp_$name.err; }
for w in c2a c2; do
EXTRA="--workload $w"
run ${w}_base
run ${w}_ring3 TGK_LIB=$L/libtgk_ring3.so
run ${w}_ring3m5 TGK_LIB=$L/libtgk_ring3m5.so
run ${w}_r64 TGK_LIB=$L/libtgk_r64.so TGK_FUSED_R=64
run ${w}_r64ring3 TGK_LIB=$L/libtgk_r64ring3.so TGK_FUSED_R=64
done
for f in gpurun_out/exp_*.json; do python -c "
import json; d=json.load(open('$f')); print('$f'.split('exp_')[1][:-5].ljust(16), round(d['ms_per_step']*1e3,1), 'us', d['config']['fused_plan']['recompute_factor'])" 2>/dev/null || echo "$f failed"; done
