#!/bin/bash
# quick performance experiments (bench lines only)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
run() { name=$1; shift; env "$@" timeout 600 python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline $EXTRA > gpurun_out/exp_$name.json 2> gpurun_out/exp_$name.err; }
EXTRA="--workload c2a"
run c2a_base
run c2a_noB TGK_FUSED_DEBUG=1
run c2a_noA TGK_FUSED_DEBUG=2
run c2a_noAB TGK_FUSED_DEBUG=3
run c2a_r128 TGK_FUSED_R=128
run c2a_r128_noB TGK_FUSED_R=128 TGK_FUSED_DEBUG=1
run c2a_r128_noA TGK_FUSED_R=128 TGK_FUSED_DEBUG=2
EXTRA="--workload c2"
run c2_base
run c2_noB TGK_FUSED_DEBUG=1
run c2_noA TGK_FUSED_DEBUG=2
for f in gpurun_out/exp_*.json; do python -c "
import json; d=json.load(open('$f')); print('$f'.split('exp_')[1][:-5].ljust(16), round(d['ms_per_step']*1e3,1), 'us')" 2>/dev/null || echo "$f failed"; done
