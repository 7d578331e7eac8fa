#!/bin/bash
# launch-bounds / rows-per-block matrix (bench lines only)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
L=paper_2602_05052_b200/lib
run() { name=$1; shift; env "$@" timeout 600 python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline $EXTRA > gpurun_out/exp_$name.json 2> gpurun_out/exp_$name.err; }
for lib in libtgk libtgk_minb1 libtgk_minb2; do
  EXTRA="--workload c2a"
  run ${lib}_c2a_r256 TGK_LIB=$L/$lib.so TGK_FUSED_R=256
  run ${lib}_c2a_r128 TGK_LIB=$L/$lib.so TGK_FUSED_R=128
  EXTRA="--workload c2"
  run ${lib}_c2_r128 TGK_LIB=$L/$lib.so TGK_FUSED_R=128
  run ${lib}_c2_r256 TGK_LIB=$L/$lib.so TGK_FUSED_R=256
done
EXTRA="--workload c2a"
run libtgk_c2a_noB TGK_FUSED_DEBUG=1
run libtgk_c2a_noA TGK_FUSED_DEBUG=2
for f in gpurun_out/exp_*.json; do python -c "
import json; d=json.load(open('$f')); print('$f'.split('exp_')[1][:-5].ljust(28), round(d['ms_per_step']*1e3,1), 'us')" 2>/dev/null || echo "$f failed"; done
