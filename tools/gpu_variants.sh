#!/bin/bash
# device-time bench of library build variants (TGK_LIB) on c2a / c2
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
L=paper_2602_05052_b200/lib
for w in ${WORKLOADS:-c2a c2}; do for v in ${VARIANTS:-libtgk}; do for R in ${RS:-128}; do
  TGK_FUSED_R=$R TGK_LIB=$L/$v.so timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --e2e-steps 0 --no-cpu-baseline > gpurun_out/var_${w}_${v}_$R.json 2> gpurun_out/var_${w}_${v}_$R.err
  python -c "
import json; d=json.load(open('gpurun_out/var_${w}_${v}_$R.json')); print('$w $v R=$R', round(d['ms_per_step']*1e3,1), 'us')" 2>/dev/null || (echo "$w $v $R failed"; tail -2 gpurun_out/var_${w}_${v}_$R.err)
done; done; done
