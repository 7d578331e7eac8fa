#!/bin/bash
# v3 + first-touch node table + owned-row stores: parity, bench, ncu
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
for w in c2a c2; do for no in 0 1; do
  TGK_NODE_ORDER=$no timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/v3b_${w}_$no.json 2> gpurun_out/v3b_${w}_$no.err
  python -c "
import json; d=json.load(open('gpurun_out/v3b_${w}_$no.json')); print('$w node_order=$no', round(d['ms_per_step']*1e3,1), 'us frac', round(d['roofline']['frac'],3))" 2>/dev/null || (echo "$w $no failed"; tail -3 gpurun_out/v3b_${w}_$no.err)
done; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 3 -c 1 \
  -o gpurun_out/prof3b_c2a python bench.py --workload c2a --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu3b.log 2>&1
