#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
cat gpurun_out/smoke.log 2>/dev/null; tail -3 gpurun_out/pytest_gpu.log 2>/dev/null
for f in gpurun_out/bench_*.json; do python -c "
import json,sys
try:
    d=json.load(open('$f'))
except Exception as e:
    print('$f', 'ERR', e); sys.exit()
print('$f'.split('/')[-1], round(d['value']/1e9,3), 'Gelem/s', round(d['ms_per_step']*1e3,1), 'us frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value']/1e6,1) if d.get('e2e') else None, 'M/s cpu', d['cpu_baseline']['value'] if d.get('cpu_baseline') else None, 'rf', round(d['config']['fused_plan']['recompute_factor'],3), d['clocks'])"; done
