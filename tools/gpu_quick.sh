#!/bin/bash
# GPU tests + device-time bench lines (+ optional ncu full capture of one workload: PROF=c2a)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for w in ${WORKLOADS:-c2a c2}; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --e2e-steps 0 --no-cpu-baseline > gpurun_out/q_$w.json 2> gpurun_out/q_$w.err
  python -c "
import json; d=json.load(open('gpurun_out/q_$w.json')); r=d['roofline']
print('$w', 'ms/step %.3f' % d['ms_per_step'], 'kernel_ms %.3f' % r.get('kernel_ms', 0), 'frac %.3f' % r['frac'])" 2>/dev/null || (echo "$w failed"; tail -3 gpurun_out/q_$w.err)
done
if [ -n "$PROF" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${PROFK:-k_fused} -s 3 -c 1 \
  -o gpurun_out/prof_q_$PROF python bench.py --workload $PROF --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_q.log 2>&1
fi
