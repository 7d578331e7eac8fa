#!/bin/bash
# Full round check on one B200: smoke, GPU tests, every bench workload, ncu launch
# list of the default bench command and full captures of the top kernels.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for w in ${WORKLOADS:-c2 c2a c1 c3 c4}; do
  timeout 900 python bench.py --workload $w --steps ${STEPS:-20} --warmup 5 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_$w.json')); r=d['roofline']; e=d['e2e'] or {}
print('$w', 'ms/step %.3f' % d['ms_per_step'], 'value %.3e' % d['value'], 'frac %.3f' % r['frac'], 'e2e %.3e' % e.get('value', 0), 'clk', d['clocks'].get('sm_mhz'), d['clocks'].get('samples'), 'cpu', (d['cpu_baseline'] or {}).get('value'))" 2>/dev/null || (echo "$w failed"; tail -5 gpurun_out/bench_$w.err)
done
if [ -z "$NONCU" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_fused|k_batched|k_adjoint|k_local|k_segment|k_interface" --csv \
  --log-file gpurun_out/launches_c2.csv python bench.py --workload c2 --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 3 -c 1 \
  -o gpurun_out/prof_c2 python bench.py --workload c2 --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_full_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_batched -s 2 -c 1 \
  -o gpurun_out/prof_c4 python bench.py --workload c4 --steps 2 --warmup 2 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_full_c4.log 2>&1
fi
ls gpurun_out | head -50
