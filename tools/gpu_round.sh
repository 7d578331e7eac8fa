#!/bin/bash
# Full round check on one B200: smoke, GPU tests, every bench workload, ncu launch
# list of the default bench command and one full capture of each workload's
# dominant kernel (-> profiles/traffic.json via tools/make_traffic.py).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; grep -E "FAILED|passed|failed" gpurun_out/pytest_gpu.log | tail -5
for w in ${WORKLOADS:-c2 c2a c1 c3 c4 c5 rm}; do
  timeout 900 python bench.py --workload $w --steps ${STEPS:-20} --warmup 5 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_$w.json')); r=d['roofline']; e=d['e2e'] or {}
print('$w', 'ms/step %.3f' % d['ms_per_step'], 'value %.3e' % d['value'], 'frac %.3f' % r['frac'], 'e2e %.3e' % e.get('value', 0), 'clk', d['clocks'].get('sm_mhz'), d['clocks'].get('samples'), 'cpu', (d['cpu_baseline'] or {}).get('value'))" 2>/dev/null || (echo "$w failed"; tail -5 gpurun_out/bench_$w.err)
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; tail -c 400 gpurun_out/bench_reference.json
if [ -z "$NONCU" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_c2.csv python bench.py --workload c2 --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch_c2.log 2>&1
for wk in ${PROF:-c2:k_fast_scalar c2a:k_fast_scalar c1:k_fast_scalar c3:k_fast_elast c4:k_batched_entries c4adj:k_adjoint_groups c5:k_fast_scalar rm:k_segment_reduce}; do
  w=${wk%%:*}; k=${wk##*:}; bw=$w; [ $w = c4adj ] && bw=c4
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 \
    -o gpurun_out/prof_$w python bench.py --workload $bw --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_full_$w.log 2>&1
done
# summaries + traffic.json on the box; keep only the reports named in KEEP (64 MiB merge limit)
TRAFFIC_OUT=gpurun_out/prof_out python tools/make_traffic.py ${PREFIX:-r02} > /dev/null
for f in gpurun_out/prof_*.ncu-rep; do
  case " ${KEEP:-c2} " in *" $(basename $f .ncu-rep | sed s/prof_//) "*) ;; *) rm -f $f ;; esac
done
fi
ls gpurun_out | head -60
