#!/bin/bash
# bench lines + ncu launch list + one full capture per workload
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for w in ${WORKLOADS:-c2 c2a c1}; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
if [ -n "$NCU" ]; then
for w in ${NCU_WORKLOADS:-c2 c2a}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 3 -c 1 \
    -o gpurun_out/prof_$w python bench.py --workload $w --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_full_$w.log 2>&1
done
fi
if [ -n "$RVAR" ]; then
  TGK_FUSED_R=128 timeout 600 python bench.py --workload c2a --steps 20 --warmup 5 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_c2a_r128.json 2> gpurun_out/bench_c2a_r128.err
  TGK_FUSED_R=256 timeout 600 python bench.py --workload c2 --steps 20 --warmup 5 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_c2_r256.json 2> gpurun_out/bench_c2_r256.err
  TGK_IEEE_DIV=1 timeout 600 python bench.py --workload c2a --steps 20 --warmup 5 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_c2a_ieee.json 2> gpurun_out/bench_c2a_ieee.err
fi
