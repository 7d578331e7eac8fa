#!/bin/bash
# bench lines for the scalar workloads (fast mode default) + reference arm for c2
for W in ${WL:-c2 c2a c1}; do
  timeout 900 python bench.py --workload $W --steps 20 --warmup 5 > gpurun_out/bench_$W.json 2> gpurun_out/bench_$W.err; echo "$W rc=$?"
done
