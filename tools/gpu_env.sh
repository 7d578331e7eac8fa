#!/bin/bash
# device-time bench under env settings: ENVS="A=1 B=2;A=0" (';'-separated cases)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
IFS=';' read -ra CASES <<< "${ENVS:-}"
for w in ${WORKLOADS:-c2a c2}; do for cs in "${CASES[@]}"; do
  tag=$(echo "$cs" | tr ' =' '_-')
  env $cs timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --e2e-steps 0 --no-cpu-baseline > gpurun_out/env_${w}_$tag.json 2> gpurun_out/env_${w}_$tag.err
  python -c "
import json; d=json.load(open('gpurun_out/env_${w}_$tag.json')); print('$w [$cs]', round(d['ms_per_step']*1e3,1), 'us')" 2>/dev/null || (echo "$w [$cs] failed"; tail -2 gpurun_out/env_${w}_$tag.err)
done; done
