#!/bin/bash
# batched-kernel (C4) sweep: tests, then batched_ms under plan/launch variants (ENVS="K=V;K=V ...")
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_features.py tests/test_gpu_parity.py -x -q -k "batched or adjoint" 2>&1 | tail -3
for e in ${ENVS:-none}; do
  ( [ "$e" != none ] && export $(echo $e | tr ';' ' '); timeout 300 python bench.py --workload c4 --steps 20 --warmup 5 --e2e-steps 0 --no-cpu-baseline 2>gpurun_out/sweep.err | python -c "
import json,sys; d=json.load(sys.stdin); print('$e', 'batched_ms %.4f' % d['config']['batched_ms'], 'frac %.3f' % d['roofline']['frac'], 'adjoint_ms %.4f' % d['config']['adjoint_ms'])" || tail -3 gpurun_out/sweep.err )
done
