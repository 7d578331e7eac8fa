#!/bin/bash
# fast-mode tests + ncu capture of k_fast_scalar on C2a
timeout 900 python -m pytest tests/test_gpu_fast.py -x -q -m gpu --durations=10 2>&1 | tail -15
timeout 600 ncu --set full --import-source on -k regex:k_fast_scalar -c 1 -o gpurun_out/fast_c2a -f python tools/fast_bench.py c2a --reps 1 --modes fast > gpurun_out/ncu_fast.log 2>&1
tail -3 gpurun_out/ncu_fast.log
