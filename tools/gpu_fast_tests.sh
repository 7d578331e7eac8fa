#!/bin/bash
# fast-mode GPU parity + quick timings (one gpurun call)
nvidia-smi --query-gpu=name,clocks.sm --format=csv
timeout 300 python tools/fast_bench.py c2a c2 c1 --reps 20 2>&1 | tail -20
timeout 900 python -m pytest tests/test_gpu_fast.py -x -q -m gpu --durations=10 2>&1 | tail -30
