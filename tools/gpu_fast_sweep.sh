#!/bin/bash
# fast-mode parity + rows-per-block / threads sweep on C2a and C2
[ -z "$NOTEST" ] && timeout 900 python -m pytest tests/test_gpu_fast.py -x -q -m gpu 2>&1 | tail -4
for RT in ${SWEEP:-24:256 32:256 48:256 48:512 64:256 64:512 96:512}; do R=${RT%:*}; T=${RT#*:}
  echo "== R=$R T=$T"; TGK_FAST_R=$R TGK_FAST_T=$T timeout 300 python tools/fast_bench.py c2a c2 --modes fast --reps 10 2>&1 | grep -v Warn
done
