#!/bin/bash
# time split of the fast kernel: skip phases via TGK_FAST_DEBUG (timings only; outputs invalid)
R=${1:-32}; T=${2:-256}
for D in 0 1 2 4 6 7 3; do echo "== debug=$D R=$R T=$T"; TGK_FAST_DEBUG=$D TGK_FAST_R=$R TGK_FAST_T=$T timeout 300 python tools/fast_bench.py c2a --modes fast --reps 10 2>&1 | grep -v Warn; done
