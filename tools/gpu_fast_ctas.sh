#!/bin/bash
# fast kernel skeleton anatomy vs CTAs per SM (TGK_FAST_DEBUG bits: 1 A, 2 B, 4 copy-out, 8 gathers, 16 record B)
for C in ${CTAS:-1 3}; do for D in ${DBG:-7 15 23 31 0}; do
  echo "== ctas=$C debug=$D"; TGK_FAST_CTAS=$C TGK_FAST_DEBUG=$D timeout 300 python tools/fast_bench.py c2a --modes fast --reps 10 2>&1 | grep c2a
done; done
