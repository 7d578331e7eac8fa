#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over every hot kernel (tools/sanitize_kernels.py)
python tools/sanitize_kernels.py > gpurun_out/sanitize_plain.log 2>&1; echo "plain rc=$?"
for T in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $T --print-limit 20 python tools/sanitize_kernels.py > gpurun_out/sanitize_$T.log 2>&1
  echo "$T rc=$?"; tail -3 gpurun_out/sanitize_$T.log
done
