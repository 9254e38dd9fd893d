#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for m in ncta1 default; do
  echo "== $m" >> gpurun_out/repro.log
  CUDA_LAUNCH_BLOCKING=1 timeout 120 python tools/repro_b16.py $m >> gpurun_out/repro.log 2>&1
  echo "rc=$?" >> gpurun_out/repro.log
done
grep -E "^==|rc=|ran;|guards|FAILED|UNFINISHED|tasks started|last 5|^b |rror" gpurun_out/repro.log
