#!/bin/bash
# scheduler knob sweep (no rebuild): reserved helper CTAs / team slack on C5 and C3
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for cfg in C3 C5; do
  for rs in 0 2 4 6 8 12; do
    for sl in 2 4; do
      echo "== $cfg reserve $rs slack $sl" >> gpurun_out/knobs.log
      timeout 300 python tools/probe_config.py $cfg --reserve $rs --team-slack $sl 2>&1 | tail -1 | cut -c1-120 >> gpurun_out/knobs.log
    done
  done
done
cat gpurun_out/knobs.log
