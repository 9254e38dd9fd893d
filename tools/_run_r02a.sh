#!/bin/bash
# Round-2 first capture: GPU tests, bench, launch list, full ncu of k_tiled_dag, panel timings.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
timeout 600 python tools/bench_panels.py > gpurun_out/panels_r02a.log 2>&1
timeout 3000 python -m pytest tests -m gpu -q -x > gpurun_out/gputest_r02a.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gputest_r02a.log
TAG=r02a bash tools/gpu_bench_profile.sh
