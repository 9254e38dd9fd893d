#!/bin/bash
# GPU tests only (log kept small)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 3000 python -X faulthandler -m pytest tests -m gpu -q -x -v -s > gpurun_out/gputest_r02.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gputest_r02.log
tail -5 gpurun_out/gputest_r02.log
