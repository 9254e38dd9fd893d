#!/bin/bash
# quick check after a kernel change: unit/golden GPU tests, rounded-addition micro-benchmarks, C3 probe
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-r02c}
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_factorize.py tests/test_gpu_scale.py -m gpu -q -x > gpurun_out/gputest_$T.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gputest_$T.log
tail -3 gpurun_out/gputest_$T.log
BATCH=148 TEAMS=0 timeout 600 python tools/bench_radd.py 512,16,16 512,32,32 512,64,64 512,100,100 512,170,170 1024,8,8 > gpurun_out/radd_${T}_noteams.log 2>&1
BATCH=8 timeout 600 python tools/bench_radd.py 512,64,64 512,100,100 512,170,170 > gpurun_out/radd_${T}_teams.log 2>&1
cat gpurun_out/radd_${T}_noteams.log gpurun_out/radd_${T}_teams.log | cut -c1-330
timeout 600 python tools/probe_config.py C3 > gpurun_out/probe_C3_$T.log 2>&1; tail -3 gpurun_out/probe_C3_$T.log | cut -c1-600
timeout 600 python tools/probe_config.py C5 > gpurun_out/probe_C5_$T.log 2>&1; tail -3 gpurun_out/probe_C5_$T.log | cut -c1-600
