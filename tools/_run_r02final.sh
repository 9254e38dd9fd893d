#!/bin/bash
# Final round-2 capture: bench + launch list + full ncu (gpu_bench_profile.sh), reference arm,
# critical paths, rounded-addition phase micro-benchmarks, panel timings.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-r02b}
TAG=$T bash tools/gpu_bench_profile.sh
timeout 900 python bench.py --impl reference > gpurun_out/bench_reference_arm_$T.json 2> gpurun_out/bench_reference_arm_$T.err
timeout 600 python tools/critical_path.py C3 gpurun_out/critical_path_C3_${T}_path.txt > gpurun_out/critical_path_C3_$T.json 2> gpurun_out/cp3.err
timeout 600 python tools/critical_path.py C5 > gpurun_out/critical_path_C5_$T.json 2> gpurun_out/cp5.err
BATCH=148 TEAMS=0 timeout 600 python tools/bench_radd.py 512,16,16 512,32,32 512,64,64 512,100,100 512,170,170 1024,8,8 > gpurun_out/radd_${T}.log 2>&1
BATCH=8 timeout 600 python tools/bench_radd.py 512,64,64 512,100,100 512,170,170 >> gpurun_out/radd_${T}.log 2>&1
timeout 600 python tools/bench_panels.py > gpurun_out/panels_$T.log 2>&1
for c in C1 C2 C4; do timeout 600 python tools/probe_config.py $c 2>&1 | tail -1 | cut -c1-200 >> gpurun_out/probes_$T.log; done
timeout 600 python tools/probe_config.py C4 --method blocked-hh 2>&1 | tail -1 | cut -c1-200 >> gpurun_out/probes_$T.log
timeout 600 python tools/probe_config.py C2 --method tiled-hh 2>&1 | tail -1 | cut -c1-200 >> gpurun_out/probes_$T.log
ls -la gpurun_out | tail -25
