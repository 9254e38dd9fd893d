#!/bin/bash
# critical paths of C3 / C5, rounded-addition phase micro-benchmarks, panel timings
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash tools/_run_repro.sh > gpurun_out/repro_stack.txt 2>&1
timeout 600 python tools/critical_path.py C3 gpurun_out/critical_path_C3_r02a_path.txt > gpurun_out/critical_path_C3_r02a.json 2> gpurun_out/cp3.err
timeout 600 python tools/critical_path.py C5 gpurun_out/critical_path_C5_r02a_path.txt > gpurun_out/critical_path_C5_r02a.json 2> gpurun_out/cp5.err
BATCH=148 TEAMS=0 timeout 600 python tools/bench_radd.py 512,16,16 512,32,32 512,64,64 512,100,100 512,150,150 512,170,170 1024,8,8 1024,16,16 > gpurun_out/radd_r02a_noteams.log 2>&1
BATCH=8 timeout 600 python tools/bench_radd.py 512,64,64 512,100,100 512,150,150 512,170,170 > gpurun_out/radd_r02a_teams.log 2>&1
timeout 600 python tools/bench_panels.py > gpurun_out/panels_r02a.log 2>&1
tail -3 gpurun_out/repro_stack.txt; tail -2 gpurun_out/cp3.err gpurun_out/cp5.err
