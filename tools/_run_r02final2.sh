#!/bin/bash
# final build: GPU tests, then bench + launch list + full ncu capture, reference arm
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash tools/_run_r02t.sh
TAG=r02e bash tools/gpu_bench_profile.sh
timeout 900 python bench.py --impl reference > gpurun_out/bench_reference_arm_r02e.json 2> gpurun_out/bench_reference_arm_r02e.err
timeout 300 python tools/repro_perm.py 30 2>&1 | tail -1 > gpurun_out/repro_perm_r02e.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02e.txt 2>&1
tail -2 gpurun_out/smoke_r02e.txt gpurun_out/repro_perm_r02e.txt
