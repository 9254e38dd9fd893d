#!/bin/bash
# final tree: GPU tests, smoke, plain bench (traffic from the r02c capture of the same kernel sources)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash tools/_run_r02t.sh
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_r02d.json 2> gpurun_out/bench_r02d.err; echo "bench rc=$?"
timeout 300 python tools/repro_perm.py 30 2>&1 | tail -2
