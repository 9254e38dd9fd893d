#!/bin/bash
# Round measurement: bench (plain), launch list under ncu, one full ncu capture
# of the dominant kernel (k_tiled_dag, C3 full size, application replay so the
# persistent kernel's 60 GB working set needs no save/restore).  Outputs under
# gpurun_out/ (CSV exports only: the .ncu-rep stays in /tmp, gpurun_out/ is
# capped at 64 MiB).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-r01}
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
echo "bench rc=$?"
CMD="python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu --no-classes"
timeout 900 $CMD > gpurun_out/plain_${TAG}.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launch_${TAG}.log 2>&1
echo "launch list rc=$?"
if [ -z "$SKIP_FULL" ]; then
CMD2="python tools/probe_config.py C3"
REP=/tmp/prof_dag_${TAG}
rm -f ${REP}.ncu-rep
timeout 600 $CMD2 > gpurun_out/plain2_${TAG}.log 2>&1 && \
timeout 2700 ncu --set full --clock-control none --import-source on --replay-mode application -k regex:k_tiled_dag -c 1 -o ${REP} $CMD2 > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "ncu full rc=$?"
ncu -i ${REP}.ncu-rep --page raw --csv > gpurun_out/ncu_full_k_tiled_dag_${TAG}_raw.csv 2>/dev/null
ncu -i ${REP}.ncu-rep --page details --csv > gpurun_out/ncu_full_k_tiled_dag_${TAG}_details.csv 2>/dev/null
ls -la ${REP}.ncu-rep gpurun_out/
fi
