#!/bin/bash
# split-arena / L2-persistence experiment: time and DRAM bytes of k_tiled_dag at C3 for several hot sizes
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for hot in 0 32768 65536 98304; do
  export BLRQR_ARENA_HOT=$hot
  echo "== hot $hot" >> gpurun_out/hot.log
  timeout 300 python tools/probe_config.py C3 2>&1 | tail -1 | cut -c1-110 >> gpurun_out/hot.log
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum --clock-control none --replay-mode application -k regex:k_tiled_dag -c 1 --csv --log-file gpurun_out/hot_$hot.csv python tools/probe_config.py C3 > gpurun_out/hot_ncu_$hot.log 2>&1
  grep -E "dram__bytes|hit_rate|time_duration" gpurun_out/hot_$hot.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}' >> gpurun_out/hot.log
done
cat gpurun_out/hot.log
