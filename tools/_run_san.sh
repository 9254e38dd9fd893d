mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
python tools/sanitize_run.py tiled,radd > gpurun_out/san_plain.log 2>&1
timeout 1500 $CS --tool memcheck --leak-check no --report-api-errors no --print-limit 50 python tools/sanitize_run.py tiled,blocked,mgs,radd > gpurun_out/san_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/san_memcheck.log
timeout 1500 $CS --tool racecheck --racecheck-report hazard --print-limit 50 python tools/sanitize_run.py tiled,radd > gpurun_out/san_racecheck.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/san_racecheck.log
timeout 1500 $CS --tool synccheck --print-limit 50 python tools/sanitize_run.py tiled,radd > gpurun_out/san_synccheck.log 2>&1; echo "synccheck rc=$?" >> gpurun_out/san_synccheck.log
timeout 1500 $CS --tool memcheck --leak-check no --report-api-errors no --print-limit 50 python tools/sanitize_run.py geqrt > gpurun_out/san_memcheck_geqrt.log 2>&1; echo "memcheck geqrt rc=$?" >> gpurun_out/san_memcheck_geqrt.log
