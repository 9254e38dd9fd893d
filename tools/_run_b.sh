mkdir -p gpurun_out
python tools/bench_panels.py --json gpurun_out/panels.json > gpurun_out/panels.log 2>&1
timeout 3000 python -m pytest tests -m gpu -q -s > gpurun_out/gputest.log 2>&1
tail -5 gpurun_out/gputest.log
