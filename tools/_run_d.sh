mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scale.py tests/test_gpu_kernels.py -q -s -x > gpurun_out/t_scale.log 2>&1
python tools/bench_panels.py --ctas 1,17 > gpurun_out/panels.log 2>&1
python tools/probe_config.py C5 > gpurun_out/probe_C5.log 2>&1
python tools/probe_config.py C3 > gpurun_out/probe_C3.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_fullsize.py -q -s -k "C5 or C3" > gpurun_out/t_full.log 2>&1
