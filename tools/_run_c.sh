mkdir -p gpurun_out
python tools/probe_config.py C3 > gpurun_out/probe_C3.log 2>&1
python tools/probe_config.py C5 > gpurun_out/probe_C5.log 2>&1
timeout 2400 python -m pytest tests/test_gpu_scale.py tests/test_gpu_kernels.py -q -s > gpurun_out/t_scale.log 2>&1
timeout 2400 python -m pytest tests/test_gpu_fullsize.py -q -s -k "C3 or C4 or C2" > gpurun_out/t_full.log 2>&1
