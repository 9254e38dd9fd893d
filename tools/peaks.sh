#!/bin/bash
# Measure FP64 peaks on the GPU box (DFMA, DMMA, torch fp64 matmul) + host info.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/peaks_smi.txt 2>&1
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/peaks_clocks.csv &
SMI=$!
./tools/fp64_peak > gpurun_out/peaks.txt 2>&1
python - >> gpurun_out/peaks.txt 2>&1 <<'PY'
import torch, time, os, json
a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda"); b = torch.randn_like(a)
for _ in range(2): c = a @ b
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
best = 1e9
for _ in range(5):
    e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
print(json.dumps({"probe": "torch_matmul_f64_8192", "tflops": 2 * 8192**3 / best * 1e-9, "ms": best}))
print(json.dumps({"cpu_count": os.cpu_count(), "affinity": len(os.sched_getaffinity(0))}))
import numpy, scipy; print("numpy", numpy.__version__, "scipy", scipy.__version__)
PY
lscpu | head -20 >> gpurun_out/peaks.txt
kill $SMI
