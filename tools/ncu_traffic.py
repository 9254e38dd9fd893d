"""profiles/ncu_traffic.json from an ncu --page raw --csv export of k_tiled_dag
(tools/gpu_bench_profile.sh): DRAM bytes per launch, keyed on the sha of the
kernel sources so bench.py only reports it for the build it was measured on.

python tools/ncu_traffic.py profiles/ncu_full_k_tiled_dag_<tag>_raw.csv [config]"""
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

path, cfg = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "C3")
rows = list(csv.reader(open(path)))
hdr, units, val = rows[0], rows[1], rows[2]
col = {h: i for i, h in enumerate(hdr)}
scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def get(name):
    i = col[name]
    return float(val[i].replace(",", "")), units[i]


rd, ru = get("dram__bytes_read.sum")
wr, wu = get("dram__bytes_write.sum")
rd *= scale[ru]
wr *= scale[wu]
dur, du = get("gpu__time_duration.sum")
dur *= {"s": 1.0, "ms": 1e-3, "us": 1e-6, "ns": 1e-9}.get(du, 1.0)
out = {cfg: {
    "kernel": "k_tiled_dag", "dram_bytes_per_launch": rd + wr, "dram_read_bytes": rd, "dram_write_bytes": wr,
    "duration_s_under_ncu": dur,
    "l2_hit_rate_pct": get("lts__t_sector_hit_rate.pct")[0],
    "fp64_pipe_active_pct": get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active")[0],
    "dmma_cycles_active_avg": get("SM_C.TriageCompute.smsp__pipe_tensor_subpipe_dmma_cycles_active.avg")[0]
    if "SM_C.TriageCompute.smsp__pipe_tensor_subpipe_dmma_cycles_active.avg" in col else None,
    "issue_active_pct": get("smsp__issue_active.avg.pct_of_peak_sustained_active")[0],
    "csrc_sha16": bench._sources_sha(),
    "source": f"ncu --set full --clock-control none --replay-mode application -k regex:k_tiled_dag "
              f"(tools/gpu_bench_profile.sh), python tools/probe_config.py {cfg}; {path}",
    "note": "algorithmic bytes of the rounded additions: ~146 GB per C3 factorization (device counter); the surplus "
            "is per-CTA arena scratch written back before reuse (DESIGN 4)"}}
dst = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
json.dump(out, open(dst, "w"), indent=1)
print(json.dumps(out, indent=1))
