"""Summarise an ncu --set full report into profiles/ncu_summary.json.

usage: python scripts/ncu_summary.py REPORT.ncu-rep OUT.json "capture description"
Keys follow bench.py's roofline kernels (k_spread_fwd = the spread kernel).
"""
import csv
import io
import json
import subprocess
import sys

rep, out, desc = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, data = rows[0], rows[2:]
KEYS = [("k_gather_cc", "k_bwd_gather"), ("k_tile_keys", "k_tile_keys"), ("k_z_tiles_ko", "k_z_tiles_ko"),
        ("k_spread_f8", "k_spread_fwd"), ("k_spread_uv", "k_spread_fwd"), ("k_dgemm_tn_tma", "k_dgemm_tn"),
        ("k_dgemm_tn", "k_dgemm_tn"), ("k_spread_mma", "k_spread_fwd"), ("k_bwd_gather", "k_bwd_gather"),
        ("k_col_scatter", "k_col_scatter"), ("k_z_sort", "k_z_sort"), ("k_tile_hist", "k_tile_hist"),
        ("k_col_scan", "k_col_scan"), ("k_tile_sort", "k_tile_sort"), ("k_z_tiles", "k_z_tiles"),
        ("k_core_sum", "k_core_sum")]
M = {"time_us": "gpu__time_duration.sum", "dram_read": "dram__bytes_read.sum",
     "dram_write": "dram__bytes_write.sum", "inst": "smsp__inst_executed.sum",
     "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
     "dmma_pct": "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
     "dmma_inst": "sm__inst_executed_pipe_tensor_subpipe_dmma.sum",
     "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
     "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
     "l1tex_pct": "l1tex__throughput.avg.pct_of_peak_sustained_active",
     "smem_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
     "dram_pct": "dram__throughput.avg.pct_of_peak_sustained_elapsed",
     "regs": "launch__registers_per_thread"}
units = rows[1]
res = {}
for d in data:
    name = d[h.index("Kernel Name")]
    key = next((k for pat, k in KEYS if pat in name), None)
    if key is None or key in res:
        continue
    e = {"name": name.split("(")[0].replace("(anonymous namespace)::", "")}
    for k, m in M.items():
        if m not in h:
            continue
        v = float(d[h.index(m)].replace(",", "") or 0)
        u = units[h.index(m)]
        if k.startswith("dram_") and not k.endswith("pct"):
            v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        if k == "time_us":
            v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}.get(u, 1)
        e[k] = v
    e["dram_bytes"] = e.get("dram_read", 0) + e.get("dram_write", 0)
    st = [(h[i], float(d[i] or 0)) for i in range(len(h))
          if h[i].startswith("smsp__average_warps_issue_stalled_") and h[i].endswith("per_issue_active.ratio")]
    e["top_stalls"] = {k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""):
                       round(v, 2) for k, v in sorted(st, key=lambda x: -x[1])[:4]}
    res[key] = e
with open(out, "w") as f:
    json.dump({"capture": desc, "kernels": res}, f, indent=1)
print(json.dumps({k: (v["name"], round(v["time_us"], 2)) for k, v in res.items()}, indent=1))
