"""Summarise an .ncu-rep into profiles/<name>.raw.txt (selected raw metrics per launch) and
profiles/<name>.details.txt (the details page): python tools/ncu_summary.py REP NAME"""
import csv
import io
import subprocess
import sys

rep, name = sys.argv[1], sys.argv[2]
KEYS = ["Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "launch__block_size", "launch__grid_size",
        "launch__cluster_dim_x", "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
        "lts__t_sector_hit_rate.pct", "sm__cycles_elapsed.avg.per_second",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "lts__t_bytes.sum"]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
with open(f"profiles/{name}.raw.txt", "w") as f:
    for li, vals in enumerate(rows[2:]):
        f.write(f"# launch {li}\n")
        for k in KEYS:
            for h, u, v in zip(hdr, units, vals):
                if h == k or h.endswith("." + k) or (k == "Kernel Name" and h == "Kernel Name"):
                    f.write(f"{k} = {v} {u}\n")
                    break
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(det)))
hdr = rows[0]
si, mi, vi, ui = hdr.index("Section Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
with open(f"profiles/{name}.details.txt", "w") as f:
    for r in rows[1:]:
        f.write(f"{r[si]:<32s} | {r[mi]:<40s} | {r[vi]:>14s} {r[ui]}\n")
print(open(f"profiles/{name}.raw.txt").read())
