"""Summarise an .ncu-rep: key raw metrics per kernel and the top SASS stall lines.
python tools/ncu_summary.py REP OUT.txt "command line" """
import csv
import subprocess
import sys

rep, out, cmd = sys.argv[1], sys.argv[2], sys.argv[3]
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__m_xbar2l1tex_read_bytes.sum",
        "lts__t_sector_hit_rate.pct", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__cycles_active.avg", "gpc__cycles_elapsed.max", "launch__registers_per_thread", "launch__grid_size"]
raw = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                     text=True).stdout.splitlines()))
lines = [f"# {cmd}"]
h, units = raw[0], raw[1]
for row in raw[2:]:
    lines.append(row[h.index("Kernel Name")])
    lines += [f"  {k} = {row[h.index(k)]} {units[h.index(k)]}" for k in KEYS if k in h]
src = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True,
                                     text=True).stdout.splitlines()))
if len(src) > 2:
    sh, data = src[1], src[2:]
    si = sh.index("Warp Stall Sampling (All Samples)")
    tot = sum(int(r[si]) for r in data if r[si].isdigit()) or 1
    cols = [c for c in sh if c.startswith("stall_") and "Not Issued" not in c]
    lines.append("top SASS lines by warp stall samples (first kernel of the report):")
    for r in sorted(data, key=lambda r: -int(r[si]) if r[si].isdigit() else 0)[:10]:
        st = sorted(((c, int(r[sh.index(c)])) for c in cols if r[sh.index(c)].isdigit()), key=lambda x: -x[1])[:2]
        lines.append(f"  {int(r[si]) / tot * 100:5.1f}%  {r[1].strip()[:64]:64s} {st}")
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
