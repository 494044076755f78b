"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per kernel count, mean, share.
python tools/launch_summary.py LIST.csv OUT.summary.txt "command line" [algorithmic_flop_of_prefill]"""
import collections
import csv
import sys

src, dst, cmd = sys.argv[1], sys.argv[2], sys.argv[3]
flop = float(sys.argv[4]) if len(sys.argv) > 4 else None
rows = [r for r in csv.reader(open(src)) if len(r) > 5]
hdr = rows[0]
ki, mi, vi, ui = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
agg = collections.OrderedDict()
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    us = float(r[vi].replace(",", "")) * scale[r[ui]]
    a = agg.setdefault(r[ki][:78], [0, 0.0])
    a[0] += 1
    a[1] += us
tot = sum(a[1] for a in agg.values())
out = [cmd, "(cold-cache, serialised launches: compare shares, not absolutes; input generation and L2 flush kernels "
       "are outside the timed step)", ""]
for n, (c, t) in agg.items():
    out.append(f"{n:80s} launches {c:3d}  mean {t / c:9.1f} us  share {100 * t / tot:5.1f}%")
if flop:
    for n, (c, t) in agg.items():
        if "prefill_tc" in n:
            out.append(f"\nprefill_tc_kernel per launch: {t / c / 1e3:.3f} ms under ncu -> "
                       f"{flop / (t / c * 1e-6) / 1e12:.0f} TFLOP/s algorithmic")
open(dst, "w").write("\n".join(out) + "\n")
print("\n".join(out))
