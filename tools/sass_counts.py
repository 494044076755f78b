"""Per-kernel counts of the SASS mnemonics that prove the tcgen05 / TMA paths (static instruction counts in
libloza.so, not executions): python tools/sass_counts.py > profiles/rNN_sass_counts.txt"""
import collections
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2512_23966_b200", "libloza.so")
KEYS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "UTMALDG", "UTMASTG", "UBLKCP", "UTMAPF", "UBLKPF", "LDTM", "STTM",
        "UTCATOMSWS", "HMMA", "FFMA2", "MUFU.EX2", "SYNCS", "STL", "LDL"]
sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
cur, counts = None, collections.OrderedDict()
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        counts[cur] = collections.Counter()
        continue
    if cur is None:
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
    if not m:
        continue
    op = m.group(1)
    for k in KEYS:
        if op == k or op.startswith(k + "."):
            counts[cur][k] += 1
dem = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True, text=True).stdout.splitlines()
print(f"static SASS mnemonic counts per kernel in {os.path.relpath(LIB, ROOT)} (cuobjdump -sass)")
for (name, c), d in zip(counts.items(), dem):
    if not any(c.values()):
        continue
    short = re.sub(r"\(.*", "", d.replace("(anonymous namespace)::", "")).replace("loza::", "")
    print(f"{short[:60]:60s} " + " ".join(f"{k}={c[k]}" for k in KEYS if c[k]))
