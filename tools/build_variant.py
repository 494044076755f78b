"""Build A/B variants of libloza.so that differ in -D flags of one source file.

usage: python tools/build_variant.py NAME SRC.cu -DFOO=1 [-DBAR=2 ...]
writes variants/libloza_NAME.so (load it with LOZA_LIB=variants/libloza_NAME.so).
"""
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2512_23966_b200 import build as B  # noqa: E402

name, src, defs = sys.argv[1], sys.argv[2], sys.argv[3:]
B.build()
out_dir = os.path.join(ROOT, "variants")
os.makedirs(out_dir, exist_ok=True)
src_path = src if os.path.sep in src else os.path.join(B.CSRC, src)
src = os.path.basename(src) if os.path.sep not in src else os.environ.get("REPLACES", os.path.basename(src))
obj = os.path.join(out_dir, f"{name}_{src[:-3]}.o")
inc = ["-I", os.path.join(ROOT, "include"), "-I", B._nccl_include()]
r = subprocess.run(["nvcc", *B.NVCC_FLAGS, *inc, *defs, "-c", src_path, "-o", obj], capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stdout + r.stderr)
objs = [o for o in sorted(glob.glob(os.path.join(B.BUILD, "*.o"))) if os.path.basename(o) != src[:-3] + ".o"] + [obj]
lib = os.path.join(out_dir, f"libloza_{name}.so")
subprocess.run(["nvcc", "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", lib, "-ldl"], check=True)
print(lib)
