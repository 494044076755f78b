"""The key-split pair decode kernel (attn_tc_decode_pair.cu, selected with LOZA_DECODE_KERNEL=pair; the default
is the pair-cooperative kernel, and the choice is read once per process) through the same decode and
ring-cache parity tests."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_split_pair_decode_parity_suite():
    env = dict(os.environ, LOZA_DECODE_KERNEL="pair")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_tc_decode.py"),
                        os.path.join(ROOT, "tests", "test_ring_cache.py")],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
