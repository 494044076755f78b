"""Host logic of bench.py (no GPU): the --gpus contract, the FLOP counter, the reference arm's line."""
import json
import os
import subprocess
import sys

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def _run(args, env_extra=None, timeout=600):
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    env.pop("WORLD_SIZE", None)
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          env=env, timeout=timeout)


def test_gpus_n_without_enough_gpus_fails_loudly():
    """`bench.py --gpus 2` never silently measures one GPU: it re-launches under torch.distributed.run or exits
    non-zero when the node has fewer GPUs."""
    r = _run(["--gpus", "2", "--steps", "1"])
    assert r.returncode == 2, r.stdout + r.stderr
    assert "needs 2 visible GPUs" in r.stderr
    assert r.stdout.strip() == ""


def test_world_size_disagreeing_with_gpus_fails():
    r = _run(["--gpus", "4", "--steps", "1"], {"WORLD_SIZE": "2", "RANK": "0"})
    assert r.returncode == 2 and "WORLD_SIZE=2 but --gpus 4" in r.stderr


def test_ssa_pairs_matches_oracle_mask():
    """The bench's FLOP counter (pairs) equals the count of allowed (query, key) pairs of the oracle's mask."""
    for n, s, l, b, q0 in [(300, 1, 3, 16, 32), (257, 2, 2, 8, 0), (64, 0, 4, 4, 16), (1000, 1, 7, 128, 0),
                           (129, 3, 1, 32, 64)]:
        brute = sum(len(oracle.allowed_keys(p, q0 + n, s, l, b)) for p in range(q0, q0 + n))
        assert bench.ssa_pairs(n, s, l, b, q0) == brute
    # SURVEY.md Appendix A
    assert bench.ssa_pairs(32768, 1, 7, 128) == 31014912
    assert bench.ssa_pairs(1 << 20, 1, 7, 128) == 1006698496


def test_reference_arm_line_at_n2():
    """--impl reference at N=2 (no torchrun: rank 0 alone) times the oracle on the N>1 workload (1M SP prefill)
    and reports the measured step time separately from the projection."""
    r = _run(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "3", "--cpu-seconds", "0.5"])
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert line["config"]["workload"] == "ssa_seqpar_prefill_1m" and line["scaling"] == "strong"
    assert line["ms_per_step"] < 60e3 < line["projected_full_step_ms"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "oracle"
