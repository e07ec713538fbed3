"""bench.py's reference arm (the CPU oracle, runnable here) prints one JSON line with the
contract's keys; the GPU arm's keys are checked on the GPU box (test_bench_gpu)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _line(args, timeout):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _line(["--impl", "reference", "--steps", "1", "--warmup", "3", "--cpu-sample", "2"], 600)
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "dtype", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["metric"] == "MoE-layer tokens/s" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"


@pytest.mark.gpu
def test_bench_gpu_line():
    d = _line(["--steps", "20", "--warmup", "3", "--no-cpu-baseline"], 900)
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "clocks", "e2e", "gpu_launches"):
        assert key in d, key
    assert d["gpu_launches"] == 20  # one launch per call
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor") and 0 < r["frac"] < 1.2
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    # the north star's other numbers in the same line
    p = d["prefill"]
    assert p["roofline"]["bound"] == "tensor" and 0 < p["roofline"]["frac"] < 1.2 and p["us_per_call"] > 0
    f = d["failover"]
    assert f["calls_errored"] == 0 and f["post_mask_outputs_bit_identical"] == f["post_mask_outputs_compared"]
    assert f["mask_host_us"] > 0 and f["reroute_ms"] > 0
