"""Multi-GPU parity through torchrun (G = all visible GPUs, 2 or 4)."""
import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(G, *args):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={G}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + G), os.path.join(ROOT, "tests", "mp_parity.py"),
           *args]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert r.returncode == 0 and lines, f"rc={r.returncode}\n{r.stdout[-3000:]}\n{r.stderr[-3000:]}"
    rep = json.loads(lines[-1])
    print(rep)
    assert rep["ok"], rep
    return rep


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("W_mult", [1, 2])
def test_tiny_multi_gpu(W_mult):
    G = torch.cuda.device_count()
    rep = _run(G, "--config", "tiny", "--W", str(G * W_mult))
    assert rep["cross_G_bit_identical"]


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_mixtral_multi_gpu():
    G = torch.cuda.device_count()
    _run(G, "--config", "mixtral_decode", "--sample", "16")


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("config", ["tiny", "mixtral_decode"])
def test_rank_fail_stop(config):
    """NEXT-3a: a whole rank fail-stops; survivors keep serving bit-identically."""
    G = torch.cuda.device_count()
    rep = _run(G, "--config", config, "--rank-fail")
    assert rep["rank_fail_dead"] == G - 1


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("config", ["tiny", "mixtral_decode"])
def test_inflight_failover(config):
    """NEXT-1: a rank crashes mid-call; the survivors repair that very call (tg_failover)."""
    G = torch.cuda.device_count()
    rep = _run(G, "--config", config, "--inflight-fail")
    assert rep["inflight_rc"] == 0


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_prefill_multi_gpu_token_dedup():
    """NEXT-2: a prefill-sized call (>= 16 MB of dispatched rows) sends each token once per peer
    rank and the peer copies it into its other pairs' rows; parity, flips and masks unchanged,
    and the G-GPU output bitwise equal to the 1-GPU run."""
    G = torch.cuda.device_count()
    rep = _run(G, "--config", "qwen_prefill", "--sample", "16")
    assert rep["cross_G_bit_identical"]


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("config", ["tiny", "qwen_prefill"])
def test_rank_with_no_tokens(config):
    """A rank with T = 0 still exchanges counts and serves rows; the others' outputs are unchanged."""
    G = torch.cuda.device_count()
    args = ["--config", config, "--empty-rank"] + (["--sample", "16"] if config != "tiny" else [])
    rep = _run(G, *args)
    assert rep["empty_rank"] == G - 1
