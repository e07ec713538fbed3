"""NEXT-4 measurement: KV-segment checkpointing between layer calls, non-interference.

    python tools/kv_ckpt.py [--config mixtral_decode] [--steps 1000]

Times bench.py's layer step (same weights, 8 rotating batches) with and without a checkpoint of the
step's KV segment (T tokens x C bytes, C = 2 H_kv (d/H_attn) S_elem = 4096 B for Mixtral; the layer's
expert traffic per token is V = 2 k d S_elem = 32 KB: C/V = 12.5 %, App. C) after every call, and
reports the step time both ways, the commit lag and the checkpoint bandwidth.  One JSON line.
"""
import argparse
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as wl  # noqa: E402
import paper_2601_01310_b200 as tg  # noqa: E402
from bench import make_weights_device  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="mixtral_decode")
    ap.add_argument("--steps", type=int, default=1000)
    a = ap.parse_args()
    sh = wl.CONFIGS[a.config]
    dev = torch.device("cuda", 0)
    pl = wl.make_placement(sh.E, 1, 1, shadows=False)
    L = make_weights_device(sh, 1001, dev, list(range(sh.E)))
    layer = tg.MoELayer(sh, pl, L, max_tokens_per_rank=sh.T, device=0)
    xs = [wl.make_tokens(sh, 1001 + 17 * i, device=dev) for i in range(8)]
    C = 2 * 8 * (sh.d // 32) * 2  # H_kv = 8, H_attn = 32 (Mixtral attention), bf16
    seg_bytes = sh.T * C
    kv = torch.randint(0, 256, (8, seg_bytes), dtype=torch.uint8, device=dev)
    ring = 64  # bucket holds the last 64 steps' segments (the store side keeps the log)
    tg.tg_kv_store_init(layer.ctx, ring * seg_bytes)
    stream = torch.cuda.current_stream()

    def run(ckpt, seq0):
        for i in range(20):
            layer(xs[i % 8])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(stream)
        for i in range(a.steps):
            layer(xs[i % 8])
            if ckpt:
                tg.tg_kv_checkpoint(layer.ctx, kv[i % 8], (i % ring) * seg_bytes, seq0 + i + 1)
        e1.record(stream)
        torch.cuda.synchronize()
        host = time.perf_counter() - t0
        if ckpt:
            while tg.tg_kv_committed(layer.ctx) < seq0 + a.steps:
                time.sleep(1e-4)
        done = time.perf_counter() - t0
        return e0.elapsed_time(e1) / a.steps, host, done

    base1, _, _ = run(False, 0)
    ck, host, done = run(True, 0)
    base2, _, _ = run(False, 0)
    base = (base1 + base2) / 2
    rep = {"config": a.config, "T": sh.T, "segment_bytes_per_token": C, "segment_bytes_per_step": seg_bytes,
           "expert_bytes_per_token": 2 * sh.k * sh.d * 2, "ms_per_step_no_ckpt": base,
           "ms_per_step_ckpt": ck, "interference_pct": 100.0 * (ck - base) / base,
           "commit_drain_after_last_step_ms": 1e3 * (done - host),
           "ckpt_GBps": seg_bytes * a.steps / (ck * 1e-3 * a.steps) / 1e9, "steps": a.steps,
           "store": "pinned host bucket, copy engine on a lowest-priority stream"}
    print(json.dumps(rep), flush=True)
    layer.close()


if __name__ == "__main__":
    main()
