"""SURVEY 8(d) measurement protocols beyond the throughput line (run with torchrun for G > 1).

  failover : stream Mixtral decode calls; before call M every rank masks EW1 (fail-stop,
             P:914-916) and its slots are NaN-poisoned; reports the host latency of
             tg_mask_worker, the reroute latency (mask call -> first post-mask call done), per-call
             latency before / after, calls that errored, and bit-identity of every post-mask
             output against an unmasked replay of the same inputs.
  flip     : alternate route table A (primaries first) / B (shadows first) every call; bitwise
             equality with a no-flip run; per-call latency flip vs no-flip (ERT-indirection
             overhead, the analog of App. F Alt-3).
  shadow   : latency with shadow replicas loaded (never read when unmasked) vs none (App. D,
             P:1545-1546).

    python tools/protocols.py --which failover|flip|shadow [--calls 400]
    torchrun --nproc-per-node G ... tools/protocols.py --which failover
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as wl  # noqa: E402
import paper_2601_01310_b200 as tg  # noqa: E402
from bench import make_weights_device  # noqa: E402


def setup(cfg, W, shadows, rank, world, local, group):
    sh = wl.CONFIGS[cfg]
    Tr = sh.T // world
    pl = wl.make_placement(sh.E, W, world, shadows=shadows)
    dev = torch.device("cuda", local)
    experts = sorted({e for ew in range(W) if pl.ew_rank[ew] == rank for e in pl.hosted[ew] if e >= 0})
    L = make_weights_device(sh, 1001, dev, experts)
    layer = tg.MoELayer(sh, pl, L, max_tokens_per_rank=Tr, rank=rank, world=world, device=local, group=group)
    return sh, pl, L, layer, Tr, dev


def timed_calls(layer, xs, outs, stream, n0, n1, on_call=None):
    """Run calls n0..n1-1; per-call CUDA-event latency (ms) and rc list."""
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n1 - n0)]
    rcs = []
    for i in range(n0, n1):
        if on_call:
            on_call(i)
        e0, e1 = evs[i - n0]
        e0.record(stream)
        rcs.append(tg.tg_moe_layer(layer.ctx, xs[i % len(xs)], outs[i], stream))
        e1.record(stream)
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in evs], rcs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--which", default="failover", choices=["failover", "flip", "shadow"])
    ap.add_argument("--config", default="mixtral_decode")
    ap.add_argument("--calls", type=int, default=400)
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        group = dist.group.WORLD
    W = max(2, world)
    res = {"protocol": a.which, "config": a.config, "n_gpus": world, "W": W}
    stream = torch.cuda.current_stream()
    if a.which in ("failover", "flip"):
        sh, pl, L, layer, Tr, dev = setup(a.config, W, True, rank, world, local, group)
        NX = 16
        xs = [wl.make_tokens(sh, 5000 + i, T=sh.T, device=dev)[rank * Tr:(rank + 1) * Tr].contiguous()
              for i in range(NX)]
        n = a.calls
        ref = [torch.empty_like(xs[0]) for _ in range(n)]
        for i in range(20):
            tg.tg_moe_layer(layer.ctx, xs[i % NX], ref[0], stream)
        lat_ref, rc_ref = timed_calls(layer, xs, ref, stream, 0, n)        # unmasked / unflipped replay
        outs = [torch.empty_like(xs[0]) for _ in range(n)]
        if a.which == "failover":
            M = n // 2
            info = {}

            def on_call(i):
                if i == M:
                    torch.cuda.synchronize()
                    if world > 1:
                        dist.barrier()
                    t0 = time.perf_counter()
                    rc = layer.mask_worker(1, 1)
                    info["mask_host_us"] = (time.perf_counter() - t0) * 1e6
                    info["mask_rc"] = rc
                    info["t0"] = t0
                    # fail-stop: the masked EW's memory is poisoned (never read again)
                    if pl.ew_rank[1] == rank:
                        nan = torch.full((sh.F, sh.d), float("nan"), dtype=torch.bfloat16, device=dev)
                        nan2 = torch.full((sh.d, sh.F), float("nan"), dtype=torch.bfloat16, device=dev)
                        for sl, e in enumerate(pl.hosted[1]):
                            if e >= 0:
                                tg.tg_load_experts(layer.ctx, 1, sl, e, nan, nan, nan2)
                    info["t_poison"] = time.perf_counter()

            lat, rcs = timed_calls(layer, xs, outs, stream, 0, M, None)
            lat2, rcs2 = [], []
            # first post-mask call: host-timed to completion
            on_call(M)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t1 = time.perf_counter()
            e0.record(stream)
            rc = tg.tg_moe_layer(layer.ctx, xs[M % NX], outs[M], stream)
            e1.record(stream)
            e1.synchronize()
            t2 = time.perf_counter()
            info["reroute_latency_us"] = (t2 - info["t0"]) * 1e6 - (info["t_poison"] - info["t0"]) * 1e6
            info["first_post_mask_call_us"] = e0.elapsed_time(e1) * 1e3
            info["first_post_mask_host_us"] = (t2 - t1) * 1e6
            lat2, rcs2 = timed_calls(layer, xs, outs, stream, M + 1, n)
            bad = [i for i in range(n) if not torch.equal(outs[i].view(torch.int16), ref[i].view(torch.int16))]
            st = layer.stats()
            res.update({
                "mask_worker_host_us": info["mask_host_us"], "mask_rc": info["mask_rc"],
                "reroute_latency_us": info["reroute_latency_us"],
                "first_post_mask_call_device_us": info["first_post_mask_call_us"],
                "pre_mask_call_us_median": float(np.median(lat_ref[:M]) * 1e3),
                "pre_mask_call_us_p95": float(np.percentile(lat_ref[:M], 95) * 1e3),
                "post_mask_call_us_median": float(np.median(lat2) * 1e3),
                "post_mask_call_us_p95": float(np.percentile(lat2, 95) * 1e3),
                "tokens_per_s_pre": sh.T / (np.median(lat_ref[:M]) / 1e3),
                "tokens_per_s_post": sh.T / (np.median(lat2) / 1e3),
                "calls_errored": int(sum(r != 0 for r in rcs + [rc] + rcs2)),
                "post_mask_outputs_bit_identical": len(bad) == 0, "mismatched_calls": bad[:10],
            })
            del st
        else:
            flipped = wl.flipped(pl.cand)

            def on_call(i):
                layer.set_route_table(flipped if i % 2 == 0 else pl.cand)

            lat, rcs = timed_calls(layer, xs, outs, stream, 0, n, on_call)
            bad = [i for i in range(n) if not torch.equal(outs[i].view(torch.int16), ref[i].view(torch.int16))]
            res.update({"flip_call_us_median": float(np.median(lat) * 1e3),
                        "noflip_call_us_median": float(np.median(lat_ref) * 1e3),
                        "flip_overhead_pct": float((np.median(lat) / np.median(lat_ref) - 1) * 100),
                        "calls_errored": int(sum(r != 0 for r in rcs)),
                        "flip_outputs_bit_identical": len(bad) == 0, "mismatched_calls": bad[:10]})
        layer.close()
    else:
        out = {}
        for shadows in (False, True):
            sh, pl, L, layer, Tr, dev = setup(a.config, W, shadows, rank, world, local, group)
            xs = [wl.make_tokens(sh, 5000 + i, T=sh.T, device=dev)[rank * Tr:(rank + 1) * Tr].contiguous()
                  for i in range(8)]
            outs = [torch.empty_like(xs[0]) for _ in range(a.calls)]
            timed_calls(layer, xs, outs, stream, 0, 20)
            lat, rcs = timed_calls(layer, xs, outs, stream, 0, a.calls)
            out[shadows] = (float(np.median(lat) * 1e3), outs[0].clone())
            layer.close()
            del L
            torch.cuda.empty_cache()
        res.update({"call_us_no_shadows": out[False][0], "call_us_shadows_loaded": out[True][0],
                    "delta_pct": (out[True][0] / out[False][0] - 1) * 100,
                    "outputs_bit_identical": bool(torch.equal(out[False][1].view(torch.int16),
                                                              out[True][1].view(torch.int16)))})
    if world > 1:
        dist.barrier()
    if rank == 0:
        print(json.dumps(res), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
