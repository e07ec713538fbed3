"""Dispatch-exchange NVLink bandwidth sweep (all-to-all vs 900 GB/s/direction).

    torchrun --nproc-per-node G --master-addr 127.0.0.1 --master-port P tools/nvlink_sweep.py [--config qwen_prefill]

For each global token count T, runs the layer, traces one call and reports per
rank: bytes this rank stored into PEER receive buffers in the dispatch phase
(P4 of k_layer: rows whose destination rank != this rank, d*2 B each,
+ 8 B metadata), the P4 duration from device timestamps, and the resulting
GB/s per direction; plus the whole-call latency.  Rank 0 prints one JSON line
per T with the max over ranks of the P4 time (the exchange completes when the
slowest rank finishes).
"""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as wl  # noqa: E402
import paper_2601_01310_b200 as tg  # noqa: E402
from bench import make_weights_device  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="qwen_prefill")
    ap.add_argument("--tokens", default="1024,2048,4096,8192,16384")
    a = ap.parse_args()
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    sh = wl.CONFIGS[a.config]
    Ts = [int(t) for t in a.tokens.split(",")]
    Tmax = max(Ts) // world
    W = world
    pl = wl.make_placement(sh.E, W, world)
    experts = sorted({e for ew in range(W) if pl.ew_rank[ew] == rank for e in pl.hosted[ew] if e >= 0})
    L = make_weights_device(sh, 1001, dev, experts)
    layer = tg.MoELayer(sh, pl, L, max_tokens_per_rank=Tmax, rank=rank, world=world, device=local,
                        group=dist.group.WORLD)
    for T in Ts:
        Tr = T // world
        x = wl.make_tokens(sh, 77, T=T, device=dev)[rank * Tr:(rank + 1) * Tr].contiguous()
        for _ in range(5):
            layer(x)
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        for _ in range(20):
            layer(x)
        ev1.record()
        torch.cuda.synchronize()
        call_us = ev0.elapsed_time(ev1) / 20 * 1e3
        tg.tg_set_trace(layer.ctx, True)
        layer(x)
        torch.cuda.synchronize()
        tr = tg.tg_get_trace(layer.ctx)
        tg.tg_set_trace(layer.ctx, False)
        st = tr["front_stamps"]
        p4_us = (st[4] - st[3]) / 1e3
        rt = layer.routing(Tr)
        dr = rt["dst_rank"].long()
        remote_pairs = int((dr != rank).sum().item())
        # token dedup: one row per (token, remote rank); every pair still sends 8 B origin + 4 B dup
        onehot = torch.zeros(dr.shape[0], world, dtype=torch.bool, device=dr.device)
        onehot.scatter_(1, dr, True)
        onehot[:, rank] = False
        remote_rows = int(onehot.sum().item())
        remote_bytes = remote_rows * sh.d * 2 + remote_pairs * 12
        v = torch.tensor([p4_us, remote_bytes, call_us], device=dev, dtype=torch.float64)
        allv = [torch.empty_like(v) for _ in range(world)]
        dist.all_gather(allv, v)
        if rank == 0:
            p4 = max(float(t[0]) for t in allv)
            rb = [float(t[1]) for t in allv]
            rep = {"config": a.config, "n_gpus": world, "T_global": T, "dispatch_p4_us_max": p4,
                   "remote_bytes_per_rank": rb, "dedup": True,
                   "dispatch_GBps_per_direction_per_gpu": (max(rb) / (p4 * 1e-6) / 1e9) if p4 > 0 else None,
                   "nvlink_frac_of_900": ((max(rb) / (p4 * 1e-6) / 1e9) / 900.0) if p4 > 0 else None,
                   "call_us_max": max(float(t[2]) for t in allv),
                   "tokens_per_s": T / (max(float(t[2]) for t in allv) * 1e-6)}
            print(json.dumps(rep), flush=True)
    layer.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
