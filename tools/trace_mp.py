"""Per-rank timeline of one layer call on G GPUs (front phases, GEMM span, tail).

    torchrun --nproc-per-node G --master-addr 127.0.0.1 --master-port P tools/trace_mp.py [--config mixtral_decode]

Same placement as bench.py at N = G (W = G EWs, spread shadows, T global split
over the ranks).  Rank 0 prints one line per rank.
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
    ap.add_argument("--config", default="mixtral_decode")
    ap.add_argument("--tokens", type=int, default=None)
    a = ap.parse_args()
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    sh = wl.CONFIGS[a.config]
    T = a.tokens or sh.T
    Tr = T // world
    pl = wl.make_placement(sh.E, world, world)
    experts = sorted({e for ew in range(world) if pl.ew_rank[ew] == rank for e in pl.hosted[ew] if e >= 0})
    L = make_weights_device(sh, 1001, dev, experts)
    layer = tg.MoELayer(sh, pl, L, max_tokens_per_rank=Tr, rank=rank, world=world, device=local,
                        group=dist.group.WORLD)
    x = wl.make_tokens(sh, 1001, T=T, device=dev)[rank * Tr:(rank + 1) * Tr].contiguous()
    for _ in range(20):
        layer(x)
    torch.cuda.synchronize()
    dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(200):
        layer(x)
    ev1.record()
    torch.cuda.synchronize()
    call_us = ev0.elapsed_time(ev1) / 200 * 1e3
    dist.barrier()
    # steady state: trace stamps are overwritten by every call; the last of a back-to-back run is read
    tg.tg_set_trace(layer.ctx, True)
    for _ in range(30):
        layer(x)
    torch.cuda.synchronize()
    tr = tg.tg_get_trace(layer.ctx)
    tg.tg_set_trace(layer.ctx, False)
    st = tr["front_stamps"]
    f = lambda i: round((st[i] - st[0]) / 1e3, 2) if st[i] else -1  # noqa: E731
    t0g = tr["start"].min()
    end = (tr["end"] - t0g) / 1e3
    fin = {}
    for e, s in zip(end, tr["smid"]):
        fin[int(s)] = max(fin.get(int(s), 0.0), float(e))
    finv = np.array(list(fin.values())) if fin else np.zeros(1)
    rep = {"rank": rank, "call_us": round(call_us, 1),
           "launch_gap": round((st[18] - st[19]) / 1e3, 2) if st[18] and st[19] else None,
           "front": {"grp0_topk": f(12), "rank0": f(13), "xchg_start": f(1), "xchg_end": f(14), "barrier": f(3),
                     "dispatch_done": f(4)},
           "gemm_start_after_front_start": round((t0g - st[0]) / 1e3, 2),
           "gemm_units": int(len(end)), "gemm_span": round(float(end.max()) if len(end) else 0, 1),
           "gemm_first_unit_end": round(float(end.min()) if len(end) else 0, 1),
           "tail_mean_idle": round(float(finv.max() - finv.mean()), 1),
           "gemm_barrier": round((st[16] - t0g) / 1e3, 1), "combine_done": round((st[17] - t0g) / 1e3, 1)}
    reps = [None] * world
    dist.all_gather_object(reps, rep)
    if rank == 0:
        for r in reps:
            print(json.dumps(r), flush=True)
    layer.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
