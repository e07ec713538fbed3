"""NVLink bytes of the dispatch / combine exchanges from the hardware counters (NVML), G ranks.

    torchrun --nproc-per-node G --master-addr 127.0.0.1 --master-port P tools/nvlink_counters.py \
        [--config qwen_prefill] [--W 2G] [--calls 50]

Every rank reads its GPU's cumulative NVLink data counters (NVML field values
THROUGHPUT_DATA_TX / RX, summed over the links, KiB) around K back-to-back
layer calls, and reports per call: bytes sent / received over NVLink, the
algorithmic exchange bytes of the call (rows this rank stored into peers' receive
buffers + expert outputs it stored into peers' combine buffers, d*2 B each), the
call time (CUDA events), the exchange phases' time from the kernel's device
timestamps (dispatch: front barrier -> data flags released; combine: last GEMM
unit -> call end), and GB/s per direction over those phases.  Rank 0 prints one
JSON line (per-rank records).  The counters, not timestamps alone, are the
evidence of the bytes moved.
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


NVML_RC = {}


def smi_kib(index):
    """Fallback: `nvidia-smi nvlink -gt d` data throughput counters (KiB, summed over the links)."""
    import re
    import subprocess
    r = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", str(index)], capture_output=True, text=True)
    tx = sum(int(v) for v in re.findall(r"Data Tx:\s*(\d+)\s*KiB", r.stdout))
    rx = sum(int(v) for v in re.findall(r"Data Rx:\s*(\d+)\s*KiB", r.stdout))
    NVML_RC["smi_tail"] = r.stdout[-300:] + r.stderr[-200:]
    return tx, rx


def nvlink_kib(handle, index, nlinks=18):
    import pynvml as p
    ids = []
    for f in (p.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, p.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX):
        for l in range(nlinks):
            ids.append((f, l))
    tx = rx = 0
    ok = False
    try:
        vals = p.nvmlDeviceGetFieldValues(handle, ids)
        for (f, _), v in zip(ids, vals):
            NVML_RC[v.nvmlReturn] = NVML_RC.get(v.nvmlReturn, 0) + 1
            if v.nvmlReturn != 0:
                continue
            ok = True
            x = v.value.ullVal
            if f == p.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX:
                tx += x
            else:
                rx += x
    except Exception as e:  # noqa: BLE001
        NVML_RC["exc"] = str(e)
    if not ok or (tx == 0 and rx == 0):
        NVML_RC["source"] = "nvidia-smi"
        return smi_kib(index)
    NVML_RC["source"] = "nvml"
    return tx, rx


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="qwen_prefill")
    ap.add_argument("--W", type=int, default=0)
    ap.add_argument("--calls", type=int, default=50)
    a = ap.parse_args()
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    import pynvml as p
    p.nvmlInit()
    h = p.nvmlDeviceGetHandleByIndex(torch.cuda.current_device() if "CUDA_VISIBLE_DEVICES" in os.environ else local)
    sh = wl.CONFIGS[a.config]
    W = a.W or world
    T = sh.T
    Tr = T // world
    pl = wl.make_placement(sh.E, W, world)
    experts = sorted({e for ew in range(W) if pl.ew_rank[ew] == rank for e in pl.hosted[ew] if e >= 0})
    L = make_weights_device(sh, 1001, dev, experts)
    layer = tg.MoELayer(sh, pl, L, max_tokens_per_rank=Tr, rank=rank, world=world, device=local,
                        group=dist.group.WORLD)
    x = wl.make_tokens(sh, 1001, T=T, device=dev)[rank * Tr:(rank + 1) * Tr].contiguous()
    out = torch.empty_like(x)
    for _ in range(10):
        layer(x, out)
    torch.cuda.synchronize()
    dist.barrier()
    tx0, rx0 = nvlink_kib(h, local)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.calls):
        layer(x, out)
    e1.record()
    torch.cuda.synchronize()
    tx1, rx1 = nvlink_kib(h, local)
    dist.barrier()
    ms = e0.elapsed_time(e1) / a.calls
    # algorithmic exchange bytes of this rank (per call): dispatched rows to peers + y rows stored in peers
    rt = layer.routing(Tr)
    dr = rt["dst_rank"].cpu().numpy()
    to_peers = int((dr != rank).sum())
    counts = rt["counts"].cpu().numpy()
    # phase times from the device trace of one more call
    tg.tg_set_trace(layer.ctx, True)
    layer(x, out)
    layer(x, out)
    torch.cuda.synchronize()
    tr = tg.tg_get_trace(layer.ctx)
    st = tr["front_stamps"]
    disp_us = (st[4] - st[3]) / 1e3 if st[4] and st[3] else None
    comb_us = (st[17] - st[16]) / 1e3 if st[17] and st[16] else None
    tg.tg_set_trace(layer.ctx, False)
    rec = {"rank": rank, "calls": a.calls, "ms_per_call": ms,
           "nvlink_tx_MB_per_call": (tx1 - tx0) * 1024 / a.calls / 1e6,
           "nvlink_rx_MB_per_call": (rx1 - rx0) * 1024 / a.calls / 1e6,
           "pairs_to_peers": to_peers, "rows_from_peers": int(counts[rank].sum()) - int((dr == rank).sum()),
           "algorithmic_dispatch_MB": to_peers * sh.d * 2 / 1e6,
           "dispatch_phase_us": disp_us, "combine_phase_us": comb_us,
           "counter_source": {str(k): v for k, v in NVML_RC.items()}}
    if disp_us:
        rec["dispatch_GBps_per_direction"] = rec["algorithmic_dispatch_MB"] * 1e6 / (disp_us * 1e-6) / 1e9
    if rec["nvlink_tx_MB_per_call"] > 0 and disp_us and comb_us:
        rec["counter_GBps_tx_over_exchange_phases"] = rec["nvlink_tx_MB_per_call"] * 1e6 / ((disp_us + comb_us) * 1e-6) / 1e9
    recs = [None] * world
    dist.all_gather_object(recs, rec)
    if rank == 0:
        print(json.dumps({"config": a.config, "T": T, "G": world, "W": W, "ranks": recs,
                          "note": "dedup on (>= 16 MB of rows): a token is sent once per peer rank" if
                          T * sh.k * sh.d * 2 >= (16 << 20) else "dedup off"}), flush=True)
    layer.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
