"""Diagnostic: G ranks, the same x every call; per call, elements differing from call 1 (and the
tokens affected), with and without a device sync between calls."""
import os, sys, json
import torch, torch.distributed as dist
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as wl
import paper_2601_01310_b200 as tg
from bench import make_weights_device

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local); dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
cfg = sys.argv[1] if len(sys.argv) > 1 else "mixtral_decode"
sh = wl.CONFIGS[cfg]; T = sh.T; Tr = T // world
pl = wl.make_placement(sh.E, world, world)
experts = sorted({e for ew in range(world) if pl.ew_rank[ew] == rank for e in pl.hosted[ew] if e >= 0})
L = make_weights_device(sh, 1001, dev, experts)
layer = tg.MoELayer(sh, pl, L, max_tokens_per_rank=Tr, rank=rank, world=world, device=local, group=dist.group.WORLD)
x = wl.make_tokens(sh, 1001, T=T, device=dev)[rank * Tr:(rank + 1) * Tr].contiguous()
res = {}
for mode in ("sync", "back2back"):
    outs = [torch.empty_like(x) for _ in range(6)]
    for i in range(6):
        layer(x, outs[i])
        if mode == "sync":
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    ref = outs[0].view(torch.int16)
    r = []
    for i in range(1, 6):
        dif = (outs[i].view(torch.int16) != ref)
        toks = dif.any(dim=1).nonzero().flatten()
        r.append({"call": i + 1, "n_diff": int(dif.sum()), "tokens": toks[:8].tolist(), "n_tokens": int(toks.numel())})
    res[mode] = r
allr = [None] * world
dist.all_gather_object(allr, {"rank": rank, **res})
if rank == 0:
    for a in allr:
        print(json.dumps(a))
layer.close(); dist.destroy_process_group()
