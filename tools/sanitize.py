"""Tiny-config layer calls meant for compute-sanitizer (memcheck / racecheck / synccheck):

    compute-sanitizer --tool memcheck python tools/sanitize.py [--config tiny] [--calls 4]

(compute-sanitizer is closed on the round-2 GPU pool — it refuses to run, rc 86 — so the script is
run plainly there: a determinism and host-path check.)

Device-path calls (two buffer sets, consecutive launches), a masked-EW call, and host-buffer calls
(copy streams ordered by device words); every output is compared with the first call's, bitwise.
"""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as wl  # noqa: E402
import paper_2601_01310_b200 as tg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="tiny")
    ap.add_argument("--calls", type=int, default=4)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    sh = wl.CONFIGS[a.config]
    L = wl.make_layer(sh, seed=1000)
    x = wl.make_tokens(sh, seed=1000).cuda()
    pl = wl.make_placement(sh.E, 2, 1)
    layer = tg.MoELayer(sh, pl, L, max_tokens_per_rank=sh.T, device=0)
    outs = [layer(x) for _ in range(a.calls)]
    torch.cuda.synchronize()
    bad = sum(int(not torch.equal(o.view(torch.int16), outs[0].view(torch.int16))) for o in outs)
    layer.mask_worker(1, 1)
    om = layer(x)
    torch.cuda.synchronize()
    bad += int(not torch.equal(om.view(torch.int16), outs[0].view(torch.int16)))
    xh = x.cpu().pin_memory()
    ohs = [torch.empty_like(xh).pin_memory() for _ in range(a.calls)]
    for o in ohs:
        assert tg.tg_moe_layer_host(layer.ctx, xh, o) == tg.TG_OK
    tg.tg_host_sync(layer.ctx)
    torch.cuda.synchronize()
    bad += sum(int(not torch.equal(o.view(torch.int16), outs[0].cpu().view(torch.int16))) for o in ohs)
    layer.close()
    print("sanitize run:", a.config, "calls", a.calls, "mismatches", bad, flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
