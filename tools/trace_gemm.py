"""Timeline of k_layer (front phases, grouped GEMM units, combine) from its device trace.

    python tools/trace_gemm.py [--config mixtral_decode] [--tokens 256]

Prints the kernel span, per-SM finish spread (tail), and per-kind unit
durations (end time minus the previous unit end on the same SM).
"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as wl  # noqa: E402
import paper_2601_01310_b200 as tg  # noqa: E402
from bench import make_weights_device  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="mixtral_decode")
    ap.add_argument("--tokens", type=int, default=None)
    ap.add_argument("--W", type=int, default=1)
    ap.add_argument("--warm", type=int, default=5, help="untraced calls first (1000+: power-capped steady state)")
    a = ap.parse_args()
    sh = wl.CONFIGS[a.config]
    T = a.tokens or sh.T
    pl = wl.make_placement(sh.E, a.W, 1, shadows=a.W > 1)
    dev = torch.device("cuda", 0)
    L = make_weights_device(sh, 1001, dev, list(range(sh.E)))
    layer = tg.MoELayer(sh, pl, L, max_tokens_per_rank=T, device=0)
    x = wl.make_tokens(sh, 1001, T=T, device=dev)
    for _ in range(a.warm):
        layer(x)
    tg.tg_set_trace(layer.ctx, True)
    layer(x)
    layer(x)  # second traced call: the first one's end stamp gives the launch gap
    torch.cuda.synchronize()
    tr = tg.tg_get_trace(layer.ctx)
    st = tr["front_stamps"]
    if st[0] > 0:
        print("front phases (us from start): group0 top-k %.2f, chunk0 rank %.2f, exchange start %.2f end %.2f, "
              "grid barrier %.2f, dispatch done %.2f" % tuple((st[i] - st[0]) / 1e3 if st[i] else -1
                                                             for i in (12, 13, 1, 14, 3, 4)))
        print("group 0: part arrivals", [round((v - st[0]) / 1e3, 2) if v else -1 for v in st[40:48]],
              "last-arriver start %.2f, logits summed %.2f, top-k done %.2f" % tuple((st[i] - st[0]) / 1e3 if st[i] else -1 for i in (30, 31, 12)))
        print("row 0 top-k: entry %.2f select %.2f slots %.2f Z %.2f stores %.2f | pass1 done %.2f pass2 done %.2f" % tuple((st[i] - st[0]) / 1e3 if st[i] else -1 for i in (32, 33, 34, 35, 36, 37, 38)))
        stc = tr["front_stamps_raw"]
        if st[32] and st[33]:
            print("row-0 select loop: %.2f us, %d SM cycles -> %.0f MHz" % ((st[33] - st[32]) / 1e3, stc[51] - stc[50], (stc[51] - stc[50]) / ((st[33] - st[32]) / 1e3)))
        print("router detail (us from front start): zero-ctr %.2f | item0: start %.2f x-tile %.2f"
              % tuple((st[i] - st[0]) / 1e3 if st[i] else -1 for i in (8, 10, 11)))
        print("block0 items (start,end) us:", [(round((st[20 + 2 * i] - st[0]) / 1e3, 2), round((st[21 + 2 * i] - st[0]) / 1e3, 2)) for i in range(5) if st[20 + 2 * i]])
        fb = (tr["front_block_p1"] - st[0]) / 1e3
        print("front P1 finish per block: min %.1f median %.1f max %.1f  argmax %d" % (fb.min(), np.median(fb), fb.max(), int(np.argmax(fb))))
        for key in ("front_block_router", "front_block_prefetch", "front_block_bar1"):
            v = tr[key]
            if (v > 0).any():
                v = (v[v > 0] - st[0]) / 1e3
                print("%s per block: min %.1f p10 %.1f median %.1f p90 %.1f max %.1f" % (
                    key, v.min(), np.percentile(v, 10), np.median(v), np.percentile(v, 90), v.max()))
        tc = tr["topk_cycles"]
        if (tc[:, 1] > 0).any():  # grid-stride top-k: each block's first (cold code) and second group
            c1, c2 = tc[:, 0][tc[:, 1] > 0], tc[:, 1][tc[:, 1] > 0]
            print("top-k kcycles per group, block's first / second: median %.1f / %.1f, max %.1f / %.1f" % (
                np.median(c1) / 1e3, np.median(c2) / 1e3, c1.max() / 1e3, c2.max() / 1e3))
        ic = tr["item_clock"]
        if ic[0] and ic[2] > ic[0]:
            print("router item 1 of block 0: %.2f us, %d cycles -> %.0f MHz" % (
                (ic[2] - ic[0]) / 1e3, ic[3] - ic[1], (ic[3] - ic[1]) / ((ic[2] - ic[0]) / 1e3)))
        td = tr["topk_detail"].reshape(2, 6)
        for i in range(2):
            if td[i, 4]:
                print("block 0 group %d top-k cycles: gather %d, select %d, slot+Z %d, stores %d" % (
                    i, td[i, 5] - td[i, 4], td[i, 1] - td[i, 0], td[i, 2] - td[i, 1], td[i, 3] - td[i, 2]))
        if st[19] and st[18]:
            print("launch gap: previous call end -> entry %.2f us, entry -> front start (PDL wait) %.2f us"
                  % ((st[18] - st[19]) / 1e3, (st[0] - st[18]) / 1e3))
        t0g = tr["start"].min()
        print("gemm: CTA start %.1f us after front start; grid barrier at %.1f, combine done %.1f us after GEMM start"
              % ((t0g - st[0]) / 1e3, (st[16] - t0g) / 1e3, (st[17] - t0g) / 1e3))
    np.savez(os.path.join(ROOT, "gpurun_out", f"trace_{a.config}_{T}.npz"), **tr)
    analyze(tr)


def analyze(tr):
    end, smid, start, kind = tr["end"], tr["smid"], tr["start"], tr["kind"]
    t0 = start.min()
    end = (end - t0) / 1e3
    print("units", len(end), "span %.1f us" % end.max())
    fin = {}
    for e, s in zip(end, smid):
        fin[s] = max(fin.get(s, 0), e)
    fin = np.array(list(fin.values()))
    print(" per-SM finish min %.1f p10 %.1f median %.1f max %.1f -> mean idle tail %.1f us" % (
        fin.min(), np.percentile(fin, 10), np.median(fin), fin.max(), fin.max() - fin.mean()))
    order = np.argsort(end)
    last = {}
    durs = {0: [], 1: [], 2: [], 3: []}
    for i in order:
        s = smid[i]
        durs[int(kind[i])].append(end[i] - last.get(s, 0.0))
        last[s] = end[i]
    for kd, v in durs.items():
        if v:
            v = np.array(v)
            print(" kind %d n %d mean %.2f p50 %.2f p90 %.2f max %.2f" % (kd, len(v), v.mean(), np.median(v),
                                                                        np.percentile(v, 90), v.max()))


if __name__ == "__main__":
    main()
