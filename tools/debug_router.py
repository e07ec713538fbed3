import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__)))); sys.path.insert(0, 'tests')
import workloads as wl, paper_2601_01310_b200 as tg
from parity_util import oracle_layer
for cfg, W in (("tiny", 2), ("mixtral_decode", 1)):
    sh = wl.CONFIGS[cfg]; L = wl.make_layer(sh, 1000); x = wl.make_tokens(sh, 1000); pl = wl.make_placement(sh.E, W, 1)
    layer = tg.MoELayer(sh, pl, L, max_tokens_per_rank=sh.T)
    out = layer(x.cuda()); torch.cuda.synchronize()
    rt = layer.routing(sh.T)
    w1 = [wl.as_u16(a) for a in L.w1]; 
    import oracle
    lg = oracle.router(wl.as_u16(x), wl.as_u16(L.wg)); idx, w, gap = oracle.select(lg, sh.k)
    gi = rt["idx"].cpu().numpy(); gw = rt["w"].cpu().numpy()
    print(cfg, "idx match frac", (gi == idx).all(1).mean())
    print(" oracle idx", idx[:4].tolist(), "gpu", gi[:4].tolist())
    print(" oracle w", w[:2].tolist(), "gpu", gw[:2].tolist())
    print(" logits row0", lg[0].tolist())
    layer.close()
