"""The multi-rank data plane on ONE GPU: G virtual ranks (one ctx each, same process, same
device) connected by device pointer (tg_connect_local), their calls run as ONE cooperative
launch (tg_moe_layer_multi: rank r on CTAs [r n_SM / G, (r + 1) n_SM / G)).  Count exchange, peer dispatch stores, the combine exchange fused into the
GEMM2 epilogue, epoch flags, token dedup, masks, rank fail-stop and in-call failover run the
same code as over NVLink (peer addresses are just other ranks' regions); only the transport
differs.  SURVEY.md 8(e), P:739 (no collective group per call), P:914-920 (in-call failover),
P:927-941 (EWs tolerate AW failures)."""
import os

import numpy as np
import pytest
import torch

import workloads as wl
from parity_util import check, collect

pytestmark = pytest.mark.gpu

NT = min(32, os.cpu_count() or 1)


def _tg():
    import paper_2601_01310_b200 as tg
    return tg


class World:
    """G virtual ranks of one layer; global batch x split contiguously (R#12)."""

    def __init__(self, cfg, G, W=None, seed=3000, T=None, fail_ms=None):
        tg = _tg()
        self.tg = tg
        self.sh = wl.CONFIGS[cfg] if isinstance(cfg, str) else cfg
        self.G, self.W = G, W or G
        self.T = T or self.sh.T
        assert self.T % G == 0
        self.Tr = self.T // G
        self.L = wl.make_layer(self.sh, seed)
        self.x = wl.make_tokens(self.sh, seed, self.T)
        self.pl = wl.make_placement(self.sh.E, self.W, G)
        self.layers = tg.local_ranks(self.sh, self.pl, self.L, self.Tr, G)
        for l in self.layers:
            l.export_stages(True)
            if fail_ms:
                tg.tg_set_failure_timeout(l.ctx, fail_ms)
        self.xs = [self.x[r * self.Tr:(r + 1) * self.Tr].contiguous().cuda() for r in range(G)]

    def call(self, skip=(), xs=None):
        rc, outs = self.tg.call_all(self.layers, xs or self.xs, skip=skip)
        torch.cuda.synchronize()
        assert rc == self.tg.TG_OK, self.tg.tg_last_error(self.layers[0].ctx)
        return outs

    def failover_all(self, outs, ranks):
        """tg_failover of every survivor (collective among them): one fused replay launch."""
        skip = [r for r in range(self.G) if r not in ranks]
        rc, failed = self.tg.failover_all(self.layers, self.xs, outs, skip=skip)
        torch.cuda.synchronize()
        return {r: (rc, failed[r]) for r in ranks}

    def check(self, outs, mask=None, tokens=None):
        views = [collect(l, o, t0=r * self.Tr) for r, (l, o) in enumerate(zip(self.layers, outs))]
        return check(views, self.L, self.x, self.pl, mask or [0] * self.W, tokens=tokens, n_threads=NT)

    def one_gpu(self):
        """P7 reference: the same layer as ONE rank with all tokens."""
        pl1 = wl.make_placement(self.sh.E, self.W, 1)
        one = self.tg.MoELayer(self.sh, pl1, self.L, max_tokens_per_rank=self.T)
        o = one(self.x.cuda())
        torch.cuda.synchronize()
        one.close()
        return o

    def close(self):
        for l in self.layers:
            l.close()


def _eq(a, b):
    return torch.equal(a.view(torch.int16), b.view(torch.int16))


@pytest.mark.parametrize("cfg,G,Wm,sample", [("tiny", 2, 1, None), ("tiny", 4, 2, None),
                                             ("mixtral_decode", 2, 1, 24), ("mixtral_decode", 4, 1, 16)])
def test_virtual_ranks_parity_mask_flip(cfg, G, Wm, sample):
    """P1-P4 on every rank (strict, per storage point), P7 output bitwise equal to one rank,
    P6 run-to-run, P5 masked EW (its slots NaN-poisoned on its rank) and route flips bit-identical,
    P8 the masked EW receives no rows."""
    w = World(cfg, G, W=G * Wm)
    outs = w.call()
    tok = None
    if sample:
        tok = np.sort(np.random.default_rng(G).choice(w.T, size=sample, replace=False)).astype(np.int32)
    rep = w.check(outs, tokens=tok)
    print(cfg, G, rep)
    full = torch.cat(outs)
    assert _eq(full, w.one_gpu()), "P7: G-rank output differs from the 1-rank output"
    assert all(_eq(a, b) for a, b in zip(outs, w.call())), "P6"
    tg, sh = w.tg, w.sh
    ew = 1
    for l in w.layers:
        assert l.mask_worker(ew, 1) == tg.TG_OK
    host = w.layers[w.pl.ew_rank[ew]]
    nan = torch.full((sh.F, sh.d), float("nan"), dtype=torch.bfloat16, device="cuda")
    nan2 = torch.full((sh.d, sh.F), float("nan"), dtype=torch.bfloat16, device="cuda")
    for sl, e in enumerate(w.pl.hosted[ew]):
        if e >= 0:
            tg.tg_load_experts(host.ctx, ew, sl, e, nan, nan, nan2)
    st0 = [l.stats() for l in w.layers]
    outs_m = w.call()
    assert all(_eq(a, b) for a, b in zip(outs, outs_m)), "P5: masked output differs"
    bank = [tg.tg_bank_slot(w.layers[0].ctx, e_, 0) for e_ in range(w.W)]
    for l, s0 in zip(w.layers, st0):
        st = l.stats() - s0
        assert all(st[w.pl.ew_rank[ew], bank[ew] + sl] == 0 for sl in range(w.pl.slots_per_ew)), "P8"
    for i in range(4):
        cand = wl.flipped(w.pl.cand) if i % 2 == 0 else w.pl.cand
        for l in w.layers:
            assert l.set_route_table(cand) == tg.TG_OK
        assert all(_eq(a, b) for a, b in zip(outs, w.call())), f"flip {i} differs"
    w.close()


def test_virtual_prefill_token_dedup():
    """NEXT-2 token dedup (>= 16 MB of dispatched rows: each token sent once per peer rank, the
    peer copies it into its other pairs' rows) on the Qwen-shaped prefill, G = 2: strict parity on
    sampled tokens, masks, and the output bitwise equal to one rank."""
    w = World("qwen_prefill", 2, W=4)
    outs = w.call()
    tok = np.sort(np.random.default_rng(7).choice(w.T, size=24, replace=False)).astype(np.int32)
    print(w.check(outs, tokens=tok))
    assert _eq(torch.cat(outs), w.one_gpu())
    for l in w.layers:
        l.mask_worker(1, 1)
    assert all(_eq(a, b) for a, b in zip(outs, w.call()))
    w.close()


@pytest.mark.parametrize("cfg,G", [("tiny", 2), ("tiny", 4), ("mixtral_decode", 2)])
def test_virtual_rank_fail_stop(cfg, G):
    """NEXT-3a: the last rank stops calling; the survivors mask it and keep
    serving bit-identically, never sending it rows."""
    w = World(cfg, G)
    outs = w.call()
    dead = G - 1
    for r in range(G - 1):
        assert w.layers[r].mask_rank(dead) == w.tg.TG_OK
    st0 = [l.stats() for l in w.layers[:-1]]
    for i in range(3):
        o = w.call(skip=(dead,))
        assert all(_eq(outs[r], o[r]) for r in range(G - 1)), f"call {i} after the rank failed differs"
    for l, s0 in zip(w.layers[:-1], st0):
        assert int((l.stats() - s0)[dead].sum()) == 0
    w.close()


@pytest.mark.parametrize("cfg,G", [("tiny", 2), ("tiny", 4), ("mixtral_decode", 2), ("mixtral_decode", 4)])
def test_virtual_inflight_failover(cfg, G):
    """NEXT-1: the last rank crashes mid-call (after its dispatch, before its expert
    outputs).  Every survivor detects it in that call (combine-flag timeout), and tg_failover
    re-dispatches the pairs it held to the next live candidate on WHICHEVER surviving rank hosts
    it: the repaired output of that very call is bitwise the unfailed one; later calls too."""
    w = World(cfg, G, fail_ms=50.0)
    ref = w.call()
    dead = G - 1
    w.tg.tg_inject_failure(w.layers[dead].ctx)
    outs = w.call()
    res = w.failover_all(outs, range(G - 1))
    for r in range(G - 1):
        rc, failed = res[r]
        assert rc == w.tg.TG_OK and failed == 1 << dead, (r, rc, failed)
        assert _eq(ref[r], outs[r]), f"rank {r}: repaired output differs"
    for i in range(2):
        o = w.call(skip=(dead,))
        assert all(_eq(ref[r], o[r]) for r in range(G - 1))
        res = w.failover_all(o, range(G - 1))
        assert all(res[r][1] == 0 for r in range(G - 1)), "spurious failure after masking"
    w.close()


@pytest.mark.parametrize("G", [2, 4])
def test_virtual_peer_dies_before_counts(G):
    """A rank that dies before publishing its counts: the survivors' count exchange times out on
    it (no trap), they take its counts as zero (EW-side partial batch), dispatch nothing
    to it, and tg_failover re-routes the pairs its EWs would have served: bitwise outputs."""
    w = World("tiny", G, fail_ms=50.0)
    ref = w.call()
    dead = G - 1
    outs = w.call(skip=(dead,))
    res = w.failover_all(outs, range(G - 1))
    for r in range(G - 1):
        rc, failed = res[r]
        assert rc == w.tg.TG_OK and failed == 1 << dead, (r, rc, failed)
        assert _eq(ref[r], outs[r]), f"rank {r}: repaired output differs"
    o = w.call(skip=(dead,))
    assert all(_eq(ref[r], o[r]) for r in range(G - 1))
    w.close()


@pytest.mark.parametrize("cfg", ["tiny", "qwen_prefill"])
def test_virtual_rank_with_no_tokens(cfg):
    """A rank with T = 0 still takes part in the count exchange and serves its EWs; the others'
    outputs are bitwise those of the full call."""
    w = World(cfg, 2)
    ref = w.call()
    xs = list(w.xs)
    xs[1] = torch.empty(0, w.sh.d, dtype=torch.bfloat16, device="cuda")
    for i in range(2):
        o = w.call(xs=xs)
        assert _eq(ref[0], o[0])
    assert all(_eq(a, b) for a, b in zip(ref, w.call()))
    w.close()
