"""GPU (sm_100a) parity of the C-ABI path against the CPU oracle (criteria P1-P8,
SURVEY.md 8(c)); every call goes through libtarragon.so via the binding, and
every bf16 storage point is checked against the oracle's exact value of that
stage (tests/parity_util.py, R#21 / R#24)."""
import os

import numpy as np
import pytest
import torch

import workloads as wl
from parity_util import check, collect, oracle_layer, single

pytestmark = pytest.mark.gpu

NT = min(32, os.cpu_count() or 1)


def _tg():
    import paper_2601_01310_b200 as tg
    return tg


def _setup(cfg, W, seed, T=None, skew=0.0, integer=False, shadows=True, T_max=None):
    tg = _tg()
    sh = wl.CONFIGS[cfg] if isinstance(cfg, str) else cfg
    T = sh.T if T is None else T
    u = None
    if skew:
        u = torch.randn(sh.d, generator=torch.Generator().manual_seed(seed + 99))
        u = u / u.norm() * sh.d ** 0.5
    L = wl.integer_layer(sh, seed) if integer else wl.make_layer(sh, seed, skew=skew, u=u)
    x = wl.integer_tokens(sh, seed, T) if integer else wl.make_tokens(sh, seed, T, skew_mu=skew, u=u)
    pl = wl.make_placement(sh.E, W, 1, shadows=shadows)
    layer = tg.MoELayer(sh, pl, L, max_tokens_per_rank=T_max or max(T, 1))
    layer.export_stages(True)
    return tg, sh, L, x, pl, layer


def _run(layer, x):
    xd = x.cuda()
    out = layer(xd)
    torch.cuda.synchronize()
    return out


def test_library_is_native_and_loaded():
    tg = _tg()
    assert os.path.exists(tg.LIB_PATH)
    with open("/proc/self/maps") as f:
        assert "libtarragon.so" in f.read()


@pytest.mark.parametrize("skew", [0.0, 0.6])
def test_tiny_parity_mask_poison_flip(skew):
    """configs[0]: tiny layer, 2 logical EWs with shadows on one B200; EW1 masked mid-run."""
    tg, sh, L, x, pl, layer = _setup("tiny", 2, seed=1000, skew=skew)
    out0 = _run(layer, x)
    rep = single(layer, out0, L, x, pl, [0, 0])
    print("tiny", skew, rep)
    # P6 determinism
    out0b = _run(layer, x)
    assert torch.equal(out0.view(torch.int16), out0b.view(torch.int16))
    # P8 shadows idle when unmasked
    st = layer.stats()
    base = [tg.tg_bank_slot(layer.ctx, ew, 0) for ew in range(pl.n_ews)]
    for ew in range(pl.n_ews):
        for sl, e in enumerate(pl.hosted[ew]):
            if e >= 0 and tuple(pl.cand[e, 0]) != (ew, sl):
                assert st[0, base[ew] + sl] == 0
    # P5 mask EW1 -> bit-identical; its slots poisoned with NaN
    assert layer.mask_worker(1, 1) == tg.TG_OK
    nan = torch.full((sh.F, sh.d), float("nan"), dtype=torch.bfloat16, device="cuda")
    nan2 = torch.full((sh.d, sh.F), float("nan"), dtype=torch.bfloat16, device="cuda")
    for sl, e in enumerate(pl.hosted[1]):
        if e >= 0:
            tg.tg_load_experts(layer.ctx, 1, sl, e, nan, nan, nan2)
    st0 = layer.stats()
    out1 = _run(layer, x)
    assert torch.equal(out0.view(torch.int16), out1.view(torch.int16)), "masked output differs"
    st1 = layer.stats() - st0
    for sl in range(pl.slots_per_ew):
        assert st1[0, base[1] + sl] == 0, "masked EW received rows"
    single(layer, out1, L, x, pl, [0, 1])


def test_route_flip_bit_identity():
    """configs[4] protocol on the tiny layer: table A (primaries first) / B (shadows first) alternate."""
    tg, sh, L, x, pl, layer = _setup("tiny", 2, seed=1001)
    outA = _run(layer, x)
    for i in range(6):
        cand = wl.flipped(pl.cand) if i % 2 == 0 else pl.cand
        assert layer.set_route_table(cand) == tg.TG_OK
        o = _run(layer, x)
        assert torch.equal(outA.view(torch.int16), o.view(torch.int16)), f"flip {i} changed output"
        pl2 = wl.Placement(pl.n_ews, pl.ew_rank, pl.slots_per_ew, pl.hosted, cand)
        single(layer, o, L, x, pl2, [0, 0])
    # stale versions are ignored
    assert tg.tg_set_route_table(layer.ctx, layer.version, pl.cand) == tg.TG_ERR_STALE_VERSION
    # a slot the active table names for another expert cannot be overwritten
    e0 = pl.hosted[0][0]
    other = (e0 + 1) % sh.E
    with pytest.raises(tg.TarragonError):
        tg.tg_load_experts(layer.ctx, 0, 0, other, L.w1[other], L.w3[other], L.w2[other])


def test_integer_ties_bit_exact():
    """Integer router inputs: logits exact in any order, so lowest-id tie breaks must match exactly."""
    tg, sh, L, x, pl, layer = _setup("tiny", 2, seed=1002, integer=True)
    out = _run(layer, x)
    ref = oracle_layer(L, x, pl, [0, 0], G=1)
    assert (ref["gap"] == 0).sum() > 10, "test needs exact ties"
    ref["gap"][:] = 1.0  # no near-tie exemption: idx and permutation bit-exact for every token
    rep = single(layer, out, L, x, pl, [0, 0], ref=ref)
    assert rep["max_dlogit"] == 0.0


@pytest.mark.parametrize("T", [1, 37, 300, 1000])
def test_ragged_and_multi_tile(T):
    """Ragged token counts; T = 1000 gives ~250 rows per expert -> 2 token tiles (128 + ragged)."""
    tg, sh, L, x, pl, layer = _setup("tiny", 2, seed=1003 + T, T=T)
    out = _run(layer, x)
    single(layer, out, L, x, pl, [0, 0])


@pytest.mark.parametrize("shape", [
    wl.Shape("k1_E1", d=64, E=1, k=1, F=128, T=200),     # dense SwiGLU FFN through the MoE path
    wl.Shape("k1_E8", d=128, E=8, k=1, F=192, T=300),    # w = 1 exactly, out = y
    wl.Shape("kE_8", d=64, E=8, k=8, F=128, T=256),      # k = E: dense softmax mixture, gap = +inf
], ids=lambda s: s.name)
def test_degenerate_k_and_E(shape):
    """The method's degenerate cases (SURVEY 8(c) special cases) through the GPU path."""
    tg, sh, L, x, pl, layer = _setup(shape, 2, seed=1020)
    out = _run(layer, x)
    rep = single(layer, out, L, x, pl, [0, 0])
    rt = layer.routing(x.shape[0])
    if sh.k == 1:
        assert torch.all(rt["w"] == 1.0)
    if sh.k == sh.E:
        assert rep["near_ties"] == 0
        assert torch.equal(rt["idx"].cpu(), torch.arange(sh.E, dtype=torch.int32).expand(x.shape[0], sh.E))
    layer.mask_worker(1, 1)
    assert torch.equal(out.view(torch.int16), _run(layer, x).view(torch.int16))


@pytest.mark.parametrize("mode", ["TG_WIDE", "TG_G2DUAL"])
@pytest.mark.parametrize("cfg,T", [("tiny", 1000), ("qwen_prefill", None), ("mixtral_decode", None)])
def test_tile_modes_parity(cfg, T, mode, monkeypatch):
    """GEMM tile variants forced on: wide token tiles (bn = 256, TMEM halves shared by a1|a3) and dual
    GEMM2 tiles (two W2 tiles per unit): same parity and mask bit-identity."""
    monkeypatch.setenv(mode, "1")
    if cfg == "tiny":
        tg, sh, L, x, pl, layer = _setup("tiny", 2, seed=1006, T=T)
        out = _run(layer, x)
        single(layer, out, L, x, pl, [0, 0])
        layer.mask_worker(1, 1)
        assert torch.equal(out.view(torch.int16), _run(layer, x).view(torch.int16))
    else:
        _big(cfg, 2004, n_sample=16, W=4 if cfg == "qwen_prefill" else 2)


@pytest.mark.parametrize("cfg", ["tiny", "mixtral_decode"])
def test_dual_and_single_gemm2_bitwise_equal(cfg, monkeypatch):
    """Two W2 tiles per GEMM2 unit (default) or one (TG_G2DUAL=0): every output element sees the
    same MMAs in the same K order, so the outputs are bitwise equal."""
    tg = _tg()
    sh = wl.CONFIGS[cfg]
    L = wl.make_layer(sh, 1010)
    x = wl.make_tokens(sh, 1010)
    pl = wl.make_placement(sh.E, 2, 1)
    outs = []
    for dual in ("0", "1"):
        monkeypatch.setenv("TG_G2DUAL", dual)
        layer = tg.MoELayer(sh, pl, L, max_tokens_per_rank=sh.T)
        outs.append(_run(layer, x).view(torch.int16).clone())
        layer.close()
    assert torch.equal(outs[0], outs[1])


def test_empty_call_and_errors():
    tg, sh, L, x, pl, layer = _setup("tiny", 2, seed=1004, T=16, T_max=64)
    empty = torch.empty(0, sh.d, dtype=torch.bfloat16, device="cuda")
    assert tg.tg_moe_layer(layer.ctx, empty, torch.empty_like(empty)) == tg.TG_OK
    torch.cuda.synchronize()
    with pytest.raises(tg.TarragonError):  # routing export is sized by the last call's tokens
        layer.routing(16)
    out = _run(layer, x)
    single(layer, out, L, x, pl, [0, 0])
    # too many tokens
    big = torch.zeros(65, sh.d, dtype=torch.bfloat16, device="cuda")
    assert tg.tg_moe_layer(layer.ctx, big, torch.empty_like(big)) == tg.TG_ERR_INVALID
    # mask both EWs -> NO_ROUTE, nothing launched; unmask recovers
    assert layer.mask_worker(0, 1) == tg.TG_OK
    assert layer.mask_worker(1, 1) == tg.TG_ERR_NO_ROUTE
    xd = x.cuda()
    assert tg.tg_moe_layer(layer.ctx, xd, torch.empty_like(xd)) == tg.TG_ERR_NO_ROUTE
    assert layer.mask_worker(0, 0) == tg.TG_OK
    o2 = _run(layer, x)
    assert torch.equal(out.view(torch.int16), o2.view(torch.int16))


@pytest.mark.parametrize("cfg,ncalls", [("tiny", 12), ("mixtral_decode", 8)])
def test_host_entry_point_e2e(cfg, ncalls):
    """tg_moe_layer_host: pinned host in/out, copies inside the call; the copy streams are
    ordered against the layer launches by device words (no stream op between the launches), over
    the two staging buffers, with a different token count per call."""
    tg, sh, L, x, pl, layer = _setup(cfg, 2, seed=1005)
    layer.export_stages(False)  # nothing else on the stream between the launches
    xh = x.pin_memory()
    oh = torch.empty_like(xh).pin_memory()
    assert tg.tg_moe_layer_host(layer.ctx, xh, oh) == tg.TG_OK
    tg.tg_host_sync(layer.ctx)
    torch.cuda.synchronize()
    od = _run(layer, x)
    assert torch.equal(oh.view(torch.int16), od.cpu().view(torch.int16))
    # pipelined calls over the two staging buffers, different inputs (and sizes) per call
    sizes = [sh.T, max(sh.T - 3, 1), max(sh.T // 2, 1), 1, 0, sh.T]  # (0: a call with no tokens)
    xs = [wl.make_tokens(sh, 2000 + i, sizes[i % len(sizes)]).pin_memory() for i in range(ncalls)]
    ohs = [torch.empty_like(v).pin_memory() for v in xs]
    for v, o in zip(xs, ohs):
        assert tg.tg_moe_layer_host(layer.ctx, v, o) == tg.TG_OK
    tg.tg_host_sync(layer.ctx)
    torch.cuda.synchronize()
    for v, o in zip(xs, ohs):
        ref = _run(layer, v.cuda()).cpu()
        assert torch.equal(o.view(torch.int16), ref.view(torch.int16))


def _big(cfg, seed, n_sample, W=2, T=None, skew=0.0):
    tg, sh, L, x, pl, layer = _setup(cfg, W, seed=seed, T=T, skew=skew)
    out = _run(layer, x)
    Tn = x.shape[0]
    if n_sample is None or n_sample >= Tn:
        tok = None
    else:
        rng = np.random.default_rng(seed)
        tok = np.sort(rng.choice(Tn, size=n_sample, replace=False)).astype(np.int32)
        tok[0] = 0
        tok[-1] = Tn - 1
    rep = single(layer, out, L, x, pl, [0] * W, tokens=tok, n_threads=NT)
    print(cfg, "skew" if skew else "", rep)
    # mask EW1: bit-identical at full size
    layer.mask_worker(1, 1)
    out1 = _run(layer, x)
    assert torch.equal(out.view(torch.int16), out1.view(torch.int16))
    layer.close()
    return rep


def test_mixtral_decode_parity_full_T():
    """configs[1]: Mixtral-shaped layer, T = 256 decode batch; routing AND the FFN of every token
    (full-T FFN parity on Mixtral decode)."""
    _big("mixtral_decode", 2001, n_sample=None)


def test_ds_v2_lite_shared_parity():
    """configs[3] shape (64 experts top-6 + 2 shared merged to 2816) at T = 1024 on one GPU."""
    _big("ds_v2_lite_decode", 2002, n_sample=48, W=8)


def test_qwen_prefill_parity():
    """configs[4] shape: 60 experts top-4, prefill T = 8192 (multi-tile slots)."""
    _big("qwen_prefill", 2003, n_sample=48, W=4)


@pytest.mark.parametrize("cfg,W", [("ds_v2_lite_decode", 8), ("qwen_prefill", 4)])
def test_skewed_routing_parity(cfg, W):
    """App. B imbalance: skewed routing (top expert ~3x the mean load) at full size."""
    _big(cfg, 2006, n_sample=32, W=W, skew=0.6)


@pytest.mark.parametrize("cfg,W", [("ds_v2_lite_decode_g1", 8), ("qwen_prefill_sg", 4)])
def test_next3b_gating_variants(cfg, W):
    """NEXT-3b: the public DS-V2-Lite / Qwen1.5-MoE gating (softmax over all E, top-k weights not
    renormalised) and Qwen's sigmoid-gated shared expert (F_sh 5632), parity + mask bit-identity."""
    _big(cfg, 2005, n_sample=32, W=W)


@pytest.mark.parametrize("cfg,ncalls", [("mixtral_decode", 240), ("ds_v2_lite_decode", 160), ("qwen_prefill", 40)])
def test_back_to_back_calls(cfg, ncalls):
    """Epoch-flag / buffer-set stress: ncalls launches back to back with no host
    synchronisation — consecutive calls overlap (PDL), decode calls start their GEMM on a ready
    word with claimed router items and row copies — alternating two inputs and, on the host-buffer
    path, ordered by device words; every output is bitwise the single call's output for its input."""
    tg, sh, L, x0, pl, layer = _setup(cfg, 2, seed=1100)
    layer.export_stages(False)
    xs = [x0.cuda(), wl.make_tokens(sh, 1101).cuda()]
    refs = [_run(layer, v).clone() for v in xs]
    outs = [torch.empty_like(xs[0]) for _ in range(ncalls)]
    for i in range(ncalls):
        layer(xs[i % 2], outs[i])
    torch.cuda.synchronize()
    bad = [i for i in range(ncalls) if not torch.equal(outs[i].view(torch.int16), refs[i % 2].view(torch.int16))]
    assert not bad, f"calls {bad[:8]} (of {len(bad)}) differ from their input's reference"
    # host-buffer path, same stress
    xh = [v.cpu().pin_memory() for v in xs]
    n_h = min(ncalls, 64) if sh.T <= 1024 else 8  # (pinned host memory)
    ohs = [torch.empty_like(xh[0]).pin_memory() for _ in range(n_h)]
    for i in range(n_h):
        assert tg.tg_moe_layer_host(layer.ctx, xh[i % 2], ohs[i]) == tg.TG_OK
    tg.tg_host_sync(layer.ctx)
    torch.cuda.synchronize()
    bad = [i for i in range(n_h) if not torch.equal(ohs[i].view(torch.int16), refs[i % 2].cpu().view(torch.int16))]
    assert not bad, f"host-path calls {bad[:8]} (of {len(bad)}) differ"
    layer.close()
