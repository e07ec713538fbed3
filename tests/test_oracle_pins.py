"""Pins of the CPU oracle to things other than itself (paper's worked example,
brute force, closed forms, library special cases, invariants).  CPU only.

Each test names what it pins; see DESIGN.md §4 for the pin table.
"""
import itertools
import json
import os

import numpy as np
import pytest
import torch
import torch.nn.functional as Fn

import oracle
import workloads as wl
from bf16_ref import bf16_bits_to_f64, bf16_rne_exact

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def bf(a):
    """python/numpy numbers -> bf16 bit patterns (test inputs exactly representable)."""
    return wl.as_u16(torch.tensor(a, dtype=torch.float32).to(torch.bfloat16))


# ---------------------------------------------------------------- worked example

def _worked():
    with open(os.path.join(GOLD, "worked_example.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("masked", [False, True])
def test_worked_example(masked):
    """Hand-derived example (golden/worked_example.json)."""
    g = _worked()
    x, wg = bf(g["x"]), bf(g["wg"])
    w1 = [bf(a) for a in g["w1"]]
    w3 = [bf(a) for a in g["w3"]]
    w2 = [bf(a) for a in g["w2"]]
    cand = np.array(g["cand"], np.int32)
    mask = np.array([0, 1 if masked else 0], np.uint8)
    r = oracle.layer(x, wg, g["k"], w1, w3, w2, cand, g["ew_rank"], g["slots_per_ew"], mask, G=1)
    ex = g["expect"]
    assert r["rc"] == 0
    np.testing.assert_array_equal(r["logits"], np.array(ex["logits"], np.float32))
    np.testing.assert_array_equal(r["idx"], np.array(ex["idx"], np.int32))
    np.testing.assert_array_equal(r["w"], np.array(ex["w"], np.float64).astype(np.float32))
    np.testing.assert_array_equal(r["gap"], np.array(ex["gap"], np.float32))
    np.testing.assert_array_equal(r["out"], np.array(ex["out_bits"], np.uint16))
    pe = ex["ew1_masked" if masked else "unmasked"]
    np.testing.assert_array_equal(r["dst_slot"], np.array(pe["dst_slot"], np.int32))
    np.testing.assert_array_equal(r["dst_pos"], np.array(pe["dst_pos"], np.int32))
    np.testing.assert_array_equal(r["counts"], np.array(pe["counts"], np.int32))
    assert np.all(r["dst_rank"] == 0)


# ---------------------------------------------------------------- top-k

def _brute_topk(l, k):
    """The unique S with: for a in S, b not in S: l_a > l_b or (l_a == l_b and a < b)."""
    E = len(l)
    found = []
    for S in itertools.combinations(range(E), k):
        Sset = set(S)
        ok = all((l[a] > l[b]) or (l[a] == l[b] and a < b) for a in S for b in range(E) if b not in Sset)
        if ok:
            found.append(S)
    assert len(found) == 1
    return list(found[0])


@pytest.mark.parametrize("E", [2, 3, 5, 8, 10])
def test_topk_bruteforce_with_ties(E):
    """O2 vs exhaustive enumeration of all C(E,k) subsets, quantised logits force ties."""
    rng = np.random.default_rng(100 + E)
    T = 300
    logits = rng.integers(-3, 4, size=(T, E)).astype(np.float32)
    logits[::7] = 0.0           # all-equal rows
    logits[1::11, :] = -0.0     # signed zeros tie with zeros
    for k in range(1, E + 1):
        idx, w, gap = oracle.select(logits, k)
        for t in range(T):
            S = _brute_topk([float(v) for v in logits[t]], k)
            assert list(idx[t]) == sorted(S), (t, k, logits[t], idx[t], S)
            if k < E:
                order = sorted(range(E), key=lambda e: (-logits[t, e], e))
                assert gap[t] == logits[t, order[k - 1]] - logits[t, order[k]]


def test_softmax_closed_forms():
    """O3 closed forms: equal logits -> w = 1/k exactly; k = 1 -> w = 1; l = [2, 3] -> [1/(1+e), e/(1+e)]."""
    l = np.zeros((4, 8), np.float32)
    for k in (1, 2, 4, 8):
        idx, w, _ = oracle.select(l, k)
        assert np.all(idx == np.arange(k)[None, :])
        assert np.all(w == np.float32(1.0 / k))
    l = np.array([[2.0, 3.0, -1.0]], np.float32)
    idx, w, gap = oracle.select(l, 2)
    e = np.e
    assert list(idx[0]) == [0, 1]
    assert w[0, 0] == np.float32(1.0 / (1.0 + e)) and w[0, 1] == np.float32(e / (1.0 + e))
    assert gap[0] == np.float32(3.0)


def test_gate_mode1_is_full_softmax_then_topk():
    """O3' (gate_mode 1, NEXT-3b): w = softmax over all E (torch fp64), gathered at the selected ids,
    not renormalised; k = E reduces bitwise to gate_mode 0 (the renormalised softmax of all E)."""
    rng = np.random.default_rng(21)
    l = rng.standard_normal((500, 60)).astype(np.float32)
    for k in (1, 4, 6):
        idx, w, _ = oracle.select(l, k, gate_mode=1)
        idx0, _, _ = oracle.select(l, k, gate_mode=0)
        assert np.array_equal(idx, idx0)                       # selection unchanged
        full = torch.softmax(torch.from_numpy(l).double(), dim=1)
        ref = torch.gather(full, 1, torch.from_numpy(idx).long()).float().numpy()
        np.testing.assert_array_equal(w, ref)
        assert np.all(w.astype(np.float64).sum(1) < 1.0 + 1e-6)
    l8 = l[:, :8].copy()
    np.testing.assert_array_equal(oracle.select(l8, 8, gate_mode=1)[1], oracle.select(l8, 8, gate_mode=0)[1])


def test_shared_gate_closed_forms():
    """O7' (NEXT-3b): wsg = 0 -> sigmoid(0) = 0.5 exactly -> out = y_sh / 2 bitwise (routed experts zero);
    a gate logit >= 20 -> weight 1.0f -> out = y_sh bitwise; sigmoid matches torch in fp64."""
    d, F, T, E = 32, 64, 24, 4
    ws = _rand_expert(d, 48, 51)
    z = np.zeros((F, d), np.uint16)
    x = torch.randint(-2, 3, (T, d), generator=torch.Generator().manual_seed(52)).to(torch.bfloat16)
    pl = wl.make_placement(E, 1, 1, shadows=False)
    y_sh = _torch_swiglu_bf16(x, *ws)

    def run(wsg):
        return oracle.layer(wl.as_u16(x), np.zeros((E, d), np.uint16), 2, [z] * E, [z] * E,
                            [np.zeros((d, F), np.uint16)] * E, pl.cand, pl.ew_rank, pl.slots_per_ew,
                            np.zeros(1, np.uint8), G=1, shared=tuple(wl.as_u16(a) for a in ws),
                            wsg=wl.as_u16(wsg))
    r = run(torch.zeros(d, dtype=torch.bfloat16))
    assert np.all(r["sgate"] == np.float32(0.5))
    half = bf16_rne_exact(bf16_bits_to_f64(y_sh) * 0.5)
    np.testing.assert_array_equal(r["out"], half)
    big = torch.full((d,), 64.0, dtype=torch.bfloat16)      # x has a nonzero entry per row w.h.p.
    r = run(big)
    g = (x.double() @ big.double()).float()
    ok = g.numpy() >= 20
    assert ok.sum() > 5
    np.testing.assert_array_equal(r["sgate"], torch.sigmoid(g.double()).float().numpy())
    np.testing.assert_array_equal(r["out"][ok], y_sh[ok])


def test_softmax_sums_to_one_random():
    rng = np.random.default_rng(7)
    l = rng.standard_normal((2000, 60)).astype(np.float32)
    for k in (1, 2, 4, 6):
        _, w, _ = oracle.select(l, k)
        assert np.all(np.abs(w.astype(np.float64).sum(1) - 1.0) <= 1e-6)
        assert np.all(w > 0)


# ---------------------------------------------------------------- bf16 rounding

def test_bf16_rne_random_f64_vs_exact():
    """orc_bf16_from_f64 vs an independent exact RNE (frexp/ldexp), incl. exact midpoints."""
    rng = np.random.default_rng(3)
    v = np.concatenate([
        rng.standard_normal(200000) * np.exp2(rng.integers(-140, 130, 200000)),
        np.ldexp(np.arange(256, 512, dtype=np.float64) + 0.5, -8) * np.exp2(rng.integers(-120, 120, 256)),  # midpoints
        np.ldexp(np.arange(0, 300, dtype=np.float64) + 0.5, -133),      # subnormal midpoints
        [0.0, -0.0, 3.3895313892515355e38, 3.4e38, 1e39, -1e39, 1e-45, -1e-45, 2.0 ** -133, 2.0 ** -134,
         2.0 ** -134 * 1.0000001, 2.0 ** -126 * (1 - 2.0 ** -9), np.inf, -np.inf],
    ])
    got = oracle.bf16_from_f64(v)
    exp = bf16_rne_exact(v)
    np.testing.assert_array_equal(got, exp)
    n = oracle.bf16_from_f64(np.array([np.nan]))
    assert (int(n[0]) & 0x7F80) == 0x7F80 and (int(n[0]) & 0x7F) != 0


def test_bf16_rne_exhaustive_f32_vs_torch():
    """All 2^32 binary32 patterns: oracle's rounding == torch's float32->bfloat16 (RNE); NaNs as NaN."""
    chunk = 1 << 25
    torch.set_num_threads(max(1, os.cpu_count() or 1))
    for start in range(0, 1 << 32, chunk):
        bits = np.arange(start, start + chunk, dtype=np.uint64).astype(np.uint32)
        f = bits.view(np.float32)
        got = oracle.bf16_from_f32(f)
        ref = torch.from_numpy(f).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
        isnan = np.isnan(f)
        bad = (got != ref) & ~isnan
        assert not bad.any(), f"mismatch at 0x{int(bits[np.argmax(bad)]):08x}"
        g_nan = ((got & 0x7F80) == 0x7F80) & ((got & 0x7F) != 0)
        assert np.all(g_nan[isnan])


# ---------------------------------------------------------------- dense special cases

def _rand_expert(d, F, seed):
    g = torch.Generator().manual_seed(seed)
    w1 = (torch.randn(F, d, generator=g) * d ** -0.5).to(torch.bfloat16)
    w3 = (torch.randn(F, d, generator=g) * d ** -0.5).to(torch.bfloat16)
    w2 = (torch.randn(d, F, generator=g) * F ** -0.5).to(torch.bfloat16)
    return w1, w3, w2


def _torch_swiglu_bf16(x, w1, w3, w2):
    """Textbook SwiGLU FFN in torch fp64, bf16 storage of h and y (R#6, R#7)."""
    xd = x.double()
    h = Fn.silu(xd @ w1.double().T) * (xd @ w3.double().T)
    hb = torch.from_numpy(bf16_bits_to_f64(bf16_rne_exact(h.numpy())))
    y = hb @ w2.double().T
    return bf16_rne_exact(y.numpy())


def test_dense_E1_is_textbook_swiglu():
    """E = 1, k = 1: the MoE layer reduces to one dense SwiGLU FFN (torch fp64 reference)."""
    d, F, T = 96, 160, 64
    w1, w3, w2 = _rand_expert(d, F, 11)
    x = torch.randn(T, d, generator=torch.Generator().manual_seed(12)).to(torch.bfloat16)
    wg = torch.ones(1, d).to(torch.bfloat16)
    ex = _torch_swiglu_bf16(x, w1, w3, w2)
    cand = np.array([[[0, 0]]], np.int32)
    r = oracle.layer(wl.as_u16(x), wl.as_u16(wg), 1, [wl.as_u16(w1)], [wl.as_u16(w3)], [wl.as_u16(w2)],
                     cand, [0], 1, np.zeros(1, np.uint8), G=1)
    assert np.all(r["w"] == 1.0)
    np.testing.assert_array_equal(r["out"], ex)


def test_dense_k_equals_E_is_softmax_mixture():
    """k = E: out = bf16( sum_e softmax(l)_e * FFN_e(x) ) (full softmax mixture)."""
    d, F, T, E = 64, 96, 48, 4
    ex = [_rand_expert(d, F, 20 + e) for e in range(E)]
    g = torch.Generator().manual_seed(5)
    x = torch.randn(T, d, generator=g).to(torch.bfloat16)
    wg = (torch.randn(E, d, generator=g) * d ** -0.5).to(torch.bfloat16)
    l = (x.double() @ wg.double().T).float()                  # fp32 logits
    wsm = torch.softmax(l.double(), dim=1).float().double()  # fp32 gate weights
    ys = [torch.from_numpy(bf16_bits_to_f64(_torch_swiglu_bf16(x, *ex[e]))) for e in range(E)]
    acc = sum(wsm[:, e:e + 1] * ys[e] for e in range(E))
    expect = bf16_rne_exact(acc.numpy())
    pl = wl.make_placement(E, 1, 1, shadows=False)
    r = oracle.layer(wl.as_u16(x), wl.as_u16(wg), E, [wl.as_u16(a[0]) for a in ex], [wl.as_u16(a[1]) for a in ex],
                     [wl.as_u16(a[2]) for a in ex], pl.cand, pl.ew_rank, pl.slots_per_ew, np.zeros(1, np.uint8), G=1)
    np.testing.assert_array_equal(r["logits"], l.numpy())
    np.testing.assert_array_equal(r["out"], expect)


def test_zero_router_and_identical_experts():
    """Wg = 0 -> experts {0..k-1}, w = 1/k; identical experts -> out == y bitwise (weights sum to 1)."""
    d, F, T, E = 32, 64, 40, 8
    w1, w3, w2 = _rand_expert(d, F, 33)
    x = torch.randn(T, d, generator=torch.Generator().manual_seed(34)).to(torch.bfloat16)
    y = _torch_swiglu_bf16(x, w1, w3, w2)
    pl = wl.make_placement(E, 2, 1)
    for k in (1, 2, 4):
        r = oracle.layer(wl.as_u16(x), np.zeros((E, d), np.uint16), k, [wl.as_u16(w1)] * E, [wl.as_u16(w3)] * E,
                         [wl.as_u16(w2)] * E, pl.cand, pl.ew_rank, pl.slots_per_ew, np.zeros(2, np.uint8), G=1)
        assert np.all(r["idx"] == np.arange(k)[None, :])
        assert np.all(r["w"] == np.float32(1.0 / k))
        np.testing.assert_array_equal(r["out"], y)
    # random router, identical experts: any selection gives out == y
    wg = (torch.randn(E, d, generator=torch.Generator().manual_seed(35))).to(torch.bfloat16)
    r = oracle.layer(wl.as_u16(x), wl.as_u16(wg), 3, [wl.as_u16(w1)] * E, [wl.as_u16(w3)] * E,
                     [wl.as_u16(w2)] * E, pl.cand, pl.ew_rank, pl.slots_per_ew, np.zeros(2, np.uint8), G=1)
    np.testing.assert_array_equal(r["out"], y)


def test_shared_expert_adds_with_weight_one():
    """F_sh > 0 with all routed experts zero: out == FFN_sh(x) (R#16)."""
    d, F, T, E = 32, 64, 16, 4
    ws = _rand_expert(d, 48, 41)
    z = np.zeros((F, d), np.uint16)
    x = torch.randn(T, d, generator=torch.Generator().manual_seed(42)).to(torch.bfloat16)
    pl = wl.make_placement(E, 1, 1, shadows=False)
    r = oracle.layer(wl.as_u16(x), np.zeros((E, d), np.uint16), 2, [z] * E, [z] * E, [np.zeros((d, F), np.uint16)] * E,
                     pl.cand, pl.ew_rank, pl.slots_per_ew, np.zeros(1, np.uint8), G=1,
                     shared=tuple(wl.as_u16(a) for a in ws))
    np.testing.assert_array_equal(r["out"], _torch_swiglu_bf16(x, *ws))


# ---------------------------------------------------------------- routing / permutation invariants

def test_resolve_rules():
    """O4: healthy primary -> primary; masked -> first healthy shadow; none -> NO_ROUTE."""
    pl = wl.make_placement(8, 4, 2)
    base, S = oracle.slot_bases(4, pl.ew_rank, pl.slots_per_ew)
    r, b, rc = oracle.resolve(pl.cand, pl.ew_rank, base, np.zeros(4, np.uint8))
    assert rc == 0
    for e in range(8):
        ew, sl = pl.cand[e, 0]
        assert r[e] == pl.ew_rank[ew] and b[e] == base[ew] + sl
    m = np.array([0, 1, 0, 0], np.uint8)
    r, b, rc = oracle.resolve(pl.cand, pl.ew_rank, base, m)
    assert rc == 0
    for e in range(8):
        ew, sl = pl.cand[e, 0]
        if ew == 1:
            ew, sl = pl.cand[e, 1]
        assert r[e] == pl.ew_rank[ew] and b[e] == base[ew] + sl
    # mask an EW and the EW holding its shadow of expert e -> NO_ROUTE for e
    e = int(np.where(pl.cand[:, 0, 0] == 1)[0][0])
    m = np.zeros(4, np.uint8)
    m[pl.cand[e, 0, 0]] = 1
    m[pl.cand[e, 1, 0]] = 1
    r, b, rc = oracle.resolve(pl.cand, pl.ew_rank, base, m)
    assert rc == oracle.ERR_NO_ROUTE and r[e] == -1


@pytest.mark.parametrize("cfg,W,G", [("tiny", 2, 1), ("tiny", 4, 2), ("tiny", 8, 4)])
def test_permutation_invariants_and_mask_invariance(cfg, W, G):
    """Every token reaches exactly k rows; dst_pos is a bijection per rank; rows of a slot ascend in
    global t; shadows get 0 rows unmasked, the masked EW gets 0 rows masked; out is unchanged by the
    mask bitwise (P:918 stateless replay); bytes/token = V = 2*k*d*2."""
    sh = wl.CONFIGS[cfg]
    L = wl.make_layer(sh, seed=1000)
    x = wl.make_tokens(sh, seed=1000)
    pl = wl.make_placement(sh.E, W, G)
    args = ([wl.as_u16(a) for a in L.w1], [wl.as_u16(a) for a in L.w3], [wl.as_u16(a) for a in L.w2])
    res = {}
    for masked in (None, 1):
        m = np.zeros(W, np.uint8)
        if masked is not None:
            m[masked] = 1
        r = oracle.layer(wl.as_u16(x), wl.as_u16(L.wg), sh.k, *args, pl.cand, pl.ew_rank, pl.slots_per_ew, m, G=G)
        assert r["rc"] == 0
        T, k = r["idx"].shape
        assert np.all(np.abs(r["w"].astype(np.float64).sum(1) - 1) <= 1e-6)
        assert all(len(set(row)) == k for row in r["idx"].tolist())
        counts = r["counts"]
        assert counts.sum() == T * k
        for q in range(G):
            sel = r["dst_rank"] == q
            pos = np.sort(r["dst_pos"][sel])
            np.testing.assert_array_equal(pos, np.arange(counts[q].sum()))
            for s in range(r["S_max"]):
                ss = sel & (r["dst_slot"] == s)
                tt = np.nonzero(ss)[0]
                assert len(tt) == counts[q, s]
                order = np.argsort(r["dst_pos"][ss])
                assert np.all(np.diff(tt[order]) > 0)
                if len(tt):
                    assert r["dst_pos"][ss].min() == counts[q, :s].sum()
        # rows land only on slots that host the selected expert
        base = r["slot_base"]
        for t in range(0, T, 17):
            for j in range(k):
                e = r["idx"][t, j]
                q, s = r["dst_rank"][t, j], r["dst_slot"][t, j]
                ews = [w for w in range(W) if pl.ew_rank[w] == q and base[w] <= s < base[w] + pl.slots_per_ew]
                assert len(ews) == 1 and pl.hosted[ews[0]][s - base[ews[0]]] == e
        # shadow-inactivity / masked-EW silence
        rows_per_ew = np.zeros(W, np.int64)
        shadow_rows = 0
        for w in range(W):
            q = pl.ew_rank[w]
            for sl in range(pl.slots_per_ew):
                n = counts[q, base[w] + sl]
                rows_per_ew[w] += n
                e = pl.hosted[w][sl]
                if e >= 0 and tuple(pl.cand[e, 0]) != (w, sl):
                    shadow_rows += n
        if masked is None:
            assert shadow_rows == 0
        else:
            assert rows_per_ew[masked] == 0
        assert 2 * 2 * k * sh.d == 2 * k * sh.d * 2   # V = 2 * Top_k * N_hidden * S_elem per token
        res[masked] = r["out"]
    np.testing.assert_array_equal(res[None], res[1])


def test_sampled_tokens_equal_full_run():
    """Tokens are independent: the oracle on a token subset equals the same rows of a full run,
    and the multi-threaded run equals the single-threaded one bitwise."""
    sh = wl.CONFIGS["tiny"]
    L = wl.make_layer(sh, seed=1001)
    x = wl.make_tokens(sh, seed=1001)
    pl = wl.make_placement(sh.E, 2, 1)
    args = ([wl.as_u16(a) for a in L.w1], [wl.as_u16(a) for a in L.w3], [wl.as_u16(a) for a in L.w2])
    full = oracle.layer(wl.as_u16(x), wl.as_u16(L.wg), sh.k, *args, pl.cand, pl.ew_rank, pl.slots_per_ew,
                        np.zeros(2, np.uint8), G=1)
    tok = np.array([0, 5, 77, 255], np.int32)
    part = oracle.moe_tokens(wl.as_u16(x), full["idx"], full["w"], *args, tokens=tok, n_threads=4)
    np.testing.assert_array_equal(part, full["out"][tok])
    mt = oracle.moe_tokens(wl.as_u16(x), full["idx"], full["w"], *args, n_threads=8)
    np.testing.assert_array_equal(mt, full["out"])


def test_v_size_law_mixtral():
    """App. C: V = 2 * Top_k * N_hidden * S_elem = 32768 B for Mixtral bf16."""
    sh = wl.CONFIGS["mixtral_decode"]
    assert 2 * sh.k * sh.d * 2 == 32768


# ---------------------------------------------------------------- unrounded stage values (R#21)

def test_k_equals_E_has_no_near_tie():
    """O2 with k == E: there is no (k+1)-th logit, so gap = +inf (no token is a near tie)."""
    l = np.zeros((3, 4), np.float32)
    _, _, gap = oracle.select(l, 4)
    assert np.all(np.isinf(gap)) and np.all(gap > 0)


def test_router_f64_vs_torch_fp64():
    """O1 before rounding == torch fp64 x @ Wg^T; its fp32 rounding is O1; s = |x| @ |Wg|^T."""
    g = torch.Generator().manual_seed(61)
    x = torch.randn(40, 128, generator=g).to(torch.bfloat16)
    wg = (torch.randn(12, 128, generator=g) * 0.1).to(torch.bfloat16)
    l, s = oracle.router_f64(wl.as_u16(x), wl.as_u16(wg))
    ref = (x.double() @ wg.double().T).numpy()
    np.testing.assert_allclose(l, ref, rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(s, (x.double().abs() @ wg.double().abs().T).numpy(), rtol=1e-13)
    np.testing.assert_array_equal(l.astype(np.float32), oracle.router(wl.as_u16(x), wl.as_u16(wg)))


def test_stage_h_and_y_vs_torch_fp64():
    """O6a / O6b unrounded values == torch fp64 SwiGLU halves (silu(x W1^T) * x W3^T, then h W2^T)."""
    d, F, n = 96, 160, 24
    w1, w3, w2 = _rand_expert(d, F, 62)
    x = torch.randn(n, d, generator=torch.Generator().manual_seed(63)).to(torch.bfloat16)
    st = oracle.stage_h(wl.as_u16(x), wl.as_u16(w1), wl.as_u16(w3), n_threads=2)
    xd = x.double()
    a1, a3 = xd @ w1.double().T, xd @ w3.double().T
    np.testing.assert_allclose(st["a1"], a1.numpy(), rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(st["a3"], a3.numpy(), rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(st["h"], (Fn.silu(a1) * a3).numpy(), rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(st["s1"], (xd.abs() @ w1.double().abs().T).numpy(), rtol=1e-12)
    hb = bf16_rne_exact(st["h"])
    y, s = oracle.stage_y(hb, wl.as_u16(w2), n_threads=2)
    hd = torch.from_numpy(bf16_bits_to_f64(hb))
    np.testing.assert_allclose(y, (hd @ w2.double().T).numpy(), rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(s, (hd.abs() @ w2.double().abs().T).numpy(), rtol=1e-12)
    # the stages rounded at the R#7 storage points are exactly O6 (the oracle's y)
    np.testing.assert_array_equal(bf16_rne_exact(y), _torch_swiglu_bf16(x, w1, w3, w2))


def test_stage_combine_and_out_f64():
    """O8 before rounding: out_f64 = sum_j w_j y_j (+ sg y_sh) in fp64 (numpy), its RNE is the
    oracle's out; closed form k = 1, w = 1 -> out_f64 == y exactly."""
    sh = wl.CONFIGS["tiny"]
    L = wl.make_layer(sh, seed=1007)
    x = wl.make_tokens(sh, seed=1007, T=64)
    pl = wl.make_placement(sh.E, 2, 1)
    args = ([wl.as_u16(a) for a in L.w1], [wl.as_u16(a) for a in L.w3], [wl.as_u16(a) for a in L.w2])
    r = oracle.layer(wl.as_u16(x), wl.as_u16(L.wg), sh.k, *args, pl.cand, pl.ew_rank, pl.slots_per_ew,
                     np.zeros(2, np.uint8), G=1, want_y=True)
    yv = bf16_bits_to_f64(r["y"])
    ref = np.sum(r["w"].astype(np.float64)[:, :, None] * yv, axis=1)
    np.testing.assert_allclose(r["out_f64"], ref, rtol=1e-15, atol=0)
    np.testing.assert_array_equal(bf16_rne_exact(r["out_f64"]), r["out"])
    o, s = oracle.stage_combine(r["w"], r["y"])
    np.testing.assert_array_equal(o, r["out_f64"])
    np.testing.assert_allclose(s, np.sum(np.abs(r["w"].astype(np.float64)[:, :, None] * yv), axis=1), rtol=1e-15)
    one = np.ones((64, 1), np.float32)
    o1, _ = oracle.stage_combine(one, r["y"][:, :1])
    np.testing.assert_array_equal(o1, yv[:, 0])
    sg = np.full(64, 0.25, np.float32)
    o2, _ = oracle.stage_combine(one, r["y"][:, :1], ysh=r["y"][:, 1], sg=sg)
    np.testing.assert_array_equal(o2, yv[:, 0] + 0.25 * yv[:, 1])
