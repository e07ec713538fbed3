"""GPU-vs-oracle parity (test infrastructure): criteria P1-P4 of SURVEY.md 8(c),
checked per storage point (R#21).

Every bf16 value the GPU path stores — h (SwiGLU activations), y (expert
outputs, in the source AW's combine buffer), y_sh, out — is checked against
the EXACT value (oracle, fp64) of the function the paper defines for that
stage, computed from the GPU's OWN inputs to that stage (the token rows it
received, the h it stored, the w and y the combine read).  The GPU value must
be a bf16 round-to-nearest-even of some real number within the fp32
accumulation bound B of the exact value:

    bf16(v_exact - B) <= v_gpu <= bf16(v_exact + B)          (every element)

B is derived from the arithmetic (R#24): a K-long bf16 dot product
accumulated in fp32 on tensor cores (one rounding per 16-wide MMA step, plus
the fixed-order split-K / warp-partial adds) has |err| <= (K/16 + 16 + adds) *
2^-22 * sum|terms|; the SwiGLU epilogue adds the propagation of those bounds
through silu(a1) * a3 (|silu'| <= 1.1) and a few ulps of expf / division /
multiply; the combine's fma chain has |err| <= (k + 2) * 2^-24 * sum|terms|.
No element is exempt and nothing is counted-and-passed.  The end-to-end error
against the oracle's own fp64 chain (north_star: max|err| <= 2e-2 * RMS) is
reported, with the number of elements beyond it: each of those is explained
by the per-stage checks above (different but correct roundings at some bf16
storage point upstream).

Routing: the oracle's top-k + softmax (O2/O3) applied to the GPU's OWN fp32
logits reproduces the GPU's idx bit-exactly for every token and its w within
(n + 6) ulps; P1 idx bit-exact vs the oracle's own routing except near ties
(oracle gap < 1e-5), and near-tie selections valid within 1e-5 of the exact
logits; P2 permutation bit-exact
when there is no near tie, and CONDITIONAL P2 always (the oracle's O4-O5
applied to the GPU's own idx must reproduce every dst_rank/slot/pos and the
counts bit-exactly, no exemption); P3 |dw| <= 1e-6 or the propagation of the
measured logit error (2 w max|dl|), whichever is larger; router logits within
5e-6 of the exact fp64 logits (so the near-tie exemption of 1e-5 covers every
GPU-vs-oracle selection difference) and within their accumulation bound.
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional

import numpy as np
import torch

import oracle
import workloads as wl

NEAR_TIE = 1e-5       # north_star: k-th vs (k+1)-th logit gap below which routing may differ
W_TOL = 1e-6          # |w_gpu - w_oracle|
OUT_TOL = 2e-2        # north_star: max|out_gpu - out_oracle| <= OUT_TOL * RMS(out_oracle) (reported)
LOGIT_TOL = 5e-6      # half the near-tie gap: GPU-vs-oracle selection differences only at near ties
U = 2.0 ** -24        # fp32 unit roundoff


def bf16_to_f64(u16: np.ndarray) -> np.ndarray:
    return (np.ascontiguousarray(u16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def dot_bound(S: np.ndarray, K: int, adds: int = 0) -> np.ndarray:
    """DESIGN.md R#24: fp32 tensor-core accumulation of a K-long dot product (16-wide MMA steps)
    plus `adds` fixed-order fp32 additions of partials: |err| <= (K/16 + 16 + adds) * 2^-22 * S."""
    return (K / 16.0 + 16.0 + adds) * 4.0 * U * S


def h_bound(a1, a3, s1, s3, d):
    """R#24 / R#26: bound on |h_fp32 - h_exact| for h = silu(a1) * a3 with a1, a3 accumulated in
    fp32 (propagated through |silu'| <= 1.1) and silu evaluated with the fast exp / divide
    (relative error <= (5 + 1.2 |a1|) ulp; + the final multiply): (8 + 1.5 |a1|) ulps here."""
    B1, B3 = dot_bound(s1, d), dot_bound(s3, d)
    sil = a1 / (1.0 + np.exp(-a1))
    prop = 1.1 * B1 * (np.abs(a3) + B3) + np.abs(sil) * B3
    return prop + (8.0 + 1.5 * (np.abs(a1) + B1)) * U * (np.abs(sil * a3) + prop)


def bracket(v_exact: np.ndarray, B: np.ndarray, gpu_u16: np.ndarray):
    """Mask of elements where gpu is a bf16 RNE of a value in [v - B, v + B]; and the used fraction."""
    lo = bf16_to_f64(oracle.bf16_from_f64(v_exact - B))
    hi = bf16_to_f64(oracle.bf16_from_f64(v_exact + B))
    g = bf16_to_f64(gpu_u16)
    ok = (g >= lo) & (g <= hi)
    # how much of the allowance was used: |g - v| against B + half a bf16 step of v
    half = np.exp2(np.floor(np.log2(np.maximum(np.abs(v_exact), 2.0 ** -126))) - 8)
    used = np.abs(g - v_exact) / (B + half)
    return ok, float(used.max()) if used.size else 0.0


def host_weights(L: wl.Layer):
    w1 = [wl.as_u16(a) for a in L.w1]
    w3 = [wl.as_u16(a) for a in L.w3]
    w2 = [wl.as_u16(a) for a in L.w2]
    sh = tuple(wl.as_u16(a) for a in L.shared) if L.shared is not None else None
    return w1, w3, w2, sh


def oracle_layer(L: wl.Layer, x: torch.Tensor, pl: wl.Placement, mask, G: int, tokens=None, n_threads=1,
                 want_y=True):
    w1, w3, w2, sh = host_weights(L)
    wsg = wl.as_u16(L.wsg) if L.wsg is not None else None
    return oracle.layer(wl.as_u16(x), wl.as_u16(L.wg), L.shape.k, w1, w3, w2, pl.cand, pl.ew_rank,
                        pl.slots_per_ew, np.asarray(mask, np.uint8), G, shared=sh, tokens=tokens,
                        n_threads=n_threads, gate_mode=L.shape.gate_mode, wsg=wsg, want_y=want_y)


@dataclasses.dataclass
class RankView:
    """What one rank's ctx exported after a call (host numpy arrays)."""
    rank: int
    t0: int                       # global index of the rank's first token
    out: np.ndarray               # u16 [T_r, d]
    routing: dict                 # idx, w, dst_rank, dst_slot, dst_pos [T_r, k]; counts [G, S_max]
    logits: Optional[np.ndarray]  # f32 [T_r, E(+1)]
    recv: np.ndarray              # u16 [R, d]
    meta: np.ndarray              # i32 [R, 2]
    H: np.ndarray                 # u16 [R, F]
    Y: np.ndarray                 # u16 [T_r, k, d]
    Hs: Optional[np.ndarray]      # u16 [T_r, F_sh]
    ysh: Optional[np.ndarray]     # u16 [T_r, d]
    sgate: Optional[np.ndarray]   # f32 [T_r]


def collect(layer, out: torch.Tensor, t0: int = 0) -> RankView:
    """Export the last call's routing and stage values of `layer` (device synchronised)."""
    import paper_2601_01310_b200 as tg
    sh = layer.shape
    T = out.shape[0]
    rt = {k: v.cpu().numpy() for k, v in layer.routing(T).items()}
    d, k, F = sh.d, sh.k, sh.F
    lg = layer.stage(tg.TG_STAGE_LOGITS) if getattr(layer, "stage_export", False) else None
    recv = layer.stage(tg.TG_STAGE_RECV)
    R = recv.size // d
    Hs = layer.stage(tg.TG_STAGE_HSH) if sh.F_sh else None
    ysh = layer.stage(tg.TG_STAGE_YSH) if sh.F_sh else None
    sg = layer.stage(tg.TG_STAGE_SGATE) if getattr(sh, "shared_gate", 0) else None
    return RankView(rank=layer.rank, t0=t0, out=wl.as_u16(out), routing=rt,
                    logits=None if lg is None else lg.reshape(T, -1),
                    recv=recv.reshape(R, d), meta=layer.stage(tg.TG_STAGE_META).reshape(R, 2),
                    H=layer.stage(tg.TG_STAGE_H).reshape(R, F), Y=layer.stage(tg.TG_STAGE_Y).reshape(T, k, d),
                    Hs=None if Hs is None else Hs.reshape(T, sh.F_sh), ysh=None if ysh is None else ysh.reshape(T, d),
                    sgate=sg)


def _cat(views, key):
    return np.concatenate([v.routing[key] for v in views])


def check(views: List[RankView], L: wl.Layer, x: torch.Tensor, pl: wl.Placement, mask, tokens=None,
          n_threads=1, nsplit=None, ref=None):
    """All parity criteria for one call of every rank (views in rank order, tokens = global
    sample for the FFN/combine checks; None = all).  Returns a report; asserts on failure."""
    sh = L.shape
    G = len(views)
    d, k, F, E = sh.d, sh.k, sh.F, sh.E
    xu = wl.as_u16(x)
    T = xu.shape[0]
    if ref is None:
        ref = oracle_layer(L, x, pl, mask, G=G, tokens=tokens, n_threads=n_threads)
    rep = {}
    idx_g, w_g = _cat(views, "idx"), _cat(views, "w")
    near = ref["gap"] < NEAR_TIE
    rep["near_ties"] = int(near.sum())
    nterm = k if sh.gate_mode == 0 else E  # exponentials summed by the softmax (O3 / O3')
    max_dl = LOGIT_TOL
    # ---- router logits (O1) against the exact fp64 logits
    if all(v.logits is not None for v in views):
        lg32 = np.ascontiguousarray(np.concatenate([v.logits for v in views])[:, :E])
        lg = lg32.astype(np.float64)
        l_ex, l_s = oracle.router_f64(xu, wl.as_u16(L.wg))
        dl = np.abs(lg - l_ex)
        rep["max_dlogit"] = max_dl = float(dl.max()) if dl.size else 0.0
        assert rep["max_dlogit"] <= LOGIT_TOL, f"router: max |dlogit| {rep['max_dlogit']:.3g} > {LOGIT_TOL}"
        assert np.all(dl <= dot_bound(l_s, d, adds=64) + U * np.abs(l_ex)), "router: logit beyond its bound"
        # ---- top-k + softmax stage (O2/O3) on the GPU's OWN logits: the selection must be
        # bit-exact for every token (no near-tie exemption: same logits, same ties) and w within
        # the fp32 evaluation bound of expf / sum / division ((nterm + 6) ulps, R#24)
        if T:
            idx_s, w_s, _ = oracle.select(lg32, k, sh.gate_mode)
            bad_s = np.any(_cat(views, "idx") != idx_s, axis=1)
            assert not bad_s.any(), f"top-k on the GPU's own logits differs at tokens {np.nonzero(bad_s)[0][:5]}"
            dws = np.abs(_cat(views, "w").astype(np.float64) - w_s.astype(np.float64))
            assert np.all(dws <= (nterm + 6) * U * w_s + 2.0 ** -149), f"softmax stage: max |dw| {dws.max():.3g}"
            rep["max_dw_stage_ulps"] = float((dws / np.maximum(w_s, 1e-30)).max() / U) if dws.size else 0.0
    # ---- P1 selection
    bad = np.any(idx_g != ref["idx"], axis=1)
    assert not (bad & ~near).any(), \
        f"P1: idx mismatch on {int((bad & ~near).sum())} non-near-tie tokens, first {np.nonzero(bad & ~near)[0][:5]}"
    rep["near_tie_flips"] = int((bad & near).sum())
    if (bad & near).any():  # several selections are correct within 1e-5: the GPU's must be one of them
        lgx = oracle.router(xu, wl.as_u16(L.wg)).astype(np.float64)
        for t in np.nonzero(bad & near)[0]:
            sel = np.zeros(E, bool)
            sel[idx_g[t]] = True
            assert lgx[t, sel].min() >= lgx[t, ~sel].max() - NEAR_TIE, f"P1: invalid near-tie selection at {t}"
    # ---- P3 gate weights against the oracle's (from ITS logits): 1e-6, or what the measured logit
    # error propagates to (|dw_j| <= 2 w_j max|dl| through the softmax, + its evaluation ulps) when
    # larger (skewed routing: |l| ~ 16, a few ulps of logit exceed 1e-6 of w; R#25)
    same = ~bad
    wr = ref["w"].astype(np.float64)
    dw = np.abs(w_g.astype(np.float64) - wr)
    tol_w = np.maximum(W_TOL, 2.0 * max_dl * wr + (nterm + 7) * U * wr)
    rep["max_dw"] = float(dw[same].max()) if same.any() else 0.0
    assert np.all((dw <= tol_w)[same]), f"P3: max |dw| = {rep['max_dw']}"
    # ---- P2 permutation: unconditional without near ties, conditional (GPU idx) always
    counts_g = views[0].routing["counts"]
    perm_g = {kk: _cat(views, kk) for kk in ("dst_rank", "dst_slot", "dst_pos")}
    if rep["near_ties"] == 0:
        for kk in perm_g:
            assert np.array_equal(perm_g[kk], ref[kk]), f"P2: {kk} mismatch at {np.argwhere(perm_g[kk] != ref[kk])[:5]}"
        assert np.array_equal(counts_g, ref["counts"]), "P2: counts mismatch"
    dr, ds, dp, cnt = oracle.permute(idx_g, ref["rank_e"], ref["bank_e"], G, ref["S_max"])
    for kk, o in (("dst_rank", dr), ("dst_slot", ds), ("dst_pos", dp)):
        assert np.array_equal(perm_g[kk], o), f"conditional P2: {kk} mismatch at {np.argwhere(perm_g[kk] != o)[:5]}"
    assert np.array_equal(counts_g, cnt), "conditional P2: counts mismatch"
    for v in views[1:]:
        assert np.array_equal(v.routing["counts"], counts_g), "counts differ between ranks"
    # ---- per-storage-point checks on the sampled tokens
    tok = np.arange(T) if tokens is None else np.asarray(tokens)
    rank_of = np.zeros(T, np.int64)
    for v in views:
        rank_of[v.t0:v.t0 + v.out.shape[0]] = v.rank
    w1, w3, w2, shw = host_weights(L)
    pairs = {}  # expert -> list of (t, j, q, pos)
    for t in tok:
        r = rank_of[t]
        tl = t - views[r].t0
        for j in range(k):
            e, q, pos = int(idx_g[t, j]), int(perm_g["dst_rank"][t, j]), int(perm_g["dst_pos"][t, j])
            V = views[q]
            assert np.array_equal(V.recv[pos], xu[t]), f"dispatch: recv row {pos} on rank {q} is not x[{t}]"
            assert tuple(V.meta[pos]) == (r, tl * k + j), f"dispatch: origin of row {pos} on rank {q}"
            pairs.setdefault(e, []).append((t, j, q, pos))
    # fixed-order split-K adds of GEMM2 (the library's rule: 2 splits when F / 64 >= 128 and even)
    nsplit = nsplit if nsplit is not None else (2 if (F // 64 >= 128 and (F // 64) % 2 == 0) else 1)
    n_h = n_y = 0
    use_h = use_y = 0.0
    for e, lst in pairs.items():
        ts = np.array([p[0] for p in lst])
        Hg = np.stack([views[p[2]].H[p[3]] for p in lst])
        st = oracle.stage_h(xu[ts], w1[e], w3[e], n_threads=n_threads)
        ok, used = bracket(st["h"], h_bound(st["a1"], st["a3"], st["s1"], st["s3"], d), Hg)
        assert ok.all(), f"h (O6a) of expert {e}: {int((~ok).sum())} of {ok.size} values outside the bound"
        n_h += ok.size
        use_h = max(use_h, used)
        yx, ys = oracle.stage_y(Hg, w2[e], n_threads=n_threads)
        Yg = np.stack([views[rank_of[p[0]]].Y[p[0] - views[rank_of[p[0]]].t0, p[1]] for p in lst])
        ok, used = bracket(yx, dot_bound(ys, F, adds=nsplit), Yg)
        assert ok.all(), f"y (O6b) of expert {e}: {int((~ok).sum())} of {ok.size} values outside the bound"
        n_y += ok.size
        use_y = max(use_y, used)
    rep.update(h_checked=n_h, y_checked=n_y, h_bound_used=use_h, y_bound_used=use_y)
    tl_of = tok - np.array([views[rank_of[t]].t0 for t in tok])
    ysh_g = sg_g = None
    if sh.F_sh:
        Hs_g = np.stack([views[rank_of[t]].Hs[tl] for t, tl in zip(tok, tl_of)])
        st = oracle.stage_h(xu[tok], shw[0], shw[1], n_threads=n_threads)
        ok, used = bracket(st["h"], h_bound(st["a1"], st["a3"], st["s1"], st["s3"], d), Hs_g)
        assert ok.all(), f"h_sh (O7): {int((~ok).sum())} values outside the bound"
        ysh_g = np.stack([views[rank_of[t]].ysh[tl] for t, tl in zip(tok, tl_of)])
        yx, ys = oracle.stage_y(Hs_g, shw[2], n_threads=n_threads)
        ok, used2 = bracket(yx, dot_bound(ys, sh.F_sh), ysh_g)
        assert ok.all(), f"y_sh (O7): {int((~ok).sum())} values outside the bound"
        rep["shared_bound_used"] = max(used, used2)
        if getattr(sh, "shared_gate", 0):
            sg_g = np.stack([views[rank_of[t]].sgate[tl] for t, tl in zip(tok, tl_of)])
            dsg = np.abs(sg_g.astype(np.float64) - ref["sgate"][tok].astype(np.float64))
            rep["max_dsgate"] = float(dsg.max())
            assert rep["max_dsgate"] <= W_TOL, f"O7': max |d sgate| = {rep['max_dsgate']}"
    Yt = np.stack([views[rank_of[t]].Y[tl] for t, tl in zip(tok, tl_of)])
    out_g = np.stack([views[rank_of[t]].out[tl] for t, tl in zip(tok, tl_of)])
    ox, os_ = oracle.stage_combine(w_g[tok], Yt, ysh_g, sg_g)
    ok, used = bracket(ox, (k + 2) * U * os_, out_g)
    assert ok.all(), f"out (O8): {int((~ok).sum())} of {ok.size} values outside the bound"
    rep["out_checked"] = int(ok.size)
    rep["out_bound_used"] = used
    # ---- end to end against the oracle's own chain (north_star tolerance, reported)
    out_ref = bf16_to_f64(ref["out"])
    sel = ~near[tok]
    err = np.abs(bf16_to_f64(out_g) - out_ref)[sel]
    rms = float(np.sqrt(np.mean(out_ref[sel] ** 2))) if sel.any() else 1.0
    rep["rms"] = rms
    rep["max_err_over_rms"] = float(err.max()) / rms if err.size else 0.0
    rep["mean_err_over_rms"] = float(err.mean()) / rms if err.size else 0.0
    rep["n_compared"] = int(err.size)
    rep["n_bit_diff"] = int((err > 0).sum())
    rep["n_over_tol_explained"] = int((err > OUT_TOL * rms).sum())
    return rep


def single(layer, out: torch.Tensor, L, x, pl, mask, tokens=None, n_threads=1, ref=None):
    """check() for a one-rank layer."""
    return check([collect(layer, out)], L, x, pl, mask, tokens=tokens, n_threads=n_threads, ref=ref)
