"""ctypes wrapper for the CPU oracle (oracle/tg_oracle.c).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module.  The product path (``paper_2601_01310_b200``) never imports it and the
oracle never imports the product: they share no code.

Each wrapper names the oracle step it calls (O1..O8, see tg_oracle.c and
DESIGN.md §3); the arithmetic lives in C, this file only marshals arrays.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tg_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OK, ERR_INVALID, ERR_NO_ROUTE = 0, -1, -2

_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle (plain gcc, no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
                               "-fPIC", "-shared", "-Wall", "-o", _LIB, _SRC, "-lm"])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i32, i64 = ctypes.c_int, ctypes.c_int64
        L.orc_bf16_from_f64.argtypes = [ctypes.c_double]
        L.orc_bf16_from_f64.restype = ctypes.c_uint16
        L.orc_bf16_from_f64_array.argtypes = [P, P, i64]
        L.orc_bf16_from_f32_array.argtypes = [P, P, i64]
        L.orc_router.argtypes = [P, P, i32, i32, i32, P]
        L.orc_select.argtypes = [P, i32, i32, i32, P, P, P]
        L.orc_select.restype = i32
        L.orc_resolve.argtypes = [i32, i32, P, P, P, P, P, P]
        L.orc_resolve.restype = i32
        L.orc_permute.argtypes = [i32, i32, P, P, P, i32, i32, P, P, P, P]
        L.orc_permute.restype = i32
        L.orc_moe_tokens.argtypes = [i32, i32, i32, i32, i32, P, P, P, P, P, P, P, P, P, P, i32, P, P, i32]
        L.orc_moe_tokens.restype = i32
        L.orc_select_mode.argtypes = [P, i32, i32, i32, i32, P, P, P]
        L.orc_select_mode.restype = i32
        L.orc_shared_gate.argtypes = [P, P, i32, i32, P]
        L.orc_moe_tokens2.argtypes = [i32, i32, i32, i32, i32, P, P, P, P, P, P, P, P, P, P, P, i32, P, P, i32, P]
        L.orc_moe_tokens2.restype = i32
        L.orc_moe_tokens3.argtypes = [i32, i32, i32, i32, i32, P, P, P, P, P, P, P, P, P, P, P, i32, P, P, i32, P, P]
        L.orc_moe_tokens3.restype = i32
        L.orc_router_f64.argtypes = [P, P, i32, i32, i32, P, P]
        L.orc_stage_h.argtypes = [P, i32, i32, i32, P, P, P, P, P, P, P, i32]
        L.orc_stage_y.argtypes = [P, i32, i32, i32, P, P, P, i32]
        L.orc_stage_combine.argtypes = [i32, i32, i32, P, P, P, P, P, P]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"], "oracle inputs must be C-contiguous"
    return a.ctypes.data_as(ctypes.c_void_p)


def _u16(a) -> np.ndarray:
    a = np.ascontiguousarray(a)
    if a.dtype != np.uint16:
        a = a.view(np.uint16) if a.dtype.itemsize == 2 else a.astype(np.uint16)
    return a


def bf16_from_f64(v: np.ndarray) -> np.ndarray:
    v = np.ascontiguousarray(v, dtype=np.float64)
    out = np.empty(v.shape, np.uint16)
    lib().orc_bf16_from_f64_array(_p(v), _p(out), v.size)
    return out


def bf16_from_f32(v: np.ndarray) -> np.ndarray:
    v = np.ascontiguousarray(v, dtype=np.float32)
    out = np.empty(v.shape, np.uint16)
    lib().orc_bf16_from_f32_array(_p(v), _p(out), v.size)
    return out


def router(x: np.ndarray, wg: np.ndarray) -> np.ndarray:
    """O1: fp32 logits [T, E] from bf16 x [T, d] and Wg [E, d]."""
    x, wg = _u16(x), _u16(wg)
    T, d = x.shape
    E = wg.shape[0]
    out = np.empty((T, E), np.float32)
    lib().orc_router(_p(x), _p(wg), T, d, E, _p(out))
    return out


def router_f64(x: np.ndarray, wg: np.ndarray):
    """O1 before the fp32 rounding: (l_exact fp64 [T, E], sum of |x Wg| fp64 [T, E])."""
    x, wg = _u16(x), _u16(wg)
    T, d = x.shape
    E = wg.shape[0]
    l = np.empty((T, E), np.float64)
    s = np.empty((T, E), np.float64)
    lib().orc_router_f64(_p(x), _p(wg), T, d, E, _p(l), _p(s))
    return l, s


def stage_h(rows_x, w1, w3, n_threads=1):
    """O6a on rows sharing one expert: dict(h, a1, a3, s1, s3), fp64 [n, F]; h = silu(a1) * a3 unrounded."""
    rows_x, w1, w3 = _u16(rows_x), _u16(w1), _u16(w3)
    n, d = rows_x.shape
    F = w1.shape[0]
    out = {k: np.empty((n, F), np.float64) for k in ("h", "a1", "a3", "s1", "s3")}
    lib().orc_stage_h(_p(rows_x), n, d, F, _p(w1), _p(w3), *(_p(out[k]) for k in ("h", "a1", "a3", "s1", "s3")),
                      int(n_threads))
    return out


def stage_y(rows_h, w2, n_threads=1):
    """O6b on stored bf16 h rows sharing one expert: (y_exact fp64 [n, d], sum |h W2| fp64 [n, d])."""
    rows_h, w2 = _u16(rows_h), _u16(w2)
    n, F = rows_h.shape
    d = w2.shape[0]
    y = np.empty((n, d), np.float64)
    s = np.empty((n, d), np.float64)
    lib().orc_stage_y(_p(rows_h), n, d, F, _p(w2), _p(y), _p(s), int(n_threads))
    return y, s


def stage_combine(w, y, ysh=None, sg=None):
    """O8 before the bf16 rounding: w fp32 [n, k], y bf16 [n, k, d], ysh bf16 [n, d] | None,
    sg fp32 [n] | None -> (out_exact fp64 [n, d], sum of |terms| fp64 [n, d])."""
    w = np.ascontiguousarray(w, dtype=np.float32)
    y = _u16(y)
    n, k, d = y.shape
    ysh = _u16(ysh) if ysh is not None else None
    sg = np.ascontiguousarray(sg, dtype=np.float32) if sg is not None else None
    out = np.empty((n, d), np.float64)
    s = np.empty((n, d), np.float64)
    lib().orc_stage_combine(n, d, k, _p(w), _p(y), _p(ysh) if ysh is not None else None,
                            _p(sg) if sg is not None else None, _p(out), _p(s))
    return out, s


def select(logits: np.ndarray, k: int, gate_mode: int = 0):
    """O2/O3 (gate_mode 0) or O2/O3' (gate_mode 1: softmax over all E, no renormalisation):
    (idx int32 [T,k] ascending id, w fp32 [T,k], gap fp32 [T])."""
    logits = np.ascontiguousarray(logits, dtype=np.float32)
    T, E = logits.shape
    idx = np.empty((T, k), np.int32)
    w = np.empty((T, k), np.float32)
    gap = np.empty((T,), np.float32)
    rc = lib().orc_select_mode(_p(logits), T, E, k, int(gate_mode), _p(idx), _p(w), _p(gap))
    if rc != OK:
        raise ValueError(f"orc_select rc={rc}")
    return idx, w, gap


def resolve(cand: np.ndarray, ew_rank, ew_slot_base, mask):
    """O4: (rank_e, bank_e, rc).  cand int32 [E, C, 2] = (ew, slot), -1 pad."""
    cand = np.ascontiguousarray(cand, dtype=np.int32)
    E, C, _ = cand.shape
    ew_rank = np.ascontiguousarray(ew_rank, dtype=np.int32)
    ew_slot_base = np.ascontiguousarray(ew_slot_base, dtype=np.int32)
    mask = np.ascontiguousarray(mask, dtype=np.uint8)
    assert mask.size == ew_rank.size, "mask needs one entry per EW"
    rank_e = np.empty(E, np.int32)
    bank_e = np.empty(E, np.int32)
    rc = lib().orc_resolve(E, C, _p(cand), _p(ew_rank), _p(ew_slot_base), _p(mask), _p(rank_e), _p(bank_e))
    return rank_e, bank_e, rc


def permute(idx: np.ndarray, rank_e, bank_e, G: int, S_max: int):
    """O5: (dst_rank, dst_slot, dst_pos int32 [T,k], counts int32 [G, S_max])."""
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    T, k = idx.shape
    rank_e = np.ascontiguousarray(rank_e, dtype=np.int32)
    bank_e = np.ascontiguousarray(bank_e, dtype=np.int32)
    dr = np.empty((T, k), np.int32)
    ds = np.empty((T, k), np.int32)
    dp = np.empty((T, k), np.int32)
    counts = np.empty((G, S_max), np.int32)
    rc = lib().orc_permute(T, k, _p(idx), _p(rank_e), _p(bank_e), G, S_max, _p(dr), _p(ds), _p(dp), _p(counts))
    if rc != OK:
        raise ValueError(f"orc_permute rc={rc}")
    return dr, ds, dp, counts


def shared_gate(x, wsg) -> np.ndarray:
    """O7': per-token sigmoid weight of the shared expert, fp32 [T]."""
    x = _u16(x)
    wsg = _u16(np.ascontiguousarray(wsg).reshape(-1))
    T, d = x.shape
    out = np.empty(T, np.float32)
    lib().orc_shared_gate(_p(x), _p(wsg), T, d, _p(out))
    return out


def moe_tokens(x, idx, w, w1, w3, w2, shared=None, tokens=None, want_y=False, n_threads=1, sgate=None,
               want_f64=False):
    """O6-O8 for the given tokens (all if None).  want_f64: also out before its bf16 rounding.

    w1/w3/w2: sequences of E bf16 arrays (W1, W3: [F, d]; W2: [d, F]).
    shared: optional (W1s, W3s, W2s) of the merged shared expert.
    Returns out bf16 [n, d] (uint16) and, if want_y, (y bf16 [n, k, d], y_sh bf16 [n, d] or None).
    """
    x = _u16(x)
    T, d = x.shape
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    w = np.ascontiguousarray(w, dtype=np.float32)
    k = idx.shape[1]
    E = len(w1)
    w1 = [_u16(a) for a in w1]
    w3 = [_u16(a) for a in w3]
    w2 = [_u16(a) for a in w2]
    F = w1[0].shape[0]
    PtrArr = ctypes.c_void_p * E
    p1 = PtrArr(*[a.ctypes.data for a in w1])
    p3 = PtrArr(*[a.ctypes.data for a in w3])
    p2 = PtrArr(*[a.ctypes.data for a in w2])
    if shared is not None:
        s1, s3, s2 = (_u16(a) for a in shared)
        F_sh = s1.shape[0]
        ps = (_p(s1), _p(s3), _p(s2))
    else:
        F_sh = 0
        ps = (None, None, None)
    if tokens is None:
        tok = None
        n = T
    else:
        tok = np.ascontiguousarray(tokens, dtype=np.int32)
        n = tok.size
    out = np.empty((n, d), np.uint16)
    y = np.empty((n, k, d), np.uint16) if want_y else None
    ysh = np.empty((n, d), np.uint16) if (want_y and shared is not None) else None
    sg = None if sgate is None else np.ascontiguousarray(sgate, dtype=np.float32)
    of = np.empty((n, d), np.float64) if want_f64 else None
    rc = lib().orc_moe_tokens3(d, E, k, F, F_sh, _p(x), _p(idx), _p(w),
                               ctypes.cast(p1, ctypes.c_void_p), ctypes.cast(p3, ctypes.c_void_p),
                               ctypes.cast(p2, ctypes.c_void_p), ps[0], ps[1], ps[2],
                               _p(sg) if sg is not None else None,
                               _p(tok) if tok is not None else None, n, _p(out),
                               _p(y) if y is not None else None, int(n_threads),
                               _p(ysh) if ysh is not None else None,
                               _p(of) if of is not None else None)
    if rc != OK:
        raise ValueError(f"orc_moe_tokens rc={rc}")
    res = (out, (y, ysh)) if want_y else out
    return (res, of) if want_f64 else res


def slot_bases(n_ews: int, ew_rank, slots_per_ew: int):
    """EWs on a rank get consecutive bank-slot ranges in ew order (R#11)."""
    ew_rank = list(ew_rank)
    base = []
    used = {}
    for ew in range(n_ews):
        r = ew_rank[ew]
        base.append(used.get(r, 0))
        used[r] = used.get(r, 0) + slots_per_ew
    return np.array(base, np.int32), max(used.values())


def layer(x, wg, k, w1, w3, w2, cand, ew_rank, slots_per_ew, mask, G, shared=None,
          tokens=None, n_threads=1, want_y=False, gate_mode=0, wsg=None):
    """The whole path O1..O8 for global tokens ``x`` (contiguous split over G ranks).

    Returns a dict with logits, idx, w, gap, rank_e, bank_e, dst_rank,
    dst_slot, dst_pos, counts, out and out_f64 (out before its bf16 rounding; for
    ``tokens`` or all tokens), y/ysh (want_y), rc.
    """
    logits = router(x, wg)
    idx, w, gap = select(logits, k, gate_mode)
    n_ews = len(ew_rank)
    base, S_max = slot_bases(n_ews, ew_rank, slots_per_ew)
    rank_e, bank_e, rc = resolve(cand, ew_rank, base, mask)
    res = dict(logits=logits, idx=idx, w=w, gap=gap, rank_e=rank_e, bank_e=bank_e, rc=rc,
               slot_base=base, S_max=S_max)
    used = np.unique(idx)
    if np.any(rank_e[used] < 0):
        res["rc"] = ERR_NO_ROUTE
        return res
    dr, ds, dp, counts = permute(idx, rank_e, bank_e, G, S_max)
    res.update(dst_rank=dr, dst_slot=ds, dst_pos=dp, counts=counts)
    sgate = shared_gate(x, wsg) if (wsg is not None and shared is not None) else None
    res["sgate"] = sgate
    r, res["out_f64"] = moe_tokens(x, idx, w, w1, w3, w2, shared=shared, tokens=tokens, n_threads=n_threads,
                                   want_y=want_y, sgate=sgate, want_f64=True)
    if want_y:
        res["out"], (res["y"], res["ysh"]) = r
    else:
        res["out"] = r
    res["rc"] = OK
    return res
