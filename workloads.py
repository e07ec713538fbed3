"""Seeded synthetic inputs shared by the tests, smoke() and bench.py.

This module holds NO arithmetic of the method (no gating, routing, FFN or
combine): it only draws random tensors and builds placement tables from the
configs in BASELINE.json.  Both the CUDA path and the oracle consume its
output; neither is imported here.

Recipe:
  x  ~ N(0, 1)            -> bf16      (token embeddings)
  Wg ~ N(0, 1/d)          -> bf16      (router; logits ~ N(0, 1))
  W1, W3 ~ N(0, 1/d), W2 ~ N(0, 1/F)  -> bf16  (so h, y are O(1))
  "skewed" routing (App. B, P:1497 imbalance): x_t = z_t + mu*u and Wg rows
  get alpha_e*u with alpha decreasing in e, so low ids draw more tokens.
All draws use torch.Generator(seed) on CPU (or on a CUDA device for bench
sizes), so a (config, seed) pair names one exact input.
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional

import numpy as np
import torch


@dataclasses.dataclass
class Shape:
    name: str
    d: int          # d_model
    E: int          # routed experts
    k: int          # top-k
    F: int          # expert FFN width
    F_sh: int = 0   # merged shared-expert width (0 = none)
    T: int = 256    # global tokens per layer call
    gate_mode: int = 0    # 0 softmax over the k selected; 1 softmax over all E, no renormalisation
    shared_gate: int = 0  # 1: shared expert scaled by sigmoid(x . wsg)


# BASELINE.json "configs" (index = position in that list).
CONFIGS = {
    "tiny": Shape("tiny", d=64, E=8, k=2, F=128, T=256),                              # configs[0]
    "mixtral_decode": Shape("mixtral_decode", d=4096, E=8, k=2, F=14336, T=256),     # configs[1], [2]
    "ds_v2_lite_decode": Shape("ds_v2_lite_decode", d=2048, E=64, k=6, F=1408, F_sh=2816, T=1024),  # configs[3]
    "qwen_prefill": Shape("qwen_prefill", d=2048, E=60, k=4, F=1408, T=8192),        # configs[4]
    # NEXT-3b: the public models' own gating (norm_topk_prob = false) and, for Qwen1.5-MoE-A2.7B,
    # its sigmoid-gated shared expert (shared_expert_intermediate_size 5632)
    "ds_v2_lite_decode_g1": Shape("ds_v2_lite_decode_g1", d=2048, E=64, k=6, F=1408, F_sh=2816, T=1024,
                                  gate_mode=1),
    "qwen_prefill_sg": Shape("qwen_prefill_sg", d=2048, E=60, k=4, F=1408, F_sh=5632, T=8192,
                             gate_mode=1, shared_gate=1),
}


def _gen(seed: int, device="cpu") -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def bf16_normal(shape, std: float, seed: int, device="cpu") -> torch.Tensor:
    """N(0, std^2) drawn in fp32, stored as bf16 (torch's round-to-nearest-even)."""
    g = _gen(seed, device)
    t = torch.randn(*shape, generator=g, device=device, dtype=torch.float32)
    return (t * std).to(torch.bfloat16)


def as_u16(t: torch.Tensor) -> np.ndarray:
    """bf16 tensor -> numpy uint16 bit patterns (host)."""
    return t.detach().cpu().contiguous().view(torch.int16).numpy().view(np.uint16)


@dataclasses.dataclass
class Layer:
    shape: Shape
    wg: torch.Tensor                 # [E, d] bf16
    w1: List[torch.Tensor]           # E x [F, d]
    w3: List[torch.Tensor]           # E x [F, d]
    w2: List[torch.Tensor]           # E x [d, F]
    shared: Optional[tuple] = None   # (W1s [F_sh,d], W3s [F_sh,d], W2s [d,F_sh])
    wsg: Optional[torch.Tensor] = None  # [d] shared-expert gate (shared_gate)


def make_layer(shape: Shape, seed: int, device="cpu", skew: float = 0.0, u: Optional[torch.Tensor] = None) -> Layer:
    d, E, F = shape.d, shape.E, shape.F
    wg = bf16_normal((E, d), d ** -0.5, seed * 1000 + 1, device)
    if skew:
        assert u is not None
        alpha = torch.linspace(skew, -skew, E, device=device)[:, None]
        wg = (wg.float() + alpha * u[None, :].to(device) * d ** -0.5).to(torch.bfloat16)
    w1 = [bf16_normal((F, d), d ** -0.5, seed * 1000 + 10 + 3 * e, device) for e in range(E)]
    w3 = [bf16_normal((F, d), d ** -0.5, seed * 1000 + 11 + 3 * e, device) for e in range(E)]
    w2 = [bf16_normal((d, F), F ** -0.5, seed * 1000 + 12 + 3 * e, device) for e in range(E)]
    shared = None
    if shape.F_sh:
        Fs = shape.F_sh
        shared = (bf16_normal((Fs, d), d ** -0.5, seed * 1000 + 2, device),
                  bf16_normal((Fs, d), d ** -0.5, seed * 1000 + 3, device),
                  bf16_normal((d, Fs), Fs ** -0.5, seed * 1000 + 4, device))
    wsg = bf16_normal((d,), d ** -0.5, seed * 1000 + 5, device) if shape.shared_gate else None
    return Layer(shape, wg, w1, w3, w2, shared, wsg)


def make_tokens(shape: Shape, seed: int, T: Optional[int] = None, device="cpu", skew_mu: float = 0.0,
                u: Optional[torch.Tensor] = None) -> torch.Tensor:
    T = shape.T if T is None else T
    x = torch.randn(T, shape.d, generator=_gen(seed * 7919 + 5, device), device=device)
    if skew_mu:
        x = x + skew_mu * u[None, :].to(device)
    return x.to(torch.bfloat16)


def integer_layer(shape: Shape, seed: int, lo: int = -2, hi: int = 2) -> Layer:
    """Small integer-valued bf16 weights: router logits are exact integers in any
    accumulation order, so exact ties occur and the lowest-id tie-break must be
    reproduced bit-exactly (no near-tie exemption)."""
    g = _gen(seed)
    d, E, F = shape.d, shape.E, shape.F

    def ri(*s):
        return torch.randint(lo, hi + 1, s, generator=g).to(torch.bfloat16)
    wg = ri(E, d)
    # FFN weights stay Gaussian (the tie test is about routing)
    base = make_layer(shape, seed)
    return Layer(shape, wg, base.w1, base.w3, base.w2, base.shared)


def integer_tokens(shape: Shape, seed: int, T: Optional[int] = None, lo: int = -1, hi: int = 1) -> torch.Tensor:
    g = _gen(seed * 31 + 7)
    T = shape.T if T is None else T
    return torch.randint(lo, hi + 1, (T, shape.d), generator=g).to(torch.bfloat16)


# ---------------------------------------------------------------- placement

def contiguous_experts(E: int, W: int) -> List[List[int]]:
    """EW w hosts experts [floor(wE/W), floor((w+1)E/W))  (R#11)."""
    return [list(range((w * E) // W, ((w + 1) * E) // W)) for w in range(W)]


def spread_shadow_ew(w: int, i: int, W: int) -> int:
    """The i-th primary of EW w is shadowed on EW (w+1+(i mod (W-1))) mod W (R#10)."""
    if W == 1:
        return w
    return (w + 1 + (i % (W - 1))) % W


@dataclasses.dataclass
class Placement:
    n_ews: int
    ew_rank: List[int]
    slots_per_ew: int
    hosted: List[List[int]]          # hosted[ew][slot] = expert id (-1 empty)
    cand: np.ndarray                 # [E, C, 2] (ew, slot), primaries first


def make_placement(E: int, W: int, G: int, shadows: bool = True) -> Placement:
    """W logical EWs on G ranks (EW w on rank w*G//W), contiguous primaries,
    spread shadows; route table = [primary, shadow] per expert."""
    prim = contiguous_experts(E, W)
    hosted = [list(p) for p in prim]
    cand = -np.ones((E, 2 if (shadows and W > 1) else 1, 2), np.int32)
    for w in range(W):
        for s, e in enumerate(prim[w]):
            cand[e, 0] = (w, s)
    if shadows and W > 1:
        for w in range(W):
            for i, e in enumerate(prim[w]):
                sw = spread_shadow_ew(w, i, W)
                hosted[sw].append(e)
                cand[e, 1] = (sw, len(hosted[sw]) - 1)
    spe = max(len(h) for h in hosted)
    for h in hosted:
        h.extend([-1] * (spe - len(h)))
    ew_rank = [(w * G) // W for w in range(W)]
    return Placement(W, ew_rank, spe, hosted, cand)


def flipped(cand: np.ndarray) -> np.ndarray:
    """Route table B of the flip protocol: candidate order reversed (shadows first)."""
    return np.ascontiguousarray(cand[:, ::-1, :])
