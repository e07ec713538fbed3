"""Independent bf16 round-to-nearest-even, written from the IEEE-754 definition
with numpy's exact frexp/ldexp (scaling by powers of two and splitting off the
integer part are exact in binary64).  Used only to pin the oracle's rounding.
"""
import numpy as np


def bf16_rne_exact(v) -> np.ndarray:
    """fp64 array -> bf16 bit patterns (uint16), exact RNE of the fp64 value."""
    v = np.asarray(v, dtype=np.float64)
    out = np.zeros(v.shape, np.uint16)
    sign = np.signbit(v).astype(np.uint32) << 15
    a = np.abs(v)
    nan = np.isnan(v)
    inf = np.isinf(v)
    fin = ~(nan | inf) & (a > 0)
    m, e = np.frexp(np.where(fin, a, 1.0))        # a = m * 2^e, m in [0.5, 1)
    # normal bf16: value = 1.f * 2^(e-1) with exponent e-1 >= -126; 8 significant bits
    exp_unb = e - 1
    # quantum exponent q: normals 2^(exp-7), subnormals 2^-133
    q = np.where(exp_unb >= -126, exp_unb - 7, -133)
    scaled = np.ldexp(np.where(fin, a, 0.0), -q)   # exact: a / 2^q
    n = np.floor(scaled)
    rem = scaled - n                               # exact
    up = (rem > 0.5) | ((rem == 0.5) & (np.mod(n, 2) == 1))
    n = n + up
    # re-encode: value = n * 2^q
    res = np.zeros(v.shape, np.uint32)
    normal = exp_unb >= -126
    # normals: n in [128, 256]
    be = exp_unb + 127
    carry = normal & (n >= 256)
    n = np.where(carry, n / 2, n)
    be = np.where(carry, be + 1, be)
    enc_norm = (be.astype(np.int64) << 7) | (n.astype(np.int64) & 0x7F)
    enc_norm = np.where(be >= 255, 0x7F80, enc_norm)
    enc_sub = n.astype(np.int64)                    # n in [0,128]; 128 -> exponent field 1
    res = np.where(normal, enc_norm, enc_sub).astype(np.uint32)
    res = np.where(fin, res, 0)
    res = np.where(inf, 0x7F80, res)
    res = np.where(nan, 0x7FC0, res)
    out = (res | sign).astype(np.uint16)
    return out


def bf16_bits_to_f64(b) -> np.ndarray:
    b = np.asarray(b, dtype=np.uint16).astype(np.uint32) << 16
    return b.view(np.float32).astype(np.float64)
