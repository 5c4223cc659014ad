"""A second, separately written integer attention for pinning the oracle.

Untiled (T_c = 1) integer softmax-attention written directly from the paper's
equations with numpy int64 and Python-level constants -- it shares no code with
oracle/qflash_oracle.c.  With block_kv >= N, Algorithm 1 has one KV
tile, the ScaleRelease terms multiply l = O = 0, and the method reduces to:

    S = Q K^T                                   Eq. 3
    m = rowmax(S)                               Eq. 4
    y = ShiftExp2(S - m)                        Alg. 2 (q by eq:q_div)
    P = min(127, (y * M_r) >> r)                Eq. 9-10, s_P = 1/127
    l = sum_c P,  O = P V                       Eq. 11, Eq. 3
    out = clamp(floor(O / l), -128, 127)        step (11)
"""
from __future__ import annotations

import math

import numpy as np


def params(s_q: float, s_k: float, d: int):
    s = (float(np.float32(s_q)) * float(np.float32(s_k))) * 1.4426950408889634 / math.sqrt(d)
    s_inv = int(math.floor(1.0 / s + 0.5))  # 1/s > 0: half-up == half-away
    ratio = 127.0 * s
    n = math.floor(math.log2(ratio))
    # guard the float log2 at exact powers of two
    while 2.0 ** n > ratio:
        n -= 1
    while 2.0 ** (n + 1) <= ratio:
        n += 1
    r = 8 - n
    m_r = int(math.floor(ratio * 2.0 ** r + 0.5))
    return s, s_inv, r, m_r


def shift_exp2(x: np.ndarray, s_inv: int) -> np.ndarray:
    x = x.astype(np.int64)
    q = (-x) // s_inv                      # eq:q_div, numpy // is floor
    r = x + q * s_inv
    t = (r >> 1) + s_inv                   # arithmetic shift = floor
    qc = np.minimum(q, 62)
    return np.where(q >= 62, 0, t >> qc)


def untiled_attention(q: np.ndarray, k: np.ndarray, v: np.ndarray, s_q: float, s_k: float):
    P, N, d = q.shape
    _, s_inv, r, m_r = params(s_q, s_k, d)
    q64, k64, v64 = q.astype(np.int64), k.astype(np.int64), v.astype(np.int64)
    S = np.einsum("pid,pjd->pij", q64, k64)
    m = S.max(axis=-1, keepdims=True)
    y = shift_exp2(S - m, s_inv)
    Pm = np.minimum(127, (y * m_r) >> r)
    l = Pm.sum(axis=-1, keepdims=True)
    O = np.einsum("pij,pjd->pid", Pm, v64)
    out = np.clip(O // l, -128, 127)
    return out.astype(np.int8), l[..., 0], O
