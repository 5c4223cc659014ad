"""Seeded synthetic inputs and the workload catalog (shared by tests, bench, smoke).

This module holds NONE of the method's arithmetic: only random draws and the
shapes of the paper's workloads.  It is the one module both the CUDA path's
tests and the oracle's tests take inputs from.

Workloads: Table 1 of arxiv 2604.25306 -- A1-A3 ViT/DeiT T/S/B
(N=197, d=64, heads 3/6/12) and A4-A7 Swin-T/S stages 1-4 (N=49, d=32,
windows 64/16/4/1, heads 3/6/12/24) -- plus BASELINE.json's Swin-B stages
(heads 4/8/16/32) and the ViT-L/14@448 stress shape (N=32*32+1=1025, 16 heads).
Problems are flattened as p = (b*W + w)*H + h (windows folded into the batch
axis, SPEC D21 S:L540); Q, K, V are [P, N, d] row-major.

Recipe (calibrated so the FP output power matches the 2.68 / 3.12
implied by Table[SQNR]): numpy default_rng(seed), fp32, draw order
mu_Q, Q, mu_K, K, mu_V, V;
  Q, K = mu + N(0, 1.5^2),  mu ~ N(0, 0.5^2) per (problem, channel);
  V    = mu_V + N(0, 0.6^2), mu_V ~ N(0, 1.6^2) (ViT) or N(0, 1.7^2) (Swin).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Workload:
    name: str
    source: str
    windows: int
    heads: int
    seq_len: int
    head_dim: int
    family: str  # "vit" | "swin"

    def problems(self, batch: int) -> int:
        return batch * self.windows * self.heads


# Table 1 + BASELINE.json configs.
CATALOG = {
    "A1": Workload("A1", "ViT/DeiT-Tiny", 1, 3, 197, 64, "vit"),
    "A2": Workload("A2", "ViT/DeiT-Small", 1, 6, 197, 64, "vit"),
    "A3": Workload("A3", "ViT/DeiT-Base", 1, 12, 197, 64, "vit"),
    "A4": Workload("A4", "Swin-T/S Stage-1", 64, 3, 49, 32, "swin"),
    "A5": Workload("A5", "Swin-T/S Stage-2", 16, 6, 49, 32, "swin"),
    "A6": Workload("A6", "Swin-T/S Stage-3", 4, 12, 49, 32, "swin"),
    "A7": Workload("A7", "Swin-T/S Stage-4", 1, 24, 49, 32, "swin"),
    "SwinB-s1": Workload("SwinB-s1", "Swin-B Stage-1", 64, 4, 49, 32, "swin"),
    "SwinB-s2": Workload("SwinB-s2", "Swin-B Stage-2", 16, 8, 49, 32, "swin"),
    "SwinB-s3": Workload("SwinB-s3", "Swin-B Stage-3", 4, 16, 49, 32, "swin"),
    "SwinB-s4": Workload("SwinB-s4", "Swin-B Stage-4", 1, 32, 49, 32, "swin"),
    "L14": Workload("L14", "ViT-L/14@448", 1, 16, 1025, 64, "vit"),
}

# BASELINE.json "configs" -> (workload, batch).
BASELINE_CONFIGS = {
    0: ("A1", 1),   # DeiT-Tiny b1 (the oracle finishes in seconds)
    1: ("A3", 8),   # ViT-Base b8 (the bench workload)
    2: ("A4", 8),   # Swin-T stage-1 b8
    3: ("SwinB-s1", 8),  # Swin-B all stages; s1 listed here, s2-s4 in CATALOG
    4: ("L14", 64),  # long-sequence stress
}


def gen_real_qkv(P: int, N: int, d: int, seed: int = 0, family: str = "vit"):
    """Real-valued fp32 Q, K, V [P, N, d] per the recipe above."""
    rng = np.random.default_rng(seed)
    mu_v_std = 1.6 if family == "vit" else 1.7
    mu_q = rng.standard_normal((P, 1, d), dtype=np.float32) * np.float32(0.5)
    q = mu_q + rng.standard_normal((P, N, d), dtype=np.float32) * np.float32(1.5)
    mu_k = rng.standard_normal((P, 1, d), dtype=np.float32) * np.float32(0.5)
    k = mu_k + rng.standard_normal((P, N, d), dtype=np.float32) * np.float32(1.5)
    mu_v = rng.standard_normal((P, 1, d), dtype=np.float32) * np.float32(mu_v_std)
    v = mu_v + rng.standard_normal((P, N, d), dtype=np.float32) * np.float32(0.6)
    return q.astype(np.float32), k.astype(np.float32), v.astype(np.float32)


def gen_workload(name: str, batch: int, seed: int = 0):
    w = CATALOG[name]
    return gen_real_qkv(w.problems(batch), w.seq_len, w.head_dim, seed, w.family)


# ------------------------------------------------ parity-only adversarial int8 sets
ADVERSARIAL_KINDS = ("uniform", "all_min", "constant_rows", "one_hot", "ties", "zeros")


def gen_int8_qkv(P: int, N: int, d: int, seed: int = 0, kind: str = "uniform"):
    """int8 Q, K, V [P, N, d] for parity-only sets (no quantizer involved).

    uniform: U[-128, 127]; all_min: Q = K = -128 (S = +d*2^14, the extreme);
    constant_rows: every row of Q/K/V constant; one_hot: Q rows aligned with one
    K row (peaky softmax); ties: K drawn from 2 distinct rows (many tied maxima);
    zeros: Q = K = 0 (uniform attention)."""
    rng = np.random.default_rng(seed)
    u = lambda *s: rng.integers(-128, 128, size=s, dtype=np.int16).astype(np.int8)
    if kind == "uniform":
        return u(P, N, d), u(P, N, d), u(P, N, d)
    if kind == "all_min":
        q = np.full((P, N, d), -128, np.int8)
        return q, q.copy(), u(P, N, d)
    if kind == "constant_rows":
        q = np.repeat(u(P, N, 1), d, axis=2)
        k = np.repeat(u(P, N, 1), d, axis=2)
        v = np.repeat(u(P, N, 1), d, axis=2)
        return q, k, v
    if kind == "one_hot":
        k = u(P, N, d)
        idx = rng.integers(0, N, size=(P, N))
        q = np.take_along_axis(k, idx[:, :, None].repeat(d, axis=2), axis=1)
        return q.copy(), k, u(P, N, d)
    if kind == "ties":
        base = u(P, 2, d)
        pick = rng.integers(0, 2, size=(P, N))
        k = np.take_along_axis(base, pick[:, :, None].repeat(d, axis=2), axis=1)
        return u(P, N, d), k.copy(), u(P, N, d)
    if kind == "zeros":
        z = np.zeros((P, N, d), np.int8)
        return z, z.copy(), u(P, N, d)
    raise ValueError(kind)


# Scales paired with the int8 adversarial sets: the regime of real workloads
# (s_q = s_k ~ amax/127 for |x| up to ~7) unless a test overrides them.
DEFAULT_INT8_SCALES = (0.055, 0.055, 0.03)


# ------------------------------------------------ problem-addressable global batches
SLAB_CHUNK = 16  # problems per independently seeded chunk


def gen_real_qkv_slab(P_total: int, N: int, d: int, begin: int, count: int, seed: int = 0,
                      family: str = "vit"):
    """Problems [begin, begin + count) of a global [P_total, N, d] batch defined chunk by
    chunk: chunk c (problems [16 c, 16 c + 16)) is gen_real_qkv(..., seed=[seed, c]).  Any
    rank can generate its own slab (multi-GPU bench), and the concatenation over a
    partition equals the slab of the whole batch."""
    assert 0 <= begin and begin + count <= P_total
    out = [np.empty((count, N, d), np.float32) for _ in range(3)]
    c0, c1 = begin // SLAB_CHUNK, (begin + count + SLAB_CHUNK - 1) // SLAB_CHUNK
    for c in range(c0, c1):
        lo, hi = c * SLAB_CHUNK, min(P_total, (c + 1) * SLAB_CHUNK)
        chunk = gen_real_qkv(hi - lo, N, d, seed=[seed, c], family=family)
        a, b = max(lo, begin), min(hi, begin + count)
        for t in range(3):
            out[t][a - begin:b - begin] = chunk[t][a - lo:b - lo]
    return tuple(out)
