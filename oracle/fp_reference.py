"""FP64 attention and error metrics -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper measures QFlash against floating-point attention with SQNR and MSE
(Table[SQNR]; definitions).  This module is that
reference: softmax(Q K^T / sqrt(d)) V in float64 with max subtraction, on the
*original real* inputs, so the measured error includes input quantization.
"""
from __future__ import annotations

import numpy as np


def attention_fp64(q: np.ndarray, k: np.ndarray, v: np.ndarray) -> np.ndarray:
    """softmax(Q K^T / sqrt(d)) V per problem; inputs [P, N, d] real."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    d = q.shape[-1]
    s = np.einsum("pid,pjd->pij", q, k) / np.sqrt(d)
    s -= s.max(axis=-1, keepdims=True)
    e = np.exp(s)
    w = e / e.sum(axis=-1, keepdims=True)
    return np.einsum("pij,pjd->pid", w, v)


def sqnr_db(ref: np.ndarray, test: np.ndarray) -> float:
    """10 log10(sum ref^2 / sum (ref - test)^2)."""
    ref = np.asarray(ref, dtype=np.float64)
    test = np.asarray(test, dtype=np.float64)
    noise = np.sum((ref - test) ** 2)
    if noise == 0.0:
        return float("inf")
    return float(10.0 * np.log10(np.sum(ref ** 2) / noise))


def mse(ref: np.ndarray, test: np.ndarray) -> float:
    ref = np.asarray(ref, dtype=np.float64)
    test = np.asarray(test, dtype=np.float64)
    return float(np.mean((ref - test) ** 2))
