"""CPU oracle for the QFlash hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package.  The product path
(``paper_2604_25306_b200`` + ``libqflash.so``) never imports it and shares no
code with it.

* ``qflash_oracle.c`` -- the integer method (Eq. 1-14, Algorithms 1 and 2 of
  arxiv 2604.25306), plain C with int64 intermediates, loaded here via ctypes.
* ``fp_reference.py`` -- the FP64 attention the paper's SQNR/MSE compare
  against (Table[SQNR]).

Parity status: every function is pinned by ``tests/test_oracle_pins.py`` except
the exact output *bits* of Algorithm 1, which the paper never prints ("parity
unpinned by the paper" -- pinned only through readings R1-R22 in DESIGN.md and
the invariants/brute-force checks listed there).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "qflash_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

# Status codes of the oracle (its own, independent of include/qflash.h).
QO_OK, QO_ERR_INVALID, QO_ERR_SHAPE, QO_ERR_SCALE = 0, 1, 2, 3


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2, no fast-math: IEEE fp32/fp64)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-D_GNU_SOURCE", "-fno-fast-math", "-ffp-contract=off",
               "-shared", "-fPIC", "-o", _LIB, _SRC, "-lm", "-lpthread"]
        subprocess.run(cmd, check=True)
    return _LIB


class _Params(ctypes.Structure):
    _fields_ = [("s", ctypes.c_double), ("s_inv", ctypes.c_int64), ("n", ctypes.c_int32),
                ("r_p", ctypes.c_int32), ("m_p", ctypes.c_int64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        L = _lib
        i64, i32, f32, vp = ctypes.c_int64, ctypes.c_int32, ctypes.c_float, ctypes.c_void_p
        L.qo_floordiv.restype = i64
        L.qo_floordiv.argtypes = [i64, i64]
        L.qo_quantize_f32.restype = ctypes.c_int
        L.qo_quantize_f32.argtypes = [vp, i64, vp, ctypes.POINTER(f32)]
        L.qo_quantize_bf16.restype = ctypes.c_int
        L.qo_quantize_bf16.argtypes = [vp, i64, vp, ctypes.POINTER(f32)]
        L.qo_dequantize.restype = None
        L.qo_dequantize.argtypes = [vp, i64, f32, vp]
        L.qo_derive_params.restype = ctypes.c_int
        L.qo_derive_params.argtypes = [f32, f32, i32, ctypes.POINTER(_Params)]
        L.qo_quotient_div.restype = i64
        L.qo_quotient_div.argtypes = [i64, i64]
        L.qo_shift_exp2.restype = i64
        L.qo_shift_exp2.argtypes = [i64, i64]
        L.qo_requantize.restype = i64
        L.qo_requantize.argtypes = [i64, i64, i32]
        L.qo_scale_release.restype = i64
        L.qo_scale_release.argtypes = [i64, i64, i64]
        L.qo_attention_mode.restype = ctypes.c_int
        L.qo_attention_mode.argtypes = [vp, vp, vp, i64, i32, i32, i32, i32, f32, f32, i32, i32,
                                        vp, ctypes.POINTER(i32)]
        L.qo_make_multiplier.restype = ctypes.c_int
        L.qo_make_multiplier.argtypes = [ctypes.c_double, i32, ctypes.POINTER(i32),
                                         ctypes.POINTER(i32), ctypes.POINTER(i64)]
        L.qo_shift_exp2_array.restype = None
        L.qo_shift_exp2_array.argtypes = [vp, i64, i64, vp]
        L.qo_normalize.restype = i64
        L.qo_normalize.argtypes = [i64, i64]
        L.qo_attention_rows_state.restype = ctypes.c_int
        L.qo_attention_rows_state.argtypes = [vp, vp, vp, i32, i32, i32, f32, f32, i64, i32, i32,
                                              vp, vp, vp]
        L.qo_attention_rows.restype = ctypes.c_int
        L.qo_attention_rows.argtypes = [vp, vp, vp, i32, i32, i32, f32, f32, i64, i32, i32, vp]
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# --------------------------------------------------------------- scalar steps
def floordiv(a: int, b: int) -> int:
    return int(lib().qo_floordiv(a, b))


def quotient_div(x: int, s_inv: int) -> int:
    """eq:q_div."""
    return int(lib().qo_quotient_div(x, s_inv))


def shift_exp2(x: int, s_inv: int) -> int:
    """Algorithm 2 with the eq:q_div quotient (R6)."""
    return int(lib().qo_shift_exp2(x, s_inv))


def requantize(y: int, m_p: int, r_p: int) -> int:
    """Eq. 10 + R8 clamp."""
    return int(lib().qo_requantize(y, m_p, r_p))


def shift_exp2_array(x: np.ndarray, s_inv: int) -> np.ndarray:
    """Vector form of Algorithm 2 (same C function per element)."""
    x = np.ascontiguousarray(x, dtype=np.int64)
    y = np.empty_like(x)
    lib().qo_shift_exp2_array(_ptr(x), x.size, s_inv, _ptr(y))
    return y


def make_multiplier(ratio: float, b: int = 8):
    """Eq. 9-10: (n, r, M_r) for a real ratio s_X / s_Y."""
    n, r, m = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int64()
    rc = lib().qo_make_multiplier(ratio, b, ctypes.byref(n), ctypes.byref(r), ctypes.byref(m))
    if rc != QO_OK:
        raise ValueError(rc)
    return n.value, r.value, m.value


def normalize(o: int, l: int) -> int:
    """Step (11): floor(O / l) saturated to int8 (R14)."""
    return int(lib().qo_normalize(o, l))


def scale_release(x: int, alpha: int, s_inv: int) -> int:
    """Eq. 14 realised per P:L408 (R10)."""
    return int(lib().qo_scale_release(x, alpha, s_inv))


def derive_params(s_q: float, s_k: float, d: int):
    """Host constants s, s_inv, n, r_P, M_P (Eq. 9-10).

    Returns a dict, or raises ValueError with the oracle status code."""
    p = _Params()
    rc = lib().qo_derive_params(ctypes.c_float(s_q), ctypes.c_float(s_k), d, ctypes.byref(p))
    if rc != QO_OK:
        raise ValueError(rc)
    return {"s": p.s, "s_inv": p.s_inv, "n": p.n, "r_p": p.r_p, "m_p": p.m_p}


# --------------------------------------------------------------- tensor steps
def quantize(x: np.ndarray):
    """Eq. 2 per-tensor int8 quantization (R1-R4).  fp32 or bf16 (as uint16)."""
    x = np.ascontiguousarray(x)
    out = np.empty(x.shape, dtype=np.int8)
    s = ctypes.c_float(0.0)
    if x.dtype == np.float32:
        rc = lib().qo_quantize_f32(_ptr(x), x.size, _ptr(out), ctypes.byref(s))
    elif x.dtype == np.uint16:  # raw bf16 bits
        rc = lib().qo_quantize_bf16(_ptr(x), x.size, _ptr(out), ctypes.byref(s))
    else:
        raise TypeError(x.dtype)
    if rc != QO_OK:
        raise ValueError(rc)
    return out, float(s.value)


def dequantize(xq: np.ndarray, s: float) -> np.ndarray:
    xq = np.ascontiguousarray(xq, dtype=np.int8)
    y = np.empty(xq.shape, dtype=np.float32)
    lib().qo_dequantize(_ptr(xq), xq.size, ctypes.c_float(s), _ptr(y))
    return y


def attention(q: np.ndarray, k: np.ndarray, v: np.ndarray, s_q: float, s_k: float,
              block_kv: int = 128, block_r: int = 128, mode: int = 0, nthreads: int = 1,
              return_overflow: bool = False):
    """Algorithm 1 over [P, N, d] int8 problems; returns int8 [P, N, d].

    mode 0 = Scale Release (Eq. 14, the method); 1 = Scale Accumulation (Eq. 13)."""
    q = np.ascontiguousarray(q, dtype=np.int8)
    k = np.ascontiguousarray(k, dtype=np.int8)
    v = np.ascontiguousarray(v, dtype=np.int8)
    assert q.shape == k.shape == v.shape and q.ndim == 3
    P, N, d = q.shape
    out = np.empty_like(q)
    ovf = ctypes.c_int32(0)
    rc = lib().qo_attention_mode(_ptr(q), _ptr(k), _ptr(v), P, N, d, block_r, block_kv,
                                 ctypes.c_float(s_q), ctypes.c_float(s_k), mode, nthreads,
                                 _ptr(out), ctypes.byref(ovf))
    if rc != QO_OK:
        raise ValueError(rc)
    if return_overflow:
        return out, bool(ovf.value)
    return out


def attention_rows(q, k, v, s_q, s_k, p: int, row_begin: int, row_end: int,
                   block_kv: int = 128) -> np.ndarray:
    """Rows [row_begin, row_end) of problem p only (sampled parity at full size)."""
    q = np.ascontiguousarray(q, dtype=np.int8)
    k = np.ascontiguousarray(k, dtype=np.int8)
    v = np.ascontiguousarray(v, dtype=np.int8)
    P, N, d = q.shape
    out = np.empty((row_end - row_begin, d), dtype=np.int8)
    rc = lib().qo_attention_rows(_ptr(q), _ptr(k), _ptr(v), N, d, block_kv,
                                 ctypes.c_float(s_q), ctypes.c_float(s_k), p, row_begin,
                                 row_end, _ptr(out))
    if rc != QO_OK:
        raise ValueError(rc)
    return out


def attention_rows_state(q, k, v, s_q, s_k, p: int, row_begin: int, row_end: int,
                         block_kv: int = 128):
    """Like attention_rows, also returning the final integer state (l, O) per row
    before normalization (test access to the fixed-point normaliser)."""
    q = np.ascontiguousarray(q, dtype=np.int8)
    k = np.ascontiguousarray(k, dtype=np.int8)
    v = np.ascontiguousarray(v, dtype=np.int8)
    P, N, d = q.shape
    rows = row_end - row_begin
    out = np.empty((rows, d), dtype=np.int8)
    l_state = np.empty((rows,), dtype=np.int64)
    o_state = np.empty((rows, d), dtype=np.int64)
    rc = lib().qo_attention_rows_state(_ptr(q), _ptr(k), _ptr(v), N, d, block_kv,
                                       ctypes.c_float(s_q), ctypes.c_float(s_k), p, row_begin,
                                       row_end, _ptr(out), _ptr(l_state), _ptr(o_state))
    if rc != QO_OK:
        raise ValueError(rc)
    return out, l_state, o_state


# --------------------------------------------------------------- per-head granularity
# one scale per (tensor, head) instead of per
# tensor.  Problems are the flattened (batch, window, head) with the head fastest
# (p = (b W + w) H + h), so head h owns the problems p = h, h + H, h + 2H, ...  Each
# head is quantized, attended and dequantized exactly as a per-tensor problem set of
# its own: the definitions below are that composition, nothing more.
def head_problems(P: int, H: int, h: int) -> np.ndarray:
    return np.arange(h, P, H)


def quantize_per_head(x: np.ndarray, H: int):
    """Eq. 2 with the amax taken over each head's problems (x: [P, N, d])."""
    P = x.shape[0]
    assert P % H == 0
    out = np.empty(x.shape, dtype=np.int8)
    scales = np.empty(H, dtype=np.float32)
    for h in range(H):
        idx = head_problems(P, H, h)
        out[idx], s = quantize(np.ascontiguousarray(x[idx]))
        scales[h] = s
    return out, scales


def attention_per_head(q, k, v, s_q, s_k, H: int, block_kv: int = 128, nthreads: int = 1):
    """Algorithm 1 with head h's constants derived from (s_q[h], s_k[h])."""
    P = q.shape[0]
    out = np.empty_like(np.asarray(q, dtype=np.int8))
    for h in range(H):
        idx = head_problems(P, H, h)
        out[idx] = attention(q[idx], k[idx], v[idx], float(s_q[h]), float(s_k[h]),
                             block_kv=block_kv, nthreads=nthreads)
    return out


def dequantize_per_head(xq: np.ndarray, s: np.ndarray, H: int) -> np.ndarray:
    P = xq.shape[0]
    y = np.empty(xq.shape, dtype=np.float32)
    for h in range(H):
        idx = head_problems(P, H, h)
        y[idx] = dequantize(np.ascontiguousarray(xq[idx]), float(s[h]))
    return y
