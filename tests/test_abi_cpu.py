"""The C ABI on a machine without a GPU: the library loads, exports every symbol
the headers declare, and its pure-host logic (constant derivation, the exact
division-free magics, argument validation, partitioning) is checked here."""
from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

from paper_2604_25306_b200 import _lib
from paper_2604_25306_b200.api import qflash_derive_params, qflash_partition

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    names = set()
    for h in ("qflash.h", "qflash_debug.h"):
        text = open(os.path.join(ROOT, "include", h)).read()
        names.update(re.findall(r"QFLASH_API\s+[\w\s\*]+?\b(qflash_\w+)\s*\(", text))
    return sorted(names)


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    names = _declared_symbols()
    assert len(names) >= 13
    for n in names:
        assert hasattr(L, n), n
    assert set(_lib.EXPORTED) <= set(names)
    assert L.qflash_version() >> 16 == 1


def test_status_strings():
    assert _lib.status_string(0) == "QFLASH_OK"
    assert _lib.status_string(3) == "QFLASH_ERR_SCALE_RANGE"


@pytest.mark.parametrize("sq,sk,d", [(0.0625, 0.0625, 64), (0.5, 0.5, 64), (0.125, 0.125, 32),
                                     (0.03125, 0.03125, 128), (0.0411, 0.0533, 64),
                                     (0.002, 0.003, 32), (0.9, 0.9, 32), (1.3e-4, 1.1e-4, 64)])
def test_derive_params_matches_oracle(orc, sq, sk, d):
    # The library derives its constants independently of the oracle.
    try:
        ref = orc.derive_params(sq, sk, d)
    except ValueError:
        with pytest.raises(_lib.QFlashError):
            qflash_derive_params(sq, sk, d)
        return
    got = qflash_derive_params(sq, sk, d)
    for key in ("s", "s_inv", "n", "r_p", "m_p"):
        assert got[key] == ref[key], key


def test_derive_params_sweep_matches_oracle_and_magic_definitions(orc):
    # 600 random scale pairs over the whole accepted range: the oracle's fields, and
    # the division magics equal their definitions ceil(2^k / s_inv) in big integers
    # (the library computes them with an fp64-estimated, remainder-corrected division)
    rng = np.random.default_rng(2604)
    checked = 0
    for i in range(600):
        d = (32, 64, 128)[i % 3]
        sq, sk = (float(np.float32(10.0 ** rng.uniform(-4.5, 0.3))) for _ in range(2))
        try:
            ref = orc.derive_params(sq, sk, d)
        except ValueError:
            with pytest.raises(_lib.QFlashError):
                qflash_derive_params(sq, sk, d)
            continue
        got = qflash_derive_params(sq, sk, d)
        for key in ("s", "s_inv", "n", "r_p", "m_p"):
            assert got[key] == ref[key], (key, sq, sk, d)
        D = got["s_inv"]
        L = (D - 1).bit_length()
        if got["q_shift"] == 0:
            assert got["q_magic"] == -(-(1 << 32) // D)
        else:
            assert got["q_shift"] == max(L - 7, 0)
            assert got["q_magic"] == -(-(1 << (32 + got["q_shift"])) // D)
        assert got["rel_shift"] == max(L - 8, 0)
        assert got["rel_magic"] == -(-(1 << (64 + got["rel_shift"])) // D)
        checked += 1
    assert checked > 300


def _s_invs():
    return [2, 3, 22, 127, 251, 1287, 1420, 2293, 8030, 11408, 11769, 12853, 65537, 250001,
            (1 << 22), (1 << 24) - 3]


@pytest.mark.parametrize("s_inv", _s_invs())
def test_quotient_magic_exact(s_inv):
    # q1 = umulhi(t, q_magic) >> q_shift must equal floor(t / s_inv) wherever the
    # ShiftExp2 output can be non-zero (q1 <= 25); beyond, both are >= 26 so the
    # shifted value (< 2^26) is 0 either way.  t ranges over [s_inv, 2^25).
    s = 1.0 / (s_inv + 0.3)                              # round(1/s) == s_inv
    sq = float(np.sqrt(s * 8.0 / 1.4426950408889634))   # d = 64
    p = qflash_derive_params(sq, sq, 64)
    if p["s_inv"] != s_inv:
        pytest.skip("float scale did not hit this s_inv exactly")
    t = np.arange(p["s_inv"], 1 << 25, dtype=np.uint64)
    est = ((t * np.uint64(p["q_magic"])) >> np.uint64(32)) >> np.uint64(p["q_shift"])
    true = t // np.uint64(s_inv)
    live = true <= 25
    assert np.array_equal(est[live], true[live])
    assert np.all(est[~live] >= 26)
    # and the value that gets shifted stays < 2^26 where the estimate is off
    off = est != true
    if off.any():
        S_minus_m = np.int64(s_inv) - t[off].astype(np.int64)  # x + s_inv
        num = (est[off].astype(np.int64) * s_inv + S_minus_m + s_inv) & 0xFFFFFFFF
        assert np.all((num >> np.minimum(est[off], 31).astype(np.int64)) == 0)


@pytest.mark.parametrize("sq,d", [(0.05, 64), (0.002, 32), (0.6, 32), (0.3, 64), (1e-3, 128)])
def test_requant_multiplier_exact(sq, d):
    p = qflash_derive_params(sq, sq, d)
    y = np.arange(0, p["s_inv"] + 1, dtype=np.uint64)
    est = ((y << np.uint64(p["p_pre"])) * np.uint64(p["p_mul"])) >> np.uint64(32)
    true = (y * np.uint64(p["m_p"])) >> np.uint64(p["r_p"])
    assert np.array_equal(est, true)
    assert p["p_max"] == int(true[-1])


@pytest.mark.parametrize("s_inv_target", [2, 22, 1420, 8030, 1 << 20])
def test_release_magic_exact(s_inv_target):
    s = 1.0 / (s_inv_target + 0.3)
    sq = float(np.sqrt(s * 8.0 / 1.4426950408889634))
    p = qflash_derive_params(sq, sq, 64)
    D = p["s_inv"]
    M, sh = p["rel_magic"], p["rel_shift"]
    rng = np.random.default_rng(D)
    ns = [0, 1, D - 1, D, (1 << 56) - 1] + [int(x) for x in rng.integers(0, 1 << 62, 2000) >> 6]
    ns += [a << 31 for a in range(0, D + 1, max(1, D // 500))]
    for n in ns:
        assert ((n * M) >> 64) >> sh == n // D


def test_partition_properties():
    for P in (0, 1, 7, 96, 1024, 1536):
        for world in (1, 2, 3, 4, 8):
            spans = [qflash_partition(P, world, r) for r in range(world)]
            assert sum(c for _, c in spans) == P
            pos = 0
            for b, c in spans:
                assert b == pos and c >= 0
                assert c in (P // world, -(-P // world))
                pos += c
    assert qflash_partition(10, 0, 0) == (0, 0)
    assert qflash_partition(10, 2, 2) == (0, 0)


def test_validation_before_any_cuda_call():
    # Invalid arguments are rejected without touching CUDA (works with no GPU).
    L = _lib.lib()
    sh = _lib.AttnShape(2, 197, 64, 128)
    vp = ctypes.c_void_p
    assert L.qflash_attention_int8(None, None, None, 0.05, 0.05, 0.05, ctypes.byref(sh), None,
                                   None, None) == _lib.QFLASH_ERR_INVALID_ARGUMENT
    bad = _lib.AttnShape(2, 197, 48, 128)
    assert L.qflash_attention_int8(vp(16), vp(32), vp(48), 0.05, 0.05, 0.05, ctypes.byref(bad),
                                   vp(64), None, None) == _lib.QFLASH_ERR_UNSUPPORTED_SHAPE
    bad = _lib.AttnShape(2, 70000, 64, 128)
    assert L.qflash_attention_int8(vp(16), vp(32), vp(48), 0.05, 0.05, 0.05, ctypes.byref(bad),
                                   vp(64), None, None) == _lib.QFLASH_ERR_UNSUPPORTED_SHAPE
    bad = _lib.AttnShape(2, 197, 64, 32)
    assert L.qflash_attention_int8(vp(16), vp(32), vp(48), 0.05, 0.05, 0.05, ctypes.byref(bad),
                                   vp(64), None, None) == _lib.QFLASH_ERR_UNSUPPORTED_SHAPE
    n = 2 * 197 * 64
    base = 1 << 20
    assert L.qflash_attention_int8(vp(base), vp(base + 4 * n), vp(base + 8 * n), 10.0, 10.0, 1.0,
                                   ctypes.byref(sh), vp(base + 12 * n), None,
                                   None) == _lib.QFLASH_ERR_SCALE_RANGE
    assert L.qflash_attention_int8(vp(base), vp(base + 4 * n), vp(base + 8 * n), 0.05, 0.05, 0.05,
                                   ctypes.byref(sh), vp(base + 16), None,
                                   None) == _lib.QFLASH_ERR_INVALID_ARGUMENT   # o aliases q
    assert L.qflash_attention_int8(vp(base + 1), vp(base + 4 * n), vp(base + 8 * n), 0.05, 0.05,
                                   0.05, ctypes.byref(sh), vp(base + 12 * n), None,
                                   None) == _lib.QFLASH_ERR_INVALID_ARGUMENT   # misaligned
    assert L.qflash_quantize_per_tensor(vp(base), 0, 10, vp(base + 64), None, None,
                                        None) == _lib.QFLASH_ERR_INVALID_ARGUMENT  # no scale ptr
    assert L.qflash_quantize_qkv(vp(base), vp(base), vp(base), 7, 10, vp(base), vp(base),
                                 vp(base), vp(base), None) == _lib.QFLASH_ERR_INVALID_ARGUMENT
    assert L.qflash_dequantize(None, 1.0, 10, None, None) == _lib.QFLASH_ERR_INVALID_ARGUMENT
    # fused step: every code buffer must be disjoint from every fp32 input and the
    # other code buffers (k_q aliasing the fp32 q input was accepted)
    f = [vp(base + i * 4 * n) for i in range(3)]                 # fp32 q, k, v
    y, sc, ws = vp(base + 12 * n), vp(base + 16 * n), vp(base + 17 * n)
    codes = [vp(base + 20 * n + i * n) for i in range(3)]
    fused = L.qflash_forward_fused
    fused.restype = ctypes.c_int
    ok_codes = fused(*f, ctypes.byref(sh), 0, *codes, None, y, sc, ws, None)
    assert ok_codes != _lib.QFLASH_ERR_INVALID_ARGUMENT          # (device check comes later)
    for bad_codes in ([codes[0], f[0], codes[2]],                 # k_q aliases the q input
                      [codes[0], codes[1], vp(base + 8 * n + 64)],  # v_q inside the v input
                      [codes[0], codes[0], codes[2]]):            # q_q == k_q
        assert fused(*f, ctypes.byref(sh), 0, *bad_codes, None, y, sc, ws,
                     None) == _lib.QFLASH_ERR_INVALID_ARGUMENT
    assert fused(*f, ctypes.byref(sh), 0, *codes, None, y, sc, f[1],
                 None) == _lib.QFLASH_ERR_INVALID_ARGUMENT       # workspace aliases k
    # configuration override of the debug header: range-checked, -1 = heuristic
    assert L.qflash_debug_force_config(4) == _lib.QFLASH_ERR_INVALID_ARGUMENT
    assert L.qflash_debug_force_config(-2) == _lib.QFLASH_ERR_INVALID_ARGUMENT
    assert L.qflash_debug_force_config(-1) == _lib.QFLASH_OK


# ----------------------------------------------------------------------------
# The kernel's division-free ScaleRelease arithmetic (qflash_attention.cu),
# emulated with Python integers and checked against floor(X alpha / s_inv):
# pins the derivation the GPU implements (the GPU parity tests pin the code).
def _hi32(a, b):
    return ((a & 0xFFFFFFFF) * (b & 0xFFFFFFFF)) >> 32


def _release_fast(X, alpha, D, bound):
    """make_biased_release + BiasedRelease.apply (valid when (2 bound + D) D < 2^32)."""
    B = bound // D + 1
    BD = (B * D) & 0xFFFFFFFF
    ident = alpha == D
    A = 0xFFFFFFFF if ident else ((((alpha << 32) // D) & 0xFFFFFFFF) + 1) & 0xFFFFFFFF
    add = ((-(B * alpha)) + (1 if ident else 0)) & 0xFFFFFFFF
    Xp = (X + BD) & 0xFFFFFFFF
    q = (_hi32(Xp, A) + add) & 0xFFFFFFFF
    return q - (1 << 32) if q >= (1 << 31) else q


def _release_slow(X, alpha, D):
    A = min((alpha << 31) // D, (1 << 31) - 1)
    q0 = (X * A) >> 31
    rem = X * alpha - q0 * D          # exact here; the kernel computes it mod 2^32
    return q0 + (1 if rem >= D else 0) - (1 if rem < 0 else 0)


@pytest.mark.parametrize("D", [2, 3, 97, 1024, 1420, 2048, 8030, 65537, (1 << 24) - 3])
def test_kernel_release_arithmetic(D):
    rng = np.random.default_rng(D)
    alphas = [0, 1, D // 2, D - 1, D] + [int(a) for a in rng.integers(0, D + 1, 40)]
    max_bound = ((1 << 32) // D - D) // 2          # (2 bound + D) D < 2^32
    for alpha in alphas:
        if max_bound > 0:
            for bound in [0, 1, max_bound] + [int(b) for b in rng.integers(0, max_bound + 1, 8)]:
                xs = [0, 1, -1, bound, -bound] + [int(x) for x in rng.integers(-bound, bound + 1, 40)]
                for X in xs:
                    assert _release_fast(X, alpha, D, bound) == (X * alpha) // D, (X, alpha, bound)
        xs = [int(x) for x in rng.integers(-(1 << 31), 1 << 31, 200)] + [(1 << 31) - 1, -(1 << 31)]
        for X in xs:
            assert _release_slow(X, alpha, D) == (X * alpha) // D, (X, alpha)


def _floor_div_kernel(O, l):
    """Emulates make_recip + floor_div (+ the exact fallback) of the kernel."""
    k = 32 - l.bit_length()                      # __clz(l), l >= 2
    ln = (l << k) & 0xFFFFFFFF
    idx = (ln >> 21) & 1023
    R = (1 << 62) // ((1 << 31) + ((2 * idx + 1) << 20))
    sh = 30 - k
    q0 = ((O * R) >> 32) >> sh                   # __mulhi (signed) then arithmetic shift
    rem = O - q0 * l
    q = q0 + (1 if rem >= l else 0) + (-1 if rem < 0 else 0)
    bad = rem >= 2 * l or rem < -l
    if bad:                                      # floor_div_exact
        un = -(O + 1) if O < 0 else O
        qq = un // l
        q = ~qq if O < 0 else qq
    return q


def test_kernel_normalize_arithmetic():
    rng = np.random.default_rng(5)
    ls = [2, 3, 126, 127, 128, 1000, 4095, 4096, 65535, 1 << 20, (1 << 31) - 1]
    ls += [int(x) for x in rng.integers(2, 1 << 31, 300)]
    for l in ls:
        Os = [0, 1, -1, l, -l, l - 1, -l - 1, 127 * l, -128 * l, (1 << 31) - 1, -(1 << 31)]
        Os += [int(x) for x in rng.integers(-130 * l, 130 * l + 1, 50)]
        Os += [int(x) for x in rng.integers(-(1 << 31), 1 << 31, 20)]
        for O in Os:
            if -(1 << 31) <= O < (1 << 31):
                assert _floor_div_kernel(O, l) == O // l, (O, l)


def test_python_wrappers_check_buffers_before_the_abi():
    # the library sizes every buffer from q's shape, so the
    # wrappers reject a k / v / out / workspace that does not match -- before any
    # pointer reaches the C ABI (these CPU tensors never get that far).
    import torch
    from paper_2604_25306_b200 import api
    q = torch.zeros((2, 64, 32), dtype=torch.int8)
    small = torch.zeros((2, 63, 32), dtype=torch.int8)
    with pytest.raises(ValueError):
        api.qflash_attention_int8(q, small, q, 0.05, 0.05, 0.05)
    with pytest.raises(ValueError):
        api.qflash_attention_int8(q, q, q, 0.05, 0.05, 0.05, out=small)
    with pytest.raises(TypeError):
        api.qflash_attention_int8(q, q.float(), q, 0.05, 0.05, 0.05)
    ws_small = torch.zeros(16, dtype=torch.int32)
    with pytest.raises(ValueError):
        api.qflash_attention_int8_prepared(q, q, q, ws_small)
    with pytest.raises(ValueError):
        api.qflash_attention_dequant_prepared(q, q, q, torch.zeros(2048, dtype=torch.int32),
                                              out=torch.zeros((2, 64, 16)))
    f = torch.zeros((2, 64, 32))
    with pytest.raises(ValueError):
        api.qflash_forward_fused(f, f, f, codes=[q, q, small])
    with pytest.raises(ValueError):
        api.qflash_forward_fused(f, f, f, scales=torch.zeros(2))
    with pytest.raises(ValueError):
        api.qflash_attention_int8_dscale(q, q, q, torch.zeros(2))
    with pytest.raises(TypeError):
        api.qflash_dequantize(f, 1.0)
