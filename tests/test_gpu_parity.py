"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by element.

Integer outputs must be bit-exact; the quantizer's int8
bytes and fp32 scale bit-identical; the dequantizer bit-identical (one IEEE fp32
multiply on both sides).  Full-size configs are checked on sampled rows the
oracle computes one by one, in the launch configuration bench.py times.
"""
from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - collected on CPU boxes too
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2604_25306_b200 as qf  # noqa: E402
from paper_2604_25306_b200 import _lib  # noqa: E402
from paper_2604_25306_b200.inputs import (CATALOG, gen_int8_qkv, gen_real_qkv,  # noqa: E402
                                          gen_workload)


def _dev(*arrs):
    return [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in arrs]


def _gpu_attention(q, k, v, sq, sk, sv=0.03, block_kv=128, variant="auto"):
    dq, dk, dv = _dev(q, k, v)
    out, s_o = qf.qflash_attention_int8(dq, dk, dv, sq, sk, sv, block_kv=block_kv, variant=variant)
    torch.cuda.synchronize()
    assert s_o == np.float32(sv)
    return out.cpu().numpy()


# ------------------------------------------------------------------ edge grid
N_GRID = [1, 2, 31, 32, 33, 48, 49, 50, 63, 64, 65, 127, 128, 129, 196, 197, 255, 256, 257]


def _config_fits(D, BC, NSEG, CS, QT):
    """Mirror of config_fits<> in qflash_attn_kernel.cuh (TMEM columns, columns per
    thread, shared memory)."""
    nums = 2 if (QT == 1 and 2 * BC + D + 16 <= 512) else 1
    smem = (QT * (2 * NSEG * 128 * D + 2 * 2 * NSEG * BC * D) + BC * D + 64 * 10
            + QT * 2 * CS * 512 + 5120 + 640 + 2048)
    cw_ok = BC // CS in (16, 32, 64) or (CS == 1 and BC == 128)
    return (QT * (nums * BC + D + 16) <= 512 and cw_ok and (D // CS) % 8 == 0
            and NSEG * (BC // 4) <= BC and smem <= 227 * 1024)


def _packable(N, d, bkv):
    """Mirror of qflash_host.cu: the row-packed tiling needs <= 4 problems per
    128-row tile and an instantiated (d, B_c, NSEG) kernel in either configuration."""
    if N < 2:
        return False
    bc = (64 if N <= 64 else 128 if N <= 128 else 256) if N <= bkv else bkv
    seg = (N + 126) // N + 1
    if seg > 4:
        return False
    nseg = 2 if seg <= 2 else 4
    return any(_config_fits(d, bc, nseg, cs, qt) for cs, qt in ((4, 1), (2, 2), (1, 2), (1, 1)))


@pytest.mark.parametrize("N", N_GRID)
@pytest.mark.parametrize("d", [32, 64, 128])
def test_edge_seq_lengths(orc, N, d):
    q, k, v = gen_int8_qkv(3, N, d, seed=N + d)
    for bkv in (64, 128, 256):
        ref = orc.attention(q, k, v, 0.05, 0.05, block_kv=bkv)
        got = _gpu_attention(q, k, v, 0.05, 0.05, block_kv=bkv, variant="generic")
        assert np.array_equal(got, ref), (N, d, bkv, int((got != ref).sum()))
        if _packable(N, d, bkv):
            got_p = _gpu_attention(q, k, v, 0.05, 0.05, block_kv=bkv, variant="packed")
            assert np.array_equal(got_p, ref), (N, d, bkv, int((got_p != ref).sum()))
        else:
            with pytest.raises(_lib.QFlashError) as e:
                _gpu_attention(q, k, v, 0.05, 0.05, block_kv=bkv, variant="packed")
            assert e.value.status == _lib.QFLASH_ERR_UNSUPPORTED_SHAPE


@pytest.mark.parametrize("N,d,P", [(43, 32, 61), (49, 32, 97), (49, 64, 40), (64, 32, 33),
                                   (100, 64, 29), (127, 32, 7), (197, 64, 151), (300, 64, 9),
                                   (1025, 64, 3)])
def test_row_packed_alignments(orc, N, d, P):
    # many problems: tiles start at every residue of 128 t mod N, span 1..4
    # segments, and (P N / 128 > 148 for some shapes) CTAs walk several tiles
    q, k, v = gen_int8_qkv(P, N, d, seed=N * 7 + P)
    for bkv in (64, 128):
        if not _packable(N, d, bkv):
            continue
        ref = orc.attention(q, k, v, 0.05, 0.05, block_kv=bkv)
        got = _gpu_attention(q, k, v, 0.05, 0.05, block_kv=bkv, variant="packed")
        bad = np.argwhere((got != ref).any(axis=2))
        assert bad.size == 0, (N, d, P, bkv, bad[:8].tolist())


@pytest.mark.parametrize("kind", ["uniform", "all_min", "constant_rows", "one_hot", "ties", "zeros"])
@pytest.mark.parametrize("N,d", [(197, 64), (49, 32), (1025, 64), (300, 128)])
def test_adversarial_sets(orc, kind, N, d):
    q, k, v = gen_int8_qkv(2, N, d, seed=11, kind=kind)
    for (sq, sk) in [(0.05, 0.05), (0.003, 0.004), (0.2, 0.25)]:
        ref = orc.attention(q, k, v, sq, sk, block_kv=128)
        got = _gpu_attention(q, k, v, sq, sk, block_kv=128)
        assert np.array_equal(got, ref), (kind, sq, int((got != ref).sum()))


def _fp32_scale_for(s, d):
    """The largest fp32 s_q = s_k whose s = s_q s_k log2(e) / sqrt(d) (fp64, the
    library's and the oracle's expression) is <= the target: the ABI's end points
    2^-24 and 0.5 are reached from inside (never skipped)."""
    sq = np.float32(np.sqrt(s * np.sqrt(d) / 1.4426950408889634))
    for _ in range(64):
        if float(sq) * float(sq) * 1.4426950408889634 / np.sqrt(d) <= s:
            break
        sq = np.nextafter(sq, np.float32(0))
    return float(sq)


@pytest.mark.parametrize("s", [2.0 ** -24 * 1.01, 1e-6, 3e-5, 2e-4, 1e-3, 7.7e-3, 0.05, 0.3, 0.5])
def test_scale_range(orc, s):
    # sweep s = s_q s_k log2e / sqrt(d) over the ABI range: exercises the fast and
    # general quotient magics, p_pre > 0 (large s) and the 127 clamp; s = 0.5 is the
    # upper end point itself (s_inv = 2).
    d = 64
    sq = _fp32_scale_for(s, d)
    p = qf.qflash_derive_params(sq, sq, d)        # must be inside the range
    assert p["s"] <= s and p["s"] >= s * (1 - 1e-6)
    if s == 0.5:
        assert p["s_inv"] == 2
    q, k, v = gen_int8_qkv(2, 197, d, seed=3)
    ref = orc.attention(q, k, v, sq, sq, block_kv=64)
    got = _gpu_attention(q, k, v, sq, sq, block_kv=64)
    assert np.array_equal(got, ref)


# Every kernel configuration (qflash_attn_inst.cuh: cfg 0 CS4xQT1, 1 CS2xQT2, 2 row
# owner + correction x QT2, 3 row owner x QT1) forced through the debug ABI on a
# representative subset: generic and row-packed tiles, ragged KV tiles, T_c = 1 and
# T_c = 9, d = 32 / 64 / 128, multi-wave grids, the fused one-launch step.
CFG_CASES = [(3, 197, 64, 128, "generic"), (3, 197, 64, 128, "packed"), (3, 197, 64, 64, "generic"),
             (97, 49, 32, 128, "packed"), (40, 49, 64, 128, "generic"), (3, 1025, 64, 128, "generic"),
             (2, 257, 128, 128, "generic"), (400, 197, 64, 128, "packed"), (5, 300, 64, 256, "generic")]


def _real_codes(orc, P, N, d, seed):
    # int8 codes with the paper-like distribution: the shared generator's fp32
    # workload quantized by the oracle (no input comes from the CUDA path)
    return [orc.quantize(x)[0] for x in gen_real_qkv(P, N, d, seed=seed)]


@pytest.mark.parametrize("cfg", [0, 1, 2, 3])
@pytest.mark.parametrize("P,N,d,bkv,variant", CFG_CASES)
def test_forced_configuration(orc, cfg, P, N, d, bkv, variant):
    if cfg % 2:
        q, k, v = gen_int8_qkv(P, N, d, seed=P + N + cfg, kind="uniform")
    else:
        q, k, v = _real_codes(orc, P, N, d, seed=P + N + cfg)
    ref = orc.attention(q, k, v, 0.05, 0.04, block_kv=bkv, nthreads=8)
    _lib.force_config(cfg)
    try:
        got = _gpu_attention(q, k, v, 0.05, 0.04, block_kv=bkv, variant=variant)
        ran, nseg = _lib.last_config()
    finally:
        _lib.force_config(-1)
    assert (nseg > 1) == (variant == "packed")
    # a configuration without an instantiation for this shape falls back to the heuristic
    if ran != cfg:
        assert not _config_fits(d, bkv if N > bkv else (64 if N <= 64 else 128 if N <= 128 else 256),
                                nseg, *{0: (4, 1), 1: (2, 2), 2: (1, 2), 3: (1, 1)}[cfg])
    assert np.array_equal(got, ref), (cfg, ran, int((got != ref).sum()))


@pytest.mark.parametrize("cfg", [0, 1, 2, 3])
@pytest.mark.parametrize("name,batch", [("A3", 8), ("A4", 1), ("A1", 1)])
def test_forced_configuration_fused_step(orc, cfg, name, batch):
    q, k, v = gen_workload(name, batch, seed=cfg)
    P, N, d = q.shape
    _lib.force_config(cfg)
    try:
        y = qf.QFlashPipeline(P, N, d, mode="fused")(*_dev(q, k, v))
        torch.cuda.synchronize()
        ran, _ = _lib.last_config()
    finally:
        _lib.force_config(-1)
    assert ran == cfg
    qq, sq = orc.quantize(q)
    kq, sk = orc.quantize(k)
    vq, sv = orc.quantize(v)
    ref = orc.dequantize(orc.attention(qq, kq, vq, sq, sk, block_kv=128, nthreads=8), sv)
    assert np.array_equal(y.cpu().numpy().view(np.uint32), ref.view(np.uint32))


def test_p_clamp_regime(orc):
    # s = 0.34: s_inv = 3 and s * s_inv = 1.02, so P = floor(y M_P / 2^r_P) reaches
    # 129 at y = s_inv before the 127 clamp of reading R8.
    sq = float(np.sqrt(0.34 * np.sqrt(32) / 1.4426950408889634))
    p = qf.qflash_derive_params(sq, sq, 32)
    assert p["s_inv"] == 3 and p["p_max"] > 127
    q, k, v = gen_int8_qkv(2, 97, 32, seed=5)
    ref = orc.attention(q, k, v, sq, sq, block_kv=64)
    got = _gpu_attention(q, k, v, sq, sq, block_kv=64)
    assert np.array_equal(got, ref)


# ------------------------------------------------------------------ workloads
@pytest.mark.parametrize("name,batch", [("A1", 1), ("A2", 1), ("A3", 1), ("A4", 1), ("A5", 1),
                                        ("A6", 1), ("A7", 1), ("A2", 8), ("A7", 8),
                                        ("SwinB-s3", 1), ("SwinB-s4", 8)])
def test_workload_parity(orc, name, batch):
    q, k, v = gen_workload(name, batch, seed=0)
    qq, sq = orc.quantize(q)
    kq, sk = orc.quantize(k)
    vq, sv = orc.quantize(v)
    ref = orc.attention(qq, kq, vq, sq, sk, block_kv=128, nthreads=8)
    got = _gpu_attention(qq, kq, vq, sq, sk, sv, block_kv=128)
    assert np.array_equal(got, ref)


def test_full_size_a3_b8_exact(orc):
    # BASELINE configs[1] at full size, every element (the oracle takes ~1 s).
    q, k, v = gen_workload("A3", 8, seed=0)
    qq, sq = orc.quantize(q)
    kq, sk = orc.quantize(k)
    vq, sv = orc.quantize(v)
    ref = orc.attention(qq, kq, vq, sq, sk, block_kv=128, nthreads=8)
    got = _gpu_attention(qq, kq, vq, sq, sk, sv)
    assert np.array_equal(got, ref)


def test_full_size_swin_b8_exact(orc):
    for name in ("A4", "SwinB-s1"):
        q, k, v = gen_workload(name, 8, seed=0)
        qq, sq = orc.quantize(q)
        kq, sk = orc.quantize(k)
        vq, sv = orc.quantize(v)
        ref = orc.attention(qq, kq, vq, sq, sk, block_kv=128, nthreads=8)
        got = _gpu_attention(qq, kq, vq, sq, sk, sv)
        assert np.array_equal(got, ref)


def test_full_size_l14_b64_sampled(orc):
    # configs[4] at full size (1024 problems x 1025 tokens): sampled rows.
    w = CATALOG["L14"]
    P = w.problems(64)
    q, k, v = gen_real_qkv(P, w.seq_len, w.head_dim, seed=0)
    qq, sq = orc.quantize(q)
    kq, sk = orc.quantize(k)
    vq, sv = orc.quantize(v)
    got = _gpu_attention(qq, kq, vq, sq, sk, sv)
    rng = np.random.default_rng(0)
    for p in list(rng.integers(0, P, 6)) + [0, P - 1]:
        for (a, b) in [(0, 3), (126, 130), (1020, 1025)]:
            ref = orc.attention_rows(qq, kq, vq, sq, sk, int(p), a, b)
            assert np.array_equal(got[p, a:b], ref), (p, a)


@pytest.mark.parametrize("d,kind", [(64, "uniform"), (64, "all_min"), (128, "uniform")])
def test_maximum_sequence_length_sampled(orc, d, kind):
    # N = 65536, the ABI maximum: |O| <= 128 * 127 * N stays below 2^31 and the
    # release / normaliser paths see their largest l; rows sampled at tile edges
    N = 65536
    q, k, v = gen_int8_qkv(1, N, d, seed=5, kind=kind)
    for (sq, sk) in [(0.05, 0.05), (0.004, 0.003)]:
        got = _gpu_attention(q, k, v, sq, sk, block_kv=128)
        for (a, b) in [(0, 2), (127, 129), (32767, 32769), (N - 2, N)]:
            ref = orc.attention_rows(q, k, v, sq, sk, 0, a, b)
            assert np.array_equal(got[0, a:b], ref), (d, kind, sq, a)


def test_empty_inputs():
    # zero elements: the quantizer is a no-op; an attention call with no problems or
    # no tokens is rejected before any launch (QFLASH_ERR_UNSUPPORTED_SHAPE)
    x = torch.zeros(0, dtype=torch.float32, device="cuda")
    xq = torch.zeros(0, dtype=torch.int8, device="cuda")
    _, sc = qf.qflash_quantize_per_tensor(x, out=xq)
    torch.cuda.synchronize()
    assert sc.item() == np.float32(1.0 / 127.0)  # amax of the empty set is 0 (R3)
    for shape in [(0, 197, 64), (3, 0, 64)]:
        q = torch.zeros(shape, dtype=torch.int8, device="cuda")
        with pytest.raises(_lib.QFlashError) as e:
            qf.qflash_attention_int8(q, q, q, 0.05, 0.05, 0.05)
        assert e.value.status == _lib.QFLASH_ERR_UNSUPPORTED_SHAPE


def test_full_size_l14_b64_fused_step_sampled(orc):
    # configs[4] through the one-launch fused step (the bench's default step form):
    # codes, scales and sampled rows of the fp32 output against the oracle
    w = CATALOG["L14"]
    P = w.problems(64)
    q, k, v = gen_real_qkv(P, w.seq_len, w.head_dim, seed=1)
    pipe = qf.QFlashPipeline(P, w.seq_len, w.head_dim, mode="fused")
    y = pipe(*_dev(q, k, v))
    torch.cuda.synchronize()
    assert int(pipe.workspace[0].item()) == 0
    qq, sq = orc.quantize(q)
    kq, sk = orc.quantize(k)
    vq, sv = orc.quantize(v)
    assert [pipe.scales[i].item() for i in range(3)] == [np.float32(x) for x in (sq, sk, sv)]
    for t, ref in enumerate((qq, kq, vq)):
        assert np.array_equal(pipe.qkv_q[t].cpu().numpy(), ref)
    got = y.cpu().numpy()
    rng = np.random.default_rng(1)
    for p in list(rng.integers(0, P, 5)) + [0, P - 1]:
        for (a, b) in [(0, 2), (127, 129), (1023, 1025)]:
            o = orc.attention_rows(qq, kq, vq, sq, sk, int(p), a, b)
            ref = orc.dequantize(o, sv)
            assert np.array_equal(got[p, a:b].view(np.uint32), ref.view(np.uint32)), (p, a)


# ------------------------------------------------------------------ quantizer
@pytest.mark.parametrize("n", [1, 3, 16, 1000, 4099, 1 << 20, 1_210_368])
@pytest.mark.parametrize("dtype", ["f32", "bf16", "f16"])
def test_quantizer_bit_exact(orc, n, dtype):
    rng = np.random.default_rng(n)
    x = (rng.standard_normal(n) * 2.5).astype(np.float32)
    if dtype == "f32":
        xt = torch.from_numpy(x).cuda()
        ref_in = x
    elif dtype == "bf16":
        xt = torch.from_numpy(x).to(torch.bfloat16).cuda()
        ref_in = xt.cpu().view(torch.int16).numpy().view(np.uint16)
    else:
        xt = torch.from_numpy(x).to(torch.float16).cuda()
        ref_in = xt.cpu().float().numpy()   # f16 -> f32 widening is exact
    xq, s = qf.qflash_quantize_per_tensor(xt)
    rq, rs = orc.quantize(ref_in)
    assert np.float32(s.item()).view(np.uint32) == np.float32(rs).view(np.uint32)
    assert np.array_equal(xq.cpu().numpy(), rq)


@pytest.mark.parametrize("amax", [1e-38, 3e-40, 1e-44])
def test_quantizer_subnormal_scale(orc, amax):
    # s = fl32(amax / 127) subnormal: r = 1/s overflows to +Inf below 2^-128, so every
    # element must take the exact IEEE-division path; amax <= 127 2^-150
    # underflows s to 0 -> s = 1/127 (R3).  Codes and scale equal the oracle's.
    rng = np.random.default_rng(7)
    x = (rng.uniform(-1.0, 1.0, 4099) * amax).astype(np.float32)
    x[0] = np.float32(amax)
    x[1:4] = [0.0, np.float32(amax) / 2, -np.float32(amax) / 2]
    rq, rs = orc.quantize(x)
    xq, s = qf.qflash_quantize_per_tensor(torch.from_numpy(x).cuda())
    assert np.float32(s.item()).view(np.uint32) == np.float32(rs).view(np.uint32)
    assert np.array_equal(xq.cpu().numpy(), rq)
    # the fused step's prologue quantizer (Q subnormal; K, V normal: s stays in range
    # only for the codes -- the attention rejects s < 2^-24, so compare codes only)
    q = x[:4096].reshape(2, 32, 64)
    k = np.ones_like(q)
    codes = [torch.empty(q.shape, dtype=torch.int8, device="cuda") for _ in range(3)]
    ws = torch.zeros(_lib.DSCALE_WORKSPACE_BYTES // 4, dtype=torch.int32, device="cuda")
    sc = torch.empty(3, dtype=torch.float32, device="cuda")
    qf.qflash_forward_fused(*_dev(q, k, k), codes=codes, scales=sc, workspace=ws)
    torch.cuda.synchronize()
    fq, fs = orc.quantize(q)
    assert np.float32(sc[0].item()).view(np.uint32) == np.float32(fs).view(np.uint32)
    assert np.array_equal(codes[0].cpu().numpy(), fq)
    # the device-derived status equals the oracle's verdict on (s_q, s_k): out of range
    # for a subnormal s_q, in range when s_q underflowed to 0 and became 1/127 (R3)
    try:
        orc.derive_params(float(fs), float(orc.quantize(k)[1]), 64)
        want = 0
    except ValueError:
        want = _lib.QFLASH_ERR_SCALE_RANGE
    assert int(ws[0].item()) == want


def test_quantizer_zero_and_ties(orc):
    z = torch.zeros(1001, device="cuda")
    xq, s = qf.qflash_quantize_per_tensor(z)
    assert s.item() == np.float32(1 / 127) and not xq.any()
    x = torch.tensor([127.0, 2.5, -2.5, 0.5, -0.5, 1.5, -127.0, 126.5] * 3, device="cuda")
    xq, s = qf.qflash_quantize_per_tensor(x)
    assert s.item() == 1.0
    assert xq.cpu().tolist()[:8] == [127, 3, -3, 1, -1, 2, -127, 127]


def test_quantizer_near_half_integers(orc):
    # values whose quotient x / s lies within a few ulps of k + 1/2: exercises the
    # exact slow path of the quantizer's rounding (quant_one) -- bit-exact vs the
    # oracle's IEEE division + roundf (readings R1, R2).
    s = np.float32(100.0) / np.float32(127.0)
    vals = [np.float32(100.0)]
    for k in range(-127, 127):
        c = np.float32((k + 0.5) * float(s))
        v = c
        for _ in range(4):
            v = np.nextafter(v, np.float32(-np.inf))
        for _ in range(9):
            vals.append(v)
            v = np.nextafter(v, np.float32(np.inf))
    x = np.array(vals, np.float32)
    x = x[np.abs(x) <= 100.0]
    xq, sg = qf.qflash_quantize_per_tensor(torch.from_numpy(x).cuda())
    rq, rs = orc.quantize(x)
    assert np.float32(sg.item()) == np.float32(rs) == s
    assert np.array_equal(xq.cpu().numpy(), rq)


def test_prepare_path_constants_and_output(orc):
    q, k, v = (torch.from_numpy(a).cuda() for a in gen_workload("A2", 1, seed=6))
    qq, kq, vq, scales, ws = qf.qflash_quantize_qkv_prepare(q, k, v)
    out = qf.qflash_attention_int8_prepared(qq, kq, vq, ws)
    torch.cuda.synchronize()
    s = scales.cpu().numpy()
    hp = qf.qflash_derive_params(float(s[0]), float(s[1]), 64)
    w = ws.cpu().numpy()
    assert w[0] == 0 and w[1] == hp["s_inv"] and np.uint32(w[2]) == hp["q_magic"]
    assert w[3] == hp["q_shift"] and np.uint32(w[4]) == hp["p_mul"] and w[5] == hp["p_pre"]
    ref, _ = qf.qflash_attention_int8(qq, kq, vq, float(s[0]), float(s[1]), float(s[2]))
    assert torch.equal(out, ref)


def test_quantize_qkv_matches_single(orc):
    q, k, v = (torch.from_numpy(a).cuda() for a in gen_workload("A2", 8, seed=3))
    qq, kq, vq, scales = qf.qflash_quantize_qkv(q, k, v)
    for t, tq, s in zip((q, k, v), (qq, kq, vq), scales.cpu().numpy()):
        rq, rs = orc.quantize(t.cpu().numpy())
        assert np.float32(s) == np.float32(rs)
        assert np.array_equal(tq.cpu().numpy(), rq)


def test_dequantizer_bit_exact(orc):
    rng = np.random.default_rng(9)
    xq = rng.integers(-128, 128, size=100_003).astype(np.int8)
    s = np.float32(0.0123)
    got = qf.qflash_dequantize(torch.from_numpy(xq).cuda(), float(s)).cpu().numpy()
    assert np.array_equal(got.view(np.uint32), orc.dequantize(xq, float(s)).view(np.uint32))
    st = torch.tensor([s], device="cuda")
    got2 = qf.qflash_dequantize(torch.from_numpy(xq).cuda(), st).cpu().numpy()
    assert np.array_equal(got2, got)


# ------------------------------------------------------------------ device-scale path
def test_dscale_matches_host_scales(orc):
    q, k, v = gen_workload("A3", 1, seed=4)
    qt, kt, vt = _dev(q, k, v)
    qq, kq, vq, scales = qf.qflash_quantize_qkv(qt, kt, vt)
    out, ws = qf.qflash_attention_int8_dscale(qq, kq, vq, scales)
    torch.cuda.synchronize()
    assert int(ws[0].item()) == 0
    s = scales.cpu().numpy()
    ref_host, _ = qf.qflash_attention_int8(qq, kq, vq, float(s[0]), float(s[1]), float(s[2]))
    assert torch.equal(out, ref_host)
    # device-derived constants equal the host-derived ones
    hp = qf.qflash_derive_params(float(s[0]), float(s[1]), 64)
    wsn = ws.cpu().numpy()
    assert wsn[1] == hp["s_inv"] and wsn[2] == np.int32(np.uint32(hp["q_magic"]))


def test_dscale_out_of_range_writes_nothing():
    q = torch.zeros((1, 64, 64), dtype=torch.int8, device="cuda")
    scales = torch.tensor([10.0, 10.0, 1.0], device="cuda")    # s = 18 > 0.5
    out = torch.full_like(q, 77)
    _, ws = qf.qflash_attention_int8_dscale(q, q.clone(), q.clone(), scales, out=out)
    torch.cuda.synchronize()
    assert int(ws[0].item()) == _lib.QFLASH_ERR_SCALE_RANGE
    assert (out == 77).all()


def test_pipeline_end_to_end_bit_exact(orc):
    # float -> quantize -> attention -> dequantize, all on the GPU, vs the oracle
    q, k, v = gen_workload("A1", 1, seed=7)
    out = qf.qflash_forward(torch.from_numpy(q), torch.from_numpy(k), torch.from_numpy(v))
    qq, sq = orc.quantize(q)
    kq, sk = orc.quantize(k)
    vq, sv = orc.quantize(v)
    ref = orc.dequantize(orc.attention(qq, kq, vq, sq, sk), sv)
    assert np.array_equal(out.numpy().view(np.uint32), ref.view(np.uint32))


@pytest.mark.parametrize("name,batch", [("A1", 1), ("A3", 8), ("A4", 8), ("A7", 1), ("SwinB-s3", 8),
                                        ("SwinB-s2", 8), ("SwinB-s1", 8)])
def test_fused_step_and_dequant_epilogue_bit_exact(orc, name, batch):
    # quantize_prepare -> attention with the DQ step fused into the epilogue (fp32 bits from
    # the quantizer's table) == oracle dequantize(attention(quantize)) == the 3-stage path
    q, k, v = gen_workload(name, batch, seed=5)
    P, N, d = q.shape
    dq, dk, dv = _dev(q, k, v)
    fused = qf.QFlashPipeline(P, N, d, mode="two")
    staged = qf.QFlashPipeline(P, N, d, mode="three")
    one = qf.QFlashPipeline(P, N, d, mode="fused")
    y_f = fused(dq, dk, dv).clone()
    y_s = staged(dq, dk, dv).clone()
    y_1 = one(dq, dk, dv).clone()
    o8_1 = torch.empty((P, N, d), dtype=torch.int8, device="cuda")
    y_1b = qf.qflash_forward_fused(dq, dk, dv, out_int8=o8_1)
    o8 = torch.empty((P, N, d), dtype=torch.int8, device="cuda")
    y_b = qf.qflash_attention_dequant_prepared(fused.qkv_q[0], fused.qkv_q[1], fused.qkv_q[2],
                                               fused.workspace, out_int8=o8)
    torch.cuda.synchronize()
    qq, sq = orc.quantize(q)
    kq, sk = orc.quantize(k)
    vq, sv = orc.quantize(v)
    o_ref = orc.attention(qq, kq, vq, sq, sk, block_kv=128)
    ref = orc.dequantize(o_ref, sv)
    for y in (y_f, y_s, y_b, y_1, y_1b):
        assert np.array_equal(y.cpu().numpy().view(np.uint32), ref.view(np.uint32))
    assert np.array_equal(o8.cpu().numpy(), o_ref)
    assert np.array_equal(o8_1.cpu().numpy(), o_ref)
    for t, (xq, sx) in enumerate(((qq, sq), (kq, sk), (vq, sv))):  # the prologue's codes and scales
        assert np.array_equal(one.qkv_q[t].cpu().numpy(), xq)
        assert one.scales[t].item() == np.float32(sx)
    assert int(one.workspace[0].item()) == 0


def test_sqnr_floor_on_gpu_output(orc):
    from oracle.fp_reference import attention_fp64, sqnr_db
    for name, batch in [("A2", 8), ("A7", 8)]:
        q, k, v = gen_workload(name, batch, seed=0)
        out = qf.qflash_forward(torch.from_numpy(q), torch.from_numpy(k), torch.from_numpy(v))
        assert sqnr_db(attention_fp64(q, k, v), out.numpy()) >= 29.0   # > I-ViT's 25.8


# ------------------------------------------------------------------ properties
def test_determinism_and_independence(orc):
    q, k, v = gen_int8_qkv(16, 197, 64, seed=8)
    a = _gpu_attention(q, k, v, 0.05, 0.05)
    b = _gpu_attention(q, k, v, 0.05, 0.05)
    assert np.array_equal(a, b)
    for p in (0, 7, 15):
        one = _gpu_attention(q[p:p + 1], k[p:p + 1], v[p:p + 1], 0.05, 0.05)
        assert np.array_equal(one[0], a[p])


def test_validation_errors():
    q = torch.zeros((2, 197, 64), dtype=torch.int8, device="cuda")
    with pytest.raises(_lib.QFlashError) as e:
        qf.qflash_attention_int8(q, q, q, 10.0, 10.0, 1.0)        # s > 0.5
    assert e.value.status == _lib.QFLASH_ERR_SCALE_RANGE
    with pytest.raises(_lib.QFlashError) as e:
        qf.qflash_attention_int8(q, q, q, 0.05, 0.05, 0.05, out=q)  # aliasing
    assert e.value.status == _lib.QFLASH_ERR_INVALID_ARGUMENT
    with pytest.raises(_lib.QFlashError) as e:
        qf.qflash_attention_int8(q, q, q, 0.05, 0.05, 0.05, block_kv=96)
    assert e.value.status == _lib.QFLASH_ERR_UNSUPPORTED_SHAPE
    q48 = torch.zeros((2, 197, 48), dtype=torch.int8, device="cuda")
    with pytest.raises(_lib.QFlashError) as e:
        qf.qflash_attention_int8(q48, q48, q48, 0.05, 0.05, 0.05)
    assert e.value.status == _lib.QFLASH_ERR_UNSUPPORTED_SHAPE
    q1 = torch.zeros((4, 20, 64), dtype=torch.int8, device="cuda")
    with pytest.raises(_lib.QFlashError):
        qf.qflash_attention_int8(q1, q1, q1, 0.05, 0.05, 0.05, variant="packed")  # N < 43


def test_host_pipeline_overlapped_batches(orc):
    # the serving loop: pinned host batches, two buffer sets / streams overlapping
    # copies and compute; every batch's output equals the oracle's
    batches = [gen_workload("A2", 1, seed=s) for s in (21, 22, 23)]
    P, N, d = batches[0][0].shape
    hp = qf.QFlashHostPipeline(P, N, d)
    outs = [torch.empty((P, N, d), dtype=torch.float32).pin_memory() for _ in batches]
    for (q, k, v), o in zip(batches, outs):
        hp(*(torch.from_numpy(x).pin_memory() for x in (q, k, v)), o)
    hp.synchronize()
    for (q, k, v), o in zip(batches, outs):
        qq, sq = orc.quantize(q)
        kq, sk = orc.quantize(k)
        vq, sv = orc.quantize(v)
        ref = orc.dequantize(orc.attention(qq, kq, vq, sq, sk), sv)
        assert np.array_equal(o.numpy().view(np.uint32), ref.view(np.uint32))


# ------------------------------------------------------- per-head granularity (N1)
def _head_spread(q, k, v, H, spread=1.5):
    gains = np.exp(np.linspace(-spread, spread, H)).astype(np.float32)
    g = np.tile(gains, q.shape[0] // H)[:, None, None]
    return q * g, k * g, v * g


@pytest.mark.parametrize("name,batch,H", [("A1", 1, 3), ("A3", 8, 12), ("A4", 8, 3),
                                          ("SwinB-s3", 1, 16), ("L14", 1, 16)])
def test_per_head_path_bit_exact(orc, name, batch, H):
    q, k, v = _head_spread(*gen_workload(name, batch, seed=3), H)
    dq, dk, dv = _dev(q, k, v)
    y, o, scales, ws = qf.qflash_forward_per_head(dq, dk, dv, H)
    torch.cuda.synchronize()
    assert int(ws[0].item()) == 0
    qh, sq = orc.quantize_per_head(q, H)
    kh, sk = orc.quantize_per_head(k, H)
    vh, sv = orc.quantize_per_head(v, H)
    assert np.array_equal(scales.cpu().numpy(), np.concatenate([sq, sk, sv]))
    o_ref = orc.attention_per_head(qh, kh, vh, sq, sk, H, nthreads=8)
    assert np.array_equal(o.cpu().numpy(), o_ref)
    ref = orc.dequantize_per_head(o_ref, sv, H)
    assert np.array_equal(y.cpu().numpy().view(np.uint32), ref.view(np.uint32))


def test_per_head_one_head_equals_per_tensor(orc):
    q, k, v = gen_workload("A2", 1, seed=4)
    dq, dk, dv = _dev(q, k, v)
    y, _, _, _ = qf.qflash_forward_per_head(dq, dk, dv, 1)
    y_t = qf.qflash_forward(dq, dk, dv)
    torch.cuda.synchronize()
    assert torch.equal(y.view(torch.int32), y_t.view(torch.int32))


@pytest.mark.parametrize("d", [32, 64, 128])
def test_device_constants_equal_host_constants(d):
    # the device derivation (derive_core on the GPU: fp64 with explicit rounding,
    # 64-bit magics, sqrt(d) constants) equals the host's field by field
    rng = np.random.default_rng(d)
    q = torch.zeros((1, 2, d), dtype=torch.int8, device="cuda")
    for _ in range(24):
        sq, sk = (float(np.float32(10.0 ** rng.uniform(-3.6, -0.4))) for _ in range(2))
        try:
            hp = qf.qflash_derive_params(sq, sk, d)
        except _lib.QFlashError:
            continue
        scales = torch.tensor([sq, sk, 0.05], dtype=torch.float32, device="cuda")
        _, ws = qf.qflash_attention_int8_dscale(q, q, q, scales)
        torch.cuda.synchronize()
        w = ws.cpu().numpy()
        s_dev = ws[16:18].cpu().numpy().view(np.float64)[0]
        rel = (int(np.uint32(w[7])) << 32) | int(np.uint32(w[6]))
        assert (w[0], w[1], np.uint32(w[2]), w[3], np.uint32(w[4]), w[5]) == (
            0, hp["s_inv"], hp["q_magic"], hp["q_shift"], hp["p_mul"], hp["p_pre"])
        assert (rel, w[8], w[9], w[10], w[11], w[12]) == (
            hp["rel_magic"], hp["rel_shift"], hp["p_max"], hp["r_p"], hp["m_p"], hp["n"])
        assert s_dev == hp["s"]


# ------------------------------------------------ sharded quantization
@pytest.mark.parametrize("name,batch,world", [("A3", 8, 2), ("A1", 8, 3), ("A4", 1, 4), ("L14", 2, 2)])
def test_sharded_fused_step_equals_single_gpu(orc, name, batch, world):
    # Strong scaling of ONE logical batch: every "rank" (here: a slab on the same GPU)
    # takes qflash_partition's contiguous problem range, computes its local amax
    # (qflash_amax_qkv), the MAX all-reduce is emulated by torch.maximum, and
    # qflash_forward_fused_amax quantizes with the global scales.  The concatenated
    # slab outputs are byte-identical to the 1-GPU fused step on the whole batch, and
    # the codes / scales to the oracle's quantizer.
    q, k, v = gen_workload(name, batch, seed=11)
    P = q.shape[0]
    dq, dk, dv = _dev(q, k, v)
    full = qf.qflash_forward_fused(dq, dk, dv).cpu().numpy()
    slabs = [qf.qflash_partition(P, world, r) for r in range(world)]
    amax = torch.zeros(3, device="cuda")
    for b, c in slabs:
        if c:
            amax = torch.maximum(amax, qf.qflash_amax_qkv(dq[b:b + c], dk[b:b + c], dv[b:b + c]))
    ref_amax = [np.float32(np.abs(x).max()) for x in (q, k, v)]
    assert [np.float32(x) for x in amax.cpu().numpy()] == ref_amax
    out = np.empty_like(full)
    for b, c in slabs:
        if not c:
            continue
        codes = [torch.empty((c,) + q.shape[1:], dtype=torch.int8, device="cuda") for _ in range(3)]
        sc = torch.empty(3, dtype=torch.float32, device="cuda")
        y = qf.qflash_forward_fused(dq[b:b + c], dk[b:b + c], dv[b:b + c], codes=codes, scales=sc,
                                    amax=amax)
        out[b:b + c] = y.cpu().numpy()
        for t, x in enumerate((q, k, v)):
            rq, rs = orc.quantize(x)
            assert np.float32(sc[t].item()).view(np.uint32) == np.float32(rs).view(np.uint32)
            assert np.array_equal(codes[t].cpu().numpy(), rq[b:b + c])
    assert np.array_equal(out.view(np.uint32), full.view(np.uint32))


def test_amax_qkv_edge_cases():
    z = torch.zeros((2, 49, 32), device="cuda")
    assert qf.qflash_amax_qkv(z, z, z).tolist() == [0.0, 0.0, 0.0]
    e = torch.zeros((0, 49, 32), device="cuda")
    assert qf.qflash_amax_qkv(e, e, e).tolist() == [0.0, 0.0, 0.0]
    x = torch.randn((3, 197, 64), device="cuda")
    x[1, 5, 7] = -1e30
    a = qf.qflash_amax_qkv(x, x * 2, -x).cpu()
    assert a.tolist() == [float(np.float32(1e30)), float(np.float32(2e30)), float(np.float32(1e30))]


# ------------------------------------------------ Scale Accumulation ablation
@pytest.mark.parametrize("N,d,bkv", [(49, 32, 64), (197, 64, 64), (197, 64, 128), (256, 64, 64),
                                     (300, 32, 64), (1025, 64, 128)])
def test_scale_accumulation_matches_oracle_mode1(orc, N, d, bkv):
    # Eq. 13 in int64 with the oracle's wrap-around, bit-exact to oracle
    # mode 1 on real-valued inputs (T_c = 1 .. 9), and the int64-overflow flag equal to
    # the oracle's; int64 overflow implies int32 overflow.
    w = "vit" if d == 64 else "swin"
    q, k, v = gen_real_qkv(3, N, d, seed=N + bkv, family=w)
    (qq, sq), (kq, sk), (vq, sv) = (orc.quantize(x) for x in (q, k, v))
    ref, ovf = orc.attention(qq, kq, vq, sq, sk, block_kv=bkv, mode=1, return_overflow=True)
    got, flags = qf.qflash_attention_int8_accum(*_dev(qq, kq, vq), sq, sk, block_kv=bkv)
    f = int(flags.item())
    assert np.array_equal(got.cpu().numpy(), ref), (N, d, bkv, int((got.cpu().numpy() != ref).sum()))
    assert bool(f & 1) == ovf
    assert not (f & 1) or (f & 2)


def test_scale_accumulation_single_tile_equals_release(orc):
    # T_c = 1: O = PV s_inv, l = rowsum s_inv -> floor(O / l) = floor(PV / rowsum), the
    # same output as Scale Release (no release ever happens); no int64 overflow
    q, k, v = gen_int8_qkv(4, 100, 64, seed=3)
    got, flags = qf.qflash_attention_int8_accum(*_dev(q, k, v), 0.05, 0.05, block_kv=128)
    rel = orc.attention(q, k, v, 0.05, 0.05, block_kv=128)
    assert np.array_equal(got.cpu().numpy(), rel)
    assert not (int(flags.item()) & 1)


# ------------------------------------------------ packed QKV projection output
def _pack_qkv(q, k, v, H):
    P, N, d = q.shape
    B = P // H
    qkv = np.empty((B, N, 3, H, d), np.float32)
    for t, x in enumerate((q, k, v)):
        qkv[:, :, t] = x.reshape(B, H, N, d).transpose(0, 2, 1, 3)
    return qkv


@pytest.mark.parametrize("name,batch", [("A1", 1), ("A3", 8), ("A4", 1), ("A7", 8), ("L14", 1)])
def test_fused_step_packed_qkv(orc, name, batch):
    # the fused step reading a [B, N, 3, H, d] projection output directly (no permute pass)
    # == the oracle on the three permuted tensors: codes, scales and fp32 output bit-exact
    w = CATALOG[name]
    q, k, v = gen_workload(name, batch, seed=21)
    H = w.heads
    qkv = torch.from_numpy(_pack_qkv(q, k, v, H)).cuda()
    codes = [torch.empty(q.shape, dtype=torch.int8, device="cuda") for _ in range(3)]
    sc = torch.empty(3, dtype=torch.float32, device="cuda")
    y = qf.qflash_forward_fused_qkv(qkv, H, codes=codes, scales=sc).cpu().numpy()
    (qq, sq), (kq, sk), (vq, sv) = (orc.quantize(x) for x in (q, k, v))
    for t, (c, s) in enumerate(((qq, sq), (kq, sk), (vq, sv))):
        assert np.array_equal(codes[t].cpu().numpy(), c)
        assert np.float32(sc[t].item()).view(np.uint32) == np.float32(s).view(np.uint32)
    ref = orc.dequantize(orc.attention(qq, kq, vq, sq, sk, block_kv=128), sv)
    assert np.array_equal(y.view(np.uint32), ref.view(np.uint32))


def test_fused_step_packed_qkv_rejects_bad_heads():
    qkv = torch.zeros((2, 49, 3, 3, 32), device="cuda")
    with pytest.raises(ValueError):
        qf.qflash_forward_fused_qkv(qkv, 4)
    shape = _lib.AttnShape(7, 49, 32, 128)
    st = _lib.lib().qflash_forward_fused_qkv(qkv.data_ptr(), 3, shape, 0, None, None, None, None, None,
                                             None, None, None)
    assert st == _lib.QFLASH_ERR_INVALID_ARGUMENT


# ------------------------------------------------ ablation steps V3 / V2
@pytest.mark.parametrize("name,batch", [("A2", 1), ("A7", 8), ("A1", 8)])
def test_ablation_variants_accuracy(orc, name, batch):
    # V3 (integer exp, FP accumulation) and V2 (FP exp2 softmax, int8 P V) are not exact:
    # both must stay in the paper's SQNR regime against FP64 attention, and V3 (same P
    # bytes as the method, exact fp32 accumulation of exact int32 P V) within a few LSB
    # of the method's dequantized output
    from oracle.fp_reference import attention_fp64, sqnr_db
    q, k, v = gen_workload(name, batch, seed=4)
    (qq, sq), (kq, sk), (vq, sv) = (orc.quantize(x) for x in (q, k, v))
    dq, dk, dv = _dev(qq, kq, vq)
    ref = attention_fp64(q, k, v)
    v4 = qf.qflash_attention_int8(dq, dk, dv, sq, sk, sv)[0].cpu().numpy().astype(np.float64) * sv
    y3 = qf.qflash_attention_ablation(dq, dk, dv, sq, sk, sv, "V3").cpu().numpy()
    y2 = qf.qflash_attention_ablation(dq, dk, dv, sq, sk, sv, "V2").cpu().numpy()
    s4, s3, s2 = sqnr_db(ref, v4), sqnr_db(ref, y3), sqnr_db(ref, y2)
    assert s3 >= 29.0 and s2 >= 29.0 and s4 >= 29.0, (s4, s3, s2)
    assert np.abs(y3 - v4).max() <= 3.0 * sv


@pytest.mark.parametrize("name,batch,H,cfg", [("L14", 2, 16, 1), ("L14", 2, 16, 0), ("A3", 8, 12, 1)])
def test_per_head_configurations(orc, name, batch, H, cfg):
    # the per-head attention in configuration 1 (two query tiles per SM, CS = 2) and 0,
    # forced, bit-exact to the oracle's per-head composition
    q, k, v = _head_spread(*gen_workload(name, batch, seed=8), H)
    dq, dk, dv = _dev(q, k, v)
    _lib.force_config(cfg)
    try:
        y, o, scales, ws = qf.qflash_forward_per_head(dq, dk, dv, H)
        torch.cuda.synchronize()
    finally:
        _lib.force_config(-1)
    qh, sq = orc.quantize_per_head(q, H)
    kh, sk = orc.quantize_per_head(k, H)
    vh, sv = orc.quantize_per_head(v, H)
    o_ref = orc.attention_per_head(qh, kh, vh, sq, sk, H, nthreads=8)
    assert np.array_equal(o.cpu().numpy(), o_ref)


@pytest.mark.parametrize("name,batch,H", [("A1", 1, 3), ("A3", 8, 12), ("A4", 8, 3), ("SwinB-s3", 1, 16),
                                          ("L14", 2, 16), ("A7", 8, 24)])
def test_fused_per_head_step_bit_exact(orc, name, batch, H):
    # the one-launch per-head step: codes, the 3H scales and y bit-exact to the oracle's
    # per-head composition, also on the second call on the same workspace
    q, k, v = _head_spread(*gen_workload(name, batch, seed=13), H)
    dq, dk, dv = _dev(q, k, v)
    codes = [torch.empty(q.shape, dtype=torch.int8, device="cuda") for _ in range(3)]
    ws = torch.zeros(_lib.PH_FUSED_WORKSPACE_BYTES // 4, dtype=torch.int32, device="cuda")
    qh, sq = orc.quantize_per_head(q, H)
    kh, sk = orc.quantize_per_head(k, H)
    vh, sv = orc.quantize_per_head(v, H)
    ref = orc.dequantize_per_head(orc.attention_per_head(qh, kh, vh, sq, sk, H, nthreads=8), sv, H)
    # call 1 on 4 Q (larger amax), call 2 on Q: stale accumulators would keep 4 amax(Q)
    for rep, x in enumerate((dq * 4.0, dq)):
        y, sc, ws = qf.qflash_forward_fused_per_head(x, dk, dv, H, codes=codes, workspace=ws)
        torch.cuda.synchronize()
        assert int(ws[0].item()) == 0
    assert np.array_equal(sc.cpu().numpy(), np.concatenate([sq, sk, sv]))
    for t, c in enumerate((qh, kh, vh)):
        assert np.array_equal(codes[t].cpu().numpy(), c)
    assert np.array_equal(y.cpu().numpy().view(np.uint32), ref.view(np.uint32))
    assert not ws[8192 // 4: 8192 // 4 + 3 * H].any()  # re-zeroed for the next call


def test_fused_per_head_one_head_equals_per_tensor():
    q, k, v = gen_workload("A2", 1, seed=4)
    dq, dk, dv = _dev(q, k, v)
    y, _, _ = qf.qflash_forward_fused_per_head(dq, dk, dv, 1)
    y_t = qf.qflash_forward(dq, dk, dv)
    torch.cuda.synchronize()
    assert torch.equal(y.view(torch.int32), y_t.view(torch.int32))


@pytest.mark.gpu
def test_pipeline_fused_fast_path_matches_and_checks():
    # QFlashPipeline's fused call marshals its own buffers once at construction; the
    # per-call path checks q, k, v itself: same bytes as qflash_forward_fused, and the
    # same rejections before anything reaches the C ABI
    w = CATALOG["A3"]
    P, N, d = w.problems(1), w.seq_len, w.head_dim
    q, k, v = _dev(*gen_real_qkv(P, N, d, seed=3))
    pipe = qf.QFlashPipeline(P, N, d, mode="fused")
    y1 = pipe(q, k, v).clone()
    y2 = qf.qflash_forward_fused(q, k, v)
    torch.cuda.synchronize()
    assert torch.equal(y1.view(torch.int32), y2.view(torch.int32))
    with pytest.raises(ValueError):
        pipe(q, k[:, :-1].contiguous(), v)                    # wrong shape
    with pytest.raises(ValueError):
        pipe(q, k, v.transpose(1, 2).contiguous().transpose(1, 2))  # not contiguous
    with pytest.raises(ValueError):
        pipe(q, k.to(torch.float16), v)                       # wrong dtype
    with pytest.raises(ValueError):
        pipe(q, k.cpu(), v)                                   # wrong device
