"""Python API over libqflash.so -- same names as the C ABI, torch tensors in/out.

PyTorch supplies device memory and the current CUDA stream only; every step of
the QFlash hot path (quantize, fused integer attention, dequantize) runs in the
library's sm_100a kernels.  There is no CPU or eager-PyTorch fallback.
"""
from __future__ import annotations

import ctypes

import torch

from . import _lib
from ._lib import AttnShape, IntParams, check, lib

_DTYPES = {torch.float32: _lib.QFLASH_F32, torch.bfloat16: _lib.QFLASH_BF16,
           torch.float16: _lib.QFLASH_F16}


def _stream(stream=None) -> ctypes.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _dev_ptr(t: torch.Tensor) -> ctypes.c_void_p:
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return ctypes.c_void_p(t.data_ptr())


def _check_like(ref: torch.Tensor, t: torch.Tensor, name: str, dtype=None) -> None:
    """t must have ref's shape (the library sizes every buffer from q's shape), the
    expected dtype and ref's device -- checked before any pointer reaches the C ABI."""
    if tuple(t.shape) != tuple(ref.shape):
        raise ValueError("%s: shape %s != %s" % (name, tuple(t.shape), tuple(ref.shape)))
    if dtype is not None and t.dtype != dtype:
        raise TypeError("%s: dtype %s, expected %s" % (name, t.dtype, dtype))
    if t.device != ref.device:
        raise ValueError("%s: device %s != %s" % (name, t.device, ref.device))


def _check_qkv(q, k, v, dtype=torch.int8) -> None:
    if q.dim() != 3:
        raise ValueError("expected [P, N, d] tensors, got %s" % (tuple(q.shape),))
    for name, t in (("q", q), ("k", k), ("v", v)):
        _check_like(q, t, name, dtype)


def _check_buffer(t: torch.Tensor, nbytes: int, name: str, device, dtype=None) -> None:
    if dtype is not None and t.dtype != dtype:
        raise TypeError("%s: dtype %s, expected %s" % (name, t.dtype, dtype))
    if t.numel() * t.element_size() < nbytes:
        raise ValueError("%s: %d bytes < %d" % (name, t.numel() * t.element_size(), nbytes))
    if t.device != device:
        raise ValueError("%s: device %s != %s" % (name, t.device, device))


def _check_workspace(ws: torch.Tensor, device) -> None:
    _check_buffer(ws, _lib.DSCALE_WORKSPACE_BYTES, "workspace", device)


def _check_scales(sc: torch.Tensor, n: int, device) -> None:
    _check_buffer(sc, 4 * n, "scales", device, torch.float32)


# ---------------------------------------------------------------- quantizer
def qflash_quantize_per_tensor(x: torch.Tensor, out: torch.Tensor | None = None,
                               scale_out: torch.Tensor | None = None, stream=None):
    """Eq. 2 per-tensor int8 quantization.  Returns (x_q int8, scale float32[1] on device)."""
    if x.dtype not in _DTYPES:
        raise TypeError(x.dtype)
    out = torch.empty(x.shape, dtype=torch.int8, device=x.device) if out is None else out
    scale_out = torch.empty(1, dtype=torch.float32, device=x.device) if scale_out is None else scale_out
    _check_like(x, out, "out", torch.int8)
    _check_scales(scale_out, 1, x.device)
    check(lib().qflash_quantize_per_tensor(_dev_ptr(x), _DTYPES[x.dtype], x.numel(), _dev_ptr(out),
                                           _dev_ptr(scale_out), None, _stream(stream)))
    return out, scale_out


def qflash_quantize_qkv(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, outs=None,
                        scales: torch.Tensor | None = None, stream=None):
    """Fused Q/K/V quantization.  Returns (q_q, k_q, v_q, scales float32[3] on device)."""
    if q.dtype not in _DTYPES:
        raise TypeError(q.dtype)
    for name, t in (("k", k), ("v", v)):
        _check_like(q, t, name, q.dtype)
    if outs is None:
        outs = [torch.empty(q.shape, dtype=torch.int8, device=q.device) for _ in range(3)]
    scales = torch.empty(3, dtype=torch.float32, device=q.device) if scales is None else scales
    for i, t in enumerate(outs):
        _check_like(q, t, "outs[%d]" % i, torch.int8)
    _check_scales(scales, 3, q.device)
    check(lib().qflash_quantize_qkv(_dev_ptr(q), _dev_ptr(k), _dev_ptr(v), _DTYPES[q.dtype],
                                    q.numel(), _dev_ptr(outs[0]), _dev_ptr(outs[1]),
                                    _dev_ptr(outs[2]), _dev_ptr(scales), _stream(stream)))
    return outs[0], outs[1], outs[2], scales


# ---------------------------------------------------------------- attention
def _shape(q: torch.Tensor, block_kv: int) -> AttnShape:
    if q.dim() != 3:
        raise ValueError("expected [P, N, d] tensors")
    P, N, d = q.shape
    return AttnShape(P, N, d, block_kv)


def qflash_attention_int8(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, s_q: float,
                          s_k: float, s_v: float, block_kv: int = 128, variant: str = "auto",
                          out: torch.Tensor | None = None, stream=None):
    """Algorithm 1 (integer-only fused attention).  int8 [P, N, d] in, (int8 out, s_O) back."""
    _check_qkv(q, k, v)
    out = torch.empty_like(q) if out is None else out
    _check_like(q, out, "out", torch.int8)
    shape = _shape(q, block_kv)
    s_o = ctypes.c_float(0.0)
    check(lib().qflash_attention_int8_ex(_dev_ptr(q), _dev_ptr(k), _dev_ptr(v), s_q, s_k, s_v,
                                         ctypes.byref(shape), _lib.VARIANTS[variant],
                                         _dev_ptr(out), ctypes.byref(s_o), _stream(stream)))
    return out, float(s_o.value)


def qflash_attention_int8_dscale(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor,
                                 scales: torch.Tensor, block_kv: int = 128, variant: str = "auto",
                                 out: torch.Tensor | None = None,
                                 workspace: torch.Tensor | None = None, stream=None):
    """Device-scale attention: scales = device float32[3] (s_q, s_k, s_v); no host sync.
    Returns (out int8, workspace) -- workspace[0] (int32) holds the status."""
    _check_qkv(q, k, v)
    out = torch.empty_like(q) if out is None else out
    if workspace is None:
        workspace = torch.empty(_lib.DSCALE_WORKSPACE_BYTES // 4, dtype=torch.int32, device=q.device)
    _check_like(q, out, "out", torch.int8)
    _check_scales(scales, 3, q.device)
    _check_workspace(workspace, q.device)
    shape = _shape(q, block_kv)
    check(lib().qflash_attention_int8_dscale(_dev_ptr(q), _dev_ptr(k), _dev_ptr(v),
                                             _dev_ptr(scales), ctypes.byref(shape),
                                             _lib.VARIANTS[variant], _dev_ptr(out),
                                             _dev_ptr(workspace), _stream(stream)))
    return out, workspace


# ---------------------------------------------------------------- dequantizer
def qflash_dequantize(x_q: torch.Tensor, scale, out: torch.Tensor | None = None, stream=None):
    """y = scale * x^ in fp32.  `scale` is a python float or a device float32 tensor."""
    if x_q.dtype != torch.int8:
        raise TypeError("x_q must be int8")
    out = torch.empty(x_q.shape, dtype=torch.float32, device=x_q.device) if out is None else out
    _check_like(x_q, out, "out", torch.float32)
    if isinstance(scale, torch.Tensor):
        _check_scales(scale, 1, x_q.device)
        check(lib().qflash_dequantize_dscale(_dev_ptr(x_q), _dev_ptr(scale), x_q.numel(),
                                             _dev_ptr(out), _stream(stream)))
    else:
        check(lib().qflash_dequantize(_dev_ptr(x_q), float(scale), x_q.numel(), _dev_ptr(out),
                                      _stream(stream)))
    return out


# ---------------------------------------------------------------- pipeline
def qflash_quantize_qkv_prepare(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, outs=None,
                                scales: torch.Tensor | None = None,
                                workspace: torch.Tensor | None = None, stream=None):
    """Fused Q/K/V quantization that also derives the attention constants on the
    device.  Returns (q_q, k_q, v_q, scales float32[3], workspace int32[32])."""
    if q.dtype not in _DTYPES:
        raise TypeError(q.dtype)
    _check_qkv(q, k, v, q.dtype)
    if outs is None:
        outs = [torch.empty(q.shape, dtype=torch.int8, device=q.device) for _ in range(3)]
    scales = torch.empty(3, dtype=torch.float32, device=q.device) if scales is None else scales
    if workspace is None:
        workspace = torch.empty(_lib.DSCALE_WORKSPACE_BYTES // 4, dtype=torch.int32, device=q.device)
    for i, t in enumerate(outs):
        _check_like(q, t, "outs[%d]" % i, torch.int8)
    _check_scales(scales, 3, q.device)
    _check_workspace(workspace, q.device)
    check(lib().qflash_quantize_qkv_prepare(_dev_ptr(q), _dev_ptr(k), _dev_ptr(v),
                                            _DTYPES[q.dtype], q.numel(), _dev_ptr(outs[0]),
                                            _dev_ptr(outs[1]), _dev_ptr(outs[2]), _dev_ptr(scales),
                                            q.shape[2], _dev_ptr(workspace), _stream(stream)))
    return outs[0], outs[1], outs[2], scales, workspace


def qflash_attention_int8_prepared(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor,
                                   workspace: torch.Tensor, block_kv: int = 128,
                                   variant: str = "auto", out: torch.Tensor | None = None,
                                   stream=None):
    """Algorithm 1 with the constants qflash_quantize_qkv_prepare left in `workspace`."""
    _check_qkv(q, k, v)
    out = torch.empty_like(q) if out is None else out
    _check_like(q, out, "out", torch.int8)
    _check_workspace(workspace, q.device)
    shape = _shape(q, block_kv)
    check(lib().qflash_attention_int8_prepared(_dev_ptr(q), _dev_ptr(k), _dev_ptr(v),
                                               ctypes.byref(shape), _lib.VARIANTS[variant],
                                               _dev_ptr(out), _dev_ptr(workspace), _stream(stream)))
    return out


def qflash_attention_dequant_prepared(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor,
                                      workspace: torch.Tensor, block_kv: int = 128,
                                      variant: str = "auto", out: torch.Tensor | None = None,
                                      out_int8: torch.Tensor | None = None, stream=None):
    """Algorithm 1 with the dequantization fused into its epilogue: fp32
    y = s_V * O^ (and optionally the int8 O^), constants and dequant table from
    `workspace` (qflash_quantize_qkv_prepare)."""
    _check_qkv(q, k, v)
    out = torch.empty(q.shape, dtype=torch.float32, device=q.device) if out is None else out
    _check_like(q, out, "out", torch.float32)
    if out_int8 is not None:
        _check_like(q, out_int8, "out_int8", torch.int8)
    _check_workspace(workspace, q.device)
    shape = _shape(q, block_kv)
    check(lib().qflash_attention_dequant_prepared(
        _dev_ptr(q), _dev_ptr(k), _dev_ptr(v), ctypes.byref(shape), _lib.VARIANTS[variant],
        _dev_ptr(out_int8) if out_int8 is not None else None, _dev_ptr(out), _dev_ptr(workspace),
        _stream(stream)))
    return out


def qflash_attention_int8_accum(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, s_q: float,
                                s_k: float, block_kv: int = 128, out: torch.Tensor | None = None,
                                stream=None):
    """Scale Accumulation ablation (Eq. 13, App. B.1 -- the paper's rejected form):
    returns (int8 O^, flags) with flags bit 0 = int64 overflow, bit 1 = int32 overflow."""
    _check_qkv(q, k, v)
    out = torch.empty_like(q) if out is None else out
    _check_like(q, out, "out", torch.int8)
    flags = torch.zeros(1, dtype=torch.int32, device=q.device)
    shape = _shape(q, block_kv)
    check(lib().qflash_attention_int8_accum(_dev_ptr(q), _dev_ptr(k), _dev_ptr(v), float(s_q),
                                            float(s_k), ctypes.byref(shape), _dev_ptr(out),
                                            _dev_ptr(flags), _stream(stream)))
    return out, flags


ABLATIONS = {"V2": 2, "V3": 3}


def qflash_attention_ablation(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, s_q: float,
                              s_k: float, s_v: float, variant: str, block_kv: int = 128,
                              out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """The paper's ablation steps on B200: "V3" integer exp + FP accumulation,
    "V2" FP exp2 softmax + int8 P V; fp32 y = s_V O / l (qflash_attention_int8 is V4)."""
    _check_qkv(q, k, v)
    out = torch.empty(q.shape, dtype=torch.float32, device=q.device) if out is None else out
    _check_like(q, out, "out", torch.float32)
    shape = _shape(q, block_kv)
    check(lib().qflash_attention_ablation(_dev_ptr(q), _dev_ptr(k), _dev_ptr(v), float(s_q), float(s_k),
                                          float(s_v), ctypes.byref(shape), ABLATIONS[variant],
                                          _dev_ptr(out), _stream(stream)))
    return out


def qflash_amax_qkv(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor,
                    out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Device float[3]: max |x| of fp32 Q, K, V (this device's slab)."""
    _check_qkv(q, k, v, torch.float32)
    out = torch.empty(3, dtype=torch.float32, device=q.device) if out is None else out
    _check_scales(out, 3, q.device)
    check(lib().qflash_amax_qkv(_dev_ptr(q), _dev_ptr(k), _dev_ptr(v), q.numel(), _dev_ptr(out),
                                _stream(stream)))
    return out


def qflash_forward_fused(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, block_kv: int = 128,
                         variant: str = "auto", out: torch.Tensor | None = None, codes=None,
                         scales: torch.Tensor | None = None, workspace: torch.Tensor | None = None,
                         out_int8: torch.Tensor | None = None, stream=None,
                         amax: torch.Tensor | None = None):
    """The whole hot path in one cooperative launch: fp32 Q, K, V [P, N, d] ->
    quantize (in the kernel's prologue) -> integer attention -> fp32 output.
    amax (device float[3], optional): per-tensor amax supplied by the caller (e.g.
    MAX-all-reduced over the ranks holding slabs of one tensor) instead of computed."""
    _check_qkv(q, k, v, torch.float32)
    if amax is not None:
        _check_scales(amax, 3, q.device)
    dev = q.device
    out = torch.empty(q.shape, dtype=torch.float32, device=dev) if out is None else out
    if codes is None:
        codes = [torch.empty(q.shape, dtype=torch.int8, device=dev) for _ in range(3)]
    scales = torch.empty(3, dtype=torch.float32, device=dev) if scales is None else scales
    if workspace is None:
        workspace = torch.zeros(_lib.DSCALE_WORKSPACE_BYTES // 4, dtype=torch.int32, device=dev)
    _check_like(q, out, "out", torch.float32)
    for i, t in enumerate(codes):
        _check_like(q, t, "codes[%d]" % i, torch.int8)
    if out_int8 is not None:
        _check_like(q, out_int8, "out_int8", torch.int8)
    _check_scales(scales, 3, dev)
    _check_workspace(workspace, dev)
    shape = _shape(q, block_kv)
    check(lib().qflash_forward_fused_amax(
        _dev_ptr(q), _dev_ptr(k), _dev_ptr(v), ctypes.byref(shape), _lib.VARIANTS[variant],
        _dev_ptr(codes[0]), _dev_ptr(codes[1]), _dev_ptr(codes[2]),
        _dev_ptr(out_int8) if out_int8 is not None else None, _dev_ptr(out), _dev_ptr(scales),
        _dev_ptr(workspace), _dev_ptr(amax) if amax is not None else None, _stream(stream)))
    return out


def qflash_forward_fused_qkv(qkv: torch.Tensor, heads: int, block_kv: int = 128, variant: str = "auto",
                             out: torch.Tensor | None = None, codes=None,
                             scales: torch.Tensor | None = None, workspace: torch.Tensor | None = None,
                             stream=None):
    """The fused step on a packed QKV projection output qkv [B, N, 3, heads, d] fp32
    (B = batch x windows): problems p = b * heads + h; returns y [B * heads, N, d]."""
    if qkv.dtype != torch.float32 or qkv.dim() != 5 or qkv.shape[2] != 3 or qkv.shape[3] != heads:
        raise ValueError("qkv must be fp32 [B, N, 3, heads, d]")
    if not qkv.is_cuda or not qkv.is_contiguous():
        raise ValueError("qkv must be a contiguous CUDA tensor")
    B, N, _, H, d = qkv.shape
    dev = qkv.device
    shp = (B * H, N, d)
    out = torch.empty(shp, dtype=torch.float32, device=dev) if out is None else out
    if codes is None:
        codes = [torch.empty(shp, dtype=torch.int8, device=dev) for _ in range(3)]
    scales = torch.empty(3, dtype=torch.float32, device=dev) if scales is None else scales
    if workspace is None:
        workspace = torch.zeros(_lib.DSCALE_WORKSPACE_BYTES // 4, dtype=torch.int32, device=dev)
    if tuple(out.shape) != shp or out.dtype != torch.float32 or out.device != dev:
        raise ValueError("out must be fp32 %s" % (shp,))
    for i, t in enumerate(codes):
        if tuple(t.shape) != shp or t.dtype != torch.int8 or t.device != dev:
            raise ValueError("codes[%d] must be int8 %s" % (i, shp))
    _check_scales(scales, 3, dev)
    _check_workspace(workspace, dev)
    shape = AttnShape(B * H, N, d, block_kv)
    check(lib().qflash_forward_fused_qkv(
        _dev_ptr(qkv), H, ctypes.byref(shape), _lib.VARIANTS[variant], _dev_ptr(codes[0]),
        _dev_ptr(codes[1]), _dev_ptr(codes[2]), None, _dev_ptr(out), _dev_ptr(scales),
        _dev_ptr(workspace), _stream(stream)))
    return out


class QFlashPipeline:
    """The whole hot path for one [P, N, d] workload with preallocated buffers.

    mode "fused" (default for fp32 inputs): one cooperative launch -- quantize in
    the attention kernel's prologue, integer attention, dequantized epilogue.
    mode "two":   qflash_quantize_qkv_prepare + attention with the fused
                  dequantize epilogue (two launches; any input dtype).
    mode "three": prepare + int8 attention + qflash_dequantize.
    No host synchronization in any mode; all are bit-identical."""

    def __init__(self, P: int, N: int, d: int, block_kv: int = 128, device="cuda",
                 variant: str = "auto", mode: str = "fused"):
        assert mode in ("fused", "two", "three")
        self.shape = (P, N, d)
        self.block_kv = block_kv
        self.variant = variant
        self.mode = mode
        dev = torch.device(device)
        self.qkv_q = [torch.empty(self.shape, dtype=torch.int8, device=dev) for _ in range(3)]
        self.scales = torch.empty(3, dtype=torch.float32, device=dev)
        self.o_q = torch.empty(self.shape, dtype=torch.int8, device=dev)
        self.workspace = torch.zeros(_lib.DSCALE_WORKSPACE_BYTES // 4, dtype=torch.int32, device=dev)
        self.out = torch.empty(self.shape, dtype=torch.float32, device=dev)
        self.device = self.out.device
        # the fused call's fixed arguments (buffers owned and sized here), marshalled once:
        # a call then checks and converts only q, k, v and the stream
        self._fused_shape = AttnShape(P, N, d, block_kv)
        self._fused_fixed = (ctypes.byref(self._fused_shape), _lib.VARIANTS[variant],
                             _dev_ptr(self.qkv_q[0]), _dev_ptr(self.qkv_q[1]), _dev_ptr(self.qkv_q[2]),
                             None, _dev_ptr(self.out), _dev_ptr(self.scales), _dev_ptr(self.workspace), None)

    def _fused_call(self, q, k, v, stream):
        for name, t in (("q", q), ("k", k), ("v", v)):
            if t.shape != self.out.shape or t.dtype != torch.float32 or t.device != self.device \
                    or not t.is_contiguous():
                raise ValueError("%s: expected a contiguous float32 %s tensor on %s, got %s %s on %s"
                                 % (name, tuple(self.shape), self.device, t.dtype, tuple(t.shape), t.device))
        f = self._fused_fixed
        check(lib().qflash_forward_fused_amax(
            ctypes.c_void_p(q.data_ptr()), ctypes.c_void_p(k.data_ptr()), ctypes.c_void_p(v.data_ptr()),
            f[0], f[1], f[2], f[3], f[4], f[5], f[6], f[7], f[8], f[9], _stream(stream)))
        return self.out

    def launches(self, dtype=torch.float32) -> int:
        """Kernel launches per call (bench.py's gpu_launches)."""
        if self.mode == "fused" and dtype == torch.float32:
            return 1
        P, N, d = self.shape
        quant = 1 if (dtype == torch.float32 and P * N * d <= 148 * 2 * 256 * 4 * 4) else 2
        return quant + (1 if self.mode == "two" else 2)

    def __call__(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, stream=None):
        if self.mode == "fused" and q.dtype == torch.float32:
            return self._fused_call(q, k, v, stream)
        _check_like(self.out, q, "q", q.dtype)   # the buffers were sized for self.shape
        qflash_quantize_qkv_prepare(q, k, v, outs=self.qkv_q, scales=self.scales,
                                    workspace=self.workspace, stream=stream)
        if self.mode != "three":
            qflash_attention_dequant_prepared(self.qkv_q[0], self.qkv_q[1], self.qkv_q[2],
                                              self.workspace, self.block_kv, self.variant,
                                              out=self.out, stream=stream)
        else:
            qflash_attention_int8_prepared(self.qkv_q[0], self.qkv_q[1], self.qkv_q[2],
                                           self.workspace, self.block_kv, self.variant,
                                           out=self.o_q, stream=stream)
            qflash_dequantize(self.o_q, self.scales[2:3], out=self.out, stream=stream)
        return self.out


# ------------------------------------------------ per-head granularity
def qflash_forward_per_head(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, heads: int,
                            block_kv: int = 128, variant: str = "auto", stream=None):
    """Per-head scales: fp32 Q, K, V [P, N, d] (head = problem mod heads) ->
    per-head quantization -> integer attention with per-head constants ->
    per-head dequantization.  Returns (y fp32, o int8, scales float32[3 heads],
    workspace) -- the int32 status of the constant derivation is workspace[0]."""
    _check_qkv(q, k, v, torch.float32)
    P, N, d = q.shape
    dev = q.device
    codes = [torch.empty(q.shape, dtype=torch.int8, device=dev) for _ in range(3)]
    scales = torch.empty(3 * heads, dtype=torch.float32, device=dev)
    check(lib().qflash_quantize_per_head(_dev_ptr(q), _dev_ptr(k), _dev_ptr(v), P, N, d, heads,
                                         _dev_ptr(codes[0]), _dev_ptr(codes[1]), _dev_ptr(codes[2]),
                                         _dev_ptr(scales), _stream(stream)))
    o = torch.empty(q.shape, dtype=torch.int8, device=dev)
    ws = torch.empty(_lib.DSCALE_WORKSPACE_BYTES // 4, dtype=torch.int32, device=dev)
    shape = _shape(q, block_kv)
    check(lib().qflash_attention_int8_per_head(_dev_ptr(codes[0]), _dev_ptr(codes[1]),
                                               _dev_ptr(codes[2]), _dev_ptr(scales), heads,
                                               ctypes.byref(shape), _lib.VARIANTS[variant],
                                               _dev_ptr(o), _dev_ptr(ws), _stream(stream)))
    y = torch.empty(q.shape, dtype=torch.float32, device=dev)
    check(lib().qflash_dequantize_per_head(_dev_ptr(o), _dev_ptr(scales[2 * heads:]), P, N, d,
                                           heads, _dev_ptr(y), _stream(stream)))
    return y, o, scales, ws


def qflash_forward_fused_per_head(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, heads: int,
                                  block_kv: int = 128, variant: str = "auto", out: torch.Tensor | None = None,
                                  codes=None, scales: torch.Tensor | None = None,
                                  workspace: torch.Tensor | None = None, stream=None):
    """The per-head step in ONE cooperative launch: fp32 Q, K, V [P, N, d] (head = problem
    mod heads) -> per-(tensor, head) quantization -> integer attention -> fp32 y.  Returns
    (y, scales float32[3 heads], workspace); the workspace must start zero-filled (a fresh
    one is allocated when None) and is re-zeroed by every call."""
    _check_qkv(q, k, v, torch.float32)
    dev = q.device
    out = torch.empty(q.shape, dtype=torch.float32, device=dev) if out is None else out
    if codes is None:
        codes = [torch.empty(q.shape, dtype=torch.int8, device=dev) for _ in range(3)]
    scales = torch.empty(3 * heads, dtype=torch.float32, device=dev) if scales is None else scales
    if workspace is None:
        workspace = torch.zeros(_lib.PH_FUSED_WORKSPACE_BYTES // 4, dtype=torch.int32, device=dev)
    _check_like(q, out, "out", torch.float32)
    for i, t in enumerate(codes):
        _check_like(q, t, "codes[%d]" % i, torch.int8)
    _check_scales(scales, 3 * heads, dev)
    _check_buffer(workspace, _lib.PH_FUSED_WORKSPACE_BYTES, "workspace", dev)
    shape = _shape(q, block_kv)
    check(lib().qflash_forward_fused_per_head(
        _dev_ptr(q), _dev_ptr(k), _dev_ptr(v), heads, ctypes.byref(shape), _lib.VARIANTS[variant],
        _dev_ptr(codes[0]), _dev_ptr(codes[1]), _dev_ptr(codes[2]), _dev_ptr(out), _dev_ptr(scales),
        _dev_ptr(workspace), _stream(stream)))
    return out, scales, workspace


class QFlashPerHeadPipeline:
    """qflash_forward_per_head with preallocated buffers (graph-capturable): per-head
    quantize (amax + quantize), constant derivation + attention, dequantize."""

    def __init__(self, P: int, N: int, d: int, heads: int, block_kv: int = 128, device="cuda",
                 variant: str = "auto", mode: str = "fused"):
        assert mode in ("fused", "multi")
        dev = torch.device(device)
        self.shape, self.heads, self.block_kv, self.variant = (P, N, d), heads, block_kv, variant
        self.mode = mode if block_kv <= 128 else "multi"  # the fused per-head step: block_kv <= 128
        self.codes = [torch.empty(self.shape, dtype=torch.int8, device=dev) for _ in range(3)]
        self.scales = torch.empty(3 * heads, dtype=torch.float32, device=dev)
        self.o_q = torch.empty(self.shape, dtype=torch.int8, device=dev)
        # zero-filled: the fused step keeps its per-(tensor, head) amax accumulators here
        self.workspace = torch.zeros(_lib.PH_FUSED_WORKSPACE_BYTES // 4, dtype=torch.int32, device=dev)
        self.out = torch.empty(self.shape, dtype=torch.float32, device=dev)

    def launches(self, dtype=torch.float32) -> int:
        # fused: one cooperative launch; multi: amax, quantize, derive, attention, dequantize
        return 1 if self.mode == "fused" else 5

    def __call__(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, stream=None):
        P, N, d = self.shape
        H = self.heads
        _check_qkv(q, k, v, torch.float32)
        _check_like(self.out, q, "q")
        if self.mode == "fused":
            qflash_forward_fused_per_head(q, k, v, H, self.block_kv, self.variant, out=self.out,
                                          codes=self.codes, scales=self.scales, workspace=self.workspace,
                                          stream=stream)
            return self.out
        c = self.codes
        check(lib().qflash_quantize_per_head(_dev_ptr(q), _dev_ptr(k), _dev_ptr(v), P, N, d, H,
                                             _dev_ptr(c[0]), _dev_ptr(c[1]), _dev_ptr(c[2]),
                                             _dev_ptr(self.scales), _stream(stream)))
        shape = AttnShape(P, N, d, self.block_kv)
        check(lib().qflash_attention_int8_per_head(_dev_ptr(c[0]), _dev_ptr(c[1]), _dev_ptr(c[2]),
                                                   _dev_ptr(self.scales), H, ctypes.byref(shape),
                                                   _lib.VARIANTS[self.variant], _dev_ptr(self.o_q),
                                                   _dev_ptr(self.workspace), _stream(stream)))
        check(lib().qflash_dequantize_per_head(_dev_ptr(self.o_q), _dev_ptr(self.scales[2 * H:]),
                                               P, N, d, H, _dev_ptr(self.out), _stream(stream)))
        return self.out

    def attention(self, stream=None):
        """The attention stage alone (constant derivation + Algorithm 1) on the codes."""
        P, N, d = self.shape
        c = self.codes
        shape = AttnShape(P, N, d, self.block_kv)
        check(lib().qflash_attention_int8_per_head(_dev_ptr(c[0]), _dev_ptr(c[1]), _dev_ptr(c[2]),
                                                   _dev_ptr(self.scales), self.heads, ctypes.byref(shape),
                                                   _lib.VARIANTS[self.variant], _dev_ptr(self.o_q),
                                                   _dev_ptr(self.workspace), _stream(stream)))
        return self.o_q


class QFlashHostPipeline:
    """Serving loop over host (pinned) fp32 batches: each call copies one batch in,
    runs the whole hot path (QFlashPipeline) and copies the fp32 result back, all
    asynchronously.  Consecutive batches alternate between `depth` device buffer
    sets on their own streams, so batch t+1's host->device copy runs while batch t
    computes and copies out (PCIe is full duplex: H2D and D2H on separate copy
    engines).  Every batch is complete -- quantized with its own per-tensor
    scales, attended, dequantized -- once synchronize() returns."""

    def __init__(self, P: int, N: int, d: int, block_kv: int = 128, device="cuda",
                 mode: str = "fused", depth: int = 2):
        dev = torch.device(device)
        self.depth = depth
        self.pipes = [QFlashPipeline(P, N, d, block_kv=block_kv, device=dev, mode=mode)
                      for _ in range(depth)]
        self.dev_in = [[torch.empty((P, N, d), dtype=torch.float32, device=dev) for _ in range(3)]
                       for _ in range(depth)]
        self.streams = [torch.cuda.Stream(device=dev) for _ in range(depth)]
        self.t = 0

    def __call__(self, hq: torch.Tensor, hk: torch.Tensor, hv: torch.Tensor, hout: torch.Tensor):
        """Enqueue one batch (host tensors; pinned for asynchronous copies)."""
        i = self.t % self.depth
        self.t += 1
        s = self.streams[i]
        with torch.cuda.stream(s):
            for dst, src in zip(self.dev_in[i], (hq, hk, hv)):
                dst.copy_(src, non_blocking=True)
            out = self.pipes[i](*self.dev_in[i], stream=s)
            hout.copy_(out, non_blocking=True)
        return hout

    def synchronize(self):
        for s in self.streams:
            s.synchronize()


def qflash_forward(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, block_kv: int = 128):
    """End-to-end QFlash attention on real inputs [P, N, d] (fp32/bf16/f16).
    Host tensors are copied to the current device and the fp32 result copied back."""
    host = not q.is_cuda
    dev = torch.device("cuda", torch.cuda.current_device())
    if host:
        q, k, v = (t.to(dev, non_blocking=True) for t in (q, k, v))
    pipe = QFlashPipeline(*q.shape, block_kv=block_kv, device=dev)
    out = pipe(q.contiguous(), k.contiguous(), v.contiguous())
    status = int(pipe.workspace[0].item())
    if status != _lib.QFLASH_OK:
        raise _lib.QFlashError(status, "device-derived scales out of range")
    return out.cpu() if host else out


# ---------------------------------------------------------------- host helpers
def qflash_derive_params(s_q: float, s_k: float, head_dim: int) -> dict:
    p = IntParams()
    check(lib().qflash_derive_params(s_q, s_k, head_dim, ctypes.byref(p)))
    return {name: getattr(p, name) for name, _ in IntParams._fields_}


def qflash_partition(num_problems: int, world: int, rank: int):
    b, c = ctypes.c_int32(), ctypes.c_int32()
    lib().qflash_partition(num_problems, world, rank, ctypes.byref(b), ctypes.byref(c))
    return b.value, c.value
