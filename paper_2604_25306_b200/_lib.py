"""ctypes loader for libqflash.so (the C ABI in include/qflash.h).

Argument marshalling only: every step of the hot path runs in the library's
CUDA kernels.  There is no fallback -- if the shared library is missing the
import fails loudly.
"""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libqflash.so")
# A/B experiments (tools/) may point at an alternative in-tree build of the same ABI.
if os.environ.get("QFLASH_LIB"):
    LIB_PATH = os.path.join(_PKG, os.path.basename(os.environ["QFLASH_LIB"]))

QFLASH_OK = 0
QFLASH_ERR_INVALID_ARGUMENT = 1
QFLASH_ERR_UNSUPPORTED_SHAPE = 2
QFLASH_ERR_SCALE_RANGE = 3
QFLASH_ERR_CUDA = 4
QFLASH_ERR_UNSUPPORTED_DEVICE = 5

QFLASH_F32, QFLASH_BF16, QFLASH_F16 = 0, 1, 2
VARIANTS = {"auto": 0, "generic": 1, "packed": 2}
DSCALE_WORKSPACE_BYTES = 8192
PH_FUSED_WORKSPACE_BYTES = 16384

EXPORTED = [
    "qflash_quantize_per_tensor", "qflash_quantize_qkv", "qflash_attention_int8",
    "qflash_attention_int8_ex", "qflash_attention_int8_dscale", "qflash_dequantize",
    "qflash_dequantize_dscale", "qflash_derive_params", "qflash_partition",
    "qflash_status_string", "qflash_last_error", "qflash_version",
    "qflash_quantize_qkv_prepare", "qflash_attention_int8_prepared",
    "qflash_attention_dequant_prepared", "qflash_forward_fused",
    "qflash_quantize_per_head", "qflash_attention_int8_per_head", "qflash_dequantize_per_head",
    "qflash_amax_qkv", "qflash_forward_fused_amax", "qflash_attention_int8_accum",
    "qflash_forward_fused_qkv", "qflash_attention_ablation", "qflash_forward_fused_per_head",
]


class QFlashError(RuntimeError):
    def __init__(self, status: int, detail: str):
        super().__init__("%s: %s" % (status_string(status), detail))
        self.status = status


class AttnShape(ctypes.Structure):
    _fields_ = [("num_problems", ctypes.c_int32), ("seq_len", ctypes.c_int32),
                ("head_dim", ctypes.c_int32), ("block_kv", ctypes.c_int32)]


class IntParams(ctypes.Structure):
    _fields_ = [("s", ctypes.c_double), ("s_inv", ctypes.c_int32), ("n", ctypes.c_int32),
                ("r_p", ctypes.c_int32), ("m_p", ctypes.c_int32), ("q_magic", ctypes.c_uint32),
                ("q_shift", ctypes.c_int32), ("p_mul", ctypes.c_uint32), ("p_pre", ctypes.c_int32),
                ("p_max", ctypes.c_int32), ("rel_magic", ctypes.c_uint64),
                ("rel_shift", ctypes.c_int32)]


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError("libqflash.so is not built (%s); run __graft_entry__.build()" % LIB_PATH)
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, f32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_float
    st = ctypes.c_int
    L.qflash_quantize_per_tensor.restype = st
    L.qflash_quantize_per_tensor.argtypes = [vp, st, i64, vp, vp, vp, vp]
    L.qflash_quantize_qkv.restype = st
    L.qflash_quantize_qkv.argtypes = [vp, vp, vp, st, i64, vp, vp, vp, vp, vp]
    L.qflash_attention_int8.restype = st
    L.qflash_attention_int8.argtypes = [vp, vp, vp, f32, f32, f32, ctypes.POINTER(AttnShape), vp,
                                        ctypes.POINTER(f32), vp]
    L.qflash_attention_int8_ex.restype = st
    L.qflash_attention_int8_ex.argtypes = [vp, vp, vp, f32, f32, f32, ctypes.POINTER(AttnShape),
                                           st, vp, ctypes.POINTER(f32), vp]
    L.qflash_attention_int8_dscale.restype = st
    L.qflash_attention_int8_dscale.argtypes = [vp, vp, vp, vp, ctypes.POINTER(AttnShape), st, vp,
                                               vp, vp]
    L.qflash_quantize_qkv_prepare.restype = st
    L.qflash_quantize_qkv_prepare.argtypes = [vp, vp, vp, st, i64, vp, vp, vp, vp, i32, vp, vp]
    L.qflash_attention_int8_prepared.restype = st
    L.qflash_attention_int8_prepared.argtypes = [vp, vp, vp, ctypes.POINTER(AttnShape), st, vp,
                                                 vp, vp]
    L.qflash_attention_dequant_prepared.restype = st
    L.qflash_attention_dequant_prepared.argtypes = [vp, vp, vp, ctypes.POINTER(AttnShape), st, vp,
                                                    vp, vp, vp]
    L.qflash_forward_fused.restype = st
    L.qflash_forward_fused.argtypes = [vp, vp, vp, ctypes.POINTER(AttnShape), st, vp, vp, vp, vp,
                                       vp, vp, vp, vp]
    L.qflash_forward_fused_amax.restype = st
    L.qflash_forward_fused_amax.argtypes = [vp, vp, vp, ctypes.POINTER(AttnShape), st, vp, vp, vp, vp,
                                            vp, vp, vp, vp, vp]
    L.qflash_forward_fused_qkv.restype = st
    L.qflash_forward_fused_qkv.argtypes = [vp, i32, ctypes.POINTER(AttnShape), st, vp, vp, vp, vp, vp, vp,
                                           vp, vp]
    L.qflash_forward_fused_per_head.restype = st
    L.qflash_forward_fused_per_head.argtypes = [vp, vp, vp, i32, ctypes.POINTER(AttnShape), st, vp, vp, vp, vp,
                                                vp, vp, vp]
    L.qflash_attention_ablation.restype = st
    L.qflash_attention_ablation.argtypes = [vp, vp, vp, f32, f32, f32, ctypes.POINTER(AttnShape), i32, vp, vp]
    L.qflash_attention_int8_accum.restype = st
    L.qflash_attention_int8_accum.argtypes = [vp, vp, vp, f32, f32, ctypes.POINTER(AttnShape), vp, vp, vp]
    L.qflash_amax_qkv.restype = st
    L.qflash_amax_qkv.argtypes = [vp, vp, vp, i64, vp, vp]
    L.qflash_quantize_per_head.restype = st
    L.qflash_quantize_per_head.argtypes = [vp, vp, vp, i32, i32, i32, i32, vp, vp, vp, vp, vp]
    L.qflash_attention_int8_per_head.restype = st
    L.qflash_attention_int8_per_head.argtypes = [vp, vp, vp, vp, i32, ctypes.POINTER(AttnShape), st,
                                                 vp, vp, vp]
    L.qflash_dequantize_per_head.restype = st
    L.qflash_dequantize_per_head.argtypes = [vp, vp, i32, i32, i32, i32, vp, vp]
    L.qflash_dequantize.restype = st
    L.qflash_dequantize.argtypes = [vp, f32, i64, vp, vp]
    L.qflash_dequantize_dscale.restype = st
    L.qflash_dequantize_dscale.argtypes = [vp, vp, i64, vp, vp]
    L.qflash_derive_params.restype = st
    L.qflash_derive_params.argtypes = [f32, f32, i32, ctypes.POINTER(IntParams)]
    L.qflash_partition.restype = None
    L.qflash_partition.argtypes = [i32, i32, i32, ctypes.POINTER(i32), ctypes.POINTER(i32)]
    L.qflash_status_string.restype = ctypes.c_char_p
    L.qflash_status_string.argtypes = [st]
    L.qflash_last_error.restype = ctypes.c_char_p
    L.qflash_last_error.argtypes = []
    L.qflash_version.restype = i32
    L.qflash_version.argtypes = []
    L.qflash_debug_attention.restype = st
    L.qflash_debug_attention.argtypes = [vp, vp, vp, f32, f32, ctypes.POINTER(AttnShape), st, vp,
                                         vp, vp, vp, vp, vp]
    L.qflash_debug_force_config.restype = st
    L.qflash_debug_force_config.argtypes = [i32]
    L.qflash_debug_last_config.restype = i32
    L.qflash_debug_last_config.argtypes = []
    _lib = L
    return L


def status_string(status: int) -> str:
    return lib().qflash_status_string(status).decode()


def last_error() -> str:
    return lib().qflash_last_error().decode()


def force_config(cfg: int) -> None:
    """Force the attention kernel configuration (-1 = heuristic); include/qflash_debug.h."""
    check(lib().qflash_debug_force_config(cfg))


def last_config() -> tuple[int, int]:
    """(configuration, row-packing segments) of this thread's last attention launch."""
    c = lib().qflash_debug_last_config()
    return (-1, 0) if c < 0 else (c & 15, c >> 4)


def check(status: int) -> None:
    if status != QFLASH_OK:
        raise QFlashError(status, last_error())
