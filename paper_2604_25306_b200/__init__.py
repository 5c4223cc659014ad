"""QFlash on B200: integer-only fused attention (arxiv 2604.25306), sm_100a.

The product is libqflash.so (C ABI, include/qflash.h); this package is its thin
Python binding (argument marshalling only) plus the seeded synthetic inputs.
"""
from .api import (QFlashHostPipeline, QFlashPerHeadPipeline, QFlashPipeline, qflash_attention_int8, qflash_attention_int8_dscale,
                  qflash_attention_int8_prepared, qflash_quantize_qkv_prepare,
                  qflash_attention_dequant_prepared, qflash_amax_qkv, qflash_attention_int8_accum, qflash_forward_fused_qkv,
                  qflash_attention_ablation, qflash_forward_fused_per_head, qflash_forward_fused,
                  qflash_forward_per_head,
                  qflash_dequantize, qflash_derive_params, qflash_forward, qflash_partition,
                  qflash_quantize_per_tensor, qflash_quantize_qkv)

__all__ = ["QFlashHostPipeline", "QFlashPerHeadPipeline", "QFlashPipeline", "qflash_attention_int8", "qflash_attention_int8_dscale",
           "qflash_attention_int8_prepared", "qflash_quantize_qkv_prepare",
           "qflash_attention_dequant_prepared", "qflash_amax_qkv", "qflash_attention_int8_accum", "qflash_forward_fused_qkv", "qflash_attention_ablation", "qflash_forward_fused_per_head", "qflash_forward_fused", "qflash_forward_per_head",
           "qflash_dequantize", "qflash_derive_params", "qflash_forward", "qflash_partition",
           "qflash_quantize_per_tensor", "qflash_quantize_qkv"]
