"""paper_2603_12646_b200 -- B200-native FusedFlashAttention (the Stage-1 hot path of arXiv 2603.12646).

Public surface mirrors the reference operator interface (see attention.py).  The compute
path is librf_fa.so (hand-written sm_100a CUDA behind the C ABI in include/rf_fa.h).
"""
from .attention import (AttentionSpec, FaPlan, FlashStats, RewriteOptions, ShapeMismatch, UnsupportedHeadDim,  # noqa: F401
                        WorkspaceAllocator, fa_memory_bytes, flash_attention, fused_flash_attention,
                        kMaskThreshold, kMaskValue, local_window_attrs, mask_memory_bytes, pad_bias_from_mask)

__all__ = [
    "AttentionSpec", "FaPlan", "FlashStats", "RewriteOptions", "ShapeMismatch", "UnsupportedHeadDim", "WorkspaceAllocator",
    "fa_memory_bytes", "flash_attention", "fused_flash_attention", "kMaskThreshold", "kMaskValue",
    "local_window_attrs", "mask_memory_bytes", "pad_bias_from_mask",
]
