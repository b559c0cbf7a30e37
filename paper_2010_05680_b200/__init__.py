"""B200-native batch-reduction kernels of TurboTransformers (arXiv 2010.05680).

The product is ``libtt.so`` (C ABI in ``include/tt.h``): in-place masked
attention softmax and fused add-bias + residual + LayerNorm, hand-written for
sm_100a.  This package is its thin ctypes binding; names follow the C ABI.
"""
from ._lib import (  # noqa: F401
    EXPORTS, TT_ERROR_CUDA, TT_ERROR_INVALID_VALUE, TT_ERROR_NOT_SUPPORTED, TT_MAX_LN_HIDDEN,
    TT_MAX_SOFTMAX_COLS, TT_SUCCESS, TTError, force_tier, layernorm_plan, lib, softmax_plan, status_string,
    tt_add_bias_layernorm, tt_add_bias_layernorm_raw, tt_add_bias_layernorm_staged,
    tt_softmax_masked, tt_softmax_masked_raw, tt_softmax_masked_staged, tiers, version,
    packed_offsets, tt_softmax_packed, softmax_packed_plan, tt_add_bias_gelu,
    tt_split_qkv_add_bias, tt_merge_heads, dp_schedule, schedule_cost, tt_attention_fwd,
    attention_variant, attention_variants, tuning_build, set_pdl, get_pdl,
    tt_softmax_masked_staged_overlap,
    tt_add_bias_layernorm_staged_overlap)

__all__ = [
    "tt_softmax_masked", "tt_softmax_packed", "packed_offsets", "tt_add_bias_layernorm", "tt_softmax_masked_staged",
    "tt_add_bias_layernorm_staged", "softmax_plan", "layernorm_plan", "TTError", "lib",
]
