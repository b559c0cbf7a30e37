/*
 * tt_tune.h -- tuning and test hooks of libtt.so (not part of the serving
 * contract in tt.h).
 *
 * Every kernel configuration ("tier") compiled into the library can be listed
 * and forced, so that tests can run each tier against the oracle and tools can
 * time them.  Forcing is process-global and meant for single-threaded tools.
 * A forced tier that cannot serve a call's shape is ignored (automatic
 * selection is used for that call).  The automatic choice is what
 * tt_softmax_masked_plan / tt_add_bias_layernorm_plan report.
 *
 * op: 0 = softmax, 1 = add-bias LayerNorm.  dtype: 0 = fp32, 1 = fp16, 2 = bf16.
 */
#ifndef TT_TUNE_H_
#define TT_TUNE_H_

#include "tt.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Number of compiled tiers for `op` (same for every dtype); -1 on a bad op. */
TT_API int ttx_tier_count(int op);
/* Static name of tier i, or NULL when out of range. */
TT_API const char* ttx_tier_name(int op, int dtype, int i);
/* Force tier i for (op, dtype); i = -1 restores automatic selection.
 * Returns TT_ERROR_INVALID_VALUE for a bad op, dtype or index. */
TT_API tt_status ttx_force_tier(int op, int dtype, int i);
/* Fused attention (tt_attention_fwd) variant: 0 = automatic, 1 = 128-key tiles
 * single-buffered (2 CTAs per SM), 2 = 128-key tiles double-buffered (1 CTA per
 * SM), 3 = 64-key tiles single-buffered (4 CTAs per SM), 4 = 64-key tiles
 * double-buffered and software-pipelined (3 CTAs per SM), 5 = warp-specialised
 * (producer warp, MMA warp, 4 softmax warps; mbarrier hand-offs, no CTA barrier
 * in the tile loop; 2 CTAs per SM), 6 / 7 = variant 4 with two threads per
 * query row (8 warps; 2 / 3 CTAs per SM), 8 = variant 4 waiting for the previous
 * P.V only after the exponentials, 9 = warp-specialised: two 128-row query tiles
 * per CTA sharing K / V loaded by TMA, a producer warp, an MMA warp and two
 * ping-ponging softmax warpgroups, P kept in TMEM (attention_fa.cu), 128-key
 * tiles; 10 = the same with 64-key tiles and two S buffers per query tile;
 * 11 = variant 4 with Q / K / V loaded by TMA tensor copies on mbarriers.
 * Variants 1..11 are compiled into the tuning build only (ttx_tuning_build);
 * TT_ERROR_INVALID_VALUE for a variant not compiled in (ttx_attention_variant_ok). */
TT_API tt_status ttx_attention_variant(int v);
/* Variant ids are 0 .. ttx_attention_variant_count() - 1; ttx_attention_variant_ok
 * says whether variant v is compiled into this library (0 always; 1..11
 * in the tuning build only). */
TT_API int ttx_attention_variant_count(void);
TT_API int ttx_attention_variant_ok(int v);
/* 1 in the tuning build (libtt_tune.so, -DTT_TUNING: every tuning candidate
 * compiled in), 0 in the product library libtt.so. */
TT_API int ttx_tuning_build(void);

/* Programmatic dependent launch (PDL, default on): every kernel is launched
 * with the programmatic-stream-serialization attribute and begins with
 * griddepcontrol.wait (before any global access) then launch_dependents, so a
 * kernel's launch and prologue overlap the tail of the previous kernel in the
 * stream while its memory accesses still follow that kernel's completion.
 * enable: 1 on, 0 off (plain stream order).  Process-wide; for tools and tests.
 * Returns TT_ERROR_INVALID_VALUE for any other value. */
TT_API tt_status ttx_set_pdl(int enable);
/* Current PDL switch (1 on, 0 off). */
TT_API int ttx_get_pdl(void);

#ifdef __cplusplus
}
#endif
#endif /* TT_TUNE_H_ */
