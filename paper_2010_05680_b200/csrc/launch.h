// launch.h -- internal interface between the C ABI (tt_api.cu) and the kernel
// translation units.  Not installed; the public contract is include/tt.h.
#pragma once

#include <cuda_runtime_api.h>
#include <stdint.h>

namespace tt {

// dtype codes: 0 = fp32, 1 = fp16, 2 = bf16.
// *supported is set false (and nothing launched) when no tier fits.
cudaError_t softmax_launch(int dtype, void* scores, const int32_t* lengths, int64_t nrows,
                           int64_t rows_per_batch, int64_t Sk, float scale, cudaStream_t stream,
                           bool* supported);
const char* softmax_tier_name(int dtype, int64_t Sk, int64_t nrows);

// Packed (padding-free) softmax: request r is a dense [H, L_r, L_r] block at
// element offset cu_blocks[r]; L_r = cu_seqlens[r+1] - cu_seqlens[r] <= max_len.
cudaError_t softmax_packed_launch(int dtype, void* scores, const int32_t* cu_seqlens,
                                  const int64_t* cu_blocks, int64_t num_req, int64_t H,
                                  int64_t total_tokens, int64_t max_len, float scale,
                                  cudaStream_t stream, bool* supported);
const char* softmax_packed_tier_name(int dtype, int64_t max_len);
int softmax_packed_max_len(int dtype);

// vec_bytes: widest vector width (bytes) that every operand's alignment and
// the row pitch allow (host-computed in tt_api.cu).
cudaError_t layernorm_launch(int dtype, void* out, const void* x, const void* residual,
                             const void* bias, const void* gamma, const void* beta, int64_t rows,
                             int64_t hidden, float eps, int vec_bytes, cudaStream_t stream,
                             bool* supported);
const char* layernorm_tier_name(int dtype, int64_t hidden, int vec_bytes, int64_t rows);

// NEXT-2 element-wise kernels (elementwise.cu).  vec_bytes: 16 when every
// operand base and row pitch is 16-byte aligned, else the element size.
cudaError_t gelu_launch(int dtype, void* out, const void* x, const void* bias, int64_t rows,
                        int64_t n, int approximate, int vec_bytes, cudaStream_t stream);
cudaError_t split_qkv_launch(int dtype, void* q, void* k, void* v, const void* qkv,
                             const void* bias, int64_t B, int64_t S, int64_t H, int64_t D,
                             int vec_bytes, cudaStream_t stream);
cudaError_t merge_heads_launch(int dtype, void* out, const void* in, int64_t B, int64_t S,
                               int64_t H, int64_t D, int vec_bytes, cudaStream_t stream);

// NEXT-3 fused attention on tcgen05 (attention.cu); dtype 1 = fp16, 2 = bf16, D = 64
cudaError_t attention_launch(int dtype, void* out, const void* q, const void* k, const void* v,
                             const int32_t* lengths, int64_t B, int64_t H, int64_t S,
                             float scale, cudaStream_t stream);
bool attention_force_variant(int v);  // 0 auto, 1..4 (5..8 in the TT_TUNING build)
int attention_variant_count();       // variant ids are 0 .. count-1
bool attention_variant_ok(int v);    // variant v compiled into this build
cudaError_t smem_optin(const void* kern, size_t smem);  // per-device dynamic-smem opt-in

// Tuning / test hooks (include/tt_tune.h): enumerate every compiled tier and
// force one (-1 = automatic selection).  A forced tier that cannot serve the
// call's shape is ignored.
int softmax_tier_count();
const char* softmax_tier_name_at(int dtype, int i);
int softmax_tier_max_cols_at(int dtype, int i);
bool softmax_force_tier(int dtype, int i);
int layernorm_tier_count();
const char* layernorm_tier_name_at(int dtype, int i);
bool layernorm_force_tier(int dtype, int i);

}  // namespace tt
