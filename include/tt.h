/*
 * tt.h -- C ABI of libtt.so: B200 (sm_100a) batch-reduction kernels for
 * transformer serving, after TurboTransformers (arXiv 2010.05680).
 *
 * The paper states the problem as "reduce a batch of 1-D arrays in parallel"
 * (§4.1.2, l.315-317): "Softmax calculates summation and maximum and
 * LayerNorm calculates the mean and variance".  Its two fused reduction
 * kernels, named `ApplyMaskAndSoftmax` and `AddBiasLayerNorm` (l.765), are
 * the non-GEMM hot spots of a BERT layer (Table 2, l.324-337).  This library
 * exports those two operations (plus host-buffer "staged" forms and plan
 * queries), in fp32, fp16 and bf16 storage with fp32 arithmetic.  Beyond the
 * hot path it also exports the SURVEY §8(f) NEXT rows: the packed
 * (padding-free) softmax, the element-wise kernels between GEMMs (bias+GELU,
 * QKV split, head merge), the tcgen05 fused attention, and -- in tt_sched.h
 * -- the DP batch scheduler (Alg. 2).
 *
 * Conventions common to every entry point
 * ---------------------------------------
 * Ownership   The caller owns every buffer.  The library never allocates,
 *             frees or synchronises, needs no workspace and keeps no handles.
 * Devices     Device pointers must be on the current CUDA device.
 * Execution   Asynchronous on `stream` (0 = legacy default stream); results
 *             are visible after the caller synchronises the stream.  Kernels
 *             are launched with programmatic dependent launch (PDL): a kernel
 *             may be scheduled while the previous kernel in the stream drains,
 *             but executes griddepcontrol.wait before its first global access,
 *             so stream order is kept for every memory effect; it signals its
 *             own dependents only after its last store.  A caller kernel that
 *             is itself launched programmatically after a libtt call must
 *             execute griddepcontrol.wait before reading libtt's output (as
 *             with any PDL producer).  ttx_set_pdl(0) (tt_tune.h) turns it off.
 * Alignment   Every tensor base pointer must be 16-byte aligned (any
 *             cudaMalloc / PyTorch allocation is); rows may have any length.
 * Errors      Arguments are validated on the host BEFORE any CUDA call:
 *               TT_ERROR_INVALID_VALUE  null pointer with a non-empty shape,
 *                                       negative dimension, element count
 *                                       overflowing int64, non-finite scale,
 *                                       negative or non-finite eps,
 *                                       out/x/residual partially overlapping;
 *               TT_ERROR_NOT_SUPPORTED  base pointer not 16-B aligned, or a
 *                                       row longer than the largest tier
 *                                       (TT_MAX_SOFTMAX_COLS / TT_MAX_LN_HIDDEN);
 *               TT_ERROR_CUDA           the launch failed (cudaGetLastError);
 *                                       the cudaError_t is kept per thread, see
 *                                       tt_last_cuda_error().
 *             An empty problem (any dimension 0) returns TT_SUCCESS with no
 *             CUDA call.  Device-side faults surface at the caller's next
 *             synchronisation, as with cuBLAS.  No C++ exception crosses the ABI.
 * Values      Input values are not validated; NaN/Inf in VALID positions
 *             propagate.  Masked (padding) positions are never read.
 * Threads     Stateless and reentrant; concurrent calls on different streams
 *             are safe.
 */
#ifndef TT_H_
#define TT_H_

#include <stdint.h>
#include <cuda_runtime_api.h> /* cudaStream_t */

#if defined(__GNUC__)
#define TT_API __attribute__((visibility("default")))
#else
#define TT_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    TT_SUCCESS = 0,
    TT_ERROR_INVALID_VALUE = 1,
    TT_ERROR_NOT_SUPPORTED = 2,
    TT_ERROR_CUDA = 3
} tt_status;

/* Largest supported row lengths (elements). */
#define TT_MAX_SOFTMAX_COLS 1073741824
#define TT_MAX_LN_HIDDEN 32768

/* ------------------------------------------------------------------------
 * Masked attention softmax, in place:  ApplyMaskAndSoftmax
 *
 * scores   DEVICE, [B, H, Sq, Sk] row-major contiguous, read and overwritten.
 *          (fp32: float*; f16: __half*; bf16: __nv_bfloat16*)
 * lengths  DEVICE int32[B]: valid key count of request b.  The padding mask
 *          is implicit (shorter requests are padded
 *          to the longest): with L_b = min(max(lengths[b], 0), Sk), for every
 *          row (b, h, i) of b:
 *              z_j = scale * x_j,                          j <  L_b
 *              y_j = exp(z_j - max_k z_k) / sum_k exp(z_k - max_k z_k)
 *              y_j = +0.0 (bit pattern 0),                 L_b <= j < Sk
 *          Key columns j >= L_b are never read.  L_b = 0 gives an all-zero
 *          row.  Padded query rows i >= L_b are normalised like any other
 *          row (only keys are masked; R2).
 * scale    finite float, applied to the logits before the max (BERT: 0.125).
 * Sk       <= TT_MAX_SOFTMAX_COLS (2^30; rows beyond 131 072 keys run on the
 *          two-pass long-row tier).
 * ---------------------------------------------------------------------- */
TT_API tt_status tt_softmax_masked_f32(float* scores, const int32_t* lengths, int64_t B, int64_t H,
                                int64_t Sq, int64_t Sk, float scale, cudaStream_t stream);
TT_API tt_status tt_softmax_masked_f16(void* scores, const int32_t* lengths, int64_t B, int64_t H,
                                int64_t Sq, int64_t Sk, float scale, cudaStream_t stream);
TT_API tt_status tt_softmax_masked_bf16(void* scores, const int32_t* lengths, int64_t B, int64_t H,
                                 int64_t Sq, int64_t Sk, float scale, cudaStream_t stream);

/* ------------------------------------------------------------------------
 * Packed (padding-free) attention softmax, in place -- SURVEY §8(f) NEXT-1:
 * the variable-length batch of PAPER.md §5 (l.576, "all requests in the batch
 * will be zero-padded with regards to the maximum length") stored WITHOUT the
 * padding.  Request r (0 <= r < num_req) has L_r = cu_seqlens[r+1] -
 * cu_seqlens[r] tokens and its scores are a dense row-major [H, L_r, L_r]
 * block starting at element cu_blocks[r]; every row is softmax(scale * x)
 * over its L_r keys (no masked keys, no padding bytes read or written).
 *
 * scores      DEVICE, storage dtype of the entry point, 16-byte aligned base.
 * cu_seqlens  DEVICE int32[num_req + 1], cu_seqlens[0] = 0, nondecreasing.
 * cu_blocks   DEVICE int64[num_req], element offset of each request's block
 *             (dense packing: cu_blocks[r] = H * sum_{i<r} L_i^2).
 * total_tokens  HOST copy of cu_seqlens[num_req] (sizes the grid).
 * max_seqlen  HOST upper bound of every L_r (selects the tier); a request
 *             longer than max_seqlen is undefined (memory-safe, values wrong).
 * Errors as above; max_seqlen > 1024 (fp32) / 2048 (fp16, bf16) or
 * H * total_tokens >= 2^32 - 1 gives TT_ERROR_NOT_SUPPORTED.
 * ---------------------------------------------------------------------- */
TT_API tt_status tt_softmax_packed_f32(float* scores, const int32_t* cu_seqlens,
                                       const int64_t* cu_blocks, int64_t num_req, int64_t H,
                                       int64_t total_tokens, int64_t max_seqlen, float scale,
                                       cudaStream_t stream);
TT_API tt_status tt_softmax_packed_f16(void* scores, const int32_t* cu_seqlens,
                                       const int64_t* cu_blocks, int64_t num_req, int64_t H,
                                       int64_t total_tokens, int64_t max_seqlen, float scale,
                                       cudaStream_t stream);
TT_API tt_status tt_softmax_packed_bf16(void* scores, const int32_t* cu_seqlens,
                                        const int64_t* cu_blocks, int64_t num_req, int64_t H,
                                        int64_t total_tokens, int64_t max_seqlen, float scale,
                                        cudaStream_t stream);

/* ------------------------------------------------------------------------
 * Fused add-bias + residual + LayerNorm:  AddBiasLayerNorm (
 * "fusing all the kernels between two GEMM kernels into a single one",
 * l.302; variance per Eq. 1, l.406-409, population form)
 *
 *   v_k = (x_k + bias_k) + residual_k
 *   out_k = (v_k - mean(v)) * rsqrt(var(v) + eps) * gamma_k + beta_k
 *
 * out, x, residual   DEVICE [rows, hidden] row-major contiguous.  `out` may
 *                    alias `x` or `residual` exactly; any other overlap is
 *                    rejected with TT_ERROR_INVALID_VALUE.
 * bias, gamma, beta  DEVICE [hidden].
 * All operands share the storage dtype of the entry point; arithmetic is fp32.
 * eps      finite, >= 0, inside the square root (eps = 0 on a constant row
 *          gives NaN, as in PyTorch).
 * hidden   <= TT_MAX_LN_HIDDEN.
 * ---------------------------------------------------------------------- */
TT_API tt_status tt_add_bias_layernorm_f32(float* out, const float* x, const float* residual,
                                    const float* bias, const float* gamma, const float* beta,
                                    int64_t rows, int64_t hidden, float eps, cudaStream_t stream);
TT_API tt_status tt_add_bias_layernorm_f16(void* out, const void* x, const void* residual,
                                    const void* bias, const void* gamma, const void* beta,
                                    int64_t rows, int64_t hidden, float eps, cudaStream_t stream);
TT_API tt_status tt_add_bias_layernorm_bf16(void* out, const void* x, const void* residual,
                                     const void* bias, const void* gamma, const void* beta,
                                     int64_t rows, int64_t hidden, float eps, cudaStream_t stream);

/* ------------------------------------------------------------------------
 * NEXT-2: the element-wise kernels of the fused graph,
 * "fused activation functions and fused transpose operations" (PAPER.md
 * l.304-308).  dtype: 0 = fp32, 1 = fp16, 2 = bf16; fp32 arithmetic.  Same
 * conventions and error codes as above; vectorised when every base pointer
 * and row pitch is 16-byte aligned (element-wise otherwise).
 *
 * tt_add_bias_gelu:  out[r, j] = gelu(x[r, j] + bias[j]) over [rows, n];
 *   approximate = 0: exact 0.5 v (1 + erf(v / sqrt 2)) (BERT's definition);
 *   approximate = 1: 0.5 v (1 + tanh(sqrt(2/pi) (v + 0.044715 v^3))).
 *   out may alias x exactly; bias must not overlap out.
 * tt_split_qkv_add_bias:  qkv [B*S, 3*H*D] (token-major QKV GEMM output,
 *   parts ordered q, k, v, then heads) + bias [3*H*D] ->
 *   q, k, v each [B, H, S, D]:  out_t[b,h,s,d] = qkv[b*S+s, (t*H+h)*D+d] + bias[(t*H+h)*D+d].
 *   Outputs must not overlap the inputs or each other.
 * tt_merge_heads:  in [B, H, S, D] -> out [B*S, H*D]: out[b*S+s, h*D+d] = in[b,h,s,d].
 *   out must not overlap in.
 * Index spaces must fit 32 bits (B*S*3*H*D < 2^32 - 1), else TT_ERROR_NOT_SUPPORTED.
 * ---------------------------------------------------------------------- */
TT_API tt_status tt_add_bias_gelu(int dtype, void* out, const void* x, const void* bias,
                                  int64_t rows, int64_t n, int approximate, cudaStream_t stream);
TT_API tt_status tt_split_qkv_add_bias(int dtype, void* q, void* k, void* v, const void* qkv,
                                       const void* bias, int64_t B, int64_t S, int64_t H,
                                       int64_t D, cudaStream_t stream);
TT_API tt_status tt_merge_heads(int dtype, void* out, const void* in, int64_t B, int64_t S,
                                int64_t H, int64_t D, cudaStream_t stream);

/* ------------------------------------------------------------------------
 * NEXT-3: the masked softmax fused into its GEMMs, on the
 * tcgen05 tensor cores -- "the scaled dot-product attention computes the dot
 * products of the query with all keys, and applies a Softmax function to
 * obtain the weights on the values":
 *   out[b,h,i,:] = sum_{j < L_b} softmax_j(scale * q[b,h,i,:] . k[b,h,j,:]) v[b,h,j,:]
 * with L_b = clamp(lengths[b], 0, S) (the padding mask of tt_softmax_masked);
 * out rows are 0 when L_b = 0.  The [B,H,S,S] scores never reach HBM.
 *
 * q, k, v, out  DEVICE [B, H, S, D] row-major (the layout tt_split_qkv_add_bias
 *               produces), dtype 1 = fp16 or 2 = bf16 (fp32 accumulation;
 *               the probabilities enter the second GEMM rounded to the storage
 *               dtype, as in flash attention).  16-byte aligned bases.
 * lengths       DEVICE int32[B].   D must be 64 (BERT), else NOT_SUPPORTED.
 * out must not overlap q, k or v.
 * ---------------------------------------------------------------------- */
TT_API tt_status tt_attention_fwd(int dtype, void* out, const void* q, const void* k,
                                  const void* v, const int32_t* lengths, int64_t B, int64_t H,
                                  int64_t S, int64_t D, float scale, cudaStream_t stream);

/* ------------------------------------------------------------------------
 * Staged (host-buffer) variants: the end-to-end serving call.  On `stream`:
 * copy the HOST inputs into the caller's DEVICE buffers, run the kernel, copy
 * the result back into the HOST buffer.  Host buffers should be pinned
 * (cudaHostAlloc / torch pin_memory) for the copies to be asynchronous.
 * Same validation and error codes as the device entry points, plus
 * TT_ERROR_CUDA for a failed copy.  dtype: 0 = fp32, 1 = fp16, 2 = bf16.
 *
 * softmax:  host_scores [B,H,Sq,Sk] in/out, host_lengths int32[B] in;
 *           dev_scores, dev_lengths are the device staging buffers.
 * layernorm: host_x, host_residual in, host_out out; dev_* device buffers of
 *           the same shapes; bias/gamma/beta are DEVICE (model weights stay
 *           resident).
 * ---------------------------------------------------------------------- */
TT_API tt_status tt_softmax_masked_staged(int dtype, void* host_scores, const int32_t* host_lengths,
                                   void* dev_scores, int32_t* dev_lengths, int64_t B, int64_t H,
                                   int64_t Sq, int64_t Sk, float scale, cudaStream_t stream);
TT_API tt_status tt_add_bias_layernorm_staged(int dtype, void* host_out, const void* host_x,
                                       const void* host_residual, void* dev_out, void* dev_x,
                                       void* dev_residual, const void* bias, const void* gamma,
                                       const void* beta, int64_t rows, int64_t hidden, float eps,
                                       cudaStream_t stream);

/* Overlapped staging: the same operation and contract, but the batch is cut
 * into `chunks` pieces (requests for the softmax, rows for LayerNorm; each piece
 * a multiple of the granule that keeps its device base 16-byte aligned).  Piece
 * i's H2D copy and kernel run on `stream` while piece i-1's result is copied
 * D2H on `copy_stream`, so the two PCIe directions overlap.  On return `stream`
 * has been made to wait for the last D2H: the host result is complete when
 * `stream` completes, and later work on `stream` may reuse the device buffers.
 * copy_stream NULL, equal to stream, or chunks <= 1: the single-stream call.
 * The library creates one CUDA event per call (destroyed before returning;
 * released by the driver when its last use completes). */
TT_API tt_status tt_softmax_masked_staged_overlap(int dtype, void* host_scores,
                                                  const int32_t* host_lengths, void* dev_scores,
                                                  int32_t* dev_lengths, int64_t B, int64_t H,
                                                  int64_t Sq, int64_t Sk, float scale,
                                                  int64_t chunks, cudaStream_t stream,
                                                  cudaStream_t copy_stream);
TT_API tt_status tt_add_bias_layernorm_staged_overlap(int dtype, void* host_out, const void* host_x,
                                                      const void* host_residual, void* dev_out,
                                                      void* dev_x, void* dev_residual,
                                                      const void* bias, const void* gamma,
                                                      const void* beta, int64_t rows,
                                                      int64_t hidden, float eps, int64_t chunks,
                                                      cudaStream_t stream,
                                                      cudaStream_t copy_stream);

/* ------------------------------------------------------------------------
 * Introspection
 * ---------------------------------------------------------------------- */
/* Static string for a status code ("TT_SUCCESS", ...). */
TT_API const char* tt_status_string(tt_status s);
/* cudaError_t of the calling thread's last TT_ERROR_CUDA (0 if none). */
TT_API int tt_last_cuda_error(void);
/* Library version, major*10000 + minor*100 + patch. */
TT_API int tt_version(void);
/* Name of the kernel tier a call with these arguments would launch, for
 * profiling and tests ("softmax_rows<f32,V16,G32,NV1,R2>", ...).  Writes at
 * most `cap` bytes (NUL-terminated) into buf; returns the status the real call
 * would return for its host-side validation (pointers are not checked). */
TT_API tt_status tt_softmax_masked_plan(int dtype, int64_t B, int64_t H, int64_t Sq, int64_t Sk,
                                 char* buf, int cap);
TT_API tt_status tt_add_bias_layernorm_plan(int dtype, int64_t rows, int64_t hidden, char* buf, int cap);
TT_API tt_status tt_softmax_packed_plan(int dtype, int64_t max_seqlen, char* buf, int cap);

#ifdef __cplusplus
}
#endif
#endif /* TT_H_ */
