#include <atomic>
#include <map>
#include <mutex>
#include <utility>
// tt_api.cu -- the C ABI of libtt.so (contract: include/tt.h).
//
// Host-side validation happens before any CUDA call; the kernels themselves
// live in softmax.cu / layernorm.cu.  No allocation, no synchronisation, no
// global state beyond a thread-local last-error slot.
#include <math.h>
#include <stdio.h>
#include <string.h>

#include "../../include/tt.h"
#include "../../include/tt_tune.h"
#include "launch.h"

namespace {

thread_local int g_last_cuda_error = 0;

constexpr int kVersion = 1 * 10000 + 0 * 100 + 0;

int elem_bytes(int dtype) { return dtype == 0 ? 4 : 2; }

bool mul_overflows(int64_t a, int64_t b, int64_t* out) {
    __int128 p = (__int128)a * (__int128)b;
    if (p > (__int128)INT64_MAX) return true;
    *out = (int64_t)p;
    return false;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

tt_status cuda_status(cudaError_t e) {
    if (e == cudaSuccess) return TT_SUCCESS;
    g_last_cuda_error = (int)e;
    return TT_ERROR_CUDA;
}

// Byte ranges [a, a+n) and [b, b+m) overlap?
bool overlaps(const void* a, int64_t n, const void* b, int64_t m) {
    const uintptr_t pa = reinterpret_cast<uintptr_t>(a), pb = reinterpret_cast<uintptr_t>(b);
    return pa < pb + (uintptr_t)m && pb < pa + (uintptr_t)n;
}

// ------------------------------------------------------------------ softmax
tt_status softmax_validate(int dtype, const void* scores, const int32_t* lengths, int64_t B,
                           int64_t H, int64_t Sq, int64_t Sk, float scale, bool check_ptrs,
                           int64_t* nrows_out, bool* empty) {
    if (dtype < 0 || dtype > 2) return TT_ERROR_INVALID_VALUE;
    if (B < 0 || H < 0 || Sq < 0 || Sk < 0) return TT_ERROR_INVALID_VALUE;
    if (!isfinite(scale)) return TT_ERROR_INVALID_VALUE;
    int64_t bh, nrows, n;
    if (mul_overflows(B, H, &bh) || mul_overflows(bh, Sq, &nrows) || mul_overflows(nrows, Sk, &n) ||
        mul_overflows(n, elem_bytes(dtype), &n))
        return TT_ERROR_INVALID_VALUE;
    *nrows_out = nrows;
    *empty = (nrows == 0 || Sk == 0);
    if (*empty) return TT_SUCCESS;
    if (check_ptrs) {
        if (!scores || !lengths) return TT_ERROR_INVALID_VALUE;
        if (!aligned16(scores) || (reinterpret_cast<uintptr_t>(lengths) & 3u))
            return TT_ERROR_NOT_SUPPORTED;
    }
    if (Sk > TT_MAX_SOFTMAX_COLS) return TT_ERROR_NOT_SUPPORTED;
    return TT_SUCCESS;
}

tt_status softmax_any(int dtype, void* scores, const int32_t* lengths, int64_t B, int64_t H,
                      int64_t Sq, int64_t Sk, float scale, cudaStream_t stream) {
    int64_t nrows = 0;
    bool empty = false;
    tt_status s = softmax_validate(dtype, scores, lengths, B, H, Sq, Sk, scale, true, &nrows, &empty);
    if (s != TT_SUCCESS || empty) return s;
    bool supported = false;
    cudaError_t e = tt::softmax_launch(dtype, scores, lengths, nrows, H * Sq, Sk, scale, stream,
                                       &supported);
    if (!supported) return TT_ERROR_NOT_SUPPORTED;
    return cuda_status(e);
}

// ---------------------------------------------------------------- layernorm
int ln_vec_bytes(int dtype, int64_t hidden, const void* const* ptrs, int nptrs) {
    const int e = elem_bytes(dtype);
    for (int vb = 32; vb >= e; vb >>= 1) {
        if ((hidden * e) % vb) continue;
        bool ok = true;
        for (int i = 0; i < nptrs; ++i)
            if (reinterpret_cast<uintptr_t>(ptrs[i]) % (uintptr_t)vb) ok = false;
        if (ok) return vb;
    }
    return e;
}

tt_status ln_validate(int dtype, const void* out, const void* x, const void* residual,
                      const void* bias, const void* gamma, const void* beta, int64_t rows,
                      int64_t hidden, float eps, bool check_ptrs, bool* empty) {
    if (dtype < 0 || dtype > 2) return TT_ERROR_INVALID_VALUE;
    if (rows < 0 || hidden < 0) return TT_ERROR_INVALID_VALUE;
    if (!isfinite(eps) || eps < 0.f) return TT_ERROR_INVALID_VALUE;
    int64_t n, nb;
    if (mul_overflows(rows, hidden, &n) || mul_overflows(n, elem_bytes(dtype), &nb))
        return TT_ERROR_INVALID_VALUE;
    *empty = (n == 0);
    if (*empty) return TT_SUCCESS;
    if (check_ptrs) {
        const void* ps[6] = {out, x, residual, bias, gamma, beta};
        for (const void* p : ps)
            if (!p) return TT_ERROR_INVALID_VALUE;
        // out may alias x or residual exactly; any partial overlap is rejected,
        // and the read-only parameters must not overlap anything written.
        const int64_t pb = hidden * elem_bytes(dtype);
        if (out != x && overlaps(out, nb, x, nb)) return TT_ERROR_INVALID_VALUE;
        if (out != residual && overlaps(out, nb, residual, nb)) return TT_ERROR_INVALID_VALUE;
        const void* params[3] = {bias, gamma, beta};
        for (const void* p : params)
            if (overlaps(out, nb, p, pb)) return TT_ERROR_INVALID_VALUE;
        for (const void* p : ps)
            if (!aligned16(p)) return TT_ERROR_NOT_SUPPORTED;
    }
    if (hidden > TT_MAX_LN_HIDDEN) return TT_ERROR_NOT_SUPPORTED;
    return TT_SUCCESS;
}

tt_status ln_any(int dtype, void* out, const void* x, const void* residual, const void* bias,
                 const void* gamma, const void* beta, int64_t rows, int64_t hidden, float eps,
                 cudaStream_t stream) {
    bool empty = false;
    tt_status s = ln_validate(dtype, out, x, residual, bias, gamma, beta, rows, hidden, eps, true,
                              &empty);
    if (s != TT_SUCCESS || empty) return s;
    const void* ps[6] = {out, x, residual, bias, gamma, beta};
    const int vb = ln_vec_bytes(dtype, hidden, ps, 6);
    bool supported = false;
    cudaError_t e = tt::layernorm_launch(dtype, out, x, residual, bias, gamma, beta, rows, hidden,
                                         eps, vb, stream, &supported);
    if (!supported) return TT_ERROR_NOT_SUPPORTED;
    return cuda_status(e);
}

// ------------------------------------------------------------------- NEXT-2
// 16 when every pointer and every pitch (bytes) is a multiple of 16, else 0
int vec16(const void* const* ptrs, int nptrs, const int64_t* pitches, int npitch) {
    for (int i = 0; i < nptrs; ++i)
        if (reinterpret_cast<uintptr_t>(ptrs[i]) & 15u) return 0;
    for (int i = 0; i < npitch; ++i)
        if (pitches[i] % 16) return 0;
    return 16;
}

tt_status gelu_any(int dtype, void* out, const void* x, const void* bias, int64_t rows, int64_t n,
                   int approximate, cudaStream_t stream) {
    if (dtype < 0 || dtype > 2 || rows < 0 || n < 0 || approximate < 0 || approximate > 1)
        return TT_ERROR_INVALID_VALUE;
    int64_t cnt, nb;
    if (mul_overflows(rows, n, &cnt) || mul_overflows(cnt, elem_bytes(dtype), &nb))
        return TT_ERROR_INVALID_VALUE;
    if (cnt == 0) return TT_SUCCESS;
    if (!out || !x || !bias) return TT_ERROR_INVALID_VALUE;
    const int64_t pb = n * elem_bytes(dtype);
    if (out != x && overlaps(out, nb, x, nb)) return TT_ERROR_INVALID_VALUE;
    if (overlaps(out, nb, bias, pb)) return TT_ERROR_INVALID_VALUE;
    if ((reinterpret_cast<uintptr_t>(out) | reinterpret_cast<uintptr_t>(x) |
         reinterpret_cast<uintptr_t>(bias)) & (uintptr_t)(elem_bytes(dtype) - 1))
        return TT_ERROR_NOT_SUPPORTED;
    if (n > 0x7fffffffLL) return TT_ERROR_NOT_SUPPORTED;
    const void* ps[3] = {out, x, bias};
    const int vb = vec16(ps, 3, &pb, 1);
    return cuda_status(tt::gelu_launch(dtype, out, x, bias, rows, n, approximate, vb, stream));
}

tt_status split_any(int dtype, void* q, void* k, void* v, const void* qkv, const void* bias,
                    int64_t B, int64_t S, int64_t H, int64_t D, cudaStream_t stream) {
    if (dtype < 0 || dtype > 2 || B < 0 || S < 0 || H < 0 || D < 0) return TT_ERROR_INVALID_VALUE;
    int64_t bs, n, nb;
    if (mul_overflows(B, S, &bs) || mul_overflows(bs, 3 * H, &n) || mul_overflows(n, D, &n) ||
        mul_overflows(n, elem_bytes(dtype), &nb))
        return TT_ERROR_INVALID_VALUE;
    if (n == 0) return TT_SUCCESS;
    if (!q || !k || !v || !qkv || !bias) return TT_ERROR_INVALID_VALUE;
    const int64_t part = nb / 3, pb = 3 * H * D * elem_bytes(dtype);
    const void* outs[3] = {q, k, v};
    for (int i = 0; i < 3; ++i) {
        if (overlaps(outs[i], part, qkv, nb) || overlaps(outs[i], part, bias, pb))
            return TT_ERROR_INVALID_VALUE;
        for (int j = i + 1; j < 3; ++j)
            if (overlaps(outs[i], part, outs[j], part)) return TT_ERROR_INVALID_VALUE;
    }
    const void* ps[5] = {q, k, v, qkv, bias};
    for (const void* p : ps)
        if (reinterpret_cast<uintptr_t>(p) & (uintptr_t)(elem_bytes(dtype) - 1))
            return TT_ERROR_NOT_SUPPORTED;
    if (n >= (int64_t)0xffffffffLL) return TT_ERROR_NOT_SUPPORTED;
    const int64_t pitch = D * elem_bytes(dtype);
    const int vb = vec16(ps, 5, &pitch, 1);
    return cuda_status(tt::split_qkv_launch(dtype, q, k, v, qkv, bias, B, S, H, D, vb, stream));
}

tt_status merge_any(int dtype, void* out, const void* in, int64_t B, int64_t S, int64_t H,
                    int64_t D, cudaStream_t stream) {
    if (dtype < 0 || dtype > 2 || B < 0 || S < 0 || H < 0 || D < 0) return TT_ERROR_INVALID_VALUE;
    int64_t bs, n, nb;
    if (mul_overflows(B, S, &bs) || mul_overflows(bs, H, &n) || mul_overflows(n, D, &n) ||
        mul_overflows(n, elem_bytes(dtype), &nb))
        return TT_ERROR_INVALID_VALUE;
    if (n == 0) return TT_SUCCESS;
    if (!out || !in) return TT_ERROR_INVALID_VALUE;
    if (overlaps(out, nb, in, nb)) return TT_ERROR_INVALID_VALUE;
    if ((reinterpret_cast<uintptr_t>(out) | reinterpret_cast<uintptr_t>(in)) &
        (uintptr_t)(elem_bytes(dtype) - 1))
        return TT_ERROR_NOT_SUPPORTED;
    if (n >= (int64_t)0xffffffffLL) return TT_ERROR_NOT_SUPPORTED;
    const void* ps[2] = {out, in};
    const int64_t pitch = D * elem_bytes(dtype);
    const int vb = vec16(ps, 2, &pitch, 1);
    return cuda_status(tt::merge_heads_launch(dtype, out, in, B, S, H, D, vb, stream));
}

tt_status attention_any(int dtype, void* out, const void* q, const void* k, const void* v,
                        const int32_t* lengths, int64_t B, int64_t H, int64_t S, int64_t D,
                        float scale, cudaStream_t stream) {
    if (dtype < 0 || dtype > 2 || B < 0 || H < 0 || S < 0 || D < 0 || !isfinite(scale))
        return TT_ERROR_INVALID_VALUE;
    int64_t bh, n, nb;
    if (mul_overflows(B, H, &bh) || mul_overflows(bh, S, &n) || mul_overflows(n, D, &n) ||
        mul_overflows(n, elem_bytes(dtype), &nb))
        return TT_ERROR_INVALID_VALUE;
    if (n == 0) return TT_SUCCESS;
    if (!out || !q || !k || !v || !lengths) return TT_ERROR_INVALID_VALUE;
    const void* ins[3] = {q, k, v};
    for (const void* p : ins)
        if (overlaps(out, nb, p, nb)) return TT_ERROR_INVALID_VALUE;
    if (dtype == 0 || D != 64) return TT_ERROR_NOT_SUPPORTED;
    const void* ps[4] = {out, q, k, v};
    for (const void* p : ps)
        if (!aligned16(p)) return TT_ERROR_NOT_SUPPORTED;
    if (reinterpret_cast<uintptr_t>(lengths) & 3u) return TT_ERROR_NOT_SUPPORTED;
    if (B > 65535 || H > 65535 || S > 0x7fffffffLL) return TT_ERROR_NOT_SUPPORTED;
    return cuda_status(tt::attention_launch(dtype, out, q, k, v, lengths, B, H, S, scale, stream));
}

// ------------------------------------------------------------------- packed
tt_status packed_validate(int dtype, const void* scores, const int32_t* cu, const int64_t* blocks,
                          int64_t num_req, int64_t H, int64_t total_tokens, int64_t max_len,
                          float scale, bool check_ptrs, bool* empty) {
    if (dtype < 0 || dtype > 2) return TT_ERROR_INVALID_VALUE;
    if (num_req < 0 || H < 0 || total_tokens < 0 || max_len < 0) return TT_ERROR_INVALID_VALUE;
    if (!isfinite(scale)) return TT_ERROR_INVALID_VALUE;
    if (num_req > 0x7fffffffLL) return TT_ERROR_INVALID_VALUE;
    *empty = (num_req == 0 || H == 0 || total_tokens == 0 || max_len == 0);
    if (*empty) return TT_SUCCESS;
    if (check_ptrs) {
        if (!scores || !cu || !blocks) return TT_ERROR_INVALID_VALUE;
        if (!aligned16(scores) || (reinterpret_cast<uintptr_t>(cu) & 3u) ||
            (reinterpret_cast<uintptr_t>(blocks) & 7u))
            return TT_ERROR_NOT_SUPPORTED;
    }
    int64_t rows;
    if (mul_overflows(H, total_tokens, &rows) || rows >= (int64_t)0xffffffffLL)
        return TT_ERROR_NOT_SUPPORTED;
    if (max_len > tt::softmax_packed_max_len(dtype)) return TT_ERROR_NOT_SUPPORTED;
    return TT_SUCCESS;
}

tt_status packed_any(int dtype, void* scores, const int32_t* cu, const int64_t* blocks,
                     int64_t num_req, int64_t H, int64_t total_tokens, int64_t max_len,
                     float scale, cudaStream_t stream) {
    bool empty = false;
    tt_status s = packed_validate(dtype, scores, cu, blocks, num_req, H, total_tokens, max_len,
                                  scale, true, &empty);
    if (s != TT_SUCCESS || empty) return s;
    bool supported = false;
    cudaError_t e = tt::softmax_packed_launch(dtype, scores, cu, blocks, num_req, H, total_tokens,
                                              max_len, scale, stream, &supported);
    if (!supported) return TT_ERROR_NOT_SUPPORTED;
    return cuda_status(e);
}

void copy_name(const char* name, char* buf, int cap) {
    if (!buf || cap <= 0) return;
    snprintf(buf, (size_t)cap, "%s", name ? name : "");
}

}  // namespace

namespace tt {
std::atomic<int> g_pdl{1};
bool pdl_enabled() { return g_pdl.load(std::memory_order_relaxed) != 0; }

// (kernel, device) -> dynamic shared memory bytes already opted in.  The
// attribute is per device context: a process driving several GPUs must set it
// on each.  Only launches above 48 KB come here.
cudaError_t smem_optin(const void* kern, size_t smem) {
    if (smem <= 48 * 1024) return cudaSuccess;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, size_t> done;
    std::lock_guard<std::mutex> lk(mu);
    size_t& have = done[{kern, dev}];
    if (have >= smem) return cudaSuccess;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess) have = smem;
    return e;
}
}  // namespace tt

extern "C" {

tt_status tt_softmax_masked_f32(float* scores, const int32_t* lengths, int64_t B, int64_t H,
                                int64_t Sq, int64_t Sk, float scale, cudaStream_t stream) {
    return softmax_any(0, scores, lengths, B, H, Sq, Sk, scale, stream);
}
tt_status tt_softmax_masked_f16(void* scores, const int32_t* lengths, int64_t B, int64_t H,
                                int64_t Sq, int64_t Sk, float scale, cudaStream_t stream) {
    return softmax_any(1, scores, lengths, B, H, Sq, Sk, scale, stream);
}
tt_status tt_softmax_masked_bf16(void* scores, const int32_t* lengths, int64_t B, int64_t H,
                                 int64_t Sq, int64_t Sk, float scale, cudaStream_t stream) {
    return softmax_any(2, scores, lengths, B, H, Sq, Sk, scale, stream);
}

tt_status tt_softmax_packed_f32(float* scores, const int32_t* cu_seqlens, const int64_t* cu_blocks,
                                int64_t num_req, int64_t H, int64_t total_tokens,
                                int64_t max_seqlen, float scale, cudaStream_t stream) {
    return packed_any(0, scores, cu_seqlens, cu_blocks, num_req, H, total_tokens, max_seqlen,
                      scale, stream);
}
tt_status tt_softmax_packed_f16(void* scores, const int32_t* cu_seqlens, const int64_t* cu_blocks,
                                int64_t num_req, int64_t H, int64_t total_tokens,
                                int64_t max_seqlen, float scale, cudaStream_t stream) {
    return packed_any(1, scores, cu_seqlens, cu_blocks, num_req, H, total_tokens, max_seqlen,
                      scale, stream);
}
tt_status tt_softmax_packed_bf16(void* scores, const int32_t* cu_seqlens,
                                 const int64_t* cu_blocks, int64_t num_req, int64_t H,
                                 int64_t total_tokens, int64_t max_seqlen, float scale,
                                 cudaStream_t stream) {
    return packed_any(2, scores, cu_seqlens, cu_blocks, num_req, H, total_tokens, max_seqlen,
                      scale, stream);
}

tt_status tt_add_bias_layernorm_f32(float* out, const float* x, const float* residual,
                                    const float* bias, const float* gamma, const float* beta,
                                    int64_t rows, int64_t hidden, float eps, cudaStream_t stream) {
    return ln_any(0, out, x, residual, bias, gamma, beta, rows, hidden, eps, stream);
}
tt_status tt_add_bias_layernorm_f16(void* out, const void* x, const void* residual,
                                    const void* bias, const void* gamma, const void* beta,
                                    int64_t rows, int64_t hidden, float eps, cudaStream_t stream) {
    return ln_any(1, out, x, residual, bias, gamma, beta, rows, hidden, eps, stream);
}
tt_status tt_add_bias_layernorm_bf16(void* out, const void* x, const void* residual,
                                     const void* bias, const void* gamma, const void* beta,
                                     int64_t rows, int64_t hidden, float eps, cudaStream_t stream) {
    return ln_any(2, out, x, residual, bias, gamma, beta, rows, hidden, eps, stream);
}

tt_status tt_attention_fwd(int dtype, void* out, const void* q, const void* k, const void* v,
                           const int32_t* lengths, int64_t B, int64_t H, int64_t S, int64_t D,
                           float scale, cudaStream_t stream) {
    return attention_any(dtype, out, q, k, v, lengths, B, H, S, D, scale, stream);
}

tt_status tt_add_bias_gelu(int dtype, void* out, const void* x, const void* bias, int64_t rows,
                           int64_t n, int approximate, cudaStream_t stream) {
    return gelu_any(dtype, out, x, bias, rows, n, approximate, stream);
}

tt_status tt_split_qkv_add_bias(int dtype, void* q, void* k, void* v, const void* qkv,
                                const void* bias, int64_t B, int64_t S, int64_t H, int64_t D,
                                cudaStream_t stream) {
    return split_any(dtype, q, k, v, qkv, bias, B, S, H, D, stream);
}

tt_status tt_merge_heads(int dtype, void* out, const void* in, int64_t B, int64_t S, int64_t H,
                         int64_t D, cudaStream_t stream) {
    return merge_any(dtype, out, in, B, S, H, D, stream);
}

tt_status tt_softmax_masked_staged(int dtype, void* host_scores, const int32_t* host_lengths,
                                   void* dev_scores, int32_t* dev_lengths, int64_t B, int64_t H,
                                   int64_t Sq, int64_t Sk, float scale, cudaStream_t stream) {
    int64_t nrows = 0;
    bool empty = false;
    tt_status s = softmax_validate(dtype, dev_scores, dev_lengths, B, H, Sq, Sk, scale, true,
                                   &nrows, &empty);
    if (s != TT_SUCCESS || empty) return s;
    if (!host_scores || !host_lengths) return TT_ERROR_INVALID_VALUE;
    const size_t bytes = (size_t)(nrows * Sk * elem_bytes(dtype));
    cudaError_t e = cudaMemcpyAsync(dev_lengths, host_lengths, (size_t)B * sizeof(int32_t),
                                    cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(dev_scores, host_scores, bytes, cudaMemcpyHostToDevice, stream);
    if (e != cudaSuccess) return cuda_status(e);
    s = softmax_any(dtype, dev_scores, dev_lengths, B, H, Sq, Sk, scale, stream);
    if (s != TT_SUCCESS) return s;
    return cuda_status(
        cudaMemcpyAsync(host_scores, dev_scores, bytes, cudaMemcpyDeviceToHost, stream));
}

tt_status tt_add_bias_layernorm_staged(int dtype, void* host_out, const void* host_x,
                                       const void* host_residual, void* dev_out, void* dev_x,
                                       void* dev_residual, const void* bias, const void* gamma,
                                       const void* beta, int64_t rows, int64_t hidden, float eps,
                                       cudaStream_t stream) {
    bool empty = false;
    tt_status s = ln_validate(dtype, dev_out, dev_x, dev_residual, bias, gamma, beta, rows, hidden,
                              eps, true, &empty);
    if (s != TT_SUCCESS || empty) return s;
    if (!host_out || !host_x || !host_residual) return TT_ERROR_INVALID_VALUE;
    // both are H2D copy targets: overlapping, the residual copy would overwrite x
    if (overlaps(dev_x, rows * hidden * elem_bytes(dtype), dev_residual,
                 rows * hidden * elem_bytes(dtype)))
        return TT_ERROR_INVALID_VALUE;
    const size_t bytes = (size_t)(rows * hidden * elem_bytes(dtype));
    cudaError_t e = cudaMemcpyAsync(dev_x, host_x, bytes, cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(dev_residual, host_residual, bytes, cudaMemcpyHostToDevice, stream);
    if (e != cudaSuccess) return cuda_status(e);
    s = ln_any(dtype, dev_out, dev_x, dev_residual, bias, gamma, beta, rows, hidden, eps, stream);
    if (s != TT_SUCCESS) return s;
    return cuda_status(cudaMemcpyAsync(host_out, dev_out, bytes, cudaMemcpyDeviceToHost, stream));
}

// ---- overlapped staging: chunks of requests (softmax) or rows (LN) go H2D and
// through the kernel on `stream` while the previous chunk's result goes D2H on
// `copy_stream` (the two copy directions run concurrently over PCIe).  `stream`
// finally waits for the last D2H, so the caller's contract is unchanged: the host
// result is ready when `stream` completes.
namespace {

int64_t gcd64(int64_t a, int64_t b) {
    while (b) {
        const int64_t t = a % b;
        a = b;
        b = t;
    }
    return a;
}

// Units per chunk: a multiple of the granule that keeps every chunk's device
// base 16-byte aligned (unit_bytes * granule % 16 == 0).
int64_t chunk_units(int64_t units, int64_t chunks, int64_t unit_bytes) {
    const int64_t gran = 16 / gcd64(unit_bytes % 16 == 0 ? 16 : unit_bytes % 16, 16);
    if (chunks < 1) chunks = 1;
    int64_t per = (units + chunks - 1) / chunks;
    per = ((per + gran - 1) / gran) * gran;
    return per > 0 ? per : 1;
}

struct EventGuard {
    cudaEvent_t ev = nullptr;
    ~EventGuard() {
        if (ev) cudaEventDestroy(ev);  // released once its last record completes
    }
};

}  // namespace

tt_status tt_softmax_masked_staged_overlap(int dtype, void* host_scores,
                                           const int32_t* host_lengths, void* dev_scores,
                                           int32_t* dev_lengths, int64_t B, int64_t H, int64_t Sq,
                                           int64_t Sk, float scale, int64_t chunks,
                                           cudaStream_t stream, cudaStream_t copy_stream) {
    if (!copy_stream || copy_stream == stream || chunks <= 1)
        return tt_softmax_masked_staged(dtype, host_scores, host_lengths, dev_scores, dev_lengths,
                                        B, H, Sq, Sk, scale, stream);
    int64_t nrows = 0;
    bool empty = false;
    tt_status s = softmax_validate(dtype, dev_scores, dev_lengths, B, H, Sq, Sk, scale, true,
                                   &nrows, &empty);
    if (s != TT_SUCCESS || empty) return s;
    if (!host_scores || !host_lengths) return TT_ERROR_INVALID_VALUE;
    const int64_t req_bytes = H * Sq * Sk * elem_bytes(dtype);
    const int64_t per = chunk_units(B, chunks, req_bytes);
    EventGuard g;
    cudaError_t e = cudaEventCreateWithFlags(&g.ev, cudaEventDisableTiming);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(dev_lengths, host_lengths, (size_t)B * sizeof(int32_t),
                            cudaMemcpyHostToDevice, stream);
    if (e != cudaSuccess) return cuda_status(e);
    for (int64_t b0 = 0; b0 < B; b0 += per) {
        const int64_t nb = B - b0 < per ? B - b0 : per;
        const size_t off = (size_t)(b0 * req_bytes), bytes = (size_t)(nb * req_bytes);
        char* d = static_cast<char*>(dev_scores) + off;
        char* h = static_cast<char*>(host_scores) + off;
        e = cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, stream);
        if (e != cudaSuccess) return cuda_status(e);
        s = softmax_any(dtype, d, dev_lengths + b0, nb, H, Sq, Sk, scale, stream);
        if (s != TT_SUCCESS) return s;
        e = cudaEventRecord(g.ev, stream);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(copy_stream, g.ev, 0);
        if (e == cudaSuccess) e = cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, copy_stream);
        if (e != cudaSuccess) return cuda_status(e);
    }
    e = cudaEventRecord(g.ev, copy_stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(stream, g.ev, 0);
    return cuda_status(e);
}

tt_status tt_add_bias_layernorm_staged_overlap(int dtype, void* host_out, const void* host_x,
                                               const void* host_residual, void* dev_out,
                                               void* dev_x, void* dev_residual, const void* bias,
                                               const void* gamma, const void* beta, int64_t rows,
                                               int64_t hidden, float eps, int64_t chunks,
                                               cudaStream_t stream, cudaStream_t copy_stream) {
    if (!copy_stream || copy_stream == stream || chunks <= 1)
        return tt_add_bias_layernorm_staged(dtype, host_out, host_x, host_residual, dev_out, dev_x,
                                            dev_residual, bias, gamma, beta, rows, hidden, eps,
                                            stream);
    bool empty = false;
    tt_status s = ln_validate(dtype, dev_out, dev_x, dev_residual, bias, gamma, beta, rows, hidden,
                              eps, true, &empty);
    if (s != TT_SUCCESS || empty) return s;
    if (!host_out || !host_x || !host_residual) return TT_ERROR_INVALID_VALUE;
    // both are H2D copy targets: overlapping, the residual copy would overwrite x
    if (overlaps(dev_x, rows * hidden * elem_bytes(dtype), dev_residual,
                 rows * hidden * elem_bytes(dtype)))
        return TT_ERROR_INVALID_VALUE;
    const int64_t row_bytes = hidden * elem_bytes(dtype);
    const int64_t per = chunk_units(rows, chunks, row_bytes);
    EventGuard g;
    cudaError_t e = cudaEventCreateWithFlags(&g.ev, cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_status(e);
    for (int64_t r0 = 0; r0 < rows; r0 += per) {
        const int64_t nr = rows - r0 < per ? rows - r0 : per;
        const size_t off = (size_t)(r0 * row_bytes), bytes = (size_t)(nr * row_bytes);
        char* dx = static_cast<char*>(dev_x) + off;
        char* dr = static_cast<char*>(dev_residual) + off;
        char* dout = static_cast<char*>(dev_out) + off;
        e = cudaMemcpyAsync(dx, static_cast<const char*>(host_x) + off, bytes,
                            cudaMemcpyHostToDevice, stream);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(dr, static_cast<const char*>(host_residual) + off, bytes,
                                cudaMemcpyHostToDevice, stream);
        if (e != cudaSuccess) return cuda_status(e);
        s = ln_any(dtype, dout, dx, dr, bias, gamma, beta, nr, hidden, eps, stream);
        if (s != TT_SUCCESS) return s;
        e = cudaEventRecord(g.ev, stream);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(copy_stream, g.ev, 0);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(static_cast<char*>(host_out) + off, dout, bytes,
                                cudaMemcpyDeviceToHost, copy_stream);
        if (e != cudaSuccess) return cuda_status(e);
    }
    e = cudaEventRecord(g.ev, copy_stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(stream, g.ev, 0);
    return cuda_status(e);
}

const char* tt_status_string(tt_status s) {
    switch (s) {
        case TT_SUCCESS: return "TT_SUCCESS";
        case TT_ERROR_INVALID_VALUE: return "TT_ERROR_INVALID_VALUE";
        case TT_ERROR_NOT_SUPPORTED: return "TT_ERROR_NOT_SUPPORTED";
        case TT_ERROR_CUDA: return "TT_ERROR_CUDA";
        default: return "TT_UNKNOWN_STATUS";
    }
}

int tt_last_cuda_error(void) { return g_last_cuda_error; }

int tt_version(void) { return kVersion; }

tt_status tt_softmax_masked_plan(int dtype, int64_t B, int64_t H, int64_t Sq, int64_t Sk,
                                 char* buf, int cap) {
    int64_t nrows = 0;
    bool empty = false;
    tt_status s = softmax_validate(dtype, nullptr, nullptr, B, H, Sq, Sk, 1.0f, false, &nrows,
                                   &empty);
    if (s != TT_SUCCESS) {
        copy_name("", buf, cap);
        return s;
    }
    copy_name(empty ? "none" : tt::softmax_tier_name(dtype, Sk, nrows), buf, cap);
    return TT_SUCCESS;
}

tt_status tt_add_bias_layernorm_plan(int dtype, int64_t rows, int64_t hidden, char* buf, int cap) {
    bool empty = false;
    tt_status s = ln_validate(dtype, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, rows,
                              hidden, 0.f, false, &empty);
    if (s != TT_SUCCESS) {
        copy_name("", buf, cap);
        return s;
    }
    if (empty) {
        copy_name("none", buf, cap);
        return TT_SUCCESS;
    }
    // plan for 256-byte-aligned operands (every cudaMalloc / PyTorch allocation)
    const int e = elem_bytes(dtype);
    int vb = e;
    for (int c = 32; c >= e; c >>= 1)
        if ((hidden * e) % c == 0) {
            vb = c;
            break;
        }
    copy_name(tt::layernorm_tier_name(dtype, hidden, vb, rows), buf, cap);
    return TT_SUCCESS;
}

tt_status tt_softmax_packed_plan(int dtype, int64_t max_seqlen, char* buf, int cap) {
    bool empty = false;
    tt_status s = packed_validate(dtype, nullptr, nullptr, nullptr, 1, 1, 1, max_seqlen, 1.0f,
                                  false, &empty);
    if (s != TT_SUCCESS) {
        copy_name("", buf, cap);
        return s;
    }
    copy_name(empty ? "none" : tt::softmax_packed_tier_name(dtype, max_seqlen), buf, cap);
    return TT_SUCCESS;
}

int ttx_tier_count(int op) {
    return op == 0 ? tt::softmax_tier_count() : op == 1 ? tt::layernorm_tier_count() : -1;
}

const char* ttx_tier_name(int op, int dtype, int i) {
    return op == 0 ? tt::softmax_tier_name_at(dtype, i)
                   : op == 1 ? tt::layernorm_tier_name_at(dtype, i) : nullptr;
}

int ttx_attention_variant_count(void) { return tt::attention_variant_count(); }

int ttx_attention_variant_ok(int v) { return tt::attention_variant_ok(v) ? 1 : 0; }

int ttx_tuning_build(void) {
#ifdef TT_TUNING
    return 1;
#else
    return 0;
#endif
}

tt_status ttx_attention_variant(int v) {
    return tt::attention_force_variant(v) ? TT_SUCCESS : TT_ERROR_INVALID_VALUE;
}

tt_status ttx_set_pdl(int enable) {
    if (enable != 0 && enable != 1) return TT_ERROR_INVALID_VALUE;
    tt::g_pdl.store(enable, std::memory_order_relaxed);
    return TT_SUCCESS;
}

int ttx_get_pdl(void) { return tt::g_pdl.load(std::memory_order_relaxed); }

tt_status ttx_force_tier(int op, int dtype, int i) {
    bool ok = op == 0 ? tt::softmax_force_tier(dtype, i)
                      : op == 1 ? tt::layernorm_force_tier(dtype, i) : false;
    return ok ? TT_SUCCESS : TT_ERROR_INVALID_VALUE;
}

}  // extern "C"
