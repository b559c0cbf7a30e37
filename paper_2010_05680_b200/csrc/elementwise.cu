// elementwise.cu -- NEXT-2: the element-wise non-GEMM kernels of
// the fused transformer graph, "fused activation functions and fused
// transpose operations" (K4 / K5 in SURVEY §2.2):
//
//   add_bias_gelu      out = gelu(x + bias) over [rows, n]   (FFN-up epilogue)
//   split_qkv_add_bias qkv [B*S, 3*H*D] + bias -> q, k, v [B, H, S, D]
//   merge_heads        [B, H, S, D] -> [B*S, H*D]            (after P.V)
//
// All three are pure streaming kernels (every byte read once, written once),
// HBM-bound like the reductions.  They move VB-byte vectors (16 B, or the
// element size when alignment / pitch forbid), fp32 arithmetic, RNE narrowing.
#include <atomic>

#include "common.cuh"
#include "launch.h"

namespace tt {

namespace {

template <typename T, int VB>
__device__ __forceinline__ void add_vec(Raw<VB>& w, const Raw<VB>& b) {
    constexpr int VE = VB / (int)sizeof(T);
    float f[VE], g[VE];
    Elem<T>::template unpack<VB>(w, f);
    Elem<T>::template unpack<VB>(b, g);
#pragma unroll
    for (int e = 0; e < VE; ++e) f[e] += g[e];
    Elem<T>::template pack<VB>(f, w);
}

int sm_count_e() {
    static int cached[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!cached[dev]) {
        int n = 0;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        cached[dev] = n > 0 ? n : 148;
    }
    return cached[dev];
}

}  // namespace

// ---------------------------------------------------------------- GELU
// erf(x) via Abramowitz & Stegun 7.1.26 (|error| <= 1.5e-7 absolute):
//   erf(|x|) = 1 - t (a1 + t (a2 + t (a3 + t (a4 + t a5)))) exp(-x^2),
//   t = 1 / (1 + p |x|)
// with the reciprocal and the exponential on the MUFU (rcp.approx,
// ex2.approx): ~12 instructions against ~25 for the libdevice erff, which
// made the kernel issue-bound.  gelu error <= 0.5 |v| * 2e-7.
__device__ __forceinline__ float erf_as(float x) {
    const float ax = fabsf(x);
    float t;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t) : "f"(fmaf(0.3275911f, ax, 1.0f)));
    float p = fmaf(1.061405429f, t, -1.453152027f);
    p = fmaf(p, t, 1.421413741f);
    p = fmaf(p, t, -0.284496736f);
    p = fmaf(p, t, 0.254829592f);
    p *= t;
    const float e = ex2_approx(-1.4426950408889634f * ax * ax);
    return copysignf(fmaf(-p, e, 1.0f), x);
}

// The same A&S 7.1.26 erf for a pair of arguments on packed fp32 (FFMA2 /
// FMUL2): the polynomial and the argument scaling cost one issue slot per two
// elements; rcp and ex2 stay on the MUFU.  Returns gelu(v) = 0.5 v (1 + erf(v / sqrt 2))
// for the pair v2.
__device__ __forceinline__ F2 gelu_erf2(F2 v2) {
    const F2 hv2 = f2_mul(v2, f2_make(0.5f, 0.5f));
    float v0, v1;
    f2_split(v2, v0, v1);
    const F2 ax2 = f2_make(fabsf(v0) * 0.7071067811865476f, fabsf(v1) * 0.7071067811865476f);
    float d0, d1;
    f2_split(f2_fma(ax2, f2_make(0.3275911f, 0.3275911f), f2_make(1.0f, 1.0f)), d0, d1);
    float t0, t1;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t0) : "f"(d0));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t1) : "f"(d1));
    const F2 t2 = f2_make(t0, t1);
    // -(a1 + t (a2 + t (a3 + t (a4 + t a5)))) t, negated coefficients
    F2 p2 = f2_fma(f2_make(-1.061405429f, -1.061405429f), t2, f2_make(1.453152027f, 1.453152027f));
    p2 = f2_fma(p2, t2, f2_make(-1.421413741f, -1.421413741f));
    p2 = f2_fma(p2, t2, f2_make(0.284496736f, 0.284496736f));
    p2 = f2_fma(p2, t2, f2_make(-0.254829592f, -0.254829592f));
    p2 = f2_mul(p2, t2);
    float a0, a1;
    f2_split(f2_mul(f2_mul(ax2, ax2), f2_make(-1.4426950408889634f, -1.4426950408889634f)), a0, a1);
    const F2 e2 = f2_make(ex2_approx(a0), ex2_approx(a1));
    float r0, r1;
    f2_split(f2_fma(p2, e2, f2_make(1.0f, 1.0f)), r0, r1);  // erf(|x|)
    const F2 erf2 = f2_make(copysignf(r0, v0), copysignf(r1, v1));
    return f2_fma(hv2, erf2, hv2);
}

__device__ __forceinline__ float tanh_approx(float x) {
    float y;
    asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// One CTA walks RPB rows; each thread takes the row's vectors tid, tid + NT, ...
// (bias vectors are the same for every row, so they stay in L1).  The tanh
// form uses MUFU.TANH (rel. error ~2^-11) for 16-bit outputs, whose own
// rounding is coarser, and the accurate tanhf for fp32.
template <typename T, int VB, bool APPROX, int NT, int U>
__global__ void __launch_bounds__(NT) add_bias_gelu_kernel(T* out, const T* x,
                                                           const T* __restrict__ bias,
                                                           int64_t rows, int n, int rpb,
                                                           FastDivU32 div_nvec) {
    PdlScope pdl_;  // griddepcontrol.wait first: no global access before it (PDL)
    constexpr int VE = VB / (int)sizeof(T);
    const int nvec = n / VE;
    const int64_t r0 = (int64_t)blockIdx.x * rpb;
    const int64_t r1 = min(rows, r0 + rpb);
    if (r1 <= r0) return;
    // the CTA's rows are one contiguous span of (r1 - r0) * nvec vectors; vector
    // f of the span uses bias vector f mod nvec.  U vectors per thread in
    // flight: every load of a batch is issued before the (MUFU-heavy) GELU
    // arithmetic of the first.
    const T* xs = x + r0 * (int64_t)n;
    T* os = out + r0 * (int64_t)n;
    const int nf = (int)(r1 - r0) * nvec;
    for (int f0 = threadIdx.x; f0 < nf; f0 += NT * U) {
        Raw<VB> wx[U], wb[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int fi = f0 + u * NT;
            if (fi < nf) {
                const int bi = fi - (int)div_nvec.div((uint32_t)fi) * nvec;
                ld_stream<VB>(xs + (int64_t)fi * VE, wx[u]);
                ld_param<VB>(bias + bi * VE, wb[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int fi = f0 + u * NT;
            if (fi >= nf) break;
            float fv[VE], g[VE];
            Elem<T>::template unpack<VB>(wx[u], fv);
            Elem<T>::template unpack<VB>(wb[u], g);
            if constexpr (APPROX) {
#pragma unroll
                for (int e = 0; e < VE; ++e) {
                    const float v = fv[e] + g[e];
                    const float hv = 0.5f * v;
                    const float uu = 0.7978845608028654f * fmaf(0.044715f * v, v * v, v);
                    const float th = sizeof(T) == 4 ? tanhf(uu) : tanh_approx(uu);
                    fv[e] = fmaf(hv, th, hv);
                }
            } else if constexpr (VE % 2 == 0) {
#pragma unroll
                for (int e = 0; e < VE; e += 2)
                    f2_split(gelu_erf2(f2_add(f2_make(fv[e], fv[e + 1]), f2_make(g[e], g[e + 1]))),
                             fv[e], fv[e + 1]);
            } else {
#pragma unroll
                for (int e = 0; e < VE; ++e) {
                    const float v = fv[e] + g[e];
                    const float hv = 0.5f * v;
                    fv[e] = fmaf(hv, erf_as(v * 0.7071067811865476f), hv);
                }
            }
            Raw<VB> wy;
            Elem<T>::template pack<VB>(fv, wy);
            st_stream<VB>(os + (int64_t)fi * VE, wy);
        }
    }
}

constexpr int64_t kGeluBigVecs = 4 << 20;  // calls of >= 4 M vectors: 4 per thread in flight
template <typename T, int VB, bool APPROX>
cudaError_t launch_gelu(void* out, const void* x, const void* bias, int64_t rows, int64_t n,
                        cudaStream_t st) {
    constexpr int NT = 256;
    const int64_t nvec = n / (VB / (int)sizeof(T));
    // rows per CTA: enough vectors per CTA to amortise, enough CTAs to fill
    // the SMs several times over
    int64_t rpb = (4 * NT + nvec - 1) / nvec;
    const int64_t max_rpb = (rows + 4 * (int64_t)sm_count_e() - 1) / (4 * (int64_t)sm_count_e());
    if (rpb > max_rpb) rpb = max_rpb > 0 ? max_rpb : 1;
    const int64_t grid = (rows + rpb - 1) / rpb;
    if (grid > 0x7fffffffLL || rpb * nvec > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
    {
        // 4 vectors per thread in flight on large calls (BERT-large FFN: 101 -> 94 us);
        // small calls, a few waves of CTAs, are latency-bound and prefer one
        // (BERT-base b20 s128: 9.3 -> 8.6 us; profiles/r02_next2/)
        auto kern = rows * nvec >= kGeluBigVecs ? add_bias_gelu_kernel<T, VB, APPROX, NT, 4>
                                                : add_bias_gelu_kernel<T, VB, APPROX, NT, 1>;
        const cudaError_t le_ = launch_k(kern, (unsigned)grid, NT, 0, st,
        static_cast<T*>(out), static_cast<const T*>(x), static_cast<const T*>(bias), rows,
        (int)n, (int)rpb, FastDivU32::make((uint32_t)nvec));
        if (le_ != cudaSuccess) return le_;
    }
    return cudaGetLastError();
}

// ---------------------------------------------------------------- QKV split
// work item = one D-vector (token, t, h): GD = D / VE lanes per item; items in
// token-major order so the qkv reads are contiguous.
template <typename T, int VB, int NT>
__global__ void __launch_bounds__(NT) split_qkv_kernel(T* q, T* k, T* v, const T* qkv,
                                                       const T* __restrict__ bias, uint32_t S,
                                                       uint32_t H, uint32_t D, uint64_t total,
                                                       FastDivU32 div_gd, FastDivU32 div_3h,
                                                       FastDivU32 div_s) {
    PdlScope pdl_;  // griddepcontrol.wait first: no global access before it (PDL)
    constexpr int VE = VB / (int)sizeof(T);
    const uint32_t gd = D / VE;
    for (uint64_t i = (uint64_t)blockIdx.x * NT + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * NT) {
        const uint32_t item = div_gd.div((uint32_t)i);
        const uint32_t lane = (uint32_t)i - item * gd;
        const uint32_t token = div_3h.div(item);
        const uint32_t th = item - token * 3 * H;  // t * H + h
        const uint32_t t = th >= 2 * H ? 2 : (th >= H ? 1 : 0);
        const uint32_t h = th - t * H;
        const uint32_t b = div_s.div(token);
        const uint32_t s = token - b * S;
        Raw<VB> w, wb;
        ld_stream<VB>(qkv + (uint64_t)item * D + lane * VE, w);
        ld_param<VB>(bias + (uint64_t)th * D + lane * VE, wb);
        add_vec<T, VB>(w, wb);
        T* dst = t == 0 ? q : (t == 1 ? k : v);
        st_stream<VB>(dst + (((uint64_t)b * H + h) * S + s) * D + lane * VE, w);
    }
}

template <typename T, int VB>
cudaError_t launch_split(void* q, void* k, void* v, const void* qkv, const void* bias,
                         int64_t B, int64_t S, int64_t H, int64_t D, cudaStream_t st) {
    constexpr int NT = 256;
    const uint64_t gd = (uint64_t)(D / (VB / (int)sizeof(T)));
    const uint64_t total = (uint64_t)B * S * 3 * H * gd;
    if (total >= 0xffffffffull) return cudaErrorInvalidConfiguration;
    const uint64_t want = (total + NT - 1) / NT;
    const uint64_t cap = (uint64_t)sm_count_e() * 16;
    const unsigned grid = (unsigned)(want < cap ? want : cap);
    {
        const cudaError_t le_ = launch_k(split_qkv_kernel<T, VB, NT>, grid, NT, 0, st,
        static_cast<T*>(q), static_cast<T*>(k), static_cast<T*>(v), static_cast<const T*>(qkv),
        static_cast<const T*>(bias), (uint32_t)S, (uint32_t)H, (uint32_t)D, total,
        FastDivU32::make((uint32_t)gd), FastDivU32::make((uint32_t)(3 * H)),
        FastDivU32::make((uint32_t)S));
        if (le_ != cudaSuccess) return le_;
    }
    return cudaGetLastError();
}

// ---------------------------------------------------------------- head merge
// work item = one D-vector (token, h) in output order (token-major, h inner)
template <typename T, int VB, int NT>
__global__ void __launch_bounds__(NT) merge_heads_kernel(T* out, const T* in, uint32_t S,
                                                         uint32_t H, uint32_t D, uint64_t total,
                                                         FastDivU32 div_gd, FastDivU32 div_h,
                                                         FastDivU32 div_s) {
    PdlScope pdl_;  // griddepcontrol.wait first: no global access before it (PDL)
    constexpr int VE = VB / (int)sizeof(T);
    const uint32_t gd = D / VE;
    for (uint64_t i = (uint64_t)blockIdx.x * NT + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * NT) {
        const uint32_t item = div_gd.div((uint32_t)i);
        const uint32_t lane = (uint32_t)i - item * gd;
        const uint32_t token = div_h.div(item);
        const uint32_t h = item - token * H;
        const uint32_t b = div_s.div(token);
        const uint32_t s = token - b * S;
        Raw<VB> w;
        ld_stream<VB>(in + (((uint64_t)b * H + h) * S + s) * D + lane * VE, w);
        st_stream<VB>(out + (uint64_t)item * D + lane * VE, w);
    }
}

template <typename T, int VB>
cudaError_t launch_merge(void* out, const void* in, int64_t B, int64_t S, int64_t H, int64_t D,
                         cudaStream_t st) {
    constexpr int NT = 256;
    const uint64_t gd = (uint64_t)(D / (VB / (int)sizeof(T)));
    const uint64_t total = (uint64_t)B * S * H * gd;
    if (total >= 0xffffffffull) return cudaErrorInvalidConfiguration;
    const uint64_t want = (total + NT - 1) / NT;
    const uint64_t cap = (uint64_t)sm_count_e() * 16;
    const unsigned grid = (unsigned)(want < cap ? want : cap);
    {
        const cudaError_t le_ = launch_k(merge_heads_kernel<T, VB, NT>, grid, NT, 0, st,
        static_cast<T*>(out), static_cast<const T*>(in), (uint32_t)S, (uint32_t)H, (uint32_t)D,
        total, FastDivU32::make((uint32_t)gd), FastDivU32::make((uint32_t)H),
        FastDivU32::make((uint32_t)S));
        if (le_ != cudaSuccess) return le_;
    }
    return cudaGetLastError();
}

// ---------------------------------------------------------------- dispatch
// vec_bytes (host-computed from pointer alignment and pitches) picks 16-byte
// vectors or the element-size fallback.
namespace {

template <typename T>
cudaError_t gelu_t(void* out, const void* x, const void* bias, int64_t rows, int64_t n,
                   int approximate, int vec_bytes, cudaStream_t st) {
    if (vec_bytes >= 16)
        return approximate ? launch_gelu<T, 16, true>(out, x, bias, rows, n, st)
                           : launch_gelu<T, 16, false>(out, x, bias, rows, n, st);
    return approximate ? launch_gelu<T, sizeof(T), true>(out, x, bias, rows, n, st)
                       : launch_gelu<T, sizeof(T), false>(out, x, bias, rows, n, st);
}

template <typename T>
cudaError_t split_t(void* q, void* k, void* v, const void* qkv, const void* bias, int64_t B,
                    int64_t S, int64_t H, int64_t D, int vec_bytes, cudaStream_t st) {
    if (vec_bytes >= 16) return launch_split<T, 16>(q, k, v, qkv, bias, B, S, H, D, st);
    return launch_split<T, sizeof(T)>(q, k, v, qkv, bias, B, S, H, D, st);
}

template <typename T>
cudaError_t merge_t(void* out, const void* in, int64_t B, int64_t S, int64_t H, int64_t D,
                    int vec_bytes, cudaStream_t st) {
    if (vec_bytes >= 16) return launch_merge<T, 16>(out, in, B, S, H, D, st);
    return launch_merge<T, sizeof(T)>(out, in, B, S, H, D, st);
}

}  // namespace

cudaError_t gelu_launch(int dtype, void* out, const void* x, const void* bias, int64_t rows,
                        int64_t n, int approximate, int vec_bytes, cudaStream_t stream) {
    switch (dtype) {
        case 0: return gelu_t<float>(out, x, bias, rows, n, approximate, vec_bytes, stream);
        case 1: return gelu_t<__half>(out, x, bias, rows, n, approximate, vec_bytes, stream);
        default:
            return gelu_t<__nv_bfloat16>(out, x, bias, rows, n, approximate, vec_bytes, stream);
    }
}

cudaError_t split_qkv_launch(int dtype, void* q, void* k, void* v, const void* qkv,
                             const void* bias, int64_t B, int64_t S, int64_t H, int64_t D,
                             int vec_bytes, cudaStream_t stream) {
    switch (dtype) {
        case 0: return split_t<float>(q, k, v, qkv, bias, B, S, H, D, vec_bytes, stream);
        case 1: return split_t<__half>(q, k, v, qkv, bias, B, S, H, D, vec_bytes, stream);
        default:
            return split_t<__nv_bfloat16>(q, k, v, qkv, bias, B, S, H, D, vec_bytes, stream);
    }
}

cudaError_t merge_heads_launch(int dtype, void* out, const void* in, int64_t B, int64_t S,
                               int64_t H, int64_t D, int vec_bytes, cudaStream_t stream) {
    switch (dtype) {
        case 0: return merge_t<float>(out, in, B, S, H, D, vec_bytes, stream);
        case 1: return merge_t<__half>(out, in, B, S, H, D, vec_bytes, stream);
        default: return merge_t<__nv_bfloat16>(out, in, B, S, H, D, vec_bytes, stream);
    }
}

}  // namespace tt
