// layernorm.cu -- fused add-bias + residual + LayerNorm over [rows, hidden]
// (TurboTransformers' AddBiasLayerNorm; fusion of everything
// between two GEMMs, l.302; LayerNorm "calculates the mean and variance",
// l.316; variance per Eq. 1 l.406-409).
//
// One group of G threads owns one row:
//   LN-1  v_k = (x_k + bias_k) + residual_k in fp32, held in registers
//   LN-2  mean = K + sum(v - K) / N (K = the row's first element, a shift
//         that keeps the accumulator small), then var = sum((v - mean)^2) / N:
//         two register butterflies over the SAME registers (one extra shuffle
//         round, zero extra HBM bytes).  The paper's one-pass E(x^2) - E(x)^2 (Eq. 1 RHS)
//         saves that round but loses ~3 digits in fp32 when |mean| >> std
//         (DESIGN R9, offset test), so it is not used.
//   LN-3  y_k = (v_k - mean) * rsqrt(var + eps) * gamma_k + beta_k, RNE
//         narrowing, vector store.  `out` may alias x or residual exactly:
//         every element of a row is loaded before any element is stored.
#include <atomic>
#include <cstring>

#include "common.cuh"
#include "launch.h"

namespace tt {

// EARLY: gamma / beta are loaded into registers together with the row (for
// small, latency-bound problems: no dependent parameter load after the
// reductions); otherwise they are loaded (L1-cached) after them.
template <typename T, int VB, int G, int NV, int R, int NT, int MINB, bool EARLY = false>
__global__ void __launch_bounds__(NT, MINB)
    ln_rows_kernel(T* out, const T* x, const T* residual, const T* __restrict__ bias,
                   const T* __restrict__ gamma, const T* __restrict__ beta, int64_t rows,
                   int hidden, float eps) {
    PdlScope pdl_;  // griddepcontrol.wait first: no global access before it (PDL)
    constexpr int VE = VB / (int)sizeof(T);
    constexpr int GPB = NT / G;
    constexpr int NWG = G > 32 ? G / 32 : 1;
    __shared__ float red_a[G > 32 ? R * NWG : 1];
    __shared__ float red_b[G > 32 ? R * NWG : 1];

    const int q = threadIdx.x % G;
    const int gi = threadIdx.x / G;
    const int64_t base = (int64_t)blockIdx.x * GPB * R;
    const int nvec = hidden / VE;
    const float invN = 1.0f / (float)hidden;

    int64_t off[R];
    bool live[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int64_t row = base + (int64_t)r * GPB + gi;
        live[r] = row < rows;
        off[r] = (live[r] ? row : 0) * (int64_t)hidden;
    }
    Raw<VB> eg[EARLY ? NV : 1], eb[EARLY ? NV : 1];
    if constexpr (EARLY) {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int vi = q + k * G;
            if (vi < nvec) {
                ld_param<VB>(gamma + vi * VE, eg[k]);
                ld_param<VB>(beta + vi * VE, eb[k]);
            }
        }
    }
    // ---- LN-1: v = (x + bias) + residual
    float v[R][NV][VE];
#pragma unroll
    for (int r = 0; r < R; ++r) {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int vi = q + k * G;
            if (live[r] && vi < nvec) {
                Raw<VB> wx, wr;
                ld_stream<VB>(x + off[r] + vi * VE, wx);
                ld_stream<VB>(residual + off[r] + vi * VE, wr);
                float fr[VE];
                Elem<T>::template unpack<VB>(wx, v[r][k]);
                Elem<T>::template unpack<VB>(wr, fr);
                Raw<VB> wb;
                ld_param<VB>(bias + vi * VE, wb);
                float fb[VE];
                Elem<T>::template unpack<VB>(wb, fb);
#pragma unroll
                for (int e = 0; e < VE; ++e) v[r][k][e] = (v[r][k][e] + fb[e]) + fr[e];
            } else {
#pragma unroll
                for (int e = 0; e < VE; ++e) v[r][k][e] = 0.f;
            }
        }
    }

    // ---- LN-2: mean, then centred second moment.  The mean is accumulated
    // on data shifted by the row's first element K (exact in fp32 for nearby
    // values), so |mean| >> std loses no digits to the accumulator.
    float shift[R], mean[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        if constexpr (G <= 32) {
            shift[r] = __shfl_sync(0xffffffffu, v[r][0][0], (int)(threadIdx.x & 31) & ~(G - 1));
        } else {
            shift[r] = live[r] ? (Elem<T>::to_f(x[off[r]]) + Elem<T>::to_f(bias[0])) +
                                     Elem<T>::to_f(residual[off[r]])
                               : 0.f;
        }
        float a = 0.f;
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int vi = q + k * G;
            if (vi < nvec) {
#pragma unroll
                for (int e = 0; e < VE; ++e) a += v[r][k][e] - shift[r];
            }
        }
        mean[r] = a;
    }
    group_sum<G, R>(mean, red_a);
    float var[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        mean[r] = fmaf(mean[r], invN, shift[r]);
        float a = 0.f;
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int vi = q + k * G;
            if (vi < nvec) {
#pragma unroll
                for (int e = 0; e < VE; ++e) {
                    const float d = v[r][k][e] - mean[r];
                    a = fmaf(d, d, a);
                }
            }
        }
        var[r] = a;
    }
    group_sum<G, R>(var, red_b);

    // ---- LN-3: normalise, affine, store
#pragma unroll
    for (int r = 0; r < R; ++r) {
        if (!live[r]) continue;
        const float rstd = rsqrtf(var[r] * invN + eps);
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int vi = q + k * G;
            if (vi < nvec) {
                Raw<VB> wg, wb;
                if constexpr (EARLY) {
                    wg = eg[k];
                    wb = eb[k];
                } else {
                    ld_param<VB>(gamma + vi * VE, wg);
                    ld_param<VB>(beta + vi * VE, wb);
                }
                float fg[VE], fb[VE], y[VE];
                Elem<T>::template unpack<VB>(wg, fg);
                Elem<T>::template unpack<VB>(wb, fb);
#pragma unroll
                for (int e = 0; e < VE; ++e) y[e] = fmaf((v[r][k][e] - mean[r]) * rstd, fg[e], fb[e]);
                Raw<VB> wy;
                Elem<T>::template pack<VB>(y, wy);
                st_stream<VB>(out + off[r] + vi * VE, wy);
            }
        }
    }
}


// ----------------------------------------------------------------------------
// Warp / sub-warp tier (G <= 32, VB >= 16), the production path for hidden up
// to 32 * NV * VE.  Persistent CTAs; per CTA, bias / gamma / beta are widened
// to fp32 ONCE into shared memory in a lane-interleaved layout (quad j of
// chunk c at float4 index (p * VE/4 + j) * nvec + c, so a warp's LDS.128 are
// conflict-free), which removes their per-row global loads and conversions.
// The first row's x / residual loads are issued before that staging so the
// staging hides under their latency; with PF = true every row's loads are
// issued one row ahead (raw registers, loop unrolled by two).  Per row:
// v = (x + bias) + residual, shifted mean, centred variance (d = v - mean kept
// in the same registers), y = d * rstd * gamma + beta.
// ----------------------------------------------------------------------------
template <typename T, int VB, int G, int NV>
struct LnRow {
    static constexpr int VE = VB / (int)sizeof(T);
    static constexpr int QV = VE / 4;
    Raw<VB> x[NV], r[NV];

    __device__ __forceinline__ void load(const T* xp, const T* rp, size_t off, int q, int nvec) {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int vi = q + k * G;
            if (vi < nvec) {
                ld_stream<VB>(xp + off + vi * VE, x[k]);
                ld_stream<VB>(rp + off + vi * VE, r[k]);
            }
        }
    }

    __device__ __forceinline__ void finish(T* out, size_t off, int q, int nvec, float invN,
                                           float eps, const float4* pb, const float4* pg,
                                           const float4* pe) const {
        // ---- LN-1
        float v[NV][VE];
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int vi = q + k * G;
            if (vi < nvec) {
                float fr[VE];
                Elem<T>::template unpack<VB>(x[k], v[k]);
                Elem<T>::template unpack<VB>(r[k], fr);
#pragma unroll
                for (int j = 0; j < QV; ++j) {
                    const float4 b = pb[j * nvec + vi];
                    v[k][4 * j + 0] = (v[k][4 * j + 0] + b.x) + fr[4 * j + 0];
                    v[k][4 * j + 1] = (v[k][4 * j + 1] + b.y) + fr[4 * j + 1];
                    v[k][4 * j + 2] = (v[k][4 * j + 2] + b.z) + fr[4 * j + 2];
                    v[k][4 * j + 3] = (v[k][4 * j + 3] + b.w) + fr[4 * j + 3];
                }
            } else {
#pragma unroll
                for (int e = 0; e < VE; ++e) v[k][e] = 0.f;
            }
        }
        // ---- LN-2: shifted mean, centred variance
        float sh[1] = {__shfl_sync(0xffffffffu, v[0][0], (int)(threadIdx.x & 31) & ~(G - 1))};
        float mean[1] = {0.f};
#pragma unroll
        for (int k = 0; k < NV; ++k)
            if (q + k * G < nvec) {
#pragma unroll
                for (int e = 0; e < VE; ++e) mean[0] += v[k][e] - sh[0];
            }
        group_sum<G, 1>(mean, nullptr);
        const float mu = fmaf(mean[0], invN, sh[0]);
        float var[1] = {0.f};
#pragma unroll
        for (int k = 0; k < NV; ++k)
            if (q + k * G < nvec) {
#pragma unroll
                for (int e = 0; e < VE; ++e) {
                    v[k][e] -= mu;
                    var[0] = fmaf(v[k][e], v[k][e], var[0]);
                }
            }
        group_sum<G, 1>(var, nullptr);
        const float rstd = rsqrtf(var[0] * invN + eps);
        // ---- LN-3
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int vi = q + k * G;
            if (vi < nvec) {
                float y[VE];
#pragma unroll
                for (int j = 0; j < QV; ++j) {
                    const float4 g = pg[j * nvec + vi], b = pe[j * nvec + vi];
                    y[4 * j + 0] = fmaf(v[k][4 * j + 0] * rstd, g.x, b.x);
                    y[4 * j + 1] = fmaf(v[k][4 * j + 1] * rstd, g.y, b.y);
                    y[4 * j + 2] = fmaf(v[k][4 * j + 2] * rstd, g.z, b.z);
                    y[4 * j + 3] = fmaf(v[k][4 * j + 3] * rstd, g.w, b.w);
                }
                Raw<VB> wy;
                Elem<T>::template pack<VB>(y, wy);
                st_stream<VB>(out + off + vi * VE, wy);
            }
        }
    }
};

template <typename T, int VB, int G, int NV, int NT, int MINB, bool PF>
__global__ void __launch_bounds__(NT, MINB)
    ln_pf_kernel(T* out, const T* x, const T* residual, const T* __restrict__ bias,
                   const T* __restrict__ gamma, const T* __restrict__ beta, uint32_t rows,
                   int hidden, float eps) {
    PdlScope pdl_;  // griddepcontrol.wait first: no global access before it (PDL)
    using Row = LnRow<T, VB, G, NV>;
    constexpr int VE = Row::VE;
    constexpr int QV = Row::QV;
    constexpr int GPB = NT / G;
    static_assert(G <= 32 && VE % 4 == 0, "warp tier with >= 4-element vectors");
    extern __shared__ __align__(16) float4 prm[];  // [3][QV][nvec] float4
    const int nvec = hidden / VE;
    const float invN = 1.0f / (float)hidden;
    const int q = threadIdx.x % G;
    const uint32_t stride = gridDim.x * GPB;
    uint32_t row = blockIdx.x * GPB + threadIdx.x / G;

    Row a, b;
    if constexpr (PF) {
        if (row < rows) a.load(x, residual, (size_t)row * hidden, q, nvec);  // in flight
    } else if (row < rows) {
        // warm L2 with the first row while the parameters are staged (no registers held)
        const size_t off = (size_t)row * hidden;
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int vi = q + k * G;
            if (vi < nvec) {
                asm volatile("prefetch.global.L2 [%0];" ::"l"(x + off + vi * VE));
                asm volatile("prefetch.global.L2 [%0];" ::"l"(residual + off + vi * VE));
            }
        }
    }

    // stage the three parameter vectors as fp32 (once per persistent CTA)
    for (int i = threadIdx.x; i < 3 * hidden; i += NT) {
        const int pi = i / hidden, col = i - pi * hidden;
        const T* src = pi == 0 ? bias : pi == 1 ? gamma : beta;
        const int c = col / VE, e = col - c * VE;
        reinterpret_cast<float*>(prm)[(((pi * QV + (e >> 2)) * nvec + c) << 2) + (e & 3)] =
            Elem<T>::to_f(src[col]);
    }
    __syncthreads();
    const float4* pb = prm;
    const float4* pg = prm + QV * nvec;
    const float4* pe = prm + 2 * QV * nvec;

    if constexpr (PF) {
        while (row < rows) {
            const uint32_t r1 = row + stride;
            if (r1 < rows) b.load(x, residual, (size_t)r1 * hidden, q, nvec);
            a.finish(out, (size_t)row * hidden, q, nvec, invN, eps, pb, pg, pe);
            if (r1 >= rows) break;
            const uint32_t r2 = r1 + stride;
            if (r2 < rows) a.load(x, residual, (size_t)r2 * hidden, q, nvec);
            b.finish(out, (size_t)r1 * hidden, q, nvec, invN, eps, pb, pg, pe);
            row = r2;
        }
    } else {
        for (; row < rows; row += stride) {
            a.load(x, residual, (size_t)row * hidden, q, nvec);
            a.finish(out, (size_t)row * hidden, q, nvec, invN, eps, pb, pg, pe);
        }
    }
}


// Non-prefetching warp tier (PF = 0): loads and unpacks interleaved per vector.
template <typename T, int VB, int G, int NV, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB)
    ln_warp_kernel(T* out, const T* x, const T* residual, const T* __restrict__ bias,
                   const T* __restrict__ gamma, const T* __restrict__ beta, uint32_t rows,
                   int hidden, float eps) {
    PdlScope pdl_;  // griddepcontrol.wait first: no global access before it (PDL)
    constexpr int VE = VB / (int)sizeof(T);
    constexpr int QV = VE / 4;  // float4 quads per vector
    constexpr int GPB = NT / G;
    static_assert(G <= 32 && VE % 4 == 0, "warp tier with >= 4-element vectors");
    extern __shared__ __align__(16) float4 prm[];  // [3][QV][nvec] float4
    const int nvec = hidden / VE;
    const float invN = 1.0f / (float)hidden;

    // stage the three parameter vectors as fp32 (once per persistent CTA)
    for (int i = threadIdx.x; i < 3 * hidden; i += NT) {
        const int pi = i / hidden, col = i - pi * hidden;
        const T* src = pi == 0 ? bias : pi == 1 ? gamma : beta;
        const int c = col / VE, e = col - c * VE;
        reinterpret_cast<float*>(prm)[(((pi * QV + (e >> 2)) * nvec + c) << 2) + (e & 3)] =
            Elem<T>::to_f(src[col]);
    }
    __syncthreads();
    const float4* pb = prm;
    const float4* pg = prm + QV * nvec;
    const float4* pe = prm + 2 * QV * nvec;

    const int q = threadIdx.x % G;
    const uint32_t stride = gridDim.x * GPB;
    for (uint32_t row = blockIdx.x * GPB + threadIdx.x / G; row < rows; row += stride) {
        const size_t off = (size_t)row * (size_t)hidden;
        // ---- LN-1
        float v[NV][VE];
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int vi = q + k * G;
            if (vi < nvec) {
                Raw<VB> wx, wr;
                ld_stream<VB>(x + off + vi * VE, wx);
                ld_stream<VB>(residual + off + vi * VE, wr);
                float fr[VE];
                Elem<T>::template unpack<VB>(wx, v[k]);
                Elem<T>::template unpack<VB>(wr, fr);
#pragma unroll
                for (int j = 0; j < QV; ++j) {
                    const float4 b = pb[j * nvec + vi];
                    v[k][4 * j + 0] = (v[k][4 * j + 0] + b.x) + fr[4 * j + 0];
                    v[k][4 * j + 1] = (v[k][4 * j + 1] + b.y) + fr[4 * j + 1];
                    v[k][4 * j + 2] = (v[k][4 * j + 2] + b.z) + fr[4 * j + 2];
                    v[k][4 * j + 3] = (v[k][4 * j + 3] + b.w) + fr[4 * j + 3];
                }
            } else {
#pragma unroll
                for (int e = 0; e < VE; ++e) v[k][e] = 0.f;
            }
        }
        // ---- LN-2: shifted mean, centred variance
        float sh[1] = {__shfl_sync(0xffffffffu, v[0][0], (int)(threadIdx.x & 31) & ~(G - 1))};
        float mean[1] = {0.f};
#pragma unroll
        for (int k = 0; k < NV; ++k)
            if (q + k * G < nvec) {
#pragma unroll
                for (int e = 0; e < VE; ++e) mean[0] += v[k][e] - sh[0];
            }
        group_sum<G, 1>(mean, nullptr);
        const float mu = fmaf(mean[0], invN, sh[0]);
        float var[1] = {0.f};
#pragma unroll
        for (int k = 0; k < NV; ++k)
            if (q + k * G < nvec) {
#pragma unroll
                for (int e = 0; e < VE; ++e) {
                    v[k][e] -= mu;
                    var[0] = fmaf(v[k][e], v[k][e], var[0]);
                }
            }
        group_sum<G, 1>(var, nullptr);
        const float rstd = rsqrtf(var[0] * invN + eps);
        // ---- LN-3
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int vi = q + k * G;
            if (vi < nvec) {
                float y[VE];
#pragma unroll
                for (int j = 0; j < QV; ++j) {
                    const float4 g = pg[j * nvec + vi], b = pe[j * nvec + vi];
                    y[4 * j + 0] = fmaf(v[k][4 * j + 0] * rstd, g.x, b.x);
                    y[4 * j + 1] = fmaf(v[k][4 * j + 1] * rstd, g.y, b.y);
                    y[4 * j + 2] = fmaf(v[k][4 * j + 2] * rstd, g.z, b.z);
                    y[4 * j + 3] = fmaf(v[k][4 * j + 3] * rstd, g.w, b.w);
                }
                Raw<VB> wy;
                Elem<T>::template pack<VB>(y, wy);
                st_stream<VB>(out + off + vi * VE, wy);
            }
        }
    }
}

// ----------------------------------------------------------------------------
// TMA-staged variant (warp per row, 16-byte chunks): persistent CTAs; each
// warp streams its rows' x and residual through a private ring of D shared-
// memory slots filled by 1-D bulk copies (cp.async.bulk, SASS UBLKCP) issued
// D rows ahead, so the bytes in flight per SM are set by the ring, not by
// the register file.  bias / gamma / beta are staged once per CTA as fp32 in
// shared memory (lane-interleaved float4 layout, conflict-free LDS.128).
// Requires hidden * sizeof(T) % 16 == 0 and 16-byte aligned operands.
// Dynamic smem: [params 3*hidden fp32][NW*D mbarriers][NW*D slots].
// ----------------------------------------------------------------------------
template <typename T, int NV, int NW>
__global__ void __launch_bounds__(NW * 32)
    ln_tma_kernel(T* out, const T* x, const T* residual, const T* __restrict__ bias,
                  const T* __restrict__ gamma, const T* __restrict__ beta, int64_t rows, int hidden,
                  float eps, int D, int slot_bytes) {
    PdlScope pdl_;  // griddepcontrol.wait first: no global access before it (PDL)
    constexpr int VE = 16 / (int)sizeof(T);
    constexpr int QV = VE / 4;
    extern __shared__ __align__(128) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nchunks = hidden / VE;
    const size_t prm_bytes = ((size_t)3 * hidden * 4 + 127) & ~(size_t)127;
    float4* prm = reinterpret_cast<float4*>(smem);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + prm_bytes) + warp * D;
    unsigned char* ring = smem + prm_bytes + ((NW * D * 8 + 127) & ~127) +
                          (size_t)warp * D * slot_bytes;
    const int64_t TW = (int64_t)gridDim.x * NW;
    const int64_t gw = (int64_t)blockIdx.x * NW + warp;
    const uint32_t rb = (uint32_t)hidden * (uint32_t)sizeof(T);  // row bytes, multiple of 16
    const float invN = 1.0f / (float)hidden;

    auto issue = [&](int64_t row, int sl) {
        if (row >= rows) return;
        unsigned char* dst = ring + (size_t)sl * slot_bytes;
        mbar_arrive_expect_tx(&bars[sl], 2 * rb);
        tma_load_1d(dst, x + row * (int64_t)hidden, rb, &bars[sl]);
        tma_load_1d(dst + rb, residual + row * (int64_t)hidden, rb, &bars[sl]);
    };
    if (lane == 0) {
        for (int s = 0; s < D; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
        fence_proxy_async_smem();
        for (int s = 0; s < D; ++s) issue(gw + s * TW, s);
    }
    for (int i = threadIdx.x; i < 3 * hidden; i += NW * 32) {
        const int pi = i / hidden, col = i - pi * hidden;
        const T* src = pi == 0 ? bias : pi == 1 ? gamma : beta;
        const int c = col / VE, e = col - c * VE;
        reinterpret_cast<float*>(prm)[(((pi * QV + (e >> 2)) * nchunks + c) << 2) + (e & 3)] =
            Elem<T>::to_f(src[col]);
    }
    __syncthreads();
    const float4* pb = prm;
    const float4* pg = prm + QV * nchunks;
    const float4* pe = prm + 2 * QV * nchunks;

    int sl = 0;
    uint32_t ph = 0;
    for (int64_t row = gw; row < rows; row += TW) {
        const unsigned char* slot = ring + (size_t)sl * slot_bytes;
        mbar_wait(&bars[sl], ph);
        // ---- LN-1
        float v[NV][VE];
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int ci = lane + 32 * k;
            if (ci < nchunks) {
                Raw<16> wx, wr;
                lds128(slot + 16 * ci, wx.w);
                lds128(slot + rb + 16 * ci, wr.w);
                float fr[VE];
                Elem<T>::template unpack<16>(wx, v[k]);
                Elem<T>::template unpack<16>(wr, fr);
#pragma unroll
                for (int j = 0; j < QV; ++j) {
                    const float4 b = pb[j * nchunks + ci];
                    v[k][4 * j + 0] = (v[k][4 * j + 0] + b.x) + fr[4 * j + 0];
                    v[k][4 * j + 1] = (v[k][4 * j + 1] + b.y) + fr[4 * j + 1];
                    v[k][4 * j + 2] = (v[k][4 * j + 2] + b.z) + fr[4 * j + 2];
                    v[k][4 * j + 3] = (v[k][4 * j + 3] + b.w) + fr[4 * j + 3];
                }
            } else {
#pragma unroll
                for (int e = 0; e < VE; ++e) v[k][e] = 0.f;
            }
        }
        float sh[1] = {__shfl_sync(0xffffffffu, v[0][0], 0)};
        // slot consumed (values are in registers): refill it D rows ahead
        __syncwarp();
        if (lane == 0) {
            fence_proxy_async_smem();
            issue(row + (int64_t)D * TW, sl);
        }
        if (++sl == D) {
            sl = 0;
            ph ^= 1;
        }
        // ---- LN-2
        float mean[1] = {0.f};
#pragma unroll
        for (int k = 0; k < NV; ++k)
            if (lane + 32 * k < nchunks) {
#pragma unroll
                for (int e = 0; e < VE; ++e) mean[0] += v[k][e] - sh[0];
            }
        group_sum<32, 1>(mean, nullptr);
        const float mu = fmaf(mean[0], invN, sh[0]);
        float var[1] = {0.f};
#pragma unroll
        for (int k = 0; k < NV; ++k)
            if (lane + 32 * k < nchunks) {
#pragma unroll
                for (int e = 0; e < VE; ++e) {
                    v[k][e] -= mu;
                    var[0] = fmaf(v[k][e], v[k][e], var[0]);
                }
            }
        group_sum<32, 1>(var, nullptr);
        const float rstd = rsqrtf(var[0] * invN + eps);
        // ---- LN-3
        T* o = out + row * (int64_t)hidden;
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int ci = lane + 32 * k;
            if (ci < nchunks) {
                float y[VE];
#pragma unroll
                for (int j = 0; j < QV; ++j) {
                    const float4 g = pg[j * nchunks + ci], b = pe[j * nchunks + ci];
                    y[4 * j + 0] = fmaf(v[k][4 * j + 0] * rstd, g.x, b.x);
                    y[4 * j + 1] = fmaf(v[k][4 * j + 1] * rstd, g.y, b.y);
                    y[4 * j + 2] = fmaf(v[k][4 * j + 2] * rstd, g.z, b.z);
                    y[4 * j + 3] = fmaf(v[k][4 * j + 3] * rstd, g.w, b.w);
                }
                Raw<16> wy;
                Elem<T>::template pack<16>(y, wy);
                st_stream<16>(o + ci * VE, wy);
            }
        }
    }
}

namespace {

int sm_count() {
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

template <typename T, int NV, int NW, int KB>
cudaError_t launch_ln_tma(void* out, const void* x, const void* res, const void* bias,
                          const void* gamma, const void* beta, int64_t rows, int hidden, float eps,
                          cudaStream_t st) {
    auto kern = ln_tma_kernel<T, NV, NW>;
    const int rb = hidden * (int)sizeof(T);
    const int slot_bytes = (2 * rb + 127) & ~127;
    // ring depth: about KB kilobytes of rows in flight per warp, 2..8 slots
    const int D = max(2, min(8, (KB * 1024) / slot_bytes));
    const size_t prm_bytes = ((size_t)3 * hidden * 4 + 127) & ~(size_t)127;
    const size_t smem =
        prm_bytes + (size_t)((NW * D * 8 + 127) & ~127) + (size_t)NW * D * slot_bytes;
    if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
    cudaError_t e = smem_optin(reinterpret_cast<const void*>(kern), smem);
    if (e != cudaSuccess) return e;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NW * 32, smem);
    if (e != cudaSuccess) return e;
    occ = max(occ, 1);
    const int64_t need = (rows + NW - 1) / NW;
    const int64_t cap = (int64_t)sm_count() * occ;
    const int64_t grid = need < cap ? need : cap;
    {
        const cudaError_t le_ = launch_k(kern, (unsigned)grid, NW * 32, smem, st,
        static_cast<T*>(out), static_cast<const T*>(x), static_cast<const T*>(res),
        static_cast<const T*>(bias), static_cast<const T*>(gamma), static_cast<const T*>(beta),
        rows, hidden, eps, D, slot_bytes);
        if (le_ != cudaSuccess) return le_;
    }
    return cudaGetLastError();
}

}  // namespace

namespace {

template <typename T, int VB, int G, int NV, int R, int NT, int MINB, bool EARLY = false>
cudaError_t launch_ln(void* out, const void* x, const void* res, const void* bias,
                      const void* gamma, const void* beta, int64_t rows, int hidden, float eps,
                      cudaStream_t st) {
    constexpr int GPB = NT / G;
    const int64_t rows_per_cta = (int64_t)GPB * R;
    const int64_t grid = (rows + rows_per_cta - 1) / rows_per_cta;
    if (grid > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
    {
        const cudaError_t le_ = launch_k(ln_rows_kernel<T, VB, G, NV, R, NT, MINB, EARLY>, (unsigned)grid, NT, 0, st,
        static_cast<T*>(out), static_cast<const T*>(x), static_cast<const T*>(res),
        static_cast<const T*>(bias), static_cast<const T*>(gamma), static_cast<const T*>(beta),
        rows, hidden, eps);
        if (le_ != cudaSuccess) return le_;
    }
    return cudaGetLastError();
}


template <typename T, int VB, int G, int NV, int NT, int MINB, bool PF>
cudaError_t launch_ln_warp(void* out, const void* x, const void* res, const void* bias,
                           const void* gamma, const void* beta, int64_t rows, int hidden,
                           float eps, cudaStream_t st) {
    constexpr int GPB = NT / G;
    if (rows >= (int64_t)0xffffffffLL)
        return launch_ln<T, VB, G, NV, 1, NT, MINB>(out, x, res, bias, gamma, beta, rows, hidden,
                                                    eps, st);
    auto kern = PF ? ln_pf_kernel<T, VB, G, NV, NT, MINB, true>
                   : ln_warp_kernel<T, VB, G, NV, NT, MINB>;
    const size_t smem = (size_t)3 * hidden * sizeof(float);
    cudaError_t e = smem_optin(reinterpret_cast<const void*>(kern), smem);
    if (e != cudaSuccess) return e;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, smem);
    if (e != cudaSuccess) return e;
    occ = occ > 0 ? occ : 1;
    const int64_t need = (rows + GPB - 1) / GPB;
    const int64_t cap = (int64_t)sm_count() * occ;
    const int64_t grid = need < cap ? need : cap;
    {
        const cudaError_t le_ = launch_k(kern, (unsigned)grid, NT, smem, st,
        static_cast<T*>(out), static_cast<const T*>(x), static_cast<const T*>(res),
        static_cast<const T*>(bias), static_cast<const T*>(gamma), static_cast<const T*>(beta),
        (uint32_t)rows, hidden, eps);
        if (le_ != cudaSuccess) return le_;
    }
    return cudaGetLastError();
}

using LnFn = cudaError_t (*)(void*, const void*, const void*, const void*, const void*,
                             const void*, int64_t, int, float, cudaStream_t);

struct LnTier {
    int vb;          // vector bytes
    int ve;          // elements per vector
    int capacity;    // G * NV * VE: largest hidden
    bool automatic;  // eligible for automatic selection (else: tuning candidate only)
    LnFn fn;
    const char* name;
};

#define TT_LN_TIER(AUTO, T, TN, VB, G, NV, R, NT, MINB)                                    \
    LnTier {                                                                               \
        VB, (VB) / (int)sizeof(T), (G) * (NV) * ((VB) / (int)sizeof(T)), AUTO,             \
            &launch_ln<T, VB, G, NV, R, NT, MINB>,                                         \
            "ln_rows<" TN ",V" #VB ",G" #G ",NV" #NV ",R" #R ",T" #NT ",M" #MINB ">"      \
    }
#define TT_LN_EARLY(AUTO, T, TN, VB, G, NV, NT)                                            \
    LnTier {                                                                               \
        VB, (VB) / (int)sizeof(T), (G) * (NV) * ((VB) / (int)sizeof(T)), AUTO,             \
            &launch_ln<T, VB, G, NV, 1, NT, 1, true>,                                      \
            "ln_rows<" TN ",V" #VB ",G" #G ",NV" #NV ",R1,T" #NT ",M1,E>"                 \
    }

#define TT_LN_WARP_P(AUTO, T, TN, VB, G, NV, NT, MINB, PF)                                 \
    LnTier {                                                                               \
        VB, (VB) / (int)sizeof(T), (G) * (NV) * ((VB) / (int)sizeof(T)), AUTO,             \
            &launch_ln_warp<T, VB, G, NV, NT, MINB, PF>,                                   \
            "ln_warp<" TN ",V" #VB ",G" #G ",NV" #NV ",T" #NT ",M" #MINB ",PF" #PF ">"    \
    }
#define TT_LN_WARP(AUTO, T, TN, VB, G, NV, NT, MINB) TT_LN_WARP_P(AUTO, T, TN, VB, G, NV, NT, MINB, 0)

#define TT_LN_TMA_K(AUTO, T, TN, NV, NW, KB)                                               \
    LnTier {                                                                               \
        16, 16 / (int)sizeof(T), 32 * (NV) * (16 / (int)sizeof(T)), AUTO,                 \
            &launch_ln_tma<T, NV, NW, KB>,                                                 \
            "ln_tma<" TN ",V16,G32,NV" #NV ",W" #NW ",K" #KB ">"                          \
    }
#define TT_LN_TMA(AUTO, T, TN, NV, NW) TT_LN_TMA_K(AUTO, T, TN, NV, NW, 8)

// Main tiers use 16- or 32-byte vectors; the scalar tiers (VB = sizeof(T))
// only serve hidden sizes whose row pitch is not a multiple of 16 bytes.
// NVC32 / NVC16 = CTA-tier vectors per thread (NV * VE = 32 registers of row
// data).  Non-automatic entries are tuning candidates (tt_tune.h).
#define TT_LN_LIST(T, TN, SB, NVC32, NVC16, MA, MB, MC)                                       \
    TT_LN_WARP(true, T, TN, 16, 4, 1, 256, 4), TT_LN_WARP(true, T, TN, 16, 8, 1, 256, 4),       \
    TT_LN_WARP(true, T, TN, 16, 16, 1, 256, 4), TT_LN_WARP(true, T, TN, 16, 32, 1, 256, 4),     \
    TT_LN_WARP(true, T, TN, 16, 32, 2, 256, MA), TT_LN_WARP(true, T, TN, 16, 32, 3, 256, MB),   \
    TT_LN_WARP(true, T, TN, 16, 32, 4, 256, MB), TT_LN_WARP(true, T, TN, 16, 32, 6, 256, MC),   \
    TT_LN_WARP(true, T, TN, 16, 32, 8, 256, MC), TT_LN_WARP(true, T, TN, 32, 4, 1, 256, 4),     \
    TT_LN_WARP(true, T, TN, 32, 8, 1, 256, 4), TT_LN_WARP(true, T, TN, 32, 16, 1, 256, 4),      \
    TT_LN_WARP(true, T, TN, 32, 32, 1, 256, MA), TT_LN_WARP(true, T, TN, 32, 32, 2, 256, MB),   \
    TT_LN_WARP(true, T, TN, 32, 32, 3, 256, MC), TT_LN_WARP(true, T, TN, 32, 32, 4, 256, MC),   \
    TT_LN_TIER(true, T, TN, 16, 128, NVC16, 1, 128, 1), TT_LN_TIER(true, T, TN, 16, 256, NVC16, 1, 256, 1), \
    TT_LN_TIER(true, T, TN, 16, 512, NVC16, 1, 512, 1), TT_LN_TIER(true, T, TN, 16, 1024, NVC16, 1, 1024, 1), \
    TT_LN_TIER(true, T, TN, 32, 128, NVC32, 1, 128, 1), TT_LN_TIER(true, T, TN, 32, 256, NVC32, 1, 256, 1), \
    TT_LN_TIER(true, T, TN, 32, 512, NVC32, 1, 512, 1), TT_LN_TIER(true, T, TN, 32, 1024, NVC32, 1, 1024, 1), \
    TT_LN_TIER(true, T, TN, SB, 32, 1, 1, 256, 1), TT_LN_TIER(true, T, TN, SB, 32, 4, 1, 256, 1), \
    TT_LN_TIER(true, T, TN, SB, 32, 16, 1, 256, 1), TT_LN_TIER(true, T, TN, SB, 256, 16, 1, 256, 1), \
    TT_LN_TIER(true, T, TN, SB, 1024, 32, 1, 1024, 1),                                      \
    TT_LN_TIER(false, T, TN, 32, 32, 2, 1, 256, 1), TT_LN_TIER(false, T, TN, 32, 32, 2, 1, 128, 6), \
    TT_LN_TIER(false, T, TN, 16, 32, 3, 1, 256, 1), TT_LN_TIER(false, T, TN, 32, 32, 3, 1, 256, 1), \
    TT_LN_TIER(false, T, TN, 32, 32, 4, 1, 256, 1), TT_LN_TIER(false, T, TN, 32, 32, 4, 1, 128, 1), \
    TT_LN_TMA(false, T, TN, 3, 8), TT_LN_TMA(false, T, TN, 4, 8), TT_LN_TMA(false, T, TN, 4, 4),       \
    TT_LN_TMA(false, T, TN, 6, 4), TT_LN_TMA(false, T, TN, 8, 4), TT_LN_TMA(false, T, TN, 2, 8),       \
    TT_LN_WARP(false, T, TN, 32, 32, 2, 256, 3), TT_LN_WARP(false, T, TN, 32, 32, 2, 256, 5),   \
    TT_LN_WARP(false, T, TN, 32, 32, 2, 256, 6), TT_LN_WARP(false, T, TN, 32, 32, 2, 128, 8),   \
    TT_LN_WARP(false, T, TN, 32, 32, 2, 128, 12), TT_LN_WARP(false, T, TN, 32, 32, 3, 128, 6),  \
    TT_LN_WARP(false, T, TN, 32, 32, 3, 256, 5), TT_LN_WARP(false, T, TN, 16, 32, 3, 256, 3),   \
    TT_LN_WARP(false, T, TN, 16, 32, 3, 256, 5), TT_LN_WARP(false, T, TN, 16, 32, 3, 128, 8),   \
    TT_LN_WARP(false, T, TN, 16, 32, 4, 256, 3), TT_LN_WARP(false, T, TN, 16, 32, 4, 256, 5),   \
    TT_LN_WARP(false, T, TN, 32, 32, 4, 128, 6),                                              \
    TT_LN_TMA_K(false, T, TN, 4, 4, 12), TT_LN_TMA_K(false, T, TN, 4, 4, 16),                   \
    TT_LN_TMA_K(false, T, TN, 4, 8, 12), TT_LN_TMA_K(false, T, TN, 3, 4, 12),                   \
    TT_LN_TMA_K(false, T, TN, 3, 8, 12), TT_LN_TMA_K(false, T, TN, 8, 4, 12),                   \
    TT_LN_TMA_K(false, T, TN, 4, 2, 16), TT_LN_TMA_K(false, T, TN, 3, 2, 16),                   \
    TT_LN_WARP_P(false, T, TN, 32, 32, 2, 256, 2, 1), TT_LN_WARP_P(false, T, TN, 32, 32, 2, 256, 3, 1), \
    TT_LN_WARP_P(false, T, TN, 32, 32, 2, 128, 6, 1), TT_LN_WARP_P(false, T, TN, 16, 32, 3, 256, 3, 1), \
    TT_LN_WARP_P(false, T, TN, 16, 32, 3, 256, 2, 1), TT_LN_WARP_P(false, T, TN, 32, 32, 3, 256, 2, 1), \
    TT_LN_WARP_P(false, T, TN, 32, 32, 3, 128, 4, 1), TT_LN_WARP_P(false, T, TN, 16, 32, 4, 256, 2, 1), \
    TT_LN_WARP_P(false, T, TN, 32, 32, 1, 256, 4, 1), TT_LN_WARP_P(false, T, TN, 32, 32, 4, 256, 2, 1), \
    TT_LN_EARLY(false, T, TN, 16, 32, 3, 256), TT_LN_EARLY(false, T, TN, 32, 32, 2, 256),        \
    TT_LN_EARLY(false, T, TN, 32, 32, 3, 256), TT_LN_EARLY(false, T, TN, 32, 32, 4, 256),        \
    TT_LN_EARLY(false, T, TN, 16, 32, 3, 128), TT_LN_EARLY(false, T, TN, 32, 32, 2, 128),        \
    TT_LN_WARP(false, T, TN, 16, 16, 6, 256, 3), TT_LN_WARP(false, T, TN, 16, 8, 12, 256, 2),   \
    TT_LN_WARP(false, T, TN, 32, 16, 3, 256, 3), TT_LN_WARP(false, T, TN, 32, 16, 6, 256, 3),   \
    TT_LN_WARP(false, T, TN, 32, 8, 6, 256, 2), TT_LN_WARP(false, T, TN, 32, 8, 12, 256, 2),    \
    TT_LN_WARP(false, T, TN, 16, 16, 6, 256, 4), TT_LN_WARP(false, T, TN, 32, 16, 3, 256, 4)

// MA / MB / MC: min CTAs/SM (register cap) for warp tiers holding about
// 16 / 24-32 / 48-64 fp32 row values per lane.
const LnTier kLn_f32[] = {TT_LN_LIST(float, "f32", 4, 4, 8, 6, 4, 3)};
const LnTier kLn_f16[] = {TT_LN_LIST(__half, "f16", 2, 2, 4, 4, 4, 2)};
const LnTier kLn_bf16[] = {TT_LN_LIST(__nv_bfloat16, "bf16", 2, 2, 4, 4, 4, 2)};
constexpr int kLnN = (int)(sizeof(kLn_f32) / sizeof(kLn_f32[0]));

std::atomic<int> g_force[3] = {{-1}, {-1}, {-1}};

const LnTier* table(int dtype) {
    switch (dtype) {
        case 0: return kLn_f32;
        case 1: return kLn_f16;
        case 2: return kLn_bf16;
        default: return nullptr;
    }
}

bool fits(const LnTier& t, int64_t hidden, int vec_bytes) {
    return t.vb <= vec_bytes && hidden % t.ve == 0 && hidden <= t.capacity;
}

// Tuned preferences (tools/tune.py on B200, profiles/*_tune.txt): for rows up
// to max_hidden, use the named tier when it can serve the call.  Anything not
// covered falls through to the generic rule below.
struct Pref {
    int dtype;
    int min_hidden, max_hidden;  // applies to min_hidden < hidden <= max_hidden
    const char* name;
};
// up to kSmallRows rows the problem is latency-bound: no per-CTA parameter
// staging, one row per group, gamma / beta loaded together with the row
// (ln_rows EARLY tiers), so no dependent load follows the reductions
// (EARLY costs registers, so only for the tiniest problems)
constexpr int64_t kTinyRows = 2048, kSmallRows = 8192;
// (f16 / f32 at hidden 768 re-tuned on C2's S = 128 .. 400 LayerNorm shapes,
// profiles/r01_tune_lnmid/: 128-thread CTAs, +1..7 % over the 256-thread tiers)
const Pref kLnPrefSmall[] = {
    {0, 512, 768, "ln_rows<f32,V32,G32,NV4,R1,T128,M1>"},
    {0, 768, 1024, "ln_rows<f32,V32,G32,NV4,R1,T256,M1>"},
    {1, 512, 768, "ln_rows<f16,V16,G32,NV3,R1,T128,M1,E>"},
    {1, 768, 1024, "ln_rows<f16,V32,G32,NV2,R1,T256,M1>"},
    {2, 512, 768, "ln_rows<bf16,V16,G32,NV3,R1,T256,M1>"},
    {2, 768, 1024, "ln_rows<bf16,V32,G32,NV2,R1,T256,M1>"},
};
// Very few rows: one CTA (four warps) per row, so the rows spread over as many
// SMs as there are rows and every thread issues only a few loads (re-tuned on
// C1 / C2 S = 10 .. 40, profiles/r01_tune_lntiny/: fp16 40 rows 2.67 -> 1.84 us,
// 200 rows 3.35 -> 1.98 us; fp32 40 rows 2.43 -> 1.90 us, 400 rows 3.90 -> 2.96 us).
constexpr int64_t kMicroRows = 256, kMiniRows = 1024;
const Pref kLnPrefMicro[] = {
    {0, 512, 768, "ln_rows<f32,V32,G128,NV4,R1,T128,M1>"},
    {1, 512, 768, "ln_rows<f16,V32,G128,NV2,R1,T128,M1>"},
};
const Pref kLnPrefMini[] = {
    {0, 512, 768, "ln_rows<f32,V32,G128,NV4,R1,T128,M1>"},
    {1, 512, 768, "ln_rows<f16,V16,G128,NV4,R1,T128,M1>"},
};
const Pref kLnPrefTiny[] = {
    {0, 512, 768, "ln_rows<f32,V32,G32,NV3,R1,T256,M1,E>"},
    {0, 768, 1024, "ln_rows<f32,V32,G32,NV4,R1,T256,M1,E>"},
    {1, 512, 768, "ln_rows<f16,V32,G32,NV2,R1,T128,M1,E>"},  // 1280 / 2000 rows: -8 / -4 %
    {1, 768, 1024, "ln_rows<f16,V32,G32,NV2,R1,T256,M1,E>"},
    {2, 512, 768, "ln_rows<bf16,V16,G32,NV3,R1,T256,M1,E>"},
    {2, 768, 1024, "ln_rows<bf16,V32,G32,NV2,R1,T256,M1,E>"},
};
const Pref kLnPref[] = {
    {0, 512, 768, "ln_rows<f32,V32,G32,NV3,R1,T256,M1>"},
    {0, 768, 1024, "ln_rows<f32,V32,G32,NV4,R1,T256,M1>"},
    {1, 512, 768, "ln_warp<f16,V16,G32,NV4,T256,M2,PF1>"},
    {1, 768, 1024, "ln_warp<f16,V16,G32,NV4,T256,M2,PF1>"},
    {2, 512, 768, "ln_warp<bf16,V16,G32,NV4,T256,M2,PF1>"},
    {2, 768, 1024, "ln_warp<bf16,V16,G32,NV4,T256,M2,PF1>"},
};

const LnTier* by_name(const LnTier* tab, const char* name) {
    for (int i = 0; i < kLnN; ++i)
        if (!strcmp(tab[i].name, name)) return &tab[i];
    return nullptr;
}

template <size_t N>
const LnTier* from_prefs(const Pref (&prefs)[N], std::atomic<int> (&idx)[N], int dtype,
                         int64_t hidden, int vec_bytes) {
    // the preference whose (min_hidden, max_hidden] holds this row
    for (size_t i = 0; i < N; ++i) {
        const Pref& pr = prefs[i];
        if (pr.dtype != dtype || hidden <= pr.min_hidden || hidden > pr.max_hidden) continue;
        int k = idx[i].load(std::memory_order_relaxed);
        if (k == 0) {
            const LnTier* found = by_name(table(dtype), pr.name);
            k = found ? (int)(found - table(dtype)) + 1 : -1;
            idx[i].store(k, std::memory_order_relaxed);
        }
        const LnTier* t = k > 0 ? table(dtype) + (k - 1) : nullptr;
        if (t && fits(*t, hidden, vec_bytes)) return t;
    }
    return nullptr;
}

const LnTier* pick_dtype(int dtype, int64_t hidden, int vec_bytes, int64_t rows) {
    const LnTier* tab = table(dtype);
    if (!tab) return nullptr;
    const int f = g_force[dtype].load(std::memory_order_relaxed);
    if (f >= 0 && f < kLnN && fits(tab[f], hidden, vec_bytes)) return &tab[f];
    // name -> tier index caches, one per preference table (benign race: every
    // thread stores the same index)
    static std::atomic<int> idx_micro[sizeof(kLnPrefMicro) / sizeof(Pref)];
    static std::atomic<int> idx_mini[sizeof(kLnPrefMini) / sizeof(Pref)];
    static std::atomic<int> idx_tiny[sizeof(kLnPrefTiny) / sizeof(Pref)];
    static std::atomic<int> idx_small[sizeof(kLnPrefSmall) / sizeof(Pref)];
    static std::atomic<int> idx_large[sizeof(kLnPref) / sizeof(Pref)];
    const LnTier* pbest =
        rows <= kMicroRows  ? from_prefs(kLnPrefMicro, idx_micro, dtype, hidden, vec_bytes)
        : rows <= kMiniRows ? from_prefs(kLnPrefMini, idx_mini, dtype, hidden, vec_bytes)
                            : nullptr;
    if (!pbest)
        pbest = rows <= kTinyRows    ? from_prefs(kLnPrefTiny, idx_tiny, dtype, hidden, vec_bytes)
                : rows <= kSmallRows ? from_prefs(kLnPrefSmall, idx_small, dtype, hidden, vec_bytes)
                                     : from_prefs(kLnPref, idx_large, dtype, hidden, vec_bytes);
    if (pbest) return pbest;
    const LnTier* best = nullptr;
    for (int i = 0; i < kLnN; ++i) {
        const LnTier& t = tab[i];
        if (!t.automatic || !fits(t, hidden, vec_bytes)) continue;
        // least padding first (fewest idle lanes), then the widest vector
        if (!best || t.capacity < best->capacity ||
            (t.capacity == best->capacity && t.vb > best->vb))
            best = &t;
    }
    return best;
}

}  // namespace

int layernorm_tier_count() { return kLnN; }

const char* layernorm_tier_name_at(int dtype, int i) {
    const LnTier* t = table(dtype);
    return (t && i >= 0 && i < kLnN) ? t[i].name : nullptr;
}

bool layernorm_force_tier(int dtype, int i) {
    if (dtype < 0 || dtype > 2 || i < -1 || i >= kLnN) return false;
    g_force[dtype].store(i);
    return true;
}

const char* layernorm_tier_name(int dtype, int64_t hidden, int vec_bytes, int64_t rows) {
    const LnTier* t = pick_dtype(dtype, hidden, vec_bytes, rows);
    return t ? t->name : nullptr;
}

cudaError_t layernorm_launch(int dtype, void* out, const void* x, const void* residual,
                             const void* bias, const void* gamma, const void* beta, int64_t rows,
                             int64_t hidden, float eps, int vec_bytes, cudaStream_t stream,
                             bool* supported) {
    const LnTier* t = pick_dtype(dtype, hidden, vec_bytes, rows);
    *supported = t != nullptr;
    if (!t) return cudaSuccess;
    return t->fn(out, x, residual, bias, gamma, beta, rows, (int)hidden, eps, stream);
}

}  // namespace tt
