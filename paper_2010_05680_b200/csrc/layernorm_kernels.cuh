// layernorm_kernels.cuh -- the LayerNorm kernels (LN-1..LN-3); tier tables,
// launchers and selection are in layernorm.cu.  See layernorm.cu for the
// design notes.
#pragma once

#include "common.cuh"

namespace tt {

// ----------------------------------------------------------------------------
// Shared row arithmetic.  Every LayerNorm kernel below goes through these three
// functions, so each robustness test (offset, aliasing, gamma = 0) covers the
// same LN-1 / LN-2 / LN-3 code in every tier.  Element pairs use the packed
// fp32 FADD2 / FFMA2 / FMUL2 (IEEE round-to-nearest, like the scalar ops):
// one issue slot per two elements.
// ----------------------------------------------------------------------------

// LN-1: v = (x + bias) + residual (fp32), VE elements.
template <int VE>
__device__ __forceinline__ void ln_add(float (&v)[VE], const float* x, const float* b,
                                       const float* r) {
    if constexpr (VE % 2 == 0) {
#pragma unroll
        for (int e = 0; e < VE; e += 2) {
            const F2 t = f2_add(f2_add(f2_make(x[e], x[e + 1]), f2_make(b[e], b[e + 1])),
                                f2_make(r[e], r[e + 1]));
            f2_split(t, v[e], v[e + 1]);
        }
    } else {
#pragma unroll
        for (int e = 0; e < VE; ++e) v[e] = (x[e] + b[e]) + r[e];
    }
}

// LN-2 (DESIGN R9; Eq. 1 LHS): mean = K + sum(v - K) / N,
// K = the row's first element (identical in every lane of the group, so
// |mean| >> std loses no digits to the accumulator), then the population
// variance of the centred values, which REPLACE v (v <- v - mean).  Slots with
// q + k * G >= nvec lie outside the row and are skipped unless EXACT.  For
// G > 32, red_a / red_b hold R * G / 32 floats each (group_sum's CTA merge).
template <int G, int R, int NV, int VE, bool EXACT>
__device__ __forceinline__ void ln_moments(float (&v)[R][NV][VE], const float (&K)[R], int q,
                                           int nvec, float invN, float eps, float* red_a,
                                           float* red_b, float (&rstd)[R]) {
    float s[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const F2 nk = f2_make(-K[r], -K[r]);
        F2 a2 = f2_make(0.f, 0.f);
        float a1 = 0.f;
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            if (EXACT || q + k * G < nvec) {
                if constexpr (VE % 2 == 0) {
#pragma unroll
                    for (int e = 0; e < VE; e += 2)
                        a2 = f2_add(a2, f2_add(f2_make(v[r][k][e], v[r][k][e + 1]), nk));
                } else {
#pragma unroll
                    for (int e = 0; e < VE; ++e) a1 += v[r][k][e] - K[r];
                }
            }
        }
        float s0, s1;
        f2_split(a2, s0, s1);
        s[r] = (s0 + s1) + a1;
    }
    group_sum<G, R>(s, red_a);
    float q2[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const float mean = fmaf(s[r], invN, K[r]);
        const F2 nm = f2_make(-mean, -mean);
        F2 a2 = f2_make(0.f, 0.f);
        float a1 = 0.f;
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            if (EXACT || q + k * G < nvec) {
                if constexpr (VE % 2 == 0) {
#pragma unroll
                    for (int e = 0; e < VE; e += 2) {
                        const F2 d = f2_add(f2_make(v[r][k][e], v[r][k][e + 1]), nm);
                        f2_split(d, v[r][k][e], v[r][k][e + 1]);
                        a2 = f2_fma(d, d, a2);
                    }
                } else {
#pragma unroll
                    for (int e = 0; e < VE; ++e) {
                        v[r][k][e] -= mean;
                        a1 = fmaf(v[r][k][e], v[r][k][e], a1);
                    }
                }
            }
        }
        float s0, s1;
        f2_split(a2, s0, s1);
        q2[r] = (s0 + s1) + a1;
    }
    group_sum<G, R>(q2, red_b);
#pragma unroll
    for (int r = 0; r < R; ++r) rstd[r] = rsqrtf(fmaf(q2[r], invN, eps));
}

// LN-3: y = (d * rstd) * gamma + beta for VE centred values d.
template <int VE>
__device__ __forceinline__ void ln_affine(float (&y)[VE], const float (&d)[VE], float rstd,
                                          const float* g, const float* b) {
    if constexpr (VE % 2 == 0) {
        const F2 rs = f2_make(rstd, rstd);
#pragma unroll
        for (int e = 0; e < VE; e += 2) {
            const F2 t = f2_fma(f2_mul(f2_make(d[e], d[e + 1]), rs), f2_make(g[e], g[e + 1]),
                                f2_make(b[e], b[e + 1]));
            f2_split(t, y[e], y[e + 1]);
        }
    } else {
#pragma unroll
        for (int e = 0; e < VE; ++e) y[e] = fmaf(d[e] * rstd, g[e], b[e]);
    }
}

// ----------------------------------------------------------------------------
// CTA / generic tier: G threads per row (G <= 1024), R rows per group, any
// vector width (VB = sizeof(T): scalar rows of any pitch).  Parameters are
// read from global memory (L1-cached, shared by the CTA's rows).
// EARLY: gamma / beta are loaded together with the row (small, latency-bound
// problems: no dependent parameter load after the reductions).
// ----------------------------------------------------------------------------
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
    // ---- LN-1
    float v[R][NV][VE];
#pragma unroll
    for (int r = 0; r < R; ++r) {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int vi = q + k * G;
            if (live[r] && vi < nvec) {
                Raw<VB> wx, wr, wb;
                ld_stream<VB>(x + off[r] + vi * VE, wx);
                ld_stream<VB>(residual + off[r] + vi * VE, wr);
                ld_param<VB>(bias + vi * VE, wb);
                float fx[VE], fr[VE], fb[VE];
                Elem<T>::template unpack<VB>(wx, fx);
                Elem<T>::template unpack<VB>(wr, fr);
                Elem<T>::template unpack<VB>(wb, fb);
                ln_add<VE>(v[r][k], fx, fb, fr);
            } else {
#pragma unroll
                for (int e = 0; e < VE; ++e) v[r][k][e] = 0.f;
            }
        }
    }
    // ---- LN-2 (the shift K: the row's first element, the same in every lane)
    float K[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        if constexpr (G <= 32) {
            K[r] = __shfl_sync(0xffffffffu, v[r][0][0], (int)(threadIdx.x & 31) & ~(G - 1));
        } else {
            K[r] = live[r] ? (Elem<T>::to_f(x[off[r]]) + Elem<T>::to_f(bias[0])) +
                                 Elem<T>::to_f(residual[off[r]])
                           : 0.f;
        }
    }
    float rstd[R];
    ln_moments<G, R, NV, VE, false>(v, K, q, nvec, invN, eps, red_a, red_b, rstd);

    // ---- LN-3
#pragma unroll
    for (int r = 0; r < R; ++r) {
        if (!live[r]) continue;
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
                ln_affine<VE>(y, v[r][k], rstd[r], fg, fb);
                Raw<VB> wy;
                Elem<T>::template pack<VB>(y, wy);
                st_stream<VB>(out + off[r] + vi * VE, wy);
            }
        }
    }
}

// ----------------------------------------------------------------------------
// Warp / sub-warp tier (G <= 32, VB >= 16), the production path for hidden up
// to G * NV * VE.  Persistent CTAs (one wave); per CTA, bias / gamma / beta
// are widened to fp32 ONCE into shared memory in a lane-interleaved layout
// (quad j of vector c at float4 index (p * VE/4 + j) * nvec + c, so a warp's
// LDS.128 are conflict-free), which removes their per-row global loads and
// conversions.  EXACT (hidden == G * NV * VE, chosen at launch): every slot
// lies in the row, so no per-vector bounds test or branch is compiled.
// PF: every row's x / residual loads are issued one row ahead (raw registers,
// loop unrolled by two); otherwise the first row is prefetched into L2 while
// the parameters are staged.
// ----------------------------------------------------------------------------
template <typename T, int VB, int G, int NV, bool EXACT>
struct LnRow {
    static constexpr int VE = VB / (int)sizeof(T);
    static constexpr int QV = VE / 4;
    Raw<VB> x[NV], r[NV];

    __device__ __forceinline__ void load(const T* xp, const T* rp, size_t off, int q, int nvec) {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int vi = q + k * G;
            if (EXACT || vi < nvec) {
                ld_stream<VB>(xp + off + vi * VE, x[k]);
                ld_stream<VB>(rp + off + vi * VE, r[k]);
            }
        }
    }

    __device__ __forceinline__ void finish(T* out, size_t off, int q, int nvec, float invN,
                                           float eps, const float4* pb, const float4* pg,
                                           const float4* pe) const {
        // ---- LN-1
        float v[1][NV][VE];
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int vi = q + k * G;
            if (EXACT || vi < nvec) {
                float fx[VE], fr[VE], fb[VE];
                Elem<T>::template unpack<VB>(x[k], fx);
                Elem<T>::template unpack<VB>(r[k], fr);
#pragma unroll
                for (int j = 0; j < QV; ++j) {
                    const float4 b = pb[j * nvec + vi];
                    fb[4 * j] = b.x, fb[4 * j + 1] = b.y, fb[4 * j + 2] = b.z, fb[4 * j + 3] = b.w;
                }
                ln_add<VE>(v[0][k], fx, fb, fr);
            } else {
#pragma unroll
                for (int e = 0; e < VE; ++e) v[0][k][e] = 0.f;
            }
        }
        // ---- LN-2
        const float K[1] = {__shfl_sync(0xffffffffu, v[0][0][0], (int)(threadIdx.x & 31) & ~(G - 1))};
        float rstd[1];
        ln_moments<G, 1, NV, VE, EXACT>(v, K, q, nvec, invN, eps, nullptr, nullptr, rstd);
        // ---- LN-3.  The fence keeps the compiler from hoisting every gamma /
        // beta LDS above the reductions (3 x NV x QV float4 live at once made
        // ptxas spill the 16-bit hidden-1024 tiers).
        asm volatile("" ::: "memory");
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int vi = q + k * G;
            if (EXACT || vi < nvec) {
                float fg[VE], fe[VE], y[VE];
#pragma unroll
                for (int j = 0; j < QV; ++j) {
                    const float4 g = pg[j * nvec + vi], b = pe[j * nvec + vi];
                    fg[4 * j] = g.x, fg[4 * j + 1] = g.y, fg[4 * j + 2] = g.z, fg[4 * j + 3] = g.w;
                    fe[4 * j] = b.x, fe[4 * j + 1] = b.y, fe[4 * j + 2] = b.z, fe[4 * j + 3] = b.w;
                }
                ln_affine<VE>(y, v[0][k], rstd[0], fg, fe);
                Raw<VB> wy;
                Elem<T>::template pack<VB>(y, wy);
                st_stream<VB>(out + off + vi * VE, wy);
            }
        }
    }
};

// bias / gamma / beta -> fp32 shared memory, [3][QV][nvec] float4 (see above)
template <typename T, int VE, int NT>
__device__ __forceinline__ void ln_stage_params(float4* prm, const T* bias, const T* gamma,
                                                const T* beta, int hidden) {
    constexpr int QV = VE / 4;
    const int nvec = hidden / VE;
    for (int i = threadIdx.x; i < 3 * hidden; i += NT) {
        const int pi = i / hidden, col = i - pi * hidden;
        const T* src = pi == 0 ? bias : pi == 1 ? gamma : beta;
        const int c = col / VE, e = col - c * VE;
        reinterpret_cast<float*>(prm)[(((pi * QV + (e >> 2)) * nvec + c) << 2) + (e & 3)] =
            Elem<T>::to_f(src[col]);
    }
}

template <typename T, int VB, int G, int NV, int NT, int MINB, bool PF, bool EXACT>
__global__ void __launch_bounds__(NT, MINB)
    ln_warp_kernel(T* out, const T* x, const T* residual, const T* __restrict__ bias,
                   const T* __restrict__ gamma, const T* __restrict__ beta, uint32_t rows,
                   int hidden, float eps) {
    PdlScope pdl_;  // griddepcontrol.wait first: no global access before it (PDL)
    using Row = LnRow<T, VB, G, NV, EXACT>;
    constexpr int VE = Row::VE;
    constexpr int QV = Row::QV;
    constexpr int GPB = NT / G;
    static_assert(G <= 32 && VE % 4 == 0, "warp tier with >= 4-element vectors");
    extern __shared__ __align__(16) float4 prm[];  // [3][QV][nvec] float4
    const int nvec = EXACT ? G * NV : hidden / VE;
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
            if (EXACT || vi < nvec) {
                asm volatile("prefetch.global.L2 [%0];" ::"l"(x + off + vi * VE));
                asm volatile("prefetch.global.L2 [%0];" ::"l"(residual + off + vi * VE));
            }
        }
    }
    ln_stage_params<T, VE, NT>(prm, bias, gamma, beta, hidden);
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

#ifdef TT_TUNING
// ----------------------------------------------------------------------------
// TMA-staged variant (tuning candidate; measured slower than the warp tier,
// DESIGN §5): persistent CTAs; each warp streams its rows' x and residual
// through a private ring of D shared-memory slots filled by 1-D bulk copies
// (cp.async.bulk, SASS UBLKCP) issued D rows ahead.  Requires hidden *
// sizeof(T) % 16 == 0 and 16-byte aligned operands.
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
    ln_stage_params<T, VE, NW * 32>(prm, bias, gamma, beta, hidden);
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
        float v[1][NV][VE];
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int ci = lane + 32 * k;
            if (ci < nchunks) {
                Raw<16> wx, wr;
                lds128(slot + 16 * ci, wx.w);
                lds128(slot + rb + 16 * ci, wr.w);
                float fx[VE], fr[VE], fb[VE];
                Elem<T>::template unpack<16>(wx, fx);
                Elem<T>::template unpack<16>(wr, fr);
#pragma unroll
                for (int j = 0; j < QV; ++j) {
                    const float4 b = pb[j * nchunks + ci];
                    fb[4 * j] = b.x, fb[4 * j + 1] = b.y, fb[4 * j + 2] = b.z, fb[4 * j + 3] = b.w;
                }
                ln_add<VE>(v[0][k], fx, fb, fr);
            } else {
#pragma unroll
                for (int e = 0; e < VE; ++e) v[0][k][e] = 0.f;
            }
        }
        const float K[1] = {__shfl_sync(0xffffffffu, v[0][0][0], 0)};
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
        float rstd[1];
        ln_moments<32, 1, NV, VE, false>(v, K, lane, nchunks, invN, eps, nullptr, nullptr, rstd);
        // ---- LN-3
        T* o = out + row * (int64_t)hidden;
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int ci = lane + 32 * k;
            if (ci < nchunks) {
                float fg[VE], fe[VE], y[VE];
#pragma unroll
                for (int j = 0; j < QV; ++j) {
                    const float4 g = pg[j * nchunks + ci], b = pe[j * nchunks + ci];
                    fg[4 * j] = g.x, fg[4 * j + 1] = g.y, fg[4 * j + 2] = g.z, fg[4 * j + 3] = g.w;
                    fe[4 * j] = b.x, fe[4 * j + 1] = b.y, fe[4 * j + 2] = b.z, fe[4 * j + 3] = b.w;
                }
                ln_affine<VE>(y, v[0][k], rstd[0], fg, fe);
                Raw<16> wy;
                Elem<T>::template pack<16>(y, wy);
                st_stream<16>(o + ci * VE, wy);
            }
        }
    }
}
#endif  // TT_TUNING

}  // namespace tt
