// softmax_kernels.cuh -- the padded masked-softmax kernels (SM-1..SM-5); tier
// tables, launchers and selection are in softmax.cu (design notes there).
#pragma once

#include "common.cuh"
#include "softmax_row.cuh"

namespace tt {

constexpr float kLog2e = 1.4426950408889634f;

template <typename T, int VB, int G, int NV, int R, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) softmax_rows_kernel(T* __restrict__ scores,
                                                          const int32_t* __restrict__ lengths,
                                                          int64_t nrows, int64_t rows_per_batch,
                                                          int Sk, float c) {
    PdlScope pdl_;  // griddepcontrol.wait first: no global access before it (PDL)
    constexpr int VE = VB / (int)sizeof(T);          // elements per vector
    constexpr int HI = (VE - 1 + G - 1) / G;         // head / tail iterations per lane
    constexpr int GPB = NT / G;                      // groups per CTA
    constexpr int NWG = G > 32 ? G / 32 : 1;         // warps per group (CTA tier)
    __shared__ float red_max[G > 32 ? R * NWG : 1];
    __shared__ float red_sum[G > 32 ? R * NWG : 1];

    const int q = threadIdx.x % G;
    const int gi = threadIdx.x / G;
    const int64_t base = (int64_t)blockIdx.x * GPB * R;

    T* p[R];
    int Lr[R], hd[R], nv[R];
    bool live[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int64_t row = base + (int64_t)r * GPB + gi;
        live[r] = row < nrows;
        const int64_t rr = live[r] ? row : 0;
        p[r] = scores + rr * (int64_t)Sk;
        const int mis = (int)((reinterpret_cast<uintptr_t>(p[r]) & (VB - 1)) / sizeof(T));
        hd[r] = mis ? min(VE - mis, Sk) : 0;
        nv[r] = (Sk - hd[r]) / VE;
        int L = live[r] ? __ldg(lengths + rr / rows_per_batch) : 0;
        Lr[r] = min(max(L, 0), Sk);
    }

    // ---- SM-2: load the valid prefix, scaled into the log2 domain
    float v[R][NV][VE];
    float hv[R][HI], tv[R][HI];
#pragma unroll
    for (int r = 0; r < R; ++r) {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int vi = q + k * G;
            const int j0 = hd[r] + vi * VE;
            if (vi < nv[r] && j0 < Lr[r]) {
                Raw<VB> w;
                ld_stream<VB>(p[r] + j0, w);
                Elem<T>::template unpack<VB>(w, v[r][k]);
                if (j0 + VE <= Lr[r]) {  // whole vector valid: no per-element mask
#pragma unroll
                    for (int e = 0; e < VE; ++e) v[r][k][e] *= c;
                } else {
#pragma unroll
                    for (int e = 0; e < VE; ++e)
                        v[r][k][e] = (j0 + e < Lr[r]) ? v[r][k][e] * c : -INFINITY;
                }
            } else {
#pragma unroll
                for (int e = 0; e < VE; ++e) v[r][k][e] = -INFINITY;
            }
        }
        const int tl0 = hd[r] + nv[r] * VE;
#pragma unroll
        for (int i = 0; i < HI; ++i) {
            const int jh = q + i * G;
            hv[r][i] = (jh < hd[r] && jh < Lr[r]) ? Elem<T>::to_f(p[r][jh]) * c : -INFINITY;
            const int jt = tl0 + q + i * G;
            tv[r][i] = (jt < Sk && jt < Lr[r]) ? Elem<T>::to_f(p[r][jt]) * c : -INFINITY;
        }
    }

    // ---- SM-3: row max
    float m[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        float a = -INFINITY;
#pragma unroll
        for (int k = 0; k < NV; ++k)
#pragma unroll
            for (int e = 0; e < VE; ++e) a = fmaxf(a, v[r][k][e]);
#pragma unroll
        for (int i = 0; i < HI; ++i) a = fmaxf(a, fmaxf(hv[r][i], tv[r][i]));
        m[r] = a;
    }
    group_max<G, R>(m, red_max);

    // ---- SM-4: exponentiate once, sum
    float s[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const float mm = (m[r] == -INFINITY) ? 0.f : m[r];  // empty row: keep e = 0
        float a = 0.f;
#pragma unroll
        for (int k = 0; k < NV; ++k)
#pragma unroll
            for (int e = 0; e < VE; ++e) {
                v[r][k][e] = ex2_approx(v[r][k][e] - mm);
                a += v[r][k][e];
            }
#pragma unroll
        for (int i = 0; i < HI; ++i) {
            hv[r][i] = ex2_approx(hv[r][i] - mm);
            tv[r][i] = ex2_approx(tv[r][i] - mm);
            a += hv[r][i] + tv[r][i];
        }
        s[r] = a;
    }
    group_sum<G, R>(s, red_sum);

    // ---- SM-5: normalise valid keys, +0.0 for padding keys, store every column
#pragma unroll
    for (int r = 0; r < R; ++r) {
        if (!live[r]) continue;
        const float inv = 1.0f / s[r];
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int vi = q + k * G;
            if (vi < nv[r]) {
                const int j0 = hd[r] + vi * VE;
                float y[VE];
                if (j0 + VE <= Lr[r]) {
#pragma unroll
                    for (int e = 0; e < VE; ++e) y[e] = v[r][k][e] * inv;
                } else {
#pragma unroll
                    for (int e = 0; e < VE; ++e) y[e] = (j0 + e < Lr[r]) ? v[r][k][e] * inv : 0.f;
                }
                Raw<VB> w;
                Elem<T>::template pack<VB>(y, w);
                st_stream<VB>(p[r] + j0, w);
            }
        }
        const int tl0 = hd[r] + nv[r] * VE;
#pragma unroll
        for (int i = 0; i < HI; ++i) {
            const int jh = q + i * G;
            if (jh < hd[r]) p[r][jh] = Elem<T>::from_f(jh < Lr[r] ? hv[r][i] * inv : 0.f);
            const int jt = tl0 + q + i * G;
            if (jt < Sk) p[r][jt] = Elem<T>::from_f(jt < Lr[r] ? tv[r][i] * inv : 0.f);
        }
    }
}


// ----------------------------------------------------------------------------
// Warp / sub-warp tier (G <= 32), the production path for rows up to
// 32 * NV * VE keys.  CTA b owns GPB * rpg consecutive rows (rpg = rows per
// group); its groups walk them GPB rows at a time.  Instruction budget per
// row is what limits this kernel on B200 once the loads are deep enough, so:
//   * the request length is looked up once per CTA when the CTA's rows all
//     belong to one request (the common case), else per row, with the next
//     row's length prefetched and the row -> request division done by a
//     multiply-high (FastDivU32);
//   * loads are never predicated off: a lane whose vector lies past the valid
//     prefix re-reads the row's first vector (a valid, cached address), so
//     no sentinel initialisation is needed, and those duplicates of valid
//     keys cannot raise the max;
//   * the max is taken over RAW values (max if scale > 0, min if < 0), so
//     each exponent is one FFMA + one MUFU.EX2: e = 2^(x*c - c*m);
//   * a row with every key valid (L == Sk) skips all masking; otherwise each
//     element is masked once, to the +-inf sentinel, which the FFMA/EX2 turns
//     into e = +0.0 (scale == 0 is mapped to a tiny positive c on the host);
//   * ALIGNED (row pitch and base are multiples of VB) drops the scalar head /
//     tail code entirely.
// ----------------------------------------------------------------------------
// Rows [first, row_end) of this CTA -- all of ONE request, so one valid
// length L -- GC lanes per row, walked in warp-uniform slabs (every lane of a
// warp runs the same number of passes).
// PF: cross-row prefetch -- the loads of a group's next row are issued
// before the current row is computed, so each warp keeps two rows in flight
// (for rows under ~1 KB one row per warp is too few bytes in flight per SM).
template <typename T, int VB, int GC, int NVC, int NT, bool ALIGNED, bool NARROW, bool UP,
          bool PF = false, bool EF = false>
__device__ __forceinline__ void softmax_cta_rows(T* __restrict__ scores, uint32_t first,
                                                 uint32_t row_end, int Sk, float c, int L) {
    constexpr int GPW = 32 / GC;  // rows per warp per pass
    const int lane = threadIdx.x & 31;
    const int q = lane % GC;
    const uint32_t step = (NT / 32) * GPW;
    uint32_t row = first + (threadIdx.x >> 5) * GPW + lane / GC;
    if constexpr (PF) {
        using RR = RowRaw<T, VB, GC, NVC, ALIGNED>;
        uint32_t base = first + (threadIdx.x >> 5) * GPW;
        if (base >= row_end) return;  // warp-uniform
        bool live = row < row_end;
        T* pc = scores + (size_t)(live ? row : first) * (size_t)Sk;
        RR cur;
        row_load<T, VB, GC, NVC, ALIGNED>(pc, live ? L : 0, Sk, q, cur);
        for (; base < row_end; base += step, row += step) {
            const uint32_t rn = row + step;
            const bool ln = rn < row_end;
            T* pn = scores + (size_t)(ln ? rn : first) * (size_t)Sk;
            RR nxt;
            if (base + step < row_end)  // warp-uniform: another pass follows
                row_load<T, VB, GC, NVC, ALIGNED>(pn, ln ? L : 0, Sk, q, nxt);
            row_finish<T, VB, GC, NVC, ALIGNED, NARROW, UP, EF>(pc, live, live ? L : 0, Sk, c, q,
                                                               cur);
            cur = nxt;
            pc = pn;
            live = ln;
        }
        return;
    }
    for (uint32_t base = first + (threadIdx.x >> 5) * GPW; base < row_end; base += step, row += step) {
        const bool live = row < row_end;
        // a dead slot re-reads the range's last row (any row of the range is a
        // valid address; `first` is then not needed inside the loop)
        T* p = scores + (size_t)(live ? row : row_end - 1) * (size_t)Sk;
        const int Lr = live ? L : 0;
        RowRaw<T, VB, GC, NVC, ALIGNED> rr;
        row_load<T, VB, GC, NVC, ALIGNED>(p, Lr, Sk, q, rr);
        row_finish<T, VB, GC, NVC, ALIGNED, NARROW, UP, EF>(p, live, Lr, Sk, c, q, rr);
    }
}

// Rows of one request with L <= G * K * VE on a tier of NV > K vectors per lane:
// run them with K vectors per lane (K = 1 .. NV-1, smallest that fits).
template <typename T, int VB, int G, int K, int NV, int NT, bool ALIGNED, bool UP, bool PF, bool EF>
__device__ __forceinline__ bool softmax_narrow_nv(T* __restrict__ scores, uint32_t first,
                                                  uint32_t row_end, int Sk, float c, int L) {
    if constexpr (K >= NV) {
        return false;
    } else {
        constexpr int VE = VB / (int)sizeof(T);
        if (L <= G * K * VE) {
            softmax_cta_rows<T, VB, G, K, NT, ALIGNED, true, UP, PF, EF>(scores, first, row_end,
                                                                          Sk, c, L);
            return true;
        }
        return softmax_narrow_nv<T, VB, G, K + 1, NV, NT, ALIGNED, UP, PF, EF>(scores, first,
                                                                               row_end, Sk, c, L);
    }
}

// One request segment [first, row_end), valid length L: the tier's full path,
// or a narrower one when L is short.
template <typename T, int VB, int G, int NV, int NT, bool ALIGNED, bool UP, bool PF, bool EF>
__device__ __forceinline__ void softmax_segment(T* __restrict__ scores, uint32_t first,
                                                uint32_t row_end, int Sk, float c, int L) {
    constexpr int VE = VB / (int)sizeof(T);
    if constexpr (G == 32 && NV == 1) {
        // short request: compute on narrower groups (more rows per warp pass)
        // and zero-fill the padding vectors
        // (unaligned rows: only widths whose scalar head / tail fit one pass,
        // GC >= VE - 1, so the narrow paths do not raise register pressure)
        constexpr bool ok4 = ALIGNED || 4 >= VE - 1, ok8 = ALIGNED || 8 >= VE - 1;
        if (L < Sk) {
            if (ok4 && L <= 4 * VE)
                return softmax_cta_rows<T, VB, 4, 1, NT, ALIGNED, ok4, UP, PF, EF>(
                    scores, first, row_end, Sk, c, L);
            if (ok8 && L <= 8 * VE)
                return softmax_cta_rows<T, VB, 8, 1, NT, ALIGNED, ok8, UP, PF, EF>(
                    scores, first, row_end, Sk, c, L);
            if (L <= 16 * VE)
                return softmax_cta_rows<T, VB, 16, 1, NT, ALIGNED, true, UP, PF, EF>(
                    scores, first, row_end, Sk, c, L);
        }
    }
    if constexpr (NV > 1) {
        // short request on a multi-vector tier: the fewest vectors per lane that
        // hold its valid keys; the padding vectors are zero-filled without
        // arithmetic (NARROW), so a row's cost follows L_b instead of Sk
        if (L < Sk) {
            if (softmax_narrow_nv<T, VB, G, 1, NV, NT, ALIGNED, UP, PF, EF>(scores, first, row_end,
                                                                            Sk, c, L))
                return;
        }
    }
    softmax_cta_rows<T, VB, G, NV, NT, ALIGNED, false, UP, PF, EF>(scores, first, row_end, Sk, c, L);
}

// CTA b owns rows [first, row_end) of ONE request: the grid is laid out as
// `cpr` CTAs per request (cpr = ceil(rows_per_request / rows_per_cta)), so the
// request -- and its valid length, loaded once -- is known per CTA and no
// per-row length lookup, division or test exists in the row loop.
template <typename T, int VB, int G, int NV, int NT, bool ALIGNED, bool UP, bool PF, bool EF>
__device__ __forceinline__ void softmax_warp_body(T* __restrict__ scores,
                                                  const int32_t* __restrict__ lengths,
                                                  FastDivU32 cpr, uint32_t rpb, int Sk, float c,
                                                  int rpg) {
    constexpr int GPB = NT / G;
    static_assert(G <= 32, "warp tier");
    const uint32_t per_cta = (uint32_t)(GPB * rpg);
    const uint32_t req = cpr.div(blockIdx.x);
    const uint32_t first = req * rpb + (blockIdx.x - req * cpr.d) * per_cta;
    const uint32_t row_end = min(first + per_cta, (req + 1) * rpb);
    const int L = min(max(__ldg(lengths + req), 0), Sk);
    softmax_segment<T, VB, G, NV, NT, ALIGNED, UP, PF, EF>(scores, first, row_end, Sk, c, L);
}

template <typename T, int VB, int G, int NV, int NT, int MINB, bool ALIGNED, bool PF, bool EF>
__global__ void __launch_bounds__(NT, MINB) softmax_warp_kernel(T* __restrict__ scores,
                                                                const int32_t* __restrict__ lengths,
                                                                FastDivU32 cpr, uint32_t rpb,
                                                                int Sk, float c, int rpg) {
    PdlScope pdl_;  // griddepcontrol.wait first: no global access before it (PDL)
    if (c > 0.f)  // uniform: the sign of the scale picks the max or min reduction
        softmax_warp_body<T, VB, G, NV, NT, ALIGNED, true, PF, EF>(scores, lengths, cpr, rpb, Sk, c,
                                                               rpg);
    else
        softmax_warp_body<T, VB, G, NV, NT, ALIGNED, false, PF, EF>(scores, lengths, cpr, rpb, Sk,
                                                                c, rpg);
}

// ----------------------------------------------------------------------------
// TMA-staged variant for warp-sized rows (G = 32): a persistent kernel where
// every warp streams its rows through a private ring of D shared-memory slots.
// Lane 0 issues one 1-D bulk copy (cp.async.bulk, SASS UBLKCP) per row, of the
// row's VALID prefix only (16-byte aligned span), D rows ahead of the row being
// computed, so the bytes in flight per SM are set by the ring depth instead of
// by the register file.  The math and the stores are those of
// softmax_rows_kernel; the body is read from shared memory in 16-byte chunks
// (lane-contiguous, conflict-free LDS.128) and written with 16-byte STG.
// ----------------------------------------------------------------------------
template <typename T, int NV, int NW>
__global__ void __launch_bounds__(NW * 32) softmax_tma_kernel(T* __restrict__ scores,
                                                              const int32_t* __restrict__ lengths,
                                                              int64_t nrows, int64_t rows_per_batch,
                                                              int Sk, float c, int D,
                                                              int slot_bytes) {
    PdlScope pdl_;  // griddepcontrol.wait first: no global access before it (PDL)
    constexpr int E = (int)sizeof(T);
    constexpr int VE = 16 / E;               // elements per 16-byte chunk
    constexpr int HI = (VE - 1 + 31) / 32;   // = 1
    extern __shared__ __align__(128) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem) + warp * D;
    unsigned char* ring = smem + ((NW * D * 8 + 127) & ~127) + (size_t)warp * D * slot_bytes;
    const int64_t TW = (int64_t)gridDim.x * NW;
    const int64_t gw = (int64_t)blockIdx.x * NW + warp;

    auto row_len = [&](int64_t row) {
        const int L = __ldg(lengths + row / rows_per_batch);
        return min(max(L, 0), Sk);
    };
    // lane 0: stage row `row` into slot `sl` (valid prefix only)
    auto issue = [&](int64_t row, int sl) {
        if (row >= nrows) return;
        const int L = row_len(row);
        const uintptr_t a = reinterpret_cast<uintptr_t>(scores + row * (int64_t)Sk);
        if (L == 0) {
            mbar_arrive(&bars[sl]);  // nothing to read: complete the phase
            return;
        }
        const uintptr_t a0 = a & ~(uintptr_t)15;
        const uint32_t bytes = (uint32_t)(((a + (uintptr_t)L * E + 15) & ~(uintptr_t)15) - a0);
        mbar_arrive_expect_tx(&bars[sl], bytes);
        tma_load_1d(ring + (size_t)sl * slot_bytes, reinterpret_cast<const void*>(a0), bytes,
                    &bars[sl]);
    };

    if (lane == 0) {
        for (int s = 0; s < D; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
        fence_proxy_async_smem();
        for (int s = 0; s < D; ++s) issue(gw + s * TW, s);
    }
    __syncwarp();

    int sl = 0;
    uint32_t ph = 0;
    for (int64_t row = gw; row < nrows; row += TW) {
        T* p = scores + row * (int64_t)Sk;
        const int L = row_len(row);
        const int off = (int)(reinterpret_cast<uintptr_t>(p) & 15);
        const int hd = off ? min((16 - off) / E, Sk) : 0;
        const int nb = (Sk - hd) / VE;
        const int tl0 = hd + nb * VE;
        const unsigned char* slot = ring + (size_t)sl * slot_bytes;
        const unsigned char* body = slot + (off ? 16 : 0);

        mbar_wait(&bars[sl], ph);

        // ---- SM-2: shared -> registers, scaled into the log2 domain
        float v[NV][VE];
        float hv[HI], tv[HI];
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int ci = lane + 32 * k;
            const int j0 = hd + ci * VE;
            if (ci < nb && j0 < L) {
                Raw<16> w;
                lds128(body + 16 * ci, w.w);
                Elem<T>::template unpack<16>(w, v[k]);
                if (j0 + VE <= L) {
#pragma unroll
                    for (int e = 0; e < VE; ++e) v[k][e] *= c;
                } else {
#pragma unroll
                    for (int e = 0; e < VE; ++e) v[k][e] = (j0 + e < L) ? v[k][e] * c : -INFINITY;
                }
            } else {
#pragma unroll
                for (int e = 0; e < VE; ++e) v[k][e] = -INFINITY;
            }
        }
#pragma unroll
        for (int i = 0; i < HI; ++i) {
            const int jh = lane + 32 * i;
            hv[i] = (jh < hd && jh < L)
                        ? Elem<T>::to_f(*reinterpret_cast<const T*>(slot + off + jh * E)) * c
                        : -INFINITY;
            const int jt = tl0 + lane + 32 * i;
            tv[i] = (jt < Sk && jt < L)
                        ? Elem<T>::to_f(*reinterpret_cast<const T*>(body + 16 * nb +
                                                                    (jt - tl0) * E)) * c
                        : -INFINITY;
        }

        // ---- SM-3: row max (consumes every staged value)
        float m[1];
        {
            float a = -INFINITY;
#pragma unroll
            for (int k = 0; k < NV; ++k)
#pragma unroll
                for (int e = 0; e < VE; ++e) a = fmaxf(a, v[k][e]);
#pragma unroll
            for (int i = 0; i < HI; ++i) a = fmaxf(a, fmaxf(hv[i], tv[i]));
            m[0] = a;
        }
        group_max<32, 1>(m, nullptr);

        // slot consumed: refill it with the row D iterations ahead
        __syncwarp();
        if (lane == 0) {
            fence_proxy_async_smem();
            issue(row + (int64_t)D * TW, sl);
        }
        if (++sl == D) {
            sl = 0;
            ph ^= 1;
        }

        // ---- SM-4: exponentiate once, sum
        const float mm = (m[0] == -INFINITY) ? 0.f : m[0];
        float s[1] = {0.f};
#pragma unroll
        for (int k = 0; k < NV; ++k)
#pragma unroll
            for (int e = 0; e < VE; ++e) {
                v[k][e] = ex2_approx(v[k][e] - mm);
                s[0] += v[k][e];
            }
#pragma unroll
        for (int i = 0; i < HI; ++i) {
            hv[i] = ex2_approx(hv[i] - mm);
            tv[i] = ex2_approx(tv[i] - mm);
            s[0] += hv[i] + tv[i];
        }
        group_sum<32, 1>(s, nullptr);

        // ---- SM-5: normalise, +0.0 for padding keys, store every column
        const float inv = 1.0f / s[0];
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int ci = lane + 32 * k;
            if (ci < nb) {
                const int j0 = hd + ci * VE;
                float y[VE];
                if (j0 + VE <= L) {
#pragma unroll
                    for (int e = 0; e < VE; ++e) y[e] = v[k][e] * inv;
                } else {
#pragma unroll
                    for (int e = 0; e < VE; ++e) y[e] = (j0 + e < L) ? v[k][e] * inv : 0.f;
                }
                Raw<16> w;
                Elem<T>::template pack<16>(y, w);
                st_stream<16>(p + j0, w);
            }
        }
#pragma unroll
        for (int i = 0; i < HI; ++i) {
            const int jh = lane + 32 * i;
            if (jh < hd) p[jh] = Elem<T>::from_f(jh < L ? hv[i] * inv : 0.f);
            const int jt = tl0 + lane + 32 * i;
            if (jt < Sk) p[jt] = Elem<T>::from_f(jt < L ? tv[i] * inv : 0.f);
        }
    }
}

// ----------------------------------------------------------------------------
// Cluster tier (rows longer than one CTA holds in registers; north_star "rows
// are mapped to warps or clusters by length"): the row is cut into segments of
// W = NT * NV * VE keys, one per CTA of a thread-block cluster of ceil(Sk / W)
// CTAs (<= 8, portable).  Each CTA keeps its segment in registers (SM-2),
// takes its local max m_c and local sum s_c = sum 2^(t - m_c) (SM-3 / SM-4),
// and publishes (m_c, s_c) in its shared memory; after one cluster barrier
// every CTA reads all partners' pairs through distributed shared memory and
// merges them, (M, S) = (max m_c, sum s_c 2^(m_c - M)) -- the (m, s) merge of
// then writes y = e 2^(m_c - M) / S (SM-5).  Every key is
// read from HBM once and written once; a second cluster barrier keeps each
// CTA's shared memory alive until its partners have read it.
// t = x * c is computed explicitly (c = scale * log2 e, either sign).
// ----------------------------------------------------------------------------
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cluster_nctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n"
                 "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// float at the same shared-memory offset in CTA `rank` of this cluster
__device__ __forceinline__ float ld_dsmem_f32(const float* local, uint32_t rank) {
    uint32_t remote;
    float v;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(local)), "r"(rank));
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(remote) : "memory");
    return v;
}

template <typename T, int VB, int NV, int NT>
__global__ void __launch_bounds__(NT, 1) softmax_cluster_kernel(T* __restrict__ scores,
                                                                const int32_t* __restrict__ lengths,
                                                                int64_t rows_per_batch, int Sk,
                                                                float c) {
    PdlScope pdl_;  // griddepcontrol.wait first: no global access before it (PDL)
    constexpr int VE = VB / (int)sizeof(T);
    constexpr int W = NT * NV * VE;          // keys per CTA segment
    constexpr int HI = (VE - 1 + NT - 1) / NT;
    constexpr int NW = NT / 32;
    __shared__ float red_m[NW], red_s[NW];
    __shared__ float part[2];                // this CTA's (m_c, s_c), read by the cluster

    const uint32_t cr = cluster_ctarank(), ncl = cluster_nctarank();
    const int64_t row = (int64_t)(blockIdx.x / ncl);
    const int q = threadIdx.x;
    const int seg0 = (int)cr * W;
    const int Sks = min(W, Sk - seg0);       // keys in this segment (>= 1)
    T* p = scores + row * (int64_t)Sk + seg0;
    const int L = min(max(__ldg(lengths + row / rows_per_batch), 0), Sk);
    const int Ls = min(max(L - seg0, 0), Sks);  // valid keys in this segment
    const int mis = (int)((reinterpret_cast<uintptr_t>(p) & (VB - 1)) / sizeof(T));
    const int hd = mis ? min(VE - mis, Sks) : 0;
    const int nv = (Sks - hd) / VE;
    const int tl0 = hd + nv * VE;

    // ---- SM-2: the valid prefix of this segment, t = x * c (log2 domain)
    float v[NV][VE], hv[HI], tv[HI];
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        const int vi = q + k * NT;
        const int j0 = hd + vi * VE;
        if (vi < nv && j0 < Ls) {
            Raw<VB> w;
            ld_stream<VB>(p + j0, w);
            Elem<T>::template unpack<VB>(w, v[k]);
#pragma unroll
            for (int e = 0; e < VE; ++e) v[k][e] = (j0 + e < Ls) ? v[k][e] * c : -INFINITY;
        } else {
#pragma unroll
            for (int e = 0; e < VE; ++e) v[k][e] = -INFINITY;
        }
    }
#pragma unroll
    for (int i = 0; i < HI; ++i) {
        const int jh = q + i * NT, jt = tl0 + q + i * NT;
        hv[i] = (jh < hd && jh < Ls) ? Elem<T>::to_f(p[jh]) * c : -INFINITY;
        tv[i] = (jt < Sks && jt < Ls) ? Elem<T>::to_f(p[jt]) * c : -INFINITY;
    }
    // ---- SM-3: local max m_c
    float m[1] = {-INFINITY};
#pragma unroll
    for (int k = 0; k < NV; ++k)
#pragma unroll
        for (int e = 0; e < VE; ++e) m[0] = fmaxf(m[0], v[k][e]);
#pragma unroll
    for (int i = 0; i < HI; ++i) m[0] = fmaxf(m[0], fmaxf(hv[i], tv[i]));
    group_max<NT, 1>(m, red_m);
    const float mc = m[0];
    const float mm = mc == -INFINITY ? 0.f : mc;  // empty segment: e = 0 everywhere
    // ---- SM-4: e = 2^(t - m_c) once, local sum s_c
    float s[1] = {0.f};
#pragma unroll
    for (int k = 0; k < NV; ++k)
#pragma unroll
        for (int e = 0; e < VE; ++e) {
            v[k][e] = ex2_approx(v[k][e] - mm);
            s[0] += v[k][e];
        }
#pragma unroll
    for (int i = 0; i < HI; ++i) {
        hv[i] = ex2_approx(hv[i] - mm);
        tv[i] = ex2_approx(tv[i] - mm);
        s[0] += hv[i] + tv[i];
    }
    group_sum<NT, 1>(s, red_s);
    // ---- the cluster merge: (M, S) over the segments' (m_c, s_c)
    if (q == 0) {
        part[0] = mc;
        part[1] = s[0];
    }
    cluster_sync_all();
    float M = -INFINITY, Sum = 0.f;
    for (uint32_t r = 0; r < ncl; ++r) M = fmaxf(M, ld_dsmem_f32(&part[0], r));
    for (uint32_t r = 0; r < ncl; ++r) {
        const float mr = ld_dsmem_f32(&part[0], r);
        if (mr != -INFINITY) Sum += ld_dsmem_f32(&part[1], r) * ex2_approx(mr - M);
    }
    cluster_sync_all();  // partners are done reading this CTA's `part`
    // ---- SM-5: y = e 2^(m_c - M) / S; +0.0 past L (e = 0 there); L = 0: all zero
    const float f = (L > 0 && mc != -INFINITY) ? ex2_approx(mc - M) / Sum : 0.f;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        const int vi = q + k * NT;
        if (vi < nv) {
            float y[VE];
#pragma unroll
            for (int e = 0; e < VE; ++e) y[e] = v[k][e] * f;
            Raw<VB> w;
            Elem<T>::template pack<VB>(y, w);
            st_stream<VB>(p + hd + vi * VE, w);
        }
    }
#pragma unroll
    for (int i = 0; i < HI; ++i) {
        const int jh = q + i * NT, jt = tl0 + q + i * NT;
        if (jh < hd) p[jh] = Elem<T>::from_f(hv[i] * f);
        if (jt < Sks) p[jt] = Elem<T>::from_f(tv[i] * f);
    }
}


// ----------------------------------------------------------------------------
// Rows of any length (beyond the cluster tier's 8 register-resident segments):
// softmax_long.  A cluster of C CTAs per row, CTA r owns the key segment
// [r W, (r + 1) W) (W = ceil(Sk / C) rounded up to 64 keys) and makes TWO
// passes over it: pass 1 streams the segment's valid keys from HBM and keeps a
// per-thread online (m, s) -- s rescaled by 2^(m_old - m_new) when the running
// max grows --, the CTA and then the cluster merge
// the pairs exactly as softmax_cluster does (distributed shared memory);
// pass 2 re-reads the valid keys (an L2 hit while the live segments fit in the
// 126 MB L2: 2 x 148 CTAs x W keys), writes y = 2^(t - M) / S and +0.0 past L.
// t = x * c is recomputed with the same fp32 multiply in both passes.  HBM
// traffic per row: L e (+ the L2 re-read) + Sk e, one write per key.
// ----------------------------------------------------------------------------
template <typename T, int NT, int U, int MINB>
__global__ void __launch_bounds__(NT, MINB) softmax_long_kernel(T* __restrict__ scores,
                                                             const int32_t* __restrict__ lengths,
                                                             int64_t rows_per_batch, int Sk,
                                                             int W, float c) {
    PdlScope pdl_;  // griddepcontrol.wait first: no global access before it (PDL)
    constexpr int VB = 16, VE = VB / (int)sizeof(T);
    __shared__ float red_m[NT / 32], red_s[NT / 32];
    __shared__ float part[2];  // this CTA's (m_c, s_c), read by the cluster

    const uint32_t cr = cluster_ctarank(), ncl = cluster_nctarank();
    const int64_t row = (int64_t)(blockIdx.x / ncl);
    const int q = threadIdx.x;
    const int seg0 = (int)min((int64_t)cr * W, (int64_t)Sk);
    const int Sks = min(W, Sk - seg0);  // keys in this segment (may be 0)
    T* p = scores + row * (int64_t)Sk + seg0;
    const int L = min(max(__ldg(lengths + row / rows_per_batch), 0), Sk);
    const int Ls = min(max(L - seg0, 0), Sks);  // valid keys in this segment
    const int mis = (int)((reinterpret_cast<uintptr_t>(p) & (VB - 1)) / sizeof(T));
    const int hd = mis ? min(VE - mis, Sks) : 0;  // scalar head up to 16-byte alignment
    const int nv = (Sks - hd) / VE;
    const int tl0 = hd + nv * VE;  // scalar tail [tl0, Sks)

    // ---- pass 1: online (m, s) over the valid keys of the segment
    float m = -INFINITY, s = 0.f;
    auto absorb = [&](float t) {  // one more valid key
        const float mn = fmaxf(m, t);
        s = s * ex2_approx(m - mn) + ex2_approx(t - mn);
        m = mn;
    };
    // U vectors per thread in flight: all loads of a batch first, then one max,
    // one rescale and the exponentials of the batch
    for (int v0 = q; v0 < nv; v0 += NT * U) {
        if (hd + v0 * VE >= Ls) break;
        float x[U][VE];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int vi = v0 + u * NT, j0 = hd + vi * VE;
            if (vi < nv && j0 < Ls) {
                Raw<VB> w;
                ld_stream<VB>(p + j0, w);
                Elem<T>::template unpack<VB>(w, x[u]);
            }
        }
        float vm = -INFINITY;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int j0 = hd + (v0 + u * NT) * VE;
#pragma unroll
            for (int e = 0; e < VE; ++e) {
                x[u][e] = (v0 + u * NT < nv && j0 + e < Ls) ? x[u][e] * c : -INFINITY;
                vm = fmaxf(vm, x[u][e]);
            }
        }
        const float mn = fmaxf(m, vm);
        float acc = 0.f;
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int e = 0; e < VE; ++e) acc += ex2_approx(x[u][e] - mn);
        s = s * ex2_approx(m - mn) + acc;
        m = mn;
    }
    if (q < hd && q < Ls) absorb(Elem<T>::to_f(p[q]) * c);
    if (tl0 + q < Ls) absorb(Elem<T>::to_f(p[tl0 + q]) * c);  // q < VE - 1 < NT
    // ---- the CTA's pair (m_c, s_c)
    float mv[1] = {m};
    group_max<NT, 1>(mv, red_m);
    const float mc = mv[0];
    float sv[1] = {m == -INFINITY ? 0.f : s * ex2_approx(m - mc)};
    group_sum<NT, 1>(sv, red_s);
    if (q == 0) {
        part[0] = mc;
        part[1] = sv[0];
    }
    // ---- the cluster merge: (M, S) over the segments' (m_c, s_c)
    cluster_sync_all();
    float M = -INFINITY, Sum = 0.f;
    for (uint32_t r = 0; r < ncl; ++r) M = fmaxf(M, ld_dsmem_f32(&part[0], r));
    for (uint32_t r = 0; r < ncl; ++r) {
        const float mr = ld_dsmem_f32(&part[0], r);
        if (mr != -INFINITY) Sum += ld_dsmem_f32(&part[1], r) * ex2_approx(mr - M);
    }
    cluster_sync_all();  // partners are done reading this CTA's `part`
    // ---- pass 2: y = 2^(t - M) / S for j < L, +0.0 past L (L = 0: all zero)
    const float f = L > 0 ? 1.0f / Sum : 0.f;
    // batches in reverse order: the keys pass 1 read last are the likeliest to
    // still be in L2 when the live segments outgrow it
    const int nb = (nv + NT * U - 1) / (NT * U);
    for (int bi = nb - 1; bi >= 0; --bi) {
        const int v0 = q + bi * NT * U;
        float y[U][VE];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int vi = v0 + u * NT, j0 = hd + vi * VE;
            if (vi < nv && j0 < Ls) {
                Raw<VB> w;
                ld_stream<VB>(p + j0, w);
                Elem<T>::template unpack<VB>(w, y[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int vi = v0 + u * NT, j0 = hd + vi * VE;
            if (vi < nv) {
#pragma unroll
                for (int e = 0; e < VE; ++e)
                    y[u][e] = (j0 + e < Ls) ? ex2_approx(y[u][e] * c - M) * f : 0.f;
                Raw<VB> o;
                Elem<T>::template pack<VB>(y[u], o);
                st_stream<VB>(p + j0, o);
            }
        }
    }
    if (q < hd) p[q] = Elem<T>::from_f(q < Ls ? ex2_approx(Elem<T>::to_f(p[q]) * c - M) * f : 0.f);
    if (tl0 + q < Sks)
        p[tl0 + q] = Elem<T>::from_f(tl0 + q < Ls ? ex2_approx(Elem<T>::to_f(p[tl0 + q]) * c - M) * f : 0.f);
}

}  // namespace tt
