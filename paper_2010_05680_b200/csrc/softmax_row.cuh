// softmax_row.cuh -- the per-row body of the warp / sub-warp softmax tiers,
// shared by the padded kernel (softmax.cu) and the packed, padding-free
// kernel (softmax_packed.cu).  See softmax.cu for the design notes.
#pragma once

#include <type_traits>

#include "common.cuh"

namespace tt {

// f16 bit pattern of the small integer n (0 <= n < 2048), exact
__host__ __device__ constexpr uint32_t f16_int_bits(int n) {
    int e = 0;
    while (n >> (e + 1)) ++e;
    return n == 0 ? 0u : (uint32_t)(((e + 15) << 10) | ((n - (1 << e)) << (10 - e)));
}
// the key indices (2 i, 2 i + 1) of word i of a vector, as an f16x2 pair
__host__ __device__ constexpr uint32_t f16_pair_index(int i) {
    return f16_int_bits(2 * i) | (f16_int_bits(2 * i + 1) << 16);
}

__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Raw bytes of one row as loaded by one lane: NVC body vectors plus the
// scalar head / tail elements (unaligned rows only).  Kept in registers
// between row_load and row_finish, so a group can issue the loads of its next
// row before it computes the current one (cross-row prefetch, PF tiers).
template <typename T, int VB, int GC, int NVC, bool ALIGNED>
struct RowRaw {
    static constexpr int VE = VB / (int)sizeof(T);
    static constexpr int HI = ALIGNED ? 0 : (VE - 1 + GC - 1) / GC;
    static constexpr int HIA = HI > 0 ? HI : 1;
    Raw<VB> raw[NVC];
    T h[HIA], t[HIA];
};

// Head length and body vector count of a row starting at p.
template <typename T, int VB, bool ALIGNED>
__device__ __forceinline__ void row_split(const T* p, int Sk, int& hd, int& nv) {
    constexpr int VE = VB / (int)sizeof(T);
    hd = 0;
    nv = Sk / VE;
    if constexpr (!ALIGNED) {
        const int mis = (int)((reinterpret_cast<uintptr_t>(p) & (VB - 1)) / sizeof(T));
        hd = mis ? min(VE - mis, Sk) : 0;
        nv = (Sk - hd) / VE;
    }
}

// ---- SM-2 (issue half): every load of the row -- body vectors and the scalar
// head / tail -- is issued before any of them is consumed, so a row costs one
// memory round trip.  Loads are never predicated off: a lane past the valid
// prefix (or every lane of an empty / dead row, L = 0) re-reads the first body
// vector, or (row shorter than its head) the VB-aligned vector containing p;
// the mask in row_finish turns those into sentinels.
template <typename T, int VB, int GC, int NVC, bool ALIGNED>
__device__ __forceinline__ void row_load(const T* __restrict__ p, int L, int Sk, int q,
                                         RowRaw<T, VB, GC, NVC, ALIGNED>& r) {
    using RR = RowRaw<T, VB, GC, NVC, ALIGNED>;
    constexpr int VE = RR::VE;
    int hd, nv;
    row_split<T, VB, ALIGNED>(p, Sk, hd, nv);
    const T* fb = nv > 0 ? p + hd
                         : reinterpret_cast<const T*>(reinterpret_cast<uintptr_t>(p) &
                                                      ~(uintptr_t)(VB - 1));
#pragma unroll
    for (int k = 0; k < NVC; ++k) {
        const int vi = q + k * GC;
        const int j0 = hd + vi * VE;
        const bool in = vi < nv && j0 < L;
        ld_stream<VB>(in ? p + j0 : fb, r.raw[k]);
    }
    if constexpr (!ALIGNED) {
        // an in-row key past L is loaded harmlessly and masked in row_finish
        const int tl0 = hd + nv * VE;
#pragma unroll
        for (int i = 0; i < RR::HI; ++i) {
            const int jh = q + i * GC, jt = tl0 + q + i * GC;
            r.h[i] = p[jh < hd ? jh : 0];
            r.t[i] = p[jt < Sk ? jt : 0];
        }
    }
}

// SM-2 (mask half) .. SM-5 for one row whose raw bytes are in r.  `live`
// false: the group has no row this step (it still joins the shuffles, which
// use the full warp mask; L must be 0).  NARROW: the request is short enough
// that every valid key lies in the head and the first GC body vectors; the
// remaining body vectors are written as zeros without any arithmetic.  UP:
// c > 0, so the row max of c*x is c*max(x) (else c*min(x)); a template
// parameter so that only one of the two reductions is compiled into each path.
template <typename T, int VB, int GC, int NVC, bool ALIGNED, bool NARROW, bool UP, bool EF = false,
          bool FULLROW = false>
__device__ __forceinline__ void row_finish(T* __restrict__ p, bool live, int L, int Sk, float c,
                                           int q, const RowRaw<T, VB, GC, NVC, ALIGNED>& r) {
    using RR = RowRaw<T, VB, GC, NVC, ALIGNED>;
    constexpr int VE = RR::VE;
    constexpr int HI = RR::HI;
    constexpr int HIA = RR::HIA;
    constexpr bool up = UP;  // max of raw x (else min); c != 0 (host)
    const float sent = up ? -INFINITY : INFINITY;
    int hd, nv;
    row_split<T, VB, ALIGNED>(p, Sk, hd, nv);
    const int tl0 = hd + nv * VE;
    // FULLROW (the packed layout: every key of every row valid, L = Sk) with at
    // least one body vector: no per-element mask.  Vector slots past the row
    // (vi >= nv) then hold a re-read copy of the row's first body vector
    // (row_load), which cannot change the max, and are left out of the sum by a
    // 0 / 1 weight (the sum's FADD2 becomes an FFMA2) and never stored.
    // Otherwise masking is needed unless every key is valid and every vector
    // slot of the group maps onto the row.  (Uniform within the group.  Not
    // compiled into the padded kernels: the extra path costs their 40-register
    // unaligned 16-bit tiers a spill, C3 fp16 -2 %.)
    const bool masked = FULLROW ? (L < Sk) || (nv == 0) : (L < Sk) || (nv != GC * NVC);
    const bool dead_slots = FULLROW && !masked && (nv != GC * NVC);

    float v[NVC][VE];
    // (not in the 16-bit G8 x NV5 tier: there the word masks made ptxas spill
    // 36-48 bytes of the row at its 64-register cap)
    constexpr bool kWordMask = sizeof(T) == 2 && !(GC == 8 && NVC == 5);
    if constexpr (kWordMask) {
        // 16-bit storage: the key mask on the packed words before unpacking --
        // per pair of keys one HSET2 (key index < nvalid, both halves at once,
        // indices as exact f16 constants) and one LOP3 that swaps the masked
        // halves for the sentinel's bit pattern: 1 instruction per key instead
        // of an ISETP + FSEL after the conversion
        constexpr uint32_t kSentH =
            std::is_same<T, __half>::value ? (UP ? 0xFC00u : 0x7C00u) : (UP ? 0xFF80u : 0x7F80u);
        constexpr uint32_t kSent2 = kSentH | (kSentH << 16);
#pragma unroll
        for (int k = 0; k < NVC; ++k) {
            Raw<VB> w = r.raw[k];
            if (masked) {
                const int vi = q + k * GC;
                const int nvalid = vi < nv ? min(max(L - (hd + vi * VE), 0), VE) : 0;
                const uint32_t h = __half_as_ushort(__int2half_rn(nvalid));
                const uint32_t h2 = h | (h << 16);
#pragma unroll
                for (int i = 0; i < Raw<VB>::W; ++i) {
                    uint32_t m;
                    asm("set.lt.u32.f16x2 %0, %1, %2;" : "=r"(m) : "r"(f16_pair_index(i)), "r"(h2));
                    w.w[i] = (w.w[i] & m) | (kSent2 & ~m);
                }
            }
            Elem<T>::template unpack<VB>(w, v[k]);
        }
    } else {
#pragma unroll
        for (int k = 0; k < NVC; ++k) Elem<T>::template unpack<VB>(r.raw[k], v[k]);
        if (masked) {
#pragma unroll
            for (int k = 0; k < NVC; ++k) {
                const int vi = q + k * GC;
                const int nvalid = vi < nv ? min(max(L - (hd + vi * VE), 0), VE) : 0;
#pragma unroll
                for (int e = 0; e < VE; ++e) v[k][e] = e < nvalid ? v[k][e] : sent;
            }
        }
    }
    float hv[HIA], tv[HIA];
    if constexpr (!ALIGNED) {
#pragma unroll
        for (int i = 0; i < HI; ++i) {
            const int jh = q + i * GC, jt = tl0 + q + i * GC;
            const bool ih = jh < hd && jh < L, it = jt < Sk && jt < L;
            hv[i] = ih ? Elem<T>::to_f(r.h[i]) : sent;
            tv[i] = it ? Elem<T>::to_f(r.t[i]) : sent;
        }
    }

    // ---- SM-3: row max of the scaled logits, c * (max or min of raw x)
    float m[1];
    {
        float a = sent;
        if constexpr (up) {
#pragma unroll
            for (int k = 0; k < NVC; ++k)
#pragma unroll
                for (int e = 0; e < VE; ++e) a = fmaxf(a, v[k][e]);
            if constexpr (!ALIGNED) {
#pragma unroll
                for (int i = 0; i < HI; ++i) a = fmaxf(a, fmaxf(hv[i], tv[i]));
            }
        } else {
#pragma unroll
            for (int k = 0; k < NVC; ++k)
#pragma unroll
                for (int e = 0; e < VE; ++e) a = fminf(a, v[k][e]);
            if constexpr (!ALIGNED) {
#pragma unroll
                for (int i = 0; i < HI; ++i) a = fminf(a, fminf(hv[i], tv[i]));
            }
        }
        m[0] = up ? a : -a;
    }
    group_max<GC, 1>(m, nullptr);
    float nm = -((up ? m[0] : -m[0]) * c);  // -max_j (c * x_j)
    if (!(fabsf(nm) <= 3.0e38f)) nm = 0.f;  // empty row (L = 0)

    // ---- SM-4: e_j = 2^(c x_j - m), once (sentinel -> +0.0); s = sum e_j
    // (pairs of keys through FFMA2 / FADD2: two running sums, one per lane of
    // the pair, added at the end)
    float s[1] = {0.f};
    {
        const F2 c2 = f2_make(c, c), nm2 = f2_make(nm, nm);
        F2 s2 = f2_make(0.f, 0.f);
#pragma unroll
        for (int k = 0; k < NVC; ++k) {
            // a slot past the row (dead_slots) is summed with weight 0
            const float w = (!dead_slots || q + k * GC < nv) ? 1.f : 0.f;
            const F2 w2 = f2_make(w, w);
#pragma unroll
            for (int e = 0; e < VE; e += 2) {
                const F2 t = f2_fma(f2_make(v[k][e], v[k][e + 1]), c2, nm2);
                float t0, t1;
                f2_split(t, t0, t1);
                v[k][e] = ex2_approx(t0);
                v[k][e + 1] = ex2_approx(t1);
                if constexpr (FULLROW)
                    s2 = f2_fma(f2_make(v[k][e], v[k][e + 1]), w2, s2);
                else
                    s2 = f2_add(s2, f2_make(v[k][e], v[k][e + 1]));
            }
        }
        float s0, s1;
        f2_split(s2, s0, s1);
        s[0] = s0 + s1;
    }
    if constexpr (!ALIGNED) {
#pragma unroll
        for (int i = 0; i < HI; ++i) {
            hv[i] = ex2_approx(fmaf(hv[i], c, nm));
            tv[i] = ex2_approx(fmaf(tv[i], c, nm));
            s[0] += hv[i] + tv[i];
        }
    }
    group_sum<GC, 1>(s, nullptr);
    // masked keys hold e = +0.0, so y = e * inv is +0.0 there; L = 0 -> inv = 0.
    // For L > 0, s >= 1 (the max key contributes 1) or NaN (NaN keys propagate).
    const float inv = L > 0 ? rcp_approx(s[0]) : 0.f;
    if (!live) return;

    // ---- SM-5: normalise and store every column.  EF (evict_first stores) is
    // chosen at launch only when every row covers whole 128-byte L2 lines: a
    // line shared with the next row (partly written) evicted early costs a
    // partial write-back; measured 6 % slower on odd-pitch C3 rows and 4.5 % on
    // 800-byte rows, +1 % on C4.
#pragma unroll
    for (int k = 0; k < NVC; ++k) {
        const int vi = q + k * GC;
        if (vi < nv) {
            float y[VE];
            const F2 inv2 = f2_make(inv, inv);
#pragma unroll
            for (int e = 0; e < VE; e += 2)
                f2_split(f2_mul(f2_make(v[k][e], v[k][e + 1]), inv2), y[e], y[e + 1]);
            Raw<VB> w;
            Elem<T>::template pack<VB>(y, w);
            st_stream<VB, EF>(p + hd + vi * VE, w);
        }
    }
    if constexpr (NARROW) {
        Raw<VB> z;
#pragma unroll
        for (int i = 0; i < Raw<VB>::W; ++i) z.w[i] = 0u;
        for (int vi = GC * NVC + q; vi < nv; vi += GC) st_stream<VB>(p + hd + vi * VE, z);
    }
    if constexpr (!ALIGNED) {
#pragma unroll
        for (int i = 0; i < HI; ++i) {
            const int jh = q + i * GC, jt = tl0 + q + i * GC;
            if (jh < hd) p[jh] = Elem<T>::from_f(hv[i] * inv);
            if (jt < Sk) p[jt] = Elem<T>::from_f(tv[i] * inv);
        }
    }
}

// One row, load then finish (no prefetch).
template <typename T, int VB, int GC, int NVC, bool ALIGNED, bool NARROW, bool UP,
          bool FULLROW = false>
__device__ __forceinline__ void softmax_row_pass(T* __restrict__ p, bool live, int L, int Sk,
                                                 float c, int q) {
    if (!live) L = 0;
    RowRaw<T, VB, GC, NVC, ALIGNED> r;
    row_load<T, VB, GC, NVC, ALIGNED>(p, L, Sk, q, r);
    row_finish<T, VB, GC, NVC, ALIGNED, NARROW, UP, false, FULLROW>(p, live, L, Sk, c, q, r);
}

}  // namespace tt
