// attention.cu -- NEXT-3: the masked softmax fused into its two
// GEMMs, o = softmax_masked(scale * q k^T) v, on the 5th-generation tensor
// cores (tcgen05.mma, accumulators in TMEM).  The [B, H, S, S] score tensor
// never reaches HBM (PAPER.md l.179-182 for the attention, l.302 for "fusing
// all the kernels between two GEMM kernels").
//
// One CTA = 128 query rows of one (b, h); 4 warps, thread t owns query row t
// (TMEM lane t).  Per tile of BN keys (64 by default):
//   1. K / V tiles arrive in shared memory by cp.async (16-byte chunks written
//      in the SWIZZLE_128B layout UMMA reads); keys >= L_b are zero-filled,
//      never read (masked keys cannot inject NaN into the MMA).
//   2. one thread issues S = Q K^T: 4 x tcgen05.mma M128 N=BN K16 (bf16/f16 in,
//      fp32 out) into TMEM columns [0, BN); tcgen05.commit -> mbarrier.
//   3. every thread tcgen05.ld's its row of S (one wait for all columns), masks
//      keys >= L_b (partial tile only), takes the row max and writes
//      p = 2^(s c - m_ref) (16-bit) into shared memory in the UMMA layout; the
//      row sum l is kept in a register (a row is one thread: no shuffles).
//   4. one thread issues O += P V: BN/16 x tcgen05.mma M128 N64 K16 (V as an
//      MN-major operand) into TMEM columns [BN, BN + 64) -- O never leaves
//      TMEM.  m_ref only moves when a tile's max exceeds it by more than 2^8;
//      then the warp rescales its O rows in TMEM (tcgen05.ld / st), which
//      after the first tiles is rare.
// Finally o = O / l, narrowed, stored row-per-thread.  Head dim D = 64.
// Schedules (ttx_attention_variant): NBUF = 2 (default, with BN = 64: 64 KB of
// shared memory, 3 CTAs per SM) double-buffers K and V and software-pipelines
// the tile loop -- S(t+1) is issued as soon as S(t) has been read out of TMEM,
// so the QK^T MMA runs under softmax(t), and P.V(t) is only waited for when P,
// O or its V buffer is reused.  NBUF = 1 keeps one K and one V buffer and runs
// the steps in order (2 CTAs per SM at BN = 128, 4 at BN = 64).
#include <atomic>
#include <type_traits>

#include "common.cuh"
#include "launch.h"
#include "tcgen05.cuh"

namespace tt {

namespace {

constexpr int kBM = 128, kD = 64, kNT = 128;
constexpr int kTile = kBM * kD * 2;  // 16 KB: 128 rows x 128 B

// tile row r (128 B = 64 x 16-bit), 16-byte chunk c -> swizzled smem offset
__device__ __forceinline__ uint32_t sw_off(int r, int c) {
    return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + ((c ^ (r & 7)) << 4));
}

// rows [row0, row0 + ROWS) of a [S, 64] 16-bit matrix into a swizzled tile;
// rows >= valid are zero-filled without reading global memory
template <typename T, int ROWS = kBM>
__device__ __forceinline__ void load_tile(uint32_t tile, const T* g, int row0, int valid) {
#pragma unroll
    for (int i = 0; i < (ROWS * 8) / kNT; ++i) {
        const int idx = threadIdx.x + i * kNT;
        const int r = idx >> 3, c = idx & 7;
        const bool in = row0 + r < valid;
        const T* src = g + (size_t)(in ? row0 + r : 0) * kD + c * 8;
        cp_async16(tile + sw_off(r, c), src, in ? 16u : 0u);
    }
}

}  // namespace

// BN keys per tile (128 or 64).  A K or V tile is BN rows of 128 B; P is
// 128 x BN 16-bit (BN / 64 SW128 tiles of 16 KB).
//   NBUF = 2, BN = 128: K / V double-buffered, 112 KB smem, 1 CTA per SM;
//   NBUF = 1, BN = 128: 80 KB, 2 CTAs per SM (one CTA's softmax runs while the
//                       other's MMAs and loads are in flight);
//   NBUF = 1, BN = 64:  48 KB and 128 TMEM columns, 4 CTAs per SM;
//   NBUF = 2, BN = 64:  64 KB, 3 CTAs per SM.
// NBUF = 2 runs the software-pipelined schedule (see the loop).
template <int NBUF, int BN>
constexpr size_t attn_smem() {
    return (size_t)kTile + (size_t)2 * NBUF * BN * 128 + (size_t)BN * 256 + 64 + 1024;
}
template <int NBUF, int BN>
constexpr int attn_minb() {
    return BN == 64 ? (NBUF == 1 ? 4 : 3) : (NBUF == 1 ? 2 : 1);
}
template <int BN>
constexpr int attn_tmem_cols() {
    return BN + kD <= 128 ? 128 : 256;
}

// TMA (NBUF = 2 only): Q, K and V arrive by cp.async.bulk.tensor.3d (tensor maps
// over [B*H, S, 64], SWIZZLE_128B) issued by one thread and completing on
// mbarriers, instead of 16-byte cp.async by every thread; V rows of keys >= L
// in the last partial tile are zeroed in shared memory before the P.V MMA.
template <typename T, int NBUF, int BN, bool UP, bool LATE = false, bool TMA = false>
__global__ void __launch_bounds__(kNT, attn_minb<NBUF, BN>())
    attention_tc_kernel(const __grid_constant__ CUtensorMap tq,
                        const __grid_constant__ CUtensorMap tk,
                        const __grid_constant__ CUtensorMap tv, T* __restrict__ out,
                        const T* __restrict__ q, const T* __restrict__ k,
                        const T* __restrict__ v, const int32_t* __restrict__ lengths, int H,
                        int S, float c) {
    PdlScope pdl_;  // griddepcontrol.wait first: no global access before it (PDL)
    constexpr int kKV = BN * 128;  // bytes of one K or V tile
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-aligned carve-up: Q | K[NBUF] | V[NBUF] | P | barriers + TMEM slot
    const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
    unsigned char* sbase = smem_raw + (base - smem_u32(smem_raw));
    const uint32_t sQ = base, sK = base + kTile, sV = base + kTile + NBUF * kKV,
                   sP = base + kTile + 2 * NBUF * kKV;
    // bars: [0] S done, [1] P.V done, [2] Q (+ K0, V0) landed, [3..4] K(b), [5..6] V(b)
    uint64_t* bars = reinterpret_cast<uint64_t*>(sbase + kTile + 2 * NBUF * kKV + BN * 256);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sbase + kTile + 2 * NBUF * kKV + BN * 256 + 56);

    const int qt = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
    const int tid = threadIdx.x, warp = tid >> 5;
    const int L = min(max(__ldg(lengths + b), 0), S);
    const size_t head = ((size_t)b * H + h) * (size_t)S * kD;
    const int row = qt * kBM + tid;  // this thread's query row

    if (L == 0) {  // no valid key: the output rows are zero
        if (row < S) {
            uint4 z = make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int i = 0; i < kD * 2 / 16; ++i)
                reinterpret_cast<uint4*>(out + head + (size_t)row * kD)[i] = z;
        }
        return;
    }

    if (warp == 0) {  // TMEM: S in columns [0,BN), O in [BN,BN+64)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "n"(attn_tmem_cols<BN>())
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    const int nkt = (L + BN - 1) / BN;
    const int bh = b * H + h;
    // TMA: K(t) into buffer t & 1 on bars[3 + (t & 1)], V(t) on bars[5 + (t & 1)]
    auto tma_k = [&](int t) {
        mbar_arrive_expect_tx(&bars[3 + (t & 1)], (uint32_t)kKV);
        tma_load_3d(sK + (t & 1) * kKV, &tk, &bars[3 + (t & 1)], 0, t * BN, bh);
    };
    auto tma_v = [&](int t) {
        mbar_arrive_expect_tx(&bars[5 + (t & 1)], (uint32_t)kKV);
        tma_load_3d(sV + (t & 1) * kKV, &tv, &bars[5 + (t & 1)], 0, t * BN, bh);
    };
    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        if constexpr (TMA) {
            for (int i = 2; i < 7; ++i) mbar_init(&bars[i], 1);
        }
        fence_mbar_init();
        if constexpr (TMA) {
            mbar_arrive_expect_tx(&bars[2], (uint32_t)kTile);
            tma_load_3d(sQ, &tq, &bars[2], 0, qt * kBM, bh);
            tma_k(0);
            tma_v(0);
            if (nkt > 1) tma_k(1);
        }
    }
    if constexpr (!TMA) {
        load_tile<T>(sQ, q + head, qt * kBM, S);
        load_tile<T, BN>(sK, k + head, 0, L);
        load_tile<T, BN>(sV, v + head, 0, L);
        cp_async_commit();
        if (NBUF == 2 && nkt > 1) load_tile<T, BN>(sK + kKV, k + head, BN, L);  // K(1)
        cp_async_commit();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    const uint32_t t_s = tmem + lane_off, t_o = tmem + BN + lane_off;

    constexpr int kFmt = sizeof(T) == 2 && std::is_same<T, __nv_bfloat16>::value ? 1 : 0;
    constexpr uint32_t idesc_s = f16_idesc(kFmt, 0, kBM, BN);
    constexpr uint32_t idesc_o = f16_idesc(kFmt, 1, kBM, kD);
    // O and l are kept relative to a reference max m_ref (log2 units, scaled);
    // m_ref only moves -- and O is rescaled in TMEM -- when a tile's max
    // exceeds it by more than kRescale, so p = 2^(s c - m_ref) <= 2^kRescale.
    constexpr float kRescale = 8.f;
    constexpr int NCH = BN / 32;
    const float sent = UP ? -INFINITY : INFINITY;
    float m_ref = -INFINITY, l_run = 0.f;
    uint32_t ph_s = 0, ph_o = 0;
    unsigned char* prow = sbase + (sP - base);

    auto issue_s = [&](int kt) {  // S = Q K(kt)^T (K-major A and B, 4 K-steps of 16)
        if (tid == 0) {
            const uint32_t kbase = sK + (NBUF == 2 ? (kt & 1) : 0) * kKV;
#pragma unroll
            for (int ks = 0; ks < kD / 16; ++ks)
                tc_mma(tmem, sw128_desc(sQ + ks * 32, 16, 1024),
                       sw128_desc(kbase + ks * 32, 16, 1024), idesc_s, ks > 0);
            tc_commit(&bars[0]);
        }
    };
    auto issue_pv = [&](int kt) {  // O += P V(kt) (P K-major; V MN-major, 2048 B per K-step)
        if (tid == 0) {
            const uint32_t vbase = sV + (NBUF == 2 ? (kt & 1) : 0) * kKV;
#pragma unroll
            for (int ks = 0; ks < BN / 16; ++ks)
                tc_mma(tmem + BN, sw128_desc(sP + (ks >> 2) * kTile + (ks & 3) * 32, 16, 1024),
                       sw128_desc(vbase + ks * 2048, 16384, 1024), idesc_o, (kt > 0 || ks > 0));
            tc_commit(&bars[1]);
        }
    };
    // this thread's row of S: BN / 32 TMEM loads in flight, one wait
    auto load_s = [&](float (&sv)[BN]) {
        uint32_t r[NCH][32];
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) tc_ld32_nowait(t_s + ch * 32, r[ch]);
        tc_wait_ld();
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
            for (int e = 0; e < 32; ++e) sv[ch * 32 + e] = __uint_as_float(r[ch][e]);
    };
    // online softmax of tile kt from registers: mask (partial tile only), max,
    // conditional O rescale (the previous P.V must have completed), then
    // p = 2^(s c - m_ref) -> P in shared memory, row sum -> l
    // wait_pv: called before O or P is touched (LATE: P.V(kt-1) is waited for
    // here, after the exponentials, instead of before the softmax)
    auto softmax_tile = [&](float (&sv)[BN], int kt, auto&& wait_pv) {
        const int key0 = kt * BN;
        if (key0 + BN > L) {
#pragma unroll
            for (int e = 0; e < BN; ++e) sv[e] = key0 + e < L ? sv[e] : sent;
        }
        // row max over four independent chains (a 16-deep FMNMX3 dependency
        // instead of 32: -1 % on every BERT shape)
        float m4[4] = {sent, sent, sent, sent};
#pragma unroll
        for (int e = 0; e < BN; ++e) m4[e & 3] = UP ? fmaxf(m4[e & 3], sv[e]) : fminf(m4[e & 3], sv[e]);
        const float mx = UP ? fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]))
                            : fminf(fminf(m4[0], m4[1]), fminf(m4[2], m4[3]));
        const float m_tile = mx * c;
        if (kt == 0) {
            m_ref = m_tile;  // nothing accumulated yet
        } else if (__any_sync(0xffffffffu, m_tile > m_ref + kRescale)) {
            wait_pv();
            const float m_new = fmaxf(m_ref, m_tile);
            const float alpha = ex2_approx(m_ref - m_new);
            l_run *= alpha;
            m_ref = m_new;
#pragma unroll
            for (int ch = 0; ch < kD / 32; ++ch) {
                float ov[32];
                tc_ld32(t_o + ch * 32, ov);
#pragma unroll
                for (int e = 0; e < 32; ++e) ov[e] *= alpha;
                tc_st32(t_o + ch * 32, ov);
            }
        }
        const F2 c2 = f2_make(c, c), nm2 = f2_make(-m_ref, -m_ref);
        F2 ps2 = f2_make(0.f, 0.f);
        if constexpr (LATE) {
            // every exponential first (in place), then wait for P.V(kt-1), then P
#pragma unroll
            for (int e = 0; e < BN; e += 2) {
                float t0, t1;
                f2_split(f2_fma(f2_make(sv[e], sv[e + 1]), c2, nm2), t0, t1);
                sv[e] = ex2_approx(t0);
                sv[e + 1] = ex2_approx(t1);
                ps2 = f2_add(ps2, f2_make(sv[e], sv[e + 1]));
            }
            wait_pv();
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    Raw<16> w;
                    Elem<T>::template pack<16>(sv + ch * 32 + 8 * j, w);
                    const uint32_t off =
                        (uint32_t)(ch >> 1) * kTile + sw_off(tid, (ch & 1) * 4 + j);
                    *reinterpret_cast<uint4*>(prow + off) =
                        make_uint4(w.w[0], w.w[1], w.w[2], w.w[3]);
                }
            float a0, a1;
            f2_split(ps2, a0, a1);
            l_run += a0 + a1;
            return;
        }
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
            float pv[32];
#pragma unroll
            for (int e = 0; e < 32; e += 2) {
                float t0, t1;
                f2_split(f2_fma(f2_make(sv[ch * 32 + e], sv[ch * 32 + e + 1]), c2, nm2), t0, t1);
                pv[e] = ex2_approx(t0);
                pv[e + 1] = ex2_approx(t1);
                ps2 = f2_add(ps2, f2_make(pv[e], pv[e + 1]));
            }
            // keys ch*32 .. ch*32+31 -> P half (ch / 2), 16-byte chunks (ch % 2) * 4 + j
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                Raw<16> w;
                Elem<T>::template pack<16>(pv + 8 * j, w);
                const uint32_t off = (uint32_t)(ch >> 1) * kTile + sw_off(tid, (ch & 1) * 4 + j);
                *reinterpret_cast<uint4*>(prow + off) = make_uint4(w.w[0], w.w[1], w.w[2], w.w[3]);
            }
        }
        float a0, a1;
        f2_split(ps2, a0, a1);
        l_run += a0 + a1;
    };
    auto sync_for_mma = [&]() {  // generic-proxy smem writes (cp.async, P) -> tensor core
        fence_proxy_async_smem();
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
    };

    if constexpr (NBUF == 1) {
        // One K and one V buffer: K(kt+1) streams in during softmax(kt), V(kt+1)
        // during the next S MMA.  cp.async groups in flight at the top of an
        // iteration: K(kt), V(kt) -- wait for K only.
        for (int kt = 0; kt < nkt; ++kt) {
            cp_async_wait<1>();
            sync_for_mma();
            issue_s(kt);
            mbar_wait_bounded(&bars[0], ph_s);
            ph_s ^= 1;
            tc_fence_after();
            if (kt + 1 < nkt) {  // K consumed: stream the next K tile in now
                load_tile<T, BN>(sK, k + head, (kt + 1) * BN, L);
                cp_async_commit();
            }
            float sv[BN];
            load_s(sv);
            softmax_tile(sv, kt, [] {});
            if (kt + 1 < nkt)  // V(kt) (K(kt + 1) may still be in flight)
                cp_async_wait<1>();
            else
                cp_async_wait<0>();
            sync_for_mma();
            issue_pv(kt);
            mbar_wait_bounded(&bars[1], ph_o);
            ph_o ^= 1;
            tc_fence_after();
            if (kt + 1 < nkt) {  // V consumed by the P.V MMA
                load_tile<T, BN>(sV, v + head, (kt + 1) * BN, L);
                cp_async_commit();
            }
        }
    } else {
        // Software-pipelined, K and V double-buffered: S(kt+1) is issued as soon
        // as S(kt) has been read out of TMEM, so it runs under softmax(kt); P.V(kt)
        // runs under the next iteration's S wait and is only waited for when its
        // buffers (P, V, O) are reused.  cp.async commit order: prologue {Q, K0,
        // V0}, {K1}; then per iteration E: {K(kt+2)}, F: {V(kt+1)}.
        if constexpr (TMA) {
            mbar_wait_bounded(&bars[2], 0);  // Q
            mbar_wait_bounded(&bars[3], 0);  // K(0)
        } else {
            cp_async_wait<1>();  // Q, K0, V0
        }
        sync_for_mma();
        issue_s(0);
        for (int kt = 0; kt < nkt; ++kt) {
            mbar_wait_bounded(&bars[0], ph_s);  // A: S(kt)
            ph_s ^= 1;
            tc_fence_after();
            float sv[BN];
            load_s(sv);  // B
            if (kt + 1 < nkt) {  // C, D: K(kt+1) ready and S read by every warp -> S(kt+1)
                if constexpr (TMA) {
                    mbar_wait_bounded(&bars[3 + ((kt + 1) & 1)], (uint32_t)((kt + 1) >> 1) & 1u);
                } else {
                    if (kt == 0)
                        cp_async_wait<0>();
                    else
                        cp_async_wait<1>();
                }
                sync_for_mma();
                issue_s(kt + 1);
            }
            // E: K(kt) buffer is free (S(kt) completed)
            if constexpr (TMA) {
                if (tid == 0 && kt + 2 < nkt) tma_k(kt + 2);
            } else {
                if (kt + 2 < nkt)
                    load_tile<T, BN>(sK + (kt & 1) * kKV, k + head, (kt + 2) * BN, L);
                cp_async_commit();
            }
            // F: P.V(kt-1) done -> P, O and V((kt+1) & 1) are free (LATE: waited
            // for inside the softmax, after the exponentials)
            bool pv_done = kt == 0;
            auto wait_pv = [&]() {
                if (!pv_done) {
                    mbar_wait_bounded(&bars[1], ph_o);
                    ph_o ^= 1;
                    tc_fence_after();
                    pv_done = true;
                }
            };
            auto load_v_next = [&]() {
                if constexpr (TMA) {
                    // (every thread has passed wait_pv: the buffer's last reader,
                    // P.V(kt-1), has completed)
                    if (tid == 0 && kt + 1 < nkt) tma_v(kt + 1);
                } else {
                    if (kt + 1 < nkt)
                        load_tile<T, BN>(sV + ((kt + 1) & 1) * kKV, v + head, (kt + 1) * BN, L);
                    cp_async_commit();
                }
            };
            if constexpr (!LATE) {
                wait_pv();
                load_v_next();
            }
            softmax_tile(sv, kt, wait_pv);
            if constexpr (LATE) {
                wait_pv();
                load_v_next();
            }
            if constexpr (TMA) {  // G: V(kt) landed; keys >= L of a partial last tile -> 0
                mbar_wait_bounded(&bars[5 + (kt & 1)], (uint32_t)(kt >> 1) & 1u);
                const int vrows = L - kt * BN;
                if (vrows < BN) {
                    unsigned char* vp = sbase + (sV + (kt & 1) * kKV - base);
                    for (int idx = vrows * 8 + tid; idx < BN * 8; idx += kNT)
                        *reinterpret_cast<uint4*>(vp + idx * 16) = make_uint4(0, 0, 0, 0);
                }
            } else {
                cp_async_wait<2>();  // G: V(kt) (K(kt+2), V(kt+1) may still be in flight)
            }
            sync_for_mma();
            issue_pv(kt);
        }
        mbar_wait_bounded(&bars[1], ph_o);  // the last P.V
        ph_o ^= 1;
        tc_fence_after();
    }

    // ---- o = O / l, narrowed, one 128-byte row per thread
    {
        uint32_t r[2][32];
        tc_ld32_nowait(t_o, r[0]);
        tc_ld32_nowait(t_o + 32, r[1]);
        tc_wait_ld();
        if (row < S) {
            const float inv = 1.0f / l_run;
            T* orow = out + head + (size_t)row * kD;
#pragma unroll
            for (int j = 0; j < kD / 8; ++j) {
                float y[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) y[e] = __uint_as_float(r[j >> 2][(j & 3) * 8 + e]) * inv;
                Raw<16> w;
                Elem<T>::template pack<16>(y, w);
                reinterpret_cast<uint4*>(orow)[j] = make_uint4(w.w[0], w.w[1], w.w[2], w.w[3]);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "n"(attn_tmem_cols<BN>())
                     : "memory");
    }
}


#ifdef TT_TUNING  // measured slower than the default: tuning build only
// ----------------------------------------------------------------------------
// Warp-specialised variant (ttx_attention_variant 5): no CTA-wide barrier in
// the tile loop.  6 warps, 128 query rows, 64-key tiles:
//   warps 0-3  softmax: thread t owns query row t (TMEM lane t);
//   warp  4    producer: cp.async of Q, K(t), V(t) into 2-stage rings;
//   warp  5    MMA issuer (one lane) and TMEM owner.
// TMEM: S double-buffered in columns [0, 64) and [64, 128), O in [128, 192).
// Shared: Q 16 KB | K 2 x 8 KB | V 2 x 8 KB | P 2 x 16 KB | mbarriers.
// Hand-offs are mbarriers, slot i = tile & 1, phase = (tile >> 1) & 1:
//   kfull/vfull  producer -> MMA (cp.async complete + proxy fence)
//   sfull        MMA commit after S(t): S ready, and K slot free for the producer
//   sfree        4 softmax warps -> MMA: S(t) read out of TMEM
//   pfull        4 softmax warps -> MMA: P(t) in shared memory (and any O rescale done)
//   pvdone       MMA commit after P.V(t): P and V slots free, O updated
// The MMA lane issues S(t+1) before waiting for P(t), so QK^T of the next tile
// runs under the softmax of this one; softmax(t) waits for P.V(t-1) only when
// it must rescale O (rare) and for P.V(t-2) before reusing its P buffer.
// ----------------------------------------------------------------------------
constexpr int kWsThreads = 192;
constexpr size_t kWsSmem = (size_t)kTile + 4 * 8192 + 2 * kTile + 16 * 8 + 16 + 1024;

// rows [row0, row0 + ROWS) of a [S, 64] 16-bit matrix by one warp
template <typename T, int ROWS>
__device__ __forceinline__ void load_tile_warp(uint32_t tile, const T* g, int row0, int valid,
                                               int lane) {
#pragma unroll
    for (int i = 0; i < (ROWS * 8) / 32; ++i) {
        const int idx = lane + i * 32;
        const int r = idx >> 3, c = idx & 7;
        const bool in = row0 + r < valid;
        const T* src = g + (size_t)(in ? row0 + r : 0) * kD + c * 8;
        cp_async16(tile + sw_off(r, c), src, in ? 16u : 0u);
    }
}

template <typename T, bool UP>
__global__ void __launch_bounds__(kWsThreads, 2)
    attention_ws_kernel(T* __restrict__ out, const T* __restrict__ q, const T* __restrict__ k,
                        const T* __restrict__ v, const int32_t* __restrict__ lengths, int H, int S,
                        float c) {
    PdlScope pdl_;  // griddepcontrol.wait first: no global access before it (PDL)
    constexpr int BN = 64;
    constexpr int kKV = BN * 128;  // 8 KB
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
    unsigned char* sbase = smem_raw + (base - smem_u32(smem_raw));
    const uint32_t sQ = base, sK = base + kTile, sV = sK + 2 * kKV, sP = sV + 2 * kKV;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sbase + kTile + 4 * kKV + 2 * kTile);
    uint64_t* kfull = bars;       // [2]
    uint64_t* vfull = bars + 2;   // [2]
    uint64_t* sfull = bars + 4;   // [2]
    uint64_t* sfree = bars + 6;   // [2]
    uint64_t* pfull = bars + 8;   // [2]
    uint64_t* pvdone = bars + 10; // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);

    const int qt = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int L = min(max(__ldg(lengths + b), 0), S);
    const size_t head = ((size_t)b * H + h) * (size_t)S * kD;

    if (L == 0) {  // no valid key: the output rows are zero
        const int row = qt * kBM + tid;
        if (tid < kBM && row < S) {
            uint4 z = make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int i = 0; i < kD * 2 / 16; ++i)
                reinterpret_cast<uint4*>(out + head + (size_t)row * kD)[i] = z;
        }
        return;
    }
    if (warp == 5) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
                         smem_u32(tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        for (int i = 0; i < 4; ++i) mbar_init(&bars[i], 1);        // kfull, vfull: producer lane 0
        for (int i = 4; i < 6; ++i) mbar_init(&bars[i], 1);        // sfull: MMA commit
        for (int i = 6; i < 10; ++i) mbar_init(&bars[i], 4);       // sfree, pfull: 4 softmax warps
        for (int i = 10; i < 12; ++i) mbar_init(&bars[i], 1);      // pvdone: MMA commit
        fence_mbar_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int nkt = (L + BN - 1) / BN;
    constexpr int kFmt = sizeof(T) == 2 && std::is_same<T, __nv_bfloat16>::value ? 1 : 0;

    if (warp == 4) {
        // ---------------- producer
        for (int t = 0; t < nkt; ++t) {
            const int s = t & 1;
            if (t >= 2) mbar_wait_bounded(&sfull[s], ((t - 2) >> 1) & 1);  // S(t-2): K slot free
            if (t == 0) load_tile_warp<T, kBM>(sQ, q + head, qt * kBM, S, lane);
            load_tile_warp<T, BN>(sK + s * kKV, k + head, t * BN, L, lane);
            cp_async_commit();
            if (t >= 2) mbar_wait_bounded(&pvdone[s], ((t - 2) >> 1) & 1);  // P.V(t-2): V slot free
            load_tile_warp<T, BN>(sV + s * kKV, v + head, t * BN, L, lane);
            cp_async_commit();
            cp_async_wait<1>();  // Q, K(t)
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&kfull[s]);
            cp_async_wait<0>();  // V(t)
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&vfull[s]);
        }
    } else if (warp == 5) {
        // ---------------- MMA issuer
        if (lane == 0) {
            constexpr uint32_t idesc_s = f16_idesc(kFmt, 0, kBM, BN);
            constexpr uint32_t idesc_o = f16_idesc(kFmt, 1, kBM, kD);
            auto issue_pv = [&](int j) {
                const int s = j & 1;
                mbar_wait_bounded(&pfull[s], (j >> 1) & 1);
                mbar_wait_bounded(&vfull[s], (j >> 1) & 1);
                tc_fence_after();
                const uint32_t pb = sP + s * kTile, vb = sV + s * kKV;
#pragma unroll
                for (int ks = 0; ks < BN / 16; ++ks)
                    tc_mma(tmem + 128, sw128_desc(pb + ks * 32, 16, 1024),
                           sw128_desc(vb + ks * 2048, 16384, 1024), idesc_o, (j > 0 || ks > 0));
                tc_commit(&pvdone[s]);
            };
            for (int t = 0; t < nkt; ++t) {
                const int s = t & 1;
                mbar_wait_bounded(&kfull[s], (t >> 1) & 1);
                if (t >= 2) mbar_wait_bounded(&sfree[s], ((t - 2) >> 1) & 1);
                tc_fence_after();
                const uint32_t kb = sK + s * kKV;
#pragma unroll
                for (int ks = 0; ks < kD / 16; ++ks)
                    tc_mma(tmem + s * BN, sw128_desc(sQ + ks * 32, 16, 1024),
                           sw128_desc(kb + ks * 32, 16, 1024), idesc_s, ks > 0);
                tc_commit(&sfull[s]);
                if (t >= 1) issue_pv(t - 1);
            }
            issue_pv(nkt - 1);
        }
        __syncwarp();
    } else {
        // ---------------- softmax warps: thread tid = query row tid
        const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
        const uint32_t t_o = tmem + 128 + lane_off;
        constexpr float kRescale = 8.f;
        const float sent = UP ? -INFINITY : INFINITY;
        float m_ref = -INFINITY, l_run = 0.f;
        unsigned char* pbase = sbase + (sP - base);
        for (int t = 0; t < nkt; ++t) {
            const int s = t & 1;
            mbar_wait_bounded(&sfull[s], (t >> 1) & 1);
            tc_fence_after();
            float sv[BN];
            {
                uint32_t r[2][32];
                tc_ld32_nowait(tmem + s * BN + lane_off, r[0]);
                tc_ld32_nowait(tmem + s * BN + 32 + lane_off, r[1]);
                tc_wait_ld();
#pragma unroll
                for (int ch = 0; ch < 2; ++ch)
#pragma unroll
                    for (int e = 0; e < 32; ++e) sv[ch * 32 + e] = __uint_as_float(r[ch][e]);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&sfree[s]);
            const int key0 = t * BN;
            if (key0 + BN > L) {
#pragma unroll
                for (int e = 0; e < BN; ++e) sv[e] = key0 + e < L ? sv[e] : sent;
            }
            float mx = sent;
#pragma unroll
            for (int e = 0; e < BN; ++e) mx = UP ? fmaxf(mx, sv[e]) : fminf(mx, sv[e]);
            const float m_tile = mx * c;
            if (t == 0) {
                m_ref = m_tile;
            } else if (__any_sync(0xffffffffu, m_tile > m_ref + kRescale)) {
                // O must hold P.V(t-1) before it is rescaled
                mbar_wait_bounded(&pvdone[(t - 1) & 1], ((t - 1) >> 1) & 1);
                tc_fence_after();
                const float m_new = fmaxf(m_ref, m_tile);
                const float alpha = ex2_approx(m_ref - m_new);
                l_run *= alpha;
                m_ref = m_new;
#pragma unroll
                for (int ch = 0; ch < kD / 32; ++ch) {
                    float ov[32];
                    tc_ld32(t_o + ch * 32, ov);
#pragma unroll
                    for (int e = 0; e < 32; ++e) ov[e] *= alpha;
                    tc_st32(t_o + ch * 32, ov);
                }
            }
            // P buffer s is free once P.V(t-2) has completed
            if (t >= 2) mbar_wait_bounded(&pvdone[s], ((t - 2) >> 1) & 1);
            const F2 c2 = f2_make(c, c), nm2 = f2_make(-m_ref, -m_ref);
            F2 ps2 = f2_make(0.f, 0.f);
            unsigned char* prow = pbase + s * kTile;
#pragma unroll
            for (int ch = 0; ch < 2; ++ch) {
                float pv[32];
#pragma unroll
                for (int e = 0; e < 32; e += 2) {
                    float t0, t1;
                    f2_split(f2_fma(f2_make(sv[ch * 32 + e], sv[ch * 32 + e + 1]), c2, nm2), t0,
                             t1);
                    pv[e] = ex2_approx(t0);
                    pv[e + 1] = ex2_approx(t1);
                    ps2 = f2_add(ps2, f2_make(pv[e], pv[e + 1]));
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    Raw<16> w;
                    Elem<T>::template pack<16>(pv + 8 * j, w);
                    *reinterpret_cast<uint4*>(prow + sw_off(tid, ch * 4 + j)) =
                        make_uint4(w.w[0], w.w[1], w.w[2], w.w[3]);
                }
            }
            float a0, a1;
            f2_split(ps2, a0, a1);
            l_run += a0 + a1;
            fence_proxy_async_smem();  // P (generic proxy) -> tensor core (async proxy)
            tc_fence_before();         // and any O rescale (tcgen05.st)
            __syncwarp();
            if (lane == 0) mbar_arrive(&pfull[s]);
        }
        // ---- o = O / l after the last P.V
        mbar_wait_bounded(&pvdone[(nkt - 1) & 1], ((nkt - 1) >> 1) & 1);
        tc_fence_after();
        uint32_t r[2][32];
        tc_ld32_nowait(t_o, r[0]);
        tc_ld32_nowait(t_o + 32, r[1]);
        tc_wait_ld();
        const int row = qt * kBM + tid;
        if (row < S) {
            const float inv = 1.0f / l_run;
            T* orow = out + head + (size_t)row * kD;
#pragma unroll
            for (int j = 0; j < kD / 8; ++j) {
                float y[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) y[e] = __uint_as_float(r[j >> 2][(j & 3) * 8 + e]) * inv;
                Raw<16> w;
                Elem<T>::template pack<16>(y, w);
                reinterpret_cast<uint4*>(orow)[j] = make_uint4(w.w[0], w.w[1], w.w[2], w.w[3]);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 5) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem)
                     : "memory");
    }
}


// ----------------------------------------------------------------------------
// Split-row variant (ttx_attention_variant 6): the pipelined 64-key schedule of
// variant 4 with TWO threads per query row.  8 warps: warp w reads TMEM lanes
// 32 (w % 4) .. +31 (its rows) and owns key half h = w / 4 of every S tile, O
// columns [32 h, 32 h + 32) and output columns likewise.  The row max is
// exchanged between the two halves through shared memory (double-buffered by
// tile parity) under a 64-thread named barrier per row group; both halves then
// take identical rescale decisions, and their partial row sums are added once
// at the end.  Half the registers per thread (32 S values), twice the warps.
// ----------------------------------------------------------------------------
constexpr int kSpNT = 256;
constexpr size_t kSpSmem = attn_smem<2, 64>() + 4 * 128 * sizeof(float);

template <typename T, int ROWS, int NT>
__device__ __forceinline__ void load_tile_nt(uint32_t tile, const T* g, int row0, int valid) {
#pragma unroll
    for (int i = 0; i < (ROWS * 8) / NT; ++i) {
        const int idx = threadIdx.x + i * NT;
        const int r = idx >> 3, c = idx & 7;
        const bool in = row0 + r < valid;
        const T* src = g + (size_t)(in ? row0 + r : 0) * kD + c * 8;
        cp_async16(tile + sw_off(r, c), src, in ? 16u : 0u);
    }
}

__device__ __forceinline__ void named_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

template <typename T, bool UP, int MINB>
__global__ void __launch_bounds__(kSpNT, MINB)
    attention_split_kernel(T* __restrict__ out, const T* __restrict__ q, const T* __restrict__ k,
                           const T* __restrict__ v, const int32_t* __restrict__ lengths, int H,
                           int S, float c) {
    PdlScope pdl_;  // griddepcontrol.wait first: no global access before it (PDL)
    constexpr int NBUF = 2, BN = 64;
    constexpr int kKV = BN * 128;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
    unsigned char* sbase = smem_raw + (base - smem_u32(smem_raw));
    const uint32_t sQ = base, sK = base + kTile, sV = base + kTile + NBUF * kKV,
                   sP = base + kTile + 2 * NBUF * kKV;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sbase + kTile + 2 * NBUF * kKV + BN * 256);
    uint32_t* tmem_slot =
        reinterpret_cast<uint32_t*>(sbase + kTile + 2 * NBUF * kKV + BN * 256 + 16);
    float* xch = reinterpret_cast<float*>(sbase + kTile + 2 * NBUF * kKV + BN * 256 + 64);
    // xch: [2 parity][2 halves][128 rows] partial maxima; reused at the end for l

    const int qt = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int rg = warp & 3, hf = warp >> 2;
    const int r = rg * 32 + lane;  // query row in the tile (= TMEM lane)
    const int L = min(max(__ldg(lengths + b), 0), S);
    const size_t head = ((size_t)b * H + h) * (size_t)S * kD;
    const int row = qt * kBM + r;

    if (L == 0) {
        if (row < S) {
            uint4 z = make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int i = 0; i < 4; ++i)
                reinterpret_cast<uint4*>(out + head + (size_t)row * kD + hf * 32)[i] = z;
        }
        return;
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
                         smem_u32(tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init();
    }
    const int nkt = (L + BN - 1) / BN;
    load_tile_nt<T, kBM, kSpNT>(sQ, q + head, qt * kBM, S);
    load_tile_nt<T, BN, kSpNT>(sK, k + head, 0, L);
    load_tile_nt<T, BN, kSpNT>(sV, v + head, 0, L);
    cp_async_commit();
    if (nkt > 1) load_tile_nt<T, BN, kSpNT>(sK + kKV, k + head, BN, L);
    cp_async_commit();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t lane_off = (uint32_t)(rg * 32) << 16;
    const uint32_t t_s = tmem + lane_off + hf * 32, t_o = tmem + BN + lane_off + hf * 32;

    constexpr int kFmt = sizeof(T) == 2 && std::is_same<T, __nv_bfloat16>::value ? 1 : 0;
    constexpr uint32_t idesc_s = f16_idesc(kFmt, 0, kBM, BN);
    constexpr uint32_t idesc_o = f16_idesc(kFmt, 1, kBM, kD);
    constexpr float kRescale = 8.f;
    const float sent = UP ? -INFINITY : INFINITY;
    float m_ref = -INFINITY, l_run = 0.f;
    uint32_t ph_s = 0, ph_o = 0;
    unsigned char* prow = sbase + (sP - base);

    auto issue_s = [&](int kt) {
        if (tid == 0) {
            const uint32_t kbase = sK + (kt & 1) * kKV;
#pragma unroll
            for (int ks = 0; ks < kD / 16; ++ks)
                tc_mma(tmem, sw128_desc(sQ + ks * 32, 16, 1024),
                       sw128_desc(kbase + ks * 32, 16, 1024), idesc_s, ks > 0);
            tc_commit(&bars[0]);
        }
    };
    auto issue_pv = [&](int kt) {
        if (tid == 0) {
            const uint32_t vbase = sV + (kt & 1) * kKV;
#pragma unroll
            for (int ks = 0; ks < BN / 16; ++ks)
                tc_mma(tmem + BN, sw128_desc(sP + ks * 32, 16, 1024),
                       sw128_desc(vbase + ks * 2048, 16384, 1024), idesc_o, (kt > 0 || ks > 0));
            tc_commit(&bars[1]);
        }
    };
    auto sync_for_mma = [&]() {
        fence_proxy_async_smem();
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
    };
    auto softmax_half = [&](float (&sv)[32], int kt) {
        const int key0 = kt * BN + hf * 32;
        if (key0 + 32 > L) {
#pragma unroll
            for (int e = 0; e < 32; ++e) sv[e] = key0 + e < L ? sv[e] : sent;
        }
        float mx = sent;
#pragma unroll
        for (int e = 0; e < 32; ++e) mx = UP ? fmaxf(mx, sv[e]) : fminf(mx, sv[e]);
        float* xb = xch + (kt & 1) * 256;
        xb[hf * 128 + r] = mx;
        named_bar(1 + rg, 64);  // warps rg and rg + 4: the two halves of these rows
        const float mo = xb[(hf ^ 1) * 128 + r];
        mx = UP ? fmaxf(mx, mo) : fminf(mx, mo);
        const float m_tile = mx * c;
        if (kt == 0) {
            m_ref = m_tile;
        } else if (__any_sync(0xffffffffu, m_tile > m_ref + kRescale)) {
            const float m_new = fmaxf(m_ref, m_tile);
            const float alpha = ex2_approx(m_ref - m_new);
            l_run *= alpha;
            m_ref = m_new;
            float ov[32];
            tc_ld32(t_o, ov);
#pragma unroll
            for (int e = 0; e < 32; ++e) ov[e] *= alpha;
            tc_st32(t_o, ov);
        }
        const F2 c2 = f2_make(c, c), nm2 = f2_make(-m_ref, -m_ref);
        F2 ps2 = f2_make(0.f, 0.f);
        float pv[32];
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
            float t0, t1;
            f2_split(f2_fma(f2_make(sv[e], sv[e + 1]), c2, nm2), t0, t1);
            pv[e] = ex2_approx(t0);
            pv[e + 1] = ex2_approx(t1);
            ps2 = f2_add(ps2, f2_make(pv[e], pv[e + 1]));
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            Raw<16> w;
            Elem<T>::template pack<16>(pv + 8 * j, w);
            *reinterpret_cast<uint4*>(prow + sw_off(r, hf * 4 + j)) =
                make_uint4(w.w[0], w.w[1], w.w[2], w.w[3]);
        }
        float a0, a1;
        f2_split(ps2, a0, a1);
        l_run += a0 + a1;
    };

    cp_async_wait<1>();
    sync_for_mma();
    issue_s(0);
    for (int kt = 0; kt < nkt; ++kt) {
        mbar_wait_bounded(&bars[0], ph_s);
        ph_s ^= 1;
        tc_fence_after();
        float sv[32];
        tc_ld32(t_s, sv);
        if (kt + 1 < nkt) {
            if (kt == 0)
                cp_async_wait<0>();
            else
                cp_async_wait<1>();
            sync_for_mma();
            issue_s(kt + 1);
        }
        if (kt + 2 < nkt)
            load_tile_nt<T, BN, kSpNT>(sK + (kt & 1) * kKV, k + head, (kt + 2) * BN, L);
        cp_async_commit();
        if (kt > 0) {
            mbar_wait_bounded(&bars[1], ph_o);
            ph_o ^= 1;
            tc_fence_after();
        }
        if (kt + 1 < nkt)
            load_tile_nt<T, BN, kSpNT>(sV + ((kt + 1) & 1) * kKV, v + head, (kt + 1) * BN, L);
        cp_async_commit();
        softmax_half(sv, kt);
        cp_async_wait<2>();
        sync_for_mma();
        issue_pv(kt);
    }
    mbar_wait_bounded(&bars[1], ph_o);
    ph_o ^= 1;
    tc_fence_after();

    // ---- o = O / l: the two halves' partial sums meet in shared memory
    xch[hf * 128 + r] = l_run;  // (the last tile's max exchange has been read: barrier above)
    {
        float ov[32];
        tc_ld32(t_o, ov);
        __syncthreads();
        const float l = xch[r] + xch[128 + r];
        if (row < S) {
            const float inv = 1.0f / l;
            T* orow = out + head + (size_t)row * kD + hf * 32;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                float y[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) y[e] = ov[j * 8 + e] * inv;
                Raw<16> w;
                Elem<T>::template pack<16>(y, w);
                reinterpret_cast<uint4*>(orow)[j] = make_uint4(w.w[0], w.w[1], w.w[2], w.w[3]);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem)
                     : "memory");
    }
}

#endif  // TT_TUNING

namespace {
std::atomic<int> g_attn_nbuf{0};  // 0 = automatic (variant 4)

template <typename T, int NBUF, int BN, bool LATE = false, bool TMA = false>
cudaError_t launch_attn(void* out, const void* q, const void* k, const void* v,
                        const int32_t* lengths, int64_t B, int64_t H, int64_t S, float scale,
                        cudaStream_t st) {
    constexpr size_t smem = attn_smem<NBUF, BN>();
    dim3 grid((unsigned)((S + kBM - 1) / kBM), (unsigned)H, (unsigned)B);
    CUtensorMap mq{}, mk{}, mv{};  // read only by the TMA instantiation
    if constexpr (TMA) {
        constexpr int dt = std::is_same<T, __half>::value ? 1 : 2;
        if (!make_map(&mq, q, dt, B * H, S, kBM) || !make_map(&mk, k, dt, B * H, S, BN) ||
            !make_map(&mv, v, dt, B * H, S, BN))
            return cudaErrorNotSupported;
    }
    // c = scale * log2(e); scale 0 -> a tiny positive c (uniform weights, as the
    // softmax kernels do), so the masked-key sentinel still maps to p = +0
    float c = scale * 1.4426950408889634f;
    if (c == 0.f) c = 1e-30f;
    auto kern = c > 0.f ? attention_tc_kernel<T, NBUF, BN, true, LATE, TMA>
                        : attention_tc_kernel<T, NBUF, BN, false, LATE, TMA>;
    {
        const cudaError_t le_ = launch_k(kern, grid, kNT, smem, st, mq, mk, mv,
            static_cast<T*>(out), static_cast<const T*>(q),
                                  static_cast<const T*>(k), static_cast<const T*>(v), lengths,
                                  (int)H, (int)S, c);
        if (le_ != cudaSuccess) return le_;
    }
    return cudaGetLastError();
}

#ifdef TT_TUNING
template <typename T>
cudaError_t launch_attn_ws(void* out, const void* q, const void* k, const void* v,
                           const int32_t* lengths, int64_t B, int64_t H, int64_t S, float scale,
                           cudaStream_t st) {
    dim3 grid((unsigned)((S + kBM - 1) / kBM), (unsigned)H, (unsigned)B);
    float c = scale * 1.4426950408889634f;
    if (c == 0.f) c = 1e-30f;
    auto kern = c > 0.f ? attention_ws_kernel<T, true> : attention_ws_kernel<T, false>;
    const cudaError_t le_ = launch_k(kern, grid, kWsThreads, kWsSmem, st, static_cast<T*>(out),
                                     static_cast<const T*>(q), static_cast<const T*>(k),
                                     static_cast<const T*>(v), lengths, (int)H, (int)S, c);
    if (le_ != cudaSuccess) return le_;
    return cudaGetLastError();
}

template <typename T, int MINB>
cudaError_t launch_attn_split(void* out, const void* q, const void* k, const void* v,
                              const int32_t* lengths, int64_t B, int64_t H, int64_t S, float scale,
                              cudaStream_t st) {
    dim3 grid((unsigned)((S + kBM - 1) / kBM), (unsigned)H, (unsigned)B);
    float c = scale * 1.4426950408889634f;
    if (c == 0.f) c = 1e-30f;
    auto kern = c > 0.f ? attention_split_kernel<T, true, MINB>
                        : attention_split_kernel<T, false, MINB>;
    const cudaError_t le_ = launch_k(kern, grid, kSpNT, kSpSmem, st, static_cast<T*>(out),
                                     static_cast<const T*>(q), static_cast<const T*>(k),
                                     static_cast<const T*>(v), lengths, (int)H, (int)S, c);
    if (le_ != cudaSuccess) return le_;
    return cudaGetLastError();
}

#endif  // TT_TUNING

}  // namespace
cudaError_t attention_fa_launch(int dtype, int bn, void* out, const void* q, const void* k,
                                const void* v, const int32_t* lengths, int64_t B, int64_t H,
                                int64_t S, float scale, cudaStream_t stream);  // attention_fa.cu
namespace {

template <typename T>
cudaError_t launch_attn_any(void* out, const void* q, const void* k, const void* v,
                            const int32_t* lengths, int64_t B, int64_t H, int64_t S, float scale,
                            cudaStream_t st) {
    // automatic: 64-key tiles, pipelined (fastest on every BERT shape measured,
    // profiles/r01_attn_bench.jsonl)
    switch (g_attn_nbuf.load(std::memory_order_relaxed)) {
#ifdef TT_TUNING
        case 9:
            return attention_fa_launch(std::is_same<T, __half>::value ? 1 : 2, 128, out, q, k, v,
                                       lengths, B, H, S, scale, st);
        case 10:
            return attention_fa_launch(std::is_same<T, __half>::value ? 1 : 2, 64, out, q, k, v,
                                       lengths, B, H, S, scale, st);
        case 1: return launch_attn<T, 1, 128>(out, q, k, v, lengths, B, H, S, scale, st);
        case 2: return launch_attn<T, 2, 128>(out, q, k, v, lengths, B, H, S, scale, st);
        case 3: return launch_attn<T, 1, 64>(out, q, k, v, lengths, B, H, S, scale, st);
        case 4: return launch_attn<T, 2, 64>(out, q, k, v, lengths, B, H, S, scale, st);
        case 5: return launch_attn_ws<T>(out, q, k, v, lengths, B, H, S, scale, st);
        case 6: return launch_attn_split<T, 2>(out, q, k, v, lengths, B, H, S, scale, st);
        case 7: return launch_attn_split<T, 3>(out, q, k, v, lengths, B, H, S, scale, st);
        case 8: return launch_attn<T, 2, 64, true>(out, q, k, v, lengths, B, H, S, scale, st);
#endif
#ifdef TT_TUNING
        case 11: return launch_attn<T, 2, 64, false, true>(out, q, k, v, lengths, B, H, S, scale, st);
#endif
        default: return launch_attn<T, 2, 64>(out, q, k, v, lengths, B, H, S, scale, st);
    }
}
}  // namespace

// Variants compiled into this build: 0 (automatic = the pipelined 64-key
// schedule) and, in the TT_TUNING build, the measured-slower schedules 1 .. 8,
// the warp-specialised TMA / two-Q-tile ones (9, 10; attention_fa.cu) and the
// default schedule fed by TMA instead of cp.async (11: 4 % slower on C4).
bool attention_variant_ok(int v) {
#ifdef TT_TUNING
    return v >= 0 && v <= 11;
#else
    return v == 0;
#endif
}

int attention_variant_count() { return 12; }

bool attention_force_variant(int v) {
    if (!attention_variant_ok(v)) return false;
    g_attn_nbuf.store(v);
    return true;
}

cudaError_t attention_launch(int dtype, void* out, const void* q, const void* k, const void* v,
                             const int32_t* lengths, int64_t B, int64_t H, int64_t S,
                             float scale, cudaStream_t stream) {
    if (dtype == 1)
        return launch_attn_any<__half>(out, q, k, v, lengths, B, H, S, scale, stream);
    return launch_attn_any<__nv_bfloat16>(out, q, k, v, lengths, B, H, S, scale, stream);
}

}  // namespace tt
