// attention_fa.cu -- NEXT-3 fused attention, warp-specialised
// for Blackwell: o = softmax_masked(scale * q k^T) v per (b, h), head dim 64,
// the [B, H, S, S] scores never leave the SM ("fusing all
// the kernels between two GEMM kernels", l.302).
//
// One CTA = two 128-row query tiles of one (b, h) that share every K / V tile;
// 10 warps with fixed roles and mbarrier hand-offs only (no CTA barrier in the
// tile loop):
//   warp 8     TMA producer: Q0, Q1 once, then K(j), V(j) (64 keys each) into a
//              3-stage ring (cp.async.bulk.tensor.3d over [B*H, S, 64] maps,
//              SWIZZLE_128B -- the UMMA K-major layout; rows past S are zeros);
//   warp 9     MMA issuer (one lane) and TMEM owner: S_i = Q_i K(j)^T
//              (tcgen05.mma M128 N64 K16, smem x smem) into one of TWO S buffers
//              per query tile, issued two tiles ahead, and O_i += P_i V(j)
//              (M128 N64 K16, A = P_i read from TMEM, V MN-major in smem);
//   warps 0-3  softmax of query tile 0 (thread t = query row t = TMEM lane t),
//   warps 4-7  softmax of query tile 1: tcgen05.ld of the 64-key S row, mask
//              (last tile only), row max, p = 2^(s c - m_ref) rounded to the
//              storage dtype and written to TMEM (tcgen05.st) as the A operand
//              of the P.V MMA; the row sum is a register.
// S is double-buffered, so S_i(j+1) is already in TMEM when softmax_i(j)
// finishes: a warpgroup only waits for the P.V MMA of its previous tile (before
// it overwrites P_i), and the two warpgroups' exponentials overlap each
// other's MMAs.  O never leaves TMEM; m_ref (and O, l with it) only moves when
// a tile's max exceeds it by more than 2^8, as in attention.cu.  Keys >= L_b:
// masked in the softmax; their V rows in the last partial tile are zeroed in
// shared memory before the P.V MMA (p = 0 times a NaN / Inf in masked V must
// not reach O).
//
// TMEM (512 columns, one CTA per SM): S_i^b at 64 (2 i + b) [0,256) | P_i at
// 256 + 32 i (16-bit pairs) | O_i at 384 + 64 i.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <mutex>
#include <type_traits>

#include "common.cuh"
#include "launch.h"
#include "tcgen05.cuh"

// Measured slower than the default schedule of attention.cu on every BERT
// shape: compiled into the TT_TUNING build only.
#ifdef TT_TUNING
namespace tt {

namespace {

constexpr int kFaBM = 128;                 // query rows per Q tile (TMEM lanes)
constexpr int kFaQT = 2;                   // Q tiles per CTA (softmax warpgroups)
constexpr int kFaD = 64;                   // head dim
constexpr int kFaThreads = 320;            // 8 softmax warps + TMA warp + MMA warp
constexpr int kFaQTile = kFaBM * 128;      // 16 KB: a Q tile (128 rows x 128 B)
constexpr uint32_t kFaTmemCols = 512;
constexpr uint32_t kColP = 256, kColO = 384;  // S below 256 (see the header)

// BN keys per K / V tile: 128 (one S buffer per query tile, K / V ring of 2)
// or 64 (two S buffers per query tile issued two tiles ahead, ring of 3).
template <int BN>
struct FaCfg {
    static constexpr int NB = BN == 64 ? 2 : 1;     // S buffers per query tile
    static constexpr int NS = BN == 64 ? 3 : 2;     // K / V ring stages
    static constexpr int KV = BN * 128;             // bytes of a K or V tile
};
template <int BN>
struct FaBars {
    uint64_t q_full;
    uint64_t k_full[FaCfg<BN>::NS], v_full[FaCfg<BN>::NS], k_empty[FaCfg<BN>::NS],
        v_empty[FaCfg<BN>::NS];
    uint64_t s_full[kFaQT][2], p_full[kFaQT], o_done[kFaQT];
    uint32_t tmem_slot;
};
template <int BN>
constexpr size_t fa_smem() {
    return 1024 + (size_t)kFaQT * kFaQTile + (size_t)2 * FaCfg<BN>::NS * FaCfg<BN>::KV +
           sizeof(FaBars<BN>);
}

// O += A B with A (M x K, K-major, 16-bit pairs per 32-bit column) read from TMEM
__device__ __forceinline__ void tc_mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                          uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// 32 consecutive TMEM columns of this thread's lane <- 32 raw words (no wait)
__device__ __forceinline__ void tc_st32_nowait(uint32_t taddr, const uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
        "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(
            taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
        "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
        "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]),
        "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]),
        "r"(v[29]), "r"(v[30]), "r"(v[31])
        : "memory");
}
__device__ __forceinline__ void tc_wait_st() {
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

template <typename T>
__device__ __forceinline__ uint32_t pack2(float a, float b) {
    Raw<4> w;
    const float f[2] = {a, b};
    Elem<T>::template pack<4>(f, w);
    return w.w[0];
}

}  // namespace

template <typename T, bool UP, int BN>
__global__ void __launch_bounds__(kFaThreads, 1)
    attention_fa_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                        const __grid_constant__ CUtensorMap tv, T* __restrict__ out,
                        const int32_t* __restrict__ lengths, int H, int S, float c) {
    PdlScope pdl_;  // griddepcontrol.wait first: no global access before it (PDL)
    constexpr int kFaBN = BN, NB = FaCfg<BN>::NB, kFaNS = FaCfg<BN>::NS, kFaKV = FaCfg<BN>::KV;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
    unsigned char* sbase = smem_raw + (base - smem_u32(smem_raw));
    const uint32_t sQ = base, sK = base + kFaQT * kFaQTile, sV = sK + kFaNS * kFaKV;
    FaBars<BN>* bar = reinterpret_cast<FaBars<BN>*>(sbase + kFaQT * kFaQTile + 2 * kFaNS * kFaKV);

    const int h = blockIdx.y, b = blockIdx.z;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int L = min(max(__ldg(lengths + b), 0), S);
    const int bh = b * H + h;
    const int q0 = blockIdx.x * (kFaQT * kFaBM);
    const int nq = min(kFaQT, (S - q0 + kFaBM - 1) / kFaBM);  // Q tiles holding rows

    if (L == 0) {  // no valid key: the output rows are zero
        if (warp < 2 * 4) {
            const int row = q0 + tid;
            if (row < S) {
                uint4* o = reinterpret_cast<uint4*>(out + ((size_t)bh * S + row) * kFaD);
#pragma unroll
                for (int i = 0; i < kFaD * 2 / 16; ++i) o[i] = make_uint4(0, 0, 0, 0);
            }
        }
        return;
    }
    const int nkt = (L + kFaBN - 1) / kFaBN;

    if (warp == 9) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&bar->tmem_slot)),
                     "n"(kFaTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        mbar_init(&bar->q_full, 1);
        for (int s = 0; s < kFaNS; ++s) {
            mbar_init(&bar->k_full[s], 1);
            mbar_init(&bar->v_full[s], 1);
            mbar_init(&bar->k_empty[s], 1);
            mbar_init(&bar->v_empty[s], 1);
        }
        for (int i = 0; i < kFaQT; ++i) {
            mbar_init(&bar->s_full[i][0], 1);
            mbar_init(&bar->s_full[i][1], 1);
            mbar_init(&bar->p_full[i], kFaBM);
            mbar_init(&bar->o_done[i], 1);
        }
        fence_mbar_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bar->tmem_slot;
    constexpr int kFmt = std::is_same<T, __nv_bfloat16>::value ? 1 : 0;

    if (warp == 8) {
        // ---------------------------------------------------------------- TMA
        if (lane == 0) {
            mbar_arrive_expect_tx(&bar->q_full, (uint32_t)(nq * kFaQTile));
            for (int i = 0; i < nq; ++i)
                tma_load_3d(sQ + i * kFaQTile, &tq, &bar->q_full, 0, q0 + i * kFaBM, bh);
            for (int j = 0; j < nkt; ++j) {
                const int st = j % kFaNS;
                const uint32_t ph = (uint32_t)(j / kFaNS) & 1u;
                if (j >= kFaNS) mbar_wait_bounded(&bar->k_empty[st], ph ^ 1u);
                mbar_arrive_expect_tx(&bar->k_full[st], kFaKV);
                tma_load_3d(sK + st * kFaKV, &tk, &bar->k_full[st], 0, j * kFaBN, bh);
                if (j >= kFaNS) mbar_wait_bounded(&bar->v_empty[st], ph ^ 1u);
                mbar_arrive_expect_tx(&bar->v_full[st], kFaKV);
                tma_load_3d(sV + st * kFaKV, &tv, &bar->v_full[st], 0, j * kFaBN, bh);
            }
        }
    } else if (warp == 9) {
        // ---------------------------------------------------------------- MMA
        constexpr uint32_t idesc_s = f16_idesc(kFmt, 0, kFaBM, kFaBN);
        constexpr uint32_t idesc_o = f16_idesc(kFmt, 1, kFaBM, kFaD);
        // S_i(j) = Q_i K(j)^T into S buffer j % NB of query tile i (4 K-steps of 16)
        auto issue_s = [&](int j, int i) {
            if (lane == 0) {
                const uint32_t kb = sK + (j % kFaNS) * kFaKV;
#pragma unroll
                for (int ks = 0; ks < kFaD / 16; ++ks)
                    tc_mma(tmem + (NB * i + j % NB) * kFaBN,
                           sw128_desc(sQ + i * kFaQTile + ks * 32, 16, 1024),
                           sw128_desc(kb + ks * 32, 16, 1024), idesc_s, ks > 0);
                tc_commit(&bar->s_full[i][j % NB]);
            }
            __syncwarp();
        };
        auto wait_k = [&](int j) {
            mbar_wait_bounded(&bar->k_full[j % kFaNS], (uint32_t)(j / kFaNS) & 1u);
            tc_fence_after();
        };
        mbar_wait_bounded(&bar->q_full, 0);
        for (int j = 0; j < NB && j < nkt; ++j) {  // every S buffer starts free
            wait_k(j);
            for (int i = 0; i < nq; ++i) issue_s(j, i);
            if (lane == 0) tc_commit(&bar->k_empty[j % kFaNS]);
            __syncwarp();
        }
        for (int j = 0; j < nkt; ++j) {
            const int st = j % kFaNS;
            const uint32_t vb = sV + st * kFaKV;
            mbar_wait_bounded(&bar->v_full[st], (uint32_t)(j / kFaNS) & 1u);
            const int vrows = L - j * kFaBN;
            if (vrows < kFaBN) {
                // last partial tile: zero the V rows of keys >= L (whole 128-byte
                // rows, so the swizzle does not matter), then hand them to the
                // async proxy
                unsigned char* vp = sbase + (vb - base);
                for (int idx = vrows * 8 + lane; idx < kFaBN * 8; idx += 32)
                    *reinterpret_cast<uint4*>(vp + idx * 16) = make_uint4(0, 0, 0, 0);
                fence_proxy_async_smem();
                __syncwarp();
            }
            for (int i = 0; i < nq; ++i) {
                mbar_wait_bounded(&bar->p_full[i], (uint32_t)j & 1u);  // P_i(j) in TMEM
                tc_fence_after();
                if (lane == 0) {
#pragma unroll
                    for (int ks = 0; ks < kFaBN / 16; ++ks)
                        tc_mma_ts(tmem + kColO + i * kFaD, tmem + kColP + i * (kFaBN / 2) + ks * 8,
                                  sw128_desc(vb + ks * 2048, 16384, 1024), idesc_o,
                                  (j > 0 || ks > 0) ? 1u : 0u);
                    tc_commit(&bar->o_done[i]);
                }
                __syncwarp();
                // S_i(j+NB) into the buffer softmax_i has just finished with
                if (j + NB < nkt) {
                    if (i == 0) wait_k(j + NB);
                    issue_s(j + NB, i);
                }
            }
            if (lane == 0) {
                tc_commit(&bar->v_empty[st]);
                if (j + NB < nkt) tc_commit(&bar->k_empty[(j + NB) % kFaNS]);
            }
            __syncwarp();
        }
    } else {
        // ------------------------------------------------------------ softmax
        const int i = warp >> 2;  // query tile of this warpgroup
        if (i < nq) {
            const int r = tid & (kFaBM - 1);  // row within the tile = TMEM lane
            const int row = q0 + i * kFaBM + r;
            const uint32_t lo = (uint32_t)((warp & 3) * 32) << 16;
            const uint32_t t_s = tmem + NB * i * kFaBN + lo;
            const uint32_t t_p = tmem + kColP + i * (kFaBN / 2) + lo;
            const uint32_t t_o = tmem + kColO + i * kFaD + lo;
            constexpr float kRescale = 8.f;
            const float sent = UP ? -INFINITY : INFINITY;
            float m_ref = 0.f, l_run = 0.f;
            for (int j = 0; j < nkt; ++j) {
                mbar_wait_bounded(&bar->s_full[i][j % NB], (uint32_t)(j / NB) & 1u);
                tc_fence_after();
                const uint32_t t_sj = t_s + (j % NB) * kFaBN;
                const int key0 = j * kFaBN;
                const bool partial = key0 + kFaBN > L;
                // the S row, 64 columns at a time (BN = 128: read twice -- max, then
                // exponentials -- so it never sits in registers whole)
                auto load64 = [&](int h0, float (&sv)[64]) {
                    uint32_t rr[2][32];
                    tc_ld32_nowait(t_sj + h0 * 64, rr[0]);
                    tc_ld32_nowait(t_sj + h0 * 64 + 32, rr[1]);
                    tc_wait_ld();
#pragma unroll
                    for (int e = 0; e < 64; ++e) sv[e] = __uint_as_float(rr[e >> 5][e & 31]);
                    if (partial) {
#pragma unroll
                        for (int e = 0; e < 64; ++e) sv[e] = key0 + h0 * 64 + e < L ? sv[e] : sent;
                    }
                };
                // row max from 8 independent partial maxima (only 8 warps per SM:
                // a dependent FMNMX chain would not be hidden)
                float sv0[64];
                float mx = sent;
                {
                    float pm[8];
#pragma unroll
                    for (int k8 = 0; k8 < 8; ++k8) pm[k8] = sent;
#pragma unroll
                    for (int h0 = 0; h0 < kFaBN / 64; ++h0) {
                        float sv[64];
                        load64(h0, sv);
#pragma unroll
                        for (int e = 0; e < 64; ++e)
                            pm[e & 7] = UP ? fmaxf(pm[e & 7], sv[e]) : fminf(pm[e & 7], sv[e]);
                        if (kFaBN == 64) {
#pragma unroll
                            for (int e = 0; e < 64; ++e) sv0[e] = sv[e];
                        }
                    }
#pragma unroll
                    for (int k8 = 0; k8 < 8; ++k8) mx = UP ? fmaxf(mx, pm[k8]) : fminf(mx, pm[k8]);
                }
                const float m_tile = mx * c;
                // P_i and O_i are free once P.V_i(j-1) has completed
                if (j > 0) {
                    mbar_wait_bounded(&bar->o_done[i], (uint32_t)(j - 1) & 1u);
                    tc_fence_after();
                }
                if (j == 0) {
                    m_ref = m_tile;  // nothing accumulated yet
                } else if (__any_sync(0xffffffffu, m_tile > m_ref + kRescale)) {
                    const float m_new = fmaxf(m_ref, m_tile);
                    const float alpha = ex2_approx(m_ref - m_new);
                    l_run *= alpha;
                    m_ref = m_new;
#pragma unroll
                    for (int ch = 0; ch < kFaD / 32; ++ch) {
                        float ov[32];
                        tc_ld32(t_o + ch * 32, ov);
#pragma unroll
                        for (int e = 0; e < 32; ++e) ov[e] *= alpha;
                        tc_st32(t_o + ch * 32, ov);
                    }
                }
                // p = 2^(s c - m_ref), rounded to T, two per TMEM column
                const F2 c2 = f2_make(c, c), nm2 = f2_make(-m_ref, -m_ref);
                F2 ps[4] = {f2_make(0.f, 0.f), f2_make(0.f, 0.f), f2_make(0.f, 0.f),
                            f2_make(0.f, 0.f)};
#pragma unroll
                for (int h0 = 0; h0 < kFaBN / 64; ++h0) {
                    float sv[64];
                    if (kFaBN == 64) {
#pragma unroll
                        for (int e = 0; e < 64; ++e) sv[e] = sv0[e];
                    } else {
                        load64(h0, sv);
                    }
                    uint32_t pw[32];
#pragma unroll
                    for (int e = 0; e < 64; e += 2) {
                        float t0, t1;
                        f2_split(f2_fma(f2_make(sv[e], sv[e + 1]), c2, nm2), t0, t1);
                        const float p0 = ex2_approx(t0), p1 = ex2_approx(t1);
                        ps[(e >> 1) & 3] = f2_add(ps[(e >> 1) & 3], f2_make(p0, p1));
                        pw[e / 2] = pack2<T>(p0, p1);
                    }
                    tc_st32_nowait(t_p + h0 * 32, pw);
                }
                const F2 ps2 = f2_add(f2_add(ps[0], ps[1]), f2_add(ps[2], ps[3]));
                tc_wait_st();
                tc_fence_before();
                mbar_arrive(&bar->p_full[i]);
                float a0, a1;
                f2_split(ps2, a0, a1);
                l_run += a0 + a1;
            }
            // ---- o = O / l after the last P.V, narrowed, one 128-byte row per thread
            mbar_wait_bounded(&bar->o_done[i], (uint32_t)(nkt - 1) & 1u);
            tc_fence_after();
            uint32_t ro[2][32];
            tc_ld32_nowait(t_o, ro[0]);
            tc_ld32_nowait(t_o + 32, ro[1]);
            tc_wait_ld();
            if (row < S) {
                const float inv = 1.0f / l_run;
                T* orow = out + ((size_t)bh * S + row) * kFaD;
#pragma unroll
                for (int jj = 0; jj < kFaD / 8; ++jj) {
                    float y[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e)
                        y[e] = __uint_as_float(ro[jj >> 2][(jj & 3) * 8 + e]) * inv;
                    Raw<16> w;
                    Elem<T>::template pack<16>(y, w);
                    reinterpret_cast<uint4*>(orow)[jj] = make_uint4(w.w[0], w.w[1], w.w[2], w.w[3]);
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 9) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "n"(kFaTmemCols)
                     : "memory");
    }
}

namespace {

template <typename T, int BN>
cudaError_t launch_fa(int dtype, void* out, const void* q, const void* k, const void* v,
                      const int32_t* lengths, int64_t B, int64_t H, int64_t S, float scale,
                      cudaStream_t st) {
    CUtensorMap mq, mk, mv;
    if (!make_map(&mq, q, dtype, B * H, S, kFaBM) || !make_map(&mk, k, dtype, B * H, S, BN) ||
        !make_map(&mv, v, dtype, B * H, S, BN))
        return cudaErrorNotSupported;
    dim3 grid((unsigned)((S + kFaQT * kFaBM - 1) / (kFaQT * kFaBM)), (unsigned)H, (unsigned)B);
    float c = scale * 1.4426950408889634f;
    if (c == 0.f) c = 1e-30f;  // uniform weights; the masked-key sentinel still maps to p = 0
    auto kern = c > 0.f ? attention_fa_kernel<T, true, BN> : attention_fa_kernel<T, false, BN>;
    const cudaError_t le = launch_k(kern, grid, kFaThreads, fa_smem<BN>(), st, mq, mk, mv,
                                    static_cast<T*>(out), lengths, (int)H, (int)S, c);
    if (le != cudaSuccess) return le;
    return cudaGetLastError();
}

}  // namespace

cudaError_t attention_fa_launch(int dtype, int bn, void* out, const void* q, const void* k,
                                const void* v, const int32_t* lengths, int64_t B, int64_t H,
                                int64_t S, float scale, cudaStream_t stream) {
    if (bn == 64) {
        if (dtype == 1)
            return launch_fa<__half, 64>(dtype, out, q, k, v, lengths, B, H, S, scale, stream);
        return launch_fa<__nv_bfloat16, 64>(dtype, out, q, k, v, lengths, B, H, S, scale, stream);
    }
    if (dtype == 1)
        return launch_fa<__half, 128>(dtype, out, q, k, v, lengths, B, H, S, scale, stream);
    return launch_fa<__nv_bfloat16, 128>(dtype, out, q, k, v, lengths, B, H, S, scale, stream);
}

}  // namespace tt
#endif  // TT_TUNING
