// softmax.cu -- in-place masked attention softmax over [B, H, Sq, Sk]
// (TurboTransformers' ApplyMaskAndSoftmax; batch reduction
// "Softmax calculates summation and maximum", §4.1.2 l.316).
//
// One group of G threads owns one row:
//   SM-1  b = row / (H*Sq);  L = clamp(lengths[b], 0, Sk)
//   SM-2  vector-load the valid prefix j < L only (masked bytes never read),
//         t_j = x_j * (scale * log2 e) in fp32
//   SM-3  m = max t_j   (per-lane max, then CREDUX / butterfly / CTA merge)
//   SM-4  e_j = 2^(t_j - m) computed ONCE and kept in registers; s = sum e_j
//   SM-5  y_j = e_j / s for j < L, +0.0 for L <= j < Sk; RNE narrow; vector store
// Every element is read at most once and written exactly once: the row lives
// in registers between the load and the store, so no smem staging or online
// (m, s) rescaling is needed up to one CTA's capacity (16 384 keys); longer
// rows (up to TT_MAX_SOFTMAX_COLS) are split over a thread-block cluster that
// merges its CTAs' (max, sum) pairs through distributed shared memory.
//
// Rows of any length: a row starts at an arbitrary element offset, so each row
// is split into an unaligned head (< VE elements, scalar), an aligned body of
// VB-byte vectors and a tail (< VE elements, scalar).
#include <algorithm>
#include <atomic>
#include <cstring>

#include "common.cuh"
#include "launch.h"
#include "softmax_row.cuh"
#include "softmax_kernels.cuh"

namespace tt {

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

// Ring depth: about 4 KB of rows in flight per warp, 2..8 slots.
int tma_depth(int slot_bytes) { return max(2, min(8, 4096 / slot_bytes + 1)); }

template <typename T, int NV, int NW>
cudaError_t launch_softmax_tma(void* scores, const int32_t* lengths, int64_t nrows, int64_t rpb,
                               int Sk, float scale, cudaStream_t st) {
    auto kern = softmax_tma_kernel<T, NV, NW>;
    const int slot_bytes = ((Sk * (int)sizeof(T) + 32) + 127) & ~127;
    const int D = tma_depth(slot_bytes);
    const size_t smem = (size_t)((NW * D * 8 + 127) & ~127) + (size_t)NW * D * slot_bytes;
    cudaError_t e = smem_optin(reinterpret_cast<const void*>(kern), smem);
    if (e != cudaSuccess) return e;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NW * 32, smem);
    if (e != cudaSuccess) return e;
    occ = max(occ, 1);
    const int64_t need = (nrows + NW - 1) / NW;
    const int64_t cap = (int64_t)sm_count() * occ;
    const int64_t grid = need < cap ? need : cap;
    {
        const cudaError_t le_ = launch_k(kern, (unsigned)grid, NW * 32, smem, st,
            static_cast<T*>(scores), lengths, nrows, rpb, Sk,
                                                scale * kLog2e, D, slot_bytes);
        if (le_ != cudaSuccess) return le_;
    }
    return cudaGetLastError();
}

}  // namespace

// ----------------------------------------------------------------------------
// Tier table.  Selection is by (dtype, Sk) only; per-row lengths only shorten
// the reads.  See DESIGN.md §5 for the choice of each entry.
// ----------------------------------------------------------------------------
namespace {

template <typename T, int VB, int G, int NV, int R, int NT, int MINB>
cudaError_t launch_softmax(void* scores, const int32_t* lengths, int64_t nrows, int64_t rpb,
                           int Sk, float scale, cudaStream_t st) {
    constexpr int GPB = NT / G;
    const int64_t rows_per_cta = (int64_t)GPB * R;
    const int64_t grid = (nrows + rows_per_cta - 1) / rows_per_cta;
    if (grid > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
    {
        const cudaError_t le_ = launch_k(softmax_rows_kernel<T, VB, G, NV, R, NT, MINB>, (unsigned)grid, NT, 0, st,
        static_cast<T*>(scores), lengths, nrows, rpb, Sk, scale * kLog2e);
        if (le_ != cudaSuccess) return le_;
    }
    return cudaGetLastError();
}


// Unaligned rows (scalar head / tail code) need a few more registers: the
// instantiations that ptxas would spill at the tier's cap run one CTA per SM
// fewer (probed for every product tier, tools/probe/probe_sm.cu).
template <typename T, int VB, int G, int NV, int MINB>
constexpr int sm_minb_unaligned() {
    constexpr bool f32 = sizeof(T) == 4;
    if constexpr ((f32 && VB == 32 && G == 32 && NV == 3 && MINB >= 5) ||
                  (!f32 && VB == 32 && G == 16 && NV == 1 && MINB >= 6) ||
                  (!f32 && VB == 32 && G == 8 && NV == 3 && MINB >= 3))
        return MINB - 1;
    return MINB;
}

template <typename T, int VB, int G, int NV, int NT, int MINB, int RPG, bool PF = false>
cudaError_t launch_softmax_warp(void* scores, const int32_t* lengths, int64_t nrows, int64_t rpb,
                                int Sk, float scale, cudaStream_t st) {
    constexpr int GPB = NT / G;
    if (nrows >= (int64_t)0xffffffffLL || rpb >= (int64_t)0x7fffffffLL)  // 64-bit indices
        return launch_softmax<T, VB, G, NV, 1, NT, 1>(scores, lengths, nrows, rpb, Sk, scale, st);
    const bool aligned = (reinterpret_cast<uintptr_t>(scores) % VB) == 0 &&
                         ((int64_t)Sk * (int64_t)sizeof(T)) % VB == 0;
    // rows made of whole 128-byte L2 lines: evict_first stores (see row_finish)
    const bool lines = aligned && (reinterpret_cast<uintptr_t>(scores) % 128) == 0 &&
                       ((int64_t)Sk * (int64_t)sizeof(T)) % 128 == 0;
    const int kv = lines ? 2 : aligned ? 1 : 0;
    // (evict_first stores compiled for every tier but the 16-bit G8 x NV5 one, where the
    // extra policy register made ptxas spill; there whole-line rows store plainly)
    constexpr bool kEF = !(sizeof(T) == 2 && G == 8 && NV == 5);
    auto kern = lines     ? softmax_warp_kernel<T, VB, G, NV, NT, MINB, true, PF, kEF>
                : aligned ? softmax_warp_kernel<T, VB, G, NV, NT, MINB, true, PF, false>
                          : softmax_warp_kernel<T, VB, G, NV, NT,
                                                sm_minb_unaligned<T, VB, G, NV, MINB>(), false, PF,
                                                false>;
    // RPG > 0: fixed rows per group; RPG = 0: one persistent wave (rows spread
    // evenly over SMs x resident CTAs).
    int rpg = RPG;
    static std::atomic<int> occ_cache[3] = {{0}, {0}, {0}};
    int occ = occ_cache[kv].load(std::memory_order_relaxed);
    if (!occ) {
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, 0);
        if (e != cudaSuccess) return e;
        occ = occ > 0 ? occ : 1;
        occ_cache[kv].store(occ);
    }
    if (RPG == 0) {
        const int64_t slots = (int64_t)sm_count() * occ * GPB;
        rpg = (int)((nrows + slots - 1) / slots);
    } else {
        // problems that fit a wave are latency-bound: the shortest chain of
        // rows per group that still keeps the call in one wave of resident
        // CTAs (every slot of every SM), rather than RPG rows per group on a
        // part-empty wave (round 1 used 2 CTAs per SM here)
        const int64_t spread = (int64_t)sm_count() * occ * GPB;
        const int64_t need = (nrows + spread - 1) / spread;
        if (need < rpg) rpg = need > 0 ? (int)need : 1;
    }
    // requests of very few rows (far fewer than a CTA's groups): the CTA-tier
    // kernel, which looks each row's length up itself
    if (rpb * 4 < GPB)
        return launch_softmax<T, VB, G, NV, 1, NT, 1>(scores, lengths, nrows, rpb, Sk, scale, st);
    if ((int64_t)GPB * rpg > rpb) rpg = (int)((rpb + GPB - 1) / GPB);
    // cpr CTAs per request, each within one request (softmax_warp_body)
    const int64_t per_cta = (int64_t)GPB * rpg;
    const int64_t cpr = (rpb + per_cta - 1) / per_cta;
    const int64_t grid = (nrows / rpb) * cpr;
    if (grid > 0x7fffffffLL || cpr > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
    // c = 0 (scale 0: uniform softmax) is mapped to a tiny positive c so the
    // masked-key sentinel still exponentiates to exactly +0.0; for finite x,
    // 2^(x * 1e-30 - m * 1e-30) rounds to exactly 1.0f.
    float c = scale * kLog2e;
    if (c == 0.f) c = 1e-30f;
    {
        const cudaError_t le_ = launch_k(kern, (unsigned)grid, NT, 0, st,
            static_cast<T*>(scores), lengths, FastDivU32::make((uint32_t)cpr), (uint32_t)rpb, Sk,
            c, rpg);
        if (le_ != cudaSuccess) return le_;
    }
    return cudaGetLastError();
}

// Rows longer than one CTA's registers hold: a cluster of ceil(Sk / W) CTAs
// per row (softmax_cluster_kernel), W = NT * NV * VE keys per CTA, <= 8 CTAs
// (portable cluster size).
template <typename T, int VB, int NV, int NT>
cudaError_t launch_softmax_cluster(void* scores, const int32_t* lengths, int64_t nrows,
                                   int64_t rpb, int Sk, float scale, cudaStream_t st) {
    constexpr int W = NT * NV * (VB / (int)sizeof(T));
    const int ncl = (Sk + W - 1) / W;
    if (ncl < 1 || ncl > 8) return cudaErrorInvalidConfiguration;
    const int64_t grid = nrows * ncl;
    if (grid > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
    const cudaError_t le = launch_kc(softmax_cluster_kernel<T, VB, NV, NT>, (unsigned)grid, NT, 0,
                                     st, (unsigned)ncl, static_cast<T*>(scores), lengths, rpb, Sk,
                                     scale * kLog2e);
    if (le != cudaSuccess) return le;
    return cudaGetLastError();
}


// Rows of any length: a cluster of C CTAs per row, two passes per key segment
// (softmax_long_kernel).  C = 8, or (KPC > 0) just enough CTAs for ~KPC keys
// each (<= 8).  Measured on B200 (profiles/r02_long/): 256 threads x 4 CTAs/SM
// and ~64 K keys per CTA beat 512 x 2 and 8 CTAs per row by 24-53 % on 131 K -
// 262 K-key rows and tie on 1 M-key rows.
constexpr int kLongMaxCols = 1 << 30;  // = TT_MAX_SOFTMAX_COLS (include/tt.h)
template <typename T, int NT, int MINB, int KPC>
cudaError_t launch_softmax_long(void* scores, const int32_t* lengths, int64_t nrows, int64_t rpb,
                                int Sk, float scale, cudaStream_t st) {
    int64_t C = 8;
    if (KPC > 0) C = std::min<int64_t>(8, std::max<int64_t>(1, ((int64_t)Sk + KPC - 1) / KPC));
    const int64_t W = (((int64_t)Sk + C - 1) / C + 63) / 64 * 64;
    const int64_t grid = nrows * C;
    if (grid > 0x7fffffffLL || W > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
    float c = scale * kLog2e;
    if (c == 0.f) c = 1e-30f;
    const cudaError_t le = launch_kc(softmax_long_kernel<T, NT, 4, MINB>, (unsigned)grid, NT, 0,
                                     st, (unsigned)C, static_cast<T*>(scores), lengths, rpb,
                                     Sk, (int)W, c);
    if (le != cudaSuccess) return le;
    return cudaGetLastError();
}

using SoftmaxFn = cudaError_t (*)(void*, const int32_t*, int64_t, int64_t, int, float,
                                  cudaStream_t);

struct SoftmaxTier {
    int max_cols;  // largest Sk this tier handles for its dtype
    bool automatic;  // eligible for automatic selection (else: tuning candidate only)
    SoftmaxFn fn;
    const char* name;
};

#define TT_SM_TIER(AUTO, T, TN, VB, G, NV, R, NT, MINB)                                    \
    SoftmaxTier {                                                                          \
        (G) * (NV) * ((VB) / (int)sizeof(T)), AUTO,                                        \
            &launch_softmax<T, VB, G, NV, R, NT, MINB>,                                    \
            "softmax_rows<" TN ",V" #VB ",G" #G ",NV" #NV ",R" #R ",T" #NT ",M" #MINB ">" \
    }

#define TT_SM_CLUSTER(AUTO, T, TN, VB, NV, NT)                                             \
    SoftmaxTier {                                                                          \
        8 * (NT) * (NV) * ((VB) / (int)sizeof(T)), AUTO,                                   \
            &launch_softmax_cluster<T, VB, NV, NT>,                                        \
            "softmax_cluster<" TN ",V" #VB ",NV" #NV ",T" #NT ",C8>"                        \
    }

#define TT_SM_LONG(AUTO, T, TN, NT, MINB, KPC)                                             \
    SoftmaxTier {                                                                          \
        kLongMaxCols, AUTO, &launch_softmax_long<T, NT, MINB, KPC>,                         \
            "softmax_long<" TN ",V16,T" #NT ",M" #MINB ",K" #KPC ">"                        \
    }

#define TT_SM_WARP_R(AUTO, T, TN, VB, G, NV, NT, MINB, RPG)                               \
    SoftmaxTier {                                                                          \
        (G) * (NV) * ((VB) / (int)sizeof(T)), AUTO,                                        \
            &launch_softmax_warp<T, VB, G, NV, NT, MINB, RPG>,                             \
            "softmax_warp<" TN ",V" #VB ",G" #G ",NV" #NV ",T" #NT ",M" #MINB ",P" #RPG ">" \
    }
// cross-row prefetch (two rows in flight per group)
#define TT_SM_WARP_F(AUTO, T, TN, VB, G, NV, NT, MINB, RPG)                               \
    SoftmaxTier {                                                                          \
        (G) * (NV) * ((VB) / (int)sizeof(T)), AUTO,                                        \
            &launch_softmax_warp<T, VB, G, NV, NT, MINB, RPG, true>,                       \
            "softmax_warp<" TN ",V" #VB ",G" #G ",NV" #NV ",T" #NT ",M" #MINB ",P" #RPG ",F>" \
    }
// default: 4 rows per group per CTA
#define TT_SM_WARP(AUTO, T, TN, VB, G, NV, NT, MINB) TT_SM_WARP_R(AUTO, T, TN, VB, G, NV, NT, MINB, 4)

#define TT_SM_TMA(AUTO, T, TN, NV, NW)                                                     \
    SoftmaxTier {                                                                          \
        32 * (NV) * (16 / (int)sizeof(T)), AUTO, &launch_softmax_tma<T, NV, NW>,           \
            "softmax_tma<" TN ",V16,G32,NV" #NV ",W" #NW ">"                              \
    }

// Automatic tiers are ordered by max_cols; the first that fits is used.
// Short rows use 16-byte vectors so that more lanes carry bytes; rows of
// >= 256 B use 32-byte vectors (LDG.256).  Sub-warp groups handle many short
// rows per warp; R = 2 rows per group in flight doubles the memory-level
// parallelism.  CTA tiers keep NV * VE = 32 fp32 registers of row data per
// thread so that a 1024-thread CTA fits the 64-register limit: NVC = 4 (fp32)
// or 2 (16-bit).  Non-automatic entries are tuning candidates (tt_tune.h).
#define TT_SM_LIST(T, TN, NVC, M2, M3, M4)                                                   \
    TT_SM_WARP(true, T, TN, 16, 4, 1, 256, 6), TT_SM_WARP(true, T, TN, 16, 8, 1, 256, 6),       \
    TT_SM_WARP(true, T, TN, 16, 16, 1, 256, 6), TT_SM_WARP(true, T, TN, 32, 16, 1, 256, 6),     \
    TT_SM_WARP(true, T, TN, 32, 32, 1, 256, 6), TT_SM_WARP(true, T, TN, 32, 32, 2, 256, M2),    \
    TT_SM_WARP(true, T, TN, 32, 32, 3, 256, M3), TT_SM_WARP(true, T, TN, 32, 32, 4, 256, M4),   \
    TT_SM_TIER(true, T, TN, 32, 64, NVC, 1, 64, 1), TT_SM_TIER(true, T, TN, 32, 128, NVC, 1, 128, 1), \
    TT_SM_TIER(true, T, TN, 32, 256, NVC, 1, 256, 1), TT_SM_TIER(true, T, TN, 32, 512, NVC, 1, 512, 1), \
    TT_SM_CLUSTER(true, T, TN, 32, NVC, 512), TT_SM_LONG(true, T, TN, 256, 4, 65536),                      \
    /* selected through the preference table kSmPref */                                      \
    TT_SM_WARP(false, T, TN, 16, 8, 2, 256, 6), TT_SM_WARP_F(false, T, TN, 16, 8, 4, 256, 3, 4), \
    TT_SM_WARP_R(false, T, TN, 32, 32, 1, 256, 6, 2), TT_SM_WARP_R(false, T, TN, 32, 32, 2, 256, 3, 2), \
    TT_SM_WARP(false, T, TN, 16, 8, 4, 256, 4), TT_SM_WARP(false, T, TN, 16, 8, 5, 256, 4),     \
    TT_SM_WARP(false, T, TN, 32, 8, 3, 256, 3)

// Tuning candidates (tools/tune.py): compiled into the TT_TUNING build only.
#define TT_SM_TUNE_LIST(T, TN)                                                                 \
    TT_SM_TIER(false, T, TN, 32, 32, 1, 1, 256, 6), TT_SM_TMA(false, T, TN, 2, 4),             \
    TT_SM_TMA(false, T, TN, 4, 8),                                                             \
    TT_SM_WARP(false, T, TN, 32, 32, 1, 256, 5), TT_SM_WARP(false, T, TN, 32, 32, 1, 128, 12),  \
    TT_SM_WARP(false, T, TN, 32, 32, 2, 256, 3), TT_SM_WARP(false, T, TN, 32, 32, 2, 256, 5),   \
    TT_SM_WARP(false, T, TN, 16, 32, 2, 256, 6), TT_SM_WARP(false, T, TN, 32, 32, 3, 256, 2),   \
    TT_SM_WARP_R(false, T, TN, 32, 32, 1, 256, 6, 8),                                         \
    TT_SM_WARP(false, T, TN, 16, 8, 6, 256, 3), TT_SM_WARP(false, T, TN, 16, 8, 7, 256, 2),     \
    TT_SM_WARP(false, T, TN, 16, 16, 3, 256, 4), TT_SM_WARP(false, T, TN, 16, 16, 4, 256, 3),   \
    TT_SM_WARP(false, T, TN, 32, 8, 2, 256, 4),                                               \
    TT_SM_WARP(false, T, TN, 32, 16, 2, 256, 3), TT_SM_WARP(false, T, TN, 16, 8, 5, 256, 3),    \
    TT_SM_WARP(false, T, TN, 16, 16, 3, 256, 5), TT_SM_WARP(false, T, TN, 16, 8, 3, 256, 5),   \
    TT_SM_WARP(false, T, TN, 32, 8, 4, 256, 2),                                               \
    TT_SM_WARP(false, T, TN, 16, 8, 8, 256, 2), TT_SM_WARP(false, T, TN, 32, 16, 2, 256, 4),    \
    TT_SM_WARP(false, T, TN, 16, 16, 4, 256, 4), TT_SM_WARP(false, T, TN, 32, 32, 1, 256, 4),   \
    TT_SM_WARP_F(false, T, TN, 32, 32, 1, 256, 6, 2), TT_SM_WARP_F(false, T, TN, 32, 32, 1, 256, 6, 4), \
    TT_SM_WARP_F(false, T, TN, 32, 32, 1, 256, 5, 4)

#ifdef TT_TUNING
#define TT_SM_ALL(T, TN, NVC, M2, M3, M4) TT_SM_LIST(T, TN, NVC, M2, M3, M4), TT_SM_TUNE_LIST(T, TN)
#else
#define TT_SM_ALL(T, TN, NVC, M2, M3, M4) TT_SM_LIST(T, TN, NVC, M2, M3, M4)
#endif

// M2..M4: min CTAs/SM (register cap) of the NV = 2..4 warp tiers, chosen so
// the row (NV * VE fp32 values per lane) fits without spilling.
const SoftmaxTier kSm_f32[] = {TT_SM_ALL(float, "f32", 4, 6, 5, 4)};
const SoftmaxTier kSm_f16[] = {TT_SM_ALL(__half, "f16", 2, 4, 3, 2)};
const SoftmaxTier kSm_bf16[] = {TT_SM_ALL(__nv_bfloat16, "bf16", 2, 4, 3, 2)};
constexpr int kSmN = (int)(sizeof(kSm_f32) / sizeof(kSm_f32[0]));

std::atomic<int> g_force[3] = {{-1}, {-1}, {-1}};

const SoftmaxTier* table(int dtype) {
    switch (dtype) {
        case 0: return kSm_f32;
        case 1: return kSm_f16;
        case 2: return kSm_bf16;
        default: return nullptr;
    }
}

// Tuned preferences (tools/tune.py on B200, profiles/*_tune.txt): for rows of
// more than min_cols and at most max_cols keys, use the named tier.
struct Pref {
    int dtype;
    int min_cols, max_cols;
    const char* name;
    int64_t min_rows;  // applies only to calls with more rows (0: any)
};
// Capacity-fitting sub-warp tiers (G8 with several vectors per lane) win where
// the warp-per-row tier would leave lanes idle; see profiles/*_tune.txt.
const Pref kSmPref[] = {
    // fp32 C2 S = 40 / 64 / 100 (profiles/r01_tune_smtiny/): -31 / -27 / -21 %; not
    // for C1-sized calls (480 rows: +6 %), hence the row threshold
    {0, 32, 64, "softmax_warp<f32,V16,G8,NV2,T256,M6,P4>", 2048},
    {0, 64, 128, "softmax_warp<f32,V16,G8,NV4,T256,M3,P4,F>", 2048},
    {0, 128, 256, "softmax_warp<f32,V32,G32,NV1,T256,M6,P2>"},
    {0, 256, 384, "softmax_warp<f32,V32,G32,NV2,T256,M6,P4>"},
    {0, 384, 512, "softmax_warp<f32,V32,G32,NV2,T256,M3,P2>"},
    {1, 64, 128, "softmax_warp<f16,V16,G8,NV2,T256,M6,P4>"},
    {1, 128, 256, "softmax_warp<f16,V16,G8,NV4,T256,M4,P4>"},
    {1, 256, 320, "softmax_warp<f16,V16,G8,NV5,T256,M4,P4>"},
    {1, 320, 384, "softmax_warp<f16,V32,G8,NV3,T256,M3,P4>"},
    {1, 384, 512, "softmax_warp<f16,V32,G32,NV1,T256,M6,P2>"},  // C3 / C2 ragged: -3..6%
    {2, 64, 128, "softmax_warp<bf16,V16,G8,NV2,T256,M6,P4>"},
    {2, 128, 256, "softmax_warp<bf16,V16,G8,NV4,T256,M4,P4>"},
    {2, 256, 320, "softmax_warp<bf16,V16,G8,NV5,T256,M4,P4>"},
    {2, 320, 384, "softmax_warp<bf16,V32,G8,NV3,T256,M3,P4>"},
};

const SoftmaxTier* pick_dtype(int dtype, int64_t Sk, int64_t nrows) {
    const SoftmaxTier* t = table(dtype);
    if (!t) return nullptr;
    const int f = g_force[dtype].load(std::memory_order_relaxed);
    if (f >= 0 && f < kSmN && Sk <= t[f].max_cols) return &t[f];
    // name -> tier index, resolved once per entry (benign race: same value)
    constexpr int NP = (int)(sizeof(kSmPref) / sizeof(kSmPref[0]));
    static std::atomic<int> pidx[NP];
    for (int p = 0; p < NP; ++p) {
        const Pref& pr = kSmPref[p];
        if (pr.dtype != dtype || Sk <= pr.min_cols || Sk > pr.max_cols || nrows <= pr.min_rows)
            continue;
        int k = pidx[p].load(std::memory_order_relaxed);
        if (k == 0) {
            k = -1;
            for (int i = 0; i < kSmN; ++i)
                if (!strcmp(t[i].name, pr.name)) k = i + 1;
            pidx[p].store(k, std::memory_order_relaxed);
        }
        if (k > 0 && Sk <= t[k - 1].max_cols) return &t[k - 1];
    }
    for (int i = 0; i < kSmN; ++i)
        if (t[i].automatic && Sk <= t[i].max_cols) return &t[i];
    return nullptr;
}

}  // namespace

int softmax_tier_count() { return kSmN; }

const char* softmax_tier_name_at(int dtype, int i) {
    const SoftmaxTier* t = table(dtype);
    return (t && i >= 0 && i < kSmN) ? t[i].name : nullptr;
}

int softmax_tier_max_cols_at(int dtype, int i) {
    const SoftmaxTier* t = table(dtype);
    return (t && i >= 0 && i < kSmN) ? t[i].max_cols : -1;
}

bool softmax_force_tier(int dtype, int i) {
    if (dtype < 0 || dtype > 2 || i < -1 || i >= kSmN) return false;
    g_force[dtype].store(i);
    return true;
}

const char* softmax_tier_name(int dtype, int64_t Sk, int64_t nrows) {
    const SoftmaxTier* t = pick_dtype(dtype, Sk, nrows);
    return t ? t->name : nullptr;
}

cudaError_t softmax_launch(int dtype, void* scores, const int32_t* lengths, int64_t nrows,
                           int64_t rows_per_batch, int64_t Sk, float scale, cudaStream_t stream,
                           bool* supported) {
    const SoftmaxTier* t = pick_dtype(dtype, Sk, nrows);
    *supported = t != nullptr;
    if (!t) return cudaSuccess;
    return t->fn(scores, lengths, nrows, rows_per_batch, (int)Sk, scale, stream);
}

}  // namespace tt
