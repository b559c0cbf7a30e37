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
#include "layernorm_kernels.cuh"

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

#ifdef TT_TUNING
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
#endif  // TT_TUNING

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


// Resident-CTA cap (launch bounds, 256 threads) at which the non-exact warp
// tier compiles without spills, by row values per lane (probed with ptxas,
// tools/probe/probe_ln.cu, for every automatic tier).
template <typename T, int VB, int NV>
constexpr int ln_minb_nonexact() {
    constexpr int vpl = NV * VB / (int)sizeof(T);
    if constexpr (sizeof(T) == 4)
        return vpl <= 8 ? 5 : vpl <= 12 ? 4 : vpl <= 16 ? 3 : vpl <= 32 ? 2 : 1;
    else
        return vpl <= 16 ? 4 : vpl <= 24 ? 3 : vpl <= 48 ? 2 : 1;
}

template <typename T, int VB, int G, int NV, int NT, int MINB, bool PF>
cudaError_t launch_ln_warp(void* out, const void* x, const void* res, const void* bias,
                           const void* gamma, const void* beta, int64_t rows, int hidden,
                           float eps, cudaStream_t st) {
    constexpr int GPB = NT / G;
    constexpr int CAP = G * NV * (VB / (int)sizeof(T));
    if (rows >= (int64_t)0xffffffffLL)  // 32-bit row indices: the generic tier (no spills at M1)
        return launch_ln<T, VB, G, NV, 1, NT, 1>(out, x, res, bias, gamma, beta, rows, hidden,
                                                 eps, st);
    // hidden < capacity: the per-vector bounds tests cost registers, so that
    // instantiation runs one CTA per SM fewer (ln_minb_nonexact; both are
    // spill-free in ptxas, tools/probe/probe_ln.cu)
    constexpr int MNX = ln_minb_nonexact<T, VB, NV>() < MINB ? ln_minb_nonexact<T, VB, NV>() : MINB;
    const bool exact = hidden == CAP;
    auto kern = exact ? ln_warp_kernel<T, VB, G, NV, NT, MINB, PF, true>
                      : ln_warp_kernel<T, VB, G, NV, NT, MNX, PF, false>;
    const size_t smem = (size_t)3 * hidden * sizeof(float);
    cudaError_t e = smem_optin(reinterpret_cast<const void*>(kern), smem);
    if (e != cudaSuccess) return e;
    // resident CTAs per SM for this (kernel, smem): cached, the kernel's
    // register and smem footprint do not change between calls
    static std::atomic<long long> occ_cache[2] = {{0}, {0}};
    const long long key = (long long)smem << 8;
    long long c = occ_cache[exact].load(std::memory_order_relaxed);
    int occ = 0;
    if ((c & ~0xffLL) == key && (c & 0xff)) {
        occ = (int)(c & 0xff);
    } else {
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, smem);
        if (e != cudaSuccess) return e;
        occ = occ > 0 ? (occ < 255 ? occ : 255) : 1;
        occ_cache[exact].store(key | occ, std::memory_order_relaxed);
    }
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
// data).  Non-automatic entries are selected through the preference tables.
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
    /* selected through the preference tables kLnPref* */                                    \
    TT_LN_TIER(false, T, TN, 32, 32, 3, 1, 256, 1), TT_LN_TIER(false, T, TN, 32, 32, 4, 1, 256, 1), \
    TT_LN_TIER(false, T, TN, 32, 32, 4, 1, 128, 1), TT_LN_TIER(false, T, TN, 32, 32, 2, 1, 256, 1), \
    TT_LN_TIER(false, T, TN, 16, 32, 3, 1, 256, 1), TT_LN_TIER(false, T, TN, 32, 16, 3, 1, 256, 1), \
    TT_LN_EARLY(false, T, TN, 16, 32, 3, 128), TT_LN_EARLY(false, T, TN, 16, 32, 3, 256),        \
    TT_LN_EARLY(false, T, TN, 32, 32, 2, 128), TT_LN_EARLY(false, T, TN, 32, 32, 2, 256),        \
    TT_LN_EARLY(false, T, TN, 32, 32, 3, 256), TT_LN_EARLY(false, T, TN, 32, 32, 4, 256),        \
    TT_LN_TIER(false, T, TN, 32, 32, 3, 1, 128, 1), TT_LN_TIER(false, T, TN, 16, 32, 3, 1, 128, 1), \
    TT_LN_TIER(false, T, TN, 32, 32, 2, 1, 128, 6), TT_LN_TIER(false, T, TN, 32, 32, 2, 1, 64, 12)

// Tuning candidates (tools/tune.py): compiled into the TT_TUNING build only.
#define TT_LN_TUNE_LIST(T, TN)                                                                 \
    TT_LN_TIER(false, T, TN, 32, 32, 2, 1, 128, 1), TT_LN_WARP_P(false, T, TN, 16, 32, 4, 256, 2, 1), \
    TT_LN_TMA(false, T, TN, 3, 8), TT_LN_TMA(false, T, TN, 4, 8), TT_LN_TMA(false, T, TN, 4, 4),       \
    TT_LN_TMA(false, T, TN, 6, 4), TT_LN_TMA(false, T, TN, 8, 4),                                    \
    TT_LN_WARP_P(false, T, TN, 16, 32, 3, 256, 2, 1), TT_LN_WARP_P(false, T, TN, 16, 32, 3, 256, 3, 1), \
    TT_LN_WARP_P(false, T, TN, 16, 32, 4, 256, 3, 1), TT_LN_WARP_P(false, T, TN, 32, 32, 2, 256, 2, 1), \
    TT_LN_WARP_P(false, T, TN, 32, 32, 2, 256, 3, 1), TT_LN_WARP_P(false, T, TN, 32, 32, 3, 256, 2, 1), \
    TT_LN_WARP_P(false, T, TN, 32, 32, 4, 256, 2, 1), TT_LN_WARP_P(false, T, TN, 16, 32, 6, 256, 2, 1), \
    TT_LN_WARP_P(false, T, TN, 16, 32, 8, 256, 2, 1),                                          \
    TT_LN_WARP(false, T, TN, 16, 32, 3, 256, 4),                                              \
    TT_LN_WARP(false, T, TN, 16, 32, 4, 256, 3), TT_LN_WARP(false, T, TN, 16, 32, 4, 256, 4),   \
    TT_LN_WARP(false, T, TN, 32, 32, 2, 256, 3), TT_LN_WARP(false, T, TN, 32, 32, 2, 256, 4),   \
    TT_LN_WARP(false, T, TN, 32, 32, 3, 256, 3), TT_LN_WARP(false, T, TN, 32, 32, 4, 256, 3),   \
    TT_LN_WARP(false, T, TN, 16, 32, 6, 256, 3), TT_LN_WARP(false, T, TN, 16, 32, 8, 256, 3),   \
    TT_LN_WARP(false, T, TN, 32, 16, 3, 256, 3), TT_LN_WARP(false, T, TN, 32, 16, 4, 256, 3),   \
    TT_LN_WARP(false, T, TN, 32, 16, 3, 256, 4), TT_LN_WARP(false, T, TN, 32, 16, 4, 256, 2),   \
    TT_LN_WARP(false, T, TN, 16, 16, 6, 256, 3), TT_LN_WARP(false, T, TN, 16, 16, 8, 256, 2),   \
    TT_LN_WARP(false, T, TN, 32, 8, 6, 256, 2), TT_LN_WARP(false, T, TN, 32, 16, 6, 256, 2),    \
    TT_LN_WARP(false, T, TN, 16, 32, 3, 128, 6), TT_LN_WARP(false, T, TN, 16, 32, 4, 128, 6),   \
    TT_LN_WARP(false, T, TN, 32, 32, 2, 128, 6), TT_LN_WARP(false, T, TN, 32, 32, 3, 128, 6),   \
    TT_LN_TIER(false, T, TN, 32, 32, 3, 2, 256, 1), TT_LN_TIER(false, T, TN, 32, 32, 4, 2, 256, 1), \
    TT_LN_TIER(false, T, TN, 32, 16, 4, 1, 256, 1),                                        \
    TT_LN_TIER(false, T, TN, 16, 32, 4, 1, 256, 1), TT_LN_TIER(false, T, TN, 16, 32, 6, 1, 256, 1), \
    TT_LN_TIER(false, T, TN, 32, 32, 2, 2, 128, 4),                                        \
    TT_LN_TIER(false, T, TN, 32, 32, 2, 1, 256, 3), TT_LN_TIER(false, T, TN, 16, 32, 4, 1, 128, 6), \
    TT_LN_TIER(false, T, TN, 16, 32, 3, 2, 128, 4), TT_LN_TIER(false, T, TN, 16, 32, 3, 1, 64, 12), \
    TT_LN_TIER(false, T, TN, 32, 32, 3, 1, 64, 10)

#ifdef TT_TUNING
#define TT_LN_ALL(T, TN, SB, NVC32, NVC16, MA, MB, MC) \
    TT_LN_LIST(T, TN, SB, NVC32, NVC16, MA, MB, MC), TT_LN_TUNE_LIST(T, TN)
#else
#define TT_LN_ALL(T, TN, SB, NVC32, NVC16, MA, MB, MC) TT_LN_LIST(T, TN, SB, NVC32, NVC16, MA, MB, MC)
#endif

// MA / MB / MC: min CTAs/SM (register cap, exact hidden) for warp tiers
// holding about 8-16 / 12-32 / 24-64 row values per lane: the largest at
// which ptxas does not spill (tools/probe/probe_ln.cu).
const LnTier kLn_f32[] = {TT_LN_ALL(float, "f32", 4, 4, 8, 6, 5, 2)};
const LnTier kLn_f16[] = {TT_LN_ALL(__half, "f16", 2, 2, 4, 6, 3, 2)};
const LnTier kLn_bf16[] = {TT_LN_ALL(__nv_bfloat16, "bf16", 2, 2, 4, 6, 3, 2)};
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
// up to kSmallRows rows: one row per warp, no per-CTA parameter staging,
// small CTAs (many per SM); up to kTinyRows gamma / beta are loaded together
// with the row (ln_rows EARLY tiers), so no dependent load follows the
// reductions.  Re-tuned in round 2 on the packed-pair build
// (profiles/r02_ln/): at hidden 768 the 128-thread ln_rows tiers win from
// 5120 to 10000 rows (fp16 10.9 us vs 11.7 for the persistent warp tier at
// 10000 rows; fp32 16.8 vs 17.9 us).
// kSmallRows re-measured on the final round-2 build (profiles/r02_ln_band/): from 12 000
// rows the large-call tiers win -- 16-bit hidden 768 persistent ln_warp (16 384 rows 15.5 vs
// 16.8 us, 12 000 rows 12.8 vs 13.1), bf16 hidden 1024 T64 (12 000 rows 14.9 vs 15.2), fp32
// hidden 1024 T128 (26.7 vs 27.1) -- while at 11 000 rows (fp16 hidden 768) the 128-thread
// tier still does (12.4 vs 12.6 us).
constexpr int64_t kTinyRows = 2048, kSmallRows = 11500;
const Pref kLnPrefSmall[] = {
    {0, 512, 768, "ln_rows<f32,V32,G32,NV3,R1,T128,M1>"},
    {0, 768, 1024, "ln_rows<f32,V32,G32,NV4,R1,T256,M1>"},
    {1, 512, 768, "ln_rows<f16,V16,G32,NV3,R1,T128,M1>"},
    {1, 768, 1024, "ln_rows<f16,V32,G32,NV2,R1,T256,M1>"},
    {2, 512, 768, "ln_rows<bf16,V16,G32,NV3,R1,T128,M1>"},
    {2, 768, 1024, "ln_rows<bf16,V32,G32,NV2,R1,T256,M1>"},
};
// Just past one full wave of the 128-thread tier (4 rows per CTA; at hidden 768
// 16-bit one wave holds ~5 300 rows): half-warp rows in 256-thread CTAs (16 rows
// per CTA) take the whole call in one wave.  tools/tune.py (profiles/r02_ln_wave/):
// 6000 rows 8.46 -> 7.34 us, while 5120 (6.39 vs 6.92) and 8000 rows (9.56 vs
// 10.88) stay on the 128-thread tier.
constexpr int64_t kWaveLo = 5400, kWaveHi = 7000;
const Pref kLnPrefWave[] = {
    {1, 512, 768, "ln_rows<f16,V32,G16,NV3,R1,T256,M1>"},
    {2, 512, 768, "ln_rows<bf16,V32,G16,NV3,R1,T256,M1>"},  // 6000 / 7000 rows: 7.1 / 7.6 us
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
// More rows (C3, C4, C5): the persistent warp tier with exact-width rows at
// hidden 768 (16-bit C3 25.4 us vs 32.9 round 1), 64-thread ln_rows (12 CTAs
// per SM) at 1024 (C4 32.4 us vs 35.1 round 1, profiles/r02_ln/) and 128-thread
// ln_rows for fp32 (C3 45.4 us vs 46.1).
const Pref kLnPref[] = {
    {0, 512, 768, "ln_rows<f32,V32,G32,NV3,R1,T128,M1>"},
    {0, 768, 1024, "ln_rows<f32,V32,G32,NV4,R1,T128,M1>"},
    {1, 512, 768, "ln_warp<f16,V16,G32,NV3,T256,M3,PF0>"},
    {1, 768, 1024, "ln_rows<f16,V32,G32,NV2,R1,T64,M12>"},
    {2, 512, 768, "ln_warp<bf16,V16,G32,NV3,T256,M3,PF0>"},
    {2, 768, 1024, "ln_rows<bf16,V32,G32,NV2,R1,T64,M12>"},
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
    static std::atomic<int> idx_wave[sizeof(kLnPrefWave) / sizeof(Pref)];
    if (!pbest && rows > kWaveLo && rows <= kWaveHi)
        pbest = from_prefs(kLnPrefWave, idx_wave, dtype, hidden, vec_bytes);
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
