// softmax_packed.cu -- padding-free (packed) attention softmax, SURVEY §8(f)
// NEXT-1: the variable-length batch of PAPER.md §5 (l.576: "all requests in
// the batch will be zero-padded with regards to the maximum length") without
// the padding.  Request r's scores are a dense [H, L_r, L_r] block at element
// offset cu_blocks[r]; every key of every row is valid, so no byte of padding
// is read or written (-55% softmax traffic on a C3 draw).
//
// Rows are numbered across requests (request r owns rows H*cu[r] ..
// H*cu[r+1]-1).  A CTA owns GPB*rpg consecutive rows; when they belong to one
// request (almost always: a request has H*L_r rows) the CTA picks its group
// width from L_r -- 4, 8, 16 or 32 lanes per row -- so short requests pack
// several rows into one warp pass.  The per-row body is softmax_row_pass, the
// same code as the padded warp tier (softmax_row.cuh).
#include <atomic>

#include "common.cuh"
#include "launch.h"
#include "softmax_row.cuh"

namespace tt {

namespace {
constexpr float kLog2eP = 1.4426950408889634f;
}

// largest r in [0, num_req) with H * cu[r] <= row (cu nondecreasing, cu[0] = 0),
// searched by one whole warp (every lane calls it with the same row; the
// result is warp-uniform): 32 evenly spaced probes per round and a ballot,
// so ceil(log32 num_req) dependent loads instead of log2 num_req, and no CTA
// barrier -- the CTA-wide search by one thread behind a __syncthreads was 25 %
// of the packed kernel's stall samples (profiles/r02_packed/).
__device__ __forceinline__ int find_req_warp(const int32_t* __restrict__ cu, int num_req,
                                             uint32_t H, uint32_t row) {
    const int lane = threadIdx.x & 31;
    int lo = 0, cnt = num_req;  // the answer lies in [lo, lo + cnt); cu[lo] qualifies
    while (true) {
        const int step = (cnt + 31) / 32;
        const bool probe = lane * step < cnt;
        const int idx = lo + (probe ? lane * step : 0);
        const bool ok = probe && (uint64_t)H * (uint32_t)__ldg(cu + idx) <= row;
        const unsigned bal = __ballot_sync(0xffffffffu, ok);  // lane 0 always set
        const int k = 31 - __clz(bal);
        if (step == 1) return lo + k;
        const int hi = lo + cnt;
        lo += k * step;
        cnt = min(step, hi - lo);
    }
}

// all rows of [first, row_end) belong to one request of length L whose block
// starts at `base` and whose first row is row0
template <typename T, int VB, int GC, int NVC, int NT, bool UP>
__device__ __forceinline__ void packed_rows(T* __restrict__ scores, uint32_t first,
                                            uint32_t row_end, int64_t base, uint32_t row0, int L,
                                            float c) {
    constexpr int GPW = 32 / GC;
    const int lane = threadIdx.x & 31;
    const int q = lane % GC;
    const uint32_t step = (NT / 32) * GPW;
    uint32_t row = first + (threadIdx.x >> 5) * GPW + lane / GC;
    for (uint32_t b = first + (threadIdx.x >> 5) * GPW; b < row_end; b += step, row += step) {
        const bool live = row < row_end;
        T* p = scores + base + (int64_t)((live ? row : first) - row0) * L;
        softmax_row_pass<T, VB, GC, NVC, false, false, UP, true>(p, live, L, L, c, q);
    }
}

template <typename T, int VB, int NV, int NT, bool UP>
__device__ __forceinline__ void packed_body(T* __restrict__ scores, const int32_t* __restrict__ cu,
                                            const int64_t* __restrict__ blocks, int num_req,
                                            uint32_t H, uint32_t total_rows, float c, int rpg) {
    constexpr int VE = VB / (int)sizeof(T);
    constexpr int GPB = NT / 32;
    constexpr int CAP = 32 * NV * VE;
    const uint32_t dev_rows = H * (uint32_t)__ldg(cu + num_req);
    const uint32_t first = blockIdx.x * (uint32_t)(GPB * rpg);
    const uint32_t row_end = min(min(total_rows, dev_rows), first + (uint32_t)(GPB * rpg));
    if (first >= row_end) return;  // uniform per CTA
    // every warp finds the requests of the CTA's first and last rows itself
    const int r0 = find_req_warp(cu, num_req, H, first);
    const int r1 = find_req_warp(cu, num_req, H, row_end - 1);
    if (r0 == r1) {
        const int L = min(__ldg(cu + r0 + 1) - __ldg(cu + r0), CAP);
        const int64_t base = __ldg(blocks + r0);
        const uint32_t row0 = H * (uint32_t)__ldg(cu + r0);
        // narrow groups only where the scalar head / tail of an odd-pitch row
        // fits one pass (GC >= VE - 1), as in the padded kernel
        constexpr bool ok4 = 4 >= VE - 1, ok8 = 8 >= VE - 1;
        if (ok4 && L <= 4 * VE)
            return packed_rows<T, VB, ok4 ? 4 : 32, 1, NT, UP>(scores, first, row_end, base, row0, L, c);
        if (ok8 && L <= 8 * VE)
            return packed_rows<T, VB, ok8 ? 8 : 32, 1, NT, UP>(scores, first, row_end, base, row0, L, c);
        if (L <= 16 * VE)
            return packed_rows<T, VB, 16, 1, NT, UP>(scores, first, row_end, base, row0, L, c);
        if (L <= 32 * VE)
            return packed_rows<T, VB, 32, 1, NT, UP>(scores, first, row_end, base, row0, L, c);
        return packed_rows<T, VB, 32, NV, NT, UP>(scores, first, row_end, base, row0, L, c);
    }
    // the CTA straddles requests: one row per warp, looked up per row
    const int lane = threadIdx.x & 31;
    for (uint32_t row = first + (threadIdx.x >> 5); row < row_end; row += GPB) {
        const int r = find_req_warp(cu, num_req, H, row);
        const int L = min(__ldg(cu + r + 1) - __ldg(cu + r), CAP);
        const uint32_t row0 = H * (uint32_t)__ldg(cu + r);
        T* p = scores + __ldg(blocks + r) + (int64_t)(row - row0) * L;
        softmax_row_pass<T, VB, 32, NV, false, false, UP, true>(p, true, L, L, c, lane);
    }
}

template <typename T, int VB, int NV, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB)
    softmax_packed_kernel(T* __restrict__ scores, const int32_t* __restrict__ cu,
                          const int64_t* __restrict__ blocks, int num_req, uint32_t H,
                          uint32_t total_rows, float c, int rpg) {
    PdlScope pdl_;  // griddepcontrol.wait first: no global access before it (PDL)
    if (c > 0.f)  // uniform: the sign of the scale picks the max or min reduction
        packed_body<T, VB, NV, NT, true>(scores, cu, blocks, num_req, H, total_rows, c, rpg);
    else
        packed_body<T, VB, NV, NT, false>(scores, cu, blocks, num_req, H, total_rows, c, rpg);
}

namespace {

int sm_count_p() {
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

template <typename T, int NV, int MINB>
cudaError_t launch_packed(void* scores, const int32_t* cu, const int64_t* blocks, int num_req,
                          int64_t H, int64_t total_rows, float scale, cudaStream_t st) {
// 4 rows per warp per CTA: measured against 8 and 16 (idle warps when short
// requests use 4-lane groups notwithstanding): C3 packed step 0.0887 / 0.0890 /
// 0.0962 ms, C5 packed stream 5.17 / 5.20 / 5.66 ms (profiles/r01_packed_rpg/)
#ifndef TT_PACKED_RPG
#define TT_PACKED_RPG 4
#endif
    constexpr int NT = 256, GPB = NT / 32, RPG = TT_PACKED_RPG;
    const int64_t per_cta = (int64_t)GPB * RPG;
    const int64_t grid = (total_rows + per_cta - 1) / per_cta;
    if (grid > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
    float c = scale * kLog2eP;
    if (c == 0.f) c = 1e-30f;  // see softmax.cu: keeps sentinel keys at exactly +0.0
    {
        const cudaError_t le_ = launch_k(softmax_packed_kernel<T, 32, NV, NT, MINB>, (unsigned)grid, NT, 0, st,
        static_cast<T*>(scores), cu, blocks, num_req, (uint32_t)H, (uint32_t)total_rows, c, RPG);
        if (le_ != cudaSuccess) return le_;
    }
    (void)sm_count_p;
    return cudaGetLastError();
}

using PackedFn = cudaError_t (*)(void*, const int32_t*, const int64_t*, int, int64_t, int64_t,
                                 float, cudaStream_t);

struct PackedTier {
    int max_len;
    PackedFn fn;
    const char* name;
};

#define TT_PK(T, TN, NV, MINB)                                                              \
    PackedTier {                                                                           \
        32 * (NV) * (32 / (int)sizeof(T)), &launch_packed<T, NV, MINB>,                    \
            "softmax_packed<" TN ",V32,NV" #NV ",T256,M" #MINB ",P4>"                      \
    }

// register caps as in the padded warp tiers (NV * VE fp32 values per lane),
// lowered by one CTA per SM where ptxas would spill at the padded tier's cap
// (f32 NV3, f16 NV1, 16-bit NV3)
const PackedTier kPk_f32[] = {TT_PK(float, "f32", 1, 6), TT_PK(float, "f32", 2, 3),
                              TT_PK(float, "f32", 3, 4), TT_PK(float, "f32", 4, 4)};
const PackedTier kPk_f16[] = {TT_PK(__half, "f16", 1, 5), TT_PK(__half, "f16", 2, 4),
                              TT_PK(__half, "f16", 3, 2), TT_PK(__half, "f16", 4, 2)};
const PackedTier kPk_bf16[] = {TT_PK(__nv_bfloat16, "bf16", 1, 5),
                               TT_PK(__nv_bfloat16, "bf16", 2, 4),
                               TT_PK(__nv_bfloat16, "bf16", 3, 2),
                               TT_PK(__nv_bfloat16, "bf16", 4, 2)};

const PackedTier* pick(int dtype, int64_t max_len) {
    const PackedTier* t = dtype == 0 ? kPk_f32 : dtype == 1 ? kPk_f16 : dtype == 2 ? kPk_bf16
                                                                                    : nullptr;
    if (!t) return nullptr;
    for (int i = 0; i < 4; ++i)
        if (max_len <= t[i].max_len) return &t[i];
    return nullptr;
}

}  // namespace

int softmax_packed_max_len(int dtype) { return dtype == 0 ? 1024 : 2048; }

const char* softmax_packed_tier_name(int dtype, int64_t max_len) {
    const PackedTier* t = pick(dtype, max_len);
    return t ? t->name : nullptr;
}

cudaError_t softmax_packed_launch(int dtype, void* scores, const int32_t* cu_seqlens,
                                  const int64_t* cu_blocks, int64_t num_req, int64_t H,
                                  int64_t total_tokens, int64_t max_len, float scale,
                                  cudaStream_t stream, bool* supported) {
    const PackedTier* t = pick(dtype, max_len);
    *supported = t != nullptr;
    if (!t) return cudaSuccess;
    return t->fn(scores, cu_seqlens, cu_blocks, (int)num_req, H, H * total_tokens, scale, stream);
}

}  // namespace tt
