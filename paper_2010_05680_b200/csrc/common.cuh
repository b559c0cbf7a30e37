// common.cuh -- vector I/O, dtype packing and group reductions shared by the
// softmax and LayerNorm kernels (sm_100a only).
//
// Design: a "group" of G consecutive threads owns one row.
//   G in {4, 8, 16, 32}  : sub-warp / warp groups, reductions are register
//                          butterflies (SHFL.BFLY) or one CREDUX for the
//                          warp-wide max -- no shared memory, no barrier.
//   G in {64 .. 1024}    : a whole CTA owns one row (long rows); warp partials
//                          go through shared memory with ONE barrier per batch
//                          of R rows (the paper's "one synchronization for X
//                          elements").
// Each group processes R rows at once so independent loads, shuffles and
// MUFU ops interleave (the paper's warpAllReduceSum_XElem ILP, l.374-383).
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include <cuda_runtime.h>
#include <utility>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ != 1000)
#error "libtt is written for sm_100a only (-gencode arch=compute_100a,code=sm_100a)"
#endif

namespace tt {

// ----------------------------------------------------------------------------
// Programmatic dependent launch (PDL).  Every kernel starts with
// `PdlScope pdl_;`: griddepcontrol.wait blocks until the preceding kernel in
// the stream has completed and its memory is visible (a no-op when the launch
// was not programmatic), so NO global access precedes it.  When the scope ends
// -- after the CTA's last store, on every return path --
// griddepcontrol.launch_dependents lets the next kernel's CTAs be scheduled
// once every CTA of this grid has got there, so the next launch's latency and
// prologue overlap our tail.  (Triggering at kernel entry instead was measured
// slower on single-wave grids: the dependents' CTAs occupy SMs early and the
// grid after them is placed unevenly.)
// ----------------------------------------------------------------------------
struct PdlScope {
    __device__ __forceinline__ PdlScope() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
    __device__ __forceinline__ ~PdlScope() {
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    }
};

bool pdl_enabled();  // tt_api.cu: process-wide switch (ttx_set_pdl), default on

// Opt `kern` into `smem` bytes of dynamic shared memory (> 48 KB) on the
// CURRENT device.  The attribute belongs to each device's context, so the
// cache in tt_api.cu is keyed by (kernel, device); a no-op at <= 48 KB.
cudaError_t smem_optin(const void* kern, size_t smem);

// A triple-chevron launch of kern(args...) with the programmatic-stream-
// serialization attribute when PDL is enabled.
template <typename... P, typename... A>
inline cudaError_t launch_k(void (*kern)(P...), dim3 grid, dim3 block, size_t smem,
                            cudaStream_t st, A&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    if (smem > 48 * 1024) {
        const cudaError_t e = smem_optin(reinterpret_cast<const void*>(kern), smem);
        if (e != cudaSuccess) return e;
    }
    return cudaLaunchKernelEx(&cfg, kern, std::forward<A>(args)...);
}

// The same, as thread-block clusters of cluster_x CTAs along x.
template <typename... P, typename... A>
inline cudaError_t launch_kc(void (*kern)(P...), dim3 grid, dim3 block, size_t smem,
                             cudaStream_t st, unsigned cluster_x, A&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cluster_x;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<A>(args)...);
}

// ----------------------------------------------------------------------------
// Raw vectors of VB bytes (VB in {2, 4, 8, 16, 32}); 32-byte accesses compile
// to LDG.E.256 / STG.E.256 on sm_100a.
// ----------------------------------------------------------------------------
template <int VB>
struct Raw {
    static constexpr int W = VB >= 4 ? VB / 4 : 1;
    uint32_t w[W];
};

// Streaming load: bypass L1 (each byte is used once by one thread).
template <int VB>
__device__ __forceinline__ void ld_stream(const void* p, Raw<VB>& r) {
    if constexpr (VB == 32) {
        asm volatile(
            "ld.global.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
            : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(r.w[4]),
              "=r"(r.w[5]), "=r"(r.w[6]), "=r"(r.w[7])
            : "l"(p));
    } else if constexpr (VB == 16) {
        asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3])
                     : "l"(p));
    } else if constexpr (VB == 8) {
        asm volatile("ld.global.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
                     : "=r"(r.w[0]), "=r"(r.w[1])
                     : "l"(p));
    } else if constexpr (VB == 4) {
        asm volatile("ld.global.L1::no_allocate.u32 %0, [%1];" : "=r"(r.w[0]) : "l"(p));
    } else {
        static_assert(VB == 2, "VB");
        unsigned short h;
        asm volatile("ld.global.L1::no_allocate.u16 %0, [%1];" : "=h"(h) : "l"(p));
        r.w[0] = h;
    }
}

// Read-only parameter load (bias / gamma / beta): cached in L1, shared by all
// rows of the CTA.  Caller guarantees no overlap with any written buffer.
template <int VB>
__device__ __forceinline__ void ld_param(const void* p, Raw<VB>& r) {
    if constexpr (VB == 32) {
        asm("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
            : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(r.w[4]),
              "=r"(r.w[5]), "=r"(r.w[6]), "=r"(r.w[7])
            : "l"(p));
    } else if constexpr (VB == 16) {
        asm("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
            : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3])
            : "l"(p));
    } else if constexpr (VB == 8) {
        asm("ld.global.nc.v2.u32 {%0,%1}, [%2];" : "=r"(r.w[0]), "=r"(r.w[1]) : "l"(p));
    } else if constexpr (VB == 4) {
        asm("ld.global.nc.u32 %0, [%1];" : "=r"(r.w[0]) : "l"(p));
    } else {
        unsigned short h;
        asm("ld.global.nc.u16 %0, [%1];" : "=h"(h) : "l"(p));
        r.w[0] = h;
    }
}

// Streaming store.  EF: with an L2 evict_first cache policy, so the output's
// dirty lines are the first the L2 writes back and a kernel drains its own
// writes instead of leaving up to ~60 MB of them for the next kernel's reads to
// compete with.  Used by the softmax warp tiers on rows made of whole 128-byte
// lines (C4 step, bench.py, 2 runs each: 0.2091 -> 0.2066 ms).  Measured slower
// elsewhere (fp16 hidden-768 LayerNorm -11 %, softmax rows sharing a line with
// the next row -4.5..-6 %: the line is evicted half-written), so every other
// store is plain.
template <int VB, bool EF = false>
__device__ __forceinline__ void st_stream(void* p, const Raw<VB>& r) {
    if constexpr (EF && (VB == 32 || VB == 16)) {
        uint64_t pol;
        asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        if constexpr (VB == 32)
            asm volatile(
                "st.global.L1::no_allocate.L2::cache_hint.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8}, %9;"
                ::"l"(p), "r"(r.w[0]), "r"(r.w[1]), "r"(r.w[2]), "r"(r.w[3]), "r"(r.w[4]),
                "r"(r.w[5]), "r"(r.w[6]), "r"(r.w[7]), "l"(pol)
                : "memory");
        else
            asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;"
                         ::"l"(p), "r"(r.w[0]), "r"(r.w[1]), "r"(r.w[2]), "r"(r.w[3]), "l"(pol)
                         : "memory");
        return;
    }
    if constexpr (VB == 32) {
        asm volatile(
            "st.global.L1::no_allocate.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p),
            "r"(r.w[0]), "r"(r.w[1]), "r"(r.w[2]), "r"(r.w[3]), "r"(r.w[4]), "r"(r.w[5]),
            "r"(r.w[6]), "r"(r.w[7])
            : "memory");
    } else if constexpr (VB == 16) {
        asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p),
                     "r"(r.w[0]), "r"(r.w[1]), "r"(r.w[2]), "r"(r.w[3])
                     : "memory");
    } else if constexpr (VB == 8) {
        asm volatile("st.global.L1::no_allocate.v2.u32 [%0], {%1,%2};" ::"l"(p), "r"(r.w[0]),
                     "r"(r.w[1])
                     : "memory");
    } else if constexpr (VB == 4) {
        asm volatile("st.global.L1::no_allocate.u32 [%0], %1;" ::"l"(p), "r"(r.w[0]) : "memory");
    } else {
        unsigned short h = (unsigned short)r.w[0];
        asm volatile("st.global.L1::no_allocate.u16 [%0], %1;" ::"l"(p), "h"(h) : "memory");
    }
}

// ----------------------------------------------------------------------------
// dtype <-> fp32.  Narrowing is round-to-nearest-even (DESIGN R12).
// ----------------------------------------------------------------------------
template <typename T>
struct Elem;

template <>
struct Elem<float> {
    static __device__ __forceinline__ float to_f(float v) { return v; }
    static __device__ __forceinline__ float from_f(float v) { return v; }
    template <int VB>
    static __device__ __forceinline__ void unpack(const Raw<VB>& r, float* f) {
#pragma unroll
        for (int i = 0; i < VB / 4; ++i) f[i] = __uint_as_float(r.w[i]);
    }
    template <int VB>
    static __device__ __forceinline__ void pack(const float* f, Raw<VB>& r) {
#pragma unroll
        for (int i = 0; i < VB / 4; ++i) r.w[i] = __float_as_uint(f[i]);
    }
};

template <>
struct Elem<__half> {
    static __device__ __forceinline__ float to_f(__half v) { return __half2float(v); }
    static __device__ __forceinline__ __half from_f(float v) { return __float2half_rn(v); }
    template <int VB>
    static __device__ __forceinline__ void unpack(const Raw<VB>& r, float* f) {
        if constexpr (VB == 2) {
            f[0] = __half2float(__ushort_as_half((unsigned short)r.w[0]));
        } else {
#pragma unroll
            for (int i = 0; i < VB / 4; ++i) {
                __half2 h = *reinterpret_cast<const __half2*>(&r.w[i]);
                float2 t = __half22float2(h);
                f[2 * i] = t.x;
                f[2 * i + 1] = t.y;
            }
        }
    }
    template <int VB>
    static __device__ __forceinline__ void pack(const float* f, Raw<VB>& r) {
        if constexpr (VB == 2) {
            r.w[0] = __half_as_ushort(__float2half_rn(f[0]));
        } else {
#pragma unroll
            for (int i = 0; i < VB / 4; ++i) {
                __half2 h = __floats2half2_rn(f[2 * i], f[2 * i + 1]);
                r.w[i] = *reinterpret_cast<const uint32_t*>(&h);
            }
        }
    }
};

template <>
struct Elem<__nv_bfloat16> {
    static __device__ __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
    static __device__ __forceinline__ __nv_bfloat16 from_f(float v) {
        return __float2bfloat16_rn(v);
    }
    template <int VB>
    static __device__ __forceinline__ void unpack(const Raw<VB>& r, float* f) {
        if constexpr (VB == 2) {
            f[0] = __uint_as_float(r.w[0] << 16);
        } else {
#pragma unroll
            for (int i = 0; i < VB / 4; ++i) {
                f[2 * i] = __uint_as_float(r.w[i] << 16);
                f[2 * i + 1] = __uint_as_float(r.w[i] & 0xffff0000u);
            }
        }
    }
    template <int VB>
    static __device__ __forceinline__ void pack(const float* f, Raw<VB>& r) {
        if constexpr (VB == 2) {
            r.w[0] = __bfloat16_as_ushort(__float2bfloat16_rn(f[0]));
        } else {
#pragma unroll
            for (int i = 0; i < VB / 4; ++i) {
                __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
                r.w[i] = *reinterpret_cast<const uint32_t*>(&h);
            }
        }
    }
};

// ----------------------------------------------------------------------------
// Scalar helpers
// ----------------------------------------------------------------------------
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Packed fp32 pairs (sm_100a FFMA2 / FADD2 / FMUL2): one issue slot does two
// IEEE round-to-nearest fp32 operations, which halves the issue cost of the
// per-element arithmetic of the issue-bound 16-bit softmax rows.
struct F2 {
    unsigned long long r;
};
__device__ __forceinline__ F2 f2_make(float a, float b) {
    F2 o;
    asm("mov.b64 %0, {%1, %2};" : "=l"(o.r) : "f"(a), "f"(b));
    return o;
}
__device__ __forceinline__ void f2_split(F2 v, float& a, float& b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v.r));
}
__device__ __forceinline__ F2 f2_fma(F2 a, F2 b, F2 c) {
    F2 o;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(o.r) : "l"(a.r), "l"(b.r), "l"(c.r));
    return o;
}
__device__ __forceinline__ F2 f2_add(F2 a, F2 b) {
    F2 o;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(o.r) : "l"(a.r), "l"(b.r));
    return o;
}
__device__ __forceinline__ F2 f2_mul(F2 a, F2 b) {
    F2 o;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(o.r) : "l"(a.r), "l"(b.r));
    return o;
}

// Warp-wide f32 max in one instruction (CREDUX.MAX.F32.NAN, sm_100a only).
__device__ __forceinline__ float warp_max_redux(float v) {
    float m;
    asm volatile("redux.sync.max.NaN.f32 %0, %1, 0xffffffff;" : "=f"(m) : "f"(v));
    return m;
}

// ----------------------------------------------------------------------------
// Group all-reduce of R independent values (one per row in flight).
// For G <= 32 the whole group is inside one warp; for G > 32 the group is the
// CTA and `smem` must hold R * (G / 32) floats (distinct buffer per call site).
// ----------------------------------------------------------------------------
template <int G, int R>
__device__ __forceinline__ void group_max(float (&v)[R], float* smem) {
    if constexpr (G >= 32) {
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = warp_max_redux(v[r]);
    } else {
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) {
#pragma unroll
            for (int r = 0; r < R; ++r) v[r] = fmaxf(v[r], __shfl_xor_sync(0xffffffffu, v[r], o));
        }
    }
    if constexpr (G > 32) {
        constexpr int NW = G / 32;
        const int warp = threadIdx.x >> 5;
        if ((threadIdx.x & 31) == 0) {
#pragma unroll
            for (int r = 0; r < R; ++r) smem[r * NW + warp] = v[r];
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < R; ++r) {
            float m = smem[r * NW];
#pragma unroll
            for (int w = 1; w < NW; ++w) m = fmaxf(m, smem[r * NW + w]);
            v[r] = m;
        }
    }
}

template <int G, int R>
__device__ __forceinline__ void group_sum(float (&v)[R], float* smem) {
    constexpr int GW = G < 32 ? G : 32;
#pragma unroll
    for (int o = GW / 2; o > 0; o >>= 1) {
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] += __shfl_xor_sync(0xffffffffu, v[r], o);
    }
    if constexpr (G > 32) {
        constexpr int NW = G / 32;
        const int warp = threadIdx.x >> 5;
        if ((threadIdx.x & 31) == 0) {
#pragma unroll
            for (int r = 0; r < R; ++r) smem[r * NW + warp] = v[r];
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < R; ++r) {
            float s = 0.f;
#pragma unroll
            for (int w = 0; w < NW; ++w) s += smem[r * NW + w];
            v[r] = s;
        }
    }
}

// ----------------------------------------------------------------------------
// Division of a 32-bit row index by a runtime constant (rows per batch) with a
// multiply-high and two shifts instead of the ~25-instruction integer divide:
// the round-up magic-number method (Granlund & Montgomery), exact for every
// n < 2^32 and 1 <= d < 2^31.
// ----------------------------------------------------------------------------
struct FastDivU32 {
    uint32_t d, m, s;
    static FastDivU32 make(uint32_t d) {
        FastDivU32 f{d, 0u, 0u};
        if (d > 1) {
            uint32_t l = 0;
            while ((1ull << l) < d) ++l;                         // l = ceil(log2 d)
            f.m = (uint32_t)((((1ull << l) - d) << 32) / d + 1);
            f.s = l;
        }
        return f;
    }
    __device__ __forceinline__ uint32_t div(uint32_t n) const {
        if (d == 1) return n;
        const uint32_t t = __umulhi(n, m);
        return (t + ((n - t) >> 1)) >> (s - 1);
    }
};

// ----------------------------------------------------------------------------
// 1-D TMA (cp.async.bulk, SASS UBLKCP) + mbarrier helpers.  A bulk copy moves
// a 16-byte-aligned, 16-byte-multiple span global -> shared and signals the
// slot's mbarrier with complete_tx; the consumer waits on the barrier phase.
// ----------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_1d(void* smem_dst, const void* gsrc, uint32_t bytes,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(smem_dst)),
        "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void lds128(const void* p, uint32_t (&w)[4]) {
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3])
                 : "r"(smem_u32(p)));
}

}  // namespace tt
