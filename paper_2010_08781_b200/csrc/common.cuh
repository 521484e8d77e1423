// paper_2010_08781_b200/csrc/common.cuh -- device helpers shared by the superstep kernels.
// sm_100a only (compiled with -gencode arch=compute_100a,code=sm_100a).
#pragma once
#ifdef __CUDACC_RTC__
// compiled at run time by NVRTC together with a user vertex program (program.cuh): no host
// headers are available there
typedef signed char int8_t;
typedef unsigned char uint8_t;
typedef short int16_t;
typedef unsigned short uint16_t;
typedef int int32_t;
typedef unsigned int uint32_t;
typedef long long int64_t;
typedef unsigned long long uint64_t;
#ifndef INT_MAX
#define INT_MAX 2147483647
#endif
#else
#include <climits>
#include <cstdint>
#include <cuda_runtime.h>
#endif

namespace ipr {

constexpr uint32_t kInf = 0xFFFFFFFFu;
constexpr unsigned kFull = 0xFFFFFFFFu;

// L2 cache policies (PTX createpolicy).  Index/weight streams are read once per superstep and
// marked evict-first so they do not push the gathered outbox values out of L2.
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ uint64_t policy_evict_normal() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// Address-range policy: the first `hot` bytes of [base, base + total) evict-last, the rest
// evict-first (vertex arrays whose ids are sorted by descending degree keep their hot prefix).
__device__ __forceinline__ uint64_t policy_range(const void* base, uint32_t hot, uint32_t total) {
    uint64_t p;
    asm volatile("createpolicy.range.global.L2::evict_last.L2::evict_first.b64 %0, [%1], %2, %3;"
                 : "=l"(p) : "l"(base), "r"(hot), "r"(total));
    return p;
}
// Gather policy selector (tuning knob, IPREGEL_GATHER_POLICY): 0 evict_normal, 1 evict_last,
// 2 evict_first, 3 range (hot prefix evict_last).
__device__ __forceinline__ uint64_t policy_for(int mode, const void* base = nullptr,
                                               uint32_t hot = 0, uint32_t total = 0) {
    if (mode == 3 && base) return policy_range(base, hot < total ? hot : total, total);
    return mode == 1 ? policy_evict_last() : (mode == 2 ? policy_evict_first() : policy_evict_normal());
}

// Compile-time variants (tuning builds): IPREGEL_GATHER_HINT 1 = gathers carry the L2 policy
// operand, 0 = plain ld.global.nc; IPREGEL_STREAM_CS 1 = index stream uses ld.global.cs (evict
// first without a policy operand), 0 = L2::cache_hint evict_first policy.
#ifndef IPREGEL_GATHER_HINT
#define IPREGEL_GATHER_HINT 1
#endif
#ifndef IPREGEL_STREAM_CS
#define IPREGEL_STREAM_CS 0
#endif

// Streamed (read-once) loads: non-coherent path, no L1 allocation, L2 evict-first.
__device__ __forceinline__ int32_t ld_stream(const int32_t* p, uint64_t pol) {
    int32_t r;
#if IPREGEL_STREAM_CS
    (void)pol;
    asm("ld.global.cs.s32 %0, [%1];" : "=r"(r) : "l"(p));
#else
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;"
                 : "=r"(r) : "l"(p), "l"(pol));
#endif
    return r;
}
__device__ __forceinline__ uint32_t ld_stream(const uint32_t* p, uint64_t pol) {
    uint32_t r;
#if IPREGEL_STREAM_CS
    (void)pol;
    asm("ld.global.cs.u32 %0, [%1];" : "=r"(r) : "l"(p));
#else
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
                 : "=r"(r) : "l"(p), "l"(pol));
#endif
    return r;
}
__device__ __forceinline__ int4 ld_stream4(const int4* p, uint64_t pol) {
    int4 r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p), "l"(pol));
    return r;
}

// Gathered outbox values (random access, reused across the superstep): read-only path with an
// explicit L2 policy.
__device__ __forceinline__ double ld_gather(const double* p, uint64_t pol) {
    double r;
#if IPREGEL_GATHER_HINT
    asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(p), "l"(pol));
#else
    (void)pol;
    asm("ld.global.nc.f64 %0, [%1];" : "=d"(r) : "l"(p));
#endif
    return r;
}
__device__ __forceinline__ uint32_t ld_gather(const uint32_t* p, uint64_t pol) {
    uint32_t r;
#if IPREGEL_GATHER_HINT
    asm("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
#else
    (void)pol;
    asm("ld.global.nc.u32 %0, [%1];" : "=r"(r) : "l"(p));
#endif
    return r;
}

// Gather with an L1 choice: hot (L1 evict-last) or cold (no L1 allocation) per lane.
__device__ __forceinline__ double ld_gather_l1(const double* p, uint64_t pol, int hot) {
    double r;
#if !IPREGEL_GATHER_HINT
    (void)pol;
    asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t"
        "@q ld.global.nc.L1::evict_last.f64 %0, [%1];\n\t"
        "@!q ld.global.nc.L1::no_allocate.f64 %0, [%1];\n\t}"
        : "=d"(r) : "l"(p), "r"(hot));
    return r;
#endif
    asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\t"
        "@q ld.global.nc.L1::evict_last.L2::cache_hint.f64 %0, [%1], %2;\n\t"
        "@!q ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;\n\t}"
        : "=d"(r) : "l"(p), "l"(pol), "r"(hot));
    return r;
}
__device__ __forceinline__ uint32_t ld_gather_l1(const uint32_t* p, uint64_t pol, int hot) {
    uint32_t r;
#if !IPREGEL_GATHER_HINT
    (void)pol;
    asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t"
        "@q ld.global.nc.L1::evict_last.u32 %0, [%1];\n\t"
        "@!q ld.global.nc.L1::no_allocate.u32 %0, [%1];\n\t}"
        : "=r"(r) : "l"(p), "r"(hot));
    return r;
#endif
    asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\t"
        "@q ld.global.nc.L1::evict_last.L2::cache_hint.u32 %0, [%1], %2;\n\t"
        "@!q ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;\n\t}"
        : "=r"(r) : "l"(p), "l"(pol), "r"(hot));
    return r;
}

// Same-size bit reinterpretation (no <cstring> under NVRTC).
template <class To, class From>
__device__ __forceinline__ To bit_cast(From f) {
    static_assert(sizeof(To) == sizeof(From), "same size");
    union {
        From f;
        To t;
    } u;
    u.f = f;
    return u.t;
}
template <bool B, class X, class Y> struct cond_type { using type = X; };
template <class X, class Y> struct cond_type<false, X, Y> { using type = Y; };

// Any other 4- or 8-byte value type (user programs: f32, i32, u64, i64) through the u32 / f64
// paths by bit pattern.
template <class T>
__device__ __forceinline__ T ld_gather(const T* p, uint64_t pol) {
    static_assert(sizeof(T) == 4 || sizeof(T) == 8, "4- or 8-byte values");
    T r;
    if constexpr (sizeof(T) == 8) {
        r = bit_cast<T>(ld_gather(reinterpret_cast<const double*>(p), pol));
    } else {
        r = bit_cast<T>(ld_gather(reinterpret_cast<const uint32_t*>(p), pol));
    }
    return r;
}
template <class T>
__device__ __forceinline__ T ld_gather_l1(const T* p, uint64_t pol, int hot) {
    static_assert(sizeof(T) == 4 || sizeof(T) == 8, "4- or 8-byte values");
    T r;
    if constexpr (sizeof(T) == 8) {
        r = bit_cast<T>(ld_gather_l1(reinterpret_cast<const double*>(p), pol, hot));
    } else {
        r = bit_cast<T>(ld_gather_l1(reinterpret_cast<const uint32_t*>(p), pol, hot));
    }
    return r;
}

// Predicated gather (no branch): returns `fallback` bits when pred == 0.
__device__ __forceinline__ double ld_gather_pred(const double* p, uint64_t pol, int pred) {
    double r;
    asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\tmov.b64 %0, 0;\n\t"
        "@q ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;\n\t}"
        : "=d"(r) : "l"(p), "l"(pol), "r"(pred));
    return r;
}
__device__ __forceinline__ uint32_t ld_gather_pred(const uint32_t* p, uint64_t pol, int pred) {
    uint32_t r;
    asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\tmov.b32 %0, 0;\n\t"
        "@q ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;\n\t}"
        : "=r"(r) : "l"(p), "l"(pol), "r"(pred));
    return r;
}

// Saturating u32 add: INF + w = INF (reading R9).
__device__ __forceinline__ uint32_t sat_add(uint32_t a, uint32_t b) {
    uint32_t s = a + b;
    return s < a ? kInf : s;
}

template <class T>
__device__ __forceinline__ T shfl_up(T v, int d) { return __shfl_up_sync(kFull, v, d); }
template <class T>
__device__ __forceinline__ T shfl_xor(T v, int d) { return __shfl_xor_sync(kFull, v, d); }
template <class T>
__device__ __forceinline__ T shfl_idx(T v, int src) { return __shfl_sync(kFull, v, src); }

}  // namespace ipr
