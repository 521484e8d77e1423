// tools/tma_gather_lab.cu -- lab: can TMA gathers (cp.async.bulk.tensor.2d ... tile::gather4) get
// the PageRank gather past the L1 -> L2 request limit of ordinary loads (ncu: the L1 -> XBAR
// request path 89 % busy in k_pr_flag)?  The outbox is viewed as a 2D tensor [N/2][2] of f64:
// one gather4 fetches 4 rows of 16 bytes (the two values of each source's 16-byte pair) into
// shared memory.  Every warp walks 128-edge chunks; lane l takes edges 4l..4l+3 of a chunk,
// issues ONE gather4 for them, and reads its four values back after the mbarrier completes;
// kStages chunks in flight per warp.  Compared with the raw stream of ordinary loads (v0).
// Not product code.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

constexpr int kChunk = 128;
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ uint64_t pol_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t pol_range(const void* base, uint32_t hot, uint32_t total) {
    uint64_t p;
    asm volatile("createpolicy.range.global.L2::evict_last.L2::evict_first.b64 %0, [%1], %2, %3;"
                 : "=l"(p) : "l"(base), "r"(hot), "r"(total));
    return p;
}
__device__ __forceinline__ int ld_s(const int* p, uint64_t pol) {
    int r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ int4 ld_s4(const int4* p, uint64_t pol) {
    int4 r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
        : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ double ld_valp(const double* base, int u, uint64_t pol) {
    double r;
    asm("{\n\t.reg .pred q;\n\tsetp.lt.s32 q, %3, 8192;\n\t"
        "@q ld.global.nc.L1::evict_last.L2::cache_hint.f64 %0, [%1], %2;\n\t"
        "@!q ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;\n\t}"
        : "=d"(r) : "l"(base + u), "l"(pol), "r"(u));
    return r;
}
__device__ __forceinline__ uint32_t saddr(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

// raw stream (the product's gather policies), lane-strided edges, blocks of 64 chunks
__global__ void __launch_bounds__(256, 3) k_raw(const int* __restrict__ idx, int64_t E,
                                                const double* __restrict__ vals, uint32_t gtotal,
                                                double* out, int* ctr) {
    const int lane = threadIdx.x & 31;
    const uint64_t pol = pol_first();
    const uint64_t gp = pol_range(vals, 64u << 20, gtotal);
    const int64_t nch = (E + kChunk - 1) / kChunk;
    double acc = 0;
    for (;;) {
        int q = lane == 0 ? atomicAdd(ctr, 1) : 0;
        q = __shfl_sync(kFull, q, 0);
        const int64_t c0 = (int64_t)q * 64;
        if (c0 >= nch) break;
        const int64_t c1 = c0 + 64 < nch ? c0 + 64 : nch;
        int a[4], b[4];
        auto ld = [&](int64_t c, int (&r)[4]) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int64_t e = c * kChunk + 32 * k + lane;
                r[k] = (c < c1 && e < E) ? ld_s(idx + e, pol) : -1;
            }
        };
        ld(c0, a);
        ld(c0 + 1, b);
        double g[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) g[k] = a[k] >= 0 ? ld_valp(vals, a[k], gp) : 0.0;
        for (int64_t c = c0; c < c1; ++c) {
            double gn[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) gn[k] = b[k] >= 0 ? ld_valp(vals, b[k], gp) : 0.0;
            ld(c + 2, b);
            acc += (g[0] + g[1]) + (g[2] + g[3]);
#pragma unroll
            for (int k = 0; k < 4; ++k) g[k] = gn[k];
        }
    }
    out[(int64_t)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// TMA gather4: kStages chunks in flight per warp.  Shared: per warp kStages x 32 lanes x 64 B
// plus kStages mbarriers.  E is a multiple of 4 (the host pads the index array with source 0
// and subtracts its contribution).
template <int kStages>
__global__ void __launch_bounds__(256, 3) k_tma(const __grid_constant__ CUtensorMap tmap,
                                                const int* __restrict__ idx, int64_t E,
                                                double* out, int* ctr) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    // 128-byte slots (TMA destinations must be 128-byte aligned; a gather4 fills 64 bytes)
    double* buf = reinterpret_cast<double*>(smem) + (size_t)wid * kStages * 32 * 16;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 8 * kStages * 32 * 128) + wid * kStages;
    const uint64_t pol = pol_first();
    if (lane == 0)
        for (int s = 0; s < kStages; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(bars + s)), "r"(32));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    uint32_t phase = 0;   // bit s: parity of stage s
    const int64_t nch = (E + kChunk - 1) / kChunk;
    double acc = 0;
    // issue chunk c into stage s: lane l's 4 edges 128c + 4l .. +3
    auto issue = [&](int64_t c, int s, int4 u) {
        const uint32_t bar = saddr(bars + s);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(64)
                     : "memory");
        const uint32_t dst = saddr(buf + ((size_t)s * 32 + lane) * 16);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::"
            "bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
            "l"(&tmap), "r"(0), "r"(u.x >> 1), "r"(u.y >> 1), "r"(u.z >> 1), "r"(u.w >> 1),
            "r"(bar)
            : "memory");
        (void)c;
    };
    for (;;) {
        int q = lane == 0 ? atomicAdd(ctr, 1) : 0;
        q = __shfl_sync(kFull, q, 0);
        const int64_t c0 = (int64_t)q * 64;
        if (c0 >= nch) break;
        const int64_t c1 = c0 + 64 < nch ? c0 + 64 : nch;
        int4 U[kStages];
#pragma unroll
        for (int s = 0; s < kStages; ++s) {
            const int64_t c = c0 + s;
            if (c < c1) {
                U[s] = ld_s4(reinterpret_cast<const int4*>(idx + c * kChunk) + lane, pol);
                issue(c, s, U[s]);
            }
        }
        for (int64_t c = c0; c < c1; ++c) {
            const int s = (int)((c - c0) % kStages);
            const uint32_t bar = saddr(bars + s);
            const uint32_t par = (phase >> s) & 1u;
            asm volatile(
                "{\n\t.reg .pred p;\n"
                "W%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                "@!p bra W%=;\n\t}" ::"r"(bar),
                "r"(par)
                : "memory");
            phase ^= 1u << s;
            const int4 u = U[s];
            const double* v = buf + ((size_t)s * 32 + lane) * 16;   // 4 rows x 2 values
            acc += (v[0 + (u.x & 1)] + v[2 + (u.y & 1)]) + (v[4 + (u.z & 1)] + v[6 + (u.w & 1)]);
            __syncwarp();
            const int64_t cn = c + kStages;
            if (cn < c1) {
                U[s] = ld_s4(reinterpret_cast<const int4*>(idx + cn * kChunk) + lane, pol);
                issue(cn, s, U[s]);
            }
        }
    }
    out[(int64_t)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                             const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                             const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

extern "C" {
// variant 0 raw, 1.. TMA with stages {1, 2, 3}[variant - 1]; box_rows: tensor-map box height.
// Returns ms per pass (mean of reps) or a negative error code.
float run_tma_lab(int variant, const int* idx, int64_t E, const double* vals, int64_t n,
                  double* out, int* ctr, int box_rows, int l2promo, int reps) {
    static EncodeFn encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult qr;
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr) !=
                cudaSuccess || !fn)
            return -1.0f;
        encode = (EncodeFn)fn;
    }
    CUtensorMap tm;
    cuuint64_t gdim[2] = {2, (cuuint64_t)(n / 2)};
    cuuint64_t gstr[1] = {16};
    cuuint32_t box[2] = {2, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    const CUtensorMapL2promotion pr = l2promo == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                                     : (l2promo == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                                                     : CU_TENSOR_MAP_L2_PROMOTION_L2_128B);
    CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)vals, gdim, gstr, box,
                        estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, pr,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        printf("encode failed %d\n", (int)r);
        return -2.0f;
    }
    const int stages = variant == 1 ? 1 : (variant == 2 ? 2 : 3);
    const size_t shm = (size_t)8 * stages * 32 * 128 + 8 * 8 * stages;
    cudaFuncSetAttribute(k_tma<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024);
    cudaFuncSetAttribute(k_tma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024);
    cudaFuncSetAttribute(k_tma<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024);
    const uint32_t gtotal = (uint32_t)(n * 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float tot = 0;
    for (int i = 0; i <= reps; ++i) {
        cudaMemset(ctr, 0, 4);
        cudaEventRecord(a);
        if (variant == 0) k_raw<<<148 * 3, 256>>>(idx, E, vals, gtotal, out, ctr);
        else if (stages == 1) k_tma<1><<<148 * 3, 256, shm>>>(tm, idx, E, out, ctr);
        else if (stages == 2) k_tma<2><<<148 * 3, 256, shm>>>(tm, idx, E, out, ctr);
        else k_tma<3><<<148 * 3, 256, shm>>>(tm, idx, E, out, ctr);
        cudaEventRecord(b);
        if (cudaEventSynchronize(b) != cudaSuccess) {
            printf("kernel failed: %s\n", cudaGetErrorString(cudaGetLastError()));
            return -3.0f;
        }
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (i > 0) tot += ms;
    }
    return tot / reps;
}
}
