// tools/split_lab.cu -- ceiling of a hot/cold split of the PageRank gather on the cfg4 CSC
// (degree-ordered): the raw gather stream acc += vals[idx[e]] over (a) every edge, (b) only the
// edges whose source is >= H (the "cold" kernel, full L1 for misses in flight), (c) only the
// edges whose source is < H, served from a shared-memory copy of vals[0, H) (the "hot" kernel;
// int32 or uint16 indices).  Plus a counter of distinct 128-byte lines per warp instruction
// (32 consecutive edges), the L1 -> L2 request count the gather issues.  Not product code.
#include <cuda_runtime.h>
#include <cstdint>

__device__ __forceinline__ uint64_t pol_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ int ld_idx(const int* p, uint64_t pol) {
    int r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ unsigned ld_idx16(const unsigned short* p, uint64_t pol) {
    unsigned short r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u16 %0, [%1], %2;" : "=h"(r) : "l"(p), "l"(pol));
    return r;
}

// warp-contiguous layout like the pull kernel: a warp reads 32 consecutive edges per load
__global__ void k_raw(const int* __restrict__ idx, int64_t e, const double* __restrict__ vals,
                      double* __restrict__ out) {
    const uint64_t pol = pol_first();
    double acc = 0;
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    // each warp takes 128-edge chunks
    for (int64_t c = w * 128; c < e; c += nw * 128) {
        int a[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int64_t i = c + 32 * k + lane;
            a[k] = i < e ? ld_idx(idx + i, pol) : -1;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) acc += a[k] >= 0 ? __ldg(vals + a[k]) : 0.0;
    }
    out[(int64_t)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <class I>
__global__ void k_hot(const I* __restrict__ idx, int64_t e, const double* __restrict__ vals, int H,
                      double* __restrict__ out) {
    extern __shared__ double s_hot[];
    for (int i = threadIdx.x; i < H; i += blockDim.x) s_hot[i] = vals[i];
    __syncthreads();
    const uint64_t pol = pol_first();
    double acc = 0;
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    for (int64_t c = w * 256; c < e; c += nw * 256) {
        unsigned a[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int64_t i = c + 32 * k + lane;
            if (sizeof(I) == 2) a[k] = i < e ? ld_idx16((const unsigned short*)idx + i, pol) : 0xFFFFFFFFu;
            else a[k] = i < e ? (unsigned)ld_idx((const int*)idx + i, pol) : 0xFFFFFFFFu;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) acc += a[k] != 0xFFFFFFFFu ? s_hot[a[k]] : 0.0;
    }
    out[(int64_t)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// distinct (idx >> shift) per aligned group of 32 edges, counting changes between neighbours
// (rows are sorted, so within a row this is exact; across row ends it may overcount a revisit)
__global__ void k_lines(const int* __restrict__ idx, int64_t e, int shift,
                        unsigned long long* cnt) {
    unsigned long long c = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < e;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int l = idx[i] >> shift;
        c += (i & 31) == 0 || (idx[i - 1] >> shift) != l;
    }
    atomicAdd(cnt, c);
}

extern "C" double lines_per_edge(const int* idx, int64_t e, int shift) {
    unsigned long long* d;
    cudaMalloc(&d, 8);
    cudaMemset(d, 0, 8);
    k_lines<<<148 * 8, 256>>>(idx, e, shift, d);
    unsigned long long h = 0;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    cudaFree(d);
    return (double)h / (double)e;
}

static float timeit(int variant, const void* idx, int64_t e, const double* vals, int H,
                    double* out, int blocks, int threads, int reps) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const size_t smem = (size_t)H * 8;
    if (variant == 1) cudaFuncSetAttribute(k_hot<int>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (variant == 2) cudaFuncSetAttribute(k_hot<unsigned short>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(a);
        if (variant == 0) k_raw<<<blocks, threads>>>((const int*)idx, e, vals, out);
        else if (variant == 1) k_hot<int><<<blocks, threads, smem>>>((const int*)idx, e, vals, H, out);
        else k_hot<unsigned short><<<blocks, threads, smem>>>((const unsigned short*)idx, e, vals, H, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return cudaGetLastError() == cudaSuccess ? best : -1.0f;
}

extern "C" float split_lab(int variant, const void* idx, int64_t e, const double* vals, int H,
                           double* out, int blocks, int threads, int reps) {
    return timeit(variant, idx, e, vals, H, out, blocks, threads, reps);
}
