// tools/gather_ceiling.cu -- microbenchmark: the raw cost of the PageRank pull's memory stream
// without any row logic.  For every edge e: acc += vals[idx[e]] (f64 or u32 values), indices
// streamed with the same L2 evict-first hint, one partial per thread written at the end.
// This bounds what any pull kernel over the same CSC can reach on this GPU.
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

template <class T>
__global__ void __launch_bounds__(256) k_gather(const int* __restrict__ idx, int64_t e,
                                                const T* __restrict__ vals, T* __restrict__ out) {
    const uint64_t pol = pol_first();
    T acc = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < e; i += 4 * stride) {
        const int a = ld_idx(idx + i, pol), b = ld_idx(idx + i + stride, pol);
        const int c = ld_idx(idx + i + 2 * stride, pol), d = ld_idx(idx + i + 3 * stride, pol);
        const T va = __ldg(vals + a), vb = __ldg(vals + b), vc = __ldg(vals + c), vd = __ldg(vals + d);
        acc += (va + vb) + (vc + vd);
    }
    for (; i < e; i += stride) acc += __ldg(vals + ld_idx(idx + i, pol));
    out[(int64_t)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

extern "C" float gather_ceiling(const int* idx, int64_t e, const void* vals, int f64, void* out,
                                int blocks, int reps) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(a);
        if (f64) k_gather<double><<<blocks, 256>>>(idx, e, (const double*)vals, (double*)out);
        else k_gather<uint32_t><<<blocks, 256>>>(idx, e, (const uint32_t*)vals, (uint32_t*)out);
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
