// tools/gather_lab.cu -- microbenchmarks of the PageRank gather stream (acc += vals[idx[e]]) on
// the cfg4 CSC, to find what bounds it: the same loop as tools/gather_ceiling.cu with the hot
// prefix of the (degree-ordered) value array served from shared memory (v=1) or pinned in L1 with
// evict-last while the rest bypasses L1 (v=2).  Not product code.
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
__device__ __forceinline__ double ld_l1(const double* p, int hot) {
    double r;
    asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t"
        "@q ld.global.nc.L1::evict_last.f64 %0, [%1];\n\t"
        "@!q ld.global.nc.L1::no_allocate.f64 %0, [%1];\n\t}"
        : "=d"(r) : "l"(p), "r"(hot));
    return r;
}

template <int V>
__device__ __forceinline__ double get(const double* __restrict__ vals, const double* s, int u, int H) {
    if (V == 1) return u < H ? s[u] : __ldg(vals + u);
    if (V == 2) return ld_l1(vals + u, u < H);
    return __ldg(vals + u);
}

template <int V>
__global__ void k_lab(const int* __restrict__ idx, int64_t e, const double* __restrict__ vals,
                      int H, double* __restrict__ out) {
    extern __shared__ double s_hot[];
    if (V == 1) {
        for (int i = threadIdx.x; i < H; i += blockDim.x) s_hot[i] = vals[i];
        __syncthreads();
    }
    const uint64_t pol = pol_first();
    double acc = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < e; i += 4 * stride) {
        const int a = ld_idx(idx + i, pol), b = ld_idx(idx + i + stride, pol);
        const int c = ld_idx(idx + i + 2 * stride, pol), d = ld_idx(idx + i + 3 * stride, pol);
        const double va = get<V>(vals, s_hot, a, H), vb = get<V>(vals, s_hot, b, H);
        const double vc = get<V>(vals, s_hot, c, H), vd = get<V>(vals, s_hot, d, H);
        acc += (va + vb) + (vc + vd);
    }
    for (; i < e; i += stride) acc += get<V>(vals, s_hot, ld_idx(idx + i, pol), H);
    out[(int64_t)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void k_count_below(const int* __restrict__ idx, int64_t e, int H,
                              unsigned long long* cnt) {
    unsigned long long c = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < e;
         i += (int64_t)gridDim.x * blockDim.x)
        c += idx[i] < H;
    atomicAdd(cnt, c);
}

extern "C" double count_below(const int* idx, int64_t e, int H) {
    unsigned long long* d;
    cudaMalloc(&d, 8);
    cudaMemset(d, 0, 8);
    k_count_below<<<148 * 8, 256>>>(idx, e, H, d);
    unsigned long long h = 0;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    cudaFree(d);
    return (double)h / (double)e;
}

extern "C" float gather_lab(int variant, const int* idx, int64_t e, const double* vals, int H,
                            double* out, int blocks, int threads, int reps) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const size_t smem = variant == 1 ? (size_t)H * 8 : 0;
    if (variant == 1)
        cudaFuncSetAttribute(k_lab<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(a);
        if (variant == 1) k_lab<1><<<blocks, threads, smem>>>(idx, e, vals, H, out);
        else if (variant == 2) k_lab<2><<<blocks, threads>>>(idx, e, vals, H, out);
        else k_lab<0><<<blocks, threads>>>(idx, e, vals, H, out);
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
