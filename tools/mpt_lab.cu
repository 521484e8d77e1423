// tools/mpt_lab.cu -- lab: a per-LANE merge-path walk (Merrill & Garland's merge-based CSR
// SpMV at thread granularity) for the PageRank gather, on the cold and hot parts of the cfg4 CSC.
// Each warp takes a range of kRange merge items (row ends + edges); lane l walks items
// [l * kRange / 32, (l + 1) * kRange / 32) of it sequentially: edges add into a register sum,
// a row end stores the sum (partial rows at lane boundaries are ignored here -- a lab of the
// cost, not a product kernel).  Gathers from global memory (cold) or from a shared-memory copy
// of vals[0, H) (hot).  Not product code.
#include <cuda_runtime.h>
#include <cstdint>

__device__ __forceinline__ uint64_t pol_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ int ld_idx(const int* p, uint64_t pol) {
    int r;
    asm("ld.global.nc.L1::evict_first.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ int ld_off(const int* p) {
    int r;
    asm("ld.global.nc.s32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ double ld_val(const double* p) {
    double r;
    asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r) : "l"(p));
    return r;
}

template <int kRange, int kBatch, bool kStaged>
__global__ void __launch_bounds__(1024) k_mpt(const int* __restrict__ off, int rows, int64_t edges,
                                             const int* __restrict__ idx,
                                             const double* __restrict__ vals, int H,
                                             double* __restrict__ out, int* __restrict__ ctr,
                                             int num_ranges) {
    extern __shared__ double s_hot[];
    if (kStaged) {
        for (int i = threadIdx.x; i < H; i += blockDim.x) s_hot[i] = vals[i];
        __syncthreads();
    }
    const int lane = threadIdx.x & 31;
    const uint64_t pol = pol_first();
    constexpr int K = kRange / 32;
    const int64_t total = (int64_t)rows + edges;
    for (;;) {
        int q = lane == 0 ? atomicAdd(ctr, 1) : 0;
        q = __shfl_sync(0xffffffffu, q, 0);
        if (q >= num_ranges) break;
        int64_t d = (int64_t)q * kRange + (int64_t)lane * K;
        if (d >= total) continue;
        int64_t dend = d + K < total ? d + K : total;
        // diagonal search: r = rows finished before diagonal d
        int64_t lo = d - edges > 0 ? d - edges : 0, hi = d < rows ? d : rows;
        while (lo < hi) {
            const int64_t m = (lo + hi) >> 1;
            if ((int64_t)ld_off(off + m + 1) <= d - m - 1) lo = m + 1; else hi = m;
        }
        int r = (int)lo;
        int e = (int)(d - lo);
        int items = (int)(dend - d);
        double sum = 0.0;
        int rend = r < rows ? ld_off(off + r + 1) : (int)edges;
        while (items > 0) {
            int ne = rend - e;
            if (ne > items) ne = items;
            // edges of row r in this lane's share, in batches
            int j = 0;
            for (; j + kBatch <= ne; j += kBatch) {
                int u[kBatch];
#pragma unroll
                for (int b = 0; b < kBatch; ++b) u[b] = ld_idx(idx + e + j + b, pol);
                double v[kBatch];
#pragma unroll
                for (int b = 0; b < kBatch; ++b) v[b] = kStaged ? s_hot[u[b]] : ld_val(vals + u[b]);
#pragma unroll
                for (int b = 0; b < kBatch; ++b) sum += v[b];
            }
            for (; j < ne; ++j) {
                const int u = ld_idx(idx + e + j, pol);
                sum += kStaged ? s_hot[u] : ld_val(vals + u);
            }
            e += ne;
            items -= ne;
            if (items == 0) break;
            // row end
            out[r] = sum;
            sum = 0.0;
            ++r;
            --items;
            rend = r < rows ? ld_off(off + r + 1) : (int)edges;
        }
    }
}

template <int kRange, int kBatch, bool kStaged>
static float run(const int* off, int rows, int64_t edges, const int* idx, const double* vals,
                 int H, double* out, int* ctr, int blocks, int threads, int reps) {
    const int64_t total = (int64_t)rows + edges;
    const int num_ranges = (int)((total + kRange - 1) / kRange);
    const size_t smem = kStaged ? (size_t)H * 8 : 0;
    if (kStaged)
        cudaFuncSetAttribute(k_mpt<kRange, kBatch, kStaged>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int i = 0; i < reps; ++i) {
        cudaMemset(ctr, 0, 4);
        cudaEventRecord(a);
        k_mpt<kRange, kBatch, kStaged><<<blocks, threads, smem>>>(off, rows, edges, idx, vals, H, out,
                                                             ctr, num_ranges);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return cudaGetLastError() == cudaSuccess ? best : -1.0f;
}

extern "C" float mpt_lab(int variant, const int* off, int rows, int64_t edges, const int* idx,
                         const double* vals, int H, double* out, int* ctr, int blocks, int threads,
                         int reps) {
    switch (variant) {
        case 0: return run<4096, 4, false>(off, rows, edges, idx, vals, H, out, ctr, blocks, threads, reps);
        case 1: return run<4096, 8, false>(off, rows, edges, idx, vals, H, out, ctr, blocks, threads, reps);
        case 2: return run<8192, 8, false>(off, rows, edges, idx, vals, H, out, ctr, blocks, threads, reps);
        case 3: return run<2048, 4, false>(off, rows, edges, idx, vals, H, out, ctr, blocks, threads, reps);
        case 10: return run<4096, 4, true>(off, rows, edges, idx, vals, H, out, ctr, blocks, threads, reps);
        case 11: return run<4096, 8, true>(off, rows, edges, idx, vals, H, out, ctr, blocks, threads, reps);
        case 12: return run<2048, 4, true>(off, rows, edges, idx, vals, H, out, ctr, blocks, threads, reps);
        default: return -2.0f;
    }
}
