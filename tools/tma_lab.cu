// tools/tma_lab.cu -- lab: memory pipeline of the PageRank range kernel without its row logic.
// Every warp walks 128-edge chunks of an index array (the cold CSC), summing vals[idx[e]]:
//   v0: indices in registers two chunks ahead, gathers one chunk ahead (the range kernel's
//       pipeline), at a chosen number of resident warps per SM;
//   v1: indices staged in shared memory by 1D bulk copies (cp.async.bulk + mbarrier, TMA
//       engine: no registers, no L1 tag lookups) kSlots chunks ahead, gathers one chunk ahead;
//   v2: as v1 with gathers two chunks ahead.
// Not product code.
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
__device__ __forceinline__ double ld_val(const double* p) {
    double r;
    asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count));
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                          uint64_t pol) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], "
        "[%1], %2, [%3], %4;" ::"r"(smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W;\n\t}" ::"r"(smem_addr(b)),
        "r"(parity)
        : "memory");
}

constexpr int kChunk = 128;

template <int kBlk>
__global__ void __launch_bounds__(256) k_v0(const int* __restrict__ idx, int64_t nchunks,
                                            const double* __restrict__ vals, double* out,
                                            int* ctr) {
    const int lane = threadIdx.x & 31;
    const uint64_t pol = pol_first();
    double acc = 0;
    // each warp takes blocks of 64 chunks from the counter
    for (;;) {
        int q = lane == 0 ? atomicAdd(ctr, 1) : 0;
        q = __shfl_sync(0xffffffffu, q, 0);
        const int64_t c0 = (int64_t)q * kBlk;
        if (c0 >= nchunks) break;
        const int64_t c1 = c0 + kBlk < nchunks ? c0 + kBlk : nchunks;
        int a[4], b[4];
        double g[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) a[k] = ld_idx(idx + c0 * kChunk + 32 * k + lane, pol);
#pragma unroll
        for (int k = 0; k < 4; ++k)
            b[k] = c0 + 1 < c1 ? ld_idx(idx + (c0 + 1) * kChunk + 32 * k + lane, pol) : 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) g[k] = ld_val(vals + a[k]);
        for (int64_t c = c0; c < c1; ++c) {
            double gn[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) gn[k] = c + 1 < c1 ? ld_val(vals + b[k]) : 0.0;
#pragma unroll
            for (int k = 0; k < 4; ++k)
                b[k] = c + 2 < c1 ? ld_idx(idx + (c + 2) * kChunk + 32 * k + lane, pol) : 0;
            acc += (g[0] + g[1]) + (g[2] + g[3]);
#pragma unroll
            for (int k = 0; k < 4; ++k) g[k] = gn[k];
        }
    }
    out[(int64_t)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int kSlots, int kAhead>
__global__ void __launch_bounds__(256) k_v1(const int* __restrict__ idx, int64_t nchunks,
                                            const double* __restrict__ vals, double* out,
                                            int* ctr) {
    __shared__ __align__(128) int s_idx[8][kSlots][kChunk];
    __shared__ __align__(8) uint64_t s_bar[8][kSlots];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint64_t pol = pol_first();
    if (lane == 0)
        for (int i = 0; i < kSlots; ++i) mbar_init(&s_bar[wid][i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    uint32_t phase[kSlots];
#pragma unroll
    for (int i = 0; i < kSlots; ++i) phase[i] = 0;
    double acc = 0;
    for (;;) {
        int q = lane == 0 ? atomicAdd(ctr, 1) : 0;
        q = __shfl_sync(0xffffffffu, q, 0);
        const int64_t c0 = (int64_t)q * 64;
        if (c0 >= nchunks) break;
        const int64_t c1 = c0 + 64 < nchunks ? c0 + 64 : nchunks;
        // prologue: slots for chunks c0 .. c0 + kSlots - 1
        if (lane == 0)
            for (int i = 0; i < kSlots; ++i)
                if (c0 + i < c1)
                    bulk_load(s_idx[wid][i], idx + (c0 + i) * kChunk, kChunk * 4, &s_bar[wid][i], pol);
        double g[kAhead][4];
#pragma unroll
        for (int a = 0; a < kAhead; ++a) {
            const int64_t c = c0 + a;
            if (c < c1) {
                mbar_wait(&s_bar[wid][a], phase[a]);
                phase[a] ^= 1;
#pragma unroll
                for (int k = 0; k < 4; ++k) g[a][k] = ld_val(vals + s_idx[wid][a][32 * k + lane]);
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) g[a][k] = 0.0;
            }
        }
        __syncwarp();
        // refill consumed slots
        if (lane == 0)
            for (int a = 0; a < kAhead; ++a)
                if (c0 + a + kSlots < c1)
                    bulk_load(s_idx[wid][a], idx + (c0 + a + kSlots) * kChunk, kChunk * 4,
                              &s_bar[wid][a], pol);
        for (int64_t c = c0; c < c1; ++c) {
            // issue the gathers of chunk c + kAhead
            const int64_t cn = c + kAhead;
            const int sl = (int)(cn % kSlots);
            double gn[4];
            if (cn < c1) {
                mbar_wait(&s_bar[wid][sl], phase[sl]);
                phase[sl] ^= 1;
#pragma unroll
                for (int k = 0; k < 4; ++k) gn[k] = ld_val(vals + s_idx[wid][sl][32 * k + lane]);
                __syncwarp();
                if (lane == 0 && cn + kSlots < c1)
                    bulk_load(s_idx[wid][sl], idx + (cn + kSlots) * kChunk, kChunk * 4,
                              &s_bar[wid][sl], pol);
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) gn[k] = 0.0;
            }
            acc += (g[0][0] + g[0][1]) + (g[0][2] + g[0][3]);
#pragma unroll
            for (int a = 0; a + 1 < kAhead; ++a)
#pragma unroll
                for (int k = 0; k < 4; ++k) g[a][k] = g[a + 1][k];
#pragma unroll
            for (int k = 0; k < 4; ++k) g[kAhead - 1][k] = gn[k];
        }
    }
    out[(int64_t)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// v5..: indices kD chunks ahead in a register ring, gathers one chunk ahead
template <int kBlk, int kD>
__global__ void __launch_bounds__(256) k_vd(const int* __restrict__ idx, int64_t nchunks,
                                            const double* __restrict__ vals, double* out,
                                            int* ctr) {
    const int lane = threadIdx.x & 31;
    const uint64_t pol = pol_first();
    double acc = 0;
    for (;;) {
        int q = lane == 0 ? atomicAdd(ctr, 1) : 0;
        q = __shfl_sync(0xffffffffu, q, 0);
        const int64_t c0 = (int64_t)q * kBlk;
        if (c0 >= nchunks) break;
        const int64_t c1 = c0 + kBlk < nchunks ? c0 + kBlk : nchunks;
        int ring[kD][4];
#pragma unroll
        for (int d = 0; d < kD; ++d)
#pragma unroll
            for (int k = 0; k < 4; ++k)
                ring[d][k] = c0 + d < c1 ? ld_idx(idx + (c0 + d) * kChunk + 32 * k + lane, pol) : 0;
        double g[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) g[k] = ld_val(vals + ring[0][k]);
        for (int64_t c = c0; c < c1; ++c) {
            double gn[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) gn[k] = c + 1 < c1 ? ld_val(vals + ring[1][k]) : 0.0;
#pragma unroll
            for (int d = 0; d + 1 < kD; ++d)
#pragma unroll
                for (int k = 0; k < 4; ++k) ring[d][k] = ring[d + 1][k];
#pragma unroll
            for (int k = 0; k < 4; ++k)
                ring[kD - 1][k] = c + kD < c1 ? ld_idx(idx + (c + kD) * kChunk + 32 * k + lane, pol) : 0;
            acc += (g[0] + g[1]) + (g[2] + g[3]);
#pragma unroll
            for (int k = 0; k < 4; ++k) g[k] = gn[k];
        }
    }
    out[(int64_t)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <class F>
static float timeit(F launch, int* ctr, int reps) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        cudaMemset(ctr, 0, 4);
        cudaEventRecord(a);
        launch();
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

// ctas_per_sm: resident CTAs of 256 threads per SM (a grid of exactly that many per SM)
extern "C" float tma_lab(int variant, const int* idx, int64_t e, const double* vals, double* out,
                         int* ctr, int ctas_per_sm, int reps) {
    const int64_t nchunks = e / kChunk;   // the tail is ignored (a lab)
    const int grid = 148 * ctas_per_sm;
    const size_t pad = 0;   // residency: the grid is ctas_per_sm waves of 148 (one each)
    switch (variant) {
        case 0:
            return timeit([&] { k_v0<64><<<grid, 256, pad>>>(idx, nchunks, vals, out, ctr); }, ctr, reps);
        case 1:
            return timeit([&] { k_v0<16><<<grid, 256, pad>>>(idx, nchunks, vals, out, ctr); }, ctr, reps);
        case 2:
            return timeit([&] { k_v0<4><<<grid, 256, pad>>>(idx, nchunks, vals, out, ctr); }, ctr, reps);
        case 3:
            return timeit([&] { k_v0<2><<<grid, 256, pad>>>(idx, nchunks, vals, out, ctr); }, ctr, reps);
        case 4:
            return timeit([&] { k_v0<256><<<grid, 256, pad>>>(idx, nchunks, vals, out, ctr); }, ctr, reps);
        case 5:
            return timeit([&] { k_vd<64, 2><<<grid, 256, pad>>>(idx, nchunks, vals, out, ctr); }, ctr, reps);
        case 6:
            return timeit([&] { k_vd<64, 3><<<grid, 256, pad>>>(idx, nchunks, vals, out, ctr); }, ctr, reps);
        case 7:
            return timeit([&] { k_vd<64, 4><<<grid, 256, pad>>>(idx, nchunks, vals, out, ctr); }, ctr, reps);
        case 8:
            return timeit([&] { k_vd<64, 6><<<grid, 256, pad>>>(idx, nchunks, vals, out, ctr); }, ctr, reps);
        default:
            return -2.0f;
    }
}
