// tools/dsmem_lab.cu -- microbenchmark: the PageRank gather stream (acc += vals[idx[e]]) with the
// hottest H sources (degree order) held in the distributed shared memory of a thread-block
// cluster (each of the C CTAs holds H / C of them; a gather of a hot source is an
// ld.shared::cluster from the owning CTA, everything else a global load).  Persistent grid:
// clusters of C CTAs, one CTA per SM.  Not product code.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace cg = cooperative_groups;

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

template <int MODE>   // 0: no hot cache; 1: hot set in the cluster's DSMEM
__global__ void k_dsmem(const int* __restrict__ idx, int64_t e, const double* __restrict__ vals,
                        int per_cta, double* __restrict__ out) {
    extern __shared__ double s_hot[];
    cg::cluster_group cluster = cg::this_cluster();
    const int C = (int)cluster.num_blocks();
    const int rank = (int)cluster.block_rank();
    if (MODE == 1) {
        for (int i = threadIdx.x; i < per_cta; i += blockDim.x) s_hot[i] = vals[rank * per_cta + i];
        cluster.sync();
    }
    const int H = per_cta * C;
    const uint64_t pol = pol_first();
    double acc = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < e; i += stride) {
        const int u = ld_idx(idx + i, pol);
        double v;
        if (MODE == 1 && u < H) {
            const double* remote = cluster.map_shared_rank(s_hot, u / per_cta);
            v = remote[u % per_cta];
        } else {
            v = __ldg(vals + u);
        }
        acc += v;
    }
    out[(int64_t)blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (MODE == 1) cluster.sync();   // nobody leaves while others may read its shared memory
}

extern "C" float dsmem_lab(int mode, const int* idx, int64_t e, const double* vals, int per_cta,
                           int cluster, int ctas, int threads, double* out, int reps) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ctas);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = mode == 1 ? (size_t)per_cta * 8 : 0;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    auto k = mode == 1 ? k_dsmem<1> : k_dsmem<0>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cfg.dynamicSmemBytes);
    if (cluster > 8) cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(a);
        cudaLaunchKernelEx(&cfg, k, idx, e, vals, per_cta, out);
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
