// inputs/rmat_gpu.cu -- seeded synthetic R-MAT graphs on the GPU (GPU twin of rmat_cpu.c) and
// the CSR / CSC arrays that ipregel_graph_create takes.
//
// INPUT GENERATION ONLY: no superstep, no combiner, no vertex program.  The edge definition is
// the one in the header of inputs/rmat_cpu.c (same splitmix64 counters, same thresholds, same
// MSB-first quadrant bits, same weights, self-loops dropped, slot order and duplicates kept);
// tests/test_inputs_gpu.py checks the two twins hash-equal.
//
// CSR/CSC layout: offsets int32 [N+1]; within a row neighbours ascend by (neighbour id, weight)
// so the arrays are deterministic.  Built by a counting scatter (atomic cursor per row) and a
// per-row sort (cub::DeviceSegmentedSort) -- fixture code, outside every timed region.
#include <cuda_runtime.h>
#include <cub/cub.cuh>
#include <cstdint>
#include <cstdio>

namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

struct Gen {
    uint64_t key, key_w;
    int scale;
    uint32_t ta, tab, tabc;
    __device__ __forceinline__ void edge(uint64_t i, uint32_t& s, uint32_t& d) const {
        uint32_t src = 0, dst = 0;
        uint64_t h = 0;
        for (int l = 0; l < scale; ++l) {
            if ((l & 1) == 0) h = splitmix64(key + 32ULL * i + (uint64_t)(l >> 1));
            const uint32_t r = (l & 1) ? (uint32_t)(h >> 32) : (uint32_t)h;
            uint32_t qs, qd;
            if (r < ta) { qs = 0; qd = 0; }
            else if (r < tab) { qs = 0; qd = 1; }
            else if (r < tabc) { qs = 1; qd = 0; }
            else { qs = 1; qd = 1; }
            src |= qs << (scale - 1 - l);
            dst |= qd << (scale - 1 - l);
        }
        s = src;
        d = dst;
    }
    __device__ __forceinline__ uint32_t weight(uint64_t i) const {
        return 1u + (uint32_t)(splitmix64(key_w + i) >> 58);
    }
};

Gen make_gen(uint64_t seed, int scale, uint32_t ta, uint32_t tab, uint32_t tabc) {
    auto sm = [](uint64_t x) {
        uint64_t z = x + 0x9E3779B97F4A7C15ULL;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        return z ^ (z >> 31);
    };
    return Gen{sm(seed), sm(seed ^ 0x5745494748545321ULL), scale, ta, tab, tabc};
}

constexpr int kThreads = 256;
constexpr int kSlotsPerBlock = 8192;

// degree histograms (counts at index + 1) and number of kept edges
__global__ void k_count(Gen g, uint64_t slots, int32_t* deg_row_by_dst, int32_t* deg_row_by_src,
                        unsigned long long* kept, const int32_t* remap) {
    unsigned long long local = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < slots;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t s, d;
        g.edge(i, s, d);
        if (s == d) continue;
        if (remap) { s = (uint32_t)remap[s]; d = (uint32_t)remap[d]; }
        ++local;
        if (deg_row_by_dst) atomicAdd(deg_row_by_dst + d + 1, 1);
        if (deg_row_by_src) atomicAdd(deg_row_by_src + s + 1, 1);
    }
    for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xFFFFFFFFu, local, o);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(kept, local);
}

// scatter keys (neighbour << 6 | (w - 1)) into rows via an atomic cursor
__global__ void k_scatter(Gen g, uint64_t slots, int by_dst, int weighted, int32_t* cursor,
                          uint64_t* keys, const int32_t* remap) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < slots;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t s, d;
        g.edge(i, s, d);
        if (s == d) continue;
        if (remap) { s = (uint32_t)remap[s]; d = (uint32_t)remap[d]; }
        const uint32_t row = by_dst ? d : s, nbr = by_dst ? s : d;
        const uint32_t w = weighted ? g.weight(i) : 1u;
        const int32_t pos = atomicAdd(cursor + row, 1);
        keys[pos] = ((uint64_t)nbr << 6) | (uint64_t)(w - 1u);
    }
}

__global__ void k_unpack(const uint64_t* keys, int64_t e, int32_t* idx, uint32_t* w) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < e;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = keys[i];
        idx[i] = (int32_t)(k >> 6);
        if (w) w[i] = (uint32_t)(k & 63u) + 1u;
    }
}

// COO in slot order: per-block kept counts, then ordered writes.
__global__ void k_block_counts(Gen g, uint64_t slots, unsigned long long* blk) {
    __shared__ unsigned long long s_c[kThreads / 32];
    const uint64_t b0 = (uint64_t)blockIdx.x * kSlotsPerBlock;
    unsigned long long c = 0;
    for (uint64_t i = b0 + threadIdx.x; i < b0 + kSlotsPerBlock && i < slots; i += kThreads) {
        uint32_t s, d;
        g.edge(i, s, d);
        c += s != d;
    }
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
    if ((threadIdx.x & 31) == 0) s_c[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int w = 0; w < kThreads / 32; ++w) t += s_c[w];
        blk[blockIdx.x] = t;
    }
}

__global__ void k_block_write(Gen g, uint64_t slots, const unsigned long long* blk_off,
                              int32_t* src, int32_t* dst, uint32_t* w) {
    __shared__ int s_warp[kThreads / 32];
    const uint64_t b0 = (uint64_t)blockIdx.x * kSlotsPerBlock;
    unsigned long long base = blk_off[blockIdx.x];
    for (uint64_t c0 = b0; c0 < b0 + kSlotsPerBlock && c0 < slots; c0 += kThreads) {
        const uint64_t i = c0 + threadIdx.x;
        uint32_t s = 0, d = 0;
        bool keep = false;
        if (i < slots && i < b0 + kSlotsPerBlock) {
            g.edge(i, s, d);
            keep = s != d;
        }
        const unsigned m = __ballot_sync(0xFFFFFFFFu, keep);
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        if (lane == 0) s_warp[warp] = __popc(m);
        __syncthreads();
        int pre = 0, tot = 0;
        for (int k = 0; k < kThreads / 32; ++k) {
            if (k < warp) pre += s_warp[k];
            tot += s_warp[k];
        }
        if (keep) {
            const unsigned long long pos = base + pre + __popc(m & ((1u << lane) - 1u));
            src[pos] = (int32_t)s;
            dst[pos] = (int32_t)d;
            if (w) w[pos] = g.weight(i);
        }
        base += tot;
        __syncthreads();
    }
}

int64_t fail(const char* what, cudaError_t e) {
    fprintf(stderr, "rmat_gpu: %s: %s\n", what, cudaGetErrorString(e));
    return -1;
}

#define CK(x)                                          \
    do {                                               \
        cudaError_t e_ = (x);                          \
        if (e_ != cudaSuccess) return fail(#x, e_);    \
    } while (0)

}  // namespace

extern "C" {

// Number of kept (non-self-loop) edges; optional in/out-degree histograms (int32 [n+1],
// zero-initialised by the caller, counts written at index + 1).
int64_t rmat_gpu_count(uint64_t seed, int scale, uint64_t slots, uint32_t ta, uint32_t tab,
                       uint32_t tabc, int32_t* deg_by_dst, int32_t* deg_by_src, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    Gen g = make_gen(seed, scale, ta, tab, tabc);
    unsigned long long* d_kept = nullptr;
    CK(cudaMallocAsync(&d_kept, 8, s));
    CK(cudaMemsetAsync(d_kept, 0, 8, s));
    k_count<<<148 * 16, kThreads, 0, s>>>(g, slots, deg_by_dst, deg_by_src, d_kept, nullptr);
    CK(cudaGetLastError());
    unsigned long long h = 0;
    CK(cudaMemcpyAsync(&h, d_kept, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaFreeAsync(d_kept, s));
    CK(cudaStreamSynchronize(s));
    return (int64_t)h;
}

// COO in slot order (device arrays of capacity >= kept).  Returns kept.
int64_t rmat_gpu_coo(uint64_t seed, int scale, uint64_t slots, uint32_t ta, uint32_t tab,
                     uint32_t tabc, int32_t* src, int32_t* dst, uint32_t* w, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    Gen g = make_gen(seed, scale, ta, tab, tabc);
    const uint64_t nb = (slots + kSlotsPerBlock - 1) / kSlotsPerBlock;
    unsigned long long* blk = nullptr;
    CK(cudaMallocAsync(&blk, (nb + 1) * 8, s));
    k_block_counts<<<(unsigned)nb, kThreads, 0, s>>>(g, slots, blk);
    CK(cudaGetLastError());
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, blk, blk, (int)nb + 1, s);
    CK(cudaMallocAsync(&tmp, tmp_bytes, s));
    // blk[nb] must be 0 before the scan so the total lands in blk[nb]
    CK(cudaMemsetAsync(blk + nb, 0, 8, s));
    cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, blk, blk, (int)nb + 1, s);
    k_block_write<<<(unsigned)nb, kThreads, 0, s>>>(g, slots, blk, src, dst, w);
    CK(cudaGetLastError());
    unsigned long long kept = 0;
    CK(cudaMemcpyAsync(&kept, blk + nb, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaFreeAsync(tmp, s));
    CK(cudaFreeAsync(blk, s));
    CK(cudaStreamSynchronize(s));
    return (int64_t)kept;
}

// One adjacency (by_dst = 1: CSC, rows are destinations; 0: CSR, rows are sources).
// off: int32 [n+1] zero-initialised by the caller; idx [kept]; w [kept] or NULL.
// Returns kept, or -1 on error.
int64_t rmat_gpu_adjacency(uint64_t seed, int scale, uint64_t slots, uint32_t ta, uint32_t tab,
                           uint32_t tabc, int by_dst, int32_t* off, int32_t* idx, uint32_t* w,
                           const int32_t* remap, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t n = (int64_t)1 << scale;
    Gen g = make_gen(seed, scale, ta, tab, tabc);
    unsigned long long* d_kept = nullptr;
    CK(cudaMallocAsync(&d_kept, 8, s));
    CK(cudaMemsetAsync(d_kept, 0, 8, s));
    k_count<<<148 * 16, kThreads, 0, s>>>(g, slots, by_dst ? off : nullptr,
                                          by_dst ? nullptr : off, d_kept, remap);
    CK(cudaGetLastError());
    unsigned long long kept = 0;
    CK(cudaMemcpyAsync(&kept, d_kept, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaFreeAsync(d_kept, s));
    CK(cudaStreamSynchronize(s));
    if (kept > 0x7FFFFFFFull) { fprintf(stderr, "rmat_gpu: E beyond int32\n"); return -1; }
    // offsets = inclusive scan of counts at index + 1
    void* tmp = nullptr;
    size_t tb = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tb, off, off, (int)(n + 1), s);
    CK(cudaMallocAsync(&tmp, tb, s));
    cub::DeviceScan::InclusiveSum(tmp, tb, off, off, (int)(n + 1), s);
    CK(cudaFreeAsync(tmp, s));
    int32_t* cursor = nullptr;
    uint64_t *keys = nullptr, *keys2 = nullptr;
    CK(cudaMallocAsync(&cursor, (n + 1) * 4, s));
    CK(cudaMemcpyAsync(cursor, off, (n + 1) * 4, cudaMemcpyDeviceToDevice, s));
    CK(cudaMallocAsync(&keys, (kept + 1) * 8, s));
    CK(cudaMallocAsync(&keys2, (kept + 1) * 8, s));
    k_scatter<<<148 * 16, kThreads, 0, s>>>(g, slots, by_dst, w != nullptr, cursor, keys, remap);
    CK(cudaGetLastError());
    CK(cudaFreeAsync(cursor, s));
    // sort each row by (neighbour, weight): deterministic arrays
    tb = 0;
    cub::DeviceSegmentedSort::SortKeys(nullptr, tb, keys, keys2, (int)kept, (int)n, off, off + 1, s);
    CK(cudaMallocAsync(&tmp, tb, s));
    cub::DeviceSegmentedSort::SortKeys(tmp, tb, keys, keys2, (int)kept, (int)n, off, off + 1, s);
    CK(cudaGetLastError());
    CK(cudaFreeAsync(tmp, s));
    CK(cudaFreeAsync(keys, s));
    k_unpack<<<148 * 16, kThreads, 0, s>>>(keys2, (int64_t)kept, idx, w);
    CK(cudaGetLastError());
    CK(cudaFreeAsync(keys2, s));
    CK(cudaStreamSynchronize(s));
    return (int64_t)kept;
}

__global__ void k_iota_u32(uint32_t* a, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) a[i] = (uint32_t)i;
}
__global__ void k_invert(const uint32_t* old_of_new, int64_t n, int32_t* new_of_old) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) new_of_old[old_of_new[i]] = (int32_t)i;
}

// Degree-descending vertex order (ties: ascending original id): a layout choice for the device
// graph, not part of the method.  old_of_new[k] = original id of internal vertex k;
// new_of_old = its inverse.  `deg_src` / `deg_dst` select which degrees are summed.
int64_t rmat_gpu_degree_order(uint64_t seed, int scale, uint64_t slots, uint32_t ta, uint32_t tab,
                              uint32_t tabc, int use_out, int use_in, int32_t* old_of_new,
                              int32_t* new_of_old, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t n = (int64_t)1 << scale;
    Gen g = make_gen(seed, scale, ta, tab, tabc);
    int32_t* deg = nullptr;
    unsigned long long* d_kept = nullptr;
    CK(cudaMallocAsync(&deg, (n + 1) * 4, s));
    CK(cudaMemsetAsync(deg, 0, (n + 1) * 4, s));
    CK(cudaMallocAsync(&d_kept, 8, s));
    CK(cudaMemsetAsync(d_kept, 0, 8, s));
    // both histograms land in the same array (counts at index + 1)
    k_count<<<148 * 16, kThreads, 0, s>>>(g, slots, use_in ? deg : nullptr,
                                          use_out ? deg : nullptr, d_kept, nullptr);
    CK(cudaGetLastError());
    uint32_t *keys_out = nullptr, *vals_in = nullptr;
    CK(cudaMallocAsync(&keys_out, n * 4, s));
    CK(cudaMallocAsync(&vals_in, n * 4, s));
    k_iota_u32<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(vals_in, n);
    void* tmp = nullptr;
    size_t tb = 0;
    const uint32_t* keys_in = reinterpret_cast<const uint32_t*>(deg + 1);
    cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, keys_in, keys_out, vals_in,
                                              (uint32_t*)old_of_new, (int)n, 0, 32, s);
    CK(cudaMallocAsync(&tmp, tb, s));
    cub::DeviceRadixSort::SortPairsDescending(tmp, tb, keys_in, keys_out, vals_in,
                                              (uint32_t*)old_of_new, (int)n, 0, 32, s);
    CK(cudaGetLastError());
    k_invert<<<(unsigned)((n + 255) / 256), 256, 0, s>>>((const uint32_t*)old_of_new, n, new_of_old);
    CK(cudaGetLastError());
    CK(cudaFreeAsync(tmp, s));
    CK(cudaFreeAsync(keys_out, s));
    CK(cudaFreeAsync(vals_in, s));
    CK(cudaFreeAsync(deg, s));
    CK(cudaFreeAsync(d_kept, s));
    CK(cudaStreamSynchronize(s));
    return n;
}

}  // extern "C"
