// paper_2010_08781_b200/csrc/setup.cuh -- superstep 0, validation, push-view construction and
// small utility kernels.
#pragma once
#include "common.cuh"
#include "pull.cuh"

namespace ipr {

// ---- superstep 0 (the `ip_is_first_superstep()` branches of Figs. 8-10) --------------------
// PageRank, Fig. 8 / PAPER.md:322: value = 1/N and, if superstep 0 < k, broadcast value/outdeg
// (a vertex without out-neighbours does not broadcast, reading R4).
// 4 rows per thread (block-strided, coalesced), their out-degrees loaded before any division
// (the loads then overlap; as k_pr_finish)
constexpr int kInitRows = 4;
__global__ void k_init_pagerank(const int32_t* __restrict__ out_off, int64_t rows, int64_t vbase,
                                double inv_n, int broadcast, int write_rank,
                                double* __restrict__ rank, double* __restrict__ contrib,
                                double* __restrict__ mass) {
    const int64_t base = (int64_t)blockIdx.x * blockDim.x * kInitRows + threadIdx.x;
    LaneCounters c;
    int32_t deg[kInitRows];
#pragma unroll
    for (int j = 0; j < kInitRows; ++j) {
        const int64_t i = base + (int64_t)j * blockDim.x;
        deg[j] = i < rows && (broadcast || mass) ? out_off[i + 1] - out_off[i] : 0;
    }
#pragma unroll
    for (int j = 0; j < kInitRows; ++j) {
        const int64_t i = base + (int64_t)j * blockDim.x;
        if (i >= rows) continue;
        if (write_rank) rank[i] = inv_n;
        if (broadcast) contrib[vbase + i] = deg[j] > 0 ? __ddiv_rn(inv_n, (double)deg[j]) : 0.0;
        if (mass) {
            c.m0 += inv_n;
            if (deg[j] > 0) c.m1 += inv_n;
        }
    }
    if (mass) flush_mass(c, mass);   // grid-uniform; whole warps (blocks of 256)
}

// User programs: broadcaster bitmap of the owned rows from the per-vertex flag bytes (bit 0),
// for the frontier compaction of a push superstep (ballot per warp).
__global__ void k_bits_from_flags(const uint8_t* __restrict__ flags, int64_t rows,
                                  uint32_t* __restrict__ bits) {
    // one thread per 32 rows: two 16-byte loads of flag bytes (the flag array is padded to a
    // multiple of 32 bytes with zeros) -> one bitmap word
    const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= (rows + 31) / 32) return;
    const uint4* f = reinterpret_cast<const uint4*>(flags + 32 * w);
    const uint4 a = f[0], b = f[1];
    const uint32_t v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    uint32_t m = 0u;
#pragma unroll
    for (int i = 0; i < 8; ++i)
        m |= ((v[i] & 1u) | ((v[i] >> 7) & 2u) | ((v[i] >> 14) & 4u) | ((v[i] >> 21) & 8u)) << (4 * i);
    bits[w] = m;
}

// Max of (INF - value) over a device list of values (SSSP: the smallest distance among a push
// superstep's broadcasters, for the absorption bound of SSSPPull).
__global__ void k_list_max_inv(const uint32_t* __restrict__ vals,
                               const unsigned long long* __restrict__ len,
                               unsigned long long* __restrict__ out) {
    const int64_t n = (int64_t)*len;
    unsigned long long m = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long x = (unsigned long long)(kInf - vals[i]);
        m = x > m ? x : m;
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        const unsigned long long o = __shfl_xor_sync(kFull, m, d);
        m = o > m ? o : m;
    }
    if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

// Min of a u32 array (SSSP: the smallest edge weight), into *out (initialised to INF).
__global__ void k_min_u32(const uint32_t* __restrict__ a, int64_t n, unsigned* __restrict__ out) {
    unsigned m = kInf;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        m = a[i] < m ? a[i] : m;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        const unsigned o = __shfl_xor_sync(kFull, m, d);
        m = o < m ? o : m;
    }
    if ((threadIdx.x & 31) == 0) atomicMin(out, m);
}

// Fill 8-byte slots with a pattern (vsz 4: the low 32 bits into a u32 array of the same count).
__global__ void k_fill_u64(uint64_t* __restrict__ a, int64_t n, uint64_t pattern, int vsz) {
    // 16 bytes per thread
    const int64_t bytes = n * vsz;
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 16;
    if (i >= bytes) return;
    uint8_t* p = reinterpret_cast<uint8_t*>(a) + i;
    if (i + 16 <= bytes) {
        const uint64_t q = vsz == 8 ? pattern : ((pattern & 0xFFFFFFFFull) | (pattern << 32));
        *reinterpret_cast<ulonglong2*>(p) = make_ulonglong2(q, q);
    } else {
        for (int64_t k = i; k < bytes; k += vsz) {
            if (vsz == 8) *reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(a) + k) = pattern;
            else *reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(a) + k) = (uint32_t)pattern;
        }
    }
}

// inv[ids[v]] = v
__global__ void k_invert_ids(const int32_t* __restrict__ ids, int64_t n, int32_t* __restrict__ inv) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) inv[ids[i]] = (int32_t)i;
}

// Hash-Min CC, Fig. 9: value = id, the ORIGINAL id under a relabelled layout (every replica
// initialises all N locally -- no exchange).
__global__ void k_init_cc(uint32_t* __restrict__ val, int64_t n, const int32_t* __restrict__ ids) {
    // grid-stride, 16-byte loads and stores where both arrays allow (pool allocations are
    // 256-byte aligned; caller-provided vertex_ids may not be)
    const bool vec = ids == nullptr || (reinterpret_cast<uintptr_t>(ids) & 15) == 0;
    const int64_t n4 = vec ? n >> 2 : 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint4* v4 = reinterpret_cast<uint4*>(val);
    for (int64_t i = t; i < n4; i += stride) {
        uint4 x;
        if (ids) {
            const int4 y = reinterpret_cast<const int4*>(ids)[i];
            x = make_uint4((uint32_t)y.x, (uint32_t)y.y, (uint32_t)y.z, (uint32_t)y.w);
        } else {
            x = make_uint4((uint32_t)(4 * i), (uint32_t)(4 * i + 1), (uint32_t)(4 * i + 2),
                           (uint32_t)(4 * i + 3));
        }
        v4[i] = x;
    }
    for (int64_t i = (n4 << 2) + t; i < n; i += stride) val[i] = ids ? (uint32_t)ids[i] : (uint32_t)i;
}

// internal id of original vertex `orig` (vertex_ids is a permutation)
__global__ void k_find_index(const int32_t* __restrict__ ids, int64_t n, int32_t orig,
                             unsigned long long* __restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        if (ids[i] == orig) *out = (unsigned long long)i;
}

// out[ids[i]] = in[i]: values in internal order -> original order
template <class T>
__global__ void k_to_original(const T* __restrict__ in, const int32_t* __restrict__ ids, int64_t n,
                              T* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[ids[i]] = in[i];
}

// permutation check: every id in [0, n) exactly once
__global__ void k_count_ids(const int32_t* __restrict__ ids, int64_t n, int32_t* __restrict__ seen,
                            unsigned* __restrict__ flags) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t v = ids[i];
    if (v < 0 || (int64_t)v >= n || atomicAdd(seen + v, 1) != 0) atomicOr(flags, 8u);
}

// SSSP, Fig. 10: source = 0, everyone else INF.
__global__ void k_init_sssp(uint32_t* __restrict__ val, int64_t n, int64_t source) {
    // grid-stride, 16-byte stores (val is 256-byte aligned: a pool allocation)
    uint4* v4 = reinterpret_cast<uint4*>(val);
    const int64_t n4 = n >> 2;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint4 x = make_uint4(kInf, kInf, kInf, kInf);
        if ((source >> 2) == i) (&x.x)[source & 3] = 0u;
        v4[i] = x;
    }
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < (n & 3)) {
        const int64_t i = (n4 << 2) + t;
        val[i] = i == source ? 0u : kInf;
    }
}

__global__ void k_fill_bits(uint32_t* __restrict__ bits, int64_t rows) {
    const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nwords = (rows + 31) >> 5;
    if (w >= nwords) return;
    const int64_t rem = rows - w * 32;
    bits[w] = rem >= 32 ? 0xFFFFFFFFu : ((1u << rem) - 1u);
}

__global__ void k_set_bit(uint32_t* __restrict__ bits, int64_t row) {
    bits[row >> 5] |= 1u << (row & 31);
}

// Scatter a global frontier's (id, value) snapshots into a replica (multi-partition push).
__global__ void k_scatter_frontier(const int32_t* __restrict__ id, const uint32_t* __restrict__ v,
                                   const unsigned long long* __restrict__ len,
                                   uint32_t* __restrict__ val) {
    const int64_t n = (int64_t)*len;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        val[id[i]] = v[i];
}

__global__ void k_iota(int32_t* __restrict__ a, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) a[i] = (int32_t)i;
}

// Owned vertices with out-degree > 0 (PageRank broadcasters).
__global__ void k_count_nondangling(const int32_t* __restrict__ out_off, int64_t rows,
                                    unsigned long long* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool p = i < rows && out_off[i + 1] > out_off[i];
    const unsigned b = __ballot_sync(kFull, p);
    if ((threadIdx.x & 31) == 0 && b) atomicAdd(out, (unsigned long long)__popc(b));
}

// ---- validation (ipregel_graph_desc.validate) ------------------------------------------------
// flags bit 0: offsets[0] != 0 or offsets[rows] != edges; bit 1: offsets decrease; bit 2: index
// outside [0, N).
__global__ void k_validate_offsets(const int32_t* __restrict__ off, int64_t rows, int64_t edges,
                                   unsigned* __restrict__ flags) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0 && (off[0] != 0 || (int64_t)off[rows] != edges)) atomicOr(flags, 1u);
    if (i < rows && off[i + 1] < off[i]) atomicOr(flags, 2u);
}
__global__ void k_validate_indices(const int32_t* __restrict__ idx, int64_t edges, int64_t n,
                                   unsigned* __restrict__ flags) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < edges;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = idx[i];
        if (v < 0 || (int64_t)v >= n) { atomicOr(flags, 4u); return; }
    }
}

// ---- push view for a destination partition (multi-GPU push mode) ---------------------------
// Source-major list of the edges whose destination is owned: built by transposing the owned
// CSC rows (u -> v) and, for CC, the owned CSR rows reversed (u <- v taken as u -> v).
// Sort-based transpose (coalesced writes; an atomic-cursor scatter writes 4-byte words at
// random, which costs ~7x the bytes in DRAM read-modify-write): every edge becomes a
// (source, row | edge << 32) pair, a stable LSD radix sort by source groups the pairs into the
// transposed rows with their destinations ascending (the input is in row order), and the unpack
// writes the indices contiguously and fetches each weight by its edge index -- so the weights
// are needed only at the very end (the host upload of them overlaps the sort).
__global__ void k_transpose_pack(const int32_t* __restrict__ off, int64_t rows, int64_t vbase,
                                 unsigned long long* __restrict__ vals) {
    const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (r >= rows) return;
    const unsigned long long v = (unsigned long long)(uint32_t)(vbase + r);
    for (int32_t e = off[r] + lane; e < off[r + 1]; e += 32)
        vals[e] = v | ((unsigned long long)(uint32_t)e << 32);
}

// As k_transpose_pack with the edge's weight in the high half instead of its position (the
// relabel's CSR: the weights are already in place, so no gather after the sort)
__global__ void k_transpose_pack_w(const int32_t* __restrict__ off, int64_t rows, int64_t vbase,
                                   const uint32_t* __restrict__ w,
                                   unsigned long long* __restrict__ vals) {
    const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (r >= rows) return;
    const unsigned long long v = (unsigned long long)(uint32_t)(vbase + r);
    for (int32_t e = off[r] + lane; e < off[r + 1]; e += 32)
        vals[e] = v | ((unsigned long long)w[e] << 32);
}
__global__ void k_unpack_w(const unsigned long long* __restrict__ vals, int64_t edges,
                           int32_t* __restrict__ out_idx, uint32_t* __restrict__ out_w) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < edges;
         i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long x = vals[i];
        out_idx[i] = (int32_t)(uint32_t)x;
        if (out_w) out_w[i] = (uint32_t)(x >> 32);
    }
}

// Run boundaries of the sorted sources: start[k] = first position of source k, end[k] = one past
// its last (both 0 for sources without edges); then count[k] = end[k] - start[k] in place.
__global__ void k_run_bounds(const int32_t* __restrict__ keys, int64_t edges,
                             int32_t* __restrict__ start, int32_t* __restrict__ end) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < edges;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t k = keys[i];
        if (i == 0 || keys[i - 1] != k) start[k] = (int32_t)i;
        if (i + 1 == edges || keys[i + 1] != k) end[k] = (int32_t)(i + 1);
    }
}
__global__ void k_run_counts(const int32_t* __restrict__ start, int64_t n,
                             int32_t* __restrict__ end_to_count) {
    const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (u < n) end_to_count[u] = end_to_count[u] ? end_to_count[u] - start[u] : 0;
}

__global__ void k_transpose_unpack(const unsigned long long* __restrict__ vals, int64_t edges,
                                   const uint32_t* __restrict__ w, int32_t* __restrict__ out_idx,
                                   uint32_t* __restrict__ out_w, int32_t* __restrict__ out_perm) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < edges;
         i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long x = vals[i];
        out_idx[i] = (int32_t)(uint32_t)x;
        if (out_perm) out_perm[i] = (int32_t)(uint32_t)(x >> 32);   // weights permuted later
        else if (out_w) out_w[i] = w ? __ldg(w + (uint32_t)(x >> 32)) : 1u;
    }
}

// ---- IPREGEL_LAYOUT_DEGREE: the library's own degree relabel (create time) -----------------
// out-degrees from CSR offsets, or counted over the CSC sources
__global__ void k_degree_from_off(const int32_t* __restrict__ off, int64_t n,
                                  uint32_t* __restrict__ deg) {
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v < n) deg[v] = (uint32_t)(off[v + 1] - off[v]);
}
// (CSC rows list their sources ascending, so a hot source recurs within a warp's 32 consecutive
// edges: the lanes holding the same id add once, by their count)
__global__ void k_degree_hist(const int32_t* __restrict__ idx, int64_t edges,
                              uint32_t* __restrict__ deg) {
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); e0 < edges;
         e0 += stride) {
        const int64_t e = e0 + lane;
        const int32_t u = e < edges ? idx[e] : -1;
        const uint32_t same = __match_any_sync(kFull, u);
        if (u >= 0 && lane == __ffs(same) - 1) atomicAdd(deg + u, (uint32_t)__popc(same));
    }
}
// sort keys: ascending ~deg = descending degree; a stable sort keeps ties in id order
__global__ void k_degree_keys(uint32_t* __restrict__ deg, int64_t n, int32_t* __restrict__ ids) {
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v < n) {
        deg[v] = ~deg[v];
        ids[v] = (int32_t)v;
    }
}
// out-degrees in the new order from the sorted keys (~degree), into roff[0..n); roff[n] = 0
__global__ void k_degree_from_keys(const uint32_t* __restrict__ keys, int64_t n,
                                   int32_t* __restrict__ roff) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) roff[i] = (int32_t)~keys[i];
    else if (i == n) roff[i] = 0;
}
__global__ void k_invert_perm(const int32_t* __restrict__ old_of_new, int64_t n,
                              int32_t* __restrict__ new_of_old) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) new_of_old[old_of_new[i]] = (int32_t)i;
}
__global__ void k_iota_u32(uint32_t* __restrict__ a, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        a[i] = (uint32_t)i;
}
// out[i] = in[perm[i]]
__global__ void k_gather_u32(const uint32_t* __restrict__ perm, int64_t n,
                             const uint32_t* __restrict__ in, uint32_t* __restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = in[perm[i]];
}
// Sort key of a relabelled source inside its row: the id itself when cbits >= bits (rows fully
// sorted), else a monotone cbits-bit class -- ids below 2^sub exactly, above that the position
// of the top bit and the sub = cbits - 5 bits below it -- so the hot low ids (a handful per
// 128-B line) keep their exact order and only cold ids, one per line anyway, share a class.
__device__ __forceinline__ uint32_t source_class(uint32_t s, int bits, int cbits) {
    if (cbits >= bits) return s;
    const int sub = cbits - 5;
    if (s < (1u << sub)) return s;
    const int hb = 32 - __clz(s);   // > sub
    return ((uint32_t)(hb - sub) << sub) | ((s >> (hb - 1 - sub)) & ((1u << sub) - 1u));
}
// relabelled edge keys: (new destination << cbits) | class of the new source, one warp per CSC
// row (the edge's CSC position travels as the sort's value)
__global__ void k_relabel_pack(const int32_t* __restrict__ off, const int32_t* __restrict__ idx,
                               int64_t rows, const int32_t* __restrict__ new_of_old, int bits,
                               int cbits, unsigned long long* __restrict__ keys,
                               int32_t* __restrict__ new_src) {
    const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (r >= rows) return;
    const unsigned long long hi = (unsigned long long)(uint32_t)new_of_old[r] << cbits;
    for (int32_t e = off[r] + lane; e < off[r + 1]; e += 32) {
        const int32_t u = new_of_old[idx[e]];
        new_src[e] = u;
        keys[e] = hi | source_class((uint32_t)u, bits, cbits);
    }
}
// sorted (key, CSC position) -> new CSC indices (the renamed source at each position, written
// by k_relabel_pack) + each edge's new row (for the run-length offsets)
__global__ void k_relabel_unpack(const unsigned long long* __restrict__ keys,
                                 const uint32_t* __restrict__ pos, int64_t edges, int cbits,
                                 const int32_t* __restrict__ new_src, int32_t* __restrict__ idx,
                                 int32_t* __restrict__ row) {
    // pos[i] lies in the old CSC row of i's row: the gather reads within one row's block
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < edges;
         i += (int64_t)gridDim.x * blockDim.x) {
        idx[i] = new_src[pos[i]];
        row[i] = (int32_t)(keys[i] >> cbits);
    }
}

// One window [lo, hi) of the deferred weight permutation: wx[i] = w[perm[i]] where perm[i] falls
// in the window (the window's upload has landed; the others are written by their own passes).
__global__ void k_permute_window(const int32_t* __restrict__ perm, int64_t edges, int64_t lo,
                                 int64_t hi, const uint32_t* __restrict__ w,
                                 uint32_t* __restrict__ wx) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < edges;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = perm[i];
        if (e >= lo && e < hi) wx[i] = __ldg(w + e);
    }
}

// Device-wide exclusive scan of int32 counts (in place), 3 passes with a u64 block scratch.
constexpr int kScanChunk = 2048;
__global__ void __launch_bounds__(256)
k_chunk_sums(const int32_t* __restrict__ a, int64_t n, unsigned long long* __restrict__ sums) {
    __shared__ unsigned long long s[8];
    const int64_t base = (int64_t)blockIdx.x * kScanChunk;
    unsigned long long t = 0;
    for (int64_t i = base + threadIdx.x; i < base + kScanChunk && i < n; i += 256) t += (unsigned)a[i];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) t += __shfl_xor_sync(kFull, t, d);
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long x = 0;
        for (int w = 0; w < 8; ++w) x += s[w];
        sums[blockIdx.x] = x;
    }
}

__global__ void __launch_bounds__(256)
k_chunk_apply(int32_t* __restrict__ a, int64_t n, const unsigned long long* __restrict__ offs) {
    __shared__ unsigned long long s_w[8];
    constexpr int kPer = kScanChunk / 256;
    const int64_t i0 = (int64_t)blockIdx.x * kScanChunk + (int64_t)threadIdx.x * kPer;
    int32_t v[kPer];
    unsigned long long t = 0;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
        v[k] = i0 + k < n ? a[i0 + k] : 0;
        t += (unsigned)v[k];
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long inc = t;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        unsigned long long o = __shfl_up_sync(kFull, inc, d);
        if (lane >= d) inc += o;
    }
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    unsigned long long pre = offs[blockIdx.x];
    for (int w = 0; w < warp; ++w) pre += s_w[w];
    pre += inc - t;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
        if (i0 + k < n) a[i0 + k] = (int32_t)pre;
        pre += (unsigned)v[k];
    }
}

}  // namespace ipr
