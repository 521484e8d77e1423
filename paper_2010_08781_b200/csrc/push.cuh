// paper_2010_08781_b200/csrc/push.cuh -- push-mode delivery and the frontier (selection bypass).
//
// Selection bypass, PAPER.md:177-189 (Sec. 4.3.1, Fig. 4): for programs with systematic halt
// (Hash-Min CC, SSSP: every vertex votes to halt after compute) the vertices
// to run in superstep s+1 are exactly the recipients of superstep s's messages.  The GPU keeps
// the equivalent set of *broadcasters* (recipients whose value did not improve only halt again,
// DESIGN.md reading R18): a bitmap of improved vertices is compacted, in ascending id order, into
// the frontier list with each vertex's value SNAPSHOT (BSP isolation).  The
// paper merges per-thread lists and splits them evenly; here a warp ballot/popc +
// block scan + a deterministic device-wide scan replaces the merge, and the expansion below is
// edge-balanced over the frontier's out-degrees instead of vertex-balanced.
//
// Push delivery, PAPER.md:195-197 (Sec. 4.3.2): the sender folds its message into the
// recipient's single-slot mailbox.  iPregel serialises this with busy-wait spinlocks and notes
// that a lock-free combine is possible when the combiner maps onto an atomic (and
// future work :706).  Here the combiner enum selects the atomic: atomicMin for Fig. 5's min,
// atomicAdd for Fig. 8's sum.  No user code is rewritten.
#pragma once
#include "common.cuh"

namespace ipr {

constexpr int kScanThreads = 256;
constexpr int kWordsPerThread = 4;
constexpr int kWordsPerBlock = kScanThreads * kWordsPerThread;   // 32768 vertices per block
constexpr int kListPerBlock = 2048;                             // list entries per scan block
#ifndef IPREGEL_EXPAND_THREADS
#define IPREGEL_EXPAND_THREADS 256
#endif
#ifndef IPREGEL_EXPAND_ITEMS
#define IPREGEL_EXPAND_ITEMS 512   // 2048: SSSP 11.85 ms, forced push 58.9; 1024: 11.45 / 41; 512: 11.32 / 34.5 (cfg4)
#endif
constexpr int kExpandThreads = IPREGEL_EXPAND_THREADS;
constexpr int kExpandItems = IPREGEL_EXPAND_ITEMS;               // edges per expand chunk

struct FrontierCounters {
    unsigned long long changed;   // vertices that broadcast (bits set)
    unsigned long long messages;  // sum of their out-degrees (symmetrised for CC)
    unsigned long long list_len;  // expand-list entries (push-view degree > 0)
    unsigned long long list_edges;// sum of push-view degrees (edges the expand touches)
};

// Adjacency a push expands over: up to two parts (CC uses out-edges then in-edges).
struct PushAdj {
    const int32_t* off1 = nullptr;  // indexed by (u - src_base)
    const int32_t* idx1 = nullptr;
    const uint32_t* w1 = nullptr;
    const int32_t* off2 = nullptr;
    const int32_t* idx2 = nullptr;
    const uint32_t* w2 = nullptr;   // weights of the second part (generic symmetric programs)
    int64_t src_base = 0;           // off arrays cover sources [src_base, src_base + src_rows)
    int64_t src_rows = 0;
    __device__ __forceinline__ int64_t degree(int64_t u) const {
        int64_t r = u - src_base;
        if (r < 0 || r >= src_rows) return 0;
        int64_t d = off1[r + 1] - off1[r];
        if (off2) d += off2[r + 1] - off2[r];
        return d;
    }
};

// Full (global-graph) degree of an owned vertex for the messages counter.
struct OwnedDegree {
    const int32_t* out_off = nullptr;  // owned CSR
    const int32_t* in_off = nullptr;   // owned CSC (CC only), else NULL
    __device__ __forceinline__ int64_t operator()(int64_t row) const {
        int64_t d = out_off[row + 1] - out_off[row];
        if (in_off) d += in_off[row + 1] - in_off[row];
        return d;
    }
};

__device__ __forceinline__ unsigned long long block_sum_u64(unsigned long long v,
                                                            unsigned long long* s_tmp) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(kFull, v, d);
    if ((threadIdx.x & 31) == 0) s_tmp[threadIdx.x >> 5] = v;
    __syncthreads();
    unsigned long long t = 0;
    if (threadIdx.x == 0)
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_tmp[w];
    __syncthreads();
    return t;  // valid in thread 0
}

// Exclusive block-wide scan of a per-thread u64 (fixed order).  Returns the exclusive prefix;
// *total receives the block total (all threads).
__device__ __forceinline__ unsigned long long block_exscan_u64(unsigned long long v,
                                                               unsigned long long* s_w,
                                                               unsigned long long* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    unsigned long long inc = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        unsigned long long o = __shfl_up_sync(kFull, inc, d);
        if (lane >= d) inc += o;
    }
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    unsigned long long wpre = 0, tot = 0;
    for (int w = 0; w < nw; ++w) {
        unsigned long long x = s_w[w];
        if (w < warp) wpre += x;
        tot += x;
    }
    __syncthreads();
    *total = tot;
    return wpre + inc - v;
}

// ---- bitmap -> frontier (3 passes: count, scan of block counts, write) ----------------------
// Pass 1: per block, number of set bits and the sum of their owned degrees.
__global__ void __launch_bounds__(kScanThreads)
k_bitmap_count(const uint32_t* __restrict__ bits, int64_t nwords, OwnedDegree deg,
               unsigned long long* __restrict__ blk_cnt, unsigned long long* __restrict__ blk_deg) {
    __shared__ unsigned long long s_tmp[kScanThreads / 32];
    const int64_t w0 = (int64_t)blockIdx.x * kWordsPerBlock;
    unsigned long long c = 0, dsum = 0;
#pragma unroll
    for (int k = 0; k < kWordsPerThread; ++k) {
        int64_t w = w0 + (int64_t)k * kScanThreads + threadIdx.x;
        if (w < nwords) {
            uint32_t b = bits[w];
            c += __popc(b);
            while (b) {
                int i = __ffs(b) - 1;
                b &= b - 1;
                dsum += deg(w * 32 + i);
            }
        }
    }
    unsigned long long tc = block_sum_u64(c, s_tmp);
    unsigned long long td = block_sum_u64(dsum, s_tmp);
    if (threadIdx.x == 0) { blk_cnt[blockIdx.x] = tc; blk_deg[blockIdx.x] = td; }
}

// Pass 2 (one CTA): exclusive scan of the block counts in place; totals into counters.
__global__ void __launch_bounds__(1024)
k_scan_blocks(unsigned long long* __restrict__ a, unsigned long long* __restrict__ b, int64_t n,
              unsigned long long* __restrict__ total_a, unsigned long long* __restrict__ total_b) {
    __shared__ unsigned long long s_w[32];
    unsigned long long carry_a = 0, carry_b = 0;
    for (int64_t base = 0; base < n; base += blockDim.x) {
        int64_t i = base + threadIdx.x;
        unsigned long long va = i < n ? a[i] : 0ull, vb = (b && i < n) ? b[i] : 0ull;
        unsigned long long ta, tb;
        unsigned long long ea = block_exscan_u64(va, s_w, &ta);
        unsigned long long eb = b ? block_exscan_u64(vb, s_w, &tb) : 0ull;
        if (i < n) { a[i] = carry_a + ea; if (b) b[i] = carry_b + eb; }
        carry_a += ta;
        if (b) carry_b += tb;
    }
    if (threadIdx.x == 0) {
        if (total_a) *total_a = carry_a;
        if (total_b && b) *total_b = carry_b;
    }
}

// Pass 3: write (global id, value snapshot) of every set bit in ascending order; clear the bits.
__global__ void __launch_bounds__(kScanThreads)
k_bitmap_write(uint32_t* __restrict__ bits, int64_t nwords, int64_t vbase,
               const uint32_t* __restrict__ vals, const unsigned long long* __restrict__ blk_off,
               int32_t* __restrict__ f_id, uint32_t* __restrict__ f_val) {
    __shared__ unsigned long long s_w[kScanThreads / 32];
    const int64_t w0 = (int64_t)blockIdx.x * kWordsPerBlock + (int64_t)threadIdx.x * kWordsPerThread;
    uint32_t wv[kWordsPerThread];
    unsigned long long c = 0;
#pragma unroll
    for (int k = 0; k < kWordsPerThread; ++k) {
        int64_t w = w0 + k;
        wv[k] = w < nwords ? bits[w] : 0u;
        c += __popc(wv[k]);
    }
    unsigned long long tot;
    unsigned long long pos = blk_off[blockIdx.x] + block_exscan_u64(c, s_w, &tot);
#pragma unroll
    for (int k = 0; k < kWordsPerThread; ++k) {
        int64_t w = w0 + k;
        uint32_t b = wv[k];
        if (w < nwords && b) {
            bits[w] = 0u;
            while (b) {
                int i = __ffs(b) - 1;
                b &= b - 1;
                int64_t v = vbase + w * 32 + i;
                f_id[pos] = (int32_t)v;
                f_val[pos] = vals ? vals[v] : 0u;
                ++pos;
            }
        }
    }
}

// ---- frontier -> expand list (entries with push-view degree > 0, with degree prefix) ---------
__global__ void __launch_bounds__(kScanThreads)
k_list_count(const int32_t* __restrict__ f_id, const unsigned long long* __restrict__ f_len,
             PushAdj adj, unsigned long long* __restrict__ blk_cnt,
             unsigned long long* __restrict__ blk_deg) {
    __shared__ unsigned long long s_tmp[kScanThreads / 32];
    const int64_t n = (int64_t)*f_len;
    const int64_t i0 = (int64_t)blockIdx.x * kListPerBlock;
    unsigned long long c = 0, d = 0;
    for (int64_t i = i0 + threadIdx.x; i < i0 + kListPerBlock && i < n; i += kScanThreads) {
        int64_t g = adj.degree(f_id[i]);
        c += g > 0;
        d += (unsigned long long)g;
    }
    unsigned long long tc = block_sum_u64(c, s_tmp);
    unsigned long long td = block_sum_u64(d, s_tmp);
    if (threadIdx.x == 0) { blk_cnt[blockIdx.x] = tc; blk_deg[blockIdx.x] = td; }
}

// Writes the expand list in frontier order: e_id, e_val (64-bit payload), e_pre (exclusive
// degree prefix).  Each thread handles kListPerBlock / kScanThreads consecutive entries.
__global__ void __launch_bounds__(kScanThreads)
k_list_write(const int32_t* __restrict__ f_id, const uint32_t* __restrict__ f_val,
             const unsigned long long* __restrict__ f_len, PushAdj adj,
             const unsigned long long* __restrict__ blk_cnt,
             const unsigned long long* __restrict__ blk_deg, int32_t* __restrict__ e_id,
             uint32_t* __restrict__ e_val, long long* __restrict__ e_pre) {
    __shared__ unsigned long long s_w[kScanThreads / 32];
    constexpr int kPer = kListPerBlock / kScanThreads;
    const int64_t n = (int64_t)*f_len;
    const int64_t i0 = (int64_t)blockIdx.x * kListPerBlock + (int64_t)threadIdx.x * kPer;
    int64_t g[kPer];
    unsigned long long c = 0, d = 0;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
        int64_t i = i0 + k;
        g[k] = i < n ? adj.degree(f_id[i]) : 0;
        c += g[k] > 0;
        d += (unsigned long long)g[k];
    }
    unsigned long long tc, td;
    unsigned long long pc = blk_cnt[blockIdx.x] + block_exscan_u64(c, s_w, &tc);
    unsigned long long pd = blk_deg[blockIdx.x] + block_exscan_u64(d, s_w, &td);
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
        if (g[k] > 0) {
            int64_t i = i0 + k;
            e_id[pc] = f_id[i];
            e_val[pc] = f_val ? f_val[i] : 0u;
            e_pre[pc] = (long long)pd;
            ++pc;
            pd += (unsigned long long)g[k];
        }
    }
}

// ---- expansion: one message per out-edge of every frontier vertex ---------------------------
// Edge-balanced over the expand list: per chunk of kExpandItems edges, the frontier entries it
// touches, each with its adjacency bases resolved once, and an owner table (edge slot -> entry)
// from a block scan of the entries' start flags -- no per-edge search, no per-edge offset loads.
// The message of edge (u -> v, w) with the sender's snapshot is folded into v's slot in two
// steps: `p = deliver.pre(u, snapshot, v, w)` issues the loads (plain reads that only filter or
// feed the fold), `deliver.fin(p, u, snapshot, v, w)` the atomics.
template <class Deliver>
__device__ __forceinline__ void expand_edges(const PushAdj& adj, const int32_t* __restrict__ e_id,
                                             const uint32_t* __restrict__ e_val,
                                             const long long* __restrict__ e_pre,
                                             const unsigned long long* __restrict__ counters_len,
                                             const unsigned long long* __restrict__ counters_edges,
                                             const Deliver& deliver) {
    constexpr int kPer = kExpandItems / kExpandThreads;
    __shared__ int32_t s_start[kExpandItems + 1];   // entry start relative to the chunk
    __shared__ int32_t s_b1[kExpandItems + 1], s_d1[kExpandItems + 1], s_b2[kExpandItems + 1];
    __shared__ uint32_t s_val[kExpandItems + 1];
    __shared__ int32_t s_id[kExpandItems + 1];
    __shared__ uint16_t s_owner[kExpandItems];
    __shared__ int s_range[2];
    __shared__ int s_wsum[kExpandThreads / 32];
    const int64_t n = (int64_t)*counters_len;
    const int64_t total = (int64_t)*counters_edges;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int64_t e0 = (int64_t)blockIdx.x * kExpandItems; e0 < total;
         e0 += (int64_t)gridDim.x * kExpandItems) {
        const int64_t e1 = e0 + kExpandItems < total ? e0 + kExpandItems : total;
        const int span = (int)(e1 - e0);
        if (warp < 2) {
            // entry owning edge e: last i with e_pre[i] <= e (e_pre[0] = 0 <= e).  A 32-way
            // search by one warp per end: each step probes 32 evenly spaced entries of [lo, hi]
            // at once, so the dependent load chain is log32(n) long instead of log2(n)
            const int64_t target = warp == 0 ? e0 : e1 - 1;
            int64_t lo = 0, hi = n - 1;
            while (lo < hi) {
                const int64_t len = hi - lo + 1;
                const int64_t stride = (len + 31) >> 5;
                const int64_t p = lo + (int64_t)lane * stride;
                const bool le = p <= hi && e_pre[p] <= target;
                const int k = __popc(__ballot_sync(kFull, le)) - 1;   // lane 0 probes lo: k >= 0
                lo += (int64_t)k * stride;
                if (stride == 1) break;
                const int64_t h = lo + stride - 1;
                hi = h < hi ? h : hi;
            }
            if (lane == 0) s_range[warp] = (int)lo;
        }
        for (int j = threadIdx.x; j < kExpandItems; j += kExpandThreads) s_owner[j] = 0;
        __syncthreads();
        const int f0 = s_range[0], nf = s_range[1] - s_range[0] + 1;
        for (int i = threadIdx.x; i < nf; i += kExpandThreads) {
            const int64_t st = e_pre[f0 + i] - e0;
            s_start[i] = (int32_t)st;
            const int32_t u = e_id[f0 + i];
            s_id[i] = u;
            s_val[i] = e_val ? e_val[f0 + i] : 0u;
            const int64_t r = (int64_t)u - adj.src_base;
            const int32_t b1 = adj.off1[r];
            s_b1[i] = b1;
            s_d1[i] = adj.off1[r + 1] - b1;
            s_b2[i] = adj.off2 ? adj.off2[r] : 0;
            if (i > 0) s_owner[st] = 1;   // start flag (entries have degree >= 1: distinct)
        }
        __syncthreads();
        // owner(j) = number of entry starts in (0, j]: block inclusive scan of the flags
        int f[kPer];
        int c = 0;
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            f[k] = s_owner[threadIdx.x * kPer + k];
            c += f[k];
        }
        int inc = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int o = __shfl_up_sync(kFull, inc, d);
            if (lane >= d) inc += o;
        }
        if (lane == 31) s_wsum[warp] = inc;
        __syncthreads();
        int pre = inc - c;
        for (int w = 0; w < warp; ++w) pre += s_wsum[w];
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            pre += f[k];
            s_owner[threadIdx.x * kPer + k] = (uint16_t)pre;
        }
        __syncthreads();
        // a thread's kPer edges in three batched phases -- all destination (and weight) loads,
        // then the deliveries' loads, then their atomics -- so kPer independent requests are in
        // flight per phase instead of one load-atomic chain per edge
        int32_t v[kPer];
        uint32_t w[kPer];
        int ow[kPer];
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const int j = threadIdx.x + k * kExpandThreads;
            ow[k] = -1;
            v[k] = 0;
            w[k] = 1u;
            if (j < span) {
                const int o = s_owner[j];
                const int32_t pos = j - s_start[o];
                ow[k] = o;
                if (pos < s_d1[o]) {
                    v[k] = adj.idx1[s_b1[o] + pos];
                    if (adj.w1) w[k] = adj.w1[s_b1[o] + pos];
                } else {
                    v[k] = adj.idx2[s_b2[o] + (pos - s_d1[o])];
                    if (adj.w2) w[k] = adj.w2[s_b2[o] + (pos - s_d1[o])];
                }
            }
        }
        typename Deliver::Pre pv[kPer];
#pragma unroll
        for (int k = 0; k < kPer; ++k)
            if (ow[k] >= 0) pv[k] = deliver.pre(s_id[ow[k]], s_val[ow[k]], v[k], w[k]);
#pragma unroll
        for (int k = 0; k < kPer; ++k)
            if (ow[k] >= 0) deliver.fin(pv[k], s_id[ow[k]], s_val[ow[k]], v[k], w[k]);
        __syncthreads();
    }
}

// The paper's programs.  Min programs (CC, SSSP): msg = snapshot (CC) or sat(snapshot + w)
// (SSSP); atomicMin into the live value of the recipient; a successful decrease marks the
// recipient in the next bitmap.  Sum program (PageRank push): atomicAdd of the sender's
// contribution into the accumulator.
template <bool B, class A, class C>
struct PickT {
    using type = A;
};
template <class A, class C>
struct PickT<false, A, C> {
    using type = C;
};

template <int kProgram>
struct BuiltinDeliver {
    int64_t dst_base;
    uint32_t* val;
    uint32_t* bits;
    const double* contrib;
    double* acc;
    // PageRank: the sender's contribution; min programs: the recipient's current value (a cheap
    // filter read before the atomics -- the atomic decides)
    using Pre = typename PickT<kProgram == 0, double, uint32_t>::type;
    __device__ __forceinline__ Pre pre(int32_t u, uint32_t, int32_t v, uint32_t) const {
        if constexpr (kProgram == 0) return contrib[u];
        else return val[v];
    }
    __device__ __forceinline__ void fin(Pre p, int32_t, uint32_t snap, int32_t v,
                                        uint32_t w) const {
        const int64_t lv = (int64_t)v - dst_base;
        if constexpr (kProgram == 0) {
            atomicAdd(acc + lv, p);
        } else {
            const uint32_t msg = kProgram == 2 ? sat_add(snap, w) : snap;
            if (msg < p) {
                const uint32_t old = atomicMin(val + v, msg);
                if (msg < old) atomicOr(bits + (lv >> 5), 1u << (lv & 31));
            }
        }
    }
};

template <int kProgram>  // 0 PageRank (sum), 1 CC (min, no weight), 2 SSSP (min + weight)
__global__ void __launch_bounds__(kExpandThreads)
k_expand(PushAdj adj, const int32_t* __restrict__ e_id, const uint32_t* __restrict__ e_val,
         const long long* __restrict__ e_pre, const unsigned long long* __restrict__ counters_len,
         const unsigned long long* __restrict__ counters_edges, int64_t dst_base,
         uint32_t* __restrict__ val, uint32_t* __restrict__ bits,
         const double* __restrict__ contrib, double* __restrict__ acc) {
    if (kProgram != 2) adj.w1 = nullptr;   // weights only matter to SSSP
    adj.w2 = nullptr;
    expand_edges(adj, e_id, e_val, e_pre, counters_len, counters_edges,
                 BuiltinDeliver<kProgram>{dst_base, val, bits, contrib, acc});
}

// ---- Hash-Min row-list pull -----------------------------------------------------------------
// Once most rows hold label 0 (the smallest id, absorbing for min: PAPER.md:341-344 never lowers
// it further), a dense pull superstep spends its time streaming rows whose result is already
// known.  The row-list pull runs the same gather-combine only over the rows NOT at 0: the owned
// rows are compacted into a list (the frontier machinery above), and the edges of the listed rows
// (CSC row + CSR row: the symmetrised neighbourhood) are expanded edge-balanced, each folding its
// neighbour's label into the row's next value with atomicMin (min is exact in any order).
struct RowMinDeliver {
    const uint32_t* cur;   // labels after superstep s-1 (replica, global ids)
    uint32_t* next;        // next[u] = cur[u] on entry (owned rows), min over neighbours on exit
    using Pre = uint2;     // (neighbour's label, row's next value before this batch)
    __device__ __forceinline__ Pre pre(int32_t u, uint32_t, int32_t v, uint32_t) const {
        return make_uint2(cur[v], next[u]);
    }
    __device__ __forceinline__ void fin(Pre p, int32_t u, uint32_t, int32_t, uint32_t) const {
        if (p.x < p.y) atomicMin(next + u, p.x);
    }
};

__global__ void __launch_bounds__(kExpandThreads)
k_rowlist_min(PushAdj adj, const int32_t* __restrict__ e_id, const long long* __restrict__ e_pre,
              const unsigned long long* __restrict__ len,
              const unsigned long long* __restrict__ edges, const uint32_t* __restrict__ cur,
              uint32_t* __restrict__ next) {
    adj.w1 = nullptr;
    adj.w2 = nullptr;
    expand_edges(adj, e_id, nullptr, e_pre, len, edges, RowMinDeliver{cur, next});
}

// Owned rows whose value is not `v0` (ballot per warp).
__global__ void k_bits_ne(const uint32_t* __restrict__ vals, int64_t rows, uint32_t v0,
                          const uint32_t* __restrict__ mask, uint32_t* __restrict__ bits) {
    // one warp per 1024 rows, as k_bitmap_from_diff
    const int lane = threadIdx.x & 31;
    const int64_t nwords = (rows + 31) >> 5;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; c * 32 < nwords;
         c += nw) {
        uint32_t mine = 0u;
#pragma unroll 8
        for (int k = 0; k < 32; ++k) {
            const int64_t i = (c * 32 + k) * 32 + lane;
            const uint32_t b = __ballot_sync(kFull, i < rows && vals[i] != v0);
            if (lane == k) mine = b;
        }
        const int64_t w = c * 32 + lane;
        if (w < nwords) bits[w] = mask ? mine & mask[w] : mine;
    }
}
// Rows with at least one neighbour in the symmetrised graph (CSC or CSR row not empty), one bit
// per owned row: the others never receive a message and keep their label, so the Hash-Min row
// list leaves them out (a third of cfg4's vertices are isolated).
__global__ void k_nbr_bits(const int32_t* __restrict__ in_off, const int32_t* __restrict__ out_off,
                           int64_t rows, uint32_t* __restrict__ bits) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool pred = i < rows && (in_off[i + 1] > in_off[i] || out_off[i + 1] > out_off[i]);
    const uint32_t b = __ballot_sync(kFull, pred);
    if ((threadIdx.x & 31) == 0 && i < rows) bits[i >> 5] = b;
}

// Hash-Min row-list superstep: only the listed rows (global ids, `len` of them) can have
// changed; mark those whose label decreased in the (zeroed) owned bitmap.
__global__ void k_bits_from_list_diff(const int32_t* __restrict__ ids,
                                      const unsigned long long* __restrict__ len,
                                      const uint32_t* __restrict__ before,
                                      const uint32_t* __restrict__ after, int64_t vbase,
                                      uint32_t* __restrict__ bits) {
    const int64_t n = (int64_t)*len;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = ids[i];
        if (after[v] < before[v]) {
            const int64_t r = v - vbase;
            atomicOr(bits + (r >> 5), 1u << (r & 31));
        }
    }
}

// Pull -> push switch: the broadcasters of a pull superstep are the vertices whose value
// decreased; mark them in the bitmap (owned range).  One warp per 1024 rows: for each of its 32
// words the lanes compare 32 consecutive rows (coalesced) and the ballot is the word, kept by
// the lane that stores it -- one coalesced 128-byte store per warp, 16 loads in flight per lane
// (one thread per row ran 262K blocks at cfg4 and took 0.19 ms).
__global__ void k_bitmap_from_diff(const uint32_t* __restrict__ before,
                                   const uint32_t* __restrict__ after, int64_t vbase, int64_t rows,
                                   uint32_t* __restrict__ bits) {
    const int lane = threadIdx.x & 31;
    const int64_t nwords = (rows + 31) >> 5;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; c * 32 < nwords;
         c += nw) {
        uint32_t mine = 0u;
#pragma unroll 8
        for (int k = 0; k < 32; ++k) {
            const int64_t i = (c * 32 + k) * 32 + lane;
            const bool pred = i < rows && after[vbase + i] < before[vbase + i];
            const uint32_t b = __ballot_sync(kFull, pred);
            if (lane == k) mine = b;
        }
        const int64_t w = c * 32 + lane;
        if (w < nwords) bits[w] = mine;
    }
}

// PageRank push apply: r = ratio + 0.85 * acc; next contribution; reset the accumulator.
// dmax != NULL (to convergence): rank holds r_{s-1}; fold max |r_s - r_{s-1}| (reading R27).
__global__ void k_pr_push_apply(double* __restrict__ acc, const int32_t* __restrict__ out_off,
                                int64_t rows, int64_t vbase, double ratio, int broadcast,
                                int write_rank, double* __restrict__ rank,
                                double* __restrict__ contrib_next,
                                unsigned long long* __restrict__ dmax, double* __restrict__ mass) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double r = 0.0;
    unsigned long long d = 0;
    if (i < rows) {
        r = __dadd_rn(ratio, __dmul_rn(0.85, acc[i]));
        if (dmax) d = (unsigned long long)__double_as_longlong(fabs(__dsub_rn(r, rank[i])));
    }
    if (mass) {   // grid-uniform; whole warps
        LaneCounters c;
        if (i < rows) {
            c.m0 = r;
            c.m1 = out_off[i + 1] > out_off[i] ? r : 0.0;
        }
        flush_mass(c, mass);
    }
    if (dmax) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long x = __shfl_xor_sync(kFull, d, o);
            d = x > d ? x : d;
        }
        if ((threadIdx.x & 31) == 0 && d) atomicMax(dmax, d);
    }
    if (i >= rows) return;
    acc[i] = 0.0;
    if (write_rank) rank[i] = r;
    if (broadcast) {
        const int32_t deg = out_off[i + 1] - out_off[i];
        contrib_next[vbase + i] = deg > 0 ? __ddiv_rn(r, (double)deg) : 0.0;
    }
}

}  // namespace ipr
