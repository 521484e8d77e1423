// paper_2010_08781_b200/csrc/pull.cuh -- pull-mode delivery: CSC gather-combine.
//
// PAPER.md:199-203 (Sec. 4.3.2): in pull mode every vertex broadcasts into a single outbox slot
// and every recipient scans the outboxes of its in-neighbours, lock-free.  Here the outbox is the
// previous superstep's value array (double-buffered, BSP isolation PAPER.md:151, :239), and one
// superstep's gather + combine + compute of all recipients is ONE kernel over the in-adjacency.
//
// Work decomposition (B200-first, not the paper's OpenMP static schedule PAPER.md:155-157):
// an edge-balanced "merge path" over the two sorted lists {row ends} and {edges}.  Every CTA
// consumes exactly kItems = rows + edges merge items, so hub rows (in-degree ~1.5M at scale 26)
// and the ~40% of rows with tiny or zero in-degree are balanced alike, with no degree binning
// pass.  Per tile:
//   1. coalesced, vectorised, L2-evict-first loads of the tile's column indices; the gathered
//      outbox values are issued in one burst (8 independent loads per thread) and staged in
//      shared memory with the tile's row ends;
//   2. every thread walks kIPT consecutive merge items out of shared memory, combining edges
//      and finishing rows;
//   3. rows cut by thread boundaries are joined by a block-wide segmented scan (fixed tree);
//      rows cut by tile boundaries are joined by pull_fixup in a fixed order.
// The combine order therefore depends only on global merge coordinates: tile boundaries are
// multiples of kItems in GLOBAL diagonal space, so PageRank is bit-identical for any
// destination partition.
#pragma once
#include "common.cuh"

namespace ipr {

constexpr int kPullThreads = 256;
constexpr int kPullIPT = 8;
constexpr int kPullItems = kPullThreads * kPullIPT;

struct PullCounters {
    unsigned long long changed;
    unsigned long long messages;
};

// Tile plan for one adjacency of one partition: merge coordinates of every tile boundary.
struct TilePlan {
    int32_t rows = 0;
    int64_t edges = 0;
    int64_t phase = 0;       // (global diagonal of local diagonal 0) mod kPullItems
    int32_t num_tiles = 0;
    int32_t* cx = nullptr;   // [num_tiles + 1] rows consumed at each boundary (local)
    int32_t* cy = nullptr;   // [num_tiles + 1] edges consumed at each boundary (local)
    int32_t num_groups = 0;
    int4* groups = nullptr;  // spanning rows: (row, first boundary a, last boundary b, 0)
    void* carry = nullptr;   // [num_tiles] partial of the row leaving the tile (8-byte slots)
    void* head = nullptr;    // [num_tiles] partial of the row entering and ending in the tile
};

// Boundary b of the plan: local diagonal clamp(b * kItems - phase, 0, rows + edges), and its
// merge coordinate via binary search (A[i] = end offset of row i, B[j] = j).
__global__ void k_plan_boundaries(const int32_t* __restrict__ off, int32_t rows, int64_t edges,
                                  int64_t phase, int32_t num_tiles, int32_t* cx, int32_t* cy) {
    int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b > num_tiles) return;
    int64_t total = (int64_t)rows + edges;
    int64_t d = b * (int64_t)kPullItems - phase;
    d = d < 0 ? 0 : (d > total ? total : d);
    int64_t lo = d - edges > 0 ? d - edges : 0;
    int64_t hi = d < rows ? d : rows;
    while (lo < hi) {
        int64_t p = (lo + hi) >> 1;
        if ((int64_t)off[p + 1] <= d - p - 1) lo = p + 1; else hi = p;
    }
    cx[b] = (int32_t)lo;
    cy[b] = (int32_t)(d - lo);
}

// ---- combine policies -------------------------------------------------------------------------
struct SumF64 {
    using T = double;
    __device__ static T identity() { return 0.0; }
    __device__ static T combine(T a, T b) { return __dadd_rn(a, b); }  // Fig. 8 ip_combine
};
struct MinU32 {
    using T = uint32_t;
    __device__ static T identity() { return kInf; }
    __device__ static T combine(T a, T b) { return a > b ? b : a; }   // Fig. 5 ip_combine
};

// ---- vertex programs (gather = message on an in-edge, finish = recipient compute) ----------
// PageRank, Fig. 8: the message of u is contrib[u] = r_u / outdeg(u); recipient compute is
// r = ratio + 0.85 * sum, then broadcast r / outdeg for the next superstep if s < k.
struct PageRankPull : SumF64 {
    const double* __restrict__ contrib_cur;   // replica, global ids
    double* __restrict__ contrib_next;        // replica, global ids
    double* __restrict__ rank;                // owned, local ids (written when write_rank)
    const int32_t* __restrict__ out_off;      // owned CSR offsets (local rows)
    int64_t vbase;
    double ratio;
    int broadcast;                            // s < k
    int write_rank;
    __device__ T gather(int64_t /*e*/, int32_t u, uint64_t /*ps*/, uint64_t pol) const {
        return ld_gather(contrib_cur + u, pol);
    }
    __device__ void finish(int32_t row, T sum, PullCounters& /*c*/) const {
        double r = __dadd_rn(ratio, __dmul_rn(0.85, sum));
        if (write_rank) rank[row] = r;
        if (broadcast) {
            int32_t deg = out_off[row + 1] - out_off[row];
            contrib_next[vbase + row] = deg > 0 ? __ddiv_rn(r, (double)deg) : 0.0;
        }
    }
};

// Hash-Min CC, Fig. 9, first half: min over the CSC row (in-neighbours' labels).
struct CCPullIn : MinU32 {
    const uint32_t* __restrict__ cur;   // replica, global ids
    uint32_t* __restrict__ next;        // replica, global ids (owned slice written)
    int64_t vbase;
    __device__ T gather(int64_t, int32_t u, uint64_t, uint64_t pol) const {
        return ld_gather(cur + u, pol);
    }
    __device__ void finish(int32_t row, T m, PullCounters&) const {
        uint32_t c = cur[vbase + row];
        next[vbase + row] = m < c ? m : c;
    }
};

// Hash-Min CC, second half: min over the CSR row (the symmetrised graph's reverse edges), then
// "if value < old: broadcast" -> changed / messages counters (degree in the symmetrised graph).
struct CCPullOut : MinU32 {
    const uint32_t* __restrict__ cur;
    uint32_t* __restrict__ next;
    const int32_t* __restrict__ in_off;   // owned CSC offsets
    const int32_t* __restrict__ out_off;  // owned CSR offsets
    int64_t vbase;
    __device__ T gather(int64_t, int32_t u, uint64_t, uint64_t pol) const {
        return ld_gather(cur + u, pol);
    }
    __device__ void finish(int32_t row, T m, PullCounters& c) const {
        uint32_t old = cur[vbase + row];
        uint32_t v = next[vbase + row];
        v = m < v ? m : v;
        next[vbase + row] = v;
        if (v < old) {
            c.changed += 1;
            c.messages += (unsigned long long)(in_off[row + 1] - in_off[row]) +
                          (unsigned long long)(out_off[row + 1] - out_off[row]);
        }
    }
};

// SSSP, Fig. 10 with weights: message on edge (u -> v, w) is sat(dist_u + w), applied at the
// recipient from the CSC weight (reading R8); "if mindist < value: broadcast".
struct SSSPPull : MinU32 {
    const uint32_t* __restrict__ cur;
    uint32_t* __restrict__ next;
    const uint32_t* __restrict__ in_w;    // owned CSC weights or NULL (= 1)
    const int32_t* __restrict__ out_off;  // owned CSR offsets
    int64_t vbase;
    __device__ T gather(int64_t e, int32_t u, uint64_t ps, uint64_t pol) const {
        uint32_t w = in_w ? ld_stream(in_w + e, ps) : 1u;
        return sat_add(ld_gather(cur + u, pol), w);
    }
    __device__ void finish(int32_t row, T m, PullCounters& c) const {
        uint32_t old = cur[vbase + row];
        uint32_t v = m < old ? m : old;
        next[vbase + row] = v;
        if (v < old) {
            c.changed += 1;
            c.messages += (unsigned long long)(out_off[row + 1] - out_off[row]);
        }
    }
};

// ---- block-wide segmented inclusive scan (flag = a row ended inside this thread) ----------
template <class Op>
__device__ __forceinline__ void block_seg_scan(int& flag, typename Op::T& val,
                                               typename Op::T* s_wval, int* s_wflag) {
    using T = typename Op::T;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        T vp = shfl_up(val, d);
        int fp = shfl_up(flag, d);
        if (lane >= d) {
            if (!flag) val = Op::combine(vp, val);
            flag |= fp;
        }
    }
    if (lane == 31) { s_wval[warp] = val; s_wflag[warp] = flag; }
    __syncthreads();
    if (warp > 0 && !flag) {
        // exclusive segmented prefix over the preceding warps, nearest first
        T pre = s_wval[warp - 1];
        int pf = s_wflag[warp - 1];
        for (int w = warp - 2; w >= 0 && !pf; --w) {
            pre = Op::combine(s_wval[w], pre);
            pf = s_wflag[w];
        }
        val = Op::combine(pre, val);
    }
}

// One tile per CTA.  tile_base = local tile index; thread j's local diagonal is
// tile * kItems - phase + j * kIPT clamped to the tile.
template <class Op>
__global__ void __launch_bounds__(kPullThreads)
k_pull_tiles(Op op, const int32_t* __restrict__ off, const int32_t* __restrict__ idx,
             const int32_t* __restrict__ cx, const int32_t* __restrict__ cy, int32_t rows,
             int64_t phase, typename Op::T* __restrict__ carry, typename Op::T* __restrict__ head,
             PullCounters* __restrict__ counters) {
    using T = typename Op::T;
    __shared__ T s_val[kPullItems];
    __shared__ int32_t s_end[kPullItems + 1];
    __shared__ T s_scan[kPullThreads];
    __shared__ T s_wval[kPullThreads / 32];
    __shared__ int s_wflag[kPullThreads / 32];
    __shared__ unsigned long long s_cnt[2];

    const int tile = blockIdx.x;
    const int32_t x0 = cx[tile], y0 = cy[tile], x1 = cx[tile + 1], y1 = cy[tile + 1];
    const int n_ends = x1 - x0;             // rows finished in this tile
    const int n_edges = y1 - y0;
    const int n_a = (x1 < rows ? x1 : rows - 1) - x0 + 1;  // row-end entries staged
    const uint64_t pol_stream = policy_evict_first();
    const uint64_t pol_gather = policy_evict_last();

    if (threadIdx.x < 2) s_cnt[threadIdx.x] = 0;
    for (int i = threadIdx.x; i < n_a; i += kPullThreads) s_end[i] = off[x0 + i + 1] - y0;

    // Column indices: scalar head up to 16-byte alignment, then int4 loads.
    {
        const int32_t* base = idx + y0;
        int head_n = (int)((16 - ((uintptr_t)base & 15)) & 15) >> 2;
        if (head_n > n_edges) head_n = n_edges;
        for (int i = threadIdx.x; i < head_n; i += kPullThreads)
            s_val[i] = op.gather((int64_t)y0 + i, ld_stream(base + i, pol_stream), pol_stream, pol_gather);
        const int n_vec = (n_edges - head_n) >> 2;
        const int4* vbase = reinterpret_cast<const int4*>(base + head_n);
        for (int q = threadIdx.x; q < n_vec; q += kPullThreads) {
            int4 u = ld_stream4(vbase + q, pol_stream);
            int i = head_n + 4 * q;
            T a = op.gather((int64_t)y0 + i, u.x, pol_stream, pol_gather);
            T b = op.gather((int64_t)y0 + i + 1, u.y, pol_stream, pol_gather);
            T c = op.gather((int64_t)y0 + i + 2, u.z, pol_stream, pol_gather);
            T d = op.gather((int64_t)y0 + i + 3, u.w, pol_stream, pol_gather);
            s_val[i] = a; s_val[i + 1] = b; s_val[i + 2] = c; s_val[i + 3] = d;
        }
        for (int i = head_n + 4 * n_vec + threadIdx.x; i < n_edges; i += kPullThreads)
            s_val[i] = op.gather((int64_t)y0 + i, ld_stream(base + i, pol_stream), pol_stream, pol_gather);
    }
    __syncthreads();

    // This thread's merge range.
    const int tile_items = n_ends + n_edges;
    int64_t lo_g = (int64_t)tile * kPullItems - phase;          // local diag of the tile grid
    int64_t tile_lo = (int64_t)x0 + y0;                         // clamped tile start (local)
    int d0 = (int)(lo_g + (int64_t)threadIdx.x * kPullIPT - tile_lo);
    d0 = d0 < 0 ? 0 : (d0 > tile_items ? tile_items : d0);
    int d1 = (int)(lo_g + (int64_t)(threadIdx.x + 1) * kPullIPT - tile_lo);
    d1 = d1 < 0 ? 0 : (d1 > tile_items ? tile_items : d1);

    int lo = d0 - n_edges > 0 ? d0 - n_edges : 0;
    int hi = d0 < n_ends ? d0 : n_ends;
    while (lo < hi) {
        int p = (lo + hi) >> 1;
        if (s_end[p] <= d0 - p - 1) lo = p + 1; else hi = p;
    }
    int x = lo, y = d0 - lo;

    PullCounters cnt{0, 0};
    T acc = Op::identity();
    T head_part = Op::identity();
    int emitted = 0;
#pragma unroll
    for (int k = 0; k < kPullIPT; ++k) {
        if (d0 + k < d1) {
            if (y < s_end[x]) {
                acc = Op::combine(acc, s_val[y]);
                ++y;
            } else {
                if (!emitted) head_part = acc;
                else op.finish(x0 + x, acc, cnt);
                emitted = 1;
                acc = Op::identity();
                ++x;
            }
        }
    }
    // Segmented scan of the tail partials; S_j = partial of the row leaving thread j.
    int flag = emitted;
    T val = acc;
    block_seg_scan<Op>(flag, val, s_wval, s_wflag);
    s_scan[threadIdx.x] = val;
    __syncthreads();

    if (emitted) {
        const int first_row = lo;  // the thread's start row is the first one it finishes
        T v = threadIdx.x > 0 ? Op::combine(s_scan[threadIdx.x - 1], head_part) : head_part;
        if (first_row == 0 && tile > 0) {
            // The row entering the tile is cut by boundary `tile`: pull_fixup finishes it.
            head[tile] = v;
        } else {
            op.finish(x0 + first_row, v, cnt);
        }
    }
    if (threadIdx.x == kPullThreads - 1) carry[tile] = val;

    // Counters: warp reduce, then one shared atomic per warp, one global atomic per CTA.
    unsigned long long c0 = cnt.changed, c1 = cnt.messages;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        c0 += __shfl_xor_sync(kFull, c0, d);
        c1 += __shfl_xor_sync(kFull, c1, d);
    }
    if ((threadIdx.x & 31) == 0 && (c0 | c1)) {
        atomicAdd(&s_cnt[0], c0);
        atomicAdd(&s_cnt[1], c1);
    }
    __syncthreads();
    if (threadIdx.x == 0 && counters && (s_cnt[0] | s_cnt[1])) {
        atomicAdd(&counters->changed, s_cnt[0]);
        atomicAdd(&counters->messages, s_cnt[1]);
    }
}

// Rows cut by tile boundaries: boundaries a..b (1 <= a <= b) carry row r; its value is
// carry[a-1] (+) carry[a] (+) ... (+) carry[b-1] (+) head[b], folded in a fixed order
// (lane-strided partials, then a fixed xor tree).  One warp per spanning row.
template <class Op>
__global__ void k_pull_fixup(Op op, const int4* __restrict__ groups, int32_t num_groups,
                             const typename Op::T* __restrict__ carry,
                             const typename Op::T* __restrict__ head,
                             PullCounters* __restrict__ counters) {
    using T = typename Op::T;
    const int lane = threadIdx.x & 31;
    const int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (g >= num_groups) return;
    const int4 G = groups[g];
    T acc = Op::identity();
    for (int t = G.y - 1 + lane; t <= G.z - 1; t += 32) acc = Op::combine(acc, carry[t]);
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        T o = shfl_xor(acc, d);
        acc = (lane & d) ? Op::combine(o, acc) : Op::combine(acc, o);
    }
    if (lane == 0) {
        acc = Op::combine(acc, head[G.z]);
        PullCounters c{0, 0};
        op.finish(G.x, acc, c);
        if (counters && (c.changed | c.messages)) {
            atomicAdd(&counters->changed, c.changed);
            atomicAdd(&counters->messages, c.messages);
        }
    }
}

}  // namespace ipr
