// paper_2010_08781_b200/csrc/pull.cuh -- pull-mode delivery: CSC gather-combine.
//
// PAPER.md:199-203 (Sec. 4.3.2): in pull mode every vertex broadcasts into a single outbox slot
// and every recipient scans the outboxes of its in-neighbours, lock-free.  Here the outbox is the
// previous superstep's value array (double-buffered, BSP isolation PAPER.md:151, :239), and one
// superstep's gather + combine + compute of all recipients is ONE kernel over the in-adjacency.
//
// Work decomposition (B200-first; the paper's OpenMP static vertex split, is
// prior art): the merge of the two sorted lists {row ends} and {in-edges} is cut into fixed
// RANGES of kRangeItems items (merge path), so every range holds the same number of edges + rows
// whatever the degree distribution (hub rows of in-degree ~1.5M at scale 26, long runs of rows
// without in-edges) -- no degree binning pass, no shared-memory staging, no block barrier.  One
// resident wave of CTAs runs; each warp takes range after range from an atomic counter,
// alternately from the two ends of the plan (long-row and short-row ranges side by side).  A warp
// walks the edges of its range in CHUNKS of 128 (4 per lane):
//   1. column indices arrive with coalesced L2-evict-first loads two chunks ahead and the
//      outbox values are gathered one chunk ahead (software pipeline, 8 gathers in flight per
//      lane); each gather instruction reads the sources of 32 consecutive edges;
//   2. a chunk inside one row (most edges: long rows) only adds into lane-private accumulators;
//   3. a chunk where exactly one row ends closes it with two masked warp folds; a chunk where
//      more rows end builds a 128-bit head-flag mask from the CSC offsets (__reduce_or_sync),
//      folds it with four 5-step segmented shuffle scans (segment starts read off the uniform
//      flag words; 8-byte values close the first and last segments with the same masked folds
//      as the one-end chunks), and each row ending there reads its sum from a per-warp slot
//      array and runs the recipient compute (fused epilogue);
//   4. a row cut by a range boundary is joined by k_pull_fixup in a fixed order.
// Range boundaries sit at multiples of kRangeItems in GLOBAL merge coordinates and chunks at
// multiples of 128 GLOBAL edge positions, so every row's combine tree depends on global positions
// only: PageRank is bit-identical for any destination partition.
#pragma once
#include "common.cuh"

namespace ipr {

// L2 prefetch distance of the index / weight stream in chunks (0 = off)
#ifndef IPREGEL_IDX_PREFETCH
#define IPREGEL_IDX_PREFETCH 0
#endif
// u32 min ops take the one-row-end path too (two redux.sync.min instead of the scan)
#ifndef IPREGEL_U32_ONE_END
#define IPREGEL_U32_ONE_END 1
#endif
#ifndef IPREGEL_CHUNK_UNROLL
#define IPREGEL_CHUNK_UNROLL 1   // chunk-loop unroll (2: CC +0.3 ms, SSSP +0.2 ms, PageRank equal; 4: all slower)
#endif
constexpr int kChunkUnroll = IPREGEL_CHUNK_UNROLL;
#ifndef IPREGEL_PR_MINBLOCKS
#define IPREGEL_PR_MINBLOCKS 3   // PageRankSum / PageRankPull CTAs per SM
#endif
#ifndef IPREGEL_PULL_MINBLOCKS
#define IPREGEL_PULL_MINBLOCKS 4
#endif
// per-op override: an op may set `static constexpr int kMinBlocks` (PageRankSum: 3, measured)
template <class...> using void_t_ = void;
template <class Op, class = void> struct PullMinBlocks { static constexpr int value = IPREGEL_PULL_MINBLOCKS; };
template <class Op> struct PullMinBlocks<Op, void_t_<decltype(Op::kMinBlocks)>> {
    static constexpr int value = Op::kMinBlocks;
};
#ifndef IPREGEL_PULL_THREADS
#define IPREGEL_PULL_THREADS 256
#endif
constexpr int kPullThreads = IPREGEL_PULL_THREADS;  // range-kernel CTA size (build knob)
constexpr int kWarpsPerCta = kPullThreads / 32;
constexpr int kChunk = 128;                       // edges per warp step
#ifndef IPREGEL_RANGE_ITEMS
#define IPREGEL_RANGE_ITEMS 8192   // 4096: PageRank +0.5 ms; 2048 / 16384 / 32768 slower (cfg4)
#endif
constexpr int kRangeItems = IPREGEL_RANGE_ITEMS;  // merge items (edges + rows) per warp range

struct PullCounters {
    unsigned long long changed;
    unsigned long long messages;
    unsigned long long dmax;   // PageRank to convergence: max |r_s - r_{s-1}| as f64 bits (>= 0)
    unsigned long long aux;    // user programs: vertices that did not vote to halt; Hash-Min:
                               // symmetrised degree of the rows at label 0 after the superstep
    unsigned long long gathered;   // absorbing ops: edges whose messages were actually gathered
};

// A thread's share of the counters while it runs, 32-bit (fewer live registers in the range
// kernels' epilogue): a thread counts rows it finishes (< 2^31) and the sum of their degrees,
// at most 2E < 2^32 for the symmetrised graph since E <= INT32_MAX (validated at create).
struct LaneCounters {
    uint32_t changed;
    uint32_t aux;
    uint32_t messages;
    unsigned long long dmax;
    double agg;        // user programs: this thread's fold of ipr_aggregate values
    uint32_t agg_n;    //   (agg_n = 0: nothing folded)
    unsigned long long mkey = ~0ull;   // user programs with ipr_settled: min broadcast (order key)
    double m0 = 0.0, m1 = 0.0;         // PageRank mass check: sum of r, sum of r over outdeg > 0
    uint32_t gathered = 0;             // absorbing ops: edges gathered (lane 0 of each warp)
};

// PageRank mass check (IPREGEL_RUN_PAGERANK_MASS): the lanes' sums of r and of r over vertices
// with out-degree > 0, warp-reduced, one f64 atomic pair per warp into this superstep's slot.
// Every lane of the warp must call it.
__device__ __forceinline__ void flush_mass(const LaneCounters& c, double* mass) {
    double a = c.m0, b = c.m1;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        a += __shfl_xor_sync(kFull, a, d);
        b += __shfl_xor_sync(kFull, b, d);
    }
    if ((threadIdx.x & 31) == 0 && (a != 0.0 || b != 0.0)) {
        atomicAdd(mass, a);
        atomicAdd(mass + 1, b);
    }
}
template <class Op, class = void> struct HasMass { static constexpr bool value = false; };
template <class Op> struct HasMass<Op, void_t_<decltype(Op::kMass)>> {
    static constexpr bool value = Op::kMass;
};

// Range plan for one adjacency of one partition.
struct TilePlan {
    int32_t rows = 0;
    int64_t edges = 0;
    int64_t phase = 0;        // (global merge diagonal of local diagonal 0) mod kRangeItems
    int64_t cphase = 0;       // (global edge index of local edge 0) mod kChunk
    int32_t num_tiles = 0;    // ranges
    int32_t* cx = nullptr;    // [num_tiles + 1] rows finished before each range boundary
    int32_t* cy = nullptr;    // [num_tiles + 1] edges consumed before each range boundary
    int32_t num_groups = 0;
    int32_t num_short = 0;    // groups[0, num_short) span <= kFixupShortSpan boundaries
    int4* groups = nullptr;   // rows cut by range boundaries: (row, first boundary a, last b, 0)
    void* carry = nullptr;    // [num_tiles] partial of the row leaving the range (8-byte slots)
    void* head = nullptr;     // [num_tiles] partial of the row entering and ending in the range
    int32_t* ctr = nullptr;   // dynamic range counter (zeroed before each launch)
};

// Range boundary b: local diagonal clamp(b * kRangeItems - phase, 0, rows + edges) and its merge
// coordinate (rows finished, edges consumed) by binary search (A[i] = end of row i, B[j] = j).
__global__ void k_plan_boundaries(const int32_t* __restrict__ off, int32_t rows, int64_t edges,
                                  int64_t phase, int32_t num_ranges, int32_t* __restrict__ cx,
                                  int32_t* __restrict__ cy) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b > num_ranges) return;
    const int64_t total = (int64_t)rows + edges;
    int64_t d = b * (int64_t)kRangeItems - phase;
    d = d < 0 ? 0 : (d > total ? total : d);
    int64_t lo = d - edges > 0 ? d - edges : 0;
    int64_t hi = d < rows ? d : rows;
    while (lo < hi) {
        const int64_t m = (lo + hi) >> 1;
        if ((int64_t)off[m + 1] <= d - m - 1) lo = m + 1; else hi = m;
    }
    cx[b] = (int32_t)lo;
    cy[b] = (int32_t)(d - lo);
}

// Row in flight at range boundary b (has edges on both sides' merge order), or -1.
__global__ void k_plan_inflight(const int32_t* __restrict__ off, const int32_t* __restrict__ cx,
                                const int32_t* __restrict__ cy, int32_t rows, int32_t num_ranges,
                                int32_t* __restrict__ infl) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= num_ranges) return;
    int32_t v = -1;
    if (b >= 1) {
        const int32_t r = cx[b];
        if (r < rows && off[r] < cy[b]) v = r;
    }
    infl[b] = v;
}

// ---- combine policies -------------------------------------------------------------------------
struct SumF64 {
    using T = double;
    __device__ static T identity() { return 0.0; }
    __device__ static T combine(T a, T b) { return __dadd_rn(a, b); }  // Fig. 8 ip_combine
};
struct MinU32 {
    using T = uint32_t;
    static constexpr bool kReduxMin = true;   // warp folds by redux.sync.min (min is exact)
    __device__ static T identity() { return kInf; }
    __device__ static T combine(T a, T b) { return a > b ? b : a; }   // Fig. 5 ip_combine
};

// Ops whose result is settled once a row's partial reaches an absorbing value (Hash-Min: label
// 0, the smallest id, cannot be lowered) stop gathering the rest of that row.
struct NotAbsorbing {
    static constexpr bool kAbsorbing = false;          // absorbed(row): the row is settled
    static constexpr bool kAbsorbingPartial = false;   // absorbing(partial): so is a row whose
                                                       // partial combine reaches this value
};

// ---- fused exchange ---------------------------------------------------------
// Every OTHER replica of the broadcast array that must receive this partition's owned slice: peer
// GPUs' replicas mapped over NVLink (CUDA IPC) for ranks of a communicator, or the other
// partitions' replicas in loopback mode.  The recipient compute stores each owned result into all
// of them in its epilogue, so the exchange that a separate AllGatherv would do after the kernel is
// carried by the kernel's own stores, overlapped with the gathers of the rest of the grid.
constexpr int kMaxPeers = 7;
template <class T>
struct PeerSlots {
    T* p[kMaxPeers];
    int n;
    __device__ __forceinline__ void store(int64_t i, T v) const {
        if (n == 0) return;   // one partition: no other replica (the common case, one test)
#pragma unroll
        for (int k = 0; k < kMaxPeers; ++k)
            if (k < n) p[k][i] = v;
    }
};

// Ops that fold a program aggregator flush it at the end of the kernel (kAggregates).
struct NoAggregate {
    static constexpr bool kAggregates = false;
};

// ---- vertex programs: gather = outbox value of the sender, message = value on the edge,
// finish = recipient compute --------------------------------------------------------------------
// PageRank, Fig. 8: the message of u is contrib[u] = r_u / outdeg(u); recipient compute is
// r = ratio + 0.85 * sum, then broadcast r / outdeg for the next superstep if s < k.
struct PageRankPull : SumF64, NotAbsorbing, NoAggregate {
    static constexpr bool kWeighted = false;
    static constexpr bool kMass = true;
    static constexpr int kMinBlocks = IPREGEL_PR_MINBLOCKS;   // as PageRankSum
    const double* __restrict__ contrib_cur;   // replica, global ids
    double* __restrict__ contrib_next;        // replica, global ids
    PeerSlots<double> peers;                  // fused exchange: other replicas (n = 0: none)
    double* __restrict__ rank;                // owned, local ids (written when write_rank)
    const int32_t* __restrict__ out_off;      // owned CSR offsets (local rows)
    int64_t vbase;
    double ratio;
    int broadcast;                            // s < k
    int write_rank;
    int track;                                // to convergence: rank holds r_{s-1}; fold |dr|
    double* mass;                             // mass check: this superstep's [sum r, sum_nd r]
    // k_pr_finish<., true>: sums by ordinal among rows with in-edges (pr_flag.cuh)
    const double* __restrict__ sumc = nullptr;
    const uint32_t* __restrict__ nzbits = nullptr;
    const int32_t* __restrict__ nzpre = nullptr;
    const void* gather_base() const { return contrib_cur; }
    __device__ const T* gptr() const { return contrib_cur; }
    __device__ bool absorbed(int32_t) const { return false; }
    __device__ static T message(T g, uint32_t) { return g; }
    __device__ void finish(int32_t row, T sum, LaneCounters& c) const {
        const int32_t deg = (broadcast || mass) ? out_off[row + 1] - out_off[row] : 0;
        finish_deg(row, sum, deg, c);
    }
    // The update with the row's out-degree given (k_pr_finish loads the degrees of all its rows
    // up front, so those loads overlap instead of serialising per row).
    __device__ __forceinline__ void finish_deg(int32_t row, T sum, int32_t deg,
                                               LaneCounters& c) const {
        const double r = __dadd_rn(ratio, __dmul_rn(0.85, sum));
        if (track) {   // max aggregator of the per-vertex change (reading R27)
            const unsigned long long d =
                (unsigned long long)__double_as_longlong(fabs(__dsub_rn(r, rank[row])));
            c.dmax = d > c.dmax ? d : c.dmax;
        }
        if (write_rank) rank[row] = r;
        if (broadcast && deg > 0) {
            // a vertex without out-edges is never gathered (it is nobody's in-neighbour): its
            // outbox slot is left as it is
            const double x = __ddiv_rn(r, (double)deg);
            contrib_next[vbase + row] = x;
            peers.store(vbase + row, x);
        }
        if (mass) {   // the invariant sum r_s = 0.15 + 0.85 sum_{outdeg>0} r_{s-1} (tests)
            c.m0 += r;
            if (deg > 0) c.m1 += r;
        }
    }
};

// PageRank with the update split out of the range kernel (IPREGEL_PR_SPLIT=1): the range kernel
// only stores each row's combined sum into its next-outbox slot, and k_pr_finish applies Fig. 8's
// update row-parallel (same operations, same result).
struct PageRankSum : SumF64, NotAbsorbing, NoAggregate {
    static constexpr bool kWeighted = false;
    // 3 CTAs per SM (80 registers, no spills) instead of 4 (64 + stack): PageRank run 77.2 ->
    // 75.4 ms at cfg4 (the u32 min ops are faster at 4)
    static constexpr int kMinBlocks = IPREGEL_PR_MINBLOCKS;
    const double* __restrict__ contrib_cur;
    double* __restrict__ sum_out;             // = contrib_next of the superstep (global ids)
    int64_t vbase;
    const void* gather_base() const { return contrib_cur; }
    __device__ const T* gptr() const { return contrib_cur; }
    __device__ bool absorbed(int32_t) const { return false; }
    __device__ static T message(T g, uint32_t) { return g; }
    __device__ void finish(int32_t row, T sum, LaneCounters&) const { sum_out[vbase + row] = sum; }
};

// Hash-Min CC, Fig. 9, first half: min over the CSC row (in-neighbours' labels).
struct CCPullIn : MinU32, NoAggregate {
    static constexpr bool kWeighted = false;
    static constexpr bool kJumpSettled = true;
#ifndef IPREGEL_CCIN_MINBLOCKS
#define IPREGEL_CCIN_MINBLOCKS 6
#endif
    static constexpr int kMinBlocks = IPREGEL_CCIN_MINBLOCKS;   // 6 CTAs/SM (40 registers + 8 B stack): Hash-Min -0.4 ms vs 4 at cfg4
    static constexpr bool kAbsorbing = true;
    static constexpr bool kAbsorbingPartial = true;
    __device__ static bool absorbing(T x) { return x == 0u; }
    const uint32_t* __restrict__ cur;   // replica, global ids
    uint32_t* __restrict__ next;        // replica, global ids (owned slice written)
    int64_t vbase;
    const void* gather_base() const { return cur; }
    __device__ const T* gptr() const { return cur; }
    // label 0 is the smallest id: a row already at 0 cannot change (skip its gathers)
    __device__ bool absorbed(int32_t row) const { return cur[vbase + row] == 0u; }
    __device__ static T message(T g, uint32_t) { return g; }
    __device__ void finish(int32_t row, T m, LaneCounters&) const {
        const uint32_t c = cur[vbase + row];
        next[vbase + row] = m < c ? m : c;
    }
};

// Hash-Min CC, second half: min over the CSR row (the symmetrised graph's reverse edges), then
// "if value < old: broadcast" -> changed / messages counters (degree in the symmetrised graph).
struct CCPullOut : MinU32, NoAggregate {
    static constexpr bool kWeighted = false;
    static constexpr bool kJumpSettled = true;
#ifndef IPREGEL_CCOUT_MINBLOCKS
#define IPREGEL_CCOUT_MINBLOCKS 5
#endif
    static constexpr int kMinBlocks = IPREGEL_CCOUT_MINBLOCKS;   // 5 CTAs/SM (48 registers): with the two below, Hash-Min 17.0 -> 16.5 ms
    static constexpr bool kAbsorbing = true;
    static constexpr bool kAbsorbingPartial = true;
    __device__ static bool absorbing(T x) { return x == 0u; }
    const uint32_t* __restrict__ cur;
    uint32_t* __restrict__ next;
    const int32_t* __restrict__ in_off;   // owned CSC offsets
    const int32_t* __restrict__ out_off;  // owned CSR offsets
    int64_t vbase;
    PeerSlots<uint32_t> peers;            // fused exchange: other replicas of `next`
    int count_all_zero;                   // aux: every row at label 0 (1), or only the rows that
                                          // reached it in this superstep (0; the host adds them up)
    const void* gather_base() const { return cur; }
    __device__ const T* gptr() const { return cur; }
    __device__ bool absorbed(int32_t row) const { return next[vbase + row] == 0u; }
    __device__ static T message(T g, uint32_t) { return g; }
    __device__ void finish(int32_t row, T m, LaneCounters& c) const {
        const uint32_t old = cur[vbase + row];
        uint32_t v = next[vbase + row];
        v = m < v ? m : v;
        next[vbase + row] = v;
        peers.store(vbase + row, v);
        // degrees only where a counter needs them: the changed rows (messages) and, for the
        // row-list decision, rows at label 0 -- all of them, or only those new at 0 (most rows
        // sit at 0 unchanged after superstep 1: their four offset loads were most of the
        // CSR pass of superstep 2)
        if (v < old || (count_all_zero && v == 0u)) {
            const uint32_t deg = (uint32_t)(in_off[row + 1] - in_off[row]) +
                                 (uint32_t)(out_off[row + 1] - out_off[row]);
            if (v < old) {
                c.changed += 1;
                c.messages += deg;
            }
            if (v == 0u) c.aux += deg;   // rows at label 0 (row-list pull decision)
        }
    }
};

// SSSP, Fig. 10 with weights: message on edge (u -> v, w) is sat(dist_u + w), applied at the
// recipient from the CSC weight (reading R8); "if mindist < value: broadcast".
//
// Absorption bound: every message of superstep s comes from a vertex that changed in s-1 (E1), so
// it is >= thr = sat(m + w_min), m the smallest distance that changed in s-1 and w_min the
// smallest edge weight; a row already at or below thr -- or whose partial reaches thr -- cannot
// change, and its remaining gathers are skipped.  finish() reports m for the next superstep (as
// INF - dist in the max-reduced dmax counter).
struct SSSPPull : MinU32, NoAggregate {
    static constexpr bool kWeighted = true;
#ifndef IPREGEL_SSSP_MINBLOCKS
#define IPREGEL_SSSP_MINBLOCKS 5
#endif
    static constexpr int kMinBlocks = IPREGEL_SSSP_MINBLOCKS;   // 5 CTAs/SM (48 registers + 32 B stack): SSSP 13.4 -> 12.8 ms (6: 72 B stack, 15.5 ms)
    static constexpr bool kAbsorbing = true;
    static constexpr bool kAbsorbingPartial = true;
    const uint32_t* __restrict__ cur;
    uint32_t* __restrict__ next;
    const int32_t* __restrict__ out_off;  // owned CSR offsets
    int64_t vbase;
    PeerSlots<uint32_t> peers;            // fused exchange: other replicas of `next`
    uint32_t thr;                         // absorption bound (0: none below the source)
    const void* gather_base() const { return cur; }
    __device__ const T* gptr() const { return cur; }
    __device__ bool absorbed(int32_t row) const { return cur[vbase + row] <= thr; }
    __device__ bool absorbing(T x) const { return x <= thr; }
    __device__ static T message(T g, uint32_t w) { return sat_add(g, w); }
    __device__ void finish(int32_t row, T m, LaneCounters& c) const {
        const uint32_t old = cur[vbase + row];
        const uint32_t v = m < old ? m : old;
        next[vbase + row] = v;
        peers.store(vbase + row, v);
        if (v < old) {
            c.changed += 1;
            c.messages += (uint32_t)(out_off[row + 1] - out_off[row]);
            const unsigned long long inv = (unsigned long long)(kInf - v);
            c.dmax = inv > c.dmax ? inv : c.dmax;
        }
    }
};

// ---- one warp, one range -----------------------------------------------------------------------
// A chunk is 128 consecutive edges on the global grid, held as 4 sub-chunks of 32: lane l owns
// edges e0 + 32k + l (k = 0..3), so each gather instruction of the warp reads the sources of 32
// CONSECUTIVE edges.  CSC rows list their sources in ascending order, so consecutive edges of a
// row often share a 128-byte line and the coalescer merges their requests (the L1 -> L2 request
// rate is what bounds this kernel; profiles/r01).
struct ChunkLoad {
    int32_t idx[4];   // column index of edge e0 + 32k + lane (-1 = outside the partition/range)
    uint32_t w[4];    // weights (SSSP; 1 otherwise)
};

template <bool kWeighted>
__device__ __forceinline__ ChunkLoad load_chunk(const int32_t* __restrict__ idx,
                                                const uint32_t* __restrict__ wts, int32_t e0,
                                                int32_t lo, int32_t hi, int lane, uint64_t pol,
                                                bool skip = false) {
    ChunkLoad L;
    if (skip) {   // warp-uniform: the chunk's messages cannot change its (absorbed) row
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            L.idx[k] = -1;
            L.w[k] = 1u;
        }
        return L;
    }
    if (e0 >= lo && e0 + kChunk <= hi) {   // warp-uniform: interior chunk, no bounds checks
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int32_t e = e0 + 32 * k + lane;
            L.idx[k] = ld_stream(idx + e, pol);
            L.w[k] = (kWeighted && wts) ? ld_stream(wts + e, pol) : 1u;
        }
        return L;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int32_t e = e0 + 32 * k + lane;
        const bool in = e >= lo && e < hi;
        L.idx[k] = in ? ld_stream(idx + e, pol) : -1;
        L.w[k] = (kWeighted && in && wts) ? ld_stream(wts + e, pol) : 1u;
    }
    return L;
}

// Outbox gathers.  l1hot < 0: default L1 allocation; else vertices below l1hot are cached in L1
// (evict-last) and the rest bypass L1 (tuning knob IPREGEL_L1_HOT).
template <class Op>
__device__ __forceinline__ typename Op::T gather_one(const Op& op, int32_t u, uint64_t pol,
                                                     int32_t l1hot) {
    if (u < 0) return Op::identity();
    if (l1hot < 0) return ld_gather(op.gptr() + u, pol);
    return ld_gather_l1(op.gptr() + u, pol, u < l1hot);
}

template <class Op>
__device__ __forceinline__ void gather_chunk(const Op& op, const ChunkLoad& L,
                                             typename Op::T (&g)[4], uint64_t pol, int32_t l1hot,
                                             bool skip = false) {
#pragma unroll
    for (int k = 0; k < 4; ++k) g[k] = gather_one(op, skip ? -1 : L.idx[k], pol, l1hot);
}

struct RangeArgs {
    const int32_t* off;
    const int32_t* idx;
    const uint32_t* wts;
    const int32_t* cx;
    const int32_t* cy;
    int32_t rows;
    int32_t cphase;
    int32_t num_ranges;
    void* carry_out;
    void* head_out;
    PullCounters* counters;
    int gather_policy;
    const void* gbase;
    uint32_t ghot, gtotal;
    int32_t l1hot;
    int32_t* range_ctr;   // non-null: warps take ranges from this zeroed counter (dynamic)
    int32_t order;        // dynamic range order (knob IPREGEL_RANGE_ORDER, see k_pull_ranges)
};

// counters: warp reduce, one shared atomic per warp, one global atomic per CTA
__device__ __forceinline__ void flush_counters(const LaneCounters& cnt, unsigned long long* s_cnt,
                                               PullCounters* counters) {
    const int lane = threadIdx.x & 31;
    unsigned long long c0 = cnt.changed, c1 = cnt.messages, c2 = cnt.dmax, c3 = cnt.aux;
    unsigned long long c4 = cnt.gathered;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        c0 += __shfl_xor_sync(kFull, c0, d);
        c1 += __shfl_xor_sync(kFull, c1, d);
        const unsigned long long o = __shfl_xor_sync(kFull, c2, d);
        c2 = o > c2 ? o : c2;
        c3 += __shfl_xor_sync(kFull, c3, d);
        c4 += __shfl_xor_sync(kFull, c4, d);
    }
    if (lane == 0 && (c0 | c1 | c2 | c3 | c4)) {
        atomicAdd(&s_cnt[0], c0);
        atomicAdd(&s_cnt[1], c1);
        atomicMax(&s_cnt[2], c2);
        atomicAdd(&s_cnt[3], c3);
        atomicAdd(&s_cnt[4], c4);
    }
    __syncthreads();
    if (threadIdx.x == 0 && counters && (s_cnt[0] | s_cnt[1] | s_cnt[2] | s_cnt[3] | s_cnt[4])) {
        atomicAdd(&counters->changed, s_cnt[0]);
        atomicAdd(&counters->messages, s_cnt[1]);
        atomicMax(&counters->dmax, s_cnt[2]);
        atomicAdd(&counters->aux, s_cnt[3]);
        atomicAdd(&counters->gathered, s_cnt[4]);
    }
}

template <class Op, class = void> struct ReduxMin { static constexpr bool value = false; };
template <class Op> struct ReduxMin<Op, void_t_<decltype(Op::kReduxMin)>> {
    static constexpr bool value = Op::kReduxMin;
};

// Fixed xor-tree reduction of a lane-private partial (result on every lane); u32 min ops use
// the warp-reduce instruction (min is order-independent, so exact either way).
template <class Op>
__device__ __forceinline__ typename Op::T warp_fold(typename Op::T x) {
    if constexpr (ReduxMin<Op>::value) return __reduce_min_sync(kFull, x);
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const typename Op::T o = shfl_xor(x, d);
        x = (lane & d) ? Op::combine(o, x) : Op::combine(x, o);
    }
    return x;
}

// Two lane-private partials reduced at once (results on every lane): the first xor step
// pairs a over the low half-warp and b over the high one, so both take 5 + 2 shuffles
// instead of 2 x 5.  The one-end chunks and the general ones close the first and last
// segments of a chunk with this same tree (bit-identical partitioned views).
template <class Op>
__device__ __forceinline__ void warp_fold2(typename Op::T a, typename Op::T b,
                                           typename Op::T& fa, typename Op::T& fb) {
    using T = typename Op::T;
    const int lane = threadIdx.x & 31;
    const bool hi = lane & 16;
    const T o = shfl_xor(hi ? a : b, 16);
    T x = hi ? Op::combine(o, b) : Op::combine(a, o);
#pragma unroll
    for (int d = 1; d < 16; d <<= 1) {
        const T y = shfl_xor(x, d);
        x = (lane & d) ? Op::combine(y, x) : Op::combine(x, y);
    }
    fa = shfl_idx(x, 0);
    fb = shfl_idx(x, 16);
}

__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// Ops that jump over the settled chunks of an absorbed row (kJumpSettled, pull_range).
template <class Op, class = void> struct JumpSettled { static constexpr bool value = false; };
template <class Op> struct JumpSettled<Op, void_t_<decltype(Op::kJumpSettled)>> {
    static constexpr bool value = Op::kJumpSettled;
};
#ifndef IPREGEL_JUMP_CHUNKS
#define IPREGEL_JUMP_CHUNKS 8   // 3 / 8 / 16 / 32 / 128 within 0.1 ms at cfg4
#endif
constexpr int32_t kJumpChunks = IPREGEL_JUMP_CHUNKS;

// One warp, one range q (see the file header).  `my_sum` is the warp's sum array: 128 slots
// by chunk position + 2 for the first / last segment of 8-byte chunks.
template <class Op>
__device__ __forceinline__ void pull_range(const Op& op, const RangeArgs& A, int64_t q,
                                           typename Op::T* my_sum, LaneCounters& cnt) {
    using T = typename Op::T;
    const int lane = threadIdx.x & 31;
    const uint64_t pol_s = policy_evict_first();
    const uint64_t pol_g = policy_for(A.gather_policy, A.gbase, A.ghot, A.gtotal);
    const int32_t x1 = A.cx[q + 1], y0 = A.cy[q], y1 = A.cy[q + 1];
    int32_t r = A.cx[q];                           // next row to finish
    int32_t Bc = r < A.rows ? A.off[r] : y1;       // first edge of row r
    int32_t Ec = r < A.rows ? A.off[r + 1] : y1;   // end of row r
    int32_t En = r + 1 < A.rows ? A.off[r + 2] : INT_MAX;   // end of row r + 1
    // the row entering the range with edges before it is finished by k_pull_fixup
    const int32_t defer = (q > 0 && r < A.rows && Bc < y0) ? r : -1;
    T carry = Op::identity();   // partial of row r from earlier slow chunks
    T la = Op::identity();      // lane-private partial of row r from fast chunks
    bool absorbed = r < x1 && op.absorbed(r);
    // chunks on the global 128-edge grid covering [y0, y1)
    const int32_t c0 = y0 - ((y0 + A.cphase) & (kChunk - 1));

    if constexpr (Op::kAbsorbing) {
        // every row of the range (and the one leaving it) is settled: no gather can change any
        // of them, so finish them straight away (runs of short rows the chunk skip cannot catch)
        const int32_t last = y1 > (x1 < A.rows ? A.off[x1] : y1) ? x1 : x1 - 1;
        bool all = true;
        for (int32_t row = r + lane; row <= last && all; row += 32)
            all = op.absorbed(row);
        if (__all_sync(kFull, all)) {
            for (int32_t row = r + lane; row < x1; row += 32) {
                if (row == defer) static_cast<T*>(A.head_out)[q] = Op::identity();
                else op.finish(row, Op::identity(), cnt);
            }
            if (lane == 0) static_cast<T*>(A.carry_out)[q] = Op::identity();
            return;
        }
    }

    // software pipeline: indices two chunks ahead, gathered values one chunk ahead
    ChunkLoad Lc = load_chunk<Op::kWeighted>(A.idx, A.wts, c0, y0, y1, lane, pol_s);
    ChunkLoad Ln = load_chunk<Op::kWeighted>(A.idx, A.wts, c0 + kChunk, y0, y1, lane, pol_s);
    T gc[4];
    gather_chunk(op, Lc, gc, pol_g, A.l1hot);
    // absorbing ops count the edges they gather (superstep model bytes, bench.py)
    auto count_gathered = [&](int32_t cpos) {
        if constexpr (Op::kAbsorbing) {
            const int32_t a = cpos > y0 ? cpos : y0;
            const int32_t b = cpos + kChunk < y1 ? cpos + kChunk : y1;
            if (lane == 0 && b > a) cnt.gathered += (uint32_t)(b - a);
        }
    };
    count_gathered(c0);

#pragma unroll kChunkUnroll
    for (int32_t e0 = c0; e0 < y1; e0 += kChunk) {
        if constexpr (JumpSettled<Op>::value) {
            // the open row is settled and runs on for several chunks: jump straight to the
            // chunk holding its end (or the range's last chunk) and restart the pipeline there
            // instead of stepping through chunks whose gathers are all skipped.  Hash-Min only:
            // measured at cfg4, Hash-Min 16.96 -> 16.6 ms, while SSSP (settled rows are shorter,
            // each jump exposes the restarted pipeline's latency) went 12.8 -> 14.4-14.8 ms at
            // 4, 5 or 6 CTAs per SM.
            if (absorbed && r < x1 && e0 >= 0) {
                const int32_t t = (Ec < y1 ? Ec : y1) - 1;
                const int32_t ej = t - ((t + A.cphase) & (kChunk - 1));
                if (ej >= e0 + kJumpChunks * kChunk) {   // warp-uniform
                    e0 = ej;
                    Lc = load_chunk<Op::kWeighted>(A.idx, A.wts, e0, y0, y1, lane, pol_s);
                    Ln = load_chunk<Op::kWeighted>(A.idx, A.wts, e0 + kChunk, y0, y1, lane, pol_s);
                    gather_chunk(op, Lc, gc, pol_g, A.l1hot);
                    count_gathered(e0);
                }
            }
        }
        T gn[4];
        // the next chunk lies inside an absorbed open row: its messages cannot change it
        const bool skip_next = absorbed && r < x1 && Ec > e0 + 2 * kChunk;
        gather_chunk(op, Ln, gn, pol_g, A.l1hot, skip_next);
        if (!skip_next) count_gathered(e0 + kChunk);
        uint32_t wc[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) wc[k] = Lc.w[k];
        Lc = Ln;
        Ln = load_chunk<Op::kWeighted>(A.idx, A.wts, e0 + 2 * kChunk, y0, y1, lane, pol_s,
                                       absorbed && r < x1 && Ec > e0 + 3 * kChunk);
#if IPREGEL_IDX_PREFETCH > 0
        {
            // the index (and weight) stream further ahead into L2: under the gathers' load the
            // DRAM latency of the loads two chunks ahead is not covered (ncu: the top stall)
            const int32_t pc = e0 + IPREGEL_IDX_PREFETCH * kChunk;
            const int32_t pe = pc + 4 * lane;
            if (pe < y1 && !(absorbed && r < x1 && Ec > pc + kChunk)) {
                prefetch_l2(A.idx + pe);
                if (Op::kWeighted && A.wts) prefetch_l2(A.wts + pe);
            }
        }
#endif
        T v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            v[k] = Op::message(gc[k], wc[k]);
            gc[k] = gn[k];
        }

        // The partition's first chunk when its first edge is not on the 128-edge grid: on one
        // GPU the previous partition's last row ends there, so it takes the slow path with a
        // segment head at the partition start (same combine tree for any partition).
        const bool part_head = e0 < 0;
        if (!part_head && (r >= x1 || Ec > e0 + kChunk)) {
            // fast path: the whole chunk belongs to row r (no row ends here)
            la = Op::combine(la, Op::combine(Op::combine(v[0], v[1]), Op::combine(v[2], v[3])));
            if constexpr (Op::kAbsorbingPartial) {
                // the open row's partial reached the absorbing value: skip its remaining gathers
                if (!absorbed) absorbed = __any_sync(kFull, op.absorbing(la));
            }
            continue;
        }
        if ((sizeof(T) == 8 || (IPREGEL_U32_ONE_END && ReduxMin<Op>::value)) && !part_head &&
            Ec > e0 && En > e0 + kChunk) {
            // exactly one row (r) ends inside the chunk and the next one runs past it -- the
            // common case for rows of a few hundred edges: two masked warp folds instead of the
            // segmented scan (positions < p close row r, the rest open row r + 1).  8-byte values
            // only: the 64-bit scan is what is expensive (measured: PageRank -6 %, while the u32
            // min programs ran 3-4 % slower with it)
            const int32_t p = Ec - e0;   // in [1, kChunk]
            T t1 = Op::identity(), t2 = Op::identity();
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (32 * k + lane < p) t1 = Op::combine(t1, v[k]);
                else t2 = Op::combine(t2, v[k]);
            }
            T f1, f2;
            if constexpr (ReduxMin<Op>::value) {   // two warp-reduce instructions
                f1 = __reduce_min_sync(kFull, t1);
                f2 = __reduce_min_sync(kFull, t2);
            } else {
                warp_fold2<Op>(t1, t2, f1, f2);
            }
            const T total = Op::combine(Op::combine(carry, warp_fold<Op>(la)), f1);
            carry = f2;
            la = Op::identity();
            if (lane == 0) {
                if (r == defer) static_cast<T*>(A.head_out)[q] = total;
                else op.finish(r, total, cnt);
            }
            r += 1;
            Bc = Ec;
            Ec = En;
            En = r + 1 < A.rows ? A.off[r + 2] : INT_MAX;
            absorbed = r < x1 && op.absorbed(r);
            if constexpr (Op::kAbsorbingPartial) {
                if (!absorbed && r < x1) absorbed = op.absorbing(carry);
            }
            continue;
        }
        // slow path: rows end in this chunk.  Fold the lane partials of row r first.
        carry = Op::combine(carry, warp_fold<Op>(la));
        la = Op::identity();

        // head flags: word k bit l <=> a row ends at chunk position 32k + l (in [1, 127])
        uint32_t f[4] = {0u, 0u, 0u, 0u};
        int32_t n_emit = 0;
        int32_t E0 = 0;   // window 0's row end for this lane (reused by the emission)
        int32_t pl = -e0;  // last row end in the chunk (the partition start if none)
        for (int32_t rw = r;; rw += 32) {
            const int32_t row = rw + lane;
            const int32_t E = row < x1 ? A.off[row + 1] : INT_MAX;
            if (rw == r) E0 = E;
            const int32_t p = E == INT_MAX ? INT_MAX : E - e0;
            const bool fl = p >= 1 && p <= 127;
            const uint32_t bit = fl ? 1u << (p & 31) : 0u;
            const int word = fl ? (p >> 5) : -1;
#pragma unroll
            for (int k = 0; k < 4; ++k) f[k] |= __reduce_or_sync(kFull, word == k ? bit : 0u);
            const int n = __popc(__ballot_sync(kFull, p <= kChunk));
            if (sizeof(T) == 8 && n > 0) pl = shfl_idx(p, n - 1);
            n_emit += n;
            if (n < 32) break;
        }
        if (part_head) {
            const int p = -e0;   // in [1, 127]
            f[p >> 5] |= 1u << (p & 31);
        }
        if constexpr (sizeof(T) == 8) {
            // the first segment (the open row r, unless the partition starts in this chunk) and
            // the last one (the row running past the chunk) are closed with the same masked
            // folds as the one-end chunks above; only rows wholly inside the chunk use the
            // scan.  Each row's combine tree then depends on its own ends only, not on how
            // many other rows end in the chunk -- which differs between a partition's view and
            // the whole graph's at partition boundaries -- so any partitioning reduces every
            // row bit-identically (E4)
            const int32_t p1 = part_head ? 0 : Ec - e0;
            T t1 = Op::identity(), t2 = Op::identity();
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int32_t pos = 32 * k + lane;
                if (pos < p1) t1 = Op::combine(t1, v[k]);
                else if (pos >= pl) t2 = Op::combine(t2, v[k]);
            }
            T f1, f2;
            warp_fold2<Op>(t1, t2, f1, f2);
            if (lane == 0) {
                my_sum[4 * 32] = Op::combine(carry, f1);
                my_sum[4 * 32 + 1] = f2;
            }
            carry = Op::identity();
        }

        // segmented scan over positions 0..127: 4 independent warp scans (segment starts from
        // the uniform flag words), then the carries are chained through the sub-chunks
        int start[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t m = f[k] & (0xFFFFFFFFu >> (31 - lane));   // flags at lanes <= l
            start[k] = m ? 31 - __clz(m) : -1;
        }
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const T y = shfl_up(v[k], d);
                if (lane >= d && lane - d >= start[k]) v[k] = Op::combine(y, v[k]);
            }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (start[k] < 0) v[k] = Op::combine(carry, v[k]);
            carry = shfl_idx(v[k], 31);
            my_sum[k * 32 + lane] = v[k];
        }
        T next_carry = carry;
        __syncwarp();

        // emit every row ending here: sum = S(p - 1); rows without in-edges get identity
        bool ended_at_end = false;
        for (int32_t k = 0; k < n_emit; k += 32) {
            const int32_t row = r + k + lane;
            const int32_t E = k == 0 ? E0 : (row < x1 ? A.off[row + 1] : INT_MAX);
            int32_t B = shfl_up(E, 1);
            const int32_t Bw = k == 0 ? Bc : A.off[r + k];   // start of the window's first row
            if (lane == 0) B = Bw;
            if (k + lane < n_emit) {
                T val = Op::identity();
                if (B < E) {
                    const int pos = E - e0 - 1;
                    val = pos >= 0 ? my_sum[(sizeof(T) == 8 && k + lane == 0 && !part_head)
                                                ? 4 * 32 : pos] : Op::identity();
                    if (E - e0 == kChunk) ended_at_end = true;
                }
                if (row == defer) static_cast<T*>(A.head_out)[q] = val;
                else op.finish(row, val, cnt);
            }
        }
        r += n_emit;
        Bc = r < A.rows ? A.off[r] : y1;
        Ec = r < A.rows ? A.off[r + 1] : y1;
        En = r + 1 < A.rows ? A.off[r + 2] : INT_MAX;
        absorbed = r < x1 && op.absorbed(r);
        if (__any_sync(kFull, ended_at_end)) next_carry = Op::identity();
        carry = sizeof(T) == 8 ? my_sum[4 * 32 + 1] : next_carry;
        if constexpr (Op::kAbsorbingPartial) {
            if (!absorbed && r < x1) absorbed = op.absorbing(carry);   // carry is warp-uniform
        }
        __syncwarp();
    }
    // rows finished after the last edge of the range (rows without in-edges)
    for (int32_t row = r + lane; row < x1; row += 32) {
        if (row == defer) static_cast<T*>(A.head_out)[q] = Op::identity();
        else op.finish(row, Op::identity(), cnt);
    }
    // partial of the row leaving the range
    const T out = Op::combine(carry, warp_fold<Op>(la));
    if (lane == 0) static_cast<T*>(A.carry_out)[q] = out;
}

template <class Op>
__global__ void __launch_bounds__(kPullThreads, PullMinBlocks<Op>::value) k_pull_ranges(Op op, RangeArgs A) {
    using T = typename Op::T;
    __shared__ T s_sum[kWarpsPerCta][4 * 32 + 2];   // chunk sums by position (conflict-free)
    __shared__ unsigned long long s_cnt[5];
    const int wid = threadIdx.x >> 5;
    const int64_t q = (int64_t)blockIdx.x * kWarpsPerCta + wid;
    if (threadIdx.x < 5) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    LaneCounters cnt{0u, 0u, 0u, 0ull, 0.0, 0u};
    // warps stride over the ranges independently (the grid may be smaller than one warp per
    // range): no warp waits for the slowest warp of its CTA before taking its next range
    if (A.range_ctr) {
        // dynamic: the next range index is fetched while the current one runs
        const int lane = threadIdx.x & 31;
        int32_t r = lane == 0 ? atomicAdd(A.range_ctr, 1) : 0;
        r = __shfl_sync(kFull, r, 0);
        const int32_t per = A.order >= 2 ? (A.num_ranges + A.order - 1) / A.order : 0;
        const int32_t limit = A.order >= 2 ? per * A.order : A.num_ranges;
        while (r < limit) {
            const int32_t nx = lane == 0 ? atomicAdd(A.range_ctr, 1) : 0;
            // order of the ranges in time (knob): 1 = alternate between the two ends of the
            // plan, so long-row ranges (low ids under the degree layout) and short-row ranges
            // run side by side; the result of every range is the same either way
            int32_t q = r;
            if (A.order == 1) {
                q = (r & 1) ? A.num_ranges - 1 - (r >> 1) : (r >> 1);
            } else if (A.order >= 2) {
                // A.order interleaved streams over equal slices of the plan (a bijection of
                // [0, per * order) onto slice-major positions; those past the plan are skipped)
                q = (r % A.order) * per + r / A.order;
                if (q >= A.num_ranges) q = -1;
            }
            if (q >= 0) pull_range<Op>(op, A, q, s_sum[wid], cnt);
            r = __shfl_sync(kFull, nx, 0);
        }
    } else {
        const int64_t nw = (int64_t)gridDim.x * kWarpsPerCta;
        for (int64_t r = q; r < A.num_ranges; r += nw) pull_range<Op>(op, A, r, s_sum[wid], cnt);
    }
    flush_counters(cnt, s_cnt, A.counters);
    if constexpr (Op::kAggregates) op.flush_aggregate(cnt);
    if constexpr (HasMass<Op>::value) if (op.mass) flush_mass(cnt, op.mass);
}

// Fig. 8's update of every owned row from the sum PageRankSum left in its next-outbox slot.  A
// thread takes kPrFinishRows rows (block-strided, coalesced) with their sums loaded up front.
#ifndef IPREGEL_PR_FINISH_ROWS
#define IPREGEL_PR_FINISH_ROWS 4
#endif
constexpr int kPrFinishRows = IPREGEL_PR_FINISH_ROWS;
// kMode: 0 general (runtime flags: to-convergence / mass-check runs), 1 broadcast only
// (supersteps 1 .. k-1 of a fixed-k run), 2 rank only (superstep k).  The fixed-k variants fix
// the flags at compile time: with them at run time the compiler versioned the row loop and the
// kernel ran 2.3x the instructions (0.31 vs 0.16 ms at cfg4).  kCompact: the sums come from the
// flagged superstep (pr_flag.cuh) by ordinal -- row v with in-edges has ordinal nzpre[v / 32] +
// (rows with in-edges below v in its bitmap word); rows without in-edges sum to 0.
template <int kMode, bool kCompact = false, int kRows = kPrFinishRows>
__global__ void __launch_bounds__(256) k_pr_finish(PageRankPull op, int64_t rows,
                                                   PullCounters* counters) {
    __shared__ unsigned long long s_cnt[5];
    if (kMode == 0 && counters && threadIdx.x < 5) s_cnt[threadIdx.x] = 0;
    if constexpr (kMode != 0) {
        op.broadcast = kMode == 1;
        op.write_rank = kMode == 2;
        op.track = 0;
        op.mass = nullptr;
    }
    LaneCounters c{0u, 0u, 0u, 0ull};
    const int64_t base = (int64_t)blockIdx.x * blockDim.x * kRows + threadIdx.x;
    const bool need_deg = op.broadcast || op.mass;
    double sum[kRows];
    int32_t deg[kRows];
    if constexpr (kCompact) {
        // branch-free: every thread loads its words, then the sums at the ordinals (sumc holds
        // nnz + 1 slots, so the ordinal of a row without in-edges -- at most nnz -- is in bounds)
        uint32_t w[kRows];
        int32_t pre[kRows];
#pragma unroll
        for (int j = 0; j < kRows; ++j) {
            const int64_t row = base + (int64_t)j * blockDim.x;
            const int64_t rr = row < rows ? row : 0;
            w[j] = op.nzbits[rr >> 5];
            pre[j] = op.nzpre[rr >> 5];
            deg[j] = row < rows && need_deg ? op.out_off[row + 1] - op.out_off[row] : 0;
        }
#pragma unroll
        for (int j = 0; j < kRows; ++j) {
            const int64_t row = base + (int64_t)j * blockDim.x;
            const uint32_t bit = 1u << (row & 31);
            const double v = op.sumc[pre[j] + __popc(w[j] & (bit - 1u))];
            sum[j] = (row < rows && (w[j] & bit)) ? v : 0.0;
        }
    } else {
#pragma unroll
        for (int j = 0; j < kRows; ++j) {
            const int64_t row = base + (int64_t)j * blockDim.x;
            sum[j] = row < rows ? op.contrib_next[op.vbase + row] : 0.0;
            deg[j] = row < rows && need_deg ? op.out_off[row + 1] - op.out_off[row] : 0;
        }
    }
#pragma unroll
    for (int j = 0; j < kRows; ++j) {
        const int64_t row = base + (int64_t)j * blockDim.x;
        if (row < rows) op.finish_deg((int32_t)row, sum[j], deg[j], c);
    }
    if constexpr (kMode == 0) {
        if (counters) {   // to-convergence runs only (grid-uniform)
            __syncthreads();
            flush_counters(c, s_cnt, counters);
        }
        if (op.mass) flush_mass(c, op.mass);
    }
}

// Rows cut by range boundaries: boundaries a..b (1 <= a <= b) carry row r; its value is
// carry[a-1] (+) carry[a] (+) ... (+) carry[b-1] (+) head[b], folded in a fixed order that
// depends on the span only (ranges sit on the global grid, so on every partitioning alike):
//   groups [0, num_short) span <= kFixupShortSpan boundaries: one thread each, a left fold;
//   the rest (hub rows): one warp each, lane-strided partials then a fixed xor tree.
// The first ceil(num_short / blockDim) blocks take the short groups (grid: fixup_grid()).
constexpr int32_t kFixupShortSpan = 16;
inline unsigned fixup_grid(int32_t num_groups, int32_t num_short) {
    return (unsigned)((num_short + 255) / 256 + ((int64_t)(num_groups - num_short) * 32 + 255) / 256);
}
template <class Op>
__global__ void k_pull_fixup(Op op, const int4* __restrict__ groups, int32_t num_groups,
                             int32_t num_short, const typename Op::T* __restrict__ carry,
                             const typename Op::T* __restrict__ head,
                             PullCounters* __restrict__ counters) {
    using T = typename Op::T;
    __shared__ unsigned long long s_cnt[5];
    const int lane = threadIdx.x & 31;
    if (threadIdx.x < 5) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    LaneCounters c{0u, 0u, 0u, 0ull, 0.0, 0u};
    const int32_t short_blocks = (num_short + (int32_t)blockDim.x - 1) / (int32_t)blockDim.x;
    if ((int32_t)blockIdx.x < short_blocks) {
        const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
        if (g < num_short) {
            const int4 G = groups[g];
            T acc = carry[G.y - 1];
            for (int t = G.y; t <= G.z - 1; ++t) acc = Op::combine(acc, carry[t]);
            op.finish(G.x, Op::combine(acc, head[G.z]), c);
        }
    } else {
        const int64_t g =
            num_short + (((int64_t)(blockIdx.x - short_blocks) * blockDim.x + threadIdx.x) >> 5);
        if (g < num_groups) {
            const int4 G = groups[g];
            T acc = Op::identity();
            for (int t = G.y - 1 + lane; t <= G.z - 1; t += 32) acc = Op::combine(acc, carry[t]);
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const T o = shfl_xor(acc, d);
                acc = (lane & d) ? Op::combine(o, acc) : Op::combine(acc, o);
            }
            if (lane == 0) {
                acc = Op::combine(acc, head[G.z]);
                op.finish(G.x, acc, c);
            }
        }
    }
    // one global atomic per CTA (not per group: the counters are shared by every group)
    flush_counters(c, s_cnt, counters);
    if constexpr (Op::kAggregates) op.flush_aggregate(c);
    if constexpr (HasMass<Op>::value) if (op.mass) flush_mass(c, op.mass);
}

}  // namespace ipr
