// paper_2010_08781_b200/csrc/pr_flag.cuh -- PageRank gather superstep over a row-end-flagged CSC.
//
// PAPER.md:199-203 (Sec. 4.3.2, pull delivery) run on Fig. 8: every recipient
// sums contrib[u] = r_u / outdeg(u) over its in-neighbours.  This is the same gather-combine as
// k_pull_ranges<PageRankSum> (pull.cuh) with the row bookkeeping moved out of the loop:
//
//  * the CSC index of each row's LAST edge carries bit 31 (fidx, a library copy of the CSC indices,
//    built once per graph before its first PageRank pull run).  A warp learns where rows end from
//    the index words it loads anyway: four ballots per 128-edge chunk, no offset loads, no
//    dependent latency.  Rows are numbered by their ORDINAL among rows with in-edges (the count
//    of ends before them), so a warp knows which row every end closes from a running count;
//  * ranges are 64 chunks (8192 edges) on the GLOBAL edge grid, warps take them from a counter
//    alternately from the two ends of the plan (as the range kernels);
//  * the combine tree of a row depends on its own edges' global positions only, whatever the
//    partitioning: chunks inside a row add into lane-private partials
//    (lane l holds positions = l mod 32); in a chunk where rows end, the row entering the chunk
//    (the lane partials folded in) and the row leaving it are closed by the paired warp fold
//    (warp_fold2) over positions before the first end / after the last end; rows wholly inside
//    the chunk are summed lane-sequentially after a shared-memory transpose (lane l holds
//    positions 4l .. 4l+3) and joined across lanes by one 5-step segmented scan.  A partition
//    whose first edge is not on the range grid sees the previous partition's last row end as a
//    phantom end at local position -1, so its first row starts a segment exactly as in the whole
//    graph's view;
//  * sums are stored by ordinal (sumc); k_pr_finish maps rows to ordinals with a bitmap of the
//    rows with in-edges plus a per-word prefix count, and rows without in-edges take sum 0;
//  * a row cut by range boundaries leaves its partial in carry[] of every range it runs through
//    and its last piece in head[]; k_flag_fixup joins them in k_pull_fixup's fixed order (the
//    groups found on the device by k_flag_groups when the plan is built).  Building the plan
//    takes no host round trip (it runs inside the first PageRank run, which end-to-end callers
//    time).
//
// The kernel runs at ~0.95 of its gather-request limit (one L1 -> L2 request per SM per clock;
// ncu: request path 89 % busy, L2 tag lookups 84 %, DRAM 42 %; profiles/r02/prf_ncu_full_s38.json).
//
// Why (profiles/r02/README.md, tools/meta_lab.cu): the range kernel's time over the raw gather
// stream went to its row logic -- CSC offset loads on the critical path and ~80 shuffles per chunk
// with several row ends (the L1 data pipe also serves the gathers).  Measured on the cfg4 CSC
// without range joins: raw stream 5.56 ms, offsets-driven bookkeeping 6.3-6.5 ms, this scheme
// 5.9-6.0.
#pragma once
#include "pull.cuh"

namespace ipr {

constexpr int kFlagChunks = 64;                    // chunks per range
constexpr int64_t kFlagRange = kFlagChunks * kChunk;   // 8192 edges per range
constexpr int32_t kFlagNoEdge = 0x7FFFFFFF;        // masked position: no gather, no end
constexpr int32_t kFlagPhantom = -1;               // masked position holding an end (bit 31)

// What the flagged PageRank superstep needs for one partition (built by ensure_flag_plan).
struct FlagPlan {
    bool ready = false;
    int64_t edges = 0;
    int32_t rows = 0;
    int64_t rphase = 0;          // (global edge index of local edge 0) mod kFlagRange
    int32_t num_ranges = 0;
    int32_t* fidx = nullptr;     // [edges] CSC indices, bit 31 set on each row's last edge
    int2* rinfo = nullptr;       // [num_ranges] (ordinal of the range's first row, it started
                                 // before the range); range 0 after a phantom end: (-1, 0)
    uint32_t* nzbits = nullptr;  // [ceil(rows / 32)] rows with in-edges
    int32_t* nzpre = nullptr;    // [ceil(rows / 32)] rows with in-edges before each word
    double* sumc = nullptr;      // [rows + 1] combined sums by ordinal (ordinals < rows; + 1:
                                 // k_pr_finish's slack slot)
    double* carry = nullptr;     // [num_ranges] partial of the row leaving the range
    double* head = nullptr;      // [num_ranges] last piece of the row entering the range
    int32_t* ctr = nullptr;      // range counter (zeroed before each launch)
    int2* rowdeg = nullptr;      // [rows] by ordinal: (row, out-degree) of each row with in-edges
                                 // (the fused update, k_pr_flag<true>)
    int4* gshort = nullptr;      // rows cut by range boundaries (ordinal, a, b, 0): spans <= 16
    int4* glong = nullptr;       //   and longer spans (hub rows), [num_ranges] each
    int32_t* gcount = nullptr;   // [2] their counts (device)
};

// ---- build ---------------------------------------------------------------------------------
// One warp per 32 rows: the bitmap word of the rows with in-edges, its count, and bit 31 on the
// last edge of each of them (fidx holds a copy of the indices already).
__global__ void k_flag_rows(const int32_t* __restrict__ off, int64_t rows, int32_t* __restrict__ fidx,
                            uint32_t* __restrict__ nzbits, int32_t* __restrict__ nzcnt) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    bool nz = false;
    if (r < rows) {
        const int32_t b = off[r], e = off[r + 1];
        nz = e > b;
        if (nz) fidx[e - 1] |= (int32_t)0x80000000u;
    }
    const uint32_t w = __ballot_sync(kFull, nz);
    if (lane == 0 && r < rows) {
        nzbits[r >> 5] = w;
        nzcnt[r >> 5] = __popc(w);
    }
}

// Range R starts at local edge max(0, R * kFlagRange - rphase): its first row (binary search over
// the offsets), that row's ordinal, and whether it started before the range.
__global__ void k_flag_ranges(const int32_t* __restrict__ off, int32_t rows, int64_t edges,
                              int64_t rphase, int32_t num_ranges,
                              const uint32_t* __restrict__ nzbits,
                              const int32_t* __restrict__ nzpre, int2* __restrict__ rinfo) {
    const int64_t R = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (R >= num_ranges) return;
    if (R == 0 && rphase > 0) {   // the phantom end at local -1 closes "row -1" first
        rinfo[0] = make_int2(-1, 0);
        return;
    }
    const int64_t e = R * kFlagRange - rphase > 0 ? R * kFlagRange - rphase : 0;
    // first row r with off[r + 1] > e (it holds edge e)
    int32_t lo = 0, hi = rows - 1;
    while (lo < hi) {
        const int32_t m = (int32_t)(((int64_t)lo + hi) >> 1);
        if ((int64_t)off[m + 1] > e) hi = m; else lo = m + 1;
    }
    const uint32_t w = nzbits[lo >> 5];
    const int32_t ord = nzpre[lo >> 5] + __popc(w & ((1u << (lo & 31)) - 1u));
    rinfo[R] = make_int2(ord, (int64_t)off[lo] < e ? 1 : 0);
}

// ---- the superstep's range kernel ------------------------------------------------------------
struct FlagArgs {
    const int32_t* fidx;
    int64_t edges;
    int64_t rphase;
    int32_t num_ranges;
    int32_t order;               // 1: ranges alternately from the two ends of the plan
    const int2* rinfo;
    double* sumc;
    double* carry;
    double* head;
    int32_t* ctr;
    const double* contrib;       // the outbox replica (global ids)
    int gather_policy;
    uint32_t ghot, gtotal;
    int32_t l1hot;
    // k_pr_flag<true>: Fig. 8's update in the epilogue (broadcasting supersteps of a fixed-k run)
    const int2* rowdeg;
    double* contrib_next;        // the next outbox replica (global ids)
    PeerSlots<double> peers;     // fused exchange: the other replicas
    int64_t vbase;
    double ratio;
};

// Fig. 8's update of the row with ordinal o and combined sum `sum` (broadcasting superstep): the
// same IEEE operations as PageRankPull::finish_deg, so the result is bit-identical to the split
// path (k_pr_finish).
__device__ __forceinline__ void flag_update(const FlagArgs& A, int32_t o, double sum) {
    const int2 rd = A.rowdeg[o];
    const double r = __dadd_rn(A.ratio, __dmul_rn(0.85, sum));
    const double x = rd.y > 0 ? __ddiv_rn(r, (double)rd.y) : 0.0;
    A.contrib_next[A.vbase + rd.x] = x;
    A.peers.store(A.vbase + rd.x, x);
}

// Per row with in-edges: its (row, out-degree) at its ordinal.
__global__ void k_flag_rowdeg(const int32_t* __restrict__ in_off, const int32_t* __restrict__ out_off,
                              int64_t rows, const uint32_t* __restrict__ nzbits,
                              const int32_t* __restrict__ nzpre, int2* __restrict__ rowdeg) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    if (in_off[r + 1] == in_off[r]) return;
    const uint32_t w = nzbits[r >> 5];
    const int32_t o = nzpre[r >> 5] + __popc(w & ((1u << (r & 31)) - 1u));
    rowdeg[o] = make_int2((int32_t)r, out_off[r + 1] - out_off[r]);
}

#ifndef IPREGEL_PRF_MINBLOCKS
#define IPREGEL_PRF_MINBLOCKS 3
#endif

// Chunk at local edge e0: the indices (bit 31 = row end; kFlagNoEdge / kFlagPhantom outside).
__device__ __forceinline__ void flag_load(const FlagArgs& A, int64_t e0, int lane, uint64_t pol,
                                          int32_t (&r)[4]) {
    if (e0 >= 0 && e0 + kChunk <= A.edges) {   // warp-uniform: interior chunk
#pragma unroll
        for (int k = 0; k < 4; ++k) r[k] = ld_stream(A.fidx + e0 + 32 * k + lane, pol);
        return;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int64_t e = e0 + 32 * k + lane;
        r[k] = (e >= 0 && e < A.edges) ? ld_stream(A.fidx + e, pol)
                                       : (e == -1 ? kFlagPhantom : kFlagNoEdge);
    }
}

// Gathers of a loaded chunk and its end words (one per 32 positions).
__device__ __forceinline__ void flag_gather(const FlagArgs& A, const int32_t (&r)[4],
                                            uint64_t pol, double (&g)[4], uint32_t (&f)[4]) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int32_t u = r[k] & kFlagNoEdge;
        g[k] = u != kFlagNoEdge ? (A.l1hot < 0 ? ld_gather(A.contrib + u, pol)
                                               : ld_gather_l1(A.contrib + u, pol, u < A.l1hot))
                                : 0.0;
        f[k] = __ballot_sync(kFull, r[k] < 0);
    }
}

template <bool kFuse>
__global__ void __launch_bounds__(kPullThreads, IPREGEL_PRF_MINBLOCKS) k_pr_flag(FlagArgs A) {
    using Op = SumF64;
    __shared__ __align__(16) double s_w[kWarpsPerCta][kChunk];
    const int lane = threadIdx.x & 31;
    double* sw = s_w[threadIdx.x >> 5];
    const uint64_t pol_s = policy_evict_first();
    const uint64_t pol_g = policy_for(A.gather_policy, A.contrib, A.ghot, A.gtotal);
    int32_t t = lane == 0 ? atomicAdd(A.ctr, 1) : 0;
    t = __shfl_sync(kFull, t, 0);
    while (t < A.num_ranges) {
        const int32_t nxt = lane == 0 ? atomicAdd(A.ctr, 1) : 0;
        const int32_t q = A.order == 1 ? ((t & 1) ? A.num_ranges - 1 - (t >> 1) : (t >> 1)) : t;
        const int64_t eb = (int64_t)q * kFlagRange - A.rphase;   // range start (local)
        const int64_t ee = eb + kFlagRange < A.edges ? eb + kFlagRange : A.edges;
        const int2 info = A.rinfo[q];
        int32_t ord = info.x;                           // ordinal of the open row
        const int32_t hord = info.y ? info.x : INT_MIN;   // its piece here goes to head[q]
        auto emit = [&](int32_t o, double v) {
            if (o == hord) A.head[q] = v;
            else if (o >= 0) {
                if constexpr (kFuse) flag_update(A, o, v);
                else A.sumc[o] = v;
            }
        };
        int32_t I[4];
        double G[4];
        uint32_t F[4];
        flag_load(A, eb, lane, pol_s, I);
        flag_gather(A, I, pol_g, G, F);
        flag_load(A, eb + kChunk, lane, pol_s, I);
        double la = 0.0, carry = 0.0;
        bool la_used = false;
        for (int64_t e0 = eb; e0 < ee; e0 += kChunk) {
            double v[4];
            uint32_t f[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                v[k] = G[k];
                f[k] = F[k];
            }
            if (e0 + kChunk < ee) {
                flag_gather(A, I, pol_g, G, F);
                if (e0 + 2 * kChunk < ee) flag_load(A, e0 + 2 * kChunk, lane, pol_s, I);
            }
            const int32_t o0 = ord;
            const int n_end = __popc(f[0]) + __popc(f[1]) + __popc(f[2]) + __popc(f[3]);
            ord += n_end;
            if (n_end == 0) {   // inside one row: lane-private partials
                la = Op::combine(la, Op::combine(Op::combine(v[0], v[1]), Op::combine(v[2], v[3])));
                la_used = true;
                continue;
            }
            // first end position q1 and last end position ql (warp-uniform)
            const int k1 = f[0] ? 0 : (f[1] ? 1 : (f[2] ? 2 : 3));
            const int kl = f[3] ? 3 : (f[2] ? 2 : (f[1] ? 1 : 0));
            const int p1 = 32 * k1 + __ffs(f[k1]);            // positions < p1: entering row
            const int pl = 32 * kl + 32 - __clz(f[kl]);       // positions >= pl: leaving row
            double t1 = la, t2 = 0.0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int pos = 32 * k + lane;
                if (pos < p1) t1 = Op::combine(t1, v[k]);
                else if (pos >= pl) t2 = Op::combine(t2, v[k]);
            }
            double f1, f2;
            warp_fold2<Op>(t1, t2, f1, f2);
            if (lane == 0) emit(o0, Op::combine(carry, f1));
            carry = f2;
            la = 0.0;
            la_used = false;
            if (n_end == 1) continue;
            // rows wholly inside the chunk: lane l takes positions 4l .. 4l + 3
#pragma unroll
            for (int k = 0; k < 4; ++k) sw[32 * k + lane] = v[k];
            __syncwarp();
            const double2 w01 = *reinterpret_cast<const double2*>(sw + 4 * lane);
            const double2 w23 = *reinterpret_cast<const double2*>(sw + 4 * lane + 2);
            __syncwarp();
            const double w[4] = {w01.x, w01.y, w23.x, w23.y};
            const uint32_t word = lane < 8 ? f[0] : (lane < 16 ? f[1] : (lane < 24 ? f[2] : f[3]));
            const uint32_t nib = (word >> (4 * (lane & 7))) & 0xFu;
            // ends before this lane's positions: the rank of its first end
            const int below = __popc(word & ((1u << (4 * (lane & 7))) - 1u)) +
                              (lane >= 8 ? __popc(f[0]) : 0) + (lane >= 16 ? __popc(f[1]) : 0) +
                              (lane >= 24 ? __popc(f[2]) : 0);
            double acc = 0.0, A0 = 0.0;
            int r = below;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                acc = Op::combine(acc, w[j]);
                if ((nib >> j) & 1u) {
                    if (r == below) A0 = acc;                // this lane's first end
                    else emit(o0 + r, acc);                  // a row inside this lane
                    ++r;
                    acc = 0.0;
                }
            }
            // segmented inclusive scan of the lanes' outgoing partials: a lane with an end
            // opens a segment (the row after its last end)
            const uint32_t ends = __ballot_sync(kFull, nib != 0u);
            const uint32_t le = ends & (0xFFFFFFFFu >> (31 - lane));
            const int start = le ? 31 - __clz(le) : -1;
            double x = acc;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const double y = __shfl_up_sync(kFull, x, d);
                if (lane >= d && lane - d >= start) x = Op::combine(y, x);
            }
            double in = __shfl_up_sync(kFull, x, 1);
            if (lane == 0) in = 0.0;
            // the first end of each lane closes the row that came in from lower lanes -- except
            // the chunk's first end (the entering row, closed by the fold above)
            if (nib != 0u && below > 0) emit(o0 + below, Op::combine(in, A0));
        }
        const double out = Op::combine(carry, la_used ? warp_fold<Op>(la) : 0.0);
        if (lane == 0) A.carry[q] = out;
        t = __shfl_sync(kFull, nxt, 0);
    }
}

// Rows cut by range boundaries.  Range b is the last range of a row that started before it when
// rinfo[b] says "continuing" and range b + 1 does not continue the same row; the row's pieces are
// carry[a - 1], carry[a], ..., carry[b - 1], head[b] for the boundaries a..b that carry it.  The
// groups (ordinal, a, b) are found once, on the device, when the plan is built (k_flag_groups:
// short spans and long ones in two lists, in any order) and joined every superstep by
// k_flag_fixup in k_pull_fixup's fixed order -- spans <= kFixupShortSpan by one thread (a left
// fold), longer ones by one warp (lane-strided partials, the xor tree) -- which depends on the
// ranges' global positions only.
__global__ void k_flag_groups(const int2* __restrict__ rinfo, int32_t num_ranges,
                              int4* __restrict__ gshort, int4* __restrict__ glong,
                              int32_t* __restrict__ counts) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= num_ranges) return;
    const int2 info = rinfo[b];
    if (!info.y) return;
    if (b + 1 < num_ranges) {
        const int2 nx = rinfo[b + 1];
        if (nx.y && nx.x == info.x) return;   // the row runs on past range b
    }
    int64_t a = b;
    while (a - 1 >= 1) {
        const int2 r = rinfo[a - 1];
        if (!(r.y && r.x == info.x)) break;
        --a;
    }
    const int4 G = make_int4(info.x, (int32_t)a, (int32_t)b, 0);
    if (b - a + 1 <= kFixupShortSpan) gshort[atomicAdd(&counts[0], 1)] = G;
    else glong[atomicAdd(&counts[1], 1)] = G;
}

// Fixed grid, grid-stride over the device-side counts: first every thread takes short groups,
// then every warp takes long ones.
template <bool kFuse>
__global__ void k_flag_fixup(const int4* __restrict__ gshort, const int4* __restrict__ glong,
                             const int32_t* __restrict__ counts, const double* __restrict__ carry,
                             const double* __restrict__ head, double* __restrict__ sumc,
                             FlagArgs A) {
    using Op = SumF64;
    const int lane = threadIdx.x & 31;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
    const int32_t ns = counts[0], nl = counts[1];
    for (int64_t i = tid; i < ns; i += nthreads) {
        const int4 G = gshort[i];
        double acc = carry[G.y - 1];
        for (int32_t t = G.y; t <= G.z - 1; ++t) acc = Op::combine(acc, carry[t]);
        acc = Op::combine(acc, head[G.z]);
        if constexpr (kFuse) flag_update(A, G.x, acc);
        else sumc[G.x] = acc;
    }
    for (int64_t w = tid >> 5; w < nl; w += nthreads >> 5) {
        const int4 G = glong[w];
        double acc = Op::identity();
        for (int32_t t = G.y - 1 + lane; t <= G.z - 1; t += 32) acc = Op::combine(acc, carry[t]);
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const double o = shfl_xor(acc, d);
            acc = (lane & d) ? Op::combine(o, acc) : Op::combine(acc, o);
        }
        if (lane == 0) {
            acc = Op::combine(acc, head[G.z]);
            if constexpr (kFuse) flag_update(A, G.x, acc);
            else sumc[G.x] = acc;
        }
    }
}

}  // namespace ipr
