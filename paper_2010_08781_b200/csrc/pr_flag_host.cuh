// paper_2010_08781_b200/csrc/pr_flag_host.cuh -- host side of the flagged PageRank superstep
// (pr_flag.cuh): the per-partition plan -- built at create for graphs the library relabelled,
// else before a graph's first PageRank pull run -- and the launch.  Part of the single
// translation unit ipregel.cu (after engine.cuh).
#pragma once

namespace {

// Tuning / A-B knob: 0 = PageRank pull supersteps through k_pull_ranges<PageRankSum> (pull.cuh).
int g_pr_flag = getenv("IPREGEL_PR_FLAG") ? atoi(getenv("IPREGEL_PR_FLAG")) : 1;
// Knob IPREGEL_PR_FUSE=1: Fig. 8's update fused into the flagged superstep's epilogue for the
// broadcasting supersteps 3 .. k-1 of a fixed-k run (supersteps 1 and 2 run k_pr_finish, which
// leaves the constant outbox values of the rows without in-edges in both buffers).  Measured
// slower at cfg4 (supersteps 6.72-6.84 vs 6.44-6.58 ms with the separate pass: the (row, degree)
// load and the division sit on the emitting warp's path, 80 registers), so off by default.
int g_pr_fuse = getenv("IPREGEL_PR_FUSE") ? atoi(getenv("IPREGEL_PR_FUSE")) : 0;

// Builds p.plan_flag on the graph's stream (library memory in p.graph_mem, reported by
// ipregel_memory_footprint), stream-ordered with no host synchronisation and no copy-engine
// work: a kernel copy of the CSC indices, one pass over the rows, a scan, one binary search per
// range.
void ensure_flag_plan(ipregel_graph* g, Partition& p) {
    FlagPlan& F = p.plan_flag;
    if (F.ready) return;
    cudaStream_t s = g->stream;
    F.edges = p.csc_edges;
    F.rows = (int32_t)p.rows;
    F.rphase = p.csc_ebase % kFlagRange;
    F.num_ranges = F.edges > 0 ? (int32_t)ceil_div(F.edges + F.rphase, kFlagRange) : 0;
    const int64_t words = ceil_div(std::max<int64_t>(p.rows, 1), 32);
    F.nzbits = p.graph_mem.alloc<uint32_t>(words, s, true);
    F.nzpre = p.graph_mem.alloc<int32_t>(words + 1, s);   // [words]: the total
    F.sumc = p.graph_mem.alloc<double>(p.rows + 1, s, true);
    DeviceBuffers tmp;
    int32_t* cnt = tmp.alloc<int32_t>(words + 1, s, true);
    if (F.edges > 0) {
        F.fidx = p.graph_mem.alloc<int32_t>(F.edges, s);
        // a kernel, not cudaMemcpyAsync: a copy-engine copy would queue behind create's
        // host uploads still in flight (weights), see compute_fence in create.cuh
        kernel_copy(F.fidx, p.csc_idx, (size_t)F.edges * sizeof(int32_t), s);
    }
    if (p.rows > 0) {
        k_flag_rows<<<grid_for(p.rows, 256), 256, 0, s>>>(p.csc_off, p.rows, F.fidx, F.nzbits, cnt);
        LAUNCH_CHECK();
    }
    size_t tb = 0;
    CU(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, F.nzpre, (int)(words + 1), s));
    void* t = tmp.alloc<char>((int64_t)tb, s);
    CU(cub::DeviceScan::ExclusiveSum(t, tb, cnt, F.nzpre, (int)(words + 1), s));
    const int32_t Q = F.num_ranges;
    if (Q > 0) {
        F.rinfo = p.graph_mem.alloc<int2>(Q, s);
        F.carry = p.graph_mem.alloc<double>(Q, s);
        F.head = p.graph_mem.alloc<double>(Q, s);
        F.ctr = p.graph_mem.alloc<int32_t>(1, s, true);
        k_flag_ranges<<<grid_for(Q, 256), 256, 0, s>>>(p.csc_off, F.rows, F.edges, F.rphase, Q,
                                                       F.nzbits, F.nzpre, F.rinfo);
        LAUNCH_CHECK();
        if (g_pr_fuse) {   // only the fused update reads it
            F.rowdeg = p.graph_mem.alloc<int2>(std::max<int64_t>(p.rows, 1), s);
            k_flag_rowdeg<<<grid_for(p.rows, 256), 256, 0, s>>>(p.csc_off, p.csr_off, p.rows,
                                                                 F.nzbits, F.nzpre, F.rowdeg);
            LAUNCH_CHECK();
        }
        F.gshort = p.graph_mem.alloc<int4>(Q, s);
        F.glong = p.graph_mem.alloc<int4>(Q, s);
        F.gcount = p.graph_mem.alloc<int32_t>(2, s, true);
        k_flag_groups<<<grid_for(Q, 256), 256, 0, s>>>(F.rinfo, Q, F.gshort, F.glong, F.gcount);
        LAUNCH_CHECK();
    }
    tmp.release();   // stream-ordered frees
    F.ready = true;
}

// Grid: every SM full once (occupancy API), never more warps than ranges.
template <bool kFuse>
unsigned pr_flag_grid(int32_t num_ranges) {
    static int per_sm = -1;
    if (per_sm < 0) {
        if (g_pull_carveout >= 0)
            CU(cudaFuncSetAttribute(k_pr_flag<kFuse>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                    g_pull_carveout));
        CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pr_flag<kFuse>, kPullThreads, 0));
        per_sm = std::max(per_sm, 1);
    }
    return (unsigned)std::max<int64_t>(
        1, std::min<int64_t>(ceil_div(num_ranges, kWarpsPerCta), (int64_t)device_sms() * per_sm));
}

// One PageRank gather superstep of partition p: the range kernel, then the joins of rows cut by
// range boundaries.  Sums land in p.plan_flag.sumc by ordinal (k_pr_finish<., true> reads them).
// fuse: Fig. 8's update in the epilogue (outbox `contrib_next`, `peers`), else sums by ordinal.
void launch_pr_flag(ipregel_graph* g, Partition& p, const double* contrib_cur, cudaStream_t s,
                    bool fuse = false, double* contrib_next = nullptr,
                    PeerSlots<double> peers = PeerSlots<double>{{}, 0}, double ratio = 0.0) {
    FlagPlan& F = p.plan_flag;
    if (F.num_ranges == 0) return;
    const uint64_t total = std::min<uint64_t>((uint64_t)g->n * sizeof(double), 0xFFFFFFFFull);
    FlagArgs A;
    A.fidx = F.fidx;
    A.edges = F.edges;
    A.rphase = F.rphase;
    A.num_ranges = F.num_ranges;
    A.order = g_range_order == 1 ? 1 : 0;
    A.rinfo = F.rinfo;
    A.sumc = F.sumc;
    A.carry = F.carry;
    A.head = F.head;
    A.ctr = F.ctr;
    A.contrib = contrib_cur;
    A.gather_policy = g->gather_policy;
    A.ghot = (uint32_t)std::min<uint64_t>(g_hot_bytes, total);
    A.gtotal = (uint32_t)total;
    A.l1hot = g_l1_hot != -2 ? g_l1_hot : (g->degree_ordered ? (int32_t)(65536 / sizeof(double)) : -1);
    A.rowdeg = F.rowdeg;
    A.contrib_next = contrib_next;
    A.peers = peers;
    A.vbase = p.vb;
    A.ratio = ratio;
    CU(cudaMemsetAsync(F.ctr, 0, sizeof(int32_t), s));
    if (fuse) k_pr_flag<true><<<pr_flag_grid<true>(F.num_ranges), kPullThreads, 0, s>>>(A);
    else k_pr_flag<false><<<pr_flag_grid<false>(F.num_ranges), kPullThreads, 0, s>>>(A);
    LAUNCH_CHECK();
    if (F.num_ranges > 1) {
        // groups <= num_ranges / 1 (short) or num_ranges / 17 (long): a fixed grid strides them
        const unsigned fg = std::max<unsigned>(
            1, std::min<unsigned>(grid_for(F.num_ranges, 256), sm_grid(4)));
        if (fuse)
            k_flag_fixup<true><<<fg, 256, 0, s>>>(F.gshort, F.glong, F.gcount, F.carry, F.head,
                                                  F.sumc, A);
        else
            k_flag_fixup<false><<<fg, 256, 0, s>>>(F.gshort, F.glong, F.gcount, F.carry, F.head,
                                                   F.sumc, A);
        LAUNCH_CHECK();
    }
}

// Fig. 8's update after the flagged superstep (k_pr_finish<mode, true>): kRows rows per thread
// (knob IPREGEL_PR_FINISH_ROWS_C: 2, 4, 8 or 16; the ordinal lookup puts a second load in each
// row's chain, so more rows per thread keep more of them in flight).
int g_pr_finish_rows_c = getenv("IPREGEL_PR_FINISH_ROWS_C") ? atoi(getenv("IPREGEL_PR_FINISH_ROWS_C")) : 4;
template <int kRows>
void launch_pr_finish_rows(const PageRankPull& op, int64_t rows, PullCounters* cnt, int mode,
                           cudaStream_t s) {
    const unsigned fg = grid_for(ceil_div(rows, kRows), 256);
    if (mode == 0) k_pr_finish<0, true, kRows><<<fg, 256, 0, s>>>(op, rows, cnt);
    else if (mode == 1) k_pr_finish<1, true, kRows><<<fg, 256, 0, s>>>(op, rows, nullptr);
    else k_pr_finish<2, true, kRows><<<fg, 256, 0, s>>>(op, rows, nullptr);
    LAUNCH_CHECK();
}
void launch_pr_finish_compact(const PageRankPull& op, int64_t rows, PullCounters* cnt, int mode,
                              cudaStream_t s) {
    if (g_pr_finish_rows_c == 2) launch_pr_finish_rows<2>(op, rows, cnt, mode, s);
    else if (g_pr_finish_rows_c == 4) launch_pr_finish_rows<4>(op, rows, cnt, mode, s);
    else if (g_pr_finish_rows_c == 16) launch_pr_finish_rows<16>(op, rows, cnt, mode, s);
    else launch_pr_finish_rows<8>(op, rows, cnt, mode, s);
}

}  // namespace
