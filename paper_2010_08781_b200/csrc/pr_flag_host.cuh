// paper_2010_08781_b200/csrc/pr_flag_host.cuh -- host side of the flagged PageRank superstep
// (pr_flag.cuh): the per-partition plan, built once before a graph's first PageRank pull run, and
// the launch.  Part of the single translation unit ipregel.cu (after engine.cuh).
#pragma once

namespace {

// Tuning / A-B knob: 0 = PageRank pull supersteps through k_pull_ranges<PageRankSum> (pull.cuh).
int g_pr_flag = getenv("IPREGEL_PR_FLAG") ? atoi(getenv("IPREGEL_PR_FLAG")) : 1;

// Builds p.plan_flag on the graph's stream (library memory in p.graph_mem, reported by
// ipregel_memory_footprint).  Device work: a copy of the CSC indices, one pass over the rows, a
// scan, one binary search per range; the host groups the rows cut by range boundaries.
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
    DeviceBuffers tmp;
    int32_t* cnt = tmp.alloc<int32_t>(words + 1, s, true);
    if (F.edges > 0) {
        F.fidx = p.graph_mem.alloc<int32_t>(F.edges, s);
        CU(cudaMemcpyAsync(F.fidx, p.csc_idx, (size_t)F.edges * sizeof(int32_t),
                           cudaMemcpyDeviceToDevice, s));
    }
    if (p.rows > 0) {
        k_flag_rows<<<grid_for(p.rows, 256), 256, 0, s>>>(p.csc_off, p.rows, F.fidx, F.nzbits, cnt);
        LAUNCH_CHECK();
    }
    size_t tb = 0;
    CU(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, F.nzpre, (int)(words + 1), s));
    void* t = tmp.alloc<char>((int64_t)tb, s);
    CU(cub::DeviceScan::ExclusiveSum(t, tb, cnt, F.nzpre, (int)(words + 1), s));
    int32_t* h = static_cast<int32_t*>(g->pinned.get(16, 0));
    kernel_copy(h, F.nzpre + words, sizeof(int32_t), s);
    CU(cudaStreamSynchronize(s));
    F.nnz = h[0];
    F.sumc = p.graph_mem.alloc<double>(std::max<int32_t>(F.nnz, 1), s);
    const int32_t Q = F.num_ranges;
    if (Q > 0) {
        F.rinfo = p.graph_mem.alloc<int2>(Q, s);
        F.carry = p.graph_mem.alloc<double>(Q, s);
        F.head = p.graph_mem.alloc<double>(Q, s);
        F.ctr = p.graph_mem.alloc<int32_t>(1, s, true);
        k_flag_ranges<<<grid_for(Q, 256), 256, 0, s>>>(p.csc_off, F.rows, F.edges, F.rphase, Q,
                                                       F.nzbits, F.nzpre, F.rinfo);
        LAUNCH_CHECK();
        // rows cut by range boundaries: consecutive boundaries carrying the same row form one
        // group (ordinal, first boundary a, last boundary b) -- as build_plan
        int2* hr = static_cast<int2*>(g->pinned.get((size_t)Q * sizeof(int2), 0));
        kernel_copy(hr, F.rinfo, (size_t)Q * sizeof(int2), s);
        CU(cudaStreamSynchronize(s));
        std::vector<int4> groups;
        for (int32_t b = 1; b < Q; ++b) {
            if (!hr[b].y) continue;
            if (!groups.empty() && groups.back().x == hr[b].x && groups.back().z == b - 1)
                groups.back().z = b;
            else
                groups.push_back(make_int4(hr[b].x, b, b, 0));
        }
        std::stable_partition(groups.begin(), groups.end(),
                              [](const int4& G) { return G.z - G.y + 1 <= kFixupShortSpan; });
        F.num_groups = (int32_t)groups.size();
        F.num_short = 0;
        for (const int4& G : groups) F.num_short += (G.z - G.y + 1 <= kFixupShortSpan) ? 1 : 0;
        if (F.num_groups) {
            F.groups = p.graph_mem.alloc<int4>(F.num_groups, s);
            int4* hg = static_cast<int4*>(g->pinned.get(groups.size() * sizeof(int4), 1));
            memcpy(hg, groups.data(), groups.size() * sizeof(int4));
            kernel_copy(F.groups, hg, groups.size() * sizeof(int4), s);
            CU(cudaStreamSynchronize(s));
        }
    }
    tmp.release();
    F.ready = true;
}

// Grid: every SM full once (occupancy API), never more warps than ranges.
unsigned pr_flag_grid(int32_t num_ranges) {
    static int per_sm = -1;
    if (per_sm < 0) {
        if (g_pull_carveout >= 0)
            CU(cudaFuncSetAttribute(k_pr_flag, cudaFuncAttributePreferredSharedMemoryCarveout,
                                    g_pull_carveout));
        CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pr_flag, kPullThreads, 0));
        per_sm = std::max(per_sm, 1);
    }
    return (unsigned)std::max<int64_t>(
        1, std::min<int64_t>(ceil_div(num_ranges, kWarpsPerCta), (int64_t)device_sms() * per_sm));
}

// One PageRank gather superstep of partition p: the range kernel, then the joins of rows cut by
// range boundaries.  Sums land in p.plan_flag.sumc by ordinal (k_pr_finish<., true> reads them).
void launch_pr_flag(ipregel_graph* g, Partition& p, const double* contrib_cur, cudaStream_t s) {
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
    CU(cudaMemsetAsync(F.ctr, 0, sizeof(int32_t), s));
    k_pr_flag<<<pr_flag_grid(F.num_ranges), kPullThreads, 0, s>>>(A);
    LAUNCH_CHECK();
    if (F.num_groups) {
        PageRankCompactSum op;
        op.sumc = F.sumc;
        k_pull_fixup<PageRankCompactSum><<<fixup_grid(F.num_groups, F.num_short), 256, 0, s>>>(
            op, F.groups, F.num_groups, F.num_short, F.carry, F.head, nullptr);
        LAUNCH_CHECK();
    }
}

}  // namespace
