// paper_2010_08781_b200/csrc/create.cuh -- graph handles: descriptor validation, partition setup
// (host uploads, the derived out-adjacency, validation), tile plans and destruction.
// Host part of the single translation unit ipregel.cu (included once, in order).
#pragma once

namespace {

void validate_desc(const ipregel_graph_desc* d, int64_t* n_out) {
    if (!d) fail(IPREGEL_ERR_INVALID_ARGUMENT, "desc is NULL");
    if (d->num_vertices < 1 || d->num_vertices > 2147483647LL)
        fail(IPREGEL_ERR_INVALID_ARGUMENT, "num_vertices %lld outside [1, 2^31-1]",
             (long long)d->num_vertices);
    if (d->num_edges < 0 || d->num_edges > 2147483647LL)
        fail(IPREGEL_ERR_UNSUPPORTED, "num_edges %lld beyond int32 indexing",
             (long long)d->num_edges);
    if (d->vertex_begin < 0 || d->vertex_end < d->vertex_begin || d->vertex_end > d->num_vertices)
        fail(IPREGEL_ERR_INVALID_ARGUMENT, "owned range [%lld, %lld) invalid",
             (long long)d->vertex_begin, (long long)d->vertex_end);
    if (d->csc_edges < 0 || d->csr_edges < 0 || d->csc_edges > d->num_edges ||
        d->csr_edges > d->num_edges)
        fail(IPREGEL_ERR_INVALID_ARGUMENT, "csc_edges/csr_edges out of range");
    const bool derive_csr = !d->csr_offsets && !d->csr_indices && !d->csr_weights;
    if (!d->csc_offsets || (!derive_csr && !d->csr_offsets) || (d->csc_edges > 0 && !d->csc_indices) ||
        (!derive_csr && d->csr_edges > 0 && !d->csr_indices))
        fail(IPREGEL_ERR_INVALID_ARGUMENT, "required CSC/CSR array is NULL");
    if (!derive_csr && (d->csc_weights == nullptr) != (d->csr_weights == nullptr))
        fail(IPREGEL_ERR_INVALID_ARGUMENT, "csc_weights and csr_weights must both be set or NULL");
    if (derive_csr && (d->vertex_begin != 0 || d->vertex_end != d->num_vertices ||
                       d->csc_edges != d->num_edges))
        fail(IPREGEL_ERR_UNSUPPORTED,
             "deriving the CSR from the CSC needs the whole graph in one partition");
    if (d->memory != IPREGEL_MEMORY_DEVICE && d->memory != IPREGEL_MEMORY_HOST)
        fail(IPREGEL_ERR_INVALID_ARGUMENT, "unknown memory kind %d", d->memory);
    if (d->reserved != 0) fail(IPREGEL_ERR_INVALID_ARGUMENT, "reserved must be 0");
    if (d->degree_ordered != 0 && d->degree_ordered != 1)
        fail(IPREGEL_ERR_INVALID_ARGUMENT, "degree_ordered must be 0 or 1");
    if ((d->vertex_end - d->vertex_begin) + std::max(d->csc_edges, d->csr_edges) > 2147483647LL)
        fail(IPREGEL_ERR_UNSUPPORTED, "rows + edges of a partition beyond int32 merge coordinates");
    *n_out = d->num_vertices;
}

__global__ void k_noop() {}

// Measured on B200 (tools/lab/stream_wait_lab3.cu): once a stream's latest operation is a host ->
// device copy, a cross-stream wait issued on it next is released only after the OTHER stream's
// queued copies finish too (it sits behind them on the copy engine) -- here that would hold the
// derived CSR's sort and the weight windows until the whole upload ends.  An empty kernel first
// puts the wait back on the compute queue.
void compute_fence(cudaStream_t s) {
    k_noop<<<1, 32, 0, s>>>();
    LAUNCH_CHECK();
}

// windows of the CSC weights' upload when the CSR is derived (the last window's permutation is
// all that remains after the upload)
constexpr int kWeightWindows = 16;   // 8: +1.3 ms, 32: +18 ms (create at cfg4)

void init_partition(ipregel_graph* g, Partition& p, const ipregel_graph_desc& d) {
    cudaStream_t s = g->stream;
    p.vb = d.vertex_begin;
    p.ve = d.vertex_end;
    p.rows = p.ve - p.vb;
    p.csc_edges = d.csc_edges;
    p.csr_edges = d.csr_edges;
    const bool derive = !d.csr_offsets && !d.csr_indices;
    p.host_cnt = static_cast<unsigned long long*>(pinned_acquire(16 * sizeof(unsigned long long)));
    if (d.memory == IPREGEL_MEMORY_HOST) {
        // uploads run on a copy stream in the order the device work needs them: the adjacency
        // structure first (validation, the derived CSR's sort and the tile plans start as soon
        // as it lands), then the weights -- in windows when the CSR is derived, each window's
        // share of the weight permutation running while the next one uploads (finish_uploads)
        if (!g->copy_stream) CU(cudaStreamCreateWithFlags(&g->copy_stream, cudaStreamNonBlocking));
        cudaStream_t cs = g->copy_stream;
        auto alloc = [&](const void* src, size_t bytes) -> void* {
            return src ? (void*)p.graph_mem.alloc<uint8_t>((int64_t)bytes, s) : nullptr;
        };
        void* off_d = alloc(d.csc_offsets, (p.rows + 1) * 4);
        void* idx_d = alloc(d.csc_indices, d.csc_edges * 4);
        void* w_d = alloc(d.csc_weights, d.csc_edges * 4);
        void* roff_d = alloc(d.csr_offsets, (p.rows + 1) * 4);
        void* ridx_d = alloc(d.csr_indices, d.csr_edges * 4);
        void* rw_d = alloc(d.csr_weights, d.csr_edges * 4);
        for (cudaEvent_t* e : {&p.up_idx, &p.up_w, &p.up_all})
            if (!*e) CU(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        CU(cudaEventRecord(p.up_all, s));              // the allocations, in stream order
        CU(cudaStreamWaitEvent(cs, p.up_all, 0));
        auto up = [&](void* dst, const void* src, size_t bytes) {
            if (src) CU(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, cs));
        };
        g_ctrace.mark("uploads begin", cs);
        up(off_d, d.csc_offsets, (p.rows + 1) * 4);
        up(idx_d, d.csc_indices, d.csc_edges * 4);
        up(roff_d, d.csr_offsets, (p.rows + 1) * 4);
        up(ridx_d, d.csr_indices, d.csr_edges * 4);
        CU(cudaEventRecord(p.up_idx, cs));
        g_ctrace.mark("uploaded structure", cs);
        int windows = (derive && w_d && d.csc_edges >= (int64_t(1) << 24)) ? kWeightWindows : 1;
        if (const char* e = getenv("IPREGEL_WEIGHT_WINDOWS"))   // test hook
            if (derive && w_d) windows = std::max(1, std::min(atoi(e), 64));
        p.wc_bounds.assign(1, 0);
        for (int c = 0; c < windows; ++c) {
            const int64_t lo = d.csc_edges * c / windows, hi = d.csc_edges * (c + 1) / windows;
            if (w_d) up((uint32_t*)w_d + lo, (const uint32_t*)d.csc_weights + lo, (hi - lo) * 4);
            cudaEvent_t e;
            CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            CU(cudaEventRecord(e, cs));
            p.up_wc.push_back(e);
            p.wc_bounds.push_back(hi);
        }
        CU(cudaEventRecord(p.up_w, cs));
        g_ctrace.mark("uploaded csc w", cs);
        up(rw_d, d.csr_weights, d.csr_edges * 4);
        CU(cudaEventRecord(p.up_all, cs));
        g_ctrace.mark("uploaded all", cs);
        // validation and everything up to the weights need the structure only
        compute_fence(s);   // s uploaded the vertex ids
        CU(cudaStreamWaitEvent(s, p.up_idx, 0));
        g_ctrace.mark("structure landed", s);
        p.csc_off = (const int32_t*)off_d;
        p.csc_idx = (const int32_t*)idx_d;
        p.csc_w = (const uint32_t*)w_d;
        p.csr_off = (const int32_t*)roff_d;
        p.csr_idx = (const int32_t*)ridx_d;
        p.csr_w = (const uint32_t*)rw_d;
    } else {
        p.csc_off = d.csc_offsets; p.csc_idx = d.csc_indices; p.csc_w = d.csc_weights;
        p.csr_off = d.csr_offsets; p.csr_idx = d.csr_indices; p.csr_w = d.csr_weights;
    }

    if (d.validate) {
        unsigned* flags = p.graph_mem.alloc<unsigned>(1, s, true);
        k_validate_offsets<<<grid_for(p.rows + 1, 256), 256, 0, s>>>(p.csc_off, p.rows, p.csc_edges, flags);
        if (p.csr_off)
            k_validate_offsets<<<grid_for(p.rows + 1, 256), 256, 0, s>>>(p.csr_off, p.rows, p.csr_edges, flags);
        LAUNCH_CHECK();
        unsigned* hf = reinterpret_cast<unsigned*>(p.host_cnt);
        kernel_copy(hf, flags, 4, s);   // not a cudaMemcpy: see compute_fence
        CU(cudaStreamSynchronize(s));
        unsigned h = *hf;
        if (h == 0) {
            if (p.csc_edges)
                k_validate_indices<<<std::min<unsigned>(grid_for(p.csc_edges, 256), 4096), 256, 0, s>>>(
                    p.csc_idx, p.csc_edges, g->n, flags);
            if (p.csr_edges && p.csr_idx)
                k_validate_indices<<<std::min<unsigned>(grid_for(p.csr_edges, 256), 4096), 256, 0, s>>>(
                    p.csr_idx, p.csr_edges, g->n, flags);
            LAUNCH_CHECK();
            kernel_copy(hf, flags, 4, s);
            CU(cudaStreamSynchronize(s));
            h = *hf;
        }
        if (h)
            fail(IPREGEL_ERR_INVALID_GRAPH, "graph validation failed (flags 0x%x: %s%s%s)", h,
                 (h & 1) ? "offsets[0]/offsets[rows] " : "", (h & 2) ? "non-monotone offsets " : "",
                 (h & 4) ? "index out of range" : "");
    }
    g_ctrace.mark("validated", s);
    if (!d.csr_offsets && !d.csr_indices) {
        // out-adjacency (and its weights) derived from the CSC on the device: the transpose of
        // the whole graph's in-edges (single partition, checked by validate_desc;
        // after the validation: the transpose indexes by the CSC sources)
        int32_t *o, *ix;
        uint32_t* wx = nullptr;
        transpose_rows(p, g->n, p.csc_off, p.csc_idx, p.csc_w, p.csc_edges, p.csc_w != nullptr, s,
                       &o, &ix, &wx, d.memory == IPREGEL_MEMORY_HOST);
        p.csr_off = o;
        p.csr_idx = ix;
        p.csr_w = wx;
        p.csr_edges = p.csc_edges;
        if (p.pend.perm) {
            // permute each weight window as it lands, on a side stream (the run stream goes
            // on with the tile plans); transpose_rows returned with perm complete
            if (!g->aux_stream) CU(cudaStreamCreateWithFlags(&g->aux_stream, cudaStreamNonBlocking));
            for (size_t c = 0; c + 1 < p.wc_bounds.size(); ++c) {
                CU(cudaStreamWaitEvent(g->aux_stream, p.up_wc[c], 0));
                k_permute_window<<<148 * 8, 256, 0, g->aux_stream>>>(
                    p.pend.perm, p.pend.edges, p.wc_bounds[c], p.wc_bounds[c + 1], p.pend.w,
                    p.pend.wx);
                LAUNCH_CHECK();
            }
            CU(cudaEventCreateWithFlags(&p.perm_done, cudaEventDisableTiming));
            CU(cudaEventRecord(p.perm_done, g->aux_stream));
            g_ctrace.mark("weights permuted", g->aux_stream);
        }
    }
    p.pull_cnt = p.graph_mem.alloc<PullCounters>(1, s, true);
    p.dscratch = p.graph_mem.alloc<unsigned long long>(64, s, true);
    p.front_cnt = p.graph_mem.alloc<FrontierCounters>(1, s, true);
    // PageRank broadcasters (out-degree > 0)
    unsigned long long* cnt = p.graph_mem.alloc<unsigned long long>(1, s, true);
    if (p.rows) {
        k_count_nondangling<<<grid_for(p.rows, 256), 256, 0, s>>>(p.csr_off, p.rows, cnt);
        LAUNCH_CHECK();
    }
    kernel_copy(p.host_cnt, cnt, 8, s);   // not a cudaMemcpy: see compute_fence
    CU(cudaStreamSynchronize(s));
    p.nondangling = (int64_t)p.host_cnt[0];
    g_ctrace.mark("partition ready", s);
}

// The tail of a create from host memory, after the tile plans: the derived CSR's weights
// permuted (aux stream, window by window as the windows landed), then every upload resident
// before create returns (the caller may free its host arrays afterwards).
void finish_uploads(ipregel_graph* g, Partition& p) {
    cudaStream_t s = g->stream;
    if (p.pend.perm) {
        CU(cudaStreamWaitEvent(s, p.perm_done, 0));
        p.pend.tmp.release();   // stream-ordered, after the permutation
        p.pend.perm = nullptr;
    }
    if (p.up_all) CU(cudaStreamWaitEvent(s, p.up_all, 0));
}

void build_plans(ipregel_graph* g) {
    for (auto& p : g->parts) {
        build_plan(p.plan_csc, p.csc_off, p.csc_idx, p.csc_w, p.rows, p.csc_edges, p.vb,
                   p.csc_ebase, p.graph_mem, g->stream, g->pinned);
        build_plan(p.plan_csr, p.csr_off, p.csr_idx, nullptr, p.rows, p.csr_edges, p.vb,
                   p.csr_ebase, p.graph_mem, g->stream, g->pinned);
    }
    CU(cudaStreamSynchronize(g->stream));
}

void destroy_graph(ipregel_graph* g) {
    if (!g) return;
    auto t0 = std::chrono::steady_clock::now();
    auto tick = [&](const char* what) {   // IPREGEL_TRACE_CREATE: host time of each phase
        if (!g_ctrace.on) return;
        const auto t = std::chrono::steady_clock::now();
        fprintf(stderr, "[ipregel destroy] %-22s %8.2f ms\n", what,
                std::chrono::duration<double, std::milli>(t - t0).count());
        t0 = t;
    };
    cudaStreamSynchronize(g->stream);
    if (g->copy_stream) cudaStreamSynchronize(g->copy_stream);   // a failed create's uploads
    if (g->aux_stream) cudaStreamSynchronize(g->aux_stream);
    tick("sync");
    for (auto& p : g->parts) {
        for (auto& S : p.st) {
            for (void* q : S.ipc_opened) cudaIpcCloseMemHandle(q);
            S.ipc_opened.clear();
            S.mem.release();
        }
        p.graph_mem.release();
        for (cudaEvent_t e : {p.up_idx, p.up_w, p.up_all})
            if (e) cudaEventDestroy(e);
        for (cudaEvent_t e : p.up_wc) cudaEventDestroy(e);
        if (p.perm_done) cudaEventDestroy(p.perm_done);
        p.perm_done = nullptr;
        p.up_wc.clear();
        p.pend.tmp.release();
        pinned_release(p.host_cnt);
        p.host_cnt = nullptr;
    }
    tick("partition memory");
    if (g->pr_graph.exec) cudaGraphExecDestroy(g->pr_graph.exec);
    if (g->capture_stream) cudaStreamDestroy(g->capture_stream);
    if (g->copy_stream) cudaStreamDestroy(g->copy_stream);
    if (g->aux_stream) cudaStreamDestroy(g->aux_stream);
    for (auto e : g->events) cudaEventDestroy(e);
    tick("graph exec, streams");
    g->graph_mem.release();
    g->pinned.release();
    cudaStreamSynchronize(g->stream);
    tick("frees synchronised");
    delete g;
}

}  // namespace
