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

void init_partition(ipregel_graph* g, Partition& p, const ipregel_graph_desc& d) {
    cudaStream_t s = g->stream;
    p.vb = d.vertex_begin;
    p.ve = d.vertex_end;
    p.rows = p.ve - p.vb;
    p.csc_edges = d.csc_edges;
    p.csr_edges = d.csr_edges;
    const bool derive = !d.csr_offsets && !d.csr_indices;
    if (d.memory == IPREGEL_MEMORY_HOST) {
        // uploads run on a copy stream in the order the device work needs them: the CSC
        // offsets and indices first (the derived CSR's sort starts as soon as they land), then
        // the weights (needed only by the sort's last pass) and the rest
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
        up(off_d, d.csc_offsets, (p.rows + 1) * 4);
        up(idx_d, d.csc_indices, d.csc_edges * 4);
        CU(cudaEventRecord(p.up_idx, cs));
        up(w_d, d.csc_weights, d.csc_edges * 4);
        CU(cudaEventRecord(p.up_w, cs));
        up(roff_d, d.csr_offsets, (p.rows + 1) * 4);
        up(ridx_d, d.csr_indices, d.csr_edges * 4);
        up(rw_d, d.csr_weights, d.csr_edges * 4);
        CU(cudaEventRecord(p.up_all, cs));
        // validation reads every array; otherwise only a derived CSR starts early
        CU(cudaStreamWaitEvent(s, (d.validate || !derive) ? p.up_all : p.up_idx, 0));
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
        unsigned h = 0;
        CU(cudaMemcpyAsync(&h, flags, 4, cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
        if (h == 0) {
            if (p.csc_edges)
                k_validate_indices<<<std::min<unsigned>(grid_for(p.csc_edges, 256), 4096), 256, 0, s>>>(
                    p.csc_idx, p.csc_edges, g->n, flags);
            if (p.csr_edges && p.csr_idx)
                k_validate_indices<<<std::min<unsigned>(grid_for(p.csr_edges, 256), 4096), 256, 0, s>>>(
                    p.csr_idx, p.csr_edges, g->n, flags);
            LAUNCH_CHECK();
            CU(cudaMemcpyAsync(&h, flags, 4, cudaMemcpyDeviceToHost, s));
            CU(cudaStreamSynchronize(s));
        }
        if (h)
            fail(IPREGEL_ERR_INVALID_GRAPH, "graph validation failed (flags 0x%x: %s%s%s)", h,
                 (h & 1) ? "offsets[0]/offsets[rows] " : "", (h & 2) ? "non-monotone offsets " : "",
                 (h & 4) ? "index out of range" : "");
    }
    if (!d.csr_offsets && !d.csr_indices) {
        // out-adjacency (and its weights) derived from the CSC on the device: the transpose of
        // the whole graph's in-edges (single partition, checked by validate_desc;
        // after the validation: the transpose indexes by the CSC sources)
        int32_t *o, *ix;
        uint32_t* wx = nullptr;
        transpose_rows(p, g->n, p.csc_off, p.csc_idx, p.csc_w, p.csc_edges, p.csc_w != nullptr, s,
                       &o, &ix, &wx, d.memory == IPREGEL_MEMORY_HOST ? p.up_w : nullptr);
        p.csr_off = o;
        p.csr_idx = ix;
        p.csr_w = wx;
        p.csr_edges = p.csc_edges;
    }
    if (d.memory == IPREGEL_MEMORY_HOST)
        CU(cudaStreamWaitEvent(s, p.up_all, 0));   // every upload resident before any run
    p.pull_cnt = p.graph_mem.alloc<PullCounters>(1, s, true);
    p.dscratch = p.graph_mem.alloc<unsigned long long>(64, s, true);
    p.front_cnt = p.graph_mem.alloc<FrontierCounters>(1, s, true);
    CU(cudaMallocHost(&p.host_cnt, 16 * sizeof(unsigned long long)));
    // PageRank broadcasters (out-degree > 0)
    unsigned long long* cnt = p.graph_mem.alloc<unsigned long long>(1, s, true);
    if (p.rows) {
        k_count_nondangling<<<grid_for(p.rows, 256), 256, 0, s>>>(p.csr_off, p.rows, cnt);
        LAUNCH_CHECK();
    }
    unsigned long long h = 0;
    CU(cudaMemcpyAsync(&h, cnt, 8, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    p.nondangling = (int64_t)h;
}

void build_plans(ipregel_graph* g) {
    for (auto& p : g->parts) {
        build_plan(p.plan_csc, p.csc_off, p.csc_idx, p.csc_w, p.rows, p.csc_edges, p.vb,
                   p.csc_ebase, p.graph_mem, g->stream);
        build_plan(p.plan_csr, p.csr_off, p.csr_idx, nullptr, p.rows, p.csr_edges, p.vb,
                   p.csr_ebase, p.graph_mem, g->stream);
    }
    CU(cudaStreamSynchronize(g->stream));
}

void destroy_graph(ipregel_graph* g) {
    if (!g) return;
    cudaStreamSynchronize(g->stream);
    for (auto& p : g->parts) {
        for (auto& S : p.st) {
            for (void* q : S.ipc_opened) cudaIpcCloseMemHandle(q);
            S.ipc_opened.clear();
            S.mem.release();
        }
        p.graph_mem.release();
        for (cudaEvent_t e : {p.up_idx, p.up_w, p.up_all})
            if (e) cudaEventDestroy(e);
        if (p.host_cnt) cudaFreeHost(p.host_cnt);
        p.host_cnt = nullptr;
    }
    if (g->pr_graph.exec) cudaGraphExecDestroy(g->pr_graph.exec);
    if (g->capture_stream) cudaStreamDestroy(g->capture_stream);
    if (g->copy_stream) cudaStreamDestroy(g->copy_stream);
    for (auto e : g->events) cudaEventDestroy(e);
    g->graph_mem.release();
    cudaStreamSynchronize(g->stream);
    delete g;
}

}  // namespace
