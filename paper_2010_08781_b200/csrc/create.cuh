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
    if (d->layout != IPREGEL_LAYOUT_AS_GIVEN && d->layout != IPREGEL_LAYOUT_DEGREE)
        fail(IPREGEL_ERR_INVALID_ARGUMENT, "unknown layout %d", d->layout);
    if (d->layout == IPREGEL_LAYOUT_DEGREE) {
        if (d->vertex_ids || d->degree_ordered)
            fail(IPREGEL_ERR_INVALID_ARGUMENT,
                 "IPREGEL_LAYOUT_DEGREE computes the layout: vertex_ids must be NULL and "
                 "degree_ordered 0");
        if (d->vertex_begin != 0 || d->vertex_end != d->num_vertices ||
            d->csc_edges != d->num_edges)
            fail(IPREGEL_ERR_UNSUPPORTED,
                 "IPREGEL_LAYOUT_DEGREE needs the whole graph in one partition");
    }
    if (d->degree_ordered != 0 && d->degree_ordered != 1)
        fail(IPREGEL_ERR_INVALID_ARGUMENT, "degree_ordered must be 0 or 1");
    // the range kernels walk int32 merge coordinates and look up to 3 chunks (3 * 128 edges)
    // past the current one: keep a margin of 4 chunks below INT32_MAX
    if ((d->vertex_end - d->vertex_begin) + std::max(d->csc_edges, d->csr_edges) >
        2147483647LL - 4 * kChunk)
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
constexpr int kWeightWindows = 16;
// IPREGEL_LAYOUT_DEGREE: bits of the relabel's edge sort key (destination + source class)
constexpr int kRelabelKeyBits = 40;   // 8: +1.3 ms, 32: +18 ms (create at cfg4)

// The library's side stream for create-time work that overlaps the run stream (the derived
// CSR's sort, weight permutations).
void ensure_aux_stream(ipregel_graph* g) {
    if (!g->aux_stream) CU(cudaStreamCreateWithFlags(&g->aux_stream, cudaStreamNonBlocking));
}

// IPREGEL_LAYOUT_DEGREE (include/ipregel.h): internal ids by decreasing out-degree (ties by id),
// the CSC rebuilt with every row's sources ascending, in library-owned memory; g->vertex_ids
// becomes the internal -> original map, so results come back in original ids.  The whole graph
// is one partition (validate_desc).
void relabel_by_degree(ipregel_graph* g, Partition& p, const ipregel_graph_desc& d) {
    cudaStream_t s = g->stream;
    const int64_t n = g->n, E = p.csc_edges;
    DeviceBuffers tmp;
    g_ctrace.mark("relabel begin", s);
    // 1. out-degrees and the degree order (stable: ties keep ascending ids)
    uint32_t* deg = p.pre_deg;   // counted window by window during the upload (init_partition)
    if (!deg) {
        deg = tmp.alloc<uint32_t>(n, s, true);
        if (p.csr_off) {
            k_degree_from_off<<<grid_for(n, 256), 256, 0, s>>>(p.csr_off, n, deg);
        } else if (E) {
            k_degree_hist<<<std::min<unsigned>(grid_for(E, 256), sm_grid(16)), 256, 0, s>>>(
                p.csc_idx, E, deg);
        }
        LAUNCH_CHECK();
    }
    int32_t* ids = tmp.alloc<int32_t>(n, s);
    k_degree_keys<<<grid_for(n, 256), 256, 0, s>>>(deg, n, ids);
    LAUNCH_CHECK();
    uint32_t* deg2 = tmp.alloc<uint32_t>(n, s);
    int32_t* old_of_new = g->graph_mem.alloc<int32_t>(n, s);
    {
        size_t tb = 0;
        CU(cub::DeviceRadixSort::SortPairs(nullptr, tb, deg, deg2, ids, old_of_new, n, 0, 32, s));
        void* t = tmp.alloc<uint8_t>((int64_t)tb, s);
        CU(cub::DeviceRadixSort::SortPairs(t, tb, deg, deg2, ids, old_of_new, n, 0, 32, s));
    }
    int32_t* new_of_old = tmp.alloc<int32_t>(n, s);
    k_invert_perm<<<grid_for(n, 256), 256, 0, s>>>(old_of_new, n, new_of_old);
    LAUNCH_CHECK();
    // the out-adjacency's offsets come from the sorted degrees already: PageRank's pull (which
    // needs only out-degrees) can run before the CSR's indices exist (step 4)
    int32_t* roff = p.graph_mem.alloc<int32_t>(n + 1, s, true);
    k_degree_from_keys<<<grid_for(n, 256), 256, 0, s>>>(deg2, n, roff);
    LAUNCH_CHECK();
    exscan_i32(roff, n + 1, tmp, s);
    g_ctrace.mark("relabel order", s);
    // 2. relabelled edges sorted by (new destination, new source), their CSC positions carried
    //    along.  The key holds the source's id when 2 x bits <= kRelabelKeyBits (every row
    //    fully sorted), else a monotone class of it in kRelabelKeyBits - bits bits
    //    (source_class): at cfg4 a 40-bit sort (5 radix passes) instead of 52 (7) -- rows keep
    //    the hot sources' exact order, and the gather supersteps run as fast as on fully sorted
    //    rows (profiles/r02/README.md)
    int bits = 1;
    while (bits < 31 && (int64_t(1) << bits) < n) ++bits;
    const int cbits = std::min(bits, std::max(kRelabelKeyBits - bits, 6));
    int32_t* off = p.graph_mem.alloc<int32_t>(n + 1, s, true);
    int32_t* idx = p.graph_mem.alloc<int32_t>(std::max<int64_t>(E, 1), s);
    uint32_t* w = p.csc_w ? p.graph_mem.alloc<uint32_t>(std::max<int64_t>(E, 1), s) : nullptr;
    if (E) {
        // every large temporary is allocated once here and reused by the CSR sort of step 4
        unsigned long long* k0 = tmp.alloc<unsigned long long>(E, s);
        unsigned long long* k1 = tmp.alloc<unsigned long long>(E, s);
        int32_t* spare = tmp.alloc<int32_t>(E, s);
        int32_t* row = tmp.alloc<int32_t>(E, s);
        DeviceBuffers tsrc;   // renamed sources in the old CSC order, until the unpack
        int32_t* new_src = tsrc.alloc<int32_t>(E, s);
        k_relabel_pack<<<grid_for(p.rows * 32, 256), 256, 0, s>>>(p.csc_off, p.csc_idx, p.rows,
                                                                  new_of_old, bits, cbits, k0,
                                                                  new_src);
        LAUNCH_CHECK();
        cub::DoubleBuffer<unsigned long long> keys(k0, k1);
        // the sort carries each edge's CSC position, so it needs the structure only (from host
        // memory the weights are still uploading); sources and weights follow by gathers
        uint32_t* pos0 = reinterpret_cast<uint32_t*>(spare);
        uint32_t* pos1 = reinterpret_cast<uint32_t*>(row);
        k_iota_u32<<<std::min<unsigned>(grid_for(E, 256), sm_grid(16)), 256, 0, s>>>(pos0, E);
        LAUNCH_CHECK();
        cub::DoubleBuffer<uint32_t> vals(pos0, pos1);
        size_t tb = 0;
        CU(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, vals, E, 0, bits + cbits, s));
        void* t = tmp.alloc<uint8_t>((int64_t)tb, s);
        CU(cub::DeviceRadixSort::SortPairs(t, tb, keys, vals, E, 0, bits + cbits, s));
        g_ctrace.mark("relabel sorted", s);
        // 3. indices + offsets (run lengths of the sorted destinations, then a scan); each
        //    edge's new row goes to the position buffer the sort did not end in
        const uint32_t* pos = vals.Current();
        int32_t* rows_of = pos == pos0 ? row : spare;
        k_relabel_unpack<<<std::min<unsigned>(grid_for(E, 256), sm_grid(16)), 256, 0, s>>>(
            keys.Current(), pos, E, cbits, new_src, idx, rows_of);
        LAUNCH_CHECK();
        tsrc.release();
        int32_t* st = tmp.alloc<int32_t>(n, s, true);
        k_run_bounds<<<std::min<unsigned>(grid_for(E, 256), sm_grid(16)), 256, 0, s>>>(rows_of, E,
                                                                                  st, off);
        k_run_counts<<<grid_for(n, 256), 256, 0, s>>>(st, n, off);
        LAUNCH_CHECK();
        exscan_i32(off, n + 1, tmp, s);
        g_ctrace.mark("relabel csc", s);
        if (w) {
            // the weights last: from host memory they land while the steps above run
            if (d.memory == IPREGEL_MEMORY_HOST) CU(cudaStreamWaitEvent(s, p.up_w, 0));
            k_gather_u32<<<std::min<unsigned>(grid_for(E, 256), sm_grid(16)), 256, 0, s>>>(
                pos, E, p.csc_w, w);
            LAUNCH_CHECK();
            g_ctrace.mark("relabel weights", s);
        }
        // 4. the out-adjacency's indices: the same edges by (new source), a stable sort of the
        //    CSC order (each CSR row lists its destinations ascending), in the buffers of step 2,
        //    on the aux stream -- launched by launch_relabel_csr once the tile plans are built
        //    (their small kernels would otherwise queue behind the sort's), and create returns
        //    without waiting; whatever reads the CSR's indices first waits for p.csr_done
        //    (wait_csr).  Its offsets are roff already.
        RelabelCsr& R = p.relabel_csr;
        R.ridx = p.graph_mem.alloc<int32_t>(E, s);
        R.rw = w ? p.graph_mem.alloc<uint32_t>(E, s) : nullptr;
        {
            cub::DoubleBuffer<int32_t> tk(row, spare);
            cub::DoubleBuffer<unsigned long long> tv(k0, k1);
            CU(cub::DeviceRadixSort::SortPairs(nullptr, R.tb, tk, tv, E, 0, bits, s));
        }
        R.t = tmp.alloc<uint8_t>((int64_t)R.tb, s);
        R.n = n;
        R.E = E;
        R.bits = bits;
        R.off = off;
        R.idx = idx;
        R.w = w;
        R.k0 = k0;
        R.k1 = k1;
        R.row = row;
        R.spare = spare;
        R.tmp = tmp;   // the temporaries live on until the CSR sort is done
        tmp.blocks.clear();
        R.armed = true;
        p.csr_pending = true;
        p.csr_idx = R.ridx;
        p.csr_w = R.rw;
    } else {
        p.csr_idx = p.graph_mem.alloc<int32_t>(1, s);
        p.csr_w = w ? p.graph_mem.alloc<uint32_t>(1, s) : nullptr;
    }
    p.csr_off = roff;
    CU(cudaStreamSynchronize(s));
    tmp.release();
    p.pre_deg_mem.release();
    p.pre_deg = nullptr;
    p.csc_off = off;
    p.csc_idx = idx;
    p.csc_w = w;
    p.csr_edges = E;
    g->vertex_ids = old_of_new;
    g->degree_ordered = true;
    g->gather_policy = g_gather_policy >= 0 ? g_gather_policy : 3;
    g_ctrace.mark("relabel done", s);
}

// Step 4 of relabel_by_degree on the aux stream (after the tile plans): the CSR's indices and
// weights by a stable sort of the new CSC by source; the temporaries are freed on the aux stream
// after it.
void launch_relabel_csr(ipregel_graph* g, Partition& p) {
    RelabelCsr& R = p.relabel_csr;
    if (!R.armed) return;
    R.armed = false;
    cudaStream_t s = g->stream;
    ensure_aux_stream(g);
    cudaStream_t a = g->aux_stream;
    if (!p.csr_done) CU(cudaEventCreateWithFlags(&p.csr_done, cudaEventDisableTiming));
    CU(cudaEventRecord(p.csr_done, s));   // the CSC and every temporary are in place
    CU(cudaStreamWaitEvent(a, p.csr_done, 0));
    int32_t* kk0 = R.row;   // E int32 each
    int32_t* kk1 = R.spare;
    CU(cudaMemcpyAsync(kk0, R.idx, R.E * sizeof(int32_t), cudaMemcpyDeviceToDevice, a));
    if (R.w) k_transpose_pack_w<<<grid_for(R.n * 32, 256), 256, 0, a>>>(R.off, R.n, 0, R.w, R.k0);
    else k_transpose_pack<<<grid_for(R.n * 32, 256), 256, 0, a>>>(R.off, R.n, 0, R.k0);
    LAUNCH_CHECK();
    cub::DoubleBuffer<int32_t> tkeys(kk0, kk1);
    cub::DoubleBuffer<unsigned long long> tvals(R.k0, R.k1);
    CU(cub::DeviceRadixSort::SortPairs(R.t, R.tb, tkeys, tvals, R.E, 0, R.bits, a));
    k_unpack_w<<<std::min<unsigned>(grid_for(R.E, 256), sm_grid(16)), 256, 0, a>>>(
        tvals.Current(), R.E, R.ridx, R.rw);
    LAUNCH_CHECK();
    CU(cudaEventRecord(p.csr_done, a));
    g_ctrace.mark("relabel csr (aux)", a);
    for (auto& b : R.tmp.blocks) b.s = a;
    R.tmp.release();
}

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
        // the library relabel's out-degree histogram over the CSC sources (no CSR given, no
        // validation pass to wait for) runs window by window as the indices land, while the rest
        // uploads -- the GPU is otherwise idle until the structure is complete
        const bool hist = d.layout == IPREGEL_LAYOUT_DEGREE && !d.csr_offsets && !d.validate &&
                          idx_d && d.csc_edges >= (int64_t(1) << 24);
        if (hist) {
            p.pre_deg = p.pre_deg_mem.alloc<uint32_t>(g->n, s, true);
            constexpr int kHistWindows = 8;
            for (int c = 0; c < kHistWindows; ++c) {
                const int64_t lo = d.csc_edges * c / kHistWindows;
                const int64_t hi = d.csc_edges * (c + 1) / kHistWindows;
                up((int32_t*)idx_d + lo, (const int32_t*)d.csc_indices + lo, (hi - lo) * 4);
                cudaEvent_t e;
                CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                CU(cudaEventRecord(e, cs));
                compute_fence(s);
                CU(cudaStreamWaitEvent(s, e, 0));
                k_degree_hist<<<std::min<unsigned>(grid_for(hi - lo, 256), sm_grid(16)), 256, 0,
                                s>>>((const int32_t*)idx_d + lo, hi - lo, p.pre_deg);
                LAUNCH_CHECK();
                p.up_hist.push_back(e);   // destroyed with the partition
            }
        } else {
            up(idx_d, d.csc_indices, d.csc_edges * 4);
        }
        up(roff_d, d.csr_offsets, (p.rows + 1) * 4);
        up(ridx_d, d.csr_indices, d.csr_edges * 4);
        CU(cudaEventRecord(p.up_idx, cs));
        g_ctrace.mark("uploaded structure", cs);
        const bool relabel = d.layout == IPREGEL_LAYOUT_DEGREE;
        int windows = (derive && !relabel && w_d && d.csc_edges >= (int64_t(1) << 24))
                          ? kWeightWindows : 1;
        if (const char* e = getenv("IPREGEL_WEIGHT_WINDOWS"))   // test hook
            if (derive && !relabel && w_d) windows = std::max(1, std::min(atoi(e), 64));
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
    const bool relabel = d.layout == IPREGEL_LAYOUT_DEGREE;
    if (relabel) relabel_by_degree(g, p, d);
    if (!relabel && !d.csr_offsets && !d.csr_indices) {
        // out-adjacency (and its weights) derived from the CSC on the device: the transpose of
        // the whole graph's in-edges (single partition, checked by validate_desc;
        // after the validation: the transpose indexes by the CSC sources)
        int32_t *o, *ix;
        uint32_t* wx = nullptr;
        transpose_rows(p, g->n, p.csc_off, p.csc_idx, p.csc_w, p.csc_edges, p.csc_w != nullptr, s,
                       &o, &ix, &wx, d.memory == IPREGEL_MEMORY_HOST && !relabel);
        p.csr_off = o;
        p.csr_idx = ix;
        p.csr_w = wx;
        p.csr_edges = p.csc_edges;
        if (p.pend.perm) {
            // permute each weight window as it lands, on a side stream (the run stream goes
            // on with the tile plans); transpose_rows returned with perm complete
            ensure_aux_stream(g);
            for (size_t c = 0; c + 1 < p.wc_bounds.size(); ++c) {
                CU(cudaStreamWaitEvent(g->aux_stream, p.up_wc[c], 0));
                k_permute_window<<<sm_grid(8), 256, 0, g->aux_stream>>>(
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
        for (cudaEvent_t e : p.up_hist) cudaEventDestroy(e);
        if (p.perm_done) cudaEventDestroy(p.perm_done);
        p.perm_done = nullptr;
        if (p.csr_done) cudaEventDestroy(p.csr_done);
        p.csr_done = nullptr;
        p.up_wc.clear();
        p.up_hist.clear();
        p.pend.tmp.release();
        p.pre_deg_mem.release();        // non-empty only after a failed create
        p.relabel_csr.tmp.release();
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
