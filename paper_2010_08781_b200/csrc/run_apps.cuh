// paper_2010_08781_b200/csrc/run_apps.cuh -- the superstep loops of the paper's programs: PageRank (Fig. 8), Hash-Min CC (Fig. 9) and SSSP (Fig. 10).
// Host part of the single translation unit ipregel.cu (included once, in order).
#pragma once

namespace {

// =============================================================================================
// PageRank (Fig. 8)
// =============================================================================================
// part_ms of every gather superstep of a PageRank pull run (after finalize_times).
void fill_part_ms(ipregel_graph* g, uint32_t k) {
    for (uint32_t s = 1; s < g->steps.size() && s <= k; ++s) {
        float a = 0;
        CU(cudaEventElapsedTime(&a, ev(g, 4 * s + 1), ev(g, 4 * (k + 1) + s)));
        g->steps[s].part_ms = a;
    }
}

// IPREGEL_TRACE_KERNELS=1: per gather superstep of a PageRank pull run, the time of the range
// kernel + fixup, of k_pr_finish, and what the superstep adds around them (events on the run
// stream, the same clocks), printed to stderr -- the attribution of a superstep's time.
void trace_pr_kernels(ipregel_graph* g, uint32_t k) {
    for (uint32_t s = 1; s < g->steps.size() && s <= k; ++s) {
        float a = 0, b = 0, t = 0;
        CU(cudaEventElapsedTime(&a, ev(g, 4 * s + 1), ev(g, 4 * (k + 1) + s)));
        CU(cudaEventElapsedTime(&b, ev(g, 4 * (k + 1) + s), ev(g, 4 * s + 2)));
        CU(cudaEventElapsedTime(&t, ev(g, 4 * s + 0), ev(g, 4 * s + 3)));
        fprintf(stderr, "[ipregel pagerank] superstep %u: range kernel + fixup %.4f ms, "
                "k_pr_finish %.4f ms, superstep %.4f ms (other %.4f ms)\n", s, a, b, t,
                t - a - b);
    }
}

// Mass check: the per-superstep device sums into the step records (summed over ranks).
void read_mass(ipregel_graph* g) {
    cudaStream_t s = g->stream;
    const size_t m = 2 * g->steps.size();
    if (multi_rank(g))
        NC(ncclAllReduce(g->pr_mass, g->pr_mass, m, ncclFloat64, ncclSum, g->comm->nccl, s));
    std::vector<double> h(m);
    CU(cudaMemcpyAsync(h.data(), g->pr_mass, m * sizeof(double), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    for (size_t i = 0; i < g->steps.size(); ++i) {
        g->steps[i].mass[0] = h[2 * i];
        g->steps[i].mass[1] = h[2 * i + 1];
    }
}

ipregel_status run_pagerank(ipregel_graph* g, uint32_t max_steps, const ipregel_run_params& P) {
    cudaStream_t s = g->stream;
    const cudaStream_t user_stream = g->stream;
    const int64_t n = g->n;
    const uint32_t k = P.pagerank_iterations;
    const double ratio = 0.15 / (double)n;   // Pregel's 0.15 / NumVertices()
    const double inv_n = 1.0 / (double)n;    // initial_value
    const uint32_t last = std::min<uint32_t>(k, max_steps - 1);
    const bool push = P.mode == IPREGEL_MODE_PUSH;
    const bool fused = !push && use_fused_exchange(g, IPREGEL_APP_PAGERANK, P.flags);
    g->last_exchange = exchange_kind(g, fused);
    // to convergence (reading R27): ranks are kept every superstep and the max
    // per-vertex change is aggregated on the device; the host halts the run once it is <= tol
    const double tol = P.pagerank_tolerance;
    const bool track = tol >= 0.0;
    // mass check (IPREGEL_RUN_PAGERANK_MASS): per-superstep device sums, slot 2 s and 2 s + 1
    const bool mass = (P.flags & IPREGEL_RUN_PAGERANK_MASS) != 0;
    if (mass && g->pr_mass_cap < k + 1) {
        g->pr_mass = g->graph_mem.alloc<double>(2 * (size_t)(k + 1), s);
        g->pr_mass_cap = k + 1;
    }
    auto mass_slot = [&](uint32_t step) { return mass ? g->pr_mass + 2 * step : nullptr; };
    // PageRank broadcasters: vertices with out-degree > 0, summed over partitions / ranks
    int64_t nondangling = 0;
    for (auto& p : g->parts) nondangling += p.nondangling;
    if (multi_rank(g)) {
        Partition& p = g->parts[0];
        p.host_cnt[0] = (unsigned long long)p.nondangling;
        CU(cudaMemcpyAsync(p.dscratch, p.host_cnt, 8, cudaMemcpyHostToDevice, s));
        NC(ncclAllReduce(p.dscratch, p.dscratch + 1, 1, ncclUint64, ncclSum, g->comm->nccl, s));
        CU(cudaMemcpyAsync(p.host_cnt + 1, p.dscratch + 1, 8, cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
        nondangling = (int64_t)p.host_cnt[1];
    }

    // Fixed-k pull runs have no host synchronisation between supersteps: the whole run (superstep
    // 0 .. k, exchanges and per-superstep timing events included) is captured once as a CUDA
    // graph and replayed by every later run with the same parameters (IPREGEL_NO_GRAPHS=1: off).
    static const bool no_graphs = getenv("IPREGEL_NO_GRAPHS") != nullptr;
    const bool graphable = !track && !push && !g_persist_bytes && !no_graphs;
    auto& G = g->pr_graph;
    if (graphable && G.valid && G.k == k && G.max_steps == max_steps && G.flags == P.flags) {
        CU(cudaGraphLaunch(G.exec, s));
        g_launches.fetch_add(G.launches, std::memory_order_relaxed);
        g->steps = G.steps;
        g->cur = G.cur;
        g->last_exchange = G.exchange;
        finalize_times(g);
        if (mass) read_mass(g);
        if (g_pr_split && !push && !track) {
            fill_part_ms(g, k);
            if (g_trace_kernels) trace_pr_kernels(g, k);
        }
        return G.status;
    }
    // the flagged plan is built (once per graph) before anything is captured
    if (!push && k > 0 && g_pr_split && g_pr_flag)
        for (auto& p : g->parts)
            if (p.rows > 0) ensure_flag_plan(g, p);
    const unsigned long long launches0 = g_launches.load(std::memory_order_relaxed);
    if (graphable) {
        for (uint32_t i = 0; i <= 5 * (k + 1); ++i) ev(g, i);   // events exist before capture
        // capture on a private stream (the caller's may be the legacy default stream, which
        // cannot be captured); the graph is then launched on the caller's stream
        if (!g->capture_stream)
            CU(cudaStreamCreateWithFlags(&g->capture_stream, cudaStreamNonBlocking));
        g->stream = s = g->capture_stream;
        CU(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    }

    // superstep 0
    g->steps.assign(1, StepRecord{});
    StepTimer T0{g, 0};
    T0.begin();
    if (mass) CU(cudaMemsetAsync(g->pr_mass, 0, 2 * sizeof(double) * (k + 1), s));
    T0.kbegin();
    for (auto& p : g->parts) {
        AppState& S = p.st[IPREGEL_APP_PAGERANK];
        if (p.rows == 0) continue;
        k_init_pagerank<<<grid_for(ceil_div(p.rows, kInitRows), 256), 256, 0, s>>>(
                                                              p.csr_off, p.rows, p.vb, inv_n,
                                                              k > 0, last == 0 || track, S.rank,
                                                              S.contrib[0], mass_slot(0));
        LAUNCH_CHECK();
    }
    T0.kend();
    if (k > 0) exchange_owned<double>(g, [](Partition& p) { return p.st[0].contrib[0]; });
    T0.end();
    g->steps[0].mode = 0;
    g->steps[0].changed = k > 0 ? (uint64_t)nondangling : 0;
    g->steps[0].messages = k > 0 ? (uint64_t)g->e : 0;
    g->steps[0].model_bytes = 12ull * (uint64_t)n;
    int cur = 0;

    // push mode: static expand list of every source with push-view degree > 0
    if (push && k > 0) {
        for (auto& p : g->parts) {
            ensure_push_view(g, p);
            AppState& S = p.st[IPREGEL_APP_PAGERANK];
            if (!S.acc) S.acc = S.mem.alloc<double>(p.rows, s, true);
            if (!S.iota) {
                S.iota = S.mem.alloc<int32_t>(n, s);
                S.iota_len = S.mem.alloc<unsigned long long>(1, s);
                unsigned long long nn = (unsigned long long)n;
                CU(cudaMemcpyAsync(S.iota_len, &nn, sizeof(nn), cudaMemcpyHostToDevice, s));
                k_iota<<<grid_for(n, 256), 256, 0, s>>>(S.iota, n);
                LAUNCH_CHECK();
                CU(cudaStreamSynchronize(s));
            }
            build_expand_list(g, p, S, p.push_sssp, S.iota, nullptr, S.iota_len, n);
        }
    }

    ipregel_status status = IPREGEL_OK;
    for (uint32_t step = 1; step <= k; ++step) {
        if (step == max_steps) { status = IPREGEL_ERR_MAX_SUPERSTEPS; break; }
        const int broadcast = step < k;
        const int write_rank = step == last || track;
        g->steps.push_back(StepRecord{});
        StepTimer T{g, step};
        T.begin();
        if (track)
            for (auto& p : g->parts) CU(cudaMemsetAsync(p.pull_cnt, 0, sizeof(PullCounters), s));
        T.kbegin();
        for (auto& p : g->parts) {
            AppState& S = p.st[IPREGEL_APP_PAGERANK];
            if (p.rows == 0) continue;
            if (!push) {
                PageRankPull op;
                op.contrib_cur = S.contrib[cur];
                op.contrib_next = S.contrib[1 - cur];
                op.peers = peer_slots<double>(S, 1 - cur, fused && broadcast);
                op.rank = S.rank;
                op.out_off = p.csr_off;
                op.vbase = p.vb;
                op.ratio = ratio;
                op.broadcast = broadcast;
                op.write_rank = write_rank;
                op.track = track;
                op.mass = mass_slot(step);
                if (g_pr_split && g_pr_flag && g_pr_fuse && step >= 3 && broadcast &&
                    !write_rank && !track && !mass) {
                    // the flagged superstep with Fig. 8's update in its epilogue (the outbox
                    // entries of rows without in-edges were written by supersteps 1 and 2)
                    launch_pr_flag(g, p, op.contrib_cur, s, true, op.contrib_next, op.peers,
                                   ratio);
                    T.rec(4 * (k + 1) + step);   // no separate update pass
                } else if (g_pr_split && g_pr_flag) {
                    // the flagged superstep (pr_flag.cuh): sums by ordinal, then Fig. 8's update
                    launch_pr_flag(g, p, op.contrib_cur, s);
                    T.rec(4 * (k + 1) + step);   // range kernel + fixup done (stats part_ms)
                    op.sumc = p.plan_flag.sumc;
                    op.nzbits = p.plan_flag.nzbits;
                    op.nzpre = p.plan_flag.nzpre;
                    launch_pr_finish_compact(op, p.rows, track ? p.pull_cnt : nullptr,
                                             track || mass || (broadcast && write_rank) ? 0
                                                 : (broadcast ? 1 : 2), s);
                } else if (g_pr_split) {
                    PageRankSum sop;
                    sop.contrib_cur = op.contrib_cur;
                    sop.sum_out = op.contrib_next;
                    sop.vbase = p.vb;
                    launch_pull(sop, p.plan_csc, p.csc_off, p.csc_idx, nullptr, nullptr, s, n,
                                g->gather_policy, g->degree_ordered);
                    T.rec(4 * (k + 1) + step);   // range kernel + fixup done (stats part_ms)
                    const unsigned fg = grid_for(ceil_div(p.rows, kPrFinishRows), 256);
                    if (track || mass || (broadcast && write_rank))
                        k_pr_finish<0><<<fg, 256, 0, s>>>(op, p.rows, track ? p.pull_cnt : nullptr);
                    else if (broadcast)
                        k_pr_finish<1><<<fg, 256, 0, s>>>(op, p.rows, nullptr);
                    else
                        k_pr_finish<2><<<fg, 256, 0, s>>>(op, p.rows, nullptr);
                    LAUNCH_CHECK();
                } else {
                    launch_pull(op, p.plan_csc, p.csc_off, p.csc_idx, nullptr,
                                track ? p.pull_cnt : nullptr, s, n, g->gather_policy,
                                g->degree_ordered);
                }
            } else {
                k_expand<0><<<1184, kExpandThreads, 0, s>>>(
                    p.push_sssp, S.e_id, S.e_val, S.e_pre, &p.front_cnt->list_len,
                    &p.front_cnt->list_edges, p.vb, nullptr, nullptr, S.contrib[cur], S.acc);
                LAUNCH_CHECK();
                k_pr_push_apply<<<grid_for(p.rows, 256), 256, 0, s>>>(
                    S.acc, p.csr_off, p.rows, p.vb, ratio, broadcast, write_rank, S.rank,
                    S.contrib[1 - cur], track ? &p.pull_cnt->dmax : nullptr, mass_slot(step));
                LAUNCH_CHECK();
            }
        }
        T.kend();
        if (broadcast) {
            const int nx = 1 - cur;
            if (fused) fused_barrier(g);
            else exchange_owned<double>(g, [nx](Partition& p) { return p.st[0].contrib[nx]; });
        }
        T.end();
        StepRecord& R = g->steps.back();
        R.mode = push ? 2 : 1;
        R.changed = broadcast ? (uint64_t)nondangling : 0;
        R.messages = broadcast ? (uint64_t)g->e : 0;
        R.edges_scanned = (uint64_t)g->e;
        // 4 B index + 8 B gathered outbox per edge; 4 B CSC offset + 4 B
        // out-degree + 8 B rank + 8 B next outbox per vertex (fixed-k pull runs write the rank in
        // the last superstep only, so 12 E + 16 N of it is what they must move; bench.py reports
        // both)
        R.model_bytes = 12ull * g->e + 24ull * n;
        if (track) R.model_bytes += 8ull * n;    // the previous rank is read every superstep
        cur = 1 - cur;
        if (track) {
            const unsigned long long bits = reduce_max_delta(g);
            double d;
            memcpy(&d, &bits, 8);
            R.delta = d;
            if (d <= tol) break;   // master halt: converged
        }
    }
    g->cur = cur;
    if (graphable) {
        cudaGraph_t graph = nullptr;
        g->stream = user_stream;
        CU(cudaStreamEndCapture(s, &graph));
        s = user_stream;
        if (G.exec) cudaGraphExecDestroy(G.exec);
        G.exec = nullptr;
        G.valid = false;
        const cudaError_t ie = cudaGraphInstantiate(&G.exec, graph, 0);
        cudaGraphDestroy(graph);
        CU(ie);
        G.valid = true;
        G.k = k;
        G.max_steps = max_steps;
        G.flags = P.flags;
        G.steps = g->steps;
        G.cur = cur;
        G.exchange = g->last_exchange;
        G.status = status;
        G.launches = g_launches.load(std::memory_order_relaxed) - launches0;
        CU(cudaGraphLaunch(G.exec, s));
    }
    finalize_times(g);
    if (mass) read_mass(g);
    if (g_pr_split && !push && !track) {
        fill_part_ms(g, k);
        if (g_trace_kernels) trace_pr_kernels(g, k);
    }
    return status;
}

// =============================================================================================
// Hash-Min CC (Fig. 9) and SSSP (Fig. 10)
// =============================================================================================
// Smallest edge weight of the graph (1 without weights), over partitions / ranks; computed once.
uint32_t min_weight(ipregel_graph* g) {
    if (g->w_min >= 0) return (uint32_t)g->w_min;
    cudaStream_t s = g->stream;
    Partition& p0 = g->parts[0];
    unsigned long long m = 1;
    if (p0.csc_w) {
        DeviceBuffers tmp;
        unsigned* d = tmp.alloc<unsigned>(2, s);
        CU(cudaMemsetAsync(d, 0xFF, 8, s));
        for (auto& p : g->parts)
            if (p.csc_edges)
                k_min_u32<<<std::min<unsigned>(grid_for(p.csc_edges, 256), 4096), 256, 0, s>>>(
                    p.csc_w, p.csc_edges, d);
        LAUNCH_CHECK();
        if (multi_rank(g))
            NC(ncclAllReduce(d, d + 1, 1, ncclUint32, ncclMin, g->comm->nccl, s));
        unsigned h[2] = {0, 0};
        CU(cudaMemcpyAsync(h, d, 8, cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
        tmp.release();
        m = multi_rank(g) ? h[1] : h[0];
    }
    g->w_min = (int64_t)m;
    return (uint32_t)m;
}

// Hash-Min row-list pull: compact every partition's owned rows whose label is not 0 into its
// f_id list (front_cnt: count, symmetrised degree sum; host_cnt[4], [5]) and return the total
// degree over all partitions / ranks (the edges a row-list superstep would touch).
double rowlist_edges(ipregel_graph* g, int app, int cur) {
    cudaStream_t s = g->stream;
    for (auto& p : g->parts) {
        AppState& S = p.st[app];
        if (p.rows && !S.nbr) {   // once per graph: rows that have a neighbour at all
            S.nbr = S.mem.alloc<uint32_t>(words_of(p.rows), s);
            k_nbr_bits<<<grid_for(p.rows, 256), 256, 0, s>>>(p.csc_off, p.csr_off, p.rows, S.nbr);
            LAUNCH_CHECK();
        }
        if (p.rows)
            k_bits_ne<<<std::max<unsigned>(1u, std::min<unsigned>(
                            grid_for(ceil_div(p.rows, 1024) * 32, 256), sm_grid(16))),
                        256, 0, s>>>(S.val[cur] + p.vb, p.rows, 0u, S.nbr, S.bits);
        LAUNCH_CHECK();
        compact_bitmap(g, p, S, S.val[cur], true);
        CU(cudaMemcpyAsync(p.host_cnt + 4, p.front_cnt, 16, cudaMemcpyDeviceToHost, s));
    }
    CU(cudaStreamSynchronize(s));
    double total = 0;
    for (auto& p : g->parts) total += (double)p.host_cnt[5];
    if (multi_rank(g)) {
        Partition& p = g->parts[0];
        CU(cudaMemcpyAsync(p.dscratch + 60, &p.front_cnt->messages, 8, cudaMemcpyDeviceToDevice, s));
        NC(ncclAllReduce(p.dscratch + 60, p.dscratch + 61, 1, ncclUint64, ncclSum, g->comm->nccl, s));
        CU(cudaMemcpyAsync(p.host_cnt + 6, p.dscratch + 61, 8, cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
        total = (double)p.host_cnt[6];
    }
    g->last_rowlist_edges = (int64_t)total;
    return total;
}

ipregel_status run_min(ipregel_graph* g, int app, uint32_t max_steps, const ipregel_run_params& P) {
    wait_csr(g);   // Hash-Min gathers over the CSR; push expands over it
    cudaStream_t s = g->stream;
    const int64_t n = g->n;
    const bool cc = app == IPREGEL_APP_HASHMIN_CC;
    const int np = (int)g->parts.size();
    const bool multi = np > 1 || multi_rank(g);
    // edges a pull superstep scans (CC gathers over CSC and CSR rows: the symmetrised graph)
    const uint64_t pull_edges = cc ? 2ull * (uint64_t)g->e : (uint64_t)g->e;
    const bool fused = P.mode != IPREGEL_MODE_PUSH && use_fused_exchange(g, app, P.flags);
    g->last_exchange = exchange_kind(g, fused);

    for (auto& p : g->parts) ensure_push_view(g, p);
    // SSSP_SOURCE is an original id; find its internal id under a relabelled layout
    int64_t source = (int64_t)P.sssp_source;
    if (!cc && g->vertex_ids) {
        Partition& p0 = g->parts[0];
        const unsigned long long none = ~0ull;
        CU(cudaMemcpyAsync(p0.dscratch + 32, &none, 8, cudaMemcpyHostToDevice, s));
        k_find_index<<<std::min<unsigned>(grid_for(n, 256), 4096), 256, 0, s>>>(
            g->vertex_ids, n, (int32_t)P.sssp_source, p0.dscratch + 32);
        LAUNCH_CHECK();
        CU(cudaMemcpyAsync(p0.host_cnt + 15, p0.dscratch + 32, 8, cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
        source = (int64_t)p0.host_cnt[15];
        if (source < 0 || source >= n) fail(IPREGEL_ERR_INVALID_GRAPH, "vertex_ids is not a permutation");
    }

    // ---------------- superstep 0
    g->steps.assign(1, StepRecord{});
    StepTimer T0{g, 0};
    T0.begin();
    T0.kbegin();
    for (auto& p : g->parts) {
        AppState& S = p.st[app];
        const unsigned ig = std::min<unsigned>(grid_for(ceil_div(n, 4), 256), sm_grid(16));
        if (cc) k_init_cc<<<ig, 256, 0, s>>>(S.val[0], n, g->vertex_ids);
        else k_init_sssp<<<ig, 256, 0, s>>>(S.val[0], n, source);
        LAUNCH_CHECK();
    }
    T0.kend();
    uint64_t changed = 0, messages = 0;
    bool lists_ready = false;
    if (cc) {
        changed = (uint64_t)n;
        messages = 2ull * (uint64_t)g->e;
    } else {
        // the source's broadcast: its frontier entry and out-degree come from the compaction
        for (auto& p : g->parts) {
            AppState& S = p.st[app];
            if (source >= p.vb && source < p.ve) {
                k_set_bit<<<1, 1, 0, s>>>(S.bits, source - p.vb);
                LAUNCH_CHECK();
            }
            compact_bitmap(g, p, S, S.val[0], false);
        }
        if (multi) exchange_frontier(g, app, frontier_counts(g), 0);
        unsigned long long c[2];
        reduce_counters(g, true, c, 2);
        changed = c[0];
        messages = c[1];
        lists_ready = true;
    }
    T0.end();
    g->steps[0].mode = 0;
    g->steps[0].changed = changed;
    g->steps[0].messages = messages;
    g->steps[0].model_bytes = 4ull * (uint64_t)n;
    int cur = 0;
    int prev_mode = 0;
    uint64_t zero_edges = 0;   // Hash-Min: symmetrised degree of the rows at label 0 (last pull)
    // SSSP absorption bound: smallest distance that changed in the last superstep (the source's
    // 0 after superstep 0) plus the smallest edge weight
    const uint32_t w_min = cc ? 0u : min_weight(g);
    uint32_t m_prev = 0;
    ipregel_status status = IPREGEL_OK;

    for (uint32_t step = 1; messages > 0; ++step) {
        if (step == max_steps) { status = IPREGEL_ERR_MAX_SUPERSTEPS; break; }
        // delivery mode for this superstep (Ligra-style switch)
        int mode;
        if (P.mode == IPREGEL_MODE_PULL) mode = 1;
        else if (P.mode == IPREGEL_MODE_PUSH) mode = 2;
        else mode = (double)messages < (double)P.push_fraction * (double)pull_edges ? 2 : 1;

        g->steps.push_back(StepRecord{});
        StepTimer T{g, step};
        T.begin();
        uint64_t frontier_len = changed;

        if (mode == 2) {
            // ---- push: make the frontier list of the previous superstep's broadcasters
            if (!lists_ready) {
                for (auto& p : g->parts) {
                    AppState& S = p.st[app];
                    if (prev_mode == 0) {
                        k_fill_bits<<<grid_for(words_of(p.rows), 256), 256, 0, s>>>(S.bits, p.rows);
                    } else {
                        // pull -> push: broadcasters = vertices whose value decreased
                        k_bitmap_from_diff<<<std::max<unsigned>(1u, std::min<unsigned>(
                                                 grid_for(ceil_div(p.rows, 1024) * 32, 256),
                                                 sm_grid(16))), 256, 0, s>>>(
                            S.val[1 - cur], S.val[cur], p.vb, p.rows, S.bits);
                    }
                    LAUNCH_CHECK();
                    compact_bitmap(g, p, S, S.val[cur], cc);
                }
                if (multi) exchange_frontier(g, app, frontier_counts(g), cur);
            }
            T.kbegin();
            for (auto& p : g->parts) {
                AppState& S = p.st[app];
                const PushAdj& adj = cc ? p.push_cc : p.push_sssp;
                build_expand_list(g, p, S, adj, S.g_id, S.g_val, S.g_len, (int64_t)frontier_len);
                const unsigned grid = (unsigned)std::min<int64_t>(
                    std::max<int64_t>(ceil_div((int64_t)messages, kExpandItems), 1), sm_grid(8));
                if (cc)
                    k_expand<1><<<grid, kExpandThreads, 0, s>>>(
                        adj, S.e_id, S.e_val, S.e_pre, &p.front_cnt->list_len,
                        &p.front_cnt->list_edges, p.vb, S.val[cur], S.bits, nullptr, nullptr);
                else
                    k_expand<2><<<grid, kExpandThreads, 0, s>>>(
                        adj, S.e_id, S.e_val, S.e_pre, &p.front_cnt->list_len,
                        &p.front_cnt->list_edges, p.vb, S.val[cur], S.bits, nullptr, nullptr);
                LAUNCH_CHECK();
            }
            T.kend();
            // broadcasters of this superstep -> next frontier (+ counters)
            for (auto& p : g->parts) compact_bitmap(g, p, p.st[app], p.st[app].val[cur], cc);

            if (multi) exchange_frontier(g, app, frontier_counts(g), cur);
            unsigned long long c[2];
            reduce_counters(g, true, c, 2);
            T.end();
            StepRecord& R = g->steps.back();
            R.mode = 2;
            R.edges_scanned = messages;
            R.model_bytes = (cc ? 8ull : 12ull) * messages + 16ull * frontier_len +
                            (uint64_t)n / 8;
            changed = c[0];
            messages = c[1];
            lists_ready = true;
        } else if (cc && g_rowlist > 0.0 &&
                   (prev_mode == 3 || (prev_mode == 1 && (double)(pull_edges - zero_edges) <
                                                             g_rowlist * (double)pull_edges))) {
            // ---- row-list pull (Hash-Min): only the rows not at label 0 gather (once a row is
            // at 0 it stays there, so the list only shrinks)
            rowlist_edges(g, app, cur);   // their list in f_id / front_cnt
            T.kbegin();
            for (auto& p : g->parts) {
                AppState& S = p.st[app];
                if (p.rows == 0) continue;
                CU(cudaMemcpyAsync(S.val[1 - cur] + p.vb, S.val[cur] + p.vb, p.rows * 4,
                                   cudaMemcpyDeviceToDevice, s));
                const PushAdj own{p.csc_off, p.csc_idx, nullptr, p.csr_off, p.csr_idx, nullptr,
                                  p.vb, p.rows};
                build_expand_list(g, p, S, own, S.f_id, nullptr, &p.front_cnt->changed,
                                  (int64_t)p.host_cnt[4]);
                const unsigned grid = (unsigned)std::min<int64_t>(
                    std::max<int64_t>(ceil_div((int64_t)p.host_cnt[5], kExpandItems), 1), sm_grid(8));
                k_rowlist_min<<<grid, kExpandThreads, 0, s>>>(
                    own, S.e_id, S.e_pre, &p.front_cnt->list_len, &p.front_cnt->list_edges,
                    S.val[cur], S.val[1 - cur]);
                LAUNCH_CHECK();
            }
            T.kend();
            // broadcasters = rows whose label decreased (only listed rows can): their count and
            // symmetrised degrees
            for (auto& p : g->parts) {
                AppState& S = p.st[app];
                CU(cudaMemsetAsync(S.bits, 0, words_of(p.rows) * sizeof(uint32_t), s));
                k_bits_from_list_diff<<<std::max<unsigned>(1u, std::min<unsigned>(
                                            grid_for((int64_t)p.host_cnt[4], 256), sm_grid(8))),
                                        256, 0, s>>>(S.f_id, &p.front_cnt->changed, S.val[cur],
                                                     S.val[1 - cur], p.vb, S.bits);
                LAUNCH_CHECK();
                compact_bitmap(g, p, S, S.val[1 - cur], true);
            }
            const int nx = 1 - cur;
            exchange_owned<uint32_t>(g, [app, nx](Partition& p) { return p.st[app].val[nx]; });
            unsigned long long c[2];
            reduce_counters(g, true, c, 2);
            T.end();
            StepRecord& R = g->steps.back();
            R.mode = 3;
            mode = 3;
            R.edges_scanned = (uint64_t)g->last_rowlist_edges;
            R.model_bytes = 12ull * (uint64_t)g->last_rowlist_edges + 16ull * (uint64_t)n;
            changed = c[0];
            messages = c[1];
            cur = 1 - cur;
            // the broadcasters were compacted above (ids + new labels): on one partition that
            // is the next push superstep's frontier as it stands (ranks / loopback partitions
            // still need the frontier exchange, done by the push branch)
            lists_ready = !multi;
        } else {
            // ---- pull: gather over CSC (and CSR for CC), value[next] = min(value, gathered)
            if (!cc && prev_mode == 2) {
                // absorption bound after a push superstep: the smallest distance among its
                // broadcasters (the owned frontier lists still hold their snapshots)
                for (auto& p : g->parts) {
                    CU(cudaMemsetAsync(&p.pull_cnt->dmax, 0, 8, s));
                    k_list_max_inv<<<std::max<unsigned>(1u, std::min<unsigned>(
                                         grid_for((int64_t)std::max<uint64_t>(changed, 1), 256),
                                         1024)),
                                     256, 0, s>>>(p.st[app].f_val, &p.front_cnt->changed,
                                                  &p.pull_cnt->dmax);
                    LAUNCH_CHECK();
                }
                m_prev = (uint32_t)(kInf - (uint32_t)reduce_max_delta(g));
            }
            for (auto& p : g->parts) CU(cudaMemsetAsync(p.pull_cnt, 0, sizeof(PullCounters), s));
            T.kbegin();
            for (auto& p : g->parts) {
                AppState& S = p.st[app];
                if (p.rows == 0) continue;
                if (cc) {
                    CCPullIn a;
                    a.cur = S.val[cur]; a.next = S.val[1 - cur]; a.vbase = p.vb;
                    // counters: only its gathered edges (the CSR pass counts the changes)
                    launch_pull(a, p.plan_csc, p.csc_off, p.csc_idx, nullptr, p.pull_cnt, s, n,
                                g->gather_policy, g->degree_ordered);
                    CCPullOut b;
                    b.cur = S.val[cur]; b.next = S.val[1 - cur]; b.in_off = p.csc_off;
                    b.out_off = p.csr_off; b.vbase = p.vb;
                    b.count_all_zero = prev_mode != 1;   // else zero_edges is kept up to date
                    b.peers = peer_slots<uint32_t>(S, 1 - cur, fused);
                    launch_pull(b, p.plan_csr, p.csr_off, p.csr_idx, nullptr, p.pull_cnt, s, n,
                                g->gather_policy, g->degree_ordered);
                } else {
                    SSSPPull a;
                    a.cur = S.val[cur]; a.next = S.val[1 - cur];
                    a.out_off = p.csr_off; a.vbase = p.vb;
                    a.peers = peer_slots<uint32_t>(S, 1 - cur, fused);
                    a.thr = sat_add_host(m_prev, w_min);
                    launch_pull(a, p.plan_csc, p.csc_off, p.csc_idx, p.csc_w, p.pull_cnt, s, n,
                                g->gather_policy, g->degree_ordered);
                }
            }
            T.kend();
            const int nx = 1 - cur;
            // fused: the epilogue already stored the owned slice into every replica; the counter
            // AllReduce below is the superstep barrier
            if (!fused)
                exchange_owned<uint32_t>(g, [app, nx](Partition& p) { return p.st[app].val[nx]; });
            unsigned long long c[5];
            reduce_counters(g, false, c, 5);
            // rows at label 0 stay there: after a plain pull superstep only the new ones count
            zero_edges = prev_mode != 1 ? c[3] : zero_edges + c[3];
            if (!cc) m_prev = (uint32_t)(kInf - (uint32_t)reduce_max_delta(g));
            T.end();
            StepRecord& R = g->steps.back();
            R.mode = 1;
            // the edges whose messages were gathered: absorbed rows / ranges skip theirs, so a
            // superstep's model bytes count only the gathers it did (SURVEY.md 8(d) per edge)
            R.edges_scanned = c[4];
            R.model_bytes = cc ? 8ull * c[4] + 16ull * n : 12ull * c[4] + 12ull * n;
            changed = c[0];
            messages = c[1];
            cur = 1 - cur;
            lists_ready = false;
        }
        prev_mode = mode;
        StepRecord& R = g->steps.back();
        R.changed = changed;
        R.messages = messages;
    }
    g->cur = cur;
    finalize_times(g);
    return status;
}

}  // namespace
