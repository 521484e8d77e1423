// paper_2010_08781_b200/csrc/run_programs.cuh -- user vertex programs: NVRTC compilation, kernel loading and the generic superstep loop.
// Host part of the single translation unit ipregel.cu (included once, in order).
#pragma once

// =============================================================================================
// user vertex programs: NVRTC compilation and the generic superstep loop
// =============================================================================================
enum { PK_INIT, PK_PULL0, PK_PULL1, PK_PULL2, PK_FIX0, PK_FIX1, PK_FIX2, PK_EXPAND, PK_APPLY,
       PK_PULL_APPLY, PK_BOUND, PK_COUNT };
static const char* const kProgKernelNames[PK_COUNT] = {
    "ipr::k_prog_init<UserProgram>",
    "ipr::k_pull_ranges<ipr::ProgPull<UserProgram, 0> >",
    "ipr::k_pull_ranges<ipr::ProgPull<UserProgram, 1> >",
    "ipr::k_pull_ranges<ipr::ProgPull<UserProgram, 2> >",
    "ipr::k_pull_fixup<ipr::ProgPull<UserProgram, 0> >",
    "ipr::k_pull_fixup<ipr::ProgPull<UserProgram, 1> >",
    "ipr::k_pull_fixup<ipr::ProgPull<UserProgram, 2> >",
    "ipr::k_prog_expand<UserProgram>",
    "ipr::k_prog_apply<UserProgram>",
    "ipr::k_prog_pull_apply<UserProgram>",
    "ipr::k_prog_bound<UserProgram>",
};

struct ipregel_program {
    int value_type = 0;   // ipregel_value_type
    int combiner = 0;     // ipregel_combiner
    int sym = 0;
    int agg_op = -1;      // aggregator (ipregel_combiner over f64), -1 none
    bool sends = false;   // the source calls ipr_send (point-to-point messages)
    bool settled = false; // the source defines ipr_settled (MIN combiner, no ipr_send)
    std::vector<char> cubin;
    std::string log;
    std::string lowered[PK_COUNT];
    cudaLibrary_t lib = nullptr;
    cudaKernel_t k[PK_COUNT] = {};
    int pull_per_sm[2] = {1, 1};   // resident CTAs per SM of the loaded range kernels
};

namespace {

// NVRTC is loaded on first use (dlopen), so the library itself loads without it.
struct Nvrtc {
    bool ok = false;
    std::string why;
    nvrtcResult (*create)(nvrtcProgram*, const char*, const char*, int, const char* const*,
                          const char* const*) = nullptr;
    nvrtcResult (*add_name)(nvrtcProgram, const char*) = nullptr;
    nvrtcResult (*compile)(nvrtcProgram, int, const char* const*) = nullptr;
    nvrtcResult (*log_size)(nvrtcProgram, size_t*) = nullptr;
    nvrtcResult (*log)(nvrtcProgram, char*) = nullptr;
    nvrtcResult (*cubin_size)(nvrtcProgram, size_t*) = nullptr;
    nvrtcResult (*cubin)(nvrtcProgram, char*) = nullptr;
    nvrtcResult (*lowered)(nvrtcProgram, const char*, const char**) = nullptr;
    nvrtcResult (*destroy)(nvrtcProgram*) = nullptr;
    const char* (*err)(nvrtcResult) = nullptr;
};

Nvrtc load_nvrtc() {
    Nvrtc N;
    const char* cands[] = {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12"};
    void* h = nullptr;
    for (const char* c : cands)
        if ((h = dlopen(c, RTLD_NOW | RTLD_LOCAL)) != nullptr) break;
    if (!h) {
        N.why = "libnvrtc.so.12 not found";
        return N;
    }
    bool ok = true;
    auto sym = [&](const char* name) {
        void* f = dlsym(h, name);
        if (!f) ok = false;
        return f;
    };
    N.create = (decltype(N.create))sym("nvrtcCreateProgram");
    N.add_name = (decltype(N.add_name))sym("nvrtcAddNameExpression");
    N.compile = (decltype(N.compile))sym("nvrtcCompileProgram");
    N.log_size = (decltype(N.log_size))sym("nvrtcGetProgramLogSize");
    N.log = (decltype(N.log))sym("nvrtcGetProgramLog");
    N.cubin_size = (decltype(N.cubin_size))sym("nvrtcGetCUBINSize");
    N.cubin = (decltype(N.cubin))sym("nvrtcGetCUBIN");
    N.lowered = (decltype(N.lowered))sym("nvrtcGetLoweredName");
    N.destroy = (decltype(N.destroy))sym("nvrtcDestroyProgram");
    N.err = (decltype(N.err))sym("nvrtcGetErrorString");
    N.ok = ok;
    if (!ok) N.why = "libnvrtc lacks a required symbol";
    return N;
}

const Nvrtc& nvrtc() {
    static Nvrtc N = load_nvrtc();
    return N;
}

// The translation unit NVRTC compiles: the library's own device headers, the user source, and
// the adapter the kernel templates are instantiated on.
std::string program_tu(const ipregel_program_desc& d) {
    const char* vt = d.value_type == IPREGEL_VALUE_F64   ? "double"
                   : d.value_type == IPREGEL_VALUE_F32 ? "float"
                   : d.value_type == IPREGEL_VALUE_I32 ? "int"
                   : d.value_type == IPREGEL_VALUE_U64 ? "unsigned long long"
                   : d.value_type == IPREGEL_VALUE_I64 ? "long long"
                                                       : "unsigned int";
    std::string s;
    s += "#include \"program.cuh\"\n";
    s += "typedef ipr::ProgCtx ipr_ctx;\n";
    s += std::string("typedef ") + vt + " ipr_value_t;\n";
    s += "#define IPR_BROADCAST 1u\n#define IPR_STAY_ACTIVE 2u\n#define IPR_INF_U32 0xFFFFFFFFu\n";
    s += "__device__ __forceinline__ unsigned ipr_sat_add(unsigned a, unsigned b) "
         "{ return ipr::sat_add(a, b); }\n";
    s += "__device__ __forceinline__ void ipr_send(const ipr_ctx& c, long long dest, "
         "ipr_value_t m) { ipr::prog_send<ipr_value_t, " + std::to_string(d.combiner) +
         ">(c, dest, m); }\n";
    s += "__device__ __forceinline__ void ipr_aggregate(const ipr_ctx& c, double x) "
         "{ ipr::prog_aggregate(c, x); }\n";
    s += "#line 1 \"user_program.cu\"\n";
    s += d.source;
    s += "\n#line 1 \"ipregel_program_adapter\"\n";
    s += "struct UserProgram {\n  typedef ipr_value_t V;\n";
    s += "  static constexpr int kCombiner = " + std::to_string(d.combiner) + ";\n";
    s += std::string("  static constexpr bool kSym = ") + (d.symmetric ? "true" : "false") + ";\n";
    s += std::string("  static constexpr bool kSends = ") +
         (strstr(d.source, "ipr_send") ? "true" : "false") + ";\n";
    s += std::string("  static constexpr bool kAggregates = ") +
         (d.aggregator != IPREGEL_AGG_NONE ? "true" : "false") + ";\n";
    const bool absorbing = strstr(d.source, "ipr_absorbing") != nullptr;
    // ipr_settled: MIN programs without point-to-point sends (their messages bypass the bound)
    const bool settled = strstr(d.source, "ipr_settled") != nullptr &&
                         d.combiner == IPREGEL_COMBINE_MIN && !strstr(d.source, "ipr_send");
    s += std::string("  static constexpr bool kSettled = ") + (settled ? "true" : "false") + ";\n";
    if (settled)
        s += "  static __device__ __forceinline__ bool settled(V v, V b) { return ipr_settled(v, b); }\n";
    else
        s += "  static __device__ __forceinline__ bool settled(V, V) { return false; }\n";
    s += std::string("  static constexpr bool kAbsorbing = ") + (absorbing ? "true" : "false") + ";\n";
    if (absorbing)
        s += "  static __device__ __forceinline__ bool absorbing(V v) { return ipr_absorbing(v); }\n";
    else
        s += "  static __device__ __forceinline__ bool absorbing(V) { return false; }\n";
    s += "  static __device__ __forceinline__ unsigned init(const ipr::ProgCtx& c, V* v, V* m) "
         "{ return ipr_init(c, v, m); }\n";
    s += "  static __device__ __forceinline__ unsigned compute(const ipr::ProgCtx& c, V* v, V mb, "
         "V* m) { return ipr_compute(c, v, mb, m); }\n";
    s += "  static __device__ __forceinline__ V edge(V m, unsigned w) { return ipr_edge(m, w); }\n";
    s += "};\n";
    return s;
}

void compile_program(ipregel_program* pr, const ipregel_program_desc& d) {
    const Nvrtc& N = nvrtc();
    if (!N.ok) fail(IPREGEL_ERR_UNSUPPORTED, "NVRTC unavailable: %s", N.why.c_str());
    const std::string tu = program_tu(d);
    nvrtcProgram prog;
    nvrtcResult r = N.create(&prog, tu.c_str(), "ipregel_program.cu", kJitHeaderCount,
                             kJitHeaderBodies, kJitHeaderNames);
    if (r != NVRTC_SUCCESS) fail(IPREGEL_ERR_CUDA, "nvrtcCreateProgram: %s", N.err(r));
    for (int i = 0; i < PK_COUNT; ++i) N.add_name(prog, kProgKernelNames[i]);
    // IEEE arithmetic as written (no FMA contraction), the oracle's convention (R7).
    // Every build-time knob of the range kernels is passed on, so the JIT kernels are the same
    // shape as the host launches them (CTA size, warps per CTA, range size, unroll, paths).
    const std::string knobs[] = {
        "-DIPREGEL_PULL_THREADS=" + std::to_string(kPullThreads),
        "-DIPREGEL_PULL_MINBLOCKS=" + std::to_string(IPREGEL_PULL_MINBLOCKS),
        "-DIPREGEL_PROG_MINBLOCKS8=" + std::to_string(IPREGEL_PROG_MINBLOCKS8),
        "-DIPREGEL_RANGE_ITEMS=" + std::to_string(kRangeItems),
        "-DIPREGEL_CHUNK_UNROLL=" + std::to_string(kChunkUnroll),
        "-DIPREGEL_U32_ONE_END=" + std::to_string(IPREGEL_U32_ONE_END),
        "-DIPREGEL_IDX_PREFETCH=" + std::to_string(IPREGEL_IDX_PREFETCH),
        "-DIPREGEL_GATHER_HINT=" + std::to_string(IPREGEL_GATHER_HINT),
        "-DIPREGEL_STREAM_CS=" + std::to_string(IPREGEL_STREAM_CS)};
    std::vector<const char*> opts = {"--gpu-architecture=sm_100a", "-std=c++17", "--fmad=false",
                                     "-lineinfo", "-default-device", "--ptxas-options=-v",
                                     "-DIPREGEL_JIT=1"};
    for (const std::string& k : knobs) opts.push_back(k.c_str());
    // tuning knob: one extra NVRTC option (e.g. -DIPREGEL_PROG_MINBLOCKS8=3 -- the launch reads
    // the resident CTAs of the loaded kernel, so it stays consistent)
    const char* extra = getenv("IPREGEL_NVRTC_OPT");
    if (extra && *extra) opts.push_back(extra);
    r = N.compile(prog, (int)opts.size(), opts.data());
    size_t ls = 0;
    N.log_size(prog, &ls);
    std::string log(ls, '\0');
    if (ls) N.log(prog, &log[0]);
    while (!log.empty() && (log.back() == '\0' || log.back() == '\n')) log.pop_back();
    pr->log = log;
    if (r != NVRTC_SUCCESS) {
        N.destroy(&prog);
        fail(IPREGEL_ERR_INVALID_ARGUMENT, "vertex program does not compile (%s):\n%.3500s",
             N.err(r), log.c_str());
    }
    size_t cs = 0;
    N.cubin_size(prog, &cs);
    pr->cubin.resize(cs);
    N.cubin(prog, pr->cubin.data());
    for (int i = 0; i < PK_COUNT; ++i) {
        const char* low = nullptr;
        if (N.lowered(prog, kProgKernelNames[i], &low) != NVRTC_SUCCESS || !low) {
            N.destroy(&prog);
            fail(IPREGEL_ERR_CUDA, "nvrtcGetLoweredName(%s) failed", kProgKernelNames[i]);
        }
        pr->lowered[i] = low;
    }
    N.destroy(&prog);
}

void ensure_program_loaded(ipregel_program* pr) {
    if (pr->lib) return;
    CU(cudaLibraryLoadData(&pr->lib, pr->cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
    for (int i = 0; i < PK_COUNT; ++i)
        CU(cudaLibraryGetKernel(&pr->k[i], pr->lib, pr->lowered[i].c_str()));
    // the range kernels launch with kPullThreads: check the loaded kernels accept that, and take
    // their resident CTAs per SM from the occupancy of the kernel actually loaded
    for (int pass = 0; pass < 2; ++pass) {
        cudaFuncAttributes fa;
        CU(cudaFuncGetAttributes(&fa, (const void*)pr->k[PK_PULL0 + pass]));
        if (fa.maxThreadsPerBlock < kPullThreads)
            fail(IPREGEL_ERR_UNSUPPORTED, "program range kernel takes %d threads per CTA, the "
                 "launch needs %d", fa.maxThreadsPerBlock, kPullThreads);
        int per_sm = 0;
        CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &per_sm, (const void*)pr->k[PK_PULL0 + pass], kPullThreads, 0));
        pr->pull_per_sm[pass] = std::max(per_sm, 1);
    }
}

void launch_jit(cudaKernel_t k, unsigned grid, unsigned block, void** args, cudaStream_t s) {
    if (grid == 0) return;
    CU(cudaLaunchKernel((const void*)k, dim3(grid), dim3(block), args, 0, s));
    LAUNCH_CHECK();
}

// Bit pattern of the program combiner's identity in an 8-byte slot (u32 in the low half).
uint64_t prog_identity_bits(const ipregel_program* pr) {
    const int c = pr->combiner;
    switch (pr->value_type) {
        case IPREGEL_VALUE_F64: {
            const double id = c == IPREGEL_COMBINE_SUM ? 0.0 : (c == IPREGEL_COMBINE_MIN ? INFINITY : -INFINITY);
            uint64_t b;
            memcpy(&b, &id, 8);
            return b;
        }
        case IPREGEL_VALUE_F32: {
            const float id = c == IPREGEL_COMBINE_SUM ? 0.0f : (c == IPREGEL_COMBINE_MIN ? INFINITY : -INFINITY);
            uint32_t b;
            memcpy(&b, &id, 4);
            return b;
        }
        case IPREGEL_VALUE_I32:
            return c == IPREGEL_COMBINE_SUM ? 0ull : (c == IPREGEL_COMBINE_MIN ? 0x7FFFFFFFull : 0x80000000ull);
        case IPREGEL_VALUE_U64:
            return c == IPREGEL_COMBINE_MIN ? ~0ull : 0ull;
        case IPREGEL_VALUE_I64:
            return c == IPREGEL_COMBINE_SUM ? 0ull
                 : (c == IPREGEL_COMBINE_MIN ? 0x7FFFFFFFFFFFFFFFull : 0x8000000000000000ull);
        default:
            return c == IPREGEL_COMBINE_MIN ? 0xFFFFFFFFull : 0ull;
    }
}

size_t value_bytes(int value_type) {
    return (value_type == IPREGEL_VALUE_F64 || value_type == IPREGEL_VALUE_U64 ||
            value_type == IPREGEL_VALUE_I64) ? 8 : 4;
}

// original -> internal id (the inverse of vertex_ids), built once per graph; NULL without a
// relabelled layout.
const int32_t* inverse_ids(ipregel_graph* g) {
    if (!g->vertex_ids) return nullptr;
    if (!g->inv_ids) {
        int32_t* inv = g->graph_mem.alloc<int32_t>(g->n, g->stream);
        k_invert_ids<<<grid_for(g->n, 256), 256, 0, g->stream>>>(g->vertex_ids, g->n, inv);
        LAUNCH_CHECK();
        g->inv_ids = inv;
    }
    return g->inv_ids;
}

// One pull pass of a program over one adjacency (the ProgPull<P, pass> instantiation).
template <class V>
void launch_pull_program(ipregel_graph* g, const ipregel_program* pr, int pass, ProgArgs<V>& a,
                         const TilePlan& P, const int32_t* off, const int32_t* idx,
                         const uint32_t* w, PullCounters* cnt) {
    if (P.num_tiles == 0) return;
    RangeArgs A = range_args(P, off, idx, w, cnt, g->stream, a.out_cur, g->n, sizeof(V),
                             g->gather_policy, g->degree_ordered);
    void* args[] = {&a, &A};
    // resident CTAs per SM of the loaded JIT kernel (its occupancy, ensure_program_loaded)
    const int64_t need = ceil_div(P.num_tiles, kWarpsPerCta);
    const int64_t resident = (int64_t)device_sms(g->device) * pr->pull_per_sm[pass];
    const unsigned grid = (unsigned)(g_pull_waves == 0 || !A.range_ctr
                                         ? need : std::min<int64_t>(need, resident * g_pull_waves));
    launch_jit(pr->k[PK_PULL0 + pass], grid, kPullThreads,
               args, g->stream);
    if (P.num_groups) {
        const int4* groups = P.groups;
        int32_t ng = P.num_groups, ns = P.num_short;
        const V* carry = static_cast<const V*>(P.carry);
        const V* head = static_cast<const V*>(P.head);
        void* fargs[] = {&a, &groups, &ng, &ns, &carry, &head, &cnt};
        launch_jit(pr->k[PK_FIX0 + pass], fixup_grid(ng, ns), 256, fargs, g->stream);
    }
}

template <class V>
ipregel_status run_program_t(ipregel_graph* g, ipregel_program* pr, uint32_t max_steps,
                             const ipregel_run_params& P, const double* params, int nparams) {
    wait_csr(g);   // symmetric pulls and push read the CSR
    cudaStream_t s = g->stream;
    const int64_t n = g->n;
    const int app = kAppProgram;
    const bool sym = pr->sym != 0;
    const bool multi = g->parts.size() > 1 || multi_rank(g);
    const uint64_t pull_edges = sym ? 2ull * (uint64_t)g->e : (uint64_t)g->e;
    ensure_program_loaded(pr);
    const bool fused = use_fused_exchange(g, app, P.flags);
    g->last_exchange = exchange_kind(g, fused);
    if (P.mode != IPREGEL_MODE_PULL)
        for (auto& p : g->parts) ensure_push_view(g, p);
    double hp[kProgParams] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int i = 0; i < nparams; ++i) hp[i] = params[i];
    // point-to-point messages and the aggregator (Fig. 2's IP_send_message; Pregel aggregators)
    const int np = (int)g->parts.size();
    if (pr->sends && multi_rank(g) && g->comm->world > 1)
        fail(IPREGEL_ERR_UNSUPPORTED, "ipr_send across ranks is not supported (loopback partitions are)");
    if (pr->sends && np > kProgMaxParts)
        fail(IPREGEL_ERR_UNSUPPORTED, "ipr_send supports at most %d partitions", kProgMaxParts);
    const uint64_t ident = prog_identity_bits(pr);
    // ipr_settled: one min-broadcast key pair and bound for the whole graph (partition 0's
    // buffers, written by every loopback partition; across ranks the superstep's key is
    // all-reduced with ncclMin)
    const bool settle = pr->settled;
    unsigned long long* mkey = settle ? g->parts[0].st[app].pv_mkey : nullptr;
    unsigned long long* bound = settle ? g->parts[0].st[app].pv_bound : nullptr;
    const uint32_t wmin = settle ? min_weight(g) : 1u;
    auto settle_allreduce = [&](uint32_t step) {
        if (settle && multi_rank(g))
            NC(ncclAllReduce(mkey + (step & 1u), mkey + (step & 1u), 1, ncclUint64, ncclMin,
                             g->comm->nccl, s));
    };
    const double agg_id = pr->agg_op == 0 ? 0.0 : (pr->agg_op == 1 ? INFINITY : -INFINITY);
    double agg_prev = agg_id;
    if (pr->sends || pr->agg_op >= 0) {
        const int32_t* inv = pr->sends ? inverse_ids(g) : nullptr;
        for (int a = 0; a < np; ++a) {
            Partition& p = g->parts[a];
            AppState& S = p.st[app];
            ProgShared h{};
            h.nparts = pr->sends ? np : 0;
            h.agg_op = pr->agg_op;
            for (int b = 0; b < np && pr->sends; ++b) {
                h.bounds[b] = g->parts[b].vb;
                h.bounds[b + 1] = g->parts[b].ve;
                for (int w = 0; w < 2; ++w) {
                    h.p2p[w][b] = g->parts[b].st[app].pv_p2p[w];
                    h.p2p_recv[w][b] = g->parts[b].st[app].pv_p2p_recv[w];
                }
            }
            h.inv_ids = inv;
            h.sends = S.pv_sends;
            h.agg = S.pv_agg;
            CU(cudaMemcpyAsync(S.pv_shared, &h, sizeof(h), cudaMemcpyHostToDevice, s));
            if (pr->sends && p.rows) {
                for (int w = 0; w < 2; ++w) {
                    k_fill_u64<<<grid_for(ceil_div(p.rows * (int64_t)sizeof(V), 16), 256), 256, 0, s>>>(
                        static_cast<uint64_t*>(S.pv_p2p[w]), p.rows, ident, (int)sizeof(V));
                    LAUNCH_CHECK();
                    CU(cudaMemsetAsync(S.pv_p2p_recv[w], 0, words_of(p.rows) * 4, s));
                }
            }
        }
        CU(cudaStreamSynchronize(s));   // `h` lives on the host stack
    }
    // per superstep: reset the send counters and aggregators; afterwards fold them
    auto reset_extras = [&]() {
        if (!pr->sends && pr->agg_op < 0) return;
        for (auto& p : g->parts) {
            AppState& S = p.st[app];
            CU(cudaMemsetAsync(S.pv_sends, 0, 8, s));
            CU(cudaMemcpyAsync(S.pv_agg, &agg_id, 8, cudaMemcpyHostToDevice, s));
        }
    };
    auto fold_extras = [&](uint64_t* sends_out, double* agg_out) {
        *sends_out = 0;
        *agg_out = agg_id;
        if (!pr->sends && pr->agg_op < 0) return;
        std::vector<unsigned long long> hs(np);
        std::vector<double> ha(np);
        for (int a = 0; a < np; ++a) {
            AppState& S = g->parts[a].st[app];
            CU(cudaMemcpyAsync(&hs[a], S.pv_sends, 8, cudaMemcpyDeviceToHost, s));
            CU(cudaMemcpyAsync(&ha[a], S.pv_agg, 8, cudaMemcpyDeviceToHost, s));
        }
        CU(cudaStreamSynchronize(s));
        double agg = agg_id;
        for (int a = 0; a < np; ++a) {
            *sends_out += hs[a];
            agg = pr->agg_op == 0 ? agg + ha[a] : (pr->agg_op == 1 ? std::min(agg, ha[a])
                                                                    : std::max(agg, ha[a]));
        }
        if (multi_rank(g) && pr->agg_op >= 0) {
            Partition& p = g->parts[0];
            double* d = reinterpret_cast<double*>(p.dscratch + 62);
            CU(cudaMemcpyAsync(d, &agg, 8, cudaMemcpyHostToDevice, s));
            const ncclRedOp_t op = pr->agg_op == 0 ? ncclSum : (pr->agg_op == 1 ? ncclMin : ncclMax);
            NC(ncclAllReduce(d, d + 1, 1, ncclFloat64, op, g->comm->nccl, s));
            CU(cudaMemcpyAsync(&agg, d + 1, 8, cudaMemcpyDeviceToHost, s));
            CU(cudaStreamSynchronize(s));
        }
        *agg_out = agg;
    };
    auto args_for = [&](Partition& p, uint32_t step, int cur) {
        AppState& S = p.st[app];
        ProgArgs<V> a;
        a.value = static_cast<V*>(S.pv_value);
        a.out_cur = static_cast<const V*>(S.pv_out[cur]);
        a.out_next = static_cast<V*>(S.pv_out[1 - cur]);
        a.peers = peer_slots<V>(S, 1 - cur, fused);
        a.mbox = static_cast<V*>(S.pv_mbox);
        a.flags = S.pv_flags;
        a.recv = S.pv_recv;
        a.out_off = p.csr_off;
        a.in_off = p.csc_off;
        a.ids = g->vertex_ids;
        a.params = S.pv_params;
        a.shared = (pr->sends || pr->agg_op >= 0) ? S.pv_shared : nullptr;
        a.p2p_in = pr->sends ? S.pv_p2p[(step & 1u) ^ 1u] : nullptr;
        a.p2p_in_recv = pr->sends ? S.pv_p2p_recv[(step & 1u) ^ 1u] : nullptr;
        a.aggregate = agg_prev;
        a.agg_op = pr->agg_op;
        a.pull_all = 0;
        a.vbase = p.vb;
        a.rows = p.rows;
        a.n = n;
        a.superstep = step;
        a.sym = sym ? 1 : 0;
        a.mkey_out = settle ? mkey + (step & 1u) : nullptr;
        a.bound = settle ? bound : nullptr;
        a.w_min = wmin;
        return a;
    };
    auto exchange = [&](int w) {
        if (!fused)
            exchange_owned<V>(g, [app, w](Partition& p) { return static_cast<V*>(p.st[app].pv_out[w]); });
    };

    // ---------------- superstep 0: init writes outbox buffer 0 (read by superstep 1)
    g->steps.assign(1, StepRecord{});
    StepTimer T0{g, 0};
    T0.begin();
    for (auto& p : g->parts) {
        AppState& S = p.st[app];
        CU(cudaMemcpyAsync(S.pv_params, hp, sizeof(hp), cudaMemcpyHostToDevice, s));
        CU(cudaMemsetAsync(p.pull_cnt, 0, sizeof(PullCounters), s));
        CU(cudaMemsetAsync(S.pv_recv, 0, words_of(p.rows) * 4, s));
    }
    if (settle) CU(cudaMemsetAsync(mkey, 0xFF, sizeof(unsigned long long), s));
    reset_extras();
    T0.kbegin();
    for (auto& p : g->parts) {
        ProgArgs<V> a = args_for(p, 0, 1);   // out_next = buffer 0
        PullCounters* cnt = p.pull_cnt;
        void* args[] = {&a, &cnt};
        launch_jit(pr->k[PK_INIT], std::min<unsigned>(grid_for(p.rows, 256), sm_grid(16)), 256, args, s);
    }
    T0.kend();
    exchange(0);
    settle_allreduce(0);
    unsigned long long c[4];
    reduce_counters(g, false, c, 4);
    uint64_t sends = 0;
    fold_extras(&sends, &agg_prev);
    T0.end();
    uint64_t changed = c[0], messages = c[1] + sends, active = c[3];
    g->steps[0].mode = 0;
    g->steps[0].changed = changed;
    g->steps[0].messages = messages;
    g->steps[0].model_bytes = (uint64_t)n * sizeof(V);
    int cur = 0;
    int prev_mode = 0;
    ipregel_status status = IPREGEL_OK;

    for (uint32_t step = 1; messages > 0 || active > 0; ++step) {
        if (step == max_steps) { status = IPREGEL_ERR_MAX_SUPERSTEPS; break; }
        int mode;
        if (P.mode == IPREGEL_MODE_PULL) mode = 1;
        else if (P.mode == IPREGEL_MODE_PUSH) mode = 2;
        else mode = (double)messages < (double)P.push_fraction * (double)pull_edges ? 2 : 1;
        g->steps.push_back(StepRecord{});
        StepTimer T{g, step};
        T.begin();
        const uint64_t frontier_len = changed;
        for (auto& p : g->parts) CU(cudaMemsetAsync(p.pull_cnt, 0, sizeof(PullCounters), s));
        if (settle) CU(cudaMemsetAsync(mkey + (step & 1u), 0xFF, sizeof(unsigned long long), s));
        reset_extras();
        if (mode == 2) {
            if (prev_mode == 1) {   // a pull left folded mailboxes behind: back to the identity
                for (auto& p : g->parts) {
                    if (!p.rows) continue;
                    k_fill_u64<<<grid_for(ceil_div(p.rows * (int64_t)sizeof(V), 16), 256), 256, 0, s>>>(
                        static_cast<uint64_t*>(p.st[app].pv_mbox), p.rows, ident, (int)sizeof(V));
                    LAUNCH_CHECK();
                }
            }
            // frontier = the broadcasters of superstep s-1 (flag bytes -> bitmap -> ids)
            for (auto& p : g->parts) {
                if (p.rows) {
                    k_bits_from_flags<<<grid_for(ceil_div(p.rows, 32), 256), 256, 0, s>>>(p.st[app].pv_flags,
                                                                           p.rows, p.st[app].bits);
                    LAUNCH_CHECK();
                }
                compact_bitmap(g, p, p.st[app], nullptr, sym);
            }
            if (multi) exchange_frontier(g, app, frontier_counts(g), cur);
            T.kbegin();
            for (auto& p : g->parts) {
                AppState& S = p.st[app];
                const PushAdj& adj = sym ? p.push_cc : p.push_sssp;
                build_expand_list(g, p, S, adj, S.g_id, nullptr, S.g_len, (int64_t)frontier_len);
                ProgArgs<V> a = args_for(p, step, cur);
                const unsigned grid = (unsigned)std::min<int64_t>(
                    std::max<int64_t>(ceil_div((int64_t)messages, kExpandItems), 1), sm_grid(8));
                PushAdj ad = adj;
                const int32_t* eid = S.e_id;
                const long long* epre = S.e_pre;
                const unsigned long long* len = &p.front_cnt->list_len;
                const unsigned long long* ecnt = &p.front_cnt->list_edges;
                void* eargs[] = {&ad, &eid, &epre, &len, &ecnt, &a};
                launch_jit(pr->k[PK_EXPAND], grid, kExpandThreads, eargs, s);
            }
            for (auto& p : g->parts) {
                ProgArgs<V> a = args_for(p, step, cur);
                PullCounters* cnt = p.pull_cnt;
                void* args[] = {&a, &cnt};
                launch_jit(pr->k[PK_APPLY], grid_for(ceil_div(p.rows, kProgApplyRows), 256), 256,
                           args, s);
            }
            T.kend();
        } else {
            T.kbegin();
            if (settle) {   // the bound of this pull from the previous superstep's broadcasts
                const unsigned long long* kin = mkey + ((step - 1) & 1u);
                uint32_t w = wmin;
                void* bargs[] = {&kin, &w, &bound};
                launch_jit(pr->k[PK_BOUND], 1, 32, bargs, s);
            }
            for (auto& p : g->parts) {
                if (p.rows == 0) continue;
                ProgArgs<V> a = args_for(p, step, cur);
                if (sym) {
                    launch_pull_program<V>(g, pr, 1, a, p.plan_csc, p.csc_off, p.csc_idx, p.csc_w,
                                           p.pull_cnt);
                    launch_pull_program<V>(g, pr, 2, a, p.plan_csr, p.csr_off, p.csr_idx, p.csr_w,
                                           p.pull_cnt);
                } else {
                    launch_pull_program<V>(g, pr, 0, a, p.plan_csc, p.csc_off, p.csc_idx, p.csc_w,
                                           p.pull_cnt);
                }
            }
            // every vertex computes on its folded mailbox (pull selection, reading R28)
            for (auto& p : g->parts) {
                ProgArgs<V> a = args_for(p, step, cur);
                PullCounters* cnt = p.pull_cnt;
                void* args[] = {&a, &cnt};
                launch_jit(pr->k[PK_PULL_APPLY],
                           std::min<unsigned>(grid_for(ceil_div(p.rows, kProgPullRows), 256), sm_grid(16)),
                           256, args, s);
            }
            T.kend();
        }
        exchange(1 - cur);
        settle_allreduce(step);
        reduce_counters(g, false, c, 4);
        fold_extras(&sends, &agg_prev);
        T.end();
        StepRecord& R = g->steps.back();
        R.mode = (uint8_t)mode;
        R.edges_scanned = mode == 1 ? pull_edges : messages;
        R.model_bytes = mode == 1
            ? (uint64_t)(4 + sizeof(V) + (g->parts[0].csc_w ? 4 : 0)) * pull_edges +
                  (uint64_t)(8 + 3 * sizeof(V)) * (uint64_t)n
            : (uint64_t)(8 + sizeof(V) + (g->parts[0].csc_w ? 4 : 0)) * messages +
                  (uint64_t)(16 + 3 * sizeof(V)) * (uint64_t)n;
        changed = c[0];
        messages = c[1] + sends;
        active = c[3];
        R.changed = changed;
        R.messages = messages;
        cur = 1 - cur;
        prev_mode = mode;
    }
    g->cur = cur;
    finalize_times(g);
    return status;
}

}  // namespace
