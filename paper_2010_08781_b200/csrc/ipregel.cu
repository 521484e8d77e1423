// paper_2010_08781_b200/csrc/ipregel.cu -- the C ABI (include/ipregel.h).  One translation unit:
// device kernels in pull.cuh / push.cuh / program.cuh / setup.cuh, host engine in engine.cuh
// (state, exchanges, frontier, timing), run_apps.cuh (the paper's three programs), create.cuh
// (graph handles) and run_programs.cuh (user programs through NVRTC).
//
// BSP loop (Sec. 4.2, Fig. 3): superstep 0 initialises every vertex and its
// first broadcast; superstep s >= 1 delivers the messages of s-1 (pull: CSC gather-combine;
// push: frontier expansion with atomic combine), runs the recipients' compute fused into the
// same kernels, counts broadcasters and messages on the device, exchanges owned values between
// partitions, and the host reads the counters to decide termination ("every active vertex has
// been processed and every outgoing message delivered").
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <nvrtc.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/ipregel.h"
#include "common.cuh"
#include "pull.cuh"
#include "pr_flag.cuh"
#include "push.cuh"
#include "program.cuh"
#include "setup.cuh"
#include "jit_headers.inc"

using namespace ipr;

#include "engine.cuh"
#include "pr_flag_host.cuh"
#include "run_apps.cuh"
#include "create.cuh"
#include "run_programs.cuh"

// =============================================================================================
// C ABI
// =============================================================================================
#define ABI_BEGIN try {
#define ABI_END                                                   \
    }                                                             \
    catch (const Failure& f_) {                                   \
        g_last_error = f_.msg;                                    \
        return f_.status;                                         \
    }                                                             \
    catch (const std::bad_alloc&) {                               \
        g_last_error = "host allocation failed";                  \
        return IPREGEL_ERR_OUT_OF_MEMORY;                         \
    }                                                             \
    catch (...) {                                                 \
        g_last_error = "unexpected C++ exception";                \
        return IPREGEL_ERR_CUDA;                                  \
    }

extern "C" {

const char* ipregel_status_string(ipregel_status s) {
    switch (s) {
        case IPREGEL_OK: return "IPREGEL_OK";
        case IPREGEL_ERR_INVALID_ARGUMENT: return "IPREGEL_ERR_INVALID_ARGUMENT";
        case IPREGEL_ERR_INVALID_GRAPH: return "IPREGEL_ERR_INVALID_GRAPH";
        case IPREGEL_ERR_OUT_OF_MEMORY: return "IPREGEL_ERR_OUT_OF_MEMORY";
        case IPREGEL_ERR_CUDA: return "IPREGEL_ERR_CUDA";
        case IPREGEL_ERR_NCCL: return "IPREGEL_ERR_NCCL";
        case IPREGEL_ERR_MAX_SUPERSTEPS: return "IPREGEL_ERR_MAX_SUPERSTEPS";
        case IPREGEL_ERR_STATE: return "IPREGEL_ERR_STATE";
        case IPREGEL_ERR_UNSUPPORTED: return "IPREGEL_ERR_UNSUPPORTED";
    }
    return "IPREGEL_UNKNOWN_STATUS";
}

const char* ipregel_last_error(void) { return g_last_error.c_str(); }

int ipregel_abi_version(void) { return IPREGEL_ABI_VERSION; }

uint64_t ipregel_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }

ipregel_status ipregel_device_check(int device) {
    ABI_BEGIN
    check_device(device);
    return IPREGEL_OK;
    ABI_END
}

ipregel_status ipregel_run_params_default(ipregel_run_params* out) {
    if (!out) { g_last_error = "out is NULL"; return IPREGEL_ERR_INVALID_ARGUMENT; }
    out->mode = IPREGEL_MODE_AUTO;
    out->pagerank_iterations = 10;
    out->sssp_source = 0;
    out->push_fraction = 0.04f;
    out->flags = 0;
    out->pagerank_tolerance = -1.0;
    return IPREGEL_OK;
}

ipregel_status ipregel_partition(const int64_t* cost_prefix, int64_t n, int world,
                                 int64_t* bounds_out) {
    ABI_BEGIN
    if (!cost_prefix || !bounds_out || n < 0 || world < 1)
        fail(IPREGEL_ERR_INVALID_ARGUMENT, "bad partition arguments");
    if (cost_prefix[0] != 0) fail(IPREGEL_ERR_INVALID_ARGUMENT, "cost_prefix[0] must be 0");
    for (int64_t i = 0; i < n; ++i)
        if (cost_prefix[i + 1] < cost_prefix[i])
            fail(IPREGEL_ERR_INVALID_ARGUMENT, "cost_prefix decreases at %lld", (long long)i);
    const int64_t total = cost_prefix[n];
    bounds_out[0] = 0;
    for (int r = 1; r < world; ++r) {
        // first vertex whose prefix reaches the r-th equal share (lower bound)
        const long double target = (long double)total * r / world;
        int64_t lo = bounds_out[r - 1], hi = n;
        while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            if ((long double)cost_prefix[mid] < target) lo = mid + 1; else hi = mid;
        }
        bounds_out[r] = lo;
    }
    bounds_out[world] = n;
    return IPREGEL_OK;
    ABI_END
}

ipregel_status ipregel_nccl_unique_id(uint8_t out[128]) {
    ABI_BEGIN
    if (!out) fail(IPREGEL_ERR_INVALID_ARGUMENT, "out is NULL");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    NC(ncclGetUniqueId(&id));
    memcpy(out, &id, 128);
    return IPREGEL_OK;
    ABI_END
}

ipregel_status ipregel_comm_create(int rank, int world, const uint8_t id[128], int device,
                                   ipregel_comm** out) {
    ABI_BEGIN
    if (!out || !id || world < 1 || rank < 0 || rank >= world)
        fail(IPREGEL_ERR_INVALID_ARGUMENT, "bad comm arguments");
    *out = nullptr;
    CU(cudaSetDevice(device));
    check_device(device);
    ncclUniqueId uid;
    memcpy(&uid, id, 128);
    ipregel_comm* c = new ipregel_comm;
    c->rank = rank;
    c->world = world;
    c->device = device;
    ncclResult_t r = ncclCommInitRank(&c->nccl, world, uid, rank);
    if (r != ncclSuccess) {
        delete c;
        fail(IPREGEL_ERR_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
    }
    *out = c;
    return IPREGEL_OK;
    ABI_END
}

void ipregel_comm_destroy(ipregel_comm* comm) {
    if (!comm) return;
    if (comm->nccl) ncclCommDestroy(comm->nccl);
    delete comm;
}

static ipregel_status create_common(const ipregel_graph_desc* descs, int np, ipregel_comm* comm,
                                    void* stream, ipregel_graph** out) {
    ABI_BEGIN
    const auto t_entry = std::chrono::steady_clock::now();
    if (!out) fail(IPREGEL_ERR_INVALID_ARGUMENT, "out is NULL");
    *out = nullptr;
    if (!descs || np < 1) fail(IPREGEL_ERR_INVALID_ARGUMENT, "no partition descriptors");
    int64_t n = 0;
    for (int i = 0; i < np; ++i) {
        int64_t ni;
        validate_desc(&descs[i], &ni);
        if (i == 0) n = ni;
        else if (ni != n || descs[i].num_edges != descs[0].num_edges)
            fail(IPREGEL_ERR_INVALID_ARGUMENT, "partitions disagree on N or E");
    }
    if (!comm || comm->world == 1) {
        int64_t expect = 0;
        for (int i = 0; i < np; ++i) {
            if (descs[i].vertex_begin != expect)
                fail(IPREGEL_ERR_INVALID_ARGUMENT, "partition %d starts at %lld, expected %lld", i,
                     (long long)descs[i].vertex_begin, (long long)expect);
            expect = descs[i].vertex_end;
        }
        if (expect != n) fail(IPREGEL_ERR_INVALID_ARGUMENT, "partitions do not cover [0, N)");
    }
    int device = 0;
    CU(cudaGetDevice(&device));
    check_device(device);
    configure_pool(device);
    ipregel_graph* g = new ipregel_graph;
    g->n = n;
    g->e = descs[0].num_edges;
    g->device = device;
    g->stream = static_cast<cudaStream_t>(stream);
    g->comm = comm;
    g->parts.resize(np);
    try {
        int64_t csc_base = 0, csr_base = 0;
        for (int i = 0; i < np; ++i) {
            g->parts[i].csc_ebase = csc_base;
            g->parts[i].csr_ebase = csr_base;
            csc_base += descs[i].csc_edges;
            csr_base += descs[i].csr_edges;
        }
        if (comm) {
            // every rank's (vb, rows, csc_edges, csr_edges) -> ranges and global edge bases
            int64_t mine[4] = {descs[0].vertex_begin, descs[0].vertex_end - descs[0].vertex_begin,
                               descs[0].csc_edges, descs[0].csr_edges};
            int64_t* dmine = nullptr;
            int64_t* dall = nullptr;
            CU(cudaMalloc(&dmine, 4 * sizeof(int64_t)));
            CU(cudaMalloc(&dall, 4 * sizeof(int64_t) * comm->world));
            CU(cudaMemcpyAsync(dmine, mine, sizeof(mine), cudaMemcpyHostToDevice, g->stream));
            NC(ncclAllGather(dmine, dall, 4, ncclInt64, comm->nccl, g->stream));
            std::vector<int64_t> all(4 * comm->world);
            CU(cudaMemcpyAsync(all.data(), dall, all.size() * sizeof(int64_t),
                               cudaMemcpyDeviceToHost, g->stream));
            CU(cudaStreamSynchronize(g->stream));
            cudaFree(dmine);
            cudaFree(dall);
            int64_t expect = 0, cb = 0, rb = 0;
            for (int r = 0; r < comm->world; ++r) {
                if (all[4 * r] != expect)
                    fail(IPREGEL_ERR_INVALID_ARGUMENT, "rank ranges do not tile [0, N)");
                g->rank_vb.push_back(all[4 * r]);
                g->rank_rows.push_back(all[4 * r + 1]);
                if (r == comm->rank) {
                    g->parts[0].csc_ebase = cb;
                    g->parts[0].csr_ebase = rb;
                }
                expect += all[4 * r + 1];
                cb += all[4 * r + 2];
                rb += all[4 * r + 3];
            }
            if (expect != n) fail(IPREGEL_ERR_INVALID_ARGUMENT, "rank ranges do not cover [0, N)");
        }
        for (int i = 0; i < np; ++i) {
            if ((descs[i].vertex_ids == nullptr) != (descs[0].vertex_ids == nullptr) ||
                descs[i].degree_ordered != descs[0].degree_ordered)
                fail(IPREGEL_ERR_INVALID_ARGUMENT, "partitions disagree on the vertex layout");
        }
        g->degree_ordered = descs[0].degree_ordered != 0;
        g->gather_policy = g_gather_policy >= 0 ? g_gather_policy : (g->degree_ordered ? 3 : 1);
        if (g_ctrace.on)
            fprintf(stderr, "[ipregel create] host entry -> begin    %9.2f ms\n",
                    std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() -
                                                              t_entry).count());
        g_ctrace.mark("create begin", g->stream);
        if (descs[0].vertex_ids) {
            if (descs[0].memory == IPREGEL_MEMORY_HOST) {
                int32_t* d = g->graph_mem.alloc<int32_t>(n, g->stream);
                CU(cudaMemcpyAsync(d, descs[0].vertex_ids, n * 4, cudaMemcpyHostToDevice, g->stream));
                g->vertex_ids = d;
            } else {
                g->vertex_ids = descs[0].vertex_ids;
            }
            if (descs[0].validate) {
                DeviceBuffers tmp;
                int32_t* seen = tmp.alloc<int32_t>(n, g->stream, true);
                unsigned* flags = tmp.alloc<unsigned>(1, g->stream, true);
                k_count_ids<<<grid_for(n, 256), 256, 0, g->stream>>>(g->vertex_ids, n, seen, flags);
                LAUNCH_CHECK();
                unsigned h = 0;
                CU(cudaMemcpyAsync(&h, flags, 4, cudaMemcpyDeviceToHost, g->stream));
                CU(cudaStreamSynchronize(g->stream));
                tmp.release();
                if (h) fail(IPREGEL_ERR_INVALID_GRAPH, "vertex_ids is not a permutation of [0, N)");
            }
        }
        for (int i = 0; i < np; ++i) init_partition(g, g->parts[i], descs[i]);
        build_plans(g);
        g_ctrace.mark("plans built", g->stream);
        for (auto& p : g->parts) launch_relabel_csr(g, p);
        // a graph the library relabelled (IPREGEL_LAYOUT_DEGREE) gets PageRank's flagged plan
        // here, on the run stream while the CSR sorts on the aux stream: its allocations then
        // come in the same order every time (a create / run / destroy loop keeps a settled
        // device pool; built lazily in the first run they met the CSR sort's asynchronous frees
        // in varying order, and some end-to-end steps paid for pool growth: 650-1040 vs 483 ms)
        for (auto& p : g->parts)
            if (p.csr_pending && p.rows > 0 && g_pr_flag && g_pr_split) ensure_flag_plan(g, p);
        for (auto& p : g->parts) finish_uploads(g, p);
        CU(cudaStreamSynchronize(g->stream));
        g_ctrace.mark("create end", g->stream);
        g_ctrace.dump();
    } catch (...) {
        destroy_graph(g);
        throw;
    }
    *out = g;
    return IPREGEL_OK;
    ABI_END
}

ipregel_status ipregel_graph_create(const ipregel_graph_desc* desc, ipregel_comm* comm,
                                    void* stream, ipregel_graph** out) {
    return create_common(desc, 1, comm, stream, out);
}

ipregel_status ipregel_graph_create_partitioned(const ipregel_graph_desc* descs,
                                                int num_partitions, void* stream,
                                                ipregel_graph** out) {
    return create_common(descs, num_partitions, nullptr, stream, out);
}

void ipregel_graph_destroy(ipregel_graph* graph) { destroy_graph(graph); }

ipregel_status ipregel_memory_footprint(ipregel_graph* g, uint64_t* graph_bytes,
                                        uint64_t* state_bytes) {
    ABI_BEGIN
    if (!g) fail(IPREGEL_ERR_INVALID_ARGUMENT, "graph is NULL");
    uint64_t gb = 0, sb = 0;
    for (auto& p : g->parts) {
        gb += p.graph_mem.bytes;
        for (auto& S : p.st) sb += S.mem.bytes;
    }
    if (graph_bytes) *graph_bytes = gb;
    if (state_bytes) *state_bytes = sb;
    return IPREGEL_OK;
    ABI_END
}

ipregel_status ipregel_run(ipregel_graph* g, ipregel_app app, ipregel_combiner combiner,
                           uint32_t max_supersteps, const ipregel_run_params* params) {
    ABI_BEGIN
    if (!g) fail(IPREGEL_ERR_INVALID_ARGUMENT, "graph is NULL");
    if (g->poisoned) fail(IPREGEL_ERR_STATE, "graph handle was poisoned by an earlier failure");
    ipregel_run_params P;
    ipregel_run_params_default(&P);
    if (params) P = *params;
    if (app < IPREGEL_APP_PAGERANK || app > IPREGEL_APP_SSSP)
        fail(IPREGEL_ERR_INVALID_ARGUMENT, "unknown app %d", (int)app);
    const ipregel_combiner want =
        app == IPREGEL_APP_PAGERANK ? IPREGEL_COMBINE_SUM : IPREGEL_COMBINE_MIN;
    if (combiner != want)
        fail(IPREGEL_ERR_INVALID_ARGUMENT,
             "combiner %d does not match the app (PageRank sums, Fig. 8; CC/SSSP take the min, "
             "Fig. 5)", (int)combiner);
    if (max_supersteps == 0) fail(IPREGEL_ERR_INVALID_ARGUMENT, "max_supersteps must be >= 1");
    if (P.mode < IPREGEL_MODE_AUTO || P.mode > IPREGEL_MODE_PUSH)
        fail(IPREGEL_ERR_INVALID_ARGUMENT, "unknown mode %d", P.mode);
    if (P.flags & ~(uint32_t)(IPREGEL_RUN_EXCHANGE_COLLECTIVE | IPREGEL_RUN_EXCHANGE_FUSED |
                              IPREGEL_RUN_PAGERANK_MASS))
        fail(IPREGEL_ERR_INVALID_ARGUMENT, "unknown flags 0x%x", P.flags);
    if ((P.flags & IPREGEL_RUN_EXCHANGE_COLLECTIVE) && (P.flags & IPREGEL_RUN_EXCHANGE_FUSED))
        fail(IPREGEL_ERR_INVALID_ARGUMENT, "EXCHANGE_COLLECTIVE and EXCHANGE_FUSED are exclusive");
    if ((P.flags & IPREGEL_RUN_PAGERANK_MASS) && app != IPREGEL_APP_PAGERANK)
        fail(IPREGEL_ERR_INVALID_ARGUMENT, "IPREGEL_RUN_PAGERANK_MASS is for PageRank only");
    if (app == IPREGEL_APP_SSSP && (int64_t)P.sssp_source >= g->n)
        fail(IPREGEL_ERR_INVALID_ARGUMENT, "sssp_source %u >= N", P.sssp_source);
    if (!(P.push_fraction >= 0.0f)) fail(IPREGEL_ERR_INVALID_ARGUMENT, "push_fraction < 0");
    if (P.pagerank_tolerance != P.pagerank_tolerance)
        fail(IPREGEL_ERR_INVALID_ARGUMENT, "pagerank_tolerance is NaN");
    if (app == IPREGEL_APP_SSSP && g->parts[0].csc_w == nullptr) {
        // unit weights (Fig. 10) -- fine
    }
    g->last_status = -1;
    g->last_app = -1;
    ipregel_status st;
    const cudaStream_t caller_stream = g->stream;
    try {
        ensure_state(g, app);
        st = app == IPREGEL_APP_PAGERANK ? run_pagerank(g, max_supersteps, P)
                                         : run_min(g, app, max_supersteps, P);
    } catch (const Failure& f) {
        // a failure inside a CUDA-graph capture: close the capture, back to the caller's stream
        if (g->capture_stream) {
            cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
            if (cudaStreamIsCapturing(g->capture_stream, &cs) == cudaSuccess &&
                cs != cudaStreamCaptureStatusNone) {
                cudaGraph_t gr = nullptr;
                cudaStreamEndCapture(g->capture_stream, &gr);
                if (gr) cudaGraphDestroy(gr);
            }
            cudaGetLastError();
        }
        g->stream = caller_stream;
        if (f.status == IPREGEL_ERR_CUDA || f.status == IPREGEL_ERR_NCCL) g->poisoned = true;
        throw;
    }
    g->last_app = app;
    g->last_vsz = app == IPREGEL_APP_PAGERANK ? 8 : 4;
    g->last_status = st;
    if (st != IPREGEL_OK) g_last_error = "superstep guard reached with work remaining";
    return st;
    ABI_END
}

ipregel_status ipregel_program_create(const ipregel_program_desc* desc, ipregel_program** out) {
    ABI_BEGIN
    if (!out) fail(IPREGEL_ERR_INVALID_ARGUMENT, "out is NULL");
    *out = nullptr;
    if (!desc || !desc->source) fail(IPREGEL_ERR_INVALID_ARGUMENT, "desc or source is NULL");
    if (desc->value_type < IPREGEL_VALUE_U32 || desc->value_type > IPREGEL_VALUE_I64)
        fail(IPREGEL_ERR_INVALID_ARGUMENT, "unknown value_type %d", desc->value_type);
    if (desc->combiner < IPREGEL_COMBINE_SUM || desc->combiner > IPREGEL_COMBINE_MAX)
        fail(IPREGEL_ERR_INVALID_ARGUMENT, "unknown combiner %d", desc->combiner);
    if (desc->symmetric != 0 && desc->symmetric != 1)
        fail(IPREGEL_ERR_INVALID_ARGUMENT, "symmetric must be 0 or 1");
    if (desc->reserved != 0) fail(IPREGEL_ERR_INVALID_ARGUMENT, "reserved must be 0");
    if (desc->aggregator < IPREGEL_AGG_NONE || desc->aggregator > IPREGEL_AGG_MAX)
        fail(IPREGEL_ERR_INVALID_ARGUMENT, "unknown aggregator %d", desc->aggregator);
    ipregel_program* pr = new ipregel_program;
    pr->value_type = desc->value_type;
    pr->combiner = desc->combiner;
    pr->sym = desc->symmetric;
    pr->agg_op = desc->aggregator - 1;   // -1 none, else SUM / MIN / MAX
    pr->sends = strstr(desc->source, "ipr_send") != nullptr;
    pr->settled = strstr(desc->source, "ipr_settled") != nullptr &&
                  desc->combiner == IPREGEL_COMBINE_MIN && !pr->sends;
    try {
        compile_program(pr, *desc);
    } catch (...) {
        delete pr;
        throw;
    }
    *out = pr;
    return IPREGEL_OK;
    ABI_END
}

const char* ipregel_program_log(const ipregel_program* program) {
    return program ? program->log.c_str() : "";
}

uint64_t ipregel_program_cubin_bytes(const ipregel_program* program) {
    return program ? (uint64_t)program->cubin.size() : 0;
}

void ipregel_program_destroy(ipregel_program* program) {
    if (!program) return;
    if (program->lib) cudaLibraryUnload(program->lib);
    delete program;
}

ipregel_status ipregel_run_program(ipregel_graph* g, ipregel_program* program,
                                   uint32_t max_supersteps, const ipregel_run_params* params,
                                   const double* program_params, int num_program_params) {
    ABI_BEGIN
    if (!g || !program) fail(IPREGEL_ERR_INVALID_ARGUMENT, "graph or program is NULL");
    if (g->poisoned) fail(IPREGEL_ERR_STATE, "graph handle was poisoned by an earlier failure");
    if (max_supersteps == 0) fail(IPREGEL_ERR_INVALID_ARGUMENT, "max_supersteps must be >= 1");
    if (num_program_params < 0 || num_program_params > kProgParams ||
        (num_program_params > 0 && !program_params))
        fail(IPREGEL_ERR_INVALID_ARGUMENT, "program parameters: 0..%d values", kProgParams);
    ipregel_run_params P;
    ipregel_run_params_default(&P);
    if (params) P = *params;
    if (P.mode < IPREGEL_MODE_AUTO || P.mode > IPREGEL_MODE_PUSH)
        fail(IPREGEL_ERR_INVALID_ARGUMENT, "unknown mode %d", P.mode);
    if (P.flags & ~(uint32_t)(IPREGEL_RUN_EXCHANGE_COLLECTIVE | IPREGEL_RUN_EXCHANGE_FUSED))
        fail(IPREGEL_ERR_INVALID_ARGUMENT, "unknown flags 0x%x", P.flags);
    if ((P.flags & IPREGEL_RUN_EXCHANGE_COLLECTIVE) && (P.flags & IPREGEL_RUN_EXCHANGE_FUSED))
        fail(IPREGEL_ERR_INVALID_ARGUMENT, "EXCHANGE_COLLECTIVE and EXCHANGE_FUSED are exclusive");
    if (!(P.push_fraction >= 0.0f)) fail(IPREGEL_ERR_INVALID_ARGUMENT, "push_fraction < 0");
    g->last_status = -1;
    g->last_app = -1;
    ipregel_status st;
    try {
        ensure_state(g, kAppProgram);
        switch (program->value_type) {
            case IPREGEL_VALUE_F64:
                st = run_program_t<double>(g, program, max_supersteps, P, program_params,
                                           num_program_params);
                break;
            case IPREGEL_VALUE_F32:
                st = run_program_t<float>(g, program, max_supersteps, P, program_params,
                                          num_program_params);
                break;
            case IPREGEL_VALUE_I32:
                st = run_program_t<int32_t>(g, program, max_supersteps, P, program_params,
                                            num_program_params);
                break;
            case IPREGEL_VALUE_U64:
                st = run_program_t<uint64_t>(g, program, max_supersteps, P, program_params,
                                             num_program_params);
                break;
            case IPREGEL_VALUE_I64:
                st = run_program_t<int64_t>(g, program, max_supersteps, P, program_params,
                                            num_program_params);
                break;
            default:
                st = run_program_t<uint32_t>(g, program, max_supersteps, P, program_params,
                                             num_program_params);
        }
    } catch (const Failure& f) {
        if (f.status == IPREGEL_ERR_CUDA || f.status == IPREGEL_ERR_NCCL) g->poisoned = true;
        throw;
    }
    g->last_app = kAppProgram;
    g->last_vsz = (int)value_bytes(program->value_type);
    g->last_status = st;
    if (st != IPREGEL_OK) g_last_error = "superstep guard reached with work remaining";
    return st;
    ABI_END
}

ipregel_status ipregel_get_values_async(ipregel_graph* g, void* out, size_t out_bytes) {
    ABI_BEGIN
    if (!g || !out) fail(IPREGEL_ERR_INVALID_ARGUMENT, "graph or out is NULL");
    if (g->poisoned) fail(IPREGEL_ERR_STATE, "graph handle was poisoned");
    if (g->last_app < 0) fail(IPREGEL_ERR_STATE, "no completed run");
    if (multi_rank(g)) fail(IPREGEL_ERR_UNSUPPORTED, "ipregel_get_values_async across ranks");
    const bool owned = g->last_app == IPREGEL_APP_PAGERANK || g->last_app == kAppProgram;
    const size_t esz = (size_t)g->last_vsz;
    if (out_bytes != (size_t)g->n * esz)
        fail(IPREGEL_ERR_INVALID_ARGUMENT, "out_bytes %zu != N * %zu", out_bytes, esz);
    cudaStream_t s = g->stream;
    try {
        if (!g->copy_stream) CU(cudaStreamCreateWithFlags(&g->copy_stream, cudaStreamNonBlocking));
        // a private staging vector in original order, built by kernels on the run stream (no
        // copy-engine work there: see compute_fence), then a device -> host copy on the copy
        // stream, after which the staging buffer goes back to the pool
        uint8_t* stage = nullptr;
        CU(cudaMallocAsync(reinterpret_cast<void**>(&stage), (size_t)g->n * esz, s));
        uint8_t* full = stage;
        if (g->vertex_ids) {
            if (!g->gather_tmp) g->gather_tmp = g->graph_mem.alloc<double>(g->n, s);
            full = reinterpret_cast<uint8_t*>(g->gather_tmp);
        }
        for (auto& p : g->parts) {
            const void* src = owned ? (g->last_app == IPREGEL_APP_PAGERANK
                                           ? (const void*)p.st[0].rank
                                           : p.st[kAppProgram].pv_value)
                                    : (const void*)(reinterpret_cast<const uint8_t*>(
                                           p.st[g->last_app].val[g->cur]) + p.vb * esz);
            if (p.rows) kernel_copy(full + p.vb * esz, src, p.rows * esz, s);
        }
        if (g->vertex_ids) {
            if (esz == 8)
                k_to_original<double><<<grid_for(g->n, 256), 256, 0, s>>>(
                    (const double*)full, g->vertex_ids, g->n, (double*)stage);
            else
                k_to_original<uint32_t><<<grid_for(g->n, 256), 256, 0, s>>>(
                    (const uint32_t*)full, g->vertex_ids, g->n, (uint32_t*)stage);
            LAUNCH_CHECK();
        }
        cudaEvent_t ready;
        CU(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
        CU(cudaEventRecord(ready, s));
        compute_fence(g->copy_stream);   // its latest op may be a copy (see compute_fence)
        CU(cudaStreamWaitEvent(g->copy_stream, ready, 0));
        CU(cudaEventDestroy(ready));     // released once the wait has been recorded
        CU(cudaMemcpyAsync(out, stage, (size_t)g->n * esz, cudaMemcpyDeviceToHost, g->copy_stream));
        CU(cudaFreeAsync(stage, g->copy_stream));
    } catch (const Failure& f) {
        if (f.status == IPREGEL_ERR_CUDA || f.status == IPREGEL_ERR_NCCL) g->poisoned = true;
        throw;
    }
    return IPREGEL_OK;
    ABI_END
}

ipregel_status ipregel_graph_sync(ipregel_graph* g) {
    ABI_BEGIN
    if (!g) fail(IPREGEL_ERR_INVALID_ARGUMENT, "graph is NULL");
    if (g->copy_stream) CU(cudaStreamSynchronize(g->copy_stream));
    CU(cudaStreamSynchronize(g->stream));
    return IPREGEL_OK;
    ABI_END
}

ipregel_status ipregel_get_values(ipregel_graph* g, void* out, size_t out_bytes,
                                  int out_is_device) {
    ABI_BEGIN
    if (!g || !out) fail(IPREGEL_ERR_INVALID_ARGUMENT, "graph or out is NULL");
    if (g->poisoned) fail(IPREGEL_ERR_STATE, "graph handle was poisoned");
    if (g->last_app < 0) fail(IPREGEL_ERR_STATE, "no completed run");
    // owned value arrays (PageRank ranks, program values) are assembled into a full vector;
    // CC/SSSP values are already full replicas
    const bool owned = g->last_app == IPREGEL_APP_PAGERANK || g->last_app == kAppProgram;
    const size_t esz = (size_t)g->last_vsz;
    if (out_bytes != (size_t)g->n * esz)
        fail(IPREGEL_ERR_INVALID_ARGUMENT, "out_bytes %zu != N * %zu", out_bytes, esz);
    cudaStream_t s = g->stream;
    const cudaMemcpyKind kind = out_is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    try {
        // full N-vector in internal order (device)
        const void* full = nullptr;
        if (owned) {
            if (!g->gather_tmp) g->gather_tmp = g->graph_mem.alloc<double>(g->n, s);
            uint8_t* base = reinterpret_cast<uint8_t*>(g->gather_tmp);
            for (auto& p : g->parts) {
                const void* src = g->last_app == IPREGEL_APP_PAGERANK ? (const void*)p.st[0].rank
                                                                      : p.st[kAppProgram].pv_value;
                if (p.rows)
                    CU(cudaMemcpyAsync(base + p.vb * esz, src, p.rows * esz,
                                       cudaMemcpyDeviceToDevice, s));
            }
            if (multi_rank(g)) {
                NC(ncclGroupStart());
                for (int r = 0; r < g->comm->world; ++r)
                    if (g->rank_rows[r])
                        NC(ncclBroadcast(base + g->rank_vb[r] * esz, base + g->rank_vb[r] * esz,
                                         (size_t)g->rank_rows[r] * esz, ncclUint8, r,
                                         g->comm->nccl, s));
                NC(ncclGroupEnd());
            }
            full = g->gather_tmp;
        } else {
            full = g->parts[0].st[g->last_app].val[g->cur];
        }
        if (g->vertex_ids) {
            if (!g->gather_tmp2) g->gather_tmp2 = g->graph_mem.alloc<double>(g->n, s);
            if (esz == 8)
                k_to_original<double><<<grid_for(g->n, 256), 256, 0, s>>>(
                    (const double*)full, g->vertex_ids, g->n, g->gather_tmp2);
            else
                k_to_original<uint32_t><<<grid_for(g->n, 256), 256, 0, s>>>(
                    (const uint32_t*)full, g->vertex_ids, g->n, (uint32_t*)g->gather_tmp2);
            LAUNCH_CHECK();
            full = g->gather_tmp2;
        }
        CU(cudaMemcpyAsync(out, full, g->n * esz, kind, s));
        CU(cudaStreamSynchronize(s));
    } catch (const Failure& f) {
        if (f.status == IPREGEL_ERR_CUDA || f.status == IPREGEL_ERR_NCCL) g->poisoned = true;
        throw;
    }
    return IPREGEL_OK;
    ABI_END
}

ipregel_status ipregel_get_stats(ipregel_graph* g, ipregel_stats* st) {
    ABI_BEGIN
    if (!g || !st) fail(IPREGEL_ERR_INVALID_ARGUMENT, "graph or stats is NULL");
    st->supersteps = (uint32_t)g->steps.size();
    st->status = g->last_status;
    st->exchange = g->last_exchange;
    const size_t m = std::min<size_t>(st->capacity, g->steps.size());
    for (size_t i = 0; i < m; ++i) {
        const StepRecord& R = g->steps[i];
        if (st->time_ms) st->time_ms[i] = R.time_ms;
        if (st->kernel_ms) st->kernel_ms[i] = R.kernel_ms;
        if (st->mode) st->mode[i] = R.mode;
        if (st->changed) st->changed[i] = R.changed;
        if (st->messages) st->messages[i] = R.messages;
        if (st->edges_scanned) st->edges_scanned[i] = R.edges_scanned;
        if (st->model_bytes) st->model_bytes[i] = R.model_bytes;
        if (st->pagerank_delta) st->pagerank_delta[i] = R.delta;
        if (st->pagerank_mass) st->pagerank_mass[i] = R.mass[0];
        if (st->pagerank_mass_nd) st->pagerank_mass_nd[i] = R.mass[1];
        if (st->part_ms) st->part_ms[i] = R.part_ms;
    }
    return IPREGEL_OK;
    ABI_END
}

}  // extern "C"
