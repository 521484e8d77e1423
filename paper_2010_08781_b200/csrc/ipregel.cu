// paper_2010_08781_b200/csrc/ipregel.cu -- the C ABI (include/ipregel.h) and the host superstep
// driver.  One translation unit; kernels live in pull.cuh / push.cuh / setup.cuh.
//
// BSP loop (Sec. 4.2, Fig. 3): superstep 0 initialises every vertex and its
// first broadcast; superstep s >= 1 delivers the messages of s-1 (pull: CSC gather-combine;
// push: frontier expansion with atomic combine), runs the recipients' compute fused into the
// same kernels, counts broadcasters and messages on the device, exchanges owned values between
// partitions, and the host reads the counters to decide termination ("every active vertex has
// been processed and every outgoing message delivered").
#include <cub/device/device_radix_sort.cuh>
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
#include "push.cuh"
#include "program.cuh"
#include "setup.cuh"
#include "jit_headers.inc"

using namespace ipr;

// =============================================================================================
// errors
// =============================================================================================
namespace {

thread_local std::string g_last_error;

struct Failure {
    ipregel_status status;
    std::string msg;
};

[[noreturn]] void fail(ipregel_status s, const char* fmt, ...) {
    char buf[640];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    throw Failure{s, buf};
}

#define CU(call)                                                                              \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess) {                                                              \
            ipregel_status st_ = e_ == cudaErrorMemoryAllocation ? IPREGEL_ERR_OUT_OF_MEMORY  \
                                                                 : IPREGEL_ERR_CUDA;          \
            fail(st_, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__);   \
        }                                                                                     \
    } while (0)

#define NC(call)                                                                              \
    do {                                                                                      \
        ncclResult_t r_ = (call);                                                             \
        if (r_ != ncclSuccess)                                                                \
            fail(IPREGEL_ERR_NCCL, "%s: %s (%s:%d)", #call, ncclGetErrorString(r_), __FILE__, \
                 __LINE__);                                                                   \
    } while (0)

std::atomic<unsigned long long> g_launches{0};
#define LAUNCH_CHECK()                                   \
    do {                                                 \
        g_launches.fetch_add(1, std::memory_order_relaxed); \
        CU(cudaGetLastError());                          \
    } while (0)

// Tuning knob read once per process: L2 policy of the pull gathers (-1 = per graph: range policy
// for degree-ordered layouts, else evict_last).
int read_gather_policy() {
    const char* e = getenv("IPREGEL_GATHER_POLICY");
    return e ? atoi(e) : -1;
}
int g_gather_policy = read_gather_policy();
// Hot-prefix bytes kept evict-last under policy 3 (IPREGEL_HOT_BYTES, default 64 MiB).
uint64_t read_hot_bytes() {
    const char* e = getenv("IPREGEL_HOT_BYTES");
    return e ? strtoull(e, nullptr, 10) : (64ull << 20);
}
uint64_t g_hot_bytes = read_hot_bytes();
// Tuning knobs: L1-cached hot vertices (IPREGEL_L1_HOT, -1 = default L1 policy) and an L2
// persisting access-policy window over the hot prefix (IPREGEL_PERSIST_BYTES, 0 = off).
// -1 (default): 64 KiB worth of the hottest vertices for degree-ordered layouts, else off.
int32_t g_l1_hot = getenv("IPREGEL_L1_HOT") ? atoi(getenv("IPREGEL_L1_HOT")) : -2;
// Tuning knob: PageRank update split out of the range kernel (IPREGEL_PR_SPLIT=1).
int g_pr_split = getenv("IPREGEL_PR_SPLIT") ? atoi(getenv("IPREGEL_PR_SPLIT")) : 1;
// Hash-Min row-list pull when the rows not yet at label 0 hold fewer than this fraction of the
// symmetrised edges (IPREGEL_ROWLIST; 0 = never).
double g_rowlist = getenv("IPREGEL_ROWLIST") ? atof(getenv("IPREGEL_ROWLIST")) : 0.05;
uint64_t g_persist_bytes =
    getenv("IPREGEL_PERSIST_BYTES") ? strtoull(getenv("IPREGEL_PERSIST_BYTES"), nullptr, 10) : 0;

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline uint32_t sat_add_host(uint32_t a, uint32_t b) {
    const uint64_t s = (uint64_t)a + b;
    return s >= 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)s;
}
inline unsigned grid_for(int64_t n, int threads) {
    int64_t g = ceil_div(std::max<int64_t>(n, 1), threads);
    return (unsigned)std::min<int64_t>(g, 0x7FFFFFFF);
}

}  // namespace

// =============================================================================================
// handles
// =============================================================================================
struct ipregel_comm {
    ncclComm_t nccl = nullptr;
    int rank = 0, world = 1, device = 0;
};

namespace {

// Device memory comes from the device's stream-ordered pool (cudaMallocAsync), which keeps up to
// IPREGEL_POOL_RETAIN_BYTES (default 96 GiB) of freed memory for the next graph instead of
// returning it to the driver: creating and destroying a graph handle per job stays cheap (a
// plain cudaMalloc/cudaFree of the 7.5 GB adjacency copies costs ~100 ms each).  Buffers another
// process maps with CUDA IPC (fused-exchange replicas of a rank) use cudaMalloc.
void configure_pool(int device) {
    static bool done[64] = {};
    if (device < 0 || device >= 64 || done[device]) return;
    done[device] = true;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    const char* e = getenv("IPREGEL_POOL_RETAIN_BYTES");
    uint64_t keep = e ? strtoull(e, nullptr, 10) : (96ull << 30);
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
}

struct DeviceBuffers {
    struct Block {
        void* p;
        cudaStream_t s;   // pooled: freed on this stream; nullptr with ipc = cudaFree
        bool ipc;
    };
    std::vector<Block> blocks;
    uint64_t bytes = 0;
    template <class T>
    T* alloc(int64_t count, cudaStream_t s, bool zero = false, bool ipc = false) {
        void* p = nullptr;
        size_t b = (size_t)std::max<int64_t>(count, 1) * sizeof(T);
        if (ipc) CU(cudaMalloc(&p, b));
        else CU(cudaMallocAsync(&p, b, s));
        blocks.push_back(Block{p, s, ipc});
        bytes += b;
        if (zero) CU(cudaMemsetAsync(p, 0, b, s));
        return static_cast<T*>(p);
    }
    void release() {
        for (const Block& k : blocks) {
            if (k.ipc) cudaFree(k.p);
            else cudaFreeAsync(k.p, k.s);
        }
        blocks.clear();
        bytes = 0;
    }
};

// Vertex state of one app on one partition: Theta(N), never a function of E
// (single-slot mailboxes).
struct AppState {
    bool ready = false;
    double* rank = nullptr;                    // PageRank: owned ranks
    double* contrib[2] = {nullptr, nullptr};   // PageRank outbox replicas [N] (s / s+1)
    double* acc = nullptr;                     // PageRank push accumulator (owned)
    uint32_t* val[2] = {nullptr, nullptr};     // CC/SSSP value replicas [N] (current / next)
    uint32_t* bits = nullptr;                  // owned bitmap of broadcasters
    int32_t* f_id = nullptr;                   // owned frontier (ascending ids) + snapshots
    uint32_t* f_val = nullptr;
    int32_t* g_id = nullptr;                   // global frontier (== f_* on one partition)
    uint32_t* g_val = nullptr;
    unsigned long long* g_len = nullptr;       // device scalar
    int32_t* e_id = nullptr;                   // expand list: push-view degree > 0
    uint32_t* e_val = nullptr;
    long long* e_pre = nullptr;
    unsigned long long* blk_a = nullptr;       // scan scratch
    unsigned long long* blk_b = nullptr;
    int32_t* iota = nullptr;                   // PageRank push: every vertex as a source
    unsigned long long* iota_len = nullptr;
    // Fused exchange: the OTHER replicas of buffer w of the broadcast array
    // (contrib[w] or val[w]) that receive this partition's owned slice from the pull epilogue.
    // Loopback: the other partitions' buffers.  Ranks: peers' buffers mapped with CUDA IPC.
    void* peer[2][kMaxPeers] = {};
    int npeer = 0;
    int peers_state = 0;                       // 0 not set up, 1 reachable, -1 not reachable
    std::vector<void*> ipc_opened;
    // user vertex programs (app slot kAppProgram): 8-byte slots hold u32 or f64 values
    void* pv_value = nullptr;                  // owned values [rows]
    void* pv_out[2] = {nullptr, nullptr};      // outbox replicas [N] (identity = no broadcast)
    void* pv_mbox = nullptr;                   // owned mailboxes [rows]
    uint8_t* pv_flags = nullptr;               // owned: bit 0 broadcast, bit 1 active
    uint32_t* pv_recv = nullptr;               // owned recipient bitmap (push)
    double* pv_params = nullptr;               // program parameters [8]
    void* pv_p2p[2] = {nullptr, nullptr};      // point-to-point mailboxes [rows] (by parity)
    uint32_t* pv_p2p_recv[2] = {nullptr, nullptr};
    ProgShared* pv_shared = nullptr;           // device copy of the run's ProgShared
    unsigned long long* pv_sends = nullptr;    // point-to-point sends of the superstep
    double* pv_agg = nullptr;                  // aggregator fold of the superstep
    DeviceBuffers mem;
};

constexpr int kAppProgram = 3;   // app slot of user programs (after the paper's three)

struct Partition {
    int64_t vb = 0, ve = 0, rows = 0;
    int64_t csc_edges = 0, csr_edges = 0;
    int64_t csc_ebase = 0, csr_ebase = 0;   // global edge offset of this partition's first row
    const int32_t* csc_off = nullptr;
    const int32_t* csc_idx = nullptr;
    const uint32_t* csc_w = nullptr;
    const int32_t* csr_off = nullptr;
    const int32_t* csr_idx = nullptr;
    const uint32_t* csr_w = nullptr;
    TilePlan plan_csc, plan_csr;
    PushAdj push_sssp, push_cc;   // out-edges of every source that land in the owned range
    bool push_view_ready = false;
    int64_t nondangling = 0;
    DeviceBuffers graph_mem;      // host copies, tile plans, push view
    cudaEvent_t up_idx = nullptr, up_w = nullptr, up_all = nullptr;   // host-upload progress
    AppState st[4];
    PullCounters* pull_cnt = nullptr;         // device
    FrontierCounters* front_cnt = nullptr;    // device
    unsigned long long* host_cnt = nullptr;   // pinned [16]
    unsigned long long* dscratch = nullptr;   // device [64] (NCCL counter buffers)
};

struct StepRecord {
    float time_ms = 0, kernel_ms = 0;
    uint8_t mode = 0;
    uint64_t changed = 0, messages = 0, edges_scanned = 0, model_bytes = 0;
    double delta = 0.0;   // PageRank: max_v |r_s(v) - r_{s-1}(v)| (to-convergence runs)
};

}  // namespace

struct ipregel_graph {
    int64_t n = 0, e = 0;
    int device = 0;
    cudaStream_t stream = nullptr;
    ipregel_comm* comm = nullptr;
    std::vector<Partition> parts;
    std::vector<int64_t> rank_vb, rank_rows;  // multi-GPU: every rank's owned range
    bool poisoned = false;
    int last_app = -1;             // ipregel_app, or kAppProgram
    int last_vsz = 0;              // value bytes of the last run (8 PageRank / f64, 4 u32)
    int last_status = -1;
    int last_exchange = 0;         // 0 none, 1 collective, 2 fused
    int64_t last_rowlist_edges = 0;
    int64_t w_min = -1;            // smallest edge weight (SSSP absorption bound), lazily
    const int32_t* inv_ids = nullptr;   // original -> internal id (user programs' ipr_send)
    cudaStream_t capture_stream = nullptr;   // private stream for CUDA-graph capture
    cudaStream_t copy_stream = nullptr;      // host -> device uploads (MEMORY_HOST create)
    // PageRank (fixed k, pull) captured once as a CUDA graph and replayed: one launch per run
    struct {
        bool valid = false;
        uint32_t k = 0, max_steps = 0, flags = 0;
        cudaGraphExec_t exec = nullptr;
        std::vector<StepRecord> steps;
        int cur = 0;
        int exchange = 0;
        ipregel_status status = IPREGEL_OK;
        unsigned long long launches = 0;
    } pr_graph;
    int cur = 0;
    std::vector<StepRecord> steps;
    std::vector<cudaEvent_t> events;
    double* gather_tmp = nullptr;  // get_values scratch (full vector, internal order)
    double* gather_tmp2 = nullptr; // get_values scratch (original order)
    const int32_t* vertex_ids = nullptr;  // internal -> original id, or NULL
    bool degree_ordered = false;
    int gather_policy = 1;
    DeviceBuffers graph_mem;       // graph-level copies (vertex_ids from host)
};

// =============================================================================================
// internals
// =============================================================================================
namespace {

// Any graph created with a communicator exchanges through NCCL (a world of 1 included, which is
// how the NCCL path is exercised on a single GPU).
bool multi_rank(const ipregel_graph* g) { return g->comm != nullptr; }

void check_device(int device) {
    cudaDeviceProp prop;
    CU(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10 || prop.minor != 0)
        fail(IPREGEL_ERR_UNSUPPORTED, "device %d is sm_%d%d; this library is built for sm_100a",
             device, prop.major, prop.minor);
}

void build_plan(TilePlan& P, const int32_t* off, const int32_t* idx, const uint32_t* w,
                int64_t rows, int64_t edges, int64_t vertex_base, int64_t edge_base,
                DeviceBuffers& mem, cudaStream_t s) {
    P.rows = (int32_t)rows;
    P.edges = edges;
    // ranges on the global merge grid (diagonal = global row + global edge index), chunks on the
    // global 128-edge grid
    P.phase = (vertex_base + edge_base) % kRangeItems;
    P.cphase = edge_base % kChunk;
    P.num_tiles = rows > 0 ? (int32_t)ceil_div(rows + edges + P.phase, kRangeItems) : 0;
    (void)idx;
    (void)w;
    if (P.num_tiles == 0) return;
    const int32_t Q = P.num_tiles;
    P.cx = mem.alloc<int32_t>(Q + 1, s);
    P.cy = mem.alloc<int32_t>(Q + 1, s);
    P.carry = mem.alloc<double>(Q, s);   // 8-byte slots hold f64 or u32
    P.head = mem.alloc<double>(Q, s);
    k_plan_boundaries<<<grid_for(Q + 1, 256), 256, 0, s>>>(off, P.rows, edges, P.phase, Q, P.cx,
                                                           P.cy);
    LAUNCH_CHECK();
    // Rows cut by range boundaries: consecutive boundaries carrying the same row form one group
    // (row, a, b).  Host pass at create time (not timed).
    DeviceBuffers tmp;
    int32_t* infl = tmp.alloc<int32_t>(Q, s);
    k_plan_inflight<<<grid_for(Q, 256), 256, 0, s>>>(off, P.cx, P.cy, P.rows, Q, infl);
    LAUNCH_CHECK();
    std::vector<int32_t> h(Q);
    CU(cudaMemcpyAsync(h.data(), infl, Q * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    tmp.release();
    std::vector<int4> groups;
    for (int32_t b = 1; b < Q; ++b) {
        if (h[b] < 0) continue;
        if (!groups.empty() && groups.back().x == h[b] && groups.back().z == b - 1)
            groups.back().z = b;
        else
            groups.push_back(make_int4(h[b], b, b, 0));
    }
    P.num_groups = (int32_t)groups.size();
    if (P.num_groups) {
        P.groups = mem.alloc<int4>(P.num_groups, s);
        CU(cudaMemcpyAsync(P.groups, groups.data(), groups.size() * sizeof(int4),
                           cudaMemcpyHostToDevice, s));
        CU(cudaStreamSynchronize(s));
    }
}

RangeArgs range_args(const TilePlan& P, const int32_t* off, const int32_t* idx, const uint32_t* w,
                     PullCounters* cnt, cudaStream_t s, const void* gbase, int64_t n_global,
                     size_t vsz, int policy, bool degree_ordered);

template <class Op>
void launch_pull(const Op& op, const TilePlan& P, const int32_t* off, const int32_t* idx,
                 const uint32_t* w, PullCounters* cnt, cudaStream_t s, int64_t n_global,
                 int policy, bool degree_ordered) {
    using T = typename Op::T;
    if (P.num_tiles == 0) return;
    RangeArgs A = range_args(P, off, idx, w, cnt, s, op.gather_base(), n_global, sizeof(T), policy,
                             degree_ordered);
    k_pull_ranges<Op><<<(unsigned)ceil_div(P.num_tiles, kWarpsPerCta), kPullThreads, 0, s>>>(op, A);
    LAUNCH_CHECK();
    if (P.num_groups) {
        k_pull_fixup<Op><<<grid_for((int64_t)P.num_groups * 32, 256), 256, 0, s>>>(
            op, P.groups, P.num_groups, static_cast<const T*>(P.carry),
            static_cast<const T*>(P.head), cnt);
        LAUNCH_CHECK();
    }
}

RangeArgs range_args(const TilePlan& P, const int32_t* off, const int32_t* idx, const uint32_t* w,
                     PullCounters* cnt, cudaStream_t s, const void* gbase, int64_t n_global,
                     size_t vsz, int policy, bool degree_ordered) {
    const uint64_t total = std::min<uint64_t>((uint64_t)n_global * vsz, 0xFFFFFFFFull);
    const uint32_t hot = (uint32_t)std::min<uint64_t>(g_hot_bytes, total);
    if (g_persist_bytes) {
        static bool limit_set = false;
        if (!limit_set) {
            CU(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, g_persist_bytes));
            limit_set = true;
        }
        cudaStreamAttrValue a = {};
        a.accessPolicyWindow.base_ptr = const_cast<void*>(gbase);
        a.accessPolicyWindow.num_bytes = std::min<uint64_t>(g_persist_bytes, total);
        a.accessPolicyWindow.hitRatio = 1.0f;
        a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        CU(cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &a));
    }
    RangeArgs A;
    A.off = off; A.idx = idx; A.wts = w; A.cx = P.cx; A.cy = P.cy; A.rows = P.rows;
    A.cphase = (int32_t)P.cphase; A.num_ranges = P.num_tiles; A.carry_out = P.carry;
    A.head_out = P.head; A.counters = cnt; A.gather_policy = policy; A.gbase = gbase;
    A.ghot = hot; A.gtotal = (uint32_t)total;
    A.l1hot = g_l1_hot != -2 ? g_l1_hot : (degree_ordered ? (int32_t)(65536 / vsz) : -1);
    return A;
}

template <class T>
ncclDataType_t nccl_type();
template <>
ncclDataType_t nccl_type<double>() { return ncclFloat64; }
template <>
ncclDataType_t nccl_type<uint32_t>() { return ncclUint32; }
template <>
ncclDataType_t nccl_type<float>() { return ncclFloat32; }
template <>
ncclDataType_t nccl_type<int32_t>() { return ncclInt32; }
template <>
ncclDataType_t nccl_type<uint64_t>() { return ncclUint64; }
template <>
ncclDataType_t nccl_type<int64_t>() { return ncclInt64; }

// Replicate every partition's owned slice of a replica array into every other replica
// (multi-GPU: in-place AllGatherv as grouped ncclBroadcast, one root per rank range).
template <class T, class Get>
void exchange_owned(ipregel_graph* g, Get get) {
    if (multi_rank(g)) {
        T* rep = get(g->parts[0]);
        NC(ncclGroupStart());
        for (int r = 0; r < g->comm->world; ++r) {
            if (g->rank_rows[r] == 0) continue;
            NC(ncclBroadcast(rep + g->rank_vb[r], rep + g->rank_vb[r], (size_t)g->rank_rows[r],
                             nccl_type<T>(), r, g->comm->nccl, g->stream));
        }
        NC(ncclGroupEnd());
        return;
    }
    const int np = (int)g->parts.size();
    for (int a = 0; a < np; ++a) {
        Partition& pa = g->parts[a];
        if (pa.rows == 0) continue;
        for (int b = 0; b < np; ++b) {
            if (a == b) continue;
            CU(cudaMemcpyAsync(get(g->parts[b]) + pa.vb, get(pa) + pa.vb,
                               (size_t)pa.rows * sizeof(T), cudaMemcpyDeviceToDevice, g->stream));
        }
    }
}

// PageRank to convergence: max over partitions / ranks of the superstep's max per-vertex change
// (f64 bits of a non-negative value, so the u64 max is the f64 max; exact, order-independent).
unsigned long long reduce_max_delta(ipregel_graph* g) {
    if (multi_rank(g)) {
        Partition& p = g->parts[0];
        NC(ncclAllReduce(&p.pull_cnt->dmax, p.dscratch + 56, 1, ncclUint64, ncclMax,
                         g->comm->nccl, g->stream));
        CU(cudaMemcpyAsync(p.host_cnt + 3, p.dscratch + 56, 8, cudaMemcpyDeviceToHost, g->stream));
        CU(cudaStreamSynchronize(g->stream));
        return p.host_cnt[3];
    }
    for (auto& p : g->parts)
        CU(cudaMemcpyAsync(p.host_cnt + 3, &p.pull_cnt->dmax, 8, cudaMemcpyDeviceToHost,
                           g->stream));
    CU(cudaStreamSynchronize(g->stream));
    unsigned long long m = 0;
    for (auto& p : g->parts) m = std::max(m, p.host_cnt[3]);
    return m;
}

// Sum u64 device counters over partitions / ranks into out[0..count).
void reduce_counters(ipregel_graph* g, bool frontier, unsigned long long* out, int count) {
    for (int i = 0; i < count; ++i) out[i] = 0;
    if (multi_rank(g)) {
        Partition& p = g->parts[0];
        void* src = frontier ? (void*)p.front_cnt : (void*)p.pull_cnt;
        NC(ncclAllReduce(src, p.dscratch, (size_t)count, ncclUint64, ncclSum, g->comm->nccl,
                         g->stream));
        CU(cudaMemcpyAsync(p.host_cnt, p.dscratch, count * sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, g->stream));
        CU(cudaStreamSynchronize(g->stream));
        for (int i = 0; i < count; ++i) out[i] = p.host_cnt[i];
        return;
    }
    for (auto& p : g->parts) {
        void* src = frontier ? (void*)p.front_cnt : (void*)p.pull_cnt;
        CU(cudaMemcpyAsync(p.host_cnt, src, count * sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, g->stream));
    }
    CU(cudaStreamSynchronize(g->stream));
    for (auto& p : g->parts)
        for (int i = 0; i < count; ++i) out[i] += p.host_cnt[i];
}

int64_t words_of(int64_t rows) { return (rows + 31) >> 5; }

void ensure_state(ipregel_graph* g, int app) {
    for (auto& p : g->parts) {
        AppState& S = p.st[app];
        if (S.ready) continue;
        cudaStream_t s = g->stream;
        const int64_t n = g->n;
        const bool ipc = multi_rank(g);   // replicas a peer maps for the fused exchange
        if (app == IPREGEL_APP_PAGERANK) {
            S.rank = S.mem.alloc<double>(p.rows, s);
            S.contrib[0] = S.mem.alloc<double>(n, s, true, ipc);
            S.contrib[1] = S.mem.alloc<double>(n, s, true, ipc);
        } else if (app == kAppProgram) {
            S.pv_value = S.mem.alloc<uint64_t>(p.rows, s, true);
            S.pv_out[0] = S.mem.alloc<uint64_t>(n, s, true, ipc);
            S.pv_out[1] = S.mem.alloc<uint64_t>(n, s, true, ipc);
            S.pv_mbox = S.mem.alloc<uint64_t>(p.rows, s, true);
            S.pv_flags = S.mem.alloc<uint8_t>(p.rows, s, true);
            S.pv_recv = S.mem.alloc<uint32_t>(words_of(p.rows), s, true);
            S.pv_params = S.mem.alloc<double>(kProgParams, s, true);
            for (int w = 0; w < 2; ++w) {
                S.pv_p2p[w] = S.mem.alloc<uint64_t>(p.rows, s);
                S.pv_p2p_recv[w] = S.mem.alloc<uint32_t>(words_of(p.rows), s, true);
            }
            S.pv_shared = S.mem.alloc<ProgShared>(1, s, true);
            S.pv_sends = S.mem.alloc<unsigned long long>(1, s, true);
            S.pv_agg = S.mem.alloc<double>(1, s, true);
            S.bits = S.mem.alloc<uint32_t>(words_of(p.rows), s, true);
            S.f_id = S.mem.alloc<int32_t>(p.rows, s);
            S.f_val = S.mem.alloc<uint32_t>(p.rows, s);
            if (g->parts.size() > 1 || multi_rank(g)) {
                S.g_id = S.mem.alloc<int32_t>(n, s);
                S.g_val = S.mem.alloc<uint32_t>(n, s);
                S.g_len = S.mem.alloc<unsigned long long>(1, s, true);
            } else {
                S.g_id = S.f_id;
                S.g_val = S.f_val;
                S.g_len = &p.front_cnt->changed;
            }
        } else {
            S.val[0] = S.mem.alloc<uint32_t>(n, s, false, ipc);
            S.val[1] = S.mem.alloc<uint32_t>(n, s, false, ipc);
            S.bits = S.mem.alloc<uint32_t>(words_of(p.rows), s, true);
            S.f_id = S.mem.alloc<int32_t>(p.rows, s);
            S.f_val = S.mem.alloc<uint32_t>(p.rows, s);
            if (g->parts.size() > 1 || multi_rank(g)) {
                S.g_id = S.mem.alloc<int32_t>(n, s);
                S.g_val = S.mem.alloc<uint32_t>(n, s);
                S.g_len = S.mem.alloc<unsigned long long>(1, s, true);
            } else {
                S.g_id = S.f_id;
                S.g_val = S.f_val;
                S.g_len = &p.front_cnt->changed;
            }
        }
        // expand list + scan scratch (PageRank needs them for push mode only; allocated lazily)
        const int64_t blk = std::max<int64_t>(ceil_div(words_of(p.rows), kWordsPerBlock),
                                              ceil_div(n, kListPerBlock)) + 1;
        S.blk_a = S.mem.alloc<unsigned long long>(blk, s);
        S.blk_b = S.mem.alloc<unsigned long long>(blk, s);
        S.ready = true;
    }
}

void ensure_expand_list(Partition& p, AppState& S, int64_t n, cudaStream_t s) {
    if (S.e_id) return;
    S.e_id = S.mem.alloc<int32_t>(n, s);
    S.e_val = S.mem.alloc<uint32_t>(n, s);
    S.e_pre = S.mem.alloc<long long>(n, s);
    (void)p;
}

// Device-wide exclusive scan of int32 counts in place (create-time helper).
void exscan_i32(int32_t* a, int64_t n, DeviceBuffers& tmp, cudaStream_t s) {
    const int64_t nb = ceil_div(n, kScanChunk);
    unsigned long long* sums = tmp.alloc<unsigned long long>(nb, s);
    k_chunk_sums<<<grid_for(nb, 1), 256, 0, s>>>(a, n, sums);
    LAUNCH_CHECK();
    k_scan_blocks<<<1, 1024, 0, s>>>(sums, nullptr, nb, nullptr, nullptr);
    LAUNCH_CHECK();
    k_chunk_apply<<<grid_for(nb, 1), 256, 0, s>>>(a, n, sums);
    LAUNCH_CHECK();
}

// Transpose of a partition's rows (row r lists neighbours u) into a source-major adjacency over all
// N sources (u lists vb + r), allocated in the partition's graph memory.  Counting sort with an
// atomic cursor per source: the order inside a row is not deterministic (every consumer of a
// transposed adjacency combines with min, or with a sum that is order-nondeterministic anyway).
void transpose_rows(Partition& p, int64_t n, const int32_t* off, const int32_t* idx,
                    const uint32_t* w, int64_t edges, bool want_w, cudaStream_t s,
                    int32_t** out_off, int32_t** out_idx, uint32_t** out_w,
                    cudaEvent_t w_ready = nullptr) {
    int32_t* o = p.graph_mem.alloc<int32_t>(n + 1, s, true);
    int32_t* ix = p.graph_mem.alloc<int32_t>(edges, s);
    uint32_t* wx = want_w ? p.graph_mem.alloc<uint32_t>(edges, s) : nullptr;
    DeviceBuffers tmp;
    if (p.rows == 0 || edges == 0) CU(cudaMemsetAsync(o, 0, (n + 1) * sizeof(int32_t), s));
    if (p.rows > 0 && edges > 0) {
        // stable radix sort of (source, row | weight << 32) by source: coalesced, and each
        // transposed row lists its destinations in ascending order
        int32_t* k0 = tmp.alloc<int32_t>(edges, s);
        int32_t* k1 = tmp.alloc<int32_t>(edges, s);
        unsigned long long* v0 = tmp.alloc<unsigned long long>(edges, s);
        unsigned long long* v1 = tmp.alloc<unsigned long long>(edges, s);
        CU(cudaMemcpyAsync(k0, idx, edges * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
        k_transpose_pack<<<grid_for(p.rows * 32, 256), 256, 0, s>>>(off, p.rows, p.vb, v0);
        LAUNCH_CHECK();
        cub::DoubleBuffer<int32_t> keys(k0, k1);
        cub::DoubleBuffer<unsigned long long> vals(v0, v1);
        int bits = 1;
        while (bits < 31 && (int64_t(1) << bits) < n) ++bits;
        size_t temp_bytes = 0;
        CU(cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, keys, vals, edges, 0, bits, s));
        void* temp = tmp.alloc<uint8_t>((int64_t)temp_bytes, s);
        CU(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys, vals, edges, 0, bits, s));
        if (w_ready) CU(cudaStreamWaitEvent(s, w_ready, 0));   // weights uploaded meanwhile
        k_transpose_unpack<<<std::min<unsigned>(grid_for(edges, 256), 148 * 16), 256, 0, s>>>(
            vals.Current(), edges, w, ix, wx);
        LAUNCH_CHECK();
        // offsets from the sorted sources: run lengths, then an exclusive scan
        int32_t* st = tmp.alloc<int32_t>(n, s, true);
        k_run_bounds<<<std::min<unsigned>(grid_for(edges, 256), 148 * 16), 256, 0, s>>>(
            keys.Current(), edges, st, o);
        k_run_counts<<<grid_for(n, 256), 256, 0, s>>>(st, n, o);
        LAUNCH_CHECK();
        exscan_i32(o, n + 1, tmp, s);
    }
    CU(cudaStreamSynchronize(s));
    tmp.release();
    *out_off = o;
    *out_idx = ix;
    if (out_w) *out_w = wx;
}

// Push adjacency of one partition.  One partition: the graph's own CSR (+ CSC for CC).  Several:
// transposes of the owned CSC (and, for CC, owned CSR) rows, over all N sources.
void ensure_push_view(ipregel_graph* g, Partition& p) {
    if (p.push_view_ready) return;
    cudaStream_t s = g->stream;
    const int64_t n = g->n;
    if (g->parts.size() == 1 && !multi_rank(g)) {
        p.push_sssp = PushAdj{p.csr_off, p.csr_idx, p.csr_w, nullptr, nullptr, nullptr, 0, n};
        p.push_cc = PushAdj{p.csr_off, p.csr_idx, p.csr_w, p.csc_off, p.csc_idx, p.csc_w, 0, n};
        p.push_view_ready = true;
        return;
    }
    auto transpose = [&](const int32_t* off, const int32_t* idx, const uint32_t* w, int64_t edges,
                         bool want_w, int32_t** out_off, int32_t** out_idx, uint32_t** out_w) {
        transpose_rows(p, n, off, idx, w, edges, want_w, s, out_off, out_idx, out_w);
    };
    int32_t *o1, *i1, *o2, *i2;
    uint32_t *w1 = nullptr, *w2 = nullptr;
    transpose(p.csc_off, p.csc_idx, p.csc_w, p.csc_edges, p.csc_w != nullptr, &o1, &i1, &w1);
    transpose(p.csr_off, p.csr_idx, p.csr_w, p.csr_edges, p.csr_w != nullptr, &o2, &i2, &w2);
    p.push_sssp = PushAdj{o1, i1, w1, nullptr, nullptr, nullptr, 0, n};
    p.push_cc = PushAdj{o1, i1, w1, o2, i2, w2, 0, n};
    p.push_view_ready = true;
}

// ---- frontier machinery ------------------------------------------------------------------
// Compact the owned bitmap into (ids, snapshots) and count broadcasters / messages.
void compact_bitmap(ipregel_graph* g, Partition& p, AppState& S, const uint32_t* vals, bool cc) {
    cudaStream_t s = g->stream;
    const int64_t nw = words_of(p.rows);
    const int64_t nb = std::max<int64_t>(ceil_div(nw, kWordsPerBlock), 1);
    OwnedDegree deg{p.csr_off, cc ? p.csc_off : nullptr};
    k_bitmap_count<<<(unsigned)nb, kScanThreads, 0, s>>>(S.bits, nw, deg, S.blk_a, S.blk_b);
    LAUNCH_CHECK();
    k_scan_blocks<<<1, 1024, 0, s>>>(S.blk_a, S.blk_b, nb, &p.front_cnt->changed,
                                     &p.front_cnt->messages);
    LAUNCH_CHECK();
    k_bitmap_write<<<(unsigned)nb, kScanThreads, 0, s>>>(S.bits, nw, p.vb, vals, S.blk_a, S.f_id,
                                                        S.f_val);
    LAUNCH_CHECK();
}

// Multi-partition: concatenate every partition's owned frontier (rank order = ascending ids)
// into every partition's global frontier and scatter the snapshots into its replica.
void exchange_frontier(ipregel_graph* g, int app, const std::vector<unsigned long long>& counts,
                       int cur) {
    auto replica = [app](Partition& p, int w) { return p.st[app].val[w]; };
    // user programs read broadcast payloads from their (exchanged) outbox replicas: ids only
    const bool scatter = app != kAppProgram;
    cudaStream_t s = g->stream;
    if (multi_rank(g)) {
        Partition& p = g->parts[0];
        AppState& S = p.st[app];
        unsigned long long total = 0;
        std::vector<unsigned long long> off(counts.size());
        for (size_t r = 0; r < counts.size(); ++r) { off[r] = total; total += counts[r]; }
        NC(ncclGroupStart());
        for (int r = 0; r < g->comm->world; ++r) {
            if (counts[r] == 0) continue;
            const void* sid = r == g->comm->rank ? (const void*)S.f_id : nullptr;
            const void* sval = r == g->comm->rank ? (const void*)S.f_val : nullptr;
            NC(ncclBroadcast(sid, S.g_id + off[r], counts[r], ncclInt32, r, g->comm->nccl, s));
            NC(ncclBroadcast(sval, S.g_val + off[r], counts[r], ncclUint32, r, g->comm->nccl, s));
        }
        NC(ncclGroupEnd());
        CU(cudaMemcpyAsync(S.g_len, &total, sizeof(total), cudaMemcpyHostToDevice, s));
        if (scatter) {
            k_scatter_frontier<<<grid_for(std::max<unsigned long long>(total, 1ull), 256) > 2048
                                     ? 2048 : grid_for(std::max<unsigned long long>(total, 1ull), 256),
                                 256, 0, s>>>(S.g_id, S.g_val, S.g_len, replica(p, cur));
            LAUNCH_CHECK();
        }
        CU(cudaStreamSynchronize(s));  // `total` lives on the host stack
        return;
    }
    const int np = (int)g->parts.size();
    if (np <= 1) return;
    unsigned long long total = 0;
    std::vector<unsigned long long> off(np);
    for (int a = 0; a < np; ++a) { off[a] = total; total += counts[a]; }
    for (int b = 0; b < np; ++b) {
        AppState& Sb = g->parts[b].st[app];
        for (int a = 0; a < np; ++a) {
            if (counts[a] == 0) continue;
            AppState& Sa = g->parts[a].st[app];
            CU(cudaMemcpyAsync(Sb.g_id + off[a], Sa.f_id, counts[a] * sizeof(int32_t),
                               cudaMemcpyDeviceToDevice, s));
            CU(cudaMemcpyAsync(Sb.g_val + off[a], Sa.f_val, counts[a] * sizeof(uint32_t),
                               cudaMemcpyDeviceToDevice, s));
        }
        CU(cudaMemcpyAsync(Sb.g_len, &total, sizeof(total), cudaMemcpyHostToDevice, s));
        if (scatter) {
            unsigned gr = grid_for(std::max<unsigned long long>(total, 1ull), 256);
            k_scatter_frontier<<<gr > 2048 ? 2048 : gr, 256, 0, s>>>(Sb.g_id, Sb.g_val, Sb.g_len,
                                                                    replica(g->parts[b], cur));
            LAUNCH_CHECK();
        }
    }
    CU(cudaStreamSynchronize(s));  // `total` lives on the host stack
}

// Build the expand list (entries of the global frontier with push-view degree > 0, with the
// exclusive degree prefix) for one partition.
void build_expand_list(ipregel_graph* g, Partition& p, AppState& S, const PushAdj& adj,
                       const int32_t* ids, const uint32_t* vals, const unsigned long long* len,
                       int64_t len_host) {
    cudaStream_t s = g->stream;
    ensure_expand_list(p, S, g->n, s);
    const int64_t nb = std::max<int64_t>(ceil_div(len_host, kListPerBlock), 1);
    k_list_count<<<(unsigned)nb, kScanThreads, 0, s>>>(ids, len, adj, S.blk_a, S.blk_b);
    LAUNCH_CHECK();
    k_scan_blocks<<<1, 1024, 0, s>>>(S.blk_a, S.blk_b, nb, &p.front_cnt->list_len,
                                     &p.front_cnt->list_edges);
    LAUNCH_CHECK();
    k_list_write<<<(unsigned)nb, kScanThreads, 0, s>>>(ids, vals, len, adj, S.blk_a, S.blk_b,
                                                      S.e_id, S.e_val, S.e_pre);
    LAUNCH_CHECK();
}

// Per-partition owned-frontier sizes, in partition / rank order.
std::vector<unsigned long long> frontier_counts(ipregel_graph* g) {
    cudaStream_t s = g->stream;
    std::vector<unsigned long long> counts;
    if (multi_rank(g)) {
        Partition& p = g->parts[0];
        NC(ncclAllGather(&p.front_cnt->changed, p.dscratch, 1, ncclUint64, g->comm->nccl, s));
        counts.assign(g->comm->world, 0);
        CU(cudaMemcpyAsync(counts.data(), p.dscratch, g->comm->world * 8, cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
        return counts;
    }
    for (auto& p : g->parts)
        CU(cudaMemcpyAsync(p.host_cnt + 2, &p.front_cnt->changed, 8, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    for (auto& p : g->parts) counts.push_back(p.host_cnt[2]);
    return counts;
}

// ---- fused exchange ----------------------------------------------------
void* replica_buf(AppState& S, int app, int w) {
    if (app == kAppProgram) return S.pv_out[w];
    return app == IPREGEL_APP_PAGERANK ? (void*)S.contrib[w] : (void*)S.val[w];
}

// Ranks: map every other rank's replica buffers into this process (CUDA IPC over NVLink /
// NVSwitch).  Collective: the handles travel by ncclAllGather and the ranks agree (AllReduce)
// that every mapping succeeded; otherwise nothing stays mapped and the run falls back to the
// collective exchange.
void setup_ipc_peers(ipregel_graph* g, int app) {
    Partition& p = g->parts[0];
    AppState& S = p.st[app];
    if (S.peers_state != 0) return;
    cudaStream_t s = g->stream;
    const int world = g->comm->world, rank = g->comm->rank;
    constexpr size_t H = sizeof(cudaIpcMemHandle_t);
    unsigned long long bad = world - 1 > kMaxPeers ? 1ull : 0ull;
    std::vector<uint8_t> mine(2 * H, 0), all(2 * H * world, 0);
    for (int w = 0; w < 2 && !bad; ++w) {
        cudaIpcMemHandle_t h;
        if (cudaIpcGetMemHandle(&h, replica_buf(S, app, w)) != cudaSuccess) {
            cudaGetLastError();
            bad = 1;
        } else {
            memcpy(mine.data() + w * H, &h, H);
        }
    }
    DeviceBuffers tmp;
    uint8_t* dsend = tmp.alloc<uint8_t>(2 * H, s);
    uint8_t* drecv = tmp.alloc<uint8_t>(2 * H * world, s);
    CU(cudaMemcpyAsync(dsend, mine.data(), 2 * H, cudaMemcpyHostToDevice, s));
    NC(ncclAllGather(dsend, drecv, 2 * H, ncclUint8, g->comm->nccl, s));
    CU(cudaMemcpyAsync(all.data(), drecv, all.size(), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    tmp.release();
    std::vector<void*> opened;
    int k = 0;
    for (int r = 0; r < world && !bad; ++r) {
        if (r == rank) continue;
        for (int w = 0; w < 2 && !bad; ++w) {
            cudaIpcMemHandle_t h;
            memcpy(&h, all.data() + (2 * r + w) * H, H);
            void* q = nullptr;
            if (cudaIpcOpenMemHandle(&q, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
                cudaGetLastError();
                bad = 1;
                break;
            }
            opened.push_back(q);
            S.peer[w][k] = q;
        }
        ++k;
    }
    // every rank must agree before any kernel stores into a peer
    p.host_cnt[0] = bad;
    CU(cudaMemcpyAsync(p.dscratch + 40, p.host_cnt, 8, cudaMemcpyHostToDevice, s));
    NC(ncclAllReduce(p.dscratch + 40, p.dscratch + 41, 1, ncclUint64, ncclSum, g->comm->nccl, s));
    CU(cudaMemcpyAsync(p.host_cnt + 1, p.dscratch + 41, 8, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    if (p.host_cnt[1] != 0) {
        for (void* q : opened) cudaIpcCloseMemHandle(q);
        S.npeer = 0;
        S.peers_state = -1;
        return;
    }
    S.ipc_opened = opened;
    S.npeer = world - 1;
    S.peers_state = 1;
}

// Whether the pull supersteps of this run exchange through the fused epilogue stores.
bool use_fused_exchange(ipregel_graph* g, int app, uint32_t flags) {
    if (flags & IPREGEL_RUN_EXCHANGE_COLLECTIVE) return false;
    const bool require = (flags & IPREGEL_RUN_EXCHANGE_FUSED) != 0;
    if (multi_rank(g)) {
        setup_ipc_peers(g, app);
        if (g->parts[0].st[app].peers_state == 1) return true;
        if (require)
            fail(IPREGEL_ERR_UNSUPPORTED, "fused exchange: peer replicas not reachable (CUDA IPC)");
        return false;
    }
    const int np = (int)g->parts.size();
    if (np == 1) return true;   // nothing to exchange: the owned slice is the whole replica
    if (np - 1 > kMaxPeers) {
        if (require)
            fail(IPREGEL_ERR_UNSUPPORTED, "fused exchange supports at most %d partitions",
                 kMaxPeers + 1);
        return false;
    }
    for (int a = 0; a < np; ++a) {
        AppState& S = g->parts[a].st[app];
        if (S.peers_state == 1) continue;
        int k = 0;
        for (int b = 0; b < np; ++b) {
            if (b == a) continue;
            for (int w = 0; w < 2; ++w) S.peer[w][k] = replica_buf(g->parts[b].st[app], app, w);
            ++k;
        }
        S.npeer = k;
        S.peers_state = 1;
    }
    return true;
}

int exchange_kind(ipregel_graph* g, bool fused) {
    if (!multi_rank(g) && g->parts.size() == 1) return 0;
    return fused ? 2 : 1;
}

template <class T>
PeerSlots<T> peer_slots(const AppState& S, int w, bool fused) {
    PeerSlots<T> ps{};
    ps.n = fused ? S.npeer : 0;
    for (int k = 0; k < ps.n; ++k) ps.p[k] = static_cast<T*>(S.peer[w][k]);
    return ps;
}

// Superstep barrier after fused stores (ranks): a one-element AllReduce on the run stream.  It
// completes on a rank only after every rank's pull kernel -- and so its peer stores -- finished.
void fused_barrier(ipregel_graph* g) {
    if (!multi_rank(g)) return;   // loopback: stream order
    Partition& p = g->parts[0];
    NC(ncclAllReduce(p.dscratch + 48, p.dscratch + 49, 1, ncclUint64, ncclSum, g->comm->nccl,
                     g->stream));
}

// ---- timing -------------------------------------------------------------------------------
cudaEvent_t ev(ipregel_graph* g, size_t i) {
    while (g->events.size() <= i) {
        cudaEvent_t e;
        CU(cudaEventCreate(&e));
        g->events.push_back(e);
    }
    return g->events[i];
}

// Per-superstep CUDA events on the run stream.  Inside a CUDA-graph capture they are recorded as
// external event nodes, so they still time the superstep when the graph is replayed.
struct StepTimer {
    ipregel_graph* g;
    size_t step;
    void rec(size_t i) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        CU(cudaStreamIsCapturing(g->stream, &cs));
        if (cs == cudaStreamCaptureStatusActive)
            CU(cudaEventRecordWithFlags(ev(g, i), g->stream, cudaEventRecordExternal));
        else
            CU(cudaEventRecord(ev(g, i), g->stream));
    }
    void begin() { rec(4 * step + 0); }
    void kbegin() { rec(4 * step + 1); }
    void kend() { rec(4 * step + 2); }
    void end() { rec(4 * step + 3); }
};

void finalize_times(ipregel_graph* g) {
    CU(cudaStreamSynchronize(g->stream));
    for (size_t s = 0; s < g->steps.size(); ++s) {
        float a = 0, b = 0;
        CU(cudaEventElapsedTime(&a, ev(g, 4 * s + 0), ev(g, 4 * s + 3)));
        CU(cudaEventElapsedTime(&b, ev(g, 4 * s + 1), ev(g, 4 * s + 2)));
        g->steps[s].time_ms = a;
        g->steps[s].kernel_ms = b;
    }
}

// =============================================================================================
// PageRank (Fig. 8)
// =============================================================================================
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
        return G.status;
    }
    const unsigned long long launches0 = g_launches.load(std::memory_order_relaxed);
    if (graphable) {
        for (uint32_t i = 0; i <= 4 * (k + 1); ++i) ev(g, i);   // events exist before capture
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
    T0.kbegin();
    for (auto& p : g->parts) {
        AppState& S = p.st[IPREGEL_APP_PAGERANK];
        if (p.rows == 0) continue;
        k_init_pagerank<<<grid_for(p.rows, 256), 256, 0, s>>>(p.csr_off, p.rows, p.vb, inv_n,
                                                              k > 0, last == 0 || track, S.rank,
                                                              S.contrib[0]);
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
                if (g_pr_split) {
                    PageRankSum sop;
                    sop.contrib_cur = op.contrib_cur;
                    sop.sum_out = op.contrib_next;
                    sop.vbase = p.vb;
                    launch_pull(sop, p.plan_csc, p.csc_off, p.csc_idx, nullptr, nullptr, s, n,
                                g->gather_policy, g->degree_ordered);
                    k_pr_finish<<<grid_for(p.rows, 256), 256, 0, s>>>(op, p.rows,
                                                                      track ? p.pull_cnt : nullptr);
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
                    S.contrib[1 - cur], track ? &p.pull_cnt->dmax : nullptr);
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
        R.model_bytes = push ? 12ull * g->e + 24ull * n : 12ull * g->e + 16ull * n;
        if (track) R.model_bytes += 16ull * n;   // rank read + write every superstep
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
        if (p.rows)
            k_bits_ne<<<grid_for(p.rows, 256), 256, 0, s>>>(S.val[cur] + p.vb, p.rows, 0u, S.bits);
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
        if (cc) k_init_cc<<<grid_for(n, 256), 256, 0, s>>>(S.val[0], n, g->vertex_ids);
        else k_init_sssp<<<grid_for(n, 256), 256, 0, s>>>(S.val[0], n, source);
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
                        k_bitmap_from_diff<<<grid_for(p.rows, 256), 256, 0, s>>>(
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
                    std::max<int64_t>(ceil_div((int64_t)messages, kExpandItems), 1), 148 * 8);
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
                    std::max<int64_t>(ceil_div((int64_t)p.host_cnt[5], kExpandItems), 1), 148 * 8);
                k_rowlist_min<<<grid, kExpandThreads, 0, s>>>(
                    own, S.e_id, S.e_pre, &p.front_cnt->list_len, &p.front_cnt->list_edges,
                    S.val[cur], S.val[1 - cur]);
                LAUNCH_CHECK();
            }
            T.kend();
            // broadcasters = rows whose label decreased; their count and symmetrised degrees
            for (auto& p : g->parts) {
                AppState& S = p.st[app];
                k_bitmap_from_diff<<<grid_for(std::max<int64_t>(p.rows, 1), 256), 256, 0, s>>>(
                    S.val[cur], S.val[1 - cur], p.vb, p.rows, S.bits);
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
            lists_ready = false;
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
                    launch_pull(a, p.plan_csc, p.csc_off, p.csc_idx, nullptr, nullptr, s, n,
                                g->gather_policy, g->degree_ordered);
                    CCPullOut b;
                    b.cur = S.val[cur]; b.next = S.val[1 - cur]; b.in_off = p.csc_off;
                    b.out_off = p.csr_off; b.vbase = p.vb;
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
            unsigned long long c[4];
            reduce_counters(g, false, c, 4);
            zero_edges = c[3];
            if (!cc) m_prev = (uint32_t)(kInf - (uint32_t)reduce_max_delta(g));
            T.end();
            StepRecord& R = g->steps.back();
            R.mode = 1;
            R.edges_scanned = pull_edges;
            R.model_bytes = cc ? 8ull * pull_edges + 16ull * n : 12ull * pull_edges + 12ull * n;
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

// =============================================================================================
// user vertex programs: NVRTC compilation and the generic superstep loop
// =============================================================================================
enum { PK_INIT, PK_PULL0, PK_PULL1, PK_PULL2, PK_FIX0, PK_FIX1, PK_FIX2, PK_EXPAND, PK_APPLY,
       PK_COUNT };
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
};

struct ipregel_program {
    int value_type = 0;   // ipregel_value_type
    int combiner = 0;     // ipregel_combiner
    int sym = 0;
    int agg_op = -1;      // aggregator (ipregel_combiner over f64), -1 none
    bool sends = false;   // the source calls ipr_send (point-to-point messages)
    std::vector<char> cubin;
    std::string log;
    std::string lowered[PK_COUNT];
    cudaLibrary_t lib = nullptr;
    cudaKernel_t k[PK_COUNT] = {};
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
    s += std::string("  static constexpr bool kSends = ") +
         (strstr(d.source, "ipr_send") ? "true" : "false") + ";\n";
    s += std::string("  static constexpr bool kAggregates = ") +
         (d.aggregator != IPREGEL_AGG_NONE ? "true" : "false") + ";\n";
    const bool absorbing = strstr(d.source, "ipr_absorbing") != nullptr;
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
    // IEEE arithmetic as written (no FMA contraction), the oracle's convention (R7)
    const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "--fmad=false", "-lineinfo",
                          "-default-device", "--ptxas-options=-v",
                          "-DIPREGEL_JIT=1"};
    r = N.compile(prog, (int)(sizeof(opts) / sizeof(opts[0])), opts);
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
    launch_jit(pr->k[PK_PULL0 + pass], (unsigned)ceil_div(P.num_tiles, kWarpsPerCta), kPullThreads,
               args, g->stream);
    if (P.num_groups) {
        const int4* groups = P.groups;
        int32_t ng = P.num_groups;
        const V* carry = static_cast<const V*>(P.carry);
        const V* head = static_cast<const V*>(P.head);
        void* fargs[] = {&a, &groups, &ng, &carry, &head, &cnt};
        launch_jit(pr->k[PK_FIX0 + pass], grid_for((int64_t)ng * 32, 256), 256, fargs, g->stream);
    }
}

template <class V>
ipregel_status run_program_t(ipregel_graph* g, ipregel_program* pr, uint32_t max_steps,
                             const ipregel_run_params& P, const double* params, int nparams) {
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
                    k_fill_u64<<<grid_for(p.rows, 256), 256, 0, s>>>(
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
        a.vbase = p.vb;
        a.rows = p.rows;
        a.n = n;
        a.superstep = step;
        a.sym = sym ? 1 : 0;
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
    reset_extras();
    T0.kbegin();
    for (auto& p : g->parts) {
        ProgArgs<V> a = args_for(p, 0, 1);   // out_next = buffer 0
        PullCounters* cnt = p.pull_cnt;
        void* args[] = {&a, &cnt};
        launch_jit(pr->k[PK_INIT], grid_for(p.rows, 256), 256, args, s);
    }
    T0.kend();
    exchange(0);
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
        reset_extras();
        if (mode == 2) {
            // frontier = the broadcasters of superstep s-1 (flag bytes -> bitmap -> ids)
            for (auto& p : g->parts) {
                if (p.rows) {
                    k_bits_from_flags<<<grid_for(p.rows, 256), 256, 0, s>>>(p.st[app].pv_flags,
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
                    std::max<int64_t>(ceil_div((int64_t)messages, kExpandItems), 1), 148 * 8);
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
                launch_jit(pr->k[PK_APPLY], grid_for(p.rows, 256), 256, args, s);
            }
            T.kend();
        } else {
            T.kbegin();
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
            T.kend();
        }
        exchange(1 - cur);
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
    }
    g->cur = cur;
    finalize_times(g);
    return status;
}

}  // namespace

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
    if (P.flags & ~(uint32_t)(IPREGEL_RUN_EXCHANGE_COLLECTIVE | IPREGEL_RUN_EXCHANGE_FUSED))
        fail(IPREGEL_ERR_INVALID_ARGUMENT, "unknown flags 0x%x", P.flags);
    if ((P.flags & IPREGEL_RUN_EXCHANGE_COLLECTIVE) && (P.flags & IPREGEL_RUN_EXCHANGE_FUSED))
        fail(IPREGEL_ERR_INVALID_ARGUMENT, "EXCHANGE_COLLECTIVE and EXCHANGE_FUSED are exclusive");
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
    }
    return IPREGEL_OK;
    ABI_END
}

}  // extern "C"
