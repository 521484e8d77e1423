// paper_2010_08781_b200/csrc/engine.cuh -- errors, device memory, the graph and partition state, launch helpers, exchanges, frontier machinery, the fused exchange and per-superstep timing.
// Host part of the single translation unit ipregel.cu (included once, in order).
#pragma once
#include <algorithm>
#include <chrono>
#include <mutex>

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

// SM count of a device (cached): grid-stride kernels launch a few CTAs per SM.
int device_sms(int device = -1) {
    static int cache[64] = {};
    if (device < 0) CU(cudaGetDevice(&device));
    if (device >= 0 && device < 64 && cache[device]) return cache[device];
    int v = 0;
    CU(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device));
    if (device >= 0 && device < 64) cache[device] = v;
    return v;
}
// grid of `per_sm` CTAs on every SM of the current device
inline unsigned sm_grid(int per_sm) { return (unsigned)(device_sms() * per_sm); }

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
// Diagnostic: per-kernel events of PageRank supersteps (IPREGEL_TRACE_KERNELS=1, stderr)
int g_trace_kernels = getenv("IPREGEL_TRACE_KERNELS") ? atoi(getenv("IPREGEL_TRACE_KERNELS")) : 0;
// Tuning knob: PageRank update split out of the range kernel (IPREGEL_PR_SPLIT=1).
int g_pr_split = getenv("IPREGEL_PR_SPLIT") ? atoi(getenv("IPREGEL_PR_SPLIT")) : 1;
// Range kernels: a grid of IPREGEL_PULL_WAVES x the resident CTAs (0: one warp per range),
// warps taking ranges from an atomic counter (IPREGEL_PULL_DYNAMIC=1) or striding (0).
int g_pull_dynamic = getenv("IPREGEL_PULL_DYNAMIC") ? atoi(getenv("IPREGEL_PULL_DYNAMIC")) : 1;
int g_pull_waves = getenv("IPREGEL_PULL_WAVES") ? std::max(atoi(getenv("IPREGEL_PULL_WAVES")), 0) : 1;
// Range kernels: order in which warps take the ranges (IPREGEL_RANGE_ORDER): 1 (default)
// alternates between the two ends of the plan, 0 plan order, k >= 2 k interleaved slices.
// cfg4: PageRank 72.2 -> 70.4 ms, Hash-Min 14.8 -> 14.1, SSSP 12.85 -> 12.0 (1 vs 0); 2-16 between
int g_range_order = getenv("IPREGEL_RANGE_ORDER") ? atoi(getenv("IPREGEL_RANGE_ORDER")) : 1;
// Range kernels: preferred shared-memory carveout in percent (IPREGEL_PULL_CARVEOUT; -1: the
// driver's default)
int g_pull_carveout = getenv("IPREGEL_PULL_CARVEOUT") ? atoi(getenv("IPREGEL_PULL_CARVEOUT")) : -1;
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
// IPREGEL_POOL_RETAIN_BYTES (default 144 GiB) of freed memory for the next graph instead of
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
    uint64_t keep = e ? strtoull(e, nullptr, 10) : (144ull << 30);
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

// IPREGEL_LAYOUT_DEGREE: what the deferred CSR sort of relabel_by_degree needs (create.cuh).
struct RelabelCsr {
    bool armed = false;
    DeviceBuffers tmp;
    int64_t n = 0, E = 0;
    int bits = 0;
    const int32_t* off = nullptr;
    const int32_t* idx = nullptr;
    const uint32_t* w = nullptr;
    unsigned long long *k0 = nullptr, *k1 = nullptr;
    int32_t *row = nullptr, *spare = nullptr;
    void* t = nullptr;
    size_t tb = 0;
    int32_t* ridx = nullptr;
    uint32_t* rw = nullptr;
};

// Pinned host blocks, cached for the process: cudaMallocHost / cudaFreeHost cost milliseconds
// (page pinning, a device synchronisation) and showed up as tens of ms of jitter per graph
// create / destroy, so blocks go back to this cache instead of being freed.
std::mutex g_pin_mu;
std::vector<std::pair<void*, size_t>> g_pin_free;
std::vector<std::pair<void*, size_t>> g_pin_sizes;   // every block ever allocated
void* pinned_acquire(size_t bytes) {
    bytes = std::max<size_t>(bytes, 4096);
    {
        std::lock_guard<std::mutex> lk(g_pin_mu);
        size_t best = g_pin_free.size();
        for (size_t i = 0; i < g_pin_free.size(); ++i)
            if (g_pin_free[i].second >= bytes &&
                (best == g_pin_free.size() || g_pin_free[i].second < g_pin_free[best].second))
                best = i;
        if (best < g_pin_free.size()) {
            void* p = g_pin_free[best].first;
            g_pin_free.erase(g_pin_free.begin() + best);
            return p;
        }
    }
    void* p = nullptr;
    CU(cudaMallocHost(&p, bytes));
    std::lock_guard<std::mutex> lk(g_pin_mu);
    g_pin_sizes.push_back({p, bytes});
    return p;
}
void pinned_release(void* p) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_pin_mu);
    for (auto& b : g_pin_sizes)
        if (b.first == p) {
            g_pin_free.push_back(b);
            return;
        }
}

// Per-graph staging slots over the cache.
struct PinnedStage {
    std::vector<std::pair<void*, size_t>> slots;
    void* get(size_t bytes, int slot) {
        if ((int)slots.size() <= slot) slots.resize(slot + 1, {nullptr, 0});
        if (slots[slot].first && slots[slot].second >= bytes) return slots[slot].first;
        pinned_release(slots[slot].first);
        slots[slot] = {pinned_acquire(bytes), std::max<size_t>(bytes, 4096)};
        return slots[slot].first;
    }
    void release() {
        for (auto& b : slots) pinned_release(b.first);
        slots.clear();
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
    uint32_t* nbr = nullptr;                   // Hash-Min: owned rows with a neighbour (bitmap)
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
    uint8_t* pv_flags = nullptr;               // owned: bit 0 broadcast, bit 1 active, bit 2
                                               // broadcast one superstep earlier (padded to 32)
    uint32_t* pv_recv = nullptr;               // owned recipient bitmap (push)
    double* pv_params = nullptr;               // program parameters [8]
    void* pv_p2p[2] = {nullptr, nullptr};      // point-to-point mailboxes [rows] (by parity)
    uint32_t* pv_p2p_recv[2] = {nullptr, nullptr};
    ProgShared* pv_shared = nullptr;           // device copy of the run's ProgShared
    unsigned long long* pv_sends = nullptr;    // point-to-point sends of the superstep
    double* pv_agg = nullptr;                  // aggregator fold of the superstep
    unsigned long long* pv_mkey = nullptr;     // ipr_settled: min broadcast key [2] (by parity)
    unsigned long long* pv_bound = nullptr;    //   and the pull superstep's bound [1]
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
    FlagPlan plan_flag;           // PageRank pull over the row-end-flagged CSC (pr_flag.cuh)
    PushAdj push_sssp, push_cc;   // out-edges of every source that land in the owned range
    bool push_view_ready = false;
    int64_t nondangling = 0;
    DeviceBuffers graph_mem;      // host copies, tile plans, push view
    cudaEvent_t up_idx = nullptr, up_w = nullptr, up_all = nullptr;   // host-upload progress
    // derived CSR weights permuted window by window as the CSC weights' windows land (create
    // from host memory): wx[i] = w[perm[i]] for perm[i] in [wc_bounds[c], wc_bounds[c + 1])
    struct {
        DeviceBuffers tmp;
        int32_t* perm = nullptr;     // [edges] CSC position of each transposed entry
        const uint32_t* w = nullptr;
        uint32_t* wx = nullptr;
        int64_t edges = 0;
    } pend;
    std::vector<cudaEvent_t> up_wc;   // one per weight window (copy stream)
    std::vector<cudaEvent_t> up_hist; // one per index window of the relabel's histogram
    cudaEvent_t perm_done = nullptr;  // the last window permuted (aux stream)
    // IPREGEL_LAYOUT_DEGREE: the CSR's indices / weights are built on the aux stream after create
    // returns; csr_off is ready.  wait_csr() orders the run stream after them (first use).
    cudaEvent_t csr_done = nullptr;
    bool csr_pending = false;
    RelabelCsr relabel_csr;           // its launch, deferred to after the tile plans
    uint32_t* pre_deg = nullptr;      // its out-degree histogram, counted during the upload
    DeviceBuffers pre_deg_mem;
    std::vector<int64_t> wc_bounds;
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
    double mass[2] = {0.0, 0.0};   // PageRank mass check: sum r_s, sum over outdeg > 0
    float part_ms = 0;             // PageRank pull: range kernel + fixup (kernel_ms - update)
};

}  // namespace

struct ipregel_graph {
    int64_t n = 0, e = 0;
    int device = 0;
    cudaStream_t stream = nullptr;
    ipregel_comm* comm = nullptr;
    std::vector<Partition> parts;
    PinnedStage pinned;                      // create's staging (kernel copies)
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
    cudaStream_t aux_stream = nullptr;       // create: weight permutation while uploading
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
    double* pr_mass = nullptr;     // PageRank mass check: [2 * pr_mass_cap] device sums
    uint32_t pr_mass_cap = 0;
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
    // the compute capability only (cudaGetDeviceProperties measured 5-190 ms per call inside
    // graph creation), checked once per device
    static int ok[64] = {};
    if (device >= 0 && device < 64 && ok[device]) return;
    int major = 0, minor = 0;
    CU(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
    CU(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device));
    if (major != 10 || minor != 0)
        fail(IPREGEL_ERR_UNSUPPORTED, "device %d is sm_%d%d; this library is built for sm_100a",
             device, major, minor);
    if (device >= 0 && device < 64) ok[device] = 1;
}

// Copies through a kernel (UVA: either side may be pinned host memory).  Create uses them for
// its small readbacks and uploads so the copy engines stay out of the host-upload window: a
// cudaMemcpy on the run stream would queue behind the upload (see compute_fence, create.cuh).
__global__ void k_copy_words(const uint32_t* __restrict__ src, uint32_t* __restrict__ dst, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}
void kernel_copy(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    if (bytes == 0) return;
    if (bytes % 4) fail(IPREGEL_ERR_INVALID_ARGUMENT, "kernel_copy of %zu bytes", bytes);
    const int64_t n = (int64_t)(bytes / 4);
    k_copy_words<<<std::min<unsigned>(grid_for(n, 256), sm_grid(8)), 256, 0, s>>>(
        static_cast<const uint32_t*>(src), static_cast<uint32_t*>(dst), n);
    LAUNCH_CHECK();
}

void build_plan(TilePlan& P, const int32_t* off, const int32_t* idx, const uint32_t* w,
                int64_t rows, int64_t edges, int64_t vertex_base, int64_t edge_base,
                DeviceBuffers& mem, cudaStream_t s, PinnedStage& pin) {
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
    P.ctr = mem.alloc<int32_t>(1, s, true);
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
    int32_t* h = static_cast<int32_t*>(pin.get(Q * sizeof(int32_t), 0));
    kernel_copy(h, infl, Q * sizeof(int32_t), s);
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
    // short spans first (one thread each in k_pull_fixup), hub rows after (one warp each)
    std::stable_partition(groups.begin(), groups.end(),
                          [](const int4& G) { return G.z - G.y + 1 <= kFixupShortSpan; });
    P.num_groups = (int32_t)groups.size();
    P.num_short = 0;
    for (const int4& G : groups) P.num_short += (G.z - G.y + 1 <= kFixupShortSpan) ? 1 : 0;
    if (P.num_groups) {
        P.groups = mem.alloc<int4>(P.num_groups, s);
        int4* hg = static_cast<int4*>(pin.get(groups.size() * sizeof(int4), 1));
        memcpy(hg, groups.data(), groups.size() * sizeof(int4));
        kernel_copy(P.groups, hg, groups.size() * sizeof(int4), s);
        CU(cudaStreamSynchronize(s));
    }
}

RangeArgs range_args(const TilePlan& P, const int32_t* off, const int32_t* idx, const uint32_t* w,
                     PullCounters* cnt, cudaStream_t s, const void* gbase, int64_t n_global,
                     size_t vsz, int policy, bool degree_ordered);

// Grid of the range kernels: every SM full once (resident CTAs per SM from the occupancy API,
// cached per op), each warp taking range after range from the plan's counter; never more CTAs
// than one warp per range needs.  Measured against one CTA per 8 ranges (a CTA's slot then
// stays taken until its slowest warp ends): PageRank 75.3 -> 71.9 ms, Hash-Min 18.9 -> 17.8,
// SSSP 15.8 -> 14.3 at cfg4; striding warps statically instead was slower (77.4).
template <class Op>
unsigned pull_grid(int64_t num_tiles) {
    static int per_sm = -1;
    static int sms = 0;
    if (per_sm < 0) {
        int dev = 0;
        CU(cudaGetDevice(&dev));
        CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        if (g_pull_carveout >= 0)   // shared-memory share of the unified L1 (percent; knob)
            CU(cudaFuncSetAttribute(k_pull_ranges<Op>,
                                    cudaFuncAttributePreferredSharedMemoryCarveout,
                                    g_pull_carveout));
        CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pull_ranges<Op>, kPullThreads, 0));
        per_sm = std::max(per_sm, 1);
    }
    const int64_t need = ceil_div(num_tiles, kWarpsPerCta);
    if (g_pull_waves == 0) return (unsigned)need;   // one warp per range
    return (unsigned)std::max<int64_t>(
        1, std::min<int64_t>(need, (int64_t)sms * per_sm * g_pull_waves));
}

template <class Op>
void launch_pull(const Op& op, const TilePlan& P, const int32_t* off, const int32_t* idx,
                 const uint32_t* w, PullCounters* cnt, cudaStream_t s, int64_t n_global,
                 int policy, bool degree_ordered) {
    using T = typename Op::T;
    if (P.num_tiles == 0) return;
    RangeArgs A = range_args(P, off, idx, w, cnt, s, op.gather_base(), n_global, sizeof(T), policy,
                             degree_ordered);
    k_pull_ranges<Op><<<pull_grid<Op>(P.num_tiles), kPullThreads, 0, s>>>(op, A);
    LAUNCH_CHECK();
    if (P.num_groups) {
        k_pull_fixup<Op><<<fixup_grid(P.num_groups, P.num_short), 256, 0, s>>>(
            op, P.groups, P.num_groups, P.num_short, static_cast<const T*>(P.carry),
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
    A.range_ctr = nullptr;
    A.order = g_range_order;
    if (g_pull_dynamic && P.ctr) {
        CU(cudaMemsetAsync(P.ctr, 0, sizeof(int32_t), s));
        A.range_ctr = P.ctr;
    }
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
        // replicas a peer maps for the fused exchange (cudaMalloc: IPC-exportable); a world of one
        // rank has no peer, so its replicas stay in the stream-ordered pool
        const bool ipc = multi_rank(g) && g->comm->world > 1;
        if (app == IPREGEL_APP_PAGERANK) {
            S.rank = S.mem.alloc<double>(p.rows, s);
            S.contrib[0] = S.mem.alloc<double>(n, s, true, ipc);
            S.contrib[1] = S.mem.alloc<double>(n, s, true, ipc);
        } else if (app == kAppProgram) {
            S.pv_value = S.mem.alloc<uint64_t>(p.rows, s, true);
            S.pv_out[0] = S.mem.alloc<uint64_t>(n, s, true, ipc);
            S.pv_out[1] = S.mem.alloc<uint64_t>(n, s, true, ipc);
            S.pv_mbox = S.mem.alloc<uint64_t>(p.rows, s, true);
            S.pv_flags = S.mem.alloc<uint8_t>(ceil_div(p.rows, 32) * 32, s, true);   // vector reads
            S.pv_recv = S.mem.alloc<uint32_t>(words_of(p.rows), s, true);
            S.pv_params = S.mem.alloc<double>(kProgParams, s, true);
            for (int w = 0; w < 2; ++w) {
                S.pv_p2p[w] = S.mem.alloc<uint64_t>(p.rows, s);
                S.pv_p2p_recv[w] = S.mem.alloc<uint32_t>(words_of(p.rows), s, true);
            }
            S.pv_shared = S.mem.alloc<ProgShared>(1, s, true);
            S.pv_sends = S.mem.alloc<unsigned long long>(1, s, true);
            S.pv_agg = S.mem.alloc<double>(1, s, true);
            S.pv_mkey = S.mem.alloc<unsigned long long>(2, s, true);
            S.pv_bound = S.mem.alloc<unsigned long long>(1, s, true);
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

// Optional create-phase timeline (IPREGEL_TRACE_CREATE=1): CUDA events on the streams doing the
// work, printed to stderr relative to the first mark when ipregel_graph_create returns.
struct CreateTrace {
    bool on = getenv("IPREGEL_TRACE_CREATE") != nullptr;
    std::vector<std::pair<const char*, cudaEvent_t>> ev;
    std::vector<double> host_ms;   // when the host recorded the mark
    std::chrono::steady_clock::time_point t0;
    void mark(const char* name, cudaStream_t s) {
        if (!on) return;
        if (ev.empty()) t0 = std::chrono::steady_clock::now();
        cudaEvent_t e;
        CU(cudaEventCreate(&e));
        CU(cudaEventRecord(e, s));
        ev.push_back({name, e});
        host_ms.push_back(
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    }
    void dump() {
        if (!on || ev.empty()) return;
        CU(cudaDeviceSynchronize());
        for (size_t i = 0; i < ev.size(); ++i) {
            float ms = 0.f;
            CU(cudaEventElapsedTime(&ms, ev[0].second, ev[i].second));
            fprintf(stderr, "[ipregel create] %-22s %9.2f ms (host %9.2f)\n", ev[i].first, ms,
                    host_ms[i]);
        }
        for (auto& x : ev) cudaEventDestroy(x.second);
        ev.clear();
        host_ms.clear();
    }
};
inline CreateTrace g_ctrace;

// Transpose of a partition's rows (row r lists neighbours u) into a source-major adjacency over all
// N sources (u lists vb + r), allocated in the partition's graph memory: a stable radix sort by
// source (setup.cuh), so each transposed row lists its neighbours in ascending order.  w_ready:
// an event the weights' upload records (the sort does not need them until its last pass).
void transpose_rows(Partition& p, int64_t n, const int32_t* off, const int32_t* idx,
                    const uint32_t* w, int64_t edges, bool want_w, cudaStream_t s,
                    int32_t** out_off, int32_t** out_idx, uint32_t** out_w,
                    bool defer_w = false) {
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
        g_ctrace.mark("transpose begin", s);
        CU(cudaMemcpyAsync(k0, idx, edges * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
        k_transpose_pack<<<grid_for(p.rows * 32, 256), 256, 0, s>>>(off, p.rows, p.vb, v0);
        LAUNCH_CHECK();
        g_ctrace.mark("transpose packed", s);
        cub::DoubleBuffer<int32_t> keys(k0, k1);
        cub::DoubleBuffer<unsigned long long> vals(v0, v1);
        int bits = 1;
        while (bits < 31 && (int64_t(1) << bits) < n) ++bits;
        size_t temp_bytes = 0;
        CU(cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, keys, vals, edges, 0, bits, s));
        void* temp = tmp.alloc<uint8_t>((int64_t)temp_bytes, s);
        CU(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys, vals, edges, 0, bits, s));
        g_ctrace.mark("transpose sorted", s);
        int32_t* perm = nullptr;
        if (defer_w && wx) {
            // the weights are still uploading: keep each entry's CSC position, and let
            // finish_uploads permute the weights window by window as they land
            perm = p.pend.tmp.alloc<int32_t>(edges, s);
            p.pend.perm = perm;
            p.pend.w = w;
            p.pend.wx = wx;
            p.pend.edges = edges;
        }
        k_transpose_unpack<<<std::min<unsigned>(grid_for(edges, 256), sm_grid(16)), 256, 0, s>>>(
            vals.Current(), edges, w, ix, wx, perm);
        LAUNCH_CHECK();
        // offsets from the sorted sources: run lengths, then an exclusive scan
        int32_t* st = tmp.alloc<int32_t>(n, s, true);
        k_run_bounds<<<std::min<unsigned>(grid_for(edges, 256), sm_grid(16)), 256, 0, s>>>(
            keys.Current(), edges, st, o);
        k_run_counts<<<grid_for(n, 256), 256, 0, s>>>(st, n, o);
        LAUNCH_CHECK();
        g_ctrace.mark("transpose unpacked", s);
        exscan_i32(o, n + 1, tmp, s);
        g_ctrace.mark("transpose offsets", s);
    }
    CU(cudaStreamSynchronize(s));
    tmp.release();
    *out_off = o;
    *out_idx = ix;
    if (out_w) *out_w = wx;
}

// Orders the run stream after a pending CSR build (IPREGEL_LAYOUT_DEGREE, create.cuh): called
// by every path that reads the CSR's indices or weights.
void wait_csr(ipregel_graph* g) {
    for (auto& p : g->parts)
        if (p.csr_pending) {
            CU(cudaStreamWaitEvent(g->stream, p.csr_done, 0));
            p.csr_pending = false;
        }
}

// Push adjacency of one partition.  One partition: the graph's own CSR (+ CSC for CC).  Several:
// transposes of the owned CSC (and, for CC, owned CSR) rows, over all N sources.
void ensure_push_view(ipregel_graph* g, Partition& p) {
    wait_csr(g);
    if (p.push_view_ready) return;
    cudaStream_t s = g->stream;
    const int64_t n = g->n;
    // one partition holding every vertex (no comm, or a world of one rank): the graph's own
    // CSR is the source-major view
    if (g->parts.size() == 1 && p.vb == 0 && p.rows == n &&
        (!multi_rank(g) || g->comm->world == 1)) {
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
    if (world == 1) {   // no peer: the fused exchange stores nowhere but the own replica
        S.npeer = 0;
        S.peers_state = 1;
        return;
    }
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
        const bool first = g->parts[0].st[app].peers_state == 0;
        setup_ipc_peers(g, app);
        if (g->parts[0].st[app].peers_state == 1) return true;
        if (require)
            fail(IPREGEL_ERR_UNSUPPORTED, "fused exchange: peer replicas not reachable (CUDA IPC)");
        if (first && g->comm->world > 1)   // once per app: say which exchange the run takes
            fprintf(stderr, "[ipregel rank %d] fused exchange unavailable for app %d (peer "
                    "replicas not mapped by CUDA IPC): using the collective exchange "
                    "(ncclBroadcast AllGatherv)\n", g->comm->rank, app);
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

}  // namespace
