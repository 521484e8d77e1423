/*
 * include/ipregel.h -- C ABI of the B200-native iPregel superstep library
 * (libipregel.so, built from paper_2010_08781_b200/csrc/).
 *
 * What it computes.  iPregel's synchronous vertex-centric superstep
 * (Sec. 4.2, Fig. 3): every active vertex runs compute(),
 * sends one message per out-edge (a broadcast), messages are
 * folded at the recipient by the program's combiner into a single-slot
 * mailbox (Sec. 4.3.3), and vertices that voted to halt are
 * skipped via selection bypass (Sec. 4.3.1).  The vertex
 * programs are the paper's three benchmarks (Sec. 6): PageRank (Fig. 8,
 * PAPER.md:276-298), Hash-Min connected components (Fig. 9, :332-350) and
 * single-source shortest paths (Fig. 10, :372-396, generalised to uint32
 * edge weights; weights == NULL is exactly Fig. 10's "+1").
 *
 * A user program is the pair (compute, combine) of Fig. 1 (PAPER.md:94-100,
 * :131).  Device code cannot cross a C ABI at run time, so compute is chosen
 * by `ipregel_app` and the combiner is passed and validated against it
 * (PageRank: SUM; CC and SSSP: MIN).  The paper's compile-time optimisation
 * flags (push/pull) become `ipregel_mode`.
 *
 * Conventions for every entry point:
 *   - Returns an ipregel_status.  Nothing aborts, throws or exits.  A
 *     thread-local message describing the last failure is available from
 *     ipregel_last_error().
 *   - Pointers are plain host or device pointers as stated per argument.
 *     Device pointers must be addresses in the current CUDA device's memory
 *     (any allocator: cudaMalloc, PyTorch's caching allocator, ...).
 *   - `stream` arguments are a cudaStream_t passed as void* (NULL = the
 *     legacy default stream).  All device work of a graph handle runs on the
 *     stream it was created with.
 *   - A CUDA or NCCL failure poisons the handle: later calls on it return
 *     IPREGEL_ERR_STATE.  Only ipregel_graph_destroy remains valid.
 *   - One host thread at a time per handle.
 *   - Library-owned device memory comes from the device's default stream-ordered pool
 *     (cudaMallocAsync); freed memory is kept for later graphs up to IPREGEL_POOL_RETAIN_BYTES
 *     (environment, default 144 GiB), so creating and destroying graphs stays cheap.
 */
#ifndef IPREGEL_H
#define IPREGEL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IPREGEL_ABI_VERSION 1

typedef enum {
    IPREGEL_OK = 0,
    IPREGEL_ERR_INVALID_ARGUMENT = 1, /* NULL required pointer, sizes out of range, app/combiner
                                         mismatch, source >= N, out_bytes mismatch,
                                         max_supersteps == 0, unknown enum                      */
    IPREGEL_ERR_INVALID_GRAPH = 2,    /* validate != 0 and: offsets[0] != 0, offsets not
                                         monotone, offsets[rows] != edge count, an index
                                         outside [0, N)                                         */
    IPREGEL_ERR_OUT_OF_MEMORY = 3,    /* device or host allocation failed; nothing leaked      */
    IPREGEL_ERR_CUDA = 4,             /* a CUDA call failed; the handle is poisoned             */
    IPREGEL_ERR_NCCL = 5,             /* an NCCL call failed; the handle is poisoned            */
    IPREGEL_ERR_MAX_SUPERSTEPS = 6,   /* the superstep guard stopped a run that had more work;
                                         values/stats hold the state after the last executed
                                         superstep                            */
    IPREGEL_ERR_STATE = 7,            /* call order violated (get_values before a run,
                                         use after poison, comm/graph mismatch)                 */
    IPREGEL_ERR_UNSUPPORTED = 8       /* device is not sm_100, size beyond int32 indexing,
                                         NCCL unavailable, mode not available for the app       */
} ipregel_status;

/* The vertex programs of PAPER.md Sec. 6 (Figs. 8, 9, 10). */
typedef enum {
    IPREGEL_APP_PAGERANK = 0,   /* values: double[N]   -- ranks after superstep k              */
    IPREGEL_APP_HASHMIN_CC = 1, /* values: uint32_t[N] -- min vertex id of the component in the
                                   symmetrised graph (every edge taken in both directions)     */
    IPREGEL_APP_SSSP = 2        /* values: uint32_t[N] -- distance from the source,
                                   IPREGEL_INF (0xFFFFFFFF) if unreachable; sums saturate      */
} ipregel_app;

/* Fig. 1's combine: Fig. 8 sums; Fig. 5 keeps the minimum (:213-221).  MAX is
 * available to user programs (ipregel_program_desc). */
typedef enum { IPREGEL_COMBINE_SUM = 0, IPREGEL_COMBINE_MIN = 1, IPREGEL_COMBINE_MAX = 2 } ipregel_combiner;

/* Message delivery (Sec. 4.3.2).  PULL: every recipient gathers from its
 * in-neighbours' outboxes (CSC gather-combine).  PUSH: every sender in the frontier folds its
 * message into the recipient's slot with a lock-free atomic combine (the optimisation the paper
 * leaves as future work).  AUTO: per superstep, push when the previous
 * superstep sent few messages, else pull (Ligra's switch the paper names). */
typedef enum { IPREGEL_MODE_AUTO = 0, IPREGEL_MODE_PULL = 1, IPREGEL_MODE_PUSH = 2 } ipregel_mode;

/* Where the arrays of an ipregel_graph_desc live. */
typedef enum {
    IPREGEL_MEMORY_DEVICE = 0, /* device pointers, BORROWED: must stay valid and unmodified until
                                  ipregel_graph_destroy; no copy is made                         */
    IPREGEL_MEMORY_HOST = 1    /* host pointers (pinned or pageable): copied into library-owned
                                  device memory during ipregel_graph_create                       */
} ipregel_memory;

#define IPREGEL_INF 0xFFFFFFFFu

typedef struct ipregel_graph ipregel_graph; /* opaque */
typedef struct ipregel_program ipregel_program; /* opaque: a compiled user vertex program */
typedef struct ipregel_comm ipregel_comm;   /* opaque; NULL means a single GPU */

/*
 * One partition of a directed graph with N vertices and E edges (self-loops are allowed but the
 * fixtures remove them; duplicate edges are kept and count with multiplicity).  A partition owns
 * the destination range [vertex_begin, vertex_end) (1D destination partition; on one GPU the
 * whole range [0, N)).  All offsets are int32 and REBASED to the partition: offsets[0] == 0,
 * offsets[rows] == number of stored edges, rows = vertex_end - vertex_begin.  All indices are
 * GLOBAL vertex ids in [0, N).
 *
 *   csc_*: in-edges of the owned vertices ("CSC", the in-adjacency of PAPER.md:123).  Row r
 *          lists the sources u of edges (u -> vertex_begin + r).  Required.
 *   csr_*: out-edges of the owned vertices (the out-adjacency).  Row r lists the destinations v
 *          of edges (vertex_begin + r -> v).  Out-degrees come from it (PageRank's r/outdeg,
 *          messages counters), Hash-Min CC gathers over it (the reverse direction of the
 *          symmetrised graph) and push mode expands over it.  If csr_offsets, csr_indices and
 *          csr_weights are ALL NULL, the library derives the out-adjacency (and its weights) by
 *          transposing the CSC on the device during create (library-owned memory; the order of
 *          neighbours inside a derived row is unspecified).  Only for a graph held whole in one
 *          partition (vertex range [0, N), csc_edges == num_edges), else UNSUPPORTED.
 *   *_weights: uint32 weight per stored edge, aligned with *_indices, used by SSSP only; NULL
 *          means every weight is 1.  csc_weights and csr_weights must both be NULL or both set.
 */
typedef struct {
    int64_t num_vertices;       /* N, 1 <= N <= 2^31 - 1                                        */
    int64_t num_edges;          /* E, global                                                    */
    int64_t vertex_begin;       /* owned destination range                                      */
    int64_t vertex_end;
    int64_t csc_edges;          /* edges stored in this partition's csc_* arrays                */
    int64_t csr_edges;          /* edges stored in this partition's csr_* arrays                */
    const int32_t* csc_offsets; /* [rows + 1]                                                   */
    const int32_t* csc_indices; /* [csc_edges]                                                  */
    const uint32_t* csc_weights;/* [csc_edges] or NULL                                          */
    const int32_t* csr_offsets; /* [rows + 1]                                                   */
    const int32_t* csr_indices; /* [csr_edges]                                                  */
    const uint32_t* csr_weights;/* [csr_edges] or NULL                                          */
    int32_t memory;             /* ipregel_memory                                               */
    int32_t validate;           /* 1: O(E) device validation during create (INVALID_GRAPH)      */
    /* Optional internal vertex layout.  vertex_ids[v] = ORIGINAL id of internal vertex v (a
     * permutation of [0, N), the full array on every partition; device or host per `memory`), or
     * NULL for the identity.  With it, Hash-Min labels are original ids, sssp_source is an
     * original id and ipregel_get_values returns values indexed by original id, so results equal
     * those on the original numbering (the layout only changes memory locality).            */
    const int32_t* vertex_ids;
    /* 1: internal ids ascend by decreasing out-degree (e.g. vertex_ids from a degree sort).  The
     * pull gathers then keep the hot prefix of the outbox arrays L2-resident (evict-last address
     * range policy) and stream the rest.                                                       */
    int32_t degree_ordered;
    /* ipregel_layout.  IPREGEL_LAYOUT_AS_GIVEN (0): the arrays are used in the given numbering.
     * IPREGEL_LAYOUT_DEGREE (1): the LIBRARY relabels the graph during create -- internal ids
     * ascend by decreasing out-degree (ties by original id), the in-adjacency is rebuilt in
     * library-owned memory with every row's sources in ascending internal order (above 2^20
     * vertices: ascending by a monotone class of the internal id -- exact for the low, hot ids,
     * the top bit and the 40 - 5 - ceil(log2 N) bits below it for the others), and the
     * out-adjacency is derived from it (csr_* may be NULL; if given, only its offsets are read,
     * for the out-degrees).  The layout is what makes the hot senders' outbox values a
     * contiguous, cache-resident prefix (the bandwidth pressure of PAPER.md:169); results, the
     * SSSP source and program ids stay ORIGINAL ids, exactly as with vertex_ids.  Requires
     * vertex_ids == NULL, degree_ordered == 0 and the whole graph in one partition without a
     * communicator (else INVALID_ARGUMENT / UNSUPPORTED).  Cost at BASELINE cfg4 (1.88e9 edges):
     * a degree sort of N keys, a 64-bit radix sort of the E relabelled edges and ~50 GB of
     * temporary device memory during create.                                                   */
    int32_t layout;
} ipregel_graph_desc;

typedef enum { IPREGEL_LAYOUT_AS_GIVEN = 0, IPREGEL_LAYOUT_DEGREE = 1 } ipregel_layout;

typedef struct {
    int32_t mode;                  /* ipregel_mode, default AUTO                                */
    uint32_t pagerank_iterations;  /* k: supersteps that broadcast (Fig. 8's 10); default 10    */
    uint32_t sssp_source;          /* SSSP_SOURCE of Fig. 10; default 0                         */
    float push_fraction;           /* AUTO: push when messages(s-1) < push_fraction * scanned
                                      edges of a pull superstep; default 0.04                  */
    uint32_t flags;                /* IPREGEL_RUN_* bits below; default 0                       */
    double pagerank_tolerance;     /* < 0 (default -1): Fig. 8 exactly, k supersteps.  >= 0: run
                                      to convergence: after each superstep s >= 1
                                      the max over vertices of |r_s(v) - r_{s-1}(v)| is
                                      aggregated (exact max, deterministic) and the run halts
                                      after the first superstep where it is <= tolerance (its
                                      broadcast is not delivered), or after superstep k.  NaN:
                                      INVALID_ARGUMENT.  DESIGN.md reading R27.                */
} ipregel_run_params;

/* Exchange of the broadcast array between partitions after a PULL superstep (ranks of a comm,
 * or loopback partitions).  Default (neither bit): FUSED when every other replica is reachable,
 * else COLLECTIVE.
 *   FUSED: the pull kernel's recipient-compute epilogue stores each owned result into every
 *     replica of the broadcast array (peer GPUs' replicas mapped with CUDA IPC over NVLink /
 *     NVSwitch; the other partitions' replicas in loopback), so the exchange overlaps the
 *     gathers tile by tile; a one-element AllReduce (PageRank) or the counter AllReduce
 *     (CC/SSSP) on the run stream is the superstep barrier.  At most 8 ranks / partitions.
 *     Requires every rank's graph to be destroyed collectively (peers stay mapped until then).
 *   COLLECTIVE: a separate in-place AllGatherv (grouped ncclBroadcast; device copies in
 *     loopback) after the kernel.
 * Push supersteps always exchange the sparse (id, value) frontier through NCCL.  Values are
 * bit-identical either way.  Setting both bits: INVALID_ARGUMENT; FUSED when peers are not
 * reachable: UNSUPPORTED.  The choice is made collectively on the first run of each app. */
#define IPREGEL_RUN_EXCHANGE_COLLECTIVE 0x1u
#define IPREGEL_RUN_EXCHANGE_FUSED 0x2u
/* PageRank (ipregel_run only): after every superstep s, also fold on the device the two sums of
 * the rank mass invariant (Pregel's PageRank):
 *   pagerank_mass[s]    = sum over all vertices of r_s(v)
 *   pagerank_mass_nd[s] = sum over vertices with out-degree > 0 of r_s(v)
 * so that pagerank_mass[s] = 0.15 + 0.85 * pagerank_mass_nd[s-1] (dangling mass is dropped,
 * DESIGN.md R4) can be checked on the GPU's own values.  f64 atomics: the summation order is not
 * deterministic (the values themselves are unaffected).  A diagnostic: off by default (it adds
 * two atomics per warp to every superstep).  Other apps: INVALID_ARGUMENT. */
#define IPREGEL_RUN_PAGERANK_MASS 0x4u

/* Per-superstep record of the last run (index = superstep, 0 = initialisation). */
typedef struct {
    uint32_t capacity;        /* in: length of every non-NULL array below                       */
    uint32_t supersteps;      /* out: supersteps executed (including superstep 0)               */
    int32_t status;           /* out: status of the last run                                    */
    int32_t exchange;         /* out: exchange of the last run's pull supersteps: 0 none (one
                                 partition), 1 COLLECTIVE, 2 FUSED (IPREGEL_RUN_EXCHANGE_*)      */
    float* time_ms;           /* superstep wall time on the stream (kernels + exchange + counters) */
    float* kernel_ms;         /* time of the superstep's main delivery kernel(s) only           */
    uint8_t* mode;            /* 0 init, 1 pull, 2 push                                         */
    uint64_t* changed;        /* vertices that broadcast in the superstep                       */
    uint64_t* messages;       /* messages sent in the superstep (sum of broadcasters' degrees)  */
    uint64_t* edges_scanned;  /* edges the superstep's delivery touched                         */
    uint64_t* model_bytes;    /* algorithmic DRAM bytes of the superstep (DESIGN.md roofline)   */
    double* pagerank_delta;   /* PageRank: max_v |r_s(v) - r_{s-1}(v)| when run to convergence,
                                 else 0                                                         */
    double* pagerank_mass;    /* PageRank with IPREGEL_RUN_PAGERANK_MASS: sum_v r_s(v), else 0  */
    double* pagerank_mass_nd; /*   and sum of r_s(v) over vertices with out-degree > 0          */
    float* part_ms;           /* PageRank pull supersteps: time of the range kernel + fixup alone
                                 (the rest of kernel_ms is the update pass, k_pr_finish); 0 else */
} ipregel_stats;

/* ---- errors / device ---------------------------------------------------------------------- */
const char* ipregel_status_string(ipregel_status status);
const char* ipregel_last_error(void);     /* thread-local, never NULL                          */
int ipregel_abi_version(void);
/* Number of CUDA kernels this library has launched in the process so far (diagnostic). */
uint64_t ipregel_kernel_launches(void);
/* IPREGEL_OK if `device` is an sm_100 (B200-class) GPU, else UNSUPPORTED / CUDA. */
ipregel_status ipregel_device_check(int device);

/* ---- run parameters ----------------------------------------------------------------------- */
/* Writes the defaults listed in ipregel_run_params into *out. */
ipregel_status ipregel_run_params_default(ipregel_run_params* out);

/* ---- multi-GPU (one process per GPU, 1D destination partition) --------------------------- */
/* Rank 0 creates the 128-byte NCCL unique id; the caller ships it to every rank (e.g. a
 * torch.distributed broadcast) -- PyTorch is plumbing, the library owns the communicator. */
ipregel_status ipregel_nccl_unique_id(uint8_t out[128]);
/* Collective over `world` ranks; `device` is this rank's CUDA ordinal. */
ipregel_status ipregel_comm_create(int rank, int world, const uint8_t id[128], int device,
                                   ipregel_comm** out);
void ipregel_comm_destroy(ipregel_comm* comm);

/* Host, deterministic.  cost_prefix[0..n] is a non-decreasing prefix sum of per-vertex cost
 * (cost_prefix[0] == 0).  Writes bounds_out[0..world] with bounds_out[0] = 0,
 * bounds_out[world] = n, non-decreasing, each range's cost as close as possible to
 * cost_prefix[n] * g / world at its left end (binary search, lower bound). */
ipregel_status ipregel_partition(const int64_t* cost_prefix, int64_t n, int world,
                                 int64_t* bounds_out);

/* ---- graph ---------------------------------------------------------------------------------- */
/* Single GPU (comm == NULL, the desc must own [0, N)) or one rank of a multi-GPU run (collective:
 * every rank calls it with its own partition; the ranges must tile [0, N) in rank order). */
ipregel_status ipregel_graph_create(const ipregel_graph_desc* desc, ipregel_comm* comm,
                                    void* stream, ipregel_graph** out);
/* Loopback: `num_partitions` partitions of one graph, all on the current device, exchanging
 * through device copies instead of NCCL (tests the partitioned path on one GPU).  descs[p] must
 * tile [0, N) in order. */
ipregel_status ipregel_graph_create_partitioned(const ipregel_graph_desc* descs,
                                                int num_partitions, void* stream,
                                                ipregel_graph** out);
void ipregel_graph_destroy(ipregel_graph* graph);

/* Device bytes held by the handle: graph-side (copies, tile plans, and once PageRank's pull has
 * run -- or at create for IPREGEL_LAYOUT_DEGREE graphs -- its row-end-flagged copy of the CSC
 * indices, 4 B per edge, with per-row bookkeeping) and vertex state (values,
 * mailboxes/outboxes, frontier).  The vertex state is Theta(N), independent of E
 * (PAPER.md:205-211, :476-480). */
ipregel_status ipregel_memory_footprint(ipregel_graph* graph, uint64_t* graph_bytes,
                                        uint64_t* state_bytes);

/* ---- run ------------------------------------------------------------------------------------ */
/* Runs supersteps 0, 1, ... of `app` until no vertex is active and no message is in flight
 * (PageRank: superstep k is the last; CC/SSSP: until a superstep sends no message), or until
 * `max_supersteps` supersteps (counting superstep 0) have executed while work remains
 * (IPREGEL_ERR_MAX_SUPERSTEPS, state kept).  Host-synchronous.  params may be NULL (defaults).
 * Collective across ranks of a comm. */
ipregel_status ipregel_run(ipregel_graph* graph, ipregel_app app, ipregel_combiner combiner,
                           uint32_t max_supersteps, const ipregel_run_params* params);

/* Copies the full N-vertex result of the last run into `out` (host or device memory per
 * out_is_device).  out_bytes must be N * 8 (PageRank, 8-byte program values) or N * 4 (CC,
 * SSSP, 4-byte program values).  Multi-GPU: every
 * rank receives all N values (collective). */
ipregel_status ipregel_get_values(ipregel_graph* graph, void* out, size_t out_bytes,
                                  int out_is_device);

/* Asynchronous ipregel_get_values into HOST memory: the last run's N values are staged on the
 * device (a private copy, so later runs -- of any app -- do not affect them) and copied to `out`
 * on the library's copy stream while the caller goes on (e.g. with the next run); `out` is
 * complete once ipregel_graph_sync returns (destroy also waits).  `out` should be pinned
 * (cudaHostAlloc / registered); pageable memory makes the copy synchronous.  Same size rules and
 * errors as ipregel_get_values; one GPU or loopback partitions (ranks: UNSUPPORTED). */
ipregel_status ipregel_get_values_async(ipregel_graph* graph, void* out, size_t out_bytes);

/* Waits for every asynchronous copy of the graph (ipregel_get_values_async). */
ipregel_status ipregel_graph_sync(ipregel_graph* graph);

/* Fills the caller-owned arrays of *inout (up to capacity entries) for the last run. */
ipregel_status ipregel_get_stats(ipregel_graph* graph, ipregel_stats* inout);

/* ---- user vertex programs (Fig. 1: the user supplies compute and combine) --------- */
/*
 * A program is CUDA C++ source compiled at run time (NVRTC, sm_100a, IEEE arithmetic as
 * written: no FMA contraction) together with the library's own superstep kernels, which are
 * then instantiated on it (pull: merge-path CSC gather-combine with compute in the epilogue;
 * push: atomic combine into single-slot mailboxes; AUTO switch, fused exchange, partitions and
 * ranks -- everything ipregel_run does).  Values, messages and mailboxes share one type
 * `ipr_value_t` (value_type).  The source must define:
 *
 *   __device__ unsigned ipr_init(const ipr_ctx& c, ipr_value_t* value, ipr_value_t* message);
 *       superstep 0: set *value (and *message); return flags.
 *   __device__ unsigned ipr_compute(const ipr_ctx& c, ipr_value_t* value, ipr_value_t mailbox,
 *                                   ipr_value_t* message);
 *       superstep s >= 1: mailbox = the combiner's fold of the messages received, its identity
 *       if none (SUM 0, MIN the type's max / +inf, MAX 0 / -inf); update *value; return flags.
 *   __device__ ipr_value_t ipr_edge(ipr_value_t message, unsigned weight);
 *       the message as delivered along one edge (weight 1 when the graph has none); must map
 *       the combiner's identity to itself (e.g. SSSP: ipr_sat_add(message, weight)).
 *
 * Flags: IPR_BROADCAST = send *message to every out-neighbour (with symmetric = 1
 * to every in- and out-neighbour); IPR_STAY_ACTIVE = do not vote to halt.
 * ipr_ctx (read-only): id (ORIGINAL vertex id under a relabelled layout), num_vertices,
 * superstep, out_degree, in_degree, params[0..7] (the run's program parameters, 0 if unset),
 * aggregate (the aggregator after the previous superstep; its identity before any fold).
 * Helpers: ipr_sat_add(a, b) (u32, saturating at IPR_INF_U32 = 0xFFFFFFFF).
 * Services (Fig. 2): ipr_send(c, dest, message) -- IP_send_message: a point-to-point message to
 * the ORIGINAL vertex id dest (ignored outside [0, N)), combined into dest's mailbox with the
 * program's combiner and delivered in the next superstep, where dest computes (it counts in
 * `messages`; one GPU: whole graph or loopback partitions; not across ranks: UNSUPPORTED);
 * ipr_aggregate(c, x) -- fold the f64 x into the run's aggregator (desc.aggregator).
 * Optional hint: __device__ bool ipr_absorbing(ipr_value_t value) -- true when a vertex holding
 * `value` ignores every message (e.g. Hash-Min's label 0): pull supersteps then skip gathering
 * its in-edges, and whole merge-path ranges of such vertices (compute still runs, with the
 * identity as mailbox).
 * Optional hint (MIN combiner, no ipr_send): __device__ bool ipr_settled(ipr_value_t value,
 * ipr_value_t bound) -- true when a vertex holding `value` cannot change if every message it
 * receives is >= `bound`.  Defining it asserts that ipr_edge is non-decreasing in both the
 * message and the weight; the library then takes bound = ipr_edge(smallest message broadcast in
 * the previous superstep, smallest edge weight) for each pull superstep and skips the gathers
 * of settled vertices (and, for integer values, of rows whose partial fold is <= bound) --
 * SSSP's "distance <= min frontier distance + min weight" (across ranks the minimum is
 * all-reduced each superstep).
 * The run ends when a superstep has no broadcast and no active vertex.
 * Selection (R28): push supersteps run compute on recipients and active vertices
 * only; pull supersteps run it on every vertex, the non-recipients getting the identity, so a
 * halted vertex given the identity must leave its value and not broadcast (Figs. 8-10 do).
 * The combiner (SUM, MIN, MAX) must be what the program folds with: it is applied in a fixed
 * order in pull mode and by atomics in push mode (SUM f64 in push is order-nondeterministic).
 */
typedef enum {
    IPREGEL_VALUE_U32 = 0, IPREGEL_VALUE_F64 = 1, IPREGEL_VALUE_F32 = 2, IPREGEL_VALUE_I32 = 3,
    IPREGEL_VALUE_U64 = 4, IPREGEL_VALUE_I64 = 5
} ipregel_value_type;   /* ipr_value_t: unsigned int, double, float, int, unsigned long long,
                           long long; values returned as 4- or 8-byte elements */
typedef enum {
    IPREGEL_AGG_NONE = 0, IPREGEL_AGG_SUM = 1, IPREGEL_AGG_MIN = 2, IPREGEL_AGG_MAX = 3
} ipregel_aggregator;

typedef struct {
    const char* source;   /* NUL-terminated CUDA C++ source (copied; the caller keeps ownership) */
    int32_t value_type;   /* ipregel_value_type                                                 */
    int32_t combiner;     /* ipregel_combiner                                                   */
    int32_t symmetric;    /* 1: messages travel along every edge in both directions (Hash-Min's
                             neighbourhood; the graph's CSR row U CSC row), 0: out-edges only   */
    int32_t aggregator;   /* ipregel_aggregator: NONE (0), or SUM / MIN / MAX folding the f64
                             values vertices pass to ipr_aggregate in a superstep; every vertex
                             reads the result as ipr_ctx.aggregate in the next one (Pregel
                             aggregators; SUM's rounding order is not deterministic)           */
    int32_t reserved;     /* must be 0                                                          */
} ipregel_program_desc;

/* Compiles the program (host only; no GPU needed).  A compile error returns INVALID_ARGUMENT
 * with the NVRTC log in ipregel_last_error(); UNSUPPORTED if NVRTC is not installed.  The
 * kernels are loaded on the current device at the first run. */
ipregel_status ipregel_program_create(const ipregel_program_desc* desc, ipregel_program** out);
/* NVRTC log of the successful compile (warnings), never NULL; owned by the program. */
const char* ipregel_program_log(const ipregel_program* program);
/* Size of the compiled sm_100a CUBIN (diagnostic). */
uint64_t ipregel_program_cubin_bytes(const ipregel_program* program);
void ipregel_program_destroy(ipregel_program* program);

/* Runs `program` on the graph like ipregel_run (same params: mode, push_fraction, exchange
 * flags; pagerank_* fields are ignored).  program_params: up to 8 doubles visible as
 * ipr_ctx.params (NULL / 0 = all zero).  ipregel_get_values then returns N values of the
 * program's value_type; ipregel_get_stats the per-superstep record.  Collective across ranks. */
ipregel_status ipregel_run_program(ipregel_graph* graph, ipregel_program* program,
                                   uint32_t max_supersteps, const ipregel_run_params* params,
                                   const double* program_params, int num_program_params);

#ifdef __cplusplus
}
#endif
#endif /* IPREGEL_H */
