// paper_2010_08781_b200/csrc/program.cuh -- user vertex programs.
//
// The paper's programming model: the user writes compute() and combine() and the framework runs
// the BSP supersteps (Fig. 1; the services of Fig. 2, :102-113).  Device
// code cannot cross the C ABI at run time, so a user program is CUDA C++ source compiled by NVRTC
// for sm_100a together with THIS header (ipregel_program_create), and the kernels below are
// instantiated on it.  They are the same superstep machinery as the paper's three programs:
//   - pull: k_pull_ranges / k_pull_fixup of pull.cuh with ProgPull as the op (merge-path warp
//     ranges; the recipient compute runs in the epilogue);
//   - push: expand_edges of push.cuh with an atomic combine into a single-slot mailbox
//     (PAPER.md:195-197, :205-211), then k_prog_apply runs compute on the recipients and on the
//     vertices that did not vote to halt (naive selection = bypass).
//
// Contract for a program (values, messages and mailboxes have one type V = u32 or f64):
//   unsigned ipr_init(const ipr_ctx&, V* value, V* message)          superstep 0
//   unsigned ipr_compute(const ipr_ctx&, V* value, V mailbox, V* message)
//       mailbox = the combiner's fold of the messages received (its identity if none: the
//       fold the paper's programs do themselves, Figs. 8-10 `while (ip_get_next_message)`);
//       returns IPR_BROADCAST (send *message to every out-neighbour) and/or
//       IPR_STAY_ACTIVE (do not vote to halt).
//   V ipr_edge(V message, unsigned weight)   the message as it travels along one edge (weight
//       1 when the graph has none); must map the combiner's identity to itself.
// Selection (reading R28): push supersteps run compute exactly on the recipients and
// the active vertices; pull supersteps run it on every vertex, with the identity as mailbox for
// the ones that received nothing, so a halted vertex given the identity must leave its value
// unchanged and not broadcast (true of Figs. 8-10 and of any "improve, then broadcast"
// program) -- the pull-all equivalence E1 of SURVEY.md 8(c).
#pragma once
#include "common.cuh"
#include "pull.cuh"
#include "push.cuh"

namespace ipr {

constexpr unsigned kProgBroadcast = 1u;
constexpr unsigned kProgStayActive = 2u;
constexpr int kProgParams = 8;

// What compute() sees of its vertex (Fig. 2's services).
struct ProgCtx {
    int64_t id;            // vertex id (the ORIGINAL id under a relabelled layout)
    int64_t num_vertices;  // N
    uint32_t superstep;
    int32_t out_degree;    // out-neighbours
    int32_t in_degree;     // in-neighbours
    int32_t reserved;
    const double* params;  // the run's program parameters [8]
};

// Kernel parameter block; its layout does not depend on the program.
template <class V>
struct ProgArgs {
    V* value;              // owned values [rows]
    const V* out_cur;      // outbox replica read this superstep [N] (identity = no broadcast)
    V* out_next;           // outbox replica written this superstep [N]
    PeerSlots<V> peers;    // fused exchange of out_next
    V* mbox;               // owned mailboxes [rows] (push accumulators; symmetric pull part 1)
    uint8_t* flags;        // owned, per vertex: bit 0 broadcast this superstep, bit 1 active
    uint32_t* recv;        // owned recipient bitmap (push)
    const int32_t* out_off;
    const int32_t* in_off;
    const int32_t* ids;    // internal -> original id, or NULL
    const double* params;  // device [kProgParams]
    int64_t vbase, rows, n;
    uint32_t superstep;
    int32_t sym;
};

// ---- combiners (commutative and associative) -----------------------------------
template <class V, int kComb> struct ProgComb;
template <> struct ProgComb<uint32_t, 0> {   // SUM (mod 2^32)
    __device__ static uint32_t identity() { return 0u; }
    __device__ static uint32_t combine(uint32_t a, uint32_t b) { return a + b; }
    __device__ static void atomic(uint32_t* p, uint32_t v) { atomicAdd(p, v); }
};
template <> struct ProgComb<uint32_t, 1> {   // MIN
    __device__ static uint32_t identity() { return 0xFFFFFFFFu; }
    __device__ static uint32_t combine(uint32_t a, uint32_t b) { return b < a ? b : a; }
    __device__ static void atomic(uint32_t* p, uint32_t v) { if (v < *p) atomicMin(p, v); }
};
template <> struct ProgComb<uint32_t, 2> {   // MAX
    __device__ static uint32_t identity() { return 0u; }
    __device__ static uint32_t combine(uint32_t a, uint32_t b) { return b > a ? b : a; }
    __device__ static void atomic(uint32_t* p, uint32_t v) { if (v > *p) atomicMax(p, v); }
};
template <> struct ProgComb<double, 0> {     // SUM
    __device__ static double identity() { return 0.0; }
    __device__ static double combine(double a, double b) { return __dadd_rn(a, b); }
    __device__ static void atomic(double* p, double v) { atomicAdd(p, v); }
};
__device__ __forceinline__ void atomic_f64_select(double* p, double v, bool want_min) {
    unsigned long long* q = reinterpret_cast<unsigned long long*>(p);
    unsigned long long old = *q;
    while (true) {
        const double cur = __longlong_as_double((long long)old);
        if (want_min ? !(v < cur) : !(v > cur)) return;
        const unsigned long long seen =
            atomicCAS(q, old, (unsigned long long)__double_as_longlong(v));
        if (seen == old) return;
        old = seen;
    }
}
template <> struct ProgComb<double, 1> {     // MIN
    __device__ static double identity() { return __longlong_as_double(0x7FF0000000000000LL); }
    __device__ static double combine(double a, double b) { return b < a ? b : a; }
    __device__ static void atomic(double* p, double v) { atomic_f64_select(p, v, true); }
};
template <> struct ProgComb<double, 2> {     // MAX
    __device__ static double identity() { return __longlong_as_double((long long)0xFFF0000000000000ULL); }
    __device__ static double combine(double a, double b) { return b > a ? b : a; }
    __device__ static void atomic(double* p, double v) { atomic_f64_select(p, v, false); }
};

template <class V>
__device__ __forceinline__ ProgCtx prog_ctx(const ProgArgs<V>& A, int64_t row) {
    ProgCtx x;
    const int64_t v = A.vbase + row;
    x.id = A.ids ? (int64_t)A.ids[v] : v;
    x.num_vertices = A.n;
    x.superstep = A.superstep;
    x.out_degree = A.out_off[row + 1] - A.out_off[row];
    x.in_degree = A.in_off[row + 1] - A.in_off[row];
    x.reserved = 0;
    x.params = A.params;
    return x;
}

// Record what one vertex did: outbox slot (identity unless it broadcast), bitmap, counters.
template <class P>
__device__ __forceinline__ void prog_emit(const ProgArgs<typename P::V>& A, int64_t row,
                                          const ProgCtx& x, unsigned f, typename P::V msg,
                                          LaneCounters& c) {
    using V = typename P::V;
    using C = ProgComb<V, P::kCombiner>;
    const bool b = (f & kProgBroadcast) != 0;
    const V ob = b ? msg : C::identity();
    A.out_next[A.vbase + row] = ob;
    A.peers.store(A.vbase + row, ob);
    const bool act = (f & kProgStayActive) != 0;
    A.flags[row] = (uint8_t)((b ? 1u : 0u) | (act ? 2u : 0u));   // plain store, no atomics
    if (b) {
        c.changed += 1;
        c.messages += (uint32_t)x.out_degree + (A.sym ? (uint32_t)x.in_degree : 0u);
    }
    c.aux += act ? 1ull : 0ull;
}

template <class P>
__device__ __forceinline__ void prog_vertex(const ProgArgs<typename P::V>& A, int64_t row,
                                            typename P::V mailbox, LaneCounters& c) {
    using V = typename P::V;
    using C = ProgComb<V, P::kCombiner>;
    const ProgCtx x = prog_ctx(A, row);
    V val = A.value[row];
    V msg = C::identity();
    const unsigned f = P::compute(x, &val, mailbox, &msg);
    A.value[row] = val;
    prog_emit<P>(A, row, x, f, msg, c);
}

// ---- superstep 0 -----------------------------------------------------------------------------
template <class P>
__global__ void __launch_bounds__(256) k_prog_init(ProgArgs<typename P::V> A,
                                                   PullCounters* counters) {
    using V = typename P::V;
    using C = ProgComb<V, P::kCombiner>;
    __shared__ unsigned long long s_cnt[4];
    if (threadIdx.x < 4) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    LaneCounters c{};
    const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (row < A.rows) {
        const ProgCtx x = prog_ctx(A, row);
        V val = C::identity();
        V msg = C::identity();
        const unsigned f = P::init(x, &val, &msg);
        A.value[row] = val;
        A.mbox[row] = C::identity();
        prog_emit<P>(A, row, x, f, msg, c);
    }
    flush_counters(c, s_cnt, counters);
}

// ---- pull: the op of pull.cuh's range kernels ------------------------------------------------
// kPass 0: directed graph (CSC: in-neighbours), then compute.  kPass 1: symmetric, first half
// (CSC) into the mailbox.  kPass 2: symmetric, second half (CSR: out-neighbours) folded with the
// mailbox, then compute.
template <class P, int kPass>
struct ProgPull : ProgArgs<typename P::V> {
    using T = typename P::V;
    using C = ProgComb<T, P::kCombiner>;
    static constexpr bool kWeighted = true;
    static constexpr bool kAbsorbing = false;
    __device__ static T identity() { return C::identity(); }
    __device__ static T combine(T a, T b) { return C::combine(a, b); }
    __device__ const T* gptr() const { return this->out_cur; }
    __device__ bool absorbed(int32_t) const { return false; }
    __device__ static T message(T g, uint32_t w) { return P::edge(g, w); }
    __device__ void finish(int32_t row, T m, LaneCounters& c) const {
        if (kPass == 1) {
            this->mbox[row] = m;
            return;
        }
        if (kPass == 2) {
            m = C::combine(this->mbox[row], m);
            this->mbox[row] = C::identity();
        }
        prog_vertex<P>(*this, row, m, c);
    }
};

// ---- push ---------------------------------------------------------------------------------------
template <class P>
struct ProgDeliver {
    using V = typename P::V;
    const V* out_cur;
    V* mbox;
    uint32_t* recv;
    int64_t vbase;
    __device__ __forceinline__ void operator()(int32_t u, uint32_t, int32_t v, uint32_t w) const {
        const int64_t lv = (int64_t)v - vbase;
        ProgComb<V, P::kCombiner>::atomic(mbox + lv, P::edge(out_cur[u], w));
        const uint32_t bit = 1u << (lv & 31);
        if (!(recv[lv >> 5] & bit)) atomicOr(recv + (lv >> 5), bit);
    }
};

template <class P>
__global__ void __launch_bounds__(kExpandThreads)
k_prog_expand(PushAdj adj, const int32_t* __restrict__ e_id, const long long* __restrict__ e_pre,
              const unsigned long long* __restrict__ len, const unsigned long long* __restrict__ edges,
              ProgArgs<typename P::V> A) {
    expand_edges(adj, e_id, nullptr, e_pre, len, edges,
                 ProgDeliver<P>{A.out_cur, A.mbox, A.recv, A.vbase});
}

// After the expansion: compute on recipients and active vertices (naive selection, PAPER.md:
// 171-175, which here equals the bypass list plus the non-halted), reset their mailboxes.
template <class P>
__global__ void __launch_bounds__(256) k_prog_apply(ProgArgs<typename P::V> A,
                                                    PullCounters* counters) {
    using V = typename P::V;
    using C = ProgComb<V, P::kCombiner>;
    __shared__ unsigned long long s_cnt[4];
    if (threadIdx.x < 4) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    LaneCounters c{};
    const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool got = false;
    if (row < A.rows) {
        got = (A.recv[row >> 5] >> (row & 31)) & 1u;
        if (got || (A.flags[row] & 2u)) {
            const V m = A.mbox[row];
            A.mbox[row] = C::identity();
            prog_vertex<P>(A, row, m, c);
        } else {
            A.out_next[A.vbase + row] = C::identity();
            A.peers.store(A.vbase + row, C::identity());
            A.flags[row] = 0;
        }
    }
    __syncwarp();
    if (row < A.rows && (row & 31) == 0) A.recv[row >> 5] = 0u;
    flush_counters(c, s_cnt, counters);
}

}  // namespace ipr
