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

constexpr int kProgMaxParts = 8;

// Point-to-point messages (Fig. 2's IP_send_message) and the aggregator of a run, one device copy
// per partition.  Messages sent in superstep s go to buffer s & 1 of the OWNER partition of the
// destination (atomic combine into its single-slot mailbox + a recipient bit) and are folded
// into the recipient's mailbox in superstep s + 1.
struct ProgShared {
    int32_t nparts;
    int32_t agg_op;                          // -1 none, else SUM / MIN / MAX (ipregel_combiner)
    int64_t bounds[kProgMaxParts + 1];       // partition p owns [bounds[p], bounds[p + 1])
    void* p2p[2][kProgMaxParts];             // mailboxes [rows_p] (8-byte slots)
    uint32_t* p2p_recv[2][kProgMaxParts];    // recipient bitmaps
    const int32_t* inv_ids;                  // original -> internal id, or NULL
    unsigned long long* sends;               // this partition's point-to-point sends
    double* agg;                             // this partition's aggregator (superstep's fold)
};

// What compute() sees of its vertex (Fig. 2's services).
struct ProgCtx {
    int64_t id;            // vertex id (the ORIGINAL id under a relabelled layout)
    int64_t num_vertices;  // N
    uint32_t superstep;
    int32_t out_degree;    // out-neighbours
    int32_t in_degree;     // in-neighbours
    int32_t wpar;          // point-to-point buffer written this superstep (superstep & 1)
    const double* params;  // the run's program parameters [8]
    double aggregate;      // the aggregator's value after the previous superstep
    const ProgShared* shared;
    mutable double agg_acc;   // this vertex's ipr_aggregate fold (folded into the thread's)
    mutable uint32_t agg_n;
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
    const ProgShared* shared;   // device, this partition's
    void* p2p_in;          // this partition's point-to-point mailboxes read this superstep
    uint32_t* p2p_in_recv; //   and their recipient bitmap (NULL: the program never sends)
    double aggregate;      // the aggregator after the previous superstep
    int32_t agg_op;        // -1 none
    int32_t pull_all;      // k_prog_apply after a pull: every vertex computes
    int64_t vbase, rows, n;
    uint32_t superstep;
    int32_t sym;
    // ipr_settled programs (NULL otherwise): the minimum message broadcast this superstep (order
    // key, folded here) and the bound every message of this superstep is at least (computed by
    // k_prog_bound from the previous superstep's minimum; ~0 = no broadcast at all)
    unsigned long long* mkey_out;
    const unsigned long long* bound;
    uint32_t w_min;        // smallest edge weight (1 without weights)
};

// Order-preserving unsigned keys of the value types (atomicMin over any of them).
template <class V> struct ProgKey;
template <> struct ProgKey<uint32_t> {
    __device__ static unsigned long long key(uint32_t x) { return x; }
    __device__ static uint32_t value(unsigned long long k) { return (uint32_t)k; }
};
template <> struct ProgKey<int32_t> {
    __device__ static unsigned long long key(int32_t x) { return (uint32_t)x ^ 0x80000000u; }
    __device__ static int32_t value(unsigned long long k) { return (int32_t)((uint32_t)k ^ 0x80000000u); }
};
template <> struct ProgKey<uint64_t> {
    __device__ static unsigned long long key(uint64_t x) { return x; }
    __device__ static uint64_t value(unsigned long long k) { return k; }
};
template <> struct ProgKey<int64_t> {
    __device__ static unsigned long long key(int64_t x) { return (unsigned long long)x ^ (1ull << 63); }
    __device__ static int64_t value(unsigned long long k) { return (int64_t)(k ^ (1ull << 63)); }
};
template <> struct ProgKey<float> {
    __device__ static unsigned long long key(float x) {
        const uint32_t b = (uint32_t)__float_as_int(x);
        return (b & 0x80000000u) ? (unsigned long long)(~b) : (unsigned long long)(b | 0x80000000u);
    }
    __device__ static float value(unsigned long long k) {
        const uint32_t b = (uint32_t)k;
        return __int_as_float((int)((b & 0x80000000u) ? (b & 0x7FFFFFFFu) : ~b));
    }
};
template <> struct ProgKey<double> {
    __device__ static unsigned long long key(double x) {
        const unsigned long long b = (unsigned long long)__double_as_longlong(x);
        return (b >> 63) ? ~b : (b | (1ull << 63));
    }
    __device__ static double value(unsigned long long k) {
        return __longlong_as_double((long long)((k >> 63) ? (k & ~(1ull << 63)) : ~k));
    }
};

// warp min of the broadcast keys, one atomic per warp
__device__ __forceinline__ void flush_mkey(unsigned long long k, unsigned long long* out) {
    if (!out) return;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        const unsigned long long o = __shfl_xor_sync(0xFFFFFFFFu, k, d);
        k = o < k ? o : k;
    }
    if ((threadIdx.x & 31) == 0 && k != ~0ull) atomicMin(out, k);
}

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

// f32 / i32 / u64 / i64 values (ipregel_value_type F32, I32, U64, I64)
template <class T>
__device__ __forceinline__ void atomic_select_cas(T* p, T v, bool want_min) {
    static_assert(sizeof(T) == 4 || sizeof(T) == 8, "4- or 8-byte values");
    using U = typename cond_type<sizeof(T) == 8, unsigned long long, unsigned int>::type;
    U* q = reinterpret_cast<U*>(p);
    U old = *q;
    while (true) {
        const T cur = bit_cast<T>(old);
        if (want_min ? !(v < cur) : !(v > cur)) return;
        const U seen = atomicCAS(q, old, bit_cast<U>(v));
        if (seen == old) return;
        old = seen;
    }
}
template <> struct ProgComb<float, 0> {
    __device__ static float identity() { return 0.0f; }
    __device__ static float combine(float a, float b) { return __fadd_rn(a, b); }
    __device__ static void atomic(float* p, float v) { atomicAdd(p, v); }
};
template <> struct ProgComb<float, 1> {
    __device__ static float identity() { return __int_as_float(0x7F800000); }
    __device__ static float combine(float a, float b) { return b < a ? b : a; }
    __device__ static void atomic(float* p, float v) { atomic_select_cas(p, v, true); }
};
template <> struct ProgComb<float, 2> {
    __device__ static float identity() { return __int_as_float((int)0xFF800000u); }
    __device__ static float combine(float a, float b) { return b > a ? b : a; }
    __device__ static void atomic(float* p, float v) { atomic_select_cas(p, v, false); }
};
template <> struct ProgComb<int32_t, 0> {
    __device__ static int32_t identity() { return 0; }
    __device__ static int32_t combine(int32_t a, int32_t b) { return (int32_t)((uint32_t)a + (uint32_t)b); }
    __device__ static void atomic(int32_t* p, int32_t v) { atomicAdd(p, v); }
};
template <> struct ProgComb<int32_t, 1> {
    __device__ static int32_t identity() { return 0x7FFFFFFF; }
    __device__ static int32_t combine(int32_t a, int32_t b) { return b < a ? b : a; }
    __device__ static void atomic(int32_t* p, int32_t v) { if (v < *p) atomicMin(p, v); }
};
template <> struct ProgComb<int32_t, 2> {
    __device__ static int32_t identity() { return (int32_t)0x80000000u; }
    __device__ static int32_t combine(int32_t a, int32_t b) { return b > a ? b : a; }
    __device__ static void atomic(int32_t* p, int32_t v) { if (v > *p) atomicMax(p, v); }
};
template <> struct ProgComb<uint64_t, 0> {
    __device__ static uint64_t identity() { return 0ull; }
    __device__ static uint64_t combine(uint64_t a, uint64_t b) { return a + b; }
    __device__ static void atomic(uint64_t* p, uint64_t v) {
        atomicAdd(reinterpret_cast<unsigned long long*>(p), (unsigned long long)v);
    }
};
template <> struct ProgComb<uint64_t, 1> {
    __device__ static uint64_t identity() { return ~0ull; }
    __device__ static uint64_t combine(uint64_t a, uint64_t b) { return b < a ? b : a; }
    __device__ static void atomic(uint64_t* p, uint64_t v) {
        if (v < *p) atomicMin(reinterpret_cast<unsigned long long*>(p), (unsigned long long)v);
    }
};
template <> struct ProgComb<uint64_t, 2> {
    __device__ static uint64_t identity() { return 0ull; }
    __device__ static uint64_t combine(uint64_t a, uint64_t b) { return b > a ? b : a; }
    __device__ static void atomic(uint64_t* p, uint64_t v) {
        if (v > *p) atomicMax(reinterpret_cast<unsigned long long*>(p), (unsigned long long)v);
    }
};
template <> struct ProgComb<int64_t, 0> {
    __device__ static int64_t identity() { return 0; }
    __device__ static int64_t combine(int64_t a, int64_t b) { return (int64_t)((uint64_t)a + (uint64_t)b); }
    __device__ static void atomic(int64_t* p, int64_t v) {
        atomicAdd(reinterpret_cast<unsigned long long*>(p), (unsigned long long)v);
    }
};
template <> struct ProgComb<int64_t, 1> {
    __device__ static int64_t identity() { return 0x7FFFFFFFFFFFFFFFLL; }
    __device__ static int64_t combine(int64_t a, int64_t b) { return b < a ? b : a; }
    __device__ static void atomic(int64_t* p, int64_t v) {
        if (v < *p) atomicMin(reinterpret_cast<long long*>(p), (long long)v);
    }
};
template <> struct ProgComb<int64_t, 2> {
    __device__ static int64_t identity() { return (int64_t)0x8000000000000000ULL; }
    __device__ static int64_t combine(int64_t a, int64_t b) { return b > a ? b : a; }
    __device__ static void atomic(int64_t* p, int64_t v) {
        if (v > *p) atomicMax(reinterpret_cast<long long*>(p), (long long)v);
    }
};

// The combiner's absorbing element z (combine(z, x) == combine(x, z) == z for every message x)
// of the integer MIN / MAX combiners: once a row's partial mailbox fold reaches z, its remaining
// messages cannot change it, so the pull skips their gathers (exact).  SUM has none; the
// floating-point MIN / MAX are left out (a NaN message would not be absorbed in every order).
template <class V, int kComb> struct ProgAbsorb {
    static constexpr bool kHas = false;
    __device__ static bool is(V) { return false; }
};
template <> struct ProgAbsorb<uint32_t, 1> {
    static constexpr bool kHas = true;
    __device__ static bool is(uint32_t x) { return x == 0u; }
};
template <> struct ProgAbsorb<uint32_t, 2> {
    static constexpr bool kHas = true;
    __device__ static bool is(uint32_t x) { return x == 0xFFFFFFFFu; }
};
template <> struct ProgAbsorb<int32_t, 1> {
    static constexpr bool kHas = true;
    __device__ static bool is(int32_t x) { return x == (int32_t)0x80000000u; }
};
template <> struct ProgAbsorb<int32_t, 2> {
    static constexpr bool kHas = true;
    __device__ static bool is(int32_t x) { return x == (int32_t)0x7FFFFFFF; }
};
template <> struct ProgAbsorb<uint64_t, 1> {
    static constexpr bool kHas = true;
    __device__ static bool is(uint64_t x) { return x == 0ull; }
};
template <> struct ProgAbsorb<uint64_t, 2> {
    static constexpr bool kHas = true;
    __device__ static bool is(uint64_t x) { return x == ~0ull; }
};
template <> struct ProgAbsorb<int64_t, 1> {
    static constexpr bool kHas = true;
    __device__ static bool is(int64_t x) { return x == (int64_t)0x8000000000000000ull; }
};
template <> struct ProgAbsorb<int64_t, 2> {
    static constexpr bool kHas = true;
    __device__ static bool is(int64_t x) { return x == (int64_t)0x7FFFFFFFFFFFFFFFll; }
};

template <class V>
__device__ __forceinline__ ProgCtx prog_ctx(const ProgArgs<V>& A, int64_t row, int32_t out_degree,
                                            int32_t in_degree) {
    ProgCtx x;
    const int64_t v = A.vbase + row;
    x.id = A.ids ? (int64_t)A.ids[v] : v;
    x.num_vertices = A.n;
    x.superstep = A.superstep;
    x.out_degree = out_degree;
    x.in_degree = in_degree;
    x.wpar = (int32_t)(A.superstep & 1u);
    x.params = A.params;
    x.aggregate = A.aggregate;
    x.shared = A.shared;
    x.agg_acc = 0.0;
    x.agg_n = 0u;
    return x;
}
template <class V>
__device__ __forceinline__ ProgCtx prog_ctx(const ProgArgs<V>& A, int64_t row) {
    return prog_ctx(A, row, A.out_off[row + 1] - A.out_off[row], A.in_off[row + 1] - A.in_off[row]);
}

// ---- Fig. 2's IP_send_message and a Pregel aggregator ------------------------------------------
// Point-to-point send of `m` to ORIGINAL vertex id `dest` (ignored if outside [0, N)).
template <class V, int kComb>
__device__ __forceinline__ void prog_send(const ProgCtx& c, long long dest, V m) {
    const ProgShared* S = c.shared;
    if (!S || dest < 0 || dest >= c.num_vertices) return;
    const int64_t v = S->inv_ids ? (int64_t)S->inv_ids[dest] : (int64_t)dest;
    int p = 0;
    while (p + 1 < S->nparts && v >= S->bounds[p + 1]) ++p;
    const int64_t lv = v - S->bounds[p];
    ProgComb<V, kComb>::atomic(static_cast<V*>(S->p2p[c.wpar][p]) + lv, m);
    uint32_t* rb = S->p2p_recv[c.wpar][p];
    const uint32_t bit = 1u << (lv & 31);
    if (!(rb[lv >> 5] & bit)) atomicOr(rb + (lv >> 5), bit);
    atomicAdd(S->sends, 1ull);
}

__device__ __forceinline__ double agg_combine(int op, double a, double b) {
    return op == 0 ? __dadd_rn(a, b) : (op == 1 ? (b < a ? b : a) : (b > a ? b : a));
}

// Fold x into this superstep's aggregator (visible to every vertex as ctx.aggregate in the next
// superstep).
__device__ __forceinline__ void prog_aggregate(const ProgCtx& c, double x) {
    if (!c.shared || c.shared->agg_op < 0) return;
    c.agg_acc = c.agg_n ? agg_combine(c.shared->agg_op, c.agg_acc, x) : x;
    c.agg_n = 1u;
}

__device__ __forceinline__ void agg_atomic(int op, double* p, double v) {
    if (op == 0) atomicAdd(p, v);
    else atomic_f64_select(p, v, op == 1);
}

// End of a kernel: warp-fold the threads' aggregator values, one atomic per warp.
__device__ __forceinline__ void flush_prog_aggregate(const LaneCounters& c, int op, double* dst) {
    if (op < 0 || !dst) return;
    const unsigned any = __ballot_sync(kFull, c.agg_n != 0u);
    if (!any) return;
    double x = c.agg;
    const bool have = c.agg_n != 0u;
    const double id = op == 0 ? 0.0 : (op == 1 ? __longlong_as_double(0x7FF0000000000000LL)
                                               : __longlong_as_double((long long)0xFFF0000000000000ULL));
    if (!have) x = id;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) x = agg_combine(op, x, __shfl_xor_sync(kFull, x, d));
    if ((threadIdx.x & 31) == 0) agg_atomic(op, dst, x);
}

// Record what one vertex did: outbox slot (identity unless it broadcast), bitmap, counters.
template <class P, bool kInit = false>
__device__ __forceinline__ void prog_emit(const ProgArgs<typename P::V>& A, int64_t row,
                                          const ProgCtx& x, unsigned f, typename P::V msg,
                                          LaneCounters& c) {
    using V = typename P::V;
    using C = ProgComb<V, P::kCombiner>;
    const bool b = (f & kProgBroadcast) != 0;
    const V ob = b ? msg : C::identity();
    if constexpr (P::kSettled) {
        if (b) {
            const unsigned long long k = ProgKey<V>::key(msg);
            c.mkey = k < c.mkey ? k : c.mkey;
        }
    }
    A.out_next[A.vbase + row] = ob;
    A.peers.store(A.vbase + row, ob);
    const bool act = (f & kProgStayActive) != 0;
    // bit 2: broadcast one superstep earlier, i.e. the outbox buffer written NEXT holds a
    // non-identity value for this row (k_prog_apply then has to clear it)
    const uint8_t hist = kInit ? 4u : (uint8_t)((A.flags[row] & 1u) << 2);
    A.flags[row] = (uint8_t)((b ? 1u : 0u) | (act ? 2u : 0u) | hist);   // plain store
    if (b) {
        c.changed += 1;
        c.messages += (uint32_t)x.out_degree + (P::kSym ? (uint32_t)x.in_degree : 0u);
    }
    c.aux += act ? 1ull : 0ull;
}

// The point-to-point messages received for `row` (sent in the previous superstep), folded into
// its mailbox; the slot is reset for the next use of this buffer.
template <class P>
__device__ __forceinline__ typename P::V prog_p2p_in(const ProgArgs<typename P::V>& A,
                                                     int64_t row, typename P::V m) {
    using V = typename P::V;
    using C = ProgComb<V, P::kCombiner>;
    if constexpr (!P::kSends) return m;
    if (!A.p2p_in_recv) return m;
    const uint32_t bit = 1u << (row & 31);
    if (!(A.p2p_in_recv[row >> 5] & bit)) return m;
    V* slot = static_cast<V*>(A.p2p_in) + row;
    m = C::combine(m, *slot);
    *slot = C::identity();
    atomicAnd(A.p2p_in_recv + (row >> 5), ~bit);
    return m;
}

// compute on one vertex whose value and degrees were loaded by the caller
template <class P>
__device__ __forceinline__ void prog_vertex_loaded(const ProgArgs<typename P::V>& A, int64_t row,
                                                   typename P::V mailbox, typename P::V val,
                                                   int32_t out_degree, int32_t in_degree,
                                                   LaneCounters& c) {
    using V = typename P::V;
    using C = ProgComb<V, P::kCombiner>;
    const ProgCtx x = prog_ctx(A, row, out_degree, in_degree);
    mailbox = prog_p2p_in<P>(A, row, mailbox);
    V msg = C::identity();
    const unsigned f = P::compute(x, &val, mailbox, &msg);
    A.value[row] = val;
    if constexpr (P::kAggregates) {
        if (x.agg_n) {
            c.agg = c.agg_n ? agg_combine(A.agg_op, c.agg, x.agg_acc) : x.agg_acc;
            c.agg_n = 1u;
        }
    }
    prog_emit<P>(A, row, x, f, msg, c);
}

template <class P>
__device__ __forceinline__ void prog_vertex(const ProgArgs<typename P::V>& A, int64_t row,
                                            typename P::V mailbox, LaneCounters& c) {
    using V = typename P::V;
    using C = ProgComb<V, P::kCombiner>;
    const ProgCtx x = prog_ctx(A, row);
    mailbox = prog_p2p_in<P>(A, row, mailbox);
    V val = A.value[row];
    V msg = C::identity();
    const unsigned f = P::compute(x, &val, mailbox, &msg);
    A.value[row] = val;
    if constexpr (P::kAggregates) {
        if (x.agg_n) {
            c.agg = c.agg_n ? agg_combine(A.agg_op, c.agg, x.agg_acc) : x.agg_acc;
            c.agg_n = 1u;
        }
    }
    prog_emit<P>(A, row, x, f, msg, c);
}

// ---- superstep 0 -----------------------------------------------------------------------------
template <class P>
__global__ void __launch_bounds__(256) k_prog_init(ProgArgs<typename P::V> A,
                                                   PullCounters* counters) {
    using V = typename P::V;
    using C = ProgComb<V, P::kCombiner>;
    __shared__ unsigned long long s_cnt[5];
    if (threadIdx.x < 5) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    LaneCounters c{};
    // grid-stride (a few waves of CTAs): one counter flush per CTA, not per 256 rows -- with
    // every vertex broadcasting, 262K CTAs' same-address atomics cost more than the init itself
    // kInitRows rows per thread, block-strided, their degrees loaded before any store
    constexpr int kInitRows = 4;
    for (int64_t blk = blockIdx.x; blk * blockDim.x * kInitRows < A.rows; blk += gridDim.x) {
        const int64_t base = blk * blockDim.x * kInitRows + threadIdx.x;
        int32_t od[kInitRows], id[kInitRows];
#pragma unroll
        for (int j = 0; j < kInitRows; ++j) {
            const int64_t row = base + (int64_t)j * blockDim.x;
            if (row < A.rows) {
                od[j] = A.out_off[row + 1] - A.out_off[row];
                id[j] = A.in_off[row + 1] - A.in_off[row];
            }
        }
#pragma unroll
        for (int j = 0; j < kInitRows; ++j) {
            const int64_t row = base + (int64_t)j * blockDim.x;
            if (row >= A.rows) continue;
            const ProgCtx x = prog_ctx(A, row, od[j], id[j]);
            V val = C::identity();
            V msg = C::identity();
            const unsigned f = P::init(x, &val, &msg);
            A.value[row] = val;
            A.mbox[row] = C::identity();
            if constexpr (P::kAggregates) {
                if (x.agg_n) {
                    c.agg = c.agg_n ? agg_combine(A.agg_op, c.agg, x.agg_acc) : x.agg_acc;
                    c.agg_n = 1u;
                }
            }
            prog_emit<P, true>(A, row, x, f, msg, c);   // buffer 1 holds a previous run's values
        }
    }
    flush_counters(c, s_cnt, counters);
    if constexpr (P::kSettled) flush_mkey(c.mkey, A.mkey_out);
    if constexpr (P::kAggregates) flush_prog_aggregate(c, A.agg_op, A.shared ? A.shared->agg : nullptr);
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
    using Z = ProgAbsorb<T, P::kCombiner>;
    // ipr_settled (MIN programs): every message of this superstep is >= *bound (k_prog_bound), so
    // a row holding a settled value needs no gathers, and (integer values) a partial fold that is
    // already <= the bound cannot drop further
    static constexpr bool kSettledPartial =
        P::kSettled && P::kCombiner == 1 && (T(3) / T(2) == T(1));   // integer types
    // optional ipr_absorbing(value): a vertex holding such a value ignores its messages, so its
    // row need not be gathered (and whole ranges of such rows are skipped).  Second half of a
    // symmetric pull: a row whose first-half mailbox already holds the combiner's absorbing
    // element needs no second-half gathers either; and any partial fold reaching it ends the
    // row's gathers (kAbsorbingPartial).
    static constexpr bool kAbsorbing = P::kAbsorbing || (kPass == 2 && Z::kHas) || P::kSettled;
    static constexpr bool kAbsorbingPartial = Z::kHas || kSettledPartial;
    // u32 / i32 MIN: warp folds by redux.sync.min (exact in any order), one-row-end chunk path
    static constexpr bool kReduxMin = sizeof(T) == 4 && P::kCombiner == 1 && (T(3) / T(2) == T(1));
    static constexpr bool kAggregates = false;   // compute runs in k_prog_apply
    // 8-byte values: 3 CTAs per SM, as PageRankSum (PageRank program 79.7 -> 78.4 ms at cfg4)
#ifndef IPREGEL_PROG_MINBLOCKS8
#define IPREGEL_PROG_MINBLOCKS8 3
#endif
    static constexpr int kMinBlocks = sizeof(T) == 8 ? IPREGEL_PROG_MINBLOCKS8 : IPREGEL_PULL_MINBLOCKS;
    __device__ void flush_aggregate(const LaneCounters&) const {}
    __device__ static T identity() { return C::identity(); }
    __device__ static T combine(T a, T b) { return C::combine(a, b); }
    __device__ const T* gptr() const { return this->out_cur; }
    __device__ bool absorbed(int32_t row) const {
        if constexpr (kPass == 2 && Z::kHas)
            if (Z::is(this->mbox[row])) return true;
        if constexpr (P::kSettled) {
            if (this->bound) {
                const unsigned long long b = *this->bound;
                if (b == ~0ull || P::settled(this->value[row], ProgKey<T>::value(b))) return true;
            }
        }
        if constexpr (P::kAbsorbing) return P::absorbing(this->value[row]);
        return false;
    }
    __device__ bool absorbing(T x) const {
        if constexpr (kSettledPartial) {
            if (this->bound) {
                const unsigned long long b = *this->bound;
                if (b == ~0ull || !(ProgKey<T>::value(b) < x)) return true;
            }
        }
        return Z::is(x);
    }
    __device__ static T message(T g, uint32_t w) { return P::edge(g, w); }
    // The range kernels only fold each row's messages into its mailbox; the user's compute
    // runs row-parallel in k_prog_apply (pull_all) -- the same split as the built-in PageRank,
    // which keeps the gather loop free of the program's registers.
    __device__ void finish(int32_t row, T m, LaneCounters&) const {
        if (kPass == 2) m = C::combine(this->mbox[row], m);
        this->mbox[row] = m;
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
    // (the sender's broadcast value, the recipient's received-bits word: a filter for the OR)
    struct Pre {
        V m;
        uint32_t r;
    };
    __device__ __forceinline__ Pre pre(int32_t u, uint32_t, int32_t v, uint32_t) const {
        const int64_t lv = (int64_t)v - vbase;
        return Pre{out_cur[u], recv[lv >> 5]};
    }
    __device__ __forceinline__ void fin(const Pre& p, int32_t, uint32_t, int32_t v, uint32_t w) const {
        const int64_t lv = (int64_t)v - vbase;
        ProgComb<V, P::kCombiner>::atomic(mbox + lv, P::edge(p.m, w));
        const uint32_t bit = 1u << (lv & 31);
        if (!(p.r & bit)) atomicOr(recv + (lv >> 5), bit);
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
// A warp owns 32 x kProgApplyRows consecutive rows; it first checks their flag bytes and
// recipient bits and skips them all when none has anything to do (the common case of a sparse
// frontier), else processes them with lane l on rows base + 32 j + l (coalesced stores).
constexpr int kProgApplyRows = 16;
constexpr int kApplyBatch = 4;
template <class P>
__global__ void __launch_bounds__(256) k_prog_apply(ProgArgs<typename P::V> A,
                                                    PullCounters* counters) {
    using V = typename P::V;
    using C = ProgComb<V, P::kCombiner>;
    __shared__ unsigned long long s_cnt[5];
    if (threadIdx.x < 5) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    LaneCounters c{};
    const int lane = threadIdx.x & 31;
    const int64_t base =
        (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * (32 * kProgApplyRows);
    // the check reads lane l's 16 consecutive rows at once: one 16-byte load of their flag bytes
    // (the array is padded to 32 bytes) and half a recipient word
    bool any = false;
    {
        const int64_t r0 = base + (int64_t)kProgApplyRows * lane;
        if (r0 < A.rows) {
            const uint4 f4 = *reinterpret_cast<const uint4*>(A.flags + r0);
            uint32_t got16 = (A.recv[r0 >> 5] >> (r0 & 31)) & 0xFFFFu;
            if constexpr (P::kSends)
                if (A.p2p_in_recv) got16 |= (A.p2p_in_recv[r0 >> 5] >> (r0 & 31)) & 0xFFFFu;
            any = (f4.x | f4.y | f4.z | f4.w | got16) != 0u;
        }
    }
    if (__any_sync(kFull, any)) {   // then every row of the warp, coalesced
        // the 16 recipient words of the warp's rows (lane j holds word j), then the rows in
        // batches of kApplyBatch: flag bytes, mailboxes, values and degrees of a batch are loaded
        // before any of its stores, so the batch's loads are in flight together
        const int64_t w0 = base >> 5;
        uint32_t words = 0u, words_p2p = 0u;
        if (lane < kProgApplyRows && base + 32 * lane < A.rows) {
            words = A.recv[w0 + lane];
            if constexpr (P::kSends)
                if (A.p2p_in_recv) words_p2p = A.p2p_in_recv[w0 + lane];
        }
#pragma unroll 1
        for (int j0 = 0; j0 < kProgApplyRows; j0 += kApplyBatch) {
            uint8_t fl[kApplyBatch];
            bool run[kApplyBatch];
            V m[kApplyBatch], val[kApplyBatch];
            int32_t od[kApplyBatch], id[kApplyBatch];
#pragma unroll
            for (int b = 0; b < kApplyBatch; ++b) {
                const int64_t row = base + 32 * (j0 + b) + lane;
                const uint32_t word = __shfl_sync(kFull, words, j0 + b);
                bool got = (word >> lane) & 1u;
                if constexpr (P::kSends)
                    got = got || ((__shfl_sync(kFull, words_p2p, j0 + b) >> lane) & 1u);
                fl[b] = row < A.rows ? A.flags[row] : (uint8_t)0;
                run[b] = row < A.rows && (got || (fl[b] & 2u));
            }
#pragma unroll
            for (int b = 0; b < kApplyBatch; ++b) {
                const int64_t row = base + 32 * (j0 + b) + lane;
                if (run[b]) {
                    m[b] = A.mbox[row];
                    val[b] = A.value[row];
                    od[b] = A.out_off[row + 1] - A.out_off[row];
                    id[b] = A.in_off[row + 1] - A.in_off[row];
                }
            }
#pragma unroll
            for (int b = 0; b < kApplyBatch; ++b) {
                const int64_t row = base + 32 * (j0 + b) + lane;
                if (run[b]) {
                    A.mbox[row] = C::identity();
                    prog_vertex_loaded<P>(A, row, m[b], val[b], od[b], id[b], c);
                } else if (fl[b]) {
                    // halted and no messages: no broadcast.  The buffer written now holds a
                    // value only if the row broadcast two supersteps ago (bit 2)
                    if (fl[b] & 4u) {
                        A.out_next[A.vbase + row] = C::identity();
                        A.peers.store(A.vbase + row, C::identity());
                    }
                    A.flags[row] = (uint8_t)((fl[b] & 1u) << 2);
                }
            }
        }
        if (words) A.recv[w0 + lane] = 0u;   // lanes < 16: every lane has read them
    }
    flush_counters(c, s_cnt, counters);
    if constexpr (P::kSettled) flush_mkey(c.mkey, A.mkey_out);
    if constexpr (P::kAggregates) flush_prog_aggregate(c, A.agg_op, A.shared ? A.shared->agg : nullptr);
}

// After a pull superstep: every vertex computes on the mailbox the range kernels folded (pull
// selection, reading R28).  kProgPullRows rows per thread, block-strided, mailboxes loaded up
// front.  The mailboxes are not reset here: the next pull overwrites them, and a switch to push
// refills them with the identity first.
constexpr int kProgPullRows = 4;
template <class P>
__global__ void __launch_bounds__(256) k_prog_pull_apply(ProgArgs<typename P::V> A,
                                                         PullCounters* counters) {
    using V = typename P::V;
    __shared__ unsigned long long s_cnt[5];
    if (threadIdx.x < 5) s_cnt[threadIdx.x] = 0;
    LaneCounters c{};
    // grid-stride over blocks of kProgPullRows x 256 rows (one counter flush per CTA)
    for (int64_t blk = blockIdx.x; blk * blockDim.x * kProgPullRows < A.rows; blk += gridDim.x) {
        const int64_t base = blk * blockDim.x * kProgPullRows + threadIdx.x;
        V m[kProgPullRows];
        if constexpr (sizeof(V) == 8) {
            // 8-byte values: the values and degrees too (PageRank program 74.9 -> 74.0 ms at
            // cfg4; with 4-byte values it measured slower: Hash-Min 16.1 -> 16.5, SSSP 13.4 -> 13.5)
            V val[kProgPullRows];
            int32_t od[kProgPullRows], id[kProgPullRows];
#pragma unroll
            for (int j = 0; j < kProgPullRows; ++j) {
                const int64_t row = base + (int64_t)j * blockDim.x;
                if (row < A.rows) {
                    m[j] = A.mbox[row];
                    val[j] = A.value[row];
                    od[j] = A.out_off[row + 1] - A.out_off[row];
                    id[j] = A.in_off[row + 1] - A.in_off[row];
                }
            }
#pragma unroll
            for (int j = 0; j < kProgPullRows; ++j) {
                const int64_t row = base + (int64_t)j * blockDim.x;
                if (row < A.rows) prog_vertex_loaded<P>(A, row, m[j], val[j], od[j], id[j], c);
            }
        } else {
#pragma unroll
            for (int j = 0; j < kProgPullRows; ++j) {
                const int64_t row = base + (int64_t)j * blockDim.x;
                if (row < A.rows) m[j] = A.mbox[row];
            }
#pragma unroll
            for (int j = 0; j < kProgPullRows; ++j) {
                const int64_t row = base + (int64_t)j * blockDim.x;
                if (row < A.rows) prog_vertex<P>(A, row, m[j], c);
            }
        }
    }
    __syncthreads();
    flush_counters(c, s_cnt, counters);
    if constexpr (P::kSettled) flush_mkey(c.mkey, A.mkey_out);
    if constexpr (P::kAggregates) flush_prog_aggregate(c, A.agg_op, A.shared ? A.shared->agg : nullptr);
}

// The bound of a pull superstep of an ipr_settled program: ipr_edge(smallest message broadcast in
// the previous superstep, smallest edge weight) -- with ipr_edge monotone (the hint's contract)
// no message of this superstep is below it.  ~0: nothing was broadcast.
template <class P>
__global__ void k_prog_bound(const unsigned long long* __restrict__ mkey_in, uint32_t w_min,
                             unsigned long long* __restrict__ bound) {
    using V = typename P::V;
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        const unsigned long long k = *mkey_in;
        *bound = k == ~0ull ? ~0ull : ProgKey<V>::key(P::edge(ProgKey<V>::value(k), w_min));
    }
}

}  // namespace ipr
