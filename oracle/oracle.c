/*
 * oracle/oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded CPU Pregel interpreter of iPregel's three
 * benchmark vertex programs (Figs. 8-10), used to check the CUDA
 * path.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  It shares no code, header, table or
 * helper with paper_2010_08781_b200/; its only common input with the CUDA
 * path is the COO edge list from inputs/.
 *
 * Compiled with -O2 -ffp-contract=off (no FMA contraction, IEEE binary64,
 * round-to-nearest-even), no OpenMP, no intrinsics.
 *
 * What it follows, step by step (PAPER.md line numbers):
 *  - BSP superstep: local computation, communications, global
 *    synchronisation; messages sent in superstep s are read in s+1
 *    (PAPER.md:145-151, Sec. 4.2, Fig. 3; :239).
 *  - Naive selection: a vertex runs in superstep s if s == 0, or it has not
 *    halted, or it received a message in s-1 (Sec. 4.3.1).
 *    Selecting a vertex re-activates it (reading R15).
 *  - Single-slot combined mailboxes: a message arriving at a non-empty
 *    mailbox is folded in with the program's combine (PAPER.md:131, :153,
 *    :205-211, Sec. 4.3.3); sum for PageRank (Fig. 8, :295-298), min for
 *    Hash-Min CC and SSSP (Fig. 5, :213-221; Fig. 9 :347-350; Fig. 10
 *    :393-396).  ip_get_next_message therefore yields at most one message.
 *  - Broadcast = one message to every out-neighbour.
 *  - PageRank, Fig. 8: superstep 0 sets value =
 *    initial_value = 1/N (:322); later supersteps set value = ratio +
 *    0.85*sum with ratio = 0.15/N (Pregel, Fig. 12; reading
 *    R2); broadcast value/outdeg while superstep < k (k = 10 in Fig. 8),
 *    else vote to halt.  A vertex with no out-neighbour does not broadcast
 *    (reading R4: Fig. 8 would divide by zero; its mass is dropped).
 *  - Hash-Min CC, Fig. 9: superstep 0 value = id and
 *    broadcast; later value = min(value, messages), broadcast if it
 *    decreased; always vote to halt.  Run on the symmetrised graph
 *    (reading R11): every directed edge (u,v) also contributes (v,u).
 *  - SSSP, Fig. 10, generalised to per-edge weights
 *    (reading R8): superstep 0 the source sets 0 and sends value + w(e) on
 *    each out-edge e, others set INF; later mindist = min(messages); if
 *    mindist < value, value = mindist and send value + w(e) on each
 *    out-edge; always vote to halt.  INF = 0xFFFFFFFF and value + w
 *    saturates at INF (reading R9).  w == NULL means w = 1, i.e. exactly
 *    Fig. 10's "me->value + 1".
 *
 *  - PageRank to convergence ("In practice however, a
 *    PageRank application would typically run until convergence is
 *    reached"; reading R27): with a tolerance eps >= 0, every
 *    vertex of superstep s >= 1 folds |value_s - value_{s-1}| into a max
 *    aggregator (Pregel's aggregators, Fig. 12 context),
 *    and the master halts the run after the first superstep s >= 1 whose
 *    aggregate is <= eps (its broadcast is never delivered), or after
 *    superstep k as in Fig. 8.  eps < 0 disables it (Fig. 8 exactly).
 *
 * Counters per executed superstep s: ran(s) = vertices computed,
 * changed(s) = vertices that broadcast, messages(s) = send() calls.
 * Termination: the run stops at the first superstep in which no vertex
 * qualifies under naive selection ("once every active vertex
 * has been processed and every outgoing message delivered"); that superstep
 * is not counted (reading R16).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

enum { APP_PAGERANK = 0, APP_HASHMIN_CC = 1, APP_SSSP = 2 };
enum { OR_OK = 0, OR_INVALID = 1, OR_NOMEM = 3, OR_GUARD = 6 };

#define INF_U32 0xFFFFFFFFu

static double now_s(void) {
    struct timespec t;
    clock_gettime(CLOCK_MONOTONIC, &t);
    return (double)t.tv_sec + 1e-9 * (double)t.tv_nsec;
}

/* Out-adjacency by stable counting sort on the source (the
 * "global adjacency array").  When sym != 0 the list is the symmetrised
 * one: edge i contributes (src[i], dst[i]) and then (dst[i], src[i]), in
 * edge order, and the counting sort is stable over that list. */
typedef struct {
    int64_t* off;     /* n + 1 */
    int32_t* nbr;     /* off[n] */
    uint32_t* w;      /* off[n] or NULL */
} adj_t;

static void adj_free(adj_t* a) {
    free(a->off); free(a->nbr); free(a->w);
    a->off = NULL; a->nbr = NULL; a->w = NULL;
}

static int adj_build(int64_t n, int64_t m, const int32_t* src, const int32_t* dst,
                     const uint32_t* w, int sym, adj_t* a) {
    int64_t total = sym ? 2 * m : m;
    a->off = (int64_t*)calloc((size_t)(n + 1), sizeof(int64_t));
    a->nbr = (int32_t*)malloc((size_t)(total > 0 ? total : 1) * sizeof(int32_t));
    a->w = NULL;
    if (w && !sym) a->w = (uint32_t*)malloc((size_t)(total > 0 ? total : 1) * sizeof(uint32_t));
    int64_t* cur = (int64_t*)malloc((size_t)(n + 1) * sizeof(int64_t));
    if (!a->off || !a->nbr || !cur || (w && !sym && !a->w)) { free(cur); adj_free(a); return OR_NOMEM; }
    for (int64_t i = 0; i < m; ++i) {
        a->off[src[i] + 1] += 1;
        if (sym) a->off[dst[i] + 1] += 1;
    }
    for (int64_t v = 0; v < n; ++v) a->off[v + 1] += a->off[v];
    memcpy(cur, a->off, (size_t)(n + 1) * sizeof(int64_t));
    for (int64_t i = 0; i < m; ++i) {
        int64_t p = cur[src[i]]++;
        a->nbr[p] = dst[i];
        if (a->w) a->w[p] = w[i];
        if (sym) {
            int64_t q = cur[dst[i]]++;
            a->nbr[q] = src[i];
        }
    }
    free(cur);
    return OR_OK;
}

/* Mailboxes: current (read in superstep s) and next (written in s). */
typedef struct {
    double* fv;        /* PageRank payloads */
    uint32_t* uv;      /* CC / SSSP payloads */
    uint8_t* has;
} mailbox_t;

typedef struct {
    int app;
    int64_t n;
    adj_t adj;
    uint32_t k;        /* PageRank supersteps that broadcast (Fig. 8's 10) */
    uint32_t source;   /* SSSP_SOURCE */
    double ratio;      /* 0.15 / N */
    double tol;        /* PageRank convergence tolerance (< 0: off) */
    double agg;        /* max |value_s - value_{s-1}| of the current superstep */
    double* fval;      /* PageRank vertex values */
    uint32_t* uval;    /* CC / SSSP vertex values */
    uint8_t* halted;
    mailbox_t cur, next;
    uint64_t changed, messages;
} machine_t;

/* IP_send_message + IP_combine into the single-slot mailbox (Sec. 4.3.3). */
static inline void send_f64(machine_t* M, int32_t t, double x) {
    M->messages += 1;
    if (M->next.has[t]) {
        double* old = &M->next.fv[t];
        *old += x;                                 /* Fig. 8 ip_combine */
    } else {
        M->next.fv[t] = x;
        M->next.has[t] = 1;
    }
}

static inline void send_u32(machine_t* M, int32_t t, uint32_t x) {
    M->messages += 1;
    if (M->next.has[t]) {
        uint32_t* old = &M->next.uv[t];
        if (*old > x) *old = x;                    /* Fig. 5 ip_combine */
    } else {
        M->next.uv[t] = x;
        M->next.has[t] = 1;
    }
}

static inline uint32_t sat_add(uint32_t a, uint32_t b) {
    uint64_t s = (uint64_t)a + (uint64_t)b;
    return s >= (uint64_t)INF_U32 ? INF_U32 : (uint32_t)s;
}

/* IP_broadcast: one message to every out-neighbour. */
static void broadcast_f64(machine_t* M, int64_t v, double x) {
    M->changed += 1;
    for (int64_t e = M->adj.off[v]; e < M->adj.off[v + 1]; ++e) send_f64(M, M->adj.nbr[e], x);
}

static void broadcast_u32(machine_t* M, int64_t v, uint32_t x) {
    M->changed += 1;
    for (int64_t e = M->adj.off[v]; e < M->adj.off[v + 1]; ++e) send_u32(M, M->adj.nbr[e], x);
}

/* SSSP's per-edge "value + w" send (reading R8); w == NULL is Fig. 10. */
static void broadcast_dist(machine_t* M, int64_t v, uint32_t d) {
    M->changed += 1;
    for (int64_t e = M->adj.off[v]; e < M->adj.off[v + 1]; ++e) {
        uint32_t w = M->adj.w ? M->adj.w[e] : 1u;
        send_u32(M, M->adj.nbr[e], sat_add(d, w));
    }
}

/* Fig. 8. */
static void compute_pagerank(machine_t* M, int64_t v, uint32_t s, int has, double m) {
    if (s == 0) {
        M->fval[v] = 1.0 / (double)M->n;                       /* initial_value */
    } else {
        double sum = 0.0;
        if (has) sum += m;                                     /* while(get_next_message) */
        double old = M->fval[v];
        M->fval[v] = M->ratio + 0.85 * sum;
        double d = M->fval[v] - old;                           /* max aggregator (R27) */
        if (d < 0.0) d = -d;
        if (d > M->agg) M->agg = d;
    }
    if (s < M->k) {
        int64_t deg = M->adj.off[v + 1] - M->adj.off[v];
        if (deg > 0) broadcast_f64(M, v, M->fval[v] / (double)deg);
    } else {
        M->halted[v] = 1;                                      /* ip_vote_to_halt */
    }
}

/* Fig. 9. */
static void compute_cc(machine_t* M, int64_t v, uint32_t s, int has, uint32_t m) {
    if (s == 0) {
        M->uval[v] = (uint32_t)v;
        broadcast_u32(M, v, M->uval[v]);
    } else {
        uint32_t old = M->uval[v];
        if (has && m < M->uval[v]) M->uval[v] = m;
        if (M->uval[v] < old) broadcast_u32(M, v, M->uval[v]);
    }
    M->halted[v] = 1;
}

/* Fig. 10 with per-edge weights. */
static void compute_sssp(machine_t* M, int64_t v, uint32_t s, int has, uint32_t m) {
    if (s == 0) {
        if ((uint32_t)v == M->source) {
            M->uval[v] = 0;
            broadcast_dist(M, v, M->uval[v]);
        } else {
            M->uval[v] = INF_U32;
        }
    } else {
        uint32_t mindist = INF_U32;
        if (has && m < mindist) mindist = m;
        if (mindist < M->uval[v]) {
            M->uval[v] = mindist;
            broadcast_dist(M, v, M->uval[v]);
        }
    }
    M->halted[v] = 1;
}

/*
 * Run one vertex program to termination.
 *   app: 0 PageRank, 1 Hash-Min CC (symmetrised), 2 SSSP.
 *   n vertices, m directed edges (src[i] -> dst[i]); w may be NULL (w = 1;
 *   ignored except for SSSP).
 *   k: PageRank broadcast supersteps (Fig. 8's 10); source: SSSP source.
 *   max_supersteps: guard (>= 1); if superstep `max_supersteps` would still
 *   have work, returns OR_GUARD with the state after the last executed one.
 *   values_out: double[n] (PageRank) or uint32_t[n].
 *   Per-superstep counters (arrays of `cap`, may be NULL): ran, changed,
 *   messages, seconds.  *supersteps_out = supersteps executed.
 *   *build_seconds_out (may be NULL) = adjacency build time (not a superstep).
 *   tol: PageRank convergence tolerance (< 0: off); delta_out (may be NULL):
 *   per superstep, max_v |value_s(v) - value_{s-1}(v)| (0 for superstep 0 and
 *   for the other apps).
 */
int oracle_run(int app, int64_t n, int64_t m, const int32_t* src, const int32_t* dst,
               const uint32_t* w, uint32_t k, uint32_t source, uint32_t max_supersteps,
               void* values_out, uint32_t* supersteps_out, uint32_t cap, uint64_t* ran_out,
               uint64_t* changed_out, uint64_t* messages_out, double* seconds_out,
               double* build_seconds_out, double tol, double* delta_out) {
    if (n < 1 || n > 2147483647LL || m < 0 || (m > 0 && (!src || !dst)) || !values_out ||
        max_supersteps == 0 || app < 0 || app > 2)
        return OR_INVALID;
    if (app == APP_SSSP && (int64_t)source >= n) return OR_INVALID;
    for (int64_t i = 0; i < m; ++i)
        if (src[i] < 0 || src[i] >= n || dst[i] < 0 || dst[i] >= n) return OR_INVALID;

    machine_t M;
    memset(&M, 0, sizeof(M));
    M.app = app; M.n = n; M.k = k; M.source = source;
    M.ratio = 0.15 / (double)n;
    M.tol = tol;

    double t0 = now_s();
    int rc = adj_build(n, m, src, dst, app == APP_SSSP ? w : NULL, app == APP_HASHMIN_CC, &M.adj);
    if (rc != OR_OK) return rc;
    if (build_seconds_out) *build_seconds_out = now_s() - t0;

    size_t un = (size_t)n;
    M.halted = (uint8_t*)calloc(un, 1);
    M.cur.has = (uint8_t*)calloc(un, 1);
    M.next.has = (uint8_t*)calloc(un, 1);
    if (app == APP_PAGERANK) {
        M.fval = (double*)calloc(un, sizeof(double));
        M.cur.fv = (double*)calloc(un, sizeof(double));
        M.next.fv = (double*)calloc(un, sizeof(double));
    } else {
        M.uval = (uint32_t*)calloc(un, sizeof(uint32_t));
        M.cur.uv = (uint32_t*)calloc(un, sizeof(uint32_t));
        M.next.uv = (uint32_t*)calloc(un, sizeof(uint32_t));
    }
    int ok = M.halted && M.cur.has && M.next.has &&
             (app == APP_PAGERANK ? (M.fval && M.cur.fv && M.next.fv)
                                  : (M.uval && M.cur.uv && M.next.uv));
    rc = ok ? OR_OK : OR_NOMEM;

    uint32_t executed = 0;
    for (uint32_t s = 0; ok; ++s) {
        if (s == max_supersteps) {
            int pending = (s == 0);
            for (int64_t v = 0; v < n && !pending; ++v)
                if (!M.halted[v] || M.cur.has[v]) pending = 1;
            if (pending) rc = OR_GUARD;
            break;
        }
        double ts = now_s();
        uint64_t ran = 0;
        M.changed = 0;
        M.messages = 0;
        M.agg = 0.0;
        for (int64_t v = 0; v < n; ++v) {
            /* naive selection */
            if (!(s == 0 || !M.halted[v] || M.cur.has[v])) continue;
            ran += 1;
            M.halted[v] = 0;
            int has = M.cur.has[v];
            if (app == APP_PAGERANK)
                compute_pagerank(&M, v, s, has, has ? M.cur.fv[v] : 0.0);
            else if (app == APP_HASHMIN_CC)
                compute_cc(&M, v, s, has, has ? M.cur.uv[v] : 0u);
            else
                compute_sssp(&M, v, s, has, has ? M.cur.uv[v] : 0u);
        }
        if (ran == 0) break;                     /* nobody qualified: not a superstep */
        /* global synchronisation: next mailboxes become current */
        mailbox_t tmp = M.cur; M.cur = M.next; M.next = tmp;
        memset(M.next.has, 0, un);
        double te = now_s();
        if (executed < cap) {
            if (ran_out) ran_out[executed] = ran;
            if (changed_out) changed_out[executed] = M.changed;
            if (messages_out) messages_out[executed] = M.messages;
            if (seconds_out) seconds_out[executed] = te - ts;
            if (delta_out) delta_out[executed] = M.agg;
        }
        executed += 1;
        /* master halt: PageRank converged (reading R27) */
        if (app == APP_PAGERANK && M.tol >= 0.0 && s >= 1 && M.agg <= M.tol) break;
    }
    if (ok) {
        if (app == APP_PAGERANK) memcpy(values_out, M.fval, un * sizeof(double));
        else memcpy(values_out, M.uval, un * sizeof(uint32_t));
    }
    if (supersteps_out) *supersteps_out = executed;
    free(M.halted); free(M.cur.has); free(M.next.has);
    free(M.fval); free(M.cur.fv); free(M.next.fv);
    free(M.uval); free(M.cur.uv); free(M.next.uv);
    adj_free(&M.adj);
    return rc;
}
