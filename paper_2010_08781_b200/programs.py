"""Vertex programs written against the user-program API (include/ipregel.h, csrc/program.cuh).

The paper's three benchmark programs (Sec. 6) transcribed from Figs. 8-10 into the
ipr_init / ipr_compute / ipr_edge form, plus a few more programs of the same model.  Each entry
is (source, value_type, combiner, symmetric); `compile(name)` builds the Program.
"""
from __future__ import annotations

from .ipregel import Program

# Fig. 8: params[0] = k, the supersteps that broadcast (Fig. 8's 10).
PAGERANK = r"""
__device__ unsigned ipr_init(const ipr_ctx& c, double* value, double* message) {
    const unsigned k = (unsigned)c.params[0];
    *value = 1.0 / (double)c.num_vertices;                 // initial_value (PAPER.md:322)
    if (k == 0) return 0;                                  // ip_vote_to_halt
    if (c.out_degree == 0) return IPR_STAY_ACTIVE;         // no out-neighbour: nothing to send
    *message = *value / (double)c.out_degree;              // ip_broadcast(value / outdeg)
    return IPR_BROADCAST | IPR_STAY_ACTIVE;
}
__device__ unsigned ipr_compute(const ipr_ctx& c, double* value, double mailbox, double* message) {
    const unsigned k = (unsigned)c.params[0];
    const double ratio = 0.15 / (double)c.num_vertices;    // Pregel's 0.15 / N (PAPER.md:521)
    *value = ratio + 0.85 * mailbox;                       // sum of the messages (combined)
    if (c.superstep >= k) return 0;                        // ip_vote_to_halt
    if (c.out_degree == 0) return IPR_STAY_ACTIVE;
    *message = *value / (double)c.out_degree;
    return IPR_BROADCAST | IPR_STAY_ACTIVE;
}
__device__ double ipr_edge(double message, unsigned) { return message; }
"""

# Fig. 9: Hash-Min on the symmetrised graph.
HASHMIN_CC = r"""
__device__ unsigned ipr_init(const ipr_ctx& c, unsigned* value, unsigned* message) {
    *value = (unsigned)c.id;
    *message = *value;
    return IPR_BROADCAST;
}
__device__ unsigned ipr_compute(const ipr_ctx&, unsigned* value, unsigned mailbox,
                                unsigned* message) {
    if (mailbox < *value) {                                // min of the messages improves
        *value = mailbox;
        *message = mailbox;
        return IPR_BROADCAST;
    }
    return 0;                                              // ip_vote_to_halt
}
__device__ unsigned ipr_edge(unsigned message, unsigned) { return message; }
// hint: label 0 (the smallest id) cannot be lowered, so such vertices need not gather
__device__ bool ipr_absorbing(unsigned value) { return value == 0u; }
"""

# Fig. 10 with u32 edge weights (reading R8): params[0] = source.
SSSP = r"""
__device__ unsigned ipr_init(const ipr_ctx& c, unsigned* value, unsigned* message) {
    if (c.id == (long long)c.params[0]) {
        *value = 0;
        *message = 0;
        return IPR_BROADCAST;
    }
    *value = IPR_INF_U32;
    return 0;
}
__device__ unsigned ipr_compute(const ipr_ctx&, unsigned* value, unsigned mailbox,
                                unsigned* message) {
    if (mailbox < *value) {
        *value = mailbox;
        *message = mailbox;
        return IPR_BROADCAST;
    }
    return 0;
}
__device__ unsigned ipr_edge(unsigned message, unsigned weight) {
    return ipr_sat_add(message, weight);                   // value + w, saturating (R9)
}
// hint: compute lowers a value only to a smaller mailbox and ipr_edge is monotone, so a vertex
// at or below the superstep's message bound cannot change (its gathers are skipped)
__device__ bool ipr_settled(unsigned value, unsigned bound) { return value <= bound; }
"""

# Breadth-first levels from params[0]: Fig. 10 exactly (every edge adds 1, weights ignored).
BFS = SSSP.replace("return ipr_sat_add(message, weight);", "return ipr_sat_add(message, 1u);")

# Widest (maximum-bottleneck) path from params[0]: max over paths of the min edge weight.
WIDEST_PATH = r"""
__device__ unsigned ipr_init(const ipr_ctx& c, unsigned* value, unsigned* message) {
    if (c.id == (long long)c.params[0]) {
        *value = IPR_INF_U32;
        *message = IPR_INF_U32;
        return IPR_BROADCAST;
    }
    *value = 0;
    return 0;
}
__device__ unsigned ipr_compute(const ipr_ctx&, unsigned* value, unsigned mailbox,
                                unsigned* message) {
    if (mailbox > *value) {
        *value = mailbox;
        *message = mailbox;
        return IPR_BROADCAST;
    }
    return 0;
}
__device__ unsigned ipr_edge(unsigned message, unsigned weight) {
    return message < weight ? message : weight;            // identity 0 stays 0
}
"""

# Max-label propagation on the symmetrised graph: every vertex ends with the largest id of its
# component (Hash-Min with the order reversed).
MAX_LABEL = r"""
__device__ unsigned ipr_init(const ipr_ctx& c, unsigned* value, unsigned* message) {
    *value = (unsigned)c.id;
    *message = *value;
    return IPR_BROADCAST;
}
__device__ unsigned ipr_compute(const ipr_ctx&, unsigned* value, unsigned mailbox,
                                unsigned* message) {
    if (mailbox > *value) {
        *value = mailbox;
        *message = mailbox;
        return IPR_BROADCAST;
    }
    return 0;
}
__device__ unsigned ipr_edge(unsigned message, unsigned) { return message; }
"""

# One-superstep sum: every vertex broadcasts 1, the value becomes the number of in-edges.
IN_DEGREE = r"""
__device__ unsigned ipr_init(const ipr_ctx&, unsigned* value, unsigned* message) {
    *value = 0;
    *message = 1;
    return IPR_BROADCAST;
}
__device__ unsigned ipr_compute(const ipr_ctx&, unsigned* value, unsigned mailbox, unsigned*) {
    *value = mailbox;
    return 0;
}
__device__ unsigned ipr_edge(unsigned message, unsigned) { return message; }
"""

# Shortest paths with f64 distances (MIN over doubles, +inf = unreached).
SSSP_F64 = r"""
__device__ unsigned ipr_init(const ipr_ctx& c, double* value, double* message) {
    if (c.id == (long long)c.params[0]) {
        *value = 0.0;
        *message = 0.0;
        return IPR_BROADCAST;
    }
    *value = __longlong_as_double(0x7FF0000000000000LL);
    return 0;
}
__device__ unsigned ipr_compute(const ipr_ctx&, double* value, double mailbox, double* message) {
    if (mailbox < *value) {
        *value = mailbox;
        *message = mailbox;
        return IPR_BROADCAST;
    }
    return 0;
}
__device__ double ipr_edge(double message, unsigned weight) { return message + (double)weight; }
// hint: compute lowers a value only to a smaller mailbox and ipr_edge is monotone, so a vertex
// at or below the superstep's message bound cannot change (its gathers are skipped)
__device__ bool ipr_settled(double value, double bound) { return value <= bound; }
"""

# PageRank to convergence with a Pregel aggregator: every vertex folds its rank
# change into a MAX aggregator; in the next superstep, if the largest change was <= params[1],
# every vertex votes to halt keeping its rank (one superstep after the built-in master halt,
# same values).  params[0] = k, the superstep cap.
PAGERANK_CONVERGE = r"""
__device__ unsigned ipr_init(const ipr_ctx& c, double* value, double* message) {
    *value = 1.0 / (double)c.num_vertices;
    if ((unsigned)c.params[0] == 0) return 0;
    if (c.out_degree == 0) return IPR_STAY_ACTIVE;
    *message = *value / (double)c.out_degree;
    return IPR_BROADCAST | IPR_STAY_ACTIVE;
}
__device__ unsigned ipr_compute(const ipr_ctx& c, double* value, double mailbox, double* message) {
    const unsigned k = (unsigned)c.params[0];
    if (c.superstep >= 2 && c.aggregate <= c.params[1]) return 0;   // converged: halt, keep
    const double old = *value;
    *value = 0.15 / (double)c.num_vertices + 0.85 * mailbox;
    ipr_aggregate(c, fabs(*value - old));
    if (c.superstep >= k) return 0;
    if (c.out_degree == 0) return IPR_STAY_ACTIVE;
    *message = *value / (double)c.out_degree;
    return IPR_BROADCAST | IPR_STAY_ACTIVE;
}
__device__ double ipr_edge(double message, unsigned) { return message; }
"""

# Point-to-point messages (Fig. 2's IP_send_message): every vertex v > 0 sends v to its parent
# (v - 1) / 2 in the implicit binary heap over the ids; a vertex's value becomes the sum of its
# children's ids.
HEAP_CHILDREN_SUM = r"""
__device__ unsigned ipr_init(const ipr_ctx& c, unsigned* value, unsigned*) {
    *value = 0;
    if (c.id > 0) ipr_send(c, (c.id - 1) / 2, (unsigned)c.id);
    return 0;
}
__device__ unsigned ipr_compute(const ipr_ctx&, unsigned* value, unsigned mailbox, unsigned*) {
    *value = mailbox;
    return 0;
}
__device__ unsigned ipr_edge(unsigned message, unsigned) { return message; }
"""

# Aggregators: superstep 0 folds 1 per vertex (SUM) -> every vertex reads N in superstep 1.
COUNT_VERTICES = r"""
__device__ unsigned ipr_init(const ipr_ctx& c, double* value, double*) {
    *value = 0.0;
    ipr_aggregate(c, 1.0);
    return IPR_STAY_ACTIVE;
}
__device__ unsigned ipr_compute(const ipr_ctx& c, double* value, double, double*) {
    *value = c.aggregate;
    return 0;
}
__device__ double ipr_edge(double message, unsigned) { return message; }
"""

# The same Fig. 10 / Fig. 9 programs over other value types (ipregel_value_type).
SSSP_F32 = r"""
__device__ unsigned ipr_init(const ipr_ctx& c, float* value, float* message) {
    if (c.id == (long long)c.params[0]) {
        *value = 0.0f;
        *message = 0.0f;
        return IPR_BROADCAST;
    }
    *value = __int_as_float(0x7F800000);                   // +inf: unreached
    return 0;
}
__device__ unsigned ipr_compute(const ipr_ctx&, float* value, float mailbox, float* message) {
    if (mailbox < *value) {
        *value = mailbox;
        *message = mailbox;
        return IPR_BROADCAST;
    }
    return 0;
}
__device__ float ipr_edge(float message, unsigned weight) { return message + (float)weight; }
// hint: compute lowers a value only to a smaller mailbox and ipr_edge is monotone, so a vertex
// at or below the superstep's message bound cannot change (its gathers are skipped)
__device__ bool ipr_settled(float value, float bound) { return value <= bound; }
"""

SSSP_I32 = r"""
__device__ unsigned ipr_init(const ipr_ctx& c, int* value, int* message) {
    if (c.id == (long long)c.params[0]) {
        *value = 0;
        *message = 0;
        return IPR_BROADCAST;
    }
    *value = 0x7FFFFFFF;                                   // INT_MAX: unreached
    return 0;
}
__device__ unsigned ipr_compute(const ipr_ctx&, int* value, int mailbox, int* message) {
    if (mailbox < *value) {
        *value = mailbox;
        *message = mailbox;
        return IPR_BROADCAST;
    }
    return 0;
}
__device__ int ipr_edge(int message, unsigned weight) {
    return message == 0x7FFFFFFF ? message : message + (int)weight;
}
// hint: compute lowers a value only to a smaller mailbox and ipr_edge is monotone, so a vertex
// at or below the superstep's message bound cannot change (its gathers are skipped)
__device__ bool ipr_settled(int value, int bound) { return value <= bound; }
"""

HASHMIN_U64 = r"""
__device__ unsigned ipr_init(const ipr_ctx& c, unsigned long long* value,
                             unsigned long long* message) {
    *value = (unsigned long long)c.id;
    *message = *value;
    return IPR_BROADCAST;
}
__device__ unsigned ipr_compute(const ipr_ctx&, unsigned long long* value,
                                unsigned long long mailbox, unsigned long long* message) {
    if (mailbox < *value) {
        *value = mailbox;
        *message = mailbox;
        return IPR_BROADCAST;
    }
    return 0;
}
__device__ unsigned long long ipr_edge(unsigned long long message, unsigned) { return message; }
"""

# Hash-Min over negated ids (signed 64-bit): every vertex ends with -(largest id of its component).
MIN_NEG_LABEL_I64 = r"""
__device__ unsigned ipr_init(const ipr_ctx& c, long long* value, long long* message) {
    *value = -(long long)c.id;
    *message = *value;
    return IPR_BROADCAST;
}
__device__ unsigned ipr_compute(const ipr_ctx&, long long* value, long long mailbox,
                                long long* message) {
    if (mailbox < *value) {
        *value = mailbox;
        *message = mailbox;
        return IPR_BROADCAST;
    }
    return 0;
}
__device__ long long ipr_edge(long long message, unsigned) { return message; }
"""

CATALOG = {
    "pagerank": (PAGERANK, "f64", "sum", False),
    "hashmin_cc": (HASHMIN_CC, "u32", "min", True),
    "sssp": (SSSP, "u32", "min", False),
    "bfs": (BFS, "u32", "min", False),
    "widest_path": (WIDEST_PATH, "u32", "max", False),
    "max_label": (MAX_LABEL, "u32", "max", True),
    "in_degree": (IN_DEGREE, "u32", "sum", False),
    "sssp_f64": (SSSP_F64, "f64", "min", False),
    "pagerank_converge": (PAGERANK_CONVERGE, "f64", "sum", False, "max"),
    "heap_children_sum": (HEAP_CHILDREN_SUM, "u32", "sum", False),
    "count_vertices": (COUNT_VERTICES, "f64", "sum", False, "sum"),
    "sssp_f32": (SSSP_F32, "f32", "min", False),
    "sssp_i32": (SSSP_I32, "i32", "min", False),
    "hashmin_u64": (HASHMIN_U64, "u64", "min", True),
    "min_neg_label_i64": (MIN_NEG_LABEL_I64, "i64", "min", True),
}


def compile(name: str) -> Program:  # noqa: A001 - mirrors the catalog verb
    src, vt, comb, sym, *agg = CATALOG[name]
    return Program(src, value_type=vt, combiner=comb, symmetric=sym,
                   aggregator=agg[0] if agg else None)
