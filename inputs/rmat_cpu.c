/*
 * inputs/rmat_cpu.c -- seeded synthetic R-MAT edge lists, CPU twin.
 *
 * This module is INPUT GENERATION ONLY.  It holds none of the method's
 * arithmetic (no superstep, no combiner, no vertex program).  Both the
 * oracle (oracle/) and the CUDA path consume what it produces; its GPU twin
 * (inputs/rmat_gpu.cu) implements the same counter-based definition and the
 * two are checked hash-equal by tests/test_inputs_gpu.py.
 *
 * Definition (frozen):
 *   splitmix64(x): z = x + 0x9E3779B97F4A7C15; z = (z^(z>>30))*0xBF58476D1CE4E5B9;
 *                  z = (z^(z>>27))*0x94D049BB133111EB; return z^(z>>31)
 *   key   = splitmix64(seed),  key_w = splitmix64(seed ^ 0x5745494748545321)
 *   slot i in [0, M), level l in [0, S):
 *       h = splitmix64(key + 32*i + l/2);  r = (l even) ? low32(h) : high32(h)
 *       r <  Ta            -> quadrant a (src bit 0, dst bit 0)
 *       r <  Tab           -> quadrant b (src bit 0, dst bit 1)
 *       r <  Tabc          -> quadrant c (src bit 1, dst bit 0)
 *       else               -> quadrant d (src bit 1, dst bit 1)
 *       the bit is S-1-l (most significant first)
 *   weight w_i = 1 + (splitmix64(key_w + i) >> 58)          (uniform in [1,64])
 *   self-loops (src == dst) are dropped; slot order and duplicates are kept;
 *   no noise, no vertex permutation.
 *   Ta/Tab/Tabc are floor(a*2^32), floor((a+b)*2^32), floor((a+b+c)*2^32),
 *   computed by the caller and passed in as integers.
 *
 * The R-MAT recursive-quadrant model and a=0.57,b=c=0.19,d=0.05 are those
 * BASELINE.json configs[0..4] name; they stand in for the paper's SNAP graphs
 * (Table 1), which are not available.
 */
#include <stdint.h>
#include <string.h>
#include <pthread.h>
#include <stdlib.h>

static inline uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

uint64_t rmat_splitmix64(uint64_t x) { return splitmix64(x); }

/* (src, dst) of one slot, before self-loop removal. */
static inline void rmat_slot(uint64_t key, int scale, uint32_t ta, uint32_t tab,
                             uint32_t tabc, uint64_t i, uint32_t* s, uint32_t* d) {
    uint32_t src = 0, dst = 0;
    uint64_t h = 0;
    for (int l = 0; l < scale; ++l) {
        if ((l & 1) == 0) h = splitmix64(key + 32ULL * i + (uint64_t)(l >> 1));
        uint32_t r = (l & 1) ? (uint32_t)(h >> 32) : (uint32_t)h;
        uint32_t qs, qd;
        if (r < ta) { qs = 0; qd = 0; }
        else if (r < tab) { qs = 0; qd = 1; }
        else if (r < tabc) { qs = 1; qd = 0; }
        else { qs = 1; qd = 1; }
        src |= qs << (scale - 1 - l);
        dst |= qd << (scale - 1 - l);
    }
    *s = src;
    *d = dst;
}

void rmat_slot_edge(uint64_t seed, int scale, uint32_t ta, uint32_t tab, uint32_t tabc,
                    uint64_t i, uint32_t* src, uint32_t* dst, uint32_t* w) {
    uint64_t key = splitmix64(seed);
    uint64_t key_w = splitmix64(seed ^ 0x5745494748545321ULL);
    rmat_slot(key, scale, ta, tab, tabc, i, src, dst);
    *w = 1u + (uint32_t)(splitmix64(key_w + i) >> 58);
}

typedef struct {
    uint64_t key, key_w;
    int scale;
    uint32_t ta, tab, tabc;
    uint64_t begin, end;       /* slot range */
    int32_t *src, *dst;        /* written from index `begin` */
    uint32_t* w;               /* may be NULL */
    int64_t kept;
} job_t;

static void* worker(void* p) {
    job_t* j = (job_t*)p;
    int64_t o = (int64_t)j->begin;
    for (uint64_t i = j->begin; i < j->end; ++i) {
        uint32_t s, d;
        rmat_slot(j->key, j->scale, j->ta, j->tab, j->tabc, i, &s, &d);
        if (s == d) continue;
        j->src[o] = (int32_t)s;
        j->dst[o] = (int32_t)d;
        if (j->w) j->w[o] = 1u + (uint32_t)(splitmix64(j->key_w + i) >> 58);
        ++o;
    }
    j->kept = o - (int64_t)j->begin;
    return NULL;
}

/*
 * Generate slots [0, num_slots) into src/dst (and w if non-NULL), each of
 * capacity num_slots.  Returns the number of kept (non-self-loop) edges,
 * which occupy indices [0, kept) in slot order; -1 on bad arguments.
 */
int64_t rmat_generate(uint64_t seed, int scale, uint64_t num_slots, uint32_t ta,
                      uint32_t tab, uint32_t tabc, int32_t* src, int32_t* dst,
                      uint32_t* w, int threads) {
    if (scale < 1 || scale > 31 || !src || !dst) return -1;
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    if ((uint64_t)threads > num_slots) threads = num_slots ? (int)num_slots : 1;
    job_t* jobs = (job_t*)calloc((size_t)threads, sizeof(job_t));
    pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
    if (!jobs || !th) { free(jobs); free(th); return -1; }
    uint64_t key = splitmix64(seed), key_w = splitmix64(seed ^ 0x5745494748545321ULL);
    for (int t = 0; t < threads; ++t) {
        jobs[t].key = key; jobs[t].key_w = key_w; jobs[t].scale = scale;
        jobs[t].ta = ta; jobs[t].tab = tab; jobs[t].tabc = tabc;
        jobs[t].begin = num_slots * (uint64_t)t / (uint64_t)threads;
        jobs[t].end = num_slots * (uint64_t)(t + 1) / (uint64_t)threads;
        jobs[t].src = src; jobs[t].dst = dst; jobs[t].w = w;
        pthread_create(&th[t], NULL, worker, &jobs[t]);
    }
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    /* compact chunks in order: destination never passes the source */
    int64_t out = 0;
    for (int t = 0; t < threads; ++t) {
        int64_t b = (int64_t)jobs[t].begin, k = jobs[t].kept;
        if (out != b && k > 0) {
            memmove(src + out, src + b, (size_t)k * sizeof(int32_t));
            memmove(dst + out, dst + b, (size_t)k * sizeof(int32_t));
            if (w) memmove(w + out, w + b, (size_t)k * sizeof(uint32_t));
        }
        out += k;
    }
    free(jobs);
    free(th);
    return out;
}
