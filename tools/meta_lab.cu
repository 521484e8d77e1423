// tools/meta_lab.cu -- lab: the PageRank gather with its row bookkeeping driven by per-chunk
// metadata built at create time instead of CSC offset loads inside the loop.
//
// Per 128-edge chunk (global grid): a 128-bit mask of the positions holding the LAST edge of a
// row (rows with in-edges only) and the ordinal, among rows with in-edges, of the row holding
// the chunk's first edge.  A warp then knows from data loaded with the index stream (two chunks
// ahead) whether a chunk is inside one row, closes one row, or several, and which rows -- no
// dependent offset loads.  Sums go to a compact array (ordinal order); the update pass maps
// ordinals back.  Same combine tree as the product's range kernel (pull.cuh): fast chunks into
// lane-private partials, first / last segment by masked folds (warp_fold2), inner rows by the
// four chained segmented scans.
//   v0: raw gather stream (no rows), warp blocks of kBlk chunks;
//   v3: v0 + the metadata-driven row logic, per-row sums written.
// Rows crossing warp-block boundaries are NOT joined (lab: their partial goes to a carry slot).
// Not product code.
#include <cuda_runtime.h>
#include <cstdint>

constexpr int kChunk = 128;
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ uint64_t pol_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t pol_range(const void* base, uint32_t hot, uint32_t total) {
    uint64_t p;
    asm volatile("createpolicy.range.global.L2::evict_last.L2::evict_first.b64 %0, [%1], %2, %3;"
                 : "=l"(p) : "l"(base), "r"(hot), "r"(total));
    return p;
}
__device__ __forceinline__ int32_t ld_s(const int32_t* p, uint64_t pol) {
    int32_t r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ uint4 ld_s4(const uint4* p, uint64_t pol) {
    uint4 r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
        : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ double ld_valp(const double* base, int32_t u, uint64_t pol) {
    double r;
    const double* p = base + u;
    asm("{\n\t.reg .pred q;\n\tsetp.lt.s32 q, %3, 8192;\n\t"
        "@q ld.global.nc.L1::evict_last.L2::cache_hint.f64 %0, [%1], %2;\n\t"
        "@!q ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;\n\t}"
        : "=d"(r) : "l"(p), "l"(pol), "r"(u));
    return r;
}
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }

__device__ __forceinline__ double warp_fold(double x) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const double o = __shfl_xor_sync(kFull, x, d);
        x = (lane & d) ? add(o, x) : add(x, o);
    }
    return x;
}
__device__ __forceinline__ void warp_fold2(double a, double b, double& fa, double& fb) {
    const int lane = threadIdx.x & 31;
    const bool hi = lane & 16;
    const double o = __shfl_xor_sync(kFull, hi ? a : b, 16);
    double x = hi ? add(o, b) : add(a, o);
#pragma unroll
    for (int d = 1; d < 16; d <<= 1) {
        const double y = __shfl_xor_sync(kFull, x, d);
        x = (lane & d) ? add(y, x) : add(x, y);
    }
    fa = __shfl_sync(kFull, x, 0);
    fb = __shfl_sync(kFull, x, 16);
}

// ---- metadata: end mask per chunk --------------------------------------------------------
// rs[e] = 1 iff e is the first edge of a row (rows with in-edges).  End at e iff e = E - 1 or
// rs[e + 1].  One warp per chunk.
__global__ void k_meta_build(const uint8_t* __restrict__ rs, int64_t E, int64_t nch, uint4* mask,
                             int32_t* cnt) {
    const int lane = threadIdx.x & 31;
    const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (c >= nch) return;
    uint32_t w[4];
    int n = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int64_t e = c * kChunk + 32 * k + lane;
        const bool end = e < E && (e == E - 1 || rs[e + 1]);
        w[k] = __ballot_sync(kFull, end);
        n += __popc(w[k]);
    }
    if (lane == 0) {
        mask[c] = make_uint4(w[0], w[1], w[2], w[3]);
        cnt[c] = n;
    }
}

__device__ int g_nrows;
__device__ int g_bad;
struct Meta {
    uint32_t f[4];   // end mask (uniform)
    int32_t ord0;    // ordinal of the row holding the chunk's first edge
};

template <int kBlk>
__global__ void __launch_bounds__(256, 3) k_raw(const int32_t* __restrict__ idx, int64_t E,
                                                int64_t nch, const double* __restrict__ vals,
                                                double* out, int* ctr, uint32_t gtotal, int order,
                                                int64_t nblk) {
    const int lane = threadIdx.x & 31;
    const uint64_t pol = pol_first();
    const uint64_t gp = pol_range(vals, 64u << 20, gtotal);
    double acc = 0;
    for (;;) {
        int t = lane == 0 ? atomicAdd(ctr, 1) : 0;
        t = __shfl_sync(kFull, t, 0);
        if (t >= nblk) break;
        const int64_t q = order ? ((t & 1) ? nblk - 1 - (t >> 1) : (t >> 1)) : t;
        const int64_t c0 = q * kBlk;
        const int64_t c1 = c0 + kBlk < nch ? c0 + kBlk : nch;
        int32_t a[4], bq[4];
        auto ld = [&](int64_t c, int32_t (&r)[4]) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int64_t e = c * kChunk + 32 * k + lane;
                r[k] = (c < c1 && e < E) ? ld_s(idx + e, pol) : -1;
            }
        };
        ld(c0, a);
        ld(c0 + 1, bq);
        double g[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) g[k] = a[k] >= 0 ? ld_valp(vals, a[k], gp) : 0.0;
        for (int64_t c = c0; c < c1; ++c) {
            double gn[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) gn[k] = bq[k] >= 0 ? ld_valp(vals, bq[k], gp) : 0.0;
            ld(c + 2, bq);
            acc += (g[0] + g[1]) + (g[2] + g[3]);
#pragma unroll
            for (int k = 0; k < 4; ++k) g[k] = gn[k];
        }
    }
    out[(int64_t)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int kBlk>
__global__ void __launch_bounds__(256, 3) k_meta(const int32_t* __restrict__ idx,
                                                 const uint4* __restrict__ mask,
                                                 const int32_t* __restrict__ ord,
                                                 int64_t E, int64_t nch,
                                                 const double* __restrict__ vals,
                                                 double* __restrict__ sumc, double* carry_out,
                                                 int* ctr, uint32_t gtotal, int order, int64_t nblk) {
    const int lane = threadIdx.x & 31;
    const uint64_t pol = pol_first();
    const uint64_t gp = pol_range(vals, 64u << 20, gtotal);
    for (;;) {
        int t = lane == 0 ? atomicAdd(ctr, 1) : 0;
        t = __shfl_sync(kFull, t, 0);
        if (t >= nblk) break;
        const int64_t q = order ? ((t & 1) ? nblk - 1 - (t >> 1) : (t >> 1)) : t;
        const int64_t c0 = q * kBlk;
        const int64_t c1 = c0 + kBlk < nch ? c0 + kBlk : nch;
        int32_t a[4], bq[4];
        Meta ma, mb;
        auto ld = [&](int64_t c, int32_t (&r)[4], Meta& m) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int64_t e = c * kChunk + 32 * k + lane;
                r[k] = (c < c1 && e < E) ? ld_s(idx + e, pol) : -1;
            }
            if (c < c1) {
                const uint4 u = ld_s4(mask + c, pol);
                m.f[0] = u.x; m.f[1] = u.y; m.f[2] = u.z; m.f[3] = u.w;
                m.ord0 = ord[c];
            } else {
                m.f[0] = m.f[1] = m.f[2] = m.f[3] = 0u;
                m.ord0 = 0;
            }
        };
        ld(c0, a, ma);
        ld(c0 + 1, bq, mb);
        double g[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) g[k] = a[k] >= 0 ? ld_valp(vals, a[k], gp) : 0.0;
        double la = 0.0, carry = 0.0;
        for (int64_t c = c0; c < c1; ++c) {
            double gn[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) gn[k] = bq[k] >= 0 ? ld_valp(vals, bq[k], gp) : 0.0;
            const Meta m = ma;
            ma = mb;
            ld(c + 2, bq, mb);
            double v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                v[k] = g[k];
                g[k] = gn[k];
            }
            const int n_end = __popc(m.f[0]) + __popc(m.f[1]) + __popc(m.f[2]) + __popc(m.f[3]);
            if (n_end == 0) {
                la = add(la, add(add(v[0], v[1]), add(v[2], v[3])));
                continue;
            }
            // first end position q1 and last end position ql
            int q1, ql;
            {
                const int k1 = m.f[0] ? 0 : (m.f[1] ? 1 : (m.f[2] ? 2 : 3));
                q1 = 32 * k1 + __ffs(m.f[k1]) - 1;
                const int kl = m.f[3] ? 3 : (m.f[2] ? 2 : (m.f[1] ? 1 : 0));
                ql = 32 * kl + 31 - __clz(m.f[kl]);
            }
            const int p1 = q1 + 1, pl = ql + 1;
            double t1 = 0.0, t2 = 0.0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int pos = 32 * k + lane;
                if (pos < p1) t1 = add(t1, v[k]);
                else if (pos >= pl) t2 = add(t2, v[k]);
            }
            double f1, f2;
            warp_fold2(t1, t2, f1, f2);
            const double first = add(add(carry, warp_fold(la)), f1);
            if (lane == 0) {
                if ((unsigned)m.ord0 < (unsigned)g_nrows) sumc[m.ord0] = first;
                else atomicAdd(&g_bad, 1);
            }
            la = 0.0;
            carry = f2;
            if (n_end == 1) continue;
            // inner rows: segment heads at (end + 1), four chained segmented scans
            uint32_t h[4];
            h[0] = m.f[0] << 1;
            h[1] = (m.f[1] << 1) | (m.f[0] >> 31);
            h[2] = (m.f[2] << 1) | (m.f[1] >> 31);
            h[3] = (m.f[3] << 1) | (m.f[2] >> 31);
            int start[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t mm = h[k] & (0xFFFFFFFFu >> (31 - lane));
                start[k] = mm ? 31 - __clz(mm) : -1;
            }
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const double y = __shfl_up_sync(kFull, v[k], d);
                    if (lane >= d && lane - d >= start[k]) v[k] = add(y, v[k]);
                }
            }
            double cc = 0.0;
            int below = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (start[k] < 0) v[k] = add(cc, v[k]);
                cc = __shfl_sync(kFull, v[k], 31);
                const int pos = 32 * k + lane;
                const bool is_end = (m.f[k] >> lane) & 1u;
                const int rank = below + __popc(m.f[k] & ((1u << lane) - 1u));
                if (is_end && pos != q1) {
                    if ((unsigned)(m.ord0 + rank) < (unsigned)g_nrows) sumc[m.ord0 + rank] = v[k];
                    else atomicAdd(&g_bad, 1);
                }
                below += __popc(m.f[k]);
            }
        }
        const double co = add(carry, warp_fold(la));
        if (lane == 0) carry_out[q] = co;
    }
}


// v4: metadata rows with a cheaper combine tree.  One-end chunks fold the lane partials of the
// open row into the first segment (one paired fold); chunks with more ends transpose the chunk
// through shared memory so lane l holds positions 4l..4l+3, sum runs lane-sequentially, and one
// 5-step segmented scan over the lanes joins rows crossing lanes.  The open row's lane partials
// are folded only when a fast chunk fed them (la_used).
template <int kBlk, int kMB, int kAbl>
__global__ void __launch_bounds__(256, kMB) k_meta4(const int32_t* __restrict__ idx,
                                                  const uint4* __restrict__ mask,
                                                  const int32_t* __restrict__ ord,
                                                  int64_t E, int64_t nch,
                                                  const double* __restrict__ vals,
                                                  double* __restrict__ sumc, double* carry_out,
                                                  int* ctr, uint32_t gtotal, int order, int64_t nblk) {
    __shared__ __align__(16) double s_w[8][128];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double* sw = s_w[wid];
    double la_sink = 0.0;
    const uint64_t pol = pol_first();
    const uint64_t gp = pol_range(vals, 64u << 20, gtotal);
    for (;;) {
        int t = lane == 0 ? atomicAdd(ctr, 1) : 0;
        t = __shfl_sync(kFull, t, 0);
        if (t >= nblk) break;
        const int64_t q = order ? ((t & 1) ? nblk - 1 - (t >> 1) : (t >> 1)) : t;
        const int64_t c0 = q * kBlk;
        const int64_t c1 = c0 + kBlk < nch ? c0 + kBlk : nch;
        int32_t a[4], bq[4];
        Meta ma, mb;
        int32_t run_ord = kAbl == 3 ? ord[c0] : 0;   // index-bit flags: ordinals by counting
        auto ld = [&](int64_t c, int32_t (&r)[4], Meta& m) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int64_t e = c * kChunk + 32 * k + lane;
                r[k] = (c < c1 && e < E) ? ld_s(idx + e, pol) : 0x7fffffff;
            }
            if (kAbl == 3) return;
            if (c < c1) {
                const uint4 u = ld_s4(mask + c, pol);
                m.f[0] = u.x; m.f[1] = u.y; m.f[2] = u.z; m.f[3] = u.w;
                m.ord0 = ord[c];
            } else {
                m.f[0] = m.f[1] = m.f[2] = m.f[3] = 0u;
                m.ord0 = 0;
            }
        };
        auto gat = [&](const int32_t (&r)[4], double (&gg)[4]) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int32_t u = r[k] & 0x7fffffff;
                gg[k] = u != 0x7fffffff ? ld_valp(vals, u, gp) : 0.0;
            }
        };
        ld(c0, a, ma);
        ld(c0 + 1, bq, mb);
        double g[4];
        gat(a, g);
        uint32_t fa[4];   // kAbl 3: end words of the chunk whose values are in g
#pragma unroll
        for (int k = 0; k < 4; ++k) fa[k] = __ballot_sync(kFull, a[k] < 0);
        double la = 0.0, carry = 0.0;
        bool la_used = false;
        for (int64_t c = c0; c < c1; ++c) {
            double gn[4];
            gat(bq, gn);
            Meta m = ma;
            if (kAbl == 3) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    m.f[k] = fa[k];
                    fa[k] = __ballot_sync(kFull, bq[k] < 0);
                }
                m.ord0 = run_ord;
            }
            ma = mb;
            ld(c + 2, bq, mb);
            double v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                v[k] = g[k];
                g[k] = gn[k];
            }
            const int n_end = __popc(m.f[0]) + __popc(m.f[1]) + __popc(m.f[2]) + __popc(m.f[3]);
            if (kAbl == 3) run_ord += n_end;
            if (kAbl == 1 || n_end == 0) {
                la = add(la, add(add(v[0], v[1]), add(v[2], v[3])));
                if (kAbl == 1) la = add(la, (double)(n_end + m.ord0));
                la_used = true;
                continue;
            }
            if (n_end == 1) {
                const int k1 = m.f[0] ? 0 : (m.f[1] ? 1 : (m.f[2] ? 2 : 3));
                const int p1 = 32 * k1 + __ffs(m.f[k1]);   // positions < p1 close the open row
                double t1 = la, t2 = 0.0;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if (32 * k + lane < p1) t1 = add(t1, v[k]);
                    else t2 = add(t2, v[k]);
                }
                double f1, f2;
                warp_fold2(t1, t2, f1, f2);
                if (kAbl == 2) la_sink = add(la_sink, f1);
                else if (lane == 0) {
                    if ((unsigned)m.ord0 < (unsigned)g_nrows) sumc[m.ord0] = add(carry, f1);
                    else atomicAdd(&g_bad, 1);
                }
                carry = f2;
                la = 0.0;
                la_used = false;
                continue;
            }
            // several ends: lane l takes positions 4l .. 4l + 3
#pragma unroll
            for (int k = 0; k < 4; ++k) sw[32 * k + lane] = v[k];
            __syncwarp();
            const double2 w01 = *reinterpret_cast<const double2*>(sw + 4 * lane);
            const double2 w23 = *reinterpret_cast<const double2*>(sw + 4 * lane + 2);
            __syncwarp();
            const double w[4] = {w01.x, w01.y, w23.x, w23.y};
            const uint32_t word = m.f[lane >> 3];
            const uint32_t nib = (word >> (4 * (lane & 7))) & 0xFu;
            // ends at positions before this lane's first: rank base
            int below = __popc(word & ((1u << (4 * (lane & 7))) - 1u));
#pragma unroll
            for (int k = 0; k < 3; ++k)
                if (k < (lane >> 3)) below += __popc(m.f[k]);
            const double L = la_used ? warp_fold(la) : 0.0;   // warp-uniform branch
            double acc = 0.0, A = 0.0;
            bool first_in_lane = true;
            int r = below;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                acc = add(acc, w[j]);
                if ((nib >> j) & 1u) {
                    if (first_in_lane) {
                        A = acc;
                        first_in_lane = false;
                    } else if (kAbl == 2) {
                        la_sink = add(la_sink, acc);
                    } else {
                        if ((unsigned)(m.ord0 + r) < (unsigned)g_nrows) sumc[m.ord0 + r] = acc;
                        else atomicAdd(&g_bad, 1);
                    }
                    ++r;
                    acc = 0.0;
                }
            }
            // segmented inclusive scan of the lanes' outgoing partials; a lane with an end
            // starts a segment (its partial after its last end opens a row)
            const bool has_end = nib != 0u;
            const uint32_t ends = __ballot_sync(kFull, has_end);
            const uint32_t le = ends & (0xFFFFFFFFu >> (31 - lane));
            const int start = le ? 31 - __clz(le) : -1;
            double x = acc;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const double y = __shfl_up_sync(kFull, x, d);
                if (lane >= d && lane - d >= start) x = add(y, x);
            }
            double in = __shfl_up_sync(kFull, x, 1);
            if (lane == 0) in = 0.0;
            const int first_lane = __ffs(ends) - 1;
            if (has_end) {
                double tot = add(in, A);
                if (lane == first_lane) tot = add(add(carry, L), tot);
                const int o = m.ord0 + below;
                if (kAbl == 2) la_sink = add(la_sink, tot);
                else if ((unsigned)o < (unsigned)g_nrows) sumc[o] = tot;
                else atomicAdd(&g_bad, 1);
            }
            carry = __shfl_sync(kFull, x, 31);
            la = 0.0;
            la_used = false;
        }
        const double co = add(carry, la_used ? warp_fold(la) : 0.0);
        if (lane == 0) carry_out[q] = co;
    }
    if (kAbl != 0 && la_sink == 1.2345) carry_out[0] = la_sink;
}

// v9/v10: index-bit row-end flags (bit 31 of the CSC index), gathers kAhead chunks ahead
__device__ __forceinline__ double ld_cold(const double* base, int32_t u, uint64_t pol) {
    double r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
        : "=d"(r) : "l"(base + u), "l"(pol));
    return r;
}
template <int kBlk, int kAhead, int kThreads = 256, int kMinB = 3, int kH = 0>
__global__ void __launch_bounds__(kThreads, kMinB) k_flag(const int32_t* __restrict__ idx,
                                                 const int32_t* __restrict__ ord, int64_t E,
                                                 int64_t nch, const double* __restrict__ vals,
                                                 double* __restrict__ sumc, double* carry_out,
                                                 int* ctr, uint32_t gtotal, int order,
                                                 int64_t nblk) {
    extern __shared__ __align__(16) double s_dyn[];
    double* s_hot = s_dyn;                       // [kH]
    double* s_wall = s_dyn + kH;                 // [warps][128]
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double* sw = s_wall + wid * 128;
    const uint64_t pol = pol_first();
    const uint64_t gp = pol_range(vals, 64u << 20, gtotal);
    if (kH > 0) {
        for (int i = threadIdx.x; i < kH; i += kThreads) s_hot[i] = vals[i];
        __syncthreads();
    }
    for (;;) {
        int t = lane == 0 ? atomicAdd(ctr, 1) : 0;
        t = __shfl_sync(kFull, t, 0);
        if (t >= nblk) break;
        const int64_t q = order ? ((t & 1) ? nblk - 1 - (t >> 1) : (t >> 1)) : t;
        const int64_t c0 = q * kBlk;
        const int64_t c1 = c0 + kBlk < nch ? c0 + kBlk : nch;
        int32_t run_ord = ord[c0];
        auto ld = [&](int64_t c, int32_t (&r)[4]) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int64_t e = c * kChunk + 32 * k + lane;
                r[k] = (c < c1 && e < E) ? ld_s(idx + e, pol) : 0x7fffffff;
            }
        };
        auto gat = [&](const int32_t (&r)[4], double (&gg)[4], uint32_t (&ff)[4]) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int32_t u = r[k] & 0x7fffffff;
                if (kH > 0) gg[k] = u < kH ? s_hot[u] : (u != 0x7fffffff ? ld_cold(vals, u, gp) : 0.0);
                else gg[k] = u != 0x7fffffff ? ld_valp(vals, u, gp) : 0.0;
                ff[k] = __ballot_sync(kFull, r[k] < 0);
            }
        };
        // ring: values + flags of chunks c .. c + kAhead - 1 gathered, indices of c + kAhead
        double G[kAhead][4];
        uint32_t F[kAhead][4];
        int32_t I[4];
#pragma unroll
        for (int a = 0; a < kAhead; ++a) {
            ld(c0 + a, I);
            gat(I, G[a], F[a]);
        }
        ld(c0 + kAhead, I);
        double la = 0.0, carry = 0.0;
        bool la_used = false;
        for (int64_t c = c0; c < c1; ++c) {
            double v[4];
            uint32_t f[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                v[k] = G[0][k];
                f[k] = F[0][k];
            }
#pragma unroll
            for (int a = 0; a + 1 < kAhead; ++a)
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    G[a][k] = G[a + 1][k];
                    F[a][k] = F[a + 1][k];
                }
            gat(I, G[kAhead - 1], F[kAhead - 1]);
            ld(c + kAhead + 1, I);
            const int32_t o0 = run_ord;
            const int n_end = __popc(f[0]) + __popc(f[1]) + __popc(f[2]) + __popc(f[3]);
            run_ord += n_end;
            if (n_end == 0) {
                la = add(la, add(add(v[0], v[1]), add(v[2], v[3])));
                la_used = true;
                continue;
            }
            if (n_end == 1) {
                const int k1 = f[0] ? 0 : (f[1] ? 1 : (f[2] ? 2 : 3));
                const int p1 = 32 * k1 + __ffs(f[k1]);
                double t1 = la, t2 = 0.0;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if (32 * k + lane < p1) t1 = add(t1, v[k]);
                    else t2 = add(t2, v[k]);
                }
                double f1, f2;
                warp_fold2(t1, t2, f1, f2);
                if (lane == 0) sumc[o0] = add(carry, f1);
                carry = f2;
                la = 0.0;
                la_used = false;
                continue;
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) sw[32 * k + lane] = v[k];
            __syncwarp();
            const double2 w01 = *reinterpret_cast<const double2*>(sw + 4 * lane);
            const double2 w23 = *reinterpret_cast<const double2*>(sw + 4 * lane + 2);
            __syncwarp();
            const double w[4] = {w01.x, w01.y, w23.x, w23.y};
            const uint32_t word = lane < 8 ? f[0] : (lane < 16 ? f[1] : (lane < 24 ? f[2] : f[3]));
            const uint32_t nib = (word >> (4 * (lane & 7))) & 0xFu;
            int below = __popc(word & ((1u << (4 * (lane & 7))) - 1u));
            below += (lane >= 8 ? __popc(f[0]) : 0) + (lane >= 16 ? __popc(f[1]) : 0) +
                     (lane >= 24 ? __popc(f[2]) : 0);
            const double L = la_used ? warp_fold(la) : 0.0;
            double acc = 0.0, A = 0.0;
            bool first_in_lane = true;
            int r = below;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                acc = add(acc, w[j]);
                if ((nib >> j) & 1u) {
                    if (first_in_lane) {
                        A = acc;
                        first_in_lane = false;
                    } else {
                        sumc[o0 + r] = acc;
                    }
                    ++r;
                    acc = 0.0;
                }
            }
            const bool has_end = nib != 0u;
            const uint32_t ends = __ballot_sync(kFull, has_end);
            const uint32_t le = ends & (0xFFFFFFFFu >> (31 - lane));
            const int start = le ? 31 - __clz(le) : -1;
            double x = acc;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const double y = __shfl_up_sync(kFull, x, d);
                if (lane >= d && lane - d >= start) x = add(y, x);
            }
            double in = __shfl_up_sync(kFull, x, 1);
            if (lane == 0) in = 0.0;
            const int first_lane = __ffs(ends) - 1;
            if (has_end) {
                double tot = add(in, A);
                if (lane == first_lane) tot = add(add(carry, L), tot);
                sumc[o0 + below] = tot;
            }
            carry = __shfl_sync(kFull, x, 31);
            la = 0.0;
            la_used = false;
        }
        const double co = add(carry, la_used ? warp_fold(la) : 0.0);
        if (lane == 0) carry_out[q] = co;
    }
}

extern "C" {
void meta_build(const uint8_t* rs, int64_t E, uint4* mask, int32_t* cnt) {
    const int64_t nch = (E + kChunk - 1) / kChunk;
    k_meta_build<<<(unsigned)((nch * 32 + 255) / 256), 256>>>(rs, E, nch, mask, cnt);
}
// variant 0 raw, 3 metadata rows; returns ms per pass (mean of reps)
int meta_bad(int nrows) {
    int b = 0;
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(&b, g_bad, 4);
    cudaMemcpyToSymbol(g_nrows, &nrows, 4);
    return b;
}
float run_meta_lab(int variant, const int32_t* idx, const uint4* mask, const int32_t* ord,
                   int64_t E, const double* vals, int64_t n_vals, double* sumc, double* carry,
                   double* out, int* ctr, int ctas_per_sm, int order, int reps) {
    constexpr int kBlk = 64;
    const int64_t nch = (E + kChunk - 1) / kChunk;
    const int64_t nblk = (nch + kBlk - 1) / kBlk;
    const int grid = 148 * ctas_per_sm;
    static bool attr = false;
    if (!attr) {
        attr = true;
        cudaFuncSetAttribute(k_flag<kBlk, 1, 768, 1, 8192>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192 * 8 + 24 * 1024);
        cudaFuncSetAttribute(k_flag<kBlk, 1, 768, 1, 16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 * 8 + 24 * 1024);
        cudaFuncSetAttribute(k_flag<kBlk, 1, 768, 1, 25088>, cudaFuncAttributeMaxDynamicSharedMemorySize, 25088 * 8 + 24 * 1024);
    }
    const uint32_t gtotal = (uint32_t)(n_vals * 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float tot = 0;
    for (int r = 0; r <= reps; ++r) {
        cudaMemset(ctr, 0, 4);
        cudaEventRecord(a);
        if (variant == 0)
            k_raw<kBlk><<<grid, 256>>>(idx, E, nch, vals, out, ctr, gtotal, order, nblk);
        else if (variant == 3)
            k_meta<kBlk><<<grid, 256>>>(idx, mask, ord, E, nch, vals, sumc, carry, ctr, gtotal,
                                        order, nblk);
        else if (variant == 4)
            k_meta4<kBlk, 3, 0><<<grid, 256>>>(idx, mask, ord, E, nch, vals, sumc, carry, ctr,
                                               gtotal, order, nblk);
        else if (variant == 5)
            k_meta4<kBlk, 3, 1><<<grid, 256>>>(idx, mask, ord, E, nch, vals, sumc, carry, ctr,
                                               gtotal, order, nblk);
        else if (variant == 6)
            k_meta4<kBlk, 3, 2><<<grid, 256>>>(idx, mask, ord, E, nch, vals, sumc, carry, ctr,
                                               gtotal, order, nblk);
        else if (variant == 13)
            k_flag<kBlk, 1, 768, 1, 8192><<<148, 768, 8192 * 8 + 24 * 1024>>>(idx, ord, E, nch, vals, sumc, carry, ctr, gtotal, order, nblk);
        else if (variant == 14)
            k_flag<kBlk, 1, 768, 1, 16384><<<148, 768, 16384 * 8 + 24 * 1024>>>(idx, ord, E, nch, vals, sumc, carry, ctr, gtotal, order, nblk);
        else if (variant == 15)
            k_flag<kBlk, 1, 768, 1, 25088><<<148, 768, 25088 * 8 + 24 * 1024>>>(idx, ord, E, nch, vals, sumc, carry, ctr, gtotal, order, nblk);
        else if (variant == 16)
            k_flag<kBlk, 1, 768, 1, 0><<<148, 768, 24 * 1024>>>(idx, ord, E, nch, vals, sumc, carry, ctr, gtotal, order, nblk);
        else if (variant == 9)
            k_flag<kBlk, 1><<<grid, 256, 8 * 1024>>>(idx, ord, E, nch, vals, sumc, carry, ctr, gtotal,
                                           order, nblk);
        else if (variant == 10)
            k_flag<kBlk, 2><<<grid, 256, 8 * 1024>>>(idx, ord, E, nch, vals, sumc, carry, ctr, gtotal,
                                           order, nblk);
        else if (variant == 11)
            k_flag<32, 2><<<grid, 256, 8 * 1024>>>(idx, ord, E, nch, vals, sumc, carry, ctr, gtotal,
                                         order, (nch + 31) / 32);
        else if (variant == 12)
            k_flag<128, 2><<<grid, 256, 8 * 1024>>>(idx, ord, E, nch, vals, sumc, carry, ctr, gtotal,
                                          order, (nch + 127) / 128);
        else if (variant == 8)
            k_meta4<kBlk, 3, 3><<<grid, 256>>>(idx, mask, ord, E, nch, vals, sumc, carry, ctr,
                                               gtotal, order, nblk);
        else
            k_meta4<kBlk, 4, 0><<<grid, 256>>>(idx, mask, ord, E, nch, vals, sumc, carry, ctr,
                                               gtotal, order, nblk);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (r > 0) tot += ms;
    }
    return tot / reps;
}
}
