// tools/compress_lab.cu -- lab: does a compressed CSC index stream lower the PageRank gather's
// ceiling?  Every warp walks 128-edge chunks (global grid) summing vals[idx[e]], the range
// kernel's memory pipeline without row logic (tools/tma_lab.cu v0), with the indices read as
//   v0: raw int32 (7.5 GB at cfg4);
//   v1: per-chunk frame of reference: base = min, b = bits(max - min), 128 b-bit fields
//       (4 b u32 words), header {word offset, base | b << 26};
//   v2: as v1, but chunks inside one row (no row starts after their first edge) store the
//       deltas to the previous edge (the row is sorted), decoded by a 128-wide prefix sum.
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
__device__ __forceinline__ uint32_t ld_s(const uint32_t* p, uint64_t pol) {
    uint32_t r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ uint2 ld_s2(const uint2* p, uint64_t pol) {
    uint2 r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
        : "=r"(r.x), "=r"(r.y) : "l"(p), "l"(pol));
    return r;
}
// the range kernel's gather policies: the first 64 MiB of the outbox evict-last in L2 (rest
// evict-first), the hottest 8192 vertices cached in L1
__device__ uint64_t g_pol;
__device__ __forceinline__ uint64_t pol_range(const void* base, uint32_t hot, uint32_t total) {
    uint64_t p;
    asm volatile("createpolicy.range.global.L2::evict_last.L2::evict_first.b64 %0, [%1], %2, %3;"
                 : "=l"(p) : "l"(base), "r"(hot), "r"(total));
    return p;
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
__device__ __forceinline__ int bits_of(uint32_t x) { return x ? 32 - __clz(x) : 0; }

// ---- encoding (one warp per chunk) -------------------------------------------------------
// rowstart[e] = 1 if e is the first edge of its row.  mode 1: FOR only; mode 2: delta for
// one-row chunks.  Pass 1 writes b (and the kind bit) per chunk; the host scans 4 b words.
__global__ void k_enc_width(const int32_t* __restrict__ idx, const uint8_t* __restrict__ rowstart,
                            int64_t E, int64_t nch, int mode, uint32_t* hdr_b, int64_t* words) {
    const int lane = threadIdx.x & 31;
    const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (c >= nch) return;
    const int64_t e0 = c * kChunk;
    uint32_t mn = 0xffffffffu, mx = 0;
    bool inner_start = false;
    uint32_t dmax = 0;
    for (int k = 0; k < 4; ++k) {
        const int64_t e = e0 + 32 * k + lane;
        if (e < E) {
            const uint32_t v = (uint32_t)idx[e];
            mn = min(mn, v);
            mx = max(mx, v);
            if (e > e0) {
                if (rowstart[e]) inner_start = true;
                else dmax = max(dmax, v - (uint32_t)idx[e - 1]);
            }
        }
    }
    mn = __reduce_min_sync(kFull, mn);
    mx = __reduce_max_sync(kFull, mx);
    dmax = __reduce_max_sync(kFull, dmax);
    inner_start = __any_sync(kFull, inner_start);
    int b = bits_of(mx - mn);
    uint32_t kind = 0;
    if (mode == 2 && !inner_start && bits_of(dmax) < b) {
        b = bits_of(dmax);
        kind = 1;
    }
    if (lane == 0) {
        hdr_b[c] = (uint32_t)b | (kind << 5);
        words[c] = 4 * b;
        // base: min (FOR) or the first edge (delta)
    }
}

__global__ void k_enc_pack(const int32_t* __restrict__ idx, int64_t E, int64_t nch,
                           const uint32_t* __restrict__ hdr_b, const int64_t* __restrict__ woff,
                           uint2* hdr, uint32_t* payload) {
    const int lane = threadIdx.x & 31;
    const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (c >= nch) return;
    const int64_t e0 = c * kChunk;
    const int b = hdr_b[c] & 31, kind = hdr_b[c] >> 5;
    uint32_t mn = 0xffffffffu;
    for (int k = 0; k < 4; ++k) {
        const int64_t e = e0 + 32 * k + lane;
        if (e < E) mn = min(mn, (uint32_t)idx[e]);
    }
    mn = __reduce_min_sync(kFull, mn);
    const uint32_t base = kind ? (uint32_t)idx[e0] : mn;
    const int64_t w0 = woff[c];
    if (lane == 0) hdr[c] = make_uint2((uint32_t)w0, base | ((uint32_t)b << 26) | ((uint32_t)kind << 31));
    if (b == 0) return;
    for (int k = 0; k < 4; ++k) {
        const int p = 32 * k + lane;
        const int64_t e = e0 + p;
        uint32_t f = 0;
        if (e < E) f = kind ? (p == 0 ? 0u : (uint32_t)idx[e] - (uint32_t)idx[e - 1]) : (uint32_t)idx[e] - mn;
        const uint32_t bit = (uint32_t)p * b;
        const uint32_t w = bit >> 5, sh = bit & 31;
        if (f) {
            atomicOr(payload + w0 + w, f << sh);
            if (sh + b > 32) atomicOr(payload + w0 + w + 1, f >> (32 - sh));
        }
    }
}

// ---- decode --------------------------------------------------------------------------
struct Raw4 { uint32_t lo[4], hi[4]; };

__device__ __forceinline__ void load_payload(const uint32_t* __restrict__ pay, uint2 h, int lane,
                                             uint64_t pol, Raw4& R) {
    const uint32_t b = (h.y >> 26) & 31;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint32_t bit = (uint32_t)(32 * k + lane) * b;
        const uint32_t w = h.x + (bit >> 5);
        R.lo[k] = b ? ld_s(pay + w, pol) : 0u;
        R.hi[k] = (b && (bit & 31) + b > 32) ? ld_s(pay + w + 1, pol) : 0u;
    }
}

template <bool kDelta>
__device__ __forceinline__ void decode(uint2 h, int lane, const Raw4& R, int32_t (&ix)[4]) {
    const uint32_t b = (h.y >> 26) & 31;
    const uint32_t base = h.y & ((1u << 26) - 1);
    const uint32_t mask = b >= 32 ? 0xffffffffu : ((1u << b) - 1);
    uint32_t f[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint32_t sh = ((uint32_t)(32 * k + lane) * b) & 31;
        f[k] = __funnelshift_r(R.lo[k], R.hi[k], sh) & mask;
    }
    if (kDelta && (h.y >> 31)) {
        // inclusive prefix sum over the 128 positions (4 warp scans, chained)
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t y = __shfl_up_sync(kFull, f[k], d);
                if (lane >= d) f[k] += y;
            }
        }
        uint32_t carry = base;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            f[k] += carry;
            carry = __shfl_sync(kFull, f[k], 31);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) ix[k] = (int32_t)f[k];
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) ix[k] = (int32_t)(base + f[k]);
    }
}

template <int kBlk>
__global__ void __launch_bounds__(256) k_raw(const int32_t* __restrict__ idx, int64_t E,
                                             int64_t nch, const double* __restrict__ vals,
                                             double* out, unsigned long long* cks, int* ctr, uint32_t gtotal) {
    const int lane = threadIdx.x & 31;
    const uint64_t pol = pol_first();
    const uint64_t gp = pol_range(vals, 64u << 20, gtotal);
    double acc = 0;
    unsigned long long ck = 0;
    for (;;) {
        int q = lane == 0 ? atomicAdd(ctr, 1) : 0;
        q = __shfl_sync(kFull, q, 0);
        const int64_t c0 = (int64_t)q * kBlk;
        if (c0 >= nch) break;
        const int64_t c1 = c0 + kBlk < nch ? c0 + kBlk : nch;
        int32_t a[4], bq[4];
        auto ld = [&](int64_t c, int32_t (&r)[4]) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int64_t e = c * kChunk + 32 * k + lane;
                r[k] = (c < c1 && e < E) ? (int32_t)ld_s((const uint32_t*)idx + e, pol) : -1;
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
            for (int k = 0; k < 4; ++k) {
                gn[k] = bq[k] >= 0 ? ld_valp(vals, bq[k], gp) : 0.0;
                if (bq[k] >= 0) ck += (unsigned)bq[k];
            }
            if (c == c0) {
#pragma unroll
                for (int k = 0; k < 4; ++k) if (a[k] >= 0) ck += (unsigned)a[k];
            }
            ld(c + 2, bq);
            acc += (g[0] + g[1]) + (g[2] + g[3]);
#pragma unroll
            for (int k = 0; k < 4; ++k) g[k] = gn[k];
        }
    }
    out[(int64_t)blockIdx.x * blockDim.x + threadIdx.x] = acc;
    atomicAdd(cks, ck);
}

template <int kBlk, bool kDelta>
__global__ void __launch_bounds__(256) k_packed(const uint2* __restrict__ hdr,
                                                const uint32_t* __restrict__ pay, int64_t E,
                                                int64_t nch, const double* __restrict__ vals,
                                                double* out, unsigned long long* cks, int* ctr, uint32_t gtotal) {
    const int lane = threadIdx.x & 31;
    const uint64_t pol = pol_first();
    const uint64_t gp = pol_range(vals, 64u << 20, gtotal);
    double acc = 0;
    unsigned long long ck = 0;
    for (;;) {
        int q = lane == 0 ? atomicAdd(ctr, 1) : 0;
        q = __shfl_sync(kFull, q, 0);
        const int64_t c0 = (int64_t)q * kBlk;
        if (c0 >= nch) break;
        const int64_t c1 = c0 + kBlk < nch ? c0 + kBlk : nch;
        // headers 3 ahead, payload 2 ahead, decoded indices 1 ahead (gathered)
        uint2 h0 = ld_s2(hdr + c0, pol);
        uint2 h1 = c0 + 1 < c1 ? ld_s2(hdr + c0 + 1, pol) : make_uint2(0, 0);
        uint2 h2 = c0 + 2 < c1 ? ld_s2(hdr + c0 + 2, pol) : make_uint2(0, 0);
        Raw4 R0, R1;
        load_payload(pay, h0, lane, pol, R0);
        load_payload(pay, h1, lane, pol, R1);
        int32_t ix[4];
        decode<kDelta>(h0, lane, R0, ix);
        double g[4];
        auto valid = [&](int64_t c, int k) { return c * kChunk + 32 * k + lane < E; };
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const bool v = valid(c0, k);
            g[k] = v ? ld_valp(vals, ix[k], gp) : 0.0;
            if (v) ck += (unsigned)ix[k];
        }
        for (int64_t c = c0; c < c1; ++c) {
            double gn[4];
            if (c + 1 < c1) {
                decode<kDelta>(h1, lane, R1, ix);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const bool v = valid(c + 1, k);
                    gn[k] = v ? ld_valp(vals, ix[k], gp) : 0.0;
                    if (v) ck += (unsigned)ix[k];
                }
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) gn[k] = 0.0;
            }
            h1 = h2;
            if (c + 2 < c1) load_payload(pay, h2, lane, pol, R1);
            h2 = c + 3 < c1 ? ld_s2(hdr + c + 3, pol) : make_uint2(0, 0);
            acc += (g[0] + g[1]) + (g[2] + g[3]);
#pragma unroll
            for (int k = 0; k < 4; ++k) g[k] = gn[k];
        }
    }
    out[(int64_t)blockIdx.x * blockDim.x + threadIdx.x] = acc;
    atomicAdd(cks, ck);
}

extern "C" {
void enc_width(const int32_t* idx, const uint8_t* rs, int64_t E, int mode, uint32_t* hdr_b,
               int64_t* words) {
    const int64_t nch = (E + kChunk - 1) / kChunk;
    k_enc_width<<<(unsigned)((nch * 32 + 255) / 256), 256>>>(idx, rs, E, nch, mode, hdr_b, words);
}
void enc_pack(const int32_t* idx, int64_t E, const uint32_t* hdr_b, const int64_t* woff,
              uint2* hdr, uint32_t* pay) {
    const int64_t nch = (E + kChunk - 1) / kChunk;
    k_enc_pack<<<(unsigned)((nch * 32 + 255) / 256), 256>>>(idx, E, nch, hdr_b, woff, hdr, pay);
}
// variant 0 raw, 1 FOR, 2 FOR + delta; returns ms per pass (mean of reps), checksum out
float run_lab(int variant, const int32_t* idx, const uint2* hdr, const uint32_t* pay, int64_t E,
              const double* vals, int64_t n_vals, double* out, unsigned long long* cks, int* ctr, int ctas_per_sm,
              int reps) {
    const int64_t nch = (E + kChunk - 1) / kChunk;
    const int grid = 148 * ctas_per_sm;
    const uint32_t gtotal = (uint32_t)(n_vals * 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float tot = 0;
    for (int r = 0; r <= reps; ++r) {
        cudaMemset(ctr, 0, 4);
        cudaMemset(cks, 0, 8);
        cudaEventRecord(a);
        if (variant == 0) k_raw<64><<<grid, 256>>>(idx, E, nch, vals, out, cks, ctr, gtotal);
        else if (variant == 1) k_packed<64, false><<<grid, 256>>>(hdr, pay, E, nch, vals, out, cks, ctr, gtotal);
        else k_packed<64, true><<<grid, 256>>>(hdr, pay, E, nch, vals, out, cks, ctr, gtotal);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (r > 0) tot += ms;
    }
    return tot / reps;
}
}
