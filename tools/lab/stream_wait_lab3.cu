// The create's copy sequence: offsets, one 7.5 GB index copy, event, 8 weight windows (an event
// created and recorded after each).  bit 0: index copy split into 4 GB pieces; bit 1: no events
// created between the window copies (pre-created).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>
__global__ void k_noop() {}
#define CK(x) do { cudaError_t err_ = (x); if (err_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(err_)); return 1; } } while (0)
int main(int argc, char** argv) {
    const int flags = argc > 1 ? atoi(argv[1]) : 0;
    const size_t E = 1879040606ull, N = 67108864ull;
    void *h_off, *h_idx, *h_w, *d_off, *d_idx, *d_w;
    CK(cudaHostAlloc(&h_off, (N + 1) * 4, 0)); CK(cudaHostAlloc(&h_idx, E * 4, 0)); CK(cudaHostAlloc(&h_w, E * 4, 0));
    memset(h_idx, 1, E * 4); memset(h_w, 2, E * 4);
    CK(cudaMalloc(&d_off, (N + 1) * 4)); CK(cudaMalloc(&d_idx, E * 4)); CK(cudaMalloc(&d_w, E * 4));
    cudaStream_t s, cs;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    cudaEvent_t t0, up_idx, ws, mk;
    CK(cudaEventCreate(&t0)); CK(cudaEventCreate(&ws)); CK(cudaEventCreate(&mk));
    CK(cudaEventCreateWithFlags(&up_idx, cudaEventDisableTiming));
    for (int rep = 0; rep < 3; ++rep) {
        CK(cudaDeviceSynchronize());
        std::vector<cudaEvent_t> pre(8);
        for (auto& e : pre) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        if (flags & 4) CK(cudaMemcpyAsync(d_off, h_off, (N + 1) * 4, cudaMemcpyHostToDevice, s));
        if (flags & 8) {   // the create's ordering: s -> event -> cs waits before its copies
            cudaEvent_t ev;
            CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            CK(cudaEventRecord(ev, s));
            CK(cudaStreamWaitEvent(cs, ev, 0));
        }
        CK(cudaEventRecord(t0, cs));
        CK(cudaMemcpyAsync(d_off, h_off, (N + 1) * 4, cudaMemcpyHostToDevice, cs));
        if (flags & 1) {
            const size_t piece = (size_t)1 << 30;   // elements of 4 B = 4 GiB
            for (size_t lo = 0; lo < E; lo += piece) {
                const size_t n = E - lo < piece ? E - lo : piece;
                CK(cudaMemcpyAsync((int*)d_idx + lo, (int*)h_idx + lo, n * 4, cudaMemcpyHostToDevice, cs));
            }
        } else {
            CK(cudaMemcpyAsync(d_idx, h_idx, E * 4, cudaMemcpyHostToDevice, cs));
        }
        CK(cudaEventRecord(up_idx, cs));
        CK(cudaEventRecord(mk, cs));
        for (int c = 0; c < 8; ++c) {
            const size_t lo = E * c / 8, hi = E * (c + 1) / 8;
            CK(cudaMemcpyAsync((int*)d_w + lo, (int*)h_w + lo, (hi - lo) * 4, cudaMemcpyHostToDevice, cs));
            cudaEvent_t e = pre[c];
            if (!(flags & 2)) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            CK(cudaEventRecord(e, cs));
        }
        if (flags & 16) k_noop<<<1, 32, 0, s>>>();
        if (flags & 32) CK(cudaMemsetAsync(d_off, 0, 4, s));
        CK(cudaStreamWaitEvent(s, up_idx, 0));
        CK(cudaEventRecord(ws, s));
        CK(cudaDeviceSynchronize());
        float tw, tm;
        cudaEventElapsedTime(&tw, t0, ws);
        cudaEventElapsedTime(&tm, t0, mk);
        printf("flags %d rep %d: structure uploaded %.2f ms, waiter released %.2f ms\n", flags, rep, tm, tw);
    }
    return 0;
}
