// The create's exact stream pattern: which ingredient makes the waiter stream wait for every copy?
//   bit 0: destinations from cudaMallocAsync on s (else cudaMalloc)
//   bit 1: s records E, cs waits on E before the copies, cs re-records E after them
//   bit 2: torch-like: s is created with default flags (blocking)
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t err_ = (x); if (err_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(err_)); return 1; } } while (0)
int main(int argc, char** argv) {
    const int flags = argc > 1 ? atoi(argv[1]) : 0;
    size_t bytes = (size_t)4 << 30;
    void *h1, *h2;
    CK(cudaHostAlloc(&h1, bytes, 0)); CK(cudaHostAlloc(&h2, bytes, 0));
    memset(h1, 1, bytes); memset(h2, 2, bytes);
    cudaStream_t s, cs;
    if (flags & 4) CK(cudaStreamCreate(&s)); else CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    cudaEvent_t t0, a, E, ws;
    CK(cudaEventCreate(&t0)); CK(cudaEventCreate(&ws));
    CK(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&E, cudaEventDisableTiming));
    for (int rep = 0; rep < 3; ++rep) {
        CK(cudaDeviceSynchronize());
        void *d1, *d2;
        if (flags & 1) { CK(cudaMallocAsync(&d1, bytes, s)); CK(cudaMallocAsync(&d2, bytes, s)); }
        else { CK(cudaMalloc(&d1, bytes)); CK(cudaMalloc(&d2, bytes)); }
        if (flags & 2) { CK(cudaEventRecord(E, s)); CK(cudaStreamWaitEvent(cs, E, 0)); }
        else if (flags & 1) { CK(cudaStreamSynchronize(s)); }
        CK(cudaEventRecord(t0, cs));
        CK(cudaMemcpyAsync(d1, h1, bytes, cudaMemcpyHostToDevice, cs));
        CK(cudaEventRecord(a, cs));
        CK(cudaMemcpyAsync(d2, h2, bytes, cudaMemcpyHostToDevice, cs));
        if (flags & 2) CK(cudaEventRecord(E, cs));
        CK(cudaStreamWaitEvent(s, a, 0));
        CK(cudaEventRecord(ws, s));
        CK(cudaDeviceSynchronize());
        float tw;
        cudaEventElapsedTime(&tw, t0, ws);
        printf("flags %d rep %d: waiter released at %.2f ms (copy1 ~77, copy2 ~154)\n", flags, rep, tw);
        if (flags & 1) { CK(cudaFreeAsync(d1, s)); CK(cudaFreeAsync(d2, s)); }
        else { CK(cudaFree(d1)); CK(cudaFree(d2)); }
    }
    return 0;
}
