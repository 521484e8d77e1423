// Does a stream waiting on an event recorded between two large H2D copies on another stream
// start when the event fires, or only after both copies?  (create-phase overlap diagnosis)
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
__global__ void k_touch(int* p) { if (threadIdx.x == 0) p[0] += 1; }
int main(int argc, char** argv) {
    size_t bytes = (size_t)4 << 30;
    int mode = argc > 1 ? atoi(argv[1]) : 0;   // 0 cudaHostAlloc, 1 cudaHostRegister
    void *h1, *h2, *d1, *d2;
    if (mode == 0) { CK(cudaHostAlloc(&h1, bytes, 0)); CK(cudaHostAlloc(&h2, bytes, 0)); }
    else { h1 = malloc(bytes); h2 = malloc(bytes); CK(cudaHostRegister(h1, bytes, 0)); CK(cudaHostRegister(h2, bytes, 0)); }
    memset(h1, 1, bytes); memset(h2, 2, bytes);
    CK(cudaMalloc(&d1, bytes)); CK(cudaMalloc(&d2, bytes));
    int* dp; CK(cudaMalloc(&dp, 4));
    cudaStream_t s, cs;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    cudaEvent_t t0, a, b, c, ws, wk;
    for (cudaEvent_t* ev : {&t0, &b, &c, &ws, &wk}) CK(cudaEventCreate(ev));
    cudaEvent_t a_nt;
    CK(cudaEventCreateWithFlags(&a_nt, cudaEventDisableTiming));
    CK(cudaEventCreate(&a));
    const bool notiming = argc > 2 && atoi(argv[2]);
    for (int rep = 0; rep < 3; ++rep) {
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(t0, cs));
        CK(cudaMemcpyAsync(d1, h1, bytes, cudaMemcpyHostToDevice, cs));
        CK(cudaEventRecord(a, cs));
        CK(cudaEventRecord(a_nt, cs));
        CK(cudaMemcpyAsync(d2, h2, bytes, cudaMemcpyHostToDevice, cs));
        CK(cudaEventRecord(b, cs));
        CK(cudaStreamWaitEvent(s, notiming ? a_nt : a, 0));
        CK(cudaEventRecord(ws, s));
        k_touch<<<1, 32, 0, s>>>(dp);
        CK(cudaEventRecord(wk, s));
        CK(cudaDeviceSynchronize());
        float ta, tb, tw, tk;
        cudaEventElapsedTime(&ta, t0, a); cudaEventElapsedTime(&tb, t0, b);
        cudaEventElapsedTime(&tw, t0, ws); cudaEventElapsedTime(&tk, t0, wk);
        printf("notiming %d mode %d rep %d: copy1 done %.2f ms, copy2 done %.2f ms, waiter event %.2f ms, waiter kernel %.2f ms\n",
               (int)notiming, mode, rep, ta, tb, tw, tk);
    }
    return 0;
}
