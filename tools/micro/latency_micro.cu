// Latency probes for the single-CTA LU panel: empty launch, barriers, shuffles,
// panel load/store, FP64 division, at 640 threads (tools/micro, GPU only).
#include <cstdio>
#include <cuda_runtime.h>
struct cplx { double re, im; };
__global__ void k_empty(int* o) { if (threadIdx.x == 1000) o[0] = 1; }
__global__ void k_bar(int* o, int steps) {
    __shared__ double sh[32];
    double v = threadIdx.x;
    for (int k = 0; k < steps; ++k) {
        for (int s = 16; s > 0; s >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, s));
        if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
        __syncthreads();
        v += sh[k & 15];
    }
    if (v == -1.0) o[0] = 1;
}
__global__ void k_load(const cplx* A, cplx* B, int rows, int w, int ld) {
    extern __shared__ cplx p[];
    const int t = threadIdx.x;
    if (t < rows) for (int j = 0; j < w; ++j) p[j * rows + t] = A[size_t(j) * ld + t];
    __syncthreads();
    if (t < rows) for (int j = 0; j < w; ++j) B[size_t(j) * ld + t] = p[j * rows + t];
}
__global__ void k_div(const double* a, double* o, int steps) {
    double x = a[threadIdx.x], y = 1.0;
    for (int k = 0; k < steps; ++k) y = x / (y + 1.0);
    o[threadIdx.x] = y;
}
int main() {
    int* o; cudaMalloc(&o, 4096);
    cplx *A, *B; cudaMalloc(&A, 608 * 608 * 16); cudaMalloc(&B, 608 * 608 * 16);
    double* d; cudaMalloc(&d, 8192); cudaMemset(d, 0, 8192);
    cudaFuncSetAttribute(k_load, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto timeit = [&](const char* name, auto launch) {
        for (int i = 0; i < 10; ++i) launch();
        cudaEventRecord(e0);
        const int R = 200;
        for (int i = 0; i < R; ++i) launch();
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("%-28s %8.2f us/launch\n", name, 1000.0 * ms / R);
    };
    timeit("empty 640 thr", [&] { k_empty<<<1, 640>>>(o); });
    timeit("16 barrier+shfl steps", [&] { k_bar<<<1, 640>>>(o, 16); });
    timeit("160 barrier+shfl steps", [&] { k_bar<<<1, 640>>>(o, 160); });
    timeit("panel load+store 608x16", [&] { k_load<<<1, 640, 608 * 16 * 16>>>(A, B, 608, 16, 608); });
    timeit("16 dependent fp64 div", [&] { k_div<<<1, 640>>>(d, d + 640, 16); });
    timeit("160 dependent fp64 div", [&] { k_div<<<1, 640>>>(d, d + 640, 160); });
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
