// Per-launch time of the 16-column LU panel kernels (count = 1, 608 rows).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../paper_1410_5003_b200/csrc/linalg.cu"
#include "../../paper_1410_5003_b200/csrc/prof.cu"
using namespace qpsb;
__global__ void fill_rand(cplx* A, size_t n, unsigned seed, int dim) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        unsigned x = unsigned(i) * 2654435761u + seed;
        x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
        const size_t e = i % (size_t(dim) * dim);
        A[i] = cplx{(x & 0xffff) / 65536.0 - 0.5 + ((e % dim) == (e / dim) ? 4.0 : 0.0), ((x >> 16) & 0xffff) / 65536.0 - 0.5};
    }
}
int main() {
    const int n = 608;
    DBuf<cplx> A; A.ensure(size_t(n) * n);
    DBuf<int> piv, sing, map; piv.ensure(n); sing.ensure(1); map.ensure(64);
    DBuf<cplx*> dA; DBuf<int*> dP;
    std::vector<cplx*> hA{A.p}; std::vector<int*> hP{piv.p};
    dA.upload(hA, 0); dP.upload(hP, 0);
    fill_rand<<<256, 256>>>(A.p, size_t(n) * n, 7, n);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (const char* v : {"sm2", "reg"}) {
        setenv("QPS_PANEL", v, 1);
        // launch_panel_fast caches the env on first call: time each variant in its own process instead
        break;
    }
    const int R = 200;
    for (int i = 0; i < 5; ++i) launch_panel_fast(n, n, dA.p, dP.p, 0, 16, sing.p, map.p, 1, 0);
    cudaEventRecord(e0);
    for (int i = 0; i < R; ++i) launch_panel_fast(n, n, dA.p, dP.p, 0, 16, sing.p, map.p, 1, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("panel (%s): %.2f us/launch\n", getenv("QPS_PANEL") ? getenv("QPS_PANEL") : "sm2", 1000.0 * ms / R);
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
