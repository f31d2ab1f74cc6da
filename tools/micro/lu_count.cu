// lu_factor_batched at one batch size, for ncu launch lists (QPS_LU selects the variant)
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
int main(int argc, char** argv) {
    const int n = 608, count = argc > 1 ? atoi(argv[1]) : 500;
    const int solve = argc > 2 ? atoi(argv[2]) : 0;
    cudaStream_t s; cudaStreamCreate(&s);
    Workspace ws;
    const size_t nn = size_t(n) * n;
    DBuf<cplx> A, B, Dinv; DBuf<int> piv, sing;
    A.ensure(nn * count); B.ensure(nn * 2 * count); Dinv.ensure(lu_dinv_elems(n) * count);
    piv.ensure(size_t(n) * count); sing.ensure(count);
    std::vector<cplx*> hA, hD, hB; std::vector<int*> hP;
    for (int b = 0; b < count; ++b) {
        hA.push_back(A.p + b * nn); hD.push_back(Dinv.p + b * lu_dinv_elems(n));
        hP.push_back(piv.p + size_t(b) * n); hB.push_back(B.p + 2 * b * nn);
    }
    fill_rand<<<1024, 256, 0, s>>>(A.p, nn * count, 17, n);
    fill_rand<<<1024, 256, 0, s>>>(B.p, nn * 2 * count, 99, n);
    sing.zero(s);
    lu_factor_batched(n, n, hA, hP, hD, sing.p, s, ws);
    if (solve) lu_solve_batched(n, n, hA, hP, hD, hB, n, 2 * n, s, ws);
    cudaStreamSynchronize(s);
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
