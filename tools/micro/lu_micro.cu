// Micro-harness: batched LU (lu_factor_batched) and LU solve with 2n right-hand
// sides at the cyclic-reduction shapes, timed with CUDA events.
// usage: ./lu_micro [n] ; QPS_LU=rec|rl selects the factorization
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../paper_1410_5003_b200/csrc/linalg.cu"
#include "../../paper_1410_5003_b200/csrc/prof.cu"
using namespace qpsb;

__global__ void fill_rand(cplx* A, size_t n, unsigned seed, int dim, int ld) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        unsigned x = unsigned(i) * 2654435761u + seed;
        x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
        const double r = (x & 0xffff) / 65536.0 - 0.5, im = ((x >> 16) & 0xffff) / 65536.0 - 0.5;
        const size_t e = i % (size_t(ld) * dim);
        const bool diag = (e % ld) == (e / ld);
        A[i] = cplx{r + (diag ? 4.0 : 0.0), im};
    }
}

int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 608;
    cudaStream_t s;
    cudaStreamCreate(&s);
    Workspace ws;
    for (int count : {1, 4, 16, 62, 125, 500}) {
        const size_t nn = size_t(n) * n;
        DBuf<cplx> A, B, Dinv;
        DBuf<int> piv, sing;
        A.ensure(nn * count);
        B.ensure(nn * 2 * count);
        Dinv.ensure(lu_dinv_elems(n) * count);
        piv.ensure(size_t(n) * count);
        sing.ensure(count);
        std::vector<cplx*> hA, hD, hB;
        std::vector<int*> hP;
        for (int b = 0; b < count; ++b) {
            hA.push_back(A.p + b * nn);
            hD.push_back(Dinv.p + b * lu_dinv_elems(n));
            hP.push_back(piv.p + size_t(b) * n);
            hB.push_back(B.p + 2 * b * nn);
        }
        cudaEvent_t e0, e1, e2;
        cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&e2);
        float tf = 0, ts = 0;
        const int reps = 3;
        for (int r = 0; r <= reps; ++r) {
            fill_rand<<<1024, 256, 0, s>>>(A.p, nn * count, 17 + r, n, n);
            fill_rand<<<1024, 256, 0, s>>>(B.p, nn * 2 * count, 99 + r, n, n);
            sing.zero(s);
            cudaEventRecord(e0, s);
            lu_factor_batched(n, n, hA, hP, hD, sing.p, s, ws);
            cudaEventRecord(e1, s);
            lu_solve_batched(n, n, hA, hP, hD, hB, n, 2 * n, s, ws);
            cudaEventRecord(e2, s);
            cudaEventSynchronize(e2);
            float a, b;
            cudaEventElapsedTime(&a, e0, e1);
            cudaEventElapsedTime(&b, e1, e2);
            if (r) { tf += a; ts += b; }
        }
        tf /= reps; ts /= reps;
        const double flf = 8.0 / 3.0 * double(n) * n * n * count, fls = 16.0 * double(n) * n * n * count;
        printf("n=%d count=%4d  factor %8.3f ms (%6.2f TF/s)  solve(2n rhs) %8.3f ms (%6.2f TF/s)\n", n, count, tf,
               flf / (tf * 1e-3) / 1e12, ts, fls / (ts * 1e-3) / 1e12);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
