// Micro-harness: batched complex GEMM shapes of the BCR/Schur hot path timed
// with CUDA events (build: make -C tools/micro; run on the GPU box).
#include <cstdio>
#include <vector>
#include "../../paper_1410_5003_b200/csrc/linalg.cu"
#include "../../paper_1410_5003_b200/csrc/prof.cu"
using namespace qpsb;
int main(int argc, char** argv) {
    struct Shape { int M, N, K, batch, nseg; double beta; };
    std::vector<Shape> shapes = {{608, 608, 608, 250, 1, 1.0}, {600, 600, 600, 250, 1, 1.0}, {600, 600, 600, 250, 2, 1.0}, {600, 600, 80, 500, 2, 1.0},
                                 {568, 600, 32, 250, 1, 1.0}, {312, 312, 288, 250, 1, 1.0}, {64, 600, 64, 500, 1, 0.0},
                                 {80, 1200, 80, 999, 1, 0.0}};
    cudaStream_t s; cudaStreamCreate(&s);
    DBuf<GemmTask> dt;
    for (auto sh : shapes) {
        const size_t a = size_t(sh.M) * sh.K, b = size_t(sh.K) * sh.N, c = size_t(sh.M) * sh.N;
        DBuf<cplx> A, B, Cm;
        A.ensure(a * 2); B.ensure(b * 2); Cm.ensure(c * sh.batch);
        cudaMemset(A.p, 0, a * 2 * 16); cudaMemset(B.p, 0, b * 2 * 16); cudaMemset(Cm.p, 0, c * sh.batch * 16);
        std::vector<GemmTask> t(sh.batch);
        for (int i = 0; i < sh.batch; ++i) {
            t[i] = GemmTask{};
            t[i].nseg = sh.nseg;
            for (int q = 0; q < sh.nseg; ++q) { t[i].A[q] = A.p + q * a; t[i].lda[q] = sh.M; t[i].B[q] = B.p + q * b; t[i].ldb[q] = sh.K; t[i].K[q] = sh.K; }
            t[i].C = Cm.p + i * c; t[i].ldc = sh.M;
        }
        cplx beta{sh.beta, 0};
        zgemm_batched(sh.M, sh.N, cplx{-1, 0}, beta, t, s, dt);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0, s);
        const int reps = 5;
        for (int r = 0; r < reps; ++r) zgemm_batched(sh.M, sh.N, cplx{-1, 0}, beta, t, s, dt);
        cudaEventRecord(e1, s); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double fl = 8.0 * sh.M * sh.N * double(sh.K) * sh.nseg * sh.batch * reps;
        printf("M=%4d N=%4d K=%4d x%d batch=%4d beta=%g : %7.3f ms/launch  %6.2f TF/s\n", sh.M, sh.N, sh.K, sh.nseg,
               sh.batch, sh.beta, ms / reps, fl / (ms * 1e-3) / 1e12);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
