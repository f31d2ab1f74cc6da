// Micro-harness: the 3M batched GEMM kernel under several tile configurations
// on the hot path's shapes (timed with CUDA events, 5 launches after one
// warm-up).  Prints ms per launch and complex-equivalent TF/s (8 M N K).
// build: make -C tools/micro gemm_cfg; run on the GPU box.
#include <cstdio>
#include <vector>
#include "../../paper_1410_5003_b200/csrc/linalg.cu"
#include "../../paper_1410_5003_b200/csrc/prof.cu"
using namespace qpsb;
struct Shape { const char* what; int M, N, K, batch; double beta; };
template <int A, int B, int C, int D, int E, int F>
float run(const Shape& sh, const GemmTask* dt, cudaStream_t s) {
    launch_z3<A, B, C, D, E, F>(sh.M, sh.N, cplx{-1, 0}, cplx{sh.beta, 0}, dt, sh.batch, s);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    for (int r = 0; r < 5; ++r) launch_z3<A, B, C, D, E, F>(sh.M, sh.N, cplx{-1, 0}, cplx{sh.beta, 0}, dt, sh.batch, s);
    cudaEventRecord(e1, s); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    return ms / 5;
}
int main() {
    std::vector<Shape> shapes = {
        {"lu top", 304, 304, 304, 1000, 1}, {"lu K16", 592, 16, 16, 1000, 1}, {"lu K32", 576, 32, 32, 1000, 1},
        {"lu K64", 544, 64, 64, 1000, 1}, {"lu mid", 448, 160, 160, 1000, 1}, {"trsm leaf", 64, 240, 64, 1000, 0},
        {"solve leaf", 64, 96, 64, 1000, 0}, {"solve upd", 320, 96, 288, 1000, 1},
        {"schur upd", 608, 608, 80, 1998, 1}, {"schur t1", 80, 1216, 160, 999, 0}, {"schur t2", 80, 1216, 80, 999, 0},
        {"schur resid", 160, 1216, 80, 999, 1}, {"sample", 608, 64, 608, 1998, 0}, {"R", 48, 608, 608, 1998, 0},
        {"qr VhY", 16, 48, 608, 1998, 0}, {"qr VW", 608, 48, 16, 1998, 1}, {"cores", 48, 48, 608, 1000, 0},
        {"wb cap", 96, 96, 608, 250, 1}, {"wb Z", 608, 96, 96, 250, 0}};
    cudaStream_t s; cudaStreamCreate(&s);
    DBuf<GemmTask> dt;
    printf("%-12s %5s %5s %5s %5s | %8s %8s %8s %8s %8s %8s %8s\n", "shape", "M", "N", "K", "batch", "64x32", "16x64",
           "64x64", "32x32", "128x32", "64x32s3", "32x64");
    for (auto sh : shapes) {
        const size_t a = size_t(sh.M) * sh.K, b = size_t(sh.K) * sh.N, c = size_t(sh.M) * sh.N;
        DBuf<cplx> A, B, Cm;
        A.ensure(a); B.ensure(b); Cm.ensure(c * sh.batch);
        cudaMemset(A.p, 0, a * 16); cudaMemset(B.p, 0, b * 16); cudaMemset(Cm.p, 0, c * sh.batch * 16);
        std::vector<GemmTask> t(sh.batch);
        for (int i = 0; i < sh.batch; ++i) {
            t[i] = GemmTask{};
            t[i].nseg = 1;
            t[i].A[0] = A.p; t[i].lda[0] = sh.M; t[i].B[0] = B.p; t[i].ldb[0] = sh.K; t[i].K[0] = sh.K;
            t[i].C = Cm.p + i * c; t[i].ldc = sh.M;
        }
        dt.upload(t, s);
        float r[7] = {run<4, 2, 2, 2, 2, 3>(sh, dt.p, s), run<2, 2, 1, 4, 2, 4>(sh, dt.p, s),
                      run<4, 4, 2, 2, 2, 2>(sh, dt.p, s), run<2, 2, 2, 2, 2, 4>(sh, dt.p, s),
                      run<4, 2, 4, 2, 2, 1>(sh, dt.p, s), run<4, 2, 2, 2, 3, 2>(sh, dt.p, s),
                      run<2, 4, 2, 2, 2, 3>(sh, dt.p, s)};
        const double fl = 8.0 * sh.M * sh.N * double(sh.K) * sh.batch;
        printf("%-12s %5d %5d %5d %5d |", sh.what, sh.M, sh.N, sh.K, sh.batch);
        for (float x : r) printf(" %8.3f", x);
        printf("   best %.1f TF/s\n", fl / (*std::min_element(r, r + 7) * 1e-3) / 1e12);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
