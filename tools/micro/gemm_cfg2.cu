// Micro-harness 2: the 3M batched GEMM under candidate tile configurations on
// the hot path's shapes with DISTINCT operands per task (as in the solver:
// every block's A and B live in HBM).  Prints ms per launch (5 launches after a
// warm-up) and the 6 M N K rate of the best configuration.
// build: make -C tools/micro gemm_cfg2; run on the GPU box.
#include <algorithm>
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
    if (cudaGetLastError() != cudaSuccess) return 1e9f;
    return ms / 5;
}
int main() {
    std::vector<Shape> shapes = {
        {"lu top", 288, 288, 320, 1000, 1}, {"lu 480x192", 480, 192, 128, 1000, 1},
        {"lu 544x64", 544, 64, 64, 1000, 1}, {"lu 160x160", 160, 160, 144, 1000, 1},
        {"solve 288", 288, 101, 320, 1000, 1}, {"solve 128", 128, 101, 192, 1000, 1},
        {"solve leaf", 64, 101, 64, 1000, 0}, {"schur 160", 608, 608, 160, 1000, 1},
        {"sample", 608, 64, 688, 1998, 0}, {"wb Z", 608, 96, 96, 250, 0}, {"wb cap", 96, 96, 608, 250, 1}};
    const char* names[] = {"64x32", "32x32", "64x64w8", "64x32w8", "64x32s3", "128x32w8", "64x32s4", "32x32s3"};
    cudaStream_t s; cudaStreamCreate(&s);
    DBuf<GemmTask> dt;
    printf("%-11s %4s %4s %4s %5s |", "shape", "M", "N", "K", "batch");
    for (auto n : names) printf(" %9s", n);
    printf("\n");
    for (auto sh : shapes) {
        const size_t a = size_t(sh.M) * sh.K, b = size_t(sh.K) * sh.N, c = size_t(sh.M) * sh.N;
        DBuf<cplx> A, B, Cm;
        A.ensure(a * sh.batch); B.ensure(b * sh.batch); Cm.ensure(c * sh.batch);
        cudaMemset(A.p, 0x3f, a * sh.batch * 16); cudaMemset(B.p, 0x3e, b * sh.batch * 16);
        cudaMemset(Cm.p, 0x3d, c * sh.batch * 16);
        std::vector<GemmTask> t(sh.batch);
        for (int i = 0; i < sh.batch; ++i) {
            t[i] = GemmTask{};
            t[i].nseg = 1;
            t[i].A[0] = A.p + i * a; t[i].lda[0] = sh.M; t[i].B[0] = B.p + i * b; t[i].ldb[0] = sh.K; t[i].K[0] = sh.K;
            t[i].C = Cm.p + i * c; t[i].ldc = sh.M;
        }
        dt.upload(t, s);
        float r[8] = {run<4, 2, 2, 2, 2, 3>(sh, dt.p, s), run<2, 2, 2, 2, 2, 4>(sh, dt.p, s),
                      run<4, 2, 2, 4, 2, 1>(sh, dt.p, s), run<2, 2, 4, 2, 2, 2>(sh, dt.p, s),
                      run<4, 2, 2, 2, 3, 2>(sh, dt.p, s), run<4, 2, 4, 2, 2, 1>(sh, dt.p, s),
                      run<4, 2, 2, 2, 4, 2>(sh, dt.p, s), run<2, 2, 2, 2, 3, 3>(sh, dt.p, s)};
        const double fl = 6.0 * sh.M * sh.N * double(sh.K) * sh.batch;
        printf("%-11s %4d %4d %4d %5d |", sh.what, sh.M, sh.N, sh.K, sh.batch);
        for (float x : r) printf(" %9.3f", x);
        const int bi = int(std::min_element(r, r + 8) - r);
        printf("  best %s %.1f TF/s (3M issued; %.0f%% of 37.1)\n", names[bi], fl / (r[bi] * 1e-3) / 1e12,
               100.0 * fl / (r[bi] * 1e-3) / 1e12 / 37.1);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
