// Micro-harness: the 3M batched GEMM with cp.async staging vs TMA bulk-copy
// staging (kBulk) on the hot path's shapes plus ragged ones (M, N, K not tile
// multiples).  Distinct random operands per task; the two outputs must agree
// bitwise (same products in the same order).  Prints ms per launch of each.
// build: make -C tools/micro gemm_bulk; run on the GPU box.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>
#include "../../paper_1410_5003_b200/csrc/linalg.cu"
#include "../../paper_1410_5003_b200/csrc/prof.cu"
using namespace qpsb;
struct Shape { const char* what; int M, N, K, batch; double beta; };
template <int A, int B, int C, int D, int E, int F, bool BULK>
float run(const Shape& sh, const GemmTask* dt, cudaStream_t s, int reps) {
    launch_z3_impl<A, B, C, D, E, F, false, BULK>(sh.M, sh.N, cplx{-1, 0.5}, cplx{sh.beta, 0}, dt, sh.batch, s,
                                                  nullptr, nullptr);
    if (reps == 0) { cudaStreamSynchronize(s); return 0.f; }
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    for (int r = 0; r < reps; ++r)
        launch_z3_impl<A, B, C, D, E, F, false, BULK>(sh.M, sh.N, cplx{-1, 0.5}, cplx{sh.beta, 0}, dt, sh.batch, s,
                                                      nullptr, nullptr);
    cudaEventRecord(e1, s); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (cudaGetLastError() != cudaSuccess) return 1e9f;
    return ms / reps;
}
template <int A, int B, int C, int D, int E, int F>
void both(const char* cfg, const Shape& sh, const GemmTask* dt, cudaStream_t s, DBuf<cplx>& Cm, size_t csz,
          const std::vector<cplx>& c0) {
    std::vector<cplx> r0(csz), r1(csz);
    // correctness: one launch each from the same C
    cudaMemcpy(Cm.p, c0.data(), csz * 16, cudaMemcpyHostToDevice);
    run<A, B, C, D, E, F, false>(sh, dt, s, 0);
    cudaMemcpy(r0.data(), Cm.p, csz * 16, cudaMemcpyDeviceToHost);
    cudaMemcpy(Cm.p, c0.data(), csz * 16, cudaMemcpyHostToDevice);
    run<A, B, C, D, E, F, true>(sh, dt, s, 0);
    cudaMemcpy(r1.data(), Cm.p, csz * 16, cudaMemcpyDeviceToHost);
    size_t bad = 0;
    for (size_t i = 0; i < csz; ++i) bad += memcmp(&r0[i], &r1[i], 16) != 0;
    const bool timing = sh.batch >= 250;
    float t0 = timing ? run<A, B, C, D, E, F, false>(sh, dt, s, 5) : 0.f;
    float t1 = timing ? run<A, B, C, D, E, F, true>(sh, dt, s, 5) : 0.f;
    const double fl = 6.0 * sh.M * sh.N * double(sh.K) * sh.batch;
    printf("%-11s %4d %4d %4d %5d %-8s cp.async %8.3f ms  bulk %8.3f ms  (%.1f -> %.1f TF/s)  mismatches %zu %s\n",
           sh.what, sh.M, sh.N, sh.K, sh.batch, cfg, t0, t1, timing ? fl / (t0 * 1e-3) / 1e12 : 0.0,
           timing ? fl / (t1 * 1e-3) / 1e12 : 0.0, bad, cudaGetErrorString(cudaGetLastError()));
}
int main() {
    std::vector<Shape> shapes = {
        {"ragged", 37, 29, 21, 7, 1}, {"ragged2", 100, 77, 45, 5, 0}, {"ragged3", 130, 5, 300, 3, 1},
        {"lu top", 288, 288, 320, 1000, 1}, {"lu 480x192", 480, 192, 128, 1000, 1},
        {"lu 544x64", 544, 64, 64, 1000, 1}, {"lu 160x160", 160, 160, 144, 1000, 1},
        {"solve 288", 288, 85, 320, 1000, 1}, {"schur 160", 600, 600, 160, 1000, 1},
        {"thin 80", 80, 600, 600, 1000, 0}, {"wb cap", 80, 80, 600, 250, 1}, {"rhs 8", 600, 5, 600, 1000, 1}};
    cudaStream_t s; cudaStreamCreate(&s);
    DBuf<GemmTask> dt;
    std::mt19937_64 rng(7);
    std::uniform_real_distribution<double> U(-1, 1);
    for (auto sh : shapes) {
        const size_t a = size_t(sh.M) * sh.K, b = size_t(sh.K) * sh.N, c = size_t(sh.M) * sh.N;
        DBuf<cplx> A, B, Cm;
        A.ensure(a * sh.batch); B.ensure(b * sh.batch); Cm.ensure(c * sh.batch);
        auto fill = [&](DBuf<cplx>& X, size_t n) {
            std::vector<cplx> h(n);
            for (auto& v : h) v = cplx{U(rng), U(rng)};
            cudaMemcpy(X.p, h.data(), n * 16, cudaMemcpyHostToDevice);
            return h;
        };
        fill(A, a * sh.batch); fill(B, b * sh.batch);
        std::vector<cplx> c0 = fill(Cm, c * sh.batch);
        std::vector<GemmTask> t(sh.batch);
        for (int i = 0; i < sh.batch; ++i) {
            t[i] = GemmTask{};
            t[i].nseg = 1;
            t[i].A[0] = A.p + i * a; t[i].lda[0] = sh.M; t[i].B[0] = B.p + i * b; t[i].ldb[0] = sh.K; t[i].K[0] = sh.K;
            t[i].C = Cm.p + i * c; t[i].ldc = sh.M;
        }
        dt.upload(t, s);
        const size_t csz = c * sh.batch;
        both<2, 2, 2, 2, 2, 4>("32x32", sh, dt.p, s, Cm, csz, c0);
        both<2, 2, 2, 2, 3, 3>("32x32s3", sh, dt.p, s, Cm, csz, c0);
        both<2, 2, 1, 4, 2, 4>("16x64", sh, dt.p, s, Cm, csz, c0);
        both<4, 2, 2, 2, 2, 3>("64x32", sh, dt.p, s, Cm, csz, c0);
        both<4, 2, 2, 2, 3, 2>("64x32s3", sh, dt.p, s, Cm, csz, c0);
        if (sh.N <= 8) both<4, 1, 4, 1, 2, 3>("128x8", sh, dt.p, s, Cm, csz, c0);
        if (sh.M <= 48) both<6, 2, 1, 4, 2, 2>("48x64", sh, dt.p, s, Cm, csz, c0);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
