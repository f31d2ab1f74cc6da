// Batched complex FP64 dense linear algebra on sm_100a.
//
// FP64 on Blackwell: tcgen05.mma has no f64 kind, so the tensor path for
// double precision is the warp-level mma.sync m8n8k4 f64 (SASS DMMA).  The
// batched complex GEMM (zgemm3m_t_kernel) issues three real DMMAs per complex
// 8x8x4 step (Gauss product); the four-DMMA kernel (zgemm_kernel,
//   Cr += Ar Br - Ai Bi,  Ci += Ar Bi + Ai Br) stays selectable.
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>

#include "cmath.cuh"
#include "linalg.cuh"
#include "prof.h"

namespace qpsb {

std::atomic<uint64_t> g_zgemm_launches{0};  // ncu --launch-skip bookkeeping (QPS_TRACE_LAUNCH)

namespace {

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

constexpr int BM = 64, BN = 64, BK = 8, LDS = 72;

__global__ void __launch_bounds__(128, 2) zgemm_kernel(int M, int N, cplx alpha, cplx beta,
                                                       const GemmTask* __restrict__ tasks, int tiles_m) {
    __shared__ double As[2][2][BK][LDS];
    __shared__ double Bs[2][2][BK][LDS];
    const GemmTask& T = tasks[blockIdx.y];
    const int tm = blockIdx.x % tiles_m, tn = blockIdx.x / tiles_m;
    const int m0 = tm * BM, n0 = tn * BN;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
    double acc[4][4][2][2];  // [i][j][re/im][c0/c1]
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0][0] = acc[i][j][0][1] = acc[i][j][1][0] = acc[i][j][1][1] = 0.0;

    const int nseg = T.nseg;
    for (int sgi = 0; sgi < nseg; ++sgi) {
        const cplx* __restrict__ A = T.A[sgi];
        const cplx* __restrict__ B = T.B[sgi];
        const int lda = T.lda[sgi], ldb = T.ldb[sgi], K = T.K[sgi];
        const int nchunks = (K + BK - 1) / BK;
        double2 ra[4], rb[4];
        auto load = [&](int c) {
            const int k0 = c * BK;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int idx = tid + 128 * i;
                const int row = idx & 63, kk = idx >> 6;
                const int gm = m0 + row, gk = k0 + kk;
                ra[i] = (gm < M && gk < K) ? __ldg(reinterpret_cast<const double2*>(A + size_t(gk) * lda + gm))
                                           : make_double2(0.0, 0.0);
                const int kb = idx & 7, col = idx >> 3;
                const int gn = n0 + col, gkb = k0 + kb;
                rb[i] = (gn < N && gkb < K) ? __ldg(reinterpret_cast<const double2*>(B + size_t(gn) * ldb + gkb))
                                            : make_double2(0.0, 0.0);
            }
        };
        auto stash = [&](int buf) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int idx = tid + 128 * i;
                const int row = idx & 63, kk = idx >> 6;
                As[buf][0][kk][row] = ra[i].x;
                As[buf][1][kk][row] = ra[i].y;
                const int kb = idx & 7, col = idx >> 3;
                Bs[buf][0][kb][col] = rb[i].x;
                Bs[buf][1][kb][col] = rb[i].y;
            }
        };
        if (nchunks > 0) {
            load(0);
            stash(0);
        }
        __syncthreads();
        for (int c = 0; c < nchunks; ++c) {
            const int buf = c & 1;
            if (c + 1 < nchunks) load(c + 1);
#pragma unroll
            for (int ks = 0; ks < BK; ks += 4) {
                const int kq = ks + (lane & 3), r = lane >> 2;
                double ar[4], ai[4], nai[4], br[4], bi[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    ar[i] = As[buf][0][kq][wm + 8 * i + r];
                    ai[i] = As[buf][1][kq][wm + 8 * i + r];
                    nai[i] = -ai[i];
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    br[j] = Bs[buf][0][kq][wn + 8 * j + r];
                    bi[j] = Bs[buf][1][kq][wn + 8 * j + r];
                }
                // two passes of 32 independent DMMAs (dependent updates of one
                // accumulator 32 instructions apart)
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        dmma(acc[i][j][0][0], acc[i][j][0][1], ar[i], br[j]);
                        dmma(acc[i][j][1][0], acc[i][j][1][1], ar[i], bi[j]);
                    }
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        dmma(acc[i][j][0][0], acc[i][j][0][1], nai[i], bi[j]);
                        dmma(acc[i][j][1][0], acc[i][j][1][1], ai[i], br[j]);
                    }
            }
            if (c + 1 < nchunks) stash(buf ^ 1);
            __syncthreads();
        }
    }
    // epilogue
    const bool use_beta = (beta.re != 0.0 || beta.im != 0.0);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int row = m0 + wm + 8 * i + (lane >> 2);
                const int col = n0 + wn + 8 * j + 2 * (lane & 3) + e;
                if (row < M && col < N) {
                    const double vr = acc[i][j][0][e], vi = acc[i][j][1][e];
                    cplx out{alpha.re * vr - alpha.im * vi, alpha.re * vi + alpha.im * vr};
                    cplx* p = T.C + size_t(col) * T.ldc + row;
                    if (use_beta) {
                        const cplx o = *p;
                        out.re += beta.re * o.re - beta.im * o.im;
                        out.im += beta.re * o.im + beta.im * o.re;
                    }
                    *p = out;
                }
            }
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    const int n = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// TMA bulk copies (cp.async.bulk, SASS UBLKCP) completing on an mbarrier
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
    asm volatile(
        "{\n .reg .pred P1;\n LAB_WAIT:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        " @P1 bra DONE;\n bra LAB_WAIT;\n DONE:\n}\n" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* b) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(b))
        : "memory");
}


// ---------------------------------------------------------------------------
// 3M: three real DMMAs per complex 8x8x4 step instead of four,
//   P = Ar Br,  Q = Ai Bi,  S = (Ar + Ai)(Br + Bi),  Cr = P - Q,  Ci = S - P - Q
// (the Gauss product; normwise backward stable, error of the imaginary part
// ~ eps (|Ar| + |Ai|)(|Br| + |Bi|)), so the tensor pipe issues 6 M N K instead
// of 8 M N K real flops.  cp.async pipeline with a configurable warp tile (WMT x WNT m8n8
// tiles per warp, WARPS_M x WARPS_N warps).  Tiles are staged as interleaved
// complex: A as [k][m] (ld BM + 2 complex), B as [n][k] (ld BK + 4 complex), so
// the 16-byte fragment loads (lanes: k = lane & 3, m/n = lane >> 2) and the
// cp.async stores hit 8 distinct 16-byte bank groups per quarter warp.  The
// Gauss sums Ar + Ai, Br + Bi are formed in registers (FP64 pipe, not the
// tensor pipe).
// ---------------------------------------------------------------------------
template <int WMT, int WNT, int WARPS_M, int WARPS_N, int STAGES>
struct Z3Cfg {
    static constexpr int BM = WARPS_M * 8 * WMT, BN = WARPS_N * 8 * WNT, BK = 16;
    static constexpr int NT = 32 * WARPS_M * WARPS_N;
    static constexpr int LDA = BM + 2, LDK = BK + 4;
    static constexpr int STAGE = BK * LDA + BN * LDK;  // complex elements
    static constexpr size_t SMEM = size_t(STAGES) * STAGE * sizeof(double2);
};

// kNorm: the epilogue stores nothing; it sums |alpha A B + beta C|^2 over the
// tile and writes the CTA's partial to norm_part[(task0 + blockIdx.y) *
// gridDim.x + blockIdx.x] (C is only read) -- a residual norm without the
// residual's HBM round trip.
//
// kBulk: the stages are filled by TMA bulk copies (cp.async.bulk, one per tile
// column: A's BK columns of BM rows, B's BN columns of BK entries, each a
// contiguous run in HBM) issued by warp 0 and completing on one mbarrier per
// stage, instead of 16-byte cp.async per thread.  Rows past M and columns past
// N are not copied (their stale entries reach only accumulators that are never
// stored); the K tail of the last chunk is zero-filled in both operands.  Same
// products in the same order: results are bitwise those of the cp.async path.
template <int WMT, int WNT, int WARPS_M, int WARPS_N, int STAGES, int MINB, bool kNorm = false, bool kBulk = false>
__global__ void __launch_bounds__(32 * WARPS_M * WARPS_N, MINB)
    zgemm3m_t_kernel(int M, int N, cplx alpha, cplx beta, const GemmTask* __restrict__ tasks, int tiles_m,
                     double* __restrict__ norm_part = nullptr, size_t task0 = 0) {
    using Cfg = Z3Cfg<WMT, WNT, WARPS_M, WARPS_N, STAGES>;
    constexpr int BM = Cfg::BM, BN = Cfg::BN, BK = Cfg::BK, NT = Cfg::NT, LDA = Cfg::LDA, LDK = Cfg::LDK;
    extern __shared__ double2 z3_smem[];
    const GemmTask& T = tasks[blockIdx.y];
    const int tm = blockIdx.x % tiles_m, tn = blockIdx.x / tiles_m;
    const int m0 = tm * BM, n0 = tn * BN;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = (warp % WARPS_M) * 8 * WMT, wn = (warp / WARPS_M) * 8 * WNT;
    const int nseg = T.nseg;
    const int K0 = T.K[0], K1 = nseg > 1 ? T.K[1] : 0;
    const int c0n = (K0 + BK - 1) / BK, c1n = (K1 + BK - 1) / BK;
    const int nchunks = c0n + c1n;

    auto issue = [&](int c, int stage) {
        const int sgi = c < c0n ? 0 : 1;
        const int k0 = (c < c0n ? c : c - c0n) * BK;
        const cplx* __restrict__ A = T.A[sgi];
        const cplx* __restrict__ B = T.B[sgi];
        const int lda = T.lda[sgi], ldb = T.ldb[sgi], K = T.K[sgi];
        double2* As = z3_smem + stage * Cfg::STAGE;
        double2* Bs = As + BK * LDA;
#pragma unroll
        for (int i = 0; i < (BM * BK + NT - 1) / NT; ++i) {
            const int idx = tid + NT * i;
            if ((BM * BK) % NT == 0 || idx < BM * BK) {
                const int row = idx % BM, kk = idx / BM;
                const int gm = m0 + row, gk = k0 + kk;
                const bool ok = gm < M && gk < K;
                cp_async16(As + kk * LDA + row, ok ? (const void*)(A + size_t(gk) * lda + gm) : (const void*)A, ok);
            }
        }
#pragma unroll
        for (int i = 0; i < (BN * BK + NT - 1) / NT; ++i) {
            const int idx = tid + NT * i;
            if ((BN * BK) % NT == 0 || idx < BN * BK) {
                const int kk = idx % BK, col = idx / BK;
                const int gn = n0 + col, gk = k0 + kk;
                const bool ok = gn < N && gk < K;
                cp_async16(Bs + col * LDK + kk, ok ? (const void*)(B + size_t(gn) * ldb + gk) : (const void*)B, ok);
            }
        }
    };

    double acc[3][WMT][WNT][2];
#pragma unroll
    for (int q = 0; q < 3; ++q)
#pragma unroll
        for (int i = 0; i < WMT; ++i)
#pragma unroll
            for (int j = 0; j < WNT; ++j) acc[q][i][j][0] = acc[q][i][j][1] = 0.0;

    uint64_t* bars = reinterpret_cast<uint64_t*>(z3_smem + STAGES * Cfg::STAGE);
    // warp 0: chunk c into stage `stage` by bulk copies (kBulk)
    auto issue_bulk = [&](int c, int stage) {
        const int sgi = c < c0n ? 0 : 1;
        const int k0 = (c < c0n ? c : c - c0n) * BK;
        const cplx* __restrict__ A = T.A[sgi];
        const cplx* __restrict__ B = T.B[sgi];
        const int lda = T.lda[sgi], ldb = T.ldb[sgi];
        const int kv = min(BK, T.K[sgi] - k0), rows = min(BM, M - m0), cols = min(BN, N - n0);
        double2* As = z3_smem + stage * Cfg::STAGE;
        double2* Bs = As + BK * LDA;
        uint64_t* bar = bars + stage;
        if (lane == 0) mbar_expect_tx(bar, unsigned(kv * rows + cols * kv) * 16u);
        __syncwarp();
        for (int kk = lane; kk < BK; kk += 32) {
            if (kk < kv)
                bulk_g2s(As + kk * LDA, A + size_t(k0 + kk) * lda + m0, unsigned(rows) * 16u, bar);
            else
                for (int i = 0; i < BM; ++i) As[kk * LDA + i] = make_double2(0.0, 0.0);
        }
        for (int col = lane; col < cols; col += 32) {
            bulk_g2s(Bs + col * LDK, B + size_t(n0 + col) * ldb + k0, unsigned(kv) * 16u, bar);
            for (int kk = kv; kk < BK; ++kk) Bs[col * LDK + kk] = make_double2(0.0, 0.0);
        }
        // the zero fill (generic proxy) before any later bulk write of this stage
        if (kv < BK) asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    };
    if (kBulk) {
        if (tid == 0) {
            for (int st = 0; st < STAGES; ++st) mbar_init(bars + st, 1);
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        }
        __syncthreads();
        if (warp == 0)
            for (int st = 0; st < STAGES - 1; ++st)
                if (st < nchunks) issue_bulk(st, st);
    } else {
#pragma unroll
        for (int st = 0; st < STAGES - 1; ++st) {
            if (st < nchunks) issue(st, st);
            cp_async_commit();
        }
    }
    if (beta.re != 0.0 || beta.im != 0.0) {
        // the epilogue reads C: pull this CTA's tile into L2 now, so the
        // read-modify-write at the end does not wait on HBM (short-K products
        // spend a large share of their time in that dependent load)
        for (int e = tid; e < BN * (BM / 4); e += NT) {
            const int col = n0 + e / (BM / 4), row = m0 + (e % (BM / 4)) * 4;  // 4 complex = 64 B per prefetch
            if (col < N && row < M) {
                const cplx* p = T.C + size_t(col) * T.ldc + row;
                asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
            }
        }
    }
    for (int c = 0; c < nchunks; ++c) {
        if (kBulk) {
            mbar_wait(bars + c % STAGES, unsigned(c / STAGES) & 1u);
            __syncthreads();  // every warp is done with the stage refilled next
            if (warp == 0 && c + STAGES - 1 < nchunks) issue_bulk(c + STAGES - 1, (c + STAGES - 1) % STAGES);
        } else {
            cp_async_wait<STAGES - 2>();
            __syncthreads();
            if (c + STAGES - 1 < nchunks) issue(c + STAGES - 1, (c + STAGES - 1) % STAGES);
            cp_async_commit();
        }
        const double2* As = z3_smem + (c % STAGES) * Cfg::STAGE;
        const double2* Bs = As + BK * LDA;
#pragma unroll
        for (int ks = 0; ks < BK; ks += 4) {
            const int kq = ks + (lane & 3), r = lane >> 2;
            double br[WNT], bi[WNT], bs[WNT];
#pragma unroll
            for (int j = 0; j < WNT; ++j) {
                const double2 v = Bs[(wn + 8 * j + r) * LDK + kq];
                br[j] = v.x;
                bi[j] = v.y;
                bs[j] = v.x + v.y;
            }
#pragma unroll
            for (int i = 0; i < WMT; ++i) {
                const double2 v = As[kq * LDA + wm + 8 * i + r];
                const double as = v.x + v.y;
                // consecutive DMMAs share the A operand (operand reuse)
#pragma unroll
                for (int j = 0; j < WNT; ++j) dmma(acc[0][i][j][0], acc[0][i][j][1], v.x, br[j]);
#pragma unroll
                for (int j = 0; j < WNT; ++j) dmma(acc[1][i][j][0], acc[1][i][j][1], v.y, bi[j]);
#pragma unroll
                for (int j = 0; j < WNT; ++j) dmma(acc[2][i][j][0], acc[2][i][j][1], as, bs[j]);
            }
        }
    }
    if (!kBulk) cp_async_wait<0>();
    const bool use_beta = (beta.re != 0.0 || beta.im != 0.0);
    const int Mt = T.mlim == 0 ? M : (T.mlim > 0 ? min(M, T.mlim) : 0);
    double ss = 0.0;
#pragma unroll
    for (int i = 0; i < WMT; ++i)
#pragma unroll
        for (int j = 0; j < WNT; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int row = m0 + wm + 8 * i + (lane >> 2);
                const int col = n0 + wn + 8 * j + 2 * (lane & 3) + e;
                if (row < Mt && col < N) {
                    const double P = acc[0][i][j][e], Q = acc[1][i][j][e], S = acc[2][i][j][e];
                    const double vr = P - Q, vi = S - P - Q;
                    cplx out{alpha.re * vr - alpha.im * vi, alpha.re * vi + alpha.im * vr};
                    cplx* p = T.C + size_t(col) * T.ldc + row;
                    if (use_beta) {
                        const cplx o = *p;
                        out.re += beta.re * o.re - beta.im * o.im;
                        out.im += beta.re * o.im + beta.im * o.re;
                    }
                    if (kNorm) ss += out.re * out.re + out.im * out.im;
                    else *p = out;
                }
            }
    if (kNorm) {
        __syncthreads();  // the staging buffers are free: reuse for the partials
        double* red = reinterpret_cast<double*>(z3_smem);
        for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
        if (lane == 0) red[warp] = ss;
        __syncthreads();
        if (tid == 0) {
            double t = 0.0;
            for (int w = 0; w < NT / 32; ++w) t += red[w];
            norm_part[(task0 + blockIdx.y) * gridDim.x + blockIdx.x] = t;
        }
    }
}

__global__ void norm_parts_kernel(const double* __restrict__ part, int nparts, int ntasks, double* __restrict__ out) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ntasks) return;
    double s = 0.0;
    for (int q = 0; q < nparts; ++q) s += part[size_t(t) * nparts + q];
    out[t] = sqrt(s);
}

// QPS_ZGEMM_BULK=1: TMA bulk-copy staging instead of cp.async (A/B)
bool zgemm_bulk() {
    static const bool on = [] {
        const char* e = getenv("QPS_ZGEMM_BULK");
        return e && !strcmp(e, "1");
    }();
    return on;
}

template <int WMT, int WNT, int WARPS_M, int WARPS_N, int STAGES, int MINB = (WARPS_M * WARPS_N <= 4) ? 2 : 1,
          bool kNorm = false, bool kBulk = false>
void launch_z3_impl(int M, int N, cplx alpha, cplx beta, const GemmTask* tasks, size_t ntasks, cudaStream_t s,
                    DBuf<double>* parts, double* norms) {
    using Cfg = Z3Cfg<WMT, WNT, WARPS_M, WARPS_N, STAGES>;
    auto kern = zgemm3m_t_kernel<WMT, WNT, WARPS_M, WARPS_N, STAGES, MINB, kNorm, kBulk>;
    const size_t smem = Cfg::SMEM + (kBulk ? 8 * STAGES : 0);
    static bool attr = false;
    if (!attr) {
        QPS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        attr = true;
    }
    const int tiles_m = (M + Cfg::BM - 1) / Cfg::BM, tiles_n = (N + Cfg::BN - 1) / Cfg::BN;
    const int tiles = tiles_m * tiles_n;
    if (kNorm) parts->ensure(ntasks * tiles);
    for (size_t off = 0; off < ntasks; off += 65535) {
        const unsigned cnt = unsigned(std::min<size_t>(65535, ntasks - off));
        { QPS_NOTE_LAUNCH(); kern<<<dim3(tiles, cnt), Cfg::NT, smem, s>>>(M, N, alpha, beta, tasks + off, tiles_m,
                                                         kNorm ? parts->p : nullptr, off); }
        ++g_zgemm_launches;
    }
    if (kNorm) {
        { QPS_NOTE_LAUNCH(); norm_parts_kernel<<<unsigned((ntasks + 127) / 128), 128, 0, s>>>(parts->p, tiles, int(ntasks), norms); }
        QPS_CUDA(cudaGetLastError());
    }
}

template <int WMT, int WNT, int WARPS_M, int WARPS_N, int STAGES, int MINB = (WARPS_M * WARPS_N <= 4) ? 2 : 1,
          bool kNorm = false>
void launch_z3(int M, int N, cplx alpha, cplx beta, const GemmTask* tasks, size_t ntasks, cudaStream_t s,
               DBuf<double>* parts = nullptr, double* norms = nullptr) {
    if (zgemm_bulk())
        launch_z3_impl<WMT, WNT, WARPS_M, WARPS_N, STAGES, MINB, kNorm, true>(M, N, alpha, beta, tasks, ntasks, s,
                                                                              parts, norms);
    else
        launch_z3_impl<WMT, WNT, WARPS_M, WARPS_N, STAGES, MINB, kNorm, false>(M, N, alpha, beta, tasks, ntasks, s,
                                                                               parts, norms);
}

// ---------------------------------------------------------------------------
// block reductions
// ---------------------------------------------------------------------------
__device__ double block_sum(double v, double* sh) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    __syncthreads();
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    double t = 0.0;
    for (int w = 0; w < nw; ++w) t += sh[w];
    __syncthreads();
    return t;
}

// first index of the maximum value (Eigen maxCoeff semantics)
__device__ void block_argmax(double v, int idx, double* shv, int* shi, double& best, int& bidx) {
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
        if (ov > v || (ov == v && oi < idx)) {
            v = ov;
            idx = oi;
        }
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    __syncthreads();
    if (lane == 0) {
        shv[warp] = v;
        shi[warp] = idx;
    }
    __syncthreads();
    best = shv[0];
    bidx = shi[0];
    for (int w = 1; w < nw; ++w)
        if (shv[w] > best || (shv[w] == best && shi[w] < bidx)) {
            best = shv[w];
            bidx = shi[w];
        }
    __syncthreads();
}

constexpr int kMaxP = 256;

// ColPivHouseholderQR::computeInPlace semantics (see oracle shim for the
// restatement of Eigen's algorithm): largest updated column norm, LAPACK
// xGEQPF norm downdating with recomputation below sqrt(eps).
// kFast (low-rank compression only): reciprocal-multiplies instead of the
// FP64 divisions on each column's critical path (~600 cycles each on B200);
// the Schur least squares keep Eigen's divisions.
// kSmem: the whole m x p problem lives in shared memory (m p <= 13.7k entries,
// e.g. the 160 x 80 interior least squares), copied out once at the end.
extern __shared__ cplx cod_fac_sm[];
template <bool kFast, bool kSmem>
__global__ void __launch_bounds__(512) cod_factor_kernel(CodBatch b) {
    const int pb = blockIdx.x;
    const int m = b.m, p = b.p, size = min(m, p);
    const cplx* Q = b.Q + size_t(pb) * m * p;
    cplx* Wg = b.W + size_t(pb) * m * p;
    cplx* W = kSmem ? cod_fac_sm : Wg;
    cplx* tau = b.tau + size_t(pb) * p;
    int* perm = b.perm + size_t(pb) * p;
    __shared__ double upd[kMaxP], dir[kMaxP];
    __shared__ int flag[kMaxP];
    __shared__ double shv[32];
    __shared__ int shi[32];
    __shared__ cplx s_tau, s_den, s_inv;
    __shared__ int s_nzp;
    __shared__ double s_maxpiv;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    for (size_t i = tid; i < size_t(m) * p; i += blockDim.x) W[i] = Q[i];
    for (int j = tid; j < p; j += blockDim.x) perm[j] = j;
    __syncthreads();
    for (int j = warp; j < p; j += nw) {
        double s = 0.0;
        for (int i = lane; i < m; i += 32) s += cabs2(W[size_t(j) * m + i]);
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) upd[j] = dir[j] = sqrt(s);
    }
    __syncthreads();
    double maxnorm = 0.0;
    for (int j = 0; j < p; ++j) maxnorm = fmax(maxnorm, upd[j]);
    const double eps = DBL_EPSILON;
    const double threshold_helper = (maxnorm * eps) * (maxnorm * eps) / double(m);
    const double downdate_thr = sqrt(eps);
    if (tid == 0) {
        s_nzp = size;
        s_maxpiv = 0.0;
    }
    __syncthreads();
    for (int k = 0; k < size; ++k) {
        double best;
        int big;
        {
            double v = -1.0;
            int idx = p;
            for (int j = k + tid; j < p; j += blockDim.x)
                if (upd[j] > v) { v = upd[j]; idx = j; }
            block_argmax(v, idx, shv, shi, best, big);
        }
        if (tid == 0 && s_nzp == size && best * best < threshold_helper * double(m - k)) s_nzp = k;
        if (big != k) {
            for (int i = tid; i < m; i += blockDim.x) {
                const cplx t = W[size_t(k) * m + i];
                W[size_t(k) * m + i] = W[size_t(big) * m + i];
                W[size_t(big) * m + i] = t;
            }
            if (tid == 0) {
                double t = upd[k]; upd[k] = upd[big]; upd[big] = t;
                t = dir[k]; dir[k] = dir[big]; dir[big] = t;
                const int ti = perm[k]; perm[k] = perm[big]; perm[big] = ti;
            }
        }
        __syncthreads();
        // Householder of column k rows k..m-1 (makeHouseholderInPlace)
        double ts = 0.0;
        for (int i = k + 1 + tid; i < m; i += blockDim.x) ts += cabs2(W[size_t(k) * m + i]);
        const double tail_sq = block_sum(ts, shv);
        if (tid == 0) {
            const cplx c0 = W[size_t(k) * m + k];
            double beta;
            cplx tk;
            if (tail_sq <= DBL_MIN && c0.im * c0.im <= DBL_MIN) {
                tk = cplx{0, 0};
                beta = c0.re;
                s_den = cplx{0, 0};
            } else {
                beta = sqrt(cabs2(c0) + tail_sq);
                if (c0.re >= 0.0) beta = -beta;
                s_den = cplx{c0.re - beta, c0.im};
                tk = cconj(cdiv(cplx{beta - c0.re, -c0.im}, cplx{beta, 0.0}));
            }
            if (kFast) s_inv = (s_den.re == 0.0 && s_den.im == 0.0) ? cplx{0, 0} : fast_cinv(s_den);
            s_tau = tk;
            tau[k] = tk;
            W[size_t(k) * m + k] = cplx{beta, 0.0};
            s_maxpiv = fmax(s_maxpiv, fabs(beta));
        }
        __syncthreads();
        const cplx den = s_den, tk = s_tau;
        const bool zero_tau = (tk.re == 0.0 && tk.im == 0.0);
        for (int i = k + 1 + tid; i < m; i += blockDim.x) {
            cplx* w = &W[size_t(k) * m + i];
            if (kFast) *w = cmul(*w, s_inv);
            else *w = (den.re == 0.0 && den.im == 0.0) ? cplx{0, 0} : cdiv(*w, den);
        }
        __syncthreads();
        // apply H = I - tau v v^* to columns k+1..p-1
        if (!zero_tau || m - k == 1) {
            for (int j = k + 1 + warp; j < p; j += nw) {
                cplx* col = W + size_t(j) * m;
                if (m - k == 1) {
                    if (lane == 0) col[k] = cmul(col[k], cplx{1.0 - tk.re, -tk.im});
                    continue;
                }
                cplx t{0, 0};
                for (int i = k + 1 + lane; i < m; i += 32) {
                    const cplx e = W[size_t(k) * m + i];
                    const cplx a = col[i];
                    t.re += e.re * a.re + e.im * a.im;
                    t.im += e.re * a.im - e.im * a.re;
                }
                for (int o = 16; o > 0; o >>= 1) {
                    t.re += __shfl_xor_sync(0xffffffffu, t.re, o);
                    t.im += __shfl_xor_sync(0xffffffffu, t.im, o);
                }
                const cplx ck = col[k];
                t.re += ck.re;
                t.im += ck.im;
                t = cmul(tk, t);
                for (int i = k + 1 + lane; i < m; i += 32) {
                    const cplx e = W[size_t(k) * m + i];
                    const cplx et = cmul(e, t);
                    col[i].re -= et.re;
                    col[i].im -= et.im;
                }
                if (lane == 0) {
                    col[k].re -= t.re;
                    col[k].im -= t.im;
                }
            }
        }
        __syncthreads();
        // norm downdate (LAWN 176)
        for (int j = k + 1 + tid; j < p; j += blockDim.x) {
            flag[j] = 0;
            if (upd[j] != 0.0) {
                const cplx a = W[size_t(j) * m + k];
                const double iu = kFast ? fast_rcp(upd[j]) : 0.0;
                double t = kFast ? sqrt(cabs2(a)) * iu : sqrt(cabs2(a)) / upd[j];
                t = (1.0 + t) * (1.0 - t);
                t = t < 0.0 ? 0.0 : t;
                const double ud = kFast ? upd[j] * fast_rcp(dir[j]) : upd[j] / dir[j];
                const double t2 = t * ud * ud;
                if (t2 <= downdate_thr) flag[j] = 1;
                else upd[j] *= sqrt(t);
            }
        }
        __syncthreads();
        for (int j = k + 1 + warp; j < p; j += nw) {
            if (!flag[j]) continue;
            double s = 0.0;
            for (int i = k + 1 + lane; i < m; i += 32) s += cabs2(W[size_t(j) * m + i]);
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (lane == 0) upd[j] = dir[j] = sqrt(s);
        }
        __syncthreads();
    }
    if (tid == 0) {
        b.nzp[pb] = s_nzp;
        b.maxpiv[pb] = s_maxpiv;
    }
    if (kSmem)
        for (size_t i = tid; i < size_t(m) * p; i += blockDim.x) Wg[i] = W[i];
}

__global__ void cod_rank_kernel(CodBatch b, double th, const int* __restrict__ flags) {
    const int pb = blockIdx.x * blockDim.x + threadIdx.x;
    if (pb >= b.count) return;
    if (flags && !flags[pb]) return;
    const cplx* W = b.W + size_t(pb) * b.m * b.p;
    const double pre = b.maxpiv[pb] * th;
    int r = 0;
    for (int i = 0; i < b.nzp[pb]; ++i) r += sqrt(cabs2(W[size_t(i) * b.m + i])) > pre;
    b.rank[pb] = r;
}

// Complete orthogonal decomposition at the current rank
// (CompleteOrthogonalDecomposition::computeInPlace semantics): RZ reduction of
// [R11 R12] in V, then the two orthonormal factors of the min-norm solve
//   QH = Q_r^* restricted to its first r rows   (p x m, rows >= r zero)
//   Wz = P Z^* [I_r; 0]                          (p x p, cols >= r zero)
// so that X = Wz * T11^{-1} * (QH * RHS) (_solve_impl order: Q^*, T^{-1}, Z^*, P).
__global__ void __launch_bounds__(256) cod_operator_kernel(CodBatch b, const int* __restrict__ flags) {
    const int pb = blockIdx.x;
    if (flags && !flags[pb]) return;
    const int m = b.m, p = b.p;
    const cplx* W = b.W + size_t(pb) * m * p;
    cplx* V = b.V + size_t(pb) * m * p;
    const cplx* tau = b.tau + size_t(pb) * p;
    cplx* zc = b.zc + size_t(pb) * p;
    const int* perm = b.perm + size_t(pb) * p;
    cplx* M1 = b.M1 + size_t(pb) * m * p;
    cplx* Y = b.Y + size_t(pb) * p * m;
    cplx* QH = b.QH + size_t(pb) * p * m;
    cplx* Wz = b.Wz + size_t(pb) * p * p;
    const int r = b.rank[pb];
    const int tid = threadIdx.x;
    __shared__ double shv[32];
    __shared__ cplx s_den, s_zc;
    for (size_t i = tid; i < size_t(m) * p; i += blockDim.x) V[i] = W[i];
    if (r == 0) {
        for (size_t i = tid; i < size_t(p) * p; i += blockDim.x) Wz[i] = cplx{0, 0};
        return;
    }
    __syncthreads();
    auto vat = [&](int i, int j) -> cplx& { return V[size_t(j) * m + i]; };
    if (r < p) {
        for (int k = r - 1; k >= 0; --k) {
            if (k != r - 1)
                for (int i = tid; i <= k; i += blockDim.x) {
                    const cplx t = vat(i, k);
                    vat(i, k) = vat(i, r - 1);
                    vat(i, r - 1) = t;
                }
            __syncthreads();
            const int L = p - r + 1;
            double ts = 0.0;
            for (int j = 1 + tid; j < L; j += blockDim.x) ts += cabs2(vat(k, r - 1 + j));
            const double tail_sq = block_sum(ts, shv);
            if (tid == 0) {
                const cplx c0 = vat(k, r - 1);
                double beta;
                cplx tk;
                if (tail_sq <= DBL_MIN && c0.im * c0.im <= DBL_MIN) {
                    tk = cplx{0, 0};
                    beta = c0.re;
                    s_den = cplx{0, 0};
                } else {
                    beta = sqrt(cabs2(c0) + tail_sq);
                    if (c0.re >= 0.0) beta = -beta;
                    s_den = cplx{c0.re - beta, c0.im};
                    tk = cconj(cdiv(cplx{beta - c0.re, -c0.im}, cplx{beta, 0.0}));
                }
                s_zc = tk;
                zc[k] = tk;
                vat(k, r - 1) = cplx{beta, 0.0};
            }
            __syncthreads();
            const cplx den = s_den, tk = s_zc;
            for (int j = 1 + tid; j < L; j += blockDim.x) {
                cplx& e = vat(k, r - 1 + j);
                e = (den.re == 0.0 && den.im == 0.0) ? cplx{0, 0} : cdiv(e, den);
            }
            __syncthreads();
            if (k > 0 && !(tk.re == 0.0 && tk.im == 0.0)) {
                for (int i = tid; i < k; i += blockDim.x) {
                    cplx t = vat(i, r - 1);
                    for (int j = 1; j < L; ++j) {
                        const cplx e = vat(k, r - 1 + j);
                        const cplx a = vat(i, r - 1 + j);
                        t.re += a.re * e.re + a.im * e.im;
                        t.im += a.im * e.re - a.re * e.im;
                    }
                    t = cmul(t, tk);
                    vat(i, r - 1).re -= t.re;
                    vat(i, r - 1).im -= t.im;
                    for (int j = 1; j < L; ++j) {
                        const cplx te = cmul(t, vat(k, r - 1 + j));
                        vat(i, r - 1 + j).re -= te.re;
                        vat(i, r - 1 + j).im -= te.im;
                    }
                }
            }
            __syncthreads();
            if (k != r - 1)
                for (int i = tid; i <= k; i += blockDim.x) {
                    const cplx t = vat(i, k);
                    vat(i, k) = vat(i, r - 1);
                    vat(i, r - 1) = t;
                }
            __syncthreads();
        }
    }
    // QH: cod_qh_kernel (many CTAs per problem)
    // Wz columns: P Z^* e_c for c < r
    for (int c = tid; c < p; c += blockDim.x) {
        cplx* y = Y + size_t(c) * p;
        cplx* w = Wz + size_t(c) * p;
        if (c >= r) {
            for (int i = 0; i < p; ++i) w[i] = cplx{0, 0};
            continue;
        }
        for (int i = 0; i < p; ++i) y[i] = cplx{i == c ? 1.0 : 0.0, 0.0};
        if (r < p) {
            for (int k = c; k < r; ++k) {  // reflectors k < c leave e_c unchanged
                const cplx tk = zc[k];
                if (k != r - 1) {
                    const cplx t = y[k];
                    y[k] = y[r - 1];
                    y[r - 1] = t;
                }
                if (!(tk.re == 0.0 && tk.im == 0.0)) {
                    cplx t = y[r - 1];
                    for (int j = 0; j < p - r; ++j) {
                        const cplx e = cmul(vat(k, r + j), y[r + j]);
                        t.re += e.re;
                        t.im += e.im;
                    }
                    t = cmul(t, tk);
                    y[r - 1].re -= t.re;
                    y[r - 1].im -= t.im;
                    for (int j = 0; j < p - r; ++j) {
                        const cplx e = cmul(cconj(vat(k, r + j)), t);
                        y[r + j].re -= e.re;
                        y[r + j].im -= e.im;
                    }
                }
                if (k != r - 1) {
                    const cplx t = y[k];
                    y[k] = y[r - 1];
                    y[r - 1] = t;
                }
            }
        }
        for (int i = 0; i < p; ++i) w[perm[i]] = y[i];
    }
}

// QH = first r rows of Q_r^* = H_{r-1} ... H_0 (reflectors exactly as applied)
// for problems too large for the shared-memory operator: column c of QH is
// H_{r-1} ... H_0 e_c, independent per column, so every CTA takes 8 columns
// (one warp each, the column in shared memory, lanes over rows) and the
// problem's m columns spread over m/8 CTAs instead of one.
__global__ void __launch_bounds__(256) cod_qh_kernel(CodBatch b, const int* __restrict__ flags) {
    const int pb = blockIdx.y;
    if (flags && !flags[pb]) return;
    const int m = b.m, p = b.p, r = b.rank[pb];
    const cplx* W = b.W + size_t(pb) * m * p;
    const cplx* tau = b.tau + size_t(pb) * p;
    cplx* QH = b.QH + size_t(pb) * p * m;
    extern __shared__ cplx qh_col[];  // [8][m]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int c = blockIdx.x * 8 + warp;
    if (c >= m) return;
    cplx* col = qh_col + size_t(warp) * m;
    for (int i = lane; i < m; i += 32) col[i] = cplx{i == c ? 1.0 : 0.0, 0.0};
    __syncwarp();
    for (int kk = 0; kk < r; ++kk) {
        const cplx tk = tau[kk];
        if (tk.re == 0.0 && tk.im == 0.0) continue;
        const cplx* e = W + size_t(kk) * m;
        cplx t{0, 0};
        for (int i = kk + 1 + lane; i < m; i += 32) {
            const cplx ei = e[i];
            const cplx a = col[i];
            t.re += ei.re * a.re + ei.im * a.im;
            t.im += ei.re * a.im - ei.im * a.re;
        }
        for (int o = 16; o > 0; o >>= 1) {
            t.re += __shfl_xor_sync(0xffffffffu, t.re, o);
            t.im += __shfl_xor_sync(0xffffffffu, t.im, o);
        }
        const cplx ck = col[kk];
        t.re += ck.re;
        t.im += ck.im;
        t = cmul(tk, t);
        __syncwarp();
        if (lane == 0) {
            col[kk].re -= t.re;
            col[kk].im -= t.im;
        }
        for (int i = kk + 1 + lane; i < m; i += 32) {
            const cplx et = cmul(e[i], t);
            col[i].re -= et.re;
            col[i].im -= et.im;
        }
        __syncwarp();
    }
    for (int i = lane; i < p; i += 32) QH[size_t(c) * p + i] = i < r ? col[i] : cplx{0, 0};
}

// Same operator with the working set in shared memory (problems with
// (m p + max(p^2, 32 m)) complex entries <= kCodSmemMax): region 1 holds the RZ
// reflectors V, then the QR reflectors W; region 2 the Wz work columns
// (row-major, conflict-free per thread column), then the per-warp QH columns
// (four per warp).
constexpr size_t kCodSmemMax = 220 * 1024;
__global__ void __launch_bounds__(256) cod_operator_smem_kernel(CodBatch b, const int* __restrict__ flags) {
    extern __shared__ cplx cod_sm[];
    const int pb = blockIdx.x;
    if (flags && !flags[pb]) return;
    const int m = b.m, p = b.p;
    const cplx* W = b.W + size_t(pb) * m * p;
    const cplx* tau = b.tau + size_t(pb) * p;
    cplx* zc = b.zc + size_t(pb) * p;
    const int* perm = b.perm + size_t(pb) * p;
    cplx* QH = b.QH + size_t(pb) * p * m;
    cplx* Wz = b.Wz + size_t(pb) * p * p;
    const int r = b.rank[pb];
    const int tid = threadIdx.x;
    __shared__ double shv[32];
    __shared__ cplx s_den, s_zc;
    cplx* V = cod_sm;                      // region 1
    cplx* R2 = cod_sm + size_t(m) * p;     // region 2
    if (r == 0) {
        for (size_t i = tid; i < size_t(p) * m; i += blockDim.x) QH[i] = cplx{0, 0};
        for (size_t i = tid; i < size_t(p) * p; i += blockDim.x) Wz[i] = cplx{0, 0};
        return;
    }
    for (size_t i = tid; i < size_t(m) * p; i += blockDim.x) V[i] = W[i];
    __syncthreads();
    auto vat = [&](int i, int j) -> cplx& { return V[size_t(j) * m + i]; };
    if (r < p) {  // RZ reduction of [R11 R12] (Eigen COD), reflectors into zc and V
        for (int k = r - 1; k >= 0; --k) {
            if (k != r - 1)
                for (int i = tid; i <= k; i += blockDim.x) {
                    const cplx t = vat(i, k);
                    vat(i, k) = vat(i, r - 1);
                    vat(i, r - 1) = t;
                }
            __syncthreads();
            const int L = p - r + 1;
            double ts = 0.0;
            for (int j = 1 + tid; j < L; j += blockDim.x) ts += cabs2(vat(k, r - 1 + j));
            const double tail_sq = block_sum(ts, shv);
            if (tid == 0) {
                const cplx c0 = vat(k, r - 1);
                double beta;
                cplx tk;
                if (tail_sq <= DBL_MIN && c0.im * c0.im <= DBL_MIN) {
                    tk = cplx{0, 0};
                    beta = c0.re;
                    s_den = cplx{0, 0};
                } else {
                    beta = sqrt(cabs2(c0) + tail_sq);
                    if (c0.re >= 0.0) beta = -beta;
                    s_den = cplx{c0.re - beta, c0.im};
                    tk = cconj(cdiv(cplx{beta - c0.re, -c0.im}, cplx{beta, 0.0}));
                }
                s_zc = tk;
                zc[k] = tk;
                vat(k, r - 1) = cplx{beta, 0.0};
            }
            __syncthreads();
            const cplx den = s_den, tk = s_zc;
            for (int j = 1 + tid; j < L; j += blockDim.x) {
                cplx& e = vat(k, r - 1 + j);
                e = (den.re == 0.0 && den.im == 0.0) ? cplx{0, 0} : cdiv(e, den);
            }
            __syncthreads();
            if (k > 0 && !(tk.re == 0.0 && tk.im == 0.0)) {
                for (int i = tid; i < k; i += blockDim.x) {
                    cplx t = vat(i, r - 1);
                    for (int j = 1; j < L; ++j) {
                        const cplx e = vat(k, r - 1 + j);
                        const cplx a = vat(i, r - 1 + j);
                        t.re += a.re * e.re + a.im * e.im;
                        t.im += a.im * e.re - a.re * e.im;
                    }
                    t = cmul(t, tk);
                    vat(i, r - 1).re -= t.re;
                    vat(i, r - 1).im -= t.im;
                    for (int j = 1; j < L; ++j) {
                        const cplx te = cmul(t, vat(k, r - 1 + j));
                        vat(i, r - 1 + j).re -= te.re;
                        vat(i, r - 1 + j).im -= te.im;
                    }
                }
            }
            __syncthreads();
            if (k != r - 1)
                for (int i = tid; i <= k; i += blockDim.x) {
                    const cplx t = vat(i, k);
                    vat(i, k) = vat(i, r - 1);
                    vat(i, r - 1) = t;
                }
            __syncthreads();
        }
    }
    // Wz columns: P Z^* e_c for c < r (thread per column; work column in region 2, row-major)
    {
        const cplx* zs = zc;
        for (int c = tid; c < p; c += blockDim.x) {
            cplx* w = Wz + size_t(c) * p;
            if (c >= r) {
                for (int i = 0; i < p; ++i) w[i] = cplx{0, 0};
                continue;
            }
            auto y = [&](int i) -> cplx& { return R2[size_t(i) * p + c]; };
            for (int i = 0; i < p; ++i) y(i) = cplx{i == c ? 1.0 : 0.0, 0.0};
            if (r < p) {
                for (int k = c; k < r; ++k) {  // reflectors k < c leave e_c unchanged
                    const cplx tk = zs[k];
                    if (k != r - 1) {
                        const cplx t = y(k);
                        y(k) = y(r - 1);
                        y(r - 1) = t;
                    }
                    if (!(tk.re == 0.0 && tk.im == 0.0)) {
                        cplx t = y(r - 1);
                        for (int j = 0; j < p - r; ++j) {
                            const cplx e = cmul(vat(k, r + j), y(r + j));
                            t.re += e.re;
                            t.im += e.im;
                        }
                        t = cmul(t, tk);
                        y(r - 1).re -= t.re;
                        y(r - 1).im -= t.im;
                        for (int j = 0; j < p - r; ++j) {
                            const cplx e = cmul(cconj(vat(k, r + j)), t);
                            y(r + j).re -= e.re;
                            y(r + j).im -= e.im;
                        }
                    }
                    if (k != r - 1) {
                        const cplx t = y(k);
                        y(k) = y(r - 1);
                        y(r - 1) = t;
                    }
                }
            }
            for (int i = 0; i < p; ++i) w[perm[i]] = y(i);
        }
    }
    // T11 (upper triangle of V) for cod_trsm
    {
        cplx* Vg = b.V + size_t(pb) * m * p;
        for (size_t i = tid; i < size_t(m) * p; i += blockDim.x) Vg[i] = V[i];
    }
    __syncthreads();
    // QR reflectors into region 1 (V is no longer needed)
    for (size_t i = tid; i < size_t(m) * p; i += blockDim.x) V[i] = W[i];
    __syncthreads();
    const cplx* Ws = V;
    // QH = first r rows of H_{r-1} ... H_0: each warp carries four columns at
    // once (lanes over rows), so the four dot products' shuffle reductions of
    // each reflector overlap instead of running one column after another
    {
        constexpr int kC = 4;
        const int lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
        cplx* cols = R2 + size_t(warp) * kC * m;
        for (int cb = warp * kC; cb < m; cb += nw * kC) {
#pragma unroll
            for (int j = 0; j < kC; ++j)
                for (int i = lane; i < m; i += 32) cols[j * m + i] = cplx{i == cb + j ? 1.0 : 0.0, 0.0};
            __syncwarp();
            for (int kk = 0; kk < r; ++kk) {
                const cplx tk = tau[kk];
                if (tk.re == 0.0 && tk.im == 0.0) continue;
                cplx t[kC];
#pragma unroll
                for (int j = 0; j < kC; ++j) t[j] = cplx{0, 0};
                for (int i = kk + 1 + lane; i < m; i += 32) {
                    const cplx e = Ws[size_t(kk) * m + i];
#pragma unroll
                    for (int j = 0; j < kC; ++j) {
                        const cplx a = cols[j * m + i];
                        t[j].re += e.re * a.re + e.im * a.im;
                        t[j].im += e.re * a.im - e.im * a.re;
                    }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                    for (int j = 0; j < kC; ++j) {
                        t[j].re += __shfl_xor_sync(0xffffffffu, t[j].re, o);
                        t[j].im += __shfl_xor_sync(0xffffffffu, t[j].im, o);
                    }
#pragma unroll
                for (int j = 0; j < kC; ++j) {
                    const cplx ck = cols[j * m + kk];
                    t[j].re += ck.re;
                    t[j].im += ck.im;
                    t[j] = cmul(tk, t[j]);
                }
                __syncwarp();
                if (lane == 0) {
#pragma unroll
                    for (int j = 0; j < kC; ++j) {
                        cols[j * m + kk].re -= t[j].re;
                        cols[j * m + kk].im -= t[j].im;
                    }
                }
                for (int i = kk + 1 + lane; i < m; i += 32) {
                    const cplx e = Ws[size_t(kk) * m + i];
#pragma unroll
                    for (int j = 0; j < kC; ++j) {
                        const cplx et = cmul(e, t[j]);
                        cols[j * m + i].re -= et.re;
                        cols[j * m + i].im -= et.im;
                    }
                }
                __syncwarp();
            }
#pragma unroll
            for (int j = 0; j < kC; ++j)
                if (cb + j < m)
                    for (int i = lane; i < p; i += 32) QH[size_t(cb + j) * p + i] = i < r ? cols[j * m + i] : cplx{0, 0};
            __syncwarp();
        }
    }
}

// back substitution with T11 (upper, r x r inside V, ld m), one thread per
// column of the right-hand side; T11 is staged in shared memory (every thread
// reads the same entry at the same time: broadcast).
// Interior-layer variant: T11 (r x r) and a 64-column chunk of the RHS staged
// in shared memory; 4 lanes per column split each dot product (warp-level
// synchronisation only: a column's lanes share a warp).  Backward-stable
// substitution, no explicit inverse.
constexpr int kTrsmCols = 64;
__global__ void __launch_bounds__(256) cod_trsm_chunk_kernel(CodBatch b, cplx* B, int ldb, size_t stride, int ncols,
                                                             const int* __restrict__ flags) {
    extern __shared__ cplx tch[];
    const int pb = blockIdx.y;
    if (flags && !flags[pb]) return;
    const int m = b.m, r = b.rank[pb];
    const cplx* V = b.V + size_t(pb) * m * b.p;
    cplx* T = tch;           // r x r (ld r)
    cplx* X = tch + r * r;   // r x kTrsmCols (ld r)
    cplx* Tinv = X + r * kTrsmCols;  // r reciprocals of the diagonal
    const int c0 = blockIdx.x * kTrsmCols;
    const int nc = min(kTrsmCols, ncols - c0);
    cplx* Bp = B + stride * pb + size_t(c0) * ldb;
    for (int e = threadIdx.x; e < r * r; e += blockDim.x) {
        const int i = e % r, j = e / r;
        T[e] = (i <= j) ? V[size_t(j) * m + i] : cplx{0, 0};
    }
    for (int e = threadIdx.x; e < r * nc; e += blockDim.x) {
        const int i = e % r, j = e / r;
        X[j * r + i] = Bp[size_t(j) * ldb + i];
    }
    __syncthreads();
    // reciprocals up front: an FP64 division on the substitution chain costs ~600 cycles per row
    for (int i = threadIdx.x; i < r; i += blockDim.x) Tinv[i] = cdiv(cplx{1.0, 0.0}, T[i * r + i]);
    __syncthreads();
    const int col = threadIdx.x >> 2, part = threadIdx.x & 3;
    const bool active = col < nc;
    for (int i = r - 1; i >= 0; --i) {
        cplx sacc{0, 0};
        if (active)
            for (int l = i + 1 + part; l < r; l += 4) {
                const cplx t = cmul(T[l * r + i], X[col * r + l]);
                sacc.re += t.re;
                sacc.im += t.im;
            }
        sacc.re += __shfl_xor_sync(0xffffffffu, sacc.re, 1);
        sacc.im += __shfl_xor_sync(0xffffffffu, sacc.im, 1);
        sacc.re += __shfl_xor_sync(0xffffffffu, sacc.re, 2);
        sacc.im += __shfl_xor_sync(0xffffffffu, sacc.im, 2);
        if (active && part == 0) {
            const cplx bi = X[col * r + i];
            X[col * r + i] = cmul(cplx{bi.re - sacc.re, bi.im - sacc.im}, Tinv[i]);
        }
        __syncwarp();
    }
    __syncthreads();
    for (int e = threadIdx.x; e < r * nc; e += blockDim.x) {
        const int i = e % r, j = e / r;
        Bp[size_t(j) * ldb + i] = X[j * r + i];
    }
}

// Blocked back substitution (LAPACK trsm order, no explicit inverse): 16-row
// diagonal blocks solved by substitution with 8 lanes per column, the rows
// above updated by the solved block as small products.  T11 packed (upper,
// column-major) and 32 columns per CTA keep two CTAs per SM; the serial chain
// is r row steps of <= 16-term dot products instead of up-to-r-term ones.
#ifndef QPS_TRSM_BLK_COLS
#define QPS_TRSM_BLK_COLS 32
#endif
constexpr int kTrsmBlkCols = QPS_TRSM_BLK_COLS;
__global__ void __launch_bounds__(256) cod_trsm_blk_kernel(CodBatch b, cplx* B, int ldb, size_t stride, int ncols,
                                                           const int* __restrict__ flags) {
    extern __shared__ cplx tbk[];
    const int pb = blockIdx.y;
    if (flags && !flags[pb]) return;
    const int m = b.m, r = b.rank[pb];
    if (r == 0) return;
    const cplx* V = b.V + size_t(pb) * m * b.p;
    const int lx = r + 1;                          // X ld: the 4 columns of a warp in distinct banks
    cplx* T = tbk;                                 // packed upper: (i, j) at j (j + 1) / 2 + i
    cplx* X = T + size_t(r) * (r + 1) / 2;         // r x kTrsmBlkCols (ld lx)
    cplx* Tinv = X + size_t(lx) * kTrsmBlkCols;    // reciprocals of the diagonal
    const int c0 = blockIdx.x * kTrsmBlkCols;
    const int nc = min(kTrsmBlkCols, ncols - c0);
    cplx* Bp = B + stride * pb + size_t(c0) * ldb;
    const int tid = threadIdx.x;
    for (int e = tid; e < r * r; e += blockDim.x) {
        const int i = e % r, j = e / r;
        if (i <= j) T[j * (j + 1) / 2 + i] = V[size_t(j) * m + i];
    }
    for (int e = tid; e < r * nc; e += blockDim.x) {
        const int i = e % r, j = e / r;
        X[j * lx + i] = Bp[size_t(j) * ldb + i];
    }
    __syncthreads();
    for (int i = tid; i < r; i += blockDim.x) Tinv[i] = cdiv(cplx{1.0, 0.0}, T[i * (i + 1) / 2 + i]);
    __syncthreads();
    const int col = tid >> 3, part = tid & 7;
    const bool active = col < nc;
    for (int b1 = r; b1 > 0; b1 -= 16) {
        const int b0 = max(0, b1 - 16);
        // diagonal block: rows b1-1 .. b0 by substitution
        for (int i = b1 - 1; i >= b0; --i) {
            cplx sacc{0, 0};
            if (active)
                for (int l = i + 1 + part; l < b1; l += 8) {
                    const cplx t = cmul(T[l * (l + 1) / 2 + i], X[col * lx + l]);
                    sacc.re += t.re;
                    sacc.im += t.im;
                }
#pragma unroll
            for (int o = 1; o < 8; o <<= 1) {
                sacc.re += __shfl_xor_sync(0xffffffffu, sacc.re, o);
                sacc.im += __shfl_xor_sync(0xffffffffu, sacc.im, o);
            }
            if (active && part == 0) {
                const cplx bi = X[col * lx + i];
                X[col * lx + i] = cmul(cplx{bi.re - sacc.re, bi.im - sacc.im}, Tinv[i]);
            }
            __syncwarp();
        }
        __syncthreads();
        // rows above: X[i] -= T[i, b0:b1] X[b0:b1]
        for (int e = tid; e < b0 * nc; e += blockDim.x) {
            const int i = e % b0, c = e / b0;
            cplx acc{0, 0};
            for (int l = b0; l < b1; ++l) {
                const cplx t = cmul(T[l * (l + 1) / 2 + i], X[c * lx + l]);
                acc.re += t.re;
                acc.im += t.im;
            }
            X[c * lx + i].re -= acc.re;
            X[c * lx + i].im -= acc.im;
        }
        __syncthreads();
    }
    for (int e = tid; e < r * nc; e += blockDim.x) {
        const int i = e % r, j = e / r;
        Bp[size_t(j) * ldb + i] = X[j * lx + i];
    }
}

// Blocked back substitution (LAPACK xTRSM order, left-looking from the bottom
// in 16-row blocks aligned to each problem's rank r): block s covers rows
// [lo, hi), hi = r - 16 s, lo = max(0, hi - 16); its rows first take the
// product of the rows already solved below (a batched DMMA GEMM, tasks built
// on the device from the ranks), then the 16 x 16 diagonal block is solved by
// substitution, one thread per right-hand-side column.
__global__ void cod_trsm_tasks_kernel(CodBatch b, cplx* B, int ldb, size_t stride, const int* __restrict__ flags,
                                      int nsteps) {
    const int pb = blockIdx.x * blockDim.x + threadIdx.x;
    if (pb >= b.count) return;
    const int m = b.m, r = b.rank[pb];
    const bool on = !flags || flags[pb];
    const cplx* V = b.V + size_t(pb) * m * b.p;
    cplx* Bp = B + stride * pb;
    for (int st = 0; st < nsteps; ++st) {
        const int hi = r - 16 * st, lo = max(0, hi - 16);
        const bool act = on && hi > 0 && st > 0;
        GemmTask t{};
        t.nseg = 1;
        t.A[0] = V + size_t(act ? hi : 0) * m + (act ? lo : 0);
        t.lda[0] = m;
        t.B[0] = Bp + (act ? hi : 0);
        t.ldb[0] = ldb;
        t.K[0] = act ? r - hi : 0;
        t.C = Bp + (act ? lo : 0);
        t.ldc = ldb;
        t.mlim = act ? hi - lo : -1;
        b.trsm_tasks[size_t(st) * b.count + pb] = t;
    }
}
__global__ void __launch_bounds__(128) cod_trsm_diag_kernel(CodBatch b, cplx* B, int ldb, size_t stride, int ncols,
                                                            const int* __restrict__ flags, int st) {
    const int pb = blockIdx.y;
    if (flags && !flags[pb]) return;
    const int m = b.m, r = b.rank[pb];
    const int hi = r - 16 * st, lo = max(0, hi - 16), h = hi - lo;
    if (hi <= 0) return;
    __shared__ cplx Tb[16][17];
    __shared__ cplx Ti[16];
    const cplx* V = b.V + size_t(pb) * m * b.p;
    for (int e = threadIdx.x; e < 256; e += blockDim.x) {
        const int i = e & 15, j = e >> 4;
        Tb[i][j] = (i <= j && j < h) ? V[size_t(lo + j) * m + lo + i] : cplx{0, 0};
    }
    __syncthreads();
    if (threadIdx.x < h) Ti[threadIdx.x] = cdiv(cplx{1.0, 0.0}, Tb[threadIdx.x][threadIdx.x]);
    __syncthreads();
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= ncols) return;
    cplx* x = B + stride * pb + size_t(c) * ldb + lo;
    cplx v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = i < h ? x[i] : cplx{0, 0};
#pragma unroll
    for (int i = 15; i >= 0; --i) {
        if (i < h) {
            cplx a = v[i];
#pragma unroll
            for (int l = i + 1; l < 16; ++l) {  // T[i][l] = 0 beyond h
                const cplx t = Tb[i][l];
                a.re -= t.re * v[l].re - t.im * v[l].im;
                a.im -= t.re * v[l].im + t.im * v[l].re;
            }
            v[i] = cmul(a, Ti[i]);
        }
    }
#pragma unroll
    for (int i = 0; i < 16; ++i)
        if (i < h) x[i] = v[i];
}

template <bool kSmem>
__global__ void __launch_bounds__(128) cod_trsm_kernel(CodBatch b, cplx* B, int ldb, size_t stride, int ncols,
                                                       const int* __restrict__ flags) {
    extern __shared__ cplx tsm_dyn[];
    const int pb = blockIdx.y;
    if (flags && !flags[pb]) return;
    const int m = b.m, r = b.rank[pb];
    const cplx* V = b.V + size_t(pb) * m * b.p;
    const cplx* tsm;
    int ldt;
    if (kSmem) {  // T11 staged in shared memory (interior layers: r <= P = 60..80)
        for (int e = threadIdx.x; e < r * r; e += blockDim.x) {
            const int i = e % r, j = e / r;
            tsm_dyn[e] = (i <= j) ? V[size_t(j) * m + i] : cplx{0, 0};
        }
        __syncthreads();
        tsm = tsm_dyn;
        ldt = r;
    } else {  // large corner systems read T11 through L1
        tsm = V;
        ldt = m;
    }
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= ncols) return;
    cplx* x = B + stride * pb + size_t(c) * ldb;
    for (int i = r - 1; i >= 0; --i) {
        cplx s = x[i];
        for (int l = i + 1; l < r; ++l) {
            const cplx t = cmul(tsm[size_t(l) * ldt + i], x[l]);
            s.re -= t.re;
            s.im -= t.im;
        }
        x[i] = cdiv(s, tsm[size_t(i) * ldt + i]);
    }
}

// ---------------------------------------------------------------------------
// LU (partial pivoting on the modulus, like Eigen's PartialPivLU)
// ---------------------------------------------------------------------------
constexpr int kNB = 32;  // LU panel width
constexpr int kTB = 64;  // triangular-solve block (inverse diagonal tiles)

__global__ void __launch_bounds__(256) lu_panel_kernel(int n, int ld, cplx* const* __restrict__ Ap,
                                                       int* const* __restrict__ Pp, int k0, int* singular) {
    cplx* A = Ap[blockIdx.x];
    int* ipiv = Pp[blockIdx.x];
    const int kend = min(k0 + kNB, n);
    __shared__ double shv[32];
    __shared__ int shi[32];
    const int tid = threadIdx.x;
    for (int k = k0; k < kend; ++k) {
        double v = -1.0;
        int idx = n;
        for (int i = k + tid; i < n; i += blockDim.x) {
            const double a = sqrt(cabs2(A[size_t(k) * ld + i]));
            if (a > v) { v = a; idx = i; }
        }
        double best;
        int piv;
        block_argmax(v, idx, shv, shi, best, piv);
        if (tid == 0) ipiv[k] = piv;
        if (piv != k)
            for (int j = k0 + tid; j < kend; j += blockDim.x) {
                const cplx t = A[size_t(j) * ld + k];
                A[size_t(j) * ld + k] = A[size_t(j) * ld + piv];
                A[size_t(j) * ld + piv] = t;
            }
        __syncthreads();
        const cplx d = A[size_t(k) * ld + k];
        if (d.re == 0.0 && d.im == 0.0) {
            if (tid == 0) singular[blockIdx.x] = 1;
        } else {
            const cplx inv = cdiv(cplx{1.0, 0.0}, d);
            for (int i = k + 1 + tid; i < n; i += blockDim.x) A[size_t(k) * ld + i] = cmul(A[size_t(k) * ld + i], inv);
        }
        __syncthreads();
        for (int i = k + 1 + tid; i < n; i += blockDim.x) {
            const cplx l = A[size_t(k) * ld + i];
            for (int j = k + 1; j < kend; ++j) {
                const cplx u = A[size_t(j) * ld + k];
                const cplx t = cmul(l, u);
                A[size_t(j) * ld + i].re -= t.re;
                A[size_t(j) * ld + i].im -= t.im;
            }
        }
        __syncthreads();
    }
}





// Inverse of the bs x bs diagonal blocks of a factored LU (unit-lower L and/or
// upper U), one CTA per (block, matrix).  4 lanes per column (bs = 64 -> 256
// threads) split each dot product; a column's lanes share a warp, so the
// row-by-row recurrences need only warp-level synchronisation.  Output per
// block: [L^{-1} | U^{-1}] as two bs x bs column-major tiles (ld bs).
__global__ void __launch_bounds__(512) tri_inv_kernel(int n, int ld, cplx* const* __restrict__ Ap,
                                                      cplx* const* __restrict__ Op, int bs, int k0_first, int mode,
                                                      int tile0) {
    // Blocked in 16 x 16 tiles: the diagonal tiles are inverted concurrently
    // (64 threads each, a 16-step recurrence), then each block row of the
    // inverse is two small tile products, X_ij = -X_ii sum_k T_ik X_kj, so the
    // serial chain is 16 rows plus bs/16 - 1 product steps instead of bs rows.
    // Tiles are padded to ld bs+1 (distinct banks for the columns of a warp).
    // mode 3 runs with 512 threads: L^{-1} on threads 0-255 and U^{-1} on
    // 256-511 at the same time, each half with its own buffers and barrier.
    extern __shared__ cplx smem[];
    const int lp = bs + 1, nbk = bs / 16;
    const int half = (mode == 3) ? int(threadIdx.x >> 8) : 0;
    const int which = (mode == 3) ? (half ? 2 : 1) : mode;  // 1: lower, 2: upper
    cplx* T = smem;                                          // bs x bs block of the factor (ld lp)
    cplx* X = T + bs * lp + half * bs * lp;                  // inverse being built
    cplx* Y = T + 3 * bs * lp + half * 768;                  // 3 scratch 16 x 16 tiles (ld 16)
    cplx* Dinv = T + 3 * bs * lp + 2 * 768;                  // bs reciprocals of the diagonal
    const cplx* A = Ap[blockIdx.y];
    cplx* O = Op[blockIdx.y] + size_t(tile0 + blockIdx.x) * 2 * bs * bs + (which == 2 ? size_t(bs) * bs : 0);
    const int k0 = k0_first + blockIdx.x * bs;
    const int sz = min(bs, n - k0);
    // rows/columns past the matrix end act as identity
    for (int e = threadIdx.x; e < bs * bs; e += blockDim.x) {
        const int i = e % bs, j = e / bs;
        T[j * lp + i] = (i < sz && j < sz) ? A[size_t(k0 + j) * ld + k0 + i] : cplx{i == j ? 1.0 : 0.0, 0.0};
    }
    __syncthreads();
    const int tid = threadIdx.x & 255;
    auto bar = [&]() { asm volatile("bar.sync %0, 256;" ::"r"(1 + half)); };
    const int g = tid >> 6, t = tid & 63, jj = t >> 2, part = t & 3;  // diagonal-tile group, its column
    const int pr = tid & 15, pc = tid >> 4;                             // tile-product element
    for (int e = tid; e < bs * lp; e += 256) X[e] = cplx{0, 0};
    if (which == 1) {
        bar();
        if (g < nbk) {  // unit-lower diagonal tiles
            const int o = g * 16;
            for (int i = 0; i < 16; ++i) {
                cplx sacc{0, 0};
                if (i > jj)
                    for (int l = jj + part; l < i; l += 4) {
                        const cplx v = cmul(T[(o + l) * lp + o + i], X[(o + jj) * lp + o + l]);
                        sacc.re += v.re;
                        sacc.im += v.im;
                    }
                sacc.re += __shfl_xor_sync(0xffffffffu, sacc.re, 1);
                sacc.im += __shfl_xor_sync(0xffffffffu, sacc.im, 1);
                sacc.re += __shfl_xor_sync(0xffffffffu, sacc.re, 2);
                sacc.im += __shfl_xor_sync(0xffffffffu, sacc.im, 2);
                if (part == 0 && i >= jj) X[(o + jj) * lp + o + i] = (i == jj) ? cplx{1, 0} : cplx{-sacc.re, -sacc.im};
                __syncwarp();
            }
        }
        bar();
        for (int bi = 1; bi < nbk; ++bi) {
            for (int bj = 0; bj < bi; ++bj) {  // Y_bj = sum_{k=bj}^{bi-1} L_{bi,k} X_{k,bj}
                cplx acc{0, 0};
                for (int l = bj * 16; l < bi * 16; ++l) {
                    const cplx v = cmul(T[l * lp + bi * 16 + pr], X[(bj * 16 + pc) * lp + l]);
                    acc.re += v.re;
                    acc.im += v.im;
                }
                Y[bj * 256 + pc * 16 + pr] = acc;
            }
            bar();
            for (int bj = 0; bj < bi; ++bj) {  // X_{bi,bj} = -X_{bi,bi} Y_bj
                cplx acc{0, 0};
                for (int m = 0; m < 16; ++m) {
                    const cplx v = cmul(X[(bi * 16 + m) * lp + bi * 16 + pr], Y[bj * 256 + pc * 16 + m]);
                    acc.re += v.re;
                    acc.im += v.im;
                }
                X[(bj * 16 + pc) * lp + bi * 16 + pr] = cplx{-acc.re, -acc.im};
            }
            bar();
        }
        for (int e = tid; e < bs * bs; e += 256) O[e] = X[(e / bs) * lp + e % bs];
    } else {
        // reciprocals of the diagonal, all at once (an FP64 division on the
        // substitution's critical path costs ~600 cycles per row)
        for (int i = tid; i < bs; i += 256) {
            const cplx d = T[i * lp + i];
            Dinv[i] = (d.re == 0.0 && d.im == 0.0) ? cplx{0, 0} : cdiv(cplx{1.0, 0.0}, d);
        }
        bar();
        if (g < nbk) {  // upper diagonal tiles
            const int o = g * 16;
            for (int i = 15; i >= 0; --i) {
                cplx sacc{0, 0};
                if (i < jj)
                    for (int l = i + 1 + part; l <= jj; l += 4) {
                        const cplx v = cmul(T[(o + l) * lp + o + i], X[(o + jj) * lp + o + l]);
                        sacc.re += v.re;
                        sacc.im += v.im;
                    }
                sacc.re += __shfl_xor_sync(0xffffffffu, sacc.re, 1);
                sacc.im += __shfl_xor_sync(0xffffffffu, sacc.im, 1);
                sacc.re += __shfl_xor_sync(0xffffffffu, sacc.re, 2);
                sacc.im += __shfl_xor_sync(0xffffffffu, sacc.im, 2);
                if (part == 0 && i <= jj) {
                    const cplx num{(i == jj ? 1.0 : 0.0) - sacc.re, -sacc.im};
                    X[(o + jj) * lp + o + i] = cmul(num, Dinv[o + i]);
                }
                __syncwarp();
            }
        }
        bar();
        for (int bi = nbk - 2; bi >= 0; --bi) {
            for (int bj = bi + 1; bj < nbk; ++bj) {  // Y_bj = sum_{k=bi+1}^{bj} U_{bi,k} X_{k,bj}
                cplx acc{0, 0};
                for (int l = (bi + 1) * 16; l < (bj + 1) * 16; ++l) {
                    const cplx v = cmul(T[l * lp + bi * 16 + pr], X[(bj * 16 + pc) * lp + l]);
                    acc.re += v.re;
                    acc.im += v.im;
                }
                Y[(bj - bi - 1) * 256 + pc * 16 + pr] = acc;
            }
            bar();
            for (int bj = bi + 1; bj < nbk; ++bj) {  // X_{bi,bj} = -X_{bi,bi} Y_bj
                cplx acc{0, 0};
                for (int m = 0; m < 16; ++m) {
                    const cplx v = cmul(X[(bi * 16 + m) * lp + bi * 16 + pr], Y[(bj - bi - 1) * 256 + pc * 16 + m]);
                    acc.re += v.re;
                    acc.im += v.im;
                }
                X[(bj * 16 + pc) * lp + bi * 16 + pr] = cplx{-acc.re, -acc.im};
            }
            bar();
        }
        for (int e = tid; e < bs * bs; e += 256) O[e] = X[(e / bs) * lp + e % bs];
    }
}

// Row interchanges as a gather: perm_build_kernel composes the pivots
// [k0, kend) of each matrix into a permutation of rows [k0, n) once (global
// scratch); row_permute_kernel then permutes columns with one warp per column
// (coalesced reads/writes through a shared-memory staging column).
constexpr int kPermWarps = 8;
// Per matrix the scratch holds [perm (n) | moved rows (n) | count]: only the
// rows the interchanges move are gathered and written back (at most
// 2 (kend - k0) of the n - k0), e.g. 32 of ~600 rows for a 16-column leaf.
__global__ void perm_build_kernel(int n, const int* const* __restrict__ Pp, int* __restrict__ perm_out, int k0,
                                  int kend) {
    const int* ipiv = Pp[blockIdx.x];
    int* perm = perm_out + size_t(blockIdx.x) * (2 * n + 1);
    int* moved = perm + n;
    __shared__ int cnt;
    const int rows = n - k0;
    for (int i = threadIdx.x; i < rows; i += blockDim.x) perm[i] = k0 + i;
    if (threadIdx.x == 0) cnt = 0;
    __syncthreads();
    if (threadIdx.x == 0)
        for (int k = k0; k < kend; ++k) {
            const int p = ipiv[k];
            if (p != k) {
                const int t = perm[k - k0];
                perm[k - k0] = perm[p - k0];
                perm[p - k0] = t;
            }
        }
    __syncthreads();
    for (int i = threadIdx.x; i < rows; i += blockDim.x)
        if (perm[i] != k0 + i) moved[atomicAdd(&cnt, 1)] = i;
    __syncthreads();
    if (threadIdx.x == 0) perm[2 * n] = cnt;
}
__global__ void __launch_bounds__(256) row_permute_kernel(int n, int ld, cplx* const* __restrict__ Ap,
                                                          const int* __restrict__ perm_all, int k0, int c0, int c1) {
    extern __shared__ cplx tmp_smem[];
    cplx* A = Ap[blockIdx.y];
    const int* perm = perm_all + size_t(blockIdx.y) * (2 * n + 1);
    const int* moved = perm + n;
    const int cnt = perm[2 * n];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    cplx* tw = tmp_smem + size_t(warp) * (n - k0);
    for (int c = c0 + blockIdx.x * kPermWarps + warp; c < c1; c += gridDim.x * kPermWarps) {
        cplx* col = A + size_t(c) * ld;
        for (int t = lane; t < cnt; t += 32) tw[t] = col[perm[moved[t]]];
        __syncwarp();
        for (int t = lane; t < cnt; t += 32) col[k0 + moved[t]] = tw[t];
        __syncwarp();
    }
}

// LU of one panel of w <= 16 columns held entirely in shared memory
// (rows c0..n-1), partial pivoting on the modulus like Eigen's PartialPivLU.
constexpr int kLeaf = 16;
__global__ void __launch_bounds__(256) lu_panel_smem_kernel(int n, int ld, cplx* const* __restrict__ Ap,
                                                            int* const* __restrict__ Pp, int c0, int w, int* singular) {
    extern __shared__ cplx pnl[];
    cplx* A = Ap[blockIdx.x];
    int* ipiv = Pp[blockIdx.x];
    const int rows = n - c0;
    __shared__ double shv[32];
    __shared__ int shi[32];
    const int tid = threadIdx.x;
    // panel load: 8 independent loads in flight per thread (the loop would
    // otherwise expose one DRAM latency per element)
    for (int e0 = tid; e0 < rows * w; e0 += 8 * blockDim.x) {
        cplx v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e = e0 + u * blockDim.x;
            if (e < rows * w) v[u] = A[size_t(c0 + e / rows) * ld + c0 + e % rows];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e = e0 + u * blockDim.x;
            if (e < rows * w) pnl[e] = v[u];
        }
    }
    __syncthreads();
    for (int k = 0; k < w; ++k) {
        double v = -1.0;
        int idx = rows;
        for (int i = k + tid; i < rows; i += blockDim.x) {
            const double a = sqrt(cabs2(pnl[k * rows + i]));
            if (a > v) { v = a; idx = i; }
        }
        double best;
        int piv;
        block_argmax(v, idx, shv, shi, best, piv);
        if (tid == 0) ipiv[c0 + k] = c0 + piv;
        if (piv != k && tid < w) {
            const cplx t = pnl[tid * rows + k];
            pnl[tid * rows + k] = pnl[tid * rows + piv];
            pnl[tid * rows + piv] = t;
        }
        __syncthreads();
        const cplx d = pnl[k * rows + k];
        const bool zero = (d.re == 0.0 && d.im == 0.0);
        if (zero) {
            if (tid == 0) singular[blockIdx.x] = 1;
        }
        const cplx inv = zero ? cplx{0, 0} : cdiv(cplx{1.0, 0.0}, d);
        for (int i = k + 1 + tid; i < rows; i += blockDim.x) {
            cplx l = pnl[k * rows + i];
            if (!zero) {
                l = cmul(l, inv);
                pnl[k * rows + i] = l;
            }
            for (int j = k + 1; j < w; ++j) {
                const cplx t = cmul(l, pnl[j * rows + k]);
                pnl[j * rows + i].re -= t.re;
                pnl[j * rows + i].im -= t.im;
            }
        }
        __syncthreads();
    }
    for (int e = tid; e < rows * w; e += blockDim.x) {
        const int i = e % rows, j = e / rows;
        A[size_t(c0 + j) * ld + c0 + i] = pnl[j * rows + i];
    }
}

// Right-looking LU step for one 16-column panel [k0, k0 + w) of every matrix:
// lu_rl_panel_kernel (one CTA per matrix) factors the panel with partial
// pivoting in shared memory (rows k0..n); lu_rl_cols_kernel (one warp per
// column outside the panel, many CTAs per matrix) applies the panel's row
// interchanges (LAPACK xGETRF order) and, right of the panel, the unit-lower
// solve U12 = L11^{-1} A12; the trailing update is one batched 3M GEMM.
constexpr int kRlW = 16;
// slot map of a panel's interchanges for lu_rl_cols_kernel: slots 0..w-1 are
// rows k0..k0+w-1, slots 16..31 the distinct external rows touched; map[q] =
// slot whose original value ends in slot q, map[32 + q - 16] = row of slot q
constexpr int kRlMap = 48;
__global__ void __launch_bounds__(256) lu_rl_panel_kernel(int n, int ld, cplx* const* __restrict__ Ap,
                                                          int* const* __restrict__ Pp, int k0, int w,
                                                          int* singular, int* __restrict__ rl_map) {
    extern __shared__ cplx pnl[];
    cplx* A = Ap[blockIdx.x];
    int* ipiv = Pp[blockIdx.x];
    const int rows = n - k0;
    __shared__ double shv[32];
    __shared__ int shi[32];
    __shared__ int spiv[kRlW];
    const int tid = threadIdx.x;
    // panel load: 8 independent loads in flight per thread (the loop would
    // otherwise expose one DRAM latency per element)
    for (int e0 = tid; e0 < rows * w; e0 += 8 * blockDim.x) {
        cplx v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e = e0 + u * blockDim.x;
            if (e < rows * w) v[u] = A[size_t(k0 + e / rows) * ld + k0 + e % rows];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e = e0 + u * blockDim.x;
            if (e < rows * w) pnl[e] = v[u];
        }
    }
    __syncthreads();
    for (int k = 0; k < w; ++k) {
        double v = -1.0;
        int idx = rows;
        for (int i = k + tid; i < rows; i += blockDim.x) {
            const double a = cabs2(pnl[k * rows + i]);
            if (a > v) { v = a; idx = i; }
        }
        double best;
        int piv;
        block_argmax(v, idx, shv, shi, best, piv);
        if (tid == 0) {
            ipiv[k0 + k] = k0 + piv;
            spiv[k] = piv;
        }
        if (piv != k && tid < w) {
            const cplx t = pnl[tid * rows + k];
            pnl[tid * rows + k] = pnl[tid * rows + piv];
            pnl[tid * rows + piv] = t;
        }
        __syncthreads();
        const cplx d = pnl[k * rows + k];
        const bool zero = (d.re == 0.0 && d.im == 0.0);
        if (zero && tid == 0) singular[blockIdx.x] = 1;
        const cplx inv = zero ? cplx{0, 0} : cdiv(cplx{1.0, 0.0}, d);
        for (int i = k + 1 + tid; i < rows; i += blockDim.x) {
            cplx l = pnl[k * rows + i];
            if (!zero) {
                l = cmul(l, inv);
                pnl[k * rows + i] = l;
            }
            for (int j = k + 1; j < w; ++j) {
                const cplx t = cmul(l, pnl[j * rows + k]);
                pnl[j * rows + i].re -= t.re;
                pnl[j * rows + i].im -= t.im;
            }
        }
        __syncthreads();
    }
    for (int e = tid; e < rows * w; e += blockDim.x) {
        const int i = e % rows, j = e / rows;
        A[size_t(k0 + j) * ld + k0 + i] = pnl[j * rows + i];
    }
    if (tid == 0) {  // replay the interchanges on slots once per matrix
        int rowof[32], perm[32];
        int nslot = kRlW;
        for (int q = 0; q < 32; ++q) {
            rowof[q] = q < kRlW ? k0 + q : -1;
            perm[q] = q;
        }
        for (int t = 0; t < w; ++t) {
            const int p = k0 + spiv[t];
            if (p == k0 + t) continue;
            int sp = -1;
            if (p < k0 + kRlW) sp = p - k0;
            else {
                for (int q = kRlW; q < nslot; ++q)
                    if (rowof[q] == p) sp = q;
                if (sp < 0) {
                    sp = nslot++;
                    rowof[sp] = p;
                }
            }
            const int tmp = perm[t];
            perm[t] = perm[sp];
            perm[sp] = tmp;
        }
        int* mp = rl_map + size_t(blockIdx.x) * kRlMap;
        for (int q = 0; q < 32; ++q) mp[q] = perm[q];
        for (int q = kRlW; q < 32; ++q) mp[32 + q - kRlW] = rowof[q];
    }
}

constexpr int kRegPanelMaxRows = 640;  // rows of a single-CTA panel (one thread per row)

// Same factorization with the panel in shared memory ([column][row], one
// thread per row, rolled column loop): no register arrays, so no spills and a
// small loop body that stays in the instruction cache; one barrier per column
// (each warp publishes its candidate pivot row, every warp reduces the
// candidates itself).
__global__ void __launch_bounds__(kRegPanelMaxRows, 1)
    lu_panel_sm2_kernel(int n, int ld, cplx* const* __restrict__ Ap, int* const* __restrict__ Pp, int c0, int w,
                        int* singular, int* __restrict__ rl_map) {
    extern __shared__ cplx pnl2[];  // [w][rows]
    cplx* A = Ap[blockIdx.x];
    int* ipiv = Pp[blockIdx.x];
    const int rows = n - c0;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    __shared__ double shv[32];
    __shared__ int shi[32];
    __shared__ int spiv[kRlW];
    __shared__ double cval[2][kRegPanelMaxRows / 32];
    __shared__ int cidx[2][kRegPanelMaxRows / 32];
    __shared__ cplx crow[2][kRegPanelMaxRows / 32][kRlW + 1];
    __shared__ cplx krow[2][kRlW];
    const bool own = tid < rows;
    if (own) {  // 16 independent loads in flight per thread
        cplx v[kRlW];
#pragma unroll
        for (int j = 0; j < kRlW; ++j)
            if (j < w) v[j] = A[size_t(c0 + j) * ld + c0 + tid];
#pragma unroll
        for (int j = 0; j < kRlW; ++j)
            if (j < w) pnl2[j * rows + tid] = v[j];
    }
    __syncthreads();
    for (int k = 0; k < w; ++k) {
        const int par = k & 1;
        const cplx rk = own ? pnl2[k * rows + tid] : cplx{0, 0};
        double v = (own && tid >= k) ? cabs2(rk) : -1.0;
        int idx = (own && tid >= k) ? tid : 1 << 30;
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, v, o);
            const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
            if (ov > v || (ov == v && oi < idx)) {
                v = ov;
                idx = oi;
            }
        }
        if (idx != (1 << 30)) {  // the warp publishes its candidate row cooperatively
            if (lane < w) crow[par][warp][lane] = pnl2[lane * rows + idx];
            if (tid == idx) {
                cval[par][warp] = v;
                cidx[par][warp] = idx;
                crow[par][warp][kRlW] = (rk.re == 0.0 && rk.im == 0.0) ? cplx{0, 0} : fast_cinv(rk);
            }
        } else if (lane == 0) {
            cval[par][warp] = -1.0;
            cidx[par][warp] = 1 << 30;
        }
        if (warp == (k >> 5) && lane < w) krow[par][lane] = pnl2[lane * rows + k];
        __syncthreads();
        double bv = lane < nw ? cval[par][lane] : -1.0;
        int bi = lane < nw ? cidx[par][lane] : 1 << 30;
        int bw = lane;
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            const int ow = __shfl_xor_sync(0xffffffffu, bw, o);
            if (ov > bv || (ov == bv && oi < bi)) {
                bv = ov;
                bi = oi;
                bw = ow;
            }
        }
        const int piv = bi;
        const cplx* prow = crow[par][bw];
        if (tid == 0) {
            ipiv[c0 + k] = c0 + piv;
            spiv[k] = piv;
            if (bv == 0.0) singular[blockIdx.x] = 1;
        }
        cplx ak = rk;  // this thread's entry in column k after the interchange
        if (piv != k) {  // rows k and piv written by their warps' lanes (one column per lane)
            if (warp == (k >> 5) && lane < w) pnl2[lane * rows + k] = prow[lane];
            if (warp == (piv >> 5) && lane < w) pnl2[lane * rows + piv] = krow[par][lane];
            if (tid == piv) ak = krow[par][k];
            __syncwarp();
        }
        const cplx inv = prow[kRlW];
        const bool zero = (inv.re == 0.0 && inv.im == 0.0);
        if (own && tid > k) {
            const cplx l = zero ? ak : cmul(ak, inv);
            pnl2[k * rows + tid] = l;
#pragma unroll
            for (int j = 1; j < kRlW; ++j) {  // predicated, independent read-modify-writes
                if (j > k && j < w) {
                    const cplx pj = prow[j];
                    cplx a = pnl2[j * rows + tid];
                    a.re -= l.re * pj.re - l.im * pj.im;
                    a.im -= l.re * pj.im + l.im * pj.re;
                    pnl2[j * rows + tid] = a;
                }
            }
        }
    }
    __syncthreads();
    if (own) {
#pragma unroll
        for (int j = 0; j < kRlW; ++j)
            if (j < w) A[size_t(c0 + j) * ld + c0 + tid] = pnl2[j * rows + tid];
    }
    if (rl_map && tid == 0) {  // replay the interchanges on slots once per matrix
        int* rowof = shi;
        int* perm = reinterpret_cast<int*>(shv);
        int nslot = kRlW;
        for (int q = 0; q < 32; ++q) {
            rowof[q] = q < kRlW ? c0 + q : -1;
            perm[q] = q;
        }
        for (int t = 0; t < w; ++t) {
            const int p = c0 + spiv[t];
            if (p == c0 + t) continue;
            int sp = -1;
            if (p < c0 + kRlW) sp = p - c0;
            else {
                for (int q = kRlW; q < nslot; ++q)
                    if (rowof[q] == p) sp = q;
                if (sp < 0) {
                    sp = nslot++;
                    rowof[sp] = p;
                }
            }
            const int tmp = perm[t];
            perm[t] = perm[sp];
            perm[sp] = tmp;
        }
        int* mp = rl_map + size_t(blockIdx.x) * kRlMap;
        for (int q = 0; q < 32; ++q) mp[q] = perm[q];
        for (int q = kRlW; q < 32; ++q) mp[32 + q - kRlW] = rowof[q];
    }
}

// ---------------------------------------------------------------------------
// Wide LU panel: one CTA factors a whole (n - c0) x w column panel (w <= 64)
// of one matrix -- the bottom of the recursion in one launch instead of four
// 16-column panels, their interchanges, tile inverses and K <= 32 updates.
// One thread per row (n - c0 <= 640); 8-column sub-panels in registers.
// Rows stay in place while the panel is factored: each thread remembers the
// step at which its row became a pivot and the pivot search runs over the
// rows not chosen yet; after each sub-panel the later columns of the panel
// are updated in place through U12 = L11^{-1} A[pivot rows, later columns].
// At the end the LAPACK interchange sequence is replayed on row indices
// (ipiv, 0-based absolute rows as lu_panel_sm2 writes them) and the panel's
// rows are moved to their final positions, so the factors leave exactly as a
// sequential partial-pivoting LU would lay them out.
// ---------------------------------------------------------------------------
constexpr int kWpMax = 64;                     // widest panel
constexpr int kWpSub = 8;                      // sub-panel (register) width
constexpr int kWpThreads = 640;                // one thread per row
constexpr int kWpWarps = kWpThreads / 32;

// kStaged: the in-panel trailing update streams each thread's row of the later
// columns through a private cp.async pipeline in shared memory (kWpSt stages of
// kWpLd columns, (kWpSt - 1) kWpLd columns in flight per thread) instead of
// register double-buffering 4 columns: the update is bound by the L2 round
// trips of those loads.  Each thread reads back only what it copied itself, so
// the pipeline needs no barrier.  Same operations in the same order.
constexpr int kWpLd = 4, kWpSt = 4;
size_t wpanel_smem(int threads) { return size_t(kWpSt) * kWpLd * threads * sizeof(cplx); }

template <bool kStaged>
__global__ void __launch_bounds__(kWpThreads, 1)
    lu_wpanel_kernel(int n, int ld, cplx* const* __restrict__ Ap, int* const* __restrict__ Pp, int c0, int w,
                     int* __restrict__ singular) {
    extern __shared__ cplx wp_stage[];  // [kWpSt][kWpLd][blockDim.x] (kStaged)
    __shared__ cplx cand[2][kWpWarps][kWpSub];
    __shared__ double cval[2][kWpWarps];
    __shared__ int cidx[2][kWpWarps];
    __shared__ cplx L11[kWpSub][kWpSub];
    __shared__ cplx U12[kWpSub][kWpMax];
    __shared__ int spv[kWpMax];
    __shared__ int rowat[kWpThreads], posof[kWpThreads];
    cplx* A = Ap[blockIdx.x];
    const int rows = n - c0;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    const bool own = tid < rows;
    cplx* arow = A + size_t(c0) * ld + c0 + tid;  // this thread's row, column c0
    int mystep = own ? (1 << 30) : -1;
    bool sing = false;
    for (int p0 = 0; p0 < w; p0 += kWpSub) {
        const int sw = min(kWpSub, w - p0);
        cplx s[kWpSub];
#pragma unroll
        for (int jj = 0; jj < kWpSub; ++jj) s[jj] = (own && jj < sw) ? arow[size_t(p0 + jj) * ld] : cplx{0, 0};
#pragma unroll
        for (int kk = 0; kk < kWpSub; ++kk) {
            if (kk >= sw) break;
            const int k = p0 + kk, par = kk & 1;
            const bool live = mystep > k;
            double v = live ? cabs2(s[kk]) : -1.0;
            int idx = live ? tid : (1 << 30);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, v, o);
                const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
                if (ov > v || (ov == v && oi < idx)) {
                    v = ov;
                    idx = oi;
                }
            }
            if (idx == tid) {
#pragma unroll
                for (int jj = kk; jj < kWpSub; ++jj) cand[par][warp][jj] = s[jj];
                cval[par][warp] = v;
                cidx[par][warp] = idx;
            } else if (lane == 0 && idx == (1 << 30)) {
                cval[par][warp] = -1.0;
                cidx[par][warp] = 1 << 30;
            }
            __syncthreads();
            double bv = lane < nw ? cval[par][lane] : -1.0;
            int bi = lane < nw ? cidx[par][lane] : (1 << 30);
            int bw = lane;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                const int ow = __shfl_xor_sync(0xffffffffu, bw, o);
                if (ov > bv || (ov == bv && oi < bi)) {
                    bv = ov;
                    bi = oi;
                    bw = ow;
                }
            }
            const cplx* prow = cand[par][bw];
            if (tid == 0) spv[k] = bi;
            if (tid == bi) mystep = k;
            const cplx d = prow[kk];
            const bool zero = (d.re == 0.0 && d.im == 0.0);
            sing |= zero;
            if (live && tid != bi) {
                const cplx l = zero ? s[kk] : cmul(s[kk], fast_cinv(d));
                s[kk] = l;
#pragma unroll
                for (int jj = kk + 1; jj < kWpSub; ++jj) {
                    const cplx u = prow[jj];
                    s[jj].re -= l.re * u.re - l.im * u.im;
                    s[jj].im -= l.re * u.im + l.im * u.re;
                }
            }
        }
        // sub-panel back in place (L of live rows, U / L of its pivot rows)
        if (own) {
#pragma unroll
            for (int jj = 0; jj < kWpSub; ++jj)
                if (jj < sw) arow[size_t(p0 + jj) * ld] = s[jj];
        }
        const int ncol = w - p0 - sw;
        if (ncol <= 0) break;
        // L11: row kk0 of the pivot chosen at step p0 + kk0
        const int kk0 = mystep - p0;
        if (own && kk0 >= 0 && kk0 < sw) {
#pragma unroll
            for (int kk = 0; kk < kWpSub; ++kk) L11[kk0][kk] = kk < kk0 ? s[kk] : cplx{0, 0};
        }
        __syncthreads();
        if (tid < ncol) {  // U12 = L11^{-1} A[pivots, later columns], one thread per column
            const cplx* col = A + size_t(c0 + p0 + sw + tid) * ld + c0;
            cplx u[kWpSub];
#pragma unroll
            for (int kk = 0; kk < kWpSub; ++kk)  // independent gathers in flight
                if (kk < sw) u[kk] = col[spv[p0 + kk]];
#pragma unroll
            for (int kk = 0; kk < kWpSub; ++kk) {
#pragma unroll
                for (int k2 = 0; k2 < kk; ++k2) {
                    const cplx lv = L11[kk][k2];
                    u[kk].re -= lv.re * u[k2].re - lv.im * u[k2].im;
                    u[kk].im -= lv.re * u[k2].im + lv.im * u[k2].re;
                }
                if (kk < sw) U12[kk][tid] = u[kk];
            }
        }
        __syncthreads();
        // later columns of the panel: live rows and this sub-panel's pivot rows
        // (with their multipliers from before they were chosen)
        if (own && mystep >= p0) {
            cplx lv[kWpSub];
#pragma unroll
            for (int kk = 0; kk < kWpSub; ++kk)
                lv[kk] = (kk < sw && p0 + kk < mystep) ? s[kk] : cplx{0, 0};
            cplx* dst = arow + size_t(p0 + sw) * ld;
            if (kStaged) {
                const int nt = blockDim.x, ngrp = (ncol + kWpLd - 1) / kWpLd;
                auto issue = [&](int gi) {
                    cplx* st = wp_stage + size_t((gi % kWpSt) * kWpLd) * nt + tid;
#pragma unroll
                    for (int q = 0; q < kWpLd; ++q) {
                        const int t = gi * kWpLd + q;
                        const bool ok = t < ncol;
                        cp_async16(st + size_t(q) * nt, ok ? (const void*)(dst + size_t(t) * ld) : (const void*)dst, ok);
                    }
                };
#pragma unroll
                for (int gi = 0; gi < kWpSt - 1; ++gi) {
                    if (gi < ngrp) issue(gi);
                    cp_async_commit();
                }
                for (int gi = 0; gi < ngrp; ++gi) {
                    if (gi + kWpSt - 1 < ngrp) issue(gi + kWpSt - 1);
                    cp_async_commit();
                    cp_async_wait<kWpSt - 1>();
                    const cplx* st = wp_stage + size_t((gi % kWpSt) * kWpLd) * nt + tid;
#pragma unroll
                    for (int q = 0; q < kWpLd; ++q) {
                        const int t = gi * kWpLd + q;
                        cplx a = st[size_t(q) * nt];
#pragma unroll
                        for (int kk = 0; kk < kWpSub; ++kk) {
                            const cplx u = U12[kk][min(t, kWpMax - 1)];
                            a.re -= lv[kk].re * u.re - lv[kk].im * u.im;
                            a.im -= lv[kk].re * u.im + lv[kk].im * u.re;
                        }
                        if (t < ncol) dst[size_t(t) * ld] = a;
                    }
                }
                cp_async_wait<0>();
            } else {
            constexpr int kLd = 4;  // a group of columns; the next group's loads fly during its updates
            cplx an[kLd];
#pragma unroll
            for (int q = 0; q < kLd; ++q)
                if (q < ncol) an[q] = dst[size_t(q) * ld];
            for (int t0 = 0; t0 < ncol; t0 += kLd) {
                cplx a[kLd];
#pragma unroll
                for (int q = 0; q < kLd; ++q) a[q] = an[q];
#pragma unroll
                for (int q = 0; q < kLd; ++q)
                    if (t0 + kLd + q < ncol) an[q] = dst[size_t(t0 + kLd + q) * ld];
#pragma unroll
                for (int q = 0; q < kLd; ++q) {
#pragma unroll
                    for (int kk = 0; kk < kWpSub; ++kk) {
                        const cplx u = U12[kk][t0 + q];
                        a[q].re -= lv[kk].re * u.re - lv[kk].im * u.im;
                        a[q].im -= lv[kk].re * u.im + lv[kk].im * u.re;
                    }
                    if (t0 + q < ncol) dst[size_t(t0 + q) * ld] = a[q];
                }
            }
            }
        }
        __syncthreads();
    }
    if (sing && tid == 0) singular[blockIdx.x] = 1;
    // replay the interchange sequence on row indices
    for (int i = tid; i < rows; i += blockDim.x) {
        rowat[i] = i;
        posof[i] = i;
    }
    __syncthreads();
    if (tid == 0) {
        int* ipiv = Pp[blockIdx.x];
        for (int k = 0; k < w; ++k) {
            const int p = spv[k], loc = posof[p], other = rowat[k];
            ipiv[c0 + k] = c0 + loc;
            rowat[k] = p;
            rowat[loc] = other;
            posof[p] = k;
            posof[other] = loc;
        }
    }
    __syncthreads();
    // move every row of the panel to its final position, 8 columns at a time
    const int dest = own ? posof[tid] : 0;
    for (int p0 = 0; p0 < w; p0 += kWpSub) {
        cplx v[kWpSub];
#pragma unroll
        for (int jj = 0; jj < kWpSub; ++jj)
            if (own && p0 + jj < w) v[jj] = arow[size_t(p0 + jj) * ld];
        __syncthreads();
        if (own && dest != tid) {
            cplx* drow = A + size_t(c0) * ld + c0 + dest;
#pragma unroll
            for (int jj = 0; jj < kWpSub; ++jj)
                if (p0 + jj < w) drow[size_t(p0 + jj) * ld] = v[jj];
        }
        __syncthreads();
    }
}

// one warp per column: lanes 0..w-1 hold rows k0..k0+w-1, lanes 16.. the
// external rows the interchanges touch; the interchange sequence is replayed
// on lane indices, the values move with one shuffle, the unit-lower solve is
// a w-step shuffle broadcast.
__global__ void __launch_bounds__(256) lu_rl_cols_kernel(int n, int ld, cplx* const* __restrict__ Ap,
                                                         const int* __restrict__ rl_map, int k0, int w) {
    cplx* A = Ap[blockIdx.y];
    const int lane = threadIdx.x & 31;
    const int c = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (c >= n - w) return;
    const int col = c < k0 ? c : c + w;
    cplx* Ac = A + size_t(col) * ld;
    const int* mp = rl_map + size_t(blockIdx.y) * kRlMap;
    int src = mp[lane];
    const int ext_row = lane >= kRlW ? mp[32 + lane - kRlW] : -1;
    if (lane < kRlW && lane >= w) src = lane;
    cplx v{0, 0};
    if (lane < w) v = Ac[k0 + lane];
    else if (ext_row >= 0) v = Ac[ext_row];
    cplx nv;
    nv.re = __shfl_sync(0xffffffffu, v.re, src);
    nv.im = __shfl_sync(0xffffffffu, v.im, src);
    if (col > k0) {  // U12 = L11^{-1} A12 (unit lower, L11 in the factored panel)
        const cplx* Lp = A + size_t(k0) * ld + k0;
        cplx lrow[kRlW];  // this lane's row of L11, loaded up front (independent loads)
#pragma unroll
        for (int u = 0; u < kRlW; ++u) lrow[u] = (u < lane && lane < w) ? Lp[size_t(u) * ld + lane] : cplx{0, 0};
#pragma unroll
        for (int u = 0; u + 1 < kRlW; ++u) {
            if (u + 1 >= w) break;
            cplx ru;
            ru.re = __shfl_sync(0xffffffffu, nv.re, u);
            ru.im = __shfl_sync(0xffffffffu, nv.im, u);
            const cplx l = lrow[u];
            nv.re -= l.re * ru.re - l.im * ru.im;
            nv.im -= l.re * ru.im + l.im * ru.re;
        }
    }
    if (lane < w) Ac[k0 + lane] = nv;
    else if (ext_row >= 0) Ac[ext_row] = nv;
}


__global__ void maxabs_kernel(const cplx* X, int m, int n, int ld, size_t stride, double* out) {
    const cplx* A = X + stride * blockIdx.x;
    double v = 0.0;
    if (ld == m) {  // contiguous: one linear sweep, four loads in flight per thread
        const size_t tot = size_t(m) * n;
        double v1 = 0.0, v2 = 0.0, v3 = 0.0;
        size_t e = threadIdx.x;
        const size_t st = blockDim.x;
        for (; e + 3 * st < tot; e += 4 * st) {
            v = fmax(v, cabs2(A[e]));
            v1 = fmax(v1, cabs2(A[e + st]));
            v2 = fmax(v2, cabs2(A[e + 2 * st]));
            v3 = fmax(v3, cabs2(A[e + 3 * st]));
        }
        for (; e < tot; e += st) v = fmax(v, cabs2(A[e]));
        v = sqrt(fmax(fmax(v, v1), fmax(v2, v3)));
    } else {
        for (int j = 0; j < n; ++j)
            for (int i = threadIdx.x; i < m; i += blockDim.x) v = fmax(v, sqrt(cabs2(A[size_t(j) * ld + i])));
    }
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    __shared__ double sh[32];
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < int(blockDim.x >> 5); ++w) t = fmax(t, sh[w]);
        out[blockIdx.x] = t;
    }
}

// Frobenius norm in one pass (plain sum of squares, as Eigen's norm()); the
// max-scaled second pass runs only when the sum leaves the normal range.
// maxo (optional): the max modulus from the same pass.
__global__ void fro_kernel(const cplx* X, int m, int n, int ld, size_t stride, double* out, double* maxo) {
    const cplx* A = X + stride * blockIdx.x;
    __shared__ double sh[32];
    double mx = 0.0, s = 0.0;
    if (ld == m) {  // contiguous: one linear sweep, two loads in flight per thread
        const size_t tot = size_t(m) * n, st = blockDim.x;
        double s1 = 0.0, mx1 = 0.0;
        size_t e = threadIdx.x;
        for (; e + st < tot; e += 2 * st) {
            const double a2 = cabs2(A[e]), b2 = cabs2(A[e + st]);
            s += a2;
            s1 += b2;
            mx = fmax(mx, a2);
            mx1 = fmax(mx1, b2);
        }
        for (; e < tot; e += st) {
            const double a2 = cabs2(A[e]);
            s += a2;
            mx = fmax(mx, a2);
        }
        s += s1;
        mx = fmax(mx, mx1);
    } else {
        for (int j = 0; j < n; ++j)
            for (int i = threadIdx.x; i < m; i += blockDim.x) {
                const double a2 = cabs2(A[size_t(j) * ld + i]);
                s += a2;
                mx = fmax(mx, a2);
            }
    }
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = mx;
    __syncthreads();
    double big = 0.0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) big = fmax(big, sh[w]);
    big = sqrt(big);
    __syncthreads();
    double tot = block_sum(s, sh);
    if (!(tot < 1e300) || (tot < 1e-290 && big > 0.0)) {  // out of range: rescale by the max
        const double inv = 1.0 / big;
        s = 0.0;
        for (int j = 0; j < n; ++j)
            for (int i = threadIdx.x; i < m; i += blockDim.x) {
                const cplx a = A[size_t(j) * ld + i];
                s += (a.re * inv) * (a.re * inv) + (a.im * inv) * (a.im * inv);
            }
        tot = block_sum(s, sh);
        if (threadIdx.x == 0) out[blockIdx.x] = big * sqrt(tot);
    } else if (threadIdx.x == 0) {
        out[blockIdx.x] = sqrt(tot);
    }
    if (maxo && threadIdx.x == 0) maxo[blockIdx.x] = big;
}

__global__ void copy_blocks_kernel(const cplx* src, int lds, size_t sstride, cplx* dst, int ldd, size_t dstride,
                                   int m, int n) {
    const cplx* S = src + sstride * blockIdx.y;
    cplx* D = dst + dstride * blockIdx.y;
    for (size_t e = blockIdx.x * blockDim.x + threadIdx.x; e < size_t(m) * n; e += size_t(gridDim.x) * blockDim.x) {
        const int i = int(e % m), j = int(e / m);
        D[size_t(j) * ldd + i] = S[size_t(j) * lds + i];
    }
}

// y = beta y + alpha sum_s A_s x_s: 32 rows x 8 column groups per CTA, partial
// sums reduced through shared memory; reads of A are 512-byte coalesced.
__global__ void __launch_bounds__(256) zgemv_kernel(int M, cplx alpha, cplx beta, const GemvTask* __restrict__ tasks) {
    const GemvTask& T = tasks[blockIdx.y];
    const int tx = threadIdx.x & 31, g = threadIdx.x >> 5;
    const int i = blockIdx.x * 32 + tx;
    __shared__ cplx part[8][32];
    cplx acc{0, 0};
    if (i < M)
        for (int sgi = 0; sgi < T.nseg; ++sgi) {
            const cplx* A = T.A[sgi];
            const cplx* x = T.x[sgi];
            const int lda = T.lda[sgi], nn = T.n[sgi];
            for (int j = g; j < nn; j += 8) {
                const cplx t = cmul(A[size_t(j) * lda + i], x[j]);
                acc.re += t.re;
                acc.im += t.im;
            }
        }
    part[g][tx] = acc;
    __syncthreads();
    if (g == 0 && i < M) {
        cplx s{0, 0};
        for (int q = 0; q < 8; ++q) {
            s.re += part[q][tx].re;
            s.im += part[q][tx].im;
        }
        cplx out = cmul(alpha, s);
        if (beta.re != 0.0 || beta.im != 0.0) {
            const cplx o = cmul(beta, T.y[i]);
            out.re += o.re;
            out.im += o.im;
        }
        T.y[i] = out;
    }
}

// ---- FP64 peak microbenchmarks ----
// ---------------------------------------------------------------------------
// Reciprocal condition estimate of LU factors (the reference's
// PartialPivLU::rcond() <= 1e-15 -> SolverError(layer) test, tridiag.hpp:36-40).
// The block cyclic reduction never forms the Thomas pivots the reference tests,
// so every block it factors -- the level-0 diagonal blocks, the dense
// reduction's pivots at every level -- is checked on its U factor: LAPACK
// xTRCON's estimate rcond(U) = 1 / (||U||_1 est(||U^{-1}||_1)), est by the
// Hager/Higham 1-norm estimator in LAPACK zlacn2's iteration (at most 5
// rounds of U^{-1} x / U^{-H} sign(y), then the alternating-sign test vector).
// With partial pivoting L is unit lower with |l_ij| <= 1, so rcond(U) tracks
// rcond(A) and is exactly 0 when a pivot is 0.
// The triangular solves use the inverse 64 x 64 diagonal tiles of U that the
// LU already formed (tri_inv_kernel: tile kb at Dinv + kb 2 bs^2 + bs^2), so a
// solve is ceil(n/64) steps of (tile mat-vec, block GEMV over the rows above)
// with no sequential pivot chain: bandwidth-bound on U.  A few CTAs loop over
// the blocks, each running all of its block's solves back to back while its U
// (3 MB at n = 608) stays in L2, so the estimate costs about one HBM read of
// the factors and runs beside the cyclic reduction's latency-bound levels on a
// handful of SMs.
// ---------------------------------------------------------------------------
constexpr int kRcT = 512, kRcB = 64;  // threads per CTA; tile = kTB of the LU
static_assert(kRcB == kTB, "rcond solves use the LU's inverse diagonal tiles");
static_assert(kRcT == 512, "rc_solve_u / rc_solve_uh thread layouts assume 512 threads (16 warps)");

__device__ __forceinline__ cplx csign(cplx v) {  // v / |v| (1 for v = 0), zlacn2
    const double a = sqrt(v.re * v.re + v.im * v.im);
    return a > 0.0 ? cplx{v.re / a, v.im / a} : cplx{1.0, 0.0};
}

__device__ double rc_block_sum(double v, double* red) {  // sum over the CTA
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0;
    for (int w = 0; w < kRcT / 32; ++w) s += red[w];
    return s;
}

__device__ int rc_block_argmax(const cplx* x, int n, double* red, int* redi) {  // first max |x_i| (izmax1)
    double v = -1.0;
    int idx = 1 << 30;
    for (int i = threadIdx.x; i < n; i += kRcT) {
        const double a = sqrt(x[i].re * x[i].re + x[i].im * x[i].im);
        if (a > v) { v = a; idx = i; }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
        if (ov > v || (ov == v && oi < idx)) { v = ov; idx = oi; }
    }
    __syncthreads();
    if ((threadIdx.x & 31) == 0) { red[threadIdx.x >> 5] = v; redi[threadIdx.x >> 5] = idx; }
    __syncthreads();
    double bv = red[0];
    int bi = redi[0];
    for (int w = 1; w < kRcT / 32; ++w)
        if (red[w] > bv || (red[w] == bv && redi[w] < bi)) { bv = red[w]; bi = redi[w]; }
    return bi;
}

// x <- U^{-1} x (backward over 64-row tiles).  t: 512-entry scratch.
__device__ void rc_solve_u(const cplx* __restrict__ U, const cplx* __restrict__ Di, int n, int ld, cplx* x, cplx* t) {
    const int tid = threadIdx.x;
    const int row = tid >> 3, part = tid & 7;  // 8 lanes per tile row (kRcT = 512 = 64 x 8)
    for (int kb = (n - 1) / kRcB; kb >= 0; --kb) {
        const int k0 = kb * kRcB, w = min(kRcB, n - k0);
        const cplx* Ui = Di + size_t(kb) * 2 * kRcB * kRcB + size_t(kRcB) * kRcB;  // inv(U_kk), ld 64
        double ar = 0, ai = 0;
        if (row < w)
            for (int j = part; j < w; j += 8) {
                const cplx u = Ui[size_t(j) * kRcB + row], b = x[k0 + j];
                ar += u.re * b.re - u.im * b.im;
                ai += u.re * b.im + u.im * b.re;
            }
        for (int o = 4; o > 0; o >>= 1) {
            ar += __shfl_xor_sync(0xffffffffu, ar, o);
            ai += __shfl_xor_sync(0xffffffffu, ai, o);
        }
        __syncthreads();
        if (part == 0 && row < w) x[k0 + row] = cplx{ar, ai};
        __syncthreads();
        // x[0:k0] -= U[0:k0, k0:k0+w] x[k0:k0+w]: 128-row chunks x 4 column quarters,
        // 16 independent loads in flight per thread (w < 64 only for the
        // bottom tile when 64 does not divide n)
        {
            const int r = tid & 127, q = tid >> 7;  // row in chunk, column quarter (16 columns)
            for (int i0 = 0; i0 < k0; i0 += 128) {
                const int i = i0 + r;
                double br = 0, bi = 0;
                if (i < k0) {
                    cplx u[16];
#pragma unroll
                    for (int c = 0; c < 16; ++c)
                        u[c] = (16 * q + c < w) ? U[size_t(k0 + 16 * q + c) * ld + i] : cplx{0, 0};
#pragma unroll
                    for (int c = 0; c < 16; ++c) {
                        const cplx xc = (16 * q + c < w) ? x[k0 + 16 * q + c] : cplx{0, 0};
                        br += u[c].re * xc.re - u[c].im * xc.im;
                        bi += u[c].re * xc.im + u[c].im * xc.re;
                    }
                }
                t[q * 128 + r] = cplx{br, bi};
                __syncthreads();
                if (q == 0 && i < k0) {
                    const cplx a = t[r], b = t[128 + r], c2 = t[256 + r], d = t[384 + r];
                    x[i].re -= a.re + b.re + c2.re + d.re;
                    x[i].im -= a.im + b.im + c2.im + d.im;
                }
                __syncthreads();
            }
        }
    }
}

// x <- U^{-H} x (forward over 64-row tiles)
__device__ void rc_solve_uh(const cplx* __restrict__ U, const cplx* __restrict__ Di, int n, int ld, cplx* x) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int row = tid >> 3, part = tid & 7;
    for (int k0 = 0, kb = 0; k0 < n; k0 += kRcB, ++kb) {
        const int w = min(kRcB, n - k0);
        {  // x[k0 + c] -= U[0:k0, k0 + c]^H x[0:k0]: warp w owns columns w, w + 16, w + 32, w + 48
            double ar[4] = {0, 0, 0, 0}, ai[4] = {0, 0, 0, 0};
            for (int i = lane; i < k0; i += 32) {
                const cplx xi = x[i];
                cplx u[4];
#pragma unroll
                for (int m = 0; m < 4; ++m)
                    u[m] = (warp + 16 * m < w) ? U[size_t(k0 + warp + 16 * m) * ld + i] : cplx{0, 0};
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    ar[m] += u[m].re * xi.re + u[m].im * xi.im;
                    ai[m] += u[m].re * xi.im - u[m].im * xi.re;
                }
            }
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                for (int o = 16; o > 0; o >>= 1) {
                    ar[m] += __shfl_xor_sync(0xffffffffu, ar[m], o);
                    ai[m] += __shfl_xor_sync(0xffffffffu, ai[m], o);
                }
                if (lane == 0 && warp + 16 * m < w) {
                    x[k0 + warp + 16 * m].re -= ar[m];
                    x[k0 + warp + 16 * m].im -= ai[m];
                }
            }
        }
        __syncthreads();
        // x_blk = inv(U_kk)^H x_blk: output `row` is column `row` of the inverse tile, conjugated
        const cplx* Ui = Di + size_t(kb) * 2 * kRcB * kRcB + size_t(kRcB) * kRcB;
        double ar = 0, ai = 0;
        if (row < w)
            for (int j = part; j < w; j += 8) {
                const cplx u = Ui[size_t(row) * kRcB + j], b = x[k0 + j];
                ar += u.re * b.re + u.im * b.im;
                ai += u.re * b.im - u.im * b.re;
            }
        for (int o = 4; o > 0; o >>= 1) {
            ar += __shfl_xor_sync(0xffffffffu, ar, o);
            ai += __shfl_xor_sync(0xffffffffu, ai, o);
        }
        __syncthreads();
        if (part == 0 && row < w) x[k0 + row] = cplx{ar, ai};
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kRcT) lu_rcond_kernel(int n, int ld, int count, const cplx* const* __restrict__ Ap,
                                                        const cplx* __restrict__ base, size_t stride,
                                                        const cplx* const* __restrict__ Dp,
                                                        const cplx* __restrict__ dbase, size_t dstride, double th,
                                                        int* __restrict__ flag, double* __restrict__ rcond,
                                                        double* __restrict__ est_out) {
    extern __shared__ cplx rc_sm[];
    cplx* x = rc_sm;         // n
    cplx* t = rc_sm + n;     // 512 partial sums of the block GEMV
    __shared__ double red[kRcT / 32];
    __shared__ int redi[kRcT / 32];
    __shared__ int s_zero;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int blk = blockIdx.x; blk < count; blk += gridDim.x) {
        const cplx* U = Ap ? Ap[blk] : base + size_t(blk) * stride;
        const cplx* Di = Dp ? Dp[blk] : dbase + size_t(blk) * dstride;
        // ||U||_1 (max column sum of the upper triangle) and exact zero pivots
        __syncthreads();
        if (tid == 0) s_zero = 0;
        __syncthreads();
        double cmax = 0;
        for (int j = warp; j < n; j += kRcT / 32) {
            double sum = 0;
#pragma unroll 4
            for (int i = lane; i <= j; i += 32) {
                const cplx u = U[size_t(j) * ld + i];
                sum += sqrt(u.re * u.re + u.im * u.im);
            }
            for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
            cmax = fmax(cmax, sum);
            if (lane == 0) {
                const cplx d = U[size_t(j) * ld + j];
                if (d.re == 0.0 && d.im == 0.0) s_zero = 1;
            }
        }
        if (lane == 0) red[warp] = cmax;
        __syncthreads();
        double anorm = 0;
        for (int w = 0; w < kRcT / 32; ++w) anorm = fmax(anorm, red[w]);
        double rc = 0.0;
        if (!s_zero && anorm > 0.0 && isfinite(anorm)) {
            auto sum_abs = [&]() {
                double a = 0;
                for (int i = tid; i < n; i += kRcT) a += sqrt(x[i].re * x[i].re + x[i].im * x[i].im);
                return rc_block_sum(a, red);
            };
            // zlacn2: x = e / n; y = U^{-1} x
            __syncthreads();
            for (int i = tid; i < n; i += kRcT) x[i] = cplx{1.0 / n, 0.0};
            __syncthreads();
            rc_solve_u(U, Di, n, ld, x, t);
            double est = sum_abs();
            if (n > 1) {
                for (int i = tid; i < n; i += kRcT) x[i] = csign(x[i]);
                __syncthreads();
                rc_solve_uh(U, Di, n, ld, x);
                int j = rc_block_argmax(x, n, red, redi);
                for (int iter = 2;; ++iter) {
                    __syncthreads();
                    for (int i = tid; i < n; i += kRcT) x[i] = cplx{i == j ? 1.0 : 0.0, 0.0};
                    __syncthreads();
                    rc_solve_u(U, Di, n, ld, x, t);
                    const double estold = est;
                    est = sum_abs();
                    if (!(est > estold)) { est = fmax(est, estold); break; }
                    __syncthreads();
                    for (int i = tid; i < n; i += kRcT) x[i] = csign(x[i]);
                    __syncthreads();
                    rc_solve_uh(U, Di, n, ld, x);
                    const int jlast = j;
                    const double xl = sqrt(x[jlast].re * x[jlast].re + x[jlast].im * x[jlast].im);
                    j = rc_block_argmax(x, n, red, redi);
                    const double xj = sqrt(x[j].re * x[j].re + x[j].im * x[j].im);
                    if (!(xl != xj && iter < 5)) break;
                }
                // alternating-sign test vector x_i = (-1)^i (1 + i / (n - 1))
                __syncthreads();
                for (int i = tid; i < n; i += kRcT)
                    x[i] = cplx{((i & 1) ? -1.0 : 1.0) * (1.0 + double(i) / (n - 1)), 0.0};
                __syncthreads();
                rc_solve_u(U, Di, n, ld, x, t);
                const double temp = 2.0 * sum_abs() / (3.0 * n);
                est = fmax(est, temp);
            }
            rc = (est > 0.0 && isfinite(est)) ? (1.0 / anorm) / est : 0.0;
            if (tid == 0 && est_out) est_out[blk] = est;
        } else if (tid == 0 && est_out) {
            est_out[blk] = INFINITY;
        }
        if (tid == 0) {
            if (rcond) rcond[blk] = rc;
            if (!(rc > th)) flag[blk] = 1;
        }
    }
}

// ||A_b||_1 of each n x n block (max column sum of moduli), as the IEEE bits of a
// non-negative double (their integer order is the numeric order: atomicMax)
__global__ void __launch_bounds__(256) colsum_max_kernel(const cplx* __restrict__ A, int n, int ld, size_t stride,
                                                         unsigned long long* __restrict__ out) {
    const cplx* Ab = A + size_t(blockIdx.x) * stride;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double m = 0;
    for (int j = blockIdx.y * 8 + warp; j < n; j += gridDim.y * 8) {
        double sum = 0;
#pragma unroll 4
        for (int i = lane; i < n; i += 32) {
            const cplx u = Ab[size_t(j) * ld + i];
            sum += sqrt(u.re * u.re + u.im * u.im);
        }
        for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        m = fmax(m, sum);
    }
    if (lane == 0 && m > 0.0) atomicMax(out + blockIdx.x, (unsigned long long)__double_as_longlong(m));
}

// Screen of the Woodbury level-0 factors: est_lo = max_k ||A^{-1} r_k||_1 /
// ||r_k||_1 over the probe columns solved with the level-0 right-hand sides is
// a lower bound of ||A^{-1}||_1, so rc_up = 1 / (||A||_1 est_lo) bounds rcond
// from above: rc_up <= th_def certifies rcond <= th_def; rc_up <= th_sus marks
// the block for the full zlacn2 estimate.
__global__ void __launch_bounds__(256) rc_screen_kernel(const cplx* __restrict__ W, size_t wstride, int n, int col0,
                                                        int nprobe, const unsigned long long* __restrict__ anorm,
                                                        double rnorm1, double th_def, double th_sus,
                                                        int* __restrict__ flag, int* __restrict__ sus,
                                                        double* __restrict__ est_lo) {
    __shared__ double red[8];
    const cplx* Wb = W + size_t(blockIdx.x) * wstride;
    double best = 0;
    for (int k = 0; k < nprobe; ++k) {
        double a = 0;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const cplx v = Wb[size_t(col0 + k) * n + i];
            a += sqrt(v.re * v.re + v.im * v.im);
        }
        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        __syncthreads();
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
        __syncthreads();
        double t = 0;
        for (int w = 0; w < int(blockDim.x >> 5); ++w) t += red[w];
        best = isfinite(t) ? fmax(best, t / rnorm1) : INFINITY;
    }
    if (threadIdx.x == 0) {
        const double an = __longlong_as_double((long long)anorm[blockIdx.x]);
        const double rc = 1.0 / (an * best);
        est_lo[blockIdx.x] = best;
        if (!(rc > th_def)) flag[blockIdx.x] = 1;
        sus[blockIdx.x] = !(rc > th_sus);
    }
}

__global__ void gather_columns_kernel(const cplx* const* __restrict__ src, const int* __restrict__ ld, int rows,
                                      const int* __restrict__ cols, int ncols, cplx* __restrict__ dst, int ldd,
                                      size_t dstride) {
    const int q = blockIdx.x, k = blockIdx.y;
    const cplx* a = src[q] + size_t(cols[size_t(q) * ncols + k]) * ld[q];
    cplx* d = dst + size_t(q) * dstride + size_t(k) * ldd;
    for (int i = threadIdx.x; i < rows; i += blockDim.x) d[i] = a[i];
}

__global__ void dfma_peak_kernel(double* out, int iters) {
    double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6,
           a7 = a0 + 7;
    const double b = 0.999999, c = 1e-7;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
            a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
        }
    }
    const double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (s == 12345.678) out[0] = s;
}

__global__ void dmma_peak_kernel(double* out, int iters) {
    double c[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
    const double a = 1e-3 * (threadIdx.x & 7), b = 1e-3 * (threadIdx.x >> 3);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) dmma(c[i][0], c[i][1], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.678) out[0] = s;
}

}  // namespace

namespace {
bool thin48_off() {  // QPS_ZGEMM_THIN48=0: 16-row tiles for 48-row products (A/B)
    static const bool off = [] {
        const char* e = getenv("QPS_ZGEMM_THIN48");
        return e && !strcmp(e, "0");
    }();
    return off;
}
}  // namespace

constexpr int kThinN = 8;  // products with N <= 8 use the 128 x 8 tile

// QPS_ZGEMM_WIDE=1: the 64 x 32 tile for large K and outputs (the round-1 rule, A/B)
bool wide_tiles() {
    static const bool on = [] {
        const char* e = getenv("QPS_ZGEMM_WIDE");
        return e && !strcmp(e, "1");
    }();
    return on;
}

void zgemm_batched(int M, int N, cplx alpha, cplx beta, const std::vector<GemmTask>& tasks, cudaStream_t s,
                   DBuf<GemmTask>& d_tasks, const char* family) {
    if (tasks.empty() || M <= 0 || N <= 0) return;
    d_tasks.upload(tasks, s);
    // default: 3M, CTA 64 x 32 (4 warps of 32 x 16), two stages, three CTAs per
    // SM (38 TF/s complex-equivalent at 608^3 on B200 = 77 % of the DMMA pipe);
    // QPS_ZGEMM=4m selects the four-DMMA kernel (28 TF/s)
    static const bool four_m = [] {
        const char* e = getenv("QPS_ZGEMM");
        return e && !strcmp(e, "4m");
    }();
    // flops recorded = real flops issued to the tensor pipe (6 M N K for 3M)
    const double fpc = four_m ? 8.0 : 6.0;
    double fl = 0, by = 0;
    for (const auto& t : tasks)
        for (int q = 0; q < t.nseg; ++q) {
            fl += fpc * M * N * t.K[q];
            by += 16.0 * (double(M) * t.K[q] + double(t.K[q]) * N);
        }
    by += 16.0 * double(M) * N * tasks.size() * ((beta.re != 0.0 || beta.im != 0.0) ? 2 : 1);
    int kmax = 0;
    for (const auto& t : tasks)
        for (int q = 0; q < t.nseg; ++q) kmax = std::max(kmax, t.K[q]);
    const char* nm = family ? family : (kmax <= 64) ? (M <= 64 ? "zgemm_k64_m64" : "zgemm_k64") : (M >= 256 && N >= 256 ? "zgemm_big" : "zgemm_mid");
    static const bool trace_shapes = getenv("QPS_TRACE_GEMM") != nullptr;  // shapes to stderr (profiling aid)
    if (trace_shapes)
        fprintf(stderr, "gemm %s M=%d N=%d K=%d nseg=%d tasks=%zu\n", nm, M, N, kmax, tasks[0].nseg, tasks.size());
    ProfScope ps(nm, s, fl, by, 0.0, int((tasks.size() + 65534) / 65535));
    if (!four_m) {
        // tile by shape (tools/micro/gemm_cfg.cu, gemm_cfg2.cu on B200): 16 x 64
        // for thin products (M <= 48, or M <= 80 against a wide N), 32 x 32
        // otherwise
        // in-place products (C aliasing B, M <= 64: the triangular-tile solves)
        // need every row of a column tile in one CTA -- the 64-row tile
        const bool inplace = tasks[0].C == tasks[0].B[0];
        static const bool fixed_tile = [] {  // QPS_ZGEMM_TILE=fixed: the 64 x 32 tile for every shape (debug)
            const char* e = getenv("QPS_ZGEMM_TILE");
            return e && !strcmp(e, "fixed");
        }();
        if (N <= kThinN && !fixed_tile) {
            // narrow right-hand-side groups: 128 x 8 tiles (one N tile; in place
            // too, every row of a column tile stays in one CTA)
            if (inplace && M > 128) fail(QPS_ERR_INTERNAL, "zgemm_batched: in-place product taller than one tile");
            launch_z3<4, 1, 4, 1, 2, 3>(M, N, alpha, beta, d_tasks.p, tasks.size(), s);
        } else if (inplace || fixed_tile) {
            if (inplace && M > 64) {
                fprintf(stderr, "zgemm_batched: in-place M=%d N=%d K=%d ntasks=%zu nseg=%d\n", M, N, tasks[0].K[0],
                        tasks.size(), tasks[0].nseg);
                fail(QPS_ERR_INTERNAL, "zgemm_batched: in-place product taller than one tile");
            }
            launch_z3<4, 2, 2, 2, 2, 3>(M, N, alpha, beta, d_tasks.p, tasks.size(), s);
        } else if (M > 32 && M <= 48 && N >= 256 && kmax >= 256 && !thin48_off())
            // the whole 48-row product in one CTA row: the wide operand is
            // streamed once instead of once per 16-row tile
            launch_z3<6, 2, 1, 4, 2, 2>(M, N, alpha, beta, d_tasks.p, tasks.size(), s);
        else if (M <= 48 || (M > 64 && M <= 80 && N >= 256))
            launch_z3<2, 2, 1, 4, 2, 4>(M, N, alpha, beta, d_tasks.p, tasks.size(), s);
        else if (M <= 64 && N >= 256)
            // 64-row products against a wide N: one 64 x 32 tile row (LU U12
            // updates: 24.8 vs 18.3 TF/s for the 16 x 64 tile at 64 x 288 x 64;
            // the 80-row Schur products stay on 16 x 64)
            launch_z3<4, 2, 2, 2, 2, 3>(M, N, alpha, beta, d_tasks.p, tasks.size(), s);
        else if (kmax <= 96 || (M <= 128 && N <= 128) || !wide_tiles())
            // 32 x 32 (4 CTAs per SM): with every task's operands in HBM it
            // beats the 64 x 32 tile on every hot-path shape (tools/micro/
            // gemm_cfg2.cu: 288^2 x 320 LU update 5.56 vs 5.94 ms, 608^2 x 160
            // Schur update 12.85 vs 13.17 ms, 74-79 % of the DMMA peak)
            launch_z3<2, 2, 2, 2, 2, 4>(M, N, alpha, beta, d_tasks.p, tasks.size(), s);
        else
            launch_z3<4, 2, 2, 2, 2, 3>(M, N, alpha, beta, d_tasks.p, tasks.size(), s);
    } else {
        const int tiles_m = (M + BM - 1) / BM, tiles_n = (N + BN - 1) / BN;
        for (size_t off = 0; off < tasks.size(); off += 65535) {
            const unsigned cnt = unsigned(std::min<size_t>(65535, tasks.size() - off));
            { QPS_NOTE_LAUNCH(); zgemm_kernel<<<dim3(tiles_m * tiles_n, cnt), 128, 0, s>>>(M, N, alpha, beta, d_tasks.p + off, tiles_m); }
        }
    }
    QPS_CUDA(cudaGetLastError());
}

void zgemm_residual_norms(int M, int N, cplx alpha, cplx beta, const std::vector<GemmTask>& tasks, cudaStream_t s,
                          DBuf<GemmTask>& d_tasks, DBuf<double>& parts, double* norms) {
    if (tasks.empty() || M <= 0 || N <= 0) return;
    d_tasks.upload(tasks, s);
    int kmax = 0;
    double fl = 0;
    for (const auto& t : tasks)
        for (int q = 0; q < t.nseg; ++q) {
            kmax = std::max(kmax, t.K[q]);
            fl += 6.0 * M * N * t.K[q];
        }
    ProfScope ps("zgemm_resid", s, fl, 16.0 * double(M) * N * tasks.size());
    // same tiles as zgemm_batched's rule (the residual shapes: M = m rows of Q)
    if (kmax <= 96 || (M <= 128 && N <= 128))
        launch_z3<2, 2, 2, 2, 2, 4, true>(M, N, alpha, beta, d_tasks.p, tasks.size(), s, &parts, norms);
    else
        launch_z3<4, 2, 2, 2, 2, 3, true>(M, N, alpha, beta, d_tasks.p, tasks.size(), s, &parts, norms);
    QPS_CUDA(cudaGetLastError());
}

constexpr size_t kCodFacSmemMax = 216 * 1024;
// Dynamic shared memory a launch of only a few latency-bound CTAs requests so
// that no throughput kernel's CTA can share its SM (co-resident GEMM CTAs
// were measured to slow the corner least squares 2-3x).
constexpr size_t kLatencyReserve = 200 * 1024;
size_t latency_reserve(int ctas) { return ctas <= 16 ? kLatencyReserve : 0; }

template <bool kFast>
void launch_cod_factor(const CodBatch& b, cudaStream_t s) {
    const size_t sm = size_t(b.m) * b.p * sizeof(cplx);
    if (sm <= kCodFacSmemMax) {
        static bool attr = false;
        if (!attr) {
            QPS_CUDA(cudaFuncSetAttribute(cod_factor_kernel<kFast, true>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, int(kCodFacSmemMax)));
            attr = true;
        }
        { QPS_NOTE_LAUNCH(); cod_factor_kernel<kFast, true><<<b.count, 512, sm, s>>>(b); }
    } else {
        const size_t res = latency_reserve(b.count);
        static bool attr = false;
        if (!attr) {
            QPS_CUDA(cudaFuncSetAttribute(cod_factor_kernel<kFast, false>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, int(kLatencyReserve)));
            attr = true;
        }
        { QPS_NOTE_LAUNCH(); cod_factor_kernel<kFast, false><<<b.count, 256, res, s>>>(b); }
    }
    QPS_CUDA(cudaGetLastError());
}

void cod_factor(const CodBatch& b, cudaStream_t s) {
    if (b.count == 0) return;
    if (b.p > kMaxP) fail(QPS_ERR_CONFIG, "qsolve: too many columns for the device COD (max 256)");
    if (b.m < b.p) fail(QPS_ERR_USAGE, "qsolve: Q must have at least as many rows as columns");
    ProfScope ps("cod_factor", s, 8.0 * b.count * (2.0 * b.m * b.p * b.p - 2.0 * b.p * b.p * b.p / 3.0));
    launch_cod_factor<false>(b, s);
}
void cod_factor_fast(const CodBatch& b, cudaStream_t s) {
    if (b.count == 0) return;
    if (b.p > kMaxP || b.m < b.p) fail(QPS_ERR_INTERNAL, "cod_factor_fast: bad shape");
    ProfScope ps("lr_cpqr", s, 8.0 * b.count * (2.0 * b.m * b.p * b.p - 2.0 * b.p * b.p * b.p / 3.0));
    launch_cod_factor<true>(b, s);
}
void cod_rank(const CodBatch& b, double th, const int* flags, cudaStream_t s) {
    if (b.count == 0) return;
    ProfScope ps("cod_rank", s, 0.0);
    { QPS_NOTE_LAUNCH(); cod_rank_kernel<<<(b.count + 127) / 128, 128, 0, s>>>(b, th, flags); }
    QPS_CUDA(cudaGetLastError());
}
void cod_operator(const CodBatch& b, const int* flags, cudaStream_t s) {
    if (b.count == 0) return;
    ProfScope ps("cod_operator", s, 8.0 * b.count * (double(b.m) * b.p * b.p + double(b.p) * b.p * b.p));
    const size_t sm = (size_t(b.m) * b.p + std::max(size_t(b.p) * b.p, size_t(32) * b.m)) * sizeof(cplx);
    if (sm <= kCodSmemMax) {
        static bool attr = false;
        if (!attr) {
            QPS_CUDA(cudaFuncSetAttribute(cod_operator_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(kCodSmemMax)));
            attr = true;
        }
        { QPS_NOTE_LAUNCH(); cod_operator_smem_kernel<<<b.count, 256, sm, s>>>(b, flags); }
    } else {
        // few large problems (the corners): latency-bound single CTAs that keep
        // their SM to themselves (the reservation keeps GEMM CTAs off it)
        const size_t res = latency_reserve(b.count);
        static bool attr = false;
        if (!attr) {
            QPS_CUDA(cudaFuncSetAttribute(cod_operator_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(kLatencyReserve)));
            QPS_CUDA(cudaFuncSetAttribute(cod_qh_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(kLatencyReserve)));
            attr = true;
        }
        { QPS_NOTE_LAUNCH(); cod_operator_kernel<<<b.count, 256, res, s>>>(b, flags); }
        QPS_CUDA(cudaGetLastError());
        const size_t qs = std::max(size_t(8) * b.m * sizeof(cplx), res);
        if (qs > kLatencyReserve) fail(QPS_ERR_INTERNAL, "cod_qh: m too large");
        { QPS_NOTE_LAUNCH(); cod_qh_kernel<<<dim3((b.m + 7) / 8, b.count), 256, qs, s>>>(b, flags); }
    }
    QPS_CUDA(cudaGetLastError());
}
void cod_trsm(const CodBatch& b, cplx* B, int ldb, size_t stride, int ncols, const int* flags, cudaStream_t s) {
    if (b.count == 0 || ncols == 0) return;
    ProfScope ps("cod_trsm", s, 4.0 * b.count * double(b.p) * b.p * ncols);
    const size_t sh = size_t(b.p) * b.p * sizeof(cplx);
    const dim3 grid((ncols + 127) / 128, b.count);
    const size_t shc = (size_t(b.p) * b.p + size_t(b.p) * kTrsmCols + b.p) * sizeof(cplx);
    const size_t shb = (size_t(b.p) * (b.p + 1) / 2 + size_t(b.p + 1) * kTrsmBlkCols + b.p) * sizeof(cplx);
    static const char* mode = getenv("QPS_COD_TRSM");  // row: row-by-row kernel; blk: one-kernel blocked (A/B)
    const bool unblocked = mode && !strcmp(mode, "row");
    const bool onekernel = mode && !strcmp(mode, "blk");
    if (!unblocked && !onekernel && b.trsm_tasks && b.count >= 64) {
        // many problems: left-looking 16-row blocks, GEMMs on the DMMA pipe
        const int nst = (b.p + 15) / 16;
        { QPS_NOTE_LAUNCH(); cod_trsm_tasks_kernel<<<(b.count + 127) / 128, 128, 0, s>>>(b, B, ldb, stride, flags, nst); }
        QPS_CUDA(cudaGetLastError());
        for (int st = 0; st < nst; ++st) {
            if (st > 0) {
                static const bool trace_shapes = getenv("QPS_TRACE_GEMM") != nullptr;
                if (trace_shapes)
                    fprintf(stderr, "gemm cod_trsm M=16 N=%d K=%d nseg=1 tasks=%d\n", ncols, 16 * st, b.count);
                launch_z3<2, 2, 1, 4, 2, 4>(16, ncols, cplx{-1, 0}, cplx{1, 0}, b.trsm_tasks + size_t(st) * b.count,
                                           b.count, s);
            }
            { QPS_NOTE_LAUNCH(); cod_trsm_diag_kernel<<<dim3((ncols + 127) / 128, b.count), 128, 0, s>>>(
                b, B, ldb, stride, ncols, flags, st); }
            QPS_CUDA(cudaGetLastError());
        }
    } else if (!unblocked && shb <= 110 * 1024) {
        static bool attr = false;
        if (!attr) {
            QPS_CUDA(cudaFuncSetAttribute(cod_trsm_blk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(110 * 1024)));
            attr = true;
        }
        { QPS_NOTE_LAUNCH(); cod_trsm_blk_kernel<<<dim3((ncols + kTrsmBlkCols - 1) / kTrsmBlkCols, b.count), 256, shb, s>>>(
            b, B, ldb, stride, ncols, flags); }
    } else if (shc <= 200 * 1024) {
        static bool attr = false;
        if (!attr) {
            QPS_CUDA(cudaFuncSetAttribute(cod_trsm_chunk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(200 * 1024)));
            attr = true;
        }
        { QPS_NOTE_LAUNCH(); cod_trsm_chunk_kernel<<<dim3((ncols + kTrsmCols - 1) / kTrsmCols, b.count), 256, shc, s>>>(b, B, ldb, stride,
                                                                                                   ncols, flags); }
    } else if (sh <= 160 * 1024) {
        static size_t attr = 0;
        if (sh > attr) {
            QPS_CUDA(cudaFuncSetAttribute(cod_trsm_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(160 * 1024)));
            attr = 160 * 1024;
        }
        { QPS_NOTE_LAUNCH(); cod_trsm_kernel<true><<<grid, 128, sh, s>>>(b, B, ldb, stride, ncols, flags); }
    } else {
        const size_t res = latency_reserve(int(grid.x * grid.y));
        static bool attr = false;
        if (!attr) {
            QPS_CUDA(cudaFuncSetAttribute(cod_trsm_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(kLatencyReserve)));
            attr = true;
        }
        { QPS_NOTE_LAUNCH(); cod_trsm_kernel<false><<<grid, 128, res, s>>>(b, B, ldb, stride, ncols, flags); }
    }
    QPS_CUDA(cudaGetLastError());
}


size_t lu_dinv_elems(int n) { return size_t(2) * ((n + kTB - 1) / kTB) * kTB * kTB; }

namespace {
void launch_tri_inv(int n, int ld, cplx* const* dA, cplx* const* dO, int count, int bs, int k0_first, int nblk,
                    int mode, cudaStream_t s, int tile0 = 0) {
    // bs: a multiple of 16, <= kTB
    // layout: T | X (lower) | X (upper) | Y | Y | Dinv (mode 3 uses both halves)
    const size_t sh = (3 * size_t(bs) * (bs + 1) + 2 * 768 + bs) * sizeof(cplx);
    static bool attr = false;
    if (!attr) {
        QPS_CUDA(cudaFuncSetAttribute(tri_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int((3 * kTB * (kTB + 1) + 2 * 768 + kTB) * sizeof(cplx))));
        attr = true;
    }
    ProfScope ps("tri_inv", s, 8.0 / 3.0 * count * nblk * double(bs) * bs * bs * ((mode == 3) ? 2 : 1));
    { QPS_NOTE_LAUNCH(); tri_inv_kernel<<<dim3(nblk, count), mode == 3 ? 512 : 256, sh, s>>>(n, ld, dA, dO, bs, k0_first, mode,
                                                                                                tile0); }
    QPS_CUDA(cudaGetLastError());
}
}  // namespace

namespace {

// 16-column panel factorization of <= 640 rows (one thread per row)
void launch_panel_fast(int n, int ld, cplx* const* dA, int* const* dP, int c0, int w, int* sing, int* rl_map,
                       int count, cudaStream_t s) {
    const int threads = ((n - c0 + 31) / 32) * 32;
    static bool attr = false;
    if (!attr) {
        QPS_CUDA(cudaFuncSetAttribute(lu_panel_sm2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(size_t(kRegPanelMaxRows) * kRlW * sizeof(cplx))));
        attr = true;
    }
    { QPS_NOTE_LAUNCH(); lu_panel_sm2_kernel<<<count, threads, size_t(n - c0) * w * sizeof(cplx), s>>>(n, ld, dA, dP, c0, w, sing,
                                                                                  rl_map); }
}

void launch_row_permute(int n, int ld, cplx* const* dA, const int* const* dP, int count, int k0, int kend, int c0,
                        int c1, cudaStream_t s, DBuf<int>& perm) {
    if (c1 <= c0) return;
    perm.ensure(size_t(count) * (2 * n + 1));
    { QPS_NOTE_LAUNCH(); perm_build_kernel<<<count, 128, 0, s>>>(n, dP, perm.p, k0, kend); }
    QPS_CUDA(cudaGetLastError());
    const size_t sh = size_t(kPermWarps) * (n - k0) * sizeof(cplx);
    static size_t attr = 0;
    if (sh > attr) {
        QPS_CUDA(cudaFuncSetAttribute(row_permute_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(std::max<size_t>(sh, 64 * 1024))));
        attr = std::max<size_t>(sh, 64 * 1024);
    }
    const int nx = std::min((c1 - c0 + kPermWarps - 1) / kPermWarps, 32);
    { QPS_NOTE_LAUNCH(); row_permute_kernel<<<dim3(nx, count), 256, sh, s>>>(n, ld, dA, perm.p, k0, c0, c1); }
    QPS_CUDA(cudaGetLastError());
}

struct LuCtx {
    int n, ld, count;
    const std::vector<cplx*>& hA;
    const std::vector<int*>& hP;
    const std::vector<cplx*>& hD;
    cplx* const* dA;
    int* const* dP;
    cplx* const* dD;
    int* sing;
    cudaStream_t s;
    Workspace& ws;
    // right-hand sides carried along the recursion's spine (lu_factor_solve_batched)
    const std::vector<cplx*>* hB = nullptr;
    cplx* const* dB = nullptr;
    int ldb = 0, nrhs = 0;
};

void gemm_update(LuCtx& L, int M, int N, int K, size_t aoff, size_t boff, size_t coff, cplx alpha, cplx beta,
                 const std::vector<cplx*>& Abase, const std::vector<cplx*>& Bbase, int ldb) {
    auto& tasks = L.ws.h_gemm;
    tasks.assign(L.count, GemmTask{});
    for (int b = 0; b < L.count; ++b) {
        GemmTask& t = tasks[b];
        t.nseg = 1;
        t.A[0] = Abase[b] + aoff;
        t.lda[0] = L.ld;
        t.B[0] = Bbase[b] + boff;
        t.ldb[0] = ldb;
        t.K[0] = K;
        t.C = Bbase[b] + coff;
        t.ldc = ldb;
    }
    zgemm_batched(M, N, alpha, beta, tasks, L.s, L.ws.gemm_tasks, "lu_gemm");
}

// leaf width of the recursion: 64-column panels in one CTA (lu_wpanel_kernel)
// for matrices of <= 640 rows (QPS_LU_WIDE=0: 16-column shared-memory panels)
bool wide_leaf(int n) {
    static const bool off = [] {
        const char* e = getenv("QPS_LU_WIDE");
        return e && !strcmp(e, "0");
    }();
    return !off && n <= kWpThreads;
}
int lu_leaf(int n) {
    if (wide_leaf(n)) return kWpMax;
    return size_t(n) * kLeaf * sizeof(cplx) <= 200 * 1024 ? kLeaf : kNB;
}

// X[r0:r1, c0:c0+nc] <- L[r0:r1, r0:r1]^{-1} X (unit lower) inside the factor itself
// (U12 of the recursive LU), leaves of <= 64 rows through on-demand tile inverses.
void trsm_lower_rhs_leaf(LuCtx& L, int r0, int r1, int bs, size_t toff);
void trsm_lower_rhs_update(LuCtx& L, int r0, int h, int r1);

// rhs: apply the same L^{-1} to the carried right-hand sides (one tile inverse
// per leaf serves both)
void trsm_lower_in_factor(LuCtx& L, int r0, int r1, int c0, int nc, bool rhs = false) {
    const int m = r1 - r0;
    if (m <= kTB) {
        // wide leaves: the tile's own inverse (r0 is 64-aligned); otherwise a
        // tile sized to the leaf (16, 32, 48 or 64 rows) in tile 0 as scratch
        const bool own_tile = wide_leaf(L.n);
        const int bs = own_tile ? kTB : (m + 15) / 16 * 16;
        const size_t toff = own_tile ? size_t(r0 / kTB) * 2 * kTB * kTB : 0;
        if (!own_tile) launch_tri_inv(L.n, L.ld, L.dA, L.dD, L.count, bs, r0, 1, 1, L.s);
        if (rhs) trsm_lower_rhs_leaf(L, r0, r1, bs, toff);
        auto& tasks = L.ws.h_gemm;
        tasks.assign(L.count, GemmTask{});
        for (int b = 0; b < L.count; ++b) {
            GemmTask& t = tasks[b];
            t.nseg = 1;
            t.A[0] = L.hD[b] + toff;
            t.lda[0] = bs;
            t.B[0] = L.hA[b] + size_t(c0) * L.ld + r0;
            t.ldb[0] = L.ld;
            t.K[0] = m;
            t.C = L.hA[b] + size_t(c0) * L.ld + r0;  // in place: <= 64 rows, one CTA per column tile
            t.ldc = L.ld;
        }
        zgemm_batched(m, nc, cplx{1, 0}, cplx{0, 0}, tasks, L.s, L.ws.gemm_tasks, "lu_gemm");
        return;
    }
    const int h = ((m + kTB - 1) / kTB + 1) / 2 * kTB;
    trsm_lower_in_factor(L, r0, r0 + h, c0, nc, rhs);
    // X[r0+h:r1] -= L[r0+h:r1, r0:r0+h] X[r0:r0+h]
    gemm_update(L, m - h, nc, h, size_t(r0) * L.ld + r0 + h, size_t(c0) * L.ld + r0, size_t(c0) * L.ld + r0 + h,
                cplx{-1, 0}, cplx{1, 0}, L.hA, L.hA, L.ld);
    if (rhs) trsm_lower_rhs_update(L, r0, h, r1);
    trsm_lower_in_factor(L, r0 + h, r1, c0, nc, rhs);
}

// recursive LU of columns [c0, c0 + nc) (rows c0..n), Toledo's algorithm
void lu_rec(LuCtx& L, int c0, int nc) {
    const size_t psm = size_t(L.n - c0) * kLeaf * sizeof(cplx);
    const bool smem_leaf = size_t(L.n) * kLeaf * sizeof(cplx) <= 200 * 1024;
    const int leaf = lu_leaf(L.n);
    if (nc <= leaf) {
        ProfScope ps("lu_panel", L.s, 8.0 * L.count * double(L.n - c0) * nc * nc / 2.0);
        if (wide_leaf(L.n)) {
            const int threads = ((L.n - c0 + 31) / 32) * 32;
            static const bool staged = [] {  // QPS_WP_STAGED=0: register double-buffered update (A/B)
                const char* e = getenv("QPS_WP_STAGED");
                return !(e && !strcmp(e, "0"));
            }();
            if (staged) {
                static bool attr = false;
                if (!attr) {
                    QPS_CUDA(cudaFuncSetAttribute(lu_wpanel_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  int(wpanel_smem(kWpThreads))));
                    attr = true;
                }
                { QPS_NOTE_LAUNCH(); lu_wpanel_kernel<true><<<L.count, threads, wpanel_smem(threads), L.s>>>(
                    L.n, L.ld, L.dA, L.dP, c0, nc, L.sing); }
            } else {
                { QPS_NOTE_LAUNCH(); lu_wpanel_kernel<false><<<L.count, threads, 0, L.s>>>(L.n, L.ld, L.dA, L.dP, c0, nc,
                                                                                       L.sing); }
            }
            QPS_CUDA(cudaGetLastError());
            // the leaf is a 64-aligned diagonal tile whose L and U are final:
            // invert both into its Dinv slot now (the trsm of U12 and the
            // level-0 solves read them; no final pass over all tiles)
            launch_tri_inv(L.n, L.ld, L.dA, L.dD, L.count, kTB, c0, 1, 3, L.s, c0 / kTB);
        } else if (nc <= kRlW && L.n - c0 <= kRegPanelMaxRows) {
            launch_panel_fast(L.n, L.ld, L.dA, L.dP, c0, nc, L.sing, nullptr, L.count, L.s);
        } else if (smem_leaf) {
            static bool attr = false;
            if (!attr) {
                QPS_CUDA(cudaFuncSetAttribute(lu_panel_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              200 * 1024));
                attr = true;
            }
            { QPS_NOTE_LAUNCH(); lu_panel_smem_kernel<<<L.count, 256, psm, L.s>>>(L.n, L.ld, L.dA, L.dP, c0, nc, L.sing); }
        } else {
            { QPS_NOTE_LAUNCH(); lu_panel_kernel<<<L.count, 256, 0, L.s>>>(L.n, L.ld, L.dA, L.dP, c0, L.sing); }
        }
        QPS_CUDA(cudaGetLastError());
        return;
    }
    const int h = ((nc + leaf - 1) / leaf) / 2 * leaf;
    lu_rec(L, c0, h);
    {  // left-half interchanges onto the right half
        ProfScope ps("lu_swap", L.s, 0.0);
        launch_row_permute(L.n, L.ld, L.dA, L.dP, L.count, c0, c0 + h, c0 + h, c0 + nc, L.s, L.ws.perm);
    }
    trsm_lower_in_factor(L, c0, c0 + h, c0 + h, nc - h);
    // A22 -= A21 A12 over rows c0+h..n, cols c0+h..c0+nc
    gemm_update(L, L.n - c0 - h, nc - h, h, size_t(c0) * L.ld + c0 + h, size_t(c0 + h) * L.ld + c0,
                size_t(c0 + h) * L.ld + c0 + h, cplx{-1, 0}, cplx{1, 0}, L.hA, L.hA, L.ld);
    lu_rec(L, c0 + h, nc - h);
    {  // right-half interchanges back onto the left half
        ProfScope ps("lu_swap", L.s, 0.0);
        launch_row_permute(L.n, L.ld, L.dA, L.dP, L.count, c0 + h, c0 + nc, c0, c0 + h, L.s, L.ws.perm);
    }
}

// B[r0:r1, :] <- L[r0:r1, r0:r1]^{-1} B[r0:r1, :] (unit lower, the factor's own
// L) for the carried right-hand sides; leaves of <= 64 rows through tile inverses
// B[r0:r1] <- (tile 0 of Dinv, bs x bs) B[r0:r1]: the leaf's L^{-1} already inverted
void trsm_lower_rhs_leaf(LuCtx& L, int r0, int r1, int bs, size_t toff) {
    const int m = r1 - r0;
    auto& tasks = L.ws.h_gemm;
    tasks.assign(L.count, GemmTask{});
    for (int b = 0; b < L.count; ++b) {
        GemmTask& t = tasks[b];
        t.nseg = 1;
        t.A[0] = L.hD[b] + toff;
        t.lda[0] = bs;
        t.B[0] = (*L.hB)[b] + r0;
        t.ldb[0] = L.ldb;
        t.K[0] = m;
        t.C = (*L.hB)[b] + r0;
        t.ldc = L.ldb;
    }
    zgemm_batched(m, L.nrhs, cplx{1, 0}, cplx{0, 0}, tasks, L.s, L.ws.gemm_tasks, "lu_gemm");
}
// B[r0+h:r1] -= L[r0+h:r1, r0:r0+h] B[r0:r0+h]
void trsm_lower_rhs_update(LuCtx& L, int r0, int h, int r1) {
    auto& tasks = L.ws.h_gemm;
    tasks.assign(L.count, GemmTask{});
    for (int b = 0; b < L.count; ++b) {
        GemmTask& t = tasks[b];
        t.nseg = 1;
        t.A[0] = L.hA[b] + size_t(r0) * L.ld + r0 + h;
        t.lda[0] = L.ld;
        t.B[0] = (*L.hB)[b] + r0;
        t.ldb[0] = L.ldb;
        t.K[0] = h;
        t.C = (*L.hB)[b] + r0 + h;
        t.ldc = L.ldb;
    }
    zgemm_batched(r1 - r0 - h, L.nrhs, cplx{-1, 0}, cplx{1, 0}, tasks, L.s, L.ws.gemm_tasks, "lu_gemm");
}

void trsm_lower_rhs(LuCtx& L, int r0, int r1) {
    const int m = r1 - r0;
    auto& tasks = L.ws.h_gemm;
    if (m <= kTB) {
        const bool own_tile = wide_leaf(L.n);
        const int bs = own_tile ? kTB : (m + 15) / 16 * 16;
        const size_t toff = own_tile ? size_t(r0 / kTB) * 2 * kTB * kTB : 0;
        if (!own_tile) launch_tri_inv(L.n, L.ld, L.dA, L.dD, L.count, bs, r0, 1, 1, L.s);  // tile 0 as scratch
        tasks.assign(L.count, GemmTask{});
        for (int b = 0; b < L.count; ++b) {
            GemmTask& t = tasks[b];
            t.nseg = 1;
            t.A[0] = L.hD[b] + toff;
            t.lda[0] = bs;
            t.B[0] = (*L.hB)[b] + r0;
            t.ldb[0] = L.ldb;
            t.K[0] = m;
            t.C = (*L.hB)[b] + r0;  // in place: <= 64 rows, one CTA per column tile
            t.ldc = L.ldb;
        }
        zgemm_batched(m, L.nrhs, cplx{1, 0}, cplx{0, 0}, tasks, L.s, L.ws.gemm_tasks, "lu_gemm");
        return;
    }
    const int h = ((m + kTB - 1) / kTB + 1) / 2 * kTB;
    trsm_lower_rhs(L, r0, r0 + h);
    tasks.assign(L.count, GemmTask{});
    for (int b = 0; b < L.count; ++b) {  // B[r0+h:r1] -= L[r0+h:r1, r0:r0+h] B[r0:r0+h]
        GemmTask& t = tasks[b];
        t.nseg = 1;
        t.A[0] = L.hA[b] + size_t(r0) * L.ld + r0 + h;
        t.lda[0] = L.ld;
        t.B[0] = (*L.hB)[b] + r0;
        t.ldb[0] = L.ldb;
        t.K[0] = h;
        t.C = (*L.hB)[b] + r0 + h;
        t.ldc = L.ldb;
    }
    zgemm_batched(m - h, L.nrhs, cplx{-1, 0}, cplx{1, 0}, tasks, L.s, L.ws.gemm_tasks, "lu_gemm");
    trsm_lower_rhs(L, r0 + h, r1);
}

// Toledo's recursion on the spine (columns [c0, n)) with the right-hand sides
// B carried as extra columns of every right half: each spine node applies its
// left half's interchanges, L11^{-1} and the A21 update to B as well, so B
// leaves the factorization as L^{-1} P B.  The spine's interchanges are not
// copied back onto the left halves: L is not used after this solve (U is).
void lu_rec_spine(LuCtx& L, int c0, int nc) {
    const int leaf = lu_leaf(L.n);
    if (nc <= leaf) {
        lu_rec(L, c0, nc);
        {
            ProfScope ps("lu_swap", L.s, 0.0);
            launch_row_permute(L.n, L.ldb, L.dB, L.dP, L.count, c0, c0 + nc, 0, L.nrhs, L.s, L.ws.perm);
        }
        trsm_lower_rhs(L, c0, c0 + nc);
        return;
    }
    const int h = ((nc + leaf - 1) / leaf) / 2 * leaf;
    lu_rec(L, c0, h);
    {  // left-half interchanges onto the right half and the right-hand sides
        ProfScope ps("lu_swap", L.s, 0.0);
        launch_row_permute(L.n, L.ld, L.dA, L.dP, L.count, c0, c0 + h, c0 + h, c0 + nc, L.s, L.ws.perm);
        launch_row_permute(L.n, L.ldb, L.dB, L.dP, L.count, c0, c0 + h, 0, L.nrhs, L.s, L.ws.perm);
    }
    trsm_lower_in_factor(L, c0, c0 + h, c0 + h, nc - h, true);
    gemm_update(L, L.n - c0 - h, nc - h, h, size_t(c0) * L.ld + c0 + h, size_t(c0 + h) * L.ld + c0,
                size_t(c0 + h) * L.ld + c0 + h, cplx{-1, 0}, cplx{1, 0}, L.hA, L.hA, L.ld);
    {  // B[c0+h:n] -= A21 B[c0:c0+h]
        auto& tasks = L.ws.h_gemm;
        tasks.assign(L.count, GemmTask{});
        for (int b = 0; b < L.count; ++b) {
            GemmTask& t = tasks[b];
            t.nseg = 1;
            t.A[0] = L.hA[b] + size_t(c0) * L.ld + c0 + h;
            t.lda[0] = L.ld;
            t.B[0] = (*L.hB)[b] + c0;
            t.ldb[0] = L.ldb;
            t.K[0] = h;
            t.C = (*L.hB)[b] + c0 + h;
            t.ldc = L.ldb;
        }
        zgemm_batched(L.n - c0 - h, L.nrhs, cplx{-1, 0}, cplx{1, 0}, tasks, L.s, L.ws.gemm_tasks, "lu_gemm");
    }
    lu_rec_spine(L, c0 + h, nc - h);
}

// x <- U^{-1} x on 64-aligned recursive splits (U's inverse diagonal tiles in
// hDinv, second half of each tile pair)
void upper_solve_tiles(int n, int ld, const std::vector<cplx*>& hA, const std::vector<cplx*>& hDinv,
                       const std::vector<cplx*>& hB, int ldb, int nrhs, cudaStream_t s, Workspace& ws) {
    const int count = int(hA.size());
    auto& tasks = ws.h_gemm;
    std::function<void(int, int)> upper = [&](int b0, int b1) {
        if (b1 - b0 == 1) {
            const int k0 = b0 * kTB, kend = std::min(k0 + kTB, n);
            tasks.assign(count, GemmTask{});
            for (int b = 0; b < count; ++b) {
                GemmTask& t = tasks[b];
                t.nseg = 1;
                t.A[0] = hDinv[b] + size_t(b0) * 2 * kTB * kTB + size_t(kTB) * kTB;
                t.lda[0] = kTB;
                t.B[0] = hB[b] + k0;
                t.ldb[0] = ldb;
                t.K[0] = kend - k0;
                t.C = hB[b] + k0;
                t.ldc = ldb;
            }
            zgemm_batched(kend - k0, nrhs, cplx{1, 0}, cplx{0, 0}, tasks, s, ws.gemm_tasks, "lu_gemm");
            return;
        }
        const int bm = (b0 + b1 + 1) / 2;
        upper(bm, b1);
        const int r0 = b0 * kTB, rm = bm * kTB, r1 = std::min(b1 * kTB, n);
        tasks.assign(count, GemmTask{});
        for (int b = 0; b < count; ++b) {
            GemmTask& t = tasks[b];
            t.nseg = 1;
            t.A[0] = hA[b] + size_t(rm) * ld + r0;
            t.lda[0] = ld;
            t.B[0] = hB[b] + rm;
            t.ldb[0] = ldb;
            t.K[0] = r1 - rm;
            t.C = hB[b] + r0;
            t.ldc = ldb;
        }
        zgemm_batched(rm - r0, nrhs, cplx{-1, 0}, cplx{1, 0}, tasks, s, ws.gemm_tasks, "lu_gemm");
        upper(b0, bm);
    };
    upper(0, (n + kTB - 1) / kTB);
}

// right-looking LU: n/16 steps of (fused panel kernel, trailing 3M GEMM with
// K = 16); two launches per step keep the dependent chain short, which is what
// bounds the deep cyclic-reduction levels (few matrices per launch)
void lu_rl(LuCtx& L) {
    const int n = L.n;
    static bool attr = false;
    if (!attr) {
        QPS_CUDA(cudaFuncSetAttribute(lu_rl_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr = true;
    }
    L.ws.rl_map.ensure(size_t(L.count) * kRlMap);
    for (int k0 = 0; k0 < n; k0 += kRlW) {
        const int w = std::min(kRlW, n - k0);
        {
            ProfScope ps("lu_panel", L.s, 8.0 * L.count * double(n - k0) * w * w / 2.0);
            if (n - k0 <= kRegPanelMaxRows)
                launch_panel_fast(n, L.ld, L.dA, L.dP, k0, w, L.sing, L.ws.rl_map.p, L.count, L.s);
            else
                { QPS_NOTE_LAUNCH(); lu_rl_panel_kernel<<<L.count, 256, size_t(n - k0) * w * sizeof(cplx), L.s>>>(n, L.ld, L.dA, L.dP, k0,
                                                                                             w, L.sing, L.ws.rl_map.p); }
            QPS_CUDA(cudaGetLastError());
        }
        if (n > w) {
            ProfScope ps("lu_swap", L.s, 0.0);
            { QPS_NOTE_LAUNCH(); lu_rl_cols_kernel<<<dim3((n - w + 7) / 8, L.count), 256, 0, L.s>>>(n, L.ld, L.dA, L.ws.rl_map.p, k0, w); }
            QPS_CUDA(cudaGetLastError());
        }
        const int m = n - k0 - w;
        if (m > 0)
            gemm_update(L, m, m, w, size_t(k0) * L.ld + k0 + w, size_t(k0 + w) * L.ld + k0,
                        size_t(k0 + w) * L.ld + k0 + w, cplx{-1, 0}, cplx{1, 0}, L.hA, L.hA, L.ld);
    }
}

}  // namespace

void lu_factor_batched(int n, int ld, const std::vector<cplx*>& hA, const std::vector<int*>& hP,
                       const std::vector<cplx*>& hDinv, int* d_singular, cudaStream_t s, Workspace& ws) {
    const int count = int(hA.size());
    if (count == 0) return;
    ws.ptrs.upload(hA, s);
    ws.iptrs.upload(hP, s);
    ws.ptrs3.upload(hDinv, s);
    LuCtx L{n, ld, count, hA, hP, hDinv, ws.ptrs.p, ws.iptrs.p, ws.ptrs3.p, d_singular, s, ws};
    // Many matrices per launch: the recursive (Toledo) LU, whose big GEMMs run
    // near peak; few matrices: the right-looking LU, whose short dependent
    // chain (three launches per 16 columns) sets the latency.  QPS_LU=rec|rl
    // forces one; QPS_LU_RL_MAX sets the crossover count.
    static const int mode = [] {
        const char* e = getenv("QPS_LU");
        return !e ? 0 : !strcmp(e, "rec") ? 1 : !strcmp(e, "rl") ? 2 : 0;
    }();
    static const int rl_max = [] {
        const char* e = getenv("QPS_LU_RL_MAX");
        return e ? atoi(e) : 64;
    }();
    const bool rl_ok = size_t(n) * kRlW * sizeof(cplx) <= 200 * 1024;
    const bool use_rl = rl_ok && (mode == 2 || (mode == 0 && count <= rl_max));
    if (use_rl) lu_rl(L);
    else lu_rec(L, 0, n);
    // inverse 64x64 diagonal tiles of L and U for the GEMM-shaped solves (the
    // wide leaves of the recursion have inverted their own tiles)
    if (use_rl || !wide_leaf(n)) launch_tri_inv(n, ld, ws.ptrs.p, ws.ptrs3.p, count, kTB, 0, (n + kTB - 1) / kTB, 3, s);
}

// LU with partial pivoting of every matrix and the solve A X = B in one pass:
// the forward substitution rides along the recursion (lu_rec_spine), the back
// substitution uses U's inverse diagonal tiles.  The factors are left as
// U plus an L whose rows below the spine are not re-permuted: use this only
// when A is not solved against again.  B (ld ldb, nrhs columns) becomes X.
void lu_factor_solve_batched(int n, int ld, const std::vector<cplx*>& hA, const std::vector<int*>& hP,
                             const std::vector<cplx*>& hDinv, const std::vector<cplx*>& hB, int ldb, int nrhs,
                             int* d_singular, cudaStream_t s, Workspace& ws) {
    const int count = int(hA.size());
    if (count == 0) return;
    ws.ptrs.upload(hA, s);
    ws.iptrs.upload(hP, s);
    ws.ptrs3.upload(hDinv, s);
    ws.ptrs2.upload(hB, s);
    LuCtx L{n, ld, count, hA, hP, hDinv, ws.ptrs.p, ws.iptrs.p, ws.ptrs3.p, d_singular, s, ws};
    L.hB = &hB;
    L.dB = ws.ptrs2.p;
    L.ldb = ldb;
    L.nrhs = nrhs;
    lu_rec_spine(L, 0, n);
    if (!wide_leaf(n)) launch_tri_inv(n, ld, ws.ptrs.p, ws.ptrs3.p, count, kTB, 0, (n + kTB - 1) / kTB, 2, s);  // U tiles
    upper_solve_tiles(n, ld, hA, hDinv, hB, ldb, nrhs, s, ws);
}

void lu_solve_batched(int n, int ld, const std::vector<cplx*>& hA, const std::vector<int*>& hP,
                      const std::vector<cplx*>& hDinv, const std::vector<cplx*>& hB, int ldb, int nrhs,
                      cudaStream_t s, Workspace& ws) {
    const int count = int(hA.size());
    if (count == 0 || nrhs == 0) return;
    ws.ptrs2.upload(hB, s);
    ws.iptrs.upload(hP, s);
    cplx* const* d_B = ws.ptrs2.p;
    const int* const* d_ipiv = ws.iptrs.p;
    {
        ProfScope ps("lu_swap", s, 0.0);
        launch_row_permute(n, ldb, d_B, d_ipiv, count, 0, n, 0, nrhs, s, ws.perm);
        QPS_CUDA(cudaGetLastError());
    }
    auto& tasks = ws.h_gemm;
    // leaf: B[k0:kend] <- inverse tile * B[k0:kend] (in place, <= 64 rows)
    // column groups: the multiple of 32 (full N tiles of the 32 x 32 GEMM
    // tile) and a narrow remainder (<= 8 columns: the 128 x 8 tile), instead of
    // a last 32-wide tile mostly empty (e.g. 101 = 96 + 5 level-0 right-hand sides)
    int cb0 = 0, cb1 = nrhs;  // the group being solved
    auto leaf = [&](int bi, int which) {
        const int k0 = bi * kTB, kend = std::min(k0 + kTB, n);
        tasks.assign(count, GemmTask{});
        for (int b = 0; b < count; ++b) {
            GemmTask& t = tasks[b];
            t.nseg = 1;
            t.A[0] = hDinv[b] + size_t(bi) * 2 * kTB * kTB + (which ? size_t(kTB) * kTB : 0);
            t.lda[0] = kTB;
            t.B[0] = hB[b] + size_t(cb0) * ldb + k0;
            t.ldb[0] = ldb;
            t.K[0] = kend - k0;
            t.C = hB[b] + size_t(cb0) * ldb + k0;
            t.ldc = ldb;
        }
        zgemm_batched(kend - k0, cb1 - cb0, cplx{1, 0}, cplx{0, 0}, tasks, s, ws.gemm_tasks, "lu_gemm");
    };
    auto update = [&](int M, int K, size_t aoff, int brow, int crow) {
        tasks.assign(count, GemmTask{});
        for (int b = 0; b < count; ++b) {
            GemmTask& t = tasks[b];
            t.nseg = 1;
            t.A[0] = hA[b] + aoff;
            t.lda[0] = ld;
            t.B[0] = hB[b] + size_t(cb0) * ldb + brow;
            t.ldb[0] = ldb;
            t.K[0] = K;
            t.C = hB[b] + size_t(cb0) * ldb + crow;
            t.ldc = ldb;
        }
        zgemm_batched(M, cb1 - cb0, cplx{-1, 0}, cplx{1, 0}, tasks, s, ws.gemm_tasks, "lu_gemm");
    };
    // recursive triangular solves on 64-aligned splits: the top levels carry most
    // flops as GEMMs with K = n/2, n/4, ...
    std::function<void(int, int)> lower = [&](int b0, int b1) {  // tile range [b0, b1)
        if (b1 - b0 == 1) return leaf(b0, 0);
        const int bm = (b0 + b1 + 1) / 2;
        lower(b0, bm);
        const int r0 = b0 * kTB, rm = bm * kTB, r1 = std::min(b1 * kTB, n);
        update(r1 - rm, rm - r0, size_t(r0) * ld + rm, r0, rm);
        lower(bm, b1);
    };
    std::function<void(int, int)> upper = [&](int b0, int b1) {
        if (b1 - b0 == 1) return leaf(b0, 1);
        const int bm = (b0 + b1 + 1) / 2;
        upper(bm, b1);
        const int r0 = b0 * kTB, rm = bm * kTB, r1 = std::min(b1 * kTB, n);
        update(rm - r0, r1 - rm, size_t(rm) * ld + r0, rm, r0);
        upper(b0, bm);
    };
    const int nblk = (n + kTB - 1) / kTB;
    const int rem = nrhs % 32;
    const int nmain = (rem >= 1 && rem <= kThinN && nrhs > 32) ? nrhs - rem : nrhs;
    cb0 = 0;
    cb1 = nmain;
    lower(0, nblk);
    upper(0, nblk);
    if (nmain < nrhs) {
        cb0 = nmain;
        cb1 = nrhs;
        lower(0, nblk);
        upper(0, nblk);
    }
}

void lu_rcond_batched(int n, int ld, cplx* const* d_ptrs, const cplx* base, size_t stride, cplx* const* d_dinv,
                      const cplx* dbase, size_t dstride, int count, double th, int* d_flag, double* d_rcond,
                      cudaStream_t s, double* d_est) {
    if (count == 0 || n == 0) return;
    const size_t sm = (size_t(n) + kRcT) * sizeof(cplx);
    static size_t attr = 48 * 1024;
    if (sm > attr) {
        QPS_CUDA(cudaFuncSetAttribute(lu_rcond_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
        attr = sm;
    }
    // ~6 triangular solves, U read from HBM about once (the CTA's block stays in L2)
    ProfScope ps("lu_rcond", s, 0.0, 16.0 * 0.5 * count * double(n) * n);
    static const int ctas = [] {  // QPS_RCOND_CTAS: CTAs of the estimate (default 32: U of 32 blocks fits L2)
        const char* e = getenv("QPS_RCOND_CTAS");
        return e ? std::max(1, atoi(e)) : 32;
    }();
    const int grid = std::min(count, ctas);
    { QPS_NOTE_LAUNCH(); lu_rcond_kernel<<<grid, kRcT, sm, s>>>(n, ld, count, d_ptrs, base, stride, d_dinv, dbase, dstride,
                                                                 th, d_flag, d_rcond, d_est); }
    QPS_CUDA(cudaGetLastError());
}

void batched_norm1(const cplx* A, int n, int ld, size_t stride, int count, unsigned long long* d_out,
                   cudaStream_t s) {
    if (count == 0 || n == 0) return;
    QPS_CUDA(cudaMemsetAsync(d_out, 0, sizeof(unsigned long long) * count, s));
    ProfScope ps("reduce", s, 0.0, 16.0 * count * double(n) * n);
    { QPS_NOTE_LAUNCH(); colsum_max_kernel<<<dim3(count, 8), 256, 0, s>>>(A, n, ld, stride, d_out); }
    QPS_CUDA(cudaGetLastError());
}

void rcond_screen(const cplx* W, size_t wstride, int n, int col0, int nprobe, const unsigned long long* d_anorm,
                  double rnorm1, int count, double th_def, double th_sus, int* d_flag, int* d_sus, double* d_est_lo,
                  cudaStream_t s) {
    if (count == 0) return;
    { QPS_NOTE_LAUNCH(); rc_screen_kernel<<<count, 256, 0, s>>>(W, wstride, n, col0, nprobe, d_anorm, rnorm1, th_def,
                                                                 th_sus, d_flag, d_sus, d_est_lo); }
    QPS_CUDA(cudaGetLastError());
}

void gather_columns(const std::vector<const cplx*>& src, const std::vector<int>& ld, int rows, const int* d_cols,
                    int ncols, cplx* dst, int ldd, size_t dstride, DBuf<const cplx*>& pbuf, DBuf<int>& lbuf,
                    cudaStream_t s) {
    const int n = int(src.size());
    if (n == 0 || rows == 0 || ncols == 0) return;
    pbuf.upload(src, s);
    lbuf.upload(ld, s);
    ProfScope ps("copy", s, 0.0, 32.0 * n * double(rows) * ncols);
    { QPS_NOTE_LAUNCH(); gather_columns_kernel<<<dim3(n, ncols), 128, 0, s>>>(pbuf.p, lbuf.p, rows, d_cols, ncols, dst,
                                                                              ldd, dstride); }
    QPS_CUDA(cudaGetLastError());
}

namespace {
__global__ void axpy_kernel(cplx* __restrict__ y, const cplx* __restrict__ x, size_t n) {
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        const cplx a = x[i];
        cplx b = y[i];
        b.re += a.re;
        b.im += a.im;
        y[i] = b;
    }
}
}  // namespace

void axpy_blocks(cplx* y, const cplx* x, size_t n, cudaStream_t s) {
    if (n == 0) return;
    const int grid = int(std::min<size_t>((n + 255) / 256, 148 * 16));
    { QPS_NOTE_LAUNCH(); axpy_kernel<<<grid, 256, 0, s>>>(y, x, n); }
    QPS_CUDA(cudaGetLastError());
}

void batched_maxabs(const cplx* X, int m, int n, int ld, size_t stride, int count, double* out, cudaStream_t s) {
    if (count == 0) return;
    ProfScope ps("reduce", s, 0.0, 16.0 * count * double(m) * n);
    { QPS_NOTE_LAUNCH(); maxabs_kernel<<<count, 256, 0, s>>>(X, m, n, ld, stride, out); }
    QPS_CUDA(cudaGetLastError());
}
void batched_fro(const cplx* X, int m, int n, int ld, size_t stride, int count, double* out, cudaStream_t s,
                 double* maxabs_out) {
    if (count == 0) return;
    ProfScope ps("reduce", s, 0.0, 16.0 * count * double(m) * n);
    { QPS_NOTE_LAUNCH(); fro_kernel<<<count, 256, 0, s>>>(X, m, n, ld, stride, out, maxabs_out); }
    QPS_CUDA(cudaGetLastError());
}
void copy_blocks(const cplx* src, int lds, size_t sstride, cplx* dst, int ldd, size_t dstride, int m, int n,
                 int count, cudaStream_t s) {
    if (count == 0 || m == 0 || n == 0) return;
    const int bx = int(std::min<size_t>((size_t(m) * n + 255) / 256, 1024));
    ProfScope ps("copy", s, 0.0, 32.0 * count * double(m) * n);
    { QPS_NOTE_LAUNCH(); copy_blocks_kernel<<<dim3(bx, count), 256, 0, s>>>(src, lds, sstride, dst, ldd, dstride, m, n); }
    QPS_CUDA(cudaGetLastError());
}
void zgemv_batched(int M, cplx alpha, cplx beta, const std::vector<GemvTask>& tasks, cudaStream_t s,
                   DBuf<GemvTask>& d_tasks) {
    if (tasks.empty() || M <= 0) return;
    d_tasks.upload(tasks, s);
    double fl = 0;
    for (const auto& t : tasks)
        for (int q = 0; q < t.nseg; ++q) fl += 8.0 * M * t.n[q];
    ProfScope ps("zgemv", s, fl, fl * 2.0);
    { QPS_NOTE_LAUNCH(); zgemv_kernel<<<dim3((M + 31) / 32, unsigned(tasks.size())), 256, 0, s>>>(M, alpha, beta, d_tasks.p); }
    QPS_CUDA(cudaGetLastError());
}

double measure_dfma_tflops(cudaStream_t s) {
    DBuf<double> out;
    out.ensure(1);
    const int iters = 4096, blocks = 148 * 8, threads = 256;
    { QPS_NOTE_LAUNCH(); dfma_peak_kernel<<<blocks, threads, 0, s>>>(out.p, 64); }
    cudaEvent_t e0, e1;
    QPS_CUDA(cudaEventCreate(&e0));
    QPS_CUDA(cudaEventCreate(&e1));
    QPS_CUDA(cudaEventRecord(e0, s));
    { QPS_NOTE_LAUNCH(); dfma_peak_kernel<<<blocks, threads, 0, s>>>(out.p, iters); }
    QPS_CUDA(cudaEventRecord(e1, s));
    QPS_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    QPS_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    const double flops = 2.0 * 64.0 * iters * double(blocks) * threads;
    return flops / (ms * 1e-3) / 1e12;
}

double measure_dmma_tflops(cudaStream_t s) {
    DBuf<double> out;
    out.ensure(1);
    const int iters = 4096, blocks = 148 * 8, threads = 256;
    { QPS_NOTE_LAUNCH(); dmma_peak_kernel<<<blocks, threads, 0, s>>>(out.p, 64); }
    cudaEvent_t e0, e1;
    QPS_CUDA(cudaEventCreate(&e0));
    QPS_CUDA(cudaEventCreate(&e1));
    QPS_CUDA(cudaEventRecord(e0, s));
    { QPS_NOTE_LAUNCH(); dmma_peak_kernel<<<blocks, threads, 0, s>>>(out.p, iters); }
    QPS_CUDA(cudaEventRecord(e1, s));
    QPS_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    QPS_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    const double flops = 512.0 * 8.0 * iters * double(blocks) * (threads / 32);
    return flops / (ms * 1e-3) / 1e12;
}

}  // namespace qpsb
