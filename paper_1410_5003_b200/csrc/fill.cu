// Nystrom fill kernels for sm_100a (FP64 CUDA-core pipe; transcendental-bound).
//
//   pair_fill_kernel   : every plain kernel block of every layer in one launch
//                        (kernel_quad_block kernels.hpp:78-97 + the alpha
//                        recombination of assembly.hpp:338-397 fused in)
//   proxy_fill_kernel  : every proxy block (proxy_block kernels.hpp:294-308;
//                        B, Q = alpha^-1 Q_p - Q_m, V) in one launch
//   alpert_kernel      : the 16th-order log correction of every self block
//                        (self_quad_parts kernels.hpp:180-280) in one launch
//
// Tiles are 32 targets x 32 sources, 128 threads; a warp covers 32 consecutive
// targets of one source column so stores to the column-major blocks are
// 512-byte coalesced; source nodes are staged in shared memory; the
// near-field Hankel table sits in shared memory, the far-field one in
// constant memory (warp-uniform reads).
#include <algorithm>
#include <cmath>

#include "alpert_table.h"
#include "fill.cuh"
#include "prof.h"

namespace qpsb {

namespace {
__constant__ double c_alpert_nodes[QPS_ALPERT_NAUX];
__constant__ double c_alpert_weights[QPS_ALPERT_NAUX];
// Lagrange weights of the unclamped stencils (alpert.hpp:73-92): identical for
// every row, computed once on the host with the kernel's own arithmetic
__device__ double g_alpert_lw[2 * QPS_ALPERT_NAUX][16];
__constant__ int c_alpert_t0[2 * QPS_ALPERT_NAUX];
double* g_near_table = nullptr;
}  // namespace

void upload_hankel_tables() {
    static bool done = false;
    if (done) return;
    QPS_CUDA(cudaMemcpyToSymbol(c_hankel_far, qps_hankel_far_coeffs, sizeof(qps_hankel_far_coeffs)));
    QPS_CUDA(cudaMemcpyToSymbol(c_alpert_nodes, qps_alpert_nodes, sizeof(qps_alpert_nodes)));
    {
        double lw[2 * QPS_ALPERT_NAUX][16];
        int t0s[2 * QPS_ALPERT_NAUX];
        for (int lane = 0; lane < 2 * QPS_ALPERT_NAUX; ++lane) {
            const int side = lane < QPS_ALPERT_NAUX ? -1 : 1;
            const double xi = side * qps_alpert_nodes[lane % QPS_ALPERT_NAUX];
            const int t0 = int(std::floor(xi)) - 16 / 2 + 1;
            t0s[lane] = t0;
            for (int rr = 0; rr < 16; ++rr) {
                double num = 1.0, den = 1.0;
                const int tr = t0 + rr;
                for (int qq = 0; qq < 16; ++qq) {
                    if (qq == rr) continue;
                    const int tq = t0 + qq;
                    num *= xi - tq;
                    den *= double(tr - tq);
                }
                lw[lane][rr] = num / den;
            }
        }
        QPS_CUDA(cudaMemcpyToSymbol(g_alpert_lw, lw, sizeof(lw)));
        QPS_CUDA(cudaMemcpyToSymbol(c_alpert_t0, t0s, sizeof(t0s)));
    }
    QPS_CUDA(cudaMemcpyToSymbol(c_alpert_weights, qps_alpert_weights, sizeof(qps_alpert_weights)));
    QPS_CUDA(cudaMalloc(&g_near_table, sizeof(qps_hankel_near_coeffs)));
    QPS_CUDA(cudaMemcpy(g_near_table, qps_hankel_near_coeffs, sizeof(qps_hankel_near_coeffs),
                        cudaMemcpyHostToDevice));
    done = true;
}
const double* device_near_table() { return g_near_table; }

namespace {

constexpr int kTile = 32;
constexpr int kThreads = 128;
#ifndef QPS_MINB_PLAIN
#define QPS_MINB_PLAIN 5  // blocks per SM: plain one-wavenumber tiles (96 registers)
#endif
#ifndef QPS_MINB_SELF
#define QPS_MINB_SELF 4   // the others (128 registers)
#endif
constexpr int kNear = 4 * QPS_HANKEL_NEAR_TERMS * QPS_HANKEL_XB;

__device__ __forceinline__ void load_near(double* s_near, const double* g_near) {
    for (int i = threadIdx.x; i < kNear; i += blockDim.x) s_near[i] = g_near[i];
}

// re-layout [interval][function][term] -> [interval][term]{J0, J1}{R0, R1}
__device__ __forceinline__ void load_near2(double2* s_near2, const double* g_near) {
    for (int e = threadIdx.x; e < QPS_HANKEL_XB * QPS_HANKEL_NEAR_TERMS * 2; e += blockDim.x) {
        const int half = e & 1, k = (e >> 1) % QPS_HANKEL_NEAR_TERMS, i = (e >> 1) / QPS_HANKEL_NEAR_TERMS;
        const double* c = g_near + i * QPS_NEAR_STRIDE;
        s_near2[e] = make_double2(c[(2 * half) * QPS_HANKEL_NEAR_TERMS + k], c[(2 * half + 1) * QPS_HANKEL_NEAR_TERMS + k]);
    }
}

__device__ __forceinline__ void cacc(cplx& a, cplx c, double s, cplx v) {
    // a += s * c * v
    const double vr = s * v.re, vi = s * v.im;
    a.re += c.re * vr - c.im * vi;
    a.im += c.re * vi + c.im * vr;
}

__device__ __forceinline__ void cmacc(cplx& a, cplx c, cplx v) {
    // a += c * v
    a.re = fma(c.re, v.re, fma(-c.im, v.im, a.re));
    a.im = fma(c.re, v.im, fma(c.im, v.re, a.im));
}

__device__ __forceinline__ void store(cplx* p, cplx v, int acc) {
    if (acc) {
        cplx o = *p;
        o.re += v.re;
        o.im += v.im;
        *p = o;
    } else {
        *p = v;
    }
}

__device__ __forceinline__ int seg_index(const PairTask& T, int m) {
    int s = 0;
    while (s + 1 < T.nseg && m >= T.seg_start[s + 1]) ++s;
    return s;
}

// body of one 32 x 32 tile, specialised on the self-block kind (0 plain, 1
// smooth self, 2 open-arc self) and the number of wavenumbers (the A_jj blocks
// sum two); the specialisation removes per-pair branches and lets the two
// wavenumber evaluations of a pair interleave
// Mirrored tiles stage the transposed block's entries in shared memory
// (s_mir: 4 kinds x 16 source rows x 32 (+1) targets) and write them
// coalesced every 16 source columns: written directly, each would be a
// separate 16-byte store and the LSU queue stalls the tile's shared loads.
constexpr int kMirRows = 16, kMirLd = kTile + 1;

template <int SELF, int NK, bool MIRROR>
__device__ __forceinline__ void pair_tile(const PairTask& T, int m0, int j0, DevPool pool, const double* sx,
                                          const double* sy, const double* snx, const double* sny, const double* sw,
                                          const double2* s_near2, int* err, bool mir, cplx* s_mir) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int m = m0 + lane;
    const bool act = m < T.nt;
    if (!MIRROR && !act) return;
    // task constants in registers
    const int nterm = T.nterm, ns = T.ns;
    constexpr int nk = NK, self = SELF;
    const double k0 = T.k[0], k1 = T.k[1], sg0 = T.ksign[0], sg1 = T.ksign[1];
    const double ik0 = 1.0 / k0, ik1 = nk > 1 ? 1.0 / k1 : 0.0;
    // per-wavenumber scale factors: sign/4, sign*k/4 and (8/k)^2 for u = (8/x)^2
    const double s40 = 0.25 * sg0, s41 = 0.25 * sg1, d40 = s40 * k0, d41 = s41 * k1;
    const double u0 = 64.0 * ik0 * ik0, u1 = 64.0 * ik1 * ik1;
    const int gt = T.t_off + (act ? m : 0);
    const double tx = pool.x[gt], ty = pool.y[gt], tnx = pool.nx[gt], tny = pool.ny[gt];
    const double wm = MIRROR ? pool.w[gt] : 0.0;  // the target's weight as a mirrored source
    bool corrected = true;
    int mseg = 0;
    if (self == 2) {
        mseg = seg_index(T, m);
        const int ml = m - T.seg_start[mseg], n = T.seg_start[mseg + 1] - T.seg_start[mseg];
        corrected = min(ml, n - 1 - ml) >= QPS_ALPERT_A;
    }
    // one (target m, source column q) entry: original into the block, mirror into (bD.. )
    auto entry = [&](int q, cplx& bD, cplx& bS, cplx& bT, cplx& bDs) {
        const int j = j0 + q;
        cplx aD{0, 0}, aS{0, 0}, aT{0, 0}, aDs{0, 0};
        const double zx0 = sx[q], zy = sy[q], znx = snx[q], zny = sny[q], w = sw[q];
        const double nn = tnx * znx + tny * zny;
#pragma unroll 1
        for (int t = 0; t < nterm; ++t) {
            const int l = T.lsh[t];
            if (self == 1) {
                const int off = j + l * ns - m;
                if (off <= QPS_ALPERT_A - 1 && off >= -(QPS_ALPERT_A - 1)) continue;
            } else if (self == 2 && l == 0) {
                if (j == m) continue;
                if (corrected && j - m <= QPS_ALPERT_A - 1 && m - j <= QPS_ALPERT_A - 1 && seg_index(T, j) == mseg)
                    continue;
            }
            const double rvx = (tx + T.tdx[t]) - (zx0 + T.sdx[t]), rvy = ty - zy;
            const double r2 = rvx * rvx + rvy * rvy;
            // coincidence test of eval_kernels (kernels.hpp:38-39), r < 1e-13 (1 + |x|):
            // the cheap prefilter r^2 < 1e-16 admits every |x| < 1e5
            if (r2 < 1e-16) {
                const double xx = tx + T.tdx[t];
                if (sqrt(r2) < 1e-13 * (1.0 + sqrt(xx * xx + ty * ty))) {
                    atomicOr(err, 1);
                    continue;
                }
            }
            const double inv_r = rsqrt(r2);
            const double r = r2 * inv_r;
            const double cn = (rvx * tnx + rvy * tny) * inv_r;
            const double cdn = (rvx * znx + rvy * zny) * inv_r;
            const double cc = cn * cdn;
            const double Bt = inv_r * (nn - 2.0 * cc);  // k-independent factor of the H1 term of T
            const double ir2 = inv_r * inv_r;
            // eval_kernels (kernels.hpp:35-52) summed over the wavenumbers with signs:
            //   S = (i/4) H0, D = (ik/4) H1 cdn, D* = -(ik/4) H1 cn,
            //   T = (ik/4) [k cn cdn H0 + (nn - 2 cn cdn)/r H1]
            cplx tD{0, 0}, tS{0, 0}, tT{0, 0}, tDs{0, 0};
#pragma unroll
            for (int kk = 0; kk < NK; ++kk) {
                const double k = kk ? k1 : k0;
                HankelOut h;
                hankel01_dev(k * r, inv_r * (kk ? ik1 : ik0), ir2 * (kk ? u1 : u0), s_near2, h);
                const double s4 = kk ? s41 : s40, d4 = kk ? d41 : d40;
                tS.re = fma(-s4, h.y0, tS.re);
                tS.im = fma(s4, h.j0, tS.im);
                const double h1r = -d4 * h.y1, h1i = d4 * h.j1;
                tD.re = fma(h1r, cdn, tD.re);
                tD.im = fma(h1i, cdn, tD.im);
                tDs.re = fma(-h1r, cn, tDs.re);
                tDs.im = fma(-h1i, cn, tDs.im);
                const double A = k * cc;
                const double br = fma(A, h.j0, Bt * h.j1), bi = fma(A, h.y0, Bt * h.y1);
                tT.re = fma(-d4, bi, tT.re);
                tT.im = fma(d4, br, tT.im);
            }
            const cplx c = T.coef[t];
            const cplx wc{w * c.re, w * c.im};
            cmacc(aD, wc, tD);
            cmacc(aS, wc, tS);
            cmacc(aT, wc, tT);
            cmacc(aDs, wc, tDs);
            if (MIRROR && mir) {
                const cplx mc = T.mcoef[t];
                const cplx wmc{wm * mc.re, wm * mc.im};
                cmacc(bD, wmc, tDs);
                cmacc(bS, wmc, tS);
                cmacc(bT, wmc, tT);
                cmacc(bDs, wmc, tD);
            }
        }
        if (T.ident && j == m) {
            aD.re -= 1.0;
            aDs.re += 1.0;
        }
        const size_t o = size_t(j) * T.ld + m;
        store(T.oD + o, aD, T.accumulate);
        store(T.oS + o, aS, T.accumulate);
        store(T.oT + o, aT, T.accumulate);
        store(T.oDs + o, aDs, T.accumulate);
    };
    if constexpr (!MIRROR) {
#pragma unroll 1
        for (int q = warp; q < kTile; q += kThreads / 32) {
            if (j0 + q >= ns) break;
            cplx bD, bS, bT, bDs;
            entry(q, bD, bS, bT, bDs);
        }
    } else {
#pragma unroll 1
        for (int half = 0; half < kTile / kMirRows; ++half) {
#pragma unroll 1
            for (int q = half * kMirRows + warp; q < (half + 1) * kMirRows; q += kThreads / 32) {
                if (!act || j0 + q >= ns) continue;
                cplx bD{0, 0}, bS{0, 0}, bT{0, 0}, bDs{0, 0};
                entry(q, bD, bS, bT, bDs);
                if (mir) {
                    const int rq = (q - half * kMirRows) * kMirLd + lane;
                    s_mir[0 * kMirRows * kMirLd + rq] = bD;
                    s_mir[1 * kMirRows * kMirLd + rq] = bS;
                    s_mir[2 * kMirRows * kMirLd + rq] = bT;
                    s_mir[3 * kMirRows * kMirLd + rq] = bDs;
                }
            }
            if (!mir) continue;  // CTA-uniform
            __syncthreads();
            // rows j0 + half*16 .. +15 of the mirror block, columns m0 .. m0+31:
            // 16 consecutive rows (256 bytes) per column
            for (int e = threadIdx.x; e < 4 * kTile * kMirRows; e += kThreads) {
                const int kind = e / (kTile * kMirRows), rem = e % (kTile * kMirRows);
                const int col = rem / kMirRows, row = rem % kMirRows;
                const int n = j0 + half * kMirRows + row, mm = m0 + col;
                if (n >= ns || mm >= T.nt) continue;
                cplx* base = kind == 0 ? T.mD : kind == 1 ? T.mS : kind == 2 ? T.mT : T.mDs;
                store(base + size_t(mm) * T.mld + n, s_mir[kind * kMirRows * kMirLd + row * kMirLd + col],
                      T.accumulate);
            }
            __syncthreads();
        }
    }
}

// one kernel per block kind (self kind x wavenumber count): each gets its own
// register allocation instead of the largest of the six
template <int SELF, int NK, bool MIRROR>
__global__ void __launch_bounds__(kThreads, (SELF == 0 && NK == 1 && !MIRROR) ? QPS_MINB_PLAIN : QPS_MINB_SELF)
    pair_fill_kernel(const PairTask* __restrict__ tasks, const int4* __restrict__ tiles, DevPool pool,
                     const double* __restrict__ g_near, int* err) {
    __shared__ double2 s_near2[QPS_HANKEL_XB * QPS_HANKEL_NEAR_TERMS * 2];
    __shared__ double sx[kTile], sy[kTile], snx[kTile], sny[kTile], sw[kTile];
    __shared__ PairTask T;
    // blockIdx.y: task of this kind {task index, row tiles, total tiles};
    // blockIdx.x: tile within the task (row tiles fastest)
    const int4 tk = tiles[blockIdx.y];
    if (int(blockIdx.x) >= tk.z) return;
    if (threadIdx.x == 0) T = tasks[tk.x];
    load_near2(s_near2, g_near);
    __syncthreads();
    // tk.w: self block on its upper tile triangle (index c (c + 1) / 2 + r, r <= c),
    // the strictly upper tiles mirrored onto the lower ones
    int tr, tc;
    if (MIRROR && tk.w) {
        const int idx = int(blockIdx.x);
        int cc = int((sqrt(8.0 * idx + 1.0) - 1.0) * 0.5);
        while (cc * (cc + 1) / 2 > idx) --cc;
        while ((cc + 1) * (cc + 2) / 2 <= idx) ++cc;
        tc = cc;
        tr = idx - cc * (cc + 1) / 2;
    } else {
        tr = int(blockIdx.x) % tk.y;
        tc = int(blockIdx.x) / tk.y;
    }
    const int m0 = tr * kTile, j0 = tc * kTile;
    const bool mir = MIRROR && !(tk.w && tr == tc);
    if (threadIdx.x < kTile) {
        const int j = j0 + threadIdx.x;
        if (j < T.ns) {
            const int g = T.s_off + j;
            sx[threadIdx.x] = pool.x[g];
            sy[threadIdx.x] = pool.y[g];
            snx[threadIdx.x] = pool.nx[g];
            sny[threadIdx.x] = pool.ny[g];
            sw[threadIdx.x] = pool.w[g];
        }
    }
    __syncthreads();
    __shared__ cplx s_mir[MIRROR ? 4 * kMirRows * kMirLd : 1];
    pair_tile<SELF, NK, MIRROR>(T, m0, j0, pool, sx, sy, snx, sny, sw, s_near2, err, mir, s_mir);
}

__global__ void __launch_bounds__(kThreads) proxy_fill_kernel(const ProxyTask* __restrict__ tasks,
                                                              const int4* __restrict__ tiles, DevPool pool,
                                                              const double* __restrict__ g_near, int* err) {
    __shared__ double s_near[kNear];
    __shared__ double sx[kTile], sy[kTile], snx[kTile], sny[kTile];
    __shared__ ProxyTask T;
    const int4 tile = tiles[blockIdx.x];
    if (threadIdx.x == 0) T = tasks[tile.x];
    load_near(s_near, g_near);
    __syncthreads();
    const int m0 = tile.y, p0 = tile.z;
    if (threadIdx.x < kTile) {
        const int p = p0 + threadIdx.x;
        if (p < T.P) {
            const int g = T.p_off + p;
            sx[threadIdx.x] = pool.x[g];
            sy[threadIdx.x] = pool.y[g];
            snx[threadIdx.x] = pool.nx[g];
            sny[threadIdx.x] = pool.ny[g];
        }
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int m = m0 + lane;
    if (m >= T.nt) return;
    const int gt = T.t_off + m;
    const double tx = pool.x[gt], ty = pool.y[gt], tnx = pool.nx[gt], tny = pool.ny[gt];
    const double k = T.k;
    for (int q = warp; q < kTile; q += kThreads / 32) {
        const int p = p0 + q;
        if (p >= T.P) break;
        cplx phi{0, 0}, dphi{0, 0};
        for (int t = 0; t < T.nterm; ++t) {
            const double xx = tx + T.tdx[t];
            const double rvx = xx - sx[q], rvy = ty - sy[q];
            const double r = sqrt(rvx * rvx + rvy * rvy);
            if (r < 1e-13 * (1.0 + sqrt(xx * xx + ty * ty))) {
                atomicOr(err, 1);
                continue;
            }
            HankelOut h;
            hankel01_eval(k * r, s_near, c_hankel_far, h);
            KVals v;
            kernel_vals(k, rvx, rvy, r, tnx, tny, snx[q], sny[q], h, v);
            // phi = D + i k S ; dphi = T + i k D*
            const cplx f{v.D.re - k * v.S.im, v.D.im + k * v.S.re};
            const cplx df{v.T.re - k * v.Ds.im, v.T.im + k * v.Ds.re};
            cacc(phi, T.coef[t], 1.0, f);
            cacc(dphi, T.coef[t], 1.0, df);
        }
        store(T.out + size_t(p) * T.ld + m, phi, T.accumulate);
        store(T.out + size_t(p) * T.ld + T.drow + m, dphi, T.accumulate);
    }
}

// ---- segment parametrisations evaluated on the device (geometry.hpp) ----
// Kress grading evaluated without FMA contraction so the auxiliary nodes
// round exactly like the host's (geometry.hpp:37-65): near a corner v(s) is a
// difference of O(1) terms and contraction changes its last bits.
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double kv(double s, int q) {
    const double pi = 3.14159265358979323846;
    const double u = (pi - s) / pi;
    return add(add(mul(mul(mul(add(1.0 / q, -0.5), u), u), u), (s - pi) / (pi * q)), 0.5);
}
__device__ __forceinline__ double kvp(double s, int q) {
    const double pi = 3.14159265358979323846;
    const double u = (pi - s) / pi;
    return add(mul(mul(mul(-3.0, add(1.0 / q, -0.5)), u), u) / pi, 1.0 / (pi * q));
}

__device__ void seg_eval(const SegDesc& sd, const double* fourier, double s, double& zx, double& zy, double& tx,
                         double& ty) {
    const double pi = 3.14159265358979323846;
    if (sd.kind == SEG_LINE) {
        const int q = sd.q;
        const double v1 = kv(s, q), v2 = kv(2.0 * pi - s, q);
        const double vq = pow(v1, double(q)), vr = pow(v2, double(q));
        const double wv = mul(2.0 * pi, vq) / add(vq, vr);
        const double d1 = mul(mul(double(q), pow(v1, double(q - 1))), kvp(s, q));
        const double d2 = mul(mul(double(-q), pow(v2, double(q - 1))), kvp(2.0 * pi - s, q));
        const double den = add(vq, vr);
        const double wp = mul(2.0 * pi, add(mul(d1, den), -mul(vq, add(d1, d2)))) / mul(den, den);
        const double f = wv / (2.0 * pi);
        zx = add(sd.Ax, mul(sd.Bx - sd.Ax, f));
        zy = add(sd.Ay, mul(sd.By - sd.Ay, f));
        tx = mul((sd.Bx - sd.Ax) / (2.0 * pi), wp);
        ty = mul((sd.By - sd.Ay) / (2.0 * pi), wp);
        return;
    }
    const double d = sd.d;
    const double x = -0.5 * d + d * s / (2.0 * pi);
    const double dxds = d / (2.0 * pi);
    double y = sd.y0, dydx = 0.0;
    if (sd.kind == SEG_SINE) {
        double sn, cs;
        sincos(2.0 * pi * x / d + sd.phase, &sn, &cs);
        y += sd.amp * sn;
        dydx = sd.amp * (2.0 * pi / d) * cs;
    } else {
        const double* cc = fourier + sd.coef_off;
        const double* ss = cc + sd.ncos;
        for (int m = 0; m < sd.ncos; ++m) {
            double sn, cs;
            sincos(2.0 * pi * double(m + 1) * x / d, &sn, &cs);
            y += cc[m] * cs;
            dydx -= cc[m] * (2.0 * pi * double(m + 1) / d) * sn;
        }
        for (int m = 0; m < sd.nsin; ++m) {
            double sn, cs;
            sincos(2.0 * pi * double(m + 1) * x / d, &sn, &cs);
            y += ss[m] * sn;
            dydx += ss[m] * (2.0 * pi * double(m + 1) / d) * cs;
        }
    }
    zx = x;
    zy = y;
    tx = dxds;
    ty = dydx * dxds;
}

constexpr int kBand = 2 * 16 + 1;  // columns m-16 .. m+16 reached by the stencils

// One warp per corrected row.  Lanes 0..29 evaluate one auxiliary node each
// (both wavenumbers), then lanes sweep the 33-column window.
__global__ void __launch_bounds__(128) alpert_kernel(const AlpertTask* __restrict__ tasks, int ntasks,
                                                     int total_rows, DevPool pool,
                                                     const SegDesc* __restrict__ segs,
                                                     const double* __restrict__ fourier,
                                                     const double* __restrict__ aux,
                                                     const double* __restrict__ g_near, int* err) {
    __shared__ double s_near[kNear];
    __shared__ cplx s_val[4][2 * QPS_ALPERT_NAUX][4];    // per warp, aux, kind
    __shared__ double s_lw[4][2 * QPS_ALPERT_NAUX][16];  // Lagrange weights
    __shared__ int s_t0[4][2 * QPS_ALPERT_NAUX];
    __shared__ double s_lwtab[2 * QPS_ALPERT_NAUX][16];  // the unclamped weights, one copy per CTA
    __shared__ int s_clamped[4];
    load_near(s_near, g_near);
    for (int e = threadIdx.x; e < 2 * QPS_ALPERT_NAUX * 16; e += blockDim.x) (&s_lwtab[0][0])[e] = (&g_alpert_lw[0][0])[e];
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // grid-stride over rows: the tables above are loaded once per CTA
    for (int row = blockIdx.x * 4 + warp; row < total_rows; row += gridDim.x * 4) {
    int lo = 0, hi = ntasks - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (tasks[mid].row_start <= row) lo = mid; else hi = mid - 1;
    }
    const AlpertTask& T = tasks[lo];
    const int m = row - T.row_start;
    // locate segment
    int sidx = 0;
    for (int s = 1; s < T.nseg; ++s)
        if (m >= segs[T.seg_first + s].offset) sidx = s;
    const SegDesc sd = segs[T.seg_first + sidx];
    const int mloc = m - sd.offset;
    if (!T.smooth && min(mloc, sd.n - 1 - mloc) < QPS_ALPERT_A) continue;  // plain fallback row
    const double pi = 3.14159265358979323846;
    const double h = 2.0 * pi / sd.n;
    const int gt = T.t_off + m;
    const double xmx = pool.x[gt], xmy = pool.y[gt], nmx = pool.nx[gt], nmy = pool.ny[gt];
    if (lane == 0) s_clamped[warp] = 0;
    __syncwarp();

    if (lane < 2 * QPS_ALPERT_NAUX) {
        const int side = lane < QPS_ALPERT_NAUX ? -1 : 1;
        const int kk = lane % QPS_ALPERT_NAUX;
        const double xi = side * c_alpert_nodes[kk];
        double zx, zy, nzx, nzy, qw;
        if (T.aux_off >= 0) {  // open arc: the host's nodes (bit-identical to the reference)
            const double* e = aux + T.aux_off + (size_t(m) * 2 * QPS_ALPERT_NAUX + lane) * 5;
            zx = e[0];
            zy = e[1];
            nzx = e[2];
            nzy = e[3];
            qw = e[4];
        } else {
            const double s_aux = (mloc + 0.5 + xi) * h;
            double tzx, tzy;
            seg_eval(sd, fourier, s_aux, zx, zy, tzx, tzy);
            const double speed = sqrt(tzx * tzx + tzy * tzy);
            nzx = tzy / speed;
            nzy = -tzx / speed;
            qw = h * c_alpert_weights[kk] * speed;
        }
        const double rvx = xmx - zx, rvy = xmy - zy;
        const double r = hypot(rvx, rvy);  // Vec2::norm, types.hpp:24
        cplx vD{0, 0}, vS{0, 0}, vT{0, 0}, vDs{0, 0};
        if (r < 1e-13 * (1.0 + sqrt(xmx * xmx + xmy * xmy))) {
            atomicOr(err, 1);
        } else {
            for (int q = 0; q < T.nk; ++q) {
                const double k = T.k[q];
                HankelOut hh;
                hankel01_eval(k * r, s_near, c_hankel_far, hh);
                KVals v;
                kernel_vals(k, rvx, rvy, r, nmx, nmy, nzx, nzy, hh, v);
                const double sg = T.ksign[q] * qw;
                vD.re += sg * v.D.re; vD.im += sg * v.D.im;
                vS.re += sg * v.S.re; vS.im += sg * v.S.im;
                vT.re += sg * v.T.re; vT.im += sg * v.T.im;
                vDs.re += sg * v.Ds.re; vDs.im += sg * v.Ds.im;
            }
        }
        s_val[warp][lane][0] = vD;
        s_val[warp][lane][1] = vS;
        s_val[warp][lane][2] = vT;
        s_val[warp][lane][3] = vDs;
        // alpert_stencil_start (alpert.hpp:90-92), clamped for open arcs (kernels.hpp:256)
        const int t0u = c_alpert_t0[lane];
        int t0 = t0u;
        if (!T.smooth) t0 = max(-mloc, min(t0, sd.n - 16 - mloc));
        s_t0[warp][lane] = t0;
        // lagrange_weights (alpert.hpp:73-87): the precomputed table unless clamped
        if (t0 != t0u) s_clamped[warp] = 1;
        if (t0 == t0u && !T.smooth) {  // open arcs: a clamped lane makes the warp use s_lw for every lane
#pragma unroll
            for (int rr = 0; rr < 16; ++rr) s_lw[warp][lane][rr] = s_lwtab[lane][rr];
        }
        if (t0 != t0u)
        for (int rr = 0; rr < 16; ++rr) {
            double num = 1.0, den = 1.0;
            const int tr = t0 + rr;
            for (int qq = 0; qq < 16; ++qq) {
                if (qq == rr) continue;
                const int tq = t0 + qq;
                num *= xi - tq;
                den *= double(tr - tq);
            }
            s_lw[warp][lane][rr] = num / den;
        }
    }
    __syncwarp();
    const int N = T.N;
    const double(*lwt)[16] = s_clamped[warp] ? s_lw[warp] : s_lwtab;  // warp-uniform
    for (int c = lane; c < kBand; c += 32) {
        const int o = c - 16;  // column offset relative to the row
        cplx acc[4] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
        for (int a = 0; a < 2 * QPS_ALPERT_NAUX; ++a) {
            const int rr = o - s_t0[warp][a];
            if (rr < 0 || rr >= 16) continue;
            const double lw = lwt[a][rr];
            for (int kd = 0; kd < 4; ++kd) {
                acc[kd].re += lw * s_val[warp][a][kd].re;
                acc[kd].im += lw * s_val[warp][a][kd].im;
            }
        }
        const int jraw = mloc + o;
        bool any = false;
        for (int kd = 0; kd < 4; ++kd) any |= (acc[kd].re != 0.0 || acc[kd].im != 0.0);
        if (T.mode == 0) {
            if (!any) continue;
            cplx ph{1.0, 0.0};
            int col;
            if (jraw >= 0 && jraw < sd.n) {
                col = sd.offset + jraw;
            } else {
                col = (jraw + N) % N;
                ph = jraw < 0 ? T.alpha_inv : T.alpha;
            }
            const size_t off = size_t(col) * T.ld + m;
            cplx* outs[4] = {T.oD, T.oS, T.oT, T.oDs};  // the four quadrants: distinct entries
            cplx v[4];
#pragma unroll
            for (int kd = 0; kd < 4; ++kd) v[kd] = outs[kd][off];  // four loads in flight
#pragma unroll
            for (int kd = 0; kd < 4; ++kd) {
                v[kd].re += ph.re * acc[kd].re - ph.im * acc[kd].im;
                v[kd].im += ph.re * acc[kd].im + ph.im * acc[kd].re;
                outs[kd][off] = v[kd];
            }
        } else {
            if (jraw >= 0 && jraw < sd.n) {
                if (!any) continue;
                const size_t off = size_t(sd.offset + jraw) * T.ld + m;
                cplx* outs[4] = {T.oD, T.oS, T.oT, T.oDs};
                cplx v[4];
#pragma unroll
                for (int kd = 0; kd < 4; ++kd) v[kd] = outs[kd][off];
#pragma unroll
                for (int kd = 0; kd < 4; ++kd) {
                    v[kd].re += acc[kd].re;
                    v[kd].im += acc[kd].im;
                    outs[kd][off] = v[kd];
                }
            } else {
                // out-of-period: Alpert spill plus (smooth) removal of the band
                // entry the plain l = +-1 neighbour block carries (kernels.hpp:229-241)
                if (T.smooth && o >= -(QPS_ALPERT_A - 1) && o <= QPS_ALPERT_A - 1) {
                    const int col = (jraw + N) % N;
                    const int l = jraw < 0 ? -1 : 1;
                    const int gs = T.t_off + col;
                    const double zx = pool.x[gs] + l * segs[T.seg_first].d, zy = pool.y[gs];
                    const double rvx = xmx - zx, rvy = xmy - zy;
                    const double r = sqrt(rvx * rvx + rvy * rvy);
                    const double wneg = -pool.w[gs];
                    for (int q = 0; q < T.nk; ++q) {
                        const double k = T.k[q];
                        HankelOut hh;
                        hankel01_eval(k * r, s_near, c_hankel_far, hh);
                        KVals v;
                        kernel_vals(k, rvx, rvy, r, nmx, nmy, pool.nx[gs], pool.ny[gs], hh, v);
                        const double sg = T.ksign[q] * wneg;
                        acc[0].re += sg * v.D.re; acc[0].im += sg * v.D.im;
                        acc[1].re += sg * v.S.re; acc[1].im += sg * v.S.im;
                        acc[2].re += sg * v.T.re; acc[2].im += sg * v.T.im;
                        acc[3].re += sg * v.Ds.re; acc[3].im += sg * v.Ds.im;
                    }
                }
                cplx* wb = T.wrap + (size_t(m) * kBand + c) * 4;
                for (int kd = 0; kd < 4; ++kd) wb[kd] = acc[kd];
            }
        }
    }
    __syncwarp();  // s_val / s_lw / s_t0 are rewritten by the warp's next row
    }
}

__global__ void hankel_batch_kernel(int n, const double* __restrict__ x, cplx* h0, cplx* h1,
                                    const double* __restrict__ g_near) {
    __shared__ double s_near[kNear];
    load_near(s_near, g_near);
    __syncthreads();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        HankelOut h;
        hankel01_eval(x[i], s_near, c_hankel_far, h);
        h0[i] = cplx{h.j0, h.y0};
        h1[i] = cplx{h.j1, h.y1};
    }
}

template <class Task>
void build_tiles(const std::vector<Task>& tasks, std::vector<int4>& tiles, int (*cols)(const Task&)) {
    tiles.clear();
    for (int t = 0; t < int(tasks.size()); ++t) {
        const int nt = tasks[t].nt, nc = cols(tasks[t]);
        for (int j0 = 0; j0 < nc; j0 += kTile)
            for (int m0 = 0; m0 < nt; m0 += kTile) tiles.push_back(make_int4(t, m0, j0, 0));
    }
}

}  // namespace

void launch_pair_fill(const std::vector<PairTask>& tasks, const DevPool& pool, int* d_err, cudaStream_t s,
                      DBuf<PairTask>& d_tasks, DBuf<int4>& d_tiles) {
    if (tasks.empty()) return;
    // one launch per block kind (self * 2 + nk - 1, plus 6 + self * 2 + nk - 1
    // for mirrored tasks) over a 2-D grid (tile, task of the kind): the tile of
    // a CTA is computed in-kernel, so no tile list is built on the host
    constexpr int kKinds = 10;
    std::vector<int4> ids[kKinds];
    int maxt[kKinds] = {0};
    for (int t = 0; t < int(tasks.size()); ++t) {
        const PairTask& T = tasks[t];
        int kind = T.self * 2 + (T.nk - 1);
        if (kind < 0 || kind > 5 || (T.mirror && T.self > 1)) fail(QPS_ERR_INTERNAL, "pair fill: unknown block kind");
        if (T.mirror) kind += 6;
        const int tm = (T.nt + kTile - 1) / kTile, tn = (T.ns + kTile - 1) / kTile;
        if (tm * tn == 0) continue;
        const bool tri = T.mirror && T.self == 1;
        if (tri && tm != tn) fail(QPS_ERR_INTERNAL, "pair fill: mirrored self block must be square");
        const int ntile = tri ? tm * (tm + 1) / 2 : tm * tn;
        ids[kind].push_back(make_int4(t, tm, ntile, tri ? 1 : 0));
        maxt[kind] = std::max(maxt[kind], ntile);
    }
    std::vector<int4> all;
    size_t off[kKinds + 1] = {0};
    for (int kind = 0; kind < kKinds; ++kind) {
        off[kind] = all.size();
        all.insert(all.end(), ids[kind].begin(), ids[kind].end());
    }
    off[kKinds] = all.size();
    if (all.empty()) return;
    d_tasks.upload(tasks, s);
    d_tiles.upload(all, s);
    double ev = 0;  // kernel evaluations produced (a mirrored pair yields two)
    for (const auto& t : tasks) ev += double(t.nt) * t.ns * t.nterm * t.nk * (t.mirror && t.self == 0 ? 2 : 1);
    ProfScope ps("fill_pair", s, 200.0 * ev, 0.0, ev);
    for (int kind = 0; kind < kKinds; ++kind) {
        const unsigned n = unsigned(off[kind + 1] - off[kind]);
        if (!n) continue;
        if (n > 65535) fail(QPS_ERR_CONFIG, "pair fill: too many blocks of one kind for one launch");
        const int4* tl = d_tiles.p + off[kind];
        const dim3 grid(unsigned(maxt[kind]), n);
        switch (kind) {
            case 0: { QPS_NOTE_LAUNCH(); pair_fill_kernel<0, 1, false><<<grid, kThreads, 0, s>>>(d_tasks.p, tl, pool, g_near_table, d_err); } break;
            case 1: { QPS_NOTE_LAUNCH(); pair_fill_kernel<0, 2, false><<<grid, kThreads, 0, s>>>(d_tasks.p, tl, pool, g_near_table, d_err); } break;
            case 2: { QPS_NOTE_LAUNCH(); pair_fill_kernel<1, 1, false><<<grid, kThreads, 0, s>>>(d_tasks.p, tl, pool, g_near_table, d_err); } break;
            case 3: { QPS_NOTE_LAUNCH(); pair_fill_kernel<1, 2, false><<<grid, kThreads, 0, s>>>(d_tasks.p, tl, pool, g_near_table, d_err); } break;
            case 4: { QPS_NOTE_LAUNCH(); pair_fill_kernel<2, 1, false><<<grid, kThreads, 0, s>>>(d_tasks.p, tl, pool, g_near_table, d_err); } break;
            case 5: { QPS_NOTE_LAUNCH(); pair_fill_kernel<2, 2, false><<<grid, kThreads, 0, s>>>(d_tasks.p, tl, pool, g_near_table, d_err); } break;
            case 6: { QPS_NOTE_LAUNCH(); pair_fill_kernel<0, 1, true><<<grid, kThreads, 0, s>>>(d_tasks.p, tl, pool, g_near_table, d_err); } break;
            case 7: { QPS_NOTE_LAUNCH(); pair_fill_kernel<0, 2, true><<<grid, kThreads, 0, s>>>(d_tasks.p, tl, pool, g_near_table, d_err); } break;
            case 8: { QPS_NOTE_LAUNCH(); pair_fill_kernel<1, 1, true><<<grid, kThreads, 0, s>>>(d_tasks.p, tl, pool, g_near_table, d_err); } break;
            default: { QPS_NOTE_LAUNCH(); pair_fill_kernel<1, 2, true><<<grid, kThreads, 0, s>>>(d_tasks.p, tl, pool, g_near_table, d_err); } break;
        }
        QPS_CUDA(cudaGetLastError());
    }
}

void launch_proxy_fill(const std::vector<ProxyTask>& tasks, const DevPool& pool, int* d_err, cudaStream_t s,
                       DBuf<ProxyTask>& d_tasks, DBuf<int4>& d_tiles) {
    if (tasks.empty()) return;
    std::vector<int4> tiles;
    build_tiles<ProxyTask>(tasks, tiles, [](const ProxyTask& t) { return t.P; });
    if (tiles.empty()) return;
    d_tasks.upload(tasks, s);
    d_tiles.upload(tiles, s);
    double ev = 0;
    for (const auto& t : tasks) ev += double(t.nt) * t.P * t.nterm;
    ProfScope ps("fill_proxy", s, 200.0 * ev, 0.0, ev);
    { QPS_NOTE_LAUNCH(); proxy_fill_kernel<<<unsigned(tiles.size()), kThreads, 0, s>>>(d_tasks.p, d_tiles.p, pool, g_near_table, d_err); }
    QPS_CUDA(cudaGetLastError());
}

void launch_alpert(const std::vector<AlpertTask>& tasks, int total_rows, const DevPool& pool,
                   const SegDesc* d_segs, const double* d_fourier, const double* d_aux, int* d_err, cudaStream_t s,
                   DBuf<AlpertTask>& d_tasks) {
    if (tasks.empty() || total_rows == 0) return;
    d_tasks.upload(tasks, s);
    const int blocks = std::min((total_rows + 3) / 4, 148 * 16);
    const double ev = 2.0 * 30.0 * total_rows;
    ProfScope ps("fill_alpert", s, 200.0 * ev, 0.0, ev);
    { QPS_NOTE_LAUNCH(); alpert_kernel<<<blocks, 128, 0, s>>>(d_tasks.p, int(tasks.size()), total_rows, pool, d_segs, d_fourier,
                                         d_aux, g_near_table, d_err); }
    QPS_CUDA(cudaGetLastError());
}

void launch_hankel_batch(int n, const double* d_x, cplx* d_h0, cplx* d_h1, cudaStream_t s) {
    if (n <= 0) return;
    const int blocks = std::min((n + 255) / 256, 148 * 8);
    ProfScope ps("hankel", s, 140.0 * n, 0.0, n);
    { QPS_NOTE_LAUNCH(); hankel_batch_kernel<<<blocks, 256, 0, s>>>(n, d_x, d_h0, d_h1, g_near_table); }
    QPS_CUDA(cudaGetLastError());
}

}  // namespace qpsb
