// Block cyclic reduction with low-rank couplings.
//
// The off-diagonal blocks of the periodized system, A'_{j,j+1} and A'_{j+1,j}
// (interface-to-interface interactions across one layer, minus the rank-P
// proxy correction), are numerically low rank: at config 4 (interfaces one
// period apart, k up to 30) their singular values fall to the fill's rounding
// (~6e-16 of the largest) after ~35 of 600 (tools/coupling_rank.py).  Each
// coupling is compressed once from a sample Y = C Omega (Omega a 64-column
// sparse sign map, sparse_sketch_kernel) by a randomized row interpolative
// decomposition (lr_id_kernel): C ~= L (L1^{-1} C[I, :]) with the r = 48
// skeleton rows I of an LU with partial pivoting of Y, L its unit-lower factor
// (|L| <= 1), rank test at a relative pivot of 1e-12 (rank > 48 -> dense
// reduction) and an a-posteriori probe on 16 random columns (1e-12).
// (QPS_LR_ID=0 keeps the orthonormal form C ~= P (P^* C) from a blocked
// Householder QR and column-pivoted QR of the sample, rank at 1e-14.)
//
// Cyclic reduction then never forms a dense D^{-1} L or D^{-1} U: with
// L = P_L R_L and U = P_U R_U (P the left factor, R the r x n right factor) an
// odd elimination needs
//   Z = D_o^{-1} [P_L P_U]                   (n x 2r solve instead of n x 2n)
//   D_e -= P_L (R_L Z_U) R_U + P_U (R_U Z_L) R_L       (rank-r updates)
//   L'_e = P_L (-(R_L Z_L) R_L(o))  U'_e = P_U (-(R_U Z_U) R_U(o))
// so fill-in couplings keep the left factor of the even block and a new r x n
// right factor, and the work per elimination drops from 50.7 n^3 to about
// n^3 (8/3 + 32 r/n) real flops -- the LU of D_o dominates.  Back-substitution:
//   eta_o = z_o - Z_L (R_L(o) eta_{o-1}) - Z_U (R_U(o) eta_{o+1}).
// The default solve (bcr_solve_wb) runs this through the Woodbury identity:
// every diagonal block is LU-factored once at level 0 and the deeper levels
// only solve 2r x 2r capacitance systems.
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>

#include <nvtx3/nvToolsExt.h>

#include "cmath.cuh"
#include "ctx.h"
#include "prof.h"

namespace qpsb {

namespace {

constexpr int kLrSample = 64;    // columns of the random sample the basis is built from
// a-posteriori test of every compressed coupling on an independent probe: 16
// seeded random columns J of C (a coordinate-vector sample; kernel matrices
// spread their residual over all columns), ||C[:,J] - P (P^* C[:,J])||_F <=
// tol ||C[:,J]||_F; a failure takes the dense reduction.  Gathering columns
// costs no GEMM over C.
constexpr int kLrProbe = 16;
constexpr int kLrCols = kLrSample;  // columns of Omega and of the sample Y
// rcond screen of the Woodbury level-0 factors (tridiag.hpp:36-40): kRcProbe
// fixed unit-modulus probe columns ride along the level-0 right-hand sides;
// blocks whose certified upper bound on rcond is <= kRcSuspect get the full
// zlacn2 estimate
constexpr int kRcProbe = 4;
constexpr double kRcSuspect = 1e-10;
constexpr double kLrProbeTol = 1e-12;
constexpr int kLrMaxRank = 48;   // beyond this the dense reduction is used
// width of the compressed bases (>= any accepted rank; QPS_LR_BASIS overrides, <= kLrSample)
int lr_basis() {
    static const int b = [] {
        const char* e = getenv("QPS_LR_BASIS");
        return e ? std::max(kLrMaxRank, std::min(kLrSample, atoi(e))) : kLrMaxRank;
    }();
    return b;
}
constexpr double kLrTol = 1e-14; // relative pivot threshold of the sample's CPQR (QPS_LR_ID=0 path)
// row ID: relative pivot threshold of the sample's LU.  The couplings' singular
// values level off at the fill's rounding (~6e-16 of the largest) and the LU
// pivots of that noise at ~1e-14; the a-posteriori probe tolerance is 1e-12
constexpr double kIdTol = 1e-12;

// P_b = first r columns of Q (Q^* = H_{r-1} ... H_0 as applied by the CPQR, so
// Q e_c = H_0^* ... H_c^* e_c), and PH_b = P_b^*.  One warp per column.
__global__ void __launch_bounds__(256) lr_form_q_kernel(int m, int p, int r, const cplx* __restrict__ W,
                                                        const cplx* __restrict__ tau, cplx* __restrict__ P, int ldp,
                                                        size_t pstride, cplx* __restrict__ PH, size_t phstride) {
    extern __shared__ cplx lrv[];  // 8 warps x m
    const int b = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const cplx* Wb = W + size_t(b) * m * p;
    const cplx* tb = tau + size_t(b) * p;
    cplx* v = lrv + size_t(warp) * m;
    for (int c = blockIdx.y * 8 + warp; c < r; c += gridDim.y * 8) {
        for (int i = lane; i < m; i += 32) v[i] = cplx{i == c ? 1.0 : 0.0, 0.0};
        __syncwarp();
        for (int k = min(c, p - 1); k >= 0; --k) {
            const cplx tk = tb[k];
            if (tk.re == 0.0 && tk.im == 0.0) continue;
            // t = w^* v, w = [0..0, 1, W[k+1.., k]]
            cplx t{0, 0};
            for (int i = k + 1 + lane; i < m; i += 32) {
                const cplx e = Wb[size_t(k) * m + i];
                const cplx a = v[i];
                t.re += e.re * a.re + e.im * a.im;
                t.im += e.re * a.im - e.im * a.re;
            }
            for (int o = 16; o > 0; o >>= 1) {
                t.re += __shfl_xor_sync(0xffffffffu, t.re, o);
                t.im += __shfl_xor_sync(0xffffffffu, t.im, o);
            }
            const cplx vk = v[k];
            t.re += vk.re;
            t.im += vk.im;
            // v -= conj(tau) w t
            const cplx ct{tk.re * t.re + tk.im * t.im, tk.re * t.im - tk.im * t.re};
            __syncwarp();
            if (lane == 0) {
                v[k].re -= ct.re;
                v[k].im -= ct.im;
            }
            for (int i = k + 1 + lane; i < m; i += 32) {
                const cplx e = Wb[size_t(k) * m + i];
                v[i].re -= e.re * ct.re - e.im * ct.im;
                v[i].im -= e.re * ct.im + e.im * ct.re;
            }
            __syncwarp();
        }
        cplx* pc = P + size_t(b) * pstride + size_t(c) * ldp;
        cplx* ph = PH + size_t(b) * phstride;
        for (int i = lane; i < m; i += 32) {
            const cplx x = v[i];
            pc[i] = x;
            ph[size_t(i) * r + c] = cplx{x.re, -x.im};
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// Blocked Householder QR of the samples (m x 64, m <= 640): four 16-column
// panels, each factored in shared memory with one thread per row (one block
// reduction per column, combining the trailing-column products and the
// compact-WY inner products), trailing updates as batched GEMMs with the
// compact WY form H_15..H_0 = I - V T^* V^* (T upper triangular, LAPACK larft
// on the conjugate reflectors).  The 64 x 64 R is then factored with column
// pivoting (rank, ordering) and the basis P = Q Q2[:, :48] is formed by
// applying the four block reflectors to [Q2; 0] -- every pass over the tall
// sample is a GEMM, none streams it once per column.
// ---------------------------------------------------------------------------
constexpr int kQrW = 16;
__global__ void __launch_bounds__(640, 1) qr_panel_kernel(int m, cplx* __restrict__ Y, size_t ystride, int col0,
                                                          cplx* __restrict__ V, cplx* __restrict__ VH,
                                                          cplx* __restrict__ T, cplx* __restrict__ TH,
                                                          size_t vstride, size_t tstride) {
    // Per column k: warp 0 forms the tail norm and the Householder scalars;
    // one warp per inner product -- s_j = v_k^* a_j for the panel columns to
    // the right, z_l = v_l^* v_k for the compact-WY factor -- each a single
    // warp reduction (the thread-per-row layout would need 16 block
    // reductions); then every thread applies H_k to its own row.
    extern __shared__ cplx qp[];  // [kQrW][m]
    const int b = blockIdx.x;
    cplx* Yb = Y + size_t(b) * ystride;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5;
    __shared__ cplx dots[kQrW + 1];  // s_j (j > k), z_l (l < k) and the tail norm of the current column
    __shared__ cplx s_tau, s_inv, s_beta;
    __shared__ cplx Ts[kQrW][kQrW];  // T~[row][col]
    const bool own = tid < m;
    if (own)
        for (int j = 0; j < kQrW; ++j) qp[j * m + tid] = Yb[size_t(col0 + j) * m + tid];
    __syncthreads();
    // v_j at row i, rebuilt from the panel (qp holds v_j below the diagonal)
    auto vat = [&](int j, int i) -> cplx {
        const int d = col0 + j;
        if (i < d) return cplx{0, 0};
        if (i == d) return cplx{1.0, 0.0};
        return qp[j * m + i];
    };
    for (int k = 0; k < kQrW; ++k) {
        const int g0 = col0 + k;
        // phase 1, one warp per task over rows > g0 with the raw column a_k
        // (v_k = a_k / den below the diagonal, so the scale is applied after):
        // tasks 0..14-k: raw_j = a_k^* a_j (j > k); next k: raw_l = v_l^* a_k
        // (l < k); task 15: the tail norm |a_k|^2
        for (int task = warp; task < kQrW; task += nwarp) {
            const int nright = kQrW - 1 - k;
            cplx acc{0, 0};
            if (task == kQrW - 1) {
                for (int i = g0 + 1 + lane; i < m; i += 32) acc.re += cabs2(qp[k * m + i]);
            } else {
                const bool right = task < nright;
                const int c = right ? k + 1 + task : task - nright;
                for (int i = g0 + 1 + lane; i < m; i += 32) {
                    const cplx ak = qp[k * m + i];
                    const cplx a = qp[c * m + i];  // a_j, or v_l (i > g0 lies below v_l's unit entry)
                    if (right) {  // conj(a_k) a_j
                        acc.re += ak.re * a.re + ak.im * a.im;
                        acc.im += ak.re * a.im - ak.im * a.re;
                    } else {      // conj(v_l) a_k
                        acc.re += a.re * ak.re + a.im * ak.im;
                        acc.im += a.re * ak.im - a.im * ak.re;
                    }
                }
            }
            for (int o = 16; o > 0; o >>= 1) {
                acc.re += __shfl_xor_sync(0xffffffffu, acc.re, o);
                acc.im += __shfl_xor_sync(0xffffffffu, acc.im, o);
            }
            if (lane == 0) dots[task == kQrW - 1 ? kQrW : (task < nright ? k + 1 + task : task - nright)] = acc;
        }
        __syncthreads();
        // phase 2 (warp 0): Householder scalars, scaled inner products, T~ column k
        if (warp == 0) {
            if (lane == 0) {
                const double t2 = dots[kQrW].re;
                const cplx c0 = qp[k * m + g0];
                if (t2 <= DBL_MIN && c0.im * c0.im <= DBL_MIN) {  // makeHouseholder's no-op case
                    s_tau = cplx{0, 0};
                    s_beta = c0;
                    s_inv = cplx{0, 0};
                } else {
                    double beta = sqrt(cabs2(c0) + t2);
                    if (c0.re >= 0.0) beta = -beta;
                    s_inv = fast_cinv(cplx{c0.re - beta, c0.im});
                    const double rb = fast_rcp(beta);
                    s_tau = cplx{(beta - c0.re) * rb, c0.im * rb};  // conj((beta - c0) / beta)
                    s_beta = cplx{beta, 0.0};
                }
            }
            __syncwarp();
            const cplx inv = s_inv;
            if (lane < kQrW && lane != k) {
                const cplx raw = dots[lane];
                if (lane > k) {  // s_j = conj(inv) raw + a_j[g0]
                    const cplx t = cmul(cconj(inv), raw);
                    const cplx a0 = qp[lane * m + g0];
                    dots[lane] = cplx{t.re + a0.re, t.im + a0.im};
                } else {         // z_l = inv raw + conj(v_l[g0])
                    const cplx t = cmul(inv, raw);
                    const cplx vl = vat(lane, g0);
                    dots[lane] = cplx{t.re + vl.re, t.im - vl.im};
                }
            }
            __syncwarp();
            if (lane < kQrW) {  // T~[k][k] = conj(tau), T~[0:k, k] = -conj(tau) T~[0:k,0:k] z
                const int l = lane;
                const cplx ct = cconj(s_tau);
                cplx val{0, 0};
                if (l < k) {
                    cplx acc{0, 0};
                    for (int q = l; q < k; ++q) {
                        const cplx t = cmul(Ts[l][q], dots[q]);
                        acc.re += t.re;
                        acc.im += t.im;
                    }
                    const cplx u = cmul(ct, acc);
                    val = cplx{-u.re, -u.im};
                } else if (l == k) {
                    val = ct;
                }
                Ts[l][k] = val;
            }
        }
        __syncthreads();
        // phase 3: apply H_k = I - tau v v^* to this row of the panel columns j > k
        const cplx tau = s_tau, inv = s_inv;
        if (own && tid >= g0) {
            const cplx vk = (tid == g0) ? cplx{1.0, 0.0} : cmul(qp[k * m + tid], inv);
            qp[k * m + tid] = (tid == g0) ? s_beta : vk;
            if (!(tau.re == 0.0 && tau.im == 0.0))
                for (int j = k + 1; j < kQrW; ++j) {
                    const cplx d = cmul(cmul(tau, dots[j]), vk);
                    qp[j * m + tid].re -= d.re;
                    qp[j * m + tid].im -= d.im;
                }
        }
        __syncthreads();
    }
    // write back R (rows <= diag) and the explicit V / V^*, T~ and T~^*
    cplx* Vb = V + size_t(b) * vstride;
    cplx* VHb = VH + size_t(b) * vstride;
    if (own) {
#pragma unroll
        for (int j = 0; j < kQrW; ++j) {
            Yb[size_t(col0 + j) * m + tid] = (tid <= col0 + j) ? qp[j * m + tid] : cplx{0, 0};
            const cplx vj = vat(j, tid);
            Vb[size_t(j) * m + tid] = vj;
            VHb[size_t(tid) * kQrW + j] = cconj(vj);
        }
    }
    if (tid < kQrW * kQrW) {
        const int r = tid % kQrW, c = tid / kQrW;
        T[size_t(b) * tstride + size_t(c) * kQrW + r] = Ts[r][c];
        TH[size_t(b) * tstride + size_t(c) * kQrW + r] = cconj(Ts[c][r]);
    }
}

// top 64 x 64 (upper triangle) of each factored sample; zeros below
__global__ void qr_take_r_kernel(int m, int p, const cplx* __restrict__ Y, size_t ystride, cplx* __restrict__ R) {
    const int b = blockIdx.x;
    for (int e = threadIdx.x; e < p * p; e += blockDim.x) {
        const int i = e % p, j = e / p;
        R[size_t(b) * p * p + e] = i <= j ? Y[size_t(b) * ystride + size_t(j) * m + i] : cplx{0, 0};
    }
}

// X = [Q2 (p x r); 0] (m x r), and its conjugate transpose later
// Compact-WY merge of nb panels of width kQrW (zlarft's block recurrence):
// T (64 x 64, upper triangular) from the panels' own T_k (kQrW x kQrW, at
// Tp + k kQrW^2 per problem, stride tpstride) and G = V^* V (only its blocks
// G_ij, i < j, are read; column-major, ld 64):
//   T_kk = T_k,  T_{0:k, k} = -T_{0:k, 0:k} (G_{0:k, k} T_k).
__global__ void __launch_bounds__(256) wy_merge_kernel(int nb, const cplx* __restrict__ Tp, size_t tpstride,
                                                       const cplx* __restrict__ G, cplx* __restrict__ Tout) {
    constexpr int W = kQrW, P = 4 * kQrW;
    extern __shared__ cplx wy_sm[];
    cplx (*T)[P + 1] = reinterpret_cast<cplx (*)[P + 1]>(wy_sm);            // T[row][col]
    cplx (*M)[W + 1] = reinterpret_cast<cplx (*)[W + 1]>(wy_sm + P * (P + 1));  // G_{0:k,k} T_k
    const int b = blockIdx.x, tid = threadIdx.x;
    const int n = nb * W;
    const cplx* Gb = G + size_t(b) * P * P;
    for (int e = tid; e < n * n; e += blockDim.x) {
        const int r = e % n, cc = e / n;
        const int kb = cc / W;
        cplx v{0, 0};
        if (r / W == kb) v = Tp[size_t(b) * tpstride + size_t(kb) * W * W + size_t(cc % W) * W + (r % W)];
        T[r][cc] = v;
    }
    __syncthreads();
    for (int k = 1; k < nb; ++k) {
        const int rows = k * W;
        for (int e = tid; e < rows * W; e += blockDim.x) {  // M = G_{0:k,k} T_k
            const int r = e % rows, j = e / rows;
            cplx acc{0, 0};
            for (int q = 0; q < W; ++q) {
                const cplx g = Gb[size_t(k * W + q) * P + r];
                const cplx t = T[k * W + q][k * W + j];
                acc.re += g.re * t.re - g.im * t.im;
                acc.im += g.re * t.im + g.im * t.re;
            }
            M[r][j] = acc;
        }
        __syncthreads();
        for (int e = tid; e < rows * W; e += blockDim.x) {  // T_{0:k,k} = -T_{0:k,0:k} M
            const int r = e % rows, j = e / rows;
            cplx acc{0, 0};
            for (int q = r; q < rows; ++q) {  // T_{0:k,0:k} is upper triangular
                const cplx t = T[r][q];
                const cplx mm = M[q][j];
                acc.re += t.re * mm.re - t.im * mm.im;
                acc.im += t.re * mm.im + t.im * mm.re;
            }
            T[r][k * W + j] = cplx{-acc.re, -acc.im};
        }
        __syncthreads();
    }
    for (int e = tid; e < P * P; e += blockDim.x) {
        const int r = e % P, cc = e / P;
        Tout[size_t(b) * P * P + e] = (r < n && cc < n) ? T[r][cc] : cplx{0, 0};
    }
}

__global__ void qr_seed_kernel(int m, int p, int r, const cplx* __restrict__ Q2, size_t q2stride,
                               cplx* __restrict__ X, size_t xstride) {
    const int b = blockIdx.x;
    for (size_t e = threadIdx.x; e < size_t(m) * r; e += blockDim.x) {
        const int i = int(e % m), j = int(e / m);
        X[size_t(b) * xstride + e] = i < p ? Q2[size_t(b) * q2stride + size_t(j) * p + i] : cplx{0, 0};
    }
}

// XH = X^* per problem (X m x r column-major, XH r x m): a CTA owns 32 rows of X,
// staged through shared memory so that both the read (down X's columns) and
// the write (XH's 32 consecutive columns = one contiguous 32 r range) coalesce
constexpr int kCtRows = 32, kCtMaxR = 64;
static_assert(kLrMaxRank <= kCtMaxR, "conj_transpose_kernel: basis wider than its tile");
__global__ void __launch_bounds__(256) conj_transpose_kernel(int m, int r, const cplx* __restrict__ X,
                                                             size_t xstride, cplx* __restrict__ XH, size_t hstride) {
    __shared__ cplx tile[kCtMaxR][kCtRows + 1];
    const int b = blockIdx.y, i0 = blockIdx.x * kCtRows;
    const int rows = min(kCtRows, m - i0);
    const cplx* Xb = X + size_t(b) * xstride;
    cplx* Hb = XH + size_t(b) * hstride + size_t(i0) * r;
    for (int e = threadIdx.x; e < kCtRows * r; e += blockDim.x) {
        const int ii = e % kCtRows, j = e / kCtRows;
        if (ii < rows) tile[j][ii] = Xb[size_t(j) * m + i0 + ii];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < rows * r; e += blockDim.x) {
        const int ii = e / r, j = e % r;
        Hb[e] = cconj(tile[j][ii]);
    }
}

// C_b = I (n x n, column-major, stride n^2)
__global__ void set_identity_kernel(int n, cplx* __restrict__ C) {
    cplx* Cb = C + size_t(blockIdx.x) * n * n;
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) Cb[e] = cplx{(e % n == e / n) ? 1.0 : 0.0, 0.0};
}

// W_j = [P_L(j) P_U(j) f_j] (zeros where a coupling is absent; f_j the n-vector
// of block j, ld n) for every block j of every system, so that one solve
// gives D^{-1} [P_L P_U] and D^{-1} f; P holds per system the I-1 sub- then
// the I-1 super-couplings
// W_j = [P_L | P_U | F_j | R] (n x (2r + m + nprobe)): the level-0 right-hand sides
__global__ void stage_bases_kernel(int I, int n, size_t per, const cplx* __restrict__ P, const cplx* __restrict__ F,
                                   int m, const cplx* __restrict__ R, int nprobe, cplx* __restrict__ W) {
    const int j = blockIdx.x, a = j / I, jj = j % I;
    const size_t qa = size_t(a) * 2 * (I - 1);
    const cplx* pl = jj >= 1 ? P + (qa + (jj - 1)) * per : nullptr;
    const cplx* pu = jj + 1 < I ? P + (qa + (I - 1) + jj) * per : nullptr;
    const size_t nf = size_t(n) * m, nr = size_t(n) * nprobe;
    cplx* w = W + size_t(j) * (2 * per + nf + nr);
    const size_t tot = per > nf ? (per > nr ? per : nr) : (nf > nr ? nf : nr);
    for (size_t e = size_t(blockIdx.y) * blockDim.x + threadIdx.x; e < tot; e += size_t(gridDim.y) * blockDim.x) {
        if (e < per) {
            w[e] = pl ? pl[e] : cplx{0, 0};
            w[per + e] = pu ? pu[e] : cplx{0, 0};
        }
        if (e < nf) w[2 * per + e] = F[size_t(j) * nf + e];
        if (e < nr) w[2 * per + nf + e] = R[e];
    }
}

// In-place inverse of each n x n matrix (n <= kGjMax, column-major, stride n^2) by
// Gauss-Jordan elimination with partial (row) pivoting, one CTA per matrix,
// the matrix resident in shared memory: n steps of (pivot search, row swap,
// scaled pivot row, rank-1 elimination of every other row), then the column
// interchanges undone in reverse.  flag[b] = 1 on an exactly zero pivot or
// when rcond(C) = 1 / (||C||_1 ||C^{-1}||_1) <= 1e-15 (the reference's
// PartialPivLU::rcond() test, tridiag.hpp:36-40, here exact: the inverse is
// formed).
constexpr int kGjMax = 112;  // 112^2 complex = 196 KB of shared memory
__global__ void __launch_bounds__(512) gj_inverse_kernel(int n, cplx* __restrict__ C, int* __restrict__ flag) {
    extern __shared__ cplx gj[];  // n x n, ld n
    __shared__ int s_piv[kGjMax];
    __shared__ cplx s_row[kGjMax], s_col[kGjMax];
    __shared__ double s_v[16];
    __shared__ int s_i[16];
    cplx* Cb = C + size_t(blockIdx.x) * n * n;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int e = tid; e < n * n; e += blockDim.x) gj[e] = Cb[e];
    __syncthreads();
    // ||C||_1 and, at the end, ||C^{-1}||_1: rcond(C), tridiag.hpp:36-40
    auto norm1 = [&]() {
        double v = 0;
        for (int jj = warp; jj < n; jj += blockDim.x / 32) {
            double cs = 0;
            for (int i = lane; i < n; i += 32) cs += hypot(gj[jj * n + i].re, gj[jj * n + i].im);
            for (int o = 16; o > 0; o >>= 1) cs += __shfl_xor_sync(0xffffffffu, cs, o);
            v = fmax(v, cs);
        }
        if (lane == 0) s_v[warp] = v;
        __syncthreads();
        double m = 0;
        for (int w = 0; w < int(blockDim.x / 32); ++w) m = fmax(m, s_v[w]);
        __syncthreads();
        return m;
    };
    const double cnorm = norm1();
    for (int k = 0; k < n; ++k) {
        // pivot: first row i >= k of largest modulus in column k
        double v = -1.0;
        int idx = 1 << 30;
        if (tid < n && tid >= k) {
            v = cabs2(gj[k * n + tid]);
            idx = tid;
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, v, o);
            const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
            if (ov > v || (ov == v && oi < idx)) {
                v = ov;
                idx = oi;
            }
        }
        if (lane == 0 && warp < 16) {
            s_v[warp] = v;
            s_i[warp] = idx;
        }
        __syncthreads();
        double bv = s_v[0];
        int p = s_i[0];
        for (int w = 1; w < (n + 31) / 32; ++w)
            if (s_v[w] > bv || (s_v[w] == bv && s_i[w] < p)) {
                bv = s_v[w];
                p = s_i[w];
            }
        if (tid == 0) {
            s_piv[k] = p;
            if (!(bv > 0.0)) flag[blockIdx.x] = 1;
        }
        if (p != k && tid < n) {  // swap rows k and p (thread = column)
            const cplx t = gj[tid * n + k];
            gj[tid * n + k] = gj[tid * n + p];
            gj[tid * n + p] = t;
        }
        __syncthreads();
        const cplx a = gj[k * n + k];
        const cplx inv = (a.re == 0.0 && a.im == 0.0) ? cplx{0, 0} : cdiv(cplx{1.0, 0.0}, a);
        if (tid < n) {
            s_row[tid] = (tid == k) ? inv : cmul(gj[tid * n + k], inv);
            s_col[tid] = (tid == k) ? cplx{0, 0} : gj[k * n + tid];
        }
        __syncthreads();
        for (int e = tid; e < n * n; e += blockDim.x) {
            const int i = e % n, j = e / n;
            if (i == k) {
                gj[e] = s_row[j];
            } else {
                const cplx f = s_col[i], r = s_row[j];
                cplx x = (j == k) ? cplx{0, 0} : gj[e];
                x.re -= f.re * r.re - f.im * r.im;
                x.im -= f.re * r.im + f.im * r.re;
                gj[e] = x;
            }
        }
        __syncthreads();
    }
    for (int k = n - 1; k >= 0; --k) {  // A^{-1} = (P A)^{-1} P: swap columns k, piv[k]
        const int p = s_piv[k];
        if (p != k && tid < n) {
            const cplx t = gj[k * n + tid];
            gj[k * n + tid] = gj[p * n + tid];
            gj[p * n + tid] = t;
        }
        __syncthreads();
    }
    const double inorm = norm1();
    if (tid == 0 && !(1.0 / (cnorm * inorm) > kRcondMin)) flag[blockIdx.x] = 1;
    for (int e = tid; e < n * n; e += blockDim.x) Cb[e] = gj[e];
}

// Register-resident variant (default): thread (j, g) = (tid / 4, tid % 4) keeps
// rows g, g + 4, ... of column j in registers for the whole elimination.  No
// physical row interchanges: step k pivots on the largest-modulus unused row
// p_k of column k and applies the Jordan exchange
//   T[p][k] = 1/a,  T[p][j] = -T[p][j]/a,  T[i][k] = T[i][k]/a,
//   T[i][j] -= T[i][k] T[p][j]/a          (a = T[p][k]),
// after which A^{-1}[k][p_k'] = T[p_k][k'] (rows and columns permuted on the
// way out).  Two barriers per step; the pivot's reciprocal is computed once.
// N (a multiple of 4) fixed at compile time: every guard folds away and the
// row loops are straight-line (96 x 96 capacitance matrices, 2r = 96).
// Thread layout tid = g N + j: a warp holds one row class g (rows g, g + 4,
// ...) of 32 columns, so "owns the pivot row" is warp-uniform and the s_col
// reads are warp-wide broadcasts; the pivot search reduces the column's four
// row classes through shared memory and every thread then computes the pivot's
// reciprocal itself (one barrier saved).
template <int N>
__global__ void __launch_bounds__(4 * N) gj_inverse_reg_kernel(cplx* __restrict__ C, int* __restrict__ flag) {
    constexpr int NR = N / 4;
    static_assert(N % 16 == 0 && NR <= 32, "gj_inverse_reg_kernel: N a multiple of 16, N <= 128");
    __shared__ cplx s_row[N], s_col[2][N];  // s_col double-buffered: written before the first barrier
    __shared__ int s_perm[N], s_pinv[N];
    __shared__ double s_cv[2][4];
    __shared__ int s_ci[2][4];
    __shared__ cplx s_ca[2][4];
    __shared__ double s_nm[4 * N / 32];
    cplx* Cb = C + size_t(blockIdx.x) * N * N;
    const int tid = threadIdx.x, g = tid / N, j = tid % N;
    // ||C||_1 = max column sum, read from global memory before (and, for
    // ||C^{-1}||_1, after) the register-resident elimination: rcond(C) for the
    // reference's test, tridiag.hpp:36-40
    auto norm1 = [&]() {
        double v = 0;
        for (int jj = tid >> 5; jj < N; jj += 4 * N / 32) {
            double cs = 0;
            for (int i = tid & 31; i < N; i += 32) cs += sqrt(cabs2(Cb[size_t(jj) * N + i]));  // |z| (no hypot: magnitudes are tame)
            for (int o = 16; o > 0; o >>= 1) cs += __shfl_xor_sync(0xffffffffu, cs, o);
            v = fmax(v, cs);
        }
        if ((tid & 31) == 0) s_nm[tid >> 5] = v;
        __syncthreads();
        double m = 0;
        for (int w = 0; w < 4 * N / 32; ++w) m = fmax(m, s_nm[w]);
        return m;
    };
    const double cnorm = norm1();
    cplx T[NR];
    unsigned used = 0;  // bit ii: row g + 4 ii already pivotal
#pragma unroll
    for (int ii = 0; ii < NR; ++ii) T[ii] = Cb[size_t(j) * N + g + 4 * ii];
    for (int k = 0; k < N; ++k) {
        const int par = k & 1;
        const bool colk = (j == k);
        if (colk) {  // this row class's candidate in column k
            double v = -1.0;
            int idx = 1 << 30;
            cplx a{0, 0};
#pragma unroll
            for (int ii = 0; ii < NR; ++ii) {
                const double m = cabs2(T[ii]);
                const bool better = !((used >> ii) & 1u) && m > v;
                v = better ? m : v;
                idx = better ? g + 4 * ii : idx;
                a.re = better ? T[ii].re : a.re;
                a.im = better ? T[ii].im : a.im;
            }
            s_cv[par][g] = v;
            s_ci[par][g] = idx;
            s_ca[par][g] = a;
#pragma unroll
            for (int ii = 0; ii < NR; ++ii) s_col[par][g + 4 * ii] = T[ii];
        }
        __syncthreads();
        double bv = s_cv[par][0];
        int p = s_ci[par][0], bg = 0;
#pragma unroll
        for (int q = 1; q < 4; ++q) {
            const double v = s_cv[par][q];
            const int i = s_ci[par][q];
            const bool better = v > bv || (v == bv && i < p);
            bv = better ? v : bv;
            p = better ? i : p;
            bg = better ? q : bg;
        }
        const cplx a = s_ca[par][bg];
        const bool zero = !(bv > 0.0);
        const cplx inv = zero ? cplx{0, 0} : fast_cinv(a);
        const int pr = p >> 2;
        const bool own_p = g == (p & 3);  // warp-uniform
        if (own_p) {
            cplx rv{0, 0};
#pragma unroll
            for (int ii = 0; ii < NR; ++ii) {
                rv.re = (ii == pr) ? T[ii].re : rv.re;
                rv.im = (ii == pr) ? T[ii].im : rv.im;
            }
            s_row[j] = rv;
        }
        if (tid == 0) {
            if (zero) flag[blockIdx.x] = 1;
            s_perm[k] = p;
            s_pinv[p] = k;
        }
        __syncthreads();
        if (colk) {  // T[i][k] = T[i][k] / a, T[p][k] = 1 / a
#pragma unroll
            for (int ii = 0; ii < NR; ++ii) {
                const cplx c = s_col[par][g + 4 * ii];
                const bool piv = own_p && ii == pr;
                T[ii].re = piv ? inv.re : c.re * inv.re - c.im * inv.im;
                T[ii].im = piv ? inv.im : c.re * inv.im + c.im * inv.re;
            }
        } else {
            const cplx r = cmul(s_row[j], inv);
            if (own_p) {
#pragma unroll
                for (int ii = 0; ii < NR; ++ii) {
                    const cplx c = s_col[par][g + 4 * ii];
                    const double bre = T[ii].re - (c.re * r.re - c.im * r.im);
                    const double bim = T[ii].im - (c.re * r.im + c.im * r.re);
                    T[ii].re = (ii == pr) ? -r.re : bre;
                    T[ii].im = (ii == pr) ? -r.im : bim;
                }
            } else {
#pragma unroll
                for (int ii = 0; ii < NR; ++ii) {
                    const cplx c = s_col[par][g + 4 * ii];
                    T[ii].re -= c.re * r.re - c.im * r.im;
                    T[ii].im -= c.re * r.im + c.im * r.re;
                }
            }
        }
        used |= own_p ? (1u << pr) : 0u;
    }
    __syncthreads();
    const int col = s_perm[j];  // A^{-1}[pinv[i]][perm[j]] = T[i][j]
#pragma unroll
    for (int ii = 0; ii < NR; ++ii) Cb[size_t(col) * N + s_pinv[g + 4 * ii]] = T[ii];
    __syncthreads();  // the block's global writes are visible to it after the barrier
    const double inorm = norm1();
    if (tid == 0 && !(1.0 / (cnorm * inorm) > kRcondMin)) flag[blockIdx.x] = 1;
}

// ---------------------------------------------------------------------------
// Interpolative compression of the couplings (randomized row ID).
//
// From the sample Y = C Omega (m x 64) an LU with partial pivoting selects 64
// pivot rows; the first r of them are the skeleton rows I, and
//   C ~= L (L1^{-1} C[I, :]),   L = the first r columns of the unit lower
// factor (original row order, |L| <= 1), L1 = L[I, :] (unit lower triangular).
// The row relations that reproduce Y from Y[I, :] reproduce C from C[I, :]
// (Y's rows are C's rows times Omega): the residual on Y is the Schur
// complement after r steps, and the a-posteriori probe tests C itself.  The
// right factor needs only the r gathered rows of C -- no projection GEMM over
// the couplings (the orthonormal form P (P^* C) read all of C a second time).
//
// lr_id_kernel: one CTA per coupling, one thread per row of Y (m <= 640),
// 16-column panels in registers.  Rows are never interchanged: each thread
// remembers the step at which its row became a pivot, a pivot search runs over
// the rows not yet chosen, and the trailing columns of the rows still live are
// updated in place in Y through U12 = L11^{-1} Y[pivots, later columns].
// ---------------------------------------------------------------------------
constexpr int kIdW = 8;                        // panel width
constexpr int kIdThreads = 640;                // one thread per sample row
constexpr int kIdWarps = kIdThreads / 32;
constexpr int kIdPanels = kLrSample / kIdW;
static_assert(kLrSample % kIdW == 0, "lr_id_kernel: sample width is a multiple of the panel");
size_t id_smem_bytes(int r) {
    return (size_t(2) * kIdWarps * kIdW + size_t(kIdW) * kLrSample + size_t(kIdW) * kIdW + size_t(r) * (r + 1)) *
           sizeof(cplx);
}

__global__ void __launch_bounds__(kIdThreads, 1)
    lr_id_kernel(int m, cplx* __restrict__ Y, size_t ys, int r, cplx* __restrict__ Lo, size_t lstride,
                 cplx* __restrict__ L1i, int* __restrict__ piv_out, int* __restrict__ rank_out, double tol) {
    extern __shared__ cplx id_sm[];
    cplx* cand = id_sm;                       // [2][kIdWarps][kIdW] candidate pivot rows (panel columns)
    cplx* U12 = cand + 2 * kIdWarps * kIdW;   // [kIdW][kLrSample]
    cplx* L11 = U12 + kIdW * kLrSample;       // [kIdW][kIdW]
    cplx* L1 = L11 + kIdW * kIdW;             // [r][r + 1]
    __shared__ double cval[2][kIdWarps];
    __shared__ int cidx[2][kIdWarps];
    __shared__ double udiag[kLrSample];
    __shared__ int spiv[kLrSample];
    const int q = blockIdx.x;
    cplx* Yq = Y + size_t(q) * ys;
    cplx* Lq = Lo + size_t(q) * lstride;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool own = tid < m;
    int mystep = own ? (1 << 30) : -1;  // step at which this row became a pivot
    for (int p = 0; p < kIdPanels; ++p) {
        const int c0 = p * kIdW;
        cplx s[kIdW];
#pragma unroll
        for (int jj = 0; jj < kIdW; ++jj) s[jj] = own ? Yq[size_t(c0 + jj) * m + tid] : cplx{0, 0};
#pragma unroll
        for (int kk = 0; kk < kIdW; ++kk) {
            const int k = c0 + kk, par = kk & 1;
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
            if (idx == tid) {  // this warp's candidate publishes its panel row
                cplx* cr = cand + (par * kIdWarps + warp) * kIdW;
#pragma unroll
                for (int jj = kk; jj < kIdW; ++jj) cr[jj] = s[jj];
                cval[par][warp] = v;
                cidx[par][warp] = idx;
            } else if (lane == 0 && idx == (1 << 30)) {
                cval[par][warp] = -1.0;
                cidx[par][warp] = 1 << 30;
            }
            __syncthreads();
            double bv = lane < kIdWarps ? cval[par][lane] : -1.0;
            int bi = lane < kIdWarps ? cidx[par][lane] : (1 << 30);
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
            const cplx* prow = cand + (par * kIdWarps + bw) * kIdW;
            if (tid == 0) {
                spiv[k] = bi;
                udiag[k] = bv > 0.0 ? sqrt(bv) : 0.0;
            }
            if (tid == bi) mystep = k;
            if (live && tid != bi) {
                const cplx d = prow[kk];
                const bool zero = (d.re == 0.0 && d.im == 0.0);
                const cplx l = zero ? cplx{0, 0} : cmul(s[kk], fast_cinv(d));
                s[kk] = l;
#pragma unroll
                for (int jj = kk + 1; jj < kIdW; ++jj) {
                    const cplx u = prow[jj];
                    s[jj].re -= l.re * u.re - l.im * u.im;
                    s[jj].im -= l.re * u.im + l.im * u.re;
                }
            }
        }
        // left factor columns c0.. (< r): L values of live rows, the unit of
        // each pivot row at its own step, zero after it
        if (own) {
#pragma unroll
            for (int kk = 0; kk < kIdW; ++kk) {
                const int k = c0 + kk;
                if (k < r) {
                    const cplx v = mystep == k ? cplx{1, 0} : (mystep < k ? cplx{0, 0} : s[kk]);
                    Lq[size_t(k) * m + tid] = v;
                }
            }
        }
        if (p + 1 == kIdPanels) break;
        // L11 of this panel: row kk0 of the pivot chosen at step c0 + kk0
        const int kk0 = mystep - c0;
        if (own && kk0 >= 0 && kk0 < kIdW) {
#pragma unroll
            for (int kk = 0; kk < kIdW; ++kk)
                L11[kk0 * kIdW + kk] = kk < kk0 ? s[kk] : (kk == kk0 ? cplx{1, 0} : cplx{0, 0});
        }
        __syncthreads();
        // U12 = L11^{-1} Y[pivots of this panel, later columns] (one thread per column)
        const int ncol = kLrSample - c0 - kIdW;
        if (tid < ncol) {
            const size_t col = size_t(c0 + kIdW + tid) * m;
#pragma unroll 1
            for (int kk = 0; kk < kIdW; ++kk) {
                cplx a = Yq[col + spiv[c0 + kk]];
                for (int k2 = 0; k2 < kk; ++k2) {
                    const cplx lv = L11[kk * kIdW + k2], u = U12[k2 * kLrSample + tid];
                    a.re -= lv.re * u.re - lv.im * u.im;
                    a.im -= lv.re * u.im + lv.im * u.re;
                }
                U12[kk * kLrSample + tid] = a;
            }
        }
        __syncthreads();
        // trailing columns of the rows still live: Y[i, j] -= sum_kk L[i, kk] U12[kk, j]
        if (own && mystep >= c0 + kIdW) {
#pragma unroll 2
            for (int t = 0; t < ncol; ++t) {
                const size_t at = size_t(c0 + kIdW + t) * m + tid;
                cplx a = Yq[at];
#pragma unroll
                for (int kk = 0; kk < kIdW; ++kk) {
                    const cplx u = U12[kk * kLrSample + t];
                    a.re -= s[kk].re * u.re - s[kk].im * u.im;
                    a.im -= s[kk].re * u.im + s[kk].im * u.re;
                }
                Yq[at] = a;
            }
        }
        __syncthreads();
    }
    __syncthreads();  // the left factor's global writes are visible to the block
    // numerical rank: last pivot above tol x the largest
    if (tid == 0) {
        double mx = 0.0;
        for (int k = 0; k < kLrSample; ++k) mx = fmax(mx, udiag[k]);
        int rk = 0;
        for (int k = 0; k < kLrSample; ++k)
            if (udiag[k] > tol * mx) rk = k + 1;
        rank_out[q] = rk;
    }
    if (tid < r) piv_out[size_t(q) * r + tid] = spiv[tid];
    // L1 = L[I, :r] (unit lower), then its inverse column by column (one warp per column)
    for (int e = tid; e < r * r; e += kIdThreads) {
        const int t = e % r, t2 = e / r;
        L1[t * (r + 1) + t2] = Lq[size_t(t2) * m + spiv[t]];
    }
    __syncthreads();
    cplx* Li = L1i + size_t(q) * r * r;
    for (int c = warp; c < r; c += kIdWarps) {
        cplx x0 = lane == c ? cplx{1, 0} : cplx{0, 0};
        cplx x1 = lane + 32 == c ? cplx{1, 0} : cplx{0, 0};
        for (int tp = c; tp + 1 < r; ++tp) {
            const cplx src = tp < 32 ? x0 : x1;
            cplx xt;
            xt.re = __shfl_sync(0xffffffffu, src.re, tp & 31);
            xt.im = __shfl_sync(0xffffffffu, src.im, tp & 31);
            if (lane > tp && lane < r) {
                const cplx lv = L1[lane * (r + 1) + tp];
                x0.re -= lv.re * xt.re - lv.im * xt.im;
                x0.im -= lv.re * xt.im + lv.im * xt.re;
            }
            if (lane + 32 > tp && lane + 32 < r) {
                const cplx lv = L1[(lane + 32) * (r + 1) + tp];
                x1.re -= lv.re * xt.re - lv.im * xt.im;
                x1.im -= lv.re * xt.im + lv.im * xt.re;
            }
        }
        if (lane < r) Li[size_t(c) * r + lane] = x0;
        if (lane + 32 < r) Li[size_t(c) * r + lane + 32] = x1;
    }
}

// rows[q][0..nr) of src_q (ld lds_q) over ncols columns -> dst_q (nr x ncols, ld nr)
__global__ void __launch_bounds__(256) gather_rows_kernel(const cplx* const* __restrict__ src,
                                                          const int* __restrict__ lds, const int* __restrict__ rows,
                                                          int nr, int ncols, cplx* __restrict__ dst, size_t dstride) {
    const int q = blockIdx.y;
    const cplx* a = src[q];
    const size_t ld = size_t(lds[q]);
    const int* rw = rows + size_t(q) * nr;
    cplx* d = dst + size_t(q) * dstride;
    const int total = nr * ncols;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
        const int t = e % nr, j = e / nr;
        d[e] = a[size_t(j) * ld + rw[t]];
    }
}

// ---------------------------------------------------------------------------
// Sparse sign sketch: Y = alpha C Omega with Omega (ncols x 64) holding
// kSkZeta = 8 entries +-1 per row (each source column of C is added, with a
// sign, to 8 of the 64 sample columns).  Replaces the dense Gaussian sample
// GEMM of the range finder: C is read once (HBM-bound) instead of 6 M N K
// tensor flops (a sparse sign map captures the couplings' range as the
// Gaussian one does: tools/sparse_sketch_check.py).  Omega is stored per
// sample column as (source column, sign) lists sorted by source column; a CTA
// covers 32 rows of one task, stages its source columns through shared memory
// 64 at a time (each read once), and warp w sums sample columns 8w..8w+7 in
// registers (each lane its own row).
// ---------------------------------------------------------------------------
constexpr int kSkCols = 64, kSkZeta = 8, kSkChunk = 32;
constexpr size_t kSkSmem = size_t(kSkChunk) * 33 * sizeof(cplx);
// col_ptr[j * (nchunks + 1) + c]: first entry of sample column j whose source
// column is >= c * kSkChunk; entries packed ((source mod kSkChunk) << 1) | negative
__global__ void __launch_bounds__(256) sparse_sketch_kernel(const cplx* const* __restrict__ src,
                                                            const int* __restrict__ lds, int M, int ncols,
                                                            const int* __restrict__ col_ptr,
                                                            const int* __restrict__ ent, cplx alpha,
                                                            cplx* __restrict__ Y, int ldy, size_t ystride) {
    extern __shared__ cplx sk_sm[];  // staged source columns [kSkChunk][33] (32 rows + pad)
    const int q = blockIdx.y, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int r0 = blockIdx.x * 32;
    const cplx* A = src[q];
    const size_t ld = size_t(lds[q]);
    const int nch = (ncols + kSkChunk - 1) / kSkChunk;
    cplx acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = cplx{0, 0};
    for (int ch = 0; ch < nch; ++ch) {
        const int c0 = ch * kSkChunk, cn = min(kSkChunk, ncols - c0);
        // each source column of the chunk read once (32 rows: 512 B per column)
#pragma unroll
        for (int u = 0; u < 32 * kSkChunk / 256; ++u) {
            const int e = tid + 256 * u, i = e >> 5, rr = e & 31;
            sk_sm[i * 33 + rr] = (i < cn && r0 + rr < M) ? A[size_t(c0 + i) * ld + r0 + rr] : cplx{0, 0};
        }
        __syncthreads();
        // warp w: sample columns 8 w .. 8 w + 7, lane: row
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int j = 8 * w + k;
            const int e0 = col_ptr[j * (nch + 1) + ch], e1 = col_ptr[j * (nch + 1) + ch + 1];
            // entries: (staged row offset << 1) | negative (offset precomputed on the host)
            for (int e = e0; e < e1; ++e) {
                const int pk = ent[e];
                const cplx v = sk_sm[(pk >> 1) * 33 + lane];
                acc[k].re += (pk & 1) ? -v.re : v.re;
                acc[k].im += (pk & 1) ? -v.im : v.im;
            }
        }
        __syncthreads();
    }
    const int row = r0 + lane;
    if (row < M) {
        cplx* y = Y + size_t(q) * ystride + row;
#pragma unroll
        for (int k = 0; k < 8; ++k) y[size_t(8 * w + k) * ldy] = cmul(alpha, acc[k]);
    }
}

// the first r2 of the r1 columns of every coupling's ID factors (adaptive
// basis width): L (nb x r1 -> nb x r2, the leading columns are contiguous),
// L1^{-1} (leading r2 x r2 block: the inverse of a leading block of a lower
// triangular matrix), skeleton rows
__global__ void __launch_bounds__(256) id_compact_kernel(int nb, int r1, int r2, const cplx* __restrict__ P1,
                                                         const cplx* __restrict__ L1, const int* __restrict__ piv1,
                                                         cplx* __restrict__ P2, cplx* __restrict__ L2,
                                                         int* __restrict__ piv2) {
    const int q = blockIdx.y;
    const size_t pn = size_t(nb) * r2;
    const cplx* src = P1 + size_t(q) * nb * r1;
    cplx* dst = P2 + size_t(q) * pn;
    for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < pn; e += size_t(gridDim.x) * blockDim.x)
        dst[e] = src[e];
    if (blockIdx.x == 0) {
        for (int e = threadIdx.x; e < r2 * r2; e += blockDim.x)
            L2[size_t(q) * r2 * r2 + e] = L1[size_t(q) * r1 * r1 + size_t(e / r2) * r1 + e % r2];
        for (int e = threadIdx.x; e < r2; e += blockDim.x) piv2[size_t(q) * r2 + e] = piv1[size_t(q) * r1 + e];
    }
}

// Two rows per lane (64 per CTA) and the whole sparse map (column pointers and
// entries, ~22 KB at nb = 608) in shared memory: every entry's index and sign
// is a broadcast shared load amortised over two rows instead of a global load
// per row, which left the one-row kernel at 1.8 TB/s waiting on L1/L2
// (long-scoreboard stalls).  Same per-row summation order, so Y is bitwise the
// one-row kernel's.
constexpr int kSkRows = 64, kSkLd = kSkRows + 1;
size_t sk2_smem_bytes(int nptr, int nent) {
    return size_t(2) * kSkChunk * kSkLd * sizeof(cplx) + sizeof(int) * size_t(nptr + nent);
}
__device__ __forceinline__ void sk_cp_async16(void* smem, const void* gmem, bool valid) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(valid ? 16 : 0));
}
__global__ void __launch_bounds__(256, 2) sparse_sketch2_kernel(const cplx* const* __restrict__ src,
                                                                const int* __restrict__ lds, int M, int ncols,
                                                                const int* __restrict__ col_ptr,
                                                                const int* __restrict__ ent, int nent, cplx alpha,
                                                                cplx* __restrict__ Y, int ldy, size_t ystride) {
    extern __shared__ cplx sk_sm[];  // two staged chunks [kSkChunk][kSkLd], then the map
    const int nch = (ncols + kSkChunk - 1) / kSkChunk, nptr = kSkCols * (nch + 1);
    int* s_ptr = reinterpret_cast<int*>(sk_sm + 2 * kSkChunk * kSkLd);
    int* s_ent = s_ptr + nptr;
    const int q = blockIdx.y, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int r0 = blockIdx.x * kSkRows;
    for (int e = tid; e < nptr; e += blockDim.x) s_ptr[e] = col_ptr[e];
    for (int e = tid; e < nent; e += blockDim.x) s_ent[e] = ent[e];
    const cplx* A = src[q];
    const size_t ld = size_t(lds[q]);
    cplx acc[8][2];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k][0] = acc[k][1] = cplx{0, 0};
    // each source column of a chunk read once (64 rows: 1 KB per column),
    // asynchronously into the other buffer while this one is summed
    auto stage = [&](int ch, int buf) {
        const int c0 = ch * kSkChunk, cn = min(kSkChunk, ncols - c0);
        cplx* dst = sk_sm + buf * kSkChunk * kSkLd;
#pragma unroll
        for (int u = 0; u < kSkRows * kSkChunk / 256; ++u) {
            const int e = tid + 256 * u, i = e / kSkRows, rr = e % kSkRows;
            const bool ok = i < cn && r0 + rr < M;
            sk_cp_async16(dst + i * kSkLd + rr, ok ? (const void*)(A + size_t(c0 + i) * ld + r0 + rr) : (const void*)A,
                          ok);
        }
        asm volatile("cp.async.commit_group;\n" ::);
    };
    stage(0, 0);
    for (int ch = 0; ch < nch; ++ch) {
        if (ch + 1 < nch) {
            stage(ch + 1, (ch + 1) & 1);
            asm volatile("cp.async.wait_group 1;\n" ::);
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::);
        }
        __syncthreads();  // chunk ch landed (and, at ch = 0, the map)
        const cplx* cur = sk_sm + (ch & 1) * kSkChunk * kSkLd;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int j = 8 * w + k;
            const int e0 = s_ptr[j * (nch + 1) + ch], e1 = s_ptr[j * (nch + 1) + ch + 1];
            for (int e = e0; e < e1; ++e) {
                const int pk = s_ent[e];
                const cplx* col = cur + (pk >> 1) * kSkLd + lane;
                const cplx v0 = col[0], v1 = col[32];
                const double sg = (pk & 1) ? -1.0 : 1.0;  // acc + (-v) == fma(-1, v, acc): same rounding
                acc[k][0].re = fma(sg, v0.re, acc[k][0].re);
                acc[k][0].im = fma(sg, v0.im, acc[k][0].im);
                acc[k][1].re = fma(sg, v1.re, acc[k][1].re);
                acc[k][1].im = fma(sg, v1.im, acc[k][1].im);
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int row = r0 + lane + 32 * h;
        if (row < M) {
            cplx* y = Y + size_t(q) * ystride + row;
#pragma unroll
            for (int k = 0; k < 8; ++k) y[size_t(8 * w + k) * ldy] = cmul(alpha, acc[k][h]);
        }
    }
}

GemmTask gemm1(const cplx* A, int lda, const cplx* B, int ldb, int K, cplx* C, int ldc) {
    GemmTask t{};
    t.nseg = 1;
    t.A[0] = A;
    t.lda[0] = lda;
    t.B[0] = B;
    t.ldb[0] = ldb;
    t.K[0] = K;
    t.C = C;
    t.ldc = ldc;
    return t;
}

GemvTask gemv1(const cplx* A, int lda, const cplx* x, int n, cplx* y) {
    GemvTask v{};
    v.nseg = 1;
    v.A[0] = A;
    v.lda[0] = lda;
    v.x[0] = x;
    v.n[0] = n;
    v.y = y;
    return v;
}

}  // namespace

namespace {
// random sample matrix (seeded, fixed), uploaded on stream s
void lr_omega_setup(Ctx& c, cudaStream_t s) {
    const int nb = c.dims.nb;
    if (c.lr_omega_n == nb) return;
    std::vector<cplx> om(size_t(nb) * kLrCols);
    uint64_t x = 0x9e3779b97f4a7c15ull;
    for (auto& z : om) {
        auto next = [&]() {
            x ^= x >> 12;
            x ^= x << 25;
            x ^= x >> 27;
            return double((x * 0x2545f4914f6cdd1dull) >> 11) * (1.0 / 9007199254740992.0) * 2.0 - 1.0;
        };
        z = cplx{next(), next()};
    }
    c.lr_omega.upload(om, s);
    // the sparse sign sketch: kSkZeta distinct sample columns per source
    // column, random signs (seeded, fixed), listed per sample column
    std::vector<std::vector<int>> colent(kSkCols);
    uint64_t y = 0x853c49e6748fea9bull;
    auto rnd = [&]() {
        y ^= y >> 12;
        y ^= y << 25;
        y ^= y >> 27;
        return (y * 0x2545f4914f6cdd1dull) >> 33;
    };
    for (int i = 0; i < nb; ++i) {
        int cols[kSkCols];
        for (int j = 0; j < kSkCols; ++j) cols[j] = j;
        for (int t = 0; t < kSkZeta; ++t) {  // partial Fisher-Yates: kSkZeta distinct columns
            const int j = t + int(rnd() % uint64_t(kSkCols - t));
            std::swap(cols[t], cols[j]);
            colent[cols[t]].push_back(((i % kSkChunk) << 1) | int(rnd() & 1u) | ((i / kSkChunk) << 20));
        }
    }
    const int nch = (nb + kSkChunk - 1) / kSkChunk;
    std::vector<int> ptr(size_t(kSkCols) * (nch + 1)), ent;
    for (int j = 0; j < kSkCols; ++j) {  // entries sorted by source column (generated in order)
        const int base = int(ent.size());
        for (int ch = 0; ch <= nch; ++ch) {  // chunk index parked in bits 20.. while sorting out the ranges
            int k = 0;
            while (k < int(colent[j].size()) && (colent[j][k] >> 20) < ch) ++k;
            ptr[size_t(j) * (nch + 1) + ch] = base + k;
        }
        for (int v : colent[j]) ent.push_back(v & ((1 << 20) - 1));
    }
    c.lr_sk_ptr.upload(ptr, s);
    c.lr_sk_ent.upload(ent, s);
    c.lr_omega_n = nb;
}

// QPS_LR_SKETCH=dense: the dense Gaussian sample GEMM (A/B)
bool sparse_sketch_on() {
    static const bool dense = [] {
        const char* e = getenv("QPS_LR_SKETCH");
        return e && !strcmp(e, "dense");
    }();
    return !dense;
}

// Y_q = alpha C_q Omega for every task (C_q: M rows, ld ld_q), 64 columns
void sparse_sketch(Ctx& c, const std::vector<const cplx*>& src, const std::vector<int>& ld, int M, cplx alpha,
                   cplx* Y, int ldy, size_t ystride, DBuf<const cplx*>& pbuf, DBuf<int>& lbuf, cudaStream_t s) {
    if (src.empty()) return;
    pbuf.upload(src, s);
    lbuf.upload(ld, s);
    ProfScope ps("lr_sketch", s, 0.0, 16.0 * double(src.size()) * M * c.dims.nb);
    const int nb = c.dims.nb, nch = (nb + kSkChunk - 1) / kSkChunk;
    const int nptr = kSkCols * (nch + 1), nent = kSkZeta * nb;
    const size_t sm2 = sk2_smem_bytes(nptr, nent);
    static const bool v1 = [] {  // QPS_LR_SKETCH=v1: the one-row-per-lane kernel (A/B)
        const char* e = getenv("QPS_LR_SKETCH");
        return e && !strcmp(e, "v1");
    }();
    if (!v1 && sm2 <= 200 * 1024) {
        static size_t attr2 = 0;
        if (sm2 > attr2) {
            QPS_CUDA(cudaFuncSetAttribute(sparse_sketch2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(200 * 1024)));
            attr2 = 200 * 1024;
        }
        { QPS_NOTE_LAUNCH(); sparse_sketch2_kernel<<<dim3((M + kSkRows - 1) / kSkRows, unsigned(src.size())), 256, sm2,
                                                      s>>>(pbuf.p, lbuf.p, M, nb, c.lr_sk_ptr.p, c.lr_sk_ent.p, nent,
                                                           alpha, Y, ldy, ystride); }
    } else {
        static bool attr = false;
        if (!attr) {
            QPS_CUDA(cudaFuncSetAttribute(sparse_sketch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(kSkSmem)));
            attr = true;
        }
        { QPS_NOTE_LAUNCH(); sparse_sketch_kernel<<<dim3((M + 31) / 32, unsigned(src.size())), 256, kSkSmem, s>>>(
            pbuf.p, lbuf.p, M, nb, c.lr_sk_ptr.p, c.lr_sk_ent.p, alpha, Y, ldy, ystride); }
    }
    QPS_CUDA(cudaGetLastError());
}
bool lr_eligible(const Ctx& c) {
    static const bool dense_only = [] {
        const char* e = getenv("QPS_BCR");
        return e && !strcmp(e, "dense");
    }();
    return !dense_only && c.dims.I >= 2 && c.dims.nb >= 4 * kLrSample;
}
}  // namespace

// The sample's A Omega part needs only the assembled couplings: it runs on a
// second stream while the Schur least squares (latency-bound) run on the main
// one.  lr_compress adds the B (-X Omega) correction once X exists.
void lr_sample_async(Ctx& c) {
    c.lr_sample_pending = false;
    if (!lr_eligible(c)) return;
    const Dims& D = c.dims;
    const int I = D.I, nb = D.nb, ns = D.nsys;
    const int nc = 2 * ns * (I - 1);
    QPS_CUDA(cudaEventRecord(c.ev_fill, c.stream));
    QPS_CUDA(cudaStreamWaitEvent(c.side2, c.ev_fill, 0));
    if (c.fill_pending) QPS_CUDA(cudaStreamWaitEvent(c.side2, c.ev_fillB, 0));  // the couplings of a split fill
    lr_omega_setup(c, c.side2);
    c.lr_Y.ensure(size_t(nc) * nb * kLrCols);
    std::vector<GemmTask> t(nc);
    std::vector<const cplx*> srcs(nc);
    for (int q = 0; q < nc; ++q) {
        const int a = q / (2 * (I - 1)), rem = q % (2 * (I - 1));
        const bool sup = rem >= I - 1;
        const int j = sup ? rem - (I - 1) : rem;
        const cplx* C = (sup ? c.Asup.p : c.Asub.p) + size_t(a) * D.sU() + size_t(j) * D.nb2();
        t[q] = gemm1(C, nb, c.lr_omega.p, nb, nb, c.lr_Y.p + size_t(q) * nb * kLrCols, nb);
        srcs[q] = C;
    }
    {
        ProfPhase phase("lowrank");
        // own family: its events on the low-priority stream span its overlap
        // with the Schur chain, so the duration is not a kernel time
        if (sparse_sketch_on())
            sparse_sketch(c, srcs, std::vector<int>(nc, nb), nb, cplx{1, 0}, c.lr_Y.p, nb, size_t(nb) * kLrCols,
                          c.lr_skp, c.lr_skl, c.side2);
        else
            zgemm_batched(nb, kLrCols, cplx{1, 0}, cplx{0, 0}, t, c.side2, c.lr_tasks, "lr_sample");
    }
    QPS_CUDA(cudaEventRecord(c.ev_sample, c.side2));
    c.lr_sample_pending = true;
}

// Accept the compression once the sample ranks and probe norms are on the host
// (ev_sample): false sends the system to the dense reduction.
static bool lr_accept(Ctx& c, int nc) {
    QPS_CUDA(cudaEventSynchronize(c.ev_sample));
    int mx = 0;
    for (int q = 0; q < nc; ++q) mx = std::max(mx, c.lr_rank_h[q]);
    c.lr_rank_max = std::max(c.lr_rank_max, mx);
    if (getenv("QPS_LR_TRACE")) {
        int mn = 1 << 30;
        double mean = 0;
        for (int q = 0; q < nc; ++q) { mn = std::min(mn, c.lr_rank_h[q]); mean += c.lr_rank_h[q]; }
        fprintf(stderr, "low-rank couplings: %d blocks, rank min %d mean %.1f max %d (sample %d)\n", nc, mn,
                mean / nc, mx, kLrSample);
    }
    if (mx > kLrMaxRank) return false;  // not low rank: the dense reduction (A untouched so far)
    static const double probe_tol = [] {  // QPS_LR_PROBE_TOL: tests force the fallback with a tiny value
        const char* e = getenv("QPS_LR_PROBE_TOL");
        return e ? atof(e) : kLrProbeTol;
    }();
    double worst = 0;
    for (int q = 0; q < nc; ++q) {
        const double rel = c.lr_pn_h[q] / std::max(c.lr_pn_h[nc + q], 1e-300);
        worst = std::isfinite(rel) ? std::max(worst, rel) : INFINITY;
    }
    c.lr_probe_worst = worst;
    if (getenv("QPS_LR_TRACE"))
        fprintf(stderr, "low-rank couplings: probe max ||(I - P P^*) C w2|| / ||C w2|| = %.3e (tol %.1e)\n",
                worst, probe_tol);
    if (!(worst <= probe_tol)) return false;  // basis misses part of a coupling's range: dense reduction
    return true;
}

// Compress every coupling of every system: c.lr_P / c.lr_R (per coupling,
// n x r ld nb and r x n ld r), ordered [system][sub 0..I-2][super 0..I-2].
bool lr_compress(Ctx& c, cplx* Au, cplx* Al) {
    const Dims& D = c.dims;
    const int I = D.I, nb = D.nb, ns = D.nsys;
    if (!lr_eligible(c)) return false;  // small blocks: dense is cheap
    cudaStream_t s = c.stream;
    ProfPhase phase("lowrank");
    const int nc = 2 * ns * (I - 1);
    lr_omega_setup(c, s);
    auto coupling = [&](int q) -> const cplx* {  // q in [0, nc)
        const int a = q / (2 * (I - 1)), rem = q % (2 * (I - 1));
        const bool sup = rem >= I - 1;
        const int j = sup ? rem - (I - 1) : rem;
        return (sup ? Au : Al) + size_t(a) * D.sU() + size_t(j) * D.nb2();
    };
    // deferred coupling Schur updates (one-shot path): C = A - Bc X, never formed
    const bool corr = c.couplings_deferred;
    auto corr_task = [&](int q) -> const GemmTask& {
        const int a = q / (2 * (I - 1)), rem = q % (2 * (I - 1));
        return rem >= I - 1 ? c.coupling_sup[size_t(a) * (I - 1) + rem - (I - 1)]
                            : c.coupling_sub[size_t(a) * (I - 1) + rem];
    };
    const int P = D.P;
    // Y = C Omega  (= A Omega + Bc (-X Omega) when deferred)
    c.lr_Y.ensure(size_t(nc) * nb * kLrCols);
    const bool early = c.lr_sample_pending && corr;  // Y already holds A Omega
    static const bool trace = getenv("QPS_BCR_TRACE") != nullptr;  // per-step timing to stderr (debug)
    cudaEvent_t te0 = nullptr, te1 = nullptr;
    if (trace) {
        QPS_CUDA(cudaEventCreate(&te0));
        QPS_CUDA(cudaEventCreate(&te1));
        QPS_CUDA(cudaEventRecord(te0, s));
    }
    auto tmark = [&](const char* what) {
        if (!trace) return;
        float ms = 0;
        QPS_CUDA(cudaEventRecord(te1, s));
        QPS_CUDA(cudaEventSynchronize(te1));
        QPS_CUDA(cudaEventElapsedTime(&ms, te0, te1));
        fprintf(stderr, "lr_compress %s: %.3f ms\n", what, ms);
        QPS_CUDA(cudaEventRecord(te0, s));
    };
    if (c.lr_sample_pending) QPS_CUDA(cudaStreamWaitEvent(s, c.ev_sample, 0));
    tmark("wait for the side-stream sample");
    c.lr_sample_pending = false;
    {
        std::vector<GemmTask> t(nc);
        if (corr) {
            c.lr_W.ensure(size_t(nc) * P * kLrCols);
            std::vector<GemmTask> w(nc);
            std::vector<const cplx*> xs(nc);
            std::vector<int> xl(nc);
            for (int q = 0; q < nc; ++q) {
                const GemmTask& u = corr_task(q);
                w[q] = gemm1(u.B[0], u.ldb[0], c.lr_omega.p, nb, nb, c.lr_W.p + size_t(q) * P * kLrCols, P);
                xs[q] = u.B[0];
                xl[q] = u.ldb[0];
            }
            if (sparse_sketch_on())
                sparse_sketch(c, xs, xl, P, cplx{-1, 0}, c.lr_W.p, P, size_t(P) * kLrCols, c.lr_skp, c.lr_skl, s);
            else
                zgemm_batched(P, kLrCols, cplx{-1, 0}, cplx{0, 0}, w, s, c.ws.gemm_tasks, "lr_compress");
        }
        for (int q = 0; q < nc && early; ++q) {  // Y += Bc (-X Omega)
            const GemmTask& u = corr_task(q);
            t[q] = gemm1(u.A[0], u.lda[0], c.lr_W.p + size_t(q) * P * kLrCols, P, P,
                         c.lr_Y.p + size_t(q) * nb * kLrCols, nb);
        }
        if (early) zgemm_batched(nb, kLrCols, cplx{1, 0}, cplx{1, 0}, t, s, c.ws.gemm_tasks, "lr_compress");
        if (!early && sparse_sketch_on()) {
            // Y = C Omega (sparse), then Y += Bc (-X Omega)
            std::vector<const cplx*> cs(nc);
            for (int q = 0; q < nc; ++q) cs[q] = coupling(q);
            sparse_sketch(c, cs, std::vector<int>(nc, nb), nb, cplx{1, 0}, c.lr_Y.p, nb, size_t(nb) * kLrCols,
                          c.lr_skp, c.lr_skl, s);
            for (int q = 0; q < nc && corr; ++q) {
                const GemmTask& u = corr_task(q);
                t[q] = gemm1(u.A[0], u.lda[0], c.lr_W.p + size_t(q) * P * kLrCols, P, P,
                             c.lr_Y.p + size_t(q) * nb * kLrCols, nb);
            }
            if (corr) zgemm_batched(nb, kLrCols, cplx{1, 0}, cplx{1, 0}, t, s, c.ws.gemm_tasks, "lr_compress");
        }
        for (int q = 0; q < nc && !early && !sparse_sketch_on(); ++q) {
            t[q] = gemm1(coupling(q), nb, c.lr_omega.p, nb, nb, c.lr_Y.p + size_t(q) * nb * kLrCols, nb);
            if (corr) {
                const GemmTask& u = corr_task(q);
                t[q].nseg = 2;
                t[q].A[1] = u.A[0];
                t[q].lda[1] = u.lda[0];
                t[q].B[1] = c.lr_W.p + size_t(q) * P * kLrCols;
                t[q].ldb[1] = P;
                t[q].K[1] = P;
            }
        }
        if (!early && !sparse_sketch_on()) {
            if (getenv("QPS_TRACE_LAUNCH"))
                fprintf(stderr, "lr_compress sample GEMM is zgemm3m launch index %llu\n",
                        (unsigned long long)g_zgemm_launches.load());
            zgemm_batched(nb, kLrCols, cplx{1, 0}, cplx{0, 0}, t, s, c.ws.gemm_tasks, "lr_compress");
        }
    }
    tmark("sample correction Y += Bc (-X Omega)");
    static const bool id_off = [] {  // QPS_LR_ID=0: the orthonormal basis P (P^* C) instead (A/B)
        const char* e = getenv("QPS_LR_ID");
        return e && !strcmp(e, "0");
    }();
    if (!id_off && nb <= kIdThreads && lr_basis() <= kLrSample) {
        int r = lr_basis();
        c.lr_r = r;
        c.lr_P.ensure(size_t(nc) * nb * r);
        c.lr_L1i.ensure(size_t(nc) * r * r);
        c.lr_piv.ensure(size_t(nc) * r);
        c.lr_rank_d.ensure(nc);
        {
            ProfScope ps("lr_id", s, 0.0);
            const size_t sm = id_smem_bytes(r);
            static size_t attr = 0;
            if (sm > attr) {
                QPS_CUDA(cudaFuncSetAttribute(lr_id_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
                attr = sm;
            }
            { QPS_NOTE_LAUNCH(); lr_id_kernel<<<nc, kIdThreads, sm, s>>>(nb, c.lr_Y.p, size_t(nb) * kLrCols, r, c.lr_P.p,
                                                                         size_t(nb) * r, c.lr_L1i.p, c.lr_piv.p,
                                                                         c.lr_rank_d.p, kIdTol); }
            QPS_CUDA(cudaGetLastError());
        }
        c.lr_rank_h.ensure(nc);
        QPS_D2H(c.lr_rank_h.p, c.lr_rank_d.p, sizeof(int) * nc, s);
        // adaptive width: the widest accepted rank rounded up to 8 columns
        // (config 4: 39 -> 40 instead of 48) -- every later product, the level-0
        // right-hand sides and the 2r x 2r capacitances shrink with it.  The
        // host waits for the ranks here; the factorization is queued already.
        static const bool adapt = [] {  // QPS_LR_ADAPT=0: always lr_basis() columns (A/B)
            const char* e = getenv("QPS_LR_ADAPT");
            return !(e && !strcmp(e, "0"));
        }();
        c.lr_width_retry = false;
        if (adapt && !c.lr_full_width) {
            if (!c.ev_rank) QPS_CUDA(cudaEventCreateWithFlags(&c.ev_rank, cudaEventDisableTiming));
            QPS_CUDA(cudaEventRecord(c.ev_rank, s));
            QPS_CUDA(cudaEventSynchronize(c.ev_rank));
            int mx = 0;
            for (int q = 0; q < nc; ++q) mx = std::max(mx, c.lr_rank_h[q]);
            const int rn = std::max(16, (mx + 7) / 8 * 8);
            if (mx <= kLrMaxRank && rn < r) {
                c.lr_Pc.ensure(size_t(nc) * nb * rn);
                c.lr_L1ic.ensure(size_t(nc) * rn * rn);
                c.lr_pivc.ensure(size_t(nc) * rn);
                { QPS_NOTE_LAUNCH(); id_compact_kernel<<<dim3(16, nc), 256, 0, s>>>(nb, r, rn, c.lr_P.p, c.lr_L1i.p,
                                                                                   c.lr_piv.p, c.lr_Pc.p,
                                                                                   c.lr_L1ic.p, c.lr_pivc.p); }
                QPS_CUDA(cudaGetLastError());
                std::swap(c.lr_P, c.lr_Pc);
                std::swap(c.lr_L1i, c.lr_L1ic);
                std::swap(c.lr_piv, c.lr_pivc);
                r = rn;
                c.lr_r = r;
            }
        }
        tmark("row ID of the samples");
        wb_level0_async(c);  // the left factors exist: level 0 on the factor stream from here
        // R = L1^{-1} C[I, :]   (C[I, :] = A[I, :] - Bc[I, :] X when deferred)
        c.lr_G.ensure(size_t(nc) * r * nb);
        c.lr_R.ensure(size_t(nc) * r * nb);
        std::vector<const cplx*> src(nc);
        std::vector<int> lds(nc, nb);
        for (int q = 0; q < nc; ++q) src[q] = coupling(q);
        auto gather_rows = [&](const std::vector<const cplx*>& sp, const std::vector<int>& ld, int ncols, cplx* dst,
                               size_t dstride) {
            c.lr_gptr.upload(sp, s);
            c.lr_gld.upload(ld, s);
            ProfScope ps("copy", s, 0.0, 32.0 * nc * double(r) * ncols);
            const int per = r * ncols;
            const dim3 grid(std::min(64, (per + 255) / 256), nc);
            { QPS_NOTE_LAUNCH(); gather_rows_kernel<<<grid, 256, 0, s>>>(c.lr_gptr.p, c.lr_gld.p, c.lr_piv.p, r, ncols,
                                                                          dst, dstride); }
            QPS_CUDA(cudaGetLastError());
        };
        gather_rows(src, lds, nb, c.lr_G.p, size_t(r) * nb);
        if (corr) {
            c.lr_W.ensure(size_t(nc) * r * P);
            std::vector<const cplx*> bs(nc);
            std::vector<int> bl(nc);
            for (int q = 0; q < nc; ++q) {
                bs[q] = corr_task(q).A[0];
                bl[q] = corr_task(q).lda[0];
            }
            gather_rows(bs, bl, P, c.lr_W.p, size_t(r) * P);
            std::vector<GemmTask> t(nc);
            for (int q = 0; q < nc; ++q)
                t[q] = gemm1(c.lr_W.p + size_t(q) * r * P, r, corr_task(q).B[0], corr_task(q).ldb[0], P,
                             c.lr_G.p + size_t(q) * r * nb, r);
            zgemm_batched(r, nb, cplx{-1, 0}, cplx{1, 0}, t, s, c.ws.gemm_tasks, "lr_compress");
        }
        {
            std::vector<GemmTask> t(nc);
            for (int q = 0; q < nc; ++q)
                t[q] = gemm1(c.lr_L1i.p + size_t(q) * r * r, r, c.lr_G.p + size_t(q) * r * nb, r, r,
                             c.lr_R.p + size_t(q) * r * nb, r);
            zgemm_batched(r, nb, cplx{1, 0}, cplx{0, 0}, t, s, c.ws.gemm_tasks, "lr_compress");
        }
        tmark("R = L1^{-1} C[I, :]");
        // a-posteriori probe: ||C[:, J] - L R[:, J]||_F against ||C[:, J]||_F
        static const bool no_probe_id = [] {
            const char* e = getenv("QPS_LR_PROBE");
            return e && !strcmp(e, "0");
        }();
        c.lr_pn_h.ensure(size_t(nc) * 2);
        if (no_probe_id) {
            for (int q = 0; q < 2 * nc; ++q) c.lr_pn_h[q] = 0.0;
        } else {
            if (c.lr_probe_n != nc * 65536 + nb) {
                std::vector<int> cols(size_t(nc) * kLrProbe);
                uint64_t x = 0xd1b54a32d192ed03ull;
                for (auto& v : cols) {
                    x ^= x >> 12;
                    x ^= x << 25;
                    x ^= x >> 27;
                    v = int(((x * 0x2545f4914f6cdd1dull) >> 33) % uint64_t(nb));
                }
                c.lr_probe_cols.upload(cols, s);
                c.lr_probe_n = nc * 65536 + nb;
            }
            std::vector<const cplx*> xp(nc), rp(nc);
            std::vector<int> xld(nc, P), rld(nc, r);
            for (int q = 0; q < nc; ++q) {
                rp[q] = c.lr_R.p + size_t(q) * r * nb;
                if (corr) {
                    xp[q] = corr_task(q).B[0];
                    xld[q] = corr_task(q).ldb[0];
                }
            }
            c.lr_Y2.ensure(size_t(nc) * nb * kLrProbe);
            c.lr_G2.ensure(size_t(nc) * (r + P) * kLrProbe);
            cplx* Rg = c.lr_G2.p;                               // r x 16 per coupling
            cplx* Xg = c.lr_G2.p + size_t(nc) * r * kLrProbe;  // P x 16 per coupling
            gather_columns(src, lds, nb, c.lr_probe_cols.p, kLrProbe, c.lr_Y2.p, nb, size_t(nb) * kLrProbe, c.lr_gptr,
                           c.lr_gld, s);
            if (corr) {
                gather_columns(xp, xld, P, c.lr_probe_cols.p, kLrProbe, Xg, P, size_t(P) * kLrProbe, c.lr_gptr,
                               c.lr_gld, s);
                std::vector<GemmTask> t(nc);
                for (int q = 0; q < nc; ++q)
                    t[q] = gemm1(corr_task(q).A[0], corr_task(q).lda[0], Xg + size_t(q) * P * kLrProbe, P, P,
                                 c.lr_Y2.p + size_t(q) * nb * kLrProbe, nb);
                zgemm_batched(nb, kLrProbe, cplx{-1, 0}, cplx{1, 0}, t, s, c.ws.gemm_tasks, "lr_compress");
            }
            gather_columns(rp, rld, r, c.lr_probe_cols.p, kLrProbe, Rg, r, size_t(r) * kLrProbe, c.lr_gptr, c.lr_gld,
                           s);
            std::vector<GemmTask> e(nc);
            for (int q = 0; q < nc; ++q)
                e[q] = gemm1(c.lr_P.p + size_t(q) * nb * r, nb, Rg + size_t(q) * r * kLrProbe, r, r,
                             c.lr_Y2.p + size_t(q) * nb * kLrProbe, nb);
            c.lr_pn.ensure(size_t(nc) * 2);
            batched_fro(c.lr_Y2.p, nb, kLrProbe, nb, size_t(nb) * kLrProbe, nc, c.lr_pn.p + nc, s);
            zgemm_residual_norms(nb, kLrProbe, cplx{-1, 0}, cplx{1, 0}, e, s, c.ws.gemm_tasks, c.lr_parts, c.lr_pn.p);
            QPS_D2H(c.lr_pn_h.p, c.lr_pn.p, sizeof(double) * 2 * nc, s);
        }
        QPS_CUDA(cudaEventRecord(c.ev_sample, s));
        tmark("probe");
        if (trace) {
            QPS_CUDA(cudaEventDestroy(te0));
            QPS_CUDA(cudaEventDestroy(te1));
        }
        tl_mark(c, "compress", s);
        const bool ok = lr_accept(c, nc);
        // a truncated width that fails (rank within the limit, probe missed):
        // the caller retries at the full width before going dense
        if (!ok && r < lr_basis() && c.lr_rank_max <= kLrMaxRank) c.lr_width_retry = true;
        return ok;
    }
    static const bool cpqr_only = [] {
        const char* e = getenv("QPS_LR_QR");
        return e && !strcmp(e, "cpqr");
    }();
    std::vector<int> rk(nc);
    int r = 0;
    bool rank_deferred = false;
    if (!cpqr_only && nb <= 640) {
        // blocked Householder QR of the samples, CPQR of the 64 x 64 R
        const int m = nb, p = kLrSample, nP = p / kQrW;
        const size_t ys = size_t(m) * p, vs = size_t(m) * kQrW, ts = size_t(kQrW) * kQrW;
        c.lr_V.ensure(size_t(nc) * nP * vs);
        c.lr_VH.ensure(size_t(nc) * nP * vs);
        c.lr_Tq.ensure(size_t(nc) * nP * ts);
        c.lr_THq.ensure(size_t(nc) * nP * ts);
        c.lr_W1.ensure(size_t(nc) * kQrW * p);
        c.lr_W2.ensure(size_t(nc) * kQrW * p);
        static bool attr = false;
        if (!attr) {
            QPS_CUDA(cudaFuncSetAttribute(qr_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(640 * kQrW * sizeof(cplx))));
            attr = true;
        }
        auto V_of = [&](int q, int pn) { return c.lr_V.p + (size_t(q) * nP + pn) * vs; };
        auto VH_of = [&](int q, int pn) { return c.lr_VH.p + (size_t(q) * nP + pn) * vs; };
        auto T_of = [&](int q, int pn) { return c.lr_Tq.p + (size_t(q) * nP + pn) * ts; };
        auto TH_of = [&](int q, int pn) { return c.lr_THq.p + (size_t(q) * nP + pn) * ts; };
        for (int pn = 0; pn < nP; ++pn) {
            const int col0 = pn * kQrW;
            {
                ProfScope ps("lr_qr", s, 0.0);
                // per-problem pointers are strided: V_of(q, pn) = base + (q nP + pn) vs
                { QPS_NOTE_LAUNCH(); qr_panel_kernel<<<nc, ((m + 31) / 32) * 32, size_t(m) * kQrW * sizeof(cplx), s>>>(
                    m, c.lr_Y.p, ys, col0, c.lr_V.p + pn * vs, c.lr_VH.p + pn * vs, c.lr_Tq.p + pn * ts,
                    c.lr_THq.p + pn * ts, size_t(nP) * vs, size_t(nP) * ts); }
                QPS_CUDA(cudaGetLastError());
            }
            const int rest = p - col0 - kQrW;
            if (rest <= 0) continue;
            std::vector<GemmTask> t1(nc), t2(nc), t3(nc);
            for (int q = 0; q < nc; ++q) {
                cplx* Yr = c.lr_Y.p + size_t(q) * ys + size_t(col0 + kQrW) * m;
                t1[q] = gemm1(VH_of(q, pn), kQrW, Yr, m, m, c.lr_W1.p + size_t(q) * kQrW * p, kQrW);
                t2[q] = gemm1(TH_of(q, pn), kQrW, c.lr_W1.p + size_t(q) * kQrW * p, kQrW, kQrW,
                              c.lr_W2.p + size_t(q) * kQrW * p, kQrW);
                t3[q] = gemm1(V_of(q, pn), m, c.lr_W2.p + size_t(q) * kQrW * p, kQrW, kQrW, Yr, m);
            }
            zgemm_batched(kQrW, rest, cplx{1, 0}, cplx{0, 0}, t1, s, c.ws.gemm_tasks, "lr_qr");
            zgemm_batched(kQrW, rest, cplx{1, 0}, cplx{0, 0}, t2, s, c.ws.gemm_tasks, "lr_qr");
            zgemm_batched(m, rest, cplx{-1, 0}, cplx{1, 0}, t3, s, c.ws.gemm_tasks, "lr_qr");
        }
        tmark("blocked QR of the samples");
        // CPQR of R (64 x 64): rank and the ordered basis Q2
        c.lr_R64.ensure(size_t(nc) * p * p);
        { QPS_NOTE_LAUNCH(); qr_take_r_kernel<<<nc, 256, 0, s>>>(m, p, c.lr_Y.p, ys, c.lr_R64.p); }
        QPS_CUDA(cudaGetLastError());
        CodSet& cs = c.lr_cod;
        cs.ensure(nc, p, p, 1);
        CodBatch b = cs.batch(c.lr_R64.p);
        cod_factor_fast(b, s);
        cod_rank(b, kLrTol, nullptr, s);
        // the ranks are checked once the basis and the projections are queued
        // (the basis width is fixed, kLrMaxRank): the host waits on this event
        // while the GPU still has that work ahead of it, instead of draining
        // the stream here
        c.lr_rank_h.ensure(nc);
        QPS_D2H(c.lr_rank_h.p, cs.rank.p, sizeof(int) * nc, s);
        QPS_CUDA(cudaEventRecord(c.ev_sample, s));
        rank_deferred = true;
        r = lr_basis();
        c.lr_r = r;
        // Q2 = first r columns of the R-CPQR's Q (64 x r)
        c.lr_Q2.ensure(size_t(nc) * p * r);
        c.lr_Q2H.ensure(size_t(nc) * p * r);
        { QPS_NOTE_LAUNCH(); lr_form_q_kernel<<<dim3(nc, (r + 7) / 8), 256, size_t(8) * p * sizeof(cplx), s>>>(
            p, p, r, cs.W.p, cs.tau.p, c.lr_Q2.p, p, size_t(p) * r, c.lr_Q2H.p, size_t(r) * p); }
        QPS_CUDA(cudaGetLastError());
        // P = Q [Q2; 0], Q = (I - V0 T0 V0^*) ... (I - V3 T3 V3^*)
        c.lr_P.ensure(size_t(nc) * nb * r);
        c.lr_PH.ensure(size_t(nc) * r * nb);
        { QPS_NOTE_LAUNCH(); qr_seed_kernel<<<nc, 256, 0, s>>>(m, p, r, c.lr_Q2.p, size_t(p) * r, c.lr_P.p, size_t(nb) * r); }
        QPS_CUDA(cudaGetLastError());
        // the four panels' reflectors as one compact WY, Q = I - V T V^* with
        // V = [V0 V1 V2 V3] (m x 64, the panels are stored contiguously) and T
        // upper triangular from the block recurrence T_{0:k,k} =
        // -T_{0:k,0:k} (V_{0:k}^* V_k) T_kk (zlarft, forward): P = [Q2; 0] -
        // V (T (V^* [Q2; 0])), where V^* [Q2; 0] only reads V's first 64 rows
        c.lr_Gq.ensure(size_t(nc) * p * p);
        c.lr_Tall.ensure(size_t(nc) * p * p);
        c.lr_W1a.ensure(size_t(nc) * p * r);
        c.lr_W2a.ensure(size_t(nc) * p * r);
        {
            std::vector<GemmTask> gt;
            gt.reserve(size_t(nc) * nP * (nP - 1) / 2);
            for (int q = 0; q < nc; ++q)
                for (int j = 1; j < nP; ++j)
                    for (int i = 0; i < j; ++i)  // G_ij = V_i^* V_j (V_j vanishes above row 16 j)
                        gt.push_back(gemm1(VH_of(q, i) + size_t(j) * kQrW * kQrW, kQrW,
                                           V_of(q, j) + size_t(j) * kQrW, m, m - j * kQrW,
                                           c.lr_Gq.p + size_t(q) * p * p + size_t(j) * kQrW * p + i * kQrW, p));
            zgemm_batched(kQrW, kQrW, cplx{1, 0}, cplx{0, 0}, gt, s, c.ws.gemm_tasks, "lr_qr");
            constexpr size_t wy_sm = (size_t(4 * kQrW) * (4 * kQrW + 1) + size_t(4 * kQrW) * (kQrW + 1)) * sizeof(cplx);
            static bool wy_attr = false;
            if (!wy_attr) {
                QPS_CUDA(cudaFuncSetAttribute(wy_merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(wy_sm)));
                wy_attr = true;
            }
            { QPS_NOTE_LAUNCH(); wy_merge_kernel<<<nc, 256, wy_sm, s>>>(nP, c.lr_Tq.p, size_t(nP) * kQrW * kQrW,
                                                                          c.lr_Gq.p, c.lr_Tall.p); }
            QPS_CUDA(cudaGetLastError());
            std::vector<GemmTask> w1(size_t(nc) * nP), w2(nc), pu(nc);
            for (int q = 0; q < nc; ++q) {
                for (int pn = 0; pn < nP; ++pn)  // W1 = V^*[0:64, :] Q2
                    w1[size_t(q) * nP + pn] = gemm1(VH_of(q, pn), kQrW, c.lr_Q2.p + size_t(q) * p * r, p, p,
                                                   c.lr_W1a.p + size_t(q) * p * r + pn * kQrW, p);
                w2[q] = gemm1(c.lr_Tall.p + size_t(q) * p * p, p, c.lr_W1a.p + size_t(q) * p * r, p, p,
                              c.lr_W2a.p + size_t(q) * p * r, p);
                pu[q] = gemm1(V_of(q, 0), m, c.lr_W2a.p + size_t(q) * p * r, p, p, c.lr_P.p + size_t(q) * nb * r, nb);
            }
            zgemm_batched(kQrW, r, cplx{1, 0}, cplx{0, 0}, w1, s, c.ws.gemm_tasks, "lr_qr");
            zgemm_batched(p, r, cplx{1, 0}, cplx{0, 0}, w2, s, c.ws.gemm_tasks, "lr_qr");
            zgemm_batched(m, r, cplx{-1, 0}, cplx{1, 0}, pu, s, c.ws.gemm_tasks, "lr_qr");
        }
        tmark("rank check, Q2, P = Q [Q2; 0]");
        { QPS_NOTE_LAUNCH(); conj_transpose_kernel<<<dim3((nb + kCtRows - 1) / kCtRows, nc), 256, 0, s>>>(nb, r, c.lr_P.p, size_t(nb) * r, c.lr_PH.p,
                                                           size_t(r) * nb); }
        QPS_CUDA(cudaGetLastError());
    } else {
// column-pivoted QR of each sample, numerical rank
        CodSet& cs = c.lr_cod;
        cs.ensure(nc, nb, kLrSample, 1);
        CodBatch b = cs.batch(c.lr_Y.p);
        cod_factor_fast(b, s);
        cod_rank(b, kLrTol, nullptr, s);
        QPS_D2H(rk.data(), cs.rank.p, sizeof(int) * nc, s);
        QPS_CUDA(cudaStreamSynchronize(s));
        for (int v : rk) r = std::max(r, v);
        c.lr_rank_max = r;
        if (getenv("QPS_LR_TRACE")) {
            int mn = 1 << 30;
            double mean = 0;
            for (int v : rk) { mn = std::min(mn, v); mean += v; }
            fprintf(stderr, "low-rank couplings: %d blocks, rank min %d mean %.1f max %d (sample %d)\n", nc, mn,
                    mean / nc, r, kLrSample);
        }
        if (r > kLrMaxRank) return false;
        // a fixed basis width keeps every system's factors independent of the batch
        // it is solved in (the sweep's batched and one-at-a-time results agree)
        r = lr_basis();
        c.lr_r = r;
        // P (n x r) and P^* (r x n)
        c.lr_P.ensure(size_t(nc) * nb * r);
        c.lr_PH.ensure(size_t(nc) * r * nb);
        {
            ProfScope ps("lr_compress", s, 0.0);
            static size_t attr = 0;
            const size_t sm = size_t(8) * nb * sizeof(cplx);
            if (sm > attr) {
                QPS_CUDA(cudaFuncSetAttribute(lr_form_q_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              int(std::max<size_t>(sm, 48 * 1024))));
                attr = std::max<size_t>(sm, 48 * 1024);
            }
            { QPS_NOTE_LAUNCH(); lr_form_q_kernel<<<dim3(nc, (r + 7) / 8), 256, size_t(8) * nb * sizeof(cplx), s>>>(
                nb, kLrSample, r, cs.W.p, cs.tau.p, c.lr_P.p, nb, size_t(nb) * r, c.lr_PH.p, size_t(r) * nb); }
            QPS_CUDA(cudaGetLastError());
        }
    }
    tmark("P^*");
    // a-posteriori test on the probe columns J (per coupling): Y2 = C[:, J]
    // (= A[:, J] - Bc X[:, J] when the coupling update is deferred),
    // ||Y2 - P R[:, J]||_F against ||Y2||_F, read back with the ranks
    static const bool no_probe = [] {  // QPS_LR_PROBE=0: skip the test (A/B timing only)
        const char* e = getenv("QPS_LR_PROBE");
        return e && !strcmp(e, "0");
    }();
    if (no_probe) {
        c.lr_pn_h.ensure(size_t(nc) * 2);
        for (int q = 0; q < 2 * nc; ++q) c.lr_pn_h[q] = 0.0;
    }
    if (!no_probe) {
        if (c.lr_probe_n != nc * 65536 + nb) {
            std::vector<int> cols(size_t(nc) * kLrProbe);
            uint64_t x = 0xd1b54a32d192ed03ull;
            for (auto& v : cols) {
                x ^= x >> 12;
                x ^= x << 25;
                x ^= x >> 27;
                v = int(((x * 0x2545f4914f6cdd1dull) >> 33) % uint64_t(nb));
            }
            c.lr_probe_cols.upload(cols, s);
            c.lr_probe_n = nc * 65536 + nb;
        }
        std::vector<const cplx*> cp(nc), xp(nc);
        std::vector<int> cld(nc, nb), xld(nc, P);
        for (int q = 0; q < nc; ++q) {
            cp[q] = coupling(q);
            if (corr) {
                xp[q] = corr_task(q).B[0];
                xld[q] = corr_task(q).ldb[0];
            }
        }
        c.lr_Y2.ensure(size_t(nc) * nb * kLrProbe);
        c.lr_G2.ensure(size_t(nc) * (r + P) * kLrProbe);
        cplx* Rg = c.lr_G2.p;                                   // r x 16 per coupling
        cplx* Xg = c.lr_G2.p + size_t(nc) * r * kLrProbe;      // P x 16 per coupling
        gather_columns(cp, cld, nb, c.lr_probe_cols.p, kLrProbe, c.lr_Y2.p, nb, size_t(nb) * kLrProbe, c.lr_gptr,
                       c.lr_gld, s);
        if (corr) {
            gather_columns(xp, xld, P, c.lr_probe_cols.p, kLrProbe, Xg, P, size_t(P) * kLrProbe, c.lr_gptr, c.lr_gld,
                           s);
            std::vector<GemmTask> t(nc);
            for (int q = 0; q < nc; ++q)
                t[q] = gemm1(corr_task(q).A[0], corr_task(q).lda[0], Xg + size_t(q) * P * kLrProbe, P, P,
                             c.lr_Y2.p + size_t(q) * nb * kLrProbe, nb);
            zgemm_batched(nb, kLrProbe, cplx{-1, 0}, cplx{1, 0}, t, s, c.ws.gemm_tasks, "lr_compress");
        }
        std::vector<GemmTask> gt(nc), e(nc);  // G = P^* Y2 (= R[:, J]), then ||Y2 - P G||
        for (int q = 0; q < nc; ++q) {
            gt[q] = gemm1(c.lr_PH.p + size_t(q) * r * nb, r, c.lr_Y2.p + size_t(q) * nb * kLrProbe, nb, nb,
                          Rg + size_t(q) * r * kLrProbe, r);
            e[q] = gemm1(c.lr_P.p + size_t(q) * nb * r, nb, Rg + size_t(q) * r * kLrProbe, r, r,
                         c.lr_Y2.p + size_t(q) * nb * kLrProbe, nb);
        }
        zgemm_batched(r, kLrProbe, cplx{1, 0}, cplx{0, 0}, gt, s, c.ws.gemm_tasks, "lr_compress");
        c.lr_pn.ensure(size_t(nc) * 2);
        batched_fro(c.lr_Y2.p, nb, kLrProbe, nb, size_t(nb) * kLrProbe, nc, c.lr_pn.p + nc, s);
        zgemm_residual_norms(nb, kLrProbe, cplx{-1, 0}, cplx{1, 0}, e, s, c.ws.gemm_tasks, c.lr_parts, c.lr_pn.p);
        c.lr_pn_h.ensure(size_t(nc) * 2);
        QPS_D2H(c.lr_pn_h.p, c.lr_pn.p, sizeof(double) * 2 * nc, s);
        // the host checks ranks and probes once this is reached, while the
        // projection R = P^* C below (the largest GEMM here) still runs
        QPS_CUDA(cudaEventRecord(c.ev_sample, s));
        if (!rank_deferred) {
            rank_deferred = true;
            c.lr_rank_h.ensure(nc);
            for (int q = 0; q < nc; ++q) c.lr_rank_h[q] = 0;  // ranks already checked above
        }
    }
    wb_level0_async(c);  // level 0 on the factor stream, overlapping the projection below
    // R = P^* C  (= P^* A + (-P^* Bc) X when deferred)
    c.lr_R.ensure(size_t(nc) * r * nb);
    {
        if (corr) {
            c.lr_G.ensure(size_t(nc) * r * P);
            std::vector<GemmTask> g(nc);
            for (int q = 0; q < nc; ++q) {
                const GemmTask& u = corr_task(q);
                g[q] = gemm1(c.lr_PH.p + size_t(q) * r * nb, r, u.A[0], u.lda[0], nb, c.lr_G.p + size_t(q) * r * P, r);
            }
            zgemm_batched(r, P, cplx{-1, 0}, cplx{0, 0}, g, s, c.ws.gemm_tasks, "lr_compress");
        }
        std::vector<GemmTask> t(nc);
        for (int q = 0; q < nc; ++q) {
            t[q] = gemm1(c.lr_PH.p + size_t(q) * r * nb, r, coupling(q), nb, nb, c.lr_R.p + size_t(q) * r * nb, r);
            if (corr) {
                const GemmTask& u = corr_task(q);
                t[q].nseg = 2;
                t[q].A[1] = c.lr_G.p + size_t(q) * r * P;
                t[q].lda[1] = r;
                t[q].B[1] = u.B[0];
                t[q].ldb[1] = u.ldb[0];
                t[q].K[1] = P;
            }
        }
        zgemm_batched(r, nb, cplx{1, 0}, cplx{0, 0}, t, s, c.ws.gemm_tasks, "lr_compress");
    }
    tmark("R = P^* C");
    if (trace) {
        QPS_CUDA(cudaEventDestroy(te0));
        QPS_CUDA(cudaEventDestroy(te1));
    }
    tl_mark(c, "compress", s);
    if (rank_deferred) return lr_accept(c, nc);
    return true;
}

void bcr_solve_lr(Ctx& c, cplx* Ad) {
    ProfPhase phase("bcr");
    ++c.n_factorizations;
    const Dims& D = c.dims;
    const int I = D.I, nb = D.nb, ns = D.nsys, r = c.lr_r;
    const size_t nb2 = D.nb2();
    cudaStream_t s = c.stream;
    const cplx one{1, 0}, mone{-1, 0}, zero{0, 0};
    c.F.ensure(size_t(ns) * I * nb);
    c.F.zero(s);
    for (int a = 0; a < ns; ++a)
        QPS_CUDA(cudaMemcpyAsync(c.F.p + size_t(a) * I * nb, c.f.p + size_t(a) * nb, sizeof(cplx) * nb,
                                 cudaMemcpyDeviceToDevice, s));
    c.ipiv.ensure(size_t(ns) * I * nb);
    const size_t dsz = lu_dinv_elems(nb);
    c.dinv.ensure(size_t(ns) * I * dsz);
    auto ipiv_of = [&](int a, int j) { return c.ipiv.p + (size_t(a) * I + j) * nb; };
    auto dinv_of = [&](int a, int j) { return c.dinv.p + (size_t(a) * I + j) * dsz; };
    // per-position state of one system at one level
    struct Pos {
        int idx;
        cplx *D, *F;
        const cplx *PL, *RL, *PU, *RU;  // couplings: L = PL RL (to the left), U = PU RU (to the right)
        cplx* Z;                        // odd positions: D^{-1} [PL PU]
    };
    using Level = std::vector<std::vector<Pos>>;  // [system][position]
    std::vector<Level> levels;
    {
        Level L0(ns);
        const size_t per = size_t(nb) * r;
        for (int a = 0; a < ns; ++a) {
            const size_t qa = size_t(a) * 2 * (I - 1);
            for (int j = 0; j < I; ++j) {
                Pos p{};
                p.idx = j;
                p.D = Ad + size_t(a) * D.sA() + j * nb2;
                p.F = c.F.p + (size_t(a) * I + j) * nb;
                if (j >= 1) {  // L_j = A'_{j,j-1} = Asub[j-1]
                    p.PL = c.lr_P.p + (qa + (j - 1)) * per;
                    p.RL = c.lr_R.p + (qa + (j - 1)) * per;
                }
                if (j + 1 < I) {  // U_j = A'_{j,j+1} = Asup[j]
                    p.PU = c.lr_P.p + (qa + (I - 1) + j) * per;
                    p.RU = c.lr_R.p + (qa + (I - 1) + j) * per;
                }
                L0[a].push_back(p);
            }
        }
        levels.push_back(std::move(L0));
    }
    int nlev = 0;
    {
        int n = I;
        while (n > 1) { n = (n + 1) / 2; ++nlev; }
    }
    c.lr_Z.resize(std::max(nlev, 1));
    c.lr_Rn.resize(std::max(nlev, 1));
    c.lr_core.ensure(size_t(ns) * I * 4 * r * r);
    c.lr_T.ensure(size_t(ns) * I * 2 * r * nb);
    c.lr_vec.ensure(size_t(ns) * I * 4 * r);
    DBuf<int> flag;
    auto factor = [&](const std::vector<cplx*>& fa, const std::vector<int*>& fp, const std::vector<cplx*>& fd,
                      const std::vector<int>& orig) {
        flag.ensure(fa.size());
        flag.zero(s);
        lu_factor_batched(nb, nb, fa, fp, fd, flag.p, s, c.ws);
        lu_rcond_batched(nb, nb, c.ws.ptrs.p, nullptr, 0, c.ws.ptrs3.p, nullptr, 0, int(fa.size()), kRcondMin, flag.p,
                         nullptr, s);
        std::vector<int> hf(fa.size());
        QPS_D2H(hf.data(), flag.p, sizeof(int) * hf.size(), s);
        QPS_CUDA(cudaStreamSynchronize(s));
        int worst = -1;
        for (size_t q = 0; q < hf.size(); ++q)
            if (hf[q] && (worst < 0 || orig[q] < worst)) worst = orig[q];
        if (worst >= 0)
            throw Error(QPS_ERR_SOLVER,
                        "singular diagonal factor (resonant parameters?) at layer " + std::to_string(worst + 1),
                        worst + 1);
    };
    static const bool trace = getenv("QPS_BCR_TRACE") != nullptr;  // per-level timing to stderr (debug)
    cudaEvent_t te0 = nullptr, te1 = nullptr;
    if (trace) {
        QPS_CUDA(cudaEventCreate(&te0));
        QPS_CUDA(cudaEventCreate(&te1));
        QPS_CUDA(cudaEventRecord(te0, s));
    }
    auto tmark = [&](const char* what, int l, int cnt) {
        if (!trace) return;
        float ms = 0;
        QPS_CUDA(cudaEventRecord(te1, s));
        QPS_CUDA(cudaEventSynchronize(te1));
        QPS_CUDA(cudaEventElapsedTime(&ms, te0, te1));
        fprintf(stderr, "lr-bcr level %d (%d odd) %s: %.3f ms\n", l, cnt, what, ms);
        QPS_CUDA(cudaEventRecord(te0, s));
    };
    int lvl = 0;
    while (levels[lvl][0].size() > 1) {
        Level& cur = levels[lvl];
        const int sz = int(cur[0].size());
        const int nodd = sz / 2;
        // 1. factor the odd positions; Z = D^{-1} [PL PU], z_f = D^{-1} f
        DBuf<cplx>& Zb = c.lr_Z[lvl];
        Zb.ensure(size_t(ns) * nodd * nb * 2 * r);
        std::vector<cplx*> fa, fd, zb, vb;
        std::vector<int*> fp;
        std::vector<int> orig;
        for (int a = 0; a < ns; ++a)
            for (int o = 1; o < sz; o += 2) {
                Pos& p = cur[a][o];
                fa.push_back(p.D);
                fp.push_back(ipiv_of(a, p.idx));
                fd.push_back(dinv_of(a, p.idx));
                orig.push_back(p.idx);
                p.Z = Zb.p + (size_t(a) * nodd + o / 2) * nb * 2 * r;
                zb.push_back(p.Z);
                vb.push_back(p.F);
            }
        factor(fa, fp, fd, orig);
        tmark("factor", lvl, int(fa.size()));
        {  // stage [PL PU] (zeros where a coupling is absent), then solve in place
            QPS_CUDA(cudaMemsetAsync(Zb.p, 0, sizeof(cplx) * size_t(ns) * nodd * nb * 2 * r, s));
            for (int a = 0; a < ns; ++a)
                for (int o = 1; o < sz; o += 2) {
                    const Pos& p = cur[a][o];
                    if (p.PL)
                        QPS_CUDA(cudaMemcpyAsync(p.Z, p.PL, sizeof(cplx) * size_t(nb) * r, cudaMemcpyDeviceToDevice,
                                                 s));
                    if (p.PU)
                        QPS_CUDA(cudaMemcpyAsync(p.Z + size_t(nb) * r, p.PU, sizeof(cplx) * size_t(nb) * r,
                                                 cudaMemcpyDeviceToDevice, s));
                }
            lu_solve_batched(nb, nb, fa, fp, fd, zb, nb, 2 * r, s, c.ws);
            lu_solve_batched(nb, nb, fa, fp, fd, vb, nb, 1, s, c.ws);
        }
        tmark("solve", lvl, int(fa.size()));
        // 2. even positions: cores, products, rank-r updates, new couplings, RHS
        const int nsz = (sz + 1) / 2;
        DBuf<cplx>& Rn = c.lr_Rn[lvl];
        Rn.ensure(size_t(ns) * nsz * 2 * r * nb);
        std::vector<GemmTask> cores, prods, newr, upd;
        std::vector<GemvTask> v1, v2;
        Level nxt(ns);
        const size_t rn = size_t(r) * nb, rr = size_t(r) * r;
        for (int a = 0; a < ns; ++a) {
            for (int e = 0; e < sz; e += 2) {
                const Pos& pe = cur[a][e];
                const int q = e / 2;
                const size_t slot = size_t(a) * nsz + q;
                cplx* core = c.lr_core.p + slot * 4 * rr;  // [LU, LL, UL, UU]
                cplx* T = c.lr_T.p + slot * 2 * rn;       // [T1; T2] as two r x n blocks
                cplx* vec = c.lr_vec.p + slot * 4 * r;
                Pos np{};
                np.idx = pe.idx;
                np.D = pe.D;
                np.F = pe.F;
                GemmTask u{};
                const bool hm = e >= 1, hp = e + 1 < sz;
                if (hm) {
                    const Pos& po = cur[a][e - 1];
                    const cplx* ZL = po.Z;
                    const cplx* ZU = po.Z + size_t(nb) * r;
                    cores.push_back(gemm1(pe.RL, r, ZU, nb, nb, core + 0 * rr, r));  // R_L(e) Z_U(o)
                    cores.push_back(gemm1(pe.RL, r, ZL, nb, nb, core + 1 * rr, r));  // R_L(e) Z_L(o)
                    prods.push_back(gemm1(core + 0 * rr, r, po.RU, r, r, T, r));     // T1 = (R_L Z_U) R_U(o)
                    u.A[u.nseg] = pe.PL; u.lda[u.nseg] = nb; u.B[u.nseg] = T; u.ldb[u.nseg] = r; u.K[u.nseg] = r;
                    ++u.nseg;
                    if (e - 2 >= 0) {  // L'_e = -P_L(e) (R_L Z_L) R_L(o)
                        cplx* Rl = Rn.p + slot * 2 * rn;
                        newr.push_back(gemm1(core + 1 * rr, r, po.RL, r, r, Rl, r));
                        np.PL = pe.PL;
                        np.RL = Rl;
                    }
                    v1.push_back(gemv1(pe.RL, r, po.F, nb, vec));  // t = R_L(e) z_f(o)
                    v2.push_back(gemv1(pe.PL, nb, vec, r, pe.F));  // f_e -= P_L t
                }
                if (hp) {
                    const Pos& po = cur[a][e + 1];
                    const cplx* ZL = po.Z;
                    const cplx* ZU = po.Z + size_t(nb) * r;
                    cores.push_back(gemm1(pe.RU, r, ZL, nb, nb, core + 2 * rr, r));  // R_U(e) Z_L(o)
                    cores.push_back(gemm1(pe.RU, r, ZU, nb, nb, core + 3 * rr, r));  // R_U(e) Z_U(o)
                    prods.push_back(gemm1(core + 2 * rr, r, po.RL, r, r, T + rn, r));  // T2 = (R_U Z_L) R_L(o)
                    u.A[u.nseg] = pe.PU; u.lda[u.nseg] = nb; u.B[u.nseg] = T + rn; u.ldb[u.nseg] = r;
                    u.K[u.nseg] = r;
                    ++u.nseg;
                    if (e + 2 < sz) {  // U'_e = -P_U(e) (R_U Z_U) R_U(o)
                        cplx* Ru = Rn.p + slot * 2 * rn + rn;
                        newr.push_back(gemm1(core + 3 * rr, r, po.RU, r, r, Ru, r));
                        np.PU = pe.PU;
                        np.RU = Ru;
                    }
                    v1.push_back(gemv1(pe.RU, r, po.F, nb, vec + r));
                    v2.push_back(gemv1(pe.PU, nb, vec + r, r, pe.F));
                }
                if (u.nseg) {
                    u.C = pe.D;
                    u.ldc = nb;
                    upd.push_back(u);
                }
                nxt[a].push_back(np);
            }
        }
        zgemm_batched(r, r, one, zero, cores, s, c.ws.gemm_tasks, "lr_core");
        zgemm_batched(r, nb, one, zero, prods, s, c.ws.gemm_tasks, "lr_core");
        zgemm_batched(r, nb, mone, zero, newr, s, c.ws.gemm_tasks, "lr_core");  // L' = P_L (-(core) R)
        zgemm_batched(nb, nb, mone, one, upd, s, c.ws.gemm_tasks, "bcr_update");
        zgemv_batched(r, one, zero, v1, s, c.ws.gemv_tasks);
        zgemv_batched(nb, mone, one, v2, s, c.ws.gemv_tasks);
        tmark("update", lvl, int(fa.size()));
        levels.push_back(std::move(nxt));
        ++lvl;
    }
    // final block of every system
    {
        std::vector<cplx*> fa, fd, vb;
        std::vector<int*> fp;
        std::vector<int> orig;
        for (int a = 0; a < ns; ++a) {
            const Pos& p = levels[lvl][a][0];
            fa.push_back(p.D);
            fd.push_back(dinv_of(a, p.idx));
            fp.push_back(ipiv_of(a, p.idx));
            vb.push_back(p.F);
            orig.push_back(p.idx);
        }
        factor(fa, fp, fd, orig);
        lu_solve_batched(nb, nb, fa, fp, fd, vb, nb, 1, s, c.ws);
        tmark("final", lvl, int(fa.size()));
    }
    // back substitution: eta_o = z_o - Z_L (R_L(o) eta_{o-1}) - Z_U (R_U(o) eta_{o+1})
    for (int l = lvl - 1; l >= 0; --l) {
        const Level& cur = levels[l];
        const int sz = int(cur[0].size());
        std::vector<GemvTask> t1, t2;
        for (int a = 0; a < ns; ++a)
            for (int o = 1; o < sz; o += 2) {
                const Pos& p = cur[a][o];
                cplx* vec = c.lr_vec.p + (size_t(a) * I + p.idx) * 4 * r;
                GemvTask w{};
                if (p.RL) {
                    t1.push_back(gemv1(p.RL, r, cur[a][o - 1].F, nb, vec));
                    w.A[w.nseg] = p.Z; w.lda[w.nseg] = nb; w.x[w.nseg] = vec; w.n[w.nseg] = r; ++w.nseg;
                }
                if (p.RU && o + 1 < sz) {
                    t1.push_back(gemv1(p.RU, r, cur[a][o + 1].F, nb, vec + r));
                    w.A[w.nseg] = p.Z + size_t(nb) * r; w.lda[w.nseg] = nb; w.x[w.nseg] = vec + r;
                    w.n[w.nseg] = r;
                    ++w.nseg;
                }
                if (w.nseg) {
                    w.y = p.F;
                    t2.push_back(w);
                }
            }
        zgemv_batched(r, one, zero, t1, s, c.ws.gemv_tasks);
        zgemv_batched(nb, mone, one, t2, s, c.ws.gemv_tasks);
    }
    tmark("backsub", lvl, 0);
    tl_mark(c, "backsub", s);
    if (trace) {
        QPS_CUDA(cudaEventDestroy(te0));
        QPS_CUDA(cudaEventDestroy(te1));
    }
    c.eta_valid = true;
}

// ---------------------------------------------------------------------------
// Cyclic reduction through the Woodbury identity.  The even-position updates
// never change a block's coupling bases: after any number of levels
//   D_j = D_j^0 - [P_L P_U] S_j,        f_j = f_j^0 - [P_L P_U] g_j
// with S_j (2r x n) and g_j (2r) accumulated from the rank-r products.  So every
// diagonal block is LU-factored ONCE, all I of them in one batch at level 0
// (W_j = D_j^0^{-1} [P_L P_U], y_j = D_j^0^{-1} f_j^0 in the same pass), and a
// block eliminated at level l >= 1 needs only its 2r x 2r capacitance matrix:
//   C = I - S W,   Z = D^{-1} [P_L P_U] = W C^{-1},
//   u = y - W g,   z = D^{-1} f = u + Z (S u).
// The deep levels (a handful of blocks each) become a few small GEMMs instead
// of a latency-bound dense LU per level; the level-0 batch runs at throughput.
// ---------------------------------------------------------------------------

// ||D_j^0||_1 of every diagonal block for the level-0 rcond screen, on the side
// stream while the couplings are compressed (Ad is final after the Schur step;
// bcr_solve_wb joins before its factorization overwrites Ad)
bool lr_eligible_pub(const Ctx& c) { return lr_eligible(c); }

bool rcond_enabled() {
    static const bool on = [] {  // QPS_RCOND=0: skip the level-0 rcond screen (A/B timing only)
        const char* e = getenv("QPS_RCOND");
        return !(e && !strcmp(e, "0"));
    }();
    return on;
}

void wb_anorm_async(Ctx& c, const cplx* Ad) {
    if (!lr_eligible(c) || !rcond_enabled()) return;
    const int npos = c.dims.nsys * c.dims.I;
    c.rc_anorm.ensure(npos);
    QPS_CUDA(cudaEventRecord(c.ev_fork, c.stream));
    QPS_CUDA(cudaStreamWaitEvent(c.side2, c.ev_fork, 0));
    batched_norm1(Ad, c.dims.nb, c.dims.nb, c.dims.nb2(), npos, c.rc_anorm.p, c.side2);
    QPS_CUDA(cudaEventRecord(c.ev_anorm, c.side2));
    c.anorm_pending = true;
}

// fixed unit-modulus probes (seeded phases), ||r_k||_1 = nb
void rc_probes(Ctx& c, int nb, cudaStream_t s) {
    if (c.rc_probe_n == nb) return;
    std::vector<cplx> pr(size_t(nb) * kRcProbe);
    uint64_t x = 0x243f6a8885a308d3ull;
    for (auto& z : pr) {
        x ^= x >> 12;
        x ^= x << 25;
        x ^= x >> 27;
        const double ph = 2.0 * kPi * double((x * 0x2545f4914f6cdd1dull) >> 11) * (1.0 / 9007199254740992.0);
        z = cplx{cos(ph), sin(ph)};
    }
    c.rc_probe.upload(pr, s);
    c.rc_probe_n = nb;
}

// single right-hand side per system: f on block 0 of every system (c.F)
void wb_stage_rhs(Ctx& c, cudaStream_t s) {
    const Dims& D = c.dims;
    const int I = D.I, nb = D.nb, ns = D.nsys;
    c.F.ensure(size_t(ns) * I * nb);
    c.F.zero(s);
    for (int a = 0; a < ns; ++a)
        QPS_CUDA(cudaMemcpyAsync(c.F.p + size_t(a) * I * nb, c.f.p + size_t(a) * nb, sizeof(cplx) * nb,
                                 cudaMemcpyDeviceToDevice, s));
}

// QPS_L0_CHUNKS (1..4, default 1): chunks of the early level-0 batch.  Measured
// at config 4: no gain (the GPU is busy throughout that window), kept for A/B
int l0_chunk_count(int npos) {
    static const int n = [] {
        const char* e = getenv("QPS_L0_CHUNKS");
        return e ? std::max(1, std::min(Ctx::kL0MaxChunks, atoi(e))) : 1;
    }();
    return npos >= 64 * n ? n : 1;
}
int l0_chunk_begin(int npos, int nch, int k) { return int((int64_t(npos) * k) / nch); }
void l0_streams(Ctx& c) {
    if (c.l0_s[0]) return;
    // below the main stream by default: the main stream's compression (whose
    // bases every chunk's solve needs) must not be starved by the factorization
    int lo = 0, hi = 0;
    QPS_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    const int main_prio = hi < lo ? hi + 1 : hi;
    const char* e = getenv("QPS_L0_PRIO");  // hi | main | below (default) | lo
    int prio = std::min(lo, main_prio + 1);
    if (e && !strcmp(e, "hi")) prio = hi;
    else if (e && !strcmp(e, "main")) prio = main_prio;
    else if (e && !strcmp(e, "lo")) prio = lo;
    for (int k = 0; k < Ctx::kL0MaxChunks; ++k) {
        QPS_CUDA(cudaStreamCreateWithPriority(&c.l0_s[k], cudaStreamNonBlocking, prio));
        QPS_CUDA(cudaEventCreateWithFlags(&c.l0_ev[k], cudaEventDisableTiming));
    }
}

// Level 0 of the Woodbury reduction on the factor stream as soon as the
// compressed bases exist: W_j = D_j^{-1} [P_L P_U f_j probes] with the factors
// of wb_factor_async, the rcond screen, y = D^{-1} f into F -- overlapping the
// projection R = P^* C that the main stream runs next (lr_compress)
void wb_level0_async(Ctx& c) {
    if (!c.factor_pending || !c.wb_Ad) return;
    const Dims& D = c.dims;
    const int I = D.I, nb = D.nb, ns = D.nsys, r = c.lr_r, r2 = 2 * r, npos = ns * I;
    const int m = std::max(1, c.nrhs);
    const size_t nb2 = D.nb2(), dsz = lu_dinv_elems(nb), fs = size_t(nb) * m, per = size_t(nb) * r;
    const int wc = r2 + m + kRcProbe;
    cudaStream_t f = c.factor_stream;
    // the right-hand sides [P_L P_U f probes] are staged on the main stream
    // (where the bases were just produced): with a chunked factorization each
    // chunk's solve then waits only for its own factors
    cudaStream_t st = c.l0_chunks > 1 ? c.stream : f;
    if (st != c.stream) {
        QPS_CUDA(cudaEventRecord(c.ev_fork, c.stream));  // the bases P are queued
        QPS_CUDA(cudaStreamWaitEvent(f, c.ev_fork, 0));
    }
    if (m == 1) wb_stage_rhs(c, st);
    rc_probes(c, nb, st);
    c.lr_W0.ensure(size_t(npos) * nb * wc);
    { QPS_NOTE_LAUNCH(); stage_bases_kernel<<<dim3(npos, 16), 256, 0, st>>>(I, nb, per, c.lr_P.p, c.F.p, m,
                                                                             c.rc_probe.p, kRcProbe, c.lr_W0.p); }
    QPS_CUDA(cudaGetLastError());
    std::vector<cplx*> fa(npos), fd(npos), wb(npos);
    std::vector<int*> fp(npos);
    for (int q = 0; q < npos; ++q) {
        fa[q] = c.wb_Ad + size_t(q) * nb2;
        fp[q] = c.ipiv.p + size_t(q) * nb;
        fd[q] = c.dinv.p + size_t(q) * dsz;
        wb[q] = c.lr_W0.p + size_t(q) * nb * wc;
    }
    nvtxRangePushA("bcr_level0");  // the level-0 batch: factorization (wb_factor_async) and this solve
    tl_mark(c, "level0-staged(side)", f);
    if (c.l0_chunks == 1) {
        lu_solve_batched(nb, nb, fa, fp, fd, wb, nb, wc, f, c.ws2);
        tl_mark(c, "level0-solved(side)", f);
    } else {
        QPS_CUDA(cudaEventRecord(c.ev_fork, st));  // staged
        for (int k = 0; k < c.l0_chunks; ++k) {
            const int b0 = l0_chunk_begin(npos, c.l0_chunks, k), b1 = l0_chunk_begin(npos, c.l0_chunks, k + 1);
            QPS_CUDA(cudaStreamWaitEvent(c.l0_s[k], c.ev_fork, 0));
            const std::vector<cplx*> ca(fa.begin() + b0, fa.begin() + b1), cd(fd.begin() + b0, fd.begin() + b1),
                cw(wb.begin() + b0, wb.begin() + b1);
            const std::vector<int*> cp(fp.begin() + b0, fp.begin() + b1);
            lu_solve_batched(nb, nb, ca, cp, cd, cw, nb, wc, c.l0_s[k], c.l0_ws[k]);
            QPS_CUDA(cudaEventRecord(c.l0_ev[k], c.l0_s[k]));
            QPS_CUDA(cudaStreamWaitEvent(f, c.l0_ev[k], 0));
        }
    }
    nvtxRangePop();
    c.bcr_flag_h.ensure(npos);
    QPS_D2H(c.bcr_flag_h.p, c.l0_flag.p, sizeof(int) * npos, f);
    c.rc_flag.ensure(npos);
    c.rc_sus.ensure(npos);
    c.rc_estlo.ensure(npos);
    QPS_CUDA(cudaMemsetAsync(c.rc_flag.p, 0, sizeof(int) * npos, f));
    QPS_CUDA(cudaMemsetAsync(c.rc_sus.p, 0, sizeof(int) * npos, f));
    if (rcond_enabled())
        rcond_screen(c.lr_W0.p, size_t(nb) * wc, nb, r2 + m, kRcProbe, c.rc_anorm.p, double(nb), npos, kRcondMin,
                     kRcSuspect, c.rc_flag.p, c.rc_sus.p, c.rc_estlo.p, f);
    c.rc_flag_h.ensure(2 * size_t(npos));
    QPS_D2H(c.rc_flag_h.p, c.rc_flag.p, sizeof(int) * npos, f);
    QPS_D2H(c.rc_flag_h.p + npos, c.rc_sus.p, sizeof(int) * npos, f);
    QPS_CUDA(cudaMemcpy2DAsync(c.F.p, sizeof(cplx) * fs, c.lr_W0.p + size_t(r2) * nb, sizeof(cplx) * nb * wc,
                               sizeof(cplx) * fs, npos, cudaMemcpyDeviceToDevice, f));
    tl_mark(c, "level0-solve(side)", f);
    QPS_CUDA(cudaEventRecord(c.ev_l0, f));
    c.l0_async = true;
}

void wb_factor_async(Ctx& c, cplx* Ad) {
    const Dims& D = c.dims;
    const int npos = D.nsys * D.I, nb = D.nb;
    const size_t nb2 = D.nb2(), dsz = lu_dinv_elems(nb);
    // high priority (the corner stream, idle by now): the GPU is throughput-
    // bound here and the factorization plus the level-0 solve are the longer
    // chain (measured 150 ms per config-4 solve vs 155 ms with the
    // factorization on the low-priority side3, QPS_FACTOR_STREAM=low)
    static const bool low = [] {
        const char* e = getenv("QPS_FACTOR_STREAM");
        return e && !strcmp(e, "low");
    }();
    cudaStream_t fs = low ? c.side3 : c.side;
    c.factor_stream = fs;
    c.wb_Ad = Ad;
    c.l0_async = false;
    QPS_CUDA(cudaEventRecord(c.ev_fork, c.stream));  // A' is final (the Schur updates are queued)
    QPS_CUDA(cudaStreamWaitEvent(fs, c.ev_fork, 0));
    // ||D_j^0||_1 for the rcond screen, on this stream before the factorization
    // overwrites Ad (not behind the compression sample on side2)
    if (rcond_enabled()) {
        c.rc_anorm.ensure(npos);
        batched_norm1(Ad, nb, nb, nb2, npos, c.rc_anorm.p, fs);
    }
    c.anorm_pending = false;
    c.ipiv.ensure(size_t(npos) * nb);
    c.dinv.ensure(size_t(npos) * dsz);
    c.l0_flag.ensure(npos);
    c.l0_flag.zero(fs);
    std::vector<cplx*> fa(npos), fd(npos);
    std::vector<int*> fp(npos);
    for (int q = 0; q < npos; ++q) {
        fa[q] = Ad + size_t(q) * nb2;
        fp[q] = c.ipiv.p + size_t(q) * nb;
        fd[q] = c.dinv.p + size_t(q) * dsz;
    }
    if (!c.ev_f0) {
        QPS_CUDA(cudaEventCreate(&c.ev_f0));
        QPS_CUDA(cudaEventCreate(&c.ev_f1));
    }
    QPS_CUDA(cudaEventRecord(c.ev_f0, fs));
    nvtxRangePushA("bcr_level0");
    c.l0_chunks = l0_chunk_count(npos);
    if (c.l0_chunks == 1) {
        lu_factor_batched(nb, nb, fa, fp, fd, c.l0_flag.p, fs, c.ws2);
    } else {
        l0_streams(c);
        QPS_CUDA(cudaEventRecord(c.ev_fork, fs));  // the norms have read Ad
        for (int k = 0; k < c.l0_chunks; ++k) {
            const int b0 = l0_chunk_begin(npos, c.l0_chunks, k), b1 = l0_chunk_begin(npos, c.l0_chunks, k + 1);
            QPS_CUDA(cudaStreamWaitEvent(c.l0_s[k], c.ev_fork, 0));
            const std::vector<cplx*> ca(fa.begin() + b0, fa.begin() + b1), cd(fd.begin() + b0, fd.begin() + b1);
            const std::vector<int*> cp(fp.begin() + b0, fp.begin() + b1);
            lu_factor_batched(nb, nb, ca, cp, cd, c.l0_flag.p + b0, c.l0_s[k], c.l0_ws[k]);
            QPS_CUDA(cudaEventRecord(c.l0_ev[k], c.l0_s[k]));
            QPS_CUDA(cudaStreamWaitEvent(fs, c.l0_ev[k], 0));  // fs joins every chunk (fallback paths wait on fs)
        }
    }
    nvtxRangePop();
    QPS_CUDA(cudaEventRecord(c.ev_f1, fs));
    tl_mark(c, "factor(side)", fs);
    QPS_CUDA(cudaEventRecord(c.ev_factor, fs));
    c.factor_pending = true;
}

void wb_refine_step(Ctx& c, cplx* Ad, int slot, bool apply);

void bcr_solve_wb(Ctx& c, cplx* Ad) {
    ProfPhase phase("bcr");
    ++c.n_factorizations;
    const Dims& D = c.dims;
    const int I = D.I, nb = D.nb, ns = D.nsys, r = c.lr_r, r2 = 2 * r;
    const size_t nb2 = D.nb2();
    cudaStream_t s = c.stream;
    const cplx one{1, 0}, mone{-1, 0}, zero{0, 0};
    const int npos = ns * I;
    // right-hand sides: m = c.nrhs columns per block (nb x m, ld nb); with m = 1
    // the system's f on block 0, with m > 1 the caller has filled c.F
    const int m = std::max(1, c.nrhs);
    if (m == 1 && !c.l0_async) wb_stage_rhs(c, s);
    const size_t fs = size_t(nb) * m;  // per-block stride of F
    RhsOps rhs{m, s, c.ws};
    c.ipiv.ensure(size_t(npos) * nb);
    const size_t dsz = lu_dinv_elems(nb);
    c.dinv.ensure(size_t(npos) * dsz);
    const int wc = r2 + m + kRcProbe;  // [W | y | rcond probes] per block
    if (!c.l0_async) c.lr_W0.ensure(size_t(npos) * nb * wc);
    c.lr_S.ensure(size_t(npos) * r2 * nb);
    c.lr_g.ensure(size_t(npos) * r2 * m);
    c.lr_S.zero(s);
    c.lr_g.zero(s);
    c.lr_core.ensure(size_t(npos) * 4 * r * r);
    c.lr_vec.ensure(size_t(npos) * r2 * m);
    static const bool trace = getenv("QPS_BCR_TRACE") != nullptr;  // per-level timing to stderr (debug)
    cudaEvent_t te0 = nullptr, te1 = nullptr;
    if (trace) {
        QPS_CUDA(cudaEventCreate(&te0));
        QPS_CUDA(cudaEventCreate(&te1));
        QPS_CUDA(cudaEventRecord(te0, s));
    }
    auto tmark = [&](const char* what, int l, int cnt) {
        if (!trace) return;
        float ms = 0;
        QPS_CUDA(cudaEventRecord(te1, s));
        QPS_CUDA(cudaEventSynchronize(te1));
        QPS_CUDA(cudaEventElapsedTime(&ms, te0, te1));
        fprintf(stderr, "wb-bcr level %d (%d blocks) %s: %.3f ms\n", l, cnt, what, ms);
        QPS_CUDA(cudaEventRecord(te0, s));
    };
    DBuf<int> flag;
    DBuf<int> capflag;  // Gauss-Jordan capacitance inverses: flags of every level, checked at the end
    capflag.ensure(size_t(npos) + ns);
    capflag.zero(s);
    std::vector<int> cap_orig;
    auto check = [&](const std::vector<int>& orig) {
        std::vector<int> hf(orig.size());
        QPS_D2H(hf.data(), flag.p, sizeof(int) * hf.size(), s);
        QPS_CUDA(cudaStreamSynchronize(s));
        int worst = -1;
        for (size_t q = 0; q < hf.size(); ++q)
            if (hf[q] && (worst < 0 || orig[q] < worst)) worst = orig[q];
        if (worst >= 0)
            throw Error(QPS_ERR_SOLVER,
                        "singular diagonal factor (resonant parameters?) at layer " + std::to_string(worst + 1),
                        worst + 1);
    };
    using Pos = WbPos;
    using Level = std::vector<std::vector<Pos>>;
    auto& levels = c.wb_levels;
    levels.clear();
    auto W0_of = [&](int j) { return c.lr_W0.p + size_t(j) * nb * wc; };
    auto S_of = [&](int j) { return c.lr_S.p + size_t(j) * r2 * nb; };
    auto g_of = [&](int j) { return c.lr_g.p + size_t(j) * r2 * m; };  // r2 x m, ld r2
    std::vector<int> l0_orig;  // level-0 positions whose singular flags are checked at the end
    bool early_factor = false;  // level 0 factored by wb_factor_async
    const bool l0_async_done = c.l0_async;  // and solved by wb_level0_async
    // ---- level 0: factor every block, W = D^{-1} [P_L P_U], y = D^{-1} f
    cudaEvent_t f0 = nullptr, f1 = nullptr;  // factor_ms of the phase times
    QPS_CUDA(cudaEventCreate(&f0));
    QPS_CUDA(cudaEventCreate(&f1));
    QPS_CUDA(cudaEventRecord(f0, s));
    nvtxRangePushA("bcr_level0");  // ncu --nvtx --nvtx-include "bcr_level0/" selects this batch
    {
        Level L0(ns);
        const size_t per = size_t(nb) * r;
        std::vector<cplx*> fa, fd, wb, vb;
        std::vector<int*> fp;
        std::vector<int> orig;
        if (!c.l0_async) rc_probes(c, nb, s);
        if (c.l0_async) {
            c.anorm_pending = false;  // the factor stream already waited for the norms and solved level 0
        } else if (c.anorm_pending) {  // ||D_j^0||_1 (side stream, before the factorization overwrites Ad)
            QPS_CUDA(cudaStreamWaitEvent(s, c.ev_anorm, 0));
            c.anorm_pending = false;
        } else if (rcond_enabled()) {
            c.rc_anorm.ensure(npos);
            batched_norm1(Ad, nb, nb, nb2, npos, c.rc_anorm.p, s);
        }
        if (!c.l0_async) {
            { QPS_NOTE_LAUNCH(); stage_bases_kernel<<<dim3(npos, 16), 256, 0, s>>>(I, nb, per, c.lr_P.p, c.F.p, m,
                                                                                    c.rc_probe.p, kRcProbe, c.lr_W0.p); }
            QPS_CUDA(cudaGetLastError());
        }
        for (int a = 0; a < ns; ++a) {
            const size_t qa = size_t(a) * 2 * (I - 1);
            for (int j = 0; j < I; ++j) {
                Pos p{};
                p.idx = j;
                p.j = a * I + j;
                p.F = c.F.p + size_t(p.j) * fs;
                if (j >= 1) {
                    p.PL = c.lr_P.p + (qa + (j - 1)) * per;
                    p.RL = c.lr_R.p + (qa + (j - 1)) * per;
                }
                if (j + 1 < I) {
                    p.PU = c.lr_P.p + (qa + (I - 1) + j) * per;
                    p.RU = c.lr_R.p + (qa + (I - 1) + j) * per;
                }
                p.Z = W0_of(p.j);
                L0[a].push_back(p);
                fa.push_back(Ad + size_t(a) * D.sA() + j * nb2);
                fp.push_back(c.ipiv.p + size_t(p.j) * nb);
                fd.push_back(c.dinv.p + size_t(p.j) * dsz);
                wb.push_back(W0_of(p.j));
                vb.push_back(p.F);
                orig.push_back(j);
            }
        }
        flag.ensure(fa.size());
        flag.zero(s);
        static const bool separate = [] {  // QPS_WB_L0=separate: factor, then solve (A/B)
            const char* e = getenv("QPS_WB_L0");
            return e && !strcmp(e, "separate");
        }();
        if (c.l0_async) {
            // factored and solved on the factor stream (wb_factor_async +
            // wb_level0_async) while the couplings were compressed
            QPS_CUDA(cudaStreamWaitEvent(s, c.ev_l0, 0));
            c.l0_async = false;
            c.factor_pending = false;
            early_factor = true;
            l0_orig = orig;
        } else if (c.factor_pending) {
            // factored on the side stream during the compression: solve only
            QPS_CUDA(cudaStreamWaitEvent(s, c.ev_factor, 0));
            c.factor_pending = false;
            early_factor = true;
            lu_solve_batched(nb, nb, fa, fp, fd, wb, nb, wc, s, c.ws);
            c.bcr_flag_h.ensure(fa.size());
            QPS_D2H(c.bcr_flag_h.p, c.l0_flag.p, sizeof(int) * fa.size(), s);
            l0_orig = orig;
            tmark("solve with the early factors", 0, int(fa.size()));
        } else if (c.refine_ready) {
            // refinement replays the solve: factors that stay usable (no spine)
            lu_factor_batched(nb, nb, fa, fp, fd, flag.p, s, c.ws);
            lu_solve_batched(nb, nb, fa, fp, fd, wb, nb, wc, s, c.ws);
            c.bcr_flag_h.ensure(fa.size());
            QPS_D2H(c.bcr_flag_h.p, flag.p, sizeof(int) * fa.size(), s);
            l0_orig = orig;
            tmark("factor, solve (refinable)", 0, int(fa.size()));
        } else if (separate) {
            lu_factor_batched(nb, nb, fa, fp, fd, flag.p, s, c.ws);
            lu_rcond_batched(nb, nb, c.ws.ptrs.p, nullptr, 0, c.ws.ptrs3.p, nullptr, 0, int(fa.size()), kRcondMin, flag.p,
                         nullptr, s);
            check(orig);
            tmark("factor", 0, int(fa.size()));
            lu_solve_batched(nb, nb, fa, fp, fd, wb, nb, wc, s, c.ws);
        } else {
            // the D_j^0 factors are used only for W_j: the forward substitution
            // rides along the factorization
            lu_factor_solve_batched(nb, nb, fa, fp, fd, wb, nb, wc, flag.p, s, c.ws);
            // singular flags read back asynchronously, checked after the levels
            c.bcr_flag_h.ensure(fa.size());
            QPS_D2H(c.bcr_flag_h.p, flag.p, sizeof(int) * fa.size(), s);
            l0_orig = orig;
            tmark("factor+solve", 0, int(fa.size()));
        }
        // rcond screen from the probe columns (certain flags + suspects), read
        // back with the singular flags
        if (!early_factor || !l0_async_done) {
        c.rc_flag.ensure(npos);
        c.rc_sus.ensure(npos);
        c.rc_estlo.ensure(npos);
        QPS_CUDA(cudaMemsetAsync(c.rc_flag.p, 0, sizeof(int) * npos, s));
        QPS_CUDA(cudaMemsetAsync(c.rc_sus.p, 0, sizeof(int) * npos, s));
        if (rcond_enabled())
            rcond_screen(c.lr_W0.p, size_t(nb) * wc, nb, r2 + m, kRcProbe, c.rc_anorm.p, double(nb), npos, kRcondMin,
                     kRcSuspect, c.rc_flag.p, c.rc_sus.p, c.rc_estlo.p, s);
        c.rc_flag_h.ensure(2 * size_t(npos));
        QPS_D2H(c.rc_flag_h.p, c.rc_flag.p, sizeof(int) * npos, s);
        QPS_D2H(c.rc_flag_h.p + npos, c.rc_sus.p, sizeof(int) * npos, s);
        }
        QPS_CUDA(cudaEventRecord(f1, s));
        tl_mark(c, "level0", s);
        nvtxRangePop();
        // y = D^{-1} f back into F (column 2r of every W_j)
        if (!l0_async_done)
            QPS_CUDA(cudaMemcpy2DAsync(c.F.p, sizeof(cplx) * fs, c.lr_W0.p + size_t(r2) * nb,
                                       sizeof(cplx) * nb * wc, sizeof(cplx) * fs, npos, cudaMemcpyDeviceToDevice, s));
        tmark("solve", 0, int(fa.size()));
        levels.push_back(std::move(L0));
    }
    int nlev = 0;
    {
        int n = I;
        while (n > 1) { n = (n + 1) / 2; ++nlev; }
    }
    c.lr_Z.resize(std::max(nlev + 1, 1));
    c.lr_Rn.resize(std::max(nlev, 1));
    const size_t rr = size_t(r) * r, rn = size_t(r) * nb;
    // eliminate the listed blocks at level lvl (updated ones through their
    // capacitance matrix); sets Z and overwrites F with z = D^{-1} f
    // the right-hand-side half of every level (u = y - W g, a = S u,
    // z = u + Z a, g += R z) runs on the side stream, one level behind the
    // factor half that only the next level's factors depend on: the deep
    // levels' latency-bound launches of the two halves overlap
    static const bool rhs_side_off = [] {  // QPS_WB_RHS_STREAM=0: both halves on the main stream (A/B)
        const char* e = getenv("QPS_WB_RHS_STREAM");
        return e && !strcmp(e, "0");
    }();
    const cudaStream_t rs = rhs_side_off ? s : c.side;
    RhsOps rhs2{m, rs, rhs_side_off ? c.ws : c.ws2};
    if (!c.ev_rhs) QPS_CUDA(cudaEventCreateWithFlags(&c.ev_rhs, cudaEventDisableTiming));
    if (rs != s) {  // the side stream starts after level 0 (y, W) is in place
        QPS_CUDA(cudaEventRecord(c.ev_rhs, s));
        QPS_CUDA(cudaStreamWaitEvent(rs, c.ev_rhs, 0));
    }
    c.lr_a.ensure(size_t(npos) * r2 * m);  // per position: the RHS half may lag a level behind
    auto eliminate = [&](std::vector<Pos*>& blk, int lvl) {
        std::vector<Pos*> up;
        for (Pos* p : blk)
            if (p->updated) up.push_back(p);
        if (up.empty()) return;
        const int cnt = int(up.size());
        c.lr_Cm.ensure(size_t(cnt) * r2 * r2);
        c.lr_Ci.ensure(size_t(cnt) * r2 * r2);
        c.lr_Cpiv.ensure(size_t(cnt) * r2);
        const size_t cds = lu_dinv_elems(r2);
        c.lr_Cdinv.ensure(size_t(cnt) * cds);
        DBuf<cplx>& Zb = c.lr_Z[lvl];
        Zb.ensure(size_t(cnt) * nb * r2);
        { QPS_NOTE_LAUNCH(); set_identity_kernel<<<cnt, 256, 0, s>>>(r2, c.lr_Cm.p); }
        QPS_CUDA(cudaGetLastError());
        static const bool cap_lu = [] {  // QPS_WB_CAP=lu: LU + solve against I instead of Gauss-Jordan
            const char* e = getenv("QPS_WB_CAP");
            return e && !strcmp(e, "lu");
        }();
        const bool gjinv = !cap_lu && r2 <= kGjMax;
        if (!gjinv) {
            { QPS_NOTE_LAUNCH(); set_identity_kernel<<<cnt, 256, 0, s>>>(r2, c.lr_Ci.p); }
            QPS_CUDA(cudaGetLastError());
        }
        std::vector<GemmTask> mt(cnt), z(cnt);
        std::vector<GemmTask> gu(cnt), ga(cnt), gz(cnt);
        std::vector<cplx*> ca, cd, ci;
        std::vector<int*> cp;
        std::vector<int> orig;
        for (int q = 0; q < cnt; ++q) {
            Pos& p = *up[q];
            const cplx* W = W0_of(p.j);
            cplx* Cm = c.lr_Cm.p + size_t(q) * r2 * r2;
            cplx* Ci = c.lr_Ci.p + size_t(q) * r2 * r2;
            mt[q] = gemm1(S_of(p.j), r2, W, nb, nb, Cm, r2);                      // C = I - S W
            z[q] = gemm1(W, nb, gjinv ? Cm : Ci, r2, r2, Zb.p + size_t(q) * nb * r2, nb);  // Z = W C^{-1}
            cplx* aq = c.lr_a.p + size_t(p.j) * r2 * m;
            gu[q] = gemm1(W, nb, g_of(p.j), r2, r2, p.F, nb);                      // u = y - W g
            ga[q] = gemm1(S_of(p.j), r2, p.F, nb, nb, aq, r2);                     // a = S u
            gz[q] = gemm1(Zb.p + size_t(q) * nb * r2, nb, aq, r2, r2, p.F, nb);    // z = u + Z a
            ca.push_back(Cm);
            ci.push_back(Ci);
            cd.push_back(c.lr_Cdinv.p + size_t(q) * cds);
            cp.push_back(c.lr_Cpiv.p + size_t(q) * r2);
            orig.push_back(p.idx);
            p.Z = Zb.p + size_t(q) * nb * r2;
        }
        zgemm_batched(r2, r2, mone, one, mt, s, c.ws.gemm_tasks, "wb_cap");
        if (gjinv) {  // C <- C^{-1} in place; singular flags checked once after all levels
            static const bool gj_smem = [] {  // QPS_WB_GJ=smem: the shared-memory kernel (always for 2r != 96)
                const char* e = getenv("QPS_WB_GJ");
                return e && !strcmp(e, "smem");
            }();
            ProfScope ps("wb_gj", s, 8.0 * cnt * double(r2) * r2 * r2);
            if (gj_smem || r2 % 16 || r2 < 32 || r2 > 96) {
                static bool attr = false;
                if (!attr) {
                    QPS_CUDA(cudaFuncSetAttribute(gj_inverse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  int(kGjMax * kGjMax * sizeof(cplx))));
                    attr = true;
                }
                { QPS_NOTE_LAUNCH(); gj_inverse_kernel<<<cnt, 512, size_t(r2) * r2 * sizeof(cplx), s>>>(r2, c.lr_Cm.p,
                                                                                  capflag.p + cap_orig.size()); }
            } else {
                int* fl = capflag.p + cap_orig.size();
                QPS_NOTE_LAUNCH();
                switch (r2) {  // 2r for the adaptive widths r = 16, 24, ..., 48
                    case 32: gj_inverse_reg_kernel<32><<<cnt, 4 * 32, 0, s>>>(c.lr_Cm.p, fl); break;
                    case 48: gj_inverse_reg_kernel<48><<<cnt, 4 * 48, 0, s>>>(c.lr_Cm.p, fl); break;
                    case 64: gj_inverse_reg_kernel<64><<<cnt, 4 * 64, 0, s>>>(c.lr_Cm.p, fl); break;
                    case 80: gj_inverse_reg_kernel<80><<<cnt, 4 * 80, 0, s>>>(c.lr_Cm.p, fl); break;
                    default: gj_inverse_reg_kernel<96><<<cnt, 4 * 96, 0, s>>>(c.lr_Cm.p, fl); break;
                }
            }
            QPS_CUDA(cudaGetLastError());
            cap_orig.insert(cap_orig.end(), orig.begin(), orig.end());
        } else {
            flag.ensure(cnt);
            flag.zero(s);
            lu_factor_batched(r2, r2, ca, cp, cd, flag.p, s, c.ws);
            lu_rcond_batched(r2, r2, c.ws.ptrs.p, nullptr, 0, c.ws.ptrs3.p, nullptr, 0, cnt, kRcondMin, flag.p, nullptr, s);
            check(orig);
            lu_solve_batched(r2, r2, ca, cp, cd, ci, r2, r2, s, c.ws);
        }
        zgemm_batched(nb, r2, one, zero, z, s, c.ws.gemm_tasks, "wb_cap");
        if (rs != s) {  // Z of this level is queued
            QPS_CUDA(cudaEventRecord(c.ev_rhs, s));
            QPS_CUDA(cudaStreamWaitEvent(rs, c.ev_rhs, 0));
        }
        rhs2.run(nb, mone, one, gu);
        rhs2.run(r2, one, zero, ga);
        rhs2.run(nb, one, one, gz);
    };
    int lvl = 0;
    nvtxRangePushA("bcr_levels");  // the levels, final block and back substitution (ncu --nvtx-include)
    while (levels[lvl][0].size() > 1) {
        Level& cur = levels[lvl];
        const int sz = int(cur[0].size());
        std::vector<Pos*> odd;
        for (int a = 0; a < ns; ++a)
            for (int o = 1; o < sz; o += 2) odd.push_back(&cur[a][o]);
        eliminate(odd, lvl);
        tmark("eliminate", lvl, int(odd.size()));
        // even positions: cores, accumulated S and g, new right factors
        const int nsz = (sz + 1) / 2;
        DBuf<cplx>& Rn = c.lr_Rn[lvl];
        Rn.ensure(size_t(ns) * nsz * 2 * rn);
        std::vector<GemmTask> cores, prods, newr;
        std::vector<GemmTask> v1;
        Level nxt(ns);
        for (int a = 0; a < ns; ++a) {
            for (int e = 0; e < sz; e += 2) {
                const Pos& pe = cur[a][e];
                const size_t slot = size_t(a) * nsz + e / 2;
                cplx* core = c.lr_core.p + slot * 4 * rr;  // [LU, LL, UL, UU]
                cplx* S = S_of(pe.j);
                cplx* g = g_of(pe.j);
                Pos np = pe;
                np.PL = np.RL = np.PU = np.RU = nullptr;
                const bool hm = e >= 1, hp = e + 1 < sz;
                if (hm) {
                    const Pos& po = cur[a][e - 1];
                    const cplx* ZL = po.Z;
                    const cplx* ZU = po.Z + size_t(nb) * r;
                    cores.push_back(gemm1(pe.RL, r, ZU, nb, nb, core + 0 * rr, r));  // R_L(e) Z_U(o)
                    cores.push_back(gemm1(pe.RL, r, ZL, nb, nb, core + 1 * rr, r));  // R_L(e) Z_L(o)
                    prods.push_back(gemm1(core + 0 * rr, r, po.RU, r, r, S, r2));     // S_L += (R_L Z_U) R_U(o)
                    if (e - 2 >= 0) {
                        cplx* Rl = Rn.p + slot * 2 * rn;
                        newr.push_back(gemm1(core + 1 * rr, r, po.RL, r, r, Rl, r));
                        np.PL = pe.PL;
                        np.RL = Rl;
                    }
                    v1.push_back(gemm1(pe.RL, r, po.F, nb, nb, g, r2));  // g_L += R_L(e) z(o)
                    np.updated = true;
                }
                if (hp) {
                    const Pos& po = cur[a][e + 1];
                    const cplx* ZL = po.Z;
                    const cplx* ZU = po.Z + size_t(nb) * r;
                    cores.push_back(gemm1(pe.RU, r, ZL, nb, nb, core + 2 * rr, r));  // R_U(e) Z_L(o)
                    cores.push_back(gemm1(pe.RU, r, ZU, nb, nb, core + 3 * rr, r));  // R_U(e) Z_U(o)
                    prods.push_back(gemm1(core + 2 * rr, r, po.RL, r, r, S + r, r2));  // S_U += (R_U Z_L) R_L(o)
                    if (e + 2 < sz) {
                        cplx* Ru = Rn.p + slot * 2 * rn + rn;
                        newr.push_back(gemm1(core + 3 * rr, r, po.RU, r, r, Ru, r));
                        np.PU = pe.PU;
                        np.RU = Ru;
                    }
                    v1.push_back(gemm1(pe.RU, r, po.F, nb, nb, g + r, r2));
                    np.updated = true;
                }
                nxt[a].push_back(np);
            }
        }
        zgemm_batched(r, r, one, zero, cores, s, c.ws.gemm_tasks, "lr_core");
        zgemm_batched(r, nb, one, one, prods, s, c.ws.gemm_tasks, "lr_core");
        zgemm_batched(r, nb, mone, zero, newr, s, c.ws.gemm_tasks, "lr_core");  // L' = P_L (-(core) R)
        rhs2.run(r, one, one, v1);
        tmark("update", lvl, int(odd.size()));
        levels.push_back(std::move(nxt));
        ++lvl;
    }
    tl_mark(c, "levels", s);
    {  // final block of every system
        std::vector<Pos*> fin;
        for (int a = 0; a < ns; ++a) fin.push_back(&levels[lvl][a][0]);
        eliminate(fin, lvl);
        tmark("final", lvl, int(fin.size()));
    }
    {
        float fms = 0;
        QPS_CUDA(cudaEventSynchronize(f1));
        int worst = -1;
        std::vector<int> suspects;
        for (size_t q = 0; q < l0_orig.size(); ++q) {
            if (c.bcr_flag_h[q] || c.rc_flag_h[q]) {
                if (worst < 0 || l0_orig[q] < worst) worst = l0_orig[q];
            } else if (c.rc_flag_h[npos + q]) {
                suspects.push_back(int(q));
            }
        }
        if (worst < 0 && !suspects.empty()) {
            // full zlacn2 estimate on U for the suspects: ||A^{-1}||_1 >= max(est_lo,
            // est(||U^{-1}||_1) / ||L||_1) with ||L||_1 <= n (|l_ij| <= 1)
            const int ns_ = int(suspects.size());
            std::vector<cplx*> ua, da;
            for (int q : suspects) {
                ua.push_back(Ad + size_t(q) * nb2);
                da.push_back(c.dinv.p + size_t(q) * dsz);
            }
            DBuf<cplx*> up, dp;
            DBuf<int> fl;
            DBuf<double> est;
            up.upload(ua, s);
            dp.upload(da, s);
            fl.ensure(ns_);
            fl.zero(s);
            est.ensure(ns_);
            lu_rcond_batched(nb, nb, up.p, nullptr, 0, dp.p, nullptr, 0, ns_, kRcondMin, fl.p, nullptr, s, est.p);
            std::vector<double> eu(ns_), el(npos);
            std::vector<unsigned long long> an(npos);
            QPS_D2H(eu.data(), est.p, sizeof(double) * ns_, s);
            QPS_D2H(el.data(), c.rc_estlo.p, sizeof(double) * npos, s);
            QPS_D2H(an.data(), c.rc_anorm.p, sizeof(unsigned long long) * npos, s);
            QPS_CUDA(cudaStreamSynchronize(s));
            for (int i = 0; i < ns_; ++i) {
                const int q = suspects[i];
                double a;
                std::memcpy(&a, &an[q], sizeof a);
                const double rc = 1.0 / (a * std::max(el[q], eu[i] / nb));
                if (!(rc > kRcondMin) && (worst < 0 || l0_orig[q] < worst)) worst = l0_orig[q];
            }
        }
        if (worst >= 0) {
            QPS_CUDA(cudaEventDestroy(f0));
            QPS_CUDA(cudaEventDestroy(f1));
            throw Error(QPS_ERR_SOLVER,
                        "singular diagonal factor (resonant parameters?) at layer " + std::to_string(worst + 1),
                        worst + 1);
        }
        QPS_CUDA(cudaEventElapsedTime(&fms, f0, f1));
        c.times.factor_ms = fms;
        if (early_factor) {  // the factorization itself ran on the side stream
            float ef = 0;
            QPS_CUDA(cudaEventElapsedTime(&ef, c.ev_f0, c.ev_f1));
            c.times.factor_ms = fms + ef;
        }
        QPS_CUDA(cudaEventDestroy(f0));
        QPS_CUDA(cudaEventDestroy(f1));
    }
    if (!cap_orig.empty()) {
        flag.ensure(cap_orig.size());
        QPS_CUDA(cudaMemcpyAsync(flag.p, capflag.p, sizeof(int) * cap_orig.size(), cudaMemcpyDeviceToDevice, s));
        check(cap_orig);
    }
    if (rs != s) {  // the right-hand-side half joins the main stream
        QPS_CUDA(cudaEventRecord(c.ev_rhs, rs));
        QPS_CUDA(cudaStreamWaitEvent(s, c.ev_rhs, 0));
    }
    // back substitution: eta_o = z_o - Z_L (R_L(o) eta_{o-1}) - Z_U (R_U(o) eta_{o+1})
    for (int l = lvl - 1; l >= 0; --l) {
        const Level& cur = levels[l];
        const int sz = int(cur[0].size());
        std::vector<GemmTask> t1, t2;
        for (int a = 0; a < ns; ++a)
            for (int o = 1; o < sz; o += 2) {
                const Pos& p = cur[a][o];
                cplx* vec = c.lr_vec.p + size_t(p.j) * r2 * m;  // r2 x m, ld r2
                GemmTask w{};
                if (p.RL) {
                    t1.push_back(gemm1(p.RL, r, cur[a][o - 1].F, nb, nb, vec, r2));
                    w.A[w.nseg] = p.Z; w.lda[w.nseg] = nb; w.B[w.nseg] = vec; w.ldb[w.nseg] = r2; w.K[w.nseg] = r;
                    ++w.nseg;
                }
                if (p.RU && o + 1 < sz) {
                    t1.push_back(gemm1(p.RU, r, cur[a][o + 1].F, nb, nb, vec + r, r2));
                    w.A[w.nseg] = p.Z + size_t(nb) * r; w.lda[w.nseg] = nb; w.B[w.nseg] = vec + r;
                    w.ldb[w.nseg] = r2;
                    w.K[w.nseg] = r;
                    ++w.nseg;
                }
                if (w.nseg) {
                    w.C = p.F;
                    w.ldc = nb;
                    t2.push_back(w);
                }
            }
        rhs.run(r, one, zero, t1);
        rhs.run(nb, mone, one, t2);
    }
    nvtxRangePop();
    tmark("backsub", lvl, 0);
    tl_mark(c, "backsub", s);
    if (trace) {
        QPS_CUDA(cudaEventDestroy(te0));
        QPS_CUDA(cudaEventDestroy(te1));
    }
    if (c.refine_ready) {
        const size_t np3 = 3 * size_t(c.dims.nsys) * c.dims.I;  // per-block norms: r before, r after, f
        c.ref_nrm.ensure(np3);
        QPS_CUDA(cudaMemsetAsync(c.ref_nrm.p, 0, np3 * sizeof(double), s));
        for (int it = 0; it < c.refine_used; ++it) wb_refine_step(c, Ad, it == 0 ? 0 : -1, true);
        static const bool check = getenv("QPS_REFINE_CHECK") != nullptr;  // residual after the last step too
        if (check) wb_refine_step(c, Ad, 1, false);
        c.ref_nrm_h.ensure(np3);
        QPS_D2H(c.ref_nrm_h.p, c.ref_nrm.p, np3 * sizeof(double), s);  // combined after the solve's final sync
        c.ref_nrm_n = int(np3 / 3);
        tl_mark(c, "refine", s);
    }
    c.refine_ready = false;
    c.eta_valid = true;
}

// One step of iterative refinement of the Woodbury solve: r = f - A' eta with
// the unfactored diagonal blocks (ref_D) and couplings (raw A minus the
// deferred proxy terms Bc X), then A' delta = r by replaying the reduction on
// r -- level-0 LU solves with the kept factors, the recorded levels' Z, S, W
// and right factors, the back substitution -- and eta += delta.  Cost: one
// pass over A' and one pass over the factors per step.  Cyclic reduction is
// less accurate than block Thomas at ill-conditioned angles; a step brings
// the solution back to the accuracy the factors' conditioning allows.
void wb_refine_step(Ctx& c, cplx* Ad, int slot, bool apply) {
    const Dims& D = c.dims;
    const int I = D.I, nb = D.nb, ns = D.nsys, r = c.lr_r, r2 = 2 * r, P = D.P;
    const int npos = ns * I, m = std::max(1, c.nrhs);
    const size_t nb2 = D.nb2(), fs = size_t(nb) * m, dsz = lu_dinv_elems(nb);
    const int wc = r2 + m + kRcProbe;
    cudaStream_t s = c.stream;
    const cplx one{1, 0}, mone{-1, 0}, zero{0, 0};
    RhsOps rhs{m, s, c.ws};
    ProfPhase phase("refine");
    cplx* eta = c.F.p;
    c.ref_R.ensure(size_t(npos) * fs);
    cplx* R = c.ref_R.p;
    // r = f
    if (m == 1) {
        QPS_CUDA(cudaMemsetAsync(R, 0, sizeof(cplx) * npos * fs, s));
        for (int a = 0; a < ns; ++a)
            QPS_CUDA(cudaMemcpyAsync(R + size_t(a) * I * fs, c.f.p + size_t(a) * nb, sizeof(cplx) * nb,
                                     cudaMemcpyDeviceToDevice, s));
    } else {
        QPS_CUDA(cudaMemcpyAsync(R, c.ref_F.p, sizeof(cplx) * npos * fs, cudaMemcpyDeviceToDevice, s));
    }
    // norms per block (one CTA each; combined on the host by the diagnostics)
    if (slot == 0) batched_fro(R, nb, m, nb, fs, npos, c.ref_nrm.p + 2 * size_t(npos), s);  // ||f||
    // r -= A' eta: D_j eta_j + L_j eta_{j-1} (one two-segment product), U_j eta_{j+1},
    // then the deferred proxy terms + Bc (X eta) of both couplings
    std::vector<GemmTask> t1, t2, tx, tb;
    c.ref_X.ensure(size_t(npos) * 2 * P * m);
    cplx* xe = c.ref_X.p;  // X eta of the two couplings per block: 2P x m, ld 2P
    const bool corr = c.couplings_deferred;
    for (int a = 0; a < ns; ++a)
        for (int j = 0; j < I; ++j) {
            const size_t q = size_t(a) * I + j;
            GemmTask g = gemm1(c.ref_D.p + q * nb2, nb, eta + q * fs, nb, nb, R + q * fs, nb);
            if (j >= 1) {
                g.nseg = 2;
                g.A[1] = c.ref_Al + size_t(a) * D.sU() + size_t(j - 1) * nb2;
                g.lda[1] = nb;
                g.B[1] = eta + (q - 1) * fs;
                g.ldb[1] = nb;
                g.K[1] = nb;
            }
            t1.push_back(g);
            if (j + 1 < I)
                t2.push_back(gemm1(c.ref_Au + size_t(a) * D.sU() + size_t(j) * nb2, nb, eta + (q + 1) * fs, nb, nb,
                                   R + q * fs, nb));
            if (corr) {
                GemmTask b{};
                b.C = R + q * fs;
                b.ldc = nb;
                if (j >= 1) {
                    const GemmTask& u = c.coupling_sub[size_t(a) * (I - 1) + j - 1];
                    tx.push_back(gemm1(u.B[0], u.ldb[0], eta + (q - 1) * fs, nb, nb, xe + q * 2 * P * m, 2 * P));
                    b.A[b.nseg] = u.A[0]; b.lda[b.nseg] = u.lda[0]; b.B[b.nseg] = xe + q * 2 * P * m;
                    b.ldb[b.nseg] = 2 * P; b.K[b.nseg] = P; ++b.nseg;
                }
                if (j + 1 < I) {
                    const GemmTask& u = c.coupling_sup[size_t(a) * (I - 1) + j];
                    tx.push_back(gemm1(u.B[0], u.ldb[0], eta + (q + 1) * fs, nb, nb, xe + q * 2 * P * m + P, 2 * P));
                    b.A[b.nseg] = u.A[0]; b.lda[b.nseg] = u.lda[0]; b.B[b.nseg] = xe + q * 2 * P * m + P;
                    b.ldb[b.nseg] = 2 * P; b.K[b.nseg] = P; ++b.nseg;
                }
                if (b.nseg) tb.push_back(b);
            }
        }
    rhs.run(nb, mone, one, t1);
    rhs.run(nb, mone, one, t2);
    if (corr) {
        RhsOps rx{m, s, c.ws};
        rx.run(P, one, zero, tx);
        rhs.run(nb, one, one, tb);
    }
    if (slot >= 0) batched_fro(R, nb, m, nb, fs, npos, c.ref_nrm.p + size_t(slot) * npos, s);
    if (!apply) return;
    // replay: level 0, delta_j = D_j^{-1} r_j with the kept LU factors
    {
        std::vector<cplx*> fa(npos), fd(npos), rb(npos);
        std::vector<int*> fp(npos);
        for (int q = 0; q < npos; ++q) {
            fa[q] = Ad + size_t(q) * nb2;
            fp[q] = c.ipiv.p + size_t(q) * nb;
            fd[q] = c.dinv.p + size_t(q) * dsz;
            rb[q] = R + size_t(q) * fs;
        }
        lu_solve_batched(nb, nb, fa, fp, fd, rb, nb, m, s, c.ws);
    }
    auto& levels = c.wb_levels;
    auto Rof = [&](const WbPos& p) { return R + size_t(p.j) * fs; };
    auto W0_of = [&](int j) { return c.lr_W0.p + size_t(j) * nb * wc; };
    auto S_of = [&](int j) { return c.lr_S.p + size_t(j) * r2 * nb; };
    c.lr_g.zero(s);
    auto g_of = [&](int j) { return c.lr_g.p + size_t(j) * r2 * m; };
    c.ref_A.ensure(size_t(npos) * r2 * m);
    auto elim = [&](const std::vector<const WbPos*>& blk) {
        std::vector<GemmTask> gu, ga, gz;
        for (const WbPos* p : blk) {
            if (!p->updated) continue;
            cplx* aq = c.ref_A.p + size_t(p->j) * r2 * m;
            cplx* F = Rof(*p);
            gu.push_back(gemm1(W0_of(p->j), nb, g_of(p->j), r2, r2, F, nb));  // u = y - W g
            ga.push_back(gemm1(S_of(p->j), r2, F, nb, nb, aq, r2));           // a = S u
            gz.push_back(gemm1(p->Z, nb, aq, r2, r2, F, nb));                 // z = u + Z a
        }
        rhs.run(nb, mone, one, gu);
        rhs.run(r2, one, zero, ga);
        rhs.run(nb, one, one, gz);
    };
    const int nlvl = int(levels.size()) - 1;  // the last entry holds the final block of every system
    for (int l = 0; l < nlvl; ++l) {
        const auto& cur = levels[l];
        const int sz = int(cur[0].size());
        std::vector<const WbPos*> odd;
        for (int a = 0; a < ns; ++a)
            for (int o = 1; o < sz; o += 2) odd.push_back(&cur[a][o]);
        elim(odd);
        std::vector<GemmTask> v1;
        for (int a = 0; a < ns; ++a)
            for (int e = 0; e < sz; e += 2) {
                const WbPos& pe = cur[a][e];
                if (e >= 1) v1.push_back(gemm1(pe.RL, r, Rof(cur[a][e - 1]), nb, nb, g_of(pe.j), r2));
                if (e + 1 < sz) v1.push_back(gemm1(pe.RU, r, Rof(cur[a][e + 1]), nb, nb, g_of(pe.j) + r, r2));
            }
        rhs.run(r, one, one, v1);
    }
    {
        std::vector<const WbPos*> fin;
        for (int a = 0; a < ns; ++a) fin.push_back(&levels[nlvl][a][0]);
        elim(fin);
    }
    for (int l = nlvl - 1; l >= 0; --l) {
        const auto& cur = levels[l];
        const int sz = int(cur[0].size());
        std::vector<GemmTask> t1b, t2b;
        for (int a = 0; a < ns; ++a)
            for (int o = 1; o < sz; o += 2) {
                const WbPos& p = cur[a][o];
                cplx* vec = c.ref_A.p + size_t(p.j) * r2 * m;
                GemmTask w{};
                if (p.RL) {
                    t1b.push_back(gemm1(p.RL, r, Rof(cur[a][o - 1]), nb, nb, vec, r2));
                    w.A[w.nseg] = p.Z; w.lda[w.nseg] = nb; w.B[w.nseg] = vec; w.ldb[w.nseg] = r2; w.K[w.nseg] = r;
                    ++w.nseg;
                }
                if (p.RU && o + 1 < sz) {
                    t1b.push_back(gemm1(p.RU, r, Rof(cur[a][o + 1]), nb, nb, vec + r, r2));
                    w.A[w.nseg] = p.Z + size_t(nb) * r; w.lda[w.nseg] = nb; w.B[w.nseg] = vec + r;
                    w.ldb[w.nseg] = r2; w.K[w.nseg] = r;
                    ++w.nseg;
                }
                if (w.nseg) {
                    w.C = Rof(p);
                    w.ldc = nb;
                    t2b.push_back(w);
                }
            }
        rhs.run(r, one, zero, t1b);
        rhs.run(nb, mone, one, t2b);
    }
    axpy_blocks(eta, R, size_t(npos) * fs, s);  // eta += delta
}

}  // namespace qpsb
