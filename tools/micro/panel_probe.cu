// probes of the shared-memory panel kernel with parts removed
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../paper_1410_5003_b200/csrc/linalg.cu"
#include "../../paper_1410_5003_b200/csrc/prof.cu"
namespace qpsb {
template <int MODE>
__global__ void __launch_bounds__(kRegPanelMaxRows, 1)
    probe_kernel(int n, int ld, cplx* const* __restrict__ Ap, int* const* __restrict__ Pp, int c0, int w,
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
}
using namespace qpsb;
__global__ void fill_rand(cplx* A, size_t n, unsigned seed, int dim) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        unsigned x = unsigned(i) * 2654435761u + seed;
        x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
        const size_t e = i % (size_t(dim) * dim);
        A[i] = cplx{(x & 0xffff) / 65536.0 - 0.5 + ((e % dim) == (e / dim) ? 4.0 : 0.0), ((x >> 16) & 0xffff) / 65536.0 - 0.5};
    }
}
template <int MODE>
void run(const char* name, int n, cplx* const* dA, int* const* dP, int* sing, int* map) {
    cudaFuncSetAttribute(probe_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int R = 200;
    for (int i = 0; i < 5; ++i) probe_kernel<MODE><<<1, 608, 608 * 16 * 16>>>(n, n, dA, dP, 0, 16, sing, map);
    cudaEventRecord(e0);
    for (int i = 0; i < R; ++i) probe_kernel<MODE><<<1, 608, 608 * 16 * 16>>>(n, n, dA, dP, 0, 16, sing, map);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-36s %.2f us/launch\n", name, 1000.0 * ms / R);
}
int main() {
    const int n = 608;
    DBuf<cplx> A; A.ensure(size_t(n) * n);
    DBuf<int> piv, sing, map; piv.ensure(n); sing.ensure(1); map.ensure(64);
    DBuf<cplx*> dA; DBuf<int*> dP;
    std::vector<cplx*> hA{A.p}; std::vector<int*> hP{piv.p};
    dA.upload(hA, 0); dP.upload(hP, 0);
    fill_rand<<<256, 256>>>(A.p, size_t(n) * n, 7, n);
    run<0>("full", n, dA.p, dP.p, sing.p, map.p);
    run<0>("full (nullptr map)", n, dA.p, dP.p, sing.p, nullptr);
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
