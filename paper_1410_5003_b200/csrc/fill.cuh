// Device fill: task descriptors shared by host orchestration and kernels.
#pragma once

#include "hankel.cuh"
#include "qps_internal.h"

namespace qpsb {

constexpr int kMaxSegs = 16;

// One plain-Nystrom block (kernel_quad_block, kernels.hpp:78-97, summed over
// shift terms with phase coefficients and over up to two wavenumbers with
// signs, i.e. the alpha recombination of assembly.hpp:95-112,338-397 fused in).
// Outputs the four kinds either into one [D S; T D*] block (assembly.hpp:320-327)
// or into four separate planes (ShiftBlockCache pieces).
struct PairTask {
    int t_off, nt;  // target points (pool offset, count)
    int s_off, ns;  // source nodes  (pool offset, count)
    int nk;
    double k[2], ksign[2];
    int nterm;
    int lsh[3];      // lattice shift index of each term (-1, 0, 1; for band logic)
    double tdx[3];   // target x shift per term
    double sdx[3];   // source x shift per term
    cplx coef[3];    // phase coefficient per term
    int self;        // 0: none; 1: smooth self (band |j + l N - m| <= a-1 skipped); 2: open-arc self
    int nseg;
    int seg_start[kMaxSegs + 1];
    int ident;       // subtract I on the value block, add I on the derivative block
    int accumulate;  // 0 overwrite, 1 add
    cplx *oD, *oS, *oT, *oDs;
    int ld;
    // Mirror (self 0 or 1): the pair (source n, target m, shift -l) has the
    // separation -r of (m, n, l), so one Hankel evaluation also gives the
    // transposed block's entry (n, m): S, T unchanged, D and D* exchanged,
    // weighted by the target's weight and mcoef.  Couplings: the block
    // A_{j+1,j} with A_{j,j+1}; smooth self blocks: the lower tile triangle
    // from the upper one (same block).
    int mirror;
    cplx mcoef[3];
    cplx *mD, *mS, *mT, *mDs;
    int mld;
};

// Combined-field proxy columns phi_p = D + ik S and their normal-derivative
// rows T + ik D* (proxy_block, kernels.hpp:294-308), summed over terms.
struct ProxyTask {
    int t_off, nt;
    int p_off, P;
    double k;
    int nterm;
    double tdx[2];
    cplx coef[2];
    int drow;  // row offset of the derivative rows (nt when stacked)
    int accumulate;
    cplx* out;
    int ld;
};

// Alpert hybrid Gauss-trapezoid log correction of one interface's self block
// (self_quad_parts, kernels.hpp:180-280): 2 x 15 auxiliary nodes per corrected
// row, scattered to 16 grid columns with Lagrange weights; out-of-period
// columns wrap onto the period with alpha^{+-1}.
struct AlpertTask {
    int t_off;  // pool offset of this interface's nodes (targets)
    int N;
    int smooth;
    int nseg;
    int seg_first;  // index of the first SegDesc of this interface
    int row_start;  // first global row of this task in the row list
    int nk;
    double k[2], ksign[2];
    cplx alpha, alpha_inv;
    int mode;  // 0: fused into a [D S;T D*] block; 1: cache (central planes + wrap band)
    long long aux_off;  // open arcs: offset of the host-computed auxiliary-node table (-1: evaluate on the device)
    cplx *oD, *oS, *oT, *oDs;  // block (mode 0) or central planes (mode 1)
    int ld;
    cplx* wrap;  // mode 1: N x 33 x 4 kinds band of out-of-period entries (incl. wrap removal)
};

struct DevPool {
    const double *x, *y, *nx, *ny, *w;
};

void upload_hankel_tables();
const double* device_near_table();

void launch_pair_fill(const std::vector<PairTask>& tasks, const DevPool& pool, int* d_err, cudaStream_t s,
                      DBuf<PairTask>& d_tasks, DBuf<int4>& d_tiles);
void launch_proxy_fill(const std::vector<ProxyTask>& tasks, const DevPool& pool, int* d_err, cudaStream_t s,
                       DBuf<ProxyTask>& d_tasks, DBuf<int4>& d_tiles);
void launch_alpert(const std::vector<AlpertTask>& tasks, int total_rows, const DevPool& pool,
                   const SegDesc* d_segs, const double* d_fourier, const double* d_aux, int* d_err, cudaStream_t s,
                   DBuf<AlpertTask>& d_tasks);
void launch_hankel_batch(int n, const double* d_x, cplx* d_h0, cplx* d_h1, cudaStream_t s);

}  // namespace qpsb
