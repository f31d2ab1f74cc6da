// Complex FP64 device arithmetic shared by the dense kernels (linalg.cu,
// bcr_lr.cu).  cplx is the interleaved {re, im} of hankel.cuh.
#pragma once

#include <cuda_runtime.h>

#include "hankel.cuh"

namespace qpsb {

__device__ __forceinline__ cplx cmul(cplx a, cplx b) {
    return cplx{a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
}
__device__ __forceinline__ cplx cconj(cplx a) { return cplx{a.re, -a.im}; }
__device__ __forceinline__ cplx cdiv(cplx a, cplx b) {
    // Smith's algorithm
    if (fabs(b.re) >= fabs(b.im)) {
        const double r = b.im / b.re, den = b.re + b.im * r;
        return cplx{(a.re + a.im * r) / den, (a.im - a.re * r) / den};
    }
    const double r = b.re / b.im, den = b.re * r + b.im;
    return cplx{(a.re * r + a.im) / den, (a.im * r - a.re) / den};
}
__device__ __forceinline__ double cabs2(cplx a) { return a.re * a.re + a.im * a.im; }

// FP64 division costs ~600 cycles of latency on B200: reciprocals on latency-
// critical paths use an FP32 seed and two Newton steps (~1 ulp), falling back
// to division outside the FP32 exponent range.
__device__ __forceinline__ double fast_rcp(double x) {
    const double ax = fabs(x);
    if (!(ax > 1e-30 && ax < 1e30)) return 1.0 / x;
    double r = double(__frcp_rn(float(x)));
    r = fma(r, fma(-x, r, 1.0), r);
    r = fma(r, fma(-x, r, 1.0), r);
    return r;
}
// 1 / d for complex d != 0 (|d|^2 in range)
__device__ __forceinline__ cplx fast_cinv(cplx d) {
    const double n2 = d.re * d.re + d.im * d.im;
    if (!(n2 > 1e-280 && n2 < 1e280)) return cdiv(cplx{1.0, 0.0}, d);
    const double r = fast_rcp(n2);
    return cplx{d.re * r, -d.im * r};
}

}  // namespace qpsb
