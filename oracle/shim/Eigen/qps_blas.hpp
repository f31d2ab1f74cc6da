// ORACLE TEST INFRASTRUCTURE — not product code.
// Thin bindings to the OpenBLAS build bundled with numpy in this image
// (numpy.libs/libscipy_openblas64_-*.so, 64-bit integer CBLAS interface,
// symbol prefix `scipy_`).  Used by the Eigen shim for large complex products
// and triangular solves so the oracle's CPU timing reflects an optimised,
// threaded BLAS the way Eigen's own GEMM kernels would.
#pragma once

#include <complex>
#include <cstdint>

extern "C" {
void scipy_cblas_zgemm64_(int order, int ta, int tb, int64_t m, int64_t n, int64_t k, const void* alpha,
                          const void* a, int64_t lda, const void* b, int64_t ldb, const void* beta, void* c,
                          int64_t ldc);
void scipy_cblas_ztrsm64_(int order, int side, int uplo, int ta, int diag, int64_t m, int64_t n,
                          const void* alpha, const void* a, int64_t lda, void* b, int64_t ldb);
void scipy_openblas_set_num_threads64_(int n);
int scipy_openblas_get_num_threads64_(void);
}

namespace qps_blas {

enum { ColMajor = 102, NoTrans = 111, Trans = 112, ConjTrans = 113, Upper = 121, Lower = 122, NonUnit = 131,
       Unit = 132, Left = 141, Right = 142 };

inline int trans_code(char t) { return t == 'N' ? NoTrans : (t == 'T' ? Trans : ConjTrans); }

inline void zgemm(char ta, char tb, int64_t m, int64_t n, int64_t k, std::complex<double> alpha,
                  const std::complex<double>* a, int64_t lda, const std::complex<double>* b, int64_t ldb,
                  std::complex<double> beta, std::complex<double>* c, int64_t ldc) {
    scipy_cblas_zgemm64_(ColMajor, trans_code(ta), trans_code(tb), m, n, k, &alpha, a, lda, b, ldb, &beta, c,
                         ldc);
}

// side 'L'/'R', uplo 'U'/'L', trans 'N'/'T'/'C', diag 'U'/'N'
inline void ztrsm(char side, char uplo, char ta, char diag, int64_t m, int64_t n, std::complex<double> alpha,
                  const std::complex<double>* a, int64_t lda, std::complex<double>* b, int64_t ldb) {
    scipy_cblas_ztrsm64_(ColMajor, side == 'L' ? Left : Right, uplo == 'U' ? Upper : Lower, trans_code(ta),
                         diag == 'U' ? Unit : NonUnit, m, n, &alpha, a, lda, b, ldb);
}

inline void set_num_threads(int n) { scipy_openblas_set_num_threads64_(n); }
inline int get_num_threads() { return scipy_openblas_get_num_threads64_(); }

}  // namespace qps_blas
