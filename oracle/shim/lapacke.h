/* Test infrastructure (oracle build only). Prototype-only LAPACKE shim for the
 * unmodified reference sources (proj/src/linalg.cpp:72,93,115,220,229,281 and
 * proj/src/optimize.cpp:143), resolved at link time against OpenBLAS 0.3.15. */
#ifndef ORACLE_SHIM_LAPACKE_H
#define ORACLE_SHIM_LAPACKE_H
#include <complex>
typedef int lapack_int;
typedef std::complex<double> lapack_complex_double;
#define LAPACK_ROW_MAJOR 101
#define LAPACK_COL_MAJOR 102
extern "C" {
lapack_int LAPACKE_zgesdd(int layout, char jobz, lapack_int m, lapack_int n, lapack_complex_double* a,
                          lapack_int lda, double* s, lapack_complex_double* u, lapack_int ldu,
                          lapack_complex_double* vt, lapack_int ldvt);
lapack_int LAPACKE_zgeqrf(int layout, lapack_int m, lapack_int n, lapack_complex_double* a,
                          lapack_int lda, lapack_complex_double* tau);
lapack_int LAPACKE_zunmqr(int layout, char side, char trans, lapack_int m, lapack_int n, lapack_int k,
                          const lapack_complex_double* a, lapack_int lda,
                          const lapack_complex_double* tau, lapack_complex_double* c, lapack_int ldc);
lapack_int LAPACKE_zungqr(int layout, lapack_int m, lapack_int n, lapack_int k,
                          lapack_complex_double* a, lapack_int lda, const lapack_complex_double* tau);
lapack_int LAPACKE_zheevd(int layout, char jobz, char uplo, lapack_int n, lapack_complex_double* a,
                          lapack_int lda, double* w);
lapack_int LAPACKE_dgesv(int layout, lapack_int n, lapack_int nrhs, double* a, lapack_int lda,
                         lapack_int* ipiv, double* b, lapack_int ldb);
}
#endif
