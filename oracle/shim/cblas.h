/* Test infrastructure (oracle build only). Prototype-only CBLAS shim so the
 * unmodified reference sources under /root/reference/proj/src compile against
 * the LP64 OpenBLAS 0.3.15 shipped in the opencv wheel (no system BLAS here).
 * Only the symbols the reference calls are declared
 * (proj/src/einsum.cpp:54 cblas_zgemm). */
#ifndef ORACLE_SHIM_CBLAS_H
#define ORACLE_SHIM_CBLAS_H
#ifdef __cplusplus
extern "C" {
#endif
enum CBLAS_ORDER { CblasRowMajor = 101, CblasColMajor = 102 };
enum CBLAS_TRANSPOSE { CblasNoTrans = 111, CblasTrans = 112, CblasConjTrans = 113 };
void cblas_zgemm(enum CBLAS_ORDER order, enum CBLAS_TRANSPOSE ta, enum CBLAS_TRANSPOSE tb, int m,
                 int n, int k, const void* alpha, const void* a, int lda, const void* b, int ldb,
                 const void* beta, void* c, int ldc);
void openblas_set_num_threads(int n);
int openblas_get_num_threads(void);
#ifdef __cplusplus
}
#endif
#endif
