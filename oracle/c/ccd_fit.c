/* ORACLE (test infrastructure only): monomial fit of the coplanarity cubic.
 *
 * Restates ``f @ _FIT.T`` of reference pkg/src/clothsim/collision/ccd.py:44
 * exactly as OpenBLAS dgemm evaluates it with k = 4 (probed in SURVEY.md section 7,
 * re-checked by tests/test_oracle_golden.py):
 *   m >= 2 : c_j = fma(f3,F[j][3], fma(f2,F[j][2], fma(f1,F[j][1], f0*F[j][0])))
 *   m == 1 : c_j = (f0*F[j][0] + f2*F[j][2]) + (f1*F[j][1] + f3*F[j][3])
 * Compiled with -ffp-contract=off so only the explicit fma() calls fuse.
 */
#include <math.h>

void oracle_ccd_fit(const double *f, long m, const double *fit, double *c)
{
    for (long i = 0; i < m; ++i) {
        const double *fi = f + 4 * i;
        double *ci = c + 4 * i;
        for (int j = 0; j < 4; ++j) {
            const double *F = fit + 4 * j;
            if (m >= 2) {
                double acc = fi[0] * F[0];
                acc = fma(fi[1], F[1], acc);
                acc = fma(fi[2], F[2], acc);
                ci[j] = fma(fi[3], F[3], acc);
            } else {
                double even = fi[0] * F[0] + fi[2] * F[2];
                double odd = fi[1] * F[1] + fi[3] * F[3];
                ci[j] = even + odd;
            }
        }
    }
}
