/* Oracle (TEST INFRASTRUCTURE): strict-sequential simulated working precision.
 *
 * Restates the "full-arithmetic" mode of the reference's Arithmetic class
 * (/root/reference/pkg/src/hodlrmp/arithmetic.py:14-67):
 *   - every scalar product and every partial sum is computed in binary64 and
 *     immediately rounded to the working format (arithmetic.py:37-46),
 *   - matrix products contract strictly left to right: acc = rnd(A[:,0]*B[0,:]),
 *     acc = rnd(acc + rnd(A[:,j]*B[j,:])) for j = 1.. (arithmetic.py:59-67),
 * with the rounding of fpsim._round_array (fpsim.py:160-177): RNE onto a grid of
 * t significand bits, subnormal floor at 2^(e_min-t+1), > x_max -> +-inf.
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -shared -fPIC (see oracle/Makefile);
 * no FMA contraction, so results are bit-identical to the Python simulation.
 * Only tests/ and bench.py's CPU baseline load this library.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

typedef struct {
    int t, e_min, e_max, subnormals;
    double x_max, x_min;
    int identity; /* fp64: rounding is the identity */
    int is_fp32;  /* IEEE binary32: a (float) cast is the same RNE rounding */
} fmt_t;

static void fmt_init(fmt_t* f, int t, int e_min, int e_max, int subnormals) {
    f->t = t; f->e_min = e_min; f->e_max = e_max; f->subnormals = subnormals;
    f->x_max = ldexp(2.0 - ldexp(1.0, 1 - t), e_max);
    f->x_min = ldexp(1.0, e_min);
    f->identity = (t >= 53 && e_min <= -1022 && e_max >= 1023 && subnormals);
    f->is_fp32 = (t == 24 && e_min == -126 && e_max == 127 && subnormals);
}

static inline double rnd(const fmt_t* f, double x) {
    if (f->identity) return x;
    if (f->is_fp32) return (double)(float)x;
    if (x == 0.0 || isnan(x) || isinf(x)) return x;
    double m = fabs(x);
    int e;
    frexp(m, &e);
    int q = e - f->t;
    if (q < f->e_min - f->t + 1) q = f->e_min - f->t + 1;
    double r = ldexp(nearbyint(ldexp(m, -q)), q);
    if (r > f->x_max) r = INFINITY;
    if (!f->subnormals && r < f->x_min) r = 0.0;
    return copysign(r, x);
}

/* Elementwise rounding (exported for the oracle self-test against round_matrix). */
void oracle_round(int t, int e_min, int e_max, int subnormals,
                  const double* x, double* y, int64_t count) {
    fmt_t f; fmt_init(&f, t, e_min, e_max, subnormals);
    for (int64_t i = 0; i < count; ++i) y[i] = rnd(&f, x[i]);
}

/* out[m x s] = A[m x q] @ B[q x s], row-major with leading dims, per-op rounding. */
void oracle_seq_matmul(int t, int e_min, int e_max, int subnormals,
                       int64_t m, int64_t q, int64_t s,
                       const double* A, int64_t lda, const double* B, int64_t ldb,
                       double* out, int64_t ldo) {
    fmt_t f; fmt_init(&f, t, e_min, e_max, subnormals);
    for (int64_t i = 0; i < m; ++i) {
        double* o = out + i * ldo;
        if (q == 0) { for (int64_t j = 0; j < s; ++j) o[j] = 0.0; continue; }
        const double* a = A + i * lda;
        for (int64_t j = 0; j < s; ++j) o[j] = rnd(&f, a[0] * B[j]);
        for (int64_t k = 1; k < q; ++k) {
            const double ak = a[k];
            const double* bk = B + k * ldb;
            for (int64_t j = 0; j < s; ++j) {
                double p = rnd(&f, ak * bk[j]);
                o[j] = rnd(&f, o[j] + p);
            }
        }
    }
}

/* b[i] = rnd(b[i] + y[i]) (arithmetic.py:39-40). */
void oracle_seq_add(int t, int e_min, int e_max, int subnormals,
                    double* b, const double* y, int64_t count) {
    fmt_t f; fmt_init(&f, t, e_min, e_max, subnormals);
    for (int64_t i = 0; i < count; ++i) b[i] = rnd(&f, b[i] + y[i]);
}
