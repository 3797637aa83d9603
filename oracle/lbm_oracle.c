/* TEST INFRASTRUCTURE ONLY — CPU oracle (see lbm_oracle.h for the map to the
 * reference). Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg load this library, and only as the checker. */
#include "lbm_oracle.h"

#include <math.h>
#include <pthread.h>
#include <string.h>

#define ORC_QMAX 27

typedef struct lattice_t {
    int q;
    int c[ORC_QMAX][3];
    double w[ORC_QMAX];
    int opp[ORC_QMAX];
} lattice_t;

/* descriptor.hpp:21-45 (frozen order; opposites adjacent). */
static const lattice_t D3Q19 = {
    19,
    {{0, 0, 0},
     {-1, 0, 0}, {1, 0, 0}, {0, -1, 0}, {0, 1, 0}, {0, 0, -1}, {0, 0, 1},
     {-1, -1, 0}, {1, 1, 0}, {-1, 1, 0}, {1, -1, 0},
     {-1, 0, -1}, {1, 0, 1}, {-1, 0, 1}, {1, 0, -1},
     {0, -1, -1}, {0, 1, 1}, {0, -1, 1}, {0, 1, -1}},
    {1.0 / 3.0,
     1.0 / 18.0, 1.0 / 18.0, 1.0 / 18.0, 1.0 / 18.0, 1.0 / 18.0, 1.0 / 18.0,
     1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0,
     1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0},
    {0, 2, 1, 4, 3, 6, 5, 8, 7, 10, 9, 12, 11, 14, 13, 16, 15, 18, 17},
};

/* D3Q27: indices 0-18 as D3Q19, corners appended as opposite
 * pairs. w = 8/27, 2/27, 1/54, 1/216 (no reference exists for this set). */
static const lattice_t D3Q27 = {
    27,
    {{0, 0, 0},
     {-1, 0, 0}, {1, 0, 0}, {0, -1, 0}, {0, 1, 0}, {0, 0, -1}, {0, 0, 1},
     {-1, -1, 0}, {1, 1, 0}, {-1, 1, 0}, {1, -1, 0},
     {-1, 0, -1}, {1, 0, 1}, {-1, 0, 1}, {1, 0, -1},
     {0, -1, -1}, {0, 1, 1}, {0, -1, 1}, {0, 1, -1},
     {-1, -1, -1}, {1, 1, 1}, {-1, -1, 1}, {1, 1, -1},
     {-1, 1, -1}, {1, -1, 1}, {1, -1, -1}, {-1, 1, 1}},
    {8.0 / 27.0,
     2.0 / 27.0, 2.0 / 27.0, 2.0 / 27.0, 2.0 / 27.0, 2.0 / 27.0, 2.0 / 27.0,
     1.0 / 54.0, 1.0 / 54.0, 1.0 / 54.0, 1.0 / 54.0, 1.0 / 54.0, 1.0 / 54.0,
     1.0 / 54.0, 1.0 / 54.0, 1.0 / 54.0, 1.0 / 54.0, 1.0 / 54.0, 1.0 / 54.0,
     1.0 / 216.0, 1.0 / 216.0, 1.0 / 216.0, 1.0 / 216.0,
     1.0 / 216.0, 1.0 / 216.0, 1.0 / 216.0, 1.0 / 216.0},
    {0, 2, 1, 4, 3, 6, 5, 8, 7, 10, 9, 12, 11, 14, 13, 16, 15, 18, 17,
     20, 19, 22, 21, 24, 23, 26, 25},
};

static const lattice_t* lattice_for(int q) {
    return q == 19 ? &D3Q19 : q == 27 ? &D3Q27 : NULL;
}

int orc_descriptor(int q, int32_t* c, double* w, int32_t* opp) {
    const lattice_t* L = lattice_for(q);
    if (!L) return 1;
    for (int i = 0; i < q; ++i) {
        for (int a = 0; a < 3; ++a) c[i * 3 + a] = L->c[i][a];
        w[i] = L->w[i];
        opp[i] = L->opp[i];
    }
    return 0;
}

/* collision.hpp:19-22 */
double orc_derive_omega_minus(double omega, double lambda) {
    const double half_minus = lambda / (1.0 / omega - 0.5);
    return 1.0 / (half_minus + 0.5);
}

/* cases.cpp:145-156 (cs2 = 1/3 from descriptor.hpp:15). */
void orc_tgv_state(int64_t L, double u_inf, int64_t z0, int64_t nz, double* rho, double* ux,
                   double* uy, double* uz) {
    const double pi = 3.14159265358979323846;
    const double scale = 2.0 * pi / (double)L;
    int64_t c = 0;
    for (int64_t k = z0; k < z0 + nz; ++k) {
        for (int64_t j = 0; j < L; ++j) {
            for (int64_t i = 0; i < L; ++i, ++c) {
                const double x = scale * ((double)i + 0.5);
                const double y = scale * ((double)j + 0.5);
                const double z = scale * ((double)k + 0.5);
                const double dp = u_inf * u_inf / 16.0 * (cos(2.0 * z) + 2.0) *
                                  (cos(2.0 * x) + cos(2.0 * y));
                rho[c] = 1.0 + dp / (1.0 / 3.0);
                ux[c] = u_inf * sin(x) * cos(y) * cos(z);
                uy[c] = -u_inf * cos(x) * sin(y) * cos(z);
                uz[c] = 0.0;
            }
        }
    }
}

#define T double
#define S(name) name##_d
#define SQRT sqrt
#include "lbm_oracle_body.inc"
#undef T
#undef S
#undef SQRT

#define T float
#define S(name) name##_f
#define SQRT sqrtf
#include "lbm_oracle_body.inc"
#undef T
#undef S
#undef SQRT
