/* TEST INFRASTRUCTURE ONLY — the CPU oracle. Never linked into the product.
 *
 * Plain-C restatement of the reference's collide-and-stream algorithm
 * (arXiv 2506.09242 restated as "dolb", /root/reference/proj), written to
 * reproduce its floating-point evaluation order so results are comparable
 * bit-for-bit when both sides are compiled without FMA contraction.
 *
 *   D3Q19 tables ......... proj/include/dolb/descriptor.hpp:13-46
 *   compute_rho_u ........ descriptor.hpp:64-76
 *   equilibrium2 / 4 ..... descriptor.hpp:79-121
 *   pi_neq ............... descriptor.hpp:126-143
 *   bgk / trt / rr ....... proj/include/dolb/collision.hpp:46-164
 *   smagorinsky_omega .... collision.hpp:169-183
 *   derive_omega_minus ... collision.hpp:19-22
 *   bounce-back / Ladd ... proj/include/dolb/boundaries.hpp:10-31
 *   regularized BCs ...... boundaries.hpp:45-133
 *   ChainRecipe::apply ... proj/include/dolb/chain.hpp:104-144
 *   lattice step ......... proj/src/reference_lattice.cpp:224-264 (pull, periodic
 *                          wrap, zero outside non-periodic faces)
 *   TGV state ............ proj/src/cases.cpp:145-156
 *   equilibrium fill ..... proj/src/multiblock.cpp:252-287 (equilibrium2 in T)
 *
 * D3Q27 has no reference ("parity unpinned"). It follows the
 * same formulas generalised to the 27-velocity set ordered as SURVEY.md A.8
 * (indices 0-18 = the frozen D3Q19 table, then 8 corners as opposite pairs),
 * with the reference's exact Hermite truncation (six aab third-order terms).
 */
#ifndef LBM_ORACLE_H
#define LBM_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* POD image of dolb::ChainRecipe<T> (chain.hpp:86-102); parameters kept in
 * double and cast to T at use exactly as compile_chain<T> does (chain.hpp:150-156). */
typedef struct orc_recipe {
    int32_t kind;            /* 0 NoDynamics, 1 BounceBack, 2 MovingBounceBack, 3 Collide */
    int32_t base;            /* 0 BGK, 1 TRT, 2 RR */
    int32_t has_regularized;
    int32_t reg_is_pressure;
    int32_t reg_axis;
    int32_t reg_orient;
    int32_t has_les;
    int32_t pad;
    double omega, lambda, smagorinsky_c, omega_bulk_ho;
    double wall_velocity[3];
    double target_rho;
} orc_recipe;

int orc_descriptor(int q, int32_t* c, double* w, int32_t* opp);
double orc_derive_omega_minus(double omega, double lambda);

void orc_equilibrium_d(int q, int order, double rho, const double* u, double* out);
void orc_equilibrium_f(int q, int order, float rho, const float* u, float* out);

/* Apply one recipe to n cells stored cell-major (f[c*q + i]). */
int orc_apply_d(int q, const orc_recipe* r, double* f, int64_t n);
int orc_apply_f(int q, const orc_recipe* r, float* f, int64_t n);

/* n cells, direction-major output f[i*n + c]: equilibrium2<T>(T(rho), T(u)). */
void orc_fill_equilibrium_d(int q, int64_t n, const double* rho, const double* ux,
                            const double* uy, const double* uz, double* f);
void orc_fill_equilibrium_f(int q, int64_t n, const double* rho, const double* ux,
                            const double* uy, const double* uz, float* f);

/* nsteps of pull-collide on a dims[0]*dims[1]*dims[2] lattice in canonical
 * order (direction-major, x fastest). slot[cell] indexes recipes. scratch has
 * the size of f. nthreads splits z; results do not depend on it. */
int orc_step_d(int q, const int64_t* dims, const int32_t* periodic, const orc_recipe* recipes,
               int nrecipes, const int32_t* slot, double* f, double* scratch, int64_t nsteps,
               int nthreads);
int orc_step_f(int q, const int64_t* dims, const int32_t* periodic, const orc_recipe* recipes,
               int nrecipes, const int32_t* slot, float* f, float* scratch, int64_t nsteps,
               int nthreads);

/* TGV initial state (cases.cpp:145-156) for planes z in [z0, z0+nz) of an L^3 box. */
void orc_tgv_state(int64_t L, double u_inf, int64_t z0, int64_t nz, double* rho, double* ux,
                   double* uy, double* uz);

#ifdef __cplusplus
}
#endif

#endif
