/*
 * pswim_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference algorithms on the MRS / rod / Parareal hot path of
 * arxiv/paper_2604_12083 (`pintswim`, /root/reference/proj).  Every function cites the
 * reference file:line it restates and evaluates in the SAME operation order, so that when
 * compiled without FP contraction (-ffp-contract=off, x86-64 SSE2) its results are
 * bitwise equal to the reference library built by oracle/Makefile into oracle/_ref/.
 * tests/test_oracle_pin.py checks that equality and the committed golden vectors in
 * tests/golden/ (generated from oracle/_ref by tests/golden/make_golden.py).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load this library — and only as the checker or the timed CPU baseline, never as the
 * product path.
 */
#ifndef PSWIM_ORACLE_H
#define PSWIM_ORACLE_H

#include <stdint.h>

#include "../include/pswim_c.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Error codes follow pswim_c.h (PSWIM_EINVAL, PSWIM_ESTIFF, ...). */

/* mt19937_64 (std::mt19937_64) + the reference's uniform helpers
 * (scenario.cpp:33, tests/oracles.hpp:41-54). */
typedef struct or_rng {
    uint64_t mt[312];
    int idx;
} or_rng;
void or_rng_seed(or_rng* g, uint64_t seed);
uint64_t or_rng_next(or_rng* g);
double or_uniform(or_rng* g, double lo, double hi);            /* oracles.hpp:41-43 */
void or_random_unit(or_rng* g, double* out3);                  /* oracles.hpp:45-50 */
void or_random_vec(or_rng* g, double scale, double* out3);     /* oracles.hpp:52-54 */

/* ---- stokes (src/stokes.cpp) ---- */
void or_h_functions(double r, double eps, double* h5);                         /* :59-74  */
int or_evaluate_velocities(const double* tgt, int64_t nt, const double* src, const double* f,
                           const double* n, int64_t ns, double eps, double mu, int wall_mode,
                           double* u, double* w);                              /* :76-113 */
int or_evaluate_velocities_rows(const double* tgt, int64_t t_begin, int64_t t_end,
                                const double* src, const double* f, const double* n, int64_t ns,
                                double eps, double mu, double* u, double* w, int threads);
int or_grand_mobility(const double* nodes, int64_t n, double eps, double mu, double* mat); /* :115-154 */

/* ---- rotation (src/rotation.cpp) ---- */
int or_from_axis_angle(const double* axis3, double angle, double* r9);         /* :19-34  */
void or_to_axis_angle(const double* r9, double* axis3, double* angle);         /* :74-89  */
void or_sqrt_rotation(const double* r9, double* s9);                           /* :91-107 */
double or_rotation_residual(const double* r9);                                 /* :10-15  */

/* ---- rod (src/rod.cpp) ---- */
/* Single rod of m nodes in packed layout (12 doubles per node). */
int or_internal_loads(const double* rod12, int64_t m, double length, const double* mat6,
                      const double* wave3, double t, double* force, double* moment); /* :36-82 */
int or_nodal_loads(const double* rod12, int64_t m, double length, const double* force,
                   const double* moment, double* f, double* n);               /* :84-109 */
void or_lj_repulsion(const double* state12, int64_t rods, int64_t m, double well_depth,
                     double sigma, int64_t self_exclusion, double* forces);   /* :124-174 */
int64_t or_reorthonormalize(double* rod12, int64_t m, double tol);             /* :176-195 */
void or_preferred_strain(double s, double t, const double* wave3, double* out3); /* :29-32 */

/* ---- scenario (src/scenario.cpp) ---- */
int or_resolve(const pswim_scenario* sc, pswim_resolved* out);                 /* :10-29  */
int or_build_initial_state(const pswim_scenario* sc, double* state12);        /* :71-120 */

/* ---- propagators (src/propagators.cpp) ---- */
int or_rhs(const pswim_scenario* sc, const double* state12, double t, const double* extra_f,
           const double* extra_n, double* u, double* w, int threads);          /* :38-91  */
int or_advance_state(const pswim_scenario* sc, const double* state12, const double* u,
                     const double* w, double dt, double* out12);               /* :93-124 */
int or_step(const pswim_scenario* sc, int scheme, const double* state12, double t, double dt,
            double* out12, int threads);                                       /* :126-133 */
int or_propagate(const pswim_scenario* sc, const double* in12, double t0, double t1, int scheme,
                 int64_t steps_per_interval, double dt, double* out12, int threads); /* :135-162 */

/* ---- io / parareal ---- */
double or_position_metric(const double* x, const double* y, int64_t len);     /* io.cpp:49-68 */
double or_pointwise_metric(const double* x, const double* y, int64_t len, int64_t dim); /* parareal.cpp:15-34 */

/* Brute-force Parareal recurrence (tests/test_parareal.cpp:41-65 == parareal.cpp:58-89)
 * with Euler(coarse_steps) / RK2(fine_steps) rod propagators; states (n+1) x len. */
int or_parareal_rod(const pswim_scenario* sc, double t0, double horizon, int intervals,
                    int iterations, int64_t fine_steps, int64_t coarse_steps, const double* x0,
                    double* states, double* eta_tilde, int threads);

/* ---- reference test oracles (tests/oracles.cpp) ---- */
void or_dense_mobility_apply(const double* nodes, int64_t n, const double* f, const double* tq,
                             double eps, double mu, double* u, double* w);    /* :87-140 */
double or_elastic_energy(const double* rod12, int64_t m, double length, const double* mat6,
                         const double* wave3, double t);                        /* :142-167 */
void or_perturbed_rod(int64_t m, double length, or_rng* g, double position_jitter,
                      double angle_jitter, double* rod12);                      /* :204-222 */

#ifdef __cplusplus
}
#endif
#endif
