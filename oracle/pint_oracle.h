/* pint_oracle — CPU restatement of the reference's Nievergelt slice-map path.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library, and only as the checker or the CPU baseline.
 * The B200 product (paper_1304_6514_b200/) never links or calls it.
 *
 * Parity pinning: every reference-backed function here is checked bit-for-bit against golden
 * vectors produced by the UNMODIFIED reference (oracle/_ref/ref_tool golden, fixtures under
 * tests/golden/, generator tests/golden/make_golden.py). Functions marked EXTENSION have no
 * reference counterpart (RK4, logistic, Lotka-Volterra, bilinear/bracket interpolation,
 * closed-form weights, tree composition, FP32): their semantics are defined here and in
 * DESIGN.md §3 and pinned by analytic known-answer tests ("parity unpinned" vs the reference).
 *
 * Conventions: compiled with -ffp-contract=off, so every a*b+c rounds twice exactly as the
 * reference's x86-64 objects do; explicit fma() appears only in EXTENSION kernels where the
 * op order is part of the definition. Matrices are row-major like pint::Matrix (linalg.hpp:11-31).
 */
#ifndef PINT_ORACLE_H
#define PINT_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- time slices (ode_core.cpp:18-45) ---- */
int64_t or_steps_for(double width, double dt);
/* returns 0, or -1 for BadGrid */
int or_decompose(double t0, double T, int64_t N, double dt, double* t_begin, double* t_end,
                 int64_t* steps, double* h);

/* ---- scalar Riccati backward Euler (ode_core.cpp:47-53) ---- */
/* returns 0 and *z, or 1 (NoRealRoot) with *z = the negative discriminant */
int or_riccati_step(double y, double dt, double* z);
/* integrate_scalar (nievergelt.cpp:29-35) over one slice: steps x dt_eff. Returns 0 or 1 as above */
int or_riccati_integrate(double y, int64_t steps, double h, double* out);
/* the N*M task ensemble of run_nievergelt (nievergelt.cpp:170-182), idx = j*M + m.
 * Returns -1 when all tasks succeed, else the lowest failing idx (parallel_map semantics,
 * exec_harness.hpp:88-99) with *fail_value = that task's discriminant. */
int64_t or_riccati_ensemble(int64_t N, int64_t M, const int64_t* steps, const double* h,
                            const double* nodes, double* endpoints, double* fail_value);

/* ---- interpolation (interp.cpp:21-80) ---- */
int or_cheb_nodes1(int64_t M, double a, double b, double* x);
int or_cheb_nodes2(int64_t M, double a, double b, double* x);
/* product-form weights; returns 0 or -1 (DuplicateNodes) */
int or_bary_weights(const double* x, int64_t M, double* w);
/* EXTENSION: closed-form second-kind weights (-1)^j * delta_j, delta = 1/2 at the ends.
 * Scale-free, so they stay finite at M = 1024 where the product form overflows. */
void or_bary_weights_closed2(int64_t M, double* w);
double or_interp_eval(const double* x, const double* w, const double* v, int64_t M, double xi);
/* compose_sweep over scalar slice maps (nievergelt.cpp:68-88). values is N x M (slice-major).
 * Writes the boundary value after each slice into lambdas (may be NULL). */
double or_scalar_sweep(const double* x, const double* w, const double* values, int64_t N, int64_t M,
                       double a, double b, double y0, double* lambdas, int64_t* extrapolations);

/* ---- linear algebra (linalg.cpp:17-93) ---- */
void or_matvec(const double* A, int64_t rows, int64_t cols, const double* x, double* y);
void or_matmul(const double* A, const double* B, int64_t n, int64_t k, int64_t m, double* C);
/* returns 0 or -1 (SingularSystem) */
int or_thomas(const double* sub, const double* diag, const double* sup, int64_t n, double* d);

/* ---- heat problem (pde_problems.cpp:14-100) ---- */
double or_heat_coefficient(double t);
double or_heat_forcing(double x, double t);
/* interior points for dx (throws BadGrid -> returns -1) */
int64_t or_heat_dim(double dx);
void or_heat_initial(double dx, int64_t n, double* u);
void or_heat_exact(double dx, int64_t n, double t, double* u);
/* the make_heat_problem integrate closure: one slice [t_begin, t_end] at nominal dt */
int or_heat_integrate(double dx, int64_t n, double t_begin, double t_end, double dt_nominal,
                      int with_forcing, double* y);
/* build_affine_propagator (nievergelt.cpp:53-66): G row-major n x n, c n */
int or_heat_build(double dx, int64_t n, double t_begin, double t_end, double dt_nominal, double* G,
                  double* c);
/* compose_sweep over affine maps (nievergelt.cpp:90-110): G is N x n x n row-major */
void or_affine_chain(const double* G, const double* c, int64_t N, int64_t n, const double* y0,
                     double* y);
/* EXTENSION: log-depth pairwise tree. Level l pairs (2p, 2p+1) -> (G_{2p+1} G_{2p},
 * G_{2p+1} c_{2p} + c_{2p+1}) with reference matmul/matvec, an odd tail is carried.
 * Overwrites G/c scratch; writes the composed map to G_out/c_out and y = G y0 + c. */
void or_affine_tree(double* G, double* c, int64_t N, int64_t n, const double* y0, double* G_out,
                    double* c_out, double* y);

/* ---- EXTENSION: RK4 ensembles (no reference stepper) ---- */
void or_logistic_rk4_ensemble(int64_t N, int64_t M, const int64_t* steps, const double* h,
                              const double* nodes, double r, double K, double* endpoints);
void or_logistic_rk4_ensemble_f32(int64_t N, int64_t M, const int64_t* steps, const double* h,
                                  const float* nodes, float r, float K, float* endpoints);
/* Lotka-Volterra u' = alpha u - beta u v, v' = delta u v - gamma v; tensor grid Mu x Mv per slice.
 * endpoints layout (N, 2, Mu, Mv): component-major per slice. */
void or_lv_rk4_ensemble(int64_t N, int64_t Mu, int64_t Mv, const int64_t* steps, const double* h,
                        const double* un, const double* vn, const double* params /*a,b,d,g*/,
                        double* endpoints);
/* trajectories [lo, hi) of the flattened (slice, iu, iv) index only: for spot checks */
void or_lv_rk4_subset(int64_t lo, int64_t hi, int64_t Mu, int64_t Mv, const int64_t* steps,
                      const double* h, const double* un, const double* vn, const double* params,
                      double* out_uv /* (hi-lo) x 2 */);

/* ---- EXTENSION: bracket search + bilinear tensor interpolation ---- */
/* upper_bound(x, xi) - 1 clamped to [0, M-2] */
int64_t or_bracket(const double* x, int64_t M, double xi);
double or_lerp(double a, double b, double t);
/* chain of bilinear slice maps over tables (N, 2, Mu, Mv); writes per-slice (u, v) and the
 * bracket indices (iu, iv) the chain used; returns the extrapolation count */
int64_t or_bilinear_sweep(const double* un, int64_t Mu, const double* vn, int64_t Mv,
                          const double* tables, int64_t N, double u0, double v0, double* lambdas,
                          int64_t* brackets);

/* uniform grid a + ((b - a) * i) / (M - 1), the node rule for the 2-D tensor grid */
void or_uniform_nodes(int64_t M, double a, double b, double* x);

#ifdef __cplusplus
}
#endif
#endif
