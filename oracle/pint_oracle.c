/* pint_oracle.c — CPU restatement of the reference slice-map path. TEST INFRASTRUCTURE ONLY
 * (see pint_oracle.h for who may load it and how it is pinned against the reference). */
#include "pint_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static const double kPi = 3.14159265358979323846;

static double dmax(double a, double b) { return a > b ? a : b; }

/* ode_core.cpp:18-24: ceil after snapping by 1e-9 relative; at least one step */
int64_t or_steps_for(double width, double dt) {
    const double ratio = width / dt;
    const double snapped = ratio - 1e-9 * dmax(1.0, ratio);
    const long long n = (long long)ceil(snapped);
    return n < 1 ? 1 : (int64_t)n;
}

/* ode_core.cpp:26-45 */
int or_decompose(double t0, double T, int64_t N, double dt, double* t_begin, double* t_end,
                 int64_t* steps, double* h) {
    if (N <= 0 || !(T > t0) || !(dt > 0.0)) return -1;
    const double width = (T - t0) / (double)N;
    for (int64_t j = 0; j < N; ++j) {
        const double tb = t0 + (double)j * width;
        const double te = (j + 1 == N) ? T : t0 + (double)(j + 1) * width;
        const int64_t s = or_steps_for(te - tb, dt);
        t_begin[j] = tb;
        t_end[j] = te;
        steps[j] = s;
        h[j] = (te - tb) / (double)s;
    }
    return 0;
}

/* ode_core.cpp:47-53: disc = 1 - (4 dt) y; z = 2y / (1 + sqrt(disc)) */
int or_riccati_step(double y, double dt, double* z) {
    const double disc = 1.0 - 4.0 * dt * y;
    if (disc < 0.0) {
        *z = disc;
        return 1;
    }
    *z = 2.0 * y / (1.0 + sqrt(disc));
    return 0;
}

/* integrate_slice (ode_core.hpp:74-86) driving the Riccati step, as integrate_scalar does */
int or_riccati_integrate(double y, int64_t steps, double h, double* out) {
    for (int64_t i = 1; i <= steps; ++i) {
        double z;
        if (or_riccati_step(y, h, &z)) {
            *out = z;
            return 1;
        }
        y = z;
    }
    *out = y;
    return 0;
}

/* nievergelt.cpp:170-182 with parallel_map's lowest-failing-index rule (exec_harness.hpp:88-99) */
int64_t or_riccati_ensemble(int64_t N, int64_t M, const int64_t* steps, const double* h,
                            const double* nodes, double* endpoints, double* fail_value) {
    int64_t fail = -1;
    for (int64_t idx = 0; idx < N * M; ++idx) {
        const int64_t j = idx / M, m = idx % M;
        double out;
        if (or_riccati_integrate(nodes[m], steps[j], h[j], &out)) {
            if (fail < 0) {
                fail = idx;
                if (fail_value) *fail_value = out;
            }
            endpoints[idx] = NAN;
            continue;
        }
        endpoints[idx] = out;
    }
    return fail;
}

/* interp.cpp:14-18 map to [a, b] then sort ascending (insertion sort: M is small and the
 * cosines arrive descending, so this is the same permutation std::sort produces) */
static void map_sorted(double* x, int64_t M, double a, double b) {
    for (int64_t i = 0; i < M; ++i) x[i] = a + (b - a) * (x[i] + 1.0) / 2.0;
    for (int64_t i = 1; i < M; ++i) {
        const double v = x[i];
        int64_t k = i - 1;
        while (k >= 0 && x[k] > v) {
            x[k + 1] = x[k];
            --k;
        }
        x[k + 1] = v;
    }
}

/* interp.cpp:21-28 */
int or_cheb_nodes1(int64_t M, double a, double b, double* x) {
    if (M <= 0) return -1;
    if (M == 1) {
        x[0] = 0.5 * (a + b);
        return 0;
    }
    for (int64_t k = 0; k < M; ++k) x[k] = cos((2.0 * (double)k + 1.0) * kPi / (2.0 * (double)M));
    map_sorted(x, M, a, b);
    return 0;
}

/* interp.cpp:30-37 */
int or_cheb_nodes2(int64_t M, double a, double b, double* x) {
    if (M <= 0) return -1;
    if (M == 1) {
        x[0] = 0.5 * (a + b);
        return 0;
    }
    for (int64_t k = 0; k < M; ++k) x[k] = cos((double)k * kPi / (double)(M - 1));
    map_sorted(x, M, a, b);
    return 0;
}

/* interp.cpp:43-55: w_j = 1 / prod_{k != j}(x_j - x_k) as sequential divides, k ascending */
int or_bary_weights(const double* x, int64_t M, double* w) {
    for (int64_t j = 0; j < M; ++j) {
        double acc = 1.0;
        for (int64_t k = 0; k < M; ++k) {
            if (k == j) continue;
            const double diff = x[j] - x[k];
            if (diff == 0.0) return -1;
            acc /= diff;
        }
        w[j] = acc;
    }
    return 0;
}

/* EXTENSION: closed-form weights for the second-kind grid (Berrut & Trefethen 2004). */
void or_bary_weights_closed2(int64_t M, double* w) {
    for (int64_t j = 0; j < M; ++j) {
        const double sgn = (j % 2 == 0) ? 1.0 : -1.0;
        w[j] = (j == 0 || j == M - 1) ? 0.5 * sgn : sgn;
    }
}

/* interp.cpp:68-80: node snap (first match), then sequential barycentric sums */
double or_interp_eval(const double* x, const double* w, const double* v, int64_t M, double xi) {
    for (int64_t j = 0; j < M; ++j)
        if (fabs(xi - x[j]) <= 1e-14 * dmax(1.0, fabs(x[j]))) return v[j];
    double num = 0.0, den = 0.0;
    for (int64_t j = 0; j < M; ++j) {
        const double r = w[j] / (xi - x[j]);
        num += r * v[j];
        den += r;
    }
    return num / den;
}

/* nievergelt.cpp:68-88 (latency/message accounting lives in the callers) */
double or_scalar_sweep(const double* x, const double* w, const double* values, int64_t N, int64_t M,
                       double a, double b, double y0, double* lambdas, int64_t* extrapolations) {
    double y = y0;
    int64_t ext = 0;
    for (int64_t j = 0; j < N; ++j) {
        if (y < a || y > b) ++ext;
        y = or_interp_eval(x, w, values + j * M, M, y);
        if (lambdas) lambdas[j] = y;
    }
    if (extrapolations) *extrapolations = ext;
    return y;
}

/* linalg.cpp:17-26 */
void or_matvec(const double* A, int64_t rows, int64_t cols, const double* x, double* y) {
    for (int64_t i = 0; i < rows; ++i) {
        double s = 0.0;
        for (int64_t j = 0; j < cols; ++j) s += A[i * cols + j] * x[j];
        y[i] = s;
    }
}

/* linalg.cpp:28-38: i-k-j with zero skip. A is n x k, B is k x m. */
void or_matmul(const double* A, const double* B, int64_t n, int64_t k, int64_t m, double* C) {
    memset(C, 0, sizeof(double) * (size_t)(n * m));
    for (int64_t i = 0; i < n; ++i)
        for (int64_t q = 0; q < k; ++q) {
            const double a = A[i * k + q];
            if (a == 0.0) continue;
            for (int64_t j = 0; j < m; ++j) C[i * m + j] += a * B[q * m + j];
        }
}

/* linalg.cpp:77-93 (n = 1 handled without touching the empty sup array) */
int or_thomas(const double* sub, const double* diag, const double* sup, int64_t n, double* d) {
    double* c = (double*)malloc(sizeof(double) * (size_t)(n > 1 ? n - 1 : 1));
    double pivot = diag[0];
    if (pivot == 0.0) {
        free(c);
        return -1;
    }
    if (n > 1) c[0] = sup[0] / pivot;
    d[0] /= pivot;
    for (int64_t i = 1; i < n; ++i) {
        pivot = diag[i] - sub[i - 1] * c[i - 1];
        if (pivot == 0.0) {
            free(c);
            return -1;
        }
        if (i < n - 1) c[i] = sup[i] / pivot;
        d[i] = (d[i] - sub[i - 1] * d[i - 1]) / pivot;
    }
    for (int64_t i = n - 1; i-- > 0;) d[i] -= c[i] * d[i + 1];
    free(c);
    return 0;
}

/* pde_problems.cpp:24 */
double or_heat_coefficient(double t) { return 1.0 + 0.25 * sin(t); }

/* pde_problems.cpp:26-29 */
double or_heat_forcing(double x, double t) {
    const double sx = sin(kPi * x);
    return -sin(t) * sx + or_heat_coefficient(t) * kPi * kPi * cos(t) * sx;
}

/* pde_problems.cpp:14-21 */
int64_t or_heat_dim(double dx) {
    const double inv = 1.0 / dx;
    const long long m = llround(inv);
    if (m < 2 || fabs(inv - (double)m) > 1e-9 * inv) return -1;
    return (int64_t)(m - 1);
}

/* pde_problems.cpp:61-74 */
void or_heat_initial(double dx, int64_t n, double* u) {
    for (int64_t i = 0; i < n; ++i) u[i] = sin(kPi * (double)(i + 1) * dx);
}
void or_heat_exact(double dx, int64_t n, double t, double* u) {
    for (int64_t i = 0; i < n; ++i) u[i] = cos(t) * sin(kPi * (double)(i + 1) * dx);
}

/* one backward-Euler heat step: forcing (pde_problems.cpp:90-94) then solve_implicit (:53-57) */
static int heat_step(double dx, int64_t n, double t_next, double h, int with_forcing, double* y,
                     double* sub, double* diag, double* sup) {
    if (with_forcing)
        for (int64_t i = 0; i < n; ++i) y[i] += h * or_heat_forcing((double)(i + 1) * dx, t_next);
    const double inv_dx2 = 1.0 / (dx * dx);
    const double r = h * or_heat_coefficient(t_next) * inv_dx2;
    for (int64_t i = 0; i < n; ++i) diag[i] = 1.0 + 2.0 * r;
    for (int64_t i = 0; i + 1 < n; ++i) {
        sub[i] = -r;
        sup[i] = -r;
    }
    return or_thomas(sub, diag, sup, n, y);
}

/* the integrate closure of make_heat_problem (pde_problems.cpp:86-98) via integrate_slice */
int or_heat_integrate(double dx, int64_t n, double t_begin, double t_end, double dt_nominal,
                      int with_forcing, double* y) {
    const int64_t steps = or_steps_for(t_end - t_begin, dt_nominal);
    const double h = (t_end - t_begin) / (double)steps;
    double* buf = (double*)malloc(sizeof(double) * (size_t)(3 * n));
    int rc = 0;
    for (int64_t i = 1; i <= steps && rc == 0; ++i) {
        const double t_next = t_begin + (double)i * h;
        rc = heat_step(dx, n, t_next, h, with_forcing, y, buf, buf + n, buf + 2 * n);
    }
    free(buf);
    return rc;
}

/* nievergelt.cpp:53-66 */
int or_heat_build(double dx, int64_t n, double t_begin, double t_end, double dt_nominal, double* G,
                  double* c) {
    memset(c, 0, sizeof(double) * (size_t)n);
    if (or_heat_integrate(dx, n, t_begin, t_end, dt_nominal, 1, c)) return -1;
    double* e = (double*)malloc(sizeof(double) * (size_t)n);
    for (int64_t j = 0; j < n; ++j) {
        memset(e, 0, sizeof(double) * (size_t)n);
        e[j] = 1.0;
        if (or_heat_integrate(dx, n, t_begin, t_end, dt_nominal, 0, e)) {
            free(e);
            return -1;
        }
        for (int64_t i = 0; i < n; ++i) G[i * n + j] = e[i];
    }
    free(e);
    return 0;
}

/* nievergelt.cpp:90-110 */
void or_affine_chain(const double* G, const double* c, int64_t N, int64_t n, const double* y0,
                     double* y) {
    double* cur = (double*)malloc(sizeof(double) * (size_t)n);
    double* nxt = (double*)malloc(sizeof(double) * (size_t)n);
    memcpy(cur, y0, sizeof(double) * (size_t)n);
    for (int64_t j = 0; j < N; ++j) {
        or_matvec(G + j * n * n, n, n, cur, nxt);
        for (int64_t i = 0; i < n; ++i) nxt[i] += c[j * n + i];
        double* t = cur;
        cur = nxt;
        nxt = t;
    }
    memcpy(y, cur, sizeof(double) * (size_t)n);
    free(cur);
    free(nxt);
}

/* EXTENSION: pairwise tree of affine products */
void or_affine_tree(double* G, double* c, int64_t N, int64_t n, const double* y0, double* G_out,
                    double* c_out, double* y) {
    const size_t nn = (size_t)(n * n);
    double* tmpG = (double*)malloc(sizeof(double) * nn);
    double* tmpc = (double*)malloc(sizeof(double) * (size_t)n);
    int64_t count = N;
    while (count > 1) {
        const int64_t pairs = count / 2;
        for (int64_t p = 0; p < pairs; ++p) {
            const double* G1 = G + (2 * p) * nn;      /* earlier slice */
            const double* G2 = G + (2 * p + 1) * nn;  /* later slice */
            const double* c1 = c + (2 * p) * n;
            const double* c2 = c + (2 * p + 1) * n;
            or_matmul(G2, G1, n, n, n, tmpG);
            or_matvec(G2, n, n, c1, tmpc);
            for (int64_t i = 0; i < n; ++i) tmpc[i] += c2[i];
            memcpy(G + p * nn, tmpG, sizeof(double) * nn);
            memcpy(c + p * n, tmpc, sizeof(double) * (size_t)n);
        }
        if (count % 2) {
            memmove(G + pairs * nn, G + (count - 1) * nn, sizeof(double) * nn);
            memmove(c + pairs * n, c + (count - 1) * n, sizeof(double) * (size_t)n);
        }
        count = pairs + (count % 2);
    }
    if (G_out) memcpy(G_out, G, sizeof(double) * nn);
    if (c_out) memcpy(c_out, c, sizeof(double) * (size_t)n);
    if (y) {
        or_matvec(G, n, n, y0, y);
        for (int64_t i = 0; i < n; ++i) y[i] += c[i];
    }
    free(tmpG);
    free(tmpc);
}

/* ---- EXTENSION: RK4 logistic, y' = r y (1 - y/K). Op order:
 *   f(y) = y * fma(-rK, y, r),  rK = r/K  (one FMA + one multiply)
 *   k1 = f(y); k2 = f(fma(h/2, k1, y)); k3 = f(fma(h/2, k2, y)); k4 = f(fma(h, k3, y))
 *   y += h/6 * ((k1 + k4) + 2 (k2 + k3))  as fma(h6, fma(2, k2 + k3, k1 + k4), y) */
static double logistic_f(double y, double r, double rK) { return y * fma(-rK, y, r); }

void or_logistic_rk4_ensemble(int64_t N, int64_t M, const int64_t* steps, const double* h,
                              const double* nodes, double r, double K, double* endpoints) {
    const double rK = r / K;
    for (int64_t j = 0; j < N; ++j) {
        const double hh = h[j], h2 = 0.5 * hh, h6 = hh / 6.0;
        for (int64_t m = 0; m < M; ++m) {
            double y = nodes[m];
            for (int64_t s = 0; s < steps[j]; ++s) {
                const double k1 = logistic_f(y, r, rK);
                const double k2 = logistic_f(fma(h2, k1, y), r, rK);
                const double k3 = logistic_f(fma(h2, k2, y), r, rK);
                const double k4 = logistic_f(fma(hh, k3, y), r, rK);
                y = fma(h6, fma(2.0, k2 + k3, k1 + k4), y);
            }
            endpoints[j * M + m] = y;
        }
    }
}

static float logistic_ff(float y, float r, float rK) { return y * fmaf(-rK, y, r); }

void or_logistic_rk4_ensemble_f32(int64_t N, int64_t M, const int64_t* steps, const double* h,
                                  const float* nodes, float r, float K, float* endpoints) {
    const float rK = r / K;
    for (int64_t j = 0; j < N; ++j) {
        const float hh = (float)h[j], h2 = 0.5f * hh, h6 = hh / 6.0f;
        for (int64_t m = 0; m < M; ++m) {
            float y = nodes[m];
            for (int64_t s = 0; s < steps[j]; ++s) {
                const float k1 = logistic_ff(y, r, rK);
                const float k2 = logistic_ff(fmaf(h2, k1, y), r, rK);
                const float k3 = logistic_ff(fmaf(h2, k2, y), r, rK);
                const float k4 = logistic_ff(fmaf(hh, k3, y), r, rK);
                y = fmaf(h6, fmaf(2.0f, k2 + k3, k1 + k4), y);
            }
            endpoints[j * M + m] = y;
        }
    }
}

/* ---- EXTENSION: Lotka-Volterra RK4 on the tensor grid. f_u = u * fma(-beta, v, alpha),
 * f_v = v * fma(delta, u, -gamma); stage/combination order as the logistic kernel. */
static void lv_traj(double u, double v, int64_t steps, double hh, const double* p, double* out) {
    const double al = p[0], be = p[1], de = p[2], ga = p[3];
    const double h2 = 0.5 * hh, h6 = hh / 6.0;
    for (int64_t s = 0; s < steps; ++s) {
        const double a1 = u * fma(-be, v, al), b1 = v * fma(de, u, -ga);
        const double u2 = fma(h2, a1, u), v2 = fma(h2, b1, v);
        const double a2 = u2 * fma(-be, v2, al), b2 = v2 * fma(de, u2, -ga);
        const double u3 = fma(h2, a2, u), v3 = fma(h2, b2, v);
        const double a3 = u3 * fma(-be, v3, al), b3 = v3 * fma(de, u3, -ga);
        const double u4 = fma(hh, a3, u), v4 = fma(hh, b3, v);
        const double a4 = u4 * fma(-be, v4, al), b4 = v4 * fma(de, u4, -ga);
        u = fma(h6, fma(2.0, a2 + a3, a1 + a4), u);
        v = fma(h6, fma(2.0, b2 + b3, b1 + b4), v);
    }
    out[0] = u;
    out[1] = v;
}

void or_lv_rk4_ensemble(int64_t N, int64_t Mu, int64_t Mv, const int64_t* steps, const double* h,
                        const double* un, const double* vn, const double* params,
                        double* endpoints) {
    const int64_t P = Mu * Mv;
    for (int64_t j = 0; j < N; ++j)
        for (int64_t iu = 0; iu < Mu; ++iu)
            for (int64_t iv = 0; iv < Mv; ++iv) {
                double o[2];
                lv_traj(un[iu], vn[iv], steps[j], h[j], params, o);
                endpoints[(j * 2 + 0) * P + iu * Mv + iv] = o[0];
                endpoints[(j * 2 + 1) * P + iu * Mv + iv] = o[1];
            }
}

void or_lv_rk4_subset(int64_t lo, int64_t hi, int64_t Mu, int64_t Mv, const int64_t* steps,
                      const double* h, const double* un, const double* vn, const double* params,
                      double* out_uv) {
    const int64_t P = Mu * Mv;
    for (int64_t idx = lo; idx < hi; ++idx) {
        const int64_t j = idx / P, q = idx % P;
        lv_traj(un[q / Mv], vn[q % Mv], steps[j], h[j], params, out_uv + 2 * (idx - lo));
    }
}

/* ---- EXTENSION: bracket search and bilinear interpolation ---- */
int64_t or_bracket(const double* x, int64_t M, double xi) {
    /* upper_bound: first index with x[i] > xi, binary search over [0, M) */
    int64_t lo = 0, len = M;
    while (len > 0) {
        const int64_t half = len / 2;
        if (!(x[lo + half] > xi)) {
            lo += half + 1;
            len -= half + 1;
        } else {
            len = half;
        }
    }
    int64_t b = lo - 1;
    if (b < 0) b = 0;
    if (b > M - 2) b = M - 2;
    return b;
}

double or_lerp(double a, double b, double t) { return fma(t, b - a, a); }

int64_t or_bilinear_sweep(const double* un, int64_t Mu, const double* vn, int64_t Mv,
                          const double* tables, int64_t N, double u0, double v0, double* lambdas,
                          int64_t* brackets) {
    const int64_t P = Mu * Mv;
    double u = u0, v = v0;
    int64_t ext = 0;
    for (int64_t j = 0; j < N; ++j) {
        if (u < un[0] || u > un[Mu - 1] || v < vn[0] || v > vn[Mv - 1]) ++ext;
        const int64_t iu = or_bracket(un, Mu, u), iv = or_bracket(vn, Mv, v);
        const double tu = (u - un[iu]) / (un[iu + 1] - un[iu]);
        const double tv = (v - vn[iv]) / (vn[iv + 1] - vn[iv]);
        double out[2];
        for (int comp = 0; comp < 2; ++comp) {
            const double* T = tables + (j * 2 + comp) * P;
            const double f00 = T[iu * Mv + iv], f10 = T[(iu + 1) * Mv + iv];
            const double f01 = T[iu * Mv + iv + 1], f11 = T[(iu + 1) * Mv + iv + 1];
            out[comp] = or_lerp(or_lerp(f00, f10, tu), or_lerp(f01, f11, tu), tv);
        }
        u = out[0];
        v = out[1];
        if (lambdas) {
            lambdas[2 * j] = u;
            lambdas[2 * j + 1] = v;
        }
        if (brackets) {
            brackets[2 * j] = iu;
            brackets[2 * j + 1] = iv;
        }
    }
    return ext;
}

void or_uniform_nodes(int64_t M, double a, double b, double* x) {
    for (int64_t i = 0; i < M; ++i) x[i] = a + ((b - a) * (double)i) / (double)(M - 1);
}
