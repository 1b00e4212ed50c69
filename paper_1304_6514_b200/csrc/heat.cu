// K3 — heat-equation slice maps: the n+1 basis/forced trajectories of every slice advanced
// together through backward-Euler steps (I - h a(t) L) x = y + h b(t).
//
// Replaces build_affine_propagator (nievergelt.cpp:53-66) -> make_heat_problem's integrate
// closure (pde_problems.cpp:86-98) -> solve_implicit (pde_problems.cpp:53-57) -> thomas_solve
// (linalg.cpp:77-93), run once per trajectory per step in the reference.
//
// B200 design:
//  * The tridiagonal factor (pivots p_i, multipliers c_i) depends only on (slice, step), never
//    on the right-hand side, so it is computed once per step by heat_factor_kernel (one thread
//    per step, all steps in parallel) instead of n+1 times. Same operations, same rounding, so
//    the solves stay bit-identical to the reference's per-trajectory Thomas solve.
//  * One thread per trajectory ("column"): column k < n of slice j starts at e_k, column n
//    starts at 0 with forcing (the c run). Columns are flattened across slices, so a warp is 32
//    consecutive columns; rows are walked sequentially (forward then back substitution).
//  * The column state lives in shared memory, lane-interleaved (row i of lane l at [i*32 + l]),
//    so every access is conflict-free; at the end row i of 32 consecutive columns is one
//    coalesced 256 B store into the row-major augmented map [G | c] (ldm = pint_affine_ldm(n)).
//    For n too large for shared memory the state lives directly in the output map (same
//    lane-contiguous rows, L1/L2 resident).
//
// Roofline: FP64 pipe (division-heavy). Algorithmic work per slice-step: factor 3n flops,
// per column 5n flops (forward: mul, sub, div; back: mul, sub) + 4n for the forcing column.
#include "pint_internal.cuh"

namespace {

using pint_dev::record_failure;

// factor[(q*n + i)] = {p_i, c_i}: the Thomas forward pivots of tridiag(-r, 1+2r, -r) at step q.
__global__ void heat_factor_kernel(long long n, long long Q, const double* __restrict__ r_tab,
                                   double2* __restrict__ factor, FailRec* fail) {
    const long long q = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= Q) return;
    const double r = r_tab[q];
    const double negr = -r;                              // sub = sup = -r (pde_problems.cpp:55)
    const double diag = __dadd_rn(1.0, __dmul_rn(2.0, r));  // 1.0 + 2.0 * r
    double2* F = factor + q * n;
    double p = diag;
    if (p == 0.0) record_failure(fail, q, PINT_E_SINGULAR, 0.0);
    double c = (n > 1) ? __ddiv_rn(negr, p) : 0.0;
    F[0] = make_double2(p, c);
    for (long long i = 1; i < n; ++i) {
        p = __dsub_rn(diag, __dmul_rn(negr, c));
        if (p == 0.0) record_failure(fail, q, PINT_E_SINGULAR, static_cast<double>(i));
        c = (i < n - 1) ? __ddiv_rn(negr, p) : 0.0;
        F[i] = make_double2(p, c);
    }
}

struct HeatTables {
    const double2* factor;
    const double* r;
    const double* fa;
    const double* fb;
    const double* sx;
};

enum class Mode { kBuild, kIntegrate };

struct ColumnPlan {
    // kBuild
    long long N;
    const int64_t* step_off;
    const double* slice_dt;
    double* maps;
    long long ldm;
    unsigned long long* per_slice_ns;
    // kIntegrate
    long long K;
    long long q0;
    long long steps;
    double h;
    int with_forcing;
    double* y;
};

// Advance one column (trajectory) through its steps; state rows at st[i * rs].
__device__ __forceinline__ void advance_column(const HeatTables& T, long long n, double* st,
                                               long long rs, long long q_begin, long long q_end,
                                               double h, bool forcing) {
    for (long long q = q_begin; q < q_end; ++q) {
        const double2* F = T.factor + q * n;
        const double negr = -T.r[q];
        double fa = 0.0, fb = 0.0;
        if (forcing) {
            fa = T.fa[q];
            fb = T.fb[q];
        }
        // forward elimination (linalg.cpp:80-90), forcing folded in (pde_problems.cpp:91-94)
        double dprev = 0.0;
        for (long long i = 0; i < n; ++i) {
            double x = st[i * rs];
            if (forcing) {
                const double s = T.sx[i];
                const double b = __dadd_rn(__dmul_rn(fa, s), __dmul_rn(fb, s));
                x = __dadd_rn(x, __dmul_rn(h, b));
            }
            const double num = (i == 0) ? x : __dsub_rn(x, __dmul_rn(negr, dprev));
            dprev = __ddiv_rn(num, F[i].x);
            st[i * rs] = dprev;
        }
        // back substitution (linalg.cpp:91)
        double dnext = dprev;
        for (long long i = n - 2; i >= 0; --i) {
            const double d = __dsub_rn(st[i * rs], __dmul_rn(F[i].y, dnext));
            st[i * rs] = d;
            dnext = d;
        }
    }
}

template <Mode kMode, bool kSmem>
__global__ void __launch_bounds__(32)
heat_columns_kernel(long long n, HeatTables T, ColumnPlan P) {
    extern __shared__ double state_s[];
    const unsigned long long t_start = pint_dev::globaltimer();
    const int lane = threadIdx.x;
    const long long g = static_cast<long long>(blockIdx.x) * 32 + lane;
    const long long total = (kMode == Mode::kBuild) ? P.N * (n + 1) : P.K;
    if (g >= total) return;  // whole trailing lanes only; no block-level sync below

    long long slice = 0, k = 0, q_begin, q_end;
    double h;
    bool forcing;
    double* gcol;     // where this column lives in global memory (row stride grs)
    long long grs;
    if (kMode == Mode::kBuild) {
        slice = g / (n + 1);
        k = g - slice * (n + 1);
        q_begin = P.step_off[slice];
        q_end = P.step_off[slice + 1];
        h = P.slice_dt[slice];
        forcing = (k == n);
        gcol = P.maps + slice * n * P.ldm + k;
        grs = P.ldm;
    } else {
        q_begin = P.q0;
        q_end = P.q0 + P.steps;
        h = P.h;
        forcing = P.with_forcing != 0;
        gcol = P.y + g * n;
        grs = 1;
    }
    double* st = kSmem ? state_s + lane : gcol;
    const long long rs = kSmem ? 32 : grs;

    for (long long i = 0; i < n; ++i) {
        double v;
        if (kMode == Mode::kBuild) v = (i == k) ? 1.0 : 0.0;  // e_k, or 0 for the c run
        else v = gcol[i];
        st[i * rs] = v;
    }
    advance_column(T, n, st, rs, q_begin, q_end, h, forcing);
    if (kSmem)
        for (long long i = 0; i < n; ++i) gcol[i * grs] = st[i * rs];
    // RunReport::per_slice_compute analogue: the warp's time, charged to lane 0's slice
    if (kMode == Mode::kBuild && P.per_slice_ns && lane == 0)
        atomicAdd(P.per_slice_ns + slice, pint_dev::globaltimer() - t_start);
}

template <Mode kMode>
int launch_columns(pint_ctx* ctx, long long n, long long columns, const HeatTables& T,
                   const ColumnPlan& P, const char* what) {
    if (columns <= 0) return PINT_OK;
    const size_t smem = sizeof(double) * 32 * static_cast<size_t>(n);
    const unsigned blocks = static_cast<unsigned>((columns + 31) / 32);
    if (smem <= 200 * 1024) {
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(heat_columns_kernel<kMode, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        heat_columns_kernel<kMode, true><<<blocks, 32, smem, ctx->stream>>>(n, T, P);
    } else {
        heat_columns_kernel<kMode, false><<<blocks, 32, 0, ctx->stream>>>(n, T, P);
    }
    return pint_check_launch(ctx, what);
}

}  // namespace

int launch_heat_factor(pint_ctx* ctx, int64_t n, int64_t total_steps, const double* r, double* factor) {
    if (n < 1 || total_steps < 0) return pint_set_error(ctx, PINT_E_INVALID, "heat_factor: bad sizes");
    if (total_steps == 0) return PINT_OK;
    const unsigned blocks = static_cast<unsigned>((total_steps + 127) / 128);
    heat_factor_kernel<<<blocks, 128, 0, ctx->stream>>>(n, total_steps, r,
                                                        reinterpret_cast<double2*>(factor), ctx->d_fail);
    return pint_check_launch(ctx, "heat_factor_kernel");
}

int launch_heat_build(pint_ctx* ctx, int64_t n, int64_t N, const int64_t* step_off,
                      const double* slice_dt, const double* factor, const double* r,
                      const double* fa, const double* fb, const double* sx, double* maps,
                      unsigned long long* per_slice_ns) {
    if (n < 1 || N < 0) return pint_set_error(ctx, PINT_E_INVALID, "heat_build: bad sizes");
    HeatTables T{reinterpret_cast<const double2*>(factor), r, fa, fb, sx};
    ColumnPlan P{};
    P.N = N;
    P.step_off = step_off;
    P.slice_dt = slice_dt;
    P.maps = maps;
    P.ldm = pint_affine_ldm(n);
    P.per_slice_ns = per_slice_ns;
    return launch_columns<Mode::kBuild>(ctx, n, N * (n + 1), T, P, "heat_columns_kernel<build>");
}

int launch_heat_integrate(pint_ctx* ctx, int64_t n, int64_t K, int64_t q0, int64_t steps, double h,
                          int with_forcing, const double* factor, const double* r,
                          const double* fa, const double* fb, const double* sx, double* y) {
    if (n < 1 || K < 0) return pint_set_error(ctx, PINT_E_INVALID, "heat_integrate: bad sizes");
    HeatTables T{reinterpret_cast<const double2*>(factor), r, fa, fb, sx};
    ColumnPlan P{};
    P.K = K;
    P.q0 = q0;
    P.steps = steps;
    P.h = h;
    P.with_forcing = with_forcing;
    P.y = y;
    return launch_columns<Mode::kIntegrate>(ctx, n, K, T, P, "heat_columns_kernel<integrate>");
}
