// K3 — heat-equation slice maps: the n+1 basis/forced trajectories of every slice advanced
// together through backward-Euler steps (I - h a(t) L) x = y + h b(t).
//
// Replaces build_affine_propagator (nievergelt.cpp:53-66) -> make_heat_problem's integrate
// closure (pde_problems.cpp:86-98) -> solve_implicit (pde_problems.cpp:53-57) -> thomas_solve
// (linalg.cpp:77-93), which the reference runs once per trajectory per step.
//
// B200 design:
//  * The tridiagonal factor depends only on (slice, step), never on the right-hand side, so
//    heat_record_kernel computes it once per step (one thread per step, all steps in parallel)
//    into a per-step record {-r, fa, fb, 0, p[n], rcp[n], c[n]} instead of n+1 times. Same
//    operations and rounding as thomas_solve, so every solve stays bit-identical.
//  * Division x / p_i is done as q0 = x * rcp_i, rem = fma(-p_i, q0, x), q = fma(rem, rcp_i, q0)
//    with rcp_i = RN(1/p_i) (__drcp_rn): Markstein's theorem makes q the correctly rounded
//    quotient (no over/underflow is possible here: p_i >= 1 and |x| >= 2^-960 is checked on
//    the exponent bits, anything else takes the IEEE __ddiv_rn path). 5 dependent FP64 ops per
//    row instead of the ~12 of a full division.
//  * One warp per (slice, 32-column group); lane = trajectory. Column k < n starts at e_k, column
//    n (the c run) at 0 with forcing. All lanes of a warp share the slice, so the step's record
//    is staged once into shared memory by cp.async one step ahead (double-buffered) and read as
//    broadcasts; the column state is lane-interleaved in shared memory (conflict-free), and the
//    final rows go out as coalesced 256 B stores into the row-major augmented map [G | c].
//
// Roofline: FP64 pipe. Algorithmic flops per slice-step: (n+1)(5n-4) + 5n (bench.py).
#include "pint_internal.cuh"

namespace {

using pint_dev::record_failure;

__host__ __device__ constexpr long long rec_stride(long long n) { return ((4 + 3 * n) + 1) / 2 * 2; }

// Per-step record: the Thomas forward pivots of tridiag(-r, 1+2r, -r) (linalg.cpp:80-90).
__global__ void heat_record_kernel(long long n, long long Q, const double* __restrict__ r_tab,
                                   const double* __restrict__ fa, const double* __restrict__ fb,
                                   double* __restrict__ rec, FailRec* fail) {
    const long long q = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= Q) return;
    const double r = r_tab[q];
    const double negr = -r;                                  // sub = sup = -r (pde_problems.cpp:55)
    const double diag = __dadd_rn(1.0, __dmul_rn(2.0, r));   // 1.0 + 2.0 * r
    double* R = rec + q * rec_stride(n);
    R[0] = negr;
    R[1] = fa[q];
    R[2] = fb[q];
    R[3] = 0.0;
    double* P = R + 4;
    double* RC = R + 4 + n;
    double* CC = R + 4 + 2 * n;
    double p = diag;
    if (p == 0.0) record_failure(fail, q, PINT_E_SINGULAR, 0.0);
    double c = (n > 1) ? __ddiv_rn(negr, p) : 0.0;
    P[0] = p;
    RC[0] = __drcp_rn(p);
    CC[0] = c;
    for (long long i = 1; i < n; ++i) {
        p = __dsub_rn(diag, __dmul_rn(negr, c));
        if (p == 0.0) record_failure(fail, q, PINT_E_SINGULAR, static_cast<double>(i));
        c = (i < n - 1) ? __ddiv_rn(negr, p) : 0.0;
        P[i] = p;
        RC[i] = __drcp_rn(p);
        CC[i] = c;
    }
}

// x / p, correctly rounded, given rcp = RN(1/p) (see header comment).
__device__ __forceinline__ double div_rcp(double x, double p, double rcp) {
    const unsigned e = (static_cast<unsigned>(__double2hiint(x)) >> 20) & 0x7ffu;
    if (e < 63u || e > 2020u) return __ddiv_rn(x, p);  // zero/subnormal/tiny/huge/non-finite
    const double q0 = __dmul_rn(x, rcp);
    const double rem = __fma_rn(-p, q0, x);
    return __fma_rn(rem, rcp, q0);
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void stage_record(double* dst, const double* src, int chunks, int lane) {
    for (int c = lane; c < chunks; c += 32)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst + 2 * c)), "l"(src + 2 * c));
    asm volatile("cp.async.commit_group;\n" ::);
}

enum class Mode { kBuild, kIntegrate };

struct ColumnPlan {
    long long n;
    const double* rec;   // per-step records
    const double* sx;    // sin(pi x_i)
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

// Dynamic smem: rec[2][RS] | sx[n] | state[n][32] (state only when kSmem).
template <Mode kMode, bool kSmem>
__global__ void __launch_bounds__(32)
heat_columns_kernel(ColumnPlan P) {
    extern __shared__ __align__(16) double smem[];
    const unsigned long long t_start = pint_dev::globaltimer();
    const long long n = P.n;
    const long long RS = rec_stride(n);
    double* recbuf = smem;
    double* sx_s = smem + 2 * RS;
    double* state_s = sx_s + ((n + 1) / 2) * 2;
    const int lane = threadIdx.x;

    long long slice = 0, k, q_begin, q_end;
    double h;
    bool active, forcing;
    double* gcol;
    long long grs;
    if (kMode == Mode::kBuild) {
        const long long wps = (n + 1 + 31) / 32;  // warps per slice
        slice = blockIdx.x / wps;
        k = (blockIdx.x % wps) * 32 + lane;
        active = k <= n;
        forcing = (k == n);
        q_begin = P.step_off[slice];
        q_end = P.step_off[slice + 1];
        h = P.slice_dt[slice];
        gcol = P.maps + slice * n * P.ldm + (active ? k : 0);
        grs = P.ldm;
    } else {
        k = static_cast<long long>(blockIdx.x) * 32 + lane;
        active = k < P.K;
        forcing = P.with_forcing != 0;
        q_begin = P.q0;
        q_end = P.q0 + P.steps;
        h = P.h;
        gcol = P.y + (active ? k : 0) * n;
        grs = 1;
    }
    // inactive lanes keep a private zero column in smem (or skip work in global mode)
    double* st = kSmem ? state_s + lane : gcol;
    const long long rs = kSmem ? 32 : grs;
    const bool work = kSmem || active;
    const int chunks = static_cast<int>(RS / 2);

    if (q_begin < q_end) stage_record(recbuf, P.rec + q_begin * RS, chunks, lane);
    const bool any_forcing = __any_sync(0xffffffffu, forcing && active);
    if (any_forcing)
        for (long long i = lane; i < n; i += 32) sx_s[i] = P.sx[i];
    if (work)
        for (long long i = 0; i < n; ++i) {
            double v;
            if (kMode == Mode::kBuild) v = (i == k) ? 1.0 : 0.0;  // e_k, or 0 for the c run
            else v = active ? gcol[i] : 0.0;
            st[i * rs] = v;
        }

    int cur = 0;
    for (long long q = q_begin; q < q_end; ++q) {
        if (q + 1 < q_end) {
            stage_record(recbuf + (cur ^ 1) * RS, P.rec + (q + 1) * RS, chunks, lane);
            asm volatile("cp.async.wait_group 1;\n" ::);
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::);
        }
        __syncwarp();
        const double* R = recbuf + cur * RS;
        if (work) {
            const double negr = R[0];
            const double* Pv = R + 4;
            const double* Rc = R + 4 + n;
            const double* Cc = R + 4 + 2 * n;
            // forward elimination (linalg.cpp:80-90), forcing folded in (pde_problems.cpp:91-94)
            double dprev = 0.0;
            if (forcing) {
                const double fa = R[1], fb = R[2];
                for (long long i = 0; i < n; ++i) {
                    const double s = sx_s[i];
                    const double b = __dadd_rn(__dmul_rn(fa, s), __dmul_rn(fb, s));
                    const double x = __dadd_rn(st[i * rs], __dmul_rn(h, b));
                    const double num = (i == 0) ? x : __dsub_rn(x, __dmul_rn(negr, dprev));
                    dprev = div_rcp(num, Pv[i], Rc[i]);
                    st[i * rs] = dprev;
                }
            } else {
                dprev = div_rcp(st[0], Pv[0], Rc[0]);
                st[0] = dprev;
#pragma unroll 4
                for (long long i = 1; i < n; ++i) {
                    const double num = __dsub_rn(st[i * rs], __dmul_rn(negr, dprev));
                    dprev = div_rcp(num, Pv[i], Rc[i]);
                    st[i * rs] = dprev;
                }
            }
            // back substitution (linalg.cpp:91)
            double dnext = dprev;
#pragma unroll 4
            for (long long i = n - 2; i >= 0; --i) {
                const double d = __dsub_rn(st[i * rs], __dmul_rn(Cc[i], dnext));
                st[i * rs] = d;
                dnext = d;
            }
        }
        __syncwarp();  // everyone is done with buffer `cur` before it is refilled
        cur ^= 1;
    }
    if (kSmem && active)
        for (long long i = 0; i < n; ++i) gcol[i * grs] = st[i * rs];
    // RunReport::per_slice_compute analogue: the warp's time, charged to its slice
    if (kMode == Mode::kBuild && P.per_slice_ns && lane == 0)
        atomicAdd(P.per_slice_ns + slice, pint_dev::globaltimer() - t_start);
}

template <Mode kMode>
int launch_columns(pint_ctx* ctx, const ColumnPlan& P, long long warps, const char* what) {
    if (warps <= 0) return PINT_OK;
    const long long n = P.n;
    const size_t base = sizeof(double) * (2 * rec_stride(n) + ((n + 1) / 2) * 2);
    const size_t with_state = base + sizeof(double) * 32 * static_cast<size_t>(n);
    const unsigned blocks = static_cast<unsigned>(warps);
    if (with_state <= 200 * 1024) {
        if (with_state > 48 * 1024)
            cudaFuncSetAttribute(heat_columns_kernel<kMode, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(with_state));
        heat_columns_kernel<kMode, true><<<blocks, 32, with_state, ctx->stream>>>(P);
    } else {
        if (base > 48 * 1024)
            cudaFuncSetAttribute(heat_columns_kernel<kMode, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(base));
        heat_columns_kernel<kMode, false><<<blocks, 32, base, ctx->stream>>>(P);
    }
    return pint_check_launch(ctx, what);
}

}  // namespace

int64_t heat_record_stride(int64_t n) { return rec_stride(n); }

int launch_heat_factor(pint_ctx* ctx, int64_t n, int64_t total_steps, const double* r, const double* fa,
                       const double* fb, double* records) {
    if (n < 1 || total_steps < 0) return pint_set_error(ctx, PINT_E_INVALID, "heat_factor: bad sizes");
    if (total_steps == 0) return PINT_OK;
    const unsigned blocks = static_cast<unsigned>((total_steps + 127) / 128);
    heat_record_kernel<<<blocks, 128, 0, ctx->stream>>>(n, total_steps, r, fa, fb, records, ctx->d_fail);
    return pint_check_launch(ctx, "heat_record_kernel");
}

int launch_heat_build(pint_ctx* ctx, int64_t n, int64_t N, const int64_t* step_off, const double* slice_dt,
                      const double* records, const double* sx, double* maps, unsigned long long* per_slice_ns) {
    if (n < 1 || N < 0) return pint_set_error(ctx, PINT_E_INVALID, "heat_build: bad sizes");
    ColumnPlan P{};
    P.n = n;
    P.rec = records;
    P.sx = sx;
    P.N = N;
    P.step_off = step_off;
    P.slice_dt = slice_dt;
    P.maps = maps;
    P.ldm = pint_affine_ldm(n);
    P.per_slice_ns = per_slice_ns;
    const long long wps = (n + 1 + 31) / 32;
    return launch_columns<Mode::kBuild>(ctx, P, N * wps, "heat_columns_kernel<build>");
}

int launch_heat_integrate(pint_ctx* ctx, int64_t n, int64_t K, int64_t q0, int64_t steps, double h,
                          int with_forcing, const double* records, const double* sx, double* y) {
    if (n < 1 || K < 0) return pint_set_error(ctx, PINT_E_INVALID, "heat_integrate: bad sizes");
    ColumnPlan P{};
    P.n = n;
    P.rec = records;
    P.sx = sx;
    P.K = K;
    P.q0 = q0;
    P.steps = steps;
    P.h = h;
    P.with_forcing = with_forcing;
    P.y = y;
    return launch_columns<Mode::kIntegrate>(ctx, P, (K + 31) / 32, "heat_columns_kernel<integrate>");
}
