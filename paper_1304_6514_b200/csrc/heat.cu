// K3 — heat-equation slice maps: the n+1 basis/forced trajectories of every slice advanced
// together through backward-Euler steps (I - h a(t) L) x = y + h b(t).
//
// Replaces build_affine_propagator (nievergelt.cpp:53-66) -> make_heat_problem's integrate
// closure (pde_problems.cpp:86-98) -> solve_implicit (pde_problems.cpp:53-57) -> thomas_solve
// (linalg.cpp:77-93), which the reference runs once per trajectory per step.
//
// B200 design:
//  * The tridiagonal factor depends only on (slice, step), never on the right-hand side, so
//    heat_record_kernel computes it once per step into a record
//        {-r, fa, fb, 0, (p_0, 1/p_0), ..., (p_{n-1}, 1/p_{n-1}), c_0, ..., c_{n-1}}
//    with exactly thomas_solve's operations, so every solve stays bit-identical.
//  * x / p_i is q0 = x*rcp, rem = fma(-p, q0, x), q = fma(rem, rcp, q0) with rcp = RN(1/p_i):
//    Markstein's theorem makes q the correctly rounded quotient whenever no intermediate
//    under/overflows. Basis columns are entrywise non-negative and bounded (each step matrix is an
//    M-matrix, p_i >= 1, |c_i| < 1) and decay by at most r/p_i per row, so their quotients stay far
//    from the subnormal range and run unguarded; the warp holding the forced column (and the
//    integrate kernel, which sees caller data) checks the exponent of x and takes __ddiv_rn
//    outside [2^-960, 2^997].
//  * Lane = trajectory: column k < n starts at e_k, k == n is the forced run from 0 (c). A CTA
//    holds all ceil((n+1)/32) warps of one slice (or one warp of it when n is large): the step
//    record is staged once per CTA into shared memory by cp.async one step ahead and read as
//    broadcasts; the first RR rows of every column live in registers, the rest lane-interleaved
//    in shared memory (conflict-free). Rows leave as coalesced 256 B stores into the row-major
//    augmented map [G | c].
//  * The forced lane's quotients are range-checked OFF the dependent chain (a sticky flag);
//    if it ever trips, the kernel reports PINT_E_RANGE_RETRY and the host re-runs the build
//    with the guarded variant (exponent check on the chain, IEEE __ddiv_rn outside the range).
//
// Roofline: FP64 pipe. Algorithmic flops per slice-step: (n+1)(5n-4) + 5n (bench.py).
#include "pint_internal.cuh"

namespace {

using pint_dev::record_failure;

constexpr int kRegRows = 64;  // rows of each column held in registers (n >= kRegRows + 2)
constexpr int kMaxCtaThreads = 32 * 8;

__host__ __device__ constexpr long long rec_stride(long long n) { return 4 + 3 * n + ((3 * n) & 1); }

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
    double2* PR = reinterpret_cast<double2*>(R + 4);
    double* CC = R + 4 + 2 * n;
    double p = diag;  // thomas_solve: pivot = diag[0]; c[0] = sup[0] / pivot (linalg.cpp:80-83)
    if (p == 0.0) record_failure(fail, q, PINT_E_SINGULAR, 0.0);
    double c = (n > 1) ? __ddiv_rn(negr, p) : 0.0;
    PR[0] = make_double2(p, __drcp_rn(p));
    CC[0] = c;
    for (long long i = 1; i < n; ++i) {  // pivot = diag - sub*c[i-1]; c[i] = sup/pivot (:84-88)
        p = __dsub_rn(diag, __dmul_rn(negr, c));
        if (p == 0.0) record_failure(fail, q, PINT_E_SINGULAR, static_cast<double>(i));
        c = (i < n - 1) ? __ddiv_rn(negr, p) : 0.0;
        PR[i] = make_double2(p, __drcp_rn(p));
        CC[i] = c;
    }
}

__device__ __forceinline__ double div_fast(double x, double2 pr) {
    const double q0 = __dmul_rn(x, pr.y);
    const double rem = __fma_rn(-pr.x, q0, x);
    return __fma_rn(rem, pr.y, q0);
}

__device__ __forceinline__ double div_guarded(double x, double2 pr) {
    const unsigned e = (static_cast<unsigned>(__double2hiint(x)) >> 20) & 0x7ffu;
    if (e - 63u > 1957u) return __ddiv_rn(x, pr.x);  // zero/subnormal/tiny/huge/non-finite
    return div_fast(x, pr);
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void stage_record(double* dst, const double* src, int chunks, int lane) {
    for (int c = lane; c < chunks; c += 32)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst + 2 * c)), "l"(src + 2 * c));
    asm volatile("cp.async.commit_group;\n" ::);
}

struct BuildPlan {
    int n;
    int N;
    int wb;             // basis warps per slice = ceil(n/32)
    int warps_per_cta;  // wb (one CTA per slice) or 1
    int ctas_per_slice;
    int forcing_ctas;   // CTAs holding the forced (c) runs, warps_per_cta * 32 slices each
    const double* rec;
    const double* sx;
    const int64_t* step_off;
    const double* slice_dt;
    double* maps;
    long long ldm;
    unsigned long long* per_slice_ns;
    FailRec* fail;
};

// Forcing (pde_problems.cpp:91-94) folded into the row update: x + h*(fa s + fb s), where
// heat_forcing(x_i, t) is fa*s + fb*s with fa = -sin t, fb = ((a pi) pi) cos t (pde_problems.cpp:26-29).
__device__ __forceinline__ double forced(double x, double h, double fa, double fb, double s) {
    return __dadd_rn(x, __dmul_rn(h, __dadd_rn(__dmul_rn(fa, s), __dmul_rn(fb, s))));
}

__device__ __forceinline__ bool out_of_range(double x) {
    const unsigned e = (static_cast<unsigned>(__double2hiint(x)) >> 20) & 0x7ffu;
    return e - 63u > 1957u;
}

// One backward-Euler step of one basis column from a record in shared memory: forward
// elimination (linalg.cpp:84-90), back substitution (linalg.cpp:91). Rows [0, RR) in reg[],
// the rest at st[32*(i-RR)].
template <int RR>
__device__ __forceinline__ void basis_step(double (&reg)[RR > 0 ? RR : 1], double* st, const double* R, int n) {
    const double negr = R[0];
    const double2* PR = reinterpret_cast<const double2*>(R + 4);
    const double* CC = R + 4 + 2 * n;
    double d = 0.0;
#pragma unroll
    for (int i = 0; i < RR; ++i) {
        const double num = (i == 0) ? reg[i] : __dsub_rn(reg[i], __dmul_rn(negr, d));
        d = div_fast(num, PR[i]);
        reg[i] = d;
    }
    {
        double* s = st;
        const double2* pr = PR + RR;
#pragma unroll 8
        for (int i = RR; i < n; ++i, s += 32, ++pr) {
            const double num = (RR == 0 && i == 0) ? *s : __dsub_rn(*s, __dmul_rn(negr, d));
            d = div_fast(num, *pr);
            *s = d;
        }
    }
    {
        double* s = st + (n - 2 - RR) * 32;
        const double* c = CC + (n - 2);
#pragma unroll 8
        for (int i = n - 2; i >= RR; --i, s -= 32, --c) {
            d = __dsub_rn(*s, __dmul_rn(*c, d));
            *s = d;
        }
    }
#pragma unroll
    for (int i = RR - 1; i >= 0; --i) {
        d = __dsub_rn(reg[i], __dmul_rn(CC[i], d));
        reg[i] = d;
    }
}

__device__ __forceinline__ void stage_record_cta(double* dst, const double* src, int chunks) {
    for (int c = threadIdx.x; c < chunks; c += blockDim.x)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst + 2 * c)), "l"(src + 2 * c));
    asm volatile("cp.async.commit_group;\n" ::);
}

// Forcing kernel: one warp per CTA holds the forced (c) runs of 32 consecutive slices, lane = slice.
// Each lane's records are private (different slices), so pivots/reciprocals and multipliers stream
// from L2 kD rows ahead through register rings; the next step's first rows are fetched during the
// current back substitution. State lives in shared memory, lane-interleaved.
// Dynamic smem: sx[n] (even) | state[n * 32]
template <bool kGuard>
__device__ void forcing_cta(const BuildPlan& P, int fcta) {
    constexpr int kD = 32;
    extern __shared__ __align__(16) double smem[];
    const int n = P.n;
    const int lane = threadIdx.x & 31;
    double* sx = smem;
    double* st = sx + ((n + 1) & ~1) + lane;
    for (int i = lane; i < n; i += 32) sx[i] = P.sx[i];
    const int slice = fcta * 32 + lane;
    const bool active = slice < P.N;
    const long long q0 = active ? P.step_off[slice] : 0;
    const int steps = active ? static_cast<int>(P.step_off[slice + 1] - q0) : 0;
    const double h = active ? P.slice_dt[slice] : 0.0;
    const int max_steps = __reduce_max_sync(0xffffffffu, steps);
    const long long RS = rec_stride(n);
    for (int i = 0; i < n; ++i) st[i * 32] = 0.0;  // c = the forced run from the zero state
    __syncwarp();

    double2 pq[kD];
    double cq[kD];
    auto load_head = [&](const double* R) {
        const double2* PR = reinterpret_cast<const double2*>(R + 4);
#pragma unroll
        for (int u = 0; u < kD; ++u) pq[u] = (u < n) ? __ldg(PR + u) : make_double2(1.0, 1.0);
    };
    if (steps > 0) load_head(P.rec + q0 * RS);
    bool bad = false;
    for (int s = 0; s < max_steps; ++s) {
        if (s >= steps) continue;
        const double* R = P.rec + (q0 + s) * RS;
        const double negr = __ldg(R), fa = __ldg(R + 1), fb = __ldg(R + 2);
        const double2* PR = reinterpret_cast<const double2*>(R + 4);
        const double* CC = R + 4 + 2 * n;
#pragma unroll
        for (int u = 0; u < kD; ++u) cq[u] = (n - 2 - u >= 0) ? __ldg(CC + (n - 2 - u)) : 0.0;
        // forward elimination with the forcing folded in (linalg.cpp:84-90, pde_problems.cpp:91-94)
        double d = 0.0;
        for (int i0 = 0; i0 < n; i0 += kD) {
#pragma unroll
            for (int u = 0; u < kD; ++u) {
                const int i = i0 + u;
                if (i < n) {
                    const double2 pr = pq[u];
                    if (i + kD < n) pq[u] = __ldg(PR + i + kD);
                    const double x = forced(st[i * 32], h, fa, fb, sx[i]);
                    const double num = (i == 0) ? x : __dsub_rn(x, __dmul_rn(negr, d));
                    if (!kGuard) bad |= out_of_range(num);
                    d = kGuard ? div_guarded(num, pr) : div_fast(num, pr);
                    st[i * 32] = d;
                }
            }
        }
        if (s + 1 < steps) load_head(R + RS);  // next step's first rows, hidden behind the back sweep
        // back substitution (linalg.cpp:91), multipliers kD rows ahead
        for (int t0 = 0; n - 2 - t0 >= 0; t0 += kD) {
#pragma unroll
            for (int u = 0; u < kD; ++u) {
                const int i = n - 2 - t0 - u;
                if (i >= 0) {
                    const double c = cq[u];
                    if (i - kD >= 0) cq[u] = __ldg(CC + i - kD);
                    d = __dsub_rn(st[i * 32], __dmul_rn(c, d));
                    st[i * 32] = d;
                }
            }
        }
    }
    if (active) {
        double* gp = P.maps + static_cast<long long>(slice) * n * P.ldm + n;
        for (int i = 0; i < n; ++i) gp[i * P.ldm] = st[i * 32];
    }
    if (bad) record_failure(P.fail, slice, PINT_E_RANGE_RETRY, static_cast<double>(n));
}

// Basis CTA = warps [c*warps_per_cta, ...) of one slice, lane = basis column e_k.
// Dynamic smem: rec[2][RS] | state[warps_per_cta][(n - RR) * 32]
template <int RR>
__device__ void basis_cta(const BuildPlan& P, int b) {
    extern __shared__ __align__(16) double smem[];
    const unsigned long long t_start = pint_dev::globaltimer();
    const int n = P.n;
    const int lane = threadIdx.x & 31, wcta = threadIdx.x >> 5;
    const int slice = b / P.ctas_per_slice;
    const int g = (b - slice * P.ctas_per_slice) * P.warps_per_cta + wcta;  // warp in slice
    const long long RS = rec_stride(n);
    double* recbuf = smem;
    double* st = smem + 2 * RS + static_cast<long long>(wcta) * (n - RR) * 32 + lane;
    const int k = g * 32 + lane;
    const long long q_begin = P.step_off[slice], q_end = P.step_off[slice + 1];
    const int chunks = static_cast<int>(RS / 2);
    const double* rec = P.rec;

    if (q_begin < q_end) stage_record_cta(recbuf, rec + q_begin * RS, chunks);
    double reg[RR > 0 ? RR : 1];
#pragma unroll
    for (int i = 0; i < RR; ++i) reg[i] = (i == k) ? 1.0 : 0.0;  // e_k
    for (int i = RR; i < n; ++i) st[(i - RR) * 32] = (i == k) ? 1.0 : 0.0;

    int cur = 0;
    for (long long q = q_begin; q < q_end; ++q) {
        if (q + 1 < q_end) {
            stage_record_cta(recbuf + (cur ^ 1) * RS, rec + (q + 1) * RS, chunks);
            asm volatile("cp.async.wait_group 1;\n" ::);
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::);
        }
        __syncthreads();  // record q visible to every warp
        basis_step<RR>(reg, st, recbuf + cur * RS, n);
        __syncthreads();  // buffer `cur` is refilled next iteration
        cur ^= 1;
    }
    if (k < n) {
        double* gp = P.maps + static_cast<long long>(slice) * n * P.ldm + k;
#pragma unroll
        for (int i = 0; i < RR; ++i) gp[i * P.ldm] = reg[i];
        for (int i = RR; i < n; ++i) gp[i * P.ldm] = st[(i - RR) * 32];
    }
    if (P.per_slice_ns && threadIdx.x == 0) atomicAdd(P.per_slice_ns + slice, pint_dev::globaltimer() - t_start);
}

// Two kernels so each gets its own register allocation; the forcing kernel runs on the context's
// side stream concurrently with the basis kernel. kGuard affects only the forced columns: basis
// columns are positive and never need it.
template <int RR>
__global__ void __launch_bounds__(kMaxCtaThreads) heat_basis_kernel(BuildPlan P) {
    basis_cta<RR>(P, blockIdx.x);
}

template <bool kGuard>
__global__ void __launch_bounds__(32) heat_forcing_kernel(BuildPlan P) {
    forcing_cta<kGuard>(P, blockIdx.x);
}

// ---- integrate: K caller columns of one slice, lane = column (guarded division) ---------------
struct IntegratePlan {
    int n;
    long long K, q0, steps;
    double h;
    int with_forcing;
    const double* rec;
    const double* sx;
    double* y;
};

__global__ void __launch_bounds__(32) heat_integrate_kernel(IntegratePlan P) {
    extern __shared__ __align__(16) double smem[];
    const int n = P.n;
    const int lane = threadIdx.x;
    const long long col = static_cast<long long>(blockIdx.x) * 32 + lane;
    const bool active = col < P.K;
    double* st = smem + lane;
    double* sx = smem + 32 * n;
    for (int i = lane; i < n; i += 32) sx[i] = P.sx[i];
    for (int i = 0; i < n; ++i) st[i * 32] = active ? P.y[col * n + i] : 0.0;
    __syncwarp();
    const long long RS = rec_stride(n);
    const bool forcing = P.with_forcing != 0;
    for (long long q = P.q0; q < P.q0 + P.steps; ++q) {
        const double* R = P.rec + q * RS;
        const double negr = __ldg(R), fa = __ldg(R + 1), fb = __ldg(R + 2);
        const double2* PR = reinterpret_cast<const double2*>(R + 4);
        const double* CC = R + 4 + 2 * n;
        double d = 0.0;
        for (int i = 0; i < n; ++i) {
            double x = st[i * 32];
            if (forcing) x = forced(x, P.h, fa, fb, sx[i]);
            const double num = (i == 0) ? x : __dsub_rn(x, __dmul_rn(negr, d));
            d = div_guarded(num, __ldg(PR + i));
            st[i * 32] = d;
        }
        for (int i = n - 2; i >= 0; --i) {
            d = __dsub_rn(st[i * 32], __dmul_rn(__ldg(CC + i), d));
            st[i * 32] = d;
        }
    }
    if (active)
        for (int i = 0; i < n; ++i) P.y[col * n + i] = st[i * 32];
}




template <class K>
void smem_attrs(K kern, size_t smem) {
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
}

template <int RR, bool kGuard>
int launch_build(pint_ctx* ctx, BuildPlan P) {
    // basis: one CTA per slice when two such CTAs fit an SM, else one CTA per warp
    const size_t state_cta = sizeof(double) * static_cast<size_t>(P.n - RR) * 32;
    const size_t rec_bytes = sizeof(double) * 2 * rec_stride(P.n);
    P.warps_per_cta = (P.wb <= kMaxCtaThreads / 32 && rec_bytes + state_cta * P.wb <= 112 * 1024) ? P.wb : 1;
    P.ctas_per_slice = P.wb / P.warps_per_cta;
    P.forcing_ctas = (P.N + 31) / 32;  // forcing kernel: one warp per CTA, 32 slices per warp
    const size_t smem_b = rec_bytes + state_cta * P.warps_per_cta;
    const size_t smem_f = sizeof(double) * (((P.n + 1) & ~1) + static_cast<size_t>(P.n) * 32);
    if (smem_b > 227 * 1024 || smem_f > 227 * 1024)
        return pint_set_error(ctx, PINT_E_INVALID, "heat_build: n too large for shared memory");
    auto kb = heat_basis_kernel<RR>;
    auto kf = heat_forcing_kernel<kGuard>;
    smem_attrs(kb, smem_b);
    smem_attrs(kf, smem_f);
    // fork: forcing runs on the side stream, overlapping the basis kernel; join before returning
    cudaEventRecord(ctx->ev_fork, ctx->stream);
    cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0);
    kf<<<static_cast<unsigned>(P.forcing_ctas), 32, smem_f, ctx->side>>>(P);
    if (const int rc = pint_check_launch(ctx, "heat_forcing_kernel")) return rc;
    kb<<<static_cast<unsigned>(static_cast<long long>(P.N) * P.ctas_per_slice), 32 * P.warps_per_cta, smem_b,
         ctx->stream>>>(P);
    if (const int rc = pint_check_launch(ctx, "heat_basis_kernel")) return rc;
    cudaEventRecord(ctx->ev_join, ctx->side);
    cudaStreamWaitEvent(ctx->stream, ctx->ev_join, 0);
    return PINT_OK;
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
                      const double* records, const double* sx, double* maps, unsigned long long* per_slice_ns,
                      int guarded) {
    if (n < 1 || N < 0) return pint_set_error(ctx, PINT_E_INVALID, "heat_build: bad sizes");
    if (N == 0) return PINT_OK;
    if (n > (1 << 20) || N > (1 << 26)) return pint_set_error(ctx, PINT_E_INVALID, "heat_build: sizes out of range");
    BuildPlan P{};
    P.n = static_cast<int>(n);
    P.N = static_cast<int>(N);
    P.wb = static_cast<int>((n + 31) / 32);
    P.rec = records;
    P.sx = sx;
    P.step_off = step_off;
    P.slice_dt = slice_dt;
    P.maps = maps;
    P.ldm = pint_affine_ldm(n);
    P.per_slice_ns = per_slice_ns;
    P.fail = ctx->d_fail;
    if (n >= kRegRows + 2)
        return guarded ? launch_build<kRegRows, true>(ctx, P) : launch_build<kRegRows, false>(ctx, P);
    return guarded ? launch_build<0, true>(ctx, P) : launch_build<0, false>(ctx, P);
}

int launch_heat_integrate(pint_ctx* ctx, int64_t n, int64_t K, int64_t q0, int64_t steps, double h,
                          int with_forcing, const double* records, const double* sx, double* y) {
    if (n < 1 || K < 0) return pint_set_error(ctx, PINT_E_INVALID, "heat_integrate: bad sizes");
    if (K == 0) return PINT_OK;
    IntegratePlan P{static_cast<int>(n), K, q0, steps, h, with_forcing, records, sx, y};
    const size_t smem = sizeof(double) * (static_cast<size_t>(n) * 32 + n);
    if (smem > 227 * 1024) return pint_set_error(ctx, PINT_E_INVALID, "heat_integrate: n too large");
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(heat_integrate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    heat_integrate_kernel<<<static_cast<unsigned>((K + 31) / 32), 32, smem, ctx->stream>>>(P);
    return pint_check_launch(ctx, "heat_integrate_kernel");
}
