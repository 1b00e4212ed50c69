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

constexpr int kRegRows = 56;  // rows of each column held in registers (n >= kRegRows + 2)
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
    int wps;            // warps per slice = ceil((n+1)/32)
    int warps_per_cta;  // wps (one CTA per slice) or 1
    int ctas_per_slice;
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
// heat_forcing is fa*s + fb*s (pde_problems.cpp:26-29). fa/fb arrive pre-multiplied by f in {0,1}.
__device__ __forceinline__ double forced(double x, double h, double fa, double fb, double s) {
    return __dadd_rn(x, __dmul_rn(h, __dadd_rn(__dmul_rn(fa, s), __dmul_rn(fb, s))));
}

__device__ __forceinline__ bool out_of_range(double x) {
    const unsigned e = (static_cast<unsigned>(__double2hiint(x)) >> 20) & 0x7ffu;
    return e - 63u > 1957u;
}

// One backward-Euler step of one column: forward elimination (linalg.cpp:84-90) with the forcing
// folded in, then back substitution (linalg.cpp:91). Rows [0, RR) in reg[], the rest at st[32*(i-RR)].
template <int RR, bool kMixed, bool kGuard>
__device__ __forceinline__ void column_step(double (&reg)[RR > 0 ? RR : 1], double* st, const double* R, int n,
                                            double h, double f, const double* sx, bool forced_lane,
                                            bool& bad) {
    const double negr = R[0];
    const double ffa = kMixed ? __dmul_rn(f, R[1]) : 0.0;  // f in {0, 1}: exact
    const double ffb = kMixed ? __dmul_rn(f, R[2]) : 0.0;
    const double2* PR = reinterpret_cast<const double2*>(R + 4);
    const double* CC = R + 4 + 2 * n;
    double d = 0.0;
#pragma unroll
    for (int i = 0; i < RR; ++i) {
        const double x = kMixed ? forced(reg[i], h, ffa, ffb, sx[i]) : reg[i];
        const double num = (i == 0) ? x : __dsub_rn(x, __dmul_rn(negr, d));
        if (kMixed && !kGuard) bad |= forced_lane && out_of_range(num);
        d = kGuard ? div_guarded(num, PR[i]) : div_fast(num, PR[i]);
        reg[i] = d;
    }
    {
        double* s = st;
        const double2* pr = PR + RR;
#pragma unroll 8
        for (int i = RR; i < n; ++i, s += 32, ++pr) {
            const double x = kMixed ? forced(*s, h, ffa, ffb, sx[i]) : *s;
            const double num = (RR == 0 && i == 0) ? x : __dsub_rn(x, __dmul_rn(negr, d));
            if (kMixed && !kGuard) bad |= forced_lane && out_of_range(num);
            d = kGuard ? div_guarded(num, *pr) : div_fast(num, *pr);
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

// CTA = warps [c*warps_per_cta, ...) of one slice. Dynamic smem:
// rec[2][RS] | sx[n] (even) | state[warps_per_cta][(n - RR) * 32]
template <int RR, bool kGuard>
__global__ void __launch_bounds__(kMaxCtaThreads) heat_build_kernel(BuildPlan P) {
    extern __shared__ __align__(16) double smem[];
    const unsigned long long t_start = pint_dev::globaltimer();
    const int n = P.n;
    const int lane = threadIdx.x & 31, wcta = threadIdx.x >> 5;
    const int slice = blockIdx.x / P.ctas_per_slice;
    const int g = (blockIdx.x - slice * P.ctas_per_slice) * P.warps_per_cta + wcta;  // warp in slice
    const long long RS = rec_stride(n);
    double* recbuf = smem;
    double* sx = smem + 2 * RS;
    double* st = sx + ((n + 1) & ~1) + static_cast<long long>(wcta) * (n - RR) * 32 + lane;
    const int k = g * 32 + lane;
    const bool active = k <= n;
    const bool forced_lane = (k == n);
    const bool mixed = (g == P.wps - 1);
    const double f = forced_lane ? 1.0 : 0.0;
    const long long q_begin = P.step_off[slice], q_end = P.step_off[slice + 1];
    const double h = P.slice_dt[slice];
    const int chunks = static_cast<int>(RS / 2);
    const double* rec = P.rec;

    if (q_begin < q_end) stage_record_cta(recbuf, rec + q_begin * RS, chunks);
    for (int i = threadIdx.x; i < n; i += blockDim.x) sx[i] = P.sx[i];
    double reg[RR > 0 ? RR : 1];
#pragma unroll
    for (int i = 0; i < RR; ++i) reg[i] = (i == k) ? 1.0 : 0.0;
    for (int i = RR; i < n; ++i) st[(i - RR) * 32] = (i == k) ? 1.0 : 0.0;

    bool bad = false;
    int cur = 0;
    for (long long q = q_begin; q < q_end; ++q) {
        if (q + 1 < q_end) {
            stage_record_cta(recbuf + (cur ^ 1) * RS, rec + (q + 1) * RS, chunks);
            asm volatile("cp.async.wait_group 1;\n" ::);
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::);
        }
        __syncthreads();  // record q (and sx) visible to every warp
        const double* R = recbuf + cur * RS;
        if (mixed) column_step<RR, true, kGuard>(reg, st, R, n, h, f, sx, forced_lane, bad);
        else column_step<RR, false, kGuard>(reg, st, R, n, h, f, sx, forced_lane, bad);
        __syncthreads();  // buffer `cur` is refilled next iteration
        cur ^= 1;
    }
    if (active) {
        double* gp = P.maps + static_cast<long long>(slice) * n * P.ldm + k;
#pragma unroll
        for (int i = 0; i < RR; ++i) gp[i * P.ldm] = reg[i];
        for (int i = RR; i < n; ++i) gp[i * P.ldm] = st[(i - RR) * 32];
    }
    if (bad) record_failure(P.fail, slice, PINT_E_RANGE_RETRY, static_cast<double>(k));
    if (P.per_slice_ns && threadIdx.x == 0) atomicAdd(P.per_slice_ns + slice, pint_dev::globaltimer() - t_start);
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


size_t build_smem(int n, int rr, int warps_per_cta) {
    return sizeof(double) * (2 * rec_stride(n) + ((n + 1) & ~1) + static_cast<size_t>(n - rr) * 32 * warps_per_cta);
}

template <int RR, bool kGuard>
int launch_build(pint_ctx* ctx, BuildPlan P) {
    // one CTA per slice when two such CTAs fit an SM, else one CTA per warp
    P.warps_per_cta = (P.wps <= kMaxCtaThreads / 32 && build_smem(P.n, RR, P.wps) <= 112 * 1024) ? P.wps : 1;
    P.ctas_per_slice = P.wps / P.warps_per_cta;
    const size_t smem = build_smem(P.n, RR, P.warps_per_cta);
    if (smem > 227 * 1024) return pint_set_error(ctx, PINT_E_INVALID, "heat_build: n too large for shared memory");
    auto kern = heat_build_kernel<RR, kGuard>;
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    const long long blocks = static_cast<long long>(P.N) * P.ctas_per_slice;
    kern<<<static_cast<unsigned>(blocks), 32 * P.warps_per_cta, smem, ctx->stream>>>(P);
    return pint_check_launch(ctx, "heat_build_kernel");
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
    P.wps = static_cast<int>((n + 1 + 31) / 32);
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
