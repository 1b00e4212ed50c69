// K3 — heat-equation slice maps: the n+1 basis/forced trajectories of every slice advanced
// together through backward-Euler steps (I - h a(t) L) x = y + h b(t).
//
// Replaces build_affine_propagator (nievergelt.cpp:53-66) -> make_heat_problem's integrate
// closure (pde_problems.cpp:86-98) -> solve_implicit (pde_problems.cpp:53-57) -> thomas_solve
// (linalg.cpp:77-93), which the reference runs once per trajectory per step.
//
// B200 design:
//  * The tridiagonal factor depends only on (slice, step), never on the right-hand side, so
//    heat_record_kernel computes it once per (slice, step) with exactly thomas_solve's operations
//    (every solve stays bit-identical). Records are stored slice-minor:
//        hdr[3][S][N] = {-r, fa, fb},  pr[S][n][N] = (p_i, RN(1/p_i)),  cc[S][n][N] = c_i
//    (plus the forcing increments h*b_i[S][n][N]) so the record kernel (thread = (step, slice))
//    writes coalesced, and a slice CTA gathers its column with 16-/8-byte cp.async chunks.
//  * x / p_i is q0 = x*rcp, rem = fma(-p, q0, x), q = fma(rem, rcp, q0) with rcp = RN(1/p_i):
//    Markstein's theorem makes q the correctly rounded quotient whenever no intermediate
//    under/overflows. Basis columns are entrywise non-negative and bounded (each step matrix is an
//    M-matrix, p_i >= 1, |c_i| < 1), so their quotients stay far from the subnormal range and run
//    unguarded. Forced columns are range-checked OFF the dependent chain (a sticky flag); if it
//    ever trips, the kernel reports PINT_E_RANGE_RETRY and the host re-runs the build with the
//    guarded variant (exponent check on the chain, IEEE __ddiv_rn outside [2^-960, 2^997]).
//  * A CTA holds the ceil((n+1)/32) warps of one slice (or one warp when n is large), lane =
//    trajectory: k < n runs from e_k, k == n is the forced run from 0 (c). The step's record is
//    staged once per CTA into shared memory one step ahead (cp.async) and read as broadcasts;
//    the first kRegRows rows of every column live in registers, the rest lane-interleaved in
//    shared memory (conflict-free). The forcing increment h*b_i is precomputed in the record, so
//    the forced lane costs one exact fma(f, hb_i, x) per row (f = 1 there, 0 on basis lanes) and
//    the slice's warps stay balanced. Rows leave as coalesced 256 B stores into the row-major
//    augmented map [G | c].
//
// Roofline: FP64 pipe. Algorithmic flops per slice-step: (n+1)(5n-4) + 5n (bench.py).

#include "pint_internal.cuh"

namespace {

using pint_dev::record_failure;

constexpr int kRegRows = 64;  // rows of each basis column held in registers (n >= kRegRows + 2)

__host__ __device__ constexpr long long even(long long x) { return (x + 1) & ~1ll; }

// doubles needed for the records of N slices x S steps x n rows
__host__ __device__ constexpr long long records_doubles(long long n, long long N, long long S) {
    return even(3 * S * N) + 4 * S * n * N;
}

struct RecView {
    const double* negr;  // [S][N]
    const double* fa;
    const double* fb;
    const double2* pr;   // [S][n][N]
    const double* cc;    // [S][n][N]
    const double* hb;    // [S][n][N]: the forcing increment h * heat_forcing(x_i, t)
    long long N;
    int n;
    __device__ __forceinline__ long long hdr(long long s, long long j) const { return s * N + j; }
    __device__ __forceinline__ long long row(long long s, int i, long long j) const { return (s * n + i) * N + j; }
};

__host__ __device__ inline RecView rec_view(const double* base, int n, long long N, long long S) {
    RecView v;
    v.negr = base;
    v.fa = base + S * N;
    v.fb = base + 2 * S * N;
    v.pr = reinterpret_cast<const double2*>(base + even(3 * S * N));
    v.cc = base + even(3 * S * N) + 2 * S * n * N;
    v.hb = base + even(3 * S * N) + 3 * S * n * N;
    v.N = N;
    v.n = n;
    return v;
}

// Thread (s, j): step s of slice j — the Thomas forward pivots of tridiag(-r, 1+2r, -r)
// (linalg.cpp:80-90, with sub = sup = -r, diag = 1 + 2r as solve_implicit builds them), and the
// forcing increment h * b_i with b_i = fa*s_i + fb*s_i = heat_forcing(x_i, t) (pde_problems.cpp:
// 26-29, 91-94), rounded exactly as `state[i] += dt_step * b[i]` consumes it.
__global__ void heat_record_kernel(int n, long long N, long long S, const int64_t* __restrict__ step_off,
                                   const double* __restrict__ slice_dt, const double* __restrict__ r_tab,
                                   const double* __restrict__ fa, const double* __restrict__ fb,
                                   const double* __restrict__ sx, double* __restrict__ rec, FailRec* fail) {
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= S * N) return;
    const long long s = t / N, j = t - s * N;
    const long long q = step_off[j] + s;
    if (q >= step_off[j + 1]) return;  // slice j has fewer steps
    const RecView V = rec_view(rec, n, N, S);
    double* negr_out = const_cast<double*>(V.negr);
    double* fa_out = const_cast<double*>(V.fa);
    double* fb_out = const_cast<double*>(V.fb);
    double2* pr_out = const_cast<double2*>(V.pr);
    double* cc_out = const_cast<double*>(V.cc);
    const double r = r_tab[q];
    const double negr = -r;                                  // pde_problems.cpp:55
    const double diag = __dadd_rn(1.0, __dmul_rn(2.0, r));   // 1.0 + 2.0 * r
    negr_out[V.hdr(s, j)] = negr;
    fa_out[V.hdr(s, j)] = fa[q];
    fb_out[V.hdr(s, j)] = fb[q];
    double p = diag;  // pivot = diag[0]; c[0] = sup[0] / pivot (linalg.cpp:80-83)
    if (p == 0.0) record_failure(fail, q, PINT_E_SINGULAR, 0.0);
    double c = (n > 1) ? __ddiv_rn(negr, p) : 0.0;
    pr_out[V.row(s, 0, j)] = make_double2(p, __drcp_rn(p));
    cc_out[V.row(s, 0, j)] = c;
    for (int i = 1; i < n; ++i) {  // pivot = diag - sub*c[i-1]; c[i] = sup / pivot (:84-88)
        p = __dsub_rn(diag, __dmul_rn(negr, c));
        if (p == 0.0) record_failure(fail, q, PINT_E_SINGULAR, static_cast<double>(i));
        c = (i < n - 1) ? __ddiv_rn(negr, p) : 0.0;
        pr_out[V.row(s, i, j)] = make_double2(p, __drcp_rn(p));
        cc_out[V.row(s, i, j)] = c;
    }
    double* hb_out = const_cast<double*>(V.hb);
    const double h = slice_dt[j], fq = fa[q], gq = fb[q];
    for (int i = 0; i < n; ++i) {
        const double si = sx[i];
        hb_out[V.row(s, i, j)] = __dmul_rn(h, __dadd_rn(__dmul_rn(fq, si), __dmul_rn(gq, si)));
    }
}

__device__ __forceinline__ double div_fast(double x, double2 pr) {
    const double q0 = __dmul_rn(x, pr.y);
    const double rem = __fma_rn(-pr.x, q0, x);
    return __fma_rn(rem, pr.y, q0);
}

__device__ __forceinline__ bool out_of_range(double x) {
    // |x| bits of the high word, window test on the biased exponent: true for zero, subnormal,
    // |x| < 2^-960, |x| >= 2^998, inf and nan (LOP3 + IADD + ISETP)
    const unsigned a = static_cast<unsigned>(__double2hiint(x)) & 0x7fffffffu;
    return a - (63u << 20) > ((2021u - 63u) << 20) - 1u;
}

__device__ __forceinline__ double div_guarded(double x, double2 pr) {
    return out_of_range(x) ? __ddiv_rn(x, pr.x) : div_fast(x, pr);
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}


struct BuildPlan {
    int n;
    int N;
    long long S;        // max steps per slice (record layout)
    int wps;            // warps (= CTAs) per slice = ceil((n+1)/32): n basis columns + the forced column
    const double* rec;
    const int64_t* step_off;
    double* maps;
    long long ldm;
    unsigned long long* per_slice_ns;
    FailRec* fail;
};

// Staged record in shared memory: [negr, pad] | (p_i, rcp_i) x n | c_i x n | h b_i x n
__host__ __device__ constexpr long long staged_doubles(long long n) { return 2 + 4 * n; }

// One backward-Euler step of one column: forcing increment (mixed warp only), forward
// elimination (linalg.cpp:84-90), back substitution (linalg.cpp:91). Rows [0, RR) in reg[], the
// rest at st[32*(i-RR)]. f is 1 on the forced lane and 0 elsewhere: fma(f, hb, x) is exactly
// x + h*b (pde_problems.cpp:93) there and exactly x on every basis lane.
// The shared-memory rows are software-pipelined two rows ahead: every load a row needs is issued
// before the stores of the rows in front of it (the compiler cannot hoist a shared load above a
// shared store it cannot disambiguate), so only the FP64 chain itself is on the critical path.
template <int RR, bool kMixed, bool kGuard>
__device__ __forceinline__ void column_step(double (&reg)[RR > 0 ? RR : 1], double* st, const double* R, int n,
                                            double f, bool forced_lane, bool& bad) {
    const double negr = R[0];
    const double2* PR = reinterpret_cast<const double2*>(R + 2);
    const double* CC = R + 2 + 2 * n;
    const double* HB = R + 2 + 3 * n;
    auto divide = [&](double num, double2 pr) {
        if (kMixed && !kGuard) bad |= forced_lane && out_of_range(num);
        return (kMixed && kGuard) ? div_guarded(num, pr) : div_fast(num, pr);
    };
    double d = 0.0;
#pragma unroll
    for (int i = 0; i < RR; ++i) {
        const double x = kMixed ? __fma_rn(f, HB[i], reg[i]) : reg[i];
        d = divide((i == 0) ? x : __dsub_rn(x, __dmul_rn(negr, d)), PR[i]);
        reg[i] = d;
    }
    double dm1 = d;  // q_{i-1} when the forward pass ends: the first back row reads it from here
    {
        const int last = n - 1 - RR;  // last shared row (>= 0: n > RR)
        double2 p0 = PR[RR], p1 = PR[RR + min(1, last)];
        double x0 = st[0], x1 = st[32 * min(1, last)];
        double h0 = kMixed ? HB[RR] : 0.0, h1 = kMixed ? HB[RR + min(1, last)] : 0.0;
#pragma unroll 4
        for (int r = 0; r <= last; ++r) {
            const int r2 = min(r + 2, last);
            const double2 p2 = PR[RR + r2];
            const double x2 = st[32 * r2];
            const double h2 = kMixed ? HB[RR + r2] : 0.0;
            const double x = kMixed ? __fma_rn(f, h0, x0) : x0;
            dm1 = d;
            d = divide((RR == 0 && r == 0) ? x : __dsub_rn(x, __dmul_rn(negr, d)), p0);
            st[32 * r] = d;
            p0 = p1, p1 = p2, x0 = x1, x1 = x2, h0 = h1, h1 = h2;
        }
    }
    double c0 = 0.0, c1 = 0.0;  // CC[RR-1], CC[RR-2] once the shared rows are done
    if (n - 2 >= RR) {
        const int top = n - 2 - RR;  // first shared row of the back pass
        double y0 = dm1, y1 = st[32 * max(top - 1, 0)];
        c0 = CC[n - 2];
        c1 = CC[max(n - 3, 0)];
#pragma unroll 4
        for (int r = top; r >= 0; --r) {
            const double y2 = st[32 * max(r - 2, 0)];
            const double c2 = CC[max(RR + r - 2, 0)];
            d = __dsub_rn(y0, __dmul_rn(c0, d));
            st[32 * r] = d;
            y0 = y1, y1 = y2, c0 = c1, c1 = c2;
        }
    } else if (RR > 0) {
        c0 = CC[RR - 1];
        c1 = CC[max(RR - 2, 0)];
    }
#pragma unroll
    for (int i = RR - 1; i >= 0; --i) {
        const double c = (i == RR - 1) ? c0 : (i == RR - 2) ? c1 : CC[i];
        d = __dsub_rn(reg[i], __dmul_rn(c, d));
        reg[i] = d;
    }
}

// Staged record of one step: [negr, pad] | (p_i, rcp_i) x n | c_i x n | h b_i x n, gathered by the
// warp's own lanes with cp.async (16-/8-byte chunks of the slice-minor records).
__device__ __forceinline__ void stage_step(double* dst, const RecView& V, long long s, long long j, bool with_hb,
                                           int lane) {
    const int n = V.n;
    double2* pr = reinterpret_cast<double2*>(dst + 2);
    double* cc = dst + 2 + 2 * n;
    double* hb = dst + 2 + 3 * n;
    const int chunks = (with_hb ? 3 * n : 2 * n) + 1;
    for (int c = lane; c < chunks; c += 32) {
        if (c < n) {
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(pr + c)), "l"(V.pr + V.row(s, c, j)));
        } else if (c < 2 * n) {
            const int i = c - n;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(cc + i)), "l"(V.cc + V.row(s, i, j)));
        } else if (c == chunks - 1) {
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(V.negr + V.hdr(s, j)));
        } else {
            const int i = c - 2 * n;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(hb + i)), "l"(V.hb + V.row(s, i, j)));
        }
    }
    asm volatile("cp.async.commit_group;\n" ::);
}

// CTA = ONE warp: warp g of slice blockIdx.x / wps; lane = trajectory k = 32g + lane (k < n: basis
// e_k, k == n: the forced run from 0, k > n: idle). Warps share nothing — each stages its own copy
// of the step record (double buffer, one step ahead) — so no CTA barrier couples a slice's warps
// and the scheduler packs the single-warp CTAs over all SMs.
// Dynamic smem: staged[2][SD] | state[(n-RR)*32]
template <int RR, bool kGuard>
__global__ void __maxnreg__(224) heat_build_kernel(BuildPlan P) {
    extern __shared__ __align__(16) double smem[];
    const unsigned long long t_start = pint_dev::globaltimer();
    const int n = P.n;
    const int lane = threadIdx.x;
    const int slice = blockIdx.x / P.wps;
    const int g = blockIdx.x - slice * P.wps;
    const long long SD = staged_doubles(n);
    double* buf = smem;
    double* st = smem + 2 * SD + lane;
    const int k = g * 32 + lane;
    const bool forced_lane = (k == n);
    const bool mixed = (g == n / 32);  // the warp holding column n
    const double f = forced_lane ? 1.0 : 0.0;
    const long long steps = P.step_off[slice + 1] - P.step_off[slice];
    const RecView V = rec_view(P.rec, n, P.N, P.S);

    if (steps > 0) stage_step(buf, V, 0, slice, mixed, lane);
    double reg[RR > 0 ? RR : 1];
#pragma unroll
    for (int i = 0; i < RR; ++i) reg[i] = (i == k) ? 1.0 : 0.0;  // e_k (all zero for k >= n)
    for (int i = RR; i < n; ++i) st[(i - RR) * 32] = (i == k) ? 1.0 : 0.0;

    bool bad = false;
    int cur = 0;
    for (long long s = 0; s < steps; ++s) {
        if (s + 1 < steps) {
            stage_step(buf + (cur ^ 1) * SD, V, s + 1, slice, mixed, lane);
            asm volatile("cp.async.wait_group 1;\n" ::);
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::);
        }
        __syncwarp();  // step s's record visible to every lane
        if (mixed) column_step<RR, true, kGuard>(reg, st, buf + cur * SD, n, f, forced_lane, bad);
        else column_step<RR, false, kGuard>(reg, st, buf + cur * SD, n, f, forced_lane, bad);
        __syncwarp();  // buffer `cur` is refilled next iteration
        cur ^= 1;
    }
    if (k <= n) {
        double* gp = P.maps + static_cast<long long>(slice) * n * P.ldm + k;
#pragma unroll
        for (int i = 0; i < RR; ++i) gp[i * P.ldm] = reg[i];
        for (int i = RR; i < n; ++i) gp[i * P.ldm] = st[(i - RR) * 32];
    }
    if (bad) record_failure(P.fail, slice, PINT_E_RANGE_RETRY, static_cast<double>(n));
    if (P.per_slice_ns && lane == 0) atomicAdd(P.per_slice_ns + slice, pint_dev::globaltimer() - t_start);
}

// ---- integrate: K caller columns of one slice (records with N = 1), guarded division ----------
struct IntegratePlan {
    int n;
    long long K, s0, steps, S;
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
    double* sx = smem;
    double* st = smem + even(n) + lane;
    for (int i = lane; i < n; i += 32) sx[i] = P.sx[i];
    for (int i = 0; i < n; ++i) st[i * 32] = active ? P.y[col * n + i] : 0.0;
    __syncwarp();
    const RecView V = rec_view(P.rec, n, 1, P.S);
    const bool forcing = P.with_forcing != 0;
    for (long long s = P.s0; s < P.s0 + P.steps; ++s) {
        const double negr = __ldg(V.negr + s);
        double d = 0.0;
        for (int i = 0; i < n; ++i) {
            double x = st[i * 32];
            if (forcing) x = __dadd_rn(x, __ldg(V.hb + V.row(s, i, 0)));  // state += h*b (pde_problems.cpp:93)
            const double num = (i == 0) ? x : __dsub_rn(x, __dmul_rn(negr, d));
            d = div_guarded(num, __ldg(V.pr + V.row(s, i, 0)));
            st[i * 32] = d;
        }
        for (int i = n - 2; i >= 0; --i) {
            d = __dsub_rn(st[i * 32], __dmul_rn(__ldg(V.cc + V.row(s, i, 0)), d));
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
    const size_t smem = sizeof(double) * (2 * staged_doubles(P.n) + static_cast<size_t>(P.n - RR) * 32);
    if (smem > 227 * 1024) return pint_set_error(ctx, PINT_E_INVALID, "heat_build: n too large for shared memory");
    auto kern = heat_build_kernel<RR, kGuard>;
    smem_attrs(kern, smem);
    kern<<<static_cast<unsigned>(static_cast<long long>(P.N) * P.wps), 32, smem, ctx->stream>>>(P);
    return pint_check_launch(ctx, "heat_build_kernel");
}

}  // namespace

int64_t heat_records_doubles(int64_t n, int64_t N, int64_t S) { return records_doubles(n, N, S); }

int launch_heat_factor(pint_ctx* ctx, int64_t n, int64_t N, int64_t S, const int64_t* step_off,
                       const double* slice_dt, const double* r, const double* fa, const double* fb,
                       const double* sx, double* records) {
    if (n < 1 || N < 0 || S < 0) return pint_set_error(ctx, PINT_E_INVALID, "heat_factor: bad sizes");
    if (N == 0 || S == 0) return PINT_OK;
    const long long threads = N * S;
    heat_record_kernel<<<static_cast<unsigned>((threads + 127) / 128), 128, 0, ctx->stream>>>(
        static_cast<int>(n), N, S, step_off, slice_dt, r, fa, fb, sx, records, ctx->d_fail);
    return pint_check_launch(ctx, "heat_record_kernel");
}

int launch_heat_build(pint_ctx* ctx, int64_t n, int64_t N, int64_t S, const int64_t* step_off,
                      const double* slice_dt, const double* records, const double* sx, double* maps,
                      unsigned long long* per_slice_ns, int guarded) {
    if (n < 1 || N < 0) return pint_set_error(ctx, PINT_E_INVALID, "heat_build: bad sizes");
    if (N == 0) return PINT_OK;
    if (n > (1 << 20) || N > (1 << 26)) return pint_set_error(ctx, PINT_E_INVALID, "heat_build: sizes out of range");
    (void)slice_dt;  // the per-slice step lives in the records (h*b) and step_off
    (void)sx;
    BuildPlan P{};
    P.n = static_cast<int>(n);
    P.N = static_cast<int>(N);
    P.S = S;
    P.wps = static_cast<int>((n + 1 + 31) / 32);
    P.rec = records;
    P.step_off = step_off;
    P.maps = maps;
    P.ldm = pint_affine_ldm(n);
    P.per_slice_ns = per_slice_ns;
    P.fail = ctx->d_fail;
    if (n >= kRegRows + 2)
        return guarded ? launch_build<kRegRows, true>(ctx, P) : launch_build<kRegRows, false>(ctx, P);
    return guarded ? launch_build<0, true>(ctx, P) : launch_build<0, false>(ctx, P);
}

int launch_heat_integrate(pint_ctx* ctx, int64_t n, int64_t K, int64_t S, int64_t s0, int64_t steps, double h,
                          int with_forcing, const double* records, const double* sx, double* y) {
    if (n < 1 || K < 0) return pint_set_error(ctx, PINT_E_INVALID, "heat_integrate: bad sizes");
    if (K == 0) return PINT_OK;
    IntegratePlan P{static_cast<int>(n), K, s0, steps, S, h, with_forcing, records, sx, y};
    const size_t smem = sizeof(double) * (static_cast<size_t>(n) * 32 + even(n));
    if (smem > 227 * 1024) return pint_set_error(ctx, PINT_E_INVALID, "heat_integrate: n too large");
    smem_attrs(heat_integrate_kernel, smem);
    heat_integrate_kernel<<<static_cast<unsigned>((K + 31) / 32), 32, smem, ctx->stream>>>(P);
    return pint_check_launch(ctx, "heat_integrate_kernel");
}
