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
//    so the record kernel (thread = (step, slice)) and the forcing warps (lane = slice) are
//    coalesced, and a basis CTA gathers its slice's column with 16-/8-byte cp.async chunks.
//  * x / p_i is q0 = x*rcp, rem = fma(-p, q0, x), q = fma(rem, rcp, q0) with rcp = RN(1/p_i):
//    Markstein's theorem makes q the correctly rounded quotient whenever no intermediate
//    under/overflows. Basis columns are entrywise non-negative and bounded (each step matrix is an
//    M-matrix, p_i >= 1, |c_i| < 1), so their quotients stay far from the subnormal range and run
//    unguarded. Forced columns are range-checked OFF the dependent chain (a sticky flag); if it
//    ever trips, the kernel reports PINT_E_RANGE_RETRY and the host re-runs the build with the
//    guarded variant (exponent check on the chain, IEEE __ddiv_rn outside [2^-960, 2^997]).
//  * Basis kernel: a CTA holds the ceil(n/32) warps of one slice (or one warp when n is large),
//    lane = trajectory e_k. The step's record is staged once per CTA into shared memory one step
//    ahead and read as broadcasts; the first kRegRows rows of every column live in registers, the
//    rest lane-interleaved in shared memory (conflict-free). Rows leave as coalesced 256 B stores
//    into the row-major augmented map [G | c].
//  * Forcing kernel (side stream, concurrent): one warp holds the c runs of 32 consecutive
//    slices (lane = slice) and streams its rows kD = 32 ahead through register rings.
//
// Roofline: FP64 pipe. Algorithmic flops per slice-step: (n+1)(5n-4) + 5n (bench.py).
#include "pint_internal.cuh"

namespace {

using pint_dev::record_failure;

constexpr int kRegRows = 64;  // rows of each basis column held in registers (n >= kRegRows + 2)
constexpr int kMaxCtaThreads = 32 * 8;
#ifndef PINT_FORCING_RING
#define PINT_FORCING_RING 16  // rows the forcing warps keep in flight from L2 (register ring)
#endif

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
    const unsigned e = (static_cast<unsigned>(__double2hiint(x)) >> 20) & 0x7ffu;
    return e - 63u > 1957u;  // zero, subnormal, |x| < 2^-960, |x| >= 2^998, inf/nan
}

__device__ __forceinline__ double div_guarded(double x, double2 pr) {
    return out_of_range(x) ? __ddiv_rn(x, pr.x) : div_fast(x, pr);
}

// Forcing (pde_problems.cpp:91-94) folded into the row update: x + h*(fa s + fb s), where
// heat_forcing(x_i, t) = fa*s + fb*s with fa = -sin t, fb = ((a pi) pi) cos t (pde_problems.cpp:26-29).
__device__ __forceinline__ double forced(double x, double h, double fa, double fb, double s) {
    return __dadd_rn(x, __dmul_rn(h, __dadd_rn(__dmul_rn(fa, s), __dmul_rn(fb, s))));
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];\n" ::"l"(p)); }

struct BuildPlan {
    int n;
    int N;
    long long S;        // max steps per slice (record layout)
    int wb;             // basis warps per slice = ceil(n/32)
    int warps_per_cta;  // wb (one CTA per slice) or 1
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

// ---- basis kernel -------------------------------------------------------------------------------
// Staged record in shared memory: [negr, pad] | (p_i, rcp_i) x n | c_i x n
__host__ __device__ constexpr long long staged_doubles(long long n) { return 2 + 3 * n + (n & 1); }

__device__ __forceinline__ void stage_step(double* dst, const RecView& V, long long s, long long j) {
    const int n = V.n;
    double2* pr = reinterpret_cast<double2*>(dst + 2);
    double* cc = dst + 2 + 2 * n;
    for (int c = threadIdx.x; c < 2 * n + 1; c += blockDim.x) {
        if (c < n) {
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(pr + c)), "l"(V.pr + V.row(s, c, j)));
        } else if (c < 2 * n) {
            const int i = c - n;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(cc + i)), "l"(V.cc + V.row(s, i, j)));
        } else {
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(V.negr + V.hdr(s, j)));
        }
    }
    asm volatile("cp.async.commit_group;\n" ::);
}

// One backward-Euler step of one basis column: forward elimination (linalg.cpp:84-90) and back
// substitution (linalg.cpp:91). Rows [0, RR) in reg[], the rest at st[32*(i-RR)].
template <int RR>
__device__ __forceinline__ void basis_step(double (&reg)[RR > 0 ? RR : 1], double* st, const double* R, int n) {
    const double negr = R[0];
    const double2* PR = reinterpret_cast<const double2*>(R + 2);
    const double* CC = R + 2 + 2 * n;
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

// CTA = warps [c*warps_per_cta, ...) of one slice, lane = basis column e_k.
// Dynamic smem: staged[2][SD] | state[warps_per_cta][(n - RR) * 32]
template <int RR>
__global__ void __launch_bounds__(kMaxCtaThreads) heat_basis_kernel(BuildPlan P) {
    extern __shared__ __align__(16) double smem[];
    const unsigned long long t_start = pint_dev::globaltimer();
    const int n = P.n;
    const int lane = threadIdx.x & 31, wcta = threadIdx.x >> 5;
    const int slice = blockIdx.x / P.ctas_per_slice;
    const int g = (blockIdx.x - slice * P.ctas_per_slice) * P.warps_per_cta + wcta;  // warp in slice
    const long long SD = staged_doubles(n);
    double* buf = smem;
    double* st = smem + 2 * SD + static_cast<long long>(wcta) * (n - RR) * 32 + lane;
    const int k = g * 32 + lane;
    const long long steps = P.step_off[slice + 1] - P.step_off[slice];
    const RecView V = rec_view(P.rec, n, P.N, P.S);

    if (steps > 0) stage_step(buf, V, 0, slice);
    double reg[RR > 0 ? RR : 1];
#pragma unroll
    for (int i = 0; i < RR; ++i) reg[i] = (i == k) ? 1.0 : 0.0;  // e_k
    for (int i = RR; i < n; ++i) st[(i - RR) * 32] = (i == k) ? 1.0 : 0.0;

    int cur = 0;
    for (long long s = 0; s < steps; ++s) {
        if (s + 1 < steps) {
            stage_step(buf + (cur ^ 1) * SD, V, s + 1, slice);
            asm volatile("cp.async.wait_group 1;\n" ::);
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::);
        }
        __syncthreads();  // step s's record visible to every warp
        basis_step<RR>(reg, st, buf + cur * SD, n);
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

// ---- forcing kernel -----------------------------------------------------------------------------
// One warp per CTA: the forced (c) runs of 32 consecutive slices, lane = slice. Row i of step s is
// one coalesced 512 B load across the warp; rows stream kD ahead through register rings and the
// next step's first rows are fetched during the current back substitution.
// Dynamic smem: state[n * 32]
template <bool kGuard>
__global__ void __launch_bounds__(32) heat_forcing_kernel(BuildPlan P) {
    constexpr int kD = PINT_FORCING_RING;
    extern __shared__ __align__(16) double smem[];
    const int n = P.n;
    const int lane = threadIdx.x;
    double* st = smem + lane;
    const int slice = blockIdx.x * 32 + lane;
    const bool active = slice < P.N;
    const int js = active ? slice : P.N - 1;  // clamp addresses of idle lanes
    const long long steps = active ? P.step_off[slice + 1] - P.step_off[slice] : 0;
    const long long max_steps = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(steps));
    const RecView V = rec_view(P.rec, n, P.N, P.S);
    for (int i = 0; i < n; ++i) st[i * 32] = 0.0;  // c = the forced run from the zero state
    __syncwarp();

    // Rings are refilled by UNCONDITIONAL loads from clamped rows: a predicated refill compiles to
    // load-into-temp + MOV, and the MOV waits for the data, which defeats the prefetch.
    const long long N = P.N;
    double2 pq[kD];
    double hq[kD];
    double cq[kD];
    double h_negr = 0.0;  // header of the step the rings were loaded for
    auto load_head = [&](long long s) {
        const long long base = V.row(s, 0, js);
#pragma unroll
        for (int u = 0; u < kD; ++u) {
            const long long off = base + static_cast<long long>(u < n ? u : n - 1) * N;
            pq[u] = __ldg(V.pr + off);
            hq[u] = __ldg(V.hb + off);
        }
        h_negr = __ldg(V.negr + V.hdr(s, js));
    };
    if (steps > 0) load_head(0);
    bool bad = false;
    for (long long s = 0; s < max_steps; ++s) {
        if (s >= steps) continue;
        const double negr = h_negr;
        const long long rbase = V.row(s, 0, js);  // row i at rbase + i*N
        const double* cbase = V.cc + rbase;
#pragma unroll
        for (int u = 0; u < kD; ++u) cq[u] = __ldg(cbase + static_cast<long long>(n - 2 - u > 0 ? n - 2 - u : 0) * N);
        // forward elimination, forcing increment added first (pde_problems.cpp:91-94, linalg.cpp:84-90)
        double d = 0.0;
        auto fwd_row = [&](int i, double2 pr, double hbi) {
            const double x = __dadd_rn(st[i * 32], hbi);
            const double num = (i == 0) ? x : __dsub_rn(x, __dmul_rn(negr, d));
            if (!kGuard) bad |= out_of_range(num);
            d = kGuard ? div_guarded(num, pr) : div_fast(num, pr);
            st[i * 32] = d;
        };
        // Each slot is consumed BEFORE it is refilled, so the refill targets the same register
        // (no temp + MOV at the back edge); the steady-state loop needs no address clamping.
        // The records were written long before (HBM-resident): while sweeping forward, pull this
        // step's multipliers into L2 for the back sweep (so the ring's loads hit L2).
        int i0 = 0;
        {
            const double2* pp = V.pr + rbase + static_cast<long long>(kD) * N;  // row i0 + kD
            const double* hp = V.hb + rbase + static_cast<long long>(kD) * N;
            const double* cpf = cbase + static_cast<long long>(n - 1) * N;
            for (; i0 + 2 * kD <= n; i0 += kD) {
#pragma unroll
                for (int u = 0; u < kD; ++u) {
                    fwd_row(i0 + u, pq[u], hq[u]);
                    pq[u] = __ldg(pp);
                    hq[u] = __ldg(hp);
                    prefetch_l2(cpf);
                    pp += N;
                    hp += N;
                    cpf -= N;
                }
            }
            for (int i = i0; i < n; ++i, cpf -= N) prefetch_l2(cpf);
        }
        for (; i0 < n; i0 += kD) {  // last one or two chunks: refills clamped to valid rows
#pragma unroll
            for (int u = 0; u < kD; ++u) {
                const int i = i0 + u;
                if (i < n) {
                    fwd_row(i, pq[u], hq[u]);
                    const long long off = rbase + static_cast<long long>(i + kD < n ? i + kD : i) * N;
                    pq[u] = __ldg(V.pr + off);
                    hq[u] = __ldg(V.hb + off);
                }
            }
        }
        if (s + 1 < steps) load_head(s + 1);  // hidden behind the back sweep
        // back substitution (linalg.cpp:91), multipliers kD rows ahead
        auto back_row = [&](int i, double c) {
            d = __dsub_rn(st[i * 32], __dmul_rn(c, d));
            st[i * 32] = d;
        };
        int t0 = 0;
        {
            // meanwhile pull the next step's pivots/increments (rows kD..) into L2
            const long long nb = V.row(s + 1 < steps ? s + 1 : s, kD < n ? kD : n - 1, js);
            const double2* npp = V.pr + nb;
            const double* nhp = V.hb + nb;
            const double* cp = cbase + static_cast<long long>(n - 2 - kD) * N;  // row n-2-kD
            for (; n - 2 - t0 - (2 * kD - 1) >= 0; t0 += kD) {
#pragma unroll
                for (int u = 0; u < kD; ++u) {
                    back_row(n - 2 - t0 - u, cq[u]);
                    cq[u] = __ldg(cp);
                    prefetch_l2(npp);
                    prefetch_l2(nhp);
                    cp -= N;
                    npp += N;
                    nhp += N;
                }
            }
        }
        for (; n - 2 - t0 >= 0; t0 += kD) {
#pragma unroll
            for (int u = 0; u < kD; ++u) {
                const int i = n - 2 - t0 - u;
                if (i >= 0) {
                    back_row(i, cq[u]);
                    cq[u] = __ldg(cbase + static_cast<long long>(i - kD >= 0 ? i - kD : 0) * N);
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
    // basis: one CTA per slice when two such CTAs fit an SM, else one CTA per warp
    const size_t state_warp = sizeof(double) * static_cast<size_t>(P.n - RR) * 32;
    const size_t staged = sizeof(double) * 2 * staged_doubles(P.n);
    P.warps_per_cta = (P.wb <= kMaxCtaThreads / 32 && staged + state_warp * P.wb <= 112 * 1024) ? P.wb : 1;
    P.ctas_per_slice = P.wb / P.warps_per_cta;
    const size_t smem_b = staged + state_warp * P.warps_per_cta;
    const size_t smem_f = sizeof(double) * static_cast<size_t>(P.n) * 32;
    if (smem_b > 227 * 1024 || smem_f > 227 * 1024)
        return pint_set_error(ctx, PINT_E_INVALID, "heat_build: n too large for shared memory");
    auto kb = heat_basis_kernel<RR>;
    auto kf = heat_forcing_kernel<kGuard>;
    smem_attrs(kb, smem_b);
    smem_attrs(kf, smem_f);
    // fork: forcing runs on the side stream, overlapping the basis kernel; join before returning
    cudaEventRecord(ctx->ev_fork, ctx->stream);
    cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0);
    kf<<<static_cast<unsigned>((P.N + 31) / 32), 32, smem_f, ctx->side>>>(P);
    if (const int rc = pint_check_launch(ctx, "heat_forcing_kernel")) return rc;
    kb<<<static_cast<unsigned>(static_cast<long long>(P.N) * P.ctas_per_slice), 32 * P.warps_per_cta, smem_b,
         ctx->stream>>>(P);
    if (const int rc = pint_check_launch(ctx, "heat_basis_kernel")) return rc;
    cudaEventRecord(ctx->ev_join, ctx->side);
    cudaStreamWaitEvent(ctx->stream, ctx->ev_join, 0);
    return PINT_OK;
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
    BuildPlan P{};
    P.n = static_cast<int>(n);
    P.N = static_cast<int>(N);
    P.S = S;
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
