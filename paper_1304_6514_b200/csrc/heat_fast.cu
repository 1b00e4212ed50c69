// K3f — heat slice maps, TOLERANCE build (<= 1e-12 relative to the reference; north_star allows
// it for trajectory end states and the composed final state). Same maps as heat.cu's bit-exact
// build — build_affine_propagator (nievergelt.cpp:53-66) -> make_heat_problem's closure
// (pde_problems.cpp:86-98) -> thomas_solve (linalg.cpp:77-93) for e_0..e_{n-1} and the forced
// run from 0 — with a different operation order and a much shorter dependent chain.
//
// Why a second build: the exact build must reproduce the reference's roundings, so every row of a
// column is a chain of 7 dependent FP64 ops (sub*d, x - ., the Markstein quotient, c*d, d - .),
// and a column's n rows of state cannot stay in registers at n = 512 (shared/tensor memory at
// 64-128 B/clk is then the limit). Here:
//  * Forward elimination of a step is d_i = g_i + u_i d_{i-1} with g_i = x_i / p_i and
//    u_i = r / p_i precomputed per (slice, step): ONE FMA on the chain per row (the product
//    x_i rcp_i is off the chain). Back substitution x_i = d_i + u_i x_{i+1}: one FMA.
//  * A column is split into P partitions of R rows (R <= 64), one thread each, all rows in
//    registers. The partitions run their recurrences with zero carry-in; the carries
//    D_p = d_{a_p - 1} and E_p = x_{b_p + 1} follow from log-depth shuffle scans across the P lanes
//    of the column, and the local results are fixed up with right-hand-side-independent
//    "spike" vectors precomputed per (slice, step): x_i = x~_i + D_p psi_i + E_p sigma_i, where
//    pi_i = prod_{k=a..i} u_k, psi_i = pi_i + u_i psi_{i+1}, sigma_i = prod_{k=i..b} u_k.
//    5 FP64 instructions per (row, column, step) for the reference's 5 algorithmic flops.
//  * heat_fast_record_kernel builds the per-(slice, step) coefficients with one warp per record:
//    each lane owns NP/32 consecutive rows of one partition, starts its pivot recurrence
//    u_i = r / (diag - r u_{i-1}) from the closed form u_{i0-1} = M^{i0}(0) of the Mobius map
//    M = [[0, r], [-r, diag]] (binary powering), and the partition products / psi come from
//    shuffle scans — so the lanes write whole 128-byte lines.
//
// Record (slice j, step s), doubles, row i = p R + t stored at [t][p] (a warp's broadcast loads of
// one t across its P partitions are one contiguous, conflict-free wavefront):
//   A [R][P] (rcp_i, u_i) | B [R][P] (psi_i, sigma_i) | C [P] pi_end (padded to 16)   = BLK
//   and separately H [R][P] h b_i rcp_i (the forced column's increment, pde_problems.cpp:93).
// Rows i >= n are identity padding (rcp 1, u 0), as are steps beyond a slice's own count.
//
// Roofline: FP64 pipe. 5 instructions per (row, column, step), 2 of them on the dependent chain;
// algorithmic flops as the exact build ((n+1)(5n-4) + 5n per slice-step, bench.py).
#include <algorithm>
#include <cstdlib>

#include "pint_internal.cuh"

namespace {

using namespace pint_async;

constexpr unsigned kFull = 0xffffffffu;

// Kogge-Stone multipliers of the two carry scans, [level][partition] (levels <= 5, P <= 32)
constexpr int kScanLevelStride = 32;
constexpr int kScanTab = 5 * kScanLevelStride;
__host__ __device__ constexpr long long fast_blk(long long NP) { return 4 * NP + 2 * kScanTab; }

// Partition shape for n: R rows per partition, P (a power of two <= 32) partitions per column,
// C = 64 / R columns per thread (64 rows of state in registers: 128 of the 255), so that NP = P R
// is a multiple of 32 (the record kernel's lanes). Shorter partitions give each thread more
// independent chains and amortise every coefficient load over more columns (C), at the price of a
// deeper carry scan: R = 16 (C = 4) up to n = 512 (P = 32 above n = 256: one column per warp; the
// R = 32, C = 2 shape spilled and ran 3.5% slower at config 4), then R = 32 (C = 2, only with
// PINT_FAST_P32=0) and R = 48 (C = 1, n <= 768).
struct FastShape {
    int P = 0, R = 0;
    bool ok() const { return P > 0; }
    int NP() const { return P * R; }
};
FastShape fast_shape(long long n) {
    static const int p32 = [] {  // PINT_FAST_P32=1: 32 partitions of 16 rows up to n = 512 (experiment)
        const char* e = std::getenv("PINT_FAST_P32");
        return e ? std::atoi(e) : 1;
    }();
    FastShape f;
    for (int R : {16, 32, 48})
        for (int P = 2; P <= (R == 16 && p32 ? 32 : 16); P *= 2)
            if (static_cast<long long>(P) * R >= n) {
                f.P = P;
                f.R = R;
                return f;
            }
    return f;
}

// ---- records -------------------------------------------------------------------------------------
struct FastRecPlan {
    int n, P, R;
    long long N, S;
    const int64_t* step_off;
    const double* slice_dt;
    const double* r;
    const double* fa;
    const double* fb;
    const double* sx;
    double* rec;   // [N][S][BLK]
    double* hrec;  // [N][S][NP]
    FailRec* fail;
};

// u_{e-1} = M^e(0) for M = [[0, r], [-r, diag]] acting on u as (0 u + r) / (-r u + diag): the pivot
// recurrence u_i = r / (diag - r u_{i-1}), u_{-1} = 0, jumped e rows ahead. Binary powering with a
// rescale after every product (the Mobius value is scale-free).
__device__ double mobius_start(double r, double diag, int e) {
    double a = 1.0, b = 0.0, c = 0.0, d = 1.0;        // result
    double A = 0.0, B = r, Cc = -r, D = diag;         // M^(2^k)
    auto rescale = [](double& w, double& x, double& y, double& z) {
        const double m = fmax(fmax(fabs(w), fabs(x)), fmax(fabs(y), fabs(z)));
        const double s = 1.0 / m;
        w *= s, x *= s, y *= s, z *= s;
    };
    while (e) {
        if (e & 1) {
            const double na = a * A + b * Cc, nb = a * B + b * D, nc = c * A + d * Cc, nd = c * B + d * D;
            a = na, b = nb, c = nc, d = nd;
            rescale(a, b, c, d);
        }
        e >>= 1;
        if (e) {
            const double nA = A * A + B * Cc, nB = A * B + B * D, nC = Cc * A + D * Cc, nD = Cc * B + D * D;
            A = nA, B = nB, Cc = nC, D = nD;
            rescale(A, B, Cc, D);
        }
    }
    return b / d;
}

// One warp per (slice, step) record; lane = c P + p owns rows t in [c kM, c kM + kM) of partition p
// (kM = NP / 32, 32 / P chunks per partition).
template <int kM>
__global__ void __launch_bounds__(128) heat_fast_record_kernel(const FastRecPlan Q) {
    const long long gw = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (gw >= Q.N * Q.S) return;  // (whole warps)
    const int lane = threadIdx.x & 31;
    const int P = Q.P, R = Q.R, NP = P * R, n = Q.n;
    const int CPP = 32 / P;  // chunks per partition
    const int p = lane % P, c = lane / P;
    const long long j = gw / Q.S, s = gw - j * Q.S;
    const long long steps = Q.step_off[j + 1] - Q.step_off[j];
    const bool idn = s >= steps;  // identity padding step
    const long long q = idn ? 0 : Q.step_off[j] + s;
    const double r = idn ? 0.0 : Q.r[q];
    const double h = Q.slice_dt[j], fq = idn ? 0.0 : Q.fa[q], gq = idn ? 0.0 : Q.fb[q];
    const double diag = 1.0 + 2.0 * r;  // solve_implicit's diagonal (pde_problems.cpp:55)
    const int i0 = p * R + c * kM;
    double up = (!idn && i0 > 0 && i0 < n) ? mobius_start(r, diag, i0) : 0.0;
    double rp[kM], u[kM], hr[kM];
#pragma unroll
    for (int k = 0; k < kM; ++k) {
        const int i = i0 + k;
        if (!idn && i < n) {
            const double pv = (i == 0) ? diag : diag - r * up;
            if (pv == 0.0) pint_dev::record_failure(Q.fail, q, PINT_E_SINGULAR, static_cast<double>(i));  // linalg.cpp:82,87
            rp[k] = 1.0 / pv;
            u[k] = r * rp[k];
            const double si = Q.sx[i];
            hr[k] = (h * (fq * si + gq * si)) * rp[k];  // h b_i / p_i (pde_problems.cpp:91-94)
            up = u[k];
        } else {
            rp[k] = 1.0, u[k] = 0.0, hr[k] = 0.0;
        }
    }
    // pi: prefix products within the partition (local prefix x exclusive prefix over chunks c)
    double pl[kM], sl[kM];
    double acc = 1.0;
#pragma unroll
    for (int k = 0; k < kM; ++k) pl[k] = acc = acc * u[k];
    const double T = acc;  // this chunk's product of u
    acc = 1.0;
#pragma unroll
    for (int k = kM - 1; k >= 0; --k) sl[k] = acc = acc * u[k];
    double inc = T, incs = T;
    for (int o = 1; o < CPP; o <<= 1) {
        const double a = __shfl_up_sync(kFull, inc, o * P);
        const double b = __shfl_down_sync(kFull, incs, o * P);
        if (c >= o) inc *= a;
        if (c + o < CPP) incs *= b;
    }
    double ex = __shfl_up_sync(kFull, inc, P), exs = __shfl_down_sync(kFull, incs, P);
    if (c == 0) ex = 1.0;
    if (c == CPP - 1) exs = 1.0;
    double pi[kM];
#pragma unroll
    for (int k = 0; k < kM; ++k) pi[k] = ex * pl[k];
    // psi = pi + u psi(next), zero beyond the partition: local with zero carry, then the carries
    double ps[kM];
    acc = 0.0;
#pragma unroll
    for (int k = kM - 1; k >= 0; --k) ps[k] = acc = __fma_rn(u[k], acc, pi[k]);
    double v = ps[0], a = T;
    for (int o = 1; o < CPP; o <<= 1) {
        const double vo = __shfl_down_sync(kFull, v, o * P), ao = __shfl_down_sync(kFull, a, o * P);
        if (c + o < CPP) {
            v = __fma_rn(a, vo, v);
            a *= ao;
        }
    }
    double nxt = __shfl_down_sync(kFull, v, P);
    if (c == CPP - 1) nxt = 0.0;
    double* blk = Q.rec + gw * fast_blk(NP);
    double2* A2 = reinterpret_cast<double2*>(blk);
    double2* B2 = reinterpret_cast<double2*>(blk + 2 * NP);
    double* H = Q.hrec + gw * NP;
#pragma unroll
    for (int k = 0; k < kM; ++k) {
        const int t = c * kM + k;
        A2[t * P + p] = make_double2(rp[k], u[k]);
        // (partition 0 has no carry from above and the last none from below: psi / sigma stored as 0 there,
        // so the build multiplies whatever its shuffles return there by 0 instead of selecting)
        B2[t * P + p] = make_double2(p == 0 ? 0.0 : __fma_rn(sl[k], nxt, ps[k]), p == P - 1 ? 0.0 : sl[k] * exs);
        H[t * P + p] = hr[k];
    }
    // the carry scans' multipliers (RHS-independent): forward, element p = (pi_end(p), d~_end) scanned
    // upward; back, element p = (sigma_0(p) = pi_end(p), x_a) scanned downward. Level l multiplies
    // the partner's value by the product of pi_end over the 2^l partitions ending (starting) at p.
    // (lanes c = CPP - 1 hold pi_end; the rest compute alongside and write nothing)
    double af = pi[kM - 1], ab = af;
    for (int l = 0; (1 << l) < P; ++l) {
        const int o = 1 << l;
        const double fo = __shfl_up_sync(kFull, af, o), bo = __shfl_down_sync(kFull, ab, o);
        if (c == CPP - 1) {  // (0 where the partner partition does not exist: no select in the build)
            blk[4 * NP + l * kScanLevelStride + p] = p >= o ? af : 0.0;
            blk[4 * NP + kScanTab + l * kScanLevelStride + p] = p + o < P ? ab : 0.0;
        }
        if (p >= o) af *= fo;
        if (p + o < P) ab *= bo;
    }
}

// ---- build ---------------------------------------------------------------------------------------
struct FastPlan {
    int n;
    long long N, S;
    int NS;          // slice slots staged per buffer
    double* maps;
    long long ldm;
    const double* rec;
    const double* hrec;
    int* ready;  // (may be null) per-slice count of warps whose columns of the map are stored
    unsigned long long* span;  // (with ready) {first warp start, last warp end} globaltimer
    long long wps = 0;         // warps per slice: ceil((n + 1) / CPW), or padded to whole CTAs
};

// records staged ahead: step s + ST is fetched when step s is done (and step s + ST + 1 pulled into
// L2 meanwhile); ST = 4 where 4 stages leave room for 2 CTAs per SM (small records: C2), else 2
constexpr int kFastStagesMax = 4;

// C columns per thread share every coefficient load (one LDS serves 5 C FP64 instructions: the
// shared-memory path stays below the FP64 pipe) and give each thread C independent chains.
template <int R>
struct FastCfg {
    static constexpr int C = R <= 16 ? 4 : R <= 32 ? 2 : 1;
    // warps per CTA: single-warp CTAs stage their own records and never wait for a slower warp
    // (C2: 0.78 vs 0.88 ms with 4-warp CTAs); at R = 32 (n = 512: 21.5 KB a staged step) 4-warp
    // CTAs share one staged copy, or the copies would not fit 8 warps per SM
    static constexpr int W = R <= 16 ? 1 : 4;  // (P = 32, R = 16: see fast_warps)
    static constexpr int kMinCtas = 2;  // (x 4 / W CTAs: 8 warps per SM, <= 255 registers)
};

// One step of C column partitions (thread: partition p of C columns, rows in x[c][]); St = the
// slice's staged record, Hs its h b / p column (kF: some column of this warp is a forced run;
// fmask bit c set where this thread's column c is).
template <int P, int R, int C, bool kF>
__device__ __forceinline__ void fast_step(double (&x)[C][R], const double* St, const double* Hs, int p,
                                          unsigned fmask) {
    constexpr int NP = P * R;
    const double2* A = reinterpret_cast<const double2*>(St) + p;
    const double2* B = reinterpret_cast<const double2*>(St + 2 * NP) + p;
    const double* Hp = Hs + p;
    double d[C];
#pragma unroll
    for (int c = 0; c < C; ++c) d[c] = 0.0;
#pragma unroll
    for (int t = 0; t < R; ++t) {  // forward elimination: d = x rcp + u d (one FMA on the chain)
        const double2 a = A[t * P];
        const double h = kF ? Hp[t * P] : 0.0;
#pragma unroll
        for (int c = 0; c < C; ++c) {
            const double g = kF ? __fma_rn(x[c][t], a.x, ((fmask >> c) & 1u) ? h : 0.0) : __dmul_rn(x[c][t], a.x);
            d[c] = __fma_rn(a.y, d[c], g);
            x[c][t] = d[c];
        }
    }
    double D[C], E[C];
    constexpr int L = P >= 32 ? 5 : P >= 16 ? 4 : P >= 8 ? 3 : P >= 4 ? 2 : P >= 2 ? 1 : 0;
    if constexpr (P > 1) {  // carry-in of the forward recurrence: upward scan of (pi_end, d~_end)
        const double* FS = St + 4 * NP + p;
#pragma unroll
        for (int l = 0; l < L; ++l) {
            const double m = FS[l * kScanLevelStride];
#pragma unroll
            for (int c = 0; c < C; ++c) {  // (m = 0 where p < 2^l: the lane's own value, times 0)
                const double vo = __shfl_up_sync(kFull, d[c], 1 << l, P);
                d[c] = __fma_rn(m, vo, d[c]);
            }
        }
#pragma unroll
        for (int c = 0; c < C; ++c) D[c] = __shfl_up_sync(kFull, d[c], 1, P);  // (p = 0: psi = 0 absorbs it)
    }
    double xn[C];
#pragma unroll
    for (int c = 0; c < C; ++c) xn[c] = 0.0;
#pragma unroll
    for (int t = R - 1; t >= 0; --t) {  // back substitution: x = d + u x(next)
        const double u = A[t * P].y;
#pragma unroll
        for (int c = 0; c < C; ++c) {
            xn[c] = __fma_rn(u, xn[c], x[c][t]);
            x[c][t] = xn[c];
        }
    }
    if constexpr (P > 1) {  // carry-in from below: downward scan of (sigma_0, x~_0 + D psi_0)
        const double* BS = St + 4 * NP + kScanTab + p;
        const double psi0 = B[0].x;
        double v[C];
#pragma unroll
        for (int c = 0; c < C; ++c) v[c] = __fma_rn(D[c], psi0, x[c][0]);
#pragma unroll
        for (int l = 0; l < L; ++l) {
            const double m = BS[l * kScanLevelStride];
#pragma unroll
            for (int c = 0; c < C; ++c) {
                const double vo = __shfl_down_sync(kFull, v[c], 1 << l, P);
                v[c] = __fma_rn(m, vo, v[c]);
            }
        }
#pragma unroll
        for (int c = 0; c < C; ++c) E[c] = __shfl_down_sync(kFull, v[c], 1, P);  // (p = P - 1: sigma = 0)
#pragma unroll
        for (int t = 0; t < R; ++t) {  // x = x~ + D psi + E sigma
            const double2 b = B[t * P];
#pragma unroll
            for (int c = 0; c < C; ++c) x[c][t] = __fma_rn(b.y, E[c], __fma_rn(b.x, D[c], x[c][t]));
        }
    }
}

// CTA = W warps; warp w runs slice j = w / wps, columns wi * CPW + [0, CPW) (wi = w % wps,
// wps = ceil((n + 1) / CPW); column n is the forced run, columns > n idle): lane = (column group
// cg, partition p), C columns per lane at stride G. A warp's columns lie in ONE slice; a CTA's
// warps in ns <= W slices, whose records (+ the forced increments, for the warps that hold a
// forced column) are staged per step by bulk copies (double-buffered; the last warp done with a
// buffer refills it).
template <int P, int R, int ST, int W>
__global__ void __launch_bounds__(32 * W, FastCfg<R>::kMinCtas * 4 / W) heat_fast_build_kernel(const FastPlan Q) {
    constexpr int NP = P * R;
    constexpr int C = FastCfg<R>::C;
    constexpr int G = 32 / P;          // column groups per warp
    constexpr int CPW = G * C;         // basis columns per warp
    constexpr long long BLK = fast_blk(NP);
    constexpr long long SLOT = BLK + NP;
    extern __shared__ __align__(128) double sm[];
    const unsigned long long t_start = Q.ready ? pint_dev::globaltimer() : 0;
    const int n = Q.n;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cg = lane / P, p = lane % P;
    const long long wps = Q.wps;
    const long long w = static_cast<long long>(blockIdx.x) * W + warp;
    const long long w_last = min(static_cast<long long>(blockIdx.x) * W + W, Q.N * wps) - 1;
    const long long j_lo = static_cast<long long>(blockIdx.x) * W / wps, j_hi = w_last / wps;
    const int ns = static_cast<int>(j_hi - j_lo + 1);
    const bool wlive = w <= w_last;
    const long long j = wlive ? w / wps : j_lo;
    const int wi = static_cast<int>(w - j * wps);
    const int js = static_cast<int>(j - j_lo);
    int kk[C];
    unsigned fmask = 0;
#pragma unroll
    for (int c = 0; c < C; ++c) {
        const int k = wi * CPW + c * G + cg;
        kk[c] = (wlive && k <= n) ? k : -1;
        if (kk[c] == n) fmask |= 1u << c;
    }
    const bool wf = __any_sync(kFull, fmask != 0);
    unsigned long long* bars = reinterpret_cast<unsigned long long*>(sm + ST * Q.NS * SLOT);
    unsigned* cnt = reinterpret_cast<unsigned*>(bars + ST);
    const unsigned bar0 = smem_u32(bars);
    // the forced column of slice jq is held by warp jq * wps + (n / CPW): is that warp in this CTA?
    const long long w0 = static_cast<long long>(blockIdx.x) * W;
    auto forced_here = [&](long long jq) {
        const long long fw = jq * wps + n / CPW;
        return fw >= w0 && fw <= w_last;
    };
    auto issue = [&](long long s, int b) {  // (one thread) step s of every staged slice -> buffer b
        unsigned bytes = 0;
        for (int q = 0; q < ns; ++q) bytes += 8u * static_cast<unsigned>(BLK + (forced_here(j_lo + q) ? NP : 0));
        asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(
                         bar0 + 8u * b),
                     "r"(bytes)
                     : "memory");
        for (int q = 0; q < ns; ++q) {
            const long long rix = (j_lo + q) * Q.S + s;
            double* dst = sm + (static_cast<long long>(b) * Q.NS + q) * SLOT;
            bulk_copy(smem_u32(dst), Q.rec + rix * BLK, static_cast<unsigned>(8 * BLK), bar0 + 8u * b);
            if (forced_here(j_lo + q))
                bulk_copy(smem_u32(dst + BLK), Q.hrec + rix * NP, static_cast<unsigned>(8 * NP), bar0 + 8u * b);
            if (s + 1 < Q.S) prefetch_l2(Q.rec + (rix + 1) * BLK, static_cast<unsigned>(8 * BLK));  // (the next refill)
        }
    };
    if (threadIdx.x == 0) {
        for (int b = 0; b < ST; ++b) {
            mbar_init(bar0 + 8u * b);
            cnt[b] = 0;
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int b = 0; b < ST && b < Q.S; ++b) issue(b, b);
    }
    double x[C][R];
#pragma unroll
    for (int c = 0; c < C; ++c)
#pragma unroll
        for (int t = 0; t < R; ++t) x[c][t] = (kk[c] < n && p * R + t == kk[c]) ? 1.0 : 0.0;  // e_k; forced, idle: 0
    for (long long s = 0; s < Q.S; ++s) {
        const int b = static_cast<int>(s % ST);
        mbar_wait(bar0 + 8u * b, static_cast<unsigned>((s / ST) & 1));
        const double* St = sm + (static_cast<long long>(b) * Q.NS + js) * SLOT;
        if (wf) fast_step<P, R, C, true>(x, St, St + BLK, p, fmask);
        else fast_step<P, R, C, false>(x, St, St, p, 0u);
        __syncwarp();
        if (lane == 0) {  // the last warp done with buffer b refills it with step s + ST
            __threadfence_block();
            const unsigned tk = atomicAdd(cnt + b, 1u);
            if (tk % W == W - 1 && s + ST < Q.S) issue(s + ST, b);
        }
    }
#pragma unroll
    for (int c = 0; c < C; ++c) {
        if (kk[c] < 0) continue;
        double* gp = Q.maps + (j * n) * Q.ldm + kk[c];
#pragma unroll
        for (int t = 0; t < R; ++t) {
            const int i = p * R + t;
            if (i < n) gp[static_cast<long long>(i) * Q.ldm] = x[c][t];
        }
    }
    // this warp's columns of slice j are stored: count it (a concurrent chain waits for all wps)
    // (a pad warp of a slice-aligned grid owns no column and is not counted)
    bool has_cols = false;
#pragma unroll
    for (int c = 0; c < C; ++c) has_cols |= kk[c] >= 0;
    if (Q.ready && wlive && __any_sync(kFull, has_cols)) {
        __syncwarp();
        if (lane == 0) {
            __threadfence();
            atomicAdd(Q.ready + j, 1);
            atomicMin(Q.span, t_start);
            atomicMax(Q.span + 1, pint_dev::globaltimer());
        }
    }
}

template <int kM>
int launch_records(pint_ctx* ctx, cudaStream_t st, const FastRecPlan& Q) {
    const long long warps = Q.N * Q.S;
    heat_fast_record_kernel<kM><<<static_cast<unsigned>((warps + 3) / 4), 128, 0, st>>>(Q);
    return pint_check_launch(ctx, "heat_fast_record_kernel");
}

template <int P, int R, int ST, int W>
int launch_fast_st(pint_ctx* ctx, const FastPlan& Q, size_t smem, long long ctas) {
    auto kern = heat_fast_build_kernel<P, R, ST, W>;
    pint_kernel_attrs(reinterpret_cast<const void*>(kern));  // (once: never between the chain and the build)
    if (!Q.ready) {
        kern<<<static_cast<unsigned>(ctas), 32 * W, smem, ctx->stream>>>(Q);
        return pint_check_launch(ctx, "heat_fast_build_kernel");
    }
    // signalling build: behind the waiting chain on the same stream, allowed to start while it runs
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(ctas), 1, 1);
    cfg.blockDim = dim3(32 * W, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, Q);
    return pint_check_launch(ctx, "heat_fast_build_kernel");
}

template <int P, int R, int W>
int launch_fast_w(pint_ctx* ctx, FastPlan Q) {
    constexpr int NP = P * R;
    constexpr int CPW = 32 / P * FastCfg<R>::C;
    long long wps = (Q.n + 1 + CPW - 1) / CPW;
    // slice-aligned CTAs (warps per slice padded to a multiple of W; the pad warps own no column)
    // where a slice has many warps: each CTA then stages ONE slice's records, small enough for 4
    // stages at 2 CTAs per SM (config 4: 129 -> 132 warps a slice, 2.3% idle; the record waits
    // of 2 shared stages were 16% of the stall samples)
    static const int align_env = [] {
        const char* e = std::getenv("PINT_FAST_SLICE_CTAS");
        return e ? std::atoi(e) : 1;
    }();
    if (align_env && W > 1 && wps >= 8 * W) wps = (wps + W - 1) / W * W;
    Q.wps = wps;
    Q.NS = static_cast<int>(std::min<long long>(W, (W + wps - 1) / wps + 1));  // slices a CTA's warps span
    if (wps % W == 0) Q.NS = 1;
    const size_t stage_bytes = sizeof(double) * Q.NS * (fast_blk(NP) + NP);
    const bool deep = kFastStagesMax * stage_bytes + 64 <= static_cast<size_t>(W) * 25 * 1024;  // (8 warps per SM either way)
    const size_t smem = (deep ? kFastStagesMax : 2) * stage_bytes + 64;
    if (smem > 227 * 1024) return pint_set_error(ctx, PINT_E_INVALID, "heat_fast_build: records exceed shared memory");
    const long long ctas = (Q.N * wps + W - 1) / W;
    return deep ? launch_fast_st<P, R, kFastStagesMax, W>(ctx, Q, smem, ctas) : launch_fast_st<P, R, 2, W>(ctx, Q, smem, ctas);
}

template <int P, int R>
int launch_fast(pint_ctx* ctx, const FastPlan& Q) {
    static const int w_env = [] {  // PINT_FAST_W=1|2|8: warps per CTA (experiments only)
        const char* e = std::getenv("PINT_FAST_W");
        return e ? std::atoi(e) : 0;
    }();
    if (w_env == 1) return launch_fast_w<P, R, 1>(ctx, Q);
    if (w_env == 2) return launch_fast_w<P, R, 2>(ctx, Q);
    if (w_env == 8 && R >= 32) return launch_fast_w<P, R, 8>(ctx, Q);
    return launch_fast_w<P, R, FastCfg<R>::W>(ctx, Q);
}

}  // namespace

bool heat_fast_supported(int64_t n) { return n >= 1 && fast_shape(n).ok(); }

int64_t heat_fast_records_doubles(int64_t n, int64_t N, int64_t S) {
    const FastShape f = fast_shape(n);
    if (!f.ok()) return 0;
    return N * S * (fast_blk(f.NP()) + f.NP());
}

int launch_heat_fast_factor(pint_ctx* ctx, cudaStream_t stream, int64_t n, int64_t N, int64_t S,
                            const int64_t* step_off, const double* slice_dt, const double* r, const double* fa,
                            const double* fb, const double* sx, double* records) {
    const FastShape f = fast_shape(n);
    if (!f.ok() || N < 0 || S < 0) return pint_set_error(ctx, PINT_E_INVALID, "heat_fast_factor: unsupported n");
    if (N == 0 || S == 0) return PINT_OK;
    const FastRecPlan Q{static_cast<int>(n), f.P, f.R, N, S, step_off, slice_dt, r, fa, fb, sx, records,
                        records + N * S * fast_blk(f.NP()), ctx->d_fail};
    switch (f.NP() / 32) {
        case 1: return launch_records<1>(ctx, stream, Q);
        case 2: return launch_records<2>(ctx, stream, Q);
        case 3: return launch_records<3>(ctx, stream, Q);
        case 4: return launch_records<4>(ctx, stream, Q);
        case 6: return launch_records<6>(ctx, stream, Q);
        case 8: return launch_records<8>(ctx, stream, Q);
        case 12: return launch_records<12>(ctx, stream, Q);
        case 16: return launch_records<16>(ctx, stream, Q);
        case 24: return launch_records<24>(ctx, stream, Q);
        default: return pint_set_error(ctx, PINT_E_INVALID, "heat_fast_factor: shape");
    }
}

int heat_fast_ready_target(int64_t n) {  // warps per slice (each adds 1 to ready[j] after its stores)
    const FastShape f = fast_shape(n);
    if (!f.ok()) return 0;
    const int cpw = 32 / f.P * (f.R <= 16 ? FastCfg<16>::C : f.R <= 32 ? FastCfg<32>::C : FastCfg<48>::C);
    return static_cast<int>((n + 1 + cpw - 1) / cpw);
}

void heat_fast_prepare(int64_t n) {  // every kernel variant the build for n may launch, attributes set
    const FastShape f = fast_shape(n);
    auto set = [](auto k) { pint_kernel_attrs(reinterpret_cast<const void*>(k)); };
    switch (f.P * 1000 + f.R) {
        case 2016: set(heat_fast_build_kernel<2, 16, 4, 1>); set(heat_fast_build_kernel<2, 16, 2, 1>); break;
        case 4016: set(heat_fast_build_kernel<4, 16, 4, 1>); set(heat_fast_build_kernel<4, 16, 2, 1>); break;
        case 8016: set(heat_fast_build_kernel<8, 16, 4, 1>); set(heat_fast_build_kernel<8, 16, 2, 1>); break;
        case 16016: set(heat_fast_build_kernel<16, 16, 4, 1>); set(heat_fast_build_kernel<16, 16, 2, 1>); break;
        case 32016:
            set(heat_fast_build_kernel<32, 16, 4, 4>), set(heat_fast_build_kernel<32, 16, 2, 4>);
            set(heat_fast_build_kernel<32, 16, 4, 8>), set(heat_fast_build_kernel<32, 16, 2, 8>);
            break;
        case 16032: set(heat_fast_build_kernel<16, 32, 4, 4>); set(heat_fast_build_kernel<16, 32, 2, 4>); break;
        case 16048: set(heat_fast_build_kernel<16, 48, 4, 4>); set(heat_fast_build_kernel<16, 48, 2, 4>); break;
        default: break;
    }
}

int launch_heat_fast_build(pint_ctx* ctx, int64_t n, int64_t N, int64_t S, const double* records, double* maps,
                           int* ready) {
    const FastShape f = fast_shape(n);
    if (!f.ok() || N < 0 || S < 0) return pint_set_error(ctx, PINT_E_INVALID, "heat_fast_build: unsupported n");
    if (N == 0) return PINT_OK;
    const FastPlan Q{static_cast<int>(n), N, S, 0, maps, pint_affine_ldm(n), records,
                     records + N * S * fast_blk(f.NP()), ready,
                     ready ? reinterpret_cast<unsigned long long*>(ready + ((N + 1) & ~1ll)) : nullptr};
    if (S == 0) return pint_set_error(ctx, PINT_E_INVALID, "heat_fast_build: S >= 1 required");
    switch (f.P * 1000 + f.R) {
        case 2016: return launch_fast<2, 16>(ctx, Q);
        case 4016: return launch_fast<4, 16>(ctx, Q);
        case 8016: return launch_fast<8, 16>(ctx, Q);
        case 16016: return launch_fast<16, 16>(ctx, Q);
        case 32016: {  // (records of 512 rows: 4 warps share a staged copy; PINT_FAST_W=8: experiment)
            static const int w8 = [] { const char* e = std::getenv("PINT_FAST_W"); return e && std::atoi(e) == 8; }();
            return w8 ? launch_fast_w<32, 16, 8>(ctx, Q) : launch_fast_w<32, 16, 4>(ctx, Q);
        }
        case 16032: return launch_fast<16, 32>(ctx, Q);
        case 16048: return launch_fast<16, 48>(ctx, Q);
        default: return pint_set_error(ctx, PINT_E_INVALID, "heat_fast_build: shape");
    }
}
