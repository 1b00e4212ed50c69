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
//    (every solve stays bit-identical), together with the forcing increments h*b_i. Each (slice,
//    step) record is one contiguous block (slice-major), so a warp stages it with two bulk copies
//    (cp.async.bulk + mbarrier) and pulls the record two steps ahead into L2.
//  * x / p_i is q0 = x*rcp, rem = fma(-p, q0, x), q = fma(rem, rcp, q0) with rcp = RN(1/p_i):
//    Markstein's theorem makes q the correctly rounded quotient whenever no intermediate
//    under/overflows. The dividends are range-checked OFF the dependent chain (forced lane: a
//    window test per row; basis lanes: a running minimum); if a check trips, the
//    kernel reports PINT_E_RANGE_RETRY and the host re-runs the build with the guarded variant
//    (exponent check on the chain, IEEE __ddiv_rn outside [2^-960, 2^997]).
//  * CTA = ONE warp, lane = trajectory: warp g of a slice runs columns 32g..32g+31 (k < n: basis
//    e_k, k == n: the forced run from 0, k > n: idle). The first kRegRows rows of every column
//    live in registers, the rest lane-interleaved in shared memory (conflict-free), read through
//    a software pipeline. Rows leave as coalesced 256 B stores into the row-major augmented map.
//
// Roofline: the per-column recurrence (S x n dependent rows of 7 FP64 ops) — latency-bound;
// algorithmic flops per slice-step: (n+1)(5n-4) + 5n (bench.py).
#include <cstdlib>
#include <cstring>

#include "pint_internal.cuh"

namespace {

using pint_dev::record_failure;
using namespace pint_async;

constexpr int kRegRows = 56;  // rows of each column held in registers (n >= kRegRows + 2)
// PINT_E_RANGE_RETRY is recorded at kRetryIndex + (slice or step): above every task index, so a
// real failure (a zero pivot at step q) always wins the lowest-index race and is never masked.
constexpr long long kRetryIndex = 1ll << 62;
// The fast division is exact for dividends in [2^-960, 2^997]. Upper side: with r <= 2^40 and
// |h*b| <= 2^900 (checked by heat_record_kernel) every state stays below 2^990 (each step map is
// a max-norm contraction). Lower side: every quotient q is checked against 2^-950 (zero allowed).
constexpr unsigned kQuotLo = (1023u - 950u) << 20;  // |hi word| of 2^-950

__host__ __device__ constexpr long long even(long long x) { return (x + 1) & ~1ll; }

// One (slice, step) record, doubles, every block a whole number of 128-byte lines (so the record
// kernel writes whole sectors and the bulk copies are aligned): [negr, 0 x 15] | (p_i, rcp_i) x n16 |
// h*b_i x n16 | c_i x n16, n16 = n rounded up to 16. Forward half = header + (p, rcp) [+ h*b].
__host__ __device__ constexpr long long n16(long long n) { return (n + 15) & ~15ll; }
__host__ __device__ constexpr long long pr_offset() { return 16; }
__host__ __device__ constexpr long long hb_offset(long long n) { return 16 + 2 * n16(n); }
__host__ __device__ constexpr long long cc_offset(long long n) { return 16 + 3 * n16(n); }
__host__ __device__ constexpr long long record_stride(long long n) { return 16 + 4 * n16(n); }

// The forced columns of 32 slices run in one warp (lane = slice), so the record kernel also
// writes a slice-group copy of the per-step data: block (s, G) for step s of slices 32G..32G+31,
// lane-minor so a warp's loads are contiguous: [-r x 32] | (p_i, rcp_i)[n16][32] | h*b_i[n16][32]
// | c_i[n16][32]. Forward half = -r, (p, rcp), h*b; back half = c.
__host__ __device__ constexpr long long fblock_pr(long long) { return 32; }
__host__ __device__ constexpr long long fblock_hb(long long n) { return 32 + 64 * n16(n); }
__host__ __device__ constexpr long long fblock_cc(long long n) { return 32 + 96 * n16(n); }
__host__ __device__ constexpr long long fblock_stride(long long n) { return 32 + 128 * n16(n); }
__host__ __device__ constexpr long long groups32(long long N) { return (N + 31) / 32; }

// Per-warp shared memory (doubles): [front pad][staged record][state (n-RR)*32][tail pad][2
// mbarriers]. The staged record mirrors one global record. The pads make the software pipeline's
// look-ahead loads (up to kBackAhead rows before the state and kFwdAhead rows after it) land
// inside the allocation; the values they read are never used.
constexpr int kFwdAhead = 3;   // forward row: 5 dependent FP64 ops (~40 cycles) vs ~52-cycle LDS
constexpr int kBackAhead = 8;  // back row: 2 dependent ops (~16 cycles)
__host__ __device__ constexpr long long front_pad(long long n) {
    return record_stride(n) >= 32 * kBackAhead ? 0 : even(32 * kBackAhead - record_stride(n));
}
// Warp roles: basis columns on the slice-major record; the forced columns of 32 slices per warp
// on the slice-group block; or — when that block does not fit in shared memory (large n) — one
// forced column per warp on the slice-major record.
enum : int { kBasis = 0, kForcedGroup = 1, kForcedSingle = 2 };
__host__ __device__ constexpr long long staged_doubles(long long n, int mode) {
    return mode == kForcedGroup ? fblock_stride(n) : record_stride(n);
}
__host__ __device__ constexpr int reg_rows(long long n) { return n >= kRegRows + 2 ? kRegRows : 0; }
__host__ __device__ constexpr long long warp_smem_doubles(long long n, int mode) {
    return (mode == kForcedGroup ? 0 : front_pad(n)) + staged_doubles(n, mode) + (n - reg_rows(n)) * 32 +
           32 * kFwdAhead + 2;
}
__host__ __device__ constexpr bool group_forced(long long n) {
    return 8 * warp_smem_doubles(n, kForcedGroup) <= 227 * 1024;
}

// doubles needed for the records of N slices x S steps x n rows: [N][S][record] | [S][N/32][block]
__host__ __device__ constexpr long long records_doubles(long long n, long long N, long long S) {
    return N * S * record_stride(n) + (group_forced(n) ? S * groups32(N) * fblock_stride(n) : 0);
}

struct RecView {
    const double* base;
    long long S, N;
    int n;
    __device__ __forceinline__ const double* rec(long long j, long long s) const {
        return base + (j * S + s) * record_stride(n);
    }
    __device__ __forceinline__ const double* fblock(long long s, long long G) const {
        return base + N * S * record_stride(n) + (s * groups32(N) + G) * fblock_stride(n);
    }
};

__host__ __device__ inline RecView rec_view(const double* base, int n, long long N, long long S) {
    return RecView{base, S, N, n};
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

// Thread t = (s, j) = s*N + j: step s of slice j — the Thomas forward pivots of tridiag(-r,
// 1+2r, -r) (linalg.cpp:80-90, with sub = sup = -r, diag = 1 + 2r as solve_implicit builds them),
// and the forcing increment h * b_i with b_i = fa*s_i + fb*s_i = heat_forcing(x_i, t)
// (pde_problems.cpp:26-29, 91-94), rounded exactly as `state[i] += dt_step * b[i]` consumes it.
// The pivot recurrence is sequential in i, so a thread owns a record; a warp holds 32 consecutive
// slices of one step. Rows are produced in chunks of kRecChunk into shared memory and leave as
// coalesced segments: per record and chunk, ONE warp store writes the 16 (p, rcp) doubles, the 8
// h*b and the 8 c doubles of the slice-major record (whole sectors), and the slice-group copy is
// written directly (32 consecutive lanes = 32 consecutive slices: contiguous).
constexpr int kRecChunk = 8;
constexpr int kRecLane = 4 * kRecChunk + 1;  // padded per-lane stride (doubles)

__global__ void __launch_bounds__(128) heat_record_kernel(int n, long long N, long long S, long long j0, long long Nc,
                                                          const int64_t* __restrict__ step_off,
                                                          const double* __restrict__ slice_dt,
                                                          const double* __restrict__ r_tab,
                                                          const double* __restrict__ fa, const double* __restrict__ fb,
                                                          const double* __restrict__ sx, double* __restrict__ rec,
                                                          FailRec* fail) {
    __shared__ double buf[4][32 * kRecLane];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const long long s = t / Nc, j = j0 + (t - s * Nc);  // slices [j0, j0 + Nc) of the N laid out
    const bool live = t < S * Nc && step_off[j] + s < step_off[j + 1];  // slice j may have fewer steps
    const long long q = live ? step_off[j] + s : 0;
    const unsigned live_mask = __ballot_sync(0xffffffffu, live);
    double* mine = buf[w] + lane * kRecLane;
    const double r = live ? r_tab[q] : 0.0;
    const double negr = -r;                                  // pde_problems.cpp:55
    const double diag = __dadd_rn(1.0, __dmul_rn(2.0, r));   // 1.0 + 2.0 * r
    const double h = live ? slice_dt[j] : 0.0, fq = live ? fa[q] : 0.0, gq = live ? fb[q] : 0.0;
    if (live && !(r >= 0.0 && r <= 0x1p40)) record_failure(fail, kRetryIndex + q, PINT_E_RANGE_RETRY, r);
    unsigned hb_max = 0;
    const bool fast_c = r >= 0x1p-960 && r <= 0x1p40;
    double* const myrec = rec + (j * S + s) * record_stride(n);  // this lane's slice-major record
    double* const fblk = rec + N * S * record_stride(n) + (s * groups32(N) + j / 32) * fblock_stride(n);
    const int fl = static_cast<int>(j & 31);  // lane slot in the slice-group block
    const bool grp = live && group_forced(n);  // the slice-group copy exists for this n
    if (live) reinterpret_cast<double4*>(myrec)[0] = make_double4(negr, 0.0, 0.0, 0.0);
    if (grp) fblk[fl] = negr;
    double p = diag, c = 0.0;
    for (int i0 = 0; i0 < n; i0 += kRecChunk) {
        const int rows = min(kRecChunk, n - i0);
        for (int u = 0; u < rows; ++u) {
            const int i = i0 + u;
            if (i > 0) p = __dsub_rn(diag, __dmul_rn(negr, c));  // pivot = diag - sub*c[i-1] (:84-88)
            if (live && p == 0.0) record_failure(fail, q, PINT_E_SINGULAR, static_cast<double>(i));
            const double rcp = __drcp_rn(p);
            // c[i] = sup / pivot: the Markstein division with the reciprocal the record carries
            // anyway when r in [2^-960, 2^40] (then p in [1 + r, 1 + 2r], |c| < 1: exact), IEEE otherwise
            c = (i < n - 1) ? (fast_c ? div_fast(negr, make_double2(p, rcp)) : __ddiv_rn(negr, p)) : 0.0;
            const double si = sx[i];
            mine[4 * u + 0] = p;
            mine[4 * u + 1] = rcp;
            const double hb = __dmul_rn(h, __dadd_rn(__dmul_rn(fq, si), __dmul_rn(gq, si)));
            hb_max = max(hb_max, static_cast<unsigned>(__double2hiint(hb)) & 0x7fffffffu);
            mine[4 * u + 2] = hb;
            mine[4 * u + 3] = c;
            if (grp) {
                reinterpret_cast<double2*>(fblk + fblock_pr(n))[i * 32 + fl] = make_double2(p, rcp);
                fblk[fblock_hb(n) + i * 32 + fl] = hb;
                fblk[fblock_cc(n) + i * 32 + fl] = c;
            }
        }
        __syncwarp();
        // this lane's slot in every record of the chunk: (p, rcp) element `lane` (lanes 0-15), h*b
        // row lane-16 (16-23) or c row lane-24 (24-31)
        const int k = lane & 7, half = (lane >> 3) & 1;
        const long long off = lane < 16 ? pr_offset() + 2 * i0 + lane : (half ? cc_offset(n) : hb_offset(n)) + i0 + k;
        const int soff = lane < 16 ? 4 * (lane >> 1) + (lane & 1) : 4 * k + 2 + half;
        const bool valid = lane < 16 ? lane < 2 * rows : k < rows;
        const unsigned mask = valid ? live_mask : 0u;
        // 16 shared loads in flight, then 16 stores (a store holds its source register until the
        // LSU drains it, so a load/store ping-pong on one register would serialise on that)
#pragma unroll
        for (int l0 = 0; l0 < 32; l0 += 16) {
            double v[16];
#pragma unroll
            for (int l = 0; l < 16; ++l) v[l] = buf[w][soff + (l0 + l) * kRecLane];
#pragma unroll
            for (int l = 0; l < 16; ++l) {  // the record of lane l0 + l
                double* dst = reinterpret_cast<double*>(__shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(myrec), l0 + l));
                if ((mask >> (l0 + l)) & 1u) dst[off] = v[l];
            }
        }
        __syncwarp();
    }
    if (live && hb_max >= ((1023u + 900u) << 20)) record_failure(fail, kRetryIndex + q, PINT_E_RANGE_RETRY, 0.0);
}

__device__ __forceinline__ double div_guarded(double x, double2 pr) {
    return out_of_range(x) ? __ddiv_rn(x, pr.x) : div_fast(x, pr);
}



struct BuildPlan {
    int n;
    int N;
    long long S;        // max steps per slice (record layout)
    int wps;            // basis warps (= CTAs) per slice = ceil(n/32); the forced columns: own grid
    const double* rec;
    const int64_t* step_off;
    double* maps;
    long long ldm;
    unsigned long long* per_slice_ns;
    FailRec* fail;
};



__device__ __forceinline__ unsigned hi_abs(double x) {
    return static_cast<unsigned>(__double2hiint(x)) & 0x7fffffffu;
}

// Record views of one warp's staged step. Basis and single-forced warps read the slice-major
// record: one broadcast value per row. Group-forced warps (lane = slice) read the slice-group
// block: row i of lane l at [i * 32 + l] (contiguous across lanes: conflict-free).
template <int kMode>
struct StagedStep {
    const double* R;
    int n, lane;
    static constexpr bool kForced = kMode != kBasis;
    static constexpr int kS = kMode == kForcedGroup ? 32 : 1;  // row stride of the per-row arrays
    __device__ __forceinline__ double negr() const { return kMode == kForcedGroup ? R[lane] : R[0]; }
    __device__ __forceinline__ const double2* pr() const {
        return kMode == kForcedGroup ? reinterpret_cast<const double2*>(R + fblock_pr(n)) + lane
                                     : reinterpret_cast<const double2*>(R + pr_offset());
    }
    __device__ __forceinline__ const double* hb() const {  // forced modes only
        return kMode == kForcedGroup ? R + fblock_hb(n) + lane : R + hb_offset(n);
    }
    __device__ __forceinline__ const double* cc() const {
        return kMode == kForcedGroup ? R + fblock_cc(n) + lane : R + cc_offset(n);
    }
};

// Forward elimination of one step (linalg.cpp:84-90). Forced warps first add the forcing
// increment, x + h*b (pde_problems.cpp:93, __dadd_rn as the reference's `state[i] += dt*b[i]`).
// Rows [0, RR) in reg[], the rest at st[32*(i-RR)], software-pipelined kFwdAhead rows ahead
// (every load is issued before the stores in front of it: the compiler cannot hoist a shared load
// above a shared store it cannot disambiguate). The quotients are range-checked by column_back,
// off the chain. Returns q_{n-1}; dm1 = q_{n-2}.
template <int RR, int kMode, bool kGuard>
__device__ __forceinline__ double column_forward(double (&reg)[RR > 0 ? RR : 1], double* st,
                                                 const StagedStep<kMode>& V, double& dm1) {
    constexpr int kS = StagedStep<kMode>::kS;
    constexpr bool kForced = StagedStep<kMode>::kForced;
    const int n = V.n;
    const double negr = V.negr();
    const double2* PR = V.pr();
    const double* HB = V.hb();
    auto divide = [&](double num, double2 pr) { return kGuard ? div_guarded(num, pr) : div_fast(num, pr); };
    // RR == 0: row 0 goes through the generic x - negr*d with d = -0.0, where negr*d is +0 (negr
    // <= 0) and x - (+0) == x bit-for-bit (even for x = -0), so the loop needs no row-0 select
    double d = -0.0;
#pragma unroll
    for (int i = 0; i < RR; ++i) {
        const double x = kForced ? __dadd_rn(reg[i], HB[i * kS]) : reg[i];
        d = divide((i == 0) ? x : __dsub_rn(x, __dmul_rn(negr, d)), PR[i * kS]);
        reg[i] = d;
    }
    dm1 = d;
    const int last = n - 1 - RR;  // last shared row (>= 0)
    const double2* pr = PR + RR * kS;
    const double* hb = HB + RR * kS;
    double2 pv[kFwdAhead];
    double xv[kFwdAhead], hv[kFwdAhead];
#pragma unroll
    for (int u = 0; u < kFwdAhead; ++u) {
        pv[u] = pr[u * kS];
        xv[u] = st[32 * u];
        hv[u] = kForced ? hb[u * kS] : 0.0;
    }
    // ring slot u holds row r + u; full blocks refill without predicates (a predicated refill
    // would turn into conditional moves that wait on the load), the < kFwdAhead tail rows are
    // already in the ring
    auto row = [&](int rr, double2 p, double x0, double h) {
        const double x = kForced ? __dadd_rn(x0, h) : x0;
        dm1 = d;
        d = divide(__dsub_rn(x, __dmul_rn(negr, d)), p);
        st[32 * rr] = d;
    };
    int r = 0;
#pragma unroll 1
    for (; r + kFwdAhead - 1 <= last; r += kFwdAhead) {
#pragma unroll
        for (int u = 0; u < kFwdAhead; ++u) {  // consume, then refill the slot in place
            row(r + u, pv[u], xv[u], hv[u]);
            pv[u] = pr[(r + u + kFwdAhead) * kS];
            xv[u] = st[32 * (r + u + kFwdAhead)];
            if (kForced) hv[u] = hb[(r + u + kFwdAhead) * kS];
        }
    }
#pragma unroll
    for (int u = 0; u < kFwdAhead - 1; ++u)
        if (r + u <= last) row(r + u, pv[u], xv[u], hv[u]);
    return d;
}

// Back substitution of one step (linalg.cpp:91): d_i = q_i - c_i d_{i+1}, shared rows pipelined
// kBackAhead rows ahead, then the register rows. qmin tracks min(|hi word of q_i| - 1) over the
// forward quotients it reads anyway (zero wraps to the maximum, so exact zeros pass): a quotient
// below 2^-950 means its dividend may have left Markstein's range (one VIADDMNMX per row).
template <int RR, int kMode>
__device__ __forceinline__ void column_back(double (&reg)[RR > 0 ? RR : 1], double* st, const StagedStep<kMode>& V,
                                            double d, double dm1, unsigned& qmin) {
    constexpr int kS = StagedStep<kMode>::kS;
    const int n = V.n;
    const double* CC = V.cc();
    const int top = n - 2 - RR;  // first shared row of the back pass
    if (top >= 0) {
        double yv[kBackAhead], cv[kBackAhead];
        const double* cc = CC + RR * kS;
#pragma unroll
        for (int u = 0; u < kBackAhead; ++u) {
            yv[u] = (u == 0) ? dm1 : st[32 * (top - u)];
            cv[u] = cc[(top - u) * kS];
        }
        // ring slot u holds row r - u (see column_forward)
        auto row = [&](int rr, double y, double c) {
            qmin = min(qmin, hi_abs(y) - 1u);
            d = __dsub_rn(y, __dmul_rn(c, d));
            st[32 * rr] = d;
        };
        int r = top;
#pragma unroll 1
        for (; r >= kBackAhead - 1; r -= kBackAhead) {
#pragma unroll
            for (int u = 0; u < kBackAhead; ++u) {  // consume, then refill the slot in place
                row(r - u, yv[u], cv[u]);
                yv[u] = st[32 * (r - u - kBackAhead)];
                cv[u] = cc[(r - u - kBackAhead) * kS];
            }
        }
#pragma unroll
        for (int u = 0; u < kBackAhead - 1; ++u)
            if (r - u >= 0) row(r - u, yv[u], cv[u]);
    }
#pragma unroll
    for (int i = RR - 1; i >= 0; --i) {
        if (i > n - 2) continue;  // (RR > 0 implies n >= RR + 2: never taken)
        qmin = min(qmin, hi_abs(reg[i]) - 1u);
        d = __dsub_rn(reg[i], __dmul_rn(CC[i * kS], d));
        reg[i] = d;
    }
}

#ifdef PINT_HEAT_PROF  // section timing for tools/heat_micro.cu only (never in the library build)
__device__ unsigned long long g_heat_prof[1 << 14][6];
__device__ unsigned long long g_heat_span[2][1 << 14][2];  // [forced][cta] = {start, end} globaltimer
#define HEAT_PROF_MARK(k)                           \
    do {                                            \
        const long long t_ = clock64();             \
        prof[k] += static_cast<unsigned long long>(t_ - t_prev); \
        t_prev = t_;                                \
    } while (0)
#else
#define HEAT_PROF_MARK(k) \
    do {                  \
    } while (0)
#endif

// CTA = ONE warp. Basis warps: warp g of slice blockIdx / wps, lane = basis column k = 32g + lane
// (k < n: e_k; beyond: idle), the slice's slice-major record broadcast to all lanes. Group-forced
// warps: lane = slice j = 32 blockIdx + lane, running that slice's forced trajectory c from 0 on
// the slice-group block. Single-forced warps (large n): slice blockIdx, lane 0 runs c. Warps share nothing — each stages its own
// copy of the step data in two halves with cp.async.bulk + mbarriers (forward half refilled during
// the back pass, back half during the forward pass) and pulls the step after next into L2 — so no
// CTA barrier couples a slice's warps and the single-warp CTAs pack over every SM. The forced
// columns run as their own grid on a side stream: no warp carries 31 idle lanes, and the basis
// grid stays at <= 2 warps per SM sub-partition at C2.
template <int RR, int kMode, bool kGuard>
__global__ void __maxnreg__(168) heat_build_kernel(BuildPlan P) {
    constexpr bool kForced = kMode != kBasis, kGroup = kMode == kForcedGroup;
    extern __shared__ __align__(16) double smem[];
    const unsigned long long t_start = pint_dev::globaltimer();
    // forced grid: let the basis grid (launched after it with programmatic stream serialization)
    // start now that this CTA is resident — its 8 large CTAs are placed before the basis CTAs
    // fill the SMs
    if (kForced) asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    const int n = P.n;
    const int lane = threadIdx.x;
    const long long slice = kGroup ? 32ll * blockIdx.x + lane : kForced ? blockIdx.x : blockIdx.x / P.wps;
    const long long g0 = kGroup ? blockIdx.x : slice;  // the block's slice group / slice
    const int k = kForced ? (kGroup || lane == 0 ? n : n + 1) : static_cast<int>(blockIdx.x - g0 * P.wps) * 32 + lane;
    const bool live = kGroup ? slice < P.N : k < n + (kForced ? 1 : 0);
    double* R = smem + (kGroup ? 0 : front_pad(n));
    double* st = R + staged_doubles(n, kMode) + lane;
    const unsigned bar_f = smem_u32(R + staged_doubles(n, kMode) + (n - RR) * 32 + 32 * kFwdAhead);
    const unsigned bar_b = bar_f + 8;
    const long long my_steps = (kGroup && !live) ? 0 : P.step_off[slice + 1] - P.step_off[slice];
    const long long steps = kGroup ? __reduce_max_sync(0xffffffffu, static_cast<unsigned>(my_steps)) : my_steps;
    const RecView V = rec_view(P.rec, n, P.N, P.S);
    auto src = [&](long long s) { return kGroup ? V.fblock(s, g0) : V.rec(g0, s); };
    // forward half: header + (p, rcp) [+ h*b for the forced modes]; back half: c
    const long long fwd_doubles = kGroup ? fblock_cc(n) : kForced ? cc_offset(n) : hb_offset(n);
    const long long back_doubles = kGroup ? 32 * n16(n) : even(n);
    const long long back_off = kGroup ? fblock_cc(n) : cc_offset(n);
    const unsigned fwd_bytes = 8u * static_cast<unsigned>(fwd_doubles);
    const unsigned back_bytes = 8u * static_cast<unsigned>(back_doubles);
    const unsigned all_bytes = 8u * static_cast<unsigned>(staged_doubles(n, kMode));
    const unsigned dst_f = smem_u32(R), dst_b = smem_u32(R + back_off);
    const StagedStep<kMode> SV{R, n, lane};

    if (lane == 0) {
        mbar_init(bar_f);
        mbar_init(bar_b);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncwarp();
    if (lane == 0 && steps > 0) {
        bulk_load(dst_f, src(0), fwd_bytes, bar_f);
        bulk_load(dst_b, src(0) + back_off, back_bytes, bar_b);
        if (steps > 1) prefetch_l2(src(1), all_bytes);
    }
    double reg[RR > 0 ? RR : 1];
#pragma unroll
    for (int i = 0; i < RR; ++i) reg[i] = (i == k) ? 1.0 : 0.0;  // e_k; the forced run starts at 0
    for (int i = RR; i < n; ++i) st[(i - RR) * 32] = (i == k) ? 1.0 : 0.0;

    unsigned qmin = 0xffffffffu;
#ifdef PINT_HEAT_PROF
    unsigned long long prof[6] = {0, 0, 0, 0, 0, 0};
    long long t_prev = clock64();
#endif
    for (long long s = 0; s < steps; ++s) {
        const unsigned parity = static_cast<unsigned>(s & 1);
        const bool active = s < my_steps;  // forced lanes of shorter slices idle at the tail
        mbar_wait(bar_f, parity);  // this step's forward half has landed
        HEAT_PROF_MARK(0);
        double d = 0.0, dm1 = 0.0;
        if (active) {
            d = column_forward<RR, kMode, kGuard>(reg, st, SV, dm1);
            qmin = min(qmin, hi_abs(d) - 1u);  // q_{n-1} (the back pass starts at row n-2)
        }
        HEAT_PROF_MARK(1);
        __syncwarp();  // every lane is done with the forward half
        if (lane == 0 && s + 1 < steps) bulk_load(dst_f, src(s + 1), fwd_bytes, bar_f);
        mbar_wait(bar_b, parity);
        HEAT_PROF_MARK(2);
        if (active) column_back<RR, kMode>(reg, st, SV, d, dm1, qmin);
        HEAT_PROF_MARK(3);
        __syncwarp();  // every lane is done with the back half
        if (lane == 0 && s + 1 < steps) {
            bulk_load(dst_b, src(s + 1) + back_off, back_bytes, bar_b);
            if (s + 2 < steps) prefetch_l2(src(s + 2), all_bytes);
        }
        HEAT_PROF_MARK(4);
    }
#ifdef PINT_HEAT_PROF
    if (lane == 0 && blockIdx.x < (1 << 14)) {
        if (!kForced)
            for (int q = 0; q < 5; ++q) g_heat_prof[blockIdx.x][q] = prof[q];
        g_heat_span[kForced ? 1 : 0][blockIdx.x][0] = t_start;
        g_heat_span[kForced ? 1 : 0][blockIdx.x][1] = pint_dev::globaltimer();
    }
#endif
    if (live) {
        double* gp = P.maps + slice * n * P.ldm + k;
#pragma unroll
        for (int i = 0; i < RR; ++i) gp[i * P.ldm] = reg[i];
        for (int i = RR; i < n; ++i) gp[i * P.ldm] = st[(i - RR) * 32];
        if (!kGuard && qmin < kQuotLo - 1u) record_failure(P.fail, kRetryIndex + slice, PINT_E_RANGE_RETRY, 0.0);
    }
    if (P.per_slice_ns && (kGroup ? live : lane == 0)) atomicAdd(P.per_slice_ns + slice, pint_dev::globaltimer() - t_start);
    // basis grid: complete only after the forced grid (so the stream order after this launch
    // holds for both); it overlapped this whole kernel, so the wait costs nothing
    if (!kForced) asm volatile("griddepcontrol.wait;\n" ::: "memory");
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
        const double* R = V.rec(0, s);
        const double2* PR = reinterpret_cast<const double2*>(R + pr_offset());
        const double* HB = R + hb_offset(n);
        const double* CC = R + cc_offset(n);
        const double negr = __ldg(R);
        double d = 0.0;
        for (int i = 0; i < n; ++i) {
            double x = st[i * 32];
            if (forcing) x = __dadd_rn(x, __ldg(HB + i));  // state += h*b (pde_problems.cpp:93)
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
    const bool grp = group_forced(P.n);
    const size_t smem = sizeof(double) * warp_smem_doubles(P.n, kBasis);
    const size_t fsmem = sizeof(double) * warp_smem_doubles(P.n, grp ? kForcedGroup : kForcedSingle);
    if (smem > 227 * 1024 || fsmem > 227 * 1024)
        return pint_set_error(ctx, PINT_E_INVALID, "heat_build: n too large for shared memory");
    auto kern = heat_build_kernel<RR, kBasis, kGuard>;
    auto fkern = grp ? heat_build_kernel<RR, kForcedGroup, kGuard> : heat_build_kernel<RR, kForcedSingle, kGuard>;
    smem_attrs(kern, smem);
    smem_attrs(fkern, fsmem);
    // forced columns first, then the basis grid with programmatic stream serialization: the
    // forced CTAs trigger it once resident, so both grids run together on one stream
    // PINT_HEAT_ONLY=basis|forced: timing experiments only (the other part of the maps is not built)
    const char* only = std::getenv("PINT_HEAT_ONLY");
    const bool run_f = !only || std::strcmp(only, "basis") != 0, run_b = !only || std::strcmp(only, "forced") != 0;
    if (run_f) fkern<<<static_cast<unsigned>(grp ? groups32(P.N) : P.N), 32, fsmem, ctx->stream>>>(P);
    if (const int rc = pint_check_launch(ctx, "heat_build_kernel (forced)")) return rc;
    if (run_b) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(static_cast<unsigned>(static_cast<long long>(P.N) * P.wps), 1, 1);
        cfg.blockDim = dim3(32, 1, 1);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = ctx->stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, kern, P);
    }
    if (const int rc = pint_check_launch(ctx, "heat_build_kernel")) return rc;
    return PINT_OK;
}

}  // namespace

int64_t heat_records_doubles(int64_t n, int64_t N, int64_t S) { return records_doubles(n, N, S); }

int launch_heat_factor_range(pint_ctx* ctx, int64_t n, int64_t N, int64_t S, int64_t j0, int64_t Nc,
                             const int64_t* step_off, const double* slice_dt, const double* r, const double* fa,
                             const double* fb, const double* sx, double* records) {
    if (n < 1 || N < 0 || S < 0 || j0 < 0 || Nc < 0 || j0 + Nc > N)
        return pint_set_error(ctx, PINT_E_INVALID, "heat_factor: bad sizes");
    if (Nc == 0 || S == 0) return PINT_OK;
    const long long threads = Nc * S;
    heat_record_kernel<<<static_cast<unsigned>((threads + 127) / 128), 128, 0, ctx->stream>>>(
        static_cast<int>(n), N, S, j0, Nc, step_off, slice_dt, r, fa, fb, sx, records, ctx->d_fail);
    return pint_check_launch(ctx, "heat_record_kernel");
}

int launch_heat_factor(pint_ctx* ctx, int64_t n, int64_t N, int64_t S, const int64_t* step_off,
                       const double* slice_dt, const double* r, const double* fa, const double* fb,
                       const double* sx, double* records) {
    return launch_heat_factor_range(ctx, n, N, S, 0, N, step_off, slice_dt, r, fa, fb, sx, records);
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
    P.wps = static_cast<int>((n + 31) / 32);
    P.rec = records;
    P.step_off = step_off;
    P.maps = maps;
    P.ldm = pint_affine_ldm(n);
    P.per_slice_ns = per_slice_ns;
    P.fail = ctx->d_fail;
    static_assert(reg_rows(kRegRows + 2) == kRegRows, "reg_rows");
    if (reg_rows(n) == kRegRows)
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
