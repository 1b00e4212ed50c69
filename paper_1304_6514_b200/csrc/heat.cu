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
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "pint_internal.cuh"

namespace {

using pint_dev::record_failure;
using namespace pint_async;

constexpr int kRegRows = 96;  // rows of each column held in registers (n >= kRegRows + 2)
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

// Slice-group block (s, G): the step-s data of slices 32G..32G+31, lane-minor, every part a whole
// number of 128-byte lines: pr2[n16+1][32] of (x, y) pairs — row 0 = (-r, 0), row i+1 = (p_i,
// rcp_i) — | h*b_i[n16][32] | c_i[n16][32]. The forced grid (lane = slice) bulk-copies a block's
// halves (forward: pr2 + h*b; back: c); a basis warp fetches its slice's column of pr2 and of c
// with a 2-D tile (TMA tensor copy), so one layout serves both grids.
__host__ __device__ constexpr long long fblock_hb(long long n) { return 64 * (n16(n) + 1); }
__host__ __device__ constexpr long long fblock_cc(long long n) { return 64 * (n16(n) + 1) + 32 * n16(n); }
__host__ __device__ constexpr long long fblock_stride(long long n) { return 64 * (n16(n) + 1) + 64 * n16(n); }
__host__ __device__ constexpr long long groups32(long long N) { return (N + 31) / 32; }
__host__ __device__ constexpr long long round16(long long x) { return (x + 15) & ~15ll; }

// Per-warp shared memory (doubles): [front pad][staged step][state (n-RR)*32][tail pad][2
// mbarriers]. The pads make the software pipeline's look-ahead loads (up to kBackAhead rows
// before the state and kFwdAhead rows after it) land inside the allocation; the values they read
// are never used.
constexpr int kFwdAhead = 3;   // forward row: 5 dependent FP64 ops (~40 cycles) vs ~52-cycle LDS
constexpr int kBackAhead = 8;  // back row: 2 dependent ops (~16 cycles)
// Warp roles. With the slice-group layout (n small enough that a forced warp stages a whole block:
// group_forced): basis columns on 2-D tiles of it (kBasisGroup) and 32 forced columns per warp on
// its halves (kForcedGroup). Otherwise (large n) slice-major records: basis columns (kBasis) and
// one forced column per warp (kForcedSingle).
enum : int { kBasis = 0, kForcedGroup = 1, kForcedSingle = 2, kBasisGroup = 3, kBasisForced = 4 };
// (kBasisForced: lane-interleaved columns on slice-major records like kBasis, each adding the forcing
// increment like kForcedSingle — the integrate closure's forced runs from caller states)
// kBasisGroup staging: [-r, 0, (p, rcp) x n][pad] | c pairs [n][2] (the 2-lane tile of c)
__host__ __device__ constexpr long long bg_fwd(long long n) { return round16(2 * (n + 1)); }
__host__ __device__ constexpr long long staged_doubles(long long n, int mode) {
    return mode == kForcedGroup ? fblock_stride(n) : mode == kBasisGroup ? bg_fwd(n) + round16(2 * n) : record_stride(n);
}
__host__ __device__ constexpr long long front_pad(long long n, int mode) {  // (multiple of 128 bytes)
    return staged_doubles(n, mode) >= 32 * kBackAhead ? 0 : round16(32 * kBackAhead - staged_doubles(n, mode));
}
__host__ __device__ constexpr int reg_rows(long long n) { return n >= kRegRows + 2 ? kRegRows : 0; }
// Shared state rows are lane-interleaved (row i of lane l at 32 i + l), except for a single-forced
// warp: its 32 lanes all run the one forced column in lockstep, so they share ONE copy (stride 1,
// every lane stores the same value).
__host__ __device__ constexpr int lane_stride(int mode) { return mode == kForcedSingle ? 1 : 32; }
// staged copies of the step data: the TMA-tiled basis warps double-buffer theirs (step s + 2 is
// fetched while step s + 1 waits in the other buffer), so no refill waits at a pass boundary
__host__ __device__ constexpr int stage_bufs(int mode) { return mode == kBasisGroup ? 2 : 1; }
__host__ __device__ constexpr long long warp_smem_doubles(long long n, int mode) {
    return front_pad(n, mode) + stage_bufs(mode) * staged_doubles(n, mode) + (n - reg_rows(n)) * lane_stride(mode) +
           lane_stride(mode) * kFwdAhead + 2 * stage_bufs(mode);
}
__host__ __device__ constexpr bool group_forced(long long n) {
    return 8 * warp_smem_doubles(n, kForcedGroup) <= 227 * 1024 && n + 1 <= 256;  // (tile rows <= 256)
}

// Rows per TMEM loop body: 2 chunks of 8 (the two register buffers alternate) and a multiple of
// both look-ahead rings (kTmAhead and kBackAhead), so every ring slot is a compile-time index.
constexpr int kTmBody = 16;
constexpr int kTmAhead = 4;  // forward (p, rcp) look-ahead over the TMEM rows
#ifndef PINT_TM_ROW_STORES
#define PINT_TM_ROW_STORES 1
#endif
constexpr bool kTmRowStores = PINT_TM_ROW_STORES;  // a tcgen05.st per row instead of per 8-row chunk
// The TMEM rows' quotient range check in the back pass, on the values it loads, instead of the
// forward pass, where the check's absolute value landed in the register an in-flight tcgen05.st
// was still reading (a write-after-read wait as long as a chain step)
#ifndef PINT_TM_BACK_CHECK
#define PINT_TM_BACK_CHECK 1
#endif
constexpr bool kTmBackCheck = PINT_TM_BACK_CHECK;

// ---- large n: heat_build_tmem_kernel --------------------------------------------------------
// When a warp's state no longer fits 4 times into shared memory (n >~ 280 with the one-warp-CTA
// build above: 134 KB per warp at n = 512, ONE warp per SM), a CTA of 5 warps runs ONE slice:
// warps 0-3 four basis column groups whose rows are split three ways — kTmRegRows in registers,
// tm_rows(n) in tensor memory (each warp owns a 32-lane quarter of the SM's 256 KB TMEM: up to 256
// doubles per thread), the rest lane-interleaved in shared memory — and warp 4 the slice's forced
// column (compact, see lane_stride) in the CTA that holds groups 0-3. The five warps share one
// staged copy of the step's record; whichever warp finishes a half last refills it.
constexpr int kTmRegRows = 64;
__host__ __device__ constexpr int tm_rows(long long n) {  // (256 doubles per thread at most)
    return n - kTmRegRows - 2 < kTmBody ? 0
           : (n - kTmRegRows - 2) / kTmBody >= 256 / kTmBody
               ? 256
               : static_cast<int>((n - kTmRegRows - 2) / kTmBody) * kTmBody;
}
__host__ __device__ constexpr long long tm_shared_rows(long long n) { return n - kTmRegRows - tm_rows(n); }
// shared memory (doubles): record | 4 x basis state [tm_shared_rows][32] | tail pad | forced state
// [n - kTmRegRows] | pad | bar_f, bar_b, counters, TMEM address
__host__ __device__ constexpr long long tm_forced_off(long long n) {
    return record_stride(n) + 4 * tm_shared_rows(n) * 32 + 32 * kFwdAhead;
}
__host__ __device__ constexpr long long tm_smem_doubles(long long n) {
    return tm_forced_off(n) + even(n - kTmRegRows + kFwdAhead) + 4;
}
__host__ __device__ constexpr bool use_tmem(long long n) {
    return !group_forced(n) && tm_rows(n) >= kTmBody && 8 * tm_smem_doubles(n) <= 227 * 1024 &&
           4 * (8 * warp_smem_doubles(n, kBasis) + 1024) > 228 * 1024;
}

// doubles of the records: slice-major [N][S][record], or slice-group [S][N/32][block]
__host__ __device__ constexpr long long records_doubles(long long n, long long N, long long S) {
    return group_forced(n) ? S * groups32(N) * fblock_stride(n) : N * S * record_stride(n);
}

struct RecView {
    const double* base;
    long long S, N;
    int n;
    __device__ __forceinline__ const double* rec(long long j, long long s) const {  // slice-major
        return base + (j * S + s) * record_stride(n);
    }
    __device__ __forceinline__ const double* fblock(long long s, long long G) const {  // slice-group
        return base + (s * groups32(N) + G) * fblock_stride(n);
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
// slices of one step. Slice-group layout: each row goes straight out (32 consecutive lanes = 32
// consecutive slices: contiguous, whole sectors). Slice-major layout (large n): rows are produced
// in chunks of kRecChunk into shared memory and leave as ONE warp store per record and chunk (the
// 16 (p, rcp), 8 h*b and 8 c doubles: whole sectors).
constexpr int kRecChunk = 8;
constexpr int kRecLane = 4 * kRecChunk + 1;  // padded per-lane stride (doubles)

__global__ void __launch_bounds__(128) heat_record_kernel(int n, long long N, long long S, long long j0, long long Nc,
                                                          long long s0, long long Sc, long long tab_pitch,
                                                          long long rec_s0, bool slice_major,
                                                          const int64_t* __restrict__ step_off,
                                                          const double* __restrict__ slice_dt,
                                                          const double* __restrict__ r_tab,
                                                          const double* __restrict__ fa, const double* __restrict__ fb,
                                                          const double* __restrict__ sx, double* __restrict__ rec,
                                                          FailRec* fail) {
    __shared__ double buf[4][32 * kRecLane];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const long long sr = t / Nc, j = j0 + (t - sr * Nc);  // slices [j0, j0 + Nc) of the N laid out,
    const long long s = s0 + sr;                           // steps [s0, s0 + Sc)
    const bool live = t < Sc * Nc && step_off[j] + s < step_off[j + 1];  // slice j may have fewer steps
    // the step tables: slice-major at step_off, or (tab_pitch > 0) this block alone at
    // [j][s - s0], pitch tab_pitch, from the pointers passed
    // table index: slice-major at step_off, or (tab_pitch > 0) this block alone at [j - j0][s - s0];
    // failures always carry the global task index step_off[j] + s (lowest-index semantics)
    const long long q = !live ? 0 : tab_pitch > 0 ? (j - j0) * tab_pitch + sr : step_off[j] + s;
    const long long qf = !live ? 0 : step_off[j] + s;
    const unsigned live_mask = __ballot_sync(0xffffffffu, live);
    double* mine = buf[w] + lane * kRecLane;
    const double r = live ? r_tab[q] : 0.0;
    const double negr = -r;                                  // pde_problems.cpp:55
    const double diag = __dadd_rn(1.0, __dmul_rn(2.0, r));   // 1.0 + 2.0 * r
    const double h = live ? slice_dt[j] : 0.0, fq = live ? fa[q] : 0.0, gq = live ? fb[q] : 0.0;
    if (live && !(r >= 0.0 && r <= 0x1p40)) record_failure(fail, kRetryIndex + qf, PINT_E_RANGE_RETRY, r);
    unsigned hb_max = 0;
    const bool fast_c = r >= 0x1p-960 && r <= 0x1p40;
    // slice-major records hold steps [rec_s0, rec_s0 + S) (the integrate path's bounded chunks)
    const bool group = group_forced(n) && !slice_major;
    double* const myrec = rec + (j * S + s - rec_s0) * record_stride(n);  // slice-major: this lane's record
    double* const fblk = rec + (s * groups32(N) + j / 32) * fblock_stride(n);  // slice-group block
    double2* const pr2 = reinterpret_cast<double2*>(fblk) + (j & 31);
    if (live && group) pr2[0] = make_double2(negr, 0.0);
    if (live && !group) reinterpret_cast<double4*>(myrec)[0] = make_double4(negr, 0.0, 0.0, 0.0);
    double p = diag, c = 0.0;
    if (group) {
        for (int i = 0; i < n; ++i) {
            if (i > 0) p = __dsub_rn(diag, __dmul_rn(negr, c));  // pivot = diag - sub*c[i-1] (:84-88)
            if (live && p == 0.0) record_failure(fail, qf, PINT_E_SINGULAR, static_cast<double>(i));
            const double rcp = __drcp_rn(p);
            c = (i < n - 1) ? (fast_c ? div_fast(negr, make_double2(p, rcp)) : __ddiv_rn(negr, p)) : 0.0;
            const double si = sx[i];
            const double hb = __dmul_rn(h, __dadd_rn(__dmul_rn(fq, si), __dmul_rn(gq, si)));
            hb_max = max(hb_max, static_cast<unsigned>(__double2hiint(hb)) & 0x7fffffffu);
            if (live) {
                pr2[(i + 1) * 32] = make_double2(p, rcp);
                fblk[fblock_hb(n) + i * 32 + (j & 31)] = hb;
                fblk[fblock_cc(n) + i * 32 + (j & 31)] = c;
            }
        }
        if (live && hb_max >= ((1023u + 900u) << 20)) record_failure(fail, kRetryIndex + qf, PINT_E_RANGE_RETRY, 0.0);
        return;
    }
    for (int i0 = 0; i0 < n; i0 += kRecChunk) {
        const int rows = min(kRecChunk, n - i0);
        for (int u = 0; u < rows; ++u) {
            const int i = i0 + u;
            if (i > 0) p = __dsub_rn(diag, __dmul_rn(negr, c));  // pivot = diag - sub*c[i-1] (:84-88)
            if (live && p == 0.0) record_failure(fail, qf, PINT_E_SINGULAR, static_cast<double>(i));
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
    if (live && hb_max >= ((1023u + 900u) << 20)) record_failure(fail, kRetryIndex + qf, PINT_E_RANGE_RETRY, 0.0);
}

__device__ __forceinline__ double div_guarded(double x, double2 pr) {
    return out_of_range(x) ? __ddiv_rn(x, pr.x) : div_fast(x, pr);
}



struct alignas(64) BuildPlan {
    CUtensorMap tm_pr;  // kBasisGroup: pr2 of the slice-group blocks as [blocks][n16+1][64] doubles
    CUtensorMap tm_cc;  // kBasisGroup: c of the slice-group blocks as [blocks][n16][32] doubles
    CUtensorMap tm_hb;  // (heat_forced_lanes_kernel: tm_pr / tm_hb / tm_cc over the slice-major records)
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
    long long s_begin, s_end;  // the steps this launch runs; s_begin > 0: resume from `maps`
    int* ready;                // (TMEM build) per-slice count of CTAs whose part of the map is stored
    unsigned long long* span;  // (with ready) {first CTA start, last CTA end} globaltimer of the launch
    int only;                  // timing experiments (PINT_HEAT_ONLY): 1 basis columns only, 2 forced only
};



__device__ __forceinline__ unsigned hi_abs(double x) {
    return static_cast<unsigned>(__double2hiint(x)) & 0x7fffffffu;
}

// Record views of one warp's staged step. kBasis / kForcedSingle: the slice-major record, one
// broadcast value per row. kBasisGroup: the slice's 2-D tiles — [-r, 0, (p, rcp) x n] and the c
// pairs [n][2] of lanes (2m, 2m+1), this slice at parity (slice & 1). kForcedGroup (lane = slice):
// the whole slice-group block, row i of lane l at [i * 32 + l] (contiguous: conflict-free).
template <int kMode>
struct StagedStep {
    const double* R;
    int n, lane, parity;
    static constexpr bool kForced = kMode == kForcedGroup || kMode == kForcedSingle || kMode == kBasisForced;
    static constexpr int kS = kMode == kForcedGroup ? 32 : 1;                             // p, rcp, h*b
    static constexpr int kSc = kMode == kForcedGroup ? 32 : kMode == kBasisGroup ? 2 : 1;  // c
    __device__ __forceinline__ double negr() const {
        return kMode == kForcedGroup ? R[2 * lane] : R[0];
    }
    __device__ __forceinline__ const double2* pr() const {
        return kMode == kForcedGroup ? reinterpret_cast<const double2*>(R) + 32 + lane
               : kMode == kBasisGroup ? reinterpret_cast<const double2*>(R) + 1
                                      : reinterpret_cast<const double2*>(R + pr_offset());
    }
    __device__ __forceinline__ const double* hb() const {  // forced modes only
        return kMode == kForcedGroup ? R + fblock_hb(n) + lane : R + hb_offset(n);
    }
    __device__ __forceinline__ const double* cc() const {
        return kMode == kForcedGroup ? R + fblock_cc(n) + lane
               : kMode == kBasisGroup ? R + bg_fwd(n) + parity
                                      : R + cc_offset(n);
    }
};

// ---- TMEM rows (large n, heat_build_tmem_kernel) --------------------------------------------
// tcgen05.ld / st, shape 32x32b: thread i of warp w <-> TMEM lane 32 (w % 4) + i; x16 = 16 32-bit
// columns = 8 doubles of that thread's own column (row r of the TMEM part at columns 2r, 2r + 1).
struct Tm8 {
    unsigned u[16];
    __device__ __forceinline__ double get(int i) const { return __hiloint2double(u[2 * i + 1], u[2 * i]); }
    __device__ __forceinline__ void put(int i, double v) {
        u[2 * i] = static_cast<unsigned>(__double2loint(v));
        u[2 * i + 1] = static_cast<unsigned>(__double2hiint(v));
    }
};
__device__ __forceinline__ void tm_ld(unsigned addr, Tm8& t) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15}, [%16];\n"
        : "=r"(t.u[0]), "=r"(t.u[1]), "=r"(t.u[2]), "=r"(t.u[3]), "=r"(t.u[4]), "=r"(t.u[5]), "=r"(t.u[6]),
          "=r"(t.u[7]), "=r"(t.u[8]), "=r"(t.u[9]), "=r"(t.u[10]), "=r"(t.u[11]), "=r"(t.u[12]), "=r"(t.u[13]),
          "=r"(t.u[14]), "=r"(t.u[15])
        : "r"(addr));
}
// the loaded registers are operands of the wait, so no use of them can be scheduled above it
__device__ __forceinline__ void tm_wait_ld(Tm8& t) {
    asm volatile("tcgen05.wait::ld.sync.aligned;\n"
                 : "+r"(t.u[0]), "+r"(t.u[1]), "+r"(t.u[2]), "+r"(t.u[3]), "+r"(t.u[4]), "+r"(t.u[5]), "+r"(t.u[6]),
                   "+r"(t.u[7]), "+r"(t.u[8]), "+r"(t.u[9]), "+r"(t.u[10]), "+r"(t.u[11]), "+r"(t.u[12]),
                   "+r"(t.u[13]), "+r"(t.u[14]), "+r"(t.u[15])
                 :
                 : "memory");
}
__device__ __forceinline__ void tm_st(unsigned addr, const Tm8& t) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16};\n" ::"r"(addr),
        "r"(t.u[0]), "r"(t.u[1]), "r"(t.u[2]), "r"(t.u[3]), "r"(t.u[4]), "r"(t.u[5]), "r"(t.u[6]), "r"(t.u[7]),
        "r"(t.u[8]), "r"(t.u[9]), "r"(t.u[10]), "r"(t.u[11]), "r"(t.u[12]), "r"(t.u[13]), "r"(t.u[14]), "r"(t.u[15])
        : "memory");  // (also keeps the look-ahead loads from being hoisted across chunks)
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
// one row (a double: two 32-bit TMEM columns) straight from the register that holds it
__device__ __forceinline__ void tm_st1(unsigned addr, double v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};\n" ::"r"(addr),
                 "r"(static_cast<unsigned>(__double2loint(v))), "r"(static_cast<unsigned>(__double2hiint(v)))
                 : "memory");
}

#ifdef PINT_HEAT_PROF  // section timing for tools/heat_micro.cu only (never in the library build)
__device__ unsigned long long g_heat_prof[1 << 14][6];
__device__ unsigned long long g_heat_prof_f[1 << 10][6];  // forced grid
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
#ifdef PINT_HEAT_PROF
// per-CTA segment cycles of thread 0's column (TMEM build): forward {reg, TMEM, shared} rows, back
// {shared, TMEM, reg} rows
__device__ unsigned long long g_heat_seg[1 << 14][8];
#define HEAT_SEG_START long long seg_prev_ = clock64()
#define HEAT_SEG_MARK(k)                                                            \
    do {                                                                            \
        if (threadIdx.x == 0) {                                                     \
            const long long t_ = clock64();                                         \
            g_heat_seg[blockIdx.x & 16383][k] += static_cast<unsigned long long>(t_ - seg_prev_); \
            seg_prev_ = t_;                                                         \
        }                                                                           \
    } while (0)
#else
#define HEAT_SEG_START \
    do {               \
    } while (0)
#define HEAT_SEG_MARK(k) \
    do {                 \
    } while (0)
#endif

// Forward rows [RR, RR + 16 nb) from TMEM (base row RR at column 0): chunk c + 1 is loaded while
// chunk c is eliminated, (p, rcp) read kTmAhead rows ahead. Quotients are range-checked here.
#ifndef PINT_TM_BODY_UNROLL
#define PINT_TM_BODY_UNROLL 2
#endif
template <bool kGuard, int kNb = 0>  // kNb > 0: nb = kNb, the body loop unrolled PINT_TM_BODY_UNROLL times
__device__ __forceinline__ void tmem_forward(unsigned tm, int nb, const double2* pr, double negr, double& d,
                                             unsigned& qmin) {
    if (kNb) nb = kNb;
    constexpr int kU = kNb ? PINT_TM_BODY_UNROLL : 1;
    auto divide = [&](double num, double2 p) { return kGuard ? div_guarded(num, p) : div_fast(num, p); };
    static_assert(kTmBody % kTmAhead == 0 && kTmBody % 16 == 0, "ring slots");
    double2 pv[kTmAhead];
#pragma unroll
    for (int u = 0; u < kTmAhead; ++u) pv[u] = pr[u];
    Tm8 A, B;
    tm_wait_st();  // the back pass's stores
    tm_ld(tm, A);
    tm_wait_ld(A);
#pragma unroll kU
    for (int b = 0; b < nb; ++b) {
#pragma unroll
        for (int c = 0; c < kTmBody / 8; ++c) {
            Tm8& cur = (c & 1) ? B : A;
            Tm8& nxt = (c & 1) ? A : B;
            const int ch = (kTmBody / 8) * b + c;
            const bool more = c + 1 < kTmBody / 8 || b + 1 < nb;
            if (more) tm_ld(tm + 16u * (ch + 1), nxt);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int rr = 8 * c + u;
                d = divide(__dsub_rn(cur.get(u), __dmul_rn(negr, d)), pv[rr % kTmAhead]);
                pv[rr % kTmAhead] = pr[kTmBody * b + rr + kTmAhead];
                if (kTmRowStores) tm_st1(tm + 16u * ch + 2u * u, d);
                else cur.put(u, d);
                if (!kTmBackCheck) qmin = min(qmin, hi_abs(d) - 1u);
            }
            if (!kTmRowStores) tm_st(tm + 16u * ch, cur);
            if (more) tm_wait_ld(nxt);
        }
    }
}

// Back substitution over the TMEM rows, last chunk first; cc = c of row RR; c read kBackAhead rows
// ahead.
template <int kNb = 0>  // (see tmem_forward)
__device__ __forceinline__ void tmem_back(unsigned tm, int nb, const double* cc, double& d, unsigned& qmin) {
    if (kNb) nb = kNb;
    constexpr int kU = kNb ? PINT_TM_BODY_UNROLL : 1;
    static_assert(kTmBody % kBackAhead == 0 && kBackAhead == 8, "ring slots");
    const int nch = nb * (kTmBody / 8);
    double cv[8];
#pragma unroll
    for (int v = 0; v < 8; ++v) cv[v] = cc[8 * nch - 1 - v];
    Tm8 A, B;
    tm_wait_st();  // the forward pass's stores
    tm_ld(tm + 16u * (nch - 1), A);
    tm_wait_ld(A);
#pragma unroll kU
    for (int b = 0; b < nb; ++b) {
#pragma unroll
        for (int c = 0; c < kTmBody / 8; ++c) {
            Tm8& cur = (c & 1) ? B : A;
            Tm8& nxt = (c & 1) ? A : B;
            const int ch = nch - 1 - ((kTmBody / 8) * b + c);
            const bool more = c + 1 < kTmBody / 8 || b + 1 < nb;
            if (more) tm_ld(tm + 16u * (ch - 1), nxt);
#pragma unroll
            for (int v = 0; v < 8; ++v) {
                const int u = 7 - v;
                const double q = cur.get(u);  // (this row's forward quotient)
                if (kTmBackCheck) qmin = min(qmin, hi_abs(q) - 1u);
                d = __dsub_rn(q, __dmul_rn(cv[v], d));
                cv[v] = cc[8 * ch + u - 8];
                if (kTmRowStores) tm_st1(tm + 16u * ch + 2u * u, d);
                else cur.put(u, d);
            }
            if (!kTmRowStores) tm_st(tm + 16u * ch, cur);
            if (more) tm_wait_ld(nxt);
        }
    }
}

// Forward elimination of one step (linalg.cpp:84-90). Forced warps first add the forcing
// increment, x + h*b (pde_problems.cpp:93, __dadd_rn as the reference's `state[i] += dt*b[i]`).
// Rows [0, RR) in reg[], the rest at st[32*(i-RR)], software-pipelined kFwdAhead rows ahead
// (every load is issued before the stores in front of it: the compiler cannot hoist a shared load
// above a shared store it cannot disambiguate). Quotients are range-checked off the chain: the
// register rows here, the shared rows in column_back. Returns q_{n-1}; dm1 = q_{n-2}.
template <int RR, int kMode, bool kGuard, int kLS = lane_stride(kMode), bool kTm = false, int kNs = 0>
__device__ __forceinline__ double column_forward(double (&reg)[RR > 0 ? RR : 1], double* st,
                                                 const StagedStep<kMode>& V, double& dm1, unsigned& qmin,
                                                 unsigned tm = 0, int tm_bodies = 0) {
    constexpr int kS = StagedStep<kMode>::kS;
    constexpr bool kForced = StagedStep<kMode>::kForced;
    // kNs > 0: n known at compile time (the TMEM build at n = kNs), so the shared-row loops unroll
    // completely and ptxas places every look-ahead load where it hides its latency (with a runtime
    // trip count it sank a whole ring's refills to the end of each iteration, right in front of
    // their first use: ~9 cycles a row)
    const int n = kNs ? kNs : V.n;
    if (kNs) tm_bodies = tm_rows(kNs) / kTmBody;
    const double negr = V.negr();
    const double2* PR = V.pr();
    const double* HB = V.hb();
    auto divide = [&](double num, double2 pr) { return kGuard ? div_guarded(num, pr) : div_fast(num, pr); };
    // RR == 0: row 0 goes through the generic x - negr*d with d = -0.0, where negr*d is +0 (negr
    // <= 0) and x - (+0) == x bit-for-bit (even for x = -0), so the loop needs no row-0 select
    double d = -0.0;
    HEAT_SEG_START;
#pragma unroll
    for (int i = 0; i < RR; ++i) {
        const double x = kForced ? __dadd_rn(reg[i], HB[i * kS]) : reg[i];
        d = divide((i == 0) ? x : __dsub_rn(x, __dmul_rn(negr, d)), PR[i * kS]);
        reg[i] = d;
        qmin = min(qmin, hi_abs(d) - 1u);  // ~40 cycles of chain per row: room for the check here
    }
    dm1 = d;
    const int B = RR + (kTm ? kTmBody * tm_bodies : 0);  // first shared row
    if (kTm) HEAT_SEG_MARK(0);
    if (kTm) tmem_forward<kGuard, kNs ? tm_rows(kNs) / kTmBody : 0>(tm, tm_bodies, PR + RR, negr, d, qmin);
    if (kTm) HEAT_SEG_MARK(1);
    const int last = n - 1 - B;  // last shared row (>= 0)
    const double2* pr = PR + B * kS;
    const double* hb = HB + B * kS;
    double2 pv[kFwdAhead];
    double xv[kFwdAhead], hv[kFwdAhead];
#pragma unroll
    for (int u = 0; u < kFwdAhead; ++u) {
        pv[u] = pr[u * kS];
        xv[u] = st[kLS * u];
        hv[u] = kForced ? hb[u * kS] : 0.0;
    }
    // ring slot u holds row r + u; full blocks refill without predicates (a predicated refill
    // would turn into conditional moves that wait on the load), the < kFwdAhead tail rows are
    // already in the ring
    auto row = [&](int rr, double2 p, double x0, double h) {
        const double x = kForced ? __dadd_rn(x0, h) : x0;
        dm1 = d;
        d = divide(__dsub_rn(x, __dmul_rn(negr, d)), p);
        st[kLS * rr] = d;
    };
    int r = 0;
    constexpr int kFwdUnroll = kNs ? (kNs - RR - tm_rows(kNs) + kFwdAhead) / kFwdAhead : 1;
#pragma unroll kFwdUnroll
    for (; r + kFwdAhead - 1 <= last; r += kFwdAhead) {
#pragma unroll
        for (int u = 0; u < kFwdAhead; ++u) {  // consume, then refill the slot in place
            row(r + u, pv[u], xv[u], hv[u]);
            pv[u] = pr[(r + u + kFwdAhead) * kS];
            xv[u] = st[kLS * (r + u + kFwdAhead)];
            if (kForced) hv[u] = hb[(r + u + kFwdAhead) * kS];
        }
    }
#pragma unroll
    for (int u = 0; u < kFwdAhead - 1; ++u)
        if (r + u <= last) row(r + u, pv[u], xv[u], hv[u]);
    if (kTm) HEAT_SEG_MARK(2);
    return d;
}

// Back substitution of one step (linalg.cpp:91): d_i = q_i - c_i d_{i+1}, shared rows pipelined
// kBackAhead rows ahead, then the register rows. qmin tracks min(|hi word of q_i| - 1) over the
// forward quotients (zero wraps to the maximum, so exact zeros pass): a quotient below 2^-950
// means its dividend may have left Markstein's range (one VIADDMNMX per row) — for the shared
// rows here, as they are read back anyway; for the register rows in column_forward.
template <int RR, int kMode, int kLS = lane_stride(kMode), bool kTm = false, int kNs = 0>
__device__ __forceinline__ void column_back(double (&reg)[RR > 0 ? RR : 1], double* st, const StagedStep<kMode>& V,
                                            double d, double dm1, unsigned& qmin, unsigned tm = 0,
                                            int tm_bodies = 0) {
    constexpr int kS = StagedStep<kMode>::kSc;
    const int n = kNs ? kNs : V.n;  // (kNs: see column_forward)
    if (kNs) tm_bodies = tm_rows(kNs) / kTmBody;
    const double* CC = V.cc();
    const int B = RR + (kTm ? kTmBody * tm_bodies : 0);  // first shared row
    const int top = n - 2 - B;                           // first shared row of the back pass
    HEAT_SEG_START;
    if (top >= 0) {
        double yv[kBackAhead], cv[kBackAhead];
        const double* cc = CC + B * kS;
#pragma unroll
        for (int u = 0; u < kBackAhead; ++u) {
            yv[u] = (u == 0) ? dm1 : st[kLS * (top - u)];
            cv[u] = cc[(top - u) * kS];
        }
        // ring slot u holds row r - u (see column_forward)
        auto row = [&](int rr, double y, double c) {
            qmin = min(qmin, hi_abs(y) - 1u);
            d = __dsub_rn(y, __dmul_rn(c, d));
            st[kLS * rr] = d;
        };
        int r = top;
        constexpr int kBackUnroll = kNs ? (kNs - RR - tm_rows(kNs) + kBackAhead) / kBackAhead : 1;
#pragma unroll kBackUnroll
        for (; r >= kBackAhead - 1; r -= kBackAhead) {
#pragma unroll
            for (int u = 0; u < kBackAhead; ++u) {  // consume, then refill the slot in place
                row(r - u, yv[u], cv[u]);
                yv[u] = st[kLS * (r - u - kBackAhead)];
                cv[u] = cc[(r - u - kBackAhead) * kS];
            }
        }
#pragma unroll
        for (int u = 0; u < kBackAhead - 1; ++u)
            if (r - u >= 0) row(r - u, yv[u], cv[u]);
    }
    if (kTm) HEAT_SEG_MARK(3);
    if (kTm) tmem_back<kNs ? tm_rows(kNs) / kTmBody : 0>(tm, tm_bodies, CC + RR, d, qmin);
    if (kTm) HEAT_SEG_MARK(4);
#pragma unroll
    for (int i = RR - 1; i >= 0; --i) {  // (RR > 0 only for n >= RR + 2: every register row is a back row)
        d = __dsub_rn(reg[i], __dmul_rn(CC[i * kS], d));  // (the register rows' quotients were checked
        reg[i] = d;                                         //  by column_forward, where they are made)
    }
    if (kTm) HEAT_SEG_MARK(5);
}


// 2-D/3-D tile copies (TMA tensor) of a slice's columns out of the slice-group blocks.
__device__ __forceinline__ void tile_load(unsigned dst, const CUtensorMap* tm, int c0, int c1, int c2,
                                          unsigned bytes, unsigned bar) {
    asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(bar),
                 "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];\n" ::"r"(dst),
        "l"(reinterpret_cast<unsigned long long>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void tile_prefetch(const CUtensorMap* tm, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];\n" ::"l"(
                     reinterpret_cast<unsigned long long>(tm)),
                 "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}

// CTA = ONE warp. Basis warps (kBasis / kBasisGroup): warp g of slice blockIdx / wps, lane = basis
// column k = 32g + lane (k < n: e_k; beyond: idle), reading the slice's step data as broadcasts.
// Group-forced warps: lane = slice j = 32 blockIdx + lane, running that slice's forced trajectory
// c from 0 on the slice-group block. Single-forced warps (large n): slice blockIdx, lane 0 runs c.
// Warps share nothing — each stages its own copy of the step data in two halves (cp.async.bulk, or
// TMA tiles for kBasisGroup, completing on mbarriers; the forward half refilled during the back
// pass, the back half during the forward pass) and pulls the step after next into L2 — so no CTA
// barrier couples a slice's warps and the single-warp CTAs pack over every SM. The forced columns
// are their own grid, launched first: no warp carries 31 idle lanes, and the basis grid stays at
// <= 2 warps per SM sub-partition at C2.
template <int RR, int kMode, bool kGuard>
__global__ void __maxnreg__(255) heat_build_kernel(const __grid_constant__ BuildPlan P) {
    constexpr bool kForced = kMode == kForcedGroup || kMode == kForcedSingle;
    constexpr bool kGroup = kMode == kForcedGroup;   // lane = slice
    constexpr bool kTiles = kMode == kBasisGroup;    // TMA tiles of the slice-group blocks
    extern __shared__ __align__(128) double smem[];
    const unsigned long long t_start = pint_dev::globaltimer();
    // forced grid: let the basis grid (launched after it with programmatic stream serialization)
    // start now that this CTA is resident — its large CTAs are placed before the basis CTAs fill
    // the SMs
    if (kForced) asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    const int n = P.n;
    const int lane = threadIdx.x;
    // group-forced: two CTAs per slice group, each running 16 of its slices on lanes 0-15 (lanes
    // 16-31 shadow them — same addresses, broadcast — and store nothing): half the shared-memory
    // wavefronts per row of a full 32-slice warp
    const int el = kGroup ? 16 * static_cast<int>(blockIdx.x & 1) + (lane & 15) : lane;
    const long long slice = kGroup ? 32ll * (blockIdx.x >> 1) + el : kForced ? blockIdx.x : blockIdx.x / P.wps;
    const long long g0 = kGroup ? (blockIdx.x >> 1) : slice;  // the block's slice group / slice
    // (single-forced: all 32 lanes run the forced column on one shared copy of the state; lane 0
    // writes it out)
    constexpr int kLS = lane_stride(kMode);
    const int k = kForced ? n : static_cast<int>(blockIdx.x - g0 * P.wps) * 32 + lane;
    const bool live = kGroup ? (lane < 16 && slice < P.N) : kForced ? lane == 0 : k < n;
    constexpr int kBufs = stage_bufs(kMode);
    double* R0 = smem + front_pad(n, kMode);  // kBufs staged copies of the step data
    double* st = R0 + kBufs * staged_doubles(n, kMode) + (kLS == 32 ? lane : 0);
    // mbarriers of buffer b: forward half at bar0 + 16 b, back half at bar0 + 16 b + 8
    const unsigned bar0 = smem_u32(R0 + kBufs * staged_doubles(n, kMode) + (n - RR) * kLS + kLS * kFwdAhead);
    const long long my_all = (kGroup && slice >= P.N) ? 0 : P.step_off[slice + 1] - P.step_off[slice];
    const long long all = kGroup ? __reduce_max_sync(0xffffffffu, static_cast<unsigned>(my_all)) : my_all;
    // this launch: steps [s_begin, s_end) of the slice, counted from s0 = s_begin below
    const long long s0 = P.s_begin;
    const long long my_steps = max(0ll, min(my_all, P.s_end) - s0);
    const long long steps = max(0ll, min(all, P.s_end) - s0);
    const RecView V = rec_view(P.rec, n, P.N, P.S);
    auto src = [&](long long s) { return kGroup ? V.fblock(s, g0) : V.rec(g0, s); };
    // forward half: header + (p, rcp) [+ h*b for the forced modes]; back half: c
    const long long fwd_doubles = kGroup ? fblock_cc(n) : kTiles ? 2 * (n + 1) : kForced ? cc_offset(n) : hb_offset(n);
    const long long back_doubles = kGroup ? 32 * n16(n) : kTiles ? 2 * n : even(n);
    const long long back_off = kGroup ? fblock_cc(n) : kTiles ? bg_fwd(n) : cc_offset(n);
    const unsigned fwd_bytes = 8u * static_cast<unsigned>(fwd_doubles);
    const unsigned back_bytes = 8u * static_cast<unsigned>(back_doubles);
    const unsigned all_bytes = 8u * static_cast<unsigned>(staged_doubles(n, kMode));
    auto buf = [&](int b) { return R0 + b * staged_doubles(n, kMode); };
    // kTiles coordinates: column 2*(slice % 32) of pr2 / lanes (slice % 32) & ~1 of c; block s*N32 + G
    const int tx = static_cast<int>(slice & 31), tg = static_cast<int>(slice >> 5), ng = static_cast<int>(groups32(P.N));
    auto load_fwd = [&](long long s, int b) {
        s += s0;
        const unsigned dst = smem_u32(buf(b)), bar = bar0 + 16u * b;
        if (kTiles) tile_load(dst, &P.tm_pr, 2 * tx, 0, static_cast<int>(s) * ng + tg, fwd_bytes, bar);
        else bulk_load(dst, src(s), fwd_bytes, bar);
    };
    auto load_back = [&](long long s, int b) {
        s += s0;
        const unsigned dst = smem_u32(buf(b) + back_off), bar = bar0 + 16u * b + 8u;
        if (kTiles) tile_load(dst, &P.tm_cc, tx & ~1, 0, static_cast<int>(s) * ng + tg, back_bytes, bar);
        else bulk_load(dst, src(s) + back_off, back_bytes, bar);
    };
    auto prefetch = [&](long long s) {
        s += s0;
        if (kTiles) {
            tile_prefetch(&P.tm_pr, 2 * tx, 0, static_cast<int>(s) * ng + tg);
            tile_prefetch(&P.tm_cc, tx & ~1, 0, static_cast<int>(s) * ng + tg);
        } else {
            prefetch_l2(src(s), all_bytes);
        }
    };

    if (lane == 0) {
        for (int b = 0; b < 2 * kBufs; ++b) mbar_init(bar0 + 8u * b);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncwarp();
    if (lane == 0 && steps > 0) {
        for (int b = 0; b < kBufs && b < steps; ++b) {
            load_fwd(b, b);
            load_back(b, b);
        }
        if (steps > kBufs) prefetch(kBufs);
    }
    double reg[RR > 0 ? RR : 1];
#pragma unroll
    for (int i = 0; i < RR; ++i) reg[i] = (i == k) ? 1.0 : 0.0;  // e_k; the forced run starts at 0
    for (int i = RR; i < n; ++i) st[(i - RR) * kLS] = (i == k) ? 1.0 : 0.0;
    // a resumed segment starts from the column the previous one stored (the group-forced shadow
    // lanes read their slice's column too)
    if (s0 > 0 && (kGroup ? slice < P.N : (kForced || k < n))) {  // (only lanes that own a column)
        const double* gp = P.maps + slice * n * P.ldm + k;
#pragma unroll
        for (int i = 0; i < RR; ++i) reg[i] = gp[i * P.ldm];
        for (int i = RR; i < n; ++i) st[(i - RR) * kLS] = gp[i * P.ldm];
    }

    unsigned qmin = 0xffffffffu;
#ifdef PINT_HEAT_PROF
    unsigned long long prof[6] = {0, 0, 0, 0, 0, 0};
    long long t_prev = clock64();
#endif
    for (long long s = 0; s < steps; ++s) {
        const int b = kBufs == 2 ? static_cast<int>(s & 1) : 0;
        const unsigned parity = static_cast<unsigned>((kBufs == 2 ? s >> 1 : s) & 1);
        const bool active = s < my_steps;  // forced lanes of shorter slices idle at the tail
        const StagedStep<kMode> SV{buf(b), n, el, static_cast<int>(slice & 1)};
        mbar_wait(bar0 + 16u * b, parity);  // this step's forward half has landed
        HEAT_PROF_MARK(0);
        double d = 0.0, dm1 = 0.0;
        if (active) {
            d = column_forward<RR, kMode, kGuard>(reg, st, SV, dm1, qmin);
            qmin = min(qmin, hi_abs(d) - 1u);  // q_{n-1} (the back pass starts at row n-2)
        }
        HEAT_PROF_MARK(1);
        if (kBufs == 1) {
            __syncwarp();  // every lane is done with the forward half
            if (lane == 0 && s + 1 < steps) load_fwd(s + 1, 0);
        }
        mbar_wait(bar0 + 16u * b + 8u, parity);
        HEAT_PROF_MARK(2);
        if (active) column_back<RR, kMode>(reg, st, SV, d, dm1, qmin);
        HEAT_PROF_MARK(3);
        __syncwarp();  // every lane is done with this step's buffer
        if (lane == 0 && s + kBufs < steps) {
            if (kBufs == 2) load_fwd(s + 2, b);
            load_back(s + kBufs, b);
            if (s + kBufs + 1 < steps) prefetch(s + kBufs + 1);
        }
        HEAT_PROF_MARK(4);
    }
#ifdef PINT_HEAT_PROF
    if (lane == 0 && blockIdx.x < (1 << 14)) {
        for (int q = 0; q < 5; ++q) (kForced ? g_heat_prof_f[blockIdx.x & 1023] : g_heat_prof[blockIdx.x])[q] = prof[q];
        g_heat_span[kForced ? 1 : 0][blockIdx.x][0] = t_start;
        g_heat_span[kForced ? 1 : 0][blockIdx.x][1] = pint_dev::globaltimer();
    }
#endif
    if (live) {
        double* gp = P.maps + slice * n * P.ldm + k;
#pragma unroll
        for (int i = 0; i < RR; ++i) gp[i * P.ldm] = reg[i];
        for (int i = RR; i < n; ++i) gp[i * P.ldm] = st[(i - RR) * kLS];
        if (!kGuard && qmin < kQuotLo - 1u) record_failure(P.fail, kRetryIndex + slice, PINT_E_RANGE_RETRY, 0.0);
    }
    if (P.per_slice_ns && (kGroup ? live : lane == 0)) atomicAdd(P.per_slice_ns + slice, pint_dev::globaltimer() - t_start);
    // basis grid: complete only after the forced grid (so the stream order after this launch
    // holds for both); it overlapped this whole kernel, so the wait costs nothing
    if (!kForced) asm volatile("griddepcontrol.wait;\n" ::: "memory");
}

template <bool kGuard, int kNs = 0>  // kNs > 0: built for n = kNs only (column_forward)
__global__ void __launch_bounds__(160, 1) heat_build_tmem_kernel(const __grid_constant__ BuildPlan P) {
    constexpr int RR = kTmRegRows;
    extern __shared__ __align__(128) double smem[];
    const unsigned long long t_start = pint_dev::globaltimer();
    const int n = kNs ? kNs : P.n;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int cps = (P.wps + 3) / 4;  // CTAs per slice
    const long long slice = blockIdx.x / cps;
    const int cta = static_cast<int>(blockIdx.x - slice * cps);
    const bool forced = warp == 4;
    const int g = 4 * cta + warp;
    const bool wlive = forced ? cta == 0 && P.only != 1 : g < P.wps && P.only != 2;  // this warp has columns
    const int k = forced ? n : 32 * g + lane;
    const int nlive = (P.only == 2 ? 0 : min(4, P.wps - 4 * cta)) + (cta == 0 && P.only != 1 ? 1 : 0);
    const int nb = tm_rows(n) / kTmBody;
    const long long M = tm_shared_rows(n);
    double* R = smem;
    double* st = forced ? R + tm_forced_off(n) : R + record_stride(n) + warp * M * 32 + lane;
    double* tail = R + tm_smem_doubles(n) - 4;
    const unsigned bar_f = smem_u32(tail), bar_b = bar_f + 8;
    unsigned* cnt = reinterpret_cast<unsigned*>(tail + 2);
    unsigned* tslot = reinterpret_cast<unsigned*>(tail + 3);
    const long long steps = P.step_off[slice + 1] - P.step_off[slice];
    const RecView V = rec_view(P.rec, n, P.N, P.S);
    const unsigned fwd_bytes = 8u * static_cast<unsigned>(cc_offset(n));  // header, (p, rcp), h*b
    const unsigned back_bytes = 8u * static_cast<unsigned>(even(n));
    auto load_fwd = [&](long long s) { bulk_load(smem_u32(R), V.rec(slice, s), fwd_bytes, bar_f); };
    auto load_back = [&](long long s) {
        bulk_load(smem_u32(R + cc_offset(n)), V.rec(slice, s) + cc_offset(n), back_bytes, bar_b);
    };
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tslot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    if (threadIdx.x == 0) {
        mbar_init(bar_f);
        mbar_init(bar_b);
        cnt[0] = cnt[1] = 0;
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const unsigned tm = *tslot + ((32u * static_cast<unsigned>(warp & 3)) << 16);
    if (threadIdx.x == 0 && steps > 0) {
        load_fwd(0);
        load_back(0);
        if (steps > 1) prefetch_l2(V.rec(slice, 1), 8u * static_cast<unsigned>(record_stride(n)));
    }
    double reg[RR];
#pragma unroll
    for (int i = 0; i < RR; ++i) reg[i] = (i == k) ? 1.0 : 0.0;  // e_k; the forced run starts at 0
    if (!forced) {
        for (int ch = 0; ch < nb * (kTmBody / 8); ++ch) {
            Tm8 t;
#pragma unroll
            for (int u = 0; u < 8; ++u) t.put(u, (RR + 8 * ch + u == k) ? 1.0 : 0.0);
            tm_st(tm + 16u * ch, t);
        }
    }
    const int kls = forced ? 1 : 32;
    for (long long i = RR + (forced ? 0 : nb * kTmBody); i < n; ++i)
        st[(i - RR - (forced ? 0 : nb * kTmBody)) * kls] = (i == k) ? 1.0 : 0.0;

    unsigned qmin = 0xffffffffu;
    const StagedStep<kBasis> SB{R, n, lane, 0};
    const StagedStep<kForcedSingle> SF{R, n, lane, 0};
#ifdef PINT_HEAT_PROF
    unsigned long long prof[6] = {0, 0, 0, 0, 0, 0};
    long long t_prev = clock64();
#endif
    if (wlive) {
        for (long long s = 0; s < steps; ++s) {
            const unsigned parity = static_cast<unsigned>(s & 1);
            mbar_wait(bar_f, parity);
            HEAT_PROF_MARK(0);
            double d, dm1 = 0.0;
            if (forced) d = column_forward<RR, kForcedSingle, kGuard>(reg, st, SF, dm1, qmin);
            else d = column_forward<RR, kBasis, kGuard, 32, true, kNs>(reg, st, SB, dm1, qmin, tm, nb);
            qmin = min(qmin, hi_abs(d) - 1u);
            HEAT_PROF_MARK(1);
            __syncwarp();
            if (lane == 0) {  // the last of the CTA's live warps to finish the forward half refills it
                __threadfence_block();
                if (atomicAdd(cnt, 1u) % nlive == static_cast<unsigned>(nlive - 1) && s + 1 < steps) load_fwd(s + 1);
            }
            mbar_wait(bar_b, parity);
            HEAT_PROF_MARK(2);
            if (forced) column_back<RR, kForcedSingle>(reg, st, SF, d, dm1, qmin);
            else column_back<RR, kBasis, 32, true, kNs>(reg, st, SB, d, dm1, qmin, tm, nb);
            HEAT_PROF_MARK(3);
            __syncwarp();
            if (lane == 0) {
                __threadfence_block();
                if (atomicAdd(cnt + 1, 1u) % nlive == static_cast<unsigned>(nlive - 1) && s + 1 < steps) {
                    load_back(s + 1);
                    if (s + 2 < steps) prefetch_l2(V.rec(slice, s + 2), 8u * static_cast<unsigned>(record_stride(n)));
                }
            }
            HEAT_PROF_MARK(4);
        }
#ifdef PINT_HEAT_PROF
        if (threadIdx.x == 0 && blockIdx.x < (1 << 14)) {
            for (int q = 0; q < 5; ++q) g_heat_prof[blockIdx.x][q] = prof[q];
            g_heat_span[0][blockIdx.x][0] = t_start;
            g_heat_span[0][blockIdx.x][1] = pint_dev::globaltimer();
        }
#endif
        const bool live = forced ? lane == 0 : k < n;
        double* gp = P.maps + slice * n * P.ldm + k;
        if (live) {
#pragma unroll
            for (int i = 0; i < RR; ++i) gp[i * P.ldm] = reg[i];
        }
        long long i0 = RR;
        if (!forced) {
            tm_wait_st();
            for (int ch = 0; ch < nb * (kTmBody / 8); ++ch) {
                Tm8 t;
                tm_ld(tm + 16u * ch, t);
                tm_wait_ld(t);
                if (live) {
#pragma unroll
                    for (int u = 0; u < 8; ++u) gp[(RR + 8 * ch + u) * P.ldm] = t.get(u);
                }
            }
            i0 += nb * kTmBody;
        }
        if (live) {
            for (long long i = i0; i < n; ++i) gp[i * P.ldm] = st[(i - i0) * kls];
            if (!kGuard && qmin < kQuotLo - 1u) record_failure(P.fail, kRetryIndex + slice, PINT_E_RANGE_RETRY, 0.0);
        }
        if (P.per_slice_ns && lane == 0) atomicAdd(P.per_slice_ns + slice, pint_dev::globaltimer() - t_start);
#ifdef PINT_HEAT_PROF
        if (threadIdx.x == 0 && blockIdx.x < (1 << 14)) g_heat_span[1][blockIdx.x][0] = pint_dev::globaltimer();  // epilogue end
#endif
    }
    tm_wait_st();
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(*tslot) : "memory");
    // this CTA's columns of the map are stored: count it (a chain consuming maps as they complete
    // waits for cps counts, launch_heat_build_chain)
    if (P.ready && threadIdx.x == 0) {
        __threadfence();
        atomicAdd(P.ready + slice, 1);
        atomicMin(P.span, t_start);
        atomicMax(P.span + 1, pint_dev::globaltimer());
    }
#ifdef PINT_HEAT_PROF
    if (threadIdx.x == 0 && blockIdx.x < (1 << 14)) g_heat_span[1][blockIdx.x][1] = pint_dev::globaltimer();  // CTA end
#endif
}

// ---- forced columns apart (TMEM range): one lane per slice --------------------------------------
// Column n of every slice's map (the forced run from 0, pde_problems.cpp:91-94) for the TMEM build,
// which then builds the basis columns only: a 5th warp in CTA 0 of every slice shared sub-partition
// 0 with basis warp 0 and made CTA 0 the slowest of its slice (basis-only build 32.4 against
// 34.6 ms). Here lane l of a one-warp CTA runs slice 32 blockIdx + l: the operations, in the
// order, of the in-CTA forced warp (column_forward / column_back in kForcedSingle mode), its state
// in registers (rows 0 .. kFlRegRows-1) and lane-interleaved shared memory. The 32 slices' records
// stream through a two-slot shared ring in 64-row chunks by TMA: the slice-major records seen as
// 4-D tensors {16 doubles, slices, 16-double blocks, steps} (strides S·RS, 128 B, RS: RS = record
// doubles) over their (p, rcp), h b and c regions, one box {16, 32, blocks, 1} per region and
// chunk with the 128-byte swizzle — [block][lane][16], so lane l's row r sits at 16-byte chunk
// (r % 8) ^ (l % 8) of its line: conflict-free. (Per-lane loads from global memory left the chain
// waiting on DRAM, 1.4 ms; per-lane bulk copies needed a 32-way issue loop each, 1.1 ms.)
constexpr int kFlRegRows = 64, kFlChunk = 64;
constexpr unsigned kFlPrBytes = 16 * 32 * 8 * 8, kFlHbBytes = 16 * 32 * 4 * 8;  // a chunk's boxes
constexpr unsigned kFlSlot = kFlPrBytes + kFlHbBytes;                            // 48 KB

__host__ __device__ constexpr int fl_chunks(long long n) { return static_cast<int>((n16(n) + kFlChunk - 1) / kFlChunk); }
size_t forced_lanes_smem(long long n) {
    return 1024 + 2 * kFlSlot + sizeof(double) * 32 * static_cast<size_t>(n - kFlRegRows) + 16;
}

template <bool kGuard>
__global__ void __launch_bounds__(32, 1) heat_forced_lanes_kernel(const __grid_constant__ BuildPlan P) {
    extern __shared__ __align__(1024) unsigned char fl_raw[];
    unsigned char* fl = fl_raw + ((((smem_u32(fl_raw) + 1023u) & ~1023u) - smem_u32(fl_raw)));
    const int n = P.n, lane = threadIdx.x;
    const long long slice = static_cast<long long>(blockIdx.x) * 32 + lane;
    const bool live = slice < P.N;
    const long long steps = live ? P.step_off[slice + 1] - P.step_off[slice] : 0;
    const unsigned long long t_start = pint_dev::globaltimer();
    const RecView V = rec_view(P.rec, n, P.N, P.S);
    const unsigned ring0 = smem_u32(fl);                                            // [2][48 KB]
    double* st = reinterpret_cast<double*>(fl + 2 * kFlSlot) + lane;                // row i at st[32 (i - RR)]
    const unsigned bar0 = smem_u32(fl + 2 * kFlSlot + sizeof(double) * 32 * static_cast<size_t>(n - kFlRegRows));
    if (lane == 0) {
        mbar_init(bar0);
        mbar_init(bar0 + 8);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncwarp();
    long long max_steps = steps;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) max_steps = max(max_steps, __shfl_xor_sync(0xffffffffu, max_steps, o));
    const int nch = fl_chunks(n);
    const int sl0 = static_cast<int>(blockIdx.x) * 32;
    // task t of a step: t < nch forward chunk t, else back chunk 2 nch - 1 - t; task q = s 2 nch + t
    // runs through slot q % 2
    auto issue = [&](long long q) {  // (lane 0)
        const long long s = q / (2 * nch);
        const int t = static_cast<int>(q - s * 2 * nch);
        const bool fwd = t < nch;
        const int c = fwd ? t : 2 * nch - 1 - t;
        const unsigned bar = bar0 + 8u * static_cast<unsigned>(q & 1), dst = ring0 + static_cast<unsigned>(q & 1) * kFlSlot;
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // (the slot's earlier reads)
        asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(bar),
                     "r"(fwd ? kFlSlot : kFlHbBytes)
                     : "memory");
        auto tma = [&](const CUtensorMap* m, unsigned d, int blk) {
            asm volatile(
                "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
                "%3, %4, %5}], [%6];\n" ::"r"(d),
                "l"(reinterpret_cast<unsigned long long>(m)), "r"(0), "r"(sl0), "r"(blk), "r"(static_cast<int>(s)),
                "r"(bar)
                : "memory");
        };
        if (fwd) {
            tma(&P.tm_pr, dst, 8 * c);
            tma(&P.tm_hb, dst + kFlPrBytes, 4 * c);
        } else {
            tma(&P.tm_cc, dst, 4 * c);
        }
    };
    const int sw = lane & 7;
    // a chunk's row r: (p, rcp) at [r / 8][lane][(r % 8) ^ sw]; h b, c at [r / 16][lane][((r % 16) / 2) ^ sw] + r % 2
    auto pr_at = [&](const unsigned char* T, int r) {
        return *reinterpret_cast<const double2*>(T + ((r >> 3) * 32 + lane) * 128 + (((r & 7) ^ sw) << 4));
    };
    auto v_at = [&](const unsigned char* T, int r) {
        return *reinterpret_cast<const double*>(T + ((r >> 4) * 32 + lane) * 128 + ((((r & 15) >> 1) ^ sw) << 4) +
                                                ((r & 1) << 3));
    };
    double reg[kFlRegRows];
#pragma unroll
    for (int i = 0; i < kFlRegRows; ++i) reg[i] = 0.0;  // the forced run starts at 0
    for (int i = kFlRegRows; i < n; ++i) st[32 * (i - kFlRegRows)] = 0.0;
    unsigned qmin = 0xffffffffu;
    auto divide = [&](double num, double2 pr) { return kGuard ? div_guarded(num, pr) : div_fast(num, pr); };
    const long long total = max_steps * 2 * nch;
    if (lane == 0) {
        if (total > 0) issue(0);
        if (total > 1) issue(1);
    }
    long long q = 0;
    auto wait_task = [&]() -> const unsigned char* {  // task q's slot (landed)
        mbar_wait(bar0 + 8u * static_cast<unsigned>(q & 1), static_cast<unsigned>((q >> 1) & 1));
        return fl + static_cast<size_t>(q & 1) * kFlSlot;
    };
    auto done_task = [&]() {  // the slot is consumed: load task q + 2 into it
        __syncwarp();
        if (lane == 0 && q + 2 < total) issue(q + 2);
        ++q;
    };
    for (long long s = 0; s < max_steps; ++s) {
        const bool act = s < steps;  // (a shorter slice's lane computes nothing at the tail)
        const double negr = act ? V.rec(slice, s)[0] : 0.0;
        // forward (linalg.cpp:84-90) with the forcing increment x + h b first (pde_problems.cpp:93)
        double d = -0.0;
        for (int c = 0; c < nch; ++c) {
            const unsigned char* T = wait_task();
            const unsigned char* H = T + kFlPrBytes;
            const int r0 = c * kFlChunk, r1 = min(n, r0 + kFlChunk);
            if (act) {
                if (r0 < kFlRegRows) {  // (the register rows: chunk 0, kFlRegRows == kFlChunk)
#pragma unroll
                    for (int i = 0; i < kFlRegRows; ++i) {
                        const double x = __dadd_rn(reg[i], v_at(H, i));
                        d = divide((i == 0) ? x : __dsub_rn(x, __dmul_rn(negr, d)), pr_at(T, i));
                        reg[i] = d;
                        qmin = min(qmin, hi_abs(d) - 1u);
                    }
                } else if (r1 - r0 == kFlChunk) {  // a full chunk: straight-line, every address fixed
                    const unsigned char* pk[8];  // this lane's swizzled 16-byte chunk k of a 128-byte line
                    const unsigned char* hk[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) pk[k] = T + lane * 128 + ((k ^ sw) << 4), hk[k] = H + lane * 128 + ((k ^ sw) << 4);
                    auto PRr = [&](int r) { return *reinterpret_cast<const double2*>(pk[r & 7] + (r >> 3) * 4096); };
                    auto HBr = [&](int r) {
                        return *reinterpret_cast<const double*>(hk[(r & 15) >> 1] + (r >> 4) * 4096 + (r & 1) * 8);
                    };
                    double* sp = st + 32 * (r0 - kFlRegRows);
                    constexpr int A = 4;  // operands A rows ahead, each loaded before the store in front of it
                    double2 pv[A];
                    double hv[A], xv[A];
#pragma unroll
                    for (int u = 0; u < A; ++u) pv[u] = PRr(u), hv[u] = HBr(u), xv[u] = sp[32 * u];
#pragma unroll
                    for (int r = 0; r < kFlChunk; ++r) {
                        const int u = r % A;
                        const double x = __dadd_rn(xv[u], hv[u]);
                        d = divide(__dsub_rn(x, __dmul_rn(negr, d)), pv[u]);
                        if (r + A < kFlChunk) pv[u] = PRr(r + A), hv[u] = HBr(r + A), xv[u] = sp[32 * (r + A)];
                        sp[32 * r] = d;
                        qmin = min(qmin, hi_abs(d) - 1u);
                    }
                } else {  // (a partial last chunk)
                    for (int i = r0; i < r1; ++i) {
                        const double x = __dadd_rn(st[32 * (i - kFlRegRows)], v_at(H, i - r0));
                        d = divide(__dsub_rn(x, __dmul_rn(negr, d)), pr_at(T, i - r0));
                        st[32 * (i - kFlRegRows)] = d;
                        qmin = min(qmin, hi_abs(d) - 1u);
                    }
                }
            }
            done_task();
        }
        // back substitution (linalg.cpp:91): x_{n-1} = q_{n-1}; x_i = q_i - c_i x_{i+1}
        for (int c = nch - 1; c >= 0; --c) {
            const unsigned char* T = wait_task();
            const int r0 = c * kFlChunk, r1 = min(n - 2, r0 + kFlChunk - 1);  // rows r1 .. r0, top n - 2
            if (act) {
                if (r0 < kFlRegRows) {
#pragma unroll
                    for (int k = kFlRegRows - 1; k >= 0; --k) {
                        d = __dsub_rn(reg[k], __dmul_rn(v_at(T, k), d));
                        reg[k] = d;
                    }
                } else if (r1 - r0 == kFlChunk - 1) {  // a full chunk: straight-line, every address fixed
                    const unsigned char* ck[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) ck[k] = T + lane * 128 + ((k ^ sw) << 4);
                    auto CCr = [&](int r) {
                        return *reinterpret_cast<const double*>(ck[(r & 15) >> 1] + (r >> 4) * 4096 + (r & 1) * 8);
                    };
                    double* sp = st + 32 * (r0 - kFlRegRows);
                    constexpr int A = 8;
                    double yv[A], cv[A];
#pragma unroll
                    for (int u = 0; u < A; ++u) yv[u] = sp[32 * (kFlChunk - 1 - u)], cv[u] = CCr(kFlChunk - 1 - u);
#pragma unroll
                    for (int r = kFlChunk - 1; r >= 0; --r) {
                        const int u = (kFlChunk - 1 - r) % A;
                        d = __dsub_rn(yv[u], __dmul_rn(cv[u], d));
                        if (r - A >= 0) yv[u] = sp[32 * (r - A)], cv[u] = CCr(r - A);
                        sp[32 * r] = d;
                    }
                } else {  // (a partial chunk: the top one, ending at row n - 2)
                    for (int i = r1; i >= r0; --i) {
                        d = __dsub_rn(st[32 * (i - kFlRegRows)], __dmul_rn(v_at(T, i - r0), d));
                        st[32 * (i - kFlRegRows)] = d;
                    }
                }
            }
            done_task();
        }
    }
    if (live) {
        double* gp = P.maps + slice * n * P.ldm + n;
#pragma unroll
        for (int k = 0; k < kFlRegRows; ++k) gp[k * P.ldm] = reg[k];
        for (int k = kFlRegRows; k < n; ++k) gp[k * P.ldm] = st[32 * (k - kFlRegRows)];
        if (!kGuard && qmin < kQuotLo - 1u) record_failure(P.fail, kRetryIndex + slice, PINT_E_RANGE_RETRY, 0.0);
        if (P.per_slice_ns) atomicAdd(P.per_slice_ns + slice, pint_dev::globaltimer() - t_start);
    }
}

// ---- integrate: K caller columns through consecutive steps of ONE slice ------------------------
// The integrate closure (pde_problems.cpp:86-98) and run_serial (nievergelt.cpp:126-143): the same
// bit-exact row recurrence as the build, one warp per 32 caller columns (lane = column; a single
// trajectory runs on lane 0 with the others idle), rows [0, RR) in registers and the rest
// lane-interleaved in shared memory, each step's slice-major record (forward half: header, (p,
// rcp), h*b; back half: c) staged by two bulk copies — the back half while the forward pass runs,
// the next forward half while the back pass runs, the step after next pulled into L2. Steps go in
// bounded chunks (launch_heat_integrate_steps): the records of one chunk at a time.
struct IntegPlan {
    int n;
    long long K, steps;  // columns; steps of this chunk (records [0, steps) of `rec`)
    const double* rec;
    double* y;           // [K][n], in place
    FailRec* fail;
    long long fail_base;  // step index of the chunk's first step (range-retry index)
    // per-slice mode (parareal's fine wave): CTA b runs ONE column (y + b n, lane 0) through its own
    // records rec + b rec_cta_stride, cta_steps[b] steps
    long long rec_cta_stride;
    const int64_t* cta_steps;
};

// One warp's state and staging for the integrate loops: rows [0, RR) of this lane's column in reg,
// the rest at st[32 (i - RR)], the step's record staged at R0 (forward half at 0, back half at
// cc_offset) completing on bar0 / bar0 + 8; `ph` counts the steps run through these barriers.
template <int RR>
struct IntegWarp {
    double reg[RR > 0 ? RR : 1];
    double* st;
    double* R0;
    unsigned bar0;
    long long ph = 0;
    unsigned qmin = 0xffffffffu;
};

// `steps` consecutive steps whose slice-major records start at `rec` (the caller's warp, all lanes)
template <int RR, int kMode, bool kGuard>
__device__ __forceinline__ void integ_run(IntegWarp<RR>& W, int n, const double* rec, long long steps) {
    const int lane = threadIdx.x & 31;
    const unsigned fwd_bytes = 8u * static_cast<unsigned>(cc_offset(n));  // header, (p, rcp), h*b
    const unsigned back_bytes = 8u * static_cast<unsigned>(even(n));
    auto recs = [&](long long s) { return rec + s * record_stride(n); };
    __syncwarp();
    if (lane == 0 && steps > 0) {
        bulk_load(smem_u32(W.R0), recs(0), fwd_bytes, W.bar0);
        bulk_load(smem_u32(W.R0 + cc_offset(n)), recs(0) + cc_offset(n), back_bytes, W.bar0 + 8u);
        if (steps > 1) prefetch_l2(recs(1), 8u * static_cast<unsigned>(record_stride(n)));
    }
    for (long long s = 0; s < steps; ++s, ++W.ph) {
        const unsigned parity = static_cast<unsigned>(W.ph & 1);
        const StagedStep<kMode> SV{W.R0, n, lane, 0};
        mbar_wait(W.bar0, parity);
        double dm1 = 0.0;
        double d = column_forward<RR, kMode, kGuard>(W.reg, W.st, SV, dm1, W.qmin);
        W.qmin = min(W.qmin, hi_abs(d) - 1u);
        __syncwarp();  // every lane is done with the forward half
        if (lane == 0 && s + 1 < steps) bulk_load(smem_u32(W.R0), recs(s + 1), fwd_bytes, W.bar0);
        mbar_wait(W.bar0 + 8u, parity);
        column_back<RR, kMode>(W.reg, W.st, SV, d, dm1, W.qmin);
        __syncwarp();
        if (lane == 0 && s + 1 < steps) {
            bulk_load(smem_u32(W.R0 + cc_offset(n)), recs(s + 1) + cc_offset(n), back_bytes, W.bar0 + 8u);
            if (s + 2 < steps) prefetch_l2(recs(s + 2), 8u * static_cast<unsigned>(record_stride(n)));
        }
    }
}

template <int RR, int kMode>
__device__ __forceinline__ void integ_setup(IntegWarp<RR>& W, int n, double* smem) {
    const int lane = threadIdx.x & 31;
    W.R0 = smem + front_pad(n, kMode);
    W.st = W.R0 + staged_doubles(n, kMode) + lane;
    W.bar0 = smem_u32(W.R0 + staged_doubles(n, kMode) + (n - RR) * 32 + 32 * kFwdAhead);
    if (lane == 0) {
        mbar_init(W.bar0);
        mbar_init(W.bar0 + 8u);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncwarp();
}

template <int RR>
__device__ __forceinline__ void integ_load(IntegWarp<RR>& W, int n, const double* y, bool live) {
#pragma unroll
    for (int i = 0; i < RR; ++i) W.reg[i] = live ? y[i] : 0.0;
    for (int i = RR; i < n; ++i) W.st[(i - RR) * 32] = live ? y[i] : 0.0;
}

template <int RR>
__device__ __forceinline__ void integ_store(IntegWarp<RR>& W, int n, double* y) {
#pragma unroll
    for (int i = 0; i < RR; ++i) y[i] = W.reg[i];
    for (int i = RR; i < n; ++i) y[i] = W.st[(i - RR) * 32];
}

template <int RR, int kMode, bool kGuard>
__global__ void __maxnreg__(255) heat_integrate_kernel(const IntegPlan P) {
    static_assert(kMode == kBasis || kMode == kBasisForced, "integrate modes");
    extern __shared__ __align__(128) double smem[];
    const int n = P.n;
    const int lane = threadIdx.x;
    const bool per_slice = P.cta_steps != nullptr;
    const long long col = per_slice ? blockIdx.x : static_cast<long long>(blockIdx.x) * 32 + lane;
    const bool live = col < P.K && (!per_slice || lane == 0);
    IntegWarp<RR> W;
    integ_setup<RR, kMode>(W, n, smem);
    integ_load<RR>(W, n, P.y + (live ? col : 0) * n, live);
    const long long steps = per_slice ? P.cta_steps[blockIdx.x] : P.steps;
    integ_run<RR, kMode, kGuard>(W, n, P.rec + (per_slice ? blockIdx.x * P.rec_cta_stride : 0), steps);
    if (live) {
        integ_store<RR>(W, n, P.y + col * n);
        if (!kGuard && W.qmin < kQuotLo - 1u) record_failure(P.fail, kRetryIndex + P.fail_base, PINT_E_RANGE_RETRY, 0.0);
    }
}

// ---- parareal's sequential correction sweep on the device (parareal.cpp:71-81, :103-117) -------
// One warp, one column (lane 0): for every slice j, G(next_j) = the coarse steps of slice j (records
// rec + j rec_stride, steps[j]); iteration 0 (fout null) stores lambda_{j+1} = g_prev_j = G, later
// iterations lambda_{j+1} = (G + fout_j) - g_prev_j and g_prev_j = G — the reference's combine, row by
// row on lane 0 (rounded exactly as g_new[i] + f[i] - g_old[i]).
struct CoarsePlan {
    int n;
    long long N;
    const double* rec;
    long long rec_stride;
    const int64_t* steps;
    const double* y0;
    const double* fout;  // [N][n] fine endpoints of this iteration, or null (iteration 0)
    double* gprev;       // [N][n]
    double* lam;         // [N + 1][n]
    FailRec* fail;
};

template <int RR, bool kGuard>
__global__ void __maxnreg__(255) heat_parareal_coarse_kernel(const CoarsePlan P) {
    extern __shared__ __align__(128) double smem[];
    constexpr int kMode = kBasisForced;
    const int n = P.n;
    const int lane = threadIdx.x;
    IntegWarp<RR> W;
    integ_setup<RR, kMode>(W, n, smem);
    integ_load<RR>(W, n, P.y0, lane == 0);
    if (lane == 0)
        for (int i = 0; i < n; ++i) P.lam[i] = P.y0[i];
    for (long long j = 0; j < P.N; ++j) {
        integ_run<RR, kMode, kGuard>(W, n, P.rec + j * P.rec_stride, P.steps[j]);
        if (lane == 0) {  // g_new = the state; next = g_new + f - g_old (or g_new at iteration 0)
            double* gp = P.gprev + j * n;
            double* lm = P.lam + (j + 1) * n;
            const double* f = P.fout ? P.fout + j * n : nullptr;
#pragma unroll
            for (int i = 0; i < RR; ++i) {
                const double g = W.reg[i];
                const double nx = f ? __dsub_rn(__dadd_rn(g, f[i]), gp[i]) : g;
                gp[i] = g;
                lm[i] = nx;
                W.reg[i] = nx;
            }
            for (int i = RR; i < n; ++i) {
                const double g = W.st[(i - RR) * 32];
                const double nx = f ? __dsub_rn(__dadd_rn(g, f[i]), gp[i]) : g;
                gp[i] = g;
                lm[i] = nx;
                W.st[(i - RR) * 32] = nx;
            }
        }
        __syncwarp();
    }
    if (lane == 0 && !kGuard && W.qmin < kQuotLo - 1u) record_failure(P.fail, kRetryIndex, PINT_E_RANGE_RETRY, 0.0);
}

template <int RR, int kMode, bool kGuard>
int launch_integ(pint_ctx* ctx, cudaStream_t stream, const IntegPlan& P) {
    const size_t smem = sizeof(double) * warp_smem_doubles(P.n, kMode);
    if (smem > 227 * 1024) return pint_set_error(ctx, PINT_E_INVALID, "heat_integrate: n too large for shared memory");
    auto kern = heat_integrate_kernel<RR, kMode, kGuard>;
    pint_kernel_attrs(reinterpret_cast<const void*>(kern));
    const long long ctas = P.cta_steps ? P.K : (P.K + 31) / 32;
    kern<<<static_cast<unsigned>(ctas), 32, smem, stream>>>(P);
    return pint_check_launch(ctx, "heat_integrate_kernel");
}

template <int RR>
int launch_integ_rr(pint_ctx* ctx, cudaStream_t stream, const IntegPlan& P, bool forcing, bool guarded) {
    if (forcing)
        return guarded ? launch_integ<RR, kBasisForced, true>(ctx, stream, P)
                       : launch_integ<RR, kBasisForced, false>(ctx, stream, P);
    return guarded ? launch_integ<RR, kBasis, true>(ctx, stream, P) : launch_integ<RR, kBasis, false>(ctx, stream, P);
}

template <class K>
void smem_attrs(K kern, size_t) {
    pint_kernel_attrs(reinterpret_cast<const void*>(kern));
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

// heat_forced_lanes_kernel's tensors: the slice-major records (record j * S + s at j S RS + s RS
// doubles) seen per region as {16 doubles, slices, 16-double blocks, steps}
int make_fl_maps(pint_ctx* ctx, BuildPlan& P) {
    auto enc = tensor_map_encoder();
    if (!enc) return pint_set_error(ctx, PINT_E_CUDA, "heat_forced_lanes: cuTensorMapEncodeTiled unavailable");
    const long long RS = record_stride(P.n);
    const cuuint32_t e1[4] = {1, 1, 1, 1};
    auto make = [&](CUtensorMap* m, long long off, long long blocks, cuuint32_t box_blocks) {
        const cuuint64_t dims[4] = {16, static_cast<cuuint64_t>(P.N), static_cast<cuuint64_t>(blocks),
                                    static_cast<cuuint64_t>(P.S)};
        const cuuint64_t str[3] = {static_cast<cuuint64_t>(8 * P.S * RS), 128, static_cast<cuuint64_t>(8 * RS)};
        const cuuint32_t box[4] = {16, 32, box_blocks, 1};
        return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(P.rec + off), dims, str, box, e1,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    };
    const long long nb = n16(P.n) / 16;
    if (!make(&P.tm_pr, pr_offset(), 2 * nb, 8) || !make(&P.tm_hb, hb_offset(P.n), nb, 4) ||
        !make(&P.tm_cc, cc_offset(P.n), nb, 4))
        return pint_set_error(ctx, PINT_E_CUDA, "heat_forced_lanes: tensor map failed");
    return PINT_OK;
}

// The kBasisGroup tiles: pr2 as [blocks][n16+1][64] doubles (box 2 x (n+1) x 1: one slice's
// (-r, 0), (p, rcp) column) and c as [blocks][n16][32] doubles (box 2 x n x 1: two slices' c).
int make_tile_maps(pint_ctx* ctx, BuildPlan& P) {
    auto enc = tensor_map_encoder();
    if (!enc) return pint_set_error(ctx, PINT_E_CUDA, "heat_build: cuTensorMapEncodeTiled unavailable");
    const cuuint64_t blocks = static_cast<cuuint64_t>(P.S * groups32(P.N));
    const cuuint64_t bstride = static_cast<cuuint64_t>(8 * fblock_stride(P.n));
    const cuuint32_t estr[3] = {1, 1, 1};
    {
        const cuuint64_t dims[3] = {64, static_cast<cuuint64_t>(n16(P.n) + 1), blocks};
        const cuuint64_t strides[2] = {64 * 8, bstride};
        const cuuint32_t box[3] = {2, static_cast<cuuint32_t>(P.n + 1), 1};
        if (enc(&P.tm_pr, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(P.rec), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return pint_set_error(ctx, PINT_E_CUDA, "heat_build: tensor map (p, rcp) failed");
    }
    {
        const cuuint64_t dims[3] = {32, static_cast<cuuint64_t>(n16(P.n)), blocks};
        const cuuint64_t strides[2] = {32 * 8, bstride};
        const cuuint32_t box[3] = {2, static_cast<cuuint32_t>(P.n), 1};
        if (enc(&P.tm_cc, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(P.rec + fblock_cc(P.n)), dims,
                strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return pint_set_error(ctx, PINT_E_CUDA, "heat_build: tensor map (c) failed");
    }
    return PINT_OK;
}

template <int RR, bool kGuard>
int launch_build(pint_ctx* ctx, BuildPlan P) {
    const bool grp = group_forced(P.n);
    const size_t smem = sizeof(double) * warp_smem_doubles(P.n, grp ? kBasisGroup : kBasis);
    size_t fsmem = sizeof(double) * warp_smem_doubles(P.n, grp ? kForcedGroup : kForcedSingle);
    // a group-forced warp is the longest chain of the launch: reserve enough shared memory that at
    // most 3 basis CTAs share its SM (one warp per sub-partition); the basis grid still fits
    if (grp) fsmem = std::max(fsmem, std::min<size_t>(227 * 1024, 228 * 1024 - 4 * (smem + 1024)) & ~size_t(127));
    if (smem > 227 * 1024 || fsmem > 227 * 1024)
        return pint_set_error(ctx, PINT_E_INVALID, "heat_build: n too large for shared memory");
    if (grp)
        if (const int rc = make_tile_maps(ctx, P)) return rc;
    auto kern = grp ? heat_build_kernel<RR, kBasisGroup, kGuard> : heat_build_kernel<RR, kBasis, kGuard>;
    auto fkern = grp ? heat_build_kernel<RR, kForcedGroup, kGuard> : heat_build_kernel<RR, kForcedSingle, kGuard>;
    smem_attrs(kern, smem);
    smem_attrs(fkern, fsmem);
    // forced columns first, then the basis grid with programmatic stream serialization: the
    // forced CTAs trigger it once resident, so both grids run together on one stream
    // PINT_HEAT_ONLY=basis|forced: timing experiments only (the other part of the maps is not built)
    const char* only = std::getenv("PINT_HEAT_ONLY");
    const bool run_f = !only || std::strcmp(only, "basis") != 0, run_b = !only || std::strcmp(only, "forced") != 0;
    if (run_f) fkern<<<static_cast<unsigned>(grp ? 2 * groups32(P.N) : P.N), 32, fsmem, ctx->stream>>>(P);
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

void* pint_tensor_map_encoder() { return reinterpret_cast<void*>(tensor_map_encoder()); }

int64_t heat_records_doubles(int64_t n, int64_t N, int64_t S) { return records_doubles(n, N, S); }

int launch_heat_factor_range(pint_ctx* ctx, int64_t n, int64_t N, int64_t S, int64_t j0, int64_t Nc,
                             const int64_t* step_off, const double* slice_dt, const double* r, const double* fa,
                             const double* fb, const double* sx, double* records) {
    return launch_heat_factor_block(ctx, ctx->stream, n, N, S, j0, Nc, 0, S, 0, step_off, slice_dt, r, fa, fb, sx,
                                    records);
}

int launch_heat_factor_block(pint_ctx* ctx, cudaStream_t stream, int64_t n, int64_t N, int64_t S, int64_t j0,
                             int64_t Nc, int64_t s0, int64_t Sc, int64_t tab_pitch, const int64_t* step_off,
                             const double* slice_dt, const double* r, const double* fa, const double* fb,
                             const double* sx, double* records, int64_t rec_s0, bool slice_major) {
    if (n < 1 || N < 0 || S < 0 || j0 < 0 || Nc < 0 || j0 + Nc > N || s0 < rec_s0 || Sc < 0 || s0 + Sc > rec_s0 + S)
        return pint_set_error(ctx, PINT_E_INVALID, "heat_factor: bad sizes");
    if (Nc == 0 || Sc == 0) return PINT_OK;
    const long long threads = Nc * Sc;
    heat_record_kernel<<<static_cast<unsigned>((threads + 127) / 128), 128, 0, stream>>>(
        static_cast<int>(n), N, S, j0, Nc, s0, Sc, tab_pitch, rec_s0, slice_major, step_off, slice_dt, r, fa, fb, sx, records, ctx->d_fail);
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
    (void)slice_dt;  // the per-slice step lives in the records (h*b) and step_off
    (void)sx;
    return launch_heat_build_steps(ctx, n, N, S, step_off, records, maps, per_slice_ns, guarded, 0, S);
}

bool heat_build_segmentable(int64_t n) { return n >= 1 && !use_tmem(n); }

// The TMEM build's forced columns: the lanes kernel above (PINT_FORCED_LANES=0: the in-CTA warp)
bool tmem_forced_lanes(long long n) {
    static const int v = [] {
        const char* e = std::getenv("PINT_FORCED_LANES");
        return e ? std::atoi(e) : 1;
    }();
    return v != 0 && n > kFlRegRows + 2 && forced_lanes_smem(n) <= 227 * 1024;
}

void heat_build_prepare(int64_t n) {
    if (use_tmem(n)) {
        smem_attrs(heat_build_tmem_kernel<false>, 0);
        smem_attrs(heat_build_tmem_kernel<true>, 0);
        smem_attrs(heat_build_tmem_kernel<false, 512>, 0);
        smem_attrs(heat_build_tmem_kernel<true, 512>, 0);
        smem_attrs(heat_forced_lanes_kernel<false>, 0);
        smem_attrs(heat_forced_lanes_kernel<true>, 0);
    }
}

// heat_build_chain: the forced columns ahead of the chain (nothing may sit between the chain and
// the build it waits on); returns PINT_OK without launching when the in-CTA warp builds them.
int launch_heat_forced_first(pint_ctx* ctx, int64_t n, int64_t N, int64_t S, const int64_t* step_off,
                             const double* records, double* maps, unsigned long long* per_slice_ns, int guarded) {
    if (!use_tmem(n) || !tmem_forced_lanes(n) || N == 0) return PINT_OK;
    BuildPlan P{};
    P.s_begin = 0;
    P.s_end = S;
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
    if (const int rc = make_fl_maps(ctx, P)) return rc;
    auto fk = guarded ? heat_forced_lanes_kernel<true> : heat_forced_lanes_kernel<false>;
    fk<<<static_cast<unsigned>((N + 31) / 32), 32, forced_lanes_smem(n), ctx->stream>>>(P);
    return pint_check_launch(ctx, "heat_forced_lanes_kernel");
}

int heat_build_ready_target(int64_t n) { return use_tmem(n) ? static_cast<int>(((n + 31) / 32 + 3) / 4) : 0; }

int launch_heat_build_steps(pint_ctx* ctx, int64_t n, int64_t N, int64_t S, const int64_t* step_off,
                            const double* records, double* maps, unsigned long long* per_slice_ns, int guarded,
                            int64_t s_begin, int64_t s_end, int* ready) {
    if (n < 1 || N < 0 || s_begin < 0 || s_end < s_begin)
        return pint_set_error(ctx, PINT_E_INVALID, "heat_build: bad sizes");
    if (N == 0 || s_end == s_begin) return PINT_OK;
    if (n > (1 << 20) || N > (1 << 26)) return pint_set_error(ctx, PINT_E_INVALID, "heat_build: sizes out of range");
    if ((s_begin > 0 || s_end < S) && !heat_build_segmentable(n))
        return pint_set_error(ctx, PINT_E_INVALID, "heat_build: step segments need the register/shared-memory build");
    BuildPlan P{};
    P.s_begin = s_begin;
    P.s_end = s_end;
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
    P.ready = ready;
    if (const char* o = std::getenv("PINT_HEAT_ONLY")) P.only = std::strcmp(o, "basis") == 0 ? 1 : std::strcmp(o, "forced") == 0 ? 2 : 0;
    P.span = ready ? reinterpret_cast<unsigned long long*>(ready + ((N + 1) & ~1ll)) : nullptr;
    if (use_tmem(n)) {
        const size_t smem = sizeof(double) * tm_smem_doubles(n);
        static const bool static512 = [] {  // PINT_TM_STATIC=0: the runtime-n kernel at n = 512 too
            const char* e = std::getenv("PINT_TM_STATIC");
            return !e || std::atoi(e) != 0;
        }();
        auto kern = (n == 512 && static512)
                        ? (guarded ? heat_build_tmem_kernel<true, 512> : heat_build_tmem_kernel<false, 512>)
                        : (guarded ? heat_build_tmem_kernel<true> : heat_build_tmem_kernel<false>);
        smem_attrs(kern, smem);
        int threads = 160;
        if (tmem_forced_lanes(n) && P.only == 0) {
            // the forced columns first, 32 slices a warp (heat_forced_lanes_kernel); the TMEM grid then
            // runs 4 basis warps a CTA. With `ready` (the chain already waits on this stream) the
            // caller has launched the forced kernel ahead of the chain: heat_build_chain.
            if (!ready) {
                auto fk = guarded ? heat_forced_lanes_kernel<true> : heat_forced_lanes_kernel<false>;
                smem_attrs(fk, forced_lanes_smem(n));
                BuildPlan F = P;
                if (const int rc = make_fl_maps(ctx, F)) return rc;
                fk<<<static_cast<unsigned>((N + 31) / 32), 32, forced_lanes_smem(n), ctx->stream>>>(F);
                if (const int rc = pint_check_launch(ctx, "heat_forced_lanes_kernel")) return rc;
            }
            P.only = 1;
            threads = 128;
        }
        const long long ctas = N * ((P.wps + 3) / 4);
        if (!ready) {
            kern<<<static_cast<unsigned>(ctas), threads, smem, ctx->stream>>>(P);
            return pint_check_launch(ctx, "heat_build_tmem_kernel");
        }
        // signalling build: launched behind the waiting chain on the same stream, allowed to start
        // while it runs (programmatic stream serialization; the chain triggers at its start)
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(static_cast<unsigned>(ctas), 1, 1);
        cfg.blockDim = dim3(threads, 1, 1);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = ctx->stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, kern, P);
        return pint_check_launch(ctx, "heat_build_tmem_kernel");
    }
    static_assert(reg_rows(kRegRows + 2) == kRegRows, "reg_rows");
    if (reg_rows(n) == kRegRows)
        return guarded ? launch_build<kRegRows, true>(ctx, P) : launch_build<kRegRows, false>(ctx, P);
    return guarded ? launch_build<0, true>(ctx, P) : launch_build<0, false>(ctx, P);
}

int64_t heat_integrate_chunk(int64_t n) {  // steps per chunk: ~16 MB of records
    return std::max<int64_t>(16, (int64_t{2} << 20) / record_stride(n));
}

int64_t heat_integrate_records_doubles(int64_t n) { return heat_integrate_chunk(n) * record_stride(n); }

int64_t heat_record_stride(int64_t n) { return record_stride(n); }

int launch_heat_integrate_slices(pint_ctx* ctx, int64_t n, int64_t N, const int64_t* steps, const double* records,
                                 int64_t rec_slice_stride, double* y, int guarded) {
    if (n < 1 || N < 0) return pint_set_error(ctx, PINT_E_INVALID, "heat_integrate_slices: bad sizes");
    if (N == 0) return PINT_OK;
    const IntegPlan P{static_cast<int>(n), N, 0, records, y, ctx->d_fail, 0, rec_slice_stride, steps};
    return reg_rows(n) == kRegRows ? launch_integ_rr<kRegRows>(ctx, ctx->stream, P, true, guarded != 0)
                                   : launch_integ_rr<0>(ctx, ctx->stream, P, true, guarded != 0);
}

template <int RR, bool kGuard>
int launch_coarse(pint_ctx* ctx, const CoarsePlan& P) {
    const size_t smem = sizeof(double) * warp_smem_doubles(P.n, kBasisForced);
    if (smem > 227 * 1024) return pint_set_error(ctx, PINT_E_INVALID, "parareal: n too large for shared memory");
    auto kern = heat_parareal_coarse_kernel<RR, kGuard>;
    pint_kernel_attrs(reinterpret_cast<const void*>(kern));
    kern<<<1, 32, smem, ctx->stream>>>(P);
    return pint_check_launch(ctx, "heat_parareal_coarse_kernel");
}

int launch_heat_parareal_coarse(pint_ctx* ctx, int64_t n, int64_t N, const double* records, int64_t rec_slice_stride,
                                const int64_t* steps, const double* y0, const double* fout, double* gprev, double* lam,
                                int guarded) {
    const CoarsePlan P{static_cast<int>(n), N, records, rec_slice_stride, steps, y0, fout, gprev, lam, ctx->d_fail};
    if (reg_rows(n) == kRegRows) return guarded ? launch_coarse<kRegRows, true>(ctx, P) : launch_coarse<kRegRows, false>(ctx, P);
    return guarded ? launch_coarse<0, true>(ctx, P) : launch_coarse<0, false>(ctx, P);
}

int launch_heat_integrate_steps(pint_ctx* ctx, cudaStream_t stream, int64_t n, int64_t K, int64_t steps,
                                int with_forcing, const double* records, double* y, FailRec* fail, int64_t fail_base,
                                int guarded) {
    if (n < 1 || K < 0 || steps < 0) return pint_set_error(ctx, PINT_E_INVALID, "heat_integrate: bad sizes");
    if (K == 0 || steps == 0) return PINT_OK;
    const IntegPlan P{static_cast<int>(n), K, steps, records, y, fail, fail_base, 0, nullptr};
    return reg_rows(n) == kRegRows ? launch_integ_rr<kRegRows>(ctx, stream, P, with_forcing != 0, guarded != 0)
                                   : launch_integ_rr<0>(ctx, stream, P, with_forcing != 0, guarded != 0);
}
