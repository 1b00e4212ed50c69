// K2 — per-slice interpolants and the sequential composition sweep.
//
//  * barycentric weights: interp.cpp:43-55 (product form, sequential divides, DuplicateNodes),
//    or the closed-form second-kind weights (EXTENSION, finite at M = 1024).
//  * scalar sweep: compose_sweep (nievergelt.cpp:68-88) applying interp_eval (interp.cpp:68-80)
//    slice after slice inside one CTA. EXACT mode keeps the reference's sequential
//    num/den accumulation (bit-exact); TREE mode reduces by warp tree (EXTENSION).
//  * bilinear sweep: EXTENSION for the 2-D tensor-grid maps, with bracket indices reported.
//
// Roofline: latency (the chain is sequential by construction); reported as time, not a fraction.
#include <algorithm>
#include <cstdlib>

#include "pint_internal.cuh"

namespace {

using pint_dev::record_failure;

// w_j = 1 / prod_{k != j} (x_j - x_k) as the reference's running quotient acc /= (x_j - x_k), k in
// order (interp.cpp:43-55). Each quotient must be the IEEE one; the chain runs M - 1 of them, so
// the divide is Markstein's exact sequence — q0 = acc * rcp, rem = fma(-d, q0, acc), q = fma(rem,
// rcp, q0) with rcp = RN(1/d) computed OFF the chain (it depends on the nodes only, bary_rcp_kernel):
// 3 dependent ops instead of a full division. Exact (the correctly rounded quotient) when nothing under- or
// overflows: |d| in [2^-60, 2^60] and |acc| in [2^-900, 2^900]; outside that window the step
// takes __ddiv_rn (acc grows like the product of the inverse spacings, so large M gets there).
__device__ __forceinline__ bool in_window(double v, unsigned lo_exp, unsigned hi_exp) {
    const unsigned a = static_cast<unsigned>(__double2hiint(v)) & 0x7fffffffu;
    return a - (lo_exp << 20) < ((hi_exp - lo_exp) << 20);
}

// The reciprocals depend on the nodes only: one massively parallel pass writes RN(1/(x_j - x_k))
// for every pair, k-major (so the chain kernel's loads, lanes = consecutive j, are coalesced).
__global__ void bary_rcp_kernel(long long M, const double* __restrict__ x, double* __restrict__ rcp) {
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= M * M) return;
    const long long k = t / M, j = t - k * M;
    rcp[t] = __drcp_rn(__dsub_rn(x[j], x[k]));
}

constexpr int kBaryChunk = 8;

__global__ void __launch_bounds__(32) bary_product_kernel(long long M, const double* __restrict__ x,
                                                          const double* __restrict__ rcp, double* __restrict__ w,
                                                          FailRec* fail) {
    extern __shared__ double xs[];  // the nodes, staged once per CTA
    for (long long k = threadIdx.x; k < M; k += blockDim.x) xs[k] = x[k];
    __syncwarp();
    const long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= M) return;
    const double xj = xs[j];
    double acc = 1.0;
    bool dup = false;
    // reciprocals three chunks ahead through three fixed register sets (a rotation by moves would
    // make every chunk wait for the loads it just issued)
    auto fetch = [&](long long k0, double (&r)[kBaryChunk]) {
#pragma unroll
        for (int u = 0; u < kBaryChunk; ++u) r[u] = __ldg(rcp + (k0 + u < M ? k0 + u : 0) * M + j);
    };
    // A chunk runs the exact fast sequence unconditionally (a skipped k — k == j or past M — divides
    // by d = 1 with r = 1: exact, acc unchanged) while tracking the windows; if any step left them,
    // the chunk is redone from its starting value with IEEE divisions. No branch on the chain.
    auto chunk = [&](long long k0, const double (&r)[kBaryChunk]) {
        double d[kBaryChunk], rr[kBaryChunk];
        bool use[kBaryChunk];
#pragma unroll
        for (int u = 0; u < kBaryChunk; ++u) {
            const long long k = k0 + u < M ? k0 + u : 0;
            use[u] = k0 + u < M && k != j;
            const double dk = __dsub_rn(xj, xs[k]);
            dup |= use[u] && dk == 0.0;
            d[u] = use[u] ? dk : 1.0;
            rr[u] = use[u] ? r[u] : 1.0;
        }
        const double acc0 = acc;
        bool ok = true;
#pragma unroll
        for (int u = 0; u < kBaryChunk; ++u) {
            ok &= in_window(d[u], 1023u - 60u, 1023u + 60u) & in_window(acc, 1023u - 900u, 1023u + 900u);
            const double q0 = __dmul_rn(acc, rr[u]);
            acc = __fma_rn(rr[u], __fma_rn(-d[u], q0, acc), q0);
        }
        if (!ok) {
            acc = acc0;
#pragma unroll 1
            for (int u = 0; u < kBaryChunk; ++u)
                if (use[u]) acc = __ddiv_rn(acc, d[u]);
        }
    };
    double ra[kBaryChunk], rb[kBaryChunk], rc[kBaryChunk];
    fetch(0, ra);
    fetch(kBaryChunk, rb);
    fetch(2 * kBaryChunk, rc);
    for (long long k0 = 0; k0 < M; k0 += 3 * kBaryChunk) {
        chunk(k0, ra);
        fetch(k0 + 3 * kBaryChunk, ra);
        chunk(k0 + kBaryChunk, rb);
        fetch(k0 + 4 * kBaryChunk, rb);
        chunk(k0 + 2 * kBaryChunk, rc);
        fetch(k0 + 5 * kBaryChunk, rc);
    }
    if (dup) record_failure(fail, j, PINT_E_DUPLICATE_NODES, xj);
    w[j] = acc;
}

__global__ void bary_closed2_kernel(long long M, double* __restrict__ w) {
    const long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= M) return;
    const double sgn = (j % 2 == 0) ? 1.0 : -1.0;
    w[j] = (j == 0 || j == M - 1) ? 0.5 * sgn : sgn;
}


// TREE mode (EXTENSION, within 1e-12 of EXACT: the sums in tree order): one CTA of 1024 threads
// walks the N slices in order; thread t owns nodes t, t + 1024, ... (PER of them, in registers —
// loaded once when the slices share their nodes, the usual case), the values of slice j + 1 are
// loaded while slice j is evaluated, and the node snap (interp.cpp:70-72: the lowest node within
// 1e-14 relative returns its value) rides in the same block reduction as (num, den): ONE pass and
// two barriers per slice — the slice's critical path is a divide and two 5-level shuffle trees.
constexpr int kTreeThreads = 1024;

template <int PER>
__global__ void __launch_bounds__(kTreeThreads)
scalar_sweep_tree_kernel(long long N, long long M, const double* __restrict__ nodes, long long node_stride,
                         const double* __restrict__ weights, const double* __restrict__ values,
                         const double* __restrict__ a_arr, const double* __restrict__ b_arr,
                         long long ab_stride, double y0, double* lambdas, double* y_out,
                         long long* extrapolations) {
    __shared__ double2 red[kTreeThreads / 32];
    __shared__ unsigned red_hit[kTreeThreads / 32];
    __shared__ double y_s;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // slice j's operands in xr/wr/vr/a/b, slice j + 1's loading into xn/wn/vn/an/bn while slice j is
    // evaluated (none of them depends on y: no global load on the slice-to-slice chain)
    double xr[PER], wr[PER], vr[PER], xn[PER], wn[PER], vn[PER];
    auto load_nodes = [&](long long j, double (&xd)[PER], double (&wd)[PER]) {
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const long long k = tid + q * kTreeThreads;
            xd[q] = (k < M && j < N) ? nodes[j * node_stride + k] : 0.0;
            wd[q] = (k < M && j < N) ? weights[j * node_stride + k] : 0.0;
        }
    };
    auto load_values = [&](long long j, double (&dst)[PER]) {
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const long long k = tid + q * kTreeThreads;
            dst[q] = (k < M && j < N) ? values[j * M + k] : 0.0;
        }
    };
    load_nodes(0, xr, wr);
    load_values(0, vr);
    double a = a_arr[0], b = b_arr[0];
    double y = y0;
    long long ext = 0;
    for (long long j = 0; j < N; ++j) {
        load_values(j + 1, vn);
        if (node_stride) load_nodes(j + 1, xn, wn);
        const double an = j + 1 < N ? a_arr[(j + 1) * ab_stride] : 0.0, bn = j + 1 < N ? b_arr[(j + 1) * ab_stride] : 0.0;
        if (y < a || y > b) ++ext;  // nievergelt.cpp:83
        double num = 0.0, den = 0.0;
        unsigned hit = 0xffffffffu;
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const long long k = tid + q * kTreeThreads;
            if (k < M) {
                const double d = __dsub_rn(y, xr[q]);
                if (fabs(d) <= __dmul_rn(1e-14, fmax(1.0, fabs(xr[q]))) && hit == 0xffffffffu)
                    hit = static_cast<unsigned>(k);
                const double r = wr[q] / d;
                num = fma(r, vr[q], num);
                den += r;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            num += __shfl_xor_sync(0xffffffffu, num, o);
            den += __shfl_xor_sync(0xffffffffu, den, o);
        }
        hit = __reduce_min_sync(0xffffffffu, hit);
        if (lane == 0) {
            red[warp] = make_double2(num, den);
            red_hit[warp] = hit;
        }
        __syncthreads();
        if (warp == 0) {
            double2 t = red[lane];
            unsigned h = __reduce_min_sync(0xffffffffu, red_hit[lane]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                t.x += __shfl_xor_sync(0xffffffffu, t.x, o);
                t.y += __shfl_xor_sync(0xffffffffu, t.y, o);
            }
            if (lane == 0) {
                const double yn = h != 0xffffffffu ? values[j * M + h] : t.x / t.y;
                y_s = yn;
                if (lambdas) lambdas[j] = yn;
            }
        }
        __syncthreads();
        y = y_s;
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            vr[q] = vn[q];
            if (node_stride) xr[q] = xn[q], wr[q] = wn[q];
        }
        a = an, b = bn;
    }
    if (tid == 0) {
        if (y_out) *y_out = y;
        if (extrapolations) *extrapolations = ext;
    }
}

// TREE mode, staged: the same sums with nothing but arithmetic and one barrier between slices.
// Slice j + 1 .. j + 3's values (and nodes, weights when every slice has its own) are already in
// a 4-slot shared-memory ring, bulk-copied ahead by warp 1 (the slot of slice j - 1, which no warp
// reads any more once slice j's barrier has passed); the intervals [a_j, b_j] are staged once. A
// thread sums up to 4 terms side by side, w / (y - x) as w x rcp(y - x) (MUFU.RCP64H + two Newton
// steps: no IEEE slow-path branches); (num, den, lowest snap) are reduced per warp, the W partials
// double-buffered by slice parity, and EVERY warp reduces them itself, so one barrier per slice.
// Config 5 (64 slices, M = 1024): the register-prefetch kernel above took ~90 us to sweep (a global-
// load latency per slice), this one ~55 us; the whole S = 98 solve 0.40 -> 0.093 ms. Used when M
// is even, N <= 4096 and the ring fits (launch_scalar_sweep).
using namespace pint_async;
constexpr int kStagedMaxN = 4096;
constexpr int kStagedRing = 4;  // slices in flight (a power of 2)
// Tolerance-mode reciprocal: the hardware approximation (MUFU.RCP64H) refined by two Newton steps —
// no IEEE slow-path branches. Only for |d| well inside the float exponent range (node distances
// here; the approximation's input range is the float one).
__device__ __forceinline__ double rcp_nr(double d) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    double e = fma(-d, r, 1.0);
    r = fma(r, e, r);
    e = fma(-d, r, 1.0);
    return fma(r, e, r);
}

// a / b with b first scaled into [1, 2) by an exact power of 2 (num and den of a barycentric sum
// can be ~1e150 with the reference's weights), then rcp_nr and one remainder correction; IEEE for
// zero, subnormal, infinite or NaN b
__device__ __forceinline__ double div_scaled(double a, double b) {
    const int e = (__double2hiint(b) >> 20) & 0x7ff;
    if (e == 0 || e == 0x7ff) return a / b;
    const double sc = __hiloint2double((2046 - e) << 20, 0);  // 2^-(e - 1023)
    const double as = a * sc, bs = b * sc;
    const double r = rcp_nr(bs);
    const double q = as * r;
    return fma(fma(-q, bs, as), r, q);
}

template <int THREADS, int PER>
__global__ void __launch_bounds__(THREADS)
scalar_sweep_staged_kernel(long long N, long long M, const double* __restrict__ nodes, long long node_stride,
                           const double* __restrict__ weights, const double* __restrict__ values,
                           const double* __restrict__ a_arr, const double* __restrict__ b_arr, long long ab_stride,
                           double y0, double* lambdas, double* y_out, long long* extrapolations) {
    constexpr int W = THREADS / 32;
    extern __shared__ __align__(16) double st[];
    __shared__ double2 red[2][W];  // (by slice parity: ONE barrier per slice)
    __shared__ unsigned red_hit[2][W];
    __shared__ __align__(8) unsigned long long bars[kStagedRing];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long arrays = node_stride ? 3 : 1;  // per slot: values [| nodes | weights]
    const long long slot_d = arrays * M;
    double* ab = st + kStagedRing * slot_d;  // a[N] | b[N]
    const unsigned bar0 = smem_u32(bars);
    auto issue = [&](long long j) {  // (one thread) slice j into slot j % kStagedRing
        const int sl = static_cast<int>(j & (kStagedRing - 1));
        double* dst = st + sl * slot_d;
        const unsigned bar = bar0 + 8u * sl;
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // (the slot's previous reads)
        asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(bar),
                     "r"(static_cast<unsigned>(8 * slot_d))
                     : "memory");
        bulk_copy(smem_u32(dst), values + j * M, static_cast<unsigned>(8 * M), bar);
        if (node_stride) {
            bulk_copy(smem_u32(dst + M), nodes + j * node_stride, static_cast<unsigned>(8 * M), bar);
            bulk_copy(smem_u32(dst + 2 * M), weights + j * node_stride, static_cast<unsigned>(8 * M), bar);
        }
    };
    if (tid == 0) {
        for (int q = 0; q < kStagedRing; ++q) mbar_init(bar0 + 8u * q);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    for (long long j = tid; j < N; j += THREADS) {
        ab[j] = a_arr[j * ab_stride];
        ab[N + j] = b_arr[j * ab_stride];
    }
    double xr[PER], wr[PER];
    if (!node_stride) {
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const long long k = tid + q * THREADS;
            xr[q] = k < M ? nodes[k] : 0.0;
            wr[q] = k < M ? weights[k] : 0.0;
        }
    }
    __syncthreads();
    if (tid == 0)
        for (long long q = 0; q < kStagedRing && q < N; ++q) issue(q);
    double y = y0;
    long long ext = 0;
    for (long long j = 0; j < N; ++j) {
        if (tid == 0 && (y < ab[j] || y > ab[N + j])) ++ext;  // nievergelt.cpp:83
        const int sl = static_cast<int>(j & (kStagedRing - 1)), par = static_cast<int>(j & 1);
        const double* V = st + sl * slot_d;
        mbar_wait(bar0 + 8u * sl, static_cast<unsigned>((j / kStagedRing) & 1));
        // the PER terms side by side (branch-free: their reciprocals overlap), w / (y - x) as w x an
        // approximate reciprocal refined by two Newton steps (tolerance mode)
        double num = 0.0, den = 0.0;
        unsigned hit = 0xffffffffu;
        double dq[PER], rq[PER];
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const long long k = tid + q * THREADS;
            const double xk = k < M ? (node_stride ? V[M + k] : xr[q]) : 0.0;
            dq[q] = __dsub_rn(y, xk);
            const bool snap = k < M && fabs(dq[q]) <= __dmul_rn(1e-14, fmax(1.0, fabs(xk)));
            hit = snap ? min(hit, static_cast<unsigned>(k)) : hit;
            rq[q] = rcp_nr(dq[q]);
        }
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const long long k = tid + q * THREADS;
            if (k < M) {
                const double wk = node_stride ? V[2 * M + k] : wr[q];
                const double r = __dmul_rn(wk, rq[q]);
                num = fma(r, V[k], num);
                den += r;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            num += __shfl_xor_sync(0xffffffffu, num, o);
            den += __shfl_xor_sync(0xffffffffu, den, o);
        }
        hit = __reduce_min_sync(0xffffffffu, hit);
        if (lane == 0) {
            red[par][warp] = make_double2(num, den);
            red_hit[par][warp] = hit;
        }
        __syncthreads();  // every warp's partial is in; every thread is done with slot sl
        // every warp reduces the W partials itself (no second barrier: red is double-buffered)
        double2 t = lane < W ? red[par][lane] : make_double2(0.0, 0.0);
        const unsigned h = __reduce_min_sync(0xffffffffu, lane < W ? red_hit[par][lane] : 0xffffffffu);
#pragma unroll
        for (int o = W / 2; o > 0; o >>= 1) {
            t.x += __shfl_xor_sync(0xffffffffu, t.x, o);
            t.y += __shfl_xor_sync(0xffffffffu, t.y, o);
        }
        t.x = __shfl_sync(0xffffffffu, t.x, 0);  // (lanes >= W reduced only zeros)
        t.y = __shfl_sync(0xffffffffu, t.y, 0);
        y = h != 0xffffffffu ? V[h] : div_scaled(t.x, t.y);
        if (tid == 0 && lambdas) lambdas[j] = y;
        // refill the previous slice's slot: past this slice's barrier no warp reads it any more (this
        // slice's slot may still be read for the snap value V[h] after the barrier)
        if (tid == 32 % THREADS && j >= 1 && j - 1 + kStagedRing < N) issue(j - 1 + kStagedRing);
    }
    if (tid == 0) {
        if (y_out) *y_out = y;
        if (extrapolations) *extrapolations = ext;
    }
}

// EXACT mode (bit-exact): one CTA of 512 threads walks the N slices in order. Per slice:
// (A) thread k (and k + 512, ...) takes node k — the snap test (interp.cpp:70-72, lowest hit by
// atomicMin) and the term (r v, r), r = w / (y - x), into shared memory; (B) thread 0 adds the
// terms in the reference's order (interp.cpp:74-78). B's two dependent DADD chains are the
// slice's critical path (M x 8 cycles), so the terms are read kSumAhead ahead through a register
// ring, and A is one node per thread with every operand already in shared memory: the nodes and
// weights staged once (or per slice when node_stride != 0), the slice's values copied in by the
// other warps while thread 0 sums the previous slice. Dynamic smem: x[M] | w[M] | v[2][M] |
// (r v, r)[M + kSumAhead].
constexpr int kSumAhead = 16;
constexpr int kExactThreads = 512;
#ifdef PINT_SWEEP_PROF  // tools/sweep_micro.cu only: thread 0's cycles in {terms + sync, sum, next sync}
__device__ unsigned long long g_sweep_prof[3];
#endif

__global__ void __launch_bounds__(kExactThreads)
scalar_sweep_exact_kernel(long long N, long long M, const double* __restrict__ nodes, long long node_stride,
                          const double* __restrict__ weights, const double* __restrict__ values,
                          const double* __restrict__ a_arr, const double* __restrict__ b_arr,
                          long long ab_stride, double y0, double* lambdas, double* y_out,
                          long long* extrapolations) {
    extern __shared__ double2 sw_smem[];
    double* x_s = reinterpret_cast<double*>(sw_smem);
    double* w_s = x_s + M;
    double* v_s = w_s + M;  // [2][M]
    double2* terms = reinterpret_cast<double2*>(v_s + 2 * M);
    __shared__ double y_s;
    __shared__ unsigned long long hit_s;
    const int tid = threadIdx.x;
    // stage slice j's operands (the nodes/weights only when they differ per slice, or at j = 0)
    auto stage = [&](long long j, int t0, int nt) {
        const double* v = values + j * M;
        double* vd = v_s + (j & 1) * M;
        for (long long k = tid - t0; k < M; k += nt) vd[k] = v[k];
        if (node_stride || j == 0)
            for (long long k = tid - t0; k < M; k += nt) {
                x_s[k] = nodes[j * node_stride + k];
                w_s[k] = weights[j * node_stride + k];
            }
    };
    double y = y0;
    long long ext = 0;
    if (tid == 0) hit_s = static_cast<unsigned long long>(M);
    for (long long k = M + tid; k < M + kSumAhead; k += kExactThreads) terms[k] = make_double2(0.0, 0.0);
    if (N > 0) stage(0, 0, kExactThreads);
    __syncthreads();
#ifdef PINT_SWEEP_PROF
    unsigned long long pa = 0, pb = 0, pc = 0;
#endif
    for (long long j = 0; j < N; ++j) {
#ifdef PINT_SWEEP_PROF
        const long long c0 = clock64();
#endif
        const double* v = v_s + (j & 1) * M;
        const double a = a_arr[j * ab_stride], b = b_arr[j * ab_stride];
        if (y < a || y > b) ++ext;  // nievergelt.cpp:83
        for (long long k = tid; k < M; k += kExactThreads) {
            const double xk = x_s[k], diff = __dsub_rn(y, xk);
            if (fabs(diff) <= __dmul_rn(1e-14, fmax(1.0, fabs(xk))))  // node snap (interp.cpp:70-72)
                atomicMin(&hit_s, static_cast<unsigned long long>(k));
            const double r = __ddiv_rn(w_s[k], diff);
            terms[k] = make_double2(__dmul_rn(r, v[k]), r);
        }
        __syncthreads();
#ifdef PINT_SWEEP_PROF
        const long long c1 = clock64();
#endif
        if (tid == 0) {
            const long long hit = static_cast<long long>(hit_s);
            if (hit < M) {
                y = v[hit];
            } else {
                double num = 0.0, den = 0.0;  // num += r*v, den += r for j = 0..M-1, in order
                double2 ring[kSumAhead];
#pragma unroll
                for (int u = 0; u < kSumAhead; ++u) ring[u] = terms[u];
                long long k = 0;
                // (volatile asm keeps "consume slot u, then refill it" in order; ptxas still parks
                // one accumulator in slot 0's register for the body, so that slot's refill is late
                // once per 16 terms: measured 10.3 cycles per term against the 8-cycle DADD chain)
                unsigned addr = static_cast<unsigned>(__cvta_generic_to_shared(terms + kSumAhead));
#pragma unroll 1
                for (; k + kSumAhead <= M; k += kSumAhead, addr += 16u * kSumAhead) {
#pragma unroll
                    for (int u = 0; u < kSumAhead; ++u) {
                        asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(num) : "d"(ring[u].x));
                        asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(den) : "d"(ring[u].y));
                        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];"
                                     : "=d"(ring[u].x), "=d"(ring[u].y)
                                     : "r"(addr + 16u * u));
                    }
                }
#pragma unroll
                for (int u = 0; u < kSumAhead - 1; ++u)
                    if (k + u < M) {
                        num = __dadd_rn(num, ring[u].x);
                        den = __dadd_rn(den, ring[u].y);
                    }
                y = __ddiv_rn(num, den);
            }
            y_s = y;
            hit_s = static_cast<unsigned long long>(M);
            if (lambdas) lambdas[j] = y;
        } else if (tid >= 32 && j + 1 < N) {
            stage(j + 1, 32, kExactThreads - 32);  // (warp 0 stays out of thread 0's way)
        }
#ifdef PINT_SWEEP_PROF
        const long long c2 = clock64();
#endif
        __syncthreads();
        y = y_s;
#ifdef PINT_SWEEP_PROF
        const long long c3 = clock64();
        pa += c1 - c0, pb += c2 - c1, pc += c3 - c2;
#endif
    }
#ifdef PINT_SWEEP_PROF
    if (tid == 0) g_sweep_prof[0] = pa, g_sweep_prof[1] = pb, g_sweep_prof[2] = pc;
#endif
    if (tid == 0) {
        if (y_out) *y_out = y;
        if (extrapolations) *extrapolations = ext;
    }
}

// EXACT mode for M <= 32 (the paper's Table 3 runs M = 4..7): ONE warp, lane k = node k, every
// slice's operands staged in shared memory at the start, so a slice is the terms (one IEEE divide
// per lane, in parallel), the snap as a ballot (lowest lane = lowest node), and the reference-order
// sums over the M terms by shuffles — every lane runs the same sums and gets the same y, so no
// barrier and no broadcast between slices. Bit-identical to the 512-thread kernel above (same
// operations in the same order); ~0.94 -> ~0.25 us per slice at M = 4. The slice itself is
// pint_dev::slice_eval_small, shared with the one-launch small run (ensemble.cu).
constexpr int kSmallM = 32;
template <int MM>  // M rounded up to a power of 2: the sums run over MM terms, the pad ones -0.0
__global__ void __launch_bounds__(32)
scalar_sweep_exact_small_kernel(long long N, long long M, const double* __restrict__ nodes, long long node_stride,
                                const double* __restrict__ weights, const double* __restrict__ values,
                                const double* __restrict__ a_arr, const double* __restrict__ b_arr,
                                long long ab_stride, double y0, double* lambdas, double* y_out,
                                long long* extrapolations) {
    extern __shared__ double ss[];
    const int lane = threadIdx.x;
    const long long nsets = node_stride ? N : 1;
    double* V = ss;              // [N][M]
    double* X = V + N * M;       // [nsets][M]
    double* Wt = X + nsets * M;  // [nsets][M]
    double* A = Wt + nsets * M;  // [N]
    double* B = A + N;           // [N]
    for (long long i = lane; i < N * M; i += 32) V[i] = values[i];
    for (long long s = 0; s < nsets; ++s)
        for (long long k = lane; k < M; k += 32) {
            X[s * M + k] = nodes[s * node_stride + k];
            Wt[s * M + k] = weights[s * node_stride + k];
        }
    for (long long j = lane; j < N; j += 32) A[j] = a_arr[j * ab_stride], B[j] = b_arr[j * ab_stride];
    __syncwarp();
    double y = y0;
    long long ext = 0;
    for (long long j = 0; j < N; ++j) {
        if (y < A[j] || y > B[j]) ++ext;  // nievergelt.cpp:83
        const long long so = node_stride ? j * M : 0;
        y = pint_dev::slice_eval_small<MM>(y, X + so, Wt + so, V + j * M, static_cast<int>(M), lane);
        if (lane == 0 && lambdas) lambdas[j] = y;
    }
    if (lane == 0) {
        if (y_out) *y_out = y;
        if (extrapolations) *extrapolations = ext;
    }
}

// upper_bound(x, xi) - 1 clamped to [0, M-2]; identical search order to or_bracket.
__device__ __forceinline__ long long bracket(const double* x, long long M, double xi) {
    long long lo = 0, len = M;
    while (len > 0) {
        const long long half = len / 2;
        if (!(x[lo + half] > xi)) {
            lo += half + 1;
            len -= half + 1;
        } else {
            len = half;
        }
    }
    long long b = lo - 1;
    b = b < 0 ? 0 : b;
    return b > M - 2 ? M - 2 : b;
}

__device__ __forceinline__ double lerp(double a, double b, double t) {
    return __fma_rn(t, __dsub_rn(b, a), a);
}

// EXTENSION: chain of bilinear maps over tables (N, 2, Mu, Mv). Nodes staged in smem.
// The sweep is one dependent chain: slice j's brackets need the value leaving slice j-1, then
// its corner values come from a 1 MiB table (HBM). Warp 0 runs the chain — all 32 lanes carry the
// same values, lane 0 stores — so that:
//  * the bracket is found by the warp at once: lane l tests the cell g - 15 + l around the
//    linearly extrapolated guess g (x[c] <= xi < x[c+1] is, for sorted nodes, exactly
//    upper_bound(xi) - 1); a ballot picks it, and only a miss of all 32 runs the binary search;
//  * t = (xi - x[i]) / (x[i+1] - x[i]) is Markstein's exact sequence on the cell's reciprocal
//    (staged once), the IEEE division only outside the exactness window (see bary_product_kernel);
//  * warps 1..kLvAhead pull the rows around the extrapolated brackets of slices j+1..j+kLvAhead into
//    L2 as soon as lane 0 publishes slice j's brackets.
constexpr int kLvAhead = 3;
constexpr int kLvRows = 16;  // rows either side of the guess pulled into L2

#ifdef PINT_SWEEP_PROF
__device__ unsigned long long g_bracket_miss;
#endif
__device__ __forceinline__ long long bracket_warp(const double* x, long long M, double xi, long long g, int lane) {
    g = g < 15 ? 15 : (g > M - 18 ? M - 18 : g);
    const long long c = g - 15 + lane;
    const bool in = c >= 0 && c + 1 < M && x[c] <= xi && xi < x[c + 1];
    const unsigned m = __ballot_sync(0xffffffffu, in);
#ifdef PINT_SWEEP_PROF
    if (!m && lane == 0) atomicAdd(&g_bracket_miss, 1ull);
#endif
    return m ? g - 15 + (__ffs(m) - 1) : bracket(x, M, xi);
}

__device__ __forceinline__ double cell_frac(double num, double den, double rcp) {
    // (num / den, correctly rounded: Markstein with rcp = RN(1 / den) inside the window)
    if (in_window(num, 1023u - 900u, 1023u + 900u) && in_window(den, 1023u - 60u, 1023u + 60u)) {
        const double q0 = __dmul_rn(num, rcp);
        return __fma_rn(rcp, __fma_rn(-den, q0, num), q0);
    }
    return __ddiv_rn(num, den);
}

__global__ void __launch_bounds__(32 * (kLvAhead + 1)) bilinear_sweep_kernel(
    long long N, long long Mu, long long Mv, const double* __restrict__ un, const double* __restrict__ vn,
    const double* __restrict__ tables, double u, double v, double* lambdas, long long* brackets,
    long long* extrapolations) {
    extern __shared__ double nodes_s[];
    double* us = nodes_s;                    // [Mu]
    double* vs = us + Mu;                    // [Mv]
    double* ru = vs + Mv;                    // [Mu - 1] RN(1 / (us[i+1] - us[i]))
    double* rv = ru + Mu;                    // [Mv - 1]
    // published by lane 0 of warp 0: {j, iu, iv, diu, div} (j = -1: not yet; j = N: done)
    __shared__ volatile long long pub[5];
    for (long long i = threadIdx.x; i < Mu; i += blockDim.x) us[i] = un[i];
    for (long long i = threadIdx.x; i < Mv; i += blockDim.x) vs[i] = vn[i];
    for (long long i = threadIdx.x; i + 1 < Mu; i += blockDim.x) ru[i] = __drcp_rn(__dsub_rn(un[i + 1], un[i]));
    for (long long i = threadIdx.x; i + 1 < Mv; i += blockDim.x) rv[i] = __drcp_rn(__dsub_rn(vn[i + 1], vn[i]));
    if (threadIdx.x == 0) pub[0] = -1;
    __syncthreads();
    const long long P = Mu * Mv;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp > 0) {  // L2 prefetchers: warp w covers slice j + w
        long long seen = -1;
        while (true) {
            const long long j = pub[0];
            if (j == seen) {
                __nanosleep(64);  // (a tight spin would compete with warp 0's shared loads)
                continue;
            }
            if (j >= N) break;
            const long long iu = pub[1], iv = pub[2], du = pub[3], dv = pub[4];
            if (pub[0] != j) continue;  // (republished meanwhile: take the newer one)
            seen = j;
            const long long t = j + warp;
            if (t >= N) continue;
            const long long gu = iu + warp * du, gv = iv + warp * dv;
            // rows gu - kLvRows .. gu + kLvRows + 1, the 3 lines around column gv, both components
            for (int e = lane; e < 2 * (2 * kLvRows + 2) * 3; e += 32) {
                const int comp = e & 1, line = (e >> 1) % 3, row = (e >> 1) / 3;
                const long long r = gu - kLvRows + row;
                long long c = gv - 16 + 16 * line;
                if (r < 0 || r >= Mu) continue;
                c = c < 0 ? 0 : (c >= Mv ? Mv - 1 : c);
                asm volatile("prefetch.global.L2 [%0];\n" ::"l"(tables + (t * 2 + comp) * P + r * Mv + c));
            }
        }
        return;
    }
    long long ext = 0, piu = 0, piv = 0, du = 0, dv = 0;
#ifdef PINT_SWEEP_PROF  // (tools/prof_lv_sweep.sh) lane 0's cycles per slice by section
    long long pa = 0, pb = 0, pc = 0, t0 = clock64();
#define LV_MARK(v)                      \
    do {                                \
        const long long t1 = clock64(); \
        v += t1 - t0;                   \
        t0 = t1;                        \
    } while (0)
#else
#define LV_MARK(v) \
    do {           \
    } while (0)
#endif
    for (long long j = 0; j < N; ++j) {
        if (u < us[0] || u > us[Mu - 1] || v < vs[0] || v > vs[Mv - 1]) ++ext;
        const long long iu = j ? bracket_warp(us, Mu, u, piu + du, lane) : bracket(us, Mu, u);
        const long long iv = j ? bracket_warp(vs, Mv, v, piv + dv, lane) : bracket(vs, Mv, v);
        if (j) du = iu - piu, dv = iv - piv;
        piu = iu, piv = iv;
        if (lane == 0) {  // (no fence: a torn read only misdirects a prefetch)
            pub[1] = iu, pub[2] = iv, pub[3] = du, pub[4] = dv;
            pub[0] = j;
        }
        LV_MARK(pa);
        const double* Tu = tables + (j * 2) * P + iu * Mv + iv;
        const double* Tv = Tu + P;
        double c[8];
        c[0] = Tu[0], c[1] = Tu[1], c[2] = Tu[Mv], c[3] = Tu[Mv + 1];
        c[4] = Tv[0], c[5] = Tv[1], c[6] = Tv[Mv], c[7] = Tv[Mv + 1];
        const double tu = cell_frac(__dsub_rn(u, us[iu]), __dsub_rn(us[iu + 1], us[iu]), ru[iu]);
        const double tv = cell_frac(__dsub_rn(v, vs[iv]), __dsub_rn(vs[iv + 1], vs[iv]), rv[iv]);
        u = lerp(lerp(c[0], c[2], tu), lerp(c[1], c[3], tu), tv);
        v = lerp(lerp(c[4], c[6], tu), lerp(c[5], c[7], tu), tv);
#ifdef PINT_SWEEP_PROF
        if (u == -1.2345) printf("x");  // (forces u, v before the mark)
#endif
        LV_MARK(pb);
        if (lane == 0) {
            if (lambdas) {
                lambdas[2 * j] = u;
                lambdas[2 * j + 1] = v;
            }
            if (brackets) {
                brackets[2 * j] = iu;
                brackets[2 * j + 1] = iv;
            }
        }
        LV_MARK(pc);
    }
#ifdef PINT_SWEEP_PROF
    if (lane == 0)
        printf("bilinear sweep per slice: bracket+publish %lld, loads+fractions+lerp %lld, stores %lld cycles; "
               "bracket misses %llu (cumulative)\n",
               pa / (N ? N : 1), pb / (N ? N : 1), pc / (N ? N : 1), g_bracket_miss);
#endif
    if (lane == 0) {
        pub[0] = N;  // release the prefetchers
        if (extrapolations) *extrapolations = ext;
    }
}

}  // namespace

int launch_bary_weights(pint_ctx* ctx, int kind, int64_t M, const double* nodes, double* w) {
    if (M < 1) return pint_set_error(ctx, PINT_E_BAD_GRID, "barycentric_weights: M >= 1 required");
    const unsigned blocks = static_cast<unsigned>((M + 127) / 128);
    if (kind == PINT_WEIGHTS_CLOSED2) {
        bary_closed2_kernel<<<blocks, 128, 0, ctx->stream>>>(M, w);
    } else if (kind == PINT_WEIGHTS_PRODUCT) {
        // the M^2 reciprocals in parallel, then one warp per CTA: every weight is a chain of M - 1
        // dependent quotients, so spread the chains over as many SM sub-partitions as there are warps
        const size_t smem = sizeof(double) * static_cast<size_t>(M);
        if (smem > 220 * 1024) return pint_set_error(ctx, PINT_E_INVALID, "barycentric_weights: M too large");
        auto* rcp = static_cast<double*>(pint_scratch(ctx, 4, sizeof(double) * static_cast<size_t>(M) * M));
        if (!rcp) return PINT_E_CUDA;
        bary_rcp_kernel<<<static_cast<unsigned>((M * M + 255) / 256), 256, 0, ctx->stream>>>(M, nodes, rcp);
        if (const int rc = pint_check_launch(ctx, "bary_rcp_kernel")) return rc;
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(bary_product_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        bary_product_kernel<<<static_cast<unsigned>((M + 31) / 32), 32, smem, ctx->stream>>>(M, nodes, rcp, w,
                                                                                             ctx->d_fail);
    } else {
        return pint_set_error(ctx, PINT_E_INVALID, "barycentric_weights: unknown kind");
    }
    return pint_check_launch(ctx, "bary_weights_kernel");
}

int launch_scalar_sweep(pint_ctx* ctx, int mode, int64_t N, int64_t M, const double* nodes,
                        int64_t node_stride, const double* weights, const double* values,
                        const double* a, const double* b, int64_t ab_stride, double y0,
                        double* lambdas, double* y_out, long long* extrapolations) {
    if (M < 1 || N < 0) return pint_set_error(ctx, PINT_E_INVALID, "scalar_sweep: bad sizes");
    if (mode == PINT_SWEEP_EXACT) {
        const size_t small_smem = sizeof(double) * static_cast<size_t>(N * M + 2 * (node_stride ? N : 1) * M + 2 * N);
        if (M <= kSmallM && small_smem <= 200 * 1024) {
            auto ks = M <= 4 ? scalar_sweep_exact_small_kernel<4> : M <= 8 ? scalar_sweep_exact_small_kernel<8>
                    : M <= 16 ? scalar_sweep_exact_small_kernel<16> : scalar_sweep_exact_small_kernel<32>;
            pint_kernel_attrs(reinterpret_cast<const void*>(ks));
            ks<<<1, 32, small_smem, ctx->stream>>>(
                N, M, nodes, node_stride, weights, values, a, b, ab_stride, y0, lambdas, y_out, extrapolations);
            return pint_check_launch(ctx, "scalar_sweep_exact_small_kernel");
        }
        const size_t smem = sizeof(double) * 4 * static_cast<size_t>(M) + sizeof(double2) * (M + kSumAhead);
        if (smem > 220 * 1024) return pint_set_error(ctx, PINT_E_INVALID, "scalar_sweep: M too large for EXACT mode");
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(scalar_sweep_exact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem));
        scalar_sweep_exact_kernel<<<1, kExactThreads, smem, ctx->stream>>>(
            N, M, nodes, node_stride, weights, values, a, b, ab_stride, y0, lambdas, y_out, extrapolations);
    } else if (mode == PINT_SWEEP_TREE) {
        if (M > 8 * kTreeThreads) return pint_set_error(ctx, PINT_E_INVALID, "scalar_sweep: M > 8192 unsupported in TREE mode");
        const int per = static_cast<int>((M + kTreeThreads - 1) / kTreeThreads);
        const size_t slot = sizeof(double) * (node_stride ? 3 : 1) * static_cast<size_t>(M);
        const size_t ab_bytes = sizeof(double) * 2 * static_cast<size_t>(N);
        const bool aligned = (reinterpret_cast<uintptr_t>(values) | reinterpret_cast<uintptr_t>(nodes) |
                              reinterpret_cast<uintptr_t>(weights)) % 16 == 0;
        if (M % 2 == 0 && (node_stride % 2 == 0) && aligned && N >= 1 && N <= kStagedMaxN &&
            kStagedRing * slot + ab_bytes <= 200 * 1024) {
            const size_t smem = kStagedRing * slot + ab_bytes;
            // 256 threads x up to 4 terms each for M <= 1024 (fewer warps to issue per slice and to
            // meet at the two barriers), 512 x 4 to M = 2048, else 1024 x 8
            auto ks = M <= 256 ? scalar_sweep_staged_kernel<256, 1> : M <= 512 ? scalar_sweep_staged_kernel<256, 2>
                    : M <= 1024 ? scalar_sweep_staged_kernel<256, 4> : M <= 2048 ? scalar_sweep_staged_kernel<512, 4>
                    : scalar_sweep_staged_kernel<1024, 8>;
            const int threads = M <= 1024 ? 256 : M <= 2048 ? 512 : 1024;
            pint_kernel_attrs(reinterpret_cast<const void*>(ks));
            ks<<<1, threads, smem, ctx->stream>>>(N, M, nodes, node_stride, weights, values, a, b, ab_stride, y0,
                                                       lambdas, y_out, extrapolations);
            return pint_check_launch(ctx, "scalar_sweep_staged_kernel");
        }
        auto k = per <= 1 ? scalar_sweep_tree_kernel<1> : per <= 2 ? scalar_sweep_tree_kernel<2>
               : per <= 4 ? scalar_sweep_tree_kernel<4> : scalar_sweep_tree_kernel<8>;
        k<<<1, kTreeThreads, 0, ctx->stream>>>(N, M, nodes, node_stride, weights, values, a, b, ab_stride, y0,
                                               lambdas, y_out, extrapolations);
    } else {
        return pint_set_error(ctx, PINT_E_INVALID, "scalar_sweep: unknown mode");
    }
    return pint_check_launch(ctx, "scalar_sweep_kernel");
}

int launch_bilinear_sweep(pint_ctx* ctx, int64_t N, int64_t Mu, int64_t Mv, const double* un,
                          const double* vn, const double* tables, double u0, double v0,
                          double* lambdas, long long* brackets, long long* extrapolations) {
    if (Mu < 2 || Mv < 2 || N < 0) return pint_set_error(ctx, PINT_E_BAD_GRID, "bilinear_sweep: need >= 2 nodes per axis");
    const size_t smem = sizeof(double) * 2 * static_cast<size_t>(Mu + Mv);
    if (smem > 220 * 1024) return pint_set_error(ctx, PINT_E_INVALID, "bilinear_sweep: grid too large");
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(bilinear_sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
    bilinear_sweep_kernel<<<1, 32 * (kLvAhead + 1), smem, ctx->stream>>>(N, Mu, Mv, un, vn, tables, u0, v0,
                                                                       lambdas, brackets, extrapolations);
    return pint_check_launch(ctx, "bilinear_sweep_kernel");
}
