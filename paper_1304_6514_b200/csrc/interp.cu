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
#include "pint_internal.cuh"

namespace {

using pint_dev::record_failure;

__global__ void bary_product_kernel(long long M, const double* __restrict__ x, double* __restrict__ w,
                                    FailRec* fail) {
    const long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= M) return;
    const double xj = x[j];
    double acc = 1.0;
    bool dup = false;
    for (long long k = 0; k < M; ++k) {
        if (k == j) continue;
        const double diff = __dsub_rn(xj, x[k]);
        if (diff == 0.0) {
            dup = true;
            break;
        }
        acc = __ddiv_rn(acc, diff);
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

constexpr int kSweepThreads = 256;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// One CTA walks the N slices in order. Dynamic smem: r[M], rv[M] (EXACT mode).
template <bool kExact>
__global__ void __launch_bounds__(kSweepThreads)
scalar_sweep_kernel(long long N, long long M, const double* __restrict__ nodes, long long node_stride,
                    const double* __restrict__ weights, const double* __restrict__ values,
                    const double* __restrict__ a_arr, const double* __restrict__ b_arr,
                    long long ab_stride, double y0, double* lambdas, double* y_out,
                    long long* extrapolations) {
    extern __shared__ double smem[];
    double* r_s = smem;
    double* rv_s = smem + M;
    __shared__ double y_s;
    __shared__ long long hit_s;
    __shared__ double red_num[kSweepThreads / 32], red_den[kSweepThreads / 32];
    const int tid = threadIdx.x;
    double y = y0;
    long long ext = 0;
    for (long long j = 0; j < N; ++j) {
        const double* x = nodes + j * node_stride;
        const double* w = weights + j * node_stride;
        const double* v = values + j * M;
        const double a = a_arr[j * ab_stride], b = b_arr[j * ab_stride];
        if (y < a || y > b) ++ext;  // nievergelt.cpp:83
        if (tid == 0) hit_s = M;
        __syncthreads();
        // node snap: the lowest node within 1e-14 (relative) returns its value (interp.cpp:70-72)
        for (long long k = tid; k < M; k += kSweepThreads) {
            const double xk = x[k];
            if (fabs(__dsub_rn(y, xk)) <= __dmul_rn(1e-14, fmax(1.0, fabs(xk)))) {
                atomicMin(reinterpret_cast<unsigned long long*>(&hit_s), static_cast<unsigned long long>(k));
                break;
            }
        }
        __syncthreads();
        const long long hit = hit_s;
        if (hit < M) {
            y = v[hit];
        } else if (kExact) {
            for (long long k = tid; k < M; k += kSweepThreads) {
                const double r = __ddiv_rn(w[k], __dsub_rn(y, x[k]));
                r_s[k] = r;
                rv_s[k] = __dmul_rn(r, v[k]);
            }
            __syncthreads();
            if (tid == 0) {
                // the reference's order: num += r*v, den += r for j = 0..M-1 (interp.cpp:74-78)
                double num = 0.0, den = 0.0;
                long long k = 0;
                for (; k + 4 <= M; k += 4) {
                    const double n0 = rv_s[k], n1 = rv_s[k + 1], n2 = rv_s[k + 2], n3 = rv_s[k + 3];
                    const double d0 = r_s[k], d1 = r_s[k + 1], d2 = r_s[k + 2], d3 = r_s[k + 3];
                    num = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(num, n0), n1), n2), n3);
                    den = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(den, d0), d1), d2), d3);
                }
                for (; k < M; ++k) {
                    num = __dadd_rn(num, rv_s[k]);
                    den = __dadd_rn(den, r_s[k]);
                }
                y_s = __ddiv_rn(num, den);
            }
            __syncthreads();
            y = y_s;
        } else {
            double num = 0.0, den = 0.0;
            for (long long k = tid; k < M; k += kSweepThreads) {
                const double r = w[k] / (y - x[k]);
                num = fma(r, v[k], num);
                den += r;
            }
            num = warp_sum(num);
            den = warp_sum(den);
            if ((tid & 31) == 0) {
                red_num[tid >> 5] = num;
                red_den[tid >> 5] = den;
            }
            __syncthreads();
            if (tid == 0) {
                double sn = 0.0, sd = 0.0;
                for (int q = 0; q < kSweepThreads / 32; ++q) {
                    sn += red_num[q];
                    sd += red_den[q];
                }
                y_s = sn / sd;
            }
            __syncthreads();
            y = y_s;
        }
        if (tid == 0 && lambdas) lambdas[j] = y;
        __syncthreads();
    }
    if (tid == 0) {
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
__global__ void bilinear_sweep_kernel(long long N, long long Mu, long long Mv,
                                      const double* __restrict__ un, const double* __restrict__ vn,
                                      const double* __restrict__ tables, double u, double v,
                                      double* lambdas, long long* brackets, long long* extrapolations) {
    extern __shared__ double nodes_s[];
    double* us = nodes_s;
    double* vs = nodes_s + Mu;
    for (long long i = threadIdx.x; i < Mu; i += blockDim.x) us[i] = un[i];
    for (long long i = threadIdx.x; i < Mv; i += blockDim.x) vs[i] = vn[i];
    __syncthreads();
    if (threadIdx.x != 0) return;
    const long long P = Mu * Mv;
    long long ext = 0;
    for (long long j = 0; j < N; ++j) {
        if (u < us[0] || u > us[Mu - 1] || v < vs[0] || v > vs[Mv - 1]) ++ext;
        const long long iu = bracket(us, Mu, u), iv = bracket(vs, Mv, v);
        const double tu = __ddiv_rn(__dsub_rn(u, us[iu]), __dsub_rn(us[iu + 1], us[iu]));
        const double tv = __ddiv_rn(__dsub_rn(v, vs[iv]), __dsub_rn(vs[iv + 1], vs[iv]));
        const double* Tu = tables + (j * 2) * P + iu * Mv + iv;
        const double* Tv = Tu + P;
        const double u00 = Tu[0], u01 = Tu[1], u10 = Tu[Mv], u11 = Tu[Mv + 1];
        const double v00 = Tv[0], v01 = Tv[1], v10 = Tv[Mv], v11 = Tv[Mv + 1];
        u = lerp(lerp(u00, u10, tu), lerp(u01, u11, tu), tv);
        v = lerp(lerp(v00, v10, tu), lerp(v01, v11, tu), tv);
        if (lambdas) {
            lambdas[2 * j] = u;
            lambdas[2 * j + 1] = v;
        }
        if (brackets) {
            brackets[2 * j] = iu;
            brackets[2 * j + 1] = iv;
        }
    }
    if (extrapolations) *extrapolations = ext;
}

}  // namespace

int launch_bary_weights(pint_ctx* ctx, int kind, int64_t M, const double* nodes, double* w) {
    if (M < 1) return pint_set_error(ctx, PINT_E_BAD_GRID, "barycentric_weights: M >= 1 required");
    const unsigned blocks = static_cast<unsigned>((M + 127) / 128);
    if (kind == PINT_WEIGHTS_CLOSED2) {
        bary_closed2_kernel<<<blocks, 128, 0, ctx->stream>>>(M, w);
    } else if (kind == PINT_WEIGHTS_PRODUCT) {
        bary_product_kernel<<<blocks, 128, 0, ctx->stream>>>(M, nodes, w, ctx->d_fail);
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
        const size_t smem = sizeof(double) * 2 * static_cast<size_t>(M);
        if (smem > 220 * 1024) return pint_set_error(ctx, PINT_E_INVALID, "scalar_sweep: M too large for EXACT mode");
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(scalar_sweep_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem));
        scalar_sweep_kernel<true><<<1, kSweepThreads, smem, ctx->stream>>>(
            N, M, nodes, node_stride, weights, values, a, b, ab_stride, y0, lambdas, y_out, extrapolations);
    } else if (mode == PINT_SWEEP_TREE) {
        scalar_sweep_kernel<false><<<1, kSweepThreads, 0, ctx->stream>>>(
            N, M, nodes, node_stride, weights, values, a, b, ab_stride, y0, lambdas, y_out, extrapolations);
    } else {
        return pint_set_error(ctx, PINT_E_INVALID, "scalar_sweep: unknown mode");
    }
    return pint_check_launch(ctx, "scalar_sweep_kernel");
}

int launch_bilinear_sweep(pint_ctx* ctx, int64_t N, int64_t Mu, int64_t Mv, const double* un,
                          const double* vn, const double* tables, double u0, double v0,
                          double* lambdas, long long* brackets, long long* extrapolations) {
    if (Mu < 2 || Mv < 2 || N < 0) return pint_set_error(ctx, PINT_E_BAD_GRID, "bilinear_sweep: need >= 2 nodes per axis");
    const size_t smem = sizeof(double) * static_cast<size_t>(Mu + Mv);
    if (smem > 220 * 1024) return pint_set_error(ctx, PINT_E_INVALID, "bilinear_sweep: grid too large");
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(bilinear_sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
    bilinear_sweep_kernel<<<1, 128, smem, ctx->stream>>>(N, Mu, Mv, un, vn, tables, u0, v0, lambdas,
                                                         brackets, extrapolations);
    return pint_check_launch(ctx, "bilinear_sweep_kernel");
}
