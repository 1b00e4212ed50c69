// Roofline probe: measured FP64 / FP32 FMA throughput of this GPU (MEASURED_PEAKS.json carries
// only HBM and bf16 figures). 8 independent FMA chains per thread, grid = 8 CTAs per SM.
#include "pint_internal.cuh"

namespace {

template <typename R>
__global__ void __launch_bounds__(256) fma_probe_kernel(int iters, R seed, R* sink) {
    R a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = seed + R(threadIdx.x + k);
    const R m = R(0.9999999), c = R(1e-7);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = fma(a[k], m, c);
    }
    R s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == R(-1)) sink[threadIdx.x] = s;  // never true; keeps the chains alive
}

// FP64 tensor-core throughput: 8 independent m8n8k4 accumulators per warp.
__global__ void __launch_bounds__(256) dmma_probe_kernel(int iters, double seed, double* sink) {
    double acc[8][2];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k][0] = acc[k][1] = seed * k;
    const double a = seed + threadIdx.x, b = 0.5 + 1e-3 * threadIdx.x;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(acc[k][0]), "+d"(acc[k][1])
                         : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += acc[k][0] + acc[k][1];
    if (s == -1.0) sink[threadIdx.x] = s;
}

// Dependent-chain latency of one warp, cycles per op: out = {DFMA, DADD, DMUL, FFMA, LDS.64};
// then cycles per ROW of the heat build's two recurrences: out[5] = forward row
// (x - negr*d, then the Markstein division: 5 dependent ops), out[6] = back row (y - c*d: 2 ops),
// out[7] = alternating DMUL/DADD, per op.
__global__ void latency_probe_kernel(double seed, double* sink, double* out, const double* table) {
    __shared__ double sh[64];
    sh[threadIdx.x] = table[threadIdx.x];
    sh[threadIdx.x + 32] = table[threadIdx.x + 32];
    __syncwarp();
    constexpr int kOps = 1024;
    double a = seed + threadIdx.x;
    long long t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < kOps; ++i) a = __fma_rn(a, 0.999999, 1e-9);
    long long t1 = clock64();
#pragma unroll 64
    for (int i = 0; i < kOps; ++i) a = __dadd_rn(a, 1e-9);
    long long t2 = clock64();
#pragma unroll 64
    for (int i = 0; i < kOps; ++i) a = __dmul_rn(a, 0.999999);
    long long t3 = clock64();
    float fa = static_cast<float>(a);
#pragma unroll 64
    for (int i = 0; i < kOps; ++i) fa = __fmaf_rn(fa, 0.999f, 1e-6f);
    long long t4 = clock64();
    int idx = static_cast<int>(fa) & 1;
#pragma unroll 64
    for (int i = 0; i < kOps; ++i) idx = static_cast<int>(sh[idx]) & 31;
    long long t5 = clock64();
    a = a + static_cast<double>(idx);
    const double negr = -0.3, p = 1.7, rcp = 1.0 / 1.7, c = -0.2;
    double x = a;
#pragma unroll 64
    for (int i = 0; i < kOps; ++i) {
        const double num = __dsub_rn(x, __dmul_rn(negr, a));
        const double q0 = __dmul_rn(num, rcp);
        const double rem = __fma_rn(-p, q0, num);
        a = __fma_rn(rem, rcp, q0);
    }
    long long t6 = clock64();
#pragma unroll 64
    for (int i = 0; i < kOps; ++i) a = __dsub_rn(x, __dmul_rn(c, a));
    long long t7 = clock64();
#pragma unroll 64
    for (int i = 0; i < kOps; ++i) a = (i & 1) ? __dadd_rn(a, 1e-9) : __dmul_rn(a, 0.999999);
    long long t8 = clock64();
    if (threadIdx.x == 0) {
        out[5] = double(t6 - t5) / kOps;
        out[6] = double(t7 - t6) / kOps;
        out[7] = double(t8 - t7) / kOps;
        out[0] = double(t1 - t0) / kOps;
        out[1] = double(t2 - t1) / kOps;
        out[2] = double(t3 - t2) / kOps;
        out[3] = double(t4 - t3) / kOps;
        out[4] = double(t5 - t4) / kOps;
    }
    if (a == -1.0 || idx == 12345) sink[0] = a + fa;
}

}  // namespace

extern "C" int pint_probe_latency(pint_ctx* ctx, double* cycles /* 8 */) {
    if (!ctx || !cycles) return PINT_E_INVALID;
    double* d = static_cast<double*>(pint_scratch(ctx, 3, 4096));
    if (!d) return PINT_E_CUDA;
    cudaMemsetAsync(d, 0, 4096, ctx->stream);  // table of zeros: the LDS chain reads sh[0]
    latency_probe_kernel<<<1, 32, 0, ctx->stream>>>(1.0, d + 256, d + 128, d);
    if (const int rc = pint_check_launch(ctx, "latency_probe_kernel")) return rc;
    if (cudaMemcpyAsync(cycles, d + 128, 8 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess ||
        cudaStreamSynchronize(ctx->stream) != cudaSuccess)
        return pint_set_error(ctx, PINT_E_CUDA, "latency probe failed");
    return PINT_OK;
}

extern "C" int pint_probe_peak(pint_ctx* ctx, int precision, double* tflops) {
    if (!ctx || !tflops) return PINT_E_INVALID;
    void* sink = pint_scratch(ctx, 3, 4096);
    if (!sink) return PINT_E_CUDA;
    const int iters = 1 << 14;
    const unsigned blocks = static_cast<unsigned>(ctx->sm_count * 8);
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(ctx->ev0, ctx->stream);
        if (precision == PINT_PROBE_DMMA)
            dmma_probe_kernel<<<blocks, 256, 0, ctx->stream>>>(iters / 8, 1.0, static_cast<double*>(sink));
        else if (precision == PINT_F32)
            fma_probe_kernel<float><<<blocks, 256, 0, ctx->stream>>>(iters, 1.0f, static_cast<float*>(sink));
        else
            fma_probe_kernel<double><<<blocks, 256, 0, ctx->stream>>>(iters, 1.0, static_cast<double*>(sink));
        cudaEventRecord(ctx->ev1, ctx->stream);
        if (const int rc = pint_check_launch(ctx, "fma_probe_kernel")) return rc;
        if (cudaEventSynchronize(ctx->ev1) != cudaSuccess) return pint_set_error(ctx, PINT_E_CUDA, "probe sync");
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
        if (rep > 0 && ms < best) best = ms;
    }
    // DMMA: 8 m8n8k4 (512 flops each) per warp per iteration
    const double flops = precision == PINT_PROBE_DMMA ? 512.0 * 8.0 * (iters / 8) * 8.0 * blocks
                                                      : 2.0 * 8.0 * iters * 256.0 * blocks;
    *tflops = flops / (best * 1e-3) / 1e12;
    return PINT_OK;
}
