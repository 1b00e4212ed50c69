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

}  // namespace

extern "C" int pint_probe_peak(pint_ctx* ctx, int precision, double* tflops) {
    if (!ctx || !tflops) return PINT_E_INVALID;
    void* sink = pint_scratch(ctx, 3, 4096);
    if (!sink) return PINT_E_CUDA;
    const int iters = 1 << 14;
    const unsigned blocks = static_cast<unsigned>(ctx->sm_count * 8);
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(ctx->ev0, ctx->stream);
        if (precision == PINT_F32)
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
    const double flops = 2.0 * 8.0 * iters * 256.0 * blocks;
    *tflops = flops / (best * 1e-3) / 1e12;
    return PINT_OK;
}
