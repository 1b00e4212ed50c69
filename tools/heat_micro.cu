// Section timing of heat_build_kernel (clock64 marks compiled in with -DPINT_HEAT_PROF): per warp,
// cycles per step in {wait fwd half, forward, stage+wait back half, back, stage next}.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -DPINT_HEAT_PROF -std=c++17 \
//        -Iinclude -Ipaper_1304_6514_b200/csrc tools/heat_micro.cu -o tools/_heat_micro
//   tools/_heat_micro n N S
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1304_6514_b200/csrc/heat.cu"

int pint_set_error(pint_ctx*, int code, const std::string& msg) {
    std::fprintf(stderr, "error %d: %s\n", code, msg.c_str());
    return code;
}
int pint_check_launch(pint_ctx*, const char* what) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) std::fprintf(stderr, "%s: %s\n", what, cudaGetErrorString(e));
    return e == cudaSuccess ? 0 : PINT_E_CUDA;
}
void* pint_scratch(pint_ctx*, int, size_t) { return nullptr; }
void pint_kernel_attrs(const void* fn) {
    cudaFuncAttributes a{};
    cudaFuncGetAttributes(&a, fn);
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024 - static_cast<int>(a.sharedSizeBytes));
}
extern "C" int64_t pint_affine_ldm(int64_t n) { return (n + 1 + 3) / 4 * 4; }

int main(int argc, char** argv) {
    const int n = argc > 1 ? std::atoi(argv[1]) : 128;
    const int N = argc > 2 ? std::atoi(argv[2]) : 1;
    const int S = argc > 3 ? std::atoi(argv[3]) : 256;
    const long long Q = static_cast<long long>(N) * S;
    std::vector<int64_t> off(N + 1);
    for (int j = 0; j <= N; ++j) off[j] = static_cast<int64_t>(j) * S;
    std::vector<double> dt(N, 1e-4), r(Q), fa(Q), fb(Q), sx(n);
    for (long long q = 0; q < Q; ++q) r[q] = 2.5 + 0.001 * (q % 7), fa[q] = -0.3, fb[q] = 0.7;
    for (int i = 0; i < n; ++i) sx[i] = std::sin(M_PI * (i + 1) / (n + 1));
    int64_t* d_off;
    double *d_dt, *d_r, *d_fa, *d_fb, *d_sx, *d_rec, *d_maps;
    cudaMalloc(&d_off, sizeof(int64_t) * (N + 1));
    cudaMalloc(&d_dt, 8 * N);
    cudaMalloc(&d_r, 8 * Q);
    cudaMalloc(&d_fa, 8 * Q);
    cudaMalloc(&d_fb, 8 * Q);
    cudaMalloc(&d_sx, 8 * n);
    cudaMemcpy(d_off, off.data(), sizeof(int64_t) * (N + 1), cudaMemcpyHostToDevice);
    cudaMemcpy(d_dt, dt.data(), 8 * N, cudaMemcpyHostToDevice);
    cudaMemcpy(d_r, r.data(), 8 * Q, cudaMemcpyHostToDevice);
    cudaMemcpy(d_fa, fa.data(), 8 * Q, cudaMemcpyHostToDevice);
    cudaMemcpy(d_fb, fb.data(), 8 * Q, cudaMemcpyHostToDevice);
    cudaMemcpy(d_sx, sx.data(), 8 * n, cudaMemcpyHostToDevice);
    cudaMalloc(&d_rec, 8 * records_doubles(n, N, S));
    const long long ldm = pint_affine_ldm(n);
    cudaMalloc(&d_maps, 8 * ldm * n * N);
    pint_ctx ctx;
    cudaStreamCreateWithFlags(&ctx.stream, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&ctx.side, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&ctx.ev_fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ctx.ev_join, cudaEventDisableTiming);
    cudaMalloc(&ctx.d_fail, sizeof(FailRec));
    cudaMemset(ctx.d_fail, 0xff, sizeof(FailRec));
    if (launch_heat_factor(&ctx, n, N, S, d_off, d_dt, d_r, d_fa, d_fb, d_sx, d_rec)) return 1;
    for (int rep = 0; rep < 2; ++rep)
        if (launch_heat_build(&ctx, n, N, S, d_off, d_dt, d_rec, d_sx, d_maps, nullptr, 0)) return 1;
    cudaDeviceSynchronize();
    const int wps = (n + 31) / 32;
    {
        std::vector<unsigned long long> span(2 * (1 << 14) * 2);
        cudaMemcpyFromSymbol(span.data(), g_heat_span, span.size() * 8);
        unsigned long long b0 = ~0ull, b1 = 0, f0 = ~0ull, f1 = 0;
        for (int b = 0; b < N * wps && b < (1 << 14); ++b) b0 = std::min(b0, span[b * 2]), b1 = std::max(b1, span[b * 2 + 1]);
        for (int b = 0; b < (N + 31) / 32; ++b) {
            const size_t o = (size_t(1) << 15) + b * 2;
            f0 = std::min(f0, span[o]), f1 = std::max(f1, span[o + 1]);
        }
        const unsigned long long t0 = std::min(b0, f0);
        std::printf("basis CTAs: start %.3f end %.3f ms; forced CTAs: start %.3f end %.3f ms\n", (b0 - t0) * 1e-6,
                    (b1 - t0) * 1e-6, (f0 - t0) * 1e-6, (f1 - t0) * 1e-6);
    }
    std::vector<unsigned long long> prof(static_cast<size_t>(1 << 14) * 6);
    cudaMemcpyFromSymbol(prof.data(), g_heat_prof, prof.size() * 8);
    const char* names[5] = {"wait_fwd", "forward", "stage_wait_back", "back", "stage_next"};
    {
        std::vector<unsigned long long> pf(size_t(1024) * 6);
        cudaMemcpyFromSymbol(pf.data(), g_heat_prof_f, pf.size() * 8);
        const int nf = (N + 31) / 32;
        double acc[5] = {0, 0, 0, 0, 0};
        for (int b = 0; b < nf && b < 1024; ++b)
            for (int q = 0; q < 5; ++q) acc[q] += pf[b * 6 + q];
        std::printf("forced warps (%d):", nf);
        double tot = 0;
        for (int q = 0; q < 5; ++q) std::printf(" %.0f", acc[q] / nf / S), tot += acc[q] / nf;
        std::printf("  per-row=%.1f\n", tot / S / n);
    }
    for (int role = 0; role < 1; ++role) {  // basis warps
        double acc[5] = {0, 0, 0, 0, 0}, worst = 0;
        int cnt = 0;
        for (int b = 0; b < N * wps && b < (1 << 14); ++b) {
            (void)role;
            double tot = 0;
            for (int q = 0; q < 5; ++q) acc[q] += prof[b * 6 + q], tot += prof[b * 6 + q];
            worst = tot > worst ? tot : worst;
            ++cnt;
        }
        if (!cnt) continue;
        std::printf("%s warps (%d):", role ? "forced-column" : "basis", cnt);
        double tot = 0;
        for (int q = 0; q < 5; ++q) {
            std::printf(" %s=%.0f", names[q], acc[q] / cnt / S);
            tot += acc[q] / cnt;
        }
        std::printf("  per-row=%.1f (worst warp %.1f)\n", tot / S / n, worst / S / n);
    }
    if (n >= 282) {  // TMEM build: thread 0's segments per step
        std::vector<unsigned long long> seg(static_cast<size_t>(1 << 14) * 8);
        cudaMemcpyFromSymbol(seg.data(), g_heat_seg, seg.size() * 8);
        const int ctas = N * ((wps + 3) / 4);
        const char* sn[6] = {"fwd_reg", "fwd_tmem", "fwd_smem", "back_smem", "back_tmem", "back_reg"};
        double acc[6] = {0, 0, 0, 0, 0, 0};
        for (int b = 0; b < ctas && b < (1 << 14); ++b)
            for (int q = 0; q < 6; ++q) acc[q] += seg[b * 8 + q];
        {  // CTA lifetime against its step loop (the last launch's spans; prof accumulates both)
            std::vector<unsigned long long> span(2 * (1 << 14) * 2), pr(static_cast<size_t>(1 << 14) * 6);
            cudaMemcpyFromSymbol(span.data(), g_heat_span, span.size() * 8);
            cudaMemcpyFromSymbol(pr.data(), g_heat_prof, pr.size() * 8);
            double life = 0, loop = 0;
            for (int b = 0; b < ctas && b < (1 << 14); ++b) {
                life += double(span[b * 2 + 1] - span[b * 2]);
                for (int q = 0; q < 5; ++q) loop += double(pr[b * 6 + q]);
            }
            double epi = 0, tail = 0;
            unsigned long long t0 = ~0ull, t1 = 0;
            const size_t o = size_t(1) << 15;  // g_heat_span[1]: {epilogue end, CTA end}
            for (int b = 0; b < ctas && b < (1 << 14); ++b) {
                epi += double(span[o + b * 2] - span[b * 2 + 1]);
                tail += double(span[o + b * 2 + 1] - span[o + b * 2]);
                t0 = std::min(t0, span[b * 2]);
                t1 = std::max(t1, span[o + b * 2 + 1]);
            }
            int sms = 0;
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
            std::printf("CTA lifetime %.1f us, step loop %.1f us (at 1.965 GHz), epilogue %.1f us, dealloc+ready %.1f us; "
                        "launch span %.3f ms = %.1f us per CTA slot on %d SMs\n", life / ctas * 1e-3,
                        loop / ctas / 1.965e3, epi / ctas * 1e-3, tail / ctas * 1e-3, (t1 - t0) * 1e-6,
                        (t1 - t0) * 1e-3 / (double(ctas) / sms), sms);
        }
        std::printf("TMEM segments, cycles per step (per row):");
        const int rows[6] = {64, 256, n - 320, n - 320 - 1, 256, 64};
        for (int q = 0; q < 6; ++q) {
            const double c = acc[q] / ctas / S / 2;  // (two launches accumulate)
            std::printf(" %s=%.0f (%.1f)", sn[q], c, c / rows[q]);
        }
        std::printf("\n");
    }
    return 0;
}
