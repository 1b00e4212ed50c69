// Section timing of the EXACT scalar sweep (clock64 marks compiled in with -DPINT_SWEEP_PROF):
// thread 0's cycles per slice in {terms + barrier, ordered sum, barrier}.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -DPINT_SWEEP_PROF -std=c++17 \
//        -Iinclude -Ipaper_1304_6514_b200/csrc tools/sweep_micro.cu -o tools/_sweep_micro
//   tools/_sweep_micro N M
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1304_6514_b200/csrc/interp.cu"

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
void pint_kernel_attrs(const void* fn) { cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024); }

int main(int argc, char** argv) {
    const int N = argc > 1 ? std::atoi(argv[1]) : 64;
    const int M = argc > 2 ? std::atoi(argv[2]) : 1024;
    std::vector<double> x(M), w(M), v(static_cast<size_t>(N) * M), ab{0.0, 1.25};
    for (int k = 0; k < M; ++k) {
        x[k] = 0.625 * (1.0 - std::cos(M_PI * k / (M - 1)));
        w[k] = ((k & 1) ? -1.0 : 1.0) * ((k == 0 || k == M - 1) ? 0.5 : 1.0);
    }
    for (size_t q = 0; q < v.size(); ++q) v[q] = 0.3 + 0.5 * x[q % M] * (1.0 - 0.1 * std::sin(0.01 * q));
    double *d_x, *d_w, *d_v, *d_ab, *d_y;
    long long* d_e;
    cudaMalloc(&d_x, 8 * M);
    cudaMalloc(&d_w, 8 * M);
    cudaMalloc(&d_v, 8 * v.size());
    cudaMalloc(&d_ab, 16);
    cudaMalloc(&d_y, 8 * (N + 1));
    cudaMalloc(&d_e, 8);
    cudaMemcpy(d_x, x.data(), 8 * M, cudaMemcpyHostToDevice);
    cudaMemcpy(d_w, w.data(), 8 * M, cudaMemcpyHostToDevice);
    cudaMemcpy(d_v, v.data(), 8 * v.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(d_ab, ab.data(), 16, cudaMemcpyHostToDevice);
    pint_ctx ctx{};
    for (int rep = 0; rep < 3; ++rep) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, ctx.stream);
        launch_scalar_sweep(&ctx, PINT_SWEEP_EXACT, N, M, d_x, 0, d_w, d_v, d_ab, d_ab + 1, 0, 0.1, d_y, d_y + N, d_e);
        cudaEventRecord(e1, ctx.stream);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long p[3];
        cudaMemcpyFromSymbol(p, g_sweep_prof, sizeof p);
        std::printf("{\"N\": %d, \"M\": %d, \"ms\": %.4f, \"per_slice_cycles\": {\"terms\": %.0f, \"sum\": %.0f, "
                    "\"barrier\": %.0f}, \"sum_cycles_per_term\": %.2f}\n",
                    N, M, ms, double(p[0]) / N, double(p[1]) / N, double(p[2]) / N, double(p[1]) / N / M);
    }
    return 0;
}
