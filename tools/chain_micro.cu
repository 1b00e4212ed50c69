// Section timing of affine_chain_cluster_kernel / affine_chain_wide_kernel (-DPINT_CHAIN_PROF):
//   tools/_chain_micro n N      (PINT_WIDE_CHAIN=2 PINT_WIDE_W=1|2|4: the wide chain)
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1304_6514_b200/csrc/compose.cu"

void* pint_tensor_map_encoder() {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess) p = nullptr;
    return p;
}
void pint_kernel_attrs(const void* f) {
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
}

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
extern "C" int64_t pint_affine_ldm(int64_t n) { return (n + 1 + 3) / 4 * 4; }

int main(int argc, char** argv) {
    const int n = argc > 1 ? std::atoi(argv[1]) : 128;
    const int N = argc > 2 ? std::atoi(argv[2]) : 64;
    const long long ldm = pint_affine_ldm(n);
    std::vector<double> h(static_cast<size_t>(N) * n * ldm, 1e-3), y0(n, 1.0);
    double *d, *dy0, *dy;
    cudaMalloc(&d, 8 * h.size());
    cudaMalloc(&dy0, 8 * n);
    cudaMalloc(&dy, 8 * n);
    cudaMemcpy(d, h.data(), 8 * h.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dy0, y0.data(), 8 * n, cudaMemcpyHostToDevice);
    pint_ctx ctx;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        launch_affine_chain(&ctx, n, N, d, dy0, dy);
        cudaEventRecord(e1);
        cudaDeviceSynchronize();
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        std::printf("chain n=%d N=%d: %.3f ms (%.2f us per map) %s\n", n, N, ms, 1e3 * ms / N,
                    cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
