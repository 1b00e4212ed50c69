// Per-slice cost of the one-warp EXACT sweep variants (M <= 8), clock64 around the slice loop.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -std=c++17 -I../include
//        -I../paper_1304_6514_b200/csrc tools/sweep_slice_micro.cu -o tools/_sweep_slice_micro
// V0: lane k = node k, __ddiv_rn, ballot + shuffles (pint_dev::slice_eval_small)
// V2: lane k = node k, div_rn_scaled below (branch-free, scaled), ballot + shuffles
// V7: a shuffle + add round alone; V8 / V9: one dependent __ddiv_rn / div_rn_scaled alone
// Measured on B200 (cycles a slice, M = 4 / 7): V0 ~480 / 563, V2 481 / 619, V7 134, V8 136, V9 130;
// every lane computing all M terms with div_rn_scaled (no shuffles, no ballot): 632 / 1343.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "pint_internal.cuh"

// a / b for any b: both scaled by the power of 2 that brings |b| into [1, 2), then
// pint_dev::div_rn_fast; ok cleared outside its window
__device__ __forceinline__ double div_rn_scaled(double a, double b, bool& ok) {
    const unsigned eb = (static_cast<unsigned>(__double2hiint(b)) >> 20) & 0x7ffu;
    const double sc = __hiloint2double(static_cast<int>((2046u - eb) << 20), 0);
    const double as = __dmul_rn(a, sc), bs = __dmul_rn(b, sc);
    const unsigned ah = static_cast<unsigned>(__double2hiint(as)) & 0x7fffffffu;
    ok &= (eb - 1u < 2045u) & (ah - ((1023u - 900u) << 20) < (1800u << 20));
    return pint_dev::div_rn_fast(as, bs);
}

template <int MM, int V>
__global__ void sweep(int N, int M, const double* X, const double* W, const double* Vals, double y0, double* lam,
                      long long* cyc) {
    extern __shared__ double sm[];  // (staged like the library kernels: X | W | V)
    const int lane = threadIdx.x;
    for (int i = lane; i < M; i += 32) sm[i] = X[i], sm[M + i] = W[i];
    for (int i = lane; i < N * M; i += 32) sm[2 * M + i] = Vals[i];
    __syncwarp();
    X = sm;
    W = sm + M;
    Vals = sm + 2 * M;
    const bool live = lane < M;
    double y = y0;
    const long long c0 = clock64();
    for (int j = 0; j < N; ++j) {
        const double* V_ = Vals + j * M;
        if (V == 8 || V == 9) {  // one dependent quotient per slice: the division latency alone
            bool ok = true;
            const double d = __dsub_rn(y, 3.0);
            y = V == 8 ? __ddiv_rn(1.5, d) : div_rn_scaled(1.5, d, ok);
            if (!ok) y = 0.0;
        } else if (V == 7) {  // the slice's adds and a shuffle round, no division
            const double vk = live ? V_[lane] : 0.0;
            const double rv = __dsub_rn(y, vk);
            double num = 0.0;
#pragma unroll
            for (int k = 0; k < MM; ++k) num = __dadd_rn(num, __shfl_sync(0xffffffffu, rv, k));
            y = __dmul_rn(num, 0.25);
        } else if (V == 10) {  // V0 without the snap branch: the snap selects at the end
            const double xk = live ? X[lane] : 0.0, wk = live ? W[lane] : 0.0, vk = live ? V_[lane] : 0.0;
            const double diff = __dsub_rn(y, xk);
            const unsigned snap =
                __ballot_sync(0xffffffffu, live && fabs(diff) <= __dmul_rn(1e-14, fmax(1.0, fabs(xk))));
            const double r = live ? __ddiv_rn(wk, diff) : -0.0;
            const double rv = live ? __dmul_rn(r, vk) : -0.0;
            const double vs = __shfl_sync(0xffffffffu, vk, snap ? __ffs(snap) - 1 : 0);
            double num = 0.0, den = 0.0;
            double tn[MM], td[MM];
#pragma unroll
            for (int k = 0; k < MM; ++k)
                tn[k] = __shfl_sync(0xffffffffu, rv, k), td[k] = __shfl_sync(0xffffffffu, r, k);
#pragma unroll
            for (int k = 0; k < MM; ++k) {
                num = __dadd_rn(num, tn[k]);
                den = __dadd_rn(den, td[k]);
            }
            const double q = __ddiv_rn(num, den);
            y = snap ? vs : q;
        } else if (V == 0) {
            y = pint_dev::slice_eval_small<MM>(y, X, W, V_, M, lane);
        } else {
            const double xk = live ? X[lane] : 0.0, wk = live ? W[lane] : 0.0, vk = live ? V_[lane] : 0.0;
            const double diff = __dsub_rn(y, xk);
            const unsigned snap =
                __ballot_sync(0xffffffffu, live && fabs(diff) <= __dmul_rn(1e-14, fmax(1.0, fabs(xk))));
            double r;
            bool ok = true;
            if (V == 0) r = live ? __ddiv_rn(wk, diff) : -0.0;
            else r = live ? div_rn_scaled(wk, diff, ok) : -0.0;
            const double rv = live ? __dmul_rn(r, vk) : -0.0;
            if (snap) {
                y = __shfl_sync(0xffffffffu, vk, __ffs(snap) - 1);
            } else {
                double num = 0.0, den = 0.0;
                double tn[MM], td[MM];
#pragma unroll
                for (int k = 0; k < MM; ++k)
                    tn[k] = __shfl_sync(0xffffffffu, rv, k), td[k] = __shfl_sync(0xffffffffu, r, k);
#pragma unroll
                for (int k = 0; k < MM; ++k) {
                    num = __dadd_rn(num, tn[k]);
                    den = __dadd_rn(den, td[k]);
                }
                if (V == 0) {
                    y = __ddiv_rn(num, den);
                } else {
                    const double q = div_rn_scaled(num, den, ok);
                    const bool all = __all_sync(0xffffffffu, ok || !live);
                    y = all ? q : __ddiv_rn(num, den);  // (not exact when a term was not: test only)
                }
            }
        }
        if (lane == 0) lam[j] = y;
    }
    if (lane == 0) *cyc = clock64() - c0;
}

template <int MM, int V>
void run(int N, int M, const double* dX, const double* dW, const double* dV, double* dl, long long* dc,
         std::vector<double>& out) {
    for (int rep = 0; rep < 3; ++rep) sweep<MM, V><<<1, 32, 8 * (2 * M + N * M)>>>(N, M, dX, dW, dV, 1.0, dl, dc);
    long long c;
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    out.resize(N);
    cudaMemcpy(out.data(), dl, 8 * N, cudaMemcpyDeviceToHost);
    std::printf("  V%d MM=%d: %.0f cycles per slice\n", V, MM, double(c) / N);
}

int main() {
    const int N = 512;
    for (int M : {4, 7}) {
        std::vector<double> x(M), w(M), v(N * M);
        for (int k = 0; k < M; ++k) x[k] = 1.0 - std::cos(M_PI * k / (M - 1));  // [0, 2]
        for (int k = 0; k < M; ++k) {
            double acc = 1.0;
            for (int j = 0; j < M; ++j)
                if (j != k) acc /= (x[k] - x[j]);
            w[k] = acc;
        }
        for (int j = 0; j < N; ++j)
            for (int k = 0; k < M; ++k) v[j * M + k] = 0.1 + 0.9 * x[k] + 0.05 * std::sin(3 * x[k] + j);
        double *dX, *dW, *dV, *dl;
        long long* dc;
        cudaMalloc(&dX, 8 * M);
        cudaMalloc(&dW, 8 * M);
        cudaMalloc(&dV, 8 * N * M);
        cudaMalloc(&dl, 8 * N);
        cudaMalloc(&dc, 8);
        cudaMemcpy(dX, x.data(), 8 * M, cudaMemcpyHostToDevice);
        cudaMemcpy(dW, w.data(), 8 * M, cudaMemcpyHostToDevice);
        cudaMemcpy(dV, v.data(), 8 * N * M, cudaMemcpyHostToDevice);
        std::printf("M = %d, N = %d\n", M, N);
        std::vector<double> l0, l2;
        if (M <= 4) {
            run<4, 0>(N, M, dX, dW, dV, dl, dc, l0);
            run<4, 2>(N, M, dX, dW, dV, dl, dc, l2);
        } else {
            run<8, 0>(N, M, dX, dW, dV, dl, dc, l0);
            run<8, 2>(N, M, dX, dW, dV, dl, dc, l2);
        }
        std::printf("  V2 == V0: %d\n", l2 == l0);
        std::vector<double> l10;
        if (M <= 4) run<4, 10>(N, M, dX, dW, dV, dl, dc, l10);
        else run<8, 10>(N, M, dX, dW, dV, dl, dc, l10);
        std::printf("  V10 == V0: %d\n", l10 == l0);
        std::vector<double> l8, l9, l7;
        run<4, 8>(N, M, dX, dW, dV, dl, dc, l8);
        run<4, 9>(N, M, dX, dW, dV, dl, dc, l9);
        run<8, 7>(N, M, dX, dW, dV, dl, dc, l7);
        std::printf("  V9 == V8: %d\n", l8 == l9);
    }
    return 0;
}
