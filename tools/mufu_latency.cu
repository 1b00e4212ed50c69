#include <cstdio>
#define PINT_ENSEMBLE_STANDALONE

__global__ void k(double seed, double* out, long long* cyc) {
    double a = seed + threadIdx.x * 1e-3;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < 1024; ++i) { double r; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a)); a = r; }
    long long t1 = clock64();
#pragma unroll 16
    for (int i = 0; i < 1024; ++i) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a)); a = r; }
    long long t2 = clock64();
#pragma unroll 16
    for (int i = 0; i < 1024; ++i) a = __dsqrt_rn(a) + 0.25;
    long long t3 = clock64();
#pragma unroll 16
    for (int i = 0; i < 1024; ++i) a = __ddiv_rn(1.0, a) + 0.5;
    long long t4 = clock64();
    float f = (float)a;
#pragma unroll 16
    for (int i = 0; i < 1024; ++i) { float r; asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(f)); f = r; }
    long long t5 = clock64();
#pragma unroll 16
    for (int i = 0; i < 1024; ++i) { a = (double)(float)a + 0.5; }
    long long t6 = clock64();
    double y = 0.5 + threadIdx.x * 1e-3;
    const double h4 = 4.0 * 1e-4;
    long long t7 = clock64();
#pragma unroll 4
    for (int i = 0; i < 1024; ++i) {
        const double disc = __dsub_rn(1.0, __dmul_rn(h4, y));
        y = __ddiv_rn(__dmul_rn(2.0, y), __dadd_rn(1.0, __dsqrt_rn(disc)));
    }
    long long t8 = clock64();
    if (threadIdx.x == 0) cyc[6] = t8 - t7;
    out[threadIdx.x] = a + f + y;
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5; }
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 256 * 8); cudaMalloc(&c, 64);
    for (int r = 0; r < 2; ++r) { k<<<1, 32>>>(1.7, o, c); cudaDeviceSynchronize(); }
    long long h[7]; cudaMemcpy(h, c, 56, cudaMemcpyDeviceToHost);
    printf("{\"rsqrt64h\": %.1f, \"rcp64h\": %.1f, \"dsqrt_rn+dadd\": %.1f, \"ddiv_rn+dadd\": %.1f, \"rcp_f32\": %.1f, \"f2f_roundtrip+dadd\": %.1f, \"riccati_step\": %.1f}\n",
           h[0] / 1024.0, h[1] / 1024.0, h[2] / 1024.0, h[3] / 1024.0, h[4] / 1024.0, h[5] / 1024.0, h[6] / 1024.0);
}
