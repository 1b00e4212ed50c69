// Check rcp.approx.ftz.f64 + 2 Newton steps against IEEE 1/x over a log sweep (tolerance sweep).
#include <cstdio>
#include <cmath>
__device__ double rcp_nr(double d) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    double e = fma(-d, r, 1.0);
    r = fma(r, e, r);
    e = fma(-d, r, 1.0);
    return fma(r, e, r);
}
__global__ void k(const double* x, double* out, double* raw, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) { out[i] = rcp_nr(x[i]); double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x[i])); raw[i] = r; }
}
int main() {
    const int n = 4096;
    double h[n], o[n], rw[n];
    for (int i = 0; i < n; ++i) h[i] = (i % 2 ? -1 : 1) * pow(10.0, -15.0 + 17.0 * i / n) * (1.0 + 0.37 * (i % 7));
    double *dx, *dy, *dr;
    cudaMalloc(&dx, sizeof h); cudaMalloc(&dy, sizeof h); cudaMalloc(&dr, sizeof h);
    cudaMemcpy(dx, h, sizeof h, cudaMemcpyHostToDevice);
    k<<<n / 256, 256>>>(dx, dy, dr, n);
    cudaMemcpy(o, dy, sizeof h, cudaMemcpyDeviceToHost);
    cudaMemcpy(rw, dr, sizeof h, cudaMemcpyDeviceToHost);
    double worst = 0; int bad = 0;
    for (int i = 0; i < n; ++i) {
        double rel = fabs(o[i] * h[i] - 1.0);
        if (!(rel < 1e-15)) { if (bad < 8) printf("x=%.17g rcp=%.17g raw=%.17g rel=%g\n", h[i], o[i], rw[i], rel); ++bad; }
        if (rel > worst) worst = rel;
    }
    printf("bad %d worst %g\n", bad, worst);
}
