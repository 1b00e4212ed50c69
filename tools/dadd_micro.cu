// Dependent-sum cost per column pair for the chain kernels: s = (s + g.x*y.x) + g.y*y.y over 512
// pairs, (a) operands in registers, (b) operands from shared memory 8 pairs ahead (LDS.128),
// (c) as (b) with the y operand also an LDS.128 broadcast.    nvcc ... tools/dadd_micro.cu
#include <cstdio>
__global__ void k(double* out, int reps, int mode) {
    __shared__ __align__(16) double g[32 * 132];
    __shared__ __align__(16) double yv[1040];
    const int lane = threadIdx.x;
    for (int i = lane; i < 32 * 132; i += 32) g[i] = 1.0 + 1e-9 * i;
    for (int i = lane; i < 1040; i += 32) yv[i] = 1e-3 * i;
    __syncwarp();
    double s = 0.0;
    const long long t0 = clock64();
    const double2* g2 = reinterpret_cast<const double2*>(g + lane * 132);
    const double2* y2 = reinterpret_cast<const double2*>(yv);
    for (int r = 0; r < reps; ++r) {
        if (mode == 0) {
            double2 a = g2[0], b = y2[lane];
#pragma unroll 8
            for (int p = 0; p < 512; ++p) {
                s = __dadd_rn(s, __dmul_rn(a.x, b.x));
                s = __dadd_rn(s, __dmul_rn(a.y, b.y));
                a.x += 1e-300;  // keep the compiler from folding
            }
        } else {
            double2 gv[8], yq[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) gv[u] = g2[u], yq[u] = y2[u];
#pragma unroll 1
            for (int p = 0; p < 512; p += 8) {
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    s = __dadd_rn(s, __dmul_rn(gv[u].x, yq[u].x));
                    s = __dadd_rn(s, __dmul_rn(gv[u].y, yq[u].y));
                    gv[u] = g2[(p + 8 + u) & 63];
                    if (mode == 2) yq[u] = y2[(p + 8 + u) & 63];
                }
            }
        }
    }
    const long long t1 = clock64();
    if (lane == 0) printf("mode %d: %.1f cycles per pair\n", mode, double(t1 - t0) / (512.0 * reps));
    out[lane] = s;
}
int main() {
    double* o;
    cudaMalloc(&o, 8 * 32);
    for (int m = 0; m < 3; ++m) { k<<<1, 32>>>(o, 20, m); cudaDeviceSynchronize(); }
    return 0;
}
