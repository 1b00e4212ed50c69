// Wave-equation slice maps: the affine propagator of the leapfrog
// discretisation of u_tt = u_xx on the Chebyshev extrema grid, built on the device.
//
// Replaces build_affine_propagator (nievergelt.cpp:53-66) driving make_wave_linear_problem's
// integrate closure (pde_problems.cpp:142-172) -> leapfrog_integrate (ode_core.cpp:65-77) with
// apply_D2 = matvec(D2, v) (linalg.cpp:17-26). State of a trajectory = [u^m; u^{m-1}] (2d).
//
// Lane = trajectory (basis column e_j of the 2d-dimensional state, or the zero state for c: the
// wave problem has no forcing). Per step and lane: acc_i = sum_k D2(i,k) u_k in matvec's
// sequential order, then u_new_i = (2 u_i - u_prev_i) + dt^2 acc_i with the reference's roundings
// (ode_core.cpp:71-72). D2 is staged once per CTA in shared memory (broadcast reads); the state is
// lane-interleaved in shared memory. Bit-exact vs the reference.
#include "pint_internal.cuh"

namespace {

struct WavePlan {
    int d;               // interior points (M - 1); state dimension 2d
    long long N;         // slices (build) or 1 (integrate)
    long long K;         // columns per slice: 2d + 1 (build) or caller columns (integrate)
    const double* D2;    // d x d row-major
    const int64_t* steps;  // per slice
    const double* h;       // per slice leapfrog step
    double* maps;          // build: augmented maps; integrate: unused
    long long ldm;
    double* y;             // integrate: K states of 2d, in place
};

// Dynamic smem: D2[d*d] | cur[d][32] | prev[d][32] | acc[d][32]
template <bool kBuild>
__global__ void __launch_bounds__(32) wave_columns_kernel(WavePlan P) {
    extern __shared__ __align__(16) double smem[];
    const int d = P.d;
    const int lane = threadIdx.x;
    const long long warps_per_slice = (P.K + 31) / 32;
    const long long slice = kBuild ? blockIdx.x / warps_per_slice : 0;
    const long long col = (blockIdx.x - slice * warps_per_slice) * 32 + lane;
    const bool active = col < P.K;
    double* D2 = smem;
    double* cur = D2 + static_cast<long long>(d) * d + lane;
    double* prev = cur + 32 * d;
    double* acc = prev + 32 * d;
    for (int i = lane; i < d * d; i += 32) D2[i] = P.D2[i];
    // initial state: basis e_col (col < 2d) or zero (col == 2d, the c run) / caller data
    for (int i = 0; i < d; ++i) {
        double u, v;
        if (kBuild) {
            u = (col == i) ? 1.0 : 0.0;
            v = (col == d + i) ? 1.0 : 0.0;
        } else {
            u = active ? P.y[col * 2 * d + i] : 0.0;
            v = active ? P.y[col * 2 * d + d + i] : 0.0;
        }
        cur[i * 32] = u;
        prev[i * 32] = v;
    }
    __syncwarp();
    const long long S = P.steps[slice];
    const double h = P.h[slice];
    const double dt2 = __dmul_rn(h, h);  // ode_core.cpp:68
    for (long long s = 0; s < S; ++s) {
        for (int i = 0; i < d; ++i) {  // apply_D2: matvec row i, sequential in k (linalg.cpp:20-22)
            const double* row = D2 + static_cast<long long>(i) * d;
            double a = 0.0;
            for (int k = 0; k < d; ++k) a = __dadd_rn(a, __dmul_rn(row[k], cur[k * 32]));
            acc[i * 32] = a;
        }
        for (int i = 0; i < d; ++i) {  // acc = 2 y_curr - y_prev + dt2 acc (ode_core.cpp:71-72)
            const double c = cur[i * 32];
            const double nxt = __dadd_rn(__dsub_rn(__dmul_rn(2.0, c), prev[i * 32]), __dmul_rn(dt2, acc[i * 32]));
            prev[i * 32] = c;
            cur[i * 32] = nxt;
        }
    }
    if (!active) return;
    if (kBuild) {  // column col of slice's augmented map: rows [u; u_prev]
        double* g = P.maps + slice * (2LL * d) * P.ldm + col;
        for (int i = 0; i < d; ++i) {
            g[static_cast<long long>(i) * P.ldm] = cur[i * 32];
            g[static_cast<long long>(d + i) * P.ldm] = prev[i * 32];
        }
    } else {
        for (int i = 0; i < d; ++i) {
            P.y[col * 2 * d + i] = cur[i * 32];
            P.y[col * 2 * d + d + i] = prev[i * 32];
        }
    }
}

template <bool kBuild>
int launch_wave(pint_ctx* ctx, const WavePlan& P, long long blocks, const char* what) {
    const size_t smem = sizeof(double) * (static_cast<size_t>(P.d) * P.d + 96ull * P.d);
    if (smem > 227 * 1024) return pint_set_error(ctx, PINT_E_INVALID, "wave: grid too large for shared memory");
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(wave_columns_kernel<kBuild>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
    if (blocks <= 0) return PINT_OK;
    wave_columns_kernel<kBuild><<<static_cast<unsigned>(blocks), 32, smem, ctx->stream>>>(P);
    return pint_check_launch(ctx, what);
}

}  // namespace

int launch_wave_build(pint_ctx* ctx, int64_t d, int64_t N, const double* D2, const int64_t* steps, const double* h,
                      double* maps) {
    if (d < 1 || N < 0) return pint_set_error(ctx, PINT_E_INVALID, "wave_build: bad sizes");
    WavePlan P{};
    P.d = static_cast<int>(d);
    P.N = N;
    P.K = 2 * d + 1;
    P.D2 = D2;
    P.steps = steps;
    P.h = h;
    P.maps = maps;
    P.ldm = pint_affine_ldm(2 * d);
    return launch_wave<true>(ctx, P, N * ((P.K + 31) / 32), "wave_columns_kernel<build>");
}

int launch_wave_integrate(pint_ctx* ctx, int64_t d, int64_t K, const double* D2, const int64_t* steps,
                          const double* h, double* y) {
    if (d < 1 || K < 0) return pint_set_error(ctx, PINT_E_INVALID, "wave_integrate: bad sizes");
    WavePlan P{};
    P.d = static_cast<int>(d);
    P.N = 1;
    P.K = K;
    P.D2 = D2;
    P.steps = steps;
    P.h = h;
    P.y = y;
    return launch_wave<false>(ctx, P, (K + 31) / 32, "wave_columns_kernel<integrate>");
}
