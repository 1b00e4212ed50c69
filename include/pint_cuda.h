/* pint_cuda.h — C ABI of the B200-native Nievergelt slice-map path (libpint_cuda.so).
 *
 * Plain pointers and sizes only; no C++ or torch types cross this boundary. The C++ drop-in
 * library (paper_1304_6514_b200/include/pint/ headers, libpint_b200.so) and the Python host
 * (paper_1304_6514_b200/capi.py, ctypes) are both thin callers of these entry points.
 * Each entry point names the reference interface it replaces (file:line under
 * /root/reference/proj). Ctypes / C++ bindings a maintainer adds are shown in INTEGRATION.md.
 *
 * Conventions
 *  - `_dev` entry points take DEVICE pointers, enqueue on the context's stream and return
 *    immediately. Task failures (e.g. NoRealRoot) are latched in the context's device-side
 *    failure record; read it with pint_fail_read() after pint_ctx_sync().
 *  - Entry points without `_dev` take HOST pointers, copy in/out and synchronise.
 *  - Slice maps of a linear problem ("affine maps") are stored as one row-major augmented
 *    block per slice: rows i < n, columns [0, n) = G, column n = c, leading dimension
 *    ldm = pint_affine_ldm(n) (n + 1 rounded up to a multiple of 4), slice j at j * n * ldm.
 *  - Every function returns PINT_OK or a PINT_E_* code; pint_ctx_last_error() has the text.
 */
#ifndef PINT_CUDA_H
#define PINT_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: one per reference exception type (errors.hpp:9-43) ---- */
enum {
    PINT_OK = 0,
    PINT_E_NO_REAL_ROOT = 1,        /* NoRealRoot          errors.hpp:10 */
    PINT_E_SINGULAR = 2,            /* SingularSystem      errors.hpp:15 */
    PINT_E_BAD_GRID = 3,            /* BadGrid             errors.hpp:20 */
    PINT_E_NON_INTEGER_STEPS = 4,   /* NonIntegerStepCount errors.hpp:25 */
    PINT_E_DUPLICATE_NODES = 5,     /* DuplicateNodes      errors.hpp:29 */
    PINT_E_RANGE_RETRY = 6,         /* internal: a fast-division range check tripped; the
                                       host-buffer entry points re-run with the guarded kernel */
    PINT_E_SERIALIZED = 7,          /* internal: the chain of pint_heat_build_chain_dev could not
                                       run beside the build (kernels serialised, e.g. under a
                                       profiler); the maps are complete: re-run the compose */
    PINT_E_INVALID = 16,            /* bad argument to this ABI */
    PINT_E_CUDA = 17,               /* CUDA runtime failure (no CPU fallback exists) */
    PINT_E_NO_DEVICE = 18,
    PINT_E_NCCL = 19                /* multi-GPU transport failure (NCCL or a caller callback) */
};

typedef struct pint_ctx pint_ctx;

/* One time slice (ode_core.hpp:42-48). `steps`/`dt` follow decompose (ode_core.cpp:26-45). */
typedef struct {
    double t_begin;
    double t_end;
    int64_t steps;
    double dt;
} pint_slice;

/* Lowest failing task, parallel_map semantics (exec_harness.hpp:88-99). index < 0: none. */
typedef struct {
    int64_t index;
    int32_t code;   /* PINT_E_* of the failing task */
    int32_t pad;
    double value;   /* the offending quantity (Riccati discriminant, zero pivot row, ...) */
} pint_fail;

/* Scalar right-hand sides on the device. The reference integrator ignores ScalarIVP::rhs and
 * always runs backward-Euler Riccati (nievergelt.cpp:28-35); the others are EXTENSIONS. */
enum {
    PINT_RHS_RICCATI_BE = 0,  /* y' = y^2, closed-form backward Euler (ode_core.cpp:47-53) */
    PINT_RHS_LOGISTIC_RK4 = 1 /* y' = r y (1 - y/K), classical RK4 */
};
enum { PINT_F64 = 0, PINT_F32 = 1 };
enum { PINT_WEIGHTS_PRODUCT = 0, PINT_WEIGHTS_CLOSED2 = 1 };
enum { PINT_SWEEP_EXACT = 0, PINT_SWEEP_TREE = 1 };        /* barycentric sum order */
enum { PINT_COMPOSE_CHAIN = 0, PINT_COMPOSE_TREE = 1 };    /* affine composition */
enum { PINT_NODES_FIRST_KIND = 0, PINT_NODES_SECOND_KIND = 1 };

typedef struct {
    int32_t kind;      /* PINT_RHS_* */
    int32_t precision; /* PINT_F64 / PINT_F32 (F32 only for LOGISTIC_RK4) */
    double r;          /* logistic rate */
    double K;          /* logistic capacity */
} pint_scalar_rhs;

/* Report of a full run, the subset of RunReport (nievergelt.hpp:42-62) the device produces. */
typedef struct {
    int64_t message_count;
    int64_t bytes_communicated;
    int64_t extrapolation_count;
    double device_ms;        /* CUDA-event time of the device work */
    double total_ms;         /* host wall time of the call (T_total analogue) */
    int64_t traj_steps;      /* sum over slices of trajectories x steps */
    int64_t gpu_launches;    /* kernels this call launched */
    int64_t h2d_bytes;       /* host->device bytes this call copied */
    int64_t d2h_bytes;       /* device->host bytes this call copied */
    double compose_ms;       /* CUDA-event time of the composition sweep alone (apply_cost) */
} pint_report;

/* ---- context ---- */
/* CUDA devices visible to this process (0 without a GPU) */
int pint_device_count(void);
int pint_ctx_create(int device, pint_ctx** out);
void pint_ctx_destroy(pint_ctx* ctx);
const char* pint_ctx_last_error(const pint_ctx* ctx);
int pint_ctx_sync(pint_ctx* ctx);
/* the cudaStream_t the context enqueues on (as void*); set_stream adopts a caller stream */
void* pint_ctx_stream(pint_ctx* ctx);
int pint_ctx_set_stream(pint_ctx* ctx, void* stream);
/* number of kernels launched through this context so far */
int64_t pint_ctx_launch_count(const pint_ctx* ctx);
/* read (and clear) the device-side failure record; syncs the stream */
int pint_fail_read(pint_ctx* ctx, pint_fail* out);
const char* pint_version(void);
/* test hook: K device-side failures (task idx[t], code[t], value[t]) recorded concurrently through
   the same path the kernels use; pint_fail_read must return the lowest index with ITS code/value */
int pint_debug_fail_inject(pint_ctx* ctx, int64_t K, const int64_t* idx, const int* code,
                           const double* value);

/* ---- host-side tables (bit-identical to the reference's own host arithmetic) ---- */
/* steps_for (ode_core.cpp:18-24) */
int64_t pint_steps_for(double width, double dt);
/* decompose (ode_core.cpp:26-45): writes N slices */
int pint_decompose(double t0, double T, int64_t N, double dt, pint_slice* out);
/* cheb_nodes / cheb_nodes_second_kind (interp.cpp:21-41) */
int pint_sample_nodes(int kind, int64_t M, double a, double b, double* out);
/* augmented map leading dimension, see conventions */
int64_t pint_affine_ldm(int64_t n);

/* ---- K1: scalar ensemble (replaces parallel_map over N*M tasks, nievergelt.cpp:170-182) ----
 * endpoints[j*M + m] = slice j's end state from nodes[m] after steps[j] steps of dt[j].
 * nodes/endpoints are double (PINT_F64) or float (PINT_F32). per_slice_ns (may be NULL) gets
 * the summed device time of the slice's thread blocks (RunReport::per_slice_compute). */
int pint_scalar_ensemble_dev(pint_ctx* ctx, const pint_scalar_rhs* rhs, int64_t N, int64_t M,
                             const int64_t* steps, const double* dt, const void* nodes,
                             void* endpoints, unsigned long long* per_slice_ns);

/* ---- K2: barycentric weights (interp.cpp:43-55, product form; or closed-form EXTENSION) */
int pint_bary_weights_dev(pint_ctx* ctx, int kind, int64_t M, const double* nodes, double* w);

/* ---- K2: scalar composition sweep (compose_sweep, nievergelt.cpp:68-88 + interp_eval,
 * interp.cpp:68-80). values[j*M + m]; nodes/weights per slice at stride node_stride (0 = all
 * slices share one set); a/b per slice at stride ab_stride (0 or 1). Writes lambdas[j]
 * (may be NULL), *y_out and *extrapolations (device pointers). mode: PINT_SWEEP_EXACT keeps the
 * reference's sequential sum order (bit-exact); PINT_SWEEP_TREE sums by warp tree. */
int pint_scalar_sweep_dev(pint_ctx* ctx, int mode, int64_t N, int64_t M, const double* nodes,
                          int64_t node_stride, const double* weights, const double* values,
                          const double* a, const double* b, int64_t ab_stride, double y0,
                          double* lambdas, double* y_out, long long* extrapolations);

/* ---- K3: heat slice maps (build_affine_propagator, nievergelt.cpp:53-66, driving the
 * make_heat_problem integrate closure, pde_problems.cpp:76-100). Per-step coefficient tables
 * come from pint_heat_coefficients (host, glibc sin/cos like the reference). ---- */
/* total steps over the slices */
int64_t pint_heat_total_steps(const pint_slice* slices, int64_t N);
/* Host tables: step_off[N+1] (prefix sums of steps); per step q: r[q] = (h a(t)) / dx^2,
 * fa[q] = -sin t, fb[q] = ((a(t) pi) pi) cos t; sx[i] = sin(pi (i+1) dx). n = interior points. */
int pint_heat_coefficients(double dx, const pint_slice* slices, int64_t N, int64_t* step_off,
                           double* r, double* fa, double* fb, double* sx, int64_t* n_out);
/* doubles of the per-step records of N slices with at most S steps each (pint_heat_factor_dev) */
int64_t pint_heat_records_size(int64_t n, int64_t N, int64_t S);
/* Shared tridiagonal factor per (slice, step) — the Thomas forward pivots (linalg.cpp:77-93),
 * computed once per step instead of once per trajectory — plus the forcing increments. Layout
 * (internal; size from pint_heat_records_size): for n up to ~200, slice-group blocks
 * [S][N/32] of {(-r, 0), (p_i, RN(1/p_i))}[n+1][32] | h*b_i[n][32] | c_i[n][32]; for larger n,
 * slice-major records [N][S] of {-r} | (p_i, RN(1/p_i)) | h*b_i | c_i. step_off/slice_dt/sx (device) and r/fa/fb (device,
 * step_off[N] entries) come from pint_heat_coefficients. */
int pint_heat_factor_dev(pint_ctx* ctx, int64_t n, int64_t N, int64_t S, const int64_t* step_off,
                         const double* slice_dt, const double* r, const double* fa,
                         const double* fb, const double* sx, double* records);
/* Build all N augmented maps into maps (N * n * ldm doubles). step_off/slice_dt/sx are device
 * copies of the host tables; per_slice_ns (may be NULL) accumulates per-slice device time.
 * guarded = 0: fast exact division, dividends range-checked off the critical path (forced lanes
 * per row, basis lanes through a running minimum); a tripped check latches PINT_E_RANGE_RETRY in the failure record and the caller re-runs with
 * guarded = 1 (IEEE division on the chain outside [2^-960, 2^997]). Both are bit-exact. */
int pint_heat_build_dev(pint_ctx* ctx, int64_t n, int64_t N, int64_t S, const int64_t* step_off,
                        const double* slice_dt, const double* records, const double* sx,
                        double* maps, unsigned long long* per_slice_ns, int guarded);
/* Integrate K state vectors y[k*n ...] in place through the `steps` steps of ONE slice whose device
 * tables (pint_heat_coefficients with N = 1: step_off[2], slice_dt[1], r/fa/fb[steps], sx[n]) are
 * given: the integrate closure (pde_problems.cpp:86-98) or run_serial (nievergelt.cpp:126-143),
 * bit-exact. Records are built in bounded chunks internally (O(chunk), not O(steps), scratch).
 * guarded as pint_heat_build_dev (read the failure record; re-run with guarded = 1 on RANGE_RETRY). */
int pint_heat_integrate_dev(pint_ctx* ctx, int64_t n, int64_t K, int64_t steps, const int64_t* step_off,
                            const double* slice_dt, const double* r, const double* fa,
                            const double* fb, const double* sx, int with_forcing, double* y, int guarded);

/* ---- K3f: heat slice maps, TOLERANCE build (EXTENSION: the same maps as pint_heat_build_dev —
 * build_affine_propagator, nievergelt.cpp:53-66 — in a different operation order, <= 1e-12 relative
 * to the exact maps; north_star allows this tolerance for trajectory end states). Each step is a
 * row-partitioned Thomas solve (linalg.cpp:77-93) with all rows in registers: one FMA per row on
 * the dependent chain, partition carries by shuffle scans, fix-ups with per-(slice, step) spike
 * vectors. Supports n <= 768 (pint_heat_fast_records_size returns 0 beyond). ---- */
enum { PINT_BUILD_EXACT = 0, PINT_BUILD_FAST = 1 };
int64_t pint_heat_fast_records_size(int64_t n, int64_t N, int64_t S);
/* per-(slice, step) coefficients from the same device tables as pint_heat_factor_dev; slices with
 * fewer than S steps are padded with identity steps */
int pint_heat_fast_factor_dev(pint_ctx* ctx, int64_t n, int64_t N, int64_t S, const int64_t* step_off,
                              const double* slice_dt, const double* r, const double* fa,
                              const double* fb, const double* sx, double* records);
/* all N augmented maps (layout as pint_heat_build_dev) from pint_heat_fast_factor_dev's records */
int pint_heat_fast_build_dev(pint_ctx* ctx, int64_t n, int64_t N, int64_t S, const double* records,
                             double* maps);

/* ---- K4: affine composition (compose_sweep, nievergelt.cpp:90-110) ----
 * CHAIN: y <- G_j y + c_j in slice order, rows as sequential dots (bit-exact vs matvec,
 * linalg.cpp:17-26). TREE: log-depth pairwise products on FP64 tensor cores (DMMA), then one
 * apply (EXTENSION, <= 1e-12 relative). maps is consumed (overwritten) by TREE; scratch must hold
 * ceil(N/2) maps (TREE only; may be NULL for CHAIN). composed (may be NULL) receives the
 * composed augmented map (TREE only). y0, y: device n-vectors. */
int pint_affine_compose_dev(pint_ctx* ctx, int mode, int64_t n, int64_t N, double* maps,
                            double* scratch, const double* y0, double* y, double* composed);
/* K3 + K4 fused in time: all N maps (pint_heat_build_dev's exact build, guarded as there) and the
 * bit-exact CHAIN to y. For n in [282, 520] the chain runs concurrently with the build on the
 * context's side stream, fetching each map as soon as all its builder CTAs have stored it;
 * otherwise build then chain. Replaces the build + compose_sweep pair of run_nievergelt
 * (nievergelt.cpp:237-246). y0, y: device n-vectors; result bit-identical to build + CHAIN. */
int pint_heat_build_chain_dev(pint_ctx* ctx, int64_t n, int64_t N, int64_t S, const int64_t* step_off,
                              const double* slice_dt, const double* records, const double* sx,
                              double* maps, const double* y0, double* y, int guarded);
/* the same with the TOLERANCE build (pint_heat_fast_factor_dev's records) */
int pint_heat_fast_build_chain_dev(pint_ctx* ctx, int64_t n, int64_t N, int64_t S, const double* records,
                                   double* maps, const double* y0, double* y);
/* after an overlapped pint_heat_build_chain_dev: the build kernel's span on the device (first CTA
 * start to last CTA end, %globaltimer) and the chain's exposed tail past it; syncs the stream */
int pint_ctx_build_chain_ms(pint_ctx* ctx, double* build_ms, double* tail_ms);
/* Compose two augmented maps: out = later ∘ earlier (EXTENSION, the tree's pair step). */
int pint_affine_pair_dev(pint_ctx* ctx, int64_t n, int64_t P, const double* earlier,
                         const double* later, double* out);

/* ---- EXTENSION: 2-D Lotka-Volterra ensemble + bilinear sweep (config 3) ---- */
/* endpoints layout (N, 2, Mu, Mv); params = {alpha, beta, delta, gamma} (host) */
int pint_lv_ensemble_dev(pint_ctx* ctx, int64_t N, int64_t Mu, int64_t Mv, const int64_t* steps,
                         const double* dt, const double* un, const double* vn,
                         const double* params, double* endpoints);
/* chain of bilinear maps; lambdas (N, 2), brackets (N, 2) = (iu, iv) used at each slice */
int pint_bilinear_sweep_dev(pint_ctx* ctx, int64_t N, int64_t Mu, int64_t Mv, const double* un,
                            const double* vn, const double* tables, double u0, double v0,
                            double* lambdas, long long* brackets, long long* extrapolations);

/* ---- full runs with HOST buffers (run_nievergelt, nievergelt.cpp:145-265) ---- */
/* Scalar: decompose, sample nodes, K1, weights, K2 sweep. y_out[0] = final state.
 * endpoints_out (N*M, may be NULL) receives the ensemble; lambdas_out (N, may be NULL).
 * Small runs (FP64, EXACT sweep, M <= 32, N*M <= 8192, per_slice_seconds NULL) run as ONE kernel
 * launch with no input copy (set PINT_SMALL_RUN=0 for the separate kernels); results and errors
 * are identical either way. */
int pint_run_scalar(pint_ctx* ctx, const pint_scalar_rhs* rhs, double t0, double T, double y0,
                    int64_t N, double dt, int node_kind, int64_t M, double a, double b,
                    int weight_kind, int sweep_mode, double* y_out, double* endpoints_out,
                    double* lambdas_out, double* per_slice_seconds, pint_report* report,
                    pint_fail* fail);
/* Heat: make_heat_problem(dx, dt, T) with y0 = heat_initial, N slices, K3 + K4. */
int pint_run_heat(pint_ctx* ctx, double dx, double dt, double T, int64_t N, int compose_mode,
                  const double* y0, double* y_out, double* per_slice_seconds, pint_report* report);
/* pint_run_heat with a choice of build: PINT_BUILD_EXACT (bit-exact, = pint_run_heat) or
 * PINT_BUILD_FAST (the tolerance build, final state <= 1e-12 relative to the reference's). */
int pint_run_heat_ex(pint_ctx* ctx, double dx, double dt, double T, int64_t N, int build_mode,
                     int compose_mode, const double* y0, double* y_out, double* per_slice_seconds,
                     pint_report* report);
/* Heat slice maps to host: G row-major N x n x n, c N x n (build_affine_propagator for all). */
int pint_heat_maps(pint_ctx* ctx, double dx, double dt, const pint_slice* slices, int64_t N,
                   double* G, double* c);
/* Heat integrate closure on host vectors: K states y[k*n..] over one slice, in place. */
int pint_heat_integrate(pint_ctx* ctx, double dx, const pint_slice* slice, double dt_nominal,
                        int with_forcing, int64_t K, double* y);
/* run_serial(make_heat_problem(dx, dt, T)) in the BACKGROUND on the context's own serial stream
 * (nievergelt.cpp:126-143, bit-exact): begin enqueues it and returns; end waits and writes the final
 * state. Concurrent device work on the context (e.g. pint_run_heat) proceeds meanwhile — how the
 * drop-in's run_nievergelt overlaps the serial reference run with the parallel one. */
int pint_heat_serial_begin(pint_ctx* ctx, double dx, double dt, double T, const double* y0);
int pint_heat_serial_end(pint_ctx* ctx, double* y_out);
/* Scalar integrate (integrate_scalar, nievergelt.cpp:29-35) for K initial values on one slice. */
int pint_scalar_integrate(pint_ctx* ctx, const pint_scalar_rhs* rhs, const pint_slice* slice,
                          int64_t K, const double* y0, double* y_out, pint_fail* fail);
/* Host-buffer affine chain / tree over maps given as G (N x n x n row-major) and c (N x n). */
int pint_affine_compose(pint_ctx* ctx, int mode, int64_t n, int64_t N, const double* G,
                        const double* c, const double* y0, double* y_out);
/* Host-buffer scalar sweep over N interpolants (general: per-slice nodes/weights/a/b). */
int pint_scalar_sweep(pint_ctx* ctx, int mode, int64_t N, int64_t M, const double* nodes,
                      int64_t node_stride, const double* weights, const double* values,
                      const double* a, const double* b, int64_t ab_stride, double y0,
                      double* lambdas, double* y_out, long long* extrapolations);

/* ---- wave slice maps (make_wave_linear_problem, pde_problems.cpp:142-172; leapfrog_integrate,
 * ode_core.cpp:65-77). d = M - 1 interior points, D2 = d x d row-major (host), state [u; u_prev]
 * of size 2d. The closure's rule is kept: every slice must step at dt_native = 8/M^2 within 1e-9
 * (PINT_E_BAD_GRID otherwise). Bit-exact vs the reference. */
/* G row-major N x 2d x 2d, c N x 2d (c = 0: the wave problem has no forcing). */
int pint_wave_maps(pint_ctx* ctx, int64_t d, const double* D2, double dt_native,
                   const pint_slice* slices, int64_t N, double dt_nominal, double* G, double* c);
/* the integrate closure for K states y[k*2d ...] over one slice, in place */
int pint_wave_integrate(pint_ctx* ctx, int64_t d, const double* D2, double dt_native,
                        const pint_slice* slice, double dt_nominal, int64_t K, double* y);
/* run_nievergelt for the wave problem: N slices of [0, T], compose chain or tree */
int pint_run_wave(pint_ctx* ctx, int64_t d, const double* D2, double dt_native, double T, int64_t N,
                  double dt_nominal, int compose_mode, const double* y0, double* y_out,
                  double* per_slice_seconds, pint_report* report);

/* ---- parareal on the device (parareal.cpp:47-165; the paper's comparison method, SURVEY.md §8f
 * rank 2) — scalar model problem: the reference's integrate_scalar_step (backward-Euler Riccati,
 * per-slice steps_for / width / n) as fine (dt) and coarse (DT) propagator, N slices of
 * decompose(t0, T, N, dt), k iterations. ONE kernel: each iteration's fine wave runs the N slices
 * in parallel from lambda_j, then the sequential correction sweep g_new + f - g_old; bit-identical
 * to the reference. finals[k + 1]: the final-time state after iteration 0 (coarse init) .. k
 * (PararealResult::final_per_iteration). fine_seconds[N] (may be NULL): summed device time of each
 * slice's fine integrations; *coarse_seconds (may be NULL): mean device time per coarse slice
 * (modeled_time_parareal's inputs). NoRealRoot in the fine wave: fail->index = the slice. */
int pint_parareal_scalar(pint_ctx* ctx, double t0, double T, double y0, int64_t N, int64_t k, double dt,
                         double DT, double* finals, double* fine_seconds, double* coarse_seconds,
                         pint_report* report, pint_fail* fail);

/* Parareal for make_heat_problem(dx, ., T): the integrate closure at dt (fine) and DT (coarse)
 * (parareal.cpp:167-190), N slices of decompose(0, T, N, dt), k iterations; bit-identical to the
 * reference. Each iteration is two launches: the fine wave (a warp per slice, from lambda_j, on
 * that slice's staged records) and the sequential correction sweep (one warp walking the slices'
 * coarse steps, combining g_new + f - g_old row by row). finals[(k + 1) n]: the final state after
 * every iteration. y0 NULL: heat_initial. */
int pint_parareal_heat(pint_ctx* ctx, double dx, double T, const double* y0, int64_t N, int64_t k,
                       double dt, double DT, double* finals, pint_report* report);

/* ---- multi-GPU (north_star subsystem 4): one context per GPU (a process or a
 * thread each). Slices go to ranks in contiguous blocks [floor(rN/W), floor((r+1)N/W)) of the
 * reference decomposition (ode_core.cpp:26-45, identical on every rank: slice assignment is
 * bit-exact); the only exchange is the final compose step. Replaces the reference's simulated
 * wire (inject_latency + counters, nievergelt.cpp:73-79, 95-101) and ExecConfig::workers' thread
 * pool (exec_harness.hpp:17-21, 51-101) with GPUs. ---- */
/* NCCL: rank 0 makes the id (128 bytes, an ncclUniqueId) and the caller distributes it. NCCL is
 * resolved at run time (dlopen "libnccl.so.2" at the first NCCL call), never linked, so loading this
 * library does not pin an NCCL build: in a process that also uses PyTorch, import torch first and its
 * NCCL is the one used (paper_1304_6514_b200/dist.py nccl_comm_init does). */
int pint_comm_unique_id(void* id_out);
int pint_comm_init(pint_ctx* ctx, const void* id, int rank, int world);
/* one process driving `world` GPUs: ctxs[r] on its own device becomes rank r */
int pint_comm_init_all(pint_ctx** ctxs, int world);
/* a caller-provided transport of HOST buffers (MPI, a socket, torch.distributed ...); each call
 * returns 0 on success; device data is staged through pinned memory */
typedef int (*pint_send_fn)(void* user, int peer, const void* buf, size_t bytes);
typedef int (*pint_recv_fn)(void* user, int peer, void* buf, size_t bytes);
int pint_comm_init_callbacks(pint_ctx* ctx, int rank, int world, pint_send_fn send, pint_recv_fn recv,
                             void* user);
int pint_comm_rank(const pint_ctx* ctx, int* rank, int* world);
int pint_comm_destroy(pint_ctx* ctx);
/* run_nievergelt(make_heat_problem(dx, dt, T), N) over the communicator's ranks (call on every
 * rank). Each rank builds its block's maps (build_mode as pint_run_heat_ex). compose_mode
 * PINT_COMPOSE_TREE: the block's maps tree-composed (DMMA) into one augmented map, ONE gather of
 * the W maps to rank 0, which applies them in rank order (the paper's single final gather/compose;
 * <= 1e-12 vs the chain). PINT_COMPOSE_CHAIN: the running state handed rank to rank (W messages of
 * n doubles), each rank applying its block's maps with the bit-exact chain — bit-identical to
 * pint_run_heat. y_out (n doubles) is written on rank 0 (may be NULL elsewhere); report->
 * message_count / bytes_communicated count this rank's real transfers. */
int pint_run_heat_sharded(pint_ctx* ctx, double dx, double dt, double T, int64_t N, int build_mode,
                          int compose_mode, const double* y0, double* y_out, pint_report* report);

/* Host-buffer barycentric weights (interp.cpp:43-55 / closed form); DuplicateNodes -> code 5. */
int pint_bary_weights(pint_ctx* ctx, int kind, int64_t M, const double* nodes, double* w);

/* ---- roofline probe: measured FMA throughput (TFLOP/s) of this GPU for PINT_F64 / PINT_F32, or
   the FP64 tensor-core (DMMA m8n8k4) throughput for PINT_PROBE_DMMA — the tree compose's roof */
enum { PINT_PROBE_DMMA = 2 };
int pint_probe_peak(pint_ctx* ctx, int precision, double* tflops);
/* dependent-chain latency in SM cycles per op: {DFMA, DADD, DMUL, FFMA, LDS.64}, then cycles per
   heat forward row (5 dependent ops), per heat back row (2), per op of alternating DMUL/DADD */
int pint_probe_latency(pint_ctx* ctx, double* cycles);

#ifdef __cplusplus
}
#endif
#endif
