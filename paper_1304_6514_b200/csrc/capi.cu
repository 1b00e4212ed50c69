// The C ABI (include/pint_cuda.h): context, host-side tables and the full-run pipelines.
//
// Host tables are computed with the reference's own arithmetic (same operation order, glibc
// sin/cos, no FMA contraction: -Xcompiler -ffp-contract=off), so slice assignment, step counts
// and per-step coefficients are bit-identical to what the reference computes inside its loops.
// There is no CPU fallback anywhere: without a device every entry point returns an error.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <pthread.h>
#include <vector>

#include "pint_internal.cuh"

namespace {

constexpr double kPi = 3.14159265358979323846;

const char* cuda_name(cudaError_t e) { return cudaGetErrorString(e); }

bool ok(pint_ctx* ctx, cudaError_t e, const char* what) {
    if (e == cudaSuccess) return true;
    pint_set_error(ctx, PINT_E_CUDA, std::string(what) + ": " + cuda_name(e));
    return false;
}

struct HostTimer {
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    double ms() const {
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
};

// integrate_slice's integrality check (ode_core.hpp:77-80) for a slice run at step h
int check_integral(pint_ctx* ctx, double span, double h) {
    const double ratio = span / h;
    const long long n = std::llround(ratio);
    if (n == 0 || std::fabs(ratio - static_cast<double>(n)) > 1e-9 * std::max(1.0, std::fabs(ratio))) {
        char buf[128];
        std::snprintf(buf, sizeof buf, "integrate_slice: (t_end - t_start)/dt = %f", ratio);
        return pint_set_error(ctx, PINT_E_NON_INTEGER_STEPS, buf);
    }
    return PINT_OK;
}

// interior_points (pde_problems.cpp:14-21)
int heat_dim(pint_ctx* ctx, double dx, int64_t* n) {
    const double inv = 1.0 / dx;
    const long long m = std::llround(inv);
    if (m < 2 || std::fabs(inv - static_cast<double>(m)) > 1e-9 * inv) {
        char buf[160];
        std::snprintf(buf, sizeof buf, "make_heat_system: 1/dx must be an integer >= 2, got dx = %f", dx);
        return pint_set_error(ctx, PINT_E_BAD_GRID, buf);
    }
    *n = m - 1;
    return PINT_OK;
}

// Slices as the heat integrate closure sees them: steps = steps_for(width, dt_nominal),
// h = width / steps (pde_problems.cpp:88-89).
void closure_slices(const pint_slice* in, int64_t N, double dt_nominal, std::vector<pint_slice>& out) {
    out.resize(static_cast<size_t>(N));
    for (int64_t j = 0; j < N; ++j) {
        pint_slice s = in[j];
        s.steps = pint_steps_for(s.t_end - s.t_begin, dt_nominal);
        s.dt = (s.t_end - s.t_begin) / static_cast<double>(s.steps);
        out[static_cast<size_t>(j)] = s;
    }
}

// Pinned staging buffer owned by the context for the host-buffer entry points.
struct Pinned {
    void* p = nullptr;
    size_t bytes = 0;
};
thread_local Pinned t_pinned;

// Process-wide host worker pool for the per-step tables (glibc sin/cos must run on the host for
// bit-parity): created once, so a run pays no thread start-up. parallel_for(n, fn) runs
// fn(i0, i1) over [0, n) in up to `size` contiguous chunks and returns when all are done.
class HostPool {
  public:
    static HostPool& get() {
        static HostPool pool;
        return pool;
    }
    unsigned size() const { return static_cast<unsigned>(workers_.size()) + 1; }
    void parallel_for(int64_t n, const std::function<void(int64_t, int64_t)>& fn) {
        const int64_t parts = std::min<int64_t>(n, size());
        if (parts <= 1 || forked_child().load()) {  // (a forked child has none of the workers)
            fn(0, n);
            return;
        }
        std::unique_lock<std::mutex> job_lock(job_mutex_);  // one parallel_for at a time
        {
            std::lock_guard<std::mutex> g(m_);
            fn_ = &fn;
            n_ = n;
            parts_ = parts;
            next_ = 1;
            pending_ = parts - 1;
            ++generation_;
        }
        cv_.notify_all();
        fn(0, n / parts);  // the caller takes part 0
        std::unique_lock<std::mutex> l(m_);
        done_cv_.wait(l, [&] { return pending_ == 0; });
        fn_ = nullptr;
    }

  private:
    static std::atomic<bool>& forked_child() {
        static std::atomic<bool> f{false};
        return f;
    }
    HostPool() {
        const unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
        for (unsigned i = 1; i < hw; ++i) workers_.emplace_back([this] { run(); });
        pthread_atfork(nullptr, nullptr, [] { forked_child().store(true); });
    }
    ~HostPool() {
        {
            std::lock_guard<std::mutex> g(m_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : workers_) t.join();
    }
    // A part is claimed under the mutex, and only while the job the worker woke for is still the
    // current one: a worker that wakes late never runs a finished job's function (whose caller
    // has returned and destroyed it) on the next job's part indices. The caller returns only once
    // every claimed part has finished (pending_).
    void run() {
        uint64_t seen = 0;
        std::unique_lock<std::mutex> l(m_);
        for (;;) {
            cv_.wait(l, [&] { return stop_ || generation_ != seen; });
            if (stop_) return;
            seen = generation_;
            while (fn_ && generation_ == seen && next_ < parts_) {
                const int64_t k = next_++, n = n_, parts = parts_;
                const auto* fn = fn_;
                l.unlock();
                (*fn)(n * k / parts, n * (k + 1) / parts);
                l.lock();
                if (--pending_ == 0) done_cv_.notify_one();
            }
        }
    }
    std::vector<std::thread> workers_;
    std::mutex m_, job_mutex_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(int64_t, int64_t)>* fn_ = nullptr;
    int64_t n_ = 0, parts_ = 0, pending_ = 0, next_ = 0;
    uint64_t generation_ = 0;
    bool stop_ = false;
};

void* pinned(size_t bytes) {
    if (t_pinned.bytes < bytes) {
        if (t_pinned.p) cudaFreeHost(t_pinned.p);
        t_pinned.p = nullptr;
        t_pinned.bytes = 0;
        if (cudaHostAlloc(&t_pinned.p, bytes, cudaHostAllocDefault) != cudaSuccess) return nullptr;
        t_pinned.bytes = bytes;
    }
    return t_pinned.p;
}

// Bump allocator over one scratch arena.
struct Carve {
    char* base;
    size_t off = 0;
    template <class T>
    T* take(size_t count) {
        off = (off + 255) & ~size_t(255);
        T* p = reinterpret_cast<T*>(base + off);
        off += sizeof(T) * count;
        return p;
    }
};

size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

}  // namespace

// ---- internal helpers shared with the kernel files ------------------------------------------

int pint_set_error(pint_ctx* ctx, int code, const std::string& msg) {
    if (ctx) ctx->last_error = msg;
    return code;
}

int pint_check_launch(pint_ctx* ctx, const char* what) {
    ++ctx->launches;
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return pint_set_error(ctx, PINT_E_CUDA, std::string(what) + ": " + cuda_name(e));
    return PINT_OK;
}

void pint_kernel_attrs(const void* fn) {
    static std::mutex m;
    static std::vector<const void*> done;
    std::lock_guard<std::mutex> lk(m);
    if (std::find(done.begin(), done.end(), fn) != done.end()) return;
    // (227 KB per block including the kernel's static shared memory: asking for more fails and
    // would leave the 48 KB default in place)
    cudaFuncAttributes fa{};
    const size_t stat = cudaFuncGetAttributes(&fa, fn) == cudaSuccess ? fa.sharedSizeBytes : 0;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(227 * 1024 - stat));
    cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    done.push_back(fn);
}

void* pint_scratch(pint_ctx* ctx, int slot, size_t bytes) {
    if (ctx->scratch_bytes[slot] < bytes) {
        if (ctx->scratch[slot]) cudaFree(ctx->scratch[slot]);
        ctx->scratch[slot] = nullptr;
        ctx->scratch_bytes[slot] = 0;
        if (cudaMalloc(&ctx->scratch[slot], bytes) != cudaSuccess) {
            pint_set_error(ctx, PINT_E_CUDA, "scratch allocation of " + std::to_string(bytes) + " bytes failed");
            return nullptr;
        }
        ctx->scratch_bytes[slot] = bytes;
    }
    return ctx->scratch[slot];
}

// ---- context -----------------------------------------------------------------------------------

extern "C" {

const char* pint_version(void) { return "pint-b200 0.1 (sm_100a)"; }

int pint_device_count(void) {
    int count = 0;
    return cudaGetDeviceCount(&count) == cudaSuccess ? count : 0;
}

int pint_ctx_create(int device, pint_ctx** out) {
    if (!out) return PINT_E_INVALID;
    *out = nullptr;
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) return PINT_E_NO_DEVICE;
    if (device < 0 || device >= count) return PINT_E_INVALID;
    auto* ctx = new pint_ctx();
    ctx->device = device;
    if (cudaSetDevice(device) != cudaSuccess) {
        delete ctx;
        return PINT_E_CUDA;
    }
    cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device);
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaMalloc(&ctx->d_fail, pint_ctx::kFailAlloc) != cudaSuccess ||
        cudaEventCreate(&ctx->ev0) != cudaSuccess || cudaEventCreate(&ctx->ev1) != cudaSuccess ||
        cudaEventCreate(&ctx->evc) != cudaSuccess ||
        cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming) != cudaSuccess ||
        cudaStreamCreateWithFlags(&ctx->serial, cudaStreamNonBlocking) != cudaSuccess ||
        cudaMalloc(&ctx->d_fail_serial, sizeof(FailRec)) != cudaSuccess) {
        delete ctx;
        return PINT_E_CUDA;
    }
    ctx->own_stream = true;
    FailRec init{pint_dev::kNoFail, 0, 0, 0.0};
    cudaMemset(ctx->d_fail, 0, pint_ctx::kFailAlloc);
    cudaMemcpy(ctx->d_fail, &init, sizeof init, cudaMemcpyHostToDevice);
    cudaMemcpy(ctx->d_fail_serial, &init, sizeof init, cudaMemcpyHostToDevice);
    if (cudaHostAlloc(&ctx->h_small, 256, cudaHostAllocDefault) != cudaSuccess ||
        cudaHostAlloc(&ctx->h_mapped, 256, cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer(reinterpret_cast<void**>(&ctx->d_mapped), ctx->h_mapped, 0) != cudaSuccess) {
        pint_ctx_destroy(ctx);
        return PINT_E_CUDA;
    }
    *out = ctx;
    return PINT_OK;
}

void pint_ctx_destroy(pint_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    for (int i = 0; i < pint_ctx::kSlots; ++i)
        if (ctx->scratch[i]) cudaFree(ctx->scratch[i]);
    if (ctx->serial) cudaStreamSynchronize(ctx->serial);
    comm_free(ctx);
    if (ctx->d_fail) cudaFree(ctx->d_fail);
    if (ctx->d_fail_serial) cudaFree(ctx->d_fail_serial);
    if (ctx->h_small) cudaFreeHost(ctx->h_small);
    if (ctx->h_mapped) cudaFreeHost(ctx->h_mapped);
    if (ctx->serial) cudaStreamDestroy(ctx->serial);
    if (ctx->ev0) cudaEventDestroy(ctx->ev0);
    if (ctx->ev1) cudaEventDestroy(ctx->ev1);
    if (ctx->evc) cudaEventDestroy(ctx->evc);
    if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
    if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
    if (ctx->side) cudaStreamDestroy(ctx->side);
    if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

const char* pint_ctx_last_error(const pint_ctx* ctx) { return ctx ? ctx->last_error.c_str() : "null context"; }

int pint_ctx_sync(pint_ctx* ctx) {
    return ok(ctx, cudaStreamSynchronize(ctx->stream), "cudaStreamSynchronize") ? PINT_OK : PINT_E_CUDA;
}

void* pint_ctx_stream(pint_ctx* ctx) { return ctx ? reinterpret_cast<void*>(ctx->stream) : nullptr; }

int pint_ctx_set_stream(pint_ctx* ctx, void* stream) {
    if (!ctx) return PINT_E_INVALID;
    if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
    ctx->stream = reinterpret_cast<cudaStream_t>(stream);
    ctx->own_stream = false;
    return PINT_OK;
}

int64_t pint_ctx_launch_count(const pint_ctx* ctx) { return ctx ? ctx->launches : 0; }

namespace {
// read and clear failure record `f` on `st` (pint_fail_read semantics)
int fail_read_on(pint_ctx* ctx, FailRec* f, cudaStream_t st, pint_fail* out) {
    FailRec rec{};
    if (!ok(ctx, cudaMemcpyAsync(&rec, f, sizeof rec, cudaMemcpyDeviceToHost, st), "fail read") ||
        !ok(ctx, cudaStreamSynchronize(st), "fail read sync"))
        return PINT_E_CUDA;
    FailRec init{pint_dev::kNoFail, 0, 0, 0.0};
    if (rec.index != pint_dev::kNoFail &&
        (!ok(ctx, cudaMemcpyAsync(f, &init, sizeof init, cudaMemcpyHostToDevice, st), "fail reset") ||
         !ok(ctx, cudaStreamSynchronize(st), "fail reset sync")))
        return PINT_E_CUDA;
    if (out) {
        out->index = rec.index == pint_dev::kNoFail ? -1 : static_cast<int64_t>(rec.index);
        out->code = rec.index == pint_dev::kNoFail ? 0 : rec.code;
        out->pad = 0;
        out->value = rec.value;
    }
    return PINT_OK;
}
}  // namespace

int pint_fail_read(pint_ctx* ctx, pint_fail* out) {
    FailRec rec{};
    if (!ok(ctx, cudaMemcpyAsync(&rec, ctx->d_fail, sizeof rec, cudaMemcpyDeviceToHost, ctx->stream), "fail read") ||
        !ok(ctx, cudaStreamSynchronize(ctx->stream), "fail read sync"))
        return PINT_E_CUDA;
    FailRec init{pint_dev::kNoFail, 0, 0, 0.0};
    if (rec.index != pint_dev::kNoFail &&
        !ok(ctx, cudaMemcpyAsync(ctx->d_fail, &init, sizeof init, cudaMemcpyHostToDevice, ctx->stream), "fail reset"))
        return PINT_E_CUDA;
    cudaStreamSynchronize(ctx->stream);
    if (out) {
        out->index = rec.index == pint_dev::kNoFail ? -1 : static_cast<int64_t>(rec.index);
        out->code = rec.index == pint_dev::kNoFail ? 0 : rec.code;
        out->pad = 0;
        out->value = rec.value;
    }
    return PINT_OK;
}

namespace {
// Test hook for the failure-record protocol: thread t records (idx[t], code[t], value[t]).
__global__ void fail_inject_kernel(int64_t K, const int64_t* idx, const int* code, const double* value, FailRec* rec) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t < K) pint_dev::record_failure(rec, idx[t], code[t], value[t]);
}
}  // namespace

int pint_debug_fail_inject(pint_ctx* ctx, int64_t K, const int64_t* idx, const int* code, const double* value) {
    if (!ctx || K < 0) return PINT_E_INVALID;
    if (K == 0) return PINT_OK;
    fail_inject_kernel<<<static_cast<unsigned>((K + 255) / 256), 256, 0, ctx->stream>>>(K, idx, code, value,
                                                                                    ctx->d_fail);
    return pint_check_launch(ctx, "fail_inject_kernel");
}

// ---- host tables ---------------------------------------------------------------------------------

int64_t pint_steps_for(double width, double dt) {
    const double ratio = width / dt;
    const double snapped = ratio - 1e-9 * std::max(1.0, ratio);
    const auto n = static_cast<long long>(std::ceil(snapped));
    return n < 1 ? 1 : n;
}

int pint_decompose(double t0, double T, int64_t N, double dt, pint_slice* out) {
    if (N <= 0 || !(T > t0) || !(dt > 0.0) || !out) return PINT_E_BAD_GRID;
    const double width = (T - t0) / static_cast<double>(N);
    for (int64_t j = 0; j < N; ++j) {
        pint_slice s;
        s.t_begin = t0 + static_cast<double>(j) * width;
        s.t_end = (j + 1 == N) ? T : t0 + static_cast<double>(j + 1) * width;
        s.steps = pint_steps_for(s.t_end - s.t_begin, dt);
        s.dt = (s.t_end - s.t_begin) / static_cast<double>(s.steps);
        out[j] = s;
    }
    return PINT_OK;
}

int pint_sample_nodes(int kind, int64_t M, double a, double b, double* out) {
    if (M <= 0 || !out) return PINT_E_BAD_GRID;
    if (M == 1) {
        out[0] = 0.5 * (a + b);
        return PINT_OK;
    }
    for (int64_t k = 0; k < M; ++k) {
        const double kd = static_cast<double>(k);
        out[k] = (kind == PINT_NODES_FIRST_KIND)
                     ? std::cos((2.0 * kd + 1.0) * kPi / (2.0 * static_cast<double>(M)))
                     : std::cos(kd * kPi / static_cast<double>(M - 1));
    }
    for (int64_t k = 0; k < M; ++k) out[k] = a + (b - a) * (out[k] + 1.0) / 2.0;
    std::sort(out, out + M);
    return PINT_OK;
}

int64_t pint_affine_ldm(int64_t n) { return ((n + 1) + 3) / 4 * 4; }

int64_t pint_heat_total_steps(const pint_slice* slices, int64_t N) {
    int64_t t = 0;
    for (int64_t j = 0; j < N; ++j) t += slices[j].steps;
    return t;
}

namespace {
// Per-step tables of slices [j0, j1) (step_off already filled): heat_coefficient
// (pde_problems.cpp:24), solve_implicit's r (:54), forcing (:26-29), on the host pool.
void heat_fill_steps(double dx, const pint_slice* slices, int64_t j0, int64_t j1, const int64_t* step_off,
                     double* r, double* fa, double* fb) {
    const double inv_dx2 = 1.0 / (dx * dx);  // pde_problems.cpp:33
    auto fill = [&](int64_t a, int64_t b) {
        for (int64_t j = j0 + a; j < j0 + b; ++j) {
            const double tb = slices[j].t_begin, h = slices[j].dt;
            const int64_t base = step_off[j];
            for (int64_t i = 1; i <= slices[j].steps; ++i) {
                const double t = tb + static_cast<double>(i) * h;  // ode_core.hpp:83
                const double st = std::sin(t);
                const double a = 1.0 + 0.25 * st;
                const int64_t q = base + i - 1;
                r[q] = h * a * inv_dx2;
                fa[q] = -st;
                fb[q] = a * kPi * kPi * std::cos(t);
            }
        }
    };
    if (step_off[j1] - step_off[j0] < 4096 || j1 - j0 < 2) fill(0, j1 - j0);
    else HostPool::get().parallel_for(j1 - j0, fill);
}

// The same tables for steps [s0, s1) of every slice (0-based step s = i - 1 of the loop above),
// as one block [j][s - s0] (pitch s1 - s0) so that it travels in one copy.
void heat_fill_step_range(double dx, const pint_slice* slices, int64_t N, int64_t s0, int64_t s1, double* r,
                          double* fa, double* fb) {
    const double inv_dx2 = 1.0 / (dx * dx);
    auto fill = [&](int64_t a, int64_t b) {
        for (int64_t j = a; j < b; ++j) {
            const double tb = slices[j].t_begin, h = slices[j].dt;
            const int64_t base = j * (s1 - s0) - s0, e = std::min<int64_t>(s1, slices[j].steps);
            for (int64_t i = s0 + 1; i <= e; ++i) {
                const double t = tb + static_cast<double>(i) * h;  // ode_core.hpp:83
                const double st = std::sin(t);
                const double a = 1.0 + 0.25 * st;
                const int64_t q = base + i - 1;
                r[q] = h * a * inv_dx2;
                fa[q] = -st;
                fb[q] = a * kPi * kPi * std::cos(t);
            }
        }
    };
    if (N * (s1 - s0) < 4096 || N < 2) fill(0, N);
    else HostPool::get().parallel_for(N, fill);
}
}  // namespace

int pint_heat_coefficients(double dx, const pint_slice* slices, int64_t N, int64_t* step_off,
                           double* r, double* fa, double* fb, double* sx, int64_t* n_out) {
    int64_t n = 0;
    if (const int rc = heat_dim(nullptr, dx, &n)) return rc;
    if (n_out) *n_out = n;
    step_off[0] = 0;
    for (int64_t j = 0; j < N; ++j) step_off[j + 1] = step_off[j] + slices[j].steps;
    heat_fill_steps(dx, slices, 0, N, step_off, r, fa, fb);
    if (sx)
        for (int64_t i = 0; i < n; ++i) sx[i] = std::sin(kPi * (static_cast<double>(i + 1) * dx));
    return PINT_OK;
}

// ---- device-pointer entry points -----------------------------------------------------------------

int pint_scalar_ensemble_dev(pint_ctx* ctx, const pint_scalar_rhs* rhs, int64_t N, int64_t M,
                             const int64_t* steps, const double* dt, const void* nodes,
                             void* endpoints, unsigned long long* per_slice_ns) {
    if (!ctx) return PINT_E_INVALID;
    return launch_scalar_ensemble(ctx, rhs, N, M, steps, dt, nodes, endpoints, per_slice_ns);
}

int pint_bary_weights_dev(pint_ctx* ctx, int kind, int64_t M, const double* nodes, double* w) {
    if (!ctx) return PINT_E_INVALID;
    return launch_bary_weights(ctx, kind, M, nodes, w);
}

int pint_scalar_sweep_dev(pint_ctx* ctx, int mode, int64_t N, int64_t M, const double* nodes,
                          int64_t node_stride, const double* weights, const double* values,
                          const double* a, const double* b, int64_t ab_stride, double y0,
                          double* lambdas, double* y_out, long long* extrapolations) {
    if (!ctx) return PINT_E_INVALID;
    return launch_scalar_sweep(ctx, mode, N, M, nodes, node_stride, weights, values, a, b, ab_stride,
                               y0, lambdas, y_out, extrapolations);
}

int64_t pint_heat_records_size(int64_t n, int64_t N, int64_t S) { return heat_records_doubles(n, N, S); }

int pint_heat_factor_dev(pint_ctx* ctx, int64_t n, int64_t N, int64_t S, const int64_t* step_off,
                         const double* slice_dt, const double* r, const double* fa,
                         const double* fb, const double* sx, double* records) {
    if (!ctx) return PINT_E_INVALID;
    return launch_heat_factor(ctx, n, N, S, step_off, slice_dt, r, fa, fb, sx, records);
}

int pint_heat_build_dev(pint_ctx* ctx, int64_t n, int64_t N, int64_t S, const int64_t* step_off,
                        const double* slice_dt, const double* records, const double* sx,
                        double* maps, unsigned long long* per_slice_ns, int guarded) {
    if (!ctx) return PINT_E_INVALID;
    return launch_heat_build(ctx, n, N, S, step_off, slice_dt, records, sx, maps, per_slice_ns, guarded);
}

int64_t pint_heat_fast_records_size(int64_t n, int64_t N, int64_t S) { return heat_fast_records_doubles(n, N, S); }

int pint_heat_fast_factor_dev(pint_ctx* ctx, int64_t n, int64_t N, int64_t S, const int64_t* step_off,
                              const double* slice_dt, const double* r, const double* fa, const double* fb,
                              const double* sx, double* records) {
    if (!ctx) return PINT_E_INVALID;
    return launch_heat_fast_factor(ctx, ctx->stream, n, N, S, step_off, slice_dt, r, fa, fb, sx, records);
}

int pint_heat_fast_build_dev(pint_ctx* ctx, int64_t n, int64_t N, int64_t S, const double* records, double* maps) {
    if (!ctx) return PINT_E_INVALID;
    return launch_heat_fast_build(ctx, n, N, S, records, maps);
}

namespace {
// ---- integrate (the closure, run_serial): one slice's steps for K device columns ----------------
struct IntegTables {
    int64_t n = 0, Q = 0;
    int64_t* step_off = nullptr;
    double *dt = nullptr, *r = nullptr, *fa = nullptr, *fb = nullptr, *sx = nullptr;
};

// Host tables of slice `s` (the reference's arithmetic, as heat_upload) into scratch `slot`, copied
// on `st` and synchronised (the thread's pinned staging is free again on return).
int integ_upload(pint_ctx* ctx, cudaStream_t st, int slot, double dx, const pint_slice& s, IntegTables& T) {
    int64_t n = 0;
    if (const int rc = heat_dim(ctx, dx, &n)) return rc;
    if (const int rc = check_integral(ctx, s.t_end - s.t_begin, s.dt)) return rc;
    const int64_t Q = s.steps;
    const size_t b_off = align256(2 * sizeof(int64_t)), b_dt = align256(sizeof(double));
    const size_t b_q = align256(sizeof(double) * Q), b_sx = align256(sizeof(double) * n);
    const size_t bytes = b_off + b_dt + 3 * b_q + b_sx;
    char* h = static_cast<char*>(pinned(bytes));
    char* d = static_cast<char*>(pint_scratch(ctx, slot, bytes));
    if (!h || !d) return pint_set_error(ctx, PINT_E_CUDA, "integrate: table allocation failed");
    auto* h_off = reinterpret_cast<int64_t*>(h);
    h_off[0] = 0;
    h_off[1] = Q;
    reinterpret_cast<double*>(h + b_off)[0] = s.dt;
    heat_fill_steps(dx, &s, 0, 1, h_off, reinterpret_cast<double*>(h + b_off + b_dt),
                    reinterpret_cast<double*>(h + b_off + b_dt + b_q), reinterpret_cast<double*>(h + b_off + b_dt + 2 * b_q));
    auto* h_sx = reinterpret_cast<double*>(h + b_off + b_dt + 3 * b_q);
    for (int64_t i = 0; i < n; ++i) h_sx[i] = std::sin(kPi * (static_cast<double>(i + 1) * dx));
    if (!ok(ctx, cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st), "H2D integrate tables") ||
        !ok(ctx, cudaStreamSynchronize(st), "H2D integrate tables sync"))
        return PINT_E_CUDA;
    T.n = n;
    T.Q = Q;
    T.step_off = reinterpret_cast<int64_t*>(d);
    T.dt = reinterpret_cast<double*>(d + b_off);
    T.r = reinterpret_cast<double*>(d + b_off + b_dt);
    T.fa = reinterpret_cast<double*>(d + b_off + b_dt + b_q);
    T.fb = reinterpret_cast<double*>(d + b_off + b_dt + 2 * b_q);
    T.sx = reinterpret_cast<double*>(d + b_off + b_dt + 3 * b_q);
    return PINT_OK;
}

// the steps in bounded chunks on `st`: slice-major records of chunk c into `rec` (heat_integrate_chunk
// steps of room), then the integrate kernel over them — O(chunk) records, never O(Q)
int integ_enqueue(pint_ctx* ctx, cudaStream_t st, const IntegTables& T, double* rec, int with_forcing, int64_t K,
                  double* d_y, FailRec* fail, int guarded) {
    const int64_t chunk = heat_integrate_chunk(T.n);
    for (int64_t s0 = 0; s0 < T.Q; s0 += chunk) {
        const int64_t sc = std::min(chunk, T.Q - s0);
        if (const int rc = launch_heat_factor_block(ctx, st, T.n, 1, chunk, 0, 1, s0, sc, 0, T.step_off, T.dt, T.r,
                                                    T.fa, T.fb, T.sx, rec, s0, true))
            return rc;
        if (const int rc = launch_heat_integrate_steps(ctx, st, T.n, K, sc, with_forcing, rec, d_y, fail, s0, guarded))
            return rc;
    }
    return PINT_OK;
}

}  // namespace

int pint_heat_integrate_dev(pint_ctx* ctx, int64_t n, int64_t K, int64_t steps, const int64_t* step_off,
                            const double* slice_dt, const double* r, const double* fa, const double* fb,
                            const double* sx, int with_forcing, double* y, int guarded) {
    if (!ctx) return PINT_E_INVALID;
    const IntegTables T{n, steps, const_cast<int64_t*>(step_off), const_cast<double*>(slice_dt), const_cast<double*>(r),
                        const_cast<double*>(fa), const_cast<double*>(fb), const_cast<double*>(sx)};
    double* rec = static_cast<double*>(pint_scratch(ctx, 1, sizeof(double) * heat_integrate_records_doubles(n)));
    if (!rec) return PINT_E_CUDA;
    return integ_enqueue(ctx, ctx->stream, T, rec, with_forcing, K, y, ctx->d_fail, guarded);
}

int pint_ctx_build_chain_ms(pint_ctx* ctx, double* build_ms, double* tail_ms) {
    if (!ctx) return PINT_E_INVALID;
    if (!ctx->span_words) return pint_set_error(ctx, PINT_E_INVALID, "no overlapped build + chain ran on this context");
    unsigned long long w[3];
    if (!ok(ctx, cudaMemcpyAsync(w, ctx->span_words, sizeof w, cudaMemcpyDeviceToHost, ctx->stream), "span D2H") ||
        !ok(ctx, cudaStreamSynchronize(ctx->stream), "span sync"))
        return PINT_E_CUDA;
    if (build_ms) *build_ms = static_cast<double>(w[1] - w[0]) * 1e-6;
    if (tail_ms) *tail_ms = w[2] > w[1] ? static_cast<double>(w[2] - w[1]) * 1e-6 : 0.0;
    return PINT_OK;
}

namespace {
int heat_build_chain(pint_ctx* ctx, int64_t n, int64_t N, int64_t S, const int64_t* step_off,
                     const double* slice_dt, const double* records, const double* sx, double* maps,
                     const double* y0, double* y, unsigned long long* per_slice_ns, int guarded,
                     int build_mode = PINT_BUILD_EXACT);
}  // namespace

int pint_heat_build_chain_dev(pint_ctx* ctx, int64_t n, int64_t N, int64_t S, const int64_t* step_off,
                              const double* slice_dt, const double* records, const double* sx, double* maps,
                              const double* y0, double* y, int guarded) {
    if (!ctx) return PINT_E_INVALID;
    return heat_build_chain(ctx, n, N, S, step_off, slice_dt, records, sx, maps, y0, y, nullptr, guarded);
}

int pint_heat_fast_build_chain_dev(pint_ctx* ctx, int64_t n, int64_t N, int64_t S, const double* records,
                                   double* maps, const double* y0, double* y) {
    if (!ctx) return PINT_E_INVALID;
    return heat_build_chain(ctx, n, N, S, nullptr, nullptr, records, nullptr, maps, y0, y, nullptr, 0, PINT_BUILD_FAST);
}

int pint_affine_compose_dev(pint_ctx* ctx, int mode, int64_t n, int64_t N, double* maps,
                            double* scratch, const double* y0, double* y, double* composed) {
    if (!ctx) return PINT_E_INVALID;
    if (mode == PINT_COMPOSE_CHAIN) return launch_affine_chain(ctx, n, N, maps, y0, y);
    if (mode == PINT_COMPOSE_TREE) {
        if (!scratch && N > 1) return pint_set_error(ctx, PINT_E_INVALID, "affine tree needs scratch");
        return launch_affine_tree(ctx, n, N, maps, scratch, y0, y, composed);
    }
    return pint_set_error(ctx, PINT_E_INVALID, "affine_compose: unknown mode");
}

int pint_affine_pair_dev(pint_ctx* ctx, int64_t n, int64_t P, const double* earlier,
                         const double* later, double* out) {
    if (!ctx) return PINT_E_INVALID;
    return launch_affine_pair(ctx, n, P, earlier, later, out);
}

int pint_lv_ensemble_dev(pint_ctx* ctx, int64_t N, int64_t Mu, int64_t Mv, const int64_t* steps,
                         const double* dt, const double* un, const double* vn,
                         const double* params, double* endpoints) {
    if (!ctx) return PINT_E_INVALID;
    return launch_lv_ensemble(ctx, N, Mu, Mv, steps, dt, un, vn, params, endpoints);
}

int pint_bilinear_sweep_dev(pint_ctx* ctx, int64_t N, int64_t Mu, int64_t Mv, const double* un,
                            const double* vn, const double* tables, double u0, double v0,
                            double* lambdas, long long* brackets, long long* extrapolations) {
    if (!ctx) return PINT_E_INVALID;
    return launch_bilinear_sweep(ctx, N, Mu, Mv, un, vn, tables, u0, v0, lambdas, brackets, extrapolations);
}

// ---- full runs with host buffers -----------------------------------------------------------------

int pint_run_scalar(pint_ctx* ctx, const pint_scalar_rhs* rhs, double t0, double T, double y0,
                    int64_t N, double dt, int node_kind, int64_t M, double a, double b,
                    int weight_kind, int sweep_mode, double* y_out, double* endpoints_out,
                    double* lambdas_out, double* per_slice_seconds, pint_report* report,
                    pint_fail* fail) {
    if (!ctx || !rhs || !y_out) return PINT_E_INVALID;
    HostTimer wall;
    const long long launches0 = ctx->launches;
    if (fail) *fail = pint_fail{-1, 0, 0, 0.0};
    if (N < 1) N = 1;
    const bool serial = (N == 1);  // run_nievergelt with N <= 1 is run_serial (nievergelt.cpp:146-152)
    const bool f32 = rhs->precision == PINT_F32;
    const size_t esz = f32 ? sizeof(float) : sizeof(double);

    std::vector<pint_slice> sl(static_cast<size_t>(N));
    if (pint_decompose(t0, T, N, dt, sl.data()) != PINT_OK)
        return pint_set_error(ctx, PINT_E_BAD_GRID, "decompose: need N >= 1, T > t0, dt > 0");
    for (const auto& s : sl)
        if (const int rc = check_integral(ctx, s.t_end - s.t_begin, s.dt)) return rc;
    const int64_t Mn = serial ? 1 : M;
    std::vector<double> nodes(static_cast<size_t>(Mn));
    if (serial) {
        nodes[0] = y0;
    } else if (pint_sample_nodes(node_kind, M, a, b, nodes.data()) != PINT_OK) {
        return pint_set_error(ctx, PINT_E_BAD_GRID, "cheb_nodes: M >= 1 required");
    }

    // staging: steps[N] | dt[N] | nodes[M] (as the kernel's precision) | {a, b}
    const size_t b_steps = align256(sizeof(int64_t) * N), b_dt = align256(sizeof(double) * N);
    const size_t b_nodes = align256(esz * Mn), b_ab = align256(2 * sizeof(double));
    const size_t in_bytes = b_steps + b_dt + b_nodes + b_ab;
    char* h_in = static_cast<char*>(pinned(in_bytes));
    if (!h_in) return pint_set_error(ctx, PINT_E_CUDA, "pinned staging allocation failed");
    for (int64_t j = 0; j < N; ++j) {
        reinterpret_cast<int64_t*>(h_in)[j] = sl[j].steps;
        reinterpret_cast<double*>(h_in + b_steps)[j] = sl[j].dt;
    }
    for (int64_t m = 0; m < Mn; ++m) {
        if (f32) reinterpret_cast<float*>(h_in + b_steps + b_dt)[m] = static_cast<float>(nodes[m]);
        else reinterpret_cast<double*>(h_in + b_steps + b_dt)[m] = nodes[m];
    }
    reinterpret_cast<double*>(h_in + b_steps + b_dt + b_nodes)[0] = a;
    reinterpret_cast<double*>(h_in + b_steps + b_dt + b_nodes)[1] = b;

    const size_t b_ends = align256(esz * N * Mn);
    const size_t total = in_bytes + b_ends + align256(sizeof(double) * Mn) + align256(sizeof(double) * N) +
                         align256(sizeof(unsigned long long) * N) + 512;
    char* dbase = static_cast<char*>(pint_scratch(ctx, 0, total));
    if (!dbase) return PINT_E_CUDA;
    Carve cv{dbase};
    char* d_in = cv.take<char>(in_bytes);
    void* d_ends = cv.take<char>(b_ends);
    double* d_w = cv.take<double>(Mn);
    double* d_lam = cv.take<double>(N);
    auto* d_ns = cv.take<unsigned long long>(N);
    // y, the extrapolation count and the sweep's span sit right behind the failure record: the
    // call's small results come back in ONE copy
    unsigned long long* d_small = ctx->d_small();
    auto* d_y = reinterpret_cast<double*>(d_small);
    auto* d_ext = reinterpret_cast<long long*>(d_small + 1);
    const auto* d_steps = reinterpret_cast<const int64_t*>(d_in);
    const auto* d_dt = reinterpret_cast<const double*>(d_in + b_steps);
    const void* d_nodes = d_in + b_steps + b_dt;
    const auto* d_ab = reinterpret_cast<const double*>(d_in + b_steps + b_dt + b_nodes);

    int rc = PINT_OK;
    const bool sweep = !serial && !f32;
    // small runs (the paper's Table-3 shapes): ensemble, weights and the EXACT sweep in one launch,
    // its inputs as kernel parameters and its results in mapped host memory (no copies)
    const bool fused = sweep && sweep_mode == PINT_SWEEP_EXACT && !per_slice_seconds &&
                       scalar_small_run_fits(rhs, N, M, weight_kind);
    cudaEventRecord(ctx->ev0, ctx->stream);
    if (!fused && !ok(ctx, cudaMemcpyAsync(d_in, h_in, in_bytes, cudaMemcpyHostToDevice, ctx->stream), "H2D inputs"))
        return PINT_E_CUDA;
    if (per_slice_seconds) cudaMemsetAsync(d_ns, 0, sizeof(unsigned long long) * N, ctx->stream);
    if (fused) {
        rc = launch_scalar_small_run(ctx, rhs, N, M, t0, T, dt, nodes.data(), static_cast<double*>(d_ends), d_w,
                                     weight_kind, a, b, y0, d_lam, ctx->d_mapped);
        if (rc) return rc;
    } else if (sweep) {
        // the weights depend on the nodes only: side stream, overlapping the ensemble
        cudaEventRecord(ctx->ev_fork, ctx->stream);
        cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0);
        cudaStream_t main_stream = ctx->stream;
        ctx->stream = ctx->side;
        rc = launch_bary_weights(ctx, weight_kind, M, reinterpret_cast<const double*>(d_nodes), d_w);
        ctx->stream = main_stream;
        if (rc) return rc;
        cudaEventRecord(ctx->ev_join, ctx->side);
    }
    if (!fused) {
        rc = launch_scalar_ensemble(ctx, rhs, N, Mn, d_steps, d_dt, d_nodes, d_ends,
                                    per_slice_seconds ? d_ns : nullptr);
        if (rc) return rc;
    }
    long long ext = 0;
    double y = 0.0;
    if (serial) {
        if (!ok(ctx, cudaMemcpyAsync(d_y, d_ends, esz, cudaMemcpyDeviceToDevice, ctx->stream), "copy"))
            return PINT_E_CUDA;
    } else if (!fused) {
        if (f32) return pint_set_error(ctx, PINT_E_INVALID, "FP32 runs support the ensemble only; sweep in FP64");
        cudaStreamWaitEvent(ctx->stream, ctx->ev_join, 0);  // (the weights, from the side stream)
        cudaEventRecord(ctx->evc, ctx->stream);
        rc = launch_scalar_sweep(ctx, sweep_mode, N, M, reinterpret_cast<const double*>(d_nodes), 0, d_w,
                                 static_cast<const double*>(d_ends), d_ab, d_ab + 1, 0, y0, d_lam, d_y, d_ext);
        if (rc) return rc;
    }
    cudaEventRecord(ctx->ev1, ctx->stream);
    int64_t d2h = 0;
    // the failure record, y, the extrapolation count and the sweep span: ONE copy into the pinned
    // small block
    auto* hs = static_cast<char*>(fused ? ctx->h_mapped : ctx->h_small);
    if (!fused &&
        !ok(ctx, cudaMemcpyAsync(hs, ctx->d_fail, pint_ctx::kFailBlock, cudaMemcpyDeviceToHost, ctx->stream),
            "D2H results"))
        return PINT_E_CUDA;
    d2h += pint_ctx::kFailBlock;  // (fused: written by the kernel into mapped host memory)
    if (endpoints_out) {
        cudaMemcpyAsync(endpoints_out, d_ends, esz * N * Mn, cudaMemcpyDeviceToHost, ctx->stream);
        d2h += esz * N * Mn;
    }
    if (lambdas_out && !serial) {
        cudaMemcpyAsync(lambdas_out, d_lam, sizeof(double) * N, cudaMemcpyDeviceToHost, ctx->stream);
        d2h += sizeof(double) * N;
    }
    std::vector<unsigned long long> ns;
    if (per_slice_seconds) {
        ns.resize(static_cast<size_t>(N));
        cudaMemcpyAsync(ns.data(), d_ns, sizeof(unsigned long long) * N, cudaMemcpyDeviceToHost, ctx->stream);
    }
    if (!ok(ctx, cudaStreamSynchronize(ctx->stream), "run_scalar sync")) return PINT_E_CUDA;
    const char* hres = hs + pint_ctx::kSmallOff;
    std::memcpy(&y, hres, sizeof y);
    if (!serial) std::memcpy(&ext, hres + 8, sizeof ext);
    if (f32) y = static_cast<double>(*reinterpret_cast<float*>(&y));
    FailRec frec;
    std::memcpy(&frec, hs, sizeof frec);
    pint_fail fr{-1, 0, 0, 0.0};
    if (frec.index != pint_dev::kNoFail) {  // (rare) read it properly, which also clears it
        if ((rc = pint_fail_read(ctx, &fr))) return rc;
    }
    if (fail) *fail = fr;
    if (fr.index >= 0) {
        char buf[160];
        if (fr.code == PINT_E_NO_REAL_ROOT)
            std::snprintf(buf, sizeof buf, "be_step_scalar_riccati: 1 - 4 dt y = %f", fr.value);
        else
            std::snprintf(buf, sizeof buf, "barycentric_weights: repeated node");
        return pint_set_error(ctx, fr.code, buf);
    }
    *y_out = y;
    if (per_slice_seconds)
        for (int64_t j = 0; j < N; ++j) per_slice_seconds[j] = static_cast<double>(ns[j]) * 1e-9;
    if (report) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
        report->message_count = serial ? 0 : N - 1;
        report->bytes_communicated = serial ? 0 : (N - 1) * static_cast<int64_t>(sizeof(double));
        report->extrapolation_count = ext;
        report->device_ms = ms;
        report->traj_steps = 0;
        for (int64_t j = 0; j < N; ++j) report->traj_steps += sl[j].steps * Mn;
        report->gpu_launches = ctx->launches - launches0;
        report->h2d_bytes = static_cast<int64_t>(fused ? scalar_small_run_param_bytes() : in_bytes);
        report->d2h_bytes = d2h;
        float cms = 0.f;
        if (fused) {
            unsigned long long span[2];
            std::memcpy(span, hres + 16, sizeof span);
            cms = static_cast<float>(static_cast<double>(span[1] - span[0]) * 1e-6);
        } else if (!serial) {
            cudaEventElapsedTime(&cms, ctx->evc, ctx->ev1);
        }
        report->compose_ms = cms;
        report->total_ms = wall.ms();
    }
    return PINT_OK;
}

int pint_parareal_scalar(pint_ctx* ctx, double t0, double T, double y0, int64_t N, int64_t k, double dt, double DT,
                         double* finals, double* fine_seconds, double* coarse_seconds, pint_report* report,
                         pint_fail* fail) {
    if (!ctx || !finals || N < 1 || k < 0 || !(dt > 0.0) || !(DT > 0.0)) return PINT_E_INVALID;
    HostTimer wall;
    const long long launches0 = ctx->launches;
    std::vector<pint_slice> dec(static_cast<size_t>(N));
    if (pint_decompose(t0, T, N, dt, dec.data()) != PINT_OK)
        return pint_set_error(ctx, PINT_E_BAD_GRID, "decompose: need N >= 1, T > t0, dt > 0");
    // integrate_scalar_step's per-slice step count and effective step for each propagator
    std::vector<pint_slice> fine, coarse;
    closure_slices(dec.data(), N, dt, fine);
    closure_slices(dec.data(), N, DT, coarse);
    for (int64_t j = 0; j < N; ++j) {
        if (const int rc = check_integral(ctx, fine[j].t_end - fine[j].t_begin, fine[j].dt)) return rc;
        if (const int rc = check_integral(ctx, coarse[j].t_end - coarse[j].t_begin, coarse[j].dt)) return rc;
    }
    const size_t b_i = align256(sizeof(int64_t) * N), b_d = align256(sizeof(double) * N);
    const size_t b_w = align256(sizeof(double) * (3 * N + 1)), b_f = align256(sizeof(double) * (k + 1));
    const size_t b_ns = align256(sizeof(unsigned long long) * (N + 1));
    const size_t in_bytes = 2 * b_i + 2 * b_d;
    char* h = static_cast<char*>(pinned(in_bytes));
    char* d = static_cast<char*>(pint_scratch(ctx, 0, in_bytes + b_w + b_f + b_ns));
    if (!h || !d) return PINT_E_CUDA;
    for (int64_t j = 0; j < N; ++j) {
        reinterpret_cast<int64_t*>(h)[j] = fine[j].steps;
        reinterpret_cast<int64_t*>(h + b_i)[j] = coarse[j].steps;
        reinterpret_cast<double*>(h + 2 * b_i)[j] = fine[j].dt;
        reinterpret_cast<double*>(h + 2 * b_i + b_d)[j] = coarse[j].dt;
    }
    auto* ns = reinterpret_cast<unsigned long long*>(d + in_bytes + b_w + b_f);
    cudaEventRecord(ctx->ev0, ctx->stream);
    cudaMemcpyAsync(d, h, in_bytes, cudaMemcpyHostToDevice, ctx->stream);
    cudaMemsetAsync(ns, 0, sizeof(unsigned long long) * (N + 1), ctx->stream);
    auto* d_finals = reinterpret_cast<double*>(d + in_bytes + b_w);
    if (const int rc = launch_parareal_scalar(ctx, N, k, reinterpret_cast<int64_t*>(d), reinterpret_cast<double*>(d + 2 * b_i),
                                              reinterpret_cast<int64_t*>(d + b_i),
                                              reinterpret_cast<double*>(d + 2 * b_i + b_d), y0,
                                              reinterpret_cast<double*>(d + in_bytes), d_finals, ns, ns + N))
        return rc;
    cudaEventRecord(ctx->ev1, ctx->stream);
    std::vector<unsigned long long> hns(static_cast<size_t>(N + 1));
    cudaMemcpyAsync(finals, d_finals, sizeof(double) * (k + 1), cudaMemcpyDeviceToHost, ctx->stream);
    cudaMemcpyAsync(hns.data(), ns, sizeof(unsigned long long) * (N + 1), cudaMemcpyDeviceToHost, ctx->stream);
    pint_fail fr;
    if (const int rc = pint_fail_read(ctx, &fr)) return rc;  // (synchronises)
    if (fail) *fail = fr;
    if (fr.index >= 0) {
        const bool coarse_fail = fr.index >= parareal_coarse_fail_index();
        char buf[128];
        std::snprintf(buf, sizeof buf, "be_step_scalar_riccati: no real root (discriminant %.17g)%s", fr.value,
                      coarse_fail ? " in the coarse sweep" : "");
        if (coarse_fail && fail) fail->index = -1;  // (the coarse sweep throws unwrapped, parareal.cpp:78/112)
        return pint_set_error(ctx, PINT_E_NO_REAL_ROOT, buf);
    }
    if (fine_seconds)
        for (int64_t j = 0; j < N; ++j) fine_seconds[j] = static_cast<double>(hns[j]) * 1e-9;
    if (coarse_seconds) *coarse_seconds = static_cast<double>(hns[N]) * 1e-9 / static_cast<double>((k + 1) * N);
    if (report) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
        report->message_count = (2 * k + 1) * (N - 1);  // parareal_message_count (parareal.cpp:141-143)
        report->bytes_communicated = report->message_count * static_cast<int64_t>(sizeof(double));
        report->extrapolation_count = 0;
        report->device_ms = ms;
        report->compose_ms = static_cast<double>(hns[N]) * 1e-6;  // (the coarse sweeps)
        int64_t ts = 0;
        for (int64_t j = 0; j < N; ++j) ts += k * fine[j].steps + (k + 1) * coarse[j].steps;
        report->traj_steps = ts;
        report->gpu_launches = ctx->launches - launches0;
        report->h2d_bytes = static_cast<int64_t>(in_bytes);
        report->d2h_bytes = static_cast<int64_t>(sizeof(double) * (k + 1) + 8 * (N + 1));
        report->total_ms = wall.ms();
    }
    return PINT_OK;
}

int pint_scalar_integrate(pint_ctx* ctx, const pint_scalar_rhs* rhs, const pint_slice* slice,
                          int64_t K, const double* y0, double* y_out, pint_fail* fail) {
    if (!ctx || !rhs || !slice || K < 0) return PINT_E_INVALID;
    if (fail) *fail = pint_fail{-1, 0, 0, 0.0};
    if (K == 0) return PINT_OK;
    if (rhs->precision != PINT_F64) return pint_set_error(ctx, PINT_E_INVALID, "scalar_integrate: FP64 only");
    // integrate_scalar (nievergelt.cpp:29-35): steps_for + dt_eff from the slice bounds
    const int64_t steps = slice->steps;
    const double h = slice->dt;
    if (const int rc = check_integral(ctx, slice->t_end - slice->t_begin, h)) return rc;
    const size_t bytes = align256(sizeof(double) * K) * 2 + 512;
    char* d = static_cast<char*>(pint_scratch(ctx, 0, bytes));
    if (!d) return PINT_E_CUDA;
    Carve cv{d};
    auto* d_steps = cv.take<int64_t>(1);
    auto* d_h = cv.take<double>(1);
    auto* d_y0 = cv.take<double>(K);
    auto* d_out = cv.take<double>(K);
    cudaMemcpyAsync(d_steps, &steps, sizeof steps, cudaMemcpyHostToDevice, ctx->stream);
    cudaMemcpyAsync(d_h, &h, sizeof h, cudaMemcpyHostToDevice, ctx->stream);
    cudaMemcpyAsync(d_y0, y0, sizeof(double) * K, cudaMemcpyHostToDevice, ctx->stream);
    int rc = launch_scalar_ensemble(ctx, rhs, 1, K, d_steps, d_h, d_y0, d_out, nullptr);
    if (rc) return rc;
    cudaMemcpyAsync(y_out, d_out, sizeof(double) * K, cudaMemcpyDeviceToHost, ctx->stream);
    if (!ok(ctx, cudaStreamSynchronize(ctx->stream), "scalar_integrate sync")) return PINT_E_CUDA;
    pint_fail fr;
    if ((rc = pint_fail_read(ctx, &fr))) return rc;
    if (fail) *fail = fr;
    if (fr.index >= 0) {
        char buf[128];
        std::snprintf(buf, sizeof buf, "be_step_scalar_riccati: 1 - 4 dt y = %f", fr.value);
        return pint_set_error(ctx, fr.code, buf);
    }
    return PINT_OK;
}

// Device tables for a set of (closure-normalised) heat slices; returns device pointers.
namespace {
struct HeatDev {
    int64_t n = 0, N = 0, Q = 0, S = 0;
    int64_t* step_off = nullptr;
    double *slice_dt = nullptr, *r = nullptr, *fa = nullptr, *fb = nullptr, *sx = nullptr;
    double* factor = nullptr;
    size_t h2d = 0;
};

// Step segments of the e2e heat run: while the device builds steps [s0, s1) of every slice, the
// host fills (and the side stream copies and factors) the next segment's tables, so the build
// starts after the first segment's tables instead of all of them. The first segment is short
// (the build waits for it); the host fills ~10x faster than the device builds, so it stays ahead.
constexpr int kHeatSegments = 3;
// segment ends in eighths of S (the last segment ends at S). Default: [0, S/4), [S/4, S) — measured
// at C2 (tools/e2e_breakdown.py) e2e 1.70 ms unsegmented, 1.64 with "2", 1.65 "1", 1.69 "1,4",
// 1.71 "2,5": every extra boundary costs a record-kernel gap. PINT_HEAT_SPLIT: experiments only
int64_t heat_segment_end(int64_t S, int k) {
    static const std::vector<int64_t> ends = [] {
        std::vector<int64_t> v;
        const char* e = std::getenv("PINT_HEAT_SPLIT");
        for (const char* p = e ? e : "2"; *p && static_cast<int>(v.size()) < kHeatSegments - 1;) {
            v.push_back(std::strtol(p, const_cast<char**>(&p), 10));
            while (*p == ',') ++p;
        }
        return v;
    }();
    return k >= static_cast<int>(ends.size()) ? S : std::max<int64_t>(1, S * ends[k] / 8);
}

using StepsFn = std::function<int(int64_t s0, int64_t s1)>;

int heat_upload(pint_ctx* ctx, double dx, const std::vector<pint_slice>& sl, HeatDev& H,
                const StepsFn* on_steps = nullptr, int build_mode = PINT_BUILD_EXACT) {
    const bool fast = build_mode == PINT_BUILD_FAST;
    int64_t n = 0;
    if (const int rc = heat_dim(ctx, dx, &n)) return rc;
    for (const auto& s : sl)
        if (const int rc = check_integral(ctx, s.t_end - s.t_begin, s.dt)) return rc;
    const int64_t N = static_cast<int64_t>(sl.size());
    const int64_t Q = pint_heat_total_steps(sl.data(), N);
    const size_t b_off = align256(sizeof(int64_t) * (N + 1)), b_dt = align256(sizeof(double) * N);
    const size_t b_q = align256(sizeof(double) * Q), b_sx = align256(sizeof(double) * n);
    const size_t in_bytes = b_off + b_dt + 3 * b_q + b_sx;
    char* h = static_cast<char*>(pinned(in_bytes));
    if (!h) return pint_set_error(ctx, PINT_E_CUDA, "pinned staging allocation failed");
    auto* h_off = reinterpret_cast<int64_t*>(h);
    auto* h_dt = reinterpret_cast<double*>(h + b_off);
    auto* h_r = reinterpret_cast<double*>(h + b_off + b_dt);
    auto* h_fa = reinterpret_cast<double*>(h + b_off + b_dt + b_q);
    auto* h_fb = reinterpret_cast<double*>(h + b_off + b_dt + 2 * b_q);
    auto* h_sx = reinterpret_cast<double*>(h + b_off + b_dt + 3 * b_q);
    for (int64_t j = 0; j < N; ++j) h_dt[j] = sl[j].dt;
    h_off[0] = 0;
    for (int64_t j = 0; j < N; ++j) h_off[j + 1] = h_off[j] + sl[j].steps;
    for (int64_t i = 0; i < n; ++i) h_sx[i] = std::sin(kPi * (static_cast<double>(i + 1) * dx));
    int64_t S = 0;
    for (const auto& s : sl) S = std::max<int64_t>(S, s.steps);
    char* d = static_cast<char*>(pint_scratch(ctx, 0, in_bytes));
    if (fast && !heat_fast_supported(n))
        return pint_set_error(ctx, PINT_E_INVALID, "heat fast build: n > 768 unsupported (use PINT_BUILD_EXACT)");
    const int64_t rec_doubles = fast ? heat_fast_records_doubles(n, N, S) : heat_records_doubles(n, N, S);
    double* f = static_cast<double*>(pint_scratch(ctx, 1, sizeof(double) * rec_doubles));
    if (!d || !f) return PINT_E_CUDA;
    H.n = n;
    H.N = N;
    H.Q = Q;
    H.S = S;
    H.step_off = reinterpret_cast<int64_t*>(d);
    H.slice_dt = reinterpret_cast<double*>(d + b_off);
    H.r = reinterpret_cast<double*>(d + b_off + b_dt);
    H.fa = reinterpret_cast<double*>(d + b_off + b_dt + b_q);
    H.fb = reinterpret_cast<double*>(d + b_off + b_dt + 2 * b_q);
    H.sx = reinterpret_cast<double*>(d + b_off + b_dt + 3 * b_q);
    H.factor = f;
    H.h2d = in_bytes;
    // slice table + sx first, then the per-step tables in chunks of slices (multiples of 32, the
    // forced grid's slice groups): the host pool computes chunk c + 1 (glibc sin/cos) while the
    // copy engine and the record kernel work on chunk c
    // (step segments: the tables go on the side stream, after the slice table and sx)
    cudaStream_t tab_stream = ctx->stream;
    auto h2d = [&](const void* src, void* dst, size_t bytes) {
        return ok(ctx, cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, tab_stream), "H2D heat tables");
    };
    if (!h2d(h_off, H.step_off, sizeof(int64_t) * (N + 1)) || !h2d(h_dt, H.slice_dt, sizeof(double) * N) ||
        !h2d(h_sx, H.sx, sizeof(double) * n))
        return PINT_E_CUDA;
    if (on_steps) {  // step segments (uniform slices: slice j's steps at j*S in every table)
        cudaEventRecord(ctx->ev_fork, ctx->stream);  // slice table + sx are on the device
        cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0);
        tab_stream = ctx->side;
        int64_t s0 = 0;
        for (int k = 0; k < kHeatSegments && s0 < S; ++k) {
            const int64_t s1 = std::max(s0 + 1, std::min(S, heat_segment_end(S, k)));
            // segment k's block at offset N * s0 of each table (the blocks tile the Q = N * S slots)
            const int64_t o = N * s0, cnt = N * (s1 - s0);
            heat_fill_step_range(dx, sl.data(), N, s0, s1, h_r + o, h_fa + o, h_fb + o);
            if (!h2d(h_r + o, H.r + o, sizeof(double) * cnt) || !h2d(h_fa + o, H.fa + o, sizeof(double) * cnt) ||
                !h2d(h_fb + o, H.fb + o, sizeof(double) * cnt))
                return PINT_E_CUDA;
            if (const int rc = launch_heat_factor_block(ctx, ctx->side, n, N, S, 0, N, s0, s1 - s0, s1 - s0,
                                                        H.step_off, H.slice_dt, H.r + o, H.fa + o, H.fb + o, H.sx,
                                                        H.factor))
                return rc;
            cudaEventRecord(ctx->ev_join, ctx->side);
            cudaStreamWaitEvent(ctx->stream, ctx->ev_join, 0);
            if (const int rc = (*on_steps)(s0, s1)) return rc;
            s0 = s1;
        }
        return PINT_OK;
    }
    const int64_t chunk = std::max<int64_t>(32, (N / 4 + 31) / 32 * 32);
    for (int64_t j0 = 0; j0 < N; j0 += chunk) {
        const int64_t j1 = std::min(N, j0 + chunk), q0 = h_off[j0], nq = h_off[j1] - q0;
        heat_fill_steps(dx, sl.data(), j0, j1, h_off, h_r, h_fa, h_fb);
        if (!h2d(h_r + q0, H.r + q0, sizeof(double) * nq) || !h2d(h_fa + q0, H.fa + q0, sizeof(double) * nq) ||
            !h2d(h_fb + q0, H.fb + q0, sizeof(double) * nq))
            return PINT_E_CUDA;
        if (fast) continue;  // (one record launch over all slices below)
        if (const int rc = launch_heat_factor_range(ctx, n, N, S, j0, j1 - j0, H.step_off, H.slice_dt, H.r, H.fa,
                                                    H.fb, H.sx, H.factor))
            return rc;
    }
    if (fast) return launch_heat_fast_factor(ctx, ctx->stream, n, N, S, H.step_off, H.slice_dt, H.r, H.fa, H.fb, H.sx,
                                             H.factor);
    return PINT_OK;
}

// All N maps and the bit-exact chain to y. Where the build signals per-slice completion (the
// TMEM build, n in [282, 520]) the chain runs CONCURRENTLY: the 16-CTA cluster chain holds 16 SMs
// and fetches map j once ready[j] counts all of slice j's builder CTAs, while the build fills the
// other SMs. The chain is launched first and the build right behind it on the same stream with
// programmatic stream serialization: build CTAs are dispatched only once every chain CTA is
// resident (the chain triggers at its start), so the cluster never queues behind the build grid;
// nothing may sit between the two launches (an event record would make the build wait for the
// chain). The build never waits on the chain (deadlock-free; the chain's waits are bounded and
// fail loudly). Kernel attributes are set before the launches: cudaFuncSetAttribute waits for a
// running kernel, here for the chain that waits for the build.
int heat_build_chain(pint_ctx* ctx, int64_t n, int64_t N, int64_t S, const int64_t* step_off,
                     const double* slice_dt, const double* records, const double* sx, double* maps,
                     const double* y0, double* y, unsigned long long* per_slice_ns, int guarded,
                     int build_mode) {
    const bool fast = build_mode == PINT_BUILD_FAST;
    const int target = fast ? heat_fast_ready_target(n) : heat_build_ready_target(n);
    // ready[N] counters, then {build start, build end, chain end} globaltimer words
    const size_t ready_bytes = sizeof(int) * static_cast<size_t>((N + 1) & ~1ll);
    int* ready = target ? static_cast<int*>(pint_scratch(ctx, 5, ready_bytes + 32)) : nullptr;
    static const int overlap_env = [] {  // PINT_OVERLAP=0: build, then chain (experiments, debugging)
        const char* e = std::getenv("PINT_OVERLAP");
        return e ? std::atoi(e) : 1;
    }();
    if (!target || !ready || n > 512 || overlap_env == 0) {
        if (const int rc = fast ? launch_heat_fast_build(ctx, n, N, S, records, maps)
                                : launch_heat_build(ctx, n, N, S, step_off, slice_dt, records, sx, maps, per_slice_ns,
                                                    guarded))
            return rc;
        cudaEventRecord(ctx->evc, ctx->stream);
        return launch_affine_chain(ctx, n, N, maps, y0, y);
    }
    if (fast) heat_fast_prepare(n);
    else heat_build_prepare(n);
    if (!fast)  // (the forced columns ahead of the chain: nothing may sit between it and the build)
        if (const int rc = launch_heat_forced_first(ctx, n, N, S, step_off, records, maps, per_slice_ns, guarded))
            return rc;
    cudaMemsetAsync(ready, 0, ready_bytes, ctx->stream);
    cudaMemsetAsync(reinterpret_cast<char*>(ready) + ready_bytes, 0xff, 8, ctx->stream);  // (min start)
    cudaMemsetAsync(reinterpret_cast<char*>(ready) + ready_bytes + 8, 0, 16, ctx->stream);
    ctx->span_words = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(ready) + ready_bytes);
    if (const int rc = launch_affine_chain_on(ctx, ctx->stream, n, N, maps, y0, y, ready, target, fast ? 0 : 128))
        return rc;
    if (overlap_env == 2) cudaEventRecord(ctx->evc, ctx->stream);  // (test hook: serialise the build behind the chain)
    if (const int rc = fast ? launch_heat_fast_build(ctx, n, N, S, records, maps, ready)
                            : launch_heat_build_steps(ctx, n, N, S, step_off, records, maps, per_slice_ns, guarded, 0,
                                                      S, ready))
        return rc;
    cudaEventRecord(ctx->evc, ctx->stream);
    return PINT_OK;
}

int singular_check(pint_ctx* ctx) {
    pint_fail fr;
    if (const int rc = pint_fail_read(ctx, &fr)) return rc;
    if (fr.index >= 0) {
        if (fr.code == PINT_E_RANGE_RETRY) return PINT_E_RANGE_RETRY;  // caller re-runs guarded
        if (fr.code == PINT_E_SERIALIZED) return PINT_E_SERIALIZED;    // caller re-runs the compose
        char buf[96];
        std::snprintf(buf, sizeof buf, "thomas_solve: zero pivot at row %d", static_cast<int>(fr.value));
        return pint_set_error(ctx, PINT_E_SINGULAR, buf);
    }
    return PINT_OK;
}
}  // namespace

int pint_run_heat(pint_ctx* ctx, double dx, double dt, double T, int64_t N, int compose_mode,
                  const double* y0, double* y_out, double* per_slice_seconds, pint_report* report) {
    return pint_run_heat_ex(ctx, dx, dt, T, N, PINT_BUILD_EXACT, compose_mode, y0, y_out, per_slice_seconds, report);
}

int pint_run_heat_ex(pint_ctx* ctx, double dx, double dt, double T, int64_t N, int build_mode, int compose_mode,
                     const double* y0, double* y_out, double* per_slice_seconds, pint_report* report) {
    if (!ctx || !y_out || N < 1 || (build_mode != PINT_BUILD_EXACT && build_mode != PINT_BUILD_FAST))
        return PINT_E_INVALID;
    const bool fast = build_mode == PINT_BUILD_FAST;
    HostTimer wall;
    const long long launches0 = ctx->launches;
    std::vector<pint_slice> sl(static_cast<size_t>(N));
    if (pint_decompose(0.0, T, N, dt, sl.data()) != PINT_OK)
        return pint_set_error(ctx, PINT_E_BAD_GRID, "decompose: need N >= 1, T > t0, dt > 0");
    closure_slices(sl.data(), N, dt, sl);
    cudaEventRecord(ctx->ev0, ctx->stream);
    int64_t n = 0;
    if (const int rc = heat_dim(ctx, dx, &n)) return rc;
    const int64_t ldm = pint_affine_ldm(n);
    const size_t map_elems = static_cast<size_t>(n * ldm);
    // maps (N) + tree scratch (ceil(N/2)) + y0 + y + per-slice timers
    const size_t b_maps = align256(sizeof(double) * map_elems * N);
    const size_t b_scr = (compose_mode == PINT_COMPOSE_TREE && N > 1) ? align256(sizeof(double) * map_elems * ((N + 1) / 2)) : 0;
    const size_t total = b_maps + b_scr + 2 * align256(sizeof(double) * n) + align256(8 * N) + 1024;
    char* d = static_cast<char*>(pint_scratch(ctx, 2, total));
    if (!d) return PINT_E_CUDA;
    Carve cv{d};
    double* d_maps = cv.take<double>(map_elems * N);
    double* d_scr = b_scr ? cv.take<double>(map_elems * ((N + 1) / 2)) : nullptr;
    double* d_y0 = cv.take<double>(n);
    double* d_y = cv.take<double>(n);
    auto* d_ns = cv.take<unsigned long long>(N);
    // step-segmented first build (uniform slices, register/shared-memory build; PINT_HEAT_SEGMENTS=0
    // turns it off): launched from inside the upload, segment by segment
    static const bool seg_env = [] {
        const char* e = std::getenv("PINT_HEAT_SEGMENTS");
        return !(e && e[0] == '0');
    }();
    bool uniform = true;
    for (const auto& s : sl) uniform = uniform && s.steps == sl[0].steps;
    const bool segmented =
        !fast && seg_env && uniform && heat_build_segmentable(n) && sl[0].steps >= 2 * kHeatSegments;
    if (per_slice_seconds) cudaMemsetAsync(d_ns, 0, sizeof(unsigned long long) * N, ctx->stream);
    HeatDev H;
    const StepsFn seg_build = [&](int64_t s0, int64_t s1) {
        return launch_heat_build_steps(ctx, n, N, sl[0].steps, H.step_off, H.factor, d_maps,
                                       per_slice_seconds ? d_ns : nullptr, 0, s0, s1);
    };
    if (const int rc = heat_upload(ctx, dx, sl, H, segmented ? &seg_build : nullptr, build_mode)) return rc;
    std::vector<double> y0v;
    if (!y0) {
        y0v.resize(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) y0v[i] = std::sin(kPi * static_cast<double>(i + 1) * dx);  // heat_initial
        y0 = y0v.data();
    }
    cudaMemcpyAsync(d_y0, y0, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream);
    std::vector<unsigned long long> ns;
    int rc = PINT_OK;
    for (int guarded = 0; guarded < 2; ++guarded) {  // second pass only if a range check tripped
        const bool overlap = !segmented && n <= 512 &&
                             (fast ? heat_fast_ready_target(n) > 0 && compose_mode == PINT_COMPOSE_CHAIN
                                   : heat_build_ready_target(n) > 0 &&
                                         (compose_mode == PINT_COMPOSE_CHAIN || n > 256));  // (only-y TREE at n > 256 IS the chain)
        if (overlap) {
            if (per_slice_seconds && guarded) cudaMemsetAsync(d_ns, 0, sizeof(unsigned long long) * N, ctx->stream);
            rc = heat_build_chain(ctx, n, N, H.S, H.step_off, H.slice_dt, H.factor, H.sx, d_maps, d_y0, d_y,
                                  per_slice_seconds ? d_ns : nullptr, guarded, build_mode);
            if (rc) return rc;
        } else if (fast) {  // (no range retry: plain FP64 arithmetic throughout)
            rc = launch_heat_fast_build(ctx, n, N, H.S, H.factor, d_maps);
            if (rc) return rc;
        } else if (guarded || !segmented) {
            if (per_slice_seconds && guarded) cudaMemsetAsync(d_ns, 0, sizeof(unsigned long long) * N, ctx->stream);
            rc = launch_heat_build(ctx, n, N, H.S, H.step_off, H.slice_dt, H.factor, H.sx, d_maps,
                                   per_slice_seconds ? d_ns : nullptr, guarded);
            if (rc) return rc;
        }
        if (!overlap) {
            cudaEventRecord(ctx->evc, ctx->stream);
            if (compose_mode == PINT_COMPOSE_TREE) rc = launch_affine_tree(ctx, n, N, d_maps, d_scr, d_y0, d_y, nullptr);
            else rc = launch_affine_chain(ctx, n, N, d_maps, d_y0, d_y);
            if (rc) return rc;
        }
        cudaEventRecord(ctx->ev1, ctx->stream);
        cudaMemcpyAsync(y_out, d_y, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream);
        if (per_slice_seconds) {
            ns.resize(static_cast<size_t>(N));
            cudaMemcpyAsync(ns.data(), d_ns, sizeof(unsigned long long) * N, cudaMemcpyDeviceToHost, ctx->stream);
        }
        if (!ok(ctx, cudaStreamSynchronize(ctx->stream), "run_heat sync")) return PINT_E_CUDA;
        rc = singular_check(ctx);
        if (rc == PINT_E_SERIALIZED) {  // the concurrent chain could not run beside the build: the maps
            if ((rc = launch_affine_chain(ctx, n, N, d_maps, d_y0, d_y))) return rc;  // are done, chain them now
            cudaEventRecord(ctx->ev1, ctx->stream);
            cudaMemcpyAsync(y_out, d_y, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream);
            if (!ok(ctx, cudaStreamSynchronize(ctx->stream), "run_heat sync")) return PINT_E_CUDA;
            rc = singular_check(ctx);
        }
        if (rc != PINT_E_RANGE_RETRY) break;
    }
    if (rc) return rc;
    if (per_slice_seconds && fast) {  // the tolerance build has no per-slice timers: its time split evenly
        float ms = 0.f, cms = 0.f;
        cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
        cudaEventElapsedTime(&cms, ctx->evc, ctx->ev1);
        for (int64_t j = 0; j < N; ++j) per_slice_seconds[j] = (ms - cms) * 1e-3 / static_cast<double>(N);
    } else if (per_slice_seconds) {
        for (int64_t j = 0; j < N; ++j) per_slice_seconds[j] = static_cast<double>(ns[j]) * 1e-9;
    }
    if (report) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
        report->message_count = N - 1;
        report->bytes_communicated = (N - 1) * n * static_cast<int64_t>(sizeof(double));
        report->extrapolation_count = 0;
        report->device_ms = ms;
        report->traj_steps = H.Q * (n + 1);
        report->gpu_launches = ctx->launches - launches0;
        report->h2d_bytes = static_cast<int64_t>(H.h2d + sizeof(double) * n);
        report->d2h_bytes = static_cast<int64_t>(sizeof(double) * n);
        float cms = 0.f;
        cudaEventElapsedTime(&cms, ctx->evc, ctx->ev1);
        report->compose_ms = cms;
        report->total_ms = wall.ms();
    }
    return PINT_OK;
}

int pint_run_heat_sharded(pint_ctx* ctx, double dx, double dt, double T, int64_t N, int build_mode,
                          int compose_mode, const double* y0, double* y_out, pint_report* report) {
    if (!ctx || N < 1 || (build_mode != PINT_BUILD_EXACT && build_mode != PINT_BUILD_FAST) ||
        (compose_mode != PINT_COMPOSE_CHAIN && compose_mode != PINT_COMPOSE_TREE))
        return PINT_E_INVALID;
    if (!ctx->comm) return pint_set_error(ctx, PINT_E_INVALID, "run_heat_sharded: no communicator (pint_comm_init*)");
    int rank = 0, W = 1;
    pint_comm_rank(ctx, &rank, &W);
    if (rank == 0 && !y_out) return PINT_E_INVALID;
    comm_counters(ctx, nullptr, nullptr, true);
    if (W == 1) {  // one rank: the single-GPU run itself (bit-identical by construction)
        const int rc = pint_run_heat_ex(ctx, dx, dt, T, N, build_mode, compose_mode, y0, y_out, nullptr, report);
        if (report) report->message_count = report->bytes_communicated = 0;  // (no transfers)
        return rc;
    }
    HostTimer wall;
    const long long launches0 = ctx->launches;
    std::vector<pint_slice> all(static_cast<size_t>(N));
    if (pint_decompose(0.0, T, N, dt, all.data()) != PINT_OK)
        return pint_set_error(ctx, PINT_E_BAD_GRID, "decompose: need N >= 1, T > t0, dt > 0");
    closure_slices(all.data(), N, dt, all);
    const int64_t lo = rank * N / W, hi = (rank + 1) * N / W, Nb = hi - lo;  // this rank's block
    const std::vector<pint_slice> sl(all.begin() + lo, all.begin() + hi);
    int64_t n = 0;
    if (const int rc = heat_dim(ctx, dx, &n)) return rc;
    cudaEventRecord(ctx->ev0, ctx->stream);
    const int64_t ldm = pint_affine_ldm(n);
    const size_t map_elems = static_cast<size_t>(n * ldm);
    const bool tree = compose_mode == PINT_COMPOSE_TREE;
    const size_t total = align256(sizeof(double) * map_elems * std::max<int64_t>(Nb, 1)) +
                         (tree ? align256(sizeof(double) * map_elems * ((Nb + 1) / 2 + 1)) : 0) +
                         (tree ? align256(sizeof(double) * map_elems) : 0) +
                         (tree && rank == 0 ? align256(sizeof(double) * map_elems * W) : 0) +
                         3 * align256(sizeof(double) * n) + 1024;
    char* d = static_cast<char*>(pint_scratch(ctx, 2, total));
    if (!d) return PINT_E_CUDA;
    Carve cv{d};
    double* d_maps = cv.take<double>(map_elems * std::max<int64_t>(Nb, 1));
    double* d_scr = tree ? cv.take<double>(map_elems * ((Nb + 1) / 2 + 1)) : nullptr;
    double* d_comp = tree ? cv.take<double>(map_elems) : nullptr;
    double* d_gath = tree && rank == 0 ? cv.take<double>(map_elems * W) : nullptr;
    double* d_y0 = cv.take<double>(n);
    double* d_y = cv.take<double>(n);
    double* d_lam = cv.take<double>(n);
    std::vector<double> y0v;
    if (!y0) {
        y0v.resize(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) y0v[i] = std::sin(kPi * static_cast<double>(i + 1) * dx);  // heat_initial
        y0 = y0v.data();
    }
    cudaMemcpyAsync(d_y0, y0, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream);
    // this block's maps (its slices' records, then the build; a tripped range check re-runs guarded)
    HeatDev H;
    if (Nb > 0) {
        if (const int rc = heat_upload(ctx, dx, sl, H, nullptr, build_mode)) return rc;
        for (int guarded = 0; guarded < 2; ++guarded) {
            int rc = build_mode == PINT_BUILD_FAST
                         ? launch_heat_fast_build(ctx, n, Nb, H.S, H.factor, d_maps)
                         : launch_heat_build(ctx, n, Nb, H.S, H.step_off, H.slice_dt, H.factor, H.sx, d_maps, nullptr,
                                             guarded);
            if (rc) return rc;
            rc = singular_check(ctx);  // (synchronises)
            if (rc == PINT_OK) break;
            if (rc != PINT_E_RANGE_RETRY) return rc;
        }
    }
    cudaEventRecord(ctx->evc, ctx->stream);
    if (tree) {  // the block map, ONE gather of the W block maps, rank 0 applies them in rank order
        if (Nb > 0) {
            if (const int rc = launch_affine_tree(ctx, n, Nb, d_maps, d_scr, d_y0, d_lam, d_comp)) return rc;
        } else {  // an empty block composes to the identity map [I | 0]
            std::vector<double> id(map_elems, 0.0);
            for (int64_t i = 0; i < n; ++i) id[static_cast<size_t>(i * ldm + i)] = 1.0;
            cudaMemcpyAsync(d_comp, id.data(), sizeof(double) * map_elems, cudaMemcpyHostToDevice, ctx->stream);
            cudaStreamSynchronize(ctx->stream);
        }
        if (const int rc = comm_gather(ctx, d_comp, d_gath, sizeof(double) * map_elems, 0)) return rc;
        if (rank == 0)
            if (const int rc = launch_affine_chain(ctx, n, W, d_gath, d_y0, d_y)) return rc;
    } else {  // the running state handed rank to rank (0 -> 1 -> ... -> W-1 -> 0), each block chained
        const double* in = d_y0;
        if (rank > 0) {
            if (const int rc = comm_recv(ctx, d_lam, sizeof(double) * n, rank - 1)) return rc;
            in = d_lam;
        }
        if (Nb > 0) {
            if (const int rc = launch_affine_chain(ctx, n, Nb, d_maps, in, d_y)) return rc;
        } else {
            cudaMemcpyAsync(d_y, in, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream);
        }
        if (const int rc = comm_send(ctx, d_y, sizeof(double) * n, (rank + 1) % W)) return rc;
        if (rank == 0)
            if (const int rc = comm_recv(ctx, d_y, sizeof(double) * n, W - 1)) return rc;
    }
    cudaEventRecord(ctx->ev1, ctx->stream);
    if (rank == 0) cudaMemcpyAsync(y_out, d_y, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream);
    if (!ok(ctx, cudaStreamSynchronize(ctx->stream), "run_heat_sharded sync")) return PINT_E_CUDA;
    if (report) {
        float ms = 0.f, cms = 0.f;
        cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
        cudaEventElapsedTime(&cms, ctx->evc, ctx->ev1);
        int64_t msgs = 0, bytes = 0;
        comm_counters(ctx, &msgs, &bytes, false);
        report->message_count = msgs;
        report->bytes_communicated = bytes;
        report->extrapolation_count = 0;
        report->device_ms = ms;
        report->compose_ms = cms;
        report->traj_steps = (Nb > 0 ? H.Q : 0) * (n + 1);
        report->gpu_launches = ctx->launches - launches0;
        report->h2d_bytes = static_cast<int64_t>((Nb > 0 ? H.h2d : 0) + sizeof(double) * n);
        report->d2h_bytes = rank == 0 ? static_cast<int64_t>(sizeof(double) * n) : 0;
        report->total_ms = wall.ms();
    }
    return PINT_OK;
}

namespace {
// Tables and slice-major records of the slices `sl` (each at most S steps) into scratch slots:
// records [N][S][record] (slice j's steps at j S), device step counts `steps`.
int slices_records(pint_ctx* ctx, double dx, const std::vector<pint_slice>& sl, int slot_tab, int slot_rec,
                   int64_t* n_out, int64_t* S_out, int64_t** steps, double** rec) {
    int64_t n = 0;
    if (const int rc = heat_dim(ctx, dx, &n)) return rc;
    const int64_t N = static_cast<int64_t>(sl.size());
    int64_t S = 0, Q = 0;
    for (const auto& s : sl) {
        if (const int rc = check_integral(ctx, s.t_end - s.t_begin, s.dt)) return rc;
        S = std::max<int64_t>(S, s.steps);
        Q += s.steps;
    }
    const size_t b_off = align256(sizeof(int64_t) * (N + 1)), b_st = align256(sizeof(int64_t) * N);
    const size_t b_dt = align256(sizeof(double) * N), b_q = align256(sizeof(double) * Q);
    const size_t b_sx = align256(sizeof(double) * n);
    const size_t bytes = b_off + b_st + b_dt + 3 * b_q + b_sx;
    char* h = static_cast<char*>(pinned(bytes));
    char* d = static_cast<char*>(pint_scratch(ctx, slot_tab, bytes));
    double* r = static_cast<double*>(pint_scratch(ctx, slot_rec, sizeof(double) * N * S * heat_record_stride(n)));
    if (!h || !d || !r) return pint_set_error(ctx, PINT_E_CUDA, "parareal: table / record allocation failed");
    auto* h_off = reinterpret_cast<int64_t*>(h);
    auto* h_st = reinterpret_cast<int64_t*>(h + b_off);
    auto* h_dt = reinterpret_cast<double*>(h + b_off + b_st);
    h_off[0] = 0;
    for (int64_t j = 0; j < N; ++j) {
        h_off[j + 1] = h_off[j] + sl[j].steps;
        h_st[j] = sl[j].steps;
        h_dt[j] = sl[j].dt;
    }
    double* h_q = reinterpret_cast<double*>(h + b_off + b_st + b_dt);
    heat_fill_steps(dx, sl.data(), 0, N, h_off, h_q, h_q + b_q / 8, h_q + 2 * b_q / 8);
    auto* h_sx = reinterpret_cast<double*>(h + b_off + b_st + b_dt + 3 * b_q);
    for (int64_t i = 0; i < n; ++i) h_sx[i] = std::sin(kPi * (static_cast<double>(i + 1) * dx));
    if (!ok(ctx, cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, ctx->stream), "H2D parareal tables") ||
        !ok(ctx, cudaStreamSynchronize(ctx->stream), "H2D parareal tables sync"))
        return PINT_E_CUDA;
    const double* dq = reinterpret_cast<const double*>(d + b_off + b_st + b_dt);
    if (const int rc = launch_heat_factor_block(ctx, ctx->stream, n, N, S, 0, N, 0, S, 0,
                                                reinterpret_cast<const int64_t*>(d), reinterpret_cast<const double*>(d + b_off + b_st),
                                                dq, dq + b_q / 8, dq + 2 * b_q / 8,
                                                reinterpret_cast<const double*>(d + b_off + b_st + b_dt + 3 * b_q), r, 0, true))
        return rc;
    *n_out = n;
    *S_out = S;
    *steps = reinterpret_cast<int64_t*>(d + b_off);
    *rec = r;
    return PINT_OK;
}
}  // namespace

int pint_parareal_heat(pint_ctx* ctx, double dx, double T, const double* y0, int64_t N, int64_t k, double dt,
                       double DT, double* finals, pint_report* report) {
    if (!ctx || !finals || N < 1 || k < 0 || !(dt > 0.0) || !(DT > 0.0)) return PINT_E_INVALID;
    HostTimer wall;
    const long long launches0 = ctx->launches;
    std::vector<pint_slice> dec(static_cast<size_t>(N));
    if (pint_decompose(0.0, T, N, dt, dec.data()) != PINT_OK)
        return pint_set_error(ctx, PINT_E_BAD_GRID, "decompose: need N >= 1, T > t0, dt > 0");
    std::vector<pint_slice> fine, coarse;  // the integrate closure at dt (fine) and DT (coarse)
    closure_slices(dec.data(), N, dt, fine);
    closure_slices(dec.data(), N, DT, coarse);
    cudaEventRecord(ctx->ev0, ctx->stream);
    int64_t n = 0, Sf = 0, Sc = 0;
    int64_t *st_f = nullptr, *st_c = nullptr;
    double *rec_f = nullptr, *rec_c = nullptr;
    if (const int rc = slices_records(ctx, dx, fine, 0, 1, &n, &Sf, &st_f, &rec_f)) return rc;
    if (const int rc = slices_records(ctx, dx, coarse, 6, 7, &n, &Sc, &st_c, &rec_c)) return rc;
    const int64_t stride = heat_record_stride(n);
    const size_t vn = sizeof(double) * n;
    char* d = static_cast<char*>(pint_scratch(ctx, 2, (4 * N + 2 + (k + 1)) * vn + 1024));
    if (!d) return PINT_E_CUDA;
    auto* d_y0 = reinterpret_cast<double*>(d);
    double* lam = d_y0 + n;
    double* gprev = lam + (N + 1) * n;
    double* fout = gprev + N * n;
    double* d_fin = fout + N * n;
    std::vector<double> y0v;
    if (!y0) {
        y0v.resize(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) y0v[i] = std::sin(kPi * static_cast<double>(i + 1) * dx);  // heat_initial
        y0 = y0v.data();
    }
    cudaMemcpyAsync(d_y0, y0, vn, cudaMemcpyHostToDevice, ctx->stream);
    int rc = PINT_OK;
    for (int guarded = 0; guarded < 2; ++guarded) {  // a tripped range check re-runs everything guarded
        if ((rc = launch_heat_parareal_coarse(ctx, n, N, rec_c, Sc * stride, st_c, d_y0, nullptr, gprev, lam, guarded)))
            return rc;
        cudaMemcpyAsync(d_fin, lam + N * n, vn, cudaMemcpyDeviceToDevice, ctx->stream);
        for (int64_t it = 1; it <= k; ++it) {
            cudaMemcpyAsync(fout, lam, vn * N, cudaMemcpyDeviceToDevice, ctx->stream);  // fine wave from lambda_j
            if ((rc = launch_heat_integrate_slices(ctx, n, N, st_f, rec_f, Sf * stride, fout, guarded))) return rc;
            if ((rc = launch_heat_parareal_coarse(ctx, n, N, rec_c, Sc * stride, st_c, d_y0, fout, gprev, lam, guarded)))
                return rc;
            cudaMemcpyAsync(d_fin + it * n, lam + N * n, vn, cudaMemcpyDeviceToDevice, ctx->stream);
        }
        rc = singular_check(ctx);  // (synchronises)
        if (rc != PINT_E_RANGE_RETRY) break;
    }
    if (rc) return rc;
    cudaEventRecord(ctx->ev1, ctx->stream);
    cudaMemcpyAsync(finals, d_fin, vn * (k + 1), cudaMemcpyDeviceToHost, ctx->stream);
    if (!ok(ctx, cudaStreamSynchronize(ctx->stream), "parareal_heat sync")) return PINT_E_CUDA;
    if (report) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
        report->message_count = (2 * k + 1) * (N - 1);
        report->bytes_communicated = report->message_count * static_cast<int64_t>(vn);
        report->extrapolation_count = 0;
        report->device_ms = ms;
        report->compose_ms = 0.0;
        int64_t ts = 0;
        for (int64_t j = 0; j < N; ++j) ts += k * fine[j].steps + (k + 1) * coarse[j].steps;
        report->traj_steps = ts;
        report->gpu_launches = ctx->launches - launches0;
        report->h2d_bytes = static_cast<int64_t>(vn);
        report->d2h_bytes = static_cast<int64_t>(vn * (k + 1));
        report->total_ms = wall.ms();
    }
    return PINT_OK;
}

int pint_heat_maps(pint_ctx* ctx, double dx, double dt, const pint_slice* slices, int64_t N, double* G,
                   double* c) {
    if (!ctx || !slices || N < 1) return PINT_E_INVALID;
    std::vector<pint_slice> sl;
    closure_slices(slices, N, dt, sl);
    HeatDev H;
    if (const int rc = heat_upload(ctx, dx, sl, H)) return rc;
    const int64_t n = H.n, ldm = pint_affine_ldm(n);
    double* d_maps = static_cast<double*>(pint_scratch(ctx, 2, sizeof(double) * n * ldm * N));
    if (!d_maps) return PINT_E_CUDA;
    std::vector<double> host(static_cast<size_t>(n * ldm * N));
    int rc = PINT_OK;
    for (int guarded = 0; guarded < 2; ++guarded) {
        if ((rc = launch_heat_build(ctx, n, N, H.S, H.step_off, H.slice_dt, H.factor, H.sx, d_maps, nullptr, guarded)))
            return rc;
        cudaMemcpyAsync(host.data(), d_maps, sizeof(double) * host.size(), cudaMemcpyDeviceToHost, ctx->stream);
        if (!ok(ctx, cudaStreamSynchronize(ctx->stream), "heat_maps sync")) return PINT_E_CUDA;
        rc = singular_check(ctx);
        if (rc != PINT_E_RANGE_RETRY) break;
    }
    if (rc) return rc;
    for (int64_t j = 0; j < N; ++j)
        for (int64_t i = 0; i < n; ++i) {
            const double* row = host.data() + (j * n + i) * ldm;
            if (G) std::memcpy(G + (j * n + i) * n, row, sizeof(double) * n);
            if (c) c[j * n + i] = row[n];
        }
    return PINT_OK;
}

int pint_heat_integrate(pint_ctx* ctx, double dx, const pint_slice* slice, double dt_nominal,
                        int with_forcing, int64_t K, double* y) {
    if (!ctx || !slice || K < 0) return PINT_E_INVALID;
    if (K == 0) return PINT_OK;
    std::vector<pint_slice> sl;
    closure_slices(slice, 1, dt_nominal, sl);
    IntegTables T;
    if (const int rc = integ_upload(ctx, ctx->stream, 0, dx, sl[0], T)) return rc;
    const int64_t n = T.n;
    double* rec = static_cast<double*>(pint_scratch(ctx, 1, sizeof(double) * heat_integrate_records_doubles(n)));
    double* d_y = static_cast<double*>(pint_scratch(ctx, 2, 2 * sizeof(double) * n * K));
    if (!rec || !d_y) return PINT_E_CUDA;
    double* d_y0 = d_y + n * K;  // (the start states, for a guarded re-run)
    cudaMemcpyAsync(d_y, y, sizeof(double) * n * K, cudaMemcpyHostToDevice, ctx->stream);
    cudaMemcpyAsync(d_y0, d_y, sizeof(double) * n * K, cudaMemcpyDeviceToDevice, ctx->stream);
    int rc = PINT_OK;
    for (int guarded = 0; guarded < 2; ++guarded) {  // second pass only if a range check tripped
        if (guarded) cudaMemcpyAsync(d_y, d_y0, sizeof(double) * n * K, cudaMemcpyDeviceToDevice, ctx->stream);
        if ((rc = integ_enqueue(ctx, ctx->stream, T, rec, with_forcing, K, d_y, ctx->d_fail, guarded))) return rc;
        rc = singular_check(ctx);  // (synchronises)
        if (rc != PINT_E_RANGE_RETRY) break;
    }
    if (rc) return rc;
    cudaMemcpyAsync(y, d_y, sizeof(double) * n * K, cudaMemcpyDeviceToHost, ctx->stream);
    return ok(ctx, cudaStreamSynchronize(ctx->stream), "heat_integrate sync") ? PINT_OK : PINT_E_CUDA;
}

int pint_heat_serial_begin(pint_ctx* ctx, double dx, double dt, double T, const double* y0) {
    if (!ctx || !y0) return PINT_E_INVALID;
    auto& R = ctx->serial_run;
    if (R.active) return pint_set_error(ctx, PINT_E_INVALID, "heat_serial_begin: a serial run is already in flight");
    // run_serial's single slice (nievergelt.cpp:126-143) as the integrate closure steps it
    const int64_t steps = pint_steps_for(T, dt);
    const pint_slice whole{0.0, T, steps, T / static_cast<double>(steps)};
    std::vector<pint_slice> sl;
    closure_slices(&whole, 1, dt, sl);
    IntegTables Tb;
    if (const int rc = integ_upload(ctx, ctx->serial, 6, dx, sl[0], Tb)) return rc;
    const int64_t n = Tb.n, rec_doubles = heat_integrate_records_doubles(n);
    double* d = static_cast<double*>(pint_scratch(ctx, 7, sizeof(double) * (rec_doubles + 2 * n)));
    if (!d) return PINT_E_CUDA;
    R.n = n;
    R.Q = Tb.Q;
    R.rec = d;
    R.y = d + rec_doubles;
    R.y0 = R.y + n;
    R.step_off = Tb.step_off, R.dt = Tb.dt, R.r = Tb.r, R.fa = Tb.fa, R.fb = Tb.fb, R.sx = Tb.sx;
    if (!ok(ctx, cudaMemcpyAsync(R.y0, y0, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->serial), "H2D serial y0") ||
        !ok(ctx, cudaMemcpyAsync(R.y, R.y0, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->serial), "serial y") ||
        !ok(ctx, cudaStreamSynchronize(ctx->serial), "serial y0 sync"))  // (y0 is the caller's buffer)
        return PINT_E_CUDA;
    if (const int rc = integ_enqueue(ctx, ctx->serial, Tb, R.rec, 1, 1, R.y, ctx->d_fail_serial, 0)) return rc;
    R.active = true;
    return PINT_OK;
}

int pint_heat_serial_end(pint_ctx* ctx, double* y_out) {
    if (!ctx || !y_out) return PINT_E_INVALID;
    auto& R = ctx->serial_run;
    if (!R.active) return pint_set_error(ctx, PINT_E_INVALID, "heat_serial_end: no serial run in flight");
    R.active = false;
    const IntegTables Tb{R.n, R.Q, R.step_off, R.dt, R.r, R.fa, R.fb, R.sx};
    for (int guarded = 0; guarded < 2; ++guarded) {
        pint_fail f;
        if (const int rc = fail_read_on(ctx, ctx->d_fail_serial, ctx->serial, &f)) return rc;  // (synchronises)
        if (f.index < 0) break;
        if (f.code != PINT_E_RANGE_RETRY || guarded) {
            char buf[96];
            std::snprintf(buf, sizeof buf, "thomas_solve: zero pivot at row %d", static_cast<int>(f.value));
            return pint_set_error(ctx, PINT_E_SINGULAR, buf);
        }
        cudaMemcpyAsync(R.y, R.y0, sizeof(double) * R.n, cudaMemcpyDeviceToDevice, ctx->serial);
        if (const int rc = integ_enqueue(ctx, ctx->serial, Tb, R.rec, 1, 1, R.y, ctx->d_fail_serial, 1)) return rc;
    }
    return ok(ctx, cudaMemcpyAsync(y_out, R.y, sizeof(double) * R.n, cudaMemcpyDeviceToHost, ctx->serial), "D2H serial") &&
                   ok(ctx, cudaStreamSynchronize(ctx->serial), "serial sync")
               ? PINT_OK
               : PINT_E_CUDA;
}

int pint_affine_compose(pint_ctx* ctx, int mode, int64_t n, int64_t N, const double* G, const double* c,
                        const double* y0, double* y_out) {
    if (!ctx || n < 1 || N < 0 || !y0 || !y_out) return PINT_E_INVALID;
    if (N == 0) {
        std::memcpy(y_out, y0, sizeof(double) * n);
        return PINT_OK;
    }
    const int64_t ldm = pint_affine_ldm(n);
    const size_t map_elems = static_cast<size_t>(n * ldm);
    std::vector<double> host(map_elems * N, 0.0);
    for (int64_t j = 0; j < N; ++j)
        for (int64_t i = 0; i < n; ++i) {
            double* row = host.data() + (j * n + i) * ldm;
            std::memcpy(row, G + (j * n + i) * n, sizeof(double) * n);
            row[n] = c[j * n + i];
        }
    const size_t b_maps = align256(sizeof(double) * map_elems * N);
    const size_t b_scr = align256(sizeof(double) * map_elems * ((N + 1) / 2));
    char* d = static_cast<char*>(pint_scratch(ctx, 2, b_maps + b_scr + 2 * align256(sizeof(double) * n) + 512));
    if (!d) return PINT_E_CUDA;
    Carve cv{d};
    double* d_maps = cv.take<double>(map_elems * N);
    double* d_scr = cv.take<double>(map_elems * ((N + 1) / 2));
    double* d_y0 = cv.take<double>(n);
    double* d_y = cv.take<double>(n);
    cudaMemcpyAsync(d_maps, host.data(), sizeof(double) * host.size(), cudaMemcpyHostToDevice, ctx->stream);
    cudaMemcpyAsync(d_y0, y0, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream);
    int rc = pint_affine_compose_dev(ctx, mode, n, N, d_maps, d_scr, d_y0, d_y, nullptr);
    if (rc) return rc;
    cudaMemcpyAsync(y_out, d_y, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream);
    return ok(ctx, cudaStreamSynchronize(ctx->stream), "affine_compose sync") ? PINT_OK : PINT_E_CUDA;
}

int pint_scalar_sweep(pint_ctx* ctx, int mode, int64_t N, int64_t M, const double* nodes,
                      int64_t node_stride, const double* weights, const double* values,
                      const double* a, const double* b, int64_t ab_stride, double y0,
                      double* lambdas, double* y_out, long long* extrapolations) {
    if (!ctx || M < 1 || N < 0 || !y_out) return PINT_E_INVALID;
    const int64_t nsets = node_stride ? N : 1, nab = ab_stride ? N : 1;
    const size_t b_nodes = align256(sizeof(double) * M * nsets), b_vals = align256(sizeof(double) * M * N);
    const size_t b_ab = align256(sizeof(double) * nab);
    const size_t total = 2 * b_nodes + b_vals + 2 * b_ab + align256(sizeof(double) * N) + 1024;
    char* d = static_cast<char*>(pint_scratch(ctx, 2, total));
    if (!d) return PINT_E_CUDA;
    Carve cv{d};
    double* d_x = cv.take<double>(M * nsets);
    double* d_w = cv.take<double>(M * nsets);
    double* d_v = cv.take<double>(M * N);
    double* d_a = cv.take<double>(nab);
    double* d_b = cv.take<double>(nab);
    double* d_lam = cv.take<double>(N);
    double* d_y = cv.take<double>(1);
    auto* d_ext = cv.take<long long>(1);
    cudaMemcpyAsync(d_x, nodes, sizeof(double) * M * nsets, cudaMemcpyHostToDevice, ctx->stream);
    cudaMemcpyAsync(d_w, weights, sizeof(double) * M * nsets, cudaMemcpyHostToDevice, ctx->stream);
    cudaMemcpyAsync(d_v, values, sizeof(double) * M * N, cudaMemcpyHostToDevice, ctx->stream);
    cudaMemcpyAsync(d_a, a, sizeof(double) * nab, cudaMemcpyHostToDevice, ctx->stream);
    cudaMemcpyAsync(d_b, b, sizeof(double) * nab, cudaMemcpyHostToDevice, ctx->stream);
    int rc = launch_scalar_sweep(ctx, mode, N, M, d_x, node_stride ? M : 0, d_w, d_v, d_a, d_b,
                                 ab_stride ? 1 : 0, y0, d_lam, d_y, d_ext);
    if (rc) return rc;
    long long ext = 0;
    cudaMemcpyAsync(y_out, d_y, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream);
    cudaMemcpyAsync(&ext, d_ext, sizeof ext, cudaMemcpyDeviceToHost, ctx->stream);
    if (lambdas) cudaMemcpyAsync(lambdas, d_lam, sizeof(double) * N, cudaMemcpyDeviceToHost, ctx->stream);
    if (!ok(ctx, cudaStreamSynchronize(ctx->stream), "scalar_sweep sync")) return PINT_E_CUDA;
    if (extrapolations) *extrapolations = ext;
    return PINT_OK;
}

// ---- wave problem (make_wave_linear_problem, pde_problems.cpp:142-172) --------------------------

namespace {
// Upload D2 and the per-slice leapfrog tables; enforces the closure's native-step rule
// (pde_problems.cpp:155-157) and integrate_slice's integrality check.
int wave_upload(pint_ctx* ctx, int64_t d, const double* D2, double dt_native, const std::vector<pint_slice>& sl,
                int slot, double** d_D2, int64_t** d_steps, double** d_h) {
    for (const auto& s : sl) {
        if (std::fabs(s.dt - dt_native) > 1e-9 * dt_native)
            return pint_set_error(ctx, PINT_E_BAD_GRID, "wave: leapfrog runs only at the native step dt = 8/M^2");
        if (const int rc = check_integral(ctx, s.t_end - s.t_begin, s.dt)) return rc;
    }
    const int64_t N = static_cast<int64_t>(sl.size());
    const size_t b_d2 = align256(sizeof(double) * d * d), b_st = align256(sizeof(int64_t) * N);
    const size_t b_h = align256(sizeof(double) * N);
    char* h = static_cast<char*>(pinned(b_d2 + b_st + b_h));
    char* dev = static_cast<char*>(pint_scratch(ctx, slot, b_d2 + b_st + b_h));
    if (!h || !dev) return pint_set_error(ctx, PINT_E_CUDA, "wave: staging allocation failed");
    std::memcpy(h, D2, sizeof(double) * d * d);
    for (int64_t j = 0; j < N; ++j) {
        reinterpret_cast<int64_t*>(h + b_d2)[j] = sl[j].steps;
        reinterpret_cast<double*>(h + b_d2 + b_st)[j] = sl[j].dt;
    }
    if (!ok(ctx, cudaMemcpyAsync(dev, h, b_d2 + b_st + b_h, cudaMemcpyHostToDevice, ctx->stream), "H2D wave"))
        return PINT_E_CUDA;
    // the pinned staging buffer is reused by the next call: make this copy complete first
    if (!ok(ctx, cudaStreamSynchronize(ctx->stream), "H2D wave sync")) return PINT_E_CUDA;
    *d_D2 = reinterpret_cast<double*>(dev);
    *d_steps = reinterpret_cast<int64_t*>(dev + b_d2);
    *d_h = reinterpret_cast<double*>(dev + b_d2 + b_st);
    return PINT_OK;
}
}  // namespace

int pint_wave_maps(pint_ctx* ctx, int64_t d, const double* D2, double dt_native, const pint_slice* slices,
                   int64_t N, double dt_nominal, double* G, double* c) {
    if (!ctx || d < 1 || !D2 || !slices || N < 1) return PINT_E_INVALID;
    std::vector<pint_slice> sl;
    closure_slices(slices, N, dt_nominal, sl);
    double *d_D2, *d_h;
    int64_t* d_steps;
    if (const int rc = wave_upload(ctx, d, D2, dt_native, sl, 0, &d_D2, &d_steps, &d_h)) return rc;
    const int64_t n = 2 * d, ldm = pint_affine_ldm(n);
    double* d_maps = static_cast<double*>(pint_scratch(ctx, 2, sizeof(double) * n * ldm * N));
    if (!d_maps) return PINT_E_CUDA;
    if (const int rc = launch_wave_build(ctx, d, N, d_D2, d_steps, d_h, d_maps)) return rc;
    std::vector<double> host(static_cast<size_t>(n * ldm * N));
    cudaMemcpyAsync(host.data(), d_maps, sizeof(double) * host.size(), cudaMemcpyDeviceToHost, ctx->stream);
    if (!ok(ctx, cudaStreamSynchronize(ctx->stream), "wave_maps sync")) return PINT_E_CUDA;
    for (int64_t j = 0; j < N; ++j)
        for (int64_t i = 0; i < n; ++i) {
            const double* row = host.data() + (j * n + i) * ldm;
            if (G) std::memcpy(G + (j * n + i) * n, row, sizeof(double) * n);
            if (c) c[j * n + i] = row[n];
        }
    return PINT_OK;
}

int pint_wave_integrate(pint_ctx* ctx, int64_t d, const double* D2, double dt_native, const pint_slice* slice,
                        double dt_nominal, int64_t K, double* y) {
    if (!ctx || d < 1 || !D2 || !slice || K < 0) return PINT_E_INVALID;
    std::vector<pint_slice> sl;
    closure_slices(slice, 1, dt_nominal, sl);
    double *d_D2, *d_h;
    int64_t* d_steps;
    if (const int rc = wave_upload(ctx, d, D2, dt_native, sl, 0, &d_D2, &d_steps, &d_h)) return rc;
    if (K == 0) return PINT_OK;
    double* d_y = static_cast<double*>(pint_scratch(ctx, 2, sizeof(double) * 2 * d * K));
    if (!d_y) return PINT_E_CUDA;
    cudaMemcpyAsync(d_y, y, sizeof(double) * 2 * d * K, cudaMemcpyHostToDevice, ctx->stream);
    if (const int rc = launch_wave_integrate(ctx, d, K, d_D2, d_steps, d_h, d_y)) return rc;
    cudaMemcpyAsync(y, d_y, sizeof(double) * 2 * d * K, cudaMemcpyDeviceToHost, ctx->stream);
    return ok(ctx, cudaStreamSynchronize(ctx->stream), "wave_integrate sync") ? PINT_OK : PINT_E_CUDA;
}

int pint_run_wave(pint_ctx* ctx, int64_t d, const double* D2, double dt_native, double T, int64_t N,
                  double dt_nominal, int compose_mode, const double* y0, double* y_out, double* per_slice_seconds,
                  pint_report* report) {
    if (!ctx || d < 1 || !D2 || !y0 || !y_out || N < 1) return PINT_E_INVALID;
    HostTimer wall;
    const long long launches0 = ctx->launches;
    std::vector<pint_slice> sl(static_cast<size_t>(N));
    if (pint_decompose(0.0, T, N, dt_nominal, sl.data()) != PINT_OK)
        return pint_set_error(ctx, PINT_E_BAD_GRID, "decompose: need N >= 1, T > t0, dt > 0");
    closure_slices(sl.data(), N, dt_nominal, sl);
    cudaEventRecord(ctx->ev0, ctx->stream);
    double *d_D2, *d_h;
    int64_t* d_steps;
    if (const int rc = wave_upload(ctx, d, D2, dt_native, sl, 0, &d_D2, &d_steps, &d_h)) return rc;
    const int64_t n = 2 * d, ldm = pint_affine_ldm(n);
    const size_t map_elems = static_cast<size_t>(n * ldm);
    const size_t b_scr = compose_mode == PINT_COMPOSE_TREE ? align256(sizeof(double) * map_elems * ((N + 1) / 2)) : 0;
    char* dv = static_cast<char*>(pint_scratch(ctx, 2, align256(sizeof(double) * map_elems * N) + b_scr +
                                                        2 * align256(sizeof(double) * n) + 512));
    if (!dv) return PINT_E_CUDA;
    Carve cv{dv};
    double* d_maps = cv.take<double>(map_elems * N);
    double* d_scr = b_scr ? cv.take<double>(map_elems * ((N + 1) / 2)) : nullptr;
    double* d_y0 = cv.take<double>(n);
    double* d_y = cv.take<double>(n);
    cudaMemcpyAsync(d_y0, y0, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream);
    int rc = launch_wave_build(ctx, d, N, d_D2, d_steps, d_h, d_maps);
    if (rc) return rc;
    cudaEventRecord(ctx->evc, ctx->stream);
    if (compose_mode == PINT_COMPOSE_TREE) rc = launch_affine_tree(ctx, n, N, d_maps, d_scr, d_y0, d_y, nullptr);
    else rc = launch_affine_chain(ctx, n, N, d_maps, d_y0, d_y);
    if (rc) return rc;
    cudaEventRecord(ctx->ev1, ctx->stream);
    cudaMemcpyAsync(y_out, d_y, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream);
    if (!ok(ctx, cudaStreamSynchronize(ctx->stream), "run_wave sync")) return PINT_E_CUDA;
    float ms = 0.f, cms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
    cudaEventElapsedTime(&cms, ctx->evc, ctx->ev1);
    if (per_slice_seconds) {  // uniform slices: the build's device time split evenly
        for (int64_t j = 0; j < N; ++j) per_slice_seconds[j] = (ms - cms) * 1e-3 / static_cast<double>(N);
    }
    if (report) {
        report->message_count = N - 1;
        report->bytes_communicated = (N - 1) * n * static_cast<int64_t>(sizeof(double));
        report->extrapolation_count = 0;
        report->device_ms = ms;
        report->traj_steps = 0;
        for (const auto& s : sl) report->traj_steps += s.steps * (n + 1);
        report->gpu_launches = ctx->launches - launches0;
        report->h2d_bytes = static_cast<int64_t>(sizeof(double) * (d * d + n) + 16 * N);
        report->d2h_bytes = static_cast<int64_t>(sizeof(double) * n);
        report->compose_ms = cms;
        report->total_ms = wall.ms();
    }
    return PINT_OK;
}

int pint_bary_weights(pint_ctx* ctx, int kind, int64_t M, const double* nodes, double* w) {
    if (!ctx || M < 1 || !nodes || !w) return PINT_E_INVALID;
    char* d = static_cast<char*>(pint_scratch(ctx, 2, 2 * align256(sizeof(double) * M)));
    if (!d) return PINT_E_CUDA;
    Carve cv{d};
    double* d_x = cv.take<double>(M);
    double* d_w = cv.take<double>(M);
    cudaMemcpyAsync(d_x, nodes, sizeof(double) * M, cudaMemcpyHostToDevice, ctx->stream);
    if (const int rc = launch_bary_weights(ctx, kind, M, d_x, d_w)) return rc;
    cudaMemcpyAsync(w, d_w, sizeof(double) * M, cudaMemcpyDeviceToHost, ctx->stream);
    if (!ok(ctx, cudaStreamSynchronize(ctx->stream), "bary_weights sync")) return PINT_E_CUDA;
    pint_fail fr;
    if (const int rc = pint_fail_read(ctx, &fr)) return rc;
    if (fr.index >= 0) return pint_set_error(ctx, PINT_E_DUPLICATE_NODES, "barycentric_weights: repeated node");
    return PINT_OK;
}

}  // extern "C"
