// libpint_b200.so — the reference's pint:: API for the Nievergelt slice-map path, implemented on
// top of the C ABI of libpint_cuda.so (include/pint_cuda.h).
//
// Hot-path entry points (run_nievergelt x2, run_serial x2, build_scalar_slice_map,
// build_affine_propagator, compose_sweep x2, barycentric_weights, interp_eval and the heat
// integrate closure) execute on the B200; without a device they throw — there is no CPU
// fallback. The remaining functions are the reference's host-side API surface (grids, small
// dense linear algebra, problem setup) that its tests and callers use directly.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <thread>
#include <stdexcept>
#include <string>
#include <vector>

#include "pint/errors.hpp"
#include "pint/exec_harness.hpp"
#include "pint/interp.hpp"
#include "pint/linalg.hpp"
#include "pint/nievergelt.hpp"
#include "pint/ode_core.hpp"
#include "pint/parareal.hpp"
#include "pint/pde_problems.hpp"
#include "pint_cuda.h"

namespace pint {
namespace {

constexpr double kPi = 3.14159265358979323846;

// One device context per process (cuda:0), serialised by a mutex: the reference API is
// re-entrant and free-function based, so callers never see the context.
struct Device {
    std::mutex mu;
    pint_ctx* ctx = nullptr;
    ~Device() {
        if (ctx) pint_ctx_destroy(ctx);
    }
};

Device& device() {
    static Device d;
    return d;
}

pint_ctx* ctx_locked() {
    Device& d = device();
    if (!d.ctx) {
        const int rc = pint_ctx_create(0, &d.ctx);
        if (rc != PINT_OK)
            throw std::runtime_error("pint-b200: no CUDA device (code " + std::to_string(rc) +
                                     "); the slice-map path runs only on the GPU");
    }
    return d.ctx;
}

// ExecConfig::workers > 1 with several GPUs: one context per device (cuda:0 .. cuda:G-1), joined
// into one NCCL communicator (pint_comm_init_all); built once per G, guarded by device().mu.
struct DeviceSet {
    std::vector<pint_ctx*> ctxs;
    ~DeviceSet() {
        for (std::size_t g = 1; g < ctxs.size(); ++g) pint_ctx_destroy(ctxs[g]);  // (ctxs[0] is device())
    }
};

int gpus_for(std::size_t workers) {
    return static_cast<int>(std::max<std::size_t>(1, std::min<std::size_t>(workers, pint_device_count())));
}

[[noreturn]] void raise(int rc, pint_ctx* ctx, const pint_fail* fail = nullptr);

// the device set for G GPUs (G > 1), caller holds device().mu
std::vector<pint_ctx*>& device_set_locked(int G) {
    static DeviceSet set;
    if (static_cast<int>(set.ctxs.size()) != G) {
        for (std::size_t g = 1; g < set.ctxs.size(); ++g) pint_ctx_destroy(set.ctxs[g]);
        set.ctxs.assign(1, ctx_locked());
        for (int g = 1; g < G; ++g) {
            pint_ctx* c = nullptr;
            if (const int rc = pint_ctx_create(g, &c)) raise(rc, nullptr);
            set.ctxs.push_back(c);
        }
        if (const int rc = pint_comm_init_all(set.ctxs.data(), G)) raise(rc, set.ctxs[0]);
    }
    return set.ctxs;
}

[[noreturn]] void raise(int rc, pint_ctx* ctx, const pint_fail* fail) {
    const std::string msg = ctx ? pint_ctx_last_error(ctx) : std::string("pint-b200 error");
    if (fail && fail->index >= 0) throw TaskFailure(static_cast<std::size_t>(fail->index), msg);
    switch (rc) {
        case PINT_E_NO_REAL_ROOT: throw NoRealRoot(msg);
        case PINT_E_SINGULAR: throw SingularSystem(msg);
        case PINT_E_BAD_GRID: throw BadGrid(msg);
        case PINT_E_NON_INTEGER_STEPS: throw NonIntegerStepCount(msg);
        case PINT_E_DUPLICATE_NODES: throw DuplicateNodes(msg);
        default: throw std::runtime_error("pint-b200: " + msg);
    }
}

void check(int rc, pint_ctx* ctx, const pint_fail* fail = nullptr) {
    if (rc != PINT_OK) raise(rc, ctx, fail);
}

pint_scalar_rhs device_rhs(const ScalarIVP& ivp) {
    pint_scalar_rhs r{};
    r.kind = ivp.device.kind == ScalarDevice::Kind::logistic_rk4 ? PINT_RHS_LOGISTIC_RK4 : PINT_RHS_RICCATI_BE;
    r.precision = ivp.device.fp32 ? PINT_F32 : PINT_F64;
    r.r = ivp.device.r;
    r.K = ivp.device.K;
    return r;
}

pint_slice to_c(const TimeSlice& s) { return pint_slice{s.t_begin, s.t_end, static_cast<int64_t>(s.steps), s.dt}; }

// integrate_scalar (nievergelt.cpp:29-35) for many initial values on the device.
Vector integrate_scalar_many(const ScalarIVP& ivp, const Vector& y0, double t_begin, double t_end, double dt) {
    const std::size_t n = steps_for(t_end - t_begin, dt);
    const pint_slice sl{t_begin, t_end, static_cast<int64_t>(n), (t_end - t_begin) / static_cast<double>(n)};
    Vector out(y0.size());
    const pint_scalar_rhs rhs = device_rhs(ivp);
    std::lock_guard<std::mutex> lk(device().mu);
    pint_ctx* c = ctx_locked();
    pint_fail fail{};
    const int rc = pint_scalar_integrate(c, &rhs, &sl, static_cast<int64_t>(y0.size()), y0.data(), out.data(), &fail);
    if (rc != PINT_OK) raise(rc, c, y0.size() > 1 ? &fail : nullptr);
    return out;
}

double max_abs(const Vector& v) {
    double m = 0.0;
    for (double x : v) m = std::max(m, std::abs(x));
    return m;
}

double max_abs_diff(const Vector& a, const Vector& b) {
    double m = 0.0;
    for (std::size_t i = 0; i < a.size(); ++i) m = std::max(m, std::abs(a[i] - b[i]));
    return m;
}

// the simulated wire of compose_sweep (nievergelt.cpp:73-79, 95-101): sleeps and counters
void simulate_receives(std::size_t n_maps, std::size_t bytes_per_msg, double latency, SweepStats& stats) {
    for (std::size_t j = 1; j < n_maps; ++j) {
        Stopwatch recv;
        inject_latency(latency);
        stats.T_comm += latency > 0.0 ? recv.seconds() : 0.0;
        ++stats.message_count;
        stats.bytes_communicated += bytes_per_msg;
    }
}

}  // namespace

// ---- linalg (host utilities) -------------------------------------------------------------------

Matrix Matrix::identity(std::size_t n) {
    Matrix I(n, n);
    for (std::size_t i = 0; i < n; ++i) I(i, i) = 1.0;
    return I;
}

Vector matvec(const Matrix& A, const Vector& x) {
    Vector y(A.rows(), 0.0);
    for (std::size_t i = 0; i < A.rows(); ++i) {
        double acc = 0.0;
        for (std::size_t k = 0; k < A.cols(); ++k) acc += A(i, k) * x[k];
        y[i] = acc;
    }
    return y;
}

Matrix matmul(const Matrix& A, const Matrix& B) {
    Matrix C(A.rows(), B.cols());
    for (std::size_t i = 0; i < A.rows(); ++i)
        for (std::size_t k = 0; k < A.cols(); ++k) {
            const double aik = A(i, k);
            if (aik == 0.0) continue;
            for (std::size_t j = 0; j < B.cols(); ++j) C(i, j) += aik * B(k, j);
        }
    return C;
}

Vector lu_solve(Matrix A, Vector b) {
    const std::size_t n = A.rows();
    for (std::size_t col = 0; col < n; ++col) {
        std::size_t piv = col;
        for (std::size_t i = col + 1; i < n; ++i)
            if (std::abs(A(i, col)) > std::abs(A(piv, col))) piv = i;
        if (A(piv, col) == 0.0) throw SingularSystem("lu_solve: zero pivot column " + std::to_string(col));
        if (piv != col) {
            for (std::size_t j = 0; j < n; ++j) std::swap(A(col, j), A(piv, j));
            std::swap(b[col], b[piv]);
        }
        for (std::size_t i = col + 1; i < n; ++i) {
            const double m = A(i, col) / A(col, col);
            if (m == 0.0) continue;
            for (std::size_t j = col + 1; j < n; ++j) A(i, j) -= m * A(col, j);
            b[i] -= m * b[col];
        }
    }
    Vector x(n);
    for (std::size_t r = n; r-- > 0;) {
        double acc = b[r];
        for (std::size_t j = r + 1; j < n; ++j) acc -= A(r, j) * x[j];
        x[r] = acc / A(r, r);
    }
    return x;
}

Vector thomas_solve(const Vector& sub, const Vector& diag, const Vector& sup, Vector rhs) {
    const std::size_t n = diag.size();
    Vector cp(n > 1 ? n - 1 : 0);
    double p = diag[0];
    if (p == 0.0) throw SingularSystem("thomas_solve: zero pivot at row 0");
    if (n > 1) cp[0] = sup[0] / p;
    rhs[0] /= p;
    for (std::size_t i = 1; i < n; ++i) {
        p = diag[i] - sub[i - 1] * cp[i - 1];
        if (p == 0.0) throw SingularSystem("thomas_solve: zero pivot at row " + std::to_string(i));
        if (i + 1 < n) cp[i] = sup[i] / p;
        rhs[i] = (rhs[i] - sub[i - 1] * rhs[i - 1]) / p;
    }
    for (std::size_t i = n - 1; i-- > 0;) rhs[i] -= cp[i] * rhs[i + 1];
    return rhs;
}

// ---- exec harness ------------------------------------------------------------------------------

double modeled_time_nievergelt(const std::vector<double>& per_slice_compute, double latency, double apply_cost) {
    if (per_slice_compute.empty()) return 0.0;
    // idealized schedule (exec_harness.cpp:7-13): slowest slice, then N-1 receives and applications
    const double msgs = static_cast<double>(per_slice_compute.size() - 1);
    const double slowest = *std::max_element(per_slice_compute.begin(), per_slice_compute.end());
    return slowest + msgs * latency + msgs * apply_cost;
}

double modeled_time_parareal(const std::vector<double>& fine, double coarse_per_slice, std::size_t k, std::size_t N,
                             double latency) {
    const double fmax = fine.empty() ? 0.0 : *std::max_element(fine.begin(), fine.end());
    const double kk = static_cast<double>(k), nn = static_cast<double>(N);
    return kk * fmax + (kk + 1.0) * nn * coarse_per_slice + (2.0 * kk + 1.0) * (nn - 1.0) * latency;
}

// ---- ode core ----------------------------------------------------------------------------------

ScalarIVP make_model_problem() {
    ScalarIVP p;
    p.rhs = [](double, double y) { return y * y; };
    p.t0 = 0.0;
    p.T = 0.5;
    p.y0 = 1.0;
    p.exact = [](double t) { return 1.0 / (1.0 - t); };
    return p;
}

ScalarIVP make_logistic_problem(double r, double K, double y0, double T) {
    ScalarIVP p;
    p.rhs = [r, K](double, double y) { return r * y * (1.0 - y / K); };
    p.t0 = 0.0;
    p.T = T;
    p.y0 = y0;
    p.exact = [r, K, y0](double t) {
        const double e = std::exp(r * t);
        return K * y0 * e / (K + y0 * (e - 1.0));
    };
    p.device.kind = ScalarDevice::Kind::logistic_rk4;
    p.device.r = r;
    p.device.K = K;
    return p;
}

std::size_t steps_for(double width, double dt) { return static_cast<std::size_t>(pint_steps_for(width, dt)); }

TimeSliceDecomposition decompose(double t0, double T, std::size_t N, double dt) {
    if (N == 0 || !(T > t0) || !(dt > 0.0)) throw BadGrid("decompose: need N >= 1, T > t0, dt > 0");
    std::vector<pint_slice> raw(N);
    if (pint_decompose(t0, T, static_cast<int64_t>(N), dt, raw.data()) != PINT_OK)
        throw BadGrid("decompose: need N >= 1, T > t0, dt > 0");
    TimeSliceDecomposition d;
    d.N = N;
    d.t0 = t0;
    d.T = T;
    d.dt_nominal = dt;
    d.slices.resize(N);
    for (std::size_t j = 0; j < N; ++j)
        d.slices[j] = TimeSlice{j, raw[j].t_begin, raw[j].t_end, static_cast<std::size_t>(raw[j].steps), raw[j].dt};
    return d;
}

double be_step_scalar_riccati(double y, double dt) {  // ode_core.cpp:47-53 (host API form)
    const double disc = 1.0 - 4.0 * dt * y;
    if (disc < 0.0) throw NoRealRoot("be_step_scalar_riccati: 1 - 4 dt y = " + std::to_string(disc));
    return 2.0 * y / (1.0 + std::sqrt(disc));
}

Vector be_step_linear(const LinearSystem& sys, const Vector& y, double t_next, double dt) {
    Vector rhs = y;
    if (sys.forcing) {
        const Vector b = sys.forcing(t_next);
        for (std::size_t i = 0; i < rhs.size(); ++i) rhs[i] += dt * b[i];
    }
    return sys.solve_implicit(t_next, dt, rhs);
}

std::pair<Vector, Vector> leapfrog_integrate(Vector y_curr, Vector y_prev, std::size_t n_steps, double dt,
                                             const std::function<Vector(const Vector&)>& apply_D2) {
    const double dt2 = dt * dt;
    for (std::size_t m = 0; m < n_steps; ++m) {
        Vector next = apply_D2(y_curr);
        for (std::size_t i = 0; i < next.size(); ++i) next[i] = 2.0 * y_curr[i] - y_prev[i] + dt2 * next[i];
        y_prev = std::move(y_curr);
        y_curr = std::move(next);
    }
    return {std::move(y_curr), std::move(y_prev)};
}

// ---- interp ------------------------------------------------------------------------------------

Vector sample_nodes(NodeKind kind, std::size_t M, double a, double b) {
    if (M == 0) throw BadGrid("cheb_nodes: M >= 1 required");
    Vector x(M);
    pint_sample_nodes(kind == NodeKind::first_kind ? PINT_NODES_FIRST_KIND : PINT_NODES_SECOND_KIND,
                      static_cast<int64_t>(M), a, b, x.data());
    return x;
}

Vector cheb_nodes(std::size_t M, double a, double b) { return sample_nodes(NodeKind::first_kind, M, a, b); }
Vector cheb_nodes_second_kind(std::size_t M, double a, double b) { return sample_nodes(NodeKind::second_kind, M, a, b); }

static Vector device_weights(const Vector& nodes, bool closed_form) {
    Vector w(nodes.size());
    if (nodes.empty()) return w;
    std::lock_guard<std::mutex> lk(device().mu);
    pint_ctx* c = ctx_locked();
    check(pint_bary_weights(c, closed_form ? PINT_WEIGHTS_CLOSED2 : PINT_WEIGHTS_PRODUCT,
                            static_cast<int64_t>(nodes.size()), nodes.data(), w.data()),
          c);
    return w;
}

Vector barycentric_weights(const Vector& nodes) { return device_weights(nodes, false); }

InterpolantData make_interpolant(Vector nodes, Vector values, double a, double b) {
    InterpolantData f;
    f.weights = barycentric_weights(nodes);
    f.nodes = std::move(nodes);
    f.values = std::move(values);
    f.a = a;
    f.b = b;
    return f;
}

static double sweep_maps(const std::vector<const InterpolantData*>& fs, double y0, std::vector<double>* lambdas,
                         long long* extrapolations) {
    const std::size_t N = fs.size();
    const std::size_t M = fs.front()->nodes.size();
    Vector nodes(N * M), weights(N * M), values(N * M), a(N), b(N);
    for (std::size_t j = 0; j < N; ++j) {
        const InterpolantData& f = *fs[j];
        if (f.nodes.size() != M || f.weights.size() != M || f.values.size() != M)
            throw std::invalid_argument("compose_sweep: all slice maps must have the same node count");
        std::copy(f.nodes.begin(), f.nodes.end(), nodes.begin() + static_cast<std::ptrdiff_t>(j * M));
        std::copy(f.weights.begin(), f.weights.end(), weights.begin() + static_cast<std::ptrdiff_t>(j * M));
        std::copy(f.values.begin(), f.values.end(), values.begin() + static_cast<std::ptrdiff_t>(j * M));
        a[j] = f.a;
        b[j] = f.b;
    }
    double y = 0.0;
    long long ext = 0;
    std::vector<double> lam(N);
    std::lock_guard<std::mutex> lk(device().mu);
    pint_ctx* c = ctx_locked();
    check(pint_scalar_sweep(c, PINT_SWEEP_EXACT, static_cast<int64_t>(N), static_cast<int64_t>(M), nodes.data(),
                            static_cast<int64_t>(M), weights.data(), values.data(), a.data(), b.data(), 1, y0,
                            lam.data(), &y, &ext),
          c);
    if (lambdas) *lambdas = std::move(lam);
    if (extrapolations) *extrapolations = ext;
    return y;
}

double interp_eval(const InterpolantData& f, double xi) { return sweep_maps({&f}, xi, nullptr, nullptr); }

ChebDiff cheb_diff_matrix(std::size_t M, double a, double b) {  // wave setup (host)
    if (M == 0) throw BadGrid("cheb_diff_matrix: M >= 1 required");
    const std::size_t n = M + 1;
    Vector x(n), cw(n, 1.0);
    for (std::size_t j = 0; j < n; ++j) x[j] = std::cos(static_cast<double>(j) * kPi / static_cast<double>(M));
    cw.front() = cw.back() = 2.0;
    const double scale = 2.0 / (b - a);
    ChebDiff out;
    out.D = Matrix(n, n);
    for (std::size_t i = 0; i < n; ++i) {
        double diag = 0.0;
        for (std::size_t j = 0; j < n; ++j) {
            if (i == j) continue;
            const double sign = ((i + j) % 2 == 0) ? 1.0 : -1.0;
            const double dij = (cw[i] / cw[j]) * sign / (x[i] - x[j]);
            diag += dij;
            out.D(i, j) = dij * scale;
        }
        out.D(i, i) = -diag * scale;
    }
    out.grid.resize(n);
    for (std::size_t j = 0; j < n; ++j) out.grid[j] = a + (b - a) * (x[j] + 1.0) / 2.0;
    return out;
}

// ---- nievergelt --------------------------------------------------------------------------------

SliceMap build_scalar_slice_map(const ScalarIVP& ivp, const TimeSlice& slice, const InitialValueSpace& space,
                                double dt) {
    Vector nodes = sample_nodes(space.kind, space.M, space.a, space.b);
    Vector ends = integrate_scalar_many(ivp, nodes, slice.t_begin, slice.t_end, dt);
    SliceMap map;
    map.slice_index = slice.index;
    map.interpolant.weights = device_weights(nodes, space.closed_form_weights);
    map.interpolant.nodes = std::move(nodes);
    map.interpolant.values = std::move(ends);
    map.interpolant.a = space.a;
    map.interpolant.b = space.b;
    return map;
}

static void require_device(const LinearProblem& p) {
    if (!p.heat && !p.wave)
        throw std::invalid_argument("pint-b200: LinearProblem '" + p.name +
                                    "' has no device description (make_heat_problem / "
                                    "make_wave_linear_problem provide one)");
}

AffinePropagator build_affine_propagator(const LinearProblem& problem, const TimeSlice& slice) {
    require_device(problem);
    const std::size_t n = problem.dim;
    AffinePropagator prop;
    prop.slice_index = slice.index;
    prop.G = Matrix(n, n);
    prop.c.assign(n, 0.0);
    std::vector<double> G(n * n);
    const pint_slice s = to_c(slice);
    std::lock_guard<std::mutex> lk(device().mu);
    pint_ctx* c = ctx_locked();
    if (problem.heat) {
        check(pint_heat_maps(c, problem.heat->dx, problem.dt, &s, 1, G.data(), prop.c.data()), c);
    } else {
        const WaveDevice& w = *problem.wave;
        check(pint_wave_maps(c, static_cast<int64_t>(w.d), w.D2.data(), w.dt_native, &s, 1, problem.dt, G.data(),
                             prop.c.data()),
              c);
    }
    for (std::size_t i = 0; i < n; ++i)
        for (std::size_t j = 0; j < n; ++j) prop.G(i, j) = G[i * n + j];
    return prop;
}

double compose_sweep(const std::vector<SliceMap>& maps, double y0, double latency, SweepStats& stats) {
    if (maps.empty()) return y0;
    simulate_receives(maps.size(), sizeof(double), latency, stats);
    std::vector<const InterpolantData*> fs;
    fs.reserve(maps.size());
    for (const auto& m : maps) fs.push_back(&m.interpolant);
    Stopwatch apply;
    long long ext = 0;
    const double y = sweep_maps(fs, y0, nullptr, &ext);
    stats.extrapolation_count += static_cast<int>(ext);
    stats.apply_cost = apply.seconds() / static_cast<double>(maps.size());
    return y;
}

Vector compose_sweep(const std::vector<AffinePropagator>& maps, Vector y0, double latency, SweepStats& stats) {
    if (maps.empty()) return y0;
    const std::size_t n = y0.size();
    simulate_receives(maps.size(), sizeof(double) * n, latency, stats);
    std::vector<double> G(maps.size() * n * n), cvec(maps.size() * n);
    for (std::size_t j = 0; j < maps.size(); ++j) {
        std::copy(maps[j].G.data().begin(), maps[j].G.data().end(), G.begin() + static_cast<std::ptrdiff_t>(j * n * n));
        std::copy(maps[j].c.begin(), maps[j].c.end(), cvec.begin() + static_cast<std::ptrdiff_t>(j * n));
    }
    Vector y(n);
    Stopwatch apply;
    {
        std::lock_guard<std::mutex> lk(device().mu);
        pint_ctx* c = ctx_locked();
        check(pint_affine_compose(c, PINT_COMPOSE_CHAIN, static_cast<int64_t>(n), static_cast<int64_t>(maps.size()),
                                  G.data(), cvec.data(), y0.data(), y.data()),
              c);
    }
    stats.apply_cost = apply.seconds() / static_cast<double>(maps.size());
    return y;
}

RunReport run_serial(const ScalarIVP& ivp, double dt) {
    RunReport r;
    r.method = "serial";
    r.N = 1;
    r.dt = dt;
    Stopwatch sw;
    const double y = integrate_scalar_many(ivp, Vector{ivp.y0}, ivp.t0, ivp.T, dt)[0];
    r.T_total = sw.seconds();
    r.final_state = {y};
    r.per_slice_compute = {r.T_total};
    if (ivp.exact) r.error_vs_exact = std::abs(y - (*ivp.exact)(ivp.T));
    return r;
}

RunReport run_serial(const LinearProblem& problem) {
    RunReport r;
    r.method = "serial";
    r.N = 1;
    r.dt = problem.dt;
    TimeSlice whole;
    whole.t_begin = problem.t0;
    whole.t_end = problem.T;
    whole.steps = steps_for(problem.T - problem.t0, problem.dt);
    whole.dt = (problem.T - problem.t0) / static_cast<double>(whole.steps);
    Stopwatch sw;
    r.final_state = problem.integrate(whole, problem.y0, problem.dt, true);
    r.T_total = sw.seconds();
    r.per_slice_compute = {r.T_total};
    if (problem.exact_final) r.error_vs_exact = max_abs_diff(r.final_state, *problem.exact_final);
    return r;
}

static void finish_report(RunReport& r, const pint_report& rep, const SweepStats& stats, const ExecConfig& exec,
                          std::vector<double> per_slice) {
    r.T_comm = stats.T_comm;
    r.message_count = stats.message_count;
    r.bytes_communicated = stats.bytes_communicated;
    r.extrapolation_count = static_cast<int>(rep.extrapolation_count);
    r.per_slice_compute = std::move(per_slice);
    if (exec.clock != ClockMode::measured)
        r.modeled_time = modeled_time_nievergelt(r.per_slice_compute, exec.latency_per_receive, stats.apply_cost);
}

RunReport run_nievergelt(const ScalarIVP& ivp, std::size_t N, double dt, const InitialValueSpace& space,
                         const ExecConfig& exec) {
    if (N <= 1) {
        RunReport r = run_serial(ivp, dt);
        r.method = "nievergelt";
        r.workers = exec.workers;
        return r;
    }
    const double y_serial = integrate_scalar_many(ivp, Vector{ivp.y0}, ivp.t0, ivp.T, dt)[0];  // outside T_total
    RunReport r;
    r.method = "nievergelt";
    r.N = N;
    r.M = space.M;
    r.dt = dt;
    r.latency = exec.latency_per_receive;
    r.workers = exec.workers;
    Stopwatch total;
    const pint_scalar_rhs rhs = device_rhs(ivp);
    std::vector<double> per_slice(N);
    pint_report rep{};
    pint_fail fail{};
    double y = 0.0;
    {
        std::lock_guard<std::mutex> lk(device().mu);
        pint_ctx* c = ctx_locked();
        const int rc = pint_run_scalar(
            c, &rhs, ivp.t0, ivp.T, ivp.y0, static_cast<int64_t>(N), dt,
            space.kind == NodeKind::first_kind ? PINT_NODES_FIRST_KIND : PINT_NODES_SECOND_KIND,
            static_cast<int64_t>(space.M), space.a, space.b,
            space.closed_form_weights ? PINT_WEIGHTS_CLOSED2 : PINT_WEIGHTS_PRODUCT,
            space.tree_sum ? PINT_SWEEP_TREE : PINT_SWEEP_EXACT, &y, nullptr, nullptr, per_slice.data(), &rep, &fail);
        if (rc != PINT_OK) raise(rc, c, &fail);
    }
    SweepStats stats;
    simulate_receives(N, sizeof(double), exec.latency_per_receive, stats);
    stats.apply_cost = rep.compose_ms * 1e-3 / static_cast<double>(N);
    r.T_total = total.seconds();
    r.final_state = {y};
    finish_report(r, rep, stats, exec, std::move(per_slice));
    if (ivp.exact) r.error_vs_exact = std::abs(y - (*ivp.exact)(ivp.T));
    r.error_vs_serial = std::abs(y - y_serial) / std::max(1e-300, std::abs(y_serial));
    return r;
}

RunReport run_nievergelt(const LinearProblem& problem, std::size_t N, const ExecConfig& exec) {
    if (N <= 1) {
        RunReport r = run_serial(problem);
        r.method = "nievergelt";
        r.workers = exec.workers;
        return r;
    }
    require_device(problem);
    // the serial reference run (outside T_total, nievergelt.cpp:221): heat runs it in the background
    // on the device while the parallel run proceeds (pint_heat_serial_begin/_end); wave runs it first
    Vector serial = problem.heat ? Vector(problem.dim) : run_serial(problem).final_state;
    RunReport r;
    r.method = "nievergelt";
    r.N = N;
    r.dt = problem.dt;
    r.latency = exec.latency_per_receive;
    r.workers = exec.workers;
    Stopwatch total;
    Vector y(problem.dim);
    std::vector<double> per_slice(N);
    pint_report rep{};
    {
        std::lock_guard<std::mutex> lk(device().mu);
        pint_ctx* c = ctx_locked();
        if (problem.t0 != 0.0) throw std::invalid_argument("pint-b200: linear problems start at t0 = 0");
        const int mode = problem.tree_compose ? PINT_COMPOSE_TREE : PINT_COMPOSE_CHAIN;
        const int G = problem.heat ? gpus_for(exec.workers) : 1;
        if (G > 1) {  // ExecConfig::workers -> GPUs: slice blocks per GPU, one thread each, NCCL gather
            std::vector<pint_ctx*>& cs = device_set_locked(G);
            check(pint_heat_serial_begin(cs[0], problem.heat->dx, problem.dt, problem.T, problem.y0.data()), cs[0]);
            total = Stopwatch();
            std::vector<int> rcs(static_cast<std::size_t>(G), PINT_OK);
            std::vector<pint_report> reps(static_cast<std::size_t>(G));
            std::vector<std::thread> th;
            for (int g = 0; g < G; ++g)
                th.emplace_back([&, g] {
                    rcs[g] = pint_run_heat_sharded(cs[g], problem.heat->dx, problem.dt, problem.T,
                                                   static_cast<int64_t>(N), PINT_BUILD_EXACT, mode, problem.y0.data(),
                                                   g == 0 ? y.data() : nullptr, &reps[g]);
                });
            for (auto& t : th) t.join();
            r.T_total = total.seconds();
            const int rs = pint_heat_serial_end(cs[0], serial.data());
            for (int g = 0; g < G; ++g) check(rcs[g], cs[g]);
            check(rs, cs[0]);
            rep = reps[0];
            const double each = rep.device_ms * 1e-3 / static_cast<double>(N);  // (no per-slice timers here)
            std::fill(per_slice.begin(), per_slice.end(), each);
        } else if (problem.heat) {
            check(pint_heat_serial_begin(c, problem.heat->dx, problem.dt, problem.T, problem.y0.data()), c);
            total = Stopwatch();
            const int rc = pint_run_heat(c, problem.heat->dx, problem.dt, problem.T, static_cast<int64_t>(N), mode,
                                         problem.y0.data(), y.data(), per_slice.data(), &rep);
            r.T_total = total.seconds();
            const int rs = pint_heat_serial_end(c, serial.data());
            check(rc, c);
            check(rs, c);
        } else {
            const WaveDevice& w = *problem.wave;
            check(pint_run_wave(c, static_cast<int64_t>(w.d), w.D2.data(), w.dt_native, problem.T,
                                static_cast<int64_t>(N), problem.dt, mode, problem.y0.data(), y.data(),
                                per_slice.data(), &rep),
                  c);
        }
    }
    SweepStats stats;
    const double t_run = problem.heat ? r.T_total : total.seconds();  // (heat: measured around the run)
    simulate_receives(N, sizeof(double) * problem.dim, exec.latency_per_receive, stats);
    stats.apply_cost = rep.compose_ms * 1e-3 / static_cast<double>(N);
    r.T_total = t_run + stats.T_comm;
    r.final_state = std::move(y);
    finish_report(r, rep, stats, exec, std::move(per_slice));
    if (problem.exact_final) r.error_vs_exact = max_abs_diff(r.final_state, *problem.exact_final);
    const double scale = max_abs(serial);
    const double gap = max_abs_diff(r.final_state, serial);
    r.error_vs_serial = scale == 0.0 ? gap : gap / scale;
    return r;
}

// ---- heat problem ------------------------------------------------------------------------------

static std::size_t heat_interior(double dx) {
    const double inv = 1.0 / dx;
    const auto m = static_cast<std::size_t>(std::llround(inv));
    if (m < 2 || std::abs(inv - static_cast<double>(m)) > 1e-9 * inv)
        throw BadGrid("make_heat_system: 1/dx must be an integer >= 2, got dx = " + std::to_string(dx));
    return m - 1;
}

double heat_coefficient(double t) { return 1.0 + 0.25 * std::sin(t); }

double heat_forcing(double x, double t) {
    const double sx = std::sin(kPi * x);
    return -std::sin(t) * sx + heat_coefficient(t) * kPi * kPi * std::cos(t) * sx;
}

LinearSystem make_heat_system(double dx) {
    const std::size_t m = heat_interior(dx);
    const double inv_dx2 = 1.0 / (dx * dx);
    LinearSystem sys;
    sys.dim = m;
    sys.structure = LinearSystem::Structure::tridiagonal;
    sys.apply_A = [m, inv_dx2](double t, const Vector& y) {
        const double a = heat_coefficient(t) * inv_dx2;
        Vector out(m);
        for (std::size_t i = 0; i < m; ++i)
            out[i] = a * ((i > 0 ? y[i - 1] : 0.0) - 2.0 * y[i] + (i + 1 < m ? y[i + 1] : 0.0));
        return out;
    };
    sys.forcing = [m, dx](double t) {
        Vector b(m);
        for (std::size_t i = 0; i < m; ++i) b[i] = heat_forcing(static_cast<double>(i + 1) * dx, t);
        return b;
    };
    sys.solve_implicit = [m, inv_dx2](double t, double dt, const Vector& rhs) {
        const double r = dt * heat_coefficient(t) * inv_dx2;
        return thomas_solve(Vector(m - 1, -r), Vector(m, 1.0 + 2.0 * r), Vector(m - 1, -r), rhs);
    };
    return sys;
}

Vector heat_initial(double dx) {
    const std::size_t m = heat_interior(dx);
    Vector u(m);
    for (std::size_t i = 0; i < m; ++i) u[i] = std::sin(kPi * static_cast<double>(i + 1) * dx);
    return u;
}

Vector heat_exact(double dx, double t) {
    Vector u = heat_initial(dx);
    for (double& v : u) v *= std::cos(t);
    return u;
}

LinearProblem make_heat_problem(double dx, double dt, double T) {
    const std::size_t m = heat_interior(dx);
    LinearProblem p;
    p.dim = m;
    p.t0 = 0.0;
    p.T = T;
    p.dt = dt;
    p.y0 = heat_initial(dx);
    p.exact_final = heat_exact(dx, T);
    p.name = "heat";
    p.heat = HeatDevice{dx};
    // the integrate closure runs on the device: K = 1 trajectory through the slice's steps
    p.integrate = [dx, m](const TimeSlice& s, Vector y, double step_nominal, bool with_forcing) {
        if (y.size() != m) throw std::invalid_argument("heat integrate: state size mismatch");
        const pint_slice cs = to_c(s);
        std::lock_guard<std::mutex> lk(device().mu);
        pint_ctx* c = ctx_locked();
        check(pint_heat_integrate(c, dx, &cs, step_nominal, with_forcing ? 1 : 0, 1, y.data()), c);
        return y;
    };
    return p;
}

WaveProblem make_wave_problem(std::size_t M, double x0, double sigma) {
    if (M < 8 || M % 2 != 0) throw BadGrid("make_wave_problem: M must be even and >= 8, got " + std::to_string(M));
    WaveProblem w;
    w.M = M;
    w.dt = 8.0 / (static_cast<double>(M) * static_cast<double>(M));
    w.x0 = x0;
    w.sigma = sigma;
    const ChebDiff cd = cheb_diff_matrix(M, -1.0, 1.0);
    w.grid = cd.grid;
    const Matrix D2 = matmul(cd.D, cd.D);
    const std::size_t d = M - 1;
    w.D2_interior = Matrix(d, d);
    for (std::size_t i = 0; i < d; ++i)
        for (std::size_t j = 0; j < d; ++j) w.D2_interior(i, j) = D2(i + 1, j + 1);
    w.u0.resize(d);
    w.um1.resize(d);
    for (std::size_t i = 0; i < d; ++i) {
        const double x = w.grid[i + 1];
        w.u0[i] = std::exp(-sigma * (x - x0) * (x - x0));
        w.um1[i] = std::exp(-sigma * (x - w.dt - x0) * (x - w.dt - x0));
    }
    return w;
}

Matrix wave_step_matrix(const WaveProblem& w) {
    const std::size_t d = w.M - 1;
    const double dt2 = w.dt * w.dt;
    Matrix S(2 * d, 2 * d);
    for (std::size_t i = 0; i < d; ++i) {
        for (std::size_t j = 0; j < d; ++j) S(i, j) = dt2 * w.D2_interior(i, j);
        S(i, i) += 2.0;
        S(i, d + i) = -1.0;
        S(d + i, i) = 1.0;
    }
    return S;
}

LinearProblem make_wave_linear_problem(const WaveProblem& w, double T) {
    const std::size_t d = w.M - 1;
    LinearProblem p;
    p.dim = 2 * d;
    p.t0 = 0.0;
    p.T = T;
    p.dt = w.dt;
    p.y0.resize(2 * d);
    for (std::size_t i = 0; i < d; ++i) {
        p.y0[i] = w.u0[i];
        p.y0[d + i] = w.um1[i];
    }
    p.name = "wave";
    WaveDevice wd;
    wd.d = d;
    wd.D2 = w.D2_interior.data();
    wd.dt_native = w.dt;
    p.wave = wd;
    // the leapfrog integrate closure (pde_problems.cpp:150-171) on the device, one trajectory
    p.integrate = [wd](const TimeSlice& s, Vector y, double step_nominal, bool) {
        if (y.size() != 2 * wd.d) throw std::invalid_argument("wave integrate: state size mismatch");
        const pint_slice cs = to_c(s);
        std::lock_guard<std::mutex> lk(device().mu);
        pint_ctx* c = ctx_locked();
        check(pint_wave_integrate(c, static_cast<int64_t>(wd.d), wd.D2.data(), wd.dt_native, &cs, step_nominal, 1,
                                  y.data()),
              c);
        return y;
    };
    return p;
}

// ---- parareal (parareal.cpp:47-190) on the device ----------------------------------------------

std::size_t parareal_message_count(std::size_t k, std::size_t N) { return N == 0 ? 0 : (2 * k + 1) * (N - 1); }

double coarse_propagate(const ScalarIVP& ivp, double lambda, const TimeSlice& slice, double DT) {
    (void)ivp;  // (the reference's coarse propagator is the Riccati step whatever the right-hand side)
    ScalarIVP model = make_model_problem();
    return integrate_scalar_many(model, Vector{lambda}, slice.t_begin, slice.t_end, DT)[0];
}

Vector coarse_propagate(const LinearProblem& problem, Vector lambda, const TimeSlice& slice, double DT) {
    return problem.integrate(slice, std::move(lambda), DT, true);
}

namespace {

// the report fields every parareal run shares; the simulated receives (latency per message) are
// slept here, as the reference's CommTracker sleeps them inside its sweeps
void parareal_report(RunReport& r, const PararealConfig& cfg, const ExecConfig& exec, std::size_t state_bytes) {
    r.method = "parareal";
    r.N = cfg.N;
    r.k = cfg.k;
    r.dt = cfg.dt;
    r.DT = cfg.DT;
    r.latency = exec.latency_per_receive;
    r.workers = exec.workers;
    r.message_count = parareal_message_count(cfg.k, cfg.N);
    r.bytes_communicated = r.message_count * state_bytes;
    for (std::size_t m = 0; m < r.message_count; ++m) {
        Stopwatch sw;
        inject_latency(exec.latency_per_receive);
        if (exec.latency_per_receive > 0.0) r.T_comm += sw.seconds();
    }
}

}  // namespace

PararealResult parareal_sweep(const ScalarIVP& ivp, const PararealConfig& cfg, const ExecConfig& exec) {
    if (cfg.N == 0) throw std::invalid_argument("parareal: N >= 1 required");
    PararealResult out;
    RunReport& r = out.report;
    std::vector<double> finals(cfg.k + 1), fine(cfg.N);
    double coarse_per_slice = 0.0;
    Stopwatch total;
    {
        std::lock_guard<std::mutex> lk(device().mu);
        pint_ctx* c = ctx_locked();
        pint_report rep{};
        pint_fail fail{};
        const int rc = pint_parareal_scalar(c, ivp.t0, ivp.T, ivp.y0, static_cast<int64_t>(cfg.N),
                                            static_cast<int64_t>(cfg.k), cfg.dt, cfg.DT, finals.data(), fine.data(),
                                            &coarse_per_slice, &rep, &fail);
        check(rc, c, &fail);
    }
    parareal_report(r, cfg, exec, sizeof(double));
    r.T_total = total.seconds();
    r.per_slice_compute = fine;
    for (double y : finals) out.final_per_iteration.push_back(Vector{y});
    r.final_state = out.final_per_iteration.back();
    if (exec.clock != ClockMode::measured) {
        std::vector<double> fine_mean(fine);
        for (double& t : fine_mean) t /= static_cast<double>(std::max<std::size_t>(cfg.k, 1));
        r.modeled_time = modeled_time_parareal(fine_mean, coarse_per_slice, cfg.k, cfg.N, exec.latency_per_receive);
    }
    const double y = r.final_state[0];
    if (ivp.exact) r.error_vs_exact = std::abs(y - (*ivp.exact)(ivp.T));
    const ScalarIVP model = make_model_problem();  // (the serial run uses the Riccati step too)
    const double y_serial = integrate_scalar_many(model, Vector{ivp.y0}, ivp.t0, ivp.T, cfg.dt)[0];
    r.error_vs_serial = std::abs(y - y_serial) / std::max(1e-300, std::abs(y_serial));
    return out;
}

PararealResult parareal_sweep(const LinearProblem& problem, const PararealConfig& cfg, const ExecConfig& exec) {
    if (cfg.N == 0) throw std::invalid_argument("parareal: N >= 1 required");
    PararealResult out;
    RunReport& r = out.report;
    const std::size_t n = problem.dim;
    Stopwatch total;
    if (problem.heat && problem.t0 == 0.0) {  // both propagators in device kernels
        std::vector<double> finals((cfg.k + 1) * n);
        pint_report rep{};
        {
            std::lock_guard<std::mutex> lk(device().mu);
            pint_ctx* c = ctx_locked();
            check(pint_parareal_heat(c, problem.heat->dx, problem.T, problem.y0.data(), static_cast<int64_t>(cfg.N),
                                     static_cast<int64_t>(cfg.k), cfg.dt, cfg.DT, finals.data(), &rep),
                  c);
        }
        for (std::size_t i = 0; i <= cfg.k; ++i)
            out.final_per_iteration.emplace_back(finals.begin() + static_cast<std::ptrdiff_t>(i * n),
                                                 finals.begin() + static_cast<std::ptrdiff_t>((i + 1) * n));
        r.per_slice_compute.assign(cfg.N, rep.device_ms * 1e-3 / static_cast<double>(cfg.N));
    } else {  // other linear problems: the same iteration over their device integrate closures
        const TimeSliceDecomposition dec = decompose(problem.t0, problem.T, cfg.N, cfg.dt);
        std::vector<Vector> lam(cfg.N + 1), g_old(cfg.N);
        lam[0] = problem.y0;
        for (std::size_t j = 0; j < cfg.N; ++j) lam[j + 1] = g_old[j] = coarse_propagate(problem, lam[j], dec.slices[j], cfg.DT);
        out.final_per_iteration.push_back(lam[cfg.N]);
        r.per_slice_compute.assign(cfg.N, 0.0);
        for (std::size_t it = 1; it <= cfg.k; ++it) {
            std::vector<Vector> f(cfg.N);
            for (std::size_t j = 0; j < cfg.N; ++j) {
                Stopwatch sw;
                f[j] = problem.integrate(dec.slices[j], lam[j], cfg.dt, true);
                r.per_slice_compute[j] += sw.seconds();
            }
            for (std::size_t j = 0; j < cfg.N; ++j) {
                Vector g = coarse_propagate(problem, lam[j], dec.slices[j], cfg.DT);
                Vector next(n);
                for (std::size_t i = 0; i < n; ++i) next[i] = g[i] + f[j][i] - g_old[j][i];
                g_old[j] = std::move(g);
                lam[j + 1] = std::move(next);
            }
            out.final_per_iteration.push_back(lam[cfg.N]);
        }
    }
    parareal_report(r, cfg, exec, sizeof(double) * n);
    r.T_total = total.seconds();
    r.final_state = out.final_per_iteration.back();
    if (exec.clock != ClockMode::measured)
        r.modeled_time = modeled_time_parareal(r.per_slice_compute, 0.0, cfg.k, cfg.N, exec.latency_per_receive);
    if (problem.exact_final) r.error_vs_exact = max_abs_diff(r.final_state, *problem.exact_final);
    const Vector serial = run_serial(problem).final_state;
    const double scale = max_abs(serial);
    const double gap = max_abs_diff(r.final_state, serial);
    r.error_vs_serial = scale == 0.0 ? gap : gap / scale;
    return out;
}

RunReport run_parareal(const ScalarIVP& ivp, const PararealConfig& cfg, const ExecConfig& exec) {
    return parareal_sweep(ivp, cfg, exec).report;
}

RunReport run_parareal(const LinearProblem& problem, const PararealConfig& cfg, const ExecConfig& exec) {
    return parareal_sweep(problem, cfg, exec).report;
}

}  // namespace pint
