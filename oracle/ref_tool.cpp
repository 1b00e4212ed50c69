// ref_tool — a driver linked against the UNMODIFIED reference library (oracle/_ref/libpint_ref.a,
// compiled from /root/reference/proj/src by oracle/Makefile). Test and baseline infrastructure
// only: it never links the B200 product code.
//
//   ref_tool golden <outdir>      dump golden vectors from the reference's own functions
//   ref_tool bench-heat  ...      time pint::run_nievergelt(make_heat_problem(...)) (CPU baseline)
//   ref_tool bench-scalar ...     time pint::run_nievergelt(make_model_problem(), ...)
//   ref_tool bench-serial --dt h  time pint::run_serial(make_model_problem(), h) (one core)
//   ref_tool fit <fixture>        pint::fit_params(load_observations(fixture), 0.5) as JSON
//
// Every vector below is produced by calling the reference API exactly as its own tests do
// (tests/test_nievergelt.cpp, tests/test_ode_core.cpp, tests/acceptance.cpp).
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <string>
#include <thread>
#include <vector>

#include "pint/cost_model.hpp"
#include "pint/exec_harness.hpp"
#include "pint/interp.hpp"
#include "pint/linalg.hpp"
#include "pint/nievergelt.hpp"
#include "pint/ode_core.hpp"
#include "pint/pde_problems.hpp"

using namespace pint;

namespace {

struct Dump {
    std::string dir;
    std::string manifest = "{\n";
    bool first = true;

    void entry(const std::string& name, const std::string& dtype, const std::vector<std::size_t>& shape,
               const void* data, std::size_t bytes) {
        const std::string file = name + "." + dtype;
        std::ofstream f(dir + "/" + file, std::ios::binary);
        f.write(static_cast<const char*>(data), static_cast<std::streamsize>(bytes));
        std::string sh = "[";
        for (std::size_t i = 0; i < shape.size(); ++i) sh += (i ? "," : "") + std::to_string(shape[i]);
        sh += "]";
        manifest += std::string(first ? "" : ",\n") + "  \"" + name + "\": {\"dtype\": \"" + dtype +
                    "\", \"shape\": " + sh + "}";
        first = false;
    }
    void f64(const std::string& name, const std::vector<double>& v, std::vector<std::size_t> shape = {}) {
        if (shape.empty()) shape = {v.size()};
        entry(name, "f64", shape, v.data(), v.size() * sizeof(double));
    }
    void i64(const std::string& name, const std::vector<std::int64_t>& v) {
        entry(name, "i64", {v.size()}, v.data(), v.size() * sizeof(std::int64_t));
    }
    void scalar(const std::string& name, double x) { f64(name, std::vector<double>{x}); }
    void close() {
        manifest += "\n}\n";
        std::ofstream(dir + "/manifest.json") << manifest;
    }
};

std::vector<double> flatten(const Matrix& A) { return A.data(); }

void dump_decomposition(Dump& d, const std::string& tag, double t0, double T, std::size_t N, double dt) {
    const auto dec = decompose(t0, T, N, dt);
    std::vector<double> tb, te, h;
    std::vector<std::int64_t> steps;
    for (const auto& s : dec.slices) {
        tb.push_back(s.t_begin);
        te.push_back(s.t_end);
        h.push_back(s.dt);
        steps.push_back(static_cast<std::int64_t>(s.steps));
    }
    d.f64(tag + "_t_begin", tb);
    d.f64(tag + "_t_end", te);
    d.f64(tag + "_dt", h);
    d.i64(tag + "_steps", steps);
}

// Scalar run: the reference RunReport fields plus every slice's sampled endpoints (via the
// public build_scalar_slice_map, nievergelt.cpp:41-51) and the boundary values the sweep visits
// (interp_eval chain, nievergelt.cpp:68-88).
void dump_scalar_run(Dump& d, const std::string& tag, std::size_t N, double dt, std::size_t M,
                     double a, double b, bool endpoints) {
    const ScalarIVP ivp = make_model_problem();
    InitialValueSpace space;
    space.M = M;
    space.a = a;
    space.b = b;
    const RunReport r = run_nievergelt(ivp, N, dt, space, ExecConfig{});
    d.scalar(tag + "_final", r.final_state.at(0));
    d.scalar(tag + "_error_vs_exact", r.error_vs_exact.value());
    d.scalar(tag + "_error_vs_serial", r.error_vs_serial.value_or(0.0));
    d.scalar(tag + "_message_count", static_cast<double>(r.message_count));
    d.scalar(tag + "_bytes", static_cast<double>(r.bytes_communicated));
    d.scalar(tag + "_extrapolation_count", static_cast<double>(r.extrapolation_count));
    if (!endpoints) return;
    const auto dec = decompose(ivp.t0, ivp.T, N, dt);
    std::vector<double> ends, lambdas;
    double y = ivp.y0;
    for (std::size_t j = 0; j < N; ++j) {
        const SliceMap map = build_scalar_slice_map(ivp, dec.slices[j], space, dt);
        ends.insert(ends.end(), map.interpolant.values.begin(), map.interpolant.values.end());
        y = interp_eval(map.interpolant, y);
        lambdas.push_back(y);
    }
    d.f64(tag + "_endpoints", ends, {N, M});
    d.f64(tag + "_lambdas", lambdas);
}

int cmd_golden(const std::string& dir) {
    Dump d{dir};

    // ---- ode_core: steps_for / decompose / Riccati step (test_ode_core.cpp:11-44)
    const double sf_w[] = {0.125, 0.125, 0.5, 0.3, 0.05, 10.0 / 64, 0.5 / 7, 1.0 / 3.0};
    const double sf_dt[] = {0.01, 1e-4, 1e-4, 0.1, 0.1, 1e-3, 1e-4, 1e-2};
    std::vector<double> w, dts;
    std::vector<std::int64_t> st;
    for (std::size_t i = 0; i < sizeof(sf_w) / sizeof(double); ++i) {
        w.push_back(sf_w[i]);
        dts.push_back(sf_dt[i]);
        st.push_back(static_cast<std::int64_t>(steps_for(sf_w[i], sf_dt[i])));
    }
    d.f64("steps_for_width", w);
    d.f64("steps_for_dt", dts);
    d.i64("steps_for_steps", st);
    dump_decomposition(d, "dec_4_001", 0.0, 0.5, 4, 0.01);
    dump_decomposition(d, "dec_64_1em4", 0.0, 0.5, 64, 1e-4);
    dump_decomposition(d, "dec_7_1em3", 0.0, 0.5, 7, 1e-3);
    dump_decomposition(d, "dec_3_1em2", 0.0, 0.5, 3, 1e-2);
    dump_decomposition(d, "dec_heat_256", 0.0, 10.0, 256, 10.0 / (256.0 * 256.0));

    std::vector<double> ry, rdt, rz;
    for (double y : {1.0, 1.7, 0.0, 0.3, 2.0, 1.999}) {
        for (double h : {0.01, 0.005, 1e-4, 9.8892405063291138e-05, 0.12}) {
            if (1.0 - 4.0 * h * y < 0.0) continue;
            ry.push_back(y);
            rdt.push_back(h);
            rz.push_back(be_step_scalar_riccati(y, h));
        }
    }
    d.f64("riccati_y", ry);
    d.f64("riccati_dt", rdt);
    d.f64("riccati_z", rz);

    // ---- interp: nodes and product-form weights (interp.cpp:21-55)
    for (std::size_t M : {1, 2, 5, 6, 7, 33, 64, 512}) {
        const Vector x2 = cheb_nodes_second_kind(M, 0.0, 2.0);
        d.f64("nodes2_" + std::to_string(M), x2);
        if (M > 1) d.f64("weights2_" + std::to_string(M), barycentric_weights(x2));
        const Vector x1 = cheb_nodes(M, 0.0, 2.0);
        d.f64("nodes1_" + std::to_string(M), x1);
    }
    {   // interp_eval on a fixed table, incl. node snaps and extrapolation
        const Vector x = cheb_nodes_second_kind(33, 0.0, 2.0);
        Vector v(x.size());
        for (std::size_t i = 0; i < x.size(); ++i) v[i] = std::exp(0.3 * x[i]) - 0.25 * x[i] * x[i];
        const InterpolantData f = make_interpolant(x, v, 0.0, 2.0);
        std::vector<double> xi, out;
        for (int k = -5; k <= 45; ++k) xi.push_back(0.05 * k);
        xi.push_back(x[3]);
        xi.push_back(x[17] + 1e-16);
        xi.push_back(x[32]);
        for (double q : xi) out.push_back(interp_eval(f, q));
        d.f64("interp33_values", v);
        d.f64("interp33_xi", xi);
        d.f64("interp33_out", out);
    }

    // ---- scalar Nievergelt runs (test_nievergelt.cpp:31-74, acceptance.cpp:45-77)
    dump_scalar_run(d, "sc_N4_M5_1em4", 4, 1e-4, 5, 0.0, 2.0, true);
    dump_scalar_run(d, "sc_N4_M6_1em4", 4, 1e-4, 6, 0.0, 2.0, true);
    dump_scalar_run(d, "sc_N4_M7_1em4", 4, 1e-4, 7, 0.0, 2.0, true);
    dump_scalar_run(d, "sc_N64_M6_1em4", 64, 1e-4, 6, 0.0, 2.0, true);
    dump_scalar_run(d, "sc_N8_M6_1em3", 8, 1e-3, 6, 0.0, 2.0, true);
    dump_scalar_run(d, "sc_N16_M33_1em3", 16, 1e-3, 33, 0.0, 2.0, true);
    dump_scalar_run(d, "sc_N64_M64_1em4", 64, 1e-4, 64, 0.0, 2.0, true);
    dump_scalar_run(d, "sc_N64_M512_1em4", 64, 1e-4, 512, 0.0, 2.0, false);
    dump_scalar_run(d, "sc_extrap_N4_M5_1em3", 4, 1e-3, 5, 0.0, 0.5, true);
    {   // acceptance criterion 1 grid (N=4): error_vs_exact per (dt, M)
        const double dtg[5] = {0.01, 0.005, 0.0025, 0.001, 0.0001};
        std::vector<double> errs;
        for (double h : dtg)
            for (std::size_t M : {3, 4, 5, 6, 7}) {
                InitialValueSpace space;
                space.M = M;
                errs.push_back(run_nievergelt(make_model_problem(), 4, h, space, ExecConfig{})
                                   .error_vs_exact.value());
            }
        d.f64("table1_errors", errs, {5, 5});
    }
    {
        const RunReport s = run_serial(make_model_problem(), 1e-4);
        d.scalar("serial_1em4_final", s.final_state[0]);
        d.scalar("serial_1em4_error", s.error_vs_exact.value());
        d.scalar("serial_1em2_final", run_serial(make_model_problem(), 1e-2).final_state[0]);
    }

    // ---- heat affine path (pde_problems.cpp:76-100, nievergelt.cpp:53-66, :213-265)
    {
        const auto heat = make_heat_problem(0.1, 0.005, 10.0);
        const auto dec = decompose(0.0, 10.0, 4, 0.005);
        std::vector<double> Gs, cs;
        for (std::size_t j = 0; j < 4; ++j) {
            const AffinePropagator p = build_affine_propagator(heat, dec.slices[j]);
            const auto g = flatten(p.G);
            Gs.insert(Gs.end(), g.begin(), g.end());
            cs.insert(cs.end(), p.c.begin(), p.c.end());
        }
        d.f64("heat9_G", Gs, {4, 9, 9});
        d.f64("heat9_c", cs, {4, 9});
        const RunReport serial = run_serial(heat);
        d.f64("heat9_serial_final", serial.final_state);
        d.scalar("heat9_serial_error", serial.error_vs_exact.value());
        const RunReport r4 = run_nievergelt(heat, 4, ExecConfig{});
        d.f64("heat9_N4_final", r4.final_state);
        d.scalar("heat9_N4_error_vs_serial", r4.error_vs_serial.value());
        d.scalar("heat9_N4_bytes", static_cast<double>(r4.bytes_communicated));
        Vector y(9);
        for (std::size_t i = 0; i < 9; ++i) y[i] = 0.1 * static_cast<double>(i) - 0.3;
        d.f64("heat9_direct_y", y);
        d.f64("heat9_direct_out", heat.integrate(dec.slices[1], y, heat.dt, true));
    }
    {   // n = 128 (config 2 shape), N = 16 slices of S = 32 steps
        const double dx = 1.0 / 129.0, dt = 10.0 / (16.0 * 32.0);
        const auto heat = make_heat_problem(dx, dt, 10.0);
        const auto dec = decompose(0.0, 10.0, 16, dt);
        const AffinePropagator p5 = build_affine_propagator(heat, dec.slices[5]);
        d.f64("heat128_slice5_G", flatten(p5.G), {128, 128});
        d.f64("heat128_slice5_c", p5.c);
        const RunReport r = run_nievergelt(heat, 16, ExecConfig{8});
        d.f64("heat128_N16_final", r.final_state);
        d.scalar("heat128_N16_error_vs_serial", r.error_vs_serial.value());
        d.scalar("heat128_N16_error_vs_exact", r.error_vs_exact.value());
        d.f64("heat128_serial_final", run_serial(heat).final_state);
    }

    // ---- wave affine path (pde_problems.cpp:102-172, leapfrog ode_core.cpp:65-77)
    {
        const WaveProblem w = make_wave_problem(16);
        const auto wave = make_wave_linear_problem(w, 16.0);
        d.f64("wave16_D2", flatten(w.D2_interior), {15, 15});
        d.scalar("wave16_dt", w.dt);
        d.f64("wave16_y0", wave.y0);
        const auto dec = decompose(0.0, 16.0, 4, wave.dt);
        const AffinePropagator p1 = build_affine_propagator(wave, dec.slices[1]);
        d.f64("wave16_slice1_G", flatten(p1.G), {30, 30});
        d.f64("wave16_slice1_c", p1.c);
        d.f64("wave16_N4_final", run_nievergelt(wave, 4, ExecConfig{}).final_state);
        d.f64("wave16_serial_final", run_serial(wave).final_state);
        const WaveProblem w40 = make_wave_problem(40);
        d.f64("wave40_D2", flatten(w40.D2_interior), {39, 39});
        d.f64("wave40_N8_final", run_nievergelt(make_wave_linear_problem(w40, 16.0), 8, ExecConfig{}).final_state);
    }

    // ---- linalg KATs (linalg.cpp:17-93)
    {
        const std::size_t n = 12;
        Vector sub(n - 1, -1.0), sup(n - 1, -1.3), diag(n), rhs(n);
        for (std::size_t i = 0; i < n; ++i) {
            diag[i] = 4.0 + 0.1 * static_cast<double>(i);
            rhs[i] = 1.0 / (1.0 + static_cast<double>(i));
        }
        d.f64("thomas12_x", thomas_solve(sub, diag, sup, rhs));
        Matrix A(5, 5);
        Vector x(5);
        for (std::size_t i = 0; i < 5; ++i) {
            x[i] = std::cos(0.3 * static_cast<double>(i));
            for (std::size_t j = 0; j < 5; ++j)
                A(i, j) = std::sin(1.0 + static_cast<double>(i * 5 + j)) * (j == 2 ? 0.0 : 1.0);
        }
        d.f64("linalg5_A", flatten(A), {5, 5});
        d.f64("linalg5_x", x);
        d.f64("linalg5_Ax", matvec(A, x));
        d.f64("linalg5_AA", flatten(matmul(A, A)), {5, 5});
    }
    d.close();
    std::printf("golden vectors written to %s\n", dir.c_str());
    return 0;
}

void write_f64(const std::string& path, const Vector& v) {
    std::ofstream f(path, std::ios::binary);
    f.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(v.size() * sizeof(double)));
}

double arg_d(std::map<std::string, std::string>& a, const char* k, double dflt) {
    return a.count(k) ? std::atof(a[k].c_str()) : dflt;
}

// Time the reference's heat path: make_heat_problem + run_nievergelt(problem, N, {workers}).
// With --sample-slices k < N the reference's own build_affine_propagator runs on the first k
// slices through parallel_map (the per-slice body of run_nievergelt, nievergelt.cpp:237-243)
// followed by its compose_sweep, so a bounded sample of a huge config stays in seconds.
int cmd_bench_heat(std::map<std::string, std::string> a) {
    const auto n = static_cast<std::size_t>(arg_d(a, "--n", 128));
    const auto N = static_cast<std::size_t>(arg_d(a, "--N", 256));
    const auto S = static_cast<std::size_t>(arg_d(a, "--S", 256));
    const double T = arg_d(a, "--T", 10.0);
    std::size_t workers = static_cast<std::size_t>(arg_d(a, "--workers", 0));
    if (workers == 0) workers = std::max(1u, std::thread::hardware_concurrency());
    const auto k = static_cast<std::size_t>(arg_d(a, "--sample-slices", static_cast<double>(N)));
    const int reps = static_cast<int>(arg_d(a, "--reps", 1));
    // --final-out <file>: the full final state of the last rep as raw little-endian f64 (golden)
    const std::string final_out = a.count("--final-out") ? a["--final-out"] : std::string();
    const double dx = 1.0 / static_cast<double>(n + 1);
    const double dt = T / static_cast<double>(N * S);
    const auto heat = make_heat_problem(dx, dt, T);
    std::printf("[");
    for (int rep = 0; rep < reps; ++rep) {
        const auto t0 = std::chrono::steady_clock::now();
        double final0 = 0.0;
        if (k >= N) {
            ExecConfig e;
            e.workers = workers;
            e.clock = ClockMode::measured;
            // run_nievergelt runs run_serial first (outside its own T_total); the wall clock
            // here is the reference's T_total only, matching what the reference reports.
            const RunReport r = run_nievergelt(heat, N, e);
            final0 = r.final_state[0];
            if (!final_out.empty()) write_f64(final_out, r.final_state);
            const double secs = r.T_total;
            std::printf("%s{\"seconds\": %.9g, \"slices\": %zu, \"traj_steps\": %.17g, \"final0\": %.17g}",
                        rep ? "," : "", secs, N, static_cast<double>(N * (n + 1) * S), final0);
        } else {
            const auto dec = decompose(0.0, T, N, dt);
            const auto maps = parallel_map<AffinePropagator>(
                k, workers, [&](std::size_t j) { return build_affine_propagator(heat, dec.slices[j]); });
            SweepStats stats;
            const Vector y = compose_sweep(maps, heat.y0, 0.0, stats);
            final0 = y[0];
            if (!final_out.empty()) write_f64(final_out, y);
            const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            std::printf("%s{\"seconds\": %.9g, \"slices\": %zu, \"traj_steps\": %.17g, \"final0\": %.17g}",
                        rep ? "," : "", secs, k, static_cast<double>(k * (n + 1) * S), final0);
        }
        std::fflush(stdout);
    }
    std::printf("]\n");
    std::fprintf(stderr, "workers=%zu\n", workers);
    return 0;
}

// Time the reference's scalar path (Riccati BE, barycentric maps, nievergelt.cpp:145-211).
int cmd_bench_scalar(std::map<std::string, std::string> a) {
    const auto N = static_cast<std::size_t>(arg_d(a, "--N", 64));
    const auto M = static_cast<std::size_t>(arg_d(a, "--M", 512));
    const auto S = static_cast<std::size_t>(arg_d(a, "--S", 79));
    std::size_t workers = static_cast<std::size_t>(arg_d(a, "--workers", 0));
    if (workers == 0) workers = std::max(1u, std::thread::hardware_concurrency());
    const int reps = static_cast<int>(arg_d(a, "--reps", 1));
    const double dt = 0.5 / static_cast<double>(N * S);
    InitialValueSpace space;
    space.M = M;
    std::printf("[");
    for (int rep = 0; rep < reps; ++rep) {
        ExecConfig e;
        e.workers = workers;
        e.clock = ClockMode::measured;
        const RunReport r = run_nievergelt(make_model_problem(), N, dt, space, e);
        std::printf("%s{\"seconds\": %.9g, \"traj_steps\": %.17g, \"final\": %.17g}", rep ? "," : "",
                    r.T_total, static_cast<double>(N * M * S), r.final_state[0]);
        std::fflush(stdout);
    }
    std::printf("]\n");
    return 0;
}

// The reference's serial scalar run (the CPU side of the cost model's ratio column).
int cmd_bench_serial(std::map<std::string, std::string> a) {
    const double dt = arg_d(a, "--dt", 6.103515625e-05);
    const int reps = static_cast<int>(arg_d(a, "--reps", 3));
    double best = 1e30, y = 0.0;
    for (int rep = 0; rep < reps; ++rep) {
        const auto t0 = std::chrono::steady_clock::now();
        const RunReport r = run_serial(make_model_problem(), dt);
        best = std::min(best, std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
        y = r.final_state[0];
    }
    std::printf("{\"seconds\": %.9g, \"final\": %.17g}\n", best, y);
    return 0;
}

// The reference's least-squares fit of (tau_F, tau_N, tau_K, tau_F_cpu) on a 5-column fixture.
int cmd_fit(const std::string& path) {
    const auto obs = load_observations(path);
    const FitResult f = fit_params(obs, 0.5);
    std::printf("{\"tau_F\": %.9g, \"tau_N\": %.9g, \"tau_K\": %.9g, \"tau_F_cpu\": %.9g, \"predicted\": [",
                f.params.tau_F, f.params.tau_N, f.params.tau_K, f.params.tau_F_cpu);
    for (std::size_t i = 0; i < f.predicted.size(); ++i) std::printf("%s%.9g", i ? ", " : "", f.predicted[i]);
    std::printf("], \"observed\": [");
    for (std::size_t i = 0; i < obs.size(); ++i) std::printf("%s%.9g", i ? ", " : "", obs[i].total_us);
    std::printf("]}\n");
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: ref_tool golden <dir> | bench-heat [--k v ...] | bench-scalar [...]\n");
        return 2;
    }
    const std::string cmd = argv[1];
    std::map<std::string, std::string> args;
    for (int i = 2; i + 1 < argc; i += 2) args[argv[i]] = argv[i + 1];
    try {
        if (cmd == "golden" && argc >= 3) return cmd_golden(argv[2]);
        if (cmd == "bench-heat") return cmd_bench_heat(args);
        if (cmd == "bench-scalar") return cmd_bench_scalar(args);
        if (cmd == "bench-serial") return cmd_bench_serial(args);
        if (cmd == "fit" && argc >= 3) return cmd_fit(argv[2]);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "ref_tool: %s\n", e.what());
        return 1;
    }
    std::fprintf(stderr, "ref_tool: unknown command %s\n", cmd.c_str());
    return 2;
}
