// Test infrastructure: the UNMODIFIED reference's parareal_sweep (parareal.cpp) final_per_iteration
// for the configurations tests/golden/make_parareal_golden.py asks for, one line per iterate:
//   scalar N k dt DT          -> "it value"
//   heat dx T N k dt DT       -> "it v0 v1 ... v(n-1)"
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "pint/parareal.hpp"
#include "pint/pde_problems.hpp"

int main(int argc, char** argv) {
    using namespace pint;
    if (argc >= 6 && std::strcmp(argv[1], "scalar") == 0) {
        PararealConfig cfg;
        cfg.N = std::strtoull(argv[2], nullptr, 10);
        cfg.k = std::strtoull(argv[3], nullptr, 10);
        cfg.dt = std::strtod(argv[4], nullptr);
        cfg.DT = std::strtod(argv[5], nullptr);
        const auto r = parareal_sweep(make_model_problem(), cfg, ExecConfig{});
        for (std::size_t i = 0; i < r.final_per_iteration.size(); ++i)
            std::printf("%zu %.17g\n", i, r.final_per_iteration[i][0]);
        std::printf("err %.17g %.17g\n", r.report.error_vs_exact.value(), r.report.error_vs_serial.value());
        return 0;
    }
    if (argc >= 8 && std::strcmp(argv[1], "heat") == 0) {
        const double dx = std::strtod(argv[2], nullptr), T = std::strtod(argv[3], nullptr);
        PararealConfig cfg;
        cfg.N = std::strtoull(argv[4], nullptr, 10);
        cfg.k = std::strtoull(argv[5], nullptr, 10);
        cfg.dt = std::strtod(argv[6], nullptr);
        cfg.DT = std::strtod(argv[7], nullptr);
        const auto r = parareal_sweep(make_heat_problem(dx, cfg.dt, T), cfg, ExecConfig{});
        for (std::size_t i = 0; i < r.final_per_iteration.size(); ++i) {
            std::printf("%zu", i);
            for (double v : r.final_per_iteration[i]) std::printf(" %.17g", v);
            std::printf("\n");
        }
        return 0;
    }
    std::fprintf(stderr, "usage: parareal_golden scalar N k dt DT | heat dx T N k dt DT\n");
    return 2;
}
