// pint-b200 drop-in: the heat and wave problems (reference pde_problems.hpp:13-45) with their
// device descriptors; both integrate closures and slice maps run on the B200.
#pragma once

#include <cstddef>

#include "pint/linalg.hpp"
#include "pint/nievergelt.hpp"
#include "pint/ode_core.hpp"

namespace pint {

double heat_coefficient(double t);
double heat_forcing(double x, double t);
LinearSystem make_heat_system(double dx);
Vector heat_initial(double dx);
Vector heat_exact(double dx, double t);
LinearProblem make_heat_problem(double dx, double dt, double T);

struct WaveProblem {
    std::size_t M = 0;
    double dt = 0.0;
    double x0 = 0.0, sigma = 200.0;
    Vector grid;
    Matrix D2_interior;
    Vector u0, um1;
};
WaveProblem make_wave_problem(std::size_t M, double x0 = 0.0, double sigma = 200.0);
Matrix wave_step_matrix(const WaveProblem& w);
LinearProblem make_wave_linear_problem(const WaveProblem& w, double T);

}  // namespace pint
