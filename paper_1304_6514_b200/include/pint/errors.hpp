// pint-b200 drop-in: exception taxonomy of the reference (errors.hpp:9-43). Every C-ABI status
// code (include/pint_cuda.h) maps back to one of these in host/pint_host.cpp.
#pragma once

#include <cstddef>
#include <stdexcept>
#include <string>

namespace pint {

#define PINT_B200_ERROR(Name) \
    struct Name : std::runtime_error { using std::runtime_error::runtime_error; }

PINT_B200_ERROR(NoRealRoot);           // backward-Euler root crossed the blow-up
PINT_B200_ERROR(SingularSystem);       // zero pivot in a linear solve
PINT_B200_ERROR(BadGrid);              // inconsistent grid parameters
PINT_B200_ERROR(NonIntegerStepCount);  // slice width is not a whole number of steps
PINT_B200_ERROR(DuplicateNodes);       // repeated interpolation node
PINT_B200_ERROR(RankDeficient);        // least-squares design without full rank
#undef PINT_B200_ERROR

// The lowest failing task of a parallel launch (exec_harness.hpp:88-99 semantics).
struct TaskFailure : std::runtime_error {
    std::size_t task_index;
    TaskFailure(std::size_t index, const std::string& what)
        : std::runtime_error("task " + std::to_string(index) + ": " + what), task_index(index) {}
};

}  // namespace pint
