// fuseplan-b200 — error taxonomy of the experience-collection path.
//
// Source-compatible with the reference's proj/include/fuseplan/errors.hpp:9-18
// so that callers (and the reference's own unit tests) catch the same types.
// Across the C ABI (include/fp_sched.h, include/fp_engine.h) these map to
// status codes: ConfigError / std::invalid_argument -> 2, InfeasibleError -> 3,
// anything else (incl. CUDA failures) -> 4, mirroring the reference CLI's exit
// codes (proj/tools/fuseplan_main.cpp:32-35).
#pragma once

#include <stdexcept>

namespace fuseplan {

/// Bad user input: unreadable length files, malformed config values.
struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

/// Well-formed input with no feasible execution, e.g. a KV pool that cannot
/// hold the reservation of even one sample.
struct InfeasibleError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

}  // namespace fuseplan
