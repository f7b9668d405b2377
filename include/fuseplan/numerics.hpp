// fuseplan-b200 — generalized advantage estimation (host reference forms).
//
// Source-compatible with proj/include/fuseplan/numerics.hpp:11-26. The GPU
// post-processing kernel (csrc/kernels/postprocess.cu) computes the same
// recursion in fp32 with a reverse warp scan; these fp64 forms are the host
// API and the conventions it must follow (T rewards, T+1 values with an
// explicit bootstrap, gamma and lambda in [0, 1]).
#pragma once

#include <vector>

namespace fuseplan {

struct GaeInputs {
  std::vector<double> rewards;  // r_0 .. r_{T-1}
  std::vector<double> values;   // V_0 .. V_T (V_T is the bootstrap)
  double gamma = 0.99;
  double lam = 0.95;
};

/// A_t = delta_t + gamma*lam*A_{t+1}, delta_t = r_t + gamma V_{t+1} - V_t.
std::vector<double> gae_recursive(const GaeInputs& in);

/// Same quantity as a dense upper-triangular product (A = U delta), summed
/// left to right per row; an independent association order for cross-checks.
std::vector<double> gae_matrix(const GaeInputs& in);

}  // namespace fuseplan
