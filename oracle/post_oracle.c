/* ORACLE — test infrastructure only; never linked into the product path.
 *
 * CPU restatement (C, fp64) of the per-token experience post-processing that
 * the GPU kernel csrc/kernels/post.cu performs in fp32:
 *
 *   kl_t      = logp_actor_t - logp_ref_t                      (builder-stated;
 *   reward_t  = -beta * kl_t + [t == R-1] * score               PPO/KL math is a
 *                                                               reference non-goal,
 *                                                               SPEC.md:512)
 *   delta_t   = reward_t + gamma * V_{t+1} - V_t,  V_R = 0 (explicit terminal
 *               bootstrap, the T+1 convention of numerics.hpp:9-10)
 *   A_t       = delta_t + gamma*lam*A_{t+1},  A_{R-1} = delta_{R-1}
 *               (gae_recursive, proj/src/numerics.cpp:11-34)
 *   return_t  = A_t + V_t
 *
 * The GAE recursion here is pinned against the reference's golden vectors
 * (test_numerics.cpp:35-49 [1.855, 1.0], :59-70 lam=0, :122-131 bootstrap)
 * and against oracle/_ref/libfuseplan_ref.so's gae_recursive on random
 * rollouts in tests/test_oracle.py.
 *
 * Packed layout: sample i owns tokens [off[i], off[i+1]) of every per-token
 * array; R_i = off[i+1] - off[i] >= 1.
 */
#include <math.h>
#include <stdint.h>

/* gae over one rollout; values has T+1 entries. Returns 0, or 2 on bad args. */
int oracle_gae(const double* rewards, const double* values, int32_t T, double gamma, double lam,
               double* adv) {
  if (T < 1 || gamma < 0.0 || gamma > 1.0 || lam < 0.0 || lam > 1.0) return 2;
  for (int32_t t = 0; t < T; ++t) adv[t] = rewards[t] + gamma * values[t + 1] - values[t];
  const double k = gamma * lam;
  for (int32_t t = T - 1; t > 0; --t) adv[t - 1] += k * adv[t];
  return 0;
}

int oracle_postprocess(int32_t n, const int32_t* off, const float* logp_actor, const float* logp_ref,
                       const float* values, const float* score, double beta, double gamma, double lam,
                       double* kl, double* reward, double* adv, double* ret) {
  if (gamma < 0.0 || gamma > 1.0 || lam < 0.0 || lam > 1.0) return 2;
  for (int32_t i = 0; i < n; ++i) {
    const int32_t b = off[i], e = off[i + 1], R = e - b;
    if (R < 1) return 2;
    for (int32_t t = 0; t < R; ++t) {
      const double d = (double)logp_actor[b + t] - (double)logp_ref[b + t];
      kl[b + t] = d;
      reward[b + t] = -beta * d + (t == R - 1 ? (double)score[i] : 0.0);
    }
    /* delta then the backward recursion, in place in adv */
    for (int32_t t = 0; t < R; ++t) {
      const double v_next = (t + 1 < R) ? (double)values[b + t + 1] : 0.0;
      adv[b + t] = reward[b + t] + gamma * v_next - (double)values[b + t];
    }
    const double k = gamma * lam;
    for (int32_t t = R - 1; t > 0; --t) adv[b + t - 1] += k * adv[b + t];
    for (int32_t t = 0; t < R; ++t) ret[b + t] = adv[b + t] + (double)values[b + t];
  }
  return 0;
}
