// fuseplan-b200 — per-token experience post-processing.
//
// One warp per sample (R response tokens, packed at [off[i], off[i+1])):
//   kl_t     = logp_actor_t - logp_ref_t
//   reward_t = -beta kl_t + [t = R-1] score
//   delta_t  = reward_t + gamma V_{t+1} - V_t,  V_R = 0 (explicit bootstrap,
//              the T+1 convention of proj/include/fuseplan/numerics.hpp:9-10)
//   A_t      = delta_t + gamma lam A_{t+1}     (gae_recursive, numerics.cpp:27-34)
//   return_t = A_t + V_t
// The backward recursion is evaluated 32 tokens at a time as a reverse
// warp scan of the affine map A -> delta + c A (c = gamma lam), carrying the
// chunk's A_0 into the preceding chunk. HBM-bound (reads 3 + writes 4
// floats per token).
#include "ops.h"
#include "ptx.cuh"

namespace fpk {

namespace {

__global__ void postprocess_kernel(int n, const int* __restrict__ off, const float* __restrict__ la,
                                   const float* __restrict__ lr, const float* __restrict__ val,
                                   const float* __restrict__ score, float beta, float gamma, float lam,
                                   float* __restrict__ kl, float* __restrict__ rew, float* __restrict__ adv,
                                   float* __restrict__ ret, PostScatter sc_out) {
  pdl_trigger();  // let the next (PDL-launched) GEMM start its prologue / weight prefetch
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  const int b = off[i], e = off[i + 1];
  const int R = e - b;
  if (R <= 0) return;
  // output offset: packed (b) or the sample's global response offset
  const int64_t ob = sc_out.off_out ? sc_out.off_out[i] : b;
  if (sc_out.score_out && lane == 0) sc_out.score_out[sc_out.sid[i]] = score[i];
  const float c = gamma * lam;
  float cp[5];  // c^1, c^2, c^4, c^8, c^16
  cp[0] = c;
#pragma unroll
  for (int k = 1; k < 5; ++k) cp[k] = cp[k - 1] * cp[k - 1];
  const float sc = score[i];
  float carry = 0.f;        // A at the first token of the chunk to the right
  float v_right = 0.f;      // V at the first token of the chunk to the right (V_R = 0)
  const int nchunks = (R + 31) / 32;
  for (int ch = nchunks - 1; ch >= 0; --ch) {
    const int t = ch * 32 + lane;
    const bool ok = t < R;
    const int g = b + t;
    float a_lp = 0.f, r_lp = 0.f, v = 0.f;
    if (ok) {
      a_lp = la[g];
      r_lp = lr[g];
      v = val[g];
    }
    const float d_kl = a_lp - r_lp;
    const float r = -beta * d_kl + (t == R - 1 ? sc : 0.f);
    // V_{t+1}: next lane, or the right chunk's first value
    float v_next = __shfl_down_sync(0xffffffffu, v, 1);
    const int last_in_chunk = min(31, R - 1 - ch * 32);
    if (lane == last_in_chunk) v_next = (t == R - 1) ? 0.f : v_right;
    const float delta = ok ? r + gamma * v_next - v : 0.f;
    // reverse inclusive scan: s_lane = sum_{j>=lane} c^{j-lane} delta_j (within chunk)
    float s = delta;
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const int o = 1 << k;
      const float y = __shfl_down_sync(0xffffffffu, s, o);
      if (lane + o < 32) s = fmaf(cp[k], y, s);
    }
    // + c^{(last+1-lane)} * carry
    float cpow = 1.f;
    int pw = last_in_chunk + 1 - lane;
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      if (pw & 1) cpow *= (k < 5 ? cp[k] : cp[4] * cp[4]);
      pw >>= 1;
    }
    const float A = ok ? fmaf(cpow, carry, s) : 0.f;
    if (ok) {
      const int64_t o = ob + t;
      kl[o] = d_kl;
      rew[o] = r;
      adv[o] = A;
      ret[o] = A + v;
      if (sc_out.off_out) {
        sc_out.logp_actor[o] = a_lp;
        sc_out.logp_ref[o] = r_lp;
        sc_out.values[o] = v;
        sc_out.tokens_out[o] = sc_out.tokens_in[g];
      }
    }
    carry = __shfl_sync(0xffffffffu, A, 0);
    v_right = __shfl_sync(0xffffffffu, v, 0);
  }
}

}  // namespace

void postprocess(int n, const int* off, const float* logp_actor, const float* logp_ref, const float* values,
                 const float* score, float beta, float gamma, float lam, float* kl, float* reward, float* adv,
                 float* ret, cudaStream_t st, const PostScatter* scatter) {
  if (n <= 0) return;
  const int warps = 4;
  PostScatter sc{};
  if (scatter) sc = *scatter;
  postprocess_kernel<<<(n + warps - 1) / warps, warps * 32, 0, st>>>(n, off, logp_actor, logp_ref, values, score, beta,
                                                                      gamma, lam, kl, reward, adv, ret, sc); fpk::count_launch();
}

}  // namespace fpk
