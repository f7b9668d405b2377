// fuseplan-b200 — LM-head epilogue: log-softmax statistics, target gather,
// greedy argmax and Gumbel-max temperature sampling, fused into the tcgen05
// head GEMM so the [rows, V] logits never reach HBM.
//
// Orientation: A = hidden rows (one token per TMEM lane / epilogue thread),
// B = head weight rows (vocab ids on the BN columns). Each CTA emits, per row
// and per vocab tile, a VocabPartial {max z, sum exp(z - max), best key,
// best id, z of best}; z = logit / temperature. vocab_finalize() merges the
// tiles of a row in tile order (deterministic), picks the token (forced
// target | argmax z | argmax z + Gumbel(Philox(seed, sample, step, v))) and
// its log-probability z_token - logsumexp(z).
#pragma once

#include <math.h>

#include "philox.cuh"
#include "ptx.cuh"

namespace fpk {

enum TokenMode : int { kForced = 0, kGreedy = 1, kSample = 2 };

struct VocabPartial {
  float m, s, key, z;
  int idx, pad_;
};

struct VocabRowInfo {
  const int* target;     // [rows] forced target id (kForced) or nullptr
  const int* sample_id;  // [rows] Philox stream id (kSample)
  const int* step;       // [rows] response position (kSample)
};

// Gumbel noise of vocab id v in the stream (sample, step).
__device__ __forceinline__ float gumbel_of(uint32_t w) {
  const float u = (static_cast<float>(w >> 8) + 0.5f) * (1.0f / 16777216.0f);  // (0, 1)
  return -logf(-logf(u));
}

struct EpiVocab {
  VocabPartial* part;   // [rows][n_tiles]
  float* tgt_z;         // [rows] z of the forced target (written by its tile)
  VocabRowInfo info;
  int mode;
  float inv_temp;
  int vocab;
  int rows;
  int n_tiles;
  uint32_t seed_lo, seed_hi;

  struct State {
    float m, s, key, z;
    int idx;
    float tz;
    int has_t;
  };
  static constexpr bool kTmaStore = false;
  __device__ void store(const uint8_t*, int, int, int) const {}

  __device__ void operator()(State& st, uint8_t*, int a0, int b0, int, int r, int half, int c0,
                             const float (&v)[32]) const {
    const int row = a0 + r;
    if (c0 == 32 * half) {
      st.m = -INFINITY;
      st.s = 0.f;
      st.key = -INFINITY;
      st.z = -INFINITY;
      st.idx = -1;
      st.has_t = 0;
      st.tz = 0.f;
    }
    if (row >= rows || c0 >= 256) return;
    const int base = b0 + c0;
    if (base >= vocab) return;
    const int nvalid = min(32, vocab - base);
    float z[32];
    float cmax = -INFINITY;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      z[j] = v[j] * inv_temp;
      if (j < nvalid) cmax = fmaxf(cmax, z[j]);
    }
    const float nm = fmaxf(st.m, cmax);
    float acc = (st.m == -INFINITY) ? 0.f : st.s * expf(st.m - nm);
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < nvalid) acc += expf(z[j] - nm);
    st.m = nm;
    st.s = acc;

    if (mode == kForced) {
      const int t = info.target[row];
      if (t >= base && t < base + nvalid) {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (base + j == t) st.tz = z[j];
        st.has_t = 1;
      }
    } else if (mode == kGreedy) {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < nvalid && z[j] > st.key) {
          st.key = z[j];
          st.z = z[j];
          st.idx = base + j;
        }
    } else {
      const uint32_t sid = static_cast<uint32_t>(info.sample_id[row]);
      const uint32_t stp = static_cast<uint32_t>(info.step[row]);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const U4 w = philox4x32_10(U4{static_cast<uint32_t>((base >> 2) + q), stp, sid, 0xF00Du}, seed_lo, seed_hi);
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int j = q * 4 + e;
          if (j < nvalid) {
            const float k = z[j] + gumbel_of(ws[e]);
            if (k > st.key) {
              st.key = k;
              st.z = z[j];
              st.idx = base + j;
            }
          }
        }
      }
    }
  }

  __device__ void finish(State& st, int a0, int, int, int r, int half) const {
    const int row = a0 + r;
    if (row >= rows) return;
    VocabPartial p;  // one per (row, vocab tile = blockIdx.y, column half)
    p.m = st.m;
    p.s = st.s;
    p.key = st.key;
    p.z = st.z;
    p.idx = st.idx;
    p.pad_ = 0;
    part[static_cast<size_t>(row) * n_tiles + 2 * blockIdx.y + half] = p;
    if (mode == kForced && st.has_t) tgt_z[row] = st.tz;
  }
};

}  // namespace fpk
