// fuseplan-b200 — LM-head epilogue: log-softmax statistics, target gather,
// greedy argmax and exact temperature sampling, fused into the tcgen05 head
// GEMM so the [rows, V] logits never reach HBM.
//
// Orientation: A = hidden rows (one token per TMEM lane), B = head weight rows
// (vocab ids on the BN = 256 columns). Each epilogue thread owns one row and
// one half of the tile's columns (the interleaved 32-column chunks of its
// warp half), and emits one VocabPartial per (row, tile, half): with
// z = logit / T and z2 = z log2(e),
//   m2 = max z2,  s = sum 2^(z2 - m2)  (exp2 on the MUFU),
//   (idx, zsel) = the half-tile's candidate token:
//       greedy: argmax z (ties: lower id);
//       sample: inverse CDF of 2^(z2 - m2) at u s, u = Philox(seed, sample,
//               step, partial index) — a second pass re-reads TMEM;
//   forced targets write their z to tgt_z.
// vocab_finalize() merges a row's partials in partial order (deterministic):
// logsumexp, and for sampling picks the half-tile by inverse CDF of
// s_t 2^(m2_t - M2) at u' (Philox counter 0xFFFFFFFF). Exact sampling from
// softmax(z): P(v) = P(tile) P(v | tile). One Philox draw per 128 vocab
// entries instead of a Gumbel variate per entry.
#pragma once

#include <math.h>

#include "philox.cuh"
#include "ptx.cuh"

namespace fpk {

enum TokenMode : int { kForced = 0, kGreedy = 1, kSample = 2 };
// Filtered sampling (top-k / top-p): the epilogue keeps the log-softmax
// statistics and writes z = logit / T to a [rows, ldv] fp32 buffer, which
// topk_sample() filters and samples from.
constexpr int kLogits = 3;
constexpr float kLog2E = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr uint32_t kRowDraw = 0xFFFFFFFFu;  // Philox counter word of the tile choice

struct VocabPartial {
  float m2, s, zsel;
  int idx;
  float pad0, pad1;
};
static_assert(sizeof(VocabPartial) == 24, "vocab_finalize stages a row of partials as 16-byte words");

struct VocabRowInfo {
  const int* target;     // [rows] forced target id (kForced) or nullptr
  const int* sample_id;  // [rows] Philox stream id (kSample)
  const int* step;       // [rows] response position (kSample)
};

// u in (0, 1) from the top 24 bits of a Philox word.
__host__ __device__ __forceinline__ float unit_open(uint32_t w) {
  return (static_cast<float>(w >> 8) + 0.5f) * (1.0f / 16777216.0f);
}

template <int MODE>
struct EpiVocab {
  VocabPartial* part;   // [rows][n_tiles]
  float* tgt_z;         // [rows] z of the forced target (written by its tile)
  VocabRowInfo info;
  float inv_temp;
  int vocab;
  int rows;
  int n_tiles;
  uint32_t seed_lo, seed_hi;
  float* logits;  // kLogits: [rows][ldv]
  int ldv;

  static constexpr bool kTmaStore = false;
  static constexpr int kPasses = MODE == kSample ? 2 : 1;
  // 2 x 48 KB ring: two CTAs per SM, so a vocab sweep of 197 column tiles at
  // small M is one wave and each CTA's (heavy) epilogue overlaps the other's
  // mainloop
  static constexpr int kStages = 2;
  __device__ void store(const uint8_t*, int, int, int) const {}

  struct State {
    float m, s;      // running max of z2, sum of 2^(z2 - m)
    float zsel;      // z of the candidate
    int idx;         // candidate id
    float thr, acc;  // sampling walk (pass 1)
    float tz;
    int has_t, pass;
  };

  __device__ void next_pass(State& st, int a0, int b0, int r, int half) const {
    st.pass = 1;
    st.acc = 0.f;
    const int row = a0 + r;
    if (row >= rows || st.m == -INFINITY) {
      st.thr = INFINITY;
      return;
    }
    const uint32_t pidx = static_cast<uint32_t>(2 * (b0 / 256) + half);
    const U4 w = philox4x32_10(U4{pidx, static_cast<uint32_t>(info.step[row]),
                                  static_cast<uint32_t>(info.sample_id[row]), 0xF00Du},
                               seed_lo, seed_hi);
    st.thr = unit_open(w.x) * st.s;
  }

  __device__ void operator()(State& st, uint8_t*, int a0, int b0, int, int r, int half, int c0,
                             const float (&v)[32]) const {
    const int row = a0 + r;
    if (c0 == 32 * half && st.pass == 0) {
      st.m = -INFINITY;
      st.s = 0.f;
      st.zsel = -INFINITY;
      st.idx = -1;
      st.has_t = 0;
      st.tz = 0.f;
      st.pass = 0;
    }
    if (row >= rows || c0 >= 256) return;
    const int base = b0 + c0;
    if (base >= vocab) return;
    const int nvalid = min(32, vocab - base);
    const float c2 = inv_temp * kLog2E;
    if (st.pass == 1) {  // sampling walk: first column whose running mass reaches thr
      if (st.acc >= st.thr) return;
      float e[32];  // the chunk's masses first (independent MUFU work), then the serial walk over them
#pragma unroll
      for (int j = 0; j < 32; ++j) e[j] = exp2f(v[j] * c2 - st.m);
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if (j < nvalid && st.acc < st.thr) {
          st.acc += e[j];
          st.idx = base + j;
          st.zsel = v[j] * inv_temp;
        }
      }
      return;
    }
    float cmax = -INFINITY;
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < nvalid) cmax = fmaxf(cmax, v[j] * c2);
    const float nm = fmaxf(st.m, cmax);
    float acc = (st.m == -INFINITY) ? 0.f : st.s * exp2f(st.m - nm);
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < nvalid) acc += exp2f(v[j] * c2 - nm);
    st.m = nm;
    st.s = acc;
    if constexpr (MODE == kLogits) {
      float* dst = logits + static_cast<size_t>(row) * ldv + base;
      if (nvalid == 32) {
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          *reinterpret_cast<float4*>(dst + j) =
              make_float4(v[j] * inv_temp, v[j + 1] * inv_temp, v[j + 2] * inv_temp, v[j + 3] * inv_temp);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (j < nvalid) dst[j] = v[j] * inv_temp;
      }
    } else if constexpr (MODE == kForced) {
      const int t = info.target[row];
      if (t >= base && t < base + nvalid) {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (base + j == t) st.tz = v[j] * inv_temp;
        st.has_t = 1;
      }
    } else if constexpr (MODE == kGreedy) {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float z = v[j] * inv_temp;
        if (j < nvalid && z > st.zsel) {
          st.zsel = z;
          st.idx = base + j;
        }
      }
    }
  }

  __device__ void finish(State& st, int a0, int b0, int, int r, int half) const {
    const int row = a0 + r;
    if (row >= rows) return;
    VocabPartial p;  // one per (row, vocab tile = blockIdx.y, column half)
    p.m2 = st.m;
    p.s = st.s;
    p.zsel = st.zsel;
    p.idx = st.idx;
    p.pad0 = p.pad1 = 0.f;
    part[static_cast<size_t>(row) * n_tiles + 2 * (b0 / 256) + half] = p;
    if (MODE == kForced && st.has_t) tgt_z[row] = st.tz;
  }
};

}  // namespace fpk
