// fuseplan-b200 — filtered sampling (top-k / top-p) over materialised logits.
//
// The unfiltered sampler never writes logits (EpiVocab: two-level exact
// sampling inside the head GEMM). A top-k / nucleus filter needs the k-th
// largest logit of the row first, so in that mode the head GEMM writes
// z = logit / T (fp32, gemm_vocab_logits) and this kernel, one CTA per row:
//   1. exact k-th largest z by a 4-pass 8-bit radix select on order-preserving
//      keys (integer histograms: deterministic);
//   2. gathers every z >= that value (ties at the boundary kept, as
//      HF's TopKLogitsWarper) and sorts them by (z desc, id asc) with a
//      bitonic sort — the candidate order is then independent of the
//      (non-deterministic) gather order;
//   3. masses e_i = exp2((z_i - z_0) log2 e) and their prefix sums in that
//      order (warp 0, lane-contiguous chunks: a fixed summation order the
//      CPU oracle replays), the nucleus = the shortest prefix whose mass
//      reaches top_p of the candidates' mass;
//   4. inverse-CDF draw in sorted order at u * mass(nucleus),
//      u = Philox4x32-10(seed; kFilterDraw, step, sample, 0xF00D).
// HBM traffic per row: the z row is read 5 times (radix passes + gather);
// it was just written by the head GEMM and is mostly L2-resident.
#include <cuda_runtime.h>

#include <stdexcept>

#include "launch.cuh"
#include "ops.h"
#include "philox.cuh"
#include "ptx.cuh"
#include "vocab.cuh"

namespace fpk {

namespace {

constexpr int kThreads = 512;
constexpr int kCand = 2 * kTopKMax;            // candidate capacity (ties beyond k)
constexpr uint32_t kFilterDraw = 0xFFFFFFFEu;  // Philox counter word of the filtered draw

__device__ __forceinline__ uint32_t order_key(float f) {
  const uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__global__ void __launch_bounds__(kThreads) topk_sample_kernel(const float* __restrict__ logits, int ldv, int V,
                                                               int top_k, float top_p,
                                                               const int* __restrict__ sample_id,
                                                               const int* __restrict__ step, uint32_t seed_lo,
                                                               uint32_t seed_hi, int* __restrict__ pick,
                                                               float* __restrict__ pick_z) {
  __shared__ unsigned int hist[256];
  __shared__ unsigned long long cand[kCand];
  __shared__ float csum[kCand];
  __shared__ uint32_t s_prefix, s_remaining;
  __shared__ int s_count;
  pdl_trigger();
  pdl_wait();  // the logits come from the head GEMM
  const int row = blockIdx.x;
  const int tid = threadIdx.x;
  const float* z = logits + static_cast<size_t>(row) * ldv;
  const int k = min(V, top_k > 0 ? min(top_k, kTopKMax) : kTopKMax);

  // 1. radix select: the key of the k-th largest z
  if (tid == 0) {
    s_prefix = 0;
    s_remaining = static_cast<uint32_t>(k);
  }
  uint32_t mask = 0;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = tid; i < 256; i += kThreads) hist[i] = 0;
    __syncthreads();
    const uint32_t prefix = s_prefix;
    for (int i = tid; i < V; i += kThreads) {
      const uint32_t key = order_key(z[i]);
      if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (tid == 0) {
      uint32_t above = 0, rem = s_remaining;
      int d = 255;
      for (; d > 0; --d) {
        if (above + hist[d] >= rem) break;
        above += hist[d];
      }
      s_remaining = rem - above;
      s_prefix = prefix | (static_cast<uint32_t>(d) << shift);
    }
    mask |= 255u << shift;
    __syncthreads();
  }
  const uint32_t kth = s_prefix;

  // 2. candidates (z >= the k-th largest), sorted by (z desc, id asc)
  if (tid == 0) s_count = 0;
  __syncthreads();
  for (int i = tid; i < V; i += kThreads) {
    const uint32_t key = order_key(z[i]);
    if (key >= kth) {
      const int p = atomicAdd(&s_count, 1);
      if (p < kCand) cand[p] = (static_cast<unsigned long long>(key) << 32) | (0xFFFFFFFFu - static_cast<uint32_t>(i));
    }
  }
  __syncthreads();
  // s_count > kCand only for a pathological tie group at the boundary; the
  // kept subset then depends on the gather order
  const int n = min(s_count, kCand);
  int np = 1;
  while (np < n) np <<= 1;
  for (int i = n + tid; i < np; i += kThreads) cand[i] = 0ull;
  __syncthreads();
  for (int size = 2; size <= np; size <<= 1) {  // bitonic sort, descending
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = tid; i < np; i += kThreads) {
        const int j = i ^ stride;
        if (j > i) {
          const bool desc = (i & size) == 0;
          const unsigned long long a = cand[i], b = cand[j];
          if ((a < b) == desc) {
            cand[i] = b;
            cand[j] = a;
          }
        }
      }
      __syncthreads();
    }
  }

  // 3./4. masses, nucleus and the draw (warp 0; fixed summation order)
  if (tid >= 32) return;
  const int lane = tid;
  auto z_of = [&](int i) { return z[0xFFFFFFFFu - static_cast<uint32_t>(cand[i])]; };
  const float z0 = z_of(0);
  const int chunk = (n + 31) / 32;
  const int c0 = min(n, lane * chunk), c1 = min(n, c0 + chunk);
  float run = 0.f;
  for (int i = c0; i < c1; ++i) {
    run += exp2f(__fmul_rn(z_of(i) - z0, kLog2E));
    csum[i] = run;  // lane-local inclusive prefix
  }
  float base = 0.f;  // exclusive prefix of the lane sums, in lane order
  for (int l = 0; l < 32; ++l) {
    const float t = __shfl_sync(0xffffffffu, run, l);
    if (l < lane) base += t;
  }
  for (int i = c0; i < c1; ++i) csum[i] += base;
  __syncwarp();
  const float total = csum[n - 1];
  // nucleus: the first index whose prefix mass reaches top_p * total
  int cut = n - 1;
  if (top_p < 1.f) {
    const float need = top_p * total;
    int first = n;
    for (int i = lane; i < n; i += 32)
      if (csum[i] >= need) {
        first = i;
        break;
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
    cut = min(first, n - 1);
  }
  const U4 w = philox4x32_10(U4{kFilterDraw, static_cast<uint32_t>(step[row]),
                                static_cast<uint32_t>(sample_id[row]), 0xF00Du},
                             seed_lo, seed_hi);
  const float thr = unit_open(w.x) * csum[cut];
  int sel = cut + 1;
  for (int i = lane; i <= cut; i += 32)
    if (csum[i] >= thr) {
      sel = i;
      break;
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sel = min(sel, __shfl_xor_sync(0xffffffffu, sel, o));
  sel = min(sel, cut);
  if (lane == 0) {
    const int id = static_cast<int>(0xFFFFFFFFu - static_cast<uint32_t>(cand[sel]));
    pick[row] = id;
    pick_z[row] = z[id];
  }
}

}  // namespace

void topk_sample(const float* logits, int ldv, int M, int V, int top_k, float top_p, const int* sample_id,
                 const int* step, uint64_t seed, int* pick, float* pick_z, cudaStream_t st) {
  if (M <= 0) return;
  if (top_k < 0 || top_k > kTopKMax || !(top_p > 0.f && top_p <= 1.f))
    throw std::invalid_argument("topk_sample: top_k must lie in [0, kTopKMax] and top_p in (0, 1]");
  launch_pdl(topk_sample_kernel, dim3(M), dim3(kThreads), 0, st, logits, ldv, V, top_k, top_p, sample_id, step,
             static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32), pick, pick_z);
  fpk::count_launch();
}

}  // namespace fpk
