// fuseplan-b200 — the residual-add + RMSNorm row shared by add_norm_kernel
// (layers.cu) and the split-K GEMM's fused norm (gemm.cuh, EpiStoreF32): one
// definition of the arithmetic, so both produce the same bits.
#pragma once

#include <cuda_bf16.h>

#include "ptx.cuh"

namespace fpk {

constexpr float kNormEps = 1e-5f;

__device__ __forceinline__ float sumsq4(const float4 v) { return v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w; }

__device__ __forceinline__ uint2 norm_scale4(const float4 v, float inv, const float4 g) {
  return make_uint2(pack_bf16x2(v.x * inv * g.x, v.y * inv * g.y), pack_bf16x2(v.z * inv * g.z, v.w * inv * g.w));
}

// Row sum over the nw warps of a named barrier group (warp-sum, then the warp
// sums in warp order through red[]) — add_norm's block_sum with blockDim =
// 32 * nw.
template <class Sync>
__device__ __forceinline__ float group_sum(float v, float* red, int w, int l, int nw, Sync sync) {
  v = warp_sum(v);
  if (l == 0) red[w] = v;
  sync();
  float t = (l < nw) ? red[l] : 0.f;
  t = warp_sum(t);
  sync();
  return t;
}

}  // namespace fpk
