// fuseplan-b200 — tcgen05/TMEM GEMM for sm_100a.
//
//   D[i][j] = sum_k A[i][k] * B[j][k]        (A, B bf16 K-major; D fp32 in TMEM)
//
// One CTA owns a 128 x BN tile of D (UMMA M=128, N=BN), loops over a K range
// of 64-element blocks (one 128-byte swizzle atom) through an S-stage
// TMA -> shared-memory ring, and hands the TMEM accumulator to an epilogue
// functor. Warp roles (192 threads):
//   warp 0      TMA producer (one elected lane)
//   warp 1      TMEM allocator + MMA issuer (one elected lane)
//   warps 2..5  epilogue: tcgen05.ld 32x32b.x32 -> registers -> Epi
// Which operand is the weight is the caller's choice: "swap-AB" (A = weight,
// B = activations) puts output features on TMEM lanes, which is what the
// decode GEMMs (batch on N <= 256) and the SwiGLU epilogue want; the vocab
// epilogue uses A = activations so that one thread owns one token row.
#pragma once

#include "ptx.cuh"

namespace fpk {

constexpr int kBK = 64;                  // K elements per stage (128 B)
constexpr int kTileA = 128 * kBK * 2;    // bytes of one A stage
constexpr int kGemmThreads = 192;

template <int BN>
struct GemmCfg {
  static constexpr int kTileB = BN * kBK * 2;
  static constexpr int kStageBytes = kTileA + kTileB;
  static constexpr int kStages = BN >= 256 ? 4 : (BN >= 128 ? 5 : 4);
  static constexpr int kSmem = kStages * kStageBytes + 1024;  // + alignment slack
  static constexpr uint32_t kTmemCols = BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : 256));
};

struct GemmGeom {
  int a_rows;        // valid rows of A
  int b_rows;        // valid rows of B
  int k_blocks;      // total 64-wide K blocks
  int kb_per_split;  // K blocks per gridDim.z slice
};

// Epilogue protocol (per epilogue thread; `State` lives in registers):
//   struct State {...};
//   __device__ void operator()(State&, int a_row0, int b_row0, int split, int r,
//                              int c0, const float (&v)[32], float* scratch) const;
//     r  = TMEM lane (A-row within tile), c0 = first of 32 B-columns;
//     scratch = drained pipeline smem, shared by the 4 epilogue warps, which
//     may synchronise with named barrier 1 (epi_bar_sync) — uniformly.
//   __device__ void finish(State&, int a_row0, int b_row0, int split, int r) const;
template <int BN, class Epi>
__global__ void __launch_bounds__(kGemmThreads, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                   GemmGeom g, Epi epi) {
  using C = GemmCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full_bar[C::kStages];
  __shared__ __align__(8) uint64_t empty_bar[C::kStages];
  __shared__ __align__(8) uint64_t acc_bar;
  __shared__ uint32_t tmem_base_smem;

  const uint32_t warp = warp_id();
  const int a_row0 = blockIdx.x * 128;
  const int b_row0 = blockIdx.y * BN;
  const int split = blockIdx.z;
  const int kb0 = split * g.kb_per_split;
  const int kb1 = min(g.k_blocks, kb0 + g.kb_per_split);
  const int nkb = kb1 - kb0;

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&map_a);
    tma_prefetch_desc(&map_b);
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(&acc_bar, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<C::kTmemCols>(&tmem_base_smem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_smem;

  if (warp == 0) {
    if (elect_one()) {
      for (int i = 0; i < nkb; ++i) {
        const int s = i % C::kStages;
        const uint32_t ph = (i / C::kStages) & 1;
        mbar_wait(&empty_bar[s], ph ^ 1);
        uint8_t* sa = smem + s * C::kStageBytes;
        uint8_t* sb = sa + kTileA;
        mbar_arrive_expect_tx(&full_bar[s], C::kStageBytes);
        tma_load_2d(sa, &map_a, &full_bar[s], (kb0 + i) * kBK, a_row0);
        tma_load_2d(sb, &map_b, &full_bar[s], (kb0 + i) * kBK, b_row0);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = idesc_bf16(128, BN);
    for (int i = 0; i < nkb; ++i) {
      const int s = i % C::kStages;
      const uint32_t ph = (i / C::kStages) & 1;
      mbar_wait(&full_bar[s], ph);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t sa = smem_u32(smem + s * C::kStageBytes);
        const uint32_t sb = sa + kTileA;
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k) {
          tc_mma_bf16(tmem, sdesc_k128(sa + k * 32), sdesc_k128(sb + k * 32), idesc, (i > 0 || k > 0) ? 1u : 0u);
        }
        tc_commit(&empty_bar[s]);
        if (i == nkb - 1) tc_commit(&acc_bar);
      }
      __syncwarp();
    }
  } else {
    // Epilogue warps 2..5 -> TMEM lane quarters (warp % 4).
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane_id();
    float* scratch = reinterpret_cast<float*>(smem);  // pipeline buffers are drained by then
    typename Epi::State st;
    if (nkb > 0) {
      mbar_wait(&acc_bar, 0);
      tc_fence_after();
    }
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
      float v[32];
      if (nkb > 0) {
        tmem_ld32(tmem + (static_cast<uint32_t>(quarter * 32) << 16) + c0, v);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = 0.f;
      }
      epi(st, a_row0, b_row0, split, r, c0, v, scratch);
    }
    epi.finish(st, a_row0, b_row0, split, r);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<C::kTmemCols>(tmem);
}

__device__ __forceinline__ void epi_bar_sync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// ---- epilogues ----------------------------------------------------------------

// swap-AB: A = weight [N, K] (rows = output features), B = activations [M, K].
// out[m * ld + n] = D[n][m] as bf16.
struct EpiStoreBF16 {
  __nv_bfloat16* out;
  int ld, n_valid, m_valid;
  struct State {};
  __device__ void operator()(State&, int a0, int b0, int, int r, int c0, const float (&v)[32], float*) const {
    const int n = a0 + r;
    if (n >= n_valid) return;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int m = b0 + c0 + j;
      if (m < m_valid) out[static_cast<size_t>(m) * ld + n] = f2bf(v[j]);
    }
  }
  __device__ void finish(State&, int, int, int, int) const {}
};

// swap-AB split-K partials: out[split][m][n] fp32 (summed by the consumer in
// split order, so each row's result is independent of the batch size).
// accumulate != 0 (single split only): out[m][n] += D — the residual add of
// the o / down projections fused into the GEMM.
struct EpiStoreF32 {
  float* out;
  size_t split_stride;
  int ld, n_valid, m_valid;
  int accumulate;
  struct State {};
  __device__ void operator()(State&, int a0, int b0, int split, int r, int c0, const float (&v)[32], float*) const {
    const int n = a0 + r;
    if (n >= n_valid) return;
    float* o = out + split * split_stride;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int m = b0 + c0 + j;
      if (m < m_valid) {
        float* dst = o + static_cast<size_t>(m) * ld + n;
        *dst = accumulate ? *dst + v[j] : v[j];
      }
    }
  }
  __device__ void finish(State&, int, int, int, int) const {}
};

// swap-AB fused SwiGLU. The gate/up weight is stored interleaved in 64-row
// groups: tile rows [0,64) are gate rows of features f0..f0+63 and rows
// [64,128) the matching up rows, f0 = a_row0 / 2. out[m][f] = silu(g) * u.
template <int BN>
struct EpiSwiGLU {
  __nv_bfloat16* out;
  int ld, f_valid, m_valid;
  struct State {};
  __device__ void operator()(State&, int a0, int b0, int, int r, int c0, const float (&v)[32], float* scratch) const {
    // scratch: [32 cols][64 lanes] of up values
    if (r >= 64) {
#pragma unroll
      for (int j = 0; j < 32; ++j) scratch[j * 64 + (r - 64)] = v[j];
    }
    epi_bar_sync();
    if (r < 64) {
      const int f = a0 / 2 + r;
      if (f < f_valid) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int m = b0 + c0 + j;
          const float gte = v[j];
          const float up = scratch[j * 64 + r];
          const float act = gte / (1.0f + __expf(-gte)) * up;
          if (m < m_valid) out[static_cast<size_t>(m) * ld + f] = f2bf(act);
        }
      }
    }
    epi_bar_sync();
  }
  __device__ void finish(State&, int, int, int, int) const {}
};

}  // namespace fpk
