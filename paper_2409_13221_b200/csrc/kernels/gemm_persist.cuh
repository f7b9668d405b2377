// fuseplan-b200 — persistent tcgen05 GEMM for the packed forwards (prefill and
// the scoring models: thousands of rows).
//
// Same math, operands, epilogue functors and per-element K order as
// tc_gemm_kernel (gemm.cuh) — so every output element has the same bits — but
// one CTA per SM walks a static list of 128 x BN output tiles:
//   warp 0      TMA producer: the ring runs across tile boundaries
//   warp 1      MMA issuer: accumulates tile i into TMEM buffer i & 1
//   warps 2..9  epilogue of tile i (TMEM buffer i & 1) while the MMA warp
//               already fills buffer (i + 1) & 1
// The epilogue stages its output in a shared-memory area of its own (the ring
// keeps streaming the next tiles), so the ring gets what the budget leaves.
// This removes the two costs the one-tile-per-CTA kernel pays at large M: the
// exposed epilogue (no mainloop runs under it) and wave quantisation (e.g.
// 192 tiles on 148 SMs = two waves for 1.3 waves of work).
#pragma once

#include "gemm.cuh"
#include "vocab.cuh"

namespace fpk {

// Shared memory the epilogue stages one output tile in (bytes).
template <int BN, class Epi>
struct EpiStaging {
  static constexpr int v = ((BN + 63) / 64) * 64 * 128 * 2;  // bf16 [round64(BN)][128]
};
template <int BN>
struct EpiStaging<BN, EpiStoreF32> {
  static constexpr int v = ((BN + 63) / 64) * 64 * 128 * 4;  // fp32
};
template <int BN>
struct EpiStaging<BN, EpiSwiGLU<BN>> {
  static constexpr int v = EpiSwiGLU<BN>::kTileBytes + 2 * 32 * 128 * 4;  // tile + gate/up exchange
};

// Residual add without staging: resid[m][n] += D[n][m] straight from the
// accumulator registers. Each element belongs to exactly one tile (no split-K),
// so a plain load-add-store gives the bits of the TMA reduce-add (one fp32 add,
// round to nearest) — and the staging smem goes to a deeper TMA ring: the
// small-K scoring GEMMs are bound by the operand bytes a CTA keeps in flight.
// A warp covers 32 consecutive features of one token per access (128 B).
struct EpiResidDirect {
  float* resid;
  int N, M;
  static constexpr bool kTmaStore = false;
  static constexpr int kPasses = 1;
  template <class S> __device__ void next_pass(S&, int, int, int, int) const {}
  struct State {};
  __device__ void operator()(State&, uint8_t*, int a0, int b0, int, int r, int, int c0, const float (&v)[32]) const {
    const int n = a0 + r;
    const int m0 = b0 + c0;
    if (n >= N || m0 >= M) return;
    float* p = resid + static_cast<size_t>(m0) * N + n;
    const int cnt = min(32, M - m0);
    float old[32];
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < cnt) old[j] = p[static_cast<size_t>(j) * N];
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < cnt) p[static_cast<size_t>(j) * N] = old[j] + v[j];
  }
  __device__ void finish(State&, int, int, int, int, int) const {}
  __device__ void store(const uint8_t*, int, int, int) const {}
};
template <int BN>
struct EpiStaging<BN, EpiResidDirect> {
  static constexpr int v = 0;
};
template <int BN, int MODE>
struct EpiStaging<BN, EpiVocab<MODE>> {  // writes its partials straight to global memory
  static constexpr int v = 0;
};

// SwiGLU with the same gate/up pairing and arithmetic as EpiSwiGLU (so the
// same bits) but the outputs go straight to global memory: per store a warp
// writes 32 consecutive features of one token (64 B). Only the gate/up
// exchange buffer stays in shared memory, which leaves room for a 4-stage ring
// at BN = 256.
template <int BN>
struct EpiSwiGLUDirect {
  __nv_bfloat16* out;
  int F, M;
  static constexpr bool kTmaStore = false;
  static constexpr int kPasses = 1;
  template <class S> __device__ void next_pass(S&, int, int, int, int) const {}
  struct State {};
  __device__ void operator()(State&, uint8_t* smem, int a0, int b0, int, int r, int half, int c0,
                             const float (&v)[32]) const {
    float* xch = reinterpret_cast<float*>(smem) + half * 32 * 128;  // [32][128]
    const uint32_t xa = smem_u32(xch) + r * 4;
#pragma unroll
    for (int j = 0; j < 32; ++j) sts_f32(xa + j * 512, v[j]);
    half_bar_sync(half);
    const int t = r;
    const int f = t & 63, j0 = (t >> 6) * 16;
    if (c0 < BN) {
      float gte[16], up[16];
      const uint32_t xr = smem_u32(xch) + (j0 * 128 + f) * 4;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        gte[j] = lds_f32(xr + j * 512);
        up[j] = lds_f32(xr + j * 512 + 256);
      }
      const int m0 = b0 + c0 + j0;
      __nv_bfloat16* o = out + static_cast<size_t>(m0) * F + a0 / 2 + f;
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (m0 + j < M) o[static_cast<size_t>(j) * F] = f2bf(__fdividef(gte[j], 1.0f + __expf(-gte[j])) * up[j]);
    }
    half_bar_sync(half);
  }
  __device__ void finish(State&, int, int, int, int, int) const {}
  __device__ void store(const uint8_t*, int, int, int) const {}
};
template <int BN>
struct EpiStaging<BN, EpiSwiGLUDirect<BN>> {
  static constexpr int v = 2 * 32 * 128 * 4;  // gate/up exchange only
};

constexpr int kPersistSmem = 227 * 1024;

template <int BN, class Epi>
struct PersistCfg {
  static constexpr int kStageBytes = kTileA + BN * kBK * 2;
  static constexpr int kStaging = EpiStaging<BN, Epi>::v + EpiSmemExtra<Epi>::value;
  static constexpr int kStages = (kPersistSmem - 1024 - kStaging - 256) / kStageBytes;
  static constexpr int kSmem = kStages * kStageBytes + kStaging + 1024 + 256;
  static constexpr uint32_t kAccCols = GemmCfg<BN>::kTmemCols;
  static constexpr uint32_t kTmemCols = 2 * kAccCols;
  static_assert(kStages >= 2, "persistent GEMM: ring too shallow");
  static_assert(kTmemCols <= 512, "persistent GEMM: two accumulators must fit TMEM");
};

struct PersistGeom {
  int a_rows, b_rows, k_blocks, a_tiles, n_tiles;
  int weight_is_a;  // 1: A (prefetched before griddepcontrol.wait) is the weight; 0: B is
  unsigned long long* trace;  // debug (fp_k_gemm_trace): per CTA, per local tile i < 8: 4 globaltimer stamps
};

__device__ __forceinline__ void persist_stamp(const PersistGeom& g, int i, int k) {
  if (g.trace && i < 8) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g.trace[(blockIdx.x * 8 + i) * 4 + k] = t;
  }
}

template <int BN, class Epi>
__global__ void __launch_bounds__(kGemmThreads, 1)
    tc_gemm_persist_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                           const PersistGeom g, const __grid_constant__ Epi epi) {
  using C = PersistCfg<BN, Epi>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* staging = smem + C::kStages * C::kStageBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(staging + C::kStaging);
  uint64_t* full_bar = bars;                    // [kStages]
  uint64_t* empty_bar = bars + C::kStages;      // [kStages]
  uint64_t* acc_full = bars + 2 * C::kStages;   // [2]
  uint64_t* acc_empty = acc_full + 2;           // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const uint32_t warp = warp_id();
  pdl_trigger();
  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&map_a);
    tma_prefetch_desc(&map_b);
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 32 * kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<C::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int nkb = g.k_blocks;

  if (warp == 0) {
    if (elect_one()) {
      // ring position it -> (local tile it / nkb, k-block it % nkb). The weight
      // operand does not depend on the previous kernel: the first kStages
      // stages of it are issued before griddepcontrol.wait, the activations
      // after it.
      const int local_tiles = g.n_tiles > static_cast<int>(blockIdx.x)
                                  ? (g.n_tiles - 1 - static_cast<int>(blockIdx.x)) / static_cast<int>(gridDim.x) + 1
                                  : 0;
      const int total = local_tiles * nkb;
      const int pre = min(total, C::kStages);
      auto rows_of = [&](int it, int& a_row0, int& b_row0) {
        const int t = blockIdx.x + (it / nkb) * gridDim.x;
        a_row0 = (t % g.a_tiles) * 128;
        b_row0 = (t / g.a_tiles) * BN;
      };
      auto load_weight = [&](uint8_t* sa, int it, int a_row0, int b_row0) {
        const int s = it % C::kStages, kb = it % nkb;
        if (g.weight_is_a)
          tma_load_2d(sa, &map_a, &full_bar[s], kb * kBK, a_row0);
        else
          tma_load_2d(sa + kTileA, &map_b, &full_bar[s], kb * kBK, b_row0);
      };
      for (int it = 0; it < pre; ++it) {
        int a_row0, b_row0;
        rows_of(it, a_row0, b_row0);
        mbar_arrive_expect_tx(&full_bar[it], C::kStageBytes);
        load_weight(smem + it * C::kStageBytes, it, a_row0, b_row0);
      }
      pdl_wait();
      for (int it = 0; it < total; ++it) {
        const int s = it % C::kStages, kb = it % nkb;
        int a_row0, b_row0;
        rows_of(it, a_row0, b_row0);
        uint8_t* sa = smem + s * C::kStageBytes;
        if (it >= pre) {
          mbar_wait(&empty_bar[s], ((it / C::kStages) & 1) ^ 1);
          mbar_arrive_expect_tx(&full_bar[s], C::kStageBytes);
          load_weight(sa, it, a_row0, b_row0);
        }
        if (g.weight_is_a)
          tma_load_2d(sa + kTileA, &map_b, &full_bar[s], kb * kBK, b_row0);
        else
          tma_load_2d(sa, &map_a, &full_bar[s], kb * kBK, a_row0);
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      constexpr uint32_t idesc = idesc_bf16(128, BN);
      const uint64_t da = sdesc_k128(smem_u32(smem)), db = sdesc_k128(smem_u32(smem) + kTileA);
      int it = 0, i = 0;
      for (int t = blockIdx.x; t < g.n_tiles; t += gridDim.x, ++i) {
        const int buf = i & 1;
        mbar_wait(&acc_empty[buf], ((i >> 1) & 1) ^ 1);  // epilogue drained this buffer (tile i - 2)
        tc_fence_after();
        const uint32_t acc = tmem + buf * C::kAccCols;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % C::kStages;
          mbar_wait(&full_bar[s], (it / C::kStages) & 1);
          if (kb == 0) persist_stamp(g, i, 0);
          tc_fence_after();
          const uint64_t off = static_cast<uint64_t>((s * C::kStageBytes) >> 4);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k)
            tc_mma_bf16(acc, da + off + 2 * k, db + off + 2 * k, idesc, (kb > 0 || k > 0) ? 1u : 0u);
          tc_commit(&empty_bar[s]);
        }
        tc_commit(&acc_full[buf]);
        persist_stamp(g, i, 1);
      }
    }
    __syncwarp();
  } else {
    const int quarter = warp & 3;
    const int half = (static_cast<int>(warp) - 2) >> 2;
    const int r = quarter * 32 + lane_id();
    pdl_wait();
    int i = 0;
    for (int t = blockIdx.x; t < g.n_tiles; t += gridDim.x, ++i) {
      const int a_row0 = (t % g.a_tiles) * 128, b_row0 = (t / g.a_tiles) * BN;
      const int buf = i & 1;
      typename Epi::State st{};
      if constexpr (EpiHasPrologue<Epi>::value) epi.prologue(st, a_row0, b_row0, staging + EpiStaging<BN, Epi>::v);
      mbar_wait(&acc_full[buf], (i >> 1) & 1);
      if (threadIdx.x == 64) persist_stamp(g, i, 2);
      tc_fence_after();
      const uint32_t acc = tmem + buf * C::kAccCols + (static_cast<uint32_t>(quarter * 32) << 16);
#pragma unroll 1
      for (int pass = 0; pass < Epi::kPasses; ++pass) {
        if (pass) epi.next_pass(st, a_row0, b_row0, r, half);
#pragma unroll 1
        for (int c0 = 32 * half; c0 < ((BN + 63) / 64) * 64; c0 += 64) {
          float v[32];
          if (c0 < BN) {
            tmem_ld32(acc + c0, v);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = 0.f;
          }
          epi(st, staging, a_row0, b_row0, 0, r, half, c0, v);
        }
      }
      tc_fence_before();
      mbar_arrive(&acc_empty[buf]);  // TMEM buffer free: the MMA warp may start tile i + 2 in it
      epi.finish(st, a_row0, b_row0, 0, r, half);
      if constexpr (Epi::kTmaStore) {
        fence_async_smem();
        epi_bar_sync();
        if (threadIdx.x == 64) {
          epi.store(staging, a_row0, b_row0, 0);
          bulk_commit_wait_read();
        }
      }
      epi_bar_sync();  // staging reusable: the store has read it / finish() is done with it
      if (threadIdx.x == 64) persist_stamp(g, i, 3);
    }
    if constexpr (EpiHasPost<Epi>::value) epi.post();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<C::kTmemCols>(tmem);
}

}  // namespace fpk
