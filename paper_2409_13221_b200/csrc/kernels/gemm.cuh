// fuseplan-b200 — tcgen05/TMEM GEMM for sm_100a.
//
//   D[i][j] = sum_k A[i][k] * B[j][k]        (A, B bf16 K-major; D fp32 in TMEM)
//
// One CTA owns a 128 x BN tile of D (UMMA M=128, N=BN), loops over a K range
// of 64-element blocks (one 128-byte swizzle atom) through an S-stage
// TMA -> shared-memory ring, and hands the TMEM accumulator to an epilogue
// functor. Warp roles (320 threads):
//   warp 0      TMA producer (one elected lane)
//   warp 1      TMEM allocator + MMA issuer (one elected lane)
//   warps 2..9  epilogue: tcgen05.ld 32x32b.x32 -> registers -> Epi; warp w
//               reads TMEM lane quarter w & 3, column half (w - 2) >> 2
// Which operand is the weight is the caller's choice: "swap-AB" (A = weight,
// B = activations) puts output features on TMEM lanes, which is what the
// decode GEMMs (batch on N <= 256) and the SwiGLU epilogue want; the vocab
// epilogue uses A = activations so that one thread owns one token row.
#pragma once

#include <type_traits>

#include "norm.cuh"
#include "ops.h"
#include "ptx.cuh"

namespace fpk {

constexpr int kBK = 64;                  // K elements per stage (128 B)
constexpr int kTileA = 128 * kBK * 2;    // bytes of one A stage
constexpr int kEpiWarps = 8;             // two per TMEM lane quarter (interleaved column chunks)
constexpr int kGemmThreads = 64 + 32 * kEpiWarps;
constexpr int kSmemBudget = 200 * 1024;

// STAGES = 0: as deep as the budget allows (the decode mainloop is latency-
// bound); an epilogue may pin a shallower ring (Epi::kStages) so that two CTAs
// share an SM and one's epilogue overlaps the other's mainloop.
template <int BN, int STAGES = 0>
struct GemmCfg {
  static constexpr int kTileB = BN * kBK * 2;
  static constexpr int kStageBytes = kTileA + kTileB;
  static constexpr int kFit = kSmemBudget / kStageBytes;
  static constexpr int kStages = STAGES > 0 ? STAGES : (kFit > 8 ? 8 : kFit);
  static constexpr int kSmem = kStages * kStageBytes + 1024;  // + alignment slack
  static constexpr uint32_t kTmemCols = BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : 256));
};

template <class E, class = void>
struct EpiHasPrologue : std::false_type {};
template <class E>
struct EpiHasPrologue<E, std::void_t<decltype(&E::prologue)>> : std::true_type {};

// Dynamic shared memory an epilogue needs beyond the ring (Epi::kSmemExtra),
// at offset kStages * kStageBytes; its prologue may fill it during the mainloop.
template <class E, class = void>
struct EpiSmemExtra {
  static constexpr int value = 0;
};
template <class E>
struct EpiSmemExtra<E, std::void_t<decltype(E::kSmemExtra)>> {
  static constexpr int value = E::kSmemExtra;
};

template <class E, class = void>
struct EpiHasPost : std::false_type {};
template <class E>
struct EpiHasPost<E, std::void_t<decltype(&E::post)>> : std::true_type {};

template <class E, class = void>
struct EpiStages {
  static constexpr int value = 0;
};
template <class E>
struct EpiStages<E, std::void_t<decltype(E::kStages)>> {
  static constexpr int value = E::kStages;
};

struct GemmGeom {
  int a_rows;        // valid rows of A
  int b_rows;        // valid rows of B
  int k_blocks;      // total 64-wide K blocks
  int kb_per_split;  // K blocks per gridDim.z slice
  int weight_is_a;   // 1: A is a weight (may be prefetched before griddepcontrol.wait)
  unsigned long long* trace;  // optional per-CTA phase stamps (globaltimer ns), 8 per CTA
};

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}


__device__ __forceinline__ void epi_bar_sync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }
// per-half barrier (128 threads: the 4 epilogue warps sharing column chunks)
__device__ __forceinline__ void half_bar_sync(int half) { asm volatile("bar.sync %0, 128;" ::"r"(2 + half) : "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void bulk_commit_wait() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
// Only until the bulk store has read its shared-memory source: enough before
// a CTA exits — the grid's completion (what the next kernel's
// griddepcontrol.wait observes) covers the global writes themselves.
__device__ __forceinline__ void bulk_commit_wait_read() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void tma_reduce_add_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}

// Epilogue protocol (per epilogue thread; `State` lives in registers):
//   struct State {...};
//   __device__ void operator()(State&, uint8_t* smem, int a_row0, int b_row0,
//                              int split, int r, int half, int c0, const float (&v)[32]) const;
//     r = TMEM lane (A-row within tile); the 8 epilogue warps form two halves
//     (warps 2-5 / 6-9, each covering the 4 lane quarters) that take
//     alternating 32-column chunks: half h processes c0 = 32 (2k + h). Every
//     half makes the same number of calls (ceil(BN / 64)); a call with
//     c0 >= BN carries zeros and must only take part in half_bar_sync(half).
//     smem = the drained pipeline buffers (tile staging / exchange).
//   __device__ void finish(State&, int a_row0, int b_row0, int split, int r, int half) const;
//   static constexpr bool kTmaStore; __device__ void store(const uint8_t* smem,
//     int a_row0, int b_row0, int split) const;   (one thread, after a barrier)
// ST > 0 overrides the ring depth (a 2-stage ring lets two CTAs share an SM:
// one's epilogue overlaps the other's mainloop — the large-M GEMMs).
template <int BN, class Epi, int ST = 0>
__global__ void __launch_bounds__(kGemmThreads, ST == 2 ? 2 : 1)  // the 2-stage shape must fit twice per SM
    tc_gemm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                   const GemmGeom g, const __grid_constant__ Epi epi) {
  using C = GemmCfg<BN, ST ? ST : EpiStages<Epi>::value>;
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
  unsigned long long* tr = nullptr;
  if (g.trace) {
    tr = g.trace + 8ull * (blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z));
    if (threadIdx.x == 0) tr[0] = gtime();
  }
  pdl_trigger();

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
  if (tr && threadIdx.x == 0) tr[1] = gtime();

  if (warp == 0) {
    if (elect_one()) {
      // Weights do not depend on the previous kernel: stream the first stages
      // of the weight operand before waiting on it (PDL overlap).
      const int pre = g.weight_is_a ? min(nkb, C::kStages) : 0;
      for (int i = 0; i < pre; ++i) {
        uint8_t* sa = smem + i * C::kStageBytes;
        mbar_arrive_expect_tx(&full_bar[i], C::kStageBytes);
        tma_load_2d(sa, &map_a, &full_bar[i], (kb0 + i) * kBK, a_row0);
      }
      pdl_wait();
      for (int i = 0; i < nkb; ++i) {
        const int s = i % C::kStages;
        const uint32_t ph = (i / C::kStages) & 1;
        uint8_t* sa = smem + s * C::kStageBytes;
        uint8_t* sb = sa + kTileA;
        if (i >= pre) {
          mbar_wait(&empty_bar[s], ph ^ 1);
          mbar_arrive_expect_tx(&full_bar[s], C::kStageBytes);
          tma_load_2d(sa, &map_a, &full_bar[s], (kb0 + i) * kBK, a_row0);
        }
        tma_load_2d(sb, &map_b, &full_bar[s], (kb0 + i) * kBK, b_row0);
      }
    }
  } else if (warp == 1) {
    // One thread issues: stage descriptors are the stage-0 ones plus the
    // stage offset (>> 4, the descriptor's address unit), so a stage costs a
    // wait, four MMAs and a commit — the issue loop, not the tensor core,
    // paces small-N decode GEMMs.
    if (elect_one()) {
      constexpr uint32_t idesc = idesc_bf16(128, BN);
      const uint64_t da = sdesc_k128(smem_u32(smem)), db = sdesc_k128(smem_u32(smem) + kTileA);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % C::kStages;
        mbar_wait(&full_bar[s], (i / C::kStages) & 1);
        if (tr && (i == 0 || i == nkb - 1)) tr[i == 0 ? 2 : 3] = gtime();
        tc_fence_after();
        const uint64_t off = static_cast<uint64_t>((s * C::kStageBytes) >> 4);
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k)
          tc_mma_bf16(tmem, da + off + 2 * k, db + off + 2 * k, idesc, (i > 0 || k > 0) ? 1u : 0u);
        tc_commit(&empty_bar[s]);
      }
      if (nkb > 0) tc_commit(&acc_bar);
    }
    __syncwarp();
  }
  // Epilogue warps 2..9 -> TMEM lane quarters (warp % 4), two halves.
  const int quarter = warp & 3;
  const int half = (static_cast<int>(warp) - 2) >> 2;
  const int r = quarter * 32 + lane_id();
  typename Epi::State st{};
  auto run_epi = [&](auto&& load) {
#pragma unroll 1
    for (int pass = 0; pass < Epi::kPasses; ++pass) {  // two-pass epilogues re-read TMEM (cheap)
      if (pass) epi.next_pass(st, a_row0, b_row0, r, half);
#pragma unroll 1
      for (int c0 = 32 * half; c0 < ((BN + 63) / 64) * 64; c0 += 64) {
        float v[32];
        load(c0, v);
        epi(st, smem, a_row0, b_row0, split, r, half, c0, v);
      }
    }
    epi.finish(st, a_row0, b_row0, split, r, half);
    if constexpr (Epi::kTmaStore) {
      fence_async_smem();
      epi_bar_sync();
      if (threadIdx.x == 64) {
        epi.store(smem, a_row0, b_row0, split);
        bulk_commit_wait_read();
      }
    }
  };
  auto tmem_load = [&](int c0, float (&v)[32]) {
    if (nkb > 0 && c0 < BN) {
      tmem_ld32(tmem + (static_cast<uint32_t>(quarter * 32) << 16) + c0, v);
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = 0.f;
    }
  };
  if (warp >= 2) {
    pdl_wait();
    // epilogue inputs that do not depend on the accumulator (e.g. positions,
    // pages, rope tables) are fetched while the mainloop runs
    if constexpr (EpiHasPrologue<Epi>::value) epi.prologue(st, a_row0, b_row0, smem + C::kStages * C::kStageBytes);
    if (nkb > 0) {
      mbar_wait(&acc_bar, 0);
      if (tr && threadIdx.x == 64) tr[4] = gtime();
      tc_fence_after();
    }
    run_epi(tmem_load);
    if (tr && threadIdx.x == 64) tr[5] = gtime();
    if constexpr (EpiHasPost<Epi>::value) epi.post();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<C::kTmemCols>(tmem);
}

// ---- epilogues ----------------------------------------------------------------
// The swap-AB epilogues stage the output tile in shared memory as
// [BN tokens][128 features] (the row-major layout of the output) and write it
// with one TMA bulk tensor store (or reduce-add), instead of 2-byte scattered
// stores: thread r (feature r) writes column r of the tile, so every st.shared
// of a warp covers 32 consecutive features (conflict-free). Out-of-range rows /
// columns are clipped by the TMA unit.

// out[m][n] = D[n][m] as bf16; map: [M rows][ld] bf16, box {128, BN}.
struct EpiStoreBF16 {
  CUtensorMap map;
  static constexpr bool kTmaStore = true;
  static constexpr int kPasses = 1;
  template <class S> __device__ void next_pass(S&, int, int, int, int) const {}
  struct State {};
  __device__ void operator()(State&, uint8_t* smem, int, int, int, int r, int, int c0, const float (&v)[32]) const {
    __nv_bfloat16* tile = reinterpret_cast<__nv_bfloat16*>(smem);
    const uint32_t t = smem_u32(tile) + (c0 * 128 + r) * 2;  // c0 < BN + 32: inside the staging area
#pragma unroll
    for (int j = 0; j < 32; ++j) sts_bf16(t + j * 256, f2bf(v[j]));
  }
  __device__ void finish(State&, int, int, int, int, int) const {}
  __device__ void store(const uint8_t* smem, int a0, int b0, int) const { tma_store_2d(&map, smem, a0, b0); }
};

// fp32 out: split-K partials out[split][m][n] (3-D map {N, M, splits}; the
// consumer sums them in split order, so each row is batch-independent), or —
// accumulate — a TMA reduce-add into the residual stream out[m][n] (2-D map):
// the residual add of the o / down projections fused into the GEMM.
struct EpiStoreF32 {
  CUtensorMap map;
  int accumulate;
  static constexpr bool kTmaStore = true;
  static constexpr int kPasses = 1;
  template <class S> __device__ void next_pass(S&, int, int, int, int) const {}
  struct State {};
  __device__ void operator()(State&, uint8_t* smem, int, int, int, int r, int, int c0, const float (&v)[32]) const {
    float* tile = reinterpret_cast<float*>(smem);
    const uint32_t t = smem_u32(tile) + (c0 * 128 + r) * 4;
#pragma unroll
    for (int j = 0; j < 32; ++j) sts_f32(t + j * 512, v[j]);
  }
  __device__ void finish(State&, int, int, int, int, int) const {}
  __device__ void store(const uint8_t* smem, int a0, int b0, int split) const {
    if (accumulate)
      tma_reduce_add_2d(&map, smem, a0, b0);
    else
      tma_store_3d(&map, smem, a0, b0, split);
  }
};

// Fused SwiGLU. The gate/up weight is stored interleaved in 64-row groups:
// tile rows [0,64) are gate rows of features f0..f0+63 and rows [64,128) the
// matching up rows, f0 = a_row0 / 2. out[m][f] = silu(g) * u; map [M][F] bf16,
// box {64, BN}. Per chunk, the half's 128 threads park gate and up in a
// [32][128] fp32 exchange buffer, then each thread computes 16 outputs
// (feature t % 64, 16 consecutive tokens): all threads share the MUFU work.
template <int BN>
struct EpiSwiGLU {
  CUtensorMap map;
  static constexpr bool kTmaStore = true;
  static constexpr int kPasses = 1;
  template <class S> __device__ void next_pass(S&, int, int, int, int) const {}
  static constexpr int kTileBytes = (BN < 64 ? 64 : BN) * 64 * 2;
  struct State {};
  __device__ void operator()(State&, uint8_t* smem, int, int, int, int r, int half, int c0,
                             const float (&v)[32]) const {
    __nv_bfloat16* tile = reinterpret_cast<__nv_bfloat16*>(smem);                       // [BN][64]
    float* xch = reinterpret_cast<float*>(smem + kTileBytes) + half * 32 * 128;          // [32][128]
    const uint32_t xa = smem_u32(xch) + r * 4;
#pragma unroll
    for (int j = 0; j < 32; ++j) sts_f32(xa + j * 512, v[j]);
    half_bar_sync(half);
    const int t = r;
    const int f = t & 63, j0 = (t >> 6) * 16;
    if (c0 < BN) {
      float gte[16], up[16];  // all loads first, then the tile stores
      const uint32_t xr = smem_u32(xch) + (j0 * 128 + f) * 4, tr = smem_u32(tile) + ((c0 + j0) * 64 + f) * 2;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        gte[j] = lds_f32(xr + j * 512);
        up[j] = lds_f32(xr + j * 512 + 256);
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) sts_bf16(tr + j * 128, f2bf(__fdividef(gte[j], 1.0f + __expf(-gte[j])) * up[j]));
    }
    half_bar_sync(half);
  }
  __device__ void finish(State&, int, int, int, int, int) const {}
  __device__ void store(const uint8_t* smem, int a0, int b0, int) const { tma_store_2d(&map, smem, a0 / 2, b0); }
};

// Decode QKV projection with RoPE + KV-cache append (swap-AB: tile rows = 128
// qkv features a0.., columns = batch rows b0..). The tile is staged as bf16 —
// the rounding of the unfused qkv output — then, after one barrier, the 256
// epilogue threads rotate pairs (i, i + hd/2) of every head in the tile with
// the position's (cos, sin) from the rope table and write q rows to q_out and
// the new token's K / V straight into its pool page. A warp covers the i of
// one (row, head), so every global store is a contiguous 64-byte run.
template <int BN>
struct EpiRopeKV {
  __nv_bfloat16* q_out;
  KvPoolView pool;
  const int* slot;
  const int* pos;
  const float2* cs;
  int layer, H, KVH, hd, M;
  __nv_bfloat16* k_out = nullptr;  // optional packed K / V [M, KVH, hd] (prefill / scoring attention)
  __nv_bfloat16* v_out = nullptr;
  int use_pool = 1;                // write the new K / V into the paged pool
  static constexpr bool kTmaStore = false;
  static constexpr int kPasses = 1;
  template <class S> __device__ void next_pass(S&, int, int, int, int) const {}
  // BN <= 64 (decode): the (cos, sin) of every column's position are fetched
  // into shared memory by the prologue, under the mainloop, instead of by
  // dependent loads after it — [column][pair index], hd / 2 <= 64 pairs.
  static constexpr bool kCache = BN <= 64;
  static constexpr int kSmemExtra = kCache ? BN * 64 * 8 : 0;
  struct State {
    uint8_t* smem;
    int pj, pagej;  // lane j: position and pool page of this warp's j-th column (prologue)
    const float2* cs_s;
  };
  __device__ void prologue(State& st, int, int b0, uint8_t* extra) const {
    const int ew = (threadIdx.x >> 5) - 2, lane = threadIdx.x & 31;
    const int nb = min(BN, M - b0);
    const int bl = ew + 8 * lane;
    st.pj = st.pagej = 0;
    if (bl < nb) {
      st.pj = pos[b0 + bl];
      if (use_pool) st.pagej = pool.block_table[slot[b0 + bl] * pool.bt_stride + st.pj / pool.page_tokens];
    }
    if constexpr (kCache) {
      float2* cache = reinterpret_cast<float2*>(extra);
      st.cs_s = cache;
      const int hh = hd >> 1;
      const int ncol = (nb - ew + 7) >> 3;
      float2 c[BN / 8][2];
#pragma unroll
      for (int k = 0; k < BN / 8; ++k) {  // all loads in flight together
        const int p = __shfl_sync(0xffffffffu, st.pj, k);
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2)
          if (k < ncol && lane + 32 * h2 < hh) c[k][h2] = __ldg(cs + p * hh + lane + 32 * h2);
      }
#pragma unroll
      for (int k = 0; k < BN / 8; ++k)
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2)
          if (k < ncol && lane + 32 * h2 < hh) cache[(ew + 8 * k) * 64 + lane + 32 * h2] = c[k][h2];
      __syncwarp();  // each warp reads back only its own columns
    }
  }
  __device__ void operator()(State& st, uint8_t* smem, int, int, int, int r, int, int c0,
                             const float (&v)[32]) const {
    st.smem = smem;
    __nv_bfloat16* tile = reinterpret_cast<__nv_bfloat16*>(smem);
    const uint32_t t = smem_u32(tile) + (c0 * 128 + r) * 2;
#pragma unroll
    for (int j = 0; j < 32; ++j) sts_bf16(t + j * 256, f2bf(v[j]));
  }
  __device__ void finish(State& st, int a0, int b0, int, int, int) const {
    epi_bar_sync();
    const uint32_t tile_s = smem_u32(st.smem);  // staged tile [column][128] bf16 (shared-space accesses below)
    const int ew = (threadIdx.x >> 5) - 2;      // epilogue warp 0..7: columns ew, ew + 8, ...
    const int lane = threadIdx.x & 31;
    const int hh = hd >> 1;
    const int nb = min(BN, M - b0);
    const int pj = st.pj, pagej = st.pagej;
    const int ncol = (nb - ew + 7) >> 3;  // columns of this warp
    // (1) rotate the q / k pairs of this warp's columns in place; per pair
    // slot k2 (lane, lane + 32) the feature is column-independent
    int fl2[2], i2[2], rot2[2];
#pragma unroll
    for (int k2 = 0; k2 < 2; ++k2) {
      const int pr = lane + 32 * k2;
      i2[k2] = pr % hh;
      fl2[k2] = (pr / hh) * hd + i2[k2];  // tile-local feature of the pair's low element
      rot2[k2] = (a0 + fl2[k2]) / hd < H + KVH;
    }
    constexpr int kG = 4;  // columns whose (cos, sin) and tile values are loaded together
    for (int k0 = 0; k0 < ncol; k0 += kG) {
      float2 c[kG][2];
      __nv_bfloat16 t1[kG][2], t2[kG][2];
#pragma unroll
      for (int kk = 0; kk < kG; ++kk) {
        const int k = min(k0 + kk, ncol - 1);
        const int p = __shfl_sync(0xffffffffu, pj, k);
#pragma unroll
        for (int k2 = 0; k2 < 2; ++k2) {
          if constexpr (kCache)
            c[kk][k2] = lds_f2(smem_u32(st.cs_s) + ((ew + 8 * k) * 64 + i2[k2]) * 8);
          else
            c[kk][k2] = rot2[k2] ? __ldg(cs + p * hh + i2[k2]) : make_float2(1.f, 0.f);
          const uint32_t ta = tile_s + ((ew + 8 * k) * 128 + fl2[k2]) * 2;
          t1[kk][k2] = lds_bf16(ta);
          t2[kk][k2] = lds_bf16(ta + hh * 2);
        }
      }
#pragma unroll
      for (int kk = 0; kk < kG; ++kk) {
        if (k0 + kk >= ncol) break;
        const int bl = ew + 8 * (k0 + kk);
#pragma unroll
        for (int k2 = 0; k2 < 2; ++k2) {
          if (!rot2[k2]) continue;  // v: stored as computed
          float r1, r2;
          rope_pair(__bfloat162float(t1[kk][k2]), __bfloat162float(t2[kk][k2]), c[kk][k2].x, c[kk][k2].y, r1, r2);
          const uint32_t ta = tile_s + (bl * 128 + fl2[k2]) * 2;
          sts_bf16(ta, f2bf(r1));
          sts_bf16(ta + hh * 2, f2bf(r2));
        }
      }
    }
    __syncwarp();
    // (2) 16-byte copies out: per column 16 chunks of 8 features, each inside
    // one head — q rows are contiguous in q_out, k / v rows go to the token's
    // pool page slot (and / or the packed buffers)
    __nv_bfloat16* pool_base = reinterpret_cast<__nv_bfloat16*>(pool.base);
    const size_t page_elems = pool.page_bytes / 2, layer_off = static_cast<size_t>(layer) * pool.layer_bytes / 2;
    for (int it = 0; it * 2 < ncol; ++it) {
      const int k = it * 2 + (lane >> 4);
      const int kc = min(k, ncol - 1);
      const int p = __shfl_sync(0xffffffffu, pj, kc), pg = __shfl_sync(0xffffffffu, pagej, kc);
      if (k >= ncol) continue;
      const int bl = ew + 8 * k, b = b0 + bl;
      const int f = (lane & 15) * 8, feat = a0 + f, head = feat / hd, e = feat - head * hd;
      const uint4 v = lds_v4(tile_s + (bl * 128 + f) * 2);
      if (head < H) {
        *reinterpret_cast<uint4*>(q_out + static_cast<size_t>(b) * H * hd + feat) = v;
      } else {
        const bool is_v = head >= H + KVH;
        const int kh = head - H - (is_v ? KVH : 0);
        if (use_pool)
          *reinterpret_cast<uint4*>(pool_base + static_cast<size_t>(pg) * page_elems + layer_off +
                                    (kh * 2 + (is_v ? 1 : 0)) * pool.page_tokens * hd +
                                    (p % pool.page_tokens) * hd + e) = v;
        __nv_bfloat16* packed = is_v ? v_out : k_out;
        if (packed) *reinterpret_cast<uint4*>(packed + (static_cast<size_t>(b) * KVH + kh) * hd + e) = v;
      }
    }
  }
  __device__ void store(const uint8_t*, int, int, int) const {}
};

}  // namespace fpk
