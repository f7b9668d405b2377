// fuseplan-b200 — persistent tcgen05 GEMM on SM pairs (cta_group::2) for the
// packed forwards.
//
// A cluster of two CTAs (two SMs) owns a 256 x 256 output tile: CTA r holds
// weight rows [a0 + 128 r, +128) (UMMA A) and token rows [b0 + 128 r, +128)
// (UMMA B) of each 64-wide K block in its own shared memory; the even CTA's
// elected thread issues tcgen05.mma.cta_group::2 (M 256, N 256), which reads
// both CTAs' halves, and CTA r's TMEM receives D rows [128 r, +128) x all 256
// token columns. Per SM this halves the B bytes loaded and read per MMA
// compared with the one-SM 128 x 256 tile — the shared-memory and L2 traffic
// that holds the one-SM kernel's mainloops at ~70 % of the MMA rate.
//
// Protocol (the same as CUTLASS's 2x1SM pipelines):
//   * both CTAs' producers wait their own `empty` slot, then TMA their halves
//     with .cta_group::2, completing bytes on the EVEN CTA's `full` barrier
//     (mapa to rank 0); only the even producer arms it (expect_tx of both
//     halves);
//   * the even MMA thread waits `full`, issues 4 MMAs per K block and commits
//     to `empty` of both CTAs (multicast); per tile it commits `acc_full` of
//     both CTAs;
//   * each CTA's 8 epilogue warps drain their own TMEM (same epilogue functors
//     as the one-SM kernel, BN = 256) and arrive on the even CTA's
//     `acc_empty` (512 arrivals: both CTAs' epilogue threads).
// Same per-element K order as the other GEMM kernels.
#pragma once

#include "gemm_persist.cuh"

namespace fpk {

// The shared::cluster address of the same object in the pair's even CTA.
__device__ __forceinline__ uint32_t peer0(const void* p) { return mapa_shared(smem_u32(p), 0); }

__device__ __forceinline__ void tma_load_2d_pair(void* smem_dst, const CUtensorMap* map, uint32_t bar_even,
                                                 int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_even), "r"(c0), "r"(c1)
      : "memory");
}

template <uint32_t kCols>
__device__ __forceinline__ void tmem_alloc_pair(uint32_t* dst_smem) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "n"(kCols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
template <uint32_t kCols>
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols));
}

__device__ __forceinline__ void tc_mma_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// Arrive (once each) on `bar` at the same offset in both CTAs of the pair when
// this thread's prior tcgen05.mma complete.
__device__ __forceinline__ void tc_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}

__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

template <class Epi, int BN_ = 256>
struct PairCfg {
  static constexpr int BN = BN_;                             // MMA N (tokens per pair tile)
  static constexpr int kStageBytes = kTileA + (BN / 2) * kBK * 2;  // this CTA's A half + B half
  static constexpr int kStaging = EpiStaging<BN, Epi>::v + EpiSmemExtra<Epi>::value;
  static constexpr int kStages = (kPersistSmem - 1024 - kStaging - 256) / kStageBytes;
  static constexpr int kSmem = kStages * kStageBytes + kStaging + 1024 + 256;
  static constexpr uint32_t kAccCols = BN;
  static constexpr uint32_t kTmemCols = 2 * BN;
  static_assert(kStages >= 2, "pair GEMM: ring too shallow");
};

// Tiles: a_tiles = ceil(a_rows / 256) weight-row pairs, tokens in BNs.
template <class Epi, int BN_ = 256>
__global__ void __launch_bounds__(kGemmThreads, 1)
    tc_gemm_pair_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                        const PersistGeom g, const __grid_constant__ Epi epi) {
  using C = PairCfg<Epi, BN_>;
  constexpr int BN = C::BN;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* staging = smem + C::kStages * C::kStageBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(staging + C::kStaging);
  uint64_t* full_bar = bars;                    // [kStages] (used on the even CTA)
  uint64_t* empty_bar = bars + C::kStages;      // [kStages]
  uint64_t* acc_full = bars + 2 * C::kStages;   // [2]
  uint64_t* acc_empty = acc_full + 2;           // [2] (used on the even CTA)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const uint32_t warp = warp_id();
  const uint32_t rank = cluster_ctarank();  // 0: issues the MMAs
  const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
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
      mbar_init(&acc_empty[b], 2 * 32 * kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair<C::kTmemCols>(tmem_slot);
  tc_fence_before();
  cluster_sync();  // both CTAs' barriers initialised before any remote arrive / complete_tx
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int nkb = g.k_blocks;

  if (warp == 0) {
    if (elect_one()) {
      int it = 0;
      bool waited = false;
      for (int t = pair; t < g.n_tiles; t += n_pairs) {
        const int a_row0 = (t % g.a_tiles) * 256 + 128 * rank, b_row0 = (t / g.a_tiles) * BN + (BN / 2) * rank;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % C::kStages;
          mbar_wait(&empty_bar[s], ((it / C::kStages) & 1) ^ 1);
          uint8_t* sa = smem + s * C::kStageBytes;
          const uint32_t fb = peer0(&full_bar[s]);
          if (rank == 0) mbar_arrive_expect_tx(&full_bar[s], 2 * C::kStageBytes);
          if (!waited && !g.weight_is_a) {
            pdl_wait();
            waited = true;
          }
          tma_load_2d_pair(sa, &map_a, fb, kb * kBK, a_row0);
          if (!waited) {
            pdl_wait();
            waited = true;
          }
          tma_load_2d_pair(sa + kTileA, &map_b, fb, kb * kBK, b_row0);
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0 && elect_one()) {
      constexpr uint32_t idesc = idesc_bf16(256, BN);
      const uint64_t da = sdesc_k128(smem_u32(smem)), db = sdesc_k128(smem_u32(smem) + kTileA);
      int it = 0, i = 0;
      for (int t = pair; t < g.n_tiles; t += n_pairs, ++i) {
        const int buf = i & 1;
        mbar_wait(&acc_empty[buf], ((i >> 1) & 1) ^ 1);  // both CTAs drained this buffer (tile i - 2)
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
            tc_mma_pair(acc, da + off + 2 * k, db + off + 2 * k, idesc, (kb > 0 || k > 0) ? 1u : 0u);
          tc_commit_pair(&empty_bar[s]);
        }
        tc_commit_pair(&acc_full[buf]);
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
    for (int t = pair; t < g.n_tiles; t += n_pairs, ++i) {
      const int a_row0 = (t % g.a_tiles) * 256 + 128 * rank, b_row0 = (t / g.a_tiles) * BN;
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
        for (int c0 = 32 * half; c0 < BN; c0 += 64) {
          float v[32];
          tmem_ld32(acc + c0, v);
          epi(st, staging, a_row0, b_row0, 0, r, half, c0, v);
        }
      }
      tc_fence_before();
      mbar_arrive_cluster(peer0(&acc_empty[buf]));  // the even CTA's MMA may reuse this buffer
      epi.finish(st, a_row0, b_row0, 0, r, half);
      if constexpr (Epi::kTmaStore) {
        fence_async_smem();
        epi_bar_sync();
        if (threadIdx.x == 64) {
          epi.store(staging, a_row0, b_row0, 0);
          bulk_commit_wait_read();
        }
      }
      epi_bar_sync();
      if (threadIdx.x == 64) persist_stamp(g, i, 3);
    }
    if constexpr (EpiHasPost<Epi>::value) epi.post();
  }
  tc_fence_before();
  cluster_sync();  // no CTA leaves while its peer may still signal its barriers or read its shared memory
  if (warp == 1) tmem_dealloc_pair<C::kTmemCols>(tmem);
}

}  // namespace fpk
