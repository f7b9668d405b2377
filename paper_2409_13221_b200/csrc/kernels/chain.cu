// fuseplan-b200 — the decode layer's GEMM chain as ONE persistent kernel.
//
// A decode step at gpt2s width is latency-bound: per layer the O projection,
// two residual-add + RMSNorms, gate/up (SwiGLU), down and the next layer's
// QKV (+ RoPE + KV append) were six dependent launches of ~3-10 us each
// against ~3 us of weight streaming (profiles/r01_step_trace_*.txt). Here one
// grid of 148 CTAs (one per SM) runs the whole chain
//
//   P0  O-proj split-K partials      parts[s][b][:] = attn[b] . Wo[:, K_s]
//   P1  residual + RMSNorm (ln2)     x[b] += sum_s parts[s][b]; h[b] = norm(x[b])
//   P2  gate/up + SwiGLU             act[b] = silu(h Wg) * (h Wu)
//   P3  down split-K partials        parts[s][b][:] = act[b] . Wd[:, K_s]
//   P4  residual + RMSNorm (ln1' / lnf)
//   P5  next layer's QKV + RoPE + KV append (EpiRopeKV)        (not after the last layer)
//
// with a grid-wide counter barrier between phases instead of a kernel
// boundary. Per CTA the warps are the GEMM's (tc_gemm_kernel) plus one:
//   warp 0      weight producer: TMA of the weight tiles of every phase,
//               in consumption order, as far ahead as the ring allows — the
//               weights do not depend on the activations, so the next phase's
//               weights stream while the current phase and the barrier run;
//   warp 10     activation producer: after the phase's input barrier, the
//               activation tiles into the same ring stages (one mbarrier per
//               stage; its tx count covers both halves);
//   warp 1      MMA issuer (tcgen05.mma, fp32 accumulators in TMEM, two
//               buffers so a tile's epilogue overlaps the next tile's MMAs);
//   warps 2..9  epilogues of the GEMM phases and the norm rows of P1 / P4.
// Numerics are the separate kernels' exactly: the same split-K factors
// (gemm_splits), the same tensor-core dot products, the partials summed in
// split order, and add_norm's reduction tree replayed with virtual threads —
// a row's bits do not change, and do not depend on the batch.
#include <cudaTypedefs.h>

#include <algorithm>
#include <stdexcept>
#include <type_traits>

#include "gemm.cuh"
#include "ops.h"

namespace fpk {

namespace {

constexpr int kChainThreads = kGemmThreads + 32;  // + the activation producer (warp 10)
constexpr int kChainSmem = 225 * 1024;  // + ~0.5 KB static: within the 227 KB per-block limit

__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// After a CTA barrier over the writers: the release orders their generic
// writes (cumulativity through bar.sync); the proxy fence covers the TMA
// (async proxy) reads of the consumers.
__device__ __forceinline__ void grid_arrive(int* cnt) {
  fence_proxy_async_global();
  asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(cnt) : "memory");
}

__device__ __forceinline__ void grid_wait(const int* cnt, int target) {
  int seen = 0;
  do {
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(seen) : "l"(cnt) : "memory");
  } while (seen < target);
  fence_proxy_async_global();
}

// The split-K phases' epilogue: stores from registers (partial_store below).
struct NoEpi {
  struct State {};
  static constexpr bool kTmaStore = false;
  __device__ void finish(State&, int, int, int, int, int) const {}
};

struct ChainPhase {
  int a_tiles;   // 128-row weight tiles
  int splits;    // K splits
  int kb_per;    // K blocks per split
  int k_blocks;  // total K blocks
};

template <int BN>
struct ChainArgs {
  CUtensorMap w[4];  // A operands: Wo [d, ao], Wgu [2F, d], Wd [d, F], Wqkv' [qw', d]
  CUtensorMap in[4]; // B operands: attn [B, ao], h [B, d], act [B, F], h [B, d]
  EpiSwiGLU<BN> swiglu;
  EpiRopeKV<BN> rope;
  ChainPhase ph[4];  // GEMM phases P0, P2, P3, P5
  float* parts;      // [splits][B][d]
  float* x;          // residual stream [B][d]
  __nv_bfloat16* h;  // norm output [B][d]
  const float* gain[2];  // P1 (ln2), P4 (next ln1 or lnf)
  int B, d;
  int has_qkv;
  int* counters;  // 8 ints: phase counters 0..4, exit; zero at launch, left zero
  unsigned long long* trace;  // optional: 16 globaltimer stamps per CTA (tools/step_trace.py)
};

// Item sequence of one CTA: GEMM phases g = 0..3 (P0, P2, P3, P5), tiles
// t = cta, cta + G, ... of phase g (t -> a-tile, b-tile, split), K blocks of
// the tile's split. The three roles walk it in the same order.
template <int BN, class F>
__device__ __forceinline__ void for_tiles(const ChainArgs<BN>& a, int g, int nb, F&& f) {
  const ChainPhase& p = a.ph[g];
  const int total = p.a_tiles * nb * p.splits;
  for (int t = blockIdx.x; t < total; t += gridDim.x) {
    const int at = t % p.a_tiles;
    const int rest = t / p.a_tiles;
    const int bt = rest % nb;
    const int split = rest / nb;
    const int kb0 = split * p.kb_per;
    const int kb1 = min(p.k_blocks, kb0 + p.kb_per);
    f(at, bt, split, kb0, kb1);
  }
}

template <int BN>
struct ChainCfg {
  static constexpr int kStageBytes = kTileA + BN * kBK * 2;
  // epilogue staging: EpiSwiGLU (tile + exchange) / EpiRopeKV (tile + cos/sin cache)
  static constexpr int kSwi = EpiSwiGLU<BN>::kTileBytes + 2 * 32 * 128 * 4;
  // the RoPE epilogue stages [max(BN, 64)][128] bf16 (its zero chunks past BN
  // land there too), its cos/sin cache follows
  static constexpr int kRopeTile = (BN < 64 ? 64 : BN) * 128 * 2;
  static constexpr int kRope = kRopeTile + EpiRopeKV<BN>::kSmemExtra;
  static constexpr int kStaging = ((kSwi > kRope ? kSwi : kRope) + 1023) & ~1023;
  static constexpr int kStages = (kChainSmem - 1024 - kStaging - 1024) / kStageBytes;
  // two accumulator buffers of >= 32 columns (an epilogue chunk reads 32)
  static constexpr uint32_t kAccCols = BN <= 32 ? 32 : BN;
  static constexpr uint32_t kTmemCols = 2 * kAccCols;
};

// Residual add + RMSNorm of rows `row0` and (if row1 >= 0) `row1` with the 256
// epilogue threads standing in for add_norm_kernel's blockDim = 32 * ceil(d /
// 128) threads (virtual thread j = 256 k + t): the same float4 per virtual
// thread, the same warp-then-warp-order reduction — the same bits. The loads
// of both rows are in flight together.
__device__ __forceinline__ void chain_norm_rows(float* x, const float* parts, int ns, size_t ps, const float* gain,
                                                __nv_bfloat16* y, int d, int row0, int row1, float (*red)[32]) {
  const int t = static_cast<int>(threadIdx.x) - 64;  // 0..255
  const int d4 = d >> 2;
  const int nthr = ((d4 + 31) / 32) * 32, nw = nthr >> 5;
  const int rounds = (nthr + 255) / 256;
  const size_t ps4 = ps >> 2;
  float4 v[2][4];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int row = q ? row1 : row0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      v[q][k] = make_float4(0.f, 0.f, 0.f, 0.f);
      const int j = 256 * k + t;
      if (row >= 0 && k < rounds && j < d4) {
        const float4* xr = reinterpret_cast<const float4*>(x + static_cast<size_t>(row) * d);
        const float4* pr = reinterpret_cast<const float4*>(parts + static_cast<size_t>(row) * d);
        float4 a = __ldcg(xr + j);
        float4 p[8];
#pragma unroll
        for (int s = 0; s < 8; ++s)
          if (s < ns) p[s] = __ldcg(pr + s * ps4 + j);  // written by other CTAs: L2
#pragma unroll
        for (int s = 0; s < 8; ++s)
          if (s < ns) a.x += p[s].x, a.y += p[s].y, a.z += p[s].z, a.w += p[s].w;
        v[q][k] = a;
      }
    }
  }
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int row = q ? row1 : row0;
    if (row < 0) continue;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int j = 256 * k + t;
      if (k < rounds && j < d4 && ns > 0) reinterpret_cast<float4*>(x + static_cast<size_t>(row) * d)[j] = v[q][k];
      if (k < rounds && j < nthr) {
        const float ws = warp_sum(sumsq4(v[q][k]));
        if ((t & 31) == 0) red[q][(256 * k + t) >> 5] = ws;
      }
    }
  }
  epi_bar_sync();
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int row = q ? row1 : row0;
    if (row < 0) continue;
    float tot = (static_cast<int>(lane_id()) < nw) ? red[q][lane_id()] : 0.f;
    tot = warp_sum(tot);
    const float inv = rsqrtf(tot / d + kNormEps);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int j = 256 * k + t;
      if (k < rounds && j < d4) {
        const float4 g = reinterpret_cast<const float4*>(gain)[j];
        reinterpret_cast<uint2*>(y + static_cast<size_t>(row) * d)[j] = norm_scale4(v[q][k], inv, g);
      }
    }
  }
  epi_bar_sync();  // red[] is reused by the next rows
}

__device__ __forceinline__ void stamp(unsigned long long* tr, int k) {
  if (tr) tr[k] = gtime();
}

template <int BN>
__global__ void __launch_bounds__(kChainThreads, 1) decode_chain_kernel(const __grid_constant__ ChainArgs<BN> a) {
  using C = ChainCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* staging = smem + C::kStages * C::kStageBytes;
  __shared__ __align__(8) uint64_t full_bar[C::kStages];
  __shared__ __align__(8) uint64_t empty_bar[C::kStages];
  __shared__ __align__(8) uint64_t acc_full[2];
  __shared__ __align__(8) uint64_t acc_empty[2];
  __shared__ uint32_t tmem_base_smem;
  __shared__ float red[2][32];

  const uint32_t warp = warp_id();
  const int nb = (a.B + BN - 1) / BN;
  const int G = gridDim.x;
  const int n_gemm = a.has_qkv ? 4 : 3;
  unsigned long long* tr = a.trace ? a.trace + 16ull * blockIdx.x : nullptr;
  if (threadIdx.x == 0) stamp(tr, 0);
  pdl_trigger();

  if (warp == 0 && elect_one()) {
    for (int i = 0; i < 4; ++i) {
      tma_prefetch_desc(&a.w[i]);
      tma_prefetch_desc(&a.in[i]);
    }
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 256);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<C::kTmemCols>(&tmem_base_smem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_smem;

  if (warp == 0) {
    // weight producer: every stage's arrive.expect_tx (A + B bytes) and its A half
    if (elect_one()) {
      int i = 0;
      for (int g = 0; g < n_gemm; ++g)
        for_tiles(a, g, nb, [&](int at, int, int, int kb0, int kb1) {
          for (int kb = kb0; kb < kb1; ++kb, ++i) {
            const int s = i % C::kStages;
            mbar_wait(&empty_bar[s], ((i / C::kStages) & 1) ^ 1);
            mbar_arrive_expect_tx(&full_bar[s], C::kStageBytes);
            tma_load_2d(smem + s * C::kStageBytes, &a.w[g], &full_bar[s], kb * kBK, at * 128);
          }
        });
    }
  } else if (warp == 10) {
    // activation producer: the B half of every stage, once the phase's input exists
    if (elect_one()) {
      int i = 0;
      for (int g = 0; g < n_gemm; ++g) {
        if (g == 0)
          pdl_wait();  // attention output of the previous kernel
        else
          grid_wait(a.counters + (g == 1 ? 1 : g == 2 ? 2 : 4), G);  // P1 / P2 / P4 done everywhere
        if (g == 1) stamp(tr, 14);
        if (g == 3) stamp(tr, 15);
        for_tiles(a, g, nb, [&](int, int bt, int, int kb0, int kb1) {
          for (int kb = kb0; kb < kb1; ++kb, ++i) {
            const int s = i % C::kStages;
            mbar_wait(&empty_bar[s], ((i / C::kStages) & 1) ^ 1);
            tma_load_2d(smem + s * C::kStageBytes + kTileA, &a.in[g], &full_bar[s], kb * kBK, bt * BN);
          }
        });
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      constexpr uint32_t idesc = idesc_bf16(128, BN);
      const uint64_t da = sdesc_k128(smem_u32(smem)), db = sdesc_k128(smem_u32(smem) + kTileA);
      int i = 0, tile = 0;
      for (int g = 0; g < n_gemm; ++g)
        for_tiles(a, g, nb, [&](int, int, int, int kb0, int kb1) {
          const int buf = tile & 1;
          if (tile >= 2) mbar_wait(&acc_empty[buf], ((tile >> 1) - 1) & 1);
          tc_fence_after();
          const uint32_t acc = tmem + buf * C::kAccCols;
          for (int kb = kb0; kb < kb1; ++kb, ++i) {
            const int s = i % C::kStages;
            mbar_wait(&full_bar[s], (i / C::kStages) & 1);
            tc_fence_after();
            const uint64_t off = static_cast<uint64_t>((s * C::kStageBytes) >> 4);
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k)
              tc_mma_bf16(acc, da + off + 2 * k, db + off + 2 * k, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
            tc_commit(&empty_bar[s]);
          }
          tc_commit(&acc_full[buf]);
          ++tile;
        });
    }
    __syncwarp();
  } else {
    // epilogue warps 2..9
    const int quarter = warp & 3;
    const int half = (static_cast<int>(warp) - 2) >> 2;
    const int r = quarter * 32 + lane_id();
    const size_t ps = static_cast<size_t>(a.B) * a.d;  // split stride of the partials
    pdl_wait();
    int tile = 0;
    const int acc_stamp[4] = {1, 5, 8, 12};
    auto gemm_phase = [&](int g, const auto& epi, auto&& store_chunk) {
      bool first = true;
      using Epi = std::remove_cvref_t<decltype(epi)>;
      typename Epi::State st{};
      for_tiles(a, g, nb, [&](int at, int bt, int split, int, int) {
        const int buf = tile & 1;
        const int a0 = at * 128, b0 = bt * BN;
        if constexpr (EpiHasPrologue<Epi>::value) epi.prologue(st, a0, b0, staging + C::kRopeTile);
        mbar_wait(&acc_full[buf], (tile >> 1) & 1);
        if (first && threadIdx.x == 64) stamp(tr, acc_stamp[g]);
        first = false;
        tc_fence_after();
        const uint32_t acc = tmem + buf * C::kAccCols + (static_cast<uint32_t>(quarter * 32) << 16);
#pragma unroll 1
        for (int c0 = 32 * half; c0 < ((BN + 63) / 64) * 64; c0 += 64) {
          float v[32];
          if (c0 < BN) {
            tmem_ld32(acc + c0, v);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = 0.f;
          }
          store_chunk(st, a0, b0, split, c0, v);
        }
        tc_fence_before();
        mbar_arrive(&acc_empty[buf]);  // the accumulator is in registers / staging now
        epi.finish(st, a0, b0, split, r, half);
        if constexpr (Epi::kTmaStore) {
          fence_async_smem();
          epi_bar_sync();
          if (threadIdx.x == 64) {
            epi.store(staging, a0, b0, split);
            bulk_commit_wait();  // complete (not only read): the barrier below publishes it
          }
        }
        epi_bar_sync();  // the staging area is free for the next tile
        ++tile;
      });
    };
    // split-K partials straight from registers: for each batch column of the
    // chunk, the warp's 32 lanes store 32 consecutive features (128 B)
    const NoEpi none{};
    auto partial_store = [&](NoEpi::State&, int a0, int b0, int split, int c0, const float (&v)[32]) {
      float* out = a.parts + static_cast<size_t>(split) * ps + a0 + r;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int b = b0 + c0 + j;
        if (c0 + j < BN && b < a.B) out[static_cast<size_t>(b) * a.d] = v[j];
      }
    };
    const int arrive_stamp[5] = {2, 4, 6, 9, 11};
    auto arrive = [&](int phase) {
      epi_bar_sync();
      if (threadIdx.x == 64) {
        grid_arrive(a.counters + phase);
        stamp(tr, arrive_stamp[phase]);
      }
    };
    auto norm_phase = [&](int phase, int ns, const float* gain) {
      if (threadIdx.x == 64) {
        grid_wait(a.counters + phase - 1, G);
        stamp(tr, phase == 1 ? 3 : 10);
      }
      epi_bar_sync();
      for (int row = blockIdx.x; row < a.B; row += 2 * G)
        chain_norm_rows(a.x, a.parts, ns, ps, gain, a.h, a.d, row, row + G < a.B ? row + G : -1, red);
      arrive(phase);
    };

    gemm_phase(0, none, partial_store);  // P0
    arrive(0);
    norm_phase(1, a.ph[0].splits, a.gain[0]);  // P1
    // (the epilogues are used in place: the SwiGLU store's tensor map must stay in parameter space)
    gemm_phase(1, a.swiglu, [&](typename EpiSwiGLU<BN>::State& st, int a0, int b0, int split, int c0,
                                const float (&v)[32]) { a.swiglu(st, staging, a0, b0, split, r, half, c0, v); });  // P2
    arrive(2);
    if (threadIdx.x == 64) {
      grid_wait(a.counters + 2, G);  // P3's partials overwrite P0's: P1 has read them
      stamp(tr, 7);
    }
    epi_bar_sync();
    gemm_phase(2, none, partial_store);  // P3
    arrive(3);
    norm_phase(4, a.ph[2].splits, a.gain[1]);  // P4
    if (a.has_qkv)
      gemm_phase(3, a.rope, [&](typename EpiRopeKV<BN>::State& st, int a0, int b0, int split, int c0,
                                const float (&v)[32]) { a.rope(st, staging, a0, b0, split, r, half, c0, v); });  // P5
    if (threadIdx.x == 64) stamp(tr, 13);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<C::kTmemCols>(tmem);
  // the last CTA out resets the counters for the next launch
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(a.counters + 5, 1) == G - 1) {
      for (int i = 0; i < 6; ++i) atomicExch(a.counters + i, 0);
    }
  }
}

}  // namespace

// Host: maps and launch (gemm.cu's map helpers are file-local; chain_maps.cu
// builds them through the shared encode cache).
CUtensorMap chain_operand_map(const void* ptr, int rows, int k, int box_rows);
CUtensorMap chain_out_map_bf16(const void* ptr, int rows, int cols, int ld, int box_cols, int box_rows);
int chain_pick_bn(int M, int a_tiles);

template <int BN>
static void launch_chain(const DecodeChain& c, cudaStream_t st) {
  using C = ChainCfg<BN>;
  static_assert(C::kStages >= 2, "chain ring too shallow");
  ChainArgs<BN> a{};
  const int d = c.d, F = c.F, ao = c.ao;
  a.w[0] = chain_operand_map(c.wo, d, ao, 128);
  a.w[1] = chain_operand_map(c.wgu, 2 * F, d, 128);
  a.w[2] = chain_operand_map(c.wd, d, F, 128);
  a.in[0] = chain_operand_map(c.attn, c.B, ao, BN);
  a.in[1] = chain_operand_map(c.h, c.B, d, BN);
  a.in[2] = chain_operand_map(c.act, c.B, F, BN);
  a.in[3] = a.in[1];
  a.has_qkv = c.wqkv != nullptr;
  const int qw = (c.H + 2 * c.KVH) * c.hd;
  if (a.has_qkv) a.w[3] = chain_operand_map(c.wqkv, qw, d, 128);
  else a.w[3] = a.w[0];
  auto phase = [](int N, int K, int splits) {
    ChainPhase p;
    p.a_tiles = (N + 127) / 128;
    p.k_blocks = K / kBK;
    splits = std::max(1, std::min(splits, p.k_blocks));
    p.kb_per = (p.k_blocks + splits - 1) / splits;
    p.splits = (p.k_blocks + p.kb_per - 1) / p.kb_per;
    return p;
  };
  a.ph[0] = phase(d, ao, gemm_splits(d, ao));
  a.ph[1] = phase(2 * F, d, 1);
  a.ph[2] = phase(d, F, gemm_splits(d, F));
  a.ph[3] = phase(qw, d, 1);
  if (a.ph[0].splits > 8 || a.ph[2].splits > 8) throw std::invalid_argument("decode_chain: at most 8 splits");
  a.swiglu = EpiSwiGLU<BN>{chain_out_map_bf16(c.act, c.B, F, F, 64, BN)};
  if (a.has_qkv) {
    a.rope = EpiRopeKV<BN>{c.q_out, c.pool, c.slot, c.pos, c.cs, c.layer + 1, c.H, c.KVH, c.hd, c.B};
    a.rope.pool.kv_map = nullptr;
  }
  a.parts = c.parts;
  a.x = c.x;
  a.h = c.h;
  a.gain[0] = c.gain_mlp;
  a.gain[1] = c.gain_next;
  a.B = c.B;
  a.d = d;
  a.counters = c.counters;

  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(decode_chain_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, kChainSmem);
    attr = true;
  }
  cudaLaunchConfig_t cfg{};
  int tiles = 0;
  for (int g = 0; g < (a.has_qkv ? 4 : 3); ++g)
    tiles = std::max(tiles, a.ph[g].a_tiles * a.ph[g].splits * ((c.B + BN - 1) / BN));
  const int ctas = std::max(1, std::min(c.ctas, tiles));  // idle SMs stay free for the scoring stream
  a.trace = trace_slot(3, ctas, 16);
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(kChainThreads);
  cfg.dynamicSmemBytes = kChainSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr_pdl[1];
  attr_pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr_pdl[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr_pdl;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, decode_chain_kernel<BN>, a);
  if (e != cudaSuccess) throw std::runtime_error(std::string("decode_chain launch: ") + cudaGetErrorString(e));
  fpk::count_launch();
}

bool decode_chain(const DecodeChain& c, cudaStream_t st) {
  if (c.d % 128 || c.d > 4096 || c.F % 64 || c.ao % 64 || 128 % c.hd) return false;
  if (c.B < 1 || c.B > 512) return false;
  switch (chain_pick_bn(c.B, (2 * c.F + 127) / 128)) {
    case 16: launch_chain<16>(c, st); break;
    case 32: launch_chain<32>(c, st); break;
    case 64: launch_chain<64>(c, st); break;
    case 128: launch_chain<128>(c, st); break;
    default: launch_chain<256>(c, st); break;
  }
  return true;
}

}  // namespace fpk
