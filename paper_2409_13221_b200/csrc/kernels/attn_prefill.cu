// fuseplan-b200 — tcgen05 causal attention over packed variable-length
// sequences: the prefill forward of the actor and the scoring forwards of the
// reference / critic / reward models (engine.cpp forward_packed), i.e. the
// attention inside RLHFuse's inference stage (reference genfuse.cpp:33-41
// schedules it; the math is standard causal softmax attention).
//
// One CTA owns a 128-query tile of one (sequence, head) and walks the causal
// key range in 64-key blocks:
//
//   S  = Q K^T            tcgen05.mma M=128 N=64  K=hd   (A, B K-major smem)
//   P  = exp2(S*c - m)    softmax warps: tcgen05.ld S -> registers -> bf16 P
//                         written to smem in the 128-byte-swizzled K-major
//                         layout the next MMA reads
//   O += P V              tcgen05.mma M=128 N=hd  K=64   (B = V MN-major)
//
// S (two 64-column buffers) and O (hd columns) live in TMEM; Q, K and V arrive by TMA
// (128 B swizzle, the K/V ring is two blocks deep). The running max is only
// moved when it grows by more than 2^8 (exp2 domain), so O is rescaled in TMEM
// (tcgen05.ld -> scale -> tcgen05.st) rarely: O and the row sum l always use
// the same stale max, so O / l is exact. Warp roles (192 threads):
//   warp 0      TMA producer (one elected lane)
//   warp 1      TMEM allocator + MMA issuer (one elected lane)
//   warps 2..5  softmax / rescale / epilogue: thread = query row = TMEM lane
// TMEM 256 columns and <= 114 KB smem per CTA: two CTAs per SM, so one CTA's
// softmax overlaps the other's MMAs.
#include <math.h>

#include <algorithm>
#include <stdexcept>

#include "ops.h"
#include "ptx.cuh"

namespace fpk {

CUtensorMap chain_operand_map(const void* ptr, int rows, int k, int box_rows);  // gemm.cu (bf16, SW128, box {64, rows})

namespace {

constexpr int kBM = 128;  // queries per CTA (UMMA M)
constexpr int kBN = 64;   // keys per block
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kRescaleThresh = 8.f;  // log2 units: P <= 2^8 between rescales
constexpr int kSoftmaxWarps = 4;  // one per TMEM lane quarter: thread = query row
constexpr int kThreads = 64 + 32 * kSoftmaxWarps;

template <int HD>
struct PrefillCfg {
  static constexpr int kQBytes = kBM * HD * 2;   // HD/64 swizzle boxes of [128][64]
  static constexpr int kKBytes = kBN * HD * 2;   // HD/64 boxes of [64][64]
  static constexpr int kPBytes = kBM * kBN * 2;  // one box [128][64]
  // K and V have rings of their own: a K block is released when its S MMA
  // retires, a V block when its PV MMA does, so loads run ahead of both.
  static constexpr int kStages = HD == 64 ? 4 : 2;
  static constexpr int kOffK = kQBytes;
  static constexpr int kOffV = kOffK + kStages * kKBytes;
  // P double-buffered where smem allows (two CTAs per SM): softmax writes P
  // of the next block while the tensor core still reads this one.
  static constexpr int kPBuf = HD == 64 ? 2 : 1;
  static constexpr int kOffP = kOffV + kStages * kKBytes;
  static constexpr int kOffBar = kOffP + kPBuf * kPBytes;
  static constexpr int kSmem = kOffBar + 256;  // two CTAs per SM: <= 113 KB each
  // TMEM: S double-buffered at columns 0 and 64 (S of the next block is
  // computed while softmax works on this one), O at column 128.
  static constexpr uint32_t kTmemCols = 256;
  static constexpr uint32_t kColO = 128;
};

// One work item: 128 queries [q0, q0 + 128) of head h in sequence [s0, s1).
struct Item {
  int h, s0, s1, q0, n_kb;
};
__device__ __forceinline__ Item get_item(int it, int H, const int* __restrict__ cu, const int* __restrict__ tiles) {
  const int t = it / H;
  Item x;
  x.h = it - t * H;
  const int seq = tiles[2 * t], qt = tiles[2 * t + 1];
  x.s0 = cu[seq];
  x.s1 = cu[seq + 1];
  x.q0 = x.s0 + qt * kBM;
  x.n_kb = (min(x.q0 + kBM, x.s1) - x.s0 + kBN - 1) / kBN;  // key blocks visible to some row
  return x;
}

// This CTA's item of round k: snake order over the cost-sorted list (even
// rounds left to right, odd rounds right to left) evens out per-CTA sums.
__device__ __forceinline__ int item_at(int k) {
  const int G = gridDim.x;
  return k * G + ((k & 1) ? G - 1 - static_cast<int>(blockIdx.x) : static_cast<int>(blockIdx.x));
}

// Walks this CTA's items; the next item's table entries are fetched one item
// early so the dependent loads (tiles -> cu) stay off the critical path.
struct ItemWalk {
  int k = 0, it, n_items, H;
  const int* cu;
  const int* tiles;
  Item cur, nxt;
  __device__ ItemWalk(int n, int h, const int* c, const int* t) : it(item_at(0)), n_items(n), H(h), cu(c), tiles(t) {
    if (it < n_items) cur = get_item(it, H, cu, tiles);
    prefetch();
  }
  __device__ void prefetch() {
    const int ni = item_at(k + 1);
    if (ni < n_items) nxt = get_item(ni, H, cu, tiles);
  }
  __device__ bool valid() const { return it < n_items; }
  __device__ void advance() {
    it = item_at(++k);
    cur = nxt;
    prefetch();
  }
};

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// MN-major operand, 128-byte swizzle: 64 contiguous MN elements per 128-byte
// row, K rows 128 B apart, 8-row K groups `sbo` apart, 64-element MN groups
// `lbo` apart (cute::UMMA canonical Major-MN SW128 layout).
__device__ __forceinline__ uint64_t sdesc_mn128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}

__device__ __forceinline__ void tmem_ld32_async(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]),
      "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]),
      "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void sts_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

// Persistent: CTA b takes one item per round of the (tile, head) list (tiles
// sorted most-keys-first, heads fastest) in snake order (item_at). The producer and MMA
// warps run ahead across item boundaries — the next item's Q / K / V loads
// and first S = Q K^T overlap this item's last softmax and its epilogue — and
// all barrier phases count blocks (g) or items (n) over the CTA's lifetime.
template <int HD>
__global__ void __launch_bounds__(kThreads, 2)
    attn_prefill_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_k,
                        const __grid_constant__ CUtensorMap map_v, int H, int KVH, int n_items,
                        const int* __restrict__ cu, const int* __restrict__ tiles, float scale_log2,
                        bf16* __restrict__ out, unsigned long long* __restrict__ trace) {
  // debug trace (fp_k_attn_prefill_trace): CTA 0's event times, [kind][64]
  unsigned long long* tr = blockIdx.x == 0 ? trace : nullptr;
  auto stamp = [&](int kind, int i) {
    if (tr && i < 64) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      tr[kind * 64 + i] = t;
    }
  };
  using C = PrefillCfg<HD>;
  pdl_trigger();
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023) != 0) __trap();  // 128 B swizzle atoms need 1 KB alignment
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  constexpr int KS = C::kStages;
  uint64_t* q_full = bars + 0;            // Q of item n landed
  uint64_t* q_free = bars + 1;            // every S MMA of item n retired (Q buffer reusable)
  uint64_t* s_full = bars + 2;            // [2] S of block g in TMEM buffer g & 1
  uint64_t* s_free = bars + 6;            // [2] softmax read S of block g
  constexpr int PB = C::kPBuf;
  uint64_t* p_full = bars + 4;            // [PB, <= 2] P of block g in buffer g % PB (O rescaled / read before it)
  uint64_t* pv_done = bars + 10;          // [PB] PV of block g retired (its P buffer free, O settled)
  uint64_t* k_full = bars + 12;           // [KS] K block g landed in stage g % KS
  uint64_t* k_empty = k_full + KS;        // [KS] S MMA of block g retired
  uint64_t* v_full = k_empty + KS;        // [KS] V block g landed
  uint64_t* v_empty = v_full + KS;        // [KS] PV MMA of block g retired
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(v_empty + KS);

  const uint32_t warp = warp_id();
  const int group = H / KVH;
  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&map_q);
    tma_prefetch_desc(&map_k);
    tma_prefetch_desc(&map_v);
    mbar_init(q_full, 1);
    mbar_init(q_free, 1);
    for (int s = 0; s < KS; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&s_free[b], 32 * kSoftmaxWarps);
    }
    for (int b = 0; b < PB; ++b) {
      mbar_init(&p_full[b], 32 * kSoftmaxWarps);
      mbar_init(&pv_done[b], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<C::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t sbase = smem_u32(smem);

  if (warp == 0) {
    if (elect_one()) {
      int g = 0, n = 0;
      for (ItemWalk w(n_items, H, cu, tiles); w.valid(); w.advance(), ++n) {
        const Item x = w.cur;
        if (n > 0) mbar_wait(q_free, (n - 1) & 1);
        mbar_arrive_expect_tx(q_full, C::kQBytes);
#pragma unroll
        for (int c = 0; c < HD / 64; ++c)
          tma_load_2d(smem + c * (kBM * 128), &map_q, q_full, x.h * HD + 64 * c, x.q0);
        const int kc = (x.h / group) * HD;
        for (int j = 0; j < x.n_kb; ++j, ++g) {
          const int s = g % KS;
          const uint32_t ph = ((g / KS) & 1) ^ 1;
          uint8_t* ks = smem + C::kOffK + s * C::kKBytes;
          uint8_t* vs = smem + C::kOffV + s * C::kKBytes;
          mbar_wait(&k_empty[s], ph);
          stamp(0, g);
          mbar_arrive_expect_tx(&k_full[s], C::kKBytes);
#pragma unroll
          for (int c = 0; c < HD / 64; ++c)
            tma_load_2d(ks + c * (kBN * 128), &map_k, &k_full[s], kc + 64 * c, x.s0 + j * kBN);
          mbar_wait(&v_empty[s], ph);
          mbar_arrive_expect_tx(&v_full[s], C::kKBytes);
#pragma unroll
          for (int c = 0; c < HD / 64; ++c)
            tma_load_2d(vs + c * (kBN * 128), &map_v, &v_full[s], kc + 64 * c, x.s0 + j * kBN);
        }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      constexpr uint32_t idesc_s = idesc_bf16(kBM, kBN);
      constexpr uint32_t idesc_o = idesc_bf16(kBM, HD) | (1u << 16);  // B (V) MN-major

      // O += P V for block gg; `first`: the item's first block (O starts from zero).
      // Its p_full also orders it after the previous item's epilogue read O.
      auto issue_pv = [&](int gg, bool first) {
        const int s = gg % KS;
        mbar_wait(&v_full[s], (gg / KS) & 1);
        const int b = gg % PB;
        mbar_wait(&p_full[b], (gg / PB) & 1);
        tc_fence_after();
        const uint32_t vs = sbase + C::kOffV + s * C::kKBytes;
        const uint64_t pa = sdesc_k128(sbase + C::kOffP + b * C::kPBytes);
#pragma unroll
        for (int kk = 0; kk < kBN / 16; ++kk)
          tc_mma_bf16(tmem + C::kColO, pa + 2 * kk, sdesc_mn128(vs + kk * 16 * 128, kBN * 128, 1024), idesc_o,
                      (first && kk == 0) ? 0u : 1u);
        tc_commit(&pv_done[b]);
        tc_commit(&v_empty[s]);
        stamp(2, gg);
      };
      int g = 0, n = 0;
      bool prev_first = false;
      for (ItemWalk w(n_items, H, cu, tiles); w.valid(); w.advance(), ++n) {
        const Item x = w.cur;
        mbar_wait(q_full, n & 1);
        for (int j = 0; j < x.n_kb; ++j, ++g) {
          const int s = g % KS;
          mbar_wait(&k_full[s], (g / KS) & 1);
          mbar_wait(&s_free[g & 1], ((g >> 1) & 1) ^ 1);  // softmax read S of block g - 2
          tc_fence_after();
          const uint32_t ks = sbase + C::kOffK + s * C::kKBytes;
#pragma unroll
          for (int c = 0; c < HD / 64; ++c) {
            const uint64_t qa = sdesc_k128(sbase + c * (kBM * 128));
            const uint64_t kb = sdesc_k128(ks + c * (kBN * 128));
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              tc_mma_bf16(tmem + (g & 1) * kBN, qa + 2 * kk, kb + 2 * kk, idesc_s, (c | kk) ? 1u : 0u);
          }
          tc_commit(&s_full[g & 1]);
          stamp(1, g);
          tc_commit(&k_empty[s]);
          if (j == x.n_kb - 1) tc_commit(q_free);
          if (g > 0) issue_pv(g - 1, prev_first);
          prev_first = j == 0;
        }
      }
      if (g > 0) issue_pv(g - 1, prev_first);
    }
    __syncwarp();
  } else {
    // softmax warps 2..5: warp w reads TMEM lanes (w & 3) * 32 .. + 31, one
    // query row per thread.
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane_id();
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
    const uint32_t prow = sbase + C::kOffP + r * 128;
    auto wait_pv = [&](int i) {
      mbar_wait(&pv_done[i % PB], (i / PB) & 1);
      tc_fence_after();
    };
    int g = 0;
    for (ItemWalk w(n_items, H, cu, tiles); w.valid(); w.advance()) {
      const Item x = w.cur;
      const int row = x.q0 + r;
      const int lim = min(row, x.s1 - 1);  // last visible key of this row
      float m_used = -INFINITY, l = 0.f;   // running max (scaled, log2 units) and row sum
      for (int j = 0; j < x.n_kb; ++j, ++g) {
        mbar_wait(&s_full[g & 1], (g >> 1) & 1);
        tc_fence_after();
        if (r == 0) stamp(3, g);
        uint32_t raw[2][32];
        tmem_ld32_async(lane_base + (g & 1) * kBN, raw[0]);
        tmem_ld32_async(lane_base + (g & 1) * kBN + 32, raw[1]);
        tmem_wait_ld();
        if (r == 0) stamp(7, g);
        tc_fence_before();
        mbar_arrive(&s_free[g & 1]);
        float sv[64];
        const int nvalid = lim - (x.s0 + j * kBN) + 1;  // keys c < nvalid are visible
        float mx[8];
        if (__all_sync(0xffffffffu, nvalid >= kBN)) {  // below the diagonal for the whole warp: no mask
#pragma unroll
          for (int c = 0; c < 64; ++c) {
            sv[c] = __uint_as_float(raw[c >> 5][c & 31]);
            mx[c & 7] = c < 8 ? sv[c] : fmaxf(mx[c & 7], sv[c]);
          }
        } else {
#pragma unroll
          for (int c = 0; c < 64; ++c) {
            sv[c] = c < nvalid ? __uint_as_float(raw[c >> 5][c & 31]) : -INFINITY;
            mx[c & 7] = c < 8 ? sv[c] : fmaxf(mx[c & 7], sv[c]);
          }
        }
        const float mt = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                               fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7]))) * scale_log2;
        const float m_new = fmaxf(m_used, mt);
        if (j == 0) {
          m_used = m_new;
        } else if (__any_sync(0xffffffffu, m_new > m_used + kRescaleThresh)) {
          wait_pv(g - 1);  // O settled
          const float f = ex2(m_used - m_new);
#pragma unroll 1
          for (int c0 = 0; c0 < HD; c0 += 32) {
            uint32_t o[32];
            tmem_ld32_async(lane_base + C::kColO + c0, o);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * f);
            tmem_st32(lane_base + C::kColO + c0, o);
          }
          tmem_wait_st();
          l *= f;
          m_used = m_new;
        }
        if (r == 0) stamp(4, g);
        const uint32_t pbuf = prow + (g % PB) * C::kPBytes;
        // exponent arguments, row sums and P in packed pairs (FFMA2 / FADD2:
        // half the FP32 instructions of the issue-bound exp phase)
        const float2 sc2 = make_float2(scale_log2, scale_log2), nm2 = make_float2(-m_used, -m_used);
        float2 rs2[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
        uint32_t wd[8][4];
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 a = __ffma2_rn(make_float2(sv[ch * 8 + 2 * e], sv[ch * 8 + 2 * e + 1]), sc2, nm2);
            const float2 pp = make_float2(ex2(a.x), ex2(a.y));
            rs2[e] = __fadd2_rn(rs2[e], pp);
            wd[ch][e] = pack_bf16x2(pp.x, pp.y);
          }
        }
        if (g >= PB) wait_pv(g - PB);  // P buffer free (checked after the exps: usually long done)
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) sts_v4(pbuf + ((ch ^ (r & 7)) << 4), wd[ch][0], wd[ch][1], wd[ch][2], wd[ch][3]);
        const float2 rsa = __fadd2_rn(__fadd2_rn(rs2[0], rs2[1]), __fadd2_rn(rs2[2], rs2[3]));
        l += rsa.x + rsa.y;
        fence_async_smem();  // generic-proxy P stores -> visible to the tensor core
        tc_fence_before();
        mbar_arrive(&p_full[g % PB]);
        if (r == 0) stamp(5, g);
      }
      // epilogue: O / l of this item
      wait_pv(g - 1);
      const float inv = l > 0.f ? 1.f / l : 0.f;
      const bool store = row < x.s1;
      bf16* dst = out + (static_cast<size_t>(row) * H + x.h) * HD;
#pragma unroll 1
      for (int c0 = 0; c0 < HD; c0 += 32) {
        uint32_t o[32];
        tmem_ld32_async(lane_base + C::kColO + c0, o);
        tmem_wait_ld();
        if (store) {
#pragma unroll
          for (int i = 0; i < 32; i += 8) {
            uint4 v;
            v.x = pack_bf16x2(__uint_as_float(o[i + 0]) * inv, __uint_as_float(o[i + 1]) * inv);
            v.y = pack_bf16x2(__uint_as_float(o[i + 2]) * inv, __uint_as_float(o[i + 3]) * inv);
            v.z = pack_bf16x2(__uint_as_float(o[i + 4]) * inv, __uint_as_float(o[i + 5]) * inv);
            v.w = pack_bf16x2(__uint_as_float(o[i + 6]) * inv, __uint_as_float(o[i + 7]) * inv);
            *reinterpret_cast<uint4*>(dst + c0 + i) = v;
          }
        }
      }
      tc_fence_before();  // O reads ordered before the next item's first p_full arrive
      if (r == 0) stamp(6, g);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<C::kTmemCols>(tmem);
}

unsigned long long* g_prefill_trace = nullptr;

int sm_count() {
  static int n = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : 148;
  }();
  return n;
}

template <int HD>
void launch_prefill(const bf16* q, const bf16* k, const bf16* v, int H, int KVH, int M, const int* cu,
                    const int* tiles, int n_tiles, bf16* out, cudaStream_t st) {
  using C = PrefillCfg<HD>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_prefill_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    attr = true;
  }
  const CUtensorMap mq = chain_operand_map(q, M, H * HD, kBM);
  const CUtensorMap mk = chain_operand_map(k, M, KVH * HD, kBN);
  const CUtensorMap mv = chain_operand_map(v, M, KVH * HD, kBN);
  const float scale = kLog2e / sqrtf(static_cast<float>(HD));
  const int n_items = n_tiles * H;
  // two CTAs per SM (TMEM 2 x 256 cols, <= 113 KB smem); one item per CTA
  // when the packed kernels must leave room for a decode step (set_packed_persistent)
  const int grid = packed_persistent() ? std::min(n_items, 2 * sm_count()) : n_items;
  attn_prefill_kernel<HD><<<grid, kThreads, C::kSmem, st>>>(mq, mk, mv, H, KVH, n_items, cu, tiles, scale, out,
                                                             g_prefill_trace);
  count_launch();
}

}  // namespace

void attn_prefill_set_trace(unsigned long long* buf) { g_prefill_trace = buf; }

bool attn_prefill_supported(int hd) { return hd == 64 || hd == 128; }

void attn_prefill(const bf16* q, const bf16* k, const bf16* v, int H, int KVH, int hd, int M, const int* cu,
                  const int* tiles, int n_tiles, bf16* out, cudaStream_t st) {
  if (n_tiles <= 0) return;
  if (hd == 64) {
    launch_prefill<64>(q, k, v, H, KVH, M, cu, tiles, n_tiles, out, st);
  } else if (hd == 128) {
    launch_prefill<128>(q, k, v, H, KVH, M, cu, tiles, n_tiles, out, st);
  } else {
    throw std::invalid_argument("attn_prefill: head_dim must be 64 or 128");
  }
}

}  // namespace fpk
