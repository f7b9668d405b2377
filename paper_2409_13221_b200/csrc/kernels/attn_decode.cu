// fuseplan-b200 — paged decode attention on tensor cores (head_dim 64 / 128).
//
// Persistent kernel, one CTA per SM (<= 148), 6-8 independent warps. A work
// item is (sample, 256-token context split, kv head); warps take items from a
// launch-wide atomic counter in the host's longest-first order (dynamic load
// balance). Each warp streams its items' 32-token K|V units with 2-D TMA
// (box 64 x 32 rows, 128-byte swizzle) into a private 2-3 stage ring on
// mbarriers, issuing kStages units ahead across item boundaries so the pipe
// never drains, and computes S = Q K^T and O += P V with mma.sync m16n8k16
// (bf16 in, fp32 accumulate), the G query heads of a GQA group as MMA rows
// (K/V read once per group) and the online softmax in registers; ldmatrix
// addresses apply the TMA swizzle (16-byte chunk c of row r lives at chunk
// c ^ (r & 7)), so fragment loads are bank-conflict free. A single-split item
// normalises in place; otherwise the last split of a (sample, kv head) to
// finish merges the (o, m, l) partials (atomic ticket), so no combine kernel
// runs. Split boundaries depend on the position only (batch-independent
// results). HBM-bound: every K/V byte of the visible context is read once.
#include <math.h>

#include <algorithm>
#include <cstdlib>

#include "launch.cuh"
#include "ops.h"
#include "ptx.cuh"

namespace fpk {

namespace {

constexpr int kPT = 64;
constexpr int kTileBytes = 32 * 128;  // one 32-row x 64-column bf16 box (a TMA box)
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ void ldsm4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm4t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Swizzled address of 16-byte chunk `c16` (along the head dim) of row r.
template <int HD>
__device__ __forceinline__ uint32_t swz(uint32_t tile_base, int r, int c16) {
  const int sub = c16 >> 3, cc = c16 & 7;
  return tile_base + sub * kTileBytes + r * 128 + ((cc ^ (r & 7)) << 4);
}

// Stages are private to the warp, so no cross-warp barrier exists.
// A stage holds K and V of one 32-token unit and, for the first unit of an
// item, the item's G query rows (bulk-copied with it, so starting an item
// never waits on a global load of q).
// Two shapes of the same per-item computation (identical numerics): WIDE —
// many warps, 2 stages each — for large batches, where warps per SM hide the
// per-unit latency; DEEP — few warps, a deep ring each — for small batches,
// where each warp streams a long item alone and needs many units in flight.
template <int HD, bool DEEP = false>
struct DecCfg {
  static constexpr int kSub = HD / 64;                  // 64-column boxes per K (or V) unit
  static constexpr int kBox = 32 * 128;                 // 32 rows x 128 B
  static constexpr int kKV = 2 * kSub * kBox;           // K + V of one 32-token unit
  static constexpr int kQSlot = HD == 64 ? 1024 : 2048; // >= 8 q rows x HD x 2 B, keeps 1 KB alignment
  static constexpr int kStageBytes = kKV + kQSlot;
  static constexpr int kWarps = DEEP ? (HD == 64 ? 4 : 3) : (HD == 64 ? 12 : 6);
  static constexpr int kStages = DEEP ? (HD == 64 ? 6 : 4) : 2;
  static constexpr int kSmem = kWarps * kStages * kStageBytes + 1024;
};

// A decoded work item: (sample b, split, kv head), its token range [t0, t1),
// the sample's context cx and number of non-empty splits nsb.
struct DecItem {
  int j, b, kvh, split, t0, t1, cx, nsb;
};
// Issue cursor: the item, its current / end 32-token unit, and (lane l) the
// pool page id of the item's l-th 64-token page — fetched once per item, so
// issuing a unit needs no dependent global load.
struct Cursor {
  DecItem it;
  int u, ue;
  int pg;
};
static_assert(kDecodeChunk / 64 <= 32, "an item's pages must fit one per lane");

template <int HD, int G, bool DEEP>
__global__ void __launch_bounds__(DecCfg<HD, DEEP>::kWarps * 32, 1) attn_decode_mma_kernel(
    const __grid_constant__ CUtensorMap kv_map, const bf16* __restrict__ q, const int* __restrict__ block_table,
    int bt_stride, int rows_per_page, int layer_rows, int layer, const int* __restrict__ slot,
    const int* __restrict__ ctx, const int* __restrict__ items, int B, int H, int KVH, int nsplit_max,
    float scale_log2,
    float* __restrict__ part_o, float* __restrict__ part_ml, bf16* __restrict__ out, int* __restrict__ counters) {
  pdl_trigger();  // let the next (PDL-launched) GEMM start its prologue / weight prefetch
  using C = DecCfg<HD, DEEP>;
  static_assert(G <= 8, "GQA group must fit the first 8 MMA rows");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full_bar[C::kWarps][C::kStages];

  __shared__ int4 ring_s[C::kWarps][8][2];  // items decoded by the issue cursor, in order, for the consumer

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* bar = full_bar[warp];
  uint8_t* my_smem = smem + warp * C::kStages * C::kStageBytes;
  int4(*ring)[2] = ring_s[warp];
  if (lane == 0) {
    if (warp == 0) tma_prefetch_desc(&kv_map);
    for (int s = 0; s < C::kStages; ++s) mbar_init(&bar[s], 1);
    fence_barrier_init();
  }
  __syncwarp();
  // items / ctx / slot / block table were uploaded before the step's first
  // kernel: readable before griddepcontrol.wait. q, the new token's K/V and
  // the work counters are not (they come from the kernels before this one).
  const int n_items = items[0] * KVH;
  const int T = gridDim.x * C::kWarps;

  // item j -> (sample b, split, kv head): pair items[1 + j / KVH] = b << 8 |
  // split (the host lists pairs longest first), kv head j % KVH
  auto decode = [&](int j, DecItem& it) {
    it.j = j;
    if (j >= n_items) return;
    const int pr = j / KVH;
    it.kvh = j - pr * KVH;
    const int e = items[1 + pr];
    it.b = e >> 8;
    it.split = e & 255;
    it.cx = ctx[it.b];
    it.t0 = it.split * kDecodeChunk;
    it.t1 = min(it.cx, it.t0 + kDecodeChunk);
    it.nsb = (it.cx + kDecodeChunk - 1) / kDecodeChunk;
  };
  int wr = 0, rd = 0;
  auto begin_item = [&](Cursor& c) {  // all lanes: page ids, hand the item to the consumer
    if (lane == 0) {
      ring[wr & 7][0] = make_int4(c.it.j, c.it.b, c.it.kvh, c.it.split);
      ring[wr & 7][1] = make_int4(c.it.t0, c.it.t1, c.it.cx, c.it.nsb);
    }
    ++wr;
    if (c.it.j < n_items) {
      c.u = c.it.t0 >> 5;
      c.ue = ((c.it.t1 - 1) >> 5) + 1;
      const int p0 = c.it.t0 >> 6, np = ((c.it.t1 - 1) >> 6) - p0 + 1;
      c.pg = lane < np ? block_table[slot[c.it.b] * bt_stride + p0 + lane] : 0;
    }
    __syncwarp();
  };
  // dynamic schedule: the first T items are static, then a launch-wide counter
  auto grab = [&](Cursor& c) {
    int j = 0;
    if (lane == 0) j = T + atomicAdd(&counters[0], 1);
    decode(__shfl_sync(0xffffffffu, j, 0), c.it);
    begin_item(c);
  };
  auto next_issue = [&](Cursor& c) {  // advance the issue cursor by one unit
    if (++c.u >= c.ue) grab(c);
  };
  auto issue = [&](const Cursor& c, int k, bool with_q = true) {  // all lanes (lane 0 issues)
    const int pid = __shfl_sync(0xffffffffu, c.pg, (c.u >> 1) - (c.it.t0 >> 6));
    if (lane != 0) return;
    const int rk = pid * rows_per_page + layer * layer_rows + c.it.kvh * 2 * kPT + (c.u & 1) * 32;
    uint8_t* dst = my_smem + k * C::kStageBytes;
    const bool first = c.u == (c.it.t0 >> 5);
    constexpr uint32_t kQBytes = G * HD * 2;
    mbar_arrive_expect_tx(&bar[k], C::kKV + (first ? kQBytes : 0u));
#pragma unroll
    for (int sub = 0; sub < C::kSub; ++sub) {
      tma_load_2d(dst + sub * C::kBox, &kv_map, &bar[k], sub * 64, rk);
      tma_load_2d(dst + (C::kSub + sub) * C::kBox, &kv_map, &bar[k], sub * 64, rk + kPT);
    }
    if (first && with_q)
      bulk_load(dst + C::kKV, q + (static_cast<size_t>(c.it.b) * H + c.it.kvh * G) * HD, kQBytes, &bar[k]);
  };

  // issue cursor: the first item is static (warp index in the grid)
  Cursor in;
  decode(warp + static_cast<int>(blockIdx.x) * C::kWarps, in.it);
  begin_item(in);
  int issued = 0;
  if (in.it.j < n_items) {
    // Before waiting on the previous kernel: stream the units of the first
    // item that hold only cached tokens (positions < ctx - 1, written by
    // earlier steps); the q rows follow after the wait.
    const int u_new = (in.it.cx - 1) >> 5;  // unit of the token appended this step
    for (; issued < C::kStages && in.u < in.ue && in.u < u_new; ++issued, ++in.u) issue(in, issued, false);
  }
  pdl_wait();
  if (issued > 0 && lane == 0)  // stage 0 (the item's first unit) already expects the q bytes
    bulk_load(my_smem + C::kKV, q + (static_cast<size_t>(in.it.b) * H + in.it.kvh * G) * HD, G * HD * 2, &bar[0]);
  if (in.it.j < n_items && in.u >= in.ue) grab(in);
  // prologue: fill the remaining stages
  for (; issued < C::kStages && in.it.j < n_items; ++issued) {
    issue(in, issued);
    next_issue(in);
  }
  // consume cursor: the issue cursor's items, in order
  DecItem cur;
  auto pop = [&]() {
    const int4 x = ring[rd & 7][0], y = ring[rd & 7][1];
    ++rd;
    cur = DecItem{x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w};
  };
  pop();
  int cu = cur.t0 >> 5, cue = ((cur.t1 - 1) >> 5) + 1;

  const int r0 = lane >> 2;
  const uint32_t base = smem_u32(my_smem);
  uint32_t qa[HD / 16][4];
  float o[HD / 8][4];
  float m_run = -INFINITY, l_run = 0.f;
  bool fresh = true;

  for (int c = 0; cur.j < n_items; ++c) {
    const int k = c % C::kStages;
    mbar_wait(&bar[k], (c / C::kStages) & 1);
    if (fresh) {  // new item: Q fragments from the stage's q slot, reset the running state
      fresh = false;
      const bf16* qs = reinterpret_cast<const bf16*>(my_smem + k * C::kStageBytes + C::kKV);
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
        const int col = kk * 16 + 2 * (lane & 3);
        const bool ok = r0 < G;
        qa[kk][0] = ok ? *reinterpret_cast<const uint32_t*>(qs + r0 * HD + col) : 0u;
        qa[kk][1] = 0u;
        qa[kk][2] = ok ? *reinterpret_cast<const uint32_t*>(qs + r0 * HD + col + 8) : 0u;
        qa[kk][3] = 0u;
      }
#pragma unroll
      for (int i = 0; i < HD / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
      m_run = -INFINITY;
      l_run = 0.f;
    }
    const uint32_t Kt = base + k * C::kStageBytes;
    const uint32_t Vt = Kt + C::kSub * C::kBox;
    const int ut0 = cu * 32;
    const int lo = max(cur.t0, ut0) - ut0, hi = min(cur.t1, ut0 + 32) - ut0;

    // S = Q K^T over 32 tokens (4 n-tiles of 8)
    float sc[4][4];
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) sc[nt][0] = sc[nt][1] = sc[nt][2] = sc[nt][3] = 0.f;
    const int mi = lane >> 3;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
#pragma unroll
      for (int nt = 0; nt < 4; nt += 2) {
        const int r = (nt + (mi >> 1)) * 8 + (lane & 7);
        uint32_t b0, b1, b2, b3;
        ldsm4(swz<HD>(Kt, r, kk * 2 + (mi & 1)), b0, b1, b2, b3);
        mma16816(sc[nt], qa[kk], b0, b1);
        mma16816(sc[nt + 1], qa[kk], b2, b3);
      }
    }
    float mx = -INFINITY;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int tok = nt * 8 + 2 * (lane & 3) + e;
        const float v = (tok >= lo && tok < hi) ? sc[nt][e] * scale_log2 : -INFINITY;
        sc[nt][e] = v;
        mx = fmaxf(mx, v);
      }
    }
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    const float nm = fmaxf(m_run, mx);
    const float corr = (m_run == -INFINITY) ? 0.f : exp2f(m_run - nm);
    m_run = nm;
    float rs = 0.f;
    uint32_t pa[2][4];
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const float p0 = (sc[nt][0] == -INFINITY) ? 0.f : exp2f(sc[nt][0] - nm);
      const float p1 = (sc[nt][1] == -INFINITY) ? 0.f : exp2f(sc[nt][1] - nm);
      rs += p0 + p1;
      const int kk2 = nt >> 1;
      if ((nt & 1) == 0) {
        pa[kk2][0] = pack_bf16x2(p0, p1);
        pa[kk2][1] = 0u;
      } else {
        pa[kk2][2] = pack_bf16x2(p0, p1);
        pa[kk2][3] = 0u;
      }
    }
    rs += __shfl_xor_sync(0xffffffffu, rs, 1);
    rs += __shfl_xor_sync(0xffffffffu, rs, 2);
    l_run = l_run * corr + rs;
#pragma unroll
    for (int dn = 0; dn < HD / 8; ++dn) {
      o[dn][0] *= corr;
      o[dn][1] *= corr;
    }
#pragma unroll
    for (int kk2 = 0; kk2 < 2; ++kk2) {
#pragma unroll
      for (int dn = 0; dn < HD / 8; dn += 2) {
        const int r = kk2 * 16 + (mi & 1) * 8 + (lane & 7);
        uint32_t b0, b1, b2, b3;
        ldsm4t(swz<HD>(Vt, r, dn + (mi >> 1)), b0, b1, b2, b3);
        mma16816(o[dn], pa[kk2], b0, b1);
        mma16816(o[dn + 1], pa[kk2], b2, b3);
      }
    }
    // refill this stage with the unit kStages ahead
    __syncwarp();
    if (in.it.j < n_items) {
      if (lane == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(in, k);
      next_issue(in);
    }
    // advance the consume cursor; flush the item's partial when it ends
    if (++cu >= cue) {
      const int nsb = cur.nsb, b = cur.b, kvh = cur.kvh, split = cur.split;
      const size_t row0 = static_cast<size_t>(b) * H + kvh * G;
      if (nsb == 1) {
        // single split: the combine is the identity (f = 1), normalise here
        if (r0 < G) {
          bf16* og = out + (row0 + r0) * HD + 2 * (lane & 3);
#pragma unroll
          for (int dn = 0; dn < HD / 8; ++dn)
            *reinterpret_cast<__nv_bfloat162*>(og + dn * 8) =
                __floats2bfloat162_rn(__fdiv_rn(o[dn][0], l_run), __fdiv_rn(o[dn][1], l_run));
        }
      } else {
        if (r0 < G) {
          const size_t pb = (row0 + r0) * nsplit_max + split;
          float* po = part_o + pb * HD + 2 * (lane & 3);
#pragma unroll
          for (int dn = 0; dn < HD / 8; ++dn)
            *reinterpret_cast<float2*>(po + dn * 8) = make_float2(o[dn][0], o[dn][1]);
          if ((lane & 3) == 0) {
            part_ml[pb * 2] = m_run;
            part_ml[pb * 2 + 1] = l_run;
          }
        }
        // the last split of (sample, kv head) to finish merges all of them:
        // a release-ordered ticket (the warp's partial stores are ordered
        // before it by __syncwarp) instead of a full __threadfence, whose L1
        // invalidation would evict every warp's cached tables; the merge
        // reads the partials through L2 (ld.global.cg).
        __syncwarp();
        int last = 0;
        if (lane == 0) {
          int old;
          asm volatile("atom.release.gpu.global.add.s32 %0, [%1], 1;"
                       : "=r"(old)
                       : "l"(counters + 2 + b * KVH + kvh)
                       : "memory");
          last = old == nsb - 1;
        }
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last) {
          if (lane == 0) counters[2 + b * KVH + kvh] = 0;  // ready for the next launch
          for (int g = 0; g < G; ++g) combine_row(part_o, part_ml, (row0 + g) * nsplit_max, nsb, HD, lane, 32,
                                                  out + (row0 + g) * HD);
        }
      }
      pop();
      cu = cur.t0 >> 5;
      cue = ((cur.t1 - 1) >> 5) + 1;
      fresh = true;
    }
  }
  // the last warp out resets the work counter for the next launch
  if (lane == 0 && atomicAdd(&counters[1], 1) == static_cast<int>(gridDim.x) * C::kWarps - 1) {
    counters[0] = 0;
    counters[1] = 0;
  }
}

template <int HD, int G, bool DEEP>
void launch_cfg(const CUtensorMap& map, const bf16* q, int B, int H, int KVH, const KvPoolView& pool, int layer,
            const int* slot, const int* ctx, const int* items, int nsplit, float* work, bf16* out, int* counters,
            cudaStream_t st) {
  using C = DecCfg<HD, DEEP>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_decode_mma_kernel<HD, G, DEEP>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    attr = true;
  }
  float* part_o = work;
  float* part_ml = work + static_cast<size_t>(B) * H * nsplit * HD;
  const int layer_rows = KVH * 2 * kPT;
  const int rows_per_page = static_cast<int>(pool.page_bytes / (static_cast<size_t>(HD) * 2));
  const float scale = kLog2e / sqrtf(static_cast<float>(HD));
  const int max_items = nsplit * B * KVH;  // upper bound of the non-empty items
  const int grid = std::max(1, std::min(148, (max_items + C::kWarps - 1) / C::kWarps));
  launch_pdl(attn_decode_mma_kernel<HD, G, DEEP>, dim3(grid), dim3(C::kWarps * 32), C::kSmem, st, map, q,
             pool.block_table, pool.bt_stride, rows_per_page, layer_rows, layer, slot, ctx, items, B, H, KVH, nsplit,
             scale, part_o, part_ml, out, counters);
  count_launch();
}

template <int HD, int G>
void launch(const CUtensorMap& map, const bf16* q, int B, int H, int KVH, const KvPoolView& pool, int layer,
            const int* slot, const int* ctx, const int* items, int nsplit, float* work, bf16* out, int* counters,
            cudaStream_t st) {
  // DEEP when the (sample, kv head) pairs cannot fill the WIDE grid's warps
  // four times over; FUSEPLAN_ATTN_DEEP=0/1 forces a shape (A/B runs)
  static const int force = [] {
    const char* e = std::getenv("FUSEPLAN_ATTN_DEEP");
    return e ? std::atoi(e) : -1;
  }();
  const bool deep = force >= 0 ? force == 1 : B * KVH * 4 <= 148 * DecCfg<HD, false>::kWarps;
  if (deep)
    launch_cfg<HD, G, true>(map, q, B, H, KVH, pool, layer, slot, ctx, items, nsplit, work, out, counters, st);
  else
    launch_cfg<HD, G, false>(map, q, B, H, KVH, pool, layer, slot, ctx, items, nsplit, work, out, counters, st);
}

}  // namespace

bool attn_decode_mma(const bf16* q, int B, int H, int KVH, int hd, const KvPoolView& pool, int layer,
                     const int* slot, const int* ctx, const int* items, int nsplit, float* work, bf16* out,
                     int* counters, cudaStream_t st) {
  if (!pool.kv_map || !counters || !items) return false;
  const int G = H / KVH;
#define FP_MMA(HD_, G_)                                                                            \
  if (hd == HD_ && G == G_) {                                                                      \
    launch<HD_, G_>(*pool.kv_map, q, B, H, KVH, pool, layer, slot, ctx, items, nsplit, work, out, counters, st);      \
    return true;                                                                                   \
  }
  FP_MMA(64, 1) FP_MMA(128, 1) FP_MMA(64, 4) FP_MMA(128, 4) FP_MMA(128, 8) FP_MMA(64, 8)
#undef FP_MMA
  return false;
}

}  // namespace fpk
