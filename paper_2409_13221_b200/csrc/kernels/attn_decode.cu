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
unsigned long long* g_attn_trace_host = nullptr;  // debug tracing (set_attn_trace)
__device__ __forceinline__ unsigned long long gtime_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
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

// Attention numerics: inside a 512-token split item, the online softmax runs
// over 128-token sub-chunks (4 units) and the sub-chunk partials are folded
// left to right with this update (explicit roundings), so the warp-per-item
// and the team kernels give the same bits for every batch size.
constexpr int kSubUnits = 4;
__device__ __forceinline__ void sub_fold(float& M, float& L, float m, float l, float& fa, float& fb) {
  const float Mn = fmaxf(M, m);
  fa = exp2f(M - Mn);
  fb = exp2f(m - Mn);
  L = __fadd_rn(__fmul_rn(L, fa), __fmul_rn(l, fb));
  M = Mn;
}
__device__ __forceinline__ float sub_fold_o(float O, float o, float fa, float fb) {
  return __fadd_rn(__fmul_rn(O, fa), __fmul_rn(o, fb));
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
template <int HD, int DEEP = 0>  // 0 wide, 1 deep
struct DecCfg {
  static constexpr int kSub = HD / 64;                  // 64-column boxes per K (or V) unit
  static constexpr int kBox = 32 * 128;                 // 32 rows x 128 B
  static constexpr int kKV = 2 * kSub * kBox;           // K + V of one 32-token unit
  static constexpr int kQSlot = HD == 64 ? 1024 : 2048; // >= 8 q rows x HD x 2 B, keeps 1 KB alignment
  static constexpr int kStageBytes = kKV + kQSlot;
  static constexpr int kWarps = DEEP == 1 ? (HD == 64 ? 4 : 3) : (HD == 64 ? 12 : 6);
  static constexpr int kStages = DEEP == 1 ? (HD == 64 ? 6 : 4) : 2;
  static constexpr int kSmem = kWarps * kStages * kStageBytes + 1024;
};

// A decoded work item: (sample b, split, kv head), its token range [t0, t1),
// the sample's context cx and number of non-empty splits nsb.
struct DecItem {
  int j, b, kvh, split, t0, t1, cx, nsb;
  int sub;  // 7: the whole split; c < 4: only sub-chunk c of it
};
// items[] entry -> (b, split, sub) and the token range of the item
__device__ __forceinline__ void item_entry(int e, int cx, DecItem& it) {
  it.b = e >> 11;
  it.split = (e >> 3) & 255;
  it.sub = e & 7;
  it.cx = cx;
  const int s0 = it.split * kDecodeChunk;
  it.t0 = it.sub == 7 ? s0 : s0 + it.sub * 32 * kSubUnits;
  it.t1 = min(cx, it.sub == 7 ? s0 + kDecodeChunk : it.t0 + 32 * kSubUnits);
  it.nsb = (cx + kDecodeChunk - 1) / kDecodeChunk;
}
// Issue cursor: the item, its current / end 32-token unit, and (lane l) the
// pool page id of the item's l-th 64-token page — fetched once per item, so
// issuing a unit needs no dependent global load.
struct Cursor {
  DecItem it;
  int u, ue;
  int pg;
};
static_assert(kDecodeChunk / 64 <= 32, "an item's pages must fit one per lane");

template <int HD, int G, int DEEP>
__global__ void __launch_bounds__(DecCfg<HD, DEEP>::kWarps * 32, 1) attn_decode_mma_kernel(
    const __grid_constant__ CUtensorMap kv_map, const bf16* __restrict__ q, const int* __restrict__ block_table,
    int bt_stride, int rows_per_page, int layer_rows, int layer, const int* __restrict__ slot,
    const int* __restrict__ ctx, const int* __restrict__ items, int B, int H, int KVH, int nsplit_max,
    float scale_log2,
    float* __restrict__ part_o, float* __restrict__ part_ml, float* __restrict__ sub_o, float* __restrict__ sub_ml,
    bf16* __restrict__ out, int* __restrict__ counters, unsigned long long* __restrict__ trace) {
  const unsigned long long t_entry = trace ? gtime_ns() : 0ull;
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
    item_entry(e, ctx[e >> 11], it);
  };
  int wr = 0, rd = 0;
  auto begin_item = [&](Cursor& c) {  // all lanes: page ids, hand the item to the consumer
    if (lane == 0) {
      ring[wr & 7][0] = make_int4(c.it.j, c.it.b, c.it.kvh, c.it.split | c.it.sub << 16);
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
    cur = DecItem{x.x, x.y, x.z, x.w & 0xffff, y.x, y.y, y.z, y.w, x.w >> 16};
  };
  pop();
  int cu = cur.t0 >> 5, cue = ((cur.t1 - 1) >> 5) + 1;

  const int r0 = lane >> 2;
  const uint32_t base = smem_u32(my_smem);
  uint32_t qa[HD / 16][4];
  float o[HD / 8][4];
  float m_run = -INFINITY, l_run = 0.f;
  float acc_m = -INFINITY, acc_l = 0.f, acc_o[HD / 8][2];  // folded sub-chunks of the current item
  bool acc_has = false;
  bool fresh = true;

  const unsigned long long t_begin = trace ? gtime_ns() : 0ull;
  int c = 0;
  for (; cur.j < n_items; ++c) {
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
    // sub-chunk boundary: fold the running softmax into the item accumulator
    ++cu;
    if (cu >= cue || ((cu - (cur.t0 >> 5)) % kSubUnits) == 0) {
      if (!acc_has) {
        acc_m = m_run;
        acc_l = l_run;
#pragma unroll
        for (int dn = 0; dn < HD / 8; ++dn) {
          acc_o[dn][0] = o[dn][0];
          acc_o[dn][1] = o[dn][1];
        }
        acc_has = true;
      } else {
        float fa, fb;
        sub_fold(acc_m, acc_l, m_run, l_run, fa, fb);
#pragma unroll
        for (int dn = 0; dn < HD / 8; ++dn) {
          acc_o[dn][0] = sub_fold_o(acc_o[dn][0], o[dn][0], fa, fb);
          acc_o[dn][1] = sub_fold_o(acc_o[dn][1], o[dn][1], fa, fb);
        }
      }
      m_run = -INFINITY;
      l_run = 0.f;
#pragma unroll
      for (int dn = 0; dn < HD / 8; ++dn) o[dn][0] = o[dn][1] = o[dn][2] = o[dn][3] = 0.f;
    }
    // flush the item's partial when it ends
    if (cu >= cue) {
      acc_has = false;
      const int nsb = cur.nsb, b = cur.b, kvh = cur.kvh, split = cur.split;
      const size_t row0 = static_cast<size_t>(b) * H + kvh * G;
      // release-ordered ticket (the warp's stores before it are ordered by
      // __syncwarp); returns whether this warp was the last of `n`. Cheaper
      // than a full __threadfence, whose L1 invalidation would evict every
      // warp's cached tables; merges read the partials through L2 (.cg).
      auto ticket = [&](int* ctr, int n) {
        __syncwarp();
        int last = 0;
        if (lane == 0) {
          int old;
          asm volatile("atom.release.gpu.global.add.s32 %0, [%1], 1;" : "=r"(old) : "l"(ctr) : "memory");
          last = old == n - 1;
          if (last) *ctr = 0;  // ready for the next launch
        }
        return __shfl_sync(0xffffffffu, last, 0) != 0;
      };
      // after the split's partial is stored: the last split to finish merges all
      auto merge_splits = [&]() {
        if (ticket(counters + 2 + b * KVH + kvh, nsb))
          for (int g = 0; g < G; ++g)
            combine_row(part_o, part_ml, (row0 + g) * nsplit_max, nsb, HD, lane, 32, out + (row0 + g) * HD);
      };
      if (cur.sub == 7) {
        if (nsb == 1) {
          // single split: the combine is the identity (f = 1), normalise here
          if (r0 < G) {
            bf16* og = out + (row0 + r0) * HD + 2 * (lane & 3);
#pragma unroll
            for (int dn = 0; dn < HD / 8; ++dn)
              *reinterpret_cast<__nv_bfloat162*>(og + dn * 8) =
                  __floats2bfloat162_rn(__fdiv_rn(acc_o[dn][0], acc_l), __fdiv_rn(acc_o[dn][1], acc_l));
          }
        } else {
          if (r0 < G) {
            const size_t pb = (row0 + r0) * nsplit_max + split;
            float* po = part_o + pb * HD + 2 * (lane & 3);
#pragma unroll
            for (int dn = 0; dn < HD / 8; ++dn)
              *reinterpret_cast<float2*>(po + dn * 8) = make_float2(acc_o[dn][0], acc_o[dn][1]);
            if ((lane & 3) == 0) {
              part_ml[pb * 2] = acc_m;
              part_ml[pb * 2 + 1] = acc_l;
            }
          }
          merge_splits();
        }
      } else {
        // one sub-chunk of a cut split: park its partial; the last sub-chunk
        // to finish folds them in order (== the whole-split fold) and flushes
        if (r0 < G) {
          const size_t sb = ((row0 + r0) * nsplit_max + split) * kSubUnits + cur.sub;
          float* so = sub_o + sb * HD + 2 * (lane & 3);
#pragma unroll
          for (int dn = 0; dn < HD / 8; ++dn)
            *reinterpret_cast<float2*>(so + dn * 8) = make_float2(acc_o[dn][0], acc_o[dn][1]);
          if ((lane & 3) == 0) {
            sub_ml[sb * 2] = acc_m;
            sub_ml[sb * 2 + 1] = acc_l;
          }
        }
        const int slen = min(cur.cx, (split + 1) * kDecodeChunk) - split * kDecodeChunk;
        const int nsub = (slen + 32 * kSubUnits - 1) / (32 * kSubUnits);
        if (ticket(counters + 2 + B * KVH + (b * KVH + kvh) * nsplit_max + split, nsub)) {
          for (int g = 0; g < G; ++g) {
            const size_t sb0 = ((row0 + g) * nsplit_max + split) * kSubUnits;
            float M = __ldcg(sub_ml + sb0 * 2), L = __ldcg(sub_ml + sb0 * 2 + 1);
            float O[HD / 32];
#pragma unroll
            for (int i = 0; i < HD / 32; ++i) O[i] = __ldcg(sub_o + sb0 * HD + lane + 32 * i);
            for (int c = 1; c < nsub; ++c) {
              float fa, fb;
              sub_fold(M, L, __ldcg(sub_ml + (sb0 + c) * 2), __ldcg(sub_ml + (sb0 + c) * 2 + 1), fa, fb);
#pragma unroll
              for (int i = 0; i < HD / 32; ++i)
                O[i] = sub_fold_o(O[i], __ldcg(sub_o + (sb0 + c) * HD + lane + 32 * i), fa, fb);
            }
            if (nsb == 1) {
#pragma unroll
              for (int i = 0; i < HD / 32; ++i)
                out[(row0 + g) * HD + lane + 32 * i] = __float2bfloat16_rn(__fdiv_rn(O[i], L));
            } else {
              const size_t pb = (row0 + g) * nsplit_max + split;
#pragma unroll
              for (int i = 0; i < HD / 32; ++i) part_o[pb * HD + lane + 32 * i] = O[i];
              if (lane == 0) {
                part_ml[pb * 2] = M;
                part_ml[pb * 2 + 1] = L;
              }
            }
          }
          if (nsb > 1) merge_splits();
        }
      }
      pop();
      cu = cur.t0 >> 5;
      cue = ((cur.t1 - 1) >> 5) + 1;
      fresh = true;
    }
  }
  if (trace && lane == 0) {  // debug: per-warp busy interval and units (tools/attn_roofline.py --trace)
    unsigned long long* t = trace + 4ull * (blockIdx.x * C::kWarps + warp);
    t[0] = t_entry;
    t[1] = t_begin;
    t[2] = gtime_ns();
    t[3] = c;
  }
  // the last warp out resets the work counter for the next launch
  if (lane == 0 && atomicAdd(&counters[1], 1) == static_cast<int>(gridDim.x) * C::kWarps - 1) {
    counters[0] = 0;
    counters[1] = 0;
  }
}

template <int HD, int G, int DEEP>
void launch_cfg(const CUtensorMap& map, const bf16* q, int B, int H, int KVH, const KvPoolView& pool, int layer,
            const int* slot, const int* ctx, const int* items, int nsplit, float* work, bf16* out, int* counters,
            cudaStream_t st, int max_ctas) {
  using C = DecCfg<HD, DEEP>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_decode_mma_kernel<HD, G, DEEP>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    attr = true;
  }
  const size_t rows = static_cast<size_t>(B) * H * nsplit;
  float* part_o = work;
  float* part_ml = part_o + rows * HD;
  float* sub_o = part_ml + rows * 2;
  float* sub_ml = sub_o + rows * kSubUnits * HD;
  const int layer_rows = KVH * 2 * kPT;
  const int rows_per_page = static_cast<int>(pool.page_bytes / (static_cast<size_t>(HD) * 2));
  const float scale = kLog2e / sqrtf(static_cast<float>(HD));
  const int max_items = nsplit * kSubUnits * B * KVH;  // upper bound of the items (cut splits included)
  const int grid = std::max(1, std::min(max_ctas, (max_items + C::kWarps - 1) / C::kWarps));
  launch_pdl(attn_decode_mma_kernel<HD, G, DEEP>, dim3(grid), dim3(C::kWarps * 32), C::kSmem, st, map, q,
             pool.block_table, pool.bt_stride, rows_per_page, layer_rows, layer, slot, ctx, items, B, H, KVH, nsplit,
             scale, part_o, part_ml, sub_o, sub_ml, out, counters,
             g_attn_trace_host ? g_attn_trace_host : trace_slot(1, grid * C::kWarps, 4));
  count_launch();
}


// ---------------------------------------------------------------------------
// Team kernel (head_dim 64, no GQA grouping). The work item is the same
// (sample, 512-token split, kv head), but a team of 4 warps shares it: warp w
// streams the item's sub-chunk w (128 tokens = 4 units) through its own
// 2-stage ring and runs the online softmax over it; the team leader then folds
// the 4 sub-partials in order (the combine_row formula) and flushes the item
// (normalised output, or a split partial + ticket as above). A warp's stream is
// 4 units per item instead of 16, so long items no longer serialise on one
// warp and the dynamic queue balances at a 4x finer grain. The sub-chunk fold
// is part of the numerics for every batch size (batch-independent results).
template <int T>  // warps per team (4: one sub-chunk each; 2: two contiguous sub-chunks each)
struct TeamCfg {
  static constexpr int kTeamWarps = T;
  static constexpr int kTeams = 12 / T;
  static constexpr int kWarps = kTeams * kTeamWarps;
  static constexpr int kStages = 2;
  static constexpr int kSubUnits = fpk::kSubUnits;                      // units per sub-chunk
  static constexpr int kSubs = kDecodeChunk / (32 * kSubUnits);         // sub-chunks per item
  static constexpr int kKV = 2 * 32 * 128;                              // K + V of one unit (hd 64)
  static constexpr int kStageBytes = kKV;                               // (q slots live after the stages)
  static constexpr int kQOff = kWarps * kStages * kStageBytes;         // q slot (warp, stage): 128 B each
  static constexpr int kSmem = kQOff + kWarps * kStages * 128 + 1024;
};
static_assert(TeamCfg<4>::kSubs % 4 == 0, "sub-chunks split evenly over team warps");

template <int T>
__device__ __forceinline__ void team_bar(int team) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + team), "r"(32 * T) : "memory");
}

template <int T>
__global__ void __launch_bounds__(TeamCfg<T>::kWarps * 32, 1) attn_decode_team_kernel(
    const __grid_constant__ CUtensorMap kv_map, const bf16* __restrict__ q, const int* __restrict__ block_table,
    int bt_stride, int rows_per_page, int layer_rows, int layer, const int* __restrict__ slot,
    const int* __restrict__ ctx, const int* __restrict__ items, int H, int KVH, int nsplit_max, float scale_log2,
    float* __restrict__ part_o, float* __restrict__ part_ml, bf16* __restrict__ out, int* __restrict__ counters,
    unsigned long long* __restrict__ trace) {
  constexpr int HD = 64;
  using C = TeamCfg<T>;
  constexpr int kSubsPerWarp = C::kSubs / T;
  const unsigned long long t_entry = trace ? gtime_ns() : 0ull;
  pdl_trigger();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full_bar[C::kWarps][C::kStages];
  __shared__ int4 ring_s[C::kTeams][4][2];                 // team item infos (decoded), items i .. i+2
  __shared__ float sub_o[C::kTeams][2][C::kSubs][HD];      // sub-chunk partials, double-buffered by item
  __shared__ float sub_ml[C::kTeams][2][C::kSubs][2];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int team = warp / C::kTeamWarps, tw = warp % C::kTeamWarps;
  uint64_t* bar = full_bar[warp];
  uint8_t* my_smem = smem + warp * C::kStages * C::kStageBytes;
  auto qslot = [&](int stage) { return smem + C::kQOff + (warp * C::kStages + stage) * 128; };
  int4(*ring)[2] = ring_s[team];
  if (lane == 0) {
    if (warp == 0) tma_prefetch_desc(&kv_map);
    for (int s2 = 0; s2 < C::kStages; ++s2) mbar_init(&bar[s2], 1);
    fence_barrier_init();
  }
  __syncwarp();
  const int n_items = items[0] * KVH;
  const int n_teams = gridDim.x * C::kTeams;

  auto decode = [&](int j, DecItem& it) {  // (the host never cuts splits for this kernel)
    it.j = j;
    it.b = it.kvh = it.split = it.t0 = it.t1 = it.cx = it.nsb = 0;
    it.sub = 7;
    if (j >= n_items) return;
    const int pr = j / KVH;
    it.kvh = j - pr * KVH;
    const int e = items[1 + pr];
    item_entry(e, ctx[e >> 11], it);
  };
  auto put = [&](int idx, int j) {  // leader lane only
    DecItem it;
    decode(j, it);
    ring[idx & 3][0] = make_int4(it.j, it.b, it.kvh, it.split);
    ring[idx & 3][1] = make_int4(it.t0, it.t1, it.cx, it.nsb);
  };
  auto get = [&](int idx) {
    const int4 x = ring[idx & 3][0], y = ring[idx & 3][1];
    return DecItem{x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w, 7};
  };
  // this warp's units of an item: its contiguous sub-chunks
  auto my_units = [&](const DecItem& it, int& ua, int& ub) {
    ua = (it.t0 >> 5) + tw * kSubsPerWarp * C::kSubUnits;
    ub = min(((it.t1 - 1) >> 5) + 1, ua + kSubsPerWarp * C::kSubUnits);
    if (it.j >= n_items || ub < ua) ub = ua;
  };

  // item 0 of each team is static (its index), so it is decoded before
  // griddepcontrol.wait; item 1 comes from the counter after it
  if (tw == 0 && lane == 0) put(0, static_cast<int>(blockIdx.x) * C::kTeams + team);
  team_bar<T>(team);
  int known = 0;  // highest item index whose info is in the ring

  // issue cursor over (item index, unit) of this warp's sub-chunks
  int in_i = 0, in_u = 0, in_ue = 0, in_ua = 0, in_pg = 0;
  DecItem in_it = get(0);
  bool in_ok = in_it.j < n_items;
  auto load_item = [&]() {  // all lanes: unit range and page ids of item in_i
    my_units(in_it, in_ua, in_ue);
    in_u = in_ua;
    const int p0 = in_ua >> 1;
    in_pg = (in_ue > in_ua && lane < 2 * kSubsPerWarp) ? block_table[slot[in_it.b] * bt_stride + p0 + lane] : 0;
  };
  if (in_ok) load_item();
  auto advance_item = [&]() {  // move past empty / finished items while their infos are known
    while (in_ok && in_u >= in_ue) {
      if (in_i + 1 > known) return;  // wait for the next team barrier
      ++in_i;
      in_it = get(in_i);
      in_ok = in_it.j < n_items;
      if (in_ok) load_item();
    }
  };
  int n_iss = 0, n_con = 0;
  auto issue_unit = [&](bool with_q) {  // all lanes
    const int k = n_iss % C::kStages;
    const int pid = __shfl_sync(0xffffffffu, in_pg, (in_u >> 1) - (in_ua >> 1));
    if (lane == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      const int rk = pid * rows_per_page + layer * layer_rows + in_it.kvh * 2 * kPT + (in_u & 1) * 32;
      uint8_t* dst = my_smem + k * C::kStageBytes;
      const bool first = in_u == in_ua;
      mbar_arrive_expect_tx(&bar[k], C::kKV + (first ? HD * 2 : 0));
      tma_load_2d(dst, &kv_map, &bar[k], 0, rk);
      tma_load_2d(dst + 32 * 128, &kv_map, &bar[k], 0, rk + kPT);
      if (first && with_q)
        bulk_load(qslot(k), q + (static_cast<size_t>(in_it.b) * H + in_it.kvh) * HD, HD * 2, &bar[k]);
    }
    ++n_iss;
    ++in_u;
  };
  auto pump = [&]() {  // all lanes
    advance_item();
    while (in_ok && in_u < in_ue && n_iss - n_con < C::kStages) {
      issue_unit(true);
      advance_item();
    }
  };
  // before waiting on the previous kernel: the cached units of item 0 (only
  // tokens written by earlier steps; the q row follows after the wait)
  bool q_late = false;
  if (in_ok && in_u < in_ue) {
    const int u_new = (in_it.cx - 1) >> 5;
    while (n_iss < C::kStages && in_u < in_ue && in_u < u_new) {
      q_late |= in_u == in_ua;
      issue_unit(false);
    }
  }
  pdl_wait();  // q, the new K/V and the counters come from earlier kernels
  const unsigned long long t_wait = trace ? gtime_ns() : 0ull;
  unsigned long long t_first = 0ull;
  if (q_late && lane == 0)  // stage 0 (the sub-chunk's first unit) already expects the q bytes
    bulk_load(qslot(0), q + (static_cast<size_t>(in_it.b) * H + in_it.kvh) * HD, HD * 2, &bar[0]);
  if (tw == 0 && lane == 0) put(1, n_teams + atomicAdd(&counters[0], 1));
  team_bar<T>(team);
  known = 1;
  pump();

  const int r0 = lane >> 2;
  const uint32_t base = smem_u32(my_smem);
  const int mi = lane >> 3;
  for (int i = 0;; ++i) {
    const DecItem it = get(i);
    if (it.j >= n_items) break;
    int ua, ub;
    my_units(it, ua, ub);
    float o[HD / 8][4];
    float m_run = -INFINITY, l_run = 0.f;
#pragma unroll
    for (int d = 0; d < HD / 8; ++d) o[d][0] = o[d][1] = o[d][2] = o[d][3] = 0.f;
    uint32_t qa[HD / 16][4];
    for (int u = ua; u < ub; ++u) {
      const int k = n_con % C::kStages;
      mbar_wait(&bar[k], (n_con / C::kStages) & 1);
      if (u == ua) {
        const bf16* qs = reinterpret_cast<const bf16*>(qslot(k));
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const int col = kk * 16 + 2 * (lane & 3);
          qa[kk][0] = r0 == 0 ? *reinterpret_cast<const uint32_t*>(qs + col) : 0u;
          qa[kk][1] = 0u;
          qa[kk][2] = r0 == 0 ? *reinterpret_cast<const uint32_t*>(qs + col + 8) : 0u;
          qa[kk][3] = 0u;
        }
      }
      const uint32_t Kt = base + k * C::kStageBytes;
      const uint32_t Vt = Kt + 32 * 128;
      const int ut0 = u * 32;
      const int lo = max(it.t0, ut0) - ut0, hi = min(it.t1, ut0 + 32) - ut0;
      float sc[4][4];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) sc[nt][0] = sc[nt][1] = sc[nt][2] = sc[nt][3] = 0.f;
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
      __syncwarp();
      ++n_con;
      pump();
      // end of a sub-chunk: park its partial (row 0 lives in lanes 0..3), restart the softmax
      const int rel = u + 1 - (it.t0 >> 5);
      if (rel % C::kSubUnits == 0 || u + 1 == ub) {
        const int sx = (rel - 1) / C::kSubUnits;
        if (lane < 4) {
#pragma unroll
          for (int dn = 0; dn < HD / 8; ++dn) {
            sub_o[team][i & 1][sx][dn * 8 + 2 * lane] = o[dn][0];
            sub_o[team][i & 1][sx][dn * 8 + 2 * lane + 1] = o[dn][1];
          }
          if (lane == 0) {
            sub_ml[team][i & 1][sx][0] = m_run;
            sub_ml[team][i & 1][sx][1] = l_run;
          }
        }
        m_run = -INFINITY;
        l_run = 0.f;
#pragma unroll
        for (int d = 0; d < HD / 8; ++d) o[d][0] = o[d][1] = o[d][2] = o[d][3] = 0.f;
      }
    }
    const int sl = i & 1;
    if (tw == 0 && lane == 0) put(i + 2, n_teams + atomicAdd(&counters[0], 1));
    team_bar<T>(team);
    if (i == 0 && trace) t_first = gtime_ns();
    known = i + 2;
    pump();
    if (tw != 0) continue;
    // leader: fold the sub-chunks in order, then flush the item
    const int nsub = (it.t1 - it.t0 + 32 * C::kSubUnits - 1) / (32 * C::kSubUnits);
    float M = sub_ml[team][sl][0][0], L = sub_ml[team][sl][0][1];
    float O0 = sub_o[team][sl][0][lane], O1 = sub_o[team][sl][0][lane + 32];
    for (int s2 = 1; s2 < nsub; ++s2) {
      float fa, fb;
      sub_fold(M, L, sub_ml[team][sl][s2][0], sub_ml[team][sl][s2][1], fa, fb);
      O0 = sub_fold_o(O0, sub_o[team][sl][s2][lane], fa, fb);
      O1 = sub_fold_o(O1, sub_o[team][sl][s2][lane + 32], fa, fb);
    }
    const size_t row0 = static_cast<size_t>(it.b) * H + it.kvh;
    if (it.nsb == 1) {
      bf16* og = out + row0 * HD;
      og[lane] = __float2bfloat16_rn(__fdiv_rn(O0, L));
      og[lane + 32] = __float2bfloat16_rn(__fdiv_rn(O1, L));
    } else {
      const size_t pb = row0 * nsplit_max + it.split;
      part_o[pb * HD + lane] = O0;
      part_o[pb * HD + lane + 32] = O1;
      if (lane == 0) {
        part_ml[pb * 2] = M;
        part_ml[pb * 2 + 1] = L;
      }
      __syncwarp();
      int last = 0;
      if (lane == 0) {
        int old;
        asm volatile("atom.release.gpu.global.add.s32 %0, [%1], 1;"
                     : "=r"(old)
                     : "l"(counters + 2 + it.b * KVH + it.kvh)
                     : "memory");
        last = old == it.nsb - 1;
      }
      last = __shfl_sync(0xffffffffu, last, 0);
      if (last) {
        if (lane == 0) counters[2 + it.b * KVH + it.kvh] = 0;
        combine_row(part_o, part_ml, row0 * nsplit_max, it.nsb, HD, lane, 32, out + row0 * HD);
      }
    }
  }
  if (trace && tw == 0 && lane == 0) {  // per CTA: entry, team 0's wait return, last team's end, team 0's first item
    unsigned long long* t = trace + 4ull * blockIdx.x;
    if (team == 0) t[0] = t_entry, t[1] = t_wait, t[3] = t_first;
    atomicMax(t + 2, gtime_ns());
  }
  // the last team out resets the work counter for the next launch
  if (tw == 0 && lane == 0 && atomicAdd(&counters[1], 1) == n_teams - 1) {
    counters[0] = 0;
    counters[1] = 0;
  }
}

template <int T>
void launch_team(const CUtensorMap& map, const bf16* q, int B, int H, int KVH, const KvPoolView& pool, int layer,
                 const int* slot, const int* ctx, const int* items, int nsplit, float* work, bf16* out, int* counters,
                 cudaStream_t st, int max_ctas) {
  using C = TeamCfg<T>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_decode_team_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    attr = true;
  }
  float* part_o = work;
  float* part_ml = work + static_cast<size_t>(B) * H * nsplit * 64;
  const int layer_rows = KVH * 2 * kPT;
  const int rows_per_page = static_cast<int>(pool.page_bytes / (static_cast<size_t>(64) * 2));
  const float scale = kLog2e / sqrtf(64.f);
  const int max_items = nsplit * B * KVH;
  const int grid = std::max(1, std::min(max_ctas, (max_items + C::kTeams - 1) / C::kTeams));
  launch_pdl(attn_decode_team_kernel<T>, dim3(grid), dim3(C::kWarps * 32), C::kSmem, st, map, q, pool.block_table,
             pool.bt_stride, rows_per_page, layer_rows, layer, slot, ctx, items, H, KVH, nsplit, scale, part_o,
             part_ml, out, counters, trace_slot(2, grid, 4));
  count_launch();
}


template <int HD, int G>
void launch(const CUtensorMap& map, const bf16* q, int B, int H, int KVH, const KvPoolView& pool, int layer,
            const int* slot, const int* ctx, const int* items, int nsplit, float* work, bf16* out, int* counters,
            cudaStream_t st, int max_ctas) {
  switch (attn_decode_variant(B, KVH, HD, G, nullptr)) {
    case 2: launch_team<4>(map, q, B, H, KVH, pool, layer, slot, ctx, items, nsplit, work, out, counters, st, max_ctas); break;
    case 1:
      launch_cfg<HD, G, 1>(map, q, B, H, KVH, pool, layer, slot, ctx, items, nsplit, work, out, counters, st,
                              max_ctas);
      break;
    default:
      launch_cfg<HD, G, 0>(map, q, B, H, KVH, pool, layer, slot, ctx, items, nsplit, work, out, counters, st,
                               max_ctas);
  }
}

}  // namespace

void set_attn_trace(unsigned long long* buf) { g_attn_trace_host = buf; }

// The team kernel (hd 64, G 1) while the (sample, kv head) pairs cannot fill
// the warp-per-item grid four times over, else deep below that for other
// shapes, else wide; identical numerics.
// (The lean "mid" shape and 2-warp teams were measured no faster,
// profiles/r02_attn_variant_sweep.txt, and are not instantiated.)
int attn_decode_variant(int B, int KVH, int hd, int G, int* warps) {
  const int wide_warps = hd == 64 ? DecCfg<64, 0>::kWarps : DecCfg<128, 0>::kWarps;
  const bool small = B * KVH * 4 <= 148 * wide_warps;
  int v = 0;
  if (hd == 64 && G == 1 && small) v = 2;
  // GQA at hd 128 (Llama-3-8B, 4 query heads per KV head): the wide shape wins
  // once B * KVH > 40 (8B B 8 / 16 / 24, long contexts: 59 / 68 / 94 vs
  // 74 / 78 / 100 us, ATTN_SHAPE=8b tools/attn_roofline.py); MHA at hd 128
  // (1.3B) keeps the deep shape (29-31 vs 35 us at B 4-12).
  else if (small && !(hd == 128 && G >= 4 && B * KVH > 40)) v = 1;
  if (warps) *warps = v == 2 ? 12 : v == 1 ? (hd == 64 ? DecCfg<64, 1>::kWarps : DecCfg<128, 1>::kWarps) : wide_warps;
  return v;
}

bool attn_decode_mma(const bf16* q, int B, int H, int KVH, int hd, const KvPoolView& pool, int layer,
                     const int* slot, const int* ctx, const int* items, int nsplit, float* work, bf16* out,
                     int* counters, cudaStream_t st, int max_ctas) {
  if (!pool.kv_map || !counters || !items) return false;
  const int G = H / KVH;
#define FP_MMA(HD_, G_)                                                                            \
  if (hd == HD_ && G == G_) {                                                                      \
    launch<HD_, G_>(*pool.kv_map, q, B, H, KVH, pool, layer, slot, ctx, items, nsplit, work, out, counters, st, max_ctas);      \
    return true;                                                                                   \
  }
  FP_MMA(64, 1) FP_MMA(128, 1) FP_MMA(64, 4) FP_MMA(128, 4) FP_MMA(128, 8) FP_MMA(64, 8)
#undef FP_MMA
  return false;
}

}  // namespace fpk
