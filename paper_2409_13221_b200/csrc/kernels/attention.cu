// fuseplan-b200 — attention kernels.
//
// attn_decode: paged-KV flash-decoding. One CTA per (kv head, sample, context
// split); a producer warp streams each 64-token page's K|V block (contiguous
// in the pool: [page][layer][kv_head][K 64 x hd | V 64 x hd]) into a 3-stage
// shared-memory ring with cp.async.bulk (TMA bulk copies, UBLKCP) signalled
// on mbarriers; four consumer warps each own 16 tokens of every page and run
// an online softmax for all G query heads of the GQA group (K read once per
// group). Split boundaries depend on the position only, so every sample's
// result is independent of the batch it decodes in. HBM-bound.
//
// attn_varlen: causal attention over packed variable-length sequences for
// prefill and the scoring models' forward; 64-query tiles x 64-key tiles,
// mma.sync m16n8k16 bf16 (fp32 accumulate), online softmax in registers.
#include <math.h>

#include <algorithm>
#include <array>
#include <vector>
#include <cstdlib>
#include <stdexcept>

#include "ops.h"
#include "ptx.cuh"

namespace fpk {

namespace {

constexpr int kPT = 64;          // tokens per KV page
constexpr int kChunk = kDecodeChunk;  // tokens per decode split
constexpr int kStages = 3;
constexpr float kLog2e = 1.4426950408889634f;

template <int HD, int G>
struct DecodeSmem {
  static constexpr int kPageElems = 2 * kPT * HD;
  static constexpr int kBytes = kStages * kPageElems * 2 + G * HD * 4 + 4 * G * HD * 4 + 4 * G * 2 * 4 + 64;
};

template <int HD, int G>
__global__ void __launch_bounds__(160) attn_decode_kernel(const bf16* __restrict__ q, KvPoolView pool, int layer,
                                                          const int* __restrict__ slot, const int* __restrict__ ctx,
                                                          int H, int nsplit_max, float scale_log2,
                                                          float* __restrict__ part_o, float* __restrict__ part_ml) {
  pdl_trigger();  // let the next (PDL-launched) GEMM start its prologue / weight prefetch
  constexpr int EPL = HD / 32;  // output dims per lane
  constexpr int WH = HD / 4;    // bf16x2 words per half row
  constexpr int kPageElems = 2 * kPT * HD;
  extern __shared__ __align__(128) uint8_t smem[];
  bf16* kv = reinterpret_cast<bf16*>(smem);
  float* q_s = reinterpret_cast<float*>(smem + kStages * kPageElems * 2);
  float* red_o = q_s + G * HD;
  float* red_ml = red_o + 4 * G * HD;
  __shared__ __align__(8) uint64_t full_bar[kStages];
  __shared__ __align__(8) uint64_t empty_bar[kStages];

  const int kvh = blockIdx.x, b = blockIdx.y, split = blockIdx.z;
  const int n_ctx = ctx[b];
  const int t0 = split * kChunk;
  if (t0 >= n_ctx) return;
  const int t1 = min(n_ctx, t0 + kChunk);
  const int pg0 = t0 / kPT, pg1 = (t1 - 1) / kPT;
  const int npages = pg1 - pg0 + 1;
  const int* bt = pool.block_table + slot[b] * pool.bt_stride;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 4);
    }
    fence_barrier_init();
  }
  for (int i = threadIdx.x; i < G * HD; i += blockDim.x) {
    const int g = i / HD, d = i % HD;
    q_s[i] = __bfloat162float(q[(static_cast<size_t>(b) * H + kvh * G + g) * HD + d]);
  }
  __syncthreads();

  if (warp == 4) {  // producer
    if (lane == 0) {
      const uint32_t bytes = kPageElems * 2;
      for (int i = 0; i < npages; ++i) {
        const int s = i % kStages;
        mbar_wait(&empty_bar[s], ((i / kStages) & 1) ^ 1);
        const uint8_t* src = pool.base + static_cast<size_t>(bt[pg0 + i]) * pool.page_bytes +
                             static_cast<size_t>(layer) * pool.layer_bytes +
                             static_cast<size_t>(kvh) * kPageElems * 2;
        mbar_arrive_expect_tx(&full_bar[s], bytes);
        bulk_load(kv + s * kPageElems, src, bytes, &full_bar[s]);
      }
    }
    return;
  }

  const int tok = warp * 16 + (lane >> 1);  // token within page this lane scores
  const int half = lane & 1;
  float m[G], l[G], acc[G][EPL];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    m[g] = -INFINITY;
    l[g] = 0.f;
#pragma unroll
    for (int e = 0; e < EPL; ++e) acc[g][e] = 0.f;
  }

  for (int i = 0; i < npages; ++i) {
    const int s = i % kStages;
    mbar_wait(&full_bar[s], (i / kStages) & 1);
    const bf16* Ks = kv + s * kPageElems;
    const bf16* Vs = Ks + kPT * HD;
    const int page_t0 = (pg0 + i) * kPT;
    const int lo = max(t0, page_t0) - page_t0;
    const int hi = min(t1, page_t0 + kPT) - page_t0;
    const bool valid = tok >= lo && tok < hi;

    float sc[G];
#pragma unroll
    for (int g = 0; g < G; ++g) sc[g] = 0.f;
    const uint32_t* krow = reinterpret_cast<const uint32_t*>(Ks + tok * HD);
#pragma unroll
    for (int it = 0; it < WH; ++it) {
      const int word = half * WH + ((it + tok + (half ? 16 : 0)) % WH);
      const uint32_t kw = krow[word];
      const __nv_bfloat162 k2 = *reinterpret_cast<const __nv_bfloat162*>(&kw);
      const float k0 = __bfloat162float(k2.x), k1 = __bfloat162float(k2.y);
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float2 qq = *reinterpret_cast<const float2*>(q_s + g * HD + 2 * word);
        sc[g] = fmaf(qq.x, k0, fmaf(qq.y, k1, sc[g]));
      }
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
      float v = sc[g] + __shfl_xor_sync(0xffffffffu, sc[g], 1);
      v = valid ? v * scale_log2 : -INFINITY;
      const float pm = warp_max(v);
      const float nm = fmaxf(m[g], pm);
      const float corr = (m[g] == -INFINITY) ? 0.f : exp2f(m[g] - nm);
      const float p = valid ? exp2f(v - nm) : 0.f;
      const float ps = warp_sum(half == 0 ? p : 0.f);
      l[g] = l[g] * corr + ps;
      m[g] = nm;
#pragma unroll
      for (int e = 0; e < EPL; ++e) acc[g][e] *= corr;
      sc[g] = p;
    }
    // P . V over this warp's 16 tokens
#pragma unroll 4
    for (int j = 0; j < 16; ++j) {
      const int tj = warp * 16 + j;
      if (tj < lo || tj >= hi) continue;  // warp-uniform
      const bf16* vr = Vs + tj * HD + lane * EPL;
      float vv[EPL];
      if constexpr (EPL == 1) {
        vv[0] = __bfloat162float(vr[0]);
      } else {
#pragma unroll
        for (int e = 0; e < EPL; e += 2) {
          const __nv_bfloat162 v2 = *reinterpret_cast<const __nv_bfloat162*>(vr + e);
          vv[e] = __bfloat162float(v2.x);
          vv[e + 1] = __bfloat162float(v2.y);
        }
      }
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float pj = __shfl_sync(0xffffffffu, sc[g], 2 * j);
#pragma unroll
        for (int e = 0; e < EPL; ++e) acc[g][e] = fmaf(pj, vv[e], acc[g][e]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_bar[s]);
  }

  // merge the 4 consumer warps
#pragma unroll
  for (int g = 0; g < G; ++g) {
#pragma unroll
    for (int e = 0; e < EPL; ++e) red_o[(warp * G + g) * HD + lane * EPL + e] = acc[g][e];
    if (lane == 0) {
      red_ml[(warp * G + g) * 2] = m[g];
      red_ml[(warp * G + g) * 2 + 1] = l[g];
    }
  }
  asm volatile("bar.sync 1, 128;" ::: "memory");
  for (int i = threadIdx.x; i < G * HD; i += 128) {
    const int g = i / HD, d = i % HD;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < 4; ++w) M = fmaxf(M, red_ml[(w * G + g) * 2]);
    float L = 0.f, O = 0.f;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const float mw = red_ml[(w * G + g) * 2];
      if (mw == -INFINITY) continue;
      const float f = exp2f(mw - M);
      L += red_ml[(w * G + g) * 2 + 1] * f;
      O += red_o[(w * G + g) * HD + d] * f;
    }
    const int h = kvh * G + g;
    const size_t base = (static_cast<size_t>(b) * H + h) * nsplit_max + split;
    part_o[base * HD + d] = O;
    if (d == 0) {
      part_ml[base * 2] = M;
      part_ml[base * 2 + 1] = L;
    }
  }
}

// Merge the context splits of each (sample, head).
__global__ void attn_decode_combine_kernel(const float* __restrict__ part_o, const float* __restrict__ part_ml,
                                           const int* __restrict__ ctx, int H, int HD, int nsplit_max,
                                           bf16* __restrict__ out) {
  pdl_trigger();  // let the next (PDL-launched) GEMM start its prologue / weight prefetch
  const int bh = blockIdx.x;
  const int b = bh / H;
  const int ns = (ctx[b] + kChunk - 1) / kChunk;
  combine_row(part_o, part_ml, static_cast<size_t>(bh) * nsplit_max, ns, HD, threadIdx.x, blockDim.x,
              out + static_cast<size_t>(bh) * HD);
}

// ---------------------------------------------------------------------------
// varlen causal attention (mma.sync m16n8k16)

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void mma_bf16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int HD>
struct VarlenCfg {
  static constexpr int kLd = HD + 8;  // padded smem row (bf16), breaks ldmatrix bank conflicts
  static constexpr int kTile = 64 * kLd;
  static constexpr int kSmem = (1 + 2 * 2) * kTile * 2;  // Q + double-buffered K, V
};

// rows [r0, r0+64) of a [*, heads, HD] tensor, head h, into smem (zero-fill past `end`)
template <int HD>
__device__ __forceinline__ void load_tile(bf16* dst, const bf16* src, int heads, int h, int r0, int end) {
  constexpr int kChunks = HD / 8;
  for (int i = threadIdx.x; i < 64 * kChunks; i += 128) {
    const int r = i / kChunks, c = i % kChunks;
    const int row = r0 + r;
    const bool ok = row < end;
    const bf16* s = src + (static_cast<size_t>(ok ? row : r0) * heads + h) * HD + c * 8;
    cp_async16(smem_u32(dst + r * VarlenCfg<HD>::kLd + c * 8), s, ok ? 16 : 0);
  }
}

template <int HD>
__global__ void __launch_bounds__(128) attn_varlen_kernel(const bf16* __restrict__ q, const bf16* __restrict__ k,
                                                          const bf16* __restrict__ v, int H, int KVH,
                                                          const int* __restrict__ cu, const int* __restrict__ tiles,
                                                          float scale_log2, bf16* __restrict__ out) {
  pdl_trigger();  // let the next (PDL-launched) GEMM start its prologue / weight prefetch
  using C = VarlenCfg<HD>;
  constexpr int LD = C::kLd;
  extern __shared__ __align__(128) uint8_t smem[];
  bf16* Qs = reinterpret_cast<bf16*>(smem);
  bf16* Ks = Qs + C::kTile;       // [2][tile]
  bf16* Vs = Ks + 2 * C::kTile;   // [2][tile]

  const int seq = tiles[2 * blockIdx.x], qt = tiles[2 * blockIdx.x + 1];
  const int h = blockIdx.y, kvh = h / (H / KVH);
  const int s0 = cu[seq], s1 = cu[seq + 1];
  const int q0 = s0 + qt * 64;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  load_tile<HD>(Qs, q, H, h, q0, s1);
  load_tile<HD>(Ks, k, KVH, kvh, s0, s1);
  load_tile<HD>(Vs, v, KVH, kvh, s0, s1);
  cp_async_commit();

  const int n_kt = qt + 1;
  uint32_t qa[HD / 16][4];
  float o[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
  const int qrow0 = q0 + warp * 16 + (lane >> 2);  // rows qrow0 and qrow0 + 8

  for (int kt = 0; kt < n_kt; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < n_kt) {
      load_tile<HD>(Ks + (buf ^ 1) * C::kTile, k, KVH, kvh, s0 + (kt + 1) * 64, s1);
      load_tile<HD>(Vs + (buf ^ 1) * C::kTile, v, KVH, kvh, s0 + (kt + 1) * 64, s1);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    if (kt == 0) {
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
        const int r = warp * 16 + (lane & 15), c = kk * 16 + (lane >> 4) * 8;
        ldsm_x4(smem_u32(Qs + r * LD + c), qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3]);
      }
    }
    const bf16* Kt = Ks + buf * C::kTile;
    const bf16* Vt = Vs + buf * C::kTile;
    float s[8][4];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
#pragma unroll
      for (int nt = 0; nt < 8; nt += 2) {
        const int mi = lane >> 3;
        const int r = (nt + (mi >> 1)) * 8 + (lane & 7), c = kk * 16 + (mi & 1) * 8;
        uint32_t b0, b1, b2, b3;
        ldsm_x4(smem_u32(Kt + r * LD + c), b0, b1, b2, b3);
        mma_bf16(s[nt], qa[kk], b0, b1);
        mma_bf16(s[nt + 1], qa[kk], b2, b3);
      }
    }
    // mask + online softmax (rows qrow0, qrow0 + 8)
    const int key0 = s0 + kt * 64 + 2 * (lane & 3);
    const bool need_mask = (kt == n_kt - 1) || (s0 + (kt + 1) * 64 > s1);
    float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = key0 + nt * 8 + (e & 1);
        const int row = qrow0 + (e >> 1) * 8;
        float val = s[nt][e] * scale_log2;
        if (need_mask && (key > row || key >= s1)) val = -INFINITY;
        s[nt][e] = val;
        mx[e >> 1] = fmaxf(mx[e >> 1], val);
      }
    }
    float corr[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
      const float nm = fmaxf(mrow[r], mx[r]);
      corr[r] = (nm == -INFINITY) ? 1.f : exp2f(mrow[r] - nm);
      mrow[r] = nm;
    }
    float rs[2] = {0.f, 0.f};
    uint32_t pa[4][4];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      float p[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float mm = mrow[e >> 1];
        p[e] = (s[nt][e] == -INFINITY) ? 0.f : exp2f(s[nt][e] - mm);
        rs[e >> 1] += p[e];
      }
      const int kk2 = nt >> 1;
      if ((nt & 1) == 0) {
        pa[kk2][0] = pack_bf16x2(p[0], p[1]);
        pa[kk2][1] = pack_bf16x2(p[2], p[3]);
      } else {
        pa[kk2][2] = pack_bf16x2(p[0], p[1]);
        pa[kk2][3] = pack_bf16x2(p[2], p[3]);
      }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      rs[r] += __shfl_xor_sync(0xffffffffu, rs[r], 1);
      rs[r] += __shfl_xor_sync(0xffffffffu, rs[r], 2);
      lrow[r] = lrow[r] * corr[r] + rs[r];
    }
#pragma unroll
    for (int dn = 0; dn < HD / 8; ++dn) {
      o[dn][0] *= corr[0];
      o[dn][1] *= corr[0];
      o[dn][2] *= corr[1];
      o[dn][3] *= corr[1];
    }
#pragma unroll
    for (int kk2 = 0; kk2 < 4; ++kk2) {
#pragma unroll
      for (int dn = 0; dn < HD / 8; dn += 2) {
        const int mi = lane >> 3;
        const int r = kk2 * 16 + (mi & 1) * 8 + (lane & 7), c = (dn + (mi >> 1)) * 8;
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(smem_u32(Vt + r * LD + c), b0, b1, b2, b3);
        mma_bf16(o[dn], pa[kk2], b0, b1);
        mma_bf16(o[dn + 1], pa[kk2], b2, b3);
      }
    }
    __syncthreads();
  }

#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int row = qrow0 + r * 8;
    if (row >= s1) continue;
    const float inv = 1.f / lrow[r];
    bf16* dst = out + (static_cast<size_t>(row) * H + h) * HD + 2 * (lane & 3);
#pragma unroll
    for (int dn = 0; dn < HD / 8; ++dn) {
      *reinterpret_cast<uint32_t*>(dst + dn * 8) = pack_bf16x2(o[dn][2 * r] * inv, o[dn][2 * r + 1] * inv);
    }
  }
}

template <int HD, int G>
void launch_decode(const bf16* q, int B, int H, int KVH, const KvPoolView& pool, int layer, const int* slot,
                   const int* ctx, int nsplit, float* work, cudaStream_t st) {
  constexpr int smem = DecodeSmem<HD, G>::kBytes;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_decode_kernel<HD, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  float* part_o = work;
  float* part_ml = work + static_cast<size_t>(B) * H * nsplit * HD;
  const float scale = kLog2e / sqrtf(static_cast<float>(HD));
  attn_decode_kernel<HD, G><<<dim3(KVH, B, nsplit), 160, smem, st>>>(q, pool, layer, slot, ctx, H, nsplit, scale,
                                                                      part_o, part_ml); fpk::count_launch();
}

}  // namespace

namespace {
thread_local int g_attn_cut = 0;  // 0 never (default), 1 always, -1 the small-batch rule below (warp-per-item kernels)
}
void set_attn_cut(int mode) { g_attn_cut = mode < 0 ? -1 : (mode ? 1 : 0); }  // fp_k_set_attn_cut

int attn_decode_items(const int* ctx, int B, int KVH, int hd, int G, int* items) {
  // One item per (sample, 512-token split), longest first (counting sort by
  // 32-token units, ties by (sample, split, sub)). Cutting splits into
  // 128-token sub-chunks (partials folded in order: the same bits) is a policy
  // (set_attn_cut): isolated, the wide kernel gains at small batches (gpt2s
  // B 48 / 96: 18.5 / 24.6 vs 26.6 / 26.6 us) and the deep kernel loses (8B
  // B 16-64: 1.2-1.8x slower); in the bench the rule below (cut when the whole
  // splits cannot give every wide-kernel warp an item) measured 549.0 vs 554.2
  // samples/s, so the default is never. The team kernel never takes cuts.
  constexpr int kU = kDecodeChunk / 32;  // units per split
  constexpr int kSubU = 4;               // units per sub-chunk (attn_decode.cu kSubUnits)
  int warps = 0;
  const int v = attn_decode_variant(B, KVH, hd, G, &warps);
  int pairs = 0;
  for (int b = 0; b < B; ++b) pairs += (ctx[b] + kDecodeChunk - 1) / kDecodeChunk;
  const bool cut = v != 2 && (g_attn_cut == 1 || (g_attn_cut < 0 && v == 0 && pairs * KVH < 148 * warps));
  int n = 0;
  for (int u = kU; u >= 1; --u)
    for (int b = 0; b < B; ++b) {
      const int ns = (ctx[b] + kDecodeChunk - 1) / kDecodeChunk;
      for (int s = 0; s < ns; ++s) {
        const int len = std::min(ctx[b], (s + 1) * kDecodeChunk) - s * kDecodeChunk;
        const int units = (len + 31) / 32;
        if (!cut || units <= kSubU) {
          if (units == u) items[1 + n++] = b << 11 | s << 3 | 7;
        } else {
          for (int c = 0; c * kSubU < units; ++c)
            if (std::min(kSubU, units - c * kSubU) == u) items[1 + n++] = b << 11 | s << 3 | c;
        }
      }
    }
  items[0] = n;
  return n;
}

size_t attn_decode_workspace(int B, int H, int hd, int max_ctx) {
  const int ns = (max_ctx + kChunk - 1) / kChunk;
  return static_cast<size_t>(B) * H * ns * (hd + 2) * 5;  // split partials + 4 sub-chunk partials per split
}

void attn_decode(const bf16* q, int B, int H, int KVH, int hd, const KvPoolView& pool, int layer, const int* slot,
                 const int* ctx, const int* items, int max_ctx, float* work, bf16* out, int* counters,
                 cudaStream_t st,
                 cudaEvent_t probe_begin,
                 cudaEvent_t probe_end, int max_ctas) {
  if (B <= 0) return;
  if (probe_begin) cudaEventRecord(probe_begin, st);
  if (pool.page_tokens != kPT) throw std::invalid_argument("attn_decode: page_tokens must be 64");
  const int ns = std::max(1, (max_ctx + kChunk - 1) / kChunk);
  const int G = H / KVH;
#define FP_DEC(HD_, G_) \
  if (hd == HD_ && G == G_) { launch_decode<HD_, G_>(q, B, H, KVH, pool, layer, slot, ctx, ns, work, st); } else
  if (attn_decode_mma(q, B, H, KVH, hd, pool, layer, slot, ctx, items, ns, work, out, counters, st, max_ctas)) {
    if (probe_end) cudaEventRecord(probe_end, st);
    return;  // splits merged in-kernel
  } else FP_DEC(32, 1) FP_DEC(64, 1) FP_DEC(128, 1) FP_DEC(64, 4) FP_DEC(128, 4) FP_DEC(128, 8) FP_DEC(64, 8) {
    throw std::invalid_argument("attn_decode: unsupported (head_dim, group) combination");
  }
#undef FP_DEC
  if (probe_end) cudaEventRecord(probe_end, st);
  const float* part_o = work;
  const float* part_ml = work + static_cast<size_t>(B) * H * ns * hd;
  attn_decode_combine_kernel<<<B * H, std::min(hd, 128), 0, st>>>(part_o, part_ml, ctx, H, hd, ns, out); fpk::count_launch();
}

int attn_varlen_tile_rows(int hd) { return attn_prefill_supported(hd) ? 128 : 64; }

int attn_tiles(const int* cu_host, int n_seq, int rows, int* tiles_host) {
  std::vector<std::array<int, 3>> t;  // (visible keys, seq, q tile)
  for (int s = 0; s < n_seq; ++s) {
    const int len = cu_host[s + 1] - cu_host[s];
    for (int q = 0; q * rows < len; ++q) t.push_back({std::min(len, (q + 1) * rows), s, q});
  }
  if (tiles_host) {
    // Most keys first (better tail); ties keep sequence order.
    std::stable_sort(t.begin(), t.end(), [](const auto& a, const auto& b) { return a[0] > b[0]; });
    for (size_t i = 0; i < t.size(); ++i) {
      tiles_host[2 * i] = t[i][1];
      tiles_host[2 * i + 1] = t[i][2];
    }
  }
  return static_cast<int>(t.size());
}

int attn_varlen_tiles(const int* cu_host, int n_seq, int hd, int* tiles_host) {
  return attn_tiles(cu_host, n_seq, attn_varlen_tile_rows(hd), tiles_host);
}

void attn_varlen(const bf16* q, const bf16* k, const bf16* v, int H, int KVH, int hd, int M, const int* cu,
                 const int* tiles, int n_tiles, bf16* out, cudaStream_t st) {
  if (attn_prefill_supported(hd))
    attn_prefill(q, k, v, H, KVH, hd, M, cu, tiles, n_tiles, out, st);
  else
    attn_varlen_mma(q, k, v, H, KVH, hd, cu, tiles, n_tiles, out, st);
}

void attn_varlen_mma(const bf16* q, const bf16* k, const bf16* v, int H, int KVH, int hd, const int* cu,
                     const int* tiles, int n_tiles, bf16* out, cudaStream_t st) {
  if (n_tiles <= 0) return;
  const float scale = kLog2e / sqrtf(static_cast<float>(hd));
#define FP_VL(HD_)                                                                                           \
  if (hd == HD_) {                                                                                           \
    static bool attr = false;                                                                                \
    if (!attr) {                                                                                             \
      cudaFuncSetAttribute(attn_varlen_kernel<HD_>, cudaFuncAttributeMaxDynamicSharedMemorySize,           \
                           VarlenCfg<HD_>::kSmem);                                                           \
      attr = true;                                                                                           \
    }                                                                                                        \
    attn_varlen_kernel<HD_><<<dim3(n_tiles, H), 128, VarlenCfg<HD_>::kSmem, st>>>(q, k, v, H, KVH, cu, tiles, \
                                                                                  scale, out); fpk::count_launch();               \
  } else
  FP_VL(32) FP_VL(64) FP_VL(128) { throw std::invalid_argument("attn_varlen: unsupported head_dim"); }
#undef FP_VL
}

}  // namespace fpk
