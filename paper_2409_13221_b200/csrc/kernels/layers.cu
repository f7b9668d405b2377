// fuseplan-b200 — memory-bound transformer pieces: synthetic weight init,
// embedding gather, fused residual-add + RMSNorm (+ optional value head),
// RoPE + KV append into the paged pool.
#include <math.h>

#include <atomic>
#include <stdexcept>

#include "launch.cuh"
#include "ops.h"
#include "philox.cuh"
#include "ptx.cuh"
#include "norm.cuh"

namespace fpk {

static std::atomic<long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
void count_launches(long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
long long launch_count() { return g_launches.load(std::memory_order_relaxed); }

namespace {

constexpr float kEps = 1e-5f;

__global__ void init_bf16_kernel(bf16* __restrict__ w, size_t n, uint64_t seed, uint64_t tag, float scale) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    const float u = unit24(hash3(seed, tag, i));
    const float t = __fsub_rn(__fmul_rn(u, 2.0f), 1.0f);
    w[i] = __float2bfloat16_rn(__fmul_rn(t, scale));
  }
}

__global__ void init_gain_kernel(float* __restrict__ g, size_t n, uint64_t seed, uint64_t tag) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    const float u = unit24(hash3(seed, tag, i));
    const float t = __fsub_rn(__fmul_rn(u, 2.0f), 1.0f);
    g[i] = __fadd_rn(1.0f, __fmul_rn(0.1f, t));
  }
}

__global__ void init_bf16_gu_kernel(bf16* __restrict__ w, int F, int d, uint64_t seed, uint64_t tag, float scale) {
  const size_t n = static_cast<size_t>(2) * F * d;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    const size_t row = i / d, col = i % d;
    const size_t grp = row / 128, within = row % 128;
    const size_t logical = within < 64 ? grp * 64 + within : static_cast<size_t>(F) + grp * 64 + (within - 64);
    const float u = unit24(hash3(seed, tag, logical * d + col));
    const float t = __fsub_rn(__fmul_rn(u, 2.0f), 1.0f);
    w[i] = __float2bfloat16_rn(__fmul_rn(t, scale));
  }
}

__global__ void assemble_kernel(AssembleArgs a) {
  pdl_trigger();  // let the next (PDL-launched) GEMM start its prologue / weight prefetch
  const int j = blockIdx.x;
  const int sid = a.sid[j], P = a.P[j], R = a.R[j], row0 = a.cu[j], r0 = a.roff[j];
  const int T = P + R;
  const int* hist = a.hist_tok[j];
  const float* hl = a.hist_logp[j];
  const int* pr = a.prompts + static_cast<size_t>(sid) * a.max_prompt;
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    a.tokens[row0 + t] = t < P ? pr[t] : hist[t - P];
    a.pos[row0 + t] = t;
  }
  for (int k = threadIdx.x; k < R; k += blockDim.x) {
    a.targets[r0 + k] = hist[k];
    a.logp_actor[r0 + k] = hl[k];
    a.gather_resp[r0 + k] = row0 + P - 1 + k;
  }
  if (threadIdx.x == 0) a.gather_last[j] = row0 + T - 1;
}

__global__ void embed_kernel(const int* __restrict__ tok, const int* __restrict__ idx, const bf16* __restrict__ E,
                             int d, float* __restrict__ x) {
  pdl_trigger();  // let the next (PDL-launched) GEMM start its prologue / weight prefetch
  pdl_wait();     // PDL-launched: the input tokens come from the previous kernel
  const int m = blockIdx.x;
  const bf16* e = E + static_cast<size_t>(tok[idx ? idx[m] : m]) * d;
  float* o = x + static_cast<size_t>(m) * d;
  for (int j = threadIdx.x * 2; j < d; j += blockDim.x * 2) {
    const __nv_bfloat162 v = *reinterpret_cast<const __nv_bfloat162*>(e + j);
    o[j] = __bfloat162float(v.x);
    o[j + 1] = __bfloat162float(v.y);
  }
}

__device__ float block_sum(float v, float* red) {
  return group_sum(v, red, threadIdx.x >> 5, threadIdx.x & 31, blockDim.x >> 5, [] { __syncthreads(); });
}

// One block per output row, one float4 of the row per thread (blockDim =
// d / 4 rounded up to a warp multiple): the x load and all NS split-K partial
// loads of a thread are in flight together, so a row costs one memory round
// trip regardless of d.
template <int NS>  // number of split-K partials
__global__ void add_norm_kernel(float* __restrict__ x, const float* __restrict__ parts, size_t split_stride,
                                const float* __restrict__ gain, bf16* __restrict__ y, int d,
                                const int* __restrict__ gather, int rows, const bf16* __restrict__ value_w,
                                float* __restrict__ value, L2Prefetch pf) {
  pdl_trigger();  // let the next (PDL-launched) GEMM start its prologue / weight prefetch
  if (threadIdx.x < 2 && pf.bytes[threadIdx.x]) {  // the next GEMMs' weights: block slices, 32 KB requests
    const size_t n = pf.bytes[threadIdx.x], per = ((n + gridDim.x - 1) / gridDim.x + 15) & ~size_t(15);
    const char* base = static_cast<const char*>(pf.p[threadIdx.x]);
    for (size_t o = blockIdx.x * per; o < min(n, (blockIdx.x + 1) * per); o += 32768)
      prefetch_l2(base + o, static_cast<uint32_t>(min(size_t(32768), min(n, (blockIdx.x + 1) * per) - o)));
  }
  pdl_wait();     // PDL-launched: x and the partials come from the previous kernels
  __shared__ float red[32];
  const int i = blockIdx.x;
  const int src = gather ? gather[i] : i;
  const int d4 = d >> 2;
  const int j = threadIdx.x;
  const bool on = j < d4;
  float4* xr = reinterpret_cast<float4*>(x + static_cast<size_t>(src) * d);
  const float4* pr = reinterpret_cast<const float4*>(parts + static_cast<size_t>(src) * d);
  const size_t ps4 = split_stride >> 2;
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  if (on) {
    v = xr[j];
    float4 p[NS > 0 ? NS : 1];
#pragma unroll
    for (int s = 0; s < NS; ++s) p[s] = pr[s * ps4 + j];
#pragma unroll
    for (int s = 0; s < NS; ++s) v.x += p[s].x, v.y += p[s].y, v.z += p[s].z, v.w += p[s].w;
    if (!gather && NS > 0) xr[j] = v;
  }
  float ss = sumsq4(v);
  ss = block_sum(ss, red);
  const float inv = rsqrtf(ss / d + kNormEps);
  float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
  if (on) g = reinterpret_cast<const float4*>(gain)[j];
  if (value_w) {
    float dot = 0.f;
    if (on) {
      const __nv_bfloat162 w01 = reinterpret_cast<const __nv_bfloat162*>(value_w)[2 * j];
      const __nv_bfloat162 w23 = reinterpret_cast<const __nv_bfloat162*>(value_w)[2 * j + 1];
      dot = v.x * inv * g.x * __bfloat162float(w01.x) + v.y * inv * g.y * __bfloat162float(w01.y) +
            v.z * inv * g.z * __bfloat162float(w23.x) + v.w * inv * g.w * __bfloat162float(w23.y);
    }
    dot = block_sum(dot, red);
    if (threadIdx.x == 0) value[i] = dot;
    return;
  }
  if (on) {
    uint2* yr = reinterpret_cast<uint2*>(y + static_cast<size_t>(i) * d);
    yr[j] = norm_scale4(v, inv, g);
  }
}

// Decode step head: the embedding gather and the first layer's RMSNorm in one
// launch — x = E[tok] (exact bf16 -> fp32) and y = RMSNorm(x) with
// add_norm_kernel<0>'s thread mapping and reduction tree, so the same bits as
// embed + add_norm.
__global__ void embed_norm_kernel(const int* __restrict__ tok, const int* __restrict__ idx,
                                  const bf16* __restrict__ E, int d, float* __restrict__ x,
                                  const float* __restrict__ gain, bf16* __restrict__ y) {
  pdl_trigger();  // let the next (PDL-launched) GEMM start its prologue / weight prefetch
  __shared__ float red[32];
  const int i = blockIdx.x;
  const int j = threadIdx.x;
  const bool on = j < (d >> 2);
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  if (on) {
    const bf16* e = E + static_cast<size_t>(tok[idx ? idx[i] : i]) * d;
    const uint2 w = reinterpret_cast<const uint2*>(e)[j];
    const __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(&w.x);
    const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&w.y);
    v = make_float4(__bfloat162float(a.x), __bfloat162float(a.y), __bfloat162float(b.x), __bfloat162float(b.y));
    reinterpret_cast<float4*>(x + static_cast<size_t>(i) * d)[j] = v;
  }
  float ss = sumsq4(v);
  ss = block_sum(ss, red);
  const float inv = rsqrtf(ss / d + kNormEps);
  float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
  if (on) g = reinterpret_cast<const float4*>(gain)[j];
  if (on) {
    uint2* yr = reinterpret_cast<uint2*>(y + static_cast<size_t>(i) * d);
    yr[j] = norm_scale4(v, inv, g);
  }
}

// Packed forward (prefill / scoring, thousands of rows): RMSNorm with one
// warp per row and 8 rows per block — no block-wide reduction, V float4 of
// the row per lane, all of them in flight at once. d = 128 V.
template <int V>
__global__ void __launch_bounds__(256) rms_norm_rows_kernel(const float* __restrict__ x, const float* __restrict__ gain,
                                                            bf16* __restrict__ y, int M) {
  pdl_trigger();  // let the next (PDL-launched) GEMM start its prologue / weight prefetch
  pdl_wait();     // PDL-launched: x comes from the previous kernel
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= M) return;
  const int lane = threadIdx.x & 31;
  constexpr int d4 = 32 * V;
  const float4* xr = reinterpret_cast<const float4*>(x) + static_cast<size_t>(row) * d4;
  float4 v[V];
#pragma unroll
  for (int k = 0; k < V; ++k) v[k] = xr[lane + 32 * k];
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < V; ++k) ss += sumsq4(v[k]);
  ss = warp_sum(ss);
  const float inv = rsqrtf(ss / (4 * d4) + kNormEps);
  uint2* yr = reinterpret_cast<uint2*>(y) + static_cast<size_t>(row) * d4;
  const float4* g4 = reinterpret_cast<const float4*>(gain);
#pragma unroll
  for (int k = 0; k < V; ++k) yr[lane + 32 * k] = norm_scale4(v[k], inv, g4[lane + 32 * k]);
}

// grid: M rows; block: 128. Rotate-half RoPE (pairs i, i + HD/2); cos/sin of
// the row's position are computed once per pair index and shared by all heads.
template <int HD>
__global__ void rope_qkv_kernel(const bf16* __restrict__ qkv, int H, int KVH, const int* __restrict__ pos,
                                float log2_theta, bf16* __restrict__ q_out, bf16* __restrict__ k_out,
                                bf16* __restrict__ v_out, KvPoolView pool, int use_pool, int layer,
                                const int* __restrict__ slot) {
  pdl_trigger();  // let the next (PDL-launched) GEMM start its prologue / weight prefetch
  constexpr int half = HD / 2;
  __shared__ float cs_s[half], sn_s[half];
  const int m = blockIdx.x;
  const int p = pos[m];
  const int width = (H + 2 * KVH) * HD;
  const bf16* in = qkv + static_cast<size_t>(m) * width;
  for (int i = threadIdx.x; i < half; i += blockDim.x) {
    const float inv_freq = exp2f(-(2.0f * i / HD) * log2_theta);
    float sn, cs;
    sincosf(static_cast<float>(p) * inv_freq, &sn, &cs);
    cs_s[i] = cs;
    sn_s[i] = sn;
  }
  __syncthreads();
  bf16* pool_base = reinterpret_cast<bf16*>(pool.base);
  int page = 0, in_page = 0;
  if (use_pool) {
    page = pool.block_table[slot[m] * pool.bt_stride + p / pool.page_tokens];
    in_page = p % pool.page_tokens;
  }
  for (int idx = threadIdx.x; idx < (H + KVH) * half; idx += blockDim.x) {
    const int h = idx / half, i = idx % half;
    const float cs = cs_s[i], sn = sn_s[i];
    const float x1 = __bfloat162float(in[h * HD + i]);
    const float x2 = __bfloat162float(in[h * HD + i + half]);
    float r1, r2;
    rope_pair(x1, x2, cs, sn, r1, r2);
    const bf16 o1 = __float2bfloat16_rn(r1);
    const bf16 o2 = __float2bfloat16_rn(r2);
    if (h < H) {
      bf16* q = q_out + (static_cast<size_t>(m) * H + h) * HD;
      q[i] = o1;
      q[i + half] = o2;
    } else {
      const int kh = h - H;
      if (k_out) {
        bf16* k = k_out + (static_cast<size_t>(m) * KVH + kh) * HD;
        k[i] = o1;
        k[i + half] = o2;
      }
      if (use_pool) {
        bf16* k = pool_base + kv_elem_offset(pool, page, layer, kh, HD, in_page, false);
        k[i] = o1;
        k[i + half] = o2;
      }
    }
  }
  // values: plain copy, 4 bytes per thread
  const uint32_t* vin = reinterpret_cast<const uint32_t*>(in + (H + KVH) * HD);
  for (int idx = threadIdx.x; idx < KVH * half; idx += blockDim.x) {
    const int kh = idx / half, j = (idx % half) * 2;
    const uint32_t v = vin[idx];
    if (v_out) *reinterpret_cast<uint32_t*>(v_out + (static_cast<size_t>(m) * KVH + kh) * HD + j) = v;
    if (use_pool)
      *reinterpret_cast<uint32_t*>(pool_base + kv_elem_offset(pool, page, layer, kh, HD, in_page, true) + j) = v;
  }
}

template <int HD>
__global__ void rope_table_kernel(float2* tab, int max_pos, float log2_theta) {
  constexpr int half = HD / 2;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= max_pos * half) return;
  const int p = idx / half, i = idx % half;
  const float inv_freq = exp2f(-(2.0f * i / HD) * log2_theta);  // the expression of rope_qkv_kernel
  float sn, cs;
  sincosf(static_cast<float>(p) * inv_freq, &sn, &cs);
  tab[idx] = make_float2(cs, sn);
}

__global__ void scatter_int_kernel(const int* __restrict__ idx, const int* __restrict__ val, int n,
                                   int* __restrict__ dst) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[idx[i]] = val[i];
}

__global__ void copy_chunks_kernel(const CopyChunk* __restrict__ list) {
  const CopyChunk c = list[blockIdx.x];
  const int4* src = static_cast<const int4*>(c.src);
  int4* dst = static_cast<int4*>(c.dst);
  const size_t n = c.bytes / 16;
  size_t i = threadIdx.x;
  for (; i + 3 * blockDim.x < n; i += 4 * blockDim.x) {
    const int4 a = src[i], b = src[i + blockDim.x], cc = src[i + 2 * blockDim.x], d = src[i + 3 * blockDim.x];
    dst[i] = a;
    dst[i + blockDim.x] = b;
    dst[i + 2 * blockDim.x] = cc;
    dst[i + 3 * blockDim.x] = d;
  }
  for (; i < n; i += blockDim.x) dst[i] = src[i];
}

__global__ void cur_from_hist_kernel(const int* __restrict__ q, int n, const int* __restrict__ hist, int max_new,
                                     const int* __restrict__ prompts, int max_prompt, int* __restrict__ cur) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int slot = q[i], sid = q[n + i], gen = q[2 * n + i], P = q[3 * n + i];
  cur[slot] = gen > 0 ? hist[static_cast<size_t>(sid) * max_new + gen - 1]
                      : prompts[static_cast<size_t>(sid) * max_prompt + P - 1];
}

int grid_for(size_t n) {
  const size_t b = (n + 255) / 256;
  return static_cast<int>(b < 148 * 16 ? (b == 0 ? 1 : b) : 148 * 16);
}

}  // namespace

void init_bf16(bf16* w, size_t n, uint64_t seed, uint64_t tag, float scale, cudaStream_t st) {
  init_bf16_kernel<<<grid_for(n), 256, 0, st>>>(w, n, seed, tag, scale); fpk::count_launch();
}

void init_gain(float* g, size_t n, uint64_t seed, uint64_t tag, cudaStream_t st) {
  init_gain_kernel<<<grid_for(n), 256, 0, st>>>(g, n, seed, tag); fpk::count_launch();
}

void init_bf16_gu(bf16* w, int F, int d, uint64_t seed, uint64_t tag, float scale, cudaStream_t st) {
  init_bf16_gu_kernel<<<grid_for(static_cast<size_t>(2) * F * d), 256, 0, st>>>(w, F, d, seed, tag, scale); fpk::count_launch();
}

void embed_norm(const int* tokens, const int* idx, int M, const bf16* E, int d, float* x, const float* gain, bf16* y,
                cudaStream_t st) {
  if (M <= 0) return;
  if (d % 4 || d > 4096) throw std::invalid_argument("embed_norm: d must be a multiple of 4 and <= 4096");
  // a plain launch, like embed(): the step's first kernel fully orders the step
  embed_norm_kernel<<<M, ((d / 4 + 31) / 32) * 32, 0, st>>>(tokens, idx, E, d, x, gain, y);
  fpk::count_launch();
}

void embed(const int* tokens, const int* idx, int M, const bf16* E, int d, float* x, cudaStream_t st) {
  if (M <= 0) return;
  // a plain launch: the step's first kernel fully orders the step after the
  // previous one (the decode attention reads cached K/V before its PDL wait)
  embed_kernel<<<M, 128, 0, st>>>(tokens, idx, E, d, x);
  fpk::count_launch();
}

// 4-byte granular gather (experience hand-off: response segments start at
// arbitrary token offsets); 16-byte vectors when both ends are aligned.
__global__ void copy_words_kernel(const CopyChunk* __restrict__ list) {
  const CopyChunk c = list[blockIdx.x];
  const size_t n = c.bytes / 4;
  const uint32_t* src = static_cast<const uint32_t*>(c.src);
  uint32_t* dst = static_cast<uint32_t*>(c.dst);
  if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
    const size_t n4 = n / 4;
    for (size_t i = threadIdx.x; i < n4; i += blockDim.x)
      reinterpret_cast<int4*>(dst)[i] = reinterpret_cast<const int4*>(src)[i];
    for (size_t i = n4 * 4 + threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
  } else {
    for (size_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
  }
}

void copy_words(const CopyChunk* d_list, int n, cudaStream_t st) {
  if (n <= 0) return;
  copy_words_kernel<<<n, 128, 0, st>>>(d_list);
  fpk::count_launch();
}

void copy_chunks(const CopyChunk* d_list, int n, cudaStream_t st) {
  if (n <= 0) return;
  copy_chunks_kernel<<<n, 256, 0, st>>>(d_list); fpk::count_launch();
}

void cur_from_hist(const int* d_quad, int n, const int* hist_tok, int max_new, const int* prompts, int max_prompt,
                   int* cur_tok, cudaStream_t st) {
  if (n <= 0) return;
  cur_from_hist_kernel<<<(n + 127) / 128, 128, 0, st>>>(d_quad, n, hist_tok, max_new, prompts, max_prompt, cur_tok); fpk::count_launch();
}

void scatter_int(const int* idx, const int* val, int n, int* dst, cudaStream_t st) {
  if (n <= 0) return;
  scatter_int_kernel<<<(n + 255) / 256, 256, 0, st>>>(idx, val, n, dst); fpk::count_launch();
}

void assemble_batch(const AssembleArgs& a, int n, cudaStream_t st) {
  if (n <= 0) return;
  assemble_kernel<<<n, 256, 0, st>>>(a); fpk::count_launch();
}

void add_norm(float* x, const float* parts, int nsplit, size_t split_stride, const float* gain, bf16* y, int M, int d,
              const int* gather, int M_out, const bf16* value_w, float* value, cudaStream_t st, const L2Prefetch& pf) {
  const int rows = gather ? M_out : M;
  if (rows <= 0) return;
  const int ns = parts ? nsplit : 0;
  if (d % 4 || d > 4096) throw std::invalid_argument("add_norm: d must be a multiple of 4 and <= 4096");
  const dim3 grid(rows), block(((d / 4 + 31) / 32) * 32);
  const size_t sm = 0;
#define FP_AN(N_) \
  case N_: launch_pdl(add_norm_kernel<N_>, dim3(grid), dim3(block), sm, st, x, parts, split_stride, gain, y, d, gather, rows, value_w, value, pf); break;
  switch (ns) {
    FP_AN(0) FP_AN(1) FP_AN(2) FP_AN(3) FP_AN(4) FP_AN(5) FP_AN(6) FP_AN(7) FP_AN(8)
    default: throw std::invalid_argument("add_norm: at most 8 split-K partials");
  }
#undef FP_AN
  fpk::count_launch();
}

void rms_norm_rows(const float* x, const float* gain, bf16* y, int M, int d, cudaStream_t st) {
  if (M <= 0) return;
  const dim3 grid((M + 7) / 8), block(256);
  switch (d) {
    case 256: launch_pdl(rms_norm_rows_kernel<2>, grid, block, 0, st, x, gain, y, M); break;
    case 768: launch_pdl(rms_norm_rows_kernel<6>, grid, block, 0, st, x, gain, y, M); break;
    case 1024: launch_pdl(rms_norm_rows_kernel<8>, grid, block, 0, st, x, gain, y, M); break;
    case 2048: launch_pdl(rms_norm_rows_kernel<16>, grid, block, 0, st, x, gain, y, M); break;
    case 4096: launch_pdl(rms_norm_rows_kernel<32>, grid, block, 0, st, x, gain, y, M); break;
    default:  // other widths: the block-per-row kernel
      add_norm(const_cast<float*>(x), nullptr, 0, 0, gain, y, M, d, nullptr, 0, nullptr, nullptr, st);
      return;
  }
  fpk::count_launch();
}

void rope_qkv(const bf16* qkv, int M, int H, int KVH, int hd, const int* pos, float rope_theta, bf16* q_out,
              bf16* k_out, bf16* v_out, const KvPoolView* pool, int layer, const int* slot, cudaStream_t st) {
  if (M <= 0) return;
  KvPoolView pv{};
  if (pool) pv = *pool;
  const float l2 = log2f(rope_theta);
  const int up = pool != nullptr ? 1 : 0;
  switch (hd) {
    case 32: rope_qkv_kernel<32><<<M, 128, 0, st>>>(qkv, H, KVH, pos, l2, q_out, k_out, v_out, pv, up, layer, slot); break;
    case 64: rope_qkv_kernel<64><<<M, 128, 0, st>>>(qkv, H, KVH, pos, l2, q_out, k_out, v_out, pv, up, layer, slot); break;
    case 128: rope_qkv_kernel<128><<<M, 128, 0, st>>>(qkv, H, KVH, pos, l2, q_out, k_out, v_out, pv, up, layer, slot); break;
    default: throw std::invalid_argument("rope_qkv: head_dim must be 32, 64 or 128");
  }
  fpk::count_launch();
}

void rope_table(float2* tab, int max_pos, int hd, float rope_theta, cudaStream_t st) {
  const float l2 = log2f(rope_theta);
  const int n = max_pos * hd / 2;
  switch (hd) {
    case 32: rope_table_kernel<32><<<(n + 255) / 256, 256, 0, st>>>(tab, max_pos, l2); break;
    case 64: rope_table_kernel<64><<<(n + 255) / 256, 256, 0, st>>>(tab, max_pos, l2); break;
    case 128: rope_table_kernel<128><<<(n + 255) / 256, 256, 0, st>>>(tab, max_pos, l2); break;
    default: throw std::invalid_argument("rope_table: head_dim must be 32, 64 or 128");
  }
  fpk::count_launch();
}

__global__ void checksum64_kernel(const unsigned long long* __restrict__ w, size_t n, unsigned long long* out) {
  unsigned long long acc = 0;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    acc += w[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, acc);  // integer sums: order-independent
}

void checksum64(const void* p, size_t bytes, unsigned long long* out, cudaStream_t st) {
  checksum64_kernel<<<296, 256, 0, st>>>(static_cast<const unsigned long long*>(p), bytes / 8, out);
  fpk::count_launch();
}

}  // namespace fpk
