// fuseplan-b200 — host-callable launchers of the sm_100a kernels.
// Every function enqueues on `st` and never synchronises.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <vector>

namespace fpk {

using bf16 = __nv_bfloat16;

// Number of kernels this library has launched (all launchers count).
void count_launch();
void count_launches(long long n);  // graph replays: the kernels the graph holds
long long launch_count();

// Packed forwards (M >= 1024 rows) take the persistent GEMM / attention
// kernels, which hold every SM for their whole duration. While the same GPU
// is still decoding, scoring turns this off (calling thread only) so its
// one-tile-per-CTA kernels leave room for the decode step's CTAs.
void set_packed_persistent(bool on);
bool packed_persistent();
void set_pair_gemm(int mode);  // packed GEMMs on SM pairs (cta_group::2): -1 auto (default), 0 never, 1 always

// ---- GEMMs (tcgen05; gemm.cu) --------------------------------------------------
// swap-AB: out[m][n] = sum_k X[m][k] W[n][k]; W [N, K], X [M, K], K % 64 == 0.
void gemm_bf16(const bf16* W, int N, int K, const bf16* X, int M, bf16* out, int ld_out, cudaStream_t st);
// fp32 split-K partials: out[s][m][n] for s < splits (see gemm_splits()).
void gemm_f32_splitk(const bf16* W, int N, int K, const bf16* X, int M, float* out, int splits, cudaStream_t st);
// resid[m][n] += sum_k X[m][k] W[n][k] (single split; residual add fused).
void gemm_f32_residual(const bf16* W, int N, int K, const bf16* X, int M, float* resid, cudaStream_t st);
// SwiGLU, W_gu [2F, K] interleaved in 64-row gate/up groups: out[m][f], ld = F.
void gemm_swiglu(const bf16* Wgu, int F, int K, const bf16* X, int M, bf16* out, cudaStream_t st);
// Decode variant: lean rings for small batches (the next GEMM's CTAs co-reside under PDL).
void gemm_swiglu_decode(const bf16* Wgu, int F, int K, const bf16* X, int M, bf16* out, cudaStream_t st);
// Split count used by gemm_f32_splitk for an (N, K) weight; a function of the
// weight shape only, so each row's result does not depend on the batch.
int gemm_splits(int N, int K);
// Debug: per-CTA phase stamps of subsequent GEMM launches (nullptr disables).
void set_gemm_trace(unsigned long long* buf);

struct VocabOut;  // fwd
// Largest top_k of the filtered sampler (topk_sample); top_p alone filters
// within the top kTopKMax logits.
constexpr int kTopKMax = 1024;
// Vocab head: rows X [M, K] against W_head [V, K]; writes per-(row, tile)
// partials into `part` (M x vocab_tiles(V) VocabPartial = 24 B each, two
// 128-column halves per 256-wide vocab tile) and, in
// forced mode, tgt_z[M]. mode: 0 forced (target[]), 1 greedy, 2 sample.
int vocab_tiles(int V);
void gemm_vocab(const bf16* X, int M, int K, const bf16* Whead, int V, int mode, float inv_temp,
                const int* target, const int* sample_id, const int* step, uint64_t seed, void* part, float* tgt_z,
                cudaStream_t st);
// Filtered sampling, step 1: the same head GEMM keeping the log-softmax
// partials and writing z = logit * inv_temp to logits [M][ldv] (fp32).
void gemm_vocab_logits(const bf16* X, int M, int K, const bf16* Whead, int V, float inv_temp, void* part,
                       float* logits, int ldv, cudaStream_t st);
// Step 2 (sampling.cu), one CTA per row: the k-th largest z by an exact
// radix select (k = top_k, or kTopKMax when top_k == 0; ties at the boundary
// kept), the candidates sorted by (z desc, id asc), the nucleus = the
// shortest sorted prefix whose softmax mass reaches top_p of the candidates'
// mass, and an inverse-CDF draw in that order with
// u = Philox(seed, sample_id, step, counter kFilterDraw). pick[row] = token,
// pick_z[row] = its z (step 3 is vocab_finalize in forced mode on pick:
// log-prob under the full temperature softmax, scatter, next input).
void topk_sample(const float* logits, int ldv, int M, int V, int top_k, float top_p, const int* sample_id,
                 const int* step, uint64_t seed, int* pick, float* pick_z, cudaStream_t st);
// Merge partials: token[row] (forced -> target), logp[row]; optional scatter
// into per-sample buffers: out_tok[dst[row]] / out_logp[dst[row]] when dst != nullptr.
// cur_tok[cur_idx[row]] = token (next decode input) when cur_tok != nullptr.
// Sampling (mode 2) draws the half-tile with Philox(seed, sample_id[row], step[row], 0xFFFFFFFF).
void vocab_finalize(const void* part, const float* tgt_z, int M, int V, int mode, const int* target,
                    const int* sample_id, const int* step, uint64_t seed, int* token, float* logp, const int* dst,
                    int* out_tok, float* out_logp, const int* cur_idx, int* cur_tok, cudaStream_t st);

// ---- elementwise / norms (layers.cu) ----------------------------------------------
void init_bf16(bf16* w, size_t n, uint64_t seed, uint64_t tag, float scale, cudaStream_t st);
void init_gain(float* g, size_t n, uint64_t seed, uint64_t tag, cudaStream_t st);
// Gate/up weight [2F, d] stored in 64-row interleaved groups (see EpiSwiGLU);
// the hash index is that of the logical [gate; up] matrix.
void init_bf16_gu(bf16* w, int F, int d, uint64_t seed, uint64_t tag, float scale, cudaStream_t st);
// x[m] = E[tokens[idx ? idx[m] : m]] (fp32 residual stream).
void embed(const int* tokens, const int* idx, int M, const bf16* E, int d, float* x, cudaStream_t st);
// embed + the first RMSNorm in one launch (decode step head): same bits as embed then add_norm (no partials).
void embed_norm(const int* tokens, const int* idx, int M, const bf16* E, int d, float* x, const float* gain, bf16* y,
                cudaStream_t st);
// Packed scoring batch: for sample j (global id sid[j], prompt P[j], response
// R[j], rows [cu[j], cu[j+1])): tokens = prompt ++ response, pos = 0..T-1;
// response-aligned outputs at [roff[j], roff[j] + R[j]): targets (response
// ids), logp_actor (from the generator's history), gather_resp (row of
// position P-1+k); gather_last[j] = row of position T-1.
struct AssembleArgs {
  const int* sid; const int* P; const int* R; const int* cu; const int* roff;
  const int* prompts; int max_prompt;            // [n_global][max_prompt]
  const int* const* hist_tok; const float* const* hist_logp;  // per sample j: base of that sample's row
  int* tokens; int* pos; int* targets; float* logp_actor; int* gather_resp; int* gather_last;
};
void assemble_batch(const AssembleArgs& a, int n, cudaStream_t st);
// For output row i (src = gather ? gather[i] : i): xs = x[src] + sum_s parts[s][src];
// if !gather, x[src] = xs. y[i] = bf16(rmsnorm(xs) * g). If value_w != nullptr,
// instead value[i] = dot(rmsnorm(xs) * g, value_w) and y is not written.
// Weight ranges to pull into L2 while a small kernel runs (the next GEMMs'
// weights: their first TMA loads then hit L2 instead of waiting on DRAM).
struct L2Prefetch {
  const void* p[2] = {nullptr, nullptr};
  size_t bytes[2] = {0, 0};
};
void add_norm(float* x, const float* parts, int nsplit, size_t split_stride, const float* gain, bf16* y, int M,
              int d, const int* gather, int M_out, const bf16* value_w, float* value, cudaStream_t st,
              const L2Prefetch& pf = L2Prefetch{});
// y = bf16(RMSNorm(x) * gain) for the packed forward (no partials / gather): one
// warp per row (layers.cu rms_norm_rows_kernel).
void rms_norm_rows(const float* x, const float* gain, bf16* y, int M, int d, cudaStream_t st);

// RoPE on q, k of a packed qkv [M, (H + 2 KVH) * hd] row block; q -> q_out
// [M, H, hd]; k, v -> either contiguous k_out/v_out [M, KVH, hd] and/or the
// paged pool (pool != nullptr): token (slot[i], pos[i]).
struct KvPoolView {
  uint8_t* base;          // page 0
  size_t page_bytes;      // bytes per page (all layers)
  size_t layer_bytes;     // bytes per layer inside a page
  int page_tokens;        // tokens per page
  const int* block_table; // [slots][max_pages]
  int bt_stride;          // max_pages
  const CUtensorMap* kv_map = nullptr;  // host copy: 2-D TMA view of the pool (make_kv_map), hd 64/128
};
#ifdef __CUDACC__
#include <math.h>
// Merge ns context splits of one (sample, head) row: partial o [ns][HD]
// (unnormalised) and (m, l) pairs at part_*[base ..]; threads t, t + nt, ...
// of the caller write out[d]. Shared by the combine kernel and the fused
// last-split merge, with explicit roundings, so both give the same bits
// (one split: f = 1 and out = o / l exactly). L2 loads: the partials were
// written by other SMs.
__device__ __forceinline__ void combine_row(const float* part_o, const float* part_ml, size_t base, int ns, int HD,
                                            int t, int nt, __nv_bfloat16* out) {
  float M = -INFINITY;
  for (int s = 0; s < ns; ++s) M = fmaxf(M, __ldcg(part_ml + (base + s) * 2));
  for (int d = t; d < HD; d += nt) {
    float L = 0.f, O = 0.f;
    for (int s = 0; s < ns; ++s) {
      const float f = exp2f(__ldcg(part_ml + (base + s) * 2) - M);
      L = __fmaf_rn(__ldcg(part_ml + (base + s) * 2 + 1), f, L);
      O = __fmaf_rn(__ldcg(part_o + (base + s) * HD + d), f, O);
    }
    out[d] = __float2bfloat16_rn(__fdiv_rn(O, L));
  }
}
// Element offset of token `tok` of (page, layer, kv head) K (or V) in the pool.
__device__ __forceinline__ size_t kv_elem_offset(const KvPoolView& p, int page, int layer, int kvh, int hd, int tok,
                                                 bool is_v) {
  const size_t head_elems = static_cast<size_t>(2) * p.page_tokens * hd;
  return (static_cast<size_t>(page) * p.page_bytes + static_cast<size_t>(layer) * p.layer_bytes) / 2 +
         kvh * head_elems + (is_v ? static_cast<size_t>(p.page_tokens) * hd : 0) + static_cast<size_t>(tok) * hd;
}
// Rotate-half RoPE of the pair (x1, x2) = (x[i], x[i + hd/2}) with (cos, sin);
// explicit roundings (no FMA contraction) so every kernel that rotates agrees
// bit-for-bit with the others and with the oracle.
__device__ __forceinline__ void rope_pair(float x1, float x2, float cs, float sn, float& o1, float& o2) {
  o1 = __fsub_rn(__fmul_rn(x1, cs), __fmul_rn(x2, sn));
  o2 = __fadd_rn(__fmul_rn(x2, cs), __fmul_rn(x1, sn));
}
#endif
// RoPE table: tab[p * hd/2 + i] = (cos, sin)(p * theta^(-2i/hd)) for p < max_pos.
void rope_table(float2* tab, int max_pos, int hd, float rope_theta, cudaStream_t st);
// Decode QKV projection with RoPE and the KV-cache append fused into the
// epilogue: qkv = X W^T (never stored); q -> q_out [M, H, hd]; the new
// token's K / V -> the pool at (slot[m], pos[m]) of `layer`. cs: rope_table.
void gemm_qkv_rope(const bf16* Wqkv, int K, const bf16* X, int M, int H, int KVH, int hd, const int* pos,
                   const float2* cs, const KvPoolView& pool, int layer, const int* slot, bf16* q_out,
                   cudaStream_t st);
// The same for packed rows (prefill / scoring): q_out [M, H, hd]; K / V into
// k_out / v_out [M, KVH, hd] (optional) and, with a pool, at (slot[m], pos[m]).
// Bit-identical to gemm_bf16 + rope_qkv (same tiles, roundings and table).
void gemm_qkv_rope_packed(const bf16* Wqkv, int K, const bf16* X, int M, int H, int KVH, int hd, const int* pos,
                          const float2* cs, const KvPoolView* pool, int layer, const int* slot, bf16* q_out,
                          bf16* k_out, bf16* v_out, cudaStream_t st);
// The decode layer's GEMM chain in one persistent launch (chain.cu): O-proj
// split-K -> residual + RMSNorm (gain_mlp) -> gate/up SwiGLU -> down split-K ->
// residual + RMSNorm (gain_next) -> [next layer's QKV + RoPE + KV append when
// wqkv != nullptr]; grid-wide barriers between the phases. Bit-identical to
// gemm_f32_splitk / add_norm / gemm_swiglu_decode / gemm_qkv_rope.
// counters: 8 ints, zero, left zero. false: shape unsupported (nothing launched).
struct DecodeChain {
  const bf16 *wo, *wgu, *wd, *wqkv;  // layer l's O / gate-up / down; layer l+1's QKV (nullptr: last layer)
  const bf16* attn;                   // [B][ao] attention output of layer l
  bf16* h;                            // [B][d] norm output (GEMM input)
  bf16* act;                          // [B][F]
  float* parts;                       // [8][B][d] split-K partials
  float* x;                           // [B][d] residual stream
  const float *gain_mlp, *gain_next;  // ln2 of layer l; ln1 of layer l+1 or the final norm
  bf16* q_out;                        // [B][H][hd] (layer l+1)
  KvPoolView pool;
  const int *slot, *pos;
  const float2* cs;
  int layer;                          // l (the QKV phase writes layer l + 1's K / V)
  int H, KVH, hd, d, F, ao, B;
  int* counters;
  int ctas;                           // persistent grid size (<= SMs)
};
bool decode_chain(const DecodeChain& c, cudaStream_t st);

// 2-D TMA map over the pool viewed as [rows, hd] bf16 rows (one row = one
// token's K or V of one (page, layer, kv head)); box {64, 32}, 128 B swizzle.
CUtensorMap make_kv_map(const void* pool, long long rows, int hd);
// Tokens per decode-attention split (position-determined).
constexpr int kDecodeChunk = 512;
// Tensor-core decode attention (attn_decode.cu); false if (hd, group) unsupported or no map.
// Work items are (sample, non-empty split, kv head) — or, for long splits when
// a batch is large enough that the warp-per-item kernel runs, one 128-token
// sub-chunk of a split (its partial is folded with the others by the last to
// finish, in sub-chunk order: the same bits as one warp folding them) —
// handed out dynamically through counters[0..1] in the order of `items`
// (attn_decode_items, longest first). The splits of a (sample, kv head) merge
// inside the kernel too (tickets). counters: attn_decode_counters ints, zero,
// left zero.
bool attn_decode_mma(const bf16* q, int B, int H, int KVH, int hd, const KvPoolView& pool, int layer,
                     const int* slot, const int* ctx, const int* items, int nsplit, float* work, bf16* out,
                     int* counters, cudaStream_t st, int max_ctas = 148);
// Debug: per-warp (entry ns, loop-begin ns, end ns, units) of subsequent
// warp-per-item decode-attention launches into buf (4 x 148 x warps); nullptr disables.
void set_attn_trace(unsigned long long* buf);
// Step timeline tracing (tools/step_trace.py): while armed, every GEMM and
// decode-attention launch gets its own slice of the arena for globaltimer
// stamps (GEMM: 8 words per CTA; attention: 4 words per warp or per team
// CTA) and a host record. Eager launches only (the engine disables the step
// graph for the traced step).
struct TraceRec {
  int kind;    // 0 GEMM, 1 warp-per-item attention, 2 team attention
  int units;   // CTAs (GEMM, team) or warps (attention)
  size_t off;  // word offset in the arena
};
void trace_arm(unsigned long long* arena, size_t words);
unsigned long long* trace_slot(int kind, int units, int words_per_unit);  // nullptr when not armed
std::vector<TraceRec> trace_disarm();
inline int attn_decode_counters(int B, int KVH, int max_ctx) {
  const int ns = (max_ctx + kDecodeChunk - 1) / kDecodeChunk;
  return 2 + B * KVH + B * KVH * ns;  // work queue, split tickets, sub-chunk tickets
}
// Which kernel shape attn_decode_mma runs for a batch: 0 warp-per-item wide,
// 1 warp-per-item deep, 2 team; `warps` = its warps per CTA.
int attn_decode_variant(int B, int KVH, int hd, int G, int* warps);
// Host: the item table from the contexts: items[0] = n, items[1..n] =
// b << 11 | split << 3 | sub (sub 7: the whole split), longest first (an LPT
// order for the dynamic schedule); ties by (b, split, sub). Splits are cut
// into 128-token sub-chunks only under set_attn_cut (default never); same bits
// either way.
// Capacity: 1 + B * ceil(max_ctx / 128) ints.
int attn_decode_items(const int* ctx, int B, int KVH, int hd, int G, int* items);
void set_attn_cut(int mode);  // calling thread: 0 never cut (default), 1 always, -1 small-batch rule
void rope_qkv(const bf16* qkv, int M, int H, int KVH, int hd, const int* pos, float rope_theta, bf16* q_out,
              bf16* k_out, bf16* v_out, const KvPoolView* pool, int layer, const int* slot, cudaStream_t st);

// ---- attention (attention.cu) -----------------------------------------------------
// Decode: q [B, H, hd] (one token per row), paged K/V of `layer`; ctx[b]
// tokens visible (including the one just appended). out [B, H, hd] bf16.
// work: float scratch of attn_decode_workspace(B, H, hd, max_ctx) floats.
size_t attn_decode_workspace(int B, int H, int hd, int max_ctx);  // split + sub-chunk partials
// counters / items (see attn_decode_mma) enable the tensor-core kernel with
// its fused split merge; nullptr runs the CUDA-core kernel + combine kernel.
// probe_begin / probe_end (optional) bracket the main split kernel (not the combine).
void attn_decode(const bf16* q, int B, int H, int KVH, int hd, const KvPoolView& pool, int layer, const int* slot,
                 const int* ctx, const int* items, int max_ctx, float* work, bf16* out, int* counters,
                 cudaStream_t st,
                 cudaEvent_t probe_begin = nullptr, cudaEvent_t probe_end = nullptr, int max_ctas = 148);
// Varlen causal attention over packed q [M, H, hd], k/v [M, KVH, hd];
// sequences [cu[i], cu[i+1]). tiles: host-built table of (seq, q_tile) pairs
// (attn_varlen_tiles; the query-tile height depends on hd). out [M, H, hd].
// hd 64 / 128 run the tcgen05 kernel (attn_prefill.cu), other head sizes the
// mma.sync kernel (attention.cu).
int attn_varlen_tile_rows(int hd);
int attn_tiles(const int* cu_host, int n_seq, int rows, int* tiles_host);  // (seq, tile) pairs, most keys first
int attn_varlen_tiles(const int* cu_host, int n_seq, int hd, int* tiles_host);
void attn_varlen(const bf16* q, const bf16* k, const bf16* v, int H, int KVH, int hd, int M, const int* cu,
                 const int* tiles, int n_tiles, bf16* out, cudaStream_t st);
bool attn_prefill_supported(int hd);
void attn_prefill_set_trace(unsigned long long* buf);  // debug: CTA 0 event times [8][64] (nullptr: off)
void attn_prefill(const bf16* q, const bf16* k, const bf16* v, int H, int KVH, int hd, int M, const int* cu,
                  const int* tiles, int n_tiles, bf16* out, cudaStream_t st);
// The mma.sync kernel for any supported hd (64-row query tiles); kept for
// hd 32 and as the cross-check of the tcgen05 kernel in the GPU tests.
void attn_varlen_mma(const bf16* q, const bf16* k, const bf16* v, int H, int KVH, int hd, const int* cu,
                     const int* tiles, int n_tiles, bf16* out, cudaStream_t st);

// ---- post-processing (post.cu) -----------------------------------------------------
// Per sample i, inputs at tokens [off[i], off[i+1]): kl, reward, advantage,
// return (fp32). Outputs go to the same packed offsets, or — with `scatter` —
// to [off_out[i], off_out[i] + R_i) of the global experience arrays, together
// with copies of logp_actor / logp_ref / values / token ids and score[sid[i]].
struct PostScatter {
  const int64_t* off_out; const int* sid; const int* tokens_in;
  float *logp_actor, *logp_ref, *values, *score_out; int* tokens_out;
};
void postprocess(int n, const int* off, const float* logp_actor, const float* logp_ref, const float* values,
                 const float* score, float beta, float gamma, float lam, float* kl, float* reward, float* adv,
                 float* ret, cudaStream_t st, const PostScatter* scatter = nullptr);
// Bulk copies (e.g. KV pages pulled from a peer GPU over NVLink, history
// rows): one CTA per chunk, 16-byte vector loads; src/dst/bytes 16-aligned.
struct CopyChunk { const void* src; void* dst; unsigned long long bytes; };
void copy_chunks(const CopyChunk* d_list, int n, cudaStream_t st);
// The same at 4-byte granularity (src/dst/bytes multiples of 4).
void copy_words(const CopyChunk* d_list, int n, cudaStream_t st);
// cur_tok[slot[i]] = gen[i] > 0 ? hist[sid[i]][gen[i]-1] : prompts[sid[i]][P[i]-1]
void cur_from_hist(const int* d_quad, int n, const int* hist_tok, int max_new, const int* prompts, int max_prompt,
                   int* cur_tok, cudaStream_t st);  // d_quad: [4][n] = slot, sid, gen, P
// *out += sum of the 64-bit words of [p, p + bytes) (bytes % 8 == 0; *out zeroed by the caller)
void checksum64(const void* p, size_t bytes, unsigned long long* out, cudaStream_t st);
// dst[idx[i]] = val[i]
void scatter_int(const int* idx, const int* val, int n, int* dst, cudaStream_t st);

}  // namespace fpk
