/* fuseplan-b200 — C ABI of the B200 experience-collection engine.
 *
 * Same conventions as fp_sched.h (status codes FP_OK / FP_EINVAL /
 * FP_EINFEASIBLE / FP_EINTERNAL, fp_last_error(), caller-owned host buffers,
 * engine-owned device memory, no exceptions across the boundary).
 *
 * What it replaces in the reference: simulate_serial / simulate_fused
 * (proj/include/fuseplan/genfuse.hpp:113-121, proj/src/genfuse.cpp:469-515)
 * model generation and scoring with cost formulas (prefill_seconds /
 * score_seconds / decode_step_base, genfuse.cpp:26-41, 243-245); fp_execute
 * runs the same schedule for real on B200s and returns the experience batch,
 * measured times, and the decision-clock result it executed (which is exactly
 * what simulate_* return, so reference callers keep their outputs).
 *
 * Multi-GPU: one process per GPU; every rank calls fp_execute with the same
 * batch / config and fp_comm{rank, world, shm_name}. cfg->num_instances must
 * equal world. Rank 0's experience is the gathered batch.
 *
 * The fp_k_* entry points expose single kernels on caller-provided device
 * pointers for parity tests (stream = cudaStream_t or NULL).
 */
#ifndef FP_ENGINE_H_
#define FP_ENGINE_H_

#include <stddef.h>
#include <stdint.h>

#include "fp_sched.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fp_model_dims {
  int32_t num_layers, hidden, num_heads, num_kv_heads, head_dim, ffn, vocab;
} fp_model_dims;

typedef struct fp_engine_setup {
  fp_model_dims actor, ref, critic, reward; /* critic/reward: vocab = embedding size only */
  uint64_t weight_seed;
  int32_t max_prompt, max_new, max_samples, max_live;
  int64_t kv_pool_bytes; /* 0: max_live x (max_prompt + max_new) tokens */
  int32_t max_prefill_tokens, max_infer_tokens;
  float rope_theta;
  int32_t device;
} fp_engine_setup;

enum { FP_TOKENS_FORCED = 0, FP_TOKENS_GREEDY = 1, FP_TOKENS_SAMPLE = 2 };
enum { FP_SCHEDULE_STAGE_BARRIER = 0, FP_SCHEDULE_FUSED = 1 };

typedef struct fp_run_options {
  int32_t token_mode, schedule;
  float temperature;
  uint64_t token_seed, sample_seed;
  float kl_beta, gamma, lam;
  int32_t claim_tokens, run_ahead;
  int32_t resident;        /* 1: prompts already resident (same as previous call), experience kept on device */
  int32_t probe_attention; /* 1: time each decode-attention launch (stats.attn_probe_*) */
  int32_t handoff_dp;      /* > 0: pack the experience into length-balanced DP mini-batches (fp_exec_handoff) */
  int32_t claim_max_live;  /* > 0: a generating rank scores only while its decode batch <= this */
  /* Free-run (north_star "retires each sample as it emits EOS"): eos_id >= 0
   * retires a sample at its first emitted eos_id (kept as the last response
   * token) or at max_new; greedy / sample modes; the fused trigger is then
   * online. eos_lag: steps between a decode step and the host reading its ids. */
  int32_t eos_id, eos_lag;
  /* 1: online fused trigger on world > 1 (fewer than r_t unfinished samples
   * batch-wide; plan_migration on the ranks' live state). 0: decision clock. */
  int32_t online_trigger;
  /* Filtered sampling (FP_TOKENS_SAMPLE): top_k in [0, 1024] (0 off), top_p in (0, 1] (1 off). */
  int32_t top_k;
  float top_p;
} fp_run_options;

typedef struct fp_comm {
  int32_t rank, world;
  const char* shm_name; /* POSIX shm name shared by all ranks ("/..."); NULL if world == 1 */
} fp_comm;

typedef struct fp_exec_stats {
  double wall_seconds, gen_seconds, trigger_seconds, migrate_seconds, infer_busy_seconds, decode_gpu_seconds;
  int64_t decode_steps, decode_rows, decode_ctx_tokens, prefill_tokens, infer_tokens, infer_samples;
  int64_t migrated_in, migrated_bytes;
  int64_t total_resp;
  int64_t gpu_launches;
  double attn_probe_ms, attn_probe_bytes;
  int64_t attn_probe_launches;
  double ipc_seconds;
  int64_t eos_retired, overrun_rows; /* free-run: EOS retirements; row-steps decoded past an unseen EOS */
  int32_t online;                    /* 1: the trigger was taken online */
} fp_exec_stats;

typedef struct fp_engine fp_engine;
typedef struct fp_exec fp_exec;

int fp_engine_create(const fp_engine_setup* setup, fp_engine** out);
void fp_engine_destroy(fp_engine* e);
/* model: 0 actor, 1 ref, 2 critic, 3 reward. Weight bytes (device) and parameter count. */
int fp_engine_model_size(const fp_engine* e, int32_t model, int64_t* bytes, int64_t* params);
/* Physical KV bytes per token of the actor (bf16 K + V, GQA-aware). */
int fp_engine_kv_bytes_per_token(const fp_engine* e, int64_t* bytes);
/* Synthetic prompt ids [n][max_prompt] for token_seed. */
int fp_synthetic_prompts(const fp_engine* e, int32_t n, uint64_t token_seed, int32_t* out);

/* Weight sync (reference: the per-iteration actor weight redistribution,
 * workflow.cpp:94-102): every rank calls it with the same
 * model slot, src rank and comm (a fresh shm name); rank r ends with src's
 * weights, pulled over NVLink (scatter + all-gather). seconds: this rank's time. */
int fp_engine_broadcast_model(fp_engine* e, int32_t model, int32_t src, const fp_comm* comm, double* seconds);
/* Device pointer and size of a model's weight blob (engine layout), e.g. for a
 * trainer writing updated weights in place before fp_engine_broadcast_model. */
int fp_engine_model_ptr(const fp_engine* e, int32_t model, void** dev_ptr, int64_t* bytes);
/* Weight loading (the models InferenceTask / GenSimConfig::actor name,
 * genfuse.hpp:45-57): copy one standard row-major host tensor into the
 * engine's layout (repacked on the way: the gate / up rows are interleaved in
 * 64-row groups for the SwiGLU epilogue). model: 0 actor, 1 ref, 2 critic,
 * 3 reward; layer: 0 for the per-model tensors. Shapes (d hidden, F ffn,
 * V vocab, H/KVH heads, hd head_dim), dtype bf16 unless noted:
 *   FP_W_EMBED [V][d]; FP_W_QKV [(H + 2 KVH) hd][d] (q heads, then k, then v);
 *   FP_W_O [d][H hd]; FP_W_GATE, FP_W_UP [F][d]; FP_W_DOWN [d][F];
 *   FP_W_ATTN_NORM, FP_W_MLP_NORM, FP_W_FINAL_NORM [d] fp32 gains;
 *   FP_W_HEAD [V][d] (actor / ref); FP_W_VALUE_HEAD [d] (critic / reward).
 * n_elems must equal the tensor's size. Synchronous. */
enum {
  FP_W_EMBED = 0, FP_W_QKV = 1, FP_W_O = 2, FP_W_GATE = 3, FP_W_UP = 4, FP_W_DOWN = 5, FP_W_ATTN_NORM = 6,
  FP_W_MLP_NORM = 7, FP_W_FINAL_NORM = 8, FP_W_HEAD = 9, FP_W_VALUE_HEAD = 10
};
int fp_engine_load_weights(fp_engine* e, int32_t model, int32_t tensor, int32_t layer, const void* host,
                           int64_t n_elems);
/* Tooling: regenerate a model's synthetic weights from `seed`; order-independent
 * 64-bit checksum of its blob. */
int fp_engine_reinit_model(fp_engine* e, int32_t model, uint64_t seed);
int fp_engine_model_checksum(fp_engine* e, int32_t model, uint64_t* sum);
/* Run the stage. prompts: [n][max_prompt] ids or NULL (synthetic). */
int fp_execute(fp_engine* e, const fp_gen_sample* batch, int32_t n, const fp_gen_config* cfg, int32_t r_t,
               const fp_run_options* opts, const fp_comm* comm, const int32_t* prompts, fp_exec** out);
int fp_exec_stats_get(const fp_exec* x, fp_exec_stats* s);
/* Experience, response-aligned (total_resp entries; sample i owns
 * [resp_off[i], resp_off[i+1])) plus score[n]. Any pointer may be NULL. */
int fp_exec_experience(const fp_exec* x, int64_t* resp_off, int32_t* tokens, float* logp_actor, float* logp_ref,
                       float* values, float* kl, float* reward, float* adv, float* ret, float* score);
/* Per sample: GPU-clock finish time (s) and the instance it finished on (-1: other rank). */
int fp_exec_finish(const fp_exec* x, double* finish_seconds, int32_t* finish_instance);
/* Decision-clock GenStageResult of the executed schedule (free with fp_result_free). */
int fp_exec_decision(const fp_exec* x, fp_result** out);
/* Trigger / plan actually executed (fused, world > 1); moves in application order. */
int fp_exec_moves(const fp_exec* x, int32_t* n_moves, int32_t* sample, int32_t* from, int32_t* to);
/* Samples this rank received at the migration, (sample, source rank) in
 * application order — what the executor actually pulled (in flight: KV
 * pages or recompute; queued: re-queued). */
int fp_exec_received(const fp_exec* x, int32_t* n, int32_t* sample, int32_t* from);
/* Trigger state the executed plan was taken on (GenState, genfuse.hpp:67-79):
 * time, and per unfinished sample id / instance / kv_bytes / generated /
 * prompt_len / admitted (fp_remaining of fp_sched.h); NULL to query the count. */
int fp_exec_trigger_state(const fp_exec* x, double* time, int32_t* n, fp_remaining* samples);
/* Experience hand-off (handoff_dp > 0; balance_minibatch, workflow.hpp:63-66):
 * order[n], group_off[dp+1], packed_off[n+1] (response-token offsets in
 * order); this rank's groups [*group_begin, *group_end) and device pointers
 * dev[9] = tokens, logp_actor, logp_ref, values, kl, reward, adv, ret, score of
 * its packed range (engine-owned, valid until the next fp_execute). Any
 * pointer may be NULL. */
int fp_exec_handoff(const fp_exec* x, int32_t* dp, int32_t* group_begin, int32_t* group_end, int32_t* order,
                    int32_t* group_off, int64_t* packed_off, void** dev, double* seconds, int64_t* bytes,
                    int64_t* peer_bytes);
/* Copy this rank's packed hand-off range to host buffers (sizes from
 * fp_exec_handoff: tokens / arrays hold packed_off[group_off[end]] -
 * packed_off[group_off[begin]] entries, score group_off[end] - group_off[begin]).
 * host[9] in the order of dev[]; NULL entries are skipped. */
int fp_exec_handoff_download(const fp_exec* x, void** host);
/* Per decode step of this rank: batch rows, GPU milliseconds and visible context tokens summed over the
 * rows (n_steps entries; NULL to query / skip). */
int fp_exec_steps(const fp_exec* x, int32_t* n_steps, int32_t* rows, float* ms, int64_t* ctx);
void fp_exec_free(fp_exec* x);

/* ---- single-kernel entry points (device pointers) ---- */
int fp_k_init_bf16(void* w, int64_t n, uint64_t seed, uint64_t tag, float scale, void* stream);
int fp_k_gemm_bf16(const void* W, int32_t N, int32_t K, const void* X, int32_t M, void* out, int32_t ld,
                   void* stream);
int fp_k_gemm_f32(const void* W, int32_t N, int32_t K, const void* X, int32_t M, float* out, int32_t splits,
                  void* stream); /* splits <= 0: fp_k_gemm_splits(N, K) */
int fp_k_gemm_splits(int32_t N, int32_t K);
/* resid[M][N] += X W^T (fp32 residual stream; TMA reduce-add epilogue). */
int fp_k_gemm_f32_residual(const void* W, int32_t N, int32_t K, const void* X, int32_t M, float* resid,
                           void* stream);
/* Debug: record 8 globaltimer stamps per CTA of subsequent GEMMs into buf (device, NULL disables). */
int fp_k_gemm_trace(void* buf);
int fp_k_gemm_swiglu(const void* Wgu, int32_t F, int32_t K, const void* X, int32_t M, void* out, void* stream);
/* The decode-step SwiGLU GEMM (lean shared-memory rings for small M, so the next GEMM's CTAs co-reside under PDL). */
int fp_k_gemm_swiglu_decode(const void* Wgu, int32_t F, int32_t K, const void* X, int32_t M, void* out,
                            void* stream);
/* Decode QKV projection with RoPE and the KV append fused (one kernel):
 * q_out [M, H, hd] = rope(bf16(X Wqkv^T))[q heads]; K, V of row m -> pool
 * (layout of fp_k_attn_decode) at token (slot[m], pos[m]) of `layer`.
 * max_pos: bound on pos (size of the cos/sin table). */
int fp_k_qkv_rope(const void* Wqkv, int32_t K, const void* X, int32_t M, int32_t H, int32_t KVH, int32_t hd,
                  const int32_t* pos, int32_t max_pos, float rope_theta, void* pool, int32_t num_layers,
                  int32_t layer, const int32_t* block_table, int32_t bt_stride, const int32_t* slot, void* q_out,
                  void* stream);
/* LM head + token choice: token[M], logp[M]. mode: FP_TOKENS_*; target/sample_id/step: [M] (device). */
int fp_k_vocab(const void* X, int32_t M, int32_t K, const void* W, int32_t V, int32_t mode, float inv_temp,
               const int32_t* target, const int32_t* sample_id, const int32_t* step, uint64_t seed, int32_t* token,
               float* logp, void* stream);
/* The decode layer's GEMM chain in one persistent kernel (chain.cu): from the
 * attention output attn [M][H hd] of layer `layer`: x += O-proj (split-K
 * partials summed in order), h = rmsnorm(x) gain_mlp, act = SwiGLU(h Wgu),
 * x += down(act), h = rmsnorm(x) gain_next, and — when Wqkv != NULL — the next
 * layer's QKV with RoPE: q_out [M][H][hd], K / V appended to the pool at
 * (slot, pos) of layer + 1 (pool layout of fp_k_attn_decode). parts: 8 x M x d
 * fp32 scratch (holds the down partials on return); act [M][F]. */
int fp_k_decode_chain(const void* Wo, const void* Wgu, const void* Wd, const void* Wqkv, const void* attn, void* h,
                      void* act, float* parts, float* x, const float* gain_mlp, const float* gain_next, void* q_out,
                      void* pool, int32_t num_layers, int32_t layer, const int32_t* block_table, int32_t bt_stride,
                      const int32_t* slot, const int32_t* pos, int32_t max_pos, float rope_theta, int32_t M,
                      int32_t d, int32_t H, int32_t KVH, int32_t hd, int32_t F, void* stream);
/* Filtered sampling (top-k / top-p) through the engine's kernels:
 * gemm_vocab_logits -> topk_sample -> vocab_finalize. z_out (optional, [M][V]
 * fp32) receives the temperature-scaled logits the filter saw. */
int fp_k_vocab_filtered(const void* X, int32_t M, int32_t K, const void* W, int32_t V, float inv_temp, int32_t top_k,
                        float top_p, const int32_t* sample_id, const int32_t* step, uint64_t seed, int32_t* token,
                        float* logp, float* z_out, void* stream);
/* Decode step head: x[m] = E[tokens[idx[m]]] (fp32) and y = RMSNorm(x) * gain in one launch
 * (idx may be NULL: row m gathers tokens[m]); the bits of an embedding gather then fp_k_add_norm with nsplit 0. */
int fp_k_embed_norm(const int32_t* tokens, const int32_t* idx, int32_t M, const void* E, int32_t d, float* x,
                    const float* gain, void* y, void* stream);
int fp_k_add_norm(float* x, const float* parts, int32_t nsplit, const float* gain, void* y, int32_t M, int32_t d,
                  void* stream);
/* y = bf16(RMSNorm(x) * gain), warp-per-row kernel of the packed (prefill / scoring) forward. */
int fp_k_rms_norm_rows(const float* x, const float* gain, void* y, int32_t M, int32_t d, void* stream);
/* Paged decode attention. pool: [num_pages][L][KVH][2][64][hd] bf16; block_table [slots][bt_stride].
 * num_pages > 0 selects the tensor-core TMA kernel (hd 64 / 128); 0 the CUDA-core kernel. */
int fp_k_attn_decode(const void* q, int32_t B, int32_t H, int32_t KVH, int32_t hd, const void* pool,
                     int32_t num_pages, int32_t num_layers, int32_t layer, const int32_t* block_table,
                     int32_t bt_stride, const int32_t* slot, const int32_t* ctx, int32_t max_ctx, void* out,
                     void* stream);
/* The same with caller-owned buffers and no host synchronisation (graph-
 * capturable; tooling / roofline): items_dev from fp_k_attn_items (host ctx),
 * workspace of fp_k_attn_workspace_bytes, zero-filled before its first use
 * (the kernel leaves its counters zero). */
/* Debug: per-warp (begin ns, end ns, units) of the next decode-attention launches (NULL disables). */
void fp_k_attn_trace(void* buf);
int64_t fp_k_attn_workspace_bytes(int32_t B, int32_t H, int32_t KVH, int32_t hd, int32_t max_ctx);
int fp_k_attn_items(const int32_t* ctx_host, int32_t B, int32_t H, int32_t KVH, int32_t hd, int32_t max_ctx,
                    int32_t* items_host); /* items_host: 1 + B * ceil(max_ctx / 128) ints */
int fp_k_attn_decode_ws(const void* q, int32_t B, int32_t H, int32_t KVH, int32_t hd, const void* pool,
                        int32_t num_pages, int32_t num_layers, int32_t layer, const int32_t* block_table,
                        int32_t bt_stride, const int32_t* slot, const int32_t* ctx, const int32_t* items_dev,
                        int32_t max_ctx, void* workspace, void* out, void* stream);
/* Varlen causal attention; cu_host: n_seq+1 offsets (host), cu_dev the same on device.
 * hd 64 / 128: tcgen05 kernel; other head sizes: mma.sync kernel. */
int fp_k_attn_varlen(const void* q, const void* k, const void* v, int32_t H, int32_t KVH, int32_t hd,
                     const int32_t* cu_host, const int32_t* cu_dev, int32_t n_seq, void* out, void* stream);
/* Packed-forward kernel policy of the calling thread: 1 (default) persistent GEMM / attention
 * kernels from 1024 rows, 0 one-tile-per-CTA kernels (what scoring uses while its GPU decodes). */
int fp_k_set_packed_persistent(int on);
/* Packed GEMMs on SM pairs (tcgen05 cta_group::2, 256 x 256 tiles) for the calling thread:
 * -1 (default) when the tiles spread evenly, 0 never, 1 always. Same bits either way. */
int fp_k_set_pair_gemm(int mode);
/* Decode-attention work table (fp_k_attn_items) for the calling thread: 0 (default) whole 512-token
 * splits, 1 cut into 128-token sub-chunks, -1 cut only for small wide-kernel batches. Same bits. */
int fp_k_set_attn_cut(int mode);
/* Debug: record CTA 0's event times of subsequent tcgen05 varlen launches into buf (8 x 64 u64, device). */
int fp_k_attn_prefill_trace(void* buf);
/* The mma.sync kernel for any supported head size (cross-check of the tcgen05 kernel). */
int fp_k_attn_varlen_mma(const void* q, const void* k, const void* v, int32_t H, int32_t KVH, int32_t hd,
                         const int32_t* cu_host, const int32_t* cu_dev, int32_t n_seq, void* out, void* stream);
int fp_k_postprocess(int32_t n, const int32_t* off, const float* logp_actor, const float* logp_ref,
                     const float* values, const float* score, float beta, float gamma, float lam, float* kl,
                     float* reward, float* adv, float* ret, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FP_ENGINE_H_ */
