// fuseplan-b200 — GPU execution of the gen+inf stage (extension of genfuse.hpp).
//
// execute() runs the experience-collection stage for real on B200s: the
// actor's batched decode (paged KV, retire-on-finish, KV-gated admission with
// the reference's reservation rule, genfuse.cpp:226-236), sample-level
// streaming of finished samples into Reference/Critic/Reward scoring, per-token
// post-processing (KL, reward, GAE, returns), and — in the fused schedule on
// G > 1 instances — the one-shot long-tail migration at the trigger.
//
// Decisions (sample -> instance assignment, trigger, m, destinations,
// migrated set, mechanism, in-flight placement) are taken on the decision
// clock (simulate_fused / fused_trigger), so they are bit-exact with the
// reference; the engine then executes them and measures wall time separately.
// One process per GPU: rank r executes instance r of cfg.num_instances.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "fuseplan/genfuse.hpp"

namespace fuseplan {

/// Transformer shape of one engine model (Llama-style: RMSNorm, RoPE, GQA, SwiGLU).
struct EngineModelDims {
  int num_layers = 0, hidden = 0, num_heads = 0, num_kv_heads = 0, head_dim = 0, ffn = 0, vocab = 0;
};

struct EngineSetup {
  EngineModelDims actor, ref, critic, reward;
  std::uint64_t weight_seed = 1234;
  int max_prompt = 128;
  int max_new = 1024;
  int max_samples = 512;
  int max_live = 512;
  std::int64_t kv_pool_bytes = 0;
  int max_prefill_tokens = 16384;
  int max_infer_tokens = 16384;
  float rope_theta = 10000.f;
  int device = 0;
};

enum class TokenMode : int { kForced = 0, kGreedy = 1, kSample = 2 };
enum class Schedule : int { kStageBarrier = 0, kFused = 1 };

struct EngineOptions {
  TokenMode token_mode = TokenMode::kForced;
  Schedule schedule = Schedule::kFused;
  float temperature = 1.0f;
  std::uint64_t token_seed = 7;    // synthetic prompts / forced responses
  std::uint64_t sample_seed = 11;  // Philox streams of the sampler
  float kl_beta = 0.05f, gamma = 1.0f, lam = 0.95f;
  int claim_tokens = 8192;         // scoring batch granularity (tokens)
  int claim_max_live = 0;          // > 0: a generating rank claims scoring work only while its decode batch <= this
  int run_ahead = 4;               // decode steps the host may enqueue ahead of the GPU
  bool resident = false;           // prompts already on the device (same ids as last call), experience left there
  bool probe_attention = false;    // time every decode-attention launch (bench roofline)
  // > 0: hand the experience off as `handoff_dp` length-balanced data-parallel
  // mini-batches (balance_minibatch over prompt + response lengths): rank r
  // packs groups [r dp / world, (r + 1) dp / world) contiguously on its GPU,
  // pulling samples scored on other GPUs over NVLink. dp % world == 0.
  int handoff_dp = 0;
  // Free-run generation (north_star: "retires each sample as it emits EOS"):
  // eos_id >= 0 retires a sample at the first emitted eos_id (kept as its last
  // response token) or at max_new; target_output_len is then unused, KV
  // reservations use prompt + max_new, and the trigger is online. Greedy or
  // sample token modes only. The host learns the emitted ids eos_lag steps
  // late (a retired row decodes at most eos_lag extra, discarded, steps).
  int eos_id = -1;
  int eos_lag = 1;
  // Trigger of the fused schedule on G > 1 instances. false: the decision
  // clock's (bit-exact with simulate_fused; teacher-forced lengths); true:
  // online — the first rank that sees fewer than r_t unfinished samples in the
  // whole batch raises the trigger, every rank pauses at its next step
  // boundary, publishes its live state, and all ranks plan with the
  // reference's plan_migration on that state (genfuse.cpp:416-467) and place
  // the migrants with apply_migration's rules (genfuse.cpp:136-208).
  bool online_trigger = false;
  // Sampling filters (token_mode kSample): top_k > 0 keeps the logits >= the
  // k-th largest (k <= 1024); top_p < 1 keeps the shortest prefix of those
  // (sorted by probability; the top 1024 when top_k == 0) whose mass reaches
  // top_p of theirs. 0 / 1: off. The reported log-prob is the token's under
  // the full temperature softmax.
  int top_k = 0;
  float top_p = 1.0f;
};

/// Multi-process coordination (G > 1): every rank passes the same shm name.
struct CommSetup {
  int rank = 0;
  int world = 1;
  std::string shm_name;  // empty when world == 1
};

struct ExperienceBatch {
  std::vector<std::int64_t> resp_off;  // n + 1 response offsets
  std::vector<int> tokens;             // response token ids
  std::vector<float> logp_actor, logp_ref, values, kl, reward, adv, ret;
  std::vector<float> score;            // per sample
};

struct ExecStats {
  double wall_seconds = 0.0;        // whole stage on this rank (host clock, start barrier -> end)
  double gen_seconds = 0.0;         // this rank's last decode step end (GPU clock from start)
  double trigger_seconds = -1.0;    // trigger reached (GPU clock), -1 if none
  double migrate_seconds = 0.0;     // migration exchange (host clock)
  double ipc_seconds = 0.0;         // opening peer mappings (host clock; cached after the first call)
  double infer_busy_seconds = 0.0;  // GPU time of this rank's scoring batches
  std::int64_t decode_steps = 0, decode_rows = 0, decode_ctx_tokens = 0;
  std::int64_t prefill_tokens = 0, infer_tokens = 0, infer_samples = 0;
  std::int64_t migrated_in = 0, migrated_bytes = 0;
  double decode_gpu_seconds = 0.0;  // sum of decode-step GPU durations
  std::int64_t gpu_launches = 0;    // kernels this rank launched
  double attn_probe_ms = 0.0, attn_probe_bytes = 0.0;  // probe_attention totals
  std::int64_t attn_probe_launches = 0;
  std::int64_t eos_retired = 0;     // free-run: samples retired on an emitted EOS (this rank)
  std::int64_t overrun_rows = 0;    // free-run: row-steps decoded after an EOS the host had not seen yet
};

// Experience hand-off (EngineOptions::handoff_dp > 0).
struct Handoff {
  int dp = 0;
  std::vector<int> order;                // n sample ids, group-major (balance_minibatch)
  std::vector<int> group_off;            // dp + 1: group g = order[group_off[g] .. group_off[g + 1])
  std::vector<std::int64_t> packed_off;  // n + 1: response-token offsets in `order`
  int group_begin = 0, group_end = 0;    // this rank's groups
  // This rank's device buffers (engine-owned, valid until the next execute):
  // response tokens [packed_off[group_off[group_begin]], packed_off[group_off[group_end]])
  // of tokens / logp_actor, logp_ref, values, kl, reward, adv, ret, and the
  // score of samples order[group_off[group_begin] ..], all in `order`.
  const int* tokens = nullptr;
  const float* arrays[7] = {};
  const float* score = nullptr;
  double seconds = 0.0;                   // GPU time of the pack
  std::int64_t bytes = 0, peer_bytes = 0;  // bytes packed; of which pulled from other GPUs
};

struct ExecResult {
  GenStageResult decision;          // decision-clock result of the same schedule (planned lengths)
  TriggerSnapshot trigger;          // plan executed (fused, G > 1): decision clock's, or the online one
  bool online = false;              // the trigger was taken online (EngineOptions::online_trigger / eos_id)
  // In-flight and queued samples this rank received at the migration:
  // (sample, source rank), in application order.
  std::vector<int> received_sample, received_from;
  std::vector<double> finish_wall;  // per sample: GPU-clock finish time (seconds), on its final instance
  std::vector<int> finish_instance;
  ExperienceBatch experience;       // complete on rank 0 (gathered), local part elsewhere
  ExecStats stats;
  std::vector<int> step_rows;       // per decode step: batch rows
  std::vector<float> step_ms;       // per decode step: GPU duration (ms)
  std::vector<std::int64_t> step_ctx;  // per decode step: visible context tokens summed over its rows
  Handoff handoff;
};

class GpuEngine;  // opaque

GpuEngine* create_engine(const EngineSetup& setup);
void destroy_engine(GpuEngine* e);

/// Synthetic prompts (hash of token_seed) of shape [n][max_prompt].
std::vector<int> synthetic_prompts(const GpuEngine* e, int n, std::uint64_t token_seed);

// Weight sync across the ranks of one box: model slot
// 0 actor, 1 ref, 2 critic, 3 reward; every rank calls it with the same src
// and comm (a fresh shm name). Returns this rank's seconds.
double broadcast_model(GpuEngine* e, int model, int src, const CommSetup& comm);
// Test / tooling helpers: regenerate a model's synthetic weights with another
// seed; an order-independent 64-bit checksum of its weight blob.
void reinit_model(GpuEngine* e, int model, std::uint64_t seed);
// Copy one row-major host tensor into the engine's layout (fp_engine.h FP_W_*).
void load_weights(GpuEngine* e, int model, int tensor, int layer, const void* host, std::int64_t n_elems);
std::uint64_t model_checksum(GpuEngine* e, int model);

ExecResult execute(GpuEngine* e, const std::vector<GenSample>& batch, const GenSimConfig& cfg, int r_t,
                   const EngineOptions& opts, const CommSetup& comm, const std::vector<int>* prompts = nullptr);

}  // namespace fuseplan
