// fuseplan-b200 — one generation/inference engine per B200 (internal C++ API).
//
// An Engine owns, on its device:
//   * the four models' weights (actor, reference, critic, reward), synthetic
//     and deterministic (hash of seed, model, layer, tensor, index);
//   * the paged KV pool of the actor: pages of 64 tokens x all layers, page
//     layout [layer][kv_head][K 64 x hd | V 64 x hd] (bf16), a host free list
//     and a device block table [slot][page];
//   * per-sample histories (response token ids and actor log-probs, indexed by
//     global sample id) and the synthetic prompts;
//   * a decode workspace (live batch rows) and a packed workspace (prefill /
//     scoring rows), and three streams: decode, infer, copy.
// Work is enqueued asynchronously; the executor (executor.cpp) drives it.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <map>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "ops.h"

namespace fpe {

using bf16 = __nv_bfloat16;

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void check(cudaError_t e, const char* what);
#define FP_CUDA(x) ::fpe::check((x), #x)

enum ModelSlot : int { kActor = 0, kRef = 1, kCritic = 2, kReward = 3 };

struct Dims {
  int L = 0, d = 0, H = 0, KVH = 0, hd = 0, F = 0, V = 0;
  int qkv_width() const { return (H + 2 * KVH) * hd; }
  size_t kv_bytes_per_token() const { return static_cast<size_t>(2) * L * KVH * hd * 2; }  // physical, bf16
};

struct LayerW {
  bf16 *wqkv = nullptr, *wo = nullptr, *wgu = nullptr, *wd = nullptr;
  float *ln1 = nullptr, *ln2 = nullptr;
};

struct ModelW {
  Dims dims;
  int id = 0;
  bool lm_head = true;  // actor/ref: LM head [V, d]; critic/reward: value head [d]
  bf16* embed = nullptr;
  std::vector<LayerW> layers;
  float* lnf = nullptr;
  bf16* head = nullptr;
  bf16* vhead = nullptr;
  void* blob = nullptr;
  size_t bytes = 0;
  size_t param_count = 0;
};

struct EngineConfig {
  Dims model[4];
  uint64_t weight_seed = 1234;
  int max_prompt = 128;
  int max_new = 1024;
  int max_samples = 512;    // global batch n (history buffers are indexed by global id)
  int max_live = 512;       // decode slots
  int64_t kv_pool_bytes = 0;  // 0: enough for max_live samples of max_prompt + max_new
  int max_prefill_tokens = 16384;
  int max_infer_tokens = 16384;
  float rope_theta = 10000.f;
  int device = 0;
};

constexpr int kPageTokens = 64;

struct PinnedRing;  // host staging for async uploads

class Engine {
 public:
  explicit Engine(const EngineConfig& cfg);
  ~Engine();
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  const EngineConfig& config() const { return cfg_; }
  const ModelW& model(int m) const { return models_[m]; }
  void reinit_model(int m, uint64_t seed);     // synthetic weights from another seed (same layout)
  // Copy one row-major host tensor (fp_engine.h FP_W_*) into the model's blob,
  // repacking the gate / up rows into the 64-row interleave. Synchronous.
  void load_tensor(int m, int tensor, int layer, const void* host, int64_t n_elems);
  uint64_t model_checksum(int m);             // sum of the blob's 64-bit words (synchronises)
  cudaStream_t decode_stream() const { return s_decode_; }
  // The scoring stream: low priority, so scoring CTAs fill the SMs decode leaves idle.
  cudaStream_t infer_stream() const { return s_infer_; }
  cudaStream_t copy_stream() const { return s_copy_; }

  // ---- batch data (global sample ids) -------------------------------------------
  // prompts [n][max_prompt] (host), uploaded on the decode stream.
  void load_prompts(const int* prompts, int n, uint64_t tag = 0);
  uint64_t prompts_tag() const { return prompts_tag_; }
  int* d_prompts() const { return d_prompts_; }
  int* d_hist_tok() const { return d_hist_tok_; }
  float* d_hist_logp() const { return d_hist_logp_; }

  // ---- KV pages and slots -----------------------------------------------------------
  int pages_for(int tokens) const { return (tokens + kPageTokens - 1) / kPageTokens; }
  int free_pages() const { return static_cast<int>(free_pages_.size()); }
  int free_slots() const { return static_cast<int>(free_slots_.size()); }
  // Reserve a slot and `tokens` worth of pages; returns the slot.
  int reserve(int tokens);
  void release(int slot);
  const std::vector<int>& pages_of(int slot) const { return slot_pages_[slot]; }
  uint8_t* pool_base() const { return pool_; }
  size_t page_bytes() const { return page_bytes_; }
  int num_pages() const { return num_pages_; }

  // ---- generation (decode stream) ---------------------------------------------------
  struct PrefillItem {
    int sid, slot, ctx_tokens;  // positions [0, ctx_tokens) are written to the pool
    const int* tokens;          // host: ctx_tokens ids
    int next_token;             // first decode input (position ctx_tokens)
  };
  void prefill(const std::vector<PrefillItem>& items);

  struct DecodeRow {
    int sid, slot, pos, step, target;  // pos: position of the input token; step: response index
  };
  // One decode step for `rows`: writes hist[sid][step] (token, logp) and the
  // next input token. mode 0 forced (target), 1 greedy, 2 sample.
  // top_k / top_p (mode 2): filtered sampling (EngineOptions::top_k / top_p).
  void decode(const std::vector<DecodeRow>& rows, int mode, float inv_temp, uint64_t sample_seed, int top_k = 0,
              float top_p = 1.f);
  void set_use_graphs(bool on) { use_graphs_ = on; }
  static int bucket_of(int B);

  // ---- scoring (infer stream) ------------------------------------------------------
  struct InferItem {
    int sid, P, R;
    const int* hist_tok;     // device pointer (local or peer) of the sample's history row
    const float* hist_logp;
  };
  // Scores items in chunks of <= max_infer_tokens rows (three frozen models),
  // post-processes, and scatters the experience into the device arrays below
  // at each sample's global response offset (set_layout).
  // yield: this GPU is still decoding — one stream, one-tile-per-CTA kernels
  // (the decode step's CTAs get SMs between scoring tiles).
  void infer(const std::vector<InferItem>& items, float beta, float gamma, float lam, bool yield = false);

  // Global response layout: resp_off[n+1]; (re)allocates the experience arrays.
  void set_layout(const std::vector<int64_t>& resp_off);
  struct Experience {
    int* tokens = nullptr;
    float *logp_actor = nullptr, *logp_ref = nullptr, *values = nullptr, *kl = nullptr, *reward = nullptr,
          *adv = nullptr, *ret = nullptr, *score = nullptr;
  };
  const Experience& experience() const { return exp_; }
  void* exp_blob() const { return exp_blob_; }  // one cudaMalloc holding the arrays above (IPC-exportable)
  // Hand-off destination: `tokens` response entries of the 8 arrays + `n` scores
  // (reallocated when too small; same member layout as Experience).
  const Experience& handoff_buffers(int64_t tokens, int n);
  const std::vector<int64_t>& resp_off() const { return resp_off_; }

  // Async host -> device copy on `st` through a pinned staging ring (the host
  // buffer may be reused as soon as this returns).
  void upload(void* d_dst, const void* h_src, size_t bytes, cudaStream_t st);

  // Block-table row upload for a slot.
  void upload_block_table(int slot, cudaStream_t st);
  int* d_cur_tok() const { return d_cur_tok_; }
  // Device scratch for small per-call tables (chunk lists, index quads) on the decode stream.
  void* decode_scratch(size_t bytes);

  void synchronize();

  // Peer mapping of another process's allocation (CUDA IPC). Mappings are cached
  // for the engine's lifetime: the peers' KV pools / histories are persistent,
  // and opening a multi-GB pool costs milliseconds per call.
  void* open_ipc(const cudaIpcMemHandle_t& h);

  // Kernel probe: when enabled, every decode-attention launch is bracketed by
  // CUDA events on the decode stream and its algorithmic bytes recorded
  // (K/V of the visible context + q), for the roofline of bench.py.
  void set_attn_probe(bool on) { probe_on_ = on; }
  struct ProbeTotals {
    double ms = 0.0;
    double bytes = 0.0;
    long long launches = 0;
  };
  ProbeTotals drain_attn_probe();  // synchronises the decode stream

 private:
  struct ProbeRec {
    cudaEvent_t a, b;
    double bytes;
  };
  bool probe_on_ = false;
  bool use_graphs_ = true;
  bool fuse_rope_ = true;  // prefill / scoring: RoPE + K/V writes in the QKV GEMM epilogue
  int decode_calls_ = 0;
  bool chain_ = true;     // decode: the GEMM chain of a layer as one persistent kernel (fpk::decode_chain)
  int chain_max_b_ = 0;   // ... for decode batches up to this many rows (off: measured no faster)
  int chain_ctas_ = 148;  // its grid: one CTA per SM
  int pad_slot_ = 0;
  struct GraphKey {
    int B, mode;
    float inv_temp;
    uint64_t seed;
    int top_k;
    float top_p;
    bool operator<(const GraphKey& o) const {
      if (B != o.B) return B < o.B;
      if (mode != o.mode) return mode < o.mode;
      if (inv_temp != o.inv_temp) return inv_temp < o.inv_temp;
      if (top_k != o.top_k) return top_k < o.top_k;
      if (top_p != o.top_p) return top_p < o.top_p;
      return seed < o.seed;
    }
  };
  struct StepGraph {
    cudaGraphExec_t exec;
    long long kernels;  // launches the graph replays (gpu_launches accounting)
  };
  std::map<GraphKey, StepGraph> graphs_;
  std::set<GraphKey> graph_seen_;
  struct DecodeWs;
  void decode_kernels(DecodeWs& dw, cudaStream_t st, int B, int max_ctx, int mode, float inv_temp,
                      uint64_t sample_seed, double ctx_sum, int attn_ctas, int top_k, float top_p);
  size_t build_rows(const DecodeRow* rows, int B, int Bb, std::vector<int>& h, int& max_ctx, double& ctx_sum);
  void run_graph(const GraphKey& key, const std::function<void()>& body);
  uint64_t prompts_tag_ = 0;
  CUtensorMap kv_map_{};
  bool has_kv_map_ = false;
  fpk::KvPoolView pool_view() const {
    fpk::KvPoolView pv{pool_, page_bytes_, layer_bytes_, kPageTokens, d_block_table_, max_pages_per_sample_};
    pv.kv_map = has_kv_map_ ? &kv_map_ : nullptr;
    return pv;
  }
  std::vector<ProbeRec> probes_;
  std::vector<cudaEvent_t> probe_pool_;
  cudaEvent_t probe_event();
  // Activations of one packed forward (per model when the scoring models run
  // concurrently).
  struct ActWs {
    float* x = nullptr;
    bf16 *h = nullptr, *qkv = nullptr, *q = nullptr, *k = nullptr, *v = nullptr, *attn = nullptr, *act = nullptr;
  };
  struct PackedWs {
    int cap = 0, cap_seq = 0;
    ActWs a[3];  // [0]: prefill / reference; [1], [2]: critic, reward (scoring only)
    int *tokens = nullptr, *pos = nullptr, *slot = nullptr, *cu = nullptr, *tiles = nullptr, *tiles128 = nullptr;
    // scoring
    int *sid = nullptr, *P = nullptr, *R = nullptr, *roff = nullptr, *targets = nullptr, *gather_resp = nullptr,
        *gather_last = nullptr;
    const int** hist_tok = nullptr;
    const float** hist_logp = nullptr;
    int64_t* off_out = nullptr;
    void* vocab_part = nullptr;
    float *tgt_z = nullptr, *logp_actor = nullptr, *logp_ref = nullptr, *values = nullptr, *score = nullptr,
          *kl = nullptr, *reward = nullptr, *adv = nullptr, *ret = nullptr;
  };
  struct DecodeWs {
    int cap = 0;
    float *x = nullptr, *parts = nullptr, *attn_work = nullptr;
    int* attn_cnt = nullptr;  // split-merge tickets of the decode attention (B x KVH, kept zero)
    int* chain_cnt = nullptr;  // grid-barrier counters of decode_chain, 8 per layer (kept zero)
    bf16 *h = nullptr, *qkv = nullptr, *q = nullptr, *attn = nullptr, *act = nullptr;
    int* rows = nullptr;  // 7 x cap: slot, pos, ctx, dst, target, sid, step
    void* vocab_part = nullptr;
    float* tgt_z = nullptr;
    float* logits = nullptr;  // filtered sampling: [cap][ldv] z (allocated on first use)
    int* pick = nullptr;      // filtered sampling: chosen token per row
  };
  int logits_ld() const { return (cfg_.model[kActor].V + 3) & ~3; }

  void init_model(int m);
  void fill_model(int m, uint64_t seed);
  void alloc_ws();
  // Both attention tile tables of one packed batch (64- and 128-query tiles);
  // forward_packed uses the one its model's head size needs. nt[0], nt[1]: counts.
  void upload_tiles(PackedWs& ws, const int* cu, int n_seq, int nt[2], cudaStream_t st);
  void forward_packed(const ModelW& w, PackedWs& ws, const ActWs& a, int M, int n_seq, const int nt[2],
                      bool use_pool, cudaStream_t st);

  EngineConfig cfg_;
  ModelW models_[4];
  cudaStream_t s_decode_ = nullptr, s_infer_ = nullptr, s_copy_ = nullptr;
  // The critic's and the reward model's forwards run beside the reference
  // model's (three independent packed forwards over the same batch): one
  // model's kernel ramp-up / drain overlaps another's mainloops.
  cudaStream_t s_score_[2] = {nullptr, nullptr};
  cudaEvent_t ev_fork_ = nullptr, ev_join_[2] = {nullptr, nullptr};
  // pool
  uint8_t* pool_ = nullptr;
  size_t page_bytes_ = 0, layer_bytes_ = 0;
  int num_pages_ = 0, max_pages_per_sample_ = 0;
  std::vector<int> free_pages_, free_slots_;
  std::vector<std::vector<int>> slot_pages_;
  std::vector<int> bt_host_;
  int* d_block_table_ = nullptr;
  int* d_cur_tok_ = nullptr;
  float2* rope_cs_ = nullptr;
  // batch
  int* d_prompts_ = nullptr;
  int* d_hist_tok_ = nullptr;
  float* d_hist_logp_ = nullptr;
  PackedWs pre_, inf_;
  Experience exp_;
  void* exp_blob_ = nullptr;
  void* handoff_blob_ = nullptr;
  size_t handoff_bytes_ = 0;
  Experience hand_;
  std::vector<int64_t> resp_off_;
  DecodeWs dec_;
  PinnedRing* ring_ = nullptr;
  void* scratch_ = nullptr;
  size_t scratch_bytes_ = 0;
  std::vector<void*> allocs_;
  std::map<std::string, void*> ipc_cache_;
  void* dalloc(size_t bytes);
};

}  // namespace fpe
