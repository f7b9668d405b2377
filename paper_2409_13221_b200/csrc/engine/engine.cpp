// fuseplan-b200 — Engine: weights, paged KV pool, prefill / decode / scoring.
#include "engine.hpp"

#include <cuda.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <functional>
#include <numeric>

#include "philox.cuh"

namespace fpe {

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string("CUDA error: ") + cudaGetErrorString(e) + " at " + what);
}

// ---------------------------------------------------------------------------
// pinned staging ring: fixed chunks, each guarded by an event

struct PinnedRing {
  static constexpr int kChunks = 64;
  static constexpr size_t kChunkBytes = 1 << 20;
  uint8_t* host = nullptr;
  cudaEvent_t ev[kChunks];
  bool used[kChunks] = {};
  int next = 0;
  PinnedRing() {
    FP_CUDA(cudaMallocHost(&host, kChunks * kChunkBytes));
    for (auto& e : ev) FP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  ~PinnedRing() {
    for (auto& e : ev) cudaEventDestroy(e);
    cudaFreeHost(host);
  }
};

void Engine::upload(void* d_dst, const void* h_src, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return;
  const uint8_t* src = static_cast<const uint8_t*>(h_src);
  uint8_t* dst = static_cast<uint8_t*>(d_dst);
  while (bytes > 0) {
    const size_t n = std::min(bytes, PinnedRing::kChunkBytes);
    const int c = ring_->next;
    ring_->next = (c + 1) % PinnedRing::kChunks;
    if (ring_->used[c]) FP_CUDA(cudaEventSynchronize(ring_->ev[c]));
    uint8_t* h = ring_->host + c * PinnedRing::kChunkBytes;
    std::memcpy(h, src, n);
    FP_CUDA(cudaMemcpyAsync(dst, h, n, cudaMemcpyHostToDevice, st));
    FP_CUDA(cudaEventRecord(ring_->ev[c], st));
    ring_->used[c] = true;
    src += n;
    dst += n;
    bytes -= n;
  }
}

void* Engine::dalloc(size_t bytes) {
  void* p = nullptr;
  bytes = (bytes + 255) & ~size_t(255);
  FP_CUDA(cudaMalloc(&p, bytes == 0 ? 256 : bytes));
  allocs_.push_back(p);
  return p;
}

// ---------------------------------------------------------------------------

Engine::Engine(const EngineConfig& cfg) : cfg_(cfg) {
  FP_CUDA(cudaSetDevice(cfg_.device));
  // Decode is the latency-critical stream (the long tail is the critical
  // path): give it the highest priority so scoring batches only fill idle SMs.
  int prio_lo = 0, prio_hi = 0;
  FP_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  FP_CUDA(cudaStreamCreateWithPriority(&s_decode_, cudaStreamNonBlocking, prio_hi));
  FP_CUDA(cudaStreamCreateWithPriority(&s_infer_, cudaStreamNonBlocking, prio_lo));
  for (int i = 0; i < 2; ++i) {
    FP_CUDA(cudaStreamCreateWithPriority(&s_score_[i], cudaStreamNonBlocking, prio_lo));
    FP_CUDA(cudaEventCreateWithFlags(&ev_join_[i], cudaEventDisableTiming));
  }
  FP_CUDA(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
  FP_CUDA(cudaStreamCreateWithFlags(&s_copy_, cudaStreamNonBlocking));
  ring_ = new PinnedRing();
  const Dims& a = cfg_.model[kActor];
  if (a.L <= 0 || a.d <= 0 || a.H <= 0 || a.KVH <= 0 || a.hd <= 0 || a.F <= 0 || a.V <= 0)
    throw std::invalid_argument("engine: actor dimensions must be positive");
  for (int m = 0; m < 4; ++m) {
    const Dims& d = cfg_.model[m];
    if (d.d % 64 || d.F % 64 || (d.H * d.hd) % 64)
      throw std::invalid_argument("engine: hidden, ffn and H*head_dim must be multiples of 64");
    if (d.H % d.KVH) throw std::invalid_argument("engine: num_heads must be a multiple of num_kv_heads");
    if (d.hd % 2) throw std::invalid_argument("engine: head_dim must be even");
  }
  for (int m = 0; m < 4; ++m) init_model(m);

  // KV pool
  layer_bytes_ = static_cast<size_t>(a.KVH) * 2 * kPageTokens * a.hd * 2;
  page_bytes_ = layer_bytes_ * a.L;
  max_pages_per_sample_ = pages_for(cfg_.max_prompt + cfg_.max_new);
  int64_t pool_bytes = cfg_.kv_pool_bytes;
  if (pool_bytes <= 0) pool_bytes = static_cast<int64_t>(cfg_.max_live) * max_pages_per_sample_ * page_bytes_;
  num_pages_ = static_cast<int>(pool_bytes / page_bytes_) + 1;  // +1: scratch page for padded rows
  pool_ = static_cast<uint8_t*>(dalloc(static_cast<size_t>(num_pages_) * page_bytes_));
  for (int p = num_pages_ - 1; p >= 1; --p) free_pages_.push_back(p);  // page 0 is the scratch page
  if (a.hd == 64 || a.hd == 128) {  // 2-D TMA view of the pool for tensor-core decode attention
    const long long rows = static_cast<long long>(num_pages_) * static_cast<long long>(page_bytes_ / (a.hd * 2));
    kv_map_ = fpk::make_kv_map(pool_, rows, a.hd);
    has_kv_map_ = true;
  }
  for (int s = cfg_.max_live - 1; s >= 0; --s) free_slots_.push_back(s);
  if (const char* g = std::getenv("FUSEPLAN_DECODE_GRAPHS")) use_graphs_ = std::atoi(g) != 0;  // A/B switch
  // decode_chain for decode batches of at most chain_max_b_ rows (FUSEPLAN_DECODE_CHAIN: that bound;
  // 0 = never) — bit-identical to the separate kernels, so the choice never changes a result
  if (const char* g = std::getenv("FUSEPLAN_DECODE_CHAIN")) chain_max_b_ = std::atoi(g);
  {
    int sms = 148;
    FP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cfg_.device));
    chain_ctas_ = sms;
  }
  if (const char* g = std::getenv("FUSEPLAN_FUSE_ROPE")) fuse_rope_ = std::atoi(g) != 0;
  pad_slot_ = cfg_.max_live;  // decode padding rows: block-table row of zeros -> scratch page 0
  slot_pages_.assign(cfg_.max_live + 1, {});
  bt_host_.assign(static_cast<size_t>(cfg_.max_live + 1) * max_pages_per_sample_, 0);
  d_block_table_ = static_cast<int*>(dalloc(bt_host_.size() * sizeof(int)));
  FP_CUDA(cudaMemsetAsync(d_block_table_, 0, bt_host_.size() * sizeof(int), s_decode_));
  d_cur_tok_ = static_cast<int*>(dalloc((cfg_.max_live + 1) * sizeof(int)));
  {  // RoPE (cos, sin) table of the actor for every position the decode step can see
    const int max_pos = cfg_.max_prompt + cfg_.max_new;
    const int hd = cfg_.model[kActor].hd;
    rope_cs_ = static_cast<float2*>(dalloc(static_cast<size_t>(max_pos) * (hd / 2) * sizeof(float2)));
    fpk::rope_table(rope_cs_, max_pos, hd, cfg_.rope_theta, s_decode_);
  }

  // one extra history row: the destination of decode padding rows
  const size_t hist = static_cast<size_t>(cfg_.max_samples + 1) * cfg_.max_new;
  d_prompts_ = static_cast<int*>(dalloc(static_cast<size_t>(cfg_.max_samples) * cfg_.max_prompt * sizeof(int)));
  d_hist_tok_ = static_cast<int*>(dalloc(hist * sizeof(int)));
  d_hist_logp_ = static_cast<float*>(dalloc(hist * sizeof(float)));
  FP_CUDA(cudaMemsetAsync(d_hist_tok_, 0, hist * sizeof(int), s_decode_));
  alloc_ws();
  FP_CUDA(cudaStreamSynchronize(s_decode_));
}

void* Engine::open_ipc(const cudaIpcMemHandle_t& h) {
  const std::string key(reinterpret_cast<const char*>(&h), sizeof(h));
  auto it = ipc_cache_.find(key);
  if (it != ipc_cache_.end()) return it->second;
  void* p = nullptr;
  FP_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  ipc_cache_.emplace(key, p);
  return p;
}

Engine::~Engine() {
  cudaSetDevice(cfg_.device);
  cudaDeviceSynchronize();
  for (auto& kv : ipc_cache_) cudaIpcCloseMemHandle(kv.second);
  for (void* p : allocs_) cudaFree(p);
  for (int m = 0; m < 4; ++m)
    if (models_[m].blob) cudaFree(models_[m].blob);
  if (exp_blob_) cudaFree(exp_blob_);
  if (handoff_blob_) cudaFree(handoff_blob_);
  if (scratch_) cudaFree(scratch_);
  for (auto& kv : graphs_) cudaGraphExecDestroy(kv.second.exec);
  for (auto& p : probes_) probe_pool_.insert(probe_pool_.end(), {p.a, p.b});
  for (cudaEvent_t e : probe_pool_) cudaEventDestroy(e);
  delete ring_;
  cudaStreamDestroy(s_decode_);
  cudaStreamDestroy(s_infer_);
  for (int i = 0; i < 2; ++i) {
    cudaStreamDestroy(s_score_[i]);
    cudaEventDestroy(ev_join_[i]);
  }
  cudaEventDestroy(ev_fork_);
  cudaStreamDestroy(s_copy_);
}

void Engine::synchronize() {
  FP_CUDA(cudaStreamSynchronize(s_decode_));
  FP_CUDA(cudaStreamSynchronize(s_infer_));
  for (cudaStream_t s : s_score_) FP_CUDA(cudaStreamSynchronize(s));
  FP_CUDA(cudaStreamSynchronize(s_copy_));
}

void Engine::init_model(int m) {
  ModelW& w = models_[m];
  const Dims& D = cfg_.model[m];
  w.dims = D;
  w.id = m;
  w.lm_head = (m == kActor || m == kRef);
  const size_t d = D.d, F = D.F, V = D.V, qw = D.qkv_width(), ao = static_cast<size_t>(D.H) * D.hd;
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  size_t bytes = al(V * d * 2);  // embedding
  const size_t per_layer = al(qw * d * 2) + al(d * ao * 2) + al(2 * F * d * 2) + al(d * F * 2) + 2 * al(d * 4);
  bytes += D.L * per_layer + al(d * 4) + (w.lm_head ? al(V * d * 2) : al(d * 2));
  FP_CUDA(cudaMalloc(&w.blob, bytes));
  FP_CUDA(cudaMemsetAsync(w.blob, 0, bytes, s_decode_));  // padding included: checksums see defined bytes
  w.bytes = bytes;
  fill_model(m, cfg_.weight_seed);
}

void Engine::reinit_model(int m, uint64_t seed) {
  fill_model(m, seed);
  FP_CUDA(cudaStreamSynchronize(s_decode_));
}

void Engine::load_tensor(int m, int tensor, int layer, const void* host, int64_t n_elems) {
  if (m < 0 || m > 3) throw std::invalid_argument("load_weights: model index out of range");
  ModelW& w = models_[m];
  const Dims& D = w.dims;
  const bool per_layer = tensor >= 1 && tensor <= 7;
  if (per_layer && (layer < 0 || layer >= D.L)) throw std::invalid_argument("load_weights: layer out of range");
  if (!per_layer && layer != 0) throw std::invalid_argument("load_weights: per-model tensors take layer 0");
  if (!host) throw std::invalid_argument("load_weights: null host tensor");
  const size_t d = D.d, F = D.F, V = D.V, qw = D.qkv_width(), ao = static_cast<size_t>(D.H) * D.hd;
  void* dst = nullptr;
  size_t elems = 0, esize = 2;
  switch (tensor) {
    case 0: dst = w.embed, elems = V * d; break;
    case 1: dst = w.layers[layer].wqkv, elems = qw * d; break;
    case 2: dst = w.layers[layer].wo, elems = d * ao; break;
    case 3:
    case 4: dst = w.layers[layer].wgu, elems = F * d; break;
    case 5: dst = w.layers[layer].wd, elems = d * F; break;
    case 6: dst = w.layers[layer].ln1, elems = d, esize = 4; break;
    case 7: dst = w.layers[layer].ln2, elems = d, esize = 4; break;
    case 8: dst = w.lnf, elems = d, esize = 4; break;
    case 9:
      if (!w.lm_head) throw std::invalid_argument("load_weights: critic / reward models have a value head, not an LM head");
      dst = w.head, elems = V * d;
      break;
    case 10:
      if (w.lm_head) throw std::invalid_argument("load_weights: actor / reference models have an LM head, not a value head");
      dst = w.vhead, elems = d;
      break;
    default: throw std::invalid_argument("load_weights: unknown tensor kind");
  }
  if (n_elems < 0 || static_cast<size_t>(n_elems) != elems)
    throw std::invalid_argument("load_weights: element count does not match the tensor's shape");
  FP_CUDA(cudaStreamSynchronize(s_decode_));
  if (tensor == 3 || tensor == 4) {
    // [F][d] gate (or up) rows -> rows (f / 64) * 128 + (up ? 64 : 0) + f % 64 of W_gu
    const size_t group = 64 * d * 2;
    uint8_t* base = static_cast<uint8_t*>(dst) + (tensor == 4 ? group : 0);
    FP_CUDA(cudaMemcpy2D(base, 2 * group, host, group, group, F / 64, cudaMemcpyHostToDevice));
  } else {
    FP_CUDA(cudaMemcpy(dst, host, elems * esize, cudaMemcpyHostToDevice));
  }
}

uint64_t Engine::model_checksum(int m) {
  unsigned long long* d = static_cast<unsigned long long*>(decode_scratch(sizeof(unsigned long long)));
  FP_CUDA(cudaMemsetAsync(d, 0, sizeof(unsigned long long), s_decode_));
  fpk::checksum64(models_[m].blob, models_[m].bytes, d, s_decode_);
  unsigned long long h = 0;
  FP_CUDA(cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, s_decode_));
  FP_CUDA(cudaStreamSynchronize(s_decode_));
  return h;
}

void Engine::fill_model(int m, uint64_t wseed) {
  ModelW& w = models_[m];
  const Dims& D = cfg_.model[m];
  const size_t d = D.d, F = D.F, V = D.V, qw = D.qkv_width(), ao = static_cast<size_t>(D.H) * D.hd;
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  uint8_t* p = static_cast<uint8_t*>(w.blob);
  auto take = [&](size_t b) {
    uint8_t* r = p;
    p += al(b);
    return r;
  };
  const uint64_t seed = wseed;
  cudaStream_t st = s_decode_;
  w.embed = reinterpret_cast<bf16*>(take(V * d * 2));
  fpk::init_bf16(w.embed, V * d, seed, fpk::weight_tag(m, 0, fpk::kTagEmbed), 1.0f, st);
  w.layers.resize(D.L);
  for (int l = 0; l < D.L; ++l) {
    LayerW& L = w.layers[l];
    L.wqkv = reinterpret_cast<bf16*>(take(qw * d * 2));
    L.wo = reinterpret_cast<bf16*>(take(d * ao * 2));
    L.wgu = reinterpret_cast<bf16*>(take(2 * F * d * 2));
    L.wd = reinterpret_cast<bf16*>(take(d * F * 2));
    L.ln1 = reinterpret_cast<float*>(take(d * 4));
    L.ln2 = reinterpret_cast<float*>(take(d * 4));
    fpk::init_bf16(L.wqkv, qw * d, seed, fpk::weight_tag(m, l, fpk::kTagWqkv), std::sqrt(3.0f / d), st);
    fpk::init_bf16(L.wo, d * ao, seed, fpk::weight_tag(m, l, fpk::kTagWo), std::sqrt(3.0f / ao), st);
    fpk::init_bf16_gu(L.wgu, D.F, D.d, seed, fpk::weight_tag(m, l, fpk::kTagWgu), std::sqrt(3.0f / d), st);
    fpk::init_bf16(L.wd, d * F, seed, fpk::weight_tag(m, l, fpk::kTagWd), std::sqrt(3.0f / F), st);
    fpk::init_gain(L.ln1, d, seed, fpk::weight_tag(m, l, fpk::kTagAttnNorm), st);
    fpk::init_gain(L.ln2, d, seed, fpk::weight_tag(m, l, fpk::kTagMlpNorm), st);
  }
  w.lnf = reinterpret_cast<float*>(take(d * 4));
  fpk::init_gain(w.lnf, d, seed, fpk::weight_tag(m, 0, fpk::kTagFinalNorm), st);
  if (w.lm_head) {
    w.head = reinterpret_cast<bf16*>(take(V * d * 2));
    fpk::init_bf16(w.head, V * d, seed, fpk::weight_tag(m, 0, fpk::kTagHead), std::sqrt(3.0f / d), st);
  } else {
    w.vhead = reinterpret_cast<bf16*>(take(d * 2));
    fpk::init_bf16(w.vhead, d, seed, fpk::weight_tag(m, 0, fpk::kTagValueHead), std::sqrt(3.0f / d), st);
  }
  w.param_count = V * d + D.L * (qw * d + d * ao + 2 * F * d + d * F) + (w.lm_head ? V * d : d);
  FP_CUDA(cudaGetLastError());
}

void Engine::alloc_ws() {
  int maxd = 0, maxq = 0, maxF = 0, maxao = 0, maxV = 0, maxkv = 0;
  for (int m = 0; m < 4; ++m) {
    const Dims& D = cfg_.model[m];
    maxd = std::max(maxd, D.d);
    maxq = std::max(maxq, D.qkv_width());
    maxF = std::max(maxF, D.F);
    maxao = std::max(maxao, D.H * D.hd);
    maxkv = std::max(maxkv, D.KVH * D.hd);
    if (m == kActor || m == kRef) maxV = std::max(maxV, D.V);
  }
  const int vt = fpk::vocab_tiles(maxV);
  auto packed = [&](PackedWs& w, int cap, bool scoring) {
    w.cap = cap;
    w.cap_seq = std::min(cap, cfg_.max_samples) + 1;
    for (int i = 0; i < (scoring ? 3 : 1); ++i) {
      ActWs& a = w.a[i];
      a.x = static_cast<float*>(dalloc(static_cast<size_t>(cap) * maxd * 4));
      a.h = static_cast<bf16*>(dalloc(static_cast<size_t>(cap) * maxd * 2));
      a.qkv = static_cast<bf16*>(dalloc(static_cast<size_t>(cap) * maxq * 2));
      a.q = static_cast<bf16*>(dalloc(static_cast<size_t>(cap) * maxao * 2));
      a.k = static_cast<bf16*>(dalloc(static_cast<size_t>(cap) * maxkv * 2));
      a.v = static_cast<bf16*>(dalloc(static_cast<size_t>(cap) * maxkv * 2));
      a.attn = static_cast<bf16*>(dalloc(static_cast<size_t>(cap) * maxao * 2));
      a.act = static_cast<bf16*>(dalloc(static_cast<size_t>(cap) * maxF * 2));
    }
    w.tokens = static_cast<int*>(dalloc(cap * 4));
    w.pos = static_cast<int*>(dalloc(cap * 4));
    w.slot = static_cast<int*>(dalloc(cap * 4));
    w.cu = static_cast<int*>(dalloc(w.cap_seq * 4));
    w.tiles = static_cast<int*>(dalloc(static_cast<size_t>(2) * (cap / 64 + w.cap_seq) * 4));
    w.tiles128 = static_cast<int*>(dalloc(static_cast<size_t>(2) * (cap / 128 + w.cap_seq) * 4));
    if (!scoring) return;
    const int cs = w.cap_seq;
    w.sid = static_cast<int*>(dalloc(cs * 4));
    w.P = static_cast<int*>(dalloc(cs * 4));
    w.R = static_cast<int*>(dalloc(cs * 4));
    w.roff = static_cast<int*>(dalloc(cs * 4));
    w.off_out = static_cast<int64_t*>(dalloc(cs * 8));
    w.hist_tok = static_cast<const int**>(dalloc(cs * 8));
    w.hist_logp = static_cast<const float**>(dalloc(cs * 8));
    w.targets = static_cast<int*>(dalloc(cap * 4));
    w.gather_resp = static_cast<int*>(dalloc(cap * 4));
    w.gather_last = static_cast<int*>(dalloc(cs * 4));
    w.vocab_part = dalloc(static_cast<size_t>(cap) * vt * 24);
    w.tgt_z = static_cast<float*>(dalloc(cap * 4));
    for (float** f : {&w.logp_actor, &w.logp_ref, &w.values, &w.kl, &w.reward, &w.adv, &w.ret})
      *f = static_cast<float*>(dalloc(cap * 4));
    w.score = static_cast<float*>(dalloc(cs * 4));
  };
  const int prefill_cap = std::max(cfg_.max_prefill_tokens, cfg_.max_prompt + cfg_.max_new);
  const int infer_cap = std::max(cfg_.max_infer_tokens, cfg_.max_prompt + cfg_.max_new);
  packed(pre_, prefill_cap, false);
  packed(inf_, infer_cap, true);

  const int Bcap = bucket_of(cfg_.max_live);
  auto decode_ws = [&](DecodeWs& dw, int B) {
    dw.cap = B;
    dw.x = static_cast<float*>(dalloc(static_cast<size_t>(B) * maxd * 4));
    dw.parts = static_cast<float*>(dalloc(static_cast<size_t>(16) * B * maxd * 4));
    dw.h = static_cast<bf16*>(dalloc(static_cast<size_t>(B) * maxd * 2));
    dw.qkv = static_cast<bf16*>(dalloc(static_cast<size_t>(B) * maxq * 2));
    dw.q = static_cast<bf16*>(dalloc(static_cast<size_t>(B) * maxao * 2));
    dw.attn = static_cast<bf16*>(dalloc(static_cast<size_t>(B) * maxao * 2));
    dw.act = static_cast<bf16*>(dalloc(static_cast<size_t>(B) * maxF * 2));
    const int items_cap = (cfg_.max_prompt + cfg_.max_new + 127) / 128;  // work items per row (attn_decode_items)
    dw.rows = static_cast<int*>(dalloc((static_cast<size_t>(7 + items_cap) * B + 1) * 4));
    dw.vocab_part = dalloc(static_cast<size_t>(B) * vt * 24);
    dw.tgt_z = static_cast<float*>(dalloc(B * 4));
    const Dims& a = cfg_.model[kActor];
    dw.attn_work = static_cast<float*>(
        dalloc(fpk::attn_decode_workspace(B, a.H, a.hd, cfg_.max_prompt + cfg_.max_new) * sizeof(float)));
    const size_t cnt =
        static_cast<size_t>(fpk::attn_decode_counters(B, a.KVH, cfg_.max_prompt + cfg_.max_new)) * sizeof(int);
    dw.attn_cnt = static_cast<int*>(dalloc(cnt));
    FP_CUDA(cudaMemsetAsync(dw.attn_cnt, 0, cnt, s_decode_));
    const size_t ccnt = static_cast<size_t>(cfg_.model[kActor].L) * 8 * sizeof(int);
    dw.chain_cnt = static_cast<int*>(dalloc(ccnt));
    FP_CUDA(cudaMemsetAsync(dw.chain_cnt, 0, ccnt, s_decode_));
  };
  decode_ws(dec_, Bcap);
}

// ---------------------------------------------------------------------------

void Engine::load_prompts(const int* prompts, int n, uint64_t tag) {
  if (n > cfg_.max_samples) throw std::invalid_argument("engine: batch larger than max_samples");
  upload(d_prompts_, prompts, static_cast<size_t>(n) * cfg_.max_prompt * sizeof(int), s_decode_);
  prompts_tag_ = tag;
}

void Engine::set_layout(const std::vector<int64_t>& resp_off) {
  if (exp_blob_ && resp_off == resp_off_) return;  // same layout: reuse (results are overwritten)
  resp_off_ = resp_off;
  const size_t n = resp_off.empty() ? 0 : resp_off.size() - 1;
  const size_t total = resp_off.empty() ? 0 : static_cast<size_t>(resp_off.back());
  if (exp_blob_) {
    FP_CUDA(cudaDeviceSynchronize());
    cudaFree(exp_blob_);
    exp_blob_ = nullptr;
  }
  const size_t al = (total * 4 + 255) & ~size_t(255);
  const size_t bytes = 8 * al + ((n * 4 + 255) & ~size_t(255));
  FP_CUDA(cudaMalloc(&exp_blob_, bytes));
  FP_CUDA(cudaMemsetAsync(exp_blob_, 0, bytes, s_decode_));
  uint8_t* p = static_cast<uint8_t*>(exp_blob_);
  exp_.tokens = reinterpret_cast<int*>(p);
  float** fs[7] = {&exp_.logp_actor, &exp_.logp_ref, &exp_.values, &exp_.kl, &exp_.reward, &exp_.adv, &exp_.ret};
  for (int i = 0; i < 7; ++i) *fs[i] = reinterpret_cast<float*>(p + (i + 1) * al);
  exp_.score = reinterpret_cast<float*>(p + 8 * al);
}

const Engine::Experience& Engine::handoff_buffers(int64_t tokens, int n) {
  const size_t al = (static_cast<size_t>(std::max<int64_t>(tokens, 1)) * 4 + 255) & ~size_t(255);
  const size_t bytes = 8 * al + ((static_cast<size_t>(std::max(n, 1)) * 4 + 255) & ~size_t(255));
  if (bytes > handoff_bytes_) {
    if (handoff_blob_) {
      FP_CUDA(cudaDeviceSynchronize());
      cudaFree(handoff_blob_);
    }
    FP_CUDA(cudaMalloc(&handoff_blob_, bytes));
    handoff_bytes_ = bytes;
  }
  uint8_t* p = static_cast<uint8_t*>(handoff_blob_);
  hand_.tokens = reinterpret_cast<int*>(p);
  float** fs[7] = {&hand_.logp_actor, &hand_.logp_ref, &hand_.values, &hand_.kl, &hand_.reward, &hand_.adv,
                   &hand_.ret};
  for (int i = 0; i < 7; ++i) *fs[i] = reinterpret_cast<float*>(p + (i + 1) * al);
  hand_.score = reinterpret_cast<float*>(p + 8 * al);
  return hand_;
}

int Engine::reserve(int tokens) {
  const int need = pages_for(tokens);
  if (need > max_pages_per_sample_) throw std::invalid_argument("engine: sample longer than max_prompt + max_new");
  if (free_slots_.empty() || static_cast<int>(free_pages_.size()) < need)
    throw std::runtime_error("engine: KV pool or decode slots exhausted");
  const int slot = free_slots_.back();
  free_slots_.pop_back();
  std::vector<int>& pages = slot_pages_[slot];
  pages.clear();
  for (int i = 0; i < need; ++i) {
    pages.push_back(free_pages_.back());
    free_pages_.pop_back();
  }
  int* row = bt_host_.data() + static_cast<size_t>(slot) * max_pages_per_sample_;
  std::fill(row, row + max_pages_per_sample_, 0);
  std::copy(pages.begin(), pages.end(), row);
  return slot;
}

void Engine::upload_block_table(int slot, cudaStream_t st) {
  const size_t off = static_cast<size_t>(slot) * max_pages_per_sample_;
  upload(d_block_table_ + off, bt_host_.data() + off, max_pages_per_sample_ * sizeof(int), st);
}

void* Engine::decode_scratch(size_t bytes) {
  if (bytes > scratch_bytes_) {
    if (scratch_) {
      FP_CUDA(cudaStreamSynchronize(s_decode_));
      cudaFree(scratch_);
    }
    scratch_bytes_ = std::max<size_t>(bytes, 1 << 20);
    FP_CUDA(cudaMalloc(&scratch_, scratch_bytes_));
  }
  return scratch_;
}

cudaEvent_t Engine::probe_event() {
  if (probe_pool_.empty()) {
    cudaEvent_t e;
    FP_CUDA(cudaEventCreate(&e));
    return e;
  }
  cudaEvent_t e = probe_pool_.back();
  probe_pool_.pop_back();
  return e;
}

Engine::ProbeTotals Engine::drain_attn_probe() {
  ProbeTotals t;
  FP_CUDA(cudaStreamSynchronize(s_decode_));
  for (const ProbeRec& p : probes_) {
    float ms = 0.f;
    FP_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
    t.ms += ms;
    t.bytes += p.bytes;
    t.launches += 1;
    probe_pool_.push_back(p.a);
    probe_pool_.push_back(p.b);
  }
  probes_.clear();
  return t;
}

void Engine::release(int slot) {
  for (int p : slot_pages_[slot]) free_pages_.push_back(p);
  slot_pages_[slot].clear();
  free_slots_.push_back(slot);
}

// ---------------------------------------------------------------------------

void Engine::upload_tiles(PackedWs& ws, const int* cu, int n_seq, int nt[2], cudaStream_t st) {
  std::vector<int> t;
  for (int i = 0; i < 2; ++i) {
    const int rows = i ? 128 : 64;
    nt[i] = fpk::attn_tiles(cu, n_seq, rows, nullptr);
    t.assign(2 * static_cast<size_t>(nt[i]), 0);
    fpk::attn_tiles(cu, n_seq, rows, t.data());
    upload(i ? ws.tiles128 : ws.tiles, t.data(), t.size() * 4, st);
  }
}

void Engine::forward_packed(const ModelW& w, PackedWs& ws, const ActWs& a, int M, int n_seq, const int nt[2],
                            bool use_pool, cudaStream_t st) {
  (void)n_seq;
  const Dims& D = w.dims;
  const bool t128 = fpk::attn_varlen_tile_rows(D.hd) == 128;
  const fpk::KvPoolView pv = pool_view();
  fpk::embed(ws.tokens, nullptr, M, w.embed, D.d, a.x, st);
  for (int l = 0; l < D.L; ++l) {
    const LayerW& L = w.layers[l];
    fpk::rms_norm_rows(a.x, L.ln1, a.h, M, D.d, st);
    if (fuse_rope_ && D.hd == models_[kActor].dims.hd) {  // the cos/sin table is the actor's head_dim
      fpk::gemm_qkv_rope_packed(L.wqkv, D.d, a.h, M, D.H, D.KVH, D.hd, ws.pos, rope_cs_, use_pool ? &pv : nullptr, l,
                                ws.slot, a.q, a.k, a.v, st);
    } else {
      fpk::gemm_bf16(L.wqkv, D.qkv_width(), D.d, a.h, M, a.qkv, D.qkv_width(), st);
      fpk::rope_qkv(a.qkv, M, D.H, D.KVH, D.hd, ws.pos, cfg_.rope_theta, a.q, a.k, a.v, use_pool ? &pv : nullptr,
                    l, ws.slot, st);
    }
    if (use_pool && l == D.L - 1) break;  // prefill only needs the last layer's K/V
    fpk::attn_varlen(a.q, a.k, a.v, D.H, D.KVH, D.hd, M, ws.cu, t128 ? ws.tiles128 : ws.tiles, nt[t128], a.attn,
                     st);
    fpk::gemm_f32_residual(L.wo, D.d, D.H * D.hd, a.attn, M, a.x, st);
    fpk::rms_norm_rows(a.x, L.ln2, a.h, M, D.d, st);
    fpk::gemm_swiglu(L.wgu, D.F, D.d, a.h, M, a.act, st);
    fpk::gemm_f32_residual(L.wd, D.d, D.F, a.act, M, a.x, st);
  }
}

void Engine::prefill(const std::vector<PrefillItem>& items) {
  cudaStream_t st = s_decode_;
  const ModelW& w = models_[kActor];
  std::vector<int> tok, pos, slot, cu, tiles, nslot, ntok;
  size_t i = 0;
  while (i < items.size()) {
    tok.clear();
    pos.clear();
    slot.clear();
    cu.assign(1, 0);
    size_t j = i;
    while (j < items.size()) {
      const int c = items[j].ctx_tokens;
      if (j > i && static_cast<int>(tok.size()) + c > pre_.cap) break;
      if (static_cast<int>(cu.size()) >= pre_.cap_seq) break;
      for (int t = 0; t < c; ++t) {
        tok.push_back(items[j].tokens[t]);
        pos.push_back(t);
        slot.push_back(items[j].slot);
      }
      cu.push_back(static_cast<int>(tok.size()));
      ++j;
    }
    const int M = static_cast<int>(tok.size());
    const int ns = static_cast<int>(cu.size()) - 1;
    if (M > 0) {
      int nt[2];
      upload_tiles(pre_, cu.data(), ns, nt, st);
      upload(pre_.tokens, tok.data(), M * 4, st);
      upload(pre_.pos, pos.data(), M * 4, st);
      upload(pre_.slot, slot.data(), M * 4, st);
      upload(pre_.cu, cu.data(), cu.size() * 4, st);
      forward_packed(w, pre_, pre_.a[0], M, ns, nt, true, st);
    }
    i = j;
  }
  // first decode input of every admitted sample
  nslot.clear();
  ntok.clear();
  for (const PrefillItem& it : items) {
    nslot.push_back(it.slot);
    ntok.push_back(it.next_token);
  }
  if (!nslot.empty()) {
    const int n = static_cast<int>(nslot.size());
    // reuse the packed slot/token buffers (stream-ordered after the forward)
    upload(pre_.slot, nslot.data(), n * 4, st);
    upload(pre_.tokens, ntok.data(), n * 4, st);
    fpk::scatter_int(pre_.slot, pre_.tokens, n, d_cur_tok_, st);
  }
  FP_CUDA(cudaGetLastError());
}

int Engine::bucket_of(int B) {
  static const int kBuckets[] = {1,  2,  4,  8,   12,  16,  24,  32,  40,  48,  56,  64,
                                 80, 96, 112, 128, 160, 192, 224, 256, 320, 384, 448, 512};
  for (int b : kBuckets)
    if (B <= b) return b;
  return ((B + 127) / 128) * 128;
}

// Host row table of one decode group, padded to Bb rows (padding rows decode a
// dummy token into the scratch slot / page / history row): [7][Bb] columns +
// the attention work-item table. Returns the ints to upload.
size_t Engine::build_rows(const DecodeRow* rows, int B, int Bb, std::vector<int>& h, int& max_ctx,
                          double& ctx_sum) {
  const int items_cap = (cfg_.max_prompt + cfg_.max_new + 127) / 128;
  h.assign(static_cast<size_t>(7 + items_cap) * Bb + 1, 0);
  max_ctx = 0;
  ctx_sum = 0.0;
  for (int b = 0; b < Bb; ++b) {
    const bool pad = b >= B;
    const DecodeRow r = pad ? DecodeRow{cfg_.max_samples, pad_slot_, 0, 0, 0} : rows[b];
    h[b] = r.slot;
    h[Bb + b] = r.pos;
    h[2 * Bb + b] = r.pos + 1;
    h[3 * Bb + b] = r.sid * cfg_.max_new + r.step;
    h[4 * Bb + b] = r.target;
    h[5 * Bb + b] = r.sid;
    h[6 * Bb + b] = r.step;
    max_ctx = std::max(max_ctx, r.pos + 1);
    if (!pad) ctx_sum += r.pos + 1;
  }
  const Dims& A = models_[kActor].dims;
  const int n_pairs = fpk::attn_decode_items(h.data() + 2 * Bb, Bb, A.KVH, A.hd, A.H / A.KVH, h.data() + 7 * Bb);
  return static_cast<size_t>(7) * Bb + 1 + n_pairs;
}

// One decode step. Rows are padded to a batch-size bucket so that the whole
// step — ~7 kernels per layer with PDL edges — replays as one CUDA graph per
// (bucket, mode, temperature, seed, top-k, top-p): host launch cost and
// inter-kernel gaps vanish. (Cutting large batches into two halves on two
// graph branches, so one half's GEMM chain overlaps the other's attention,
// measured no faster and was removed.) The probe mode (per-launch CUDA events)
// and the traced step run eagerly.
void Engine::decode(const std::vector<DecodeRow>& rows, int mode, float inv_temp, uint64_t sample_seed, int top_k,
                    float top_p) {
  if (mode != 2 || top_p >= 1.f) top_p = 1.f;
  if (mode != 2) top_k = 0;
  const int B = static_cast<int>(rows.size());
  if (B == 0) return;
  // FUSEPLAN_TRACE_STEP=k: the engine's k-th decode step runs eagerly with
  // globaltimer stamps in every GEMM / attention launch (tools/step_trace.py)
  static const int trace_step = [] {
    const char* e = std::getenv("FUSEPLAN_TRACE_STEP");
    return e ? std::atoi(e) : -1;
  }();
  const bool tracing = ++decode_calls_ == trace_step;
  const bool graph = use_graphs_ && !probe_on_ && !tracing;
  cudaStream_t st = s_decode_;
  const int ctx_cap = cfg_.max_prompt + cfg_.max_new;
  const int Bb = graph ? bucket_of(B) : B;
  if (Bb > dec_.cap) throw std::invalid_argument("engine: decode batch exceeds max_live");
  std::vector<int> h;
  int max_ctx;
  double ctx_sum;
  const size_t n = build_rows(rows.data(), B, Bb, h, max_ctx, ctx_sum);
  upload(dec_.rows, h.data(), n * 4, st);
  if (!graph) {
    unsigned long long* arena = nullptr;
    const size_t words = size_t(1) << 22;
    if (tracing) {
      FP_CUDA(cudaMalloc(&arena, words * 8));
      FP_CUDA(cudaMemsetAsync(arena, 0, words * 8, st));
      FP_CUDA(cudaStreamSynchronize(st));
      fpk::trace_arm(arena, words);
    }
    decode_kernels(dec_, st, Bb, max_ctx, mode, inv_temp, sample_seed, ctx_sum, 148, top_k, top_p);
    if (tracing) {
      FP_CUDA(cudaStreamSynchronize(st));
      const std::vector<fpk::TraceRec> recs = fpk::trace_disarm();
      size_t used = 0;
      auto wpu_of = [](int kind) { return kind == 0 ? 8 : kind == 3 ? 16 : 4; };  // stamps per unit
      for (const auto& r : recs) used = std::max(used, r.off + static_cast<size_t>(r.units) * wpu_of(r.kind));
      std::vector<unsigned long long> th(used);
      FP_CUDA(cudaMemcpy(th.data(), arena, used * 8, cudaMemcpyDeviceToHost));
      cudaFree(arena);
      const char* path = std::getenv("FUSEPLAN_TRACE_OUT");
      FILE* f = std::fopen(path ? path : "fp_step_trace.json", "w");
      if (f) {
        std::fprintf(f, "{\"B\": %d, \"max_ctx\": %d, \"ctx_sum\": %.0f, \"launches\": [", B, max_ctx, ctx_sum);
        for (size_t i = 0; i < recs.size(); ++i) {
          const int wpu = wpu_of(recs[i].kind);
          std::fprintf(f, "%s{\"kind\": %d, \"units\": %d, \"data\": [", i ? ", " : "", recs[i].kind, recs[i].units);
          for (int u = 0; u < recs[i].units * wpu; ++u)
            std::fprintf(f, "%s%llu", u ? "," : "", th[recs[i].off + u]);
          std::fprintf(f, "]}");
        }
        std::fprintf(f, "]}\n");
        std::fclose(f);
      }
    }
    return;
  }
  run_graph(GraphKey{Bb, mode, inv_temp, sample_seed, top_k, top_p},
            [&]() { decode_kernels(dec_, st, Bb, ctx_cap, mode, inv_temp, sample_seed, 0.0, 148, top_k, top_p); });
}

// Replay the step graph of `key`; the first sight of a key runs eagerly (sets
// kernel attributes, fills the tensor-map cache), the second captures.
void Engine::run_graph(const GraphKey& key, const std::function<void()>& body) {
  cudaStream_t st = s_decode_;
  auto it = graphs_.find(key);
  if (it == graphs_.end()) {
    if (!graph_seen_.count(key)) {
      graph_seen_.insert(key);
      body();
      return;
    }
    cudaGraph_t g = nullptr;
    const long long n0 = fpk::launch_count();
    FP_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    body();
    FP_CUDA(cudaStreamEndCapture(st, &g));
    const long long nk = fpk::launch_count() - n0;
    fpk::count_launches(-nk);  // captured, not launched: counted at each replay
    cudaGraphExec_t ex = nullptr;
    FP_CUDA(cudaGraphInstantiate(&ex, g, 0));
    cudaGraphDestroy(g);
    it = graphs_.emplace(key, StepGraph{ex, nk}).first;
  }
  FP_CUDA(cudaGraphLaunch(it->second.exec, st));
  fpk::count_launches(it->second.kernels);
}

void Engine::decode_kernels(DecodeWs& dw, cudaStream_t st, int B, int max_ctx, int mode, float inv_temp,
                            uint64_t sample_seed, double ctx_sum, int attn_ctas, int top_k, float top_p) {
  const ModelW& w = models_[kActor];
  const Dims& D = w.dims;
  const int* slot = dw.rows;
  const int* pos = dw.rows + B;
  const int* ctx = dw.rows + 2 * B;
  const int* dst = dw.rows + 3 * B;
  const int* target = dw.rows + 4 * B;
  const int* sid = dw.rows + 5 * B;
  const int* step = dw.rows + 6 * B;
  const int* items = dw.rows + 7 * B;
  const fpk::KvPoolView pv = pool_view();
  const size_t stride = static_cast<size_t>(B) * D.d;
  const int so = fpk::gemm_splits(D.d, D.H * D.hd);
  const int sd = fpk::gemm_splits(D.d, D.F);

  fpk::embed_norm(d_cur_tok_, slot, B, w.embed, D.d, dw.x, w.layers[0].ln1, dw.h, st);
  fpk::gemm_qkv_rope(w.layers[0].wqkv, D.d, dw.h, B, D.H, D.KVH, D.hd, pos, rope_cs_, pv, 0, slot, dw.q, st);
  for (int l = 0; l < D.L; ++l) {
    const LayerW& L = w.layers[l];
    const bool last = l + 1 == D.L;
    const float* next_gain = last ? w.lnf : w.layers[l + 1].ln1;
    if (probe_on_) {
      ProbeRec pr{probe_event(), probe_event(), 0.0};
      const double kv_tok = 2.0 * D.KVH * D.hd * 2.0;  // K + V of one layer, bf16
      pr.bytes = ctx_sum * kv_tok + static_cast<double>(B) * D.H * D.hd * 2.0;
      fpk::attn_decode(dw.q, B, D.H, D.KVH, D.hd, pv, l, slot, ctx, items, max_ctx, dw.attn_work, dw.attn, dw.attn_cnt, st, pr.a,
                       pr.b);
      probes_.push_back(pr);
    } else {
      fpk::attn_decode(dw.q, B, D.H, D.KVH, D.hd, pv, l, slot, ctx, items, max_ctx, dw.attn_work, dw.attn, dw.attn_cnt, st,
                       nullptr, nullptr, attn_ctas);
    }
    // O -> norm -> gate/up -> down -> norm -> next QKV: one persistent launch
    // (decode_chain), or the six kernels it replaces (bit-identical)
    if (chain_ && B <= chain_max_b_) {
      fpk::DecodeChain c{};
      c.wo = L.wo, c.wgu = L.wgu, c.wd = L.wd, c.wqkv = last ? nullptr : w.layers[l + 1].wqkv;
      c.attn = dw.attn, c.h = dw.h, c.act = dw.act, c.parts = dw.parts, c.x = dw.x;
      c.gain_mlp = L.ln2, c.gain_next = next_gain;
      c.q_out = dw.q, c.pool = pv, c.slot = slot, c.pos = pos, c.cs = rope_cs_, c.layer = l;
      c.H = D.H, c.KVH = D.KVH, c.hd = D.hd, c.d = D.d, c.F = D.F, c.ao = D.H * D.hd, c.B = B;
      c.counters = dw.chain_cnt + 8 * l;
      c.ctas = chain_ctas_;
      if (fpk::decode_chain(c, st)) continue;
    }
    fpk::gemm_f32_splitk(L.wo, D.d, D.H * D.hd, dw.attn, B, dw.parts, so, st);
    fpk::add_norm(dw.x, dw.parts, so, stride, L.ln2, dw.h, B, D.d, nullptr, 0, nullptr, nullptr, st);
    fpk::gemm_swiglu_decode(L.wgu, D.F, D.d, dw.h, B, dw.act, st);
    fpk::gemm_f32_splitk(L.wd, D.d, D.F, dw.act, B, dw.parts, sd, st);
    fpk::add_norm(dw.x, dw.parts, sd, stride, next_gain, dw.h, B, D.d, nullptr, 0, nullptr, nullptr, st);
    if (!last)
      fpk::gemm_qkv_rope(w.layers[l + 1].wqkv, D.d, dw.h, B, D.H, D.KVH, D.hd, pos, rope_cs_, pv, l + 1, slot, dw.q,
                         st);
  }
  if (top_k > 0 || top_p < 1.f) {  // filtered sampling: z materialised, radix-select filter, then forced finalize
    if (!dw.logits) {  // first use runs eagerly (run_graph), never inside a capture
      dw.logits = static_cast<float*>(dalloc(static_cast<size_t>(dw.cap) * logits_ld() * sizeof(float)));
      dw.pick = static_cast<int*>(dalloc(static_cast<size_t>(dw.cap) * sizeof(int)));
    }
    fpk::gemm_vocab_logits(dw.h, B, D.d, w.head, D.V, inv_temp, dw.vocab_part, dw.logits, logits_ld(), st);
    fpk::topk_sample(dw.logits, logits_ld(), B, D.V, top_k, top_p, sid, step, sample_seed, dw.pick, dw.tgt_z, st);
    fpk::vocab_finalize(dw.vocab_part, dw.tgt_z, B, D.V, 0, dw.pick, sid, step, sample_seed, nullptr, nullptr, dst,
                        d_hist_tok_, d_hist_logp_, slot, d_cur_tok_, st);
  } else {
    fpk::gemm_vocab(dw.h, B, D.d, w.head, D.V, mode, inv_temp, target, sid, step, sample_seed, dw.vocab_part,
                    dw.tgt_z, st);
    fpk::vocab_finalize(dw.vocab_part, dw.tgt_z, B, D.V, mode, target, sid, step, sample_seed, nullptr, nullptr, dst,
                        d_hist_tok_, d_hist_logp_, slot, d_cur_tok_, st);
  }
  FP_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------

void Engine::infer(const std::vector<InferItem>& items, float beta, float gamma, float lam, bool yield) {
  struct PersistGuard {
    bool prev;
    explicit PersistGuard(bool on) : prev(fpk::packed_persistent()) { fpk::set_packed_persistent(on); }
    ~PersistGuard() { fpk::set_packed_persistent(prev); }
  } guard(!yield);
  cudaStream_t st = infer_stream();
  PackedWs& ws = inf_;
  std::vector<int> sid, P, R, cu, roff, tiles;
  std::vector<int64_t> off_out;
  std::vector<const void*> ht, hl;
  size_t i = 0;
  while (i < items.size()) {
    sid.clear(), P.clear(), R.clear(), roff.clear(), off_out.clear(), ht.clear(), hl.clear();
    cu.assign(1, 0);
    roff.push_back(0);
    size_t j = i;
    while (j < items.size()) {
      const int T = items[j].P + items[j].R;
      if (j > i && cu.back() + T > ws.cap) break;
      if (static_cast<int>(cu.size()) >= ws.cap_seq) break;
      sid.push_back(items[j].sid);
      P.push_back(items[j].P);
      R.push_back(items[j].R);
      cu.push_back(cu.back() + T);
      roff.push_back(roff.back() + items[j].R);
      off_out.push_back(resp_off_.at(items[j].sid));
      ht.push_back(items[j].hist_tok);
      hl.push_back(items[j].hist_logp);
      ++j;
    }
    const int n = static_cast<int>(sid.size());
    const int M = cu.back();
    const int NR = roff.back();
    int nt[2];
    upload_tiles(ws, cu.data(), n, nt, st);
    upload(ws.sid, sid.data(), n * 4, st);
    upload(ws.P, P.data(), n * 4, st);
    upload(ws.R, R.data(), n * 4, st);
    upload(ws.cu, cu.data(), cu.size() * 4, st);
    upload(ws.roff, roff.data(), roff.size() * 4, st);
    upload(ws.off_out, off_out.data(), n * 8, st);
    upload(ws.hist_tok, ht.data(), n * 8, st);
    upload(ws.hist_logp, hl.data(), n * 8, st);
    fpk::AssembleArgs a{ws.sid,        ws.P,      ws.R,         ws.cu,           ws.roff,
                        d_prompts_,    cfg_.max_prompt, ws.hist_tok, ws.hist_logp,
                        ws.tokens,     ws.pos,    ws.targets,   ws.logp_actor,   ws.gather_resp,
                        ws.gather_last};
    fpk::assemble_batch(a, n, st);

    // The three frozen models read the same packed batch and write disjoint
    // outputs: the critic and the reward model run on streams of their own.
    cudaStream_t s_cr = yield ? st : s_score_[0], s_rw = yield ? st : s_score_[1];
    if (!yield) {
      FP_CUDA(cudaEventRecord(ev_fork_, st));
      for (cudaStream_t s2 : s_score_) FP_CUDA(cudaStreamWaitEvent(s2, ev_fork_, 0));
    }
    // reference model: log-prob of every response token
    const ModelW& ref = models_[kRef];
    const ActWs& ar = ws.a[0];
    forward_packed(ref, ws, ar, M, n, nt, false, st);
    fpk::add_norm(ar.x, nullptr, 0, 0, ref.lnf, ar.h, M, ref.dims.d, ws.gather_resp, NR, nullptr, nullptr, st);
    fpk::gemm_vocab(ar.h, NR, ref.dims.d, ref.head, ref.dims.V, 0 /* forced */, 1.0f, ws.targets, nullptr, nullptr, 0,
                    ws.vocab_part, ws.tgt_z, st);
    fpk::vocab_finalize(ws.vocab_part, ws.tgt_z, NR, ref.dims.V, 0 /* forced */, ws.targets, nullptr, nullptr, 0, nullptr, ws.logp_ref,
                        nullptr, nullptr, nullptr, nullptr, nullptr, st);
    // critic: value of the state before each response token
    const ModelW& cr = models_[kCritic];
    forward_packed(cr, ws, ws.a[1], M, n, nt, false, s_cr);
    fpk::add_norm(ws.a[1].x, nullptr, 0, 0, cr.lnf, nullptr, M, cr.dims.d, ws.gather_resp, NR, cr.vhead, ws.values,
                  s_cr);
    // reward model: scalar score at the last token
    const ModelW& rw = models_[kReward];
    forward_packed(rw, ws, ws.a[2], M, n, nt, false, s_rw);
    fpk::add_norm(ws.a[2].x, nullptr, 0, 0, rw.lnf, nullptr, M, rw.dims.d, ws.gather_last, n, rw.vhead, ws.score,
                  s_rw);
    for (int k = 0; k < 2 && !yield; ++k) {
      FP_CUDA(cudaEventRecord(ev_join_[k], s_score_[k]));
      FP_CUDA(cudaStreamWaitEvent(st, ev_join_[k], 0));
    }

    fpk::PostScatter sc{ws.off_out,   ws.sid,          ws.targets,  exp_.logp_actor, exp_.logp_ref,
                        exp_.values,  exp_.score,      exp_.tokens};
    fpk::postprocess(n, ws.roff, ws.logp_actor, ws.logp_ref, ws.values, ws.score, beta, gamma, lam, exp_.kl,
                     exp_.reward, exp_.adv, exp_.ret, st, &sc);
    FP_CUDA(cudaGetLastError());
    i = j;
  }
}

}  // namespace fpe
