// fuseplan-b200 — C ABI of the engine (include/fp_engine.h).
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "engine.hpp"
#include "fp_engine.h"
#include "fuseplan/engine.hpp"
#include "fuseplan/errors.hpp"
#include "ops.h"

void fp_set_last_error_internal(const char* msg);             // sched_capi.cpp
const fpe::Engine& fp_engine_internal(const fuseplan::GpuEngine* g);  // executor.cpp

struct fp_engine {
  fuseplan::GpuEngine* g = nullptr;
  fuseplan::EngineSetup setup;
};
struct fp_exec {
  fuseplan::ExecResult r;
};
// fp_result is defined by sched_capi.cpp with this exact layout.
struct fp_result {
  fuseplan::GenStageResult r;
};

namespace {

// fp_last_error() lives in sched_capi.cpp; its storage is shared through a setter.
template <typename F>
int guarded(F&& body) {
  try {
    body();
    return FP_OK;
  } catch (const fuseplan::InfeasibleError& e) {
    fp_set_last_error_internal(e.what());
    return FP_EINFEASIBLE;
  } catch (const fuseplan::ConfigError& e) {
    fp_set_last_error_internal(e.what());
    return FP_EINVAL;
  } catch (const std::invalid_argument& e) {
    fp_set_last_error_internal(e.what());
    return FP_EINVAL;
  } catch (const std::exception& e) {
    fp_set_last_error_internal(e.what());
    return FP_EINTERNAL;
  } catch (...) {
    fp_set_last_error_internal("unknown error");
    return FP_EINTERNAL;
  }
}

void need(const void* p, const char* what) {
  if (!p) throw std::invalid_argument(std::string("null argument: ") + what);
}

fuseplan::EngineModelDims dims(const fp_model_dims& m) {
  return {m.num_layers, m.hidden, m.num_heads, m.num_kv_heads, m.head_dim, m.ffn, m.vocab};
}

fuseplan::ModelSpec model_of(const fp_model_spec& m) {
  fuseplan::ModelSpec s;
  s.name = m.name ? m.name : "";
  s.num_layers = m.num_layers;
  s.num_heads = m.num_heads;
  s.hidden_size = m.hidden_size;
  s.intermediate_size = m.intermediate_size;
  return s;
}

fuseplan::GenSimConfig config_of(const fp_gen_config* c) {
  need(c, "cfg");
  fuseplan::GenSimConfig g;
  g.actor = model_of(c->actor);
  g.num_instances = c->num_instances;
  g.instance_gpus = c->instance_gpus;
  for (int i = 0; i < c->num_tasks; ++i) {
    fuseplan::InferenceTask t;
    t.model = model_of(c->tasks[i]);
    t.name = (c->task_names && c->task_names[i]) ? c->task_names[i] : t.model.name;
    g.tasks.push_back(t);
  }
  g.cluster.num_gpus = c->cluster.num_gpus;
  g.cluster.gpus_per_node = c->cluster.gpus_per_node;
  g.cluster.activation_capacity_per_stage = c->cluster.activation_capacity_per_stage;
  g.cluster.kv_capacity_per_instance = c->cluster.kv_capacity_per_instance;
  g.cluster.bs_max = c->cluster.bs_max;
  g.cluster.interconnect_bandwidth = c->cluster.interconnect_bandwidth;
  g.cost.time_per_token_coeff = c->cost.time_per_token_coeff;
  g.cost.backward_forward_ratio = c->cost.backward_forward_ratio;
  g.cost.activation_bytes_coeff = c->cost.activation_bytes_coeff;
  g.cost.decode_step_base = c->cost.decode_step_base;
  g.cost.comm_bandwidth = c->cost.comm_bandwidth;
  return g;
}

cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }
using bf16 = __nv_bfloat16;

void after_launch() {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw fpe::CudaError(std::string("kernel launch: ") + cudaGetErrorString(e));
}

}  // namespace

extern "C" {

int fp_engine_create(const fp_engine_setup* s, fp_engine** out) {
  return guarded([&] {
    need(s, "setup");
    need(out, "out");
    fuseplan::EngineSetup es;
    es.actor = dims(s->actor);
    es.ref = dims(s->ref);
    es.critic = dims(s->critic);
    es.reward = dims(s->reward);
    es.weight_seed = s->weight_seed;
    es.max_prompt = s->max_prompt;
    es.max_new = s->max_new;
    es.max_samples = s->max_samples;
    es.max_live = s->max_live;
    es.kv_pool_bytes = s->kv_pool_bytes;
    es.max_prefill_tokens = s->max_prefill_tokens;
    es.max_infer_tokens = s->max_infer_tokens;
    es.rope_theta = s->rope_theta;
    es.device = s->device;
    if (es.max_prompt < 1 || es.max_new < 1 || es.max_samples < 1 || es.max_live < 1)
      throw std::invalid_argument("engine setup: sizes must be positive");
    auto* e = new fp_engine;
    e->setup = es;
    try {
      e->g = fuseplan::create_engine(es);
    } catch (...) {
      delete e;
      throw;
    }
    *out = e;
  });
}

void fp_engine_destroy(fp_engine* e) {
  if (!e) return;
  fuseplan::destroy_engine(e->g);
  delete e;
}

int fp_engine_model_size(const fp_engine* e, int32_t model, int64_t* bytes, int64_t* params) {
  return guarded([&] {
    need(e, "engine");
    if (model < 0 || model > 3) throw std::invalid_argument("model index out of range");
    const fpe::ModelW& w = fp_engine_internal(e->g).model(model);
    if (bytes) *bytes = static_cast<int64_t>(w.bytes);
    if (params) *params = static_cast<int64_t>(w.param_count);
  });
}

int fp_engine_broadcast_model(fp_engine* e, int32_t model, int32_t src, const fp_comm* comm, double* seconds) {
  return guarded([&] {
    need(e, "engine");
    need(comm, "comm");
    fuseplan::CommSetup c;
    c.rank = comm->rank;
    c.world = comm->world;
    c.shm_name = comm->shm_name ? comm->shm_name : "";
    const double t = fuseplan::broadcast_model(e->g, model, src, c);
    if (seconds) *seconds = t;
  });
}

int fp_engine_model_ptr(const fp_engine* e, int32_t model, void** dev_ptr, int64_t* bytes) {
  return guarded([&] {
    need(e, "engine");
    if (model < 0 || model > 3) throw std::invalid_argument("model index out of range");
    const fpe::ModelW& w = fp_engine_internal(e->g).model(model);
    if (dev_ptr) *dev_ptr = w.blob;
    if (bytes) *bytes = static_cast<int64_t>(w.bytes);
  });
}

int fp_engine_load_weights(fp_engine* e, int32_t model, int32_t tensor, int32_t layer, const void* host,
                           int64_t n_elems) {
  return guarded([&] {
    need(e, "engine");
    fuseplan::load_weights(e->g, model, tensor, layer, host, n_elems);
  });
}

int fp_engine_reinit_model(fp_engine* e, int32_t model, uint64_t seed) {
  return guarded([&] {
    need(e, "engine");
    if (model < 0 || model > 3) throw std::invalid_argument("model index out of range");
    fuseplan::reinit_model(e->g, model, seed);
  });
}

int fp_engine_model_checksum(fp_engine* e, int32_t model, uint64_t* sum) {
  return guarded([&] {
    need(e, "engine");
    need(sum, "sum");
    if (model < 0 || model > 3) throw std::invalid_argument("model index out of range");
    *sum = fuseplan::model_checksum(e->g, model);
  });
}

int fp_engine_kv_bytes_per_token(const fp_engine* e, int64_t* bytes) {
  return guarded([&] {
    need(e, "engine");
    need(bytes, "bytes");
    *bytes = static_cast<int64_t>(fp_engine_internal(e->g).config().model[fpe::kActor].kv_bytes_per_token());
  });
}

int fp_synthetic_prompts(const fp_engine* e, int32_t n, uint64_t token_seed, int32_t* out) {
  return guarded([&] {
    need(e, "engine");
    need(out, "out");
    const std::vector<int> p = fuseplan::synthetic_prompts(e->g, n, token_seed);
    std::memcpy(out, p.data(), p.size() * 4);
  });
}

int fp_execute(fp_engine* e, const fp_gen_sample* batch, int32_t n, const fp_gen_config* cfg, int32_t r_t,
               const fp_run_options* o, const fp_comm* comm, const int32_t* prompts, fp_exec** out) {
  return guarded([&] {
    need(e, "engine");
    need(o, "opts");
    need(out, "out");
    if (n < 1) throw std::invalid_argument("execute: empty batch");
    need(batch, "batch");
    std::vector<fuseplan::GenSample> b(n);
    for (int i = 0; i < n; ++i)
      b[i] = {batch[i].id, batch[i].prompt_len, batch[i].target_output_len, batch[i].generated, batch[i].kv_bytes};
    fuseplan::EngineOptions eo;
    if (o->token_mode < 0 || o->token_mode > 2) throw std::invalid_argument("token_mode out of range");
    eo.token_mode = static_cast<fuseplan::TokenMode>(o->token_mode);
    eo.schedule = o->schedule == FP_SCHEDULE_FUSED ? fuseplan::Schedule::kFused : fuseplan::Schedule::kStageBarrier;
    eo.temperature = o->temperature > 0.f ? o->temperature : 1.0f;
    eo.token_seed = o->token_seed;
    eo.sample_seed = o->sample_seed;
    eo.kl_beta = o->kl_beta;
    eo.gamma = o->gamma;
    eo.lam = o->lam;
    if (eo.gamma < 0.f || eo.gamma > 1.f || eo.lam < 0.f || eo.lam > 1.f)
      throw std::invalid_argument("GaeInputs: gamma and lam must lie in [0, 1]");
    eo.claim_tokens = o->claim_tokens > 0 ? o->claim_tokens : 8192;
    eo.run_ahead = o->run_ahead > 0 ? o->run_ahead : 4;
    eo.resident = o->resident != 0;
    eo.probe_attention = o->probe_attention != 0;
    eo.handoff_dp = o->handoff_dp;
    eo.claim_max_live = o->claim_max_live;
    eo.eos_id = o->eos_id;
    eo.eos_lag = o->eos_lag;
    eo.online_trigger = o->online_trigger != 0;
    eo.top_k = o->top_k;
    eo.top_p = o->top_p;
    fuseplan::CommSetup cs;
    if (comm) {
      cs.rank = comm->rank;
      cs.world = comm->world;
      cs.shm_name = comm->shm_name ? comm->shm_name : "";
    }
    if (cs.world > 1 && cs.shm_name.empty()) throw std::invalid_argument("comm: shm_name required for world > 1");
    std::vector<int> pv;
    if (prompts) pv.assign(prompts, prompts + static_cast<size_t>(n) * e->setup.max_prompt);
    auto* x = new fp_exec;
    try {
      x->r = fuseplan::execute(e->g, b, config_of(cfg), r_t, eo, cs, prompts ? &pv : nullptr);
    } catch (...) {
      delete x;
      throw;
    }
    *out = x;
  });
}

int fp_exec_stats_get(const fp_exec* x, fp_exec_stats* s) {
  return guarded([&] {
    need(x, "exec");
    need(s, "stats");
    const fuseplan::ExecStats& t = x->r.stats;
    s->wall_seconds = t.wall_seconds;
    s->gen_seconds = t.gen_seconds;
    s->trigger_seconds = t.trigger_seconds;
    s->migrate_seconds = t.migrate_seconds;
    s->infer_busy_seconds = t.infer_busy_seconds;
    s->decode_gpu_seconds = t.decode_gpu_seconds;
    s->decode_steps = t.decode_steps;
    s->decode_rows = t.decode_rows;
    s->decode_ctx_tokens = t.decode_ctx_tokens;
    s->prefill_tokens = t.prefill_tokens;
    s->infer_tokens = t.infer_tokens;
    s->infer_samples = t.infer_samples;
    s->migrated_in = t.migrated_in;
    s->migrated_bytes = t.migrated_bytes;
    s->total_resp = x->r.experience.resp_off.empty() ? 0 : x->r.experience.resp_off.back();
    s->gpu_launches = t.gpu_launches;
    s->attn_probe_ms = t.attn_probe_ms;
    s->attn_probe_bytes = t.attn_probe_bytes;
    s->attn_probe_launches = t.attn_probe_launches;
    s->ipc_seconds = t.ipc_seconds;
    s->eos_retired = t.eos_retired;
    s->overrun_rows = t.overrun_rows;
    s->online = x->r.online ? 1 : 0;
  });
}

int fp_exec_experience(const fp_exec* x, int64_t* resp_off, int32_t* tokens, float* logp_actor, float* logp_ref,
                       float* values, float* kl, float* reward, float* adv, float* ret, float* score) {
  return guarded([&] {
    need(x, "exec");
    const fuseplan::ExperienceBatch& b = x->r.experience;
    auto cp = [](auto* dst, const auto& v) {
      if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(v[0]));
    };
    cp(resp_off, b.resp_off);
    cp(tokens, b.tokens);
    cp(logp_actor, b.logp_actor);
    cp(logp_ref, b.logp_ref);
    cp(values, b.values);
    cp(kl, b.kl);
    cp(reward, b.reward);
    cp(adv, b.adv);
    cp(ret, b.ret);
    cp(score, b.score);
  });
}

int fp_exec_finish(const fp_exec* x, double* finish_seconds, int32_t* finish_instance) {
  return guarded([&] {
    need(x, "exec");
    if (finish_seconds) std::memcpy(finish_seconds, x->r.finish_wall.data(), x->r.finish_wall.size() * 8);
    if (finish_instance)
      for (size_t i = 0; i < x->r.finish_instance.size(); ++i) finish_instance[i] = x->r.finish_instance[i];
  });
}

int fp_exec_decision(const fp_exec* x, fp_result** out) {
  return guarded([&] {
    need(x, "exec");
    need(out, "out");
    *out = new fp_result{x->r.decision};
  });
}

int fp_exec_moves(const fp_exec* x, int32_t* n_moves, int32_t* sample, int32_t* from, int32_t* to) {
  return guarded([&] {
    need(x, "exec");
    const auto& t = x->r.trigger;
    if (n_moves) *n_moves = static_cast<int32_t>(t.move_sample.size());
    for (size_t i = 0; i < t.move_sample.size(); ++i) {
      if (sample) sample[i] = t.move_sample[i];
      if (from) from[i] = t.move_from[i];
      if (to) to[i] = t.move_to[i];
    }
  });
}

int fp_exec_received(const fp_exec* x, int32_t* n, int32_t* sample, int32_t* from) {
  return guarded([&] {
    need(x, "exec");
    const auto& r = x->r;
    if (n) *n = static_cast<int32_t>(r.received_sample.size());
    for (size_t i = 0; i < r.received_sample.size(); ++i) {
      if (sample) sample[i] = r.received_sample[i];
      if (from) from[i] = r.received_from[i];
    }
  });
}

int fp_exec_trigger_state(const fp_exec* x, double* time, int32_t* n, fp_remaining* samples) {
  return guarded([&] {
    need(x, "exec");
    const fuseplan::GenState& st = x->r.trigger.state;
    if (time) *time = st.time;
    if (n) *n = static_cast<int32_t>(st.samples.size());
    if (samples)
      for (size_t i = 0; i < st.samples.size(); ++i) {
        const auto& r = st.samples[i];
        samples[i] = fp_remaining{r.id, r.instance, r.kv_bytes, r.generated, r.prompt_len, r.admitted ? 1 : 0};
      }
  });
}

int fp_exec_handoff(const fp_exec* x, int32_t* dp, int32_t* group_begin, int32_t* group_end, int32_t* order,
                    int32_t* group_off, int64_t* packed_off, void** dev, double* seconds, int64_t* bytes,
                    int64_t* peer_bytes) {
  return guarded([&] {
    need(x, "exec");
    const fuseplan::Handoff& h = x->r.handoff;
    if (dp) *dp = h.dp;
    if (group_begin) *group_begin = h.group_begin;
    if (group_end) *group_end = h.group_end;
    if (order) std::copy(h.order.begin(), h.order.end(), order);
    if (group_off) std::copy(h.group_off.begin(), h.group_off.end(), group_off);
    if (packed_off) std::copy(h.packed_off.begin(), h.packed_off.end(), packed_off);
    if (dev) {
      dev[0] = const_cast<int*>(h.tokens);
      for (int k = 0; k < 7; ++k) dev[1 + k] = const_cast<float*>(h.arrays[k]);
      dev[8] = const_cast<float*>(h.score);
    }
    if (seconds) *seconds = h.seconds;
    if (bytes) *bytes = h.bytes;
    if (peer_bytes) *peer_bytes = h.peer_bytes;
  });
}

int fp_exec_handoff_download(const fp_exec* x, void** host) {
  return guarded([&] {
    need(x, "exec");
    need(host, "host");
    const fuseplan::Handoff& h = x->r.handoff;
    if (h.dp == 0) throw std::invalid_argument("handoff: the run had handoff_dp = 0");
    const int k0 = h.group_off[h.group_begin], k1 = h.group_off[h.group_end];
    const size_t toks = static_cast<size_t>(h.packed_off[k1] - h.packed_off[k0]);
    const void* src[9] = {h.tokens, h.arrays[0], h.arrays[1], h.arrays[2], h.arrays[3],
                          h.arrays[4], h.arrays[5], h.arrays[6], h.score};
    for (int a = 0; a < 9; ++a) {
      const size_t bytes = (a == 8 ? static_cast<size_t>(k1 - k0) : toks) * 4;
      if (host[a] && bytes) fpe::check(cudaMemcpy(host[a], src[a], bytes, cudaMemcpyDeviceToHost), "handoff d2h");
    }
  });
}

int fp_exec_steps(const fp_exec* x, int32_t* n_steps, int32_t* rows, float* ms, int64_t* ctx) {
  return guarded([&] {
    need(x, "exec");
    if (n_steps) *n_steps = static_cast<int32_t>(x->r.step_rows.size());
    for (size_t i = 0; i < x->r.step_rows.size(); ++i) {
      if (rows) rows[i] = x->r.step_rows[i];
      if (ms) ms[i] = i < x->r.step_ms.size() ? x->r.step_ms[i] : 0.f;
      if (ctx) ctx[i] = i < x->r.step_ctx.size() ? x->r.step_ctx[i] : 0;
    }
  });
}

void fp_exec_free(fp_exec* x) { delete x; }

// ---- single kernels ----------------------------------------------------------------

int fp_k_init_bf16(void* w, int64_t n, uint64_t seed, uint64_t tag, float scale, void* stream) {
  return guarded([&] {
    fpk::init_bf16(static_cast<bf16*>(w), static_cast<size_t>(n), seed, tag, scale, S(stream));
    after_launch();
  });
}

int fp_k_gemm_bf16(const void* W, int32_t N, int32_t K, const void* X, int32_t M, void* out, int32_t ld,
                   void* stream) {
  return guarded([&] {
    fpk::gemm_bf16(static_cast<const bf16*>(W), N, K, static_cast<const bf16*>(X), M, static_cast<bf16*>(out), ld,
                   S(stream));
    after_launch();
  });
}

int fp_k_gemm_f32_residual(const void* W, int32_t N, int32_t K, const void* X, int32_t M, float* resid,
                           void* stream) {
  return guarded([&] {
    fpk::gemm_f32_residual(static_cast<const bf16*>(W), N, K, static_cast<const bf16*>(X), M, resid, S(stream));
    after_launch();
  });
}

int fp_k_gemm_splits(int32_t N, int32_t K) { return fpk::gemm_splits(N, K); }

int fp_k_gemm_f32(const void* W, int32_t N, int32_t K, const void* X, int32_t M, float* out, int32_t splits,
                  void* stream) {
  return guarded([&] {
    fpk::gemm_f32_splitk(static_cast<const bf16*>(W), N, K, static_cast<const bf16*>(X), M, out,
                         splits > 0 ? splits : fpk::gemm_splits(N, K), S(stream));
    after_launch();
  });
}

int fp_k_gemm_swiglu(const void* Wgu, int32_t F, int32_t K, const void* X, int32_t M, void* out, void* stream) {
  return guarded([&] {
    fpk::gemm_swiglu(static_cast<const bf16*>(Wgu), F, K, static_cast<const bf16*>(X), M, static_cast<bf16*>(out),
                     S(stream));
    after_launch();
  });
}

int fp_k_gemm_swiglu_decode(const void* Wgu, int32_t F, int32_t K, const void* X, int32_t M, void* out,
                            void* stream) {
  return guarded([&] {
    fpk::gemm_swiglu_decode(static_cast<const bf16*>(Wgu), F, K, static_cast<const bf16*>(X), M,
                            static_cast<bf16*>(out), S(stream));
    after_launch();
  });
}

int fp_k_qkv_rope(const void* Wqkv, int32_t K, const void* X, int32_t M, int32_t H, int32_t KVH, int32_t hd,
                  const int32_t* pos, int32_t max_pos, float rope_theta, void* pool, int32_t num_layers,
                  int32_t layer, const int32_t* block_table, int32_t bt_stride, const int32_t* slot, void* q_out,
                  void* stream) {
  return guarded([&] {
    const size_t layer_bytes = static_cast<size_t>(KVH) * 2 * 64 * hd * 2;
    fpk::KvPoolView pv{static_cast<uint8_t*>(pool), layer_bytes * num_layers, layer_bytes, 64, block_table,
                       bt_stride};
    float2* cs = nullptr;
    const size_t cb = static_cast<size_t>(max_pos) * (hd / 2) * sizeof(float2);
    fpe::check(cudaMallocAsync(reinterpret_cast<void**>(&cs), cb, S(stream)), "alloc");
    fpk::rope_table(cs, max_pos, hd, rope_theta, S(stream));
    fpk::gemm_qkv_rope(static_cast<const bf16*>(Wqkv), K, static_cast<const bf16*>(X), M, H, KVH, hd, pos, cs, pv,
                       layer, slot, static_cast<bf16*>(q_out), S(stream));
    after_launch();
    fpe::check(cudaFreeAsync(cs, S(stream)), "free");
  });
}

int fp_k_vocab(const void* X, int32_t M, int32_t K, const void* W, int32_t V, int32_t mode, float inv_temp,
               const int32_t* target, const int32_t* sample_id, const int32_t* step, uint64_t seed, int32_t* token,
               float* logp, void* stream) {
  return guarded([&] {
    void* part = nullptr;
    float* tz = nullptr;
    fpe::check(cudaMallocAsync(&part, static_cast<size_t>(M) * fpk::vocab_tiles(V) * 24 + 256, S(stream)), "alloc");
    fpe::check(cudaMallocAsync(reinterpret_cast<void**>(&tz), static_cast<size_t>(M) * 4 + 256, S(stream)), "alloc");
    fpk::gemm_vocab(static_cast<const bf16*>(X), M, K, static_cast<const bf16*>(W), V, mode, inv_temp, target,
                    sample_id, step, seed, part, tz, S(stream));
    fpk::vocab_finalize(part, tz, M, V, mode, target, sample_id, step, seed, token, logp, nullptr, nullptr, nullptr, nullptr, nullptr,
                        S(stream));
    after_launch();
    fpe::check(cudaFreeAsync(part, S(stream)), "free");
    fpe::check(cudaFreeAsync(tz, S(stream)), "free");
  });
}

int fp_k_decode_chain(const void* Wo, const void* Wgu, const void* Wd, const void* Wqkv, const void* attn, void* h,
                      void* act, float* parts, float* x, const float* gain_mlp, const float* gain_next, void* q_out,
                      void* pool, int32_t num_layers, int32_t layer, const int32_t* block_table, int32_t bt_stride,
                      const int32_t* slot, const int32_t* pos, int32_t max_pos, float rope_theta, int32_t M,
                      int32_t d, int32_t H, int32_t KVH, int32_t hd, int32_t F, void* stream) {
  return guarded([&] {
    const size_t layer_bytes = static_cast<size_t>(KVH) * 2 * 64 * hd * 2;
    float2* cs = nullptr;
    const size_t cb = static_cast<size_t>(max_pos) * (hd / 2) * sizeof(float2);
    fpe::check(cudaMallocAsync(reinterpret_cast<void**>(&cs), cb, S(stream)), "alloc");
    fpk::rope_table(cs, max_pos, hd, rope_theta, S(stream));
    int* cnt = nullptr;
    fpe::check(cudaMallocAsync(reinterpret_cast<void**>(&cnt), 64, S(stream)), "alloc");
    fpe::check(cudaMemsetAsync(cnt, 0, 64, S(stream)), "memset");
    fpk::DecodeChain c{};
    c.wo = static_cast<const bf16*>(Wo), c.wgu = static_cast<const bf16*>(Wgu), c.wd = static_cast<const bf16*>(Wd);
    c.wqkv = static_cast<const bf16*>(Wqkv);
    c.attn = static_cast<const bf16*>(attn), c.h = static_cast<bf16*>(h), c.act = static_cast<bf16*>(act);
    c.parts = parts, c.x = x, c.gain_mlp = gain_mlp, c.gain_next = gain_next;
    c.q_out = static_cast<bf16*>(q_out);
    c.pool = fpk::KvPoolView{static_cast<uint8_t*>(pool), layer_bytes * num_layers, layer_bytes, 64, block_table, bt_stride};
    c.slot = slot, c.pos = pos, c.cs = cs, c.layer = layer;
    c.H = H, c.KVH = KVH, c.hd = hd, c.d = d, c.F = F, c.ao = H * hd, c.B = M;
    c.counters = cnt;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    c.ctas = sms;
    if (!fpk::decode_chain(c, S(stream))) throw std::invalid_argument("fp_k_decode_chain: unsupported shape");
    after_launch();
    fpe::check(cudaFreeAsync(cs, S(stream)), "free");
    fpe::check(cudaFreeAsync(cnt, S(stream)), "free");
  });
}

int fp_k_vocab_filtered(const void* X, int32_t M, int32_t K, const void* W, int32_t V, float inv_temp, int32_t top_k,
                        float top_p, const int32_t* sample_id, const int32_t* step, uint64_t seed, int32_t* token,
                        float* logp, float* z_out, void* stream) {
  return guarded([&] {
    void* part = nullptr;
    float *tz = nullptr, *z = z_out;
    int* pick = nullptr;
    const int ldv = z_out ? V : (V + 3) & ~3;
    if (z_out && V % 4) throw std::invalid_argument("fp_k_vocab_filtered: z_out needs V % 4 == 0");
    fpe::check(cudaMallocAsync(&part, static_cast<size_t>(M) * fpk::vocab_tiles(V) * 24 + 256, S(stream)), "alloc");
    fpe::check(cudaMallocAsync(reinterpret_cast<void**>(&tz), static_cast<size_t>(M) * 4 + 256, S(stream)), "alloc");
    fpe::check(cudaMallocAsync(reinterpret_cast<void**>(&pick), static_cast<size_t>(M) * 4 + 256, S(stream)), "alloc");
    if (!z) fpe::check(cudaMallocAsync(reinterpret_cast<void**>(&z), static_cast<size_t>(M) * ldv * 4 + 256, S(stream)), "alloc");
    fpk::gemm_vocab_logits(static_cast<const bf16*>(X), M, K, static_cast<const bf16*>(W), V, inv_temp, part, z, ldv,
                           S(stream));
    fpk::topk_sample(z, ldv, M, V, top_k, top_p, sample_id, step, seed, pick, tz, S(stream));
    fpk::vocab_finalize(part, tz, M, V, 0, pick, sample_id, step, seed, token, logp, nullptr, nullptr, nullptr, nullptr,
                        nullptr, S(stream));
    after_launch();
    fpe::check(cudaFreeAsync(part, S(stream)), "free");
    fpe::check(cudaFreeAsync(tz, S(stream)), "free");
    fpe::check(cudaFreeAsync(pick, S(stream)), "free");
    if (!z_out) fpe::check(cudaFreeAsync(z, S(stream)), "free");
  });
}

int fp_k_embed_norm(const int32_t* tokens, const int32_t* idx, int32_t M, const void* E, int32_t d, float* x,
                    const float* gain, void* y, void* stream) {
  return guarded([&] {
    fpk::embed_norm(tokens, idx, M, static_cast<const bf16*>(E), d, x, gain, static_cast<bf16*>(y), S(stream));
    after_launch();
  });
}

int fp_k_add_norm(float* x, const float* parts, int32_t nsplit, const float* gain, void* y, int32_t M, int32_t d,
                  void* stream) {
  return guarded([&] {
    fpk::add_norm(x, parts, nsplit, static_cast<size_t>(M) * d, gain, static_cast<bf16*>(y), M, d, nullptr, 0, nullptr,
                  nullptr, S(stream));
    after_launch();
  });
}

int fp_k_rms_norm_rows(const float* x, const float* gain, void* y, int32_t M, int32_t d, void* stream) {
  return guarded([&] {
    fpk::rms_norm_rows(x, gain, static_cast<bf16*>(y), M, d, S(stream));
    after_launch();
  });
}

int fp_k_attn_decode(const void* q, int32_t B, int32_t H, int32_t KVH, int32_t hd, const void* pool,
                     int32_t num_pages, int32_t num_layers, int32_t layer, const int32_t* block_table,
                     int32_t bt_stride, const int32_t* slot, const int32_t* ctx, int32_t max_ctx, void* out,
                     void* stream) {
  return guarded([&] {
    const size_t layer_bytes = static_cast<size_t>(KVH) * 2 * 64 * hd * 2;
    fpk::KvPoolView pv{static_cast<uint8_t*>(const_cast<void*>(pool)), layer_bytes * num_layers, layer_bytes, 64,
                       block_table, bt_stride};
    CUtensorMap map;
    if (num_pages > 0 && (hd == 64 || hd == 128)) {
      map = fpk::make_kv_map(pool, static_cast<long long>(num_pages) * (layer_bytes * num_layers / (hd * 2)), hd);
      pv.kv_map = &map;
    }
    float* work = nullptr;
    const size_t wb = fpk::attn_decode_workspace(B, H, hd, max_ctx) * 4 + 256;
    const size_t cb = static_cast<size_t>(fpk::attn_decode_counters(B, KVH, max_ctx)) * 4;
    const size_t ob = (1 + static_cast<size_t>(B) * ((max_ctx + 127) / 128)) * 4;
    fpe::check(cudaMallocAsync(reinterpret_cast<void**>(&work), wb + cb + ob, S(stream)), "alloc");
    int* counters = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(work) + wb);
    int* items = counters + fpk::attn_decode_counters(B, KVH, max_ctx);
    fpe::check(cudaMemsetAsync(counters, 0, cb, S(stream)), "memset");
    std::vector<int> hc(B), hi(ob / 4);
    {  // work-item table from the contexts (host; this entry is a test / tooling path)
      fpe::check(cudaMemcpyAsync(hc.data(), ctx, B * 4, cudaMemcpyDeviceToHost, S(stream)), "ctx d2h");
      fpe::check(cudaStreamSynchronize(S(stream)), "sync");
      for (int b = 0; b < B; ++b)
        if (hc[b] < 1 || hc[b] > max_ctx) throw std::invalid_argument("attn_decode: ctx out of [1, max_ctx]");
      fpk::attn_decode_items(hc.data(), B, KVH, hd, H / KVH, hi.data());
      fpe::check(cudaMemcpyAsync(items, hi.data(), ob, cudaMemcpyHostToDevice, S(stream)), "items h2d");
    }
    fpk::attn_decode(static_cast<const bf16*>(q), B, H, KVH, hd, pv, layer, slot, ctx, items, max_ctx, work,
                     static_cast<bf16*>(out), counters, S(stream));
    after_launch();
    fpe::check(cudaFreeAsync(work, S(stream)), "free");
  });
}

void fp_k_attn_trace(void* buf) { fpk::set_attn_trace(static_cast<unsigned long long*>(buf)); }

int64_t fp_k_attn_workspace_bytes(int32_t B, int32_t H, int32_t KVH, int32_t hd, int32_t max_ctx) {
  return static_cast<int64_t>(fpk::attn_decode_workspace(B, H, hd, max_ctx)) * 4 + 256 +
         static_cast<int64_t>(fpk::attn_decode_counters(B, KVH, max_ctx)) * 4;
}

int fp_k_attn_items(const int32_t* ctx_host, int32_t B, int32_t H, int32_t KVH, int32_t hd, int32_t max_ctx,
                    int32_t* items_host) {
  return guarded([&] {
    for (int b = 0; b < B; ++b)
      if (ctx_host[b] < 1 || ctx_host[b] > max_ctx) throw std::invalid_argument("attn_items: ctx out of [1, max_ctx]");
    fpk::attn_decode_items(ctx_host, B, KVH, hd, H / KVH, items_host);
  });
}

int fp_k_attn_decode_ws(const void* q, int32_t B, int32_t H, int32_t KVH, int32_t hd, const void* pool,
                        int32_t num_pages, int32_t num_layers, int32_t layer, const int32_t* block_table,
                        int32_t bt_stride, const int32_t* slot, const int32_t* ctx, const int32_t* items_dev,
                        int32_t max_ctx, void* workspace, void* out, void* stream) {
  return guarded([&] {
    const size_t layer_bytes = static_cast<size_t>(KVH) * 2 * 64 * hd * 2;
    fpk::KvPoolView pv{static_cast<uint8_t*>(const_cast<void*>(pool)), layer_bytes * num_layers, layer_bytes, 64,
                       block_table, bt_stride};
    CUtensorMap map;
    if (num_pages > 0 && (hd == 64 || hd == 128)) {
      map = fpk::make_kv_map(pool, static_cast<long long>(num_pages) * (layer_bytes * num_layers / (hd * 2)), hd);
      pv.kv_map = &map;
    }
    float* work = static_cast<float*>(workspace);
    int* counters = reinterpret_cast<int*>(static_cast<uint8_t*>(workspace) +
                                           fpk::attn_decode_workspace(B, H, hd, max_ctx) * 4 + 256);
    fpk::attn_decode(static_cast<const bf16*>(q), B, H, KVH, hd, pv, layer, slot, ctx, items_dev, max_ctx, work,
                     static_cast<bf16*>(out), counters, S(stream));
    after_launch();
  });
}

namespace {
int attn_varlen_call(const void* q, const void* k, const void* v, int H, int KVH, int hd, const int32_t* cu_host,
                     const int32_t* cu_dev, int n_seq, void* out, void* stream, bool mma) {
  return guarded([&] {
    const int rows = mma ? 64 : fpk::attn_varlen_tile_rows(hd);
    const int nt = fpk::attn_tiles(cu_host, n_seq, rows, nullptr);
    std::vector<int> tiles(2 * static_cast<size_t>(nt));
    fpk::attn_tiles(cu_host, n_seq, rows, tiles.data());
    int* dt = nullptr;
    fpe::check(cudaMallocAsync(reinterpret_cast<void**>(&dt), tiles.size() * 4 + 256, S(stream)), "alloc");
    fpe::check(cudaMemcpyAsync(dt, tiles.data(), tiles.size() * 4, cudaMemcpyHostToDevice, S(stream)), "copy");
    const auto* qb = static_cast<const bf16*>(q);
    const auto* kb = static_cast<const bf16*>(k);
    const auto* vb = static_cast<const bf16*>(v);
    if (mma)
      fpk::attn_varlen_mma(qb, kb, vb, H, KVH, hd, cu_dev, dt, nt, static_cast<bf16*>(out), S(stream));
    else
      fpk::attn_varlen(qb, kb, vb, H, KVH, hd, cu_host[n_seq], cu_dev, dt, nt, static_cast<bf16*>(out), S(stream));
    after_launch();
    fpe::check(cudaStreamSynchronize(S(stream)), "sync");  // tiles lives on the host stack
    fpe::check(cudaFreeAsync(dt, S(stream)), "free");
  });
}
}  // namespace

int fp_k_set_packed_persistent(int on) {
  return guarded([&] { fpk::set_packed_persistent(on != 0); });
}

int fp_k_set_attn_cut(int mode) {
  return guarded([&] { fpk::set_attn_cut(mode); });
}

int fp_k_set_pair_gemm(int mode) {
  return guarded([&] { fpk::set_pair_gemm(mode); });
}

int fp_k_attn_prefill_trace(void* buf) {
  return guarded([&] { fpk::attn_prefill_set_trace(static_cast<unsigned long long*>(buf)); });
}

int fp_k_attn_varlen(const void* q, const void* k, const void* v, int32_t H, int32_t KVH, int32_t hd,
                     const int32_t* cu_host, const int32_t* cu_dev, int32_t n_seq, void* out, void* stream) {
  return attn_varlen_call(q, k, v, H, KVH, hd, cu_host, cu_dev, n_seq, out, stream, false);
}

int fp_k_attn_varlen_mma(const void* q, const void* k, const void* v, int32_t H, int32_t KVH, int32_t hd,
                         const int32_t* cu_host, const int32_t* cu_dev, int32_t n_seq, void* out, void* stream) {
  return attn_varlen_call(q, k, v, H, KVH, hd, cu_host, cu_dev, n_seq, out, stream, true);
}

int fp_k_postprocess(int32_t n, const int32_t* off, const float* logp_actor, const float* logp_ref,
                     const float* values, const float* score, float beta, float gamma, float lam, float* kl,
                     float* reward, float* adv, float* ret, void* stream) {
  return guarded([&] {
    if (gamma < 0.f || gamma > 1.f || lam < 0.f || lam > 1.f)
      throw std::invalid_argument("GaeInputs: gamma and lam must lie in [0, 1]");
    fpk::postprocess(n, off, logp_actor, logp_ref, values, score, beta, gamma, lam, kl, reward, adv, ret, S(stream));
    after_launch();
  });
}

}  // extern "C"

extern "C" int fp_k_gemm_trace(void* buf) {
  fpk::set_gemm_trace(static_cast<unsigned long long*>(buf));
  return FP_OK;
}
