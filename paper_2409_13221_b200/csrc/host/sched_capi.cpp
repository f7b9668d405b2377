// fuseplan-b200 — C ABI adapter of the scheduler (include/fp_sched.h).
//
// Uses only the public fuseplan C++ API (genfuse.hpp, numerics.hpp,
// errors.hpp). It is therefore compiled twice: into the product library
// against this repo's include/fuseplan, and by oracle/Makefile against the
// reference's proj/include/fuseplan + proj/src sources, yielding an oracle
// library with an identical ABI.
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "fp_sched.h"
#include "fuseplan/errors.hpp"
#include "fuseplan/genfuse.hpp"
#include "fuseplan/minibatch.hpp"
#include "fuseplan/numerics.hpp"

struct fp_result {
  fuseplan::GenStageResult r;
};
struct fp_plan {
  fuseplan::MigrationPlan p;
};

namespace {

thread_local std::string g_error;

template <typename F>
int guarded(F&& body) {
  try {
    body();
    return FP_OK;
  } catch (const fuseplan::InfeasibleError& e) {
    g_error = e.what();
    return FP_EINFEASIBLE;
  } catch (const fuseplan::ConfigError& e) {
    g_error = e.what();
    return FP_EINVAL;
  } catch (const std::invalid_argument& e) {
    g_error = e.what();
    return FP_EINVAL;
  } catch (const std::exception& e) {
    g_error = e.what();
    return FP_EINTERNAL;
  } catch (...) {
    g_error = "unknown error";
    return FP_EINTERNAL;
  }
}

void need(const void* p, const char* what) {
  if (p == nullptr) throw std::invalid_argument(std::string("null argument: ") + what);
}

fuseplan::ModelSpec to_model(const fp_model_spec& m) {
  fuseplan::ModelSpec s;
  s.name = m.name ? m.name : "";
  s.num_layers = m.num_layers;
  s.num_heads = m.num_heads;
  s.hidden_size = m.hidden_size;
  s.intermediate_size = m.intermediate_size;
  return s;
}

fuseplan::GenSimConfig to_config(const fp_gen_config* c) {
  need(c, "cfg");
  fuseplan::GenSimConfig g;
  g.actor = to_model(c->actor);
  g.num_instances = c->num_instances;
  g.instance_gpus = c->instance_gpus;
  if (c->num_tasks < 0) throw std::invalid_argument("num_tasks < 0");
  if (c->num_tasks > 0) need(c->tasks, "cfg.tasks");
  for (int i = 0; i < c->num_tasks; ++i) {
    fuseplan::InferenceTask t;
    t.model = to_model(c->tasks[i]);
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

fuseplan::LengthDistribution to_dist(const fp_length_dist* d) {
  need(d, "dist");
  fuseplan::LengthDistribution out;
  out.kind = d->kind == 1 ? fuseplan::LengthDistribution::Kind::kEmpirical
                          : fuseplan::LengthDistribution::Kind::kLognormal;
  out.median = d->median;
  out.p999_ratio = d->p999_ratio;
  out.max_len = d->max_len;
  if (d->n_empirical > 0) {
    need(d->empirical, "dist.empirical");
    out.empirical.assign(d->empirical, d->empirical + d->n_empirical);
  }
  return out;
}

std::vector<fuseplan::GenSample> to_batch(const fp_gen_sample* b, int n) {
  if (n < 0) throw std::invalid_argument("negative batch size");
  if (n > 0) need(b, "batch");
  std::vector<fuseplan::GenSample> v(n);
  for (int i = 0; i < n; ++i) {
    v[i].id = b[i].id;
    v[i].prompt_len = b[i].prompt_len;
    v[i].target_output_len = b[i].target_output_len;
    v[i].generated = b[i].generated;
    v[i].kv_bytes = b[i].kv_bytes;
  }
  return v;
}

int kind_code(const std::string& k) {
  static const char* const names[] = {"admit",      "finish",         "trigger", "migrate_out",
                                      "migrate_in", "join_inference", "gen_end", "inf_end"};
  for (int i = 0; i < 8; ++i)
    if (k == names[i]) return i;
  return -1;
}

void fill_plan(const fuseplan::MigrationPlan& p, fp_plan_info* info) {
  info->trigger_time = p.trigger_time;
  info->r_t = p.r_t;
  info->m = p.m;
  info->mechanism = static_cast<int32_t>(p.mechanism);
  info->no_op = p.no_op ? 1 : 0;
  info->overhead = p.overhead;
  info->n_destinations = static_cast<int32_t>(p.destinations.size());
  info->n_migrated = static_cast<int32_t>(p.migrated.size());
}

}  // namespace

void fp_set_last_error_internal(const char* msg) { g_error = msg ? msg : ""; }

extern "C" {

const char* fp_last_error(void) { return g_error.c_str(); }

int fp_sample_lengths(const fp_length_dist* dist, int32_t n, uint64_t seed, int32_t* out) {
  return guarded([&] {
    need(out, "out");
    const std::vector<int> v = fuseplan::sample_lengths(to_dist(dist), n, seed);
    std::memcpy(out, v.data(), v.size() * sizeof(int32_t));
  });
}

int fp_load_length_file(const char* path, int32_t* out, int32_t cap, int32_t* count) {
  return guarded([&] {
    need(path, "path");
    need(count, "count");
    const std::vector<int> v = fuseplan::load_length_file(path);
    *count = static_cast<int32_t>(v.size());
    if (out != nullptr)
      for (int i = 0; i < cap && i < static_cast<int>(v.size()); ++i) out[i] = v[i];
  });
}

int fp_make_batch(const fp_length_dist* dist, int32_t n, int32_t prompt_len, const fp_model_spec* actor,
                  uint64_t seed, fp_gen_sample* out) {
  return guarded([&] {
    need(actor, "actor");
    need(out, "out");
    const auto b = fuseplan::make_batch(to_dist(dist), n, prompt_len, to_model(*actor), seed);
    for (std::size_t i = 0; i < b.size(); ++i)
      out[i] = {b[i].id, b[i].prompt_len, b[i].target_output_len, b[i].generated, b[i].kv_bytes};
  });
}

int fp_kv_bytes_per_token(const fp_model_spec* spec, double* out) {
  return guarded([&] {
    need(spec, "spec");
    need(out, "out");
    *out = fuseplan::kv_bytes_per_token(to_model(*spec));
  });
}

int fp_plan_migration(double time, const fp_remaining* samples, int32_t n, int32_t r_t,
                      const fp_gen_config* cfg, fp_plan** out) {
  return guarded([&] {
    need(out, "out");
    if (n > 0) need(samples, "samples");
    fuseplan::GenState st;
    st.time = time;
    for (int i = 0; i < n; ++i) {
      fuseplan::GenState::Remaining r;
      r.id = samples[i].id;
      r.instance = samples[i].instance;
      r.kv_bytes = samples[i].kv_bytes;
      r.generated = samples[i].generated;
      r.prompt_len = samples[i].prompt_len;
      r.admitted = samples[i].admitted != 0;
      st.samples.push_back(r);
    }
    auto* p = new fp_plan{fuseplan::plan_migration(st, r_t, to_config(cfg))};
    *out = p;
  });
}

int fp_plan_info_get(const fp_plan* p, fp_plan_info* info, int32_t* destinations, int32_t* migrated) {
  return guarded([&] {
    need(p, "plan");
    if (info) fill_plan(p->p, info);
    if (destinations)
      for (std::size_t i = 0; i < p->p.destinations.size(); ++i) destinations[i] = p->p.destinations[i];
    if (migrated)
      for (std::size_t i = 0; i < p->p.migrated.size(); ++i) migrated[i] = p->p.migrated[i];
  });
}

void fp_plan_free(fp_plan* p) { delete p; }

int fp_simulate_serial(const fp_gen_sample* batch, int32_t n, const fp_gen_config* cfg, fp_result** out) {
  return guarded([&] {
    need(out, "out");
    *out = new fp_result{fuseplan::simulate_serial(to_batch(batch, n), to_config(cfg))};
  });
}

int fp_simulate_fused(const fp_gen_sample* batch, int32_t n, const fp_gen_config* cfg, int32_t r_t,
                      fp_result** out) {
  return guarded([&] {
    need(out, "out");
    *out = new fp_result{fuseplan::simulate_fused(to_batch(batch, n), to_config(cfg), r_t)};
  });
}

int fp_result_info_get(const fp_result* r, fp_result_info* info) {
  return guarded([&] {
    need(r, "result");
    need(info, "info");
    info->gen_end = r->r.gen_end;
    info->inf_end = r->r.inf_end;
    info->total = r->r.total;
    info->triggered = r->r.triggered ? 1 : 0;
    info->n_samples = static_cast<int32_t>(r->r.finish_time.size());
    info->n_events = static_cast<int32_t>(r->r.events.size());
    fill_plan(r->r.plan, &info->plan);
  });
}

int fp_result_arrays(const fp_result* r, double* finish, fp_event* events, int32_t* destinations,
                     int32_t* migrated) {
  return guarded([&] {
    need(r, "result");
    const auto& g = r->r;
    if (finish)
      for (std::size_t i = 0; i < g.finish_time.size(); ++i) finish[i] = g.finish_time[i];
    if (events)
      for (std::size_t i = 0; i < g.events.size(); ++i)
        events[i] = {g.events[i].time, g.events[i].instance, kind_code(g.events[i].kind), g.events[i].sample};
    if (destinations)
      for (std::size_t i = 0; i < g.plan.destinations.size(); ++i) destinations[i] = g.plan.destinations[i];
    if (migrated)
      for (std::size_t i = 0; i < g.plan.migrated.size(); ++i) migrated[i] = g.plan.migrated[i];
  });
}

int fp_result_timeline(const fp_result* r, char* buf, size_t cap, size_t* len) {
  return guarded([&] {
    need(r, "result");
    const std::string text = fuseplan::timeline_text(r->r);
    if (len) *len = text.size();
    if (buf && cap > 0) {
      const size_t k = text.size() < cap - 1 ? text.size() : cap - 1;
      std::memcpy(buf, text.data(), k);
      buf[k] = '\0';
    }
  });
}

void fp_result_free(fp_result* r) { delete r; }

int fp_sweep_threshold(const fp_gen_sample* batch, int32_t n, const fp_gen_config* cfg, const double* ratios,
                       int32_t n_ratios, fp_sweep_point* curve, int32_t* n_curve, int32_t* best_index,
                       double* serial_total) {
  return guarded([&] {
    need(curve, "curve");
    std::vector<double> grid;
    if (n_ratios > 0) {
      need(ratios, "ratios");
      grid.assign(ratios, ratios + n_ratios);
    }
    const fuseplan::SweepResult s = fuseplan::sweep_threshold(to_batch(batch, n), to_config(cfg), grid);
    for (std::size_t i = 0; i < s.curve.size(); ++i) curve[i] = {s.curve[i].ratio, s.curve[i].r_t, s.curve[i].fused_total};
    if (n_curve) *n_curve = static_cast<int32_t>(s.curve.size());
    if (best_index) *best_index = s.best_index;
    if (serial_total) *serial_total = s.serial_total;
  });
}

#ifdef FUSEPLAN_B200_EXTENSIONS
int fp_fused_trigger(const fp_gen_sample* batch, int32_t n, const fp_gen_config* cfg, int32_t r_t,
                     int32_t* triggered, fp_plan_info* plan, fp_remaining* state, int32_t* n_state,
                     int32_t* move_sample, int32_t* move_from, int32_t* move_to, int32_t* n_moves) {
  return guarded([&] {
    const fuseplan::TriggerSnapshot t = fuseplan::fused_trigger(to_batch(batch, n), to_config(cfg), r_t);
    if (triggered) *triggered = t.triggered ? 1 : 0;
    if (plan) fill_plan(t.plan, plan);
    if (n_state) *n_state = static_cast<int32_t>(t.state.samples.size());
    if (state)
      for (std::size_t i = 0; i < t.state.samples.size(); ++i) {
        const auto& r = t.state.samples[i];
        state[i] = {r.id, r.instance, r.kv_bytes, r.generated, r.prompt_len, r.admitted ? 1 : 0};
      }
    if (n_moves) *n_moves = static_cast<int32_t>(t.move_sample.size());
    for (std::size_t i = 0; i < t.move_sample.size(); ++i) {
      if (move_sample) move_sample[i] = t.move_sample[i];
      if (move_from) move_from[i] = t.move_from[i];
      if (move_to) move_to[i] = t.move_to[i];
    }
  });
}
#endif

static int gae_common(bool matrix, const double* rewards, const double* values, int32_t T, double gamma,
                      double lam, double* adv_out) {
  return guarded([&] {
    need(adv_out, "adv_out");
    if (T < 0) throw std::invalid_argument("GaeInputs: need T >= 1 rewards and T+1 values");
    fuseplan::GaeInputs in;
    if (T > 0) {
      need(rewards, "rewards");
      need(values, "values");
      in.rewards.assign(rewards, rewards + T);
      in.values.assign(values, values + T + 1);
    }
    in.gamma = gamma;
    in.lam = lam;
    const std::vector<double> a = matrix ? fuseplan::gae_matrix(in) : fuseplan::gae_recursive(in);
    std::memcpy(adv_out, a.data(), a.size() * sizeof(double));
  });
}

int fp_balance_minibatch(const int32_t* lengths, int32_t n, int32_t dp, int32_t* group_of, int32_t* order,
                         int32_t* group_off) {
  return guarded([&] {
    if (n < 0) throw std::invalid_argument("balance_minibatch: n must be >= 0");
    if (n > 0) need(lengths, "lengths");
    const std::vector<int> len(lengths, lengths + n);
    const auto groups = fuseplan::balance_minibatch(len, dp);
    int k = 0;
    for (int g = 0; g < static_cast<int>(groups.size()); ++g) {
      if (group_off) group_off[g] = k;
      for (const int s : groups[g]) {
        if (group_of) group_of[s] = g;
        if (order) order[k] = s;
        ++k;
      }
    }
    if (group_off) group_off[groups.size()] = k;
  });
}

int fp_gae_recursive(const double* rewards, const double* values, int32_t T, double gamma, double lam,
                     double* adv_out) {
  return gae_common(false, rewards, values, T, gamma, lam, adv_out);
}

int fp_gae_matrix(const double* rewards, const double* values, int32_t T, double gamma, double lam,
                  double* adv_out) {
  return gae_common(true, rewards, values, T, gamma, lam, adv_out);
}

}  // extern "C"
