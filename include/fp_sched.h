/* fuseplan-b200 — C ABI of the gen+inf scheduler (decision clock).
 *
 * Plain C: pointers, sizes and POD structs; no C++ or torch types cross this
 * boundary, and no exceptions: every function returns a status
 *   FP_OK (0), FP_EINVAL (2: std::invalid_argument / ConfigError),
 *   FP_EINFEASIBLE (3: InfeasibleError), FP_EINTERNAL (4: anything else)
 * mirroring the reference CLI exit codes (proj/tools/fuseplan_main.cpp:32-35).
 * fp_last_error() returns the thread-local message of the last failure.
 *
 * Each entry point replaces one function of the reference's C++ API in
 * proj/include/fuseplan/genfuse.hpp / numerics.hpp (cited per function).
 * The same header is implemented twice: by the product library
 * (paper_2409_13221_b200/lib/libfuseplan_b200.so, over this repo's
 * include/fuseplan/) and by the oracle build of the reference sources
 * (oracle/_ref/libfuseplan_ref.so), which is what makes bit-exact parity
 * checks between the two a one-line comparison.
 */
#ifndef FP_SCHED_H_
#define FP_SCHED_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { FP_OK = 0, FP_EINVAL = 2, FP_EINFEASIBLE = 3, FP_EINTERNAL = 4 };

/* Event kinds, in the reference's tie-break order (genfuse.cpp:56-65). */
enum {
  FP_EV_ADMIT = 0, FP_EV_FINISH = 1, FP_EV_TRIGGER = 2, FP_EV_MIGRATE_OUT = 3,
  FP_EV_MIGRATE_IN = 4, FP_EV_JOIN_INFERENCE = 5, FP_EV_GEN_END = 6, FP_EV_INF_END = 7
};

/* ModelSpec (core.hpp:14-20). `name` must be non-empty. */
typedef struct fp_model_spec {
  const char* name;
  int32_t num_layers, num_heads, hidden_size, intermediate_size;
} fp_model_spec;

/* CostModel (core.hpp:31-44). */
typedef struct fp_cost_model {
  double time_per_token_coeff, backward_forward_ratio, activation_bytes_coeff;
  double decode_step_base, comm_bandwidth;
} fp_cost_model;

/* ClusterSpec (core.hpp:46-57). */
typedef struct fp_cluster_spec {
  int32_t num_gpus, gpus_per_node;
  double activation_capacity_per_stage, kv_capacity_per_instance;
  int32_t bs_max;
  double interconnect_bandwidth;
} fp_cluster_spec;

/* GenSimConfig (genfuse.hpp:45-57); tasks[i] is InferenceTask{task_names[i], tasks[i]}. */
typedef struct fp_gen_config {
  fp_model_spec actor;
  int32_t num_instances, instance_gpus;
  int32_t num_tasks;
  const fp_model_spec* tasks;
  const char* const* task_names;
  fp_cluster_spec cluster;
  fp_cost_model cost;
} fp_gen_config;

/* GenSample (genfuse.hpp:32-41). */
typedef struct fp_gen_sample {
  int32_t id, prompt_len, target_output_len, generated;
  double kv_bytes;
} fp_gen_sample;

/* LengthDistribution (genfuse.hpp:15-24); kind 0 lognormal, 1 empirical. */
typedef struct fp_length_dist {
  int32_t kind;
  double median, p999_ratio;
  int32_t max_len;
  const int32_t* empirical;
  int32_t n_empirical;
} fp_length_dist;

/* GenState::Remaining (genfuse.hpp:67-79). */
typedef struct fp_remaining {
  int32_t id, instance;
  double kv_bytes;
  int32_t generated, prompt_len, admitted;
} fp_remaining;

/* GenTimelineEvent (genfuse.hpp:59-64) with the kind as FP_EV_*. */
typedef struct fp_event {
  double time;
  int32_t instance, kind, sample;
} fp_event;

/* Scalar part of MigrationPlan (genfuse.hpp:83-92). */
typedef struct fp_plan_info {
  double trigger_time;
  int32_t r_t, m, mechanism, no_op;
  double overhead;
  int32_t n_destinations, n_migrated;
} fp_plan_info;

/* Scalar part of GenStageResult (genfuse.hpp:100-108). */
typedef struct fp_result_info {
  double gen_end, inf_end, total;
  int32_t triggered;
  int32_t n_samples, n_events;
  fp_plan_info plan;
} fp_result_info;

typedef struct fp_sweep_point { double ratio; int32_t r_t; double fused_total; } fp_sweep_point;

typedef struct fp_result fp_result; /* opaque GenStageResult */
typedef struct fp_plan fp_plan;     /* opaque MigrationPlan */

const char* fp_last_error(void);

/* sample_lengths (genfuse.hpp:29; genfuse.cpp:376-401). out[n]. */
int fp_sample_lengths(const fp_length_dist* dist, int32_t n, uint64_t seed, int32_t* out);
/* load_length_file (genfuse.hpp:26; genfuse.cpp:354-374). Writes min(count, cap). */
int fp_load_length_file(const char* path, int32_t* out, int32_t cap, int32_t* count);
/* make_batch (genfuse.hpp:43-44; genfuse.cpp:403-414). out[n]. */
int fp_make_batch(const fp_length_dist* dist, int32_t n, int32_t prompt_len,
                  const fp_model_spec* actor, uint64_t seed, fp_gen_sample* out);
/* kv_bytes_per_token (core.hpp:84; core.cpp:90-93). */
int fp_kv_bytes_per_token(const fp_model_spec* spec, double* out);

/* plan_migration (genfuse.hpp:94-98; genfuse.cpp:416-467). */
int fp_plan_migration(double time, const fp_remaining* samples, int32_t n, int32_t r_t,
                      const fp_gen_config* cfg, fp_plan** out);
int fp_plan_info_get(const fp_plan* p, fp_plan_info* info, int32_t* destinations,
                     int32_t* migrated);
void fp_plan_free(fp_plan* p);

/* simulate_serial / simulate_fused (genfuse.hpp:113, 120-121). */
int fp_simulate_serial(const fp_gen_sample* batch, int32_t n, const fp_gen_config* cfg,
                       fp_result** out);
int fp_simulate_fused(const fp_gen_sample* batch, int32_t n, const fp_gen_config* cfg,
                      int32_t r_t, fp_result** out);
int fp_result_info_get(const fp_result* r, fp_result_info* info);
/* Arrays sized by fp_result_info: finish[n_samples], events[n_events],
 * destinations[plan.n_destinations], migrated[plan.n_migrated]; any may be NULL. */
int fp_result_arrays(const fp_result* r, double* finish, fp_event* events,
                     int32_t* destinations, int32_t* migrated);
/* timeline_text (genfuse.hpp:141). Returns the byte length in *len (without
 * NUL); copies min(len, cap-1) bytes plus NUL when buf != NULL. */
int fp_result_timeline(const fp_result* r, char* buf, size_t cap, size_t* len);
void fp_result_free(fp_result* r);

/* sweep_threshold (genfuse.hpp:137-138; genfuse.cpp:517-534); n_ratios == 0
 * selects the default 5%..95% grid (curve must then hold 19 points). */
int fp_sweep_threshold(const fp_gen_sample* batch, int32_t n, const fp_gen_config* cfg,
                       const double* ratios, int32_t n_ratios, fp_sweep_point* curve,
                       int32_t* n_curve, int32_t* best_index, double* serial_total);

/* Extension (product library only; not in the reference API): the fused
 * trigger as the GPU executor takes it — trigger time, the GenState handed to
 * plan_migration (genfuse.cpp:492-495), the plan, and the samples
 * apply_migration (genfuse.cpp:136-208) moves, in application order. Pass
 * NULL arrays to query n_state / n_moves first. */
int fp_fused_trigger(const fp_gen_sample* batch, int32_t n, const fp_gen_config* cfg, int32_t r_t,
                     int32_t* triggered, fp_plan_info* plan, fp_remaining* state, int32_t* n_state,
                     int32_t* move_sample, int32_t* move_from, int32_t* move_to, int32_t* n_moves);

/* gae_recursive / gae_matrix (numerics.hpp:18-25). values has T+1 entries. */
/* balance_minibatch (workflow.hpp:63-66; workflow.cpp:160-182): LPT packing
 * of n sample lengths into dp groups. Outputs: group_of[n] (group of each
 * sample), order[n] (sample indices group-major, insertion order within a
 * group) and group_off[dp+1] (group g = order[group_off[g] .. group_off[g+1])).
 * FP_EINVAL for dp < 1 or n < dp. */
int fp_balance_minibatch(const int32_t* lengths, int32_t n, int32_t dp, int32_t* group_of, int32_t* order,
                         int32_t* group_off);

int fp_gae_recursive(const double* rewards, const double* values, int32_t T, double gamma,
                     double lam, double* adv_out);
int fp_gae_matrix(const double* rewards, const double* values, int32_t T, double gamma,
                  double lam, double* adv_out);

#ifdef __cplusplus
}
#endif
#endif /* FP_SCHED_H_ */
