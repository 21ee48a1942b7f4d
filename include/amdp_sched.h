/*
 * amdp_sched.h — C-ABI over the ppsim-compatible schedule library (include/ppsim/ppsim.hpp).
 *
 * What a non-C++ host (the Python mirror paper_2605_29664_b200/ppsim.py, or a ctypes /
 * cffi binding) binds to reach the reference API without C++ types:
 *   ppsim::build            (builder.hpp:145)    -> amdp_schedule_build
 *   ppsim::simulate         (engine.hpp:28)      -> amdp_schedule_simulate
 *   ppsim::bubble_ratio     (engine.hpp:166)     -> amdp_schedule_bubble
 *   ppsim::mismatch_report / window_mismatch / memory_report / validate_causality /
 *   validate_non_overlap    (analysis.hpp:28,126,226; validate.hpp:118,164)
 *                                                -> amdp_schedule_report_json
 *   ppsim::timeline_csv     (serialize.hpp:41)   -> amdp_schedule_text(.., AMDP_TEXT_TIMELINE_CSV)
 *   ppsim::validate_cluster / validate_policy (validate.hpp:12,49) -> amdp_validate
 *   map_stage_to_device / default_num_pipelines / preload_count (builder.hpp:81-104)
 * Errors: functions returning int give 0 on success, AMDP_SCHED_EINVAL for what the
 * reference throws std::invalid_argument for, AMDP_SCHED_ERUNTIME for runtime_error
 * (dependency cycle / deadlock), AMDP_SCHED_EARITH for overflow/domain errors; the
 * exception text is copied into `err` (NUL-terminated, truncated to errlen).
 */
#ifndef AMDP_SCHED_H_
#define AMDP_SCHED_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#pragma GCC visibility push(default)

#define AMDP_SCHED_EINVAL (-1)
#define AMDP_SCHED_ERUNTIME (-2)
#define AMDP_SCHED_EARITH (-3)
#define AMDP_SCHED_ESTATE (-4)

typedef struct amdp_rat {
  int64_t num, den;
} amdp_rat;

/* Policy ids follow ppsim::Policy: 0 AMDP, 1 DAPPLE, 2 GPipe, 3 Interleaved1F1B,
 * 4 Chimera, 5 PipeDreamAsync.  Kind ids follow ppsim::Kind: 0 Forward, 1 Backward,
 * 2 Reduce, 3 Broadcast, 4 Update. */
typedef struct amdp_cluster_spec {
  int depth, devices;
  const amdp_rat* fwd_cost; /* n_fwd entries (normally depth) */
  int n_fwd;
  const amdp_rat* bwd_cost;
  int n_bwd;
  amdp_rat update_cost, comm_cost;
  int num_nodes;           /* 0 = one node */
  const int* node_sizes;   /* num_nodes entries */
  const int* node_devices; /* concatenated node members */
  int has_inter_node_cost;
  amdp_rat inter_node_cost;
} amdp_cluster_spec;

typedef struct amdp_policy_config {
  int policy, injection_limit, num_pipelines, accumulation_threshold, num_minibatches;
  int zero_enabled, injection_override;
} amdp_policy_config;

typedef struct amdp_task_info {
  int kind, stage, minibatch, pipeline, device, window, preloaded;
  amdp_rat duration;
} amdp_task_info;

typedef struct amdp_event {
  int kind, stage, minibatch, pipeline, device, window, preloaded;
  amdp_rat start, duration;
} amdp_event;

typedef struct amdp_schedule amdp_schedule; /* TaskGraph + declared cluster + Timeline */

/* validate_cluster + validate_policy: returns the number of violations; messages are
 * written '\n'-separated into buf.  The _cluster/_policy variants run one rule set. */
int amdp_validate(const amdp_policy_config* cfg, const amdp_cluster_spec* cl, char* buf,
                  size_t len);
int amdp_validate_cluster(const amdp_cluster_spec* cl, char* buf, size_t len);
int amdp_validate_policy(const amdp_policy_config* cfg, const amdp_cluster_spec* cl, char* buf,
                         size_t len);

int amdp_map_stage_to_device(int pipeline, int stage, int depth, int* out, char* err,
                             size_t errlen);
int amdp_default_num_pipelines(int depth, int* out, char* err, size_t errlen);
int amdp_preload_count(amdp_rat bwd, amdp_rat fwd, int* out, char* err, size_t errlen);

/* build(): NULL on error (text in err). */
amdp_schedule* amdp_schedule_build(const amdp_policy_config* cfg, const amdp_cluster_spec* cl,
                                   char* err, size_t errlen);
/* A hand-assembled TaskGraph (the reference's tests build these directly). */
amdp_schedule* amdp_graph_new(int policy, int depth, int devices, int threshold,
                              const amdp_cluster_spec* cl);
int amdp_graph_add_task(amdp_schedule* s, const amdp_task_info* t); /* returns task id */
int amdp_graph_add_dep(amdp_schedule* s, int pred, int succ);
int amdp_graph_add_lane(amdp_schedule* s, const int* ids, int n);
/* A bare Timeline (e.g. measured on the GPU) for the analysis calls. */
amdp_schedule* amdp_timeline_new(int policy, int depth, int devices, int threshold,
                                 const amdp_event* events, int n, const amdp_cluster_spec* cl);
amdp_schedule* amdp_schedule_clone(const amdp_schedule* s);
void amdp_schedule_free(amdp_schedule* s);

int amdp_schedule_simulate(amdp_schedule* s, char* err, size_t errlen);
int amdp_schedule_num_tasks(const amdp_schedule* s);
int amdp_schedule_tasks(const amdp_schedule* s, amdp_task_info* out, int cap);
int amdp_schedule_num_deps(const amdp_schedule* s);
int amdp_schedule_deps(const amdp_schedule* s, int* out_pairs, int cap);
/* global dispatch order (task ids), a topological order of the DAG */
int amdp_schedule_order(const amdp_schedule* s, int* out, int cap);
int amdp_schedule_num_events(const amdp_schedule* s);
/* events device-major, each device in execution order */
int amdp_schedule_events(const amdp_schedule* s, amdp_event* out, int cap);
int amdp_schedule_makespan(const amdp_schedule* s, amdp_rat* out);
int amdp_schedule_bubble(const amdp_schedule* s, int warmup, amdp_rat* out, char* err,
                         size_t errlen);

enum amdp_text_kind {
  AMDP_TEXT_TIMELINE_CSV = 0,
  AMDP_TEXT_VERSION_CSV = 1,
  AMDP_TEXT_TIMELINE_JSON = 2
};
/* Returns the full text length; copies min(len-1, length) bytes + NUL into buf. */
size_t amdp_schedule_text(const amdp_schedule* s, int which, char* buf, size_t len);
/* summary.json-style report: makespan, bubble (warmup), mismatch entries / per-stage max /
 * missing, window report, memory report (unit model), causality/overlap issue lists. */
size_t amdp_schedule_report_json(const amdp_schedule* s, const amdp_policy_config* cfg,
                                 int warmup, char* buf, size_t len);

#pragma GCC visibility pop
#ifdef __cplusplus
}
#endif

#endif /* AMDP_SCHED_H_ */
