/*
 * amdp_engine.h — C-ABI of the AMDP stage executor on B200s.
 *
 * This is `simulate()` (ppsim engine.hpp:28) made real: the same TaskGraph
 * (builder.hpp:145, under a declared ClusterSpec) is executed on GPUs, and the result
 * comes back as the same Timeline type with measured times.  One engine per process /
 * GPU; logical devices (AMDP requires devices == depth, validate.hpp:62) are folded
 * onto world_size GPUs, depth/world_size per GPU.
 *
 * Per task (dispatch order of the declared simulation, a topological order):
 *   Forward(i,j)   -> GPT stage i forward on minibatch j (embedding on stage 0,
 *                     final LayerNorm + LM head + cross-entropy on stage depth-1)
 *   Backward(i,j)  -> stage i backward; weight gradients accumulate (fp32) into the
 *                     stage's window gradient buffer
 *   Reduce(w,i)    -> replica gradient sum to the stage owner (NCCL reduce on the
 *                     stage's replica group; no-op when all replicas share one GPU)
 *   Broadcast(w,i) -> fused optimizer step on the owner + weight broadcast
 * Cross-GPU stage boundaries move activations / activation-gradients with NCCL
 * send/recv on a communication stream; same-GPU boundaries are device copies.
 */
#ifndef AMDP_ENGINE_H_
#define AMDP_ENGINE_H_

#include <stddef.h>
#include <stdint.h>

#include "amdp_kernels.h"
#include "amdp_sched.h"

#ifdef __cplusplus
extern "C" {
#endif
#pragma GCC visibility push(default)

typedef struct amdp_model_config {
  int layers, hidden, heads, ffn, vocab, seq;
  int seqs_per_minibatch; /* tokens per minibatch = seqs_per_minibatch * seq */
  int causal;             /* 1 = GPT (causal LM), 0 = bidirectional */
  float init_std;         /* N(0, init_std); residual projections scaled by 1/sqrt(2L) */
  float ln_eps;
  uint64_t seed;
  /* stage partition: layers_per_stage[depth] (NULL = balanced automatically) */
  const int* layers_per_stage;
  /* 1 = keep neither f = gelu(u) nor the attention output o per minibatch: the backward
   * recomputes both from u / qkv (weight-independent, so exact under AMDP's staleness);
   * activation slots shrink by 5/16 (the rebuilt o / f live in the shared workspace). */
  int recompute;
  /* 1 = fp32 validation mode: activations, weights and every product in fp32 on the CUDA
   * cores (amdp_f32_* kernels) instead of the bf16 tcgen05 path, so that losses / weights
   * match the fp64 CPU oracle at a tolerance far below bf16's (north_star).  Slow; for
   * correctness runs, not throughput. */
  int fp32_validation;
  /* bidirectional (BERT) models: token id > 0 that marks padding (0 = no padding).  Each
   * sequence's valid length is the position of its first pad token; attention gives padded
   * keys no weight (their labels must be -1).  amdp_synthetic_tokens pads such models to a
   * length drawn in [seq / 2, seq]. */
  int pad_token;
} amdp_model_config;

typedef struct amdp_run_config {
  amdp_policy_config policy;   /* AMDP: injection 2, pipelines depth/2, zero on  */
  amdp_rat declared_fwd;       /* declared per-stage costs the order is built on */
  amdp_rat declared_bwd;
  amdp_opt_args optimizer;
  int world_size, rank;        /* GPUs in the job and this process's rank        */
  int record_events;           /* 1 = per-task CUDA events (measured Timeline)   */
  uint64_t data_seed;
  int plan_only;               /* 1 = plan (hosting/slots/comm program) without  */
                               /*     touching CUDA or NCCL; see plan_json       */
  int depth;                   /* stages = devices; 0 = 2 x num_pipelines (AMDP).  */
                               /* Policies: AMDP (ZeRO on), or DAPPLE / GPipe with */
                               /* one pipeline and per-window Update tasks         */
  int comm_backend;            /* world_size > 1: AMDP_COMM_IPC (default, this     */
                               /* library's peer-memory data plane; also several   */
                               /* ranks on one GPU) or AMDP_COMM_NCCL              */
} amdp_run_config;

#define AMDP_COMM_IPC 0
#define AMDP_COMM_NCCL 1

typedef struct amdp_engine amdp_engine;

/* NCCL unique id for world_size > 1 (rank 0 creates; the host broadcasts 128 bytes). */
int amdp_nccl_unique_id(uint8_t out[128]);

/* Creates the engine on the current CUDA device: builds + orders the schedule, plans
 * stage hosting / activation slots / communication, allocates and initialises weights.
 * nccl_id may be NULL when world_size == 1.  Returns NULL on error (text in err). */
amdp_engine* amdp_engine_create(const amdp_model_config* model, const amdp_run_config* run,
                                const uint8_t* nccl_id, char* err, size_t errlen);
void amdp_engine_destroy(amdp_engine* e);

/* world_size > 1 with AMDP_COMM_IPC: after every rank created its engine, each exports a
 * descriptor of the memory its peers may map (IPC handles of the boundary arena, of the
 * per-stage gradient / weight buffers and of its flag array, plus its send table); the host
 * all-gathers them (any transport: torch.distributed, MPI, files) and passes all world_size
 * descriptors, in rank order, to amdp_engine_comm_connect.  Export returns the descriptor
 * size (copies at most len bytes into buf; call with buf = NULL to size it).  No-ops for
 * world_size 1 and for NCCL.                                                        */
size_t amdp_engine_comm_export(amdp_engine* e, uint8_t* buf, size_t len);
int amdp_engine_comm_connect(amdp_engine* e, const uint8_t* const* blobs, const size_t* lens,
                             int count, char* err, size_t errlen);

/* Pinned host memory for the token streams (host -> device copies overlap compute). */
void* amdp_host_alloc(size_t bytes);
void amdp_host_free(void* p);

/* Deterministic synthetic data: inputs/labels [num_minibatches][tokens_per_minibatch]
 * (arithmetic-progression token streams, splitmix64-keyed; oracle/gpt_oracle.py restates). */
int amdp_synthetic_tokens(const amdp_model_config* model, uint64_t data_seed,
                          int first_minibatch, int num_minibatches, int32_t* inputs,
                          int32_t* labels);

/* Executes the whole schedule (policy.num_minibatches minibatches = windows * threshold)
 * once.  inputs/labels are HOST arrays [num_minibatches][tokens] (pinned for overlap);
 * each window's tokens are copied to the device when its first entry forward issues.
 * losses_out (host, [num_minibatches], may be NULL) receives the per-minibatch mean loss
 * (valid on the rank hosting the last stage).  Returns when the device work is done. */
int amdp_engine_run(amdp_engine* e, const int32_t* inputs, const int32_t* labels,
                    float* losses_out, char* err, size_t errlen);
/* Runs the tasks of windows [0, num_windows) of the schedule in dispatch order (a window
 * prefix: the pipeline starts empty and drains at the end; the next window's preloaded
 * forwards are not run).  resident != 0: the token arrays were already copied to the
 * device by amdp_engine_stage_tokens and no host->device copy happens inside the run. */
int amdp_engine_run_windows(amdp_engine* e, int num_windows, const int32_t* inputs,
                            const int32_t* labels, float* losses_out, int resident,
                            char* err, size_t errlen);
/* Copies all token arrays to the device now (synchronously). */
int amdp_engine_stage_tokens(amdp_engine* e, const int32_t* inputs, const int32_t* labels);

/* Per-kernel-class CUDA-event timing inside runs (adds two events per launch). */
typedef struct amdp_kernel_class_stats {
  char name[24];
  int64_t launches;
  double total_ms;
  double flops; /* algorithmic (tensor-pipe work) */
  double bytes; /* algorithmic HBM bytes (memory-bound classes) */
} amdp_kernel_class_stats;
int amdp_engine_set_kernel_timing(amdp_engine* e, int enable);
/* CUDA graphs of whole runs (default on; one GPU only): a configuration's second run is
 * captured and later runs replay it.  Host buffers must be pinned (amdp_host_alloc) or the
 * run resident; otherwise, and with kernel timing on, runs are issued eagerly. */
int amdp_engine_set_graphs(amdp_engine* e, int enable);
/* Concurrent compute streams (one GPU, ZeRO AMDP; one per logical device by default, capped by
 * free HBM): use the first n of them (1 = the serial executor, e.g. for isolated per-task
 * times).  Returns the number in use. */
int amdp_engine_set_streams(amdp_engine* e, int n);
int amdp_engine_kernel_stats(const amdp_engine* e, amdp_kernel_class_stats* out, int cap);

/* Stats of the last run: device-timed milliseconds from the first task to the last,
 * tasks / kernels launched by this rank, bytes copied H2D / D2H. */
typedef struct amdp_run_stats {
  double device_ms;
  int64_t tasks_executed;
  int64_t kernels_launched;
  int64_t h2d_bytes, d2h_bytes;
  int64_t p2p_bytes_sent, collective_bytes;
  double busy_ms; /* sum of measured task durations on this GPU (record_events) */
  double host_issue_ms; /* host wall time spent issuing the run (launches, events, NCCL) */
  int64_t graph_replayed; /* 1: the run was one CUDA-graph launch (captured run, replayed) */
} amdp_run_stats;
int amdp_engine_stats(const amdp_engine* e, amdp_run_stats* out);

/* Measured Timeline of the last run (record_events = 1): ppsim events, times in ns,
 * logical devices hosted by this rank only.  Pass to amdp_timeline_new for analyses. */
int amdp_engine_num_events(const amdp_engine* e);
int amdp_engine_events(const amdp_engine* e, amdp_event* out, int cap);
/* The window machinery's own intervals: ZeRO Reduce (collective stream) and Broadcast
 * (optimizer step + weight broadcast on the update stream) run beside the compute stream;
 * the Timeline above shows each where the compute stream passed it (the reference's
 * one-task-per-device model, so its validators apply), these events their real extent. */
int amdp_engine_num_lane_events(const amdp_engine* e);
int amdp_engine_lane_events(const amdp_engine* e, amdp_event* out, int cap);
/* Parameter version each Forward/Backward actually read on the GPU (device-side
 * counter per stage, bumped by the optimizer step), as version_trace_csv text. */
size_t amdp_engine_version_trace(const amdp_engine* e, char* buf, size_t len);
/* The declared (reference-order) timeline the engine replays. */
amdp_schedule* amdp_engine_schedule(const amdp_engine* e);

/* Parameters of one stage (flat, see amdp_engine_param_layout) copied to host (fp32 master,
 * only valid on the stage's owner rank), for parity checks. */
int64_t amdp_engine_stage_numel(const amdp_engine* e, int stage);
int amdp_engine_get_stage_params(const amdp_engine* e, int stage, float* out, int64_t n);
int amdp_engine_set_stage_params(amdp_engine* e, int stage, const float* in, int64_t n);
/* JSON: per stage, the list of {name, offset, rows, cols} in the flat buffer, plus the
 * memory plan (activation slots per stage, bytes). */
size_t amdp_engine_plan_json(const amdp_engine* e, char* buf, size_t len);

#pragma GCC visibility pop
#ifdef __cplusplus
}
#endif

#endif /* AMDP_ENGINE_H_ */
