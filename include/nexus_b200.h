/*
 * nexus_b200.h — C-ABI boundary of the B200-native Nexus intra-GPU
 * prefill/decode executor.
 *
 * The reference (`/root/reference/proj`, "nexussim") exposes its path as a C++
 * library API in `proj/core/include/nexussim/` headers. Every entry point below
 * replaces one of those interfaces; the citation on each line names the one
 * it stands in for. Conventions:
 *   - plain C, POD structs, plain pointers + sizes; no C++ or torch types;
 *   - every function returns an `int` status (NX_OK == 0) unless it is a pure
 *     scalar query; nothing throws across the ABI (the reference throws
 *     std::invalid_argument / std::runtime_error, e.g. costmodel.cpp:10-11,
 *     simulator.cpp:61-93 — those become NX_EINVAL / NX_ERUNTIME plus a
 *     message readable through nx_last_error());
 *   - the caller owns input arrays and allocates output arrays; an engine
 *     owns its weights, KV cache, streams and green contexts;
 *   - one engine per host thread, not re-entrant.
 */
#ifndef NEXUS_B200_H
#define NEXUS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes -------------------------------------------------------- */
#define NX_OK 0
#define NX_EINVAL 1    /* precondition violated (reference: std::invalid_argument) */
#define NX_ERUNTIME 2  /* I/O, parse or CUDA error (reference: std::runtime_error) */
#define NX_ENOMEM 3    /* device / pool allocation failed */
#define NX_EAGAIN 4    /* nothing to do yet (device clock: event not ready) */
#define NX_EDONE 5     /* engine drained: no pending event remains */
#define NX_ENODEV 6    /* CUDA path requested but no usable sm_100 device */

/* Thread-local message of the last failing call (empty string if none). */
const char* nx_last_error(void);
/* Version / build identification, e.g. "nexus_b200 0.1 sm_100a". */
const char* nx_version(void);
/* sizeof(nx_sim_config) as compiled: FFI mirrors check their struct layout against it. */
size_t nx_sim_config_size(void);

/* ---- domain types (reference: domain.hpp:14-103) ------------------------- */

/* ModelConfig (domain.hpp:14-34). Cost-model/ledger view of the model:
 * kv_bytes_per_token = 2*L*d*elem exactly (domain.cpp:54-58). */
typedef struct nx_model_config {
  int64_t hidden_dim;
  int64_t ffn_dim;
  int32_t num_layers;
  int32_t num_heads;
  int32_t element_bytes;
  int32_t _pad0;
  int64_t kv_bytes_per_token;
  int64_t weight_bytes_per_layer_dense;
  int64_t weight_bytes_per_layer_attn;
} nx_model_config;

/* GpuSpec (domain.hpp:36-41). */
typedef struct nx_gpu_spec {
  int32_t total_sm;
  int32_t _pad0;
  double peak_compute;   /* FLOP/s */
  double peak_bandwidth; /* B/s */
  int64_t kv_capacity_bytes;
} nx_gpu_spec;

/* SaturationCurve / KernelProfile (domain.hpp:45-56). */
typedef struct nx_saturation_curve {
  double r_sat;
  double lambda;
} nx_saturation_curve;

typedef struct nx_kernel_profile {
  nx_saturation_curve qkv_proj;
  nx_saturation_curve attn_prefill;
  nx_saturation_curve attn_decode;
  nx_saturation_curve attn_out_proj;
  nx_saturation_curve ffn;
} nx_kernel_profile;

/* ControllerConfig (domain.hpp:80-89). */
typedef struct nx_controller_config {
  double alpha;
  double beta;
  double kv_switch_fraction;
  double gamma;
  int32_t delta_pp;
  int32_t max_decode_batch;
  int64_t chunk_size;
  int64_t token_budget;
} nx_controller_config;

/* PartitionState (domain.hpp:74-78). */
typedef struct nx_partition_state {
  int32_t r_p;
  int32_t r_d;
  int32_t last_applied_r_p;
} nx_partition_state;

/* EngineKind (simulator.hpp:30) — EngineLevelDisagg is out of scope. */
#define NX_ENGINE_NEXUS 0
#define NX_ENGINE_MONOLITHIC 1
#define NX_ENGINE_STATIC 2
/* PrefillPolicy (simulator.hpp:31) */
#define NX_PREFILL_SPF 0
#define NX_PREFILL_FCFS 1
/* Clock modes of the step executor (new). */
#define NX_CLOCK_VIRTUAL 0 /* batch latency = cost model (reference semantics) */
#define NX_CLOCK_DEVICE 1  /* batch latency = measured on the B200 partitions */
#define NX_CLOCK_REPLAY 2  /* batch latency = caller-supplied list, in launch order */

/* EngineConfig (simulator.hpp:33-43) + executor selection. */
typedef struct nx_engine_config {
  int32_t kind;
  int32_t static_r_p;
  int32_t prefill_policy;
  int32_t clock_mode;
  double timeout_sim_s;
  uint64_t max_events;
} nx_engine_config;

/* Cost-model extension (new, off by default => reference-exact): the HBM
 * bandwidth an operator can draw grows with its SM share until bw_sat,
 *   mem_s = bytes / (B * min(1, share / bw_sat[kind])),
 * because on B200 one SM streams only ~1/90 of peak HBM bandwidth. The
 * reference's memory time ignores the share (costmodel.cpp:33), which makes
 * its controller starve decode of SMs. */
typedef struct nx_cost_ext {
  int32_t enabled;
  int32_t contention; /* 1: co-located decode = isolated x (c0 + c1 p + c2 p^2), p = prefill share */
  double bw_sat[5]; /* per operator kind, in (0, 1] */
  /* Measured co-location slowdown of a decode batch beside a prefill batch
   * (paper_2507_06608_b200.calibrate), replacing the B_decode bandwidth split
   * (costmodel.cpp:56-64) when `contention` is set: on B200 the shared power
   * / clock budget, not HBM bandwidth, dominates the slowdown. */
  double contention_c[3];
  /* > 0: decode-step target (seconds) of Algorithm 1's prefill-priority mode
   * (optimizer.cpp:22-61). A prefill share also fits when the decode batch's
   * co-located step (isolated x the contention factor above when
   * `contention` is set) stays within this target, so prefill takes every SM
   * the decode lane does not need to hold its step time; the reference rule
   * (decode <= beta x T_decode(100%)) stays the floor. 0 = reference. */
  double decode_target_s;
} nx_cost_ext;

/* SimConfig (simulator.hpp:45-51) + the cost-model extension. */
typedef struct nx_sim_config {
  nx_model_config model;
  nx_gpu_spec gpu;
  nx_controller_config ctrl;
  nx_kernel_profile profile;
  nx_engine_config engine;
  nx_cost_ext ext;
} nx_sim_config;

/* Request (domain.hpp:58-72), trace view. */
typedef struct nx_request {
  uint64_t id;
  double arrival_s;
  int64_t prompt_len;
  int64_t output_len;
} nx_request;

/* ModelConfig::derive (domain.cpp:7-24). */
nx_model_config nx_model_derive(int64_t hidden_dim, int64_t ffn_dim, int32_t num_layers,
                                int32_t num_heads, int32_t element_bytes);
/* Defaults: ControllerConfig{} (domain.hpp:80-89), KernelProfile{} (domain.hpp:50-56),
 * EngineConfig{} (simulator.hpp:33-43), PartitionState{} (domain.hpp:74-78). */
nx_controller_config nx_controller_config_default(void);
nx_kernel_profile nx_kernel_profile_default(void);
nx_engine_config nx_engine_config_default(void);
/* validate_config + describe (domain.cpp:42-95). Returns the number of
 * violations; writes "field: reason; ..." into msg (truncated to msg_cap). */
int nx_validate_config(const nx_model_config* model, const nx_gpu_spec* gpu,
                       const nx_controller_config* ctrl, const nx_kernel_profile* prof,
                       char* msg, size_t msg_cap);

/* ---- operator model (reference: opcost.hpp:22-66) ------------------------ */
#define NX_OP_QKV_PROJ 0
#define NX_OP_ATTN_PREFILL 1
#define NX_OP_ATTN_DECODE 2
#define NX_OP_ATTN_OUT_PROJ 3
#define NX_OP_FFN 4

typedef struct nx_op_workload {
  int32_t kind;
  int32_t is_attention;
  double flops;
  double mem_bytes;
  double kv_bytes;
} nx_op_workload;

#define NX_MAX_OPS 8

/* prefill_batch_workloads (opcost.cpp:99-126): chunk i has chunk_tokens[i]
 * new tokens attending context_len[i]. Writes 4 ops. */
int nx_prefill_batch_workloads(const nx_model_config* model, const int64_t* chunk_tokens,
                               const int64_t* context_len, size_t n_chunks,
                               nx_op_workload* out_ops, size_t* n_ops);
/* decode_op_workloads (opcost.cpp:128-148). Writes 4 ops. */
int nx_decode_op_workloads(const nx_model_config* model, const int64_t* context_lens,
                           size_t n, nx_op_workload* out_ops, size_t* n_ops);
/* mixed_batch_workloads (opcost.cpp:150-189). Writes 4 or 5 ops. */
int nx_mixed_batch_workloads(const nx_model_config* model, const int64_t* chunk_tokens,
                             const int64_t* context_len, size_t n_chunks,
                             const int64_t* decode_context_lens, size_t n_decode,
                             nx_op_workload* out_ops, size_t* n_ops);

/* ---- cost model (reference: costmodel.hpp:19-80) ------------------------- */
typedef struct nx_op_latency {
  int32_t kind;
  int32_t memory_bound;
  double compute_s;
  double mem_s;
} nx_op_latency;

typedef struct nx_breakdown {
  double total_s;
  double attn_mem_time_s;
  int32_t n_ops;
  int32_t _pad0;
  nx_op_latency per_op[NX_MAX_OPS];
} nx_breakdown;

/* compute_latency, Eq. 5 (costmodel.cpp:8-14). Returns NX_EINVAL for share <= 0. */
int nx_compute_latency(double flops, double share, nx_saturation_curve curve,
                       double peak_compute, double* out_s);
/* Installs a cost-model extension for the nx_phase_latency_isolated /
 * nx_decode_latency_contended calls of this thread (NULL = reference model). */
int nx_set_cost_ext(const nx_cost_ext* ext);
/* phase_latency_isolated (costmodel.cpp:43-49). */
int nx_phase_latency_isolated(const nx_op_workload* ops, size_t n_ops, double share,
                              const nx_gpu_spec* gpu, const nx_kernel_profile* prof,
                              nx_breakdown* out);
/* effective_decode_bandwidth (costmodel.cpp:56-64). */
int nx_effective_decode_bandwidth(double p_attn, double m_d, double m_p1, double m_p2,
                                  double peak_bandwidth, double* out_bps);
/* decode_latency_contended (costmodel.cpp:85-96). prefill may be NULL (isolated). */
int nx_decode_latency_contended(const nx_op_workload* decode_ops, size_t n_decode,
                                double share, const nx_breakdown* prefill_bd,
                                const nx_op_workload* prefill_ops, size_t n_prefill,
                                const nx_gpu_spec* gpu, const nx_kernel_profile* prof,
                                nx_breakdown* out);
/* min_phase_latency (costmodel.cpp:98-102); n_ops == 0 -> 0. */
double nx_min_phase_latency(const nx_op_workload* ops, size_t n_ops, const nx_gpu_spec* gpu,
                            const nx_kernel_profile* prof);

/* ---- controller (reference: optimizer.hpp:14-77) ------------------------- */
#define NX_MODE_PREFILL 0 /* ObjectiveMode::PrefillPrioritized */
#define NX_MODE_DECODE 1  /* ObjectiveMode::DecodePrioritized */
#define NX_PHASE_PREFILL 0
#define NX_PHASE_DECODE 1

/* PhaseModel (optimizer.hpp:23-26): std::function becomes fn-ptr + user. */
typedef struct nx_phase_model {
  int32_t active;
  double (*latency_at)(void* user, int32_t share_pct);
  void* user;
} nx_phase_model;

typedef struct nx_adjust_outcome {
  int32_t r_p;
  int32_t r_d;
  int32_t infeasible;
  int32_t queries;
} nx_adjust_outcome;

typedef struct nx_decision {
  int32_t r_p;
  int32_t r_d;
  int32_t mode;
  int32_t switched;
  int32_t infeasible;
  int32_t candidate_r_p;
  int32_t iterations_searched;
  int32_t _pad0;
} nx_decision;

/* select_mode (optimizer.cpp:13-20). Returns NX_MODE_* or -1 on invalid input. */
int nx_select_mode(int64_t kv_used, int64_t kv_capacity, double kv_switch_fraction);
/* adjust_partition, Algorithm 1 (optimizer.cpp:22-61). */
int nx_adjust_partition(int32_t target_phase, const nx_partition_state* cur,
                        const nx_phase_model* prefill, const nx_phase_model* decode,
                        const nx_controller_config* cfg, nx_adjust_outcome* out);
/* PartitionController (optimizer.hpp:60-77). */
typedef struct nx_controller nx_controller;
int nx_controller_create(const nx_partition_state* initial, const nx_controller_config* cfg,
                         nx_controller** out);
void nx_controller_destroy(nx_controller* c);
int nx_controller_decide(nx_controller* c, int64_t kv_used, int64_t kv_capacity,
                         const nx_phase_model* prefill, const nx_phase_model* decode,
                         nx_decision* out);
int nx_controller_state(const nx_controller* c, nx_partition_state* out);

/* ---- schedulers (reference: schedulers.hpp:12-59) ------------------------ */
typedef struct nx_prefill_entry {
  uint64_t id;
  int64_t remaining;
  double arrival_s;
} nx_prefill_entry;

typedef struct nx_decode_candidate {
  uint64_t id;
  double arrival_s;
} nx_decode_candidate;

typedef struct nx_batch_member {
  uint64_t id;
  int64_t tokens;
} nx_batch_member;

/* All schedulers write at most `cap` members and the total token count. */
int nx_spf_schedule(const nx_prefill_entry* queue, size_t n, int64_t token_budget,
                    double gamma, double now_s, int32_t skip_non_fitting,
                    nx_batch_member* out, size_t cap, size_t* n_out, int64_t* total_tokens);
int nx_fcfs_prefill_schedule(const nx_prefill_entry* queue, size_t n, int64_t token_budget,
                             nx_batch_member* out, size_t cap, size_t* n_out,
                             int64_t* total_tokens);
int nx_fcfs_decode_schedule(const nx_decode_candidate* active, size_t n, int32_t max_batch,
                            nx_batch_member* out, size_t cap, size_t* n_out,
                            int64_t* total_tokens);
int nx_chunked_mixed_schedule(const nx_prefill_entry* queue, size_t n_queue,
                              const nx_decode_candidate* decodes, size_t n_decodes,
                              int64_t token_budget, int32_t max_batch, int64_t chunk_size,
                              nx_batch_member* out, size_t cap, size_t* n_out,
                              int64_t* total_tokens);

/* ---- traces (reference: workload.hpp:20-81, presets.hpp:28-43) ----------- */
/* generate_trace/mix_traces via workload_preset + realize (presets.cpp:70-105).
 * preset: "long-data" | "arxiv" | "sharegpt" | "mixed" (reference) or, new,
 * "longbench" (uniform 4096..16384-token prompts, ShareGPT outputs) and
 * "bursty" ("mixed" lengths, Gamma inter-arrivals with CV 4). Writes min(count, cap). */
int nx_workload_preset_trace(const char* preset, double rate_rps, int64_t count, uint64_t seed,
                             nx_request* out, size_t cap, size_t* n_out);
/* Trace file text "# nexustrace v1" (workload.cpp:200-243). */
int nx_trace_to_text(const nx_request* trace, size_t n, char* buf, size_t cap, size_t* len);
int nx_trace_from_text(const char* text, nx_request* out, size_t cap, size_t* n_out);

/* Calibration file text "<op> <r_sat> <lambda>" (presets.cpp:109-170). */
int nx_kernel_profile_to_text(const nx_kernel_profile* prof, char* buf, size_t cap, size_t* len);
int nx_kernel_profile_from_text(const char* text, nx_kernel_profile* out, char* warnings,
                                size_t warn_cap);

/* ---- step executor (reference: simulator.hpp:53-80, simulator.cpp:142-501) */

/* Event log lanes / kinds (eventlog.hpp:20-21). */
#define NX_LANE_NONE 0
#define NX_LANE_PREFILL 1
#define NX_LANE_DECODE 2
#define NX_LANE_MIXED 3
#define NX_EV_ARRIVAL 0
#define NX_EV_LAUNCH 1
#define NX_EV_COMPLETE 2
#define NX_EV_FINISH 3
#define NX_EV_TIMEOUT 4

typedef struct nx_engine nx_engine;

/* Creates a host engine (scheduler, controller, KV ledger + block manager).
 * With clock_mode NX_CLOCK_DEVICE the engine must be bound to a device
 * executor (nx_engine_bind_device) before the first step. */
int nx_engine_create(const nx_sim_config* cfg, nx_engine** out);
void nx_engine_destroy(nx_engine* eng);
const char* nx_engine_last_error(const nx_engine* eng);

/* An arrival (simulator.cpp:171-175). Requests must be submitted in
 * non-decreasing arrival order with unique ids (simulator.cpp:72-93). */
int nx_submit(nx_engine* eng, const nx_request* req);
/* Submits a whole trace (same checks as the SimBase constructor). */
int nx_submit_trace(nx_engine* eng, const nx_request* reqs, size_t n);

/* One loop iteration of IntraGpuSim::run (simulator.cpp:152-177): launch
 * idle lanes, then retire exactly one event in the reference tie order.
 * Returns NX_OK, NX_EDONE when drained, or NX_EAGAIN (device clock) when
 * no event is due yet. */
int nx_step(nx_engine* eng);
/* Steps until drained or timeout (the run() equivalent, simulator.cpp:760). */
int nx_run(nx_engine* eng);
/* Replay clock: latencies for successive launches (in launch order). */
int nx_engine_set_replay_latencies(nx_engine* eng, const double* lat_s, size_t n);

typedef struct nx_engine_stats {
  uint64_t events;
  uint64_t decisions;
  uint64_t switches;
  uint64_t launches;
  uint64_t completed_requests;
  int32_t timed_out;
  int32_t current_r_p;
  double clock_s;
  int64_t kv_used;
  int64_t kv_reserved;
  int64_t kv_capacity;
} nx_engine_stats;
int nx_engine_get_stats(const nx_engine* eng, nx_engine_stats* out);

/* Logs, byte-compatible with serialize_event_log (eventlog.cpp:72-128) and
 * decision_log_text (simulator.cpp:25-36); summary with summary_json
 * (metrics.cpp:125-150). Size query with buf == NULL. */
int nx_engine_event_log(const nx_engine* eng, char* buf, size_t cap, size_t* len);
int nx_engine_decision_log(const nx_engine* eng, char* buf, size_t cap, size_t* len);
int nx_engine_summary_json(const nx_engine* eng, const char* label, char* buf, size_t cap,
                           size_t* len);
/* Per-launch latencies in launch order (the replay artefact). */
int nx_engine_launch_latencies(const nx_engine* eng, double* out, size_t cap, size_t* n);
/* Per-launch device time (ms, CUDA events on the lane stream); 0 without a device. */
int nx_engine_launch_device_ms(const nx_engine* eng, double* out, size_t cap, size_t* n);
/* Arrival with caller-provided prompt token ids (prompt_len of them). */
int nx_submit_with_tokens(nx_engine* eng, const nx_request* req, const int32_t* tokens);
/* Turn the event log / page log off for long benchmark runs (default on). */
int nx_engine_set_logging(nx_engine* eng, int32_t events, int32_t pages);
/* SLOs for goodput (new; the reference has no SLO metric). */
int nx_engine_set_slo(nx_engine* eng, double ttft_s, double tbt_p99_s);

typedef struct nx_goodput {
  uint64_t completed;
  uint64_t slo_met;
  double makespan_s;
  double goodput_tok_s; /* output tokens of SLO-meeting requests / makespan */
  double output_tokens; /* all output tokens of completed requests */
  double ttft_p50, ttft_p99, tbt_p50, tbt_p99;
} nx_goodput;
int nx_engine_goodput(const nx_engine* eng, nx_goodput* out);
/* Token ids of a request: prompt followed by generated tokens. */
int nx_engine_tokens(const nx_engine* eng, uint64_t id, int32_t* out, size_t cap, size_t* n);

/* Per-request outcome. */
typedef struct nx_request_state {
  uint64_t id;
  double arrival_s;
  int64_t prompt_len;
  int64_t output_len;
  int64_t prefilled_len;
  int64_t decoded_len;
  double first_token_s; /* -1 if none */
  double finish_s;      /* -1 if not finished */
} nx_request_state;
int nx_engine_requests(const nx_engine* eng, nx_request_state* out, size_t cap, size_t* n);
/* Emission times of one request's tokens (first token included). */
int nx_engine_token_times(const nx_engine* eng, uint64_t id, double* out, size_t cap, size_t* n);

/* ---- KV ledger + paged block manager (new; reference keeps bytes only,
 *      simulator.cpp:96-98,223-244,443-492) ---------------------------------- */
int nx_kv_usage(const nx_engine* eng, int64_t* used, int64_t* reserved, int64_t* capacity);
/* Current page ids of a live request, in position order. */
int nx_kv_block_table(const nx_engine* eng, uint64_t id, int32_t* pages, size_t cap,
                      size_t* n);
/* Page-assignment log: one record per allocation ("alloc id page") or release
 * ("free id page"), in order — the block-table parity artefact. */
int nx_kv_page_log(const nx_engine* eng, char* buf, size_t cap, size_t* len);
/* Page size (tokens) and pool size (pages); set before the first submit. */
int nx_kv_configure(nx_engine* eng, int32_t page_tokens, int32_t num_pages);

/* ---- device executor (new: the reference has no GPU path) ----
 * The kernels that replace the analytic operators (opcost.hpp:22):
 * QkvProj/AttnOutProj/Ffn -> tcgen05 GEMMs, AttnPrefill/AttnDecode -> paged
 * attention kernels, plus RMSNorm/RoPE/embedding/lm_head+argmax. */

/* Llama/Qwen-style decoder geometry (the reference's ModelConfig stays the
 * cost-model view; this is the kernel view). head_dim must be 128; hidden,
 * ffn and vocab multiples of 128. */
typedef struct nx_arch {
  int32_t hidden;
  int32_t n_layers;
  int32_t n_heads;
  int32_t n_kv_heads;
  int32_t head_dim;
  int32_t ffn;
  int32_t vocab;
  int32_t qkv_bias; /* 1: QKV projection has a bias (Qwen2.5) */
  float rope_theta;
  float rms_eps;
} nx_arch;

/* Tensor-parallel shard of one rank: QKV / gate-up
 * column-parallel, O / down row-parallel + all-reduce, vocab-parallel lm_head. */
typedef struct nx_tp_shard {
  int32_t tp_size, rank;
  int32_t q_head0, n_q_heads;
  int32_t kv_head0, n_kv_heads;
  int32_t ffn0, ffn_local;
  int32_t vocab0, vocab_local, vocab_valid, vocab_padded;
} nx_tp_shard;
int nx_tp_shard_plan(const nx_arch* arch, int32_t tp_size, int32_t rank, nx_tp_shard* out);
/* NCCL unique id (128 bytes) for a communicator; rank 0 creates, the caller
 * distributes (e.g. torch.distributed), every rank passes it to nx_device_create. */
int nx_nccl_unique_id(uint8_t out[128]);

/* Tensor-parallel execution modes.
 * NX_TP_NCCL: one process per GPU; this nx_device is rank tp_rank and talks
 *   to its peers through NCCL (all engines must issue identical batches).
 * NX_TP_PEER: this nx_device drives all tp_size ranks itself, rank r on CUDA
 *   device (device + r), collectives are peer-memory kernels over NVLink.
 * NX_TP_PEER_COLOCATED: as NX_TP_PEER with every rank on `device` (tests). */
enum { NX_TP_NCCL = 0, NX_TP_PEER = 1, NX_TP_PEER_COLOCATED = 2 };

typedef struct nx_device_config {
  nx_arch arch;
  int32_t device;             /* CUDA ordinal */
  int32_t page_tokens;        /* KV page size in tokens (16) */
  int32_t num_pages;          /* KV pool size in pages */
  int32_t max_prefill_tokens; /* token budget (+ decode batch for mixed lanes) */
  int32_t max_decode_batch;
  int32_t green_contexts;     /* 1: partition SMs per lane with CUDA green contexts */
  uint64_t weight_seed;
  float weight_gain;   /* weights ~ U(+-gain * sqrt(3/K)) -> unit-variance outputs */
  float lm_head_gain;  /* larger gain on lm_head widens the logit spread */
  int32_t tp_size;     /* 1 = single GPU */
  int32_t tp_rank;     /* NX_TP_NCCL: this process's rank */
  int32_t tp_mode;     /* NX_TP_NCCL / NX_TP_PEER / NX_TP_PEER_COLOCATED */
  int32_t tp_pad;
  uint8_t nccl_id[2][128]; /* NX_TP_NCCL: one communicator per lane (prefill, decode) */
} nx_device_config;

typedef struct nx_device nx_device;

typedef struct nx_device_info {
  int32_t sm_count;
  int32_t n_layouts;        /* green-context layouts (0 if disabled) */
  int32_t layout_decode_sms[32];
  int32_t layout_prefill_sms[32];
  uint64_t weight_bytes;
  uint64_t kv_bytes;
  uint64_t workspace_bytes;
} nx_device_info;

/* Allocates weights (deterministic random init on device), the paged KV
 * cache, per-lane workspaces, and pre-instantiates every green-context SM
 * layout. NX_ENODEV without a usable sm_100 GPU. */
int nx_device_create(const nx_device_config* cfg, nx_device** out);
void nx_device_destroy(nx_device* dev);
int nx_device_get_info(const nx_device* dev, nx_device_info* out);
/* Binds a device to an engine (before submitting requests); every launched
 * batch then runs on the device; tokens are greedy. */
int nx_engine_bind_device(nx_engine* eng, nx_device* dev);

/* Weight tensors, raw device layout (bf16). layer is ignored for global ones. */
#define NX_W_EMBED 0
#define NX_W_ATTN_NORM 1
#define NX_W_QKV 2      /* [(H + 2 Hkv) hd, hidden] */
#define NX_W_QKV_BIAS 3 /* [(H + 2 Hkv) hd] */
#define NX_W_O 4        /* [hidden, H hd] */
#define NX_W_FFN_NORM 5
#define NX_W_GATE_UP 6 /* [2 ffn, hidden]; 128-row blocks = 64 gate rows then the 64 matching up rows */
#define NX_W_DOWN 7    /* [hidden, ffn] */
#define NX_W_FINAL_NORM 8
#define NX_W_LM_HEAD 9 /* [vocab, hidden] */
int nx_device_weight(const nx_device* dev, int32_t tensor, int32_t layer, void* host,
                     size_t cap_bytes, size_t* bytes);

/* One forward batch, synchronous (kernel-level tests and the bench). Members
 * are described by parallel arrays; tokens holds sum(n_tokens) ids; pages
 * holds each member's page list back to back (n_pages each). lane: 0 prefill
 * / mixed lane, 1 decode lane; sm_pct picks the partition layout. Writes one
 * sampled token per member with sample[i] != 0 and, if logits != NULL, their
 * fp32 logits (row-major [n_sampled, vocab]). */
typedef struct nx_batch_desc {
  int32_t lane;
  int32_t sm_pct;
  int32_t n_members;
  int32_t _pad0;
  const int32_t* n_tokens;
  const int64_t* start_pos;
  const int32_t* sample;
  const int32_t* tokens;
  const int32_t* n_pages;
  const int32_t* pages;
} nx_batch_desc;
int nx_device_forward(nx_device* dev, const nx_batch_desc* b, int32_t* sampled, float* logits,
                      double* device_ms);
/* Asynchronous halves of nx_device_forward: launch on the lane's partition
 * stream and return; wait for that lane's batch (co-location experiments). */
int nx_device_launch(nx_device* dev, const nx_batch_desc* b);
int nx_device_wait(nx_device* dev, int32_t lane, int32_t* sampled, float* logits,
                   double* device_ms);

/* Launch observer (new): called on every engine launch, before the bound
 * device (if any) sees it, with the batch in nx_batch_desc form (tokens NULL
 * when the engine holds no token ids, i.e. no device bound). The pointers are
 * valid during the call only. Under NX_TP_NCCL the ranks' devices must run
 * identical batches in identical per-lane order: rank 0's engine serves on
 * the device clock and its observer forwards each batch to the followers,
 * which replay it with nx_device_launch (paper_2507_06608_b200.device
 * tp_follow). */
typedef void (*nx_launch_observer)(void* user, const nx_batch_desc* batch);
int nx_engine_set_launch_observer(nx_engine* eng, nx_launch_observer fn, void* user);

/* Kernel-class timing (CUDA events on the launching stream, every
 * `sample_every`-th batch per lane; 0 disables) with algorithmic work. */
#define NX_K_GEMM_DECODE 0  /* projections on the decode lane (HBM-bound weight stream) */
#define NX_K_GEMM_PREFILL 1 /* projections on the prefill / mixed lane (tensor-bound) */
#define NX_K_ATTN_DECODE 2  /* split-KV paged decode attention (HBM-bound KV stream) */
#define NX_K_ATTN_PREFILL 3 /* causal paged prefill attention */
#define NX_K_OTHER 4        /* norms, RoPE/KV write, embedding, argmax */
#define NX_K_CLASSES 5
typedef struct nx_kernel_stats {
  double ms[NX_K_CLASSES];
  double bytes[NX_K_CLASSES];  /* algorithmic bytes moved */
  double flops[NX_K_CLASSES];  /* algorithmic FLOPs */
  uint64_t launches[NX_K_CLASSES];
  uint64_t batches_sampled;
  double batch_ms_sampled; /* whole-batch device time of the sampled batches */
  uint64_t kernel_launches; /* every kernel this device launched (all batches) */
  uint64_t batches;         /* every batch this device ran */
  double sm_ms[NX_K_CLASSES]; /* sum of (lane SM count x event ms): / ms = mean partition size */
  /* the same sampled event time charged to the reference operator a kernel
   * belongs to (NX_OP_*: the projection GEMM with its norm / fold / RoPE /
   * all-reduce kernels, or the attention); embedding, lm_head and sampling
   * are not operators of the cost model and are not charged */
  double op_ms[5];
  uint64_t op_launches[5];
} nx_kernel_stats;
int nx_device_set_profiling(nx_device* dev, int32_t sample_every);
int nx_device_kernel_stats(const nx_device* dev, nx_kernel_stats* out);
int nx_device_reset_kernel_stats(nx_device* dev);

/* ---- raw device plumbing + single-op entry points (tests / profiling) --- */
int nx_dev_malloc(size_t bytes, void** p);
int nx_dev_free(void* p);
int nx_dev_h2d(void* dst, const void* src, size_t bytes);
int nx_dev_d2h(void* dst, const void* src, size_t bytes);
int nx_dev_sync(void);
/* out = epilogue(x[tokens, K] . w[rows, K]^T) with the tcgen05 GEMM; mode is
 * the epilogue (0 store, 1 bias, 2 residual, 3 bias+residual, 4 SwiGLU,
 * 6 fp32; 16 / 17: the decode GEMM (tokens <= 128) with deferred fold /
 * direct, fp32 out). sm_count caps the persistent grid; splits 0 = automatic,
 * -2 = the CTA-pair (cta_group::2) prefill kernel.
 * Returns the device time of `iters` launches in *ms (may be NULL). */
/* Diagnostics: per-CTA %globaltimer milestones of the last GEMM launched with
 * NX_GEMM_DBG & 16 set ([cta][8] u64); returns the count copied. */
size_t nx_dbg_gemm_trace(uint64_t* out, size_t n);
int nx_op_gemm(const void* x, const void* w, int32_t tokens, int32_t rows, int32_t K, int32_t mode,
               void* out, int32_t ldo, const void* bias, const void* residual, int32_t ldr,
               int32_t sm_count, int32_t splits, int32_t iters, float* ms);

#ifdef __cplusplus
}
#endif

#endif /* NEXUS_B200_H */
