/*
 * superneurons.h -- C ABI of the B200-native SuperNeurons memory-scheduled
 * training step (planner: libsnplan.so, executor: libsnexec.so).
 *
 * The reference (memsched 0.1.0, pure Python) has no FFI; its boundary is the
 * Python API re-exported by pkg/src/memsched/__init__.py:69-130.  Each entry
 * point below replaces one reference call; the Python facade
 * paper_1801_04380_b200/ keeps the reference's names on top of these.
 *
 *   sn_plan_create      <- memsched.simulator._Simulation.__init__ + run()
 *                          (pkg/src/memsched/simulator.py:192-259, 500-548);
 *                          i.e. run_simulation(net, cfg) (simulator.py:734-735)
 *   sn_plan_report/rows/selections/modes
 *                       <- SimReport fields (simulator.py:134-170, 683-731)
 *   sn_plan_tape        <- (new) the physical event tape the reference only
 *                          implies: BlockPool.alloc/free (poolalloc.py:80-124),
 *                          _TransferEngine.submit (simulator.py:181-188),
 *                          LruCache ops (offload.py:100-129), replays
 *                          (simulator.py:417-423) and compute points
 *                          (simulator.py:562-565, 612-615)
 *   sn_plan_costs       <- costmodel.build_costs (costmodel.py:171-204)
 *   sn_plan_order       <- netgraph.build_schedule (netgraph.py:300-309)
 *   sn_plan_demands     <- recompute.step_demands / min_pool_bytes
 *                          (recompute.py:173-205, 242-244)
 *   sn_exec_*           <- (new) the device executor; no reference counterpart
 *                          (the reference models compute/transfer time only,
 *                          costmodel.py:181-202, simulator.py:173-188).
 *
 * Return codes: SN_OK, or an SN_ERR_* class; sn_last_error() gives the message
 * and sn_last_error_kind() the exact reference exception type (SN_EK_*).
 * Errors are thread-local.  No function allocates device memory except
 * sn_exec_create (one arena, one parameter block, pinned host stash).
 */
#ifndef SUPERNEURONS_H
#define SUPERNEURONS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- return codes (CLI exit-code classes, reference cli.py:250-260) ---- */
#define SN_OK 0
#define SN_ERR_OTHER 1
#define SN_ERR_CONFIG 2 /* ConfigError / NetError / CostError / PoolError class */
#define SN_ERR_SCHED 3  /* SchedulingError class */
#define SN_ERR_CUDA 4   /* CUDA / NCCL failure (executor only) */

/* ---- exact exception kinds (reference errors.py:8-17 and subclasses) ---- */
enum sn_error_kind {
  SN_EK_NONE = 0,
  SN_EK_CONFIG = 1,      /* ConfigError */
  SN_EK_SCHED = 2,       /* SchedulingError */
  SN_EK_COST = 3,        /* costmodel.CostError */
  SN_EK_NETVALID = 4,    /* netgraph.NetValidationError */
  SN_EK_POOL = 5,        /* poolalloc.PoolError */
  SN_EK_POOLEXH = 6,     /* poolalloc.PoolExhausted */
  SN_EK_ALLLOCKED = 7,   /* offload.AllLockedError */
  SN_EK_ZERODIV = 8,     /* ZeroDivisionError (stride 0 in a window) */
  SN_EK_INTERNAL = 9,    /* implementation limit (e.g. int64 overflow) */
  SN_EK_CUDA = 10,       /* executor: CUDA / NCCL error */
  SN_EK_UNSUPPORTED = 11 /* executor: graph not executable numerically */
};

const char* sn_version(void);
const char* sn_last_error(void);
int sn_last_error_kind(void);

/* ---- layer kinds (netgraph.py:35-45), in declaration order ---- */
enum sn_layer_kind {
  SN_DATA = 0, SN_CONV, SN_POOL, SN_ACT, SN_LRN, SN_BN, SN_FC, SN_DROPOUT, SN_SOFTMAX, SN_JOIN
};

/* Integer layer parameters read by the cost model (costmodel.py:113-168). */
enum sn_param { SN_P_C = 0, SN_P_H, SN_P_W, SN_P_OUT, SN_P_K, SN_P_S, SN_P_P, SN_NPARAM };

typedef struct sn_net_desc {
  const char* name;
  int32_t n_layers;
  const int32_t* kinds;              /* sn_layer_kind per layer id */
  const char* const* names;          /* layer names */
  const char* const* name_reprs;     /* Python repr() of each name, for messages */
  const int32_t* prev_off;           /* CSR: prev ids of layer i are      */
  const int32_t* prev_idx;           /*   prev_idx[prev_off[i]..prev_off[i+1]) */
  const int32_t* next_off;           /* CSR, edge declaration order */
  const int32_t* next_idx;
  const int8_t* param_state;         /* [n_layers][SN_NPARAM]: 0 absent, 1 int, 2 other */
  const int64_t* param_int;          /* [n_layers][SN_NPARAM] value when state == 1 */
  const char* const* param_repr;     /* [n_layers][SN_NPARAM] repr() when state == 2 */
} sn_net_desc;

/* Recompute policies (recompute.py:35). */
enum sn_recompute { SN_RC_NONE = 0, SN_RC_SPEED = 1, SN_RC_MEMORY = 2, SN_RC_COST_AWARE = 3 };

/* SimConfig (simulator.py:108-117) with CostConfig (costmodel.py:32-51) and
 * the *normalized* Features (simulator.py:56-63). */
typedef struct sn_sim_config {
  int64_t pool_bytes;
  int32_t liveness, offload, cache, recompute, convselect;
  int64_t batch, dtype_bytes;
  double time_per_elem, heavy_time_per_elem, backward_time_factor, bandwidth_bytes_per_s;
} sn_sim_config;

typedef struct sn_report {
  int32_t num_layers, num_steps;
  int64_t peak_bytes;
  int32_t peak_step, peak_layer;
  int64_t peak_live_count, peak_working_bytes, peak_stash_bytes;
  int64_t min_pool_bytes, baseline_peak_bytes, liveness_peak_bytes;
  double compute_s, stall_s, stall_prefetch_s, stall_demand_s, stall_backup_s;
  double transfer_busy_s, total_s;
  int64_t scheduled_transfer_bytes, scheduled_transfer_count;
  int64_t demand_transfer_bytes, demand_transfer_count;
  int64_t cache_hits, evictions, extra_forward_steps, planned_extra_forward_steps;
  int64_t pool_high_water_bytes;
  int32_t n_rows, n_selections, n_modes;
} sn_report;

/* StepRow (simulator.py:120-131); phase 0 forward, 1 backward, 2 replay. */
typedef struct sn_step_row {
  double index;
  int32_t layer, phase;
  int64_t resident_bytes, live_count, pool_used_bytes;
  double compute_s, stall_s;
  int64_t transfer_bytes;
} sn_step_row;

/* Selection (convselect.py:41-49); algo 0 implicit-gemm, 1 gemm-workspace, 2 fft. */
typedef struct sn_selection {
  double step;
  int32_t layer, phase, algo, pad_;
  int64_t workspace_bytes, free_bytes;
} sn_selection;

/* One physical event of the iteration, in execution order.
 *   'A' alloc   a=key kind (0 act,1 grad,2 ws) b=key id c=block offset d=blocks e=high
 *   'F' free    a=key kind b=key id
 *   'C' forward compute of layer b, e=algo (-1 none), d=workspace key step (-1 none)
 *   'B' backward compute of layer b, e/d as for 'C'
 *   'R' replayed forward of layer b            'O' copy-out (D2H) of layer b
 *   'P' scheduled fetch (H2D) of layer b       'D' demand fetch (H2D) of layer b
 *   'I' cache insert b   'T' cache touch b   'X' cache discard b   'E' evict b
 *   'H' cache hit b      'V' revive pending-drop copy b            'S' end of step b */
typedef struct sn_event {
  char op;
  char pad_[3];
  int32_t a, b, e;
  int64_t c, d;
} sn_event;

/* Per-layer cost (costmodel.py:54-64); shape padded with 0s. */
typedef struct sn_layer_cost {
  int32_t ndim;
  int32_t pad_;
  int64_t shape[3];
  int64_t out_elems, out_bytes, device_bytes, grad_bytes, param_bytes;
  double fwd_time, bwd_time;
} sn_layer_cost;

typedef struct sn_plan sn_plan;

int sn_plan_create(const sn_net_desc* net, const sn_sim_config* cfg, sn_plan** out);
void sn_plan_destroy(sn_plan* plan);
int sn_plan_report(const sn_plan* plan, sn_report* out);
int sn_plan_rows(const sn_plan* plan, sn_step_row* rows, size_t cap, size_t* n);
int sn_plan_selections(const sn_plan* plan, sn_selection* sel, size_t cap, size_t* n);
int sn_plan_modes(const sn_plan* plan, int32_t* modes, size_t cap, size_t* n); /* 1 speed 2 memory */
int sn_plan_tape(const sn_plan* plan, const sn_event** events, size_t* n);
int sn_plan_costs(const sn_plan* plan, sn_layer_cost* costs, size_t cap, size_t* n);
int sn_plan_order(const sn_plan* plan, int32_t* forward_ids, size_t cap, size_t* n);
int sn_plan_demands(const sn_plan* plan, int64_t* demands, size_t cap, size_t* n);

/* Planning without simulation (analysis entry points of the reference API):
 * shapes/costs, forward order, per-step demands; cfg->pool_bytes ignored. */
int sn_analyze(const sn_net_desc* net, const sn_sim_config* cfg, sn_plan** out);
/* Cost table only, with costmodel.build_costs' error semantics (no schedule). */
int sn_build_costs(const sn_net_desc* net, const sn_sim_config* cfg, sn_plan** out);

/* The planner's block pool on its own (poolalloc.BlockPool, poolalloc.py:35-163):
 * 1 KiB blocks, two-ended first fit, coalescing free.  Keys are caller ids. */
typedef struct sn_pool sn_pool;
int sn_pool_create(int64_t capacity_bytes, sn_pool** out);
void sn_pool_destroy(sn_pool* pool);
int sn_pool_alloc(sn_pool* pool, int64_t key, int64_t nbytes, int32_t high, int64_t* block_offset);
int sn_pool_free(sn_pool* pool, int64_t key);
int sn_pool_check(const sn_pool* pool);
/* used / free / high-water in bytes, capacity in blocks, number of live keys */
int sn_pool_stats(const sn_pool* pool, int64_t* used, int64_t* free_bytes, int64_t* high_water,
                  int64_t* capacity_blocks, int64_t* n_keys);
/* Free spans (is_free=1) or allocated spans with their keys (is_free=0), by offset. */
int sn_pool_spans(const sn_pool* pool, int32_t is_free, int64_t* offsets, int64_t* lengths, int64_t* keys,
                  size_t cap, size_t* n);

/* Test hook: CPython set iteration order emulation (see planner/pool.hpp). */
int sn_debug_pyset(const int64_t* a, size_t na, const int64_t* b, size_t nb, const int64_t* a2,
                   size_t na2, int64_t* out, size_t cap, size_t* n);

/* ======================================================================
 * Executor (libsnexec.so): replays a plan's tape on one B200.
 * ====================================================================== */

/* Numeric constants the reference leaves open; per layer. */
typedef struct sn_layer_numerics {
  int32_t pool_mode;    /* 0 max, 1 avg (count includes padding) */
  int32_t lrn_size;     /* cross-channel window (odd) */
  float lrn_alpha, lrn_beta, lrn_k;
  float dropout_rate;
  float bn_eps, bn_momentum;
} sn_layer_numerics;

typedef struct sn_exec_options {
  int32_t device;
  int32_t elide_backups;  /* 1: skip copy-outs the tape never fetches back */
  int32_t use_graph;      /* 1: capture the iteration into a CUDA graph */
  int32_t num_classes;    /* labels in [0, num_classes) */
  uint64_t seed;          /* dropout mask seed */
  float lr;               /* SGD learning rate */
  float grad_scale;       /* multiply gradients before the update (1/world) */
  int32_t precision;      /* CONV / FC math: 0 tf32 tensor cores (fp32 accumulate),
                             1 fp32-faithful 3xTF32 split operands (~3x the MMA work) */
  int32_t stash;          /* where copied-out tensors live: 0 pinned host memory (PCIe),
                             1 device memory of stash_device (an NVLink peer's spare HBM;
                             the executor's own device = same-device loopback) */
  int32_t stash_device;
  int32_t autotune;       /* 1: benchmark the CONV kernel variants per layer shape at create time
                             and run the fastest (non-parity mode: summation orders differ);
                             sn_exec_catalog reports the measurements */
  /* Data-parallel replica; dp_comm NULL = single replica.  The
   * weight gradients are summed over the dp_world ranks by ncclAllReduce in
   * buckets of about dp_bucket_bytes, each issued on a communication stream
   * as soon as the backward steps of its layers are done (overlapping the
   * rest of the backward), and each bucket's SGD update (grad_scale applied,
   * normally 1/world) follows its all-reduce on that stream. */
  void* dp_comm;          /* ncclComm_t from sn_dp_comm_create, owned by the caller */
  int32_t dp_world, dp_rank;
  int64_t dp_bucket_bytes; /* 0: default (8 MiB) */
} sn_exec_options;

typedef struct sn_step_timing {
  float step_ms;            /* device time of the whole iteration */
  float h2d_ms, d2h_ms;     /* copy-engine busy time (events) */
  int64_t kernels;          /* kernel launches in the iteration */
  int64_t d2h_bytes, h2d_bytes;
  int64_t arena_high_water; /* bytes of the arena touched (from the tape) */
} sn_step_timing;

typedef struct sn_exec sn_exec;

/* Executor errors (thread-local, separate from the planner's). */
const char* sn_exec_last_error(void);
int sn_exec_last_error_kind(void);

int sn_exec_create(const sn_plan* plan, const sn_net_desc* net, const sn_layer_numerics* numerics,
                   const sn_exec_options* opts, sn_exec** out);
void sn_exec_destroy(sn_exec* ex);
/* Device pointers of the flat fp32 parameter and gradient blocks. */
int sn_exec_params(sn_exec* ex, float** params, float** grads, int64_t* n_floats);
/* Offset/count (floats) of layer `layer`'s weights (w) and bias/affine (b). */
int sn_exec_param_slice(sn_exec* ex, int32_t layer, int64_t* w_off, int64_t* w_n, int64_t* b_off,
                        int64_t* b_n);
/* Device input buffers owned by the executor (NHWC fp32 images, int32 labels). */
int sn_exec_inputs(sn_exec* ex, float** images, int32_t** labels, int64_t* image_floats);
/* Forward + backward (+ optional SGD update) of one iteration on the
 * executor's input buffers.  update=0 leaves parameters untouched. */
int sn_exec_step(sn_exec* ex, int32_t update, float* loss_host, sn_step_timing* timing);
/* End-to-end: copy host images/labels in, run the step, read the loss back. */
int sn_exec_step_host(sn_exec* ex, const float* images_host, const int32_t* labels_host,
                      int32_t update, float* loss_host, sn_step_timing* timing);
/* End-to-end with a one-batch input pipeline (the data layer's prefetch):
 * runs the step on images_host/labels_host and, while it computes, copies
 * next_images_host/next_labels_host (may be NULL) in: the images straight into
 * the executor's input buffer as soon as this step's DATA layer has laid its
 * own out, the labels into a staging buffer.  A call whose images_host is the
 * batch staged by the previous call only waits for what is left of that copy;
 * otherwise it stages it first.  The next_* host buffers must stay unchanged
 * until the following call returns; other entry points (sn_exec_step,
 * sn_exec_step_host, sn_exec_inputs) drop a staged batch. */
int sn_exec_step_host_pipelined(sn_exec* ex, const float* images_host, const int32_t* labels_host,
                                const float* next_images_host, const int32_t* next_labels_host, int32_t update,
                                float* loss_host, sn_step_timing* timing);
/* End to end over n host batches (images NHWC fp32, labels int32; pinned for
 * overlap) in one call -- the reference's training loop (memsched
 * run_training iterations) on the B200: batch k+1 is copied in while step k
 * computes (as sn_exec_step_host_pipelined), and every step's loss is read
 * back into losses[k] while the next step runs, so the device never idles on
 * the host between steps.  timing->step_ms = device ms per step (mean). */
int sn_exec_train_host(sn_exec* ex, int32_t n, const float* const* images_host, const int32_t* const* labels_host,
                       int32_t update, float* losses, sn_step_timing* timing);
/* Copy a layer's current forward output (if resident in the arena) or its
 * gradient buffer to device memory `dst`; used by parity tests. */
int sn_exec_read_tensor(sn_exec* ex, int32_t kind, int32_t layer, float* dst, int64_t n_floats);
/* Run one iteration eagerly with a CUDA event between consecutive actions on
 * the compute stream; per action: device ms, layer id (-1 none) and type
 * (0 forward, 1 replay, 2 backward, 3 copy/sync).  For roofline accounting:
 * the weight gradients run on the compute stream too (serial), so each
 * action's interval holds exactly its own kernels. */
int sn_exec_profile(sn_exec* ex, float* action_ms, int32_t* action_layer, int32_t* action_type, size_t cap,
                    size_t* n);
/* Per-action kernel census of one iteration (for per-launch tables): action i
 * of sn_exec_profile launched action_kernels[i] kernels; `names` receives
 * their mangled function names, '\n'-terminated, each action's list closed
 * by a 0x1e byte (truncated to names_cap).  Captured from one serial
 * iteration (weight gradients on the compute stream), nothing executed. */
int sn_exec_census(sn_exec* ex, int32_t* action_kernels, size_t cap, char* names, size_t names_cap, size_t* n);
/* Per-kernel CUDA-event time of one iteration: the serial iteration of
 * sn_exec_census replayed node by node on the compute stream (copies and
 * memsets too), an event pair around every kernel, median of `reps` replays.
 * us[k] / action[k] for the k-th kernel in issue order (n = count; call with
 * us = NULL first to size the buffers). */
int sn_exec_kernel_times(sn_exec* ex, int32_t reps, float* us, int32_t* action, size_t cap, size_t* n);
/* Launch the SGD update alone (after an external gradient all-reduce). */
int sn_exec_apply_update(sn_exec* ex, float lr, float grad_scale);
/* CONV weight gradients whose split-K partials live in the conv workspace the
 * plan granted their step (reference simulator.py:624-654, the dynamic
 * workspace) vs in executor scratch outside the pool (workspace too small). */
int sn_exec_workspace_use(const sn_exec* ex, int32_t* wgrad_in_pool, int32_t* wgrad_outside);
/* Transfers of the last iteration (offload copy-outs and fetches the tape
 * issued, reference simulator.py:378-413): bytes and copy-engine busy time per
 * direction, and the time the compute stream stood blocked on fetches (the
 * exposed, non-overlapped transfer time).  Synchronises the compute stream. */
int sn_exec_transfer_stats(sn_exec* ex, int64_t* d2h_bytes, double* d2h_ms, int64_t* h2d_bytes, double* h2d_ms,
                           double* exposed_ms);
/* Device (and pinned host) memory the executor allocated, by purpose.  The
 * arena is the one pool allocation (ceil_KiB(pool_bytes), reference
 * simulator.py:204); everything else is outside the reference's residency
 * accounting (parameters and gradients, costmodel.py:3-6) or executor-owned. */
typedef struct sn_exec_mem {
  int64_t arena_bytes;
  int64_t params_grads_bytes;
  int64_t layer_state_bytes;    /* BN saved / running statistics, max-pool argmax bytes */
  int64_t input_bytes;          /* images, labels, the stem's padded copy, staging */
  int64_t wgrad_scratch_bytes;  /* weight-gradient scratch outside the pool (partials that
                                   did not fit their granted workspace, reductions) */
  int64_t other_scratch_bytes;  /* FC split-K, weight transposes, BN tile statistics, ... */
  int64_t host_stash_bytes;     /* pinned host memory of copied-out tensors (stash 0) */
  int64_t device_stash_bytes;   /* stash 1 on this device (loopback) */
  int64_t peer_stash_bytes;     /* stash 1 on a peer device's HBM */
  int64_t device_total_bytes;   /* sum of this device's categories (arena .. device stash) */
  int64_t wgrad_partials_outside_pool_bytes;
  int64_t planned_arena_high_water; /* the planner's BlockPool high water */
} sn_exec_mem;
int sn_exec_memory(const sn_exec* ex, sn_exec_mem* out);
/* Measured arena use: sn_exec_arena_fill writes a sentinel (0xFF bytes, a NaN
 * no kernel produces) over the whole arena; after a step, sn_exec_arena_scan
 * returns the end of the highest 1 KiB block any kernel or copy wrote
 * (high_water_bytes) and the bytes of all written blocks. */
int sn_exec_arena_fill(sn_exec* ex);
int sn_exec_arena_scan(sn_exec* ex, int64_t* high_water_bytes, int64_t* touched_bytes);
/* The measured CONV kernel-variant catalog (autotune): one entry per (layer
 * shape, op, variant): the representative layer, op 0 forward / 1 dgrad /
 * 2 wgrad, the dispatch knobs (halo 0 off / 1 by shape, pairs 0 off / 1 by
 * size, bn 0 policy / forced im2col tile width, subpix 0 off / 1 on), the
 * median event time in microseconds, and whether it was chosen. */
typedef struct sn_catalog_entry {
  int32_t layer, op;
  int32_t halo, pairs, bn, subpix;
  float us;
  int32_t chosen;
} sn_catalog_entry;
int sn_exec_catalog(const sn_exec* ex, sn_catalog_entry* out, size_t cap, size_t* n);
/* Stream the executor launches on (for cross-library ordering). */
void* sn_exec_stream(sn_exec* ex);

/* ======================================================================
 * Data-parallel replicas: one process per GPU, NCCL (libnccl.so.2 loaded at
 * run time) for the one collective of the path, the weight-gradient sum.
 * ====================================================================== */
typedef struct sn_dp_id {
  char bytes[128]; /* ncclUniqueId: made by rank 0, broadcast by the caller */
} sn_dp_id;
const char* sn_dp_last_error(void);
int sn_dp_nccl_version(int32_t* version);
int sn_dp_unique_id(sn_dp_id* out);
int sn_dp_comm_create(const sn_dp_id* id, int32_t world, int32_t rank, int32_t device, void** comm_out);
void sn_dp_comm_destroy(void* comm);
/* The all-reduce buckets of a plan (host only, no device needed): bucket i
 * covers floats [lo[i], hi[i]) of the flat gradient block and is issued right
 * after the backward step of layer after_layer[i]; buckets are in issue
 * (backward) order and cover every parameter float exactly once. */
int sn_dp_buckets(const sn_plan* plan, int64_t bucket_bytes, int64_t* lo, int64_t* hi, int32_t* after_layer,
                  size_t cap, size_t* n);

#ifdef __cplusplus
}
#endif

#endif /* SUPERNEURONS_H */
