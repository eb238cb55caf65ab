/*
 * opscale_b200.h -- C ABI of the B200-native candidate-evaluation path.
 *
 * This library replaces the search core of the opscaler planners
 * (arXiv 2511.02248 reference, pkg/src/opscaler/autoscaler.py):
 *
 *   opsc_menu_build        <- _Evaluator.predict_op menu loops
 *                             (autoscaler.py:743-757; perfmodel.py:62-64,133-171;
 *                              queueing.py:54-87)
 *   opsc_stability_check   <- init_configs NoStableConfig pre-check that the
 *                             brute-force oracle inherits from its greedy warm
 *                             start (autoscaler.py:254-294, 771)
 *   opsc_compose_argmin    <- brute_force_autoscale descend + leaf mask +
 *                             lexicographic argmin (autoscaler.py:786-826)
 *   opsc_menu_fallback     <- infeasible-SLO per-op fallback (autoscaler.py:828-841)
 *   opsc_decode_decisions  <- best_assign -> OperatorConfig (autoscaler.py:843-845)
 *   opsc_model_grid        <- model_level_autoscale (autoscaler.py:596-681)
 *   opsc_materialize       <- _Evaluator.evaluate + _make_plan
 *                             (autoscaler.py:196-247; opgraph.py:199-244),
 *                             metrics.request_energy (metrics.py:84-102),
 *                             provisioned_memory (metrics.py:130-132) and
 *                             default_stream_place.devices_used
 *                             (placement.py:358-385, 465-491)
 *   opsc_greedy            <- greedy_autoscale (autoscaler.py:334-589)
 *   opsc_plan_windows_host <- runner.plan_for_mode looped over windows
 *                             (runner.py:38-52, cli.py:135-150), host buffers in
 *                             and out, one call per batch of windows.
 *
 * Conventions
 *   - Operators are indexed by their rank in sorted(node_ids) ("lex rank").
 *     That is the brute-force menu order (autoscaler.py:725).
 *   - All floating point is IEEE binary64, evaluated in exactly the
 *     reference's association order with no FMA contraction.
 *   - Device-pointer entry points take a cudaStream_t (passed as void*) and
 *     never allocate or synchronise. Host-buffer entry points go through an
 *     opaque context that owns its device workspace.
 *   - Every entry point returns an int status (OPSC_OK = 0); no exception
 *     crosses the ABI. Per-window semantic outcomes (NoStableConfig, ...) are
 *     reported in per-window status words (OPSC_W_* bits).
 */
#ifndef OPSCALE_B200_H
#define OPSCALE_B200_H

#include <stdint.h>
#include <stddef.h>

#if defined(__GNUC__)
#define OPSC_API __attribute__((visibility("default")))
#else
#define OPSC_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define OPSC_ABI_VERSION 1

#define OPSC_MAX_OPS 32
#define OPSC_MAX_EDGES 256
#define OPSC_MAX_P 8
#define OPSC_MAX_DEVICES 1024
#define OPSC_PRED_FIELDS 7 /* op_latency, lam, mu, utilization, wait, service, comm */

/* call status codes */
#define OPSC_OK 0
#define OPSC_ERR_ARG 1      /* bad argument / size limit exceeded        */
#define OPSC_ERR_CUDA 2     /* CUDA runtime error                          */
#define OPSC_ERR_SPACE 3    /* candidate space exceeds the 2^40 key field  */
#define OPSC_ERR_NODEVICE 4 /* no CUDA device / extension unusable         */

/* per-window status bits */
#define OPSC_W_NO_STABLE_BOUNDS 0x1u   /* NoStableConfig: op has no stable entry in bounds (autoscaler.py:835) */
#define OPSC_W_NO_STABLE_PARAMS 0x2u   /* NoStableConfig: init_configs pre-check failed (autoscaler.py:289) */
#define OPSC_W_NO_STABLE_MODEL 0x4u    /* NoStableConfig: model-level found no stable batch (autoscaler.py:678) */
#define OPSC_W_ZERO_DIVISION 0x8u      /* reference would raise ZeroDivisionError (T*layers == 0) */
#define OPSC_W_UNSTABLE_ROUNDING 0x10u /* lam < R*mu but lam/(R*mu) rounds to 1.0: reference raises Unstable */
#define OPSC_W_FLEET_EXHAUSTED 0x20u   /* default-stream placement ran out of devices (placement.py:183-187) */
#define OPSC_W_INFEASIBLE_PLACEMENT 0x40u /* a replica exceeds device memory (placement.py:379-383, 485-489) */
#define OPSC_W_IDLE 0x80u              /* qps <= 0: no plan (cli.py:138-144) */

/* planning modes (runner.py:38-52) */
#define OPSC_MODE_ORACLE 0   /* brute_force_autoscale, exhaustive */
#define OPSC_MODE_MODEL 1    /* model_level_autoscale */
#define OPSC_MODE_OPERATOR 2 /* greedy_autoscale (operator level, Alg. 1 as coded) */

#define OPSC_W_NO_STABLE_INIT 0x100u    /* NoStableConfig from init_configs (autoscaler.py:289) in greedy mode */
#define OPSC_W_TRACE_TRUNCATED 0x200u   /* more trace entries than trace_cap */
#define OPSC_W_ORDER_SENSITIVE 0x400u   /* brute force, opt-in certificate (OPSC_PLAN_CERTIFY /
                                           opsc_certify_order): the decision could depend on the
                                           reference's frozenset-ordered leaf sum (autoscaler.py:792-796),
                                           i.e. argmin over lat <= slo - band != argmin over
                                           lat <= slo + band (band = OPSC_CERTIFY_BAND_ULPS ulps of slo) */
/* OR'ed into the mode of opsc_plan_windows_host: brute force also runs the
 * order certificate and sets OPSC_W_ORDER_SENSITIVE (ignored by the other modes,
 * whose latencies are the canonical critical_path_latency, opgraph.py:223-244) */
#define OPSC_PLAN_CERTIFY 0x100
#define OPSC_CERTIFY_BAND_ULPS 64.0
/* Which operator the reference's NoStableConfig message names (so the host can
 * raise it with the reference's exact text):
 *   bits 16..21: 1 + position in dag.node_ids order of the first operator
 *                init_configs finds unstable at every (B, P) (autoscaler.py:289-292;
 *                set with OPSC_W_NO_STABLE_PARAMS / OPSC_W_NO_STABLE_INIT);
 *   bits 22..27: 1 + lexicographic rank of the first operator without a finite
 *                menu entry (autoscaler.py:833-837; set with OPSC_W_NO_STABLE_BOUNDS). */
#define OPSC_W_INIT_OP_SHIFT 16
#define OPSC_W_BOUNDS_OP_SHIFT 22
#define OPSC_W_OP_FIELD 0x3fu

/* greedy trace actions (autoscaler.py:363, 446-454, 478-486, 549-557, 579-587) */
#define OPSC_ACT_UPSCALE 1
#define OPSC_ACT_DOWNSCALE 2
#define OPSC_ACT_HEADROOM 3
#define OPSC_ACT_PRUNE 4
#define OPSC_ACT_RESEED 5

#define OPSC_KEY_INFEASIBLE 0x7fffffffffffffffLL
#define OPSC_KEY_LEX_BITS 40

/* Static DAG + profile tables, indexed by lex rank.
 * Built once per planning instance by the host (opgraph.py:71-148,
 * perfmodel.py:79-130). Passed by value to every kernel. */
typedef struct OpscDag {
  int32_t n_ops;
  int32_t n_edges;
  int32_t topo[OPSC_MAX_OPS];        /* lex ranks in OperatorDag.topo_order   */
  int32_t node_order[OPSC_MAX_OPS];  /* lex ranks in OperatorDag.node_ids order */
  int32_t layer_count[OPSC_MAX_OPS];
  uint32_t pred_mask[OPSC_MAX_OPS];  /* bit p set iff edge p -> v              */
  uint32_t sink_mask;                /* bit v set iff v has no successor       */
  uint32_t has_phase[2];             /* bit v set iff profile of v models phase (0 prefill, 1 decode) */
  double c0[2][OPSC_MAX_OPS];        /* LatencyModel per phase (perfmodel.py:50-64) */
  double c1[2][OPSC_MAX_OPS];
  double c2[2][OPSC_MAX_OPS];
  double eta[OPSC_MAX_OPS];
  double weight_mem[OPSC_MAX_OPS];
  double m0[OPSC_MAX_OPS];
  double m1[OPSC_MAX_OPS];
  double s0[OPSC_MAX_OPS];
  double s1[OPSC_MAX_OPS];
  int32_t out_ptr[OPSC_MAX_OPS + 1]; /* out edges of v: [out_ptr[v], out_ptr[v+1]) in dag.out_edges order */
  double out_v0[OPSC_MAX_EDGES];     /* volume_ref profile v0 / v1 of each out edge */
  double out_v1[OPSC_MAX_EDGES];
  double link_bw;
} OpscDag;

/* Brute-force candidate grid (BruteForceBounds, autoscaler.py:688-700).
 * Menu of op v: entries e in lexicographic (P, R, B) order,
 * e = (pi * r_max + (r - 1)) * b_max[v] + (b - 1). */
typedef struct OpscGrid {
  int32_t r_max;
  int32_t n_p[OPSC_MAX_OPS];
  int32_t p_vals[OPSC_MAX_OPS][OPSC_MAX_P]; /* ascending, duplicates kept */
  int32_t b_max[OPSC_MAX_OPS];
  int32_t menu_off[OPSC_MAX_OPS + 1];       /* prefix sum of menu sizes      */
  /* AutoscaleParams view used by the init_configs pre-check */
  int32_t r_cap;
  int32_t params_n_p[OPSC_MAX_OPS];
  int32_t params_p_vals[OPSC_MAX_OPS][OPSC_MAX_P];
  int32_t params_b_max[OPSC_MAX_OPS];
} OpscGrid;

/* Model-level grid (autoscaler.py:612-615). */
typedef struct OpscModelSpec {
  int32_t p_base[OPSC_MAX_OPS]; /* smallest allowed P per op */
  int32_t b_cap;                /* min over ops of b_max     */
  int32_t r_cap;
} OpscModelSpec;

/* Greedy operator-level planner knobs (AutoscaleParams, autoscaler.py:102-131).
 * The uniform reseed (autoscaler.py:357-367, 492-500) uses `model`. */
typedef struct OpscGreedySpec {
  int32_t n_p[OPSC_MAX_OPS];
  int32_t p_vals[OPSC_MAX_OPS][OPSC_MAX_P]; /* params.parallelism_for(op): sorted, duplicates kept */
  int32_t b_max[OPSC_MAX_OPS];
  int32_t r_cap;
  int32_t max_iterations;
  int32_t prune_excess_replicas;
  OpscModelSpec model;
} OpscGreedySpec;

/* One accepted greedy move (ScalingPlan.trace entry). */
typedef struct OpscTraceEntry {
  double latency;     /* trial latency (reseed: unused)        */
  int32_t objective;  /* objective after the move               */
  int16_t to_r, to_b, to_p;
  int8_t op;          /* lex rank; -1 for reseed_uniform        */
  uint8_t action;     /* OPSC_ACT_*                              */
  int32_t reserved;   /* zero (explicit padding to 24 bytes)     */
} OpscTraceEntry;

/* Default-stream placement + energy inputs (placement.py:465-491, metrics.py:34-47). */
typedef struct OpscPlaceSpec {
  int32_t n_devices;     /* fleet size; devices in sorted-id order */
  int32_t uniform_cap;   /* 1: every device has mem_cap[0] */
  double alpha;
  double beta;
  const double* mem_cap; /* [n_devices] host or device pointer (see entry point) */
} OpscPlaceSpec;

/* Per-window planning inputs, structure of arrays (workload.py:38-54). */
typedef struct OpscWindows {
  int32_t n;
  const double* qps;
  const int32_t* seq_len;
  const uint8_t* phase; /* 0 prefill, 1 decode */
  const double* slo;
  const double* eps;
} OpscWindows;

/* Per-window decided plan, structure of arrays (autoscaler.py:76-99). */
typedef struct OpscDecisions {
  int64_t* key;       /* [W] best packed key (cost << 40 | lex index) or OPSC_KEY_INFEASIBLE */
  int16_t* cfg;       /* [W][n_ops][3] P, R, B (lex-rank order)              */
  uint8_t* feasible;  /* [W]                                                 */
  uint32_t* status;   /* [W] OPSC_W_* bits                                   */
  double* latency;    /* [W] iteration_latency (critical path)               */
  int32_t* objective; /* [W] sum P*R                                         */
  int8_t* path;       /* [W][n_ops] critical path, lex ranks, -1 padded      */
  double* pred;       /* [W][n_ops][7] PredictedSojourn fields               */
  uint8_t* stable;    /* [W][n_ops]                                          */
  double* energy;     /* [W] request_energy under default-stream placement   */
  double* memory;     /* [W] provisioned_memory under default-stream placement */
  int32_t* devices;   /* [W] devices_used under default-stream placement     */
  int32_t trace_cap;  /* entries per window in `trace` (operator mode)       */
  int32_t* trace_len; /* [W] number of moves (may exceed trace_cap)          */
  OpscTraceEntry* trace; /* [W][trace_cap]; entries >= trace_len[w] are unspecified */
} OpscDecisions;

/* ---- library info ---- */
OPSC_API int opsc_abi_version(void);
OPSC_API const char* opsc_status_string(int status);
OPSC_API int opsc_device_count(int* count);

/* ---- device-pointer entry points (stream passed as cudaStream_t cast to void*) ---- */

/* menu_w: [W][grid.menu_off[n_ops]] critical-path weight of every menu entry
 * ((W+T/B)+C)*layers, +inf when unstable. status |= ZERO_DIVISION / UNSTABLE_ROUNDING. */
OPSC_API int opsc_menu_build(const OpscDag* dag, const OpscGrid* grid, OpscWindows win,
                    double* menu_w, uint32_t* status, void* stream);

/* status |= OPSC_W_NO_STABLE_PARAMS when some op has no (P, B) in AutoscaleParams
 * whose strict-stability replica floor is <= r_cap. */
OPSC_API int opsc_stability_check(const OpscDag* dag, const OpscGrid* grid, OpscWindows win,
                         uint32_t* status, void* stream);

/* Diagnostic (not on the planning path): per window, ADDS to count_out the
 * number of candidates whose canonical critical-path latency is finite and
 * within band_ulps ulps of slo -- the only ones whose feasibility could
 * depend on the reference's frozenset-ordered sum() (autoscaler.py:792-794).
 * count_out must be zeroed by the caller. */
OPSC_API int opsc_compose_boundary(const OpscDag* dag, const OpscGrid* grid, OpscWindows win,
                                   const double* menu_w, double band_ulps, int64_t* count_out, void* stream);

/* Opt-in summation-order certificate of brute-force decisions
 * (autoscaler.py:765, 792-796: the reference's leaf sums path weights over a
 * frozenset, so its order depends on PYTHONHASHSEED). Runs the compose argmin
 * twice more with slo -/+ band_ulps ulps and ORs OPSC_W_ORDER_SENSITIVE into
 * status where the two keys differ. Windows left unflagged decide identically
 * under every summation order whose error stays inside the band.
 * workspace: opsc_certify_workspace(win.n) bytes of device memory. */
OPSC_API size_t opsc_certify_workspace(int32_t n_windows);
OPSC_API int opsc_certify_order(const OpscDag* dag, const OpscGrid* grid, OpscWindows win,
                                const double* menu_w, double band_ulps, void* workspace,
                                size_t workspace_bytes, uint32_t* status, void* stream);

/* Exhaustive compose + SLO mask + lexicographic argmin over the shard
 * [shard/n_shards] of every window's candidate space. key_out must be
 * initialised to OPSC_KEY_INFEASIBLE (opsc_fill_keys); results are min-merged. */
OPSC_API int opsc_compose_argmin(const OpscDag* dag, const OpscGrid* grid, OpscWindows win,
                        const double* menu_w, int32_t shard, int32_t n_shards,
                        int64_t* key_out, void* stream);

OPSC_API int opsc_fill_keys(int64_t* key, int32_t n, void* stream);

/* Per-window prologue: status = OPSC_W_IDLE for qps <= 0 (cli.py:138-144)
 * else 0; key = OPSC_KEY_INFEASIBLE; feasible = 0. key/feasible may be NULL. */
OPSC_API int opsc_init_windows(OpscWindows win, uint32_t* status, int64_t* key, uint8_t* feasible,
                               void* stream);

/* fb_entry: [W][n_ops] argmin over finite menu weights of (weight, entry), -1 if none. */
OPSC_API int opsc_menu_fallback(const OpscDag* dag, const OpscGrid* grid, int32_t n_windows,
                       const double* menu_w, int32_t* fb_entry, void* stream);

/* key (+ fallback) -> cfg[W][n_ops][3], feasible, status |= NO_STABLE_BOUNDS. */
OPSC_API int opsc_decode_decisions(const OpscDag* dag, const OpscGrid* grid, int32_t n_windows,
                          const int64_t* key, const int32_t* fb_entry,
                          int16_t* cfg, uint8_t* feasible, uint32_t* status, void* stream);

/* model_level_autoscale per window -> cfg, feasible, status |= NO_STABLE_MODEL. */
OPSC_API int opsc_model_grid(const OpscDag* dag, const OpscModelSpec* spec, OpscWindows win,
                    int16_t* cfg, uint8_t* feasible, uint32_t* status, void* stream);

/* cfg -> predicted, latency, path, objective, energy, memory, devices.
 * config_order: 0 = lex-rank order (brute force), 1 = node order (model level).
 * place.mem_cap must be a device pointer here. */
OPSC_API int opsc_materialize(const OpscDag* dag, OpscWindows win, int32_t config_order,
                     const OpscPlaceSpec* place, OpscDecisions out, void* stream);

/* Fused forms of the per-window brute-force chain (fewer launches on the
 * W=1 decision path; same bits as the separate entry points):
 *   opsc_menu_stability    = opsc_menu_build + opsc_stability_check
 *                            (autoscaler.py:743-757 and its init_configs pre-check :254-294, 771);
 *   opsc_decode_materialize = opsc_menu_fallback + opsc_decode_decisions + opsc_materialize
 *                            with config_order 0 (autoscaler.py:828-847, 196-247, metrics.py:84-132). */
OPSC_API int opsc_menu_stability(const OpscDag* dag, const OpscGrid* grid, OpscWindows win, double* menu_w,
                                 uint32_t* status, void* stream);
OPSC_API int opsc_decode_materialize(const OpscDag* dag, const OpscGrid* grid, OpscWindows win,
                                     const int64_t* key, const double* menu_w, const OpscPlaceSpec* place,
                                     OpscDecisions out, void* stream);

/* greedy_autoscale per window (autoscaler.py:334-589): init_configs, the
 * bottleneck up/downscale loop, uniform reseed + prune, headroom restore and
 * the optional prune pass. uniform_cfg / uniform_feasible / uniform_status are
 * opsc_model_grid's outputs for the same windows (_uniform_optimum, :492-500).
 * Writes out.cfg (lex-rank order), out.feasible, out.status
 * (OPSC_W_NO_STABLE_INIT), out.trace_len and out.trace. */
OPSC_API int opsc_greedy(const OpscDag* dag, const OpscGreedySpec* spec, OpscWindows win,
                         const int16_t* uniform_cfg, const uint8_t* uniform_feasible,
                         const uint32_t* uniform_status, OpscDecisions out, void* stream);

/* The same planner split in two launches: phase 1 = init_configs + first
 * greedy loop (needs no model-level input), phase 2 = uniform reseed,
 * headroom restore, prune, outputs. Lets the caller run opsc_model_grid
 * concurrently with phase 1. `state` holds opsc_greedy_state_bytes(W) bytes. */
OPSC_API size_t opsc_greedy_state_bytes(int32_t n_windows);
OPSC_API int opsc_greedy_phase(const OpscDag* dag, const OpscGreedySpec* spec, OpscWindows win,
                               int32_t phase, void* state, const int16_t* uniform_cfg,
                               const uint8_t* uniform_feasible, const uint32_t* uniform_status,
                               OpscDecisions out, void* stream);

/* Small-batch model level: every (B, R) point of every window is tabulated in
 * parallel (same arithmetic as the in-warp probes, so the same bits) and the
 * reference's probe/bisect then walks the table. Needs
 * opsc_model_table_bytes(spec, W, n_ops) bytes of device workspace. */
OPSC_API size_t opsc_model_table_bytes(const OpscModelSpec* spec, int32_t n_windows, int32_t n_ops);
OPSC_API int opsc_model_grid_table(const OpscDag* dag, const OpscModelSpec* spec, OpscWindows win,
                                   int16_t* cfg, uint8_t* feasible, uint32_t* status,
                                   void* workspace, size_t workspace_bytes, void* stream);

/* ---- shared (interference-aware) placement, Alg. 2 (placement.py:399-462) ---- */

/* Fleet (DeviceSpec, devices in sorted-id order), PlacementParams,
 * InterferenceParams and EnergyParams (placement.py:46-55, 112-117;
 * perfmodel.py:67-76; metrics.py:34-47). */
typedef struct OpscPlaceShared {
  int32_t n_devices;
  const double* mem_cap;     /* [n_devices] */
  const double* compute_cap; /* [n_devices] */
  double slo;                /* PlacementParams.slo */
  double slack_weight_mem;
  double slack_weight_compute;
  double max_sm_load;
  double theta;              /* InterferenceParams */
  double exponent;           /* 1.0 / 2.0 / 0.5 bit-exact; other values use pow() */
  double alpha;              /* EnergyParams */
  double beta;
  int32_t flags;             /* OPSC_PLACE_* */
} OpscPlaceShared;

/* OpscPlaceShared.flags */
#define OPSC_PLACE_DEFAULT_STREAM 0x1 /* default_stream_place (placement.py:465-491): every extra
                                         replica on a dedicated device, no probing */
#define OPSC_PLACE_WINDOW_SLO 0x2     /* PlacementParams.slo per window = OpscWindows.slo[w]
                                         (runner.run_point, runner.py:70), else .slo */

/* Placement of each window's plan; per-window capacities. */
typedef struct OpscPlacement {
  int32_t cap_assign;    /* assignment slots per window (>= sum of R)        */
  int32_t cap_dev;       /* device-load slots per window                     */
  int32_t* n_assign;     /* [W]                                              */
  int32_t* devices_used; /* [W]                                              */
  uint8_t* feasible;     /* [W] recomputed latency <= slo                    */
  uint32_t* status;      /* [W] OPSC_W_FLEET_EXHAUSTED / INFEASIBLE_PLACEMENT; when set, the
                            window's other outputs are unspecified */
  double* latency;       /* [W] recomputed_latency                           */
  double* energy;        /* [W] request_energy under this placement          */
  double* memory;        /* [W] provisioned_memory                           */
  int8_t* a_op;          /* [W][cap_assign] lex rank                         */
  int16_t* a_replica;
  int32_t* a_device;     /* sorted-id device index                          */
  int16_t* a_share;      /* sm_share percent                                 */
  double* a_latency;     /* interference_adjusted_latency                    */
  double* d_mem;         /* [W][cap_dev] DeviceLoad.mem_used                 */
  double* d_sm;          /* DeviceLoad.sm_demand (standing load)             */
  double* d_energy;      /* fill_device_energy                              */
} OpscPlacement;

/* place() + request_energy + fill_device_energy + provisioned_memory for the
 * decided plan of every window (cfg [W][n][3] lex-rank order, plan feasible
 * flags; config_order as in opsc_materialize). Windows whose plan is not
 * feasible or idle are skipped (n_assign = 0). */
OPSC_API size_t opsc_place_shared_workspace(int32_t n_windows, int32_t cap_assign, int32_t cap_dev,
                                            int32_t n_ops);
OPSC_API int opsc_place_shared(const OpscDag* dag, const OpscPlaceShared* fleet, OpscWindows win,
                               const int16_t* cfg, const uint8_t* plan_feasible,
                               int32_t config_order, OpscPlacement out, void* workspace,
                               size_t workspace_bytes, void* stream);

/* ---- trace windowing (workload.py:107-158) ---- */

/* A request trace as structure of arrays (RequestRecord, workload.py:31-35). */
typedef struct OpscTraceRecords {
  int64_t n;
  const double* arrival;     /* seconds, >= 0, any order */
  const int32_t* input_len;  /* >= 1 */
  const int32_t* output_len; /* >= 0 */
} OpscTraceRecords;

/* Bytes of device workspace opsc_windowize needs. */
OPSC_API size_t opsc_windowize_workspace(int64_t n_records, int32_t max_windows);

/* windowize(records, window_len, quantile) on the device: n_windows =
 * max(1, ceil(horizon/len + 1e-12)), record -> min(int(t/len), n-1); per
 * window prefill qps = count/len, prefill seq_len = max(1, q-"higher"
 * quantile of input lengths), decode qps = sum(output)/len (decode seq_len is
 * 1). Empty windows give qps 0 and seq_len 1. `n_windows` is a device int32;
 * if it exceeds max_windows it is written but no window is produced and the
 * call returns OPSC_ERR_ARG at the next synchronisation of the host path. */
OPSC_API int opsc_windowize(OpscTraceRecords rec, double window_len, double quantile,
                            int32_t max_windows, int32_t* n_windows, double* prefill_qps,
                            int32_t* prefill_len, double* decode_qps, void* workspace,
                            size_t workspace_bytes, void* stream);

/* ---- host-buffer path: one call plans a batch of windows end to end ---- */
typedef struct OpscContext OpscContext;

OPSC_API int opsc_ctx_create(int32_t device, int32_t max_windows, OpscContext** out);
OPSC_API int opsc_ctx_destroy(OpscContext* ctx);

/* win / out / place.mem_cap are HOST pointers. Copies in, runs the mode's
 * kernels on the context stream, copies out, synchronises. */
OPSC_API int opsc_plan_windows_host(OpscContext* ctx, int32_t mode, const OpscDag* dag,
                           const OpscGrid* grid, const OpscModelSpec* model,
                           const OpscGreedySpec* greedy, const OpscPlaceSpec* place,
                           OpscWindows win, OpscDecisions out);

/* Number of kernels the last opsc_plan_windows_host call launched. */
OPSC_API int opsc_ctx_last_launches(const OpscContext* ctx, int32_t* launches);

/* Device time (CUDA events on the context stream) of the last
 * opsc_plan_windows_host call, from its first host->device copy to its last
 * device->host copy. OPSC_ERR_ARG before any call. */
OPSC_API int opsc_ctx_last_ms(OpscContext* ctx, float* ms);

/* ---- measurement helper: FP64 add throughput microbenchmark ----
 * Runs `iters` dependent-chain DADD/DSETP pairs per thread on a full grid;
 * writes elapsed milliseconds and the executed FP64 op count. */
OPSC_API int opsc_fp64_peak(int32_t iters, float* ms, double* fp64_ops, void* stream);

/* ---- multi-GPU key merge over NVLink peer memory ----
 * The MIN merge of per-window keys (dist.merge_keys' NCCL all-reduce,
 * SURVEY §8(e)) fused into the compose kernel: every CTA's atomicMin goes
 * straight to the key buffer of every rank (peer pointers mapped with CUDA
 * IPC), then one device-side flag barrier orders the merge before decode.
 * Buffers are double-buffered by the caller (paper_2511_02248_b200/dist.py
 * PeerMerge): the buffer for step s+1 is reset before the barrier of step s. */
#define OPSC_MAX_PEERS 8

/* cudaMalloc + zero + cudaIpcGetMemHandle; handle = 64 bytes */
OPSC_API int opsc_ipc_alloc(size_t bytes, void** dptr, void* handle);
/* cudaIpcOpenMemHandle (lazy peer access) of a handle from another process */
OPSC_API int opsc_ipc_open(const void* handle, void** dptr);
OPSC_API int opsc_ipc_close(void* dptr);
OPSC_API int opsc_ipc_free(void* dptr);

/* opsc_compose_argmin with the merge fused: peer_keys[0..n_peers) are the
 * [W] int64 key buffers of every rank (this rank's included). */
OPSC_API int opsc_compose_argmin_peers(const OpscDag* dag, const OpscGrid* grid, OpscWindows win,
                                       const double* menu_w, int32_t shard, int32_t n_shards,
                                       int64_t* const* peer_keys, int32_t n_peers, void* stream);

/* Stream-ordered device copy of n int64 keys (merged keys -> decisions). */
OPSC_API int opsc_copy_keys(int64_t* dst, const int64_t* src, int32_t n, void* stream);

/* Device flag barrier over n ranks: flags[p] is rank p's [n] uint32 arrival
 * array (this rank's own pointer at index `rank`); `epoch` increases by one
 * per barrier. Release/acquire at system scope; a wait longer than
 * timeout_ms sets *err = 1 instead of hanging. */
OPSC_API int opsc_peer_barrier(uint32_t* const* flags, int32_t rank, int32_t n, uint32_t epoch,
                               int32_t timeout_ms, int32_t* err, void* stream);

/* Diagnostic: out[i] = excess ** exponent as the placement kernel evaluates
 * it inside interference_factor (perfmodel.py:174-187): exact for exponents
 * 1, 2 and 0.5, otherwise rounded to nearest from a double-double
 * evaluation. Device pointers, n >= 0. */
OPSC_API int opsc_interference_pow(const double* x, const double* e, double* out, int64_t n, void* stream);

/* Candidate-loop probe: the compose inner loop on synthetic register menus
 * (kind 1: DADD + DSETP + select per candidate, kind 2: DSETP + select).
 * Gives the instruction-mix ceiling of the compose kernel on this GPU. */
OPSC_API int opsc_candidate_probe(int32_t kind, int32_t iters, float* ms, double* candidates,
                                  void* stream);

#ifdef __cplusplus
}
#endif
#endif /* OPSCALE_B200_H */
