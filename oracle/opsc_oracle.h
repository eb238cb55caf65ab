/*
 * opsc_oracle.h -- CPU restatement of the reference planner's search path.
 *
 * TEST INFRASTRUCTURE ONLY. This is the checker the parity tests, smoke()
 * and bench.py's cpu_baseline / --impl reference legs compare against; the
 * product path (paper_2511_02248_b200/) never links or calls it.
 *
 * Parity pinned against the reference: the JSON vectors in tests/golden/ were produced by
 * running /root/reference's own functions (tests/golden/make_golden.py) and
 * tests/test_oracle_golden.py checks every function here bit-exactly
 * against them.
 *
 * Every routine mirrors the ABI of include/opscale_b200.h (same structs,
 * same outputs) with the stream argument replaced by a thread count.
 */
#ifndef OPSC_ORACLE_H
#define OPSC_ORACLE_H

#include "../include/opscale_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* scalar primitives (perfmodel.py, queueing.py) */
double orc_op_latency(double c0, double c1, double c2, double eta, int64_t b, int64_t l, int64_t p);
double orc_comm_time(double v0, double v1, int64_t b, int64_t l, double bw);
double orc_op_memory(double weight_mem, double m0, double m1, int64_t b, int64_t l, int64_t p);
double orc_erlang_c(int32_t r, double rho);
double orc_expected_wait(double lam, double mu, int32_t r);
int32_t orc_strict_min_replicas(double lam, double mu, int32_t r_cap); /* -1 = None */
double orc_py_sum(const double* x, int32_t n); /* CPython 3.12 builtin sum() over floats */

/* PredictedSojourn of op v (lex rank) under (p, r, b); returns stable flag. */
int32_t orc_predict(const OpscDag* dag, double qps, int32_t seq_len, int32_t phase,
                    int32_t v, int32_t p, int32_t r, int32_t b, double* out7,
                    uint32_t* status);

/* critical_path_latency over per-op weights (lex-rank indexed). */
double orc_critical_path(const OpscDag* dag, const double* weight, int8_t* path);

int orc_menu_build(const OpscDag* dag, const OpscGrid* grid, OpscWindows win,
                   double* menu_w, uint32_t* status, int32_t n_threads);
int orc_stability_check(const OpscDag* dag, const OpscGrid* grid, OpscWindows win,
                        uint32_t* status, int32_t n_threads);
int orc_compose_argmin(const OpscDag* dag, const OpscGrid* grid, OpscWindows win,
                       const double* menu_w, int32_t shard, int32_t n_shards,
                       int64_t* key_out, int32_t n_threads);
int orc_menu_fallback(const OpscDag* dag, const OpscGrid* grid, int32_t n_windows,
                      const double* menu_w, int32_t* fb_entry);
int orc_decode_decisions(const OpscDag* dag, const OpscGrid* grid, int32_t n_windows,
                         const int64_t* key, const int32_t* fb_entry, int16_t* cfg,
                         uint8_t* feasible, uint32_t* status);
int orc_model_grid(const OpscDag* dag, const OpscModelSpec* spec, OpscWindows win,
                   int16_t* cfg, uint8_t* feasible, uint32_t* status, int32_t n_threads);
int orc_materialize(const OpscDag* dag, OpscWindows win, int32_t config_order,
                    const OpscPlaceSpec* place, OpscDecisions out, int32_t n_threads);

/* greedy_autoscale (opsc_oracle_greedy.c); uniform_* = orc_model_grid outputs. */
int orc_greedy(const OpscDag* dag, const OpscGreedySpec* spec, OpscWindows win,
               const int16_t* uniform_cfg, const uint8_t* uniform_feasible,
               const uint32_t* uniform_status, OpscDecisions out, int32_t n_threads);

/* shared placement + placement metrics (opsc_oracle_place.c) */
int orc_place_shared(const OpscDag* dag, const OpscPlaceShared* fleet, OpscWindows win,
                     const int16_t* cfg, const uint8_t* plan_feasible, int32_t config_order,
                     OpscPlacement out, int32_t n_threads);

/* windowize (workload.py:107-158); returns n_windows or -1 if > max_windows. */
int32_t orc_windowize(OpscTraceRecords rec, double window_len, double quantile,
                      int32_t max_windows, double* prefill_qps, int32_t* prefill_len,
                      double* decode_qps);

/* Whole pipeline of one planning mode over a batch of windows. */
int orc_plan_windows(int32_t mode, const OpscDag* dag, const OpscGrid* grid,
                     const OpscModelSpec* model, const OpscGreedySpec* greedy,
                     const OpscPlaceSpec* place, OpscWindows win, OpscDecisions out,
                     int32_t n_threads);

#ifdef __cplusplus
}
#endif
#endif
