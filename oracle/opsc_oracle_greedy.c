/*
 * opsc_oracle_greedy.c -- CPU restatement of greedy_autoscale
 * (reference autoscaler.py:254-589). TEST INFRASTRUCTURE (see opsc_oracle.h).
 *
 * Pinned by tests/golden/greedy.json (reference outputs, bit-exact floats).
 * Every move set, selection key and loop guard follows the reference code:
 *   init_configs          :254-294
 *   _bottleneck           :301-303
 *   _upscale_moves        :306-317 (distinct (B, P) with R+1)
 *   _downscale_moves      :320-331 (distinct (B >= b, P) with R-1)
 *   greedy_autoscale      :334-380
 *   _greedy_loop          :383-489
 *   _restore_headroom     :503-559
 *   _prune_pass           :562-589
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "opsc_oracle.h"

typedef struct { int p, r, b; } GCfg;

typedef struct {
  double sojourn[OPSC_MAX_OPS];
  double weight[OPSC_MAX_OPS];
  int stable;
  double latency;
  int8_t path[OPSC_MAX_OPS];
} GEval;

typedef struct {
  const OpscDag* d;
  const OpscGreedySpec* s;
  double qps, slo, eps;
  int L, ph;
  uint32_t st;
  int init_fail; /* 1 + node-order position of the op init_configs could not seed */
  OpscTraceEntry* trace;
  int32_t cap, len;
  int np_distinct[OPSC_MAX_OPS];
  int p_distinct[OPSC_MAX_OPS][OPSC_MAX_P];
} G;

static void g_eval(G* g, const GCfg* c, GEval* e) {
  const OpscDag* d = g->d;
  e->stable = 1;
  for (int v = 0; v < d->n_ops; ++v) {
    double o[7];
    int s = orc_predict(d, g->qps, g->L, g->ph, v, c[v].p, c[v].r, c[v].b, o, &g->st);
    e->stable &= s;
    e->sojourn[v] = o[4] + o[5];
    e->weight[v] = ((o[4] + o[5]) + o[6]) * (double)d->layer_count[v];
  }
  if (e->stable) {
    e->latency = orc_critical_path(d, e->weight, e->path);
  } else {
    e->latency = INFINITY;
    for (int v = 0; v < d->n_ops; ++v) e->path[v] = -1;
  }
}

static int objective(const G* g, const GCfg* c) {
  int o = 0;
  for (int v = 0; v < g->d->n_ops; ++v) o += c[v].p * c[v].r;
  return o;
}

/* largest sojourn on the critical path; ties to the smallest id */
static int bottleneck(const G* g, const GEval* e) {
  int best = -1;
  for (int i = 0; i < g->d->n_ops && e->path[i] >= 0; ++i) {
    int v = e->path[i];
    if (best < 0 || e->sojourn[v] > e->sojourn[best] ||
        (e->sojourn[v] == e->sojourn[best] && v < best))
      best = v;
  }
  return best;
}

static void push_trace(G* g, int action, int op, const GCfg* to, double lat, int obj) {
  if (g->len < g->cap) {
    OpscTraceEntry* t = &g->trace[g->len];
    t->latency = lat;
    t->objective = obj;
    t->to_r = (int16_t)(to ? to->r : 0);
    t->to_b = (int16_t)(to ? to->b : 0);
    t->to_p = (int16_t)(to ? to->p : 0);
    t->op = (int8_t)op;
    t->action = (uint8_t)action;
    t->reserved = 0;
  }
  g->len++;
}

/* efficiency = reduction / max(obj_trial - base_obj, 1e-9) (Python max(int, float)) */
static double efficiency(double cur_lat, double lat, int dobj) {
  double cost = dobj >= 1 ? (double)dobj : 1e-9;
  return (cur_lat - lat) / cost;
}

typedef struct {
  int have;
  double k0, k1;  /* float keys */
  int k2, b, p;   /* int keys */
  GCfg to;
  double lat;
} Best;

/* lexicographic tuple comparison of (k0, k1, k2, b, p) */
static int key_less(double a0, double a1, int a2, int ab, int ap, const Best* y) {
  if (a0 != y->k0) return a0 < y->k0;
  if (a1 != y->k1) return a1 < y->k1;
  if (a2 != y->k2) return a2 < y->k2;
  if (ab != y->b) return ab < y->b;
  return ap < y->p;
}

static void consider(Best* x, double k0, double k1, int k2, int b, int p, GCfg to, double lat) {
  if (!x->have || key_less(k0, k1, k2, b, p, x)) {
    x->have = 1; x->k0 = k0; x->k1 = k1; x->k2 = k2; x->b = b; x->p = p; x->to = to; x->lat = lat;
  }
}

/* One upscale step at the bottleneck (greedy loop when `headroom` == 0,
 * _restore_headroom otherwise). Returns 1 if a move was applied. */
static int upscale_step(G* g, GCfg* c, GEval* e, double target, double fallback_bound, int headroom) {
  const int op = bottleneck(g, e);
  const GCfg cur = c[op];
  if (cur.r + 1 > g->s->r_cap) return 0;
  const int base_obj = objective(g, c);
  Best ach = {0}, ach2 = {0}, imp = {0};
  GCfg trial[OPSC_MAX_OPS];
  memcpy(trial, c, sizeof(GCfg) * g->d->n_ops);
  for (int b = 1; b <= g->s->b_max[op]; ++b) {
    for (int pi = 0; pi < g->np_distinct[op]; ++pi) {
      const int p = g->p_distinct[op][pi];
      GCfg to = {p, cur.r + 1, b};
      trial[op] = to;
      GEval te;
      g_eval(g, trial, &te);
      if (!te.stable) continue;
      const int obj = base_obj - cur.p * cur.r + p * (cur.r + 1);
      if (te.latency <= target) consider(&ach, (double)obj, te.latency, 0, b, p, to, te.latency);
      if (!headroom && te.latency <= fallback_bound)
        consider(&ach2, (double)obj, te.latency, 0, b, p, to, te.latency);
      const int improving = headroom ? te.latency < e->latency - 1e-9 * g->slo : te.latency < e->latency;
      if (improving) {
        double eff = efficiency(e->latency, te.latency, obj - base_obj);
        if (headroom) consider(&imp, -eff, te.latency, 0, b, p, to, te.latency);
        else consider(&imp, -eff, te.latency, obj, b, p, to, te.latency);
      }
    }
  }
  const Best* pick = ach.have ? &ach : (!headroom && ach2.have) ? &ach2 : imp.have ? &imp : NULL;
  if (!pick) return 0;
  c[op] = pick->to;
  g_eval(g, c, e);
  push_trace(g, headroom ? OPSC_ACT_HEADROOM : OPSC_ACT_UPSCALE, op, &pick->to, e->latency,
             objective(g, c));
  return 1;
}

static int downscale_step(G* g, GCfg* c, GEval* e) {
  const int op = bottleneck(g, e);
  const GCfg cur = c[op];
  if (cur.r - 1 < 1) return 0;
  const int base_obj = objective(g, c);
  const double bound = g->slo - g->eps;
  Best best = {0};
  GCfg trial[OPSC_MAX_OPS];
  memcpy(trial, c, sizeof(GCfg) * g->d->n_ops);
  for (int b = cur.b; b <= g->s->b_max[op]; ++b) {
    for (int pi = 0; pi < g->np_distinct[op]; ++pi) {
      const int p = g->p_distinct[op][pi];
      GCfg to = {p, cur.r - 1, b};
      trial[op] = to;
      GEval te;
      g_eval(g, trial, &te);
      if (!te.stable || te.latency > bound) continue;
      const int obj = base_obj - cur.p * cur.r + p * (cur.r - 1);
      if (obj >= base_obj) continue;
      consider(&best, (double)obj, 0.0, 0, b, p, to, te.latency);
    }
  }
  if (!best.have) return 0;
  c[op] = best.to;
  g_eval(g, c, e);
  push_trace(g, OPSC_ACT_DOWNSCALE, op, &best.to, e->latency, objective(g, c));
  return 1;
}

static void greedy_loop(G* g, GCfg* c, GEval* e) {
  const double slo = g->slo, eps = g->eps;
  for (int it = 0; it < g->s->max_iterations; ++it) {
    if (e->latency > slo) {
      if (!upscale_step(g, c, e, slo - eps, slo, 0)) break;
    } else if (e->latency <= slo - eps) {
      if (!downscale_step(g, c, e)) break;
    } else {
      break;
    }
  }
}

static void prune_pass(G* g, GCfg* c, GEval* e) {
  const double target = g->slo - g->eps;
  int changed = 1;
  while (changed) {
    changed = 0;
    for (int v = 0; v < g->d->n_ops; ++v) {
      if (c[v].r <= 1) continue;
      GCfg trial[OPSC_MAX_OPS];
      memcpy(trial, c, sizeof(GCfg) * g->d->n_ops);
      trial[v].r -= 1;
      GEval te;
      g_eval(g, trial, &te);
      if (te.stable && te.latency <= target) {
        memcpy(c, trial, sizeof(GCfg) * g->d->n_ops);
        *e = te;
        push_trace(g, OPSC_ACT_PRUNE, v, &c[v], e->latency, objective(g, c));
        changed = 1;
      }
    }
  }
}

/* init_configs: per op (node order) the first P with a stable B, argmin
 * sojourn (strict <, lowest B), R at the strict-stability floor. */
static int init_configs(G* g, GCfg* c) {
  const OpscDag* d = g->d;
  for (int i = 0; i < d->n_ops; ++i) {
    const int v = d->node_order[i];
    int chosen = 0;
    for (int pi = 0; pi < g->s->n_p[v] && !chosen; ++pi) {
      const int p = g->s->p_vals[v][pi];
      int have = 0, bb = 0, br = 0;
      double bs = 0.0;
      for (int b = 1; b <= g->s->b_max[v]; ++b) {
        double t = orc_op_latency(d->c0[g->ph][v], d->c1[g->ph][v], d->c2[g->ph][v], d->eta[v], b,
                                  g->L, p);
        double tl = t * (double)d->layer_count[v];
        if (tl == 0.0) g->st |= OPSC_W_ZERO_DIVISION;
        double mu = 1.0 / tl, lam = g->qps / (double)b;
        int r = orc_strict_min_replicas(lam, mu, g->s->r_cap);
        if (r < 0) continue;
        double util = lam / ((double)r * mu);
        if (util >= 1.0 || util <= 0.0) g->st |= OPSC_W_UNSTABLE_ROUNDING;
        double soj = orc_expected_wait(lam, mu, r) + t / (double)b;
        if (!have || soj < bs) { have = 1; bs = soj; bb = b; br = r; }
      }
      if (have) {
        c[v].p = p; c[v].r = br; c[v].b = bb;
        chosen = 1;
      }
    }
    if (!chosen) {
      g->init_fail = i + 1;
      return 0;
    }
  }
  return 1;
}

int orc_greedy(const OpscDag* d, const OpscGreedySpec* s, OpscWindows win, const int16_t* ucfg,
               const uint8_t* ufeas, const uint32_t* ustatus, OpscDecisions out, int32_t n_threads) {
  const int n = d->n_ops;
#pragma omp parallel for num_threads(n_threads) schedule(dynamic, 1)
  for (int w = 0; w < win.n; ++w) {
    out.feasible[w] = 0;
    out.trace_len[w] = 0;
    if (!(win.qps[w] > 0.0)) continue;
    G g;
    memset(&g, 0, sizeof(g));
    g.d = d; g.s = s;
    g.qps = win.qps[w]; g.slo = win.slo[w]; g.eps = win.eps[w];
    g.L = win.seq_len[w]; g.ph = win.phase[w];
    g.trace = out.trace + (size_t)w * out.trace_cap;
    g.cap = out.trace_cap;
    for (int v = 0; v < n; ++v) {
      int k = 0;
      for (int i = 0; i < s->n_p[v]; ++i) {
        int dup = 0;
        for (int j = 0; j < k; ++j) dup |= g.p_distinct[v][j] == s->p_vals[v][i];
        if (!dup) g.p_distinct[v][k++] = s->p_vals[v][i];
      }
      g.np_distinct[v] = k;
    }
    GCfg c[OPSC_MAX_OPS];
    if (!init_configs(&g, c)) {
      out.status[w] |= g.st | OPSC_W_NO_STABLE_INIT | ((uint32_t)g.init_fail << OPSC_W_INIT_OP_SHIFT);
      continue;
    }
    GEval e;
    g_eval(&g, c, &e);
    greedy_loop(&g, c, &e);
    /* uniform reseed (model_level_autoscale; NoStableConfig -> None) */
    const uint32_t us = ustatus[w];
    g.st |= us & (OPSC_W_ZERO_DIVISION | OPSC_W_UNSTABLE_ROUNDING);
    if (!(us & OPSC_W_NO_STABLE_MODEL) && ufeas[w]) {
      GCfg u[OPSC_MAX_OPS];
      for (int v = 0; v < n; ++v) {
        u[v].p = ucfg[(w * n + v) * 3];
        u[v].r = ucfg[(w * n + v) * 3 + 1];
        u[v].b = ucfg[(w * n + v) * 3 + 2];
      }
      if (objective(&g, u) < objective(&g, c)) {
        push_trace(&g, OPSC_ACT_RESEED, -1, NULL, 0.0, objective(&g, u));
        GEval ue;
        g_eval(&g, u, &ue);
        prune_pass(&g, u, &ue);
        greedy_loop(&g, u, &ue);
        if (objective(&g, u) < objective(&g, c)) {
          memcpy(c, u, sizeof(c));
          e = ue;
        }
      }
    }
    if (g.eps > 0 && e.latency <= g.slo) {
      while (e.latency > g.slo - g.eps) {
        if (!upscale_step(&g, c, &e, g.slo - g.eps, g.slo, 1)) break;
      }
    }
    if (s->prune_excess_replicas && e.latency <= g.slo) prune_pass(&g, c, &e);
    out.feasible[w] = (uint8_t)(e.stable && e.latency <= g.slo);
    for (int v = 0; v < n; ++v) {
      out.cfg[(w * n + v) * 3] = (int16_t)c[v].p;
      out.cfg[(w * n + v) * 3 + 1] = (int16_t)c[v].r;
      out.cfg[(w * n + v) * 3 + 2] = (int16_t)c[v].b;
    }
    out.trace_len[w] = g.len;
    if (g.cap > 0 && g.len > g.cap) g.st |= OPSC_W_TRACE_TRUNCATED;
    out.status[w] |= g.st;
  }
  return OPSC_OK;
}
