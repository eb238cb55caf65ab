/*
 * opsc_oracle_place.c -- CPU restatement of the reference's shared
 * (interference-aware) placement, Alg. 2, and the placement-dependent
 * metrics. TEST INFRASTRUCTURE (see opsc_oracle.h).
 *
 * Pinned by tests/golden/place.json (reference outputs, bit-exact floats):
 *   _deploy_base_instances   placement.py:358-385
 *   _extra_replicas          placement.py:388-396
 *   place                    placement.py:399-462
 *   _interference_per_replica placement.py:209-231 (+ interference_factor,
 *                            perfmodel.py:174-187)
 *   _adjusted_ops / latency  placement.py:245-284
 *   _finalize                placement.py:494-515
 *   weighted_slack           placement.py:338-351
 *   request_energy / fill_device_energy / provisioned_memory  metrics.py:84-132
 * Python's builtin sum() over floats is Neumaier-compensated (CPython 3.12);
 * every sum the reference takes with sum() is emulated as such.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "opsc_oracle.h"

typedef struct { double f, c; int started; } PS;
static void ps_add(PS* s, double x) {
  if (!s->started) { s->f = 0.0 + x; s->c = 0.0; s->started = 1; return; }
  double t = s->f + x;
  if (fabs(s->f) >= fabs(x)) s->c += (s->f - t) + x;
  else s->c += (x - t) + s->f;
  s->f = t;
}
static double ps_val(const PS* s) {
  if (!s->started) return 0.0;
  return (s->c != 0.0 && isfinite(s->c)) ? s->f + s->c : s->f;
}

typedef struct {
  int op, k, dev, group, share;
  double dem, mem, factor;
} Asg;

typedef struct {
  const OpscDag* d;
  const OpscPlaceShared* f;
  int n, L, ph;
  double qps, slo; /* PlacementParams.slo of this window */
  int p[OPSC_MAX_OPS], r[OPSC_MAX_OPS], b[OPSC_MAX_OPS];
  double T[OPSC_MAX_OPS], comm[OPSC_MAX_OPS], dem[OPSC_MAX_OPS], mem[OPSC_MAX_OPS];
  int order[OPSC_MAX_OPS]; /* plan.configs order */
  Asg* a;
  int na, cap;
  int used;
} PL;

static double pow_expo(double x, double e) {
  if (e == 1.0) return x;
  if (e == 2.0) return x * x;
  if (e == 0.5) return sqrt(x);
  return pow(x, e);
}

/* interference_factor(device_load, adding) (perfmodel.py:174-187) */
static double interference(const PL* s, double load, double adding) {
  double excess = load + adding - 1.0;
  if (excess <= 0.0) return 1.0;
  return 1.0 + s->f->theta * pow_expo(excess, s->f->exponent);
}

/* group maxima of device `dev` (insertion order), optionally with an extra
 * member; returns count; fills gid[] / gmax[] */
static int dev_groups(const PL* s, int dev, const Asg* extra, int* gid, double* gmax) {
  int ng = 0;
  for (int i = 0; i <= s->na; ++i) {
    const Asg* a = i < s->na ? &s->a[i] : extra;
    if (!a || a->dev != dev) continue;
    int j = 0;
    while (j < ng && gid[j] != a->group) ++j;
    if (j == ng) { gid[ng] = a->group; gmax[ng] = 0.0; ++ng; }
    gmax[j] = gmax[j] >= a->dem ? gmax[j] : a->dem; /* max(old, new) */
  }
  return ng;
}

static double dev_load(const PL* s, int dev, const Asg* extra) {
  int* gid = (int*)malloc(sizeof(int) * (s->na + 1));
  double* gmax = (double*)malloc(sizeof(double) * (s->na + 1));
  int ng = dev_groups(s, dev, extra, gid, gmax);
  PS t = {0, 0, 0};
  for (int j = 0; j < ng; ++j) ps_add(&t, gmax[j]);
  free(gid);
  free(gmax);
  return ps_val(&t);
}

static double dev_mem(const PL* s, int dev) {
  PS t = {0, 0, 0};
  for (int i = 0; i < s->na; ++i)
    if (s->a[i].dev == dev) ps_add(&t, s->a[i].mem);
  return ps_val(&t);
}

/* factors of all members of `dev` (+extra) -> out_f[assignment index], extra -> *extra_f */
static void dev_factors(const PL* s, int dev, const Asg* extra, double* out_f, double* extra_f) {
  int* gid = (int*)malloc(sizeof(int) * (s->na + 1));
  double* gmax = (double*)malloc(sizeof(double) * (s->na + 1));
  int ng = dev_groups(s, dev, extra, gid, gmax);
  PS t = {0, 0, 0};
  for (int j = 0; j < ng; ++j) ps_add(&t, gmax[j]);
  double total = ps_val(&t);
  for (int i = 0; i <= s->na; ++i) {
    const Asg* a = i < s->na ? &s->a[i] : extra;
    if (!a || a->dev != dev) continue;
    int j = 0;
    while (gid[j] != a->group) ++j;
    double f = interference(s, total - gmax[j], a->dem);
    if (i < s->na) out_f[i] = f;
    else *extra_f = f;
  }
  free(gid);
  free(gmax);
}

/* adjusted per-op figures (placement.py:245-273) given per-assignment
 * factors `fac` (+ optional extra with factor ef) */
typedef struct { double t_eff, wait; int stable; } Adj;

static void adjusted(const PL* s, const double* fac, const Asg* extra, double ef, Adj* out) {
  for (int v = 0; v < s->n; ++v) {
    PS sum = {0, 0, 0};
    for (int k = 1; k <= s->r[v]; ++k) {
      double f = 1.0;
      for (int i = 0; i < s->na; ++i)
        if (s->a[i].op == v && s->a[i].k == k) { f = fac[i]; break; }
      if (extra && extra->op == v && extra->k == k) f = ef;
      ps_add(&sum, f);
    }
    double t_eff = (s->T[v] * ps_val(&sum)) / (double)s->r[v];
    double layers = (double)s->d->layer_count[v];
    double mu = 1.0 / (t_eff * layers), lam = s->qps / (double)s->b[v];
    int st = lam < (double)s->r[v] * mu;
    out[v].t_eff = t_eff;
    out[v].stable = st;
    out[v].wait = st ? orc_expected_wait(lam, mu, s->r[v]) : INFINITY;
  }
}

static double latency_of(const PL* s, const Adj* adj) {
  double wt[OPSC_MAX_OPS];
  for (int v = 0; v < s->n; ++v) {
    if (!adj[v].stable) return INFINITY;
    double soj = adj[v].wait + adj[v].t_eff / (double)s->b[v];
    wt[v] = (soj + s->comm[v]) * (double)s->d->layer_count[v];
  }
  return orc_critical_path(s->d, wt, NULL);
}

static double* current_factors(const PL* s) {
  double* fac = (double*)malloc(sizeof(double) * (s->na + 1));
  for (int dev = 0; dev < s->used; ++dev) dev_factors(s, dev, NULL, fac, NULL);
  return fac;
}

static void push(PL* s, int op, int k, int dev, int group, int share) {
  Asg* a = &s->a[s->na++];
  a->op = op; a->k = k; a->dev = dev; a->group = group; a->share = share;
  a->dem = s->dem[op]; a->mem = s->mem[op]; a->factor = 1.0;
}

typedef struct { double key; int v; } OK;
static int ok_cmp(const void* x, const void* y) {
  const OK* a = (const OK*)x;
  const OK* b = (const OK*)y;
  if (a->key < b->key) return -1;
  if (a->key > b->key) return 1;
  return a->v - b->v;
}

static uint32_t place_one(PL* s) {
  const OpscDag* d = s->d;
  const OpscPlaceShared* f = s->f;
  int n = s->n, k_base = 1 << 30;
  for (int v = 0; v < n; ++v) k_base = s->r[v] < k_base ? s->r[v] : k_base;
  /* base instances: first-fit decreasing by (-(weight_mem / P), id) */
  OK ord[OPSC_MAX_OPS];
  for (int v = 0; v < n; ++v) { ord[v].key = -(d->weight_mem[v] / (double)s->p[v]); ord[v].v = v; }
  qsort(ord, n, sizeof(OK), ok_cmp);
  for (int inst = 1; inst <= k_base; ++inst) {
    int inst_dev[OPSC_MAX_OPS], nd = 0;
    for (int i = 0; i < n; ++i) {
      int v = ord[i].v, target = -1;
      for (int j = 0; j < nd; ++j)
        if (dev_mem(s, inst_dev[j]) + s->mem[v] <= f->mem_cap[inst_dev[j]]) { target = inst_dev[j]; break; }
      if (target < 0) {
        if (s->used >= f->n_devices) return OPSC_W_FLEET_EXHAUSTED;
        target = s->used++;
        if (s->mem[v] > f->mem_cap[target]) return OPSC_W_INFEASIBLE_PLACEMENT;
        inst_dev[nd++] = target;
      }
      push(s, v, inst, target, inst - 1, 100);
    }
  }
  /* extras, heaviest op_latency first: (-T, id, k) */
  OK xo[OPSC_MAX_OPS];
  for (int v = 0; v < n; ++v) { xo[v].key = -s->T[v]; xo[v].v = v; }
  qsort(xo, n, sizeof(OK), ok_cmp);
  int next_group = k_base;
  Adj adj[OPSC_MAX_OPS];
  for (int i = 0; i < n; ++i) {
    int v = xo[i].v;
    for (int k = k_base + 1; k <= s->r[v]; ++k) {
      int group = next_group++;
      double mem = s->mem[v], demand = s->dem[v];
      double sh = nearbyint(demand * 100.0);
      int share = sh < 1.0 ? 1 : (sh > 100.0 ? 100 : (int)sh);
      double* fac = current_factors(s);
      int best = -1;
      double best_score = 0.0;
      /* default_stream_place (placement.py:465-491): no probing */
      const int n_probe = (f->flags & OPSC_PLACE_DEFAULT_STREAM) ? 0 : s->used;
      for (int dev = 0; dev < n_probe; ++dev) {
        double mu = dev_mem(s, dev);
        if (mu + mem > f->mem_cap[dev]) continue;
        double load = dev_load(s, dev, NULL);
        if (load + demand > f->max_sm_load) continue;
        Asg t = {v, k, dev, group, share, demand, mem, 1.0};
        double* tf = (double*)malloc(sizeof(double) * (s->na + 1));
        memcpy(tf, fac, sizeof(double) * s->na);
        double ef = 1.0;
        dev_factors(s, dev, &t, tf, &ef);
        adjusted(s, tf, &t, ef, adj);
        double lat = latency_of(s, adj);
        free(tf);
        if (lat > s->slo) continue;
        double ms = f->mem_cap[dev] - (mu + mem), cs = f->compute_cap[dev] - (load + demand);
        double mf = (0.0 >= ms ? 0.0 : ms) / f->mem_cap[dev];
        double cf = (0.0 >= cs ? 0.0 : cs) / f->compute_cap[dev];
        double score = f->slack_weight_mem * mf + f->slack_weight_compute * cf;
        if (best < 0 || score > best_score) { best = dev; best_score = score; }
      }
      free(fac);
      if (best >= 0) {
        push(s, v, k, best, group, share);
      } else {
        if (s->used >= f->n_devices) return OPSC_W_FLEET_EXHAUSTED;
        int dev = s->used++;
        if (mem > f->mem_cap[dev]) return OPSC_W_INFEASIBLE_PLACEMENT;
        push(s, v, k, dev, group, 100);
      }
    }
  }
  return 0;
}

int orc_place_shared(const OpscDag* d, const OpscPlaceShared* f, OpscWindows win, const int16_t* cfg,
                     const uint8_t* plan_feasible, int32_t config_order, OpscPlacement out,
                     int32_t n_threads) {
  const int n = d->n_ops;
#pragma omp parallel for num_threads(n_threads) schedule(dynamic, 1)
  for (int w = 0; w < win.n; ++w) {
    out.n_assign[w] = 0; out.devices_used[w] = 0; out.feasible[w] = 0; out.status[w] = 0;
    out.latency[w] = 0.0; out.energy[w] = 0.0; out.memory[w] = 0.0;
    if (!(win.qps[w] > 0.0) || !plan_feasible[w]) continue;
    PL s;
    memset(&s, 0, sizeof(s));
    s.d = d; s.f = f; s.n = n;
    s.slo = (f->flags & OPSC_PLACE_WINDOW_SLO) ? win.slo[w] : f->slo; s.qps = win.qps[w]; s.L = win.seq_len[w]; s.ph = win.phase[w];
    int total_r = 0;
    for (int v = 0; v < n; ++v) {
      s.p[v] = cfg[(w * n + v) * 3]; s.r[v] = cfg[(w * n + v) * 3 + 1]; s.b[v] = cfg[(w * n + v) * 3 + 2];
      double o[7];
      orc_predict(d, s.qps, s.L, s.ph, v, s.p[v], s.r[v], s.b[v], o, NULL);
      s.T[v] = o[0]; s.comm[v] = o[6];
      double dm = d->s0[v] + (d->s1[v] * (double)s.b[v]) * (double)s.L;
      s.dem[v] = 1.0 <= dm ? 1.0 : dm; /* min(1.0, ...) */
      s.mem[v] = orc_op_memory(d->weight_mem[v], d->m0[v], d->m1[v], s.b[v], s.L, s.p[v]);
      s.order[v] = config_order == 0 ? v : d->node_order[v];
      total_r += s.r[v];
    }
    s.cap = total_r + 1;
    s.a = (Asg*)calloc(s.cap, sizeof(Asg));
    uint32_t err = place_one(&s);
    if (err || s.na > out.cap_assign || s.used > out.cap_dev) {
      out.status[w] = err ? err : OPSC_W_TRACE_TRUNCATED;
      free(s.a);
      continue;
    }
    /* _finalize */
    double* fac = current_factors(&s);
    Adj adj[OPSC_MAX_OPS];
    adjusted(&s, fac, NULL, 1.0, adj);
    double lat = latency_of(&s, adj);
    out.latency[w] = lat;
    out.feasible[w] = lat <= s.slo;
    out.devices_used[w] = s.used;
    out.n_assign[w] = s.na;
    PS memsum = {0, 0, 0};
    double* de = out.d_energy + (size_t)w * out.cap_dev;
    for (int dev = 0; dev < s.used; ++dev) {
      out.d_mem[(size_t)w * out.cap_dev + dev] = dev_mem(&s, dev);
      out.d_sm[(size_t)w * out.cap_dev + dev] = dev_load(&s, dev, NULL);
      de[dev] = 0.0;
    }
    for (int i = 0; i < s.na; ++i) {
      const Asg* a = &s.a[i];
      size_t o = (size_t)w * out.cap_assign + i;
      out.a_op[o] = (int8_t)a->op;
      out.a_replica[o] = (int16_t)a->k;
      out.a_device[o] = a->dev;
      out.a_share[o] = (int16_t)a->share;
      out.a_latency[o] = s.T[a->op] * fac[i];
      ps_add(&memsum, a->mem);
      /* fill_device_energy (metrics.py:105-127) */
      double layers = (double)d->layer_count[a->op];
      double sh = ((f->alpha * (double)s.p[a->op]) * (adj[a->op].wait + adj[a->op].t_eff)) * layers;
      sh += ((f->beta * adj[a->op].t_eff) * layers) / (double)s.r[a->op];
      de[a->dev] += sh;
    }
    out.memory[w] = ps_val(&memsum);
    double total = 0.0;
    for (int i = 0; i < n; ++i) {
      int v = s.order[i];
      double layers = (double)d->layer_count[v];
      double wl = adj[v].wait * layers, sl = adj[v].t_eff * layers;
      total += ((f->alpha * (double)s.p[v]) * (double)s.r[v]) * (wl + sl);
      total += f->beta * sl;
    }
    out.energy[w] = total;
    free(fac);
    free(s.a);
  }
  return OPSC_OK;
}
