// k_materialize.cu -- K4: decided configs -> ScalingPlan fields + metrics.
//
// Per window (one thread each; this is per-decision work, not per-candidate):
//   * _Evaluator.evaluate of the decided configs (autoscaler.py:196-206):
//     PredictedSojourn per op and the critical path with the reference's
//     lexicographic path tie-break (opgraph.py:199-244); objective = sum P*R;
//   * default_stream_place (placement.py:358-396, 465-491): devices_used and
//     provisioned memory (metrics.py:130-132, CPython-3.12 float sum order);
//   * request_energy (metrics.py:84-102) with every interference factor equal
//     to 1 (single-group devices under default-stream placement), i.e.
//     t_eff = (T * R) / R as _adjusted_ops computes it (placement.py:257).
#include <cstring>

#include "opsc_common.cuh"

namespace opsc {

__device__ __forceinline__ double op_memory(const OpscDag& d, int v, int p, int b, int L) {
  return (d.weight_mem[v] / (double)p + d.m0[v]) + (d.m1[v] * (double)b) * (double)L;
}

// Per-warp shared scratch of the serial lane-0 section: a one-shot walk over
// cold local memory would pay an L2 round trip per access.
struct MatScratch {
  double mem[OPSC_MAX_OPS];
  double val[OPSC_MAX_OPS];
  double ds_f[OPSC_MAX_OPS], ds_c[OPSC_MAX_OPS];  // per-device PySum state (Neumaier)
  int order[OPSC_MAX_OPS], xord[OPSC_MAX_OPS], inst_dev[OPSC_MAX_OPS];
  int cp[OPSC_MAX_OPS], cr[OPSC_MAX_OPS], cb[OPSC_MAX_OPS];  // decided (P, R, B), loaded once by the lanes
  double ratio[OPSC_MAX_OPS];
  int k_base;
  int8_t parent[OPSC_MAX_OPS];
};

// Warp-parallel part of default_stream_place (lane v = operator v): memory
// per replica, and the two stable sorts as ranks -- (-(weight_mem/P), id)
// for base instances and (-op_latency, id) for extra replicas
// (placement.py:358-396, 465-491).
__device__ __forceinline__ void place_prepare(const OpscDag& d, const double* T, int L, MatScratch& S, int lane) {
  const int n = d.n_ops;
  int kb = 1 << 30;
  if (lane < n) S.ratio[lane] = -(d.weight_mem[lane] / (double)S.cp[lane]);
  __syncwarp();
  if (lane < n) {
    const int v = lane;
    S.mem[v] = op_memory(d, v, S.cp[v], S.cb[v], L);
    const double rv = S.ratio[v];
    const double tv = -T[v];
    int r1 = 0, r2 = 0;
    for (int u = 0; u < n; ++u) {
      const double ru = S.ratio[u];
      const double tu = -T[u];
      r1 += ru < rv || (ru == rv && u < v);
      r2 += tu < tv || (tu == tv && u < v);
    }
    S.order[r1] = v;
    S.xord[r2] = v;
    kb = S.cr[v];
  }
  kb = __reduce_min_sync(0xffffffffu, kb);
  if (lane == 0) S.k_base = kb;
  __syncwarp();
}

// default_stream_place (lane 0, sequential as the reference); returns 0 or an error bit
__device__ uint32_t place_default_stream(const OpscPlaceSpec& pl, int n, MatScratch& S, int* devices,
                                         double* memory) {
  const int k_base = S.k_base;
  PySum total;
  total.reset();
  int used = 0;
  auto cap_of = [&](int dev) { return pl.uniform_cap ? pl.mem_cap[0] : pl.mem_cap[dev]; };
  auto dev_value = [&](int j) { const double f = S.ds_f[j], cc = S.ds_c[j]; return (cc != 0.0 && isfinite(cc)) ? f + cc : f; };
  // base instances (placement.py:358-385)
  const int full_sim = pl.uniform_cap ? 1 : k_base;  // uniform caps: every instance packs alike
  int per_inst = 0;
  for (int inst = 1; inst <= full_sim; ++inst) {
    int nd = 0;
    for (int i = 0; i < n; ++i) {
      const int v = S.order[i];
      const double m = S.mem[v];
      int t = -1;
      for (int j = 0; j < nd; ++j)
        if (dev_value(j) + m <= cap_of(S.inst_dev[j])) { t = j; break; }
      if (t < 0) {
        if (used >= pl.n_devices) return OPSC_W_FLEET_EXHAUSTED;
        const int dev = used++;
        if (m > cap_of(dev)) return OPSC_W_INFEASIBLE_PLACEMENT;
        S.inst_dev[nd] = dev;
        S.ds_f[nd] = 0.0 + m;  // PySum's first add
        S.ds_c[nd] = 0.0;
        t = nd++;
      } else {
        PySum ds;
        ds.f = S.ds_f[t];
        ds.c = S.ds_c[t];
        ds.started = true;
        ds.add(m);
        S.ds_f[t] = ds.f;
        S.ds_c[t] = ds.c;
      }
      total.add(m);
    }
    per_inst = nd;
  }
  if (pl.uniform_cap && k_base > 1) {
    if ((long long)used + (long long)(k_base - 1) * per_inst > (long long)pl.n_devices)
      return OPSC_W_FLEET_EXHAUSTED;
    used += (k_base - 1) * per_inst;
    for (int inst = 2; inst <= k_base; ++inst)
      for (int i = 0; i < n; ++i) total.add(S.mem[S.order[i]]);
  }
  // extra replicas on dedicated devices, heaviest op_latency first (placement.py:388-396, 482-490)
  for (int i = 0; i < n; ++i) {
    const int v = S.xord[i];
    const double m = S.mem[v];
    for (int k = k_base + 1; k <= S.cr[v]; ++k) {
      if (used >= pl.n_devices) return OPSC_W_FLEET_EXHAUSTED;
      const int dev = used++;
      if (m > cap_of(dev)) return OPSC_W_INFEASIBLE_PLACEMENT;
      total.add(m);
    }
  }
  *devices = used;
  *memory = total.value();
  return 0;
}

// Two warps per window. Warp A: lane v predicts operator v (its Erlang-B
// recurrences run in parallel lanes) and its Eq. 9 energy terms, then the
// critical path (a chain's weights summed left to right by shuffles; any
// other DAG by lane 0 with the reference's lexicographic path tie-break) and
// the energy sum in the plan's config order. Warp B, at the same time: the
// default-stream placement, which needs only the configs, op latencies and
// memory (lane-parallel sorts, then lane 0's sequential packing, as the
// reference). A named barrier per window joins them.
constexpr int kMatWin = 2;  // windows per CTA (2 warps each)

// Brute-force decode in the window's warp (DECODE): the per-op fallback
// argmin when no candidate met the SLO (autoscaler.py:828-841: min over
// finite weights of (weight, entry), one warp reduction per op) or the
// winner's lexicographic index split into menu entries (:843-845), then the
// (P, R, B) configs -- the work of fallback_kernel + decode_kernel, fused so
// the per-window chain is one launch shorter by two.
struct DecodeIn {
  OpscGrid g;
  const unsigned long long* key;
  const double* menu_w;
};

__device__ __forceinline__ void decode_window(const OpscDag& d, const DecodeIn& dc, const OpscDecisions& out, int w,
                                              int lane) {
  const int n = d.n_ops;
  int16_t* cw = out.cfg + (size_t)w * n * 3;
  for (int i = lane; i < n * 3; i += 32) cw[i] = 0;  // defined output for idle / error windows
  if (lane == 0) out.feasible[w] = 0;
  __syncwarp();
  if (out.status[w] & OPSC_W_IDLE) return;
  const unsigned long long key = dc.key[w];
  const OpscGrid& g = dc.g;
  if (key != (unsigned long long)OPSC_KEY_INFEASIBLE) {
    if (lane == 0) {
      unsigned long long lex = key & OPSC_LEXMASK;
      for (int v = n - 1; v >= 0; --v) {
        const unsigned long long m = (unsigned long long)(g.menu_off[v + 1] - g.menu_off[v]);
        const int e = (int)(lex % m);
        lex /= m;
        int p, r, b;
        entry_prb(g, v, e, p, r, b);
        cw[v * 3] = (int16_t)p;
        cw[v * 3 + 1] = (int16_t)r;
        cw[v * 3 + 2] = (int16_t)b;
      }
      out.feasible[w] = 1;
    }
    __syncwarp();
    return;
  }
  const int E = g.menu_off[n];
  int bad = 0;  // 1 + rank of the first operator without a finite entry (autoscaler.py:833-837)
  for (int v = 0; v < n; ++v) {
    const double* mw = dc.menu_w + (size_t)w * E + g.menu_off[v];
    const int m = g.menu_off[v + 1] - g.menu_off[v];
    double bw = OPSC_INF;
    int be = 0x7fffffff;
    for (int e = lane; e < m; e += 32) {
      const double x = mw[e];
      if (isfinite(x) && (x < bw || (x == bw && e < be))) { bw = x; be = e; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double x = __shfl_xor_sync(0xffffffffu, bw, o);
      const int e = __shfl_xor_sync(0xffffffffu, be, o);
      if (x < bw || (x == bw && e < be)) { bw = x; be = e; }
    }
    if (be == 0x7fffffff) {
      if (!bad) bad = v + 1;
    } else if (lane == 0 && !bad) {
      int p, r, b;
      entry_prb(g, v, be, p, r, b);
      cw[v * 3] = (int16_t)p;
      cw[v * 3 + 1] = (int16_t)r;
      cw[v * 3 + 2] = (int16_t)b;
    }
  }
  if (bad) {  // configs stay zero, as decode_kernel leaves them
    for (int i = lane; i < n * 3; i += 32) cw[i] = 0;
    __syncwarp();
    if (lane == 0) out.status[w] |= OPSC_W_NO_STABLE_BOUNDS | ((uint32_t)bad << OPSC_W_BOUNDS_OP_SHIFT);
  }
  __syncwarp();
}

// the two warps of window `pair` (barrier ids 1, 2 as immediates: ptxas
// reserves only what it sees)
__device__ __forceinline__ void pair_barrier(int pair) {
  static_assert(kMatWin == 2, "one named barrier per window of the CTA");
  // non-.aligned form: a warp may arrive with its lanes not yet reconverged
  // (compute-sanitizer synccheck flags bar.sync = barrier.sync.aligned there)
  __syncwarp();
  if (pair == 0) asm volatile("barrier.sync 1, 64;" ::: "memory");
  else asm volatile("barrier.sync 2, 64;" ::: "memory");
}

struct MatPlace {
  uint32_t err;
  int devices;
  double memory;
};

template <bool DECODE>
__global__ void __launch_bounds__(64 * kMatWin) materialize_kernel(const __grid_constant__ OpscDag d,
                                                                   const __grid_constant__ OpscWindows win,
                                                                   int config_order,
                                                                   const __grid_constant__ OpscPlaceSpec pl,
                                                                   const __grid_constant__ OpscDecisions out,
                                                                   const __grid_constant__ DecodeIn dc) {
  pdl_trigger();
  pdl_wait();
  __shared__ double s_wt[kMatWin][OPSC_MAX_OPS], s_T[kMatWin][OPSC_MAX_OPS];
  __shared__ double s_e1[kMatWin][OPSC_MAX_OPS], s_e2[kMatWin][OPSC_MAX_OPS];
  __shared__ MatScratch s_scr[kMatWin];
  __shared__ MatPlace s_pl[kMatWin];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = warp >> 1;
  const bool A = (warp & 1) == 0;
  const int w = blockIdx.x * kMatWin + pair;
  if (w >= win.n) return;  // both warps of a window leave together
  const int n = d.n_ops;
  if (DECODE && A) decode_window(d, dc, out, w, lane);
  if (DECODE) pair_barrier(pair);
  const uint32_t st0 = out.status[w];
  if (A) {
    if (lane < n) {
      out.path[(size_t)w * n + lane] = -1;
      out.stable[(size_t)w * n + lane] = 0;
      for (int f = 0; f < OPSC_PRED_FIELDS; ++f) out.pred[((size_t)w * n + lane) * OPSC_PRED_FIELDS + f] = 0.0;
    }
    if (lane == 0) {
      out.latency[w] = OPSC_INF;
      out.objective[w] = 0;
      out.energy[w] = 0.0;
      out.memory[w] = 0.0;
      out.devices[w] = 0;
    }
  }
  if (st0 & (OPSC_W_IDLE | OPSC_W_NO_STABLE_BOUNDS | OPSC_W_NO_STABLE_PARAMS | OPSC_W_NO_STABLE_MODEL |
             OPSC_W_NO_STABLE_INIT))
    return;
  const int16_t* c = out.cfg + (size_t)w * n * 3;
  const double qps = win.qps[w];
  const int L = win.seq_len[w], ph = win.phase[w];
  const bool feas = out.feasible[w] != 0;
  MatScratch& S = s_scr[pair];
  if (!A) {  // ---- warp B: default-stream placement (placement.py:358-396, 465-491)
    if (feas) {
      if (lane < n) {
        const int v = lane;
        const int p = c[v * 3], r = c[v * 3 + 1], b = c[v * 3 + 2];
        S.cp[v] = p;
        S.cr[v] = r;
        S.cb[v] = b;
        s_T[pair][v] = op_latency(d, ph, v, b, L, p);
      }
      __syncwarp();
      place_prepare(d, s_T[pair], L, S, lane);
      if (lane == 0) {
        MatPlace& P = s_pl[pair];
        P.devices = 0;
        P.memory = 0.0;
        P.err = place_default_stream(pl, n, S, &P.devices, &P.memory);
      }
    }
    pair_barrier(pair);
    return;
  }
  // ---- warp A: evaluate (autoscaler.py:196-206) and request_energy terms
  uint32_t st = 0;
  bool stable = true;
  int cpv = 0, crv = 0;
  if (lane < n) {
    const int v = lane;
    const int p = c[v * 3], r = c[v * 3 + 1], b = c[v * 3 + 2];
    cpv = p;
    crv = r;
    const Pred o = predict(d, qps, L, ph, v, p, r, b, &st);
    double* pf = out.pred + ((size_t)w * n + v) * OPSC_PRED_FIELDS;
    pf[0] = o.t; pf[1] = o.lam; pf[2] = o.mu; pf[3] = o.util;
    pf[4] = o.wait; pf[5] = o.service; pf[6] = o.comm;
    out.stable[(size_t)w * n + v] = o.stable;
    stable = o.stable;
    s_wt[pair][v] = weight(o, d.layer_count[v]);
  }
  // request_energy terms under default-stream placement: factors 1,
  // t_eff = (T * R) / R (placement.py:257), wait re-derived from t_eff -- a
  // second Erlang-B chain per op, run in lanes n..2n-1 next to the predict
  // chains of lanes 0..n-1 (in lane v itself when n > 16)
  const int ev = n <= 16 ? lane - n : lane;
  if (feas && ev >= 0 && ev < n) {
    const int v = ev;
    const int p = c[v * 3], r = c[v * 3 + 1], b = c[v * 3 + 2];
    const double layers = (double)d.layer_count[v];
    const double t = op_latency(d, ph, v, b, L, p);
    const double t_eff = (t * (double)r) / (double)r;
    const double mu = 1.0 / (t_eff * layers), lam = qps / (double)b;
    // the wait only enters fl(wait * layers + t_eff * layers): wait_for_sum
    // against t_eff gives the same bits (a W below 2^-56 t_eff scales to
    // below half an ulp of t_eff * layers)
    const double wait = lam < (double)r * mu
                            ? wait_for_sum(r, lam / ((double)r * mu), (double)r * mu - lam, t_eff)
                            : OPSC_INF;
    const double wl = wait * layers, sl = t_eff * layers;
    s_e1[pair][v] = ((pl.alpha * (double)p) * (double)r) * (wl + sl);
    s_e2[pair][v] = pl.beta * sl;
  }
  const bool all = __all_sync(0xffffffffu, stable);
  st = __reduce_or_sync(0xffffffffu, st);
  const int obj = __reduce_add_sync(0xffffffffu, cpv * crv);
  __syncwarp();
  if (all) {
    if (is_chain(d)) {  // one source-sink path: val = val(prev) + w in order, the path is every op
      const int u = lane < n ? d.topo[lane] : 0;
      const double wl = lane < n ? s_wt[pair][u] : 0.0;
      double acc = 0.0;
      for (int i = 0; i < n; ++i) {
        const double wi = __shfl_sync(0xffffffffu, wl, i);
        acc = i == 0 ? wi : acc + wi;
      }
      if (lane < n) out.path[(size_t)w * n + lane] = (int8_t)u;
      if (lane == 0) out.latency[w] = acc;
    } else if (lane == 0) {
      out.latency[w] = critical_path_lex(d, s_wt[pair], out.path + (size_t)w * n, S.val, S.parent);
    }
  }
  double total = 0.0;
  if (feas && lane == 0) {  // the energy sum in the plan's config order
    for (int i = 0; i < n; ++i) {
      const int v = config_order == 0 ? i : d.node_order[i];
      total = total + s_e1[pair][v];
      total = total + s_e2[pair][v];
    }
  }
  pair_barrier(pair);  // warp B's placement is in s_pl
  if (lane != 0) return;
  out.objective[w] = obj;
  st |= st0;
  if (feas) {
    const MatPlace& P = s_pl[pair];
    st |= P.err;
    if (!P.err) {
      out.devices[w] = P.devices;
      out.memory[w] = P.memory;
      out.energy[w] = total;
    }
  }
  out.status[w] = st;
}

cudaError_t launch_materialize(const OpscDag& d, OpscWindows w, int config_order, const OpscPlaceSpec& p,
                               OpscDecisions out, cudaStream_t s) {
  if (w.n <= 0) return cudaSuccess;
  DecodeIn dc;
  memset(&dc, 0, sizeof(dc));
  return launch_pdl(materialize_kernel<false>, dim3((w.n + kMatWin - 1) / kMatWin), dim3(64 * kMatWin), 0, s, d, w,
                    config_order, p, out, dc);
}

cudaError_t launch_decode_materialize(const OpscDag& d, const OpscGrid& g, OpscWindows w,
                                      const unsigned long long* key, const double* menu_w, const OpscPlaceSpec& p,
                                      OpscDecisions out, cudaStream_t s) {
  if (w.n <= 0) return cudaSuccess;
  DecodeIn dc;
  dc.g = g;
  dc.key = key;
  dc.menu_w = menu_w;
  return launch_pdl(materialize_kernel<true>, dim3((w.n + kMatWin - 1) / kMatWin), dim3(64 * kMatWin), 0, s, d, w,
                    0, p, out, dc);
}

}  // namespace opsc
