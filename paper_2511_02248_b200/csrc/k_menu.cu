// k_menu.cu -- K1 menu_build and the small per-window kernels around it.
//
//   menu_build      <- predict_op loops of brute_force_autoscale (autoscaler.py:743-757)
//   stability_check <- init_configs NoStableConfig check (autoscaler.py:254-294, 771)
//   menu_fallback   <- infeasible-SLO per-op argmin (autoscaler.py:828-841)
//   decode          <- best_assign -> configs (autoscaler.py:843-845)
//
// K1 is one thread per (window, menu entry): ~30 FP64 ops incl. ~8 divisions
// plus the R-step Erlang-B recurrence (R more divisions). Entries of one
// window are contiguous, so the weight stores coalesce.
#include "opsc_common.cuh"

namespace opsc {

__global__ void init_kernel(int n, const double* __restrict__ qps, uint32_t* __restrict__ status,
                            unsigned long long* __restrict__ key, uint8_t* __restrict__ feasible) {
  pdl_trigger();
  pdl_wait();
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= n) return;
  status[w] = qps[w] > 0.0 ? 0u : OPSC_W_IDLE;
  if (key) key[w] = (unsigned long long)OPSC_KEY_INFEASIBLE;
  if (feasible) feasible[w] = 0;
}

cudaError_t launch_init(int n, const double* qps, uint32_t* status, unsigned long long* key,
                        uint8_t* feasible, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  return launch_pdl(init_kernel, dim3((n + 255) / 256), dim3(256), 0, s, n, qps, status, key, feasible);
}

__global__ void fill_keys_kernel(unsigned long long* key, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) key[i] = (unsigned long long)OPSC_KEY_INFEASIBLE;
}

cudaError_t launch_fill_keys(unsigned long long* key, int n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  fill_keys_kernel<<<(n + 255) / 256, 256, 0, s>>>(key, n);
  return cudaGetLastError();
}

__device__ __forceinline__ void menu_build_body(const OpscDag& d, const OpscGrid& g, const OpscWindows& win,
                                                double* __restrict__ menu_w, uint32_t* __restrict__ status,
                                                int block) {
  const int E = g.menu_off[d.n_ops];
  const long long idx = (long long)block * blockDim.x + threadIdx.x;
  if (idx >= (long long)win.n * E) return;
  const int w = (int)(idx / E);
  const int j = (int)(idx - (long long)w * E);
  const double qps = win.qps[w];
  if (!(qps > 0.0)) {
    menu_w[idx] = OPSC_INF;
    return;
  }
  int v = 0;
  while (j >= g.menu_off[v + 1]) ++v;
  int p, r, b;
  entry_prb(g, v, j - g.menu_off[v], p, r, b);
  uint32_t st = 0;
  const Pred o = predict<true>(d, qps, win.seq_len[w], win.phase[w], v, p, r, b, &st);
  // the reference skips every non-finite weight (autoscaler.py:800-801, 833):
  // NaN (possible only with NaN profile data) is stored as +inf so that every
  // compose level excludes it, not just the innermost one
  const double wt = weight(o, d.layer_count[v]);
  menu_w[idx] = (o.stable && !isnan(wt)) ? wt : OPSC_INF;
  if (st) atomicOr(&status[w], st);
}

__global__ void __launch_bounds__(256) menu_build_kernel(const __grid_constant__ OpscDag d,
                                                         const __grid_constant__ OpscGrid g,
                                                         const __grid_constant__ OpscWindows win,
                                                         double* __restrict__ menu_w,
                                                         uint32_t* __restrict__ status) {
  pdl_trigger();
  pdl_wait();
  menu_build_body(d, g, win, menu_w, status, blockIdx.x);
}

cudaError_t launch_menu_build(const OpscDag& d, const OpscGrid& g, OpscWindows w, double* menu_w,
                              uint32_t* status, cudaStream_t s) {
  const long long total = (long long)w.n * g.menu_off[d.n_ops];
  if (total <= 0) return cudaSuccess;
  return launch_pdl(menu_build_kernel, dim3((unsigned)((total + 255) / 256)), dim3(256), 0, s, d, g, w, menu_w, status);
}

// One warp per (window, op): does some (P in params, B <= params.b_max) have
// a strict-stability replica floor within r_cap? P in ascending order (the
// reference's init_configs pre-check, autoscaler.py:254-294), all B of one P
// across the lanes; flags accumulate over every (P, B) visited up to and
// including the first P with a stable B, as in the sequential scan.
__device__ __forceinline__ void stability_body(const OpscDag& d, const OpscGrid& g, const OpscWindows& win,
                                               uint32_t* __restrict__ status, int block) {
  const int gw = (block * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= win.n * d.n_ops) return;
  const int w = gw / d.n_ops, v = gw - w * d.n_ops;
  const double qps = win.qps[w];
  if (!(qps > 0.0)) return;
  const int L = win.seq_len[w], ph = win.phase[w];
  uint32_t st = 0;
  bool found = false;
  for (int pi = 0; pi < g.params_n_p[v] && !found; ++pi) {
    const int p = g.params_p_vals[v][pi];
    bool mine = false;
    for (int b = lane + 1; b <= g.params_b_max[v]; b += 32) {
      const double tl = op_latency(d, ph, v, b, L, p) * (double)d.layer_count[v];
      if (tl == 0.0) st |= OPSC_W_ZERO_DIVISION;
      const double mu = 1.0 / tl, lam = qps / (double)b;
      const int r = strict_min_replicas(lam, mu, g.r_cap);
      if (r < 0) continue;
      const double util = lam / ((double)r * mu);
      if (util >= 1.0 || util <= 0.0) st |= OPSC_W_UNSTABLE_ROUNDING;
      mine = true;
    }
    found = __any_sync(0xffffffffu, mine);
  }
  st = __reduce_or_sync(0xffffffffu, st);
  if (lane != 0) return;
  if (found) {
    if (st) atomicOr(&status[w], st);
    return;
  }
  // NoStableConfig names the first unstable operator in dag.node_ids order
  // (autoscaler.py:268, 289-292): keep the minimum position over the warps
  int pos = 0;
  while (d.node_order[pos] != v) ++pos;
  const uint32_t mine = (uint32_t)(pos + 1);
  st |= OPSC_W_NO_STABLE_PARAMS;
  uint32_t old = status[w], assumed;
  do {
    assumed = old;
    const uint32_t cur = (assumed >> OPSC_W_INIT_OP_SHIFT) & OPSC_W_OP_FIELD;
    uint32_t nv = assumed | st;
    if (cur == 0 || mine < cur)
      nv = (nv & ~(OPSC_W_OP_FIELD << OPSC_W_INIT_OP_SHIFT)) | (mine << OPSC_W_INIT_OP_SHIFT);
    old = atomicCAS(&status[w], assumed, nv);
  } while (old != assumed);
}

__global__ void stability_kernel(const __grid_constant__ OpscDag d, const __grid_constant__ OpscGrid g,
                                 const __grid_constant__ OpscWindows win, uint32_t* __restrict__ status) {
  pdl_trigger();
  pdl_wait();
  stability_body(d, g, win, status, blockIdx.x);
}

// K1 + K1b in one launch (the per-window chains of the host-buffer path and
// DevicePlanner): the first nb_menu blocks build menus, the rest run the
// init_configs stability pre-check; both only OR into status.
__global__ void __launch_bounds__(256) menu_stability_kernel(const __grid_constant__ OpscDag d,
                                                             const __grid_constant__ OpscGrid g,
                                                             const __grid_constant__ OpscWindows win,
                                                             double* __restrict__ menu_w,
                                                             uint32_t* __restrict__ status, int nb_menu) {
  pdl_trigger();
  pdl_wait();
  if ((int)blockIdx.x < nb_menu) menu_build_body(d, g, win, menu_w, status, blockIdx.x);
  else stability_body(d, g, win, status, blockIdx.x - nb_menu);
}

cudaError_t launch_menu_stability(const OpscDag& d, const OpscGrid& g, OpscWindows w, double* menu_w,
                                  uint32_t* status, cudaStream_t s) {
  if (w.n <= 0) return cudaSuccess;
  const long long menu_threads = (long long)w.n * g.menu_off[d.n_ops];
  const long long stab_threads = (long long)w.n * d.n_ops * 32;
  const long long nb_menu = (menu_threads + 255) / 256, nb_stab = (stab_threads + 255) / 256;
  if (nb_menu + nb_stab > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  return launch_pdl(menu_stability_kernel, dim3((unsigned)(nb_menu + nb_stab)), dim3(256), 0, s, d, g, w, menu_w,
                    status, (int)nb_menu);
}

cudaError_t launch_stability(const OpscDag& d, const OpscGrid& g, OpscWindows w, uint32_t* status,
                             cudaStream_t s) {
  const long long threads = (long long)w.n * d.n_ops * 32;
  if (threads <= 0) return cudaSuccess;
  return launch_pdl(stability_kernel, dim3((unsigned)((threads + 127) / 128)), dim3(128), 0, s, d, g, w, status);
}

// One warp per (window, op): min over finite entries of (weight, entry).
__global__ void fallback_kernel(int n_ops, int n_windows, const __grid_constant__ OpscGrid g,
                                const double* __restrict__ menu_w, int32_t* __restrict__ fb) {
  pdl_trigger();
  pdl_wait();
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= n_windows * n_ops) return;
  const int w = gw / n_ops, v = gw - w * n_ops;
  const int E = g.menu_off[n_ops];
  const double* mw = menu_w + (size_t)w * E + g.menu_off[v];
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
  if (lane == 0) fb[w * n_ops + v] = be == 0x7fffffff ? -1 : be;
}

cudaError_t launch_fallback(const OpscDag& d, const OpscGrid& g, int n_windows, const double* menu_w,
                            int32_t* fb, cudaStream_t s) {
  const long long threads = (long long)n_windows * d.n_ops * 32;
  if (threads <= 0) return cudaSuccess;
  return launch_pdl(fallback_kernel, dim3((unsigned)((threads + 255) / 256)), dim3(256), 0, s, d.n_ops, n_windows, g,
                    menu_w, fb);
}

__global__ void decode_kernel(int n_ops, int n_windows, const __grid_constant__ OpscGrid g,
                              const unsigned long long* __restrict__ key, const int32_t* __restrict__ fb,
                              int16_t* __restrict__ cfg, uint8_t* __restrict__ feasible,
                              uint32_t* __restrict__ status) {
  pdl_trigger();
  pdl_wait();
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= n_windows) return;
  feasible[w] = 0;
  int16_t* cw = cfg + (size_t)w * n_ops * 3;
  for (int i = 0; i < n_ops * 3; ++i) cw[i] = 0;  // defined output for idle / error windows
  if (status[w] & OPSC_W_IDLE) return;
  int ent[OPSC_MAX_OPS];
  if (key[w] != (unsigned long long)OPSC_KEY_INFEASIBLE) {
    unsigned long long lex = key[w] & OPSC_LEXMASK;
    for (int v = n_ops - 1; v >= 0; --v) {
      const unsigned long long m = (unsigned long long)(g.menu_off[v + 1] - g.menu_off[v]);
      ent[v] = (int)(lex % m);
      lex /= m;
    }
    feasible[w] = 1;
  } else {
    int bad = 0;  // 1 + rank of the first operator without a finite entry (autoscaler.py:833-837)
    for (int v = 0; v < n_ops; ++v) {
      ent[v] = fb[w * n_ops + v];
      if (ent[v] < 0 && !bad) bad = v + 1;
    }
    if (bad) {
      status[w] |= OPSC_W_NO_STABLE_BOUNDS | ((uint32_t)bad << OPSC_W_BOUNDS_OP_SHIFT);
      return;
    }
  }
  for (int v = 0; v < n_ops; ++v) {
    int p, r, b;
    entry_prb(g, v, ent[v], p, r, b);
    int16_t* c = cfg + ((size_t)w * n_ops + v) * 3;
    c[0] = (int16_t)p;
    c[1] = (int16_t)r;
    c[2] = (int16_t)b;
  }
}

cudaError_t launch_decode(const OpscDag& d, const OpscGrid& g, int n_windows,
                          const unsigned long long* key, const int32_t* fb, int16_t* cfg,
                          uint8_t* feasible, uint32_t* status, cudaStream_t s) {
  if (n_windows <= 0) return cudaSuccess;
  return launch_pdl(decode_kernel, dim3((n_windows + 127) / 128), dim3(128), 0, s, d.n_ops, n_windows, g, key, fb,
                    cfg, feasible, status);
}

}  // namespace opsc
