// k_model.cu -- K3 model_grid: model_level_autoscale on the device.
//
// Mirrors autoscaler.py:596-681 exactly, including its search sequence:
// for every batch size B the replica floor is the max strict-stability floor
// over operators (:643-656), then the smallest R meeting slo - eps (else slo)
// is found with the reference's exponential probe + bisection (:620-639), so
// the evaluated (B, R) points -- and hence the bits of every latency -- are
// the reference's. Argmin of R * sum(P_base) with strict `<` (smallest B
// wins), fallback = min latency at r_cap (first B wins).
//
// One CTA per window, one warp per batch size, one lane per operator: a
// candidate evaluation runs all operators' Erlang-B recurrences in parallel
// lanes and the critical-path DP on lane 0.
#include "opsc_common.cuh"

namespace opsc {

struct ModelArgs {
  OpscDag d;
  OpscModelSpec m;
};

// evaluate(uniform(b, r)) latency (autoscaler.py:196-206, opgraph.py:199-244)
__device__ double eval_uniform(const OpscDag& d, const OpscModelSpec& m, double qps, int L, int ph,
                               int b, int r, double* wsh, uint32_t* st) {
  const int lane = threadIdx.x & 31;
  const int n = d.n_ops;
  bool stable = true;
  if (lane < n) {
    const Pred o = predict<true>(d, qps, L, ph, lane, m.p_base[lane], r, b, st);
    stable = o.stable;
    wsh[lane] = weight(o, d.layer_count[lane]);
  }
  const bool all = __all_sync(0xffffffffu, stable);
  __syncwarp();
  double lat = OPSC_INF;
  if (lane == 0 && all) {
    double val[OPSC_MAX_OPS];
    for (int i = 0; i < n; ++i) {
      const int v = d.topo[i];
      double in = 0.0;
      uint32_t pm = d.pred_mask[v];
      while (pm) {
        const int p = __ffs(pm) - 1;
        pm &= pm - 1;
        in = fmax(in, val[p]);
      }
      val[v] = in + wsh[v];
    }
    lat = 0.0;
    for (int v = 0; v < n; ++v)
      if (d.sink_mask >> v & 1u) lat = fmax(lat, val[v]);
  }
  __syncwarp();
  return __shfl_sync(0xffffffffu, lat, 0);
}

// One (B, R) probe: evaluated in-warp, or looked up in the precomputed
// table of the small-batch path (same arithmetic, so the same bits; the
// table's per-point status bits are ORed only for points the reference visits).
template <bool TABLE>
__device__ __forceinline__ double probe(const OpscDag& d, const OpscModelSpec& m, double qps, int L, int ph,
                                        int b, int r, double* wsh, uint32_t* st, const double* lt,
                                        const uint8_t* ls) {
  if (TABLE) {  // lt / ls: this B's row (R = 1 .. r_cap)
    *st |= ls[r - 1];
    return lt[r - 1];
  }
  return eval_uniform(d, m, qps, L, ph, b, r, wsh, st);
}

// autoscaler.py:620-639
template <bool TABLE>
__device__ int smallest_r(const OpscDag& d, const OpscModelSpec& m, double qps, int L, int ph, int b,
                          int r_floor, double bound, double* wsh, uint32_t* st, double* lat_out,
                          const double* lt, const uint8_t* ls) {
  const double lo_lat = probe<TABLE>(d, m, qps, L, ph, b, r_floor, wsh, st, lt, ls);
  if (lo_lat <= bound) {
    *lat_out = lo_lat;
    return r_floor;
  }
  int hi = r_floor;
  double hi_lat = lo_lat;
  while (hi_lat > bound && hi < m.r_cap) {
    hi = min(hi * 2, m.r_cap);
    hi_lat = probe<TABLE>(d, m, qps, L, ph, b, hi, wsh, st, lt, ls);
  }
  if (hi_lat > bound) {
    *lat_out = hi_lat;
    return -1;
  }
  int lo = r_floor;
  while (hi - lo > 1) {
    const int mid = (lo + hi) / 2;
    const double ml = probe<TABLE>(d, m, qps, L, ph, b, mid, wsh, st, lt, ls);
    if (ml <= bound) {
      hi = mid;
      hi_lat = ml;
    } else {
      lo = mid;
    }
  }
  *lat_out = hi_lat;
  return hi;
}

template <bool TABLE>
__global__ void __launch_bounds__(1024) model_grid_kernel(const __grid_constant__ ModelArgs a,
                                                          const __grid_constant__ OpscWindows win,
                                                          int16_t* __restrict__ cfg,
                                                          uint8_t* __restrict__ feasible,
                                                          uint32_t* __restrict__ status,
                                                          const double* __restrict__ lt_all,
                                                          const uint8_t* __restrict__ ls_all, int rows_smem) {
  pdl_trigger();
  pdl_wait();
  const OpscDag& d = a.d;
  const OpscModelSpec& m = a.m;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int nwarps = blockDim.x >> 5;
  double* wsh_all = reinterpret_cast<double*>(smem_raw);       // [nwarps][32]
  double* res_lat = wsh_all + nwarps * 32;                      // [b_cap]
  int32_t* res_r = reinterpret_cast<int32_t*>(res_lat + m.b_cap);  // [b_cap]; -2 skip, -1 fallback
  __shared__ uint32_t st_sh;

  const int w = blockIdx.x;
  const double qps = win.qps[w];
  for (int i = threadIdx.x; i < d.n_ops * 3; i += blockDim.x) cfg[(size_t)w * d.n_ops * 3 + i] = 0;
  if (!(qps > 0.0)) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) st_sh = 0;
  __syncthreads();
  const int L = win.seq_len[w], ph = win.phase[w];
  const double slo = win.slo[w], target = win.slo[w] - win.eps[w];
  double* wsh = wsh_all + warp * 32;
  uint32_t st = 0;
  const size_t tab = (size_t)m.b_cap * m.r_cap;
  const double* lt_w = TABLE ? lt_all + (size_t)w * tab : nullptr;
  const uint8_t* ls_w = TABLE ? ls_all + (size_t)w * tab : nullptr;
  // table path: each warp stages its B's row of latencies / status bits in
  // shared memory first (coalesced), so the probe + bisection's dependent
  // lookups cost a shared-memory load instead of an L2 round trip each
  double* row_lt = reinterpret_cast<double*>(res_r + m.b_cap + (m.b_cap & 1)) + (size_t)warp * m.r_cap;
  uint8_t* row_ls = reinterpret_cast<uint8_t*>(reinterpret_cast<double*>(res_r + m.b_cap + (m.b_cap & 1)) +
                                               (size_t)nwarps * m.r_cap) + (size_t)warp * m.r_cap;

  for (int b = warp + 1; b <= m.b_cap; b += nwarps) {
    const double* lt = nullptr;
    const uint8_t* ls = nullptr;
    if (TABLE) {
      lt = lt_w + (size_t)(b - 1) * m.r_cap;
      ls = ls_w + (size_t)(b - 1) * m.r_cap;
      if (rows_smem) {
        for (int r = lane; r < m.r_cap; r += 32) {
          row_lt[r] = lt[r];
          row_ls[r] = ls[r];
        }
        __syncwarp();
        lt = row_lt;
        ls = row_ls;
      }
    }
    int rm = 1;
    bool bad = false;
    if (lane < d.n_ops) {
      const double tl = op_latency(d, ph, lane, b, L, m.p_base[lane]) * (double)d.layer_count[lane];
      if (tl == 0.0) st |= OPSC_W_ZERO_DIVISION;
      rm = strict_min_replicas(qps / (double)b, 1.0 / tl, m.r_cap);
      bad = rm < 0;
    }
    const bool unstable = __any_sync(0xffffffffu, bad);
    const int r_floor = max(1, __reduce_max_sync(0xffffffffu, bad ? 1 : rm));
    if (unstable) {
      if (lane == 0) res_r[b - 1] = -2;
      continue;
    }
    double lat;
    int r = smallest_r<TABLE>(d, m, qps, L, ph, b, r_floor, target, wsh, &st, &lat, lt, ls);
    if (r < 0) r = smallest_r<TABLE>(d, m, qps, L, ph, b, r_floor, slo, wsh, &st, &lat, lt, ls);
    if (lane == 0) {
      res_r[b - 1] = r;
      res_lat[b - 1] = lat;
    }
    __syncwarp();  // the row buffer is reused by this warp's next B
  }
  if (st) atomicOr(&st_sh, st);
  __syncthreads();
  if (threadIdx.x == 0) {
    int p_sum = 0;
    for (int v = 0; v < d.n_ops; ++v) p_sum += m.p_base[v];
    int best_b = -1, best_r = 0, best_obj = 0, fb_b = -1;
    double fb_lat = 0.0;
    for (int b = 1; b <= m.b_cap; ++b) {
      const int r = res_r[b - 1];
      if (r == -2) continue;
      if (r == -1) {
        if (fb_b < 0 || res_lat[b - 1] < fb_lat) {
          fb_b = b;
          fb_lat = res_lat[b - 1];
        }
        continue;
      }
      const int obj = r * p_sum;
      if (best_b < 0 || obj < best_obj) {
        best_b = b;
        best_r = r;
        best_obj = obj;
      }
    }
    uint32_t s = st_sh;
    int bb = -1, rr = 0;
    feasible[w] = 0;
    if (best_b >= 0) {
      bb = best_b;
      rr = best_r;
      feasible[w] = 1;
    } else if (fb_b >= 0) {
      bb = fb_b;
      rr = m.r_cap;
    } else {
      s |= OPSC_W_NO_STABLE_MODEL;
    }
    if (bb > 0) {
      for (int v = 0; v < d.n_ops; ++v) {
        int16_t* c = cfg + ((size_t)w * d.n_ops + v) * 3;
        c[0] = (int16_t)m.p_base[v];
        c[1] = (int16_t)rr;
        c[2] = (int16_t)bb;
      }
    }
    status[w] |= s;
  }
}

// ---- small-batch path: every (B, R) point tabulated in parallel ----------
// thread per (window, B, R, op): weight of op under uniform (B, R) at P_base
__global__ void model_tab_weights(const __grid_constant__ ModelArgs a, const __grid_constant__ OpscWindows win,
                                  double* __restrict__ wt, uint8_t* __restrict__ wst) {
  pdl_trigger();
  pdl_wait();
  const OpscDag& d = a.d;
  const OpscModelSpec& m = a.m;
  const int n = d.n_ops;
  const long long total = (long long)win.n * m.b_cap * m.r_cap * n;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int v = (int)(i % n);
    long long t = i / n;
    const int r = (int)(t % m.r_cap) + 1;
    t /= m.r_cap;
    const int b = (int)(t % m.b_cap) + 1;
    const int w = (int)(t / m.b_cap);
    const double qps = win.qps[w];
    if (!(qps > 0.0)) continue;
    uint32_t st = 0;
    const Pred o = predict<true>(d, qps, win.seq_len[w], win.phase[w], v, m.p_base[v], r, b, &st);
    wt[i] = o.stable ? weight(o, d.layer_count[v]) : OPSC_INF;
    wst[i] = (uint8_t)st;
  }
}

// thread per (window, B, R): evaluate(uniform(B, R)).latency (inf if unstable)
__global__ void model_tab_latency(const __grid_constant__ ModelArgs a, int n_windows,
                                  const double* __restrict__ wt, const uint8_t* __restrict__ wst,
                                  double* __restrict__ lt, uint8_t* __restrict__ ls) {
  pdl_trigger();
  pdl_wait();
  const OpscDag& d = a.d;
  const int n = d.n_ops;
  const long long total = (long long)n_windows * a.m.b_cap * a.m.r_cap;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const double* x = wt + i * n;
    uint8_t st = 0;
    bool all = true;
    for (int v = 0; v < n; ++v) {
      st |= wst[i * n + v];
      all &= x[v] != OPSC_INF;
    }
    double lat = OPSC_INF;
    if (all) {
      double val[OPSC_MAX_OPS];
      lat = 0.0;
      for (int k = 0; k < n; ++k) {
        const int v = d.topo[k];
        double in = 0.0;
        uint32_t pm = d.pred_mask[v];
        while (pm) {
          const int p = __ffs(pm) - 1;
          pm &= pm - 1;
          in = fmax(in, val[p]);
        }
        val[v] = in + x[v];
        if (d.sink_mask >> v & 1u) lat = fmax(lat, val[v]);
      }
    }
    lt[i] = lat;
    ls[i] = st;
  }
}

size_t model_table_bytes(int n_windows, const OpscModelSpec& m, int n_ops) {
  const size_t pts = (size_t)n_windows * m.b_cap * m.r_cap;
  return pts * (size_t)n_ops * 9 + pts * 9 + 64;
}

cudaError_t launch_model_grid(const OpscDag& d, const OpscModelSpec& m, OpscWindows w, int16_t* cfg,
                              uint8_t* feasible, uint32_t* status, cudaStream_t s, void* table_ws,
                              size_t table_bytes) {
  if (w.n <= 0) return cudaSuccess;
  if (m.b_cap < 1 || m.r_cap < 1) return cudaErrorInvalidValue;
  ModelArgs a;
  a.d = d;
  a.m = m;
  const int nwarps = m.b_cap < 32 ? m.b_cap : 32;
  const size_t smem0 = (size_t)nwarps * 32 * sizeof(double) + (size_t)m.b_cap * sizeof(double) +
                       (size_t)(m.b_cap + (m.b_cap & 1)) * sizeof(int32_t);
  const bool table = table_ws && table_bytes >= model_table_bytes(w.n, m, d.n_ops);
  const size_t rows = (size_t)nwarps * m.r_cap * (sizeof(double) + 1);
  const int rows_smem = table && smem0 + rows <= (size_t)200 * 1024;
  const size_t smem = smem0 + (rows_smem ? rows : 0);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(table ? model_grid_kernel<true> : model_grid_kernel<false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  if (!table) {
    return launch_pdl(model_grid_kernel<false>, dim3(w.n), dim3(nwarps * 32), smem, s, a, w, cfg, feasible, status,
                      (const double*)nullptr, (const uint8_t*)nullptr, 0);
  }
  const size_t pts = (size_t)w.n * m.b_cap * m.r_cap;
  double* wt = (double*)table_ws;
  double* lt = wt + pts * d.n_ops;
  uint8_t* wst = (uint8_t*)(lt + pts);
  uint8_t* ls = wst + pts * d.n_ops;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long t1 = (long long)pts * d.n_ops;
  const int g1 = (int)((t1 + 127) / 128 < (long long)sms * 32 ? (t1 + 127) / 128 : (long long)sms * 32);
  cudaError_t e = launch_pdl(model_tab_weights, dim3(g1), dim3(128), 0, s, a, w, wt, wst);
  if (e != cudaSuccess) return e;
  const int g2 = (int)(((long long)pts + 127) / 128 < (long long)sms * 32 ? ((long long)pts + 127) / 128
                                                                          : (long long)sms * 32);
  e = launch_pdl(model_tab_latency, dim3(g2), dim3(128), 0, s, a, w.n, (const double*)wt, (const uint8_t*)wst, lt, ls);
  if (e != cudaSuccess) return e;
  return launch_pdl(model_grid_kernel<true>, dim3(w.n), dim3(nwarps * 32), smem, s, a, w, cfg, feasible, status,
                    (const double*)lt, (const uint8_t*)ls, rows_smem);
}

}  // namespace opsc
