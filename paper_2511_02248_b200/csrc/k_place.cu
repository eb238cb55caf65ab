// k_place.cu -- K6: shared (interference-aware) placement, Alg. 2 of the
// reference (placement.py:399-462), or with OPSC_PLACE_DEFAULT_STREAM its
// no-sharing variant (default_stream_place, :465-491: same base instances
// and _finalize, every extra replica on an unused device), with the
// placement-dependent metrics
// (request_energy, fill_device_energy, provisioned_memory; metrics.py:84-132).
//
// One CTA per window. Base instances are packed first-fit-decreasing
// (placement.py:358-385, sequential, thread 0; each base device then holds
// one instance's group, refreshed one device per thread). Each extra replica,
// heaviest op_latency first (:388-396), probes every used device; a probe
// needs the interference factors of the device's members with the tentative
// replica added (:209-231), the adjusted service time and Erlang-C wait of
// every operator with a replica there (:245-273) and the critical path.
// Stage 1 (a thread per device) admits the devices and lists the (device,
// operator) pairs to re-evaluate; stage 2 runs those Erlang-B recurrences, one
// listed pair per thread; stage 3 (a thread per device) checks the critical
// path against the SLO and scores by weighted slack (:338-351), reduced to the
// best score, ties to the lowest device id; thread 0 commits, and the new
// load and factors of the chosen device are updated incrementally.
// Sums the reference takes with Python's sum() use CPython 3.12's Neumaier
// summation (PySum), in the reference's iteration order.
#include <cstdio>

#include "opsc_common.cuh"
#include "opsc_pow.cuh"

namespace opsc {

constexpr int kPlaceThreads = 128;
static_assert(kPlaceThreads == 128, "the extra-replica commit is split over exactly four warps");
constexpr int kMaxDevProbe = 128;  // device probes per chunk held in smem
constexpr size_t kPlaceSmemMax = 200 * 1024;  // static PShared + per-window workspace

struct PlaceArgs {
  OpscDag d;
  OpscPlaceShared f;
  int probe_smem;  // the probe store of the first kMaxDevProbe devices fits in shared memory
};

struct PWork {  // per-window workspace (shared memory when it fits, else global)
  int32_t* a_op;    // operator of assignment i
  int32_t* a_dev;   // device of assignment i
  double* a_gmax;   // max demand over the members of i's group on i's device
  double* dev_lf;   // standing load of each device: the PySum state (f, c, started) of its
  double* dev_lc;   //   group maxima in first-occurrence order, kept current at every push
  int32_t* dev_ls;
  uint32_t* dev_mask;  // operators with a member on each device
  int32_t* a_group;
  int32_t* a_next;
  double* a_dem;
  double* a_mem;
  double* a_fac;
  int32_t* dev_head;
  int32_t* dev_tail;
  int32_t* dev_cnt;
  double* dev_mem_f;
  double* dev_mem_c;
  int32_t* rep;  // [sum R] assignment index per (op, replica), -1 unplaced
};

// per-window global store of the stage-2 probe results (t_eff, wait,
// weight, stable) of every (device, operator) pair: after a commit the chosen
// device's entries ARE the operators' new figures (same factors, same sums)
__host__ __device__ inline size_t probe_bytes(int D, int n) {
  return (((size_t)D * n * (8 + 8 + 8 + 1)) + 15) & ~(size_t)15;
}

struct ProbeStore {
  double* teff;
  double* wait;
  double* wt;
  uint8_t* ok;
};

// the store's arrays for `devs` devices, indexed [device * n + op]
__device__ __forceinline__ ProbeStore probe_store(unsigned char* base, int devs, int n) {
  ProbeStore p;
  p.teff = reinterpret_cast<double*>(base);
  p.wait = p.teff + (size_t)devs * n;
  p.wt = p.wait + (size_t)devs * n;
  p.ok = reinterpret_cast<uint8_t*>(p.wt + (size_t)devs * n);
  return p;
}

__host__ __device__ inline size_t pw_bytes(int A, int D, int n) {
  (void)n;
  // rounded to 16 B so every window's double arrays stay 8-byte aligned
  const size_t b = (size_t)A * (4 + 4 + 4 + 4 + 8 + 8 + 8 + 8) + (size_t)D * (4 + 4 + 4 + 8 + 8 + 8 + 8 + 4 + 4) +
                   (size_t)A * 4 + 64;
  return (b + 15) & ~(size_t)15;
}

__device__ PWork carve(unsigned char* base, int A, int D) {
  PWork p;
  double* dp = (double*)base;
  p.a_dem = dp; dp += A;
  p.a_mem = dp; dp += A;
  p.a_fac = dp; dp += A;
  p.dev_mem_f = dp; dp += D;
  p.dev_mem_c = dp; dp += D;
  p.a_gmax = dp; dp += A;
  p.dev_lf = dp; dp += D;
  p.dev_lc = dp; dp += D;
  int32_t* ip = (int32_t*)dp;
  p.dev_ls = ip; ip += D;
  p.dev_mask = (uint32_t*)ip; ip += D;
  p.a_op = ip; ip += A;
  p.a_dev = ip; ip += A;
  p.a_group = ip; ip += A;
  p.a_next = ip; ip += A;
  p.dev_head = ip; ip += D;
  p.dev_tail = ip; ip += D;
  p.dev_cnt = ip; ip += D;
  p.rep = ip;
  return p;
}

// excess ** exponent: exact forms for 1, 2 and 0.5. Any other exponent runs
// the GP instantiation (chosen on the host): rounded to nearest from a
// double-double evaluation (opsc_pow.cuh), which equals glibc's pow -- the
// reference's `**` -- wherever glibc rounds correctly. The default
// instantiation keeps the library pow as an unreachable fallback, so its
// register allocation is not shaped by the double-double code.
template <bool GP>
__device__ __forceinline__ double pow_expo(double x, double e) {
  if (e == 1.0) return x;
  if (e == 2.0) return x * x;
  if (e == 0.5) return sqrt(x);
  return GP ? opsc_pow::pow_rn(x, e) : pow(x, e);
}

template <bool GP>
__device__ __forceinline__ double interference(const OpscPlaceShared& f, double load, double adding) {
  const double excess = load + adding - 1.0;
  if (excess <= 0.0) return 1.0;
  return 1.0 + f.theta * pow_expo<GP>(excess, f.exponent);
}

__device__ __forceinline__ double psum_value(double f, double c, bool started) {
  if (!started) return 0.0;
  return (c != 0.0 && isfinite(c)) ? f + c : f;
}

// interference factor of member i of `dev` with an optional extra (group xg, demand xd)
template <bool GP>
__device__ double member_factor(const PWork& P, const OpscPlaceShared& f, int dev, int i, int xg, double xd,
                                double total) {
  (void)dev;
  double gm = P.a_gmax[i];  // = the scan over dev's members of i's group, kept by push
  if (xg == P.a_group[i]) gm = gm >= xd ? gm : xd;
  return interference<GP>(f, total - gm, P.a_dem[i]);
}

__device__ __forceinline__ PySum cached_load(const PWork& P, int dev) {
  PySum t;
  t.f = P.dev_lf[dev];
  t.c = P.dev_lc[dev];
  t.started = P.dev_ls[dev] != 0;
  return t;
}

struct OpAdj {
  double t_eff, wait, wt;
  bool stable;
};

// adjusted figures of op u: factors of its replicas (k = 1..R) with the
// members of `dev` re-evaluated under the extra (xg, xd, xop, xk, xf)
template <bool GP>
__device__ OpAdj adjust_op(const OpscDag& d, const OpscPlaceShared& f, const PWork& P, const int* rep_off,
                           const int32_t* adev, int u, int p, int r, int b, double T, double comm, double qps,
                           int dev, int xg, double xd, int xop, int xk, double xf, double total) {
  PySum s;
  s.reset();
  for (int k = 1; k <= r; ++k) {
    const int idx = P.rep[rep_off[u] + k - 1];
    double fk = 1.0;
    if (idx >= 0) {
      const bool on_dev = dev >= 0 && adev[idx] == dev;
      fk = on_dev ? member_factor<GP>(P, f, dev, idx, xg, xd, total) : P.a_fac[idx];
    } else if (u == xop && k == xk) {
      fk = xf;
    }
    s.add(fk);
  }
  OpAdj o;
  o.t_eff = (T * s.value()) / (double)r;
  const double layers = (double)d.layer_count[u];
  const double mu = 1.0 / (o.t_eff * layers), lam = qps / (double)b;
  o.stable = lam < (double)r * mu;
  o.wait = o.stable ? expected_wait(lam, mu, r) : OPSC_INF;
  o.wt = ((o.wait + o.t_eff / (double)b) + comm) * layers;
  return o;
}

__device__ double dp_latency(const OpscDag& d, const double* wt) {
  double val[OPSC_MAX_OPS];
  double top = 0.0;
  for (int i = 0; i < d.n_ops; ++i) {
    const int v = d.topo[i];
    double in = 0.0;
    uint32_t pm = d.pred_mask[v];
    while (pm) {
      const int q = __ffs(pm) - 1;
      pm &= pm - 1;
      in = fmax(in, val[q]);
    }
    val[v] = in + wt[v];
    if (d.sink_mask >> v & 1u) top = fmax(top, val[v]);
  }
  return top;
}

struct PShared {
  int p[OPSC_MAX_OPS], r[OPSC_MAX_OPS], b[OPSC_MAX_OPS];
  double T[OPSC_MAX_OPS], comm[OPSC_MAX_OPS], dem[OPSC_MAX_OPS], mem[OPSC_MAX_OPS];
  int rep_off[OPSC_MAX_OPS + 1];
  double cur_wt[OPSC_MAX_OPS], cur_teff[OPSC_MAX_OPS], cur_wait[OPSC_MAX_OPS];
  bool cur_stable[OPSC_MAX_OPS];
  double dev_load0[kMaxDevProbe];   // standing load of device d (without the tentative replica)
  double dev_total[kMaxDevProbe];   // ... with it
  double dev_xf[kMaxDevProbe];      // tentative replica's factor on d
  uint16_t items[kMaxDevProbe * OPSC_MAX_OPS];  // stage 2 work list: (d << 5 | op)
  int n_items;
  uint8_t dev_ok[kMaxDevProbe];
  double probe_wt[kMaxDevProbe][OPSC_MAX_OPS];
  double dev_score[kMaxDevProbe];   // weighted slack of each admissible device
  double ototal;                    // a commit's device: standing load with the extra
#ifdef OPSC_PLACE_PROF
  long long prof[7];  // stage1+2, stage3+select, commit, refresh, -, extras, device probes
  long long ph[6];    // phase timestamps: start, setup, base, initial figures, extras, end
#endif
  double red_score[kPlaceThreads / 32];
  int red_dj[kPlaceThreads / 32];
  int used, na, err, best;
};

template <bool SMEM, bool GP>
__global__ void __launch_bounds__(kPlaceThreads) place_kernel(const __grid_constant__ PlaceArgs a,
                                                              const __grid_constant__ OpscWindows win,
                                                              const int16_t* __restrict__ cfg,
                                                              const uint8_t* __restrict__ plan_feasible,
                                                              int config_order,
                                                              const __grid_constant__ OpscPlacement out,
                                                              unsigned char* __restrict__ ws) {
  __shared__ PShared S;
  extern __shared__ __align__(16) unsigned char pw_smem[];
  const OpscDag& d = a.d;
  const OpscPlaceShared& f = a.f;
  const int n = d.n_ops;
  const int w = blockIdx.x;
  const int A = out.cap_assign, D = out.cap_dev;
  if (threadIdx.x == 0) {
    out.n_assign[w] = 0; out.devices_used[w] = 0; out.feasible[w] = 0; out.status[w] = 0;
    out.latency[w] = 0.0; out.energy[w] = 0.0; out.memory[w] = 0.0;
  }
  const double qps = win.qps[w];
  if (!(qps > 0.0) || !plan_feasible[w]) return;
  const int L = win.seq_len[w], ph = win.phase[w];
  const double slo = (f.flags & OPSC_PLACE_WINDOW_SLO) ? win.slo[w] : f.slo;
  const bool probe = !(f.flags & OPSC_PLACE_DEFAULT_STREAM);
  const bool chain = is_chain(d);  // stage 3's critical path without the DAG walk
  // the window's assignment lists / device tables are walked by every probe:
  // in shared memory when they fit (smem_ws), else in its global slice
  // (SMEM: a compile-time choice, so the walks compile to shared-memory loads)
  unsigned char* wbase = ws + (size_t)w * (pw_bytes(A, D, n) + probe_bytes(D, n));
  PWork P = carve(SMEM ? pw_smem : wbase, A, D);
  const ProbeStore pg = probe_store(wbase + pw_bytes(A, D, n), D, n);
  // while no more than kMaxDevProbe devices are in use, the probe store in
  // shared memory (behind the workspace) when the launch reserved it
  const ProbeStore pss = probe_store(pw_smem + pw_bytes(A, D, n), kMaxDevProbe, n);
  const int32_t* adev = P.a_dev;
  if (threadIdx.x == 0) {
    S.rep_off[0] = 0;
    for (int v = 0; v < n; ++v) {
      S.p[v] = cfg[((size_t)w * n + v) * 3];
      S.r[v] = cfg[((size_t)w * n + v) * 3 + 1];
      S.b[v] = cfg[((size_t)w * n + v) * 3 + 2];
      S.rep_off[v + 1] = S.rep_off[v] + S.r[v];
    }
    S.err = S.rep_off[n] > A ? OPSC_W_TRACE_TRUNCATED : 0;
#ifdef OPSC_PLACE_PROF
    for (int q = 0; q < 7; ++q) S.prof[q] = 0;
    S.ph[0] = clock64();
#endif
    S.used = 0;
    S.na = 0;
    S.n_items = 0;
  }
  __syncthreads();
  if (S.err) {
    if (threadIdx.x == 0) out.status[w] = S.err;
    return;
  }
  for (int v = threadIdx.x; v < n; v += blockDim.x) {
    uint32_t st = 0;
    const Pred o = predict(d, qps, L, ph, v, S.p[v], S.r[v], S.b[v], &st);
    S.T[v] = o.t;
    S.comm[v] = o.comm;
    const double dm = d.s0[v] + (d.s1[v] * (double)S.b[v]) * (double)L;
    S.dem[v] = 1.0 <= dm ? 1.0 : dm;
    S.mem[v] = (d.weight_mem[v] / (double)S.p[v] + d.m0[v]) + (d.m1[v] * (double)S.b[v]) * (double)L;
  }
  for (int i = threadIdx.x; i < S.rep_off[n]; i += blockDim.x) P.rep[i] = -1;
  for (int i = threadIdx.x; i < D; i += blockDim.x) {
    P.dev_head[i] = -1; P.dev_tail[i] = -1; P.dev_cnt[i] = 0;
    P.dev_mem_f[i] = 0.0; P.dev_mem_c[i] = 0.0;
    P.dev_lf[i] = 0.0; P.dev_lc[i] = 0.0; P.dev_ls[i] = 0; P.dev_mask[i] = 0u;
  }
  __syncthreads();
#ifdef OPSC_PLACE_PROF
  if (threadIdx.x == 0) S.ph[1] = clock64();
#endif

  // thread 0 helpers -------------------------------------------------------
  auto push = [&](int v, int k, int dev, int group, int share) {
    const int i = S.na++;
    P.a_group[i] = group;
    P.a_next[i] = -1;
    P.a_dem[i] = S.dem[v];
    P.a_mem[i] = S.mem[v];
    P.a_fac[i] = 1.0;
    if (P.dev_tail[dev] >= 0) P.a_next[P.dev_tail[dev]] = i;
    else P.dev_head[dev] = i;
    P.dev_tail[dev] = i;
    // device memory: Python sum over members in order
    const double x = S.mem[v];
    if (P.dev_cnt[dev] == 0) {
      P.dev_mem_f[dev] = 0.0 + x;
      P.dev_mem_c[dev] = 0.0;
    } else {
      const double fs = P.dev_mem_f[dev], t = fs + x;
      if (fabs(fs) >= fabs(x)) P.dev_mem_c[dev] += (fs - t) + x;
      else P.dev_mem_c[dev] += (x - t) + fs;
      P.dev_mem_f[dev] = t;
    }
    P.dev_cnt[dev]++;
    P.rep[S.rep_off[v] + k - 1] = i;
    P.dev_mask[dev] |= 1u << v;  // group maxima, load sum and factors: by the caller
    const size_t o = (size_t)w * A + i;
    P.a_op[i] = v;
    P.a_dev[i] = dev;
    out.a_op[o] = (int8_t)v;
    out.a_replica[o] = (int16_t)k;
    out.a_device[o] = dev;
    out.a_share[o] = (int16_t)share;
  };
  auto dev_mem = [&](int dev) { return psum_value(P.dev_mem_f[dev], P.dev_mem_c[dev], P.dev_cnt[dev] > 0); };
  // a base device after the first-fit pass: every device is opened within one
  // instance and only that instance's pushes go to it (first fit over the
  // devices opened for the instance), so its members form ONE group: each
  // member's group maximum is the maximum over the device's list (the scan
  // member_factor made per call, in list order), the standing load is that one
  // term, and every member's interference factor follows from it
  auto refresh_base_device = [&](int dev) {
    double gm = 0.0;
    for (int j = P.dev_head[dev]; j >= 0; j = P.a_next[j]) gm = gm >= P.a_dem[j] ? gm : P.a_dem[j];
    PySum ls;
    ls.reset();
    ls.add(gm);
    P.dev_lf[dev] = ls.f;
    P.dev_lc[dev] = ls.c;
    P.dev_ls[dev] = 1;
    const double total = ls.value();
    for (int i = P.dev_head[dev]; i >= 0; i = P.a_next[i]) {
      P.a_gmax[i] = gm;
      P.a_fac[i] = interference<GP>(f, total - gm, P.a_dem[i]);
    }
  };

  // ---- base instances (placement.py:358-385), thread 0
  int k_base = 1 << 30;
  for (int v = 0; v < n; ++v) k_base = min(k_base, S.r[v]);
  if (threadIdx.x == 0) {
    int order[OPSC_MAX_OPS];
    double key[OPSC_MAX_OPS];
    for (int v = 0; v < n; ++v) { order[v] = v; key[v] = -(d.weight_mem[v] / (double)S.p[v]); }
    for (int i = 1; i < n; ++i) {
      const int x = order[i];
      int j = i - 1;
      while (j >= 0 && key[order[j]] > key[x]) { order[j + 1] = order[j]; --j; }
      order[j + 1] = x;
    }
    for (int inst = 1; inst <= k_base && !S.err; ++inst) {
      int idev[OPSC_MAX_OPS], nd = 0;
      for (int i = 0; i < n && !S.err; ++i) {
        const int v = order[i];
        int target = -1;
        for (int j = 0; j < nd; ++j)
          if (dev_mem(idev[j]) + S.mem[v] <= f.mem_cap[idev[j]]) { target = idev[j]; break; }
        if (target < 0) {
          if (S.used >= f.n_devices || S.used >= D) { S.err = OPSC_W_FLEET_EXHAUSTED; break; }
          target = S.used++;
          if (S.mem[v] > f.mem_cap[target]) { S.err = OPSC_W_INFEASIBLE_PLACEMENT; break; }
          idev[nd++] = target;
        }
        push(v, inst, target, inst - 1, 100);
      }
    }
  }
  __syncthreads();
  for (int dev = threadIdx.x; dev < S.used; dev += blockDim.x) refresh_base_device(dev);  // in parallel
  __syncthreads();
#ifdef OPSC_PLACE_PROF
  if (threadIdx.x == 0) S.ph[2] = clock64();
#endif
  if (S.err) {
    if (threadIdx.x == 0) out.status[w] = S.err;
    return;
  }
  // current adjusted figures of every op (parallel over ops)
  for (int v = threadIdx.x; v < n; v += blockDim.x) {
    const OpAdj o = adjust_op<GP>(d, f, P, S.rep_off, adev, v, S.p[v], S.r[v], S.b[v], S.T[v], S.comm[v], qps, -1, -1,
                              0.0, -1, 0, 1.0, 0.0);
    S.cur_wt[v] = o.wt; S.cur_teff[v] = o.t_eff; S.cur_wait[v] = o.wait; S.cur_stable[v] = o.stable;
  }
  __syncthreads();
#ifdef OPSC_PLACE_PROF
  if (threadIdx.x == 0) S.ph[3] = clock64();
#endif

  // ---- extra replicas, heaviest op_latency first (-T, id, k)
  int xord[OPSC_MAX_OPS];
  for (int v = 0; v < n; ++v) xord[v] = v;
  for (int i = 1; i < n; ++i) {
    const int x = xord[i];
    int j = i - 1;
    while (j >= 0 && -S.T[xord[j]] > -S.T[x]) { xord[j + 1] = xord[j]; --j; }
    xord[j + 1] = x;
  }
  int group = k_base;
  for (int xi = 0; xi < n; ++xi) {
    const int v = xord[xi];
    for (int k = k_base + 1; k <= S.r[v]; ++k, ++group) {
      const double mem = S.mem[v], demand = S.dem[v];
      const double shf = nearbyint(demand * 100.0);
      const int share = shf < 1.0 ? 1 : (shf > 100.0 ? 100 : (int)shf);
      // default-stream placement never shares: straight to take_unused.
      // The device count is read once: thread 0 bumps S.used in the commit,
      // while other threads may still be evaluating the chunk loop's exit
      // condition (compute-sanitizer racecheck; a fleet with a multiple of
      // kMaxDevProbe used devices would otherwise split the CTA across
      // __syncthreads).
      const int n_used = S.used, na0 = S.na;  // both change only in the commit below
      // without probes (default stream) no stage barrier separates these reads
      // and the previous extra's flags from this extra's commit
      if (!probe) __syncthreads();
      const ProbeStore ps = SMEM && a.probe_smem && n_used <= kMaxDevProbe ? pss : pg;
      const double xg_max = 0.0 >= demand ? 0.0 : demand;  // the extra's (fresh) group maximum
      int best_dev = -1;  // lane 0 of every warp: best admissible device over the chunks
      double best_score = 0.0;
#ifdef OPSC_PLACE_PROF
      long long q0 = clock64(), q1 = q0, q2 = q0;
#endif
      for (int c0 = 0; probe && c0 < n_used; c0 += kMaxDevProbe) {
      const int U = min(n_used - c0, kMaxDevProbe);
      // stage 1, one thread per device: admission (memory, standing SM load)
      // and the standing load with the tentative replica -- extras own a fresh
      // group (groups count up per extra replica), so dev_load with the extra
      // is the device's cached sum plus one more term max(0, demand); the
      // (device, operator) pairs to re-evaluate (operators with a replica
      // there) are appended to a compact work list, so that stage 2 spreads
      // the Erlang chains over the CTA instead of over a (device x op) grid
      // where most items are empty and the warps run in lockstep
      for (int dj = threadIdx.x; dj < U; dj += blockDim.x) {
        const int dev = c0 + dj;
        const double mu = dev_mem(dev);
        const PySum ls = cached_load(P, dev);
        const double load = ls.value();
        const bool ok = !(mu + mem > f.mem_cap[dev]) && !(load + demand > f.max_sm_load);
        S.dev_ok[dj] = ok;
        S.dev_load0[dj] = load;
        if (!ok) continue;
        PySum lt = ls;
        lt.add(xg_max);
        const double total = lt.value();
        S.dev_total[dj] = total;
        S.dev_xf[dj] = interference<GP>(f, total - xg_max, demand);
        uint32_t m = P.dev_mask[dev] | (1u << v);
        int at = atomicAdd(&S.n_items, __popc(m));
        for (; m; m &= m - 1) S.items[at++] = (uint16_t)(dj << 5 | (__ffs(m) - 1));
      }
      __syncthreads();
      // stage 2: the listed (device, operator) re-evaluations in parallel
      for (int it = threadIdx.x; it < S.n_items; it += blockDim.x) {
        const int dj = S.items[it] >> 5, u = S.items[it] & 31;
        const int dev = c0 + dj;
        const OpAdj o = adjust_op<GP>(d, f, P, S.rep_off, adev, u, S.p[u], S.r[u], S.b[u], S.T[u], S.comm[u], qps,
                                  dev, group, demand, v, k, S.dev_xf[dj], S.dev_total[dj]);
        S.probe_wt[dj][u] = o.stable ? o.wt : OPSC_INF;
        const size_t pi = (size_t)dev * n + u;
        ps.teff[pi] = o.t_eff;
        ps.wait[pi] = o.wait;
        ps.wt[pi] = o.wt;
        ps.ok[pi] = o.stable;
      }
      __syncthreads();
#ifdef OPSC_PLACE_PROF
      q1 = clock64();
#endif
      // stage 3: recomputed latency must meet the SLO (placement.py:434-438),
      // and the weighted slack score of every admissible device (:338-351)
      bool nan_score = false;
      int my_dj = -1;
      double my_score = 0.0;
      for (int dj = threadIdx.x; dj < U; dj += blockDim.x) {
        if (!S.dev_ok[dj]) continue;
        const uint32_t m = P.dev_mask[c0 + dj] | (1u << v);  // operators stage 2 re-evaluated
        bool fin = true;
        double lat;
        if (chain) {  // dp_latency's operations on a chain, in registers
          double x = 0.0;
          for (int i = 0; i < n; ++i) {
            const int u = d.topo[i];
            const double wt = (m >> u & 1u) ? S.probe_wt[dj][u] : (S.cur_stable[u] ? S.cur_wt[u] : OPSC_INF);
            fin &= wt != OPSC_INF;
            x = fmax(0.0, x) + wt;
          }
          lat = fin ? fmax(0.0, x) : OPSC_INF;
        } else {
          for (int u = 0; u < n; ++u) {
            if (!(m >> u & 1u)) S.probe_wt[dj][u] = S.cur_stable[u] ? S.cur_wt[u] : OPSC_INF;
            fin &= S.probe_wt[dj][u] != OPSC_INF;
          }
          lat = fin ? dp_latency(d, S.probe_wt[dj]) : OPSC_INF;
        }
        if (lat > slo) {
          S.dev_ok[dj] = 0;
          continue;
        }
        const int dev = c0 + dj;
        const double mu = dev_mem(dev), load = S.dev_load0[dj];
        const double ms = f.mem_cap[dev] - (mu + mem), cs = f.compute_cap[dev] - (load + demand);
        const double mf = (0.0 >= ms ? 0.0 : ms) / f.mem_cap[dev];
        const double cf = (0.0 >= cs ? 0.0 : cs) / f.compute_cap[dev];
        const double score = f.slack_weight_mem * mf + f.slack_weight_compute * cf;
        S.dev_score[dj] = score;
        nan_score |= score != score;
        if (my_dj < 0 || score > my_score) { my_dj = dj; my_score = score; }  // ascending dj per thread
      }
      // best score, ties to the lowest device id: a block-wide (score, -dj)
      // maximum -- the reference's in-order scan with a strict '>' -- unless a
      // score is NaN, where only the literal scan reproduces it (thread 0)
      for (int o = 16; o > 0; o >>= 1) {
        const double os = __shfl_xor_sync(0xffffffffu, my_score, o);
        const int od = __shfl_xor_sync(0xffffffffu, my_dj, o);
        if (od >= 0 && (my_dj < 0 || os > my_score || (os == my_score && od < my_dj))) {
          my_score = os;
          my_dj = od;
        }
      }
      nan_score = __any_sync(0xffffffffu, nan_score);
      if ((threadIdx.x & 31) == 0) {
        S.red_score[threadIdx.x >> 5] = my_score;
        S.red_dj[threadIdx.x >> 5] = nan_score ? -2 : my_dj;
      }
      __syncthreads();
      if ((threadIdx.x & 31) == 0) {  // every warp's lane 0 selects (the same device): all commit below
        bool any_nan = false;
        for (int wi = 0; wi < kPlaceThreads / 32; ++wi) any_nan |= S.red_dj[wi] == -2;
        int bd = -1;
        double bs = 0.0;
        if (any_nan) {
          for (int dj = 0; dj < U; ++dj)
            if (S.dev_ok[dj] && (bd < 0 || S.dev_score[dj] > bs)) { bd = dj; bs = S.dev_score[dj]; }
        } else {
          for (int wi = 0; wi < kPlaceThreads / 32; ++wi) {
            const int od = S.red_dj[wi];
            const double os = S.red_score[wi];
            if (od >= 0 && (bd < 0 || os > bs || (os == bs && od < bd))) { bd = od; bs = os; }
          }
        }
        // across device chunks: a later chunk wins only with a strictly greater score
        if (bd >= 0 && (best_dev < 0 || bs > best_score)) { best_dev = c0 + bd; best_score = bs; }
      }
      if (threadIdx.x == 0) S.n_items = 0;  // stage 1's list, empty for the next chunk / extra (a barrier comes first)
      if (c0 + kMaxDevProbe < n_used) __syncthreads();  // the next chunk reuses the stage arrays
      }
#ifdef OPSC_PLACE_PROF
      q2 = clock64();
#endif
      __shared__ int s_probed, s_fresh_same;
      // commit: the lane 0 of each warp takes the same decision (best device,
      // or the next unused one: take_unused) from the same state and writes
      // its part of the push, so the four parts run side by side
      if ((threadIdx.x & 31) == 0) {
        const bool probed = best_dev >= 0;
        int best = best_dev, err = 0;
        if (!probed) {
          if (n_used >= f.n_devices || n_used >= D) err = OPSC_W_FLEET_EXHAUSTED;
          else if (mem > f.mem_cap[best = n_used]) err = OPSC_W_INFEASIBLE_PLACEMENT;
        }
        const int i = na0, part = threadIdx.x >> 5;
        if (part == 0) {  // status, the assignment's list entry and index tables
          S.err = err;
          S.best = best;
          s_probed = probed;
          if (!probed) S.used = n_used + 1;
          if (!err) {
            S.na = i + 1;
            P.a_group[i] = group;
            P.a_next[i] = -1;
            const int tail = P.dev_tail[best];
            if (tail >= 0) P.a_next[tail] = i;
            else P.dev_head[best] = i;
            P.dev_tail[best] = i;
            P.dev_cnt[best] += 1;
            P.rep[S.rep_off[v] + k - 1] = i;
            P.a_op[i] = v;
            P.a_dev[i] = best;
          }
        } else if (part == 1 && !err) {  // device memory: Python sum over members in order
          P.a_dem[i] = demand;
          P.a_mem[i] = mem;
          P.a_fac[i] = 1.0;  // (overwritten with the device's other members after the barrier)
          if (!probed) {  // a fresh device: its first member
            P.dev_mem_f[best] = 0.0 + mem;
            P.dev_mem_c[best] = 0.0;
          } else {
            const double fs = P.dev_mem_f[best], t = fs + mem;
            if (fabs(fs) >= fabs(mem)) P.dev_mem_c[best] += (fs - t) + mem;
            else P.dev_mem_c[best] += (mem - t) + fs;
            P.dev_mem_f[best] = t;
          }
        } else if (part == 2 && !err) {
          // the extra owns a fresh group, appended last in first-occurrence
          // order: the device's standing load is its cached PySum plus one
          // more term (what a from-scratch dev_load would build, and what
          // stage 1 probed), the other members' group maxima are unchanged
          PySum lt = cached_load(P, best);
          lt.add(xg_max);
          P.dev_lf[best] = lt.f;
          P.dev_lc[best] = lt.c;
          P.dev_ls[best] = lt.started ? 1 : 0;
          P.a_gmax[i] = xg_max;
          S.ototal = lt.value();
          // a replica placed alone on a fresh device gets factor 1.0 (the
          // factor the loop below gives it) -- exactly the factor its
          // operator's figures already counted it with while it was unplaced
          // (adjust_op), so those figures are unchanged
          s_fresh_same = !probed && interference<GP>(f, S.ototal - xg_max, demand) == 1.0;
        } else if (part == 3 && !err) {  // the output row and the device's operator mask
          P.dev_mask[best] |= 1u << v;
          const size_t o = (size_t)w * A + i;
          out.a_op[o] = (int8_t)v;
          out.a_replica[o] = (int16_t)k;
          out.a_device[o] = best;
          out.a_share[o] = (int16_t)(probed ? share : 100);
        }
      }
      __syncthreads();
      if (S.err) {
        if (threadIdx.x == 0) out.status[w] = S.err;
        return;
      }
#ifdef OPSC_PLACE_PROF
      const long long q3 = clock64();
#endif
      // every member's interference factor under the new load, in parallel
      // over the assignments (member_factor with no extra); the cached figures
      // of the ops with a replica on the chosen device: the probe of this
      // device computed exactly these figures (same factors, same sums)
      const int bdev = S.best;
      for (int i = threadIdx.x; i < S.na; i += blockDim.x)
        if (adev[i] == bdev) P.a_fac[i] = interference<GP>(f, S.ototal - P.a_gmax[i], P.a_dem[i]);
      const uint32_t bmask = P.dev_mask[bdev];
      if (s_probed) {
        for (int u = threadIdx.x; u < n; u += blockDim.x) {
          if (!(bmask >> u & 1u)) continue;
          const size_t pi = (size_t)bdev * n + u;
          S.cur_wt[u] = ps.wt[pi]; S.cur_teff[u] = ps.teff[pi]; S.cur_wait[u] = ps.wait[pi];
          S.cur_stable[u] = ps.ok[pi] != 0;
        }
      }
      __syncthreads();
      if (!s_probed && !s_fresh_same) {  // a fresh device whose factor is not 1.0 (NaN demand)
        for (int u = threadIdx.x; u < n; u += blockDim.x) {
          if (!(bmask >> u & 1u)) continue;
          const OpAdj o = adjust_op<GP>(d, f, P, S.rep_off, adev, u, S.p[u], S.r[u], S.b[u], S.T[u], S.comm[u], qps, -1,
                                    -1, 0.0, -1, 0, 1.0, 0.0);
          S.cur_wt[u] = o.wt; S.cur_teff[u] = o.t_eff; S.cur_wait[u] = o.wait; S.cur_stable[u] = o.stable;
        }
        __syncthreads();
      }
#ifdef OPSC_PLACE_PROF
      if (threadIdx.x == 0) {
        S.prof[0] += q1 - q0; S.prof[1] += q2 - q1; S.prof[2] += q3 - q2; S.prof[3] += clock64() - q3;
        S.prof[5] += 1; S.prof[6] += n_used;
      }
#endif
    }
  }
#ifdef OPSC_PLACE_PROF
  if (threadIdx.x == 0) S.ph[4] = clock64();
#endif

  // ---- _finalize + metrics
  // per assignment, in parallel: its op latency and its share of the request
  // energy (metrics.py); the shares are kept in a_gmax, dead after the extras
  double* a_sh = P.a_gmax;
  for (int i = threadIdx.x; i < S.na; i += blockDim.x) {
    const size_t o = (size_t)w * A + i;
    const int u = P.a_op[i];
    out.a_latency[o] = S.T[u] * P.a_fac[i];
    const double layers = (double)d.layer_count[u];
    double sh = ((f.alpha * (double)S.p[u]) * (S.cur_wait[u] + S.cur_teff[u])) * layers;
    sh += ((f.beta * S.cur_teff[u]) * layers) / (double)S.r[u];
    a_sh[i] = sh;
  }
  __syncthreads();
  // per device, in parallel: the shares of its members added in assignment
  // order (the device's list is in assignment order), as the reference's loop
  // over the assignments adds each to its device's entry
  for (int dev = threadIdx.x; dev < S.used; dev += blockDim.x) {
    double e = 0.0;
    for (int i = P.dev_head[dev]; i >= 0; i = P.a_next[i]) e += a_sh[i];
    out.d_energy[(size_t)w * D + dev] = e;
    out.d_mem[(size_t)w * D + dev] = dev_mem(dev);
    out.d_sm[(size_t)w * D + dev] = cached_load(P, dev).value();
  }
  // the scalar sums, by one thread of the last warp (alongside the devices)
  if (threadIdx.x == kPlaceThreads - 32) {
    bool all = true;
    for (int u = 0; u < n; ++u) all &= S.cur_stable[u];
    const double lat = all ? dp_latency(d, S.cur_wt) : OPSC_INF;
    out.latency[w] = lat;
    out.feasible[w] = lat <= slo;
    out.devices_used[w] = S.used;
    out.n_assign[w] = S.na;
    PySum memsum;
    memsum.reset();
    for (int i = 0; i < S.na; ++i) memsum.add(P.a_mem[i]);
    out.memory[w] = memsum.value();
    double total = 0.0;
    for (int i = 0; i < n; ++i) {
      const int u = config_order == 0 ? i : d.node_order[i];
      const double layers = (double)d.layer_count[u];
      const double wl = S.cur_wait[u] * layers, sl = S.cur_teff[u] * layers;
      total += ((f.alpha * (double)S.p[u]) * (double)S.r[u]) * (wl + sl);
      total += f.beta * sl;
    }
    out.energy[w] = total;
  }
#ifdef OPSC_PLACE_PROF
  __syncthreads();
  if (threadIdx.x == 0)
    printf("phases w%d: setup %lld base %lld initial %lld extras %lld finalize %lld | %lld extras, %lld device probes, "
           "stage1+2 %lld stage3+select %lld commit %lld refresh %lld\n", w, S.ph[1] - S.ph[0], S.ph[2] - S.ph[1],
           S.ph[3] - S.ph[2], S.ph[4] - S.ph[3], clock64() - S.ph[4], S.prof[5], S.prof[6], S.prof[0], S.prof[1],
           S.prof[2], S.prof[3]);
#endif
}

size_t place_shared_workspace(int n_windows, int A, int D, int n) {
  return (size_t)(n_windows > 0 ? n_windows : 1) * (pw_bytes(A, D, n) + probe_bytes(D, n));
}

cudaError_t launch_place_shared(const OpscDag& d, const OpscPlaceShared& f, OpscWindows w, const int16_t* cfg,
                                const uint8_t* feas, int config_order, OpscPlacement out, void* ws,
                                size_t ws_bytes, cudaStream_t s) {
  if (w.n <= 0) return cudaSuccess;
  if (!ws || ws_bytes < place_shared_workspace(w.n, out.cap_assign, out.cap_dev, d.n_ops))
    return cudaErrorInvalidValue;
  PlaceArgs a;
  a.d = d;
  a.f = f;
  const size_t pw = pw_bytes(out.cap_assign, out.cap_dev, d.n_ops);
  const size_t pss = probe_bytes(kMaxDevProbe, d.n_ops);
  const bool smem_ws = pw + sizeof(PShared) + 1024 <= kPlaceSmemMax;
  a.probe_smem = smem_ws && pw + pss + sizeof(PShared) + 1024 <= kPlaceSmemMax;
  const size_t dyn = smem_ws ? pw + (a.probe_smem ? pss : 0) : 0;
  // static PShared + dynamic workspace may pass the 48 KB default: raise the
  // kernel's dynamic limit (once per size increase, per device)
  static int set_dyn[64];
  int dev = 0;
  cudaGetDevice(&dev);
  const bool gp = !(f.exponent == 1.0 || f.exponent == 2.0 || f.exponent == 0.5);
  if (dyn > 0 && dev < 64 && (int)dyn > set_dyn[dev]) {
    cudaError_t e = cudaFuncSetAttribute(place_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(place_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    if (e != cudaSuccess) return e;
    set_dyn[dev] = (int)dyn;
  }
  unsigned char* wsb = (unsigned char*)ws;
  if (smem_ws && gp)
    place_kernel<true, true><<<w.n, kPlaceThreads, dyn, s>>>(a, w, cfg, feas, config_order, out, wsb);
  else if (smem_ws)
    place_kernel<true, false><<<w.n, kPlaceThreads, dyn, s>>>(a, w, cfg, feas, config_order, out, wsb);
  else if (gp)
    place_kernel<false, true><<<w.n, kPlaceThreads, 0, s>>>(a, w, cfg, feas, config_order, out, wsb);
  else
    place_kernel<false, false><<<w.n, kPlaceThreads, 0, s>>>(a, w, cfg, feas, config_order, out, wsb);
  return cudaGetLastError();
}

// Diagnostic: the placement's excess ** exponent on arbitrary inputs
// (opsc_interference_pow; tests/test_gpu_pow.py).
__global__ void interference_pow_kernel(const double* __restrict__ x, const double* __restrict__ e,
                                        double* __restrict__ out, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = pow_expo<true>(x[i], e[i]);
}

cudaError_t launch_interference_pow(const double* x, const double* e, double* out, long long n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const long long blocks = (n + 255) / 256;
  interference_pow_kernel<<<(int)(blocks < 148 * 16 ? blocks : 148 * 16), 256, 0, s>>>(x, e, out, n);
  return cudaGetLastError();
}

}  // namespace opsc
