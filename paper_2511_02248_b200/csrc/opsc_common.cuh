// opsc_common.cuh -- shared device arithmetic for the sm_100a planner kernels.
//
// Bit-exactness contract: every expression below keeps
// the reference's Python association order, the whole library is compiled
// with --fmad=false (no DFMA contraction), and double division is CUDA's
// IEEE round-to-nearest `/`. Integers convert to double exactly.
#pragma once

#include <cuda_runtime.h>
#include <cstdlib>
#include <math_constants.h>
#include <stdint.h>

#include "../../include/opscale_b200.h"

#define OPSC_INF CUDART_INF
#define OPSC_LEXMASK ((1ull << OPSC_KEY_LEX_BITS) - 1ull)

namespace opsc {

// Programmatic dependent launch (sm_90+): the planning pipeline's kernels are
// launched with programmatic stream serialization, so a kernel's launch and
// CTA rasterisation overlap its predecessor's tail. Every such kernel calls
// pdl_wait() before touching memory a predecessor wrote (griddepcontrol.wait
// returns once the preceding grid has completed and its writes are visible);
// small kernels call pdl_trigger() first to release their dependents early.
// Without the launch attribute both are no-ops.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// perfmodel.py:62-64 and :133-157. At the planners' sm_share = 1.0 the
// SM-share factor is exactly 1: demand = min(1, s0+s1*B*L) <= 1 gives
// 1/demand >= 1, so effective = min(1, 1/demand) = 1.0 and base/1.0 = base.
// (The CPU oracle evaluates the factor literally; the golden tests pin both.)
__device__ __forceinline__ double op_latency(const OpscDag& d, int ph, int v, long long b,
                                             long long l, long long p) {
  const long long bl = b * l;
  const double base = (d.c0[ph][v] + d.c1[ph][v] * (double)bl) + (d.c2[ph][v] * (double)bl) * (double)l;
  return base / (d.eta[v] * (double)p);
}

// queueing.py:54-75: Erlang-B recurrence recomputed with a = R*rho.
// Once b underflows to +0 every later step is exactly +0 (a*0 = 0, k+0 = k,
// 0/k = +0), so the loop stops there: the same bits without the remaining
// steps, whose zero-numerator divisions take the slow path (~3x a normal
// step on B200; tools/probe/erlang_probe.cu).
__device__ __forceinline__ double erlang_c(int r, double rho) {
  const double a = (double)r * rho;
  double b = 1.0;
  for (int k = 1; k <= r; ++k) {
    const double ab = a * b;
    b = ab / ((double)k + ab);
    if (b == 0.0) break;
  }
  return ((double)r * b) / ((double)r - a * (1.0 - b));
}

// queueing.py:78-87
__device__ __forceinline__ double expected_wait(double lam, double mu, int r) {
  const double rho = lam / ((double)r * mu);
  return erlang_c(r, rho) / ((double)r * mu - lam);
}

// The M/M/R wait for consumers that only use it inside fl(W + service)
// (sojourn = wait + T/B, and the critical-path weight built from it): the
// reference's exact recurrence, except that it returns +0.0 as soon as the
// final W is provably below 2^-56 * service. Then W < half an ulp of service,
// so fl(W + service) == service == fl(+0 + service): the same bits, without
// the tail of a long Erlang-B chain. Proof sketch: for k >= a = R*rho every
// later step multiplies b by a / (k + a b) <= 1 (rounding adds at most a
// relative 1e-13 over 512 steps), so b_R <= b_k; C_R = R b_R / (R - a(1 - b_R))
// <= R b_k / (R - a); W = C_R / (R mu - lam). The bound below carries a 4x
// margin on top. `den` = R*mu - lam as the reference computes it.
__device__ __forceinline__ double wait_for_sum(int r, double rho, double den, double service) {
  const double a = (double)r * rho;
  const double cut = service * 0x1p-56 * den * ((double)r - a) * 0.25;  // on R*b_k
  double b = 1.0;
  for (int k = 1; k <= r; ++k) {
    const double ab = a * b;
    b = ab / ((double)k + ab);
    if (b == 0.0) break;
    if ((double)k >= a && (double)r * b < cut) return 0.0;
  }
  return (((double)r * b) / ((double)r - a * (1.0 - b))) / den;
}

// autoscaler.py:224-228; -1 == None
__device__ __forceinline__ int strict_min_replicas(double lam, double mu, int r_cap) {
  const double q = ceil(lam / mu);
  if (!(q <= (double)r_cap)) return -1;
  int r = q < 1.0 ? 1 : (int)q;
  while (lam >= (double)r * mu) {
    if (++r > r_cap) return -1;
  }
  return r;
}

// perfmodel.py:167-171 via autoscaler.py:163-172 (max over out edges, strict >)
__device__ __forceinline__ double comm_time(const OpscDag& d, int v, long long b, long long l) {
  double best = 0.0;
  for (int e = d.out_ptr[v]; e < d.out_ptr[v + 1]; ++e) {
    const double t = (d.out_v0[e] + (d.out_v1[e] * (double)b) * (double)l) / d.link_bw;
    if (t > best) best = t;
  }
  return best;
}

// Critical path with the reference's lexicographic path tie-break
// (opgraph.py:199-244): best[v] = max over predecessors of best[p] + w[v],
// ties to the lexicographically smallest path tuple (op ids are lex ranks),
// latency = max over sinks with the same tie-break. Kept as parent pointers:
// O(n + E) per call; paths are materialised only to break an exact tie.
__device__ __forceinline__ int cp_path_of(const int8_t* parent, int v, int8_t* buf) {
  int8_t tmp[OPSC_MAX_OPS];
  int len = 0;
  for (int u = v; u >= 0; u = parent[u]) tmp[len++] = (int8_t)u;
  for (int i = 0; i < len; ++i) buf[i] = tmp[len - 1 - i];
  return len;
}

__device__ __forceinline__ bool cp_seq_less(const int8_t* a, int la, const int8_t* b, int lb) {
  const int n = la < lb ? la : lb;
  for (int i = 0; i < n; ++i)
    if (a[i] != b[i]) return a[i] < b[i];
  return la < lb;
}

// val / parent: caller scratch (shared memory in K4, where cold local
// memory would cost an L2 round trip per access of a one-shot serial walk).
static __device__ __forceinline__ double critical_path_lex_body(const OpscDag& d, const double* wt, int8_t* path_out,
                                                                double* val, int8_t* parent) {
  const int n = d.n_ops;
  for (int i = 0; i < n; ++i) {
    const int v = d.topo[i];
    uint32_t pm = d.pred_mask[v];
    if (!pm) {
      val[v] = wt[v];
      parent[v] = -1;
      continue;
    }
    int cand = -1;
    double cv = 0.0;
    while (pm) {
      const int p = __ffs(pm) - 1;
      pm &= pm - 1;
      const double ev = val[p] + wt[v];
      bool take = cand < 0 || ev > cv;
      if (!take && ev == cv) {  // path(p) + (v,) < path(cand) + (v,) ?
        int8_t pa[OPSC_MAX_OPS], pb[OPSC_MAX_OPS];
        const int la = cp_path_of(parent, p, pa), lb = cp_path_of(parent, cand, pb);
        pa[la] = (int8_t)v;
        pb[lb] = (int8_t)v;
        take = cp_seq_less(pa, la + 1, pb, lb + 1);
      }
      if (take) {
        cand = p;
        cv = ev;
      }
    }
    val[v] = cv;
    parent[v] = (int8_t)cand;
  }
  int tv = -1;
  double top = 0.0;
  for (int s = 0; s < n; ++s) {
    if (!(d.sink_mask >> s & 1u)) continue;
    bool take = tv < 0 || val[s] > top;
    if (!take && val[s] == top) {
      int8_t pa[OPSC_MAX_OPS], pb[OPSC_MAX_OPS];
      const int la = cp_path_of(parent, s, pa), lb = cp_path_of(parent, tv, pb);
      take = cp_seq_less(pa, la, pb, lb);
    }
    if (take) {
      tv = s;
      top = val[s];
    }
  }
  int len = 0;
  for (int u = tv; u >= 0; u = parent[u]) ++len;
  int i = len;
  for (int u = tv; u >= 0; u = parent[u]) path_out[--i] = (int8_t)u;
  for (int k = len; k < n; ++k) path_out[k] = (int8_t)-1;
  return top;
}

static __device__ __noinline__ double critical_path_lex(const OpscDag& d, const double* wt, int8_t* path_out,
                                                        double* val, int8_t* parent) {
  return critical_path_lex_body(d, wt, path_out, val, parent);
}

static __device__ __forceinline__ double critical_path_lex(const OpscDag& d, const double* wt, int8_t* path_out) {
  double val[OPSC_MAX_OPS];
  int8_t parent[OPSC_MAX_OPS];
  return critical_path_lex(d, wt, path_out, val, parent);
}

// the DAG is a single path: topo[0] a source, every later op fed by exactly
// the previous one, the last op the only sink (critical path = the whole
// chain, its latency the left-to-right sum of the weights)
__device__ __forceinline__ bool is_chain(const OpscDag& d) {
  const int n = d.n_ops;
  if (d.pred_mask[d.topo[0]] != 0u || d.sink_mask != (1u << d.topo[n - 1])) return false;
  for (int i = 1; i < n; ++i)
    if (d.pred_mask[d.topo[i]] != (1u << d.topo[i - 1])) return false;
  return true;
}

struct Pred {
  double t, lam, mu, util, wait, service, comm;
  bool stable;
};

// autoscaler.py:174-194 predict_op; status bits flag the reference's
// ZeroDivisionError / Unstable raises. SUM_ONLY: the caller uses `wait` only
// through wait + service (sojourn, weight) -- wait_for_sum may then return
// +0.0 for a wait below half an ulp of the service time (same sojourn bits).
// Reported PredictedSojourn fields (K4) use the exact form.
template <bool SUM_ONLY = false>
__device__ __forceinline__ Pred predict(const OpscDag& d, double qps, int L, int ph, int v, int p,
                                        int r, int b, uint32_t* st) {
  Pred o;
  o.t = op_latency(d, ph, v, b, L, p);
  const double tl = o.t * (double)d.layer_count[v];
  if (tl == 0.0) *st |= OPSC_W_ZERO_DIVISION;
  o.mu = 1.0 / tl;
  o.lam = qps / (double)b;
  o.stable = o.lam < (double)r * o.mu;
  o.util = o.lam / ((double)r * o.mu);
  o.wait = OPSC_INF;
  o.service = o.t / (double)b;
  if (o.stable) {
    if (o.util >= 1.0 || o.util <= 0.0) *st |= OPSC_W_UNSTABLE_ROUNDING;
    const double den = (double)r * o.mu - o.lam;
    o.wait = SUM_ONLY ? wait_for_sum(r, o.util, den, o.service) : erlang_c(r, o.util) / den;
  }
  o.comm = comm_time(d, v, b, L);
  return o;
}

// ((W + T/B) + C) * layers (autoscaler.py:751-755, opgraph.py:218)
__device__ __forceinline__ double weight(const Pred& o, int layers) {
  return ((o.wait + o.service) + o.comm) * (double)layers;
}

// menu entry -> (P, R, B), lexicographic (P, R, B) order (autoscaler.py:747-749)
__host__ __device__ __forceinline__ void entry_prb(const OpscGrid& g, int v, int e, int& p, int& r, int& b) {
  const int bm = g.b_max[v];
  b = e % bm + 1;
  r = (e / bm) % g.r_max + 1;
  p = g.p_vals[v][e / (bm * g.r_max)];
}

// CPython 3.12 builtin sum() over floats (Neumaier), used by placement memory
// bookkeeping and provisioned_memory (placement.py:171-172, metrics.py:130-132).
struct PySum {
  double f, c;
  bool started;
  __device__ void reset() { f = 0.0; c = 0.0; started = false; }
  __device__ void add(double x) {
    if (!started) { f = 0.0 + x; c = 0.0; started = true; return; }
    // both compensation terms, then a select: the same ops as the
    // reference's branch, but the f -> t chain (one DADD per element) is the
    // only serial dependency left (long replica sums in K4 / K6)
    const double t = f + x;
    const double d1 = (f - t) + x;
    const double d2 = (x - t) + f;
    c += fabs(f) >= fabs(x) ? d1 : d2;
    f = t;
  }
  __device__ double value() const {
    if (!started) return 0.0;
    return (c != 0.0 && isfinite(c)) ? f + c : f;
  }
};

// warp / block minimum of a u64 key
__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long x = __shfl_xor_sync(0xffffffffu, v, o);
    v = x < v ? x : v;
  }
  return v;
}

}  // namespace opsc

// ---------------------------------------------------------------- compose cfg
#define OPSC_CMAX (OPSC_MAX_OPS + 2)

// Host-computed view of one compose launch (topological positions).
struct ComposeCfg {
  int32_t n;            // positions (>= 2, virtual positions prepended when needed)
  int32_t il;           // inner levels held by one thread (>= 2)
  int32_t E;            // menu entries per window (window stride of menu_w)
  int32_t n_real_ops;
  int32_t m[OPSC_CMAX];        // menu size per position
  int32_t off[OPSC_CMAX];      // menu offset per position (virtual -> E)
  unsigned long long stride[OPSC_CMAX];  // lexicographic stride per position (0 virtual)
  uint32_t pmask[OPSC_CMAX];   // predecessor positions
  uint32_t sinkmask;           // sink positions
  uint32_t m_out;              // outer index space per window
  uint32_t lo, hi;             // this shard's outer index range
  uint32_t mid_count;          // product of middle-level menu sizes
  int32_t blocks_per_window;
  int32_t spc;                 // 256-thread slices per CTA (tile kernel)
  int32_t nj;                  // register tile of the innermost menu
  int32_t chain;               // j's only predecessor is k and k is not a sink
  int32_t tkey;                // 32-bit in-thread keys span the middle levels too (cs over all in-thread positions)
  uint32_t cs[OPSC_CMAX];      // compact in-thread lexicographic strides (local key index = sum dig * cs)
  int32_t path_dag;            // in-thread positions form a path ending in the only in-thread sink (middle-level odometer)
  int32_t flat;                // menus too large for the shared-memory tile: flat kernel over the candidate index
  int32_t vop[OPSC_CMAX];      // real operator per position (-1 virtual)
  unsigned long long flo, fhi; // flat kernel: this shard's candidate index range
};

namespace opsc {
// Host launch with the programmatic-stream-serialization attribute (see
// pdl_wait); OPSC_NO_PDL=1 launches plainly (A/B switch).
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* f = getenv("OPSC_NO_PDL");
    return !(f && f[0] == '1');
  }();
  return on;
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

// launchers (defined in the k_*.cu files), all asynchronous on `s`
cudaError_t launch_init(int n_windows, const double* qps, uint32_t* status, unsigned long long* key,
                        uint8_t* feasible, cudaStream_t s);
cudaError_t launch_menu_build(const OpscDag& d, const OpscGrid& g, OpscWindows w, double* menu_w,
                              uint32_t* status, cudaStream_t s);
cudaError_t launch_stability(const OpscDag& d, const OpscGrid& g, OpscWindows w, uint32_t* status,
                             cudaStream_t s);
cudaError_t launch_fallback(const OpscDag& d, const OpscGrid& g, int n_windows, const double* menu_w,
                            int32_t* fb, cudaStream_t s);
cudaError_t launch_decode(const OpscDag& d, const OpscGrid& g, int n_windows,
                          const unsigned long long* key, const int32_t* fb, int16_t* cfg,
                          uint8_t* feasible, uint32_t* status, cudaStream_t s);
cudaError_t launch_fill_keys(unsigned long long* key, int n, cudaStream_t s);
int compose_setup(const OpscDag& d, const OpscGrid& g, int n_windows, int shard, int n_shards,
                  ComposeCfg* cfg);
// peer key buffers for the fused multi-GPU merge (n = 0: local atomics only)
struct PeerKeys {
  unsigned long long* p[OPSC_MAX_PEERS];
  int32_t n;
};
struct PeerFlags {
  uint32_t* p[OPSC_MAX_PEERS];
};
cudaError_t launch_compose(const ComposeCfg& c, const OpscGrid& g, int n_windows,
                           const double* menu_w, const double* slo, const double* qps,
                           unsigned long long* key, cudaStream_t s, const PeerKeys* peers = nullptr);
cudaError_t launch_compose_boundary(const ComposeCfg& c, const OpscGrid& g, int n_windows, const double* menu_w,
                                    const double* slo, const double* qps, double band_ulps,
                                    unsigned long long* count, cudaStream_t s);
size_t certify_workspace(int n_windows);
cudaError_t launch_certify(const ComposeCfg& c, const OpscGrid& g, int n_windows, const double* menu_w,
                           const double* slo, const double* qps, double band_ulps, void* ws, uint32_t* status,
                           cudaStream_t s);
cudaError_t launch_peer_barrier(const PeerFlags& f, int rank, int n, uint32_t epoch, int timeout_ms,
                                int32_t* err, cudaStream_t s);
cudaError_t launch_model_grid(const OpscDag& d, const OpscModelSpec& m, OpscWindows w, int16_t* cfg,
                              uint8_t* feasible, uint32_t* status, cudaStream_t s,
                              void* table_ws = nullptr, size_t table_bytes = 0);
size_t model_table_bytes(int n_windows, const OpscModelSpec& m, int n_ops);
cudaError_t launch_materialize(const OpscDag& d, OpscWindows w, int config_order,
                               const OpscPlaceSpec& p, OpscDecisions out, cudaStream_t s);
cudaError_t launch_menu_stability(const OpscDag& d, const OpscGrid& g, OpscWindows w, double* menu_w,
                                  uint32_t* status, cudaStream_t s);
cudaError_t launch_decode_materialize(const OpscDag& d, const OpscGrid& g, OpscWindows w,
                                      const unsigned long long* key, const double* menu_w, const OpscPlaceSpec& p,
                                      OpscDecisions out, cudaStream_t s);
cudaError_t launch_fp64_peak(int iters, double* sink, int* blocks, int* threads, cudaStream_t s);
cudaError_t launch_greedy(const OpscDag& d, const OpscGreedySpec& s, OpscWindows w, const int16_t* ucfg,
                          const uint8_t* ufeas, const uint32_t* ustatus, OpscDecisions out, cudaStream_t st,
                          int phase = 0, void* save = nullptr);
size_t greedy_state_bytes(int n_windows);
size_t windowize_workspace(long long n, int max_w);
size_t place_shared_workspace(int n_windows, int A, int D, int n);
cudaError_t launch_interference_pow(const double* x, const double* e, double* out, long long n, cudaStream_t s);
cudaError_t launch_place_shared(const OpscDag& d, const OpscPlaceShared& f, OpscWindows w, const int16_t* cfg,
                                const uint8_t* feas, int config_order, OpscPlacement out, void* ws,
                                size_t ws_bytes, cudaStream_t s);
cudaError_t launch_windowize(OpscTraceRecords rec, double len, double q, int max_w, int32_t* n_windows,
                             double* pq, int32_t* pl, double* dq, void* ws, size_t ws_bytes, cudaStream_t s);
}  // namespace opsc
