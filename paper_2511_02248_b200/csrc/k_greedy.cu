// k_greedy.cu -- K5: greedy_autoscale (operator-level planner) on the device.
//
// One CTA per window runs the reference's sequential algorithm
// (autoscaler.py:334-589) with the data-parallel parts spread over threads:
//   * init_configs (:254-294): (op, B) pairs in parallel per parallelism rank;
//   * every upscale / downscale / headroom step evaluates its whole move set
//     (all distinct (B, P) at R +- 1 for the bottleneck operator, :306-331) in
//     parallel -- one thread per move: predict_op for the moved operator and
//     the critical-path DP with that operator's weight replaced;
//   * the reference's selection keys are lexicographic minima with a unique
//     (B, P) tie-break, so each is a block-wide reduction (warp shuffles);
//     thread 0 applies the pick and recomputes the critical path (with its
//     lexicographic tie-break) for the bottleneck of the next step; the
//     prune pass is sequential as in :562-589.
// The uniform reseed uses K3's model-level result for the same window.
// The step functions are __noinline__: inlined at every call site the kernel
// was 32k instructions (512 KB of SASS) and a single-window run spent ~22% of
// its warp samples waiting on instruction fetch (ncu stall "no_inst").
#include <cstdio>
#include <cstring>

#include "opsc_common.cuh"

namespace opsc {

#ifndef OPSC_GREEDY_THREADS
#define OPSC_GREEDY_THREADS 384  // 128 evaluate and commit a move, 256 speculate the next move sets
#endif
constexpr int kGreedyThreads = OPSC_GREEDY_THREADS;
constexpr int kMaxMoves = 256;                   // move-set chunk (larger sets run in chunks)
constexpr int kInitChunk = 64;                   // init_configs B chunk per operator
constexpr int kCore = 128;                       // threads that evaluate, reduce and commit a step
constexpr int kSpecMoves = 128;                  // largest speculated move set (one per spec thread)
static_assert(kGreedyThreads == kCore || kGreedyThreads == kCore + 2 * kSpecMoves, "core + two speculated sets");

struct GreedyArgs {
  OpscDag d;
  OpscGreedySpec s;
};

constexpr size_t kGreedyArgsWords = (sizeof(GreedyArgs) + 15) / 16;  // dynamic smem: copied args first

struct GShared {
  int p[OPSC_MAX_OPS], r[OPSC_MAX_OPS], b[OPSC_MAX_OPS];
  double soj[OPSC_MAX_OPS], wt[OPSC_MAX_OPS];
  int8_t path[OPSC_MAX_OPS];
  double lat;
  int stable;
  // move results
  double m_lat[kMaxMoves], m_soj[kMaxMoves], m_wt[kMaxMoves];
  uint8_t m_ok[kMaxMoves];
  // init scratch (one B chunk) and the running per-op argmin over chunks
  double i_soj[OPSC_MAX_OPS][kInitChunk];
  int i_r[OPSC_MAX_OPS][kInitChunk];
  double i_bs[OPSC_MAX_OPS];
  int i_bb[OPSC_MAX_OPS], i_br[OPSC_MAX_OPS];
  int chosen[OPSC_MAX_OPS];
  // control
  int op, applied, flag;
  int np_d[OPSC_MAX_OPS];
  int pd[OPSC_MAX_OPS][OPSC_MAX_P];
  uint32_t st;
  int trace_len;
  int bneck;                     // bottleneck of the current path (set with the path)
  double cpv[OPSC_MAX_OPS];      // critical-path DP values of the current weights (thread 0's walk)
  int8_t cppar[OPSC_MAX_OPS];
  int8_t tpos[OPSC_MAX_OPS];     // topological position of every op
  int cpv_ok;                    // cpv matches wt and every weight is >= 0 (trial_latency prefix)
  int chain;                     // the DAG is one path (each op feeds the next in topological order)
  // speculated move sets, [parity][set]: predict_op of (op, P, R, B >= B_lo)
  // for a key (op, R, B_lo) -- a pure function of the key, so valid whenever
  // it matches; step c consumes parity c & 1 and fills parity (c + 1) & 1
  double n_wt[2][2][kSpecMoves], n_soj[2][2][kSpecMoves];
  uint8_t n_ok[2][2][kSpecMoves];
  int n_op[2][2], n_r[2][2], n_blo[2][2], n_M[2][2], n_valid[2][2];
  uint32_t n_st[2][2];           // status bits of the speculated points, ORed in when consumed
};

// barrier of the kCore threads that run a step's evaluation, reduction and
// commit (the speculating threads only meet them at the step's end)
__device__ __forceinline__ void core_sync() {
  if (kGreedyThreads == kCore) __syncthreads();
  else asm volatile("barrier.sync 1, %0;" ::"n"(kCore) : "memory");
}


// latency of the current plan with op `v`'s weight replaced (value only).
// prefix: S.cpv holds the DP values of the current weights and every weight
// is >= 0 (S.cpv_ok) -- then the values of v's topological predecessors in
// the order are unchanged and the DP restarts at v (for weights >= 0 the
// critical-path DP and this one, which clamps dp_in at 0, agree bit for bit).
__device__ double trial_latency(const GShared& S, const OpscDag& d, const double* wt, int v, double wv,
                                bool prefix) {
  if (!prefix && S.chain) {  // a chain, literally the DP below: t = max(0, t) + w in topological order
    double t = 0.0;
    for (int i = 0; i < d.n_ops; ++i) {
      const int u = d.topo[i];
      t = fmax(0.0, t) + (u == v ? wv : wt[u]);
    }
    return fmax(0.0, t);
  }
  if (prefix && S.chain) {  // a chain: one running value from v's predecessor on
    const int n = d.n_ops, i0 = S.tpos[v];
    double t = i0 > 0 ? S.cpv[d.topo[i0 - 1]] : 0.0;  // >= 0 (all weights >= 0)
    t = t + wv;
    for (int i = i0 + 1; i < n; ++i) t = t + wt[d.topo[i]];
    return fmax(0.0, t);
  }
  double val[OPSC_MAX_OPS];
  double top = 0.0;
  int i0 = 0;
  if (prefix) {
    i0 = S.tpos[v];
    for (int i = 0; i < i0; ++i) {
      const int u = d.topo[i];
      if (d.sink_mask >> u & 1u) top = fmax(top, S.cpv[u]);
    }
  }
  for (int i = i0; i < d.n_ops; ++i) {
    const int u = d.topo[i];
    double in = 0.0;
    uint32_t pm = d.pred_mask[u];
    while (pm) {
      const int p = __ffs(pm) - 1;
      pm &= pm - 1;
      in = fmax(in, S.tpos[p] < i0 ? S.cpv[p] : val[p]);
    }
    val[u] = in + (u == v ? wv : wt[u]);
    if (d.sink_mask >> u & 1u) top = fmax(top, val[u]);
  }
  return top;
}

__device__ int objective(const GShared& S, int n) {
  int o = 0;
  for (int v = 0; v < n; ++v) o += S.p[v] * S.r[v];
  return o;
}

__device__ int bottleneck(const GShared& S, int n) {
  int best = -1;
  for (int i = 0; i < n && S.path[i] >= 0; ++i) {
    const int v = S.path[i];
    if (best < 0 || S.soj[v] > S.soj[best] || (S.soj[v] == S.soj[best] && v < best)) best = v;
  }
  return best;
}

// thread 0: critical path of the current weights with the reference's
// lexicographic path tie-break (opgraph.py:223-244), DP scratch in shared
// memory, and the bottleneck the next step starts from (:306-331) -- so the
// steps need no serial section of their own before evaluating moves
__device__ __noinline__ void set_path(GShared& S, const OpscDag& d) {
  if (S.chain) {  // one source-sink path: val[v] = val[prev] + w[v] in order, the path is every op
    const int n = d.n_ops;
    double acc = 0.0;
    for (int i = 0; i < n; ++i) {
      const int u = d.topo[i];
      acc = i == 0 ? S.wt[u] : acc + S.wt[u];
      S.cpv[u] = acc;
      S.path[i] = (int8_t)u;
    }
    S.lat = acc;
  } else {
    S.lat = critical_path_lex_body(d, S.wt, S.path, S.cpv, S.cppar);
  }
  S.bneck = bottleneck(S, d.n_ops);
  bool nonneg = true;
  for (int v = 0; v < d.n_ops; ++v) nonneg &= S.wt[v] >= 0.0;
  S.cpv_ok = nonneg;
}

__device__ void push_trace(GShared& S, const OpscDecisions& out, int w, int action, int op, int r,
                           int b, int p, double lat, int obj) {
  if (S.trace_len < out.trace_cap) {
    OpscTraceEntry* t = out.trace + (size_t)w * out.trace_cap + S.trace_len;
    t->latency = lat;
    t->objective = obj;
    t->to_r = (int16_t)r;
    t->to_b = (int16_t)b;
    t->to_p = (int16_t)p;
    t->op = (int8_t)op;
    t->action = (uint8_t)action;
    t->reserved = 0;
  }
  S.trace_len++;
}

// one out-of-line copy of predict_op for the whole kernel (instruction-cache
// footprint; called per thread, the call overhead is a few instructions)
__device__ __noinline__ Pred gpredict(const OpscDag& d, double qps, int L, int ph, int v, int p, int r, int b,
                                      uint32_t* st) {
  return predict<true>(d, qps, L, ph, v, p, r, b, st);
}

// predict_op of (v, P, R, B) for window w as the steps use it
struct GPt {
  double wt, soj;
  bool ok;
};

__device__ __forceinline__ GPt gpoint(const GreedyArgs& a, int w, double qps, int L, int ph, int v, int p, int r,
                                      int b, uint32_t* st) {
  (void)w;
  const Pred o = gpredict(a.d, qps, L, ph, v, p, r, b, st);
  return GPt{weight(o, a.d.layer_count[v]), o.wait + o.service, o.stable};
}

__device__ __noinline__ void set_path_warp(GShared& S, const OpscDag& d);

// full evaluation of the current configs (all threads; ends synchronised)
__device__ __noinline__ void eval_full(GShared& S, const GreedyArgs& a, int w, double qps, int L, int ph) {
  const OpscDag& d = a.d;
  __shared__ int s_unstable;
  if (threadIdx.x == 0) s_unstable = 0;
  __syncthreads();
  for (int v = threadIdx.x; v < d.n_ops; v += blockDim.x) {
    uint32_t st = 0;
    const GPt o = gpoint(a, w, qps, L, ph, v, S.p[v], S.r[v], S.b[v], &st);
    S.soj[v] = o.soj;
    S.wt[v] = o.wt;
    if (!o.ok) atomicOr(&s_unstable, 1);
    if (st) atomicOr(&S.st, st);
  }
  __syncthreads();
  if (threadIdx.x < 32) {  // warp 0
    const bool stable = !s_unstable;
    if (stable) {
      set_path_warp(S, d);
    } else if (threadIdx.x == 0) {
      S.lat = OPSC_INF;
      for (int i = 0; i < d.n_ops; ++i) S.path[i] = -1;
      S.bneck = -1;
      S.cpv_ok = 0;
    }
    if (threadIdx.x == 0) S.stable = stable;
  }
  __syncthreads();
}

// Evaluate moves [m0, m0 + kMaxMoves) of the move set of `op` at replica
// count r_new (move m = (B = b_lo + m / np, P = pd[m % np]), all distinct P)
// into the scratch slots m - m0 (the kCore threads; ends core-synchronised).
// Returns the size of the whole set; sets larger than kMaxMoves run in
// chunks. A speculated set of parity `par` with this key supplies the
// predict_op values.
__device__ __noinline__ int eval_moves(GShared& S, const GreedyArgs& a, int w, int op, int r_new, int b_lo, double qps,
                                       int L, int ph, int m0, int par) {
  const int np = S.np_d[op];
  const int nb = a.s.b_max[op] - b_lo + 1;
  const int M = nb * np;
  const int m1 = min(M, m0 + kMaxMoves);
  int spec = -1;
  if (m0 == 0)
    for (int q = 0; q < 2; ++q)
      if (S.n_valid[par][q] && S.n_op[par][q] == op && S.n_r[par][q] == r_new && S.n_blo[par][q] == b_lo &&
          S.n_M[par][q] == M)
        spec = q;
  for (int m = m0 + threadIdx.x; m < m1; m += kCore) {
    const int b = b_lo + m / np, p = S.pd[op][m % np];
    uint32_t st = 0;
    const GPt o = spec >= 0 ? GPt{S.n_wt[par][spec][m], S.n_soj[par][spec][m], S.n_ok[par][spec][m] != 0}
                            : gpoint(a, w, qps, L, ph, op, p, r_new, b, &st);
    const int i = m - m0;
    S.m_ok[i] = o.ok;
    if (o.ok) {
      S.m_wt[i] = o.wt;
      S.m_soj[i] = o.soj;
      S.m_lat[i] = trial_latency(S, a.d, S.wt, op, S.m_wt[i], S.cpv_ok);
    }
    if (st) atomicOr(&S.st, st);
  }
  core_sync();
  if (threadIdx.x == 0 && m0 == 0) {  // consumed or superseded
    if (spec >= 0) S.st |= S.n_st[par][spec];
    S.n_valid[par][0] = S.n_valid[par][1] = 0;
  }
  return M;
}

// Speculation (threads kCore.. of an upscale step, concurrently with the
// step's evaluation / reduction / commit): on a chain the next bottleneck is
// either the moved operator itself or, whatever the pick, the argmax of the
// other operators' sojourns -- so the two upscale move sets the next step can
// need, (op, R + 2, 1) and (op2, R_op2 + 1, 1), are evaluated now into the
// buffers of parity `par`. Wrong guesses (a downscale next, or an early
// stop) only cost idle threads' work: a set is used on an exact key match.
__device__ void speculate_up(GShared& S, const GreedyArgs& a, int w, double qps, int L, int ph, int op, int cur_r,
                             int par) {
  const int t = (int)threadIdx.x - kCore;  // 0 .. 2 * kSpecMoves - 1
  const int q = t / kSpecMoves, m = t - q * kSpecMoves;
  const int n = a.d.n_ops;
  int v = op, r = cur_r + 2;
  if (q == 1) {  // bottleneck() over every op but `op` (the chain's path is every op, topological order)
    v = -1;
    double sv = 0.0;
    for (int i = 0; i < n; ++i) {
      const int u = a.d.topo[i];
      if (u == op) continue;
      const double su = S.soj[u];
      if (v < 0 || su > sv || (su == sv && u < v)) {
        v = u;
        sv = su;
      }
    }
    if (v < 0) return;
    r = S.r[v] + 1;
  }
  const int np = S.np_d[v];
  const int M = a.s.b_max[v] * np;
  if (r > a.s.r_cap || M > kSpecMoves) return;
  uint32_t st = 0;
  if (m < M) {
    const GPt o = gpoint(a, w, qps, L, ph, v, S.pd[v][m % np], r, 1 + m / np, &st);
    S.n_wt[par][q][m] = o.wt;
    S.n_soj[par][q][m] = o.soj;
    S.n_ok[par][q][m] = o.ok;
  }
  if (st) atomicOr(&S.n_st[par][q], st);
  if (m == 0) {
    S.n_op[par][q] = v;
    S.n_r[par][q] = r;
    S.n_blo[par][q] = 1;
    S.n_M[par][q] = M;
    S.n_valid[par][q] = 1;
  }
}

// A move's selection key (k0, k1, k2, B, P) for one of the reference's
// criteria. Keys end in the move's unique (B, P), so the lexicographic
// minimum is a total order: the block reduction below picks exactly the move
// the reference's in-order scan picks. (k2, B, P) travel packed in one u64
// (k2 >= 0, B and P < 2^16); "no candidate" is (+inf, +inf, ~0) -- k0 and
// k1 of a real move are never +inf (objectives, -(dlat/dobj) and stable
// latencies). The move index is recovered from (B, P) (move_index).
struct PK {
  double k0, k1;
  unsigned long long tie;
};

__device__ __forceinline__ PK pk_none() { return PK{OPSC_INF, OPSC_INF, ~0ull}; }
__device__ __forceinline__ PK pk_make(double k0, double k1, int k2, int b, int p) {
  return PK{k0, k1, ((unsigned long long)(uint32_t)k2 << 32) | ((unsigned long long)b << 16) | (unsigned long long)p};
}
__device__ __forceinline__ bool pk_valid(const PK& x) { return x.tie != ~0ull; }
__device__ __forceinline__ int pk_b(const PK& x) { return (int)((x.tie >> 16) & 0xffffu); }
__device__ __forceinline__ int pk_p(const PK& x) { return (int)(x.tie & 0xffffu); }

// branch-free lexicographic (k0, k1, tie) compare (NaN compares false
// everywhere, as in the branchy form)
__device__ __forceinline__ bool pk_less(const PK& x, const PK& y) {
  const bool e0 = x.k0 == y.k0, e1 = x.k1 == y.k1;
  return (x.k0 < y.k0) | (e0 & ((x.k1 < y.k1) | (e1 & (x.tie < y.tie))));
}

__device__ __forceinline__ PK pk_shfl(const PK& x, int off) {
  PK y;
  y.k0 = __shfl_xor_sync(0xffffffffu, x.k0, off);
  y.k1 = __shfl_xor_sync(0xffffffffu, x.k1, off);
  y.tie = __shfl_xor_sync(0xffffffffu, x.tie, off);
  return y;
}

// index m of move (B, P) in the move set of `op` starting at b_lo
__device__ __forceinline__ int move_index(const GShared& S, int op, int b_lo, int b, int p) {
  const int np = S.np_d[op];
  int pi = 0;
  while (pi < np - 1 && S.pd[op][pi] != p) ++pi;
  return (b - b_lo) * np + pi;
}

// Block-wide minimum of NK keys per thread (warp shuffles, then one warp
// over the per-warp minima). The kCore threads; the result in x[] on every
// thread (W0: on warp 0 only -- the steps' commit runs there -- and no
// closing barrier: the buffer is next written after the step's end)
template <int NK, bool W0 = false>
__device__ void block_min(PK (&x)[NK]) {  // the kCore threads
  __shared__ PK red[kCore / 32][NK];
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int k = 0; k < NK; ++k) {
      const PK y = pk_shfl(x[k], off);
      if (pk_less(y, x[k])) x[k] = y;
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < NK; ++k) red[warp][k] = x[k];
  core_sync();
  if (W0 && warp != 0) return;
#pragma unroll
  for (int k = 0; k < NK; ++k) {
    PK v = red[0][k];
    for (int w2 = 1; w2 < kCore / 32; ++w2)
      if (pk_less(red[w2][k], v)) v = red[w2][k];
    x[k] = v;
  }
  if (!W0) core_sync();
}

// warp 0 (all lanes): set_path's results with the serial parts spread over
// the lanes -- a chain's weights gathered by shuffles and summed left to
// right in every lane (lane i keeps the DP value of position i), the
// bottleneck as a warp (sojourn, -id) max by integer reductions (literal
// scan if a sojourn is NaN), the non-negativity check as a vote. Same values as set_path.
// Out of line: one copy serves the step commits, the prune pass and
// eval_full (the kernel's code is larger than the instruction cache, and a
// step's serial tail runs cold code otherwise).
__device__ __noinline__ void set_path_warp(GShared& S, const OpscDag& d) {
  const int lane = threadIdx.x & 31, n = d.n_ops;
  if (S.chain) {
    const int u = lane < n ? d.topo[lane] : 0;
    const double wl = lane < n ? S.wt[u] : 0.0;
    double acc = 0.0, mine = 0.0;
    for (int i = 0; i < n; ++i) {
      const double wi = __shfl_sync(0xffffffffu, wl, i);
      acc = i == 0 ? wi : acc + wi;
      if (lane == i) mine = acc;
    }
    if (lane < n) {
      S.cpv[u] = mine;
      S.path[lane] = (int8_t)u;
    }
    if (lane == 0) S.lat = acc;
  } else if (lane == 0) {
    S.lat = critical_path_lex_body(d, S.wt, S.path, S.cpv, S.cppar);
  }
  __syncwarp();
  const int v = lane < n ? S.path[lane] : -1;
  const double sj = v >= 0 ? S.soj[v] : 0.0;
  const bool nan = __any_sync(0xffffffffu, v >= 0 && sj != sj);
  // (sojourn, -id) maximum as three warp reductions over an order-preserving
  // integer image of the sojourn: the highest word, then the low word among
  // those, then the lowest id among the equal ones (-0.0 is folded into +0.0,
  // they compare equal as doubles; a NaN takes the literal scan below)
  const long long sb = __double_as_longlong(sj + 0.0);
  const unsigned long long key = sb < 0 ? ~(unsigned long long)sb : (unsigned long long)sb | 0x8000000000000000ull;
  const unsigned hi = v >= 0 ? (unsigned)(key >> 32) : 0u, lo = v >= 0 ? (unsigned)key : 0u;
  const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
  const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
  const int bv = (int)__reduce_min_sync(0xffffffffu, v >= 0 && hi == mh && lo == ml ? (unsigned)v : 0xffffffffu);
  const bool nonneg = __all_sync(0xffffffffu, lane >= n || S.wt[lane] >= 0.0);
  if (lane == 0) {
    S.bneck = nan ? bottleneck(S, n) : bv;
    S.cpv_ok = nonneg;
  }
  __syncwarp();
}

__device__ __forceinline__ int objective_warp(const GShared& S, int n) {
  const int lane = threadIdx.x & 31;
  return __reduce_add_sync(0xffffffffu, lane < n ? S.p[lane] * S.r[lane] : 0);
}

// warp 0: apply move m of `op` (new r; lane 0 updates the config and the
// move's weight / sojourn -- from the scratch when its chunk is the last one
// evaluated, else recomputed, same bits) and the path (set_path_warp)
__device__ __forceinline__ void apply_move_warp(GShared& S, const GreedyArgs& a, int w, int op, int m, int r_new, int b_lo,
                                             int m0, double qps, int L, int ph) {
  if ((threadIdx.x & 31) == 0) {
    const int np = S.np_d[op];
    S.p[op] = S.pd[op][m % np];
    S.b[op] = b_lo + m / np;
    S.r[op] = r_new;
    if (m >= m0 && m < m0 + kMaxMoves) {
      S.wt[op] = S.m_wt[m - m0];
      S.soj[op] = S.m_soj[m - m0];
    } else {
      uint32_t st = 0;
      const GPt o = gpoint(a, w, qps, L, ph, op, S.p[op], r_new, S.b[op], &st);
      S.wt[op] = o.wt;
      S.soj[op] = o.soj;
    }
    S.stable = 1;
  }
  __syncwarp();
  set_path_warp(S, a.d);
}

// One upscale step (greedy loop when headroom == false, _restore_headroom
// otherwise). All threads; returns (via S.applied) whether a move was made.
// Selection (autoscaler.py:395-455; headroom :503-557): first the cheapest
// move reaching slo - eps (objective, latency, B, P), then (loop only) the
// cheapest reaching slo, else the most efficient improving move
// (-(dlat / dobj), latency, objective, B, P) -- each a block-wide minimum.
__device__ __forceinline__ void upscale_core(GShared& S, const GreedyArgs& a, const OpscDecisions& out, int w,
                                             double qps, int L, int ph, double slo, double eps, bool headroom, int c,
                                             int op, int cur_p, int cur_r);
__device__ __forceinline__ void downscale_core(GShared& S, const GreedyArgs& a, const OpscDecisions& out, int w,
                                               double qps, int L, int ph, double slo, double eps, int c, int op,
                                               int cur_p, int cur_r, int cur_b);

__device__ __noinline__ void upscale_step(GShared& S, const GreedyArgs& a, const OpscDecisions& out, int w, double qps,
                                          int L, int ph, double slo, double eps, bool headroom, int c) {
  const int op = S.bneck;  // set with the current path (every writer ends synchronised)
  const int cur_p = S.p[op], cur_r = S.r[op];
  if (cur_r + 1 > a.s.r_cap) {
    __syncthreads();
    if (threadIdx.x == 0) S.applied = 0;
    __syncthreads();
    return;
  }
  if ((int)threadIdx.x >= kCore) {  // speculate the next step's two candidate move sets
    if (S.chain) speculate_up(S, a, w, qps, L, ph, op, cur_r, (c + 1) & 1);
  } else {
    upscale_core(S, a, out, w, qps, L, ph, slo, eps, headroom, c, op, cur_p, cur_r);
  }
  __syncthreads();  // one barrier instruction for the whole CTA
}

// the kCore threads' part of an upscale step
__device__ __forceinline__ void upscale_core(GShared& S, const GreedyArgs& a, const OpscDecisions& out, int w,
                                             double qps, int L, int ph, double slo, double eps, bool headroom, int c,
                                             int op, int cur_p, int cur_r) {
  const int np = S.np_d[op];
  const int base = objective_warp(S, a.d.n_ops);  // every warp: one add-reduction
  const double target = slo - eps, cur_lat = S.lat;
  PK k[3];  // ach, ach2, imp
  for (int i = 0; i < 3; ++i) k[i] = pk_none();
  int M = 0, m0 = 0;
#ifdef OPSC_GREEDY_PROF
  const long long u0 = clock64();
  long long u1 = 0;
#endif
  do {
    if (m0 > 0) core_sync();  // previous chunk's scratch fully read
    M = eval_moves(S, a, w, op, cur_r + 1, 1, qps, L, ph, m0, c & 1);
#ifdef OPSC_GREEDY_PROF
    u1 = clock64();
#endif
    for (int m = m0 + threadIdx.x; m < min(M, m0 + kMaxMoves); m += kCore) {
      if (!S.m_ok[m - m0]) continue;
      const int b = 1 + m / np, p = S.pd[op][m % np];
      const double lat = S.m_lat[m - m0];
      const int obj = base - cur_p * cur_r + p * (cur_r + 1);
      const PK reach = pk_make((double)obj, lat, 0, b, p);
      if (lat <= target && pk_less(reach, k[0])) k[0] = reach;
      if (!headroom && lat <= slo && pk_less(reach, k[1])) k[1] = reach;
      const bool improving = headroom ? lat < cur_lat - 1e-9 * slo : lat < cur_lat;
      if (improving) {
        const int dobj = obj - base;
        const double cost = dobj >= 1 ? (double)dobj : 1e-9;
        const PK eff = pk_make(-((cur_lat - lat) / cost), lat, headroom ? 0 : obj, b, p);
        if (pk_less(eff, k[2])) k[2] = eff;
      }
    }
    m0 += kMaxMoves;
  } while (m0 < M);
  m0 -= kMaxMoves;  // the chunk still in the scratch
#ifdef OPSC_GREEDY_PROF
  const long long u2 = clock64();
#endif
  block_min<3, true>(k);
#ifdef OPSC_GREEDY_PROF
  const long long u3 = clock64();
#endif
  if (threadIdx.x < 32) {  // warp 0 applies the pick (every thread holds the same minima)
    const PK& pick = pk_valid(k[0]) ? k[0] : (!headroom && pk_valid(k[1])) ? k[1] : k[2];
    const int m = pk_valid(pick) ? move_index(S, op, 1, pk_b(pick), pk_p(pick)) : -1;
    if (threadIdx.x == 0) S.applied = m >= 0;
    if (m >= 0) {
#if defined(OPSC_GREEDY_PROF) && defined(OPSC_GREEDY_PROF_STEPS)
      const long long a0 = clock64();
#endif
      apply_move_warp(S, a, w, op, m, cur_r + 1, 1, m0, qps, L, ph);
#if defined(OPSC_GREEDY_PROF) && defined(OPSC_GREEDY_PROF_STEPS)
      const long long a1 = clock64();
#endif
      const int obj = objective_warp(S, a.d.n_ops);
      if (threadIdx.x == 0)
        push_trace(S, out, w, headroom ? OPSC_ACT_HEADROOM : OPSC_ACT_UPSCALE, op, S.r[op], S.b[op], S.p[op],
                   S.lat, obj);
#if defined(OPSC_GREEDY_PROF) && defined(OPSC_GREEDY_PROF_STEPS)
      if (threadIdx.x == 0) printf("    apply: pick %lld move+path %lld trace %lld\n", a0 - u3, a1 - a0, clock64() - a1);
#endif
    }
  }
#if defined(OPSC_GREEDY_PROF) && defined(OPSC_GREEDY_PROF_STEPS)  // per-step split (slows the loop)
  if (threadIdx.x == 0)
    printf("  up step op %d r %d M %d: eval %lld keys %lld reduce %lld apply %lld cycles\n", op, cur_r + 1, M,
           u1 - u0, u2 - u1, u3 - u2, clock64() - u3);
#endif
}

// Downscale (autoscaler.py:456-486): the cheapest (objective, B, P) move at
// R - 1 that stays within slo - eps and lowers the objective.
__device__ __noinline__ void downscale_step(GShared& S, const GreedyArgs& a, const OpscDecisions& out, int w,
                                            double qps, int L, int ph, double slo, double eps, int c) {
  const int op = S.bneck;  // set with the current path (every writer ends synchronised)
  const int cur_p = S.p[op], cur_r = S.r[op], cur_b = S.b[op];
  if (cur_r - 1 < 1) {
    __syncthreads();
    if (threadIdx.x == 0) S.applied = 0;
    __syncthreads();
    return;
  }
  if ((int)threadIdx.x < kCore) downscale_core(S, a, out, w, qps, L, ph, slo, eps, c, op, cur_p, cur_r, cur_b);
  __syncthreads();  // one barrier instruction for the whole CTA (nothing speculated after a downscale)
}

__device__ __forceinline__ void downscale_core(GShared& S, const GreedyArgs& a, const OpscDecisions& out, int w,
                                               double qps, int L, int ph, double slo, double eps, int c, int op,
                                               int cur_p, int cur_r, int cur_b) {
  const int np = S.np_d[op];
  const int base = objective_warp(S, a.d.n_ops);  // every warp: one add-reduction
  const double bound = slo - eps;
  PK k[1];
  k[0] = pk_none();
  int M = 0, m0 = 0;
  do {
    if (m0 > 0) core_sync();  // previous chunk's scratch fully read
    M = eval_moves(S, a, w, op, cur_r - 1, cur_b, qps, L, ph, m0, c & 1);
    for (int m = m0 + threadIdx.x; m < min(M, m0 + kMaxMoves); m += kCore) {
      if (!S.m_ok[m - m0] || S.m_lat[m - m0] > bound) continue;
      const int b = cur_b + m / np, p = S.pd[op][m % np];
      const int obj = base - cur_p * cur_r + p * (cur_r - 1);
      if (obj >= base) continue;
      const PK cand = pk_make((double)obj, 0.0, 0, b, p);
      if (pk_less(cand, k[0])) k[0] = cand;
    }
    m0 += kMaxMoves;
  } while (m0 < M);
  m0 -= kMaxMoves;
  block_min<1, true>(k);
  if (threadIdx.x < 32) {
    const int best = pk_valid(k[0]) ? move_index(S, op, cur_b, pk_b(k[0]), pk_p(k[0])) : -1;
    if (threadIdx.x == 0) S.applied = best >= 0;
    if (best >= 0) {
      apply_move_warp(S, a, w, op, best, cur_r - 1, cur_b, m0, qps, L, ph);
      const int obj = objective_warp(S, a.d.n_ops);
      if (threadIdx.x == 0)
        push_trace(S, out, w, OPSC_ACT_DOWNSCALE, op, S.r[op], S.b[op], S.p[op], S.lat, obj);
    }
  }
}

__device__ __noinline__ void greedy_loop(GShared& S, const GreedyArgs& a, const OpscDecisions& out, int w, double qps,
                            int L, int ph, double slo, double eps) {
  for (int it = 0; it < a.s.max_iterations; ++it) {
    const double lat = S.lat;
    if (lat > slo) {
      upscale_step(S, a, out, w, qps, L, ph, slo, eps, false, it);
    } else if (lat <= slo - eps) {
      downscale_step(S, a, out, w, qps, L, ph, slo, eps, it);
    } else {
      break;
    }
    if (!S.applied) break;
  }
}

// _prune_pass (:562-589). The sweep itself is sequential (each accepted
// prune changes the state the next trial sees), but a trial's predict_op
// depends only on its own operator's config, so the Erlang-B recurrences of
// all pending trials run in parallel threads; thread 0 then sweeps in id
// order with the cheap DP, and only accepted operators are re-predicted
// before the next pass (the same set of evaluations the reference makes).
__device__ __noinline__ void prune_pass(GShared& S, const GreedyArgs& a, const OpscDecisions& out, int w, double qps, int L,
                           int ph, double target) {
  __shared__ double t_wt[OPSC_MAX_OPS], t_soj[OPSC_MAX_OPS];
  __shared__ uint8_t t_ok[OPSC_MAX_OPS], t_need[OPSC_MAX_OPS];
  __shared__ int changed;
  __shared__ int r_base[OPSC_MAX_OPS];
  const OpscDag& d = a.d;
  const int n = d.n_ops;
  // Every pass prunes an operator by at most one replica and its P and B stay,
  // so the trials a pass can need are predict_op(v, P_v, R_v - depth, B_v):
  // all threads tabulate depth 1 .. kGreedyThreads / n of every operator at
  // once (one Erlang chain each); a pass then looks its trials up (status bits
  // ORed when used), computing only past the table's depth.
  extern __shared__ __align__(16) unsigned char g_dyn[];
  double* pt_wt = reinterpret_cast<double*>(g_dyn + kGreedyArgsWords * 16);
  double* pt_soj = pt_wt + kGreedyThreads;
  uint32_t* pt_st = reinterpret_cast<uint32_t*>(pt_soj + kGreedyThreads);
  uint8_t* pt_ok = reinterpret_cast<uint8_t*>(pt_st + kGreedyThreads);
  const int depth = kGreedyThreads / n;
  for (int v = threadIdx.x; v < n; v += blockDim.x) {
    t_need[v] = 1;
    r_base[v] = S.r[v];
  }
  {
    const int e = threadIdx.x, v = e % n, dd = e / n + 1;
    if (dd <= depth && S.r[v] - dd >= 1) {
      uint32_t st = 0;
      const GPt o = gpoint(a, w, qps, L, ph, v, S.p[v], S.r[v] - dd, S.b[v], &st);
      pt_wt[e] = o.wt;
      pt_soj[e] = o.soj;
      pt_ok[e] = o.ok;
      pt_st[e] = st;
    }
  }
  __syncthreads();
  while (true) {
    for (int v = threadIdx.x; v < n; v += blockDim.x) {
      if (!t_need[v] || S.r[v] <= 1) continue;
      uint32_t st = 0;
      const int dd = r_base[v] - (S.r[v] - 1);
      if (dd >= 1 && dd <= depth) {
        const int e = (dd - 1) * n + v;
        st = pt_st[e];
        t_ok[v] = pt_ok[e];
        t_wt[v] = pt_wt[e];
        t_soj[v] = pt_soj[e];
      } else {
        const GPt o = gpoint(a, w, qps, L, ph, v, S.p[v], S.r[v] - 1, S.b[v], &st);
        t_ok[v] = o.ok;
        t_wt[v] = o.wt;
        t_soj[v] = o.soj;
      }
      if (st) atomicOr(&S.st, st);
      t_need[v] = 0;
    }
    __syncthreads();
    // The sweep in id order (each accepted prune changes the state the next
    // trial sees), by warp 0 with one lane per operator: every remaining
    // operator's trial runs at once against the current state, the lowest id
    // that passes is accepted -- exactly the one the sequential sweep accepts
    // next, since the ids before it failed against the same state -- and the
    // sweep resumes after it.
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x, n = d.n_ops;
      bool any = false;
      int obj = objective_warp(S, n);  // kept current per accepted prune (-P_v, exact)
      for (int start = 0; start < n;) {
        const bool cand = lane >= start && lane < n && S.r[lane] > 1 && t_ok[lane];
        double lat = OPSC_INF;
        if (cand) lat = trial_latency(S, d, S.wt, lane, t_wt[lane], false);  // S.wt moves inside the pass
        const unsigned pass = __ballot_sync(0xffffffffu, cand && lat <= target);
        if (!pass) break;
        const int v = __ffs(pass) - 1;
        const double lv = __shfl_sync(0xffffffffu, lat, v);
        if (lane == 0) {
          S.r[v] -= 1;
          S.wt[v] = t_wt[v];
          S.soj[v] = t_soj[v];
          // the accepted trial's DP value IS the new critical-path latency
          // (max over predecessors commutes with the monotone + w); the path
          // itself is only needed after the pass
          S.lat = lv;
          S.cpv_ok = 0;
          t_need[v] = 1;
          push_trace(S, out, w, OPSC_ACT_PRUNE, v, S.r[v], S.b[v], S.p[v], S.lat, obj - S.p[v]);
        }
        obj -= S.p[v];  // R_v dropped by one, P_v unchanged
        __syncwarp();
        any = true;
        start = v + 1;
      }
      if (lane == 0) changed = any;
      if (!any) set_path_warp(S, d);  // path (and the same value) for what follows
    }
    __syncthreads();
    if (!changed) break;
  }
}

// Greedy state carried from phase 1 (init + first loop) to phase 2 (reseed,
// headroom, prune), so K3 -- needed only by phase 2 -- can run concurrently
// with phase 1 on another stream.
struct GSave {
  int p[OPSC_MAX_OPS], r[OPSC_MAX_OPS], b[OPSC_MAX_OPS];
  double soj[OPSC_MAX_OPS], wt[OPSC_MAX_OPS];
  double lat;
  int8_t path[OPSC_MAX_OPS];
  int stable, trace_len, ok;
  uint32_t st;
};

size_t greedy_state_bytes(int n_windows) { return sizeof(GSave) * (size_t)(n_windows > 0 ? n_windows : 1); }

__device__ void distinct_p(GShared& S, const GreedyArgs& a, int n) {
  for (int v = 0; v < n; ++v) {
    int k = 0;
    for (int i = 0; i < a.s.n_p[v]; ++i) {
      bool dup = false;
      for (int j = 0; j < k; ++j) dup |= S.pd[v][j] == a.s.p_vals[v][i];
      if (!dup) S.pd[v][k++] = a.s.p_vals[v][i];
    }
    S.np_d[v] = k;
  }
}

// phase 0: whole planner; phase 1: init_configs + first greedy loop, state
// saved; phase 2: state loaded, uniform reseed, headroom, prune, outputs.
// The DAG and spec tables are read per operator by lane-varying indices
// (init pairs, the path update, the prune sweep): from the kernel's parameter
// (constant) bank every such load serialises over the distinct addresses of a
// warp, so the CTA first copies them to shared memory (16-byte words).

__global__ void __launch_bounds__(kGreedyThreads) greedy_kernel(
    const __grid_constant__ GreedyArgs ga, const __grid_constant__ OpscWindows win,
    const int16_t* __restrict__ ucfg, const uint8_t* __restrict__ ufeas, const uint32_t* __restrict__ ustatus,
    const __grid_constant__ OpscDecisions out, int phase, GSave* __restrict__ save) {
  // programmatic dependent launch: release the next kernel (phase 2, K4) so
  // its CTAs are resident when this grid ends, then wait for the previous one
  pdl_trigger();
  pdl_wait();
  __shared__ GShared S;
  extern __shared__ __align__(16) unsigned char g_args[];
  {
    const uint4* src = reinterpret_cast<const uint4*>(&ga);
    uint4* dst = reinterpret_cast<uint4*>(g_args);
    for (int i = threadIdx.x; i < (int)(sizeof(GreedyArgs) / 16); i += blockDim.x) dst[i] = src[i];
    if (threadIdx.x == 0 && sizeof(GreedyArgs) % 16) {
      const unsigned char* sb = reinterpret_cast<const unsigned char*>(&ga);
      for (size_t k = sizeof(GreedyArgs) / 16 * 16; k < sizeof(GreedyArgs); ++k) g_args[k] = sb[k];
    }
    __syncthreads();
  }
  const GreedyArgs& a = *reinterpret_cast<const GreedyArgs*>(g_args);
  const OpscDag& d = a.d;
  const int n = d.n_ops;
  const int w = blockIdx.x;
  const double qps = win.qps[w];
  const int L = win.seq_len[w], ph = win.phase[w];
  const double slo = win.slo[w], eps = win.eps[w];
  if (phase == 2) {
    if (!(qps > 0.0)) return;
    if (threadIdx.x == 0) {
      const GSave& g = save[w];
      distinct_p(S, a, n);
      for (int v = 0; v < n; ++v) {
        S.p[v] = g.p[v]; S.r[v] = g.r[v]; S.b[v] = g.b[v];
        S.soj[v] = g.soj[v]; S.wt[v] = g.wt[v]; S.path[v] = g.path[v];
      }
      S.lat = g.lat;
      S.stable = g.stable;
      S.trace_len = g.trace_len;
      S.st = g.st;
      S.flag = g.ok;
      S.bneck = bottleneck(S, n);
      S.cpv_ok = 0;
      for (int i = 0; i < n; ++i) S.tpos[d.topo[i]] = (int8_t)i;
      S.chain = is_chain(d);
      for (int q = 0; q < 4; ++q) {
        S.n_valid[q >> 1][q & 1] = 0;
        S.n_st[q >> 1][q & 1] = 0;
      }
    }
    __syncthreads();
    if (!S.flag) return;
  } else {
  if (threadIdx.x == 0) {
    out.feasible[w] = 0;
    out.trace_len[w] = 0;
    if (phase == 1) save[w].ok = 0;
  }
  for (int i = threadIdx.x; i < n * 3; i += blockDim.x) out.cfg[(size_t)w * n * 3 + i] = 0;
  if (!(qps > 0.0)) return;
  for (int v = threadIdx.x; v < n; v += blockDim.x) {  // distinct P per operator, one thread each
    int k = 0;
    for (int i = 0; i < a.s.n_p[v]; ++i) {
      bool dup = false;
      for (int j = 0; j < k; ++j) dup |= S.pd[v][j] == a.s.p_vals[v][i];
      if (!dup) S.pd[v][k++] = a.s.p_vals[v][i];
    }
    S.np_d[v] = k;
    S.chosen[v] = 0;
    S.tpos[d.topo[v]] = (int8_t)v;
  }
  if (threadIdx.x == 0) {
    S.st = 0;
    S.trace_len = 0;
    S.cpv_ok = 0;
    S.chain = is_chain(d);
    for (int q = 0; q < 4; ++q) {
      S.n_valid[q >> 1][q & 1] = 0;
      S.n_st[q >> 1][q & 1] = 0;
    }
  }
  __syncthreads();

#ifdef OPSC_GREEDY_PROF
  const long long t_init0 = clock64();
#endif
  // ---- init_configs (:254-294): per parallelism rank, (op, B) pairs in parallel
  int max_np = 0;
  for (int v = 0; v < n; ++v) max_np = max(max_np, a.s.n_p[v]);
  int max_b = 0;
  for (int v = 0; v < n; ++v) max_b = max(max_b, a.s.b_max[v]);
  for (int pi = 0; pi < max_np; ++pi) {
    for (int v = threadIdx.x; v < n; v += blockDim.x) S.i_bb[v] = -1;
    for (int b0 = 0; b0 < max_b; b0 += kInitChunk) {
    __syncthreads();
    for (int k = threadIdx.x; k < n * kInitChunk; k += blockDim.x) {
      // B-major: a round of threads covers a few B values of every operator,
      // so the long Erlang chains of small B (R ~ qps T_B / B) share rounds
      // instead of setting every round's length
      const int v = k % n, b = b0 + k / n + 1;
      if (S.chosen[v] || pi >= a.s.n_p[v] || b > a.s.b_max[v]) continue;
      const int p = a.s.p_vals[v][pi];
      const double t = op_latency(d, ph, v, b, L, p);
      const double tl = t * (double)d.layer_count[v];
      uint32_t st = 0;
      if (tl == 0.0) st |= OPSC_W_ZERO_DIVISION;
      const double mu = 1.0 / tl, lam = qps / (double)b;
      const int r = strict_min_replicas(lam, mu, a.s.r_cap);
      const int j = b - b0 - 1;
      S.i_r[v][j] = r;
      if (r >= 0) {
        const double util = lam / ((double)r * mu);
        if (util >= 1.0 || util <= 0.0) st |= OPSC_W_UNSTABLE_ROUNDING;
        const double service = t / (double)b;  // sojourn key: wait only inside wait + service
        S.i_soj[v][j] = wait_for_sum(r, lam / ((double)r * mu), (double)r * mu - lam, service) + service;
      }
      if (st) atomicOr(&S.st, st);
    }
    __syncthreads();
    // running argmin over the chunks: min sojourn, ties to the lowest B
    // (the reference's strict '<' over ascending B), one warp per operator:
    // lanes reduce the chunk's (sojourn, B) minimum over the non-NaN entries;
    // a chunk whose first valid entry is NaN (which the strict scan would keep
    // when nothing precedes it) goes through the literal scan
    for (int v = threadIdx.x >> 5; v < n; v += blockDim.x >> 5) {
      if (S.chosen[v] || pi >= a.s.n_p[v]) continue;
      const int lane = threadIdx.x & 31;
      const int bend = min(a.s.b_max[v], b0 + kInitChunk);
      int fv = 0x7fffffff, bb = 0x7fffffff;
      double bs = 0.0;
      for (int b = b0 + 1 + lane; b <= bend; b += 32) {
        const int j = b - b0 - 1;
        if (S.i_r[v][j] < 0) continue;
        fv = min(fv, b);
        const double x = S.i_soj[v][j];
        if (x == x && (bb == 0x7fffffff || x < bs || (x == bs && b < bb))) { bs = x; bb = b; }
      }
      fv = __reduce_min_sync(0xffffffffu, fv);
      for (int o = 16; o > 0; o >>= 1) {
        const double ox = __shfl_xor_sync(0xffffffffu, bs, o);
        const int ob = __shfl_xor_sync(0xffffffffu, bb, o);
        if (ob != 0x7fffffff && (bb == 0x7fffffff || ox < bs || (ox == bs && ob < bb))) { bs = ox; bb = ob; }
      }
      if (lane == 0 && fv != 0x7fffffff) {  // (no valid entry in this chunk: nothing to do)
      const double first = S.i_soj[v][fv - b0 - 1];
      if (first != first || S.i_bs[v] != S.i_bs[v]) {  // NaN in play: the literal scan
        for (int b = b0 + 1; b <= bend; ++b) {
          const int j = b - b0 - 1;
          if (S.i_r[v][j] < 0) continue;
          if (S.i_bb[v] < 0 || S.i_soj[v][j] < S.i_bs[v]) {
            S.i_bb[v] = b;
            S.i_bs[v] = S.i_soj[v][j];
            S.i_br[v] = S.i_r[v][j];
          }
        }
      } else if (bb != 0x7fffffff && (S.i_bb[v] < 0 || bs < S.i_bs[v])) {
        S.i_bb[v] = bb;
        S.i_bs[v] = bs;
        S.i_br[v] = S.i_r[v][bb - b0 - 1];
      }
      }
      __syncwarp();
    }
    }
    __syncthreads();
    for (int v = threadIdx.x; v < n; v += blockDim.x) {
      if (S.chosen[v] || pi >= a.s.n_p[v] || S.i_bb[v] < 0) continue;
      S.p[v] = a.s.p_vals[v][pi];
      S.b[v] = S.i_bb[v];
      S.r[v] = S.i_br[v];
      S.chosen[v] = 1;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    // 0, or 1 + dag.node_ids position of the first operator without a stable
    // (B, P): the one the reference's NoStableConfig names (autoscaler.py:289-292)
    int fail = 0;
    for (int pos = n - 1; pos >= 0; --pos)
      if (!S.chosen[d.node_order[pos]]) fail = pos + 1;
    S.flag = fail;
  }
  __syncthreads();
  if (S.flag) {
    if (threadIdx.x == 0)
      out.status[w] |= S.st | OPSC_W_NO_STABLE_INIT | ((uint32_t)S.flag << OPSC_W_INIT_OP_SHIFT);
    return;
  }
#ifdef OPSC_GREEDY_PROF
  const long long t_init1 = clock64();
#endif
  eval_full(S, a, w, qps, L, ph);
#ifdef OPSC_GREEDY_PROF
  const long long t_eval1 = clock64();
#endif
  greedy_loop(S, a, out, w, qps, L, ph, slo, eps);
#ifdef OPSC_GREEDY_PROF
  if (threadIdx.x == 0)  // dev build only (tools): cycles of init / first evaluation / loop
    printf("greedy w%d phase %d: init %lld eval %lld loop %lld cycles, trace %d\n", w, phase, t_init1 - t_init0,
           t_eval1 - t_init1, clock64() - t_eval1, S.trace_len);
#endif
  if (phase == 1) {
    if (threadIdx.x == 0) {
      GSave& g = save[w];
      for (int v = 0; v < n; ++v) {
        g.p[v] = S.p[v]; g.r[v] = S.r[v]; g.b[v] = S.b[v];
        g.soj[v] = S.soj[v]; g.wt[v] = S.wt[v]; g.path[v] = S.path[v];
      }
      g.lat = S.lat;
      g.stable = S.stable;
      g.trace_len = S.trace_len;
      g.st = S.st;
      g.ok = 1;
    }
    return;
  }
  }  // phase != 2

  // ---- uniform reseed (:357-367)
  const uint32_t us = ustatus[w];
  if (threadIdx.x == 0) S.st |= us & (OPSC_W_ZERO_DIVISION | OPSC_W_UNSTABLE_ROUNDING);
  if (!(us & OPSC_W_NO_STABLE_MODEL) && ufeas[w]) {
    __shared__ int keep_p[OPSC_MAX_OPS], keep_r[OPSC_MAX_OPS], keep_b[OPSC_MAX_OPS];
    __shared__ double keep_soj[OPSC_MAX_OPS], keep_wt[OPSC_MAX_OPS], keep_lat;
    __shared__ int8_t keep_path[OPSC_MAX_OPS];
    __shared__ int reseed, base_obj;
    if (threadIdx.x == 0) {
      base_obj = objective(S, n);
      int uobj = 0;
      for (int v = 0; v < n; ++v) uobj += ucfg[((size_t)w * n + v) * 3] * ucfg[((size_t)w * n + v) * 3 + 1];
      reseed = uobj < base_obj;
      if (reseed) {
        push_trace(S, out, w, OPSC_ACT_RESEED, -1, 0, 0, 0, 0.0, uobj);
        for (int v = 0; v < n; ++v) {
          keep_p[v] = S.p[v]; keep_r[v] = S.r[v]; keep_b[v] = S.b[v];
          keep_soj[v] = S.soj[v]; keep_wt[v] = S.wt[v]; keep_path[v] = S.path[v];
          S.p[v] = ucfg[((size_t)w * n + v) * 3];
          S.r[v] = ucfg[((size_t)w * n + v) * 3 + 1];
          S.b[v] = ucfg[((size_t)w * n + v) * 3 + 2];
        }
        keep_lat = S.lat;
      }
    }
    __syncthreads();
    if (reseed) {
#ifdef OPSC_GREEDY_PROF
      const long long z0 = clock64();
      const int tr0 = S.trace_len;
#endif
      eval_full(S, a, w, qps, L, ph);
#ifdef OPSC_GREEDY_PROF
      const long long z1 = clock64();
#endif
      prune_pass(S, a, out, w, qps, L, ph, slo - eps);
#ifdef OPSC_GREEDY_PROF
      const long long z2 = clock64();
      const int tr1 = S.trace_len;
#endif
      greedy_loop(S, a, out, w, qps, L, ph, slo, eps);
#ifdef OPSC_GREEDY_PROF
      if (threadIdx.x == 0)
        printf("greedy w%d phase 2 reseed: eval %lld prune %lld (%d moves) loop %lld (%d moves) cycles\n", w, z1 - z0,
               z2 - z1, tr1 - tr0, clock64() - z2, S.trace_len - tr1);
#endif
      if (threadIdx.x == 0 && !(objective(S, n) < base_obj)) {
        for (int v = 0; v < n; ++v) {
          S.p[v] = keep_p[v]; S.r[v] = keep_r[v]; S.b[v] = keep_b[v];
          S.soj[v] = keep_soj[v]; S.wt[v] = keep_wt[v]; S.path[v] = keep_path[v];
        }
        S.lat = keep_lat;
        S.stable = 1;
        S.bneck = bottleneck(S, n);
        S.cpv_ok = 0;  // cpv belongs to the discarded reseeded plan
      }
      __syncthreads();
    }
  }
  // ---- headroom restore (:369-374, 503-559)
  if (eps > 0 && S.lat <= slo) {
    for (int c = 0; S.lat > slo - eps; ++c) {
      upscale_step(S, a, out, w, qps, L, ph, slo, eps, true, c);
      if (!S.applied) break;
    }
  }
  // ---- optional prune (:376-377)
  if (a.s.prune_excess_replicas && S.lat <= slo) prune_pass(S, a, out, w, qps, L, ph, slo - eps);

  if (threadIdx.x == 0) {
    out.feasible[w] = (uint8_t)(S.stable && S.lat <= slo);
    for (int v = 0; v < n; ++v) {
      int16_t* c = out.cfg + ((size_t)w * n + v) * 3;
      c[0] = (int16_t)S.p[v];
      c[1] = (int16_t)S.r[v];
      c[2] = (int16_t)S.b[v];
    }
    out.trace_len[w] = S.trace_len;
    uint32_t st = S.st;
    // trace_cap == 0: the caller asked for no trace (e.g. capacity search)
    if (out.trace_cap > 0 && S.trace_len > out.trace_cap) st |= OPSC_W_TRACE_TRUNCATED;
    out.status[w] |= st;
  }
}

cudaError_t launch_greedy(const OpscDag& d, const OpscGreedySpec& s, OpscWindows w, const int16_t* ucfg,
                          const uint8_t* ufeas, const uint32_t* ustatus, OpscDecisions out, cudaStream_t st,
                          int phase, void* save) {
  if (w.n <= 0) return cudaSuccess;
  if (phase < 0 || phase > 2 || (phase != 0 && !save)) return cudaErrorInvalidValue;
  for (int v = 0; v < d.n_ops; ++v)
    if (s.b_max[v] < 1 || s.n_p[v] < 1) return cudaErrorInvalidValue;
  GreedyArgs a;
  a.d = d;
  a.s = s;
  // dynamic smem: the copied args, then the prune pass's trial table
  const size_t dyn = kGreedyArgsWords * 16 + (size_t)kGreedyThreads * (8 + 8 + 4 + 1);
  static int set_dyn[64];  // raise the dynamic limit once per device (static GShared + args pass 48 KB)
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !set_dyn[dev]) {
    const cudaError_t e = cudaFuncSetAttribute(greedy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    if (e != cudaSuccess) return e;
    set_dyn[dev] = 1;
  }
  return launch_pdl(greedy_kernel, dim3(w.n), dim3(kGreedyThreads), dyn, st, a, w, ucfg, ufeas, ustatus, out, phase,
                    (GSave*)save);
}

}  // namespace opsc
