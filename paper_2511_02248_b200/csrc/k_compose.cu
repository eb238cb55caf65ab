// k_compose.cu -- K2 compose_mask_argmin: exhaustive enumeration of every
// window's (P,R,B)^n candidate space, SLO mask, and lexicographic argmin.
//
// Replaces brute_force_autoscale's descend / leaf test (autoscaler.py:786-826)
// with a literal enumeration: every candidate's iteration latency is composed
// as the critical-path DP of opgraph.py:223-244 (max over predecessors, then
// + own weight, in topological order), masked with `<= slo`, and reduced with
// key = (objective << 40) | lexicographic index (ops sorted by id, per op
// (P,R,B) ascending; autoscaler.py:725, 747-749, 795). The key carries the
// global lexicographic index, so traversal order, sharding and reduction
// order cannot change the winner.
//
// Work split (one CTA = 256 threads, one window):
//   * positions = topological order; the last two are the k and j levels,
//     `il-2` middle levels sit above them, the rest are "outer" and fixed per
//     thread (decoded from the thread's outer index);
//   * the j menu (innermost op) is staged SORTED by its key (P*R, entry) and
//     held in registers; per candidate the thread issues exactly
//         DADD  lat = B_j + w_j          (path extension, the DP's last add)
//         DSETP lat <= slo               (SLO mask)
//         @P MOV inner = rank            (descending scan: the last hit is the
//                                         cheapest feasible j of this prefix)
//     with no loop-carried dependency, so warps issue back to back;
//   * per k entry the cheapest feasible (k, j) pair is folded into a u64 key
//     from shared-memory key tables; CTA result = warp-shuffle u64 min ->
//     smem -> one atomicMin per CTA.
#include <algorithm>
#include <cstring>

#include "opsc_common.cuh"

namespace opsc {

#ifndef OPSC_COMPOSE_THREADS
#define OPSC_COMPOSE_THREADS 256
#endif
#ifndef OPSC_COMPOSE_MINB
#define OPSC_COMPOSE_MINB 4  // 64 registers: 32 warps/SM hide the DADD->DSETP->SEL latency (+12% vs 3)
#endif
constexpr int kComposeThreads = OPSC_COMPOSE_THREADS;
constexpr unsigned long long kSentinel = 1ull << 62;  // > any real key (objective < 2^17)

__device__ __forceinline__ double dp_in(uint32_t pm, const double* val) {
  double in = 0.0;
  while (pm) {
    const int p = __ffs(pm) - 1;
    pm &= pm - 1;
    in = fmax(in, val[p]);
  }
  return in;
}

struct ComposeSmem {
  double* w;                 // [E+1] weights (entry E = virtual, 0.0)
  int32_t* cost;             // [E+1] P*R per entry
  unsigned long long* kk;    // [m_k] (cost_k << 40) + a * kstride
  double* jw;                // [m_j] j weights sorted by key
  unsigned long long* jk;    // [m_j + 1] sorted j keys, jk[m_j] = sentinel
};

template <int NJ, bool CHAIN>
__global__ void __launch_bounds__(kComposeThreads, OPSC_COMPOSE_MINB)
compose_kernel(const __grid_constant__ ComposeCfg c, const __grid_constant__ OpscGrid g,
               const double* __restrict__ menu_w, const double* __restrict__ slo_w,
               const double* __restrict__ qps_w, unsigned long long* __restrict__ key_out,
               const __grid_constant__ PeerKeys peers) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ unsigned long long warp_best[kComposeThreads / 32];
  __shared__ __align__(8) unsigned long long tma_bar;
  const int jp = c.n - 1, kp = c.n - 2;
  const int mj = c.m[jp], mk = c.m[kp];
  ComposeSmem s;
  s.w = reinterpret_cast<double*>(smem_raw);  // offset 0: 16-byte aligned TMA target
  s.kk = reinterpret_cast<unsigned long long*>(s.w + c.E + 1);
  s.jk = s.kk + mk;
  s.jw = reinterpret_cast<double*>(s.jk + mj + 1);
  s.cost = reinterpret_cast<int32_t*>(s.jw + mj);

  const int w = blockIdx.x / c.blocks_per_window;
  const int bw = blockIdx.x - w * c.blocks_per_window;
  const double* src = menu_w + (size_t)w * c.E;
  // The window's menu slab is one contiguous tile: when it is 16-byte sized
  // and aligned, one thread moves it with a TMA bulk copy (cp.async.bulk,
  // completion on an mbarrier) while the CTA builds the cost table.
  const uint32_t slab = (uint32_t)c.E * 8u;
  const bool use_tma = (slab % 16u) == 0u && ((reinterpret_cast<uintptr_t>(src) & 15u) == 0u) && slab > 0u;
  const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&tma_bar);
  if (use_tma) {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();  // the barrier is initialised before anyone polls it
  }
  if (use_tma && threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(slab) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            (uint32_t)__cvta_generic_to_shared(s.w)),
        "l"(src), "r"(slab), "r"(bar)
        : "memory");
  }
  for (int i = threadIdx.x; i < c.E; i += kComposeThreads) {
    if (!use_tma) s.w[i] = src[i];
    int v = 0;
    while (i >= g.menu_off[v + 1]) ++v;
    int p, r, b;
    entry_prb(g, v, i - g.menu_off[v], p, r, b);
    s.cost[i] = p * r;  // objective contribution (autoscaler.py:220-221, 756)
  }
  if (threadIdx.x == 0) {
    s.w[c.E] = 0.0;
    s.cost[c.E] = 0;
  }
  if (use_tma) {
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
          : "=r"(done)
          : "r"(bar)
          : "memory");
    }
  }
  __syncthreads();
  const int koff = c.off[kp], joff = c.off[jp];
  for (int a = threadIdx.x; a < mk; a += kComposeThreads)
    s.kk[a] = ((unsigned long long)s.cost[koff + a] << OPSC_KEY_LEX_BITS) + (unsigned long long)a * c.stride[kp];
  for (int i = threadIdx.x; i < mj; i += kComposeThreads) {
    // rank of entry i in (cost, entry) order == order of its key
    const int ci = s.cost[joff + i];
    int rank = 0;
    for (int q = 0; q < mj; ++q) {
      const int cq = s.cost[joff + q];
      rank += (cq < ci) || (cq == ci && q < i);
    }
    s.jw[rank] = s.w[joff + i];
    s.jk[rank] = ((unsigned long long)ci << OPSC_KEY_LEX_BITS) + (unsigned long long)i * c.stride[jp];
  }
  if (threadIdx.x == 0) s.jk[mj] = kSentinel;
  __syncthreads();

  const double slo = slo_w[w];
  unsigned long long best = kSentinel;
  const uint32_t o = c.lo + (uint32_t)bw * kComposeThreads + threadIdx.x;
  if (qps_w[w] > 0.0 && o < c.hi) {
    const int nout = c.n - c.il;
    double wj[NJ > 0 ? NJ : 1];
#pragma unroll
    for (int i = 0; i < NJ; ++i) wj[i] = i < mj ? s.jw[i] : OPSC_INF;
    double val[OPSC_CMAX];
    int dig[OPSC_CMAX];
    uint32_t rem = o;
    for (int pos = nout - 1; pos >= 0; --pos) {
      const uint32_t mm = (uint32_t)c.m[pos];
      const uint32_t q = rem / mm;
      dig[pos] = (int)(rem - q * mm);
      rem = q;
    }
    long long cost0 = 0;
    unsigned long long lex0 = 0;
    for (int pos = 0; pos < nout; ++pos) {
      const int e = c.off[pos] + dig[pos];
      val[pos] = dp_in(c.pmask[pos], val) + s.w[e];
      cost0 += s.cost[e];
      lex0 += (unsigned long long)dig[pos] * c.stride[pos];
    }
    const uint32_t kmask = 1u << kp, jmask = 1u << jp;
    const bool k_to_j = (c.pmask[jp] & kmask) != 0;
    const bool k_sink = (c.sinkmask & kmask) != 0;

    for (uint32_t mid = 0; mid < c.mid_count; ++mid) {
      uint32_t r2 = mid;
      for (int pos = kp - 1; pos >= nout; --pos) {
        const uint32_t mm = (uint32_t)c.m[pos];
        const uint32_t q = r2 / mm;
        dig[pos] = (int)(r2 - q * mm);
        r2 = q;
      }
      long long cost1 = cost0;
      unsigned long long lex1 = lex0;
      for (int pos = nout; pos < kp; ++pos) {
        const int e = c.off[pos] + dig[pos];
        val[pos] = dp_in(c.pmask[pos], val) + s.w[e];
        cost1 += s.cost[e];
        lex1 += (unsigned long long)dig[pos] * c.stride[pos];
      }
      double in_k = dp_in(c.pmask[kp], val);
      const double bj0 = dp_in(c.pmask[jp] & ~kmask, val);
      const double lo0 = dp_in(c.sinkmask & ~(kmask | jmask), val);
      if (CHAIN && !(lo0 <= slo)) in_k = OPSC_INF;  // another sink already misses the SLO

      unsigned long long mbest = kSentinel;
      for (int a = 0; a < mk; ++a) {
        const double bk = in_k + s.w[koff + a];
        double bj;
        if (CHAIN) {
          bj = bk;  // j's only predecessor is k, k is not a sink
        } else {
          bj = k_to_j ? fmax(bj0, bk) : bj0;
          const double lo = k_sink ? fmax(lo0, bk) : lo0;
          if (!(lo <= slo)) bj = OPSC_INF;
        }
        int inner = mj;
        if (NJ > 0) {
#pragma unroll
          for (int i = NJ - 1; i >= 0; --i) {
            const double lat = bj + wj[i];
            if (lat <= slo) inner = i;
          }
        } else {
          for (int i = mj - 1; i >= 0; --i) {
            const double lat = bj + s.jw[i];
            if (lat <= slo) inner = i;
          }
        }
        const unsigned long long kl = s.kk[a] + s.jk[inner];
        mbest = kl < mbest ? kl : mbest;
      }
      if (mbest < kSentinel) {
        const unsigned long long key = ((unsigned long long)cost1 << OPSC_KEY_LEX_BITS) + lex1 + mbest;
        best = key < best ? key : best;
      }
    }
  }
  best = warp_min_u64(best);
  if ((threadIdx.x & 31) == 0) warp_best[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x < 32) {
    unsigned long long b = threadIdx.x < kComposeThreads / 32 ? warp_best[threadIdx.x] : kSentinel;
    b = warp_min_u64(b);
    if (threadIdx.x == 0 && b < kSentinel) {
      if (peers.n == 0) {
        atomicMin(&key_out[w], b);
      } else {
        // fused multi-GPU merge: the CTA's minimum straight into every
        // rank's key buffer over NVLink (IPC-mapped peer memory)
        for (int p = 0; p < peers.n; ++p) atomicMin(peers.p[p] + w, b);
        __threadfence_system();
      }
    }
  }
}

// Host: topological positions, lexicographic strides, level split.
int compose_setup(const OpscDag& d, const OpscGrid& g, int n_windows, int shard, int n_shards,
                  ComposeCfg* cfg) {
  ComposeCfg c;
  memset(&c, 0, sizeof(c));
  const int nr = d.n_ops;
  if (nr < 1 || nr > OPSC_MAX_OPS || n_shards < 1 || shard < 0 || shard >= n_shards) return OPSC_ERR_ARG;
  const int nvirt = nr < 2 ? 2 - nr : 0;
  c.n = nr + nvirt;
  c.n_real_ops = nr;
  c.E = g.menu_off[nr];
  unsigned long long lexstride[OPSC_MAX_OPS];
  double space = 1.0;
  unsigned long long s = 1;
  for (int v = nr - 1; v >= 0; --v) {
    const int m = g.menu_off[v + 1] - g.menu_off[v];
    if (m < 1 || m > 65535) return OPSC_ERR_ARG;
    lexstride[v] = s;
    s *= (unsigned long long)m;
    space *= (double)m;
  }
  if (space >= (double)(1ull << OPSC_KEY_LEX_BITS)) return OPSC_ERR_SPACE;
  int pos_of[OPSC_MAX_OPS];
  for (int i = 0; i < nr; ++i) pos_of[d.topo[i]] = i + nvirt;
  for (int pos = 0; pos < c.n; ++pos) {
    if (pos < nvirt) {
      c.m[pos] = 1;
      c.off[pos] = c.E;
      continue;
    }
    const int v = d.topo[pos - nvirt];
    c.m[pos] = g.menu_off[v + 1] - g.menu_off[v];
    c.off[pos] = g.menu_off[v];
    c.stride[pos] = lexstride[v];
    uint32_t pm = 0;
    for (int p = 0; p < nr; ++p)
      if (d.pred_mask[v] >> p & 1u) pm |= 1u << pos_of[p];
    c.pmask[pos] = pm;
    if (d.sink_mask >> v & 1u) c.sinkmask |= 1u << pos;
  }
  // the objective of any candidate must stay below 2^17 (key headroom under the sentinel)
  long long max_obj = 0;
  for (int v = 0; v < nr; ++v) {
    int pmax = 0;
    for (int i = 0; i < g.n_p[v]; ++i) pmax = std::max(pmax, g.p_vals[v][i]);
    max_obj += (long long)pmax * g.r_max;
  }
  if (max_obj >= (1 << 17)) return OPSC_ERR_ARG;
  // level split: enough in-thread candidates to amortise the outer decode,
  // while keeping at least half a wave of threads
  auto prod = [&](int lo, int hi) {
    double x = 1.0;
    for (int pos = lo; pos < hi; ++pos) x *= c.m[pos];
    return x;
  };
  const double min_threads = 148.0 * 512.0;
  int il = 2;
  while (il < c.n && il < 6) {
    const bool too_many = prod(0, c.n - il) >= 4294967295.0;
    if (!too_many && prod(c.n - il, c.n) >= 2048.0) break;
    if (!too_many && (double)n_windows * prod(0, c.n - il - 1) < min_threads) break;
    ++il;
  }
  if (prod(0, c.n - il) >= 4294967295.0) return OPSC_ERR_SPACE;
  c.il = il;
  c.m_out = (uint32_t)prod(0, c.n - il);
  const double mid = prod(c.n - il, c.n - 2);
  if (mid >= 4294967295.0) return OPSC_ERR_SPACE;
  c.mid_count = (uint32_t)mid;
  c.lo = (uint32_t)((unsigned long long)c.m_out * shard / n_shards);
  c.hi = (uint32_t)((unsigned long long)c.m_out * (shard + 1) / n_shards);
  c.blocks_per_window = (int)((c.hi - c.lo + kComposeThreads - 1) / kComposeThreads);
  if (c.blocks_per_window < 1) c.blocks_per_window = 1;
  const int mj = c.m[c.n - 1];
  c.nj = mj <= 4 ? 4 : mj <= 8 ? 8 : mj <= 12 ? 12 : mj <= 16 ? 16 : mj <= 24 ? 24 : mj <= 32 ? 32 : 0;
  // chain fast path: j's only predecessor is k and k is not a sink
  const int jp = c.n - 1, kp = c.n - 2;
  c.chain = (c.pmask[jp] == (1u << kp)) && !(c.sinkmask >> kp & 1u);
  *cfg = c;
  return OPSC_OK;
}

template <int NJ, bool CHAIN>
static cudaError_t launch_t(const ComposeCfg& c, const OpscGrid& g, int n_windows, const double* menu_w,
                            const double* slo, const double* qps, unsigned long long* key, cudaStream_t s,
                            const PeerKeys& pk) {
  const int mj = c.m[c.n - 1], mk = c.m[c.n - 2];
  const size_t smem = (size_t)mk * 8 + (size_t)(mj + 1) * 8 + (size_t)(c.E + 1) * 8 + (size_t)mj * 8 +
                      (size_t)(c.E + 1) * 4;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(compose_kernel<NJ, CHAIN>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  const long long blocks = (long long)n_windows * c.blocks_per_window;
  if (blocks > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  compose_kernel<NJ, CHAIN><<<(unsigned)blocks, kComposeThreads, smem, s>>>(c, g, menu_w, slo, qps, key, pk);
  return cudaGetLastError();
}

template <int NJ>
static cudaError_t launch_nj(const ComposeCfg& c, const OpscGrid& g, int n_windows, const double* menu_w,
                             const double* slo, const double* qps, unsigned long long* key, cudaStream_t s,
                             const PeerKeys& pk) {
  return c.chain ? launch_t<NJ, true>(c, g, n_windows, menu_w, slo, qps, key, s, pk)
                 : launch_t<NJ, false>(c, g, n_windows, menu_w, slo, qps, key, s, pk);
}

cudaError_t launch_compose(const ComposeCfg& c, const OpscGrid& g, int n_windows, const double* menu_w,
                           const double* slo, const double* qps, unsigned long long* key, cudaStream_t s,
                           const PeerKeys* peers) {
  if (n_windows <= 0 || c.hi <= c.lo) return cudaSuccess;
  PeerKeys pk;
  memset(&pk, 0, sizeof(pk));
  if (peers) pk = *peers;
  switch (c.nj) {
    case 4: return launch_nj<4>(c, g, n_windows, menu_w, slo, qps, key, s, pk);
    case 8: return launch_nj<8>(c, g, n_windows, menu_w, slo, qps, key, s, pk);
    case 12: return launch_nj<12>(c, g, n_windows, menu_w, slo, qps, key, s, pk);
    case 16: return launch_nj<16>(c, g, n_windows, menu_w, slo, qps, key, s, pk);
    case 24: return launch_nj<24>(c, g, n_windows, menu_w, slo, qps, key, s, pk);
    case 32: return launch_nj<32>(c, g, n_windows, menu_w, slo, qps, key, s, pk);
    default: return launch_nj<0>(c, g, n_windows, menu_w, slo, qps, key, s, pk);
  }
}

}  // namespace opsc
