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
//   * the j menu (innermost op) is staged in shared memory sorted by WEIGHT
//     and held in registers. For a fixed prefix (everything but j) the
//     candidate latency fl(B_j + w_j) is monotone in w_j, so the feasible j
//     form a prefix of that order and the cheapest feasible j is a table
//     lookup pm[count] (prefix minimum of the j keys in weight order). Per
//     candidate the thread issues exactly
//         DADD  lat = B_j + w_j          (path extension, the DP's last add)
//         DSETP lat <= slo               (SLO mask)
//         SEL   count = i + 1            (ascending scan: the last hit is the
//                                         length of the feasible prefix)
//     with no loop-carried dependency, so warps issue back to back. (A
//     high-word mask on the FMA pipe and integer-pipe compares were measured
//     and rejected: DESIGN.md, instruction-mix paragraph;
//     tools/probe/cand_probe.cu);
//   * keys: each thread keeps one 32-bit running minimum over all its
//     in-thread candidates (cost << 20 | compact lexicographic index of the
//     middle, k and j digits), one fused add+min per k entry, decoded to the
//     u64 key once per 256-thread slice; CTA result = warp-shuffle u64 min ->
//     smem -> one atomicMin per CTA;
//   * the middle levels run as a register odometer over a plain inner loop
//     (the last middle level); template MODE 2 ("path suffix") covers every
//     DAG whose in-thread positions form a path (the chains and the
//     multimodal DAG); a CTA takes `spc` consecutive slices of its window;
//   * launched with programmatic stream serialization (pdl_wait at entry).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "opsc_common.cuh"

namespace opsc {

#ifndef OPSC_COMPOSE_THREADS
#define OPSC_COMPOSE_THREADS 256
#endif
#ifndef OPSC_COMPOSE_MINB_SMALL
// path-suffix kernels with register tiles of <= 8 entries fit 40 registers
// without spills: 6 CTAs (48 warps) per SM instead of 3 -- cfg2 5.2e12 ->
// 6.2e12, cfg3 5.6e12 -> 6.5e12 candidates/s (tools/variants_minb_small.sh;
// the generic-DAG modes spill there and keep OPSC_COMPOSE_MINB)
#define OPSC_COMPOSE_MINB_SMALL 6
#endif
#ifndef OPSC_COMPOSE_MINB_PATH
#define OPSC_COMPOSE_MINB_PATH 4  // path-suffix kernels with 12..32-entry tiles: 64 registers, no spills (cfg5 8.16e12 -> 8.20e12; 5 / 6: 8.15 / 8.16, tools/variants_minb_path.sh)
#endif
#ifndef OPSC_COMPOSE_MINB
#define OPSC_COMPOSE_MINB 3  // 80 registers, no spills: 7.38e12 vs 7.28e12 candidates/s at 4 CTAs/SM (64 regs, spills)
#endif
#ifndef OPSC_COMPOSE_KUNROLL
#define OPSC_COMPOSE_KUNROLL 3  // k-loop unroll of the exact form: +5% on 6-entry menus, neutral on 24
#endif
#ifndef OPSC_COMPOSE_LUNROLL
#define OPSC_COMPOSE_LUNROLL 2  // +1.5% on 6-entry menus (cfg2 / cfg3), neutral on cfg5 (tools/variants_lunroll.sh)
#endif
constexpr int kComposeThreads = OPSC_COMPOSE_THREADS;
constexpr int kLUnroll = OPSC_COMPOSE_LUNROLL;  // unroll of the last middle level's loop
constexpr int kOdoLevels = 4;
constexpr int kKUnroll = OPSC_COMPOSE_KUNROLL;  // middle levels kept in registers on path DAGs (il <= 6)
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
  double* jw;                // [m_j] j weights in ascending order (NaN as +inf)
  unsigned long long* pmk;   // [m_j + 1] pmk[c] = min key of the c lightest j entries, pmk[0] = sentinel
  uint32_t* kk32;            // [m_k] local form (register-tile path): cost_k << 20 | a * ks
  uint32_t* pm32;            // [m_j + 1] local form of pmk: cost_j << 20 | i * js, pm32[0] = 2^31
  uint32_t* lk32;            // [E + 1] local key contribution of every entry of an in-thread position (tkey)
};

// Local (k, j) keys of the register-tile path: cost_k + cost_j < 2^11 in
// bits 20..30 and the (k, j) index in lexicographic order in bits 0..19, so
// key order is the u64 key order restricted to one prefix, any sum with
// pm32[0] = 2^31 is >= 2^31 (infeasible), and nothing overflows.
constexpr uint32_t kLocalInfeasible = 1u << 31;

__device__ __forceinline__ uint32_t opaque_u32(uint32_t x) {
  asm volatile("mov.b32 %0, %0;" : "+r"(x));
  return x;
}

// 32-bit shared-window loads (the k loop keeps 32-bit addresses live instead
// of 64-bit generic pointers)
__device__ __forceinline__ double lds_f64(uint32_t a) {
  double v;
  asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}

// max(0, x) for the path-suffix DP: dp_in of a position fed by one
// predecessor (in = 0.0, then max with its value). Three instructions
// (DSETP + two selects) instead of fmax's NaN/-0 sequence; differs from fmax
// only in the sign of a zero, which no later add or SLO compare can see.
__device__ __forceinline__ double clamp0(double x) {
  double r;  // inline PTX: the front end would turn the select back into fmax
  asm("{ .reg .pred p; setp.gt.f64 p, %1, 0d0000000000000000; selp.f64 %0, %1, 0d0000000000000000, p; }"
      : "=d"(r)
      : "d"(x));
  return r;
}

// Exact count: the feasible j form a prefix in weight order.
template <int NJ>
__device__ __forceinline__ uint32_t exact_count(double bj, const double (&wj)[NJ], double slo) {
  uint32_t cnt = 0;
#pragma unroll
  for (int i = 0; i < NJ; ++i)
    if (bj + wj[i] <= slo) cnt = (uint32_t)i + 1u;
  return cnt;
}

template <bool CHAIN>
__device__ __forceinline__ double j_base(double bk, double bj0, double lo0, bool k_to_j, bool k_sink, double slo) {
  if (CHAIN) return bk;  // j's only predecessor is k, k is not a sink
  const double bj = k_to_j ? fmax(bj0, bk) : bj0;
  const double lo = k_sink ? fmax(lo0, bk) : lo0;
  return lo <= slo ? bj : OPSC_INF;
}

// The k and j levels for one prefix. Register-tile path (NJ > 0): returns
// the minimum local key (>= kLocalInfeasible if no candidate is feasible).
// a_wk / a_kk / a_pm: shared addresses of w[koff], kk32, pm32. The +inf
// padding past m_j never passes (slo <= DBL_MAX), so the count needs no clamp.
template <int NJ, bool CHAIN>
__device__ __forceinline__ uint32_t k_level_tile(uint32_t a_wk, uint32_t a_kk, uint32_t a_pm, int mk,
                                                 const double (&wj)[NJ], double in_k, double bj0, double lo0,
                                                 bool k_to_j, bool k_sink, double slo) {
  uint32_t mbest = kLocalInfeasible;  // min with any infeasible kl (>= 2^31) stays 2^31
  const uint32_t a_end = a_kk + 4u * (uint32_t)mk;
#pragma unroll(kKUnroll)
  for (; a_kk < a_end; a_kk += 4u, a_wk += 8u) {
    const double bj = j_base<CHAIN>(in_k + lds_f64(a_wk), bj0, lo0, k_to_j, k_sink, slo);
    const uint32_t cnt = exact_count<NJ>(bj, wj, slo);
    const uint32_t kl = lds_u32(a_kk) + lds_u32(a_pm + 4u * cnt);
    mbest = kl < mbest ? kl : mbest;
  }
  return mbest;
}

// Small menus (m_k <= NJ <= 8): the k menu in registers too, fully unrolled
// (padding: w = +inf never passes, local key 0 + pm32[0] = infeasible).
template <int NJ, bool CHAIN>
__device__ __forceinline__ uint32_t k_level_reg(uint32_t a_pm, const double (&wk)[NJ],
                                                const uint32_t (&kk)[NJ], const double (&wj)[NJ], double in_k,
                                                double bj0, double lo0, bool k_to_j, bool k_sink, double slo) {
  uint32_t mbest = kLocalInfeasible;
#pragma unroll
  for (int a = 0; a < NJ; ++a) {
    const double bj = j_base<CHAIN>(in_k + wk[a], bj0, lo0, k_to_j, k_sink, slo);
    const uint32_t kl = kk[a] + lds_u32(a_pm + 4u * exact_count<NJ>(bj, wj, slo));
    mbest = kl < mbest ? kl : mbest;
  }
  return mbest;
}

// Shared-memory path for large j menus (NJ == 0): u64 keys, exact compares.
template <bool CHAIN>
__device__ __forceinline__ unsigned long long k_level_smem(const ComposeSmem& s, int mk, int mj, int koff,
                                                           double in_k, double bj0, double lo0, bool k_to_j,
                                                           bool k_sink, double slo) {
  unsigned long long mbest = kSentinel;
  for (int a = 0; a < mk; ++a) {
    const double bk = in_k + s.w[koff + a];
    double bj;
    if (CHAIN) {
      bj = bk;
    } else {
      bj = k_to_j ? fmax(bj0, bk) : bj0;
      const double lo = k_sink ? fmax(lo0, bk) : lo0;
      if (!(lo <= slo)) bj = OPSC_INF;
    }
    int cnt = 0;
    for (int i = 0; i < mj; ++i)
      if (bj + s.jw[i] <= slo) cnt = i + 1;
    const unsigned long long kl = s.kk[a] + s.pmk[cnt];
    mbest = kl < mbest ? kl : mbest;
  }
  return mbest;
}

// CTA minimum -> one atomicMin per CTA into this GPU's key (or, for the
// fused multi-GPU merge, into EVERY rank's key buffer over NVLink peer memory).
__device__ __forceinline__ void cta_min_commit(unsigned long long best, int w, unsigned long long* key_out,
                                               const PeerKeys& peers, unsigned long long* warp_best) {
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
        for (int p = 0; p < peers.n; ++p) atomicMin(peers.p[p] + w, b);
        __threadfence_system();
      }
    }
  }
}

// Large-menu path (menus that do not fit the shared-memory tile, or a menu
// over 65535 entries): one thread per candidate index of the window's
// lexicographic space, weights read from the global menu slab (L1/L2
// resident), the same critical-path DP (max over predecessors, then + own
// weight, topological order) and the same key. Literal and exact, slower per
// candidate; only reachable with few operators (the reference's 1e7 guard).
//
// COUNT = true is the boundary diagnostic (opsc_compose_boundary): instead of
// the argmin it counts the candidates whose canonical latency lies within
// `band` of slo, i.e. those whose feasibility could depend on the reference's
// own summation order (a frozenset-ordered, Neumaier-compensated sum(),
// autoscaler.py:792-794). A zero count certifies the window's decision
// independent of that order.
template <bool COUNT>
__global__ void __launch_bounds__(kComposeThreads)
compose_flat_kernel(const __grid_constant__ ComposeCfg c, const __grid_constant__ OpscGrid g,
                    const double* __restrict__ menu_w, const double* __restrict__ slo_w,
                    const double* __restrict__ qps_w, unsigned long long* __restrict__ key_out,
                    const __grid_constant__ PeerKeys peers, double band_ulps = 0.0) {
  pdl_wait();
  __shared__ unsigned long long warp_best[kComposeThreads / 32];
  const int w = blockIdx.x / c.blocks_per_window;
  const int bw = blockIdx.x - w * c.blocks_per_window;
  const double slo = fmin(slo_w[w], 1.7976931348623157e308);
  const double* mw = menu_w + (size_t)w * c.E;
  unsigned long long best = kSentinel;
  // band = band_ulps ulps of slo (ulp from the exponent of slo)
  const double band = COUNT ? band_ulps * (nextafter(slo, OPSC_INF) - slo) : 0.0;
  unsigned long long near = 0;
  if (qps_w[w] > 0.0) {
    const unsigned long long step = (unsigned long long)c.blocks_per_window * kComposeThreads;
    for (unsigned long long idx = c.flo + (unsigned long long)bw * kComposeThreads + threadIdx.x; idx < c.fhi;
         idx += step) {
      int dig[OPSC_CMAX];
      unsigned long long rem = idx;
      for (int pos = c.n - 1; pos >= 0; --pos) {
        const unsigned long long mm = (unsigned long long)c.m[pos];
        const unsigned long long q = rem / mm;
        dig[pos] = (int)(rem - q * mm);
        rem = q;
      }
      double val[OPSC_CMAX];
      long long cost = 0;
      unsigned long long lex = 0;
      double lat = 0.0;
      for (int pos = 0; pos < c.n; ++pos) {
        double wt = 0.0;
        if (c.vop[pos] >= 0) {
          wt = mw[c.off[pos] + dig[pos]];
          int p, r, b;
          entry_prb(g, c.vop[pos], dig[pos], p, r, b);
          cost += p * r;
          lex += (unsigned long long)dig[pos] * c.stride[pos];
        }
        val[pos] = dp_in(c.pmask[pos], val) + wt;
        if (c.sinkmask >> pos & 1u) lat = fmax(lat, val[pos]);
      }
      if (COUNT) {
        near += lat < OPSC_INF && fabs(lat - slo) <= band;
      } else if (lat <= slo) {
        const unsigned long long key = ((unsigned long long)cost << OPSC_KEY_LEX_BITS) + lex;
        best = key < best ? key : best;
      }
    }
  }
  if (COUNT) {
    for (int o = 16; o > 0; o >>= 1) near += __shfl_xor_sync(0xffffffffu, near, o);
    if ((threadIdx.x & 31) == 0 && near) atomicAdd(&key_out[w], near);
    return;
  }
  cta_min_commit(best, w, key_out, peers, warp_best);
}

// MODE: 0 generic DAG, 1 CHAIN (j's only predecessor is k, k no sink),
// 2 path suffix (every in-thread position fed by the previous one only, j the
// only in-thread sink; outer sinks checked once per thread).
template <int NJ, int MODE, bool KREG>
__global__ void __launch_bounds__(kComposeThreads,
                                  NJ > 0 && NJ <= 8 && MODE == 2   ? OPSC_COMPOSE_MINB_SMALL
                                  : NJ > 8 && MODE == 2            ? OPSC_COMPOSE_MINB_PATH
                                                                   : OPSC_COMPOSE_MINB)
compose_kernel(const __grid_constant__ ComposeCfg c, const __grid_constant__ OpscGrid g,
               const double* __restrict__ menu_w, const double* __restrict__ slo_w,
               const double* __restrict__ qps_w, unsigned long long* __restrict__ key_out,
               const __grid_constant__ PeerKeys peers) {
  pdl_wait();
  constexpr bool CHAIN = MODE >= 1, PATH = MODE == 2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ unsigned long long warp_best[kComposeThreads / 32];
  __shared__ __align__(8) unsigned long long tma_bar;
  const int jp = c.n - 1, kp = c.n - 2;
  const int mj = c.m[jp], mk = c.m[kp];
  ComposeSmem s;
  s.w = reinterpret_cast<double*>(smem_raw);  // offset 0: 16-byte aligned TMA target
  s.kk = reinterpret_cast<unsigned long long*>(s.w + c.E + 1);
  s.pmk = s.kk + mk;
  s.jw = reinterpret_cast<double*>(s.pmk + mj + 1);
  s.cost = reinterpret_cast<int32_t*>(s.jw + mj);
  s.kk32 = reinterpret_cast<uint32_t*>(s.cost + c.E + 1);
  s.pm32 = s.kk32 + mk;
  s.lk32 = s.pm32 + mj + 1;

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
    if (c.tkey) {
      int pos = 0;
      while (c.vop[pos] != v) ++pos;
      s.lk32[i] = ((uint32_t)(p * r) << 20) + (uint32_t)(i - g.menu_off[v]) * c.cs[pos];
    }
  }
  if (threadIdx.x == 0) {
    s.w[c.E] = 0.0;
    s.cost[c.E] = 0;
    s.lk32[c.E] = 0;
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
  const uint32_t ks = c.cs[kp], js = c.cs[jp];
  for (int a = threadIdx.x; a < mk; a += kComposeThreads) {
    s.kk[a] = ((unsigned long long)s.cost[koff + a] << OPSC_KEY_LEX_BITS) + (unsigned long long)a * c.stride[kp];
    s.kk32[a] = ((uint32_t)s.cost[koff + a] << 20) + (uint32_t)a * ks;
  }
  for (int i = threadIdx.x; i < mj; i += kComposeThreads) {
    // rank of entry i in (weight, entry) order; NaN never passes a compare,
    // exactly like +inf, so it sorts as +inf
    double wi = s.w[joff + i];
    wi = wi != wi ? OPSC_INF : wi;
    int rank = 0;
    for (int q = 0; q < mj; ++q) {
      double wq = s.w[joff + q];
      wq = wq != wq ? OPSC_INF : wq;
      rank += (wq < wi) || (wq == wi && q < i);
    }
    s.jw[rank] = wi;
    s.pmk[rank + 1] = ((unsigned long long)s.cost[joff + i] << OPSC_KEY_LEX_BITS) +
                      (unsigned long long)i * c.stride[jp];
    s.pm32[rank + 1] = ((uint32_t)s.cost[joff + i] << 20) + (uint32_t)i * js;
  }
  __syncthreads();
  if (threadIdx.x < 32) {  // pmk[1..mj] = running minimum (warp scan in chunks of 32)
    unsigned long long carry = kSentinel;
    uint32_t carry32 = 0xffffffffu;
    for (int base = 0; base < mj; base += 32) {
      const int i = base + threadIdx.x;
      unsigned long long v = i < mj ? s.pmk[i + 1] : kSentinel;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long u = __shfl_up_sync(0xffffffffu, v, o);
        if ((int)threadIdx.x >= o) v = u < v ? u : v;
      }
      v = carry < v ? carry : v;
      if (i < mj) s.pmk[i + 1] = v;
      carry = __shfl_sync(0xffffffffu, v, 31);
      uint32_t v32 = i < mj ? s.pm32[i + 1] : 0xffffffffu;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, v32, o);
        if ((int)threadIdx.x >= o) v32 = u < v32 ? u : v32;
      }
      v32 = carry32 < v32 ? carry32 : v32;
      if (i < mj) s.pm32[i + 1] = v32;
      carry32 = __shfl_sync(0xffffffffu, v32, 31);
    }
    if (threadIdx.x == 0) {
      s.pmk[0] = kSentinel;
      s.pm32[0] = kLocalInfeasible;
    }
  }
  __syncthreads();

  // An infinite SLO admits every candidate whose weights are all finite (the
  // reference skips non-finite menu weights, autoscaler.py:800-801): compare
  // against DBL_MAX, which keeps the INF-weighted (unstable) entries out.
  const double slo = fmin(slo_w[w], 1.7976931348623157e308);
  // opaque copies: keeps the k loop from rematerialising the addresses
  // (CgaCtaId + parameter loads) in every iteration under register pressure
  const uint32_t a_wk = opaque_u32((uint32_t)__cvta_generic_to_shared(s.w + koff));
  const uint32_t a_kk = opaque_u32((uint32_t)__cvta_generic_to_shared(s.kk32));
  const uint32_t a_pm = opaque_u32((uint32_t)__cvta_generic_to_shared(s.pm32));
  const int mk_r = (int)opaque_u32((uint32_t)mk);
  unsigned long long best = kSentinel;
  if (qps_w[w] > 0.0) {
    const int nout = c.n - c.il;
    double wj[NJ > 0 ? NJ : 1];
#pragma unroll
    for (int i = 0; i < NJ; ++i) wj[i] = i < mj ? s.jw[i] : OPSC_INF;
    constexpr int NK = KREG ? NJ : 1;
    double wk[NK];
    uint32_t kkr[NK];
#pragma unroll
    for (int i = 0; i < NK; ++i) {
      wk[i] = KREG && i < mk ? s.w[koff + i] : OPSC_INF;
      kkr[i] = KREG && i < mk ? s.kk32[i] : 0u;
    }
    // c.spc consecutive 256-thread slices of this window per CTA: the
    // shared tables above are built once per CTA and amortised over them
    for (int sl = 0; sl < c.spc; ++sl) {
      const uint32_t o = c.lo + (uint32_t)(bw * c.spc + sl) * kComposeThreads + threadIdx.x;
      if (o >= c.hi) break;
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

      // register tiles (NJ > 0, compose_setup guarantees c.tkey): the thread's
      // running minimum as one 32-bit local key over the middle, k and j levels
      // (pb = the middle levels' part), decoded once
      constexpr bool tkey = NJ > 0;
      uint32_t best32 = 0xffffffffu;
      // The k and j levels for one prefix (middle digits fixed): pb / cost1 /
      // lex1 are the prefix's key parts (local key, or objective and index).
      auto kj_levels = [&](double in_k, double bj0, double lo0, uint32_t pb, long long cost1,
                           unsigned long long lex1) {
        if constexpr (NJ > 0) {
          uint32_t m32;
          if constexpr (KREG) {
            m32 = k_level_reg<NJ, CHAIN>(a_pm, wk, kkr, wj, in_k, bj0, lo0, k_to_j, k_sink, slo);
          } else {
            m32 = k_level_tile<NJ, CHAIN>(a_wk, a_kk, a_pm, mk_r, wj, in_k, bj0, lo0, k_to_j, k_sink, slo);
          }
          // m32 < 2^31 + (kk part) and kk part + pb < 2^31 (the host's local-key
          // budget), so m32 + pb never wraps and stays >= 2^31 when infeasible
          const uint32_t t = m32 + pb;
          best32 = t < best32 ? t : best32;
        } else {
          const unsigned long long mbest = k_level_smem<CHAIN>(s, mk, mj, koff, in_k, bj0, lo0, k_to_j, k_sink, slo);
          if (mbest < kSentinel) {
            const unsigned long long key = ((unsigned long long)cost1 << OPSC_KEY_LEX_BITS) + lex1 + mbest;
            best = key < best ? key : best;
          }
        }
      };

      // Middle levels (<= kOdoLevels of them): the last one is a plain loop
      // over its menu, the ones above it an odometer, all DP values in
      // registers (no per-index digit divisions, no DP through local memory).
      // A dp_in is a max over predecessors (exact, order-free), so it splits
      // into the outer predecessors' part, fixed per thread, and the middle ones'.
      const int nmid = kp - nout;  // <= kOdoLevels (compose_setup: il <= kOdoLevels + 2)
      {
        const uint32_t outer = (1u << nout) - 1u;
        const int nm1 = nmid > 0 ? nmid - 1 : 0;  // odometer levels above the last middle level
        const int lpos = nout + nmid - 1;         // the last middle level (nmid > 0)
        const uint32_t m_last = nmid > 0 ? (uint32_t)c.m[lpos] : 1u;
        const uint32_t n_pre = c.mid_count / m_last;
        int od[kOdoLevels];
        double o_in[kOdoLevels], mv[kOdoLevels];
  #pragma unroll
        for (int l = 0; l < kOdoLevels; ++l) {
          od[l] = 0;
          mv[l] = 0.0;
          o_in[l] = (!PATH && l < nmid) ? dp_in(c.pmask[nout + l] & outer, val) : 0.0;
        }
        const double o_k = !PATH ? dp_in(c.pmask[kp] & outer, val) : 0.0;
        const double o_j = !PATH ? dp_in(c.pmask[jp] & ~kmask & outer, val) : 0.0;
        const double o_lo = !PATH ? dp_in(c.sinkmask & ~(kmask | jmask) & outer, val) : 0.0;
        // path suffix: the first in-thread position's dp_in (outer predecessors
        // only), +inf if an outer sink already misses the SLO
        double pv0 = 0.0;
        if constexpr (PATH) {
          pv0 = dp_in(c.pmask[nout], val);
          if (!(dp_in(c.sinkmask & outer, val) <= slo)) pv0 = OPSC_INF;
        }
        const uint32_t bit_last = nmid > 0 ? 1u << lpos : 0u;
        const bool last_to_k = (c.pmask[kp] & bit_last) != 0;
        const bool last_to_j = (c.pmask[jp] & ~kmask & bit_last) != 0;
        const bool last_sink = (c.sinkmask & bit_last) != 0;
        const int off_last = nmid > 0 ? c.off[lpos] : c.E;  // entry E: weight +0.0, cost 0, local key 0
        const unsigned long long stride_last = nmid > 0 ? c.stride[lpos] : 0ull;

        for (uint32_t pre = 0; pre < n_pre; ++pre) {
          if (pre > 0) {  // advance the odometer (innermost level fastest)
            bool carry = true;
  #pragma unroll
            for (int l = kOdoLevels - 1; l >= 0; --l) {
              if (l < nm1 && carry) {
                if (++od[l] == c.m[nout + l]) od[l] = 0;
                else carry = false;
              }
            }
          }
          // prefix state over the odometer levels
          long long pc = cost0;
          unsigned long long pl = lex0;
          uint32_t pbp = 0;
          double pv = pv0;                                 // PATH: dp_in of the next position
          double in_k = o_k, bj0 = o_j, lo0 = o_lo, in_last = 0.0;  // generic
          if (!PATH && nmid > 0) in_last = o_in[nmid - 1];
  #pragma unroll
          for (int l = 0; l < kOdoLevels; ++l) {
            if (l < nm1) {
              const int pos = nout + l;
              const int e = c.off[pos] + od[l];
              if constexpr (PATH) {
                pv = clamp0(pv + s.w[e]);  // val[pos], then the next position's dp_in
              } else {
                double in = o_in[l];
  #pragma unroll
                for (int l2 = 0; l2 < l; ++l2)
                  if (c.pmask[pos] >> (nout + l2) & 1u) in = fmax(in, mv[l2]);
                mv[l] = in + s.w[e];
                const uint32_t bit = 1u << pos;
                if (c.pmask[kp] & bit) in_k = fmax(in_k, mv[l]);
                if (c.pmask[jp] & ~kmask & bit) bj0 = fmax(bj0, mv[l]);
                if (c.sinkmask & bit) lo0 = fmax(lo0, mv[l]);
                if (c.pmask[lpos] & bit) in_last = fmax(in_last, mv[l]);
              }
              if constexpr (tkey) {
                pbp += s.lk32[e];
              } else {
                pc += s.cost[e];
                pl += (unsigned long long)od[l] * c.stride[pos];
              }
            }
          }
  #pragma unroll(kLUnroll)
          for (uint32_t i = 0; i < m_last; ++i) {  // the last middle level (none: the virtual entry E)
            const int e = off_last + (int)i;
            const double wl = s.w[e];
            const uint32_t pb = tkey ? pbp + s.lk32[e] : 0u;
            const long long cost1 = tkey ? 0 : pc + s.cost[e];
            const unsigned long long lex1 = tkey ? 0ull : pl + (unsigned long long)i * stride_last;
            if constexpr (PATH) {
              kj_levels(clamp0(pv + wl), 0.0, 0.0, pb, cost1, lex1);
            } else {
              const double v = in_last + wl;
              double ik = last_to_k ? fmax(in_k, v) : in_k;
              const double b0 = last_to_j ? fmax(bj0, v) : bj0;
              const double l0 = last_sink ? fmax(lo0, v) : lo0;
              if (CHAIN && !(l0 <= slo)) ik = OPSC_INF;  // another sink already misses the SLO
              kj_levels(ik, b0, l0, pb, cost1, lex1);
            }
          }
        }
      }
      if (NJ > 0 && best32 < kLocalInfeasible) {  // decode the slice's in-thread minimum once
        const uint32_t loc = best32 & 0xfffffu;
        unsigned long long lex = lex0;
        for (int pos = nout; pos < c.n; ++pos)
          lex += (unsigned long long)((loc / c.cs[pos]) % (uint32_t)c.m[pos]) * c.stride[pos];
        const unsigned long long key = ((unsigned long long)(cost0 + (best32 >> 20)) << OPSC_KEY_LEX_BITS) + lex;
        best = key < best ? key : best;
      }
    }
  }
  cta_min_commit(best, w, key_out, peers, warp_best);
}

// Dynamic shared memory of the tile kernel: menu slab + costs, k / j tables.
static size_t compose_smem_bytes(int E, int mk, int mj) {
  return (size_t)mk * 8 + (size_t)(mj + 1) * 8 + (size_t)(E + 1) * 8 + (size_t)mj * 8 + (size_t)(E + 1) * 4 +
         (size_t)mk * 4 + (size_t)(mj + 1) * 4 + (size_t)(E + 1) * 4;
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
    if (m < 1) return OPSC_ERR_ARG;
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
      c.vop[pos] = -1;
      continue;
    }
    const int v = d.topo[pos - nvirt];
    c.vop[pos] = v;
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
  // Large menus: the shared-memory tile needs every window's menu slab plus
  // the k / j tables on chip; past ~200 KB (or a menu over 65535 entries)
  // the flat kernel runs instead.
  {
    const size_t mj = (size_t)c.m[c.n - 1], mk = (size_t)c.m[c.n - 2];
    const size_t need = compose_smem_bytes(c.E, (int)mk, (int)mj);
    int big = 0;
    for (int pos = 0; pos < c.n; ++pos) big |= c.m[pos] > 65535;
    if (big || need > 200 * 1024) {
      c.flat = 1;
      c.flo = s * (unsigned long long)shard / (unsigned long long)n_shards;
      c.fhi = s * (unsigned long long)(shard + 1) / (unsigned long long)n_shards;
      const unsigned long long per_cta = (unsigned long long)kComposeThreads * 64ull;
      unsigned long long bpw = (c.fhi - c.flo + per_cta - 1) / per_cta;
      const unsigned long long cap = (unsigned long long)(148 * 8 * 4) / (unsigned long long)(n_windows > 0 ? n_windows : 1) + 1;
      bpw = bpw < 1 ? 1 : bpw;
      bpw = bpw > cap ? cap : bpw;
      c.blocks_per_window = (int)bpw;
      *cfg = c;
      return OPSC_OK;
    }
  }
  // level split: enough in-thread candidates to amortise the outer decode,
  // while keeping at least half a wave of threads
  auto prod = [&](int lo, int hi) {
    double x = 1.0;
    for (int pos = lo; pos < hi; ++pos) x *= c.m[pos];
    return x;
  };
  const double min_threads = 148.0 * 512.0;
  // thread counts are per rank: a shard enumerates 1/n_shards of the outer space
  const double per_rank = (double)n_windows / (double)(n_shards > 0 ? n_shards : 1);
  int il = 2;
  while (il < c.n && il < kOdoLevels + 2) {
    const bool too_many = prod(0, c.n - il) >= 4294967295.0;
    // in-thread candidates amortise the outer decode: >= 1024, or >= 4096
    // while the next split still leaves >= 1.8M threads (~8 waves; cfg3's
    // 12-op DAG: il 4 -> 5 is +7%, tools/quick_time.py with OPSC_COMPOSE_IL)
    const double in_thread = prod(c.n - il, c.n);
    if (!too_many && in_thread >= 1024.0 &&
        (in_thread >= 4096.0 || per_rank * prod(0, c.n - il - 1) < 1.8e6))
      break;
    if (!too_many && per_rank * prod(0, c.n - il - 1) < min_threads) break;
    ++il;
  }
  if (const char* f = getenv("OPSC_COMPOSE_IL")) {  // dev override (tools/w1_latency.py)
    const int want = atoi(f);
    if (want >= 2 && want <= kOdoLevels + 2 && want <= c.n && prod(0, c.n - want) < 4294967295.0) il = want;
  }
  if (prod(0, c.n - il) >= 4294967295.0) return OPSC_ERR_SPACE;
  c.il = il;
  c.m_out = (uint32_t)prod(0, c.n - il);
  const double mid = prod(c.n - il, c.n - 2);
  if (mid >= 4294967295.0) return OPSC_ERR_SPACE;
  c.mid_count = (uint32_t)mid;
  c.lo = (uint32_t)((unsigned long long)c.m_out * shard / n_shards);
  c.hi = (uint32_t)((unsigned long long)c.m_out * (shard + 1) / n_shards);
  // slices of 256 outer indices; a CTA takes `spc` consecutive slices of its
  // window so the per-CTA table setup (menu slab, cost / key tables, weight
  // sort, prefix-minimum scan) is amortised over >= ~2M candidates, while
  // keeping >= 24 waves of CTAs (tail). cfg3: +6%; cfg5 / cfg2 stay at 1
  // (tools/variants_spc.sh)
  const long long nslices = std::max<long long>(1, ((long long)c.hi - c.lo + kComposeThreads - 1) / kComposeThreads);
  const double per_cta = (double)kComposeThreads * prod(c.n - il, c.n);
  long long spc = (long long)std::ceil(2.0e6 / per_cta);
  const long long min_ctas = 148LL * OPSC_COMPOSE_MINB * 24;
  spc = std::min<long long>(spc, ((long long)n_windows * nslices) / min_ctas);
  spc = std::max<long long>(1, std::min<long long>(spc, 16));
  if (const char* f = getenv("OPSC_COMPOSE_SPC")) spc = std::max(1, atoi(f));  // dev override
  c.spc = (int)spc;
  c.blocks_per_window = (int)((nslices + spc - 1) / spc);
  const int mj = c.m[c.n - 1], mk = c.m[c.n - 2];
  // register tile widths (padded entries are +inf and still cost their
  // DADD/DSETP/SEL, so common menu sizes get exact tiles: 6 = P{1,2} x R<=3)
  c.nj = mj <= 4 ? 4 : mj <= 6 ? 6 : mj <= 8 ? 8 : mj <= 12 ? 12 : mj <= 16 ? 16 : mj <= 24 ? 24 : mj <= 32 ? 32 : 0;
  // register-tile local keys: cost << 20 | compact index, index < 2^20 and
  // cost < 2^11. The compact index of a set of positions orders them by
  // lexicographic significance (global stride), so within one thread's
  // prefix it orders candidates exactly as the global key does.
  auto max_cost = [&](int pos) {
    int mx = 0;
    for (int e = 0; e < c.m[pos]; ++e) {
      if (c.off[pos] >= c.E) break;  // virtual position: cost 0
      const int v = d.topo[pos - nvirt];
      int p, r, b;
      opsc::entry_prb(g, v, e, p, r, b);
      mx = std::max(mx, p * r);
    }
    return mx;
  };
  auto compact = [&](int lo) {  // cs over positions lo..n-1; false if the local key does not fit
    double space = 1.0;
    long long cmax = 0;
    for (int p = lo; p < c.n; ++p) {
      space *= c.m[p];
      cmax += max_cost(p);
      unsigned long long cs = 1;
      for (int q = lo; q < c.n; ++q)
        if (c.stride[q] < c.stride[p]) cs *= (unsigned long long)c.m[q];
      c.cs[p] = (uint32_t)std::min(cs, 0xffffffffull);
    }
    return space < (double)(1 << 20) && cmax < (1 << 11);
  };
  // register tiles keep one 32-bit running minimum per thread over all its
  // in-thread levels, decoded to the global key once; when the in-thread
  // space or cost does not fit the local key, the u64 shared-memory path runs
  c.tkey = c.nj > 0 && compact(c.n - il) ? 1 : 0;
  if (!c.tkey) c.nj = 0;
  // chain fast path: j's only predecessor is k and k is not a sink
  const int jp = c.n - 1, kp = c.n - 2;
  c.chain = (c.pmask[jp] == (1u << kp)) && !(c.sinkmask >> kp & 1u);
  // path suffix: the in-thread positions form a path (each fed by the
  // previous one only; the first by outer positions only) ending in the only
  // in-thread sink j. Sinks among the outer positions are checked once per
  // thread. True for the chain DAGs (7B, 70B) and for DAGs whose branches
  // merge above the in-thread levels (the multimodal DAG).
  {
    const int nout = c.n - il;
    const uint32_t inner = ~((1u << nout) - 1u);
    c.path_dag = (c.sinkmask & inner) == (1u << jp);
    for (int pos = nout + 1; pos < c.n; ++pos) c.path_dag &= c.pmask[pos] == (1u << (pos - 1));
  }
  *cfg = c;
  return OPSC_OK;
}

template <int NJ, int MODE, bool KREG>
static cudaError_t launch_t(const ComposeCfg& c, const OpscGrid& g, int n_windows, const double* menu_w,
                            const double* slo, const double* qps, unsigned long long* key, cudaStream_t s,
                            const PeerKeys& pk) {
  const int mj = c.m[c.n - 1], mk = c.m[c.n - 2];
  const size_t smem = compose_smem_bytes(c.E, mk, mj);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(compose_kernel<NJ, MODE, KREG>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  const long long blocks = (long long)n_windows * c.blocks_per_window;
  if (blocks > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  return launch_pdl(compose_kernel<NJ, MODE, KREG>, dim3((unsigned)blocks), dim3(kComposeThreads), smem, s, c, g, menu_w,
                    slo, qps, key, pk);
}

template <int NJ, bool KREG>
static cudaError_t launch_mode(const ComposeCfg& c, const OpscGrid& g, int n_windows, const double* menu_w,
                               const double* slo, const double* qps, unsigned long long* key, cudaStream_t s,
                               const PeerKeys& pk) {
  if (c.path_dag) return launch_t<NJ, 2, KREG>(c, g, n_windows, menu_w, slo, qps, key, s, pk);
  if (c.chain) return launch_t<NJ, 1, KREG>(c, g, n_windows, menu_w, slo, qps, key, s, pk);
  return launch_t<NJ, 0, false>(c, g, n_windows, menu_w, slo, qps, key, s, pk);  // k registers spill there
}

template <int NJ>
static cudaError_t launch_nj(const ComposeCfg& c, const OpscGrid& g, int n_windows, const double* menu_w,
                             const double* slo, const double* qps, unsigned long long* key, cudaStream_t s,
                             const PeerKeys& pk) {
  if constexpr (NJ > 0 && NJ <= 8) {
    if (c.m[c.n - 2] <= NJ && !getenv("OPSC_COMPOSE_NO_KREG"))
      return launch_mode<NJ, true>(c, g, n_windows, menu_w, slo, qps, key, s, pk);
  }
  return launch_mode<NJ, false>(c, g, n_windows, menu_w, slo, qps, key, s, pk);
}

cudaError_t launch_compose(const ComposeCfg& c, const OpscGrid& g, int n_windows, const double* menu_w,
                           const double* slo, const double* qps, unsigned long long* key, cudaStream_t s,
                           const PeerKeys* peers) {
  if (n_windows <= 0 || (!c.flat && c.hi <= c.lo)) return cudaSuccess;
  PeerKeys pk;
  memset(&pk, 0, sizeof(pk));
  if (peers) pk = *peers;
  if (c.flat) {
    if (c.fhi <= c.flo) return cudaSuccess;
    const long long blocks = (long long)n_windows * c.blocks_per_window;
    if (blocks > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
    return launch_pdl(compose_flat_kernel<false>, dim3((unsigned)blocks), dim3(kComposeThreads), 0, s, c, g, menu_w, slo,
                      qps, key, pk, 0.0);
  }
  switch (c.nj) {
    case 4: return launch_nj<4>(c, g, n_windows, menu_w, slo, qps, key, s, pk);
    case 6: return launch_nj<6>(c, g, n_windows, menu_w, slo, qps, key, s, pk);
    case 8: return launch_nj<8>(c, g, n_windows, menu_w, slo, qps, key, s, pk);
    case 12: return launch_nj<12>(c, g, n_windows, menu_w, slo, qps, key, s, pk);
    case 16: return launch_nj<16>(c, g, n_windows, menu_w, slo, qps, key, s, pk);
    case 24: return launch_nj<24>(c, g, n_windows, menu_w, slo, qps, key, s, pk);
    case 32: return launch_nj<32>(c, g, n_windows, menu_w, slo, qps, key, s, pk);
    default: return launch_nj<0>(c, g, n_windows, menu_w, slo, qps, key, s, pk);
  }
}

// Boundary diagnostic over the whole candidate space (flat kernel, literal).
cudaError_t launch_compose_boundary(const ComposeCfg& c0, const OpscGrid& g, int n_windows, const double* menu_w,
                                    const double* slo, const double* qps, double band_ulps,
                                    unsigned long long* count, cudaStream_t s) {
  if (n_windows <= 0) return cudaSuccess;
  ComposeCfg c = c0;
  unsigned long long space = 1;
  for (int pos = 0; pos < c.n; ++pos) space *= (unsigned long long)c.m[pos];
  c.flo = 0;
  c.fhi = space;
  const unsigned long long per_cta = (unsigned long long)kComposeThreads * 256ull;
  unsigned long long bpw = (space + per_cta - 1) / per_cta;
  const unsigned long long cap = 148ull * 16ull * 8ull / (unsigned long long)n_windows + 1ull;
  bpw = bpw < 1 ? 1 : (bpw > cap ? cap : bpw);
  c.blocks_per_window = (int)bpw;
  const long long blocks = (long long)n_windows * c.blocks_per_window;
  if (blocks > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  PeerKeys pk;
  memset(&pk, 0, sizeof(pk));
  compose_flat_kernel<true><<<(unsigned)blocks, kComposeThreads, 0, s>>>(c, g, menu_w, slo, qps, count, pk,
                                                                          band_ulps);
  return cudaGetLastError();
}


// Summation-order certificate (opt-in, OPSC_PLAN_CERTIFY / opsc_certify_order).
// The reference accepts a leaf when its frozenset-ordered plain and Neumaier
// path sums are <= slo (autoscaler.py:792-796); any such sum of the same
// weights lies within a few ulps of the canonical DP latency. With
// band = band_ulps * ulp(slo), every candidate the reference could accept is
// in F_hi = {lat <= slo + band} and every candidate it must accept is in
// F_lo = {lat <= slo - band}. The reference's argmin is squeezed between
// argmin(F_hi) and argmin(F_lo) (the same key order), so equal keys certify
// the window's decision for every PYTHONHASHSEED (both empty: the per-op
// fallback, which does not depend on the SLO). Unequal keys set
// OPSC_W_ORDER_SENSITIVE. Cost: two more compose launches over the window.
__global__ void certify_prep_kernel(int n, const double* __restrict__ slo, double band_ulps, double* __restrict__ lo,
                                    double* __restrict__ hi, unsigned long long* __restrict__ klo,
                                    unsigned long long* __restrict__ khi) {
  pdl_trigger();
  pdl_wait();
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= n) return;
  const double s = slo[w];
  double band = 0.0;
  if (s < OPSC_INF) band = band_ulps * (nextafter(s, OPSC_INF) - s);
  lo[w] = s - band;
  hi[w] = s + band;
  klo[w] = (unsigned long long)OPSC_KEY_INFEASIBLE;
  khi[w] = (unsigned long long)OPSC_KEY_INFEASIBLE;
}

__global__ void certify_mark_kernel(int n, const unsigned long long* __restrict__ klo,
                                    const unsigned long long* __restrict__ khi, uint32_t* __restrict__ status) {
  pdl_trigger();
  pdl_wait();
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w < n && klo[w] != khi[w]) status[w] |= OPSC_W_ORDER_SENSITIVE;
}

size_t certify_workspace(int n_windows) { return n_windows > 0 ? (size_t)n_windows * 32u : 0u; }

cudaError_t launch_certify(const ComposeCfg& c, const OpscGrid& g, int n_windows, const double* menu_w,
                           const double* slo, const double* qps, double band_ulps, void* ws, uint32_t* status,
                           cudaStream_t s) {
  if (n_windows <= 0) return cudaSuccess;
  double* lo = (double*)ws;
  double* hi = lo + n_windows;
  unsigned long long* klo = (unsigned long long*)(hi + n_windows);
  unsigned long long* khi = klo + n_windows;
  const unsigned nb = (unsigned)((n_windows + 255) / 256);
  cudaError_t e = launch_pdl(certify_prep_kernel, dim3(nb), dim3(256), 0, s, n_windows, slo, band_ulps, lo, hi, klo, khi);
  if (e == cudaSuccess) e = launch_compose(c, g, n_windows, menu_w, lo, qps, klo, s);
  if (e == cudaSuccess) e = launch_compose(c, g, n_windows, menu_w, hi, qps, khi, s);
  if (e == cudaSuccess) e = launch_pdl(certify_mark_kernel, dim3(nb), dim3(256), 0, s, n_windows,
                                       (const unsigned long long*)klo, (const unsigned long long*)khi, status);
  return e;
}

}  // namespace opsc
