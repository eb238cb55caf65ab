// k_compose.cu -- K2 compose_mask_argmin: exhaustive enumeration of every
// window's (P,R,B)^n candidate space, SLO mask, and lexicographic argmin.
//
// Replaces brute_force_autoscale's descend / leaf test (autoscaler.py:786-826)
// with a literal enumeration: every candidate's iteration latency is composed
// as the critical-path DP of opgraph.py:223-244 (max over predecessors, then
// + own weight, in topological order), masked with `<= slo`, and reduced with
// key = (objective << 40) | lexicographic index (ops sorted by id, per op
// (P,R,B) ascending; autoscaler.py:725, 747-749, 795). Because the key carries
// the global lexicographic index, traversal order, sharding and reduction
// order cannot change the winner.
//
// Work split (one CTA = 256 threads of one window):
//   * positions = topological order of the ops; the last two positions are the
//     k and j levels, `il-2` middle levels sit above them, the rest are
//     "outer" and fixed per thread (decoded from the thread's outer index);
//   * the j menu (innermost) lives in registers: per candidate the thread does
//     one DADD (path extension), one DSETP (SLO mask) and one predicated
//     32-bit min of (P*R << 16 | j) -- prefix hoisting keeps the rest of the
//     DP out of the inner loop;
//   * menus + per-entry costs are staged once per CTA in shared memory; the
//     k level reads them as warp-broadcast LDS;
//   * CTA result = warp-shuffle u64 min -> smem -> one atomicMin per CTA.
#include <algorithm>
#include <cstring>

#include "opsc_common.cuh"

namespace opsc {

constexpr int kComposeThreads = 256;

__device__ __forceinline__ double dp_in(uint32_t pm, const double* val) {
  double in = 0.0;
  while (pm) {
    const int p = __ffs(pm) - 1;
    pm &= pm - 1;
    in = fmax(in, val[p]);
  }
  return in;
}

template <int NJ>
__global__ void __launch_bounds__(kComposeThreads, 2)
compose_kernel(const __grid_constant__ ComposeCfg c, const __grid_constant__ OpscGrid g,
               const double* __restrict__ menu_w, const double* __restrict__ slo_w,
               const double* __restrict__ qps_w, unsigned long long* __restrict__ key_out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* sw = reinterpret_cast<double*>(smem_raw);
  int32_t* sc = reinterpret_cast<int32_t*>(sw + c.E + 1);
  __shared__ unsigned long long warp_best[kComposeThreads / 32];

  const int w = blockIdx.x / c.blocks_per_window;
  const int bw = blockIdx.x - w * c.blocks_per_window;
  const double* src = menu_w + (size_t)w * c.E;
  for (int i = threadIdx.x; i < c.E; i += kComposeThreads) {
    sw[i] = src[i];
    int v = 0;
    while (i >= g.menu_off[v + 1]) ++v;
    int p, r, b;
    entry_prb(g, v, i - g.menu_off[v], p, r, b);
    sc[i] = p * r;  // objective contribution (autoscaler.py:220-221, 756)
  }
  if (threadIdx.x == 0) {  // the virtual entry (weight 0, cost 0)
    sw[c.E] = 0.0;
    sc[c.E] = 0;
  }
  __syncthreads();

  const double slo = slo_w[w];
  unsigned long long best = (unsigned long long)OPSC_KEY_INFEASIBLE;
  const uint32_t o = c.lo + (uint32_t)bw * kComposeThreads + threadIdx.x;
  if (qps_w[w] > 0.0 && o < c.hi) {
    const int jp = c.n - 1, kp = c.n - 2, nout = c.n - c.il;
    const int joff = c.off[jp], mj = c.m[jp];
    double wj[NJ > 0 ? NJ : 1];
    uint32_t kj[NJ > 0 ? NJ : 1];
#pragma unroll
    for (int i = 0; i < NJ; ++i) {
      const bool ok = i < mj;
      wj[i] = ok ? sw[joff + i] : OPSC_INF;
      kj[i] = ok ? ((uint32_t)sc[joff + i] << 16 | (uint32_t)i) : 0xffffffffu;
    }
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
      val[pos] = dp_in(c.pmask[pos], val) + sw[e];
      cost0 += sc[e];
      lex0 += (unsigned long long)dig[pos] * c.stride[pos];
    }
    const uint32_t kmask = 1u << kp, jmask = 1u << jp;
    const bool k_to_j = (c.pmask[jp] & kmask) != 0;
    const bool k_sink = (c.sinkmask & kmask) != 0;
    const int koff = c.off[kp], mk = c.m[kp];
    const unsigned long long kstride = c.stride[kp], jstride = c.stride[jp];

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
        val[pos] = dp_in(c.pmask[pos], val) + sw[e];
        cost1 += sc[e];
        lex1 += (unsigned long long)dig[pos] * c.stride[pos];
      }
      const double in_k = dp_in(c.pmask[kp], val);
      const double bj0 = dp_in(c.pmask[jp] & ~kmask, val);
      const double lo0 = dp_in(c.sinkmask & ~(kmask | jmask), val);

      for (int a = 0; a < mk; ++a) {
        const double bk = in_k + sw[koff + a];
        double bj = k_to_j ? fmax(bj0, bk) : bj0;
        const double lo = k_sink ? fmax(lo0, bk) : lo0;
        if (!(lo <= slo)) bj = OPSC_INF;
        uint32_t in0 = 0xffffffffu, in1 = 0xffffffffu;
        if (NJ > 0) {
#pragma unroll
          for (int i = 0; i < NJ; i += 2) {
            const double l0 = bj + wj[i];
            if (l0 <= slo) in0 = min(in0, kj[i]);
            if (i + 1 < NJ) {
              const double l1 = bj + wj[i + 1];
              if (l1 <= slo) in1 = min(in1, kj[i + 1]);
            }
          }
        } else {
          for (int i = 0; i < mj; ++i) {
            const double l0 = bj + sw[joff + i];
            if (l0 <= slo) in0 = min(in0, (uint32_t)sc[joff + i] << 16 | (uint32_t)i);
          }
        }
        const uint32_t inner = min(in0, in1);
        if (inner != 0xffffffffu) {
          const unsigned long long cst =
              (unsigned long long)(cost1 + sc[koff + a] + (long long)(inner >> 16));
          const unsigned long long lx = lex1 + (unsigned long long)a * kstride +
                                        (unsigned long long)(inner & 0xffffu) * jstride;
          const unsigned long long key = cst << OPSC_KEY_LEX_BITS | lx;
          best = key < best ? key : best;
        }
      }
    }
  }
  best = warp_min_u64(best);
  if ((threadIdx.x & 31) == 0) warp_best[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x < 32) {
    unsigned long long b = threadIdx.x < kComposeThreads / 32 ? warp_best[threadIdx.x]
                                                               : (unsigned long long)OPSC_KEY_INFEASIBLE;
    b = warp_min_u64(b);
    if (threadIdx.x == 0 && b != (unsigned long long)OPSC_KEY_INFEASIBLE) atomicMin(&key_out[w], b);
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
      c.stride[pos] = 0;
      c.pmask[pos] = 0;
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
  // entry costs: P*R of each entry (multiplies of <= 8 x r_max) must fit 15 bits
  for (int v = 0; v < nr; ++v)
    for (int i = 0; i < g.n_p[v]; ++i)
      if ((long long)g.p_vals[v][i] * g.r_max > 32767) return OPSC_ERR_ARG;
  // level split: as many in-thread levels as keep >= ~1 wave of threads
  auto m_out = [&](int il) {
    double x = 1.0;
    for (int pos = 0; pos < c.n - il; ++pos) x *= c.m[pos];
    return x;
  };
  const double target = 148.0 * 1024.0;
  int il = 2;
  while (il < c.n && il < 6 &&
         (m_out(il) >= 4294967295.0 || (double)n_windows * m_out(il + 1) >= target))
    ++il;
  if (m_out(il) >= 4294967295.0) return OPSC_ERR_SPACE;
  c.il = il;
  c.m_out = (uint32_t)m_out(il);
  double mid = 1.0;
  for (int pos = c.n - il; pos < c.n - 2; ++pos) mid *= c.m[pos];
  if (mid >= 4294967295.0) return OPSC_ERR_SPACE;
  c.mid_count = (uint32_t)mid;
  c.lo = (uint32_t)((unsigned long long)c.m_out * shard / n_shards);
  c.hi = (uint32_t)((unsigned long long)c.m_out * (shard + 1) / n_shards);
  c.blocks_per_window = (int)((c.hi - c.lo + kComposeThreads - 1) / kComposeThreads);
  if (c.blocks_per_window < 1) c.blocks_per_window = 1;
  const int mj = c.m[c.n - 1];
  c.nj = mj <= 4 ? 4 : mj <= 8 ? 8 : mj <= 12 ? 12 : mj <= 16 ? 16 : mj <= 24 ? 24 : mj <= 32 ? 32 : 0;
  *cfg = c;
  return OPSC_OK;
}

template <int NJ>
static cudaError_t launch_nj(const ComposeCfg& c, const OpscGrid& g, int n_windows,
                             const double* menu_w, const double* slo, const double* qps,
                             unsigned long long* key, cudaStream_t s) {
  const size_t smem = (size_t)(c.E + 1) * (sizeof(double) + sizeof(int32_t));
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(compose_kernel<NJ>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  const long long blocks = (long long)n_windows * c.blocks_per_window;
  if (blocks > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  compose_kernel<NJ><<<(unsigned)blocks, kComposeThreads, smem, s>>>(c, g, menu_w, slo, qps, key);
  return cudaGetLastError();
}

cudaError_t launch_compose(const ComposeCfg& c, const OpscGrid& g, int n_windows,
                           const double* menu_w, const double* slo, const double* qps,
                           unsigned long long* key, cudaStream_t s) {
  if (n_windows <= 0 || c.hi <= c.lo) return cudaSuccess;
  switch (c.nj) {
    case 4: return launch_nj<4>(c, g, n_windows, menu_w, slo, qps, key, s);
    case 8: return launch_nj<8>(c, g, n_windows, menu_w, slo, qps, key, s);
    case 12: return launch_nj<12>(c, g, n_windows, menu_w, slo, qps, key, s);
    case 16: return launch_nj<16>(c, g, n_windows, menu_w, slo, qps, key, s);
    case 24: return launch_nj<24>(c, g, n_windows, menu_w, slo, qps, key, s);
    case 32: return launch_nj<32>(c, g, n_windows, menu_w, slo, qps, key, s);
    default: return launch_nj<0>(c, g, n_windows, menu_w, slo, qps, key, s);
  }
}

}  // namespace opsc
