// k_windowize.cu -- trace -> per-window demand points on the device
// (reference workload.py:107-158).
//
//   horizon      = max arrival            (block max -> atomicMax on the IEEE bits)
//   n_windows    = max(1, ceil(horizon / len + 1e-12))
//   window(r)    = min(int(t / len), n - 1)   (count + output-token sum atomics)
//   grouping     = exclusive scan of counts + scatter of input lengths
//   q-quantile   = k-th smallest input length, k = max(0, ceil(q*count) - 1)
//                  ("higher" empirical quantile), by a per-window CTA radix
//                  select (3 passes of 11/11/10 bits over the uint32 values)
// Integer counts / sums are exact, so qps = count/len and sum/len are the
// reference's bits.
#include "opsc_common.cuh"

namespace opsc {

struct WzWork {
  unsigned long long* horizon_bits;
  uint32_t* err;
  uint32_t* counts;
  unsigned long long* sums;
  unsigned long long* offsets;
  uint32_t* cursors;
  uint32_t* widx;
  uint32_t* grouped;
};

static size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }

size_t windowize_workspace(long long n, int max_w) {
  size_t s = 0;
  s += align16(8) + align16(4);
  s += align16(4ull * max_w) + align16(8ull * max_w) + align16(8ull * (max_w + 1)) + align16(4ull * max_w);
  s += align16(4ull * (size_t)n) * 2;
  return s;
}

static WzWork carve(void* ws, long long n, int max_w) {
  char* p = (char*)ws;
  WzWork w;
  w.horizon_bits = (unsigned long long*)p; p += align16(8);
  w.err = (uint32_t*)p; p += align16(4);
  w.counts = (uint32_t*)p; p += align16(4ull * max_w);
  w.sums = (unsigned long long*)p; p += align16(8ull * max_w);
  w.offsets = (unsigned long long*)p; p += align16(8ull * (max_w + 1));
  w.cursors = (uint32_t*)p; p += align16(4ull * max_w);
  w.widx = (uint32_t*)p; p += align16(4ull * (size_t)n);
  w.grouped = (uint32_t*)p;
  return w;
}

__global__ void wz_zero(WzWork w, int max_w) {
  pdl_trigger();  // dependents launch early; each waits for its predecessor first
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) {
    *w.horizon_bits = 0ull;
    *w.err = 0u;
  }
  if (i < max_w) {
    w.counts[i] = 0;
    w.sums[i] = 0;
    w.cursors[i] = 0;
  }
}

// non-negative doubles order like their unsigned bit patterns
__global__ void wz_horizon(const double* __restrict__ t, long long n, WzWork w) {
  pdl_trigger();  // dependents launch early; each waits for its predecessor first
  pdl_wait();
  unsigned long long m = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(t[i]);
    m = b > m ? b : m;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long x = __shfl_xor_sync(0xffffffffu, m, o);
    m = x > m ? x : m;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(w.horizon_bits, m);
}

__global__ void wz_nwin(WzWork w, double len, int max_w, int32_t* n_windows) {
  pdl_trigger();  // dependents launch early; each waits for its predecessor first
  pdl_wait();
  const double horizon = __longlong_as_double((long long)*w.horizon_bits);
  const double nw = ceil(horizon / len + 1e-12);
  long long n = nw < 1.0 ? 1 : (long long)nw;
  if (n > max_w) {
    *w.err = 1u;
    n = n > 0x7fffffffLL ? 0x7fffffffLL : n;
  }
  *n_windows = (int32_t)n;
}

// exact sum (mod 2^64, as the u64 atomics) of x over the lanes of `grp`:
// four 16-bit slices, each slice sum < 2^21
__device__ __forceinline__ unsigned long long group_sum_u64(unsigned grp, unsigned long long x) {
  unsigned long long s = 0;
#pragma unroll
  for (int sh = 0; sh < 64; sh += 16)
    s += (unsigned long long)__reduce_add_sync(grp, (unsigned)((x >> sh) & 0xffffull)) << sh;
  return s;
}

// Records of a trace arrive (nearly) in time order, so the lanes of a warp
// mostly share a window: lanes are grouped by window (__match_any_sync) and
// one leader per group adds the group's count and output-token sum -- integer
// sums, so the totals are the same in any grouping (no same-address atomic
// storm on a handful of window counters).
__global__ void wz_count(OpscTraceRecords rec, double len, WzWork w, const int32_t* __restrict__ n_windows) {
  pdl_trigger();  // dependents launch early; each waits for its predecessor first
  pdl_wait();
  if (*w.err) return;
  const long long n = *n_windows;
  const int lane = threadIdx.x & 31;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long base = (long long)blockIdx.x * blockDim.x; base < rec.n; base += stride) {
    const long long i = base + threadIdx.x;  // whole warps iterate together
    uint32_t k = 0xffffffffu;
    unsigned long long out = 0;
    if (i < rec.n) {
      long long kk = (long long)(rec.arrival[i] / len);  // int() truncates (t >= 0)
      if (kk > n - 1) kk = n - 1;
      k = (uint32_t)kk;
      w.widx[i] = k;
      out = (unsigned long long)rec.output_len[i];
    }
    const unsigned grp = __match_any_sync(0xffffffffu, k);
    const unsigned long long sum = group_sum_u64(grp, out);
    if (k != 0xffffffffu && lane == __ffs(grp) - 1) {
      atomicAdd(&w.counts[k], (uint32_t)__popc(grp));
      atomicAdd(&w.sums[k], sum);
    }
  }
}

// single-CTA exclusive scan of counts (chunks of 1024)
__global__ void __launch_bounds__(1024) wz_scan(WzWork w, const int32_t* __restrict__ n_windows) {
  pdl_trigger();  // dependents launch early; each waits for its predecessor first
  pdl_wait();
  __shared__ unsigned long long part[1024];
  __shared__ unsigned long long carry;
  if (*w.err) return;
  const int n = *n_windows;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < n; base += 1024) {
    const int i = base + threadIdx.x;
    const unsigned long long v = i < n ? w.counts[i] : 0;
    part[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
      const unsigned long long add = threadIdx.x >= o ? part[threadIdx.x - o] : 0;
      __syncthreads();
      part[threadIdx.x] += add;
      __syncthreads();
    }
    if (i < n) w.offsets[i] = carry + part[threadIdx.x] - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry += part[1023];
    __syncthreads();
  }
  if (threadIdx.x == 0) w.offsets[n] = carry;
}

// the same grouping: one cursor reservation per (warp, window), lanes take
// consecutive slots (the order inside a window does not matter to the select)
__global__ void wz_scatter(OpscTraceRecords rec, WzWork w) {
  pdl_trigger();  // dependents launch early; each waits for its predecessor first
  pdl_wait();
  if (*w.err) return;
  const int lane = threadIdx.x & 31;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long base = (long long)blockIdx.x * blockDim.x; base < rec.n; base += stride) {
    const long long i = base + threadIdx.x;
    const uint32_t k = i < rec.n ? w.widx[i] : 0xffffffffu;
    const unsigned grp = __match_any_sync(0xffffffffu, k);
    const int leader = __ffs(grp) - 1;
    uint32_t at = 0;
    if (k != 0xffffffffu && lane == leader) at = atomicAdd(&w.cursors[k], (uint32_t)__popc(grp));
    at = __shfl_sync(grp, at, leader);
    if (k != 0xffffffffu) {
      const uint32_t rank = (uint32_t)__popc(grp & ((1u << lane) - 1u));
      w.grouped[w.offsets[k] + at + rank] = (uint32_t)rec.input_len[i];
    }
  }
}

__global__ void __launch_bounds__(256) wz_select(WzWork w, double len, double q, const int32_t* __restrict__ n_windows,
                                                 double* __restrict__ pq, int32_t* __restrict__ pl,
                                                 double* __restrict__ dq) {
  pdl_trigger();  // dependents launch early; each waits for its predecessor first
  pdl_wait();
  __shared__ uint32_t hist[2048];
  __shared__ uint32_t s_prefix, s_mask;
  __shared__ long long s_k;
  __shared__ unsigned long long s_wsum[8];
  if (*w.err) return;
  const int win = blockIdx.x;
  if (win >= *n_windows) return;
  const unsigned long long c = w.counts[win];
  if (c == 0) {
    if (threadIdx.x == 0) {
      pq[win] = 0.0;
      pl[win] = 1;
      dq[win] = 0.0;
    }
    return;
  }
  const unsigned long long off = w.offsets[win];
  if (threadIdx.x == 0) {
    long long k = (long long)ceil(q * (double)c) - 1;
    s_k = k < 0 ? 0 : k;
    s_prefix = 0;
    s_mask = 0;
  }
  const int shifts[3] = {21, 10, 0};
  const int bits[3] = {11, 11, 10};
  for (int pass = 0; pass < 3; ++pass) {
    const int nb = 1 << bits[pass];
    for (int b = threadIdx.x; b < nb; b += blockDim.x) hist[b] = 0;
    __syncthreads();
    const uint32_t prefix = s_prefix, mask = s_mask;
    for (unsigned long long i = threadIdx.x; i < c; i += blockDim.x) {
      const uint32_t v = w.grouped[off + i];
      if ((v & mask) == prefix) atomicAdd(&hist[(v >> shifts[pass]) & (uint32_t)(nb - 1)], 1u);
    }
    __syncthreads();
    // the bin holding the k-th value: each thread sums a run of nb / 256 bins,
    // a block scan of the run sums finds the run, its thread walks the run
    {
      const int per = nb / (int)blockDim.x;  // 8 or 4 bins
      const int b0 = threadIdx.x * per;
      unsigned long long run = 0;
      for (int b = 0; b < per; ++b) run += hist[b0 + b];
      unsigned long long incl = run;  // inclusive scan over the block (warp shuffles + warp totals)
      const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long x = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += x;
      }
      if (lane == 31) s_wsum[wid] = incl;
      __syncthreads();
      unsigned long long before = 0;
      for (int j = 0; j < wid; ++j) before += s_wsum[j];
      incl += before;
      const unsigned long long excl = incl - run;
      const long long k = s_k;
      __syncthreads();  // everyone has read s_k
      if ((long long)excl <= k && k < (long long)incl) {  // exactly one run holds the k-th value
        unsigned long long cum = excl;
        int sel = b0 + per - 1;
        for (int b = 0; b < per; ++b) {
          if ((long long)(cum + hist[b0 + b]) > k) {
            sel = b0 + b;
            break;
          }
          cum += hist[b0 + b];
        }
        s_k = k - (long long)cum;
        s_prefix = prefix | ((uint32_t)sel << shifts[pass]);
        s_mask = mask | ((uint32_t)(nb - 1) << shifts[pass]);
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const int v = (int)s_prefix;
    pq[win] = (double)c / len;
    pl[win] = v < 1 ? 1 : v;
    dq[win] = (double)w.sums[win] / len;
  }
}

cudaError_t launch_windowize(OpscTraceRecords rec, double len, double q, int max_w, int32_t* n_windows,
                             double* pq, int32_t* pl, double* dq, void* ws, size_t ws_bytes, cudaStream_t s) {
  if (rec.n <= 0 || max_w < 1) return cudaErrorInvalidValue;
  if (ws_bytes < windowize_workspace(rec.n, max_w)) return cudaErrorInvalidValue;
  WzWork w = carve(ws, rec.n, max_w);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long rb = (rec.n + 255) / 256;
  const int grid = (int)(rb < (long long)sms * 8 ? rb : (long long)sms * 8);
  // the chain runs under programmatic dependent launch (launch_pdl): every
  // kernel releases its successor at entry and waits for its predecessor
  cudaError_t e = launch_pdl(wz_zero, dim3((max_w + 255) / 256), dim3(256), 0, s, w, max_w);
  if (e == cudaSuccess) e = launch_pdl(wz_horizon, dim3(grid), dim3(256), 0, s, (const double*)rec.arrival, rec.n, w);
  if (e == cudaSuccess) e = launch_pdl(wz_nwin, dim3(1), dim3(1), 0, s, w, len, max_w, n_windows);
  if (e == cudaSuccess) e = launch_pdl(wz_count, dim3(grid), dim3(256), 0, s, rec, len, w, (const int32_t*)n_windows);
  if (e == cudaSuccess) e = launch_pdl(wz_scan, dim3(1), dim3(1024), 0, s, w, (const int32_t*)n_windows);
  if (e == cudaSuccess) e = launch_pdl(wz_scatter, dim3(grid), dim3(256), 0, s, rec, w);
  if (e == cudaSuccess)
    e = launch_pdl(wz_select, dim3(max_w), dim3(256), 0, s, w, len, q, (const int32_t*)n_windows, pq, pl, dq);
  return e;
}

}  // namespace opsc
