// Candidate inner-loop variants for K2 (dev probe, not product code).
// Each variant evaluates 24 candidates lat_i = bj + w_i against slo per
// outer iteration and yields the smallest i with lat_i <= slo.
//   1: DADD + DSETP + SEL                       (current K2)
//   2: DADD + ISETP(hi word) + SEL, exact check (superset mask on the high word)
//   3: DADD + ISETP(hi) packed with P2R         (mask of 24 bits, FLO once)
//   4: DADD + IMAD/SHF funnel mask              (sign-bit gather)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cand_probe cand_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int KIND>
__global__ void __launch_bounds__(256, 4) probe(int iters, double seed, double* sink, uint32_t two) {
  double wj[24];
#pragma unroll
  for (int i = 0; i < 24; ++i) wj[i] = seed * (1.0 + 0.01 * i) + 1e-3 * threadIdx.x;
  const double slo = seed * 1.2;
  const uint32_t H = (uint32_t)(__double_as_longlong(slo) >> 32);
  const float HB = __int_as_float((int)H + 1) * 16777216.0f;
  double bj = 1e-4 * (threadIdx.x & 7);
  int acc = 0;
  for (int it = 0; it < iters; ++it) {
    int inner = 24;
    if (KIND == 1) {
#pragma unroll
      for (int i = 23; i >= 0; --i) {
        const double lat = bj + wj[i];
        if (lat <= slo) inner = i;
      }
    } else if (KIND == 2) {
#pragma unroll
      for (int i = 23; i >= 0; --i) {
        const double lat = bj + wj[i];
        if ((uint32_t)__double2hiint(lat) <= H) inner = i;
      }
    } else if (KIND == 3) {
      uint32_t m = 0;
#pragma unroll
      for (int i = 0; i < 24; ++i) {
        const double lat = bj + wj[i];
        m |= ((uint32_t)__double2hiint(lat) <= H ? 1u : 0u) << i;
      }
      inner = m ? __ffs(m) - 1 : 24;
    } else if (KIND == 5) {
#pragma unroll
      for (int i = 23; i >= 0; --i) {
        const double lat = bj + wj[i];
        asm("{.reg .pred p; setp.le.u32 p, %1, %2; @p mov.u32 %0, %3;}" : "+r"(inner) : "r"((uint32_t)__double2hiint(lat)), "r"(H), "r"(i));
      }
    } else if (KIND == 6) {
      // 2 candidates per select: hi words compared, results combined by IMAD arithmetic
#pragma unroll
      for (int i = 23; i >= 0; --i) {
        const double lat = bj + wj[i];
        const uint32_t v = (uint32_t)__double2hiint(lat) - H - 1u;  // bit31 set <=> hi(lat) <= H
        inner = (int)v < 0 ? i : inner;
      }
    } else if (KIND == 7) {
      // weight-sorted menu: count hi-word failures (superset mask), exact fix-up later
      uint32_t fails = 0;
#pragma unroll
      for (int i = 0; i < 24; ++i) {
        const double lat = bj + wj[i];
        fails += (H - (uint32_t)__double2hiint(lat)) >> 31;
      }
      inner = (int)fails;
    } else if (KIND == 8) {
      uint32_t fails = 0;
#pragma unroll
      for (int i = 0; i < 24; ++i) {
        const double lat = bj + wj[i];
        const uint32_t x = H - (uint32_t)__double2hiint(lat);
        asm("mad.hi.u32 %0, %1, %2, %0;" : "+r"(fails) : "r"(x), "r"(two));
      }
      inner = (int)fails;
    } else if (KIND == 9) {
      // count of hi32(lat) <= H in FP32 on the FMA pipe: t = sat(HB - f*BIG)
      float acc0 = 0.f, acc1 = 0.f;
#pragma unroll
      for (int i = 0; i < 24; ++i) {
        const double lat = bj + wj[i];
        const float f = __int_as_float(__double2hiint(lat));
        const float t = __saturatef(__fmaf_rn(f, -16777216.0f, HB));
        if (i & 1) acc1 += t; else acc0 += t;
      }
      inner = (int)(acc0 + acc1);
    } else if (KIND == 10) {
      // DSETP only, predicates AND-chained (DSETP.LE.AND P, ..., P)
      bool ok = true;
#pragma unroll
      for (int i = 0; i < 24; ++i) ok = ok & (wj[i] <= bj);
      inner = ok;
    } else if (KIND == 11) {
      // DADD + DSETP, predicates AND-chained (no select)
      bool ok = true;
#pragma unroll
      for (int i = 0; i < 24; ++i) ok = ok & (bj + wj[i] <= slo);
      inner = ok;
    } else if (KIND == 12) {
      // DADD only: hi words OR-ed (DADD + LOP3 per candidate)
      uint32_t m = 0;
#pragma unroll
      for (int i = 0; i < 24; i += 2) m |= (uint32_t)__double2hiint(bj + wj[i]) ^ (uint32_t)__double2hiint(bj + wj[i + 1]);
      inner = (int)m;
    } else {
      uint32_t m = 0;
#pragma unroll
      for (int i = 23; i >= 0; --i) {
        const double lat = bj + wj[i];
        const uint32_t v = H - (uint32_t)__double2hiint(lat);  // bit31 set <=> hi(lat) > H
        m = __funnelshift_l(v, m, 1);
      }
      m = ~m & 0xffffffu;  // bit (23-i) set <=> hi(lat_i) <= H
      inner = m ? 23 - (31 - __clz(m)) : 24;
    }
    acc += inner;
    bj = bj + 1e-7;
  }
  if (acc == 12345) sink[blockIdx.x] = bj;
}

template <int K>
static float run(int iters, double* sink, int blocks) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  probe<K><<<blocks, 256>>>(iters / 10, 1.0, sink, 2u);
  cudaEventRecord(a);
  probe<K><<<blocks, 256>>>(iters, 1.0, sink, 2u);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  double* sink;
  cudaMalloc(&sink, 1 << 20);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 4 * 8;
  const int iters = 20000;
  const double cands = (double)blocks * 256 * iters * 24;
  float t[13];
  t[1] = run<1>(iters, sink, blocks); t[2] = run<2>(iters, sink, blocks); t[3] = run<3>(iters, sink, blocks);
  t[4] = run<4>(iters, sink, blocks); t[5] = run<5>(iters, sink, blocks); t[6] = run<6>(iters, sink, blocks);
  t[7] = run<7>(iters, sink, blocks); t[8] = run<8>(iters, sink, blocks); t[9] = run<9>(iters, sink, blocks);
  t[10] = run<10>(iters, sink, blocks); t[11] = run<11>(iters, sink, blocks); t[12] = run<12>(iters, sink, blocks);
  for (int k = 1; k <= 12; ++k) printf("kind%d %.3e cand/s\n", k, cands / t[k] * 1e3);
  return 0;
}
