// k_peer.cu -- device flag barrier for the fused multi-GPU key merge.
//
// The compose kernel (k_compose.cu) min-reduces each CTA's key straight into
// every rank's key buffer over NVLink; before any rank decodes its keys,
// every rank's atomics must have landed. One thread per rank:
//   fence.acq_rel.sys; st.release.sys flags_p[rank] = epoch   (for every p)
//   ld.acquire.sys own_flags[q] until >= epoch                  (for every q)
// The kernel boundary after it orders the decode. A wait longer than
// timeout_ms (globaltimer) sets *err instead of hanging the GPU.
#include "opsc_common.cuh"

namespace opsc {

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void peer_barrier_kernel(const __grid_constant__ PeerFlags f, int rank, int n, uint32_t epoch,
                                    long long timeout_ns, int32_t* err) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  for (int p = 0; p < n; ++p)
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f.p[p] + rank), "r"(epoch) : "memory");
  const uint32_t* mine = f.p[rank];
  const unsigned long long t0 = global_ns();
  for (int q = 0; q < n; ++q) {
    while (true) {
      uint32_t v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mine + q) : "memory");
      if ((int32_t)(v - epoch) >= 0) break;
      if ((long long)(global_ns() - t0) > timeout_ns) {
        atomicExch(err, 1);
        return;
      }
      __nanosleep(200);
    }
  }
}

cudaError_t launch_peer_barrier(const PeerFlags& f, int rank, int n, uint32_t epoch, int timeout_ms,
                                int32_t* err, cudaStream_t s) {
  peer_barrier_kernel<<<1, 32, 0, s>>>(f, rank, n, epoch, (long long)timeout_ms * 1000000LL, err);
  return cudaGetLastError();
}

}  // namespace opsc
