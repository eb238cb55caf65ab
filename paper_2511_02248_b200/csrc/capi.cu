// capi.cu -- extern "C" entry points of libopscale_b200.so (include/opscale_b200.h).
//
// Device-pointer entry points only enqueue kernels on the caller's stream.
// The host-buffer path owns a per-context stream and device workspace, so
// concurrent callers (runner.sweep's threads, runner.py:237-240) each use
// their own context and never share mutable state.
#include <cstdio>
#include <cstring>
#include <new>

#include "opsc_common.cuh"

using namespace opsc;

namespace {

int from_cuda(cudaError_t e) { return e == cudaSuccess ? OPSC_OK : OPSC_ERR_CUDA; }

__global__ void fp64_peak_kernel(int iters, double seed, double* sink) {
  // 8 independent DADD chains per thread; DADD throughput bound
  double a0 = seed + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  double a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double x = seed * 1e-300;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      a0 = a0 + x; a1 = a1 + x; a2 = a2 + x; a3 = a3 + x;
      a4 = a4 + x; a5 = a5 + x; a6 = a6 + x; a7 = a7 + x;
    }
  }
  const double s = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
  if (s == 12345.678) sink[blockIdx.x] = s;
}

// Candidate-loop probes: kind 1 = literal (DADD + DSETP + select) per
// candidate, kind 2 = threshold form (DSETP + select) per candidate. Each
// iteration evaluates 24 candidates against a register-resident menu.
template <int KIND>
__global__ void __launch_bounds__(256, 3) cand_probe_kernel(int iters, double seed, double* sink) {
  double wj[24];
#pragma unroll
  for (int i = 0; i < 24; ++i) wj[i] = seed * (1.0 + 0.01 * i) + 1e-3 * threadIdx.x;
  const double slo = seed * 1.2;
  double bj = 1e-4 * (threadIdx.x & 7);
  int acc = 0;
  for (int it = 0; it < iters; ++it) {
    int inner = 24;
#pragma unroll
    for (int i = 23; i >= 0; --i) {
      if (KIND == 1) {
        const double lat = bj + wj[i];
        if (lat <= slo) inner = i;
      } else {
        if (wj[i] <= bj) inner = i;
      }
    }
    acc += inner;
    bj = bj + 1e-7;
  }
  if (acc == 12345) sink[blockIdx.x] = bj;
}

}  // namespace

namespace opsc {
cudaError_t launch_fp64_peak(int iters, double* sink, int* blocks, int* threads, cudaStream_t s) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  *blocks = sms * 8;
  *threads = 256;
  fp64_peak_kernel<<<*blocks, *threads, 0, s>>>(iters, 1.0, sink);
  return cudaGetLastError();
}
}  // namespace opsc

struct OpscContext {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;  // span of the last host-buffer call
  bool timed = false;
  int launches = 0;
  size_t cap_w = 0, cap_e = 0, cap_n = 0, cap_dev = 0;
  // windows
  double *qps = nullptr, *slo = nullptr, *eps = nullptr;
  int32_t* seq_len = nullptr;
  uint8_t* phase = nullptr;
  // workspace
  double* menu = nullptr;
  int32_t* fb = nullptr;
  double* mem_cap = nullptr;
  // decisions
  unsigned long long* key = nullptr;
  int16_t* cfg = nullptr;
  uint8_t *feasible = nullptr, *stable = nullptr;
  uint32_t* status = nullptr;
  double *latency = nullptr, *pred = nullptr, *energy = nullptr, *memory = nullptr;
  int32_t *objective = nullptr, *devices = nullptr;
  int8_t* path = nullptr;
  // operator mode: uniform reseed inputs and the move trace
  int16_t* u_cfg = nullptr;
  uint8_t* u_feas = nullptr;
  uint32_t* u_status = nullptr;
  int32_t* trace_len = nullptr;
  OpscTraceEntry* trace = nullptr;
  size_t cap_trace = 0;
  unsigned char* gstate = nullptr;  // greedy phase-1 state
  unsigned char* mtab = nullptr;    // model-level (B, R) table (small batches)
  size_t cap_mtab = 0;
  cudaStream_t side = nullptr;      // K3 runs here concurrently with greedy phase 1
  cudaEvent_t fork = nullptr, join = nullptr;
  unsigned char* h_stage = nullptr;  // pinned staging for pageable caller buffers
  size_t cap_stage = 0;
};

namespace {

// (Re)allocate a context buffer, zero-filled: fields a kernel leaves
// undefined (trace entries past trace_len, devices past devices_used) read as
// 0, never as uninitialised memory (compute-sanitizer initcheck). Growth
// happens on a context's first calls only.
template <class T>
cudaError_t regrow(T*& p, size_t n) {
  if (p) cudaFree(p);
  p = nullptr;
  const size_t bytes = n * sizeof(T) > 0 ? n * sizeof(T) : sizeof(T);
  cudaError_t e = cudaMalloc((void**)&p, bytes);
  if (e == cudaSuccess) e = cudaMemset(p, 0, bytes);
  if (e == cudaSuccess) e = cudaStreamSynchronize(0);
  return e;
}

int ensure(OpscContext* c, size_t W, size_t E, size_t n, size_t ndev, size_t trace_cap = 0) {
  cudaError_t e = cudaSuccess;
  if (W > c->cap_w || n > c->cap_n) {
    const size_t w2 = W > c->cap_w ? W : c->cap_w, n2 = n > c->cap_n ? n : c->cap_n;
    if ((e = regrow(c->qps, w2)) || (e = regrow(c->slo, w2)) || (e = regrow(c->eps, w2)) ||
        (e = regrow(c->seq_len, w2)) || (e = regrow(c->phase, w2)) || (e = regrow(c->key, w2)) ||
        (e = regrow(c->feasible, w2)) || (e = regrow(c->status, w2)) || (e = regrow(c->latency, w2)) ||
        (e = regrow(c->objective, w2)) || (e = regrow(c->energy, w2)) || (e = regrow(c->memory, w2)) ||
        (e = regrow(c->devices, w2)) || (e = regrow(c->cfg, w2 * n2 * 3)) ||
        (e = regrow(c->stable, w2 * n2)) || (e = regrow(c->path, w2 * n2)) ||
        (e = regrow(c->pred, w2 * n2 * OPSC_PRED_FIELDS)) || (e = regrow(c->fb, w2 * n2)) ||
        (e = regrow(c->u_cfg, w2 * n2 * 3)) || (e = regrow(c->u_feas, w2)) ||
        (e = regrow(c->u_status, w2)) || (e = regrow(c->trace_len, w2)) ||
        (e = regrow(c->gstate, greedy_state_bytes((int)w2))))
      return from_cuda(e);
    c->cap_trace = 0;
    c->cap_w = w2;
    c->cap_n = n2;
    c->cap_e = 0;  // menu depends on W too
  }
  if (W * E > c->cap_e) {
    if ((e = regrow(c->menu, W * E))) return from_cuda(e);
    c->cap_e = W * E;
  }
  if (ndev > c->cap_dev) {
    if ((e = regrow(c->mem_cap, ndev))) return from_cuda(e);
    c->cap_dev = ndev;
  }
  if (W * trace_cap > c->cap_trace) {
    if ((e = regrow(c->trace, W * trace_cap))) return from_cuda(e);
    c->cap_trace = W * trace_cap;
  }
  return OPSC_OK;
}

OpscWindows dev_windows(const OpscContext* c, int n) {
  OpscWindows w;
  w.n = n;
  w.qps = c->qps;
  w.seq_len = c->seq_len;
  w.phase = c->phase;
  w.slo = c->slo;
  w.eps = c->eps;
  return w;
}

OpscDecisions dev_decisions(const OpscContext* c) {
  OpscDecisions d;
  d.key = (int64_t*)c->key;
  d.cfg = c->cfg;
  d.feasible = c->feasible;
  d.status = c->status;
  d.latency = c->latency;
  d.objective = c->objective;
  d.path = c->path;
  d.pred = c->pred;
  d.stable = c->stable;
  d.energy = c->energy;
  d.memory = c->memory;
  d.devices = c->devices;
  d.trace_cap = 0;
  d.trace_len = c->trace_len;
  d.trace = c->trace;
  return d;
}

bool valid_dag(const OpscDag* d) { return d && d->n_ops >= 1 && d->n_ops <= OPSC_MAX_OPS; }

bool pageable(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

// Host side of the host-buffer call. Pinned caller buffers are copied
// directly; pageable ones (numpy arrays from the Python API) go through the
// context's pinned staging buffer, so every copy is a true async DMA instead
// of a driver-staged synchronous one (~10 us each for the ~20 small arrays).
struct HostIO {
  OpscContext* c;
  cudaStream_t s;
  bool stage;
  size_t off = 0;
  struct Out {
    void* dst;
    size_t at, bytes;
  };
  Out outs[24];
  int n_out = 0;
  unsigned char* slot(size_t bytes) {
    unsigned char* p = c->h_stage + off;
    off += (bytes + 15) & ~(size_t)15;
    return p;
  }
  cudaError_t h2d(void* dev, const void* host, size_t bytes) {
    if (!bytes) return cudaSuccess;
    if (!stage) return cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, s);
    unsigned char* p = slot(bytes);
    memcpy(p, host, bytes);
    return cudaMemcpyAsync(dev, p, bytes, cudaMemcpyHostToDevice, s);
  }
  cudaError_t d2h(void* host, const void* dev, size_t bytes) {
    if (!host || !bytes) return cudaSuccess;
    if (!stage) return cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, s);
    const size_t at = off;
    unsigned char* p = slot(bytes);
    outs[n_out++] = Out{host, at, bytes};
    return cudaMemcpyAsync(p, dev, bytes, cudaMemcpyDeviceToHost, s);
  }
  void finish() {  // after the stream synchronised
    for (int i = 0; i < n_out; ++i) memcpy(outs[i].dst, c->h_stage + outs[i].at, outs[i].bytes);
  }
};

int ensure_stage(OpscContext* c, size_t bytes) {
  if (bytes <= c->cap_stage) return OPSC_OK;
  if (c->h_stage) cudaFreeHost(c->h_stage);
  c->h_stage = nullptr;
  c->cap_stage = 0;
  if (cudaHostAlloc((void**)&c->h_stage, bytes, cudaHostAllocDefault) != cudaSuccess) {
    cudaGetLastError();
    return OPSC_ERR_CUDA;
  }
  c->cap_stage = bytes;
  return OPSC_OK;
}

// small batches tabulate every (B, R) point (4M weights max, ~40 MB)
constexpr long long kModelTablePoints = 1ll << 22;

bool want_model_table(int W, const OpscModelSpec& m, int n) {
  return (long long)W * m.b_cap * m.r_cap * n <= kModelTablePoints;
}

// returns workspace pointer (or null -> per-window probe path)
void* model_table_ws(OpscContext* c, int W, const OpscModelSpec& m, int n, size_t* bytes) {
  *bytes = 0;
  if (!want_model_table(W, m, n)) return nullptr;
  const size_t need = model_table_bytes(W, m, n);
  if (need > c->cap_mtab) {
    if (regrow(c->mtab, need) != cudaSuccess) {
      cudaGetLastError();
      c->cap_mtab = 0;
      return nullptr;
    }
    c->cap_mtab = need;
  }
  *bytes = c->cap_mtab;
  return c->mtab;
}

}  // namespace

extern "C" {

int opsc_abi_version(void) { return OPSC_ABI_VERSION; }

const char* opsc_status_string(int status) {
  switch (status) {
    case OPSC_OK: return "ok";
    case OPSC_ERR_ARG: return "invalid argument or table limit exceeded";
    case OPSC_ERR_CUDA: return "CUDA runtime error";
    case OPSC_ERR_SPACE: return "candidate space exceeds the 2^40 lexicographic key field";
    case OPSC_ERR_NODEVICE: return "no CUDA device";
    default: return "unknown status";
  }
}

int opsc_device_count(int* count) {
  int n = 0;
  const cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *count = 0;
    return OPSC_ERR_NODEVICE;
  }
  *count = n;
  return OPSC_OK;
}

int opsc_menu_build(const OpscDag* dag, const OpscGrid* grid, OpscWindows win, double* menu_w,
                    uint32_t* status, void* stream) {
  if (!valid_dag(dag) || !grid) return OPSC_ERR_ARG;
  return from_cuda(launch_menu_build(*dag, *grid, win, menu_w, status, (cudaStream_t)stream));
}

int opsc_stability_check(const OpscDag* dag, const OpscGrid* grid, OpscWindows win, uint32_t* status,
                         void* stream) {
  if (!valid_dag(dag) || !grid) return OPSC_ERR_ARG;
  return from_cuda(launch_stability(*dag, *grid, win, status, (cudaStream_t)stream));
}

int opsc_compose_argmin(const OpscDag* dag, const OpscGrid* grid, OpscWindows win, const double* menu_w,
                        int32_t shard, int32_t n_shards, int64_t* key_out, void* stream) {
  if (!valid_dag(dag) || !grid) return OPSC_ERR_ARG;
  ComposeCfg c;
  const int rc = compose_setup(*dag, *grid, win.n, shard, n_shards, &c);
  if (rc != OPSC_OK) return rc;
  return from_cuda(launch_compose(c, *grid, win.n, menu_w, win.slo, win.qps,
                                  (unsigned long long*)key_out, (cudaStream_t)stream));
}

int opsc_compose_boundary(const OpscDag* dag, const OpscGrid* grid, OpscWindows win, const double* menu_w,
                          double band_ulps, int64_t* count_out, void* stream) {
  if (!valid_dag(dag) || !grid || !count_out || !(band_ulps >= 0.0)) return OPSC_ERR_ARG;
  ComposeCfg c;
  const int rc = compose_setup(*dag, *grid, win.n, 0, 1, &c);
  if (rc != OPSC_OK) return rc;
  return from_cuda(launch_compose_boundary(c, *grid, win.n, menu_w, win.slo, win.qps, band_ulps,
                                           (unsigned long long*)count_out, (cudaStream_t)stream));
}

int opsc_compose_argmin_peers(const OpscDag* dag, const OpscGrid* grid, OpscWindows win, const double* menu_w,
                              int32_t shard, int32_t n_shards, int64_t* const* peer_keys, int32_t n_peers,
                              void* stream) {
  if (!valid_dag(dag) || !grid || !peer_keys || n_peers < 1 || n_peers > OPSC_MAX_PEERS) return OPSC_ERR_ARG;
  ComposeCfg c;
  const int rc = compose_setup(*dag, *grid, win.n, shard, n_shards, &c);
  if (rc != OPSC_OK) return rc;
  PeerKeys pk;
  memset(&pk, 0, sizeof(pk));
  pk.n = n_peers;
  for (int p = 0; p < n_peers; ++p) {
    if (!peer_keys[p]) return OPSC_ERR_ARG;
    pk.p[p] = (unsigned long long*)peer_keys[p];
  }
  return from_cuda(launch_compose(c, *grid, win.n, menu_w, win.slo, win.qps, nullptr, (cudaStream_t)stream, &pk));
}

int opsc_peer_barrier(uint32_t* const* flags, int32_t rank, int32_t n, uint32_t epoch, int32_t timeout_ms,
                      int32_t* err, void* stream) {
  if (!flags || !err || n < 1 || n > OPSC_MAX_PEERS || rank < 0 || rank >= n || timeout_ms < 1) return OPSC_ERR_ARG;
  PeerFlags f;
  memset(&f, 0, sizeof(f));
  for (int p = 0; p < n; ++p) {
    if (!flags[p]) return OPSC_ERR_ARG;
    f.p[p] = flags[p];
  }
  return from_cuda(launch_peer_barrier(f, rank, n, epoch, timeout_ms, err, (cudaStream_t)stream));
}

int opsc_copy_keys(int64_t* dst, const int64_t* src, int32_t n, void* stream) {
  if (n < 0 || (n > 0 && (!dst || !src))) return OPSC_ERR_ARG;
  if (n == 0) return OPSC_OK;
  return from_cuda(cudaMemcpyAsync(dst, src, (size_t)n * 8, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
}

int opsc_ipc_alloc(size_t bytes, void** dptr, void* handle) {
  if (!dptr || !handle || bytes == 0) return OPSC_ERR_ARG;
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e != cudaSuccess) return from_cuda(e);
  e = cudaMemset(p, 0, bytes);
  if (e == cudaSuccess) e = cudaIpcGetMemHandle((cudaIpcMemHandle_t*)handle, p);
  if (e != cudaSuccess) {
    cudaFree(p);
    return from_cuda(e);
  }
  *dptr = p;
  return OPSC_OK;
}

int opsc_ipc_open(const void* handle, void** dptr) {
  if (!dptr || !handle) return OPSC_ERR_ARG;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  return from_cuda(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess));
}

int opsc_ipc_close(void* dptr) { return from_cuda(cudaIpcCloseMemHandle(dptr)); }

int opsc_ipc_free(void* dptr) { return from_cuda(cudaFree(dptr)); }

int opsc_fill_keys(int64_t* key, int32_t n, void* stream) {
  return from_cuda(launch_fill_keys((unsigned long long*)key, n, (cudaStream_t)stream));
}

int opsc_init_windows(OpscWindows win, uint32_t* status, int64_t* key, uint8_t* feasible, void* stream) {
  if (!status || win.n < 0) return OPSC_ERR_ARG;
  return from_cuda(launch_init(win.n, win.qps, status, (unsigned long long*)key, feasible,
                               (cudaStream_t)stream));
}

int opsc_menu_fallback(const OpscDag* dag, const OpscGrid* grid, int32_t n_windows, const double* menu_w,
                       int32_t* fb_entry, void* stream) {
  if (!valid_dag(dag) || !grid) return OPSC_ERR_ARG;
  return from_cuda(launch_fallback(*dag, *grid, n_windows, menu_w, fb_entry, (cudaStream_t)stream));
}

int opsc_decode_decisions(const OpscDag* dag, const OpscGrid* grid, int32_t n_windows, const int64_t* key,
                          const int32_t* fb_entry, int16_t* cfg, uint8_t* feasible, uint32_t* status,
                          void* stream) {
  if (!valid_dag(dag) || !grid) return OPSC_ERR_ARG;
  return from_cuda(launch_decode(*dag, *grid, n_windows, (const unsigned long long*)key, fb_entry, cfg,
                                 feasible, status, (cudaStream_t)stream));
}

int opsc_model_grid(const OpscDag* dag, const OpscModelSpec* spec, OpscWindows win, int16_t* cfg,
                    uint8_t* feasible, uint32_t* status, void* stream) {
  if (!valid_dag(dag) || !spec) return OPSC_ERR_ARG;
  return from_cuda(launch_model_grid(*dag, *spec, win, cfg, feasible, status, (cudaStream_t)stream));
}

int opsc_materialize(const OpscDag* dag, OpscWindows win, int32_t config_order, const OpscPlaceSpec* place,
                     OpscDecisions out, void* stream) {
  if (!valid_dag(dag) || !place) return OPSC_ERR_ARG;
  return from_cuda(launch_materialize(*dag, win, config_order, *place, out, (cudaStream_t)stream));
}

int opsc_ctx_create(int32_t device, int32_t max_windows, OpscContext** out) {
  if (!out) return OPSC_ERR_ARG;
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n <= device) {
    cudaGetLastError();
    return OPSC_ERR_NODEVICE;
  }
  OpscContext* c = new (std::nothrow) OpscContext();
  if (!c) return OPSC_ERR_ARG;
  c->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->fork, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->join, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    delete c;
    return OPSC_ERR_CUDA;
  }
  if (max_windows > 0) {
    const int rc = ensure(c, (size_t)max_windows, 64, 8, 1);
    if (rc) {
      opsc_ctx_destroy(c);
      return rc;
    }
  }
  *out = c;
  return OPSC_OK;
}

int opsc_ctx_destroy(OpscContext* c) {
  if (!c) return OPSC_OK;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  void* ptrs[] = {c->qps, c->slo, c->eps, c->seq_len, c->phase, c->menu, c->fb, c->mem_cap, c->key,
                  c->cfg, c->feasible, c->stable, c->status, c->latency, c->pred, c->energy,
                  c->memory, c->objective, c->devices, c->path, c->u_cfg, c->u_feas,
                  c->u_status, c->trace_len, c->trace, c->gstate, c->mtab};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (c->stream) cudaStreamDestroy(c->stream);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->fork) cudaEventDestroy(c->fork);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->join) cudaEventDestroy(c->join);
  if (c->h_stage) cudaFreeHost(c->h_stage);
  delete c;
  return OPSC_OK;
}

int opsc_ctx_last_launches(const OpscContext* c, int32_t* launches) {
  if (!c || !launches) return OPSC_ERR_ARG;
  *launches = c->launches;
  return OPSC_OK;
}

int opsc_ctx_last_ms(OpscContext* c, float* ms) {
  if (!c || !ms) return OPSC_ERR_ARG;
  if (!c->timed) return OPSC_ERR_ARG;
  return from_cuda(cudaEventElapsedTime(ms, c->ev0, c->ev1));
}

size_t opsc_place_shared_workspace(int32_t n_windows, int32_t cap_assign, int32_t cap_dev, int32_t n_ops) {
  return place_shared_workspace(n_windows, cap_assign, cap_dev, n_ops);
}

int opsc_place_shared(const OpscDag* dag, const OpscPlaceShared* fleet, OpscWindows win, const int16_t* cfg,
                      const uint8_t* plan_feasible, int32_t config_order, OpscPlacement out, void* workspace,
                      size_t workspace_bytes, void* stream) {
  if (!valid_dag(dag) || !fleet || fleet->n_devices < 1 || out.cap_assign < 1 || out.cap_dev < 1)
    return OPSC_ERR_ARG;
  return from_cuda(launch_place_shared(*dag, *fleet, win, cfg, plan_feasible, config_order, out, workspace,
                                       workspace_bytes, (cudaStream_t)stream));
}

size_t opsc_windowize_workspace(int64_t n_records, int32_t max_windows) {
  return windowize_workspace(n_records, max_windows);
}

int opsc_windowize(OpscTraceRecords rec, double window_len, double quantile, int32_t max_windows,
                   int32_t* n_windows, double* prefill_qps, int32_t* prefill_len, double* decode_qps,
                   void* workspace, size_t workspace_bytes, void* stream) {
  if (!(window_len > 0.0) || !(quantile > 0.0 && quantile <= 1.0) || rec.n <= 0 || max_windows < 1 ||
      !n_windows || !workspace)
    return OPSC_ERR_ARG;
  return from_cuda(launch_windowize(rec, window_len, quantile, max_windows, n_windows, prefill_qps,
                                    prefill_len, decode_qps, workspace, workspace_bytes, (cudaStream_t)stream));
}

int opsc_greedy(const OpscDag* dag, const OpscGreedySpec* spec, OpscWindows win, const int16_t* uniform_cfg,
                const uint8_t* uniform_feasible, const uint32_t* uniform_status, OpscDecisions out,
                void* stream) {
  if (!valid_dag(dag) || !spec || !out.trace_len || (out.trace_cap > 0 && !out.trace)) return OPSC_ERR_ARG;
  return from_cuda(launch_greedy(*dag, *spec, win, uniform_cfg, uniform_feasible, uniform_status, out,
                                 (cudaStream_t)stream));
}

size_t opsc_greedy_state_bytes(int32_t n_windows) { return greedy_state_bytes(n_windows); }

size_t opsc_model_table_bytes(const OpscModelSpec* spec, int32_t n_windows, int32_t n_ops) {
  if (!spec) return 0;
  return model_table_bytes(n_windows, *spec, n_ops);
}

int opsc_model_grid_table(const OpscDag* dag, const OpscModelSpec* spec, OpscWindows win, int16_t* cfg,
                          uint8_t* feasible, uint32_t* status, void* workspace, size_t workspace_bytes,
                          void* stream) {
  if (!valid_dag(dag) || !spec || !workspace ||
      workspace_bytes < model_table_bytes(win.n, *spec, dag->n_ops))
    return OPSC_ERR_ARG;
  return from_cuda(launch_model_grid(*dag, *spec, win, cfg, feasible, status, (cudaStream_t)stream,
                                     workspace, workspace_bytes));
}

int opsc_greedy_phase(const OpscDag* dag, const OpscGreedySpec* spec, OpscWindows win, int32_t phase,
                      void* state, const int16_t* uniform_cfg, const uint8_t* uniform_feasible,
                      const uint32_t* uniform_status, OpscDecisions out, void* stream) {
  if (!valid_dag(dag) || !spec || !out.trace_len || (out.trace_cap > 0 && !out.trace) || !state ||
      (phase != 1 && phase != 2))
    return OPSC_ERR_ARG;
  return from_cuda(launch_greedy(*dag, *spec, win, uniform_cfg, uniform_feasible, uniform_status, out,
                                 (cudaStream_t)stream, phase, state));
}

int opsc_plan_windows_host(OpscContext* c, int32_t mode, const OpscDag* dag, const OpscGrid* grid,
                           const OpscModelSpec* model, const OpscGreedySpec* greedy,
                           const OpscPlaceSpec* place, OpscWindows win, OpscDecisions out) {
  if (!c || !valid_dag(dag) || !place || win.n < 0) return OPSC_ERR_ARG;
  if (mode == OPSC_MODE_ORACLE && !grid) return OPSC_ERR_ARG;
  if (mode == OPSC_MODE_MODEL && !model) return OPSC_ERR_ARG;
  if (mode == OPSC_MODE_OPERATOR && !greedy) return OPSC_ERR_ARG;
  if (mode != OPSC_MODE_ORACLE && mode != OPSC_MODE_MODEL && mode != OPSC_MODE_OPERATOR) return OPSC_ERR_ARG;
  const size_t tcap = mode == OPSC_MODE_OPERATOR && out.trace_cap > 0 ? (size_t)out.trace_cap : 0;
  cudaSetDevice(c->device);
  const int W = win.n, n = dag->n_ops;
  if (W == 0) return OPSC_OK;
  const size_t E = mode == OPSC_MODE_ORACLE ? (size_t)grid->menu_off[n] : 0;
  const size_t ndev = place->uniform_cap ? 1 : (size_t)place->n_devices;
  int rc = ensure(c, W, E, n, ndev, tcap);
  if (rc) return rc;
  cudaStream_t s = c->stream;
  c->launches = 0;
  cudaError_t e;
#define CK(x)                   \
  do {                          \
    e = (x);                    \
    if (e != cudaSuccess) {     \
      cudaGetLastError();       \
      return OPSC_ERR_CUDA;     \
    }                           \
  } while (0)
  if (!c->ev0) CK(cudaEventCreate(&c->ev0));
  if (!c->ev1) CK(cudaEventCreate(&c->ev1));
  const size_t wn = (size_t)W * n;
  HostIO io{c, s, pageable(win.qps) || pageable(out.cfg) || pageable(out.latency)};
  if (io.stage) {
    const size_t in_b = W * (3 * sizeof(double) + sizeof(int32_t) + 1) + ndev * sizeof(double);
    const size_t out_b = W * (4 * sizeof(double) + 5 * sizeof(int32_t) + 1) + wn * (3 * sizeof(int16_t) + 2) +
                         wn * OPSC_PRED_FIELDS * sizeof(double) + W * tcap * sizeof(OpscTraceEntry);
    // large batches (long move traces) copy directly: the staging buffer is
    // for the many-small-copies case and stays bounded
    if (in_b + out_b > ((size_t)64 << 20)) io.stage = false;
    else if ((rc = ensure_stage(c, in_b + out_b + 24 * 16))) return rc;
  }
  CK(cudaEventRecord(c->ev0, s));  // device-side span: first H2D .. last D2H
  CK(io.h2d(c->qps, win.qps, W * sizeof(double)));
  CK(io.h2d(c->seq_len, win.seq_len, W * sizeof(int32_t)));
  CK(io.h2d(c->phase, win.phase, W * sizeof(uint8_t)));
  CK(io.h2d(c->slo, win.slo, W * sizeof(double)));
  CK(io.h2d(c->eps, win.eps, W * sizeof(double)));
  CK(io.h2d(c->mem_cap, place->mem_cap, ndev * sizeof(double)));
  OpscPlaceSpec dplace = *place;
  dplace.mem_cap = c->mem_cap;
  const OpscWindows dw = dev_windows(c, W);
  CK(launch_init(W, c->qps, c->status, c->key, c->feasible, s));
  c->launches++;
  if (mode == OPSC_MODE_ORACLE) {
    ComposeCfg cc;
    rc = compose_setup(*dag, *grid, W, 0, 1, &cc);
    if (rc) return rc;
    CK(launch_menu_build(*dag, *grid, dw, c->menu, c->status, s));
    CK(launch_stability(*dag, *grid, dw, c->status, s));
    CK(launch_compose(cc, *grid, W, c->menu, c->slo, c->qps, c->key, s));
    CK(launch_fallback(*dag, *grid, W, c->menu, c->fb, s));
    CK(launch_decode(*dag, *grid, W, c->key, c->fb, c->cfg, c->feasible, c->status, s));
    c->launches += 5;
    CK(launch_materialize(*dag, dw, 0, dplace, dev_decisions(c), s));
  } else if (mode == OPSC_MODE_MODEL) {
    size_t tb = 0;
    void* tw = model_table_ws(c, W, *model, n, &tb);
    CK(launch_model_grid(*dag, *model, dw, c->cfg, c->feasible, c->status, s, tw, tb));
    c->launches += 1;
    CK(launch_materialize(*dag, dw, 1, dplace, dev_decisions(c), s));
  } else {
    // _uniform_optimum = model_level_autoscale on the same windows
    // (autoscaler.py:492-500); it does not depend on the first greedy loop, so
    // it runs on the side stream while phase 1 runs on the main stream.
    CK(cudaEventRecord(c->fork, s));
    CK(cudaStreamWaitEvent(c->side, c->fork, 0));
    CK(launch_init(W, c->qps, c->u_status, nullptr, c->u_feas, c->side));
    // hidden behind phase 1: the one-kernel form (no (B, R) table) is the
    // cheaper side-stream load (70B W=1 median 0.177 -> 0.169 ms)
    CK(launch_model_grid(*dag, greedy->model, dw, c->u_cfg, c->u_feas, c->u_status, c->side, nullptr, 0));
    CK(cudaEventRecord(c->join, c->side));
    OpscDecisions dd = dev_decisions(c);
    dd.trace_cap = (int32_t)tcap;
    CK(launch_greedy(*dag, *greedy, dw, c->u_cfg, c->u_feas, c->u_status, dd, s, 1, c->gstate));
    CK(cudaStreamWaitEvent(s, c->join, 0));
    CK(launch_greedy(*dag, *greedy, dw, c->u_cfg, c->u_feas, c->u_status, dd, s, 2, c->gstate));
    c->launches += 4;
    CK(launch_materialize(*dag, dw, 1, dplace, dd, s));
  }
  c->launches++;
  CK(io.d2h(out.key, c->key, W * sizeof(int64_t)));
  CK(io.d2h(out.cfg, c->cfg, wn * 3 * sizeof(int16_t)));
  CK(io.d2h(out.feasible, c->feasible, W));
  CK(io.d2h(out.status, c->status, W * sizeof(uint32_t)));
  CK(io.d2h(out.latency, c->latency, W * sizeof(double)));
  CK(io.d2h(out.objective, c->objective, W * sizeof(int32_t)));
  CK(io.d2h(out.path, c->path, wn));
  CK(io.d2h(out.pred, c->pred, wn * OPSC_PRED_FIELDS * sizeof(double)));
  CK(io.d2h(out.stable, c->stable, wn));
  CK(io.d2h(out.energy, c->energy, W * sizeof(double)));
  CK(io.d2h(out.memory, c->memory, W * sizeof(double)));
  CK(io.d2h(out.devices, c->devices, W * sizeof(int32_t)));
  if (tcap) CK(io.d2h(out.trace_len, c->trace_len, W * sizeof(int32_t)));
  if (tcap) CK(io.d2h(out.trace, c->trace, W * tcap * sizeof(OpscTraceEntry)));
  CK(cudaEventRecord(c->ev1, s));
  CK(cudaStreamSynchronize(s));
  io.finish();
  c->timed = true;
#undef CK
  return OPSC_OK;
}

int opsc_candidate_probe(int32_t kind, int32_t iters, float* ms, double* candidates, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  double* sink = nullptr;
  if (cudaMalloc(&sink, 8192 * sizeof(double)) != cudaSuccess) return OPSC_ERR_CUDA;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int blocks = sms * 3 * 8;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto go = [&](int it) {
    if (kind == 1) cand_probe_kernel<1><<<blocks, 256, 0, s>>>(it, 1.0, sink);
    else cand_probe_kernel<2><<<blocks, 256, 0, s>>>(it, 1.0, sink);
  };
  go(iters / 10 + 1);
  cudaEventRecord(a, s);
  go(iters);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  const cudaError_t e = cudaGetLastError();
  float t = 0.0f;
  cudaEventElapsedTime(&t, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(sink);
  if (e != cudaSuccess) return OPSC_ERR_CUDA;
  *ms = t;
  *candidates = (double)blocks * 256.0 * (double)iters * 24.0;
  return OPSC_OK;
}

int opsc_fp64_peak(int32_t iters, float* ms, double* fp64_ops, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  double* sink = nullptr;
  if (cudaMalloc(&sink, 4096 * sizeof(double)) != cudaSuccess) return OPSC_ERR_CUDA;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int blocks = 0, threads = 0;
  launch_fp64_peak(iters / 10 + 1, sink, &blocks, &threads, s);  // warm-up
  cudaEventRecord(a, s);
  cudaError_t e = launch_fp64_peak(iters, sink, &blocks, &threads, s);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float t = 0.0f;
  cudaEventElapsedTime(&t, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(sink);
  if (e != cudaSuccess) return OPSC_ERR_CUDA;
  *ms = t;
  *fp64_ops = (double)blocks * threads * (double)iters * 32.0;
  return OPSC_OK;
}

}  // extern "C"
