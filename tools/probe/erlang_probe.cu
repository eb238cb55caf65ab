// Dev probe: cycles per Erlang-B recurrence step vs rho (one warp, clock64).
#include <cstdio>
__global__ void k(const double* rhos, int n, int r, long long* cyc, double* out) {
  int i = threadIdx.x;
  if (i >= n) return;
  double rho = rhos[i];
  long long t0 = clock64();
  const double a = (double)r * rho;
  double b = 1.0;
  int steps_zero = -1;
  for (int k = 1; k <= r; ++k) {
    const double ab = a * b;
    b = ab / ((double)k + ab);
    if (b == 0.0 && steps_zero < 0) steps_zero = k;
  }
  long long t1 = clock64();
  cyc[i] = t1 - t0;
  out[i] = b + steps_zero;
}
int main() {
  const int n = 8;
  double h[n] = {0.9, 0.5, 0.2, 0.1, 0.05, 0.02, 0.01, 0.001};
  double *d, *o; long long* c;
  cudaMalloc(&d, n * 8); cudaMalloc(&o, n * 8); cudaMalloc(&c, n * 8);
  cudaMemcpy(d, h, n * 8, cudaMemcpyHostToDevice);
  for (int r : {32, 128, 512}) {
    for (int rep = 0; rep < 2; ++rep) {
      // one thread at a time, so the numbers are pure latency per chain
      for (int j = 0; j < n; ++j) {
        k<<<1, 1>>>(d + j, 1, r, c + j, o + j);
      }
      cudaDeviceSynchronize();
    }
    long long hc[n]; double ho[n];
    cudaMemcpy(hc, c, n * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(ho, o, n * 8, cudaMemcpyDeviceToHost);
    for (int j = 0; j < n; ++j) printf("R=%d rho=%.3f cycles=%lld per_step=%.1f zero_at=%.0f\n", r, h[j], hc[j], (double)hc[j] / r, ho[j]);
  }
  return 0;
}
