// Microbenchmark: latency / throughput of FP64 ops on this GPU (diagnostic only).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat_dfma(double *out, long long *cyc, int n) {
  double a = out[0], b = out[1], c = out[2];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = fma(a, b, c);
  long long t1 = clock64();
  out[3] = a; cyc[0] = t1 - t0;
}
__global__ void lat_rsqrt(double *out, long long *cyc, int n) {
  double a = out[0] + 2.0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = rsqrt(a) + 1.5;
  long long t1 = clock64();
  out[4] = a; cyc[1] = t1 - t0;
}
__global__ void lat_div(double *out, long long *cyc, int n) {
  double a = out[0] + 2.0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = 3.0 / a + 1.0;
  long long t1 = clock64();
  out[5] = a; cyc[2] = t1 - t0;
}
__global__ void lat_lds(double *out, long long *cyc, int n) {
  __shared__ double s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (double)((i * 7 + 1) % 1024);
  __syncthreads();
  int idx = 0; double acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { double v = s[idx]; idx = (int)v; acc += v; }
  long long t1 = clock64();
  out[6] = acc; cyc[3] = t1 - t0;
}
__global__ void tput_dfma(double *out, long long *cyc, int n) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 1.0000001, c = 1e-9;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
    a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[4] = t1 - t0;
  out[8 + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void bar_lat(long long *cyc, int n) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[5] = t1 - t0;
}
int main() {
  double *d; long long *c; cudaMalloc(&d, 8192 * 8); cudaMalloc(&c, 64 * 8);
  double h[3] = {1.0, 0.999999, 1e-7}; cudaMemcpy(d, h, 24, cudaMemcpyHostToDevice);
  const int n = 4096;
  lat_dfma<<<1, 1>>>(d, c, n); lat_rsqrt<<<1, 1>>>(d, c, n); lat_div<<<1, 1>>>(d, c, n); lat_lds<<<1, 32>>>(d, c, n);
  tput_dfma<<<1, 1024>>>(d, c, n); bar_lat<<<1, 512>>>(c, n);
  cudaDeviceSynchronize();
  long long hc[8]; cudaMemcpy(hc, c, 64, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.1f cyc\n", (double)hc[0] / n);
  printf("rsqrt(double)+add dependent latency: %.1f cyc\n", (double)hc[1] / n);
  printf("double div+add dependent latency: %.1f cyc\n", (double)hc[2] / n);
  printf("LDS.64 pointer-chase latency: %.1f cyc\n", (double)hc[3] / n);
  printf("DFMA throughput (1024 thr, 8 indep chains): %.1f DFMA/cyc/SM\n", 1024.0 * 8 * n / hc[4]);
  printf("__syncthreads (512 thr) cost: %.1f cyc\n", (double)hc[5] / n);
  for (int thr : {32, 64, 128, 256, 512}) {
    tput_dfma<<<1, thr>>>(d, c, n);
    cudaDeviceSynchronize();
    cudaMemcpy(hc, c, 64, cudaMemcpyDeviceToHost);
    printf("DFMA throughput %4d threads: %.2f DFMA/cyc/SM  (%.2f cyc per warp-instr per warp)\n", thr,
           (double)thr * 8 * n / hc[4], (double)hc[4] / (8.0 * n));
  }
  return 0;
}
