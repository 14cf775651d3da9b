// DMMA (mma.sync m8n8k4 f64) latency / throughput on this GPU (diagnostic only).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int CH>
__global__ void k_dmma(double *out, long long *cyc, int n) {
  double c[CH][2];
  for (int i = 0; i < CH; ++i) { c[i][0] = threadIdx.x; c[i][1] = 1.0; }
  double a = 1.0000001, b = 0.999999;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < CH; ++j) dmma(c[j][0], c[j][1], a, b);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  double s = 0;
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  out[threadIdx.x] = s;
}
int main() {
  double *d; long long *c; cudaMalloc(&d, 8192 * 8); cudaMalloc(&c, 64);
  const int n = 2048;
  long long hc;
  k_dmma<1><<<1, 32>>>(d, c, n); cudaDeviceSynchronize(); cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
  printf("DMMA dependent latency: %.1f cyc\n", (double)hc / n);
  for (int w : {1, 2, 4, 8, 16}) {
    k_dmma<8><<<1, 32 * w>>>(d, c, n); cudaDeviceSynchronize(); cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
    printf("DMMA %2d warps x 8 chains: %.1f FMA/cyc/SM (%.1f cyc per DMMA per warp)\n", w, (double)w * 8 * n * 256 / hc, (double)hc / (8.0 * n));
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
