// Latency of the 8x8 in-register pivot-block sweep (warp_sweep8 of kernels_chain.cu) and of its
// building blocks on sm_100a (diagnostic only).
#include "../../paper_2307_00719_b200/csrc/kernels_chain.cu"
#include <cstdio>
namespace strb200 {
void prepare_f64_attrs() {}
void launch_fit_reduce(const double2 *, int64_t, double *, cudaStream_t) {}
}  // namespace strb200
using namespace strb200;

__global__ void k_sweep_lat(double *out, long long *cyc, int iters) {
  const int lane = threadIdx.x, g = lane >> 2, tg = lane & 3;
  double d[2];
  for (int e = 0; e < 2; ++e) {
    const int j = 2 * tg + e;
    d[e] = (g == j) ? 4.0 : 0.1 / (1 + g + j);
  }
  __syncwarp();
  long long t0 = clock64();
  bool bad = false;
  for (int i = 0; i < iters; ++i) {
    bad |= warp_sweep8(d, g, tg);
    d[0] = -d[0]; d[1] = -d[1];
  }
  long long t1 = clock64();
  out[lane] = d[0] + d[1] + bad;
  if (lane == 0) cyc[0] = (t1 - t0) / iters;
}

__global__ void k_ops_lat(double *out, long long *cyc, int iters) {
  double x = 1.0 + threadIdx.x * 1e-3, y = 0.5;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, y, 0.25);
  long long t1 = clock64();
  for (int i = 0; i < iters; ++i) x = rcp_nr(x) + 0.5;
  long long t2 = clock64();
  for (int i = 0; i < iters; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) * 0.999 + 0.001;
  long long t3 = clock64();
  float xf = (float)x;
  for (int i = 0; i < iters; ++i) xf = __frcp_rn(xf) + 0.5f;
  long long t4 = clock64();
  for (int i = 0; i < iters; ++i) { double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r + 0.5; }
  long long t5 = clock64();
  out[threadIdx.x] = x + xf;
  if (threadIdx.x == 0) {
    cyc[1] = (t1 - t0) / iters;
    cyc[2] = (t2 - t1) / iters;
    cyc[3] = (t3 - t2) / iters;
    cyc[4] = (t4 - t3) / iters;
    cyc[5] = (t5 - t4) / iters;
  }
}

int main() {
  double *out;
  long long *cyc, h[8] = {0};
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaMalloc(&cyc, 8 * sizeof(long long));
  for (int r = 0; r < 2; ++r) {
    k_sweep_lat<<<1, 32>>>(out, cyc, 200);
    k_ops_lat<<<1, 32>>>(out, cyc, 1000);
    cudaDeviceSynchronize();
  }
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  printf("warp_sweep8 %lld cycles | dfma chain %lld | rcp_nr+add %lld | shfl+dfma %lld | frcp+fadd %lld | rcp.approx.f64+add %lld  (%s)\n",
         h[0], h[1], h[2], h[3], h[4], h[5], cudaGetErrorString(cudaGetLastError()));
  return 0;
}
