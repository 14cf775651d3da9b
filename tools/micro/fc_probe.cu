// Phase timing of the SPD-inverse kernel (chain_factor.cu) for one S (diagnostic):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -DFC_PROBE -I../../include -I../../paper_2307_00719_b200/csrc \
//        -o fc_probe fc_probe.cu && ./fc_probe 100
#include "../../paper_2307_00719_b200/csrc/chain_factor.cu"
#include <cstdio>
#include <cstdlib>
#include <vector>
using namespace strb200;
__global__ void k_chol8_bench(int reps) {
  __shared__ __align__(16) double M[8 * 12];
  __shared__ __align__(16) double T[8 * 12];
  const int lane = threadIdx.x;
  for (int i = lane; i < 64; i += 32) M[(i / 8) * 12 + i % 8] = (i / 8 == i % 8) ? 4.0 : 0.1;
  __syncwarp();
  bool bad = false;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    chol8_inv8(M, 12, T, bad);
    __syncwarp();
    if (lane == 0) M[0] = 4.0 + T[0] * 1e-30;
    __syncwarp();
  }
  long long t1 = clock64();
  if (lane == 0) g_fc_probe[50] = (t1 - t0) / reps + (bad ? 1000000 : 0);
}
__global__ void k_lat(double seed, long long *out) {
  const int lane = threadIdx.x;
  double x = seed + lane * 1e-9, y = 1.0000001;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) { x = fma(x, y, 1e-12); x = fma(x, y, 1e-12); x = fma(x, y, 1e-12); x = fma(x, y, 1e-12); }
  t1 = clock64();
  if (lane == 0) out[0] = (t1 - t0);
  // DMUL chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) { x = x * y; x = x * y; x = x * y; x = x * y; }
  t1 = clock64();
  if (lane == 0) out[1] = (t1 - t0);
  // SHFL f64 chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) { x = __shfl_sync(0xffffffffu, x, (lane + 1) & 31); x = __shfl_sync(0xffffffffu, x, (lane + 3) & 31); x = __shfl_sync(0xffffffffu, x, (lane + 5) & 31); x = __shfl_sync(0xffffffffu, x, (lane + 7) & 31); }
  t1 = clock64();
  if (lane == 0) out[2] = (t1 - t0);
  // MUFU rsqrt f64 approx chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k) { double r; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r + 1.0; }
  }
  t1 = clock64();
  if (lane == 0) out[3] = (t1 - t0);
  // DMMA chain (accumulator dependence)
  double c0 = x, c1 = y;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) { dmma(c0, c1, x, y); dmma(c0, c1, x, y); dmma(c0, c1, x, y); dmma(c0, c1, x, y); }
  t1 = clock64();
  if (lane == 0) out[4] = (t1 - t0);
  // DMMA throughput: 8 independent accumulators
  double a[16];
  for (int k = 0; k < 16; ++k) a[k] = k;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 128; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) dmma(a[2 * k], a[2 * k + 1], x, y);
  }
  t1 = clock64();
  if (lane == 0) out[5] = (t1 - t0);
  float f = (float)x;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) { f = fmaf(f, 1.0001f, 1e-6f); f = fmaf(f, 1.0001f, 1e-6f); f = fmaf(f, 1.0001f, 1e-6f); f = fmaf(f, 1.0001f, 1e-6f); }
  t1 = clock64();
  if (lane == 0) out[6] = (t1 - t0);
  double s = 0;
  for (int k = 0; k < 16; ++k) s += a[k];
  if (lane == 0) out[7] = (long long)(x + c0 + c1 + s + f) & 1;
}

int main(int argc, char **argv) {
  {
    long long *d_out, h[8];
    cudaMalloc(&d_out, sizeof(h));
    k_lat<<<1, 32>>>(1.0, d_out);
    k_lat<<<1, 32>>>(1.0, d_out);
    cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
    printf("latency (cycles/op): DFMA %.1f DMUL %.1f SHFL.f64 %.1f RSQ64H+add %.1f DMMA-dep %.1f DMMA-8indep %.1f/op FFMA %.1f\n",
           h[0] / 1024.0, h[1] / 1024.0, h[2] / 1024.0, h[3] / 1024.0, h[4] / 1024.0, h[5] / 1024.0, h[6] / 1024.0);
  }
  const int S = argc > 1 ? atoi(argv[1]) : 100;
  std::vector<double> Q(S * S);
  srand(1);
  std::vector<double> A(2 * S * S);
  for (auto &v : A) v = (rand() / (double)RAND_MAX) - 0.5;
  for (int i = 0; i < S; ++i)
    for (int j = 0; j < S; ++j) {
      double s = 0;
      for (int k = 0; k < 2 * S; ++k) s += A[k * S + i] * A[k * S + j];
      Q[i * S + j] = s;
    }
  double *dQ, *dQi, *ws;
  int *info;
  cudaMalloc(&dQ, S * S * 8);
  cudaMalloc(&dQi, spd_factor_doubles(S) * 8);
  cudaMalloc(&ws, 8);
  cudaMalloc(&info, 4);
  cudaMemcpy(dQ, Q.data(), S * S * 8, cudaMemcpyHostToDevice);
  for (int it = 0; it < 5; ++it) launch_spd_factor(dQ, S, dQi, info, 0);
  cudaDeviceSynchronize();
  long long pr[64];
  cudaMemcpyFromSymbol(pr, g_fc_probe, sizeof(pr));
  const int nt = (S + 7) / 8;
  printf("S=%d load %lld +sym %lld (sym2 split %lld / %lld)  steps:", S, pr[44] - pr[0], pr[1] - pr[44], pr[45] - pr[44], pr[1] - pr[45]);
  long long prev = pr[1];
  for (int p = 0; p < nt; ++p) {
    printf(" %lld", pr[4 + p] - prev);
    prev = pr[4 + p];
  }
  printf("\n  pivot warp busy per step:");
  prev = pr[1];
  for (int p = 0; p < nt; ++p) {
    printf(" %lld", pr[20 + p] - prev);
    prev = pr[4 + p];
  }
  printf("\n  step 5 pivot warp: panel row %lld, diag update %lld, chol8 %lld, V write %lld",
         pr[54] - pr[8], pr[55] - pr[54], pr[56] - pr[55], pr[25] - pr[56]);
  printf("\n  tail(last gamma) %lld  total %lld cycles\n", pr[2] - prev, pr[3] - pr[0]);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int it = 0; it < 100; ++it) launch_spd_factor(dQ, S, dQi, info, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("  %.2f us per launch\n", ms * 10);
  printf("  step0 detail: prologue-chol %lld  sync %lld  alpha %lld  sync %lld\n", pr[40] - pr[1], pr[41] - pr[40],
         pr[42] - pr[41], pr[43] - pr[42]);
  // chol8_inv latency in isolation (one warp, dependent chain of calls)
  k_chol8_bench<<<1, 32>>>(100);
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(pr, g_fc_probe, sizeof(pr));
  printf("  chol8_inv: %lld cycles per call\n", pr[50]);
  return 0;
}
