// Phase timing of k_chol_solve on a random SPD system (diagnostic only).
#define STR_CHOL_PROBE 1
#include "../../paper_2307_00719_b200/csrc/kernels_small.cu"
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
using namespace strb200;
int main(int argc, char **argv) {
  int S = argc > 1 ? atoi(argv[1]) : 100, I = argc > 2 ? atoi(argv[2]) : 40;
  std::vector<double> A(S * S), Q(S * S, 0.0), P(I * S);
  srand(1);
  for (auto &v : A) v = rand() / (double)RAND_MAX - 0.5;
  for (int i = 0; i < S; ++i) for (int j = 0; j < S; ++j) { double s = 0; for (int k = 0; k < S; ++k) s += A[i * S + k] * A[j * S + k]; Q[i * S + j] = s + (i == j ? S : 0); }
  for (auto &v : P) v = rand() / (double)RAND_MAX - 0.5;
  double *dQ, *dP, *dG; int *info; long long *probe;
  cudaMalloc(&dQ, 8 * S * S); cudaMalloc(&dP, 8 * I * S); cudaMalloc(&dG, 8 * I * S); cudaMalloc(&info, 4); cudaMalloc(&probe, 64);
  cudaMemcpy(dQ, Q.data(), 8 * S * S, cudaMemcpyHostToDevice); cudaMemcpy(dP, P.data(), 8 * I * S, cudaMemcpyHostToDevice);
  cudaMemset(info, 0, 4);
  cudaMemcpyToSymbol(g_probe, &probe, sizeof(probe));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int it = 0; it < 3; ++it) launch_chol_solve(dQ, S, dP, I, dG, info, 0);
  cudaEventRecord(e0);
  for (int it = 0; it < 20; ++it) launch_chol_solve(dQ, S, dP, I, dG, info, 0);
  cudaEventRecord(e1); cudaDeviceSynchronize();
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long hp[4]; cudaMemcpy(hp, probe, 32, cudaMemcpyDeviceToHost);
  std::vector<double> G(I * S); cudaMemcpy(G.data(), dG, 8 * I * S, cudaMemcpyDeviceToHost);
  double err = 0, nrm = 0;
  for (int r = 0; r < I; ++r) for (int c = 0; c < S; ++c) { double s = 0; for (int k = 0; k < S; ++k) s += G[r * S + k] * Q[k * S + c]; err += (s - P[r * S + c]) * (s - P[r * S + c]); nrm += P[r * S + c] * P[r * S + c]; }
  printf("S=%d I=%d: %.2f us/launch (events), residual %.2e, err=%s\n", S, I, 1000 * ms / 20, sqrt(err / nrm), cudaGetErrorString(cudaGetLastError()));
  printf("cycles: load %lld  B-phases %lld  C-phases %lld  solves %lld\n", hp[0], hp[1], hp[2], hp[3]);
  return 0;
}
