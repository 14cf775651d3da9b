// Isolated timing of the serial-chain kernels of kernels_chain.cu (diagnostic only).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../include -I../../paper_2307_00719_b200/csrc \
//        -o chain_bench chain_bench.cu && ./chain_bench
#define INV_PROBE 1
#include "../../paper_2307_00719_b200/csrc/kernels_chain.cu"
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
namespace strb200 {
void prepare_f64_attrs() {}
void launch_fit_reduce(const double2 *, int64_t, double *, cudaStream_t) {}
}  // namespace strb200
using namespace strb200;

template <typename F>
static float time_us(F f, int iters = 50) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int i = 0; i < 5; ++i) f();
  cudaEventRecord(e0);
  for (int i = 0; i < iters; ++i) f();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return 1000.f * ms / iters;
}

// skeleton of the sweep loop: MODE 0: LDS + 64 FMA + barrier; 1: no barrier; 2: no LDS (registers)
template <int MODE>
__global__ void k_skel8(double *out, int steps, long long *cyc) {
  __shared__ __align__(16) double2 vb[2][4][16];
  const int t = threadIdx.x;
  for (int i = t; i < 128; i += blockDim.x) ((double *)vb)[i] = 1.0 + 1e-3 * i;
  double a[8][8];
  for (int r = 0; r < 8; ++r) for (int q = 0; q < 8; ++q) a[r][q] = r + q + t;
  const int ib = t % 13, jb = (t * 3) % 13;
  double vi[8], vj[8];
  for (int u = 0; u < 8; ++u) { vi[u] = 1e-3 * u; vj[u] = 2e-3 * u; }
  __syncthreads();
  long long t0 = clock64();
  for (int c = 0; c < steps; ++c) {
    const int buf = c & 1;
    const double p = 0.5 + 1e-9 * c;
    if (MODE != 2) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double2 xv = vb[buf][u][ib], yv = vb[buf][u][jb];
        vi[2 * u] = xv.x; vi[2 * u + 1] = xv.y; vj[2 * u] = yv.x; vj[2 * u + 1] = yv.y;
      }
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const double sr = vi[r] * p;
#pragma unroll
      for (int q = 0; q < 8; ++q) a[r][q] = fma(-sr, vj[q], a[r][q]);
    }
    if (MODE != 2 && t == 0) vb[buf ^ 1][c & 3][c % 13] = make_double2(a[0][0], a[1][1]);
    if (MODE == 0) __syncthreads();
    if (MODE == 2) { vi[c & 7] += 1e-12; }
  }
  long long t1 = clock64();
  if (t == 0) cyc[0] = t1 - t0;
  double sacc = 0;
  for (int r = 0; r < 8; ++r) for (int q = 0; q < 8; ++q) sacc += a[r][q];
  out[t] = sacc;
}

__global__ void k_empty_n() {}
__global__ void k_copy_d(const double *__restrict__ a, double *__restrict__ b, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) b[i] = a[i];
}
__global__ void k_dep_loads(const double *__restrict__ a, double *__restrict__ b, int n) {
  // one thread chain of n dependent L2 loads
  int idx = threadIdx.x;
  double acc = 0;
  for (int i = 0; i < n; ++i) { double v = a[idx]; acc += v; idx = ((int)v + i * 97 + threadIdx.x) & 4095; }
  b[threadIdx.x] = acc;
}

int main(int argc, char **argv) {
  {
    double *a, *b; cudaMalloc(&a, 8 << 20); cudaMalloc(&b, 8 << 20); cudaMemset(a, 0, 8 << 20);
    float e1 = time_us([&] { k_empty_n<<<1, 32>>>(); });
    float e2 = time_us([&] { k_empty_n<<<1600, 512>>>(); });
    float e3 = time_us([&] { k_empty_n<<<148, 1024>>>(); });
    float c1 = time_us([&] { k_copy_d<<<625, 256>>>(a, b, 160000); });
    float c2 = time_us([&] { k_copy_d<<<4096, 256>>>(a, b, 1 << 20); });
    float d1 = time_us([&] { k_dep_loads<<<1, 32>>>(a, b, 100); });
    printf("empty 1x32 %.2f | empty 1600x512 %.2f | empty 148x1024 %.2f | copy 1.28MB %.2f | copy 8MB %.2f | 100 dep loads %.2f us\n",
           e1, e2, e3, c1, c2, d1);
  }
  {
    double *o; long long *cy; cudaMalloc(&o, 8 * 1024); cudaMalloc(&cy, 64);
    for (int thr : {32, 96}) {
      long long hc[3];
      k_skel8<0><<<1, thr>>>(o, 100, cy); cudaDeviceSynchronize(); cudaMemcpy(&hc[0], cy, 8, cudaMemcpyDeviceToHost);
      k_skel8<1><<<1, thr>>>(o, 100, cy); cudaDeviceSynchronize(); cudaMemcpy(&hc[1], cy, 8, cudaMemcpyDeviceToHost);
      k_skel8<2><<<1, thr>>>(o, 100, cy); cudaDeviceSynchronize(); cudaMemcpy(&hc[2], cy, 8, cudaMemcpyDeviceToHost);
      printf("skel8 %d thr: LDS+FMA+bar %.0f | no bar %.0f | regs only %.0f cycles/step\n", thr, hc[0] / 100.0,
             hc[1] / 100.0, hc[2] / 100.0);
    }
    // instrumented real kernel: per-step cycles from clock64 around the whole kernel
  }
  const int S = argc > 1 ? atoi(argv[1]) : 100;
  const int I = argc > 2 ? atoi(argv[2]) : 40;
  std::vector<double> A(S * S), Q(S * S, 0.0), P(I * S);
  srand(1);
  for (auto &v : A) v = rand() / (double)RAND_MAX - 0.5;
  for (int i = 0; i < S; ++i)
    for (int j = 0; j < S; ++j) {
      double s = 0;
      for (int k = 0; k < S; ++k) s += A[i * S + k] * A[j * S + k];
      Q[i * S + j] = s + (i == j ? 1.0 : 0);
    }
  for (auto &v : P) v = rand() / (double)RAND_MAX - 0.5;
  double *dQ, *dQi, *dP, *dG, *dA, *dB, *dC;
  int *info;
  cudaMalloc(&dQ, 8 * S * S);
  cudaMalloc(&dQi, 8 * S * S);
  cudaMalloc(&dP, 8 * I * S);
  cudaMalloc(&dG, 8 * I * S);
  cudaMalloc(&dA, 8 * 256 * 256);
  cudaMalloc(&dB, 8 * 256 * 256);
  cudaMalloc(&dC, 8 * 256 * 256);
  cudaMalloc(&info, 4);
  cudaMemcpy(dQ, Q.data(), 8 * S * S, cudaMemcpyHostToDevice);
  cudaMemcpy(dP, P.data(), 8 * I * S, cudaMemcpyHostToDevice);
  cudaMemcpy(dA, Q.data(), 8 * S * S, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, Q.data(), 8 * S * S, cudaMemcpyHostToDevice);
  cudaMemset(info, 0, 4);
  // empty-kernel floor
  float t_empty = time_us([&] { k_axpy_any<double><<<1, 32>>>(dP, dG, 0, 0); });
  float t_inv = time_us([&] { launch_spd_inv(dQ, S, dQi, info, 0); });
  float t_rows = time_us([&] { launch_rows_mm(dP, dQi, S, I, dG, 0); });
  float t_gemm = time_us([&] { launch_chain_gemm(dA, dB, dC, S, S, S, QEpi{nullptr, 0, 0, 0}, 0); });
  float t_gram = time_us([&] { launch_gram_z2(dP, I, 10, 10, dC, 0, 0); });
  // graph of 40 serially dependent empty kernels: per-node cost
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  for (int i = 0; i < 40; ++i) k_axpy_any<double><<<1, 32, 0, st>>>(dP, dG, 0, 0);
  cudaStreamEndCapture(st, &g);
  cudaGraphInstantiate(&ge, g, 0);
  float t_graph = time_us([&] { cudaGraphLaunch(ge, st); }, 20) / 40.f;
  cudaStreamSynchronize(st);
  // graph of 40 spd_inv
  cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  for (int i = 0; i < 10; ++i) launch_spd_inv(dQ, S, dQi, info, st);
  cudaStreamEndCapture(st, &g);
  cudaGraphInstantiate(&ge, g, 0);
  float t_ginv = time_us([&] { cudaGraphLaunch(ge, st); }, 10) / 10.f;
  cudaStreamSynchronize(st);
  printf("graph: %.2f us per empty node, %.2f us per spd_inv node\n", t_graph, t_ginv);
  // graph-node cost of the chain GEMM (S x S x S and I x S x S) per staging mode
  for (int mode = 0; mode < 4; ++mode) {
    g_gemm_stage = mode;
    float tg[2];
    for (int w = 0; w < 2; ++w) {
      cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
      for (int i = 0; i < 20; ++i) {
        if (w == 0) launch_chain_gemm(dA, dB, dC, S, S, S, QEpi{nullptr, 0, 0, 0}, st);
        else launch_rows_mm(dP, dQi, S, I, dG, st);
      }
      cudaStreamEndCapture(st, &g);
      cudaGraphInstantiate(&ge, g, 0);
      tg[w] = time_us([&] { cudaGraphLaunch(ge, st); }, 10) / 20.f;
      cudaStreamSynchronize(st);
    }
    printf("graph: chain_gemm stage %d: %.2f us per %dx%dx%d node, %.2f us per rows_mm (%d rows) node\n", mode, tg[0], S, S,
           S, tg[1], I);
  }
  g_gemm_stage = -1;
  {
    // C5-shaped absorbs: Y_L (i1, i2, t) 40 x 40 x 8 entries 10x10 (fp32), contract i2 with G_2 slices
    float *Yf; double *Ad, *Od, *Wd;
    cudaMalloc(&Yf, sizeof(float) * 12800 * 100);
    cudaMalloc(&Ad, sizeof(double) * 40 * 100);
    cudaMalloc(&Od, sizeof(double) * 12800 * 100);
    cudaMalloc(&Wd, sizeof(double) * 1600 * 100);
    cudaMemset(Yf, 0, sizeof(float) * 12800 * 100);
    cudaMemset(Ad, 0, sizeof(double) * 40 * 100);
    cudaMemset(Wd, 0, sizeof(double) * 1600 * 100);
    AbsorbDesc ad{};
    ad.nd = 3; ad.d[0] = 40; ad.d[1] = 40; ad.d[2] = 8; ad.pos = 1; ad.P = 10; ad.Q = 10; ad.left = 1; ad.A = Ad; ad.Ra = 10; ad.Rb = 10;
    float t1 = time_us([&] { launch_absorb2(ad, Yf, true, Od, 0, 0); });
    ad.pos = 2; ad.left = 0;   // W: contract t (I = 8) on the right
    ad.A = Ad;
    float t2 = time_us([&] { launch_absorb2(ad, Yf, true, Od, 0, 0); });
    AbsorbDesc am{};
    am.nd = 2; am.d[0] = 40; am.d[1] = 40; am.pos = 1; am.P = 10; am.Q = 10; am.left = 1; am.A = Ad; am.Ra = 10; am.Rb = 10;
    float t3 = time_us([&] { launch_absorb2(am, Wd, false, Od, 1, 0); });
    // T_L table: 12800 entries of G_N(t) G_1(i1) G_2(i2), tf32 tiles
    TableDesc td{};
    td.fl.n = 3;
    td.fl.f[0] = Factor{Ad, 8, 10, 10, 1600};
    td.fl.f[1] = Factor{Ad, 40, 10, 10, 1};
    td.fl.f[2] = Factor{Ad, 40, 10, 10, 40};
    td.Lk = 1600; td.tk = 8; td.Npad = 112;
    float *tiles; cudaMalloc(&tiles, sizeof(float) * 400 * 2 * 112 * 32);
    float t4 = time_us([&] { launch_build_table2(td, nullptr, tiles, 0); });
    for (int cps : {1, 2, 3, 4}) {
      g_absorb_cps = cps;
      ad.pos = 1; ad.left = 1;
      float u1 = time_us([&] { launch_absorb2(ad, Yf, true, Od, 0, 0); });
      ad.pos = 2; ad.left = 0;
      float u2 = time_us([&] { launch_absorb2(ad, Yf, true, Od, 0, 0); });
      float u3 = time_us([&] { launch_absorb2(am, Wd, false, Od, 1, 0); });
      printf("absorb CTAs/SM target %d: %.2f | %.2f | %.2f us\n", cps, u1, u2, u3);
    }
    g_absorb_cps = 3;
    printf("absorb Y_L->mode2 (320 rest) %.2f us | absorb W over t (1600 rest) %.2f us | mode absorb (40 rest) %.2f us | table T_L %.2f us\n",
           t1, t2, t3, t4);
  }
  // correctness: G Q = P
  std::vector<double> G(I * S);
  cudaMemcpy(G.data(), dG, 8 * I * S, cudaMemcpyDeviceToHost);
  double err = 0, nrm = 0;
  for (int r = 0; r < I; ++r)
    for (int c = 0; c < S; ++c) {
      double s = 0;
      for (int k = 0; k < S; ++k) s += G[r * S + k] * Q[k * S + c];
      err += (s - P[r * S + c]) * (s - P[r * S + c]);
      nrm += P[r * S + c] * P[r * S + c];
    }
  int hinfo;
  cudaMemcpy(&hinfo, info, 4, cudaMemcpyDeviceToHost);
  printf("S=%d I=%d  empty %.2f us | spd_inv %.2f us | rows_mm %.2f us | chain_gemm %.2f us | gram %.2f us\n", S, I,
         t_empty, t_inv, t_rows, t_gemm, t_gram);
  long long pr[8];
  {
    long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_inv_probe, z, sizeof(z));
    launch_spd_inv(dQ, S, dQi, info, 0);
    cudaDeviceSynchronize();
  }
  cudaMemcpyFromSymbol(pr, g_inv_probe, sizeof(pr));
  {
    const int nt = (S + 7) / 8;
    printf("cluster inverse, per step (mean over the 4 CTAs, warp 0): W %.0f  updates %.0f  barrier %.0f cycles; "
           "pivot sweeps %.0f cycles each\n", pr[1] / 4.0 / (nt + 1), pr[2] / 4.0 / (nt + 1), pr[3] / 4.0 / (nt + 1),
           pr[4] / (double)nt);
  }


  printf("residual ||G Q - P||/||P|| = %.2e  info=%d  err=%s\n", sqrt(err / nrm), hinfo,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
