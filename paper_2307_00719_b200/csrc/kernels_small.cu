// kernels_small.cu — fp64 kernels for everything R^2-sized on the STR hot path:
// chained slice tables (⊠₂ chains, Def. 6), second-level "absorb" contractions,
// core Grams Z_n (Alg. 4 l.2/l.18), Gram-chain links (×_{2,4}^{1,3}, Def. 5 /
// Prop. 1), the Q_n accumulation (Alg. 4 l.16) and the Cholesky solve
// G_n(2) = P_n Q_n^{-1} (Alg. 4 l.9/l.17).
#include "common.cuh"
#include "kernels.h"

#include <cmath>

namespace strb200 {

// ------------------------------------------------------------------------------------------
// Chained slice table.  Entry e is the product F_0(i_0) F_1(i_1) ... F_{n-1}(i_{n-1}) of the
// factor slices (each factor reads its own index from e), stored row-major Ra_0 x Rb_last.
// One thread per (entry, row p): a row vector is carried through the chain in registers.
__global__ void k_build_table(FactorList fl, int64_t E, double *__restrict__ out) {
  const int R0 = fl.f[0].Ra;
  int Rl = fl.f[0].Rb;
  int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (gid >= E * R0) return;
  int64_t e = gid / R0;
  int p = (int)(gid % R0);
  double v[STR_MAXR], w[STR_MAXR];
  {
    const Factor F = fl.f[0];
    int64_t i = (e / F.stride) % F.I;
    const double *S = F.G + i * (int64_t)F.Ra * F.Rb;
#pragma unroll
    for (int b = 0; b < STR_MAXR; ++b) v[b] = (b < F.Rb) ? S[p + F.Ra * b] : 0.0;
  }
#pragma unroll
  for (int f = 1; f < kMaxFactors; ++f) {
    if (f < fl.n) {
      const Factor F = fl.f[f];
      Rl = F.Rb;
      int64_t i = (e / F.stride) % F.I;
      const double *S = F.G + i * (int64_t)F.Ra * F.Rb;
#pragma unroll
      for (int b = 0; b < STR_MAXR; ++b) {
        double acc = 0.0;
        if (b < F.Rb) {
#pragma unroll
          for (int a = 0; a < STR_MAXR; ++a)
            if (a < F.Ra) acc = fma(v[a], S[a + F.Ra * b], acc);
        }
        w[b] = acc;
      }
#pragma unroll
      for (int b = 0; b < STR_MAXR; ++b) v[b] = w[b];
    }
  }
  double *o = out + e * (int64_t)R0 * Rl + (int64_t)p * Rl;
#pragma unroll
  for (int q = 0; q < STR_MAXR; ++q)
    if (q < Rl) o[q] = v[q];
}

void launch_build_table(const FactorList &fl, int64_t E, double *out, cudaStream_t s) {
  int64_t n = E * fl.f[0].Ra;
  int threads = 256;
  k_build_table<<<(unsigned)cdiv(n, threads), threads, 0, s>>>(fl, E, out);
}

// ------------------------------------------------------------------------------------------
// Absorb: contract index `pos` of the matrix-valued tensor Y with core slices (AbsorbDesc).
//   left : out[rest][po][qo] = sum_i sum_p A(i)[po][p] Y(rest, i)[p][qo]
//   right: out[rest][po][qo] = sum_i sum_q Y(rest, i)[po][q] A(i)[q][qo]
// Thread layout: g adjacent lanes per output element split the contracted index i and reduce
// with shuffles; a CTA covers 256/g consecutive outputs (several `rest` entries), with the A
// slices of a chunk of i staged once per CTA in shared memory; Y is read through L1/L2.
constexpr int kAbsorbThreads = 256, kAbsorbSmemDoubles = 4096;

template <typename TY>
__global__ void __launch_bounds__(kAbsorbThreads) k_absorb(AbsorbDesc ad, const TY *__restrict__ Y,
                                                           double *__restrict__ out, int accumulate, int g, int ichunk,
                                                           int64_t before, int64_t I, int64_t n_out) {
  __shared__ double As[kAbsorbSmemDoubles];
  const int Po = ad.left ? ad.Ra : ad.P;
  const int Qo = ad.left ? ad.Q : ad.Rb;
  const int O = Po * Qo;
  const int PQ = ad.P * ad.Q, AB = ad.Ra * ad.Rb;
  const int64_t gid = blockIdx.x * (int64_t)kAbsorbThreads + threadIdx.x;
  const int64_t oi = gid / g;                 // global output index
  const int sub = (int)(gid % g);
  const bool active = oi < n_out;
  const int64_t rest = active ? oi / O : 0;
  const int o = (int)(oi % O);
  const int po = o / Qo, qo = o % Qo;
  // Y multi-index = b + before*(i + I*a) with b < before, a < after; rest = b + before*a.
  const int64_t b0 = rest % before, a0 = rest / before;
  const TY *ybase = Y + (b0 + before * I * a0) * PQ;
  const int64_t ystride = before * PQ;        // between consecutive i
  double acc = 0.0;
  for (int64_t i0 = 0; i0 < I; i0 += ichunk) {
    const int ic = (int)((I - i0) < ichunk ? (I - i0) : ichunk);
    __syncthreads();
    const double *Ag = ad.A + i0 * AB;
    for (int e = threadIdx.x; e < ic * AB; e += kAbsorbThreads) As[e] = Ag[e];
    __syncthreads();
    if (active) {
      // fully unrolled (predicated) inner loop: the STR_MAXR loads of one i issue back to back
      if (ad.left) {
        for (int i = sub; i < ic; i += g) {
          const double *a = As + i * AB + po;
          const TY *y = ybase + (i0 + i) * ystride + qo;
          double yv[STR_MAXR];
#pragma unroll
          for (int p = 0; p < STR_MAXR; ++p) yv[p] = (p < ad.P) ? (double)y[p * ad.Q] : 0.0;
#pragma unroll
          for (int p = 0; p < STR_MAXR; ++p)
            if (p < ad.P) acc = fma(a[ad.Ra * p], yv[p], acc);
        }
      } else {
        for (int i = sub; i < ic; i += g) {
          const double *a = As + i * AB + ad.Ra * qo;
          const TY *y = ybase + (i0 + i) * ystride + po * ad.Q;
          double yv[STR_MAXR];
#pragma unroll
          for (int q = 0; q < STR_MAXR; ++q) yv[q] = (q < ad.Q) ? (double)y[q] : 0.0;
#pragma unroll
          for (int q = 0; q < STR_MAXR; ++q)
            if (q < ad.Q) acc = fma(yv[q], a[q], acc);
        }
      }
    }
  }
  for (int sh = g / 2; sh > 0; sh >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, sh);
  if (active && sub == 0) {
    double *dst = out + oi;
    if (accumulate) *dst += acc; else *dst = acc;
  }
}

void launch_absorb(const AbsorbDesc &ad, const void *Y, bool y_f32, double *out, int accumulate, cudaStream_t s) {
  int64_t rest = 1, before = 1;
  for (int j = 0; j < ad.nd; ++j)
    if (j != ad.pos) rest *= ad.d[j];
  for (int j = 0; j < ad.pos; ++j) before *= ad.d[j];
  const int Po = ad.left ? ad.Ra : ad.P;
  const int Qo = ad.left ? ad.Q : ad.Rb;
  const int64_t I = ad.d[ad.pos];
  const int64_t K = I * (ad.left ? ad.P : ad.Q);
  int g = K <= 64 ? 1 : (K <= 160 ? 2 : (K <= 320 ? 4 : (K <= 640 ? 8 : 16)));
  const int64_t n_out = rest * Po * Qo;
  int ichunk = kAbsorbSmemDoubles / (ad.Ra * ad.Rb);
  if (ichunk > I) ichunk = (int)I;
  const unsigned grid = (unsigned)cdiv(n_out * g, kAbsorbThreads);
  if (y_f32)
    k_absorb<float><<<grid, kAbsorbThreads, 0, s>>>(ad, (const float *)Y, out, accumulate, g, ichunk, before, I, n_out);
  else
    k_absorb<double><<<grid, kAbsorbThreads, 0, s>>>(ad, (const double *)Y, out, accumulate, g, ichunk, before, I,
                                                     n_out);
}

// ------------------------------------------------------------------------------------------
// Gram tensor as a chain matrix: Zm[(a + Rb c)][(b + Ra d)] = sum_i G(i)(b,a) G(i)(d,c)
// (Z(a,b,c,d) of P:228 with rows = (1st,3rd) index pair, columns = (2nd,4th)), G(i) = Ra x Rb
// slices in G(2) layout.  accumulate != 0 adds (used for sharded partial Grams).
__global__ void k_gram_z(const double *__restrict__ G, int64_t I, int Ra, int Rb, double *__restrict__ Zm,
                         int accumulate) {
  int rows = Rb * Rb, cols = Ra * Ra;
  int gid = blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= rows * cols) return;
  int row = gid / cols, col = gid % cols;
  int a = row % Rb, c = row / Rb, b = col % Ra, d = col / Ra;
  const int64_t ssz = (int64_t)Ra * Rb;
  const double *g1 = G + b + Ra * a, *g2 = G + d + Ra * c;
  double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
  int64_t i = 0;
  for (; i + 4 <= I; i += 4) {
    acc0 = fma(g1[i * ssz], g2[i * ssz], acc0);
    acc1 = fma(g1[(i + 1) * ssz], g2[(i + 1) * ssz], acc1);
    acc2 = fma(g1[(i + 2) * ssz], g2[(i + 2) * ssz], acc2);
    acc3 = fma(g1[(i + 3) * ssz], g2[(i + 3) * ssz], acc3);
  }
  for (; i < I; ++i) acc0 = fma(g1[i * ssz], g2[i * ssz], acc0);
  const double acc = (acc0 + acc1) + (acc2 + acc3);
  if (accumulate) Zm[gid] += acc; else Zm[gid] = acc;
}

void launch_gram_z(const double *G, int64_t I, int Ra, int Rb, double *Zm, int accumulate, cudaStream_t s) {
  int n = Ra * Ra * Rb * Rb;
  k_gram_z<<<cdiv(n, 128), 128, 0, s>>>(G, I, Ra, Rb, Zm, accumulate);
}

// ------------------------------------------------------------------------------------------
// Small row-major fp64 GEMM C[M][N] = A[M][K] B[K][N] (Gram-chain links).  16x16 output tiles
// (one per thread block of 256), K staged 32 at a time, 4 independent accumulator chains.
__global__ void __launch_bounds__(256) k_dgemm(const double *__restrict__ A, const double *__restrict__ B,
                                               double *__restrict__ C, int M, int N, int K) {
  __shared__ double As[16][33], Bs[32][17];
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * 16 + tx;
  const int row = blockIdx.y * 16 + ty, col = blockIdx.x * 16 + tx;
  double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
  for (int k0 = 0; k0 < K; k0 += 32) {
    for (int e = tid; e < 16 * 32; e += 256) {
      const int r = e / 32, kk = e % 32;
      const int gr = blockIdx.y * 16 + r;
      As[r][kk] = (gr < M && k0 + kk < K) ? A[(int64_t)gr * K + k0 + kk] : 0.0;
      const int kr = e / 16, cc = e % 16;
      const int gc = blockIdx.x * 16 + cc;
      Bs[kr][cc] = (k0 + kr < K && gc < N) ? B[(int64_t)(k0 + kr) * N + gc] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 32; kk += 4) {
      acc0 = fma(As[ty][kk], Bs[kk][tx], acc0);
      acc1 = fma(As[ty][kk + 1], Bs[kk + 1][tx], acc1);
      acc2 = fma(As[ty][kk + 2], Bs[kk + 2][tx], acc2);
      acc3 = fma(As[ty][kk + 3], Bs[kk + 3][tx], acc3);
    }
    __syncthreads();
  }
  if (row < M && col < N) C[(int64_t)row * N + col] = (acc0 + acc1) + (acc2 + acc3);
}

void launch_dgemm(const double *A, const double *B, double *C, int M, int N, int K, cudaStream_t s) {
  dim3 blk(16, 16), grd((unsigned)cdiv(N, 16), (unsigned)cdiv(M, 16));
  k_dgemm<<<grd, blk, 0, s>>>(A, B, C, M, N, K);
}

// ------------------------------------------------------------------------------------------
// Q (+)= symmetrized H_<2>, where H_<2>[i1 + Rn i2][r1 + Rn r2] = Hm[i1 + Rn r1][i2 + Rn1 r2]
// (Def. 1 P:126 applied to the chain result; reading R5 symmetrizes).  One thread per (x <= y).
__global__ void k_q_accum(const double *__restrict__ Hm, int Rn, int Rn1, double *__restrict__ Q, int accumulate) {
  int S = Rn * Rn1;
  int gid = blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= S * S) return;
  int x = gid / S, y = gid % S;
  if (y < x) return;
  auto h2 = [&](int u, int v) {
    int i1 = u % Rn, i2 = u / Rn, r1 = v % Rn, r2 = v / Rn;
    return Hm[(int64_t)(i1 + Rn * r1) * (Rn1 * Rn1) + (i2 + Rn1 * r2)];
  };
  double h = 0.5 * (h2(x, y) + h2(y, x));
  double v = accumulate ? Q[(int64_t)x * S + y] + h : h;
  Q[(int64_t)x * S + y] = v;
  Q[(int64_t)y * S + x] = v;
}

void launch_q_accum(const double *Hm, int Rn, int Rn1, double *Q, int accumulate, cudaStream_t s) {
  int S = Rn * Rn1;
  k_q_accum<<<cdiv(S * S, 128), 128, 0, s>>>(Hm, Rn, Rn1, Q, accumulate);
}

// ------------------------------------------------------------------------------------------
__global__ void k_axpy(const double *__restrict__ x, double *__restrict__ y, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) y[i] += x[i];
}

void launch_axpy(const double *x, double *y, int64_t n, cudaStream_t s) {
  k_axpy<<<(unsigned)cdiv(n, 256), 256, 0, s>>>(x, y, n);
}

__global__ void k_set_identity(double *A, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n * n) A[i] = (i / n == i % n) ? 1.0 : 0.0;
}

void launch_set_identity(double *A, int n, cudaStream_t s) {
  k_set_identity<<<cdiv(n * n, 256), 256, 0, s>>>(A, n);
}

}  // namespace strb200
