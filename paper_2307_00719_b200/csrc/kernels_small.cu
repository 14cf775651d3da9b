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
  const int Rl = fl.f[fl.n - 1].Rb;
  int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (gid >= E * R0) return;
  int64_t e = gid / R0;
  int p = (int)(gid % R0);
  double v[STR_MAXR], w[STR_MAXR];
  {
    const Factor &F = fl.f[0];
    int64_t i = (e / F.stride) % F.I;
    const double *S = F.G + i * (int64_t)F.Ra * F.Rb;
    for (int b = 0; b < F.Rb; ++b) v[b] = S[p + F.Ra * b];
  }
  for (int f = 1; f < fl.n; ++f) {
    const Factor &F = fl.f[f];
    int64_t i = (e / F.stride) % F.I;
    const double *S = F.G + i * (int64_t)F.Ra * F.Rb;
    for (int b = 0; b < F.Rb; ++b) {
      double acc = 0.0;
      for (int a = 0; a < F.Ra; ++a) acc = fma(v[a], S[a + F.Ra * b], acc);
      w[b] = acc;
    }
    for (int b = 0; b < F.Rb; ++b) v[b] = w[b];
  }
  double *o = out + e * (int64_t)R0 * Rl + (int64_t)p * Rl;
  for (int q = 0; q < Rl; ++q) o[q] = v[q];
}

void launch_build_table(const FactorList &fl, int64_t E, double *out, cudaStream_t s) {
  int64_t n = E * fl.f[0].Ra;
  int threads = 256;
  k_build_table<<<(unsigned)cdiv(n, threads), threads, 0, s>>>(fl, E, out);
}

// ------------------------------------------------------------------------------------------
// Absorb: contract index `pos` of the matrix-valued tensor Y with core slices (AbsorbDesc).
// One thread per output element.  accumulate != 0 adds into `out`.
__global__ void k_absorb(AbsorbDesc ad, const double *__restrict__ Y, double *__restrict__ out,
                         int64_t n_out, int accumulate) {
  int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (gid >= n_out) return;
  const int Po = ad.left ? ad.Ra : ad.P;
  const int Qo = ad.left ? ad.Q : ad.Rb;
  int64_t rest = gid / (Po * Qo);
  int pq = (int)(gid % (Po * Qo));
  int po = pq / Qo, qo = pq % Qo;
  // Decompose `rest` over the dims without pos; compute base offset of Y entries and stride of pos.
  int64_t base = 0, stride = 1, pos_stride = 0;
  int64_t r = rest;
  for (int j = 0; j < ad.nd; ++j) {
    if (j == ad.pos) {
      pos_stride = stride;
    } else {
      int64_t ij = r % ad.d[j];
      r /= ad.d[j];
      base += ij * stride;
    }
    stride *= ad.d[j];
  }
  const int64_t esz = (int64_t)ad.P * ad.Q;
  const int64_t I = ad.d[ad.pos];
  const int64_t ssz = (int64_t)ad.Ra * ad.Rb;
  double acc = 0.0;
  if (ad.left) {
    // out[po][qo] = sum_i sum_p A(i)[po][p] Y(i)[p][qo]
    for (int64_t i = 0; i < I; ++i) {
      const double *y = Y + (base + i * pos_stride) * esz;
      const double *A = ad.A + i * ssz;
      for (int p = 0; p < ad.P; ++p) acc = fma(A[po + ad.Ra * p], y[p * ad.Q + qo], acc);
    }
  } else {
    // out[po][qo] = sum_i sum_q Y(i)[po][q] A(i)[q][qo]
    for (int64_t i = 0; i < I; ++i) {
      const double *y = Y + (base + i * pos_stride) * esz;
      const double *A = ad.A + i * ssz;
      for (int q = 0; q < ad.Q; ++q) acc = fma(y[po * ad.Q + q], A[q + ad.Ra * qo], acc);
    }
  }
  if (accumulate) out[gid] += acc; else out[gid] = acc;
}

void launch_absorb(const AbsorbDesc &ad, const double *Y, double *out, int accumulate, cudaStream_t s) {
  int64_t rest = 1;
  for (int j = 0; j < ad.nd; ++j)
    if (j != ad.pos) rest *= ad.d[j];
  const int Po = ad.left ? ad.Ra : ad.P;
  const int Qo = ad.left ? ad.Q : ad.Rb;
  int64_t n = rest * Po * Qo;
  k_absorb<<<(unsigned)cdiv(n, 128), 128, 0, s>>>(ad, Y, out, n, accumulate);
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
  double acc = 0.0;
  for (int64_t i = 0; i < I; ++i) acc = fma(G[i * ssz + b + Ra * a], G[i * ssz + d + Ra * c], acc);
  if (accumulate) Zm[gid] += acc; else Zm[gid] = acc;
}

void launch_gram_z(const double *G, int64_t I, int Ra, int Rb, double *Zm, int accumulate, cudaStream_t s) {
  int n = Ra * Ra * Rb * Rb;
  k_gram_z<<<cdiv(n, 128), 128, 0, s>>>(G, I, Ra, Rb, Zm, accumulate);
}

// ------------------------------------------------------------------------------------------
// Small row-major fp64 GEMM C[M][N] = A[M][K] B[K][N] (Gram-chain links).  16x16 tiles.
__global__ void k_dgemm(const double *__restrict__ A, const double *__restrict__ B, double *__restrict__ C, int M,
                        int N, int K) {
  __shared__ double As[16][17], Bs[16][17];
  int tx = threadIdx.x, ty = threadIdx.y;
  int row = blockIdx.y * 16 + ty, col = blockIdx.x * 16 + tx;
  double acc = 0.0;
  for (int k0 = 0; k0 < K; k0 += 16) {
    As[ty][tx] = (row < M && k0 + tx < K) ? A[(int64_t)row * K + k0 + tx] : 0.0;
    Bs[ty][tx] = (k0 + ty < K && col < N) ? B[(int64_t)(k0 + ty) * N + col] : 0.0;
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) acc = fma(As[ty][kk], Bs[kk][tx], acc);
    __syncthreads();
  }
  if (row < M && col < N) C[(int64_t)row * N + col] = acc;
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
// G = P Q^{-1} for SPD Q (S x S, S <= 128) and I right-hand-side rows P (I x S), both
// row-major.  Each CTA factors Q = L L^T in shared memory (right-looking), then solves
// L L^T g^T = p^T for a chunk of rows.  A non-positive or non-finite pivot sets *info.
constexpr int kSolveChunk = 32;

__global__ void __launch_bounds__(256) k_chol_solve(const double *__restrict__ Q, int S, const double *__restrict__ P,
                                                     int64_t I, double *__restrict__ Gout, int *info) {
  extern __shared__ double sm[];
  double *L = sm;              // S*S
  double *B = sm + S * S;      // chunk*S, row-major [r][s]
  __shared__ double piv;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t row0 = (int64_t)blockIdx.x * kSolveChunk;
  const int rows = (int)((I - row0) < kSolveChunk ? (I - row0) : kSolveChunk);
  for (int e = tid; e < S * S; e += nt) L[e] = Q[e];
  for (int e = tid; e < rows * S; e += nt) B[e] = P[(row0 + e / S) * S + e % S];
  __syncthreads();
  for (int k = 0; k < S; ++k) {
    if (tid == 0) {
      double d = L[k * S + k];
      if (!(d > 0.0) || !isfinite(d)) {
        if (info) atomicExch(info, 1);
        d = nan("");
      }
      piv = sqrt(d);
      L[k * S + k] = piv;
    }
    __syncthreads();
    const double inv = 1.0 / piv;
    for (int i = k + 1 + tid; i < S; i += nt) L[i * S + k] *= inv;
    __syncthreads();
    const int n = S - k - 1;
    for (int e = tid; e < n * n; e += nt) {
      int i = k + 1 + e / n, j = k + 1 + e % n;
      if (j <= i) L[i * S + j] -= L[i * S + k] * L[j * S + k];
    }
    __syncthreads();
  }
  // forward: L y = b (row r of B holds b^T)
  for (int k = 0; k < S; ++k) {
    const double inv = 1.0 / L[k * S + k];
    for (int r = tid; r < rows; r += nt) B[r * S + k] *= inv;
    __syncthreads();
    const int n = S - k - 1;
    for (int e = tid; e < rows * n; e += nt) {
      int r = e / n, i = k + 1 + e % n;
      B[r * S + i] -= L[i * S + k] * B[r * S + k];
    }
    __syncthreads();
  }
  // backward: L^T x = y
  for (int k = S - 1; k >= 0; --k) {
    const double inv = 1.0 / L[k * S + k];
    for (int r = tid; r < rows; r += nt) B[r * S + k] *= inv;
    __syncthreads();
    for (int e = tid; e < rows * k; e += nt) {
      int r = e / k, i = e % k;
      B[r * S + i] -= L[k * S + i] * B[r * S + k];
    }
    __syncthreads();
  }
  for (int e = tid; e < rows * S; e += nt) Gout[(row0 + e / S) * S + e % S] = B[e];
}

void launch_chol_solve(const double *Q, int S, const double *P, int64_t I, double *Gout, int *info, cudaStream_t s) {
  size_t smem = sizeof(double) * ((size_t)S * S + (size_t)kSolveChunk * S);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_chol_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr_set = true;
  }
  k_chol_solve<<<(unsigned)cdiv(I, kSolveChunk), 256, smem, s>>>(Q, S, P, I, Gout, info);
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
