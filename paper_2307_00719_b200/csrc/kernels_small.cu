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
// One CTA per remaining multi-index ("rest"); the Y entries and A slices of a chunk of the
// contracted index are staged in shared memory; each output entry is accumulated by a group
// of g threads (g | 32) that split the contracted index and combine with shuffles.
constexpr int kAbsorbThreads = 256, kAbsorbSmemDoubles = 6144;

__global__ void __launch_bounds__(kAbsorbThreads) k_absorb(AbsorbDesc ad, const double *__restrict__ Y,
                                                           double *__restrict__ out, int accumulate, int g, int ichunk,
                                                           int64_t before, int64_t I) {
  __shared__ double sm[kAbsorbSmemDoubles];
  const int Po = ad.left ? ad.Ra : ad.P;
  const int Qo = ad.left ? ad.Q : ad.Rb;
  const int O = Po * Qo;
  const int PQ = ad.P * ad.Q, AB = ad.Ra * ad.Rb;
  // Y multi-index = b + before*(i + I*a) with b < before, a < after; rest = b + before*a.
  const int64_t rest = blockIdx.x;
  const int64_t b0 = rest % before, a0 = rest / before;
  const int64_t base = b0 + before * I * a0, pos_stride = before;
  double *Ys = sm;
  double *As = sm + (int64_t)ichunk * PQ;
  const int tid = threadIdx.x;
  const int o = tid / g, sub = tid % g;
  const int po = o / Qo, qo = o % Qo;
  double acc = 0.0;
  for (int64_t i0 = 0; i0 < I; i0 += ichunk) {
    const int ic = (int)((I - i0) < ichunk ? (I - i0) : ichunk);
    __syncthreads();
    for (int e = tid; e < ic * PQ; e += kAbsorbThreads) {
      int i = e / PQ, w = e % PQ;
      Ys[e] = Y[(base + (i0 + i) * pos_stride) * PQ + w];
    }
    const double *Ag = ad.A + i0 * AB;
    for (int e = tid; e < ic * AB; e += kAbsorbThreads) As[e] = Ag[e];
    __syncthreads();
    if (o < O) {
      if (ad.left) {
        for (int i = sub; i < ic; i += g) {
          const double *a = As + i * AB + po;
          const double *y = Ys + i * PQ + qo;
#pragma unroll 4
          for (int p = 0; p < ad.P; ++p) acc = fma(a[ad.Ra * p], y[p * ad.Q], acc);
        }
      } else {
        for (int i = sub; i < ic; i += g) {
          const double *a = As + i * AB + ad.Ra * qo;
          const double *y = Ys + i * PQ + po * ad.Q;
#pragma unroll 4
          for (int q = 0; q < ad.Q; ++q) acc = fma(y[q], a[q], acc);
        }
      }
    }
  }
  for (int sh = g / 2; sh > 0; sh >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, sh);
  if (o < O && sub == 0) {
    double *dst = out + rest * O + o;
    if (accumulate) *dst += acc; else *dst = acc;
  }
}

void launch_absorb(const AbsorbDesc &ad, const double *Y, double *out, int accumulate, cudaStream_t s) {
  int64_t rest = 1, before = 1;
  for (int j = 0; j < ad.nd; ++j)
    if (j != ad.pos) rest *= ad.d[j];
  for (int j = 0; j < ad.pos; ++j) before *= ad.d[j];
  const int Po = ad.left ? ad.Ra : ad.P;
  const int Qo = ad.left ? ad.Q : ad.Rb;
  const int O = Po * Qo;
  int g = 1;
  while (g < 8 && O * g * 2 <= kAbsorbThreads) g *= 2;
  int per = ad.P * ad.Q + ad.Ra * ad.Rb;
  int ichunk = kAbsorbSmemDoubles / per;
  if (ichunk > ad.d[ad.pos]) ichunk = (int)ad.d[ad.pos];
  k_absorb<<<(unsigned)rest, kAbsorbThreads, 0, s>>>(ad, Y, out, accumulate, g, ichunk, before, ad.d[ad.pos]);
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
// G = P Q^{-1} for SPD Q (S x S, S <= 128) and I right-hand-side rows P (I x S), row-major.
// Blocked right-looking Cholesky (block 8): the packed lower triangle lives in registers
// (entry e belongs to thread e % 256).  Per block column: the panel is published to shared
// memory, every row thread factors the 8x8 diagonal block redundantly (rsqrt pivots) and solves
// its own row, the first 8 threads also emit the inverse of the diagonal block, then a rank-8
// update hits the trailing entries.  Forward / backward substitution use the inverted diagonal
// blocks.  Each CTA factors Q (redundantly) and solves a chunk of <= 64 RHS rows.
// A non-positive or non-finite pivot sets *info.
constexpr int kNB = 8, kNT = 256, kMaxE = 33, kSolveChunk = 16;

__global__ void __launch_bounds__(kNT, 1) k_chol_solve(const double *__restrict__ Q, int S,
                                                        const double *__restrict__ P, int64_t I,
                                                        double *__restrict__ Gout, int *info) {
  extern __shared__ double sm[];
  const int S2 = (S * S + 3) & ~3;          // regions padded to 32-byte multiples
  double *Lf = sm;                          // S*S, final L (lower), row-major
  double *Bm = Lf + S2;                     // kSolveChunk * S RHS rows
  double *Pn = Bm + kSolveChunk * S;        // S * 8 panel (input)
  double *Ln = Pn + S * kNB;                // S * 8 panel (output)
  double *Di = Ln + S * kNB;                // (S/8+1) * 64 inverted diagonal blocks (lower)
  const int tid = threadIdx.x;
  const int64_t row0 = (int64_t)blockIdx.x * kSolveChunk;
  const int rows = (int)((I - row0) < kSolveChunk ? (I - row0) : kSolveChunk);
  const int ntri = S * (S + 1) / 2;
  double val[kMaxE];
  int ij[kMaxE];
#pragma unroll
  for (int r = 0; r < kMaxE; ++r) {
    int e = tid + kNT * r;
    ij[r] = -1;
    val[r] = 0.0;
    if (e < ntri) {
      int i = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
      while (i * (i + 1) / 2 > e) --i;
      while ((i + 1) * (i + 2) / 2 <= e) ++i;
      int j = e - i * (i + 1) / 2;
      ij[r] = (i << 8) | j;
      val[r] = Q[(int64_t)i * S + j];
    }
  }
  for (int e = tid; e < rows * S; e += kNT) Bm[e] = P[(row0 + e / S) * S + e % S];
  bool bad = false;
  for (int kb = 0; kb < S; kb += kNB) {
    const int nbk = (S - kb) < kNB ? (S - kb) : kNB;
#pragma unroll
    for (int r = 0; r < kMaxE; ++r) {
      int i = ij[r] >> 8, j = ij[r] & 255;
      if (ij[r] >= 0 && j >= kb && j < kb + nbk) Pn[i * kNB + (j - kb)] = val[r];
    }
    __syncthreads();
    if (tid < S - kb) {
      const int i = kb + tid;
      double Ld[kNB][kNB], rd[kNB];
#pragma unroll
      for (int a = 0; a < kNB; ++a)
#pragma unroll
        for (int b = 0; b <= a; ++b) Ld[a][b] = (a < nbk) ? Pn[(kb + a) * kNB + b] : 0.0;
#pragma unroll
      for (int c = 0; c < kNB; ++c) {
        double d = Ld[c][c], r = 0.0;
        if (c < nbk) {
          if (!(d > 0.0) || !isfinite(d)) bad = true;
          r = rsqrt(d);
          Ld[c][c] = d * r;
        }
        rd[c] = r;
#pragma unroll
        for (int a = c + 1; a < kNB; ++a) Ld[a][c] *= r;
#pragma unroll
        for (int a = c + 1; a < kNB; ++a)
#pragma unroll
          for (int b = c + 1; b <= a; ++b) Ld[a][b] = fma(-Ld[a][c], Ld[b][c], Ld[a][b]);
      }
      double l[kNB];
      if (i < kb + nbk) {
#pragma unroll
        for (int m = 0; m < kNB; ++m) {
          double x = 0.0;
#pragma unroll
          for (int a = 0; a < kNB; ++a)
            if (m <= a && a == i - kb) x = Ld[a][m];
          l[m] = x;
        }
        // column (i - kb) of the inverse diagonal block
        const int c = i - kb;
        double x[kNB];
#pragma unroll
        for (int a = 0; a < kNB; ++a) {
          double v = (a == c) ? 1.0 : 0.0;
#pragma unroll
          for (int q = 0; q < a; ++q) v = fma(-Ld[a][q], x[q], v);
          x[a] = v * rd[a];
        }
        double *D = Di + (kb / kNB) * kNB * kNB;
#pragma unroll
        for (int a = 0; a < kNB; ++a) D[a * kNB + c] = x[a];
      } else {
#pragma unroll
        for (int m = 0; m < kNB; ++m) {
          double a = (m < nbk) ? Pn[i * kNB + m] : 0.0;
#pragma unroll
          for (int q = 0; q < m; ++q) a = fma(-l[q], Ld[m][q], a);
          l[m] = a * rd[m];
        }
      }
#pragma unroll
      for (int m = 0; m < kNB; ++m) Ln[i * kNB + m] = l[m];
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kMaxE; ++r) {
      if (ij[r] < 0) continue;
      int i = ij[r] >> 8, j = ij[r] & 255;
      if (j >= kb && j < kb + nbk) {
        val[r] = Ln[i * kNB + (j - kb)];
      } else if (j >= kb + nbk) {
        const double2 *li = (const double2 *)(Ln + i * kNB);
        const double2 *lj = (const double2 *)(Ln + j * kNB);
        double acc = val[r];
#pragma unroll
        for (int m = 0; m < kNB / 2; ++m) {
          double2 x = li[m], y = lj[m];
          acc = fma(-x.x, y.x, acc);
          acc = fma(-x.y, y.y, acc);
        }
        val[r] = acc;
      }
    }
  }
  if (bad && info) atomicExch(info, 1);
  for (int e = tid; e < S * S; e += kNT) Lf[e] = 0.0;
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kMaxE; ++r)
    if (ij[r] >= 0) Lf[(ij[r] >> 8) * S + (ij[r] & 255)] = val[r];
  __syncthreads();
  const int ti = tid & 127, tr = tid >> 7;
  const int nblk = (S + kNB - 1) / kNB;
  // forward substitution, L y = b, for every RHS row (rows of Bm hold b^T)
  for (int bi = 0; bi < nblk; ++bi) {
    const int kb = bi * kNB;
    const int nbk = (S - kb) < kNB ? (S - kb) : kNB;
    const double *D = Di + bi * kNB * kNB;
    double yv[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      int w = tid + kNT * u, r1 = w / kNB, m1 = w % kNB;
      yv[u] = 0.0;
      if (r1 < rows && m1 < nbk)
#pragma unroll
        for (int q = 0; q < kNB; ++q) yv[u] = fma(D[m1 * kNB + q], (q < nbk) ? Bm[r1 * S + kb + q] : 0.0, yv[u]);
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      int w = tid + kNT * u, r1 = w / kNB, m1 = w % kNB;
      if (r1 < rows && m1 < nbk) Bm[r1 * S + kb + m1] = yv[u];
    }
    __syncthreads();
    if (ti >= kb + nbk && ti < S) {
      double lrow[kNB];
#pragma unroll
      for (int m = 0; m < kNB; ++m) lrow[m] = (m < nbk) ? Lf[ti * S + kb + m] : 0.0;
      for (int r = tr; r < rows; r += kNT / 128) {
        double acc = Bm[r * S + ti];
        const double *y = Bm + r * S + kb;
#pragma unroll
        for (int m = 0; m < kNB; ++m) acc = fma(-lrow[m], (m < nbk) ? y[m] : 0.0, acc);
        Bm[r * S + ti] = acc;
      }
    }
    __syncthreads();
  }
  // backward substitution, L^T x = y
  for (int bi = nblk - 1; bi >= 0; --bi) {
    const int kb = bi * kNB;
    const int nbk = (S - kb) < kNB ? (S - kb) : kNB;
    const double *D = Di + bi * kNB * kNB;
    double xv[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      int w = tid + kNT * u, r1 = w / kNB, m1 = w % kNB;
      xv[u] = 0.0;
      if (r1 < rows && m1 < nbk)
#pragma unroll
        for (int q = 0; q < kNB; ++q) xv[u] = fma(D[q * kNB + m1], (q < nbk) ? Bm[r1 * S + kb + q] : 0.0, xv[u]);
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      int w = tid + kNT * u, r1 = w / kNB, m1 = w % kNB;
      if (r1 < rows && m1 < nbk) Bm[r1 * S + kb + m1] = xv[u];
    }
    __syncthreads();
    if (ti < kb) {
      double lcol[kNB];
#pragma unroll
      for (int m = 0; m < kNB; ++m) lcol[m] = (m < nbk) ? Lf[(kb + m) * S + ti] : 0.0;
      for (int r = tr; r < rows; r += kNT / 128) {
        double acc = Bm[r * S + ti];
        const double *x = Bm + r * S + kb;
#pragma unroll
        for (int m = 0; m < kNB; ++m) acc = fma(-lcol[m], (m < nbk) ? x[m] : 0.0, acc);
        Bm[r * S + ti] = acc;
      }
    }
    __syncthreads();
  }
  for (int e = tid; e < rows * S; e += kNT) Gout[(row0 + e / S) * S + e % S] = Bm[e];
}

size_t chol_solve_smem(int S) {
  return sizeof(double) * ((size_t)((S * S + 3) & ~3) + (size_t)kSolveChunk * S + 2 * (size_t)S * kNB +
                           (size_t)(S / kNB + 1) * kNB * kNB);
}

void launch_chol_solve(const double *Q, int S, const double *P, int64_t I, double *Gout, int *info, cudaStream_t s) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_chol_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr_set = true;
  }
  k_chol_solve<<<(unsigned)cdiv(I, kSolveChunk), kNT, chol_solve_smem(S), s>>>(Q, S, P, I, Gout, info);
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
