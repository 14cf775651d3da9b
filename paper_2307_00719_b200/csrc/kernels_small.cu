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
// G = P Q^{-1} for SPD Q (S x S, S <= 128) and I right-hand-side rows P (I x S), row-major.
// Blocked right-looking Cholesky (block 8) on the shared-memory copy of Q, written as compact
// loops (the code must stay small: the kernel runs one CTA and is latency/I-cache bound):
//   B-phase: one thread per row i >= kb factors the 8x8 diagonal block in registers
//            (rsqrt pivots), solves its row of the panel and (rows in the block) emits one
//            column of the inverted diagonal block;
//   C-phase: warps own rows, lanes own columns: the panel is finalized and the trailing
//            entries take the rank-8 update.
// Forward / backward substitution then use the inverted diagonal blocks.  Each CTA factors Q
// (cheap, redundant) and solves a chunk of <= 16 RHS rows.  A non-positive pivot sets *info.
constexpr int kNB = 8, kNT = 512, kSolveChunk = 4;    // RHS rows per CTA (the factorization is repeated per CTA)
#ifdef STR_CHOL_PROBE
__device__ long long *g_probe = nullptr;
#endif

__global__ void __launch_bounds__(kNT, 1) k_chol_solve(const double *__restrict__ Q, int S,
                                                        const double *__restrict__ P, int64_t I,
                                                        double *__restrict__ Gout, int *info) {
  extern __shared__ double sm[];
  const int LD = S + 1;                      // padded row stride of A
  const int nblk = (S + kNB - 1) / kNB;
  double *A = sm;                            // S x LD
  double *Bm = A + ((S * LD + 3) & ~3);      // kSolveChunk x LD (RHS rows)
  double *LnT = Bm + ((kSolveChunk * LD + 3) & ~3);   // 8 x S panel of L, m-major
  double *Ln = LnT + ((kNB * S + 3) & ~3);            // S x 8 panel of L, row-major
  double *Di = Ln + kNB * S;                          // nblk x 64 inverted diagonal blocks (zero padded)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = kNT / 32;
  const int64_t row0 = (int64_t)blockIdx.x * kSolveChunk;
  const int rows = (int)((I - row0) < kSolveChunk ? (I - row0) : kSolveChunk);
#ifdef STR_CHOL_PROBE
  long long t_start = clock64();
#endif
  for (int e = tid; e < S * S; e += kNT) A[(e / S) * LD + e % S] = Q[e];
  for (int e = tid; e < rows * S; e += kNT) Bm[(e / S) * LD + e % S] = P[(row0 + e / S) * S + e % S];
  for (int e = tid; e < nblk * kNB * kNB; e += kNT) Di[e] = 0.0;
  __syncthreads();
#ifdef STR_CHOL_PROBE
  long long t_loaded = clock64();
  long long tB = 0, tC = 0;
#endif
  bool bad = false;
  for (int kb = 0; kb < S; kb += kNB) {
    const int nbk = (S - kb) < kNB ? (S - kb) : kNB;
#ifdef STR_CHOL_PROBE
    long long t0 = clock64();
#endif
    if (tid < S - kb) {
      const int i = kb + tid;
      double Ld[kNB][kNB], rd[kNB], l[kNB];
#pragma unroll
      for (int a = 0; a < kNB; ++a)
#pragma unroll
        for (int b = 0; b <= a; ++b) Ld[a][b] = (a < nbk) ? A[(kb + a) * LD + kb + b] : 0.0;
#pragma unroll
      for (int c = 0; c < kNB; ++c) {
        double d = Ld[c][c], r = 0.0;
        if (c < nbk) {
          if (!(d > 0.0)) bad = true;
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
      const int c = i - kb;                    // < nbk for rows inside the diagonal block
#pragma unroll
      for (int m = 0; m < kNB; ++m) {
        double a = (m < nbk && m <= c) ? A[i * LD + kb + m] : 0.0;
#pragma unroll
        for (int q = 0; q < m; ++q) a = fma(-l[q], Ld[m][q], a);
        l[m] = (m <= c) ? a * rd[m] : 0.0;
      }
#pragma unroll
      for (int m = 0; m < kNB; ++m) LnT[m * S + i] = l[m];
      double4 *lr = (double4 *)(Ln + i * kNB);
      lr[0] = make_double4(l[0], l[1], l[2], l[3]);
      lr[1] = make_double4(l[4], l[5], l[6], l[7]);
      if (c < nbk) {
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
      }
    }
    __syncthreads();
#ifdef STR_CHOL_PROBE
    long long t1 = clock64();
    tB += t1 - t0;
#endif
    // panel write-back, then rank-8 update of the trailing lower triangle: a warp task is a strip
    // of up to 8 rows x 32 columns; lane j keeps y = L[j][kb..kb+7] in registers and reads the
    // row values x = L[i][kb..kb+7] as broadcasts from the row-major copy Ln.
    for (int e = tid; e < (S - kb) * nbk; e += kNT) {
      const int i = kb + e / nbk, m = e % nbk;
      A[i * LD + kb + m] = LnT[m * S + i];
    }
    {
      const int j0 = kb + nbk;
      const int nch = (S - j0 + 31) / 32;
      const int nrg = (S - j0 + 7) / 8;
      for (int task = warp; task < nch * nrg; task += nw) {
        const int ch = task % nch, rg = task / nch;
        const int j = j0 + ch * 32 + lane;
        const int ib = j0 + rg * 8;
        if (ib + 7 < j0 + ch * 32) continue;               // strip entirely above the diagonal
        double y[kNB];
#pragma unroll
        for (int m = 0; m < kNB; ++m) y[m] = (j < S && m < nbk) ? LnT[m * S + j] : 0.0;
        // two groups of 4 rows: all shared loads of a group are issued before its stores
#pragma unroll
        for (int g4 = 0; g4 < 8; g4 += 4) {
          double4 xa[4][2];
          double av[4];
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            const int i = ib + g4 + a;
            const bool ok = i < S;
            const double4 *xr = (const double4 *)(Ln + (ok ? i : kb) * kNB);
            xa[a][0] = xr[0];
            xa[a][1] = xr[1];
            av[a] = (ok && j <= i) ? A[i * LD + j] : 0.0;
          }
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            const int i = ib + g4 + a;
            double acc0 = av[a], acc1 = 0.0;
            acc0 = fma(-xa[a][0].x, y[0], acc0);
            acc1 = fma(-xa[a][0].y, y[1], acc1);
            acc0 = fma(-xa[a][0].z, y[2], acc0);
            acc1 = fma(-xa[a][0].w, y[3], acc1);
            acc0 = fma(-xa[a][1].x, y[4], acc0);
            acc1 = fma(-xa[a][1].y, y[5], acc1);
            acc0 = fma(-xa[a][1].z, y[6], acc0);
            acc1 = fma(-xa[a][1].w, y[7], acc1);
            if (i < S && j <= i) A[i * LD + j] = acc0 + acc1;
          }
        }
      }
    }
    __syncthreads();
#ifdef STR_CHOL_PROBE
    tC += clock64() - t1;
#endif
  }
  if (bad && info) atomicExch(info, 1);
#ifdef STR_CHOL_PROBE
  long long t_fact = clock64();
#endif
  // forward substitution L y = b (rows of Bm hold b^T), then backward L^T x = y, block by block:
  // (1) threads (r, m) form y_blk = Dinv b_blk, (2) store, (3) threads (i, r) take the rank-8 update.
  const int ti = tid & 127, tr = tid >> 7;
  for (int pass = 0; pass < 2; ++pass) {
    for (int bb = 0; bb < nblk; ++bb) {
      const int bi = pass == 0 ? bb : nblk - 1 - bb;
      const int kb = bi * kNB;
      const int nbk = (S - kb) < kNB ? (S - kb) : kNB;
      const double *D = Di + bi * kNB * kNB;
      const int r1 = tid >> 3, m1 = tid & 7;
      const bool act = (r1 < rows) && (m1 < nbk);
      double v0 = 0.0, v1 = 0.0;
      if (act) {
#pragma unroll
        for (int q = 0; q < kNB; q += 2) {
          const double d0 = pass == 0 ? D[m1 * kNB + q] : D[q * kNB + m1];
          const double d1 = pass == 0 ? D[m1 * kNB + q + 1] : D[(q + 1) * kNB + m1];
          v0 = fma(d0, (q < nbk) ? Bm[r1 * LD + kb + q] : 0.0, v0);
          v1 = fma(d1, (q + 1 < nbk) ? Bm[r1 * LD + kb + q + 1] : 0.0, v1);
        }
      }
      __syncthreads();
      if (act) Bm[r1 * LD + kb + m1] = v0 + v1;
      __syncthreads();
      const bool upd = ti < S && (pass == 0 ? (ti >= kb + nbk) : (ti < kb));
      if (upd) {
        double lv[kNB];
#pragma unroll
        for (int m = 0; m < kNB; ++m)
          lv[m] = (m < nbk) ? (pass == 0 ? A[ti * LD + kb + m] : A[(kb + m) * LD + ti]) : 0.0;
        for (int r = tr; r < rows; r += kNT / 128) {
          const double *yb = Bm + r * LD + kb;
          double acc0 = Bm[r * LD + ti], acc1 = 0.0;
#pragma unroll
          for (int m = 0; m < kNB; m += 2) {
            acc0 = fma(-lv[m], (m < nbk) ? yb[m] : 0.0, acc0);
            acc1 = fma(-lv[m + 1], (m + 1 < nbk) ? yb[m + 1] : 0.0, acc1);
          }
          Bm[r * LD + ti] = acc0 + acc1;
        }
      }
      __syncthreads();
    }
  }
  for (int e = tid; e < rows * S; e += kNT) Gout[(row0 + e / S) * S + e % S] = Bm[(e / S) * LD + e % S];
#ifdef STR_CHOL_PROBE
  if (tid == 0 && blockIdx.x == 0 && g_probe) {
    g_probe[0] = t_loaded - t_start; g_probe[1] = tB; g_probe[2] = tC; g_probe[3] = clock64() - t_fact;
  }
#endif
}

size_t chol_solve_smem(int S) {
  const int nblk = (S + kNB - 1) / kNB;
  return sizeof(double) * ((size_t)((S * (S + 1) + 3) & ~3) + (size_t)((kSolveChunk * (S + 1) + 3) & ~3) +
                           (size_t)((S * kNB + 3) & ~3) + (size_t)S * kNB + (size_t)nblk * kNB * kNB);
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
