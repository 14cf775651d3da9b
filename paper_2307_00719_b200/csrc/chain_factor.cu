// chain_factor.cu — Q^{-1} of the SPD normal-equation matrices (the "^{-1}" of G_n(2) = P_n Q_n^{-1},
// Alg. 4 l.17 P:379, and of the temporal solve l.9 P:370) by a block Cholesky factorization on one
// SM (one CTA: the matrix and every intermediate stay in its shared memory).
//
// Block Cholesky with 8 x 8 pivot blocks (no pivoting: Q is SPD).  With A^(0) = sym(Q) = (Q + Q^T)/2
// (reading R5), step p:
//   L_pp L_pp^T = A_pp^(p),  T_p = L_pp^{-1}            (one warp, in registers)
//   L_ip = A_ip^(p) T_p^T                               (i > p)
//   A_ij^(p+1) = A_ij^(p) - L_ip L_jp^T                 (p < j <= i)
// so sym(Q) = L L^T.  V = L^{-1} (block lower) follows row block by row block one step behind,
//   V_pp = T_p,   V_pk = -T_p sum_{k<=m<p} L_pm V_mk,
// and Q^{-1} = V^T V.  (The square-root form keeps the multipliers L_ip bounded by ||A||^{1/2}; a block
// LDL^T with explicitly inverted pivot blocks, W_ip = A_ip D_p^{-1}, is not stable at cond 1e8.)
//
// Schedule (one CTA, 256 threads).  The matrix lives in shared memory (lower tiles: A, then L in
// place; upper tiles: V^T; T_p in a panel); warp 0 is the pivot warp — after the panel of step p it
// updates the next pivot block and factors it at once (look-ahead), while warps 1-7 apply the trailing
// update of step p and form V's row block p.  Two CTA barriers per step; the latency floor is the
// chain of 8 dependent pivots per block.  Then the CTA assembles Q^{-1} = V^T V from shared memory.
// The code is kept compact (rolled pivot loop, one copy of the 8 x 8 factorization): the kernel is
// latency-bound, and on a cold SM every 128-byte line of straight-line code costs an L2 round trip.
// A non-positive (or NaN) pivot sets *info = 1.
#include <cuda_runtime.h>

#include "common.cuh"
#include "dmma.cuh"
#include "kernels.h"

namespace strb200 {

#ifdef FC_PROBE
__device__ long long g_fc_probe[64];
#define FCP(i)                                         \
  do {                                                 \
    if (threadIdx.x == 0) g_fc_probe[(i)] = clock64(); \
  } while (0)
#else
#define FCP(i) \
  do {         \
  } while (0)
#endif

constexpr int kFcThreads = 256;
constexpr int kPL = 12;    // leading dimension of 8-wide panels (T blocks, the L panel, scratch): conflict-free

// 1/sqrt(x) to full double precision: hardware approximation + two Newton steps
__device__ __forceinline__ double rsqrt_full(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);
  y = y * fma(-hx * y, y, 1.5);
  return y;
}

// Cholesky factor and its inverse of the SPD 8 x 8 block M (shared memory, row-major, leading
// dimension ldm; the lower triangle is read) in ONE thread's registers: M = L L^T, T = L^{-1}
// (written lower-triangular, zeros above, to Tout with leading dimension kPL).  No shuffles on the
// pivot chain: per pivot one full-precision reciprocal square root and one dependent update; the
// inverse rows are independent FMA chains the scheduler interleaves with the later pivots.  A
// non-positive or NaN pivot sets bad.
__device__ __noinline__ void chol8_inv1(const double *M, int ldm, double *Tout, bool &bad) {
  double a[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j <= i; ++j) a[i][j] = M[i * ldm + j];
  double r[8];
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    const double piv = a[m][m];
    bad = bad || !(piv > 0.0);
    r[m] = rsqrt_full(piv);
#pragma unroll
    for (int i = m + 1; i < 8; ++i) a[i][m] *= r[m];   // column m of L
#pragma unroll
    for (int i = m + 1; i < 8; ++i)
#pragma unroll
      for (int j = m + 1; j <= i; ++j) a[i][j] = fma(-a[i][m], a[j][m], a[i][j]);
  }
  // T = L^{-1}: T[i][i] = r_i, T[i][j] = -r_i sum_{j<=k<i} L[i][k] T[k][j]
  double tt[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    tt[i][i] = r[i];
#pragma unroll
    for (int j = 0; j < i; ++j) {
      double s = 0.0;
#pragma unroll
      for (int k = j; k < i; ++k) s = fma(a[i][k], tt[k][j], s);
      tt[i][j] = -r[i] * s;
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) Tout[i * kPL + j] = (j <= i) ? tt[i][j] : 0.0;
}

// Block Cholesky of sym(Q) (S x S, row-major, global) on one CTA, V = L^{-1} alongside, and
// Q^{-1} = V^T V (S x S, row-major, global).  Shared memory: fc_smem_bytes.  Returns bad.
__device__ bool cta_bchol_inv(const double *__restrict__ Q, int S, double *sm, double *__restrict__ Qinv) {
  const int nt = (S + 7) >> 3, Sp = nt * 8, LD = ld_frag(Sp);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  double *As = sm;                    // [Sp][LD]
  double *Ds = As + Sp * LD;          // [nt][8][kPL]  T_p = L_pp^{-1}
  double *Wp0 = Ds + nt * 8 * kPL;    // [2][Sp][kPL]  panel L_ip of step p (double-buffered by parity:
                                      // step p+1's panel is written while step p's is still copied)
  double *Xs = Wp0 + 2 * Sp * kPL;    // [8 warps][8][kPL] scratch
  FCP(0);
  // Q rows into shared memory (coalesced; 16-byte copies when the rows allow), then
  // sym(Q) = (Q + Q^T)/2 into the lower tiles (diagonal tiles in full), identity padding beyond S
  if ((S & 1) == 0 && ((uintptr_t)Q & 15) == 0) {
    const int h2 = S >> 1;
    for (int e = threadIdx.x; e < S * h2; e += kFcThreads) {
      const int i = e / h2, j = 2 * (e - i * h2);
      cpa16cg(As + i * LD + j, Q + (int64_t)i * S + j);
    }
  } else {
    for (int e = threadIdx.x; e < S * S; e += kFcThreads) {
      const int i = e / S, j = e - (e / S) * S;
      cpa8(As + i * LD + j, Q + e);
    }
  }
  cpa_commit();
  cpa_wait<0>();
  __syncthreads();
  {
    // lower tile (ti, tj) per warp iteration; lane -> 2 elements (a, b), (a + 4, b) of the tile
    const int ntl = nt * (nt + 1) / 2;
    for (int e = warp; e < ntl; e += kFcThreads / 32) {
      int ti = (int)((sqrtf(8.0f * (float)e + 1.0f) - 1.0f) * 0.5f);
      while ((ti + 1) * (ti + 2) / 2 <= e) ++ti;
      while (ti * (ti + 1) / 2 > e) --ti;
      const int tj = e - ti * (ti + 1) / 2;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int a = (lane >> 3) + 4 * h, b = lane & 7;
        const int i = 8 * ti + a, j = 8 * tj + b;
        if (ti == tj && j > i) continue;
        double v;
        if (i < S && j < S) v = 0.5 * (As[i * LD + j] + As[j * LD + i]);
        else v = (i == j) ? 1.0 : 0.0;
        As[i * LD + j] = v;
        if (ti == tj) As[j * LD + i] = v;
      }
    }
  }
  __syncthreads();
  FCP(1);
  bool bad = false;
  if (threadIdx.x == 0) chol8_inv1(As, LD, Ds, bad);
  FCP(40);
  __syncthreads();
  FCP(41);
  for (int p = 0; p < nt; ++p) {
    const double *Tp = Ds + p * 8 * kPL;
    double *Wp = Wp0 + (p & 1) * Sp * kPL;
    // (alpha) panel L_ip = A_ip T_p^T, i > p (warp 0 takes the next pivot row block)
    {
      const int first = (warp == 0) ? p + 1 : p + 2 + (warp - 1);
      const int step = (warp == 0) ? nt : 7;
      for (int i = first; i < nt; i += step) {
        double c[2] = {0.0, 0.0};
        dmma8_tn(c, As + (8 * i) * LD + 8 * p, LD, Tp, kPL, g, t);
        frag_store(c, Wp + 8 * i * kPL, kPL, g, t);
      }
    }
    if (p == 0) FCP(42);
    __syncthreads();
    if (p == 0) FCP(43);
    if (warp == 0) {
      // (beta, pivot warp) A_{p+1,p+1} -= L_{p+1,p} L_{p+1,p}^T, then factor it (look-ahead)
      if (p + 1 < nt) {
        const int q = p + 1;
        double c[2];
        frag_load(c, As + (8 * q) * LD + 8 * q, LD, g, t);
        const double *pw = Wp + 8 * q * kPL;
        dmma(c[0], c[1], -pw[g * kPL + t], pw[g * kPL + t]);
        dmma(c[0], c[1], -pw[g * kPL + 4 + t], pw[g * kPL + 4 + t]);
        frag_store(c, As + (8 * q) * LD + 8 * q, LD, g, t);
        __syncwarp();
        if (lane == 0) chol8_inv1(As + (8 * q) * LD + 8 * q, LD, Ds + q * 8 * kPL, bad);
        __syncwarp();
      }
    } else {
      // (beta, workers) trailing update A_ij -= L_ip L_jp^T, p < j <= i, except (p+1, p+1)
      const int m = nt - 1 - p;
      const int npairs = m * (m + 1) / 2;
      for (int e = warp - 1; e < npairs; e += 7) {
        int ii = (int)((sqrtf(8.0f * (float)e + 1.0f) - 1.0f) * 0.5f);
        while ((ii + 1) * (ii + 2) / 2 <= e) ++ii;
        while (ii * (ii + 1) / 2 > e) --ii;
        const int jj = e - ii * (ii + 1) / 2;
        const int i = p + 1 + ii, j = p + 1 + jj;
        if (i == p + 1 && j == p + 1) continue;
        double c[2];
        frag_load(c, As + (8 * i) * LD + 8 * j, LD, g, t);
        const double *pa = Wp + 8 * i * kPL, *pb = Wp + 8 * j * kPL;
        dmma(c[0], c[1], -pa[g * kPL + t], pb[g * kPL + t]);
        dmma(c[0], c[1], -pa[g * kPL + 4 + t], pb[g * kPL + 4 + t]);
        frag_store(c, As + (8 * i) * LD + 8 * j, LD, g, t);
      }
      // (beta, workers) V row block p: V_pk = -T_p sum_{k<=m<p} L_pm V_mk (V_kk = T_k), stored
      // transposed in the upper tile (k, p): As[8k + a][8p + b] = V[8p + b][8k + a]
      double *xs = Xs + warp * 8 * kPL;
      for (int k = warp - 1; k < p; k += 7) {
        double c[2] = {0.0, 0.0};
        dmma8_nn(c, As + (8 * p) * LD + 8 * k, LD, Ds + k * 8 * kPL, kPL, g, t);   // L_pk T_k
        for (int mm = k + 1; mm < p; ++mm)   // L_pm V_mk, V_mk[kk][n] = As[8k + n][8mm + kk]
          dmma8_tn(c, As + (8 * p) * LD + 8 * mm, LD, As + (8 * k) * LD + 8 * mm, LD, g, t);
        frag_store(c, xs, kPL, g, t);
        __syncwarp();
        double v[2] = {0.0, 0.0};
        dmma8_nn(v, Tp, kPL, xs, kPL, g, t);
        __syncwarp();
#pragma unroll
        for (int e2 = 0; e2 < 2; ++e2) As[(8 * k + 2 * t + e2) * LD + 8 * p + g] = -v[e2];
      }
    }
    __syncthreads();
    FCP(4 + p);
    // (gamma) L_ip replaces A_ip; the next alpha reads column p+1 only
    for (int e = threadIdx.x; e < (nt - 1 - p) * 64; e += kFcThreads) {
      const int i = 8 * (p + 1) + (e >> 3), b = e & 7;
      As[i * LD + 8 * p + b] = Wp[i * kPL + b];
    }
  }
  __syncthreads();
  FCP(2);
  // Q^{-1} = V^T V, tile (r, c), r <= c: sum_{b >= c} V_br^T V_bc, with V_bb = T_b (Ds) and, for b > k,
  // V_bk stored transposed in the upper tile (k, b): V_bk[kk][n] = As[8k + n][8b + kk].  A warp owns a
  // column tile c and keeps the accumulators of every r <= c (independent DMMA chains).
  for (int c = warp; c < nt; c += kFcThreads / 32) {
    double acc[16][2];
#pragma unroll
    for (int r = 0; r < 16; ++r) acc[r][0] = acc[r][1] = 0.0;
    // b = c: r < c: V_cr^T T_c (V_cr^T rows at As[8r][8c]); r = c: T_c^T T_c
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      if (r < c) dmma8_nn(acc[r], As + (8 * r) * LD + 8 * c, LD, Ds + c * 8 * kPL, kPL, g, t);
      else if (r == c) dmma8_tnn(acc[r], Ds + r * 8 * kPL, kPL, Ds + c * 8 * kPL, kPL, g, t);
    }
    for (int bb = c + 1; bb < nt; ++bb) {   // B = V_bc (transposed rows As[8c][8bb]), fragments reused over r
      const double *pb = As + (8 * c) * LD + 8 * bb;
      const double b0 = pb[g * LD + t], b1 = pb[g * LD + 4 + t];
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        if (r <= c) {
          const double *pa = As + (8 * r) * LD + 8 * bb;   // A = V_br^T rows
          dmma(acc[r][0], acc[r][1], pa[g * LD + t], b0);
          dmma(acc[r][0], acc[r][1], pa[g * LD + 4 + t], b1);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      if (r > c) continue;
      const int row = 8 * r + g;
#pragma unroll
      for (int e2 = 0; e2 < 2; ++e2) {
        const int col = 8 * c + 2 * t + e2;
        if (row < S && col < S) {
          Qinv[(int64_t)row * S + col] = acc[r][e2];
          if (r != c) Qinv[(int64_t)col * S + row] = acc[r][e2];
        }
      }
    }
  }
  FCP(3);
  return bad;
}

size_t fc_smem_bytes(int S) {
  const int nt = (S + 7) / 8, Sp = 8 * nt;
  return sizeof(double) * ((size_t)Sp * ld_frag(Sp) + (size_t)(nt * 8 + 2 * Sp + 64) * kPL);
}

// Q^{-1} for one SPD matrix (S <= STR_MAXW) on one CTA.
__global__ void __launch_bounds__(kFcThreads, 1)
    k_spd_inv_chol(const double *__restrict__ Q, int S, double *__restrict__ Qinv, int *info) {
  PDL_PROLOGUE();
  extern __shared__ __align__(16) double fsm[];
  const bool bad = cta_bchol_inv(Q, S, fsm, Qinv);
  if (bad && threadIdx.x == 0 && info) atomicExch(info, 1);
}

size_t spd_inv_ws_doubles(int S) {
  const int nt = (S + 7) / 8, Sp = 8 * nt;
  (void)nt;
  return (size_t)Sp * Sp;
}

void launch_spd_inv_chol(const double *Q, int S, double *Qinv, double *ws, int *info, cudaStream_t s) {
  static PerDeviceOnce once;
  once_per_device(once, [] {
    cudaFuncSetAttribute(k_spd_inv_chol, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fc_smem_bytes(STR_MAXW));
    prefer_max_smem(k_spd_inv_chol);
  });
  (void)ws;
  pdl_launch(kPdlInv, k_spd_inv_chol, dim3(1), dim3(kFcThreads), fc_smem_bytes(S), s, Q, S, Qinv, info);
}

}  // namespace strb200
