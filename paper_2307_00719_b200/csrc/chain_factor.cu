// chain_factor.cu — Q^{-1} of the SPD normal-equation matrices (the "^{-1}" of G_n(2) = P_n Q_n^{-1},
// Alg. 4 l.17 P:379, and of the temporal solve l.9 P:370) by a block Cholesky factorization on one
// SM plus a cluster-wide assembly of the inverse.
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
// Schedule (one cluster of kFcCS CTAs, 256 threads each).  CTA 0 factors: the matrix lives in shared
// memory (lower tiles: A, then L in place; upper tiles: V^T); warp 0 is the pivot warp — after the
// panel of step p it updates the next pivot block and factors it at once (look-ahead), while warps
// 1-7 apply the trailing update of step p and form V's row block p.  Two CTA barriers per step; the
// latency floor is the chain of 8 dependent pivots per block.  Then V goes to global memory and every
// CTA of the cluster assembles row tiles of Q^{-1} = V^T V.  A non-positive (or NaN) pivot sets
// *info = 1.
#include <cuda_runtime.h>

#include "common.cuh"
#include "dmma.cuh"
#include "kernels.h"

namespace strb200 {

constexpr int kFcThreads = 256;
constexpr int kFcCS = kInvClusterCTAs;   // CTAs per cluster (the SMs the contraction's persistent grid leaves free)
constexpr int kPL = 12;    // leading dimension of 8-wide panels (T blocks, the L panel, scratch): conflict-free

// Cholesky factor and its inverse of the SPD 8 x 8 block M held by one warp in accumulator layout
// (lane (g, t) holds M[g][2t], M[g][2t+1]): on return the lane holds T[g][2t], T[g][2t+1] with
// T = L^{-1}, M = L L^T (T lower triangular).  A non-positive or NaN pivot sets bad.
__device__ __forceinline__ void chol8_inv(double (&d)[2], int g, int t, bool &bad) {
  double rdg = 0.0;   // 1 / L[g][g]
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    const int src = m >> 1;
    const double piv = __shfl_sync(0xffffffffu, d[m & 1], m * 4 + src);
    const double cg = __shfl_sync(0xffffffffu, d[m & 1], g * 4 + src);
    const double c0 = __shfl_sync(0xffffffffu, d[m & 1], (2 * t) * 4 + src);
    const double c1 = __shfl_sync(0xffffffffu, d[m & 1], (2 * t + 1) * 4 + src);
    bad = bad || !(piv > 0.0);
    const double r = rsqrt(piv);   // 1 / L[m][m]
    const double lg = cg * r;       // L[g][m]
    if (g == m) rdg = r;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int j = 2 * t + e;
      if (j == m) d[e] = (g >= m) ? lg : 0.0;
      else if (j > m) d[e] = (g > m) ? fma(-lg, (e ? c1 : c0) * r, d[e]) : 0.0;
    }
  }
  // T = L^{-1} row by row: T[g][c] = (delta_gc - sum_{k<g} L[g][k] T[k][c]) / L[g][g]; the sum is
  // accumulated as the rows k are finalized (row k broadcast to the lanes of the same column pair)
  double Lrow[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) Lrow[k] = __shfl_sync(0xffffffffu, d[k & 1], g * 4 + (k >> 1));
  double acc0 = 0.0, acc1 = 0.0, T0 = 0.0, T1 = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const double t0 = ((2 * t == k ? 1.0 : 0.0) + acc0) * rdg;
    const double t1 = ((2 * t + 1 == k ? 1.0 : 0.0) + acc1) * rdg;
    if (g == k) {
      T0 = t0;
      T1 = t1;
    }
    const double b0 = __shfl_sync(0xffffffffu, t0, k * 4 + t);
    const double b1 = __shfl_sync(0xffffffffu, t1, k * 4 + t);
    acc0 = fma(-Lrow[k], b0, acc0);
    acc1 = fma(-Lrow[k], b1, acc1);
  }
  d[0] = T0;
  d[1] = T1;
}

// Block Cholesky of sym(Q) (S x S, row-major, global) on one CTA; writes V = L^{-1} (Sp x Sp dense,
// row-major, lower, zero above) to Vg.  Shared memory: fc_smem_bytes.  Returns bad.
__device__ bool cta_bchol(const double *__restrict__ Q, int S, double *sm, double *__restrict__ Vg) {
  const int nt = (S + 7) >> 3, Sp = nt * 8, LD = ld_frag(Sp);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  double *As = sm;                    // [Sp][LD]
  double *Ds = As + Sp * LD;          // [nt][8][kPL]  T_p = L_pp^{-1}
  double *Wp = Ds + nt * 8 * kPL;     // [Sp][kPL]     panel L_ip of the current step
  double *Xs = Wp + Sp * kPL;         // [8 warps][8][kPL] scratch
  // sym(Q) into the lower tiles (diagonal tiles in full), identity padding beyond S
  for (int e = threadIdx.x; e < Sp * Sp; e += kFcThreads) {
    const int i = e / Sp, j = e - (e / Sp) * Sp;
    if ((j >> 3) > (i >> 3)) continue;
    double v;
    if (i < S && j < S) v = 0.5 * (Q[(int64_t)i * S + j] + Q[(int64_t)j * S + i]);
    else v = (i == j) ? 1.0 : 0.0;
    As[i * LD + j] = v;
  }
  __syncthreads();
  bool bad = false;
  if (warp == 0) {
    double d[2];
    frag_load(d, As, LD, g, t);
    chol8_inv(d, g, t, bad);
    frag_store(d, Ds, kPL, g, t);
  }
  __syncthreads();
  for (int p = 0; p < nt; ++p) {
    const double *Tp = Ds + p * 8 * kPL;
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
    __syncthreads();
    if (warp == 0) {
      // (beta, pivot warp) A_{p+1,p+1} -= L_{p+1,p} L_{p+1,p}^T, then factor it (look-ahead)
      if (p + 1 < nt) {
        const int q = p + 1;
        double c[2];
        frag_load(c, As + (8 * q) * LD + 8 * q, LD, g, t);
        const double *pw = Wp + 8 * q * kPL;
        dmma(c[0], c[1], -pw[g * kPL + t], pw[g * kPL + t]);
        dmma(c[0], c[1], -pw[g * kPL + 4 + t], pw[g * kPL + 4 + t]);
        chol8_inv(c, g, t, bad);
        frag_store(c, Ds + q * 8 * kPL, kPL, g, t);
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
    // (gamma) L_ip replaces A_ip; the next alpha reads column p+1 only
    for (int e = threadIdx.x; e < (nt - 1 - p) * 64; e += kFcThreads) {
      const int i = 8 * (p + 1) + (e >> 3), b = e & 7;
      As[i * LD + 8 * p + b] = Wp[i * kPL + b];
    }
  }
  __syncthreads();
  // V (dense, lower) to global memory: off-diagonal blocks from the upper tiles, T_p on the diagonal
  for (int e = threadIdx.x; e < Sp * Sp; e += kFcThreads) {
    const int i = e / Sp, j = e - (e / Sp) * Sp;
    double v;
    if ((j >> 3) < (i >> 3)) v = As[j * LD + i];
    else if ((j >> 3) == (i >> 3) && j <= i) v = Ds[(i >> 3) * 8 * kPL + (i & 7) * kPL + (j & 7)];
    else v = 0.0;
    Vg[e] = v;
  }
  return bad;
}

size_t fc_smem_bytes(int S) {
  const int nt = (S + 7) / 8, Sp = 8 * nt;
  const size_t bldl = (size_t)Sp * ld_frag(Sp) + (size_t)(nt * 8 + Sp + 64) * kPL;
  const size_t qinv = (size_t)Sp * ld_frag(Sp);
  return sizeof(double) * (bldl > qinv ? bldl : qinv);
}

// Row tiles r (of 8) of Q^{-1} = V^T V: (Q^{-1})_rc = sum_{b >= max(r,c)} V_br^T V_bc, V staged whole.
__device__ void cta_qinv(const double *__restrict__ Vg, int S, int rank, int ncta, double *sm,
                         double *__restrict__ Qinv) {
  const int nt = (S + 7) >> 3, Sp = nt * 8, LD = ld_frag(Sp);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  if (rank >= nt) return;
  double *Vs = sm;   // [Sp][LD]
  for (int e = threadIdx.x; e < Sp * (Sp / 2); e += kFcThreads) {
    const int i = e / (Sp / 2), j2 = 2 * (e - i * (Sp / 2));
    cpa16cg(Vs + i * LD + j2, Vg + (int64_t)i * Sp + j2);
  }
  cpa_commit();
  cpa_wait<0>();
  __syncthreads();
  for (int r = rank; r < nt; r += ncta) {
    for (int c0 = warp; c0 < nt; c0 += 8) {
      double c[2] = {0.0, 0.0};
      const int b0 = r > c0 ? r : c0;
      for (int b = b0; b < nt; ++b)   // A = V_br^T (rows of V at 8b, columns 8r..), B = V_bc rows
        dmma8_tnn(c, Vs + (8 * b) * LD + 8 * r, LD, Vs + (8 * b) * LD + 8 * c0, LD, g, t);
      const int row = 8 * r + g;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = 8 * c0 + 2 * t + e;
        if (row < S && col < S) Qinv[(int64_t)row * S + col] = c[e];
      }
    }
  }
}

// Q^{-1} for one SPD matrix (S <= STR_MAXW): CTA 0 factors, the cluster assembles.
__global__ void __cluster_dims__(kFcCS, 1, 1) __launch_bounds__(kFcThreads, 1)
    k_spd_inv_chol(const double *__restrict__ Q, int S, double *__restrict__ Qinv, double *__restrict__ ws,
                   int *info) {
  PDL_PROLOGUE();
  extern __shared__ __align__(16) double fsm[];
  const uint32_t rank = cluster_rank();
  if (rank == 0) {
    const bool bad = cta_bchol(Q, S, fsm, ws);
    if (bad && threadIdx.x == 0 && info) atomicExch(info, 1);
  }
  cluster_sync_all();   // V in global memory, visible to the cluster
  cta_qinv(ws, S, (int)rank, kFcCS, fsm, Qinv);
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
  pdl_launch(kPdlInv, k_spd_inv_chol, dim3(kFcCS), dim3(kFcThreads), fc_smem_bytes(S), s, Q, S, Qinv, ws, info);
}

}  // namespace strb200
