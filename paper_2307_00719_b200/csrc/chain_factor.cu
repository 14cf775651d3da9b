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
// Schedule (one CTA, kFcThreads = 512 threads).  The matrix lives in shared memory (lower tiles: A, then L in
// place; upper tiles: V^T; T_p in a panel); warp 0 is the pivot warp — after the panel of step p it
// updates the next pivot block and factors it at once (look-ahead), while the worker warps apply the trailing
// update of step p and form V's row block p.  Two CTA barriers per step; the latency floor is the
// chain of 8 dependent pivots per block.  Then the CTA assembles Q^{-1} = V^T V from shared memory.
// The code is kept compact (rolled pivot loop, one copy of the 8 x 8 factorization): the kernel is
// latency-bound, and on a cold SM every 128-byte line of straight-line code costs an L2 round trip.
// A non-positive (or NaN) pivot sets *info = 1.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include <cooperative_groups.h>

#include "common.cuh"
#include "dmma.cuh"
#include "kernels.h"
#include "tc_ptx.cuh"

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

#ifndef FC_THREADS
#define FC_THREADS 512
#endif
constexpr int kFcThreads = FC_THREADS;          // factor CTA: warp 0 pivots, the rest are workers
#ifndef FC_BULK
#define FC_BULK 0
#endif
#ifndef FC_WHATIF
#define FC_WHATIF 0
#endif
#ifndef FC_EXCL
#define FC_EXCL 1
#endif
// With FC_EXCL the pivot warp has its SM sub-partition to itself (warps 4, 8, ... share warp 0's
// scheduler and only join the barriers); the other warps are the workers, numbered wid = 0, 1, ...
constexpr int kFcWarps = kFcThreads / 32;
constexpr int kFcWorkers = FC_EXCL ? kFcWarps - kFcWarps / 4 : kFcWarps - 1;
__device__ __forceinline__ int fc_worker_id(int warp) { return FC_EXCL ? ((warp & 3) ? warp - warp / 4 - 1 : -1) : warp - 1; }
constexpr int kRsThreads = 512;                 // rows-solve CTA (16 warps, one column tile each: S <= 128)
#ifndef FC_SPLIT_MIN_S
#define FC_SPLIT_MIN_S 32
#endif
constexpr int kSplitMinS = FC_SPLIT_MIN_S;      // the two-CTA factor above this S (measured: gains at S = 64 and 100)
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
// dimension ldm; the lower triangle is read): M = L L^T, T = L^{-1} (written lower-triangular, zeros
// above, to Tout with leading dimension kPL).  Called by lanes 0..7 of one warp: every lane runs the
// factorization in its own registers (one instruction stream, broadcast shared-memory reads, no
// shuffles on the pivot chain: per pivot one full-precision reciprocal square root and one dependent
// update), then lane c solves L x = e_c for column c of T — 8 independent forward substitutions in
// parallel instead of the whole triangular inverse in one thread.  Called by a whole warp (lanes
// 8-31 duplicate lanes 0-7 and store nothing).  A non-positive or NaN pivot sets bad (on every lane).
__device__ __noinline__ void chol8_inv8(const double *M, int ldm, double *Tout, bool &bad) {
  const int c = threadIdx.x & 7;
  double a[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j <= i; ++j) a[i][j] = M[i * ldm + j];
  double r[8];
  // pivots in pairs: for the leading 2 x 2 block [[x, y], [y, z]] of the current Schur complement,
  // L = [[sqrt x, 0], [y / sqrt x, sqrt(d / x)]] with d = x z - y^2, so both reciprocal square roots
  // (of x and of d) start together: half the dependent rsqrt latencies of the scalar recursion
#pragma unroll
  for (int m = 0; m < 8; m += 2) {
    const double x = a[m][m], y = a[m + 1][m], z = a[m + 1][m + 1];
    const double d = fma(x, z, -y * y);
    bad = bad || !(x > 0.0) || !(d > 0.0);
    const double rx = rsqrt_full(x), rdd = rsqrt_full(d);
    const double l10 = y * rx;               // L[m+1][m]
    r[m] = rx;                               // 1 / L[m][m]
    r[m + 1] = rdd * (x * rx);               // 1 / L[m+1][m+1] = sqrt(x) / sqrt(d)
#pragma unroll
    for (int i = m + 2; i < 8; ++i) {
      a[i][m] *= rx;                                          // L[i][m]
      a[i][m + 1] = fma(-a[i][m], l10, a[i][m + 1]) * r[m + 1];   // L[i][m+1]
    }
#pragma unroll
    for (int i = m + 2; i < 8; ++i)
#pragma unroll
      for (int j = m + 2; j <= i; ++j)
        a[i][j] = fma(-a[i][m + 1], a[j][m + 1], fma(-a[i][m], a[j][m], a[i][j]));
    a[m + 1][m] = l10;
  }
  // column c of T = L^{-1}: x_i = r_i (delta_ic - sum_{k<i} L[i][k] x_k) (x_i = 0 for i < c); the
  // sum runs k ascending so that x_{i-1}, the latest operand, enters last
  double xv[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    double s = (i == c) ? 1.0 : 0.0;
#pragma unroll
    for (int k = 0; k < i; ++k) s = fma(-a[i][k], xv[k], s);
    xv[i] = s * r[i];
  }
  if ((threadIdx.x & 31) < 8)
#pragma unroll
    for (int i = 0; i < 8; ++i) Tout[i * kPL + c] = xv[i];
}

// st.async of two doubles into another CTA of the cluster (shared::cluster addresses), signalling
// complete_tx on that CTA's mbarrier: the consumer's mbarrier wait then also makes the data visible.
__device__ __forceinline__ void st_async_f64x2(uint32_t raddr, double a, double b, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(raddr),
               "d"(a), "d"(b), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ uint32_t cluster_map_u32(const void *p, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"((uint32_t)__cvta_generic_to_shared(p)), "r"(rank));
  return r;
}

// Block Cholesky of sym(Q) (S x S, row-major, global) on one CTA with V = L^{-1} alongside, written
// to Vout (Sp x Sp, row-major; Sp = S rounded up to 8, identity padding) row block by row block as
// it is formed: only the blocks on and below the block diagonal are written (the diagonal blocks
// T_p are lower triangular with explicit zeros), so Q^{-1} = V^T V.  Shared memory: fc_smem_bytes.
// Returns bad.
__device__ bool cta_bchol(const double *__restrict__ Q, int S, double *sm, double *__restrict__ Vout,
                          uint64_t *vbar = nullptr) {
  const int nt = (S + 7) >> 3, Sp = nt * 8, LD = ld_frag(Sp);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  const int wid = fc_worker_id(warp);
  double *As = sm;                    // [Sp][LD]
  double *Ds = As + Sp * LD;          // [nt][8][kPL]  T_p = L_pp^{-1}
  double *Wp0 = Ds + nt * 8 * kPL;    // [2][Sp][kPL]  panel L_ip of step p (double-buffered by parity:
                                      // step p+1's panel is written while step p's is still copied)
  double *Xs = Wp0 + 2 * Sp * kPL;    // [kFcWarps][8][kPL] scratch
  FCP(0);
  // Q rows into shared memory: one bulk (TMA) copy per row when the rows are 16-byte multiples,
  // else 16- / 8-byte cp.async
#if FC_BULK
  __shared__ __align__(8) uint64_t qbar;
  if ((S & 1) == 0 && ((uintptr_t)Q & 15) == 0) {
    if (threadIdx.x == 0) {
      tc::mbar_init(&qbar, 1);
      tc::fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) tc::mbar_arrive_expect_tx(&qbar, (uint32_t)(S * S * 8));
    __syncthreads();
    if (threadIdx.x < S) tc::bulk_load(As + threadIdx.x * LD, Q + (int64_t)threadIdx.x * S, (uint32_t)(S * 8), &qbar);
    tc::mbar_wait(&qbar, 0);
  } else
#endif
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
  FCP(44);
  // sym(Q) = (Q + Q^T)/2 into the lower tiles (the factorization never reads above the diagonal; the
  // upper halves of the diagonal tiles are zeroed), identity padding beyond S.  One 8 x 8 lower tile
  // per warp iteration, lane (a, b) = (lane / 8, lane % 8) on (8I + a (+4), 8J + b): both the tile
  // and its mirror are read at most two-way bank-conflicted (a row walk would be eight-way).  Every
  // lane reads before any lane of the warp writes (a diagonal tile's upper half is zeroed while its
  // lower half reads it); no other warp touches the tile or its mirror.
#ifdef FC_SYM2   // (probe only: the pass twice, the second timed on warm code; wrong results)
  for (int rep = 0; rep < 2; ++rep) {
    if (rep == 1) {
      __syncthreads();
      FCP(45);
    }
#else
  {
#endif
    const int a0 = lane >> 3, b0 = lane & 7, ntl = nt * (nt + 1) / 2;
    int I = 0, J = warp;   // tile (I, J), J <= I, of the row-major lower enumeration; advanced incrementally
    while (J > I) { J -= I + 1; ++I; }
    for (int tt = warp; tt < ntl; tt += kFcWarps) {
      const int i0 = 8 * I + a0, j = 8 * J + b0;
      // all four reads first (padding rows / columns read whatever is there and are not selected)
      const double x0 = As[i0 * LD + j], y0 = As[j * LD + i0];
      const double x1 = As[(i0 + 4) * LD + j], y1 = As[j * LD + i0 + 4];
      const bool jin = j < S;
      const double v0 = (i0 < S && jin) ? (j <= i0 ? 0.5 * (x0 + y0) : 0.0) : (i0 == j ? 1.0 : 0.0);
      const double v1 = (i0 + 4 < S && jin) ? (j <= i0 + 4 ? 0.5 * (x1 + y1) : 0.0) : (i0 + 4 == j ? 1.0 : 0.0);
      __syncwarp();
      As[i0 * LD + j] = v0;
      As[(i0 + 4) * LD + j] = v1;
      J += kFcWarps;
      while (J > I) { J -= I + 1; ++I; }
    }
  }
  __syncthreads();
  FCP(1);
  bool bad = false;
  // split (vbar: the V CTA's per-step mbarriers): L's column blocks and the T_p go to the same
  // positions of the V CTA's tiles by st.async, step p's bytes counted on its mbarrier vbar[p]
  const bool split = vbar != nullptr;
  if (split) asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");   // (phase 0: its barriers are set up)
  const uint32_t rsm0 = split ? cluster_map_u32(sm, 1) : 0u, rbar0 = split ? cluster_map_u32(vbar, 1) : 0u;
  auto push_t = [&](int q, int step) {   // T_q (the 8 x 8 of its [8][kPL] block, 512 bytes) by one warp
    const int r = lane >> 2, c2 = 2 * (lane & 3);
    const double *src = Ds + q * 8 * kPL + r * kPL + c2;
    st_async_f64x2(rsm0 + (uint32_t)(sizeof(double) * (Sp * LD + q * 8 * kPL + r * kPL + c2)), src[0], src[1],
                   rbar0 + 8u * step);
  };
  if (warp == 0) chol8_inv8(As, LD, Ds, bad);
  if (split && warp == 0) {
    __syncwarp();
    push_t(0, 0);
  }
  FCP(40);
  __syncthreads();
  if (warp == 0)
    for (int e = lane; e < 64; e += 32) Vout[(int64_t)(e >> 3) * Sp + (e & 7)] = Ds[(e >> 3) * kPL + (e & 7)];
  FCP(41);
  // Step p (after the CTA barrier of step p-1):
  //   warp 0   L_{p+1,p} = A_{p+1,p} T_p^T (its own panel row) -> named-barrier arrive -> the pivot
  //            block A_{p+1,p+1} -= L_{p+1,p} L_{p+1,p}^T -> T_{p+1} (lanes 0-7 store)
  //   workers  V_pp = T_p (one warp), copy step p-1's panel into the lower tiles, the rest of the
  //            panel L_ip (i >= p+2), named barrier (the whole panel is there), trailing update,
  //            V's row block p
  //   CTA barrier
  // so the pivot chain (warp 0) never waits for the panel copies or the trailing updates of step p.
  for (int p = 0; p < nt; ++p) {
    const double *Tp = Ds + p * 8 * kPL;
    double *Wp = Wp0 + (p & 1) * Sp * kPL;
    if (warp == 0) {
      if (p + 1 < nt) {
        const int q = p + 1;
        double c[2] = {0.0, 0.0};
        dmma8_tn(c, As + (8 * q) * LD + 8 * p, LD, Tp, kPL, g, t);
        frag_store(c, Wp + 8 * q * kPL, kPL, g, t);
        __syncwarp();
        if (p == 5) FCP(54);
        asm volatile("bar.arrive 1, %0;" ::"n"(kFcThreads) : "memory");
        double d[2];
        frag_load(d, As + (8 * q) * LD + 8 * q, LD, g, t);
        const double *pw = Wp + 8 * q * kPL;
        dmma(d[0], d[1], -pw[g * kPL + t], pw[g * kPL + t]);
        dmma(d[0], d[1], -pw[g * kPL + 4 + t], pw[g * kPL + 4 + t]);
        frag_store(d, As + (8 * q) * LD + 8 * q, LD, g, t);
        __syncwarp();
        if (p == 5) FCP(55);
#if FC_WHATIF & 2   // (probe only: timing without the pivot-block factorization; wrong results)
        if (p < 0)
#endif
        chol8_inv8(As + (8 * q) * LD + 8 * q, LD, Ds + q * 8 * kPL, bad);
        if (split) {   // T_q to the V CTA (counted on step p's barrier)
          __syncwarp();
          push_t(q, p);
        }
        __syncwarp();
        if (p == 5) FCP(56);
      } else {
        asm volatile("bar.arrive 1, %0;" ::"n"(kFcThreads) : "memory");
      }
      FCP(20 + p);   // (probe: the pivot warp's work of step p is done)
    } else if (wid < 0) {
      asm volatile("bar.sync 1, %0;" ::"n"(kFcThreads) : "memory");   // idle warp on the pivot warp's sub-partition
    } else {
      if (p > 0 && wid == kFcWorkers - 1)   // V_pp = T_p (factored by the pivot warp in step p-1)
        for (int e = lane; e < 64; e += 32)
          Vout[(int64_t)(8 * p + (e >> 3)) * Sp + 8 * p + (e & 7)] = Ds[p * 8 * kPL + (e >> 3) * kPL + (e & 7)];
      // the previous step's panel replaces A_{i,p-1} (read below as L_{p,p-1} by V's row block p)
      if (p > 0) {
        const double *Wq = Wp0 + ((p - 1) & 1) * Sp * kPL;
        for (int e = wid * 32 + lane; e < (nt - p) * 64; e += kFcWorkers * 32) {
          const int i = 8 * p + (e >> 3), b = e & 7;
          As[i * LD + 8 * (p - 1) + b] = Wq[i * kPL + b];
        }
        if (split)   // L's column block p-1, rows >= 8p, to the V CTA: pairs of doubles
          for (int e = wid * 32 + lane; e < (nt - p) * 32; e += kFcWorkers * 32) {
            const int i = 8 * p + (e >> 2), b = 2 * (e & 3);
            st_async_f64x2(rsm0 + (uint32_t)(sizeof(double) * (i * LD + 8 * (p - 1) + b)), Wq[i * kPL + b],
                           Wq[i * kPL + b + 1], rbar0 + 8u * p);
          }
      }
      for (int i = p + 2 + wid; i < nt; i += kFcWorkers) {   // panel L_ip = A_ip T_p^T, i >= p+2
        double c[2] = {0.0, 0.0};
        dmma8_tn(c, As + (8 * i) * LD + 8 * p, LD, Tp, kPL, g, t);
        frag_store(c, Wp + 8 * i * kPL, kPL, g, t);
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kFcThreads) : "memory");   // the whole panel is there
#if FC_WHATIF & 1   // (probe only: timing without the trailing update and V's row blocks; wrong results)
      if (p >= 0) goto step_end;
#endif
      // (beta, workers) trailing update A_ij -= L_ip L_jp^T, p < j <= i, except (p+1, p+1); pairs
      // (ii, jj), jj <= ii < m, enumerated row by row, two tiles per iteration (independent chains)
      const int m = nt - 1 - p;
      auto norm = [](int &ii, int &jj) {
        while (jj > ii) {
          jj -= ii + 1;
          ++ii;
        }
      };
      int ii = 0, jj = wid;
      norm(ii, jj);
      while (ii < m) {
        int ii2 = ii, jj2 = jj + kFcWorkers;
        norm(ii2, jj2);
        const bool one = !(ii == 0 && jj == 0), two = ii2 < m;
        const int i1 = p + 1 + ii, j1 = p + 1 + jj, i2 = p + 1 + ii2, j2 = p + 1 + jj2;
        double c1[2] = {0.0, 0.0}, c2[2] = {0.0, 0.0};
        if (one) frag_load(c1, As + (8 * i1) * LD + 8 * j1, LD, g, t);
        if (two) frag_load(c2, As + (8 * i2) * LD + 8 * j2, LD, g, t);
        if (one) {
          const double *pa = Wp + 8 * i1 * kPL, *pb = Wp + 8 * j1 * kPL;
          dmma(c1[0], c1[1], -pa[g * kPL + t], pb[g * kPL + t]);
          dmma(c1[0], c1[1], -pa[g * kPL + 4 + t], pb[g * kPL + 4 + t]);
        }
        if (two) {
          const double *pa = Wp + 8 * i2 * kPL, *pb = Wp + 8 * j2 * kPL;
          dmma(c2[0], c2[1], -pa[g * kPL + t], pb[g * kPL + t]);
          dmma(c2[0], c2[1], -pa[g * kPL + 4 + t], pb[g * kPL + 4 + t]);
        }
        if (one) frag_store(c1, As + (8 * i1) * LD + 8 * j1, LD, g, t);
        if (two) frag_store(c2, As + (8 * i2) * LD + 8 * j2, LD, g, t);
        ii = ii2;
        jj = jj2 + kFcWorkers;
        norm(ii, jj);
      }
      // (beta, workers) V row block p: V_pk = -T_p sum_{k<=m<p} L_pm V_mk (V_kk = T_k), stored
      // transposed in the upper tile (k, p): As[8k + a][8p + b] = V[8p + b][8k + a]
      double *xs = Xs + warp * 8 * kPL;
      for (int k = wid; k < (split ? 0 : p); k += kFcWorkers) {   // (split: on the V CTA)
        // two accumulator chains (even / odd m) halve the dependent-DMMA latency of the long rows
        double c[2] = {0.0, 0.0}, c2[2] = {0.0, 0.0};
        dmma8_nn(c, As + (8 * p) * LD + 8 * k, LD, Ds + k * 8 * kPL, kPL, g, t);   // L_pk T_k
        int mm = k + 1;
        for (; mm + 1 < p; mm += 2) {   // L_pm V_mk, V_mk[kk][n] = As[8k + n][8mm + kk]
          dmma8_tn(c2, As + (8 * p) * LD + 8 * mm, LD, As + (8 * k) * LD + 8 * mm, LD, g, t);
          dmma8_tn(c, As + (8 * p) * LD + 8 * (mm + 1), LD, As + (8 * k) * LD + 8 * (mm + 1), LD, g, t);
        }
        if (mm < p) dmma8_tn(c2, As + (8 * p) * LD + 8 * mm, LD, As + (8 * k) * LD + 8 * mm, LD, g, t);
        c[0] += c2[0];
        c[1] += c2[1];
        frag_store(c, xs, kPL, g, t);
        __syncwarp();
        double v[2] = {0.0, 0.0};
        dmma8_nn(v, Tp, kPL, xs, kPL, g, t);
        __syncwarp();
#pragma unroll
        for (int e2 = 0; e2 < 2; ++e2) As[(8 * k + 2 * t + e2) * LD + 8 * p + g] = -v[e2];
        *(double2 *)(Vout + (int64_t)(8 * p + g) * Sp + 8 * k + 2 * t) = make_double2(-v[0], -v[1]);   // V_pk
      }
    }
#if FC_WHATIF & 1
  step_end:
#endif
    __syncthreads();
    FCP(4 + p);
  }
  __syncthreads();
  FCP(2);
  FCP(3);
  return bad;
}

size_t fc_smem_bytes(int S) {
  const int nt = (S + 7) / 8, Sp = 8 * nt;
  return sizeof(double) * ((size_t)Sp * ld_frag(Sp) + (size_t)(nt * 8 + 2 * Sp + 8 * kFcWarps) * kPL);
}

// The factor V = L^{-1} of one SPD matrix (S <= STR_MAXW) on one CTA.
__global__ void __launch_bounds__(kFcThreads, 1)
    k_spd_factor(const double *__restrict__ Q, int S, double *__restrict__ V, int *info) {
  PDL_PROLOGUE();
  extern __shared__ __align__(16) double fsm[];
  const bool bad = cta_bchol(Q, S, fsm, V);
  if (bad && threadIdx.x == 0 && info) atomicExch(info, 1);
}

// The second CTA of the two-CTA factor: V's row blocks (V_pk = -T_p sum_{k<=m<p} L_pm V_mk, k < p),
// one step behind the factoring CTA.  That CTA pushes L's column blocks and the T_p into this CTA's
// tiles by st.async (distributed shared memory, the same positions as its own copies), counted in
// bytes on this CTA's mbarrier of the step, so this CTA waits on its own barriers and reads only its
// own shared memory.  V^T goes to the upper tiles here (the later rows read it) and V to Vout; the
// diagonal blocks V_pp = T_p are written by the factoring CTA.  So the factor's worker warps carry
// only the trailing updates.
__device__ void cta_vrows(int S, double *sm, double *__restrict__ Vout, uint64_t *vbar) {
  const int nt = (S + 7) >> 3, Sp = nt * 8, LD = ld_frag(Sp);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  double *As = sm, *Ds = As + Sp * LD, *Xs = Ds + nt * 8 * kPL + 2 * Sp * kPL;
  for (int p = 1; p < nt; ++p) {
    if (p == 1) tc::mbar_wait(&vbar[0], 0);   // step 0: T_0, T_1
    tc::mbar_wait(&vbar[p], 0);               // step p: L's column block p-1 (rows >= 8p), T_{p+1}
    const double *Tp = Ds + p * 8 * kPL;
    double *xs = Xs + warp * 8 * kPL;
    for (int k = warp; k < p; k += kFcWarps) {
      double c[2] = {0.0, 0.0}, c2[2] = {0.0, 0.0};
      dmma8_nn(c, As + (8 * p) * LD + 8 * k, LD, Ds + k * 8 * kPL, kPL, g, t);   // L_pk T_k
      int mm = k + 1;
      for (; mm + 1 < p; mm += 2) {   // L_pm V_mk, V_mk[kk][n] = As[8k + n][8mm + kk]
        dmma8_tn(c2, As + (8 * p) * LD + 8 * mm, LD, As + (8 * k) * LD + 8 * mm, LD, g, t);
        dmma8_tn(c, As + (8 * p) * LD + 8 * (mm + 1), LD, As + (8 * k) * LD + 8 * (mm + 1), LD, g, t);
      }
      if (mm < p) dmma8_tn(c2, As + (8 * p) * LD + 8 * mm, LD, As + (8 * k) * LD + 8 * mm, LD, g, t);
      c[0] += c2[0];
      c[1] += c2[1];
      frag_store(c, xs, kPL, g, t);
      __syncwarp();
      double v[2] = {0.0, 0.0};
      dmma8_nn(v, Tp, kPL, xs, kPL, g, t);
      __syncwarp();
#pragma unroll
      for (int e2 = 0; e2 < 2; ++e2) As[(8 * k + 2 * t + e2) * LD + 8 * p + g] = -v[e2];
      *(double2 *)(Vout + (int64_t)(8 * p + g) * Sp + 8 * k + 2 * t) = make_double2(-v[0], -v[1]);   // V_pk
    }
    __syncthreads();   // V's row block p is read by the later rows
  }
}

// The factor on a cluster of two CTAs: CTA 0 factors (cta_bchol without V's rows), CTA 1 forms V's rows.
__global__ void __launch_bounds__(kFcThreads, 1)
    k_spd_factor2(const double *__restrict__ Q, int S, double *__restrict__ V, int *info) {
  PDL_PROLOGUE();
  extern __shared__ __align__(16) double fsm[];
  __shared__ __align__(8) uint64_t vbar[STR_MAXW / 8];   // (CTA 1's copies are used)
  const unsigned rank = cluster_rank();
  const int nt = (S + 7) >> 3;
  if (rank == 1 && threadIdx.x == 0) {   // the bytes each step of CTA 0 pushes here
    for (int p = 0; p < nt; ++p) {
      tc::mbar_init(&vbar[p], 1);
      const uint32_t tbytes = (p + 1 < nt ? 512u : 0u) + (p == 0 ? 512u : 0u), lbytes = p > 0 ? 512u * (nt - p) : 0u;
      tc::mbar_arrive_expect_tx(&vbar[p], tbytes + lbytes);
    }
    tc::fence_barrier_init();
  }
  // phase 0 of the cluster barrier: CTA 1's barriers exist before CTA 0 pushes (CTA 0 waits for the
  // phase only after loading Q, so its factorization starts at once)
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  if (rank == 0) {
    const bool bad = cta_bchol(Q, S, fsm, V, vbar);
    if (bad && threadIdx.x == 0 && info) atomicExch(info, 1);
  } else {
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    cta_vrows(S, fsm, V, vbar);
  }
  cluster_sync_all();   // (no CTA leaves while the other may still address its shared memory)
}

size_t spd_factor_doubles(int S) {
  const int Sp = (S + 7) / 8 * 8;
  return (size_t)Sp * Sp;
}

void launch_spd_factor(const double *Q, int S, double *V, int *info, cudaStream_t s) {
  if (g_dbg_skip & 1) return;
  static PerDeviceOnce once;
  once_per_device(once, [] {
    cudaFuncSetAttribute(k_spd_factor, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fc_smem_bytes(STR_MAXW));
    prefer_max_smem(k_spd_factor);
  });
  static int split = -1;
  if (split < 0) {
    const char *e = getenv("STR_FACTOR_SPLIT");   // A/B knob: 0 = the one-CTA factor
    split = (e && e[0] == '0') ? 0 : 1;
  }
  if (split && S > kSplitMinS) {
    static PerDeviceOnce once2;
    once_per_device(once2, [] {
      cudaFuncSetAttribute(k_spd_factor2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fc_smem_bytes(STR_MAXW));
      prefer_max_smem(k_spd_factor2);
    });
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2);
    cfg.blockDim = dim3(kFcThreads);
    cfg.dynamicSmemBytes = fc_smem_bytes(S);
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = (pdl_mask() & kPdlInv) ? 2 : 1;
    if (cudaLaunchKernelEx(&cfg, k_spd_factor2, Q, S, V, info) == cudaSuccess) return;
    cudaGetLastError();   // (not sticky) fall back to one CTA
  }
  pdl_launch(kPdlInv, k_spd_factor, dim3(1), dim3(kFcThreads), fc_smem_bytes(S), s, Q, S, V, info);
}

// ------------------------------------------------------------------------------------------
// out = P Q^{-1} = (P V^T) V for I rows of P (I x S, row-major) with the factor V of
// launch_spd_factor (the G_n(2) = P_n Q_n^{-1} of Alg. 4 l.17 P:379 and G_N^new = M_N (H^{≠N}_<2>)^{-1}
// of l.9 P:370).  One CTA per 8-row tile: V's lower blocks staged in shared memory (cp.async), then
// Y = P V^T column tile by column tile over the 8 warps (Y[:, c] = sum_{k <= c} P[:, k] V[c][k]),
// then out = Y V (out[:, c] = sum_{k >= c} Y[:, k] V[k][c]).
__global__ void __launch_bounds__(kRsThreads, 1)
    k_rows_solve(const double *__restrict__ P, const double *__restrict__ V, int S, int64_t I,
                 double *__restrict__ out) {
  PDL_PROLOGUE();
  extern __shared__ __align__(16) double rsm[];
  const int nt = (S + 7) >> 3, Sp = nt * 8, LD = ld_frag(Sp);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  double *Vs = rsm;              // [Sp][LD]  (blocks on and below the diagonal)
  double *Ps = Vs + Sp * LD;     // [8][LD]  the P rows, then Y
  const int64_t r0 = (int64_t)blockIdx.x * 8;
  const int nr = (int)((I - r0) < 8 ? (I - r0) : 8);
  for (int e = threadIdx.x; e < Sp * (Sp / 2); e += kRsThreads) {
    const int i = e / (Sp / 2), j = 2 * (e - i * (Sp / 2));
    if ((j >> 3) <= (i >> 3)) cpa16cg(Vs + i * LD + j, V + (int64_t)i * Sp + j);
  }
  for (int e = threadIdx.x; e < 8 * Sp; e += kRsThreads) {
    const int i = e / Sp, j = e - (e / Sp) * Sp;
    if (i < nr && j < S) cpa8(Ps + i * LD + j, P + (r0 + i) * S + j);
    else Ps[i * LD + j] = 0.0;
  }
  cpa_commit();
  cpa_wait<0>();
  __syncthreads();
  // one column tile per warp (nt <= 16); each product runs on two accumulator chains (even / odd k)
  const int c = warp;
  const bool act = c < nt;
  double y[2] = {0.0, 0.0}, y2[2] = {0.0, 0.0};
  if (act) {   // Y[:, c] = sum_{k <= c} P[:, k] V[c][k]  (B[k][n] = V[n][k]: tn, V rows at c)
    int k = 0;
    for (; k + 1 <= c; k += 2) {
      dmma8_tn(y, Ps + 8 * k, LD, Vs + (8 * c) * LD + 8 * k, LD, g, t);
      dmma8_tn(y2, Ps + 8 * (k + 1), LD, Vs + (8 * c) * LD + 8 * (k + 1), LD, g, t);
    }
    if (k <= c) dmma8_tn(y, Ps + 8 * k, LD, Vs + (8 * c) * LD + 8 * k, LD, g, t);
    y[0] += y2[0];
    y[1] += y2[1];
  }
  __syncthreads();   // every warp has read P
  if (act) frag_store(y, Ps + 8 * c, LD, g, t);
  __syncthreads();
  if (!act) return;
  double o[2] = {0.0, 0.0}, o2[2] = {0.0, 0.0};   // out[:, c] = sum_{k >= c} Y[:, k] V[k][c]  (B = V rows at k: nn)
  int k = c;
  for (; k + 1 < nt; k += 2) {
    dmma8_nn(o, Ps + 8 * k, LD, Vs + (8 * k) * LD + 8 * c, LD, g, t);
    dmma8_nn(o2, Ps + 8 * (k + 1), LD, Vs + (8 * (k + 1)) * LD + 8 * c, LD, g, t);
  }
  if (k < nt) dmma8_nn(o, Ps + 8 * k, LD, Vs + (8 * k) * LD + 8 * c, LD, g, t);
  o[0] += o2[0];
  o[1] += o2[1];
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int col = 8 * c + 2 * t + e;
    if (g < nr && col < S) out[(r0 + g) * S + col] = o[e];
  }
}

void launch_rows_solve(const double *P, const double *V, int S, int64_t I, double *out, cudaStream_t s) {
  if (g_dbg_skip & 32) return;
  if (I <= 0) return;
  const int Sp = (S + 7) / 8 * 8;
  const size_t smem = sizeof(double) * (size_t)(Sp + 8) * ld_frag(Sp);
  static PerDeviceOnce once;
  once_per_device(once, [] {
    cudaFuncSetAttribute(k_rows_solve, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(sizeof(double) * (STR_MAXW + 8) * ld_frag(STR_MAXW)));
    prefer_max_smem(k_rows_solve);
  });
  pdl_launch(kPdlDmma, k_rows_solve, dim3((unsigned)cdiv(I, 8)), dim3(kRsThreads), smem, s, P, V, S, I, out);
}

}  // namespace strb200
