// kernels_contract_f64.cu — FP64 contraction of X_new with a chained-slice table.
//
// The two passes of the exact two-pass schedule evaluate
// the products X^new_[n] G^{≠n}_[2] of Alg. 4 l.9 and l.14 for every mode:
//   pass 1: Y_L[(l,t)][w] = sum_r  X[l + L r + L Rr t] T_R[r][w]       (M = L*t, K = Rr)
//   pass 2: Y_R[r][w]     = sum_{l,t} X[l + L r + L Rr t] T_L[l + L t][w]  (M = Rr, K = L*t)
// where l runs over the left modes (1..k), r over the right modes (k+1..N-1), and the tables
// hold products of TR-core lateral slices (Def. 3).  This file is the FP64 path
// (FP64 tensor cores, fp64 accumulation; used where cond(Q_n) demands it and as the reference-
// precision GPU path).  Split-K partials are reduced in a fixed order, so results are deterministic.
#include "common.cuh"
#include "kernels.h"

namespace strb200 {

constexpr int BM = 64, BK = 16;   // M tile and K granule of the split-K partition

// FP64 tensor-core (DMMA m8n8k4) version: CTA tile 64 (M) x 128 (N = W padded), 8 warps as
// 2 (M) x 4 (N), each warp 32 x 32 = 4 x 4 fragments.  Fragment layouts (m8n8k4, f64): A (8 x 4,
// row) lane holds A[lane/4][lane%4]; B (4 x 8, col) lane holds B[lane%4][lane/4]; C (8 x 8) lane
// holds C[lane/4][2 (lane%4) + {0,1}].  Shared tiles As[m][k], Bs[n][k] with row stride 20 doubles:
// the 32 fragment reads of a warp hit every 8-byte slot of two wavefronts exactly once.  The X
// offsets of the rows (pass 1) / columns (pass 2) a thread loads are formed once per tile, not per
// element.
constexpr int DBM = 64, DBN = 128, DBK = 16, DLD = DBK + 4;

__device__ __forceinline__ void dmma884_f(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <typename T, int PASS>
__global__ void __launch_bounds__(256) k_contract_f64_dmma(const void *const *Xp, const double *__restrict__ Btab, int W,
                                                           int64_t L, int64_t Rr, int64_t M, int64_t K, int64_t kchunk,
                                                           double *__restrict__ part) {
  const T *__restrict__ X = (const T *)*Xp;
  __shared__ __align__(16) double As[DBM][DLD];
  __shared__ __align__(16) double Bs[DBN][DLD];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3;                 // warp tile rows wm*32.., cols wn*32..
  const int64_t m0 = (int64_t)blockIdx.x * DBM;
  const int64_t k0 = (int64_t)blockIdx.y * kchunk;
  const int64_t k1 = min(K, k0 + kchunk);
  const int64_t LRr = L * Rr;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  // A-tile load mapping (DBM x DBK = 1024 elements, 4 per thread):
  //   pass 1: element (mm, kk), mm = tid % 64 (contiguous l), kk = tid / 64 + 4 q; X offset of row m
  //           = l + LRr t (m = l + L t), formed once; + L k per k.
  //   pass 2: element (mm, kk), kk = tid % 16 (contiguous l), mm = tid / 16 + 16 q; X offset of
  //           column k = l + LRr t (k = l + L t), advanced per chunk; + L m per row.
  int64_t rowoff = 0;
  bool rowok = true;
  int amm = 0, akk = 0;
  if (PASS == 1) {   // a warp stores 8 consecutive rows x 4 k: all 16 8-byte slots of 2 wavefronts
    amm = 8 * warp + (lane & 7);
    akk = lane >> 3;
    const int64_t m = m0 + amm;
    rowok = m < M;
    if (rowok) rowoff = (m % L) + LRr * (m / L);
  } else {
    akk = tid % DBK;
    amm = tid / DBK;
  }
  // software pipeline: the global values of tile kb + DBK are loaded into registers while the
  // fragments of tile kb are multiplied, then stored to shared memory
  double ra[4], rb[8];
  auto gload = [&](int64_t kb) {
    if (PASS == 1) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t k = kb + akk + 4 * q;
        ra[q] = (rowok && k < k1) ? (double)X[rowoff + L * k] : 0.0;
      }
    } else {
      const int64_t k = kb + akk;
      const bool kok = k < k1;
      const int64_t coloff = kok ? (k % L) + LRr * (k / L) : 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t m = m0 + amm + 16 * q;
        ra[q] = (kok && m < M) ? (double)X[coloff + L * m] : 0.0;
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {   // B: w = 8 (warp + 8 (q / 4)) + lane % 8, kk = lane / 8 + 4 (q % 4)
      const int w = 8 * (warp + 8 * (q >> 2)) + (lane & 7), kk = (lane >> 3) + 4 * (q & 3);
      const int64_t k = kb + kk;
      rb[q] = (k < k1 && w < W) ? Btab[k * W + w] : 0.0;
    }
  };
  auto sstore = [&]() {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (PASS == 1) As[amm][akk + 4 * q] = ra[q];
      else As[amm + 16 * q][akk] = ra[q];
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) Bs[8 * (warp + 8 * (q >> 2)) + (lane & 7)][(lane >> 3) + 4 * (q & 3)] = rb[q];
  };
  if (k0 < k1) gload(k0);
  for (int64_t kb = k0; kb < k1; kb += DBK) {
    sstore();
    __syncthreads();
    if (kb + DBK < k1) gload(kb + DBK);
#pragma unroll
    for (int ks = 0; ks < DBK / 4; ++ks) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[wm * 32 + i * 8 + (lane >> 2)][ks * 4 + (lane & 3)];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[wn * 32 + j * 8 + (lane >> 2)][ks * 4 + (lane & 3)];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884_f(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
    __syncthreads();
  }
  double *o = part + (int64_t)blockIdx.y * M * W;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t m = m0 + wm * 32 + i * 8 + (lane >> 2);
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int w = wn * 32 + j * 8 + 2 * (lane & 3);
      if (w < W) o[m * W + w] = acc[i][j][0];
      if (w + 1 < W) o[m * W + w + 1] = acc[i][j][1];
    }
  }
}

__global__ void k_reduce_splits(const double *__restrict__ part, int splits, int64_t n, double *__restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int j = 0; j < splits; ++j) s += part[j * n + i];
  out[i] = s;
}

template <typename T, int PASS>
static void dispatch_w(const void *const *X, const double *B, int W, int64_t L, int64_t Rr, int64_t tn, int64_t M, int64_t K,
                       int64_t kchunk, int splits, double *part, cudaStream_t s) {
  (void)tn;
  dim3 g((unsigned)cdiv(M, DBM), (unsigned)splits);   // W <= 128 (str_init)
  k_contract_f64_dmma<T, PASS><<<g, 256, 0, s>>>(X, B, W, L, Rr, M, K, kchunk, part);
}

int contract_f64_splits(int64_t M, int64_t K) {
  int64_t mt = cdiv(M, BM);
  // ~2 CTAs per SM, and K chunks of at most ~640 (long chunks leave the few M-tiles of a
  // large-K pass latency-bound: C5 FP64 pass 2, 12 -> 20 splits, 347 -> ~250 us; tools/runs/gpu_r2bl.sh)
  int64_t want = std::max<int64_t>(cdiv(2 * 148, mt), cdiv(K, 640));
  int64_t maxs = std::min<int64_t>(64, cdiv(K, 2 * BK));
  int64_t s = want < maxs ? want : maxs;
  if (s < 1) s = 1;
  // Whole waves: a grid that just spills into another wave of resident CTAs wastes most of it (C5 FP64
  // pass 1: 3 splits = 600 CTAs = 2.03 waves of 2 x 148, ncu: the FP64 pipe 50% busy;
  // profiles/r02f_ncu_contract_f64.txt).  Two CTAs resident on an SM share its FP64 pipe, so the
  // cost of a split count is scored at both granularities — waves of 296 CTAs (residency) and of 148
  // (one CTA's work per SM) — times the chunk length, plus the split's share of the reduce (its
  // partial written and read once, in units of one CTA's K step); the best of s .. 2s is taken
  // (measured: C5 FP64 0.705 -> 0.634 ms per step with 5 / 23 splits, C4 FP64 best with 37 / 3).
  auto cost = [&](int64_t c) {
    const int64_t chunk = cdiv(cdiv(K, c), BK) * BK;
    const int64_t real = cdiv(K, chunk);
    return (double)((cdiv(mt * real, 296) + cdiv(mt * real, 148)) * chunk) +
           (real > 1 ? (double)real * (double)M * 4e-3 : 0.0);
  };
  int64_t best = s;
  for (int64_t c = s + 1; c <= std::min<int64_t>(maxs, 2 * s); ++c)
    if (cost(c) < cost(best) * 0.995) best = c;
  return (int)best;
}

// Returns the number of kernel launches.
int launch_contract_f64(const void *const *X, bool x_is_f64, int pass, const double *Btab, int W, int64_t L, int64_t Rr,
                        int64_t tn, double *out, double *ws, cudaStream_t s) {
  int64_t M = pass == 1 ? L * tn : Rr;
  int64_t K = pass == 1 ? Rr : L * tn;
  int splits = contract_f64_splits(M, K);
  int64_t kchunk = cdiv(cdiv(K, splits), BK) * BK;
  splits = (int)cdiv(K, kchunk);
  double *part = splits == 1 ? out : ws;
  if (x_is_f64) {
    if (pass == 1) dispatch_w<double, 1>(X, Btab, W, L, Rr, tn, M, K, kchunk, splits, part, s);
    else dispatch_w<double, 2>(X, Btab, W, L, Rr, tn, M, K, kchunk, splits, part, s);
  } else {
    if (pass == 1) dispatch_w<float, 1>(X, Btab, W, L, Rr, tn, M, K, kchunk, splits, part, s);
    else dispatch_w<float, 2>(X, Btab, W, L, Rr, tn, M, K, kchunk, splits, part, s);
  }
  if (splits == 1) return 1;
  int64_t n = M * W;
  k_reduce_splits<<<(unsigned)cdiv(n, 256), 256, 0, s>>>(ws, splits, n, out);
  return 2;
}

size_t contract_f64_ws_doubles(int64_t M, int64_t K, int W) {
  int splits = contract_f64_splits(M, K);
  return (size_t)splits * M * W;
}

// ------------------------------------------------------------------------------------------
// Fit partial sums over temporal rows: X̂[l + L r + L Rr t] = sum_{p,q} TLf[(l,t)][p][q] TR[r][q][p]
// (Tr(G_1...G_{N-1} G_N(t)) = Tr(TLf TR)).  Per block: sum (X - X̂)^2 and sum X^2.
template <typename T>
__global__ void __launch_bounds__(256) k_fit_partial(const T *__restrict__ X, const double *__restrict__ TLf,
                                                     const double *__restrict__ TR, int Ra, int Rb, int64_t L,
                                                     int64_t Rr, int64_t tn, double2 *__restrict__ out) {
  // grid: x = l-blocks, y = r, z = t
  extern __shared__ double trs[];   // Rb x Ra (TR[r] row-major q*Ra + p)
  const int64_t r = blockIdx.y, t = blockIdx.z;
  const int W = Ra * Rb;
  for (int e = threadIdx.x; e < W; e += blockDim.x) trs[e] = TR[r * W + e];
  __syncthreads();
  int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double res = 0.0, nx = 0.0;
  if (l < L) {
    const double *tl = TLf + (l + L * t) * W;   // Ra x Rb row-major p*Rb + q
    double xh = 0.0;
    for (int p = 0; p < Ra; ++p)
      for (int q = 0; q < Rb; ++q) xh = fma(tl[p * Rb + q], trs[q * Ra + p], xh);
    double x = (double)X[l + L * r + L * Rr * t];
    double d = x - xh;
    res = d * d;
    nx = x * x;
  }
  for (int o = 16; o > 0; o >>= 1) {
    res += __shfl_xor_sync(0xffffffffu, res, o);
    nx += __shfl_xor_sync(0xffffffffu, nx, o);
  }
  __shared__ double sr[8], sn[8];
  int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (lane == 0) { sr[warp] = res; sn[warp] = nx; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) { a += sr[w]; b += sn[w]; }
    int64_t bid = blockIdx.x + (int64_t)gridDim.x * (blockIdx.y + (int64_t)gridDim.y * blockIdx.z);
    out[bid] = make_double2(a, b);
  }
}

__global__ void k_fit_reduce(const double2 *__restrict__ in, int64_t n, double *__restrict__ acc2) {
  // single block, fixed-order strided sums then tree
  __shared__ double sa[256], sb[256];
  double a = 0.0, b = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) { a += in[i].x; b += in[i].y; }
  sa[threadIdx.x] = a;
  sb[threadIdx.x] = b;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) { sa[threadIdx.x] += sa[threadIdx.x + o]; sb[threadIdx.x] += sb[threadIdx.x + o]; }
    __syncthreads();
  }
  if (threadIdx.x == 0) { acc2[0] += sa[0]; acc2[1] += sb[0]; }
}

size_t fit_partials(int64_t L, int64_t Rr, int64_t tn) { return (size_t)cdiv(L, 256) * Rr * tn; }

int launch_fit(const void *X, bool x_is_f64, const double *TLf, const double *TR, int Ra, int Rb, int64_t L,
               int64_t Rr, int64_t tn, double2 *partials, double *acc2, cudaStream_t s) {
  dim3 grid((unsigned)cdiv(L, 256), (unsigned)Rr, (unsigned)tn);
  size_t smem = sizeof(double) * Ra * Rb;
  if (x_is_f64)
    k_fit_partial<double><<<grid, 256, smem, s>>>((const double *)X, TLf, TR, Ra, Rb, L, Rr, tn, partials);
  else
    k_fit_partial<float><<<grid, 256, smem, s>>>((const float *)X, TLf, TR, Ra, Rb, L, Rr, tn, partials);
  k_fit_reduce<<<1, 256, 0, s>>>(partials, (int64_t)grid.x * grid.y * grid.z, acc2);
  return 2;
}

__global__ void k_set_ptr(const void **slot, const void *p) { *slot = p; }

void launch_set_ptr(const void **slot, const void *p, cudaStream_t s) { k_set_ptr<<<1, 1, 0, s>>>(slot, p); }
void *set_ptr_kernel() { return (void *)k_set_ptr; }

// Appends the t_new fresh temporal rows (scratch GNnew) to the temporal core at the device-side
// row counter *dT (graph-invariant: no host T in the arguments), then advances *dT.
__global__ void k_append_rows(double *__restrict__ GN, int64_t *dT, const double *__restrict__ GNnew, int64_t n,
                              int64_t tn, int SN) {
  const int64_t T = *dT;
  double *dst = GN + T * SN;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = GNnew[i];
  __syncthreads();
  if (threadIdx.x == 0) *dT = T + tn;
}

void launch_append_rows(double *GN, int64_t *dT, const double *GNnew, int64_t tn, int SN, cudaStream_t s) {
  k_append_rows<<<1, 512, 0, s>>>(GN, dT, GNnew, tn * SN, tn, SN);
}

void launch_fit_reduce(const double2 *partials, int64_t n, double *acc2, cudaStream_t s) {
  k_fit_reduce<<<1, 256, 0, s>>>(partials, n, acc2);
}

void prepare_f64_attrs() {
  prefer_max_smem(k_set_ptr);
  prefer_max_smem(k_append_rows);
  prefer_max_smem(k_reduce_splits);
  prefer_max_smem(k_contract_f64_dmma<float, 1>);
  prefer_max_smem(k_contract_f64_dmma<float, 2>);
  prefer_max_smem(k_contract_f64_dmma<double, 1>);
  prefer_max_smem(k_contract_f64_dmma<double, 2>);
}

}  // namespace strb200
