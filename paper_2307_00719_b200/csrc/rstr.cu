// rstr.cu — randomized streaming TR (rSTR) with uniform (Alg. 7) and
// leverage-score (Alg. 8) row sampling.
//
// Per draw (mode k, time step tau) m indices are drawn with replacement from a SplitMix64 stream
// keyed by (seed, tau, k) (reading R11; the oracle re-implements the same generator
// independently).  The draws run ON THE DEVICE in counter form (draw j = mix(key + (j+1) GOLDEN)),
// bit-identical to the host sampler, which is kept only for index tables the caller injects
// (str_set_index_table) and for the STR_RSTR_HOST_DRAWS=1 diagnostic.  Leverage probabilities
// p_k(i) = l_i(G_k(2)) / rank (Lemma 1) are computed on the device (Gram + SPD inverse:
// l_i = g_i^T (G^T G)^{-1} g_i when I_k > R_kR_{k+1}; uniform when I_k <= R_kR_{k+1}, reading R10)
// and drawn by inverse CDF on the device.  Everything else runs in device kernels:
//   * sampled slices (G_k)_S = G_k(:, idxs(:,k), :)                       (Alg. 7 l.4)
//   * sampled subchain G^{≠n}_S by the ⊡₂ chain of sampled slices         (Alg. 3 l.5-7, Def. 7)
//   * zipped fibers X_S[n] (I_n x m) gathered from X                      (reading R7)
//   * P_n += X_S[n] G_S[2], Q_n += G_S[2]^T G_S[2], G_n = P_n Q_n^{-1}     (Alg. 7 l.36-38)
//   * temporal rows G_N^new = X_S[N] G_S (G_S^T G_S)^{-1}                (reading R4)
// rSTR-K (Alg. 9) runs the same schedule on KSRFT-mixed data (ksrft.cu): every step
// draws sign flips and mixes the batch, the sampled slices are rows of the mixed cores, the chain
// is complex and written as the stacked real [Re; Im] matrix (2m rows), the fibers are unmixed on
// their own mode, so the same real GEMMs with K = 2m give Re(X~ conj G^) and Re(G^T conj G^); the
// temporal solve takes the real halves (K = m; readings R17-R22).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.h"
#include "str_internal.h"

namespace strb200 {

// ------------------------------------------------------------------------------------------ kernels
// out[s][c] = G[idx[s]][c]  (rows of a G(2) matrix with S columns)
__global__ void k_gather_rows(const double *__restrict__ G, int S, const int32_t *__restrict__ idx, int64_t m,
                              double *__restrict__ out) {
  PDL_PROLOGUE();
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= m * S) return;
  int64_t s = e / S;
  int c = (int)(e % S);
  out[e] = G[(int64_t)idx[s] * S + c];
}

// Zipped fibers: XS[i][s] = X(idx(s,1), ..., i (mode n), ..., idx(s,N)), X in the P:119 layout.
// idx is [N][m] (mode-major); strides[j] = element stride of mode j+1 (time last).
struct GatherDesc {
  int N, n;                 // order, target mode (1-based)
  int64_t stride[8];
  int64_t In, m;
};

template <typename T>
__global__ void k_gather_fibers(const void *const *__restrict__ Xp, const int32_t *__restrict__ idx, GatherDesc gd,
                                double *__restrict__ XS) {
  PDL_PROLOGUE();
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= gd.In * gd.m) return;
  const T *__restrict__ X = (const T *)*Xp;   // the batch, through the device slot set_x fills
  int64_t s = e % gd.m, i = e / gd.m;
  int64_t off = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    if (j < gd.N) {
      int64_t ij = (j == gd.n - 1) ? i : (int64_t)idx[j * gd.m + s];
      off += ij * gd.stride[j];
    }
  }
  XS[e] = (double)X[off];
}

// Device SplitMix64 draws, bit-identical to the host sampler below (and to the oracle's): output j
// of the stream keyed by (seed, tau, k) is mix(key + (j + 1) GOLDEN), so every draw is independent
// (counter-based) and one thread makes one draw.  tau lives on the device so that a captured step
// graph advances it itself.
__device__ __forceinline__ uint64_t splitmix_at(uint64_t key, uint64_t j) {
  uint64_t z = key + (j + 1) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t draw_key(uint64_t seed, int64_t tau, int k, int N) {
  return seed ^ (0x9E3779B97F4A7C15ull * (uint64_t)(1 + tau * (N + 1) + k));
}

__global__ void k_tau_advance(int64_t *tau) { *tau += 1; }

// uniform draw fused with the gather of the sampled rows (one node fewer per draw): thread (s, c)
// recomputes draw s (counter-based), writes idx[s] when c == 0 and copies G[idx_s][c]
__global__ void k_draw_gather_uniform(uint64_t seed, const int64_t *__restrict__ tau, int k, int N, int64_t I,
                                      int64_t m, const double *__restrict__ G, int S, int32_t *__restrict__ idx,
                                      double *__restrict__ out) {
  PDL_PROLOGUE();
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= m * S) return;
  const int64_t s = e / S;
  const int c = (int)(e - s * S);
  const uint64_t u = splitmix_at(draw_key(seed, *tau, k, N), (uint64_t)s);
  const int64_t ix = (int64_t)__umul64hi(u, (uint64_t)I);
  if (c == 0) idx[s] = (int32_t)ix;
  out[e] = G[ix * S + c];
}

// weighted by p (nullptr: 1/I each): one CTA; the CDF is summed by one thread in index order (as the
// host does), then each thread inverts it for its draws: first i with cdf[i] > (u >> 11) 2^-53 cdf[I-1]
__global__ void k_draw_weighted(const double *__restrict__ p, int64_t I, uint64_t seed, const int64_t *__restrict__ tau,
                                int k, int N, int64_t m, int32_t *__restrict__ out) {
  extern __shared__ double cdf[];
  if (threadIdx.x == 0) {
    double acc = 0.0;
    const double pu = 1.0 / (double)I;
    for (int64_t i = 0; i < I; ++i) {
      acc = acc + (p ? p[i] : pu);
      cdf[i] = acc;
    }
  }
  __syncthreads();
  const uint64_t key = draw_key(seed, *tau, k, N);
  const double total = cdf[I - 1];
  for (int64_t j = threadIdx.x; j < m; j += blockDim.x) {
    const uint64_t u = splitmix_at(key, (uint64_t)j);
    const double target = (double)(u >> 11) * 0x1.0p-53 * total;
    int64_t lo = 0, hi = I;   // upper_bound
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (cdf[mid] <= target) lo = mid + 1; else hi = mid;
    }
    out[j] = (int32_t)(lo < I - 1 ? lo : I - 1);
  }
}

// p_i = (sum_c Y[i][c] G[i][c]) / rank   (leverage of row i, Def. 8 via g_i^T (G^T G)^{-1} g_i)
__global__ void k_rowdot_scale(const double *__restrict__ Y, const double *__restrict__ G, int64_t I, int S,
                               double inv_rank, double *__restrict__ p) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= I) return;
  double acc = 0.0;
  for (int c = 0; c < S; ++c) acc = fma(Y[i * S + c], G[i * S + c], acc);
  p[i] = acc * inv_rank;
}

}  // namespace strb200

using namespace strb200;

#define RCU(call)                                                        \
  do {                                                                   \
    cudaError_t _e = (call);                                             \
    if (_e != cudaSuccess) {                                             \
      h->err = std::string(#call) + ": " + cudaGetErrorString(_e);       \
      h->poisoned = true;                                                \
      return STR_E_CUDA;                                                 \
    }                                                                    \
  } while (0)
#define RTRY(call)                 \
  do {                             \
    str_status _s = (call);        \
    if (_s != STR_OK) return _s;   \
  } while (0)

// ------------------------------------------------------------------------------------------ sampler
// SplitMix64 (reading R11): key = seed ^ (GOLDEN * (1 + tau*(N+1) + k)); uniform index =
// (u * I) >> 64; weighted: first i with cdf[i] > (u >> 11) * 2^-53 * cdf[I-1].
static const uint64_t kGolden = 0x9E3779B97F4A7C15ull;

static inline uint64_t splitmix_next(uint64_t &s) {
  s += kGolden;
  uint64_t z = s;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static void draw_uniform(uint64_t seed, int64_t tau, int k, int N, int64_t I, int64_t m, std::vector<int32_t> &out) {
  uint64_t s = seed ^ (kGolden * (uint64_t)(1 + tau * (N + 1) + k));
  out.resize(m);
  for (int64_t j = 0; j < m; ++j) {
    unsigned __int128 prod = (unsigned __int128)splitmix_next(s) * (unsigned __int128)(uint64_t)I;
    out[j] = (int32_t)(uint64_t)(prod >> 64);
  }
}

static void draw_weighted(uint64_t seed, int64_t tau, int k, int N, const std::vector<double> &p, int64_t m,
                          std::vector<int32_t> &out) {
  uint64_t s = seed ^ (kGolden * (uint64_t)(1 + tau * (N + 1) + k));
  const int64_t I = (int64_t)p.size();
  std::vector<double> c(I);
  double acc = 0.0;
  for (int64_t i = 0; i < I; ++i) {
    acc = acc + p[i];
    c[i] = acc;
  }
  out.resize(m);
  for (int64_t j = 0; j < m; ++j) {
    uint64_t u = splitmix_next(s);
    double target = (double)(u >> 11) * 0x1.0p-53 * c[I - 1];
    int64_t idx = std::upper_bound(c.begin(), c.end(), target) - c.begin();
    out[j] = (int32_t)std::min<int64_t>(idx, I - 1);
  }
}

// ------------------------------------------------------------------------------------------ helpers
static inline int RRr(const str_state *h, int n) { return h->R[(n - 1) % h->N]; }

static str_status ensure_dev(str_state *h, DevBuf &b, size_t bytes) {
  if (b.bytes >= bytes) return STR_OK;
  if (h->capturing) {   // a cudaFree inside the stream capture would invalidate it (rstr_workspace pre-sizes)
    h->err = "internal: rSTR workspace grows during graph capture";
    h->poisoned = true;
    return STR_E_CUDA;
  }
  if (b.p) {   // captured graphs may hold the old pointer
    h->reset_graphs();
    cudaFree(b.p);
  }
  b.p = nullptr;
  b.bytes = 0;
  if (cudaMalloc(&b.p, bytes) != cudaSuccess) {
    cudaGetLastError();
    h->err = "cudaMalloc failed (rSTR workspace)";
    h->poisoned = true;
    return STR_E_OOM;
  }
  b.bytes = bytes;
  return STR_OK;
}

// out = B A^{-1} for SPD A (S x S) and `rows` rows of B: the block-Cholesky factor V^T of A, then the
// two triangular products (B V^T) V (the "†" of reading R3/R4 on the device).  Ai: factor scratch.
static void solve_right(str_state *h, const double *A, int S, double *Ai, const double *B, int64_t rows, double *out) {
  launch_spd_factor(A, S, Ai, h->d_info, h->st);
  tl_mark(h, "spd_factor");
  launch_rows_solve(B, Ai, S, rows, out, h->st);
  tl_mark(h, "rows_solve");
}

static void gemm(str_state *h, const double *A, int64_t sai, int64_t sak, const double *B, int64_t sbk, int64_t sbj,
                 double *C, int M, int N, int64_t K, int acc, int sym = 0, bool side_ws = false) {
  const int nl = launch_gemm_sk(A, sai, sak, B, sbk, sbj, C, M, N, K, acc,
                                (double *)(side_ws ? h->sSk2.p : h->sSk.p), h->st, sym);
  tl_mark(h, "gemm_sk", nl);
}

// Fork / join of the side stream inside one rSTR step (graph branches when capturing): the Gram
// G_S^T G_S and its inverse run beside X_S G_S; the diagnostic timeline keeps one stream.
static str_status rs_fork(str_state *h) {
  h->st_main = h->st;
  if (h->timeline) return STR_OK;
  RCU(cudaEventRecord(h->ev_fork, h->st));
  RCU(cudaStreamWaitEvent(h->st2, h->ev_fork, 0));
  h->st = h->st2;
  return STR_OK;
}
static void rs_main(str_state *h) { h->st = h->st_main; }
static str_status rs_join(str_state *h) {
  if (h->timeline) return STR_OK;
  RCU(cudaEventRecord(h->ev_join, h->st2));
  RCU(cudaStreamWaitEvent(h->st, h->ev_join, 0));
  return STR_OK;
}

// Core k's slices as G(2) rows: k < N -> current core; k == N -> temporal rows [t0, t0 + rows).
static const double *core_rows(const str_state *h, int k, int64_t t0) {
  if (k == h->N) return (const double *)h->GN.p + t0 * h->SN;
  return (const double *)h->md[k - 1].G.p;
}

// ---- rSTR-K helpers
static bool ks_f64(const str_state *h) { return h->contract == STR_CONTRACT_F64; }

// dims of the batch being mixed: I_1..I_{N-1}, tn
static void ks_dims(const str_state *h, int64_t tn, int64_t *dims) {
  for (int j = 0; j < h->N - 1; ++j) dims[j] = h->md[j].I;
  dims[h->N - 1] = tn;
}

// Sign flips of this step (tau on the device) and X^ = X x_1 (F_1 D_1) ... x_N (F_N D_N) (Alg. 9
// l.21-22 P:1224-1225; Alg. 5 l.3 P:651).  The batch enters through the device slot dX.
static str_status ks_mix(str_state *h, int64_t tn) {
  int64_t dims[16];
  ks_dims(h, tn, dims);
  int64_t off = 0;
  for (int j = 0; j < h->N; ++j) {
    h->ks_off[j] = off;
    off += dims[j];
  }
  launch_draw_signs(h->seed, (const int64_t *)h->dTau.p, h->N, off, (double *)h->ksSign.p, h->st);
  tl_mark(h, "draw_signs");
  prof_mark(h, 0);   // profiling replay: events around the N mixing passes (bench roofline)
  for (int j = 0; j < h->N; ++j) {
    if (launch_mix_mode((const void *const *)h->dX.p, h->dtype == STR_F64, h->ksXh.p, ks_f64(h), dims, h->N, j,
                        (const double *)h->ksSign.p + h->ks_off[j], h->st) != 0) {
      h->err = "KSRFT mixing: mode too long for the shared-memory DFT";
      return STR_E_ARG;
    }
    tl_mark(h, "mix_mode");
  }
  prof_mark(h, 1);
  return STR_OK;
}

// (G^_k)_S = (G_k x_2 F_k D_k)(:, idxs(:,k), :) for the rows of G_k (I rows), into dst (m x S complex)
static str_status ks_sample(str_state *h, int k, const double *rows, int64_t I, double *dst) {
  const int S = RRr(h, k) * RRr(h, k + 1);
  const int32_t *dix = (const int32_t *)h->sIdxDev.p + (int64_t)(k - 1) * h->m;
  const int nl = launch_mix_sample(rows, I, S, dix, h->m, (const double *)h->ksSign.p + h->ks_off[k - 1],
                                   (double2 *)dst, (double2 *)h->ksCore.p, h->st);
  if (nl < 0) {
    h->err = "KSRFT: mode too long for the sampled mixing kernel";
    return STR_E_ARG;
  }
  tl_mark(h, "mix_sample", nl);
  return STR_OK;
}

// Leverage probabilities of an I x S matrix G (device rows), left on the device: returns the
// pointer, or nullptr when I <= S (every score is 1: the uniform distribution, reading R10).
static str_status leverage_probs_dev(str_state *h, const double *G, int64_t I, int S, const double **pout) {
  *pout = nullptr;
  if (I <= S) return STR_OK;
  RTRY(ensure_dev(h, h->sGram, sizeof(double) * S * S));
  RTRY(ensure_dev(h, h->sTmp, sizeof(double) * (I * S + I)));
  double *K = (double *)h->sGram.p;
  double *Y = (double *)h->sTmp.p;
  double *pd = Y + I * S;
  gemm(h, G, 1, S, G, S, 1, K, S, S, I, 0);                         // K = G^T G
  solve_right(h, K, S, (double *)h->Hq.p, G, I, Y);                 // Y = G K^{-1}
  k_rowdot_scale<<<(unsigned)cdiv(I, 128), 128, 0, h->st>>>(Y, G, I, S, 1.0 / (double)S, pd);
  tl_mark(h, "k_rowdot_scale");
  *pout = pd;
  return STR_OK;
}

// Leverage probabilities of an I x S matrix G (device rows) -> host vector p.
static str_status leverage_probs(str_state *h, const double *G, int64_t I, int S, std::vector<double> &p) {
  p.assign(I, 1.0 / (double)I);
  if (I <= S) return STR_OK;   // full row rank: every score is 1 (reading R10)
  RTRY(ensure_dev(h, h->sGram, sizeof(double) * S * S));
  RTRY(ensure_dev(h, h->sTmp, sizeof(double) * (I * S + I)));
  double *K = (double *)h->sGram.p;
  double *Y = (double *)h->sTmp.p;
  double *pd = Y + I * S;
  gemm(h, G, 1, S, G, S, 1, K, S, S, I, 0);                         // K = G^T G
  solve_right(h, K, S, (double *)h->Hq.p, G, I, Y);                 // Y = G K^{-1}
  k_rowdot_scale<<<(unsigned)cdiv(I, 128), 128, 0, h->st>>>(Y, G, I, S, 1.0 / (double)S, pd);
  tl_mark(h, "k_rowdot_scale");
  RCU(cudaMemcpyAsync(p.data(), pd, sizeof(double) * I, cudaMemcpyDeviceToHost, h->st));
  RCU(cudaStreamSynchronize(h->st));
  int info = 0;
  RCU(cudaMemcpy(&info, h->d_info, sizeof(int), cudaMemcpyDeviceToHost));
  if (info) {
    h->err = "leverage: G^T G not positive definite";
    h->poisoned = true;
    return STR_E_NUMERIC;
  }
  return STR_OK;
}

constexpr int64_t kDevCdfMax = 24576;   // leverage CDF in shared memory (192 KB)

// idxs(:,k) <- Randsample(I_k, m[, p_k]) on the device (no host round trip; capturable)
static str_status draw_mode_dev(str_state *h, int k, const double *rows, int64_t I) {
  const int S = RRr(h, k) * RRr(h, k + 1);
  int32_t *dix = (int32_t *)h->sIdxDev.p + (int64_t)(k - 1) * h->m;
  const int64_t *tau = (const int64_t *)h->dTau.p;
  ModeBuf &mbu = h->md[std::min(k, h->N - 1) - 1];
  double *dstu = (k == h->N) ? (double *)h->sG.p : (double *)mbu.samp.p;
  if (h->variant == STR_SAMPLE_UNIFORM) {   // draw + gather in one kernel
    h->idx_dev[k] = true;
    pdl_launch(kPdlRstr, k_draw_gather_uniform, dim3((unsigned)cdiv(h->m * S, 256)), dim3(256), 0, h->st, h->seed, tau,
               k, h->N, I, h->m, rows, S, dix, dstu);
    tl_mark(h, "draw_gather");
    return STR_OK;
  }
  if (h->variant == STR_SAMPLE_KSRFT) {     // mixed core, then draw + gather of its sampled rows
    h->idx_dev[k] = true;
    const int nl = launch_mix_sample_draw(rows, I, S, h->seed, tau, k, h->N, h->m,
                                          (const double *)h->ksSign.p + h->ks_off[k - 1], (double2 *)dstu,
                                          (double2 *)h->ksCore.p, dix, h->st);
    if (nl < 0) {
      h->err = "KSRFT: mode too long for the sampled mixing kernel";
      return STR_E_ARG;
    }
    tl_mark(h, "mix_sample_draw", nl);
    return STR_OK;
  }
  // leverage: probabilities, weighted draw (one CTA, CDF in shared memory), gather
  const double *pd = nullptr;
  RTRY(leverage_probs_dev(h, rows, I, S, &pd));
  k_draw_weighted<<<1, 1024, sizeof(double) * I, h->st>>>(pd, I, h->seed, tau, k, h->N, h->m, dix);
  tl_mark(h, "draw_weighted");
  h->idx_dev[k] = true;
  k_gather_rows<<<(unsigned)cdiv(h->m * S, 256), 256, 0, h->st>>>(rows, S, dix, h->m, dstu);
  tl_mark(h, "k_gather_rows");
  return STR_OK;
}

// idxs(:,k) <- Randsample(I_k, m[, p_k]); (G_k)_S <- G_k(:, idxs(:,k), :)
static str_status draw_mode(str_state *h, int k, const double *rows, int64_t I) {
  const int S = RRr(h, k) * RRr(h, k + 1);
  if (h->forced_idx[k].empty() && h->rstr_dev && (h->variant != STR_SAMPLE_LEVERAGE || I <= kDevCdfMax))
    return draw_mode_dev(h, k, rows, I);
  h->idx_dev[k] = false;
  std::vector<int32_t> &ix = h->last_idx[k];
  if (!h->forced_idx[k].empty()) {
    ix = h->forced_idx[k];
  } else if (h->variant != STR_SAMPLE_LEVERAGE) {
    draw_uniform(h->seed, h->tau, k, h->N, I, h->m, ix);
  } else {
    std::vector<double> p;
    RTRY(leverage_probs(h, rows, I, S, p));
    draw_weighted(h->seed, h->tau, k, h->N, p, h->m, ix);
  }
  int32_t *dix = (int32_t *)h->sIdxDev.p + (int64_t)(k - 1) * h->m;
  // pinned staging slot per mode: wait only until the previous upload from this slot has run
  int32_t *slot = h->idx_pinned + (int64_t)(k - 1) * h->m;
  RCU(cudaEventSynchronize(h->idx_ev[k]));
  std::copy(ix.begin(), ix.end(), slot);
  RCU(cudaMemcpyAsync(dix, slot, sizeof(int32_t) * h->m, cudaMemcpyHostToDevice, h->st));
  RCU(cudaEventRecord(h->idx_ev[k], h->st));
  ModeBuf &mb = h->md[std::min(k, h->N - 1) - 1];
  double *dst = (k == h->N) ? (double *)h->sG.p : (double *)mb.samp.p;
  if (h->ksrft()) return ks_sample(h, k, rows, I, dst);
  k_gather_rows<<<(unsigned)cdiv(h->m * S, 256), 256, 0, h->st>>>(rows, S, dix, h->m, dst);
  tl_mark(h, "k_gather_rows");
  return STR_OK;
}

// G_S[2] (m x R_nR_{n+1}) = ⊡₂ chain of sampled slices in order n+1..N, 1..n-1 (identity start).
static str_status sampled_chain(str_state *h, int n, double *out) {
  if (h->ksrft()) {   // complex slices -> stacked [Re; Im] (2m x S)
    const double2 *G[kMaxFactors];
    int Ra[kMaxFactors], Rb[kMaxFactors], nf = 0;
    const int N = h->N;
    auto add = [&](int k) {
      G[nf] = (const double2 *)((k == N) ? h->sG.p : h->md[k - 1].samp.p);
      Ra[nf] = RRr(h, k);
      Rb[nf] = RRr(h, k + 1);
      ++nf;
    };
    for (int k = n + 1; k <= N; ++k) add(k);
    for (int k = 1; k < n; ++k) add(k);
    if (launch_chain_complex(G, Ra, Rb, nf, h->m, out, h->st) != 0) {
      h->err = "complex sampled chain: bad factor list";
      return STR_E_ARG;
    }
    tl_mark(h, "chain_complex");
    return STR_OK;
  }
  FactorList fl;
  fl.n = 0;
  const int N = h->N;
  for (int k = n + 1; k <= N; ++k) {
    Factor f;
    f.G = (k == N) ? (const double *)h->sG.p : (const double *)h->md[k - 1].samp.p;
    f.I = (int32_t)h->m;
    f.Ra = RRr(h, k);
    f.Rb = RRr(h, k + 1);
    f.stride = 1;
    fl.f[fl.n++] = f;
  }
  for (int k = 1; k < n; ++k) {
    Factor f;
    f.G = (const double *)h->md[k - 1].samp.p;
    f.I = (int32_t)h->m;
    f.Ra = RRr(h, k);
    f.Rb = RRr(h, k + 1);
    f.stride = 1;
    fl.f[fl.n++] = f;
  }
  TableDesc td;
  td.fl = fl;
  td.Lk = h->m;
  td.tk = 1;
  td.Npad = 0;
  if (launch_build_table2(td, out, nullptr, h->st) != 0) {
    h->err = "sampled chain needs too much shared memory";
    return STR_E_ARG;
  }
  tl_mark(h, "table_sampled");
  return STR_OK;
}

static str_status gather_fibers(str_state *h, const void *X, int n, int64_t tn, double *XS) {
  if (h->ksrft()) {   // X~_S[n] = D_n F_n^* X^_S[n], stacked [Re | Im] (I_n x 2m)
    int64_t dims[16];
    ks_dims(h, tn, dims);
    if (launch_gather_unmix(h->ksXh.p, ks_f64(h), dims, h->N, n, (const int32_t *)h->sIdxDev.p, h->m,
                            (const double *)h->ksSign.p + h->ks_off[n - 1], XS, h->st) != 0) {
      h->err = "KSRFT: fiber too long for the unmixing kernel";
      return STR_E_ARG;
    }
    tl_mark(h, "gather_unmix");
    return STR_OK;
  }
  GatherDesc gd;
  gd.N = h->N;
  gd.n = n;
  int64_t st = 1;
  for (int j = 0; j < h->N - 1; ++j) {
    gd.stride[j] = st;
    st *= h->md[j].I;
  }
  gd.stride[h->N - 1] = st;
  for (int j = h->N; j < 8; ++j) gd.stride[j] = 0;
  gd.In = (n == h->N) ? tn : h->md[n - 1].I;
  gd.m = h->m;
  const unsigned grid = (unsigned)cdiv(gd.In * gd.m, 256);
  if (h->dtype == STR_F64)
    pdl_launch(kPdlRstr, k_gather_fibers<double>, dim3(grid), dim3(256), 0, h->st, (const void *const *)h->dX.p,
               (const int32_t *)h->sIdxDev.p, gd, XS);
  else
    pdl_launch(kPdlRstr, k_gather_fibers<float>, dim3(grid), dim3(256), 0, h->st, (const void *const *)h->dX.p,
               (const int32_t *)h->sIdxDev.p, gd, XS);
  tl_mark(h, "gather_fibers");
  return STR_OK;
}

static str_status rstr_workspace(str_state *h, int64_t tn) {
  static PerDeviceOnce attr_once;
  once_per_device(attr_once, [&] {
    cudaFuncSetAttribute(k_draw_weighted, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kDevCdfMax * 8));
  });
  if (!h->idx_pinned) {
    RCU(cudaMallocHost(&h->idx_pinned, sizeof(int32_t) * h->N * h->m));
    for (int k = 0; k <= h->N; ++k) RCU(cudaEventCreateWithFlags(&h->idx_ev[k], cudaEventDisableTiming));
  }
  int64_t maxI = tn;
  int maxS = 0;
  for (auto &mb : h->md) {
    maxI = std::max<int64_t>(maxI, mb.I);
    maxS = std::max(maxS, mb.Ra * mb.Rb);
  }
  maxS = std::max(maxS, h->SN);
  RTRY(ensure_dev(h, h->sIdxDev, sizeof(int32_t) * h->N * h->m));
  RTRY(ensure_dev(h, h->GNnew, sizeof(double) * tn * h->SN));
  if (!h->dTau.p) {
    RTRY(ensure_dev(h, h->dTau, sizeof(int64_t)));
    RCU(cudaMemsetAsync(h->dTau.p, 0, sizeof(int64_t), h->st));
  }
  const int64_t cw = h->ksrft() ? 2 : 1;   // rSTR-K: complex slices, stacked [Re; Im] rows
  RTRY(ensure_dev(h, h->sX, sizeof(double) * maxI * h->m * cw));
  RTRY(ensure_dev(h, h->sG, sizeof(double) * h->m * maxS * cw));
  RTRY(ensure_dev(h, h->sidx, sizeof(double) * h->m * maxS * cw));   // G_S[2]
  RTRY(ensure_dev(h, h->sGram, sizeof(double) * maxS * maxS));
  RTRY(ensure_dev(h, h->sTmp, sizeof(double) * (maxI * maxS + maxI)));   // leverage scores (leverage_probs_dev)
  RTRY(ensure_dev(h, h->sSk,
                  sizeof(double) * gemm_sk_ws_doubles((int)std::max<int64_t>(maxI, maxS), maxS, h->m * cw)));
  RTRY(ensure_dev(h, h->sSk2, sizeof(double) * gemm_sk_ws_doubles(maxS, maxS, h->m * cw)));
  RTRY(ensure_dev(h, h->Mt, sizeof(double) * std::max<int64_t>(maxI, tn) * maxS));
  for (auto &mb : h->md) RTRY(ensure_dev(h, mb.samp, sizeof(double) * h->m * mb.Ra * mb.Rb * cw));
  if (h->ksrft()) {
    int64_t slice = 1, sumI = tn;
    for (auto &mb : h->md) {
      slice *= mb.I;
      sumI += mb.I;
    }
    RTRY(ensure_dev(h, h->ksXh, (ks_f64(h) ? sizeof(double2) : sizeof(float2)) * slice * tn));
    RTRY(ensure_dev(h, h->ksSign, sizeof(double) * sumI));
    RTRY(ensure_dev(h, h->ksCore, sizeof(double2) * maxI * maxS));   // whole mixed core (k_mix_core)
  }
  return STR_OK;
}

// G_S[2] and X_S[n] of mode n (Alg. 7 l.12-14): both need only the index table.  For rSTR-K the
// gather (which also unmixes the fibers, Alg. 9 l.27) runs on the side stream beside the complex
// sampled chain (C4: 0.662 -> 0.628 ms per step); for rSTR-U/L the plain gather is too short to pay
// for the graph's cross-stream join (measured: 0.163 -> 0.182 ms), so the two stay in stream order.
static str_status chain_and_fibers(str_state *h, const void *X, int n, int64_t tn, double *GS, double *XS) {
  if (!h->ksrft()) {
    RTRY(sampled_chain(h, n, GS));
    return gather_fibers(h, X, n, tn, XS);
  }
  RTRY(rs_fork(h));
  RTRY(gather_fibers(h, X, n, tn, XS));
  rs_main(h);
  RTRY(sampled_chain(h, n, GS));
  return rs_join(h);
}

// Accumulate the sampled normal equations of mode n (1..N-1) from X (tn slices): P_n (+)= X_S G_S,
// Q_n (+)= G_S^T G_S (Alg. 7 l.15-16 / l.36-37); with `solve`, then G_n = P_n Q_n^{-1} (l.38).  The
// Gram and the inverse run on the side stream beside X_S G_S.
static str_status sampled_normal_eq(str_state *h, const void *X, int n, int64_t tn, int acc, bool solve) {
  ModeBuf &mb = h->md[n - 1];
  const int S = mb.Ra * mb.Rb;
  double *GS = (double *)h->sidx.p;
  double *XS = (double *)h->sX.p;
  const int64_t K = h->ksrft() ? 2 * h->m : h->m;   // rSTR-K: [Re X~, Im X~][Re G^; Im G^] (reading R21)
  RTRY(chain_and_fibers(h, X, n, tn, GS, XS));
  RTRY(rs_fork(h));
  gemm(h, GS, 1, S, GS, S, 1, (double *)mb.Q.p, S, S, K, acc, 1, true);   // Q_n += sym(G_S^T G_S)
  if (solve) {
    launch_spd_factor((const double *)mb.Q.p, S, (double *)mb.Qi.p, h->d_info, h->st);
    tl_mark(h, "spd_factor");
  }
  rs_main(h);
  gemm(h, XS, K, 1, GS, S, 1, (double *)mb.P.p, (int)mb.I, S, K, acc);
  RTRY(rs_join(h));
  if (solve) {
    launch_rows_solve((const double *)mb.P.p, (const double *)mb.Qi.p, S, mb.I, (double *)mb.G.p, h->st);
    tl_mark(h, "rows_solve");
  }
  return STR_OK;
}

str_status rstr_init(str_state *h, const void *X, int64_t tn) {
  RTRY(rstr_workspace(h, tn));
  h->tau = 0;
  RCU(cudaMemsetAsync(h->dTau.p, 0, sizeof(int64_t), h->st));
  launch_set_ptr((const void **)h->dX.p, X, h->st);
  tl_mark(h, "set_x");
  const int N = h->N;
  if (h->ksrft()) RTRY(ks_mix(h, tn));   // Alg. 9 l.2-4
  // Alg. 7 l.2-5 / Alg. 8 l.2-6 / Alg. 9 l.5-8: draws for k = 1..N (I_N = t_init)
  for (int k = 1; k <= N; ++k) RTRY(draw_mode(h, k, core_rows(h, k, 0), k == N ? tn : h->md[k - 1].I));
  for (int n = 1; n < N; ++n) RTRY(sampled_normal_eq(h, X, n, tn, 0, false));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    h->err = std::string("rstr_init: ") + cudaGetErrorString(e);
    h->poisoned = true;
    return STR_E_CUDA;
  }
  return STR_OK;
}

// One rSTR step enqueued without host synchronization (Alg. 7 l.6-38 / Alg. 8): the batch enters
// through the device slot, tau advances on the device, the new temporal rows go to the scratch
// GNnew and are appended at the device row counter (as in the STR step), so the whole step can be
// captured as a graph when every draw runs on the device.
static str_status rstr_enqueue(str_state *h, const void *X, int64_t tn) {
  const int N = h->N;
  launch_set_ptr((const void **)h->dX.p, X, h->st);
  tl_mark(h, "set_x");
  if (h->capturing) {
    cudaStreamCaptureStatus cs;
    const cudaGraphNode_t *deps = nullptr;
    size_t nd = 0;
    RCU(cudaStreamGetCaptureInfo(h->st, &cs, nullptr, nullptr, &deps, &nd));
    if (nd != 1) {
      h->err = "cannot locate the captured set_x node";
      return STR_E_CUDA;
    }
    h->gs[h->cur_slot].setx = deps[0];
  }
  k_tau_advance<<<1, 1, 0, h->st>>>((int64_t *)h->dTau.p);
  tl_mark(h, "tau");
  if (h->ksrft()) {   // Alg. 9 l.21-23: new D_j, mixed batch, sampled rows of the re-mixed cores (R19)
    RTRY(ks_mix(h, tn));
    for (int k = 1; k < N; ++k)
      RTRY(ks_sample(h, k, (const double *)h->md[k - 1].G.p, h->md[k - 1].I, (double *)h->md[k - 1].samp.p));
  }
  // temporal: G_N^new = X_S[N] G_S (G_S^T G_S)^{-1}  (Alg. 7 l.17-23, reading R4)
  const int SN = h->SN;
  double *GS = (double *)h->sidx.p;
  double *XS = (double *)h->sX.p;
  double *K = (double *)h->sGram.p;
  double *M = (double *)h->Mt.p;
  double *GN_new = (double *)h->GNnew.p;
  RTRY(chain_and_fibers(h, X, N, tn, GS, XS));
  // rSTR-K: the real halves only, Re(X~) Re(G^) (Re(G^)^T Re(G^))^{-1} (reading R22)
  RTRY(rs_fork(h));   // the Gram and its inverse beside X_S G_S
  gemm(h, GS, 1, SN, GS, SN, 1, K, SN, SN, h->m, 0, 1, true);
  launch_spd_factor(K, SN, (double *)h->Hi.p, h->d_info, h->st);
  tl_mark(h, "spd_factor");
  rs_main(h);
  gemm(h, XS, h->ksrft() ? 2 * h->m : h->m, 1, GS, SN, 1, M, (int)tn, SN, h->m, 0);
  RTRY(rs_join(h));
  launch_rows_solve(M, (const double *)h->Hi.p, SN, tn, GN_new, h->st);
  tl_mark(h, "rows_solve");
  // idxs(:,N) over [t_new]; (G_N^new)_S  (Alg. 7 l.24-25; Alg. 8 l.25-27, reading R9)
  RTRY(draw_mode(h, N, GN_new, tn));
  for (int n = 1; n < N; ++n) {
    ModeBuf &mb = h->md[n - 1];
    RTRY(sampled_normal_eq(h, X, n, tn, 1, true));
    RTRY(draw_mode(h, n, (const double *)mb.G.p, mb.I));
  }
  launch_append_rows((double *)h->GN.p, (int64_t *)h->dT.p, GN_new, tn, SN, h->st);
  tl_mark(h, "append");
  return STR_OK;
}

str_status rstr_update(str_state *h, const void *X, int64_t tn) {
  RTRY(rstr_workspace(h, tn));
  const int N = h->N;
  h->tau++;   // host mirror of the device counter (host-side draws use it)
  RTRY(ensure_temporal_capacity(h, h->T + tn));
  bool forced = false;
  for (int k = 1; k <= N; ++k) forced = forced || !h->forced_idx[k].empty();
  bool dev_ok = h->variant == STR_SAMPLE_UNIFORM;
  if (!dev_ok) {   // weighted draws on the device need each I_k in the shared-memory CDF
    dev_ok = tn <= kDevCdfMax;
    for (auto &mb : h->md) dev_ok = dev_ok && mb.I <= kDevCdfMax;
  }
  const bool graph = h->use_graph && !h->timeline && h->rstr_dev && dev_ok && !forced;
  if (h->profiling && !h->pev[0]) {
    for (auto &e : h->pev) RCU(cudaEventCreate(&e));
  }
  const bool prof = h->profiling && h->ksrft();   // rSTR-K: time the mixing passes
  if (!graph) {
    h->cur_slot = 0;
    RTRY(rstr_enqueue(h, X, tn));
  } else {
    const int slot = prof ? 1 : 0;
    str_state::GraphSlot &g = h->gs[slot];
    if (!g.exec || g.tn != tn) {
      g.reset();
      RCU(cudaStreamBeginCapture(h->st, cudaStreamCaptureModeThreadLocal));
      h->capturing = true;
      h->cur_slot = slot;
      const int64_t l0 = h->launches;
      str_status st = rstr_enqueue(h, X, tn);
      h->capturing = false;
      cudaGraph_t cg = nullptr;
      cudaError_t e = cudaStreamEndCapture(h->st, &cg);
      if (st != STR_OK) {
        if (cg) cudaGraphDestroy(cg);
        return st;
      }
      if (e != cudaSuccess) {
        h->err = std::string("rSTR graph capture: ") + cudaGetErrorString(e);
        return STR_E_CUDA;
      }
      e = cudaGraphInstantiate(&g.exec, cg, h->chain_prio ? cudaGraphInstantiateFlagUseNodePriority : 0);
      if (e != cudaSuccess) {
        cudaGraphDestroy(cg);
        h->err = std::string("rSTR graph instantiate: ") + cudaGetErrorString(e);
        return STR_E_CUDA;
      }
      g.graph = cg;
      g.tn = tn;
      g.launches = h->launches - l0;
      h->launches = l0;
    } else {
      void *slotp = h->dX.p;
      const void *xp = X;
      void *args[2] = {&slotp, &xp};
      cudaKernelNodeParams kp = {};
      kp.func = set_ptr_kernel();
      kp.gridDim = dim3(1);
      kp.blockDim = dim3(1);
      kp.kernelParams = args;
      RCU(cudaGraphExecKernelNodeSetParams(g.exec, g.setx, &kp));
    }
    RCU(cudaGraphLaunch(g.exec, h->st));
    h->launches += g.launches;
    for (int k = 1; k <= N; ++k) h->idx_dev[k] = true;
  }
  if (prof) {
    RCU(cudaStreamSynchronize(h->st));
    float ms = 0.0f;
    if (cudaEventElapsedTime(&ms, h->pev[0], h->pev[1]) == cudaSuccess) {
      h->prof_ms[0] += ms;
      h->prof_n[0] += 1;
    }
  }
  h->T += tn;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    h->err = std::string("rstr_update: ") + cudaGetErrorString(e);
    h->poisoned = true;
    return STR_E_CUDA;
  }
  return STR_OK;
}

extern "C" STR_API str_status str_get_index_table(str_state *h, int32_t mode, int32_t *idx, int64_t m) {
  if (!h || !idx) return STR_E_ARG;
  if (h->variant != STR_DET && mode >= 1 && mode <= h->N && m == h->m && h->idx_dev[mode]) {
    RCU(cudaStreamSynchronize(h->st));   // the table was drawn on the device
    h->last_idx[mode].resize(m);
    RCU(cudaMemcpy(h->last_idx[mode].data(), (const int32_t *)h->sIdxDev.p + (int64_t)(mode - 1) * m,
                   sizeof(int32_t) * m, cudaMemcpyDeviceToHost));
  }
  if (h->variant == STR_DET || mode < 1 || mode > h->N || m != h->m || h->last_idx[mode].empty()) {
    h->err = "no index table for this mode";
    return STR_E_ARG;
  }
  std::copy(h->last_idx[mode].begin(), h->last_idx[mode].end(), idx);
  return STR_OK;
}

extern "C" STR_API str_status str_set_index_table(str_state *h, int32_t mode, const int32_t *idx, int64_t m) {
  if (!h) return STR_E_ARG;
  if (h->variant == STR_DET || mode < 1 || mode > h->N) {
    h->err = "index tables exist only for rSTR modes 1..N";
    return STR_E_ARG;
  }
  if (!idx || m == 0) {
    h->forced_idx[mode].clear();
    return STR_OK;
  }
  if (m != h->m) {
    h->err = "index table length must equal sketch_rows";
    return STR_E_ARG;
  }
  h->forced_idx[mode].assign(idx, idx + m);
  return STR_OK;
}
