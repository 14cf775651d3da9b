// kernels_chain.cu — the fp64 kernels on the serial part of an STR batch (everything R^2-sized):
//   k_chain_gemm_dmma Gram-chain links (×_{2,4}^{1,3} as a matrix product, Def. 5 / Prop. 1)
//                  with the Q_n (+)= H_<2> epilogue (Alg. 4 l.16);
//   k_gram_z2      core Grams Z_n (Alg. 4 l.2/l.18);
//   k_absorb2      second-level contractions of the two-pass intermediates with core slices;
//   k_build_table2 chained-slice tables (⊠₂ chains, Def. 6), fp64 rows and/or the
//                  pre-tiled 3xTF32 hi/lo operand blocks of the tensor-core contraction.
#include <algorithm>

#include <cooperative_groups.h>

#include "common.cuh"
#include "dmma.cuh"
#include "kernels.h"
#include "tc_ptx.cuh"

namespace strb200 {

#ifdef STR_DIAG
int g_dbg_skip = 0;
#endif
constexpr int kAbsorbCps = 3;   // target absorb CTAs per SM (several CTAs overlap staging with compute)

void prepare_kernel_attrs();

__device__ __forceinline__ void cp_async8(void *smem, const void *g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)), "l"(g)
               : "memory");
}
__device__ __forceinline__ void cp_async4(void *smem, const void *g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)), "l"(g)
               : "memory");
}
template <typename T>
__device__ __forceinline__ void cp_async_el(T *smem, const T *g) {
  if (sizeof(T) == 8) cp_async8(smem, g); else cp_async4(smem, g);
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

// ------------------------------------------------------------------------------------------
// 16-byte cp.async (16-byte aligned source and destination)
__device__ __forceinline__ void cp_async16(void *smem, const void *g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)), "l"(g)
               : "memory");
}


// C = A B (fp64, row-major) on the FP64 tensor-core fragments (mma.sync m8n8k4): one 16 x 16
// output tile per CTA (2 x 2 DMMA tiles), 8 warps = 4 tiles x 2 halves of K, so each warp runs one
// accumulator chain over ceil(K/8) k-steps and the halves meet in shared memory.  A rows (stride
// Ka = K rounded to 4 mod 16) and B rows (stride 20) make the fragment loads of a half-warp hit 32
// distinct banks.  Epilogue (q.mode): 0 store C; 1 Q = H_<2>; 2 Q += H_<2>, where C is the chain
// matrix Hm (rows (i1 + Rn r1), columns (i2 + Rn1 r2)) and H_<2>[i1 + Rn i2][r1 + Rn r2] = Hm[..][..]
// (Def. 1 P:126 applied to the chain result; Q is left unsymmetrized, the factorization symmetrizes);
// 3 the Gram regrouping below; 4 the fit sums of str_fit.
constexpr int kGbS = 20;   // B row stride (doubles)
__host__ __device__ inline int gemm_ka(int K) { return (K + 11) / 16 * 16 + 4; }
// TA: A is given transposed (K x M row-major, A_eff[m][k] = A[k M + m]) and staged like B.
// q.mode 3: Gram-chain epilogue, C = G^T G -> Z[(a + Rb c)][(b + Ra d)] = C[b + Ra a][d + Ra c]
// (Ra = q.Rn, Rb = q.Rn1; the layout of k_gram_z2).
template <bool AL16, bool TA>
__global__ void __launch_bounds__(256) k_chain_gemm_dmma(const double *__restrict__ A, const double *__restrict__ B,
                                                         double *__restrict__ C, int M, int N, int K, QEpi q) {
  // PDL: the dependents may launch at once; the old Q values of the accumulate epilogue (written only
  // by this kernel's instance in the previous step) are fetched before the wait for the predecessor,
  // A and B after it (under stream capture every dependency of a programmatic launch, event-joined
  // ones included, becomes programmatic, so no operand is known complete at launch)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ __align__(16) double gsm[];
  const int Ka = TA ? 0 : gemm_ka(K), K4 = (K + 3) / 4 * 4;
  double *As = gsm;                 // [16][Ka], or TA: [K4][kGbS]
  double *Bs = gsm + (TA ? K4 * kGbS : 16 * Ka);   // [K4][kGbS]
  double *Rs = Bs + K4 * kGbS;      // [4 tiles][32 lanes][2] partials of the upper K half
  const int row0 = blockIdx.y * 16, col0 = blockIdx.x * 16;
  const int mr = min(16, M - row0), nc = min(16, N - col0);
  // zero-fill: A rows >= mr and k >= K; B rows k >= K and columns >= nc
  if (TA) {
    for (int e = threadIdx.x; e < (K4 - K) * 16; e += 256) As[(K + e / 16) * kGbS + e % 16] = 0.0;
    if (mr < 16)
      for (int e = threadIdx.x; e < K * (16 - mr); e += 256) As[(e / (16 - mr)) * kGbS + mr + e % (16 - mr)] = 0.0;
  } else {
    for (int e = threadIdx.x; e < 16 * (K4 - K); e += 256) As[(e / (K4 - K)) * Ka + K + e % (K4 - K)] = 0.0;
    for (int e = threadIdx.x; e < (16 - mr) * K; e += 256) As[(mr + e / K) * Ka + e % K] = 0.0;
  }
  for (int e = threadIdx.x; e < (K4 - K) * 16; e += 256) Bs[(K + e / 16) * kGbS + e % 16] = 0.0;
  if (nc < 16)
    for (int e = threadIdx.x; e < K * (16 - nc); e += 256) Bs[(e / (16 - nc)) * kGbS + nc + e % (16 - nc)] = 0.0;
  auto stage_b = [&]() {
    if (AL16) {
      const int n2 = nc >> 1;
      for (int e = threadIdx.x; e < K * n2; e += 256) {
        const int k = e / n2, c = 2 * (e - k * n2);
        cp_async16(Bs + k * kGbS + c, B + (int64_t)k * N + col0 + c);
      }
    } else {
      for (int e = threadIdx.x; e < K * nc; e += 256) {
        const int k = e / nc, c = e - k * nc;
        cp_async8(Bs + k * kGbS + c, B + (int64_t)k * N + col0 + c);
      }
    }
  };
  // the accumulate epilogue's old values (warps 0-3 store; Q is not written by the predecessor)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tg = lane & 3;
  const int tile = warp & 3, half = warp >> 2, ti = tile >> 1, tj = tile & 1;
  const int row = row0 + 8 * ti + g;
  double *qd[2] = {nullptr, nullptr};
  double qo[2] = {0.0, 0.0};
  if (!half && (q.mode == 1 || q.mode == 2)) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int col = col0 + 8 * tj + 2 * tg + e;
      if (row < M && col < N) {
        const int i1 = row % q.Rn, r1 = row / q.Rn, i2 = col % q.Rn1, r2 = col / q.Rn1;
        const int S = q.Rn * q.Rn1;
        qd[e] = q.Q + (int64_t)(i1 + q.Rn * i2) * S + (r1 + q.Rn * r2);
        if (q.mode == 2) qo[e] = *qd[e];
      }
    }
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  stage_b();
  if (AL16) {
    const int K2 = K >> 1, m2 = mr >> 1;
    if (TA) {
      for (int e = threadIdx.x; e < K * m2; e += 256) {
        const int k = e / m2, c = 2 * (e - k * m2);
        cp_async16(As + k * kGbS + c, A + (int64_t)k * M + row0 + c);
      }
    } else {
      for (int e = threadIdx.x; e < mr * K2; e += 256) {
        const int r = e / K2, c = 2 * (e - r * K2);
        cp_async16(As + r * Ka + c, A + (int64_t)(row0 + r) * K + c);
      }
    }
  } else {
    if (TA) {
      for (int e = threadIdx.x; e < K * mr; e += 256) {
        const int k = e / mr, c = e - k * mr;
        cp_async8(As + k * kGbS + c, A + (int64_t)k * M + row0 + c);
      }
    } else {
      for (int e = threadIdx.x; e < mr * K; e += 256) {
        const int r = e / K, c = e - r * K;
        cp_async8(As + r * Ka + c, A + (int64_t)(row0 + r) * K + c);
      }
    }
  }
  cp_async_wait_all();
  __syncthreads();
  const int nks = K4 / 4, ks0 = half ? (nks + 1) / 2 : 0, ks1 = half ? nks : (nks + 1) / 2;
  double c0 = 0.0, c1 = 0.0;
  const double *bp = Bs + tg * kGbS + 8 * tj + g;
  if (TA) {
    const double *ap = As + tg * kGbS + 8 * ti + g;
#pragma unroll 4
    for (int ks = ks0; ks < ks1; ++ks) dmma(c0, c1, ap[4 * ks * kGbS], bp[4 * ks * kGbS]);
  } else {
    const double *ap = As + (8 * ti + g) * Ka + tg;
#pragma unroll 4
    for (int ks = ks0; ks < ks1; ++ks) dmma(c0, c1, ap[4 * ks], bp[4 * ks * kGbS]);
  }
  if (half) {
    Rs[(tile * 32 + lane) * 2] = c0;
    Rs[(tile * 32 + lane) * 2 + 1] = c1;
  }
  __syncthreads();
  if (half) return;
  c0 += Rs[(tile * 32 + lane) * 2];
  c1 += Rs[(tile * 32 + lane) * 2 + 1];
  if (q.mode == 4) {   // fit: residual and norm sums of this tile (warps 0-3), fixed-order partials
    double d2 = 0.0, x2 = 0.0;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int col = col0 + 8 * tj + 2 * tg + e;
      if (row < M && col < N) {
        const int64_t l = row % q.L, t = row / q.L;
        const int64_t off = l + q.L * col + q.L * q.Rr * t;
        const double x = q.xf64 ? ((const double *)q.X)[off] : (double)((const float *)q.X)[off];
        const double dv = x - (e ? c1 : c0);
        d2 = fma(dv, dv, d2);
        x2 = fma(x, x, x2);
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      d2 += __shfl_xor_sync(0xffffffffu, d2, o);
      x2 += __shfl_xor_sync(0xffffffffu, x2, o);
    }
    if (lane == 0) {
      Rs[256 + 2 * warp] = d2;
      Rs[256 + 2 * warp + 1] = x2;
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");   // the four epilogue warps
    if (threadIdx.x == 0)
      q.part[blockIdx.x + (int64_t)gridDim.x * blockIdx.y] =
          make_double2((Rs[256] + Rs[258]) + (Rs[260] + Rs[262]), (Rs[257] + Rs[259]) + (Rs[261] + Rs[263]));
    return;
  }
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int col = col0 + 8 * tj + 2 * tg + e;
    const double v = e ? c1 : c0;
    if (row < M && col < N) {
      if (q.mode == 0) {
        C[(int64_t)row * N + col] = v;
      } else if (q.mode == 3) {
        const int Ra = q.Rn, Rb = q.Rn1;
        const int a = row / Ra, b = row - a * Ra, c = col / Ra, d = col - c * Ra;
        q.Q[(int64_t)(a + Rb * c) * (Ra * Ra) + (b + Ra * d)] = v;
      } else {
        *qd[e] = qo[e] + v;   // (modes 1 / 2: every old value of this tile was loaded above)
      }
    }
  }
}

static size_t gemm_dmma_smem(int K) {
  const size_t k4 = (size_t)(K + 3) / 4 * 4;
  return sizeof(double) * (std::max((size_t)16 * gemm_ka(K), k4 * kGbS) + k4 * kGbS + 4 * 32 * 2 + 8);
}

// TRp[p Rb + q][r] = TR[r][q Ra + p]: T_R rows as the K x N operand of the fit GEMM
__global__ void k_fit_perm_tr(const double *__restrict__ TR, int Ra, int Rb, int64_t Rr, double *__restrict__ TRp) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int W = Ra * Rb;
  if (e >= (int64_t)W * Rr) return;
  const int64_t w = e / Rr, r = e - w * Rr;
  const int p = (int)(w / Rb), qq = (int)(w - (int64_t)p * Rb);
  TRp[e] = TR[r * W + qq * Ra + p];
}

// ||X - TL TR^T||^2 and ||X||^2 of tn slices on the fragment GEMM with the fit epilogue.
template <bool AL16, bool TA>
static void launch_dmma_pdl(dim3 gd, size_t smd, cudaStream_t s, const double *A, const double *B, double *C, int M,
                            int N, int K, QEpi q);

int launch_fit_gemm(const void *X, bool x_is_f64, const double *TLf, const double *TR, int Ra, int Rb, int64_t L,
                    int64_t Rr, int64_t tn, double *TRp, double2 *partials, double *acc2, cudaStream_t s) {
  prepare_kernel_attrs();
  const int W = Ra * Rb;
  k_fit_perm_tr<<<(unsigned)cdiv((int64_t)W * Rr, 256), 256, 0, s>>>(TR, Ra, Rb, Rr, TRp);
  const int M = (int)(L * tn), N = (int)Rr;
  dim3 gd((unsigned)cdiv(N, 16), (unsigned)cdiv(M, 16));
  QEpi q{nullptr, 0, 0, 4};
  q.X = X;
  q.L = L;
  q.Rr = Rr;
  q.xf64 = x_is_f64 ? 1 : 0;
  q.part = partials;
  const size_t smd = gemm_dmma_smem(W);
  const bool al16 = (W % 2 == 0) && (N % 2 == 0);
  if (al16)
    launch_dmma_pdl<true, false>(gd, smd, s, TLf, TRp, nullptr, M, N, W, q);
  else
    launch_dmma_pdl<false, false>(gd, smd, s, TLf, TRp, nullptr, M, N, W, q);
  launch_fit_reduce(partials, (int64_t)gd.x * gd.y, acc2, s);
  return 3;
}
size_t fit_gemm_partials(int64_t L, int64_t Rr, int64_t tn) { return (size_t)cdiv(Rr, 16) * cdiv(L * tn, 16); }

// k_chain_gemm_dmma with the programmatic-stream-serialization attribute (PDL; STR_PDL=0 disables)
template <bool AL16, bool TA>
static void launch_dmma_pdl(dim3 gd, size_t smd, cudaStream_t s, const double *A, const double *B, double *C, int M,
                            int N, int K, QEpi q) {
  const bool on = (pdl_mask() & kPdlDmma) != 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = gd;
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smd;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = on ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k_chain_gemm_dmma<AL16, TA>, A, B, C, M, N, K, q);
}

void launch_chain_gemm(const double *A, const double *B, double *C, int M, int N, int K, QEpi q, cudaStream_t s) {
  if (g_dbg_skip & 16) return;
  prepare_kernel_attrs();
  constexpr int kMaxRows = 65535 * 16;   // gridDim.y limit: taller plain products run in row chunks
  if (M > kMaxRows && q.mode == 0) {
    for (int r0 = 0; r0 < M; r0 += kMaxRows)
      launch_chain_gemm(A + (int64_t)r0 * K, B, C + (int64_t)r0 * N, std::min(kMaxRows, M - r0), N, K, q, s);
    return;
  }
  const bool al16 = (K % 2 == 0) && (N % 2 == 0) && ((uintptr_t)A % 16 == 0) && ((uintptr_t)B % 16 == 0);
  dim3 gd((unsigned)cdiv(N, 16), (unsigned)cdiv(M, 16));
  const size_t smd = gemm_dmma_smem(K);
  if (al16)
    launch_dmma_pdl<true, false>(gd, smd, s, A, B, C, M, N, K, q);
  else
    launch_dmma_pdl<false, false>(gd, smd, s, A, B, C, M, N, K, q);
}


// ------------------------------------------------------------------------------------------
// Gram tensor as a chain matrix: Zm[(a + Rb c)][(b + Ra d)] = sum_i G(i)(b,a) G(i)(d,c) (Z of
// P:228, rows = (1st,3rd) index pair, columns = (2nd,4th)); G(i) = Ra x Rb slices in G(2) layout.
// Thread per output entry; rows of G staged in shared memory in chunks.
constexpr int kGramSmem = 6144;   // doubles

__global__ void __launch_bounds__(256) k_gram_z2(const double *__restrict__ G, int64_t I, int Ra, int Rb,
                                                 double *__restrict__ Zm, int accumulate) {
  __shared__ double Gs[kGramSmem];
  const int AB = Ra * Rb;
  const int ch = kGramSmem / AB;
  const int rows = Rb * Rb, cols = Ra * Ra;
  const int gid = blockIdx.x * 256 + threadIdx.x;
  const bool act = gid < rows * cols;
  const int row = act ? gid / cols : 0, col = act ? gid % cols : 0;
  const int a = row % Rb, c = row / Rb, b = col % Ra, d = col / Ra;
  const int o1 = b + Ra * a, o2 = d + Ra * c;
  double acc0 = 0.0, acc1 = 0.0;
  for (int64_t i0 = 0; i0 < I; i0 += ch) {
    const int ic = (int)((I - i0) < ch ? (I - i0) : ch);
    __syncthreads();
    for (int e = threadIdx.x; e < ic * AB; e += 256) cp_async8(Gs + e, G + i0 * AB + e);
    cp_async_wait_all();
    __syncthreads();
    int i = 0;
    for (; i + 2 <= ic; i += 2) {
      acc0 = fma(Gs[i * AB + o1], Gs[i * AB + o2], acc0);
      acc1 = fma(Gs[(i + 1) * AB + o1], Gs[(i + 1) * AB + o2], acc1);
    }
    if (i < ic) acc0 = fma(Gs[i * AB + o1], Gs[i * AB + o2], acc0);
  }
  if (act) {
    const double v = acc0 + acc1;
    if (accumulate) Zm[gid] += v; else Zm[gid] = v;
  }
}

void launch_gram_z2(const double *G, int64_t I, int Ra, int Rb, double *Zm, int accumulate, cudaStream_t s) {
  if (g_dbg_skip & 64) return;
  const int S = Ra * Rb;
  const size_t smd = gemm_dmma_smem((int)I);
  if (!accumulate && I > 0 && smd <= 160 * 1024) {   // G^T G on the FP64 tensor-core fragments
    prepare_kernel_attrs();
    dim3 gd((unsigned)cdiv(S, 16), (unsigned)cdiv(S, 16));
    const QEpi q{Zm, Ra, Rb, 3};
    if (S % 2 == 0 && (uintptr_t)G % 16 == 0)
      launch_dmma_pdl<true, true>(gd, smd, s, G, G, nullptr, S, S, (int)I, q);
    else
      launch_dmma_pdl<false, true>(gd, smd, s, G, G, nullptr, S, S, (int)I, q);
    return;
  }
  const int n = Ra * Ra * Rb * Rb;
  k_gram_z2<<<(unsigned)cdiv(n, 256), 256, 0, s>>>(G, I, Ra, Rb, Zm, accumulate);
}

// ------------------------------------------------------------------------------------------
// Absorb (AbsorbDesc): contract index `pos` of the matrix-valued tensor Y with core slices.
//   left : out[rest][po][qo] = sum_i sum_p A(i)[po][p] Y(rest, i)[p][qo]
//   right: out[rest][po][qo] = sum_i sum_q Y(rest, i)[po][q] A(i)[q][qo]
// Generic form: out vector index u (po | qo, length L), vector index v (qo | po, V of them),
// contracted p (p | q, R).  A thread owns VB consecutive v of one rest and one k-split ks of the
// contracted index i; it keeps VB x L accumulators in registers (register-blocked micro-GEMM:
// per (i, p) L broadcast loads of A from shared memory and VB loads of Y feed VB x L FMAs).  The
// A slices are staged in shared memory (cp.async) in chunks of i; the KS partials are reduced in
// shared memory in a fixed order (deterministic).
constexpr int kAbsVB = 2;

template <typename TY, int MR, bool LEFT>
__global__ void __launch_bounds__(256) k_absorb4(AbsorbDesc ad, const TY *__restrict__ Y, double *__restrict__ out,
                                                 int accumulate, int64_t before, int64_t I, int64_t nrest, int KS,
                                                 int ic_max) {
  extern __shared__ __align__(16) double asm_[];
  const int AB = ad.Ra * ad.Rb, PQ = ad.P * ad.Q;
  const int Po = LEFT ? ad.Ra : ad.P, Qo = LEFT ? ad.Q : ad.Rb;
  const int L = LEFT ? Po : Qo, V = LEFT ? Qo : Po, R = LEFT ? ad.P : ad.Q;
  const int nvb = (V + kAbsVB - 1) / kAbsVB;
  const int per_ks = blockDim.x / KS;                      // (rest, vblk) pairs per CTA
  double *As = asm_;                                        // ic_max * AB
  double *red = asm_ + ((ic_max * AB + 1) & ~1);           // KS * per_ks * kAbsVB * MR
  const int tid = threadIdx.x;
  const int ks = tid / per_ks, pr = tid % per_ks;
  const int64_t pair = (int64_t)blockIdx.x * per_ks + pr;
  const int64_t rest = pair / nvb;
  const int v0 = (int)(pair % nvb) * kAbsVB;
  const bool act = rest < nrest && ks < KS;        // (threads beyond KS * per_ks idle)
  const int64_t b0 = act ? rest % before : 0, a0 = act ? rest / before : 0;
  const TY *yb = Y + (b0 + before * I * a0) * PQ;
  const int64_t ystride = before * PQ;
  const int a_ps = LEFT ? ad.Ra : 1, a_us = LEFT ? 1 : ad.Ra;     // A(i): p and u strides
  const int y_ps = LEFT ? ad.Q : 1, y_vs = LEFT ? 1 : ad.Q;       // Y(rest,i): p and v strides
  double acc[kAbsVB][MR];
#pragma unroll
  for (int b = 0; b < kAbsVB; ++b)
#pragma unroll
    for (int u = 0; u < MR; ++u) acc[b][u] = 0.0;
  for (int64_t i0 = 0; i0 < I; i0 += ic_max) {
    const int ic = (int)((I - i0) < ic_max ? (I - i0) : ic_max);
    __syncthreads();
    for (int e = tid; e < ic * AB; e += blockDim.x) cp_async8(As + e, ad.A + i0 * AB + e);
    cp_async_wait_all();
    __syncthreads();
    if (act) {
      // this thread's i in the chunk: i = i0 + j with (i0 + j) % KS == ks
      int j = (int)((ks - i0 % KS + KS) % KS);
      for (; j < ic; j += KS) {
        const double *Ai = As + j * AB;
        const TY *yi = yb + (i0 + j) * ystride;
        // all Y loads of this slice first (one memory latency per slice), then the FMAs
        double yv[MR][kAbsVB];
#pragma unroll
        for (int p = 0; p < MR; ++p)
#pragma unroll
          for (int b = 0; b < kAbsVB; ++b)
            yv[p][b] = (p < R && v0 + b < V) ? (double)__ldg(yi + p * y_ps + (v0 + b) * y_vs) : 0.0;
#pragma unroll
        for (int p = 0; p < MR; ++p) {
          if (p < R) {
            double av[MR];
#pragma unroll
            for (int u = 0; u < MR; ++u) av[u] = (u < L) ? Ai[p * a_ps + u * a_us] : 0.0;
#pragma unroll
            for (int b = 0; b < kAbsVB; ++b)
#pragma unroll
              for (int u = 0; u < MR; ++u) acc[b][u] = fma(av[u], yv[p][b], acc[b][u]);
          }
        }
      }
    }
  }
  if (KS > 1) {
    __syncthreads();
    if (ks < KS) {
      double *rp = red + ((int64_t)ks * per_ks + pr) * (kAbsVB * MR);
#pragma unroll
      for (int b = 0; b < kAbsVB; ++b)
#pragma unroll
        for (int u = 0; u < MR; ++u) rp[b * MR + u] = acc[b][u];
    }
    __syncthreads();
    if (ks != 0) return;
    for (int k = 1; k < KS; ++k) {
      const double *rk = red + ((int64_t)k * per_ks + pr) * (kAbsVB * MR);
#pragma unroll
      for (int b = 0; b < kAbsVB; ++b)
#pragma unroll
        for (int u = 0; u < MR; ++u) acc[b][u] += rk[b * MR + u];
    }
  }
  if (!act) return;
  const int O = Po * Qo;
#pragma unroll
  for (int b = 0; b < kAbsVB; ++b) {
    if (v0 + b >= V) continue;
#pragma unroll
    for (int u = 0; u < MR; ++u) {
      if (u < L) {
        const int po = LEFT ? u : v0 + b, qo = LEFT ? v0 + b : u;
        double *dst = out + rest * O + po * Qo + qo;
        if (accumulate) *dst += acc[b][u]; else *dst = acc[b][u];
      }
    }
  }
}

// Absorb on the FP64 tensor-core fragments (mma.sync m8n8k4).  For a CTA of RB rests the absorb is
// a GEMM whose large dimension stacks (rest, free rank) and whose small dimension is the new rank:
//   left:  D[u][(r, q)] = sum_{(i, p)} A(i)[u][p] Y(r, i)[p][q]     (M = Ra small, N = RB Q)
//   right: D[(r, p)][v] = sum_{(i, q)} Y(r, i)[p][q] A(i)[q][v]     (M = RB P, N = Rb small)
// K runs over (i, c) with the contracted rank c padded to a multiple of 4 (zero fragments), split
// over KW warp groups that meet in shared memory.  Y blocks and A chunks arrive by bulk copies.
template <typename TY, bool LEFT>
__global__ void __launch_bounds__(256) k_absorb6(AbsorbDesc ad, const TY *__restrict__ Y, double *__restrict__ out,
                                                 int accumulate, int before, int I, int nrest, int RB, int ic, int KW) {
  PDL_PROLOGUE();
  extern __shared__ __align__(16) double asm6[];
  const int AB = ad.Ra * ad.Rb, PQ = ad.P * ad.Q;
  const int Cb = LEFT ? ad.Q : ad.P;        // free rank carried along the large dimension
  const int Sm = LEFT ? ad.Ra : ad.Rb;      // new rank (small dimension, <= 16)
  const int C = LEFT ? ad.P : ad.Q;         // contracted rank
  const int O = LEFT ? ad.Ra * ad.Q : ad.P * ad.Rb;
  const int nc4 = (C + 3) >> 2;
  double *As = asm6;                                              // [ic][AB]
  TY *Ys = (TY *)(asm6 + ((ic * AB + 1) & ~1));                   // [RB][ic][PQ]
  double *Rd = (double *)(Ys + ((RB * ic * PQ * (int)sizeof(TY) + 15) / 16) * (16 / (int)sizeof(TY)));
  __shared__ __align__(8) uint64_t bar;
  const int rest0 = blockIdx.x * RB;
  const int nr = min(RB, nrest - rest0);
  const int NB = RB * Cb, nbt = (NB + 7) >> 3;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tg = lane & 3;
  const int bt = warp % nbt, kw = warp / nbt;
  const bool wact = kw < KW;
  // this lane's large-dimension index (fragment row/col g of big tile bt)
  const int nb = 8 * bt + g;
  const int rb = nb / Cb, cb = nb - rb * Cb;
  const bool nbv = rb < nr;
  // accumulator fragment: row g, columns 2 tg + e of the 8 x 8 tile.  The destinations and, when
  // accumulating, their old values (P_n of the previous step: nothing in this step writes them
  // before this kernel) are fetched here, before the staging and the products, so their latency
  // overlaps them; every old value is loaded before any store (a load-add-store per element
  // would serialize on the possible aliasing).  Only the storing warps (kw == 0) fetch.
  double *dsts[2][2];
  double olds[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
  for (int s2 = 0; s2 < 2; ++s2) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      dsts[s2][e] = nullptr;
      int rest, idx;
      if (LEFT) {   // D[u][n]: u = 8 s2 + g, n = 8 bt + 2 tg + e
        const int u = 8 * s2 + g, n = 8 * bt + 2 * tg + e, r = n / Cb, q = n - r * Cb;
        if (u >= Sm || r >= nr) continue;
        rest = rest0 + r;
        idx = u * ad.Q + q;
      } else {      // D[m][v]: m = 8 bt + g, v = 8 s2 + 2 tg + e
        const int v = 8 * s2 + 2 * tg + e;
        if (v >= Sm || !nbv) continue;
        rest = rest0 + rb;
        idx = cb * ad.Rb + v;
      }
      dsts[s2][e] = out + (int64_t)rest * O + idx;
      if (accumulate && kw == 0 && wact) olds[s2][e] = *dsts[s2][e];
    }
  }
  double c[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_barrier_init();
  }
  uint32_t ph = 0;
  for (int i0 = 0; i0 < I; i0 += ic) {
    const int icn = min(ic, I - i0);
    __syncthreads();
    if (threadIdx.x < 32) {
      if (threadIdx.x == 0)
        tc::mbar_arrive_expect_tx(&bar, (uint32_t)(icn * AB * 8 + nr * icn * PQ * (int)sizeof(TY)));
      __syncwarp();
      if (threadIdx.x == 0) tc::bulk_load(As, ad.A + (int64_t)i0 * AB, (uint32_t)(icn * AB * 8), &bar);
      for (int e = threadIdx.x; e < nr * icn; e += 32) {
        const int r = e / icn, ii = e - r * icn, rr = rest0 + r;
        const int b0 = rr % before, a0 = rr / before;
        tc::bulk_load(Ys + (r * ic + ii) * PQ, Y + ((int64_t)b0 + (int64_t)before * (i0 + ii + (int64_t)I * a0)) * PQ,
                      (uint32_t)(PQ * sizeof(TY)), &bar);
      }
    }
    tc::mbar_wait(&bar, ph);
    ph ^= 1;
    if (wact) {
      // K = (i, c): warp group kw takes i = kw, kw + KW, ...; per i ceil(C/4) k-steps of 4 ranks
      const TY *yrow = Ys + (size_t)rb * ic * PQ + (LEFT ? cb : cb * ad.Q);   // + i PQ + (LEFT ? c Q : c)
      const int ystep = LEFT ? 4 * ad.Q : 4, yoff = LEFT ? tg * ad.Q : tg;
      const int sm0 = g, sm1 = 8 + g;
      const int aoff0 = LEFT ? sm0 + ad.Ra * tg : tg + ad.Ra * sm0;
      const int aoff1 = LEFT ? sm1 + ad.Ra * tg : tg + ad.Ra * sm1;
      const int astep = LEFT ? 4 * ad.Ra : 4;
      const bool two = Sm > 8;
      for (int i = kw; i < icn; i += KW) {
        const TY *yi = yrow + i * PQ + yoff;
        const double *Ai = As + i * AB;
        for (int j = 0; j < nc4; ++j) {
          const bool cv = 4 * j + tg < C;
          const double yv = (nbv && cv) ? (double)yi[j * ystep] : 0.0;
          const double av0 = (sm0 < Sm && cv) ? Ai[aoff0 + j * astep] : 0.0;
          if (LEFT) dmma(c[0][0], c[0][1], av0, yv); else dmma(c[0][0], c[0][1], yv, av0);
          if (two) {
            const double av1 = (sm1 < Sm && cv) ? Ai[aoff1 + j * astep] : 0.0;
            if (LEFT) dmma(c[1][0], c[1][1], av1, yv); else dmma(c[1][0], c[1][1], yv, av1);
          }
        }
      }
    }
  }
  if (KW > 1) {
    if (wact && kw > 0) {
      double *rp = Rd + ((size_t)((kw - 1) * nbt + bt) * 32 + lane) * 4;
      rp[0] = c[0][0];
      rp[1] = c[0][1];
      rp[2] = c[1][0];
      rp[3] = c[1][1];
    }
    __syncthreads();
    if (!wact || kw > 0) return;
    for (int k2 = 1; k2 < KW; ++k2) {
      const double *rp = Rd + ((size_t)((k2 - 1) * nbt + bt) * 32 + lane) * 4;
      c[0][0] += rp[0];
      c[0][1] += rp[1];
      c[1][0] += rp[2];
      c[1][1] += rp[3];
    }
  } else if (!wact) {
    return;
  }
#pragma unroll
  for (int s2 = 0; s2 < 2; ++s2)
#pragma unroll
    for (int e = 0; e < 2; ++e)
      if (dsts[s2][e]) *dsts[s2][e] = olds[s2][e] + c[s2][e];
}

template <typename TY>
static bool absorb6_launch(const AbsorbDesc &ad, const TY *Y, double *out, int accumulate, int64_t nrest, int64_t before,
                           int64_t I, cudaStream_t s) {
  const bool left = ad.left != 0;
  const int Sm = left ? ad.Ra : ad.Rb, Cb = left ? ad.Q : ad.P;
  const int AB = ad.Ra * ad.Rb, PQ = ad.P * ad.Q;
  if (Sm > 16 || nrest >= ((int64_t)1 << 31) || before * I * nrest >= ((int64_t)1 << 40)) return false;
  if ((PQ * (int)sizeof(TY)) % 16 != 0 || (AB * 8) % 16 != 0 || (uintptr_t)Y % 16 != 0 || (uintptr_t)ad.A % 16 != 0)
    return false;
  // rests per CTA: enough CTAs to cover the GPU, at most 8 big tiles (one warp each)
  int RB = (int)std::max<int64_t>(1, std::min<int64_t>(nrest / (148 * kAbsorbCps), 64 / std::max(1, Cb)));
  const int nbt = (RB * Cb + 7) / 8;
  const int KW = (int)std::max<int64_t>(1, std::min<int64_t>(8 / nbt, I));
  const int threads = std::max(32, std::min(256, nbt * KW * 32));
  const size_t per_i = 8 * (size_t)AB + sizeof(TY) * (size_t)RB * PQ;
  const int ic = (int)std::min<int64_t>(I, std::max<int64_t>(1, (96 * 1024) / (int64_t)per_i));
  const size_t ybytes = ((size_t)RB * ic * PQ * sizeof(TY) + 15) / 16 * 16;
  const size_t smem = sizeof(double) * (((size_t)ic * AB + 1) & ~1) + ybytes + sizeof(double) * (size_t)(KW - 1) * nbt * 32 * 4;
  if (smem > 160 * 1024) return false;
  const unsigned grid = (unsigned)cdiv(nrest, RB);
  if (left)
    pdl_launch(kPdlAbsorb, k_absorb6<TY, true>, grid, dim3(threads), smem, s, ad, Y, out, accumulate, (int)before, (int)I, (int)nrest,
               RB, ic, KW);
  else
    pdl_launch(kPdlAbsorb, k_absorb6<TY, false>, grid, dim3(threads), smem, s, ad, Y, out, accumulate, (int)before, (int)I,
               (int)nrest, RB, ic, KW);
  return true;
}

template <typename TY, int MR>
static void absorb_launch(const AbsorbDesc &ad, const TY *Y, double *out, int accumulate, int64_t nrest,
                          int64_t before, int64_t I, cudaStream_t s) {
  const bool left = ad.left != 0;
  const int Po = left ? ad.Ra : ad.P, Qo = left ? ad.Q : ad.Rb;
  const int V = left ? Qo : Po;
  const int nvb = (V + kAbsVB - 1) / kAbsVB;
  const int64_t pairs = nrest * nvb;
  // k-splits: aim for ~148 x 128 threads, each thread >= 2 contracted slices
  int KS = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(148 * 128, pairs), I / 2));
  if (KS > 32) KS = 32;
  int threads = 128;
  while (threads < 256 && threads / KS < 4) threads *= 2;
  if (KS > threads) KS = threads;
  const int per_ks = threads / KS;
  const int AB = ad.Ra * ad.Rb;
  int ic = (int)std::min<int64_t>(I, std::max<int64_t>(1, 8192 / AB));   // <= 64 KB of A per chunk
  const size_t smem = sizeof(double) * (((size_t)ic * AB + 1) & ~1) +
                      (KS > 1 ? sizeof(double) * KS * per_ks * kAbsVB * MR : 0);
  const unsigned grid = (unsigned)cdiv(pairs, per_ks);
  if (left)
    k_absorb4<TY, MR, true><<<grid, threads, smem, s>>>(ad, Y, out, accumulate, before, I, nrest, KS, ic);
  else
    k_absorb4<TY, MR, false><<<grid, threads, smem, s>>>(ad, Y, out, accumulate, before, I, nrest, KS, ic);
}

template <typename TY>
static void absorb_dispatch(const AbsorbDesc &ad, const TY *Y, double *out, int accumulate, int64_t nrest,
                            int64_t before, int64_t I, cudaStream_t s) {
  // k_absorb6 (FP64 tensor-core fragments) unless the shape or alignment rules it out (e.g. fp32 Y
  // blocks that are not a whole number of 16-byte chunks); then the register-blocked k_absorb4
  if (absorb6_launch<TY>(ad, Y, out, accumulate, nrest, before, I, s)) return;
  // MR bounds both the accumulator length (Ra | Rb) and the contracted rank (P | Q)
  const int L = std::max(ad.left ? ad.Ra : ad.Rb, ad.left ? ad.P : ad.Q);
  if (L <= 4)
    absorb_launch<TY, 4>(ad, Y, out, accumulate, nrest, before, I, s);
  else if (L <= 8)
    absorb_launch<TY, 8>(ad, Y, out, accumulate, nrest, before, I, s);
  else if (L <= 10)
    absorb_launch<TY, 10>(ad, Y, out, accumulate, nrest, before, I, s);
  else
    absorb_launch<TY, STR_MAXR>(ad, Y, out, accumulate, nrest, before, I, s);
}

template <typename TY>
static void absorb_attrs() {
  const int mx = 160 * 1024;
  cudaFuncSetAttribute(k_absorb6<TY, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(k_absorb6<TY, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  prefer_max_smem(k_absorb6<TY, true>);
  prefer_max_smem(k_absorb6<TY, false>);
  cudaFuncSetAttribute(k_absorb4<TY, 4, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(k_absorb4<TY, 4, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(k_absorb4<TY, 8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(k_absorb4<TY, 8, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(k_absorb4<TY, 10, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(k_absorb4<TY, 10, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(k_absorb4<TY, STR_MAXR, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(k_absorb4<TY, STR_MAXR, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  prefer_max_smem(k_absorb4<TY, 4, true>);
  prefer_max_smem(k_absorb4<TY, 4, false>);
  prefer_max_smem(k_absorb4<TY, 8, true>);
  prefer_max_smem(k_absorb4<TY, 8, false>);
  prefer_max_smem(k_absorb4<TY, 10, true>);
  prefer_max_smem(k_absorb4<TY, 10, false>);
  prefer_max_smem(k_absorb4<TY, STR_MAXR, true>);
  prefer_max_smem(k_absorb4<TY, STR_MAXR, false>);
}

void launch_absorb2(const AbsorbDesc &ad, const void *Y, bool y_f32, double *out, int accumulate, cudaStream_t s) {
  if (g_dbg_skip & 8) return;
  prepare_kernel_attrs();
  int64_t rest = 1, before = 1;
  for (int j = 0; j < ad.nd; ++j)
    if (j != ad.pos) rest *= ad.d[j];
  for (int j = 0; j < ad.pos; ++j) before *= ad.d[j];
  const int64_t I = ad.d[ad.pos];
  if (y_f32)
    absorb_dispatch<float>(ad, (const float *)Y, out, accumulate, rest, before, I, s);
  else
    absorb_dispatch<double>(ad, (const double *)Y, out, accumulate, rest, before, I, s);
}

// ------------------------------------------------------------------------------------------
// Chained slice table over work units (t', lb): entries e = l + Lk t' for l in [32 lb, 32 lb + 32)
// ∩ [0, Lk).  Entry e is F_0(i_0) F_1(i_1) ... (i_f = (e / stride_f) % I_f), R0 x Rl.  The slices
// a unit touches (a contiguous index range per factor) are staged in shared memory; thread
// (entry, row p) carries row p through the chain in registers.  Outputs: fp64 rows
// out64[e][p][q] (optional) and/or the pre-tiled 3xTF32 operand block kt = t' nlb + lb: rows
// n < Np hold hi(w = p Rl + q), rows Np + n hold lo, 32 k-columns, 16-byte chunk c of row n at
// chunk c ^ (n % 8) (128B swizzle) — assembled in shared memory, stored contiguously.
__device__ __forceinline__ float tf32_rna(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}

template <int MR>
__global__ void k_build_table2(TableDesc td, double *__restrict__ out64, float *__restrict__ tiles) {
  if (td.zero)   // the next contraction's output (one node fewer per pass)
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < td.zero_n4; i += (int64_t)gridDim.x * blockDim.x)
      td.zero[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  // all index arithmetic in 32 bits (the host checks Lk * tk < 2^31): 64-bit division and modulo
  // are emulated and used to dominate this kernel
  extern __shared__ __align__(16) double tsm[];
  const int Lk = (int)td.Lk;
  const int nlb = (Lk + 31) / 32;
  const int unit = blockIdx.x;
  const int tp = unit / nlb;
  const int lb = unit - tp * nlb;
  const int l0 = lb * 32;
  const int l1 = (l0 + 32 < Lk) ? l0 + 32 : Lk;
  const int e_lo = l0 + Lk * tp, e_hi = l1 - 1 + Lk * tp;
  const FactorList &fl = td.fl;
  // stage slices (offsets into the shared array, so every later access is a shared-space load)
  int boff[kMaxFactors], first[kMaxFactors], cnt[kMaxFactors];
  {
    int off = 0;
#pragma unroll
    for (int f = 0; f < kMaxFactors; ++f) {
      if (f < fl.n) {
        const Factor &F = fl.f[f];
        const int st = (int)F.stride;
        const int q0 = e_lo / st, q1 = e_hi / st;
        const int c = (q1 - q0 + 1) < F.I ? (q1 - q0 + 1) : F.I;
        boff[f] = off;
        first[f] = q0;
        cnt[f] = c;
        const int AB = F.Ra * F.Rb, span = F.I * AB;
        const int s0 = (q0 % F.I) * AB;   // slices (q0 + j) mod I, j < c, wrap at most once
        for (int e = threadIdx.x; e < c * AB; e += blockDim.x) {
          int idx = s0 + e;
          if (idx >= span) idx -= span;
          cp_async8(tsm + off + e, F.G + idx);
        }
        off += ((c * AB + 1) & ~1);
      }
    }
  }
  const int R0 = fl.f[0].Ra;
  const int Rl = fl.f[fl.n - 1].Rb;
  const int W = R0 * Rl;
  float *tile = nullptr;
  const int Np = td.Npad;
  if (tiles) {
    // tile staging area after the slices (float, 2 Np x 32)
    int off = 0;
#pragma unroll
    for (int f = 0; f < kMaxFactors; ++f)
      if (f < fl.n) off += ((cnt[f] * fl.f[f].Ra * fl.f[f].Rb + 1) & ~1);
    tile = (float *)(tsm + off);
    for (int e = threadIdx.x; e < 2 * Np * 8; e += blockDim.x) ((float4 *)tile)[e] = make_float4(0, 0, 0, 0);
  }
  cp_async_wait_all();
  __syncthreads();
  const int el = threadIdx.x / R0, pr = threadIdx.x - (threadIdx.x / R0) * R0;
  const int l = l0 + el;
  if (el < 32 && l < l1) {
    const int e = l + Lk * tp;
    double v[MR], w[MR];
    auto slice = [&](int f) -> const double * {
      const Factor &F = fl.f[f];
      int j = e / (int)F.stride - first[f];
      while (j >= cnt[f]) j -= cnt[f];   // only when the unit spans more than I slices
      return tsm + boff[f] + j * (F.Ra * F.Rb);
    };
    {
      const Factor &F = fl.f[0];
      const double *S = slice(0);
#pragma unroll
      for (int b = 0; b < MR; ++b) v[b] = (b < F.Rb) ? S[pr + F.Ra * b] : 0.0;
    }
#pragma unroll
    for (int f = 1; f < kMaxFactors; ++f) {
      if (f < fl.n) {
        const Factor &F = fl.f[f];
        const double *S = slice(f);
#pragma unroll
        for (int b = 0; b < MR; ++b) {
          double acc = 0.0;
          if (b < F.Rb) {
#pragma unroll
            for (int a = 0; a < MR; ++a)
              if (a < F.Ra) acc = fma(v[a], S[a + F.Ra * b], acc);
          }
          w[b] = acc;
        }
#pragma unroll
        for (int b = 0; b < MR; ++b) v[b] = w[b];
      }
    }
    if (out64) {
      double *o = out64 + (int64_t)e * W + pr * Rl;
#pragma unroll
      for (int q = 0; q < MR; ++q)
        if (q < Rl) o[q] = v[q];
    }
    if (td.out32) {
      float *o = td.out32 + (int64_t)e * W + pr * Rl;
#pragma unroll
      for (int q = 0; q < MR; ++q)
        if (q < Rl) o[q] = (float)v[q];
    }
    if (tiles) {
      const int kk = el, chunk = kk >> 2, within = kk & 3;
#pragma unroll
      for (int q = 0; q < MR; ++q) {
        if (q < Rl) {
          const int n = pr * Rl + q;
          const float hi = tf32_rna((float)v[q]);
          const float lo = tf32_rna((float)(v[q] - (double)hi));
          tile[n * 32 + ((chunk ^ (n & 7)) << 2) + within] = hi;
          const int n2 = Np + n;
          tile[n2 * 32 + ((chunk ^ (n2 & 7)) << 2) + within] = lo;
        }
      }
    }
  }
  if (tiles) {
    __syncthreads();
    float4 *dst = (float4 *)(tiles + (int64_t)unit * (2 * Np * 32));
    const float4 *src = (const float4 *)tile;
    for (int e = threadIdx.x; e < 2 * Np * 8; e += blockDim.x) dst[e] = src[e];
  }
}

// Uniform-rank variant (every factor R x R, R even): two output rows per thread (R/2 threads per
// entry), slice columns read as 16-byte pairs, compile-time strides.  Same staging and outputs as
// k_build_table2.
template <int R>
__global__ void __launch_bounds__(256) k_build_table3(TableDesc td, double *__restrict__ out64, float *__restrict__ tiles) {
  if (td.zero)   // the next contraction's output (one node fewer per pass)
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < td.zero_n4; i += (int64_t)gridDim.x * blockDim.x)
      td.zero[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  extern __shared__ __align__(16) double tsm[];
  constexpr int AB = R * R, H = R / 2;
  const int Lk = (int)td.Lk;
  const int nlb = (Lk + 31) / 32;
  const int unit = blockIdx.x;
  const int tp = unit / nlb;
  const int lb = unit - tp * nlb;
  const int l0 = lb * 32;
  const int l1 = (l0 + 32 < Lk) ? l0 + 32 : Lk;
  const int e_lo = l0 + Lk * tp, e_hi = l1 - 1 + Lk * tp;
  const FactorList &fl = td.fl;
  int boff[kMaxFactors], first[kMaxFactors], cnt[kMaxFactors];
  int off = 0;
#pragma unroll
  for (int f = 0; f < kMaxFactors; ++f) {
    if (f < fl.n) {
      const Factor &F = fl.f[f];
      const int st = (int)F.stride;
      const int q0 = e_lo / st, q1 = e_hi / st;
      const int c = (q1 - q0 + 1) < F.I ? (q1 - q0 + 1) : F.I;
      boff[f] = off;
      first[f] = q0;
      cnt[f] = c;
      const int span = F.I * AB, s0 = (q0 % F.I) * AB;
      for (int e = threadIdx.x; e < c * (AB / 2); e += blockDim.x) {   // 16-byte chunks (AB even)
        int idx = s0 + 2 * e;
        if (idx >= span) idx -= span;
        cp_async16(tsm + off + 2 * e, F.G + idx);
      }
      off += c * AB;
    }
  }
  const int Np = td.Npad;
  float *tile = (float *)(tsm + off);
  if (tiles)
    for (int e = threadIdx.x; e < 2 * Np * 8; e += blockDim.x) ((float4 *)tile)[e] = make_float4(0, 0, 0, 0);
  cp_async_wait_all();
  __syncthreads();
  const int el = threadIdx.x / H, pr = 2 * (threadIdx.x - el * H);
  const int l = l0 + el;
  if (el < 32 && l < l1) {
    const int e = l + Lk * tp;
    auto slice = [&](int f) -> const double * {
      int j = e / (int)fl.f[f].stride - first[f];
      while (j >= cnt[f]) j -= cnt[f];
      return tsm + boff[f] + j * AB;
    };
    double v[2][R];
    {
      const double *S = slice(0);
#pragma unroll
      for (int b = 0; b < R; ++b) {
        v[0][b] = S[pr + R * b];
        v[1][b] = S[pr + 1 + R * b];
      }
    }
#pragma unroll
    for (int f = 1; f < kMaxFactors; ++f) {
      if (f < fl.n) {
        const double *S = slice(f);
        double w[2][R];
#pragma unroll
        for (int b = 0; b < R; ++b) {
          double a0 = 0.0, a1 = 0.0;
#pragma unroll
          for (int a = 0; a < R; a += 2) {
            const double2 col = *(const double2 *)(S + a + R * b);
            a0 = fma(v[0][a], col.x, a0);
            a1 = fma(v[1][a], col.x, a1);
            a0 = fma(v[0][a + 1], col.y, a0);
            a1 = fma(v[1][a + 1], col.y, a1);
          }
          w[0][b] = a0;
          w[1][b] = a1;
        }
#pragma unroll
        for (int b = 0; b < R; ++b) {
          v[0][b] = w[0][b];
          v[1][b] = w[1][b];
        }
      }
    }
    if (out64) {
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        double *o = out64 + (int64_t)e * AB + (pr + r) * R;
#pragma unroll
        for (int q = 0; q < R; ++q) o[q] = v[r][q];
      }
    }
    if (td.out32) {
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        float *o = td.out32 + (int64_t)e * AB + (pr + r) * R;
#pragma unroll
        for (int q = 0; q < R; ++q) o[q] = (float)v[r][q];
      }
    }
    if (tiles) {
      const int kk = el, chunk = kk >> 2, within = kk & 3;
#pragma unroll
      for (int r = 0; r < 2; ++r) {
#pragma unroll
        for (int q = 0; q < R; ++q) {
          const int n = (pr + r) * R + q;
          const float hi = tf32_rna((float)v[r][q]);
          const float lo = tf32_rna((float)(v[r][q] - (double)hi));
          tile[n * 32 + ((chunk ^ (n & 7)) << 2) + within] = hi;
          const int n2 = Np + n;
          tile[n2 * 32 + ((chunk ^ (n2 & 7)) << 2) + within] = lo;
        }
      }
    }
  }
  if (tiles) {
    __syncthreads();
    float4 *dst = (float4 *)(tiles + (int64_t)unit * (2 * Np * 32));
    const float4 *src = (const float4 *)tile;
    for (int e = threadIdx.x; e < 2 * Np * 8; e += blockDim.x) dst[e] = src[e];
  }
}

size_t table2_smem(const TableDesc &td) {
  size_t n = 0;
  for (int f = 0; f < td.fl.n; ++f) {
    const Factor &F = td.fl.f[f];
    int64_t c = 31 / F.stride + 2;
    if (c > F.I) c = F.I;
    n += (size_t)((c * F.Ra * F.Rb + 1) & ~1);
  }
  size_t bytes = n * sizeof(double);
  if (td.Npad > 0) bytes += (size_t)2 * td.Npad * 32 * sizeof(float);
  return bytes;
}

int launch_build_table2(const TableDesc &td, double *out64, float *tiles, cudaStream_t s) {
  if (g_dbg_skip & 2) return 0;
  const size_t smem = table2_smem(td);
  if (smem > 200 * 1024) return -1;
  if (td.Lk * td.tk >= (int64_t)1 << 31) return -1;   // 32-bit entry indices
  prepare_kernel_attrs();
  const int64_t units = td.tk * cdiv(td.Lk, 32);
  {   // uniform rank R (all factors R x R) with 16-byte aligned slices: the specialized kernel
    const int R = td.fl.f[0].Ra;
    bool uni = (R == 4 || R == 8 || R == 10 || R == 16);
    for (int f = 0; f < td.fl.n && uni; ++f)
      uni = td.fl.f[f].Ra == R && td.fl.f[f].Rb == R && (uintptr_t)td.fl.f[f].G % 16 == 0;
    if (uni) {
      const int th = (int)cdiv(16 * R, 32) * 32;
      if (R == 4) k_build_table3<4><<<(unsigned)units, th, smem, s>>>(td, out64, tiles);
      else if (R == 8) k_build_table3<8><<<(unsigned)units, th, smem, s>>>(td, out64, tiles);
      else if (R == 10) k_build_table3<10><<<(unsigned)units, th, smem, s>>>(td, out64, tiles);
      else k_build_table3<16><<<(unsigned)units, th, smem, s>>>(td, out64, tiles);
      return 0;
    }
  }
  const int threads = (int)cdiv(32 * td.fl.f[0].Ra, 32) * 32;
  int mr = 0;
  for (int f = 0; f < td.fl.n; ++f) mr = std::max(mr, std::max(td.fl.f[f].Ra, td.fl.f[f].Rb));
  if (mr <= 4)
    k_build_table2<4><<<(unsigned)units, threads, smem, s>>>(td, out64, tiles);
  else if (mr <= 8)
    k_build_table2<8><<<(unsigned)units, threads, smem, s>>>(td, out64, tiles);
  else if (mr <= 10)
    k_build_table2<10><<<(unsigned)units, threads, smem, s>>>(td, out64, tiles);
  else
    k_build_table2<STR_MAXR><<<(unsigned)units, threads, smem, s>>>(td, out64, tiles);
  return 0;
}

// ------------------------------------------------------------------------------------------
// A = I (n x n): the identity chain matrix (an empty Gram-chain product).
__global__ void k_set_identity(double *A, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n * n) A[i] = (i / n == i % n) ? 1.0 : 0.0;
}

void launch_set_identity(double *A, int n, cudaStream_t s) {
  k_set_identity<<<(unsigned)cdiv((int64_t)n * n, 256), 256, 0, s>>>(A, n);
}

// ------------------------------------------------------------------------------------------
// dst (+)= x for fp32 or fp64 x (accumulate = 0 copies).
template <typename T>
__global__ void k_axpy_any(const T *__restrict__ x, double *__restrict__ y, int64_t n, int accumulate) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) y[i] = accumulate ? y[i] + (double)x[i] : (double)x[i];
}

void launch_axpy_any(const void *x, bool x_f32, double *y, int64_t n, int accumulate, cudaStream_t s) {
  if (x_f32)
    k_axpy_any<float><<<(unsigned)cdiv(n, 256), 256, 0, s>>>((const float *)x, y, n, accumulate);
  else
    k_axpy_any<double><<<(unsigned)cdiv(n, 256), 256, 0, s>>>((const double *)x, y, n, accumulate);
}

// ------------------------------------------------------------------------------------------
// Split-K fp64 GEMM with strided operands (rSTR sampled normal equations, Alg. 7 l.15-16:
// P_n += X_S G_S, Q_n += G_S^T G_S, temporal G_S^T G_S and X_S[N] G_S with K = m sampled rows):
//   part[ks][i][j] = sum_{k in range ks} A(i, k) B(k, j),  A(i,k) = A[i sai + k sak], B(k,j) = B[k sbk + j sbj]
// One 32x32 output tile per CTA and K-range; chunks of 32 k staged in shared memory by cp.async;
// then k_reduce_sk sums the KS partials in a fixed order into C (= or +=): deterministic.
constexpr int kSkKC = 32;

__global__ void __launch_bounds__(256) k_gemm_sk(const double *__restrict__ A, int64_t sai, int64_t sak,
                                                 const double *__restrict__ B, int64_t sbk, int64_t sbj, int M, int N,
                                                 int64_t K, int64_t kper, double *__restrict__ part) {
  PDL_PROLOGUE();
  // two chunk buffers: the cp.async of chunk c+1 is in flight while chunk c is multiplied
  __shared__ __align__(16) double As[2][kSkKC][34], Bs[2][kSkKC][32];   // As rows padded (transposed loads)
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int row0 = blockIdx.y * 32, col0 = blockIdx.x * 32;
  const int64_t k0 = (int64_t)blockIdx.z * kper;
  const int64_t k1 = (k0 + kper < K) ? k0 + kper : K;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  auto load = [&](int buf, int64_t kc) {
    for (int e = threadIdx.x; e < 32 * kSkKC; e += 256) {
      // A: consecutive threads along whichever of (row, k) is contiguous in memory
      const int kk = (sak == 1) ? (e & 31) : (e >> 5), r = (sak == 1) ? (e >> 5) : (e & 31);
      const int64_t k = kc + kk;
      if (k < k1 && row0 + r < M) cp_async8(&As[buf][kk][r], A + (int64_t)(row0 + r) * sai + k * sak);
      else As[buf][kk][r] = 0.0;
      const int kb = e >> 5, cb = e & 31;
      const int64_t kq = kc + kb;
      if (kq < k1 && col0 + cb < N) cp_async8(&Bs[buf][kb][cb], B + kq * sbk + (int64_t)(col0 + cb) * sbj);
      else Bs[buf][kb][cb] = 0.0;
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  int buf = 0;
  if (k0 < k1) load(0, k0);
  for (int64_t kc = k0; kc < k1; kc += kSkKC, buf ^= 1) {
    if (kc + kSkKC < k1) {
      load(buf ^ 1, kc + kSkKC);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < kSkKC; ++kk) {
      const double b = Bs[buf][kk][tx];
      const double2 a01 = *(const double2 *)&As[buf][kk][4 * ty];
      const double2 a23 = *(const double2 *)&As[buf][kk][4 * ty + 2];
      acc[0] = fma(a01.x, b, acc[0]);
      acc[1] = fma(a01.y, b, acc[1]);
      acc[2] = fma(a23.x, b, acc[2]);
      acc[3] = fma(a23.y, b, acc[3]);
    }
    __syncthreads();   // buf is refilled two chunks later
  }
  double *pp = part + (int64_t)blockIdx.z * M * N;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int row = row0 + 4 * ty + u, col = col0 + tx;
    if (row < M && col < N) pp[(int64_t)row * N + col] = acc[u];
  }
}

// sym (square C only): C[i][j] (+)= (S[i][j] + S[j][i]) / 2 — the (A + A^T)/2 of reading R5 applied
// to the increment (equal to symmetrizing the sum when C is symmetric).
__global__ void k_reduce_sk(const double *__restrict__ part, int KS, int64_t n, int N, double *__restrict__ C, int acc,
                            int sym) {
  // PDL: the accumulated value (P_n / Q_n of the previous step: only this kernel writes it) is loaded
  // before the wait for the split-K products, the partials after it
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const double old = (acc && i < n) ? C[i] : 0.0;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (i >= n) return;
  // all partials are loaded before the (fixed-order) sums, so the loads overlap
  double v[32], w[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) v[k] = k < KS ? part[k * n + i] : 0.0;
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 32; ++k)
    if (k < KS) s += v[k];
  if (sym) {
    const int64_t r = i / N, c = i % N;
#pragma unroll
    for (int k = 0; k < 32; ++k) w[k] = k < KS ? part[k * n + c * N + r] : 0.0;
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < 32; ++k)
      if (k < KS) t += w[k];
    s = 0.5 * (s + t);
  }
  C[i] = acc ? old + s : s;
}

size_t gemm_sk_ws_doubles(int M, int N, int64_t K) {
  (void)K;
  return (size_t)32 * M * N;   // up to 32 K-splits
}

int launch_gemm_sk(const double *A, int64_t sai, int64_t sak, const double *B, int64_t sbk, int64_t sbj, double *C,
                   int M, int N, int64_t K, int acc, double *ws, cudaStream_t s, int sym) {
  const int tiles = (int)(cdiv(M, 32) * cdiv(N, 32));
  int KS = (int)std::min<int64_t>(32, std::max<int64_t>(1, std::min<int64_t>(cdiv(2 * 148, tiles), cdiv(K, 64))));
  const int64_t kper = cdiv(cdiv(K, KS), kSkKC) * kSkKC;
  KS = (int)cdiv(K, kper);
  dim3 grid((unsigned)cdiv(N, 32), (unsigned)cdiv(M, 32), (unsigned)KS);
  pdl_launch(kPdlRstr, k_gemm_sk, grid, dim3(256), 0, s, A, sai, sak, B, sbk, sbj, M, N, K, kper, ws);
  const int64_t n = (int64_t)M * N;
  pdl_launch(kPdlRstr, k_reduce_sk, dim3((unsigned)cdiv(n, 256)), dim3(256), 0, s, (const double *)ws, KS, n, N, C, acc,
             sym);
  return 2;
}

// Dynamic shared-memory opt-ins, done once outside any stream capture.
void prepare_kernel_attrs() {
  static PerDeviceOnce once;
  once_per_device(once, [] {
  cudaFuncSetAttribute(k_chain_gemm_dmma<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gemm_dmma_smem(256));
  cudaFuncSetAttribute(k_chain_gemm_dmma<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gemm_dmma_smem(256));
  cudaFuncSetAttribute(k_chain_gemm_dmma<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  cudaFuncSetAttribute(k_chain_gemm_dmma<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  prefer_max_smem(k_chain_gemm_dmma<true, false>);
  prefer_max_smem(k_chain_gemm_dmma<false, false>);
  prefer_max_smem(k_chain_gemm_dmma<true, true>);
  prefer_max_smem(k_chain_gemm_dmma<false, true>);
  absorb_attrs<float>();
  absorb_attrs<double>();
  cudaFuncSetAttribute(k_build_table2<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_build_table2<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_build_table2<10>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_build_table2<STR_MAXR>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_build_table3<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_build_table3<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_build_table3<10>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_build_table3<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  prefer_max_smem(k_build_table3<4>);
  prefer_max_smem(k_build_table3<8>);
  prefer_max_smem(k_build_table3<10>);
  prefer_max_smem(k_build_table3<16>);
  prefer_max_smem(k_gram_z2);
  prefer_max_smem(k_build_table2<4>);
  prefer_max_smem(k_build_table2<8>);
  prefer_max_smem(k_build_table2<10>);
  prefer_max_smem(k_build_table2<STR_MAXR>);
  prefer_max_smem(k_axpy_any<float>);
  prefer_max_smem(k_axpy_any<double>);
  prefer_max_smem(k_gemm_sk);
  prefer_max_smem(k_reduce_sk);
  prepare_f64_attrs();
  });
}

}  // namespace strb200
