// ksrft.cu — the KSRFT kernels of rSTR-K (Def. 10; Alg. 5 P:643-661;
// Alg. 9).  DESIGN.md readings R17-R22; the host orchestration is in rstr.cu.
//
//   k_draw_signs     D_1..D_N for the step (SplitMix64 stream k = 0 of reading R11; R18)
//   k_mix_mode       X^ <- X^ x_j (F_j D_j), one mode per launch, complex in place (the first
//                    mode reads the real batch through the device slot).  HBM-bound: each launch
//                    streams the tensor once.  The length-I DFT of every fiber runs in shared
//                    memory as two passes of a p x q factorization (I = p q, Cooley-Tukey without
//                    recursion), p + q complex MACs per output instead of I.
//   k_mix_sample     (G^_k)_S(s, :) = sum_i (F_k D_k)(idxs(s,k), i) G_k(i, :)  (only the sampled
//                    rows of the mixed core are formed; reading R19)
//   k_chain_complex  the ⊡₂ chain of complex sampled slices, written as the stacked real matrix
//                    [Re G^_S[2]; Im G^_S[2]] (2m x R_nR_{n+1}) so that the real GEMMs of rSTR give
//                    Re(X~ conj G^) = [Re X~, Im X~][Re G^; Im G^] and Re(G^T conj G^) = stacked Gram
//                    (reading R21)
//   k_gather_unmix   X~_S[n] = D_n F_n^* X^_S[n] on the zipped fibers, stacked [Re | Im] (I_n x 2m)
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace strb200 {

template <typename T> struct C2;
template <> struct C2<float> { using t = float2; };
template <> struct C2<double> { using t = double2; };

__device__ __forceinline__ uint64_t ks_splitmix_at(uint64_t key, uint64_t j) {
  uint64_t z = key + (j + 1) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// d[j] = +1 / -1 from the top bit of draw j of the stream (seed, tau, k = 0)  (reading R18)
__global__ void k_draw_signs(uint64_t seed, const int64_t *__restrict__ tau, int N, int64_t total, double *__restrict__ d) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= total) return;
  const uint64_t key = seed ^ (0x9E3779B97F4A7C15ull * (uint64_t)(1 + (*tau) * (N + 1)));
  d[j] = (ks_splitmix_at(key, (uint64_t)j) >> 63) ? -1.0 : 1.0;
}

// Mode-j mixing of a tensor viewed as [A, I, B] (element (a, i, b) at a + A (i + I b)).  A CTA owns
// WA x WB fibers (a-chunk x b-chunk): loads them into xs[i][f] (f = fa + WA fb), runs
//   stage 1: T[k1 q + n2][f] = w^{n2 k1} sum_{n1 < p} w^{q n1 k1} x[q n1 + n2][f]
//   stage 2: y[k1 + p k2][f] = sum_{n2 < q} w^{p n2 k2} T[k1 q + n2][f]          (w = e^{-2 pi i / I})
// and stores y back over the same positions.  x is scaled by d_i / sqrt(I) on load.
constexpr int kMixQMax = 20;   // register-blocked sub-DFT length (p <= q <= 20: I <= 400)

struct MixDesc {
  int64_t A, B;
  int I, p, q;
  int WA, WB;                 // fibers per CTA: WA consecutive a x WB consecutive b (WA WB <= 32)
  int64_t nA;                 // a-chunks
  int inc0, inc1, inc2;       // +256 in the mixed radix (WA, I, WB) of the load/store order
  const double *d;            // D_j diagonal
};

// element e = fa + WA (i + I fb) of the tile; walking e += 256 with carries (no divisions)
struct TileWalk {
  int fa, i, fb;
  __device__ __forceinline__ void init(int t, const MixDesc &md) {
    fa = t % md.WA;
    i = (t / md.WA) % md.I;
    fb = t / (md.WA * md.I);
  }
  __device__ __forceinline__ void step(const MixDesc &md) {
    fa += md.inc0;
    if (fa >= md.WA) { fa -= md.WA; ++i; }
    i += md.inc1;
    if (i >= md.I) { i -= md.I; ++fb; }
    fb += md.inc2;
  }
};

template <typename TIn, typename TC, bool FIRST>
__global__ void __launch_bounds__(256) k_mix_mode(const void *const *__restrict__ xslot, typename C2<TC>::t *__restrict__ Y,
                                                  MixDesc md) {
  using c2 = typename C2<TC>::t;
  extern __shared__ __align__(16) unsigned char ks_smem[];
  const int WF = md.WA * md.WB;
  const int ld = WF + 1;                                 // padded row (bank spread for the transposed loads)
  c2 *xs = (c2 *)ks_smem;                                // [I][ld]
  c2 *ts = xs + (size_t)md.I * ld;                       // [I][ld]
  c2 *tw = ts + (size_t)md.I * ld;                       // [I] twiddles w^k
  TC *ds = (TC *)(tw + md.I);                            // [I] d_i / sqrt(I)
  const int I = md.I, p = md.p, q = md.q;
  const double scale = rsqrt((double)I);
  for (int k = threadIdx.x; k < I; k += blockDim.x) {
    double s, c;
    sincospi(-2.0 * (double)k / (double)I, &s, &c);
    tw[k].x = (TC)c;
    tw[k].y = (TC)s;
    ds[k] = (TC)(md.d[k] * scale);
  }
  __syncthreads();
  const int64_t tile = blockIdx.x;
  const int64_t a0 = (tile % md.nA) * md.WA, b0 = (tile / md.nA) * md.WB;
  const int n_el = WF * I;
  const int64_t A = md.A;
  const int aval = (int)(A - a0 < md.WA ? A - a0 : md.WA), bval = (int)(md.B - b0 < md.WB ? md.B - b0 : md.WB);
  const int64_t base = a0 + A * (int64_t)I * b0;
  // load (a fastest, then i, then b: coalesced along a, or along i when A == 1)
  {
    TileWalk w;
    w.init(threadIdx.x, md);
    for (int e = threadIdx.x; e < n_el; e += 256, w.step(md)) {
      c2 v;
      v.x = 0;
      v.y = 0;
      if (w.fa < aval && w.fb < bval) {
        const int64_t off = base + w.fa + A * (w.i + (int64_t)I * w.fb);
        const TC sc = ds[w.i];
        if (FIRST) {
          const TIn *X = (const TIn *)*xslot;
          v.x = (TC)X[off] * sc;
        } else {
          v = Y[off];
          v.x *= sc;
          v.y *= sc;
        }
      }
      xs[w.i * ld + w.fa + md.WA * w.fb] = v;
    }
  }
  __syncthreads();
  // Stage 1, item (f, n2): all p outputs T[k1 q + n2][f] from one pass over x[q n1 + n2][f]
  // (register-blocked, twiddles w^{q (n1 k1 mod p)} broadcast from shared memory).  Stage 2, item
  // (f, k1): all q outputs y[k1 + p k2][f] from T[k1 q + n2][f], twiddles w^{p (n2 k2 mod q)}.
  if (q <= kMixQMax) {
    for (int it = threadIdx.x; it < WF * q; it += 256) {
      const int f = it % WF, n2 = it / WF;
      TC ax[kMixQMax], ay[kMixQMax];
#pragma unroll
      for (int k = 0; k < kMixQMax; ++k) ax[k] = ay[k] = 0;
      for (int n1 = 0; n1 < p; ++n1) {
        const c2 x = xs[(q * n1 + n2) * ld + f];
        int m = 0;                                       // n1 k1 mod p
#pragma unroll
        for (int k1 = 0; k1 < kMixQMax; ++k1) {
          if (k1 < p) {
            const c2 w = tw[q * m];
            ax[k1] += x.x * w.x - x.y * w.y;
            ay[k1] += x.x * w.y + x.y * w.x;
            m += n1;
            if (m >= p) m -= p;
          }
        }
      }
      int m = 0;                                         // n2 k1 (< I)
#pragma unroll
      for (int k1 = 0; k1 < kMixQMax; ++k1) {
        if (k1 < p) {
          const c2 w = tw[m];
          c2 t;
          t.x = ax[k1] * w.x - ay[k1] * w.y;
          t.y = ax[k1] * w.y + ay[k1] * w.x;
          ts[(k1 * q + n2) * ld + f] = t;
          m += n2;
        }
      }
    }
    __syncthreads();
    for (int it = threadIdx.x; it < WF * p; it += 256) {
      const int f = it % WF, k1 = it / WF;
      TC ax[kMixQMax], ay[kMixQMax];
#pragma unroll
      for (int k = 0; k < kMixQMax; ++k) ax[k] = ay[k] = 0;
      for (int n2 = 0; n2 < q; ++n2) {
        const c2 t = ts[(k1 * q + n2) * ld + f];
        int m = 0;                                       // n2 k2 mod q
#pragma unroll
        for (int k2 = 0; k2 < kMixQMax; ++k2) {
          if (k2 < q) {
            const c2 w = tw[p * m];
            ax[k2] += t.x * w.x - t.y * w.y;
            ay[k2] += t.x * w.y + t.y * w.x;
            m += n2;
            if (m >= q) m -= q;
          }
        }
      }
#pragma unroll
      for (int k2 = 0; k2 < kMixQMax; ++k2) {
        if (k2 < q) {
          c2 y;
          y.x = ax[k2];
          y.y = ay[k2];
          xs[(k1 + p * k2) * ld + f] = y;
        }
      }
    }
  } else {   // long prime-ish factor: one output per item (direct sums)
    for (int it = threadIdx.x; it < WF * I; it += 256) {
      const int f = it % WF, r = it / WF;                // r = k1 q + n2
      const int k1 = r / q, n2 = r % q;
      TC ax = 0, ay = 0;
      int widx = 0;
      for (int n1 = 0; n1 < p; ++n1) {
        const c2 x = xs[(q * n1 + n2) * ld + f];
        const c2 w = tw[widx];
        ax += x.x * w.x - x.y * w.y;
        ay += x.x * w.y + x.y * w.x;
        widx += q * k1;
        if (widx >= I) widx -= I;
      }
      const c2 w = tw[(n2 * k1) % I];
      c2 t;
      t.x = ax * w.x - ay * w.y;
      t.y = ax * w.y + ay * w.x;
      ts[r * ld + f] = t;
    }
    __syncthreads();
    for (int it = threadIdx.x; it < WF * I; it += 256) {
      const int f = it % WF, r = it / WF;                // output k = k1 + p k2
      const int k1 = r % p, k2 = r / p;
      TC ax = 0, ay = 0;
      int widx = 0;
      for (int n2 = 0; n2 < q; ++n2) {
        const c2 t = ts[(k1 * q + n2) * ld + f];
        const c2 w = tw[widx];
        ax += t.x * w.x - t.y * w.y;
        ay += t.x * w.y + t.y * w.x;
        widx += p * k2;
        if (widx >= I) widx -= I;
      }
      c2 y;
      y.x = ax;
      y.y = ay;
      xs[r * ld + f] = y;
    }
  }
  __syncthreads();
  {
    TileWalk w;
    w.init(threadIdx.x, md);
    for (int e = threadIdx.x; e < n_el; e += 256, w.step(md))
      if (w.fa < aval && w.fb < bval) Y[base + w.fa + A * (w.i + (int64_t)I * w.fb)] = xs[w.i * ld + w.fa + md.WA * w.fb];
  }
}

// Compile-time p x q variant (the fp32 mixing path): the sub-DFT twiddles are the p-th / q-th roots
// of unity, held in registers and indexed by compile-time (n1 k1 mod p), (n2 k2 mod q), so every
// complex MAC is 2 packed FFMA2 (products with w^0 = 1 folded away).  Same tile layout as k_mix_mode,
// with direct address walks for the two common tile shapes.
template <int P, int Q, typename TIn, bool FIRST>
__global__ void __launch_bounds__(256) k_mix_pq(const void *const *__restrict__ xslot, float2 *__restrict__ Y, MixDesc md) {
  constexpr int I = P * Q;
  extern __shared__ __align__(16) unsigned char ks_smem[];
  const int WF = md.WA * md.WB;
  const int ld = WF + 1;
  float2 *xs = (float2 *)ks_smem;                        // [I][ld]
  float2 *ts = xs + (size_t)I * ld;                      // [I][ld]
  float2 *tw = ts + (size_t)I * ld;                      // [I] w^k
  float *ds = (float *)(tw + I);                         // [I] d_i / sqrt(I)
  const double scale = rsqrt((double)I);
  for (int k = threadIdx.x; k < I; k += blockDim.x) {
    double s, c;
    sincospi(-2.0 * (double)k / (double)I, &s, &c);
    tw[k] = make_float2((float)c, (float)s);
    ds[k] = (float)(md.d[k] * scale);
  }
  __syncthreads();
  const int64_t tile = blockIdx.x;
  const int64_t a0 = (tile % md.nA) * md.WA, b0 = (tile / md.nA) * md.WB;
  const int n_el = WF * I;
  const int64_t A = md.A;
  const int aval = (int)(A - a0 < md.WA ? A - a0 : md.WA), bval = (int)(md.B - b0 < md.WB ? md.B - b0 : md.WB);
  const int64_t base = a0 + A * (int64_t)I * b0;
  // tile shapes: (a) WA = 32, WB = 1: lane = fa, rows i = warp + 8 k (offset += 8 A);
  //              (b) A = 1: the tile is one contiguous run of WB fibers (offset = e);  (c) general walk
  const bool shape_a = (md.WA == 32 && md.WB == 1), shape_b = (A == 1);
  auto load_el = [&](int64_t off, int i) -> float2 {
    const float sc = ds[i];
    if (FIRST) return make_float2((float)((const TIn *)*xslot)[off] * sc, 0.f);
    float2 v = Y[off];
    return make_float2(v.x * sc, v.y * sc);
  };
  if (shape_a) {
    const int fa = threadIdx.x & 31;
    const bool ok = fa < aval;
    for (int i = threadIdx.x >> 5; i < I; i += 8)
      xs[i * ld + fa] = ok ? load_el(base + fa + A * i, i) : make_float2(0.f, 0.f);
  } else if (shape_b) {
    const int lim = bval * I;
    int i = threadIdx.x % I, fb = threadIdx.x / I;
    const int di = 256 % I, dfb = 256 / I;
    for (int e = threadIdx.x; e < n_el; e += 256) {
      xs[i * ld + fb] = e < lim ? load_el(base + e, i) : make_float2(0.f, 0.f);
      i += di;
      fb += dfb;
      if (i >= I) { i -= I; ++fb; }
    }
  } else {
    TileWalk w;
    w.init(threadIdx.x, md);
    for (int e = threadIdx.x; e < n_el; e += 256, w.step(md)) {
      const bool ok = w.fa < aval && w.fb < bval;
      xs[w.i * ld + w.fa + md.WA * w.fb] =
          ok ? load_el(base + w.fa + A * (w.i + (int64_t)I * w.fb), w.i) : make_float2(0.f, 0.f);
    }
  }
  __syncthreads();
  const bool pow2 = (WF & (WF - 1)) == 0;
  const int lgWF = 31 - __clz(WF);
  // complex MAC on packed fp32 pairs: acc += x w = x (w.x, w.x) + (-x.y, x.x) (w.y, w.y)  (2 FFMA2)
  {
    float2 wxx[P], wyy[P];                               // w_P^j = w^{Q j}
#pragma unroll
    for (int j = 0; j < P; ++j) {
      const float2 w = tw[Q * j];
      wxx[j] = make_float2(w.x, w.x);
      wyy[j] = make_float2(w.y, w.y);
    }
    for (int it = threadIdx.x; it < WF * Q; it += 256) {   // stage 1, item (f, n2)
      int f, n2;
      if constexpr (P * Q <= 32) {   // short modes: cheap items, power-of-two tile widths use shifts
        f = pow2 ? (it & (WF - 1)) : it % WF;
        n2 = pow2 ? (it >> lgWF) : it / WF;
      } else {
        f = it % WF;
        n2 = it / WF;
      }
      float2 x[P], xr[P];
#pragma unroll
      for (int n1 = 0; n1 < P; ++n1) {
        x[n1] = xs[(Q * n1 + n2) * ld + f];
        xr[n1] = make_float2(-x[n1].y, x[n1].x);
      }
#pragma unroll
      for (int k1 = 0; k1 < P; ++k1) {
        float2 acc = x[0];
#pragma unroll
        for (int n1 = 1; n1 < P; ++n1) {
          const int j = (n1 * k1) % P;
          if (j == 0) {
            acc.x += x[n1].x;
            acc.y += x[n1].y;
          } else {
            acc = __ffma2_rn(x[n1], wxx[j], acc);
            acc = __ffma2_rn(xr[n1], wyy[j], acc);
          }
        }
        float2 t = acc;
        if (k1 != 0) {
          const float2 w = tw[n2 * k1];                  // w^{n2 k1}, n2 k1 < I
          t = __fmul2_rn(acc, make_float2(w.x, w.x));
          t = __ffma2_rn(make_float2(-acc.y, acc.x), make_float2(w.y, w.y), t);
        }
        ts[(k1 * Q + n2) * ld + f] = t;
      }
    }
  }
  __syncthreads();
  {
    float2 wxx[Q], wyy[Q];                               // w_Q^j = w^{P j}
#pragma unroll
    for (int j = 0; j < Q; ++j) {
      const float2 w = tw[P * j];
      wxx[j] = make_float2(w.x, w.x);
      wyy[j] = make_float2(w.y, w.y);
    }
    for (int it = threadIdx.x; it < WF * P; it += 256) {   // stage 2, item (f, k1)
      int f, k1;
      if constexpr (P * Q <= 32) {
        f = pow2 ? (it & (WF - 1)) : it % WF;
        k1 = pow2 ? (it >> lgWF) : it / WF;
      } else {
        f = it % WF;
        k1 = it / WF;
      }
      float2 t[Q], tr[Q];
#pragma unroll
      for (int n2 = 0; n2 < Q; ++n2) {
        t[n2] = ts[(k1 * Q + n2) * ld + f];
        tr[n2] = make_float2(-t[n2].y, t[n2].x);
      }
#pragma unroll
      for (int k2 = 0; k2 < Q; ++k2) {
        float2 acc = t[0];
#pragma unroll
        for (int n2 = 1; n2 < Q; ++n2) {
          const int j = (n2 * k2) % Q;
          if (j == 0) {
            acc.x += t[n2].x;
            acc.y += t[n2].y;
          } else {
            acc = __ffma2_rn(t[n2], wxx[j], acc);
            acc = __ffma2_rn(tr[n2], wyy[j], acc);
          }
        }
        xs[(k1 + P * k2) * ld + f] = acc;
      }
    }
  }
  __syncthreads();
  if (shape_a) {
    const int fa = threadIdx.x & 31;
    if (fa < aval)
      for (int i = threadIdx.x >> 5; i < I; i += 8) Y[base + fa + A * i] = xs[i * ld + fa];
  } else if (shape_b) {
    const int lim = bval * I;
    int i = threadIdx.x % I, fb = threadIdx.x / I;
    const int di = 256 % I, dfb = 256 / I;
    for (int e = threadIdx.x; e < lim; e += 256) {
      Y[base + e] = xs[i * ld + fb];
      i += di;
      fb += dfb;
      if (i >= I) { i -= I; ++fb; }
    }
  } else {
    TileWalk w;
    w.init(threadIdx.x, md);
    for (int e = threadIdx.x; e < n_el; e += 256, w.step(md))
      if (w.fa < aval && w.fb < bval) Y[base + w.fa + A * (w.i + (int64_t)I * w.fb)] = xs[w.i * ld + w.fa + md.WA * w.fb];
  }
}

typedef void (*MixPQFn)(const void *const *, float2 *, MixDesc);
struct MixPQEntry {
  int p, q;
  MixPQFn first_f32, first_f64, rest;
};
#define KS_PQ(P, Q) {P, Q, k_mix_pq<P, Q, float, true>, k_mix_pq<P, Q, double, true>, k_mix_pq<P, Q, float, false>}
// the mode lengths of the workloads (factor_p: p = largest divisor <= sqrt(I)); others use k_mix_mode
static const MixPQEntry kMixPQ[] = {
    KS_PQ(1, 2),  KS_PQ(1, 3),  KS_PQ(2, 2),   KS_PQ(1, 5),   KS_PQ(2, 3),   KS_PQ(1, 7),   KS_PQ(2, 4),
    KS_PQ(3, 3),  KS_PQ(2, 5),  KS_PQ(3, 4),   KS_PQ(4, 4),   KS_PQ(4, 5),   KS_PQ(4, 6),   KS_PQ(5, 5),
    KS_PQ(5, 6),  KS_PQ(6, 6),  KS_PQ(5, 8),   KS_PQ(6, 8),   KS_PQ(7, 7),   KS_PQ(5, 10),  KS_PQ(6, 10),
    KS_PQ(8, 8),  KS_PQ(8, 10), KS_PQ(10, 10), KS_PQ(10, 12), KS_PQ(8, 16),  KS_PQ(10, 16), KS_PQ(10, 20),
    KS_PQ(15, 16), KS_PQ(16, 16), KS_PQ(16, 20)};
#undef KS_PQ

// (G^_k)_S(s, c) = sum_i w^{idx_s i} d_i / sqrt(I) G(i, c)   (G: I x S rows, fp64; out: m x S complex)
__global__ void k_mix_sample(const double *__restrict__ G, int64_t I, int S, const int32_t *__restrict__ idx, int64_t m,
                             const double *__restrict__ d, double2 *__restrict__ out) {
  extern __shared__ double2 tws[];                      // w^k, k < I
  for (int64_t k = threadIdx.x; k < I; k += blockDim.x) {
    double s, c;
    sincospi(-2.0 * (double)k / (double)I, &s, &c);
    tws[k] = make_double2(c, s);
  }
  __syncthreads();
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= m * S) return;
  const int64_t s = e / S;
  const int c = (int)(e % S);
  const int64_t a = idx[s];
  double ax = 0.0, ay = 0.0;
  int64_t widx = 0;
  for (int64_t i = 0; i < I; ++i) {
    const double g = d[i] * G[i * S + c];
    const double2 w = tws[widx];
    ax = fma(g, w.x, ax);
    ay = fma(g, w.y, ay);
    widx += a;
    if (widx >= I) widx -= I;
  }
  const double sc = rsqrt((double)I);
  out[e] = make_double2(ax * sc, ay * sc);
}

// Whole mixed core G^(a, c) = sum_i w^{a i} d_i / sqrt(I) G(i, c) for every a < I (I x S complex),
// then the sampled rows are gathered: I^2 S MACs instead of m I S when I < m.
__global__ void k_mix_core(const double *__restrict__ G, int I, int S, const double *__restrict__ d,
                           double2 *__restrict__ out) {
  extern __shared__ double2 tws[];
  for (int k = threadIdx.x; k < I; k += blockDim.x) {
    double s, c;
    sincospi(-2.0 * (double)k / (double)I, &s, &c);
    tws[k] = make_double2(c, s);
  }
  __syncthreads();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= I * S) return;
  const int a = e / S, c = e % S;
  double ax = 0.0, ay = 0.0;
  int widx = 0;
  for (int i = 0; i < I; ++i) {
    const double g = d[i] * G[i * S + c];
    const double2 w = tws[widx];
    ax = fma(g, w.x, ax);
    ay = fma(g, w.y, ay);
    widx += a;
    if (widx >= I) widx -= I;
  }
  const double sc = rsqrt((double)I);
  out[e] = make_double2(ax * sc, ay * sc);
}

__global__ void k_gather_crows(const double2 *__restrict__ Gh, int S, const int32_t *__restrict__ idx, int64_t m,
                               double2 *__restrict__ out) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= m * S) return;
  const int64_t s = e / S;
  out[e] = Gh[(int64_t)idx[s] * S + (e - s * S)];
}

// One thread per (sample s, row a of the chain product): row a of F_1(s) F_2(s) ... F_L(s), each F
// an Ra x Rb complex slice stored as G(2) rows (entry (a, b) at a + Ra b).  Output column
// b + Rb_last a (r_n + R_n r_{n+1}), Re part in row s, Im part in row m + s.
struct CFactorList {
  const double2 *G[kMaxFactors];
  int32_t Ra[kMaxFactors], Rb[kMaxFactors];
  int32_t n;
};

__global__ void __launch_bounds__(128) k_chain_complex(CFactorList fl, int64_t m, double *__restrict__ out) {
  const int R0 = fl.Ra[0];
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= m * R0) return;
  const int64_t s = e / R0;
  const int a = (int)(e % R0);
  double2 row[16], nr[16];
  {
    const int Ra = fl.Ra[0], Rb = fl.Rb[0];
    const double2 *F = fl.G[0] + s * (int64_t)(Ra * Rb);
#pragma unroll
    for (int c = 0; c < 16; ++c) row[c] = (c < Rb) ? F[a + Ra * c] : make_double2(0.0, 0.0);
  }
  int Rcur = fl.Rb[0];
  for (int l = 1; l < fl.n; ++l) {
    const int Ra = fl.Ra[l], Rb = fl.Rb[l];
    const double2 *F = fl.G[l] + s * (int64_t)(Ra * Rb);
#pragma unroll
    for (int c = 0; c < 16; ++c) nr[c] = make_double2(0.0, 0.0);
#pragma unroll
    for (int b = 0; b < 16; ++b) {
      if (b < Ra) {
        const double2 x = row[b];
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          if (c < Rb) {
            const double2 f = F[b + Ra * c];
            nr[c].x = fma(x.x, f.x, fma(-x.y, f.y, nr[c].x));
            nr[c].y = fma(x.x, f.y, fma(x.y, f.x, nr[c].y));
          }
        }
      }
    }
#pragma unroll
    for (int c = 0; c < 16; ++c) row[c] = nr[c];
    Rcur = Rb;
  }
  const int S = R0 * Rcur;
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    if (c < Rcur) {
      out[s * S + c + Rcur * a] = row[c].x;
      out[(m + s) * S + c + Rcur * a] = row[c].y;
    }
  }
}

// X~_S[n](i, s) = d_i / sqrt(I) sum_k w^{-i k} X^(idx_s with mode n = k); out I x 2m: [Re | Im]
struct UnmixDesc {
  int N, n;                    // order, mode (1-based)
  int64_t stride[8];
  int64_t I, m;
  const int32_t *idx;          // [N][m]
  const double *d;             // D_n
};

constexpr int kUnmixSB = 2;   // samples per CTA (m / 2 CTAs: the whole GPU busy at m = 2000)

template <typename TC>
__global__ void __launch_bounds__(128) k_gather_unmix(const typename C2<TC>::t *__restrict__ Xh, UnmixDesc ud,
                                                      double *__restrict__ out) {
  extern __shared__ double2 us[];                        // [SB][I] fibers, then w^{-k}
  const int I = (int)ud.I;
  double2 *tw = us + kUnmixSB * I;
  const int64_t s0 = (int64_t)blockIdx.x * kUnmixSB;
  for (int k = threadIdx.x; k < I; k += blockDim.x) {
    double s, c;
    sincospi(2.0 * (double)k / (double)I, &s, &c);
    tw[k] = make_double2(c, s);
  }
  for (int sl = 0; sl < kUnmixSB; ++sl) {
    const int64_t s = s0 + sl;
    int64_t base = 0;
    if (s < ud.m) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j < ud.N && j != ud.n - 1) base += (int64_t)ud.idx[j * ud.m + s] * ud.stride[j];
    }
    const int64_t sn = ud.stride[ud.n - 1];
    for (int k = threadIdx.x; k < I; k += blockDim.x) {
      double2 v = make_double2(0.0, 0.0);
      if (s < ud.m) {
        const typename C2<TC>::t x = Xh[base + k * sn];
        v = make_double2((double)x.x, (double)x.y);
      }
      us[sl * I + k] = v;
    }
  }
  __syncthreads();
  const double sc = rsqrt((double)I);
  for (int o = threadIdx.x; o < kUnmixSB * I; o += blockDim.x) {
    const int sl = o % kUnmixSB, i = o / kUnmixSB;
    const int64_t s = s0 + sl;
    if (s >= ud.m) continue;
    double ax = 0.0, ay = 0.0;
    int widx = 0;
    const double2 *x = us + sl * I;
    for (int k = 0; k < I; ++k) {
      const double2 v = x[k], w = tw[widx];
      ax = fma(v.x, w.x, fma(-v.y, w.y, ax));
      ay = fma(v.x, w.y, fma(v.y, w.x, ay));
      widx += i;
      if (widx >= I) widx -= I;
    }
    const double di = ud.d[i] * sc;
    out[(int64_t)i * 2 * ud.m + s] = ax * di;
    out[(int64_t)i * 2 * ud.m + ud.m + s] = ay * di;
  }
}

// ------------------------------------------------------------------------------------------ launchers
static int factor_p(int I) {
  int p = 1;
  for (int c = 1; (int64_t)c * c <= I; ++c)
    if (I % c == 0) p = c;
  return p;
}

void launch_draw_signs(uint64_t seed, const int64_t *tau, int N, int64_t total, double *d, cudaStream_t st) {
  k_draw_signs<<<(unsigned)cdiv(total, 256), 256, 0, st>>>(seed, tau, N, total, d);
}

size_t mix_mode_smem(int I, bool f64, int64_t A, int *WA, int *WB) {
  const size_t cb = f64 ? 16 : 8;
  auto bytes = [&](int wf) { return (2 * (size_t)I * (wf + 1) + 2 * I) * cb; };
  int WF = 32;
  while (WF > 1 && bytes(WF) > 200 * 1024) WF /= 2;
  while (WF < 1024 && (int64_t)WF * I < 4096 && bytes(2 * WF) <= 64 * 1024) WF *= 2;   // small I: wider tiles
  if (A >= WF) {
    *WA = WF;
    *WB = 1;
  } else {
    *WA = (int)A;
    *WB = WF / (int)A > 0 ? WF / (int)A : 1;
  }
  const int wf = *WA * *WB;
  return (2 * (size_t)I * (wf + 1) + I) * cb + (size_t)I * (cb / 2);
}

// X^ (complex, TC = float if !f64) <- X^ x_j (F_j D_j); first: X^ <- X x_1 (F_1 D_1) from the real batch.
int launch_mix_mode(const void *const *xslot, bool x_f64, void *Xh, bool f64, const int64_t *dims, int N, int j,
                    const double *d, cudaStream_t st) {
  MixDesc md;
  md.A = 1;
  for (int l = 0; l < j; ++l) md.A *= dims[l];
  md.B = 1;
  for (int l = j + 1; l < N; ++l) md.B *= dims[l];
  md.I = (int)dims[j];
  md.p = factor_p(md.I);
  md.q = md.I / md.p;
  const size_t smem = mix_mode_smem(md.I, f64, md.A, &md.WA, &md.WB);
  if (smem > 227 * 1024) return -1;
  md.nA = cdiv(md.A, md.WA);
  md.inc0 = 256 % md.WA;
  md.inc1 = (256 / md.WA) % md.I;
  md.inc2 = 256 / (md.WA * md.I);
  md.d = d;
  const int64_t tiles = md.nA * cdiv(md.B, md.WB);
  const unsigned grid = (unsigned)tiles;
  static PerDeviceOnce attr_once;   // once, before any capture (the first call comes from the uncaptured init)
  once_per_device(attr_once, [&] {
    const int mx = 227 * 1024;
    cudaFuncSetAttribute(k_mix_mode<double, double, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    cudaFuncSetAttribute(k_mix_mode<double, float, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    cudaFuncSetAttribute(k_mix_mode<float, double, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    cudaFuncSetAttribute(k_mix_mode<float, float, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    cudaFuncSetAttribute(k_mix_mode<double, double, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    cudaFuncSetAttribute(k_mix_mode<float, float, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  });
  if (!f64) {   // the fp32 mixing path: compile-time p x q kernels where the factorization is listed
    static PerDeviceOnce pq_once;
    once_per_device(pq_once, [&] {
      for (const MixPQEntry &e : kMixPQ) {
        cudaFuncSetAttribute(e.first_f32, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        cudaFuncSetAttribute(e.first_f64, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        cudaFuncSetAttribute(e.rest, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      }
    });
    for (const MixPQEntry &e : kMixPQ) {
      if (e.p != md.p || e.q != md.q) continue;
      MixPQFn fn = j > 0 ? e.rest : (x_f64 ? e.first_f64 : e.first_f32);
      fn<<<grid, 256, smem, st>>>(xslot, (float2 *)Xh, md);
      return 0;
    }
  }
#define KS_MIX(TI, TC, F) k_mix_mode<TI, TC, F><<<grid, 256, smem, st>>>(xslot, (typename C2<TC>::t *)Xh, md)
  if (j == 0) {
    if (x_f64 && f64) KS_MIX(double, double, true);
    else if (x_f64) KS_MIX(double, float, true);
    else if (f64) KS_MIX(float, double, true);
    else KS_MIX(float, float, true);
  } else {
    if (f64) KS_MIX(double, double, false);
    else KS_MIX(float, float, false);
  }
#undef KS_MIX
  return 0;
}

int launch_mix_sample(const double *G, int64_t I, int S, const int32_t *idx, int64_t m, const double *d, double2 *out,
                      double2 *core_ws, cudaStream_t st) {
  const size_t smem = sizeof(double2) * (size_t)I;
  if (smem > 200 * 1024) return -1;
  static PerDeviceOnce attr_once;
  once_per_device(attr_once, [&] {
    cudaFuncSetAttribute(k_mix_sample, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_mix_core, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  });
  if (core_ws && I <= m) {
    k_mix_core<<<(unsigned)cdiv(I * S, 128), 128, smem, st>>>(G, (int)I, S, d, core_ws);
    k_gather_crows<<<(unsigned)cdiv(m * S, 256), 256, 0, st>>>(core_ws, S, idx, m, out);
    return 2;
  }
  k_mix_sample<<<(unsigned)cdiv(m * S, 256), 256, smem, st>>>(G, I, S, idx, m, d, out);
  return 1;
}

// the mixed core, then the uniform draw fused with the gather of its sampled rows (draw s of the
// stream (seed, tau, k) recomputed per thread, counter-based; idx[s] written by c == 0)
__global__ void k_draw_gather_crows(uint64_t seed, const int64_t *__restrict__ tau, int k, int N, int64_t I, int64_t m,
                                    const double2 *__restrict__ Gh, int S, int32_t *__restrict__ idx,
                                    double2 *__restrict__ out) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= m * S) return;
  const int64_t s = e / S;
  const int c = (int)(e - s * S);
  const uint64_t key = seed ^ (0x9E3779B97F4A7C15ull * (uint64_t)(1 + (*tau) * (N + 1) + k));
  const int64_t ix = (int64_t)__umul64hi(ks_splitmix_at(key, (uint64_t)s), (uint64_t)I);
  if (c == 0) idx[s] = (int32_t)ix;
  out[e] = Gh[ix * S + c];
}

int launch_mix_sample_draw(const double *G, int64_t I, int S, uint64_t seed, const int64_t *tau, int k, int N, int64_t m,
                           const double *d, double2 *out, double2 *core_ws, int32_t *idx, cudaStream_t st) {
  const size_t smem = sizeof(double2) * (size_t)I;
  if (smem > 200 * 1024 || !core_ws) return -1;
  static PerDeviceOnce attr_once;
  once_per_device(attr_once, [&] {
    cudaFuncSetAttribute(k_mix_core, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  });
  k_mix_core<<<(unsigned)cdiv(I * S, 128), 128, smem, st>>>(G, (int)I, S, d, core_ws);
  k_draw_gather_crows<<<(unsigned)cdiv(m * S, 256), 256, 0, st>>>(seed, tau, k, N, I, m, core_ws, S, idx, out);
  return 2;
}

int launch_chain_complex(const double2 *const *G, const int *Ra, const int *Rb, int nf, int64_t m, double *out,
                         cudaStream_t st) {
  if (nf < 1 || nf > kMaxFactors) return -1;
  CFactorList fl;
  fl.n = nf;
  for (int l = 0; l < nf; ++l) {
    if (Ra[l] > 16 || Rb[l] > 16) return -1;
    fl.G[l] = G[l];
    fl.Ra[l] = Ra[l];
    fl.Rb[l] = Rb[l];
  }
  k_chain_complex<<<(unsigned)cdiv(m * Ra[0], 128), 128, 0, st>>>(fl, m, out);
  return 0;
}

int launch_gather_unmix(const void *Xh, bool f64, const int64_t *dims, int N, int n, const int32_t *idx, int64_t m,
                        const double *d, double *out, cudaStream_t st) {
  UnmixDesc ud;
  ud.N = N;
  ud.n = n;
  int64_t sd = 1;
  for (int j = 0; j < 8; ++j) {
    ud.stride[j] = j < N ? sd : 0;
    if (j < N) sd *= dims[j];
  }
  ud.I = dims[n - 1];
  ud.m = m;
  ud.idx = idx;
  ud.d = d;
  const size_t smem = sizeof(double2) * (size_t)(kUnmixSB + 1) * ud.I;
  if (smem > 200 * 1024) return -1;
  static PerDeviceOnce attr_once;
  once_per_device(attr_once, [&] {
    cudaFuncSetAttribute(k_gather_unmix<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_gather_unmix<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  });
  const unsigned grid = (unsigned)cdiv(m, kUnmixSB);
  if (f64) k_gather_unmix<double><<<grid, 128, smem, st>>>((const double2 *)Xh, ud, out);
  else k_gather_unmix<float><<<grid, 128, smem, st>>>((const float2 *)Xh, ud, out);
  return 0;
}

}  // namespace strb200
