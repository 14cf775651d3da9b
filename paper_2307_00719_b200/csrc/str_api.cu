// str_api.cu — C ABI (include/str.h) and the per-batch orchestration of STR (Alg. 4,
// PAPER.md P:353-384) on one B200 (and its mode-1-sharded multi-GPU form).
//
// Per batch ("exact two-pass schedule"):
//   0. Gram-chain suffixes Sf_n = Z_{N-1} ... Z_{n+1} from the current Z's, and
//      H^{≠N} = Sf_1 Z_1 (Alg. 4 l.8).
//   1. table T_R = G_{k+1}(i_{k+1}) ... G_{N-1}(i_{N-1}) (old cores) and pass 1 over X_new -> Y_L.
//   2. temporal: M_N = sum_l (G_1...G_k)(l) Y_L(l,t); G_N^new = M_N (H^{≠N}_<2>)^{-1}
//      (l.9); append (l.10); Z_N^new.
//   3. left modes j = 1..k: M_j from Y_L, G_N^new and the current cores; P_j += M_j (l.14);
//      Q_j += (Lp_j Z_N^new Sf_j)_<2> (l.15-16, Prop. 1); G_j = P_j Q_j^{-1} (l.17); Z_j (l.18).
//   4. table T_L = G_N^new(t) G_1(i_1)...G_k(i_k) (new cores) and pass 2 over X_new -> Y_R.
//   5. right modes j = k+1..N-1: as 3, from Y_R.
// Everything is enqueued on one stream; no host synchronization inside a batch (STR).
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"
#include "kernels.h"
#include "str.h"
#include "str_internal.h"

using namespace strb200;

// ------------------------------------------------------------------------------------ helpers
#define CU(call)                                                                     \
  do {                                                                               \
    cudaError_t _e = (call);                                                         \
    if (_e != cudaSuccess) return fail(h, STR_E_CUDA, std::string(#call) + ": " +    \
                                       cudaGetErrorString(_e));                     \
  } while (0)

#define TRY(call)                  \
  do {                             \
    str_status _s = (call);        \
    if (_s != STR_OK) return _s;   \
  } while (0)

static str_status fail(str_state *h, str_status s, const std::string &msg) {
  if (h) {
    h->err = msg;
    if (s == STR_E_CUDA || s == STR_E_NUMERIC || s == STR_E_NCCL || s == STR_E_OOM) h->poisoned = true;
  }
  return s;
}

static str_status ensure(str_state *h, DevBuf &b, size_t bytes) {
  if (b.bytes >= bytes) return STR_OK;
  if (b.p) {   // captured graphs may hold the old pointer
    h->reset_graphs();
    cudaFree(b.p);
  }
  b.p = nullptr;
  b.bytes = 0;
  if (bytes == 0) return STR_OK;
  cudaError_t e = cudaMalloc(&b.p, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(h, STR_E_OOM, std::string("cudaMalloc failed: ") + cudaGetErrorString(e));
  }
  b.bytes = bytes;
  return STR_OK;
}

static str_status check_launch(str_state *h, const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(h, STR_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return STR_OK;
}

// ------------------------------------------------------------------------------------ collectives
// Sum-allreduce of device data across the mode-1 shards (no-op on one GPU), on the handle's current
// stream: NCCL or the in-process loopback group (comm.cu).
static str_status allreduce(str_state *h, void *buf, size_t n, bool f32 = false) {
  if (h->p == 1 || n == 0) return STR_OK;
  const std::string e = h->comm->allreduce(buf, n, f32, h->st);
  if (!e.empty()) return fail(h, STR_E_NCCL, e);
  h->collectives++;
  return STR_OK;
}

// ------------------------------------------------------------------------------------ geometry
static inline int RR(const str_state *h, int n) { return h->R[(n - 1) % h->N]; }   // R_n, n in 1..N+1

static Factor core_factor(const str_state *h, int n, int64_t stride) {
  const ModeBuf &m = h->md[n - 1];
  Factor f;
  f.G = (const double *)m.G.p;
  f.I = (int32_t)m.I;
  f.Ra = m.Ra;
  f.Rb = m.Rb;
  f.stride = stride;
  return f;
}

static Factor temporal_factor_at(const str_state *h, const double *rows0, int64_t rows, int64_t stride) {
  Factor f;
  f.G = rows0;
  f.I = (int32_t)rows;
  f.Ra = RR(h, h->N);
  f.Rb = RR(h, 1);
  f.stride = stride;
  return f;
}

static Factor temporal_factor(const str_state *h, int64_t row0, int64_t rows, int64_t stride) {
  Factor f;
  f.G = (const double *)h->GN.p + row0 * (int64_t)h->SN;
  f.I = (int32_t)rows;
  f.Ra = RR(h, h->N);
  f.Rb = RR(h, 1);
  f.stride = stride;
  return f;
}

// ------------------------------------------------------------------------------------ absorbs
struct AOp {
  int mode;      // mode id whose index is contracted (N = time)
  int left;
  Factor A;      // slices (stride unused)
};

// Runs a sequence of absorbs starting from Y (multi-index over `modes`, entries P x Q; fp32 when
// y_f32, else fp64).  The final result is written (accumulate=0) or added (accumulate=1) into dst.
static str_status run_absorbs(str_state *h, const void *Y, bool y_f32, std::vector<int> modes,
                              std::vector<int64_t> dims, int P, int Q, const std::vector<AOp> &ops, double *dst,
                              int accumulate) {
  if (ops.empty()) {
    int64_t n = (int64_t)P * Q;
    for (auto d : dims) n *= d;
    launch_axpy_any(Y, y_f32, dst, n, accumulate, h->st);
    tl_mark(h, "axpy");
    return check_launch(h, "axpy");
  }
  const void *cur = Y;
  bool cur_f32 = y_f32;
  for (size_t s = 0; s < ops.size(); ++s) {
    const AOp &op = ops[s];
    AbsorbDesc ad;
    ad.nd = (int)dims.size();
    for (int j = 0; j < ad.nd; ++j) ad.d[j] = dims[j];
    ad.pos = (int)(std::find(modes.begin(), modes.end(), op.mode) - modes.begin());
    ad.P = P;
    ad.Q = Q;
    ad.left = op.left;
    ad.A = op.A.G;
    ad.Ra = op.A.Ra;
    ad.Rb = op.A.Rb;
    bool last = s + 1 == ops.size();
    double *out = last ? dst : (double *)((s % 2 == 0) ? h->tmpA.p : h->tmpB.p);
    launch_absorb2(ad, cur, cur_f32, out, last ? accumulate : 0, h->st);
    tl_mark(h, "absorb");
    TRY(check_launch(h, "absorb"));
    if (op.left) P = op.A.Ra; else Q = op.A.Rb;
    modes.erase(modes.begin() + ad.pos);
    dims.erase(dims.begin() + ad.pos);
    cur = out;
    cur_f32 = false;
  }
  return STR_OK;
}

// ------------------------------------------------------------------------------------ chains
// out = A (MxK) * B (KxN) (Gram-chain matrices), with identity flags.
static str_status chain_mul(str_state *h, const double *A, bool A_id, const double *B, bool B_id, double *out, int M,
                            int N, int K) {
  if (A_id && B_id) {
    launch_set_identity(out, M, h->st);
  } else if (A_id) {
    CU(cudaMemcpyAsync(out, B, sizeof(double) * K * N, cudaMemcpyDeviceToDevice, h->st));
    return STR_OK;
  } else if (B_id) {
    CU(cudaMemcpyAsync(out, A, sizeof(double) * M * K, cudaMemcpyDeviceToDevice, h->st));
    return STR_OK;
  } else {
    launch_chain_gemm(A, B, out, M, N, K, QEpi{nullptr, 0, 0, 0}, h->st);
  }
  tl_mark(h, "chain_gemm");
  return check_launch(h, "chain_gemm");
}

// Suffix Sf_n (1 <= n <= N-2).  Sf_{N-2} = Z_{N-1} itself (no copy): Z_{N-1} changes only at the
// last mode's Gram refresh, after every use of the suffixes in the step.
static const double *sf(const str_state *h, int n) {
  return (const double *)(n == h->N - 2 ? h->md[h->N - 2].Zm.p : h->Sf[n].p);
}

// Sf_n = Z_{N-1} ... Z_{n+1} (Sf_{N-1} = I), from the current Z's (Alg. 4 l.15 right part).
static str_status build_suffixes(str_state *h) {
  const int N = h->N;
  for (int n = N - 3; n >= 1; --n) {
    // Sf_n = Sf_{n+1} * Zm_{n+1};  Sf_{n+1}: R_N^2 x R_{n+2}^2, Zm_{n+1}: R_{n+2}^2 x R_{n+1}^2
    int M = RR(h, N) * RR(h, N), K = RR(h, n + 2) * RR(h, n + 2), Nc = RR(h, n + 1) * RR(h, n + 1);
    TRY(chain_mul(h, sf(h, n + 1), false, (const double *)h->md[n].Zm.p, false, (double *)h->Sf[n].p, M, Nc, K));
  }
  return STR_OK;
}

// H = Lp * Zmid * Sf_n (Prop. 1 chain), then Q (+)= H_<2> (l.16) in the epilogue
// of the last chain product.  Lp and Sf are never both identities for N >= 3.
static str_status q_update(str_state *h, int n, const double *Lp, bool Lp_id, const double *Zmid, int accumulate,
                           double *Qout) {
  const int N = h->N;
  int a = RR(h, n) * RR(h, n), b = RR(h, 1) * RR(h, 1), c = RR(h, N) * RR(h, N), d = RR(h, n + 1) * RR(h, n + 1);
  bool Sf_id = (n == N - 1);
  QEpi q{Qout, RR(h, n), RR(h, n + 1), accumulate ? 2 : 1};
  if (Lp_id) {
    launch_chain_gemm(Zmid, sf(h, n), nullptr, b, d, c, q, h->st);
  } else if (Sf_id) {
    launch_chain_gemm(Lp, Zmid, nullptr, a, c, b, q, h->st);
  } else {
    TRY(chain_mul(h, Lp, false, Zmid, false, (double *)h->T1.p, a, c, b));
    launch_chain_gemm((const double *)h->T1.p, sf(h, n), nullptr, a, d, c, q, h->st);
  }
  tl_mark(h, "chain_gemm_q");
  return check_launch(h, "chain_gemm_q");
}

// ------------------------------------------------------------------------------------ tables
// T_R[r] = G_{k+1}(i_{k+1}) ... G_{N-1}(i_{N-1})   (R_{k+1} x R_N) over the right multi-index r.
static TableDesc desc_TR(const str_state *h) {
  TableDesc td;
  td.fl.n = 0;
  int64_t stride = 1;
  for (int i = h->k + 1; i <= h->N - 1; ++i) {
    td.fl.f[td.fl.n++] = core_factor(h, i, stride);
    stride *= h->md[i - 1].I;
  }
  td.Lk = h->Rr;
  td.tk = 1;
  td.Npad = 0;
  return td;
}

// T_L[l + L t] = G_N(t0 + t) G_1(i_1) ... G_k(i_k)   (R_N x R_{k+1}) over (l, t).
static TableDesc desc_TL_at(const str_state *h, const double *rows0, int64_t tn) {
  TableDesc td;
  td.fl.n = 0;
  td.fl.f[td.fl.n++] = temporal_factor_at(h, rows0, tn, h->L);
  int64_t stride = 1;
  for (int i = 1; i <= h->k; ++i) {
    td.fl.f[td.fl.n++] = core_factor(h, i, stride);
    stride *= h->md[i - 1].I;
  }
  td.Lk = h->L;
  td.tk = tn;
  td.Npad = 0;
  return td;
}

static str_status build_table(str_state *h, TableDesc td, double *out64, float *tiles, const char *name) {
  if (launch_build_table2(td, out64, tiles, h->st) != 0)
    return fail(h, STR_E_ARG, "chained-slice table needs too much shared memory for this shape");
  tl_mark(h, name);
  return check_launch(h, name);
}

static TableDesc desc_TL(const str_state *h, int64_t t0, int64_t tn) {
  return desc_TL_at(h, (const double *)h->GN.p + t0 * (int64_t)h->SN, tn);
}

// ------------------------------------------------------------------------------------ contraction
// One pass of the two-pass schedule over X.  The pass's table operand (pass 1: T_R from
// the current cores; pass 2: T_L from the new temporal rows [trows, +tn) and the updated left cores) is
// built by build_pass_table — on the step graph's third branch, overlapping other work: T_L beside
// Z_k's Gram, and the NEXT step's T_R at the end of this step beside Z_{N-1}'s Gram and the append
// (the right-group cores are final by then) — and run_pass contracts.  For 3xTF32 the table kernel also
// clears the pass output (the contraction accumulates into it with TMA reduce-adds); pass 1's output
// is cleared at its full capacity, since the next step's t_new is not known when it is built.
static str_status build_pass_table(str_state *h, int pass, const double *trows, int64_t tn) {
  const int W = RR(h, h->k + 1) * RR(h, h->N);
  if (pass == 2 && tf32_gen_rank(h) > 0) {
    // fused generation: only the prefix rows F[(f, t)] = G_N(t) G_1(i_1) ... G_{k-1}(i_{k-1}) (fp32,
    // tn Lf rows); the contraction multiplies each K-tile's rows by G_k itself
    TableDesc td = desc_TL_at(h, trows, tn);
    td.fl.n -= 1;   // drop G_k
    int64_t Lf = 1;
    for (int i = 1; i <= h->k - 1; ++i) Lf *= h->md[i - 1].I;
    td.fl.f[0].stride = Lf;
    td.Lk = Lf;
    td.out32 = (float *)h->F32.p;
    td.zero = (float4 *)h->tf_part2.p;
    td.zero_n4 = (h->Rr * W + 3) / 4;
    return build_table(h, td, nullptr, nullptr, "table_F");
  }
  TableDesc td = pass == 1 ? desc_TR(h) : desc_TL_at(h, trows, tn);
  if (h->contract == STR_CONTRACT_3XTF32) {
    td.Npad = tf32_npad(W);
    td.zero = (float4 *)(pass == 1 ? h->tf_part.p : h->tf_part2.p);
    td.zero_n4 = ((pass == 1 ? h->L * h->ws_t : h->Rr) * W + 3) / 4;
    TRY(build_table(h, td, nullptr, (float *)(pass == 1 ? h->tab_split.p : h->tab_split2.p),
                    pass == 1 ? "table_TR" : "table_TL"));
  } else {
    TRY(build_table(h, td, (double *)(pass == 1 ? h->TR.p : h->TL.p), nullptr, pass == 1 ? "table_TR" : "table_TL"));
  }
  if (pass == 1) h->tr_ready = true;
  return STR_OK;
}

static str_status run_pass(str_state *h, const void *X, int pass, int64_t tn, const void **Y, bool *y_f32) {
  const int W = RR(h, h->k + 1) * RR(h, h->N);
  if (h->contract == STR_CONTRACT_3XTF32) {
    float *out = (float *)(pass == 1 ? h->tf_part.p : h->tf_part2.p);
    if (launch_contract_tf32(h, X, pass, W, tn, out, true) != 0)
      return fail(h, STR_E_CUDA, "tf32 contraction launch failed: " + h->err);
    *Y = out;
    *y_f32 = true;
  } else {
    const double *tab = (const double *)(pass == 1 ? h->TR.p : h->TL.p);
    double *out = (double *)(pass == 1 ? h->YL.p : h->YR.p);
    prof_mark(h, 2 * (pass - 1));
    int nl = launch_contract_f64((const void *const *)h->dX.p, h->dtype == STR_F64, pass, tab, W, h->L, h->Rr, tn,
                                 out, (double *)h->ws.p, h->st);
    tl_mark(h, pass == 1 ? "contract_f64_p1" : "contract_f64_p2", nl);
    prof_mark(h, 2 * (pass - 1) + 1);
    *Y = out;
    *y_f32 = false;
  }
  if (pass == 1) h->tr_ready = false;   // the pass-1 output now holds this pass's sums
  return check_launch(h, pass == 1 ? "contract pass 1" : "contract pass 2");
}

// Table build and pass in sequence on the current stream (init, test hooks).
static str_status contract(str_state *h, const void *X, int pass, const double *trows, int64_t tn, const void **Y,
                           bool *y_f32) {
  TRY(build_pass_table(h, pass, trows, tn));
  return run_pass(h, X, pass, tn, Y, y_f32);
}

// ------------------------------------------------------------------------------------ workspaces
static str_status ensure_workspace(str_state *h, int64_t tn) {
  if (tn <= h->ws_t) return STR_OK;
  h->tr_ready = false;   // the pass outputs may be reallocated (and the pass-1 zeroing covers ws_t)
  const int N = h->N, k = h->k;
  const int W1 = RR(h, k + 1) * RR(h, N);
  const int64_t Lt = h->L * tn;
  TRY(ensure(h, h->Wt, sizeof(double) * h->L * RR(h, k + 1) * RR(h, 1)));
  int64_t big = std::max<int64_t>(Lt, h->Rr) * STR_MAXR * STR_MAXR;
  TRY(ensure(h, h->tmpA, sizeof(double) * big));
  TRY(ensure(h, h->tmpB, sizeof(double) * big));
  int64_t mt = tn * h->SN;
  for (auto &m : h->md) mt = std::max<int64_t>(mt, m.I * m.Ra * m.Rb);
  TRY(ensure(h, h->Mt, sizeof(double) * mt));
  TRY(ensure(h, h->GNnew, sizeof(double) * tn * h->SN));
  if (h->contract == STR_CONTRACT_3XTF32) {
    TRY(tf32_ensure_workspace(h, tn));
  } else {
    TRY(ensure(h, h->TR, sizeof(double) * h->Rr * W1));
    TRY(ensure(h, h->TL, sizeof(double) * Lt * W1));
    TRY(ensure(h, h->YL, sizeof(double) * Lt * W1));
    TRY(ensure(h, h->YR, sizeof(double) * h->Rr * W1));
    size_t ws = std::max(contract_f64_ws_doubles(Lt, h->Rr, W1), contract_f64_ws_doubles(h->Rr, Lt, W1));
    TRY(ensure(h, h->ws, sizeof(double) * ws));
  }
  h->ws_t = tn;
  return STR_OK;
}

str_status ensure_temporal_capacity(str_state *h, int64_t need) {
  if (need <= h->Tcap) return STR_OK;
  int64_t cap = std::max<int64_t>(need, 2 * h->Tcap);
  DevBuf nb;
  TRY(ensure(h, nb, sizeof(double) * cap * h->SN));
  if (h->T > 0) CU(cudaMemcpyAsync(nb.p, h->GN.p, sizeof(double) * h->T * h->SN, cudaMemcpyDeviceToDevice, h->st));
  CU(cudaStreamSynchronize(h->st));
  cudaFree(h->GN.p);
  h->GN = nb;
  h->Tcap = cap;
  h->reset_graphs();   // the captured append nodes point at the old buffer
  return STR_OK;
}

// X into the device slot h->dX (read by the f64 contraction); recorded as a graph node when
// capturing so that replays can point it at the new batch.
static str_status set_x(str_state *h, const void *X) {
  launch_set_ptr((const void **)h->dX.p, X, h->st);
  tl_mark(h, "set_x");
  if (h->capturing) {
    cudaStreamCaptureStatus cs;
    const cudaGraphNode_t *deps = nullptr;
    size_t nd = 0;
    CU(cudaStreamGetCaptureInfo(h->st, &cs, nullptr, nullptr, &deps, &nd));
    if (nd != 1) return fail(h, STR_E_CUDA, "cannot locate the captured set_x node");
    h->gs[h->cur_slot].setx = deps[0];
  }
  return check_launch(h, "set_x");
}

// ------------------------------------------------------------------------------------ left/right modes
// Absorb ops producing M_j for a left-group mode j (1 <= j <= k) from W (modes 1..k, entries
// R_{k+1} x R_1): right with G_1..G_{j-1} (current = new), left with G_k..G_{j+1} (old).
static std::vector<AOp> left_ops(const str_state *h, int j) {
  std::vector<AOp> ops;
  for (int i = 1; i < j; ++i) ops.push_back({i, 0, core_factor(h, i, 1)});
  for (int i = h->k; i > j; --i) ops.push_back({i, 1, core_factor(h, i, 1)});
  return ops;
}

// M_j for a right-group mode j (k < j < N) from Y_R (modes k+1..N-1, entries R_N x R_{k+1}):
// left with G_{N-1}..G_{j+1} (old), right with G_{k+1}..G_{j-1} (new).
static std::vector<AOp> right_ops(const str_state *h, int j) {
  std::vector<AOp> ops;
  for (int i = h->N - 1; i > j; --i) ops.push_back({i, 1, core_factor(h, i, 1)});
  for (int i = h->k + 1; i < j; ++i) ops.push_back({i, 0, core_factor(h, i, 1)});
  return ops;
}

static void left_modes(const str_state *h, std::vector<int> &modes, std::vector<int64_t> &dims) {
  modes.clear();
  dims.clear();
  for (int i = 1; i <= h->k; ++i) {
    modes.push_back(i);
    dims.push_back(h->md[i - 1].I);
  }
}

static void right_modes(const str_state *h, std::vector<int> &modes, std::vector<int64_t> &dims) {
  modes.clear();
  dims.clear();
  for (int i = h->k + 1; i <= h->N - 1; ++i) {
    modes.push_back(i);
    dims.push_back(h->md[i - 1].I);
  }
}


// G_j = P_j Q_j^{-1} (Alg. 4 l.17).
static str_status finish_rows(str_state *h, int j) {
  ModeBuf &m = h->md[j - 1];
  const int S = m.Ra * m.Rb;
  launch_rows_solve((const double *)m.P.p, (const double *)m.Qi.p, S, m.I, (double *)m.G.p, h->st);
  tl_mark(h, "rows_solve");
  return check_launch(h, "rows_solve");
}

// Z_j (l.18), reduced across the shards of the row-sharded G_1.
static str_status finish_gram(str_state *h, int j) {
  ModeBuf &m = h->md[j - 1];
  launch_gram_z2((const double *)m.G.p, m.I, m.Ra, m.Rb, (double *)m.Zm.p, 0, h->st);
  tl_mark(h, "gram_z");
  TRY(check_launch(h, "gram_z"));
  if (j == 1) TRY(allreduce(h, m.Zm.p, (size_t)m.Ra * m.Ra * m.Rb * m.Rb));   // G_1 row-sharded
  return STR_OK;
}

static str_status finish_mode(str_state *h, int j) {
  TRY(finish_rows(h, j));
  return finish_gram(h, j);
}

// Q (+)= (A B)_<2> (the last link of a Prop. 1 chain with the l.16 regrouping; the chain GEMM's Q
// epilogue), then the factor V of sym(Q) (l.17's ^{-1}; chain_factor.cu).
static str_status gram_link_factor(str_state *h, const double *A, const double *B, int M, int Nc, int K, int Rn,
                                   int Rn1, int accumulate, double *Q, int S, double *V) {
  launch_chain_gemm(A, B, nullptr, M, Nc, K, QEpi{Q, Rn, Rn1, accumulate ? 2 : 1}, h->st);
  tl_mark(h, "chain_gemm_q");
  TRY(check_launch(h, "chain_gemm_q"));
  launch_spd_factor(Q, S, V, h->d_info, h->st);
  tl_mark(h, "spd_factor");
  return check_launch(h, "spd_factor");
}

// The Gram chains that need only the Z's of the previous step (Alg. 4 l.8 and the right parts of
// l.15): the suffixes Sf_n = Z_{N-1} R_n (n <= N-3; Sf_{N-2} is Z_{N-1} itself) and
// Hq = H^{≠N}_<2> = (Z_{N-1} R_0)_<2>, with R_n = Z_{N-2} ... Z_{n+1} (R_{N-3} = Z_{N-2}).  A step
// forms them at its end from its final Z's — R_n on the data stream while the last mode's chain
// runs (they need Z_1..Z_{N-2} only), then one product per chain after Z_{N-1}, beside the next
// pass-1 table — so that the next step starts with the factor of Hq alone beside pass 1 (pass-1 CTAs
// never wait for SMs held by these products).  side_ready: they hold the current Z's.
static const double *rc(const str_state *h, int n) {
  return (const double *)(n == h->N - 3 ? h->md[h->N - 3].Zm.p : h->Rc[n].p);
}
static str_status side_r_chain(str_state *h) {   // R_n, n = N-4 .. 0 (needs Z_1 .. Z_{N-2})
  const int N = h->N;
  for (int n = N - 4; n >= 0; --n) {
    // R_n = R_{n+1} Z_{n+1}:  R_{N-1}^2 x R_{n+2}^2 . R_{n+2}^2 x R_{n+1}^2
    TRY(chain_mul(h, rc(h, n + 1), false, (const double *)h->md[n].Zm.p, false, (double *)h->Rc[n].p,
                  RR(h, N - 1) * RR(h, N - 1), RR(h, n + 1) * RR(h, n + 1), RR(h, n + 2) * RR(h, n + 2)));
  }
  return STR_OK;
}
static str_status side_sf(str_state *h) {        // Sf_n = Z_{N-1} R_n, n = 1 .. N-3 (needs Z_{N-1})
  const int N = h->N;
  for (int n = 1; n <= N - 3; ++n)
    TRY(chain_mul(h, (const double *)h->md[N - 2].Zm.p, false, rc(h, n), false, (double *)h->Sf[n].p,
                  RR(h, N) * RR(h, N), RR(h, n + 1) * RR(h, n + 1), RR(h, N - 1) * RR(h, N - 1)));
  return STR_OK;
}
static str_status side_hq(str_state *h) {        // Hq = (Z_{N-1} R_0)_<2>  (needs Z_{N-1})
  const int N = h->N;
  launch_chain_gemm((const double *)h->md[N - 2].Zm.p, rc(h, 0), nullptr, RR(h, N) * RR(h, N), RR(h, 1) * RR(h, 1),
                    RR(h, N - 1) * RR(h, N - 1), QEpi{(double *)h->Hq.p, RR(h, N), RR(h, 1), 1}, h->st);
  tl_mark(h, "chain_gemm_q");
  return check_launch(h, "chain_gemm_q (Hq)");
}
static str_status side_prepare(str_state *h) {   // all of it, in order, on the current stream
  TRY(side_r_chain(h));
  TRY(side_sf(h));
  TRY(side_hq(h));
  h->side_ready = true;
  return STR_OK;
}

// The step's first side-branch work: the factor of Hq (Alg. 4 l.9's ^{-1}).
static str_status side_start(str_state *h) {
  launch_spd_factor((const double *)h->Hq.p, h->SN, (double *)h->Hi.p, h->d_info, h->st);
  tl_mark(h, "spd_factor");
  return check_launch(h, "spd_factor (Hq)");
}

// ------------------------------------------------------------------------------------ update (STR)
// Enqueues one STR step (no host synchronization, no host-side T): the new temporal rows go to the
// scratch GNnew and are appended at the device row counter at the end.
//
// Two streams (graph branches when capturing) plus a third for the pass tables.  The serial chain
// of the step — per mode: H_j = Z_{j-1} B_j with Q_j += H_<2>, the factor of Q_j, the rows
// G_j = P_j Q_j^{-1}, the Gram Z_j — runs on the CHAIN stream (h->st2) as one sequence of
// programmatically dependent launches; the X-dependent work (passes, absorbs, allreduces) and the
// off-path chain products T1 / B run on the DATA stream (h->st at entry).  They meet through
// events: the data stream hands over M_N / P_j (evP) and B_{j+1} (evB); the chain stream hands over
// G_j (evR) and Z_j (evZ).  So the chain's kernel-to-kernel edges are same-stream (their launch
// latency hides behind the predecessor), and the data stream's waits sit off the critical path.
static str_status update_det_enqueue(str_state *h, const void *X, int64_t tn) {
  const int N = h->N, k = h->k;
  const bool serial = h->timeline != 0;   // the diagnostic timeline runs everything on one stream
  cudaStream_t D = h->st;
  cudaStream_t C = serial ? D : h->st2;
  cudaStream_t T3 = serial ? D : h->st3;
  auto rec = [&](cudaEvent_t e, cudaStream_t s) -> cudaError_t {
    return serial ? cudaSuccess : cudaEventRecord(e, s);
  };
  auto wait = [&](cudaStream_t s, cudaEvent_t e) -> cudaError_t {
    return serial ? cudaSuccess : cudaStreamWaitEvent(s, e, 0);
  };
  cudaEvent_t evP = h->ev_fork, evB = h->ev_join, evZ = h->ev_z;
  struct Restore {   // the handle's stream is D again on every exit path
    str_state *h;
    cudaStream_t d;
    ~Restore() { h->st = d; }
  } restore{h, D};

  h->st = D;
  TRY(set_x(h, X));
  // chain: suffix chains, H^{≠N} = Sf_1 Z_1 (Alg. 4 l.8) -> Hq and its factor (old state only)
  CU(rec(evP, D));
  CU(wait(C, evP));
  h->st = C;
  TRY(side_start(h));
  // data: pass 1 with the old cores (its table was built at the end of the previous step, or just
  // before this step: update_det), then M_N = (G_1...G_k) Y_L summed over l
  h->st = D;
  const void *YL;
  bool yl32;
  TRY(run_pass(h, X, 1, tn, &YL, &yl32));
  std::vector<int> modes;
  std::vector<int64_t> dims;
  left_modes(h, modes, dims);
  modes.push_back(N);
  dims.push_back(tn);
  std::vector<AOp> ops;
  for (int i = k; i >= 1; --i) ops.push_back({i, 1, core_factor(h, i, 1)});
  double *Mt = (double *)h->Mt.p;
  TRY(run_absorbs(h, YL, yl32, modes, dims, RR(h, k + 1), RR(h, N), ops, Mt, 0));
  TRY(allreduce(h, Mt, (size_t)tn * h->SN));                                   // site C1
  CU(rec(evP, D));
  // chain: G_N^new = M_N Hq^{-1} (l.9) and Z_N^new
  h->st = C;
  CU(wait(C, evP));
  double *GN_new = (double *)h->GNnew.p;
  launch_rows_solve(Mt, (const double *)h->Hi.p, h->SN, tn, GN_new, h->st);    // l.9
  tl_mark(h, "rows_solve");
  TRY(check_launch(h, "temporal solve"));
  launch_gram_z2(GN_new, tn, RR(h, N), RR(h, 1), (double *)h->ZmN.p, 0, h->st);  // Z_N^new
  tl_mark(h, "gram_z");
  TRY(check_launch(h, "gram_z"));
  CU(rec(evZ, C));   // (also certifies G_N^new)
  // modes 1..N-1 in order (Gauss-Seidel).  Gram chain of mode j (Prop. 1 with the new Z's before
  // j and the old ones after): H_j = Lp_j Z_N^new Sf_j, Lp_j = Z_{j-1} ... Z_1.  Carried as
  // T1_j = Lp_j Z_N^new (T1_1 = Z_N^new, T1_{j+1} = Z_j T1_j) and B_{j+1} = T1_j Sf_{j+1}, both
  // formed on the data stream while mode j's factor runs, so that once Z_j is known the chain's
  // only product before Q_{j+1}'s factor is H_{j+1} = Z_j B_{j+1}.
  const double *T1cur = (const double *)h->ZmN.p;   // T1_j (R_j^2 x R_N^2)
  int t1buf = 0;
  const double *Bj = nullptr;                       // B_j (R_{j-1}^2 x R_{j+1}^2), j >= 2
  const void *YR = nullptr;
  bool yr32 = false;
  const int k2 = tf32_gen_rank(h) > 0 ? k - 1 : k;   // the mode after whose rows pass 2's table is built
  for (int j = 1; j <= N - 1; ++j) {
    ModeBuf &m = h->md[j - 1];
    const int S = RR(h, j) * RR(h, j + 1);
    // chain: Q_j += H_j<2> (l.15-16) and the factor of Q_j (l.17's ^{-1})
    h->st = C;
    if (j == 1) {   // H_1 = Z_N^new Sf_1  (R_1^2 x R_N^2 . R_N^2 x R_2^2)
      if (N - 1 == 1) return fail(h, STR_E_ARG, "order N >= 3 required");
      TRY(gram_link_factor(h, (const double *)h->ZmN.p, sf(h, 1), RR(h, 1) * RR(h, 1), RR(h, 2) * RR(h, 2),
                           RR(h, N) * RR(h, N), RR(h, j), RR(h, j + 1), 1, (double *)m.Q.p, S, (double *)m.Qi.p));
    } else {        // H_j = Z_{j-1} B_j  (R_j^2 x R_{j-1}^2 . R_{j-1}^2 x R_{j+1}^2)
      CU(wait(C, evB));
      TRY(gram_link_factor(h, (const double *)h->md[j - 2].Zm.p, Bj, RR(h, j) * RR(h, j),
                           RR(h, j + 1) * RR(h, j + 1), RR(h, j - 1) * RR(h, j - 1), RR(h, j), RR(h, j + 1), 1,
                           (double *)m.Q.p, S, (double *)m.Qi.p));
    }
    // data: T1_j and B_{j+1} for the next mode (need Z_{j-1}, or Z_N^new for j = 1)
    h->st = D;
    CU(wait(D, evZ));
    if (j == N - 1) TRY(side_r_chain(h));   // next step's chains: R_n (Z_1 .. Z_{N-2} are final)
    if (j + 1 <= N - 1) {
      if (j >= 2) {   // T1_j = Z_{j-1} T1_{j-1}
        double *t1n = (double *)h->Lp[t1buf].p;
        TRY(chain_mul(h, (const double *)h->md[j - 2].Zm.p, false, T1cur, false, t1n, RR(h, j) * RR(h, j),
                      RR(h, N) * RR(h, N), RR(h, j - 1) * RR(h, j - 1)));
        T1cur = t1n;
        t1buf ^= 1;
      }
      if (j + 1 == N - 1) {
        Bj = T1cur;   // Sf_{N-1} = I
      } else {        // B_{j+1} = T1_j Sf_{j+1}  (R_j^2 x R_N^2 . R_N^2 x R_{j+2}^2)
        // (ping-pong: the chain stream may still be reading B_j while B_{j+1} is formed)
        double *bn = (double *)((j & 1) ? h->T1.p : h->H.p);
        TRY(chain_mul(h, T1cur, false, sf(h, j + 1), false, bn, RR(h, j) * RR(h, j),
                      RR(h, j + 2) * RR(h, j + 2), RR(h, N) * RR(h, N)));
        Bj = bn;
      }
      CU(rec(evB, D));
    }
    // data: P_j += X_new[j] G^{≠j}_new (l.13-14), with the new G_1..G_{j-1} (evZ above also
    // certifies G_{j-1}: the chain stream writes Z_{j-1} after G_{j-1})
    if (j <= k) {
      left_modes(h, modes, dims);
      if (j == 1) {
        // W = Y_L absorbed over t with G_N^new on the right: modes 1..k, entries R_{k+1} x R_1
        std::vector<int> m2 = modes;
        std::vector<int64_t> d2 = dims;
        m2.push_back(N);
        d2.push_back(tn);
        std::vector<AOp> o1 = {{N, 0, temporal_factor_at(h, GN_new, tn, 1)}};
        TRY(run_absorbs(h, YL, yl32, m2, d2, RR(h, k + 1), RR(h, N), o1, (double *)h->Wt.p, 0));
      }
      auto lo = left_ops(h, j);
      if (j == 1 || h->p == 1) {
        TRY(run_absorbs(h, h->Wt.p, false, modes, dims, RR(h, k + 1), RR(h, 1), lo, (double *)m.P.p, 1));
      } else {   // M_j sums over the sharded i_1: reduce before accumulating (site C2)
        TRY(run_absorbs(h, h->Wt.p, false, modes, dims, RR(h, k + 1), RR(h, 1), lo, Mt, 0));
        TRY(allreduce(h, Mt, (size_t)m.I * m.Ra * m.Rb));
        launch_axpy_any(Mt, false, (double *)m.P.p, m.I * m.Ra * m.Rb, 1, h->st);
        tl_mark(h, "axpy");
      }
    } else {
      if (j == k + 1) {   // pass 2 with the new cores (table built on the third branch after mode k's rows)
        if (!serial) CU(cudaStreamWaitEvent(D, h->ev_join3, 0));
        TRY(run_pass(h, X, 2, tn, &YR, &yr32));
        TRY(allreduce(h, const_cast<void *>(YR), (size_t)h->Rr * RR(h, k + 1) * RR(h, N), yr32));   // site C2'
      }
      right_modes(h, modes, dims);
      TRY(run_absorbs(h, YR, yr32, modes, dims, RR(h, N), RR(h, k + 1), right_ops(h, j), (double *)m.P.p, 1));
    }
    CU(rec(evP, D));
    // chain: G_j = P_j Q_j^{-1} (l.17), then Z_j (l.18)
    h->st = C;
    CU(wait(C, evP));
    TRY(finish_rows(h, j));
    if (j == k2 || j == N - 1) {
      // third branch: pass 2's table (G_N^new and the new G_1..G_k) beside Z_k -- with the fused
      // generation only its prefix rows (G_N^new, G_1..G_{k-1}), beside Z_{k-1} -- or the next
      // step's pass-1 table (final right-group cores) beside Z_{N-1}
      CU(rec(h->ev_fork3, C));
      CU(wait(T3, h->ev_fork3));
      h->st = T3;
      TRY(build_pass_table(h, j == k2 ? 2 : 1, j == k2 ? GN_new : nullptr, tn));
      CU(rec(h->ev_join3, T3));
      h->st = C;
    }
    TRY(finish_gram(h, j));
    CU(rec(evZ, C));
    if (j == N - 1) {   // next step's Hq (chain stream, after Z_{N-1})
      TRY(side_hq(h));
      CU(rec(h->ev_hq, C));
    }
  }
  // data: l.10, append the new temporal rows (G_N^new certified by the first evZ wait); the next
  // step's suffixes after Z_{N-1}; then the step ends when the chain (Hq) and the third branch
  // (next pass-1 table) are done
  h->st = D;
  launch_append_rows((double *)h->GN.p, (int64_t *)h->dT.p, GN_new, tn, h->SN, h->st);
  tl_mark(h, "append");
  TRY(check_launch(h, "append"));
  CU(wait(D, evZ));
  TRY(side_sf(h));
  CU(wait(D, h->ev_hq));
  CU(wait(D, h->ev_join3));
  return STR_OK;
}

// One STR step: replays the captured graph of update_det_enqueue (capturing it on first use or
// when t_new changes).  Profiling replays a second graph that also records events around the two
// contraction passes (accumulated by str_profile); the timeline diagnostic runs eagerly.
static str_status update_det(str_state *h, const void *X, int64_t tn) {
  TRY(ensure_workspace(h, tn));
  TRY(ensure_temporal_capacity(h, h->T + tn));
  if (h->profiling && !h->pev[0]) {
    for (auto &e : h->pev) CU(cudaEventCreate(&e));
  }
  if (!h->tr_ready) TRY(build_pass_table(h, 1, nullptr, tn));   // (outside the graph: first step, after init)
  if (!h->side_ready) TRY(side_prepare(h));                       // (likewise)
  const bool graph = h->use_graph && !h->timeline;
  if (!graph) {
    TRY(update_det_enqueue(h, X, tn));
  } else {
    const int slot = h->profiling ? 1 : 0;
    str_state::GraphSlot &g = h->gs[slot];
    if (!g.exec || g.tn != tn) {
      g.reset();
      CU(cudaStreamBeginCapture(h->st, cudaStreamCaptureModeThreadLocal));
      h->capturing = true;
      h->cur_slot = slot;
      const int64_t l0 = h->launches;
      str_status st = update_det_enqueue(h, X, tn);
      h->capturing = false;
      cudaGraph_t cg = nullptr;
      cudaError_t e = cudaStreamEndCapture(h->st, &cg);
      if (st != STR_OK) {
        if (cg) cudaGraphDestroy(cg);
        return st;
      }
      if (e != cudaSuccess) return fail(h, STR_E_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
      e = cudaGraphInstantiate(&g.exec, cg, h->chain_prio ? cudaGraphInstantiateFlagUseNodePriority : 0);
      if (e != cudaSuccess) {
        cudaGraphDestroy(cg);
        return fail(h, STR_E_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
      }
      g.graph = cg;
      g.tn = tn;
      g.launches = h->launches - l0;
      h->launches = l0;
    } else {
      // point the replay at this batch
      void *slotp = h->dX.p;
      const void *xp = X;
      void *args[2] = {&slotp, &xp};
      cudaKernelNodeParams kp = {};
      kp.func = set_ptr_kernel();
      kp.gridDim = dim3(1);
      kp.blockDim = dim3(1);
      kp.kernelParams = args;
      CU(cudaGraphExecKernelNodeSetParams(g.exec, g.setx, &kp));
      if (h->contract == STR_CONTRACT_3XTF32) {
        TRY(tf32_graph_update(h, slot, 1, X, tn));
        TRY(tf32_graph_update(h, slot, 2, X, tn));
      }
    }
    CU(cudaGraphLaunch(g.exec, h->st));
    h->launches += g.launches;
  }
  if (h->profiling) {   // pass times of this step (events on the library stream)
    CU(cudaStreamSynchronize(h->st));
    for (int ps = 0; ps < 2; ++ps) {
      float ms = 0.0f;
      if (cudaEventElapsedTime(&ms, h->pev[2 * ps], h->pev[2 * ps + 1]) == cudaSuccess) {
        h->prof_ms[ps] += ms;
        h->prof_n[ps] += 1;
      }
    }
  }
  h->T += tn;
  return STR_OK;
}

// ------------------------------------------------------------------------------------ loopback driver
// Test hook (not part of include/str.h): one STR step of all p in-process ranks of a loopback group
// (STR_COMM_LOOPBACK).  graph = 0: every rank's step is enqueued eagerly by its own host thread (the
// ranks meet at the collective sites on the host).  graph = 1: the p steps are captured once into
// ONE CUDA graph — p stream branches joined by the collective sites' sum nodes — and replayed; the
// X buffers must then be the same on every call (the graph holds their addresses).
extern "C" STR_API str_status strdbg_loopback_step(str_state **hs, int32_t p, const void **X, int64_t tn,
                                                   int32_t graph) {
  if (!hs || !X || p < 1 || tn < 1) return STR_E_ARG;
  for (int r = 0; r < p; ++r)
    if (!hs[r] || hs[r]->poisoned || hs[r]->p != p || !hs[r]->loop_group || hs[r]->variant != STR_DET)
      return STR_E_ARG;
  std::vector<str_status> st(p, STR_OK);
  if (!graph) {
    std::vector<std::thread> th;
    for (int r = 0; r < p; ++r) th.emplace_back([&, r] { st[r] = str_update_batch(hs[r], X[r], tn); });
    for (auto &t : th) t.join();
    for (int r = 0; r < p; ++r)
      if (st[r] != STR_OK) return st[r];
    return STR_OK;
  }
  str_state *h = hs[0];
  cudaSetDevice(h->device);
  int64_t *etn = nullptr;
  std::vector<const void *> *ex = nullptr;
  cudaGraphExec_t &exec = loopback_exec(loopback_group_of(h->comm), &etn, &ex);
  bool fresh = false;
  for (int r = 0; r < p; ++r) {
    const void *old = hs[r]->GN.p;
    const int64_t old_ws = hs[r]->ws_t;
    TRY(ensure_workspace(hs[r], tn));
    TRY(ensure_temporal_capacity(hs[r], hs[r]->T + tn));
    if (hs[r]->GN.p != old || hs[r]->ws_t != old_ws) fresh = true;   // (the group's graph holds old buffers)
    if (!hs[r]->tr_ready) TRY(build_pass_table(hs[r], 1, nullptr, tn));   // first step: pass-1 table
    if (!hs[r]->side_ready) TRY(side_prepare(hs[r]));
  }
  bool same = exec && *etn == tn && !fresh && (int)ex->size() == p;
  for (int r = 0; same && r < p; ++r) same = (*ex)[r] == X[r];
  if (!same) {
    if (exec) cudaGraphExecDestroy(exec);
    exec = nullptr;
    cudaEvent_t fork_ev, join_ev[16];
    CU(cudaEventCreateWithFlags(&fork_ev, cudaEventDisableTiming));
    for (int r = 0; r < p; ++r) CU(cudaEventCreateWithFlags(&join_ev[r], cudaEventDisableTiming));
    CU(cudaStreamBeginCapture(h->st, cudaStreamCaptureModeRelaxed));
    cudaEventRecord(fork_ev, h->st);
    for (int r = 1; r < p; ++r) cudaStreamWaitEvent(hs[r]->st, fork_ev, 0);
    std::vector<std::thread> th;
    for (int r = 0; r < p; ++r)
      th.emplace_back([&, r] {
        cudaSetDevice(hs[r]->device);
        st[r] = update_det_enqueue(hs[r], X[r], tn);
      });
    for (auto &t : th) t.join();
    for (int r = 1; r < p; ++r) {
      cudaEventRecord(join_ev[r], hs[r]->st);
      cudaStreamWaitEvent(h->st, join_ev[r], 0);
    }
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(h->st, &g);
    cudaEventDestroy(fork_ev);
    for (int r = 0; r < p; ++r) cudaEventDestroy(join_ev[r]);
    for (int r = 0; r < p; ++r)
      if (st[r] != STR_OK) {
        if (g) cudaGraphDestroy(g);
        return st[r];
      }
    if (e != cudaSuccess) return fail(h, STR_E_CUDA, std::string("loopback capture: ") + cudaGetErrorString(e));
    e = cudaGraphInstantiate(&exec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return fail(h, STR_E_CUDA, std::string("loopback instantiate: ") + cudaGetErrorString(e));
    *etn = tn;
    ex->assign(X, X + p);
  }
  CU(cudaGraphLaunch(exec, h->st));
  for (int r = 0; r < p; ++r) hs[r]->T += tn;
  return STR_OK;
}

// ------------------------------------------------------------------------------------ init (STR)
// Alg. 4 l.1-5: Z_1..Z_N, P_n = X_init[n] G^{≠n}_[2], Q_n = H^{≠n}_<2> with all init cores.
static str_status init_det(str_state *h, const void *X, int64_t tn) {
  const int N = h->N, k = h->k;
  TRY(ensure_workspace(h, tn));
  // Z_N over the whole init temporal core
  launch_gram_z2((const double *)h->GN.p, tn, RR(h, N), RR(h, 1), (double *)h->ZmN.p, 0, h->st);
  tl_mark(h, "gram_z");
  TRY(build_suffixes(h));
  // pass 1 (init cores), W from the init temporal rows
  TRY(set_x(h, X));
  const void *YL;
  bool yl32;
  TRY(contract(h, X, 1, nullptr, tn, &YL, &yl32));
  std::vector<int> modes;
  std::vector<int64_t> dims;
  left_modes(h, modes, dims);
  modes.push_back(N);
  dims.push_back(tn);
  {
    std::vector<AOp> o1 = {{N, 0, temporal_factor(h, 0, tn, 1)}};
    TRY(run_absorbs(h, YL, yl32, modes, dims, RR(h, k + 1), RR(h, N), o1, (double *)h->Wt.p, 0));
  }
  double *Mt = (double *)h->Mt.p;
  bool Lp_id = true;
  int lp_cur = 0;
  const void *YR = nullptr;
  bool yr32 = false;
  for (int j = 1; j <= N - 1; ++j) {
    ModeBuf &m = h->md[j - 1];
    if (j <= k) {
      left_modes(h, modes, dims);
      auto lo = left_ops(h, j);
      TRY(run_absorbs(h, h->Wt.p, false, modes, dims, RR(h, k + 1), RR(h, 1), lo, Mt, 0));
      if (j > 1) TRY(allreduce(h, Mt, (size_t)m.I * m.Ra * m.Rb));
    } else {
      if (j == k + 1) {
        TRY(contract(h, X, 2, (const double *)h->GN.p, tn, &YR, &yr32));
        TRY(allreduce(h, const_cast<void *>(YR), (size_t)h->Rr * RR(h, k + 1) * RR(h, N), yr32));
      }
      right_modes(h, modes, dims);
      TRY(run_absorbs(h, YR, yr32, modes, dims, RR(h, N), RR(h, k + 1), right_ops(h, j), Mt, 0));
    }
    CU(cudaMemcpyAsync(m.P.p, Mt, sizeof(double) * m.I * m.Ra * m.Rb, cudaMemcpyDeviceToDevice, h->st));
    TRY(q_update(h, j, (const double *)h->Lp[lp_cur].p, Lp_id, (const double *)h->ZmN.p, 0, (double *)m.Q.p));
    if (j < N - 1) {
      int M = RR(h, j + 1) * RR(h, j + 1), K = RR(h, j) * RR(h, j), Nc = RR(h, 1) * RR(h, 1);
      TRY(chain_mul(h, (const double *)m.Zm.p, false, (const double *)h->Lp[lp_cur].p, Lp_id,
                    (double *)h->Lp[1 - lp_cur].p, M, Nc, K));
      lp_cur = 1 - lp_cur;
      Lp_id = false;
    }
  }
  h->side_ready = false;   // the next step forms Sf_n / Hq from these Z's first
  return STR_OK;
}

// ------------------------------------------------------------------------------------ ABI
static str_status deferred_check(str_state *h) {
  if (h->poisoned) return STR_E_POISONED;
  cudaError_t e = cudaStreamSynchronize(h->st);
  if (e != cudaSuccess) return fail(h, STR_E_CUDA, std::string("stream: ") + cudaGetErrorString(e));
  int info = 0;
  e = cudaMemcpy(&info, h->d_info, sizeof(int), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return fail(h, STR_E_CUDA, std::string("info: ") + cudaGetErrorString(e));
  if (info && !g_dbg_skip) return fail(h, STR_E_NUMERIC, "SPD inversion of Q_n met a non-positive pivot");
  return STR_OK;
}

static int auto_split(const std::vector<int64_t> &dims, int N) {
  // choose k in [1, N-2] minimizing |Y_L| + |Y_R| relative sizes (prod of left dims ~ small)
  int best = 1;
  double bestc = 1e300;
  for (int k = 1; k <= N - 2; ++k) {
    double L = 1, Rr = 1;
    for (int i = 0; i < k; ++i) L *= (double)dims[i];
    for (int i = k; i < N - 1; ++i) Rr *= (double)dims[i];
    double c = L + Rr;
    if (c < bestc) {
      bestc = c;
      best = k;
    }
  }
  return best;
}

extern "C" str_status str_init(const str_config *cfg, const void *X_init, int64_t t_init,
                               const double *const *init_cores, str_state **out) {
  if (!cfg || !out || !init_cores || !X_init) return STR_E_ARG;
  *out = nullptr;
  const int N = cfg->order;
  if (N < 3 || !cfg->dims || !cfg->ranks) return STR_E_ARG;
  if (t_init < 1) return STR_E_SHAPE;
  for (int n = 0; n < N; ++n)
    if (cfg->ranks[n] < 1 || cfg->ranks[n] > STR_MAXR) return STR_E_ARG;
  for (int n = 0; n < N; ++n)
    if (cfg->ranks[n] * cfg->ranks[(n + 1) % N] > STR_MAXW) return STR_E_ARG;
  for (int n = 0; n < N - 1; ++n)
    if (cfg->dims[n] < 1) return STR_E_SHAPE;
  const int p = cfg->world_size < 1 ? 1 : cfg->world_size;
  if (cfg->rank < 0 || cfg->rank >= p) return STR_E_ARG;
  if (cfg->dims[0] % p != 0) return STR_E_PRECOND;
  if (cfg->split_k < 0 || cfg->split_k > N - 2) return STR_E_ARG;
  if (cfg->dtype != STR_F32 && cfg->dtype != STR_F64) return STR_E_ARG;
  if (cfg->variant < STR_DET || cfg->variant > STR_SAMPLE_KSRFT) return STR_E_ARG;
  if (cfg->variant != STR_DET && p > 1) return STR_E_PRECOND;   // rSTR runs as replicas only
  if (cfg->variant != STR_DET) {
    int64_t need = 0;
    for (int n = 0; n < N; ++n) need = std::max<int64_t>(need, (int64_t)cfg->ranks[n] * cfg->ranks[(n + 1) % N]);
    if (cfg->sketch_rows < need) return STR_E_PRECOND;
  }

  str_state *h = new str_state();
  h->N = N;
  h->dims_g.assign(cfg->dims, cfg->dims + N - 1);
  h->R.assign(cfg->ranks, cfg->ranks + N);
  h->dtype = cfg->dtype;
  h->contract = cfg->contract;
  h->variant = cfg->variant;
  h->m = cfg->sketch_rows;
  h->seed = cfg->seed;
  h->p = p;
  h->rank = cfg->rank;
  h->device = cfg->device;
  h->k = cfg->split_k ? cfg->split_k : auto_split(h->dims_g, N);
  if (h->variant == STR_DET && cfg->ranks[h->k] * cfg->ranks[N - 1] > STR_MAXW) {
    // the two-pass outputs carry R_{k+1} R_N columns: one tensor-core N tile / one
    // 128-wide DMMA tile
    delete h;
    return STR_E_ARG;
  }
  h->xbytes = cfg->dtype == STR_F64 ? 8 : 4;

#ifdef STR_DIAG
  if (const char *sk = getenv("STR_DBG_SKIP")) {   // what-if timing diagnostic (tools/gpu_whatif.sh)
    g_dbg_skip = atoi(sk);
    if (g_dbg_skip)
      fprintf(stderr, "libstr: STR_DBG_SKIP=%d skips kernel classes: results are WRONG (what-if timing only)\n",
              g_dbg_skip);
  }
#endif
  cudaError_t e = cudaSetDevice(cfg->device);
  if (e != cudaSuccess) {
    delete h;
    return STR_E_CUDA;
  }
  if (cudaDeviceGetAttribute(&h->nsm, cudaDevAttrMultiProcessorCount, cfg->device) != cudaSuccess) h->nsm = 148;
  // STR_CHAIN_PRIO=1 (A/B knob): the chain stream at the highest priority, kept by the step graph's
  // kernel nodes (cudaGraphInstantiateFlagUseNodePriority), so the serial chain's small kernels are
  // placed ahead of queued absorb / table CTAs
  int prio_lo = 0, prio_hi = 0;
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  h->chain_prio = getenv("STR_CHAIN_PRIO") && getenv("STR_CHAIN_PRIO")[0] == '1';
  if (cudaStreamCreateWithPriority(&h->st2, cudaStreamNonBlocking, h->chain_prio ? prio_hi : 0) != cudaSuccess ||
      cudaStreamCreateWithFlags(&h->st3, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_fork3, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_join3, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_z, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_hq, cudaEventDisableTiming) != cudaSuccess) {
    delete h;
    return STR_E_CUDA;
  }
  if (cfg->stream) {
    h->st = (cudaStream_t)cfg->stream;
    h->own_stream = false;
  } else {
    // blocking w.r.t. the legacy default stream, so X produced there is ordered before the step
    if (cudaStreamCreateWithFlags(&h->st, cudaStreamDefault) != cudaSuccess) {
      delete h;
      return STR_E_CUDA;
    }
    h->own_stream = true;
  }
  if (p > 1) {
    std::string why;
    if (cfg->comm == STR_COMM_LOOPBACK) {
      h->comm = comm_loopback(const_cast<void *>(cfg->nccl_id), p, cfg->rank, h, why);
      h->loop_group = const_cast<void *>(cfg->nccl_id);
      h->use_graph_forced_off = true;   // the group captures all ranks' steps into one graph
    } else {
      h->comm = comm_nccl(p, cfg->rank, cfg->nccl_id, why);
    }
    if (!h->comm) {
      h->err = why;
      *out = h;   // the caller reads str_error_string, then str_destroy
      return cfg->comm == STR_COMM_LOOPBACK ? STR_E_ARG : STR_E_NCCL;
    }
  }
  *out = h;

  // geometry (mode 1 sharded)
  h->md.resize(N - 1);
  h->i1_off = (cfg->dims[0] / p) * cfg->rank;
  for (int n = 1; n <= N - 1; ++n) {
    ModeBuf &m = h->md[n - 1];
    m.I = (n == 1) ? cfg->dims[0] / p : cfg->dims[n - 1];
    m.I_glob = cfg->dims[n - 1];
    m.Ra = RR(h, n);
    m.Rb = RR(h, n + 1);
  }
  h->SN = RR(h, N) * RR(h, 1);
  h->L = 1;
  for (int i = 1; i <= h->k; ++i) h->L *= h->md[i - 1].I;
  h->Rr = 1;
  for (int i = h->k + 1; i <= N - 1; ++i) h->Rr *= h->md[i - 1].I;

  // state buffers
  for (int n = 1; n <= N - 1; ++n) {
    ModeBuf &m = h->md[n - 1];
    const int S = m.Ra * m.Rb;
    TRY(ensure(h, m.G, sizeof(double) * m.I * S));
    TRY(ensure(h, m.P, sizeof(double) * m.I * S));
    TRY(ensure(h, m.Q, sizeof(double) * S * S));
    TRY(ensure(h, m.Zm, sizeof(double) * S * S));
    TRY(ensure(h, m.Qi, sizeof(double) * spd_factor_doubles(S)));
  }
  h->Tcap = std::max<int64_t>(cfg->t_capacity > 0 ? cfg->t_capacity : 4096, t_init);
  TRY(ensure(h, h->GN, sizeof(double) * h->Tcap * h->SN));
  int maxR2 = 0;
  for (int n = 0; n < N; ++n) maxR2 = std::max(maxR2, h->R[n] * h->R[n]);
  const size_t sq = (size_t)maxR2 * maxR2;
  TRY(ensure(h, h->ZmN, sizeof(double) * sq));
  h->Sf.resize(N);
  for (int n = 1; n <= N - 1; ++n) TRY(ensure(h, h->Sf[n], sizeof(double) * sq));
  h->Rc.resize(N);
  for (int n = 0; n <= N - 4; ++n) TRY(ensure(h, h->Rc[n], sizeof(double) * sq));
  TRY(ensure(h, h->Lp[0], sizeof(double) * sq));
  TRY(ensure(h, h->Lp[1], sizeof(double) * sq));
  TRY(ensure(h, h->T1, sizeof(double) * sq));
  TRY(ensure(h, h->H, sizeof(double) * sq));
  TRY(ensure(h, h->Hq, sizeof(double) * STR_MAXW * STR_MAXW));
  TRY(ensure(h, h->Hi, sizeof(double) * STR_MAXW * STR_MAXW));
  {
    DevBuf info;
    TRY(ensure(h, info, sizeof(int)));
    h->info_buf = info;
    h->d_info = (int *)info.p;
    CU(cudaMemsetAsync(h->d_info, 0, sizeof(int), h->st));
  }
  if (h->contract == STR_CONTRACT_3XTF32 && h->variant == STR_DET) TRY(tf32_prepare(h));   // rSTR has no dense pass
  TRY(ensure(h, h->dT, sizeof(int64_t)));
  TRY(ensure(h, h->dX, sizeof(void *)));
  prepare_kernel_attrs();
  {
    const char *ev = getenv("STR_NO_GRAPH");
    h->use_graph = !(ev && ev[0] == '1') && !h->use_graph_forced_off;
    const char *hd = getenv("STR_RSTR_HOST_DRAWS");   // diagnostic: the host sampler for rSTR draws
    h->rstr_dev = !(hd && hd[0] == '1');
  }

  // upload init cores: paper layout (a, i, b) at a + Ra*(i + I*b) -> G(2) rows [i][a + Ra*b]
  for (int n = 1; n <= N - 1; ++n) {
    ModeBuf &m = h->md[n - 1];
    const int S = m.Ra * m.Rb;
    std::vector<double> buf((size_t)m.I * S);
    int64_t off = (n == 1) ? h->i1_off : 0;
    for (int64_t i = 0; i < m.I; ++i)
      for (int b = 0; b < m.Rb; ++b)
        for (int a = 0; a < m.Ra; ++a)
          buf[i * S + a + m.Ra * b] = init_cores[n - 1][a + (int64_t)m.Ra * ((i + off) + m.I_glob * b)];
    CU(cudaMemcpyAsync(m.G.p, buf.data(), sizeof(double) * buf.size(), cudaMemcpyHostToDevice, h->st));
    CU(cudaStreamSynchronize(h->st));
    launch_gram_z2((const double *)m.G.p, m.I, m.Ra, m.Rb, (double *)m.Zm.p, 0, h->st);
    tl_mark(h, "gram_z");
    if (n == 1) TRY(allreduce(h, m.Zm.p, (size_t)S * S));
  }
  {
    const int RN = RR(h, N), R1 = RR(h, 1);
    std::vector<double> buf((size_t)t_init * h->SN);
    for (int64_t t = 0; t < t_init; ++t)
      for (int b = 0; b < R1; ++b)
        for (int a = 0; a < RN; ++a) buf[t * h->SN + a + RN * b] = init_cores[N - 1][a + (int64_t)RN * (t + t_init * b)];
    CU(cudaMemcpyAsync(h->GN.p, buf.data(), sizeof(double) * buf.size(), cudaMemcpyHostToDevice, h->st));
    CU(cudaStreamSynchronize(h->st));
  }
  h->T = t_init;
  {
    int64_t t0 = t_init;
    CU(cudaMemcpy(h->dT.p, &t0, sizeof(t0), cudaMemcpyHostToDevice));
  }
  str_status s = (h->variant == STR_DET) ? init_det(h, X_init, t_init) : rstr_init(h, X_init, t_init);
  if (s != STR_OK) return s;
  return deferred_check(h);
}

extern "C" str_status str_update_batch(str_state *h, const void *X_new, int64_t t_new) {
  if (!h) return STR_E_ARG;
  if (h->poisoned) return STR_E_POISONED;
  if (!X_new || t_new < 1) return fail(h, STR_E_ARG, "X_new must be non-NULL and t_new >= 1");
  cudaSetDevice(h->device);
  return (h->variant == STR_DET) ? update_det(h, X_new, t_new) : rstr_update(h, X_new, t_new);
}

extern "C" str_status str_update_batch_host(str_state *h, const void *X_host, int64_t t_new) {
  if (!h) return STR_E_ARG;
  if (h->poisoned) return STR_E_POISONED;
  if (!X_host || t_new < 1) return fail(h, STR_E_ARG, "X_new must be non-NULL and t_new >= 1");
  cudaSetDevice(h->device);
  size_t bytes = (size_t)h->L * h->Rr * t_new * h->xbytes;
  TRY(ensure(h, h->Xstage, bytes));
  CU(cudaMemcpyAsync(h->Xstage.p, X_host, bytes, cudaMemcpyHostToDevice, h->st));
  return str_update_batch(h, h->Xstage.p, t_new);
}

// Batch TR-ALS (include/str.h): each sweep is update_det over X with the history cleared
// (P_n = Q_n = 0, no temporal rows), i.e. Alg. 1 in the mode order N, 1..N-1; then Alg. 4's init.
extern "C" str_status str_tr_als(str_state *h, const void *X, int64_t t, int32_t sweeps, double *rel_err) {
  if (!h) return STR_E_ARG;
  if (h->poisoned) return STR_E_POISONED;
  if (!X || t < 1 || sweeps < 0) return fail(h, STR_E_ARG, "X must be non-NULL, t >= 1, sweeps >= 0");
  if (h->variant != STR_DET) return fail(h, STR_E_ARG, "str_tr_als needs an STR (deterministic) handle");
  cudaSetDevice(h->device);
  TRY(deferred_check(h));
  TRY(ensure_temporal_capacity(h, t));
  for (int s = 0; s < sweeps; ++s) {
    for (auto &m : h->md) {
      CU(cudaMemsetAsync(m.P.p, 0, sizeof(double) * m.I * m.Ra * m.Rb, h->st));
      CU(cudaMemsetAsync(m.Q.p, 0, sizeof(double) * (size_t)m.Ra * m.Rb * m.Ra * m.Rb, h->st));
    }
    const int64_t zero = 0;
    CU(cudaMemcpyAsync(h->dT.p, &zero, sizeof(zero), cudaMemcpyHostToDevice, h->st));
    CU(cudaStreamSynchronize(h->st));   // (the host value of zero must outlive the copy)
    h->T = 0;
    TRY(update_det(h, X, t));            // h->T = t afterwards
    TRY(deferred_check(h));
  }
  // Alg. 4 l.1-5 from the fitted cores: Z_N over all t rows, P_n, Q_n, Z_n
  h->T = t;
  {
    const int64_t tt = t;
    CU(cudaMemcpyAsync(h->dT.p, &tt, sizeof(tt), cudaMemcpyHostToDevice, h->st));
    CU(cudaStreamSynchronize(h->st));
  }
  TRY(init_det(h, X, t));   // (eager; not part of the step graph)
  TRY(deferred_check(h));
  if (rel_err) TRY(str_fit(h, X, 0, t, rel_err));
  return STR_OK;
}

extern "C" str_status str_sync(str_state *h) {
  if (!h) return STR_E_ARG;
  return deferred_check(h);
}

extern "C" str_status str_get_cores(str_state *h, int32_t n, double *host_out, int64_t capacity) {
  if (!h || !host_out) return STR_E_ARG;
  if (n < 1 || n > h->N) return fail(h, STR_E_ARG, "mode out of range");
  TRY(deferred_check(h));
  if (n == h->N) {
    const int RN = RR(h, h->N), R1 = RR(h, 1);
    if (capacity < h->T * h->SN) return fail(h, STR_E_ARG, "capacity too small");
    std::vector<double> buf((size_t)h->T * h->SN);
    CU(cudaMemcpy(buf.data(), h->GN.p, sizeof(double) * buf.size(), cudaMemcpyDeviceToHost));
    for (int64_t t = 0; t < h->T; ++t)
      for (int b = 0; b < R1; ++b)
        for (int a = 0; a < RN; ++a) host_out[a + (int64_t)RN * (t + h->T * b)] = buf[t * h->SN + a + RN * b];
    return STR_OK;
  }
  ModeBuf &m = h->md[n - 1];
  const int S = m.Ra * m.Rb;
  if (capacity < m.I_glob * S) return fail(h, STR_E_ARG, "capacity too small");
  std::vector<double> buf((size_t)m.I_glob * S);
  if (n == 1 && h->p > 1 && h->loop_group) {
    // in-process ranks: read every rank's shard of G_1 directly (no collective: the callers are
    // not concurrent here)
    for (int r = 0; r < h->p; ++r) {
      str_state *o = loopback_member(h->loop_group, r);
      if (!o) return fail(h, STR_E_ARG, "loopback rank missing");
      TRY(deferred_check(o));
      CU(cudaMemcpy(buf.data() + (size_t)r * m.I * S, o->md[0].G.p, sizeof(double) * m.I * S, cudaMemcpyDeviceToHost));
    }
  } else if (n == 1 && h->p > 1) {
    DevBuf gathered;
    TRY(ensure(h, gathered, sizeof(double) * m.I_glob * S));
    const std::string e = h->comm->allgather((const double *)m.G.p, (double *)gathered.p, (size_t)m.I * S, h->st);
    if (!e.empty()) {
      cudaFree(gathered.p);
      return fail(h, STR_E_NCCL, e);
    }
    CU(cudaStreamSynchronize(h->st));
    CU(cudaMemcpy(buf.data(), gathered.p, sizeof(double) * buf.size(), cudaMemcpyDeviceToHost));
    cudaFree(gathered.p);
  } else {
    CU(cudaMemcpy(buf.data(), m.G.p, sizeof(double) * buf.size(), cudaMemcpyDeviceToHost));
  }
  for (int64_t i = 0; i < m.I_glob; ++i)
    for (int b = 0; b < m.Rb; ++b)
      for (int a = 0; a < m.Ra; ++a) host_out[a + (int64_t)m.Ra * (i + m.I_glob * b)] = buf[i * S + a + m.Ra * b];
  return STR_OK;
}

extern "C" str_status str_get_temporal_rows(str_state *h, int64_t t0, int64_t t, double *host_out) {
  if (!h || !host_out) return STR_E_ARG;
  if (t0 < 0 || t < 0 || t0 + t > h->T) return fail(h, STR_E_ARG, "temporal range out of bounds");
  TRY(deferred_check(h));
  CU(cudaMemcpyAsync(host_out, (double *)h->GN.p + t0 * h->SN, sizeof(double) * t * h->SN, cudaMemcpyDeviceToHost,
                     h->st));
  CU(cudaStreamSynchronize(h->st));
  return STR_OK;
}

extern "C" str_status str_fit(str_state *h, const void *X, int64_t t0, int64_t t, double *rel_err) {
  if (!h || !X || !rel_err) return STR_E_ARG;
  if (t0 < 0 || t < 1 || t0 + t > h->T) return fail(h, STR_E_ARG, "temporal range out of bounds");
  TRY(deferred_check(h));
  const int N = h->N, k = h->k;
  const int Ra = RR(h, N), Rb = RR(h, k + 1);
  const int64_t chunk = 16;
  DevBuf tr, tl, parts, acc, trp;
  TRY(ensure(h, tr, sizeof(double) * h->Rr * Ra * Rb));
  TRY(ensure(h, trp, sizeof(double) * h->Rr * Ra * Rb));
  TRY(build_table(h, desc_TR(h), (double *)tr.p, nullptr, "table_TR"));
  TRY(ensure(h, tl, sizeof(double) * h->L * chunk * Ra * Rb));
  TRY(ensure(h, parts, sizeof(double2) * std::max(fit_partials(h->L, h->Rr, chunk), fit_gemm_partials(h->L, h->Rr, chunk))));
  TRY(ensure(h, acc, sizeof(double) * 2));
  CU(cudaMemsetAsync(acc.p, 0, sizeof(double) * 2, h->st));
  for (int64_t c0 = 0; c0 < t; c0 += chunk) {
    int64_t tn = std::min(chunk, t - c0);
    TRY(build_table(h, desc_TL(h, t0 + c0, tn), (double *)tl.p, nullptr, "table_TL"));
    const char *xp = (const char *)X + (size_t)h->L * h->Rr * c0 * h->xbytes;
    // X^hat = T_L T_R^T on the FP64 tensor-core fragments, residual sums in the epilogue (the row
    // GEMM needs L tn and R_r below 2^31 and the ranks' W <= 256)
    const bool fg = h->L * tn < ((int64_t)1 << 31) && cdiv(h->L * tn, 16) <= 65535 && h->Rr < ((int64_t)1 << 31) &&
                    Ra * Rb <= 256;
    int nf = fg ? launch_fit_gemm(xp, h->dtype == STR_F64, (const double *)tl.p, (const double *)tr.p, Ra, Rb, h->L,
                                  h->Rr, tn, (double *)trp.p, (double2 *)parts.p, (double *)acc.p, h->st)
                : launch_fit(xp, h->dtype == STR_F64, (const double *)tl.p, (const double *)tr.p, Ra, Rb, h->L,
                             h->Rr, tn, (double2 *)parts.p, (double *)acc.p, h->st);
    tl_mark(h, "fit", nf);
    TRY(check_launch(h, "fit"));
  }
  TRY(allreduce(h, (double *)acc.p, 2));
  double sums[2];
  CU(cudaMemcpyAsync(sums, acc.p, sizeof(sums), cudaMemcpyDeviceToHost, h->st));
  CU(cudaStreamSynchronize(h->st));
  cudaFree(tr.p);
  cudaFree(trp.p);
  cudaFree(tl.p);
  cudaFree(parts.p);
  cudaFree(acc.p);
  if (sums[1] == 0.0) return fail(h, STR_E_ARG, "||X|| = 0: relative error undefined");
  *rel_err = std::sqrt(sums[0] / sums[1]);
  return STR_OK;
}

extern "C" int64_t str_processed(const str_state *h) { return h ? h->T : 0; }
extern "C" const char *str_error_string(const str_state *h) { return h ? h->err.c_str() : "null handle"; }
extern "C" int64_t str_kernel_launches(const str_state *h) { return h ? h->launches : 0; }

extern "C" str_status str_set_profiling(str_state *h, int32_t enable) {
  if (!h) return STR_E_ARG;
  cudaStreamSynchronize(h->st);
  h->prof_ms[0] = h->prof_ms[1] = 0.0;
  h->prof_n[0] = h->prof_n[1] = 0;
  h->profiling = enable != 0;
  return STR_OK;
}

// Contraction pipeline trace (diagnostic, not in include/str.h): enable allocates a device buffer
// the tensor-core kernel fills (per pass a block of kTfDbgWords: per-unit timestamps of one CTA,
// then per-CTA globaltimer entry / setup / last MMA / exit); disable copies both blocks out.
extern "C" STR_API str_status strdbg_tftrace(str_state *h, int32_t enable, long long *host_out) {
  if (!h) return STR_E_ARG;
  cudaStreamSynchronize(h->st);
  if (enable) {
    if (!h->tf_dbg) {
      CU(cudaMalloc(&h->tf_dbg, 2 * str_state::kTfDbgWords * sizeof(long long)));
    }
    CU(cudaMemset(h->tf_dbg, 0, 2 * str_state::kTfDbgWords * sizeof(long long)));
  } else if (h->tf_dbg) {
    if (host_out) CU(cudaMemcpy(host_out, h->tf_dbg, 2 * str_state::kTfDbgWords * sizeof(long long), cudaMemcpyDeviceToHost));
    cudaFree(h->tf_dbg);
    h->tf_dbg = nullptr;
    h->reset_graphs();   // captured contraction nodes may point at the freed trace buffer
  }
  return STR_OK;
}

// Launch timeline (diagnostic, not in include/str.h): enable clears it; dump aggregates the
// in-stream time between consecutive marks per kernel name as "name total_ms count" lines.
extern "C" STR_API str_status strdbg_timeline(str_state *h, int32_t enable) {
  if (!h) return STR_E_ARG;
  cudaStreamSynchronize(h->st);
  for (auto &e : h->tl) cudaEventDestroy(e.second);
  h->tl.clear();
  h->timeline = enable != 0;
  if (h->timeline) tl_mark(h, "begin", 0);
  return STR_OK;
}

extern "C" STR_API int64_t strdbg_timeline_dump(str_state *h, char *buf, int64_t cap) {
  if (!h || !buf || cap < 1) return -1;
  cudaStreamSynchronize(h->st);
  std::vector<std::string> names;
  std::vector<double> ms;
  std::vector<int64_t> cnt;
  for (size_t i = 1; i < h->tl.size(); ++i) {
    float t = 0;
    cudaEventElapsedTime(&t, h->tl[i - 1].second, h->tl[i].second);
    std::string nm = h->tl[i].first;
    size_t j = std::find(names.begin(), names.end(), nm) - names.begin();
    if (j == names.size()) {
      names.push_back(nm);
      ms.push_back(0);
      cnt.push_back(0);
    }
    ms[j] += t;
    cnt[j]++;
  }
  std::string out;
  for (size_t j = 0; j < names.size(); ++j)
    out += names[j] + " " + std::to_string(ms[j]) + " " + std::to_string(cnt[j]) + "\n";
  int64_t n = std::min<int64_t>((int64_t)out.size(), cap - 1);
  memcpy(buf, out.data(), n);
  buf[n] = 0;
  return n;
}

extern "C" str_status str_profile(str_state *h, double *p1_ms, int64_t *p1_n, double *p2_ms, int64_t *p2_n) {
  if (!h) return STR_E_ARG;
  CU(cudaStreamSynchronize(h->st));
  if (p1_ms) *p1_ms = h->prof_ms[0];
  if (p1_n) *p1_n = h->prof_n[0];
  if (p2_ms) *p2_ms = h->prof_ms[1];
  if (p2_n) *p2_n = h->prof_n[1];
  return STR_OK;
}

extern "C" void str_destroy(str_state *h) {
  if (!h) return;
  cudaSetDevice(h->device);
  cudaStreamSynchronize(h->st);
  h->free_all();
  delete h->comm;
  h->comm = nullptr;
  if (h->st2) {
    cudaStreamSynchronize(h->st2);
    cudaStreamDestroy(h->st2);
  }
  if (h->st3) {
    cudaStreamSynchronize(h->st3);
    cudaStreamDestroy(h->st3);
  }
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_join) cudaEventDestroy(h->ev_join);
  if (h->ev_fork3) cudaEventDestroy(h->ev_fork3);
  if (h->ev_join3) cudaEventDestroy(h->ev_join3);
  if (h->ev_z) cudaEventDestroy(h->ev_z);
  if (h->ev_hq) cudaEventDestroy(h->ev_hq);
  if (h->own_stream) cudaStreamDestroy(h->st);
  delete h;
}

// ------------------------------------------------------------------------------------ test hook
// Not part of include/str.h: runs one contraction pass with the current cores (pass 1: T_R;
// pass 2: T_L over temporal rows [0, tn)) and copies Y (fp64) to host.  Used by the GPU unit
// tests of the contraction kernels.
extern "C" STR_API str_status strdbg_contract(str_state *h, const void *X, int32_t pass, int64_t tn, double *host_out) {
  if (!h || !X || !host_out || (pass != 1 && pass != 2) || tn < 1 || tn > h->T) return STR_E_ARG;
  TRY(ensure_workspace(h, tn));
  const int W1 = RR(h, h->k + 1) * RR(h, h->N);
  const void *Y;
  bool y32;
  TRY(set_x(h, X));
  TRY(contract(h, X, pass, (const double *)h->GN.p, tn, &Y, &y32));
  CU(cudaStreamSynchronize(h->st));
  size_t n = (size_t)(pass == 1 ? h->L * tn : h->Rr) * W1;
  if (y32) {
    std::vector<float> f(n);
    CU(cudaMemcpy(f.data(), Y, n * sizeof(float), cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < n; ++i) host_out[i] = f[i];
  } else {
    CU(cudaMemcpy(host_out, Y, n * sizeof(double), cudaMemcpyDeviceToHost));
  }
  return STR_OK;
}

// Test hook (not in include/str.h): the uniform rank of pass 2's in-kernel table generation for this
// handle (0: pass 2 reads the pre-tiled table).
extern "C" STR_API int32_t strdbg_tf32_gen_rank(const str_state *h) { return h ? tf32_gen_rank(h) : -1; }

// Launch-cost probe (diagnostic, not in include/str.h): builds the pass's table once, then times
// `reps` back-to-back launches of only the contraction (memset + kernel) between two events on the
// library stream; returns the average milliseconds per launch in *ms.
extern "C" STR_API str_status strdbg_contract_repeat(str_state *h, const void *X, int32_t pass, int64_t tn, int32_t reps,
                                                     double *ms) {
  if (!h || !X || !ms || (pass != 1 && pass != 2) || tn < 1 || tn > h->T || reps < 1) return STR_E_ARG;
  if (h->contract != STR_CONTRACT_3XTF32) return STR_E_ARG;
  TRY(ensure_workspace(h, tn));
  const int W = RR(h, h->k + 1) * RR(h, h->N);
  const void *Y;
  bool y32;
  TRY(set_x(h, X));
  TRY(contract(h, X, pass, (const double *)h->GN.p, tn, &Y, &y32));
  cudaEvent_t e0, e1;
  CU(cudaEventCreate(&e0));
  CU(cudaEventCreate(&e1));
  float *out = (float *)(pass == 1 ? h->tf_part.p : h->tf_part2.p);
  CU(cudaEventRecord(e0, h->st));
  for (int i = 0; i < reps; ++i)
    if (launch_contract_tf32(h, X, pass, W, tn, out, false) != 0) return fail(h, STR_E_CUDA, h->err);
  CU(cudaEventRecord(e1, h->st));
  CU(cudaEventSynchronize(e1));
  float t = 0.0f;
  CU(cudaEventElapsedTime(&t, e0, e1));
  *ms = t / reps;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return STR_OK;
}

// Test hook (not part of include/str.h): Q^{-1} of `count` SPD S x S matrices (host, row-major)
// through the library's SPD-inverse kernel on `device`; returns the pivot-failure flag in *info.
extern "C" STR_API str_status strdbg_spd_inv(int32_t device, int32_t S, int32_t count, const double *Q_host,
                                              double *Qinv_host, int32_t *info_host, int32_t reps, float *us) {
  if (S < 1 || S > STR_MAXW || count < 1 || !Q_host || !Qinv_host) return STR_E_ARG;
  if (cudaSetDevice(device) != cudaSuccess) return STR_E_CUDA;
  const size_t n = (size_t)S * S;
  // Q^{-1} = I Q^{-1} through the factor kernel and the row solve with P = I
  double *dQ = nullptr, *dQi = nullptr, *ws = nullptr, *dI = nullptr;
  int *dinfo = nullptr;
  str_status st = STR_OK;
  if (cudaMalloc(&dQ, n * count * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&dQi, n * count * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&ws, spd_factor_doubles(S) * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&dI, n * sizeof(double)) != cudaSuccess || cudaMalloc(&dinfo, sizeof(int)) != cudaSuccess) {
    st = STR_E_OOM;
  } else {
    std::vector<double> eye(n, 0.0);
    for (int i = 0; i < S; ++i) eye[(size_t)i * S + i] = 1.0;
    cudaMemcpy(dI, eye.data(), n * sizeof(double), cudaMemcpyHostToDevice);
    cudaMemcpy(dQ, Q_host, n * count * sizeof(double), cudaMemcpyHostToDevice);
    cudaMemset(dinfo, 0, sizeof(int));
    for (int c = 0; c < count; ++c) {
      launch_spd_factor(dQ + c * n, S, ws, dinfo, 0);
      launch_rows_solve(dI, ws, S, S, dQi + c * n, 0);
    }
    if (cudaDeviceSynchronize() != cudaSuccess) st = STR_E_CUDA;
    if (reps > 0 && us && st == STR_OK) {   // average time per inverse, back-to-back launches
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0, 0);
      for (int r = 0; r < reps; ++r) launch_spd_factor(dQ, S, ws, dinfo, 0);
      cudaEventRecord(e1, 0);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      *us = 1000.f * ms / reps;
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
    }
    cudaMemcpy(Qinv_host, dQi, n * count * sizeof(double), cudaMemcpyDeviceToHost);
    int inf = 0;
    cudaMemcpy(&inf, dinfo, sizeof(int), cudaMemcpyDeviceToHost);
    if (info_host) *info_host = inf;
  }
  cudaFree(dQ);
  cudaFree(dQi);
  cudaFree(ws);
  cudaFree(dI);
  cudaFree(dinfo);
  return st;
}
