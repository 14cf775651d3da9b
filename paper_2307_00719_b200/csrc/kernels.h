// kernels.h — host-side launchers of the STR device kernels (internal to libstr).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace strb200 {

// Diagnostic what-if knob, compiled in only with -DSTR_DIAG (tools/gpu_whatif.sh builds such a
// library; STR_DBG_SKIP is read at str_init): launchers whose bit is set enqueue nothing, so a
// timing run shows how much of the step each kernel class holds.  Results are meaningless while
// it is non-zero.  1 spd_inv, 2 tables, 4 contraction, 8 absorbs, 16 chain GEMMs, 32 row GEMMs,
// 64 Z Grams.  Release builds: the constant 0 (every skip test folds away).
#ifdef STR_DIAG
extern int g_dbg_skip;
#else
constexpr int g_dbg_skip = 0;
#endif
// SMs the contraction's persistent grid leaves to the side stream's concurrent kernels (the Gram
// chain links and the single-CTA factorizations run beside a pass)
constexpr int kSideSMs = 4;

// kernels_chain.cu
void launch_set_identity(double *A, int n, cudaStream_t s);
// chain_factor.cu: the factor V = L^{-1} (Sp x Sp, Sp = S rounded up to 8, blocks on and below the
// diagonal; sym(Q) = L L^T) of an SPD S x S matrix (S <= STR_MAXW), so Q^{-1} = V^T V; a non-positive
// pivot sets *info = 1.
void launch_spd_factor(const double *Q, int S, double *V, int *info, cudaStream_t s);
size_t spd_factor_doubles(int S);
// out = P Q^{-1} = (P V^T) V for I rows of P (I x S, row-major).
void launch_rows_solve(const double *P, const double *V, int S, int64_t I, double *out, cudaStream_t s);

void launch_chain_gemm(const double *A, const double *B, double *C, int M, int N, int K, QEpi q, cudaStream_t s);
void launch_gram_z2(const double *G, int64_t I, int Ra, int Rb, double *Zm, int accumulate, cudaStream_t s);
void launch_absorb2(const AbsorbDesc &ad, const void *Y, bool y_f32, double *out, int accumulate, cudaStream_t s);
int launch_build_table2(const TableDesc &td, double *out64, float *tiles, cudaStream_t s);
int launch_gemm_sk(const double *A, int64_t sai, int64_t sak, const double *B, int64_t sbk, int64_t sbj, double *C,
                   int M, int N, int64_t K, int acc, double *ws, cudaStream_t s, int sym = 0);
size_t gemm_sk_ws_doubles(int M, int N, int64_t K);
void launch_axpy_any(const void *x, bool x_f32, double *y, int64_t n, int accumulate, cudaStream_t s);

// kernels_contract_f64.cu
int launch_contract_f64(const void *const *X, bool x_is_f64, int pass, const double *Btab, int W, int64_t L, int64_t Rr,
                        int64_t tn, double *out, double *ws, cudaStream_t s);
void launch_set_ptr(const void **slot, const void *p, cudaStream_t s);
void *set_ptr_kernel();
void prepare_kernel_attrs();
// Every kernel of the step prefers the maximum shared-memory carve-out, so the SMs never switch
// their L1 / shared split between the 227 KB contraction and its neighbours (a switch drains the
// SM and costs microseconds per launch).
template <class F>
inline void prefer_max_smem(F *f) {
  cudaFuncSetAttribute((const void *)f, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
}
void prepare_f64_attrs();
int launch_fit_gemm(const void *X, bool x_is_f64, const double *TLf, const double *TR, int Ra, int Rb, int64_t L,
                    int64_t Rr, int64_t tn, double *TRp, double2 *partials, double *acc2, cudaStream_t s);
size_t fit_gemm_partials(int64_t L, int64_t Rr, int64_t tn);
void launch_fit_reduce(const double2 *partials, int64_t n, double *acc2, cudaStream_t s);
void launch_append_rows(double *GN, int64_t *dT, const double *GNnew, int64_t tn, int SN, cudaStream_t s);
size_t contract_f64_ws_doubles(int64_t M, int64_t K, int W);
size_t fit_partials(int64_t L, int64_t Rr, int64_t tn);
int launch_fit(const void *X, bool x_is_f64, const double *TLf, const double *TR, int Ra, int Rb, int64_t L,
               int64_t Rr, int64_t tn, double2 *partials, double *acc2, cudaStream_t s);


// ksrft.cu (rSTR-K)
void launch_draw_signs(uint64_t seed, const int64_t *tau, int N, int64_t total, double *d, cudaStream_t st);
int launch_mix_mode(const void *const *xslot, bool x_f64, void *Xh, bool f64, const int64_t *dims, int N, int j,
                    const double *d, cudaStream_t st);
int launch_mix_sample(const double *G, int64_t I, int S, const int32_t *idx, int64_t m, const double *d, double2 *out,
                      double2 *core_ws, cudaStream_t st);   // returns the number of launches (< 0: error)
int launch_mix_sample_draw(const double *G, int64_t I, int S, uint64_t seed, const int64_t *tau, int k, int N, int64_t m,
                           const double *d, double2 *out, double2 *core_ws, int32_t *idx, cudaStream_t st);
int launch_chain_complex(const double2 *const *G, const int *Ra, const int *Rb, int nf, int64_t m, double *out,
                         cudaStream_t st);
int launch_gather_unmix(const void *Xh, bool f64, const int64_t *dims, int N, int n, const int32_t *idx, int64_t m,
                        const double *d, double *out, cudaStream_t st);

}  // namespace strb200
