// dmma.cuh — FP64 tensor-core fragments (mma.sync m8n8k4 f64) and cluster helpers shared by the
// fp64 chain kernels (sm_100a has no fp64 tcgen05 kind: DMMA is the FP64 tensor path).
//
// Fragment layout of mma.sync.aligned.m8n8k4.row.col.f64 (lane l, g = l >> 2, t = l & 3):
//   A (8 x 4, row-major):  lane holds A[g][t]
//   B (4 x 8, col-major):  lane holds B[t][g]
//   C (8 x 8):             lane holds C[g][2t], C[g][2t + 1]
// Shared-memory tiles used as A (element [row][k] at row * ld + k) or as B through its transpose
// (element [n][k] at n * ld + k) are read conflict-free when ld % 16 == 4 (the 16 lanes of a
// 64-bit access phase hit 16 distinct 8-byte slots: 4 g + t).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace strb200 {

__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// 8 x 8 x 8 product: c += A B with A given as rows (A[g][k] at pa[g * lda + k]) and B given
// through its transpose (B[k][n] = BT[n][k] at pb[n * ldb + k]).
__device__ __forceinline__ void dmma8_tn(double (&c)[2], const double *pa, int lda, const double *pb, int ldb, int g,
                                         int t) {
  dmma(c[0], c[1], pa[g * lda + t], pb[g * ldb + t]);
  dmma(c[0], c[1], pa[g * lda + 4 + t], pb[g * ldb + 4 + t]);
}
// c += A B with B given as rows (B[k][n] at pb[k * ldb + n]).
__device__ __forceinline__ void dmma8_nn(double (&c)[2], const double *pa, int lda, const double *pb, int ldb, int g,
                                         int t) {
  dmma(c[0], c[1], pa[g * lda + t], pb[t * ldb + g]);
  dmma(c[0], c[1], pa[g * lda + 4 + t], pb[(4 + t) * ldb + g]);
}
// c += A^T B with A given as rows of A^T... (A[m][k] = AT[k][m] at pa[k * lda + m]) and B as rows.
__device__ __forceinline__ void dmma8_tnn(double (&c)[2], const double *pa, int lda, const double *pb, int ldb, int g,
                                          int t) {
  dmma(c[0], c[1], pa[t * lda + g], pb[t * ldb + g]);
  dmma(c[0], c[1], pa[(4 + t) * lda + g], pb[(4 + t) * ldb + g]);
}

__device__ __forceinline__ void frag_load(double (&c)[2], const double *p, int ld, int g, int t) {
  const double2 v = *(const double2 *)(p + g * ld + 2 * t);
  c[0] = v.x;
  c[1] = v.y;
}
__device__ __forceinline__ void frag_store(const double (&c)[2], double *p, int ld, int g, int t) {
  *(double2 *)(p + g * ld + 2 * t) = make_double2(c[0], c[1]);
}

// reciprocal to full double precision: hardware approximation + two Newton steps
__device__ __forceinline__ double rcp_full(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  r = fma(r, fma(-d, r, 1.0), r);
  r = fma(r, fma(-d, r, 1.0), r);
  return r;
}

// Leading dimension (doubles) >= n with ld % 16 == 4 (conflict-free fragment loads).
__host__ __device__ constexpr int ld_frag(int n) { return (n + 11) / 16 * 16 + 4; }

__device__ __forceinline__ void cpa8(void *smem, const void *g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)), "l"(g)
               : "memory");
}
__device__ __forceinline__ void cpa16cg(void *smem, const void *g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)), "l"(g)
               : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cpa_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ---------------------------------------------------------------------------------- clusters
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_size() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
// Cluster-wide barrier with release / acquire semantics: every memory access (shared, global)
// made by any thread of the cluster before the barrier is visible to every thread after it.
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

}  // namespace strb200
