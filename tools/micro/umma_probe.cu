// Pure tcgen05.mma.kind::tf32 issue/execute throughput (diagnostic): the MMA thread issues
// `iters` groups of 3 MMAs (M=128, N, K=8) with A from TMEM (TS) or shared memory (SS) and B from
// shared memory, committing every group; reports cycles per group and % of the 2048 MAC/clk
// dense TF32 rate.  Operand contents are zero (timing only).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2307_00719_b200/csrc/tc_ptx.cuh"
using namespace strb200;

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a), "l"(b),
               "r"(idesc), "r"(acc) : "memory");
}

template <bool TS>
__global__ void k_probe(int N, int iters, long long *out, int commit_every) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t tslot;
  uint8_t *s = (uint8_t *)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((float *)s)[i] = 0.f;
  if (threadIdx.x < 32) tc::tmem_alloc(&tslot, 512);
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::mbar_init(&bar2, 1); tc::fence_barrier_init(); }
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tb = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = tc::idesc_tf32(128, N, 0, 0);
    const uint32_t a_s = tc::smem_u32(s), b_s = tc::smem_u32(s + 32768);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const uint64_t bd = tc::smem_desc_sw128(b_s + ks * 32, 16, 1024);
        if (TS) {
          mma_ts(tb, tb + 256 + ks * 8, bd, idesc, 1);
          mma_ts(tb, tb + 256 + ks * 8, bd, idesc, 1);
          mma_ts(tb, tb + 288 + ks * 8, bd, idesc, 1);
        } else {
          const uint64_t ad = tc::smem_desc_sw128(a_s + ks * 32, 16, 1024);
          tc::mma_tf32(tb, ad, bd, idesc, 1);
          tc::mma_tf32(tb, ad, bd, idesc, 1);
          tc::mma_tf32(tb, ad, bd, idesc, 1);
        }
      }
      if (commit_every && (it % commit_every) == 0) { tc::mma_commit(&bar2); tc::mma_commit(&bar2); }
    }
    tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[0] = t1 - t0;
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (threadIdx.x < 32) tc::tmem_dealloc(tb, 512);
}

int main() {
  long long *d; cudaMalloc(&d, 64);
  cudaFuncSetAttribute(k_probe<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaFuncSetAttribute(k_probe<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int iters = 2000;
  for (int ce : {0, 1}) for (int N : {64, 96, 104, 112, 128, 256}) {
    for (int ts = 1; ts >= 0; --ts) {
      printf("commit every %d: ", ce);
      if (ts) k_probe<true><<<1, 128, 100 * 1024>>>(N, iters, d, ce); else k_probe<false><<<1, 128, 100 * 1024>>>(N, iters, d, ce);
      cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
      double per = (double)c / iters;           // 12 MMAs of 128 x N x 8 per iteration
      double macs = 12.0 * 128 * N * 8;
      printf("N=%3d %s: %7.1f cycles per 12 MMAs -> %.0f MAC/clk (%.0f%% of 2048)  err=%s\n", N, ts ? "TS" : "SS", per,
             macs / per, 100.0 * macs / per / 2048, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
