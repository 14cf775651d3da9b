// The contraction kernel's per-unit MMA sequence in isolation (diagnostic): 2 M-tiles x 4 k-steps
// x 3 tcgen05.mma (TS, N=112) with the kernel's TMEM addresses, commits per unit; variants.
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

// variant bits: 1 = two accumulators (else one), 2 = alternate A slots, 4 = commit per unit, 8 = wait on own commit each unit
__global__ void k_probe(int units, int variant, long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[6];
  __shared__ uint32_t tslot;
  uint8_t *s = (uint8_t *)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x)
    ((float *)s)[i] = (variant & 512) ? (float)((i * 2654435761u) >> 8) * 1e-7f : 0.f;
  if (threadIdx.x < 32) tc::tmem_alloc(&tslot, 512);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 6; ++i) tc::mbar_init(&bar[i], 1);
    tc::mbar_arrive(&bar[4]);     // phase 0 of bar[4] complete
    tc::fence_barrier_init();
  }
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tb = tslot;
  if (threadIdx.x == 0 && (variant & 512)) {   // random-ish operand data: fill TMEM A region via smem? use smem B random
  }
  if (threadIdx.x == 0) {
    const uint32_t idesc = tc::idesc_tf32(128, 112, 0, 0);
    const uint32_t b0 = tc::smem_u32(s);
    uint32_t ph = 0;
    long long t0 = clock64();
    for (int u = 0; u < units; ++u) {
      const int a = (variant & 2) ? (u & 1) : 0;
      for (int mt = 0; mt < 2; ++mt) {
        const uint32_t d = tb + ((variant & 1) ? (uint32_t)(mt * 128) : 0u);
        const uint32_t ahi = tb + 256 + (uint32_t)((2 * a + mt) * 64);
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const uint64_t bhi = tc::smem_desc_sw128(b0 + ks * 32, 16, 1024);
          const uint64_t blo = tc::smem_desc_sw128(b0 + 112 * 128 + ks * 32, 16, 1024);
          mma_ts(d, ahi + ks * 8, bhi, idesc, 1u);
          mma_ts(d, ahi + ks * 8, blo, idesc, 1u);
          mma_ts(d, ahi + 32 + ks * 8, bhi, idesc, 1u);
        }
      }
      if (variant & 4) { tc::mma_commit(&bar[0]); tc::mma_commit(&bar[1]); }
      if (variant & 8) { tc::mma_commit(&bar[2]); tc::mbar_wait(&bar[2], ph); ph ^= 1; }
      if (variant & 16) tc::mbar_wait(&bar[4], 0);          // already complete
      if (variant & 128) tc::tc_fence_after();              // tcgen05.fence::after_thread_sync
      if (variant & 256) tc::tc_fence_before();             // tcgen05.fence::before_thread_sync
      if (variant & 32) {                                      // test_wait on the completed barrier
        uint32_t ok;
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(tc::smem_u32(&bar[4])) : "memory");
        if (!ok) out[1] = 1;
      }
    }
    tc::mma_commit(&bar[3]);
    tc::mbar_wait(&bar[3], 0);
    if (blockIdx.x == 0) out[0] = clock64() - t0;
    tc::mbar_arrive(&bar[5]);   // release the spinners
  } else if ((variant & 64) && threadIdx.x >= 32) {
    tc::mbar_wait(&bar[5], 0);  // other warps spin on an mbarrier until the MMA thread is done
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (threadIdx.x < 32) tc::tmem_dealloc(tb, 512);
}

int main() {
  long long *d; cudaMalloc(&d, 64);
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int v : {7 + 16, 7 + 16 + 512}) for (int ctas : {1, 148}) {
    printf("%3d CTAs: ", ctas);
    k_probe<<<ctas, 128, 100 * 1024>>>(2000, v, d);
    cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("variant %2d (2acc=%d altA=%d commit=%d waitown=%d trywait-done=%d testwait-done=%d): %.1f cycles per unit (ideal 1344)  err=%s\n", v, v & 1,
           (v >> 1) & 1, (v >> 2) & 1, (v >> 3) & 1, (v >> 4) & 1, (v >> 5) & 1, c / 2000.0, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
