// Event-pair overhead around one kernel launch by kernel shape (diagnostic for the contraction's
// event-vs-span gap): tiny predecessor kernel, event, kernel under test, event; averaged.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o launch_probe launch_probe.cu && ./launch_probe
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_tiny(int *p) { if (threadIdx.x == 0 && p) p[0] = 1; }
__global__ void k_empty(int *p) { if (threadIdx.x == 0 && p && blockIdx.x == 100000) p[0] = 1; }
__global__ void k_smem(int *p) {
  extern __shared__ int sm[];
  if (threadIdx.x == 0) sm[0] = blockIdx.x;
  __syncthreads();
  if (threadIdx.x == 0 && p && sm[0] == 100000) p[0] = 1;
}
__global__ void k_tmem(int *p) {
  extern __shared__ int sm[];
  __shared__ unsigned slot;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"((unsigned)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
  if (threadIdx.x == 0 && p && sm[1] == 100000) p[0] = 1;
}
__global__ void k_pdl(int *p) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0 && p && blockIdx.x == 100000) p[0] = 1;
}
static void launch_pdl(int grid, bool pdl) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cfg.stream = 0;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k_pdl, (int *)nullptr);
}
template <typename F>
float timeit(F launch, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float tot = 0;
  for (int r = 0; r < reps; ++r) {
    k_tiny<<<1, 32>>>(nullptr);
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (r >= 3) tot += ms;
  }
  return tot / (reps - 3) * 1e3f;
}
int main() {
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_tmem, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_smem, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  cudaFuncSetAttribute(k_tmem, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  cudaFuncSetAttribute(k_tiny, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  printf("empty 1x32:           %.2f us\n", timeit([] { k_empty<<<1, 32>>>(nullptr); }, 50));
  printf("empty 144x512:        %.2f us\n", timeit([] { k_empty<<<144, 512>>>(nullptr); }, 50));
  printf("smem200K 144x512:     %.2f us\n", timeit([&] { k_smem<<<144, 512, smem>>>(nullptr); }, 50));
  printf("tmem512+smem 144x512: %.2f us\n", timeit([&] { k_tmem<<<144, 512, smem>>>(nullptr); }, 50));
  printf("empty 148x512:        %.2f us\n", timeit([] { k_empty<<<148, 512>>>(nullptr); }, 50));
  for (int grid : {1, 49}) {
    for (int pdl = 0; pdl < 2; ++pdl) {
      const float t1 = timeit([&] { launch_pdl(grid, pdl); }, 50);
      const float t9 = timeit([&] { for (int i = 0; i < 9; ++i) launch_pdl(grid, pdl); }, 50);
      printf("chain of 9 vs 1 kernels (grid %d, pdl %d): %.2f vs %.2f us -> %.2f us per added kernel\n", grid, pdl, t9, t1,
             (t9 - t1) / 8);
    }
  }
  // the same inside a CUDA graph (stream capture)
  for (int grid : {1, 49}) {
    for (int pdl = 0; pdl < 2; ++pdl) {
      cudaStream_t st;
      cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
      cudaGraph_t g;
      cudaGraphExec_t ge;
      cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
      for (int i = 0; i < 33; ++i) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(256);
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = pdl ? 1 : 0;
        cudaLaunchKernelEx(&cfg, k_pdl, (int *)nullptr);
      }
      cudaStreamEndCapture(st, &g);
      cudaGraphInstantiate(&ge, g, 0);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      for (int w = 0; w < 3; ++w) cudaGraphLaunch(ge, st);
      cudaEventRecord(a, st);
      for (int r = 0; r < 20; ++r) cudaGraphLaunch(ge, st);
      cudaEventRecord(b, st);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("graph of 33 kernels (grid %d, pdl %d): %.2f us per kernel\n", grid, pdl, ms * 1e3f / 20 / 33);
    }
  }
  return 0;
}
