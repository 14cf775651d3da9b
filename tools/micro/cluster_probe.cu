// Cluster barrier and DSMEM store latency on this GPU (diagnostic only).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
template <int NC>
__global__ void __cluster_dims__(NC, 1, 1) k_cl(long long *out, int iters) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double buf[64];
  cl.sync();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) cl.sync();
  long long t1 = clock64();
  // remote store + barrier
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x < 32) {
      double *r = cl.map_shared_rank(buf, (cl.block_rank() + 1) % NC);
      r[threadIdx.x] = i;
    }
    cl.sync();
  }
  long long t2 = clock64();
  if (threadIdx.x == 0 && cl.block_rank() == 0) {
    out[0] = (t1 - t0) / iters;
    out[1] = (t2 - t1) / iters;
  }
}
int main() {
  long long *d, h[2];
  cudaMalloc(&d, 16);
  k_cl<2><<<2, 256>>>(d, 1000); cudaDeviceSynchronize(); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("cluster 2: barrier %lld cyc, store+barrier %lld cyc\n", h[0], h[1]);
  k_cl<4><<<4, 256>>>(d, 1000); cudaDeviceSynchronize(); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("cluster 4: barrier %lld cyc, store+barrier %lld cyc\n", h[0], h[1]);
  k_cl<8><<<8, 256>>>(d, 1000); cudaDeviceSynchronize(); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("cluster 8: barrier %lld cyc, store+barrier %lld cyc (%s)\n", h[0], h[1], cudaGetErrorString(cudaGetLastError()));
  return 0;
}
