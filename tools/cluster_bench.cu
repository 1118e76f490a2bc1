// Cluster-size cost on this GPU: CTAs of one cluster exchange a value with every
// peer over DSMEM and meet at a cluster barrier, R rounds; cluster sizes 2..16.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2407_04991_b200/csrc \
//        tools/cluster_bench.cu -o tools/bin/cluster_bench
#include <cstdio>
#include "common.cuh"

using namespace tf;

__global__ void __launch_bounds__(128, 1) xchg(int rounds, long long* out) {
  __shared__ float red[16][32];
  const uint32_t rank = cluster_ctarank();
  uint32_t nr;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(nr));
  cluster_arrive();
  cluster_wait();
  long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  float acc = 0.f;
  for (int r = 0; r < rounds; ++r) {
    if (threadIdx.x < 32)
      for (uint32_t p = 0; p < nr; ++p)
        asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(dsmem_addr(smem_u32(&red[rank][threadIdx.x]), p)),
                     "f"(acc + r)
                     : "memory");
    cluster_arrive();
    cluster_wait();
    if (threadIdx.x < 32)
      for (uint32_t p = 0; p < nr; ++p) acc += red[p][threadIdx.x];
  }
  long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0 + (acc == 12345.f);
}

template <typename K>
void run(K kern, int csize, int grid, int rounds, long long* d) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = csize;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, rounds, d);
  cudaDeviceSynchronize();
  long long h[16];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("cluster %2d grid %3d rounds %d: %7.2f us per round (CTA0)  %s\n", csize, grid, rounds, h[0] / 1e3 / rounds,
         cudaGetErrorString(e ? e : cudaGetLastError()));
}

int main() {
  long long* d;
  cudaMalloc(&d, 4096);
  cudaFuncSetAttribute(xchg, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int c : {2, 4, 6, 8, 12, 16})
    for (int rounds : {1, 10}) run(xchg, c, c, rounds, d);
  return 0;
}
