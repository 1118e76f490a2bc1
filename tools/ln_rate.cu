// Cost of the in-smem LayerNorm of a 32 x 768 operand tile (dgemm.cuh
// dg_ln_rows) in isolation: 8 warps x 4 rows, clock64 around the call.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2407_04991_b200/csrc \
//        tools/ln_rate.cu -o tools/bin/ln_rate
#include <cstdio>
#include "dgemm.cuh"

using namespace tf;

__global__ void __launch_bounds__(256, 1) lnk(const float* g, const float* b, long long* out, int mode,
                                              const uint8_t* big) {
  __shared__ uint64_t bar;
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  const int bn = 32, H = 768;
  for (int i = threadIdx.x; i < 12 * bn * 128 / 4; i += 256) reinterpret_cast<uint32_t*>(s)[i] = 0x3c003c00u + i;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float4 gv[6], bv[6];
  ln_load_gb<3>(H, g, b, lane, gv, bv);
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (mode >= 2 && threadIdx.x == 0) {
    // 48 KB of bulk loads in flight (from a cold 256 MB buffer) into the upper smem
    mbar_expect_tx(smem_u32(&bar), 49152);
    for (int i = 0; i < 3; ++i)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16384, [%2];"
                   ::"r"(smem_u32(s + 60 * 1024 + i * 16384)), "l"(big + (size_t)blockIdx.x * 65536 + i * 16384),
                   "r"(smem_u32(&bar)) : "memory");
  }
  if (mode == 3 && threadIdx.x == 0)
    for (int i = 0; i < 4; ++i) l2_prefetch_bulk(big + (64u << 20) + i * 32768, 32768);
  __syncthreads();
  long long t0 = clock64();
  if (mode == 0 || mode >= 2) {
    dg_ln_rows<3, 4>(smem_u32(s), bn, warp, 8, bn, H, gv, bv, lane);
  } else {
    for (int r = warp; r < bn; r += 8) dg_ln_rows<3, 1>(smem_u32(s), bn, r, 8, bn, H, gv, bv, lane);
  }
  if (mode >= 2) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[mode] = t1 - t0;
  if (mode >= 2) mbar_wait(smem_u32(&bar), 0);
}

int main() {
  float *g, *b;
  long long* d;
  cudaMalloc(&g, 4096);
  cudaMalloc(&b, 4096);
  cudaMemset(g, 0, 4096);
  cudaMemset(b, 0, 4096);
  cudaMalloc(&d, 64);
  uint8_t* big;
  cudaMalloc(&big, 256u << 20);
  uint8_t* fl;
  cudaMalloc(&fl, 256u << 20);
  cudaFuncSetAttribute(lnk, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
  for (int rep = 0; rep < 3; ++rep)
    for (int mode = 0; mode < 4; ++mode) {
      cudaMemset(fl, rep, 256u << 20);
      lnk<<<1, 256, 120 * 1024>>>(g, b, d, mode, big);
    }
  cudaDeviceSynchronize();
  long long h[4];
  cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
  printf("4-row interleaved: %lld cyc; 1 row at a time: %lld cyc; +fence w/ 48KB bulk in flight: %lld; + L2 prefetch: %lld (%s)\n",
         h[0], h[1], h[2], h[3], cudaGetErrorString(cudaGetLastError()));
  return 0;
}
