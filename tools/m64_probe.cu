// Probe of the TMEM accumulator layout of tcgen05.mma cta_group::1 M=64:
// D[r][n] = (r + 1) + 100 n; dumps TMEM lanes 0..127, columns 0..15.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2407_04991_b200/csrc \
//        tools/m64_probe.cu -o tools/bin/m64_probe
#include <cuda_fp16.h>
#include <cstdio>
#include "common.cuh"

using namespace tf;

__device__ void put(uint8_t* base, int r, int k, float v) {
  uint8_t* p = base + (r >> 3) * 1024 + (r & 7) * 128 + (((k >> 3) ^ (r & 7)) * 16) + (k & 7) * 2;
  *reinterpret_cast<__half*>(p) = __float2half(v);
}

__global__ void probe(float* out, int M) {
  __shared__ __align__(1024) uint8_t a[128 * 128];
  __shared__ __align__(1024) uint8_t b[32 * 128];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 128 * 128 / 4; i += 128) reinterpret_cast<uint32_t*>(a)[i] = 0;
  for (int i = threadIdx.x; i < 32 * 128 / 4; i += 128) reinterpret_cast<uint32_t*>(b)[i] = 0;
  __syncthreads();
  if (threadIdx.x < M) {
    put(a, threadIdx.x, 0, threadIdx.x + 1);
    put(a, threadIdx.x, 1, 1.0f);
  }
  if (threadIdx.x < 32) {
    put(b, threadIdx.x, 0, 1.0f);
    put(b, threadIdx.x, 1, 100.0f * threadIdx.x);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    fence_mbar_init();
  }
  if ((threadIdx.x >> 5) == 0) tmem_alloc(smem_u32(&slot), 32);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | ((32u >> 3) << 17) | (((uint32_t)M >> 4) << 24);
    tc_mma_f16(tmem, umma_desc_sw128(smem_u32(a)), umma_desc_sw128(smem_u32(b)), idesc, 0u);
    tc_commit(smem_u32(&bar));
  }
  mbar_wait(smem_u32(&bar), 0);
  tc_fence_after();
  const int warp = threadIdx.x >> 5;
  float v[16];
  tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16), v);
  for (int j = 0; j < 16; ++j) out[threadIdx.x * 16 + j] = v[j];
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 32);
}

int main() {
  float* d;
  cudaMalloc(&d, 128 * 16 * 4);
  float h[128 * 16];
  for (int M : {64, 128}) {
    cudaMemset(d, 0, 128 * 16 * 4);
    probe<<<1, 128>>>(d, M);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("M=%d err=%s\n", M, cudaGetErrorString(e));
    for (int lane = 0; lane < 128; ++lane) {
      printf("lane %3d:", lane);
      for (int j = 0; j < 4; ++j) printf(" %7.0f", h[lane * 16 + j]);
      printf("\n");
    }
  }
  return 0;
}
