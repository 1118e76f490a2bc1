// tcgen05.mma issue-to-completion time for the decode GEMM shapes: n MMAs of
// M x N x 16 (f16 -> f32) issued back to back by one thread, then commit; the
// other warps either spin on the mbarrier or sleep. One CTA, smem operands.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2407_04991_b200/csrc \
//        tools/mma_rate.cu -o tools/bin/mma_rate
#include <cstdio>
#include "common.cuh"

using namespace tf;

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 r;\n\telect.sync r|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(pred));
  return pred != 0;
}

__global__ void __launch_bounds__(128, 1) rate(int M, int N, int n, int spin, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    fence_mbar_init();
  }
  if ((threadIdx.x >> 5) == 0) tmem_alloc(smem_u32(&slot), 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  long long t0 = clock64(), t1 = 0, t2 = 0;
  if (spin == 3 && threadIdx.x < 32) {
    // fully unrolled 48 MMAs (12 k-blocks), descriptors = base + compile-time offsets
    const uint32_t idesc = (1u << 4) | (((uint32_t)N >> 3) << 17) | (((uint32_t)M >> 4) << 24);
    const uint64_t da0 = umma_desc_sw128(smem_u32(s)), db0 = umma_desc_sw128(smem_u32(s + 8 * M * 128));
    const uint32_t astep = (uint32_t)(M * 128) >> 4, bstep = (uint32_t)(N * 128) >> 4;
    if (elect_one()) {
#pragma unroll
      for (int i = 0; i < 48; ++i) {
        const int kb = (i / 4) % 8, k = i % 4;
        tc_mma_f16(tmem, da0 + kb * astep + 2 * k, db0 + kb * bstep + 2 * k, idesc, i ? 1u : 0u);
      }
    }
    __syncwarp();
    t1 = clock64();
    if (threadIdx.x == 0) tc_commit(smem_u32(&bar));
  } else if (spin >= 2 && threadIdx.x < 32) {
    // whole warp runs the loop (warp-uniform control flow), one elected lane issues
    const uint32_t idesc = (1u << 4) | (((uint32_t)N >> 3) << 17) | (((uint32_t)M >> 4) << 24);
    const int abytes = M * 128, bbytes = N * 128;
    const uint32_t a0 = smem_u32(s), b0 = smem_u32(s + 8 * abytes);
    for (int i = 0; i < n; ++i) {
      const int kb = i / 4, k = i % 4;
      const uint64_t da = umma_desc_sw128(a0 + (uint32_t)((kb % 8) * abytes)) + 2 * k;
      const uint64_t db = umma_desc_sw128(b0 + (uint32_t)((kb % 8) * bbytes)) + 2 * k;
      asm volatile(
          "{\n\t.reg .pred p, q;\n\t.reg .b32 r;\n\t"
          "elect.sync r|p, 0xffffffff;\n\t"
          "setp.ne.b32 q, %4, 0;\n\t"
          "@p tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, q;\n\t}" ::"r"(tmem),
          "l"(da), "l"(db), "r"(idesc), "r"(i)
          : "memory");
    }
    t1 = clock64();
    if (threadIdx.x == 0) tc_commit(smem_u32(&bar));
  } else if (spin < 2 && threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | (((uint32_t)N >> 3) << 17) | (((uint32_t)M >> 4) << 24);
    const int abytes = M * 128, bbytes = N * 128;
    for (int i = 0; i < n; ++i) {
      const int kb = i / 4, k = i % 4;
      const uint64_t da = umma_desc_sw128(smem_u32(s + (size_t)(kb % 8) * abytes));
      const uint64_t db = umma_desc_sw128(smem_u32(s + 8 * abytes + (size_t)(kb % 8) * bbytes));
      tc_mma_f16(tmem, da + 2 * k, db + 2 * k, idesc, i ? 1u : 0u);
    }
    t1 = clock64();
    tc_commit(smem_u32(&bar));
  }
  if (spin >= 2) spin = 1;
  if (spin || threadIdx.x == 0)
    mbar_wait(smem_u32(&bar), 0);
  else
    mbar_wait_sleep(smem_u32(&bar), 0);
  if (threadIdx.x == 0) {
    t2 = clock64();
    out[0] = t1 - t0;
    out[1] = t2 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if ((threadIdx.x >> 5) == 0) tmem_dealloc(tmem, 256);
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int M : {64, 128})
    for (int N : {32, 64})
      for (int n : {48})
        for (int spin = 1; spin < 4; ++spin) {
          long long h[2];
          for (int rep = 0; rep < 3; ++rep) {
            rate<<<1, 128, 200 * 1024>>>(M, N, n, spin, d);
            cudaDeviceSynchronize();
          }
          cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
          printf("M=%3d N=%3d n=%3d spin=%d: issue %6lld cyc, done %6lld cyc (%.1f cyc/mma)\n", M, N, n, spin, h[0],
                 h[1], (double)h[1] / n);
        }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
