// Weight packing on the device: model upload and TINF direct-to-device loading.
//
// The reference stores every projection [in, out] row-major in F32 or F16
// (model.py:190-207, TINF v1 tensor.py:179-232). The decode/prefill GEMMs
// stream f16 W^T [out, pad64(in)] K-major tiles, and the LayerNorm-folded
// decode GEMMs use W' = q16(W * gamma) plus per-feature terms c = sum_k W'[:, k]
// and d = sum_k beta_k W[:, k] (gemm_tc.cuh ln_fold). These kernels build all of
// that from the raw tensors once they are in HBM, so a TINF file goes file ->
// pinned host -> device with no host-side f32 materialisation or transposes.
//
// Bits: f16 rounding is the reference's saturating RNE (f16_sat); the W * gamma
// product of two f16 values is exact in f32; c is a sum of f16 values, exact
// in f64 for any order (<= 2^12 terms of magnitude 2^-24 .. 2^16 span < 53 bits),
// d is accumulated in f64 in a fixed order and rounded once to f32.
#pragma once

#include "common.cuh"

namespace tf {

// src [K, N] row-major (f32 or f16) -> dst [N, ldk] f16; k >= K zero-filled.
// With gamma: dst = q16(q16(src) * gamma[k]) (the LayerNorm-folded copy).
// 32 x 32 tiles through shared memory: coalesced reads along N, writes along K.
template <bool F32SRC>
__global__ void __launch_bounds__(256) pack_kmajor_kernel(const void* __restrict__ src, int K, int N,
                                                          const float* __restrict__ gamma,
                                                          __half* __restrict__ dst, int ldk) {
  __shared__ float tile[32][33];
  const int k0 = blockIdx.y * 32, n0 = blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int k = k0 + ty + 8 * i, n = n0 + tx;
    float v = 0.0f;
    if (k < K && n < N) {
      const size_t idx = (size_t)k * N + n;
      v = F32SRC ? q16(static_cast<const float*>(src)[idx]) : __half2float(static_cast<const __half*>(src)[idx]);
      if (gamma != nullptr) v = q16(__fmul_rn(v, gamma[k]));
    }
    tile[ty + 8 * i][tx] = v;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int n = n0 + ty + 8 * i, k = k0 + tx;
    if (n < N && k < ldk) dst[(size_t)n * ldk + k] = __float2half_rn(tile[tx][ty + 8 * i]);
  }
}

// c[n] = sum_k w_ln[n, k], d[n] = sum_k beta[k] * w[n, k] in f64, one warp per
// feature row: lane-strided partial sums, then a fixed xor tree.
__global__ void __launch_bounds__(256) fold_terms_kernel(const __half* __restrict__ w, const __half* __restrict__ w_ln,
                                                         const float* __restrict__ beta, int K, int N, int ldk,
                                                         float* __restrict__ c, float* __restrict__ d) {
  const int n = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (n >= N) return;
  double sc = 0.0, sd = 0.0;
  for (int k = lane; k < K; k += 32) {
    sc += (double)__half2float(w_ln[(size_t)n * ldk + k]);
    sd += (double)beta[k] * (double)__half2float(w[(size_t)n * ldk + k]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sc += __shfl_xor_sync(0xffffffffu, sc, o);
    sd += __shfl_xor_sync(0xffffffffu, sd, o);
  }
  if (lane == 0) {
    c[n] = (float)sc;
    d[n] = (float)sd;
  }
}

// dst[i] = q16(src[i]), stored as f16 or as f32 (biases, LayerNorm parameters:
// f32 holding the f16-rounded value)
__global__ void __launch_bounds__(256) convert_kernel(const void* __restrict__ src, int src_f32, long long n,
                                                      void* __restrict__ dst, int dst_f32) {
  for (long long i = blockIdx.x * 256ll + threadIdx.x; i < n; i += (long long)gridDim.x * 256) {
    const float v = src_f32 ? q16(static_cast<const float*>(src)[i]) : __half2float(static_cast<const __half*>(src)[i]);
    if (dst_f32)
      static_cast<float*>(dst)[i] = v;
    else
      static_cast<__half*>(dst)[i] = __float2half_rn(v);
  }
}

}  // namespace tf
