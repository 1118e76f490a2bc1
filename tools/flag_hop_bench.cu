// Cost of one dependent hop when the dependency is a release/acquire counter
// instead of a kernel boundary: every CTA of hop k reads one value from every
// CTA of hop k-1 (all-to-all data dependency, like a GEMM whose consumers need
// all producer tiles), then publishes its own value and arrives on hop k's
// counter (st + fence.acq_rel.gpu + red.release.gpu.add).
//   mode 0: one persistent kernel runs all N hops (grid-wide counters)
//   mode 1: N kernels, PDL-launched early, each waits on its predecessor's
//           counter instead of griddepcontrol.wait
//   mode 2: N kernels, griddepcontrol.wait (the current chain's mechanism)
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/flag_hop_bench.cu -o gpurun_out/flag_hop_bench
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void hop_body(int k, const float* vals, float* out_vals, int G, unsigned* cnt, int wait_flag,
                                         unsigned epoch) {
  if (wait_flag && k > 0) {
    if (threadIdx.x == 0) {
      while (ld_acquire(cnt + k - 1) < epoch * (unsigned)G) {
      }
    }
    __syncthreads();
  }
  // all-to-all read of the previous hop's values
  float s = 0.f;
  const float* prev = vals + (size_t)((k + 1) & 1) * 1024;
  for (int i = threadIdx.x; i < G; i += blockDim.x) s += __ldcg(prev + i);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  __shared__ float red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    __stcg(out_vals + (size_t)(k & 1) * 1024 + blockIdx.x, t * 0.5f + 1.f);
    if (wait_flag) red_release(cnt + k, 1u);  // release orders the store above
  }
}

__global__ void persistent(float* vals, int N, unsigned* cnt, unsigned epoch) {
  for (int k = 0; k < N; ++k) hop_body(k, vals, vals, gridDim.x, cnt, 1, epoch);
}

__global__ void one_hop(float* vals, int k, unsigned* cnt, int mode, unsigned epoch) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (mode == 2) asm volatile("griddepcontrol.wait;" ::: "memory");
  hop_body(k, vals, vals, gridDim.x, cnt, mode == 1, epoch);
}

int main() {
  const int N = 64;
  float* vals;
  unsigned* cnt;
  cudaMalloc(&vals, 2 * 1024 * sizeof(float));
  cudaMalloc(&cnt, N * sizeof(unsigned));
  cudaMemset(vals, 0, 2 * 1024 * sizeof(float));
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  int grids[] = {32, 96, 148};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mode = 0; mode < 3; ++mode)
    for (int gi = 0; gi < 3; ++gi) {
      const int G = grids[gi];
      cudaGraph_t g;
      cudaGraphExec_t ge;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
      cudaMemsetAsync(cnt, 0, N * sizeof(unsigned), s);
      if (mode == 0) {
        persistent<<<G, 128, 0, s>>>(vals, N, cnt, 1u);
      } else {
        for (int k = 0; k < N; ++k) {
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3(G);
          cfg.blockDim = dim3(128);
          cfg.stream = s;
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          at[0].val.programmaticStreamSerializationAllowed = 1;
          cfg.attrs = at;
          cfg.numAttrs = 1;
          cudaLaunchKernelEx(&cfg, one_hop, vals, k, cnt, mode, 1u);
        }
      }
      cudaStreamEndCapture(s, &g);
      cudaGraphInstantiate(&ge, g, 0);
      float best = 1e30f;
      for (int rep = 0; rep < 20; ++rep) {
        cudaEventRecord(e0, s);
        cudaGraphLaunch(ge, s);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 2 && ms < best) best = ms;
      }
      cudaGraphExecDestroy(ge);
      cudaGraphDestroy(g);
      printf("mode=%d (%s) grid=%3d  per-hop %.3f us\n", mode,
             mode == 0 ? "persistent, counters" : (mode == 1 ? "PDL launch, counter wait" : "PDL griddepcontrol.wait"),
             G, best * 1e3 / N);
    }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
