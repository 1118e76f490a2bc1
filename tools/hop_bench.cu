// Floor of a dependent-kernel chain on this GPU: N kernels captured in one CUDA
// graph, each reading what its predecessor wrote. Variants: plain stream order,
// PDL (griddepcontrol) with early trigger, and grid sizes 1 / 96 / 148 / 296.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/hop_bench.cu -o gpurun_out/hop_bench
#include <cstdio>
#include <cuda_runtime.h>

__global__ void hop(const float* __restrict__ in, float* __restrict__ out, int pdl, int work) {
  if (pdl) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  float v = in[i];
  for (int k = 0; k < work; ++k) v = v * 1.0001f + 0.5f;
  out[i] = v + 1.f;
}

int main() {
  const int N = 87;
  float *a, *b;
  cudaMalloc(&a, 1 << 24);
  cudaMalloc(&b, 1 << 24);
  cudaMemset(a, 0, 1 << 24);
  cudaMemset(b, 0, 1 << 24);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  int grids[] = {1, 96, 148, 296, 592};
  for (int pdl = 0; pdl < 2; ++pdl)
    for (int gi = 0; gi < 5; ++gi)
      for (int work = 0; work <= 2000; work += 2000) {
        cudaGraph_t g;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        for (int k = 0; k < N; ++k) {
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3(grids[gi]);
          cfg.blockDim = dim3(128);
          cfg.stream = s;
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          at[0].val.programmaticStreamSerializationAllowed = 1;
          cfg.attrs = at;
          cfg.numAttrs = pdl ? 1 : 0;
          cudaLaunchKernelEx(&cfg, hop, (const float*)(k & 1 ? b : a), (k & 1 ? a : b), pdl, work);
        }
        cudaStreamEndCapture(s, &g);
        cudaGraphInstantiate(&ge, g, 0);
        for (int w = 0; w < 5; ++w) cudaGraphLaunch(ge, s);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, s);
        const int R = 50;
        for (int r = 0; r < R; ++r) cudaGraphLaunch(ge, s);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("pdl=%d grid=%4d work=%4d  per-hop %.2f us  (chain of %d: %.1f us)\n", pdl, grids[gi], work,
               ms * 1e3 / R / N, N, ms * 1e3 / R);
        cudaGraphExecDestroy(ge);
        cudaGraphDestroy(g);
      }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
