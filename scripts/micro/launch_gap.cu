// Microbenchmark: back-to-back period of near-empty kernels in a CUDA graph,
// as a function of cluster size, dynamic smem and PDL — the fixed per-launch
// cost the µs-scale fused µGraph kernels pay.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o launch_gap launch_gap.cu
#include <cuda_runtime.h>
#include <cstdio>

__global__ void k_empty(float *out, int spin_ns) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  if (spin_ns) {
    unsigned long long t;
    do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); } while (t - t0 < (unsigned long long)spin_ns);
  }
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (threadIdx.x == 0 && out) out[blockIdx.x] = 1.f;
}

float run(int ctas, int cluster, int smem, int pdl, int spin) {
  cudaFuncSetAttribute(k_empty, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaStream_t st;
  cudaStreamCreate(&st);
  float *out;
  cudaMalloc(&out, 4096 * 4);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(192);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cluster;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 2 : 1;
  const int N = 200;
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < N; ++i) cudaLaunchKernelEx(&cfg, k_empty, out, spin);
  cudaStreamEndCapture(st, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, st);
  cudaStreamSynchronize(st);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0, st);
    cudaGraphLaunch(ge, st);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  cudaError_t e = cudaGetLastError();
  if (e) printf("error %s\n", cudaGetErrorString(e));
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  cudaFree(out);
  cudaStreamDestroy(st);
  return best * 1000.f / N;
}

int main() {
  printf("ctas cluster smem pdl spin_ns  period_us\n");
  int cfgs[][5] = {{128, 1, 0, 0, 0},      {128, 1, 0, 1, 0},      {128, 4, 0, 0, 0},
                   {128, 4, 0, 1, 0},      {128, 1, 200000, 0, 0}, {128, 1, 200000, 1, 0},
                   {128, 4, 200000, 0, 0}, {128, 4, 200000, 1, 0}, {128, 2, 200000, 1, 0},
                   {128, 4, 110000, 1, 0}, {112, 1, 200000, 1, 0}, {148, 1, 200000, 1, 0},
                   {128, 4, 200000, 1, 5000}, {128, 1, 200000, 1, 5000}, {128, 4, 200000, 0, 5000},
                   {128, 4, 110000, 1, 5000}};
  for (auto &c : cfgs)
    printf("%4d %7d %6d %3d %7d  %8.3f\n", c[0], c[1], c[2], c[3], c[4], run(c[0], c[1], c[2], c[3], c[4]));
  return 0;
}
