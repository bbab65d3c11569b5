// Microbenchmark: legacy warp-level integer MMA (mma.sync m16n8k32 u8 ->
// s32, SASS IMMA.16832) against dp4a on this GPU — dependent-chain latency
// and issue throughput per SM.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
template <int CHAINS>
__global__ void k_imma(const uint32_t *a, uint32_t *o, int iters) {
  uint32_t a0 = a[threadIdx.x], a1 = a[threadIdx.x + 32], a2 = a[threadIdx.x + 64], a3 = a[threadIdx.x + 96];
  uint32_t b0 = a[threadIdx.x + 128], b1 = a[threadIdx.x + 160];
  int c[CHAINS][4] = {};
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int h = 0; h < CHAINS; ++h)
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+r"(c[h][0]), "+r"(c[h][1]), "+r"(c[h][2]), "+r"(c[h][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  int s = 0;
#pragma unroll
  for (int h = 0; h < CHAINS; ++h) s += c[h][0] + c[h][1] + c[h][2] + c[h][3];
  o[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int CHAINS>
__global__ void k_dp4a(const uint32_t *a, uint32_t *o, int iters) {
  uint32_t x = a[threadIdx.x], y = a[threadIdx.x + 32];
  uint32_t c[CHAINS] = {};
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int h = 0; h < CHAINS; ++h) c[h] = __dp4a(x, y + h, c[h]);
  uint32_t s = 0;
#pragma unroll
  for (int h = 0; h < CHAINS; ++h) s += c[h];
  o[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  uint32_t *a, *o;
  cudaMalloc(&a, 4096);
  cudaMemset(a, 1, 4096);
  cudaMalloc(&o, 1 << 24);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
  auto run = [&](const char *name, void (*k)(const uint32_t *, uint32_t *, int), int grid, int block, double ops_per_warp_iter) {
    k<<<grid, block>>>(a, o, iters);
    cudaEventRecord(e0);
    k<<<grid, block>>>(a, o, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double warps = double(grid) * block / 32;
    const double ns_per_iter = ms * 1e6 / iters;
    printf("%-22s grid %4d block %4d: %8.2f ns/iter (per warp chain step)  %10.3f T MAC/s\n", name, grid, block,
           ns_per_iter, warps * iters * ops_per_warp_iter / (ms * 1e-3) / 1e12);
  };
  // latency: one warp, one chain
  run("imma 1 chain", k_imma<1>, 1, 32, 4096);
  run("imma 4 chains", k_imma<4>, 1, 32, 4 * 4096);
  run("dp4a 1 chain", k_dp4a<1>, 1, 32, 32 * 4);
  // throughput: all SMs, 8 warps/SM
  run("imma 4 chains x 8w", k_imma<4>, 148, 256, 4 * 4096);
  run("imma 4 chains x 32w", k_imma<4>, 148, 1024, 4 * 4096);
  run("dp4a 8 chains x 32w", k_dp4a<8>, 148, 1024, 8 * 32 * 4);
  return 0;
}
