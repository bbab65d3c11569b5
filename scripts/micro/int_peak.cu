// Microbenchmark: integer issue ceilings of the verifier's arithmetic on
// B200 — IMAD (32-bit multiply-add), IDP4A (4-way u8 dot product) and
// LOP3 — with 16 independent chains per thread, grid = SMs x 8 CTAs x 256
// threads.  Prints ops/s (1 IMAD = 1 op; 1 DP4A = 4 MACs reported
// separately).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o int_peak int_peak.cu
#include <cuda_runtime.h>
#include <cstdio>

constexpr int kIters = 4096;

__global__ void k_imad(unsigned *out, unsigned seed) {
  unsigned a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = seed + threadIdx.x * 16 + i;
  const unsigned m = seed | 1;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = a[i] * m + (unsigned)i;  // IMAD
  }
  unsigned r = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) r ^= a[i];
  if (r == 0x12345u) out[0] = r;
}

__global__ void k_dp4a(unsigned *out, unsigned seed) {
  int a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = int(seed + threadIdx.x * 16 + i);
  const int m = int(seed | 0x01010101);
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = __dp4a(m, a[i] & 0x7f7f7f7f, a[i]);
  }
  unsigned r = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) r ^= unsigned(a[i]);
  if (r == 0x12345u) out[0] = r;
}

template <class K>
double rate(K kern, int ops_per_inner, int sms) {
  unsigned *out;
  cudaMalloc(&out, 4);
  const int grid = sms * 8, block = 256;
  kern<<<grid, block>>>(out, 3);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    kern<<<grid, block>>>(out, 3 + r);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  cudaFree(out);
  const double ops = double(grid) * block * kIters * 16.0 * ops_per_inner;
  return ops / (best * 1e-3);
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double imad = rate(k_imad, 1, sms);
  // dp4a loop: 1 LOP3 (mask) + 1 IDP4A per inner step
  const double dp4a = rate(k_dp4a, 1, sms);
  printf("{\"sms\": %d, \"clock_khz\": %d, \"imad_per_s\": %.4e, \"dp4a_per_s\": %.4e, "
         "\"imad_per_clk_per_sm_at_max\": %.1f}\n",
         sms, clk, imad, dp4a, imad / (double(sms) * clk * 1e3));
  cudaError_t e = cudaGetLastError();
  if (e) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
