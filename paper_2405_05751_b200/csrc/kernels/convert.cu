// B200 backend — fp32 -> bf16 input conversion for host-buffer evaluation
// (tpo_gpu_eval_mugraph_host with TPO_DTYPE_F32 inputs): round-to-nearest-even,
// 8 elements per thread with 32-byte loads / 16-byte stores, grid sized to
// the SM count.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

__global__ void __launch_bounds__(256) f32_to_bf16(const float *__restrict__ in,
                                                    __nv_bfloat16 *__restrict__ out, size_t n) {
  const size_t n8 = n / 8;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n8;
       i += size_t(gridDim.x) * blockDim.x) {
    const float4 a = reinterpret_cast<const float4 *>(in)[2 * i];
    const float4 b = reinterpret_cast<const float4 *>(in)[2 * i + 1];
    __nv_bfloat162 r[4] = {__floats2bfloat162_rn(a.x, a.y), __floats2bfloat162_rn(a.z, a.w),
                           __floats2bfloat162_rn(b.x, b.y), __floats2bfloat162_rn(b.z, b.w)};
    reinterpret_cast<uint4 *>(out)[i] = *reinterpret_cast<uint4 *>(r);
  }
  for (size_t i = n8 * 8 + size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x)
    out[i] = __float2bfloat16_rn(in[i]);
}

}  // namespace

extern "C" int tpo_convert_f32_bf16(const float *in, void *out, size_t n, int num_sms,
                                    cudaStream_t st) {
  if (!n) return 0;
  const size_t want = (n / 8 + 255) / 256 + 1;
  const int grid = int(want < size_t(num_sms) * 8 ? want : size_t(num_sms) * 8);
  f32_to_bf16<<<grid, 256, 0, st>>>(in, static_cast<__nv_bfloat16 *>(out), n);
  return int(cudaGetLastError());
}

// bf16 -> fp32 (exact), for the generic-VM evaluation of µGraphs without a
// fused kernel.
namespace {
__global__ void __launch_bounds__(256) bf16_to_f32(const __nv_bfloat16 *__restrict__ in,
                                                    float *__restrict__ out, size_t n) {
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    out[i] = __bfloat162float(in[i]);
}
}  // namespace

extern "C" int tpo_convert_bf16_f32(const void *in, float *out, size_t n, int num_sms, cudaStream_t st) {
  if (!n) return 0;
  const size_t want = (n + 255) / 256;
  const int grid = int(want < size_t(num_sms) * 8 ? want : size_t(num_sms) * 8);
  bf16_to_f32<<<grid, 256, 0, st>>>(static_cast<const __nv_bfloat16 *>(in), out, n);
  return int(cudaGetLastError());
}
