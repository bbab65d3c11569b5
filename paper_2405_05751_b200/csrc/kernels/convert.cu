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

// ---------------------------------------------------------------------------
// Precision-policy conversions for the fused kernels (tpo_gpu.h TPO_PREC_*):
// inputs of any caller dtype (TPO_DTYPE_F32 = 0, _BF16 = 1, _F64 = 2) become
// the operand forms the kernels read.
//   planes: hi = bf16(x), lo = bf16(x - hi)  (x = hi + lo to ~2^-16 relative)
//   rows:   [batch][R][C] -> [batch][2P][C] with hi rows r < R at r, lo rows
//           at P + r, zeros elsewhere (the B-operand hi / lo token rows)
//   f32 / bf16: plain conversions (round to nearest even)
namespace {

template <class T>
__device__ __forceinline__ double ld_in(const void *in, size_t i);
template <>
__device__ __forceinline__ double ld_in<float>(const void *in, size_t i) {
  return double(static_cast<const float *>(in)[i]);
}
template <>
__device__ __forceinline__ double ld_in<double>(const void *in, size_t i) {
  return static_cast<const double *>(in)[i];
}
template <>
__device__ __forceinline__ double ld_in<__nv_bfloat16>(const void *in, size_t i) {
  return double(__bfloat162float(static_cast<const __nv_bfloat16 *>(in)[i]));
}

__device__ __forceinline__ void split2(double x, __nv_bfloat16 &hi, __nv_bfloat16 &lo) {
  hi = __float2bfloat16_rn(float(x));
  lo = __float2bfloat16_rn(float(x - double(__bfloat162float(hi))));
}

// 8 elements per thread: 32-64 B loads, one 16-B store per plane.  The
// residual x - hi is exact in the input precision (hi is x to 8 bits).
template <class T>
__global__ void __launch_bounds__(256) k_planes(const void *__restrict__ in, __nv_bfloat16 *__restrict__ hi,
                                                __nv_bfloat16 *__restrict__ lo, size_t n, int vec) {
  const size_t n8 = vec ? n / 8 : 0;
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n8; i += stride) {
    double x[8];
    if constexpr (sizeof(T) == 4) {
      const float4 a = reinterpret_cast<const float4 *>(in)[2 * i], b = reinterpret_cast<const float4 *>(in)[2 * i + 1];
      x[0] = a.x, x[1] = a.y, x[2] = a.z, x[3] = a.w, x[4] = b.x, x[5] = b.y, x[6] = b.z, x[7] = b.w;
    } else if constexpr (sizeof(T) == 8) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const double2 d = reinterpret_cast<const double2 *>(in)[4 * i + j];
        x[2 * j] = d.x, x[2 * j + 1] = d.y;
      }
    } else {
      const uint4 v = reinterpret_cast<const uint4 *>(in)[i];
      const __nv_bfloat16 *b = reinterpret_cast<const __nv_bfloat16 *>(&v);
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = __bfloat162float(b[j]);
    }
    __align__(16) __nv_bfloat16 h[8], l[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) split2(x[j], h[j], l[j]);
    reinterpret_cast<uint4 *>(hi)[i] = *reinterpret_cast<const uint4 *>(h);
    reinterpret_cast<uint4 *>(lo)[i] = *reinterpret_cast<const uint4 *>(l);
  }
  for (size_t i = n8 * 8 + size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    __nv_bfloat16 h, l;
    split2(ld_in<T>(in, i), h, l);
    hi[i] = h;
    lo[i] = l;
  }
}

template <class T>
__global__ void __launch_bounds__(256) k_rows(const void *__restrict__ in, __nv_bfloat16 *__restrict__ out,
                                              size_t batch, size_t R, size_t C, size_t P) {
  const size_t n = batch * 2 * P * C;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    const size_t c = i % C, rr = (i / C) % (2 * P), bt = i / (C * 2 * P);
    const size_t r = rr < P ? rr : rr - P;
    __nv_bfloat16 v = __float2bfloat16_rn(0.f);
    if (r < R) {
      __nv_bfloat16 h, l;
      split2(ld_in<T>(in, (bt * R + r) * C + c), h, l);
      v = rr < P ? h : l;
    }
    out[i] = v;
  }
}

template <class T>
__global__ void __launch_bounds__(256) k_f32(const void *__restrict__ in, float *__restrict__ out, size_t n) {
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    out[i] = float(ld_in<T>(in, i));
}

template <class T>
__global__ void __launch_bounds__(256) k_f64(const void *__restrict__ in, double *__restrict__ out, size_t n) {
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    out[i] = ld_in<T>(in, i);
}

template <class T>
__global__ void __launch_bounds__(256) k_bf16(const void *__restrict__ in, __nv_bfloat16 *__restrict__ out,
                                              size_t n) {
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    out[i] = __float2bfloat16_rn(float(ld_in<T>(in, i)));
}

int grid_for(size_t n, int num_sms) {
  const size_t want = (n + 255) / 256;
  return int(want < size_t(num_sms) * 8 ? (want ? want : 1) : size_t(num_sms) * 8);
}

}  // namespace

#define TPO_DISPATCH(dtype, KERN, ...)                                              \
  switch (dtype) {                                                                  \
    case 0: KERN<float><<<grid, 256, 0, st>>>(__VA_ARGS__); break;                  \
    case 1: KERN<__nv_bfloat16><<<grid, 256, 0, st>>>(__VA_ARGS__); break;          \
    case 2: KERN<double><<<grid, 256, 0, st>>>(__VA_ARGS__); break;                 \
    default: return int(cudaErrorInvalidValue);                                     \
  }

extern "C" int tpo_convert_planes(const void *in, int dtype, void *hi, void *lo, size_t n, int num_sms,
                                  cudaStream_t st) {
  if (!n) return 0;
  // the vector path needs 16-B aligned buffers (else element by element)
  const int vec = ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(hi) |
                    reinterpret_cast<uintptr_t>(lo)) & 15) == 0;
  const int grid = grid_for(vec ? n / 8 + 1 : n, num_sms);
  TPO_DISPATCH(dtype, k_planes, in, static_cast<__nv_bfloat16 *>(hi), static_cast<__nv_bfloat16 *>(lo), n, vec)
  return int(cudaGetLastError());
}

extern "C" int tpo_convert_rows(const void *in, int dtype, void *out, size_t batch, size_t R, size_t C,
                                size_t P, int num_sms, cudaStream_t st) {
  const size_t n = batch * 2 * P * C;
  if (!n) return 0;
  if (R > P) return int(cudaErrorInvalidValue);
  const int grid = grid_for(n, num_sms);
  TPO_DISPATCH(dtype, k_rows, in, static_cast<__nv_bfloat16 *>(out), batch, R, C, P)
  return int(cudaGetLastError());
}

extern "C" int tpo_convert_to_f32(const void *in, int dtype, float *out, size_t n, int num_sms,
                                  cudaStream_t st) {
  if (!n) return 0;
  const int grid = grid_for(n, num_sms);
  TPO_DISPATCH(dtype, k_f32, in, out, n)
  return int(cudaGetLastError());
}

extern "C" int tpo_convert_to_f64(const void *in, int dtype, double *out, size_t n, int num_sms,
                                  cudaStream_t st) {
  if (!n) return 0;
  const int grid = grid_for(n, num_sms);
  TPO_DISPATCH(dtype, k_f64, in, out, n)
  return int(cudaGetLastError());
}

extern "C" int tpo_convert_to_bf16(const void *in, int dtype, void *out, size_t n, int num_sms,
                                   cudaStream_t st) {
  if (!n) return 0;
  const int grid = grid_for(n, num_sms);
  TPO_DISPATCH(dtype, k_bf16, in, static_cast<__nv_bfloat16 *>(out), n)
  return int(cudaGetLastError());
}
#undef TPO_DISPATCH
