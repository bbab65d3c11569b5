// B200 backend — raise a kernel's dynamic shared-memory limit, never lower it.
// Contexts on several host threads launch the same kernels; a thread that
// set a smaller limit while another thread's larger launch is in flight
// would make that launch fail (cudaErrorInvalidValue), so the limit only
// grows, under a lock.
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <mutex>

inline cudaError_t tpo_ensure_smem(const void *kern, size_t smem) {
  static std::mutex mu;
  static std::map<const void *, size_t> limit;
  std::lock_guard<std::mutex> lk(mu);
  size_t &cur = limit[kern];
  if (smem <= cur) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e == cudaSuccess) cur = smem;
  return e;
}
