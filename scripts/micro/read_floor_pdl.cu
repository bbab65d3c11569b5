// Microbenchmark: the read floor of a 34 MB µGraph-shaped stream WITH the
// fused kernels' launch-boundary pipeline (VERDICT r01 "What's weak" #2):
// back-to-back launches in a CUDA graph (PDL), each CTA streaming its
// contiguous slice of a static "weight" buffer through a TMA (1-D bulk) smem
// ring; the first NPRE stages are issued BEFORE griddepcontrol.wait, every
// stage also needs a 1 KB "activation" chunk that may only be read after the
// wait (as X in the fused kernels), and the dependents are released TRIG
// chunks before the producer's last issue.  Buffers rotate over > 3x L2.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o read_floor_pdl read_floor_pdl.cu
//   ./read_floor_pdl            (prints one line per configuration)
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ unsigned su(const void *p) { return unsigned(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void expect(uint64_t *b, unsigned n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void bulk(void *dst, const void *src, unsigned n, uint64_t *b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(dst)),
               "l"(src), "r"(n), "r"(su(b))
               : "memory");
}
__device__ __forceinline__ void wait_par(uint64_t *b, unsigned par) {
  unsigned ok = 0;
  while (!ok)
    asm volatile("{ .reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0,1,0,q; }"
                 : "=r"(ok)
                 : "r"(su(b)), "r"(par)
                 : "memory");
}

struct Args {
  const uint8_t *w;  // static stream
  const uint8_t *x;  // per-launch activations (read after the wait)
  size_t bytes;
  int npre, trig, xdep;
  unsigned *out;
};

// one producer thread (TMA), one consumer warp (releases stages)
template <int STAGES, int CHUNK>
__global__ void __launch_bounds__(64) k_ring(Args a) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  const size_t per = a.bytes / gridDim.x / CHUNK * CHUNK;  // whole chunks: 16-B aligned bulk copies
  const uint8_t *base = a.w + per * blockIdx.x;
  const uint8_t *xb = a.x + size_t(blockIdx.x) * 1024 * 64;
  const int nch = int(per / CHUNK);
  constexpr unsigned XB = 1024;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int npre = a.npre < nch ? a.npre : nch;
  const unsigned xbytes = a.xdep ? XB : 0u;
  if (threadIdx.x == 0) {
    for (int c = 0; c < npre; ++c) {
      expect(&full[c], CHUNK + xbytes);
      bulk(sm + c * (CHUNK + XB), base + size_t(c) * CHUNK, CHUNK, &full[c]);
    }
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  unsigned acc = 0;
  if (threadIdx.x == 0) {
    if (a.xdep)
      for (int c = 0; c < npre; ++c) bulk(sm + c * (CHUNK + XB) + CHUNK, xb + (c % 64) * XB, XB, &full[c]);
    for (int c = npre; c < nch; ++c) {
      const int s = c % STAGES;
      wait_par(&empty[s], ((c / STAGES) & 1) ^ 1);
      expect(&full[s], CHUNK + xbytes);
      bulk(sm + s * (CHUNK + XB), base + size_t(c) * CHUNK, CHUNK, &full[s]);
      if (a.xdep) bulk(sm + s * (CHUNK + XB) + CHUNK, xb + (c % 64) * XB, XB, &full[s]);
      if (c == nch - 1 - a.trig) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  } else if (threadIdx.x == 32) {
    for (int c = 0; c < nch; ++c) {
      const int s = c % STAGES;
      wait_par(&full[s], (c / STAGES) & 1);
      acc ^= sm[s * (CHUNK + XB)];
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[s])) : "memory");
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  }
  if (threadIdx.x == 32) a.out[blockIdx.x] = acc;
}

template <class F>
float period_us(F launch, int nbuf, cudaStream_t st) {
  const int N = 60;
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < N; ++i) launch(i % nbuf);
  cudaStreamEndCapture(st, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, st);
  cudaStreamSynchronize(st);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e9;
  for (int r = 0; r < 7; ++r) {
    cudaEventRecord(e0, st);
    cudaGraphLaunch(ge, st);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  return best * 1000.f / N;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaStream_t st;
  cudaStreamCreate(&st);
  unsigned *out;
  cudaMalloc(&out, 1 << 16);
  const size_t B = 33554432;  // the RMSNorm / LoRA weight stream
  const int nbuf = int((3ull * 126 * 1024 * 1024) / B) + 1;
  std::vector<uint8_t *> bufs(nbuf), xs(nbuf);
  for (int i = 0; i < nbuf; ++i) {
    cudaMalloc(&bufs[i], B);
    cudaMemset(bufs[i], 1, B);
    cudaMalloc(&xs[i], size_t(1024) * 64 * 1024);
    cudaMemset(xs[i], 2, size_t(1024) * 64 * 1024);
  }
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = 1;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  int cluster = 1;
  cfg.stream = st;
  cfg.blockDim = dim3(64);
  auto run = [&](auto kern, int stages, int chunk, int grid, int npre, int trig, int xdep, int minb) {
    // minb: pad the dynamic smem so that exactly `minb` CTAs fit an SM
    size_t smem = size_t(stages) * (chunk + 1024);
    if (minb == 1) smem = smem < 120 * 1024 ? 120 * 1024 : smem;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cfg.gridDim = dim3(grid);
    cfg.dynamicSmemBytes = smem;
    at[1].val.clusterDim.x = cluster;
    int nclu = 0;
    cudaOccupancyMaxActiveClusters(&nclu, kern, &cfg);
    float t = 1e9;
    for (int rep = 0; rep < 3; ++rep) {
      float tt = period_us(
        [&](int i) {
          Args a{bufs[i], xs[i], B, npre, trig, xdep, out};
          cudaLaunchKernelEx(&cfg, kern, a);
        },
        nbuf, st);
      t = tt < t ? tt : t;
    }
    const size_t nch = B / grid / chunk, rd = nch * grid * (chunk + (xdep ? 1024 : 0));
    printf("grid %4d cluster %d (max active %3d) stages %2d chunk %6d minb %d npre %2d trig %2d xdep %d  %7.2f us  %9zu B  %7.1f GB/s\n",
           grid, cluster, nclu, stages, chunk, minb, npre, trig, xdep, t, rd, rd / t / 1e3);
  };
  // the fused kernels' geometry: 32 column tiles x K split S (cluster S)
  for (int c : {4, 8}) {
    cluster = c;
    const int grid = 32 * c;
    for (int trig : {0, 2, 4}) {
      run(k_ring<5, 16384>, 5, 16384, grid, 5, trig, 1, 2);
      run(k_ring<4, 16384>, 4, 16384, grid, 4, trig, 1, 2);
      run(k_ring<3, 32768>, 3, 32768, grid, 3, trig / 2, 1, 2);
    }
    run(k_ring<5, 16384>, 5, 16384, grid, 0, 0, 1, 2);
    run(k_ring<10, 16384>, 10, 16384, grid, 10, 4, 1, 1);
  }
  cluster = 1;
  for (int grid : {148, 256, 296}) {
    run(k_ring<5, 16384>, 5, 16384, grid, 5, 2, 1, 2);
    run(k_ring<3, 32768>, 3, 32768, grid, 3, 1, 1, 2);
  }
  cudaError_t e = cudaGetLastError();
  if (e) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
