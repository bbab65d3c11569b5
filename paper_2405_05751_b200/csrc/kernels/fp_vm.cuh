// B200 backend — launch contract of the floating-point µGraph VM (fp_vm.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "vm.h"

namespace tpo_fp {

constexpr int kThreads = 256;

struct EvalArgs {
  const TpoVmInstr *code;        // the graph's bytecode (device)
  uint32_t code_len, code_bytes; // instructions; smem bytes reserved for them
  TpoVmGraph graph;              // output placement
  uint32_t n_in;                 // input elements (graph-input order, concatenated)
  const void *inputs;            // device, T[n_in]
  void *out;                     // device, T[sum of output sizes]
};

struct StabilityArgs {
  const TpoVmInstr *code;        // batch bytecode
  const TpoVmGraph *graphs;      // graphs[0] = program
  uint32_t code_bytes;           // smem bytes for program + largest candidate code (0: read in place)
  const uint32_t *cand_graph;    // graph index per candidate
  const uint64_t *seeds;         // per-candidate seed (null: `seed` for all)
  uint64_t seed, n;
  uint32_t n_in;
  int trials;
  double tol, scale;
  unsigned long long *counter;   // work queue head
  int8_t *ok;                    // per candidate: 1 pass, 0 fail, -1 error
};

}  // namespace tpo_fp

extern "C" int tpo_fp_launch_eval(const tpo_fp::EvalArgs *a, int f32, size_t smem, cudaStream_t st);
extern "C" int tpo_fp_launch_stability(const tpo_fp::StabilityArgs *a, int grid, size_t smem,
                                       cudaStream_t st);
extern "C" int tpo_fp_stability_occupancy(size_t smem);
extern "C" int tpo_fp_launch_instr(void *W, int f32, const TpoVmInstr *I, uint32_t it, int num_sms,
                                   cudaStream_t st);
extern "C" int tpo_fp_launch_normals(double *W, uint64_t seed, int trial, uint64_t n, double scale,
                                     int num_sms, cudaStream_t st);
extern "C" int tpo_fp_launch_stab_compare(const double *r, const double *o, uint64_t n, double tol, int *fail,
                                          int num_sms, cudaStream_t st);
