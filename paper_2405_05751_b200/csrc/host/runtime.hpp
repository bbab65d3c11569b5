// B200 backend — host runtime objects behind the C-ABI handles.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../kernels/ff_vm.cuh"
#include "fused.hpp"
#include "lower.hpp"
#include "tpo/ir/graph.hpp"

namespace tpo::gpu {

// Grow-only device buffer.
struct DevBuf {
  void *ptr = nullptr;
  size_t cap = 0;
  void *get(size_t bytes);
  DevBuf() = default;
  DevBuf(const DevBuf &) = delete;
  DevBuf &operator=(const DevBuf &) = delete;
  DevBuf(DevBuf &&o) noexcept : ptr(o.ptr), cap(o.cap) { o.ptr = nullptr, o.cap = 0; }
  ~DevBuf();
};

struct FieldState {
  tpo_ff::FieldConst fc{};
  std::vector<uint16_t> host_tables;  // inv_p, inv_q, sqrt_p, sqrt_q
  DevBuf dev;
};

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 0;
  // keyed by the full (p, q, omega_base) triple
  std::map<std::tuple<uint32_t, uint32_t, uint32_t>, std::unique_ptr<FieldState>> fields;
  DevBuf code, graphs, pool, cand, seeds, verdicts, accept, counter, out, status, inputs, ws;
  DevBuf shared_w, shared_tab, shared_meta;  // same-seed verification batches
  uint64_t last_draws = 0;                     // splitmix64 draws of the last verify call (attempts requested)
  DevBuf vm_in, vm_out;                       // generic-VM evaluation of unfused µGraphs
  // host-buffer fp evaluation (tpo_gpu_eval_mugraph_host): per-input device
  // copies (bf16), fp32 staging for converted inputs, per-output buffers
  std::vector<DevBuf> h_in, h_out;
  std::vector<DevBuf> fused_scratch;  // fused-kernel operand conversions (TPO_PREC_*)
  FieldState &field(uint32_t p, uint32_t q, uint32_t wbase);
};

struct Graph {
  ir::KernelGraph g;
  bool lax = true;
  int64_t madds = 0;
  int64_t in_elems = 0, out_elems = 0;
  mutable int64_t vm_words = -1;  // -2: not computed yet (tpo_gpu_graph_info)
  // The fused-kernel match (fused_kind == 0 when no hand-written kernel
  // matches), computed on first use: verification never needs it, so a
  // search stream of candidates does not pay for it.
  const FusedPlan &fused_plan() const {
    std::call_once(plan_once, [this] {
      const uint64_t st = plan.static_inputs;
      plan = match_fused(g);
      plan.static_inputs = st;
    });
    return plan;
  }
  mutable FusedPlan plan;
  mutable std::once_flag plan_once;
  int precision = 0;  // TPO_PREC_* (tpo_gpu_graph_set_precision)
  // VM lowerings by (region base, 0/1 field pinned-outputs | 2 fp): a handle is
  // immutable, so batches over the same graphs reuse their bytecode
  mutable std::mutex ff_mu;
  mutable std::map<std::pair<uint32_t, int>, std::shared_ptr<const VmProgram>> ff_cache;
  // global-memory fp executor: the instruction launches captured once per
  // (mode, VM arena) as a CUDA graph and replayed
  mutable std::map<std::pair<int, void *>, cudaGraphExec_t> vm_graphs;
  Graph() = default;
  Graph(const Graph &) = delete;
  Graph &operator=(const Graph &) = delete;
  ~Graph() {
    for (auto &kv : vm_graphs) cudaGraphExecDestroy(kv.second);
  }
};

// lower_vm(G.g, 0, region, pin, /*field=*/true), memoised on the handle.
const VmProgram &lowered_ff(const Graph &G, uint32_t region, bool pin);
// lower_vm(G.g, 0, inputs) in floating-point mode, memoised on the handle.
const VmProgram &lowered_fp(const Graph &G);

// Throws tpo::Error on failure.
void check_cuda(cudaError_t e, const char *what);

}  // namespace tpo::gpu
