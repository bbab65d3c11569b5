// B200 backend — lowering of a KernelGraph to block-batched VM bytecode
// (kernels/vm.h) and to the fused-kernel plans of csrc/host/fused.hpp.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../kernels/vm.h"
#include "tpo/ir/graph.hpp"

namespace tpo::gpu {

struct VmProgram {
  std::vector<TpoVmInstr> code;
  TpoVmGraph desc{};                       // code_off is assigned at upload
  std::vector<ir::TensorShape> out_shapes;
  std::vector<ir::TensorShape> in_shapes;
  uint32_t region_words = 0;               // words past region_base (peak)
  uint32_t pinned_words = 0;               // outputs pinned at region_base (pin_outputs)
  bool poisoned = false;                   // an EwExp consumes a q-undefined value
  bool has_silu = false;
  int64_t madds = 0;                       // reference op_madds work (SURVEY §8d unit)
};

// Inputs occupy [input_base, input_base + sum(numel)) in graph-input order
// (the order sample_inputs draws them, ffeval.cpp:29-40); every other tensor
// is placed from region_base upward by a liveness-based planner.  With
// pin_outputs the graph outputs occupy [region_base, region_base +
// pinned_words) and everything above is scratch that is dead once the
// program finishes.  Throws tpo::Error on graphs outside the supported
// fragment.
// `field`: the program runs in Z_p x Z_q, where sums are exact and may be
// reassociated: a φ-accumulated Matmul whose operand views advance by one
// k tile per for-loop iteration is hoisted out of the loop as ONE Matmul
// over the whole K range (not done for floating point, which must keep the
// reference's per-iteration summation order).
VmProgram lower_vm(const ir::KernelGraph &g, uint32_t input_base, uint32_t region_base,
                   bool pin_outputs = false, bool field = false);

int64_t graph_madds(const ir::KernelGraph &g);

// Marks VM_NOSYNC on every instruction whose successor may run in the same
// barrier phase (no read/write conflicts; physical addresses).  Run by
// lower_vm after memory planning.
void mark_phases(std::vector<TpoVmInstr> &code);
int64_t input_elems(const ir::KernelGraph &g);

}  // namespace tpo::gpu
