// B200 backend — Definition-1 validity checks.  API mirror of the reference's
// tpo/ir/validate.hpp (proj/core/include/tpo/ir/validate.hpp:27-66).  The GPU
// compile path validates with B200 limits (kB200Limits: 227 KiB of shared
// memory per CTA), SURVEY §8d "Validation limits".
#pragma once

#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "tpo/ir/graph.hpp"

namespace tpo::ir {

struct MemLimits {
  int64_t smem_bytes = 48 * 1024;
  int64_t reg_elems = 512;
  int64_t elem_size = 2;
};

inline constexpr MemLimits kB200Limits{232448, 512, 2};

enum class ViolationKind { OperatorSpec, MemoryCapacity, PathRule };

struct Violation {
  ViolationKind kind;
  std::string detail;
};

struct ValidityReport {
  std::vector<Violation> violations;
  bool valid() const { return violations.empty(); }
};

ValidityReport validate(const KernelGraph &g, const MemLimits &limits = {});
std::map<Scope, int64_t> memory_usage(const KernelGraph &g, const MemLimits &limits = {});
int64_t block_shared_bytes(const BlockGraph &bg, int64_t elem_size);

struct LaxReport {
  bool lax = true;
  std::string offending;
};

LaxReport lax_check(const KernelGraph &g);

// New (the reference's lax_check rejects every GraphDef, validate.cpp:199-205):
// a µGraph-level check that no EwExp consumes a value already downstream of
// an EwExp, across kernel and block levels.  The verifier rejects candidates
// failing it up front (status PoisonedExponent).
LaxReport mugraph_lax_check(const KernelGraph &g);

}  // namespace tpo::ir
