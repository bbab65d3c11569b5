// B200 backend — dimension labels of a computation graph: (tensor, dim)
// pairs unified through its ops (broadcast elementwise, matmul batch / m /
// n / k, full-group Sum), with the contracted labels recorded.  Shared by
// the fusion generator (generator.cpp) and Algorithm 1's enumerator
// (enumerate.cpp), which derive InIter / OutSaver maps from them.
#pragma once

#include <numeric>
#include <set>
#include <string>
#include <vector>

#include "tpo/ir/graph.hpp"

namespace tpo::ir::labels {

inline bool supported(OpType t) {
  switch (t) {
    case OpType::Matmul:
    case OpType::Sum:
    case OpType::EwAdd:
    case OpType::EwMul:
    case OpType::EwDiv:
    case OpType::EwExp:
    case OpType::Sqr:
    case OpType::Sqrt:
    case OpType::SiLU:
      return true;
    default:
      return false;
  }
}

inline bool unary(OpType t) {
  return t == OpType::EwExp || t == OpType::Sqr || t == OpType::Sqrt || t == OpType::SiLU;
}

struct Labels {
  std::vector<int> off, parent;
  std::set<int> contracted;  // roots of contracted labels
  int find(int x) {
    while (parent[size_t(x)] != x) x = parent[size_t(x)] = parent[size_t(parent[size_t(x)])];
    return x;
  }
  void unite(int a, int b) { parent[size_t(find(a))] = find(b); }
};

// (tensor, dim) label roots; -1 for extent-1 dims.  Throws Unsupported.
inline Labels label(const KernelGraph &p) {
  Labels L;
  int n = 0;
  for (const TensorInfo &t : p.tensors) L.off.push_back(n), n += t.shape.rank();
  L.parent.resize(size_t(n));
  std::iota(L.parent.begin(), L.parent.end(), 0);
  auto at = [&](TensorId t, int d) { return L.off[size_t(t)] + d; };
  auto dim = [&](TensorId t, int d) { return p.tensor(t).shape.dims[size_t(d)]; };
  std::vector<std::pair<TensorId, int>> contr;
  for (const Op &op : p.ops) {
    if (!supported(op.type)) throw Error(ErrCode::Unsupported, std::string("generator: op ") + op_name(op.type));
    const TensorId o = op.outputs[0];
    const int R = p.tensor(o).shape.rank();
    if (unary(op.type)) {
      for (int d = 0; d < R; ++d) L.unite(at(op.inputs[0], d), at(o, d));
    } else if (op.type == OpType::Matmul) {
      const TensorId a = op.inputs[0], b = op.inputs[1];
      for (int d = 0; d + 2 < R; ++d) {
        if (dim(a, d) > 1) L.unite(at(a, d), at(o, d));
        if (dim(b, d) > 1) L.unite(at(b, d), at(o, d));
      }
      L.unite(at(a, R - 2), at(o, R - 2));
      L.unite(at(b, R - 1), at(o, R - 1));
      L.unite(at(a, R - 1), at(b, R - 2));
      contr.emplace_back(a, R - 1);
    } else if (op.type == OpType::Sum) {
      const auto &sa = std::get<SumAttrs>(op.attrs);
      const TensorId a = op.inputs[0];
      if (sa.group != dim(a, sa.dim)) throw Error(ErrCode::Unsupported, "generator: partial-group Sum");
      for (int d = 0; d < R; ++d)
        if (d != sa.dim) L.unite(at(a, d), at(o, d));
      contr.emplace_back(a, sa.dim);
    } else {  // broadcast elementwise: right-aligned, equal extents > 1
      for (TensorId t : op.inputs) {
        const int r = p.tensor(t).shape.rank();
        for (int k = 1; k <= r; ++k)
          if (dim(t, r - k) > 1 && dim(t, r - k) == dim(o, R - k)) L.unite(at(t, r - k), at(o, R - k));
      }
    }
  }
  for (auto [t, d] : contr) L.contracted.insert(L.find(at(t, d)));
  return L;
}

}  // namespace tpo::ir::labels
