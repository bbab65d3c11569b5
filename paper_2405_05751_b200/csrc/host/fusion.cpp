// B200 backend — thread-graph construction; see
// tpo/ir/fusion.hpp.
#include "tpo/ir/fusion.hpp"

#include <algorithm>
#include <map>
#include <numeric>
#include <vector>

#include "tpo/ir/ops.hpp"

namespace tpo::ir {

void construct_thread_groups(BlockGraph &bg) {
  const size_t nops = bg.ops.size(), nt = bg.tensors.size();
  // producer op index and consumer ops of every block tensor
  std::vector<int> prod(nt, -1);
  std::vector<std::vector<int>> cons(nt);
  for (size_t k = 0; k < nops; ++k) {
    for (TensorId t : bg.ops[k].outputs) prod[size_t(t)] = int(k);
    for (TensorId t : bg.ops[k].inputs) {
      auto &c = cons[size_t(t)];
      if (c.empty() || c.back() != int(k)) c.push_back(int(k));
    }
  }
  // phase: post-loop iff Accum output or a descendant (eval_core.hpp:277-294)
  std::vector<char> post_t(nt, 0), post_op(nops, 0);
  for (size_t k = 0; k < nops; ++k) {
    const Op &op = bg.ops[k];
    if (op.type == OpType::Accum) {
      post_t[size_t(op.outputs[0])] = 1;
      continue;
    }
    if (op.type == OpType::InIter || op.type == OpType::OutSaver) continue;
    for (TensorId t : op.inputs)
      if (post_t[size_t(t)]) post_op[k] = 1;
    if (post_op[k])
      for (TensorId t : op.outputs) post_t[size_t(t)] = 1;
  }
  std::vector<int> parent(nops);
  std::iota(parent.begin(), parent.end(), 0);
  auto find = [&](int x) {
    while (parent[size_t(x)] != x) x = parent[size_t(x)] = parent[size_t(parent[size_t(x)])];
    return x;
  };
  for (size_t k = 0; k < nops; ++k) {
    const Op &b = bg.ops[k];
    if (!op_elementwise(b.type)) continue;
    for (TensorId t : b.inputs) {
      const int a = prod[size_t(t)];
      if (a < 0 || !op_elementwise(bg.ops[size_t(a)].type)) continue;
      if (cons[size_t(t)].size() != 1) continue;  // fan-out: not fused past it
      if (post_op[size_t(a)] != post_op[k]) continue;
      parent[size_t(find(int(k)))] = find(a);
    }
  }
  std::map<int, std::vector<int>> groups;
  for (size_t k = 0; k < nops; ++k)
    if (op_elementwise(bg.ops[k].type)) groups[find(int(k))].push_back(bg.ops[k].id);
  bg.thread_groups.clear();
  for (auto &[root, ids] : groups) {
    if (ids.size() < 2) continue;
    std::sort(ids.begin(), ids.end());
    ThreadGroup tg;
    tg.op_ids = ids;
    tg.block_dims = {128, 1, 1};
    tg.forloop = post_op[size_t(root)] ? 1 : int(bg.forloop);
    bg.thread_groups.push_back(std::move(tg));
  }
  std::sort(bg.thread_groups.begin(), bg.thread_groups.end(),
            [](const ThreadGroup &x, const ThreadGroup &y) { return x.op_ids[0] < y.op_ids[0]; });
}

KernelGraph construct_thread_graphs(const KernelGraph &g) {
  KernelGraph out = g;
  for (Op &op : out.ops)
    if (op.type == OpType::GraphDef && op.block) {
      auto bg = std::make_shared<BlockGraph>(*op.block);
      construct_thread_groups(*bg);
      op.block = bg;
    }
  return out;
}

}  // namespace tpo::ir
