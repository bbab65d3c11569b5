// B200 backend — Algorithm 1's op-by-op µGraph enumeration; see
// tpo/ir/enumerate.hpp.
#include "tpo/ir/enumerate.hpp"

#include <algorithm>
#include <array>
#include <atomic>
#include <map>
#include <mutex>
#include <set>
#include <thread>

#include "labels.hpp"
#include "tpo/ir/absexpr.hpp"
#include "tpo/ir/shape_infer.hpp"

namespace tpo::ir {

namespace {

using absx::Id;
using absx::Pool;

// ------------------------------------------------ abstract expressions (Table 2)

Id op_expr(Pool &P, OpType t, const OpAttrs &at, const std::vector<Id> &in, const std::vector<TensorShape> &sh) {
  switch (t) {
    case OpType::Matmul:
      return P.sum(uint64_t(sh[0].dims.back()), P.mul(in[0], in[1]));
    case OpType::ConcatMatmul:  // W·Y + X·Z
      return P.add(P.sum(uint64_t(sh[0].dims.back()), P.mul(in[0], in[2])),
                   P.sum(uint64_t(sh[1].dims.back()), P.mul(in[1], in[3])));
    case OpType::Sum:
      return P.sum(uint64_t(std::get<SumAttrs>(at).group), in[0]);
    case OpType::EwAdd: return P.add(in[0], in[1]);
    case OpType::EwMul: return P.mul(in[0], in[1]);
    case OpType::EwDiv: return P.div(in[0], in[1]);
    case OpType::EwExp: return P.exp(in[0]);
    case OpType::Sqr: return P.mul(in[0], in[0]);
    case OpType::Sqrt: return P.sqrt(in[0]);
    case OpType::SiLU: return P.silu(in[0]);
    case OpType::Repeat:
    case OpType::Reshape:
      return in[0];
    default:
      throw Error(ErrCode::Unsupported, std::string("abstract expression of ") + op_name(t));
  }
}

// Expressions of every kernel tensor of `g` (GraphDefs inlined, PAPER.md
// §4.3): InIter / OutSaver pass through, φ-Accum sums over the for-loop.
std::vector<Id> graph_exprs(Pool &P, const KernelGraph &g) {
  std::vector<Id> e(g.tensors.size(), 0);
  for (size_t i = 0; i < g.inputs.size(); ++i) e[size_t(g.inputs[i])] = P.var(uint32_t(i));
  for (const Op &op : g.ops) {
    if (op.type != OpType::GraphDef) {
      std::vector<Id> in;
      std::vector<TensorShape> sh;
      for (TensorId t : op.inputs) in.push_back(e[size_t(t)]), sh.push_back(g.tensor(t).shape);
      e[size_t(op.outputs[0])] = op_expr(P, op.type, op.attrs, in, sh);
      continue;
    }
    const BlockGraph &bg = *op.block;
    std::vector<Id> be(bg.tensors.size(), 0);
    size_t saver = 0;
    for (const Op &b : bg.ops) {
      if (b.type == OpType::InIter) {
        be[size_t(b.outputs[0])] = e[size_t(op.inputs[size_t(std::get<InIterAttrs>(b.attrs).operand)])];
      } else if (b.type == OpType::OutSaver) {
        if (saver < op.outputs.size()) e[size_t(op.outputs[saver])] = be[size_t(b.inputs[0])];
        ++saver;
      } else if (b.type == OpType::Accum) {
        const bool phi = std::get<AccumAttrs>(b.attrs).fmap.targets[0] == kReplica;
        be[size_t(b.outputs[0])] = phi ? P.sum(uint64_t(bg.forloop), be[size_t(b.inputs[0])]) : be[size_t(b.inputs[0])];
      } else {
        std::vector<Id> in;
        std::vector<TensorShape> sh;
        for (TensorId t : b.inputs) in.push_back(be[size_t(t)]), sh.push_back(bg.tensor(t).shape);
        be[size_t(b.outputs[0])] = op_expr(P, b.type, b.attrs, in, sh);
      }
    }
  }
  return e;
}

// Output shape of a block-level op the enumerator generates, written into
// `out` without allocating (capacity reused): 1 = shape, 0 = no shape, -1 =
// not covered (use infer_output_shape).  The same rules as
// infer_output_shape at Level::Block (ir_core.cpp: contract, broadcast_shapes,
// Sum, elementwise, Accum) for these ops — inputs are inferred shapes, so
// valid.
int block_shape(OpType t, const OpAttrs &at, const std::vector<TensorShape> &in, TensorShape &out) {
  auto contract = [](const TensorShape &a, const TensorShape &b) {
    const int r = a.rank();
    if (r < 2 || b.rank() != r) return false;
    for (int i = 0; i + 2 < r; ++i)
      if (a.dims[size_t(i)] != b.dims[size_t(i)]) return false;
    return a.dims[size_t(r - 1)] == b.dims[size_t(r - 2)];
  };
  auto set_contract = [&](const TensorShape &a, const TensorShape &b) {
    out.dims.assign(a.dims.begin(), a.dims.end());
    out.dims.back() = b.dims.back();
  };
  switch (t) {
    case OpType::Matmul:
      if (in.size() != 2 || !contract(in[0], in[1])) return 0;
      set_contract(in[0], in[1]);
      return 1;
    case OpType::ConcatMatmul: {
      if (in.size() != 4 || !contract(in[0], in[2]) || !contract(in[1], in[3])) return 0;
      // both products' shapes (a's dims with b's last) must agree
      const TensorShape &a = in[0], &c = in[1];
      if (a.rank() != c.rank() || in[2].dims.back() != in[3].dims.back()) return 0;
      for (int i = 0; i + 1 < a.rank(); ++i)
        if (a.dims[size_t(i)] != c.dims[size_t(i)]) return 0;
      set_contract(in[0], in[2]);
      return 1;
    }
    case OpType::Sum: {
      if (in.size() != 1) return 0;
      const auto &a = std::get<SumAttrs>(at);
      if (a.dim < 0 || a.dim >= in[0].rank() || a.group < 1 || in[0].dims[size_t(a.dim)] % a.group) return 0;
      out.dims.assign(in[0].dims.begin(), in[0].dims.end());
      out.dims[size_t(a.dim)] /= a.group;
      return 1;
    }
    case OpType::EwAdd:
    case OpType::EwMul:
    case OpType::EwDiv: {
      if (in.size() != 2) return 0;
      const TensorShape &a = in[0], &b = in[1];
      const int r = std::max(a.rank(), b.rank());
      out.dims.resize(size_t(r));
      for (int i = 0; i < r; ++i) {
        const int ia = i - (r - a.rank()), ib = i - (r - b.rank());
        const int64_t x = ia >= 0 ? a.dims[size_t(ia)] : 1, y = ib >= 0 ? b.dims[size_t(ib)] : 1;
        if (x != y && x != 1 && y != 1) return 0;
        out.dims[size_t(i)] = x > y ? x : y;
      }
      return 1;
    }
    case OpType::EwExp:
    case OpType::Sqr:
    case OpType::Sqrt:
    case OpType::SiLU:
      if (in.size() != 1) return 0;
      out.dims.assign(in[0].dims.begin(), in[0].dims.end());
      return 1;
    case OpType::Accum: {
      if (in.size() != 1) return 0;
      const auto &a = std::get<AccumAttrs>(at);
      if (a.fmap.axes() != 1) return 0;
      const int d = a.fmap.targets[0];
      if (d != kReplica && (d < 0 || d >= in[0].rank())) return 0;
      out.dims.assign(in[0].dims.begin(), in[0].dims.end());
      return 1;
    }
    default:
      return -1;
  }
}

// ------------------------------------------------------------ search jobs

// A kernel-level prefix: pre-defined ops (in rank order) over the program's
// inputs, then the GraphDef's operands and partition.
struct KOp {
  OpType type;
  OpAttrs attrs;
  std::vector<int> in;  // kernel tensor indices (inputs first, then prefix outputs)
};

struct Job {
  std::vector<KOp> kops;             // pre-defined kernel ops
  std::vector<TensorShape> kshape;   // shapes of every kernel tensor of the prefix
  std::vector<int> operands;         // GraphDef operands (kernel tensor indices)
  std::vector<DimMap> imap, fmap;    // per operand
  std::vector<int> ldim;             // per operand: the dim sliced by the loop (-1 none)
  std::vector<std::vector<int>> dlab;  // per operand: the label of every dim (-1: extent 1)
  std::set<int> mm_labels, sum_labels;  // labels the program contracts by Matmul / by Sum
  int64_t gx = 1, fl = 1;
  int out_dim = 0;                   // output dim assembled over grid x
};

// ------------------------------------------------------------ block search

struct BT {  // block tensor of a prefix
  TensorShape shape;
  Id e = 0;
  uint8_t acc = 1;   // bit0: an InIter path with no Accum reaches it; bit1: one Accum
  int8_t ldim = -1;  // dim sliced by the for-loop (concatenating Accum)
  bool partial = false;  // holds a partial sum over a loop-sliced dim (what a φ-Accum completes)
  std::array<int, 4> lab{-1, -1, -1, -1};  // program label of every dim (-1: extent 1)
  int users = 0;
};

struct BOp {
  OpType type;
  OpAttrs attrs;
  std::array<int, 4> in{-1, -1, -1, -1};
  int nin = 0;
};

using Rank = std::array<int, 6>;  // (max input, inputs..., type): canonical form (see below)

class BlockSearch {
 public:
  BlockSearch(const KernelGraph &prog, const Job &job, const EnumConfig &cfg, uint64_t budget, EnumStats &st,
              std::vector<KernelGraph> &out)
      : prog_(prog), job_(job), cfg_(cfg), st_(st), out_(out), budget_local_(budget) {}

  void run() {
    // kernel expressions: program inputs, then the prefix ops
    std::vector<Id> ke;
    for (size_t i = 0; i < prog_.inputs.size(); ++i) ke.push_back(P_.var(uint32_t(i)));
    for (const KOp &k : job_.kops) {
      std::vector<Id> in;
      std::vector<TensorShape> sh;
      for (int t : k.in) in.push_back(ke[size_t(t)]), sh.push_back(job_.kshape[size_t(t)]);
      ke.push_back(op_expr(P_, k.type, k.attrs, in, sh));
    }
    eo_ = graph_exprs(P_, prog_)[size_t(prog_.outputs[0])];
    out_shape_ = prog_.tensor(prog_.outputs[0]).shape;
    // InIters: the partition's tiles
    for (size_t i = 0; i < job_.operands.size(); ++i) {
      const TensorShape &ks = job_.kshape[size_t(job_.operands[i])];
      ShapeResult a = partition_shape(ks, job_.imap[i], {job_.gx});
      if (a) a = partition_shape(*a.shape, job_.fmap[i], {job_.fl});
      if (!a) return;  // this operand does not tile under the partition
      BT t;
      t.shape = *a.shape;
      t.e = ke[size_t(job_.operands[i])];
      t.acc = 1;
      t.ldim = int8_t(job_.ldim[i]);
      for (int d = 0; d < t.shape.rank() && d < 4; ++d) t.lab[size_t(d)] = t.shape.dims[size_t(d)] > 1 ? job_.dlab[i][size_t(d)] : -1;
      bytes_ += t.shape.elem_count() * cfg_.limits.elem_size;
      T_.push_back(t);
    }
    if (bytes_ > cfg_.limits.smem_bytes) return;
    n_iniers_ = int(T_.size());
    contraction_.assign(T_.size(), 0);
    unconsumed_ = n_iniers_;
    last_.fill(-2);
    // additions are useful only if some term of the program's expression is
    // a sum of several monomials (else add(x, y) is never a subexpression)
    adds_ = has_sum(eo_);
    max_dec_ = cfg_.concat_matmul && adds_ ? 3 : 1;
    dfs();
  }

 private:
  // the prefix budget is split evenly over the partitions, so the result
  // does not depend on thread scheduling
  bool exhausted() {
    if (st_.prefixes >= budget_local_) {
      st_.budget_exhausted = true;
      return true;
    }
    return false;
  }

  bool has_sum(Id e) {
    const absx::Poly &p = P_.poly(e);
    if (p.monos.size() > 1) return true;
    for (const absx::Mono &m : p.monos)
      for (Id a : m.atoms)
        if (P_.atom_of(a).kind != absx::AtomKind::Var && has_sum(P_.atom_of(a).arg)) return true;
    return false;
  }

  static Rank rank_of(const BOp &o) {
    Rank r;
    r.fill(-1);
    int mx = -1;
    for (int i = 0; i < o.nin; ++i) mx = std::max(mx, o.in[size_t(i)]);
    r[0] = mx;
    for (int i = 0; i < o.nin; ++i) r[size_t(1 + i)] = o.in[size_t(i)];
    r[5] = int(o.type);
    return r;
  }

  void dfs() {
    if (exhausted()) return;
    complete();
    const int used = int(ops_.size());
    if (used >= cfg_.max_block_ops) return;
    // every tensor must end up consumed: each op consumes at most
    // (arity - 1) more than it creates
    if (unconsumed_ - 1 > (cfg_.max_block_ops - used) * max_dec_) return;
    const int n = int(T_.size());
    // canonical form: ranks (max input, inputs, type) strictly increase; an
    // op's max input is >= the previous op's (greedy min-rank order of any
    // µGraph is increasing, so every block graph has one canonical order)
    const int lo = std::max(0, last_[0]);
    // the new op's max input m is >= the previous op's (rank order): only
    // operand tuples whose largest index is m in [lo, n) are generated
    for (int m = lo; m < n; ++m) {
      // (copies: construct() grows T_)
      const TensorShape shm = T_[size_t(m)].shape;
      const int ldm = T_[size_t(m)].ldim;
      for (OpType t : {OpType::EwExp, OpType::Sqr, OpType::Sqrt, OpType::SiLU}) try1(t, NoAttrs{}, m);
      for (int d = 0; d < shm.rank(); ++d)
        if (shm.dims[size_t(d)] > 1) try1(OpType::Sum, SumAttrs{d, shm.dims[size_t(d)]}, m);
      try1(OpType::Accum, AccumAttrs{DimMap(std::vector<int>{kReplica})}, m);
      if (ldm >= 0) try1(OpType::Accum, AccumAttrs{DimMap(std::vector<int>{ldm})}, m);
      for (int o = 0; o <= m; ++o) {
        // commutative ops: (o, m) only
        if (adds_) try2(OpType::EwAdd, o, m);
        try2(OpType::EwMul, o, m);
        try2(OpType::EwDiv, o, m);
        try2(OpType::Matmul, o, m);
        if (o < m) {
          try2(OpType::EwDiv, m, o);
          try2(OpType::Matmul, m, o);
        }
      }
    }
    if (cfg_.concat_matmul && adds_) {
      // products W·Y whose matmul alone would pass the shape / label checks
      std::vector<std::pair<int, int>> prods;
      for (int w = 0; w < n; ++w)
        for (int y = 0; y < n; ++y) {
          const BT &a = T_[size_t(w)], &b = T_[size_t(y)];
          const int R = a.shape.rank();
          if (R < 2 || b.shape.rank() != R || a.shape.dims[size_t(R - 1)] != b.shape.dims[size_t(R - 2)]) continue;
          const int ka = a.lab[size_t(R - 1)];
          if (ka != b.lab[size_t(R - 2)] || (ka >= 0 && !job_.mm_labels.count(ka))) continue;
          prods.push_back({w, y});
        }
      for (size_t i = 0; i < prods.size(); ++i)
        for (size_t j = i + 1; j < prods.size(); ++j) {  // W·Y + X·Z = X·Z + W·Y: ordered pairs
          const auto [w, y] = prods[i];
          const auto [x, z] = prods[j];
          if (std::max(std::max(w, x), std::max(y, z)) < lo) continue;
          BOp o;
          o.type = OpType::ConcatMatmul;
          o.in = {w, x, y, z};
          o.nin = 4;
          construct(o);
        }
    }
  }

  void try1(OpType t, OpAttrs at, int a) {
    BOp o;
    o.type = t;
    o.attrs = std::move(at);
    o.in[0] = a;
    o.nin = 1;
    construct(o);
  }
  void try2(OpType t, int a, int b) {
    BOp o;
    o.type = t;
    o.in[0] = a;
    o.in[1] = b;
    o.nin = 2;
    construct(o);
  }

  // ConstructOp (Alg. 1): rank, shape, accumulation rule, expression,
  // duplicate value, memory; then recurse
  void construct(const BOp &o) {
    const Rank r = rank_of(o);
    if (!(r > last_)) return;
    // scratch tensor, reused across attempts (copied into T_ on success;
    // nothing reads it after the recursion)
    BT &nt = nt_;
    nt.e = 0, nt.acc = 1, nt.ldim = -1, nt.partial = false, nt.users = 0;
    nt.lab.fill(-1);
    uint8_t acc = 0;
    for (int i = 0; i < o.nin; ++i) acc |= T_[size_t(o.in[size_t(i)])].acc;
    if (o.type == OpType::Accum) {
      const bool phi = std::get<AccumAttrs>(o.attrs).fmap.targets[0] == kReplica;
      // only loop values accumulate; a φ-Accum completes a partial sum over
      // the loop (with a one-iteration loop: any contraction result)
      const BT &x = T_[size_t(o.in[0])];
      if (acc != 1 || (phi && !(job_.fl > 1 ? x.partial : contraction_[size_t(o.in[0])]))) {
        ++st_.pruned_structure;
        return;
      }
      nt.acc = 2;
    } else {
      if (acc == 3) {  // a loop value meets an accumulated one: a path without an Accum reaches the output
        ++st_.pruned_structure;
        return;
      }
      nt.acc = acc;
    }
    // per-arity scratch reused across attempts (element assignment keeps
    // the dims' capacity: no allocation per attempt)
    std::vector<TensorShape> &sh = shv_[size_t(o.nin)];
    if (sh.size() != size_t(o.nin)) sh.resize(size_t(o.nin));
    for (int i = 0; i < o.nin; ++i) sh[size_t(i)] = T_[size_t(o.in[size_t(i)])].shape;
    const int fs = block_shape(o.type, o.attrs, sh, nt.shape);
    if (fs == 0) {
      ++st_.pruned_shape;
      return;
    }
    if (fs < 0) {  // an op block_shape does not cover: the generic inference
      ShapeResult s = infer_output_shape(o.type, o.attrs, sh, Level::Block);
      if (!s) {
        ++st_.pruned_shape;
        return;
      }
      nt.shape = *s.shape;
    }
    const BT &a0 = T_[size_t(o.in[0])];
    // dimension labels: operands must agree on what their aligned dims mean
    // (a shape that matches by coincidence is not a candidate), reductions
    // only over labels the program reduces the same way
    if (!labels_of(o, nt)) {
      ++st_.pruned_shape;
      return;
    }
    if (o.type == OpType::Accum) {
      const int d = std::get<AccumAttrs>(o.attrs).fmap.targets[0];
      if (d != kReplica) nt.shape.dims[size_t(d)] *= job_.fl;
      nt.ldim = -1;
    } else if (o.type == OpType::Matmul) {
      const int R = nt.shape.rank();
      const BT &b0 = T_[size_t(o.in[1])];
      nt.ldim = a0.ldim == R - 2 ? int8_t(R - 2) : b0.ldim == R - 1 ? int8_t(R - 1) : int8_t(-1);
    } else if (o.type == OpType::Sum) {
      nt.ldim = a0.ldim == std::get<SumAttrs>(o.attrs).dim ? int8_t(-1) : a0.ldim;
    } else if (o.type == OpType::ConcatMatmul) {
      nt.ldim = -1;
    } else {
      nt.ldim = -1;
      for (int i = 0; i < o.nin; ++i) {
        const BT &x = T_[size_t(o.in[size_t(i)])];
        if (x.shape == nt.shape && x.ldim >= 0) nt.ldim = x.ldim;
      }
    }
    if (o.type == OpType::Matmul) {
      const int R = nt.shape.rank();
      nt.partial = (a0.ldim == R - 1 && T_[size_t(o.in[1])].ldim == R - 2) || a0.partial || T_[size_t(o.in[1])].partial;
    } else if (o.type == OpType::Sum) {
      nt.partial = a0.partial || a0.ldim == std::get<SumAttrs>(o.attrs).dim;
    } else if (o.type == OpType::ConcatMatmul) {
      nt.partial = true;
      for (int i = 0; i < 4; ++i) nt.partial = nt.partial && T_[size_t(o.in[size_t(i)])].ldim >= 0;
    } else if (o.type != OpType::Accum) {
      for (int i = 0; i < o.nin; ++i) nt.partial = nt.partial || T_[size_t(o.in[size_t(i)])].partial;
    }
    // the abstract expression (Table 2) and the expr check
    std::vector<Id> &ie = iev_[size_t(o.nin)];
    ie.resize(size_t(o.nin));
    for (int i = 0; i < o.nin; ++i) ie[size_t(i)] = T_[size_t(o.in[size_t(i)])].e;
    if (o.type == OpType::Accum) {
      nt.e = std::get<AccumAttrs>(o.attrs).fmap.targets[0] == kReplica ? P_.sum(uint64_t(job_.fl), ie[0]) : ie[0];
    } else {
      nt.e = op_expr(P_, o.type, o.attrs, ie, sh);
    }
    // subexpression-of-the-program test, memoised densely by expression id
    if (sub_eo_.size() <= nt.e) sub_eo_.resize(size_t(nt.e) + 1024, -1);
    int8_t &se = sub_eo_[nt.e];
    if (se < 0) se = P_.subexpr(nt.e, eo_) ? 1 : 0;
    if (!se) {
      ++st_.pruned_expr;
      return;
    }
    // a value the prefix already holds (same tile, expression and phase)
    for (const BT &x : T_)
      if (x.e == nt.e && x.acc == nt.acc && x.shape == nt.shape) {
        ++st_.pruned_structure;
        return;
      }
    const int64_t b = nt.shape.elem_count() * cfg_.limits.elem_size;
    if (bytes_ + b > cfg_.limits.smem_bytes) {
      ++st_.pruned_memory;
      return;
    }
    // push
    ++st_.prefixes;
    const Rank saved = last_;
    int freed = 0;
    for (int i = 0; i < o.nin; ++i) {
      BT &x = T_[size_t(o.in[size_t(i)])];
      if (x.users++ == 0) ++freed;
    }
    T_.push_back(nt);
    contraction_.push_back(o.type == OpType::Matmul || o.type == OpType::Sum || o.type == OpType::ConcatMatmul);
    ops_.push_back(o);
    bytes_ += b;
    unconsumed_ += 1 - freed;
    last_ = r;
    dfs();
    last_ = saved;
    unconsumed_ -= 1 - freed;
    bytes_ -= b;
    ops_.pop_back();
    contraction_.pop_back();
    T_.pop_back();
    for (int i = 0; i < o.nin; ++i) --T_[size_t(o.in[size_t(i)])].users;
  }

  // Labels of the new tensor's dims; false when operands disagree.
  bool labels_of(const BOp &o, BT &nt) const {
    const int R = nt.shape.rank();
    auto lab = [&](int i, int d) { return T_[size_t(o.in[size_t(i)])].lab[size_t(d)]; };
    auto rk = [&](int i) { return T_[size_t(o.in[size_t(i)])].shape.rank(); };
    nt.lab.fill(-1);
    if (R > 4) return false;
    switch (o.type) {
      case OpType::Matmul:
      case OpType::ConcatMatmul: {
        // pairs (A, B): (0, 1) for Matmul; (0, 2) and (1, 3) for ConcatMatmul
        const int np = o.type == OpType::Matmul ? 1 : 2;
        for (int p = 0; p < np; ++p) {
          const int A = o.type == OpType::Matmul ? 0 : p, B = o.type == OpType::Matmul ? 1 : p + 2;
          const int ka = lab(A, rk(A) - 1), kb = lab(B, rk(B) - 2);
          if (ka != kb || (ka >= 0 && !job_.mm_labels.count(ka))) return false;
          const int m = lab(A, R - 2), n = lab(B, R - 1);
          if ((nt.lab[size_t(R - 2)] >= 0 && m >= 0 && nt.lab[size_t(R - 2)] != m) ||
              (nt.lab[size_t(R - 1)] >= 0 && n >= 0 && nt.lab[size_t(R - 1)] != n))
            return false;
          if (m >= 0) nt.lab[size_t(R - 2)] = m;
          if (n >= 0) nt.lab[size_t(R - 1)] = n;
          for (int d = 0; d + 2 < R; ++d) {
            const int x = std::max(lab(A, d), lab(B, d));
            if (lab(A, d) >= 0 && lab(B, d) >= 0 && lab(A, d) != lab(B, d)) return false;
            nt.lab[size_t(d)] = x;
          }
        }
        break;
      }
      case OpType::Sum: {
        const int d = std::get<SumAttrs>(o.attrs).dim;
        const int l = lab(0, d);
        if (l < 0 || !job_.sum_labels.count(l)) return false;
        for (int k = 0; k < R; ++k) nt.lab[size_t(k)] = k == d ? -1 : lab(0, k);
        break;
      }
      case OpType::Accum: {
        for (int k = 0; k < R; ++k) nt.lab[size_t(k)] = lab(0, k);
        break;
      }
      default: {  // elementwise, right-aligned broadcast: aligned dims of extent > 1 agree
        for (int i = 0; i < o.nin; ++i) {
          const int r = rk(i);
          for (int k = 1; k <= r; ++k) {
            const int l = lab(i, r - k);
            if (l < 0) continue;
            int &dst = nt.lab[size_t(R - k)];
            if (dst >= 0 && dst != l) return false;
            dst = l;
          }
        }
      }
    }
    for (int k = 0; k < R; ++k)
      if (nt.shape.dims[size_t(k)] <= 1) nt.lab[size_t(k)] = -1;
    return true;
  }

  // "all shared tensors consumed" and the program's expression behind one
  // Accum: emit the µGraph
  void complete() {
    if (unconsumed_ != 1 || ops_.empty()) return;
    const int t = int(T_.size()) - 1;  // the newest tensor is unconsumed (nothing read it yet)
    const BT &o = T_[size_t(t)];
    if (o.users || o.acc != 2 || o.e != eo_) return;
    const DimMap omap(std::vector<int>{job_.out_dim});
    ShapeResult whole = assemble_output_shape(o.shape, omap, {job_.gx});
    if (!whole || *whole.shape != out_shape_) return;
    ++st_.completed;
    // build it
    GraphBuilder gb;
    std::vector<TensorId> kt;
    for (TensorId x : prog_.inputs) kt.push_back(gb.input(prog_.tensor(x).shape));
    for (const KOp &k : job_.kops) {
      std::vector<TensorId> in;
      for (int x : k.in) in.push_back(kt[size_t(x)]);
      kt.push_back(gb.op(k.type, in, k.attrs));
    }
    std::vector<TensorShape> oshapes;
    std::vector<TensorId> ops_in;
    for (int x : job_.operands) oshapes.push_back(job_.kshape[size_t(x)]), ops_in.push_back(kt[size_t(x)]);
    try {
      BlockBuilder bb({job_.gx, 1, 1}, job_.fl, oshapes);
      std::vector<TensorId> bt;
      for (size_t i = 0; i < job_.operands.size(); ++i) bt.push_back(bb.initer(int(i), job_.imap[i], job_.fmap[i]));
      for (const BOp &op : ops_) {
        std::vector<TensorId> in;
        for (int i = 0; i < op.nin; ++i) in.push_back(bt[size_t(op.in[size_t(i)])]);
        bt.push_back(bb.op(op.type, in, op.attrs));
      }
      bb.outsaver(bt[size_t(t)], omap);
      const TensorId go = gb.graphdef(ops_in, bb.finish(), bb.out_shapes());
      KernelGraph g = gb.finish({go});
      if (!validate(g, cfg_.limits).valid()) {
        ++st_.rejected_validate;
        return;
      }
      out_.push_back(std::move(g));
    } catch (const Error &) {
      ++st_.rejected_validate;
    }
  }

  const KernelGraph &prog_;
  const Job &job_;
  const EnumConfig &cfg_;
  EnumStats &st_;
  std::vector<KernelGraph> &out_;
  std::array<std::vector<TensorShape>, 5> shv_;
  BT nt_;
  std::vector<int8_t> sub_eo_;  // expression id -> subexpr(e, eo_) (-1: not yet asked)
  std::array<std::vector<Id>, 5> iev_;
  Pool P_;
  Id eo_ = 0;
  TensorShape out_shape_;
  std::vector<BT> T_;
  std::vector<char> contraction_;  // tensor produced by Matmul / Sum / ConcatMatmul
  std::vector<BOp> ops_;
  int n_iniers_ = 0, unconsumed_ = 0, max_dec_ = 1;
  bool adds_ = true;
  uint64_t budget_local_ = 0;
  int64_t bytes_ = 0;
  Rank last_;
};

// ------------------------------------------------------------ kernel level

struct KernelSearch {
  const KernelGraph &prog;
  const EnumConfig &cfg;
  EnumStats &st;
  Pool P;
  Id eo = 0;
  std::vector<Job> jobs;

  // partitions of a GraphDef over `operands` of the prefix `kops`
  void partitions(const std::vector<KOp> &kops, const std::vector<TensorShape> &kshape, const std::vector<int> &operands) {
    // labels over the program's ops plus the prefix ops, on the same inputs
    KernelGraph aug = prog;
    std::vector<TensorId> kt(prog.inputs.begin(), prog.inputs.end());
    for (const KOp &k : kops) {
      Op op;
      op.id = int(aug.ops.size());
      op.type = k.type;
      op.attrs = k.attrs;
      for (int x : k.in) op.inputs.push_back(kt[size_t(x)]);
      TensorInfo ti;
      ti.id = TensorId(aug.tensors.size());
      ti.shape = kshape[kt.size()];
      ti.producer_op = op.id;
      aug.tensors.push_back(ti);
      op.outputs.push_back(ti.id);
      aug.ops.push_back(op);
      kt.push_back(ti.id);
    }
    labels::Labels L;
    try {
      L = labels::label(aug);
    } catch (const Error &) {
      return;
    }
    auto lab = [&](TensorId t, int d) {
      return aug.tensor(t).shape.dims[size_t(d)] > 1 ? L.find(L.off[size_t(t)] + d) : -1;
    };
    auto extent = [&](int l) -> int64_t {
      for (size_t t = 0; t < aug.tensors.size(); ++t)
        for (int d = 0; d < aug.tensors[t].shape.rank(); ++d)
          if (lab(TensorId(t), d) == l) return aug.tensors[t].shape.dims[size_t(d)];
      return 1;
    };
    std::set<int> mm_labels, sum_labels;
    for (const Op &op : aug.ops) {
      const TensorId a = op.inputs[0];
      if (op.type == OpType::Matmul) {
        const int l = lab(a, aug.tensor(a).shape.rank() - 1);
        if (l >= 0) mm_labels.insert(l);
      } else if (op.type == OpType::Sum) {
        const int l = lab(a, std::get<SumAttrs>(op.attrs).dim);
        if (l >= 0) sum_labels.insert(l);
      }
    }
    const TensorId o = prog.outputs[0];
    std::vector<std::pair<int, int>> glabels{{-1, 0}};  // (label, output dim)
    for (int d = 0; d < prog.tensor(o).shape.rank(); ++d) {
      const int l = lab(o, d);
      if (l >= 0 && !L.contracted.count(l)) glabels.push_back({l, d});
    }
    std::vector<int> cl;  // contracted labels present on some operand
    for (int l : L.contracted)
      for (int x : operands)
        for (int d = 0; d < kshape[size_t(x)].rank(); ++d)
          if (lab(kt[size_t(x)], d) == l && std::find(cl.begin(), cl.end(), l) == cl.end()) cl.push_back(l);
    // loop label lists, in priority order: an operand carrying several of
    // them is sliced along the first (LoRA: A along h, B along r)
    std::vector<std::vector<int>> fsets{{}};
    for (size_t i = 0; i < cl.size(); ++i) {
      fsets.push_back({cl[i]});
      if (cfg.max_loop_labels >= 2)
        for (size_t j = 0; j < cl.size(); ++j)
          if (j != i) fsets.push_back({cl[i], cl[j]});
    }
    for (auto [g, od] : glabels)
      for (int64_t gx : (g < 0 ? std::vector<int64_t>{1} : cfg.grids)) {
        if (g >= 0 && (gx <= 1 || extent(g) % gx)) continue;
        for (const auto &F : fsets)
          for (int64_t fl : (F.empty() ? std::vector<int64_t>{1} : cfg.loops)) {
            if (!F.empty() && fl <= 1) continue;
            bool ok = true;
            for (int l : F) ok = ok && l != g && extent(l) % fl == 0;
            if (!ok) continue;
            Job j;
            j.mm_labels = mm_labels;
            j.sum_labels = sum_labels;
            j.kops = kops;
            j.kshape = kshape;
            j.operands = operands;
            j.gx = gx;
            j.fl = fl;
            j.out_dim = g < 0 ? 0 : od;
            for (int x : operands) {
              int dg = -1, df = -1, fpri = int(F.size());
              for (int d = 0; d < kshape[size_t(x)].rank(); ++d) {
                const int l = lab(kt[size_t(x)], d);
                if (l < 0) continue;
                if (l == g) ok = ok && dg < 0, dg = d;
                const int pri = int(std::find(F.begin(), F.end(), l) - F.begin());
                if (pri < int(F.size())) {
                  ok = ok && pri != fpri;  // the same label on two dims
                  if (pri < fpri) fpri = pri, df = d;
                }
              }
              std::vector<int> dl;
              for (int d = 0; d < kshape[size_t(x)].rank(); ++d) dl.push_back(lab(kt[size_t(x)], d));
              j.dlab.push_back(dl);
              j.imap.emplace_back(std::vector<int>{dg >= 0 ? dg : kReplica});
              j.fmap.emplace_back(std::vector<int>{df >= 0 ? df : kReplica});
              j.ldim.push_back(df);
            }
            if (ok) jobs.push_back(std::move(j));
          }
      }
  }

  // GraphDef operand sets for a prefix: every unconsumed kernel tensor, plus
  // up to two consumed ones
  void graphdefs(const std::vector<KOp> &kops, const std::vector<TensorShape> &kshape, const std::vector<int> &users) {
    std::vector<int> must, may;
    for (size_t t = 0; t < kshape.size(); ++t) (users[t] ? may : must).push_back(int(t));
    std::vector<std::vector<int>> extra{{}};
    for (size_t i = 0; i < may.size(); ++i) {
      extra.push_back({may[i]});
      for (size_t j = i + 1; j < may.size(); ++j) extra.push_back({may[i], may[j]});
    }
    for (const auto &x : extra) {
      if (kops.empty() && !x.empty()) continue;  // no prefix: every input is unconsumed already
      std::vector<int> ops = must;
      ops.insert(ops.end(), x.begin(), x.end());
      std::sort(ops.begin(), ops.end());
      partitions(kops, kshape, ops);
    }
  }

  void dfs(std::vector<KOp> &kops, std::vector<TensorShape> &kshape, std::vector<Id> &ke, std::vector<int> &users,
           std::array<int, 4> last) {
    graphdefs(kops, kshape, users);
    if (int(kops.size()) >= cfg.max_kernel_ops) return;
    const int n = int(kshape.size());
    auto attempt = [&](OpType t, OpAttrs at, std::vector<int> in) {
      std::array<int, 4> r{-1, -1, -1, int(t)};
      int mx = -1;
      for (int x : in) mx = std::max(mx, x);
      r[0] = mx;
      for (size_t i = 0; i < in.size() && i < 2; ++i) r[1 + i] = in[i];
      if (!(r > last)) return;
      std::vector<TensorShape> sh;
      std::vector<Id> ie;
      for (int x : in) sh.push_back(kshape[size_t(x)]), ie.push_back(ke[size_t(x)]);
      ShapeResult s = infer_output_shape(t, at, sh, Level::Kernel);
      if (!s) return;
      const Id e = op_expr(P, t, at, ie, sh);
      if (!P.subexpr(e, eo) || e == eo) return;  // e == eo: the program itself, no GraphDef left to build
      for (size_t i = 0; i < ke.size(); ++i)
        if (ke[i] == e && kshape[i] == *s.shape) return;
      ++st.kernel_prefixes;
      kops.push_back({t, at, in});
      kshape.push_back(*s.shape);
      ke.push_back(e);
      for (int x : in) ++users[size_t(x)];
      users.push_back(0);
      dfs(kops, kshape, ke, users, r);
      users.pop_back();
      for (int x : in) --users[size_t(x)];
      ke.pop_back();
      kshape.pop_back();
      kops.pop_back();
    };
    for (int a = 0; a < n; ++a) {
      for (OpType t : {OpType::EwExp, OpType::Sqr, OpType::Sqrt, OpType::SiLU}) attempt(t, NoAttrs{}, {a});
      for (int d = 0; d < kshape[size_t(a)].rank(); ++d)
        if (kshape[size_t(a)].dims[size_t(d)] > 1) attempt(OpType::Sum, SumAttrs{d, kshape[size_t(a)].dims[size_t(d)]}, {a});
      for (int b = 0; b < n; ++b) {
        if (a <= b) attempt(OpType::EwAdd, NoAttrs{}, {a, b}), attempt(OpType::EwMul, NoAttrs{}, {a, b});
        attempt(OpType::EwDiv, NoAttrs{}, {a, b});
        attempt(OpType::Matmul, NoAttrs{}, {a, b});
      }
    }
  }
};

}  // namespace

std::string abstract_expression(const KernelGraph &g) {
  Pool P;
  return P.str(graph_exprs(P, g)[size_t(g.outputs.at(0))]);
}

std::vector<KernelGraph> enumerate_mugraphs(const KernelGraph &program, const EnumConfig &cfg, EnumStats *stats) {
  if (program.outputs.size() != 1) throw Error(ErrCode::Unsupported, "enumerator: single-output programs");
  for (const Op &op : program.ops)
    if (!labels::supported(op.type)) throw Error(ErrCode::Unsupported, std::string("enumerator: op ") + op_name(op.type));
  EnumStats st;
  KernelSearch ks{program, cfg, st};
  ks.eo = graph_exprs(ks.P, program)[size_t(program.outputs[0])];
  {
    std::vector<KOp> kops;
    std::vector<TensorShape> kshape;
    std::vector<Id> ke;
    for (size_t i = 0; i < program.inputs.size(); ++i) {
      kshape.push_back(program.tensor(program.inputs[i]).shape);
      ke.push_back(ks.P.var(uint32_t(i)));
    }
    std::vector<int> users(kshape.size(), 0);
    ks.dfs(kops, kshape, ke, users, {-2, -2, -2, -2});
  }
  st.partitions = ks.jobs.size();
  // block searches in parallel, one pool per search; results merged in job
  // order (deterministic while the prefix budget holds)
  std::vector<std::vector<KernelGraph>> res(ks.jobs.size());
  std::vector<EnumStats> jst(ks.jobs.size());
  const uint64_t per_job = std::max<uint64_t>(1000, cfg.max_prefixes / std::max<size_t>(1, ks.jobs.size()));
  std::atomic<size_t> next{0};
  const int nt = std::max(1, std::min<int>(cfg.threads > 0 ? cfg.threads : int(std::thread::hardware_concurrency()),
                                           int(ks.jobs.size())));
  auto work = [&] {
    for (;;) {
      const size_t j = next.fetch_add(1);
      if (j >= ks.jobs.size()) return;
      BlockSearch(program, ks.jobs[j], cfg, per_job, jst[j], res[j]).run();
    }
  };
  std::vector<std::thread> th;
  for (int i = 1; i < nt; ++i) th.emplace_back(work);
  work();
  for (auto &t : th) t.join();
  std::vector<KernelGraph> out;
  std::set<std::string> seen;
  for (size_t j = 0; j < res.size(); ++j) {
    const EnumStats &s = jst[j];
    st.prefixes += s.prefixes, st.pruned_expr += s.pruned_expr, st.pruned_shape += s.pruned_shape;
    st.pruned_memory += s.pruned_memory, st.pruned_structure += s.pruned_structure;
    st.completed += s.completed, st.rejected_validate += s.rejected_validate;
    st.budget_exhausted = st.budget_exhausted || s.budget_exhausted;
    for (KernelGraph &g : res[j]) {
      if (out.size() >= cfg.max_candidates) break;
      if (!seen.insert(canonical_key(g)).second) {
        ++st.duplicates;
        continue;
      }
      out.push_back(std::move(g));
    }
  }
  if (stats) *stats = st;
  return out;
}

}  // namespace tpo::ir
