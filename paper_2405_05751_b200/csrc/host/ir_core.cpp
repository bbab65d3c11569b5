// B200 backend — IR core: names, operator table, shape inference, builders.
// Behaviour follows the reference's ops.cpp:38-148, shape_infer.cpp:27-217,
// graph.cpp:36-161 and shape.cpp:20-81 (same results, independent code).
#include <algorithm>
#include <sstream>

#include "tpo/ir/graph.hpp"
#include "tpo/ir/shape_infer.hpp"

namespace tpo {

const char *err_name(ErrCode c) {
  static const char *const kNames[] = {
      "ShapeMismatch", "NotDivisible", "ReplicaInOmap", "Unsupported", "DivByZero",
      "NonResidue",    "PoisonedExponent", "BudgetExhausted", "Infeasible", "DoesNotFit",
      "ParseError",    "NotLax",        "UnknownSuite", "ConfigError"};
  int i = int(c);
  return (i >= 0 && i < int(sizeof(kNames) / sizeof(kNames[0]))) ? kNames[i] : "Unknown";
}

namespace ir {

// ---------------------------------------------------------------- names ---

std::string to_string(const TensorShape &s) {
  std::string r = "[";
  for (size_t i = 0; i < s.dims.size(); ++i) r += (i ? "," : "") + std::to_string(s.dims[i]);
  return r + "]";
}

const char *scope_name(Scope s) {
  return s == Scope::Device ? "device" : s == Scope::Shared ? "shared" : "register";
}

std::string to_string(const DimMap &m, bool grid_axes) {
  static const char *const kAxes[] = {"x", "y", "z"};
  std::string r = "{";
  for (int a = 0; a < m.axes(); ++a) {
    if (a) r += ",";
    r += grid_axes ? kAxes[a] : "i";
    r += "<->";
    int t = m.targets[size_t(a)];
    r += t == kReplica ? std::string("phi") : std::to_string(t);
  }
  return r + "}";
}

// ------------------------------------------------------------ op table ---

namespace {
struct OpInfo {
  const char *name;
  int arity;        // -1 variable
  bool kernel, block, thread;
  bool elementwise;
};
// Order == OpType ordinals.
constexpr OpInfo kOps[kNumOpTypes] = {
    {"initer", 0, false, true, false, false},
    {"outsaver", 1, false, true, false, false},
    {"matmul", 2, true, true, true, false},
    {"sum", 1, true, true, true, false},
    {"ewadd", 2, true, true, true, true},
    {"ewmul", 2, true, true, true, true},
    {"ewdiv", 2, true, true, true, true},
    {"ewexp", 1, true, true, true, true},
    {"repeat", 1, true, true, false, false},
    {"reshape", 1, true, true, false, false},
    {"sqr", 1, true, true, false, true},
    {"sqrt", 1, true, true, false, true},
    {"silu", 1, true, true, false, true},
    {"accum", 1, false, true, false, false},
    {"concatmatmul", 4, true, true, false, false},
    {"graphdef", -1, true, false, false, false},
};
}  // namespace

const char *op_name(OpType t) { return kOps[int(t)].name; }

OpType op_from_name(const std::string &name) {
  for (int i = 0; i < kNumOpTypes; ++i)
    if (name == kOps[i].name) return OpType(i);
  throw Error(ErrCode::ParseError, "unknown op type '" + name + "'");
}

bool op_allowed_at(OpType t, Level level) {
  const OpInfo &o = kOps[int(t)];
  return level == Level::Kernel ? o.kernel : level == Level::Block ? o.block : o.thread;
}

int op_arity(OpType t) { return kOps[int(t)].arity; }
bool op_elementwise(OpType t) { return kOps[int(t)].elementwise; }
bool op_commutative(OpType t) { return t == OpType::EwAdd || t == OpType::EwMul; }

namespace {
std::string map_key(const DimMap &m) {
  std::string r = "[";
  for (int t : m.targets) r += std::to_string(t) + ",";
  return r + "]";
}
}  // namespace

std::string attr_key(const OpAttrs &a) {
  struct V {
    std::string operator()(const NoAttrs &) const { return "-"; }
    std::string operator()(const SumAttrs &s) const {
      return "sum:" + std::to_string(s.dim) + ":" + std::to_string(s.group);
    }
    std::string operator()(const AccumAttrs &s) const { return "accum:" + map_key(s.fmap); }
    std::string operator()(const ReshapeAttrs &s) const { return "reshape:" + to_string(s.target); }
    std::string operator()(const RepeatAttrs &s) const { return "repeat:" + to_string(s.target); }
    std::string operator()(const InIterAttrs &s) const {
      return "initer:" + std::to_string(s.operand) + ":" + map_key(s.imap) + map_key(s.fmap);
    }
    std::string operator()(const OutSaverAttrs &s) const { return "outsaver:" + map_key(s.omap); }
  };
  return std::visit(V{}, a);
}

// ------------------------------------------------------ shape inference ---

namespace {
ShapeResult ok(TensorShape s) { return ShapeResult{std::move(s), ErrCode::ShapeMismatch}; }
ShapeResult bad(ErrCode c = ErrCode::ShapeMismatch) { return ShapeResult{std::nullopt, c}; }

// Batched contraction of a's last dim with b's second-to-last; equal rank
// and identical leading (batch) dims.
ShapeResult contract(const TensorShape &a, const TensorShape &b) {
  int r = a.rank();
  if (r < 2 || b.rank() != r) return bad();
  if (!std::equal(a.dims.begin(), a.dims.end() - 2, b.dims.begin())) return bad();
  if (a.dims[size_t(r - 1)] != b.dims[size_t(r - 2)]) return bad();
  TensorShape o = a;
  o.dims.back() = b.dims.back();
  return ok(o);
}
}  // namespace

std::optional<TensorShape> broadcast_shapes(const TensorShape &a, const TensorShape &b) {
  const int r = std::max(a.rank(), b.rank());
  TensorShape o;
  o.dims.resize(size_t(r));
  for (int i = 0; i < r; ++i) {
    int ia = i - (r - a.rank()), ib = i - (r - b.rank());
    int64_t x = ia >= 0 ? a.dims[size_t(ia)] : 1;
    int64_t y = ib >= 0 ? b.dims[size_t(ib)] : 1;
    if (x != y && x != 1 && y != 1) return std::nullopt;
    o.dims[size_t(i)] = x > y ? x : y;
  }
  return o;
}

ShapeResult infer_output_shape(OpType op, const OpAttrs &attrs,
                               const std::vector<TensorShape> &in, Level level) {
  if (!op_allowed_at(op, level)) return bad(ErrCode::Unsupported);
  for (const auto &s : in)
    if (!s.valid()) return bad();
  const size_t n = in.size();
  switch (op) {
    case OpType::Matmul:
      return n == 2 ? contract(in[0], in[1]) : bad();
    case OpType::ConcatMatmul: {
      if (n != 4) return bad();
      ShapeResult l = contract(in[0], in[2]), r = contract(in[1], in[3]);
      if (!l || !r || *l.shape != *r.shape) return bad();
      return l;
    }
    case OpType::Sum: {
      if (n != 1) return bad();
      const auto &s = std::get<SumAttrs>(attrs);
      if (s.dim < 0 || s.dim >= in[0].rank() || s.group < 1) return bad();
      TensorShape o = in[0];
      if (o.dims[size_t(s.dim)] % s.group) return bad();
      o.dims[size_t(s.dim)] /= s.group;
      return ok(o);
    }
    case OpType::EwAdd:
    case OpType::EwMul:
    case OpType::EwDiv: {
      if (n != 2) return bad();
      auto s = broadcast_shapes(in[0], in[1]);
      return s ? ok(*s) : bad();
    }
    case OpType::EwExp:
    case OpType::Sqr:
    case OpType::Sqrt:
    case OpType::SiLU:
      return n == 1 ? ok(in[0]) : bad();
    case OpType::Repeat: {
      if (n != 1) return bad();
      const auto &t = std::get<RepeatAttrs>(attrs).target;
      if (!t.valid()) return bad();
      auto s = broadcast_shapes(in[0], t);
      return (s && *s == t) ? ok(t) : bad();
    }
    case OpType::Reshape: {
      if (n != 1) return bad();
      const auto &t = std::get<ReshapeAttrs>(attrs).target;
      return (t.valid() && t.elem_count() == in[0].elem_count()) ? ok(t) : bad();
    }
    case OpType::InIter:
    case OpType::OutSaver:
      if (op == OpType::OutSaver && n != 1) return bad();
      return n ? ok(in[0]) : bad();
    case OpType::Accum: {
      if (n != 1) return bad();
      const auto &a = std::get<AccumAttrs>(attrs);
      if (a.fmap.axes() != 1) return bad();
      int t = a.fmap.targets[0];
      if (t != kReplica && (t < 0 || t >= in[0].rank())) return bad();
      return ok(in[0]);  // concat extent (x forloop) applied by the builder
    }
    case OpType::GraphDef:
      return bad(ErrCode::Unsupported);
  }
  return bad(ErrCode::Unsupported);
}

TensorShape infer_output_shape_or_throw(OpType op, const OpAttrs &attrs,
                                        const std::vector<TensorShape> &in, Level level) {
  ShapeResult r = infer_output_shape(op, attrs, in, level);
  if (!r) throw Error(r.err, std::string("infer_output_shape(") + op_name(op) + ")");
  return *r.shape;
}

ShapeResult partition_shape(const TensorShape &shape, const DimMap &map,
                            const std::vector<int64_t> &ext) {
  if (size_t(map.axes()) != ext.size() || !map.targets_distinct()) return bad();
  TensorShape o = shape;
  for (size_t a = 0; a < ext.size(); ++a) {
    int t = map.targets[a];
    if (t == kReplica) continue;
    if (t < 0 || t >= shape.rank()) return bad();
    if (ext[a] < 1 || o.dims[size_t(t)] % ext[a]) return bad(ErrCode::NotDivisible);
    o.dims[size_t(t)] /= ext[a];
  }
  return ok(o);
}

ShapeResult assemble_output_shape(const TensorShape &per_block, const DimMap &omap,
                                  const std::vector<int64_t> &grid) {
  if (size_t(omap.axes()) != grid.size() || !omap.targets_distinct()) return bad();
  TensorShape o = per_block;
  for (size_t a = 0; a < grid.size(); ++a) {
    int t = omap.targets[a];
    if (t == kReplica) return bad(ErrCode::ReplicaInOmap);
    if (t < 0 || t >= per_block.rank()) return bad();
    o.dims[size_t(t)] *= grid[a];
  }
  return ok(o);
}

TensorShape partition_or_throw(const TensorShape &s, const DimMap &m,
                               const std::vector<int64_t> &e) {
  ShapeResult r = partition_shape(s, m, e);
  if (!r) throw Error(r.err, "partition_shape " + to_string(s));
  return *r.shape;
}

TensorShape assemble_or_throw(const TensorShape &s, const DimMap &m,
                              const std::vector<int64_t> &g) {
  ShapeResult r = assemble_output_shape(s, m, g);
  if (!r) throw Error(r.err, "assemble_output_shape " + to_string(s));
  return *r.shape;
}

int64_t op_madds(OpType op, const OpAttrs &, const std::vector<TensorShape> &in,
                 const TensorShape &out) {
  switch (op) {
    case OpType::Matmul:
      return out.elem_count() * in[0].dims.back();
    case OpType::ConcatMatmul:
      return out.elem_count() * (in[0].dims.back() + in[1].dims.back());
    case OpType::Sum:
    case OpType::Accum:
      return in[0].elem_count();
    default:
      return op_elementwise(op) ? out.elem_count() : 0;
  }
}

// ------------------------------------------------------------- builders ---

std::vector<TensorId> KernelGraph::dangling() const {
  std::vector<char> used(tensors.size(), 0);
  for (const Op &op : ops)
    for (TensorId t : op.inputs) used[size_t(t)] = 1;
  for (TensorId t : inputs) used[size_t(t)] = 1;
  std::vector<TensorId> out;
  for (const TensorInfo &t : tensors)
    if (!used[size_t(t.id)]) out.push_back(t.id);
  return out;
}

TensorId GraphBuilder::input(TensorShape shape) {
  TensorId id = TensorId(g_.tensors.size());
  g_.tensors.push_back(TensorInfo{id, std::move(shape), Scope::Device, -1, 0, std::nullopt});
  g_.inputs.push_back(id);
  return id;
}

TensorId GraphBuilder::op(OpType type, std::vector<TensorId> inputs, OpAttrs attrs) {
  std::vector<TensorShape> shapes;
  for (TensorId t : inputs) shapes.push_back(g_.tensor(t).shape);
  TensorShape out = infer_output_shape_or_throw(type, attrs, shapes, Level::Kernel);
  const int op_id = int(g_.ops.size());
  const TensorId out_id = TensorId(g_.tensors.size());
  g_.tensors.push_back(TensorInfo{out_id, std::move(out), Scope::Device, op_id, 0, std::nullopt});
  Op o;
  o.id = op_id;
  o.type = type;
  o.attrs = std::move(attrs);
  o.inputs = std::move(inputs);
  o.outputs = {out_id};
  g_.ops.push_back(std::move(o));
  return out_id;
}

TensorId GraphBuilder::graphdef(std::vector<TensorId> inputs, std::shared_ptr<BlockGraph> block,
                                const std::vector<TensorShape> &out_shapes) {
  Op o;
  o.id = int(g_.ops.size());
  o.type = OpType::GraphDef;
  o.inputs = std::move(inputs);
  o.block = std::move(block);
  for (size_t i = 0; i < out_shapes.size(); ++i) {
    TensorId id = TensorId(g_.tensors.size());
    g_.tensors.push_back(TensorInfo{id, out_shapes[i], Scope::Device, o.id, int(i), std::nullopt});
    o.outputs.push_back(id);
  }
  TensorId first = o.outputs.empty() ? -1 : o.outputs[0];
  g_.ops.push_back(std::move(o));
  return first;
}

KernelGraph GraphBuilder::finish(std::vector<TensorId> outputs) {
  g_.outputs = std::move(outputs);
  return g_;
}

BlockBuilder::BlockBuilder(std::array<int64_t, 3> grid, int64_t forloop,
                           std::vector<TensorShape> operand_shapes)
    : bg_(std::make_shared<BlockGraph>()), operand_shapes_(std::move(operand_shapes)) {
  bg_->grid = grid;
  bg_->forloop = forloop;
}

namespace {
std::vector<int64_t> grid_prefix(const std::array<int64_t, 3> &g, int axes) {
  std::vector<int64_t> e(g.begin(), g.end());
  e.resize(size_t(axes), 1);
  return e;
}
}  // namespace

TensorId BlockBuilder::initer(int operand, DimMap imap, DimMap fmap) {
  const TensorShape &dev = operand_shapes_.at(size_t(operand));
  TensorShape tile = partition_or_throw(dev, imap, grid_prefix(bg_->grid, imap.axes()));
  tile = partition_or_throw(tile, fmap, {bg_->forloop});
  Op o;
  o.id = int(bg_->ops.size());
  o.type = OpType::InIter;
  TensorId out = TensorId(bg_->tensors.size());
  bg_->tensors.push_back(TensorInfo{out, tile, Scope::Shared, o.id, 0, std::nullopt});
  o.attrs = InIterAttrs{operand, std::move(imap), std::move(fmap)};
  o.outputs = {out};
  bg_->ops.push_back(std::move(o));
  return out;
}

TensorId BlockBuilder::op(OpType type, std::vector<TensorId> inputs, OpAttrs attrs) {
  std::vector<TensorShape> shapes;
  for (TensorId t : inputs) shapes.push_back(bg_->tensor(t).shape);
  TensorShape out = infer_output_shape_or_throw(type, attrs, shapes, Level::Block);
  if (type == OpType::Accum) {
    int t = std::get<AccumAttrs>(attrs).fmap.targets[0];
    if (t != kReplica) out.dims[size_t(t)] *= bg_->forloop;
  }
  Op o;
  o.id = int(bg_->ops.size());
  o.type = type;
  o.attrs = std::move(attrs);
  o.inputs = std::move(inputs);
  TensorId id = TensorId(bg_->tensors.size());
  bg_->tensors.push_back(TensorInfo{id, std::move(out), Scope::Shared, o.id, 0, std::nullopt});
  o.outputs = {id};
  bg_->ops.push_back(std::move(o));
  return id;
}

TensorShape BlockBuilder::outsaver(TensorId value, DimMap omap) {
  TensorShape out =
      assemble_or_throw(bg_->tensor(value).shape, omap, grid_prefix(bg_->grid, omap.axes()));
  Op o;
  o.id = int(bg_->ops.size());
  o.type = OpType::OutSaver;
  o.attrs = OutSaverAttrs{std::move(omap)};
  o.inputs = {value};
  bg_->ops.push_back(std::move(o));
  out_shapes_.push_back(out);
  return out;
}

std::shared_ptr<BlockGraph> BlockBuilder::finish() { return bg_; }

// ------------------------------------------------------- canonical key ---

namespace {
void key_ops(std::ostringstream &os, const std::vector<Op> &ops);

void key_block(std::ostringstream &os, const BlockGraph &bg) {
  os << "B(" << bg.grid[0] << ',' << bg.grid[1] << ',' << bg.grid[2] << ';' << bg.forloop << ';';
  key_ops(os, bg.ops);
  os << ')';
}

void key_ops(std::ostringstream &os, const std::vector<Op> &ops) {
  for (const Op &op : ops) {
    os << op_name(op.type) << attr_key(op.attrs) << '<';
    for (TensorId t : op.inputs) os << t << ',';
    os << '>';
    if (op.block) key_block(os, *op.block);
  }
}
}  // namespace

// Same key string as the reference (graph.cpp:128-157) so keys can be
// compared across implementations.
std::string canonical_key(const KernelGraph &g) {
  std::ostringstream os;
  os << "K(";
  for (TensorId t : g.inputs) os << to_string(g.tensor(t).shape) << ';';
  key_ops(os, g.ops);
  os << "|out:";
  for (TensorId t : g.outputs) os << t << ',';
  os << ')';
  return os.str();
}

bool isomorphic(const KernelGraph &a, const KernelGraph &b) {
  return canonical_key(a) == canonical_key(b);
}

}  // namespace ir
}  // namespace tpo
