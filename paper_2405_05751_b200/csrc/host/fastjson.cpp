// B200 backend — fast path for the JSON wire format.
//
// A search loop hands the backend tens of thousands of distinct candidate
// graphs per second as JSON text (serialize.hpp schema); a generic DOM
// parser spends ~60 µs per 2 KB graph allocating maps and strings.  This
// path tokenises the text into a flat node array (no per-value
// allocation) and builds the KernelGraph straight from it.  It is strict:
// any input it does not fully understand — non-integer numbers, escapes,
// duplicate keys, values outside int range, unknown scopes or op names,
// structural surprises — makes it return false, and the caller falls back
// to the nlohmann path, which produces the canonical result or error.  On
// every input it accepts it yields exactly what kernel_graph_from_json
// yields (tests/test_abi.py checks both on every golden graph).
#include <charconv>
#include <cstring>
#include <span>
#include <string_view>

#include "tpo/ir/serialize.hpp"

namespace tpo::ir {

namespace {

struct Node {
  enum Kind : uint8_t { Obj, Arr, Str, Int, Lit } kind;
  uint32_t a = 0, b = 0;  // Obj: [a, b) key/value pairs in `kv`; Arr: [a, b) in `items`; Str: bytes
  int64_t i = 0;
};

class Tok {
 public:
  Tok(const char *s, size_t n) : p_(s), e_(s + n), base_(s) {
    // ~1 node per 6 bytes of the schema's compact text
    nodes.reserve(n / 4 + 16);
    kv.reserve(n / 12 + 8);
    items.reserve(n / 8 + 8);
    kstk_.reserve(64);
    istk_.reserve(256);
  }

  bool parse(uint32_t &root) {
    ws();
    if (!value(root, 0)) return false;
    ws();
    return p_ == e_;
  }

  const Node &node(uint32_t k) const { return nodes[k]; }
  std::string_view str(uint32_t k) const { return {base_ + nodes[k].a, nodes[k].b - nodes[k].a}; }

  // child of object `o` under `key`, or -1
  int64_t get(uint32_t o, std::string_view key) const {
    const Node &n = nodes[o];
    for (uint32_t c = n.a; c < n.b; ++c)
      if (str(kv[c].first) == key) return kv[c].second;
    return -1;
  }

  std::vector<Node> nodes;
  std::vector<std::pair<uint32_t, uint32_t>> kv;  // (key string node, value node)
  std::vector<uint32_t> items;

 private:
  const char *p_, *e_, *base_;
  std::vector<std::pair<uint32_t, uint32_t>> kstk_;  // open objects' pairs
  std::vector<uint32_t> istk_;                       // open arrays' items

  void ws() {
    while (p_ < e_ && (*p_ == ' ' || *p_ == '\n' || *p_ == '\r' || *p_ == '\t')) ++p_;
  }

  uint32_t push(Node n) {
    nodes.push_back(n);
    return uint32_t(nodes.size() - 1);
  }

  bool string(uint32_t &out) {
    if (p_ >= e_ || *p_ != '"') return false;
    const char *s = ++p_;
    while (p_ < e_ && *p_ != '"') {
      const unsigned char ch = static_cast<unsigned char>(*p_);
      if (ch == '\\' || ch < 0x20 || ch >= 0x80) return false;  // escapes, non-ASCII: slow path
      ++p_;
    }
    if (p_ >= e_) return false;
    Node n{Node::Str};
    n.a = uint32_t(s - base_), n.b = uint32_t(p_ - base_);
    ++p_;
    out = push(n);
    return true;
  }

  bool value(uint32_t &out, int depth) {
    if (depth > 32 || p_ >= e_) return false;
    const char c = *p_;
    if (c == '{') {
      ++p_;
      // children collect on a shared stack (no allocation per container)
      // and move to `kv` when the object closes
      const size_t base = kstk_.size();
      ws();
      if (p_ < e_ && *p_ == '}') {
        ++p_;
      } else {
        for (;;) {
          ws();
          uint32_t k, v;
          if (!string(k)) return false;
          ws();
          if (p_ >= e_ || *p_ != ':') return false;
          ++p_;
          ws();
          if (!value(v, depth + 1)) return false;
          for (size_t c = base; c < kstk_.size(); ++c)
            if (str(kstk_[c].first) == str(k)) return false;  // duplicate key: slow path decides
          kstk_.emplace_back(k, v);
          ws();
          if (p_ < e_ && *p_ == ',') {
            ++p_;
            continue;
          }
          if (p_ < e_ && *p_ == '}') {
            ++p_;
            break;
          }
          return false;
        }
      }
      Node n{Node::Obj};
      n.a = uint32_t(kv.size());
      kv.insert(kv.end(), kstk_.begin() + std::ptrdiff_t(base), kstk_.end());
      kstk_.resize(base);
      n.b = uint32_t(kv.size());
      out = push(n);
      return true;
    }
    if (c == '[') {
      ++p_;
      const size_t base = istk_.size();
      ws();
      if (p_ < e_ && *p_ == ']') {
        ++p_;
      } else {
        for (;;) {
          ws();
          uint32_t v;
          if (!value(v, depth + 1)) return false;
          istk_.push_back(v);
          ws();
          if (p_ < e_ && *p_ == ',') {
            ++p_;
            continue;
          }
          if (p_ < e_ && *p_ == ']') {
            ++p_;
            break;
          }
          return false;
        }
      }
      Node n{Node::Arr};
      n.a = uint32_t(items.size());
      items.insert(items.end(), istk_.begin() + std::ptrdiff_t(base), istk_.end());
      istk_.resize(base);
      n.b = uint32_t(items.size());
      out = push(n);
      return true;
    }
    if (c == '"') return string(out);
    if (c == '-' || (c >= '0' && c <= '9')) {
      const char *d = c == '-' ? p_ + 1 : p_;
      if (d + 1 < e_ && *d == '0' && d[1] >= '0' && d[1] <= '9') return false;  // leading zero: invalid JSON
      int64_t v = 0;
      auto r = std::from_chars(p_, e_, v);
      if (r.ec != std::errc()) return false;
      if (r.ptr < e_ && (*r.ptr == '.' || *r.ptr == 'e' || *r.ptr == 'E')) return false;  // not an integer
      p_ = r.ptr;
      Node n{Node::Int};
      n.i = v;
      out = push(n);
      return true;
    }
    return false;  // true / false / null: not in the schema's fast subset
  }
};

struct Fail {};

class Builder {
 public:
  explicit Builder(const Tok &t) : t_(t) {}

  KernelGraph graph(uint32_t root) {
    obj(root);
    KernelGraph g;
    g.tensors = tensors(need(root, "tensors"));
    for (uint32_t o : arr(need(root, "ops"))) {
      Op op = parse_op(o);
      ids_ok(op.inputs, g.tensors.size());
      ids_ok(op.outputs, g.tensors.size());
      int k = 0;
      for (TensorId t : op.outputs) {
        g.tensor(t).producer_op = op.id;
        g.tensor(t).producer_out = k++;
      }
      g.ops.push_back(std::move(op));
    }
    g.inputs = ints<TensorId>(need(root, "inputs"));
    g.outputs = ints<TensorId>(need(root, "outputs"));
    ids_ok(g.inputs, g.tensors.size());
    ids_ok(g.outputs, g.tensors.size());
    return g;
  }

 private:
  const Tok &t_;

  void obj(uint32_t n) const {
    if (t_.node(n).kind != Node::Obj) throw Fail{};
  }
  uint32_t need(uint32_t o, std::string_view k) const {
    obj(o);
    const int64_t v = t_.get(o, k);
    if (v < 0) throw Fail{};
    return uint32_t(v);
  }
  std::span<const uint32_t> arr(uint32_t n) const {
    const Node &x = t_.node(n);
    if (x.kind != Node::Arr) throw Fail{};
    return {t_.items.data() + x.a, size_t(x.b - x.a)};
  }
  int64_t i64(uint32_t n) const {
    const Node &x = t_.node(n);
    if (x.kind != Node::Int) throw Fail{};
    return x.i;
  }
  int i32(uint32_t n) const {
    const int64_t v = i64(n);
    if (v < INT32_MIN || v > INT32_MAX) throw Fail{};
    return int(v);
  }
  template <class I>
  std::vector<I> ints(uint32_t n) const {
    const auto a = arr(n);
    std::vector<I> out;
    out.reserve(a.size());
    for (uint32_t c : a) out.push_back(I(sizeof(I) == 8 ? i64(c) : i32(c)));
    return out;
  }
  std::string_view sv(uint32_t n) const {
    if (t_.node(n).kind != Node::Str) throw Fail{};
    return t_.str(n);
  }
  static void ids_ok(const std::vector<TensorId> &ids, size_t n) {
    for (TensorId t : ids)
      if (t < 0 || size_t(t) >= n) throw Fail{};
  }

  std::vector<TensorInfo> tensors(uint32_t a) const {
    std::vector<TensorInfo> ts;
    for (uint32_t e : arr(a)) {
      TensorInfo t;
      t.id = i32(need(e, "id"));
      if (t.id != int(ts.size())) throw Fail{};
      t.shape = TensorShape(ints<int64_t>(need(e, "shape")));
      const std::string_view sc = sv(need(e, "scope"));
      if (sc == "device")
        t.scope = Scope::Device;
      else if (sc == "shared")
        t.scope = Scope::Shared;
      else if (sc == "register")
        t.scope = Scope::Register;
      else
        throw Fail{};
      if (t_.get(e, "layout") >= 0) t.layout = i32(need(e, "layout"));
      ts.push_back(std::move(t));
    }
    return ts;
  }

  DimMap dmap(uint32_t o, bool grid) const {
    static const char *const kGrid[] = {"x", "y", "z"};
    obj(o);
    DimMap m;
    for (int a = 0; a < (grid ? 3 : 1); ++a) {
      const int64_t v = t_.get(o, grid ? kGrid[a] : "i");
      if (v < 0) break;
      if (t_.node(uint32_t(v)).kind == Node::Str) {
        if (t_.str(uint32_t(v)) != "phi") throw Fail{};
        m.targets.push_back(kReplica);
      } else {
        m.targets.push_back(i32(uint32_t(v)));
      }
    }
    return m;
  }

  OpAttrs attrs(OpType t, int64_t j) const {
    auto at = [&](std::string_view k) {
      if (j < 0) throw Fail{};
      return need(uint32_t(j), k);
    };
    switch (t) {
      case OpType::Sum:
        return SumAttrs{i32(at("dim")), i64(at("group"))};
      case OpType::Accum:
        return AccumAttrs{dmap(at("fmap"), false)};
      case OpType::Reshape:
        return ReshapeAttrs{TensorShape(ints<int64_t>(at("target")))};
      case OpType::Repeat:
        return RepeatAttrs{TensorShape(ints<int64_t>(at("target")))};
      case OpType::InIter:
        return InIterAttrs{i32(at("operand")), dmap(at("imap"), true), dmap(at("fmap"), false)};
      case OpType::OutSaver:
        return OutSaverAttrs{dmap(at("omap"), true)};
      default:
        if (j >= 0) obj(uint32_t(j));
        return NoAttrs{};
    }
  }

  Op parse_op(uint32_t o) const {
    Op op;
    op.id = i32(need(o, "id"));
    OpType ty;
    try {
      ty = op_from_name(std::string(sv(need(o, "type"))));
    } catch (const Error &) {
      throw Fail{};
    }
    op.type = ty;
    op.attrs = attrs(ty, t_.get(o, "attrs"));
    op.inputs = ints<TensorId>(need(o, "inputs"));
    op.outputs = ints<TensorId>(need(o, "outputs"));
    const int64_t b = t_.get(o, "blockGraph");
    if (b >= 0) op.block = block(uint32_t(b));
    return op;
  }

  std::shared_ptr<BlockGraph> block(uint32_t j) const {
    auto bg = std::make_shared<BlockGraph>();
    const auto grid = ints<int64_t>(need(j, "grid"));
    if (grid.size() != 3) throw Fail{};
    for (int a = 0; a < 3; ++a) bg->grid[size_t(a)] = grid[size_t(a)];
    bg->forloop = i64(need(j, "forloop"));
    bg->tensors = tensors(need(j, "tensors"));
    for (uint32_t jo : arr(need(j, "ops"))) {
      Op op = parse_op(jo);
      ids_ok(op.inputs, bg->tensors.size());
      ids_ok(op.outputs, bg->tensors.size());
      for (TensorId t : op.outputs) bg->tensor(t).producer_op = op.id;
      bg->ops.push_back(std::move(op));
    }
    const int64_t tg = t_.get(j, "threadGroups");
    if (tg >= 0)
      for (uint32_t g : arr(uint32_t(tg))) {
        ThreadGroup group;
        group.op_ids = ints<int>(need(g, "ops"));
        const auto bd = ints<int>(need(g, "blockDims"));
        for (size_t i = 0; i < 3 && i < bd.size(); ++i) group.block_dims[i] = bd[i];
        group.forloop = i32(need(g, "forloop"));
        bg->thread_groups.push_back(std::move(group));
      }
    return bg;
  }
};

}  // namespace

bool kernel_graph_from_text_fast(const char *text, size_t n, KernelGraph &out) {
  Tok t(text, n);
  uint32_t root;
  if (!t.parse(root)) return false;
  try {
    out = Builder(t).graph(root);
    return true;
  } catch (const Fail &) {
    return false;
  }
}

}  // namespace tpo::ir
