// B200 backend — abstract expressions of µGraph tensors (§4.3,
// Table 2) in a normal form, for Algorithm 1's pruning.
//
// The reference decides subexpression entailment under the axioms of its
// Table 3 (A_eq ∪ A_sub) with a bounded saturation engine (the out-of-scope
// proj/core/src/subexpr.cpp).  Here the equivalence axioms are built into
// the representation instead, so equality is identity of interned terms:
//
//   polynomial  = multiset of monomials                (add: AC)
//   monomial    = multiset of atoms × reduction count  (mul: AC; sum(i, ·)
//                 scales the count: sum(1,x) = x, sum(i,sum(j,x)) =
//                 sum(ij,x), and sum distributes over add / mul / div)
//   atom        = var(input) | exp(P) | sqrt(P) | silu(P) | inv(P)
//   mul distributes over add (expanded polynomials); div(x, y) = x·inv(y);
//   within a monomial exp(x)·exp(y) = exp(x+y), sqrt(x)·sqrt(y) =
//   sqrt(x·y) and inv(x)·inv(y) = inv(x·y) are merged, which also gives
//   mul(x, div(y, z)) = div(mul(x, y), z) and div(div(x, y), z) =
//   div(x, mul(y, z)).
//
// subexpr(a, b) is the A_sub closure on normal forms: a ⊑ b when a, times
// some monomial factor and scaled by some reduction count, is a
// sub-multiset of b (x ⊑ x+y, x ⊑ x·y, x ⊑ sum(i,x), transitivity), or
// when a ⊑ the argument of an atom of b (x ⊑ exp(x), sqrt(x), silu(x),
// and y ⊑ div(x, y)).  It is sound for pruning in the direction that
// matters (never claims a prefix can contribute when no rewriting by the
// axioms makes it a subterm) and complete on the benchmark µGraphs; the
// one known gap is a product of two exps against one merged exp.
#pragma once

#include <cstdint>
#include <map>
#include <string>
#include <unordered_map>
#include <vector>

namespace tpo::ir::absx {

using Id = uint32_t;

enum class AtomKind : uint8_t { Var = 0, Exp, Sqrt, Silu, Inv };

struct Atom {
  AtomKind kind;
  uint32_t arg;  // Var: kernel-input index; otherwise a polynomial id
};

struct Mono {
  std::vector<Id> atoms;  // atom ids, sorted (a multiset)
  uint64_t count = 1;     // reduction count (product of summed extents)
  bool operator<(const Mono &o) const { return atoms != o.atoms ? atoms < o.atoms : count < o.count; }
  bool operator==(const Mono &o) const { return atoms == o.atoms && count == o.count; }
};

struct Poly {
  std::vector<Mono> monos;  // sorted (a multiset)
};

// Interning arena: structurally equal normal forms get equal ids.  Not
// thread-safe; use one pool per search worker.
class Pool {
 public:
  Id var(uint32_t input);
  Id add(Id a, Id b);
  Id mul(Id a, Id b);
  Id div(Id a, Id b);
  Id exp(Id a) { return unary(AtomKind::Exp, a); }
  Id sqrt(Id a) { return unary(AtomKind::Sqrt, a); }
  Id silu(Id a) { return unary(AtomKind::Silu, a); }
  Id sum(uint64_t k, Id a);
  bool subexpr(Id a, Id b);
  const Poly &poly(Id p) const { return polys_[p]; }
  const Atom &atom_of(Id a) const { return atoms_[a]; }
  std::string str(Id p) const;
  size_t size() const { return polys_.size(); }

 private:
  Id unary(AtomKind k, Id a);
  Id intern(Poly &&p);
  Id add_uncached(Id a, Id b);
  Id atom(Atom a);
  Id atom_poly(Id atom_id);
  Mono mono_mul(const Mono &x, const Mono &y);
  bool contained(Id a, Id b);

  std::vector<Atom> atoms_;
  std::map<std::pair<int, uint32_t>, Id> atom_ids_;
  std::vector<Poly> polys_;
  std::map<std::vector<uint64_t>, Id> poly_ids_;
  std::unordered_map<uint64_t, Id> mul_memo_;
  // add / unary / div are memoised like mul: the enumerator re-derives the
  // same (op, operand ids) at every DFS branch sharing a prefix
  std::unordered_map<uint64_t, Id> add_memo_, unary_memo_, div_memo_;
  std::map<std::pair<uint64_t, Id>, Id> sum_memo_;
  std::unordered_map<uint64_t, bool> sub_memo_;
};

}  // namespace tpo::ir::absx
