// B200 backend — abstract expressions in normal form; see tpo/ir/absexpr.hpp.
#include "tpo/ir/absexpr.hpp"

#include <algorithm>

namespace tpo::ir::absx {

namespace {

uint64_t sat_mul(uint64_t a, uint64_t b) {
  if (a && b > (uint64_t(1) << 62) / a) return uint64_t(1) << 62;
  return a * b;
}

// multiset inclusion of sorted sequences
template <class T>
bool includes(const std::vector<T> &big, const std::vector<T> &small) {
  return std::includes(big.begin(), big.end(), small.begin(), small.end());
}

}  // namespace

Id Pool::intern(Poly &&p) {
  std::sort(p.monos.begin(), p.monos.end());
  std::vector<uint64_t> key;
  for (const Mono &m : p.monos) {
    key.push_back(m.count);
    key.push_back(m.atoms.size());
    key.insert(key.end(), m.atoms.begin(), m.atoms.end());
  }
  auto it = poly_ids_.find(key);
  if (it != poly_ids_.end()) return it->second;
  const Id id = Id(polys_.size());
  polys_.push_back(std::move(p));
  poly_ids_.emplace(std::move(key), id);
  return id;
}

Id Pool::atom(Atom a) {
  auto key = std::make_pair(int(a.kind), a.arg);
  auto it = atom_ids_.find(key);
  if (it != atom_ids_.end()) return it->second;
  const Id id = Id(atoms_.size());
  atoms_.push_back(a);
  atom_ids_.emplace(key, id);
  return id;
}

Id Pool::atom_poly(Id atom_id) {
  Poly p;
  p.monos.push_back(Mono{{atom_id}, 1});
  return intern(std::move(p));
}

Id Pool::var(uint32_t input) { return atom_poly(atom({AtomKind::Var, input})); }

Id Pool::unary(AtomKind k, Id a) { return atom_poly(atom({k, a})); }

Id Pool::add(Id a, Id b) {
  Poly p;
  p.monos = polys_[a].monos;
  const auto &bm = polys_[b].monos;
  p.monos.insert(p.monos.end(), bm.begin(), bm.end());
  return intern(std::move(p));
}

Id Pool::sum(uint64_t k, Id a) {
  if (k == 1) return a;
  auto it = sum_memo_.find({k, a});
  if (it != sum_memo_.end()) return it->second;
  Poly p = polys_[a];
  for (Mono &m : p.monos) m.count = sat_mul(m.count, k);
  const Id r = intern(std::move(p));
  sum_memo_.emplace(std::make_pair(k, a), r);
  return r;
}

// Product of two monomials, then the per-monomial merges: all exp atoms into
// one exp of the sum of their arguments, sqrt atoms into one sqrt of the
// product, inv atoms into one inv of the product.
Mono Pool::mono_mul(const Mono &x, const Mono &y) {
  Mono m;
  m.count = sat_mul(x.count, y.count);
  std::vector<Id> all = x.atoms;
  all.insert(all.end(), y.atoms.begin(), y.atoms.end());
  std::vector<Id> ex, sq, iv;
  for (Id t : all) {
    switch (atoms_[t].kind) {
      case AtomKind::Exp: ex.push_back(t); break;
      case AtomKind::Sqrt: sq.push_back(t); break;
      case AtomKind::Inv: iv.push_back(t); break;
      default: m.atoms.push_back(t);
    }
  }
  auto merge = [&](std::vector<Id> &v, AtomKind k, bool additive) {
    if (v.empty()) return;
    if (v.size() == 1) {
      m.atoms.push_back(v[0]);
      return;
    }
    Id acc = atoms_[v[0]].arg;
    for (size_t i = 1; i < v.size(); ++i) acc = additive ? add(acc, atoms_[v[i]].arg) : mul(acc, atoms_[v[i]].arg);
    m.atoms.push_back(atom({k, acc}));
  };
  merge(ex, AtomKind::Exp, true);
  merge(sq, AtomKind::Sqrt, false);
  merge(iv, AtomKind::Inv, false);
  std::sort(m.atoms.begin(), m.atoms.end());
  return m;
}

Id Pool::mul(Id a, Id b) {
  const uint64_t key = (uint64_t(std::min(a, b)) << 32) | std::max(a, b);
  auto it = mul_memo_.find(key);
  if (it != mul_memo_.end()) return it->second;
  Poly p;
  // copies: mono_mul may intern (and reallocate polys_)
  const std::vector<Mono> am = polys_[a].monos, bm = polys_[b].monos;
  for (const Mono &x : am)
    for (const Mono &y : bm) p.monos.push_back(mono_mul(x, y));
  const Id r = intern(std::move(p));
  mul_memo_.emplace(key, r);
  return r;
}

Id Pool::div(Id a, Id b) {
  const uint64_t key = (uint64_t(a) << 32) | b;
  auto it = div_memo_.find(key);
  if (it != div_memo_.end()) return it->second;
  const Id r = mul(a, unary(AtomKind::Inv, b));
  div_memo_.emplace(key, r);
  return r;
}

// a·f scaled by c is a sub-multiset of b, for the monomial f and count c
// that align a's first monomial with one of b's
bool Pool::contained(Id a, Id b) {
  const std::vector<Mono> A = polys_[a].monos, B = polys_[b].monos;
  if (A.empty() || A.size() > B.size()) return false;
  const Mono &n0 = A[0];
  for (const Mono &m : B) {
    if (m.count % n0.count || !includes(m.atoms, n0.atoms)) continue;
    Mono f;
    std::set_difference(m.atoms.begin(), m.atoms.end(), n0.atoms.begin(), n0.atoms.end(),
                        std::back_inserter(f.atoms));
    Poly fp;
    fp.monos.push_back(f);
    const Id x = sum(m.count / n0.count, mul(a, intern(std::move(fp))));
    if (includes(B, polys_[x].monos)) return true;
  }
  return false;
}

bool Pool::subexpr(Id a, Id b) {
  if (a == b) return true;
  const uint64_t key = (uint64_t(a) << 32) | b;
  auto it = sub_memo_.find(key);
  if (it != sub_memo_.end()) return it->second;
  sub_memo_[key] = false;  // guards recursion (terms are finite trees)
  bool r = contained(a, b);
  if (!r) {
    const std::vector<Mono> B = polys_[b].monos;
    Id prev = ~Id(0);
    for (const Mono &m : B)
      for (Id t : m.atoms) {
        if (r) break;
        if (t == prev || atoms_[t].kind == AtomKind::Var) continue;
        prev = t;
        r = subexpr(a, atoms_[t].arg);
      }
  }
  sub_memo_[key] = r;
  return r;
}

std::string Pool::str(Id p) const {
  static const char *names[] = {"x", "exp", "sqrt", "silu", "inv"};
  std::string s;
  const Poly &P = polys_[p];
  for (size_t i = 0; i < P.monos.size(); ++i) {
    const Mono &m = P.monos[i];
    if (i) s += " + ";
    if (m.count != 1) s += "Σ" + std::to_string(m.count) + "·";
    for (size_t j = 0; j < m.atoms.size(); ++j) {
      const Atom &a = atoms_[m.atoms[j]];
      if (j) s += "*";
      if (a.kind == AtomKind::Var)
        s += "x" + std::to_string(a.arg);
      else
        s += std::string(names[int(a.kind)]) + "(" + str(a.arg) + ")";
    }
  }
  return s.empty() ? "0" : s;
}

}  // namespace tpo::ir::absx
