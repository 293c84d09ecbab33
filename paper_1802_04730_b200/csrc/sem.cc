// sem.cc — concrete range inference, specialization and static checks.
#include "sem.h"

#include <algorithm>
#include <cctype>
#include <functional>
#include <limits>
#include <optional>
#include <set>

namespace tcb {
namespace sem {

using lang::EK;
using lang::Expr;
using lang::ExprP;
using lang::Role;

const Range& CStmt::range(const std::string& it) const {
  auto f = ranges.find(it);
  TCB_CHECK(f != ranges.end(), "no range for iterator '" << it << "'");
  return f->second;
}

namespace {

int64_t floorDiv(int64_t a, int64_t b) {  // b > 0
  int64_t q = a / b;
  if ((a % b != 0) && (a < 0)) --q;
  return q;
}
int64_t ceilDiv(int64_t a, int64_t b) { return -floorDiv(-a, b); }

bool numeric(const std::string& s) {
  return !s.empty() && std::all_of(s.begin(), s.end(), [](unsigned char c) { return std::isdigit(c); });
}

// A subscript with every symbol concrete: sum(coef * iter) + cst.
struct Lin {
  std::map<std::string, int64_t> coef;
  int64_t cst = 0;
};

struct Access {
  std::string tensor;
  const std::vector<ExprP>* subs;
};

void collectReads(const ExprP& e, std::vector<Access>& out) {
  if (!e) return;
  if (e->k == EK::Access && !e->builtin) out.push_back({e->name, &e->kids});
  for (const auto& k : e->kids) collectReads(k, out);
}

class Inference {
 public:
  Inference(const lang::Validated& v, std::map<std::string, int64_t>& sizes,
            std::map<std::string, std::vector<int64_t>>& shapes)
      : v_(v), sizes_(sizes), shapes_(shapes) {
    size_t n = v.def.stmts.size();
    resolved_.resize(n);
    iterSet_.resize(n);
    acc_.resize(n);
    for (size_t s = 0; s < n; ++s) {
      iterSet_[s].insert(v.iters[s].begin(), v.iters[s].end());
      const auto& st = v.def.stmts[s];
      acc_[s].push_back({st.lhs, &st.idx});
      collectReads(st.rhs, acc_[s]);
      writers_[st.lhs].push_back(s);
    }
  }

  std::vector<std::map<std::string, Range>> run() {
    size_t n = v_.def.stmts.size();
    while (true) {
      std::vector<std::map<std::string, Range>> prop(n);
      auto propose = [&](size_t s, const std::string& u, Range r) {
        auto [it, fresh] = prop[s].emplace(u, r);
        if (!fresh) {
          it->second.lo = std::max(it->second.lo, r.lo);
          it->second.hi = std::min(it->second.hi, r.hi);
        }
      };
      for (size_t s = 0; s < n; ++s) {
        const auto& st = v_.def.stmts[s];
        for (const auto& w : st.where) {
          if (resolved_[s].count(w.var)) continue;
          auto lo = lin(w.lo, s), hi = lin(w.hi, s);
          if (!lo || !hi) continue;
          TCB_CHECK(lo->coef.empty() && hi->coef.empty(), "where bounds must not reference iterators");
          propose(s, w.var, Range{std::max<int64_t>(0, lo->cst), hi->cst});
        }
        for (const auto& a : acc_[s]) {
          auto sh = shapes_.find(a.tensor);
          if (sh == shapes_.end()) continue;
          for (size_t d = 0; d < a.subs->size() && d < sh->second.size(); ++d) {
            auto l = lin((*a.subs)[d], s);
            if (!l) continue;  // data-dependent or non-affine
            std::string u;
            int unresolved = 0;
            for (const auto& [it, c] : l->coef) {
              if (!resolved_[s].count(it)) {
                u = it;
                ++unresolved;
              }
            }
            if (unresolved != 1) continue;
            propose(s, u, solve(*l, u, sh->second[d], s));
          }
        }
      }
      bool progress = false;
      for (size_t s = 0; s < n; ++s) {
        for (const auto& [it, r] : prop[s]) {
          if (r.hi - r.lo <= 0)
            fail(ErrorKind::EmptyRange,
                 "inferred range [" + std::to_string(r.lo) + ", " + std::to_string(r.hi) + ") of iterator '" +
                     it + "' is empty",
                 v_.def.stmts[s].pos);
          resolved_[s].emplace(it, r);
          progress = true;
        }
      }
      for (const auto& [t, ws] : writers_) {
        if (shapes_.count(t)) continue;
        std::optional<std::vector<int64_t>> settled;
        for (size_t w : ws) {
          const auto& st = v_.def.stmts[w];
          std::vector<int64_t> dims;
          bool complete = true;
          for (const auto& ix : st.idx) {
            auto f = resolved_[w].find(ix->name);
            if (f == resolved_[w].end()) {
              complete = false;
              break;
            }
            dims.push_back(f->second.hi);
          }
          if (!complete) continue;
          if (!settled) settled = dims;
          else if (*settled != dims)
            fail(ErrorKind::Ambiguous, "writers of tensor '" + t + "' disagree on its shape", st.pos);
        }
        if (settled) {
          shapes_[t] = *settled;
          progress = true;
        }
      }
      if (!progress) break;
    }
    for (size_t s = 0; s < n; ++s)
      for (const auto& it : v_.iters[s])
        if (!resolved_[s].count(it))
          fail(ErrorKind::UnderConstrained, "cannot infer the range of iterator '" + it + "'",
               v_.def.stmts[s].pos);
    return resolved_;
  }

 private:
  std::optional<Lin> lin(const ExprP& e, size_t s) const {
    switch (e->k) {
      case EK::Int: return Lin{{}, e->ival};
      case EK::Ident: {
        if (iterSet_[s].count(e->name)) return Lin{{{e->name, 1}}, 0};
        auto z = sizes_.find(e->name);
        if (z == sizes_.end()) return std::nullopt;  // e.g. an int scalar parameter
        return Lin{{}, z->second};
      }
      case EK::DimOf: {
        auto f = shapes_.find(e->name);
        if (f == shapes_.end()) return std::nullopt;  // retry next round
        if (e->dim < 0 || e->dim >= static_cast<int>(f->second.size()))
          fail(ErrorKind::Name, "dimension " + std::to_string(e->dim) + " out of range for tensor '" + e->name + "'",
               e->pos);
        return Lin{{}, f->second[e->dim]};
      }
      case EK::Unary: {
        if (e->op != "-") return std::nullopt;
        auto a = lin(e->kids[0], s);
        if (!a) return std::nullopt;
        for (auto& kv : a->coef) kv.second = -kv.second;
        a->cst = -a->cst;
        return a;
      }
      case EK::Binary: {
        auto a = lin(e->kids[0], s), b = lin(e->kids[1], s);
        if (!a || !b) return std::nullopt;
        if (e->op == "+" || e->op == "-") {
          int64_t sg = e->op == "-" ? -1 : 1;
          for (const auto& [it, c] : b->coef) {
            a->coef[it] += sg * c;
            if (a->coef[it] == 0) a->coef.erase(it);
          }
          a->cst += sg * b->cst;
          return a;
        }
        if (e->op == "*") {
          const Lin* sc = b->coef.empty() ? &*b : (a->coef.empty() ? &*a : nullptr);
          const Lin* vec = b->coef.empty() ? &*a : &*b;
          if (!sc) return std::nullopt;
          Lin r;
          for (const auto& [it, c] : vec->coef)
            if (c * sc->cst != 0) r.coef[it] = c * sc->cst;
          r.cst = vec->cst * sc->cst;
          return r;
        }
        return std::nullopt;
      }
      default: return std::nullopt;
    }
  }

  // interval of the subscript without `skip`, over the resolved iterators
  std::pair<int64_t, int64_t> rest(const Lin& l, const std::string& skip, size_t s) const {
    int64_t lo = l.cst, hi = l.cst;
    for (const auto& [it, c] : l.coef) {
      if (it == skip) continue;
      const Range& r = resolved_[s].at(it);
      int64_t a = c * r.lo, b = c * (r.hi - 1);
      lo += std::min(a, b);
      hi += std::max(a, b);
    }
    return {lo, hi};
  }

  Range solve(const Lin& l, const std::string& u, int64_t extent, size_t s) const {
    auto [rlo, rhi] = rest(l, u, s);
    int64_t c = l.coef.at(u);
    Range r;
    if (c > 0) {  // 0 <= c*u + rest <= extent-1 for every rest
      r.lo = std::max<int64_t>(0, ceilDiv(-rlo, c));
      r.hi = floorDiv(extent - 1 - rhi, c) + 1;
    } else {
      int64_t m = -c;
      r.lo = std::max<int64_t>(0, ceilDiv(rhi - extent + 1, m));
      r.hi = floorDiv(rlo, m) + 1;
    }
    return r;
  }

  const lang::Validated& v_;
  std::map<std::string, int64_t>& sizes_;
  std::map<std::string, std::vector<int64_t>>& shapes_;
  std::vector<std::map<std::string, Range>> resolved_;
  std::vector<std::set<std::string>> iterSet_;
  std::vector<std::vector<Access>> acc_;
  std::map<std::string, std::vector<size_t>> writers_;
};

std::string subsKey(const std::vector<ExprP>& subs) {
  std::string k;
  for (const auto& s : subs) k += lang::printExpr(*s) + ";";
  return k;
}

void forEachAccess(const ExprP& e, const std::function<void(const Expr&)>& fn) {
  if (!e) return;
  if (e->k == EK::Access && !e->builtin) fn(*e);
  for (const auto& k : e->kids) forEachAccess(k, fn);
}

// checks.cc:166-181 — a statement may read its own LHS tensor only at the
// exact subscripts it writes.
void checkInPlace(const lang::Validated& v) {
  for (const auto& st : v.def.stmts) {
    std::string key = subsKey(st.idx);
    forEachAccess(st.rhs, [&](const Expr& a) {
      if (a.name == st.lhs && subsKey(a.kids) != key)
        fail(ErrorKind::LivenessInterference,
             "statement reads '" + a.name + "' at subscripts other than the ones it writes", a.pos);
    });
  }
}

// checks.cc:183-205 — temporaries must be written before they are read.
void checkSymbolicInit(const lang::Validated& v) {
  std::set<std::string> written;
  for (const auto& st : v.def.stmts) {
    auto need = [&](const std::string& t, SrcPos pos) {
      auto f = v.tensors.find(t);
      if (f == v.tensors.end() || f->second.role != Role::Temp) return;
      if (!written.count(t))
        fail(ErrorKind::UninitializedRead, "temporary '" + t + "' is read before any statement writes it", pos);
    };
    forEachAccess(st.rhs, [&](const Expr& a) { need(a.name, a.pos); });
    if (lang::isReduction(st.op) && !lang::hasInit(st.op)) need(st.lhs, st.pos);
    written.insert(st.lhs);
  }
}

}  // namespace

std::vector<std::string> opaqueReturns(const lang::Validated& v) {
  std::vector<std::string> out;
  for (const auto& r : v.def.rets) {
    const auto& t = v.tensors.at(r);
    if (t.read && !t.written) out.push_back(r);
  }
  return out;
}

std::vector<std::string> inoutReturns(const lang::Validated& v) {
  std::set<std::string> written, inout;
  for (const auto& st : v.def.stmts) {
    forEachAccess(st.rhs, [&](const Expr& a) {
      auto f = v.tensors.find(a.name);
      if (f != v.tensors.end() && f->second.role == Role::Output && !written.count(a.name)) inout.insert(a.name);
    });
    if (lang::isReduction(st.op) && !lang::hasInit(st.op) && !written.count(st.lhs)) inout.insert(st.lhs);
    written.insert(st.lhs);
  }
  std::vector<std::string> out;
  for (const auto& r : v.def.rets)
    if (inout.count(r)) out.push_back(r);
  return out;
}

Specialized specialize(const lang::Validated& v,
                       const std::map<std::string, std::vector<int64_t>>& provided) {
  checkInPlace(v);
  checkSymbolicInit(v);

  Specialized out;
  out.v = v;
  // bind size symbols from the declared dims of the provided parameters
  for (const auto& p : v.def.params) {
    if (p.scalar()) continue;
    auto f = provided.find(p.name);
    if (f == provided.end()) fail(ErrorKind::MissingBinding, "no shape provided for input '" + p.name + "'");
    if (f->second.size() != p.dims.size())
      fail(ErrorKind::ShapeMismatch, "input '" + p.name + "' has rank " + std::to_string(f->second.size()) +
                                          ", declared rank " + std::to_string(p.dims.size()));
    for (size_t d = 0; d < p.dims.size(); ++d) {
      int64_t e = f->second[d];
      if (e < 1) fail(ErrorKind::MissingBinding, "size symbol '" + p.dims[d] + "' bound to non-positive " + std::to_string(e));
      const std::string& sym = p.dims[d];
      if (numeric(sym)) {
        if (std::stoll(sym) != e)
          fail(ErrorKind::ShapeMismatch, "input '" + p.name + "' dimension " + std::to_string(d) + " is " +
                                              std::to_string(e) + ", declared " + sym);
        continue;
      }
      auto [it, fresh] = out.sizes.emplace(sym, e);
      if (!fresh && it->second != e)
        fail(ErrorKind::ShapeMismatch, "size symbol '" + sym + "' bound to both " + std::to_string(it->second) +
                                            " and " + std::to_string(e));
    }
    out.shapes[p.name] = f->second;
  }
  // opaque returns take the caller's extents (synthesized symbols R__d)
  for (const auto& r : opaqueReturns(v)) {
    auto f = provided.find(r);
    if (f == provided.end())
      fail(ErrorKind::MissingBinding, "size symbol '" + r + "__0' has no binding (return '" + r +
                                          "' is read but never written; pass its shape)");
    if (static_cast<int>(f->second.size()) != v.tensors.at(r).rank)
      fail(ErrorKind::ShapeMismatch, "return '" + r + "' has the wrong rank");
    for (size_t d = 0; d < f->second.size(); ++d) {
      if (f->second[d] < 1) fail(ErrorKind::MissingBinding, "extent of '" + r + "' must be positive");
      out.sizes[r + "__" + std::to_string(d)] = f->second[d];
    }
    out.shapes[r] = f->second;
  }

  std::vector<std::map<std::string, Range>> ranges = Inference(v, out.sizes, out.shapes).run();

  for (const auto& [t, dims] : out.shapes)
    for (size_t d = 0; d < dims.size(); ++d)
      if (dims[d] < 1)
        fail(ErrorKind::EmptyRange, "dimension " + std::to_string(d) + " of tensor '" + t + "' is empty at these sizes");
  // a provided in/out return must agree with the inferred shape
  for (const auto& [name, shp] : provided) {
    auto f = out.shapes.find(name);
    if (f != out.shapes.end() && f->second != shp)
      fail(ErrorKind::ShapeMismatch, "tensor '" + name + "' does not match the shape inferred at these sizes");
  }

  for (size_t s = 0; s < v.def.stmts.size(); ++s) {
    const lang::Stmt& src = v.def.stmts[s];
    if (lang::hasInit(src.op)) {
      CStmt init;
      init.stmt.lhs = src.lhs;
      init.stmt.idx = src.idx;
      init.stmt.op = lang::Op::Set;
      auto c = std::make_shared<Expr>();
      c->k = EK::Float;
      switch (src.op) {
        case lang::Op::AddInit: c->fval = 0.0; break;
        case lang::Op::MulInit: c->fval = 1.0; break;
        case lang::Op::MinInit: c->fval = std::numeric_limits<double>::infinity(); break;
        default: c->fval = -std::numeric_limits<double>::infinity(); break;
      }
      init.stmt.rhs = c;
      init.stmt.pos = src.pos;
      init.neutral = c->fval;
      for (const auto& ix : src.idx) {
        init.iters.push_back(ix->name);
        init.ranges[ix->name] = ranges[s].at(ix->name);
      }
      init.orig = s;
      init.synthInit = true;
      out.stmts.push_back(init);
    }
    CStmt cs;
    cs.stmt = src;
    cs.stmt.op = lang::dropInit(src.op);
    cs.iters = v.iters[s];
    cs.ranges = ranges[s];
    cs.orig = s;
    out.stmts.push_back(cs);
  }

  // checks.cc:319-350 — every affine access stays inside its tensor
  for (const auto& cs : out.stmts) {
    auto check = [&](const std::string& t, const std::vector<ExprP>& subs, SrcPos pos) {
      auto sh = out.shapes.find(t);
      if (sh == out.shapes.end()) return;
      for (size_t d = 0; d < subs.size() && d < sh->second.size(); ++d) {
        // concrete linearization over this statement's ranges
        std::function<std::optional<std::pair<int64_t, int64_t>>(const ExprP&)> ext =
            [&](const ExprP& e) -> std::optional<std::pair<int64_t, int64_t>> {
          switch (e->k) {
            case EK::Int: return std::make_pair(e->ival, e->ival);
            case EK::Ident: {
              auto r = cs.ranges.find(e->name);
              if (r != cs.ranges.end()) return std::make_pair(r->second.lo, r->second.hi - 1);
              auto z = out.sizes.find(e->name);
              if (z == out.sizes.end()) return std::nullopt;
              return std::make_pair(z->second, z->second);
            }
            case EK::DimOf: {
              auto f = out.shapes.find(e->name);
              if (f == out.shapes.end()) return std::nullopt;
              return std::make_pair(f->second[e->dim], f->second[e->dim]);
            }
            default: return std::nullopt;
          }
        };
        // affine walk with per-iterator coefficients (so i - i folds to 0)
        std::function<std::optional<Lin>(const ExprP&)> L = [&](const ExprP& e) -> std::optional<Lin> {
          switch (e->k) {
            case EK::Int: return Lin{{}, e->ival};
            case EK::Ident: {
              if (cs.ranges.count(e->name)) return Lin{{{e->name, 1}}, 0};
              auto z = out.sizes.find(e->name);
              if (z == out.sizes.end()) return std::nullopt;
              return Lin{{}, z->second};
            }
            case EK::DimOf: {
              auto x = ext(e);
              if (!x) return std::nullopt;
              return Lin{{}, x->first};
            }
            case EK::Unary: {
              if (e->op != "-") return std::nullopt;
              auto a = L(e->kids[0]);
              if (!a) return std::nullopt;
              for (auto& kv : a->coef) kv.second = -kv.second;
              a->cst = -a->cst;
              return a;
            }
            case EK::Binary: {
              auto a = L(e->kids[0]), b = L(e->kids[1]);
              if (!a || !b) return std::nullopt;
              if (e->op == "+" || e->op == "-") {
                int64_t sg = e->op == "-" ? -1 : 1;
                for (const auto& [it, c] : b->coef) {
                  a->coef[it] += sg * c;
                  if (a->coef[it] == 0) a->coef.erase(it);
                }
                a->cst += sg * b->cst;
                return a;
              }
              if (e->op == "*") {
                if (b->coef.empty()) {
                  for (auto& kv : a->coef) kv.second *= b->cst;
                  a->cst *= b->cst;
                  return a;
                }
                if (a->coef.empty()) {
                  for (auto& kv : b->coef) kv.second *= a->cst;
                  b->cst *= a->cst;
                  return b;
                }
              }
              return std::nullopt;
            }
            default: return std::nullopt;
          }
        };
        auto l = L(subs[d]);
        if (!l) continue;  // data-dependent; checked at run time
        int64_t lo = l->cst, hi = l->cst;
        for (const auto& [it, c] : l->coef) {
          const Range& r = cs.ranges.at(it);
          int64_t a = c * r.lo, b = c * (r.hi - 1);
          lo += std::min(a, b);
          hi += std::max(a, b);
        }
        if (lo < 0 || hi >= sh->second[d])
          fail(ErrorKind::OutOfBounds,
               "subscript " + lang::printExpr(*subs[d]) + " of '" + t + "' spans [" + std::to_string(lo) + ", " +
                   std::to_string(hi) + "] but dimension " + std::to_string(d) + " has extent " +
                   std::to_string(sh->second[d]),
               pos);
      }
    };
    check(cs.stmt.lhs, cs.stmt.idx, cs.stmt.pos);
    forEachAccess(cs.stmt.rhs, [&](const Expr& a) { check(a.name, a.kids, a.pos); });
  }
  return out;
}

}  // namespace sem
}  // namespace tcb
