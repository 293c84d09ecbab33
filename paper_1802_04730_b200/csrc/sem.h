// sem.h — shape binding, range inference and specialization.
//
// tc-b200 compiles for exact shapes (the caller's tensors are known at
// compile time), so inference runs on concrete integers rather than the
// reference's symbolic SizeExpr (proj/src/sem/ranges.cc:445-595). The
// algorithm is the same: rounds to a fixpoint; inside a round every
// affine subscript with exactly one unresolved iterator proposes the
// interval that keeps the subscript inside the accessed extent for every
// value of the already-resolved iterators; `where` clauses propose their
// interval; same-round proposals intersect; lower bounds clamp to 0; a
// written tensor takes the upper bounds of its first fully-resolved
// writer's LHS iterators. Specialization then desugars `op=!` into a
// neutral-element store + plain reduction (specialize.cc:118-138).
#pragma once

#include <map>
#include <string>
#include <vector>

#include "lang.h"

namespace tcb {
namespace sem {

struct Range {
  int64_t lo = 0, hi = 0;  // half-open
  int64_t extent() const { return hi - lo; }
};

struct CStmt {
  lang::Stmt stmt;                 // op has its init stripped
  std::vector<std::string> iters;  // canonical loop order, LHS first
  std::map<std::string, Range> ranges;
  size_t orig = 0;
  bool synthInit = false;  // the neutral store of a desugared `op=!`
  double neutral = 0;      // its value
  const Range& range(const std::string& it) const;
};

struct Specialized {
  lang::Validated v;
  std::map<std::string, int64_t> sizes;
  std::map<std::string, std::vector<int64_t>> shapes;  // every tensor
  std::vector<CStmt> stmts;
};

// `provided` holds the shapes of the caller's tensors: every tensor
// parameter, and every return that is read before being written (it is
// in/out and its extents are otherwise unknowable — ranges.cc:458-466).
// Errors: MissingBinding (a needed shape absent), ShapeMismatch (one size
// symbol bound to two values, a rank or literal extent mismatch),
// UnderConstrained / Ambiguous / EmptyRange (inference), OutOfBounds
// (checks.cc:319-350), LivenessInterference (checks.cc:166-181),
// UninitializedRead (checks.cc:183-205).
Specialized specialize(const lang::Validated& v,
                       const std::map<std::string, std::vector<int64_t>>& provided);

// Returns that the definition reads before any statement writes them —
// these must be supplied by the caller (C3's `+=` target, MLP3's O1).
std::vector<std::string> inoutReturns(const lang::Validated& v);
// Returns read but never written (their shapes must be provided).
std::vector<std::string> opaqueReturns(const lang::Validated& v);

}  // namespace sem
}  // namespace tcb
