// lang.h — the TC language front end of tc-b200: lexer, parser, printer,
// name validation.
//
// Surface grammar and diagnostics follow the reference front end
// (proj/src/lang/lexer.cc:161-382, parser.cc:66-209, validate.cc:38-365) so
// that any definition the reference accepts parses here to the same tree,
// and the pretty-printer reproduces the reference printer's text
// byte-for-byte (printer.cc:151-179) — the canonical cache key depends on it.
#pragma once

#include <map>
#include <memory>
#include <set>
#include <string>
#include <vector>

#include "common.h"

namespace tcb {
namespace lang {

enum class EK { Int, Float, Ident, Access, Unary, Binary, Ternary, DimOf };

struct Expr;
using ExprP = std::shared_ptr<Expr>;

struct Expr {
  EK k = EK::Int;
  SrcPos pos;
  int64_t ival = 0;
  double fval = 0;
  std::string name;  // Ident / Access / DimOf
  std::string op;    // Unary / Binary
  std::vector<ExprP> kids;
  int dim = 0;           // DimOf
  bool builtin = false;  // Access that validation classified as a builtin call
};

ExprP cloneExpr(const ExprP& e);

// Assignment operators; the *Init forms are the `op=!` spellings.
enum class Op { Set, Add, AddInit, Mul, MulInit, Min, MinInit, Max, MaxInit };
bool isReduction(Op op);
bool hasInit(Op op);
Op dropInit(Op op);
const char* opToken(Op op);

struct Where {
  std::string var;
  ExprP lo, hi;
  SrcPos pos;
};

struct Stmt {
  std::string lhs;
  std::vector<ExprP> idx;
  Op op = Op::Set;
  ExprP rhs;
  std::vector<Where> where;
  SrcPos pos;
  bool defCall = false;  // `(a,b) = f(...)` / `a = f(...)` (rejected by validation)
  std::vector<std::string> callResults;
};

enum class Elem { Float, Int };

struct Param {
  Elem elem = Elem::Float;
  std::vector<std::string> dims;  // empty ⇒ scalar
  std::string name;
  SrcPos pos;
  bool scalar() const { return dims.empty(); }
};

struct Def {
  std::string name;
  std::vector<Param> params;
  std::vector<std::string> rets;
  std::vector<Stmt> stmts;
  SrcPos pos;
  const Param* param(const std::string& n) const;
};

struct Program {
  std::vector<Def> defs;
  const Def* find(const std::string& n) const;
};

Program parse(const std::string& source);  // Error(Parse)

std::string printExpr(const Expr& e);
std::string printStmt(const Stmt& s);
std::string printDef(const Def& d);

// ---- name validation (validate.cc) ----
enum class Role { Input, Output, Temp };

struct TensorInfo {
  Elem elem = Elem::Float;
  int rank = -1;
  std::vector<std::string> dims;  // declared dims (inputs only)
  Role role = Role::Input;
  bool written = false, read = false;
};

struct Validated {
  Def def;
  std::map<std::string, TensorInfo> tensors;
  std::map<std::string, Elem> scalars;
  std::set<std::string> sizeSyms;
  // per statement: all index variables in first-use order (LHS first), and
  // the ones that appear only on the right-hand side
  std::vector<std::vector<std::string>> iters, redIters;
};

bool isBuiltin(const std::string& n);
Validated validate(const Def& def, const Program* siblings);  // Error(Name/UnsupportedCall)

// Picks the named def (or the only one).
const Def& selectDef(const Program& p, const std::string& name);

}  // namespace lang
}  // namespace tcb
