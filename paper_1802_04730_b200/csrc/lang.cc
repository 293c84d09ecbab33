// lang.cc — lexer, recursive-descent parser, printer and name validation.
// See lang.h for the reference correspondences.
#include "lang.h"

#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdio>

namespace tcb {

std::string hex16(uint64_t v) {
  char b[17];
  std::snprintf(b, sizeof(b), "%016llx", static_cast<unsigned long long>(v));
  return b;
}

const char* errorKindName(ErrorKind k) {
  static const char* names[] = {
      "Parse",           "Name",
      "UnsupportedCall", "UnderConstrained",
      "Ambiguous",       "EmptyRange",
      "LivenessInterference", "OutOfBounds",
      "UninitializedRead", "InvalidSchedule",
      "NoParallelOuterBand", "NotSinkable",
      "MappingInvalid",  "PromotionBudget",
      "PromotionLogic",  "IndexOutOfRange",
      "RaceDetected",    "BarrierDivergence",
      "DegeneratePopulation", "NoViableCandidate",
      "CorruptStore",    "MissingBinding",
      "ShapeMismatch",   "Io",
      "Internal",        "NoKernel",
      "Cuda",
  };
  int i = static_cast<int>(k);
  return (i >= 0 && i < static_cast<int>(sizeof(names) / sizeof(names[0]))) ? names[i] : "?";
}

namespace lang {

ExprP cloneExpr(const ExprP& e) {
  if (!e) return nullptr;
  auto c = std::make_shared<Expr>(*e);
  for (auto& k : c->kids) k = cloneExpr(k);
  return c;
}

bool isReduction(Op op) { return op != Op::Set; }
bool hasInit(Op op) {
  return op == Op::AddInit || op == Op::MulInit || op == Op::MinInit || op == Op::MaxInit;
}
Op dropInit(Op op) {
  switch (op) {
    case Op::AddInit: return Op::Add;
    case Op::MulInit: return Op::Mul;
    case Op::MinInit: return Op::Min;
    case Op::MaxInit: return Op::Max;
    default: return op;
  }
}
const char* opToken(Op op) {
  switch (op) {
    case Op::Set: return "=";
    case Op::Add: return "+=";
    case Op::AddInit: return "+=!";
    case Op::Mul: return "*=";
    case Op::MulInit: return "*=!";
    case Op::Min: return "min=";
    case Op::MinInit: return "min=!";
    case Op::Max: return "max=";
    case Op::MaxInit: return "max=!";
  }
  return "=";
}

const Param* Def::param(const std::string& n) const {
  for (const auto& p : params)
    if (p.name == n) return &p;
  return nullptr;
}
const Def* Program::find(const std::string& n) const {
  for (const auto& d : defs)
    if (d.name == n) return &d;
  return nullptr;
}

// ============================================================== lexer ====
namespace {

enum class Tk {
  End, Id, IntLit, FloatLit, Def, Where, Float, Int,
  LPar, RPar, LBr, RBr, Comma, Arrow, Dot, Quest, Colon,
  Assign, AddEq, AddEqB, MulEq, MulEqB, MinEq, MinEqB, MaxEq, MaxEqB,
  Plus, Minus, Star, Slash, Not, Lt, Gt, Le, Ge, EqEq, Ne, And, Or,
};

const char* tkName(Tk t) {
  switch (t) {
    case Tk::End: return "end of input";
    case Tk::Id: return "identifier";
    case Tk::IntLit: return "integer literal";
    case Tk::FloatLit: return "float literal";
    case Tk::Def: return "'def'";
    case Tk::Where: return "'where'";
    case Tk::Float: return "'float'";
    case Tk::Int: return "'int'";
    case Tk::LPar: return "'('";
    case Tk::RPar: return "')'";
    case Tk::LBr: return "'{'";
    case Tk::RBr: return "'}'";
    case Tk::Comma: return "','";
    case Tk::Arrow: return "'->'";
    case Tk::Dot: return "'.'";
    case Tk::Quest: return "'?'";
    case Tk::Colon: return "':'";
    case Tk::Assign: return "'='";
    case Tk::AddEq: return "'+='";
    case Tk::AddEqB: return "'+=!'";
    case Tk::MulEq: return "'*='";
    case Tk::MulEqB: return "'*=!'";
    case Tk::MinEq: return "'min='";
    case Tk::MinEqB: return "'min=!'";
    case Tk::MaxEq: return "'max='";
    case Tk::MaxEqB: return "'max=!'";
    case Tk::Plus: return "'+'";
    case Tk::Minus: return "'-'";
    case Tk::Star: return "'*'";
    case Tk::Slash: return "'/'";
    case Tk::Not: return "'!'";
    case Tk::Lt: return "'<'";
    case Tk::Gt: return "'>'";
    case Tk::Le: return "'<='";
    case Tk::Ge: return "'>='";
    case Tk::EqEq: return "'=='";
    case Tk::Ne: return "'!='";
    case Tk::And: return "'&&'";
    case Tk::Or: return "'||'";
  }
  return "?";
}

struct Tok {
  Tk t = Tk::End;
  std::string text;
  int64_t i = 0;
  double f = 0;
  SrcPos pos;
};

bool wordChar(char c) { return std::isalnum(static_cast<unsigned char>(c)) || c == '_'; }
bool digit(char c) { return std::isdigit(static_cast<unsigned char>(c)) != 0; }

std::vector<Tok> tokenize(const std::string& s) {
  std::vector<Tok> out;
  size_t p = 0;
  uint32_t line = 1, col = 1;
  auto at = [&](size_t k) -> char { return p + k < s.size() ? s[p + k] : '\0'; };
  auto bump = [&]() -> char {
    char c = s[p++];
    if (c == '\n') {
      ++line;
      col = 1;
    } else {
      ++col;
    }
    return c;
  };
  auto emit = [&](Tk t, SrcPos pos, std::string text = {}) {
    Tok k;
    k.t = t;
    k.pos = pos;
    k.text = std::move(text);
    out.push_back(std::move(k));
  };
  while (p < s.size()) {
    char c = at(0);
    SrcPos pos{line, col};
    if (std::isspace(static_cast<unsigned char>(c))) {
      bump();
      continue;
    }
    if (c == '#') {
      while (p < s.size() && at(0) != '\n') bump();
      continue;
    }
    if (wordChar(c)) {
      std::string w;
      while (p < s.size() && wordChar(at(0))) w += bump();
      if (std::all_of(w.begin(), w.end(), digit)) {
        // number: the '.' joins only when a digit follows (so `A.0` lexes as
        // Id Dot Int), an exponent only when a digit (or sign+digit) follows
        bool fl = false;
        if (at(0) == '.' && digit(at(1))) {
          fl = true;
          w += bump();
          while (digit(at(0))) w += bump();
        }
        if ((at(0) == 'e' || at(0) == 'E') &&
            (digit(at(1)) || ((at(1) == '+' || at(1) == '-') && digit(at(2))))) {
          fl = true;
          w += bump();
          if (at(0) == '+' || at(0) == '-') w += bump();
          while (digit(at(0))) w += bump();
        }
        Tok k;
        k.pos = pos;
        k.text = w;
        if (fl) {
          k.t = Tk::FloatLit;
          k.f = std::stod(w);
        } else {
          k.t = Tk::IntLit;
          k.i = std::stoll(w);
        }
        out.push_back(k);
        continue;
      }
      if ((w == "min" || w == "max") && at(0) == '=' && at(1) != '=') {
        bump();
        bool bang = at(0) == '!';
        if (bang) bump();
        Tk t = w == "min" ? (bang ? Tk::MinEqB : Tk::MinEq) : (bang ? Tk::MaxEqB : Tk::MaxEq);
        emit(t, pos, w + (bang ? "=!" : "="));
        continue;
      }
      Tk t = Tk::Id;
      if (w == "def") t = Tk::Def;
      else if (w == "where") t = Tk::Where;
      else if (w == "float") t = Tk::Float;
      else if (w == "int") t = Tk::Int;
      emit(t, pos, w);
      continue;
    }
    bump();
    auto two = [&](char next, Tk yes, Tk no) {
      if (at(0) == next) {
        bump();
        emit(yes, pos);
      } else {
        emit(no, pos);
      }
    };
    switch (c) {
      case '(': emit(Tk::LPar, pos); break;
      case ')': emit(Tk::RPar, pos); break;
      case '{': emit(Tk::LBr, pos); break;
      case '}': emit(Tk::RBr, pos); break;
      case ',': emit(Tk::Comma, pos); break;
      case '.': emit(Tk::Dot, pos); break;
      case '?': emit(Tk::Quest, pos); break;
      case ':': emit(Tk::Colon, pos); break;
      case '/': emit(Tk::Slash, pos); break;
      case '+':
      case '*': {
        bool plus = c == '+';
        if (at(0) == '=') {
          bump();
          if (at(0) == '!') {
            bump();
            emit(plus ? Tk::AddEqB : Tk::MulEqB, pos);
          } else {
            emit(plus ? Tk::AddEq : Tk::MulEq, pos);
          }
        } else {
          emit(plus ? Tk::Plus : Tk::Star, pos);
        }
        break;
      }
      case '-': two('>', Tk::Arrow, Tk::Minus); break;
      case '=': two('=', Tk::EqEq, Tk::Assign); break;
      case '!': two('=', Tk::Ne, Tk::Not); break;
      case '<': two('=', Tk::Le, Tk::Lt); break;
      case '>': two('=', Tk::Ge, Tk::Gt); break;
      case '&':
        if (at(0) != '&') fail(ErrorKind::Parse, "stray '&'", pos);
        bump();
        emit(Tk::And, pos);
        break;
      case '|':
        if (at(0) != '|') fail(ErrorKind::Parse, "stray '|'", pos);
        bump();
        emit(Tk::Or, pos);
        break;
      default:
        fail(ErrorKind::Parse, std::string("unexpected character '") + c + "'", pos);
    }
  }
  Tok e;
  e.t = Tk::End;
  e.pos = {line, col};
  out.push_back(e);
  return out;
}

// ============================================================= parser ====
// Binary operator levels, loosest first; each level is left-associative.
struct Level {
  std::vector<std::pair<Tk, const char*>> ops;
};
const Level kLevels[] = {
    {{{Tk::Or, "||"}}},
    {{{Tk::And, "&&"}}},
    {{{Tk::EqEq, "=="}, {Tk::Ne, "!="}}},
    {{{Tk::Lt, "<"}, {Tk::Gt, ">"}, {Tk::Le, "<="}, {Tk::Ge, ">="}}},
    {{{Tk::Plus, "+"}, {Tk::Minus, "-"}}},
    {{{Tk::Star, "*"}, {Tk::Slash, "/"}}},
};
constexpr int kAdditiveLevel = 4;
constexpr int kNumLevels = 6;

class Parser {
 public:
  explicit Parser(const std::string& src) : toks_(tokenize(src)) {}

  Program program() {
    Program p;
    while (cur().t != Tk::End) p.defs.push_back(def());
    if (p.defs.empty()) fail(ErrorKind::Parse, "no def found in input", cur().pos);
    return p;
  }

 private:
  const Tok& cur() const { return toks_[i_]; }
  const Tok& ahead(size_t k) const { return toks_[std::min(i_ + k, toks_.size() - 1)]; }
  Tok take() { return toks_[i_++]; }
  bool eat(Tk t) {
    if (cur().t != t) return false;
    ++i_;
    return true;
  }
  Tok need(Tk t) {
    if (cur().t != t) {
      std::string m = std::string("expected ") + tkName(t) + ", got " + tkName(cur().t);
      if (!cur().text.empty()) m += " '" + cur().text + "'";
      fail(ErrorKind::Parse, m, cur().pos);
    }
    return take();
  }

  Def def() {
    Def d;
    d.pos = need(Tk::Def).pos;
    d.name = need(Tk::Id).text;
    need(Tk::LPar);
    if (cur().t != Tk::RPar) {
      do d.params.push_back(param());
      while (eat(Tk::Comma));
    }
    need(Tk::RPar);
    need(Tk::Arrow);
    need(Tk::LPar);
    do d.rets.push_back(need(Tk::Id).text);
    while (eat(Tk::Comma));
    need(Tk::RPar);
    need(Tk::LBr);
    while (cur().t != Tk::RBr) d.stmts.push_back(stmt());
    need(Tk::RBr);
    if (d.stmts.empty()) fail(ErrorKind::Parse, "def has no statements", d.pos);
    return d;
  }

  Param param() {
    Param p;
    p.pos = cur().pos;
    if (eat(Tk::Float)) p.elem = Elem::Float;
    else if (eat(Tk::Int)) p.elem = Elem::Int;
    else fail(ErrorKind::Parse, "expected parameter type 'float' or 'int'", cur().pos);
    if (eat(Tk::LPar)) {
      do p.dims.push_back(need(Tk::Id).text);
      while (eat(Tk::Comma));
      need(Tk::RPar);
    }
    p.name = need(Tk::Id).text;
    return p;
  }

  Stmt stmt() {
    Stmt s;
    s.pos = cur().pos;
    if (eat(Tk::LPar)) {  // (a, b) = callee(...)
      s.defCall = true;
      do s.callResults.push_back(need(Tk::Id).text);
      while (eat(Tk::Comma));
      need(Tk::RPar);
      need(Tk::Assign);
      s.rhs = primary();
      return s;
    }
    Tok lhs = need(Tk::Id);
    s.lhs = lhs.text;
    if (cur().t == Tk::Assign && ahead(1).t == Tk::Id && ahead(2).t == Tk::LPar) {
      take();  // a = callee(...)
      s.defCall = true;
      s.callResults.push_back(lhs.text);
      s.rhs = primary();
      return s;
    }
    need(Tk::LPar);
    if (cur().t != Tk::RPar) {
      do s.idx.push_back(expr());
      while (eat(Tk::Comma));
    }
    need(Tk::RPar);
    switch (cur().t) {
      case Tk::Assign: s.op = Op::Set; break;
      case Tk::AddEq: s.op = Op::Add; break;
      case Tk::AddEqB: s.op = Op::AddInit; break;
      case Tk::MulEq: s.op = Op::Mul; break;
      case Tk::MulEqB: s.op = Op::MulInit; break;
      case Tk::MinEq: s.op = Op::Min; break;
      case Tk::MinEqB: s.op = Op::MinInit; break;
      case Tk::MaxEq: s.op = Op::Max; break;
      case Tk::MaxEqB: s.op = Op::MaxInit; break;
      default: fail(ErrorKind::Parse, "expected an assignment operator", cur().pos);
    }
    take();
    s.rhs = expr();
    if (eat(Tk::Where)) {
      do {
        Where w;
        Tok v = need(Tk::Id);
        w.var = v.text;
        w.pos = v.pos;
        Tok kw = need(Tk::Id);
        if (kw.text != "in") fail(ErrorKind::Parse, "expected 'in' after range variable", kw.pos);
        w.lo = binary(kAdditiveLevel);
        need(Tk::Colon);
        w.hi = binary(kAdditiveLevel);
        s.where.push_back(std::move(w));
      } while (eat(Tk::Comma));
    }
    return s;
  }

  ExprP expr() {  // ternary, right-nested
    ExprP c = binary(0);
    if (cur().t != Tk::Quest) return c;
    SrcPos pos = take().pos;
    ExprP a = expr();
    need(Tk::Colon);
    ExprP b = expr();
    auto e = std::make_shared<Expr>();
    e->k = EK::Ternary;
    e->pos = pos;
    e->kids = {c, a, b};
    return e;
  }

  ExprP binary(int level) {
    if (level == kNumLevels) return unary();
    ExprP lhs = binary(level + 1);
    while (true) {
      const char* sym = nullptr;
      for (const auto& o : kLevels[level].ops)
        if (cur().t == o.first) sym = o.second;
      if (!sym) return lhs;
      SrcPos pos = take().pos;
      auto e = std::make_shared<Expr>();
      e->k = EK::Binary;
      e->op = sym;
      e->pos = pos;
      e->kids = {lhs, binary(level + 1)};
      lhs = e;
    }
  }

  ExprP unary() {
    if (cur().t == Tk::Minus || cur().t == Tk::Not) {
      auto e = std::make_shared<Expr>();
      e->k = EK::Unary;
      e->op = cur().t == Tk::Minus ? "-" : "!";
      e->pos = take().pos;
      e->kids = {unary()};
      return e;
    }
    return primary();
  }

  ExprP primary() {
    auto e = std::make_shared<Expr>();
    e->pos = cur().pos;
    if (cur().t == Tk::IntLit) {
      e->k = EK::Int;
      e->ival = take().i;
      return e;
    }
    if (cur().t == Tk::FloatLit) {
      e->k = EK::Float;
      e->fval = take().f;
      return e;
    }
    if (eat(Tk::LPar)) {
      ExprP inner = expr();
      need(Tk::RPar);
      return inner;
    }
    if (cur().t == Tk::Id) {
      e->name = take().text;
      if (eat(Tk::LPar)) {
        e->k = EK::Access;
        if (cur().t != Tk::RPar) {
          do e->kids.push_back(expr());
          while (eat(Tk::Comma));
        }
        need(Tk::RPar);
        return e;
      }
      if (cur().t == Tk::Dot && ahead(1).t == Tk::IntLit) {
        take();
        e->k = EK::DimOf;
        e->dim = static_cast<int>(take().i);
        return e;
      }
      e->k = EK::Ident;
      return e;
    }
    fail(ErrorKind::Parse, std::string("expected an expression, got ") + tkName(cur().t), cur().pos);
  }

  std::vector<Tok> toks_;
  size_t i_ = 0;
};

// ============================================================ printer ====
int prec(const Expr& e) {
  switch (e.k) {
    case EK::Ternary: return 1;
    case EK::Binary:
      if (e.op == "||") return 2;
      if (e.op == "&&") return 3;
      if (e.op == "==" || e.op == "!=") return 4;
      if (e.op == "<" || e.op == ">" || e.op == "<=" || e.op == ">=") return 5;
      if (e.op == "+" || e.op == "-") return 6;
      return 7;
    case EK::Unary: return 8;
    default: return 9;
  }
}

void printRec(std::string& o, const Expr& e, int parent) {
  int p = prec(e);
  bool par = p < parent;
  if (par) o += '(';
  switch (e.k) {
    case EK::Int: o += std::to_string(e.ival); break;
    case EK::Float: {
      // default ostream formatting (%g, precision 6); integral values get
      // a ".0" suffix (printer.cc:57-64)
      char b[64];
      std::snprintf(b, sizeof(b), "%g", e.fval);
      o += b;
      if (e.fval == std::floor(e.fval) && std::fabs(e.fval) < 1e15) o += ".0";
      break;
    }
    case EK::Ident: o += e.name; break;
    case EK::Access:
      o += e.name;
      o += '(';
      for (size_t i = 0; i < e.kids.size(); ++i) {
        if (i) o += ", ";
        printRec(o, *e.kids[i], 0);
      }
      o += ')';
      break;
    case EK::Unary:
      o += e.op;
      printRec(o, *e.kids[0], p);
      break;
    case EK::Binary:
      printRec(o, *e.kids[0], p);
      o += ' ';
      o += e.op;
      o += ' ';
      printRec(o, *e.kids[1], p + 1);
      break;
    case EK::Ternary:
      printRec(o, *e.kids[0], p + 1);
      o += " ? ";
      printRec(o, *e.kids[1], p + 1);
      o += " : ";
      printRec(o, *e.kids[2], p);
      break;
    case EK::DimOf:
      o += e.name + "." + std::to_string(e.dim);
      break;
  }
  if (par) o += ')';
}

}  // namespace

Program parse(const std::string& source) { return Parser(source).program(); }

std::string printExpr(const Expr& e) {
  std::string o;
  printRec(o, e, 0);
  return o;
}

std::string printStmt(const Stmt& s) {
  std::string o;
  if (s.defCall) {
    if (s.callResults.size() > 1) {
      o += '(';
      for (size_t i = 0; i < s.callResults.size(); ++i) o += (i ? ", " : "") + s.callResults[i];
      o += ')';
    } else {
      o += s.callResults.front();
    }
    return o + " = " + printExpr(*s.rhs);
  }
  o += s.lhs + "(";
  for (size_t i = 0; i < s.idx.size(); ++i) {
    if (i) o += ", ";
    o += printExpr(*s.idx[i]);
  }
  o += ") ";
  o += opToken(s.op);
  o += " " + printExpr(*s.rhs);
  if (!s.where.empty()) {
    o += " where ";
    for (size_t i = 0; i < s.where.size(); ++i) {
      if (i) o += ", ";
      o += s.where[i].var + " in " + printExpr(*s.where[i].lo) + ":" + printExpr(*s.where[i].hi);
    }
  }
  return o;
}

std::string printDef(const Def& d) {
  std::string o = "def " + d.name + "(";
  for (size_t i = 0; i < d.params.size(); ++i) {
    const Param& p = d.params[i];
    if (i) o += ", ";
    o += p.elem == Elem::Float ? "float" : "int";
    if (!p.dims.empty()) {
      o += '(';
      for (size_t k = 0; k < p.dims.size(); ++k) o += (k ? "," : "") + p.dims[k];
      o += ')';
    }
    o += " " + p.name;
  }
  o += ") -> (";
  for (size_t i = 0; i < d.rets.size(); ++i) o += (i ? ", " : "") + d.rets[i];
  o += ") {\n";
  for (const auto& s : d.stmts) o += "  " + printStmt(s) + "\n";
  o += "}\n";
  return o;
}

// ========================================================= validation ====
namespace {

struct Builtin {
  const char* name;
  int arity;
};
const Builtin kBuiltins[] = {{"fmaxf", 2}, {"fminf", 2}, {"exp", 1},  {"log", 1},
                             {"tanh", 1},  {"sigmoid", 1}, {"abs", 1}};

int arityOf(const std::string& n) {
  for (const auto& b : kBuiltins)
    if (n == b.name) return b.arity;
  return -1;
}

class Validator {
 public:
  Validator(const Def& d, const Program* sib) : sib_(sib) { v_.def = d; }

  Validated run() {
    declare();
    for (auto& s : v_.def.stmts) stmt(s);
    for (const auto& [n, t] : v_.tensors) {
      if (t.role == Role::Output && !t.written && !t.read)
        fail(ErrorKind::Name, "return '" + n + "' is never defined or used", v_.def.pos);
      if (t.role == Role::Temp && !t.written)
        fail(ErrorKind::Name, "temporary '" + n + "' is read but never defined", v_.def.pos);
    }
    return std::move(v_);
  }

 private:
  bool isTensor(const std::string& n) const { return v_.tensors.count(n) != 0; }
  bool isScalar(const std::string& n) const { return v_.scalars.count(n) != 0; }
  bool isSize(const std::string& n) const { return v_.sizeSyms.count(n) != 0; }

  void declare() {
    std::set<std::string> seen;
    for (const Param& p : v_.def.params) {
      if (!seen.insert(p.name).second) fail(ErrorKind::Name, "duplicate parameter '" + p.name + "'", p.pos);
      if (p.scalar()) {
        v_.scalars[p.name] = p.elem;
        continue;
      }
      TensorInfo t;
      t.elem = p.elem;
      t.rank = static_cast<int>(p.dims.size());
      t.dims = p.dims;
      t.role = Role::Input;
      v_.tensors[p.name] = t;
      for (const auto& d : p.dims) v_.sizeSyms.insert(d);
    }
    for (const auto& r : v_.def.rets) {
      if (!seen.insert(r).second) fail(ErrorKind::Name, "return '" + r + "' shadows a parameter", v_.def.pos);
      TensorInfo t;
      t.elem = Elem::Float;
      t.role = Role::Output;
      v_.tensors[r] = t;
    }
  }

  TensorInfo& tensor(const std::string& n, SrcPos pos) {
    auto it = v_.tensors.find(n);
    if (it != v_.tensors.end()) return it->second;
    if (sib_ && sib_->find(n))
      fail(ErrorKind::UnsupportedCall,
           "'" + n + "' is another def; defs cannot call other defs, inline the computation instead", pos);
    fail(ErrorKind::Name, "unknown tensor '" + n + "'", pos);
  }

  void use(const std::string& n, int rank, bool write, SrcPos pos) {
    TensorInfo& t = tensor(n, pos);
    if (t.rank < 0) {
      t.rank = rank;
    } else if (t.rank != rank) {
      fail(ErrorKind::Name,
           "tensor '" + n + "' used with " + std::to_string(rank) + " subscripts but has rank " +
               std::to_string(t.rank),
           pos);
    }
    if (write) {
      if (t.role == Role::Input) fail(ErrorKind::Name, "cannot write to input parameter '" + n + "'", pos);
      t.written = true;
    } else {
      t.read = true;
    }
  }

  void stmt(Stmt& s) {
    if (s.defCall)
      fail(ErrorKind::UnsupportedCall,
           "defs cannot call other defs; '" + (s.rhs ? s.rhs->name : std::string("?")) + "' must be inlined",
           s.pos);
    if (!isTensor(s.lhs)) {
      if (isScalar(s.lhs) || isSize(s.lhs)) fail(ErrorKind::Name, "'" + s.lhs + "' is not a tensor", s.pos);
      TensorInfo t;
      t.role = Role::Temp;
      v_.tensors[s.lhs] = t;
    }
    std::vector<std::string> iters;
    auto note = [&](const std::string& n) {
      if (std::find(iters.begin(), iters.end(), n) == iters.end()) iters.push_back(n);
    };
    std::set<std::string> lhsIters;
    for (const auto& ix : s.idx) {
      if (ix->k != EK::Ident) fail(ErrorKind::Name, "left-hand side subscripts must be plain iterators", ix->pos);
      if (isScalar(ix->name) || isSize(ix->name) || isTensor(ix->name))
        fail(ErrorKind::Name, "left-hand side subscript '" + ix->name + "' is not an iterator", ix->pos);
      note(ix->name);
      lhsIters.insert(ix->name);
    }
    use(s.lhs, static_cast<int>(s.idx.size()), true, s.pos);
    expr(*s.rhs, false, note);
    for (const auto& w : s.where) {
      if (std::find(iters.begin(), iters.end(), w.var) == iters.end())
        fail(ErrorKind::Name, "where clause constrains '" + w.var + "' which is not used in the statement", w.pos);
      bound(*w.lo);
      bound(*w.hi);
    }
    std::vector<std::string> red;
    for (const auto& it : iters)
      if (!lhsIters.count(it)) red.push_back(it);
    v_.iters.push_back(iters);
    v_.redIters.push_back(red);
  }

  template <typename Note>
  void expr(Expr& e, bool inSub, Note& note) {
    switch (e.k) {
      case EK::Int:
      case EK::Float: return;
      case EK::Ident:
        if (isTensor(e.name)) fail(ErrorKind::Name, "tensor '" + e.name + "' used without subscripts", e.pos);
        if (isScalar(e.name)) {
          if (inSub && v_.scalars[e.name] != Elem::Int)
            fail(ErrorKind::Name, "float scalar '" + e.name + "' cannot appear in a subscript", e.pos);
          return;
        }
        if (isSize(e.name)) return;
        note(e.name);
        return;
      case EK::Access: {
        int ar = arityOf(e.name);
        if (ar >= 0) {
          if (isTensor(e.name)) fail(ErrorKind::Name, "'" + e.name + "' is both a tensor and a builtin", e.pos);
          e.builtin = true;
          if (static_cast<int>(e.kids.size()) != ar)
            fail(ErrorKind::Name,
                 "builtin '" + e.name + "' takes " + std::to_string(ar) + " argument(s), got " +
                     std::to_string(e.kids.size()),
                 e.pos);
          for (auto& k : e.kids) expr(*k, false, note);
          return;
        }
        use(e.name, static_cast<int>(e.kids.size()), false, e.pos);
        for (auto& k : e.kids) expr(*k, true, note);
        return;
      }
      case EK::Unary: expr(*e.kids[0], inSub, note); return;
      case EK::Binary:
        expr(*e.kids[0], inSub, note);
        expr(*e.kids[1], inSub, note);
        return;
      case EK::Ternary:
        for (auto& k : e.kids) expr(*k, inSub, note);
        return;
      case EK::DimOf: {
        TensorInfo& t = tensor(e.name, e.pos);
        if (t.rank >= 0 && (e.dim < 0 || e.dim >= t.rank))
          fail(ErrorKind::Name,
               "dimension " + std::to_string(e.dim) + " out of range for rank-" + std::to_string(t.rank) +
                   " tensor '" + e.name + "'",
               e.pos);
        return;
      }
    }
  }

  void bound(const Expr& e) {
    switch (e.k) {
      case EK::Int:
      case EK::DimOf: return;
      case EK::Ident:
        if (isSize(e.name)) return;
        if (isScalar(e.name)) {
          if (v_.scalars[e.name] != Elem::Int)
            fail(ErrorKind::Name, "float scalar '" + e.name + "' cannot bound a range", e.pos);
          return;
        }
        fail(ErrorKind::Name, "range bounds may only use size symbols and constants, not '" + e.name + "'", e.pos);
      case EK::Binary:
        if (e.op == "+" || e.op == "-" || e.op == "*" || e.op == "/") {
          bound(*e.kids[0]);
          bound(*e.kids[1]);
          return;
        }
        break;
      case EK::Unary:
        if (e.op == "-") {
          bound(*e.kids[0]);
          return;
        }
        break;
      default: break;
    }
    fail(ErrorKind::Name, "unsupported expression in range bound", e.pos);
  }

  Validated v_;
  const Program* sib_;
};

}  // namespace

bool isBuiltin(const std::string& n) { return arityOf(n) >= 0; }

Validated validate(const Def& def, const Program* siblings) { return Validator(def, siblings).run(); }

const Def& selectDef(const Program& p, const std::string& name) {
  if (name.empty()) {
    if (p.defs.size() != 1)
      fail(ErrorKind::Name, "buffer holds " + std::to_string(p.defs.size()) + " defs; name the entry point");
    return p.defs.front();
  }
  const Def* d = p.find(name);
  if (!d) fail(ErrorKind::Name, "no def named '" + name + "' in buffer");
  return *d;
}

}  // namespace lang
}  // namespace tcb
