#include "json.h"

#include <cmath>
#include <cstdio>
#include <stdexcept>

namespace tcb {

namespace {

[[noreturn]] void bad(const std::string& m) { throw std::runtime_error("json: " + m); }

void escapeTo(std::string& out, const std::string& s) {
  out += '"';
  for (unsigned char c : s) {
    switch (c) {
      case '"': out += "\\\""; break;
      case '\\': out += "\\\\"; break;
      case '\b': out += "\\b"; break;
      case '\f': out += "\\f"; break;
      case '\n': out += "\\n"; break;
      case '\r': out += "\\r"; break;
      case '\t': out += "\\t"; break;
      default:
        if (c < 0x20) {
          char buf[8];
          std::snprintf(buf, sizeof(buf), "\\u%04x", c);
          out += buf;
        } else {
          out += static_cast<char>(c);
        }
    }
  }
  out += '"';
}

class Reader {
 public:
  explicit Reader(const std::string& s) : s_(s) {}

  Json value() {
    ws();
    if (p_ >= s_.size()) bad("unexpected end of input");
    char c = s_[p_];
    if (c == '{') return object();
    if (c == '[') return array();
    if (c == '"') return Json(string());
    if (c == 't') return lit("true", Json(true));
    if (c == 'f') return lit("false", Json(false));
    if (c == 'n') return lit("null", Json());
    return number();
  }

  void end() {
    ws();
    if (p_ != s_.size()) bad("trailing characters");
  }

 private:
  void ws() {
    while (p_ < s_.size() && (s_[p_] == ' ' || s_[p_] == '\n' || s_[p_] == '\t' || s_[p_] == '\r')) ++p_;
  }
  void expect(char c) {
    ws();
    if (p_ >= s_.size() || s_[p_] != c) bad(std::string("expected '") + c + "'");
    ++p_;
  }
  Json lit(const char* word, Json v) {
    size_t n = std::char_traits<char>::length(word);
    if (s_.compare(p_, n, word) != 0) bad("bad literal");
    p_ += n;
    return v;
  }
  Json object() {
    Json o = Json::object();
    expect('{');
    ws();
    if (p_ < s_.size() && s_[p_] == '}') {
      ++p_;
      return o;
    }
    while (true) {
      ws();
      std::string k = string();
      expect(':');
      o[k] = value();
      ws();
      if (p_ < s_.size() && s_[p_] == ',') {
        ++p_;
        continue;
      }
      expect('}');
      return o;
    }
  }
  Json array() {
    Json a = Json::array();
    expect('[');
    ws();
    if (p_ < s_.size() && s_[p_] == ']') {
      ++p_;
      return a;
    }
    while (true) {
      a.push(value());
      ws();
      if (p_ < s_.size() && s_[p_] == ',') {
        ++p_;
        continue;
      }
      expect(']');
      return a;
    }
  }
  std::string string() {
    if (p_ >= s_.size() || s_[p_] != '"') bad("expected string");
    ++p_;
    std::string out;
    while (true) {
      if (p_ >= s_.size()) bad("unterminated string");
      char c = s_[p_++];
      if (c == '"') return out;
      if (c != '\\') {
        out += c;
        continue;
      }
      if (p_ >= s_.size()) bad("bad escape");
      char e = s_[p_++];
      switch (e) {
        case '"': out += '"'; break;
        case '\\': out += '\\'; break;
        case '/': out += '/'; break;
        case 'b': out += '\b'; break;
        case 'f': out += '\f'; break;
        case 'n': out += '\n'; break;
        case 'r': out += '\r'; break;
        case 't': out += '\t'; break;
        case 'u': {
          if (p_ + 4 > s_.size()) bad("bad \\u escape");
          unsigned cp = std::stoul(s_.substr(p_, 4), nullptr, 16);
          p_ += 4;
          if (cp < 0x80) {
            out += static_cast<char>(cp);
          } else if (cp < 0x800) {
            out += static_cast<char>(0xC0 | (cp >> 6));
            out += static_cast<char>(0x80 | (cp & 0x3F));
          } else {
            out += static_cast<char>(0xE0 | (cp >> 12));
            out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
            out += static_cast<char>(0x80 | (cp & 0x3F));
          }
          break;
        }
        default: bad("bad escape");
      }
    }
  }
  Json number() {
    size_t start = p_;
    bool isFloat = false;
    if (s_[p_] == '-') ++p_;
    while (p_ < s_.size()) {
      char c = s_[p_];
      if (c >= '0' && c <= '9') {
        ++p_;
      } else if (c == '.' || c == 'e' || c == 'E' || c == '+' || c == '-') {
        isFloat = true;
        ++p_;
      } else {
        break;
      }
    }
    std::string t = s_.substr(start, p_ - start);
    if (t.empty() || t == "-") bad("bad number");
    try {
      if (isFloat) return Json(std::stod(t));
      if (t[0] == '-') return Json(static_cast<int64_t>(std::stoll(t)));
      uint64_t u = std::stoull(t);
      if (u <= static_cast<uint64_t>(INT64_MAX)) return Json(static_cast<int64_t>(u));
      return Json(u);
    } catch (const std::exception&) {
      bad("number out of range");
    }
  }

  const std::string& s_;
  size_t p_ = 0;
};

}  // namespace

Json Json::parse(const std::string& text) {
  Reader r(text);
  Json v = r.value();
  r.end();
  return v;
}

bool Json::asBool() const {
  if (t_ != T::Bool) bad("not a boolean");
  return b_;
}
int64_t Json::asInt() const {
  if (t_ == T::Int) return i_;
  if (t_ == T::UInt && u_ <= static_cast<uint64_t>(INT64_MAX)) return static_cast<int64_t>(u_);
  bad("not an integer");
}
uint64_t Json::asUInt() const {
  if (t_ == T::UInt) return u_;
  if (t_ == T::Int && i_ >= 0) return static_cast<uint64_t>(i_);
  bad("not an unsigned integer");
}
const std::string& Json::asStr() const {
  if (t_ != T::Str) bad("not a string");
  return s_;
}
const std::vector<Json>& Json::items() const {
  if (t_ != T::Arr) bad("not an array");
  return a_;
}
const std::map<std::string, Json>& Json::fields() const {
  if (t_ != T::Obj) bad("not an object");
  return o_;
}
Json& Json::operator[](const std::string& k) {
  if (t_ == T::Null) t_ = T::Obj;
  if (t_ != T::Obj) bad("not an object");
  return o_[k];
}
const Json& Json::at(const std::string& k) const {
  if (t_ != T::Obj) bad("not an object");
  auto it = o_.find(k);
  if (it == o_.end()) bad("missing field '" + k + "'");
  return it->second;
}

void Json::dumpTo(std::string& out) const {
  switch (t_) {
    case T::Null: out += "null"; break;
    case T::Bool: out += b_ ? "true" : "false"; break;
    case T::Int: out += std::to_string(i_); break;
    case T::UInt: out += std::to_string(u_); break;
    case T::Float: {
      char buf[32];
      std::snprintf(buf, sizeof(buf), "%.17g", d_);
      out += buf;
      break;
    }
    case T::Str: escapeTo(out, s_); break;
    case T::Arr: {
      out += '[';
      for (size_t i = 0; i < a_.size(); ++i) {
        if (i) out += ',';
        a_[i].dumpTo(out);
      }
      out += ']';
      break;
    }
    case T::Obj: {
      out += '{';
      bool first = true;
      for (const auto& kv : o_) {
        if (!first) out += ',';
        first = false;
        escapeTo(out, kv.first);
        out += ':';
        kv.second.dumpTo(out);
      }
      out += '}';
      break;
    }
  }
}

std::string Json::dump() const {
  std::string out;
  dumpTo(out);
  return out;
}

}  // namespace tcb
