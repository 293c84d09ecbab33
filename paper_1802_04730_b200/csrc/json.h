// json.h — a small JSON value with a sorted-key object and a compact
// serializer. The output format is chosen to be byte-identical to the
// compact dump the reference stores use (sorted keys, no whitespace,
// minimal string escaping; options.cc:82-96, cache.cc:213-222), so option
// digests and cache files stay interchangeable.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

namespace tcb {

class Json {
 public:
  enum class T { Null, Bool, Int, UInt, Float, Str, Arr, Obj };

  Json() = default;
  Json(std::nullptr_t) {}
  Json(bool b) : t_(T::Bool), b_(b) {}
  Json(int v) : t_(T::Int), i_(v) {}
  Json(int64_t v) : t_(T::Int), i_(v) {}
  Json(uint64_t v) : t_(T::UInt), u_(v) {}
  Json(double v) : t_(T::Float), d_(v) {}
  Json(const char* s) : t_(T::Str), s_(s) {}
  Json(std::string s) : t_(T::Str), s_(std::move(s)) {}
  template <typename V>
  Json(const std::vector<V>& v) : t_(T::Arr) {
    for (const auto& x : v) a_.emplace_back(x);
  }

  static Json array() {
    Json j;
    j.t_ = T::Arr;
    return j;
  }
  static Json object() {
    Json j;
    j.t_ = T::Obj;
    return j;
  }
  static Json parse(const std::string& text);  // throws std::runtime_error

  T type() const { return t_; }
  bool isObj() const { return t_ == T::Obj; }
  bool isArr() const { return t_ == T::Arr; }
  bool isStr() const { return t_ == T::Str; }
  bool isBool() const { return t_ == T::Bool; }
  bool isInt() const { return t_ == T::Int || t_ == T::UInt; }

  // accessors throw std::runtime_error on a type mismatch
  bool asBool() const;
  int64_t asInt() const;
  uint64_t asUInt() const;
  const std::string& asStr() const;
  const std::vector<Json>& items() const;
  const std::map<std::string, Json>& fields() const;

  Json& operator[](const std::string& k);  // object insert/access
  const Json& at(const std::string& k) const;
  bool has(const std::string& k) const { return t_ == T::Obj && o_.count(k) != 0; }
  void push(Json v) {
    t_ = T::Arr;
    a_.push_back(std::move(v));
  }
  size_t size() const { return t_ == T::Arr ? a_.size() : o_.size(); }

  std::string dump() const;

 private:
  void dumpTo(std::string& out) const;
  T t_ = T::Null;
  bool b_ = false;
  int64_t i_ = 0;
  uint64_t u_ = 0;
  double d_ = 0;
  std::string s_;
  std::vector<Json> a_;
  std::map<std::string, Json> o_;
};

}  // namespace tcb
