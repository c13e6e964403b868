// Minimal JSON value / parser / writer for the planner's host-side interface (no dependencies).
#pragma once
#include <cstdio>
#include <map>
#include <memory>
#include <stdexcept>
#include <cmath>
#include <string>
#include <vector>

namespace fcm {
namespace json {

struct Value {
  enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
  bool b = false;
  double n = 0;
  std::string s;
  std::vector<Value> a;
  std::vector<std::pair<std::string, Value>> o;

  const Value* get(const std::string& k) const {
    for (auto& kv : o)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
  double num(const std::string& k, double dflt) const {
    const Value* v = get(k);
    return (v && v->kind == Num) ? v->n : dflt;
  }
  std::string str(const std::string& k, const std::string& dflt) const {
    const Value* v = get(k);
    return (v && v->kind == Str) ? v->s : dflt;
  }
};

class Parser {
 public:
  explicit Parser(const char* p) : p_(p) {}
  Value parse() {
    Value v = value();
    ws();
    if (*p_) throw std::runtime_error("trailing characters in JSON");
    return v;
  }

 private:
  const char* p_;
  void ws() {
    while (*p_ == ' ' || *p_ == '\n' || *p_ == '\t' || *p_ == '\r') ++p_;
  }
  Value value() {
    ws();
    Value v;
    if (*p_ == '{') {
      v.kind = Value::Obj;
      ++p_;
      ws();
      if (*p_ == '}') { ++p_; return v; }
      for (;;) {
        ws();
        std::string k = string();
        ws();
        if (*p_++ != ':') throw std::runtime_error("expected ':'");
        v.o.emplace_back(k, value());
        ws();
        if (*p_ == ',') { ++p_; continue; }
        if (*p_ == '}') { ++p_; break; }
        throw std::runtime_error("expected ',' or '}'");
      }
    } else if (*p_ == '[') {
      v.kind = Value::Arr;
      ++p_;
      ws();
      if (*p_ == ']') { ++p_; return v; }
      for (;;) {
        v.a.push_back(value());
        ws();
        if (*p_ == ',') { ++p_; continue; }
        if (*p_ == ']') { ++p_; break; }
        throw std::runtime_error("expected ',' or ']'");
      }
    } else if (*p_ == '"') {
      v.kind = Value::Str;
      v.s = string();
    } else if (!strncmp_(p_, "true")) {
      v.kind = Value::Bool; v.b = true; p_ += 4;
    } else if (!strncmp_(p_, "false")) {
      v.kind = Value::Bool; p_ += 5;
    } else if (!strncmp_(p_, "null")) {
      p_ += 4;
    } else {
      char* end = nullptr;
      v.n = strtod(p_, &end);
      if (end == p_) throw std::runtime_error("bad JSON value");
      if (!std::isfinite(v.n)) throw std::runtime_error("non-finite JSON number");
      v.kind = Value::Num;
      p_ = end;
    }
    return v;
  }
  static int strncmp_(const char* a, const char* lit) {
    for (; *lit; ++a, ++lit)
      if (*a != *lit) return 1;
    return 0;
  }
  std::string string() {
    if (*p_ != '"') throw std::runtime_error("expected string");
    ++p_;
    std::string r;
    while (*p_ && *p_ != '"') {
      if (*p_ == '\\') {
        ++p_;
        if (!*p_) break;  // a backslash right before the terminator: unterminated (never read past NUL)
        char c = *p_++;
        r.push_back(c == 'n' ? '\n' : c == 't' ? '\t' : c);
      } else {
        r.push_back(*p_++);
      }
    }
    if (*p_ != '"') throw std::runtime_error("unterminated string");
    ++p_;
    return r;
  }
};

inline std::string quote(const std::string& s) {
  std::string r = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') r.push_back('\\');
    r.push_back(c);
  }
  return r + "\"";
}

inline std::string num(double d) {
  char buf[64];
  if (!std::isfinite(d)) throw std::runtime_error("non-finite number in JSON output");
  if (d < 9e15 && d > -9e15 && d == static_cast<double>(static_cast<long long>(d)))
    snprintf(buf, sizeof buf, "%lld", static_cast<long long>(d));
  else
    snprintf(buf, sizeof buf, "%.17g", d);
  return buf;
}

}  // namespace json
}  // namespace fcm
