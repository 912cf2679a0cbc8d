// json_mini.hpp -- a small strict JSON reader for the reference's
// configuration objects (b3d_scene_from_json, b3d_infer config, library
// manifests) and a compact writer; the reference uses nlohmann::json, which
// this image does not ship.  Numbers are parsed with strtod and written as
// nlohmann's dump writes them (shortest round-trip digits); object keys keep
// their order.
#pragma once

#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace b3d200 {
namespace json {

struct Value {
  enum Kind { Null, Bool, Number, String, Array, Object } kind = Null;
  bool b = false;
  double num = 0;
  bool integral = false;  // written without fraction / exponent
  std::string str;
  std::vector<Value> arr;
  std::vector<std::pair<std::string, Value>> obj;

  bool is_object() const { return kind == Object; }
  bool is_array() const { return kind == Array; }
  const Value* find(const std::string& k) const {
    for (const auto& kv : obj)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
};

struct ParseError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

class Parser {
 public:
  explicit Parser(const std::string& s) : s_(s) {}
  Value parse() {
    Value v = value();
    ws();
    if (i_ != s_.size()) throw ParseError("trailing characters");
    return v;
  }

 private:
  const std::string& s_;
  size_t i_ = 0;
  void ws() {
    while (i_ < s_.size() && (s_[i_] == ' ' || s_[i_] == '\t' || s_[i_] == '\n' || s_[i_] == '\r'))
      ++i_;
  }
  bool eat(char c) {
    ws();
    if (i_ < s_.size() && s_[i_] == c) {
      ++i_;
      return true;
    }
    return false;
  }
  void expect(char c) {
    if (!eat(c)) throw ParseError(std::string("expected '") + c + "'");
  }
  Value value() {
    ws();
    if (i_ >= s_.size()) throw ParseError("unexpected end");
    const char c = s_[i_];
    Value v;
    if (c == '{') {
      ++i_;
      v.kind = Value::Object;
      if (eat('}')) return v;
      do {
        ws();
        std::string k = string();
        expect(':');
        v.obj.emplace_back(std::move(k), value());
      } while (eat(','));
      expect('}');
    } else if (c == '[') {
      ++i_;
      v.kind = Value::Array;
      if (eat(']')) return v;
      do v.arr.push_back(value());
      while (eat(','));
      expect(']');
    } else if (c == '"') {
      v.kind = Value::String;
      v.str = string();
    } else if (s_.compare(i_, 4, "true") == 0) {
      i_ += 4;
      v.kind = Value::Bool;
      v.b = true;
    } else if (s_.compare(i_, 5, "false") == 0) {
      i_ += 5;
      v.kind = Value::Bool;
    } else if (s_.compare(i_, 4, "null") == 0) {
      i_ += 4;
    } else {
      const char* b = s_.c_str() + i_;
      char* e = nullptr;
      v.num = std::strtod(b, &e);
      if (e == b) throw ParseError("invalid value");
      v.kind = Value::Number;
      v.integral = true;
      for (const char* q = b; q < e; ++q)
        if (*q == '.' || *q == 'e' || *q == 'E') v.integral = false;
      i_ += (size_t)(e - b);
    }
    return v;
  }
  std::string string() {
    if (i_ >= s_.size() || s_[i_] != '"') throw ParseError("expected a string");
    ++i_;
    std::string out;
    while (i_ < s_.size() && s_[i_] != '"') {
      char c = s_[i_++];
      if (c == '\\') {
        if (i_ >= s_.size()) break;
        const char e = s_[i_++];
        switch (e) {
          case 'n': c = '\n'; break;
          case 't': c = '\t'; break;
          case 'r': c = '\r'; break;
          case 'b': c = '\b'; break;
          case 'f': c = '\f'; break;
          case 'u': {
            if (i_ + 4 > s_.size()) throw ParseError("bad escape");
            const unsigned cp = (unsigned)std::strtoul(s_.substr(i_, 4).c_str(), nullptr, 16);
            i_ += 4;
            if (cp < 0x80) {
              c = (char)cp;
            } else {  // UTF-8 (BMP only)
              if (cp < 0x800) {
                out += (char)(0xC0 | (cp >> 6));
              } else {
                out += (char)(0xE0 | (cp >> 12));
                out += (char)(0x80 | ((cp >> 6) & 0x3F));
              }
              c = (char)(0x80 | (cp & 0x3F));
            }
            break;
          }
          default: c = e;
        }
      }
      out += c;
    }
    if (i_ >= s_.size()) throw ParseError("unterminated string");
    ++i_;
    return out;
  }
};

inline Value parse(const std::string& s) { return Parser(s).parse(); }

// A double as nlohmann::json::dump writes it: the shortest digits that read
// back to the same value (std::to_chars; nlohmann's Grisu2 agrees except in
// rare cases where Grisu2 is one digit longer), fixed notation for decimal
// exponents in (-4, 15] with ".0" on integral values, else d.ddde+XX;
// "null" for non-finite values.
inline std::string num(double x) {
  if (!std::isfinite(x)) return "null";
  std::string out = std::signbit(x) ? "-" : "";
  if (x == 0) return out + "0.0";
  char buf[64];
  const auto r = std::to_chars(buf, buf + sizeof buf, std::fabs(x), std::chars_format::scientific);
  const std::string s(buf, r.ptr);  // d[.ddd]e(+|-)XX
  const size_t epos = s.find('e');
  std::string digits = s.substr(0, 1) + (epos > 2 ? s.substr(2, epos - 2) : std::string());
  const int k = (int)digits.size();
  const int n = std::atoi(s.c_str() + epos + 1) + 1;  // digits before the decimal point
  if (k <= n && n <= 15) {
    out += digits + std::string(n - k, '0') + ".0";
  } else if (0 < n && n <= 15) {
    out += digits.substr(0, n) + "." + digits.substr(n);
  } else if (-4 < n && n <= 0) {
    out += "0." + std::string(-n, '0') + digits;
  } else {
    out += digits.substr(0, 1);
    if (k > 1) out += "." + digits.substr(1);
    const int e = n - 1;
    out += e < 0 ? "e-" : "e+";
    const int ae = e < 0 ? -e : e;
    if (ae < 10) out += '0';
    out += std::to_string(ae);
  }
  return out;
}
inline std::string quote(const std::string& s) {
  std::string o = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') o += '\\';
    if (c == '\n') {
      o += "\\n";
      continue;
    }
    o += c;
  }
  return o + "\"";
}

}  // namespace json
}  // namespace b3d200
