// json_mini.hpp -- a small strict JSON reader for the reference's
// configuration objects (b3d_scene_from_json, b3d_infer config, library
// manifests) and a compact writer; the reference uses nlohmann::json, which
// this image does not ship, and the reader accepts exactly what its parser
// accepts (RFC 8259; objects keyed like its std::map, in byte order, the last
// of repeated keys kept).  Numbers keep their integer literal (int64 /
// uint64) or strtod value and are written as nlohmann's dump writes them
// (shortest round-trip digits).
#pragma once

#include <algorithm>
#include <cerrno>
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
  // an integer literal that fits (nlohmann: number_integer if negative,
  // number_unsigned otherwise); any other number is a float
  int int_kind = 0;  // 0 float, 1 int64 (i), 2 uint64 (u)
  long long i = 0;
  unsigned long long u = 0;
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
    if (s_.compare(0, 3, "\xEF\xBB\xBF") == 0) i_ = 3;  // a leading UTF-8 BOM is skipped
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
      // nlohmann's object is a std::map: keys in byte order, a repeated key
      // keeps its last value
      std::stable_sort(v.obj.begin(), v.obj.end(),
                       [](const auto& a, const auto& b) { return a.first < b.first; });
      std::vector<std::pair<std::string, Value>> uniq;
      for (auto& kv : v.obj) {
        if (!uniq.empty() && uniq.back().first == kv.first)
          uniq.back().second = std::move(kv.second);
        else
          uniq.push_back(std::move(kv));
      }
      v.obj = std::move(uniq);
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
    } else {  // JSON number grammar: -?(0|[1-9]d*)(.d+)?([eE][+-]?d+)?
      const size_t b0 = i_;
      size_t q = i_;
      auto digit = [&](size_t k) { return k < s_.size() && s_[k] >= '0' && s_[k] <= '9'; };
      if (q < s_.size() && s_[q] == '-') ++q;
      if (!digit(q)) throw ParseError("invalid value");
      if (s_[q] == '0') ++q;
      else
        while (digit(q)) ++q;
      bool is_int = true;
      if (q < s_.size() && s_[q] == '.') {
        is_int = false;
        ++q;
        if (!digit(q)) throw ParseError("invalid number");
        while (digit(q)) ++q;
      }
      if (q < s_.size() && (s_[q] == 'e' || s_[q] == 'E')) {
        is_int = false;
        ++q;
        if (q < s_.size() && (s_[q] == '+' || s_[q] == '-')) ++q;
        if (!digit(q)) throw ParseError("invalid number");
        while (digit(q)) ++q;
      }
      const std::string lit = s_.substr(b0, q - b0);
      v.kind = Value::Number;
      v.num = std::strtod(lit.c_str(), nullptr);
      if (is_int) {
        errno = 0;
        if (lit[0] == '-') {
          const long long x = std::strtoll(lit.c_str(), nullptr, 10);
          if (errno == 0) {
            v.int_kind = 1;
            v.i = x;
          }
        } else {
          const unsigned long long x = std::strtoull(lit.c_str(), nullptr, 10);
          if (errno == 0) {
            v.int_kind = 2;
            v.u = x;
          }
        }
      }
      i_ = q;
    }
    return v;
  }
  std::string string() {
    // RFC 8259 strings as nlohmann's lexer reads them: no raw control
    // characters, the eight escapes and \uXXXX (surrogate pairs combined,
    // lone surrogates rejected), well-formed UTF-8 otherwise
    if (i_ >= s_.size() || s_[i_] != '"') throw ParseError("expected a string");
    ++i_;
    std::string out;
    auto put_utf8 = [&](unsigned cp) {
      if (cp < 0x80) {
        out += (char)cp;
      } else if (cp < 0x800) {
        out += (char)(0xC0 | (cp >> 6));
        out += (char)(0x80 | (cp & 0x3F));
      } else if (cp < 0x10000) {
        out += (char)(0xE0 | (cp >> 12));
        out += (char)(0x80 | ((cp >> 6) & 0x3F));
        out += (char)(0x80 | (cp & 0x3F));
      } else {
        out += (char)(0xF0 | (cp >> 18));
        out += (char)(0x80 | ((cp >> 12) & 0x3F));
        out += (char)(0x80 | ((cp >> 6) & 0x3F));
        out += (char)(0x80 | (cp & 0x3F));
      }
    };
    auto hex4 = [&]() -> unsigned {
      if (i_ + 4 > s_.size()) throw ParseError("bad escape");
      unsigned v = 0;
      for (int k = 0; k < 4; ++k) {
        const char h = s_[i_++];
        v <<= 4;
        if (h >= '0' && h <= '9') v |= (unsigned)(h - '0');
        else if (h >= 'a' && h <= 'f') v |= (unsigned)(h - 'a' + 10);
        else if (h >= 'A' && h <= 'F') v |= (unsigned)(h - 'A' + 10);
        else throw ParseError("bad escape");
      }
      return v;
    };
    for (;;) {
      if (i_ >= s_.size()) throw ParseError("unterminated string");
      const unsigned char c = (unsigned char)s_[i_++];
      if (c == '"') break;
      if (c < 0x20) throw ParseError("control character in string");
      if (c == '\\') {
        if (i_ >= s_.size()) throw ParseError("bad escape");
        const char e = s_[i_++];
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
            unsigned cp = hex4();
            if (cp >= 0xD800 && cp <= 0xDBFF) {  // a high surrogate needs its low half
              if (i_ + 2 > s_.size() || s_[i_] != '\\' || s_[i_ + 1] != 'u')
                throw ParseError("lone surrogate");
              i_ += 2;
              const unsigned lo = hex4();
              if (lo < 0xDC00 || lo > 0xDFFF) throw ParseError("lone surrogate");
              cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
            } else if (cp >= 0xDC00 && cp <= 0xDFFF) {
              throw ParseError("lone surrogate");
            }
            put_utf8(cp);
            break;
          }
          default: throw ParseError("bad escape");
        }
        continue;
      }
      if (c < 0x80) {
        out += (char)c;
        continue;
      }
      // a multi-byte UTF-8 sequence, checked (shortest form, no surrogates)
      int n = 0;
      unsigned cp = 0;
      if ((c & 0xE0) == 0xC0) n = 1, cp = c & 0x1F;
      else if ((c & 0xF0) == 0xE0) n = 2, cp = c & 0x0F;
      else if ((c & 0xF8) == 0xF0) n = 3, cp = c & 0x07;
      else throw ParseError("ill-formed UTF-8");
      if (i_ + n > s_.size()) throw ParseError("ill-formed UTF-8");
      for (int k = 0; k < n; ++k) {
        const unsigned char d = (unsigned char)s_[i_ + k];
        if ((d & 0xC0) != 0x80) throw ParseError("ill-formed UTF-8");
        cp = (cp << 6) | (d & 0x3F);
      }
      if ((n == 1 && cp < 0x80) || (n == 2 && cp < 0x800) || (n == 3 && cp < 0x10000) ||
          cp > 0x10FFFF || (cp >= 0xD800 && cp <= 0xDFFF))
        throw ParseError("ill-formed UTF-8");
      out.append(s_, i_ - 1, (size_t)n + 1);
      i_ += (size_t)n;
    }
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
