// json_lite.hpp -- just enough JSON for this layer: cost-model files, eval_cache.jsonl lines.
//
// The reference leans on nlohmann/json; this layer has two needs only: (1) read objects / arrays /
// numbers / strings, (2) write numbers exactly as nlohmann's dump() does, so that the cache file
// stays byte-compatible (evaluator.cpp:178-192; key order fixed by ordered_json).
#pragma once

#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <map>
#include <memory>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

namespace mmxhost::json {

struct Value;
using Array = std::vector<Value>;
using Object = std::vector<std::pair<std::string, Value>>;  // insertion order kept

struct Value {
  enum class Kind { Null, Bool, Number, String, Array, Object } kind = Kind::Null;
  bool boolean = false;
  double number = 0.0;
  bool is_integer = false;  // number written without '.', 'e', 'E'
  std::string string;
  std::shared_ptr<Array> array;
  std::shared_ptr<Object> object;

  bool is_object() const { return kind == Kind::Object; }
  bool is_array() const { return kind == Kind::Array; }
  bool is_number() const { return kind == Kind::Number; }
  bool is_string() const { return kind == Kind::String; }
  const Value* find(std::string_view key) const {
    if (!is_object()) return nullptr;
    const Value* hit = nullptr;
    for (const auto& kv : *object)
      if (kv.first == key) hit = &kv.second;  // last duplicate wins, as in nlohmann
    return hit;
  }
};

class Parser {
 public:
  explicit Parser(std::string_view text) : s_(text) {}

  // false on any syntax error or trailing garbage
  bool parse(Value& out) {
    skip_ws();
    if (!value(out, 0)) return false;
    skip_ws();
    return pos_ == s_.size();
  }

 private:
  std::string_view s_;
  std::size_t pos_ = 0;

  void skip_ws() {
    while (pos_ < s_.size() && (s_[pos_] == ' ' || s_[pos_] == '\t' || s_[pos_] == '\n' || s_[pos_] == '\r')) ++pos_;
  }
  bool literal(std::string_view word) {
    if (s_.substr(pos_, word.size()) != word) return false;
    pos_ += word.size();
    return true;
  }
  static void put_utf8(std::string& out, unsigned cp) {
    if (cp < 0x80) out.push_back(static_cast<char>(cp));
    else if (cp < 0x800) { out.push_back(static_cast<char>(0xC0 | (cp >> 6))); out.push_back(static_cast<char>(0x80 | (cp & 0x3F))); }
    else if (cp < 0x10000) { out.push_back(static_cast<char>(0xE0 | (cp >> 12))); out.push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3F))); out.push_back(static_cast<char>(0x80 | (cp & 0x3F))); }
    else { out.push_back(static_cast<char>(0xF0 | (cp >> 18))); out.push_back(static_cast<char>(0x80 | ((cp >> 12) & 0x3F))); out.push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3F))); out.push_back(static_cast<char>(0x80 | (cp & 0x3F))); }
  }
  bool hex4(unsigned& cp) {
    if (pos_ + 4 > s_.size()) return false;
    cp = 0;
    for (int k = 0; k < 4; ++k) {
      const char ch = s_[pos_++];
      cp <<= 4;
      if (ch >= '0' && ch <= '9') cp |= static_cast<unsigned>(ch - '0');
      else if (ch >= 'a' && ch <= 'f') cp |= static_cast<unsigned>(ch - 'a' + 10);
      else if (ch >= 'A' && ch <= 'F') cp |= static_cast<unsigned>(ch - 'A' + 10);
      else return false;
    }
    return true;
  }
  bool string(std::string& out) {
    if (pos_ >= s_.size() || s_[pos_] != '"') return false;
    ++pos_;
    while (pos_ < s_.size()) {
      const char ch = s_[pos_++];
      if (ch == '"') return true;
      if (static_cast<unsigned char>(ch) < 0x20) return false;
      if (ch != '\\') { out.push_back(ch); continue; }
      if (pos_ >= s_.size()) return false;
      const char esc = s_[pos_++];
      switch (esc) {
        case '"': out.push_back('"'); break;
        case '\\': out.push_back('\\'); break;
        case '/': out.push_back('/'); break;
        case 'b': out.push_back('\b'); break;
        case 'f': out.push_back('\f'); break;
        case 'n': out.push_back('\n'); break;
        case 'r': out.push_back('\r'); break;
        case 't': out.push_back('\t'); break;
        case 'u': {
          unsigned cp = 0;
          if (!hex4(cp)) return false;
          if (cp >= 0xD800 && cp <= 0xDBFF) {  // surrogate pair
            unsigned lo = 0;
            if (!literal("\\u") || !hex4(lo) || lo < 0xDC00 || lo > 0xDFFF) return false;
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          }
          put_utf8(out, cp);
          break;
        }
        default: return false;
      }
    }
    return false;
  }
  bool number(Value& out) {
    const std::size_t start = pos_;
    if (pos_ < s_.size() && s_[pos_] == '-') ++pos_;
    if (pos_ >= s_.size()) return false;
    if (s_[pos_] == '0') ++pos_;
    else if (s_[pos_] >= '1' && s_[pos_] <= '9') while (pos_ < s_.size() && std::isdigit(static_cast<unsigned char>(s_[pos_]))) ++pos_;
    else return false;
    bool integer = true;
    if (pos_ < s_.size() && s_[pos_] == '.') {
      integer = false;
      ++pos_;
      if (pos_ >= s_.size() || !std::isdigit(static_cast<unsigned char>(s_[pos_]))) return false;
      while (pos_ < s_.size() && std::isdigit(static_cast<unsigned char>(s_[pos_]))) ++pos_;
    }
    if (pos_ < s_.size() && (s_[pos_] == 'e' || s_[pos_] == 'E')) {
      integer = false;
      ++pos_;
      if (pos_ < s_.size() && (s_[pos_] == '+' || s_[pos_] == '-')) ++pos_;
      if (pos_ >= s_.size() || !std::isdigit(static_cast<unsigned char>(s_[pos_]))) return false;
      while (pos_ < s_.size() && std::isdigit(static_cast<unsigned char>(s_[pos_]))) ++pos_;
    }
    const std::string text(s_.substr(start, pos_ - start));
    out.kind = Value::Kind::Number;
    out.number = std::strtod(text.c_str(), nullptr);  // correctly rounded, like nlohmann's lexer
    out.is_integer = integer;
    return true;
  }
  bool value(Value& out, int depth) {
    if (depth > 64 || pos_ >= s_.size()) return false;
    const char ch = s_[pos_];
    if (ch == '{') {
      ++pos_;
      out.kind = Value::Kind::Object;
      out.object = std::make_shared<Object>();
      skip_ws();
      if (pos_ < s_.size() && s_[pos_] == '}') { ++pos_; return true; }
      for (;;) {
        skip_ws();
        std::string key;
        if (!string(key)) return false;
        skip_ws();
        if (pos_ >= s_.size() || s_[pos_] != ':') return false;
        ++pos_;
        skip_ws();
        Value v;
        if (!value(v, depth + 1)) return false;
        out.object->emplace_back(std::move(key), std::move(v));
        skip_ws();
        if (pos_ < s_.size() && s_[pos_] == ',') { ++pos_; continue; }
        if (pos_ < s_.size() && s_[pos_] == '}') { ++pos_; return true; }
        return false;
      }
    }
    if (ch == '[') {
      ++pos_;
      out.kind = Value::Kind::Array;
      out.array = std::make_shared<Array>();
      skip_ws();
      if (pos_ < s_.size() && s_[pos_] == ']') { ++pos_; return true; }
      for (;;) {
        skip_ws();
        Value v;
        if (!value(v, depth + 1)) return false;
        out.array->push_back(std::move(v));
        skip_ws();
        if (pos_ < s_.size() && s_[pos_] == ',') { ++pos_; continue; }
        if (pos_ < s_.size() && s_[pos_] == ']') { ++pos_; return true; }
        return false;
      }
    }
    if (ch == '"') { out.kind = Value::Kind::String; return string(out.string); }
    if (ch == 't') { out.kind = Value::Kind::Bool; out.boolean = true; return literal("true"); }
    if (ch == 'f') { out.kind = Value::Kind::Bool; out.boolean = false; return literal("false"); }
    if (ch == 'n') { out.kind = Value::Kind::Null; return literal("null"); }
    return number(out);
  }
};

inline bool parse(std::string_view text, Value& out) { return Parser(text).parse(out); }

// A double as nlohmann::json::dump() prints it: shortest digits that round-trip, laid out as
// a plain decimal when the decimal exponent is in (-4, 15], with a trailing ".0" for integral
// values, otherwise d[.ddd]e±XX with at least two exponent digits.
inline std::string dump_number(double v) {
  if (!std::isfinite(v)) return "null";
  if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
  char sci[64];
  const auto res = std::to_chars(sci, sci + sizeof(sci), std::fabs(v), std::chars_format::scientific);
  std::string_view text(sci, static_cast<std::size_t>(res.ptr - sci));  // d[.ddd]e±XX, shortest
  const std::size_t epos = text.find('e');
  std::string digits;
  for (char ch : text.substr(0, epos))
    if (ch != '.') digits.push_back(ch);
  const int exp10 = std::atoi(std::string(text.substr(epos + 1)).c_str());
  const int k = static_cast<int>(digits.size());
  const int n = exp10 + 1;  // value = 0.digits * 10^n
  std::string out = std::signbit(v) ? "-" : "";
  if (k <= n && n <= 15) {
    out += digits + std::string(static_cast<std::size_t>(n - k), '0') + ".0";
  } else if (0 < n && n <= 15) {
    out += digits.substr(0, static_cast<std::size_t>(n)) + "." + digits.substr(static_cast<std::size_t>(n));
  } else if (-4 < n && n <= 0) {
    out += "0." + std::string(static_cast<std::size_t>(-n), '0') + digits;
  } else {
    out += digits.substr(0, 1);
    if (k > 1) out += "." + digits.substr(1);
    const int e = n - 1;
    out += e < 0 ? "e-" : "e+";
    const int ae = e < 0 ? -e : e;
    if (ae < 10) out += "0";
    out += std::to_string(ae);
  }
  return out;
}

// Strings in this layer are genomes and status names: ASCII without quotes or control bytes;
// escape the JSON-mandatory set anyway.
inline std::string dump_string(std::string_view s) {
  std::string out = "\"";
  for (char ch : s) {
    switch (ch) {
      case '"': out += "\\\""; break;
      case '\\': out += "\\\\"; break;
      case '\n': out += "\\n"; break;
      case '\r': out += "\\r"; break;
      case '\t': out += "\\t"; break;
      default:
        if (static_cast<unsigned char>(ch) < 0x20) {
          char buf[8];
          std::snprintf(buf, sizeof(buf), "\\u%04x", ch);
          out += buf;
        } else {
          out.push_back(ch);
        }
    }
  }
  return out + "\"";
}

}  // namespace mmxhost::json
