// Minimal JSON value/parser/printer for the profile, cluster and plan wire
// formats (reference schemas: SPEC.md:88).  The reference uses
// nlohmann/json; this is a self-contained replacement so the product has no
// third-party dependency.  Integers and floats are kept apart the way the
// reference's require_int / require_number distinguish them
// (model.cpp:30-42): a number token without '.', 'e' or 'E' is an integer.
#pragma once

#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace dpl::json {

class Value {
 public:
  enum class Type { null, boolean, integer, number, string, array, object };

  Value() = default;
  Value(std::nullptr_t) {}
  Value(bool b) : type_(Type::boolean), b_(b) {}
  Value(int v) : type_(Type::integer), i_(v), d_(v) {}
  Value(long v) : type_(Type::integer), i_(v), d_(static_cast<double>(v)) {}
  Value(long long v) : type_(Type::integer), i_(v), d_(static_cast<double>(v)) {}
  Value(double v) : type_(Type::number), d_(v) {}
  Value(const char* s) : type_(Type::string), s_(s) {}
  Value(std::string s) : type_(Type::string), s_(std::move(s)) {}
  template <typename T>
  Value(const std::vector<T>& v) : type_(Type::array) {
    for (const auto& e : v) a_.emplace_back(e);
  }

  static Value array() { Value v; v.type_ = Type::array; return v; }
  static Value object() { Value v; v.type_ = Type::object; return v; }

  Type type() const { return type_; }
  bool is_null() const { return type_ == Type::null; }
  bool is_bool() const { return type_ == Type::boolean; }
  bool is_integer() const { return type_ == Type::integer; }
  bool is_number() const { return type_ == Type::integer || type_ == Type::number; }
  bool is_string() const { return type_ == Type::string; }
  bool is_array() const { return type_ == Type::array; }
  bool is_object() const { return type_ == Type::object; }

  bool as_bool() const { expect(Type::boolean, "boolean"); return b_; }
  double as_double() const {
    if (!is_number()) throw std::runtime_error("json: number expected");
    return d_;
  }
  std::int64_t as_int() const {
    if (type_ == Type::integer) return i_;
    if (type_ == Type::number) return static_cast<std::int64_t>(d_);
    throw std::runtime_error("json: integer expected");
  }
  const std::string& as_string() const { expect(Type::string, "string"); return s_; }
  const std::vector<Value>& items() const { expect(Type::array, "array"); return a_; }
  std::vector<Value>& items() { expect(Type::array, "array"); return a_; }
  std::size_t size() const { return is_array() ? a_.size() : is_object() ? o_.size() : 0; }
  bool empty() const { return size() == 0; }
  const Value& operator[](std::size_t i) const { return items().at(i); }

  bool contains(const std::string& key) const {
    if (!is_object()) return false;
    for (const auto& kv : o_) if (kv.first == key) return true;
    return false;
  }
  const Value& at(const std::string& key) const {
    if (is_object()) for (const auto& kv : o_) if (kv.first == key) return kv.second;
    throw std::runtime_error("json: missing key '" + key + "'");
  }
  Value& operator[](const std::string& key) {
    if (type_ == Type::null) type_ = Type::object;
    expect(Type::object, "object");
    for (auto& kv : o_) if (kv.first == key) return kv.second;
    o_.emplace_back(key, Value());
    return o_.back().second;
  }
  const std::vector<std::pair<std::string, Value>>& members() const { expect(Type::object, "object"); return o_; }
  void push_back(Value v) {
    if (type_ == Type::null) type_ = Type::array;
    expect(Type::array, "array");
    a_.push_back(std::move(v));
  }

  std::vector<int> as_int_vector() const {
    std::vector<int> out;
    for (const auto& e : items()) out.push_back(static_cast<int>(e.as_int()));
    return out;
  }
  std::vector<double> as_double_vector() const {
    std::vector<double> out;
    for (const auto& e : items()) out.push_back(e.as_double());
    return out;
  }

  std::string dump(int indent = -1) const {
    std::string out;
    write(out, indent, 0);
    return out;
  }

  static Value parse(const std::string& text);

 private:
  void expect(Type t, const char* what) const {
    if (type_ != t) throw std::runtime_error(std::string("json: ") + what + " expected");
  }

  static void write_double(std::string& out, double d) {
    if (!std::isfinite(d)) { out += "null"; return; }
    char buf[40];
    // shortest representation that round-trips exactly
    for (int prec = 15; prec <= 17; ++prec) {
      std::snprintf(buf, sizeof buf, "%.*g", prec, d);
      if (std::strtod(buf, nullptr) == d) break;
    }
    out += buf;
    if (!std::strpbrk(buf, ".eEn")) out += ".0";
  }

  static void write_string(std::string& out, const std::string& s) {
    out += '"';
    for (char c : s) {
      switch (c) {
        case '"': out += "\\\""; break;
        case '\\': out += "\\\\"; break;
        case '\n': out += "\\n"; break;
        case '\t': out += "\\t"; break;
        case '\r': out += "\\r"; break;
        default:
          if (static_cast<unsigned char>(c) < 0x20) {
            char buf[8];
            std::snprintf(buf, sizeof buf, "\\u%04x", c);
            out += buf;
          } else {
            out += c;
          }
      }
    }
    out += '"';
  }

  void write(std::string& out, int indent, int depth) const {
    auto newline = [&](int d) {
      if (indent < 0) return;
      out += '\n';
      out.append(static_cast<std::size_t>(indent * d), ' ');
    };
    switch (type_) {
      case Type::null: out += "null"; break;
      case Type::boolean: out += b_ ? "true" : "false"; break;
      case Type::integer: out += std::to_string(i_); break;
      case Type::number: write_double(out, d_); break;
      case Type::string: write_string(out, s_); break;
      case Type::array:
        out += '[';
        for (std::size_t k = 0; k < a_.size(); ++k) {
          if (k) out += ',';
          newline(depth + 1);
          a_[k].write(out, indent, depth + 1);
        }
        if (!a_.empty()) newline(depth);
        out += ']';
        break;
      case Type::object: {
        // keys in lexicographic order, as nlohmann::json (std::map) writes
        // them, so files round-trip byte-identically with the reference
        std::vector<const std::pair<std::string, Value>*> order;
        for (const auto& kv : o_) order.push_back(&kv);
        std::sort(order.begin(), order.end(), [](const auto* a, const auto* b) { return a->first < b->first; });
        out += '{';
        for (std::size_t k = 0; k < order.size(); ++k) {
          if (k) out += ',';
          newline(depth + 1);
          write_string(out, order[k]->first);
          out += indent < 0 ? ":" : ": ";
          order[k]->second.write(out, indent, depth + 1);
        }
        if (!o_.empty()) newline(depth);
        out += '}';
        break;
      }
    }
  }

  Type type_ = Type::null;
  bool b_ = false;
  std::int64_t i_ = 0;
  double d_ = 0.0;
  std::string s_;
  std::vector<Value> a_;
  std::vector<std::pair<std::string, Value>> o_;

  friend class Parser;
};

class Parser {
 public:
  explicit Parser(const std::string& t) : t_(t) {}

  Value parse_document() {
    Value v = parse_value();
    skip_ws();
    if (p_ != t_.size()) fail("trailing characters");
    return v;
  }

 private:
  [[noreturn]] void fail(const std::string& why) {
    throw std::runtime_error("json parse error at byte " + std::to_string(p_) + ": " + why);
  }
  void skip_ws() {
    while (p_ < t_.size() && (t_[p_] == ' ' || t_[p_] == '\n' || t_[p_] == '\t' || t_[p_] == '\r')) ++p_;
  }
  bool consume(const char* lit) {
    const std::size_t n = std::strlen(lit);
    if (t_.compare(p_, n, lit) == 0) { p_ += n; return true; }
    return false;
  }
  Value parse_value() {
    skip_ws();
    if (p_ >= t_.size()) fail("unexpected end of input");
    const char c = t_[p_];
    if (c == '{') return parse_object();
    if (c == '[') return parse_array();
    if (c == '"') return Value(parse_string());
    if (consume("true")) return Value(true);
    if (consume("false")) return Value(false);
    if (consume("null")) return Value();
    if (c == '-' || (c >= '0' && c <= '9')) return parse_number();
    fail(std::string("unexpected character '") + c + "'");
  }
  Value parse_number() {
    const std::size_t start = p_;
    bool is_float = false;
    if (t_[p_] == '-') ++p_;
    while (p_ < t_.size()) {
      const char c = t_[p_];
      if (c >= '0' && c <= '9') { ++p_; continue; }
      if (c == '.' || c == 'e' || c == 'E' || c == '+' || c == '-') { is_float = true; ++p_; continue; }
      break;
    }
    const std::string tok = t_.substr(start, p_ - start);
    if (tok == "-" || tok.empty()) fail("bad number");
    if (!is_float) {
      errno = 0;
      char* end = nullptr;
      const long long v = std::strtoll(tok.c_str(), &end, 10);
      if (errno == 0 && end && *end == '\0') return Value(v);
    }
    char* end = nullptr;
    const double d = std::strtod(tok.c_str(), &end);
    if (!end || *end != '\0') fail("bad number '" + tok + "'");
    return Value(d);
  }
  std::string parse_string() {
    ++p_;  // opening quote
    std::string out;
    while (true) {
      if (p_ >= t_.size()) fail("unterminated string");
      const char c = t_[p_++];
      if (c == '"') break;
      if (c != '\\') { out += c; continue; }
      if (p_ >= t_.size()) fail("bad escape");
      const char e = t_[p_++];
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
          if (p_ + 4 > t_.size()) fail("bad unicode escape");
          const unsigned cp = static_cast<unsigned>(std::strtoul(t_.substr(p_, 4).c_str(), nullptr, 16));
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
        default: fail("bad escape");
      }
    }
    return out;
  }
  Value parse_array() {
    ++p_;
    Value v = Value::array();
    skip_ws();
    if (p_ < t_.size() && t_[p_] == ']') { ++p_; return v; }
    while (true) {
      v.a_.push_back(parse_value());
      skip_ws();
      if (p_ >= t_.size()) fail("unterminated array");
      if (t_[p_] == ',') { ++p_; continue; }
      if (t_[p_] == ']') { ++p_; break; }
      fail("expected ',' or ']'");
    }
    return v;
  }
  Value parse_object() {
    ++p_;
    Value v = Value::object();
    skip_ws();
    if (p_ < t_.size() && t_[p_] == '}') { ++p_; return v; }
    while (true) {
      skip_ws();
      if (p_ >= t_.size() || t_[p_] != '"') fail("expected key");
      std::string key = parse_string();
      skip_ws();
      if (p_ >= t_.size() || t_[p_] != ':') fail("expected ':'");
      ++p_;
      Value val = parse_value();
      bool replaced = false;
      for (auto& kv : v.o_) {
        if (kv.first == key) { kv.second = std::move(val); replaced = true; break; }
      }
      if (!replaced) v.o_.emplace_back(std::move(key), std::move(val));
      skip_ws();
      if (p_ >= t_.size()) fail("unterminated object");
      if (t_[p_] == ',') { ++p_; continue; }
      if (t_[p_] == '}') { ++p_; break; }
      fail("expected ',' or '}'");
    }
    return v;
  }

  const std::string& t_;
  std::size_t p_ = 0;
};

inline Value Value::parse(const std::string& text) { return Parser(text).parse_document(); }

}  // namespace dpl::json
