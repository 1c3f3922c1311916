// Minimal JSON reader for network configs (objects, arrays, strings,
// numbers, true/false/null).  Integers written without sign, fraction or
// exponent are "unsigned" (the reference config rules accept only those for
// extents).  Errors throw std::runtime_error with a byte offset.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace lcnn::json {

struct Value {
  enum class Type { Null, Bool, Number, String, Array, Object } type = Type::Null;
  bool b = false;
  double num = 0.0;
  bool is_unsigned = false;
  std::uint64_t u = 0;
  std::string str;
  std::vector<Value> arr;
  std::vector<std::pair<std::string, Value>> obj;

  bool is_object() const { return type == Type::Object; }
  bool is_array() const { return type == Type::Array; }
  bool is_string() const { return type == Type::String; }
  bool is_number_unsigned() const { return type == Type::Number && is_unsigned; }
  const Value* find(const std::string& key) const {
    for (const auto& kv : obj)
      if (kv.first == key) return &kv.second;
    return nullptr;
  }
};

class Parser {
 public:
  explicit Parser(const std::string& text) : s_(text) {}
  Value parse() {
    Value v = value();
    ws();
    if (i_ != s_.size()) fail("trailing characters");
    return v;
  }

 private:
  [[noreturn]] void fail(const std::string& why) const {
    throw std::runtime_error("parse error at byte " + std::to_string(i_) + ": " + why);
  }
  void ws() {
    while (i_ < s_.size() && (s_[i_] == ' ' || s_[i_] == '\t' || s_[i_] == '\n' || s_[i_] == '\r'))
      ++i_;
  }
  char peek() {
    ws();
    if (i_ >= s_.size()) fail("unexpected end of input");
    return s_[i_];
  }
  void expect(char c) {
    if (peek() != c) fail(std::string("expected '") + c + "'");
    ++i_;
  }
  bool literal(const char* word) {
    const std::string w(word);
    if (s_.compare(i_, w.size(), w) == 0) {
      i_ += w.size();
      return true;
    }
    return false;
  }
  Value value() {
    const char c = peek();
    Value v;
    if (c == '{') {
      v.type = Value::Type::Object;
      ++i_;
      if (peek() == '}') {
        ++i_;
        return v;
      }
      for (;;) {
        if (peek() != '"') fail("expected object key");
        std::string key = string_body();
        expect(':');
        v.obj.emplace_back(std::move(key), value());
        const char d = peek();
        ++i_;
        if (d == '}') break;
        if (d != ',') fail("expected ',' or '}'");
      }
    } else if (c == '[') {
      v.type = Value::Type::Array;
      ++i_;
      if (peek() == ']') {
        ++i_;
        return v;
      }
      for (;;) {
        v.arr.push_back(value());
        const char d = peek();
        ++i_;
        if (d == ']') break;
        if (d != ',') fail("expected ',' or ']'");
      }
    } else if (c == '"') {
      v.type = Value::Type::String;
      v.str = string_body();
    } else if (literal("true")) {
      v.type = Value::Type::Bool;
      v.b = true;
    } else if (literal("false")) {
      v.type = Value::Type::Bool;
    } else if (literal("null")) {
      v.type = Value::Type::Null;
    } else if (c == '-' || (c >= '0' && c <= '9')) {
      v = number();
    } else {
      fail("unexpected character");
    }
    return v;
  }
  std::string string_body() {
    ++i_;  // opening quote
    std::string out;
    while (i_ < s_.size() && s_[i_] != '"') {
      char c = s_[i_++];
      if (c == '\\') {
        if (i_ >= s_.size()) fail("bad escape");
        const char e = s_[i_++];
        switch (e) {
          case 'n': out += '\n'; break;
          case 't': out += '\t'; break;
          case 'r': out += '\r'; break;
          case 'b': out += '\b'; break;
          case 'f': out += '\f'; break;
          case 'u': {
            if (i_ + 4 > s_.size()) fail("bad \\u escape");
            const unsigned cp = std::stoul(s_.substr(i_, 4), nullptr, 16);
            i_ += 4;
            if (cp < 0x80) out += static_cast<char>(cp);
            else out += '?';
            break;
          }
          default: out += e;
        }
      } else {
        out += c;
      }
    }
    if (i_ >= s_.size()) fail("unterminated string");
    ++i_;
    return out;
  }
  Value number() {
    const std::size_t start = i_;
    bool integral = true, negative = false;
    if (s_[i_] == '-') {
      negative = true;
      ++i_;
    }
    while (i_ < s_.size() && std::isdigit(static_cast<unsigned char>(s_[i_]))) ++i_;
    if (i_ < s_.size() && s_[i_] == '.') {
      integral = false;
      ++i_;
      while (i_ < s_.size() && std::isdigit(static_cast<unsigned char>(s_[i_]))) ++i_;
    }
    if (i_ < s_.size() && (s_[i_] == 'e' || s_[i_] == 'E')) {
      integral = false;
      ++i_;
      if (i_ < s_.size() && (s_[i_] == '+' || s_[i_] == '-')) ++i_;
      while (i_ < s_.size() && std::isdigit(static_cast<unsigned char>(s_[i_]))) ++i_;
    }
    const std::string tok = s_.substr(start, i_ - start);
    if (tok == "-" || tok.empty()) fail("bad number");
    Value v;
    v.type = Value::Type::Number;
    v.num = std::stod(tok);
    if (integral && !negative && tok.size() <= 19) {
      v.is_unsigned = true;
      v.u = std::stoull(tok);
    }
    return v;
  }

  const std::string& s_;
  std::size_t i_ = 0;
};

inline Value parse(const std::string& text) { return Parser(text).parse(); }

}  // namespace lcnn::json
