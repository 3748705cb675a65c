// Minimal JSON value, reader and canonical writer for the planning core.
// Reader: RFC 8259 subset sufficient for SPEC's topology documents (objects, arrays,
// strings with escapes, numbers via strtod (correctly rounded), true/false/null).
// Writer helpers produce the canonical compact form used for plan parity
// (sorted keys, "," and ":" separators, ASCII-only strings with \uXXXX escapes).
#pragma once

#include <cstdint>
#include <cstdlib>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace gtar {

struct JsonError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Json {
  enum Kind { Null, Bool, Number, String, Array, Object } kind = Null;
  bool b = false;
  double num = 0.0;
  bool is_integer = false;   // lexically an integer (no '.', 'e')
  long long ival = 0;
  std::string str;
  std::vector<Json> arr;
  std::vector<std::pair<std::string, Json>> obj;  // document order

  const Json *get(const std::string &k) const {
    for (auto &kv : obj)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
};

class JsonReader {
 public:
  explicit JsonReader(const std::string &s) : s_(s) {}
  Json parse() {
    Json v = value();
    ws();
    if (p_ != s_.size()) fail("trailing characters");
    return v;
  }

 private:
  const std::string &s_;
  size_t p_ = 0;
  [[noreturn]] void fail(const char *m) {
    throw JsonError(std::string("syntax error: ") + m + " at offset " + std::to_string(p_));
  }
  void ws() {
    while (p_ < s_.size() && (s_[p_] == ' ' || s_[p_] == '\n' || s_[p_] == '\r' || s_[p_] == '\t')) p_++;
  }
  bool lit(const char *w) {
    size_t n = std::char_traits<char>::length(w);
    if (s_.compare(p_, n, w) == 0) {
      p_ += n;
      return true;
    }
    return false;
  }
  static void put_utf8(std::string &o, uint32_t cp) {
    if (cp < 0x80) o += char(cp);
    else if (cp < 0x800) { o += char(0xC0 | (cp >> 6)); o += char(0x80 | (cp & 0x3F)); }
    else if (cp < 0x10000) {
      o += char(0xE0 | (cp >> 12)); o += char(0x80 | ((cp >> 6) & 0x3F)); o += char(0x80 | (cp & 0x3F));
    } else {
      o += char(0xF0 | (cp >> 18)); o += char(0x80 | ((cp >> 12) & 0x3F));
      o += char(0x80 | ((cp >> 6) & 0x3F)); o += char(0x80 | (cp & 0x3F));
    }
  }
  uint32_t hex4() {
    if (p_ + 4 > s_.size()) fail("bad \\u escape");
    uint32_t v = 0;
    for (int i = 0; i < 4; i++) {
      char c = s_[p_++];
      v <<= 4;
      if (c >= '0' && c <= '9') v |= c - '0';
      else if (c >= 'a' && c <= 'f') v |= c - 'a' + 10;
      else if (c >= 'A' && c <= 'F') v |= c - 'A' + 10;
      else fail("bad hex digit");
    }
    return v;
  }
  std::string string_body() {
    std::string o;
    while (true) {
      if (p_ >= s_.size()) fail("unterminated string");
      char c = s_[p_++];
      if (c == '"') return o;
      if ((unsigned char)c < 0x20) fail("control character in string");
      if (c != '\\') { o += c; continue; }
      if (p_ >= s_.size()) fail("bad escape");
      char e = s_[p_++];
      switch (e) {
        case '"': o += '"'; break;
        case '\\': o += '\\'; break;
        case '/': o += '/'; break;
        case 'b': o += '\b'; break;
        case 'f': o += '\f'; break;
        case 'n': o += '\n'; break;
        case 'r': o += '\r'; break;
        case 't': o += '\t'; break;
        case 'u': {
          uint32_t cp = hex4();
          if (cp >= 0xD800 && cp < 0xDC00 && p_ + 6 <= s_.size() && s_[p_] == '\\' && s_[p_ + 1] == 'u') {
            p_ += 2;
            uint32_t lo = hex4();
            if (lo >= 0xDC00 && lo < 0xE000) cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
            else { put_utf8(o, cp); cp = lo; }
          }
          put_utf8(o, cp);
          break;
        }
        default: fail("bad escape");
      }
    }
  }
  Json value() {
    ws();
    if (p_ >= s_.size()) fail("unexpected end");
    Json v;
    char c = s_[p_];
    if (c == '{') {
      p_++;
      v.kind = Json::Object;
      ws();
      if (p_ < s_.size() && s_[p_] == '}') { p_++; return v; }
      while (true) {
        ws();
        if (p_ >= s_.size() || s_[p_] != '"') fail("expected key");
        p_++;
        std::string k = string_body();
        ws();
        if (p_ >= s_.size() || s_[p_] != ':') fail("expected ':'");
        p_++;
        for (auto &kv : v.obj)
          if (kv.first == k) fail("duplicate key");
        v.obj.emplace_back(k, value());
        ws();
        if (p_ < s_.size() && s_[p_] == ',') { p_++; continue; }
        if (p_ < s_.size() && s_[p_] == '}') { p_++; return v; }
        fail("expected ',' or '}'");
      }
    }
    if (c == '[') {
      p_++;
      v.kind = Json::Array;
      ws();
      if (p_ < s_.size() && s_[p_] == ']') { p_++; return v; }
      while (true) {
        v.arr.push_back(value());
        ws();
        if (p_ < s_.size() && s_[p_] == ',') { p_++; continue; }
        if (p_ < s_.size() && s_[p_] == ']') { p_++; return v; }
        fail("expected ',' or ']'");
      }
    }
    if (c == '"') {
      p_++;
      v.kind = Json::String;
      v.str = string_body();
      return v;
    }
    if (lit("true")) { v.kind = Json::Bool; v.b = true; return v; }
    if (lit("false")) { v.kind = Json::Bool; v.b = false; return v; }
    if (lit("null")) { v.kind = Json::Null; return v; }
    // number: -?(0|[1-9][0-9]*)(\.[0-9]+)?([eE][+-]?[0-9]+)?
    size_t st = p_;
    bool integer = true;
    if (s_[p_] == '-') p_++;
    if (p_ >= s_.size() || !isdigit((unsigned char)s_[p_])) fail("bad value");
    if (s_[p_] == '0') p_++;
    else while (p_ < s_.size() && isdigit((unsigned char)s_[p_])) p_++;
    if (p_ < s_.size() && s_[p_] == '.') {
      integer = false;
      p_++;
      if (p_ >= s_.size() || !isdigit((unsigned char)s_[p_])) fail("bad fraction");
      while (p_ < s_.size() && isdigit((unsigned char)s_[p_])) p_++;
    }
    if (p_ < s_.size() && (s_[p_] == 'e' || s_[p_] == 'E')) {
      integer = false;
      p_++;
      if (p_ < s_.size() && (s_[p_] == '+' || s_[p_] == '-')) p_++;
      if (p_ >= s_.size() || !isdigit((unsigned char)s_[p_])) fail("bad exponent");
      while (p_ < s_.size() && isdigit((unsigned char)s_[p_])) p_++;
    }
    std::string tok = s_.substr(st, p_ - st);
    v.kind = Json::Number;
    v.num = std::strtod(tok.c_str(), nullptr);
    v.is_integer = integer;
    if (integer) v.ival = std::strtoll(tok.c_str(), nullptr, 10);
    return v;
  }
};

// Python json.dumps(ensure_ascii=True) string escaping.
inline void json_escape(std::string &o, const std::string &s) {
  static const char *hx = "0123456789abcdef";
  o += '"';
  size_t i = 0;
  auto u4 = [&](uint32_t v) {
    o += "\\u";
    o += hx[(v >> 12) & 15]; o += hx[(v >> 8) & 15]; o += hx[(v >> 4) & 15]; o += hx[v & 15];
  };
  while (i < s.size()) {
    unsigned char c = (unsigned char)s[i];
    if (c < 0x80) {
      i++;
      switch (c) {
        case '"': o += "\\\""; break;
        case '\\': o += "\\\\"; break;
        case '\n': o += "\\n"; break;
        case '\r': o += "\\r"; break;
        case '\t': o += "\\t"; break;
        case '\b': o += "\\b"; break;
        case '\f': o += "\\f"; break;
        default:
          if (c < 0x20) u4(c);
          else o += char(c);
      }
      continue;
    }
    uint32_t cp;
    int len;
    if ((c & 0xE0) == 0xC0) { cp = c & 0x1F; len = 2; }
    else if ((c & 0xF0) == 0xE0) { cp = c & 0x0F; len = 3; }
    else { cp = c & 0x07; len = 4; }
    for (int k = 1; k < len && i + k < s.size(); k++) cp = (cp << 6) | ((unsigned char)s[i + k] & 0x3F);
    i += len;
    if (cp >= 0x10000) {
      cp -= 0x10000;
      u4(0xD800 + (cp >> 10));
      u4(0xDC00 + (cp & 0x3FF));
    } else {
      u4(cp);
    }
  }
  o += '"';
}

}  // namespace gtar
