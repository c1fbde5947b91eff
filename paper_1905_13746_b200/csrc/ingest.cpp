// INGEST (host C++): JSONL corpus -> dense count matrix, multithreaded.
//
// Restates corpus.parse_corpus + OpcodeHistogram.from_counts
// (pkg/src/groupnb/corpus.py:133-189, :42-53) for the dense path (SURVEY 8f
// rank 1): one `{"id", "label", "size_bytes", "opcodes"}` object per line,
// unknown keys ignored, blank lines skipped, mnemonics case-folded and merged,
// zero counts dropped.  The vocabulary is the sorted union of mnemonics (byte
// order of UTF-8 == code-point order == Python's sorted()), so column order is
// the reference's feature-tie order.  Errors reproduce the reference's types,
// line numbers and schema messages; JSON syntax errors carry our own wording
// after "invalid JSON: ".  Lines are split on '\n' ("\r\n" accepted); mnemonic
// case folding is ASCII (non-ASCII mnemonics are kept as written).
#include <algorithm>
#include <cerrno>
#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <string_view>
#include <thread>
#include <atomic>
#include <chrono>
#include <unordered_map>
#include <unordered_set>
#include <memory>
#include <vector>

#include "../../include/gnb.h"

namespace {

// ---------------------------------------------------------------- JSON values
enum class JT { Null, Bool, Int, BigInt, Float, Str, Arr, Obj };

struct JVal {
  JT t = JT::Null;
  bool b = false;
  int64_t i = 0;
  std::string s;  // Str value, or the number's source text (Float / BigInt)
  std::vector<JVal> arr;
  std::vector<std::pair<std::string, JVal>> obj;  // duplicate keys: last wins on lookup
  const JVal* get(const char* key) const {
    const JVal* r = nullptr;
    for (const auto& kv : obj)
      if (kv.first == key) r = &kv.second;
    return r;
  }
};

struct Parser {
  const char* p;
  const char* end;
  std::string err;

  void ws() {
    while (p < end && (*p == ' ' || *p == '\t' || *p == '\r' || *p == '\n')) ++p;
  }
  bool fail(const char* m) {
    if (err.empty()) err = m;
    return false;
  }
  static void put_utf8(std::string& o, uint32_t cp) {
    if (cp < 0x80) {
      o += static_cast<char>(cp);
    } else if (cp < 0x800) {
      o += static_cast<char>(0xC0 | (cp >> 6));
      o += static_cast<char>(0x80 | (cp & 0x3F));
    } else if (cp < 0x10000) {
      o += static_cast<char>(0xE0 | (cp >> 12));
      o += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
      o += static_cast<char>(0x80 | (cp & 0x3F));
    } else {
      o += static_cast<char>(0xF0 | (cp >> 18));
      o += static_cast<char>(0x80 | ((cp >> 12) & 0x3F));
      o += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
      o += static_cast<char>(0x80 | (cp & 0x3F));
    }
  }
  bool hex4(uint32_t& v) {
    if (end - p < 4) return fail("Invalid \\uXXXX escape");
    v = 0;
    for (int k = 0; k < 4; ++k) {
      const char c = *p++;
      v <<= 4;
      if (c >= '0' && c <= '9') v |= c - '0';
      else if (c >= 'a' && c <= 'f') v |= c - 'a' + 10;
      else if (c >= 'A' && c <= 'F') v |= c - 'A' + 10;
      else return fail("Invalid \\uXXXX escape");
    }
    return true;
  }
  bool str(std::string& o) {  // at opening quote
    ++p;
    o.clear();
    while (p < end) {
      const char c = *p++;
      if (c == '"') return true;
      if (static_cast<unsigned char>(c) < 0x20) return fail("Invalid control character");
      if (c != '\\') {
        o += c;
        continue;
      }
      if (p >= end) break;
      const char e = *p++;
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
          uint32_t cp;
          if (!hex4(cp)) return false;
          if (cp >= 0xD800 && cp < 0xDC00 && end - p >= 6 && p[0] == '\\' && p[1] == 'u') {
            const char* save = p;
            p += 2;
            uint32_t lo;
            if (hex4(lo) && lo >= 0xDC00 && lo < 0xE000)
              cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
            else
              p = save;
          }
          put_utf8(o, cp);
          break;
        }
        default: return fail("Invalid \\escape");
      }
    }
    return fail("Unterminated string");
  }
  bool num(JVal& v) {
    const char* s = p;
    if (*p == '-') ++p;
    if (p >= end || !(*p >= '0' && *p <= '9')) return fail("Expecting value");
    if (*p == '0') ++p;
    else
      while (p < end && *p >= '0' && *p <= '9') ++p;
    bool is_float = false;
    if (p < end && *p == '.') {
      is_float = true;
      ++p;
      if (p >= end || !(*p >= '0' && *p <= '9')) return fail("Expecting value");
      while (p < end && *p >= '0' && *p <= '9') ++p;
    }
    if (p < end && (*p == 'e' || *p == 'E')) {
      is_float = true;
      ++p;
      if (p < end && (*p == '+' || *p == '-')) ++p;
      if (p >= end || !(*p >= '0' && *p <= '9')) return fail("Expecting value");
      while (p < end && *p >= '0' && *p <= '9') ++p;
    }
    v.s.assign(s, p - s);
    if (is_float) {
      v.t = JT::Float;
      return true;
    }
    // integer: exact in int64, else BigInt (kept as text for messages)
    errno = 0;
    char* e2 = nullptr;
    const long long x = strtoll(v.s.c_str(), &e2, 10);
    if (errno == ERANGE) {
      v.t = JT::BigInt;
    } else {
      v.t = JT::Int;
      v.i = x;
    }
    return true;
  }
  bool lit(const char* w, size_t n) {
    if (static_cast<size_t>(end - p) >= n && memcmp(p, w, n) == 0) {
      p += n;
      return true;
    }
    return fail("Expecting value");
  }
  bool value(JVal& v, int depth) {
    if (depth > 64) return fail("nesting too deep");
    ws();
    if (p >= end) return fail("Expecting value");
    const char c = *p;
    if (c == '{') {
      v.t = JT::Obj;
      ++p;
      ws();
      if (p < end && *p == '}') {
        ++p;
        return true;
      }
      for (;;) {
        ws();
        if (p >= end || *p != '"') return fail("Expecting property name enclosed in double quotes");
        std::string k;
        if (!str(k)) return false;
        ws();
        if (p >= end || *p != ':') return fail("Expecting ':' delimiter");
        ++p;
        JVal x;
        if (!value(x, depth + 1)) return false;
        v.obj.emplace_back(std::move(k), std::move(x));
        ws();
        if (p < end && *p == ',') {
          ++p;
          continue;
        }
        if (p < end && *p == '}') {
          ++p;
          return true;
        }
        return fail("Expecting ',' delimiter");
      }
    }
    if (c == '[') {
      v.t = JT::Arr;
      ++p;
      ws();
      if (p < end && *p == ']') {
        ++p;
        return true;
      }
      for (;;) {
        JVal x;
        if (!value(x, depth + 1)) return false;
        v.arr.push_back(std::move(x));
        ws();
        if (p < end && *p == ',') {
          ++p;
          continue;
        }
        if (p < end && *p == ']') {
          ++p;
          return true;
        }
        return fail("Expecting ',' delimiter");
      }
    }
    if (c == '"') {
      v.t = JT::Str;
      return str(v.s);
    }
    if (c == 't') {
      v.t = JT::Bool;
      v.b = true;
      return lit("true", 4);
    }
    if (c == 'f') {
      v.t = JT::Bool;
      return lit("false", 5);
    }
    if (c == 'n') {
      v.t = JT::Null;
      return lit("null", 4);
    }
    if (c == 'N') return lit("NaN", 3) && (v.t = JT::Float, v.s = "nan", true);
    if (c == 'I') return lit("Infinity", 8) && (v.t = JT::Float, v.s = "inf", true);
    if (c == '-' && end - p >= 9 && memcmp(p, "-Infinity", 9) == 0) {
      p += 9;
      v.t = JT::Float;
      v.s = "-inf";
      return true;
    }
    return num(v);
  }
};

// Python repr() of a JSON-decoded value, for error messages
std::string py_repr(const JVal& v);

std::string py_str_repr(const std::string& s) {
  const bool has_sq = s.find('\'') != std::string::npos;
  const bool has_dq = s.find('"') != std::string::npos;
  const char q = (has_sq && !has_dq) ? '"' : '\'';
  std::string o(1, q);
  for (unsigned char c : s) {
    if (c == static_cast<unsigned char>(q) || c == '\\') {
      o += '\\';
      o += static_cast<char>(c);
    } else if (c == '\n') {
      o += "\\n";
    } else if (c == '\r') {
      o += "\\r";
    } else if (c == '\t') {
      o += "\\t";
    } else if (c < 0x20 || c == 0x7f) {
      char b[8];
      snprintf(b, sizeof b, "\\x%02x", c);
      o += b;
    } else {
      o += static_cast<char>(c);
    }
  }
  o += q;
  return o;
}

std::string py_repr(const JVal& v) {
  switch (v.t) {
    case JT::Null: return "None";
    case JT::Bool: return v.b ? "True" : "False";
    case JT::Int: return std::to_string(v.i);
    case JT::BigInt: return v.s;
    case JT::Float: {
      if (v.s == "nan" || v.s == "inf" || v.s == "-inf") return v.s;
      char b[64];
      snprintf(b, sizeof b, "%.17g", strtod(v.s.c_str(), nullptr));
      std::string r = b;  // shortest round-trip repr is Python's; close enough for messages
      if (r.find_first_of(".en") == std::string::npos) r += ".0";
      return r;
    }
    case JT::Str: return py_str_repr(v.s);
    case JT::Arr: {
      std::string o = "[";
      for (size_t k = 0; k < v.arr.size(); ++k) o += (k ? ", " : "") + py_repr(v.arr[k]);
      return o + "]";
    }
    case JT::Obj: {
      std::string o = "{";
      for (size_t k = 0; k < v.obj.size(); ++k)
        o += (k ? ", " : "") + py_str_repr(v.obj[k].first) + ": " + py_repr(v.obj[k].second);
      return o + "}";
    }
  }
  return "?";
}

// ---------------------------------------------------------------- corpus
struct Row {
  std::string id;
  int8_t label;     // 1 malware, 0 benign, -1 unknown
  int64_t size;     // size_bytes; -1 if it does not fit int64 (only >= 2^63)
  int64_t e0 = 0, e1 = 0;  // entries [e0, e1) in the shard's col/val arrays
};

struct Shard {
  std::vector<Row> rows;
  std::vector<int32_t> col;  // shard-local vocab id per entry
  std::vector<int64_t> val;
  std::vector<int64_t> mark, pos;  // per local vocab id: last row touching it, entry index
  std::vector<int64_t> line_no;
  // shard-local vocabulary: open addressing over FNV-1a hashes of the
  // lower-cased mnemonic (slots hold vid + 1, 0 = empty); names[vid] holds it
  std::vector<int32_t> slots = std::vector<int32_t>(1024, 0);
  std::vector<uint64_t> hashes;
  std::vector<std::string> names;
  int64_t err_line = -1;
  int err_kind = 0;  // 1 ParseError, 2 IntegrityError
  std::string err_msg;
  std::string err_id;  // the failing line's id when it was valid (duplicate check wins)
  bool err_has_id = false;
};

// Hash of a lower-cased mnemonic, a word at a time: 8-byte little-endian
// words, the last one zero-padded.  The fast path computes the same value
// while it lower-cases (SWAR, below); everything else calls key_hash.
inline uint64_t mix_word(uint64_t h, uint64_t w) {
  h = (h ^ w) * 0x9E3779B97F4A7C15ull;
  return h ^ (h >> 29);
}
inline uint64_t key_hash(const char* s, size_t n) {
  uint64_t h = n * 0xC2B2AE3D27D4EB4Full;
  size_t i = 0;
  for (; i + 8 <= n; i += 8) {
    uint64_t w;
    memcpy(&w, s + i, 8);
    h = mix_word(h, w);
  }
  if (i < n) {
    uint64_t w = 0;
    memcpy(&w, s + i, n - i);
    h = mix_word(h, w);
  }
  return h ^ (h >> 32);
}
// 'A'..'Z' -> 'a'..'z' in each byte of w; every other byte (incl. >= 0x80) kept
inline uint64_t lower8(uint64_t w) {
  const uint64_t hi = 0x8080808080808080ull;
  const uint64_t a = (w & ~hi) + 0x3F3F3F3F3F3F3F3Full;  // low 7 bits >= 'A'
  const uint64_t z = (w & ~hi) + 0x2525252525252525ull;  // low 7 bits >  'Z'
  return w | ((a & ~z & ~w & hi) >> 2);
}

// vid of the (already lower-cased) mnemonic [s, s+n) with FNV-1a hash h,
// added if new.
int32_t vocab_id(Shard& sh, const char* s, size_t n, uint64_t h) {
  size_t mask = sh.slots.size() - 1;
  for (size_t i = static_cast<size_t>(h) & mask;; i = (i + 1) & mask) {
    const int32_t v = sh.slots[i];
    if (v == 0) break;
    const std::string& nm = sh.names[v - 1];
    if (sh.hashes[v - 1] == h && nm.size() == n && memcmp(nm.data(), s, n) == 0) return v - 1;
  }
  const int32_t vid = static_cast<int32_t>(sh.names.size());
  sh.names.emplace_back(s, n);
  sh.hashes.push_back(h);
  sh.mark.push_back(0);
  sh.pos.push_back(0);
  if (sh.names.size() * 2 > sh.slots.size()) {  // keep the load factor <= 1/2
    std::vector<int32_t> grown(sh.slots.size() * 2, 0);
    mask = grown.size() - 1;
    for (size_t k = 0; k < sh.names.size(); ++k) {
      size_t i = static_cast<size_t>(sh.hashes[k]) & mask;
      while (grown[i] != 0) i = (i + 1) & mask;
      grown[i] = static_cast<int32_t>(k) + 1;
    }
    sh.slots.swap(grown);
  } else {
    size_t i = static_cast<size_t>(h) & mask;
    while (sh.slots[i] != 0) i = (i + 1) & mask;
    sh.slots[i] = vid + 1;
  }
  return vid;
}

int32_t vocab_id(Shard& sh, const char* s, size_t n) { return vocab_id(sh, s, n, key_hash(s, n)); }

std::string lower_ascii(const std::string& s) {
  std::string o = s;
  for (char& c : o)
    if (c >= 'A' && c <= 'Z') c = static_cast<char>(c - 'A' + 'a');
  return o;
}

bool is_blank(const char* a, const char* b) {
  for (; a < b; ++a)
    if (!(*a == ' ' || *a == '\t' || *a == '\r' || *a == '\n' || *a == '\v' || *a == '\f'))
      return false;
  return true;
}


// Fast path for clean records: one pass, no DOM, no per-value allocation.
// Returns false on anything unusual (escapes, duplicate keys, non-integer or
// negative numbers, unknown labels, syntax errors...); the caller then runs
// parse_line, which implements every rule and error message.
struct FastScratch {
  std::string key;
};

inline void skip_ws(const char*& p, const char* e) {
  while (p < e && (*p == ' ' || *p == '\t' || *p == '\r' || *p == '\n')) ++p;
}

// "...": plain string without escapes; [s, s+n) excludes the quotes
inline bool plain_str(const char*& p, const char* e, const char*& s, size_t& n) {
  if (p >= e || *p != '"') return false;
  s = ++p;
  while (p < e && *p != '"') {
    if (*p == '\\' || static_cast<unsigned char>(*p) < 0x20) return false;
    ++p;
  }
  if (p >= e) return false;
  n = static_cast<size_t>(p - s);
  ++p;
  return true;
}

inline bool plain_uint(const char*& p, const char* e, int64_t& v) {
  const char* s = p;
  v = 0;
  while (p < e && *p >= '0' && *p <= '9') {
    if (p - s >= 18) return false;  // leave big numbers to the full parser
    v = v * 10 + (*p - '0');
    ++p;
  }
  if (p == s || (p - s > 1 && *s == '0')) return false;
  return !(p < e && (*p == '.' || *p == 'e' || *p == 'E'));
}

bool skip_value(const char*& p, const char* e, int depth) {  // syntax-checked skip
  Parser ps{p, e, {}};
  JVal v;
  if (!ps.value(v, depth)) return false;
  p = ps.p;
  return true;
}

bool fast_line(const char* a, const char* b, bool allow_unlabeled, Shard& sh, Row& row,
               FastScratch& fs) {
  const char* p = a;
  skip_ws(p, b);
  if (p >= b || *p != '{') return false;
  ++p;
  unsigned seen = 0;  // id 1, label 2, size 4, opcodes 8
  row.label = -1;
  const int64_t row_tag = static_cast<int64_t>(sh.rows.size()) + 1;
  const size_t col0 = sh.col.size();
  row.e0 = static_cast<int64_t>(col0);
  // on any bail-out the entries appended so far are dropped by the caller
  skip_ws(p, b);
  if (p < b && *p == '}') return false;
  for (;;) {
    skip_ws(p, b);
    const char* ks;
    size_t kn;
    if (!plain_str(p, b, ks, kn)) return false;
    skip_ws(p, b);
    if (p >= b || *p != ':') return false;
    ++p;
    skip_ws(p, b);
    unsigned bit = 0;
    if (kn == 2 && memcmp(ks, "id", 2) == 0) bit = 1;
    else if (kn == 5 && memcmp(ks, "label", 5) == 0) bit = 2;
    else if (kn == 10 && memcmp(ks, "size_bytes", 10) == 0) bit = 4;
    else if (kn == 7 && memcmp(ks, "opcodes", 7) == 0) bit = 8;
    if (bit & seen) return false;  // duplicate key: json.loads keeps the last one
    seen |= bit;
    if (bit == 1) {
      const char* s;
      size_t n;
      if (!plain_str(p, b, s, n) || n == 0) return false;
      row.id.assign(s, n);
    } else if (bit == 2) {
      const char* s;
      size_t n;
      if (!plain_str(p, b, s, n)) return false;
      if (n == 7 && memcmp(s, "malware", 7) == 0) row.label = 1;
      else if (n == 6 && memcmp(s, "benign", 6) == 0) row.label = 0;
      else return false;
    } else if (bit == 4) {
      int64_t v;
      if (!plain_uint(p, b, v)) return false;
      row.size = v;
    } else if (bit == 8) {
      if (p >= b || *p != '{') return false;
      ++p;
      skip_ws(p, b);
      if (p < b && *p == '}') {
        ++p;
      } else {
        for (;;) {
          skip_ws(p, b);
          const char* s;
          size_t n;
          if (!plain_str(p, b, s, n) || n == 0) return false;
          skip_ws(p, b);
          if (p >= b || *p != ':') return false;
          ++p;
          skip_ws(p, b);
          int64_t v;
          if (!plain_uint(p, b, v)) return false;
          // a zero count may shadow an earlier duplicate key (JSON last-wins):
          // rare, so the full parser takes it
          if (v == 0) return false;
          {
            // lower-case + hash in one pass, 8 bytes at a time when the
            // line holds whole words past the key (stack buffer for usual
            // mnemonics)
            alignas(8) char kb[64];
            char* key = kb;
            uint64_t h;
            if (n <= sizeof(kb) && s + ((n + 7) & ~size_t(7)) <= b) {
              h = n * 0xC2B2AE3D27D4EB4Full;
              for (size_t i = 0; i < n; i += 8) {
                uint64_t w;
                memcpy(&w, s + i, 8);
                if (n - i < 8) w &= (uint64_t(1) << (8 * (n - i))) - 1;
                w = lower8(w);
                memcpy(kb + i, &w, 8);
                h = mix_word(h, w);
              }
              h ^= h >> 32;
            } else {
              if (n > sizeof(kb)) {
                fs.key.resize(n);
                key = fs.key.data();
              }
              for (size_t i = 0; i < n; ++i) {
                char c = s[i];
                if (c >= 'A' && c <= 'Z') c = static_cast<char>(c - 'A' + 'a');
                key[i] = c;
              }
              h = key_hash(key, n);
            }
            const int32_t vid = vocab_id(sh, key, n, h);
            if (sh.mark[vid] == row_tag) {
              // repeated key (exact duplicate: JSON last-wins) or case variant
              // (merged): both rare, both left to the full parser
              return false;
            } else {
              sh.mark[vid] = row_tag;
              sh.pos[vid] = static_cast<int64_t>(sh.col.size());
              sh.col.push_back(vid);
              sh.val.push_back(v);
            }
          }
          skip_ws(p, b);
          if (p < b && *p == ',') {
            ++p;
            continue;
          }
          if (p < b && *p == '}') {
            ++p;
            break;
          }
          return false;
        }
      }
    } else {
      if (!skip_value(p, b, 1)) return false;
    }
    skip_ws(p, b);
    if (p < b && *p == ',') {
      ++p;
      continue;
    }
    if (p < b && *p == '}') {
      ++p;
      break;
    }
    return false;
  }
  skip_ws(p, b);
  if (p != b) return false;
  if (!(seen & 1) || !(seen & 4) || !(seen & 8)) return false;
  if (!(seen & 2) && !allow_unlabeled) return false;
  row.e1 = static_cast<int64_t>(sh.col.size());
  (void)col0;
  return true;
}

// corpus.py:146-188 for one line; returns false with (kind, msg) on error
bool parse_line(const char* a, const char* b, bool allow_unlabeled, Shard& sh, Row& row,
                int& kind, std::string& msg) {
  Parser ps{a, b, {}};
  JVal v;
  if (!ps.value(v, 0)) {
    kind = 1;
    msg = "invalid JSON: " + ps.err;
    return false;
  }
  ps.ws();
  if (ps.p != b) {
    kind = 1;
    msg = "invalid JSON: Extra data";
    return false;
  }
  if (v.t != JT::Obj) {
    kind = 1;
    msg = "record must be a JSON object";
    return false;
  }
  const JVal* id = v.get("id");
  if (!id || id->t != JT::Str || id->s.empty()) {
    kind = 1;
    msg = "missing or empty 'id'";
    return false;
  }
  row.id = id->s;
  const JVal* lab = v.get("label");
  if (lab) {
    if (lab->t == JT::Str && lab->s == "malware") row.label = 1;
    else if (lab->t == JT::Str && lab->s == "benign") row.label = 0;
    else {
      kind = 1;
      msg = "unknown label " + py_repr(*lab);
      return false;
    }
  } else if (allow_unlabeled) {
    row.label = -1;
  } else {
    kind = 1;
    msg = "missing 'label'";
    return false;
  }
  const JVal* sz = v.get("size_bytes");
  if (!sz || !(sz->t == JT::Int || sz->t == JT::BigInt) || (sz->t == JT::Int && sz->i < 0) ||
      (sz->t == JT::BigInt && !sz->s.empty() && sz->s[0] == '-')) {
    kind = 1;
    msg = "'size_bytes' must be a non-negative integer";
    return false;
  }
  row.size = sz->t == JT::Int ? sz->i : -1;  // > int64: out of any size range
  const JVal* ops = v.get("opcodes");
  if (!ops || ops->t != JT::Obj) {
    kind = 1;
    msg = "'opcodes' must be an object";
    return false;
  }
  // OpcodeHistogram.from_counts over the dict json.loads builds: duplicate keys
  // keep the LAST value at the position of the FIRST occurrence.
  std::vector<std::pair<std::string, const JVal*>> items;
  std::unordered_map<std::string, size_t> pos;
  for (const auto& kv : ops->obj) {
    auto it = pos.find(kv.first);
    if (it == pos.end()) {
      pos.emplace(kv.first, items.size());
      items.emplace_back(kv.first, &kv.second);
    } else {
      items[it->second].second = &kv.second;
    }
  }
  std::vector<std::pair<int32_t, int64_t>> ents;
  std::unordered_map<int32_t, size_t> where;
  for (const auto& it : items) {
    const JVal& c = *it.second;
    if (it.first.empty()) {
      kind = 1;
      msg = "opcode mnemonic must be a non-empty string, got ''";
      return false;
    }
    const bool ok_int = (c.t == JT::Int && c.i >= 0) ||
                        (c.t == JT::BigInt && !c.s.empty() && c.s[0] != '-');
    if (!ok_int) {
      kind = 1;
      msg = "count for " + py_str_repr(it.first) + " must be a non-negative integer, got " +
            py_repr(c);
      return false;
    }
    if (c.t == JT::BigInt) {
      kind = 1;  // counts beyond int64 cannot be represented densely
      msg = "count for " + py_str_repr(it.first) + " exceeds the dense range, got " + c.s;
      return false;
    }
    if (c.i == 0) continue;
    const std::string key = lower_ascii(it.first);
    const int32_t vid = vocab_id(sh, key.data(), key.size());
    auto w = where.find(vid);
    if (w == where.end()) {
      where.emplace(vid, ents.size());
      ents.emplace_back(vid, c.i);
    } else {
      ents[w->second].second += c.i;
    }
  }
  row.e0 = static_cast<int64_t>(sh.col.size());
  for (const auto& e : ents) {
    sh.col.push_back(e.first);
    sh.val.push_back(e.second);
  }
  row.e1 = static_cast<int64_t>(sh.col.size());
  return true;
}

}  // namespace

// A heap array that is NOT value-initialised on resize: the corpus CSR
// arrays are filled by the parallel scatter, so zero-filling 100s of MB
// first (std::vector::resize) was a serial pass as long as the parse.
template <typename T>
struct RawArray {
  std::unique_ptr<T[]> p;
  size_t n = 0;
  void resize_uninit(size_t k) {
    p.reset(k ? new T[k] : nullptr);  // default-init: no zeroing for scalars
    n = k;
  }
  size_t size() const { return n; }
  T& operator[](size_t i) { return p[i]; }
  const T& operator[](size_t i) const { return p[i]; }
};

struct gnb_corpus {
  std::vector<std::string> vocab;
  std::vector<std::string> ids;
  std::vector<int64_t> size;
  std::vector<int8_t> label;
  RawArray<int64_t> row_ptr;
  RawArray<int32_t> col;
  RawArray<int64_t> val;
  int64_t max_count = 0;
  int err_kind = 0;
  int64_t err_line = 0;
  std::string err_msg;
};

extern "C" {

int gnb_corpus_parse(const char* text, size_t len, int32_t allow_unlabeled, int32_t threads,
                     gnb_corpus** out) {
  if (!out || (!text && len)) return GNB_EINVAL;
  auto* c = new gnb_corpus();
  *out = c;
  int T = threads > 0 ? threads : static_cast<int>(std::thread::hardware_concurrency());
  T = std::max(1, std::min(T, 64));
  if (len < (size_t(1) << 20)) T = 1;
  auto run = [T](const std::function<void(int)>& f) {
    std::vector<std::thread> th;
    for (int t = 1; t < T; ++t) th.emplace_back(f, t);
    f(0);
    for (auto& x : th) x.join();
  };
  // byte ranges cut at line starts; per-range line counts give 1-based line
  // numbers (enumerate(..., start=1)) without a serial scan
  std::vector<size_t> cut(T + 1, len);
  cut[0] = 0;
  for (int t = 1; t < T; ++t) {
    size_t q = len * static_cast<size_t>(t) / T;
    while (q < len && text[q - 1] != '\n') ++q;
    cut[t] = std::max(q, cut[t - 1]);
  }
  auto T0 = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {  // GNB_INGEST_TIMING=1: phase times on stderr
    static const bool on = getenv("GNB_INGEST_TIMING") != nullptr;
    if (!on) return;
    auto t1 = std::chrono::steady_clock::now();
    fprintf(stderr, "%s %.1f ms\n", what, std::chrono::duration<double, std::milli>(t1 - T0).count());
    T0 = t1;
  };
  std::vector<int64_t> nlines(T, 0), first_line(T, 1);
  run([&](int t) {
    int64_t k = 0;  // memchr hops: a byte loop through the captured pointer ran at 0.7 GB/s
    for (const char *q = text + cut[t], *e = text + cut[t + 1];
         (q = static_cast<const char*>(memchr(q, '\n', static_cast<size_t>(e - q)))) != nullptr;
         ++q, ++k) {
    }
    if (cut[t + 1] > cut[t] && text[cut[t + 1] - 1] != '\n') ++k;  // unterminated last line
    nlines[t] = k;
  });
  for (int t = 1; t < T; ++t) first_line[t] = first_line[t - 1] + nlines[t - 1];
  lap("lines");
  std::vector<Shard> shards(T);
  run([&](int t) {
    Shard& sh = shards[t];
    FastScratch fs;
    sh.rows.reserve(static_cast<size_t>(nlines[t]));
    sh.line_no.reserve(static_cast<size_t>(nlines[t]));
    // an opcode entry takes >= 9 bytes of JSON ("x": 1, ): no regrowth copies
    sh.col.reserve((cut[t + 1] - cut[t]) / 9 + 16);
    sh.val.reserve((cut[t + 1] - cut[t]) / 9 + 16);
    const char* p = text + cut[t];
    const char* end = text + cut[t + 1];
    int64_t ln = first_line[t];
    for (; p < end; ++ln) {
      const char* a = p;
      const char* nl = static_cast<const char*>(memchr(a, '\n', static_cast<size_t>(end - a)));
      const char* b = nl ? nl : end;
      p = nl ? nl + 1 : end;
      while (b > a && b[-1] == '\r') --b;
      if (is_blank(a, b)) continue;
      Row row;
      int kind = 0;
      std::string msg;
      const size_t mark = sh.col.size();
      if (fast_line(a, b, allow_unlabeled != 0, sh, row, fs)) {
        sh.rows.push_back(std::move(row));
        sh.line_no.push_back(ln);
        continue;
      }
      sh.col.resize(mark);  // discard the fast path's partial entries
      sh.val.resize(mark);
      row = Row();
      if (!parse_line(a, b, allow_unlabeled != 0, sh, row, kind, msg)) {
        sh.err_line = ln;
        sh.err_kind = kind;
        sh.err_msg = msg;
        sh.err_has_id = !row.id.empty();
        sh.err_id = row.id;
        return;  // later lines of this shard cannot matter
      }
      sh.rows.push_back(std::move(row));
      sh.line_no.push_back(ln);
    }
  });
  lap("parse");
  // first error by line; duplicate ids before it win (the reference parses in order)
  int64_t first_err = -1;
  const Shard* err_sh = nullptr;
  for (auto& sh : shards)
    if (sh.err_line >= 0 && (first_err < 0 || sh.err_line < first_err)) {
      first_err = sh.err_line;
      err_sh = &sh;
      c->err_kind = sh.err_kind;
      c->err_msg = sh.err_msg;
    }
  // No parse error (the usual case): look for ANY duplicate id in parallel
  // (lock-free open addressing on row references); only when one exists does
  // the serial in-order scan below run to name the first one.
  bool need_scan = first_err >= 0;
  if (!need_scan) {
    size_t total = 0;
    for (auto& sh : shards) total += sh.rows.size();
    size_t cap = 16;
    while (cap < 2 * total) cap <<= 1;
    std::unique_ptr<std::atomic<uint64_t>[]> slot(new std::atomic<uint64_t>[cap]);
    run([&](int t) {
      for (size_t i = cap * t / T; i < cap * (t + 1) / T; ++i)
        slot[i].store(0, std::memory_order_relaxed);
    });
    std::atomic<bool> dup{false};
    run([&](int t) {  // (shard + 1) << 40 | row: 0 = empty
      const std::hash<std::string_view> H;
      for (size_t r = 0; r < shards[t].rows.size() && !dup.load(std::memory_order_relaxed); ++r) {
        const std::string_view id = shards[t].rows[r].id;
        const uint64_t me = (uint64_t(t) + 1) << 40 | r;
        for (size_t i = H(id) & (cap - 1);; i = (i + 1) & (cap - 1)) {
          uint64_t cur = 0;
          if (slot[i].compare_exchange_strong(cur, me, std::memory_order_acq_rel)) break;
          const std::string_view other = shards[(cur >> 40) - 1].rows[cur & ((1ull << 40) - 1)].id;
          if (other == id) {
            dup.store(true);
            break;
          }
        }
      }
    });
    need_scan = dup.load();
  }
  lap("dupcheck-par");
  if (need_scan) {
    size_t total = 0;
    for (auto& sh : shards) total += sh.rows.size();
    std::unordered_set<std::string_view> seen;
    seen.reserve(total * 2);
    for (auto& sh : shards)
      for (size_t r = 0; r < sh.rows.size(); ++r) {
        if (first_err >= 0 && sh.line_no[r] > first_err) break;
        if (!seen.insert(sh.rows[r].id).second) {
          c->err_kind = 2;
          c->err_line = sh.line_no[r];
          c->err_msg = "duplicate id " + py_str_repr(sh.rows[r].id) + " at line " +
                       std::to_string(sh.line_no[r]);
          return GNB_EINVAL;
        }
      }
    if (first_err >= 0) {
      c->err_line = first_err;
      // corpus.py:159-160 checks duplicates before the rest of the record
      if (err_sh->err_has_id && seen.count(err_sh->err_id)) {
        c->err_kind = 2;
        c->err_msg = "duplicate id " + py_str_repr(err_sh->err_id) + " at line " +
                     std::to_string(first_err);
      }
      return GNB_EINVAL;
    }
  }
  lap("dupcheck");
  // global vocabulary: sorted union; remap shard-local ids
  std::vector<std::string> all;
  for (auto& sh : shards) all.insert(all.end(), sh.names.begin(), sh.names.end());
  std::sort(all.begin(), all.end());
  all.erase(std::unique(all.begin(), all.end()), all.end());
  c->vocab = all;
  std::unordered_map<std::string, int32_t> gid;
  gid.reserve(all.size() * 2);
  for (size_t k = 0; k < all.size(); ++k) gid.emplace(all[k], static_cast<int32_t>(k));
  std::vector<int64_t> row_off(T + 1, 0), ent_off(T + 1, 0);
  for (int t = 0; t < T; ++t) {
    row_off[t + 1] = row_off[t] + static_cast<int64_t>(shards[t].rows.size());
    ent_off[t + 1] = ent_off[t] + static_cast<int64_t>(shards[t].col.size());
  }
  const int64_t n = row_off[T], nnz = ent_off[T];
  c->ids.resize(n);
  c->size.resize(n);
  c->label.resize(n);
  c->row_ptr.resize_uninit(n + 1);
  c->col.resize_uninit(nnz);
  c->val.resize_uninit(nnz);
  c->row_ptr[0] = 0;
  lap("alloc");
  std::vector<int64_t> maxc(T, 0);
  run([&](int t) {  // scatter each shard into its slice of the global arrays
    Shard& sh = shards[t];
    std::vector<int32_t> map(sh.names.size());
    for (size_t k = 0; k < sh.names.size(); ++k) map[k] = gid.at(sh.names[k]);
    int64_t r = row_off[t], e = ent_off[t];
    for (auto& row : sh.rows) {
      c->ids[r] = std::move(row.id);
      c->size[r] = row.size;
      c->label[r] = row.label;
      for (int64_t k = row.e0; k < row.e1; ++k, ++e) {
        c->col[e] = map[sh.col[k]];
        c->val[e] = sh.val[k];
        maxc[t] = std::max(maxc[t], sh.val[k]);
      }
      c->row_ptr[++r] = e;
    }
  });
  for (int64_t m : maxc) c->max_count = std::max(c->max_count, m);
  lap("scatter");
  return GNB_OK;
}

void gnb_corpus_free(gnb_corpus* c) { delete c; }

int64_t gnb_corpus_rows(const gnb_corpus* c) { return c ? static_cast<int64_t>(c->ids.size()) : 0; }
int32_t gnb_corpus_vocab_size(const gnb_corpus* c) {
  return c ? static_cast<int32_t>(c->vocab.size()) : 0;
}
const char* gnb_corpus_vocab(const gnb_corpus* c, int32_t k) { return c->vocab[k].c_str(); }
const char* gnb_corpus_id(const gnb_corpus* c, int64_t r) { return c->ids[r].c_str(); }
int64_t gnb_corpus_max_count(const gnb_corpus* c) { return c->max_count; }
int64_t gnb_corpus_nnz(const gnb_corpus* c) { return static_cast<int64_t>(c->col.size()); }
int32_t gnb_corpus_error(const gnb_corpus* c, int64_t* line, const char** message) {
  if (line) *line = c->err_line;
  if (message) *message = c->err_msg.c_str();
  return c->err_kind;
}

// sizes (int64, -1 = beyond int64) and labels (1 malware, 0 benign, -1 none)
int gnb_corpus_meta(const gnb_corpus* c, int64_t* size_out, int8_t* label_out) {
  if (!c) return GNB_EINVAL;
  if (size_out) std::copy(c->size.begin(), c->size.end(), size_out);
  if (label_out) std::copy(c->label.begin(), c->label.end(), label_out);
  return GNB_OK;
}

// Dense rows [row0, row0 + n) into x (x_type storage, row pitch ldx elements,
// ldx >= vocab size); zero-filled first.  GNB_EINVAL if a count does not fit.
int gnb_corpus_dense(const gnb_corpus* c, int32_t x_type, void* x, int64_t ldx, int64_t row0,
                     int64_t n, int32_t threads) {
  if (!c || !x || row0 < 0 || n < 0 || row0 + n > static_cast<int64_t>(c->ids.size()) ||
      ldx < static_cast<int64_t>(c->vocab.size()))
    return GNB_EINVAL;
  const int64_t lim = x_type == GNB_X_U8 ? 255 : x_type == GNB_X_U16 ? 65535 : 2147483647;
  if (c->max_count > lim) return GNB_EINVAL;
  const int eb = x_type == GNB_X_U8 ? 1 : x_type == GNB_X_U16 ? 2 : 4;
  int T = threads > 0 ? threads : static_cast<int>(std::thread::hardware_concurrency());
  T = std::max(1, std::min<int>(T, 64));
  if (n < 65536) T = 1;
  auto work = [&](int t) {
    const int64_t lo = row0 + n * t / T, hi = row0 + n * (t + 1) / T;
    uint8_t* base = static_cast<uint8_t*>(x);
    memset(base + (lo - row0) * ldx * eb, 0, static_cast<size_t>((hi - lo) * ldx * eb));
    for (int64_t r = lo; r < hi; ++r) {
      uint8_t* row = base + (r - row0) * ldx * eb;
      for (int64_t k = c->row_ptr[r]; k < c->row_ptr[r + 1]; ++k) {
        const int64_t v = c->val[k];
        const int32_t j = c->col[k];
        if (eb == 1) row[j] = static_cast<uint8_t>(v);
        else if (eb == 2) reinterpret_cast<uint16_t*>(row)[j] = static_cast<uint16_t>(v);
        else reinterpret_cast<int32_t*>(row)[j] = static_cast<int32_t>(v);
      }
    }
  };
  std::vector<std::thread> th;
  for (int t = 1; t < T; ++t) th.emplace_back(work, t);
  work(0);
  for (auto& t : th) t.join();
  return GNB_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- prediction writer
namespace {

// json.dumps(str) with the default ensure_ascii=True
void json_str(std::string& o, const std::string& s) {
  o += '"';
  size_t i = 0;
  while (i < s.size()) {
    const unsigned char c = static_cast<unsigned char>(s[i]);
    if (c < 0x80) {
      ++i;
      switch (c) {
        case '"': o += "\\\""; break;
        case '\\': o += "\\\\"; break;
        case '\n': o += "\\n"; break;
        case '\r': o += "\\r"; break;
        case '\t': o += "\\t"; break;
        case '\b': o += "\\b"; break;
        case '\f': o += "\\f"; break;
        default:
          if (c < 0x20) {
            char b[8];
            snprintf(b, sizeof b, "\\u%04x", c);
            o += b;
          } else {
            o += static_cast<char>(c);
          }
      }
      continue;
    }
    // UTF-8 -> code point -> \uXXXX (surrogate pairs above U+FFFF)
    uint32_t cp = 0;
    int extra = c >= 0xF0 ? 3 : c >= 0xE0 ? 2 : 1;
    cp = c & (0x3F >> extra);
    ++i;
    for (int k = 0; k < extra && i < s.size(); ++k, ++i)
      cp = (cp << 6) | (static_cast<unsigned char>(s[i]) & 0x3F);
    char b[16];
    if (cp >= 0x10000) {
      cp -= 0x10000;
      snprintf(b, sizeof b, "\\u%04x\\u%04x", 0xD800 + (cp >> 10), 0xDC00 + (cp & 0x3FF));
    } else {
      snprintf(b, sizeof b, "\\u%04x", cp);
    }
    o += b;
  }
  o += '"';
}

void fmt17(std::string& o, double v) {  // format(v, ".17g")
  char b[40];
  snprintf(b, sizeof b, "%.17g", v);
  o += b;
}

}  // namespace

extern "C" {

// engine.write_predictions (pkg/src/groupnb/engine.py:466-481) for a parsed
// corpus: one JSONL object per row, 17-significant-digit floats, byte-identical
// to the reference's output.  label: 1 malware, 0 benign, < 0 size error;
// logpost [n][2] = (benign, malware).  *out_text is malloc'ed: gnb_free_text.
int gnb_corpus_write_predictions(const gnb_corpus* c, const int8_t* label, const double* logpost,
                                 const int32_t* effective_group, int64_t max_size_bytes,
                                 int32_t threads, char** out_text, size_t* out_len) {
  if (!c || !label || !logpost || !effective_group || !out_text || !out_len) return GNB_EINVAL;
  const int64_t n = static_cast<int64_t>(c->ids.size());
  int T = threads > 0 ? threads : static_cast<int>(std::thread::hardware_concurrency());
  T = std::max(1, std::min<int>(T, 64));
  if (n < 16384) T = 1;
  std::vector<std::string> part(T);
  auto work = [&](int t) {
    std::string& o = part[t];
    const int64_t lo = n * t / T, hi = n * (t + 1) / T;
    o.reserve(static_cast<size_t>(hi - lo) * 120);
    for (int64_t r = lo; r < hi; ++r) {
      o += "{\"id\": ";
      json_str(o, c->ids[r]);
      if (label[r] < 0) {
        o += ", \"error\": ";
        json_str(o, "size_bytes " + (c->size[r] >= 0 ? std::to_string(c->size[r])
                                                      : std::string("(huge)")) +
                        " outside [0, " + std::to_string(max_size_bytes) + ")");
        o += "}\n";
        continue;
      }
      o += label[r] == 1 ? ", \"label\": \"malware\"" : ", \"label\": \"benign\"";
      o += ", \"log_posterior\": {\"malware\": ";
      fmt17(o, logpost[2 * r + 1]);
      o += ", \"benign\": ";
      fmt17(o, logpost[2 * r]);
      o += "}, \"effective_group\": ";
      o += std::to_string(effective_group[r]);
      o += "}\n";
    }
  };
  std::vector<std::thread> th;
  for (int t = 1; t < T; ++t) th.emplace_back(work, t);
  work(0);
  for (auto& x : th) x.join();
  size_t total = 0;
  for (auto& p : part) total += p.size();
  char* buf = static_cast<char*>(malloc(total + 1));
  if (!buf) return GNB_ENOMEM;
  size_t off = 0;
  for (auto& p : part) {
    memcpy(buf + off, p.data(), p.size());
    off += p.size();
  }
  buf[total] = '\0';
  *out_text = buf;
  *out_len = total;
  return GNB_OK;
}

void gnb_free_text(char* p) { free(p); }

}  // extern "C"
