// Trace-record parser of the JSONL ingest:
// ingest_trace (reference: src/workload.cpp:115-153) restated as a
// per-line, allocation-free, host/device parser.
//
// A line is what std::getline yields (the bytes between '\n's).  Per line the
// reference does:
//   * skip it if it holds only " \t\r" (workload.cpp:121-122);
//   * nlohmann::json::parse(line) (3.11.3, workload.cpp:125): one JSON value,
//     surrounded by whitespace, a UTF-8 BOM allowed as the very first bytes;
//     strict RFC 8259 grammar, UTF-8 validated inside strings, surrogate
//     escapes paired, numbers that strtod rounds to infinity rejected
//     (out_of_range.406); duplicate object keys keep the LAST value;
//   * require an object containing "text_tokens" (workload.cpp:131-133);
//   * get<int64_t>() of text_tokens and get<vector<int64_t>>() of
//     image_subseqs / audio_subseqs when present (workload.cpp:134-142):
//     booleans, null, strings, arrays, objects are type errors; unsigned
//     integers are cast (wrapping) to int64, integers out of 64-bit range and
//     numbers with a fraction or exponent go through strtod and then
//     static_cast<int64_t> — truncation toward zero, INT64_MIN when the value
//     is outside the int64 range (x86 cvttsd2si);
//   * Sample::valid (src/core.cpp:97-113) in its order.
// Every failure before valid() is a TraceError "ParseError", valid()'s are
// "InvariantViolation" (errors.hpp:35-47).
//
// Number conversion is exact without big integers: only trunc(strtod(x)) and
// "strtod(x) is finite" are observable, and those need the correctly rounded
// double only when 0.1 <= |x| < 1e20 (u64 integer part + a comparison of the
// fraction digits with 1 - 2^-j) or 1e308 <= |x| < 1e309 (a comparison with
// the digits of the DBL_MAX/2^1024 midpoint); elsewhere the answer follows
// from the decimal magnitude alone.  Constants: jsonl_tables.cuh
// (tools/gen_jsonl_tables.py).
//
// Limits of this ABI (reported as J_UNSUPPORTED, never silently different):
// nesting deeper than kJMaxDepth, and values that pass valid() only through
// int64 wrap-around of the token total but do not fit the int32 CSR.
#pragma once

#ifdef __CUDACC__
#define DTB_HD __host__ __device__
#else
#define DTB_HD
#endif

#include "jsonl_tables.cuh"

namespace dtb {

enum JStatus : int { J_OK = 0, J_BLANK = 1, J_PARSE = 2, J_INVARIANT = 3, J_UNSUPPORTED = 4 };
enum JReason : int {
  JR_NONE = 0,
  JR_SYNTAX = 1,           // nlohmann parse_error.101
  JR_NUMBER_OVERFLOW = 2,  // nlohmann out_of_range.406
  JR_NOT_RECORD = 3,       // "record must be an object with text_tokens"
  JR_TEXT_TYPE = 4,        // type_error.302 on text_tokens
  JR_IMAGE_TYPE = 5,       // type_error.302 on image_subseqs
  JR_AUDIO_TYPE = 6,       // type_error.302 on audio_subseqs
  JR_NEG_TEXT = 10,        // "negative text token count"
  JR_NEG_SUBSEQ = 11,      // "negative subsequence token count"
  JR_NO_TOKENS = 12,       // "sample has no tokens"
  JR_OVER_CAP = 13,        // "sample exceeds the sequence length cap"
  JR_TOO_DEEP = 20,        // nesting beyond kJMaxDepth
  JR_INT32 = 21,           // a token count that does not fit the int32 CSR
};
constexpr int kJMaxDepth = 1024;

struct JLine {
  int status, reason;
  long long text;
  int n_img, n_aud;
  int img_at, aud_at;  // byte offset of the last image / audio value, -1 if absent
};

DTB_HD inline bool j_ws(int c) { return c == ' ' || c == '\t' || c == '\n' || c == '\r'; }
DTB_HD inline bool j_digit(int c) { return c >= '0' && c <= '9'; }
DTB_HD inline int j_hex(int c) {
  if (c >= '0' && c <= '9') return c - '0';
  if (c >= 'a' && c <= 'f') return c - 'a' + 10;
  if (c >= 'A' && c <= 'F') return c - 'A' + 10;
  return -1;
}
DTB_HD inline int j_bitlen(unsigned long long x) {
#ifdef __CUDA_ARCH__
  return 64 - __clzll(static_cast<long long>(x));
#else
  return x ? 64 - __builtin_clzll(x) : 0;
#endif
}

template <class B>
DTB_HD inline int j_hex4(const B& at, int p) {
  int v = 0;
  for (int k = 0; k < 4; ++k) {
    const int h = j_hex(at(p + k));
    if (h < 0) return -1;
    v = (v << 4) | h;
  }
  return v;
}

// String body starting after the opening quote; returns the position after
// the closing quote, -1 on a lexer error.  *key = 1/2/3 when the decoded
// string is "text_tokens" / "image_subseqs" / "audio_subseqs", else 0.
template <class B>
DTB_HD inline int j_string(const B& at, int p, int* key) {
  int cand = 0, k = 0;
  bool alive = true;
  auto name_at = [&](int i) -> int {
    const char* nm = cand == 1 ? "text_tokens" : cand == 2 ? "image_subseqs" : "audio_subseqs";
    return nm[i];
  };
  auto feed = [&](int byte) {  // byte < 0: a non-ASCII code point
    if (!alive) return;
    if (k == 0) cand = byte == 't' ? 1 : byte == 'i' ? 2 : byte == 'a' ? 3 : 0;
    if (cand == 0 || name_at(k) == 0 || name_at(k) != byte) {
      alive = false;
      return;
    }
    ++k;
  };
  for (;;) {
    const int c = at(p++);
    if (c < 0) return -1;
    if (c == '"') break;
    if (c == '\\') {
      const int e = at(p++);
      switch (e) {
        case '"': feed('"'); break;
        case '\\': feed('\\'); break;
        case '/': feed('/'); break;
        case 'b': feed(8); break;
        case 'f': feed(12); break;
        case 'n': feed(10); break;
        case 'r': feed(13); break;
        case 't': feed(9); break;
        case 'u': {
          int cp = j_hex4(at, p);
          if (cp < 0) return -1;
          p += 4;
          if (cp >= 0xD800 && cp <= 0xDBFF) {
            if (at(p) != '\\' || at(p + 1) != 'u') return -1;
            const int lo = j_hex4(at, p + 2);
            if (lo < 0xDC00 || lo > 0xDFFF) return -1;
            p += 6;
            cp = 0x10000;  // non-ASCII
          } else if (cp >= 0xDC00 && cp <= 0xDFFF) {
            return -1;
          }
          feed(cp < 0x80 ? cp : -1);
          break;
        }
        default: return -1;
      }
      continue;
    }
    if (c < 0x20) return -1;
    if (c < 0x80) {
      feed(c);
      continue;
    }
    // UTF-8 (nlohmann lexer::scan_string byte ranges)
    int lo1 = 0x80, hi1 = 0xBF, more = 0;
    if (c >= 0xC2 && c <= 0xDF) more = 1;
    else if (c == 0xE0) { more = 2; lo1 = 0xA0; }
    else if ((c >= 0xE1 && c <= 0xEC) || c == 0xEE || c == 0xEF) more = 2;
    else if (c == 0xED) { more = 2; hi1 = 0x9F; }
    else if (c == 0xF0) { more = 3; lo1 = 0x90; }
    else if (c >= 0xF1 && c <= 0xF3) more = 3;
    else if (c == 0xF4) { more = 3; hi1 = 0x8F; }
    else return -1;
    for (int q = 0; q < more; ++q) {
      const int b = at(p++);
      const int lo = q == 0 ? lo1 : 0x80, hi = q == 0 ? hi1 : 0xBF;
      if (b < lo || b > hi) return -1;
    }
    feed(-1);
  }
  *key = alive && cand != 0 && name_at(k) == 0 ? cand : 0;
  return p;
}

// End of the number token at p (RFC 8259 grammar), -1 if malformed.
template <class B>
DTB_HD inline int j_number_end(const B& at, int p) {
  if (at(p) == '-') ++p;
  const int c = at(p);
  if (c == '0') {
    ++p;
  } else if (c >= '1' && c <= '9') {
    while (j_digit(at(p))) ++p;
  } else {
    return -1;
  }
  if (at(p) == '.') {
    ++p;
    if (!j_digit(at(p))) return -1;
    while (j_digit(at(p))) ++p;
  }
  const int e = at(p);
  if (e == 'e' || e == 'E') {
    ++p;
    if (at(p) == '+' || at(p) == '-') ++p;
    if (!j_digit(at(p))) return -1;
    while (j_digit(at(p))) ++p;
  }
  return p;
}

// static_cast<int64_t>(value) of the number token [s, e) as nlohmann +
// libstdc++ compute it; returns 1 when strtod overflows (parse error).
template <class B>
DTB_HD inline int j_number_value(const B& at, int s, int e, long long* out) {
  constexpr long long kMin = static_cast<long long>(0x8000000000000000ull);
  int p = s;
  const bool neg = at(p) == '-';
  if (neg) ++p;
  const int i0 = p;
  while (p < e && j_digit(at(p))) ++p;
  const int i1 = p;
  int f0 = i1, f1 = i1;
  bool is_int = true;
  if (p < e && at(p) == '.') {
    is_int = false;
    f0 = ++p;
    while (p < e && j_digit(at(p))) ++p;
    f1 = p;
  }
  long long ex = 0;
  if (p < e) {  // exponent
    is_int = false;
    ++p;
    bool en = false;
    if (at(p) == '+' || at(p) == '-') {
      en = at(p) == '-';
      ++p;
    }
    for (; p < e; ++p)
      if (ex < 1000000000000ll) ex = ex * 10 + (at(p) - '0');
    if (en) ex = -ex;
  }
  if (is_int) {  // strtoull / strtoll when in range (lexer::scan_number)
    unsigned long long m = 0;
    bool ovf = false;
    for (int q = i0; q < i1; ++q) {
      const unsigned d = static_cast<unsigned>(at(q) - '0');
      if (m > (~0ull - d) / 10) {
        ovf = true;
        break;
      }
      m = m * 10 + d;
    }
    if (!ovf) {
      if (!neg) {
        *out = static_cast<long long>(m);
        return 0;
      }
      if (m <= 0x8000000000000000ull) {
        *out = static_cast<long long>(0ull - m);
        return 0;
      }
    }
  }
  // strtod + static_cast<int64_t>
  const long long nI = i1 - i0, nF = f1 - f0, nC = nI + nF;
  auto C = [&](long long k) -> int {
    return k < nI ? at(i0 + static_cast<int>(k)) - '0' : at(f0 + static_cast<int>(k - nI)) - '0';
  };
  long long z = 0;
  while (z < nC && C(z) == 0) ++z;
  if (z == nC) {
    *out = 0;
    return 0;
  }
  const long long mag = nI + ex - z;  // value in [10^(mag-1), 10^mag)
  auto S = [&](long long j) -> int { return z + j < nC ? C(z + j) : 0; };
  auto tail_nonzero = [&](long long j) -> bool {
    for (long long k = z + j; k < nC; ++k)
      if (C(k) != 0) return true;
    return false;
  };
  if (mag < 0) {  // |value| < 0.1
    *out = 0;
    return 0;
  }
  if (mag >= 310) return 1;
  if (mag == 309) {  // overflow iff >= 2^1024 - 2^970 (ties round to 2^1024)
    const char* M = jmax_digits();
    for (int j = 0; j < 309; ++j) {
      const int d = S(j), md = M[j] - '0';
      if (d != md) {
        if (d > md) return 1;
        *out = kMin;
        return 0;
      }
    }
    return 1;
  }
  if (mag >= 20) {  // 1e19 <= |value| < 1e308: finite, rounds to >= 2^63
    *out = kMin;
    return 0;
  }
  unsigned long long n = 0;  // integer part, < 1e19
  for (long long j = 0; j < mag; ++j) n = n * 10 + static_cast<unsigned>(S(j));
  // fraction 0.F (digits S(mag), S(mag+1), ...) against 1 - 2^-jj
  auto frac_cmp = [&](int jj) -> int {
    const char* T = jt_all() + jj * (jj - 1) / 2;
    for (int i = 0; i < jj; ++i) {
      const int d = S(mag + i), t = T[i] - '0';
      if (d != t) return d > t ? 1 : -1;
    }
    return tail_nonzero(mag + jj) ? 1 : 0;
  };
  unsigned long long m;
  const int b = j_bitlen(n);
  if (n == 0) {  // [0.1, 1): rounds to 1.0 iff >= 1 - 2^-54
    m = frac_cmp(54) >= 0 ? 1 : 0;
  } else if (b <= 53) {  // spacing 2^(b-53) <= 1: up to n+1 iff F >= 1 - 2^(b-54)
    const int c = frac_cmp(54 - b);
    const bool up = c > 0 || (c == 0 && (b <= 52 || (n & 1)));
    m = up ? n + 1 : n;
  } else {  // spacing u = 2^(b-53) >= 2
    const int sh = b - 53;
    const unsigned long long u = 1ull << sh, r = n & (u - 1), half = u >> 1, n0 = n - r;
    const bool fz = !tail_nonzero(mag);
    const bool up = r > half || (r == half && (!fz || ((n0 >> sh) & 1)));
    m = up ? n0 + u : n0;
  }
  if (m >= 0x8000000000000000ull) *out = kMin;
  else *out = neg ? -static_cast<long long>(m) : static_cast<long long>(m);
  return 0;
}

template <class B>
DTB_HD inline bool j_number_start(const B& at, int p) {
  const int c = at(p);
  return c == '-' || j_digit(c);
}

// Pass 1: parse and validate one line of `len` bytes.
template <class B>
DTB_HD inline JLine j_parse_line(const B& at, int len, long long seq_len_cap) {
  JLine r;
  r.status = J_OK;
  r.reason = JR_NONE;
  r.text = 0;
  r.n_img = r.n_aud = 0;
  r.img_at = r.aud_at = -1;
  bool blank = true;
  for (int i = 0; i < len; ++i) {
    const int c = at(i);
    if (c != ' ' && c != '\t' && c != '\r') {
      blank = false;
      break;
    }
  }
  if (blank) {
    r.status = J_BLANK;
    return r;
  }
  auto fail = [&](int st, int why) {
    r.status = st;
    r.reason = why;
    return r;
  };
  int p = 0;
  if (at(0) == 0xEF) {
    if (at(1) != 0xBB || at(2) != 0xBF) return fail(J_PARSE, JR_SYNTAX);
    p = 3;
  }
  unsigned stk[kJMaxDepth / 32];
  int depth = 0, text_at = -1, pending = 0;
  bool top_obj = false, want_value = true;
  auto is_obj = [&]() { return (stk[(depth - 1) >> 5] >> ((depth - 1) & 31)) & 1u; };
  auto push = [&](bool obj) {
    const unsigned bit = 1u << (depth & 31);
    if (obj) stk[depth >> 5] |= bit;
    else stk[depth >> 5] &= ~bit;
    ++depth;
  };
  auto key_then_colon = [&]() -> bool {  // at '"' of a key
    if (at(p) != '"') return false;
    int key = 0;
    p = j_string(at, p + 1, &key);
    if (p < 0) return false;
    while (j_ws(at(p))) ++p;
    if (at(p) != ':') return false;
    ++p;
    pending = depth == 1 ? key : 0;
    return true;
  };
  for (;;) {
    while (j_ws(at(p))) ++p;
    if (want_value) {
      if (pending != 0) {
        if (pending == 1) text_at = p;
        else if (pending == 2) r.img_at = p;
        else r.aud_at = p;
        pending = 0;
      }
      const int c = at(p);
      if (c == '{' || c == '[') {
        if (depth == kJMaxDepth) return fail(J_UNSUPPORTED, JR_TOO_DEEP);
        if (depth == 0) top_obj = c == '{';
        push(c == '{');
        ++p;
        while (j_ws(at(p))) ++p;
        if (at(p) == (c == '{' ? '}' : ']')) {
          ++p;
          --depth;
          want_value = false;
          continue;
        }
        if (c == '{' && !key_then_colon()) return fail(J_PARSE, JR_SYNTAX);
        continue;  // a value follows
      }
      if (c == '"') {
        int key = 0;
        p = j_string(at, p + 1, &key);
        if (p < 0) return fail(J_PARSE, JR_SYNTAX);
      } else if (c == 't' || c == 'f' || c == 'n') {
        const char* lit = c == 't' ? "true" : c == 'f' ? "false" : "null";
        for (int k = 0; lit[k]; ++k)
          if (at(p + k) != lit[k]) return fail(J_PARSE, JR_SYNTAX);
        p += c == 'f' ? 5 : 4;
      } else if (j_number_start(at, p)) {
        const int e = j_number_end(at, p);
        if (e < 0) return fail(J_PARSE, JR_SYNTAX);
        long long v;
        if (j_number_value(at, p, e, &v)) return fail(J_PARSE, JR_NUMBER_OVERFLOW);
        p = e;
      } else {
        return fail(J_PARSE, JR_SYNTAX);
      }
      want_value = false;
      continue;
    }
    if (depth == 0) {
      if (at(p) != -1) return fail(J_PARSE, JR_SYNTAX);  // expected end of input
      break;
    }
    const int c = at(p);
    const bool obj = is_obj();
    if (c == ',') {
      ++p;
      if (obj) {
        while (j_ws(at(p))) ++p;
        if (!key_then_colon()) return fail(J_PARSE, JR_SYNTAX);
      }
      want_value = true;
      continue;
    }
    if (c == (obj ? '}' : ']')) {
      ++p;
      --depth;
      continue;
    }
    return fail(J_PARSE, JR_SYNTAX);
  }
  if (!top_obj || text_at < 0) return fail(J_PARSE, JR_NOT_RECORD);
  // get<int64_t> / get<vector<int64_t>> (type errors before valid())
  if (!j_number_start(at, text_at)) return fail(J_PARSE, JR_TEXT_TYPE);
  j_number_value(at, text_at, j_number_end(at, text_at), &r.text);
  unsigned long long total = static_cast<unsigned long long>(r.text);
  bool neg_sub = false, big = r.text > 0x7fffffff;
  auto array = [&](int a, int* cnt) -> bool {
    if (at(a) != '[') return false;
    int q = a + 1;
    for (;;) {
      while (j_ws(at(q))) ++q;
      if (at(q) == ']') return true;
      if (!j_number_start(at, q)) return false;
      const int e = j_number_end(at, q);
      long long v;
      j_number_value(at, q, e, &v);
      ++*cnt;
      if (v < 0) neg_sub = true;
      if (v > 0x7fffffff) big = true;
      total += static_cast<unsigned long long>(v);
      q = e;
      while (j_ws(at(q))) ++q;
      if (at(q) == ',') ++q;
    }
  };
  if (r.img_at >= 0 && !array(r.img_at, &r.n_img)) return fail(J_PARSE, JR_IMAGE_TYPE);
  const bool neg_img = neg_sub;
  if (r.aud_at >= 0 && !array(r.aud_at, &r.n_aud)) return fail(J_PARSE, JR_AUDIO_TYPE);
  // Sample::valid (src/core.cpp:97-113); total_tokens wraps like int64
  if (r.text < 0) return fail(J_INVARIANT, JR_NEG_TEXT);
  if (neg_img || neg_sub) return fail(J_INVARIANT, JR_NEG_SUBSEQ);
  const long long tot = static_cast<long long>(total);
  if (tot < 1) return fail(J_INVARIANT, JR_NO_TOKENS);
  if (tot > seq_len_cap) return fail(J_INVARIANT, JR_OVER_CAP);
  if (big) return fail(J_UNSUPPORTED, JR_INT32);
  return r;
}

// Fast path for the canonical record layout write_trace produces
// (src/workload.cpp:157-165, nlohmann dump: no whitespace, keys in order):
//   {"text_tokens":N[,"image_subseqs":[N,...]][,"audio_subseqs":[N,...]]}
// with N = 0 | [1-9][0-9]{0,8}.  On such a line the general parser's result
// is exactly: text = N, the arrays' values, no duplicate keys, nothing else
// to validate but the token total (no int64 wrap: every N < 1e9).  Any other
// byte sequence returns false and the caller runs j_parse_line.
template <class B>
DTB_HD inline bool j_fast_uint(const B& at, int* p, long long* v) {
  int c = at(*p);
  if (c < '0' || c > '9') return false;
  long long x = c - '0';
  ++*p;
  if (x == 0) {
    c = at(*p);
    if (c >= '0' && c <= '9') return false;
    *v = 0;
    return true;
  }
  for (int k = 1;; ++k) {
    c = at(*p);
    if (c < '0' || c > '9') break;
    if (k == 9) return false;
    x = x * 10 + (c - '0');
    ++*p;
  }
  *v = x;
  return true;
}

// literal match, unrolled so every character is an immediate
template <class B, int N>
DTB_HD inline bool j_fast_lit(const B& at, int* p, const char (&lit)[N]) {
#pragma unroll
  for (int k = 0; k < N - 1; ++k)
    if (at(*p + k) != static_cast<unsigned char>(lit[k])) return false;
  *p += N - 1;
  return true;
}

template <class B>
DTB_HD inline bool j_fast_list(const B& at, int* p, int* cnt, long long* sum) {
  if (at(*p) == ']') {
    ++*p;
    return true;
  }
  for (;;) {
    long long v;
    if (!j_fast_uint(at, p, &v)) return false;
    ++*cnt;
    *sum += v;
    const int c = at(*p);
    ++*p;
    if (c == ']') return true;
    if (c != ',') return false;
  }
}

template <class B>
DTB_HD inline bool j_fast_line(const B& at, int len, long long seq_len_cap, JLine* r) {
  int p = 0;
  if (!j_fast_lit(at, &p, "{\"text_tokens\":")) return false;
  long long text, sum = 0;
  if (!j_fast_uint(at, &p, &text)) return false;
  int n_img = 0, n_aud = 0, img_at = -1, aud_at = -1;
  if (at(p) == ',' && at(p + 2) == 'i') {
    if (!j_fast_lit(at, &p, ",\"image_subseqs\":[")) return false;
    img_at = p - 1;
    if (!j_fast_list(at, &p, &n_img, &sum)) return false;
  }
  if (at(p) == ',') {
    if (!j_fast_lit(at, &p, ",\"audio_subseqs\":[")) return false;
    aud_at = p - 1;
    if (!j_fast_list(at, &p, &n_aud, &sum)) return false;
  }
  if (at(p) != '}' || p + 1 != len) return false;
  r->text = text;
  r->n_img = n_img;
  r->n_aud = n_aud;
  r->img_at = img_at;
  r->aud_at = aud_at;
  const long long tot = text + sum;
  r->status = J_OK;
  r->reason = JR_NONE;
  if (tot < 1) {
    r->status = J_INVARIANT;
    r->reason = JR_NO_TOKENS;
  } else if (tot > seq_len_cap) {
    r->status = J_INVARIANT;
    r->reason = JR_OVER_CAP;
  }
  return true;
}

// One line: the canonical fast path, else the general parser.
template <class B>
DTB_HD inline JLine j_parse_record(const B& at, int len, long long seq_len_cap, bool* fast) {
  JLine r;
  *fast = j_fast_line(at, len, seq_len_cap, &r);
  if (*fast) return r;
  return j_parse_line(at, len, seq_len_cap);
}

// Pass 2 on a fast-path line: plain unsigned digits.
template <class B>
DTB_HD inline void j_write_array_fast(const B& at, int a, int* dst) {
  int q = a + 1, k = 0;
  if (at(q) == ']') return;
  for (;;) {
    int v = 0, c;
    while ((c = at(q)) >= '0' && c <= '9') {
      v = v * 10 + (c - '0');
      ++q;
    }
    dst[k++] = v;
    if (at(q++) == ']') return;
  }
}

// Pass 2: the values of a validated array at byte a, as int32.
template <class B>
DTB_HD inline void j_write_array(const B& at, int a, int* dst) {
  int q = a + 1, k = 0;
  for (;;) {
    while (j_ws(at(q))) ++q;
    if (at(q) == ']') return;
    const int e = j_number_end(at, q);
    long long v;
    j_number_value(at, q, e, &v);
    dst[k++] = static_cast<int>(v);
    q = e;
    while (j_ws(at(q))) ++q;
    if (at(q) == ',') ++q;
  }
}

}  // namespace dtb
