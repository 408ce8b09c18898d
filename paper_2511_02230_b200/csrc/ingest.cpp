// ingest.cpp — host-side trace ingest (NEXT-4): the tool-call parser of §5.2 /
// App. A and the JSONL trace loader (SPEC.md:144-178 interfaces).
// Host code only: no CUDA call.  Readings R33-R35.
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string>
#include <unordered_set>
#include <utility>
#include <vector>

#include "ct_internal.h"

namespace {

// ---- a small strict JSON reader (RFC 8259 grammar; duplicate keys: the last one wins) ----------
struct JVal {
  enum Kind { NUL, BOOL, NUM, STR, ARR, OBJ } k = NUL;
  bool b = false;
  std::string s;  // STR: decoded UTF-8; NUM: the number's text
  std::vector<JVal> a;
  std::vector<std::pair<std::string, JVal>> o;

  const JVal* get(const char* key) const {
    if (k != OBJ) return nullptr;
    for (size_t i = o.size(); i-- > 0;)
      if (o[i].first == key) return &o[i].second;
    return nullptr;
  }
};

struct JParser {
  const char* p;
  const char* e;
  bool ok = true;

  static bool ws(char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\r'; }
  void skip() {
    while (p < e && ws(*p)) ++p;
  }
  bool lit(const char* w) {
    size_t n = strlen(w);
    if ((size_t)(e - p) < n || memcmp(p, w, n) != 0) return false;
    p += n;
    return true;
  }
  static void put_utf8(std::string& out, uint32_t cp) {
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
  }
  bool hex4(uint32_t& v) {
    if (e - p < 4) return false;
    v = 0;
    for (int i = 0; i < 4; ++i) {
      char c = *p++;
      v <<= 4;
      if (c >= '0' && c <= '9') v |= (uint32_t)(c - '0');
      else if (c >= 'a' && c <= 'f') v |= (uint32_t)(c - 'a' + 10);
      else if (c >= 'A' && c <= 'F') v |= (uint32_t)(c - 'A' + 10);
      else return false;
    }
    return true;
  }
  bool str(std::string& out) {
    if (p >= e || *p != '"') return false;
    ++p;
    while (p < e) {
      unsigned char c = (unsigned char)*p++;
      if (c == '"') return true;
      if (c < 0x20) return false;
      if (c != '\\') {
        out += (char)c;
        continue;
      }
      if (p >= e) return false;
      char x = *p++;
      switch (x) {
        case '"': out += '"'; break;
        case '\\': out += '\\'; break;
        case '/': out += '/'; break;
        case 'b': out += '\b'; break;
        case 'f': out += '\f'; break;
        case 'n': out += '\n'; break;
        case 'r': out += '\r'; break;
        case 't': out += '\t'; break;
        case 'u': {
          uint32_t v;
          if (!hex4(v)) return false;
          if (v >= 0xD800 && v < 0xDC00 && e - p >= 6 && p[0] == '\\' && p[1] == 'u') {
            const char* save = p;
            p += 2;
            uint32_t lo;
            if (hex4(lo) && lo >= 0xDC00 && lo < 0xE000) {
              v = 0x10000 + ((v - 0xD800) << 10) + (lo - 0xDC00);
            } else {
              p = save;
            }
          }
          put_utf8(out, v);
          break;
        }
        default:
          return false;
      }
    }
    return false;
  }
  bool num(std::string& out) {
    const char* s = p;
    if (p < e && *p == '-') ++p;
    if (p >= e) return false;
    if (*p == '0') {
      ++p;
    } else if (*p >= '1' && *p <= '9') {
      while (p < e && *p >= '0' && *p <= '9') ++p;
    } else {
      return false;
    }
    if (p < e && *p == '.') {
      ++p;
      const char* d = p;
      while (p < e && *p >= '0' && *p <= '9') ++p;
      if (p == d) return false;
    }
    if (p < e && (*p == 'e' || *p == 'E')) {
      ++p;
      if (p < e && (*p == '+' || *p == '-')) ++p;
      const char* d = p;
      while (p < e && *p >= '0' && *p <= '9') ++p;
      if (p == d) return false;
    }
    out.assign(s, p);
    return true;
  }
  bool value(JVal& v, int depth) {
    if (depth > 64) return false;
    skip();
    if (p >= e) return false;
    char c = *p;
    if (c == '{') {
      ++p;
      v.k = JVal::OBJ;
      skip();
      if (p < e && *p == '}') { ++p; return true; }
      for (;;) {
        skip();
        std::string key;
        if (!str(key)) return false;
        skip();
        if (p >= e || *p != ':') return false;
        ++p;
        v.o.emplace_back(std::move(key), JVal());
        if (!value(v.o.back().second, depth + 1)) return false;
        skip();
        if (p < e && *p == ',') { ++p; continue; }
        if (p < e && *p == '}') { ++p; return true; }
        return false;
      }
    }
    if (c == '[') {
      ++p;
      v.k = JVal::ARR;
      skip();
      if (p < e && *p == ']') { ++p; return true; }
      for (;;) {
        v.a.emplace_back();
        if (!value(v.a.back(), depth + 1)) return false;
        skip();
        if (p < e && *p == ',') { ++p; continue; }
        if (p < e && *p == ']') { ++p; return true; }
        return false;
      }
    }
    if (c == '"') { v.k = JVal::STR; return str(v.s); }
    if (lit("true")) { v.k = JVal::BOOL; v.b = true; return true; }
    if (lit("false")) { v.k = JVal::BOOL; v.b = false; return true; }
    if (lit("null")) { v.k = JVal::NUL; return true; }
    v.k = JVal::NUM;
    return num(v.s);
  }
};

// Parses exactly one JSON document spanning [b, e) (surrounding JSON whitespace allowed).
bool parse_json(const char* b, const char* e, JVal& out) {
  JParser q{b, e};
  if (!q.value(out, 0)) return false;
  q.skip();
  return q.p == e;
}

// ---- tool-call parsing (App. A) ----------------------------------------------
bool is_space(char c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\v' || c == '\f';
}

std::string trim(const std::string& s) {
  size_t b = 0, e = s.size();
  while (b < e && is_space(s[b])) ++b;
  while (e > b && is_space(s[e - 1])) --e;
  return s.substr(b, e - b);
}

// App. A: "locate the single bash code block, split the command string on && or ||, then parse
// each sub-command: the first token is the executable/function name"; "use the
// first word as the tool call name".  Reading R33: the name is the first token of the first
// sub-command; the ```bash fence is used when present, else the whole text is the command.
std::string bash_name(const std::string& msg) {
  std::string cmd = msg;
  size_t f = msg.find("```bash");
  if (f != std::string::npos) {
    size_t b = msg.find('\n', f);
    b = b == std::string::npos ? msg.size() : b + 1;
    size_t c = msg.find("```", b);
    cmd = msg.substr(b, (c == std::string::npos ? msg.size() : c) - b);
  }
  size_t cut = cmd.size();
  size_t a1 = cmd.find("&&"), a2 = cmd.find("||");
  if (a1 != std::string::npos) cut = std::min(cut, a1);
  if (a2 != std::string::npos) cut = std::min(cut, a2);
  size_t i = 0;
  while (i < cut && is_space(cmd[i])) ++i;
  size_t j = i;
  while (j < cut && !is_space(cmd[j])) ++j;
  return cmd.substr(i, j - i);
}

bool call_type(const std::string& t) {
  return t == "function_call" || t == "function" || t == "tool_call" || t == "tool_use";
}

// The name of an OpenAI-schema call block: "name", else "function"."name".
const JVal* call_name(const JVal& blk) {
  const JVal* n = blk.get("name");
  if (n && n->k == JVal::STR) return n;
  const JVal* fn = blk.get("function");
  if (fn) {
    n = fn->get("name");
    if (n && n->k == JVal::STR) return n;
  }
  return nullptr;
}

// The blocks of a structured message: an array's elements, the "tool_calls" / "output" array
// of a message object, else the object itself.
std::vector<const JVal*> blocks_of(const JVal& v) {
  std::vector<const JVal*> out;
  const JVal* arr = nullptr;
  if (v.k == JVal::ARR) arr = &v;
  else if (const JVal* t = v.get("tool_calls"); t && t->k == JVal::ARR) arr = t;
  else if (const JVal* o = v.get("output"); o && o->k == JVal::ARR) arr = o;
  if (arr) {
    for (const JVal& x : arr->a) out.push_back(&x);
  } else {
    out.push_back(&v);
  }
  return out;
}

enum Res { R_NONE = 0, R_NAME = 1, R_BAD = 2 };

// OPENAI rule: the first block whose type indicates a call gives its name.
// With `name_rule`, a block without "type" that has a string "name" also counts (Qwen-3, App. A).
Res json_rule(const JVal& v, bool type_rule, bool name_rule, std::string& name) {
  for (const JVal* blk : blocks_of(v)) {
    if (blk->k != JVal::OBJ) continue;
    const JVal* t = blk->get("type");
    if (type_rule && t) {
      if (t->k == JVal::STR && call_type(t->s)) {
        const JVal* n = call_name(*blk);
        if (!n || n->s.empty()) return R_BAD;
        name = n->s;
        return R_NAME;
      }
      continue;
    }
    if (name_rule && !t) {
      const JVal* n = blk->get("name");
      if (!n) continue;
      if (n->k != JVal::STR || n->s.empty()) return R_BAD;
      name = n->s;
      return R_NAME;
    }
  }
  return R_NONE;
}

Res terminal_rule(const JVal& v, std::string& name) {
  const JVal* c = v.get("commands");
  if (!c) return R_NONE;
  if (c->k != JVal::ARR) return R_BAD;
  if (c->a.empty()) return R_NONE;
  const JVal* ks = c->a[0].get("keystrokes");
  if (!ks || ks->k != JVal::STR) return R_BAD;
  name = bash_name(ks->s);
  return name.empty() ? R_NONE : R_NAME;
}

bool ident_start(char c) { return (c >= 'A' && c <= 'Z') || (c >= 'a' && c <= 'z') || c == '_'; }
bool ident_char(char c) { return ident_start(c) || (c >= '0' && c <= '9') || c == '.'; }

// Llama-3 style "f(p1=v1, ...)" or "[f(...), g(...)]" (App. A): the first call's identifier.
Res pythonic_rule(const std::string& msg, std::string& name) {
  std::string t = trim(msg);
  if (t.size() >= 2 && t.front() == '[' && t.back() == ']') t = trim(t.substr(1, t.size() - 2));
  if (t.empty() || !ident_start(t[0]) || t.back() != ')') return R_NONE;
  size_t i = 1;
  while (i < t.size() && ident_char(t[i])) ++i;
  size_t j = i;
  while (j < t.size() && is_space(t[j])) ++j;
  if (j >= t.size() || t[j] != '(') return R_NONE;
  name = t.substr(0, i);
  return R_NAME;
}

Res parse_message(const std::string& msg, int fmt, std::string& name) {
  name.clear();
  std::string t = trim(msg);
  switch (fmt) {
    case CT_TOOLFMT_BASH: {
      name = bash_name(msg);
      return name.empty() ? R_NONE : R_NAME;
    }
    case CT_TOOLFMT_PYTHONIC:
      return pythonic_rule(msg, name);
    case CT_TOOLFMT_OPENAI:
    case CT_TOOLFMT_NAME:
    case CT_TOOLFMT_TERMINAL: {
      JVal v;
      if (!parse_json(t.data(), t.data() + t.size(), v)) return R_BAD;
      if (fmt == CT_TOOLFMT_TERMINAL) return terminal_rule(v, name);
      return json_rule(v, fmt == CT_TOOLFMT_OPENAI, fmt == CT_TOOLFMT_NAME, name);
    }
    default:
      break;
  }
  // AUTO (reading R33): structured blocks first, then a bash fence, then a pythonic call.
  static const char kOpen[] = "<tool_call>", kClose[] = "</tool_call>";
  if (t.compare(0, sizeof kOpen - 1, kOpen) == 0) {
    size_t c = t.find(kClose);
    t = trim(t.substr(sizeof kOpen - 1, (c == std::string::npos ? t.size() : c) - (sizeof kOpen - 1)));
  }
  if (!t.empty() && (t[0] == '{' || t[0] == '[')) {
    JVal v;
    if (!parse_json(t.data(), t.data() + t.size(), v)) return R_BAD;
    if (v.get("commands")) return terminal_rule(v, name);
    return json_rule(v, true, true, name);
  }
  if (msg.find("```bash") != std::string::npos) {
    name = bash_name(msg);
    return name.empty() ? R_NONE : R_NAME;
  }
  return pythonic_rule(msg, name);
}

// ---- number conversions ------------------------------------------------------------------------
// A JSON number's exact decimal value times 10^6, rounded half away from zero (R34).
bool decimal_to_us(const std::string& num, int64_t& out) {
  size_t i = 0;
  bool neg = false;
  if (i < num.size() && num[i] == '-') { neg = true; ++i; }
  std::string digits;
  int64_t exp10 = 6;
  while (i < num.size() && num[i] >= '0' && num[i] <= '9') digits += num[i++];
  if (i < num.size() && num[i] == '.') {
    ++i;
    while (i < num.size() && num[i] >= '0' && num[i] <= '9') { digits += num[i++]; --exp10; }
  }
  if (i < num.size() && (num[i] == 'e' || num[i] == 'E')) {
    ++i;
    bool eneg = false;
    if (i < num.size() && (num[i] == '+' || num[i] == '-')) eneg = num[i++] == '-';
    int64_t x = 0;
    while (i < num.size() && num[i] >= '0' && num[i] <= '9') {
      x = std::min<int64_t>(x * 10 + (num[i++] - '0'), 1000000);
    }
    exp10 += eneg ? -x : x;
  }
  size_t nz = digits.find_first_not_of('0');
  digits = nz == std::string::npos ? std::string() : digits.substr(nz);
  unsigned __int128 v = 0;
  const unsigned __int128 lim = (unsigned __int128)1 << 62;
  if (exp10 >= 0) {
    for (char c : digits) {
      v = v * 10 + (unsigned)(c - '0');
      if (v >= lim) return false;
    }
    for (int64_t k = 0; k < exp10 && v != 0; ++k) {
      v *= 10;
      if (v >= lim) return false;
    }
  } else {
    int64_t keep = (int64_t)digits.size() + exp10;  // digits left of the rounding point
    for (int64_t k = 0; k < keep; ++k) {
      v = v * 10 + (unsigned)(digits[k] - '0');
      if (v >= lim) return false;
    }
    if (keep >= 0 && keep < (int64_t)digits.size() && digits[keep] >= '5') ++v;
  }
  if (v >= lim) return false;
  out = neg ? -(int64_t)v : (int64_t)v;
  return true;
}

// A JSON integer (no fraction, no exponent) in [lo, hi].
bool json_int(const JVal& v, int64_t lo, int64_t hi, int64_t& out) {
  if (v.k != JVal::NUM) return false;
  if (v.s.find_first_of(".eE") != std::string::npos) return false;
  if (v.s.size() > 19) return false;
  long long x = strtoll(v.s.c_str(), nullptr, 10);
  if (x < lo || x > hi) return false;
  out = x;
  return true;
}

struct LTurn {
  int32_t nw, dec;
  std::string tool;  // empty on the final turn
  int64_t dur;
};
struct LProg {
  int64_t arr;
  int64_t line;
  std::vector<LTurn> turns;
};

int fail_line(int64_t* counts, int64_t line, const std::string& what) {
  char buf[600];
  snprintf(buf, sizeof buf, "line %lld: %s", (long long)line, what.c_str());
  ct::set_last_error(buf);
  if (counts) counts[4] = line;
  return CT_EINVAL;
}

int fail_msg(const char* what) {
  ct::set_last_error(what);
  return CT_EINVAL;
}

}  // namespace

extern "C" {

int ct_parse_tool_name(const char* msg, int64_t len, int32_t format, char* name, int32_t name_cap,
                       int32_t* name_len, int32_t* malformed) {
  if (!msg || len < 0 || !name || name_cap < 1 || !name_len || !malformed)
    return fail_msg("ct_parse_tool_name: NULL pointer or negative length");
  if (format < CT_TOOLFMT_AUTO || format > CT_TOOLFMT_TERMINAL)
    return fail_msg("ct_parse_tool_name: unknown format");
  std::string s;
  Res r;
  try {
    r = parse_message(std::string(msg, (size_t)len), format, s);
  } catch (...) {
    return fail_msg("ct_parse_tool_name: allocation failed");
  }
  *malformed = r == R_BAD ? 1 : 0;
  if (r != R_NAME) s.clear();
  if ((int64_t)s.size() > (int64_t)name_cap - 1) return fail_msg("ct_parse_tool_name: name_cap too small");
  memcpy(name, s.data(), s.size());
  name[s.size()] = 0;
  *name_len = (int32_t)s.size();
  return CT_OK;
}

int ct_load_trace_jsonl(const char* path, int32_t format, int64_t ctx_window, char* tool_names,
                        int32_t n_known, ct_program* programs, int64_t programs_cap,
                        ct_turn* turns, int64_t turns_cap, int64_t* counts) {
  if (!path || !counts) return fail_msg("ct_load_trace_jsonl: NULL path or counts");
  for (int i = 0; i < 5; ++i) counts[i] = 0;
  if (format < CT_TOOLFMT_AUTO || format > CT_TOOLFMT_TERMINAL)
    return fail_msg("ct_load_trace_jsonl: unknown format");
  if (n_known < 0 || n_known > CT_MAX_TOOLS || (n_known > 0 && !tool_names))
    return fail_msg("ct_load_trace_jsonl: n_known out of range or tool_names NULL");
  try {
    std::vector<std::string> names;
    for (int i = 0; i < n_known; ++i) {
      const char* e = tool_names + 64 * i;
      size_t n = strnlen(e, 64);
      if (n == 0 || n > 63) return fail_msg("ct_load_trace_jsonl: known tool names must be 1..63 bytes");
      std::string nm(e, n);
      if (std::find(names.begin(), names.end(), nm) != names.end())
        return fail_msg("ct_load_trace_jsonl: duplicate known tool name");
      names.push_back(nm);
    }
    std::ifstream in(path, std::ios::binary);
    if (!in) return fail_msg("ct_load_trace_jsonl: cannot open file");
    std::vector<LProg> progs;
    std::unordered_set<std::string> ids;
    std::string line;
    int64_t ln = 0, warnings = 0;
    const int64_t kI32 = 0x7FFFFFFF;
    while (std::getline(in, line)) {
      ++ln;
      if (!line.empty() && line.back() == '\r') line.pop_back();
      if (trim(line).empty()) continue;
      JVal rec;
      if (!parse_json(line.data(), line.data() + line.size(), rec)) return fail_line(counts, ln, "invalid JSON");
      if (rec.k != JVal::OBJ) return fail_line(counts, ln, "record is not an object");
      const JVal* pid = rec.get("program_id");
      if (!pid || (pid->k != JVal::STR && pid->k != JVal::NUM))
        return fail_line(counts, ln, "program_id: missing or not a string/number");
      if (!ids.insert(pid->s).second) return fail_line(counts, ln, "program_id: duplicate '" + pid->s + "'");
      const JVal* at = rec.get("arrival_time_s");
      LProg pr;
      pr.line = ln;
      // arr_q = arrival µs replays at gap_us = 2^20, so arrivals stay below 2^42 µs
      // (ct_simulate_batch: arr_q x gap < 2^62)
      if (!at || at->k != JVal::NUM || !decimal_to_us(at->s, pr.arr) || pr.arr < 0 ||
          pr.arr >= (1ll << 42))
        return fail_line(counts, ln, "arrival_time_s: missing, negative or out of range");
      const JVal* ts = rec.get("turns");
      if (!ts || ts->k != JVal::ARR || ts->a.empty())
        return fail_line(counts, ln, "turns: missing, not a list or empty");
      if (ts->a.size() > CT_MAX_TURNS) return fail_line(counts, ln, "turns: more than CT_MAX_TURNS");
      int64_t cum = 0;
      for (size_t k = 0; k < ts->a.size(); ++k) {
        const JVal& tv = ts->a[k];
        const std::string tk = "turns[" + std::to_string(k) + "].";
        if (tv.k != JVal::OBJ) return fail_line(counts, ln, tk + ": not an object");
        const bool last = k + 1 == ts->a.size();
        LTurn t;
        int64_t x;
        const JVal* f = tv.get("new_prompt_tokens");
        if (!f || !json_int(*f, 0, kI32, x)) return fail_line(counts, ln, tk + "new_prompt_tokens: missing or not an integer >= 0");
        t.nw = (int32_t)x;
        f = tv.get("decode_tokens");
        if (!f || !json_int(*f, 1, kI32, x)) return fail_line(counts, ln, tk + "decode_tokens: missing or not an integer >= 1");
        t.dec = (int32_t)x;
        cum += (int64_t)t.nw + t.dec;
        if (cum > CT_MAX_CONTEXT)
          return fail_line(counts, ln, tk + "new_prompt_tokens: total context above CT_MAX_CONTEXT");
        if (ctx_window > 0 && cum > ctx_window)
          return fail_line(counts, ln, tk + "new_prompt_tokens: cumulative context exceeds the context window");
        const JVal* tn = tv.get("tool_name");
        const JVal* td = tv.get("tool_duration_s");
        const JVal* ms = tv.get("message");
        if (last) {
          if (tn || td) return fail_line(counts, ln, tk + "tool_name: present on the final turn");
          t.dur = 0;
        } else {
          if (!td) return fail_line(counts, ln, tk + "tool_duration_s: missing on a non-final turn");
          if (td->k != JVal::NUM || !decimal_to_us(td->s, t.dur) || t.dur < 0)
            return fail_line(counts, ln, tk + "tool_duration_s: not a number >= 0 or out of range");
          if (t.dur < 1) t.dur = 1;  // R25: a tool call lasts at least 1 µs
          if (t.dur > kI32) return fail_line(counts, ln, tk + "tool_duration_s: above 2^31 µs");
          if (tn) {
            if (tn->k != JVal::STR || tn->s.empty() || tn->s.size() > 63)
              return fail_line(counts, ln, tk + "tool_name: not a string of 1..63 bytes");
            t.tool = tn->s;
          } else if (ms) {
            if (ms->k != JVal::STR) return fail_line(counts, ln, tk + "message: not a string");
            std::string nm;
            Res r = parse_message(ms->s, format, nm);
            if (r != R_NAME || nm.size() > 63) {  // R35: absent / malformed -> "unknown" + warning
              ++warnings;
              nm = "unknown";
            }
            t.tool = nm;
          } else {
            return fail_line(counts, ln, tk + "tool_name: missing on a non-final turn");
          }
        }
        pr.turns.push_back(std::move(t));
      }
      progs.push_back(std::move(pr));
    }
    std::stable_sort(progs.begin(), progs.end(),
                     [](const LProg& a, const LProg& b) { return a.arr < b.arr; });
    int64_t nt = 0;
    for (auto& pr : progs) {
      nt += (int64_t)pr.turns.size();
      for (auto& t : pr.turns) {
        if (t.tool.empty()) continue;
        if (std::find(names.begin(), names.end(), t.tool) == names.end()) {
          if ((int)names.size() >= CT_MAX_TOOLS) return fail_line(counts, pr.line, "tool_name: more than CT_MAX_TOOLS tools");
          names.push_back(t.tool);
        }
      }
    }
    counts[0] = (int64_t)progs.size();
    counts[1] = nt;
    counts[2] = (int64_t)names.size();
    counts[3] = warnings;
    if (nt > kI32) return fail_msg("ct_load_trace_jsonl: more than 2^31 turns");
    if (!programs || !turns) return CT_OK;
    if (programs_cap < (int64_t)progs.size() || turns_cap < nt)
      return fail_msg("ct_load_trace_jsonl: programs_cap or turns_cap too small (see counts)");
    int64_t o = 0;
    for (size_t i = 0; i < progs.size(); ++i) {
      programs[i].arr_q = progs[i].arr;
      programs[i].turn0 = (int32_t)o;
      programs[i].nturns = (int32_t)progs[i].turns.size();
      for (auto& t : progs[i].turns) {
        ct_turn& r = turns[o++];
        r.new_tokens = t.nw;
        r.decode_tokens = t.dec;
        r.tool = t.tool.empty() ? -1
                                : (int32_t)(std::find(names.begin(), names.end(), t.tool) - names.begin());
        r.dur_us = (int32_t)t.dur;
      }
    }
    if (tool_names) {
      for (size_t i = (size_t)n_known; i < names.size(); ++i) {
        char* e = tool_names + 64 * i;
        memset(e, 0, 64);
        memcpy(e, names[i].data(), names[i].size());
      }
    }
    return CT_OK;
  } catch (...) {
    ct::set_last_error("ct_load_trace_jsonl: host allocation failed");
    return CT_ENOMEM;
  }
}

}  // extern "C"
