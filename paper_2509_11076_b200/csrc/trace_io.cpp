// trace_io.cpp -- Detailed-record files (SURVEY §8(b) plumbing `chm_trace_load`
// save/load with a byte-offset parse error, "DetailedRecord serializable in the same
// JSON-lines format"): one JSON object per line, LF endings.
//
//   line 1  {"chm_trace":1,"t_iter_s":T,"tensors":[[nbytes,dtype],...]}
//   op      {"op":"aten::mm","tok":7,"phase":0,"in":[i,...],"out":[i,...],"free":[i,...],"live":B}
//   swap    {"swap":[from,to,nbytes]}            (Fig. 3 swap log; to = -1: still out)
//
// Tensor ids are indices into the header's table.  An op's "op" name is tokenized through the
// ctx (its "tok" is used only when the name is absent); "live" is optional (-1).  A tensor that
// no op outputs is live at iteration start (static); one that is output twice is an error.
#include <cerrno>
#include <cinttypes>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "internal.h"

using namespace chm;

namespace {

// ------------------------------------------------------------------ minimal JSON reader
struct JVal {
  enum Kind { NUL, BOOL, NUM, STR, ARR, OBJ } kind = NUL;
  bool b = false;
  bool is_int = false;
  int64_t i = 0;
  double d = 0.0;
  std::string s;
  std::vector<JVal> a;
  std::vector<std::pair<std::string, JVal>> o;
  const JVal *get(const char *k) const {
    for (const auto &kv : o)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
};

struct Parser {
  const char *p, *end, *base;
  size_t err = SIZE_MAX;
  const char *msg = "";
  bool fail(const char *m) {
    if (err == SIZE_MAX) { err = size_t(p - base); msg = m; }
    return false;
  }
  void ws() { while (p < end && (*p == ' ' || *p == '\t' || *p == '\r')) p++; }
  bool lit(const char *w) {
    size_t n = std::strlen(w);
    if (size_t(end - p) < n || std::memcmp(p, w, n)) return fail("bad literal");
    p += n;
    return true;
  }
  bool str(std::string &out) {
    if (p >= end || *p != '"') return fail("expected string");
    p++;
    while (p < end && *p != '"') {
      if (*p == '\n') return fail("newline in string");
      if (*p == '\\') {
        if (++p >= end) return fail("truncated escape");
        switch (*p) {
          case '"': out += '"'; break;
          case '\\': out += '\\'; break;
          case '/': out += '/'; break;
          case 'n': out += '\n'; break;
          case 't': out += '\t'; break;
          case 'r': out += '\r'; break;
          case 'b': out += '\b'; break;
          case 'f': out += '\f'; break;
          default: return fail("unsupported escape");
        }
        p++;
      } else {
        out += *p++;
      }
    }
    if (p >= end) return fail("unterminated string");
    p++;
    return true;
  }
  bool num(JVal &v) {
    const char *s = p;
    if (p < end && *p == '-') p++;
    if (p >= end || *p < '0' || *p > '9') { p = s; return fail("expected number"); }
    while (p < end && *p >= '0' && *p <= '9') p++;
    bool frac = false;
    if (p < end && (*p == '.' || *p == 'e' || *p == 'E')) {
      frac = true;
      if (*p == '.') { p++; while (p < end && *p >= '0' && *p <= '9') p++; }
      if (p < end && (*p == 'e' || *p == 'E')) {
        p++;
        if (p < end && (*p == '+' || *p == '-')) p++;
        if (p >= end || *p < '0' || *p > '9') return fail("bad exponent");
        while (p < end && *p >= '0' && *p <= '9') p++;
      }
    }
    std::string t(s, size_t(p - s));
    v.kind = JVal::NUM;
    v.d = std::strtod(t.c_str(), nullptr);
    if (!frac) {
      errno = 0;
      long long x = std::strtoll(t.c_str(), nullptr, 10);
      if (errno == ERANGE) { p = s; return fail("integer out of range"); }
      v.is_int = true;
      v.i = int64_t(x);
    }
    return true;
  }
  bool value(JVal &v, int depth) {
    if (depth > 8) return fail("nesting too deep");
    ws();
    if (p >= end) return fail("unexpected end of line");
    switch (*p) {
      case '{': {
        v.kind = JVal::OBJ;
        p++;
        ws();
        if (p < end && *p == '}') { p++; return true; }
        for (;;) {
          ws();
          std::string k;
          if (!str(k)) return false;
          ws();
          if (p >= end || *p != ':') return fail("expected ':'");
          p++;
          v.o.emplace_back(std::move(k), JVal());
          if (!value(v.o.back().second, depth + 1)) return false;
          ws();
          if (p < end && *p == ',') { p++; continue; }
          if (p < end && *p == '}') { p++; return true; }
          return fail("expected ',' or '}'");
        }
      }
      case '[': {
        v.kind = JVal::ARR;
        p++;
        ws();
        if (p < end && *p == ']') { p++; return true; }
        for (;;) {
          v.a.emplace_back();
          if (!value(v.a.back(), depth + 1)) return false;
          ws();
          if (p < end && *p == ',') { p++; continue; }
          if (p < end && *p == ']') { p++; return true; }
          return fail("expected ',' or ']'");
        }
      }
      case '"': v.kind = JVal::STR; return str(v.s);
      case 't': v.kind = JVal::BOOL; v.b = true; return lit("true");
      case 'f': v.kind = JVal::BOOL; return lit("false");
      case 'n': return lit("null");
      default: return num(v);
    }
  }
  // one object per line; the cursor is left after the line's LF
  bool line(JVal &v) {
    if (!value(v, 0)) return false;
    ws();
    if (p < end && *p != '\n') return fail("trailing characters");
    if (p < end) p++;
    if (v.kind != JVal::OBJ) { return fail("line is not an object"); }
    return true;
  }
};

bool int_array(const JVal *v, std::vector<int64_t> &out) {
  out.clear();
  if (!v) return true;
  if (v->kind != JVal::ARR) return false;
  for (const JVal &x : v->a) {
    if (x.kind != JVal::NUM || !x.is_int) return false;
    out.push_back(x.i);
  }
  return true;
}

}  // namespace

#define PARSE_FAIL(off, ...)                          \
  do {                                                \
    if (err_offset) *err_offset = int64_t(off);       \
    CHM_FAIL(CHM_E_PARSE, __VA_ARGS__);               \
  } while (0)

extern "C" chm_status chm_trace_load(chm_ctx *ctx, const char *text, size_t len, const chm_trace_params *params,
                                     chm_trace **out, int64_t *err_offset) {
  if (err_offset) *err_offset = -1;
  if (!ctx || (!text && len) || !params || !out) CHM_FAIL(CHM_E_INVAL, "chm_trace_load: NULL argument");
  *out = nullptr;
  Parser ps{text, text + len, text};
  IterRecord R;
  R.detailed = true;
  JVal hdr;
  if (!ps.line(hdr)) PARSE_FAIL(ps.err, "chm_trace_load: byte %zu: %s", ps.err, ps.msg);
  const JVal *ver = hdr.get("chm_trace");
  if (!ver || !ver->is_int || ver->i != 1) PARSE_FAIL(0, "chm_trace_load: byte 0: header lacks \"chm_trace\":1");
  const JVal *ti = hdr.get("t_iter_s");
  if (ti && ti->kind == JVal::NUM) R.t_iter = ti->d;
  const JVal *tt = hdr.get("tensors");
  if (!tt || tt->kind != JVal::ARR) PARSE_FAIL(0, "chm_trace_load: byte 0: header lacks a \"tensors\" array");
  for (const JVal &e : tt->a) {
    if (e.kind != JVal::ARR || e.a.size() != 2 || !e.a[0].is_int || !e.a[1].is_int || e.a[0].i <= 0 ||
        e.a[1].i < 0 || e.a[1].i > 255)
      PARSE_FAIL(0, "chm_trace_load: byte 0: tensor %zu must be [nbytes > 0, dtype 0..255]", R.tensors.size());
    TensorRec r;
    r.nbytes = e.a[0].i;
    r.dtype = uint8_t(e.a[1].i);
    R.tensors.push_back(r);
  }
  const int64_t T = int64_t(R.tensors.size());
  std::vector<int64_t> ins, outs, frees, sw;
  while (ps.p < ps.end) {
    const size_t at = size_t(ps.p - ps.base);
    if (*ps.p == '\n') { ps.p++; continue; }  // blank line
    JVal v;
    if (!ps.line(v)) PARSE_FAIL(ps.err, "chm_trace_load: byte %zu: %s", ps.err, ps.msg);
    if (const JVal *s = v.get("swap")) {
      if (!int_array(s, sw) || sw.size() != 3 || sw[0] < 0 || sw[2] <= 0)
        PARSE_FAIL(at, "chm_trace_load: byte %zu: swap must be [from >= 0, to, nbytes > 0]", at);
      R.swaps.push_back({int32_t(sw[0]), sw[1] < 0 ? INT32_MAX : int32_t(sw[1]), sw[2], 0});
      continue;
    }
    const JVal *nm = v.get("op"), *tk = v.get("tok"), *ph = v.get("phase");
    int32_t token = 0;
    if (nm && nm->kind == JVal::STR) {
      chm_status st = chm_tokenize(ctx, nm->s.c_str(), &token);
      if (st != CHM_OK) return st;
    } else if (tk && tk->is_int && tk->i >= 1 && tk->i <= INT32_MAX) {
      token = int32_t(tk->i);
    } else {
      PARSE_FAIL(at, "chm_trace_load: byte %zu: op line needs \"op\" (name) or \"tok\" >= 1", at);
    }
    if (!ph || !ph->is_int || ph->i < 0 || ph->i > 2) PARSE_FAIL(at, "chm_trace_load: byte %zu: phase must be 0, 1 or 2", at);
    if (!R.phase.empty() && uint8_t(ph->i) < R.phase.back())
      PARSE_FAIL(at, "chm_trace_load: byte %zu: phases interleave (FWD* BWD* OPT* required)", at);
    if (!int_array(v.get("in"), ins) || !int_array(v.get("out"), outs) || !int_array(v.get("free"), frees))
      PARSE_FAIL(at, "chm_trace_load: byte %zu: in / out / free must be integer arrays", at);
    const int32_t i = int32_t(R.tokens.size());
    R.tokens.push_back(token);
    R.phase.push_back(uint8_t(ph->i));
    const JVal *lv = v.get("live");
    R.live_bytes.push_back(lv && lv->is_int ? lv->i : -1);
    const size_t use_begin = R.use_idx.size();
    auto add_use = [&](int32_t t, bool is_in) {
      for (size_t u = use_begin; u < R.use_idx.size(); u++)
        if (R.use_idx[u] == t) return;
      R.use_idx.push_back(t);
      R.use_is_in.push_back(is_in ? 1 : 0);
    };
    for (int64_t t : ins) {
      if (t < 0 || t >= T) PARSE_FAIL(at, "chm_trace_load: byte %zu: input tensor %" PRId64 " not in the table", at, t);
      if (R.tensors[t].freed >= 0) PARSE_FAIL(at, "chm_trace_load: byte %zu: tensor %" PRId64 " used after its free", at, t);
      add_use(int32_t(t), true);
    }
    for (int64_t t : outs) {
      if (t < 0 || t >= T) PARSE_FAIL(at, "chm_trace_load: byte %zu: output tensor %" PRId64 " not in the table", at, t);
      if (R.tensors[t].producer >= 0) PARSE_FAIL(at, "chm_trace_load: byte %zu: tensor %" PRId64 " output twice", at, t);
      R.tensors[t].producer = i;
      R.out_idx.push_back(int32_t(t));
      R.alloc_bytes += R.tensors[t].nbytes;
      add_use(int32_t(t), false);
    }
    for (int64_t t : frees) {
      if (t < 0 || t >= T || R.tensors[t].freed >= 0)
        PARSE_FAIL(at, "chm_trace_load: byte %zu: bad or repeated free of tensor %" PRId64, at, t);
      R.tensors[t].freed = i;
      R.free_idx.push_back(int32_t(t));
    }
    R.use_ptr.push_back(int32_t(R.use_idx.size()));
    R.out_ptr.push_back(int32_t(R.out_idx.size()));
    R.free_ptr.push_back(int32_t(R.free_idx.size()));
  }
  if (R.tokens.empty()) CHM_FAIL(CHM_E_STATE, "chm_trace_load: the file has no ops");
  // a tensor used before its producer: only static tensors may be read before any output
  for (int32_t i = 0; i < int32_t(R.tokens.size()); i++)
    for (int32_t u = R.use_ptr[i]; u < R.use_ptr[i + 1]; u++) {
      const TensorRec &r = R.tensors[R.use_idx[u]];
      if (R.use_is_in[u] && r.producer > i)
        CHM_FAIL(CHM_E_PARSE, "chm_trace_load: op %d reads tensor %d before op %d outputs it", i, R.use_idx[u], r.producer);
    }
  return build_trace(ctx, R, params, out);
}

// ------------------------------------------------------------------ writer
namespace {
struct Out {
  char *buf;
  size_t cap, n = 0;
  void put(const char *s, size_t k) {
    if (n + k <= cap && buf) std::memcpy(buf + n, s, k);
    n += k;
  }
  void str(const char *s) { put(s, std::strlen(s)); }
  void i64(int64_t v) {
    char t[32];
    int k = std::snprintf(t, sizeof t, "%" PRId64, v);
    put(t, size_t(k));
  }
  void dbl(double v) {
    char t[40];
    int k = std::snprintf(t, sizeof t, "%.17g", v);
    put(t, size_t(k));
  }
  void jstr(const std::string &s) {
    put("\"", 1);
    for (char c : s) {
      if (c == '"' || c == '\\') { put("\\", 1); put(&c, 1); }
      else if (c == '\n') put("\\n", 2);
      else put(&c, 1);
    }
    put("\"", 1);
  }
};
}  // namespace

extern "C" chm_status chm_record_save(chm_ctx *ctx, char *buf, size_t cap, size_t *len) {
  if (!ctx || !len || (cap && !buf)) CHM_FAIL(CHM_E_INVAL, "chm_record_save: NULL argument");
  const IterRecord &R = ctx->last_detailed;
  if (R.tokens.empty()) CHM_FAIL(CHM_E_STATE, "chm_record_save: no Detailed-mode iteration recorded");
  std::vector<const std::string *> name;
  for (const auto &kv : ctx->tokens) {
    if (size_t(kv.second) >= name.size()) name.resize(size_t(kv.second) + 1, nullptr);
    name[size_t(kv.second)] = &kv.first;
  }
  Out o{buf, cap};
  o.str("{\"chm_trace\":1,\"t_iter_s\":");
  o.dbl(R.t_iter);
  o.str(",\"tensors\":[");
  for (size_t t = 0; t < R.tensors.size(); t++) {
    o.str(t ? ",[" : "[");
    o.i64(R.tensors[t].nbytes);
    o.str(",");
    o.i64(R.tensors[t].dtype);
    o.str("]");
  }
  o.str("]}\n");
  for (size_t i = 0; i < R.tokens.size(); i++) {
    o.str("{");
    const int32_t tok = R.tokens[i];
    if (tok >= 0 && size_t(tok) < name.size() && name[size_t(tok)]) {
      o.str("\"op\":");
      o.jstr(*name[size_t(tok)]);
      o.str(",");
    }
    o.str("\"tok\":");
    o.i64(tok);
    o.str(",\"phase\":");
    o.i64(R.phase[i]);
    const char *keys[3] = {",\"in\":[", ",\"out\":[", ",\"free\":["};
    for (int which = 0; which < 3; which++) {
      o.str(keys[which]);
      bool first = true;
      auto emit = [&](int32_t t) { if (!first) o.str(","); o.i64(t); first = false; };
      if (which == 0) {
        for (int32_t u = R.use_ptr[i]; u < R.use_ptr[i + 1]; u++)
          if (R.use_is_in[u]) emit(R.use_idx[u]);
      } else if (which == 1) {
        for (int32_t u = R.out_ptr[i]; u < R.out_ptr[i + 1]; u++) emit(R.out_idx[u]);
      } else {
        for (int32_t u = R.free_ptr[i]; u < R.free_ptr[i + 1]; u++) emit(R.free_idx[u]);
      }
      o.str("]");
    }
    if (i < R.live_bytes.size() && R.live_bytes[i] >= 0) {
      o.str(",\"live\":");
      o.i64(R.live_bytes[i]);
    }
    o.str("}\n");
  }
  for (const auto &sp : R.swaps) {
    o.str("{\"swap\":[");
    o.i64(sp.from);
    o.str(",");
    o.i64(sp.to == INT32_MAX ? -1 : sp.to);
    o.str(",");
    o.i64(sp.nbytes);
    o.str("]}\n");
  }
  *len = o.n;
  if (o.n > cap) CHM_FAIL(CHM_E_NOMEM, "chm_record_save: %zu bytes needed, buffer has %zu", o.n, cap);
  return CHM_OK;
}
