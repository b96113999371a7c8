// trace_v1.cpp -- native reader of the relsim-trace-v1 file format, the
// on-disk trace both sides share (pkg/docs/trace-schema.md; written by
// workload.save_trace, pkg/src/relsim/workload.py:324-347, read by
// load_trace, :349-384).  Only the counts are parsed -- what the device SoA
// needs (arrival, rel_id, output_limit, prefix_len, per-request tok / out);
// token IDs are never materialised (the device models the prefix cache from
// counts).  A hand-written scanner for this one schema.
#include <errno.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <string>
#include <vector>

#include "../../include/relserve.h"

struct rs_trace_file {
  double rate = 0.0;
  long long seed = 0;
  std::vector<long long> rel_id;
  std::vector<double> arrival;
  std::vector<int> output_limit, prefix_len;
  std::vector<long long> row_off{0};
  std::vector<int> tok, out;
};

namespace {

thread_local std::string g_trace_err;

struct Scanner {
  const char* p;
  const char* end;
  long long line;
  bool ok = true;
  std::string err;

  void fail(const std::string& m) {
    if (ok) err = "line " + std::to_string(line) + ": " + m;
    ok = false;
  }
  void ws() {
    while (p < end && (*p == ' ' || *p == '\t' || *p == '\r')) ++p;
  }
  bool eat(char ch) {
    ws();
    if (p < end && *p == ch) {
      ++p;
      return true;
    }
    return false;
  }
  void expect(char ch) {
    if (!eat(ch)) fail(std::string("expected '") + ch + "'");
  }
  struct Key {  // a view of the key's characters (no allocation per key)
    const char* s;
    size_t n;
    bool operator==(const char* lit) const { return strlen(lit) == n && memcmp(s, lit, n) == 0; }
  };
  Key key() {
    ws();
    if (p >= end || *p != '"') {
      fail("expected a key");
      return {p, 0};
    }
    const char* s = ++p;
    while (p < end && *p != '"') p += (*p == '\\') ? 2 : 1;
    const Key k{s, (size_t)((p < end ? p : end) - s)};
    if (p < end) ++p;
    expect(':');
    return k;
  }
  long long integer() {  // a JSON integer (the counts): plain digit loop, strtoll is locale-bound and slow
    ws();
    const bool neg = p < end && *p == '-';
    if (neg) ++p;
    const char* d0 = p;
    unsigned long long v = 0;
    while (p < end && *p >= '0' && *p <= '9' && p - d0 < 19) v = v * 10 + (unsigned long long)(*p++ - '0');
    if (p == d0 || (p < end && ((*p >= '0' && *p <= '9') || *p == '.' || *p == 'e' || *p == 'E')))
      fail("expected an integer");
    return neg ? -(long long)v : (long long)v;
  }
  double number() {  // strtod rounds correctly: the same double as Python's float(repr(x))
    ws();
    char* q = nullptr;
    const double v = strtod(p, &q);
    if (q == p) fail("expected a number");
    p = q;
    return v;
  }
  void skip_value() {  // any JSON value (keys the schema does not name)
    ws();
    if (p >= end) return fail("truncated value");
    const char ch = *p;
    if (ch == '"') {
      ++p;
      while (p < end && *p != '"') p += (*p == '\\') ? 2 : 1;
      ++p;
    } else if (ch == '{' || ch == '[') {
      const char close = ch == '{' ? '}' : ']';
      ++p;
      if (eat(close)) return;
      do {
        if (ch == '{') key();
        skip_value();
      } while (ok && eat(','));
      expect(close);
    } else {
      while (p < end && *p != ',' && *p != '}' && *p != ']' && *p != '\n') ++p;
    }
  }
};

bool parse_header(Scanner& s, rs_trace_file& f) {
  s.expect('{');
  bool schema_ok = false;
  do {
    const Scanner::Key k = s.key();
    if (k == "schema") {
      s.ws();
      schema_ok = s.end - s.p >= 17 && strncmp(s.p, "\"relsim-trace-v1\"", 17) == 0;
      s.skip_value();
    } else if (k == "rate") {
      f.rate = s.number();
    } else if (k == "seed") {
      f.seed = s.integer();
    } else {
      s.skip_value();
    }
  } while (s.ok && s.eat(','));
  s.expect('}');
  if (!schema_ok) s.fail("not a relsim-trace-v1 file");
  return s.ok;
}

bool parse_relquery(Scanner& s, rs_trace_file& f) {
  long long rel_id = 0, size = -1;
  double arrival = 0.0;
  int limit = 0, plen = 0;
  bool have_reqs = false;
  const size_t first = f.tok.size();
  std::vector<int> req_plen;
  s.expect('{');
  do {
    const Scanner::Key k = s.key();
    if (k == "rel_id") rel_id = s.integer();
    else if (k == "arrival_s") arrival = s.number();
    else if (k == "size") size = s.integer();
    else if (k == "output_limit") limit = (int)s.integer();
    else if (k == "prefix_len") plen = (int)s.integer();
    else if (k == "requests") {
      have_reqs = true;
      s.expect('[');
      if (!s.eat(']')) {
        do {
          int tok = 0, out = 0, rp = 0;
          bool has_tok = false, has_out = false, has_plen = false;
          s.expect('{');
          do {
            const Scanner::Key rk = s.key();
            if (rk == "tok") tok = (int)s.integer(), has_tok = true;
            else if (rk == "out") out = (int)s.integer(), has_out = true;
            else if (rk == "prefix_len") rp = (int)s.integer(), has_plen = true;
            else s.skip_value();
          } while (s.ok && s.eat(','));
          s.expect('}');
          if (!(has_tok && has_out && has_plen)) s.fail("request without tok / out / prefix_len");
          f.tok.push_back(tok);
          f.out.push_back(out);
          req_plen.push_back(rp);
        } while (s.ok && s.eat(','));
        s.expect(']');
      }
    } else {
      s.skip_value();
    }
  } while (s.ok && s.eat(','));
  s.expect('}');
  if (!s.ok) return false;
  const long long n = (long long)(f.tok.size() - first);
  if (!have_reqs) s.fail("relQuery without requests");
  if (size >= 0 && size != n) s.fail("relQuery " + std::to_string(rel_id) + ": size != len(requests)");
  for (int rp : req_plen)
    if (rp != plen) s.fail("relQuery " + std::to_string(rel_id) + ": per-request prefix_len differs");
  if (!s.ok) return false;
  f.rel_id.push_back(rel_id);
  f.arrival.push_back(arrival);
  f.output_limit.push_back(limit);
  f.prefix_len.push_back(plen);
  f.row_off.push_back((long long)f.tok.size());
  return true;
}

}  // namespace

extern "C" {

const char* rs_trace_v1_error(void) { return g_trace_err.c_str(); }

int rs_trace_v1_load(const char* path, rs_trace_file** out) {
  *out = nullptr;
  FILE* fp = fopen(path, "rb");
  if (!fp) {
    g_trace_err = std::string("cannot open ") + path;
    return RS_EINVAL;
  }
  std::vector<char> buf;
  fseek(fp, 0, SEEK_END);
  const long sz = ftell(fp);
  fseek(fp, 0, SEEK_SET);
  buf.resize(sz > 0 ? (size_t)sz : 0);
  const size_t got = sz > 0 ? fread(buf.data(), 1, (size_t)sz, fp) : 0;
  fclose(fp);
  buf.push_back('\0');  // strtod / strtoll stop at it past the last line
  if ((long)got != sz) {
    g_trace_err = std::string("short read of ") + path;
    return RS_EINVAL;
  }
  rs_trace_file* f = new rs_trace_file();
  const char* p = buf.data();
  const char* end = p + buf.size() - 1;
  long long line = 1;
  bool header = true;
  while (p < end) {
    const char* nl = (const char*)memchr(p, '\n', (size_t)(end - p));
    const char* le = nl ? nl : end;
    Scanner s{p, le, line};
    s.ws();
    if (s.p < le) {
      const bool ok = header ? parse_header(s, *f) : parse_relquery(s, *f);
      if (ok) {
        s.ws();
        if (s.p != le) s.fail("trailing characters");
      }
      if (!s.ok) {
        g_trace_err = s.err;
        delete f;
        return RS_EINVAL;
      }
      header = false;
    }
    p = nl ? nl + 1 : end;
    ++line;
  }
  if (header) {
    g_trace_err = "empty trace file";
    delete f;
    return RS_EINVAL;
  }
  *out = f;
  return RS_OK;
}

int rs_trace_v1_info(const rs_trace_file* f, int64_t* num_relqueries, int64_t* num_requests, double* rate,
                     int64_t* seed) {
  if (!f) return RS_EINVAL;
  *num_relqueries = (int64_t)f->rel_id.size();
  *num_requests = (int64_t)f->tok.size();
  *rate = f->rate;
  *seed = f->seed;
  return RS_OK;
}

int rs_trace_v1_columns(const rs_trace_file* f, int64_t* rel_id, double* arrival, int32_t* output_limit,
                        int32_t* prefix_len, int64_t* row_off, int32_t* tok, int32_t* out) {
  if (!f) return RS_EINVAL;
  const size_t R = f->rel_id.size(), N = f->tok.size();
  memcpy(rel_id, f->rel_id.data(), R * sizeof(int64_t));
  memcpy(arrival, f->arrival.data(), R * sizeof(double));
  memcpy(output_limit, f->output_limit.data(), R * sizeof(int32_t));
  memcpy(prefix_len, f->prefix_len.data(), R * sizeof(int32_t));
  memcpy(row_off, f->row_off.data(), (R + 1) * sizeof(int64_t));
  memcpy(tok, f->tok.data(), N * sizeof(int32_t));
  memcpy(out, f->out.data(), N * sizeof(int32_t));
  return RS_OK;
}

void rs_trace_v1_free(rs_trace_file* f) { delete f; }

}  // extern "C"
