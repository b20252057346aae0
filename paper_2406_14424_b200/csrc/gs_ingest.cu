// gs_ingest.cu — validation ingest (host side of the C ABI): the reference's
// validation JSONL (formats.save_validation / load_validation,
// /root/reference/pkg/src/gearserve/formats.py:75-106: one record per line,
// {"sample_id": int, "models": {"<id>": {"scores": [...], "correct": bool}}})
// parsed into columnar arrays with all host threads, so a 1M-record file
// feeds the device sweep in a fraction of a second instead of a Python loop.
//
// Semantics follow the reference reader: blank lines are skipped; unknown
// keys are ignored; sample_id goes through int() (integer tokens exactly,
// float tokens truncated, NaN / inf rejected, decimal strings and bools as
// int() takes them); correct through bool(); every score through float()
// (correctly rounded strtod); number tokens follow json.loads: the JSON
// grammar plus NaN / Infinity / -Infinity, nothing else; a line that is not such an
// object fails with its 1-based line number.  Cross-record checks (unique
// non-negative ids, one model set, non-empty scores) are reported per line
// too.  Model order is the first record's key order.
#include <cctype>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <string>
#include <thread>
#include <vector>

#include "../../include/gearserve_b200.h"

namespace {

// one parsed record (scratch, M <= GS_JSONL_MAX_MODELS)
struct Line {
  int64_t sample_id = 0;
  int32_t len[GS_JSONL_MAX_MODELS];
  uint8_t correct[GS_JSONL_MAX_MODELS];
  size_t off[GS_JSONL_MAX_MODELS];  // offsets into the chunk's score buffer
};

// the records of one thread's line range, flat
struct Chunk {
  std::vector<int64_t> sample_id, lineno;
  std::vector<int32_t> len;      // [lines][M]
  std::vector<uint8_t> correct;  // [lines][M]
  std::vector<size_t> off;       // [lines][M]
  std::vector<double> scores;
  int64_t err_line = 0;
  std::string err;
};

struct Parser {
  const char* p;
  const char* end;
  std::string err;

  void ws() {
    while (p < end && (*p == ' ' || *p == '\t' || *p == '\r' || *p == '\n')) ++p;
  }
  bool eat(char c) {
    ws();
    if (p < end && *p == c) {
      ++p;
      return true;
    }
    return false;
  }
  bool fail(const char* m) {
    if (err.empty()) err = m;
    return false;
  }
  bool string(std::string* out) {
    ws();
    if (p >= end || *p != '"') return fail("expected a string");
    ++p;
    if (out) out->clear();
    while (p < end && *p != '"') {
      char c = *p++;
      if (c == '\\') {
        if (p >= end) return fail("bad escape");
        c = *p++;
        if (c == 'u') {  // keep the escape verbatim (ids are compared as written)
          if (end - p < 4) return fail("bad escape");
          if (out) out->append("\\u").append(p, 4);
          p += 4;
          continue;
        }
        switch (c) {
          case 'n': c = '\n'; break;
          case 't': c = '\t'; break;
          case 'r': c = '\r'; break;
          case 'b': c = '\b'; break;
          case 'f': c = '\f'; break;
          default: break;  // \" \\ \/
        }
      }
      if (out) out->push_back(c);
    }
    if (p >= end) return fail("unterminated string");
    ++p;
    return true;
  }
  // A number token as json.loads reads it: the JSON grammar
  // -?(0|[1-9][0-9]*)(.[0-9]+)?([eE][+-]?[0-9]+)? or the literals NaN,
  // Infinity, -Infinity (json.loads accepts them); is_int: no fraction or
  // exponent (json.loads returns an int).  Nothing else (hex, "inf", "nan",
  // a leading '+') is accepted.
  bool number_token(std::string* tok, bool* is_int) {
    ws();
    const char* q = p;
    auto lit = [&](const char* w) {
      const size_t n = std::strlen(w);
      return (size_t)(end - q) >= n && !std::strncmp(q, w, n) ? n : (size_t)0;
    };
    size_t n = lit("NaN");
    if (!n) n = lit("Infinity");
    if (!n) n = lit("-Infinity");
    *is_int = false;
    if (!n) {
      const char* r = q;
      if (r < end && *r == '-') ++r;
      if (r >= end || !std::isdigit((unsigned char)*r)) return fail("expected a number");
      if (*r == '0') ++r;
      else
        while (r < end && std::isdigit((unsigned char)*r)) ++r;
      *is_int = true;
      if (r < end && *r == '.') {
        ++r;
        if (r >= end || !std::isdigit((unsigned char)*r)) return fail("bad number");
        while (r < end && std::isdigit((unsigned char)*r)) ++r;
        *is_int = false;
      }
      if (r < end && (*r == 'e' || *r == 'E')) {
        ++r;
        if (r < end && (*r == '+' || *r == '-')) ++r;
        if (r >= end || !std::isdigit((unsigned char)*r)) return fail("bad number");
        while (r < end && std::isdigit((unsigned char)*r)) ++r;
        *is_int = false;
      }
      n = (size_t)(r - q);
    }
    tok->assign(q, n);
    p += n;
    return true;
  }
  bool number(double* v) {
    std::string tok;
    bool is_int;
    if (!number_token(&tok, &is_int)) return false;
    if (tok == "NaN") *v = NAN;
    else if (tok == "Infinity") *v = INFINITY;
    else if (tok == "-Infinity") *v = -INFINITY;
    else *v = std::strtod(tok.c_str(), nullptr);  // the C locale's '.': correctly rounded
    return true;
  }
  // int(value) of a JSON value, as the reference's int(rec["sample_id"]):
  // an integer token exactly, a float token truncated (NaN / inf raise), a
  // string through int(str) (optional sign and surrounding whitespace), a
  // bool as 0 / 1
  bool integer(int64_t* v) {
    ws();
    if (end - p >= 4 && !std::strncmp(p, "true", 4)) { p += 4; *v = 1; return true; }
    if (end - p >= 5 && !std::strncmp(p, "false", 5)) { p += 5; *v = 0; return true; }
    std::string tok;
    bool is_int = false;
    if (p < end && *p == '"') {
      if (!string(&tok)) return false;
      size_t a = 0, b = tok.size();
      while (a < b && std::isspace((unsigned char)tok[a])) ++a;
      while (b > a && std::isspace((unsigned char)tok[b - 1])) --b;
      tok = tok.substr(a, b - a);
      size_t i = (!tok.empty() && (tok[0] == '-' || tok[0] == '+')) ? 1 : 0;
      if (i >= tok.size()) return fail("invalid literal for int()");
      for (; i < tok.size(); ++i)
        if (!std::isdigit((unsigned char)tok[i])) return fail("invalid literal for int()");
      is_int = true;
    } else if (!number_token(&tok, &is_int)) {
      return false;
    }
    errno = 0;
    if (is_int) {
      char* e = nullptr;
      const long long x = std::strtoll(tok.c_str(), &e, 10);
      if (errno == ERANGE) return fail("integer out of range");
      *v = (int64_t)x;
      return true;
    }
    double d;
    if (!number_token_value(tok, &d)) return false;
    if (!std::isfinite(d)) return fail("cannot convert float NaN or infinity to integer");
    if (!(d > -9.3e18 && d < 9.3e18)) return fail("integer out of range");
    *v = (int64_t)d;  // int(float): truncation toward zero
    return true;
  }
  bool number_token_value(const std::string& tok, double* d) {
    if (tok == "NaN") *d = NAN;
    else if (tok == "Infinity") *d = INFINITY;
    else if (tok == "-Infinity") *d = -INFINITY;
    else *d = std::strtod(tok.c_str(), nullptr);
    return true;
  }
  // any JSON value (for ignored keys)
  bool skip() {
    ws();
    if (p >= end) return fail("unexpected end of line");
    if (*p == '"') return string(nullptr);
    if (*p == '{' || *p == '[') {
      const char open = *p, close = open == '{' ? '}' : ']';
      ++p;
      if (eat(close)) return true;
      do {
        if (open == '{') {
          if (!string(nullptr) || !eat(':')) return fail("bad object");
        }
        if (!skip()) return false;
      } while (eat(','));
      return eat(close) ? true : fail("bad container");
    }
    bool b;
    return truth(&b);
  }
  // bool(value): true/false, numbers (!= 0), null -> false
  bool truth(bool* out) {
    ws();
    if (end - p >= 4 && !std::strncmp(p, "true", 4)) { p += 4; *out = true; return true; }
    if (end - p >= 5 && !std::strncmp(p, "false", 5)) { p += 5; *out = false; return true; }
    if (end - p >= 4 && !std::strncmp(p, "null", 4)) { p += 4; *out = false; return true; }
    double d;
    if (!number(&d)) return false;
    *out = d != 0.0;
    return true;
  }
};

int model_index(const std::vector<std::string>& ids, const std::string& id) {
  for (size_t i = 0; i < ids.size(); ++i)
    if (ids[i] == id) return (int)i;
  return -1;
}

// Parse one record line.  ids empty: discover the model ids (first record).
bool parse_line(Parser& ps, std::vector<std::string>& ids, bool discover, Line* ln,
                std::vector<double>* scores) {
  if (!ps.eat('{')) return ps.fail("expected an object");
  bool have_id = false, have_models = false;
  const size_t M = ids.size();
  if (!ps.eat('}')) {
    do {
      std::string key;
      if (!ps.string(&key) || !ps.eat(':')) return ps.fail("bad key");
      if (key == "sample_id") {
        if (!ps.integer(&ln->sample_id)) return false;  // int(value)
        have_id = true;
      } else if (key == "models") {
        if (!ps.eat('{')) return ps.fail("models must be an object");
        have_models = true;
        uint8_t seen[GS_JSONL_MAX_MODELS] = {};
        size_t count = 0;
        if (!ps.eat('}')) {
          do {
            std::string mid;
            if (!ps.string(&mid) || !ps.eat(':')) return ps.fail("bad model key");
            int m;
            if (discover) {
              if (model_index(ids, mid) >= 0) return ps.fail("duplicate model id");
              if ((int)ids.size() >= GS_JSONL_MAX_MODELS) return ps.fail("too many models");
              ids.push_back(mid);
              m = (int)ids.size() - 1;
              ln->len[m] = 0;
              ln->correct[m] = 0;
              ln->off[m] = 0;
            } else {
              m = model_index(ids, mid);
              if (m < 0 || seen[m]) return ps.fail("model set differs from the first record");
              seen[m] = 1;
            }
            ++count;
            if (!ps.eat('{')) return ps.fail("model output must be an object");
            bool have_scores = false, have_corr = false;
            if (!ps.eat('}')) {
              do {
                std::string k2;
                if (!ps.string(&k2) || !ps.eat(':')) return ps.fail("bad key");
                if (k2 == "scores") {
                  if (!ps.eat('[')) return ps.fail("scores must be a list");
                  ln->off[m] = scores->size();
                  int32_t n = 0;
                  if (!ps.eat(']')) {
                    do {
                      double v;
                      ps.ws();
                      if (ps.p < ps.end && *ps.p == '"') {  // float("1.5"), as the reference allows
                        std::string str;
                        if (!ps.string(&str)) return false;
                        char* e = nullptr;
                        v = std::strtod(str.c_str(), &e);
                        while (e && (*e == ' ' || *e == '\t' || *e == '\n')) ++e;
                        if (str.empty() || !e || *e) return ps.fail("could not convert string to float");
                      } else if (!ps.number(&v)) {
                        return false;
                      }
                      scores->push_back(v);
                      ++n;
                    } while (ps.eat(','));
                    if (!ps.eat(']')) return ps.fail("bad scores list");
                  }
                  if (n == 0) return ps.fail("scores must be non-empty");
                  ln->len[m] = n;
                  have_scores = true;
                } else if (k2 == "correct") {
                  bool b;
                  if (!ps.truth(&b)) return false;
                  ln->correct[m] = b ? 1 : 0;
                  have_corr = true;
                } else if (!ps.skip()) {
                  return false;
                }
              } while (ps.eat(','));
              if (!ps.eat('}')) return ps.fail("bad model output");
            }
            if (!have_scores) return ps.fail("'scores'");
            if (!have_corr) return ps.fail("'correct'");
          } while (ps.eat(','));
          if (!ps.eat('}')) return ps.fail("bad models object");
        }
        if (!discover && count != M) return ps.fail("model set differs from the first record");
        if (discover && count == 0) return ps.fail("validation records cover no models");
      } else if (!ps.skip()) {
        return false;
      }
    } while (ps.eat(','));
    if (!ps.eat('}')) return ps.fail("bad record");
  }
  ps.ws();
  if (ps.p != ps.end) return ps.fail("trailing characters");
  if (!have_id) return ps.fail("'sample_id'");
  if (!have_models) return ps.fail("'models'");
  if (ln->sample_id < 0) return ps.fail("sample_id must be a non-negative integer");
  return true;
}

struct Handle {
  std::vector<std::string> ids;
  std::vector<Chunk> chunks;
  int64_t n = 0;
  std::vector<int32_t> width;
};

bool blank(const char* a, const char* b) {
  for (; a < b; ++a)
    if (!(*a == ' ' || *a == '\t' || *a == '\r')) return false;
  return true;
}

}  // namespace

extern "C" int gs_jsonl_open(const char* path, int32_t n_threads, void** handle,
                             gs_jsonl_info* info) {
  if (!path || !handle || !info) return GS_EINVAL;
  *handle = nullptr;
  std::memset(info, 0, sizeof(*info));
  FILE* f = std::fopen(path, "rb");
  if (!f) {
    std::snprintf(info->error, sizeof(info->error), "cannot open file");
    return GS_EINVAL;
  }
  std::fseek(f, 0, SEEK_END);
  const long size = std::ftell(f);
  std::fseek(f, 0, SEEK_SET);
  std::string buf((size_t)std::max(size, 0L), '\0');
  const size_t got = size > 0 ? std::fread(&buf[0], 1, (size_t)size, f) : 0;
  std::fclose(f);
  if ((long)got != size) {
    std::snprintf(info->error, sizeof(info->error), "read failed");
    return GS_EINVAL;
  }
  // line starts
  std::vector<size_t> starts;
  starts.reserve(buf.size() / 64 + 1);
  size_t pos = 0;
  while (pos < buf.size()) {
    starts.push_back(pos);
    const void* nl = std::memchr(buf.data() + pos, '\n', buf.size() - pos);
    pos = nl ? (size_t)((const char*)nl - buf.data()) + 1 : buf.size();
  }
  const int64_t n_lines = (int64_t)starts.size();
  auto line_end = [&](int64_t i) {
    size_t e = i + 1 < n_lines ? starts[i + 1] : buf.size();
    while (e > starts[i] && (buf[e - 1] == '\n')) --e;
    return e;
  };
  auto* h = new Handle();
  // the first non-blank line fixes the model ids
  int64_t first = 0;
  while (first < n_lines && blank(buf.data() + starts[first], buf.data() + line_end(first))) ++first;
  if (first == n_lines) {
    std::snprintf(info->error, sizeof(info->error), "validation set is empty");
    delete h;
    return GS_EINVAL;
  }
  {
    Parser ps{buf.data() + starts[first], buf.data() + line_end(first), {}};
    Line ln;
    std::vector<double> sc;
    if (!parse_line(ps, h->ids, true, &ln, &sc)) {
      info->err_line = first + 1;
      std::snprintf(info->error, sizeof(info->error), "%s", ps.err.c_str());
      delete h;
      return GS_EINVAL;
    }
  }
  if ((int)h->ids.size() > GS_JSONL_MAX_MODELS) {
    std::snprintf(info->error, sizeof(info->error), "more than %d models", GS_JSONL_MAX_MODELS);
    delete h;
    return GS_EUNSUPPORTED;
  }
  const int T = std::max(1, std::min<int>(n_threads > 0 ? n_threads : 1, 256));
  h->chunks.resize(T);
  std::vector<std::thread> pool;
  for (int t = 0; t < T; ++t) {
    pool.emplace_back([&, t] {
      Chunk& ck = h->chunks[t];
      const int64_t lo = n_lines * t / T, hi = n_lines * (t + 1) / T;
      std::vector<std::string> ids = h->ids;
      const size_t M = ids.size();
      for (int64_t i = lo; i < hi; ++i) {
        const char* a = buf.data() + starts[i];
        const char* b = buf.data() + line_end(i);
        if (blank(a, b)) continue;
        Parser ps{a, b, {}};
        Line ln;
        if (!parse_line(ps, ids, false, &ln, &ck.scores)) {
          ck.err_line = i + 1;
          ck.err = ps.err;
          return;
        }
        ck.sample_id.push_back(ln.sample_id);
        ck.lineno.push_back(i + 1);
        ck.len.insert(ck.len.end(), ln.len, ln.len + M);
        ck.correct.insert(ck.correct.end(), ln.correct, ln.correct + M);
        ck.off.insert(ck.off.end(), ln.off, ln.off + M);
      }
    });
  }
  for (auto& th : pool) th.join();
  const size_t M = h->ids.size();
  h->width.assign(M, 0);
  for (auto& ck : h->chunks) {
    if (ck.err_line) {  // the first failing line in file order
      info->err_line = ck.err_line;
      std::snprintf(info->error, sizeof(info->error), "%s", ck.err.c_str());
      delete h;
      return GS_EINVAL;
    }
    h->n += (int64_t)ck.sample_id.size();
    for (size_t i = 0; i < ck.len.size(); ++i)
      h->width[i % M] = std::max(h->width[i % M], ck.len[i]);
  }
  info->n_records = h->n;
  info->n_models = (int32_t)M;
  for (size_t m = 0; m < M; ++m) {
    info->width[m] = h->width[m];
    std::snprintf(info->model_ids[m], sizeof(info->model_ids[m]), "%s", h->ids[m].c_str());
    if (h->ids[m].size() >= sizeof(info->model_ids[m])) {
      std::snprintf(info->error, sizeof(info->error), "model id longer than %d bytes",
                    (int)sizeof(info->model_ids[m]) - 1);
      delete h;
      return GS_EUNSUPPORTED;
    }
  }
  *handle = h;
  return GS_OK;
}

extern "C" int gs_jsonl_read(void* handle, int64_t* sample_id, int64_t* line_no,
                             double* const* scores, int32_t* row_len, uint8_t* correct) {
  auto* h = static_cast<Handle*>(handle);
  if (!h || !sample_id || !scores || !row_len || !correct) return GS_EINVAL;
  const size_t M = h->ids.size();
  int64_t r = 0;
  for (auto& ck : h->chunks) {
    for (size_t i = 0; i < ck.sample_id.size(); ++i, ++r) {
      sample_id[r] = ck.sample_id[i];
      if (line_no) line_no[r] = ck.lineno[i];
      for (size_t m = 0; m < M; ++m) {
        const int32_t w = h->width[m], len = ck.len[i * M + m];
        double* dst = scores[m] + r * w;
        std::memcpy(dst, ck.scores.data() + ck.off[i * M + m], sizeof(double) * len);
        for (int32_t j = len; j < w; ++j) dst[j] = 0.0;
        row_len[r * M + m] = len;
        correct[r * M + m] = ck.correct[i * M + m];
      }
    }
  }
  return GS_OK;
}

extern "C" void gs_jsonl_close(void* handle) { delete static_cast<Handle*>(handle); }
