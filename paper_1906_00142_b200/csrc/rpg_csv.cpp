// rpg_csv.cpp — the sample CSV of the reference's data kit (data::
// parse_samples / format_samples, datakit.hpp:272-415) at scale: columnar
// output (the layout the fit consumes), multi-threaded parsing and
// formatting, the same schema, checks, error precedence and CsvError
// messages as the sequential reference.
//
// Parse: the header (and the comments / provenance line before it) is read
// sequentially; the body is cut into chunks at line boundaries, one per
// thread; each thread parses its lines into local columns and stops at its
// first error.  The reported error is the one the sequential reader meets
// first: the lowest failing line, where a duplicate (data tuple, config)
// key counts as failing at its second occurrence (the set insert of
// datakit.hpp:404-409).  Duplicates are found by hashing every row,
// bucketing the hashes by thread and sorting each bucket — no sequential
// pass over the rows.
// Format: std::to_chars shortest round-trip for the reals (datakit.hpp:
// 225-230), rows formatted in parallel chunks and concatenated in order.
#include <algorithm>
#include <cctype>
#include <cerrno>
#include <charconv>
#include <cmath>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "rpg.h"

struct rpg_samples {
  int64_t n = 0;
  int32_t d = 0;
  std::vector<std::string> names;
  std::vector<int64_t> data, configs;
  std::vector<double> values;
  int32_t prov_kind = 0;  // 0 measured, 1 synthetic
  uint64_t seed = 0;
  double noise_rel = 0.0;
};

namespace {

int cerr_(char* err, size_t errlen, const char* fmt, ...) {
  if (err && errlen) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(err, errlen, fmt, ap);
    va_end(ap);
  }
  return RPG_E_CSV;
}

// split_csv (datakit.hpp:232-243): fields at ',', dropping '\r', ' ', '\t'.
void split(const char* b, const char* e, std::vector<std::string>* out) {
  out->clear();
  out->emplace_back();
  for (const char* p = b; p < e; ++p) {
    const char c = *p;
    if (c == ',') out->emplace_back();
    else if (c != '\r' && c != ' ' && c != '\t') out->back().push_back(c);
  }
}

struct Err {
  int64_t line = INT64_MAX;
  std::string msg;
};

bool blank(const char* b, const char* e) {
  for (const char* p = b; p < e; ++p)
    if (*p != ' ' && *p != '\t') return false;
  return true;
}

// One parsed field; returns false with the reference's message.
bool int_field(const std::string& s, int64_t line, const std::string& what, int64_t* v,
               std::string* msg) {
  long long x = 0;
  auto r = std::from_chars(s.data(), s.data() + s.size(), x);
  if (r.ec != std::errc() || r.ptr != s.data() + s.size()) {
    *msg = "line " + std::to_string(line) + ": bad integer " + what + " '" + s + "'";
    return false;
  }
  *v = x;
  return true;
}

bool real_field(const std::string& s, int64_t line, const std::string& what, double* v,
                std::string* msg) {
  double x = 0;
  auto r = std::from_chars(s.data(), s.data() + s.size(), x);
  if (r.ec != std::errc() || r.ptr != s.data() + s.size()) {
    *msg = "line " + std::to_string(line) + ": bad value for " + what + " '" + s + "'";
    return false;
  }
  if (!std::isfinite(x)) {
    *msg = "line " + std::to_string(line) + ": non-finite value for " + what;
    return false;
  }
  *v = x;
  return true;
}

struct Chunk {
  const char* b;
  const char* e;
  int64_t first_line;  // line number of the chunk's first line
  std::vector<int64_t> data, cfg, line;
  std::vector<double> val;
  Err err;
};

void parse_chunk_rows(Chunk& ch, int32_t d, const std::vector<std::string>& names);

// Parses the chunk; on an error the partial row is dropped (only complete
// rows before the failing line are kept).
void parse_chunk(Chunk& ch, int32_t d, const std::vector<std::string>& names) {
  parse_chunk_rows(ch, d, names);
  const size_t r = ch.line.size();
  ch.data.resize(r * (size_t)d);
  ch.cfg.resize(r * 3);
  ch.val.resize(r * names.size());
}

void parse_chunk_rows(Chunk& ch, int32_t d, const std::vector<std::string>& names) {
  std::vector<std::string> f;
  const size_t want = (size_t)d + 3 + names.size();
  int64_t ln = ch.first_line;
  for (const char* p = ch.b; p < ch.e; ++ln) {
    const char* q = static_cast<const char*>(memchr(p, '\n', (size_t)(ch.e - p)));
    const char* le = q ? q : ch.e;
    const char* next = q ? q + 1 : ch.e;
    const char* lend = (le > p && le[-1] == '\r') ? le - 1 : le;
    if (blank(p, lend)) {
      p = next;
      continue;
    }
    if (*p == '#') {
      ch.err = {ln, "line " + std::to_string(ln) + ": comments are only allowed before the header"};
      return;
    }
    split(p, lend, &f);
    if (f.size() != want) {
      ch.err = {ln, "line " + std::to_string(ln) + ": expected " + std::to_string(want) +
                        " fields, found " + std::to_string(f.size())};
      return;
    }
    std::string msg;
    int64_t v;
    for (int32_t i = 0; i < d; ++i) {
      if (!int_field(f[i], ln, "D" + std::to_string(i + 1), &v, &msg)) {
        ch.err = {ln, msg};
        return;
      }
      ch.data.push_back(v);
    }
    int64_t c3[3];
    const char* cn[3] = {"bx", "by", "bz"};
    for (int k = 0; k < 3; ++k)
      if (!int_field(f[d + k], ln, cn[k], &c3[k], &msg)) {
        ch.err = {ln, msg};
        return;
      }
    if (c3[0] < 1 || c3[1] < 1 || c3[2] < 1) {
      ch.err = {ln, "line " + std::to_string(ln) + ": block dimensions must be positive"};
      return;
    }
    ch.cfg.insert(ch.cfg.end(), c3, c3 + 3);
    for (size_t k = 0; k < names.size(); ++k) {
      double x;
      if (!real_field(f[d + 3 + k], ln, names[k], &x, &msg)) {
        ch.err = {ln, msg};
        return;
      }
      ch.val.push_back(x);
    }
    ch.line.push_back(ln);
    p = next;
  }
}

uint64_t mix(uint64_t h, uint64_t v) {
  h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
  return h * 0xff51afd7ed558ccdull;
}

int threads_for(int32_t n_threads, size_t bytes) {
  int t = n_threads > 0 ? n_threads : (int)std::thread::hardware_concurrency();
  t = std::max(1, std::min(t, 64));
  return (int)std::max<size_t>(1, std::min<size_t>((size_t)t, bytes / (1 << 16) + 1));
}

}  // namespace

extern "C" {

int rpg_samples_parse(const char* text, size_t len, int32_t n_threads, rpg_samples** out,
                      char* err, size_t errlen) {
  if (!out || (len && !text)) return cerr_(err, errlen, "rpg_samples_parse: null argument");
  *out = nullptr;
  rpg_samples S;
  // Header and the comments before it (datakit.hpp:336-379).
  const char* p = text;
  const char* end = text + len;
  int64_t ln = 0;
  bool have_header = false;
  std::vector<std::string> f;
  while (p < end && !have_header) {
    ++ln;
    const char* q = static_cast<const char*>(memchr(p, '\n', (size_t)(end - p)));
    const char* le = q ? q : end;
    const char* next = q ? q + 1 : end;
    const char* lend = (le > p && le[-1] == '\r') ? le - 1 : le;
    const std::string line(p, lend);
    p = next;
    if (blank(line.data(), line.data() + line.size())) continue;
    if (line[0] == '#') {
      // "# provenance: <kind> [key=value ...]" (whitespace-separated tokens)
      std::vector<std::string> tok;
      size_t i = 0;
      while (i < line.size()) {
        while (i < line.size() && isspace((unsigned char)line[i])) ++i;
        size_t j = i;
        while (j < line.size() && !isspace((unsigned char)line[j])) ++j;
        if (j > i) tok.push_back(line.substr(i, j - i));
        i = j;
      }
      const std::string tag = tok.size() > 1 ? tok[1] : "", kind = tok.size() > 2 ? tok[2] : "";
      if (tag == "provenance:") {
        if (kind == "measured") {
          S.prov_kind = 0;
          S.seed = 0;
          S.noise_rel = 0.0;
        } else if (kind == "synthetic") {
          S.prov_kind = 1;
          for (size_t k = 3; k < tok.size(); ++k) {
            const size_t eq = tok[k].find('=');
            if (eq == std::string::npos) continue;
            const std::string key = tok[k].substr(0, eq), val = tok[k].substr(eq + 1);
            if (key == "seed") {
              // std::stoull: optional blanks and sign, decimal digits (prefix)
              char* e2 = nullptr;
              errno = 0;
              const unsigned long long s = strtoull(val.c_str(), &e2, 10);
              if (e2 == val.c_str() || errno == ERANGE)
                return cerr_(err, errlen, "line %lld: bad provenance seed '%s'", (long long)ln,
                             val.c_str());
              S.seed = s;
            } else if (key == "noise_rel") {
              std::string msg;
              if (!real_field(val, ln, "noise_rel", &S.noise_rel, &msg))
                return cerr_(err, errlen, "%s", msg.c_str());
            }
          }
        } else {
          return cerr_(err, errlen, "line %lld: unknown provenance kind '%s'", (long long)ln,
                       kind.c_str());
        }
      }
      continue;
    }
    split(line.data(), line.data() + line.size(), &f);
    size_t i = 0;
    while (i < f.size() && f[i] == "D" + std::to_string(i + 1)) ++i;
    const size_t d = i;
    if (d == 0)
      return cerr_(err, errlen, "line %lld: header must start with data-parameter columns D1,...,Dd",
                   (long long)ln);
    if (f.size() < d + 4)
      return cerr_(err, errlen, "line %lld: header is missing block-dimension or metric columns",
                   (long long)ln);
    if (f[d] != "bx" || f[d + 1] != "by" || f[d + 2] != "bz")
      return cerr_(err, errlen, "line %lld: header must list bx,by,bz after the data parameters",
                   (long long)ln);
    for (size_t k = d + 3; k < f.size(); ++k) {
      if (f[k].empty()) return cerr_(err, errlen, "line %lld: empty metric column name", (long long)ln);
      if (std::find(S.names.begin(), S.names.end(), f[k]) != S.names.end())
        return cerr_(err, errlen, "line %lld: duplicate metric column '%s'", (long long)ln,
                     f[k].c_str());
      S.names.push_back(f[k]);
    }
    S.d = (int32_t)d;
    have_header = true;
  }
  if (!have_header) return cerr_(err, errlen, "no header row found");

  // Body: chunks at line boundaries, one thread each.
  const int T = threads_for(n_threads, (size_t)(end - p));
  std::vector<const char*> cut{p};
  for (int t = 1; t < T; ++t) {
    const char* c = p + (size_t)(end - p) * t / T;
    if (c < cut.back()) c = cut.back();
    const char* q = static_cast<const char*>(memchr(c, '\n', (size_t)(end - c)));
    cut.push_back(q ? q + 1 : end);
  }
  cut.push_back(end);
  std::vector<Chunk> chunks(T);
  std::vector<int64_t> nl(T, 0);
  {
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
      th.emplace_back([&, t] {
        int64_t k = 0;
        for (const char* c = cut[t]; c < cut[t + 1]; ++c) k += *c == '\n';
        nl[t] = k;
      });
    for (auto& x : th) x.join();
  }
  int64_t first = ln + 1;
  for (int t = 0; t < T; ++t) {
    chunks[t].b = cut[t];
    chunks[t].e = cut[t + 1];
    chunks[t].first_line = first;
    first += nl[t];
  }
  {
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t) th.emplace_back([&, t] { parse_chunk(chunks[t], S.d, S.names); });
    for (auto& x : th) x.join();
  }
  // Rows in file order up to the first parse error.
  Err perr;
  for (const Chunk& c : chunks)
    if (c.err.line < perr.line) perr = c.err;
  int64_t n = 0;
  for (const Chunk& c : chunks) n += (int64_t)c.line.size();
  const int32_t d = S.d, k = (int32_t)S.names.size();
  S.n = n;
  S.data.resize((size_t)n * d);
  S.configs.resize((size_t)n * 3);
  S.values.resize((size_t)n * k);
  std::vector<int64_t> line(n);
  {
    int64_t o = 0;
    for (const Chunk& c : chunks) {
      const int64_t r = (int64_t)c.line.size();
      std::copy(c.data.begin(), c.data.end(), S.data.begin() + o * d);
      std::copy(c.cfg.begin(), c.cfg.end(), S.configs.begin() + o * 3);
      std::copy(c.val.begin(), c.val.end(), S.values.begin() + o * k);
      std::copy(c.line.begin(), c.line.end(), line.begin() + o);
      o += r;
    }
  }
  // Duplicate keys: hash rows, bucket by hash across threads, sort buckets;
  // the failing line of a duplicated key is its second occurrence.
  std::vector<uint64_t> h(n);
  {
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
      th.emplace_back([&, t] {
        for (int64_t r = n * t / T; r < n * (t + 1) / T; ++r) {
          uint64_t x = 0x243f6a8885a308d3ull;
          for (int32_t i = 0; i < d; ++i) x = mix(x, (uint64_t)S.data[r * d + i]);
          for (int i = 0; i < 3; ++i) x = mix(x, (uint64_t)S.configs[r * 3 + i]);
          h[r] = x;
        }
      });
    for (auto& x : th) x.join();
  }
  std::vector<int64_t> dup(T, INT64_MAX);
  {
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
      th.emplace_back([&, t] {
        std::vector<std::pair<uint64_t, int64_t>> b;
        for (int64_t r = 0; r < n; ++r)
          if ((int)(h[r] % (uint64_t)T) == t) b.emplace_back(h[r], r);
        std::sort(b.begin(), b.end());
        auto same = [&](int64_t x, int64_t y) {
          for (int32_t i = 0; i < d; ++i)
            if (S.data[x * d + i] != S.data[y * d + i]) return false;
          for (int i = 0; i < 3; ++i)
            if (S.configs[x * 3 + i] != S.configs[y * 3 + i]) return false;
          return true;
        };
        for (size_t i = 0; i < b.size();) {
          size_t j = i;
          while (j < b.size() && b[j].first == b[i].first) ++j;
          // within one hash value: for each row, is an earlier row the same key?
          bool found = false;
          for (size_t a = i + 1; a < j && !found; ++a)
            for (size_t c = i; c < a; ++c)
              if (same(b[c].second, b[a].second)) {
                dup[t] = std::min(dup[t], b[a].second);
                found = true;
                break;
              }
          i = j;
        }
      });
    for (auto& x : th) x.join();
  }
  const int64_t drow = *std::min_element(dup.begin(), dup.end());
  if (drow != INT64_MAX && line[drow] < perr.line)
    return cerr_(err, errlen, "line %lld: duplicate sample for the same point and configuration",
                 (long long)line[drow]);
  if (perr.line != INT64_MAX) return cerr_(err, errlen, "%s", perr.msg.c_str());
  *out = new rpg_samples(std::move(S));
  return RPG_OK;
}

int rpg_samples_info(const rpg_samples* s, int64_t* n_rows, int32_t* d, int32_t* n_metrics,
                     int32_t* provenance_kind, uint64_t* seed, double* noise_rel) {
  if (!s) return RPG_E_INVALID;
  if (n_rows) *n_rows = s->n;
  if (d) *d = s->d;
  if (n_metrics) *n_metrics = (int32_t)s->names.size();
  if (provenance_kind) *provenance_kind = s->prov_kind;
  if (seed) *seed = s->seed;
  if (noise_rel) *noise_rel = s->noise_rel;
  return RPG_OK;
}

const char* rpg_samples_metric_name(const rpg_samples* s, int32_t k) {
  if (!s || k < 0 || k >= (int32_t)s->names.size()) return nullptr;
  return s->names[k].c_str();
}

int rpg_samples_copy(const rpg_samples* s, int64_t* data, int64_t* configs, double* values) {
  if (!s) return RPG_E_INVALID;
  if (data) std::copy(s->data.begin(), s->data.end(), data);
  if (configs) std::copy(s->configs.begin(), s->configs.end(), configs);
  if (values) std::copy(s->values.begin(), s->values.end(), values);
  return RPG_OK;
}

void rpg_samples_free(rpg_samples* s) { delete s; }

int64_t rpg_samples_format(const int64_t* data, const int64_t* configs, const double* values,
                           int64_t n, int32_t d, const char* const* metric_names,
                           int32_t n_metrics, int32_t provenance_kind, uint64_t seed,
                           double noise_rel, int32_t n_threads, char* buf, size_t buflen,
                           char* err, size_t errlen) {
  if (n <= 0) return cerr_(err, errlen, "cannot format an empty sample set");
  if (d < 0 || n_metrics < 0 || !configs || (d > 0 && !data) || (n_metrics > 0 && (!values || !metric_names)))
    return cerr_(err, errlen, "rpg_samples_format: null argument");
  auto fmt = [](double v, char* o) -> char* {
    return std::to_chars(o, o + 64, v).ptr;
  };
  // non-finite values: the reference names the first metric it meets
  for (int64_t r = 0; r < n; ++r)
    for (int32_t k = 0; k < n_metrics; ++k)
      if (!std::isfinite(values[r * n_metrics + k]))
        return cerr_(err, errlen, "metric '%s' has a non-finite value", metric_names[k]);
  std::string head;
  char tmp[64];
  if (provenance_kind == 1) {
    head = "# provenance: synthetic seed=" + std::to_string(seed) + " noise_rel=";
    head.append(tmp, fmt(noise_rel, tmp));
    head += "\n";
  } else {
    head = "# provenance: measured\n";
  }
  for (int32_t i = 1; i <= d; ++i) head += "D" + std::to_string(i) + ",";
  head += "bx,by,bz";
  for (int32_t k = 0; k < n_metrics; ++k) head += std::string(",") + metric_names[k];
  head += "\n";
  const int T = threads_for(n_threads, (size_t)n * 32);
  std::vector<std::string> part(T);
  {
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
      th.emplace_back([&, t] {
        std::string& o = part[t];
        char b[64];
        for (int64_t r = n * t / T; r < n * (t + 1) / T; ++r) {
          for (int32_t i = 0; i < d; ++i) {
            o.append(b, std::to_chars(b, b + 64, (long long)data[r * d + i]).ptr);
            o += ',';
          }
          for (int i = 0; i < 3; ++i) {
            if (i) o += ',';
            o.append(b, std::to_chars(b, b + 64, (long long)configs[r * 3 + i]).ptr);
          }
          for (int32_t k = 0; k < n_metrics; ++k) {
            o += ',';
            o.append(b, fmt(values[r * n_metrics + k], b));
          }
          o += '\n';
        }
      });
    for (auto& x : th) x.join();
  }
  size_t total = head.size();
  for (const auto& s : part) total += s.size();
  if (buf && buflen > 0) {
    size_t o = 0;
    auto put = [&](const std::string& s) {
      const size_t c = std::min(s.size(), buflen - 1 - std::min(o, buflen - 1));
      memcpy(buf + o, s.data(), c);
      o += c;
    };
    put(head);
    for (const auto& s : part) put(s);
    buf[std::min(o, buflen - 1)] = 0;
  }
  return (int64_t)total;
}

}  // extern "C"
