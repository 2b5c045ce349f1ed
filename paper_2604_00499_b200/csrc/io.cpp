// Input formats on either side of the path, host C++:
//   * request traces, JSONL one object per line -- save_trace / load_trace
//     (proj/src/workload.cpp:82-161): id, arrival_s, prompt_tokens, output_tokens,
//     max_tokens, optional mu / sigma; load fills missing arrivals from
//     poisson_arrivals(rps, count, seed) (workload.cpp:37-48) and stable-sorts by arrival;
//   * fit inputs (proj/tools/main.cpp:432-495): CSV with header "prompt_id,length" (rows
//     grouped by prompt id in first-seen order) or JSONL {"prompt_id": str, "lengths": [int]};
//     lengths are integers >= 1;
//   * a ragged fit report over such inputs: prompts grouped by sample count, one batched
//     GPU report (tie_fit_report_host) per group.
// The JSON reader is a small flat-object parser (the reference uses nlohmann-json): objects
// of scalar / string / flat-array members, which is everything these formats contain.
// Errors keep the reference's messages: load_trace's std::runtime_error text and the CLI's
// ConfigError "path:line: message" (both surface as TIE_EINVALID).
#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <set>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/tie_cuda.h"
#include "host_numerics.hpp"

namespace tie {
namespace capi {
int set_error(int code, const std::string& msg);
}
}  // namespace tie

namespace {

using tie::capi::set_error;

struct JVal {
  enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
  bool b = false;
  bool is_int = false;  // integer literal (no fraction / exponent), as nlohmann's is_number_integer
  bool neg = false;
  double num = 0.0;
  uint64_t u = 0;       // magnitude of an integer literal
  std::string str;
  std::vector<JVal> arr;
};

struct JParser {
  const char* p;
  const char* e;
  bool ok = true;
  void ws() {
    while (p < e && (*p == ' ' || *p == '\t' || *p == '\r' || *p == '\n')) ++p;
  }
  bool lit(const char* s) {
    const size_t n = std::strlen(s);
    if ((size_t)(e - p) >= n && std::memcmp(p, s, n) == 0) {
      p += n;
      return true;
    }
    return false;
  }
  bool string(std::string& out) {
    if (p >= e || *p != '"') return false;
    ++p;
    while (p < e && *p != '"') {
      if (*p == '\\') {
        if (++p >= e) return false;
        switch (*p) {
          case '"': out += '"'; break;
          case '\\': out += '\\'; break;
          case '/': out += '/'; break;
          case 'b': out += '\b'; break;
          case 'f': out += '\f'; break;
          case 'n': out += '\n'; break;
          case 'r': out += '\r'; break;
          case 't': out += '\t'; break;
          case 'u': {
            if (e - p < 5) return false;
            const unsigned cp = (unsigned)std::strtoul(std::string(p + 1, p + 5).c_str(), nullptr, 16);
            if (cp < 0x80) {
              out += (char)cp;
            } else if (cp < 0x800) {
              out += (char)(0xC0 | (cp >> 6));
              out += (char)(0x80 | (cp & 0x3F));
            } else {
              out += (char)(0xE0 | (cp >> 12));
              out += (char)(0x80 | ((cp >> 6) & 0x3F));
              out += (char)(0x80 | (cp & 0x3F));
            }
            p += 4;
            break;
          }
          default: return false;
        }
        ++p;
      } else {
        out += *p++;
      }
    }
    if (p >= e) return false;
    ++p;
    return true;
  }
  bool number(JVal& v) {
    const char* s = p;
    if (p < e && *p == '-') ++p;
    const char* digits = p;
    while (p < e && *p >= '0' && *p <= '9') ++p;
    if (p == digits) return false;
    bool frac = false;
    if (p < e && *p == '.') {
      frac = true;
      ++p;
      while (p < e && *p >= '0' && *p <= '9') ++p;
    }
    if (p < e && (*p == 'e' || *p == 'E')) {
      frac = true;
      ++p;
      if (p < e && (*p == '+' || *p == '-')) ++p;
      while (p < e && *p >= '0' && *p <= '9') ++p;
    }
    const std::string tok(s, p);
    v.kind = JVal::Num;
    v.num = std::strtod(tok.c_str(), nullptr);
    v.is_int = !frac;
    v.neg = tok[0] == '-';
    if (v.is_int) v.u = std::strtoull(digits, nullptr, 10);
    return true;
  }
  bool value(JVal& v, int depth) {
    ws();
    if (p >= e || depth > 8) return false;
    if (*p == '"') {
      v.kind = JVal::Str;
      return string(v.str);
    }
    if (*p == '{') {
      ++p;
      v.kind = JVal::Obj;
      ws();
      if (p < e && *p == '}') {
        ++p;
        return true;
      }
      while (true) {
        ws();
        JVal kv;  // (key, value) pair: kv.str = key, kv.arr[0] = value
        if (!string(kv.str)) return false;
        ws();
        if (p >= e || *p != ':') return false;
        ++p;
        kv.arr.emplace_back();
        if (!value(kv.arr[0], depth + 1)) return false;
        v.arr.push_back(std::move(kv));
        ws();
        if (p < e && *p == ',') {
          ++p;
          continue;
        }
        if (p < e && *p == '}') {
          ++p;
          return true;
        }
        return false;
      }
    }
    if (*p == '[') {
      ++p;
      v.kind = JVal::Arr;
      ws();
      if (p < e && *p == ']') {
        ++p;
        return true;
      }
      while (true) {
        JVal item;
        if (!value(item, depth + 1)) return false;
        v.arr.push_back(std::move(item));
        ws();
        if (p < e && *p == ',') {
          ++p;
          continue;
        }
        if (p < e && *p == ']') {
          ++p;
          return true;
        }
        return false;
      }
    }
    if (lit("true")) {
      v.kind = JVal::Bool;
      v.b = true;
      return true;
    }
    if (lit("false")) {
      v.kind = JVal::Bool;
      return true;
    }
    if (lit("null")) return true;
    return number(v);
  }
};

// parse one line; false on malformed JSON
bool parse_line(const std::string& line, JVal& out) {
  JParser jp{line.data(), line.data() + line.size()};
  if (!jp.value(out, 0)) return false;
  jp.ws();
  return jp.p == jp.e;
}

const JVal* member(const JVal& obj, const char* key) {
  for (const JVal& kv : obj.arr)
    if (kv.str == key) return &kv.arr[0];
  return nullptr;
}

// nlohmann get<T>() of a number (numeric conversions are static_casts)
uint64_t as_u64(const JVal& v) {
  if (v.is_int) return v.neg ? (uint64_t)(-(int64_t)v.u) : v.u;
  return (uint64_t)v.num;
}

struct Trace {
  std::vector<uint64_t> id;
  std::vector<double> arrival;
  std::vector<uint32_t> prompt, output, max_tokens;
  std::vector<double> mu, sigma;  // NaN = absent
};

struct FitInput {
  std::vector<std::string> ids;
  std::vector<uint64_t> offsets{0};
  std::vector<double> lengths;
};

}  // namespace

struct tie_trace : Trace {};
struct tie_fit_input : FitInput {};

extern "C" {

// ---------------------------------------------------------------- traces
int tie_trace_load(const char* path, double fill_rps, uint64_t seed, tie_trace** out) {
  if (!path || !out) return set_error(TIE_EINVALID, "tie_trace_load: null argument");
  *out = nullptr;
  std::ifstream in(path);
  if (!in) return set_error(TIE_EINVALID, std::string("load_trace: cannot open ") + path);
  auto* t = new tie_trace();
  std::vector<size_t> missing;
  std::set<uint64_t> seen;
  std::string line;
  size_t lineno = 0;
  auto fail = [&](const std::string& msg) {
    delete t;
    return set_error(TIE_EINVALID, "load_trace: " + std::string(path) + ":" +
                                       std::to_string(lineno) + ": " + msg);
  };
  while (std::getline(in, line)) {
    ++lineno;
    if (line.empty()) continue;
    JVal j;
    if (!parse_line(line, j) || j.kind != JVal::Obj) return fail("bad JSON");
    for (const char* f : {"id", "prompt_tokens", "output_tokens", "max_tokens"})
      if (!member(j, f)) return fail(std::string("missing field '") + f + "'");
    for (const char* f : {"id", "prompt_tokens", "output_tokens", "max_tokens", "arrival_s",
                          "mu", "sigma"}) {
      const JVal* v = member(j, f);
      if (v && v->kind != JVal::Num) return fail(std::string("field '") + f + "' is not a number");
    }
    const uint64_t id = as_u64(*member(j, "id"));
    if (!seen.insert(id).second) return fail("duplicate id " + std::to_string(id));
    t->id.push_back(id);
    t->prompt.push_back((uint32_t)as_u64(*member(j, "prompt_tokens")));
    t->output.push_back((uint32_t)as_u64(*member(j, "output_tokens")));
    t->max_tokens.push_back((uint32_t)as_u64(*member(j, "max_tokens")));
    if (const JVal* a = member(j, "arrival_s")) {
      t->arrival.push_back(a->num);
    } else {
      t->arrival.push_back(-1.0);
      missing.push_back(t->id.size() - 1);
    }
    const JVal* m = member(j, "mu");
    const JVal* s = member(j, "sigma");
    t->mu.push_back(m ? m->num : std::nan(""));
    t->sigma.push_back(s ? s->num : std::nan(""));
  }
  if (!missing.empty()) {
    if (!(fill_rps > 0.0)) {
      delete t;
      return set_error(TIE_EINVALID, std::string("load_trace: ") + path +
                                         ": records missing arrival_s but no fill rate supplied");
    }
    if (!std::isfinite(fill_rps)) {
      delete t;
      return set_error(TIE_EDOMAIN, "poisson_arrivals: rps must be finite and > 0");
    }
    tie::host::Sampler rng(seed);  // poisson_arrivals (workload.cpp:37-48)
    double acc = 0.0;
    for (size_t k = 0; k < missing.size(); ++k) t->arrival[missing[k]] = (acc += rng.exponential(fill_rps));
  }
  // stable sort by arrival (workload.cpp:157-159)
  std::vector<size_t> perm(t->id.size());
  for (size_t i = 0; i < perm.size(); ++i) perm[i] = i;
  std::stable_sort(perm.begin(), perm.end(),
                   [&](size_t a, size_t b) { return t->arrival[a] < t->arrival[b]; });
  auto apply = [&](auto& v) {
    auto c = v;
    for (size_t i = 0; i < perm.size(); ++i) v[i] = c[perm[i]];
  };
  apply(t->id);
  apply(t->arrival);
  apply(t->prompt);
  apply(t->output);
  apply(t->max_tokens);
  apply(t->mu);
  apply(t->sigma);
  *out = t;
  return TIE_OK;
}

uint64_t tie_trace_size(const tie_trace* t) { return t ? t->id.size() : 0; }
const uint64_t* tie_trace_ids(const tie_trace* t) { return t ? t->id.data() : nullptr; }
const double* tie_trace_arrival(const tie_trace* t) { return t ? t->arrival.data() : nullptr; }
const uint32_t* tie_trace_prompt_tokens(const tie_trace* t) { return t ? t->prompt.data() : nullptr; }
const uint32_t* tie_trace_output_tokens(const tie_trace* t) { return t ? t->output.data() : nullptr; }
const uint32_t* tie_trace_max_tokens(const tie_trace* t) { return t ? t->max_tokens.data() : nullptr; }
const double* tie_trace_mu(const tie_trace* t) { return t ? t->mu.data() : nullptr; }
const double* tie_trace_sigma(const tie_trace* t) { return t ? t->sigma.data() : nullptr; }
void tie_trace_free(tie_trace* t) { delete t; }

// save_trace (workload.cpp:82-104): one object per request in the given order; mu / sigma
// written when given and not NaN.  Doubles with 17 significant digits (round-trip exact).
int tie_trace_save(const char* path, uint64_t n, const uint64_t* ids, const double* arrival,
                   const uint32_t* prompt_tokens, const uint32_t* output_tokens,
                   const uint32_t* max_tokens, const double* mu, const double* sigma) {
  if (!path) return set_error(TIE_EINVALID, "tie_trace_save: null path");
  FILE* f = std::fopen(path, "w");
  if (!f) return set_error(TIE_EINVALID, std::string("save_trace: cannot open ") + path);
  char buf[512];
  for (uint64_t i = 0; i < n; ++i) {
    int k = std::snprintf(buf, sizeof(buf),
                          "{\"arrival_s\":%.17g,\"id\":%llu,\"max_tokens\":%u,", arrival[i],
                          (unsigned long long)ids[i], max_tokens[i]);
    if (mu && !std::isnan(mu[i])) k += std::snprintf(buf + k, sizeof(buf) - k, "\"mu\":%.17g,", mu[i]);
    k += std::snprintf(buf + k, sizeof(buf) - k, "\"output_tokens\":%u,\"prompt_tokens\":%u",
                       output_tokens[i], prompt_tokens[i]);
    if (sigma && !std::isnan(sigma[i]))
      k += std::snprintf(buf + k, sizeof(buf) - k, ",\"sigma\":%.17g", sigma[i]);
    std::fputs(buf, f);
    std::fputs("}\n", f);
  }
  const bool bad = std::ferror(f) != 0;
  std::fclose(f);
  if (bad) return set_error(TIE_EINVALID, std::string("save_trace: write failed on ") + path);
  return TIE_OK;
}

// ---------------------------------------------------------------- fit inputs
int tie_fit_input_load(const char* path, tie_fit_input** out) {
  if (!path || !out) return set_error(TIE_EINVALID, "tie_fit_input_load: null argument");
  *out = nullptr;
  const std::string sp(path);
  std::ifstream in(sp);
  if (!in) return set_error(TIE_EINVALID, "cannot open input: " + sp);
  auto* fi = new tie_fit_input();
  std::vector<std::vector<double>> rows;
  std::unordered_map<std::string, size_t> index;
  std::string line;
  int lineno = 0;
  auto fail = [&](const std::string& msg) {
    delete fi;
    return set_error(TIE_EINVALID, sp + ":" + std::to_string(lineno) + ": " + msg);
  };
  const bool csv = sp.size() >= 4 && sp.substr(sp.size() - 4) == ".csv";
  if (csv) {
    if (!std::getline(in, line)) {
      delete fi;
      return set_error(TIE_EINVALID, sp + ": empty file");
    }
    lineno = 1;
    if (!line.empty() && line.back() == '\r') line.pop_back();
    if (line != "prompt_id,length") return fail("expected header prompt_id,length");
    while (std::getline(in, line)) {
      ++lineno;
      if (!line.empty() && line.back() == '\r') line.pop_back();
      if (line.empty()) continue;
      const size_t comma = line.find(',');
      if (comma == std::string::npos) return fail("expected prompt_id,length");
      const std::string id = line.substr(0, comma);
      const std::string num = line.substr(comma + 1);
      // std::stoll with the used-count check (main.cpp:454-464)
      const char* b = num.c_str();
      while (*b == ' ' || *b == '\t' || *b == '\n' || *b == '\v' || *b == '\f' || *b == '\r') ++b;
      char* endp = nullptr;
      errno = 0;
      const long long len = std::strtoll(b, &endp, 10);
      if (endp == b || errno == ERANGE || *endp != '\0') return fail("length must be an integer");
      if (len < 1) return fail("length must be >= 1");
      auto it = index.find(id);
      if (it == index.end()) {
        it = index.emplace(id, rows.size()).first;
        fi->ids.push_back(id);
        rows.emplace_back();
      }
      rows[it->second].push_back((double)len);
    }
  } else {
    while (std::getline(in, line)) {
      ++lineno;
      if (!line.empty() && line.back() == '\r') line.pop_back();
      if (line.empty()) continue;
      JVal rec;
      if (!parse_line(line, rec)) return fail("invalid JSON");
      const JVal* pid = rec.kind == JVal::Obj ? member(rec, "prompt_id") : nullptr;
      const JVal* lens = rec.kind == JVal::Obj ? member(rec, "lengths") : nullptr;
      if (!pid || !lens) return fail("expected {\"prompt_id\", \"lengths\"}");
      if (pid->kind != JVal::Str) return fail("prompt_id must be a string");
      if (lens->kind != JVal::Arr) return fail("lengths must be an array");
      if (index.count(pid->str)) return fail("duplicate prompt_id " + pid->str);
      index[pid->str] = rows.size();
      fi->ids.push_back(pid->str);
      rows.emplace_back();
      for (const JVal& v : lens->arr) {
        if (v.kind != JVal::Num || !v.is_int || v.neg || v.u < 1)
          return fail("lengths must be integers >= 1");
        rows.back().push_back((double)v.u);
      }
    }
  }
  if (rows.empty()) {
    delete fi;
    return set_error(TIE_EINVALID, sp + ": no prompts found");
  }
  for (const auto& r : rows) {
    fi->lengths.insert(fi->lengths.end(), r.begin(), r.end());
    fi->offsets.push_back(fi->lengths.size());
  }
  *out = fi;
  return TIE_OK;
}

uint64_t tie_fit_input_count(const tie_fit_input* f) { return f ? f->ids.size() : 0; }
const char* tie_fit_input_prompt_id(const tie_fit_input* f, uint64_t i) {
  return f && i < f->ids.size() ? f->ids[i].c_str() : nullptr;
}
const uint64_t* tie_fit_input_offsets(const tie_fit_input* f) { return f ? f->offsets.data() : nullptr; }
const double* tie_fit_input_lengths(const tie_fit_input* f) { return f ? f->lengths.data() : nullptr; }
void tie_fit_input_free(tie_fit_input* f) { delete f; }

// Ragged fit report: prompt p's samples are lengths[offsets[p] .. offsets[p+1]); prompts are
// grouped by sample count and each group runs as one dense batch; fits[4][10][P], tail[5][P]
// as tie_fit_report.  Every prompt needs >= 5 samples (cmd_fit, main.cpp:517-519).
int tie_fit_report_ragged_host(tie_ctx* ctx, const double* lengths, const uint64_t* offsets,
                               uint64_t P, double nu, unsigned families, double* fits,
                               double* tail) {
  if (!lengths || !offsets || !fits) return set_error(TIE_EINVALID, "tie_fit_report_ragged_host: null pointer");
  std::map<uint64_t, std::vector<uint64_t>> groups;
  for (uint64_t p = 0; p < P; ++p) {
    const uint64_t K = offsets[p + 1] - offsets[p];
    if (K < 5)
      return set_error(TIE_EINVALID, "prompt " + std::to_string(p) + " has fewer than 5 samples");
    groups[K].push_back(p);
  }
  for (const auto& [K, ps] : groups) {
    const uint64_t m = ps.size();
    std::vector<double> x(m * K), f(4 * 10 * m), t(5 * m);
    for (uint64_t j = 0; j < m; ++j)
      std::memcpy(&x[j * K], lengths + offsets[ps[j]], 8 * K);
    for (int fam = 0; fam < 4; ++fam)
      for (int fld = 0; fld < 10; ++fld)
        for (uint64_t j = 0; j < m; ++j)
          f[((uint64_t)fam * 10 + fld) * m + j] = fits[((uint64_t)fam * 10 + fld) * P + ps[j]];
    if (int rc = tie_fit_report_host(ctx, x.data(), m, K, nu, families, f.data(),
                                     tail ? t.data() : nullptr))
      return rc;
    for (int fam = 0; fam < 4; ++fam)
      for (int fld = 0; fld < 10; ++fld)
        for (uint64_t j = 0; j < m; ++j)
          fits[((uint64_t)fam * 10 + fld) * P + ps[j]] = f[((uint64_t)fam * 10 + fld) * m + j];
    if (tail)
      for (int fld = 0; fld < 5; ++fld)
        for (uint64_t j = 0; j < m; ++j) tail[(uint64_t)fld * P + ps[j]] = t[(uint64_t)fld * m + j];
  }
  return TIE_OK;
}

}  // extern "C"
