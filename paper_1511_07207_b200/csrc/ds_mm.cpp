// ds_mm.cpp — native Matrix Market reader (host side of the input path).
//
// Restates harness.read_matrix_market (/root/reference/pkg/src/densolve/harness.py:130-220):
// 'array' and 'coordinate' formats, field 'real', symmetry 'general' or
// 'symmetric' (mirrored on read), 1-based indices, unlisted coordinate entries
// zero, comment ('%') and blank lines skipped, every error tagged with the
// offending 1-based line number (MatrixMarketError.line).  The file is parsed
// once with a single pass over an mmap-free buffered read; values go straight
// into the caller's column-major buffer (which may be pinned host memory the
// caller then uploads with one copy).
#include <cctype>
#include <cerrno>
#include <cmath>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/densolve_b200.h"

namespace {

thread_local std::string g_mm_err;

int mm_fail(int64_t line, int64_t* err_line, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_mm_err = "line " + std::to_string(line) + ": " + buf;
  if (err_line) *err_line = line;
  return DS_EMM;
}

std::vector<std::string> split_ws(const std::string& s) {
  std::vector<std::string> out;
  size_t i = 0;
  while (i < s.size()) {
    while (i < s.size() && isspace((unsigned char)s[i])) ++i;
    size_t j = i;
    while (j < s.size() && !isspace((unsigned char)s[j])) ++j;
    if (j > i) out.emplace_back(s.substr(i, j - i));
    i = j;
  }
  return out;
}

std::string strip(const std::string& s) {
  size_t a = 0, b = s.size();
  while (a < b && isspace((unsigned char)s[a])) ++a;
  while (b > a && isspace((unsigned char)s[b - 1])) --b;
  return s.substr(a, b - a);
}

std::string lower(std::string s) {
  for (auto& c : s) c = (char)tolower((unsigned char)c);
  return s;
}

// Python int(): optional sign, decimal digits (underscores between digits allowed)
bool parse_int(const std::string& t, int64_t* v) {
  size_t i = 0;
  bool neg = false;
  if (i < t.size() && (t[i] == '+' || t[i] == '-')) neg = t[i++] == '-';
  if (i >= t.size()) return false;
  int64_t x = 0;
  bool prev_digit = false;
  for (; i < t.size(); ++i) {
    const char c = t[i];
    if (c == '_' && prev_digit && i + 1 < t.size() && isdigit((unsigned char)t[i + 1])) {
      prev_digit = false;
      continue;
    }
    if (!isdigit((unsigned char)c)) return false;
    x = x * 10 + (c - '0');
    prev_digit = true;
  }
  *v = neg ? -x : x;
  return true;
}

// Python float(): decimal / exponent forms, inf/infinity/nan (any case, signed); no hex
bool parse_float(const std::string& t, double* v) {
  if (t.empty()) return false;
  std::string u;
  u.reserve(t.size());
  for (size_t i = 0; i < t.size(); ++i) {
    const char c = t[i];
    if (c == '_') {
      if (i == 0 || i + 1 >= t.size() || !isdigit((unsigned char)t[i - 1]) || !isdigit((unsigned char)t[i + 1]))
        return false;
      continue;
    }
    u.push_back(c);
  }
  const std::string l = lower(u);
  size_t k = (l[0] == '+' || l[0] == '-') ? 1 : 0;
  if (l.compare(k, std::string::npos, "x") == 0 || l.find("0x", k) == k) return false;  // no hex
  errno = 0;
  char* end = nullptr;
  const double d = strtod(u.c_str(), &end);
  if (end != u.c_str() + u.size()) return false;
  *v = d;
  return true;
}

}  // namespace

extern "C" {

const char* ds_mm_last_error(void) { return g_mm_err.c_str(); }

int ds_mm_read(const char* path, double* out, int64_t cap, int64_t* rows_out, int64_t* cols_out,
               int64_t* err_line) {
  if (err_line) *err_line = 0;
  FILE* fh = fopen(path, "rb");
  if (!fh) {
    g_mm_err = std::string("No such file or directory: '") + path + "'";
    return DS_ENOFILE;
  }
  std::vector<std::string> lines;
  {
    std::string cur;
    char buf[1 << 16];
    size_t got;
    while ((got = fread(buf, 1, sizeof buf, fh)) > 0) {
      for (size_t i = 0; i < got; ++i) {
        cur.push_back(buf[i]);
        if (buf[i] == '\n') {
          lines.emplace_back(std::move(cur));
          cur.clear();
        }
      }
    }
    if (!cur.empty()) lines.emplace_back(std::move(cur));
    fclose(fh);
  }
  if (lines.empty()) return mm_fail(1, err_line, "empty file");
  const auto header = split_ws(lines[0]);
  if (header.size() != 5 || header[0] != "%%MatrixMarket" || header[1] != "matrix")
    return mm_fail(1, err_line, "malformed header '%s'", strip(lines[0]).c_str());
  const std::string fmt = lower(header[2]), field = lower(header[3]), sym = lower(header[4]);
  if (fmt != "array" && fmt != "coordinate") return mm_fail(1, err_line, "unsupported format '%s'", fmt.c_str());
  if (field != "real") return mm_fail(1, err_line, "unsupported field '%s' (only 'real')", field.c_str());
  if (sym != "general" && sym != "symmetric") return mm_fail(1, err_line, "unsupported symmetry '%s'", sym.c_str());
  const bool symmetric = sym == "symmetric";

  // body: (1-based line number, stripped text) of non-blank, non-comment lines
  std::vector<std::pair<int64_t, std::string>> body;
  for (size_t i = 1; i < lines.size(); ++i) {
    const std::string t = strip(lines[i]);
    if (t.empty() || t[0] == '%') continue;
    body.emplace_back((int64_t)i + 1, t);
  }
  if (body.empty()) return mm_fail((int64_t)lines.size(), err_line, "missing size line");
  const int64_t size_ln = body[0].first;
  const auto parts = split_ws(body[0].second);
  int64_t rows = 0, cols = 0, nnz = -1;
  if (fmt == "array") {
    if (parts.size() != 2 || !parse_int(parts[0], &rows) || !parse_int(parts[1], &cols))
      return mm_fail(size_ln, err_line, "bad size line '%s'", body[0].second.c_str());
  } else {
    if (parts.size() != 3 || !parse_int(parts[0], &rows) || !parse_int(parts[1], &cols) ||
        !parse_int(parts[2], &nnz))
      return mm_fail(size_ln, err_line, "bad size line '%s'", body[0].second.c_str());
  }
  if (rows < 0 || cols < 0) return mm_fail(size_ln, err_line, "negative dimensions");
  *rows_out = rows;
  *cols_out = cols;
  if (out == nullptr || cap < rows * cols) return DS_OK;  // size query
  for (int64_t e = 0; e < rows * cols; ++e) out[e] = 0.0;
  const size_t nent = body.size() - 1;
  const int64_t last_ln = nent ? body.back().first : size_ln;
  if (fmt == "array") {
    int64_t expected = rows * cols;
    if (symmetric) {
      expected = 0;
      for (int64_t j = 0; j < cols; ++j) expected += rows - j;
    }
    if ((int64_t)nent != expected)
      return mm_fail(last_ln, err_line, "expected %lld values, found %lld", (long long)expected, (long long)nent);
    size_t idx = 1;
    for (int64_t j = 0; j < cols; ++j) {
      for (int64_t i = symmetric ? j : 0; i < rows; ++i) {
        const auto& e = body[idx++];
        const auto tok = split_ws(e.second);
        double v = 0.0;
        if (tok.empty() || !parse_float(tok[0], &v)) return mm_fail(e.first, err_line, "bad value '%s'", e.second.c_str());
        out[i + j * rows] = v;
        if (symmetric && i != j) out[j + i * rows] = v;
      }
    }
  } else {
    if ((int64_t)nent != nnz)
      return mm_fail(last_ln, err_line, "expected %lld entries, found %lld", (long long)nnz, (long long)nent);
    for (size_t k = 1; k < body.size(); ++k) {
      const auto& e = body[k];
      const auto tok = split_ws(e.second);
      if (tok.size() != 3) return mm_fail(e.first, err_line, "expected 'i j value', got '%s'", e.second.c_str());
      int64_t i = 0, j = 0;
      double v = 0.0;
      if (!parse_int(tok[0], &i) || !parse_int(tok[1], &j) || !parse_float(tok[2], &v))
        return mm_fail(e.first, err_line, "bad entry '%s'", e.second.c_str());
      if (!(1 <= i && i <= rows && 1 <= j && j <= cols))
        return mm_fail(e.first, err_line, "index (%lld, %lld) out of range for %lldx%lld", (long long)i,
                       (long long)j, (long long)rows, (long long)cols);
      out[(i - 1) + (j - 1) * rows] = v;
      if (symmetric && i != j) out[(j - 1) + (i - 1) * rows] = v;
    }
  }
  return DS_OK;
}

}  // extern "C"
