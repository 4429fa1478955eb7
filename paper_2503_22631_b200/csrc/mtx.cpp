// Matrix Market and plain-text vector interchange (host side of the ABI).
//
// Restates the reference's sparse::load_matrix_market / save_matrix_market /
// load_vector / save_vector (proj/src/sparse.cpp:140-242, declared at
// include/rkmf/sparse.hpp:55-66): "coordinate real {general|symmetric}"
// only, symmetric inputs expanded to full storage, 1-based indices
// converted, duplicates summed, rows sorted (from_triplets, sparse.cpp:14-47);
// vectors as one decimal value per line with '%' comments and blank lines
// skipped; writes at 17 significant digits. Parse failures carry
// "path:line: what" with the reference's messages (ParseError -> status
// RKMF_PARSE_ERROR). These feed the reference's `external` problem workflow
// (problems.cpp:494-508) into the device path: rkmf_matrix_load_mtx uploads
// the parsed CSR through rkmf_matrix_create_host.
//
// The parser reads the whole file once and scans it with strtol/strtod
// (correctly rounded, like the istream extraction the reference uses)
// instead of one istringstream per line: an order of magnitude faster on
// the 10^7-10^8-line files the device path is sized for.
#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "rkmf_b200.h"

namespace {

struct Fail : std::runtime_error {
  int code;
  Fail(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] void parse_fail(const std::string& path, long line, const std::string& what) {
  throw Fail(RKMF_PARSE_ERROR, path + ":" + std::to_string(line) + ": " + what);
}

int report(const Fail& f, char* err, int64_t cap) {
  if (err && cap > 0) {
    std::strncpy(err, f.what(), size_t(cap - 1));
    err[cap - 1] = '\0';
  }
  return f.code;
}

std::string read_all(const std::string& path) {
  FILE* fp = std::fopen(path.c_str(), "rb");
  if (!fp) throw Fail(RKMF_PARSE_ERROR, path + ": cannot open");
  std::string buf;
  char chunk[1 << 16];
  size_t got;
  while ((got = std::fread(chunk, 1, sizeof(chunk), fp)) > 0) buf.append(chunk, got);
  std::fclose(fp);
  return buf;
}

// Lines of a buffer (std::getline semantics: '\n' separated, a trailing
// '\r' kept, the last line needs no terminator).
struct Lines {
  const std::string& s;
  size_t pos = 0;
  long lineno = 0;
  explicit Lines(const std::string& b) : s(b) {}
  bool next(const char*& b, const char*& e) {
    if (pos >= s.size()) return false;
    const size_t nl = s.find('\n', pos);
    const size_t end = nl == std::string::npos ? s.size() : nl;
    b = s.data() + pos;
    e = s.data() + end;
    pos = nl == std::string::npos ? s.size() : nl + 1;
    ++lineno;
    return true;
  }
};

std::string lower(std::string x) {
  for (char& c : x) c = char(std::tolower(static_cast<unsigned char>(c)));
  return x;
}

bool is_space(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }

// istream >> long / >> double on [p, e): skip blanks, parse, advance p.
bool get_long(const char*& p, const char* e, long& out) {
  while (p < e && is_space(*p)) ++p;
  if (p >= e) return false;
  std::string tok;
  const char* q = p;
  while (q < e && !is_space(*q)) ++q;
  tok.assign(p, q);
  char* end = nullptr;
  errno = 0;
  const long v = std::strtol(tok.c_str(), &end, 10);
  if (end == tok.c_str() || errno == ERANGE) return false;
  p += (end - tok.c_str());
  out = v;
  return true;
}
bool get_double(const char*& p, const char* e, double& out) {
  while (p < e && is_space(*p)) ++p;
  if (p >= e) return false;
  const char* q = p;
  while (q < e && !is_space(*q)) ++q;
  std::string tok(p, q);
  // istream extraction takes decimal numbers only (no inf / nan / hex)
  for (char c : tok)
    if (!(std::isdigit(static_cast<unsigned char>(c)) || c == '+' || c == '-' || c == '.' ||
          c == 'e' || c == 'E'))
      return false;
  char* end = nullptr;
  const double v = std::strtod(tok.c_str(), &end);
  if (end == tok.c_str()) return false;
  p += (end - tok.c_str());
  out = v;
  return true;
}
bool rest_blank(const char* p, const char* e) {
  while (p < e && is_space(*p)) ++p;
  return p >= e;
}
bool skip_line(const char* b, const char* e) { return b == e || *b == '%'; }

struct Trip {
  int64_t r, c;
  double v;
};

// from_triplets (sparse.cpp:14-47): sort by (row, col), sum duplicates
void to_csr(int64_t n_rows, int64_t n_cols, std::vector<Trip>& t, std::vector<int64_t>& rp,
            std::vector<int32_t>& ci, std::vector<double>& v) {
  if (n_rows < 0 || n_cols < 0) throw Fail(RKMF_PARAMETER_ERROR, "negative matrix size");
  if (n_cols > (int64_t(1) << 31) - 1)
    throw Fail(RKMF_SHAPE_ERROR, "rkmf_b200: column indices must fit int32");
  std::stable_sort(t.begin(), t.end(), [](const Trip& a, const Trip& b) {
    return a.r != b.r ? a.r < b.r : a.c < b.c;
  });
  rp.assign(size_t(n_rows) + 1, 0);
  ci.clear();
  v.clear();
  ci.reserve(t.size());
  v.reserve(t.size());
  size_t i = 0;
  while (i < t.size()) {
    const int64_t r = t[i].r, c = t[i].c;
    double s = t[i].v;
    ++i;
    while (i < t.size() && t[i].r == r && t[i].c == c) s += t[i++].v;  // duplicates summed
    ci.push_back(int32_t(c));
    v.push_back(s);
    ++rp[size_t(r) + 1];
  }
  for (int64_t r = 0; r < n_rows; ++r) rp[size_t(r) + 1] += rp[size_t(r)];
}

void load_mtx(const std::string& path, int64_t& nr, int64_t& nc, std::vector<int64_t>& rp,
              std::vector<int32_t>& ci, std::vector<double>& v) {
  const std::string buf = read_all(path);
  Lines L(buf);
  const char *b, *e;
  if (!L.next(b, e)) parse_fail(path, 1, "empty file");
  {
    std::vector<std::string> w;
    const char* p = b;
    while (p < e) {
      while (p < e && is_space(*p)) ++p;
      const char* q = p;
      while (q < e && !is_space(*q)) ++q;
      if (q > p) w.emplace_back(p, q);
      p = q;
    }
    w.resize(std::max<size_t>(w.size(), 5));
    if (w[0] != "%%MatrixMarket" || lower(w[1]) != "matrix")
      parse_fail(path, L.lineno, "malformed MatrixMarket header");
    if (lower(w[2]) != "coordinate") parse_fail(path, L.lineno, "only coordinate format is supported");
    if (lower(w[3]) != "real") parse_fail(path, L.lineno, "only real field is supported");
    const std::string sym = lower(w[4]);
    if (sym != "general" && sym != "symmetric")
      parse_fail(path, L.lineno, "only general/symmetric qualifiers are supported");
    w[4] = sym;
    long rows = -1, cols = -1, declared = -1;
    while (L.next(b, e)) {
      if (skip_line(b, e)) continue;
      const char* p = b;
      if (!(get_long(p, e, rows) && get_long(p, e, cols) && get_long(p, e, declared)))
        parse_fail(path, L.lineno, "malformed size line");
      break;
    }
    if (rows < 0 || cols < 0 || declared < 0) parse_fail(path, L.lineno, "missing size line");
    const bool symmetric = w[4] == "symmetric";
    std::vector<Trip> t;
    t.reserve(size_t(declared) * (symmetric ? 2 : 1));
    long seen = 0;
    while (L.next(b, e)) {
      if (skip_line(b, e)) continue;
      const char* p = b;
      long r = 0, c = 0;
      double x = 0.0;
      if (!(get_long(p, e, r) && get_long(p, e, c) && get_double(p, e, x)))
        parse_fail(path, L.lineno, "malformed coordinate line (expected: row col real-value)");
      if (r < 1 || r > rows || c < 1 || c > cols) parse_fail(path, L.lineno, "index out of range");
      t.push_back({r - 1, c - 1, x});
      if (symmetric && r != c) t.push_back({c - 1, r - 1, x});
      ++seen;
    }
    if (seen != declared) parse_fail(path, L.lineno, "entry count does not match header");
    nr = rows;
    nc = cols;
    to_csr(rows, cols, t, rp, ci, v);
  }
}

template <class T>
T* host_copy(const std::vector<T>& x) {
  T* p = static_cast<T*>(std::malloc(sizeof(T) * std::max<size_t>(x.size(), 1)));
  if (!p) throw Fail(RKMF_INTERNAL_ERROR, "out of host memory");
  if (!x.empty()) std::memcpy(p, x.data(), sizeof(T) * x.size());
  return p;
}

void fmt17(char* buf, size_t cap, double x) { std::snprintf(buf, cap, "%.17g", x); }

}  // namespace

extern "C" {

void rkmf_host_free(void* p) { std::free(p); }

int rkmf_mtx_load(const char* path, int64_t* n_rows, int64_t* n_cols, int64_t* nnz,
                  int64_t** h_row_ptr, int32_t** h_col_idx, double** h_values, char* err,
                  int64_t err_cap) {
  try {
    std::vector<int64_t> rp;
    std::vector<int32_t> ci;
    std::vector<double> v;
    int64_t nr = 0, nc = 0;
    load_mtx(path, nr, nc, rp, ci, v);
    *n_rows = nr;
    *n_cols = nc;
    *nnz = int64_t(v.size());
    *h_row_ptr = host_copy(rp);
    *h_col_idx = host_copy(ci);
    *h_values = host_copy(v);
    return RKMF_OK;
  } catch (const Fail& f) {
    return report(f, err, err_cap);
  } catch (const std::exception& x) {
    return report(Fail(RKMF_INTERNAL_ERROR, x.what()), err, err_cap);
  }
}

int rkmf_mtx_save(const char* path, int64_t n_rows, int64_t n_cols, const int64_t* h_row_ptr,
                  const int32_t* h_col_idx, const double* h_values, char* err, int64_t err_cap) {
  try {
    FILE* fp = std::fopen(path, "wb");
    if (!fp) throw Fail(RKMF_INTERNAL_ERROR, std::string(path) + ": cannot open for writing");
    const int64_t nnz = n_rows > 0 ? h_row_ptr[n_rows] : 0;
    std::string out = "%%MatrixMarket matrix coordinate real general\n" + std::to_string(n_rows) +
                      " " + std::to_string(n_cols) + " " + std::to_string(nnz) + "\n";
    char num[64];
    bool ok = true;
    for (int64_t r = 0; r < n_rows && ok; ++r) {
      for (int64_t k = h_row_ptr[r]; k < h_row_ptr[r + 1]; ++k) {
        fmt17(num, sizeof(num), h_values[k]);
        out += std::to_string(r + 1);
        out += ' ';
        out += std::to_string(int64_t(h_col_idx[k]) + 1);
        out += ' ';
        out += num;
        out += '\n';
      }
      if (out.size() > (size_t(1) << 24)) {
        ok = std::fwrite(out.data(), 1, out.size(), fp) == out.size();
        out.clear();
      }
    }
    if (ok && !out.empty()) ok = std::fwrite(out.data(), 1, out.size(), fp) == out.size();
    if (std::fclose(fp) != 0) ok = false;
    if (!ok) throw Fail(RKMF_INTERNAL_ERROR, std::string(path) + ": write failure");
    return RKMF_OK;
  } catch (const Fail& f) {
    return report(f, err, err_cap);
  }
}

int rkmf_vector_load(const char* path, int64_t* n, double** h_out, char* err, int64_t err_cap) {
  try {
    const std::string p(path);
    const std::string buf = read_all(p);
    Lines L(buf);
    const char *b, *e;
    std::vector<double> vals;
    while (L.next(b, e)) {
      if (skip_line(b, e)) continue;
      const char* q = b;
      double x = 0.0;
      if (!get_double(q, e, x)) parse_fail(p, L.lineno, "expected one decimal value");
      if (!rest_blank(q, e)) parse_fail(p, L.lineno, "expected one value per line");
      vals.push_back(x);
    }
    *n = int64_t(vals.size());
    *h_out = host_copy(vals);
    return RKMF_OK;
  } catch (const Fail& f) {
    return report(f, err, err_cap);
  }
}

int rkmf_vector_save(const char* path, int64_t n, const double* h_v, char* err, int64_t err_cap) {
  try {
    FILE* fp = std::fopen(path, "wb");
    if (!fp) throw Fail(RKMF_INTERNAL_ERROR, std::string(path) + ": cannot open for writing");
    std::string out;
    char num[64];
    bool ok = true;
    for (int64_t i = 0; i < n && ok; ++i) {
      fmt17(num, sizeof(num), h_v[i]);
      out += num;
      out += '\n';
      if (out.size() > (size_t(1) << 24)) {
        ok = std::fwrite(out.data(), 1, out.size(), fp) == out.size();
        out.clear();
      }
    }
    if (ok && !out.empty()) ok = std::fwrite(out.data(), 1, out.size(), fp) == out.size();
    if (std::fclose(fp) != 0) ok = false;
    if (!ok) throw Fail(RKMF_INTERNAL_ERROR, std::string(path) + ": write failure");
    return RKMF_OK;
  } catch (const Fail& f) {
    return report(f, err, err_cap);
  }
}

}  // extern "C"
