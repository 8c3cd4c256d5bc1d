// Sparse Matrix Market ingestion: the reference's
// reader (proj/src/matrix_market.cpp:37-100, matrix_market.hpp:10-16) reads
// into a dense Eigen matrix; this one reads the same files into CSR, the
// operator format of the product.  Same accepted subset and diagnostics:
//   * `array` and `coordinate` formats, `general` or `symmetric` symmetry,
//     `real` or `integer` fields (integers read as reals);
//   * symmetric coordinate entries expand to (j, i) as well (off-diagonal),
//     symmetric arrays list the lower triangle column by column;
//   * duplicate coordinates are summed in file order from +0 (the
//     reference's `A(i-1, j-1) += value` on a zero matrix), so the CSR values
//     equal the reference's dense entries bit for bit;
//   * messages "matrix market: <path>: <what>" for the reference's failures.
// The CSR keeps the file's structural entries (every entry of an `array`
// file), columns ascending.  Numbers follow the reference's stream
// extraction (get_long / get_double below).
#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/phx.h"

namespace phx_mm {

struct Fail {
  std::string msg;
};

[[noreturn]] void fail(const std::string& path, const std::string& what) {
  throw Fail{"matrix market: " + path + ": " + what};
}

std::string lower(std::string s) {
  for (char& c : s) c = char(std::tolower(static_cast<unsigned char>(c)));
  return s;
}

// line cursor over the whole file (next_data_line of the reference:
// skips empty, '%' and blank lines; strips CR)
struct Lines {
  const char* p;
  const char* end;
  bool next(const char** b, const char** e) {
    while (p < end) {
      const char* s = p;
      const char* nl = static_cast<const char*>(std::memchr(p, '\n', size_t(end - p)));
      const char* t = nl ? nl : end;
      p = nl ? nl + 1 : end;
      const char* te = t;
      while (te > s && (te[-1] == '\r' || te[-1] == '\n')) --te;
      if (te == s || s[0] == '%') continue;
      bool blank = true;
      for (const char* q = s; q < te; ++q)
        if (*q != ' ' && *q != '\t') {
          blank = false;
          break;
        }
      if (blank) continue;
      *b = s;
      *e = te;
      return true;
    }
    return false;
  }
};

// The reference parses with `stream >> long` / `stream >> double` in the
// classic locale (libstdc++ num_get): skip whitespace, collect the longest
// prefix of the decimal grammar -- [sign] digits for integers;
// [sign] digits [. digits] [(e|E) [sign] digits] for reals, so no inf / nan /
// hex -- then convert with strtol / strtod, failing when the conversion does
// not consume the whole collected token or overflows (underflow is kept).
const char* skip_ws(const char* q, const char* e) {
  while (q < e && std::isspace(static_cast<unsigned char>(*q))) ++q;
  return q;
}
bool is_digit(char c) { return c >= '0' && c <= '9'; }

bool get_long(const char*& q, const char* e, long* out) {
  q = skip_ws(q, e);
  const char* s = q;
  if (q < e && (*q == '+' || *q == '-')) ++q;
  while (q < e && is_digit(*q)) ++q;
  const std::string tok(s, size_t(q - s));
  char* stop = nullptr;
  errno = 0;
  const long v = std::strtol(tok.c_str(), &stop, 10);
  if (tok.empty() || *stop != '\0' || errno == ERANGE) return false;
  *out = v;
  return true;
}

bool get_double(const char*& q, const char* e, double* out) {
  q = skip_ws(q, e);
  const char* s = q;
  if (q < e && (*q == '+' || *q == '-')) ++q;
  bool digits = false;
  while (q < e && is_digit(*q)) ++q, digits = true;
  if (q < e && *q == '.') {
    ++q;
    while (q < e && is_digit(*q)) ++q, digits = true;
  }
  if (digits && q < e && (*q == 'e' || *q == 'E')) {
    ++q;
    if (q < e && (*q == '+' || *q == '-')) ++q;
    while (q < e && is_digit(*q)) ++q;
  }
  const std::string tok(s, size_t(q - s));
  char* stop = nullptr;
  const double v = std::strtod(tok.c_str(), &stop);
  if (tok.empty() || *stop != '\0' || std::isinf(v)) return false;
  *out = v;
  return true;
}

struct Csr {
  int64_t n = 0;
  std::vector<int64_t> rp;
  std::vector<int32_t> ci;
  std::vector<double> av;
};

Csr read(const std::string& path) {
  FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) fail(path, "cannot open file");
  std::vector<char> buf;
  {
    char chunk[1 << 16];
    size_t got;
    while ((got = std::fread(chunk, 1, sizeof chunk, f)) > 0) buf.insert(buf.end(), chunk, chunk + got);
    std::fclose(f);
  }
  const char* p = buf.data();
  const char* end = p + buf.size();
  if (buf.empty()) fail(path, "empty file");
  // header line (the first physical line)
  const char* nl = static_cast<const char*>(std::memchr(p, '\n', buf.size()));
  std::string header(p, nl ? nl : end);
  while (!header.empty() && (header.back() == '\r' || header.back() == '\n')) header.pop_back();
  std::vector<std::string> tok;
  {
    size_t i = 0;
    while (i < header.size() && tok.size() < 5) {
      while (i < header.size() && std::isspace(static_cast<unsigned char>(header[i]))) ++i;
      size_t j = i;
      while (j < header.size() && !std::isspace(static_cast<unsigned char>(header[j]))) ++j;
      if (j > i) tok.emplace_back(header.substr(i, j - i));
      i = j;
    }
    while (tok.size() < 5) tok.emplace_back();
  }
  if (lower(tok[0]) != "%%matrixmarket" || lower(tok[1]) != "matrix")
    fail(path, "malformed header line");
  const std::string format = lower(tok[2]), field = lower(tok[3]), symmetry = lower(tok[4]);
  if (format != "array" && format != "coordinate") fail(path, "unsupported format '" + format + "'");
  if (field != "real" && field != "integer") fail(path, "non-real field '" + field + "'");
  if (symmetry != "general" && symmetry != "symmetric")
    fail(path, "unsupported symmetry '" + symmetry + "'");
  const bool symmetric = symmetry == "symmetric";

  Lines L{nl ? nl + 1 : end, end};
  const char *b, *e;
  if (!L.next(&b, &e)) fail(path, "missing size line");
  long rows = 0, cols = 0, nnz = 0;
  {
    const char* q = b;
    if (!get_long(q, e, &rows) || !get_long(q, e, &cols)) fail(path, "malformed size line");
    if (format == "coordinate" && !get_long(q, e, &nnz)) fail(path, "missing entry count");
  }
  if (rows <= 0 || cols <= 0) fail(path, "non-positive dimensions");
  if (rows != cols)
    fail(path, "matrix is " + std::to_string(rows) + "x" + std::to_string(cols) + ", expected square");
  if (rows >= (int64_t(1) << 31)) fail(path, "dimension exceeds the int32 column range");

  Csr out;
  out.n = rows;
  const int64_t n = rows;
  if (format == "array") {
    // column-major listing; symmetric files store the lower triangle
    if (double(n) * double(n) > 2.0e9) fail(path, "array file too large for a dense listing");
    std::vector<double> A(size_t(n) * size_t(n), 0.0);
    for (int64_t j = 0; j < n; ++j)
      for (int64_t i = symmetric ? j : 0; i < n; ++i) {
        if (!L.next(&b, &e)) fail(path, "truncated array data");
        const char* q = b;
        double v = 0.0;
        if (!get_double(q, e, &v)) fail(path, "malformed entry");
        A[size_t(i) + size_t(j) * size_t(n)] = v;
        if (symmetric) A[size_t(j) + size_t(i) * size_t(n)] = v;
      }
    out.rp.resize(size_t(n) + 1);
    out.ci.resize(size_t(n) * size_t(n));
    out.av.resize(size_t(n) * size_t(n));
    for (int64_t i = 0; i < n; ++i) {
      out.rp[size_t(i)] = i * n;
      for (int64_t j = 0; j < n; ++j) {
        out.ci[size_t(i * n + j)] = int32_t(j);
        out.av[size_t(i * n + j)] = A[size_t(i) + size_t(j) * size_t(n)];
      }
    }
    out.rp[size_t(n)] = n * n;
  } else {
    struct E {
      int32_t i, j;
      int64_t ord;  // file order, for summing duplicates in order
      double v;
    };
    std::vector<E> ent;
    if (nnz > 0) ent.reserve(size_t(std::min<long>(nnz, long(1) << 28)) * (symmetric ? 2 : 1));
    int64_t ord = 0;
    for (long k = 0; k < nnz; ++k) {
      if (!L.next(&b, &e)) fail(path, "truncated coordinate data");
      const char* q = b;
      long i = 0, j = 0;
      double v = 0.0;
      if (!get_long(q, e, &i) || !get_long(q, e, &j) || !get_double(q, e, &v))
        fail(path, "malformed entry");
      if (i < 1 || i > rows || j < 1 || j > cols) fail(path, "entry index out of range");
      ent.push_back(E{int32_t(i - 1), int32_t(j - 1), ord++, v});
      if (symmetric && i != j) ent.push_back(E{int32_t(j - 1), int32_t(i - 1), ord++, v});
    }
    std::sort(ent.begin(), ent.end(), [](const E& x, const E& y) {
      return x.i != y.i ? x.i < y.i : (x.j != y.j ? x.j < y.j : x.ord < y.ord);
    });
    out.rp.assign(size_t(n) + 1, 0);
    for (size_t k = 0; k < ent.size();) {
      size_t m = k;
      double acc = 0.0;  // A(i, j) += value on a zero matrix, in file order
      while (m < ent.size() && ent[m].i == ent[k].i && ent[m].j == ent[k].j) acc = acc + ent[m++].v;
      out.ci.push_back(ent[k].j);
      out.av.push_back(acc);
      out.rp[size_t(ent[k].i) + 1]++;
      k = m;
    }
    for (int64_t i = 0; i < n; ++i) out.rp[size_t(i) + 1] += out.rp[size_t(i)];
  }
  for (double v : out.av)
    if (!std::isfinite(v)) fail(path, "non-finite entries");
  return out;
}

}  // namespace phx_mm

namespace phx {
void set_last_error(const char* msg);  // the product's error channel (phx_host.cpp)
}

extern "C" {

phx_status phx_mm_read_csr(const char* path, int64_t* n, int64_t* nnz, int64_t* row_ptr,
                           int32_t* col_idx, double* vals, int64_t cap_nnz) {
  if (!path || !n || !nnz) {
    phx::set_last_error("matrix market: null argument");
    return PHX_EINVAL;
  }
  try {
    const phx_mm::Csr c = phx_mm::read(path);
    *n = c.n;
    *nnz = int64_t(c.ci.size());
    if (row_ptr && col_idx && vals && cap_nnz >= int64_t(c.ci.size())) {
      std::copy(c.rp.begin(), c.rp.end(), row_ptr);
      std::copy(c.ci.begin(), c.ci.end(), col_idx);
      std::copy(c.av.begin(), c.av.end(), vals);
    }
    return PHX_OK;
  } catch (const phx_mm::Fail& f) {
    phx::set_last_error(f.msg.c_str());
    return PHX_ENUMERIC;
  } catch (const std::bad_alloc&) {
    phx::set_last_error("host allocation failed");
    return PHX_ENOMEM;
  }
}

phx_status phx_mm_write_csr(const char* path, int64_t n, const int64_t* row_ptr,
                            const int32_t* col_idx, const double* vals) {
  if (!path || n < 1 || !row_ptr || !col_idx || !vals) {
    phx::set_last_error("matrix market: null argument");
    return PHX_EINVAL;
  }
  FILE* f = std::fopen(path, "wb");
  if (!f) {
    phx::set_last_error((std::string("matrix market: ") + path + ": cannot open file for writing").c_str());
    return PHX_ENUMERIC;
  }
  std::fprintf(f, "%%%%MatrixMarket matrix coordinate real general\n");
  std::fprintf(f, "%lld %lld %lld\n", (long long)n, (long long)n, (long long)row_ptr[n]);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e)
      std::fprintf(f, "%lld %lld %.17g\n", (long long)(i + 1), (long long)col_idx[e] + 1, vals[e]);
  const bool ok = std::ferror(f) == 0;
  std::fclose(f);
  if (!ok) {
    phx::set_last_error((std::string("matrix market: ") + path + ": write failed").c_str());
    return PHX_ENUMERIC;
  }
  return PHX_OK;
}

phx_status phx_op_create_mm(const char* path, int32_t device, phx_op* out) {
  if (!path || !out) {
    phx::set_last_error("matrix market: null argument");
    return PHX_EINVAL;
  }
  try {
    const phx_mm::Csr c = phx_mm::read(path);
    return phx_op_create_csr(c.n, c.rp.data(), c.ci.data(), c.av.data(), device, out);
  } catch (const phx_mm::Fail& f) {
    phx::set_last_error(f.msg.c_str());
    return PHX_ENUMERIC;
  } catch (const std::bad_alloc&) {
    phx::set_last_error("host allocation failed");
    return PHX_ENOMEM;
  }
}

}  // extern "C"
