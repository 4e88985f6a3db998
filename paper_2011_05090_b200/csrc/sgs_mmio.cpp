// Matrix Market coordinate ingest (the reference's io.read_matrix_market,
// io.py:24-70), native: the whole file is read once and parsed in place with
// strtoll / strtod instead of a Python loop over lines (SiO2-sized inputs,
// millions of entries, parse in well under a second).  Same acceptance rules
// and messages as the reference: header "%%MatrixMarket matrix coordinate
// {real|integer|double} {general|symmetric}", '%' comment lines, a square size
// line, exactly three tokens per entry line, 1-based indices in bounds.
// Entries are returned 0-based and unsorted; the Python layer builds the CSR
// (duplicates summed, symmetric storage mirrored) as krylov.SparseMatrix.from_coo.

#include <cctype>
#include <cerrno>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/sketchgs_b200.h"

namespace sgs {
void set_error(const char* fmt, ...);
}

namespace {

struct MmFile {
  std::vector<char> buf;
  size_t pos = 0;
  bool next_line(const char*& b, const char*& e) {
    if (pos >= buf.size()) return false;
    b = buf.data() + pos;
    const char* nl = static_cast<const char*>(memchr(b, '\n', buf.size() - pos));
    e = nl ? nl : buf.data() + buf.size();
    pos = (size_t)(e - buf.data()) + (nl ? 1 : 0);
    if (e > b && e[-1] == '\r') --e;
    return true;
  }
};

bool load(const char* path, MmFile& f) {
  FILE* fh = fopen(path, "rb");
  if (!fh) {
    sgs::set_error("cannot open %s: %s", path, strerror(errno));
    return false;
  }
  fseek(fh, 0, SEEK_END);
  const long sz = ftell(fh);
  fseek(fh, 0, SEEK_SET);
  f.buf.resize(sz > 0 ? (size_t)sz : 0);
  const size_t got = sz > 0 ? fread(f.buf.data(), 1, (size_t)sz, fh) : 0;
  fclose(fh);
  if ((long)got != sz) {
    sgs::set_error("short read on %s", path);
    return false;
  }
  return true;
}

std::vector<std::string> split(const char* b, const char* e) {
  std::vector<std::string> out;
  while (b < e) {
    while (b < e && isspace((unsigned char)*b)) ++b;
    const char* s = b;
    while (b < e && !isspace((unsigned char)*b)) ++b;
    if (b > s) out.emplace_back(s, b);
  }
  return out;
}

std::string lower(std::string s) {
  for (auto& c : s) c = (char)tolower((unsigned char)c);
  return s;
}

bool parse_int(const std::string& t, int64_t& v) {
  char* end = nullptr;
  errno = 0;
  v = strtoll(t.c_str(), &end, 10);
  return errno == 0 && end && *end == '\0' && !t.empty();
}

// header + size line; leaves f.pos at the first entry line
int mm_header(MmFile& f, int64_t* nrows, int64_t* ncols, int64_t* nnz, int* symmetric) {
  const char *b, *e;
  if (!f.next_line(b, e)) {
    sgs::set_error("malformed Matrix Market header: ''");
    return SGS_EINVAL;
  }
  const std::string header(b, e);
  auto parts = split(b, e);
  if (parts.size() != 5 || parts[0] != "%%MatrixMarket" || lower(parts[1]) != "matrix") {
    sgs::set_error("malformed Matrix Market header: '%s'", header.c_str());
    return SGS_EINVAL;
  }
  const std::string fmt = lower(parts[2]), fld = lower(parts[3]), symm = lower(parts[4]);
  if (fmt != "coordinate") {
    sgs::set_error("unsupported format '%s' (coordinate only)", fmt.c_str());
    return SGS_EINVAL;
  }
  if (fld != "real" && fld != "integer" && fld != "double") {
    sgs::set_error("unsupported field '%s'", fld.c_str());
    return SGS_EINVAL;
  }
  if (symm != "general" && symm != "symmetric") {
    sgs::set_error("unsupported symmetry '%s'", symm.c_str());
    return SGS_EINVAL;
  }
  bool have = f.next_line(b, e);
  while (have) {
    const char* s = b;
    while (s < e && isspace((unsigned char)*s)) ++s;
    if (s < e && *s == '%') {
      have = f.next_line(b, e);
      continue;
    }
    break;
  }
  auto sizes = have ? split(b, e) : std::vector<std::string>{};
  int64_t r = 0, c = 0, z = 0;
  if (sizes.size() != 3 || !parse_int(sizes[0], r) || !parse_int(sizes[1], c) ||
      !parse_int(sizes[2], z) || z < 0) {
    sgs::set_error("malformed size line: '%s'", have ? std::string(b, e).c_str() : "");
    return SGS_EINVAL;
  }
  if (r != c) {
    sgs::set_error("matrix is %lldx%lld, expected square", (long long)r, (long long)c);
    return SGS_EINVAL;
  }
  *nrows = r;
  *ncols = c;
  *nnz = z;
  *symmetric = symm == "symmetric";
  return SGS_OK;
}

}  // namespace

extern "C" int sgs_mm_read_header(const char* path, int64_t* nrows, int64_t* ncols, int64_t* nnz,
                                  int* symmetric) {
  if (!path || !nrows || !ncols || !nnz || !symmetric) {
    sgs::set_error("mm_read_header: null argument");
    return SGS_EINVAL;
  }
  MmFile f;
  if (!load(path, f)) return SGS_EINVAL;
  return mm_header(f, nrows, ncols, nnz, symmetric);
}

extern "C" int sgs_mm_read_entries(const char* path, int64_t nnz, int64_t* rows, int64_t* cols,
                                   double* vals) {
  if (!path || (nnz > 0 && (!rows || !cols || !vals))) {
    sgs::set_error("mm_read_entries: null argument");
    return SGS_EINVAL;
  }
  MmFile f;
  if (!load(path, f)) return SGS_EINVAL;
  int64_t nr, nc, z;
  int sym;
  const int rc = mm_header(f, &nr, &nc, &z, &sym);
  if (rc != SGS_OK) return rc;
  if (z != nnz) {
    sgs::set_error("mm_read_entries: nnz %lld does not match the file (%lld)", (long long)nnz,
                   (long long)z);
    return SGS_EINVAL;
  }
  for (int64_t t = 0; t < nnz; ++t) {
    const char *b = nullptr, *e = nullptr;
    const bool have = f.next_line(b, e);
    // three whitespace-separated tokens: i j value
    const char* p = have ? b : nullptr;
    int ntok = 0;
    int64_t iv = 0, jv = 0;
    double v = 0.0;
    bool ok = have;
    while (ok && p < e) {
      while (p < e && isspace((unsigned char)*p)) ++p;
      if (p >= e) break;
      const char* s = p;
      while (p < e && !isspace((unsigned char)*p)) ++p;
      const std::string tok(s, p);
      char* end = nullptr;
      errno = 0;
      if (ntok == 0 || ntok == 1) {
        const long long x = strtoll(tok.c_str(), &end, 10);
        ok = errno == 0 && *end == '\0';
        (ntok == 0 ? iv : jv) = x;
      } else if (ntok == 2) {
        v = strtod(tok.c_str(), &end);
        ok = *end == '\0';
      }
      ++ntok;
    }
    if (!ok || ntok != 3) {
      sgs::set_error("malformed entry line %lld: '%s'", (long long)(t + 1),
                     have ? std::string(b, e).c_str() : "");
      return SGS_EINVAL;
    }
    if (!(1 <= iv && iv <= nr && 1 <= jv && jv <= nc)) {
      sgs::set_error("entry (%lld, %lld) out of bounds for %lldx%lld", (long long)iv,
                     (long long)jv, (long long)nr, (long long)nc);
      return SGS_EINVAL;
    }
    rows[t] = iv - 1;
    cols[t] = jv - 1;
    vals[t] = v;
  }
  return SGS_OK;
}
