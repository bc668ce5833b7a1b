// io.cpp — value files for the exact-sum path.
//
// Replaces exsum::parse_format / read_values / write_values (io.cpp:71-159,
// io.hpp:23-37) behind the C ABI:
//   bin   raw little-endian IEEE-754 doubles, 8 bytes each; a size that is not
//         a multiple of 8 is an error (io.cpp:96-99)
//   text  one value per line; only the first whitespace-separated token of a
//         line counts, blank lines are skipped (io.cpp:111-123); a token that
//         starts with 0x / 0X (and is longer than 2) is a hexadecimal bit
//         pattern that must fill the token (io.cpp:51-61), any other token must
//         parse completely with strtod (io.cpp:62-67).  Written as %.17g for
//         finite values and 0x%016llx for Inf/NaN (io.cpp:143-153).
// The reference throws std::runtime_error("<path>: <what>"); here the call
// returns EXSUM_EIO and exsum_io_error() returns the same message (per thread).
// The file sum itself (exsum_context_sum_file) lives in context.cu.

#include <errno.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <string>
#include <vector>

#include "exsum_b200.h"

namespace {

thread_local std::string g_error;

int fail(const char *path, const std::string &what) {
  g_error = std::string(path) + ": " + what;
  return EXSUM_EIO;
}

bool is_space(char c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\v' || c == '\f';
}

int hex_digit(char c) {
  if (c >= '0' && c <= '9') return c - '0';
  if (c >= 'a' && c <= 'f') return c - 'a' + 10;
  if (c >= 'A' && c <= 'F') return c - 'A' + 10;
  return -1;
}

// The first token of one line -> value; false on a parse error.
bool parse_token(const char *tok, size_t len, double *out) {
  if (len > 2 && tok[0] == '0' && (tok[1] == 'x' || tok[1] == 'X')) {
    uint64_t bits = 0;
    for (size_t i = 2; i < len; ++i) {
      const int d = hex_digit(tok[i]);
      if (d < 0 || bits >> 60) return false;  // not hex, or more than 64 bits
      bits = (bits << 4) | static_cast<uint64_t>(d);
    }
    memcpy(out, &bits, 8);
    return true;
  }
  const std::string t(tok, len);  // strtod needs a terminated string
  char *end = nullptr;
  const double v = strtod(t.c_str(), &end);
  if (end == t.c_str() || end != t.c_str() + t.size()) return false;
  *out = v;
  return true;
}

int read_text(const char *path, std::vector<double> &values) {
  FILE *f = fopen(path, "rb");
  if (!f) return fail(path, "cannot open");
  std::vector<char> buf;
  char chunk[1 << 16];
  size_t got;
  while ((got = fread(chunk, 1, sizeof chunk, f)) > 0) buf.insert(buf.end(), chunk, chunk + got);
  const bool bad = ferror(f) != 0;
  fclose(f);
  if (bad) return fail(path, "read error");
  size_t pos = 0, lineno = 0;
  const size_t n = buf.size();
  while (pos < n) {
    size_t eol = pos;
    while (eol < n && buf[eol] != '\n') ++eol;
    ++lineno;
    size_t b = pos;
    while (b < eol && is_space(buf[b])) ++b;
    if (b < eol) {
      size_t e = b;
      while (e < eol && !is_space(buf[e])) ++e;
      double v;
      if (!parse_token(buf.data() + b, e - b, &v)) {
        const bool hex = e - b > 2 && buf[b] == '0' && (buf[b + 1] == 'x' || buf[b + 1] == 'X');
        return fail(path, std::string(hex ? "bad bit pattern on line " : "bad value on line ") +
                              std::to_string(lineno));
      }
      values.push_back(v);
    }
    pos = eol + 1;
  }
  return EXSUM_OK;
}

int read_bin(const char *path, std::vector<double> &values) {
  FILE *f = fopen(path, "rb");
  if (!f) return fail(path, "cannot open");
  if (fseeko(f, 0, SEEK_END) != 0) {
    fclose(f);
    return fail(path, "read error");
  }
  const off_t size = ftello(f);
  fseeko(f, 0, SEEK_SET);
  if (size < 0) {
    fclose(f);
    return fail(path, "read error");
  }
  if (size % 8 != 0) {
    fclose(f);
    return fail(path, "size is not a multiple of 8 bytes");
  }
  values.resize(static_cast<size_t>(size) / 8);
  const size_t got = values.empty() ? 0 : fread(values.data(), 8, values.size(), f);
  fclose(f);
  if (got != values.size()) return fail(path, "short read");
  // files are little-endian; so is every host this library builds for
  return EXSUM_OK;
}

}  // namespace

extern "C" {

const char *exsum_io_error(void) { return g_error.c_str(); }

int exsum_parse_format(const char *name) {
  if (name && strcmp(name, "bin") == 0) return EXSUM_FORMAT_BIN;
  if (name && strcmp(name, "text") == 0) return EXSUM_FORMAT_TEXT;
  return -1;  // the reference throws std::invalid_argument (io.cpp:71-79)
}

int exsum_read_values(const char *path, int format, double **values, size_t *n) {
  if (!path || !values || !n || (format != EXSUM_FORMAT_BIN && format != EXSUM_FORMAT_TEXT))
    return EXSUM_EINVAL;
  *values = nullptr;
  *n = 0;
  std::vector<double> v;
  const int st = format == EXSUM_FORMAT_BIN ? read_bin(path, v) : read_text(path, v);
  if (st != EXSUM_OK) return st;
  double *out = static_cast<double *>(malloc(v.empty() ? 8 : v.size() * 8));
  if (!out) return EXSUM_ENOMEM;
  if (!v.empty()) memcpy(out, v.data(), v.size() * 8);
  *values = out;
  *n = v.size();
  return EXSUM_OK;
}

void exsum_free_values(double *values) { free(values); }

int exsum_write_values(const char *path, const double *values, size_t n, int format) {
  if (!path || (n && !values) || (format != EXSUM_FORMAT_BIN && format != EXSUM_FORMAT_TEXT))
    return EXSUM_EINVAL;
  FILE *f = fopen(path, "wb");
  if (!f) return fail(path, "cannot open for writing");
  bool ok = true;
  if (format == EXSUM_FORMAT_BIN) {
    ok = n == 0 || fwrite(values, 8, n, f) == n;
  } else {
    char buf[40];
    for (size_t i = 0; i < n && ok; ++i) {
      uint64_t bits;
      memcpy(&bits, &values[i], 8);
      const bool finite = ((bits >> 52) & 0x7FF) != 0x7FF;
      const int len = finite ? snprintf(buf, sizeof buf, "%.17g\n", values[i])
                             : snprintf(buf, sizeof buf, "0x%016llx\n",
                                        static_cast<unsigned long long>(bits));
      ok = fwrite(buf, 1, static_cast<size_t>(len), f) == static_cast<size_t>(len);
    }
  }
  ok = (fclose(f) == 0) && ok;
  return ok ? EXSUM_OK : fail(path, "write error");
}

}  // extern "C"
