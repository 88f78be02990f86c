// LIBSVM text ingest (host code): the line loop of load_libsvm
// (pkg/src/syscd/dataset.py:169-233) as a two-pass, multi-threaded parser.
//
// The buffer is cut into n_threads byte ranges at line boundaries.  Pass 1
// (scan) tokenises and validates every line of a range and counts lines,
// examples and nonzeros; the lowest failing line number over all ranges is
// the one reported, which is the error the reference's sequential loop
// raises first.  Pass 2 (fill) re-counts per range (tokenising only), takes
// prefix sums and writes labels / example pointers / features / values in
// place, so the caller owns every array.
//
// Token grammar follows Python: float() for labels and values (optional sign,
// digits with single underscores between digits, optional fraction and
// exponent, or inf / infinity / nan in any case), int() base 10 for indices.
// Line terminators follow universal newlines (\n, \r, \r\n); whitespace is
// the ASCII set str.split() uses.
#include <cerrno>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"

namespace syscd {
namespace {

enum { kOk = 0, kBadLabel = 1, kBadEntry = 2, kNotOneBased = 3, kNotAscending = 4, kTooLarge = 5 };

inline bool is_ws(char c) {
  return c == ' ' || c == '\t' || c == '\v' || c == '\f' || (c >= 0x1c && c <= 0x1f);
}
inline bool is_nl(char c) { return c == '\n' || c == '\r'; }
inline bool is_digit(char c) { return c >= '0' && c <= '9'; }

// digits with single underscores strictly between digits; appends the digits
// to out and advances i.  Returns false if no digit was consumed or an
// underscore is misplaced.
bool digit_part(const char* s, int64_t n, int64_t& i, std::string& out) {
  if (i >= n || !is_digit(s[i])) return false;
  out.push_back(s[i++]);
  while (i < n) {
    if (is_digit(s[i])) {
      out.push_back(s[i++]);
    } else if (s[i] == '_' && i + 1 < n && is_digit(s[i + 1])) {
      ++i;
    } else {
      break;
    }
  }
  return true;
}

bool ieq(const char* s, int64_t n, const char* lit) {
  const int64_t m = (int64_t)strlen(lit);
  if (n != m) return false;
  for (int64_t k = 0; k < n; ++k) {
    char c = s[k];
    if (c >= 'A' && c <= 'Z') c = (char)(c - 'A' + 'a');
    if (c != lit[k]) return false;
  }
  return true;
}

// Python float(token)
bool parse_float(const char* s, int64_t n, double* out, std::string& tmp) {
  tmp.clear();
  int64_t i = 0;
  bool neg = false;
  if (i < n && (s[i] == '+' || s[i] == '-')) {
    neg = s[i] == '-';
    tmp.push_back(s[i]);
    ++i;
  }
  if (ieq(s + i, n - i, "inf") || ieq(s + i, n - i, "infinity")) {
    *out = neg ? -INFINITY : INFINITY;
    return true;
  }
  if (ieq(s + i, n - i, "nan")) {
    *out = NAN;
    return true;
  }
  bool mant = false;
  if (i < n && is_digit(s[i])) {
    if (!digit_part(s, n, i, tmp)) return false;
    mant = true;
  }
  if (i < n && s[i] == '.') {
    tmp.push_back('.');
    ++i;
    if (i < n && is_digit(s[i])) {
      if (!digit_part(s, n, i, tmp)) return false;
      mant = true;
    }
  }
  if (!mant) return false;
  if (i < n && (s[i] == 'e' || s[i] == 'E')) {
    tmp.push_back('e');
    ++i;
    if (i < n && (s[i] == '+' || s[i] == '-')) tmp.push_back(s[i++]);
    if (!digit_part(s, n, i, tmp)) return false;
  }
  if (i != n) return false;
  errno = 0;
  *out = strtod(tmp.c_str(), nullptr);  // correctly rounded, like Python
  return true;
}

// Python int(token) for base 10.  *big is set when |value| exceeds int64.
bool parse_int(const char* s, int64_t n, int64_t* out, bool* big, std::string& tmp) {
  tmp.clear();
  int64_t i = 0;
  bool neg = false;
  if (i < n && (s[i] == '+' || s[i] == '-')) neg = s[i++] == '-';
  if (!digit_part(s, n, i, tmp) || i != n) return false;
  *big = false;
  __int128 v = 0;
  for (char c : tmp) {
    v = v * 10 + (c - '0');
    if (v > (__int128)INT64_MAX) {
      *big = true;
      v = (__int128)INT64_MAX;
      break;
    }
  }
  *out = neg ? -(int64_t)v : (int64_t)v;
  return true;
}

struct Range {
  int64_t lo = 0, hi = 0;
  // pass-1 results
  int64_t lines = 0, examples = 0, nnz = 0, max_feat = 0;
  int32_t err = kOk;
  int64_t err_line = 0;  // local, 1-based
  int64_t tok_off = 0, tok_len = 0, err_index = 0;
};

// next line boundary at or after p (position just past a terminator), or len
int64_t align_to_line(const char* buf, int64_t len, int64_t p) {
  if (p <= 0) return 0;
  // p is a boundary if the previous byte ends a line (and does not split \r\n)
  while (p < len) {
    const char prev = buf[p - 1];
    if (prev == '\n') return p;
    if (prev == '\r' && buf[p] != '\n') return p;
    ++p;
  }
  return len;
}

std::vector<Range> split(const char* buf, int64_t len, int n_threads) {
  int T = n_threads > 0 ? n_threads : (int)std::thread::hardware_concurrency();
  if (T < 1) T = 1;
  if (len < (int64_t)T * 4096) T = (int)std::max<int64_t>(1, len / 4096);
  if (T < 1) T = 1;
  std::vector<Range> r(T);
  int64_t prev = 0;
  for (int t = 0; t < T; ++t) {
    r[t].lo = prev;
    r[t].hi = t == T - 1 ? len : align_to_line(buf, len, std::max(prev, len * (t + 1) / T));
    prev = r[t].hi;
  }
  return r;
}

// Walk the lines of one range.  emit(label, feats...) is called per example
// when Fill is set; validation only stops at the first error of the range.
template <bool Fill>
void walk(const char* buf, Range& R, double* labels, int64_t* ex_ptr, int32_t* feat,
          double* vals, int64_t ex0, int64_t nz0) {
  std::string tmp;
  int64_t p = R.lo, line = 0, ex = ex0, nz = nz0;
  while (p < R.hi) {
    int64_t e = p;
    while (e < R.hi && !is_nl(buf[e])) ++e;
    ++line;
    const int64_t next = (e < R.hi && buf[e] == '\r' && e + 1 < R.hi && buf[e + 1] == '\n')
                             ? e + 2
                             : e + 1;
    // tokens of [p, e)
    int64_t i = p;
    while (i < e && is_ws(buf[i])) ++i;
    if (i < e) {
      // label
      int64_t t0 = i;
      while (i < e && !is_ws(buf[i])) ++i;
      double label;
      if (!parse_float(buf + t0, i - t0, &label, tmp)) {
        if (!Fill) {
          R.err = kBadLabel;
          R.err_line = line;
          R.tok_off = t0;
          R.tok_len = i - t0;
          R.lines = line;
          return;
        }
      }
      if (Fill) {
        labels[ex] = label;
        ex_ptr[ex] = nz;
      }
      int64_t prev_idx = 0;
      while (true) {
        while (i < e && is_ws(buf[i])) ++i;
        if (i >= e) break;
        t0 = i;
        while (i < e && !is_ws(buf[i])) ++i;
        const char* tok = buf + t0;
        const int64_t tl = i - t0;
        int32_t code = kOk;
        int64_t idx = 0;
        double val = 0.0;
        const char* colon = (const char*)memchr(tok, ':', (size_t)tl);
        bool big = false;
        if (!colon || !parse_int(tok, colon - tok, &idx, &big, tmp) ||
            !parse_float(colon + 1, tok + tl - (colon + 1), &val, tmp)) {
          code = kBadEntry;
        } else if (idx < 1) {
          code = kNotOneBased;
        } else if (idx <= prev_idx) {
          code = kNotAscending;
        } else if (big || idx > (int64_t)INT32_MAX) {
          code = kTooLarge;
        }
        if (code != kOk) {
          if (!Fill) {
            R.err = code;
            R.err_line = line;
            R.tok_off = t0;
            R.tok_len = tl;
            R.err_index = idx;
            R.lines = line;
            return;
          }
          continue;
        }
        prev_idx = idx;
        if (Fill) {
          feat[nz] = (int32_t)(idx - 1);
          vals[nz] = val;
        }
        ++nz;
      }
      if (prev_idx > R.max_feat) R.max_feat = prev_idx;
      ++ex;
    }
    p = next;
  }
  R.lines = line;
  R.examples = ex - ex0;
  R.nnz = nz - nz0;
}

template <typename F>
void run_parallel(int T, F&& f) {
  if (T == 1) {
    f(0);
    return;
  }
  std::vector<std::thread> th;
  th.reserve(T);
  for (int t = 0; t < T; ++t) th.emplace_back(f, t);
  for (auto& x : th) x.join();
}

}  // namespace
}  // namespace syscd

using namespace syscd;

extern "C" int syscd_libsvm_scan(const char* buf, int64_t len, int32_t n_threads,
                                 syscd_libsvm_info* info) {
  if (!info || len < 0 || (len > 0 && !buf)) {
    set_error("syscd_libsvm_scan: invalid arguments");
    return SYSCD_EINVAL;
  }
  memset(info, 0, sizeof(*info));
  if (len == 0) return SYSCD_OK;
  std::vector<Range> R = split(buf, len, n_threads);
  const int T = (int)R.size();
  run_parallel(T, [&](int t) { walk<false>(buf, R[t], nullptr, nullptr, nullptr, nullptr, 0, 0); });
  int64_t line0 = 0;
  for (int t = 0; t < T; ++t) {
    if (R[t].err != kOk) {
      info->err = R[t].err;
      info->err_line = line0 + R[t].err_line;
      info->err_tok_off = R[t].tok_off;
      info->err_tok_len = R[t].tok_len;
      info->err_index = R[t].err_index;
      return SYSCD_OK;
    }
    line0 += R[t].lines;
    info->n_examples += R[t].examples;
    info->nnz += R[t].nnz;
    if (R[t].max_feat > info->max_feature) info->max_feature = R[t].max_feat;
  }
  return SYSCD_OK;
}

extern "C" int syscd_libsvm_fill(const char* buf, int64_t len, int32_t n_threads, double* labels,
                                 int64_t* ex_ptr, int32_t* feat_idx, double* vals) {
  if (len < 0 || (len > 0 && (!buf || !labels || !ex_ptr)) || !ex_ptr) {
    set_error("syscd_libsvm_fill: invalid arguments");
    return SYSCD_EINVAL;
  }
  if (len == 0) {
    ex_ptr[0] = 0;
    return SYSCD_OK;
  }
  std::vector<Range> R = split(buf, len, n_threads);
  const int T = (int)R.size();
  run_parallel(T, [&](int t) { walk<false>(buf, R[t], nullptr, nullptr, nullptr, nullptr, 0, 0); });
  std::vector<int64_t> ex0(T + 1, 0), nz0(T + 1, 0);
  for (int t = 0; t < T; ++t) {
    if (R[t].err != kOk) {
      set_error("syscd_libsvm_fill: buffer does not validate (call syscd_libsvm_scan first)");
      return SYSCD_EINVAL;
    }
    ex0[t + 1] = ex0[t] + R[t].examples;
    nz0[t + 1] = nz0[t] + R[t].nnz;
  }
  if (nz0[T] > 0 && (!feat_idx || !vals)) {
    set_error("syscd_libsvm_fill: invalid arguments");
    return SYSCD_EINVAL;
  }
  run_parallel(T, [&](int t) {
    Range r2;
    r2.lo = R[t].lo;
    r2.hi = R[t].hi;
    walk<true>(buf, r2, labels, ex_ptr, feat_idx, vals, ex0[t], nz0[t]);
  });
  ex_ptr[ex0[T]] = nz0[T];
  return SYSCD_OK;
}

extern "C" int syscd_csr_transpose(int64_t n_rows, int64_t n_cols, const int64_t* ptr,
                                   const int32_t* idx, const double* vals, int64_t* t_ptr,
                                   int32_t* t_idx, double* t_vals) {
  if (n_rows < 0 || n_cols < 0 || !ptr || !t_ptr ||
      (ptr[n_rows] > 0 && (!idx || !vals || !t_idx || !t_vals))) {
    set_error("syscd_csr_transpose: invalid arguments");
    return SYSCD_EINVAL;
  }
  const int64_t nnz = ptr[n_rows];
  std::vector<int64_t> cnt(n_cols + 1, 0);
  for (int64_t e = 0; e < nnz; ++e) {
    const int32_t c = idx[e];
    if (c < 0 || c >= n_cols) {
      set_error("syscd_csr_transpose: column index out of range");
      return SYSCD_EINVAL;
    }
    ++cnt[c + 1];
  }
  for (int64_t c = 0; c < n_cols; ++c) cnt[c + 1] += cnt[c];
  memcpy(t_ptr, cnt.data(), sizeof(int64_t) * (n_cols + 1));
  for (int64_t r = 0; r < n_rows; ++r) {
    for (int64_t e = ptr[r]; e < ptr[r + 1]; ++e) {
      const int64_t o = cnt[idx[e]]++;
      t_idx[o] = (int32_t)r;
      t_vals[o] = vals[e];
    }
  }
  return SYSCD_OK;
}
