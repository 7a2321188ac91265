// Host-side matrix wire format of the reference (textio.py:70-119), multi-threaded:
//   "n\n" then n lines of n single-space separated fields, each a nonnegative integer or
//   the literal INF (INF_RAW in the int64 domain), '\n' terminated.
// The Python mirror (paper_2310_03983_b200/textio.py) keeps the reference's header and
// error handling; these two entry points do the O(n^2) field work.
#include <algorithm>
#include <atomic>
#include <charconv>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>
#include "../../include/apsp_b200.h"
#include "common.cuh"

namespace {

int workers(int64_t rows) {
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  return int(std::min<int64_t>(hw, std::max<int64_t>(1, rows / 64)));
}

template <typename F>
void parallel_rows(int64_t rows, F fn) {
  const int w = workers(rows);
  if (w <= 1) {
    fn(0, rows, 0);
    return;
  }
  std::vector<std::thread> th;
  const int64_t per = (rows + w - 1) / w;
  for (int t = 0; t < w; t++) {
    const int64_t a = t * per, b = std::min(rows, a + per);
    if (a >= b) break;
    th.emplace_back(fn, a, b, t);
  }
  for (auto& x : th) x.join();
}

inline int field_len(int64_t v) {
  if (v == apsp::INF_RAW) return 3;
  int len = 1;
  while (v >= 10) {
    v /= 10;
    len++;
  }
  return len;
}

}  // namespace

extern "C" {

int64_t apsp_format_matrix_i64(const int64_t* m, int64_t n, char* out, int64_t cap) {
  if (n < 1) return -1;
  // pass 1: bytes per row
  std::vector<int64_t> row_bytes(size_t(n) + 1, 0);
  std::atomic<bool> negative{false};
  parallel_rows(n, [&](int64_t a, int64_t b, int) {
    for (int64_t i = a; i < b; i++) {
      int64_t len = n;  // n - 1 separators + '\n'
      for (int64_t j = 0; j < n; j++) {
        const int64_t v = m[i * n + j];
        if (v < 0) negative.store(true, std::memory_order_relaxed);
        len += field_len(v);
      }
      row_bytes[size_t(i) + 1] = len;
    }
  });
  if (negative.load()) return -2;
  char head[32];
  const auto hr = std::to_chars(head, head + sizeof(head), n);
  const int64_t head_len = int64_t(hr.ptr - head) + 1;
  std::vector<int64_t> off(size_t(n) + 1, head_len);
  for (int64_t i = 0; i < n; i++) off[size_t(i) + 1] = off[size_t(i)] + row_bytes[size_t(i) + 1];
  const int64_t total = off[size_t(n)];
  if (!out || cap < total) return total;   // caller retries with this capacity
  std::memcpy(out, head, size_t(head_len - 1));
  out[head_len - 1] = '\n';
  parallel_rows(n, [&](int64_t a, int64_t b, int) {
    for (int64_t i = a; i < b; i++) {
      char* p = out + off[size_t(i)];
      for (int64_t j = 0; j < n; j++) {
        const int64_t v = m[i * n + j];
        if (v == apsp::INF_RAW) {
          std::memcpy(p, "INF", 3);
          p += 3;
        } else {
          p = std::to_chars(p, p + 20, v).ptr;
        }
        *p++ = (j + 1 < n) ? ' ' : '\n';
      }
    }
  });
  return total;
}

// Parses the n body lines (text starts after the header line).  Returns 0, or
// -(1 + row) for a row with the wrong field count / malformed field, or -(1 + n) for a wrong
// number of lines.  *bad_col receives the column of a malformed or negative field.
int64_t apsp_parse_matrix_i64(const char* text, int64_t len, int64_t n, int64_t* out, int64_t* bad_col) {
  if (n < 1) return -1;
  // line starts
  std::vector<int64_t> starts;
  starts.reserve(size_t(n) + 1);
  int64_t pos = 0;
  while (pos < len) {
    starts.push_back(pos);
    const void* nl = std::memchr(text + pos, '\n', size_t(len - pos));
    if (!nl) {
      pos = len + 1;   // last line without newline
      break;
    }
    pos = static_cast<const char*>(nl) - text + 1;
  }
  if (int64_t(starts.size()) != n) return -(1 + n);
  starts.push_back(pos > len ? len + 1 : len);
  std::vector<int64_t> err(size_t(workers(n)) + 1, 0), col(size_t(workers(n)) + 1, 0);
  parallel_rows(n, [&](int64_t a, int64_t b, int t) {
    for (int64_t i = a; i < b && !err[size_t(t)]; i++) {
      const char* p = text + starts[size_t(i)];
      const char* e = text + starts[size_t(i) + 1] - 1;   // excludes '\n'
      if (e > text + len) e = text + len;
      int64_t j = 0;
      while (true) {
        const char* f = p;
        while (p < e && *p != ' ') p++;
        if (j >= n) {
          err[size_t(t)] = -(1 + i);
          col[size_t(t)] = j;
          break;
        }
        if (p - f == 3 && std::memcmp(f, "INF", 3) == 0) {
          out[i * n + j] = apsp::INF_RAW;
        } else {
          int64_t v = 0;
          const char* g = (p - f > 1 && *f == '+') ? f + 1 : f;   // int() accepts a leading '+'
          const auto r = std::from_chars(g, p, v);
          if (r.ec != std::errc() || r.ptr != p || v < 0 || g == p) {
            err[size_t(t)] = -(1 + i);
            col[size_t(t)] = j;
            break;
          }
          out[i * n + j] = v;
        }
        j++;
        if (p >= e) break;
        p++;   // the separator
      }
      if (!err[size_t(t)] && j != n) {
        err[size_t(t)] = -(1 + i);
        col[size_t(t)] = j;
      }
    }
  });
  for (size_t t = 0; t < err.size(); t++)
    if (err[t]) {
      if (bad_col) *bad_col = col[t];
      return err[t];
    }
  return 0;
}

}  // extern "C"
