// json.cu — canonical JSON of the Mapper graph's node array (host code).
//
// Reference: nervemap/nerve.py:119-188 (_write_canonical / _fmt_float): keys
// sorted, no whitespace, floats as "%.9g" with "-0" written as "0",
// non-finite floats rejected. The node objects are the bulk of the graph file
// (1.4M row ids and 55k floats at cfg3); the Python host keeps the small parts
// (manifest, edges, composition objects) and splices this array in. SURVEY §8f
// row 2 ("canonical JSON writer in C++").
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <mutex>
#include <string>
#include <charconv>
#include <thread>
#include <vector>

#include "common.cuh"

namespace bm {
namespace {

// two decimal digits per step
constexpr char kDigits2[] =
    "00010203040506070809101112131415161718192021222324252627282930313233343536373839"
    "40414243444546474849505152535455565758596061626364656667686970717273747576777879"
    "8081828384858687888990919293949596979899";

// decimal text of v at p (no bounds check; <= 20 bytes), returns the end
inline char* fmt_int(char* p, int64_t v) {
  uint64_t u = v < 0 ? (uint64_t)(-(v + 1)) + 1 : (uint64_t)v;
  if (v < 0) *p++ = '-';
  char t[20];
  int n = 20;
  while (u >= 100) {
    const unsigned r = (unsigned)(u % 100);
    u /= 100;
    n -= 2;
    t[n] = kDigits2[2 * r];
    t[n + 1] = kDigits2[2 * r + 1];
  }
  if (u >= 10) {
    n -= 2;
    t[n] = kDigits2[2 * u];
    t[n + 1] = kDigits2[2 * u + 1];
  } else {
    t[--n] = (char)('0' + u);
  }
  memcpy(p, t + n, 20 - n);
  return p + 20 - n;
}

struct Out {
  char* buf;
  int64_t cap, len = 0;
  void put(const char* s, int64_t n) {
    if (buf && len + n <= cap) memcpy(buf + len, s, n);
    len += n;
  }
  void put(const char* s) { put(s, (int64_t)strlen(s)); }
  void put_int(int64_t v) {
    char t[24];
    put(t, fmt_int(t, v) - t);
  }
  // comma-separated ints; unchecked fast path when the worst case fits
  void put_ints(const int64_t* a, int64_t n) {
    if (buf && len + 21 * n <= cap) {
      char* p = buf + len;
      for (int64_t i = 0; i < n; ++i) {
        if (i) *p++ = ',';
        p = fmt_int(p, a[i]);
      }
      len = p - buf;
      return;
    }
    for (int64_t i = 0; i < n; ++i) {
      if (i) put(",", 1);
      put_int(a[i]);
    }
  }
  // "%.9g" exactly as Python's '%.9g' % v (both correctly rounded; same
  // exponent rules), "-0" -> "0"
  bool put_num(double v) {
    if (!(v == v) || v == __builtin_inf() || v == -__builtin_inf()) return false;
    char t[40];
    // std::to_chars with a precision is specified as printf's "%.*g" in the
    // C locale (correctly rounded), ~4x faster than snprintf
    const int n = (int)(std::to_chars(t, t + sizeof t, v, std::chars_format::general, 9).ptr - t);
    if (n == 2 && t[0] == '-' && t[1] == '0') {
      put("0", 1);
    } else {
      put(t, n);
    }
    return true;
  }
};

}  // namespace
}  // namespace bm

using namespace bm;

namespace {

// nodes [v0, v1) into o; false on a non-finite value
bool write_nodes(Out& o, int64_t v0, int64_t v1, const int64_t* h_node_rows,
                 const int64_t* h_node_off, const int32_t* h_elem, const double* h_stats,
                 int64_t d, const int32_t* h_stat_order, const char* h_names,
                 const int64_t* h_name_off, const double* h_fmean, int32_t m, const char* h_comp,
                 const int64_t* h_comp_off) {
  for (int64_t v = v0; v < v1; ++v) {
    if (v) o.put(",", 1);
    // keys in sorted order: composition, element, filter_mean, id, rows, size, stats
    o.put("{\"composition\":");
    o.put(h_comp + h_comp_off[v], h_comp_off[v + 1] - h_comp_off[v]);
    o.put(",\"element\":");
    if (h_elem[2 * v + 1] < 0) {
      o.put_int(h_elem[2 * v]);
    } else {
      o.put("[", 1);
      o.put_int(h_elem[2 * v]);
      o.put(",", 1);
      o.put_int(h_elem[2 * v + 1]);
      o.put("]", 1);
    }
    o.put(",\"filter_mean\":[");
    for (int32_t a = 0; a < m; ++a) {
      if (a) o.put(",", 1);
      if (!o.put_num(h_fmean[v * m + a])) return false;
    }
    o.put("],\"id\":");
    o.put_int(v);
    o.put(",\"rows\":[");
    o.put_ints(h_node_rows + h_node_off[v], h_node_off[v + 1] - h_node_off[v]);
    o.put("],\"size\":");
    o.put_int(h_node_off[v + 1] - h_node_off[v]);
    o.put(",\"stats\":{");
    for (int64_t i = 0; i < d; ++i) {
      if (i) o.put(",", 1);
      const int32_t c = h_stat_order[i];  // i-th key in sorted order -> column
      o.put(h_names + h_name_off[i], h_name_off[i + 1] - h_name_off[i]);  // quoted key
      o.put(":", 1);
      if (!o.put_num(h_stats[v * d + c])) return false;
    }
    o.put("}}", 2);
  }
  return true;
}

}  // namespace

extern "C" int bm_json_nodes(int64_t n_nodes, const int64_t* h_node_rows,
                             const int64_t* h_node_off, const int32_t* h_elem,
                             const double* h_stats, int64_t d, const int32_t* h_stat_order,
                             const char* h_names, const int64_t* h_name_off,
                             const double* h_fmean, int32_t m, const char* h_comp,
                             const int64_t* h_comp_off, char* out, int64_t cap,
                             int64_t* h_len) {
  BM_REQUIRE(n_nodes >= 0 && d >= 0 && m >= 0, "bad sizes");
  BM_REQUIRE(h_len, "null output length");
  BM_REQUIRE(n_nodes == 0 || (h_node_rows && h_node_off && h_elem && h_comp && h_comp_off),
             "null node table");
  BM_REQUIRE(d == 0 || (h_stats && h_stat_order && h_names && h_name_off), "null stats table");
  BM_REQUIRE(m == 0 || h_fmean, "null filter means");
  // node ranges of balanced byte volume are written by host threads into
  // private buffers (kept across calls: no page faults on reuse), then copied
  // in order into out by the same threads. A sizing call (out == NULL) keeps
  // its formatted parts for this thread, and the next call with the same
  // arguments only copies them.
  struct Key {
    const void* p[10];
    int64_t n, d;
    int32_t m;
    bool operator==(const Key& o) const {
      return n == o.n && d == o.d && m == o.m && memcmp(p, o.p, sizeof p) == 0;
    }
  };
  const Key key{{h_node_rows, h_node_off, h_elem, h_stats, h_stat_order, h_names, h_name_off,
                 h_fmean, h_comp, h_comp_off},
                n_nodes, d, m};
  struct Cache {
    bool valid = false;
    Key key{};
    std::vector<std::vector<char>> parts;
    std::vector<int64_t> len;
  };
  thread_local Cache cache;
  static std::mutex pool_mu;
  static std::vector<std::vector<char>> pool;  // idle part buffers
  auto give_back = [&](std::vector<std::vector<char>>& parts) {
    std::lock_guard<std::mutex> lk(pool_mu);
    for (auto& p : parts)
      if (pool.size() < 64) pool.emplace_back(std::move(p));
    parts.clear();
  };
  const unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  auto run = [&](int nt, auto fn) {
    if (nt == 1) {
      fn(0);
      return;
    }
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t) th.emplace_back(fn, t);
    for (auto& x : th) x.join();
  };
  std::vector<std::vector<char>> parts;
  std::vector<int64_t> len;
  if (out && cache.valid && cache.key == key) {
    parts.swap(cache.parts);
    len.swap(cache.len);
    cache.valid = false;
  } else {
    if (cache.valid) {
      give_back(cache.parts);
      cache.valid = false;
    }
    // cost of node v ~ its row ids + kNumCost per formatted number (one
    // "%.9g" costs about as much as 30 row ids)
    constexpr int64_t kNumCost = 30;
    auto work = [&](int64_t v) { return h_node_off[v] + v * (d + m) * kNumCost; };
    const int64_t total = n_nodes ? work(n_nodes) : 0;
    const int nt = (int)std::min<int64_t>(hw, std::max<int64_t>(1, total / 32768));
    std::vector<int64_t> cut(nt + 1, n_nodes);
    cut[0] = 0;
    for (int t = 1, v = 0; t < nt; ++t) {
      while (v < n_nodes && work(v) < total * t / nt) ++v;
      cut[t] = v;
    }
    parts.resize(nt);
    {
      std::lock_guard<std::mutex> lk(pool_mu);
      for (int t = 0; t < nt && !pool.empty(); ++t) {
        parts[t].swap(pool.back());
        pool.pop_back();
      }
    }
    len.assign(nt, 0);
    std::vector<int> ok(nt, 1);
    run(nt, [&](int t) {
      const int64_t v0 = cut[t], v1 = std::max(cut[t], cut[t + 1]);
      const int64_t est =
          (h_node_off[v1] - h_node_off[v0]) * 8 + (v1 - v0) * (d + m + 8) * 18 + 64;
      if ((int64_t)parts[t].size() < est) parts[t].resize(est);
      for (;;) {
        Out o{parts[t].data(), (int64_t)parts[t].size()};
        ok[t] = write_nodes(o, v0, v1, h_node_rows, h_node_off, h_elem, h_stats, d,
                            h_stat_order, h_names, h_name_off, h_fmean, m, h_comp, h_comp_off);
        len[t] = o.len;
        if (o.len <= (int64_t)parts[t].size()) return;
        parts[t].resize(o.len);  // estimate too small: rewrite at the exact size
      }
    });
    for (int t = 0; t < nt; ++t)
      if (!ok[t]) {
        give_back(parts);
        set_error("non-finite value in graph JSON");
        return BM_ERR_DATA;
      }
  }
  const int nt = (int)parts.size();
  std::vector<int64_t> at(nt + 1, 1);  // "[" first
  for (int t = 0; t < nt; ++t) at[t + 1] = at[t] + len[t];
  *h_len = at[nt] + 1;  // "]"
  if (!out) {  // sizing call: keep the parts for the writing call
    cache.parts.swap(parts);
    cache.len.swap(len);
    cache.key = key;
    cache.valid = true;
    return BM_OK;
  }
  if (*h_len > cap) {
    give_back(parts);
    set_error("output buffer too small (%lld < %lld)", (long long)cap, (long long)*h_len);
    return BM_ERR_DATA;
  }
  out[0] = '[';
  run(nt, [&](int t) { memcpy(out + at[t], parts[t].data(), len[t]); });
  out[at[nt]] = ']';
  give_back(parts);
  return BM_OK;
}
