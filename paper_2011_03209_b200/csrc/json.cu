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

#include <string>
#include <vector>

#include "common.cuh"

namespace bm {
namespace {

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
    int n = 0;
    uint64_t u = v < 0 ? (uint64_t)(-(v + 1)) + 1 : (uint64_t)v;
    do {
      t[23 - n++] = (char)('0' + u % 10);
      u /= 10;
    } while (u);
    if (v < 0) t[23 - n++] = '-';
    put(t + 24 - n, n);
  }
  // "%.9g" exactly as Python's '%.9g' % v (both correctly rounded; same
  // exponent rules), "-0" -> "0"
  bool put_num(double v) {
    if (!(v == v) || v == __builtin_inf() || v == -__builtin_inf()) return false;
    char t[40];
    const int n = snprintf(t, sizeof t, "%.9g", v);
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
  Out o{out, out ? cap : 0};
  o.put("[", 1);
  for (int64_t v = 0; v < n_nodes; ++v) {
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
      if (!o.put_num(h_fmean[v * m + a])) {
        set_error("non-finite value in graph JSON");
        return BM_ERR_DATA;
      }
    }
    o.put("],\"id\":");
    o.put_int(v);
    o.put(",\"rows\":[");
    for (int64_t e = h_node_off[v]; e < h_node_off[v + 1]; ++e) {
      if (e > h_node_off[v]) o.put(",", 1);
      o.put_int(h_node_rows[e]);
    }
    o.put("],\"size\":");
    o.put_int(h_node_off[v + 1] - h_node_off[v]);
    o.put(",\"stats\":{");
    for (int64_t i = 0; i < d; ++i) {
      if (i) o.put(",", 1);
      const int32_t c = h_stat_order[i];  // i-th key in sorted order -> column
      o.put(h_names + h_name_off[i], h_name_off[i + 1] - h_name_off[i]);  // quoted key
      o.put(":", 1);
      if (!o.put_num(h_stats[v * d + c])) {
        set_error("non-finite value in graph JSON");
        return BM_ERR_DATA;
      }
    }
    o.put("}}", 2);
  }
  o.put("]", 1);
  *h_len = o.len;
  if (out && o.len > cap) {
    set_error("output buffer too small (%lld < %lld)", (long long)cap, (long long)o.len);
    return BM_ERR_DATA;
  }
  return BM_OK;
}
