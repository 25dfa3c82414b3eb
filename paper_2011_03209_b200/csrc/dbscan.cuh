// dbscan.cuh — shared layout of the per-element DBSCAN engine.
//
// Layout in HBM (one batch of elements):
//   entry e   = position of a membership entry in the batch (element-major,
//               ascending rows inside an element: the reference's order)
//   padded index p = pbase[k] + i: element k's rows in a SPATIALLY GROUPED
//               order (nearest-seed groups, stable), padded to kTile rows;
//               ent[p] = e (-1 for pads), inv[e] = p. Every order-dependent
//               rule of the reference (border -> smallest core neighbour,
//               clusters ordered by smallest member) is evaluated on e.
//   Xg   : P x d fp64   rows gathered in padded order (pads are zero)
//   tiles: the KEPT tile pairs (I <= J) of every element, sorted by (k, I, J):
//          pairs whose rigorous centroid/radius bound puts every row pair
//          beyond eps are pruned (they hold no bit). Slot s of the list owns
//          the 128x128 bit tile adj[s] (128 rows x 4 uint32 words, 2 KiB).
//   cnt  : int32 per p   eps-neighbour counts (self included)
//   core : uint8 per p
//   par  : int32 per p   union-find parent (root = min padded index)
//   bmin : int32 per p   smallest-ENTRY core neighbour of a non-core point
#pragma once
#include "common.cuh"

namespace bm {

constexpr int kTile = 128;
constexpr int kTileWords = kTile * kTile / 32;  // 512
constexpr int kNoCore = 0x7fffffff;

struct ElemTables {
  const int64_t* tp_off;  // n_el+1 dense tile-pair prefix (pruning flags)
  const int32_t* pbase;   // n_el+1 padded base
  const int32_t* nrows;   // n_el
  const int32_t* ntiles;  // n_el
  const uint8_t* order;   // n_el (BM_ORDER_*)
  const int32_t* ent;     // P: batch entry of padded row p (-1: pad)
  int64_t n_el;
};

// Where the coordinates of padded row p come from: the gathered copy Xg
// (xrow == nullptr: Xg + p * d) or the dataset X itself (X + xrow[p] * d,
// xrow[p] = rows[ent[p]], -1 for pads; valid p only). The tensor-core engine
// reads X directly (no gathered copy); the exact engine reads Xg.
struct RowSrc {
  const double* X;
  const int64_t* xrow;  // padded index -> dataset row (null: X is Xg)
  __device__ __forceinline__ int64_t index(int64_t p) const { return xrow ? xrow[p] : p; }
  __device__ __forceinline__ const double* row(int64_t p, int64_t d) const {
    return X + index(p) * d;
  }
};

// kept tile pair: element k, row tile I, column tile J (slot = list index)
struct TileRef {
  int32_t k, I, J, pad;
};

// row-tile work unit: element k, row tile I, slots [off, off + cnt) of the
// window's kept-tile list (all with row tile I, ascending J)
struct TileUnit {
  int32_t k, I, off, cnt;
};

__device__ __forceinline__ int64_t tri_index(int64_t I, int64_t J, int64_t T) {
  return I * T - I * (I - 1) / 2 + (J - I);
}

// Decode a global tile-pair index into (element, I, J).
__device__ __forceinline__ void decode_tile(const ElemTables& et, int64_t g, int& k, int& I,
                                            int& J) {
  int64_t a = 0, b = et.n_el;  // find last k with tp_off[k] <= g
  while (b - a > 1) {
    int64_t mid = (a + b) >> 1;
    if (et.tp_off[mid] <= g) a = mid; else b = mid;
  }
  k = (int)a;
  int64_t t = g - et.tp_off[k];
  int64_t T = et.ntiles[k];
  int64_t lo = 0, hi = T;  // last I with tri_index(I, I) <= t
  while (hi - lo > 1) {
    int64_t mid = (lo + hi) >> 1;
    if (tri_index(mid, mid, T) <= t) lo = mid; else hi = mid;
  }
  I = (int)lo;
  J = (int)(lo + (t - tri_index(lo, lo, T)));
}

__device__ __forceinline__ int uf_find(int* par, int x) {
  BM_DASSERT(x >= 0);
  while (true) {
    int p = __ldcg(par + x);
    if (p == x) return x;
    int gp = __ldcg(par + p);
    if (gp == p) return p;
    par[x] = gp;  // path halving; gp is an ancestor, the race is benign
    x = gp;
  }
}

__device__ __forceinline__ void uf_union(int* par, int a, int b) {
  while (true) {
    a = uf_find(par, a);
    b = uf_find(par, b);
    if (a == b) return;
    if (a > b) { int t = a; a = b; b = t; }
    int old = atomicCAS(par + b, b, a);  // hook the larger root under the smaller
    if (old == b) return;
    b = old;
  }
}

}  // namespace bm

namespace bm {

// Exact squared distance of one pair in the reference's fp64 order, reading
// both rows from global memory (one thread per pair). Sequential = scipy
// cdist; pairwise = numpy add.reduce over the squared difference row.
__device__ __forceinline__ double pw_leaf_diff2(const double* __restrict__ a,
                                                const double* __restrict__ b, int start,
                                                int len) {
  auto t = [&](int i) {
    double df = __dsub_rn(a[start + i], b[start + i]);
    return __dmul_rn(df, df);
  };
  if (len < 8) {
    double r = -0.0;
    for (int i = 0; i < len; ++i) r = __dadd_rn(r, t(i));
    return r;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = t(j);
  const int body = len - (len % 8);
  for (int i = 8; i < body; i += 8)
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], t(i + j));
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (int i = body; i < len; ++i) res = __dadd_rn(res, t(i));
  return res;
}

__device__ __forceinline__ double exact_dist2(const double* __restrict__ a,
                                              const double* __restrict__ b, int64_t d, int order,
                                              const PwProgram& prog) {
  if (order == BM_ORDER_SEQUENTIAL) {
    double s = 0.0;
    for (int64_t c = 0; c < d; ++c) {
      double df = __dsub_rn(a[c], b[c]);
      s = __dadd_rn(s, __dmul_rn(df, df));
    }
    return s;
  }
  PwStack st;
#pragma unroll
  for (int i = 0; i < kMaxStack; ++i) st.s[i] = 0.0;
  for (int li = 0; li < prog.n_leaves; ++li) {
    st.push(pw_leaf_diff2(a, b, prog.leaf[li].start, prog.leaf[li].len));
    for (int p = 0; p < prog.leaf[li].pops; ++p) st.reduce();
  }
  return __dadd_rn(0.0, st.s[0]);
}

}  // namespace bm
