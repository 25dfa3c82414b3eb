// dbscan.cu — K3..K6: per-element DBSCAN over cover elements.
//
// Reference: nervemap/clustering.py:151-198 (dbscan), 201-208 (order
// choice), 238-316 (cluster_all). Semantics reproduced exactly:
//   count(i) = #{j : dist(i,j) <= eps}, self included          (:166)
//   core     = count >= min_pts                                  (:167)
//   clusters = connected components of core points under eps    (:169-182)
//   border   = non-core with a core neighbour joins the cluster of its
//              smallest-index core neighbour                     (:184-190)
//   clusters ordered by smallest member (borders included)       (:192-197)
// dist(i,j) is the fp64 value the reference computes for that element:
// scipy cdist (sequential sum, no FMA) or numpy's pairwise row sum, then
// sqrt, compared with eps AFTER the sqrt.
//
// Pipeline per batch of elements (see dbscan.cuh for the HBM layout):
//   spatial grouping of each element's rows (nearest of 64 chained seeds,
//   stable sort) -> gather -> tile centres/radii -> pruning of tile pairs
//   that provably hold no eps pair -> device-built lists of kept tiles and
//   work units -> adjacency bitmap of the kept tiles (tcgen05 candidates +
//   exact recheck, tc_engine.cu; or the exact fp64 tile engine) -> counts ->
//   core -> union-find over core-core bits (diagonal tiles first, then
//   off-diagonal with empty/uniform-root tiles skipped) + border minima on
//   entry indices -> canonical relabel on entry indices.
#include <algorithm>
#include <vector>

#include "dbscan.cuh"

namespace bm {

bool tc_supported(int64_t d);
struct TcPrep;
int tc_prepare(const RowSrc src, int64_t d, const ElemTables& et, int64_t P, double eps,
               const std::vector<int32_t>& h_nrows, cudaStream_t stream, TcPrep** out,
               double* cen, double* rad, const double* tminmax);
void tc_release(TcPrep* tp);
int tc_window(TcPrep* tp, const RowSrc src, const ElemTables& et, const TileRef* tiles,
              int64_t slot0, int64_t n_tiles, const TileUnit* units, int64_t n_units,
              int64_t pairs, uint32_t* adj, int32_t* nonempty, int32_t* cnt, bool accumulate,
              bool sync_check, int64_t* stats, cudaStream_t stream);
void tc_set_queue_scale(TcPrep* tp, double s);
void tc_set_min_pts(TcPrep* tp, int32_t m);
int tc_collect(TcPrep* tp, int64_t* rechecked, bool* overflow, cudaStream_t stream);
int tc_tile_project(TcPrep* tp, const ElemTables& et, const int32_t* tseed,
                    const int8_t* seeds_q, const double* unorm, double* proj,
                    cudaStream_t stream);
int64_t tc_kpad(int64_t d);

namespace {


// ---------------------------------------------------------------------------
// gather: Xg[p] = X[rows[ent[p]]] (zero for pads). One warp per padded row.
// ---------------------------------------------------------------------------
__global__ void gather_kernel(const double* __restrict__ X, int64_t d,
                              const int64_t* __restrict__ rows,  // batch entries
                              ElemTables et, int64_t P, double* __restrict__ Xg) {
  const int lane = threadIdx.x & 31;
  const int64_t wpb = blockDim.x >> 5;
  for (int64_t p = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5); p < P;
       p += (int64_t)gridDim.x * wpb) {
    const int e = et.ent[p];
    double* dst = Xg + p * d;
    if (e >= 0) {
      const double* src = X + rows[e] * d;
      for (int64_t c = lane; c < d; c += 32) dst[c] = src[c];
    } else {
      for (int64_t c = lane; c < d; c += 32) dst[c] = 0.0;
    }
  }
}

// Per-tile column statistics the tensor-core engine needs (min, max, mean =
// the tile centre of the pruning bound), read from X through the membership;
// with Xg != null the rows are also gathered. One CTA per 128-row tile, one
// thread per column, rows in order.
__global__ void __launch_bounds__(256)
gather_tiles_kernel(const double* __restrict__ X, int64_t d, const int64_t* __restrict__ rows,
                    ElemTables et, double* __restrict__ Xg, double* __restrict__ tmin,
                    double* __restrict__ tmax, double* __restrict__ cen) {
  const int64_t tile = blockIdx.x;
  const int64_t p0 = tile * kTile;
  __shared__ int64_t src[kTile];
  __shared__ int nvalid;
  if (threadIdx.x == 0) nvalid = 0;
  __syncthreads();
  if (threadIdx.x < kTile) {
    const int e = et.ent[p0 + threadIdx.x];
    src[threadIdx.x] = e >= 0 ? rows[e] : -1;
    if (e >= 0) atomicAdd(&nvalid, 1);
  }
  __syncthreads();
  const int valid = nvalid;  // valid rows are the tile's first rows (pads at the end)
  for (int64_t c = threadIdx.x; c < d; c += blockDim.x) {
    double mn = __longlong_as_double(0x7ff0000000000000ll), mx = -mn, sm = 0.0;
#pragma unroll 8
    for (int r = 0; r < kTile; ++r) {
      double v = 0.0;
      if (r < valid) {
        v = X[src[r] * d + c];
        // the quantisation grid spans the FINITE values: a non-finite row
        // then only poisons its own tile's error bound (rechecked), not the
        // element's scale
        if (isfinite(v)) {
          mn = fmin(mn, v);
          mx = fmax(mx, v);
        }
        sm += v;
      }
      if (Xg) Xg[(p0 + r) * d + c] = v;
    }
    tmin[tile * d + c] = mn;
    tmax[tile * d + c] = mx;
    cen[tile * d + c] = sm / (double)valid;
  }
}

// The same statistics without the gather (the tensor-core engine reading X
// directly; d even): 2 columns per thread (16-byte loads), 8 rows in flight.
__device__ __forceinline__ void stat_acc(double v, double& mn, double& mx, double& sm) {
  if (isfinite(v)) {  // finite grid: see gather_tiles_kernel
    mn = fmin(mn, v);
    mx = fmax(mx, v);
  }
  sm += v;
}

#ifndef BM_STAT_ROWS
#define BM_STAT_ROWS 4
#endif
constexpr int kStatRows = BM_STAT_ROWS;  // row loads in flight per thread

__global__ void __launch_bounds__(128)
tile_stats_kernel(const double* __restrict__ X, int64_t d, const int64_t* __restrict__ xrow,
                  double* __restrict__ tmin, double* __restrict__ tmax,
                  double* __restrict__ cen) {
  const int64_t tile = blockIdx.x;
  const int64_t p0 = tile * kTile;
  __shared__ int64_t src[kTile];
  const int64_t xr = xrow[p0 + threadIdx.x];  // blockDim.x == kTile
  src[threadIdx.x] = xr;
  const int valid = __syncthreads_count(xr >= 0);  // pads at the tile's end
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  for (int64_t c = 2 * threadIdx.x; c < d; c += 2 * blockDim.x) {
    double mn0 = inf, mx0 = -inf, sm0 = 0.0, mn1 = inf, mx1 = -inf, sm1 = 0.0;
    int r = 0;
    for (; r + kStatRows <= valid; r += kStatRows) {
      double2 v[kStatRows];
#pragma unroll
      for (int u = 0; u < kStatRows; ++u)
        v[u] = __ldg(reinterpret_cast<const double2*>(X + src[r + u] * d + c));
#pragma unroll
      for (int u = 0; u < kStatRows; ++u) {
        stat_acc(v[u].x, mn0, mx0, sm0);
        stat_acc(v[u].y, mn1, mx1, sm1);
      }
    }
    for (; r < valid; ++r) {
      const double2 v = __ldg(reinterpret_cast<const double2*>(X + src[r] * d + c));
      stat_acc(v.x, mn0, mx0, sm0);
      stat_acc(v.y, mn1, mx1, sm1);
    }
    *reinterpret_cast<double2*>(tmin + tile * d + c) = make_double2(mn0, mn1);
    *reinterpret_cast<double2*>(tmax + tile * d + c) = make_double2(mx0, mx1);
    *reinterpret_cast<double2*>(cen + tile * d + c) =
        make_double2(sm0 / (double)valid, sm1 / (double)valid);
  }
}

// ---------------------------------------------------------------------------
// Spatial grouping inside an element (performance only — any order gives the
// same result, the order-dependent rules run on entry indices). Each entry
// picks the nearest of S evenly spaced seed entries of its element over the
// first kGroupDims dims (fp32); a stable sort by (element, seed) makes row
// tiles compact, so tile pairs of far-apart groups can be pruned.
// ---------------------------------------------------------------------------
constexpr int kGroupSeeds = 64;
static_assert(kGroupSeeds == 64, "seed_order / tile_project / prune kernels are written for 64 seeds");
constexpr int kGroupDims = 32;
constexpr int kGroupMinRows = 3 * kTile;  // smaller elements keep their order
constexpr int kSeedTab = kGroupSeeds * (kGroupDims + 1);  // floats per element seed table
#ifndef BM_GROUP_TC
#define BM_GROUP_TC 1
#endif
constexpr bool kGroupTc = BM_GROUP_TC;  // seed assignment on the tensor cores (mma.sync tf32)

struct GroupItem {
  int32_t k, e0, e1, pad;  // element, entries [e0, e1) (batch-relative)
};

// Seed order per grouped element: a greedy nearest-neighbour chain from
// seed 0 over the seeds' first kGroupDims dims, so that consecutive groups
// (and the tiles straddling their boundaries) are spatially close. One CTA
// per element; rank[k * kGroupSeeds + s] = position of seed s in the chain.
__global__ void __launch_bounds__(256)
seed_order_kernel(const double* __restrict__ X, int64_t d, const int64_t* __restrict__ rows,
                  const int64_t* __restrict__ offs, const int32_t* __restrict__ elems,
                  int32_t* __restrict__ rank, int32_t* __restrict__ order,
                  float* __restrict__ seed_tab) {
  __shared__ float sd[kGroupSeeds][kGroupDims + 1];
  __shared__ float dist[kGroupSeeds][kGroupSeeds + 1];
  __shared__ int used[kGroupSeeds];
  const int k = elems[blockIdx.x];
  const int64_t ek = offs[k], nk = offs[k + 1] - ek;
  const int S = nk < kGroupSeeds ? (int)nk : kGroupSeeds;
  const int D = d < kGroupDims ? (int)d : kGroupDims;
  for (int i = threadIdx.x; i < kGroupSeeds * kGroupDims; i += blockDim.x) {
    const int j = i / kGroupDims, dim = i % kGroupDims;
    sd[j][dim] = (j < S && dim < D) ? (float)X[rows[ek + (j * nk) / S] * d + dim] : 0.0f;
  }
  if (threadIdx.x < kGroupSeeds) used[threadIdx.x] = threadIdx.x >= S;
  __syncthreads();
  {
    // the element's seed table for group_assign: 64 x kGroupDims coordinates
    // then the 64 squared norms (one contiguous block per element)
    float* tab = seed_tab + (int64_t)k * kSeedTab;
    for (int i = threadIdx.x; i < kGroupSeeds * kGroupDims; i += blockDim.x)
      tab[i] = sd[i / kGroupDims][i % kGroupDims];
    if (threadIdx.x < kGroupSeeds) {
      float q = 0.0f;
      for (int c = 0; c < kGroupDims; ++c) q = fmaf(sd[threadIdx.x][c], sd[threadIdx.x][c], q);
      tab[kGroupSeeds * kGroupDims + threadIdx.x] = q;
    }
  }
  for (int i = threadIdx.x; i < kGroupSeeds * kGroupSeeds; i += blockDim.x) {
    const int a = i / kGroupSeeds, b = i % kGroupSeeds;
    float acc = 0.0f;
    for (int dim = 0; dim < D; ++dim) {
      const float df = sd[a][dim] - sd[b][dim];
      acc = fmaf(df, df, acc);
    }
    dist[a][b] = acc;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    int cur = 0;
    if (lane == 0) {
      rank[(int64_t)k * kGroupSeeds] = 0;
      for (int r = 0; r < kGroupSeeds; ++r) order[(int64_t)k * kGroupSeeds + r] = r ? -1 : 0;
      used[0] = 1;
    }
    __syncwarp();
    for (int step = 1; step < S; ++step) {
      float best = 3.0e38f;
      int bi = kGroupSeeds;
      for (int c = lane; c < kGroupSeeds; c += 32)
        if (!used[c] && (dist[cur][c] < best || (dist[cur][c] == best && c < bi))) {
          best = dist[cur][c];
          bi = c;
        }
      for (int o = 16; o; o >>= 1) {
        const float ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob < best || (ob == best && oi < bi)) {
          best = ob;
          bi = oi;
        }
      }
      cur = bi;
      if (lane == 0) {
        rank[(int64_t)k * kGroupSeeds + cur] = step;
        order[(int64_t)k * kGroupSeeds + step] = cur;
        used[cur] = 1;
      }
      __syncwarp();
    }
  }
}

// One thread per entry: its first kGroupDims coordinates in registers
// (fp32), the 64 seeds broadcast from shared memory, 4 dims per 16-byte
// load; nearest seed by |s|^2 - 2 <x, s> (one FMA per dim; smallest index on
// ties) -> key (element, seed rank). The grouping only orders rows for the
// pruning; any assignment gives the same clusters.
__global__ void __launch_bounds__(128, 6)
group_assign_kernel(const double* __restrict__ X, int64_t d, const int64_t* __restrict__ rows,
                    const int64_t* __restrict__ offs, const GroupItem* __restrict__ items,
                    const int32_t* __restrict__ seed_rank, const float* __restrict__ seed_tab,
                    uint64_t* __restrict__ keys, int64_t* __restrict__ vals) {
  __shared__ __align__(16) float sd[kGroupSeeds][kGroupDims];  // seed coordinates
  __shared__ float sn[kGroupSeeds];                              // |s|^2
  const GroupItem it = items[blockIdx.x];
  const int64_t ek = offs[it.k], nk = offs[it.k + 1] - ek;
  const int S = nk < kGroupSeeds ? (int)nk : kGroupSeeds;
  const int D = d < kGroupDims ? (int)d : kGroupDims;
  {  // the element's seed table (seed_order_kernel), coalesced
    const float4* tab = reinterpret_cast<const float4*>(seed_tab + (int64_t)it.k * kSeedTab);
    for (int i = threadIdx.x; i < kSeedTab / 4; i += blockDim.x) {
      const float4 v = tab[i];
      if (i < kGroupSeeds * kGroupDims / 4)
        reinterpret_cast<float4*>(&sd[0][0])[i] = v;
      else
        reinterpret_cast<float4*>(sn)[i - kGroupSeeds * kGroupDims / 4] = v;
    }
  }
  __syncthreads();
  for (int e = it.e0 + threadIdx.x; e < it.e1; e += blockDim.x) {
    const double* xr = X + rows[e] * d;
    float x[kGroupDims];
#pragma unroll
    for (int c = 0; c < kGroupDims; ++c) x[c] = c < D ? -2.0f * (float)xr[c] : 0.0f;
    float best = 3.0e38f;
    int bi = 0;
    for (int j = 0; j < S; ++j) {
      float acc = sn[j];
#pragma unroll
      for (int c = 0; c < kGroupDims; c += 4) {
        const float4 sv = *reinterpret_cast<const float4*>(&sd[j][c]);
        acc = fmaf(x[c], sv.x, acc);
        acc = fmaf(x[c + 1], sv.y, acc);
        acc = fmaf(x[c + 2], sv.z, acc);
        acc = fmaf(x[c + 3], sv.w, acc);
      }
      if (acc < best) {
        best = acc;
        bi = j;
      }
    }
    keys[e] = ((uint64_t)it.k << 7) | (uint64_t)seed_rank[(int64_t)it.k * kGroupSeeds + bi];
    vals[e] = e;
  }
}

// Tensor-core variant (mma.sync tf32, m16n8k8): a warp takes 16 entries, the
// scores |s|^2 - 2 <x, s> of all 64 seeds come from 4 k-steps x 8 seed tiles
// of MMAs, and each row's argmin (smallest seed index on ties) is reduced
// across its quad. The entries' first kGroupDims coordinates are read
// coalesced (lane = dim) and transposed through shared memory.
__device__ __forceinline__ uint32_t to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

constexpr int kGaWarps = 4;

__global__ void __launch_bounds__(kGaWarps * 32)
group_assign_tc_kernel(const double* __restrict__ X, int64_t d, const int64_t* __restrict__ rows,
                       const int64_t* __restrict__ offs, const GroupItem* __restrict__ items,
                       const int32_t* __restrict__ seed_rank, const float* __restrict__ seed_tab,
                       uint64_t* __restrict__ keys, int64_t* __restrict__ vals) {
  __shared__ uint32_t sb[kGroupSeeds][kGroupDims + 4];    // seeds (tf32), padded
  __shared__ float sn[kGroupSeeds];                       // |s|^2
  __shared__ uint32_t sa[kGaWarps][16][kGroupDims + 4];   // per warp: 16 entries (tf32)
  const GroupItem it = items[blockIdx.x];
  const int64_t nk = offs[it.k + 1] - offs[it.k];
  const int S = nk < kGroupSeeds ? (int)nk : kGroupSeeds;
  const int D = d < kGroupDims ? (int)d : kGroupDims;
  {
    const float* tab = seed_tab + (int64_t)it.k * kSeedTab;
    for (int i = threadIdx.x; i < kGroupSeeds * kGroupDims; i += blockDim.x)
      sb[i / kGroupDims][i % kGroupDims] = to_tf32(tab[i]);
    for (int i = threadIdx.x; i < kGroupSeeds; i += blockDim.x)
      sn[i] = i < S ? tab[kGroupSeeds * kGroupDims + i] : 3.0e38f;  // absent seeds never win
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  uint32_t(*A)[kGroupDims + 4] = sa[wid];
  for (int64_t e0 = it.e0 + wid * 16; e0 < it.e1; e0 += kGaWarps * 16) {
    // 16 entries x kGroupDims dims, coalesced along the dims
#pragma unroll 4
    for (int i = 0; i < 16; ++i) {
      const int64_t e = e0 + i;
      float v = 0.0f;
      if (e < it.e1 && lane < D) v = (float)X[rows[e] * d + lane];
      A[i][lane] = to_tf32(v);
    }
    __syncwarp();
    float acc[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.0f;
#pragma unroll
    for (int kk = 0; kk < kGroupDims / 8; ++kk) {
      const uint32_t a0 = A[g][kk * 8 + t], a1 = A[g + 8][kk * 8 + t];
      const uint32_t a2 = A[g][kk * 8 + t + 4], a3 = A[g + 8][kk * 8 + t + 4];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t b0 = sb[j * 8 + g][kk * 8 + t], b1 = sb[j * 8 + g][kk * 8 + t + 4];
        asm volatile(
            "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
            "{%8,%9}, {%0,%1,%2,%3};"
            : "+f"(acc[j][0]), "+f"(acc[j][1]), "+f"(acc[j][2]), "+f"(acc[j][3])
            : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
      }
    }
    __syncwarp();
    // rows g (acc[.][0..1]) and g + 8 (acc[.][2..3]); seed n = 8 j + 2 t + {0, 1}
    float best0 = 3.4e38f, best1 = 3.4e38f;
    int bi0 = kGroupSeeds, bi1 = kGroupSeeds;
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int n = j * 8 + 2 * t + h;
        const float s0 = fmaf(-2.0f, acc[j][h], sn[n]);
        const float s1 = fmaf(-2.0f, acc[j][2 + h], sn[n]);
        if (s0 < best0) { best0 = s0; bi0 = n; }  // n ascending per lane: first min kept
        if (s1 < best1) { best1 = s1; bi1 = n; }
      }
#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {
      const float ob0 = __shfl_xor_sync(0xffffffffu, best0, o);
      const int oi0 = __shfl_xor_sync(0xffffffffu, bi0, o);
      const float ob1 = __shfl_xor_sync(0xffffffffu, best1, o);
      const int oi1 = __shfl_xor_sync(0xffffffffu, bi1, o);
      if (ob0 < best0 || (ob0 == best0 && oi0 < bi0)) { best0 = ob0; bi0 = oi0; }
      if (ob1 < best1 || (ob1 == best1 && oi1 < bi1)) { best1 = ob1; bi1 = oi1; }
    }
    if (t == 0) {
      const int64_t ea = e0 + g, eb = e0 + g + 8;
      const int32_t* rk = seed_rank + (int64_t)it.k * kGroupSeeds;
      if (ea < it.e1) {
        keys[ea] = ((uint64_t)it.k << 7) | (uint64_t)rk[bi0 < S ? bi0 : 0];
        vals[ea] = ea;
      }
      if (eb < it.e1) {
        keys[eb] = ((uint64_t)it.k << 7) | (uint64_t)rk[bi1 < S ? bi1 : 0];
        vals[eb] = eb;
      }
    }
  }
}

// identity order (key = element) for the entries of elements with fewer than
// min_rows rows
__global__ void group_identity_kernel(const int64_t* __restrict__ offs, int64_t n_el,
                                      int64_t n_entries, int64_t min_rows,
                                      uint64_t* __restrict__ keys, int64_t* __restrict__ vals) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n_entries;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = 0, b = n_el;
    while (b - a > 1) {
      const int64_t mid = (a + b) >> 1;
      if (offs[mid] <= e) a = mid; else b = mid;
    }
    if (offs[a + 1] - offs[a] < min_rows) {
      keys[e] = (uint64_t)a << 7;
      vals[e] = e;
    }
  }
}

// sorted entries -> ent (per padded row) and inv (per entry)
__global__ void perm_kernel(const int64_t* __restrict__ sorted, const int64_t* __restrict__ offs,
                            ElemTables et, int64_t P, int32_t* __restrict__ ent,
                            int32_t* __restrict__ inv, const int64_t* __restrict__ rows,
                            int64_t* __restrict__ xrow) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P;
       p += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = 0, b = et.n_el;
    while (b - a > 1) {
      const int64_t mid = (a + b) >> 1;
      if (et.pbase[mid] <= p) a = mid; else b = mid;
    }
    const int64_t i = p - et.pbase[a];
    if (i < et.nrows[a]) {
      const int e = (int)sorted[offs[a] + i];
      ent[p] = e;
      inv[e] = (int32_t)p;
      if (xrow) xrow[p] = rows[e];
    } else {
      ent[p] = -1;
      if (xrow) xrow[p] = -1;
    }
  }
}

// ---------------------------------------------------------------------------
// Direction bound (second pruning test). Every grouped element keeps its 64
// seed points s_g (full d, fp64). Row tile T is labelled with the seed a of
// its middle row; for every seed g the kernel below stores
//   proj_T[g] <= min_{x in T} <x, s_a - s_g>
// (fp32 dot products, minus a rigorous bound of their rounding). For tiles I
// (seed a) and J (seed b != a), u = s_a - s_b gives for all x in I, y in J
//   |x - y| >= <x - y, u>/|u| = (<x,u> + <y,-u>)/|u| >= (proj_I[b] + proj_J[a]) / |u|,
// which prunes most tile pairs of different seed groups that the centre/radius
// bound cannot (the groups are far apart along u, wide across it).
// ---------------------------------------------------------------------------
// per row tile: its seed (-1: element not grouped)
__global__ void tile_seed_kernel(ElemTables et, const int64_t* __restrict__ offs, int64_t n_rt,
                                 const uint64_t* __restrict__ skeys,
                                 const int32_t* __restrict__ order, int64_t min_rows,
                                 int32_t* __restrict__ tseed) {
  for (int64_t rt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; rt < n_rt;
       rt += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p0 = rt * kTile;
    int64_t a = 0, b = et.n_el;
    while (b - a > 1) {
      const int64_t mid = (a + b) >> 1;
      if (et.pbase[mid] <= p0) a = mid; else b = mid;
    }
    const int k = (int)a;
    int seed = -1;
    if (et.nrows[k] >= min_rows) {
      const int64_t i0 = p0 - et.pbase[k];
      const int64_t valid = min((int64_t)kTile, (int64_t)et.nrows[k] - i0);
      const uint64_t key = skeys[offs[k] + i0 + valid / 2];
      seed = order[(int64_t)k * kGroupSeeds + (int)(key & 127)];
    }
    tseed[rt] = seed;
  }
}

// per (grouped element, seed a) (one CTA): fp32 copy and fp64 norm of seed a,
// fp64 distances from seed a to every seed (one warp per seed b)
__global__ void __launch_bounds__(256)
seed_data_kernel(const double* __restrict__ X, int64_t d, const int64_t* __restrict__ rows,
                 const int64_t* __restrict__ offs, const int32_t* __restrict__ elems,
                 float* __restrict__ sf, double* __restrict__ snorm,
                 double* __restrict__ sdist) {
  const int k = elems[blockIdx.x / kGroupSeeds];
  const int ga = blockIdx.x % kGroupSeeds;
  const int64_t ek = offs[k], nk = offs[k + 1] - ek;
  const int S = nk < kGroupSeeds ? (int)nk : kGroupSeeds;
  float* sfa = sf + ((int64_t)k * kGroupSeeds + ga) * d;
  const double* xa = ga < S ? X + rows[ek + (ga * nk) / S] * d : nullptr;
  for (int64_t c = threadIdx.x; c < d; c += blockDim.x) sfa[c] = xa ? (float)xa[c] : 0.0f;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int gb = w; gb < kGroupSeeds; gb += blockDim.x >> 5) {
    double acc = 0.0, na = 0.0;
    if (xa && gb < S) {
      const double* xb = X + rows[ek + (gb * nk) / S] * d;
      for (int64_t c = lane; c < d; c += 32) {
        const double df = xa[c] - xb[c];
        acc = fma(df, df, acc);
        if (gb == 0) na = fma(xa[c], xa[c], na);
      }
    }
    for (int o = 16; o; o >>= 1) {
      acc += __shfl_xor_sync(0xffffffffu, acc, o);
      na += __shfl_xor_sync(0xffffffffu, na, o);
    }
    if (lane == 0) {
      sdist[((int64_t)k * kGroupSeeds + ga) * kGroupSeeds + gb] = sqrt(acc);
      if (gb == 0) snorm[(int64_t)k * kGroupSeeds + ga] = sqrt(na);
    }
  }
}

// int8 seeds of the tensor-core direction bound (tc_engine.cu
// tile_project_i8_kernel): per grouped element (one CTA),
//   s'_g = clamp(rint((s_g - m) / sigma), +-127),  m = mean of the seeds,
//   sigma = max_{g,c} |s_g,c - m_c| / 127,
// zero-padded to kpad bytes, and |s'_a - s'_b| (exact integer sum of squares,
// square root rounded up). Any integer direction gives a valid bound; this
// one follows the seed differences to ~1% in 256 dimensions.
__global__ void __launch_bounds__(256)
seed_quant_kernel(const double* __restrict__ X, int64_t d, const int64_t* __restrict__ rows,
                  const int64_t* __restrict__ offs, const int32_t* __restrict__ elems,
                  int64_t kpad, int8_t* __restrict__ seeds_q, double* __restrict__ unorm) {
  const int k = elems[blockIdx.x];
  const int64_t ek = offs[k], nk = offs[k + 1] - ek;
  const int S = nk < kGroupSeeds ? (int)nk : kGroupSeeds;
  __shared__ int64_t srow[kGroupSeeds];
  __shared__ double smean[256];
  __shared__ double sdev[8];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  if (t < kGroupSeeds) srow[t] = t < S ? rows[ek + (t * nk) / S] : -1;
  __syncthreads();
  double dev = 0.0;
  for (int64_t c = t; c < d; c += blockDim.x) {
    double m = 0.0;
    for (int g = 0; g < S; ++g) m += X[srow[g] * d + c];
    m /= (double)S;
    smean[c] = m;
    for (int g = 0; g < S; ++g) dev = fmax(dev, fabs(X[srow[g] * d + c] - m));
  }
  for (int o = 16; o; o >>= 1) dev = fmax(dev, __shfl_xor_sync(0xffffffffu, dev, o));
  if (lane == 0) sdev[w] = dev;
  __syncthreads();
  double dmax = 0.0;
  for (int i = 0; i < 8; ++i) dmax = fmax(dmax, sdev[i]);
  const double sigma = (dmax > 0.0 && dmax < 1e300) ? dmax / 127.0 : 1.0;
  int8_t* sq = seeds_q + (int64_t)k * kGroupSeeds * kpad;
  constexpr int kSS = 256 + 4;  // smem row (bytes): 65 words, conflict-free columns
  __shared__ __align__(16) int8_t ssq[kGroupSeeds * kSS];
  for (int64_t i = t; i < (int64_t)kGroupSeeds * kpad; i += blockDim.x) {
    const int g = (int)(i / kpad);
    const int64_t c = i % kpad;
    double v = 0.0;
    if (g < S && c < d) v = fmin(fmax(rint((X[srow[g] * d + c] - smean[c]) / sigma), -127.0), 127.0);
    const int8_t q = (int8_t)(v == v ? (int)v : 0);
    sq[i] = q;
    ssq[g * kSS + c] = q;
  }
  __syncthreads();
  // |s'_a - s'_b|^2 = |a|^2 + |b|^2 - 2 a.b, exact in int32 (dp4a over words)
  for (int pr = t; pr < kGroupSeeds * kGroupSeeds; pr += blockDim.x) {
    const int ga = pr / kGroupSeeds, gb = pr % kGroupSeeds;
    int dot = 0, na = 0, nb = 0;
    for (int64_t c = 0; c < kpad; c += 4) {
      const int wa = *reinterpret_cast<const int*>(ssq + ga * kSS + c);
      const int wb = *reinterpret_cast<const int*>(ssq + gb * kSS + c);
      dot = __dp4a(wa, wb, dot);
      na = __dp4a(wa, wa, na);
      nb = __dp4a(wb, wb, nb);
    }
    unorm[((int64_t)k * kGroupSeeds + ga) * kGroupSeeds + gb] = __dsqrt_ru((double)(na + nb - 2 * dot));
  }
}

constexpr int kProjKC = 16;  // dims staged per step (register-prefetched)

// one CTA per grouped row tile: D[x][g] = <x, s_g> for its 128 rows and the 64
// seeds (fp32, 4 x 8 per thread), then proj[rt][g] = min_x (D[x][a] - D[x][g])
// minus the rounding bound (d + 4) 2^-23 (|c_T| + r_T)(|s_a| + |s_g|)
__global__ void __launch_bounds__(256, 3)
tile_project_kernel(const double* __restrict__ Xg, int64_t d, ElemTables et, int64_t n_rt,
                    const int32_t* __restrict__ tseed, const float* __restrict__ sf,
                    const double* __restrict__ snorm, const double* __restrict__ cen,
                    const double* __restrict__ rad, double* __restrict__ proj) {
  // staging (xs, ss) during the dot products; the dot matrix dd afterwards
  constexpr int kStage = kProjKC * (kTile + 4) + kProjKC * (kGroupSeeds + 4);
  constexpr int kDot = kTile * (kGroupSeeds + 1);
  __shared__ __align__(16) float sbuf[kStage > kDot ? kStage : kDot];
  float(*xs)[kTile + 4] = reinterpret_cast<float(*)[kTile + 4]>(sbuf);
  float(*ss)[kGroupSeeds + 4] =
      reinterpret_cast<float(*)[kGroupSeeds + 4]>(sbuf + kProjKC * (kTile + 4));
  float(*dd)[kGroupSeeds + 1] = reinterpret_cast<float(*)[kGroupSeeds + 1]>(sbuf);
  __shared__ double cn;
  const int64_t rt = blockIdx.x;
  const int a = tseed[rt];
  if (a < 0) return;  // block-uniform
  const int64_t p0 = rt * kTile;
  int64_t lo = 0, hi = et.n_el;
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (et.pbase[mid] <= p0) lo = mid; else hi = mid;
  }
  const int k = (int)lo;
  const int valid = min(kTile, (int)(et.nrows[k] - (p0 - et.pbase[k])));
  const float* sfk = sf + (int64_t)k * kGroupSeeds * d;
  // points 4ty.., seeds 8tx..; a warp covers 8 point groups x 4 seed groups,
  // so its shared-memory operand loads touch 8 + 4 distinct 16-byte vectors
  // (no bank conflicts; 3 wavefronts per k step)
  const int t = threadIdx.x, lane = t & 31, wp = t >> 5;
  const int ty = (lane & 7) + 8 * (wp & 3), tx = (lane >> 3) + 4 * (wp >> 2);
  float acc[4][8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.0f;
  // each thread stages 8 row values and 4 seed values per step; the next
  // step's values are loaded into registers while the current one computes
  constexpr int kXv = kTile * kProjKC / 256, kSv = kGroupSeeds * kProjKC / 256;
  double xr[kXv];
  float sr[kSv];
  auto fetch = [&](int64_t c0) {
#pragma unroll
    for (int u = 0; u < kXv; ++u) {
      const int i = t + u * 256, pnt = i / kProjKC, c = i % kProjKC;
      xr[u] = (c0 + c < d && pnt < valid) ? Xg[(p0 + pnt) * d + c0 + c] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kSv; ++u) {
      const int i = t + u * 256, g = i / kProjKC, c = i % kProjKC;
      sr[u] = c0 + c < d ? sfk[(int64_t)g * d + c0 + c] : 0.0f;
    }
  };
  auto stage = [&]() {
    bool all_ok = true;
    float xf[kXv];
#pragma unroll
    for (int u = 0; u < kXv; ++u) {
      bool ok;
      xf[u] = f64_to_f32_rz(xr[u], &ok);
      all_ok &= ok;
    }
    if (!__all_sync(0xffffffffu, all_ok)) {  // rare: outside the fp32 normal range
#pragma unroll
      for (int u = 0; u < kXv; ++u) xf[u] = (float)xr[u];
    }
#pragma unroll
    for (int u = 0; u < kXv; ++u) {
      const int i = t + u * 256;
      xs[i % kProjKC][i / kProjKC] = xf[u];
    }
#pragma unroll
    for (int u = 0; u < kSv; ++u) {
      const int i = t + u * 256;
      ss[i % kProjKC][i / kProjKC] = sr[u];
    }
  };
  fetch(0);
  for (int64_t c0 = 0; c0 < d; c0 += kProjKC) {
    __syncthreads();
    stage();
    __syncthreads();
    if (c0 + kProjKC < d) fetch(c0 + kProjKC);
#pragma unroll
    for (int c = 0; c < kProjKC; ++c) {
      const float4 xa = *reinterpret_cast<const float4*>(&xs[c][4 * ty]);
      const float4 s0 = *reinterpret_cast<const float4*>(&ss[c][8 * tx]);
      const float4 s1 = *reinterpret_cast<const float4*>(&ss[c][8 * tx + 4]);
      const float xv[4] = {xa.x, xa.y, xa.z, xa.w};
      const float sv[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(xv[i], sv[j], acc[i][j]);
    }
  }
  __syncthreads();  // staging buffers are reused for dd
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) dd[4 * ty + i][8 * tx + j] = acc[i][j];
  if (t < 32) {  // |c_T| (fp64)
    double q = 0.0;
    for (int64_t c = t; c < d; c += 32) q = fma(cen[rt * d + c], cen[rt * d + c], q);
    for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
    if (t == 0) cn = sqrt(q);
  }
  __syncthreads();
  if (t < kGroupSeeds) {
    float m = 3.0e38f;
    for (int pnt = 0; pnt < valid; ++pnt) m = fminf(m, dd[pnt][a] - dd[pnt][t]);
    // |fl(<x,s>) - <x,s>| <= (d+2) 2^-24 |x||s| for the fp32 inputs and FMA
    // chain; x is rounded toward zero (2^-23) and s to nearest (2^-24), and
    // the difference of two dots is rounded once more: (d+6) 2^-24 in all,
    // below the (2d+8) 2^-24 used
    const double xmax = (cn + rad[rt]) * (1.0 + 1e-12);
    const double err = ((double)d + 4.0) * 1.1920928955078125e-07 * xmax *
                       (snorm[(int64_t)k * kGroupSeeds + a] + snorm[(int64_t)k * kGroupSeeds + t]) *
                       (1.0 + 1e-9);
    const double v = (double)m - err;
    proj[rt * kGroupSeeds + t] = (m == m && rad[rt] == rad[rt]) ? v : -1.0e300;
  }
}

// ---------------------------------------------------------------------------
// Tile geometry and pruning. Per 128-row tile: a centre c (the fp64 mean of
// its rows — any point works) and a radius r >= max |x - c| (fp64 norm plus
// a relative margin far above its rounding error). For I != J, every pair of
// rows is at true distance >= |c_I - c_J| - r_I - r_J, and the reference's
// fp64 distance is within a factor (1 +- gamma) of the true one, so
//   (|c_I - c_J| (1 - 1e-12) - r_I - r_J) (1 - gamma) > eps
// proves that no pair of the tile pair is an eps-neighbour. NaN/inf rows make
// the bound NaN and keep the tile pair.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
tile_geom_kernel(const double* __restrict__ Xg, int64_t d, ElemTables et,
                 const int32_t* __restrict__ tile_elem, double* __restrict__ cen,
                 double* __restrict__ rad) {
  const int64_t t = blockIdx.x;
  const int k = tile_elem[t];
  const int64_t p0 = t * kTile;
  const int valid = min(kTile, (int)(et.nrows[k] - (p0 - et.pbase[k])));
  double* c = cen + t * d;
  for (int64_t j = threadIdx.x; j < d; j += blockDim.x) {
    double s = 0.0;
    for (int r = 0; r < valid; ++r) s += Xg[(p0 + r) * d + j];
    c[j] = s / (double)valid;
  }
  __syncthreads();
  __shared__ double wmax[8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double m = 0.0;
  bool nan = false;
  for (int r = w; r < valid; r += 8) {
    double s = 0.0;
    for (int64_t j = lane; j < d; j += 32) {
      const double df = Xg[(p0 + r) * d + j] - c[j];
      s += df * df;
    }
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (s == s) m = fmax(m, sqrt(s));
    else nan = true;  // NaN poisons the radius (keeps every tile pair)
  }
  if (lane == 0) wmax[w] = nan ? __longlong_as_double(0x7ff8000000000000ll) : m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double mm = 0.0;
    bool any_nan = false;
    for (int i = 0; i < 8; ++i) {
      if (wmax[i] == wmax[i]) mm = fmax(mm, wmax[i]);
      else any_nan = true;
    }
    rad[t] = any_nan ? __longlong_as_double(0x7ff8000000000000ll) : mm;
  }
}

constexpr int kPruneB = 64;   // 64 x 64 tile pairs per CTA (4 x 4 per thread)
constexpr int kPruneDC = 32;  // centre dims staged per step

struct PruneBlock {
  int32_t k, bi, bj, pad;
};

// flags[g] = 1 if dense tile pair g of the batch must be computed
#ifndef BM_PRUNE_MINB
#define BM_PRUNE_MINB 3
#endif
__global__ void __launch_bounds__(256, BM_PRUNE_MINB)
tile_prune_kernel(ElemTables et, int64_t d, const int32_t* __restrict__ tbase,
                  const PruneBlock* __restrict__ blocks, const double* __restrict__ cen,
                  const double* __restrict__ rad, double eps, double gamma,
                  const int32_t* __restrict__ tseed, const double* __restrict__ proj,
                  const double* __restrict__ sdist, int32_t* __restrict__ flags) {
  __shared__ double sa[kPruneDC][kPruneB + 1], sb[kPruneDC][kPruneB + 1];
  const PruneBlock pbk = blocks[blockIdx.x];
  const int k = pbk.k, T = et.ntiles[k];
  const int64_t tb = tbase[k];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int i0 = pbk.bi * kPruneB, j0 = pbk.bj * kPruneB;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  for (int64_t c0 = 0; c0 < d; c0 += kPruneDC) {
    const int dc = (d - c0) < kPruneDC ? (int)(d - c0) : kPruneDC;
    __syncthreads();
    for (int i = threadIdx.x; i < kPruneB * kPruneDC; i += blockDim.x) {
      const int t = i / kPruneDC, c = i % kPruneDC;
      const bool okc = c < dc;
      sa[c][t] = (okc && i0 + t < T) ? cen[(tb + i0 + t) * d + c0 + c] : 0.0;
      sb[c][t] = (okc && j0 + t < T) ? cen[(tb + j0 + t) * d + c0 + c] : 0.0;
    }
    __syncthreads();
    for (int c = 0; c < dc; ++c) {
      double av[4], bv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = sa[c][ty + 16 * a];
#pragma unroll
      for (int b = 0; b < 4; ++b) bv[b] = sb[c][tx + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const double df = av[a] - bv[b];
          acc[a][b] = fma(df, df, acc[a][b]);
        }
    }
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int I = i0 + ty + 16 * a, J = j0 + tx + 16 * b;
      if (I >= T || J >= T || J < I) continue;
      int keep = 1;
      if (I != J) {
        // radii: raw fp64 maxima of |x - c|, inflated far above their rounding error
        const double rsum = (rad[tb + I] + rad[tb + J]) * (1.0 + 1e-12) + 1e-300;
        const double lb = (sqrt(acc[a][b]) * (1.0 - 1e-12) - rsum) * (1.0 - gamma);
        keep = lb > eps ? 0 : 1;
        if (keep && tseed) {  // direction bound between the tiles' seed groups
          const int sa = tseed[tb + I], sb = tseed[tb + J];
          if (sa >= 0 && sb >= 0 && sa != sb) {
            const double u = sdist[((int64_t)k * kGroupSeeds + sa) * kGroupSeeds + sb];
            const double num =
                __dadd_rd(proj[(tb + I) * kGroupSeeds + sb], proj[(tb + J) * kGroupSeeds + sa]);
            if (u > 0.0 && num > 0.0 && (num / (u * (1.0 + 1e-12))) * (1.0 - gamma) > eps) keep = 0;
          }
        }
      }
      flags[et.tp_off[k] + tri_index(I, J, T)] = keep;
    }
}

__global__ void fill_ones_kernel(int32_t* __restrict__ f, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    f[i] = 1;
}

// Per row tile rt = tbase[k] + I (one warp): its kept tiles into the list at
// pos[g] (ascending J), the row's first slot and the distinct row pairs of
// its kept tiles.
__global__ void emit_tiles_kernel(ElemTables et, const int32_t* __restrict__ row_elem,
                                  const int32_t* __restrict__ tbase, int64_t n_rt,
                                  const int32_t* __restrict__ flags,
                                  const int64_t* __restrict__ pos, TileRef* __restrict__ tiles,
                                  int64_t* __restrict__ row_first, int64_t* __restrict__ row_pairs) {
  const int lane = threadIdx.x & 31;
  const int64_t wpb = blockDim.x >> 5;
  for (int64_t rt = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5); rt < n_rt;
       rt += (int64_t)gridDim.x * wpb) {
    const int k = row_elem[rt];
    const int I = (int)(rt - tbase[k]);
    const int T = et.ntiles[k], nk = et.nrows[k];
    const int64_t g0 = et.tp_off[k] + tri_index(I, I, T);
    const int64_t vI = min(kTile, nk - I * kTile);
    int64_t pr = 0;
    for (int J = I + lane; J < T; J += 32) {
      const int64_t g = g0 + (J - I);
      if (flags[g]) {
        tiles[pos[g]] = TileRef{k, I, J, 0};
        const int64_t vJ = min(kTile, nk - J * kTile);
        pr += J == I ? vI * (vI - 1) / 2 : vI * vJ;
      }
    }
    for (int o = 16; o; o >>= 1) pr += __shfl_xor_sync(0xffffffffu, pr, o);
    if (lane == 0) {
      row_first[rt] = pos[g0];
      row_pairs[rt] = pr;
    }
  }
}

// tensor-core work units hold up to kTcUnit column tiles (the row tile's A
// operand is loaded once per unit)
#ifndef BM_TC_UNIT
#define BM_TC_UNIT 16
#endif
constexpr int kTcUnit = BM_TC_UNIT;

// unit counts per row tile (from the kept slots of consecutive rows)
__global__ void unit_counts_kernel(const int64_t* __restrict__ row_first, int64_t n_rt,
                                   int64_t* __restrict__ n_off, int64_t* __restrict__ n_tc) {
  for (int64_t rt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; rt < n_rt;
       rt += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = row_first[rt + 1] - row_first[rt];
    n_off[rt] = (c - 1 + 31) / 32;
    n_tc[rt] = (c + kTcUnit - 1) / kTcUnit;
  }
}

// units of every row tile: diagonal unit rt; off-diagonal units at
// off_pos[rt] (slots after the diagonal); tensor-core units at tc_pos[rt]
__global__ void emit_units_kernel(const int32_t* __restrict__ row_elem,
                                  const int32_t* __restrict__ tbase, int64_t n_rt,
                                  const int64_t* __restrict__ row_first,
                                  const int64_t* __restrict__ off_pos,
                                  const int64_t* __restrict__ tc_pos, TileUnit* __restrict__ diag,
                                  TileUnit* __restrict__ off, TileUnit* __restrict__ tcu) {
  for (int64_t rt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; rt < n_rt;
       rt += (int64_t)gridDim.x * blockDim.x) {
    const int k = row_elem[rt];
    const int I = (int)(rt - tbase[k]);
    const int64_t f = row_first[rt];
    const int c = (int)(row_first[rt + 1] - f);
    diag[rt] = TileUnit{k, I, (int32_t)f, 1};
    int64_t o = off_pos[rt];
    for (int j = 1; j < c; j += 32) off[o++] = TileUnit{k, I, (int32_t)(f + j), min(32, c - j)};
    o = tc_pos[rt];
    for (int j = 0; j < c; j += kTcUnit)
      tcu[o++] = TileUnit{k, I, (int32_t)(f + j), min(kTcUnit, c - j)};
  }
}

// ---------------------------------------------------------------------------
// Exact fp64 tile engine: every pair of a 128x128 tile in the reference's
// exact order. 256 threads, 4x4 pairs per thread per 64x64 quadrant; the
// rows of the current leaf (<=128 dims) are staged transposed in smem.
// ---------------------------------------------------------------------------
constexpr int kQ = 64;
constexpr int kKC = 128;
constexpr int kLd = kQ + 1;  // padded leading dimension (doubles)
constexpr size_t kExactSmem = 2 * kKC * kLd * sizeof(double);

struct Frag {
  double v[16];
};

__device__ __forceinline__ void frag_zero(Frag& f, double z) {
#pragma unroll
  for (int i = 0; i < 16; ++i) f.v[i] = z;
}

// f += (a - b)^2 for dim index `c` of the staged leaf (no FMA contraction)
__device__ __forceinline__ void frag_step(Frag& f, const double* As, const double* Bs, int c,
                                          int ty, int tx) {
  double a[4], b[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) a[i] = As[c * kLd + ty + 16 * i];
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = Bs[c * kLd + tx + 16 * i];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      double df = __dsub_rn(a[i], b[j]);
      f.v[i * 4 + j] = __dadd_rn(f.v[i * 4 + j], __dmul_rn(df, df));
    }
}

__device__ __forceinline__ void frag_first(Frag& f, const double* As, const double* Bs, int c,
                                           int ty, int tx) {
  double a[4], b[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) a[i] = As[c * kLd + ty + 16 * i];
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = Bs[c * kLd + tx + 16 * i];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      double df = __dsub_rn(a[i], b[j]);
      f.v[i * 4 + j] = __dmul_rn(df, df);
    }
}

__device__ __forceinline__ void frag_add(Frag& a, const Frag& b) {
#pragma unroll
  for (int i = 0; i < 16; ++i) a.v[i] = __dadd_rn(a.v[i], b.v[i]);
}

// accumulator j of a pairwise leaf: sequential over i = j, j+8, ... < body
__device__ __forceinline__ void leaf_acc(Frag& f, const double* As, const double* Bs, int j,
                                         int body, int ty, int tx) {
  frag_first(f, As, Bs, j, ty, tx);
  for (int i = j + 8; i < body; i += 8) frag_step(f, As, Bs, i, ty, tx);
}

// numpy pairwise_sum of one staged leaf of length len (loops_utils.h.src)
__device__ __forceinline__ void leaf_pairwise(Frag& A, const double* As, const double* Bs,
                                              int len, int ty, int tx) {
  if (len < 8) {
    frag_zero(A, -0.0);
    for (int i = 0; i < len; ++i) frag_step(A, As, Bs, i, ty, tx);
    return;
  }
  const int body = len - (len % 8);
  Frag B, C, D;
  leaf_acc(A, As, Bs, 0, body, ty, tx);
  leaf_acc(B, As, Bs, 1, body, ty, tx);
  frag_add(A, B);  // r0 + r1
  leaf_acc(B, As, Bs, 2, body, ty, tx);
  leaf_acc(C, As, Bs, 3, body, ty, tx);
  frag_add(B, C);  // r2 + r3
  frag_add(A, B);  // (r0+r1)+(r2+r3)
  leaf_acc(B, As, Bs, 4, body, ty, tx);
  leaf_acc(C, As, Bs, 5, body, ty, tx);
  frag_add(B, C);
  leaf_acc(C, As, Bs, 6, body, ty, tx);
  leaf_acc(D, As, Bs, 7, body, ty, tx);
  frag_add(C, D);
  frag_add(B, C);  // (r4+r5)+(r6+r7)
  frag_add(A, B);
  for (int i = body; i < len; ++i) frag_step(A, As, Bs, i, ty, tx);
}

__device__ __forceinline__ void stage_rows(double* S, const double* __restrict__ Xg, int64_t d,
                                           int64_t prow0, int nvalid, int c0, int len) {
  const int total = kQ * len;
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
    int r = idx / len, c = idx - r * len;
    double v = 0.0;
    if (r < nvalid) v = Xg[(prow0 + r) * d + c0 + c];
    S[c * kLd + r] = v;
  }
}

template <int DEPTH>
__global__ void __launch_bounds__(256, 1)
adjacency_exact_kernel(const double* __restrict__ Xg, int64_t d, ElemTables et, double eps,
                       const TileRef* __restrict__ tiles, uint32_t* __restrict__ adj,
                       int32_t* __restrict__ nonempty, int64_t tile0,
                       const __grid_constant__ PwProgram c_prog) {
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + kKC * kLd;
  __shared__ uint32_t bits[kTile * 4];

  const int64_t g = tile0 + blockIdx.x;  // slot
  const TileRef tr = tiles[g];
  const int k = tr.k, I = tr.I, J = tr.J;
  const int n_k = et.nrows[k];
  const int64_t pb = et.pbase[k];
  const int mode = et.order[k];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  for (int i = threadIdx.x; i < kTile * 4; i += blockDim.x) bits[i] = 0u;

  for (int q = 0; q < 4; ++q) {
    const int qa = q >> 1, qb = q & 1;
    const int ra = I * kTile + qa * kQ, rb = J * kTile + qb * kQ;  // local rows
    if (ra >= n_k || rb >= n_k) continue;  // uniform
    const int va = min(kQ, n_k - ra), vb = min(kQ, n_k - rb);
    Frag acc;
    Frag stk[DEPTH];
    if (mode == BM_ORDER_SEQUENTIAL) {
      frag_zero(acc, 0.0);
      for (int c0 = 0; c0 < d; c0 += kKC) {
        const int len = (int)((d - c0) < kKC ? (d - c0) : kKC);
        __syncthreads();
        stage_rows(As, Xg, d, pb + ra, va, c0, len);
        stage_rows(Bs, Xg, d, pb + rb, vb, c0, len);
        __syncthreads();
        for (int c = 0; c < len; ++c) frag_step(acc, As, Bs, c, ty, tx);
      }
    } else {
      for (int li = 0; li < c_prog.n_leaves; ++li) {
        const PwLeaf lf = c_prog.leaf[li];
        __syncthreads();
        stage_rows(As, Xg, d, pb + ra, va, lf.start, lf.len);
        stage_rows(Bs, Xg, d, pb + rb, vb, lf.start, lf.len);
        __syncthreads();
        Frag leaf;
        leaf_pairwise(leaf, As, Bs, lf.len, ty, tx);
        // push
#pragma unroll
        for (int s = DEPTH - 1; s > 0; --s) stk[s] = stk[s - 1];
        stk[0] = leaf;
        if constexpr (DEPTH > 1) {
          for (int p = 0; p < lf.pops; ++p) {
            frag_add(stk[1], stk[0]);
#pragma unroll
            for (int s = 0; s < DEPTH - 1; ++s) stk[s] = stk[s + 1];
          }
        }
      }
      acc = stk[0];
    }
    // decisions -> bit words (see header comment for the lane mapping)
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int rl = ty + 16 * a;
#pragma unroll
      for (int bw = 0; bw < 2; ++bw) {
        bool in0, in1;
        {
          const int cl = tx + 16 * (2 * bw);
          double dist = __dsqrt_rn(__dadd_rn(0.0, acc.v[a * 4 + 2 * bw]));
          in0 = rl < va && cl < vb && dist <= eps;
        }
        {
          const int cl = tx + 16 * (2 * bw + 1);
          double dist = __dsqrt_rn(__dadd_rn(0.0, acc.v[a * 4 + 2 * bw + 1]));
          in1 = rl < va && cl < vb && dist <= eps;
        }
        unsigned m0 = __ballot_sync(0xffffffffu, in0);
        unsigned m1 = __ballot_sync(0xffffffffu, in1);
        const int R_even = qa * kQ + 2 * warp + 16 * a;
        const int word = qb * 2 + bw;
        if (lane == 0) bits[R_even * 4 + word] = (m0 & 0xffffu) | (m1 << 16);
        if (lane == 16) bits[(R_even + 1) * 4 + word] = (m0 >> 16) | (m1 & 0xffff0000u);
      }
    }
  }
  __syncthreads();
  uint32_t* dst = adj + g * kTileWords;
  int any = 0;
  for (int i = threadIdx.x; i < kTileWords; i += blockDim.x) {
    dst[i] = bits[i];
    any |= bits[i] != 0u;
  }
  any = __syncthreads_or(any);
  if (threadIdx.x == 0) nonempty[g] = any;
}

// ---------------------------------------------------------------------------
// counts from the bitmap: rows of every tile, columns of off-diagonal tiles
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128)
count_kernel(const uint32_t* __restrict__ adj, ElemTables et, const TileUnit* __restrict__ units,
             const TileRef* __restrict__ tiles, int64_t slot0, int64_t n_units,
             int32_t* __restrict__ cnt) {
  __shared__ uint32_t bits[kTileWords];
  for (int64_t u = blockIdx.x; u < n_units; u += gridDim.x) {
    const TileUnit un = units[u];
    const int64_t pb = et.pbase[un.k];
    int rc = 0;
    for (int t = 0; t < un.cnt; ++t) {
      const int64_t g = un.off + t;
      const int J = tiles[g].J;
      __syncthreads();
      const uint4 w = reinterpret_cast<const uint4*>(adj + (g - slot0) * kTileWords)[threadIdx.x];
      reinterpret_cast<uint4*>(bits)[threadIdx.x] = w;
      rc += __popc(w.x) + __popc(w.y) + __popc(w.z) + __popc(w.w);
      if (J != un.I) {
        __syncthreads();
        const int c = threadIdx.x, wd = c >> 5, sh = c & 31;
        int cc = 0;
#pragma unroll 8
        for (int r = 0; r < kTile; ++r) cc += (bits[r * 4 + wd] >> sh) & 1u;
        if (cc) atomicAdd(cnt + pb + J * kTile + c, cc);
      }
    }
    if (rc) atomicAdd(cnt + pb + un.I * kTile + threadIdx.x, rc);
  }
}

__global__ void core_init_kernel(const int32_t* __restrict__ cnt, ElemTables et, int64_t P,
                                 int32_t min_pts, uint8_t* __restrict__ core,
                                 int32_t* __restrict__ par, int32_t* __restrict__ bmin) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P;
       p += (int64_t)gridDim.x * blockDim.x) {
    core[p] = cnt[p] >= min_pts ? 1 : 0;  // pads have count 0 and min_pts >= 1
    par[p] = (int32_t)p;
    bmin[p] = kNoCore;
  }
}

// ---------------------------------------------------------------------------
// union-find + border over the bitmap. DIAG selects the diagonal-tile pass
// (run first) or the off-diagonal pass.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int lfind(int* lp, int x) {
  while (true) {
    int p = lp[x];
    if (p == x) return x;
    int gp = lp[p];
    lp[x] = gp;
    x = gp;
  }
}
__device__ __forceinline__ bool lunion(int* lp, int a, int b) {
  while (true) {
    a = lfind(lp, a);
    b = lfind(lp, b);
    if (a == b) return false;
    if (a > b) { int t = a; a = b; b = t; }
    if (atomicCAS(lp + b, b, a) == b) return true;
  }
}

// one step of the in-warp 32x32 bit transpose: lane j ends with bit i = the
// input word of lane i, bit j
__device__ __forceinline__ uint32_t bit_transpose_step(uint32_t w, int s, uint32_t m, int lane) {
  const uint32_t t = __shfl_xor_sync(0xffffffffu, w, s);
  return (lane & s) ? ((w & ~m) | ((t >> s) & m)) : ((w & m) | ((t << s) & ~m));
}

#ifdef BM_COMP_STATS
// dev counters (-DBM_COMP_STATS): tiles by path, unions, merges
__device__ unsigned long long g_comp_stats[8];
#define COMP_STAT(i) (threadIdx.x == 0 ? atomicAdd(&g_comp_stats[i], 1ull) : 0ull)
#else
#define COMP_STAT(i) 0ull
#endif

// off-diagonal phases: tile pairs [kCompCuts[i-1], kCompCuts[i]) of every unit,
// with a compression of the forest between phases
#ifndef BM_DIAG_BFS
#define BM_DIAG_BFS 1
#endif
constexpr bool kDiagBfs = BM_DIAG_BFS;  // diagonal pass: mask BFS (diag_bfs_kernel)

#ifndef BM_COMP_CUT1
#define BM_COMP_CUT1 6
#endif
#ifndef BM_COMP_CUT2
#define BM_COMP_CUT2 0
#endif
#if BM_COMP_CUT2 > 0
constexpr int kCompCuts[] = {0, BM_COMP_CUT1, BM_COMP_CUT2, 1 << 30};
#else
constexpr int kCompCuts[] = {0, BM_COMP_CUT1, 1 << 30};
#endif
constexpr int kCompPhases = (int)(sizeof(kCompCuts) / sizeof(kCompCuts[0])) - 1;

template <bool DIAG>
__global__ void __launch_bounds__(128, 16)
components_kernel(const uint32_t* __restrict__ adj, ElemTables et,
                  const TileUnit* __restrict__ units, const TileRef* __restrict__ tiles,
                  int64_t slot0, int64_t n_units, const uint8_t* __restrict__ core,
                  int32_t* __restrict__ par, int32_t* __restrict__ bmin,
                  const int32_t* __restrict__ uni, const int32_t* __restrict__ nonempty,
                  int s_lo, int s_hi) {
  __shared__ uint32_t bits[kTileWords];
  __shared__ int groot[2 * kTile];  // global root of each tile node (-1: not core)
  __shared__ int lp[2 * kTile];     // local union-find over tile nodes
  __shared__ uint32_t coreJ[4], coreI[4];
  __shared__ int any_merge;
  __shared__ int rmm[4][4];  // per warp: min/max core root of rows, of columns
  __shared__ int2 grp[4][32];  // off-diagonal: per column word, (root, lanes) of each root group
  __shared__ int ngrp[4];
  const int t = threadIdx.x;
  for (int64_t u = blockIdx.x; u < n_units; u += gridDim.x) {
    const TileUnit un = units[u];
    const int k = un.k, I = un.I;
    const int64_t pb = et.pbase[k];
    const int nk = et.nrows[k];
    const int pI = (int)(pb + I * kTile);
    BM_DASSERT(k >= 0 && k < et.n_el && I >= 0 && I < et.ntiles[k]);
    // row side once per unit (stale roots later only cost redundant unions)
    const bool ci = core[pI + t];
    int gr = ci ? uf_find(par, pI + t) : -1;
    __syncthreads();
    {
      const unsigned bi = __ballot_sync(0xffffffffu, ci);
      if ((t & 31) == 0) coreI[t >> 5] = bi;
    }
    const int uI = DIAG ? -1 : uni[(pb >> 7) + I];
    const int s_end = un.cnt < s_hi ? un.cnt : s_hi;
    for (int s = s_lo; s < s_end; ++s) {
      const int64_t g = un.off + s;
      const int J = tiles[g].J;
      BM_DASSERT(tiles[g].k == k && tiles[g].I == I && J >= I && J < et.ntiles[k]);
      const int pJ = (int)(pb + J * kTile);
      (void)COMP_STAT(0);
      if (!DIAG) {
        if (!nonempty[g - slot0]) {
          (void)COMP_STAT(1);
          continue;  // no bit: nothing to join (block-uniform)
        }
        if (uI >= 0) {
          // both tiles all-core with one root each: the tile's bits can only
          // join the two roots (border rules need non-core rows: none here)
          const int uJ = uni[(pb >> 7) + J];
          if (uJ >= 0) {
            (void)COMP_STAT(2);
            if (t == 0 && uI != uJ) uf_union(par, uI, uJ);
            continue;  // block-uniform
          }
        }
      }
      __syncthreads();
      reinterpret_cast<uint4*>(bits)[t] =
          reinterpret_cast<const uint4*>(adj + (g - slot0) * kTileWords)[t];
      const bool cj = DIAG ? ci : (bool)core[pJ + t];
      if (!DIAG) {
        const unsigned bj = __ballot_sync(0xffffffffu, cj);
        if ((t & 31) == 0) coreJ[t >> 5] = bj;
      }
      groot[t] = gr;
      const int grj = (!DIAG && cj) ? uf_find(par, pJ + t) : -1;
      groot[kTile + t] = grj;
      lp[t] = t;
      lp[kTile + t] = kTile + t;
      if (t == 0) any_merge = 0;
      if (!DIAG) {  // per-warp min/max of the core roots of rows and columns
        const int w = t >> 5;
        const unsigned mnI = __reduce_min_sync(0xffffffffu, ci ? (unsigned)gr : 0x7fffffffu);
        const int mxI = __reduce_max_sync(0xffffffffu, ci ? gr : -1);
        const unsigned mnJ = __reduce_min_sync(0xffffffffu, cj ? (unsigned)grj : 0x7fffffffu);
        const int mxJ = __reduce_max_sync(0xffffffffu, cj ? grj : -1);
        if ((t & 31) == 0) {
          rmm[0][w] = (int)mnI;
          rmm[1][w] = mxI;
          rmm[2][w] = (int)mnJ;
          rmm[3][w] = mxJ;
        }
        // the word's core columns grouped by global root (after the diagonal
        // pass a word holds few roots): a row joins each group it touches once
        // instead of visiting every neighbouring column
        const int lane = t & 31;
        const unsigned eq = __match_any_sync(0xffffffffu, cj ? grj : -1);
        const bool lead = cj && (__ffs(eq) - 1 == lane);
        const unsigned lm = __ballot_sync(0xffffffffu, lead);
        if (lead) grp[w][__popc(lm & ((1u << lane) - 1u))] = make_int2(grj, (int)eq);
        if (lane == 0) ngrp[w] = __popc(lm);
      }
      __syncthreads();
      const int r = t;
      bool uniform = false;
      if (!DIAG) {
        // every core row in one (possibly stale) root RI and every core column
        // in one root RJ: one union(RI, RJ) covers all core-core bits
        const int mnI = min(min(rmm[0][0], rmm[0][1]), min(rmm[0][2], rmm[0][3]));
        const int mxI = max(max(rmm[1][0], rmm[1][1]), max(rmm[1][2], rmm[1][3]));
        const int mnJ = min(min(rmm[2][0], rmm[2][1]), min(rmm[2][2], rmm[2][3]));
        const int mxJ = max(max(rmm[3][0], rmm[3][1]), max(rmm[3][2], rmm[3][3]));
        uniform = (mxI < 0 || mnI == mxI) && (mxJ < 0 || mnJ == mxJ);
        (void)COMP_STAT(uniform ? 3 : 4);
        if (uniform) {
          const bool hit = ci && (((bits[r * 4] & coreJ[0]) | (bits[r * 4 + 1] & coreJ[1]) |
                                   (bits[r * 4 + 2] & coreJ[2]) | (bits[r * 4 + 3] & coreJ[3])) != 0u);
          const int any = __syncthreads_or(hit && mnI != mnJ);
          if (any) {
            if (t == 0) uf_union(par, mnI, mnJ);
            __syncthreads();
            if (ci) gr = uf_find(par, gr);
          }
        }
      }
      // --- core-core edges between nodes with different global roots; a row
      //     joins each distinct neighbouring global root once (consecutive
      //     bits mostly share the root, so `last` skips the repeats)
      if (ci && !uniform) {
        int last = gr;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          uint32_t m = bits[r * 4 + w] & (DIAG ? coreI[w] : coreJ[w]);
          if (DIAG) {
            // the diagonal tile is symmetric (the ε relation is): row r joins
            // only its neighbours c < r, each edge is visited once
            const int lo = r - w * 32;
            m &= lo >= 32 ? 0xffffffffu : (lo <= 0 ? 0u : (1u << lo) - 1u);
          } else if (m && ngrp[w] <= __popc(m)) {
            // walk the word's root groups (one group: every core column has
            // the same root): one join with the first neighbour of a group
            // stands for all of its columns
            const int ng = ngrp[w];
            for (int q = 0; q < ng; ++q) {
              const int2 G = grp[w][q];
              const uint32_t mm = m & (uint32_t)G.y;
              if (mm && G.x != gr && G.x != last) {
                last = G.x;
                if (lunion(lp, r, kTile + w * 32 + __ffs(mm) - 1)) any_merge = 1;
              }
            }
            continue;
          }
          while (m) {
            const int c = w * 32 + __ffs(m) - 1;
            m &= m - 1;
            const int node = DIAG ? c : kTile + c;
            const int gn = groot[node];
            if (gn != gr && (DIAG || gn != last)) {
              last = gn;
              if (lunion(lp, r, node)) any_merge = 1;
            }
          }
        }
      }
      // --- border: non-core row r -> its core neighbour of smallest ENTRY
      if (!ci && r < nk - I * kTile) {
        const int cb = DIAG ? pI : pJ;
        int best = kNoCore;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          uint32_t m = bits[r * 4 + w] & (DIAG ? coreI[w] : coreJ[w]);
          while (m) {
            const int c = w * 32 + __ffs(m) - 1;
            m &= m - 1;
            best = min(best, et.ent[cb + c]);
          }
        }
        if (best < __ldcg(bmin + pI + r)) atomicMin(bmin + pI + r, best);
      }
      // --- border: non-core column c -> its core row of smallest entry
      //     (off-diagonal only). Warp w owns columns 32w..32w+31 = word w: four
      //     32x32 bit transposes give each lane its column's row bits, so only
      //     the set bits are visited.
      if (!DIAG) {
        const bool need = !cj && t < nk - J * kTile;
        if (__any_sync(0xffffffffu, need)) {  // warp-uniform
          const int lane = t & 31, wd = t >> 5;
          int best = kNoCore;
#pragma unroll
          for (int rb = 0; rb < 4; ++rb) {
            uint32_t x = bits[(rb * 32 + lane) * 4 + wd];
            x = bit_transpose_step(x, 16, 0x0000FFFFu, lane);
            x = bit_transpose_step(x, 8, 0x00FF00FFu, lane);
            x = bit_transpose_step(x, 4, 0x0F0F0F0Fu, lane);
            x = bit_transpose_step(x, 2, 0x33333333u, lane);
            x = bit_transpose_step(x, 1, 0x55555555u, lane);
            uint32_t m = need ? (x & coreI[rb]) : 0u;  // bit i: row 32 rb + i, core
            while (m) {
              const int i = __ffs(m) - 1;
              m &= m - 1;
              best = min(best, et.ent[pI + rb * 32 + i]);
            }
          }
          if (need && best < __ldcg(bmin + pJ + t)) atomicMin(bmin + pJ + t, best);
        }
      }
      __syncthreads();
      if (any_merge) (void)COMP_STAT(5);
      // --- propagate local merges to the global forest
      if (any_merge) {
        for (int x = t; x < 2 * kTile; x += blockDim.x) {
          if (groot[x] < 0) continue;
          const int lr = lfind(lp, x);
          if (lr != x && groot[lr] != groot[x]) uf_union(par, groot[x], groot[lr]);
        }
        if (ci) gr = uf_find(par, gr);  // refresh the row roots after merges
      }
    }
  }
}

// Diagonal pass as a breadth-first search over 128-bit masks. Each row is in
// exactly one diagonal tile, so a tile's components are found inside its CTA
// and every core row is joined to its component's smallest row by one union
// (uncontended: each row hooks its own root). Per component, each
// BFS level ORs the bitmap rows of the frontier with one block reduction;
// a dense tile is one component found in 2-3 levels instead of a walk over
// its ~8k bits. Isolated core rows are settled before the search.
__global__ void __launch_bounds__(128)
diag_bfs_kernel(const uint32_t* __restrict__ adj, ElemTables et,
                const TileUnit* __restrict__ units, const TileRef* __restrict__ tiles,
                int64_t slot0, int64_t n_units, const uint8_t* __restrict__ core,
                int32_t* __restrict__ par, int32_t* __restrict__ bmin) {
  __shared__ uint32_t s_core[4];
  __shared__ uint32_t s_red[4][4];
  __shared__ uint32_t s_rem[4];
  const int t = threadIdx.x, lane = t & 31, wq = t >> 5;
  for (int64_t u = blockIdx.x; u < n_units; u += gridDim.x) {
    const TileUnit un = units[u];
    const int k = un.k, I = un.I;
    const int64_t g = un.off;  // the row tile's first kept tile: its diagonal
    BM_DASSERT(tiles[g].k == k && tiles[g].I == I && tiles[g].J == I);
    const int64_t pb = et.pbase[k];
    const int nk = et.nrows[k];
    const int pI = (int)(pb + I * kTile);
    const uint4 rw = reinterpret_cast<const uint4*>(adj + (g - slot0) * kTileWords)[t];
    const bool ci = core[pI + t];
    __syncthreads();  // the previous unit's readers of s_core / s_rem are done
    {
      const unsigned b = __ballot_sync(0xffffffffu, ci);
      if (lane == 0) s_core[wq] = b;
    }
    __syncthreads();
    const uint32_t c0 = s_core[0], c1 = s_core[1], c2 = s_core[2], c3 = s_core[3];
    // my row's core neighbours other than myself
    uint32_t nb[4] = {rw.x & c0, rw.y & c1, rw.z & c2, rw.w & c3};
#pragma unroll
    for (int w = 0; w < 4; ++w)
      if (w == wq) nb[w] &= ~(1u << lane);  // static indices: no local memory
    const bool lonely = ci && !(nb[0] | nb[1] | nb[2] | nb[3]);
    int lab = ci ? t : -1;  // component's smallest row (lonely rows: themselves)
    {
      const unsigned b = __ballot_sync(0xffffffffu, ci && !lonely);
      if (lane == 0) s_rem[wq] = b;
    }
    __syncthreads();
    uint32_t rem[4] = {s_rem[0], s_rem[1], s_rem[2], s_rem[3]};  // block-uniform
    while (rem[0] | rem[1] | rem[2] | rem[3]) {
      const int wseed = rem[0] ? 0 : rem[1] ? 1 : rem[2] ? 2 : 3;
      const uint32_t rs = rem[0] ? rem[0] : rem[1] ? rem[1] : rem[2] ? rem[2] : rem[3];
      const int seed = wseed * 32 + __ffs(rs) - 1;
      uint32_t comp[4], front[4];
#pragma unroll
      for (int w = 0; w < 4; ++w) comp[w] = front[w] = w == wseed ? 1u << (seed & 31) : 0u;
      while (true) {
        const uint32_t fw = wq == 0 ? front[0] : wq == 1 ? front[1] : wq == 2 ? front[2] : front[3];
        const bool in_front = (fw >> lane) & 1u;
        uint32_t m[4];
#pragma unroll
        for (int w = 0; w < 4; ++w) m[w] = in_front ? nb[w] : 0u;
#pragma unroll
        for (int w = 0; w < 4; ++w) m[w] = __reduce_or_sync(0xffffffffu, m[w]);
        if (lane == 0) {
#pragma unroll
          for (int w = 0; w < 4; ++w) s_red[wq][w] = m[w];
        }
        __syncthreads();
        uint32_t any = 0u;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const uint32_t all = s_red[0][w] | s_red[1][w] | s_red[2][w] | s_red[3][w];
          front[w] = all & ~comp[w];
          comp[w] |= front[w];
          any |= front[w];
        }
        __syncthreads();  // s_red is rewritten by the next level
        if (!any) break;  // block-uniform
      }
      const uint32_t cwq = wq == 0 ? comp[0] : wq == 1 ? comp[1] : wq == 2 ? comp[2] : comp[3];
      if ((cwq >> lane) & 1u) lab = seed;
#pragma unroll
      for (int w = 0; w < 4; ++w) rem[w] &= ~comp[w];
    }
    if (ci) {
      // a union, not a store: in row windows (huge elements) an earlier
      // window's off-diagonal pass may already have hooked these rows
      if (lab != t) uf_union(par, pI + t, pI + lab);
    } else if (t < nk - I * kTile) {
      // border: non-core row -> its core neighbour of smallest ENTRY
      int best = kNoCore;
      const uint32_t cw[4] = {rw.x & c0, rw.y & c1, rw.z & c2, rw.w & c3};
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        uint32_t m = cw[w];
        while (m) {
          best = min(best, et.ent[pI + w * 32 + __ffs(m) - 1]);
          m &= m - 1;
        }
      }
      if (best < __ldcg(bmin + pI + t)) atomicMin(bmin + pI + t, best);
    }
  }
}

// Debug check (B200MAP_CHECK_SYMMETRY=1): every diagonal tile bitmap equals
// its transpose. The diagonal components pass joins only the bits c < r of
// row r, so it relies on this invariant: the eps relation is symmetric, and
// every engine must produce (r, c) and (c, r) alike (the tensor-core epilogue
// reaches them by different routes: per-row bounds, floor(N_j / U) on the
// column side, the recheck queue; each route is rigorous, hence they agree).
__global__ void __launch_bounds__(128)
diag_symmetry_kernel(const uint32_t* __restrict__ adj, const TileUnit* __restrict__ units,
                     const TileRef* __restrict__ tiles, int64_t slot0, int64_t n_units,
                     unsigned long long* __restrict__ bad) {
  __shared__ uint32_t bits[kTileWords];
  for (int64_t u = blockIdx.x; u < n_units; u += gridDim.x) {
    const TileUnit un = units[u];
    for (int s = 0; s < un.cnt; ++s) {
      const int64_t g = un.off + s;
      if (tiles[g].J != un.I) continue;  // block-uniform
      __syncthreads();
      reinterpret_cast<uint4*>(bits)[threadIdx.x] =
          reinterpret_cast<const uint4*>(adj + (g - slot0) * kTileWords)[threadIdx.x];
      __syncthreads();
      const int r = threadIdx.x;
      int nbad = 0;
      for (int c = 0; c < kTile; ++c) {
        const uint32_t a = (bits[r * 4 + (c >> 5)] >> (c & 31)) & 1u;
        const uint32_t b = (bits[c * 4 + (r >> 5)] >> (r & 31)) & 1u;
        nbad += a != b;
      }
      if (nbad) atomicAdd(bad, (unsigned long long)nbad);
    }
  }
}

bool check_symmetry() {
  const char* e = getenv("B200MAP_CHECK_SYMMETRY");
  return e && e[0] == '1';
}

// per 128-row tile: the common root of its rows if every valid row is core
// and all share one root (stale roots are fine: still in the component), else -1
__global__ void tile_uniform_kernel(ElemTables et, int64_t n_rt, const uint8_t* __restrict__ core,
                                    int32_t* __restrict__ par, int32_t* __restrict__ uni) {
  const int lane = threadIdx.x & 31;
  const int64_t wpb = blockDim.x >> 5;
  for (int64_t rt = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5); rt < n_rt;
       rt += (int64_t)gridDim.x * wpb) {
    bool ok = true;
    int mn = 0x7fffffff, mx = -1;
    for (int i = lane; i < kTile; i += 32) {
      const int64_t p = rt * kTile + i;
      if (et.ent[p] < 0) continue;
      if (!core[p]) {
        ok = false;
        continue;
      }
      const int r = uf_find(par, (int)p);
      mn = min(mn, r);
      mx = max(mx, r);
    }
    ok = __all_sync(0xffffffffu, ok);
    mn = (int)__reduce_min_sync(0xffffffffu, (unsigned)mn);
    mx = __reduce_max_sync(0xffffffffu, mx);
    if (lane == 0) uni[rt] = (ok && mx >= 0 && mn == mx) ? mn : -1;
  }
}

__global__ void compress_kernel(int32_t* __restrict__ par, const uint8_t* __restrict__ core,
                                int64_t P) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P;
       p += (int64_t)gridDim.x * blockDim.x)
    if (core[p]) par[p] = uf_find(par, (int)p);
}

// root label per padded index (-1 noise); cluster's smallest ENTRY via atomicMin
__global__ void label_kernel(ElemTables et, int64_t P, const uint8_t* __restrict__ core,
                             int32_t* __restrict__ par, const int32_t* __restrict__ bmin,
                             const int32_t* __restrict__ inv, int32_t* __restrict__ lab,
                             int32_t* __restrict__ cmin) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P;
       p += (int64_t)gridDim.x * blockDim.x) {
    int root = -1;
    if (core[p]) root = uf_find(par, (int)p);
    else if (bmin[p] != kNoCore) root = uf_find(par, inv[bmin[p]]);
    lab[p] = root;
    if (root >= 0) atomicMin(cmin + root, et.ent[p]);
  }
}

// head[e] = entry e is the smallest member of its cluster
__global__ void head_kernel(int64_t n_entries, const int32_t* __restrict__ inv,
                            const int32_t* __restrict__ lab, const int32_t* __restrict__ cmin,
                            int32_t* __restrict__ head) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n_entries;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int r = lab[inv[e]];
    head[e] = (r >= 0 && cmin[r] == (int)e) ? 1 : 0;
  }
}

// cluster rank of every entry inside its element (clusters ordered by their
// smallest entry, clustering.py:192-197), -1 for noise
__global__ void output_kernel(ElemTables et, const int64_t* __restrict__ offsets,
                              int64_t n_entries, const int32_t* __restrict__ inv,
                              const int32_t* __restrict__ lab, const int32_t* __restrict__ cmin,
                              const int64_t* __restrict__ hscan, int32_t* __restrict__ out) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n_entries;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = 0, b = et.n_el;
    while (b - a > 1) {
      int64_t mid = (a + b) >> 1;
      if (offsets[mid] <= e) a = mid; else b = mid;
    }
    const int r = lab[inv[e]];
    out[e] = r >= 0 ? (int32_t)(hscan[cmin[r]] - hscan[offsets[a]]) : -1;
  }
}

__global__ void fill_total_kernel(int64_t* hs, const int32_t* hd, int64_t n) {
  hs[n] = (n > 0 ? hs[n - 1] + hd[n - 1] : 0);
}

__global__ void nclusters_kernel(ElemTables et, const int64_t* __restrict__ offsets,
                                 const int64_t* __restrict__ hscan, int32_t* __restrict__ ncl) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < et.n_el) ncl[k] = (int32_t)(hscan[offsets[k + 1]] - hscan[offsets[k]]);
}

inline unsigned grid_for(int64_t n, int threads, int per_sm = 8) {
  int64_t b = ceil_div(n, threads);
  int64_t cap = (int64_t)num_sms() * per_sm;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (unsigned)b;
}

template <int DEPTH>
int launch_exact_depth(const double* Xg, int64_t d, const ElemTables& et, const TileRef* tiles,
                       int64_t n_tiles, double eps, uint32_t* adj, int32_t* nonempty,
                       const PwProgram& prog, cudaStream_t stream) {
  BM_TRY(ensure_dyn_smem((const void*)adjacency_exact_kernel<DEPTH>, (int)kExactSmem));
  const int64_t kMaxGrid = 1ll << 30;
  for (int64_t t0 = 0; t0 < n_tiles; t0 += kMaxGrid) {
    int64_t nb = std::min<int64_t>(kMaxGrid, n_tiles - t0);
    adjacency_exact_kernel<DEPTH><<<(unsigned)nb, 256, kExactSmem, stream>>>(
        Xg, d, et, eps, tiles, adj, nonempty, t0, prog);
    BM_CHECK_LAUNCH();
  }
  return BM_OK;
}

int exact_build_adjacency(const double* Xg, int64_t d, const ElemTables& et, const TileRef* tiles,
                          int64_t n_tiles, double eps, uint32_t* adj, int32_t* nonempty,
                          cudaStream_t stream) {
  if (n_tiles == 0) return BM_OK;
  PwProgram prog;
  BM_TRY(make_pw_program(d, &prog));
  switch (prog.depth) {
    case 1: return launch_exact_depth<1>(Xg, d, et, tiles, n_tiles, eps, adj, nonempty, prog, stream);
    case 2: return launch_exact_depth<2>(Xg, d, et, tiles, n_tiles, eps, adj, nonempty, prog, stream);
    case 3: return launch_exact_depth<3>(Xg, d, et, tiles, n_tiles, eps, adj, nonempty, prog, stream);
    case 4: return launch_exact_depth<4>(Xg, d, et, tiles, n_tiles, eps, adj, nonempty, prog, stream);
    default: return launch_exact_depth<kMaxStack>(Xg, d, et, tiles, n_tiles, eps, adj, nonempty, prog, stream);
  }
}

// full distance matrix of a row subset in one exact order (API helper)
__global__ void pairwise_matrix_kernel(const double* __restrict__ X, int64_t d,
                                       const int64_t* __restrict__ rows, int64_t n, int order,
                                       double* __restrict__ out,
                                       const __grid_constant__ PwProgram c_prog) {
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n * n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / n, j = idx - i * n;
    const double s = exact_dist2(X + rows[i] * d, X + rows[j] * d, d, order, c_prog);
    out[idx] = __dsqrt_rn(s);
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// One batch of elements resident on the device: the grouping permutation,
// gathered rows, per-row work arrays, tables, the pruned tile list and (tensor-
// core engine) the quantised planes. Bits are produced per WINDOW of tile rows:
// the whole batch at once, or — for an element whose bitmap exceeds the device
// budget — row blocks [I0, I1) of a single-element batch,
// in two passes (counts for every block, then components per block,
// recomputing the blocks that are not resident). A window is a contiguous run
// of the kept-tile list (sorted by element, row tile, column tile); its slots
// are renumbered from 0 and adj[slot] holds the bits.
// ---------------------------------------------------------------------------
struct WindowBufs {
  const TileRef* tiles = nullptr;  // the batch's full kept list (absolute slots)
  const TileUnit *diag = nullptr, *off = nullptr, *tcu = nullptr;
  int64_t slot0 = 0, n_tiles = 0, n_diag = 0, n_off = 0, n_tc = 0, pairs = 0;
};

// eps outside [1e-140, 1e140]: squared differences near eps can underflow
// to subnormals or overflow, where the relative error model behind the
// pruning bound (and the tensor-core band) does not hold — every tile pair is
// computed and every tensor-core decision is rechecked in exact fp64.
bool eps_in_model(double eps) { return eps >= 1e-140 && eps <= 1e140; }

bool prune_enabled(int64_t d, double eps) {
  const char* e = getenv("B200MAP_NO_PRUNE");  // tests: identity order, every tile pair
  return !(e && e[0] == '1') && d <= 512 && eps_in_model(eps);
}

struct BatchCtx {
  cudaStream_t stream = nullptr;
  int64_t d = 0;
  double eps = 0.0;
  int32_t min_pts = 1;
  bool use_tc = false;
  double qscale = 1.0;  // recheck queue capacity factor (batch retried on overflow)
  int64_t nb_el = 0, n_tp = 0, P = 0, n_entries = 0, n_rt = 0;
  std::vector<int64_t> tp_off, offs;
  std::vector<int32_t> pbase, nrows, ntiles, tbase;
  std::vector<uint8_t> order;
  // kept tile pairs (device list sorted by (k, I, J)) and, per global row
  // tile rt = tbase[k] + I, host copies of: first slot (n_rt+1 entries, last =
  // n_kept), first off-diagonal / tensor-core unit (n_rt+1), row pairs
  int64_t n_kept = 0;
  std::vector<int64_t> row_first, off_pos, tc_pos, row_pairs;
  Scratch tabs, xg, work, perm, s_units, s_geo, s_dir, s_seed;
  // dense per-tile-pair arrays (flags, positions, the kept list with room for
  // every pair): cached buffers, not pool blocks — at cfg5 they are ~6 GB,
  // and re-mapping them through the pool cost ~0.4 s per call
  BigScratch s_tiles, b_flags, b_pos;
  // direction bound: per row tile its seed (s_dir), per grouped element the
  // seeds (fp32), their norms and pairwise distances (s_seed); null if none
  int32_t* tseed = nullptr;
  float* seed_f = nullptr;
  double *seed_norm = nullptr, *seed_dist = nullptr;
  // direct: the tensor-core engine reads X through the membership (no
  // gathered fp64 copy Xg) and the direction bound runs on the limb planes
  // with int8 seeds (seeds_q; seed_dist then holds |s'_a - s'_b|)
  bool direct = false;
  RowSrc src{};
  Scratch s_seedq;
  int8_t* seeds_q = nullptr;
  TileRef* d_tiles = nullptr;
  TileUnit *d_diag = nullptr, *d_off = nullptr, *d_tcu = nullptr;
  ElemTables et{};
  int32_t *cnt = nullptr, *par = nullptr, *bmin = nullptr, *lab = nullptr, *cmin = nullptr,
          *head = nullptr, *ent = nullptr, *inv = nullptr;
  int64_t* xrow = nullptr;  // padded index -> dataset row (-1: pad)
  int64_t* hscan = nullptr;
  uint8_t* core = nullptr;
  int64_t* d_offs = nullptr;
  TcPrep* tc = nullptr;
  BatchCtx() = default;
  BatchCtx(const BatchCtx&) = delete;
  ~BatchCtx() { tc_release(tc); }

  int setup(const double* d_X, const int64_t* d_rows, const int64_t* h_offsets,
            const uint8_t* h_order, int64_t k0, int64_t k1, int64_t* stats) {
    nb_el = k1 - k0;
    tp_off.assign(nb_el + 1, 0);
    offs.assign(nb_el + 1, 0);
    pbase.assign(nb_el + 1, 0);
    tbase.assign(nb_el + 1, 0);
    nrows.assign(nb_el, 0);
    ntiles.assign(nb_el, 0);
    order.assign(nb_el, 0);
    for (int64_t i = 0; i < nb_el; ++i) {
      const int64_t k = k0 + i;
      const int64_t nk = h_offsets[k + 1] - h_offsets[k];
      const int64_t T = ceil_div(nk, kTile);
      nrows[i] = (int32_t)nk;
      ntiles[i] = (int32_t)T;
      order[i] = h_order[k];
      tp_off[i + 1] = tp_off[i] + T * (T + 1) / 2;
      pbase[i + 1] = (int32_t)(pbase[i] + T * kTile);
      tbase[i + 1] = (int32_t)(tbase[i] + T);
      offs[i] = h_offsets[k] - h_offsets[k0];
    }
    offs[nb_el] = h_offsets[k1] - h_offsets[k0];
    n_tp = tp_off[nb_el];
    P = pbase[nb_el];
    n_rt = tbase[nb_el];
    n_entries = offs[nb_el];
    if (n_entries == 0) return BM_OK;

    const size_t tab_bytes = (nb_el + 1) * 8 * 2 + (nb_el + 1) * 4 * 4 + nb_el + 64;
    BM_TRY(scratch_alloc(tabs, tab_bytes, stream));
    char* tp = tabs.as<char>();
    int64_t* d_tp_off = (int64_t*)tp;
    d_offs = d_tp_off + nb_el + 1;
    int32_t* d_pbase = (int32_t*)(d_offs + nb_el + 1);
    int32_t* d_nrows = d_pbase + nb_el + 1;
    int32_t* d_ntiles = d_nrows + nb_el + 1;
    int32_t* d_tbase = d_ntiles + nb_el + 1;
    uint8_t* d_order = (uint8_t*)(d_tbase + nb_el + 1);
    BM_CHECK_CUDA(cudaMemcpyAsync(d_tp_off, tp_off.data(), (nb_el + 1) * 8, cudaMemcpyHostToDevice, stream));
    BM_CHECK_CUDA(cudaMemcpyAsync(d_offs, offs.data(), (nb_el + 1) * 8, cudaMemcpyHostToDevice, stream));
    BM_CHECK_CUDA(cudaMemcpyAsync(d_pbase, pbase.data(), (nb_el + 1) * 4, cudaMemcpyHostToDevice, stream));
    BM_CHECK_CUDA(cudaMemcpyAsync(d_nrows, nrows.data(), nb_el * 4, cudaMemcpyHostToDevice, stream));
    BM_CHECK_CUDA(cudaMemcpyAsync(d_ntiles, ntiles.data(), nb_el * 4, cudaMemcpyHostToDevice, stream));
    BM_CHECK_CUDA(cudaMemcpyAsync(d_tbase, tbase.data(), (nb_el + 1) * 4, cudaMemcpyHostToDevice, stream));
    BM_CHECK_CUDA(cudaMemcpyAsync(d_order, order.data(), nb_el, cudaMemcpyHostToDevice, stream));
    BM_TRY(scratch_alloc(perm, (size_t)(P + n_entries) * 4 + 16 + (size_t)P * 8, stream));
    ent = perm.as<int32_t>();
    inv = ent + P;
    xrow = reinterpret_cast<int64_t*>(((uintptr_t)(inv + n_entries) + 15) & ~(uintptr_t)15);
    et = ElemTables{d_tp_off, d_pbase, d_nrows, d_ntiles, d_order, ent, nb_el};
    const int64_t* rows_b = d_rows + h_offsets[k0];
    const bool prune = prune_enabled(d, eps);
    // per-row bulk copies of X rows need 16-byte row sizes (d even);
    // B200MAP_NO_DIRECT=1 keeps the gathered copy (A/B checks)
    const char* no_direct = getenv("B200MAP_NO_DIRECT");
    direct = use_tc && (d % 2 == 0) && !(no_direct && no_direct[0] == '1');

    trace_mark("setup:tables", stream);
    // ---- row order inside each element: grouped (stable by seed) or identity
    {
      Scratch s_k, s_v, s_it;
      BM_TRY(scratch_alloc(s_k, (size_t)n_entries * 8, stream));
      BM_TRY(scratch_alloc(s_v, (size_t)n_entries * 8, stream));
      std::vector<GroupItem> items;
      bool any_small = false;
      const int64_t min_rows = prune ? kGroupMinRows : (1ll << 62);
      for (int64_t i = 0; i < nb_el; ++i) {
        if (nrows[i] >= min_rows) {
          for (int64_t e = offs[i]; e < offs[i + 1]; e += 256)
            items.push_back({(int32_t)i, (int32_t)e, (int32_t)std::min<int64_t>(e + 256, offs[i + 1]), 0});
        } else if (nrows[i] > 0) {
          any_small = true;
        }
      }
      if (any_small) {
        group_identity_kernel<<<grid_for(n_entries, 256), 256, 0, stream>>>(
            d_offs, nb_el, n_entries, min_rows, s_k.as<uint64_t>(), s_v.as<int64_t>());
        BM_CHECK_LAUNCH();
      }
      if (!items.empty()) {
        std::vector<int32_t> gel;
        for (int64_t i = 0; i < nb_el; ++i)
          if (nrows[i] >= min_rows) gel.push_back((int32_t)i);
        Scratch s_rank, s_gel;
        BM_TRY(scratch_alloc(s_rank, (size_t)nb_el * kGroupSeeds * 4 * 2, stream));
        BM_TRY(scratch_alloc(s_gel, gel.size() * 4, stream));
        BM_CHECK_CUDA(cudaMemcpyAsync(s_gel.ptr, gel.data(), gel.size() * 4,
                                      cudaMemcpyHostToDevice, stream));
        int32_t* d_order = s_rank.as<int32_t>() + nb_el * kGroupSeeds;
        Scratch s_tab;
        BM_TRY(scratch_alloc(s_tab, (size_t)nb_el * kSeedTab * 4, stream));
        seed_order_kernel<<<(unsigned)gel.size(), 256, 0, stream>>>(
            d_X, d, rows_b, d_offs, s_gel.as<int32_t>(), s_rank.as<int32_t>(), d_order,
            s_tab.as<float>());
        BM_CHECK_LAUNCH();
        // seeds for the direction bound (fp32 copy, norms, pair distances;
        // direct: int8 seeds and their integer difference norms)
        BM_TRY(scratch_alloc(s_seed, (size_t)nb_el * kGroupSeeds * (d * 4 + 8 + kGroupSeeds * 8),
                             stream));
        seed_norm = s_seed.as<double>();
        seed_dist = seed_norm + nb_el * kGroupSeeds;
        seed_f = reinterpret_cast<float*>(seed_dist + (int64_t)nb_el * kGroupSeeds * kGroupSeeds);
        if (direct) {
          const int64_t kpad = tc_kpad(d);
          BM_TRY(scratch_alloc(s_seedq, (size_t)nb_el * kGroupSeeds * kpad, stream));
          seeds_q = s_seedq.as<int8_t>();
          seed_quant_kernel<<<(unsigned)gel.size(), 256, 0, stream>>>(
              d_X, d, rows_b, d_offs, s_gel.as<int32_t>(), kpad, seeds_q, seed_dist);
        } else {
          seed_data_kernel<<<(unsigned)(gel.size() * kGroupSeeds), 256, 0, stream>>>(
              d_X, d, rows_b, d_offs, s_gel.as<int32_t>(), seed_f, seed_norm, seed_dist);
        }
        BM_CHECK_LAUNCH();
        BM_TRY(scratch_alloc(s_it, items.size() * sizeof(GroupItem), stream));
        BM_CHECK_CUDA(cudaMemcpyAsync(s_it.ptr, items.data(), items.size() * sizeof(GroupItem),
                                      cudaMemcpyHostToDevice, stream));
        if (kGroupTc)
          group_assign_tc_kernel<<<(unsigned)items.size(), kGaWarps * 32, 0, stream>>>(
              d_X, d, rows_b, d_offs, s_it.as<GroupItem>(), s_rank.as<int32_t>(),
              s_tab.as<float>(), s_k.as<uint64_t>(), s_v.as<int64_t>());
        else
          group_assign_kernel<<<(unsigned)items.size(), 128, 0, stream>>>(
              d_X, d, rows_b, d_offs, s_it.as<GroupItem>(), s_rank.as<int32_t>(),
              s_tab.as<float>(), s_k.as<uint64_t>(), s_v.as<int64_t>());
        BM_CHECK_LAUNCH();
        int bits = 7;
        while (bits < 64 && ((uint64_t)nb_el << 7) >> bits) ++bits;
        BM_TRY(sort_pairs_u64(s_k.as<uint64_t>(), s_v.as<int64_t>(), n_entries, bits, stream));
        BM_TRY(scratch_alloc(s_dir, (size_t)n_rt * 4, stream));
        tseed = s_dir.as<int32_t>();
        tile_seed_kernel<<<grid_for(n_rt, 256), 256, 0, stream>>>(
            et, d_offs, n_rt, s_k.as<uint64_t>(), d_order, min_rows, tseed);
        BM_CHECK_LAUNCH();
      }
      perm_kernel<<<grid_for(P, 256), 256, 0, stream>>>(s_v.as<int64_t>(), d_offs, et, P, ent,
                                                        inv, rows_b, xrow);
      BM_CHECK_LAUNCH();
    }

    trace_mark("setup:grouped", stream);
    // ---- gather rows (fp64, padded order) — the exact engine only
    if (!direct) BM_TRY(scratch_alloc(xg, (size_t)P * d * sizeof(double), stream));
    src = direct ? RowSrc{d_X, xrow} : RowSrc{xg.as<double>(), nullptr};
    // tile centres / radii for the pruning bound; with the tensor-core engine
    // the centres (and the column ranges of the quantisation) come out of the
    // gather itself, the radii out of the quantisation pass
    if (prune) BM_TRY(scratch_alloc(s_geo, (size_t)n_rt * (d + 1) * 8, stream));
    double* cen = prune ? s_geo.as<double>() : nullptr;
    double* rad = prune ? cen + n_rt * d : nullptr;
    Scratch s_mm;
    if (use_tc && prune) {
      BM_TRY(scratch_alloc(s_mm, (size_t)n_rt * d * 16, stream));
      if (direct)
        tile_stats_kernel<<<(unsigned)n_rt, kTile, 0, stream>>>(
            d_X, d, xrow, s_mm.as<double>(), s_mm.as<double>() + n_rt * d, cen);
      else
        gather_tiles_kernel<<<(unsigned)n_rt, 256, 0, stream>>>(
            d_X, d, rows_b, et, xg.as<double>(), s_mm.as<double>(), s_mm.as<double>() + n_rt * d,
            cen);
      BM_CHECK_LAUNCH();
    } else if (!direct) {
      gather_kernel<<<grid_for(P, 8, 64), 256, 0, stream>>>(d_X, d, rows_b, et, P,
                                                            xg.as<double>());
      BM_CHECK_LAUNCH();
    }

    // ---- per-row work arrays (counts accumulate over the adjacency windows)
    const size_t wbytes = (size_t)P * (4 + 1 + 4 + 4 + 4 + 4 + 4) + (size_t)(P + 1) * 8 + 64;
    BM_TRY(scratch_alloc(work, wbytes, stream));
    cnt = work.as<int32_t>();
    par = cnt + P;
    bmin = par + P;
    lab = bmin + P;
    cmin = lab + P;
    head = cmin + P;
    hscan = (int64_t*)(((uintptr_t)(head + P) + 15) & ~(uintptr_t)15);
    core = (uint8_t*)(hscan + P + 1);
    BM_CHECK_CUDA(cudaMemsetAsync(cnt, 0, P * 4, stream));
    BM_CHECK_CUDA(cudaMemsetAsync(cmin, 0x7f, P * 4, stream));
    trace_mark("setup:gathered", stream);
    if (use_tc) {
      const double* tmm = s_mm.ptr ? s_mm.as<double>() : nullptr;
      BM_TRY(tc_prepare(src, d, et, P, eps, nrows, stream, &tc, cen, rad, tmm));
      tc_set_queue_scale(tc, qscale);
      tc_set_min_pts(tc, min_pts);
    }

    // ---- kept tile pairs and work units (device-built)
    trace_mark("setup:quantised", stream);
    BM_TRY(build_tiles(d_tbase, prune));
    trace_mark("setup:tiles", stream);
    s_geo.release();
    stats[3] += n_tp;
    stats[2] += n_tp - n_kept;
    return BM_OK;
  }

  int build_tiles(const int32_t* d_tbase, bool prune) {
    std::vector<int32_t> row_elem(n_rt);
    std::vector<PruneBlock> blocks;
    for (int64_t i = 0; i < nb_el; ++i) {
      for (int32_t t = 0; t < ntiles[i]; ++t) row_elem[tbase[i] + t] = (int32_t)i;
      const int32_t nbk = (int32_t)ceil_div(ntiles[i], kPruneB);
      for (int32_t bi = 0; bi < nbk; ++bi)
        for (int32_t bj = bi; bj < nbk; ++bj) blocks.push_back({(int32_t)i, bi, bj, 0});
    }
    Scratch s_re, s_rows;
    BM_TRY(scratch_alloc(s_re, n_rt * 4, stream));
    BM_CHECK_CUDA(cudaMemcpyAsync(s_re.ptr, row_elem.data(), n_rt * 4, cudaMemcpyHostToDevice, stream));
    BM_TRY(big_scratch(b_flags, (size_t)std::max<int64_t>(n_tp, 1) * 4, stream));
    int32_t* flags = b_flags.as<int32_t>();
    if (prune) {
      Scratch s_blk;
      double* cen = s_geo.as<double>();
      double* rad = cen + n_rt * d;
      if (!use_tc) {
        tile_geom_kernel<<<(unsigned)n_rt, 256, 0, stream>>>(xg.as<double>(), d, et,
                                                             s_re.as<int32_t>(), cen, rad);
        BM_CHECK_LAUNCH();
      }
      const int64_t nblk = (int64_t)blocks.size();
      BM_TRY(scratch_alloc(s_blk, (size_t)nblk * sizeof(PruneBlock), stream));
      BM_CHECK_CUDA(cudaMemcpyAsync(s_blk.ptr, blocks.data(), nblk * sizeof(PruneBlock),
                                    cudaMemcpyHostToDevice, stream));
      const double gamma = ((double)d + 16.0) * 1.5 * 1.1102230246251565e-16;
      Scratch s_proj;
      double* proj = nullptr;
      if (tseed) {
        BM_TRY(scratch_alloc(s_proj, (size_t)n_rt * kGroupSeeds * 8, stream));
        proj = s_proj.as<double>();
        if (direct) {
          BM_TRY(tc_tile_project(tc, et, tseed, seeds_q, seed_dist, proj, stream));
        } else {
          tile_project_kernel<<<(unsigned)n_rt, 256, 0, stream>>>(
              xg.as<double>(), d, et, n_rt, tseed, seed_f, seed_norm, cen, rad, proj);
          BM_CHECK_LAUNCH();
        }
      }
      for (int64_t b0 = 0; b0 < nblk; b0 += (1ll << 30)) {
        const int64_t nb = std::min<int64_t>(1ll << 30, nblk - b0);
        tile_prune_kernel<<<(unsigned)nb, 256, 0, stream>>>(
            et, d, d_tbase, s_blk.as<PruneBlock>() + b0, cen, rad, eps, gamma, tseed, proj,
            seed_dist, flags);
        BM_CHECK_LAUNCH();
      }
    } else {
      fill_ones_kernel<<<grid_for(n_tp, 256), 256, 0, stream>>>(flags, n_tp);
      BM_CHECK_LAUNCH();
    }
    BM_TRY(big_scratch(b_pos, (size_t)(n_tp + 1) * 8, stream));
    int64_t* pos = b_pos.as<int64_t>();
    BM_TRY(exclusive_scan_i32_to_i64(flags, pos, n_tp, stream));
    fill_total_kernel<<<1, 1, 0, stream>>>(pos, flags, n_tp);  // pos[n_tp] = n_kept
    BM_CHECK_LAUNCH();
    // capacity for every tile pair: the list is built before its length is
    // known on the host (one synchronisation for all row tables below)
    BM_TRY(big_scratch(s_tiles, (size_t)std::max<int64_t>(n_tp, 1) * sizeof(TileRef), stream));
    d_tiles = s_tiles.as<TileRef>();
    // row tables: first slot, pairs, unit positions (exclusive scans)
    BM_TRY(scratch_alloc(s_rows, (size_t)(n_rt + 1) * 8 * 6, stream));
    int64_t* d_first = s_rows.as<int64_t>();
    int64_t* d_pairs = d_first + (n_rt + 1);
    int64_t* d_noff = d_pairs + (n_rt + 1);
    int64_t* d_ntc = d_noff + (n_rt + 1);
    int64_t* d_offp = d_ntc + (n_rt + 1);
    int64_t* d_tcp = d_offp + (n_rt + 1);
    emit_tiles_kernel<<<grid_for(n_rt, 8, 32), 256, 0, stream>>>(
        et, s_re.as<int32_t>(), d_tbase, n_rt, flags, pos, d_tiles, d_first, d_pairs);
    BM_CHECK_LAUNCH();
    BM_CHECK_CUDA(cudaMemcpyAsync(d_first + n_rt, pos + n_tp, 8, cudaMemcpyDeviceToDevice, stream));
    unit_counts_kernel<<<grid_for(n_rt, 256), 256, 0, stream>>>(d_first, n_rt, d_noff, d_ntc);
    BM_CHECK_LAUNCH();
    // exclusive scans over n_rt + 1 entries: entry n_rt of the output is the
    // total (input entry n_rt is never read into it)
    BM_TRY(exclusive_scan_i64(d_noff, d_offp, n_rt + 1, stream));
    BM_TRY(exclusive_scan_i64(d_ntc, d_tcp, n_rt + 1, stream));
    row_first.resize(n_rt + 1);
    row_pairs.resize(n_rt + 1);
    off_pos.resize(n_rt + 1);
    tc_pos.resize(n_rt + 1);
    BM_CHECK_CUDA(cudaMemcpyAsync(row_first.data(), d_first, (n_rt + 1) * 8, cudaMemcpyDeviceToHost, stream));
    BM_CHECK_CUDA(cudaMemcpyAsync(row_pairs.data(), d_pairs, n_rt * 8, cudaMemcpyDeviceToHost, stream));
    BM_CHECK_CUDA(cudaMemcpyAsync(off_pos.data(), d_offp, (n_rt + 1) * 8, cudaMemcpyDeviceToHost, stream));
    BM_CHECK_CUDA(cudaMemcpyAsync(tc_pos.data(), d_tcp, (n_rt + 1) * 8, cudaMemcpyDeviceToHost, stream));
    BM_CHECK_CUDA(cudaStreamSynchronize(stream));
    n_kept = row_first[n_rt];
    BM_REQUIRE(n_kept < (1ll << 31), "too many tile pairs (%lld)", (long long)n_kept);
    const int64_t n_off_u = off_pos[n_rt], n_tc_u = tc_pos[n_rt];
    BM_TRY(scratch_alloc(s_units, (size_t)(n_rt + n_off_u + n_tc_u + 1) * sizeof(TileUnit), stream));
    d_diag = s_units.as<TileUnit>();
    d_off = d_diag + n_rt;
    d_tcu = d_off + n_off_u;
    emit_units_kernel<<<grid_for(n_rt, 256), 256, 0, stream>>>(
        s_re.as<int32_t>(), d_tbase, n_rt, d_first, d_offp, d_tcp, d_diag, d_off, d_tcu);
    BM_CHECK_LAUNCH();
    return BM_OK;
  }

  // kept slots [s0, s1) and row tiles [r0, r1) of the tile rows [I0, I1) of
  // element 0 (I0 < 0: the whole batch)
  void rows_of(int32_t I0, int32_t I1, int64_t& r0, int64_t& r1) const {
    if (I0 < 0) {
      r0 = 0;
      r1 = n_rt;
    } else {
      r0 = tbase[0] + I0;
      r1 = tbase[0] + I1;
    }
  }

  // device views of the window's tiles and work units (no copies: the
  // window is a contiguous run of rows, hence of slots and of every unit list)
  int window(int32_t I0, int32_t I1, WindowBufs& w) {
    if (I0 >= 0)
      BM_REQUIRE(nb_el == 1 && I0 < I1 && I1 <= ntiles[0], "bad row window [%d, %d)", I0, I1);
    int64_t r0 = 0, r1 = 0;
    rows_of(I0, I1, r0, r1);
    w.slot0 = row_first[r0];
    w.n_tiles = row_first[r1] - row_first[r0];
    w.tiles = d_tiles;
    w.diag = d_diag + r0;
    w.n_diag = r1 - r0;
    w.off = d_off + off_pos[r0];
    w.n_off = off_pos[r1] - off_pos[r0];
    w.tcu = d_tcu + tc_pos[r0];
    w.n_tc = tc_pos[r1] - tc_pos[r0];
    w.pairs = 0;
    for (int64_t r = r0; r < r1; ++r) w.pairs += row_pairs[r];
    return BM_OK;
  }

  // Bits of the window into adj; counts added into cnt_acc (nullptr: the
  // counts of this window were already taken).
  int adjacency(int32_t I0, int32_t I1, uint32_t* adj, int32_t* cnt_acc, int64_t* stats) {
    WindowBufs w;
    BM_TRY(window(I0, I1, w));
    int32_t* nonempty = reinterpret_cast<int32_t*>(adj + w.n_tiles * kTileWords);
    if (use_tc) {
      // windows (huge elements, row blocks) check the recheck queue at once so
      // that their counts accumulate exactly once; a whole batch defers it
      BM_TRY(tc_window(tc, src, et, w.tiles, w.slot0, w.n_tiles, w.tcu, w.n_tc,
                       w.pairs, adj, nonempty, cnt_acc, I0 >= 0, I0 >= 0, stats, stream));
    } else {
      BM_TRY(exact_build_adjacency(xg.as<double>(), d, et, w.tiles + w.slot0, w.n_tiles, eps,
                                   adj, nonempty, stream));
      if (cnt_acc) {
        if (w.n_diag > 0) {
          count_kernel<<<grid_for(w.n_diag, 1, 32), 128, 0, stream>>>(
              adj, et, w.diag, w.tiles, w.slot0, w.n_diag, cnt_acc);
          BM_CHECK_LAUNCH();
        }
        if (w.n_off > 0) {
          count_kernel<<<grid_for(w.n_off, 1, 32), 128, 0, stream>>>(
              adj, et, w.off, w.tiles, w.slot0, w.n_off, cnt_acc);
          BM_CHECK_LAUNCH();
        }
      }
      stats[0] += w.pairs;
    }
    stats[4] = std::max<int64_t>(stats[4], w.n_tiles * kTileWords * 4);
    return BM_OK;
  }

  int init_core(const int32_t* counts, int32_t* par_out, int32_t* bmin_out) {
    core_init_kernel<<<grid_for(P, 256), 256, 0, stream>>>(counts, et, P, min_pts, core, par_out,
                                                           bmin_out);
    BM_CHECK_LAUNCH();
    return BM_OK;
  }

  // union-find over the core-core bits and border minima of the window
  // (adj: the window's bitmap followed by its per-slot nonempty flags)
  int components(int32_t I0, int32_t I1, uint32_t* adj, int32_t* par_w, int32_t* bmin_w) {
    WindowBufs w;
    BM_TRY(window(I0, I1, w));
    int32_t* nonempty = reinterpret_cast<int32_t*>(adj + w.n_tiles * kTileWords);
    if (w.n_diag > 0 && check_symmetry()) {
      Scratch s_bad;
      BM_TRY(scratch_alloc(s_bad, 8, stream));
      BM_CHECK_CUDA(cudaMemsetAsync(s_bad.ptr, 0, 8, stream));
      diag_symmetry_kernel<<<grid_for(w.n_diag, 1, 32), 128, 0, stream>>>(
          adj, w.diag, w.tiles, w.slot0, w.n_diag, s_bad.as<unsigned long long>());
      BM_CHECK_LAUNCH();
      unsigned long long h_bad = 0;
      BM_CHECK_CUDA(cudaMemcpyAsync(&h_bad, s_bad.ptr, 8, cudaMemcpyDeviceToHost, stream));
      BM_CHECK_CUDA(cudaStreamSynchronize(stream));
      BM_REQUIRE_INTERNAL(h_bad == 0, "asymmetric diagonal tile bitmap (%llu bits)", h_bad);
    }
    if (w.n_diag > 0) {
      if (kDiagBfs)
        diag_bfs_kernel<<<grid_for(w.n_diag, 1, 32), 128, 0, stream>>>(
            adj, et, w.diag, w.tiles, w.slot0, w.n_diag, core, par_w, bmin_w);
      else
        components_kernel<true><<<grid_for(w.n_diag, 1, 32), 128, 0, stream>>>(
            adj, et, w.diag, w.tiles, w.slot0, w.n_diag, core, par_w, bmin_w, nullptr, nonempty, 0,
            1 << 30);
      BM_CHECK_LAUNCH();
    }
    compress_kernel<<<grid_for(P, 256), 256, 0, stream>>>(par_w, core, P);
    BM_CHECK_LAUNCH();
    if (w.n_off > 0) {
      Scratch s_uni;
      BM_TRY(scratch_alloc(s_uni, (size_t)n_rt * 4, stream));
      tile_uniform_kernel<<<grid_for(n_rt, 8, 32), 256, 0, stream>>>(et, n_rt, core, par_w,
                                                                     s_uni.as<int32_t>());
      BM_CHECK_LAUNCH();
#ifdef BM_COMP_STATS
      {
        unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        BM_CHECK_CUDA(cudaMemcpyToSymbolAsync(g_comp_stats, z, sizeof(z), 0,
                                              cudaMemcpyHostToDevice, stream));
      }
#endif
      // two phases: the first 6 tile pairs of every unit (its nearest kept
      // column tiles) join most of each cluster's tiles; after a compression
      // the remaining pairs mostly see one root per tile side and take the
      // one-union path instead of walking their bits (cfg3: 1.04 -> 0.84 ms)
      for (int phase = 0; phase < kCompPhases; ++phase) {
        if (phase > 0) {
          compress_kernel<<<grid_for(P, 256), 256, 0, stream>>>(par_w, core, P);
          BM_CHECK_LAUNCH();
          tile_uniform_kernel<<<grid_for(n_rt, 8, 32), 256, 0, stream>>>(et, n_rt, core, par_w,
                                                                         s_uni.as<int32_t>());
          BM_CHECK_LAUNCH();
        }
        components_kernel<false><<<grid_for(w.n_off, 1, 32), 128, 0, stream>>>(
            adj, et, w.off, w.tiles, w.slot0, w.n_off, core, par_w, bmin_w, s_uni.as<int32_t>(),
            nonempty, kCompCuts[phase], kCompCuts[phase + 1]);
        BM_CHECK_LAUNCH();
      }
#ifdef BM_COMP_STATS
      {
        unsigned long long h[8];
        BM_CHECK_CUDA(cudaMemcpyFromSymbolAsync(h, g_comp_stats, sizeof(h), 0,
                                                cudaMemcpyDeviceToHost, stream));
        BM_CHECK_CUDA(cudaStreamSynchronize(stream));
        std::vector<int32_t> hu(n_rt);
        BM_CHECK_CUDA(cudaMemcpy(hu.data(), s_uni.ptr, n_rt * 4, cudaMemcpyDeviceToHost));
        int64_t nu = 0;
        for (auto v : hu) nu += v >= 0;
        fprintf(stderr, "[comp-stats] off-diag tiles %llu: empty %llu, both-uniform %llu, "
                "rmm-uniform %llu, full %llu, merged %llu; uniform row tiles %lld / %lld\n",
                h[0], h[1], h[2], h[3], h[4], h[5], (long long)nu, (long long)n_rt);
      }
#endif
    }
    return BM_OK;
  }

  // bytes of the bitmap of the row tiles [I0, I1) (all: I0 < 0)
  size_t window_bytes(int32_t I0, int32_t I1) const {
    int64_t r0 = 0, r1 = 0;
    rows_of(I0, I1, r0, r1);
    return (size_t)std::max<int64_t>(row_first[r1] - row_first[r0], 1) * (kTileWords * 4 + 4);
  }

  // canonical labels of every entry (element-relative cluster ids, -1 noise)
  int finish(int32_t* par_w, const int32_t* bmin_w, int32_t* d_out, int32_t* h_ncl) {
    label_kernel<<<grid_for(P, 256), 256, 0, stream>>>(et, P, core, par_w, bmin_w, inv, lab, cmin);
    BM_CHECK_LAUNCH();
    head_kernel<<<grid_for(n_entries, 256), 256, 0, stream>>>(n_entries, inv, lab, cmin, head);
    BM_CHECK_LAUNCH();
    BM_TRY(exclusive_scan_i32_to_i64(head, hscan, n_entries, stream));
    fill_total_kernel<<<1, 1, 0, stream>>>(hscan, head, n_entries);  // hscan[n] = #heads
    BM_CHECK_LAUNCH();
    Scratch ncl_d;
    BM_TRY(scratch_alloc(ncl_d, nb_el * 4, stream));
    nclusters_kernel<<<(unsigned)ceil_div(nb_el, 128), 128, 0, stream>>>(et, d_offs, hscan,
                                                                          ncl_d.as<int32_t>());
    BM_CHECK_LAUNCH();
    output_kernel<<<grid_for(n_entries, 256), 256, 0, stream>>>(et, d_offs, n_entries, inv, lab,
                                                                cmin, hscan, d_out);
    BM_CHECK_LAUNCH();
    BM_CHECK_CUDA(cudaMemcpyAsync(h_ncl, ncl_d.ptr, nb_el * 4, cudaMemcpyDeviceToHost, stream));
    BM_CHECK_CUDA(cudaStreamSynchronize(stream));
    return BM_OK;
  }
};

// Row windows of element 0 holding at most max_tiles kept tiles each (every
// window has at least one tile row), in ascending row order. Built from the
// bottom so that the LAST window — the one whose bits stay resident between
// the two passes — is the full one and the recomputed remainder is as small
// as possible.
std::vector<std::pair<int32_t, int32_t>> row_windows(const BatchCtx& bc, int64_t max_tiles) {
  const int64_t T = bc.ntiles[0];
  auto first = [&](int64_t I) { return bc.row_first[bc.tbase[0] + I]; };
  // first(I) = slot of row I's diagonal; rows [I, I1) hold first(I1) - first(I) tiles
  std::vector<std::pair<int32_t, int32_t>> w;
  int64_t I1 = T;
  while (I1 > 0) {
    int64_t I = I1 - 1;
    while (I > 0 && first(I1) - first(I - 1) <= max_tiles) --I;
    w.push_back({(int32_t)I, (int32_t)I1});
    I1 = I;
  }
  std::reverse(w.begin(), w.end());
  return w;
}

int64_t row_window_cap() {
  // B200MAP_WINDOW_TILES forces small windows (tests of the row-block path)
  const char* e = getenv("B200MAP_WINDOW_TILES");
  return e ? std::max<int64_t>(1, atoll(e)) : 0;
}

// bytes per kept tile besides its bitmap: tile ref, thresholds, recheck queue
constexpr double kTileAux = 16.0 + 24.0 + 16.0 * 16384.0 / 2000.0;

}  // namespace bm

using namespace bm;

extern "C" int bm_cluster_elements(const double* d_X, int64_t n, int64_t d,
                                   const int64_t* d_rows, const int64_t* h_offsets,
                                   int64_t n_el, double eps, int32_t min_pts,
                                   const uint8_t* h_order, int engine, int32_t* d_labels,
                                   int32_t* h_n_clusters, int64_t* h_stats, void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  trace_mark("cluster:entry", stream);
  BM_REQUIRE(n >= 0 && d >= 1 && n_el >= 0, "bad shapes");
  BM_REQUIRE(eps > 0.0, "eps must be positive");
  BM_REQUIRE(min_pts >= 1, "min-pts must be >= 1");
  BM_REQUIRE(h_offsets && h_n_clusters && h_order, "null host table");
  BM_REQUIRE(engine == BM_ENGINE_AUTO || engine == BM_ENGINE_EXACT || engine == BM_ENGINE_TC,
             "unknown engine %d", engine);
  int64_t stats_local[8] = {0};
  int64_t* stats = h_stats ? h_stats : stats_local;
  for (int i = 0; i < 8; ++i) stats[i] = 0;
  for (int64_t k = 0; k < n_el; ++k) h_n_clusters[k] = 0;
  if (n_el == 0) return BM_OK;
  for (int64_t k = 0; k < n_el; ++k) {
    BM_REQUIRE(h_offsets[k + 1] >= h_offsets[k], "offsets must be non-decreasing");
    BM_REQUIRE(h_order[k] == BM_ORDER_SEQUENTIAL || h_order[k] == BM_ORDER_PAIRWISE,
               "bad order flag");
  }
  if (h_offsets[n_el] == h_offsets[0]) return BM_OK;
  BM_REQUIRE(d_X && d_rows && d_labels, "null device pointer");
  BM_REQUIRE(h_offsets[n_el] - h_offsets[0] < (1ll << 31), "too many membership entries");
  BM_REQUIRE(n < (1ll << 31), "more than 2^31 - 1 points");
  PwProgram probe;
  BM_TRY(make_pw_program(d, &probe));

  bool use_tc = false;
  if (engine == BM_ENGINE_TC) {
    BM_REQUIRE(tc_supported(d), "tensor-core engine does not support d=%lld", (long long)d);
    use_tc = true;
  } else if (engine == BM_ENGINE_AUTO) {
    use_tc = tc_supported(d);
  }
  // outside the error model every tensor-core decision would be queued for
  // the exact recheck: run the exact engine directly (same bits)
  if (!eps_in_model(eps)) use_tc = false;

  // ---- batches bounded by the device budget (dense bitmap estimate); an
  //      element whose dense bitmap alone exceeds it is processed by itself in
  //      row windows sized on its kept tiles
  // free memory is queried only when the work could come near it: the query
  // (cudaMemGetInfo + pool attributes) intermittently stalls for tens of ms
  const int64_t forced_cap = row_window_cap();
  double need = 0.0;
  for (int64_t k = 0; k < n_el; ++k) {
    const int64_t T = ceil_div(h_offsets[k + 1] - h_offsets[k], kTile);
    need += (double)(T * (T + 1) / 2) * (kTileWords * 4 + kTileAux) +
            (double)T * kTile * (d * 8.0 + 4 * 9 + 1 + 24 + d * 3.0);
  }
  size_t free_b = device_total_bytes();
  if (need > 0.2 * (double)free_b || forced_cap > 0) BM_TRY(device_free_bytes(&free_b));
  const double budget = 0.55 * (double)free_b;
  struct Batch {
    int64_t k0, k1;
    bool windowed;  // single huge element in row windows
  };
  std::vector<Batch> batches;
  {
    int64_t k0 = 0;
    double acc = 0;
    for (int64_t k = 0; k < n_el; ++k) {
      const int64_t nk = h_offsets[k + 1] - h_offsets[k];
      const int64_t T = ceil_div(nk, kTile);
      BM_REQUIRE(T * kTile < (1ll << 31), "element %lld too large", (long long)k);
      const double row_bytes = (double)T * kTile * (d * 8.0 + 4 * 9 + 1 + 24 + d * 3.0);
      const double bytes = (double)(T * (T + 1) / 2) * (kTileWords * 4 + kTileAux) + row_bytes;
      if (bytes > budget || (forced_cap > 0 && T * (T + 1) / 2 > forced_cap)) {
        if (k > k0) batches.push_back({k0, k, false});
        batches.push_back({k, k + 1, true});
        k0 = k + 1;
        acc = 0;
        continue;
      }
      if (acc + bytes > budget && k > k0) {
        batches.push_back({k0, k, false});
        k0 = k;
        acc = 0;
      }
      acc += bytes;
    }
    if (k0 < n_el) batches.push_back({k0, n_el, false});
  }

  for (const Batch& bt : batches) {
    cudaEvent_t evs = nullptr, ev0 = nullptr, ev1 = nullptr, ev2 = nullptr;
    BM_CHECK_CUDA(cudaEventCreate(&evs));
    BM_CHECK_CUDA(cudaEventCreate(&ev0));
    BM_CHECK_CUDA(cudaEventCreate(&ev1));
    BM_CHECK_CUDA(cudaEventCreate(&ev2));
    struct EvGuard {
      cudaEvent_t* e[4];
      ~EvGuard() {
        for (auto p : e) cudaEventDestroy(*p);
      }
    } evg{{&evs, &ev0, &ev1, &ev2}};
    // a batch whose deferred recheck-queue check overflows is rerun with a
    // larger queue (rare: the capacity is ~10x the typical need)
    int64_t bst[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    bool empty = false;
    for (int attempt = 0;; ++attempt) {
      for (auto& v : bst) v = 0;
      BM_CHECK_CUDA(cudaEventRecord(evs, stream));
      trace_mark("batch:start", stream);
      BatchCtx bc;
      bc.stream = stream;
      bc.d = d;
      bc.eps = eps;
      bc.min_pts = min_pts;
      bc.use_tc = use_tc;
      // (the last attempt holds every pair of the window)
      bc.qscale = attempt == 0 ? 1.0 : (attempt == 1 ? 8.0 : 2000.0);
      BM_TRY(bc.setup(d_X, d_rows, h_offsets, h_order, bt.k0, bt.k1, bst));
      if (bc.n_entries == 0) {
        empty = true;
        break;
      }
      int32_t* d_out = d_labels + h_offsets[bt.k0];
      std::vector<std::pair<int32_t, int32_t>> wins;
      if (bt.windowed) {
        // the window plan is a function of the device size (not of the free
        // memory of the moment), so repeated calls reuse the cached bitmap
        // buffer: at most 45% of the device, less if it is not free
        size_t free_now = 0;
        BM_TRY(device_free_bytes(&free_now));
        const double avail = std::min(0.45 * (double)device_total_bytes(),
                                      0.85 * (double)free_now - (double)(2ll << 30));
        int64_t cap = (int64_t)(avail / (kTileWords * 4.0 + kTileAux));
        if (forced_cap > 0) cap = forced_cap;  // windows still hold >= 1 tile row
        wins = row_windows(bc, std::max<int64_t>(cap, 1));
      } else {
        wins.push_back({-1, -1});
      }
      size_t max_w = 0;
      for (auto& w : wins) max_w = std::max(max_w, bc.window_bytes(w.first, w.second));
      // the bitmap: a cached buffer (released after finish() synchronised)
      BigScratch adj;
      BM_TRY(big_scratch(adj, max_w, stream));
      trace_mark("batch:bitmap allocated", stream);
      BM_CHECK_CUDA(cudaEventRecord(ev0, stream));
      // pass 1: counts of every window (the last window's bits stay resident);
      // pass 2: components of the resident window, then of the others with
      // their bits recomputed (bit-identical: the decision is a pure function
      // of the pair)
      for (auto& w : wins)
        BM_TRY(bc.adjacency(w.first, w.second, adj.as<uint32_t>(), bc.cnt, bst));
      trace_mark("adjacency", stream);
      BM_CHECK_CUDA(cudaEventRecord(ev1, stream));
      BM_TRY(bc.init_core(bc.cnt, bc.par, bc.bmin));
      for (size_t i = wins.size(); i-- > 0;) {
        if (i + 1 != wins.size())
          BM_TRY(bc.adjacency(wins[i].first, wins[i].second, adj.as<uint32_t>(), nullptr, bst));
        BM_TRY(bc.components(wins[i].first, wins[i].second, adj.as<uint32_t>(), bc.par, bc.bmin));
      }
      trace_mark("components", stream);
      BM_TRY(bc.finish(bc.par, bc.bmin, d_out, h_n_clusters + bt.k0));  // synchronises
      trace_mark("finished", stream);
      BM_CHECK_CUDA(cudaEventRecord(ev2, stream));
      bool overflow = false;
      if (bc.tc) BM_TRY(tc_collect(bc.tc, &bst[1], &overflow, stream));
      if (!overflow) break;
      if (attempt == 2) {
        set_error("recheck queue overflow");
        return BM_ERR_INTERNAL;
      }
    }
    if (empty) continue;
    for (int i = 0; i < 5; ++i) stats[i] = i == 4 ? std::max(stats[4], bst[4]) : stats[i] + bst[i];
    float ms = 0.f, ms_pre = 0.f, ms_post = 0.f;
    BM_CHECK_CUDA(cudaEventSynchronize(ev2));
    BM_CHECK_CUDA(cudaEventElapsedTime(&ms, ev0, ev1));
    BM_CHECK_CUDA(cudaEventElapsedTime(&ms_pre, evs, ev0));
    BM_CHECK_CUDA(cudaEventElapsedTime(&ms_post, ev1, ev2));
    stats[5] += (int64_t)(ms * 1e6);       // adjacency (distance) stage, ns on the launch stream
    stats[6] += (int64_t)(ms_pre * 1e6);   // grouping, gather, quantisation, pruning
    stats[7] += (int64_t)(ms_post * 1e6);  // core, union-find, border, relabel (+ recomputed windows)
  }
  trace_mark("cluster:return", stream);
  trace_dump();
  return BM_OK;
}

// ---------------------------------------------------------------------------
// Row-block protocol for one huge element sharded over ranks:
// every rank opens the element, takes the counts of its row windows,
// all-reduce(sum) of counts, core + forest init, union-find of its windows,
// forests merged on rank 0 (bm_merge_forest), all-reduce(min) of border
// minima, labels on rank 0. The collectives stay in the host (NCCL through
// torch.distributed); these entry points are the per-rank compute steps.
// ---------------------------------------------------------------------------
namespace bm {
namespace {

struct BigElement {
  BatchCtx bc;
  Scratch adj;
  size_t adj_bytes = 0;
  int32_t w0 = -1, w1 = -1;  // window whose bits are resident in adj
  int64_t stats[8] = {0, 0, 0, 0, 0, 0, 0, 0};

  int bits(int32_t I0, int32_t I1, int32_t* cnt_acc) {
    BM_REQUIRE(I0 >= 0 && I0 < I1 && I1 <= bc.ntiles[0], "bad row window [%d, %d)", I0, I1);
    const size_t need = bc.window_bytes(I0, I1);
    if (need > adj_bytes) {
      BM_TRY(scratch_alloc(adj, need, bc.stream));
      adj_bytes = need;
    }
    w0 = w1 = -1;
    BM_TRY(bc.adjacency(I0, I1, adj.as<uint32_t>(), cnt_acc, stats));
    w0 = I0;
    w1 = I1;
    return BM_OK;
  }
};

__global__ void merge_forest_kernel(int32_t* __restrict__ par, const int32_t* __restrict__ other,
                                    int64_t n) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int q = __ldg(other + p);
    if (q != (int)p) uf_union(par, (int)p, q);
  }
}

}  // namespace
}  // namespace bm

extern "C" int bm_big_open(const double* d_X, int64_t n, int64_t d, const int64_t* d_rows,
                           int64_t n_rows, double eps, int32_t min_pts, int order, int engine,
                           void* stream, void** handle, int64_t* h_tiles) {
  BM_REQUIRE(handle && h_tiles, "null output");
  *handle = nullptr;
  BM_REQUIRE(n >= 0 && n < (1ll << 31) && d >= 1 && n_rows >= 1, "bad shapes");
  BM_REQUIRE(d_X && d_rows, "null device pointer");
  BM_REQUIRE(eps > 0.0, "eps must be positive");
  BM_REQUIRE(min_pts >= 1, "min-pts must be >= 1");
  BM_REQUIRE(order == BM_ORDER_SEQUENTIAL || order == BM_ORDER_PAIRWISE, "bad order flag");
  BM_REQUIRE(engine == BM_ENGINE_AUTO || engine == BM_ENGINE_EXACT || engine == BM_ENGINE_TC,
             "unknown engine %d", engine);
  BM_REQUIRE(ceil_div(n_rows, kTile) * kTile < (1ll << 31), "element too large");
  PwProgram probe;
  BM_TRY(make_pw_program(d, &probe));
  bool use_tc = engine == BM_ENGINE_TC || (engine == BM_ENGINE_AUTO && tc_supported(d));
  BM_REQUIRE(!use_tc || tc_supported(d), "tensor-core engine does not support d=%lld",
             (long long)d);
  if (!eps_in_model(eps)) use_tc = false;  // see bm_cluster_elements
  BigElement* be = new BigElement();
  be->bc.stream = (cudaStream_t)stream;
  be->bc.d = d;
  be->bc.eps = eps;
  be->bc.min_pts = min_pts;
  be->bc.use_tc = use_tc;
  const int64_t offs[2] = {0, n_rows};
  const uint8_t ord = (uint8_t)order;
  const int rc = be->bc.setup(d_X, d_rows, offs, &ord, 0, 1, be->stats);
  if (rc != BM_OK) {
    delete be;
    return rc;
  }
  *handle = be;
  *h_tiles = be->bc.ntiles[0];
  return BM_OK;
}

extern "C" int bm_big_counts(void* handle, int32_t I0, int32_t I1, int32_t* d_cnt) {
  BM_REQUIRE(handle && d_cnt, "null argument");
  return static_cast<BigElement*>(handle)->bits(I0, I1, d_cnt);
}

extern "C" int bm_big_init(void* handle, const int32_t* d_cnt, int32_t* d_par, int32_t* d_bmin) {
  BM_REQUIRE(handle && d_cnt && d_par && d_bmin, "null argument");
  return static_cast<BigElement*>(handle)->bc.init_core(d_cnt, d_par, d_bmin);
}

extern "C" int bm_big_components(void* handle, int32_t I0, int32_t I1, int32_t* d_par,
                                 int32_t* d_bmin) {
  BM_REQUIRE(handle && d_par && d_bmin, "null argument");
  BigElement* be = static_cast<BigElement*>(handle);
  if (be->w0 != I0 || be->w1 != I1) BM_TRY(be->bits(I0, I1, nullptr));
  return be->bc.components(I0, I1, be->adj.as<uint32_t>(), d_par, d_bmin);
}

extern "C" int bm_big_labels(void* handle, int32_t* d_par, const int32_t* d_bmin,
                             int32_t* d_labels, int32_t* h_n_clusters) {
  BM_REQUIRE(handle && d_par && d_bmin && d_labels && h_n_clusters, "null argument");
  BigElement* be = static_cast<BigElement*>(handle);
  return be->bc.finish(d_par, d_bmin, d_labels, h_n_clusters);
}

extern "C" int bm_big_stats(void* handle, int64_t* h_stats) {
  BM_REQUIRE(handle && h_stats, "null argument");
  BigElement* be = static_cast<BigElement*>(handle);
  for (int i = 0; i < 8; ++i) h_stats[i] = be->stats[i];
  if (be->bc.tc) {
    bool overflow = false;  // windows check their queue synchronously
    BM_TRY(tc_collect(be->bc.tc, &h_stats[1], &overflow, be->bc.stream));
  }
  return BM_OK;
}

extern "C" int bm_big_row_tiles(void* handle, int64_t* h_row_first) {
  BM_REQUIRE(handle && h_row_first, "null argument");
  const BatchCtx& bc = static_cast<BigElement*>(handle)->bc;
  const int64_t T = bc.ntiles[0];
  for (int64_t I = 0; I <= T; ++I)
    h_row_first[I] = bc.row_first[bc.tbase[0] + I] - bc.row_first[bc.tbase[0]];
  return BM_OK;
}

extern "C" int bm_element_work(const double* d_X, int64_t n, int64_t d, const int64_t* d_rows,
                               const int64_t* h_offsets, int64_t n_el, double eps,
                               int64_t* h_kept_tiles, void* stream_) {
  BM_REQUIRE(n >= 0 && d >= 1 && n_el >= 0, "bad shapes");
  BM_REQUIRE(eps > 0.0, "eps must be positive");
  BM_REQUIRE(h_offsets && h_kept_tiles, "null host table");
  for (int64_t k = 0; k < n_el; ++k) {
    BM_REQUIRE(h_offsets[k + 1] >= h_offsets[k], "offsets must be non-decreasing");
    h_kept_tiles[k] = 0;
  }
  if (n_el == 0 || h_offsets[n_el] == h_offsets[0]) return BM_OK;
  BM_REQUIRE(d_X && d_rows, "null device pointer");
  BM_REQUIRE(h_offsets[n_el] - h_offsets[0] < (1ll << 31), "too many membership entries");
  // chunks of elements bounded by the dense tile-pair count (flag and tile
  // lists are sized for every pair of a chunk)
  std::vector<uint8_t> order(n_el, (uint8_t)BM_ORDER_SEQUENTIAL);
  int64_t k0 = 0;
  while (k0 < n_el) {
    int64_t k1 = k0, pairs = 0;
    while (k1 < n_el) {
      const int64_t T = ceil_div(h_offsets[k1 + 1] - h_offsets[k1], kTile);
      if (k1 > k0 && pairs + T * (T + 1) / 2 > (1ll << 27)) break;
      pairs += T * (T + 1) / 2;
      ++k1;
    }
    BatchCtx bc;
    bc.stream = (cudaStream_t)stream_;
    bc.d = d;
    bc.eps = eps;
    bc.min_pts = 1;
    bc.use_tc = false;  // geometry from the gathered rows; no quantisation
    int64_t st[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    BM_TRY(bc.setup(d_X, d_rows, h_offsets, order.data(), k0, k1, st));
    if (bc.n_entries > 0)
      for (int64_t i = 0; i < bc.nb_el; ++i)
        h_kept_tiles[k0 + i] = bc.row_first[bc.tbase[i + 1]] - bc.row_first[bc.tbase[i]];
    k0 = k1;
  }
  return BM_OK;
}

extern "C" int bm_big_close(void* handle) {
  if (handle) {
    BigElement* be = static_cast<BigElement*>(handle);
    cudaStream_t s = be->bc.stream;
    delete be;
    BM_CHECK_CUDA(cudaStreamSynchronize(s));
  }
  return BM_OK;
}

extern "C" int bm_merge_forest(int32_t* d_par, const int32_t* d_other, int64_t n, void* stream) {
  BM_REQUIRE(n >= 0, "bad size");
  if (n == 0) return BM_OK;
  BM_REQUIRE(d_par && d_other, "null device pointer");
  merge_forest_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(d_par, d_other, n);
  BM_CHECK_LAUNCH();
  return BM_OK;
}

extern "C" int bm_pairwise_distances(const double* d_X, int64_t n, int64_t d,
                                     const int64_t* d_rows, int64_t n_rows, int order,
                                     double* d_out, void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  BM_REQUIRE(n >= 0 && d >= 1 && n_rows >= 0, "bad shapes");
  BM_REQUIRE(order == BM_ORDER_SEQUENTIAL || order == BM_ORDER_PAIRWISE, "bad order");
  if (n_rows == 0) return BM_OK;
  BM_REQUIRE(d_X && d_rows && d_out, "null pointer");
  PwProgram prog;
  BM_TRY(make_pw_program(d, &prog));
  pairwise_matrix_kernel<<<grid_for(n_rows * n_rows, 128, 32), 128, 0, stream>>>(
      d_X, d, d_rows, n_rows, order, d_out, prog);
  BM_CHECK_LAUNCH();
  return BM_OK;
}
