// graph.cu — nodes (stable grouping), K7 nerve edges, node payload.
//
// Reference: nervemap/nerve.py:77-114 (build_graph), 60-62 (_node_stats),
// 96 (filter_mean). Node ids are dense in (element, cluster) order; node v's
// rows are ascending. Edges (s,t,w), s<t, w = |rows_s ∩ rows_t| > 0, sorted.
//
// Both grouping and edges are stable LSD radix sorts (8-bit digits) whose
// scatter is one warp per 4096-item chunk processed in order with
// __match_any_sync ranks — stable by construction, no atomics on positions.
#include <algorithm>
#include <vector>

#include "common.cuh"

namespace bm {
namespace {

constexpr int kRChunk = 1024;
constexpr int kRBits = 8;
constexpr int kRBins = 1 << kRBits;

__global__ void radix_hist_kernel(const uint64_t* __restrict__ keys, int64_t n, int shift,
                                  int64_t n_chunks, int64_t* __restrict__ C) {
  __shared__ int h[kRBins];
  for (int i = threadIdx.x; i < kRBins; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const int64_t c = blockIdx.x;
  const int64_t b0 = c * kRChunk, b1 = min(n, b0 + kRChunk);
  for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x)
    atomicAdd(&h[(keys[i] >> shift) & (kRBins - 1)], 1);
  __syncthreads();
  for (int i = threadIdx.x; i < kRBins; i += blockDim.x) C[(int64_t)i * n_chunks + c] = h[i];
}

constexpr int kScatterWarps = 4;

__global__ void radix_scatter_kernel(const uint64_t* __restrict__ kin,
                                     const int64_t* __restrict__ vin, int64_t n, int shift,
                                     int64_t n_chunks, const int64_t* __restrict__ Cscan,
                                     uint64_t* __restrict__ kout, int64_t* __restrict__ vout) {
  __shared__ int64_t cur[kScatterWarps][kRBins];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t c = (int64_t)blockIdx.x * kScatterWarps + w;
  if (c >= n_chunks) return;
  for (int i = lane; i < kRBins; i += 32) cur[w][i] = Cscan[(int64_t)i * n_chunks + c];
  __syncwarp();
  const unsigned lt = (1u << lane) - 1u;
  const int64_t b0 = c * kRChunk, b1 = min(n, b0 + kRChunk);
  for (int64_t base = b0; base < b1; base += 32) {
    const int64_t i = base + lane;
    const bool ok = i < b1;
    uint64_t k = ok ? kin[i] : 0;
    int dg = ok ? (int)((k >> shift) & (kRBins - 1)) : kRBins;
    unsigned peers = __match_any_sync(0xffffffffu, dg);
    if (ok) {
      int leader = __ffs(peers) - 1;
      int64_t bp = 0;
      if (lane == leader) bp = cur[w][dg];
      bp = __shfl_sync(peers, bp, leader);
      int64_t pos = bp + __popc(peers & lt);
      kout[pos] = k;
      if (vin) vout[pos] = vin[i];
      __syncwarp(peers);
      if (lane == leader) cur[w][dg] = bp + __popc(peers);
    }
    __syncwarp();
  }
}

// Stable sort of (keys, vals) by the low `key_bits` bits of keys. Result in
// (keys, vals) (vals may be null).
int radix_sort_pairs(uint64_t* keys, int64_t* vals, int64_t n, int key_bits, cudaStream_t s) {
  if (n <= 1 || key_bits <= 0) return BM_OK;
  const int64_t n_chunks = ceil_div(n, kRChunk);
  Scratch kb, vb, C;
  BM_TRY(scratch_alloc(kb, n * 8, s));
  if (vals) BM_TRY(scratch_alloc(vb, n * 8, s));
  BM_TRY(scratch_alloc(C, (size_t)kRBins * n_chunks * 8, s));
  uint64_t* k0 = keys;
  int64_t* v0 = vals;
  uint64_t* k1 = kb.as<uint64_t>();
  int64_t* v1 = vals ? vb.as<int64_t>() : nullptr;
  int passes = 0;
  for (int shift = 0; shift < key_bits; shift += kRBits, ++passes) {
    radix_hist_kernel<<<(unsigned)n_chunks, 256, 0, s>>>(k0, n, shift, n_chunks, C.as<int64_t>());
    BM_CHECK_LAUNCH();
    BM_TRY(exclusive_scan_i64(C.as<int64_t>(), C.as<int64_t>(), (int64_t)kRBins * n_chunks, s));
    radix_scatter_kernel<<<(unsigned)ceil_div(n_chunks, kScatterWarps), 32 * kScatterWarps, 0, s>>>(
        k0, v0, n, shift, n_chunks, C.as<int64_t>(), k1, v1);
    BM_CHECK_LAUNCH();
    std::swap(k0, k1);
    std::swap(v0, v1);
  }
  if (passes & 1) {  // result lives in the scratch buffers: copy back
    BM_CHECK_CUDA(cudaMemcpyAsync(keys, k0, n * 8, cudaMemcpyDeviceToDevice, s));
    if (vals) BM_CHECK_CUDA(cudaMemcpyAsync(vals, v0, n * 8, cudaMemcpyDeviceToDevice, s));
  }
  return BM_OK;
}

inline int bits_for(uint64_t maxv) {
  int b = 0;
  while (b < 64 && (maxv >> b) != 0) ++b;
  return b;
}

// ---- grouping --------------------------------------------------------------
__global__ void node_keys_kernel(const int64_t* __restrict__ rows, const int64_t* __restrict__ offs,
                                 const int64_t* __restrict__ node_base, int64_t n_el,
                                 int64_t n_entries, const int32_t* __restrict__ labels,
                                 int64_t n_nodes, uint64_t* __restrict__ keys,
                                 int64_t* __restrict__ vals, int32_t* __restrict__ counts) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n_entries;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = 0, b = n_el;
    while (b - a > 1) {
      int64_t mid = (a + b) >> 1;
      if (offs[mid] <= e) a = mid; else b = mid;
    }
    const int32_t l = labels[e];
    const int64_t key = l >= 0 ? node_base[a] + l : n_nodes;
    keys[e] = (uint64_t)key;
    vals[e] = rows[e];
    // warp-aggregated count (a few hundred nodes share ~1M entries: one
    // atomic per distinct node in the warp instead of one per entry)
    const unsigned act = __activemask();
    const unsigned same = __match_any_sync(act, key);
    if (l >= 0 && (__ffs(same) - 1) == (int)(threadIdx.x & 31)) atomicAdd(counts + key, __popc(same));
  }
}

// ---- edges -----------------------------------------------------------------
__global__ void entry_pairs_kernel(const int64_t* __restrict__ node_rows,
                                   const int64_t* __restrict__ node_off, int64_t n_nodes,
                                   int64_t total, uint64_t* __restrict__ keys,
                                   int64_t* __restrict__ vals) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = 0, b = n_nodes;
    while (b - a > 1) {
      int64_t mid = (a + b) >> 1;
      if (node_off[mid] <= i) a = mid; else b = mid;
    }
    keys[i] = (uint64_t)node_rows[i];
    vals[i] = a;
  }
}

// For each run of equal rows (sorted), count its node pairs.
__global__ void run_pairs_count_kernel(const uint64_t* __restrict__ keys, int64_t total,
                                       int64_t* __restrict__ npairs) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t c = 0;
    if (i == 0 || keys[i] != keys[i - 1]) {
      int64_t m = 1;
      while (i + m < total && keys[i + m] == keys[i]) ++m;
      c = m * (m - 1) / 2;
    }
    npairs[i] = c;
  }
}

__global__ void run_pairs_dense_kernel(const uint64_t* __restrict__ keys,
                                       const int64_t* __restrict__ vals, int64_t total,
                                       int64_t n_nodes, int32_t* __restrict__ bins) {
  const unsigned lt = (1u << (threadIdx.x & 31)) - 1u;
  (void)lt;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i == 0 || keys[i] != keys[i - 1]) {
      int64_t m = 1;
      while (i + m < total && keys[i + m] == keys[i]) ++m;
      for (int64_t x = 0; x < m; ++x)
        for (int64_t y = x + 1; y < m; ++y)
          atomicAdd(bins + vals[i + x] * n_nodes + vals[i + y], 1);
    }
  }
}

__global__ void run_pairs_emit_kernel(const uint64_t* __restrict__ keys,
                                      const int64_t* __restrict__ vals, int64_t total,
                                      int64_t n_nodes, const int64_t* __restrict__ pos,
                                      uint64_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i == 0 || keys[i] != keys[i - 1]) {
      int64_t m = 1;
      while (i + m < total && keys[i + m] == keys[i]) ++m;
      int64_t p = pos[i];
      for (int64_t x = 0; x < m; ++x)
        for (int64_t y = x + 1; y < m; ++y)
          out[p++] = (uint64_t)vals[i + x] * (uint64_t)n_nodes + (uint64_t)vals[i + y];
    }
  }
}

__global__ void nonzero_flags_kernel(const int32_t* __restrict__ bins, int64_t nb,
                                     int32_t* __restrict__ flags) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nb;
       i += (int64_t)gridDim.x * blockDim.x)
    flags[i] = bins[i] != 0;
}

__global__ void dense_edges_kernel(const int32_t* __restrict__ bins, int64_t n_nodes,
                                   const int64_t* __restrict__ pos, int64_t* __restrict__ edges) {
  const int64_t nb = n_nodes * n_nodes;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nb;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (bins[i]) {
      int64_t p = pos[i];
      edges[3 * p] = i / n_nodes;
      edges[3 * p + 1] = i % n_nodes;
      edges[3 * p + 2] = bins[i];
    }
  }
}

// Sort-free dense edges: every point lists the (few) nodes that hold it in
// kSlots slots (one per cover element it lies in at most); the pairs of a
// point's nodes are counted into the n_nodes^2 bins with warp-aggregated
// atomics (few distinct edges). A point in more than kSlots nodes sets the
// overflow flag and the caller takes the sorting path.
constexpr int kSlots = 8;
#ifndef BM_EDGE_SLOTS
#define BM_EDGE_SLOTS 1
#endif
constexpr bool kEdgeSlots = BM_EDGE_SLOTS;

__global__ void point_slots_kernel(const int64_t* __restrict__ node_rows,
                                   const int64_t* __restrict__ node_off, int64_t n_nodes,
                                   int64_t total, int32_t* __restrict__ cnt,
                                   int32_t* __restrict__ slots, int32_t* __restrict__ overflow) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = 0, b = n_nodes;
    while (b - a > 1) {
      const int64_t mid = (a + b) >> 1;
      if (node_off[mid] <= i) a = mid; else b = mid;
    }
    const int64_t p = node_rows[i];
    const int k = atomicAdd(cnt + p, 1);
    if (k < kSlots) slots[p * kSlots + k] = (int32_t)a;
    else *overflow = 1;
  }
}

__global__ void point_pairs_kernel(const int32_t* __restrict__ cnt,
                                   const int32_t* __restrict__ slots, int64_t n_points,
                                   int64_t n_nodes, int32_t* __restrict__ bins) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n_points;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int c = min(cnt[p], kSlots);
    // the common case, one pair per point: warp-aggregated by bin
    int64_t bin = -1;
    if (c == 2) {
      const int32_t u = slots[p * kSlots], v = slots[p * kSlots + 1];
      bin = (int64_t)min(u, v) * n_nodes + max(u, v);
    }
    const unsigned act = __activemask();
    const unsigned same = __match_any_sync(act, bin);
    if (bin >= 0 && (__ffs(same) - 1) == (int)(threadIdx.x & 31)) atomicAdd(bins + bin, __popc(same));
    if (c > 2)
      for (int x = 0; x < c; ++x)
        for (int y = x + 1; y < c; ++y) {
          const int32_t u = slots[p * kSlots + x], v = slots[p * kSlots + y];
          atomicAdd(bins + (int64_t)min(u, v) * n_nodes + max(u, v), 1);
        }
  }
}

__global__ void run_start_flags_kernel(const uint64_t* __restrict__ keys, int64_t n,
                                       int32_t* __restrict__ flags) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    flags[i] = (i == 0 || keys[i] != keys[i - 1]);
}

__global__ void sparse_edges_kernel(const uint64_t* __restrict__ keys, int64_t n,
                                    int64_t n_nodes, const int64_t* __restrict__ pos,
                                    int64_t* __restrict__ edges) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i == 0 || keys[i] != keys[i - 1]) {
      int64_t m = 1;
      while (i + m < n && keys[i + m] == keys[i]) ++m;
      int64_t p = pos[i];
      edges[3 * p] = (int64_t)(keys[i] / (uint64_t)n_nodes);
      edges[3 * p + 1] = (int64_t)(keys[i] % (uint64_t)n_nodes);
      edges[3 * p + 2] = m;
    }
  }
}

// ---- node payload ------------------------------------------------------------
// stats: numpy X[rows].mean(axis=0) = sequential row sum per column / size.
// The row sum is an inherently serial fp64 chain per column, so the time is
// set by how many row loads are in flight per chain: one warp per (node, 32
// columns) streams its rows through a shared-memory ring of kNsStages chunks
// of 32 rows with cp.async (each lane copies, and then adds, its own column;
// 192 rows in flight per warp), row ids prefetched a chunk ahead.
#ifndef BM_NS_STAGES
#define BM_NS_STAGES 6
#endif
constexpr int kNsStages = BM_NS_STAGES;  // 8 KB of static shared memory each
#ifndef BM_NS_LPT
#define BM_NS_LPT 1
#endif
constexpr bool kNsLpt = BM_NS_LPT;

__device__ __forceinline__ void cp_async8(void* dst, const void* src, bool pred) {
  const unsigned sz = pred ? 8u : 0u;  // src-size 0: zero-fill, no read
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(
                   (unsigned)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(sz)
               : "memory");
}

__global__ void __launch_bounds__(32)
node_stats_kernel(const double* __restrict__ X, int64_t d, const int64_t* __restrict__ node_rows,
                  const int64_t* __restrict__ node_off, const int32_t* __restrict__ order,
                  int64_t n_nodes, double* __restrict__ stats) {
  __shared__ __align__(16) double ring[kNsStages][32][32];
  const int64_t v = order[blockIdx.y];  // largest nodes first (their chains are the longest)
  const int lane = threadIdx.x;
  const int64_t c = (int64_t)blockIdx.x * 32 + lane;
  const bool col = c < d;
  const int64_t a = node_off[v], b = node_off[v + 1];
  const int64_t n_chunks = (b - a + 31) / 32;
  const double* Xc = X + (col ? c : 0);
  int64_t idx = a + lane < b ? node_rows[a + lane] : 0;  // row ids of the next chunk to issue
  int64_t q = 0;                                          // next chunk to issue
  auto issue = [&]() {
    if (q < n_chunks) {
      const int64_t base = a + q * 32;
      const int64_t nxt = base + 32 + lane;
      const int64_t idx_next = nxt < b ? node_rows[nxt] : 0;
      double(*st)[32] = ring[q % kNsStages];
#pragma unroll 8
      for (int j = 0; j < 32; ++j) {
        const int64_t r = __shfl_sync(0xffffffffu, idx, j);
        cp_async8(&st[j][lane], Xc + r * d, col && base + j < b);
      }
      idx = idx_next;
    }
    ++q;
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
#pragma unroll 1
  for (int s0 = 0; s0 < kNsStages - 1; ++s0) issue();
  double s = 0.0;
  for (int64_t k = 0; k < n_chunks; ++k) {
    issue();
    asm volatile("cp.async.wait_group %0;" ::"n"(kNsStages - 1) : "memory");
    const double(*st)[32] = ring[k % kNsStages];
    const int nv = (int)min((int64_t)32, b - (a + k * 32));
    if (nv == 32) {
#pragma unroll
      for (int j = 0; j < 32; ++j) s = __dadd_rn(s, st[j][lane]);
    } else {
      for (int j = 0; j < nv; ++j) s = __dadd_rn(s, st[j][lane]);
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  if (col) stats[v * d + c] = __ddiv_rn(s, (double)(b - a));
}

// numpy 1-D mean of the filter values of every node, in two parallel steps:
// every pairwise-sum leaf (<= 128 rows, 8 strided accumulators) of every node
// at once, then per node the leaf sums combined in the recursion's order
// (leaf program built on the host from the node sizes).
__device__ double pairwise_leaf_at(const double* __restrict__ f, int m, int ax,
                                   const int64_t* __restrict__ rows, int64_t n) {
  if (n < 8) {
    double r = -0.0;
    for (int64_t i = 0; i < n; ++i) r = __dadd_rn(r, f[rows[i] * m + ax]);
    return r;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = f[rows[j] * m + ax];
  int64_t i = 8;
  for (; i < n - (n % 8); i += 8)
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], f[rows[i + j] * m + ax]);
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, f[rows[i] * m + ax]);
  return res;
}

struct NodeLeaf {
  int64_t start;  // first entry of the leaf (absolute, into node_rows)
  int32_t len, pops;
};

__global__ void node_leaf_kernel(const double* __restrict__ f, int m,
                                 const int64_t* __restrict__ node_rows,
                                 const NodeLeaf* __restrict__ leaves, int64_t n_leaves,
                                 double* __restrict__ lsum) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_leaves * m) return;
  const NodeLeaf L = leaves[t / m];
  const int ax = (int)(t % m);
  lsum[t] = pairwise_leaf_at(f, m, ax, node_rows + L.start, L.len);
}

__global__ void node_combine_kernel(const NodeLeaf* __restrict__ leaves,
                                    const int64_t* __restrict__ leaf_off, int m,
                                    const double* __restrict__ lsum,
                                    const int64_t* __restrict__ node_off, int64_t n_nodes,
                                    double* __restrict__ fmean) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_nodes * m) return;
  const int64_t v = t / m;
  const int ax = (int)(t % m);
  constexpr int kS = 48;
  double st[kS];
  int sp = 0;
  for (int64_t l = leaf_off[v]; l < leaf_off[v + 1]; ++l) {
    st[sp++] = lsum[l * m + ax];
    for (int q = 0; q < leaves[l].pops; ++q) {
      st[sp - 2] = __dadd_rn(st[sp - 2], st[sp - 1]);
      --sp;
    }
  }
  const int64_t n = node_off[v + 1] - node_off[v];
  fmean[t] = __ddiv_rn(__dadd_rn(0.0, sp > 0 ? st[0] : 0.0), (double)n);
}

inline unsigned grid1(int64_t n, int threads = 256) {
  int64_t b = ceil_div(n, threads);
  int64_t cap = (int64_t)num_sms() * 16;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (unsigned)b;
}

}  // namespace

int sort_pairs_u64(uint64_t* keys, int64_t* vals, int64_t n, int key_bits, cudaStream_t s) {
  return radix_sort_pairs(keys, vals, n, key_bits, s);
}

}  // namespace bm

using namespace bm;

extern "C" int bm_group_nodes(const int64_t* d_rows, const int64_t* h_offsets, int64_t n_el,
                              const int32_t* d_labels, const int32_t* h_n_clusters,
                              int64_t* d_node_rows, int64_t* d_node_offsets, int64_t* h_total,
                              void* stream_) {
  cudaStream_t s = (cudaStream_t)stream_;
  BM_REQUIRE(n_el >= 0 && h_offsets && h_n_clusters && h_total, "bad arguments");
  std::vector<int64_t> node_base(n_el + 1, 0);
  for (int64_t k = 0; k < n_el; ++k) {
    BM_REQUIRE(h_n_clusters[k] >= 0, "negative cluster count");
    node_base[k + 1] = node_base[k] + h_n_clusters[k];
  }
  const int64_t n_nodes = node_base[n_el];
  const int64_t n_entries = n_el ? h_offsets[n_el] - h_offsets[0] : 0;
  *h_total = 0;
  BM_REQUIRE(d_node_offsets, "null node offsets");
  if (n_nodes == 0 || n_entries == 0) {
    BM_CHECK_CUDA(cudaMemsetAsync(d_node_offsets, 0, (n_nodes + 1) * 8, s));
    BM_CHECK_CUDA(cudaStreamSynchronize(s));
    return BM_OK;
  }
  BM_REQUIRE(d_rows && d_labels && d_node_rows, "null device pointer");
  std::vector<int64_t> offs(n_el + 1);
  for (int64_t k = 0; k <= n_el; ++k) offs[k] = h_offsets[k] - h_offsets[0];
  Scratch tab, kv, cnt;
  BM_TRY(scratch_alloc(tab, (2 * n_el + 2) * 8, s));
  int64_t* d_offs = tab.as<int64_t>();
  int64_t* d_nb = d_offs + n_el + 1;
  BM_CHECK_CUDA(cudaMemcpyAsync(d_offs, offs.data(), (n_el + 1) * 8, cudaMemcpyHostToDevice, s));
  BM_CHECK_CUDA(cudaMemcpyAsync(d_nb, node_base.data(), (n_el + 1) * 8, cudaMemcpyHostToDevice, s));
  BM_TRY(scratch_alloc(kv, n_entries * 16, s));
  uint64_t* keys = kv.as<uint64_t>();
  int64_t* vals = (int64_t*)(keys + n_entries);
  BM_TRY(scratch_alloc(cnt, (n_nodes + 1) * 4, s));
  BM_CHECK_CUDA(cudaMemsetAsync(cnt.ptr, 0, (n_nodes + 1) * 4, s));
  node_keys_kernel<<<grid1(n_entries), 256, 0, s>>>(d_rows + h_offsets[0], d_offs, d_nb, n_el,
                                                    n_entries, d_labels + h_offsets[0], n_nodes,
                                                    keys, vals, cnt.as<int32_t>());
  BM_CHECK_LAUNCH();
  BM_TRY(radix_sort_pairs(keys, vals, n_entries, bits_for((uint64_t)n_nodes), s));
  BM_TRY(exclusive_scan_i32_to_i64(cnt.as<int32_t>(), d_node_offsets, n_nodes + 1, s));
  int64_t total = 0;
  BM_CHECK_CUDA(cudaMemcpyAsync(&total, d_node_offsets + n_nodes, 8, cudaMemcpyDeviceToHost, s));
  BM_CHECK_CUDA(cudaStreamSynchronize(s));
  if (total > 0)
    BM_CHECK_CUDA(cudaMemcpyAsync(d_node_rows, vals, total * 8, cudaMemcpyDeviceToDevice, s));
  *h_total = total;
  return BM_OK;
}

extern "C" int bm_nerve_edges(const int64_t* d_node_rows, const int64_t* d_node_offsets,
                              int64_t n_nodes, int64_t n_points, int64_t* d_edges,
                              int64_t* h_n_edges, void* stream_) {
  cudaStream_t s = (cudaStream_t)stream_;
  BM_REQUIRE(h_n_edges && n_nodes >= 0 && n_points >= 0, "bad arguments");
  *h_n_edges = 0;
  if (n_nodes < 2) return BM_OK;
  BM_REQUIRE(d_node_rows && d_node_offsets, "null device pointer");
  int64_t total = 0;
  BM_CHECK_CUDA(cudaMemcpyAsync(&total, d_node_offsets + n_nodes, 8, cudaMemcpyDeviceToHost, s));
  BM_CHECK_CUDA(cudaStreamSynchronize(s));
  if (total == 0) return BM_OK;
  Scratch kv;
  uint64_t* keys = nullptr;
  int64_t* vals = nullptr;
  auto sort_entries = [&]() -> int {  // (row, node) entries sorted by row
    BM_TRY(scratch_alloc(kv, total * 16 + 16, s));
    keys = kv.as<uint64_t>();
    vals = (int64_t*)(keys + total);
    entry_pairs_kernel<<<grid1(total), 256, 0, s>>>(d_node_rows, d_node_offsets, n_nodes, total,
                                                    keys, vals);
    BM_CHECK_LAUNCH();
    return radix_sort_pairs(keys, vals, total,
                            bits_for((uint64_t)std::max<int64_t>(n_points, 1)), s);
  };
  const bool dense = n_nodes <= 4096;
  if (dense) {
    const int64_t nb = n_nodes * n_nodes;
    Scratch bins, flags, pos;
    BM_TRY(scratch_alloc(bins, nb * 4, s));
    BM_TRY(scratch_alloc(flags, nb * 4, s));
    BM_TRY(scratch_alloc(pos, (nb + 1) * 8, s));
    BM_CHECK_CUDA(cudaMemsetAsync(bins.ptr, 0, nb * 4, s));
    bool sorted_path = !kEdgeSlots;
    if (kEdgeSlots) {
      Scratch sc;
      BM_TRY(scratch_alloc(sc, (size_t)n_points * 4 * (1 + kSlots) + 16, s));
      int32_t* cnt = sc.as<int32_t>();
      int32_t* slots = cnt + n_points;
      int32_t* ovf = slots + n_points * kSlots;
      BM_CHECK_CUDA(cudaMemsetAsync(cnt, 0, n_points * 4, s));
      BM_CHECK_CUDA(cudaMemsetAsync(ovf, 0, 4, s));
      point_slots_kernel<<<grid1(total), 256, 0, s>>>(d_node_rows, d_node_offsets, n_nodes, total,
                                                      cnt, slots, ovf);
      BM_CHECK_LAUNCH();
      int32_t h_ovf = 0;
      BM_CHECK_CUDA(cudaMemcpyAsync(&h_ovf, ovf, 4, cudaMemcpyDeviceToHost, s));
      BM_CHECK_CUDA(cudaStreamSynchronize(s));
      if (h_ovf) {
        sorted_path = true;
      } else {
        point_pairs_kernel<<<grid1(n_points), 256, 0, s>>>(cnt, slots, n_points, n_nodes,
                                                           bins.as<int32_t>());
        BM_CHECK_LAUNCH();
      }
    }
    if (sorted_path) {
      BM_TRY(sort_entries());
      run_pairs_dense_kernel<<<grid1(total), 256, 0, s>>>(keys, vals, total, n_nodes,
                                                          bins.as<int32_t>());
      BM_CHECK_LAUNCH();
    }
    nonzero_flags_kernel<<<grid1(nb), 256, 0, s>>>(bins.as<int32_t>(), nb, flags.as<int32_t>());
    BM_CHECK_LAUNCH();
    BM_TRY(exclusive_scan_i32_to_i64(flags.as<int32_t>(), pos.as<int64_t>(), nb, s));
    int64_t last_pos = 0;
    int32_t last_flag = 0;
    BM_CHECK_CUDA(cudaMemcpyAsync(&last_pos, pos.as<int64_t>() + nb - 1, 8, cudaMemcpyDeviceToHost, s));
    BM_CHECK_CUDA(cudaMemcpyAsync(&last_flag, flags.as<int32_t>() + nb - 1, 4, cudaMemcpyDeviceToHost, s));
    BM_CHECK_CUDA(cudaStreamSynchronize(s));
    const int64_t n_edges = last_pos + last_flag;
    *h_n_edges = n_edges;
    if (d_edges && n_edges) {
      dense_edges_kernel<<<grid1(nb), 256, 0, s>>>(bins.as<int32_t>(), n_nodes, pos.as<int64_t>(),
                                                  d_edges);
      BM_CHECK_LAUNCH();
      BM_CHECK_CUDA(cudaStreamSynchronize(s));
    }
    return BM_OK;
  }
  // sparse: materialise pair keys, sort, run-length encode
  BM_TRY(sort_entries());
  Scratch np, pk, fl, ps;
  BM_TRY(scratch_alloc(np, (total + 1) * 8, s));
  run_pairs_count_kernel<<<grid1(total), 256, 0, s>>>(keys, total, np.as<int64_t>());
  BM_CHECK_LAUNCH();
  int64_t last_cnt = 0;
  BM_CHECK_CUDA(cudaMemcpyAsync(&last_cnt, np.as<int64_t>() + total - 1, 8, cudaMemcpyDeviceToHost, s));
  BM_TRY(exclusive_scan_i64(np.as<int64_t>(), np.as<int64_t>(), total, s));
  int64_t last_pos = 0;
  BM_CHECK_CUDA(cudaMemcpyAsync(&last_pos, np.as<int64_t>() + total - 1, 8, cudaMemcpyDeviceToHost, s));
  BM_CHECK_CUDA(cudaStreamSynchronize(s));
  const int64_t n_pairs = last_pos + last_cnt;
  if (n_pairs == 0) return BM_OK;
  BM_TRY(scratch_alloc(pk, n_pairs * 8, s));
  run_pairs_emit_kernel<<<grid1(total), 256, 0, s>>>(keys, vals, total, n_nodes, np.as<int64_t>(),
                                                     pk.as<uint64_t>());
  BM_CHECK_LAUNCH();
  BM_TRY(radix_sort_pairs(pk.as<uint64_t>(), nullptr, n_pairs,
                          bits_for((uint64_t)n_nodes * (uint64_t)n_nodes), s));
  BM_TRY(scratch_alloc(fl, n_pairs * 4, s));
  BM_TRY(scratch_alloc(ps, n_pairs * 8, s));
  run_start_flags_kernel<<<grid1(n_pairs), 256, 0, s>>>(pk.as<uint64_t>(), n_pairs, fl.as<int32_t>());
  BM_CHECK_LAUNCH();
  BM_TRY(exclusive_scan_i32_to_i64(fl.as<int32_t>(), ps.as<int64_t>(), n_pairs, s));
  int64_t lp = 0;
  int32_t lf = 0;
  BM_CHECK_CUDA(cudaMemcpyAsync(&lp, ps.as<int64_t>() + n_pairs - 1, 8, cudaMemcpyDeviceToHost, s));
  BM_CHECK_CUDA(cudaMemcpyAsync(&lf, fl.as<int32_t>() + n_pairs - 1, 4, cudaMemcpyDeviceToHost, s));
  BM_CHECK_CUDA(cudaStreamSynchronize(s));
  *h_n_edges = lp + lf;
  if (d_edges && *h_n_edges) {
    sparse_edges_kernel<<<grid1(n_pairs), 256, 0, s>>>(pk.as<uint64_t>(), n_pairs, n_nodes,
                                                      ps.as<int64_t>(), d_edges);
    BM_CHECK_LAUNCH();
    BM_CHECK_CUDA(cudaStreamSynchronize(s));
  }
  return BM_OK;
}

extern "C" int bm_node_stats(const double* d_X, int64_t d, const double* d_f, int m,
                             const int64_t* d_node_rows, const int64_t* d_node_offsets,
                             int64_t n_nodes, double* d_stats, double* d_fmean, void* stream_) {
  cudaStream_t s = (cudaStream_t)stream_;
  BM_REQUIRE(d >= 1 && (m == 1 || m == 2) && n_nodes >= 0, "bad arguments");
  if (n_nodes == 0) return BM_OK;
  BM_REQUIRE(n_nodes <= 65535, "node_stats: at most 65535 nodes per call");
  // node sizes on the host: launch order of the column chains (largest
  // first) and the pairwise leaf programs of the filter means
  std::vector<int64_t> off(n_nodes + 1);
  BM_CHECK_CUDA(cudaMemcpyAsync(off.data(), d_node_offsets, (n_nodes + 1) * 8,
                                cudaMemcpyDeviceToHost, s));
  BM_CHECK_CUDA(cudaStreamSynchronize(s));
  Scratch s_order;
  if (d_stats) {
    BM_REQUIRE(d_X, "null points");
    std::vector<int32_t> order(n_nodes);
    for (int64_t v = 0; v < n_nodes; ++v) order[v] = (int32_t)v;
    if (kNsLpt)
      std::stable_sort(order.begin(), order.end(), [&](int32_t x, int32_t y) {
        return off[x + 1] - off[x] > off[y + 1] - off[y];
      });
    BM_TRY(scratch_alloc(s_order, (size_t)n_nodes * 4, s));
    BM_CHECK_CUDA(cudaMemcpyAsync(s_order.ptr, order.data(), n_nodes * 4, cudaMemcpyHostToDevice, s));
    dim3 grid((unsigned)ceil_div(d, 32), (unsigned)n_nodes);
    node_stats_kernel<<<grid, 32, 0, s>>>(d_X, d, d_node_rows, d_node_offsets,
                                          s_order.as<int32_t>(), n_nodes, d_stats);
    BM_CHECK_LAUNCH();
  }
  if (d_fmean) {
    BM_REQUIRE(d_f, "null filter values");
    std::vector<NodeLeaf> lv;
    std::vector<int64_t> loff(n_nodes + 1, 0);
    for (int64_t v = 0; v < n_nodes; ++v) {
      const int64_t n = off[v + 1] - off[v];
      BM_REQUIRE(n >= 1 && n < (1ll << 31), "bad node size");
      for (const PwLeaf& L : pw_plan((int)n)) lv.push_back({off[v] + L.start, L.len, L.pops});
      loff[v + 1] = (int64_t)lv.size();
    }
    const int64_t nl = (int64_t)lv.size();
    Scratch sl, so, ss;
    BM_TRY(scratch_alloc(sl, nl * sizeof(NodeLeaf), s));
    BM_TRY(scratch_alloc(so, (n_nodes + 1) * 8, s));
    BM_TRY(scratch_alloc(ss, (size_t)nl * m * 8, s));
    BM_CHECK_CUDA(cudaMemcpyAsync(sl.ptr, lv.data(), nl * sizeof(NodeLeaf),
                                  cudaMemcpyHostToDevice, s));
    BM_CHECK_CUDA(cudaMemcpyAsync(so.ptr, loff.data(), (n_nodes + 1) * 8,
                                  cudaMemcpyHostToDevice, s));
    node_leaf_kernel<<<(unsigned)ceil_div(nl * m, 128), 128, 0, s>>>(
        d_f, m, d_node_rows, sl.as<NodeLeaf>(), nl, ss.as<double>());
    BM_CHECK_LAUNCH();
    node_combine_kernel<<<(unsigned)ceil_div(n_nodes * m, 64), 64, 0, s>>>(
        sl.as<NodeLeaf>(), so.as<int64_t>(), m, ss.as<double>(), d_node_offsets, n_nodes,
        d_fmean);
    BM_CHECK_LAUNCH();
  }
  return BM_OK;
}
