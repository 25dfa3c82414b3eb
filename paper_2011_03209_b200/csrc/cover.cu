// cover.cu — K2: cover binning + stable compaction of per-element row lists.
//
// Reference: nervemap/cover.py:122-140 (membership). Row i is in element k
// iff lo <= f(i) <= hi on every axis (closed intervals; NaN is in nothing).
// Per axis the intervals are sorted (lo_k, hi_k non-decreasing, cover.py:
// 97-104), so a point's axis-memberships form one contiguous range found by
// two binary searches; a 2-D element k = (i, j) is row-major (cover.py:56-61).
//
// Both passes process the points in chunks of kChunk rows with one warp per
// chunk, in row order, so the compaction is stable (ascending rows) without
// a sort: pass 1 counts rows per (element, chunk) into C[k][chunk]; the flat
// exclusive scan of C (element-major) is every chunk's write cursor; pass 2
// replays the chunk and scatters rows. HBM traffic: 2*N*m*8 (f read twice)
// + sum(n_k)*8 (rows written) + N_chunks*n_el*8 (cursor table).
#include "common.cuh"

namespace bm {
namespace {

constexpr int kChunk = 256;  // rows per warp-chunk

struct AxisTable {
  const double* lo;  // concatenated
  const double* hi;
  int n0, n1;        // intervals per axis (n1 = 1 for m = 1)
  int m;
};

// first k with hi[k] >= v ; n if none
__device__ __forceinline__ int lower_hi(const double* hi, int n, double v) {
  int a = 0, b = n;
  while (a < b) {
    int mid = (a + b) >> 1;
    if (hi[mid] < v) a = mid + 1; else b = mid;
  }
  return a;
}
// number of k with lo[k] <= v
__device__ __forceinline__ int count_lo(const double* lo, int n, double v) {
  int a = 0, b = n;
  while (a < b) {
    int mid = (a + b) >> 1;
    if (lo[mid] <= v) a = mid + 1; else b = mid;
  }
  return a;
}

// Axis range [first, last] (empty when first > last). Uses the exact closed
// test of cover.py:133 on the boundary intervals so NaN and ties follow it.
__device__ __forceinline__ void axis_range(const double* lo, const double* hi, int n, double v,
                                           int& first, int& last) {
  first = lower_hi(hi, n, v);
  last = count_lo(lo, n, v) - 1;
  if (!(v == v)) { first = 1; last = 0; }
}

// PASS 1 (COUNT=true) / PASS 2 (COUNT=false): one warp per chunk of rows.
// SMEM: the warp keeps its chunk's cursors of all n_el elements in shared
// memory (loaded once, written back once) instead of a global load/store per
// served element.
constexpr int kSmemEl = 256;  // largest element count with shared-memory cursors

template <bool COUNT, bool SMEM>
__global__ void membership_kernel(const double* __restrict__ f, int64_t n, AxisTable t,
                                  int64_t n_chunks, int64_t* __restrict__ cursor,
                                  int64_t* __restrict__ rows_out) {
  extern __shared__ int64_t s_cur[];
  const int lane = threadIdx.x & 31;
  const int64_t chunk = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (chunk >= n_chunks) return;
  const int n_el = t.n0 * t.n1;
  int64_t* const wc = SMEM ? s_cur + (threadIdx.x >> 5) * (int64_t)n_el : nullptr;
  if (SMEM) {
    for (int k = lane; k < n_el; k += 32) wc[k] = cursor[(int64_t)k * n_chunks + chunk];
    __syncwarp();
  }
  const int64_t r0 = chunk * kChunk;
  const int64_t r1 = min(n, r0 + kChunk);
  const unsigned lt = (1u << lane) - 1u;
  for (int64_t base = r0; base < r1; base += 32) {
    const int64_t r = base + lane;
    int f0 = 1, l0 = 0, f1 = 0, l1 = 0;
    if (r < r1) {
      axis_range(t.lo, t.hi, t.n0, f[r * t.m], f0, l0);
      if (t.m == 2) axis_range(t.lo + t.n0, t.hi + t.n0, t.n1, f[r * t.m + 1], f1, l1);
    }
    int c0 = l0 >= f0 ? l0 - f0 + 1 : 0;
    int c1 = t.m == 2 ? (l1 >= f1 ? l1 - f1 + 1 : 0) : 1;
    const int mult = c0 * c1;
    // A lane's element keys ascend with its slot s (row-major (i, j)), so
    // the warp repeatedly serves the smallest pending key: every element is
    // served once per 32-row batch with its lanes in row order (stable).
    int s = 0;
    while (true) {
      int key = 0x7fffffff;
      if (s < mult) {
        int i = f0 + s / c1;
        int j = t.m == 2 ? f1 + s % c1 : 0;
        key = i * t.n1 + j;
      }
      const int kmin = __reduce_min_sync(0xffffffffu, key);
      if (kmin == 0x7fffffff) break;
      const bool mine = key == kmin;
      const unsigned peers = __ballot_sync(0xffffffffu, mine);
      const int leader = __ffs(peers) - 1;
      int64_t* cur = SMEM ? &wc[kmin] : &cursor[(int64_t)kmin * n_chunks + chunk];
      int64_t basepos = 0;
      if (lane == leader) basepos = *cur;
      basepos = __shfl_sync(0xffffffffu, basepos, leader);
      if (mine) {
        if (!COUNT) rows_out[basepos + __popc(peers & lt)] = r;
        ++s;
      }
      if (lane == leader) *cur = basepos + __popc(peers);
      __syncwarp();
    }
  }
  if (SMEM && COUNT)
    for (int k = lane; k < n_el; k += 32) cursor[(int64_t)k * n_chunks + chunk] = wc[k];
}

template <bool COUNT>
void launch_membership(const double* f, int64_t n, const AxisTable& t, int64_t n_chunks,
                       int64_t* cursor, int64_t* rows_out, cudaStream_t stream) {
  const int warps = 4;
  const unsigned blocks = (unsigned)ceil_div(n_chunks, warps);
  const int64_t n_el = (int64_t)t.n0 * t.n1;
  if (n_el <= kSmemEl)
    membership_kernel<COUNT, true><<<blocks, warps * 32, warps * n_el * sizeof(int64_t), stream>>>(
        f, n, t, n_chunks, cursor, rows_out);
  else
    membership_kernel<COUNT, false><<<blocks, warps * 32, 0, stream>>>(f, n, t, n_chunks, cursor,
                                                                      rows_out);
}

// counts[k] = sum over chunks of C[k][chunk]
__global__ void element_totals_kernel(const int64_t* __restrict__ C, int64_t n_chunks,
                                      int64_t n_el, int64_t* __restrict__ totals) {
  int64_t k = blockIdx.x;
  if (k >= n_el) return;
  int64_t s = 0;
  for (int64_t c = threadIdx.x; c < n_chunks; c += blockDim.x) s += C[k * n_chunks + c];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  __shared__ int64_t ws[32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += ws[w];
    totals[k] = t;
  }
}

// element-major exclusive scan of C, shifted so chunk cursors start at the
// caller's d_offsets[k] (equal to the scan when offsets are the count scan).
__global__ void add_offsets_kernel(int64_t* __restrict__ C, int64_t n_chunks, int64_t n_el,
                                   const int64_t* __restrict__ offsets,
                                   const int64_t* __restrict__ scan_first) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_chunks * n_el) return;
  int64_t k = i / n_chunks;
  C[i] = C[i] - scan_first[k] + offsets[k];
}

__global__ void gather_first_kernel(const int64_t* __restrict__ C, int64_t n_chunks,
                                    int64_t n_el, int64_t* __restrict__ first) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n_el) first[k] = C[k * n_chunks];
}

struct Prepared {
  Scratch tab;  // lo|hi on device
  AxisTable t;
  int64_t n_el = 0;
  int64_t n_chunks = 0;
};

int prepare(const double* h_lo, const double* h_hi, const int32_t* h_n_axis, int m, int64_t n,
            cudaStream_t stream, Prepared& p) {
  BM_REQUIRE(m == 1 || m == 2, "cover needs 1 or 2 axes, got %d", m);
  BM_REQUIRE(h_lo && h_hi && h_n_axis, "null cover table");
  int n0 = h_n_axis[0], n1 = m == 2 ? h_n_axis[1] : 1;
  BM_REQUIRE(n0 >= 1 && n1 >= 1, "interval counts must be >= 1");
  int64_t tot = (int64_t)n0 + (m == 2 ? n1 : 0);
  BM_TRY(scratch_alloc(p.tab, 2 * tot * sizeof(double), stream));
  double* lo = p.tab.as<double>();
  double* hi = lo + tot;
  BM_CHECK_CUDA(cudaMemcpyAsync(lo, h_lo, tot * sizeof(double), cudaMemcpyHostToDevice, stream));
  BM_CHECK_CUDA(cudaMemcpyAsync(hi, h_hi, tot * sizeof(double), cudaMemcpyHostToDevice, stream));
  p.t = AxisTable{lo, hi, n0, n1, m};
  p.n_el = (int64_t)n0 * n1;
  p.n_chunks = ceil_div(n, kChunk);
  return BM_OK;
}

int count_table(const double* f, int64_t n, Prepared& p, Scratch& C, cudaStream_t stream) {
  int64_t cells = p.n_el * p.n_chunks;
  BM_TRY(scratch_alloc(C, (cells + 1) * sizeof(int64_t), stream));
  BM_CHECK_CUDA(cudaMemsetAsync(C.ptr, 0, (cells + 1) * sizeof(int64_t), stream));
  if (n == 0) return BM_OK;
  launch_membership<true>(f, n, p.t, p.n_chunks, C.as<int64_t>(), nullptr, stream);
  BM_CHECK_LAUNCH();
  return BM_OK;
}

}  // namespace
}  // namespace bm

using namespace bm;

extern "C" int bm_membership_count(const double* d_f, int64_t n, int m, const double* h_lo,
                                   const double* h_hi, const int32_t* h_n_axis,
                                   int64_t* h_counts, void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  BM_REQUIRE(n >= 0, "negative row count");
  BM_REQUIRE(h_counts, "null counts");
  BM_REQUIRE(n == 0 || d_f, "null filter values");
  Prepared p;
  BM_TRY(prepare(h_lo, h_hi, h_n_axis, m, n, stream, p));
  Scratch C, tot;
  BM_TRY(count_table(d_f, n, p, C, stream));
  BM_TRY(scratch_alloc(tot, p.n_el * sizeof(int64_t), stream));
  if (p.n_chunks > 0) {
    element_totals_kernel<<<(unsigned)p.n_el, 256, 0, stream>>>(C.as<int64_t>(), p.n_chunks,
                                                                p.n_el, tot.as<int64_t>());
    BM_CHECK_LAUNCH();
  } else {
    BM_CHECK_CUDA(cudaMemsetAsync(tot.ptr, 0, p.n_el * sizeof(int64_t), stream));
  }
  BM_CHECK_CUDA(cudaMemcpyAsync(h_counts, tot.ptr, p.n_el * sizeof(int64_t),
                                cudaMemcpyDeviceToHost, stream));
  BM_CHECK_CUDA(cudaStreamSynchronize(stream));
  return BM_OK;
}

extern "C" int bm_membership_fill(const double* d_f, int64_t n, int m, const double* h_lo,
                                  const double* h_hi, const int32_t* h_n_axis,
                                  const int64_t* d_offsets, int64_t* d_rows, void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  BM_REQUIRE(n >= 0, "negative row count");
  BM_REQUIRE(d_offsets, "null offsets");
  if (n == 0) return BM_OK;
  BM_REQUIRE(d_f && d_rows, "null pointer");
  Prepared p;
  BM_TRY(prepare(h_lo, h_hi, h_n_axis, m, n, stream, p));
  Scratch C, first;
  BM_TRY(count_table(d_f, n, p, C, stream));
  int64_t cells = p.n_el * p.n_chunks;
  // cursors: element-major exclusive scan, re-based on the caller's offsets
  BM_TRY(exclusive_scan_i64(C.as<int64_t>(), C.as<int64_t>(), cells, stream));
  BM_TRY(scratch_alloc(first, p.n_el * sizeof(int64_t), stream));
  gather_first_kernel<<<(unsigned)ceil_div(p.n_el, 256), 256, 0, stream>>>(
      C.as<int64_t>(), p.n_chunks, p.n_el, first.as<int64_t>());
  BM_CHECK_LAUNCH();
  add_offsets_kernel<<<(unsigned)ceil_div(cells, 256), 256, 0, stream>>>(
      C.as<int64_t>(), p.n_chunks, p.n_el, d_offsets, first.as<int64_t>());
  BM_CHECK_LAUNCH();
  launch_membership<false>(d_f, n, p.t, p.n_chunks, C.as<int64_t>(), d_rows, stream);
  BM_CHECK_LAUNCH();
  return BM_OK;
}
