// lens.cu — K1: lens evaluation and normalisation in exact fp64.
//
// Reference: nervemap/filters.py:133-140 (evaluate), dataset.py:165-186
// (normalize). The l2-norm lens is np.sqrt((X**2).sum(axis=1)): numpy's
// pairwise summation of the squared row (loops_utils.h.src pairwise_sum,
// 8 strided accumulators over blocks of <=128, recursive halving), then an
// IEEE sqrt. One warp evaluates one row: lanes 8g..8g+7 run the 8
// accumulators of leaf g of a group of 4 leaves, the 8-way combine is a
// butterfly (fp add is commutative, so the butterfly reproduces
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) bit for bit), and lane 0 replays the
// post-order leaf program. HBM-bound: N*d*8 bytes read, N*8 written.
#include "common.cuh"

namespace bm {
namespace {


constexpr int kLensWarps = 8;

// Sum of squares (or plain values) of one leaf owned by 8 lanes starting at
// `lane0` of the leaf group. Returns the leaf sum on every lane of the group.
template <bool SQUARE>
__device__ __forceinline__ double leaf_sum_8lanes(const double* __restrict__ row, int start,
                                                  int len, int j) {
  auto term = [&](int i) -> double {
    double v = row[start + i];
    return SQUARE ? __dmul_rn(v, v) : v;
  };
  if (len < 8) {
    // numpy: res = -0.0; res += a[i] sequentially. One lane suffices; the
    // group leader computes it and broadcasts.
    double res = -0.0;
    for (int i = 0; i < len; ++i) res = __dadd_rn(res, term(i));
    return res;
  }
  double r = term(j);
  const int body = len - (len % 8);
  for (int i = 8; i < body; i += 8) r = __dadd_rn(r, term(i + j));
  // butterfly over 8 lanes (xor 1, 2, 4) == the numpy combine tree
  r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 1));
  r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 2));
  r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 4));
  for (int i = body; i < len; ++i) r = __dadd_rn(r, term(i));
  return r;
}

// numpy pairwise sum of squares of one row (whole warp cooperates).
template <bool SQUARE>
__device__ double warp_pairwise_row(const double* __restrict__ row, const PwProgram& prog,
                                    double* s_leaf) {
  const int lane = threadIdx.x & 31;
  const int g = lane >> 3, j = lane & 7;
  for (int base = 0; base < prog.n_leaves; base += 4) {
    int li = base + g;
    double v = 0.0;
    bool active = li < prog.n_leaves;
    int start = active ? prog.leaf[li].start : 0;
    int len = active ? prog.leaf[li].len : 8;
    // all 32 lanes must reach the shuffles: inactive groups use a dummy leaf
    // of length 8 over the row's first elements (result discarded).
    if (!active) start = 0, len = (prog.leaf[0].len >= 8 ? 8 : prog.leaf[0].len);
    if (len >= 8) {
      v = leaf_sum_8lanes<SQUARE>(row, start, len, j);
    } else {
      v = leaf_sum_8lanes<SQUARE>(row, start, len, j);  // uniform per group
    }
    if (active && j == 0) s_leaf[li] = v;
  }
  __syncwarp();
  double total = 0.0;
  if (lane == 0) {
    PwStack st;
#pragma unroll
    for (int i = 0; i < kMaxStack; ++i) st.s[i] = 0.0;
    for (int li = 0; li < prog.n_leaves; ++li) {
      st.push(s_leaf[li]);
      for (int p = 0; p < prog.leaf[li].pops; ++p) st.reduce();
    }
    total = st.s[0];
  }
  __syncwarp();
  return __shfl_sync(0xffffffffu, total, 0);
}

// Packed form for rows of 1, 2 or 4 full leaves (8 <= d <= 512 with every
// leaf >= 8 long): the 4 lane groups of a warp cover 4 / n_leaves rows at
// once, each lane loads its (<= 16) strided values of the leaf up front, and
// the leader of each row replays the leaf program. Same additions, same order
// as warp_pairwise_row.
__device__ __forceinline__ double packed_leaf(const double* __restrict__ row, int start, int len,
                                              int j) {
  double v[16];
  const int body = len - (len % 8);
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = (8 * i < body) ? __ldg(row + start + 8 * i + j) : 0.0;
  double r = __dmul_rn(v[0], v[0]);
#pragma unroll
  for (int i = 1; i < 16; ++i)
    if (8 * i < body) r = __dadd_rn(r, __dmul_rn(v[i], v[i]));
  r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 1));
  r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 2));
  r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 4));
  for (int i = body; i < len; ++i) {
    const double t = row[start + i];
    r = __dadd_rn(r, __dmul_rn(t, t));
  }
  return r;
}

__global__ void __launch_bounds__(kLensWarps * 32)
lens_l2_kernel(const double* __restrict__ X, int64_t n, int64_t d, double* __restrict__ out,
               const __grid_constant__ PwProgram c_prog_lens, int packed) {
  __shared__ double s_leaf[kLensWarps][kMaxLeaves];
  const int warp = threadIdx.x >> 5;
  if (packed) {
    const int nl = c_prog_lens.n_leaves, rpw = 4 / nl;
    const int lane = threadIdx.x & 31, g = lane >> 3, j = lane & 7;
    const int sub = g / nl, li = g % nl;
    const PwLeaf L = c_prog_lens.leaf[li];
    for (int64_t r0 = ((int64_t)blockIdx.x * kLensWarps + warp) * rpw; r0 < n;
         r0 += (int64_t)gridDim.x * kLensWarps * rpw) {
      const int64_t r = min(r0 + sub, n - 1);  // tail: duplicate work, not stored
      const double v = packed_leaf(X + r * d, L.start, L.len, j);
      if (j == 0) s_leaf[warp][g] = v;
      __syncwarp();
      if (j == 0 && li == 0 && r0 + sub < n) {
        PwStack st;
#pragma unroll
        for (int i = 0; i < kMaxStack; ++i) st.s[i] = 0.0;
        for (int k = 0; k < nl; ++k) {
          st.push(s_leaf[warp][g + k]);
          for (int p = 0; p < c_prog_lens.leaf[k].pops; ++p) st.reduce();
        }
        // reduction result = identity(+0.0) + pairwise(...)
        out[r0 + sub] = __dsqrt_rn(__dadd_rn(0.0, st.s[0]));
      }
      __syncwarp();
    }
    return;
  }
  for (int64_t r = (int64_t)blockIdx.x * kLensWarps + warp; r < n;
       r += (int64_t)gridDim.x * kLensWarps) {
    double s = warp_pairwise_row<true>(X + r * d, c_prog_lens, s_leaf[warp]);
    // reduction result = identity(+0.0) + pairwise(...)
    s = __dadd_rn(0.0, s);
    if ((threadIdx.x & 31) == 0) out[r] = __dsqrt_rn(s);
  }
}

__global__ void lens_linf_kernel(const double* __restrict__ X, int64_t n, int64_t d,
                                 double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int warps = blockDim.x >> 5;
  for (int64_t r = (int64_t)blockIdx.x * warps + (threadIdx.x >> 5); r < n;
       r += (int64_t)gridDim.x * warps) {
    const double* row = X + r * d;
    double m = -1.0;
    bool nan = false;
    for (int64_t c = lane; c < d; c += 32) {
      double v = fabs(row[c]);
      if (v != v) nan = true;
      m = v > m ? v : m;
    }
    for (int o = 16; o; o >>= 1) {
      double y = __shfl_xor_sync(0xffffffffu, m, o);
      m = y > m ? y : m;
    }
    nan = __any_sync(0xffffffffu, nan);
    if (lane == 0) out[r] = nan ? __longlong_as_double(0x7ff8000000000000ll) : m;
  }
}

__global__ void lens_column_kernel(const double* __restrict__ X, int64_t n, int64_t d,
                                   int64_t col, double* __restrict__ out) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x)
    out[r] = X[r * d + col];
}

// ---- normalisation ---------------------------------------------------------
// minmax: per-column min/max (exact), span==0 -> 1, (x - lo) / span.
__global__ void colminmax_kernel(const double* __restrict__ X, int64_t n, int64_t d,
                                 double* __restrict__ lo, double* __restrict__ hi) {
  // one block per column chunk of 32 columns; threads stride rows
  int64_t c = (int64_t)blockIdx.x * 32 + (threadIdx.x & 31);
  int rgrp = threadIdx.x >> 5, ngrp = blockDim.x >> 5;
  double mn = __longlong_as_double(0x7ff0000000000000ll), mx = -mn;
  bool nan = false;
  if (c < d) {
    for (int64_t r = rgrp; r < n; r += ngrp) {
      double v = X[r * d + c];
      if (v != v) nan = true;
      mn = v < mn ? v : mn;
      mx = v > mx ? v : mx;
    }
  }
  __shared__ double smn[32][33], smx[32][33];
  __shared__ int snan[32][33];
  smn[rgrp][threadIdx.x & 31] = mn;
  smx[rgrp][threadIdx.x & 31] = mx;
  snan[rgrp][threadIdx.x & 31] = nan;
  __syncthreads();
  if (rgrp == 0 && c < d) {
    for (int g = 1; g < ngrp; ++g) {
      double a = smn[g][threadIdx.x], b = smx[g][threadIdx.x];
      mn = a < mn ? a : mn;
      mx = b > mx ? b : mx;
      nan = nan || snan[g][threadIdx.x];
    }
    double qnan = __longlong_as_double(0x7ff8000000000000ll);
    lo[c] = nan ? qnan : mn;
    hi[c] = nan ? qnan : mx;
  }
}

__global__ void minmax_apply_kernel(const double* __restrict__ X, int64_t n, int64_t d,
                                    const double* __restrict__ lo,
                                    const double* __restrict__ hi, double* __restrict__ out) {
  int64_t total = n * d;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t c = i % d;
    double span = __dsub_rn(hi[c], lo[c]);
    if (span == 0.0) span = 1.0;
    out[i] = __ddiv_rn(__dsub_rn(X[i], lo[c]), span);
  }
}

__global__ void l2_apply_kernel(const double* __restrict__ X, int64_t n, int64_t d,
                                const double* __restrict__ norms, double* __restrict__ out) {
  int64_t total = n * d;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    double nv = norms[i / d];
    if (nv == 0.0) nv = 1.0;
    out[i] = __ddiv_rn(X[i], nv);
  }
}

int lens_l2(const double* X, int64_t n, int64_t d, double* out, cudaStream_t stream) {
  PwProgram prog;
  BM_TRY(make_pw_program(d, &prog));
  int packed = prog.n_leaves == 1 || prog.n_leaves == 2 || prog.n_leaves == 4;
  for (int i = 0; i < prog.n_leaves; ++i) packed &= prog.leaf[i].len >= 8 && prog.leaf[i].len <= 135;
  const int rpw = packed ? 4 / prog.n_leaves : 1;
  int64_t blocks = ceil_div(ceil_div(n, rpw), kLensWarps);
  int64_t cap = (int64_t)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  lens_l2_kernel<<<(unsigned)blocks, kLensWarps * 32, 0, stream>>>(X, n, d, out, prog, packed);
  BM_CHECK_LAUNCH();
  return BM_OK;
}

}  // namespace
}  // namespace bm

using namespace bm;

extern "C" int bm_lens_f64(int kind, const double* d_X, int64_t n, int64_t d, int64_t col,
                           double* d_out, void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  BM_REQUIRE(n >= 0 && d >= 1, "bad lens shape n=%lld d=%lld", (long long)n, (long long)d);
  if (n == 0) return BM_OK;
  BM_REQUIRE(d_X && d_out, "null pointer");
  int64_t blocks;
  switch (kind) {
    case BM_LENS_COLUMN:
      BM_REQUIRE(col >= 0 && col < d, "column %lld out of range", (long long)col);
      blocks = std::min<int64_t>(ceil_div(n, 256), (int64_t)num_sms() * 8);
      lens_column_kernel<<<(unsigned)blocks, 256, 0, stream>>>(d_X, n, d, col, d_out);
      BM_CHECK_LAUNCH();
      return BM_OK;
    case BM_LENS_L2:
      return lens_l2(d_X, n, d, d_out, stream);
    case BM_LENS_LINF:
      blocks = std::min<int64_t>(ceil_div(n, 8), (int64_t)num_sms() * 16);
      lens_linf_kernel<<<(unsigned)blocks, 256, 0, stream>>>(d_X, n, d, d_out);
      BM_CHECK_LAUNCH();
      return BM_OK;
    default:
      set_error("unknown lens kind %d", kind);
      return BM_ERR_DATA;
  }
}

extern "C" int bm_normalize_f64(int scheme, const double* d_X, int64_t n, int64_t d,
                                double* d_out, void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  BM_REQUIRE(n >= 0 && d >= 1, "bad shape");
  BM_REQUIRE(scheme == 1 || scheme == 2, "unknown normalization scheme %d", scheme);
  if (n == 0) return BM_OK;
  BM_REQUIRE(d_X && d_out && d_X != d_out, "bad pointers");
  int64_t blocks = std::min<int64_t>(ceil_div(n * d, 256), (int64_t)num_sms() * 16);
  if (scheme == 1) {
    Scratch s;
    BM_TRY(scratch_alloc(s, 2 * d * sizeof(double), stream));
    double* lo = s.as<double>();
    double* hi = lo + d;
    colminmax_kernel<<<(unsigned)ceil_div(d, 32), 1024, 0, stream>>>(d_X, n, d, lo, hi);
    BM_CHECK_LAUNCH();
    minmax_apply_kernel<<<(unsigned)blocks, 256, 0, stream>>>(d_X, n, d, lo, hi, d_out);
    BM_CHECK_LAUNCH();
  } else {
    Scratch s;
    BM_TRY(scratch_alloc(s, n * sizeof(double), stream));
    BM_TRY(lens_l2(d_X, n, d, s.as<double>(), stream));
    l2_apply_kernel<<<(unsigned)blocks, 256, 0, stream>>>(d_X, n, d, s.as<double>(), d_out);
    BM_CHECK_LAUNCH();
  }
  return BM_OK;
}
