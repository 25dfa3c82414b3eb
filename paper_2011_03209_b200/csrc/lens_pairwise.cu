// lens_pairwise.cu — the O(N x M) lenses: eccentricity and density
// (nervemap/filters.py:103-150).
//
//   d_ij        = scipy cdist: sqrt of the sequential fp64 sum of (x_i - y_j)^2
//                 (no FMA), y_j over the target rows (all points, or the
//                 seed-1729 subsample of 50k rows when N is larger)
//   eccentricity p = 1 : mean_j d_ij           (numpy pairwise row sum / M)
//                p = 2 : sqrt(mean_j d_ij^2)   (numpy fast paths: square, sqrt)
//                p = inf: max_j d_ij
//                other p: pow(mean_j pow(d, p), 1/p)  (CUDA pow: ulp-level)
//   density          : sum_j exp(-(d_ij^2) / (2 sigma^2))  (CUDA exp: ulp-level)
//   nearest neighbour: min_{j, row_j != row_i} d_ij (the default bandwidth's
//                      1000-point helper, filters.py:103-118)
// Every d_ij is bit-identical to scipy's; p in {1, 2, inf} and the nearest
// neighbour are bit-identical to the reference; exp/pow may differ by an ulp.
//
// One CTA per 64 query rows; target rows stream in chunks of 64: exact d for
// the 64 x 64 tile (4 x 4 per thread, dims staged transposed in shared
// memory), then one thread per query row folds its 64 values in target order
// into numpy's pairwise-sum state (leaf program over M, 8 strided
// accumulators per leaf, explicit stack).
#include <math.h>

#include <algorithm>
#include <vector>

#include "common.cuh"

namespace bm {
namespace {

constexpr int kLq = 64;   // query rows per CTA
constexpr int kLt = 64;   // target rows per chunk
constexpr int kLk = 32;   // dims per staging step
constexpr int kLd = 65;   // padded leading dimension (doubles)
constexpr int kLStack = 20;
constexpr size_t kLSmem = (size_t)(2 * kLk * kLd + kLq * kLd) * sizeof(double);

enum { kEccSum = 0, kEccSq = 1, kEccPow = 2, kEccMax = 3, kDensity = 4, kNnMin = 5 };

template <int MODE>
__global__ void __launch_bounds__(256)
pairwise_lens_kernel(const double* __restrict__ X, int64_t d, const int64_t* __restrict__ qrows,
                     int64_t nq, const int64_t* __restrict__ trows, int64_t m,
                     const PwLeaf* __restrict__ leaves, double param, double* __restrict__ out) {
  extern __shared__ double lsm[];
  double* As = lsm;                  // [kLk][kLd] query dims
  double* Bs = lsm + kLk * kLd;      // [kLk][kLd] target dims
  double* Ds = lsm + 2 * kLk * kLd;  // [kLq][kLd] distances of the chunk
  const int t = threadIdx.x, tx = t & 15, ty = t >> 4;
  const int64_t q0 = (int64_t)blockIdx.x * kLq;
  const int nqv = (int)min((int64_t)kLq, nq - q0);
  // consumer state (threads 0..63: one query row each)
  double r8[8], st[kLStack], res = 0.0, ext = MODE == kNnMin ? INFINITY : -INFINITY;
#pragma unroll
  for (int j = 0; j < 8; ++j) r8[j] = 0.0;
#pragma unroll
  for (int j = 0; j < kLStack; ++j) st[j] = 0.0;
  int li = 0;
  const int64_t my_row = (t < nqv) ? (qrows ? qrows[q0 + t] : q0 + t) : -1;

  for (int64_t c0 = 0; c0 < m; c0 += kLt) {
    const int ntv = (int)min((int64_t)kLt, m - c0);
    double acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
    for (int64_t k0 = 0; k0 < d; k0 += kLk) {
      const int len = (int)min((int64_t)kLk, d - k0);
      __syncthreads();
      for (int i = t; i < kLq * kLk; i += blockDim.x) {
        const int r = i / kLk, c = i % kLk;
        double a = 0.0, b = 0.0;
        if (c < len && r < nqv) a = X[(qrows ? qrows[q0 + r] : q0 + r) * d + k0 + c];
        if (c < len && r < ntv) b = X[(trows ? trows[c0 + r] : c0 + r) * d + k0 + c];
        As[c * kLd + r] = a;
        Bs[c * kLd + r] = b;
      }
      __syncthreads();
      for (int c = 0; c < len; ++c) {
        double av[4], bv[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) av[a] = As[c * kLd + ty + 16 * a];
#pragma unroll
        for (int b = 0; b < 4; ++b) bv[b] = Bs[c * kLd + tx + 16 * b];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const double df = __dsub_rn(av[a], bv[b]);
            acc[a][b] = __dadd_rn(acc[a][b], __dmul_rn(df, df));
          }
      }
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) Ds[(ty + 16 * a) * kLd + tx + 16 * b] = __dsqrt_rn(acc[a][b]);
    __syncthreads();
    if (t < nqv) {
      if (MODE == kEccMax || MODE == kNnMin) {
        for (int j = 0; j < ntv; ++j) {
          const double v = Ds[t * kLd + j];
          if (MODE == kEccMax) {
            ext = (v > ext || v != v) ? v : ext;  // numpy max propagates NaN
          } else if ((trows ? trows[c0 + j] : c0 + j) != my_row) {
            ext = (v < ext || v != v) ? v : ext;
          }
        }
      } else {
        for (int g = 0; g < kLt / 8; ++g) {
          const int64_t gb = c0 + 8 * g;
          if (gb >= m) break;
          const int nv = (int)min((int64_t)8, m - gb);
          double v[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const double x = j < nv ? Ds[t * kLd + 8 * g + j] : 0.0;
            if (MODE == kEccSum) v[j] = x;
            else if (MODE == kEccSq) v[j] = __dmul_rn(x, x);
            else if (MODE == kEccPow) v[j] = pow(x, param);
            else v[j] = exp(__ddiv_rn(-__dmul_rn(x, x), param));  // kDensity: param = 2 sigma^2
          }
          // numpy pairwise_sum over the M targets: the 8-group lies in one leaf
          // (leaf starts are multiples of 8), accumulator j <-> position j
          const PwLeaf L = leaves[li];
          const int pos = (int)(gb - L.start);
          const int body = L.len - (L.len & 7);
          bool finish = false;
          if (L.len < 8) {
            double rr = -0.0;
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (j < L.len) rr = __dadd_rn(rr, v[j]);
            res = rr;
            finish = true;
          } else if (pos < body) {
#pragma unroll
            for (int j = 0; j < 8; ++j) r8[j] = pos == 0 ? v[j] : __dadd_rn(r8[j], v[j]);
            if (pos + 8 == body) {
              res = __dadd_rn(__dadd_rn(__dadd_rn(r8[0], r8[1]), __dadd_rn(r8[2], r8[3])),
                              __dadd_rn(__dadd_rn(r8[4], r8[5]), __dadd_rn(r8[6], r8[7])));
              finish = body == L.len;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (j < L.len - body) res = __dadd_rn(res, v[j]);
            finish = true;
          }
          if (finish) {
#pragma unroll
            for (int j = kLStack - 1; j > 0; --j) st[j] = st[j - 1];
            st[0] = res;
            for (int q = 0; q < L.pops; ++q) {
              st[0] = __dadd_rn(st[1], st[0]);
#pragma unroll
              for (int j = 1; j < kLStack - 1; ++j) st[j] = st[j + 1];
            }
            ++li;
          }
        }
      }
    }
  }
  if (t < nqv) {
    double o;
    if (MODE == kEccMax || MODE == kNnMin) {
      o = ext;
    } else {
      const double s = __dadd_rn(0.0, st[0]);  // numpy add.reduce of the row
      if (MODE == kDensity) o = s;
      else {
        const double mean = __ddiv_rn(s, (double)m);
        if (MODE == kEccSum) o = mean;
        else if (MODE == kEccSq) o = __dsqrt_rn(mean);
        else o = pow(mean, 1.0 / param);
      }
    }
    out[q0 + t] = o;
  }
}

template <int MODE>
int launch_lens(const double* X, int64_t d, const int64_t* q, int64_t nq, const int64_t* tr,
                int64_t m, const PwLeaf* leaves, double param, double* out, cudaStream_t s) {
  BM_TRY(ensure_dyn_smem((const void*)pairwise_lens_kernel<MODE>, (int)kLSmem));
  pairwise_lens_kernel<MODE><<<(unsigned)ceil_div(nq, kLq), 256, kLSmem, s>>>(
      X, d, q, nq, tr, m, leaves, param, out);
  BM_CHECK_LAUNCH();
  return BM_OK;
}

}  // namespace
}  // namespace bm

using namespace bm;

extern "C" int bm_pairwise_lens(int kind, double param, const double* d_X, int64_t n, int64_t d,
                                const int64_t* d_qrows, int64_t nq, const int64_t* d_trows,
                                int64_t m, double* d_out, void* stream_) {
  cudaStream_t s = (cudaStream_t)stream_;
  BM_REQUIRE(n >= 0 && d >= 1 && nq >= 0 && m >= 0, "bad shapes");
  BM_REQUIRE(kind >= BM_PLENS_ECC_MEAN && kind <= BM_PLENS_NN_MIN, "unknown pairwise lens %d",
             kind);
  if (nq == 0) return BM_OK;
  BM_REQUIRE(m >= 1, "pairwise lens needs at least one target row");
  BM_REQUIRE(d_X && d_out, "null device pointer");
  BM_REQUIRE(nq < (1ll << 31) * kLq && m < (1ll << 31), "too many rows");
  std::vector<PwLeaf> lv = pw_plan((int)m);
  int depth = 0, maxd = 0;
  for (auto& x : lv) {
    maxd = std::max(maxd, ++depth);
    depth -= x.pops;
  }
  BM_REQUIRE(maxd <= kLStack, "target count %lld too large", (long long)m);
  Scratch sl;
  BM_TRY(scratch_alloc(sl, lv.size() * sizeof(PwLeaf), s));
  BM_CHECK_CUDA(cudaMemcpyAsync(sl.ptr, lv.data(), lv.size() * sizeof(PwLeaf),
                                cudaMemcpyHostToDevice, s));
  const PwLeaf* L = sl.as<PwLeaf>();
  switch (kind) {
    case BM_PLENS_ECC_MEAN:
      return launch_lens<kEccSum>(d_X, d, d_qrows, nq, d_trows, m, L, param, d_out, s);
    case BM_PLENS_ECC_RMS:
      return launch_lens<kEccSq>(d_X, d, d_qrows, nq, d_trows, m, L, param, d_out, s);
    case BM_PLENS_ECC_POW:
      BM_REQUIRE(param >= 1.0 && param < INFINITY, "eccentricity exponent must be finite >= 1");
      return launch_lens<kEccPow>(d_X, d, d_qrows, nq, d_trows, m, L, param, d_out, s);
    case BM_PLENS_ECC_MAX:
      return launch_lens<kEccMax>(d_X, d, d_qrows, nq, d_trows, m, L, param, d_out, s);
    case BM_PLENS_DENSITY:
      BM_REQUIRE(param > 0.0, "density needs 2 sigma^2 > 0");
      return launch_lens<kDensity>(d_X, d, d_qrows, nq, d_trows, m, L, param, d_out, s);
    default:
      return launch_lens<kNnMin>(d_X, d, d_qrows, nq, d_trows, m, L, param, d_out, s);
  }
}
