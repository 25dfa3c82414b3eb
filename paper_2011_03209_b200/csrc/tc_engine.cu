// tc_engine.cu — eps-adjacency on the 5th-gen tensor cores (tcgen05 + TMEM +
// TMA), with an exact fp64 recheck of the pairs the tensor cores cannot
// decide. Reference decision: sqrt(fp64 sum (x_i - x_j)^2 in the element's
// order) <= eps (clustering.py:113,137-139,166-187).
//
// Why integers: the reference's decision is an fp64 comparison, so the
// candidate distance must come with a RIGOROUS error bound. Floating-point
// MMA accumulation has no documented rounding model; integer MMA
// (kind::i8, s32 accumulate) is exact. Each element is centred (c_k) and
// quantised to 22-bit fixed point q = rint((x - c_k) / s_k), |q| < 2^21, split
// into three limbs q = H*2^14 + M*2^7 + L (H signed byte, M, L in [0,127]).
// Six of the nine limb products run on the tensor cores, accumulated per
// shift class in three TMEM accumulators (N = 128 columns each):
//   A0 = H.H   A1 = H.M + M.H   A2 = H.L + M.M + L.H
// The omitted A3 = M.L + L.M and L.L terms are non-negative and bounded
// (Cauchy-Schwarz on per-tile limb norms), so D2c = N_i + N_j - 2 (A0<<28 + A1<<21 + A2<<14)
// brackets D2_q = |q_i - q_j|^2 from both sides with known slack.
// Per point the quantisation error e_i = |x_i - c - s q_i| is measured in
// fp64 (tile maxima, tile_u); by the triangle inequality
// |d_true - s sqrt(D2_q)| <= e_i + e_j, and the reference's fp64 result
// satisfies |d_ref - d_true| <= gamma d_true, gamma = 1.5 (d+16) 2^-53.
// Each tile pair gets thresholds t_in <= t_out on D2c (tile_thr_kernel):
//   D2c <= t_in  -> certainly inside (d_ref <= eps)
//   D2c >  t_out -> certainly outside
//   otherwise    -> queued and decided by the exact fp64 recheck kernel in
//                   the element's summation order (~3e-5 of the pairs).
// In the epilogue one int32 per pair decides: y = 2^7 a0 + a1 + (a2 >> 7)
// - floor(N_j / 2^22) against per-row integer bounds r_in/r_out (the
// floors and shifts are absorbed by +-2 margins, see tile_thr_kernel).
//
// Kernel (tc_adjacency_kernel): persistent, one CTA per SM, 768 threads.
//   warp 0      TMA producer: per tile the three B limb planes (128 rows x
//               Kpad bytes each, SWIZZLE_128B 3-D tensor map) into a 2-stage
//               ring, plus the tile's info (column norms, thresholds, J) by
//               bulk copy into a 3-deep ring
//   warp 1      MMA issuer (whole warp, elect.sync): tcgen05.mma.cta_group::1
//               .kind::i8, M = N = 128, K = 32; accumulator-major order:
//               phase 1 (A0, A1) then phase 2 (A2), each released separately
//   warp 2      TMEM allocator (512 columns: A's H/M planes 128 + 3 x 128)
//   warps 4-19  epilogue: 4 warps per TMEM lane quarter x 32 columns each;
//               tcgen05.ld -> y -> two sign bits per pair -> bitmap word,
//               row counts, nonempty flag, undecided pairs to the queue
//   warps 20-23 A loaders: H/M limb planes of the unit's row tile into TMEM
//               (tcgen05.st; the MMA reads A from TMEM), L plane by TMA to smem
// A work unit is (element, 128-row tile I, <= 32 kept column tiles J) over
// the pruned tile list (dbscan.cu); column counts of off-diagonal tiles come
// from colcount_kernel, then recheck_kernel decides the queued pairs.
#include <cuda.h>

#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "dbscan.cuh"

namespace bm {

namespace {

constexpr int kBM = 128;        // A rows (TMEM lanes)
constexpr int kBN = 128;        // B rows per tile (MMA N)
constexpr int kKC = 128;        // bytes per swizzle-128B row chunk
constexpr int kStages = 2;      // B ring depth (full-K B tiles)
constexpr int kInfo = 3;        // per-tile info ring depth (smem)
constexpr int kEpiWarps = 16;   // epilogue warps 4..19 (4 per TMEM lane quarter)
constexpr int kEpiCols = kBN / (kEpiWarps / 4);  // columns per epilogue warp (32)
constexpr int kLoadWarps = 4;   // A-loader warps 20..23
constexpr int kThreads = 128 + 32 * (kEpiWarps + kLoadWarps);
constexpr int kLimb = 7;        // bits of the M and L limbs
constexpr int kQBits = 2 * kLimb + 7;   // |q| <= 2^21 - 1: H = q >> 14 is a signed byte
constexpr int kYShift = 3 * kLimb + 1;  // y is in units of 2^22 of D2


// ---------------------------------------------------------------------------
// PTX helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
// try_wait with a suspend-time hint: a waiting warp sleeps until the phase
// completes (or the hint expires) instead of re-issuing try_wait, which left
// the spinning warps (A loaders, producer, waiting epilogue warps) with ~30%
// of the SM's issued instructions, taken from the epilogue's decisions
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity), "r"(0x989680u)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"((uint64_t)src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
// One elected lane of a converged warp issues; operands stay warp-uniform.
__device__ __forceinline__ void mma_ts_elect(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_ss_elect(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void commit_elect(uint64_t* b) {
  asm volatile(
      "{\n"
      ".reg .pred e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
      "}\n" ::"r"(smem_u32(b))
      : "memory");
}
__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Shared-memory matrix descriptor: K-major, SWIZZLE_128B, 8-row groups 1024 B
// apart (SBO), version 1 (sm_100).
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                 // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;       // SBO
  d |= (uint64_t)1 << 46;                 // version
  d |= (uint64_t)2 << 61;                 // SWIZZLE_128B
  return d;
}

// Instruction descriptor, kind::i8: D=s32, A/B K-major, M=128, N=64.
__host__ __device__ constexpr uint32_t idesc_i8(bool a_signed, bool b_signed) {
  return (2u << 4) | ((a_signed ? 1u : 0u) << 7) | ((b_signed ? 1u : 0u) << 10) |
         ((uint32_t)(kBN >> 3) << 17) | ((uint32_t)(kBM >> 4) << 24);
}

struct TileThr {
  int32_t k_in, k_out;  // integer fast-path offsets (kNever: never certain)
  double t_in, t_out;   // exact-path thresholds on D2c
};
constexpr int32_t kNever = 0x7fffffff;
#ifdef BM_TC_PROFILE
#define EP_START() long long te = clock64()
#define EP_MARK(i) (ep[i] += clock64() - te, te = clock64())
#else
#define EP_START() ((void)0)
#define EP_MARK(i) ((void)0)
#endif
constexpr int kYMax = 850000000;  // bound on |y| (kLimb = 7, Kpad <= 256): see tc_engine header

struct TcParams {
  ElemTables et;
  const TileThr* thr;     // per kept tile (slot)
  const TileRef* tiles;   // kept tiles of the batch (absolute slot -> k, I, J)
  int64_t slot0;          // first slot of the window (adj, thr, queue use slot - slot0)
  const TileUnit* units;
  int64_t n_units;
  const int64_t* nq;      // per padded row: sum q^2
  const int32_t* cq;      // per padded row: floor(sum q^2 / 2^kYShift)
  const double* tile_u;   // per 128-row tile: max quantisation error / s_k (quantised units)
  const int32_t* tbase;   // per element: first global 128-row tile index
  const double* a_in;     // per element: eps / (1 + gamma) / s_k
  const double* a_out;    // per element: eps / (1 - gamma) / s_k
  const uint32_t* limb_sq;  // per 128-row tile: max over rows of |M|^2, |L|^2 (limb planes)
  int nkc;                // Kpad / 128
  uint32_t* adj;
  int32_t* nonempty;      // per window slot: 1 if the tile holds any bit (zeroed by the host)
  int32_t* cnt;           // eps-neighbour counts per padded row (self included)
  int4* queue;            // undecided pairs: (p_i, p_j, slot, element)
  const uint8_t* planes;  // limb planes [3][P][kpad]
  int64_t P;
  unsigned long long* qcount;
  unsigned long long qcap;
  long long* prof;        // optional [grid][8] cycle counters of the MMA warp (B200MAP_TC_PROFILE)
};

constexpr double kBig = 4.0e18;

// Bounds of the omitted non-negative terms from the tiles' limb norms
// (Cauchy-Schwarz): L.L <= |L_i||L_j|, A3 = M.L + L.M <= |M_i||L_j| + |L_i||M_j|,
// rounded up (per-tile maxima of the row norms; far below the worst case
// 127^2 Kpad, which narrows the recheck band ~3x).
__device__ __forceinline__ double limb_norm(const TcParams& P, int64_t t, int which) {
  return __dsqrt_ru((double)P.limb_sq[2 * t + which]);
}
__device__ __forceinline__ double ll_bound(const TcParams& P, int64_t tI, int64_t tJ) {
  return __dmul_ru(limb_norm(P, tI, 1), limb_norm(P, tJ, 1)) * (1.0 + 1e-12);
}
__device__ __forceinline__ double a3_bound(const TcParams& P, int64_t tI, int64_t tJ) {
  return __dadd_ru(__dmul_ru(limb_norm(P, tI, 0), limb_norm(P, tJ, 1)),
                   __dmul_ru(limb_norm(P, tI, 1), limb_norm(P, tJ, 0))) * (1.0 + 1e-12);
}

// fp64 thresholds on D2c for one (row tile, column tile) pair; the +-64
// margins cover the fp64 rounding of S = N_i + N_j and of the fast D2.
__device__ __forceinline__ void thresholds(const TcParams& P, int k, int64_t tI, int64_t tJ,
                                           double& t_in, double& t_out) {
  const double du = P.tile_u[tI] + P.tile_u[tJ];
  if (!(du < 1e300)) {  // NaN/inf inputs: every pair of the tile goes to the recheck
    t_in = -kBig;
    t_out = kBig;
    return;
  }
  const double ri = P.a_in[k] - du;
  t_in = ri > 0.0 ? ri * ri * (1.0 - 1e-12) - 64.0 : -kBig;
  const double ro = P.a_out[k] + du;
  t_out = ro * ro * (1.0 + 1e-12) + 2.0 * ll_bound(P, tI, tJ) + 64.0;
}

// Per bitmap tile pair: exact thresholds t_in/t_out on D2c and the integer
// offsets of the fast path (see the epilogue): with U = 2^kYShift and
// niU = floor(N_i/U),
//   r_in  = niU + ceil(-t_in/U) + 3   >= (N_i - t_in)/U + 2
//   r_out = niU + floor(-(t_out + a3)/U) - 2 <= (N_i - t_out - a3)/U - 1
// with a3 = 2^(kLimb+1) a3_bound (the A3 term's weight in D2).
__global__ void tile_thr_kernel(TcParams P, int64_t n_tiles, TileThr* __restrict__ out) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_tiles) return;
  const TileRef tr = P.tiles[P.slot0 + g];
  const int k = tr.k, I = tr.I, J = tr.J;
  double t_in, t_out;
  thresholds(P, k, P.tbase[k] + I, P.tbase[k] + J, t_in, t_out);
  TileThr th;
  th.t_in = t_in;
  th.t_out = t_out;
  const double sc = 1.0 / (double)(1ll << kYShift);
  th.k_in = t_in > -1e18 ? (int32_t)fmin(fmax(ceil(-t_in * sc) + 3.0, -1073741824.0), 1073741824.0)
                         : kNever;
  // clamping k_in down is conservative (fewer certain-inside pairs); k_out
  // must never be raised, so out-of-range values disable the certain-outside test
  const double a3 = (double)(2 << kLimb) * a3_bound(P, P.tbase[k] + I, P.tbase[k] + J);
  const double ko = floor(-(t_out + a3) * sc) - 2.0;
  th.k_out = (t_out < 1e18 && ko >= -1073741824.0) ? (int32_t)ko : kNever;
  out[g] = th;
}

// one step of the in-warp 32x32 bit-matrix transpose (lane i holds row i)
__device__ __forceinline__ uint32_t bit_transpose_step(uint32_t w, int s, uint32_t m, int lane) {
  const uint32_t t = __shfl_xor_sync(0xffffffffu, w, s);
  return (lane & s) ? ((w & ~m) | ((t >> s) & m)) : ((w & m) | ((t << s) & ~m));
}


__device__ __forceinline__ void tmem_ld16(uint32_t taddr, int32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
        "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
      "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(
          taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
      "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]),
      "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]),
      "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}

// Warp roles (512 threads): 0 TMA producer, 1 MMA issuer, 2 TMEM allocator,
// 4..11 epilogue, 12..15 A loaders (TMEM lane quarter = warp % 4).
// TMEM columns: [0, kpad/2) A limb planes H|M (row = lane, 4 int8 of K per
// column); [128, 512) accumulators A0 | A1 | A2 (N = 128 columns each).
// Shared memory: A limb plane L (SW128 K-major, resident per unit) and a
// 2-stage ring of full-K B tiles (3 limb planes x 128 rows).
template <int NKC>
__global__ void __launch_bounds__(kThreads, 1)
tc_adjacency_kernel(const __grid_constant__ CUtensorMap qmap, TcParams P) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // the SW128 operand tiles need 1024-byte alignment; the dynamic window starts
  // after the 1 KB reserved block, which is 1024-aligned (checked, not assumed)
  if ((smem_u32(smem_raw) & 1023u) != 0u) __trap();
  uint8_t* smem = smem_raw;
  constexpr int nkc = NKC;
  constexpr int kpad = nkc * kKC;
  const uint32_t blk = (uint32_t)kBN * kKC;            // one (plane, K-chunk) block: 16 KB
  const uint32_t aL_bytes = (uint32_t)nkc * blk;
  const uint32_t b_plane_bytes = (uint32_t)nkc * blk;
  const uint32_t b_bytes = 3 * b_plane_bytes;
  uint8_t* sAL = smem;
  uint8_t* sB = smem + aL_bytes;
  uint64_t* bars = (uint64_t*)(sB + kStages * b_bytes);
  uint64_t* a_tm_full = bars + 0;             // H/M planes stored to TMEM (4 loader warps)
  uint64_t* a_sm_full = bars + 1;             // L plane landed in smem (TMA tx)
  uint64_t* a_empty = bars + 2;               // MMAs of the unit done
  uint64_t* b_full = bars + 3;                // [kStages]
  uint64_t* b_empty = b_full + kStages;       // [kStages]
  uint64_t* acc_full = b_empty + kStages;     // [2]: (A0, A1), A2
  uint64_t* acc_empty = acc_full + 2;         // [2]
  uint32_t* tmem_slot = (uint32_t*)(acc_empty + 2);
  // per-tile info ring, filled ahead by the producer: floor(N_j/U) of the
  // tile's 128 columns (bulk TMA) + the tile's integer threshold offsets
  struct TileInfo {
    int32_t cq[kBN];
    int2 th;
    int32_t J;  // column tile
    int32_t pad;
  };
  TileInfo* info = (TileInfo*)(((uintptr_t)(tmem_slot + 4) + 15) & ~(uintptr_t)15);
  uint64_t* info_full = (uint64_t*)(info + kInfo);        // [kInfo]
  uint64_t* info_empty = info_full + kInfo;               // [kInfo]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(a_tm_full, kLoadWarps);
    mbar_init(a_sm_full, 1);
    mbar_init(a_empty, 1);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(b_full + s, 1);
      mbar_init(b_empty + s, 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(acc_full + s, 1);
      mbar_init(acc_empty + s, kEpiWarps);
    }
    for (int s = 0; s < kInfo; ++s) {
      mbar_init(info_full + s, 1);
      mbar_init(info_empty + s, kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t tacc0 = tmem_base + 128;  // accumulator columns

  if (warp == 0) {
    // ------------------------------------------------------------ producer (TMA)
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&qmap) : "memory");
      // per-slot phases as bit masks (a dynamically indexed array would live in local memory)
      uint32_t stage = 0, ph_empty = 0, a_empty_ph = 0;
      uint32_t islot = 0, ph_info = 0;
      for (int64_t u = blockIdx.x; u < P.n_units; u += gridDim.x) {
        const TileUnit un = P.units[u];
        const int pb = P.et.pbase[un.k];
        // A limb plane L of row tile I (resident for the unit)
        mbar_wait(a_empty, a_empty_ph ^ 1);
        a_empty_ph ^= 1;
        mbar_expect_tx(a_sm_full, aL_bytes);
        for (int c = 0; c < nkc; ++c)
          for (int h = 0; h < 2; ++h)
            tma_load_3d(sAL + c * blk + h * 64 * kKC, &qmap, a_sm_full, c * kKC,
                        pb + un.I * kBM + h * 64, 2);
        for (int t = 0; t < un.cnt; ++t) {
          const int b = P.tiles[un.off + t].J;
          // tile info for the epilogue (runs ahead by up to kInfo tiles)
          mbar_wait(info_empty + islot, ((ph_info >> islot) & 1u) ^ 1u);
          ph_info ^= 1u << islot;
          info[islot].th = *reinterpret_cast<const int2*>(P.thr + (un.off + t - P.slot0));
          info[islot].J = b;
          mbar_expect_tx(info_full + islot, kBN * 4);
          bulk_load(info[islot].cq, P.cq + pb + b * kBN, kBN * 4, info_full + islot);
          islot = (islot + 1) % kInfo;
          mbar_wait(b_empty + stage, ((ph_empty >> stage) & 1u) ^ 1u);
          ph_empty ^= 1u << stage;
          mbar_expect_tx(b_full + stage, b_bytes);
          uint8_t* dst = sB + stage * b_bytes;
          for (int pl = 0; pl < 3; ++pl)
            for (int c = 0; c < nkc; ++c)
              for (int h = 0; h < 2; ++h)
                tma_load_3d(dst + pl * b_plane_bytes + c * blk + h * 64 * kKC, &qmap,
                            b_full + stage, c * kKC, pb + b * kBN + h * 64, pl);
          stage = (stage + 1) % kStages;
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // The whole warp runs the loop so every descriptor lives in uniform
    // registers; one elected lane issues (elect.sync inside the asm).
    constexpr uint32_t ID_SS = idesc_i8(true, true);
    constexpr uint32_t ID_SU = idesc_i8(true, false);
    constexpr uint32_t ID_US = idesc_i8(false, true);
    constexpr uint32_t ID_UU = idesc_i8(false, false);
    constexpr int KSTEPS = NKC * 4;
    constexpr uint32_t NCOL_PLANE = NKC * 32;          // TMEM columns per limb plane
    constexpr uint32_t BLK = kBN * kKC;                // bytes of one (plane, K-chunk) block
    constexpr uint32_t BPLANE = NKC * BLK;
    uint32_t a_ph = 0, stage = 0, ph_full = 0;  // per-stage phase bits
    uint32_t ph_acc[2] = {0, 0};
    const uint32_t aH = tmem_base, aM = tmem_base + NCOL_PLANE;
    const uint64_t aL_desc = smem_desc(smem_u32(sAL));
    const uint64_t b_desc0 = smem_desc(smem_u32(sB));
    long long prof_a = 0, prof_b = 0, prof_e0 = 0, prof_e1 = 0;
    const long long prof_t0 = clock64();
    for (int64_t u = blockIdx.x; u < P.n_units; u += gridDim.x) {
      const TileUnit un = P.units[u];
      long long tw = clock64();
      mbar_wait(a_tm_full, a_ph);
      mbar_wait(a_sm_full, a_ph);
      prof_a += clock64() - tw;
      a_ph ^= 1;
      tc_fence_after();
      for (int t = 0; t < un.cnt; ++t) {
        tw = clock64();
        mbar_wait(b_full + stage, (ph_full >> stage) & 1u);
        prof_b += clock64() - tw;
        ph_full ^= 1u << stage;
        const uint64_t bd = b_desc0 + ((stage * 3 * BPLANE) >> 4);
        // descriptor of (B plane pl, K-step ks): start address advances in 16-byte units
#define BDESC(pl, ks) (bd + ((uint64_t)((pl) * BPLANE + ((ks) >> 2) * BLK + ((ks) & 3) * 32) >> 4))
        // phase 1 — shift classes 2^32, 2^24: A0 = H.H, A1 = H.M + M.H
        tw = clock64();
        mbar_wait(acc_empty + 0, ph_acc[0] ^ 1);
        prof_e0 += clock64() - tw;
        tc_fence_after();
#pragma unroll
        for (int ks = 0; ks < KSTEPS; ++ks) {
          mma_ts_elect(tacc0 + 0 * kBN, aH + ks * 8, BDESC(0, ks), ID_SS, ks > 0);
          mma_ts_elect(tacc0 + 1 * kBN, aH + ks * 8, BDESC(1, ks), ID_SU, ks > 0);
          mma_ts_elect(tacc0 + 1 * kBN, aM + ks * 8, BDESC(0, ks), ID_US, 1u);
        }
        commit_elect(acc_full + 0);
        // phase 2 — shift class 2^16: A2 = H.L + M.M + L.H (L of A from smem)
        tw = clock64();
        mbar_wait(acc_empty + 1, ph_acc[1] ^ 1);
        prof_e1 += clock64() - tw;
        tc_fence_after();
#pragma unroll
        for (int ks = 0; ks < KSTEPS; ++ks) {
          mma_ts_elect(tacc0 + 2 * kBN, aH + ks * 8, BDESC(2, ks), ID_SU, ks > 0);
          mma_ts_elect(tacc0 + 2 * kBN, aM + ks * 8, BDESC(1, ks), ID_UU, 1u);
          mma_ss_elect(tacc0 + 2 * kBN,
                       aL_desc + ((uint64_t)((ks >> 2) * BLK + (ks & 3) * 32) >> 4),
                       BDESC(0, ks), ID_US, 1u);
        }
#undef BDESC
        commit_elect(acc_full + 1);
        commit_elect(b_empty + stage);   // B slot reusable once these MMAs finish
        ph_acc[0] ^= 1;
        ph_acc[1] ^= 1;
        stage = (stage + 1) % kStages;
      }
      commit_elect(a_empty);             // A planes reusable
    }
    if (P.prof && lane == 0) {
      long long* pr = P.prof + blockIdx.x * 8;
      pr[0] = clock64() - prof_t0;
      pr[1] = prof_a;
      pr[2] = prof_b;
      pr[3] = prof_e0;
      pr[4] = prof_e1;
    }
  } else if (warp >= 4 + kEpiWarps) {
    // ------------------------------------------------------------ A loaders (H, M -> TMEM)
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const uint32_t ncol_plane = (uint32_t)kpad / 4;
    uint32_t a_empty_ph = 0;
    for (int64_t u = blockIdx.x; u < P.n_units; u += gridDim.x) {
      const TileUnit un = P.units[u];
      const int64_t prow = (int64_t)P.et.pbase[un.k] + un.I * kBM + row;
      mbar_wait(a_empty, a_empty_ph ^ 1);
      a_empty_ph ^= 1;
      tc_fence_after();
      // both planes' chunk loads in flight together: half the dependent
      // global round trips per unit (the MMA warp waits on this at unit
      // boundaries)
      const uint4* srcH = reinterpret_cast<const uint4*>(P.planes + prow * kpad);
      const uint4* srcM = reinterpret_cast<const uint4*>(P.planes + P.P * kpad + prow * kpad);
      for (int c0 = 0; c0 < kpad / 4; c0 += 32) {
        uint32_t vh[32], vm[32];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint4 w = __ldg(srcH + c0 / 4 + i);
          const uint4 x = __ldg(srcM + c0 / 4 + i);
          vh[4 * i] = w.x, vh[4 * i + 1] = w.y, vh[4 * i + 2] = w.z, vh[4 * i + 3] = w.w;
          vm[4 * i] = x.x, vm[4 * i + 1] = x.y, vm[4 * i + 2] = x.z, vm[4 * i + 3] = x.w;
        }
        tmem_st32(tmem_base + ((uint32_t)(q * 32) << 16) + c0, vh);
        tmem_st32(tmem_base + ((uint32_t)(q * 32) << 16) + ncol_plane + c0, vm);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(a_tm_full);
      // warm L2 with the next unit's A rows
      const int64_t un_next = u + gridDim.x;
      if (un_next < P.n_units) {
        const TileUnit nx = P.units[un_next];
        const int64_t nrow = (int64_t)P.et.pbase[nx.k] + nx.I * kBM + row;
        for (int pl = 0; pl < 2; ++pl)
          for (int off = 0; off < kpad; off += 128)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(P.planes + (int64_t)pl * P.P * kpad +
                                                          nrow * kpad + off));
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    // warp (q, ch): TMEM lane quarter q (rows 32q..32q+31), column quarter ch
    // (kEpiCols = 32 columns). Row counts here; column counts of the
    // off-diagonal tiles by colcount_kernel from the stored bits.
    const int ew = warp - 4;
    const int q = warp & 3;            // tcgen05.ld lane window = warp % 4
    const int ch = ew >> 2;
    const int row = q * 32 + lane;
    uint32_t ph_acc[2] = {0, 0};
    uint32_t islot = 0, ph_info = 0;  // per-slot phase bits
#ifdef BM_TC_PROFILE
    long long ep[7] = {0, 0, 0, 0, 0, 0, 0};
    const long long ep_t0 = clock64();
#endif
    // the next unit's descriptor and row data are fetched one unit ahead
    // (dependent global loads off the per-tile critical path)
    TileUnit un_nx = blockIdx.x < P.n_units ? P.units[blockIdx.x] : TileUnit{0, 0, 0, 0};
    int pb_nx = P.et.pbase[un_nx.k], nk_nx = P.et.nrows[un_nx.k];
    int32_t cq_nx = (int32_t)(P.nq[pb_nx + un_nx.I * kBM + row] >> kYShift);
#ifdef BM_TC_PROFILE
    long long tu_end = clock64();  // end of the previous unit's last tile
    ep[5] = 0;
#endif
    for (int64_t u = blockIdx.x; u < P.n_units; u += gridDim.x) {
#ifdef BM_TC_PROFILE
      const long long tu0 = clock64();
#endif
      const TileUnit un = un_nx;
      const int k = un.k;
      const int pb = pb_nx;
      const int n_k = nk_nx;
      const int gi = un.I * kBM + row;                // local row index
      const bool row_ok = gi < n_k;
      const int niU = cq_nx;
      if (u + gridDim.x < P.n_units) {
        un_nx = P.units[u + gridDim.x];
        pb_nx = P.et.pbase[un_nx.k];
        nk_nx = P.et.nrows[un_nx.k];
        cq_nx = (int32_t)(P.nq[pb_nx + un_nx.I * kBM + row] >> kYShift);
      }
      int row_count = 0;
#ifdef BM_TC_PROFILE
      ep[5] += clock64() - tu0;  // unit setup (descriptor + next-unit prefetch)
      (void)tu_end;
#endif
      for (int t = 0; t < un.cnt; ++t) {
        const int64_t tile = un.off + t - P.slot0;    // window slot of the kept tile
        // Integer decision. With y = 2^7 a0 + a1 + (a2 >> 7) - floor(N_j/U):
        //   y >= r_in  => D2c <= t_in (certainly inside; a3, L.L >= 0)
        //   y <= r_out => D2c >  t_out (certainly outside; a3, L.L bounded)
        //   otherwise  => exact fp64 recheck in the element's order
        // r = floor(N_i/U) + per-tile constant (tile_thr_kernel, with the
        // margins that absorb every rounding).
        EP_START();
        mbar_wait(info_full + islot, (ph_info >> islot) & 1u);
        ph_info ^= 1u << islot;
        const int2 th = info[islot].th;
        const int J = info[islot].J;
        const int col0 = J * kBN + ch * kEpiCols;     // first local column of this warp
        const int cown = info[islot].cq[ch * kEpiCols + lane];
        __syncwarp();
        if (lane == 0) mbar_arrive(info_empty + islot);
        islot = (islot + 1) % kInfo;
        // |y| <= kYMax for every pair, so clamping the bounds to +-(kYMax + 2)
        // keeps every decision and rules out int32 overflow below
        const int rin1 = th.x == kNever ? kYMax + 2 : max(-kYMax - 2, min(kYMax + 2, niU + th.x - 1));
        const int ro1 = th.y == kNever ? -kYMax - 2 : max(-kYMax - 2, min(kYMax + 2, niU + th.y + 1));
        const uint32_t colmask = __ballot_sync(0xffffffffu, col0 + lane < n_k);
        const uint32_t tq = tacc0 + ((uint32_t)(q * 32) << 16) + ch * kEpiCols;
        // --- phase 1: t1 = 2^7 a0 + a1 (exact int32), then release A0/A1
        mbar_wait(acc_full + 0, ph_acc[0]);
        EP_MARK(0);
        tc_fence_after();
        static_assert(kEpiCols == 32, "two 16-column TMEM loads per accumulator");
        int32_t t1[kEpiCols];
        {
          // all four loads in flight, one wait: A0/A1 are released sooner
          int32_t x0a[16], x0b[16], x1a[16], x1b[16];
          tmem_ld16(tq + 0 * kBN, x0a);
          tmem_ld16(tq + 0 * kBN + 16, x0b);
          tmem_ld16(tq + 1 * kBN, x1a);
          tmem_ld16(tq + 1 * kBN + 16, x1b);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            t1[j] = x0a[j] * (1 << kLimb) + x1a[j];
            t1[16 + j] = x0b[j] * (1 << kLimb) + x1b[j];
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(acc_empty + 0);
        // --- phase 2: fold A2 into t1 (t1 + (a2 >> 7)), release A2 at once,
        //     then decide from registers while the next tile's MMAs run
        EP_MARK(2);
        mbar_wait(acc_full + 1, ph_acc[1]);
        EP_MARK(1);
        tc_fence_after();
        {
          int32_t a2a[16], a2b[16];
          tmem_ld16(tq + 2 * kBN, a2a);
          tmem_ld16(tq + 2 * kBN + 16, a2b);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            t1[j] += a2a[j] >> kLimb;
            t1[16 + j] += a2b[j] >> kLimb;
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(acc_empty + 1);
        ph_acc[0] ^= 1;
        ph_acc[1] ^= 1;

        // Decision per pair from two sign bits (no predicates, no selects):
        //   (r_in - 1) - y < 0  <=> certainly inside
        //   y - (r_out + 1) < 0 <=> certainly outside
        // each funnel-shifted into the row word (columns 31..0 -> bits 31..0);
        // neither => undecided -> exact recheck queue.
        EP_MARK(3);
        uint32_t wi_hi = 0, wi_lo = 0, wo_hi = 0, wo_lo = 0;
#pragma unroll
        for (int jj = 15; jj >= 0; --jj) {
          const int y_hi = t1[16 + jj] - __shfl_sync(0xffffffffu, cown, 16 + jj);
          const int y_lo = t1[jj] - __shfl_sync(0xffffffffu, cown, jj);
          wi_hi = __funnelshift_l((uint32_t)(rin1 - y_hi), wi_hi, 1);
          wi_lo = __funnelshift_l((uint32_t)(rin1 - y_lo), wi_lo, 1);
          wo_hi = __funnelshift_l((uint32_t)(y_hi - ro1), wo_hi, 1);
          wo_lo = __funnelshift_l((uint32_t)(y_lo - ro1), wo_lo, 1);
        }
        const uint32_t valid = row_ok ? colmask : 0u;
        const uint32_t iw = (wi_hi << 16) | wi_lo, ow = (wo_hi << 16) | wo_lo;
        const uint32_t in_w = iw & valid;
        const uint32_t amb_w = valid & ~iw & ~ow;
        // bitmap word (row, 32 columns) of the tile
        BM_DASSERT(tile >= 0 && row < kTile && ch < 4);
        P.adj[tile * kTileWords + row * 4 + ch] = in_w;
        if (__any_sync(0xffffffffu, in_w != 0u) && lane == 0) P.nonempty[tile] = 1;
        row_count += __popc(in_w);
        EP_MARK(4);
        // undecided pairs -> exact recheck queue (one atomic per warp)
        if (__any_sync(0xffffffffu, amb_w != 0u)) {
          const int nb = __popc(amb_w);
          int incl = nb;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
          }
          const int tot = __shfl_sync(0xffffffffu, incl, 31);
          unsigned long long base = 0;
          if (lane == 31) base = atomicAdd(P.qcount, (unsigned long long)tot);
          base = __shfl_sync(0xffffffffu, base, 31);
          unsigned long long i = base + (unsigned long long)(incl - nb);
          uint32_t band = amb_w;
          while (band) {
            const int j = __ffs(band) - 1;
            band &= band - 1;
            if (i < P.qcap) P.queue[i] = make_int4(pb + gi, pb + col0 + j, (int)tile, k);
            ++i;
          }
        }
        EP_MARK(6);
      }
      if (row_count) atomicAdd(P.cnt + pb + gi, row_count);
    }
#ifdef BM_TC_PROFILE
    if (P.prof && ew == 0 && lane == 0) {
      long long* pr = P.prof + 148 * 8 + blockIdx.x * 8;
      for (int i = 0; i < 7; ++i) pr[i] = ep[i];
      pr[7] = clock64() - ep_t0;
    }
#endif
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
  }
}


// ---------------------------------------------------------------------------
// preparation: per-element centre / scale, quantisation, per-tile error max
// ---------------------------------------------------------------------------
// per 128-row tile (global tile index t): column min/max over valid rows, and
// (when cen != null) the tile centre = column means, for the pruning bound
__global__ void tile_minmax_kernel(const RowSrc src, int64_t d, ElemTables et,
                                   const int32_t* __restrict__ tile_elem, int64_t n_tiles,
                                   double* __restrict__ tmin, double* __restrict__ tmax,
                                   double* __restrict__ cen) {
  const int64_t t = blockIdx.x;
  if (t >= n_tiles) return;
  const int k = tile_elem[t];
  const int64_t p0 = t * kTile;  // padded base of this tile
  const int valid = min(kTile, (int)(et.nrows[k] - (p0 - et.pbase[k])));
  for (int64_t c = threadIdx.x; c < d; c += blockDim.x) {
    double mn = __longlong_as_double(0x7ff0000000000000ll), mx = -mn, sm = 0.0;
    for (int r = 0; r < valid; ++r) {
      const double v = src.row(p0 + r, d)[c];
      if (isfinite(v)) {  // see gather_tiles_kernel
        mn = fmin(mn, v);
        mx = fmax(mx, v);
      }
      sm += v;
    }
    tmin[t * d + c] = mn;
    tmax[t * d + c] = mx;
    if (cen) cen[t * d + c] = sm / (double)valid;
  }
}

// per element: centre c = (min+max)/2 per column, half-range R, scale s
// per element: centre c = (min+max)/2 per column (CTA per element x 32
// columns, 8 tile strides reduced in smem) and the half-range R (max over
// columns, atomicMax on the non-negative double's bits)
__global__ void __launch_bounds__(256)
elem_center_kernel(int64_t d, ElemTables et, const int32_t* __restrict__ tbase,
                   const double* __restrict__ tmin, const double* __restrict__ tmax,
                   double* __restrict__ center, unsigned long long* __restrict__ rbits) {
  const int k = blockIdx.x;
  const int lane = threadIdx.x & 31, tg = threadIdx.x >> 5;
  const int64_t c = (int64_t)blockIdx.y * 32 + lane;
  const int64_t t0 = tbase[k], t1 = tbase[k] + et.ntiles[k];
  __shared__ double smn[8][32], smx[8][32];
  double mn = __longlong_as_double(0x7ff0000000000000ll), mx = -mn;
  if (c < d)
    for (int64_t t = t0 + tg; t < t1; t += 8) {
      mn = fmin(mn, tmin[t * d + c]);
      mx = fmax(mx, tmax[t * d + c]);
    }
  smn[tg][lane] = mn;
  smx[tg][lane] = mx;
  __syncthreads();
  if (tg == 0) {
    for (int i = 1; i < 8; ++i) {
      mn = fmin(mn, smn[i][lane]);
      mx = fmax(mx, smx[i][lane]);
    }
    double R = 0.0;
    if (c < d) {
      double cc = t1 > t0 ? 0.5 * mn + 0.5 * mx : 0.0;
      if (!(cc == cc) || t1 == t0) cc = 0.0;
      center[(int64_t)k * d + c] = cc;
      if (t1 > t0) R = fmax(fmax(mx - cc, cc - mn), 0.0);
    }
    for (int o = 16; o; o >>= 1) R = fmax(R, __shfl_xor_sync(0xffffffffu, R, o));
    if (lane == 0 && R > 0.0) atomicMax(rbits + k, (unsigned long long)__double_as_longlong(R));
  }
}

__global__ void elem_scale_kernel(int64_t n_el, const unsigned long long* __restrict__ rbits,
                                  double* __restrict__ scale) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n_el) return;
  const double Rk = __longlong_as_double((long long)rbits[k]) * (1.0 + 1e-12);
  scale[k] = Rk > 0.0 ? Rk / (double)((1 << kQBits) - 2) : 1.0;
}

// Quantise one padded row (one half-warp; both half-warps of a warp call this
// together): limbs into the three planes (4 columns per lane per pass, packed
// 32-bit stores) and the row sums over the half-warp: N = sum q^2 (exact),
// |M|^2, |L|^2, sum e^2 (e = x - c - s q, fp64), sum y^2, and with ct != null
// the squared distance to the tile centre.
struct QRow {
  unsigned long long nsum;
  uint32_t msq, lsq;
  double esum, ysum, rsum;
};
__device__ __forceinline__ QRow quantize_row(const double* __restrict__ xr,
                                             const double* __restrict__ ck,
                                             const double* __restrict__ ct, bool valid, int64_t d,
                                             int64_t kpad, double sc, double inv,
                                             int8_t* __restrict__ hrow_p,
                                             int8_t* __restrict__ mrow_p,
                                             int8_t* __restrict__ lrow_p, int hl, int half) {
  constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52
  constexpr double kQMax = (double)((1 << kQBits) - 1);
  const bool vec = (d & 1) == 0;  // 16-byte aligned rows
  uint32_t msq = 0, lsq = 0;  // |M|^2, |L|^2 of the row's limb planes (exact)
  double esum = 0.0, ysum = 0.0, rsum = 0.0;
  long long nsi = 0;
  // Fast path (full 4-column groups of a valid row): rint and the integer
  // conversion by the 1.5 * 2^52 trick (exact rint, ties to even, for
  // |v| < 2^51), byte packing with PRMT, limb norms with DP4A, sum q^2 in
  // fp64 (per lane <= 16 * 2^42: exact). A row with any |v| >= qmax
  // (clamping, inf, NaN) is redone by the generic path.
  bool bad = false;
  auto quant4 = [&](const double (&xv)[4], const double (&cv)[4], const double (&tv)[4],
                    int (&q)[4]) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const double y = xv[j] - cv[j];
      const double v = y * inv;
      bad |= !(fabs(v) < kQMax);
      const double tq = __dadd_rn(v, kMagic);
      const double qd = __dsub_rn(tq, kMagic);
      q[j] = __double2loint(tq);
      const double e = y - qd * sc;
      esum += e * e;
      nsi += (long long)q[j] * q[j];  // exact, on the integer pipe
      if (ct) {
        const double dr = xv[j] - tv[j];
        rsum += dr * dr;
      }
    }
  };
  if (valid && vec) {
    // 64-column blocks; lane hl takes columns b + 2hl, b + 2hl + 1 and
    // b + 32 + 2hl, b + 33 + 2hl: every 16-byte shared load of a quarter-warp
    // phase is contiguous (no bank conflicts; 4 consecutive columns per lane
    // read at a 32-byte stride were 2-way conflicted), limbs stored as 16-bit
    // pairs
    for (int64_t b = 0; b + 64 <= d; b += 64) {
      const int64_t c0 = b + 2 * hl, c1 = b + 32 + 2 * hl;
      double xv[4], cv[4], tv[4];
      const double2 u0 = *reinterpret_cast<const double2*>(xr + c0);
      const double2 u1 = *reinterpret_cast<const double2*>(xr + c1);
      xv[0] = u0.x, xv[1] = u0.y, xv[2] = u1.x, xv[3] = u1.y;
      const double2 k0 = *reinterpret_cast<const double2*>(ck + c0);
      const double2 k1 = *reinterpret_cast<const double2*>(ck + c1);
      cv[0] = k0.x, cv[1] = k0.y, cv[2] = k1.x, cv[3] = k1.y;
      if (ct) {
        const double2 t0 = *reinterpret_cast<const double2*>(ct + c0);
        const double2 t1 = *reinterpret_cast<const double2*>(ct + c1);
        tv[0] = t0.x, tv[1] = t0.y, tv[2] = t1.x, tv[3] = t1.y;
      } else {
        tv[0] = tv[1] = tv[2] = tv[3] = 0.0;
      }
      int q[4];
      quant4(xv, cv, tv, q);
      // bytes (q0, q1 | q2, q3): low half-word -> columns c0, c0 + 1, high -> c1, c1 + 1
      const uint32_t lw = __byte_perm(__byte_perm(q[0], q[1], 0x0040),
                                      __byte_perm(q[2], q[3], 0x0040), 0x5410) & 0x7f7f7f7fu;
      const uint32_t mw = __byte_perm(__byte_perm(q[0] >> kLimb, q[1] >> kLimb, 0x0040),
                                      __byte_perm(q[2] >> kLimb, q[3] >> kLimb, 0x0040),
                                      0x5410) & 0x7f7f7f7fu;
      const uint32_t hw = __byte_perm(
          __byte_perm(q[0] >> (2 * kLimb), q[1] >> (2 * kLimb), 0x0040),
          __byte_perm(q[2] >> (2 * kLimb), q[3] >> (2 * kLimb), 0x0040), 0x5410);
      msq = __dp4a(mw, mw, msq);
      lsq = __dp4a(lw, lw, lsq);
      *reinterpret_cast<uint16_t*>(hrow_p + c0) = (uint16_t)hw;
      *reinterpret_cast<uint16_t*>(hrow_p + c1) = (uint16_t)(hw >> 16);
      *reinterpret_cast<uint16_t*>(mrow_p + c0) = (uint16_t)mw;
      *reinterpret_cast<uint16_t*>(mrow_p + c1) = (uint16_t)(mw >> 16);
      *reinterpret_cast<uint16_t*>(lrow_p + c0) = (uint16_t)lw;
      *reinterpret_cast<uint16_t*>(lrow_p + c1) = (uint16_t)(lw >> 16);
    }
  } else if (valid) {
    for (int64_t c4 = 4 * hl; c4 < kpad && c4 + 4 <= d; c4 += 64) {
      double xv[4], cv[4], tv[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        xv[j] = xr[c4 + j];
        cv[j] = ck[c4 + j];
        tv[j] = ct ? ct[c4 + j] : 0.0;
      }
      int q[4];
      quant4(xv, cv, tv, q);
      const uint32_t lw = __byte_perm(__byte_perm(q[0], q[1], 0x0040),
                                      __byte_perm(q[2], q[3], 0x0040), 0x5410) & 0x7f7f7f7fu;
      const uint32_t mw = __byte_perm(__byte_perm(q[0] >> kLimb, q[1] >> kLimb, 0x0040),
                                      __byte_perm(q[2] >> kLimb, q[3] >> kLimb, 0x0040),
                                      0x5410) & 0x7f7f7f7fu;
      const uint32_t hw = __byte_perm(
          __byte_perm(q[0] >> (2 * kLimb), q[1] >> (2 * kLimb), 0x0040),
          __byte_perm(q[2] >> (2 * kLimb), q[3] >> (2 * kLimb), 0x0040), 0x5410);
      msq = __dp4a(mw, mw, msq);
      lsq = __dp4a(lw, lw, lsq);
      *reinterpret_cast<uint32_t*>(hrow_p + c4) = hw;
      *reinterpret_cast<uint32_t*>(mrow_p + c4) = mw;
      *reinterpret_cast<uint32_t*>(lrow_p + c4) = lw;
    }
  }
  // fast path: every |y| < qmax * s, so sum y^2 < d (qmax s)^2 bounds the
  // row's term of the tile error bound (1e-15 sqrt(max ysum), see the tile
  // maxima) without a multiply-add per coordinate
  unsigned long long nsum = (unsigned long long)nsi;
  if (valid) ysum = (double)d * (kQMax * sc) * (kQMax * sc) * (1.0 + 1e-12);
  const bool redo = ((__ballot_sync(0xffffffffu, bad) >> (16 * half)) & 0xffffu) != 0;
  if (redo) nsum = 0, msq = lsq = 0, esum = ysum = rsum = 0.0;
  // generic path: the tail columns (or the whole row when redo / padding);
  // the fast path covered whole 64-column blocks (vec) or 4-column groups,
  // so a fast row starts after its last whole 64-column block
  const int64_t g0 = (!redo && valid) ? (d / 64) * 64 : 0;
  for (int64_t c4 = g0 + 4 * hl; c4 < kpad; c4 += 64) {
    if (!redo && valid && (vec ? (c4 - c4 % 64) + 64 <= d : c4 + 4 <= d)) continue;
    uint32_t hw = 0, mw = 0, lw = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t c = c4 + j;
      int q = 0;
      if (valid && c < d) {
        const double x = xr[c];
        const double y = x - ck[c];
        double qd = rint(y * inv);
        qd = fmin(fmax(qd, -kQMax), kQMax);
        q = (int)qd;
        const double e = y - qd * sc;
        esum += e * e;
        ysum += y * y;
        if (ct) {
          const double dr = x - ct[c];
          rsum += dr * dr;
        }
      }
      nsum += (unsigned long long)((long long)q * q);
      const uint32_t mq = (q >> kLimb) & ((1 << kLimb) - 1), lq = q & ((1 << kLimb) - 1);
      msq += mq * mq;
      lsq += lq * lq;
      hw |= (uint32_t)(uint8_t)(int8_t)(q >> (2 * kLimb)) << (8 * j);
      mw |= mq << (8 * j);
      lw |= lq << (8 * j);
    }
    *reinterpret_cast<uint32_t*>(hrow_p + c4) = hw;
    *reinterpret_cast<uint32_t*>(mrow_p + c4) = mw;
    *reinterpret_cast<uint32_t*>(lrow_p + c4) = lw;
  }
    // row sums over the 16 lanes of the half-warp
#pragma unroll
  for (int o = 8; o; o >>= 1) {
    esum += __shfl_xor_sync(0xffffffffu, esum, o);
    ysum += __shfl_xor_sync(0xffffffffu, ysum, o);
    rsum += __shfl_xor_sync(0xffffffffu, rsum, o);
    nsum += __shfl_xor_sync(0xffffffffu, nsum, o);
    msq += __shfl_xor_sync(0xffffffffu, msq, o);
    lsq += __shfl_xor_sync(0xffffffffu, lsq, o);
  }
  return QRow{nsum, msq, lsq, esum, ysum, rsum};
}

// One block per tile (grid-stride), one HALF-warp per padded row: limbs into
// the three planes (4 columns per lane per pass, packed 32-bit stores),
// N = sum q^2 (exact), e = |x - c - s q| (fp64) -> tile max (bit pattern, one
// atomicMax per tile); with cen != null also the row's distance to its tile
// centre -> tile radius (raw max, NaN-propagating). The block's rows stream
// through a shared-memory ring of kQRows-row stages filled by cp.async.bulk
// (16 contiguous rows of Xg per stage, or — reading X through the membership
// — one bulk copy per row, issued by the lanes of warp 0); the element and
// tile centres are staged once per tile. Two rows per warp halve the per-row reduction and
// bookkeeping instructions (the kernel is issue-bound, not HBM-bound).
constexpr int kQWarps = 8;            // blockDim.x == 256
constexpr int kQRows = 2 * kQWarps;   // rows per ring stage (one per half-warp)
constexpr int kQIters = kTile / kQRows;
constexpr int kQMaxStages = 4;
constexpr int kQSmem = 96 * 1024;     // ring budget (d <= 256: 2 stages of 32 KB + centres)

__global__ void __launch_bounds__(256, 3)
quantize_kernel(const RowSrc src, int64_t d, int64_t kpad, ElemTables et, int64_t P,
                const double* __restrict__ center, const double* __restrict__ scale,
                int8_t* __restrict__ planes, int64_t* __restrict__ nq, int32_t* __restrict__ cq,
                unsigned long long* __restrict__ tile_e, const double* __restrict__ cen,
                unsigned long long* __restrict__ rad_bits, uint32_t* __restrict__ limb_sq,
                int n_stages) {
  extern __shared__ __align__(128) double q_ring[];
  __shared__ __align__(8) uint64_t q_full[kQMaxStages];
  __shared__ unsigned long long s_red[5][2 * kQWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int half = lane >> 4, hl = lane & 15, hrow = 2 * warp + half;
  const int64_t n_tiles = P / kTile;
  const int64_t my_tiles = n_tiles > blockIdx.x ? (n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t n_it = my_tiles * kQIters;
  const uint32_t stage_bytes = (uint32_t)(kQRows * d * 8);
  double* const s_c = q_ring + n_stages * kQRows * d;  // element centre, tile centre
  // iteration i into ring slot sl; called by all lanes of warp 0
  auto issue = [&](int64_t i, int sl) {
    const int64_t row0 = (blockIdx.x + (i / kQIters) * gridDim.x) * kTile + (i % kQIters) * kQRows;
    uint64_t* bar = q_full + sl;
    if (!src.xrow) {
      if (lane == 0) {
        mbar_expect_tx(bar, stage_bytes);
        bulk_load(q_ring + sl * kQRows * d, src.X + row0 * d, stage_bytes, bar);
      }
      return;
    }
    const int64_t xrow = lane < kQRows ? src.xrow[row0 + lane] : -1;
    const unsigned m = __ballot_sync(0xffffffffu, xrow >= 0);
    if (lane == 0) mbar_expect_tx(bar, (uint32_t)(__popc(m) * d * 8));
    __syncwarp();
    if (xrow >= 0)  // pad rows are not loaded (never read: `valid` below)
      bulk_load(q_ring + (sl * kQRows + lane) * d, src.X + xrow * d, (uint32_t)(d * 8), bar);
  };
  if (threadIdx.x == 0) {
    for (int i = 0; i < n_stages; ++i) mbar_init(q_full + i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0)
    for (int i = 0; i < n_stages && i < n_it; ++i) issue(i, i);
  int k = 0;
  double sc = 1.0, inv = 1.0;
  // per-half-warp maxima over its rows (lane hl == 0): |M|^2, |L|^2 and the
  // bit patterns of the squared error / |y|^2 / radius sums (roots per tile)
  unsigned long long w_m = 0, w_l = 0, w_e = 0, w_y = 0, w_r = 0;
  bool w_valid = false;
  int slot = 0;
  uint32_t phase = 0;
  int64_t t = blockIdx.x;
  int sub = 0;  // row group within the tile
  for (int64_t i = 0; i < n_it; ++i) {
    if (sub == 0) {
      int64_t a = 0, bb = et.n_el;
      while (bb - a > 1) {
        int64_t mid = (a + bb) >> 1;
        if (et.pbase[mid] <= t * kTile) a = mid; else bb = mid;
      }
      k = (int)a;  // tiles never straddle elements
      sc = scale[k];
      inv = 1.0 / sc;
      w_m = w_l = w_e = w_y = w_r = 0;
      w_valid = false;
      for (int64_t c = threadIdx.x; c < d; c += blockDim.x) {
        s_c[c] = center[(int64_t)k * d + c];
        s_c[d + c] = cen ? cen[t * d + c] : 0.0;
      }
      __syncthreads();
    }
    const int64_t p = t * kTile + sub * kQRows + hrow;
    mbar_wait(q_full + slot, phase);
    const double* xr = q_ring + slot * kQRows * d + hrow * d;
    const bool valid = (p - et.pbase[k]) < et.nrows[k];
    const double* ck = s_c;
    const double* ct = cen ? s_c + d : nullptr;
    const QRow qr = quantize_row(xr, ck, ct, valid, d, kpad, sc, inv, planes + p * kpad,
                                 planes + P * kpad + p * kpad, planes + 2 * P * kpad + p * kpad,
                                 hl, half);
    const unsigned long long nsum = qr.nsum;
    const uint32_t msq = qr.msq, lsq = qr.lsq;
    const double esum = qr.esum, ysum = qr.ysum, rsum = qr.rsum;
    // every half-warp is done with this stage: refill it
    __syncthreads();
    if (warp == 0 && i + n_stages < n_it) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(i + n_stages, slot);
    }
    if (++slot == n_stages) slot = 0, phase ^= 1u;
    if (hl == 0) {
      nq[p] = (int64_t)nsum;
      cq[p] = (int32_t)((int64_t)nsum >> kYShift);
      w_m = max(w_m, (unsigned long long)msq);  // pads are all-zero rows
      w_l = max(w_l, (unsigned long long)lsq);
      if (valid) {
        // NaN (any sign) -> the positive quiet NaN, above every finite value
        auto bits = [](double v) {
          return (unsigned long long)__double_as_longlong(
              v == v ? v : __longlong_as_double(0x7ff8000000000000ll));
        };
        w_e = max(w_e, bits(esum));
        w_y = max(w_y, bits(ysum));
        w_r = max(w_r, bits(rsum));
        w_valid = true;
      }
    }
    if (++sub == kQIters) {
      // tile maxima: one atomic per tile and array (the arrays start zeroed).
      // sqrt is monotonic, so the tile's error bound
      //   sqrt(max esum) (1 + 1e-12) + 1e-15 sqrt(max ysum) + 1e-300
      // bounds every row's |x - c - s q| (the fp64 evaluation of each
      // coordinate of e is off by <= 3.1u|y_k|, u = 2^-53), and
      // sqrt(max rsum) is the max row distance to the tile centre.
      if (hl == 0) {
        const int h2 = 2 * warp + half;
        s_red[0][h2] = w_m, s_red[1][h2] = w_l;
        s_red[2][h2] = w_valid ? w_e + 1 : 0;  // +1: nonzero marks "has valid rows"
        s_red[3][h2] = w_y;
        s_red[4][h2] = w_r;
      }
      __syncthreads();
      if (threadIdx.x < 5) {
        unsigned long long m = 0;
#pragma unroll
        for (int w = 0; w < 2 * kQWarps; ++w) m = max(m, s_red[threadIdx.x][w]);
        s_red[threadIdx.x][0] = m;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        atomicMax(limb_sq + 2 * t, (uint32_t)s_red[0][0]);
        atomicMax(limb_sq + 2 * t + 1, (uint32_t)s_red[1][0]);
        if (s_red[2][0]) {
          const double es = __longlong_as_double((long long)(s_red[2][0] - 1));
          const double ys = __longlong_as_double((long long)s_red[3][0]);
          const double e = sqrt(es) * (1.0 + 1e-12) + 1e-15 * sqrt(ys) + 1e-300;
          atomicMax(tile_e + t, (unsigned long long)__double_as_longlong(
                                    e == e ? e : __longlong_as_double(0x7ff8000000000000ll)));
          if (rad_bits) {
            const double rr = sqrt(__longlong_as_double((long long)s_red[4][0]));
            atomicMax(rad_bits + t, (unsigned long long)__double_as_longlong(
                                        rr == rr ? rr : __longlong_as_double(0x7ff8000000000000ll)));
          }
        }
      }
      __syncthreads();
      sub = 0;
      t += gridDim.x;
    }
  }
}

// Warp-private rings (d even): the CTA walks its tiles; each warp quantises 16
// rows of the current tile two at a time (a half-warp per row), streaming
// them through its own ring of kWStages two-row stages that lanes 0 and 1
// fill with one bulk copy per row (the next source rows are looked up one
// step ahead). No CTA barrier per stage: three per tile, for the centres
// and the tile maxima.
constexpr int kWStages = 2;
constexpr int kQWarpsR = 8;  // blockDim.x == 256

__global__ void __launch_bounds__(256, 3)
quantize_rows_kernel(const RowSrc src, int64_t d, int64_t kpad, ElemTables et, int64_t P,
                     const double* __restrict__ center, const double* __restrict__ scale,
                     int8_t* __restrict__ planes, int64_t* __restrict__ nq,
                     int32_t* __restrict__ cq, unsigned long long* __restrict__ tile_e,
                     const double* __restrict__ cen, unsigned long long* __restrict__ rad_bits,
                     uint32_t* __restrict__ limb_sq) {
  extern __shared__ __align__(128) double q_smem[];
  __shared__ __align__(8) uint64_t wbar[kQWarpsR][kWStages];
  __shared__ unsigned long long s_red[5][2 * kQWarpsR];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int half = lane >> 4, hl = lane & 15;
  double* const ring = q_smem + (int64_t)warp * kWStages * 2 * d;
  double* const s_c = q_smem + (int64_t)kQWarpsR * kWStages * 2 * d;  // element, tile centre
  const int64_t n_tiles = P / kTile;
  const int64_t my_tiles = n_tiles > blockIdx.x ? (n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  constexpr int kIt = kTile / (2 * kQWarpsR);  // iterations per tile and warp (8)
  const int64_t n_it = my_tiles * kIt;
  auto row_of = [&](int64_t i, int h) -> int64_t {
    const int64_t tile = blockIdx.x + (i / kIt) * gridDim.x;
    return tile * kTile + warp * (2 * kIt) + (i % kIt) * 2 + h;
  };
  // dataset (or Xg) row of iteration i for lanes 0, 1 (-1: pad / none)
  auto src_row = [&](int64_t i) -> int64_t {
    if (lane >= 2 || i >= n_it) return -1;
    return src.index(row_of(i, lane));
  };
  auto issue = [&](int sl, int64_t xr) {  // all lanes of the warp
    uint64_t* bar = &wbar[warp][sl];
    const unsigned m = __ballot_sync(0xffffffffu, xr >= 0);
    if (lane == 0) mbar_expect_tx(bar, (uint32_t)(__popc(m) * d * 8));
    __syncwarp();
    if (xr >= 0) bulk_load(ring + (sl * 2 + lane) * d, src.X + xr * d, (uint32_t)(d * 8), bar);
  };
  if (lane == 0) {
    for (int sl = 0; sl < kWStages; ++sl) mbar_init(&wbar[warp][sl], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  int64_t nx = src_row(0);
  for (int sl = 0; sl < kWStages && sl < n_it; ++sl) {
    issue(sl, nx);
    nx = src_row(sl + 1);
  }
  int slot = 0;
  uint32_t phase = 0;
  int64_t tile = blockIdx.x;
  for (int64_t tl = 0; tl < my_tiles; ++tl, tile += gridDim.x) {
    int64_t a = 0, bb = et.n_el;
    while (bb - a > 1) {
      const int64_t mid = (a + bb) >> 1;
      if (et.pbase[mid] <= tile * kTile) a = mid; else bb = mid;
    }
    const int k = (int)a;  // tiles never straddle elements
    const double sc = scale[k], inv = 1.0 / sc;
    const int64_t p_end = et.pbase[k] + et.nrows[k];  // first pad row of the element
    __syncthreads();  // the previous tile's readers of s_c / s_red are done
    for (int64_t c = threadIdx.x; c < d; c += blockDim.x) {
      s_c[c] = center[(int64_t)k * d + c];
      s_c[d + c] = cen ? cen[tile * d + c] : 0.0;
    }
    __syncthreads();
    unsigned long long w_m = 0, w_l = 0, w_e = 0, w_y = 0, w_r = 0;
    bool w_valid = false;
    for (int j = 0; j < kIt; ++j) {
      const int64_t i = tl * kIt + j;
      const int64_t p = tile * kTile + warp * (2 * kIt) + j * 2 + half;
      BM_DASSERT(p < P);
      mbar_wait(&wbar[warp][slot], phase);
      const bool valid = p < p_end;
      const QRow qr = quantize_row(ring + (slot * 2 + half) * d, s_c, cen ? s_c + d : nullptr,
                                   valid, d, kpad, sc, inv, planes + p * kpad,
                                   planes + P * kpad + p * kpad, planes + 2 * P * kpad + p * kpad,
                                   hl, half);
      __syncwarp();  // both rows of the stage are consumed: refill it
      if (i + kWStages < n_it) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(slot, nx);
        nx = src_row(i + kWStages + 1);
      }
      if (++slot == kWStages) slot = 0, phase ^= 1u;
      if (hl == 0) {
        nq[p] = (int64_t)qr.nsum;
        cq[p] = (int32_t)((int64_t)qr.nsum >> kYShift);
        w_m = max(w_m, (unsigned long long)qr.msq);  // pads are all-zero rows
        w_l = max(w_l, (unsigned long long)qr.lsq);
        if (valid) {
          auto bits = [](double v) {  // NaN -> the positive quiet NaN (max)
            return (unsigned long long)__double_as_longlong(
                v == v ? v : __longlong_as_double(0x7ff8000000000000ll));
          };
          w_e = max(w_e, bits(qr.esum));
          w_y = max(w_y, bits(qr.ysum));
          w_r = max(w_r, bits(qr.rsum));
          w_valid = true;
        }
      }
    }
    // tile maxima (see quantize_kernel): one atomic per tile and array
    if (hl == 0) {
      const int h2 = 2 * warp + half;
      s_red[0][h2] = w_m, s_red[1][h2] = w_l;
      s_red[2][h2] = w_valid ? w_e + 1 : 0;
      s_red[3][h2] = w_y;
      s_red[4][h2] = w_r;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long m[5] = {0, 0, 0, 0, 0};
      for (int x = 0; x < 5; ++x)
        for (int w = 0; w < 2 * kQWarpsR; ++w) m[x] = max(m[x], s_red[x][w]);
      atomicMax(limb_sq + 2 * tile, (uint32_t)m[0]);
      atomicMax(limb_sq + 2 * tile + 1, (uint32_t)m[1]);
      if (m[2]) {
        const double es = __longlong_as_double((long long)(m[2] - 1));
        const double ys = __longlong_as_double((long long)m[3]);
        const double e = sqrt(es) * (1.0 + 1e-12) + 1e-15 * sqrt(ys) + 1e-300;
        atomicMax(tile_e + tile, (unsigned long long)__double_as_longlong(
                                     e == e ? e : __longlong_as_double(0x7ff8000000000000ll)));
        if (rad_bits) {
          const double rr = sqrt(__longlong_as_double((long long)m[4]));
          atomicMax(rad_bits + tile, (unsigned long long)__double_as_longlong(
                                         rr == rr ? rr : __longlong_as_double(0x7ff8000000000000ll)));
        }
      }
    }
  }
}

// per tile: quantisation-error bound in quantised units; per element: the
// eps radii a_in = eps/(1+gamma)/s, a_out = eps/(1-gamma)/s
__global__ void thresholds_prep_kernel(const unsigned long long* __restrict__ tile_e_bits,
                                       const int32_t* __restrict__ tile_elem, int64_t n_tiles,
                                       const double* __restrict__ scale, int64_t n_el, double eps,
                                       double gamma, double* __restrict__ tile_u,
                                       double* __restrict__ a_in, double* __restrict__ a_out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_tiles) {
    const double e = __longlong_as_double((long long)tile_e_bits[i]);
    // round the quotient up: u >= e / s
    tile_u[i] = __ddiv_ru(e, scale[tile_elem[i]]);
  }
  if (i < n_el) {
    const double s = scale[i];
    if (eps >= 1e-140 && eps <= 1e140) {
      a_in[i] = __ddiv_rd(__ddiv_rd(eps, 1.0 + gamma), s);
      a_out[i] = __ddiv_ru(__ddiv_ru(eps, 1.0 - gamma), s);
    } else {
      // squares near eps would underflow/overflow (dbscan.cu eps_in_model):
      // no certain decision, every pair of the element is rechecked
      a_in[i] = -1e300;
      a_out[i] = 1e300;
    }
  }
}

// ---------------------------------------------------------------------------
// Direction-bound projections from the limb planes (int8 mma.sync): per
// grouped row tile I (seed a) and every seed g of its element k,
//   proj[I][g] = s_k (min_{x in I} <2^14 H_x + 2^7 M_x, u'_ag> - Lmax_I |u'_ag|)
//                - e_I |u'_ag|                                 (rounded down)
// where u'_ag = s'_a - s'_g is the difference of the element's int8-quantised
// seeds (dbscan.cu seed_quant_kernel), q_x = 2^14 H + 2^7 M + L the row's
// limbs, Lmax_I = max_x |L_x| (limb norms, quantize_kernel; then
// <L_x, u'> >= -Lmax_I |u'|, ~2^-14 of the H term) and e_I bounds
// |x - c_k - s_k q_x| over the tile. For every direction u,
//   <x, u> = <c_k, u> + s_k <q_x, u> + <e_x, u>,
// so proj[I][g] + <c_k, u'_ag> <= min_x <x, u'_ag>. In tile_prune_kernel the
// two tiles of a pair use u'_ab and u'_ba = -u'_ab, the <c_k, u'> terms
// cancel, and (proj[I][b] + proj[J][a]) / |u'_ab| <= |x - y| for every x in
// I, y in J. <H_x, s'_g>, <M_x, s'_g> are exact int32 sums (|.| <= 128 * 127
// * 256), combined in int64. One CTA per row tile, 8 warps x 16 rows, all 64
// seeds (8 n-tiles); the next K step's A fragments load while this one's MMAs
// run.
// ---------------------------------------------------------------------------
constexpr int kPjSeeds = 64;

__device__ __forceinline__ void mma_s8_16832(int (&c)[4], const uint32_t (&a)[4],
                                             uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int NKC>
__global__ void __launch_bounds__(256, 2)
tile_project_i8_kernel(const int8_t* __restrict__ planes, int64_t P, ElemTables et,
                       const int32_t* __restrict__ tile_elem, const int32_t* __restrict__ tseed,
                       const int8_t* __restrict__ seeds_q, const double* __restrict__ unorm,
                       const double* __restrict__ scale,
                       const unsigned long long* __restrict__ tile_e,
                       const uint32_t* __restrict__ limb_sq, double* __restrict__ proj) {
  constexpr int kpad = NKC * kKC;
  constexpr int kS = kpad + 16;  // padded smem row: conflict-free B fragments
  __shared__ __align__(16) int8_t sS[kPjSeeds * kS];
  __shared__ long long red[8][kPjSeeds];
  const int64_t rt = blockIdx.x;
  const int a = tseed[rt];
  if (a < 0) return;  // block-uniform: element not grouped
  const int k = tile_elem[rt];
  BM_DASSERT(k >= 0 && k < et.n_el && a < kPjSeeds);
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  const int r0 = w * 16 + gid;  // this thread's rows: r0, r0 + 8
  const int64_t p0 = rt * kTile;
  // A fragments (H and M planes) of K step ks: rows r0 / r0 + 8, bytes
  // 4 tig.. and 4 tig + 16.. of the step's 32
  const int8_t* arow = planes + (p0 + r0) * (int64_t)kpad + tig * 4;
  auto load_a = [&](int ks, uint32_t (&af)[2][4]) {
#pragma unroll
    for (int l = 0; l < 2; ++l) {
      const int8_t* b = arow + (int64_t)l * P * kpad + ks * 32;
      af[l][0] = __ldg(reinterpret_cast<const uint32_t*>(b));
      af[l][1] = __ldg(reinterpret_cast<const uint32_t*>(b + 8 * kpad));
      af[l][2] = __ldg(reinterpret_cast<const uint32_t*>(b + 16));
      af[l][3] = __ldg(reinterpret_cast<const uint32_t*>(b + 8 * kpad + 16));
    }
  };
  uint32_t afc[2][4];
  load_a(0, afc);  // in flight while the seeds are staged
  const int8_t* sk = seeds_q + (int64_t)k * kPjSeeds * kpad;
  for (int i = t; i < kPjSeeds * kpad / 16; i += 256) {
    const int g = i / (kpad / 16), c = i % (kpad / 16);
    *reinterpret_cast<int4*>(sS + g * kS + c * 16) =
        reinterpret_cast<const int4*>(sk + (int64_t)g * kpad)[c];
  }
  __syncthreads();
  const int valid = min(kTile, (int)(et.nrows[k] - (p0 - et.pbase[k])));
  int acc[2][8][4];
#pragma unroll
  for (int l = 0; l < 2; ++l)
#pragma unroll
    for (int n = 0; n < 8; ++n)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[l][n][j] = 0;
#pragma unroll
  for (int ks = 0; ks < kpad / 32; ++ks) {
    uint32_t afn[2][4];
    if (ks + 1 < kpad / 32) load_a(ks + 1, afn);
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      const int8_t* bp = sS + (n * 8 + gid) * kS + ks * 32 + tig * 4;
      const uint32_t b0 = *reinterpret_cast<const uint32_t*>(bp);
      const uint32_t b1 = *reinterpret_cast<const uint32_t*>(bp + 16);
#pragma unroll
      for (int l = 0; l < 2; ++l) mma_s8_16832(acc[l][n], afc[l], b0, b1);
    }
    if (ks + 1 < kpad / 32) {
#pragma unroll
      for (int l = 0; l < 2; ++l)
#pragma unroll
        for (int j = 0; j < 4; ++j) afc[l][j] = afn[l][j];
    }
  }
  // <2^14 H_x + 2^7 M_x, s'_g> of row r0 (j = 0, 1) or r0 + 8 (j = 2, 3),
  // column n * 8 + 2 tig + (j & 1)
#define BM_PJ_COMB(n, j) \
  ((long long)acc[0][n][j] * (1ll << (2 * kLimb)) + (long long)acc[1][n][j] * (1 << kLimb))
  // <., s'_a> of my two rows, from the lane of the same row group owning
  // column a (static register indices only: selects, no indexed arrays)
  const int na = a >> 3, ca = a & 7;
  const bool odd = ca & 1;
  long long da_lo = 0, da_hi = 0;
#pragma unroll
  for (int n = 0; n < 8; ++n)
    if (n == na) {
      da_lo = odd ? BM_PJ_COMB(n, 1) : BM_PJ_COMB(n, 0);
      da_hi = odd ? BM_PJ_COMB(n, 3) : BM_PJ_COMB(n, 2);
    }
  const int src_lane = (lane & ~3) | (ca >> 1);
  da_lo = __shfl_sync(0xffffffffu, da_lo, src_lane);
  da_hi = __shfl_sync(0xffffffffu, da_hi, src_lane);
  constexpr long long kMax = 0x7fffffffffffffffll;
  const bool ok_lo = r0 < valid, ok_hi = r0 + 8 < valid;
#pragma unroll
  for (int n = 0; n < 8; ++n)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      long long m = min(ok_lo ? da_lo - BM_PJ_COMB(n, j) : kMax,
                        ok_hi ? da_hi - BM_PJ_COMB(n, 2 + j) : kMax);
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (gid == 0) red[w][n * 8 + tig * 2 + j] = m;
    }
#undef BM_PJ_COMB
  __syncthreads();
  if (t < kPjSeeds) {
    long long m = red[0][t];
#pragma unroll
    for (int i = 1; i < 8; ++i) m = min(m, red[i][t]);
    const double e = __longlong_as_double((long long)tile_e[rt]);
    const double u = unorm[((int64_t)k * kPjSeeds + a) * kPjSeeds + t];
    const double lmax = __dsqrt_ru((double)limb_sq[2 * rt + 1]);
    // s_k (m - Lmax |u'|) - e |u'|, every step rounded down
    const double inner = __dsub_rd((double)m, __dmul_ru(lmax, u));
    double v = __dsub_rd(__dmul_rd(scale[k], inner), __dmul_ru(e, u));
    if (!(e == e) || m == kMax || !(v == v)) v = -1.0e300;  // NaN/inf rows: no bound
    proj[rt * kPjSeeds + t] = v;
  }
}

__device__ __forceinline__ void set_inside(const ElemTables& et, int4 pr,
                                           uint32_t* __restrict__ adj, int32_t* __restrict__ nonempty,
                                           int32_t* __restrict__ cnt,
                                           unsigned long long* __restrict__ n_inside) {
  const int k = pr.w;
  BM_DASSERT(k >= 0 && k < et.n_el);
  const int li = pr.x - et.pbase[k], lj = pr.y - et.pbase[k];
  BM_DASSERT(li >= 0 && li < et.nrows[k] && lj >= 0 && lj < et.nrows[k]);
  const int I = li / kTile, J = lj / kTile, r = li % kTile, c = lj % kTile;
  BM_DASSERT(I <= J && pr.z >= 0);
  const int64_t tile = pr.z;
  atomicOr(adj + tile * kTileWords + r * 4 + (c >> 5), 1u << (c & 31));
  nonempty[tile] = 1;
  atomicAdd(cnt + pr.x, 1);
  if (I != J) atomicAdd(cnt + pr.y, 1);  // off-diagonal bits stand for both orders
  atomicAdd(n_inside, 1ull);
}

// exact recheck of the queued pairs in the element's fp64 order. One lane per
// pair, 32 pairs per warp: the warp stages 32-dim chunks of the squared
// differences of its 32 pairs in shared memory with coalesced row loads, then
// each lane folds its own pair's squares in dim order. Both reference orders
// consume the dims left to right: sequential is s += v; pairwise (numpy's
// add.reduce, PwProgram) keeps 8 strided accumulators per leaf. Leaf starts
// are multiples of 8 (every left half has a length divisible by 8), so each
// 8-dim group lies inside one leaf and maps accumulator j to dim 8g+j
// statically; the leaf walk is uniform across lanes.
constexpr int kRcWarps = 4;

template <int DEPTH>
__global__ void __launch_bounds__(kRcWarps * 32, 6)
    recheck_kernel(const RowSrc src, int64_t d, ElemTables et,
                   const int4* __restrict__ queue, const unsigned long long* __restrict__ nq_ptr,
                   unsigned long long qcap, double eps,
                   uint32_t* __restrict__ adj, int32_t* __restrict__ nonempty,
                   int32_t* __restrict__ cnt, const __grid_constant__ PwProgram c_prog_tc,
                   unsigned long long* __restrict__ n_inside) {
  __shared__ double sq_all[kRcWarps][32][33];
  const int64_t nq = (int64_t)(*nq_ptr < qcap ? *nq_ptr : qcap);
  const int lane = threadIdx.x & 31;
  double(*S)[33] = sq_all[threadIdx.x >> 5];
  const int64_t stride = (int64_t)gridDim.x * kRcWarps * 32;
  for (int64_t base = ((int64_t)blockIdx.x * kRcWarps + (threadIdx.x >> 5)) * 32; base < nq;
       base += stride) {
    const int64_t i = base + lane;
    const bool have = i < nq;
    const int4 pr = have ? queue[i] : make_int4(0, 0, 0, 0);
    const int k = pr.w;
    // dataset rows of the lane's pair (the queue holds valid padded rows)
    // (dataset row ids fit int32: bm_cluster_elements requires n < 2^31)
    const int xa = have ? (int)src.index(pr.x) : 0, xb = have ? (int)src.index(pr.y) : 0;
    BM_DASSERT(xa >= 0 && xb >= 0);
    const int np = (nq - base) < 32 ? (int)(nq - base) : 32;
    double s_seq = 0.0, res = 0.0;
    double r[8];
    double st[DEPTH];  // pairwise partial sums (register stack, static indexing)
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = 0.0;
#pragma unroll
    for (int j = 0; j < DEPTH; ++j) st[j] = 0.0;
    int li = 0;
    for (int64_t c0 = 0; c0 < d; c0 += 32) {
      const bool cv = c0 + lane < d;
      // 8 pairs per step: all 16 row loads issued before any is consumed
      for (int p0 = 0; p0 < np; p0 += 8) {
        double va[8], vb[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int p = p0 + u;
          const int64_t ra = __shfl_sync(0xffffffffu, xa, p & 31);
          const int64_t rb = __shfl_sync(0xffffffffu, xb, p & 31);
          const bool ok = cv && p < np;
          va[u] = ok ? __ldg(src.X + ra * d + c0 + lane) : 0.0;
          vb[u] = ok ? __ldg(src.X + rb * d + c0 + lane) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const double df = __dsub_rn(va[u], vb[u]);
          S[(p0 + u) & 31][lane] = __dmul_rn(df, df);
        }
      }
      __syncwarp();
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const int64_t gb = c0 + 8 * g;
        if (gb >= d) break;
        const int nv = (d - gb) < 8 ? (int)(d - gb) : 8;
        double v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = S[lane][8 * g + j];
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (j < nv) s_seq = __dadd_rn(s_seq, v[j]);
        const PwLeaf L = c_prog_tc.leaf[li];
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
          for (int j = 0; j < 8; ++j) r[j] = pos == 0 ? v[j] : __dadd_rn(r[j], v[j]);
          if (pos + 8 == body) {
            res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                            __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
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
          for (int j = DEPTH - 1; j > 0; --j) st[j] = st[j - 1];
          st[0] = res;
          for (int q = 0; q < L.pops; ++q) {
            st[0] = __dadd_rn(st[1 < DEPTH ? 1 : 0], st[0]);
#pragma unroll
            for (int j = 1; j < DEPTH - 1; ++j) st[j] = st[j + 1];
          }
          ++li;
        }
      }
      __syncwarp();
    }
    if (have) {
      const double s2 = et.order[k] == BM_ORDER_SEQUENTIAL ? s_seq : __dadd_rn(0.0, st[0]);
      if (__dsqrt_rn(s2) <= eps) set_inside(et, pr, adj, nonempty, cnt, n_inside);
    }
  }
}

// Column counts of the off-diagonal kept tiles of a window (the epilogue takes
// the row counts): one warp per (tile, 32-column word), 4 row quarters
// transposed in registers (lane j then holds column j), popc, one atomic per
// column. Runs before the recheck, which counts the bits it adds itself.
// One warp per kept off-diagonal tile: the 128 x 4 words arrive as four
// 16-byte loads per lane (row 32 rb + lane), issued before any transpose; the
// next tile's flags are fetched one tile ahead.
// Rows whose count is still below min_pts after the tile pairs' ROW counts
// (K3): only their column counts can change a core decision (core = count >=
// min_pts; counts only grow), so colcount counts only these columns. Per
// 128-row tile, 4 words of candidate bits.
__global__ void cand_mask_kernel(const int32_t* __restrict__ cnt, ElemTables et, int64_t P,
                                 int32_t min_pts, uint32_t* __restrict__ cand) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // blockDim % 32 == 0
  const bool c = p < P && et.ent[p] >= 0 && cnt[p] < min_pts;
  const unsigned w = __ballot_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0 && p < P) cand[p >> 5] = w;
}

__global__ void __launch_bounds__(256)
colcount_kernel(const uint32_t* __restrict__ adj, const int32_t* __restrict__ nonempty,
                const TileRef* __restrict__ tiles, int64_t slot0, int64_t n_tiles,
                ElemTables et, int32_t* __restrict__ cnt, const uint32_t* __restrict__ cand) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int64_t s = w0;
  int ne = s < n_tiles ? nonempty[s] : 0;
  for (; s < n_tiles; s += nw) {
    const int ne_cur = ne;
    ne = s + nw < n_tiles ? nonempty[s + nw] : 0;
    if (!ne_cur) continue;
    const TileRef tr = tiles[slot0 + s];
    if (tr.I == tr.J) continue;
    const uint4* b = reinterpret_cast<const uint4*>(adj + s * kTileWords);
    uint4 r[4];
    if (cand) {
      // candidate columns only: one ballot per 32-row block and column; a
      // tile without candidate columns is not even read (most of them: rows
      // reach min_pts from their row counts alone)
      const int64_t pj = et.pbase[tr.k] + tr.J * kTile;
      const uint4 cm = *reinterpret_cast<const uint4*>(cand + (pj >> 5));
      if ((cm.x | cm.y | cm.z | cm.w) == 0u) continue;  // warp-uniform
#pragma unroll
      for (int rb = 0; rb < 4; ++rb) r[rb] = b[rb * 32 + lane];
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        uint32_t m = w == 0 ? cm.x : w == 1 ? cm.y : w == 2 ? cm.z : cm.w;
        while (m) {  // warp-uniform
          const int c = __ffs(m) - 1;
          m &= m - 1;
          int acc = 0;
#pragma unroll
          for (int rb = 0; rb < 4; ++rb) {
            const uint32_t x = w == 0 ? r[rb].x : w == 1 ? r[rb].y : w == 2 ? r[rb].z : r[rb].w;
            acc += __popc(__ballot_sync(0xffffffffu, (x >> c) & 1u));
          }
          if (acc && lane == 0) atomicAdd(cnt + pj + w * 32 + c, acc);
        }
      }
      continue;
    }
#pragma unroll
    for (int rb = 0; rb < 4; ++rb) r[rb] = b[rb * 32 + lane];
    const int64_t base = et.pbase[tr.k] + tr.J * kTile + lane;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      int acc = 0;
#pragma unroll
      for (int rb = 0; rb < 4; ++rb) {
        uint32_t x = w == 0 ? r[rb].x : w == 1 ? r[rb].y : w == 2 ? r[rb].z : r[rb].w;
        x = bit_transpose_step(x, 16, 0x0000FFFFu, lane);
        x = bit_transpose_step(x, 8, 0x00FF00FFu, lane);
        x = bit_transpose_step(x, 4, 0x0F0F0F0Fu, lane);
        x = bit_transpose_step(x, 2, 0x33333333u, lane);
        x = bit_transpose_step(x, 1, 0x55555555u, lane);
        acc += __popc(x);
      }
      if (acc) atomicAdd(cnt + base + w * 32, acc);
    }
  }
}

// ---------------------------------------------------------------------------
// TMA descriptor through the driver entry point (no libcuda link dependency)
// ---------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int make_qmap(CUtensorMap* map, void* planes, int64_t P, int64_t kpad) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    BM_CHECK_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess) {
      set_error("cuTensorMapEncodeTiled unavailable");
      return BM_ERR_INTERNAL;
    }
    fn = (EncodeTiledFn)p;
  }
  cuuint64_t dims[3] = {(cuuint64_t)kpad, (cuuint64_t)P, 3};
  cuuint64_t strides[2] = {(cuuint64_t)kpad, (cuuint64_t)(P * kpad)};
  cuuint32_t box[3] = {(cuuint32_t)kKC, (cuuint32_t)64, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, planes, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
    return BM_ERR_INTERNAL;
  }
  return BM_OK;
}

inline unsigned grid_cap(int64_t n, int threads, int per_sm) {
  int64_t b = ceil_div(n, threads);
  int64_t cap = (int64_t)num_sms() * per_sm;
  return (unsigned)std::max<int64_t>(1, std::min(b, cap));
}

}  // namespace

bool tc_supported(int64_t d) { return d >= 32 && d <= 256; }

// Per-batch state of the tensor-core engine: quantised limb planes, row
// norms, per-tile error bounds and element thresholds. Built once per batch
// and reused by every row window (a huge element is processed in windows of
// tile rows, twice: counts, then components).
struct TcPrep {
  int64_t d = 0, P = 0, n_el = 0, n_tiles = 0, kpad = 0;
  int nkc = 0, depth = 1;  // depth: pairwise-sum stack depth of d (PwProgram)
  PwProgram prog{};       // numpy pairwise-sum program of d (a kernel argument: no
                          // shared constant memory, so concurrent calls are safe)
  double eps = 0.0;
  int32_t min_pts = 0;  // > 0: column counts only for rows not already core by their rows
  std::vector<int32_t> nrows;
  Scratch s_tab, s_mm, s_cs, s_pl, s_nq, s_te, s_thr, s_cntw, s_flag, s_lim;
  // deferred recheck-queue check: [0] largest overflowing request, [1] pairs
  // rechecked (device); the caller reads them at its next synchronisation
  unsigned long long* d_flag = nullptr;
  double qscale = 1.0;  // recheck queue capacity factor (raised on overflow)
  int32_t* d_tile_elem = nullptr;
  int32_t* d_tbase = nullptr;
  double* tile_u = nullptr;
  double* a_in = nullptr;
  double* a_out = nullptr;
  CUtensorMap qmap;
};

// tminmax (optional): per-tile column min [n_tiles][d] then max, and cen the
// tile centres, already computed (by the fused gather)
int tc_prepare(const RowSrc src, int64_t d, const ElemTables& et, int64_t P, double eps,
               const std::vector<int32_t>& h_nrows, cudaStream_t stream, TcPrep** out,
               double* cen, double* rad, const double* tminmax) {
  *out = nullptr;
  const int64_t kpad = ceil_div(d, kKC) * kKC;
  const int nkc = (int)(kpad / kKC);
  BM_REQUIRE(nkc >= 1 && nkc <= 2, "tensor-core engine supports d <= 256");
  PwProgram prog;
  BM_TRY(make_pw_program(d, &prog));
  TcPrep* tp = new TcPrep();
  struct Guard {
    TcPrep*& p;
    ~Guard() { delete p; }
  } guard{tp};
  const int64_t n_el = et.n_el;
  tp->d = d;
  tp->P = P;
  tp->n_el = n_el;
  tp->kpad = kpad;
  tp->nkc = nkc;
  tp->depth = prog.depth;
  tp->prog = prog;
  tp->eps = eps;
  tp->nrows = h_nrows;
  const int64_t n_tiles = P / kTile;
  tp->n_tiles = n_tiles;
  std::vector<int32_t> tile_elem(n_tiles), tbase(n_el + 1, 0);
  for (int64_t k = 0; k < n_el; ++k) {
    const int64_t T = ceil_div(h_nrows[k], kTile);
    tbase[k + 1] = (int32_t)(tbase[k] + T);
    for (int64_t t = 0; t < T; ++t) tile_elem[tbase[k] + t] = (int32_t)k;
  }
  BM_TRY(scratch_alloc(tp->s_tab, (n_tiles + n_el + 1) * 4 + 16, stream));
  tp->d_tile_elem = tp->s_tab.as<int32_t>();
  tp->d_tbase = tp->d_tile_elem + n_tiles;
  BM_CHECK_CUDA(cudaMemcpyAsync(tp->d_tile_elem, tile_elem.data(), n_tiles * 4,
                                cudaMemcpyHostToDevice, stream));
  BM_CHECK_CUDA(cudaMemcpyAsync(tp->d_tbase, tbase.data(), (n_el + 1) * 4, cudaMemcpyHostToDevice,
                                stream));
  const double* tmin = tminmax;
  const double* tmax = tminmax ? tminmax + n_tiles * d : nullptr;
  if (!tminmax) {
    BM_TRY(scratch_alloc(tp->s_mm, (size_t)n_tiles * d * 16, stream));
    tmin = tp->s_mm.as<double>();
    tmax = tmin + n_tiles * d;
  }
  BM_TRY(scratch_alloc(tp->s_cs, (size_t)(n_el * d + n_el) * 8, stream));
  double* center = tp->s_cs.as<double>();
  double* scale = center + n_el * d;
  BM_TRY(scratch_alloc(tp->s_pl, (size_t)3 * P * kpad, stream));
  BM_TRY(scratch_alloc(tp->s_nq, (size_t)P * 12, stream));
  BM_TRY(scratch_alloc(tp->s_te, (size_t)n_tiles * 8, stream));
  BM_CHECK_CUDA(cudaMemsetAsync(tp->s_te.ptr, 0, n_tiles * 8, stream));

  trace_mark("tc:prep start", stream);
  if (!tminmax) {
    tile_minmax_kernel<<<(unsigned)n_tiles, 256, 0, stream>>>(
        src, d, et, tp->d_tile_elem, n_tiles, const_cast<double*>(tmin), const_cast<double*>(tmax),
        cen);
    BM_CHECK_LAUNCH();
  }
  {
    Scratch s_r;
    BM_TRY(scratch_alloc(s_r, (size_t)n_el * 8, stream));
    BM_CHECK_CUDA(cudaMemsetAsync(s_r.ptr, 0, n_el * 8, stream));
    elem_center_kernel<<<dim3((unsigned)n_el, (unsigned)ceil_div(d, 32)), 256, 0, stream>>>(
        d, et, tp->d_tbase, tmin, tmax, center, s_r.as<unsigned long long>());
    BM_CHECK_LAUNCH();
    elem_scale_kernel<<<(unsigned)ceil_div(n_el, 128), 128, 0, stream>>>(
        n_el, s_r.as<unsigned long long>(), scale);
    BM_CHECK_LAUNCH();
  }
  if (rad) BM_CHECK_CUDA(cudaMemsetAsync(rad, 0, n_tiles * 8, stream));
  BM_TRY(scratch_alloc(tp->s_lim, (size_t)n_tiles * 8, stream));
  BM_CHECK_CUDA(cudaMemsetAsync(tp->s_lim.ptr, 0, n_tiles * 8, stream));
  if (d % 2 == 0) {  // per-row bulk copies (16-byte multiples) into warp-private rings
    const size_t smem = ((size_t)kQWarpsR * kWStages * 2 * d + 2 * d) * 8;
    BM_TRY(ensure_dyn_smem((const void*)quantize_rows_kernel, (int)smem));
    quantize_rows_kernel<<<(unsigned)std::min<int64_t>(n_tiles, (int64_t)num_sms() * 3), 256,
                           smem, stream>>>(
        src, d, kpad, et, P, center, scale, tp->s_pl.as<int8_t>(), tp->s_nq.as<int64_t>(),
        reinterpret_cast<int32_t*>(tp->s_nq.as<int64_t>() + P), tp->s_te.as<unsigned long long>(),
        cen, reinterpret_cast<unsigned long long*>(rad), tp->s_lim.as<uint32_t>());
    BM_CHECK_LAUNCH();
  } else {
    const int64_t stage = (int64_t)kQRows * d * 8;
    const int n_stages = (int)std::min<int64_t>(kQMaxStages, (kQSmem - 16 * d) / stage);
    BM_REQUIRE(n_stages >= 2, "quantiser ring: d=%lld too large", (long long)d);
    BM_TRY(ensure_dyn_smem((const void*)quantize_kernel, kQSmem));
    const size_t smem = (size_t)n_stages * stage + 16 * d;  // ring + two centres
    const int per_sm = std::max<int>(1, std::min<int>(3, (int)((220 * 1024) / smem)));
    quantize_kernel<<<(unsigned)std::min<int64_t>(n_tiles, (int64_t)num_sms() * per_sm), 256, smem,
                      stream>>>(
        src, d, kpad, et, P, center, scale, tp->s_pl.as<int8_t>(), tp->s_nq.as<int64_t>(),
        reinterpret_cast<int32_t*>(tp->s_nq.as<int64_t>() + P), tp->s_te.as<unsigned long long>(),
        cen, reinterpret_cast<unsigned long long*>(rad), tp->s_lim.as<uint32_t>(), n_stages);
    BM_CHECK_LAUNCH();
  }
  BM_TRY(make_qmap(&tp->qmap, tp->s_pl.ptr, P, kpad));

  const double gamma = ((double)d + 16.0) * 1.5 * 1.1102230246251565e-16;
  BM_TRY(scratch_alloc(tp->s_thr, (size_t)(n_tiles + 2 * n_el) * 8, stream));
  tp->tile_u = tp->s_thr.as<double>();
  tp->a_in = tp->tile_u + n_tiles;
  tp->a_out = tp->a_in + n_el;
  thresholds_prep_kernel<<<(unsigned)ceil_div(std::max<int64_t>(n_tiles, n_el), 256), 256, 0,
                           stream>>>(tp->s_te.as<unsigned long long>(), tp->d_tile_elem, n_tiles,
                                     scale, n_el, eps, gamma, tp->tile_u, tp->a_in, tp->a_out);
  BM_CHECK_LAUNCH();
  BM_TRY(scratch_alloc(tp->s_flag, 16, stream));
  tp->d_flag = tp->s_flag.as<unsigned long long>();
  BM_CHECK_CUDA(cudaMemsetAsync(tp->d_flag, 0, 16, stream));
  *out = tp;
  tp = nullptr;  // disarm the guard
  return BM_OK;
}

int tc_tile_project(TcPrep* tp, const ElemTables& et, const int32_t* tseed,
                    const int8_t* seeds_q, const double* unorm, double* proj,
                    cudaStream_t stream) {
  const double* scale = tp->s_cs.as<double>() + tp->n_el * tp->d;
  const unsigned grid = (unsigned)tp->n_tiles;
  if (grid == 0) return BM_OK;
  if (tp->nkc == 1)
    tile_project_i8_kernel<1><<<grid, 256, 0, stream>>>(
        tp->s_pl.as<int8_t>(), tp->P, et, tp->d_tile_elem, tseed, seeds_q, unorm, scale,
        tp->s_te.as<unsigned long long>(), tp->s_lim.as<uint32_t>(), proj);
  else
    tile_project_i8_kernel<2><<<grid, 256, 0, stream>>>(
        tp->s_pl.as<int8_t>(), tp->P, et, tp->d_tile_elem, tseed, seeds_q, unorm, scale,
        tp->s_te.as<unsigned long long>(), tp->s_lim.as<uint32_t>(), proj);
  BM_CHECK_LAUNCH();
  return BM_OK;
}

int64_t tc_kpad(int64_t d) { return ceil_div(d, kKC) * kKC; }

void tc_release(TcPrep* tp) { delete tp; }

void tc_set_queue_scale(TcPrep* tp, double s) { tp->qscale = s; }
void tc_set_min_pts(TcPrep* tp, int32_t m) { tp->min_pts = m; }

// after a synchronisation of the stream: pairs rechecked so far and whether a
// window's recheck queue overflowed (then its bits are incomplete: rerun with
// a larger tc_set_queue_scale)
int tc_collect(TcPrep* tp, int64_t* rechecked, bool* overflow, cudaStream_t stream) {
  unsigned long long h[2] = {0, 0};
  BM_CHECK_CUDA(cudaMemcpyAsync(h, tp->d_flag, 16, cudaMemcpyDeviceToHost, stream));
  BM_CHECK_CUDA(cudaStreamSynchronize(stream));
  *rechecked = (int64_t)h[1];
  *overflow = h[0] != 0;
  return BM_OK;
}

__global__ void queue_check_kernel(const unsigned long long* __restrict__ qcount,
                                   unsigned long long qcap, unsigned long long* __restrict__ flag) {
  const unsigned long long c = qcount[0];
  if (c > qcap) flag[0] = c > flag[0] ? c : flag[0];
  flag[1] += c < qcap ? c : qcap;
}

__global__ void add_counts_kernel(int32_t* __restrict__ dst, const int32_t* __restrict__ src,
                                  int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (src[i]) dst[i] += src[i];
}

// Adjacency bits and eps-neighbour counts of one window of kept tiles:
// slots [slot0, slot0 + n_tiles) of the batch list `tiles`, work units over
// them; adj[slot - slot0] written.
// accumulate: add the window's counts into cnt instead of overwriting it;
// cnt == nullptr: the counts of this window are not wanted (recomputed window).
// pairs = distinct row pairs inside the window's tiles (stats and queue size).
//
// sync_check: synchronise after the MMA pass and retry it with a larger queue
// on overflow (counts are accumulated exactly once); otherwise nothing
// synchronises and an overflow is reported by tc_collect.
int tc_window(TcPrep* tp, const RowSrc src, const ElemTables& et, const TileRef* tiles,
              int64_t slot0, int64_t n_tiles, const TileUnit* units, int64_t n_units,
              int64_t pairs, uint32_t* adj, int32_t* nonempty, int32_t* cnt, bool accumulate,
              bool sync_check, int64_t* stats, cudaStream_t stream) {
  const int64_t P = tp->P, d = tp->d;
  const int nkc = tp->nkc;
  if (n_units == 0) return BM_OK;
  Scratch s_cnt, s_tt;
  BigScratch s_q;  // cached across calls: mapping ~100 MB per call costs ~1 ms
  int32_t* cnt_run = cnt;
  if (accumulate || !cnt) {  // window counts go to a private buffer first
    if (!tp->s_cntw.ptr) BM_TRY(scratch_alloc(tp->s_cntw, (size_t)P * 4, stream));
    cnt_run = tp->s_cntw.as<int32_t>();
  }

  // ---- MMA pass (re-run with a larger recheck queue on overflow)
  unsigned long long qcap = std::max<unsigned long long>(
      1ull << 20, (unsigned long long)(tp->qscale * (double)pairs / 2000.0));
  static const char* force_q = getenv("B200MAP_TEST_QCAP");  // tests: tiny queue
  if (force_q) qcap = (unsigned long long)(tp->qscale * (double)atoll(force_q));
  BM_TRY(scratch_alloc(s_cnt, 16, stream));
  unsigned long long* d_cnt = s_cnt.as<unsigned long long>();
  const size_t smem = (size_t)nkc * kKC * kBN * (1 + 3 * kStages) + 256 + 1024 + 1600 + 64;
  BM_TRY(ensure_dyn_smem((const void*)tc_adjacency_kernel<1>, 227 * 1024));
  BM_TRY(ensure_dyn_smem((const void*)tc_adjacency_kernel<2>, 227 * 1024));
  BM_TRY(scratch_alloc(s_tt, (size_t)n_tiles * sizeof(TileThr), stream));
  trace_mark("tc:thr allocated", stream);
  unsigned long long h_cnt[2] = {0, 0};
  for (int attempt = 0; attempt < 3; ++attempt) {
    {
      size_t qb = (size_t)16 << 20;  // power-of-two size classes
      while (qb < qcap * sizeof(int4)) qb <<= 1;
      BM_TRY(big_scratch(s_q, qb, stream));
    }
    trace_mark("tc:queue allocated", stream);
    BM_CHECK_CUDA(cudaMemsetAsync(d_cnt, 0, 16, stream));
    BM_CHECK_CUDA(cudaMemsetAsync(cnt_run, 0, (size_t)P * 4, stream));
    BM_CHECK_CUDA(cudaMemsetAsync(nonempty, 0, (size_t)n_tiles * 4, stream));
    TcParams prm{};
    prm.et = et;
    prm.units = units;
    prm.tiles = tiles;
    prm.slot0 = slot0;
    prm.n_units = n_units;
    prm.nq = tp->s_nq.as<int64_t>();
    prm.cq = reinterpret_cast<const int32_t*>(tp->s_nq.as<int64_t>() + P);
    prm.tile_u = tp->tile_u;
    prm.tbase = tp->d_tbase;
    prm.a_in = tp->a_in;
    prm.a_out = tp->a_out;
    prm.limb_sq = tp->s_lim.as<uint32_t>();
    prm.nkc = nkc;
    prm.adj = adj;
    prm.nonempty = nonempty;
    prm.cnt = cnt_run;
    prm.queue = s_q.as<int4>();
    prm.planes = tp->s_pl.as<uint8_t>();
    prm.P = P;
    prm.qcount = d_cnt;
    prm.qcap = qcap;
    static const bool tc_prof = getenv("B200MAP_TC_PROFILE") != nullptr;
    Scratch s_prof;
    if (tc_prof) {
      BM_TRY(scratch_alloc(s_prof, 148 * 8 * 8 * 2, stream));
      BM_CHECK_CUDA(cudaMemsetAsync(s_prof.ptr, 0, 148 * 8 * 8 * 2, stream));
      prm.prof = s_prof.as<long long>();
    }
    prm.thr = s_tt.as<TileThr>();
    if (attempt == 0) {
      tile_thr_kernel<<<(unsigned)ceil_div(n_tiles, 256), 256, 0, stream>>>(prm, n_tiles,
                                                                             s_tt.as<TileThr>());
      BM_CHECK_LAUNCH();
    }
    const unsigned grid = (unsigned)std::min<int64_t>(num_sms(), n_units);
    if (nkc == 1)
      tc_adjacency_kernel<1><<<grid, kThreads, smem, stream>>>(tp->qmap, prm);
    else
      tc_adjacency_kernel<2><<<grid, kThreads, smem, stream>>>(tp->qmap, prm);
    BM_CHECK_LAUNCH();
    trace_mark("tc:mma launched", stream);
    if (!sync_check && !tc_prof) break;
    BM_CHECK_CUDA(cudaMemcpyAsync(h_cnt, d_cnt, 8, cudaMemcpyDeviceToHost, stream));
    BM_CHECK_CUDA(cudaStreamSynchronize(stream));
    if (tc_prof) {
      std::vector<long long> pr(148 * 8 * 2);
      BM_CHECK_CUDA(cudaMemcpy(pr.data(), s_prof.ptr, pr.size() * 8, cudaMemcpyDeviceToHost));
      double t[5] = {0, 0, 0, 0, 0};
      for (int b = 0; b < 148; ++b)
        for (int i = 0; i < 5; ++i) t[i] += pr[b * 8 + i];
      fprintf(stderr, "[tc-profile] MMA warp cycles/CTA: total %.3g  wait A %.1f%%  wait B %.1f%%  "
              "wait acc01 %.1f%%  wait acc2 %.1f%%  (units %lld)\n", t[0] / 148,
              100 * t[1] / t[0], 100 * t[2] / t[0], 100 * t[3] / t[0], 100 * t[4] / t[0],
              (long long)n_units);
      double e[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (int b = 0; b < 148; ++b)
        for (int i = 0; i < 8; ++i) e[i] += pr[148 * 8 + b * 8 + i];
      fprintf(stderr, "[tc-profile] epilogue warp: wait acc01 %.1f%%  E1 %.1f%%  wait acc2 %.1f%%  "
              "fold %.1f%%  decide+pack %.1f%%  unit setup %.1f%%  flush+queue %.1f%%  rest %.1f%%\n",
              100 * e[0] / e[7], 100 * e[2] / e[7], 100 * e[1] / e[7], 100 * e[3] / e[7],
              100 * e[4] / e[7], 100 * e[5] / e[7], 100 * e[6] / e[7],
              100 * (e[7] - e[0] - e[1] - e[2] - e[3] - e[4] - e[5] - e[6]) / e[7]);
    }
    if (h_cnt[0] <= qcap || !sync_check) break;
    qcap = h_cnt[0] + 1024;
    if (attempt == 2) {
      set_error("recheck queue overflow");
      return BM_ERR_INTERNAL;
    }
  }
  // the whole batch in one window: every row's count from its own tile row is
  // complete here, so only the rows still below min_pts need column counts
  Scratch s_cand;
  uint32_t* cand = nullptr;
  if (!accumulate && cnt && tp->min_pts > 0) {
    BM_TRY(scratch_alloc(s_cand, (size_t)(P / 32 + 4) * 4, stream));
    cand = s_cand.as<uint32_t>();
    cand_mask_kernel<<<(unsigned)ceil_div(P, 256), 256, 0, stream>>>(cnt_run, et, P, tp->min_pts,
                                                                    cand);
    BM_CHECK_LAUNCH();
  }
  colcount_kernel<<<grid_cap(n_tiles, 8, 8), 256, 0, stream>>>(adj, nonempty, tiles, slot0,
                                                               n_tiles, et, cnt_run, cand);
  BM_CHECK_LAUNCH();
  {
    // the queue length stays on the device: the recheck grid covers the
    // capacity and each warp reads the count
    const unsigned rg = grid_cap((int64_t)qcap, kRcWarps * 32, 6);
    const int4* q = s_q.as<int4>();
    switch (tp->depth) {
      case 1:
        recheck_kernel<1><<<rg, kRcWarps * 32, 0, stream>>>(src, d, et, q, d_cnt, qcap, tp->eps,
                                                            adj, nonempty, cnt_run, tp->prog,
                                                            d_cnt + 1);
        break;
      case 2:
        recheck_kernel<2><<<rg, kRcWarps * 32, 0, stream>>>(src, d, et, q, d_cnt, qcap, tp->eps,
                                                            adj, nonempty, cnt_run, tp->prog,
                                                            d_cnt + 1);
        break;
      default:
        recheck_kernel<4><<<rg, kRcWarps * 32, 0, stream>>>(src, d, et, q, d_cnt, qcap, tp->eps,
                                                            adj, nonempty, cnt_run, tp->prog,
                                                            d_cnt + 1);
        break;
    }
    BM_CHECK_LAUNCH();
    queue_check_kernel<<<1, 1, 0, stream>>>(d_cnt, qcap, tp->d_flag);
    BM_CHECK_LAUNCH();
    trace_mark("tc:recheck launched", stream);
  }
  if (accumulate && cnt) {
    add_counts_kernel<<<grid_cap(P, 256, 8), 256, 0, stream>>>(cnt, cnt_run, P);
    BM_CHECK_LAUNCH();
  }
  stats[0] += pairs;
  return BM_OK;
}

}  // namespace bm
