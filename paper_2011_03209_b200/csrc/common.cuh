// common.cuh — shared plumbing for libb200map: error state, scratch buffers,
// device-wide scans, and the exact fp64 summation orders of the reference.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string>
#include <vector>

#include "../../include/b200map.h"

namespace bm {

// ---------------------------------------------------------------------------
// Error plumbing: C++ never throws across the ABI; every entry point returns
// a status and leaves a per-thread message.
// ---------------------------------------------------------------------------
void set_error(const char* fmt, ...);
const char* get_error();

struct Status {
  int code = BM_OK;
};

#define BM_CHECK_CUDA(expr)                                                   \
  do {                                                                        \
    cudaError_t _e = (expr);                                                  \
    if (_e != cudaSuccess) {                                                  \
      ::bm::set_error("%s:%d %s -> %s", __FILE__, __LINE__, #expr,            \
                      cudaGetErrorString(_e));                                \
      return _e == cudaErrorMemoryAllocation ? BM_ERR_NOMEM : BM_ERR_INTERNAL; \
    }                                                                         \
  } while (0)

// Every kernel launch site ends with BM_CHECK_LAUNCH(), which also counts the
// launch (bm_launch_count) so benchmarks can report how many of the
// library's kernels ran.
void count_launch();
#define BM_CHECK_LAUNCH()       \
  do {                          \
    ::bm::count_launch();       \
    BM_CHECK_CUDA(cudaGetLastError()); \
  } while (0)

#define BM_REQUIRE(cond, ...)        \
  do {                               \
    if (!(cond)) {                   \
      ::bm::set_error(__VA_ARGS__);  \
      return BM_ERR_DATA;            \
    }                                \
  } while (0)

// Device-side bounds assertions of the debug build (-DBM_DEBUG_BOUNDS,
// B200MAP_NVCC_FLAGS): a violated index traps the kernel (the launch's
// sticky error surfaces as InternalError). Compiled out otherwise.
#ifdef BM_DEBUG_BOUNDS
#define BM_DASSERT(cond)                                                          \
  do {                                                                            \
    if (!(cond)) {                                                                \
      printf("BM_DASSERT failed %s:%d: %s\n", __FILE__, __LINE__, #cond);         \
      __trap();                                                                   \
    }                                                                             \
  } while (0)
#else
#define BM_DASSERT(cond) ((void)0)
#endif

#define BM_REQUIRE_INTERNAL(cond, ...) \
  do {                                 \
    if (!(cond)) {                     \
      ::bm::set_error(__VA_ARGS__);    \
      return BM_ERR_INTERNAL;          \
    }                                  \
  } while (0)

#define BM_TRY(expr)        \
  do {                      \
    int _rc = (expr);       \
    if (_rc != BM_OK) return _rc; \
  } while (0)

// Stream-ordered scratch buffer released on scope exit (cudaFreeAsync).
void big_release(int slot, cudaStream_t stream);

struct Scratch {
  void* ptr = nullptr;
  size_t bytes = 0;
  cudaStream_t stream = nullptr;
  int slot = -1;  // >= 0: a cached large buffer (big_acquire), not the stream pool
  Scratch() = default;
  Scratch(const Scratch&) = delete;
  Scratch& operator=(const Scratch&) = delete;
  ~Scratch() { release(); }
  void release() {
    if (slot >= 0) {
      big_release(slot, stream);
    } else if (ptr) {
      cudaFreeAsync(ptr, stream);
    }
    ptr = nullptr;
    slot = -1;
    bytes = 0;
  }
  template <typename T>
  T* as() const { return reinterpret_cast<T*>(ptr); }
};

// Stream-ordered scratch; at least kScratchBig bytes come from the cached
// large buffers (big_acquire) instead of the stream-ordered pool.
constexpr size_t kScratchBig = size_t(16) << 20;
int scratch_alloc(Scratch& s, size_t bytes, cudaStream_t stream);

// Stable sort of (keys, vals) by the low key_bits bits of keys (LSD radix,
// graph.cu); result in place. vals may be null.
int sort_pairs_u64(uint64_t* keys, int64_t* vals, int64_t n, int key_bits, cudaStream_t s);

// Dev tracing (B200MAP_TRACE=1): host time and a device event per mark;
// trace_dump() (after a synchronisation) prints both timelines.
void trace_mark(const char* name, cudaStream_t s);
void trace_dump();

// A large buffer kept across calls (cudaMalloc'd once per size class, reused
// by later calls; bm_release_scratch frees the idle ones). Release records an
// event on the holder's stream and the next holder's stream waits on it, so
// reuse is stream-ordered without host synchronisation.
int big_acquire(size_t bytes, cudaStream_t stream, void** out, int* slot);
void big_release(int slot, cudaStream_t stream);
struct BigScratch {
  void* ptr = nullptr;
  int slot = -1;
  cudaStream_t stream = nullptr;
  BigScratch() = default;
  BigScratch(const BigScratch&) = delete;
  BigScratch& operator=(const BigScratch&) = delete;
  ~BigScratch() { big_release(slot, stream); }
  template <typename T>
  T* as() const { return reinterpret_cast<T*>(ptr); }
};
inline int big_scratch(BigScratch& b, size_t bytes, cudaStream_t stream) {
  big_release(b.slot, b.stream);
  b.slot = -1;
  b.stream = stream;
  return big_acquire(bytes, stream, &b.ptr, &b.slot);
}

// Free device memory including what the stream-ordered pool retains unused.
int device_free_bytes(size_t* free_b);

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Number of SMs on the current device (cached per device).
int num_sms();
// Opt the kernel `fn` into `bytes` of dynamic shared memory on the CURRENT
// device. The attribute is per (device context, function), so the guard is
// keyed on both and taken under a lock (re-entrant ABI calls from several
// host threads, and one process driving several GPUs).
int ensure_dyn_smem(const void* fn, int bytes);
// Total memory of the current device (cached per device).
size_t device_total_bytes();

// fp64 -> fp32 rounding toward zero in integer ops, for |x| in the normal
// fp32 range or x == +-0 (*ok true); other inputs leave *ok false and need
// the conversion instruction. sm_100's fp64 conversions run on a narrow unit
// (~2 per clock per SM), so bulk conversions go through here. Relative error
// < 2^-23.
__device__ __forceinline__ float f64_to_f32_rz(double x, bool* ok) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(x);
  const unsigned hi = (unsigned)(b >> 32);
  const unsigned e = (hi >> 20) & 0x7ffu;
  *ok = (e - 897u <= 253u) || (b << 1) == 0;
  const unsigned m = (unsigned)(b >> 29) & 0x7fffffu;
  return __uint_as_float((hi & 0x80000000u) | (e ? ((e - 896u) << 23) | m : 0u));
}

// ---------------------------------------------------------------------------
// Device-wide exclusive scan over int64 (in-place allowed). n may be 0.
// ---------------------------------------------------------------------------
int exclusive_scan_i64(const int64_t* d_in, int64_t* d_out, int64_t n,
                       cudaStream_t stream);
int exclusive_scan_i32_to_i64(const int32_t* d_in, int64_t* d_out, int64_t n,
                              cudaStream_t stream);

// ---------------------------------------------------------------------------
// numpy pairwise summation (numpy/_core/src/umath/loops_utils.h.src,
// pairwise_sum; PW_BLOCKSIZE = 128) as a post-order program of leaves.
// Leaf = contiguous run of <= 128 terms summed with 8 strided accumulators
// (or sequentially from 0.0 when shorter than 8). After each leaf, `pops`
// additions combine the top of the stack (left + right).
// ---------------------------------------------------------------------------
struct PwLeaf {
  int32_t start;
  int32_t len;
  int32_t pops;  // number of stack reductions after pushing this leaf
};

inline void pw_plan_rec(int start, int n, std::vector<PwLeaf>& out) {
  if (n <= 128) {
    out.push_back({start, n, 0});
    return;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  pw_plan_rec(start, n2, out);
  pw_plan_rec(start + n2, n - n2, out);
  out.back().pops += 1;
}

inline std::vector<PwLeaf> pw_plan(int n) {
  std::vector<PwLeaf> out;
  if (n <= 0) return out;
  pw_plan_rec(0, n, out);
  return out;
}

constexpr int kMaxLeaves = 64;  // supports d <= 64*128 = 8192 dims
constexpr int kMaxStack = 8;

struct PwProgram {
  int32_t n_leaves;
  int32_t depth;  // max stack depth
  PwLeaf leaf[kMaxLeaves];
};

int make_pw_program(int64_t d, PwProgram* prog);

// Shift-register stack of partial sums in registers (static indexing only).
struct PwStack {
  double s[kMaxStack];
  __device__ __forceinline__ void push(double v) {
#pragma unroll
    for (int i = kMaxStack - 1; i > 0; --i) s[i] = s[i - 1];
    s[0] = v;
  }
  __device__ __forceinline__ void reduce() {
    s[0] = __dadd_rn(s[1], s[0]);
#pragma unroll
    for (int i = 1; i < kMaxStack - 1; ++i) s[i] = s[i + 1];
  }
};

}  // namespace bm
