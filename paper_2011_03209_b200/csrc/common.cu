// common.cu — error state, scratch allocation and device-wide scans.
#include <stdarg.h>
#include <stdlib.h>

#include <algorithm>
#include <atomic>
#include <map>
#include <mutex>

#include <chrono>
#include <cstdlib>

#include "common.cuh"

namespace bm {

static thread_local std::string g_err;
static std::atomic<long long> g_launches{0};

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
}

const char* get_error() { return g_err.c_str(); }

// Scratch comes from the device's default stream-ordered pool. Its release
// threshold is raised once per device so freed blocks stay mapped between
// calls: re-mapping the ~12 GB a 1M-point build uses costs ~0.5 s per call.
// B200MAP_POOL_RELEASE=1 restores the CUDA default (return memory at sync).
static void retain_pool_once() {
  static std::mutex mu;
  static bool done[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (dev >= 64 || done[dev]) return;
  done[dev] = true;
  const char* env = getenv("B200MAP_POOL_RELEASE");
  if (env && env[0] == '1') return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  cudaGetLastError();
}

namespace {
struct TraceMark {
  const char* name;
  double host_ms;
  cudaEvent_t ev;
};
std::vector<TraceMark>& trace_marks() {
  static thread_local std::vector<TraceMark> m;
  return m;
}
bool trace_on() {
  static const bool on = getenv("B200MAP_TRACE") != nullptr;
  return on;
}
}  // namespace

void trace_mark(const char* name, cudaStream_t s) {
  if (!trace_on()) return;
  static const auto t0 = std::chrono::steady_clock::now();
  TraceMark m{name, std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(), nullptr};
  cudaEventCreate(&m.ev);
  cudaEventRecord(m.ev, s);
  trace_marks().push_back(m);
}

void trace_dump() {
  if (!trace_on()) return;
  auto& m = trace_marks();
  if (m.empty()) return;
  cudaEventSynchronize(m.back().ev);
  fprintf(stderr, "[trace] %-28s %10s %10s\n", "mark", "host ms", "device ms");
  for (auto& x : m) {
    float dev = 0.f;
    cudaEventElapsedTime(&dev, m.front().ev, x.ev);
    fprintf(stderr, "[trace] %-28s %10.3f %10.3f\n", x.name, x.host_ms - m.front().host_ms, dev);
  }
  for (auto& x : m) cudaEventDestroy(x.ev);
  m.clear();
}

size_t big_idle_bytes(int dev);

int device_free_bytes(size_t* free_b) {
  size_t total = 0;
  BM_CHECK_CUDA(cudaMemGetInfo(free_b, &total));
  int dev = 0;
  cudaGetDevice(&dev);
  // idle cached large buffers are reusable too: counting them keeps the
  // window plan of a huge element the same from call to call
  *free_b += big_idle_bytes(dev);
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t reserved = 0, used = 0;
    if (cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved) ==
            cudaSuccess &&
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used) == cudaSuccess &&
        reserved > used)
      *free_b += (size_t)(reserved - used);  // retained by the pool, reusable
  }
  cudaGetLastError();
  return BM_OK;
}

// ---------------------------------------------------------------------------
// Cached large buffers (see BigScratch): mapping tens of GB through the
// stream-ordered pool costs ~60 ms per GB whenever the pool cannot reuse one
// contiguous block, so the bitmap of a huge element is kept between calls.
// ---------------------------------------------------------------------------
namespace {
struct BigBuf {
  void* p;
  size_t bytes;
  int dev;
  bool busy;
  cudaEvent_t ev;  // recorded on the holder's stream at release
  bool pending;    // ev recorded and not yet waited on by a host free
};
std::mutex g_big_mu;
std::vector<BigBuf> g_big;

void big_free_locked(BigBuf& b) {  // g_big_mu held; b idle
  if (b.pending) cudaEventSynchronize(b.ev);
  b.pending = false;
  cudaFree(b.p);
  b.p = nullptr;
  b.bytes = 0;
}
}  // namespace

// Size classes of the cached buffers: requests are rounded up to 1/16 of
// their power-of-two magnitude (<= 6.25% over-allocation), so a request that
// varies slightly between calls (window plans follow the free memory) reuses
// the cached buffer instead of mapping tens of GB afresh.
static size_t big_class(size_t bytes) {
  size_t p2 = 1;
  while (p2 < bytes) p2 <<= 1;
  const size_t g = std::max<size_t>(p2 >> 4, (size_t)1 << 20);
  return (bytes + g - 1) / g * g;
}

size_t big_idle_bytes(int dev) {
  std::lock_guard<std::mutex> lk(g_big_mu);
  size_t b = 0;
  for (const auto& x : g_big)
    if (!x.busy && x.p && x.dev == dev) b += x.bytes;
  return b;
}

int big_acquire(size_t bytes, cudaStream_t stream, void** out, int* slot) {
  int dev = 0;
  cudaGetDevice(&dev);
  bytes = big_class(bytes);
  std::lock_guard<std::mutex> lk(g_big_mu);
  int best = -1;
  for (int i = 0; i < (int)g_big.size(); ++i) {
    const BigBuf& b = g_big[i];
    if (!b.busy && b.p && b.dev == dev && b.bytes >= bytes &&
        (best < 0 || b.bytes < g_big[best].bytes))
      best = i;
  }
  static const bool trace_mem = getenv("B200MAP_TRACE_MEM") != nullptr;
  if (best < 0) {
    void* p = nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) {
      // first the memory the stream-ordered pool retains unused, then the
      // idle cached buffers
      cudaGetLastError();
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        cudaDeviceSynchronize();
        cudaMemPoolTrimTo(pool, 0);
      }
      cudaGetLastError();
      e = cudaMalloc(&p, bytes);
    }
    if (e != cudaSuccess) {  // give back the idle cached buffers and retry once
      cudaGetLastError();
      for (auto& b : g_big)
        if (!b.busy && b.dev == dev && b.p) big_free_locked(b);
      e = cudaMalloc(&p, bytes);
    }
    if (trace_mem)
      fprintf(stderr, "[mem] big_acquire miss %.2f GB: cudaMalloc %s in %.1f ms\n", bytes / 1e9,
              e == cudaSuccess ? "ok" : "FAILED",
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                  .count());
    if (e != cudaSuccess) {
      cudaGetLastError();
      set_error("device allocation of %zu bytes failed: %s", bytes, cudaGetErrorString(e));
      return BM_ERR_NOMEM;
    }
    for (int i = 0; i < (int)g_big.size() && best < 0; ++i)
      if (!g_big[i].p && g_big[i].dev == dev) best = i;  // reuse an emptied entry
    if (best < 0) {
      BigBuf nb{};
      nb.dev = dev;
      if (cudaEventCreateWithFlags(&nb.ev, cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        cudaFree(p);
        set_error("cudaEventCreate failed");
        return BM_ERR_INTERNAL;
      }
      g_big.push_back(nb);
      best = (int)g_big.size() - 1;
    }
    g_big[best].p = p;
    g_big[best].bytes = bytes;
    g_big[best].pending = false;
  } else {
    if (trace_mem) fprintf(stderr, "[mem] big_acquire hit %.2f GB\n", bytes / 1e9);
    if (g_big[best].pending)  // the previous holder's work precedes this stream's use
      cudaStreamWaitEvent(stream, g_big[best].ev, 0);
  }
  g_big[best].busy = true;
  *out = g_big[best].p;
  *slot = best;
  return BM_OK;
}

void big_release(int slot, cudaStream_t stream) {
  std::lock_guard<std::mutex> lk(g_big_mu);
  if (slot < 0 || slot >= (int)g_big.size()) return;
  BigBuf& b = g_big[slot];
  if (cudaEventRecord(b.ev, stream) == cudaSuccess) {
    b.pending = true;
  } else {  // cannot order the next use: drain the stream instead
    cudaGetLastError();
    cudaStreamSynchronize(stream);
    b.pending = false;
  }
  b.busy = false;
}

void big_trim() {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_big_mu);
  for (auto& b : g_big)
    if (!b.busy && b.dev == dev && b.p) big_free_locked(b);
}

void release_pool() {
  big_trim();
  int dev = 0;
  cudaGetDevice(&dev);
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
  cudaGetLastError();
}

int scratch_alloc(Scratch& s, size_t bytes, cudaStream_t stream) {
  retain_pool_once();
  s.release();
  s.bytes = bytes;
  s.stream = stream;
  if (bytes == 0) bytes = 16;
  // large scratch comes from the cached large buffers: growing the
  // stream-ordered pool by GBs was measured to stall for 0.1-2.5 s when its
  // reserve is fragmented (cfg5's windows)
  if (bytes >= kScratchBig) return big_acquire(bytes, stream, &s.ptr, &s.slot);
  static const bool trace_mem = getenv("B200MAP_TRACE_MEM") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  cudaError_t e = cudaMallocAsync(&s.ptr, bytes, stream);
  if (trace_mem) {
    const double ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (ms > 1.0) fprintf(stderr, "[mem] scratch %.3f GB took %.1f ms\n", bytes / 1e9, ms);
  }
  if (e != cudaSuccess) {  // idle cached large buffers hold the memory: free them, retry
    cudaGetLastError();
    if (getenv("B200MAP_TRACE_MEM"))
      fprintf(stderr, "[mem] pool allocation of %.2f GB failed: trimming cached buffers\n",
              bytes / 1e9);
    big_trim();
    e = cudaMallocAsync(&s.ptr, bytes, stream);
  }
  if (e != cudaSuccess) {
    s.ptr = nullptr;
    cudaGetLastError();
    set_error("device scratch allocation of %zu bytes failed: %s", bytes,
              cudaGetErrorString(e));
    return BM_ERR_NOMEM;
  }
  return BM_OK;
}

size_t device_total_bytes() {
  static std::mutex mu;
  static size_t cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (dev < 64 && cache[dev]) return cache[dev];
  size_t f = 0, t = 0;
  if (cudaMemGetInfo(&f, &t) != cudaSuccess) {
    cudaGetLastError();
    t = 0;
  }
  if (dev < 64) cache[dev] = t;
  return t;
}

int ensure_dyn_smem(const void* fn, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int> done;
  int dev = 0;
  BM_CHECK_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_pair(dev, fn);
  auto it = done.find(key);
  if (it != done.end() && it->second >= bytes) return BM_OK;
  BM_CHECK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  done[key] = bytes;
  return BM_OK;
}

int num_sms() {
  static std::mutex mu;
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (dev < 64 && cache[dev]) return cache[dev];
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
  if (v <= 0) v = 148;
  if (dev < 64) cache[dev] = v;
  return v;
}

int make_pw_program(int64_t d, PwProgram* prog) {
  std::vector<PwLeaf> leaves = pw_plan((int)d);
  if ((int)leaves.size() > kMaxLeaves) {
    set_error("dimension %lld too large for the pairwise program (max %d)",
              (long long)d, kMaxLeaves * 128);
    return BM_ERR_DATA;
  }
  prog->n_leaves = (int32_t)leaves.size();
  int depth = 0, maxd = 0;
  for (size_t i = 0; i < leaves.size(); ++i) {
    prog->leaf[i] = leaves[i];
    depth += 1;
    if (depth > maxd) maxd = depth;
    depth -= leaves[i].pops;
  }
  if (maxd > kMaxStack) {
    set_error("pairwise program stack depth %d exceeds %d", maxd, kMaxStack);
    return BM_ERR_DATA;
  }
  prog->depth = maxd;
  return BM_OK;
}

// ---------------------------------------------------------------------------
// Exclusive scan (int64), three phases. Chunk = 4096 elements per block.
// ---------------------------------------------------------------------------
namespace {

constexpr int kScanThreads = 512;
constexpr int kScanPer = 8;
constexpr int kScanChunk = kScanThreads * kScanPer;

template <typename T>
__device__ __forceinline__ int64_t load_as_i64(const T* p, int64_t i, int64_t n) {
  return i < n ? (int64_t)p[i] : 0;
}

// Block-wide exclusive scan of one value per thread; returns the exclusive
// prefix and writes the block total to *total.
__device__ int64_t block_exclusive_scan(int64_t v, int64_t* total) {
  __shared__ int64_t warp_sums[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int nw = blockDim.x >> 5;
    int64_t w = lane < nw ? warp_sums[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < nw) warp_sums[lane] = w;
  }
  __syncthreads();
  int64_t warp_prefix = warp ? warp_sums[warp - 1] : 0;
  *total = warp_sums[(blockDim.x >> 5) - 1];
  __syncthreads();
  return warp_prefix + x - v;
}

template <typename T>
__global__ void scan_reduce_kernel(const T* in, int64_t n, int64_t* block_sums) {
  int64_t base = (int64_t)blockIdx.x * kScanChunk;
  int64_t s = 0;
  for (int j = 0; j < kScanPer; ++j) s += load_as_i64(in, base + j * kScanThreads + threadIdx.x, n);
  int64_t total;
  block_exclusive_scan(s, &total);
  if (threadIdx.x == 0) block_sums[blockIdx.x] = total;
}

__global__ void scan_blocksums_kernel(int64_t* sums, int64_t nb) {
  int64_t carry = 0;
  for (int64_t base = 0; base < nb; base += blockDim.x) {
    int64_t i = base + threadIdx.x;
    int64_t v = i < nb ? sums[i] : 0;
    int64_t total;
    int64_t ex = block_exclusive_scan(v, &total);
    if (i < nb) sums[i] = carry + ex;
    carry += total;
  }
}

template <typename T>
__global__ void scan_apply_kernel(const T* in, int64_t* out, int64_t n,
                                  const int64_t* block_sums) {
  int64_t base = (int64_t)blockIdx.x * kScanChunk;
  // blocked arrangement: thread t owns kScanPer consecutive items
  int64_t v[kScanPer];
  int64_t s = 0;
  for (int j = 0; j < kScanPer; ++j) {
    v[j] = load_as_i64(in, base + (int64_t)threadIdx.x * kScanPer + j, n);
    s += v[j];
  }
  int64_t total;
  int64_t ex = block_exclusive_scan(s, &total) + block_sums[blockIdx.x];
  for (int j = 0; j < kScanPer; ++j) {
    int64_t i = base + (int64_t)threadIdx.x * kScanPer + j;
    if (i < n) out[i] = ex;
    ex += v[j];
  }
}

template <typename T>
int exclusive_scan_impl(const T* d_in, int64_t* d_out, int64_t n, cudaStream_t stream) {
  if (n <= 0) return BM_OK;
  int64_t nb = ceil_div(n, kScanChunk);
  Scratch sums;
  BM_TRY(scratch_alloc(sums, nb * sizeof(int64_t), stream));
  scan_reduce_kernel<T><<<(unsigned)nb, kScanThreads, 0, stream>>>(d_in, n, sums.as<int64_t>());
  BM_CHECK_LAUNCH();
  scan_blocksums_kernel<<<1, 1024, 0, stream>>>(sums.as<int64_t>(), nb);
  BM_CHECK_LAUNCH();
  scan_apply_kernel<T><<<(unsigned)nb, kScanThreads, 0, stream>>>(d_in, d_out, n, sums.as<int64_t>());
  BM_CHECK_LAUNCH();
  return BM_OK;
}

}  // namespace

int exclusive_scan_i64(const int64_t* d_in, int64_t* d_out, int64_t n, cudaStream_t stream) {
  return exclusive_scan_impl<int64_t>(d_in, d_out, n, stream);
}

int exclusive_scan_i32_to_i64(const int32_t* d_in, int64_t* d_out, int64_t n,
                              cudaStream_t stream) {
  return exclusive_scan_impl<int32_t>(d_in, d_out, n, stream);
}

}  // namespace bm

extern "C" {

int bm_abi_version(void) { return 1; }

int64_t bm_launch_count(void) { return bm::g_launches.load(); }

int bm_release_scratch(void) {
  bm::release_pool();
  return BM_OK;
}

const char* bm_last_error(void) { return bm::get_error(); }

int bm_device_free_bytes(int64_t* out) {
  BM_REQUIRE(out, "null output");
  size_t f = 0;
  BM_TRY(bm::device_free_bytes(&f));
  *out = (int64_t)f;
  return BM_OK;
}

int bm_device_count(int* out) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  if (out) *out = n;
  return BM_OK;
}

}  // extern "C"
