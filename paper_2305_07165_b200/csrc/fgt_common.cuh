// Shared helpers for libfgtcuda (sm_100a).
#pragma once
#include <cstdlib>
#include <chrono>
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>
#include <string>
#include <stdexcept>
#include <vector>

#include "../../include/fgt_cuda.h"

namespace fgt {

// ---------------------------------------------------------------- errors
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string& msg);
void count_launch(int n = 1);

#define FGT_CUDA(expr)                                                              \
  do {                                                                              \
    cudaError_t _e = (expr);                                                        \
    if (_e != cudaSuccess) {                                                        \
      throw ::fgt::Error(_e == cudaErrorMemoryAllocation ? FGT_ENOMEM : FGT_ECUDA,  \
                         std::string(#expr) + ": " + cudaGetErrorString(_e) +      \
                             " (" + __FILE__ + ":" + std::to_string(__LINE__) + ")"); \
    }                                                                               \
  } while (0)

#define FGT_LAUNCHED()                 \
  do {                                 \
    FGT_CUDA(cudaPeekAtLastError());   \
    ::fgt::count_launch();             \
  } while (0)

#define FGT_REQUIRE(cond, code, msg)                   \
  do {                                                 \
    if (!(cond)) throw ::fgt::Error((code), (msg));    \
  } while (0)

// Run a body, translating exceptions into C status codes.
template <class F>
int guarded(F&& f) {
  try {
    f();
    return FGT_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return FGT_ENOMEM;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return FGT_ECUDA;
  }
}

// Keep freed pool memory mapped (default release threshold 0 trims the pool at every
// synchronisation, so multi-GB scratch would be unmapped/remapped on each call).
void ensure_pool_retained();

// Large buffers (>= BIG_BYTES) bypass the stream-ordered pool: carving multi-GB blocks
// out of a fragmented pool makes the driver remap physical pages, which blocks the host
// for 100s of ms while the GPU idles.  A process-lifetime cache of cudaMalloc'd blocks
// serves them instead: a freed block records an event on its stream and a later user on
// another stream waits on it, so reuse keeps stream order (api.cu).
constexpr size_t BIG_BYTES = size_t(64) << 20;
void* big_alloc(size_t bytes, cudaStream_t st);
void big_free(void* p, cudaStream_t st);

// ---------------------------------------------------------------- device buffers
// Stream-ordered device allocation (cudaMallocAsync pool): frees are ordered after
// the work already queued on the stream, so scratch never needs a device sync.
template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  DBuf() = default;
  DBuf(size_t count, cudaStream_t st) { alloc(count, st); }
  bool big = false;
  void alloc(size_t count, cudaStream_t st) {
    release();
    ensure_pool_retained();
    s = st;
    n = count;
    big = count * sizeof(T) >= BIG_BYTES;
    if (big) p = static_cast<T*>(big_alloc(count * sizeof(T), st));
    else if (count) FGT_CUDA(cudaMallocAsync((void**)&p, count * sizeof(T), st));
  }
  void zero() {
    if (n) FGT_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
  }
  void release() {
    if (p) {
      if (big) big_free(p, s);
      else cudaFreeAsync(p, s);
    }
    p = nullptr;
    n = 0;
    big = false;
  }
  ~DBuf() { release(); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), s(o.s), big(o.big) { o.p = nullptr; o.n = 0; o.big = false; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p; n = o.n; s = o.s; big = o.big;
      o.p = nullptr; o.n = 0; o.big = false;
    }
    return *this;
  }
  T* get() const { return p; }
  size_t size() const { return n; }
  void to_host(T* h, size_t count) const {
    if (count) FGT_CUDA(cudaMemcpyAsync(h, p, count * sizeof(T), cudaMemcpyDeviceToHost, s));
  }
  void from_host(const T* h, size_t count) {
    if (count) FGT_CUDA(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, s));
  }
};

// Grow-only device buffer for batch loops: one pool allocation serves every batch that
// fits (re-allocating per batch lets the stream-ordered pool fragment and grow, and pool
// growth blocks the host for milliseconds while the GPU idles).
template <class T>
struct BufView {  // a DBuf-like view of the first n elements of a GrowBuf
  T* p;
  size_t n;
  cudaStream_t s;
  T* get() const { return p; }
  size_t size() const { return n; }
  void from_host(const T* h, size_t count) {
    if (count) FGT_CUDA(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  void to_host(T* h, size_t count) const {
    if (count) FGT_CUDA(cudaMemcpyAsync(h, p, count * sizeof(T), cudaMemcpyDeviceToHost, s));
  }
  void zero() {
    if (n) FGT_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
  }
};

template <class T>
struct GrowBuf {
  DBuf<T> b;
  T* get(size_t count, cudaStream_t st) {
    if (b.size() < count) b.alloc(count + count / 4, st);
    return b.get();
  }
  BufView<T> view(size_t count, cudaStream_t st) { return BufView<T>{get(count, st), count, st}; }
};

// CUDA-event pair bracketing one kernel launch (device time of that kernel alone).
// Several begin/end intervals may be recorded; ms() returns their sum.
struct KClock {
  std::vector<cudaEvent_t> ev;
  void begin(cudaStream_t st) {
    cudaEvent_t a, b;
    FGT_CUDA(cudaEventCreate(&a));
    FGT_CUDA(cudaEventCreate(&b));
    FGT_CUDA(cudaEventRecord(a, st));
    ev.push_back(a);
    ev.push_back(b);
  }
  void end(cudaStream_t st) { FGT_CUDA(cudaEventRecord(ev.back(), st)); }
  double ms() const {
    double tot = 0.0;
    for (size_t i = 0; i + 1 < ev.size(); i += 2) {
      float v = 0.f;
      FGT_CUDA(cudaEventSynchronize(ev[i + 1]));
      FGT_CUDA(cudaEventElapsedTime(&v, ev[i], ev[i + 1]));
      tot += v;
    }
    return tot;
  }
  KClock() = default;
  KClock(const KClock&) = delete;
  KClock& operator=(const KClock&) = delete;
  ~KClock() {
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
  }
};

// Timeline tracing (FGT_TRACE=1): trace_mark records a CUDA event and the host clock;
// trace_dump prints, per mark, the device and host times since the first mark (device
// time that jumps while the host time advances = the GPU waited on the host).
struct TraceMark {
  const char* label;
  cudaEvent_t ev;
  double host_ms;
};
inline std::vector<TraceMark>& trace_marks() {
  static std::vector<TraceMark> m;
  return m;
}
inline bool trace_on() {
  static int on = -1;
  if (on < 0) {
    const char* e = std::getenv("FGT_TRACE");
    on = (e && *e && *e != '0') ? 1 : 0;
  }
  return on == 1;
}
inline void trace_mark(cudaStream_t st, const char* label) {
  if (!trace_on()) return;
  TraceMark m;
  m.label = label;
  cudaEventCreate(&m.ev);
  cudaEventRecord(m.ev, st);
  m.host_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
  trace_marks().push_back(m);
}
inline void trace_dump() {
  if (!trace_on() || trace_marks().empty()) return;
  auto& m = trace_marks();
  cudaEventSynchronize(m.back().ev);
  double prev = 0.0;
  std::fprintf(stderr, "%-28s %9s %9s %9s\n", "mark", "gpu_ms", "d_gpu", "host_ms");
  for (auto& x : m) {
    float g = 0.f;
    cudaEventElapsedTime(&g, m[0].ev, x.ev);
    std::fprintf(stderr, "%-28s %9.3f %9.3f %9.3f\n", x.label, g, g - prev, x.host_ms - m[0].host_ms);
    prev = g;
  }
  for (auto& x : m) cudaEventDestroy(x.ev);
  m.clear();
  int dev = 0;
  cudaMemPool_t pool;
  if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t rc = 0, rh = 0, uc = 0, uh = 0;
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &rc);
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemHigh, &rh);
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &uc);
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &uh);
    std::fprintf(stderr, "pool reserved %.2f GB (high %.2f), used %.2f GB (high %.2f)\n", rc / 1e9, rh / 1e9,
                 uc / 1e9, uh / 1e9);
  }
}

inline unsigned grid_for(int64_t n, int block, int64_t cap = 148 * 64) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (unsigned)g;
}

// ---------------------------------------------------------------- device math
// Box centre per axis exactly as tree._Builder.center (tree.py:141-143):
//   (root_center - 0.5*root_side) + (coord + 0.5) * s,  s = root_side / 2**level.
// Each operation is rounded separately (no FMA contraction), which is what numpy does.
__device__ __forceinline__ double box_center_1d(double root_low, int64_t coord, double s) {
  return __dadd_rn(root_low, __dmul_rn((double)coord + 0.5, s));
}

__host__ __device__ __forceinline__ int pow2i(int k) { return 1 << k; }

// Morton helpers: a box at level l with integer coords g (each < 2^l) has code
//   sum_{lv<l} childno(lv) << (d*(l-1-lv)),  childno = sum_k bit_k << k
// (child c has axis-k bit (c>>k)&1, tree.py:131-132), so code(parent) = code >> d.
__host__ __device__ __forceinline__ uint64_t morton_encode(const int64_t* g, int d, int l) {
  uint64_t code = 0;
  for (int b = l - 1; b >= 0; --b) {
    uint64_t c = 0;
    for (int k = 0; k < d; ++k) c |= (uint64_t)((g[k] >> b) & 1) << k;
    code = (code << d) | c;
  }
  return code;
}
__host__ __device__ __forceinline__ void morton_decode(uint64_t code, int d, int l, int64_t* g) {
  for (int k = 0; k < d; ++k) g[k] = 0;
  for (int b = 0; b < l; ++b) {
    uint64_t c = (code >> (d * b)) & ((1u << d) - 1);
    for (int k = 0; k < d; ++k) g[k] |= (int64_t)((c >> k) & 1) << b;
  }
}

// Global box key: level in the top 6 bits, Morton code below (level-major order).
constexpr int KEY_LEVEL_SHIFT = 58;
__host__ __device__ __forceinline__ uint64_t box_key(int level, uint64_t code) {
  return ((uint64_t)level << KEY_LEVEL_SHIFT) | code;
}
__host__ __device__ __forceinline__ int key_level(uint64_t key) {
  return (int)(key >> KEY_LEVEL_SHIFT);
}
__host__ __device__ __forceinline__ uint64_t key_code(uint64_t key) {
  return key & ((1ull << KEY_LEVEL_SHIFT) - 1);
}

// lower_bound on a sorted device array.
template <class T>
__device__ __forceinline__ int64_t lower_bound_dev(const T* a, int64_t n, T v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}
template <class T>
__device__ __forceinline__ int64_t find_dev(const T* a, int64_t n, T v) {
  int64_t i = lower_bound_dev(a, n, v);
  return (i < n && a[i] == v) ? i : -1;
}

}  // namespace fgt
