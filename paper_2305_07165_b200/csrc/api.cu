// extern "C" surface of libfgtcuda.so (declared in include/fgt_cuda.h).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <map>
#include <memory>

#include <cub/cub.cuh>

#include "k_kernels.cuh"
#include "k_nufft.cuh"

namespace fgt {

static thread_local std::string g_last_error;
static thread_local int64_t g_launches = 0;

void set_last_error(const std::string& msg) { g_last_error = msg; }

void ensure_pool_retained() {
  static thread_local int done_dev = -1;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev == done_dev) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done_dev = dev;
}
void count_launch(int n) { g_launches += n; }

namespace {
struct BigBlock {
  void* p;
  size_t bytes;
  int dev;
  bool busy;
  cudaStream_t last;
  cudaEvent_t ev;
};
std::mutex& big_mu() {
  static std::mutex m;
  return m;
}
std::vector<BigBlock>& big_blocks() {
  static auto* v = new std::vector<BigBlock>();  // process lifetime
  return *v;
}
}  // namespace

void* big_alloc(size_t bytes, cudaStream_t st) {
  const size_t rounded = (bytes + (size_t(2) << 20) - 1) & ~((size_t(2) << 20) - 1);
  int dev = 0;
  FGT_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(big_mu());
  auto& v = big_blocks();
  // best fit among idle blocks of this device no larger than 2x the request
  BigBlock* best = nullptr;
  for (auto& b : v)
    if (!b.busy && b.dev == dev && b.bytes >= rounded && b.bytes <= 2 * rounded &&
        (!best || b.bytes < best->bytes))
      best = &b;
  if (best) {
    best->busy = true;
    if (best->last != st) FGT_CUDA(cudaStreamWaitEvent(st, best->ev, 0));
    return best->p;
  }
  BigBlock b;
  b.bytes = rounded;
  b.dev = dev;
  b.busy = true;
  b.last = st;
  cudaError_t e = cudaMalloc(&b.p, rounded);
  if (e != cudaSuccess) {
    // release idle cached blocks of this device and retry once
    cudaGetLastError();
    FGT_CUDA(cudaDeviceSynchronize());
    for (auto it = v.begin(); it != v.end();) {
      if (!it->busy && it->dev == dev) {
        cudaFree(it->p);
        cudaEventDestroy(it->ev);
        it = v.erase(it);
      } else {
        ++it;
      }
    }
    e = cudaMalloc(&b.p, rounded);
    if (e == cudaErrorMemoryAllocation) throw Error(FGT_ENOMEM, "device allocation failed");
    FGT_CUDA(e);
  }
  FGT_CUDA(cudaEventCreateWithFlags(&b.ev, cudaEventDisableTiming));
  v.push_back(b);
  return b.p;
}

void big_free(void* p, cudaStream_t st) {
  std::lock_guard<std::mutex> lock(big_mu());
  for (auto& b : big_blocks())
    if (b.p == p) {
      cudaEventRecord(b.ev, st);
      b.last = st;
      b.busy = false;
      return;
    }
}

// RAII stream for host-pointer entry points
struct OwnedStream {
  cudaStream_t s = nullptr;
  OwnedStream() { FGT_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }
  ~OwnedStream() {
    if (s) {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  }
};

// Phase boundaries as events on the stream, read once at the end (no host stall between
// phases).
struct PhaseMarks {
  std::vector<cudaEvent_t> ev;
  cudaStream_t st;
  explicit PhaseMarks(cudaStream_t s) : st(s) { mark(); }
  void mark() {
    cudaEvent_t e;
    FGT_CUDA(cudaEventCreate(&e));
    FGT_CUDA(cudaEventRecord(e, st));
    ev.push_back(e);
  }
  // elapsed ms between marks i and i + 1 (or i and j)
  double ms(size_t i) const { return ms(i, i + 1); }
  double ms(size_t i, size_t j) const {
    FGT_CUDA(cudaEventSynchronize(ev[j]));
    float v = 0;
    FGT_CUDA(cudaEventElapsedTime(&v, ev[i], ev[j]));
    return v;
  }
  ~PhaseMarks() {
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
  }
};

// Streams of the host-buffer entry points: created once per (host thread, device) and kept
// (creating and destroying two streams costs ~0.1 ms per call).  s = the transform, side =
// the overlapped charge upload.
struct HostStreams {
  cudaStream_t s = nullptr, side = nullptr;
};
static HostStreams& host_streams() {
  static thread_local std::map<int, HostStreams> per_dev;
  int dev = 0;
  FGT_CUDA(cudaGetDevice(&dev));
  HostStreams& h = per_dev[dev];
  if (!h.s) {
    FGT_CUDA(cudaStreamCreateWithFlags(&h.s, cudaStreamNonBlocking));
    FGT_CUDA(cudaStreamCreateWithFlags(&h.side, cudaStreamNonBlocking));
  }
  return h;
}

struct Event {
  cudaEvent_t e = nullptr;
  Event() { FGT_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming)); }
  ~Event() { cudaEventDestroy(e); }
};

struct Timer {
  cudaEvent_t a, b;
  cudaStream_t st;
  explicit Timer(cudaStream_t s) : st(s) {
    FGT_CUDA(cudaEventCreate(&a));
    FGT_CUDA(cudaEventCreate(&b));
    FGT_CUDA(cudaEventRecord(a, st));
  }
  double lap() {
    FGT_CUDA(cudaEventRecord(b, st));
    FGT_CUDA(cudaEventSynchronize(b));
    float ms = 0;
    FGT_CUDA(cudaEventElapsedTime(&ms, a, b));
    std::swap(a, b);
    return ms;
  }
  ~Timer() {
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
};

__global__ void scatter_kernel(const double* __restrict__ us, const int64_t* __restrict__ perm, int64_t n,
                               double* __restrict__ u) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    u[perm[i]] = us[i];
}

// multi-GPU shares: the potentials of the listed boxes' targets only (a warp per box; u was
// zeroed, and a share's targets all sit in its direct target leaves or its psi boxes)
__global__ void scatter_boxes_kernel(const int64_t* __restrict__ ids, int64_t n, const int64_t* __restrict__ start,
                                     const int64_t* __restrict__ count, const double* __restrict__ us,
                                     const int64_t* __restrict__ perm, double* __restrict__ u) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarp = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t k = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); k < n; k += nwarp) {
    const int64_t b = ids[k], s0 = start[b], m = count[b];
    for (int64_t i = lane; i < m; i += 32) u[perm[s0 + i]] = us[s0 + i];
  }
}




// the rank's direct target leaves (positions into the replicated CSR): ids, begin, end
__global__ void restrict_direct_kernel(const int64_t* __restrict__ pos, int64_t n, const int64_t* __restrict__ tl,
                                       const int64_t* __restrict__ off, int64_t* __restrict__ ids,
                                       int64_t* __restrict__ beg, int64_t* __restrict__ end) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = pos[i];
    ids[i] = tl[p];
    beg[i] = off[p];
    end[i] = off[p + 1];
  }
}

std::vector<int64_t> partition_bounds(const std::vector<double>& cost, int parts) {
  const int64_t n = (int64_t)cost.size();
  std::vector<int64_t> b(parts + 1, n);
  b[0] = 0;
  double total = 0;
  for (double c : cost) total += c;
  double acc = 0;
  int r = 1;
  for (int64_t i = 0; i < n && r < parts; ++i) {
    acc += cost[i];
    while (r < parts && acc >= total * r / parts) b[r++] = i + 1;
  }
  for (; r < parts; ++r) b[r] = n;
  return b;
}

// Multi-GPU shares (one process per GPU).  Every rank builds the same tree and lists,
// then keeps a cost-balanced contiguous range of target leaves (canonical = Morton order
// at each level).  P-box expansions either get recomputed by every rank that needs them
// (exchange = false: a one-box halo of extra form work, no communication) or are formed
// only by their owner -- the rank whose leaf range holds the box -- and the one-box halo
// is exchanged (exchange = true: ExchangePlan, then an all-to-all of the packed slots).
struct ExchangePlan {
  int rank = 0, world = 1;
  std::vector<int64_t> send_off, recv_off;  // (world + 1) slot offsets per peer
  DBuf<int64_t> send_slots, recv_slots;     // dense slots, concatenated in peer order
};

__global__ void pack_slots_kernel(const double2* __restrict__ phi, const int64_t* __restrict__ slots,
                                  int64_t n, int64_t NH, double2* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n * NH;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = i / NH, e = i - k * NH;
    out[i] = phi[slots[k] * NH + e];
  }
}

__global__ void unpack_slots_kernel(double2* __restrict__ phi, const int64_t* __restrict__ slots,
                                    int64_t n, int64_t NH, const double2* __restrict__ in) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n * NH;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = i / NH, e = i - k * NH;
    phi[slots[k] * NH + e] = in[i];
  }
}

// ---- share planning on the device: per target leaf its cost, its Morton key across levels
// (code at l_c of its first cell) and its psi index; the leaves are sorted by that key, the
// cost prefix sum cut into `size` balanced ranges, every P-box's owner found from its key
// and every rank's needs marked with a bit per rank (one pass over the P entries).  Only
// per-rank bounds and per-slot owner / need words (n_dense entries) come back to the host.
__device__ __forceinline__ uint64_t deep_key(uint64_t key, int d, int l_c) {
  return key_code(key) << (d * (l_c - key_level(key)));
}

__global__ void share_leaf_kernel(const int64_t* __restrict__ tl, int64_t n, const int64_t* __restrict__ d_off,
                                  const int64_t* __restrict__ d_src, const int64_t* __restrict__ scount,
                                  const int64_t* __restrict__ tcount, const int64_t* __restrict__ dense_slot,
                                  const int64_t* __restrict__ psi_ids, int64_t nps, const int64_t* __restrict__ p_off,
                                  const uint64_t* __restrict__ bkey, int d, int l_c, double NH, double form_ns,
                                  double* __restrict__ cost, uint64_t* __restrict__ dk, int64_t* __restrict__ iota,
                                  uint8_t* __restrict__ has_psi) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t T = tl[i];
    double src = 0;
    for (int64_t e = d_off[i]; e < d_off[i + 1]; ++e) src += (double)scount[d_src[e]];
    const double nt = (double)tcount[T];
    // cost in ns, calibrated on the B200 kernels: direct ~10 ps per pair, eval 8 N_H flops
    // per target at ~21 TFLOP/s, gather ~2.4 ps per stored mode per P entry; with the
    // exchange a P-box's form (~2.4 ns per source at w = 11, ~w^3) is charged to its leaf
    double c = 0.01 * nt * src + (dense_slot[T] >= 0 ? form_ns * (double)scount[T] : 0.0);
    const int64_t j = find_dev(psi_ids, nps, T);
    if (j >= 0) c += 8.0 * NH * nt / 21e3 + 2.4e-3 * NH * (double)(p_off[j + 1] - p_off[j]);
    cost[i] = c;
    dk[i] = deep_key(bkey[T], d, l_c);
    iota[i] = i;
    has_psi[i] = j >= 0;
  }
}

__global__ void share_order_kernel(const int64_t* __restrict__ ord, int64_t n, const double* __restrict__ cost,
                                   const uint8_t* __restrict__ has_psi, double* __restrict__ cost_o,
                                   int64_t* __restrict__ psi_flag_o) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    cost_o[k] = cost[ord[k]];
    psi_flag_o[k] = has_psi[ord[k]];
  }
}

// one thread: b[r] (leaf ranges, the host partition_bounds rule on the inclusive prefix),
// pb[r] (psi index ranges: psi boxes appear in ascending index along the Morton order),
// thr[r] (first Morton key of rank r); out = [b (P+1) | pb (P+1) | thr (P+1)]
__global__ void share_bounds_kernel(const double* __restrict__ pre, const int64_t* __restrict__ psi_cnt,
                                    const uint64_t* __restrict__ dks, int64_t n, int64_t nps, int P,
                                    int64_t* __restrict__ out) {
  if (threadIdx.x || blockIdx.x) return;
  const double total = n > 0 ? pre[n - 1] : 0.0;
  int64_t* b = out;
  int64_t* pb = out + P + 1;
  uint64_t* thr = reinterpret_cast<uint64_t*>(out + 2 * (P + 1));
  b[0] = 0;
  b[P] = n;
  for (int r = 1; r < P; ++r) {
    const double t = total * r / P;
    int64_t lo = 0, hi = n;  // first i with pre[i] >= t
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (pre[mid] >= t) hi = mid; else lo = mid + 1;
    }
    b[r] = lo < n ? lo + 1 : n;
    if (b[r] < b[r - 1]) b[r] = b[r - 1];
  }
  for (int r = 0; r <= P; ++r) {
    pb[r] = b[r] < n ? psi_cnt[b[r]] : nps;
    thr[r] = b[r] < n ? dks[b[r]] : ~(uint64_t)0;
  }
  thr[0] = 0;
}

__global__ void share_need_kernel(const int64_t* __restrict__ bounds, int P, int64_t nps,
                                  const int64_t* __restrict__ p_off, const int64_t* __restrict__ p_src,
                                  unsigned long long* __restrict__ need) {
  const int64_t* pb = bounds + P + 1;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nps; j += (int64_t)gridDim.x * blockDim.x) {
    int r = 0;
    while (r + 1 < P && pb[r + 1] <= j) ++r;
    const unsigned long long bit = 1ull << r;
    for (int64_t e = p_off[j]; e < p_off[j + 1]; ++e) atomicOr(&need[p_src[e]], bit);
  }
}

__global__ void share_owner_kernel(const int64_t* __restrict__ bounds, int P, const int64_t* __restrict__ dense_ids,
                                   int64_t nd, const uint64_t* __restrict__ bkey, int d, int l_c,
                                   int32_t* __restrict__ owner) {
  const uint64_t* thr = reinterpret_cast<const uint64_t*>(bounds + 2 * (P + 1));
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < nd; s += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = deep_key(bkey[dense_ids[s]], d, l_c);
    int r = 0;
    while (r + 1 < P && thr[r + 1] <= key) ++r;
    owner[s] = r;
  }
}

// boxes whose points a rank touches: its target leaves and their D-list sources, its psi
// boxes, and the P-boxes whose expansions it forms
__global__ void need_leaf_kernel(const int64_t* __restrict__ ids, const int64_t* __restrict__ off,
                                 const int64_t* __restrict__ end, int64_t n, const int64_t* __restrict__ d_src,
                                 uint8_t* __restrict__ need_src, uint8_t* __restrict__ need_tgt) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    need_tgt[ids[i]] = 1;
    for (int64_t e = off[i]; e < end[i]; ++e) need_src[d_src[e]] = 1;
  }
}
__global__ void need_ids_kernel(const int64_t* __restrict__ ids, const uint8_t* __restrict__ sel, int64_t n,
                                uint8_t* __restrict__ need) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (!sel || sel[i]) need[ids[i]] = 1;
}

// leaf-ordered points of the rank's share only (after plan_share)
static void gather_share_points(TreeDev& T, const double* src, const double* q, const double* tgt) {
  cudaStream_t st = T.st;
  DBuf<uint8_t> ns(std::max<int64_t>(T.nb, 1), st), nt(std::max<int64_t>(T.nb, 1), st);
  ns.zero();
  nt.zero();
  if (T.n_dtgt > 0) {
    need_leaf_kernel<<<grid_for(T.n_dtgt, 256), 256, 0, st>>>(T.d_tgt_ids.get(), T.d_off.get(), T.d_end.get(), T.n_dtgt,
                                                             T.d_src.get(), ns.get(), nt.get());
    FGT_LAUNCHED();
  }
  if (T.n_psi > 0) {
    need_ids_kernel<<<grid_for(T.n_psi, 256), 256, 0, st>>>(T.psi_ids.get(), nullptr, T.n_psi, nt.get());
    FGT_LAUNCHED();
  }
  if (T.n_dense > 0) {
    DBuf<uint8_t> sel(T.n_dense, st);
    sel.from_host(T.dense_need.data(), T.n_dense);
    need_ids_kernel<<<grid_for(T.n_dense, 256), 256, 0, st>>>(T.dense_ids.get(), sel.get(), T.n_dense, ns.get());
    FGT_LAUNCHED();
    // (dense_need is pageable host memory: the copy above has left it when it returned)
  }
  order_leaf_points(T, ns.get(), nt.get());
  gather_needed_points(T, src, q, tgt, ns.get(), nt.get());
}

static void plan_share(TreeDev& T, int rank, int size, int64_t NH, int w, bool exchange, ExchangePlan* X) {
  cudaStream_t st = T.st;
  FGT_REQUIRE(size <= 64, FGT_ERANGE, "at most 64 ranks");
  const int64_t n = T.n_dtgt, nps = T.n_psi, nd = T.n_dense;
  const int P = size;
  const double form_ns = exchange ? 2.4 * std::pow(w / 11.0, 3) : 0.0;
  DBuf<double> cost(std::max<int64_t>(n, 1), st), cost_o(std::max<int64_t>(n, 1), st), pre(std::max<int64_t>(n, 1), st);
  DBuf<uint64_t> dk(std::max<int64_t>(n, 1), st), dks(std::max<int64_t>(n, 1), st);
  DBuf<int64_t> iota(std::max<int64_t>(n, 1), st), ord(std::max<int64_t>(n, 1), st),
      psi_flag(std::max<int64_t>(n, 1), st), psi_cnt(std::max<int64_t>(n, 1), st), bounds(3 * (P + 1), st);
  DBuf<uint8_t> has_psi(std::max<int64_t>(n, 1), st);
  DBuf<unsigned long long> need(std::max<int64_t>(nd, 1), st);
  DBuf<int32_t> owner(std::max<int64_t>(nd, 1), st);
  DBuf<uint8_t> tmp;
  if (n > 0) {
    share_leaf_kernel<<<grid_for(n, 256), 256, 0, st>>>(T.d_tgt_ids.get(), n, T.d_off.get(), T.d_src.get(),
                                                        T.src_count.get(), T.tgt_count.get(), T.dense_slot.get(),
                                                        T.psi_ids.get(), nps, T.p_off.get(), T.bkey.get(), T.d, T.l_c,
                                                        (double)NH, form_ns, cost.get(), dk.get(), iota.get(),
                                                        has_psi.get());
    FGT_LAUNCHED();
    size_t bytes = 0;
    const int bits = std::max(1, T.d * T.l_c);
    FGT_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, dk.get(), dks.get(), iota.get(), ord.get(), (int)n, 0, bits, st));
    tmp.alloc(bytes, st);
    FGT_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), bytes, dk.get(), dks.get(), iota.get(), ord.get(), (int)n, 0, bits, st));
    count_launch();
    share_order_kernel<<<grid_for(n, 256), 256, 0, st>>>(ord.get(), n, cost.get(), has_psi.get(), cost_o.get(),
                                                         psi_flag.get());
    FGT_LAUNCHED();
    bytes = 0;
    FGT_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, cost_o.get(), pre.get(), (int)n, st));
    if (bytes > tmp.size()) tmp.alloc(bytes, st);
    FGT_CUDA(cub::DeviceScan::InclusiveSum(tmp.get(), bytes, cost_o.get(), pre.get(), (int)n, st));
    bytes = 0;
    FGT_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, psi_flag.get(), psi_cnt.get(), (int)n, st));
    if (bytes > tmp.size()) tmp.alloc(bytes, st);
    FGT_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), bytes, psi_flag.get(), psi_cnt.get(), (int)n, st));
    count_launch();
  }
  share_bounds_kernel<<<1, 1, 0, st>>>(pre.get(), psi_cnt.get(), dks.get(), n, nps, P, bounds.get());
  FGT_LAUNCHED();
  if (nd > 0) {
    need.zero();
    share_need_kernel<<<grid_for(std::max<int64_t>(nps, 1), 256), 256, 0, st>>>(bounds.get(), P, nps, T.p_off.get(),
                                                                                 T.p_src.get(), need.get());
    FGT_LAUNCHED();
    share_owner_kernel<<<grid_for(nd, 256), 256, 0, st>>>(bounds.get(), P, T.dense_ids.get(), nd, T.bkey.get(), T.d,
                                                          T.l_c, owner.get());
    FGT_LAUNCHED();
  }
  // read back: bounds (3 (P + 1)), need (nd), owner (nd) into one pinned block
  static thread_local char* hbuf = nullptr;
  static thread_local size_t hcap = 0;
  const size_t o_need = 3 * (P + 1) * sizeof(int64_t), o_own = o_need + nd * sizeof(uint64_t),
               tot = o_own + nd * sizeof(int32_t);
  if (tot > hcap) {
    if (hbuf) FGT_CUDA(cudaFreeHost(hbuf));
    hcap = std::max(tot, 2 * hcap);
    FGT_CUDA(cudaMallocHost((void**)&hbuf, hcap));
  }
  trace_mark(st, "share:plan(device)");
  FGT_CUDA(cudaMemcpyAsync(hbuf, bounds.get(), o_need, cudaMemcpyDeviceToHost, st));
  if (nd > 0) {
    FGT_CUDA(cudaMemcpyAsync(hbuf + o_need, need.get(), nd * sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    FGT_CUDA(cudaMemcpyAsync(hbuf + o_own, owner.get(), nd * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  }
  FGT_CUDA(cudaStreamSynchronize(st));
  trace_mark(st, "share:d2h(sync)");
  const int64_t* hb = reinterpret_cast<const int64_t*>(hbuf);
  const int64_t* hpb = hb + P + 1;
  const uint64_t* hneed = reinterpret_cast<const uint64_t*>(hbuf + o_need);
  const int32_t* hown = reinterpret_cast<const int32_t*>(hbuf + o_own);
  const int64_t lo = hb[rank], hi = hb[rank + 1];
  const int64_t plo = hpb[rank], phi = hpb[rank + 1];
  const uint64_t me = (uint64_t)1 << rank;
  T.dense_need.assign(nd, 0);
  if (!exchange) {
    for (int64_t s = 0; s < nd; ++s) T.dense_need[s] = (hneed[s] & me) != 0;
  } else {
    X->rank = rank;
    X->world = size;
    X->send_off.assign(size + 1, 0);
    X->recv_off.assign(size + 1, 0);
    // per peer, slots in ascending order on both sides: the owner sends what the peer needs,
    // the peer receives what it needs from that owner
    std::vector<std::vector<int64_t>> sendr(size), recvr(size);
    for (int64_t s = 0; s < nd; ++s) {
      const uint64_t m = hneed[s];
      if (!m) continue;
      if (hown[s] == rank) {
        T.dense_need[s] = 1;
        for (int r = 0; r < size; ++r)
          if (r != rank && ((m >> r) & 1)) sendr[r].push_back(s);
      } else if (m & me) {
        recvr[hown[s]].push_back(s);
      }
    }
    std::vector<int64_t> send, recv;
    for (int r = 0; r < size; ++r) {
      send.insert(send.end(), sendr[r].begin(), sendr[r].end());
      recv.insert(recv.end(), recvr[r].begin(), recvr[r].end());
      X->send_off[r + 1] = (int64_t)send.size();
      X->recv_off[r + 1] = (int64_t)recv.size();
    }
    X->send_slots.alloc(send.size(), st);
    X->send_slots.from_host(send.data(), send.size());
    X->recv_slots.alloc(recv.size(), st);
    X->recv_slots.from_host(recv.data(), recv.size());
  }
  trace_mark(st, "share:plans");
  // restrict the direct lists to the rank's leaves (begin / end per leaf into the
  // replicated entry arrays)
  {
    const int64_t m = hi - lo;
    DBuf<int64_t> ids(std::max<int64_t>(m, 1), st), beg(std::max<int64_t>(m, 1), st), end(std::max<int64_t>(m, 1), st);
    if (m > 0) {
      restrict_direct_kernel<<<grid_for(m, 256), 256, 0, st>>>(ord.get() + lo, m, T.d_tgt_ids.get(), T.d_off.get(),
                                                               ids.get(), beg.get(), end.get());
      FGT_LAUNCHED();
    }
    T.d_tgt_ids = std::move(ids);
    T.d_off = std::move(beg);
    T.d_end = std::move(end);
    T.n_dtgt = m;
  }
  // restrict psi boxes
  {
    DBuf<int64_t> ids(phi - plo, st), off(phi - plo + 1, st);
    if (phi > plo) FGT_CUDA(cudaMemcpyAsync(ids.get(), T.psi_ids.get() + plo, (phi - plo) * sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
    FGT_CUDA(cudaMemcpyAsync(off.get(), T.p_off.get() + plo, (phi - plo + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
    T.psi_ids = std::move(ids);
    T.p_off = std::move(off);
    T.n_psi = phi - plo;
  }
}

// One transform split at the exchange point: begin = tree, lists, share, own expansions;
// finish = translation, evaluation, near field, scatter.
struct PointsRun {
  cudaStream_t st = nullptr;
  cudaStream_t sb = nullptr;  // side stream of the overlapped single-GPU path (else null)
  cudaEvent_t ev_direct = nullptr;
  KClock k_lists;             // lists on the side stream
  TreeDev T;
  PwDev P;
  const NufftPlan* NP = nullptr;
  DBuf<double> us, ud;        // ud: near-field sums of the overlapped path
  fgt_tree_params tp;
  fgt_pw_params pw;
  std::vector<double> w1d;
  ExchangePlan X;
  std::unique_ptr<PhaseMarks> pm;
  int64_t l0 = 0, nt = 0;
  ~PointsRun() {
    if (ev_direct) cudaEventDestroy(ev_direct);
  }
};

// Side stream of the overlapped pipeline: one per (host thread, device), kept.
static cudaStream_t side_stream() {
  static thread_local std::map<int, cudaStream_t> per_dev;
  int dev = 0;
  FGT_CUDA(cudaGetDevice(&dev));
  cudaStream_t& s = per_dev[dev];
  if (!s) FGT_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  return s;
}

__global__ void scatter_add_kernel(const double* __restrict__ us, const double* __restrict__ ud,
                                   const int64_t* __restrict__ perm, int64_t n, double* __restrict__ u) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    u[perm[i]] = us[i] + ud[i];
}

static void points_begin(PointsRun& R, const double* src, int64_t ns, const double* q, const double* tgt,
                         int64_t nt, const fgt_tree_params& tp, const fgt_pw_params& pw, cudaStream_t st,
                         bool exchange, cudaEvent_t q_ready = nullptr) {
  FGT_REQUIRE(tp.dim == pw.dim, FGT_EINVAL, "tree/plane-wave dim mismatch");
  R.st = st;
  R.tp = tp;
  R.pw = pw;
  R.w1d.assign(pw.weights_1d, pw.weights_1d + pw.n_f);
  R.pw.weights_1d = R.w1d.data();
  R.nt = nt;
  R.l0 = g_launches;
  R.pm.reset(new PhaseMarks(st));  // marks: 0 start, 1 tree, 2 lists, 3 form, 4 gather+eval, 5 direct
  trace_mark(st, "start");
  TreeDev& T = R.T;
  {
    const char* env_min = std::getenv("FGT_SHARE_GATHER_MIN");
    T.defer_order = tp.part_size > 1 && ns + nt >= (env_min ? atoll(env_min) : ((int64_t)1 << 23));
  }
  build_tree(T, src, ns, tgt, nt, tp, st);
  if (q_ready) FGT_CUDA(cudaStreamWaitEvent(st, q_ready, 0));  // charges copied on a side stream
  // multi-GPU shares gather the leaf-ordered points after the share is planned, and only
  // the rank's own (plan_share needs counts, not coordinates)
  // (below ~8M points the full gather is cheaper than planning the restricted one;
  // FGT_SHARE_GATHER_MIN overrides the threshold for tests)
  const bool shared = T.defer_order;
  if (!shared) gather_sorted_points(T, src, q, tgt);
  R.pm->mark();
  trace_mark(st, "tree");
  const double D0 = tp.D0;
  const double tol = 0.3 * std::exp(-pw.D0 * pw.D0);
  if (tp.part_size <= 1 && !exchange && T.n_dense > 0) {
    // Single GPU: the form needs only the tree, the lists only the tree, and the near
    // field only the lists.  The form is enqueued on st first (its one host round trip
    // waits on st only); then the lists, the psi metadata and the near-field sums run on
    // a side stream, on the GPU alongside the form's kernels.  Gather / eval (st) wait for
    // the lists; the final scatter waits for the near field and adds it (u = eval + near,
    // the same single addition per target as the sequential path).
    cudaStream_t sb = side_stream();
    R.sb = sb;
    Event e_tree, e_lists;
    FGT_CUDA(cudaEventRecord(e_tree.e, st));
    FGT_CUDA(cudaStreamWaitEvent(sb, e_tree.e, 0));
    R.pm->mark();  // (lists: on the side stream, timed by k_lists)
    T.st = sb;
    // side-stream busy time only: two intervals (enumeration; compaction + psi metadata),
    // not the span in between while the host enqueues the form
    R.k_lists.begin(sb);
    build_lists_begin(T);  // list enumeration, no host wait
    R.k_lists.end(sb);
    T.st = st;
    R.us.alloc(nt, st);
    R.us.zero();
    pw_setup_dense(R.P, T, R.pw);
    trace_mark(st, "setup");
    const double X = 0.5 * R.P.side_lc * R.P.sc * (1.0 + 1e-12);
    R.NP = &nufft_plan_cached(pw.n_f, tol, X, R.w1d.data(), st);
    pw_form(R.P, T, R.NP);
    R.pm->mark();
    trace_mark(st, "form(enqueued)");
    T.st = sb;
    R.k_lists.begin(sb);
    build_lists_end(T);
    pw_setup_psi(R.P, T);
    R.k_lists.end(sb);
    FGT_CUDA(cudaEventRecord(e_lists.e, sb));
    R.ud.alloc(nt, sb);
    R.ud.zero();
    direct_lists(T, 1.0 / tp.delta, D0 * D0 * tp.delta, R.ud.get(), &R.P.k_direct);
    FGT_CUDA(cudaEventCreateWithFlags(&R.ev_direct, cudaEventDisableTiming));
    FGT_CUDA(cudaEventRecord(R.ev_direct, sb));
    T.st = st;
    FGT_CUDA(cudaStreamWaitEvent(st, e_lists.e, 0));
    trace_mark(st, "form");
    return;
  }
  build_lists(T);
  // stored modes (half spectrum for d >= 2) and the NUFFT width the plan will use
  int64_t NH = pw.dim >= 2 ? pw.n_f / 2 + 1 : pw.n_f;
  for (int k = 1; k < pw.dim; ++k) NH *= pw.n_f;
  const int w = std::max(2, std::min((int)std::ceil(std::log10(1.0 / tol) - 1e-9) + 1, 16));
  if (tp.part_size > 1) {
    FGT_REQUIRE(tp.part_rank >= 0 && tp.part_rank < tp.part_size, FGT_EINVAL, "bad part_rank");
    plan_share(T, tp.part_rank, tp.part_size, NH, w, exchange, &R.X);
    if (shared) gather_share_points(T, src, q, tgt);
  }
  R.pm->mark();
  trace_mark(st, "lists");
  R.us.alloc(nt, st);
  R.us.zero();
  if (T.n_dense > 0) {
    pw_setup(R.P, T, R.pw);
    trace_mark(st, "setup");
    // box-local NUFFT plan at tolerance eps/10; eps = 3 exp(-D0^2)
    const double X = 0.5 * R.P.side_lc * R.P.sc * (1.0 + 1e-12);
    R.NP = &nufft_plan_cached(pw.n_f, tol, X, R.w1d.data(), st);
    trace_mark(st, "nufft_plan");
    pw_form(R.P, T, R.NP);
  }
  R.pm->mark();
  trace_mark(st, "form");
}

// u_host (optional): the result's device->host copy is enqueued right behind the scatter,
// before the phase timings are read (which waits on the stream).
static void points_finish(PointsRun& R, double* u, fgt_phase_times* times, double* u_host = nullptr) {
  // phases of finish are timed from its own start: with the exchange path other ranks'
  // work and the all-to-all sit between begin and finish on a shared GPU
  const size_t m_fin = R.pm->ev.size();
  R.pm->mark();
  cudaStream_t st = R.st;
  TreeDev& T = R.T;
  PwDev& P = R.P;
  if (T.n_dense > 0) {
    pw_gather_eval(P, T, R.us.get(), R.NP);
    P.phi.release();
    P.psi.release();
  }
  R.pm->mark();
  trace_mark(st, "gather+eval");
  if (R.sb) {
    // overlapped path: the near field ran on the side stream into ud
    FGT_CUDA(cudaStreamWaitEvent(st, R.ev_direct, 0));
    if (R.nt > 0) {
      scatter_add_kernel<<<grid_for(R.nt, 256), 256, 0, st>>>(R.us.get(), R.ud.get(), T.tgt_perm.get(), R.nt, u);
      FGT_LAUNCHED();
    }
  } else {
    const double D0 = R.tp.D0;
    direct_lists(T, 1.0 / R.tp.delta, D0 * D0 * R.tp.delta, R.us.get(), &P.k_direct);
    if (R.nt > 0 && T.defer_order) {
      // a share of a large transform: zero u, then write the share's own targets only
      FGT_CUDA(cudaMemsetAsync(u, 0, R.nt * sizeof(double), st));
      if (T.n_dtgt > 0) {
        scatter_boxes_kernel<<<grid_for(T.n_dtgt, 8), 256, 0, st>>>(T.d_tgt_ids.get(), T.n_dtgt, T.tgt_start.get(),
                                                                    T.tgt_count.get(), R.us.get(), T.tgt_perm.get(), u);
        FGT_LAUNCHED();
      }
      if (T.n_psi > 0) {
        scatter_boxes_kernel<<<grid_for(T.n_psi, 8), 256, 0, st>>>(T.psi_ids.get(), T.n_psi, T.tgt_start.get(),
                                                                   T.tgt_count.get(), R.us.get(), T.tgt_perm.get(), u);
        FGT_LAUNCHED();
      }
    } else if (R.nt > 0) {
      scatter_kernel<<<grid_for(R.nt, 256), 256, 0, st>>>(R.us.get(), T.tgt_perm.get(), R.nt, u);
      FGT_LAUNCHED();
    }
  }
  R.pm->mark();
  trace_mark(st, "direct");
  fgt_phase_times t;
  std::memset(&t, 0, sizeof(t));
  if (u_host) {
    Timer tm(st);
    if (R.nt > 0) FGT_CUDA(cudaMemcpyAsync(u_host, u, R.nt * sizeof(double), cudaMemcpyDeviceToHost, st));
    t.d2h_ms = tm.lap();
  }
  PhaseMarks& pm = *R.pm;
  t.tree_ms = pm.ms(0);
  t.lists_ms = R.sb ? R.k_lists.ms() : pm.ms(1);  // overlapped: side-stream time
  t.form_ms = pm.ms(2);
  t.gather_ms = P.k_gather.ms();
  t.eval_ms = pm.ms(m_fin, m_fin + 1) - t.gather_ms;
  t.direct_ms = pm.ms(m_fin + 1, m_fin + 2);
  trace_dump();
  // device time on the launching stream: begin (tree, lists, form) + finish (the overlapped
  // lists are not on it; the exchange between begin and finish is not counted)
  t.total_ms = t.tree_ms + pm.ms(1) + t.form_ms + pm.ms(m_fin, m_fin + 2);
  t.launches = g_launches - R.l0;
  t.k_form_ms = P.k_form.ms();
  t.k_gather_ms = P.k_gather.ms();
  t.k_eval_ms = P.k_eval.ms();
  t.k_direct_ms = P.k_direct.ms();
  t.n_boxes = T.nb;
  t.n_dense = T.n_dense;
  t.n_psi = T.n_psi;
  t.n_src_dense = P.n_src_dense;
  t.n_tgt_psi = P.n_tgt_psi;
  t.n_p_entries = T.n_p;
  t.n_direct_pairs = direct_pairs(T);
  t.n_modes = P.NF;
  t.n_spread_boxes = P.n_spread_boxes;
  t.n_src_spread = P.n_src_spread;
  t.n_spread_psi = P.n_spread_psi;
  t.n_tgt_spread = P.n_tgt_spread;
  t.nufft_w = R.NP ? R.NP->w : 0;
  t.nufft_G = R.NP ? R.NP->G : 0;
  if (times) *times = t;
}

static void points_pipeline(const double* src, int64_t ns, const double* q, const double* tgt,
                            int64_t nt, const fgt_tree_params& tp, const fgt_pw_params& pw,
                            double* u, cudaStream_t st, fgt_phase_times* times,
                            cudaEvent_t q_ready = nullptr, double* u_host = nullptr) {
  PointsRun R;
  points_begin(R, src, ns, q, tgt, nt, tp, pw, st, false, q_ready);
  points_finish(R, u, times, u_host);
}

// ---------------------------------------------------------------- microbenchmarks
__global__ void fp64_dfma_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1e-10, a2 = a0 + 2e-10, a3 = a0 + 3e-10;
  double a4 = a0 + 4e-10, a5 = a0 + 5e-10, a6 = a0 + 6e-10, a7 = a0 + 7e-10;
  const double b = 0.999999, c = 1e-12;
  for (int i = 0; i < iters; ++i) {
    a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
    a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
  }
  double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 12345.0) out[0] = s;
}

__global__ void fp64_dmma_kernel(double* out, int iters) {
  double d[8][2];
  for (int i = 0; i < 8; ++i) d[i][0] = d[i][1] = 0.0;
  double a = threadIdx.x * 1e-6, b = 1.0 - threadIdx.x * 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d[t][0]), "+d"(d[t][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1];
  if (s == 12345.0) out[0] = s;
}

}  // namespace fgt

using namespace fgt;

extern "C" {

const char* fgt_last_error(void) { return g_last_error.c_str(); }
const char* fgt_version(void) { return "0.1.0+sm_100a"; }
int64_t fgt_launch_count(void) { return g_launches; }
void fgt_reset_launch_count(void) { g_launches = 0; }

int fgt_gauss_direct_dev(const double* tgt, int64_t nt, const double* src, int64_t ns,
                         const double* q, int d, double inv_delta, double r2_cut, int periodic,
                         double* out, void* stream) {
  return guarded([&] {
    FGT_REQUIRE(d >= 1 && d <= 3, FGT_EINVAL, "dim must be 1, 2, or 3");
    FGT_REQUIRE(nt >= 0 && ns >= 0, FGT_EINVAL, "negative size");
    launch_gauss_direct_allpairs(tgt, nt, src, ns, q, d, inv_delta, r2_cut, periodic != 0, out,
                                 (cudaStream_t)stream);
  });
}

int fgt_gauss_direct(const double* tgt, int64_t nt, const double* src, int64_t ns,
                     const double* q, int d, double inv_delta, double r2_cut, int periodic,
                     double* out) {
  return guarded([&] {
    FGT_REQUIRE(d >= 1 && d <= 3, FGT_EINVAL, "dim must be 1, 2, or 3");
    FGT_REQUIRE(nt >= 0 && ns >= 0, FGT_EINVAL, "negative size");
    if (nt == 0) return;
    OwnedStream os;
    DBuf<double> dt(nt * d, os.s), ds(ns * d, os.s), dq(ns, os.s), dout(nt, os.s);
    dt.from_host(tgt, nt * d);
    ds.from_host(src, ns * d);
    dq.from_host(q, ns);
    dout.from_host(out, nt);
    launch_gauss_direct_allpairs(dt.get(), nt, ds.get(), ns, dq.get(), d, inv_delta, r2_cut,
                                 periodic != 0, dout.get(), os.s);
    dout.to_host(out, nt);
    FGT_CUDA(cudaStreamSynchronize(os.s));
  });
}

int fgt_nufft_spread_dev(const double* x, int64_t M, int d, const double* vals, int64_t n_r,
                         int m_sp, double tau, double* grid, void* stream) {
  return guarded([&] {
    FGT_REQUIRE(d >= 1 && d <= 3, FGT_EINVAL, "dim must be 1, 2, or 3");
    FGT_REQUIRE(n_r >= 1 && m_sp >= 0 && tau > 0, FGT_EINVAL, "bad spreading parameters");
    launch_nufft_spread(x, M, d, vals, n_r, m_sp, tau, grid, (cudaStream_t)stream);
  });
}

int fgt_nufft_spread(const double* x, int64_t M, int d, const double* vals, int64_t n_r, int m_sp,
                     double tau, double* grid) {
  return guarded([&] {
    FGT_REQUIRE(d >= 1 && d <= 3, FGT_EINVAL, "dim must be 1, 2, or 3");
    FGT_REQUIRE(n_r >= 1 && m_sp >= 0 && tau > 0, FGT_EINVAL, "bad spreading parameters");
    int64_t ng = 1;
    for (int k = 0; k < d; ++k) ng *= n_r;
    OwnedStream os;
    DBuf<double> dx(M * d, os.s), dv(2 * M, os.s), dg(2 * ng, os.s);
    dx.from_host(x, M * d);
    dv.from_host(vals, 2 * M);
    dg.from_host(grid, 2 * ng);
    launch_nufft_spread(dx.get(), M, d, dv.get(), n_r, m_sp, tau, dg.get(), os.s);
    dg.to_host(grid, 2 * ng);
    FGT_CUDA(cudaStreamSynchronize(os.s));
  });
}

int fgt_nufft_interp_dev(const double* x, int64_t M, int d, const double* grid, int64_t n_r,
                         int m_sp, double tau, double* out, void* stream) {
  return guarded([&] {
    FGT_REQUIRE(d >= 1 && d <= 3, FGT_EINVAL, "dim must be 1, 2, or 3");
    FGT_REQUIRE(n_r >= 1 && m_sp >= 0 && tau > 0, FGT_EINVAL, "bad spreading parameters");
    launch_nufft_interp(x, M, d, grid, n_r, m_sp, tau, out, (cudaStream_t)stream);
  });
}

int fgt_nufft_interp(const double* x, int64_t M, int d, const double* grid, int64_t n_r, int m_sp,
                     double tau, double* out) {
  return guarded([&] {
    FGT_REQUIRE(d >= 1 && d <= 3, FGT_EINVAL, "dim must be 1, 2, or 3");
    FGT_REQUIRE(n_r >= 1 && m_sp >= 0 && tau > 0, FGT_EINVAL, "bad spreading parameters");
    if (M == 0) return;
    int64_t ng = 1;
    for (int k = 0; k < d; ++k) ng *= n_r;
    OwnedStream os;
    DBuf<double> dx(M * d, os.s), dg(2 * ng, os.s), dout(2 * M, os.s);
    dx.from_host(x, M * d);
    dg.from_host(grid, 2 * ng);
    launch_nufft_interp(dx.get(), M, d, dg.get(), n_r, m_sp, tau, dout.get(), os.s);
    dout.to_host(out, 2 * M);
    FGT_CUDA(cudaStreamSynchronize(os.s));
  });
}

struct fgt_tree {
  TreeDev T;
};

int fgt_tree_build_dev(const double* src, int64_t ns, const double* tgt, int64_t nt,
                       const fgt_tree_params* prm, void* stream, fgt_tree** out) {
  return guarded([&] {
    FGT_REQUIRE(prm && out, FGT_EINVAL, "null argument");
    auto t = std::make_unique<fgt_tree>();
    build_tree(t->T, src, ns, tgt, nt, *prm, (cudaStream_t)stream);
    FGT_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    *out = t.release();
  });
}

int fgt_tree_get_info(const fgt_tree* t, fgt_tree_info* info) {
  return guarded([&] {
    FGT_REQUIRE(t && info, FGT_EINVAL, "null argument");
    const TreeDev& T = t->T;
    std::memset(info, 0, sizeof(*info));
    info->dim = T.d;
    info->l_c = T.l_c;
    info->n_levels = T.n_levels;
    info->periodic = T.periodic;
    info->n_boxes = T.nb;
    info->n_leaves = T.n_leaves;
    info->n_dense = T.n_dense;
    info->n_sources = T.ns;
    info->n_targets = T.nt;
    for (int k = 0; k < 3; ++k) info->root_center[k] = T.root_center[k];
    info->root_side = T.root_side;
  });
}

int fgt_tree_copy_out(const fgt_tree* t, int64_t* level, int64_t* parent, int64_t* children,
                      int64_t* coords, uint8_t* is_leaf, int64_t* src_perm, int64_t* tgt_perm,
                      int64_t* src_start, int64_t* src_count, int64_t* tgt_start,
                      int64_t* tgt_count, int64_t* n_points) {
  return guarded([&] {
    FGT_REQUIRE(t, FGT_EINVAL, "null tree");
    const TreeDev& T = t->T;
    cudaStream_t st = T.st;
    const int64_t nb = T.nb;
    if (level) {
      std::vector<int32_t> l32(nb);
      T.level.to_host(l32.data(), nb);
      FGT_CUDA(cudaStreamSynchronize(st));
      for (int64_t i = 0; i < nb; ++i) level[i] = l32[i];
    }
    if (parent) T.parent.to_host(parent, nb);
    if (children) T.children.to_host(children, nb << T.d);
    if (coords) T.coords.to_host(coords, nb * T.d);
    if (is_leaf) T.is_leaf.to_host(is_leaf, nb);
    if (src_perm) T.src_perm.to_host(src_perm, T.ns);
    if (tgt_perm) T.tgt_perm.to_host(tgt_perm, T.nt);
    if (src_start) T.src_start.to_host(src_start, nb);
    if (src_count) T.src_count.to_host(src_count, nb);
    if (tgt_start) T.tgt_start.to_host(tgt_start, nb);
    if (tgt_count) T.tgt_count.to_host(tgt_count, nb);
    if (n_points) T.n_points.to_host(n_points, nb);
    FGT_CUDA(cudaStreamSynchronize(st));
  });
}

int fgt_tree_lists(fgt_tree* t, fgt_list_info* info) {
  return guarded([&] {
    FGT_REQUIRE(t, FGT_EINVAL, "null tree");
    build_lists(t->T);
    FGT_CUDA(cudaStreamSynchronize(t->T.st));
    if (info) {
      info->n_p_entries = t->T.n_p;
      info->n_d_entries = t->T.n_d;
      info->n_psi_boxes = t->T.n_psi;
      info->n_direct_pairs = direct_pairs(t->T);
    }
  });
}

int fgt_tree_copy_lists(const fgt_tree* t, int64_t* p_tgt, int64_t* p_src, int64_t* p_v,
                        int64_t* d_tgt, int64_t* d_src, int64_t* d_v) {
  return guarded([&] {
    FGT_REQUIRE(t && t->T.lists_built, FGT_EINVAL, "lists not built");
    const TreeDev& T = t->T;
    cudaStream_t st = T.st;
    const int d = T.d;
    std::vector<int64_t> slot(T.n_p), dense(T.n_dense);
    std::vector<int32_t> pv(T.n_p * d), dv(T.n_d * d);
    T.p_src.to_host(slot.data(), T.n_p);
    T.dense_ids.to_host(dense.data(), T.n_dense);
    T.p_v.to_host(pv.data(), T.n_p * d);
    T.d_v.to_host(dv.data(), T.n_d * d);
    if (p_tgt) T.p_tgt.to_host(p_tgt, T.n_p);
    if (d_tgt) T.d_tgt.to_host(d_tgt, T.n_d);
    if (d_src) T.d_src.to_host(d_src, T.n_d);
    FGT_CUDA(cudaStreamSynchronize(st));
    if (p_src)
      for (int64_t i = 0; i < T.n_p; ++i) p_src[i] = dense[slot[i]];
    if (p_v)
      for (int64_t i = 0; i < T.n_p * d; ++i) p_v[i] = pv[i];
    if (d_v)
      for (int64_t i = 0; i < T.n_d * d; ++i) d_v[i] = dv[i];
  });
}

void fgt_tree_free(fgt_tree* t) {
  if (t) {
    cudaStreamSynchronize(t->T.st);
    delete t;
  }
}

int fgt_points_dev(const double* src, int64_t ns, const double* charges, const double* tgt,
                   int64_t nt, const fgt_tree_params* tp, const fgt_pw_params* pw, double* u,
                   void* stream, fgt_phase_times* times) {
  return guarded([&] {
    FGT_REQUIRE(tp && pw, FGT_EINVAL, "null parameters");
    points_pipeline(src, ns, charges, tgt, nt, *tp, *pw, u, (cudaStream_t)stream, times);
  });
}

struct fgt_points_run {
  PointsRun R;
};

int fgt_points_begin(const double* src, int64_t ns, const double* charges, const double* tgt,
                     int64_t nt, const fgt_tree_params* tp, const fgt_pw_params* pw, void* stream,
                     fgt_points_run** out) {
  return guarded([&] {
    FGT_REQUIRE(tp && pw && out, FGT_EINVAL, "null argument");
    auto r = std::make_unique<fgt_points_run>();
    points_begin(r->R, src, ns, charges, tgt, nt, *tp, *pw, (cudaStream_t)stream, true);
    *out = r.release();
  });
}

int fgt_points_exchange_counts(const fgt_points_run* r, int64_t* send_slots, int64_t* recv_slots,
                               int64_t* slot_doubles) {
  return guarded([&] {
    FGT_REQUIRE(r, FGT_EINVAL, "null run");
    const ExchangePlan& X = r->R.X;
    for (int p = 0; p < X.world; ++p) {
      if (send_slots) send_slots[p] = X.send_off.empty() ? 0 : X.send_off[p + 1] - X.send_off[p];
      if (recv_slots) recv_slots[p] = X.recv_off.empty() ? 0 : X.recv_off[p + 1] - X.recv_off[p];
    }
    if (slot_doubles) *slot_doubles = 2 * r->R.P.NH;
  });
}

int fgt_points_pack(fgt_points_run* r, double* send_buf) {
  return guarded([&] {
    FGT_REQUIRE(r, FGT_EINVAL, "null run");
    PointsRun& R = r->R;
    const int64_t n = R.X.send_slots.size();
    if (n == 0) return;
    pack_slots_kernel<<<grid_for(n * R.P.NH, 256), 256, 0, R.st>>>(
        reinterpret_cast<const double2*>(R.P.phi.get()), R.X.send_slots.get(), n, R.P.NH,
        reinterpret_cast<double2*>(send_buf));
    FGT_LAUNCHED();
  });
}

int fgt_points_unpack(fgt_points_run* r, const double* recv_buf) {
  return guarded([&] {
    FGT_REQUIRE(r, FGT_EINVAL, "null run");
    PointsRun& R = r->R;
    const int64_t n = R.X.recv_slots.size();
    if (n == 0) return;
    unpack_slots_kernel<<<grid_for(n * R.P.NH, 256), 256, 0, R.st>>>(
        reinterpret_cast<double2*>(R.P.phi.get()), R.X.recv_slots.get(), n, R.P.NH,
        reinterpret_cast<const double2*>(recv_buf));
    FGT_LAUNCHED();
  });
}

int fgt_points_finish(fgt_points_run* r, double* u, fgt_phase_times* times) {
  return guarded([&] {
    FGT_REQUIRE(r, FGT_EINVAL, "null run");
    points_finish(r->R, u, times);
  });
}

void fgt_points_run_free(fgt_points_run* r) {
  if (r) {
    cudaStreamSynchronize(r->R.st);
    delete r;
  }
}

int fgt_points(const double* src, int64_t ns, const double* charges, const double* tgt, int64_t nt,
               const fgt_tree_params* tp, const fgt_pw_params* pw, double* u,
               fgt_phase_times* times) {
  return guarded([&] {
    FGT_REQUIRE(tp && pw, FGT_EINVAL, "null parameters");
    const int d = tp->dim;
    HostStreams& os = host_streams();
    Timer tm(os.s);
    DBuf<double> ds(ns * d, os.s), dq(ns, os.s), dt(nt * d, os.s), du(nt, os.s);
    // coordinates first (the tree needs all of them); the charges follow on a side stream
    // and land while the tree is built (gather_sorted_points waits for them).  The copy
    // is timed by events read after the pipeline: no host wait between the copy and the
    // tree's first kernels.
    Event q_alloc, q_ready;
    FGT_CUDA(cudaEventRecord(q_alloc.e, os.s));
    ds.from_host(src, ns * d);
    dt.from_host(tgt, nt * d);
    FGT_CUDA(cudaEventRecord(tm.b, os.s));
    FGT_CUDA(cudaStreamWaitEvent(os.side, q_alloc.e, 0));
    if (ns > 0) FGT_CUDA(cudaMemcpyAsync(dq.get(), charges, ns * sizeof(double), cudaMemcpyHostToDevice, os.side));
    FGT_CUDA(cudaEventRecord(q_ready.e, os.side));
    fgt_phase_times t;
    std::memset(&t, 0, sizeof(t));
    points_pipeline(ds.get(), ns, dq.get(), dt.get(), nt, *tp, *pw, du.get(), os.s, &t, q_ready.e, u);
    FGT_CUDA(cudaStreamSynchronize(os.s));  // (points_finish timed the copy: u is on the host)
    float h2d = 0.f;
    FGT_CUDA(cudaEventElapsedTime(&h2d, tm.a, tm.b));
    t.h2d_ms = h2d;
    if (times) *times = t;
  });
}

int fgt_box_dev(const fgt_box_plan* plan, const double* values, double* u, void* stream,
                fgt_phase_times* times) {
  return guarded([&] {
    FGT_REQUIRE(plan, FGT_EINVAL, "null plan");
    const int64_t l0 = g_launches;
    fgt_phase_times t;
    std::memset(&t, 0, sizeof(t));
    box_fgt(*plan, values, u, (cudaStream_t)stream, &t);
    t.launches = g_launches - l0;
    if (times) *times = t;
  });
}

int fgt_box_interp_dev(const fgt_interp_tree* t, const double* x, int64_t n, double* out, void* stream) {
  return guarded([&] {
    FGT_REQUIRE(t, FGT_EINVAL, "null tree");
    box_interp(*t, x, n, out, (cudaStream_t)stream);
  });
}

int fgt_box_interp(const fgt_interp_tree* t, const double* x, int64_t n, double* out) {
  return guarded([&] {
    FGT_REQUIRE(t, FGT_EINVAL, "null tree");
    OwnedStream os;
    DBuf<double> dx(n * t->dim, os.s), dout(n, os.s);
    dx.from_host(x, n * t->dim);
    box_interp(*t, dx.get(), n, dout.get(), os.s);
    dout.to_host(out, n);
    FGT_CUDA(cudaStreamSynchronize(os.s));
  });
}

int fgt_box(const fgt_box_plan* plan, const double* values, double* u, fgt_phase_times* times) {
  return guarded([&] {
    FGT_REQUIRE(plan, FGT_EINVAL, "null plan");
    int64_t kd = 1;
    for (int i = 0; i < plan->dim; ++i) kd *= plan->k;
    const int64_t n = plan->n_leaves * kd;
    OwnedStream os;
    Timer tm(os.s);
    DBuf<double> dv(n, os.s), du(n, os.s);
    dv.from_host(values, n);
    const double h2d = tm.lap();
    const int64_t l0 = g_launches;
    fgt_phase_times t;
    std::memset(&t, 0, sizeof(t));
    box_fgt(*plan, dv.get(), du.get(), os.s, &t);
    t.launches = g_launches - l0;
    tm.lap();
    du.to_host(u, n);
    FGT_CUDA(cudaStreamSynchronize(os.s));
    t.h2d_ms = h2d;
    t.d2h_ms = tm.lap();
    if (times) *times = t;
  });
}

// ---- Alg 3 / 5 / 6 on the device: tail test, grid nodes, level restriction, retained psi
int fgt_box_tail_dev(const double* values, int64_t n, int dim, int k, const double* val_to_pol,
                     const double* weights, double* tail, double* wsq, void* stream) {
  return guarded([&] {
    FGT_REQUIRE(n >= 0 && (n == 0 || (values && tail)) && val_to_pol && weights, FGT_EINVAL, "bad arguments");
    FGT_REQUIRE(k >= 2 && k <= 24, FGT_ERANGE, "polynomial order outside [2, 24]");
    cudaStream_t st = (cudaStream_t)stream;
    DBuf<double> m((size_t)k * k, st), w((size_t)k, st);
    m.from_host(val_to_pol, (size_t)k * k);
    w.from_host(weights, (size_t)k);
    box_tail(values, n, dim, k, m.get(), w.get(), tail, wsq, st);
    FGT_CUDA(cudaStreamSynchronize(st));  // the host tables may go out of scope
  });
}

int fgt_box_tail(const double* values, int64_t n, int dim, int k, const double* val_to_pol,
                 const double* weights, double* tail, double* wsq) {
  return guarded([&] {
    FGT_REQUIRE(n >= 0 && (n == 0 || (values && tail)) && val_to_pol && weights, FGT_EINVAL, "bad arguments");
    FGT_REQUIRE(dim >= 1 && dim <= 3, FGT_EINVAL, "dim must be 1, 2, or 3");
    FGT_REQUIRE(k >= 2 && k <= 24, FGT_ERANGE, "polynomial order outside [2, 24]");
    int64_t kd = 1;
    for (int i = 0; i < dim; ++i) kd *= k;
    OwnedStream os;
    DBuf<double> dv(n * kd, os.s), dt(n, os.s), dw(n, os.s), m((size_t)k * k, os.s), w((size_t)k, os.s);
    dv.from_host(values, n * kd);
    m.from_host(val_to_pol, (size_t)k * k);
    w.from_host(weights, (size_t)k);
    box_tail(dv.get(), n, dim, k, m.get(), w.get(), dt.get(), dw.get(), os.s);
    dt.to_host(tail, n);
    if (wsq) dw.to_host(wsq, n);
    FGT_CUDA(cudaStreamSynchronize(os.s));
  });
}

int fgt_box_nodes_dev(const int32_t* level, const int64_t* coords, int64_t n, int dim, int k,
                      const double* nodes, const double* root_low, double root_side, double* pts,
                      void* stream) {
  return guarded([&] {
    FGT_REQUIRE(n >= 0 && (n == 0 || (level && coords && pts)) && nodes && root_low, FGT_EINVAL, "bad arguments");
    FGT_REQUIRE(dim >= 1 && dim <= 3, FGT_EINVAL, "dim must be 1, 2, or 3");
    FGT_REQUIRE(k >= 1 && k <= 64, FGT_ERANGE, "grid order out of range");
    for (int64_t i = 0; i < n; ++i) FGT_REQUIRE(level[i] >= 0 && level[i] <= 57 / dim, FGT_ERANGE, "level out of range");
    cudaStream_t st = (cudaStream_t)stream;
    DBuf<int32_t> dl(n, st);
    DBuf<int64_t> dc(n * dim, st);
    DBuf<double> dn((size_t)k, st);
    dl.from_host(level, n);
    dc.from_host(coords, n * dim);
    dn.from_host(nodes, (size_t)k);
    box_nodes(dl.get(), dc.get(), n, dim, k, dn.get(), root_low, root_side, pts, st);
    FGT_CUDA(cudaStreamSynchronize(st));
  });
}

int fgt_box_balance_flags(const int32_t* level, const int64_t* coords, const uint8_t* is_leaf,
                          int64_t n, int dim, int periodic, uint8_t* flags) {
  return guarded([&] {
    FGT_REQUIRE(n >= 0 && (n == 0 || (level && coords && is_leaf && flags)), FGT_EINVAL, "bad arguments");
    FGT_REQUIRE(dim >= 1 && dim <= 3, FGT_EINVAL, "dim must be 1, 2, or 3");
    // sorted (level, Morton) keys of the box set; flags come back in the caller's order
    std::vector<std::pair<uint64_t, int64_t>> kv(n);
    for (int64_t i = 0; i < n; ++i) {
      FGT_REQUIRE(level[i] >= 0 && level[i] * dim <= 57, FGT_ERANGE, "level out of range");
      kv[i] = {box_key(level[i], morton_encode(coords + i * dim, dim, level[i])), i};
    }
    std::sort(kv.begin(), kv.end());
    std::vector<uint64_t> hk(n);
    std::vector<uint8_t> hl(n), hf(n);
    for (int64_t i = 0; i < n; ++i) {
      hk[i] = kv[i].first;
      hl[i] = is_leaf[kv[i].second];
      FGT_REQUIRE(i == 0 || hk[i] != hk[i - 1], FGT_EINVAL, "duplicate box");
    }
    OwnedStream os;
    DBuf<uint64_t> dk(n, os.s);
    DBuf<uint8_t> dl(n, os.s), df(n, os.s);
    dk.from_host(hk.data(), n);
    dl.from_host(hl.data(), n);
    box_balance_flags(dk.get(), dl.get(), n, dim, periodic, df.get(), os.s);
    df.to_host(hf.data(), n);
    FGT_CUDA(cudaStreamSynchronize(os.s));
    for (int64_t i = 0; i < n; ++i) flags[kv[i].second] = hf[i];
  });
}

struct fgt_box_state {
  OwnedStream os;
  BoxState st;
};

int fgt_box_retain(const fgt_box_plan* plan, const double* values, double* u, fgt_phase_times* times,
                   fgt_box_state** state) {
  return guarded([&] {
    FGT_REQUIRE(plan && state && values && u, FGT_EINVAL, "null argument");
    int64_t kd = 1;
    for (int i = 0; i < plan->dim; ++i) kd *= plan->k;
    const int64_t n = plan->n_leaves * kd;
    std::unique_ptr<fgt_box_state> s(new fgt_box_state);
    cudaStream_t st = s->os.s;
    s->st.st = st;
    s->st.values.alloc(n, st);
    s->st.n_values = plan->n_leaves;
    s->st.values.from_host(values, n);
    DBuf<double> du(n, st);
    const int64_t l0 = g_launches;
    fgt_phase_times t;
    std::memset(&t, 0, sizeof(t));
    box_fgt(*plan, s->st.values.get(), du.get(), st, &t, &s->st, nullptr);
    t.launches = g_launches - l0;
    du.to_host(u, n);
    FGT_CUDA(cudaStreamSynchronize(st));
    du.release();
    if (times) *times = t;
    *state = s.release();
  });
}

int fgt_box_refine(fgt_box_state* state, const fgt_box_plan* rplan, double* u_new,
                   fgt_phase_times* times) {
  return guarded([&] {
    FGT_REQUIRE(state && rplan && (rplan->n_leaves == 0 || u_new), FGT_EINVAL, "null argument");
    cudaStream_t st = state->os.s;
    for (int64_t p = 0; p < rplan->n_dpairs; ++p)
      FGT_REQUIRE(rplan->d_src[p] >= 0 && rplan->d_src[p] < state->st.n_values, FGT_EINVAL,
                  "direct source outside the retained leaf grids");
    const int64_t n = rplan->n_leaves * state->st.KD;
    DBuf<double> du(std::max<int64_t>(n, 1), st);
    const int64_t l0 = g_launches;
    fgt_phase_times t;
    std::memset(&t, 0, sizeof(t));
    box_fgt(*rplan, state->st.values.get(), du.get(), st, &t, nullptr, &state->st);
    t.launches = g_launches - l0;
    du.to_host(u_new, n);
    FGT_CUDA(cudaStreamSynchronize(st));
    du.release();
    if (times) *times = t;
  });
}

int fgt_box_state_free(fgt_box_state* state) {
  return guarded([&] {
    if (!state) return;
    state->st.psi.release();
    state->st.values.release();
    delete state;
  });
}

int fgt_partition_bounds(const double* cost, int64_t n, int32_t parts, int64_t* bounds) {
  return guarded([&] {
    FGT_REQUIRE(parts >= 1 && n >= 0 && (n == 0 || cost) && bounds, FGT_EINVAL, "bad arguments");
    std::vector<double> c(cost, cost + n);
    for (double v : c) FGT_REQUIRE(v >= 0, FGT_EINVAL, "negative cost");
    std::vector<int64_t> b = partition_bounds(c, parts);
    for (int r = 0; r <= parts; ++r) bounds[r] = b[r];
  });
}

int fgt_bench_fp64_peak(int use_dmma, double* tflops) {
  return guarded([&] {
    OwnedStream os;
    DBuf<double> out(1, os.s);
    int dev = 0, nsm = 0;
    FGT_CUDA(cudaGetDevice(&dev));
    FGT_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    const int block = 256, grid = nsm * 8;
    const int iters = use_dmma ? 4096 : 16384;
    for (int rep = 0; rep < 2; ++rep) {
      Timer tm(os.s);
      if (use_dmma) fp64_dmma_kernel<<<grid, block, 0, os.s>>>(out.get(), iters);
      else fp64_dfma_kernel<<<grid, block, 0, os.s>>>(out.get(), iters);
      FGT_LAUNCHED();
      double ms = tm.lap();
      double flops = use_dmma ? (double)grid * (block / 32) * iters * 8 * 256 * 2
                              : (double)grid * block * iters * 8 * 2;
      *tflops = flops / (ms * 1e-3) / 1e12;
    }
  });
}

}  // extern "C"
