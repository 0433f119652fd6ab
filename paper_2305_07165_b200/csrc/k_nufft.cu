// Box-local NUFFT (spread / separable DFT / interpolate) for heavy P-boxes and psi boxes.
//
// The reference forms phi with nufft_type1 (nufft.py:139-162: Gaussian spreading onto a
// periodic 2x grid, radix-2/3/5 FFT, bin selection, deconvolution) and evaluates psi
// with nufft_type2 (nufft.py:165-183).  On B200 the same transform is organised as:
//   1. spreading with the exponential-of-semicircle kernel (w taps/axis instead of the
//      reference Gaussian's 2w+1) into a NON-periodic grid that covers only the box
//      (2X/Delta + w cells per axis), held in shared-memory plane slabs in which every
//      warp owns whole planes: plain read-modify-write, no atomics;
//   2. the grid -> mode map as d separable complex GEMMs on the FP64 tensor cores
//      (mma.sync m8n8k4 .f64) with the deconvolution 1/fh(m) and the plane-wave weights
//      folded into the 1-D matrices, written straight into phi (no FFT, no bin gather:
//      only n_f of the 2 n_f modes are ever needed);
//   3. evaluation runs the transposed chain and interpolates with the same kernel.
// Partial grids of K-split boxes are summed in a fixed order (deterministic).
#include <algorithm>
#include <cmath>
#include <string>
#include <mutex>
#include <map>
#include <cstdlib>
#include <cstring>

#include <cub/cub.cuh>

#include "k_gemm.cuh"
#include "k_nufft.cuh"

namespace fgt {

namespace {

struct CubTmpBuf {
  DBuf<uint8_t> buf;
  void* get(size_t bytes, cudaStream_t st) {
    if (bytes > buf.size()) buf.alloc(bytes + 256, st);
    return buf.get();
  }
};

__global__ void iota_i64_kernel(int64_t* a, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    a[i] = i;
}

void iota_i64(int64_t* a, int64_t n, cudaStream_t st) {
  if (n == 0) return;
  iota_i64_kernel<<<grid_for(n, 256), 256, 0, st>>>(a, n);
  FGT_LAUNCHED();
}

template <class K>
void sort_pairs_key(CubTmpBuf& tmp, const K* kin, K* kout, const int64_t* vin,
                    int64_t* vout, int64_t n, int bits, cudaStream_t st) {
  if (n == 0) return;
  size_t bytes = 0;
  FGT_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kin, kout, vin, vout, (int)n, 0, bits, st));
  FGT_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(bytes, st), bytes, kin, kout, vin, vout, (int)n, 0, bits, st));
  count_launch();
}


__host__ __device__ __forceinline__ double es_kernel(double z, double beta) {
  double s = 1.0 - z * z;
  return s > 0.0 ? exp(beta * (sqrt(s) - 1.0)) : 0.0;
}

constexpr int MAXW = 16;
constexpr int PROXY_PMAX = 48;  // proxy-point form: Chebyshev nodes per axis

// ------------------------------------------------------------------ spreading
// Pass 1 (one thread per point): first tap a_k (0-based grid index) and the w kernel
// weights of every axis, computed once, plus a sort key.  Pass 2: points sorted by the
// key, so every job's points form one contiguous range:
//   d = 3: key (box, a_0, a_1); job = (box, grid plane p), points with a_0 in [p-w+1, p];
//   d = 2: key (box, a_0);      job = (box), the whole G x G grid;
//   d = 1: key (box, a_0);      job = (box, cell p).
// Pass 3 (d = 2, 3) spreads on the FP64 tensor cores: a point's contribution to a plane
// is the rank-1 update c w1 (x) w2, so four points make one m8n8k4 DMMA per 8 x 8 tile;
// one warp keeps its whole plane (NB x NB tiles) in registers -- no shared-memory
// read-modify-write, no atomics.  Per group of 4 points only the tiles their taps touch
// are issued (warp-uniform predicates).
struct WeightArgs {
  const double* src;
  const double* q;
  const double* center;
  const int64_t* dense_ids;
  const int64_t* src_start;
  const int64_t* slots;  // batch box -> dense slot
  const int64_t* boff;   // (nbat+1) point offsets of the batch boxes
  int64_t npts, nbat;
  double* wts;           // (npts, MAXW), d = 1 only
  double* tt;            // (npts, D) coordinates in grid units
  int* ai;               // (npts, D)
  double* qb;            // (npts)
  uint64_t* key;         // (npts)
  double sc, inv_delta, beta;
  int w, gmin, G;
};

// Pass 1, one thread per (point, axis): the scaled coordinate tt (grid units) and the
// first tap a_k; no kernel weights yet (d >= 2 evaluates them after the sort, directly in
// sorted order; d = 1 evaluates them here for the line kernel).
template <int D>
__global__ void __launch_bounds__(256) spread_taps_kernel(WeightArgs a) {
  const double s = a.sc * a.inv_delta, half = 0.5 * a.w, inv_half = 2.0 / a.w;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < a.npts * D;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / D;
    const int k = (int)(t - i * D);
    int64_t lo = 0, hi = a.nbat;  // batch box of point i
    while (hi - lo > 1) {
      int64_t mid = (lo + hi) >> 1;
      if (a.boff[mid] <= i) lo = mid; else hi = mid;
    }
    const int64_t box = a.dense_ids[a.slots[lo]];
    const int64_t sidx = a.src_start[box] + (i - a.boff[lo]);
    const double tt = (a.src[sidx * D + k] - a.center[box * D + k]) * s;
    const double a0 = ceil(tt - half);
    a.tt[i * D + k] = tt;
    a.ai[i * D + k] = max(0, min((int)a0 - a.gmin, a.G - a.w));
    if (D == 1) {
      double* wp = a.wts + i * MAXW;
#pragma unroll
      for (int o = 0; o < MAXW; ++o) wp[o] = o < a.w ? es_kernel((a0 + o - tt) * inv_half, a.beta) : 0.0;
    }
    if (k == 0) {
      a.qb[i] = a.q[sidx];
      a.key[i] = (uint64_t)lo;  // box part; spread_keys_kernel adds the taps
    }
  }
}

// interleave two 8-bit values (x in the odd bits)
__device__ __forceinline__ uint64_t morton2_8(unsigned x, unsigned y) {
  uint64_t r = 0;
#pragma unroll
  for (int b = 0; b < 8; ++b) r |= (uint64_t)(((x >> b) & 1u) << (2 * b + 1)) | (uint64_t)(((y >> b) & 1u) << (2 * b));
  return r;
}

// key = (box, a_0, Morton(a_1, a_2)) for d = 3, (box, Morton(a_0, a_1)) for d = 2 (16 bits
// for the last two taps), (box, a_0) for d = 1: a plane job is one key range (a_0 major) and
// consecutive points are spatially compact, so a 4-point DMMA group touches few tiles
// d = 3 row class of a first tap: 8-row blocks cut at a = 0 and a = 1 - w (mod 8), so the
// taps [a, a + w) touch row block b exactly for the classes [cls(8b - w + 1), cls(8b + 7)]
__host__ __device__ __forceinline__ int row_class(int a, int w) {
  const int r = ((1 - w) % 8 + 8) % 8;
  return 2 * (a >> 3) + ((a & 7) >= r ? 1 : 0);
}

// d = 3 key (box, row class of a_1, a_0, a_2) in 16 tap bits (G <= 64): a pencil's row
// range is one key range
template <int D>
__global__ void spread_keys_kernel(uint64_t* __restrict__ key, const int* __restrict__ ai, int64_t n, int w) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k = key[i];
    if (D == 1) k = (k << 8) | (uint64_t)ai[i];
    if (D == 2) k = (k << 16) | morton2_8((unsigned)ai[i * 2], (unsigned)ai[i * 2 + 1]);
    if (D == 3)
      k = (k << 16) | ((uint64_t)row_class(ai[i * 3 + 1], w) << 12) | ((uint64_t)ai[i * 3] << 6) |
          (uint64_t)ai[i * 3 + 2];  // G <= 64: taps < 64, classes < 16
    key[i] = k;
  }
}

// job ranges in the sorted keys: d = 3 per (box, row block), d = 1 per (box, cell), d = 2
// per box
template <int D>
__global__ void job_ranges_kernel(const uint64_t* __restrict__ key, int64_t npts, int64_t nbat, int G,
                                  int w, int* __restrict__ range) {
  const int NB = (G + 7) / 8;
  const int64_t njob = D == 2 ? nbat : (D == 3 ? nbat * NB : nbat * G);
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < njob;
       t += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k0, k1;
    if (D == 2) {
      k0 = (uint64_t)t << 16;
      k1 = (uint64_t)(t + 1) << 16;
    } else if (D == 3) {
      const uint64_t bx = (uint64_t)(t / NB);
      const int b = (int)(t % NB);
      const int clo = row_class(max(0, 8 * b - w + 1), w), chi = row_class(8 * b + 7, w);
      k0 = (bx << 16) | ((uint64_t)clo << 12);
      k1 = (bx << 16) + ((uint64_t)(chi + 1) << 12);  // chi + 1 may be 16: the next box
    } else {
      const uint64_t b = (uint64_t)(t / G), p = (uint64_t)(t % G);
      const uint64_t plo = (uint64_t)max(0, (int)p - w + 1);
      const int sh = 8 * (D - 1);  // bits below the a_0 byte
      k0 = (((b << 8) | plo) << sh);
      k1 = (((b << 8) | (p + 1)) << sh);
    }
    range[2 * t] = (int)lower_bound_dev(key, npts, k0);
    range[2 * t + 1] = (int)lower_bound_dev(key, npts, k1);
  }
}

// Sorted point records for the spreading kernels, one gather after the sort so every job's
// staging is a contiguous, coalesced copy instead of a perm -> index -> weights chase:
//   d = 2: rw (n, 32) = [axis-0 weights | axis-1 weights], rq (n) charge;
//   d = 3: rw (n, 48) = [q x axis-1 weights | axis-2 weights | axis-0 weights];
// ra (n, 4) = first taps (a_0, a_1, a_2).
// Block = 32 sorted points; warp a evaluates axis a (lane = point).  Interior taps by the
// plan's Horner polynomials (16 independent accumulators), the two edge taps -- where the
// kernel has its square-root branch point -- exactly; then each warp writes its 32 x 16
// weights through shared memory as 128-byte rows.
constexpr int REC_PTS = 32;
constexpr int PEN_REC = 48;  // d = 3 record: [q w1 | w2 | w0], 16 zero-padded taps each
constexpr int HC_MAX = 25;  // max polynomial degree + 1
template <int D, int W>  // W: kernel width (taps evaluated; the rest of the 16 are zero)
__global__ void __launch_bounds__(D * 32) sort_records_kernel(
    const int64_t* __restrict__ perm, int64_t n, const double* __restrict__ tt, const int* __restrict__ ai,
    const double* __restrict__ qb, double beta, const double* __restrict__ hc, int K,
    double* __restrict__ rw, double* __restrict__ rq, int* __restrict__ ra, double* __restrict__ rw0) {
  __shared__ double s_c[HC_MAX * 16];
  __shared__ double s_w[D][REC_PTS][17];
  for (int i = threadIdx.x; i < (K + 1) * 16; i += blockDim.x) s_c[i] = hc[i];
  __syncthreads();
  const int ax = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t j0 = (int64_t)blockIdx.x * REC_PTS, j = j0 + lane;
  constexpr int w = W;
  const double half = 0.5 * w, inv_half = 2.0 / w;
  if (j < n) {
    const int64_t i = perm[j];
    const double x = tt[i * D + ax];
    const double a0 = ceil(x - half);
    const double y = 2.0 * ((a0 - x) + half) - 1.0;
    double acc[W];
#pragma unroll
    for (int t = 0; t < W; ++t) acc[t] = s_c[K * 16 + t];
    for (int p = K - 1; p >= 0; --p) {
#pragma unroll
      for (int t = 0; t < W; ++t) acc[t] = fma(acc[t], y, s_c[p * 16 + t]);
    }
    const double cq = (D == 3 && ax == 1) ? qb[i] : 1.0;  // d = 3: charge folded into w1
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      double v = 0.0;
      if (t < W) {
        v = acc[t < W ? t : 0];
        if (t == 0 || t == W - 1) v = es_kernel((a0 + t - x) * inv_half, beta);
        v *= cq;
      }
      s_w[ax][lane][t] = v;
    }
    if (ax == 0) {
      if (D != 3) rq[j] = qb[i];
      int4 a;
      a.x = ai[i * D];
      a.y = D > 1 ? ai[i * D + 1] : 0;
      a.z = D > 2 ? ai[i * D + 2] : 0;
      a.w = 0;
      reinterpret_cast<int4*>(ra)[j] = a;
    }
  }
  __syncwarp();
  // d = 3: rw (n, 48) = [q w1 | w2 | w0], 16 zero-padded taps each (pencil kernel);
  // d = 2: rw (n, 32) = [w0 (16) | w1 (16)]
  double* dst = rw;
  (void)rw0;
  if (D == 3) {
    const int off = ax == 1 ? 0 : (ax == 2 ? 16 : 32);
    for (int e = lane; e < REC_PTS * 16; e += 32) {
      const int pt = e >> 4, t = e & 15;
      if (j0 + pt < n) dst[(j0 + pt) * 48 + off + t] = s_w[ax][pt][t];
    }
  } else {
    const int off = (ax == D - 1) ? 16 : 0;
    for (int e = lane; e < REC_PTS * 16; e += 32) {
      const int pt = e >> 4, t = e & 15;
      if (j0 + pt < n) dst[(j0 + pt) * 32 + off + t] = s_w[ax][pt][t];
    }
  }
}

struct PlaneArgs {
  const int4* jobs;       // (job id, first sorted point, count, scratch index or -1)
  int njobs;
  const int64_t* perm;    // sorted position -> batch point
  const double* wts;
  const int* ai;
  const double* qb;
  double* grid;           // (nbat, G^D)
  double* scratch;        // (nscratch, plane)
  const double* rw;       // sorted records (tile kernel)
  const double* rq;
  const int* ra;
  const double* rw0;
  int w, G;
};

// staged weights per point: w1 at [0, 16), w2 at [20, 36); row stride 40 doubles (80 words,
// = 16 mod 32) so the 4 point rows read by one fragment load fall on 2 disjoint bank sets
constexpr int TILE_RS = 40;
constexpr int TILE_W2 = 20;

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

#ifndef FGT_TILE_PTS
#define FGT_TILE_PTS 32
#endif
constexpr int TILE_PTS = FGT_TILE_PTS;                  // points per staged batch (<= 32)
constexpr int TILE_BUF = TILE_PTS * TILE_RS;            // doubles per staged batch
constexpr size_t TILE_SMEM = 4 * (2 * TILE_BUF * sizeof(double) + 32 * (sizeof(double) + 2 * sizeof(int)));

// rank-4 update of the 3x3 tile window at (BL, TL) (tile kernel, see below)
template <int NB, int BL, int TL>
__device__ __forceinline__ void tile_window(double (&acc)[NB][NB][2], const double* __restrict__ w1,
                                            const double* __restrict__ w2, int jr, double cj, int a1,
                                            int a2, bool valid, int w, int lane) {
  double A[3], B[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const int d = 8 * (BL + i) + (lane >> 2) - a1;
    A[i] = (valid && (unsigned)d < (unsigned)w) ? cj * w1[jr + d] : 0.0;
    const int e = 8 * (TL + i) + (lane >> 2) - a2;
    B[i] = (valid && (unsigned)e < (unsigned)w) ? w2[jr + e] : 0.0;
  }
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int k = 0; k < 3; ++k) dmma2(acc[BL + i][TL + k][0], acc[BL + i][TL + k][1], A[i], B[k]);
}

template <int NB>
__device__ __forceinline__ void window_dispatch(int widx, double (&acc)[NB][NB][2], const double* w1,
                                                const double* w2, int jr, double cj, int a1, int a2,
                                                bool valid, int w, int lane) {
  constexpr int NW = NB - 2;
  switch (widx & 63) {  // dense: one indirect branch
#define FGT_WIN(K)                                                                        \
  case K:                                                                                 \
    if constexpr ((K) < NW * NW) tile_window<NB, (K) / NW, (K) % NW>(acc, w1, w2, jr, cj, a1, a2, valid, w, lane); \
    break;
#define FGT_WIN8(K) FGT_WIN(K) FGT_WIN(K + 1) FGT_WIN(K + 2) FGT_WIN(K + 3) FGT_WIN(K + 4) FGT_WIN(K + 5) FGT_WIN(K + 6) FGT_WIN(K + 7)
    FGT_WIN8(0) FGT_WIN8(8) FGT_WIN8(16) FGT_WIN8(24) FGT_WIN8(32) FGT_WIN8(40) FGT_WIN8(48) FGT_WIN8(56)
#undef FGT_WIN8
#undef FGT_WIN
  }
}

template <int D, int NB>
#ifndef FGT_TILE_MINB
#define FGT_TILE_MINB 2
#endif
__global__ void __launch_bounds__(128, FGT_TILE_MINB) spread_tile_kernel(PlaneArgs a) {
  extern __shared__ double tsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* wbuf = tsm + (size_t)warp * 2 * TILE_BUF;             // 2 staged batches
  double* s_c = tsm + 4 * 2 * TILE_BUF + warp * 32;
  int* s_a1 = reinterpret_cast<int*>(tsm + 4 * 2 * TILE_BUF + 4 * 32) + warp * 64;
  int* s_a2 = s_a1 + 32;
  const int job = blockIdx.x * 4 + warp;
  if (job >= a.njobs) return;  // warp-uniform; only __syncwarp below
  const int G = a.G, w = a.w;
  const int4 jb = a.jobs[job];
  const int p = D == 3 ? jb.x % G : 0;
  double acc[NB][NB][2];
#pragma unroll
  for (int b = 0; b < NB; ++b)
#pragma unroll
    for (int t = 0; t < NB; ++t) acc[b][t][0] = acc[b][t][1] = 0.0;
  const int jend = jb.y + jb.z;
  const int nbatch = (jb.z + TILE_PTS - 1) / TILE_PTS;
  // lane layout of one staged weight row: w1 -> [0, 16), w2 -> [TILE_W2, TILE_W2 + 16)
  const int dst_off = lane < 16 ? lane : TILE_W2 + lane - 16;
  auto issue = [&](int bi) {
    const int base = jb.y + TILE_PTS * bi, cnt = min(TILE_PTS, jend - base);
    double* dst = wbuf + (bi & 1) * TILE_BUF;
    const double* src = a.rw + (int64_t)base * 32 + lane;
    for (int it = 0; it < cnt; ++it) cp_async8(dst + it * TILE_RS + dst_off, src + it * 32);
    cp_async_commit();
  };
  // per-point scalars of a batch, lane-parallel, kept in registers until published
  double nc = 0.0;
  int na1 = 0, na2 = 0;
  auto fetch = [&](int bi) {
    const int base = jb.y + TILE_PTS * bi, cnt = min(TILE_PTS, jend - base);
    if (lane < cnt) {
      const int64_t j = base + lane;
      const int4 r = *reinterpret_cast<const int4*>(a.ra + 4 * j);
      double c = a.rq[j];
      if (D == 3) c *= a.rw0[j * 16 + (p - r.x)];
      nc = c;
      na1 = D == 3 ? r.y : r.x;
      na2 = D == 3 ? r.z : r.y;
    }
  };
  issue(0);
  fetch(0);
  for (int bi = 0; bi < nbatch; ++bi) {
    const int cnt = min(TILE_PTS, jend - (jb.y + TILE_PTS * bi));
    __syncwarp();
    s_c[lane] = nc;
    s_a1[lane] = na1;
    s_a2[lane] = na2;
    if (bi + 1 < nbatch) {
      issue(bi + 1);
      fetch(bi + 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncwarp();
    const double* w1 = wbuf + (bi & 1) * TILE_BUF;
    const double* w2 = w1 + TILE_W2;
    for (int g = 0; 4 * g < cnt; ++g) {
      const int j = 4 * g + (lane & 3);
      const bool valid = j < cnt;
      const double cj = valid ? s_c[j] : 0.0;
      const int a1 = valid ? s_a1[j] : 0, a2 = valid ? s_a2[j] : 0;
      // rows / columns the group touches (warp-uniform: reductions over its <= 4 points)
      const int rlo = __reduce_min_sync(0xffffffffu, valid ? a1 : 1 << 20);
      const int rhi = __reduce_max_sync(0xffffffffu, valid ? a1 + w - 1 : -1);
      const int clo = __reduce_min_sync(0xffffffffu, valid ? a2 : 1 << 20);
      const int chi = __reduce_max_sync(0xffffffffu, valid ? a2 + w - 1 : -1);
      const int bl = rlo >> 3, bh = rhi >> 3, tl = clo >> 3, th = chi >> 3;
      if constexpr (NB >= 3) {
        // a 3x3-tile window covers every 4-point group (span <= 11 + 7 + spread): one
        // straight-line block of 9 unpredicated DMMAs per window position
        if (bh - bl <= 2 && th - tl <= 2) {
          const int wb = min(bl, NB - 3), wt = min(tl, NB - 3);
          window_dispatch<NB>(wb * (NB - 2) + wt, acc, w1, w2, j * TILE_RS, cj, a1, a2, valid, w, lane);
          continue;
        }
      }
      // wide groups: fragments only for the touched tiles (uniform branches skip the rest)
      double B[NB];
#pragma unroll
      for (int t = 0; t < NB; ++t) {
        B[t] = 0.0;
        if (t >= tl && t <= th) {
          const int e = 8 * t + (lane >> 2) - a2;
          if (valid && (unsigned)e < (unsigned)w) B[t] = w2[j * TILE_RS + e];
        }
      }
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        if (b < bl || b > bh) continue;
        const int d = 8 * b + (lane >> 2) - a1;
        const double A = (valid && (unsigned)d < (unsigned)w) ? cj * w1[j * TILE_RS + d] : 0.0;
#pragma unroll
        for (int t = 0; t < NB; ++t) {
          if (t < tl || t > th) continue;
          dmma2(acc[b][t][0], acc[b][t][1], A, B[t]);
        }
      }
    }
  }
  // write the plane: lane holds cells (8b + lane/4, 8t + 2 (lane%4) + {0, 1})
  const int64_t plane = (int64_t)G * G;
  const int bx = D == 3 ? jb.x / G : jb.x;
  double* out = jb.w < 0 ? a.grid + (int64_t)bx * plane * (D == 3 ? G : 1) + (int64_t)p * plane
                         : a.scratch + (int64_t)jb.w * plane;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const int r = 8 * b + (lane >> 2);
#pragma unroll
    for (int t = 0; t < NB; ++t) {
#pragma unroll
      for (int i2 = 0; i2 < 2; ++i2) {
        const int c = 8 * t + 2 * (lane & 3) + i2;
        if (r < G && c < G) out[(int64_t)r * G + c] = acc[b][t][i2];
      }
    }
  }
}

// ---------------------------------------------------------------- d = 3 pencil spreading
// A pencil is the 8 x 8 x PH block of grid cells (rows 8b + [0, 8), columns 8t + [0, 8),
// planes h PH + [0, PH)); one warp keeps it as PH DMMA accumulator tiles in registers.
// Points are sorted by (box, row class, a_0, a_2), where the row classes cut every 8 rows
// at a = 0 and a = 1 - w (mod 8): the points whose row taps [a_1, a_1 + w) touch block b
// are then ONE contiguous key range per (box, b) (a "row job", split at 4096 points).
// Work item = (row job, pencil (t, h)); warps are persistent and take items from a global
// counter (largest row jobs first), so no warp waits on another.  Per item the warp scans
// the range 32 points at a time, keeps (ballot) the points whose column and axis-0 taps
// touch its pencil and stages one row per kept point by cp.async (double-buffered): the
// 8 row weights q w1[8b + r - a_1], the 8 column weights w2[8t + c - a_2] (zero-filled
// outside the taps), a zero band, the 16 axis-0 weights.  A group of 4 kept points then
// issues one rank-4 DMMA per plane,
//   C_p += (q w1[rows] w0[p - a_0]) (x) w2[cols],
// as a straight-line block of NPL planes chosen by a jump table on the group's first
// plane; planes past a point's taps read the zero band / zero padding of its staged row,
// so the plane loop is one shared load, one multiply and one DMMA per plane.  Kept rows go
// to a ring, so groups stay full across chunk boundaries.
constexpr int PEN_PH = 24;    // planes per pencil part (2 PEN_PH accumulator doubles per lane)
constexpr int PEN_RS = 38;    // staged row: A 8 | B 8 | zeros 6 | w0 16
constexpr int PEN_W0 = 22;    // offset of w0 in a staged row (zero band >= NPL - w)
constexpr int PEN_WARPS = 2;  // warps per CTA (each independent)
// staged rows form a ring: <= 3 rows left over + the kept rows of the chunk being
// processed + those of the chunk in flight
#ifndef FGT_PEN_CH
#define FGT_PEN_CH 32
#endif
constexpr int PEN_CH = FGT_PEN_CH;            // points scanned per chunk (<= 32)
#ifndef FGT_PEN_RING
#define FGT_PEN_RING 48
#endif
// ring of staged rows: a chunk is staged only when PEN_CH rows are free (else the staged
// rows are processed first), so any size >= PEN_CH + 3 is correct
constexpr int PEN_RING = FGT_PEN_RING;
// per warp: the row ring, its a_0 ring, 32 (j, a_1, a_2) metas
constexpr size_t PEN_WSMEM = PEN_RING * PEN_RS * sizeof(double) + PEN_RING * sizeof(int) + 32 * sizeof(int4);
constexpr size_t PEN_SMEM = PEN_WARPS * PEN_WSMEM;

struct PencilArgs {
  const int4* jobs;  // row jobs: (box * NB + b, first sorted point, count, scratch base or -1)
  const int* njobs;  // number of row jobs (device; items = row jobs x per)
  int* counter;      // work-item counter (zeroed before the launch)
  const double* rw;  // sorted records (n, PEN_REC) [q w1 | w2 | w0]
  const int* ra;     // (n, 4) first taps (a_0, a_1, a_2, -)
  double* grid;      // (nbat, G^3)
  double* scratch;   // (nscr, PEN_PH * 64) partial pencils
  int w, G, NB, nparts, PH, per;
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}

__device__ __forceinline__ void cp_async8_zfill(void* smem, const void* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(valid ? 8 : 0));
}

// planes [s, s + NPL) of the part, s = S - 15 >= 1 - w, clipped to [0, PEN_PH) at compile
// time; the lane's axis-0 weight at plane s + q is w0row[q] (zero outside its taps)
// Planes [NPL_HEAD(NPL), NPL) are issued only when the group spans them (cnt > head): a
// group whose points share their first tap (up to +1) stops after the head.
template <int NPL>
__host__ __device__ constexpr int npl_head() { return NPL == 16 ? 12 : (NPL == 12 ? 9 : 6); }

template <int NPL, int S>
__device__ __forceinline__ void pencil_planes(double (&acc)[PEN_PH][2], const double* __restrict__ w0row,
                                              double A, double B, int cnt) {
  constexpr int H = npl_head<NPL>();
  double wq[NPL];  // all loads first: the DMUL -> DMMA chains then issue back to back
#pragma unroll
  for (int q = 0; q < H; ++q) {
    const int pl = S - 15 + q;
    if (pl >= 0 && pl < PEN_PH) wq[q] = w0row[q];
  }
#pragma unroll
  for (int q = 0; q < H; ++q) {
    const int pl = S - 15 + q;
    if (pl >= 0 && pl < PEN_PH) dmma2(acc[pl][0], acc[pl][1], A * wq[q], B);
  }
  if (cnt > H) {
#pragma unroll
    for (int q = H; q < NPL; ++q) {
      const int pl = S - 15 + q;
      if (pl >= 0 && pl < PEN_PH) wq[q] = w0row[q];
    }
#pragma unroll
    for (int q = H; q < NPL; ++q) {
      const int pl = S - 15 + q;
      if (pl >= 0 && pl < PEN_PH) dmma2(acc[pl][0], acc[pl][1], A * wq[q], B);
    }
  }
}

template <int NPL>
__device__ __forceinline__ void pencil_dispatch(int S, double (&acc)[PEN_PH][2], const double* w0row, double A,
                                                double B, int cnt) {
  // S in [0, 39); a dense 64-entry switch lowers to one indirect branch
  switch (S & 63) {
#define FGT_PL(K) \
  case K: pencil_planes<NPL, K>(acc, w0row, A, B, cnt); break;
#define FGT_PL8(K) FGT_PL(K) FGT_PL(K + 1) FGT_PL(K + 2) FGT_PL(K + 3) FGT_PL(K + 4) FGT_PL(K + 5) FGT_PL(K + 6) FGT_PL(K + 7)
    FGT_PL8(0) FGT_PL8(8) FGT_PL8(16) FGT_PL8(24) FGT_PL8(32) FGT_PL8(40) FGT_PL8(48) FGT_PL8(56)
#undef FGT_PL8
#undef FGT_PL
  }
}

template <int NPL>
__global__ void __launch_bounds__(PEN_WARPS * 32, 5) spread_pencil_kernel(PencilArgs a) {
  extern __shared__ double psm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  char* wsm = reinterpret_cast<char*>(psm) + warp * PEN_WSMEM;
  double* stg = reinterpret_cast<double*>(wsm);
  int4* s_meta = reinterpret_cast<int4*>(stg + PEN_RING * PEN_RS);
  int* s_a0 = reinterpret_cast<int*>(s_meta + 32);
  const int NB = a.NB, G = a.G, w = a.w;
  // zero band of every staged row (never written by the staging)
  for (int e = lane; e < PEN_RING * 6; e += 32) stg[(e / 6) * PEN_RS + 16 + e % 6] = 0.0;
  const int4* ra4 = reinterpret_cast<const int4*>(a.ra);
  while (true) {
    int item = 0;
    if (lane == 0) item = atomicAdd(a.counter, 1);
    item = __shfl_sync(0xffffffffu, item, 0);
    if (item >= *a.njobs * a.per) break;
    const int4 jb = a.jobs[item / a.per];
    const int th = item - (item / a.per) * a.per;  // t * nparts + h
    const int t = th / a.nparts, h = th - t * a.nparts;
    const int box = jb.x / NB, b = jb.x - box * NB;
    const int P0 = h * a.PH, PHc = min(a.PH, G - P0);
    const int c_lo = 8 * t - w + 1, c_hi = 8 * t + 7;
    const int p_lo = P0 - w + 1, p_hi = P0 + PHc - 1;
    double acc[PEN_PH][2];
#pragma unroll
    for (int i = 0; i < PEN_PH; ++i) acc[i][0] = acc[i][1] = 0.0;
    const int nchunk = (jb.z + PEN_CH - 1) / PEN_CH;
    auto load_ra = [&](int c) {
      int4 r = make_int4(0, 0, -1000, 0);
      if (lane < PEN_CH && PEN_CH * c + lane < jb.z) r = ra4[jb.y + PEN_CH * c + lane];
      return r;
    };
    // keep the chunk's points that touch the pencil; stage their rows at the ring's tail
    // (ring positions: monotone counters mod PEN_RING)
    int head = 0, tail = 0;
    auto stage = [&](int c, int4 r) {
      const bool ok = r.z >= c_lo && r.z <= c_hi && r.x >= p_lo && r.x <= p_hi;
      const unsigned mask = __ballot_sync(0xffffffffu, ok);
      const int nok = __popc(mask);
      if (ok) s_meta[__popc(mask & ((1u << lane) - 1u))] = make_int4(jb.y + PEN_CH * c + lane, r.y, r.z, r.x);
      __syncwarp();
      // four lanes per kept point (8 points per pass): lane quarter q copies row weights
      // 2q, 2q + 1, column weights 2q, 2q + 1 (8-byte, zero-filled outside the taps) and
      // axis-0 weights [4q, 4q + 4) (two 16-byte copies)
      const int q = lane & 3;
      const int ts = tail % PEN_RING;
      for (int i = lane >> 2; i < nok; i += 8) {
        const int4 m = s_meta[i];
        const int slot = ts + i >= PEN_RING ? ts + i - PEN_RING : ts + i;
        double* dst = stg + slot * PEN_RS;
        const double* rec = a.rw + (int64_t)m.x * PEN_REC;
        if (q == 0) s_a0[slot] = m.w;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int ia = 8 * b + 2 * q + e - m.y, ib = 8 * t + 2 * q + e - m.z;
          const bool va = (unsigned)ia < 16u, vb = (unsigned)ib < 16u;
          cp_async8_zfill(dst + 2 * q + e, rec + (va ? ia : 0), va);
          cp_async8_zfill(dst + 8 + 2 * q + e, rec + 16 + (vb ? ib : 0), vb);
          cp_async16(dst + PEN_W0 + 4 * q + 2 * e, rec + 32 + 4 * q + 2 * e);  // axis-0 weights
        }
      }
      cp_async_commit();
      __syncwarp();
      tail += nok;
    };
    int4 r_next = make_int4(0, 0, -1000, 0);
    if (nchunk > 0) {
      stage(0, load_ra(0));
      if (nchunk > 1) r_next = load_ra(1);
    }
    // full groups of 4 from [head, end) of the ring (the partial group too when all = true)
    auto process = [&](int end, bool all) {
      const int avail = end - head;
      const int ngr = all ? (avail + 3) >> 2 : avail >> 2;
      const int hs = head % PEN_RING;
      for (int g = 0; g < ngr; ++g) {
        const int k = 4 * g + (lane & 3);
        const bool valid = k < avail;
        const int kk = hs + (valid ? k : 0);
        const int slot = kk >= PEN_RING ? kk - PEN_RING : kk;
        const double* row = stg + slot * PEN_RS;
        const double A = valid ? row[lane >> 2] : 0.0;
        const double B = valid ? row[8 + (lane >> 2)] : 0.0;
        const int a0i = valid ? s_a0[slot] : (1 << 20);
        bool pend = valid;
        while (true) {
          const int m = __reduce_min_sync(0xffffffffu, pend ? a0i : (1 << 20));
          if (m == (1 << 20)) break;
          const bool sel = pend && a0i <= m + NPL - w;
          const int mx = __reduce_max_sync(0xffffffffu, sel ? a0i : -(1 << 20));
          // the lane's axis-0 weights from plane m on: m - a0i in [w - NPL, 0] for a
          // selected lane (the zero band before its taps, zero padding after)
          const double* w0row = row + PEN_W0 + (sel ? m - a0i : 0);
          pencil_dispatch<NPL>(m - P0 + 15, acc, w0row, sel ? A : 0.0, B, mx + w - m);
          pend = pend && !sel;
        }
      }
      head += min(avail, 4 * ngr);
    };
    for (int c = 0; c < nchunk; ++c) {
      const int ready = tail;  // rows of chunks <= c
      const bool last = c + 1 >= nchunk;
      if (!last) {
        if (tail - head + PEN_CH > PEN_RING) {
          // no room for another chunk: finish the staged rows first
          cp_async_wait<0>();
          __syncwarp();
          process(ready, false);
          __syncwarp();
        }
        stage(c + 1, r_next);
        if (c + 2 < nchunk) r_next = load_ra(c + 2);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncwarp();
      process(ready, last);
      __syncwarp();
    }
    // write the pencil: lane holds rows 8b + lane/4, columns 8t + 2 (lane % 4) + {0, 1}
    const int r = lane >> 2, cc = 2 * (lane & 3);
    if (jb.w < 0) {
      double* out = a.grid + (int64_t)box * G * G * G;
      const int gr = 8 * b + r, gc = 8 * t + cc;
#pragma unroll
      for (int pl = 0; pl < PEN_PH; ++pl) {
        if (pl < PHc && gr < G) {
          double* o = out + ((int64_t)(P0 + pl) * G + gr) * G + gc;
          if (gc < G) o[0] = acc[pl][0];
          if (gc + 1 < G) o[1] = acc[pl][1];
        }
      }
    } else {
      double* o = a.scratch + ((int64_t)jb.w + th) * (PEN_PH * 64) + r * 8 + cc;
#pragma unroll
      for (int pl = 0; pl < PEN_PH; ++pl) {
        o[pl * 64] = acc[pl][0];
        o[pl * 64 + 1] = acc[pl][1];
      }
    }
  }
}

// partial pencils of K-split (box, b) ranges: red = (box * NB + b, first scratch, chunks, -);
// chunk k's pencil (t, h) is scratch[first + k * NB * nparts + t * nparts + h]; summed in
// chunk order (deterministic) and scattered into the grid
__global__ void pencil_reduce_kernel(const double* __restrict__ scratch, const int4* __restrict__ red,
                                     const int* __restrict__ nred, int NB, int nparts, int PH, int G,
                                     double* __restrict__ grid) {
  if ((int)blockIdx.y >= *nred) return;  // launched for the host's upper bound
  const int4 rd = red[blockIdx.y];
  const int th = blockIdx.z, t = th / nparts, h = th - t * nparts;
  const int box = rd.x / NB, b = rd.x - box * NB;
  const int P0 = h * PH, PHc = min(PH, G - P0);
  const int64_t stride = (int64_t)NB * nparts * PEN_PH * 64;
  for (int e = threadIdx.x; e < PEN_PH * 64; e += blockDim.x) {
    const int pl = e >> 6, r = (e >> 3) & 7, c = e & 7;
    const int gr = 8 * b + r, gc = 8 * t + c;
    if (pl >= PHc || gr >= G || gc >= G) continue;
    const double* src = scratch + ((int64_t)rd.y + th) * (PEN_PH * 64) + e;
    double s = 0.0;
    for (int k = 0; k < rd.z; ++k) s += src[k * stride];
    grid[(int64_t)box * G * G * G + ((int64_t)(P0 + pl) * G + gr) * G + gc] = s;
  }
}

// Pencil job list on the device (no host round trip): per row job (box, row block) with
// n points, nc = max(1, ceil(n / PCH)) chunks; row jobs split in more than one chunk keep
// partial pencils in scratch (per slots each) and get a reduce entry.  One CTA scans the
// row jobs in tiles of 1024; outputs the unsorted chunk list with sort keys PCH - count
// (largest chunks first after a stable ascending sort; padding up to the host's bound sorts
// last) and counts[0] = chunks, counts[1] = reduce entries.
__global__ void __launch_bounds__(1024) pencil_jobs_kernel(const int* __restrict__ range, int njob, int PCH,
                                                          int per, int bound, int4* __restrict__ jobs_tmp,
                                                          uint64_t* __restrict__ key, int64_t* __restrict__ val,
                                                          int4* __restrict__ reds, int* __restrict__ counts) {
  typedef cub::BlockScan<int, 1024> Scan;
  __shared__ typename Scan::TempStorage ts;
  __shared__ int carry[3];
  if (threadIdx.x < 3) carry[threadIdx.x] = 0;
  __syncthreads();
  for (int base = 0; base < njob; base += 1024) {
    const int jid = base + (int)threadIdx.x;
    int n = 0, lo = 0, nc = 0, red = 0;
    if (jid < njob) {
      lo = range[2 * jid];
      n = range[2 * jid + 1] - lo;
      nc = n <= PCH ? 1 : (n + PCH - 1) / PCH;
      red = n > PCH;
    }
    int o_job, o_red, o_scr, t_job, t_red, t_scr;
    Scan(ts).ExclusiveSum(nc, o_job, t_job);
    __syncthreads();
    Scan(ts).ExclusiveSum(red, o_red, t_red);
    __syncthreads();
    Scan(ts).ExclusiveSum(red ? nc * per : 0, o_scr, t_scr);
    const int cj = carry[0], cr = carry[1], cs = carry[2];
    if (jid < njob) {
      for (int c = 0; c < nc; ++c) {
        const int idx = cj + o_job + c, len = min(PCH, n - c * PCH);
        jobs_tmp[idx] = make_int4(jid, lo + c * PCH, max(0, len), red ? cs + o_scr + c * per : -1);
        key[idx] = (uint64_t)(PCH - max(0, len));
        val[idx] = idx;
      }
      if (red) reds[cr + o_red] = make_int4(jid, cs + o_scr, nc, 0);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      carry[0] = cj + t_job;
      carry[1] = cr + t_red;
      carry[2] = cs + t_scr;
    }
    __syncthreads();
  }
  for (int idx = carry[0] + (int)threadIdx.x; idx < bound; idx += blockDim.x) {
    key[idx] = (uint64_t)(PCH + 1);
    val[idx] = idx;
  }
  if (threadIdx.x == 0) {
    counts[0] = carry[0];
    counts[1] = carry[1];
  }
}

__global__ void gather_jobs_kernel(const int4* __restrict__ tmp, const int64_t* __restrict__ perm,
                                   const int* __restrict__ counts, int4* __restrict__ jobs) {
  const int n = counts[0];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) jobs[i] = tmp[perm[i]];
}

// d = 1: one warp per (box, cell) job sums c w0[p - a0] over its points
__global__ void __launch_bounds__(128) spread_line_kernel(PlaneArgs a) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int job = blockIdx.x * 4 + warp;
  if (job >= a.njobs) return;
  const int4 jb = a.jobs[job];
  const int G = a.G, p = jb.x % G;
  double sum = 0.0;
  for (int j = jb.y + lane; j < jb.y + jb.z; j += 32) {
    const int64_t i = a.perm[j];
    sum += a.qb[i] * a.wts[i * MAXW + (p - a.ai[i])];
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
  if (lane == 0) {
    if (jb.w < 0) a.grid[(int64_t)(jb.x / G) * G + p] = sum;
    else a.scratch[jb.w] = sum;
  }
}

__global__ void plane_reduce_kernel(const double* __restrict__ scratch, const int4* __restrict__ red,
                                    int64_t plane, int64_t job_stride, double* __restrict__ grid) {
  const int4 r = red[blockIdx.y];  // (job id, first scratch, count, -); job id -> offset job*plane
  double* out = grid + (int64_t)r.x * plane;
  (void)job_stride;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < plane;
       e += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int t = 0; t < r.z; ++t) s += scratch[(int64_t)(r.y + t) * plane + e];
    out[e] = s;
  }
}

// ------------------------------------------------------------------ interpolation
struct InterpArgs {
  const double* tgt;
  const double* center;
  const int64_t* psi_ids;
  const int64_t* list;   // list index -> psi index
  const int64_t* tgt_start;
  const int64_t* tgt_count;
  const double* grid;    // (list, G^D) real
  double* u;
  double sc, inv_delta, beta;
  int w, gmin, G;
};

// d = 2 interpolation with the kernel width W a compile-time constant (taps and weights in
// registers) and the box's G x G grid staged in shared memory: one CTA per psi box, one
// thread per target.
template <int W>
__global__ void __launch_bounds__(256) interp2_kernel(InterpArgs a) {
  extern __shared__ double s_grid[];
  const int64_t li = blockIdx.x;
  const int64_t T = a.psi_ids[a.list[li]];
  const int64_t t0 = a.tgt_start[T];
  const int nt = (int)a.tgt_count[T];
  const int G = a.G;
  const double* grid = a.grid + li * (int64_t)G * G;
  for (int i = threadIdx.x; i < G * G; i += blockDim.x) s_grid[i] = grid[i];
  __syncthreads();
  const double c0 = a.center[T * 2], c1 = a.center[T * 2 + 1];
  const double s = a.sc * a.inv_delta, half = 0.5 * W, inv_half = 2.0 / W;
  for (int j = threadIdx.x; j < nt; j += blockDim.x) {
    const double t_0 = (a.tgt[(t0 + j) * 2] - c0) * s, t_1 = (a.tgt[(t0 + j) * 2 + 1] - c1) * s;
    const double a0 = ceil(t_0 - half), a1 = ceil(t_1 - half);
    const int i0 = max(0, min((int)a0 - a.gmin, G - W)), i1 = max(0, min((int)a1 - a.gmin, G - W));
    double w0[W], w1[W];
#pragma unroll
    for (int o = 0; o < W; ++o) {
      w0[o] = es_kernel((a0 + o - t_0) * inv_half, a.beta);
      w1[o] = es_kernel((a1 + o - t_1) * inv_half, a.beta);
    }
    double acc = 0.0;
#pragma unroll
    for (int o0 = 0; o0 < W; ++o0) {
      const double* row = s_grid + (i0 + o0) * G + i1;
      double part = 0.0;
#pragma unroll
      for (int o1 = 0; o1 < W; ++o1) part += w1[o1] * row[o1];
      acc += w0[o0] * part;
    }
    a.u[t0 + j] += acc;
  }
}

template <int D>
__global__ void __launch_bounds__(256) interp_kernel(InterpArgs a) {
  __shared__ double s_w[8][D][MAXW];
  const int64_t li = blockIdx.x;
  const int64_t T = a.psi_ids[a.list[li]];
  const int64_t t0 = a.tgt_start[T];
  const int nt = (int)a.tgt_count[T];
  const int G = a.G, w = a.w;
  const int64_t GD = D == 3 ? (int64_t)G * G * G : (D == 2 ? (int64_t)G * G : G);
  const double* grid = a.grid + li * GD;
  double ctr[D];
#pragma unroll
  for (int k = 0; k < D; ++k) ctr[k] = a.center[T * D + k];
  const double s = a.sc * a.inv_delta, half = 0.5 * w, inv_half = 2.0 / w;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (D == 3) {
    // one warp per target; lanes over the (o1, o2) taps of each o0 plane
    for (int j = warp; j < nt; j += 8) {
      int ai[D];
#pragma unroll
      for (int k = 0; k < D; ++k) {
        const double tt = (a.tgt[(t0 + j) * D + k] - ctr[k]) * s;
        const double a0 = ceil(tt - half);
        ai[k] = max(0, min((int)a0 - a.gmin, G - w));
        for (int o = lane; o < w; o += 32) s_w[warp][k][o] = es_kernel((a0 + o - tt) * inv_half, a.beta);
      }
      __syncwarp();
      double acc = 0.0;
      for (int o0 = 0; o0 < w; ++o0) {
        const double* pl = grid + ((int64_t)(ai[0] + o0) * G) * G;
        double part = 0.0;
        for (int idx = lane; idx < w * w; idx += 32) {
          const int o1 = idx / w, o2 = idx - o1 * w;
          part += s_w[warp][1][o1] * s_w[warp][2][o2] * pl[(ai[1] + o1) * G + ai[2] + o2];
        }
        acc += s_w[warp][0][o0] * part;
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
      if (lane == 0) a.u[t0 + j] += acc;
      __syncwarp();
    }
  } else {
    for (int j = threadIdx.x; j < nt; j += blockDim.x) {
      double wk[D][MAXW];
      int ai[D];
#pragma unroll
      for (int k = 0; k < D; ++k) {
        const double tt = (a.tgt[(t0 + j) * D + k] - ctr[k]) * s;
        const double a0 = ceil(tt - half);
        ai[k] = max(0, min((int)a0 - a.gmin, G - w));
        for (int o = 0; o < MAXW; ++o) wk[k][o] = o < w ? es_kernel((a0 + o - tt) * inv_half, a.beta) : 0.0;
      }
      double acc = 0.0;
      if (D == 2) {
        for (int o0 = 0; o0 < w; ++o0) {
          const double* row = grid + (int64_t)(ai[0] + o0) * G + ai[1];
          double part = 0.0;
          for (int o1 = 0; o1 < w; ++o1) part += wk[1][o1] * row[o1];
          acc += wk[0][o0] * part;
        }
      } else {
        for (int o0 = 0; o0 < w; ++o0) acc += wk[0][o0] * grid[ai[0] + o0];
      }
      a.u[t0 + j] += acc;
    }
  }
}

// ------------------------------------------------------------------ proxy charges
// grid[b][a_0][a_1 ..] = sum_j q_j prod_k L_{a_k}(x_jk): per box one real GEMM on the DMMA
// pipe, M = p (axis 0), N = p^(d-1) (last axis padded to 8-column tiles), K = the box's
// points.  CTA = (box, 8-row m-tile, n-chunk); per chunk of 32 points the d x p Lagrange
// values of every point go to shared memory once (barycentric form at the Chebyshev
// nodes; a point on a node takes the Kronecker row), then each warp feeds its n-tiles:
// A[a_0][j] = q_j L_{a_0}(x_j0), B[j][(a_1 a_2)] = L_{a_1}(x_j1) L_{a_2}(x_j2).
constexpr int PROXY_NT = 16;  // n-tiles per warp
struct ProxyArgs {
  const double* src;
  const double* q;
  const double* center;
  const int64_t* dense_ids;
  const int64_t* src_start;
  const int64_t* slots;
  const int64_t* boff;
  const double* cheb_x;
  const double* cheb_lam;
  double* grid;  // (nbat, p^D)
  double sc;
  int p;
};

template <int D>
__global__ void __launch_bounds__(256) proxy_charges_kernel(ProxyArgs a) {
  __shared__ double sL[D][32][PROXY_PMAX + 1];
  __shared__ double sq[32];
  __shared__ double sx[PROXY_PMAX], slam[PROXY_PMAX];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int p = a.p, P8 = (p + 7) / 8;  // 8-column tiles along the last axis
  const int ntiles = D == 1 ? 1 : (D == 2 ? P8 : p * P8);
  const int64_t bx = blockIdx.x;
  const int mt = blockIdx.y;
  const int nt0 = (blockIdx.z * 8 + warp) * PROXY_NT;
  const int64_t box = a.dense_ids[a.slots[bx]];
  const int64_t s0 = a.src_start[box], n = a.boff[bx + 1] - a.boff[bx];
  for (int i = threadIdx.x; i < p; i += blockDim.x) {
    sx[i] = a.cheb_x[i];
    slam[i] = a.cheb_lam[i];
  }
  double acc[PROXY_NT][2];
#pragma unroll
  for (int t = 0; t < PROXY_NT; ++t) acc[t][0] = acc[t][1] = 0.0;
  __syncthreads();
  for (int64_t c0 = 0; c0 < n; c0 += 32) {
    // Lagrange rows of the chunk: thread (point, axis)
    if (threadIdx.x < 32 * D) {
      const int pt = threadIdx.x / D, k = threadIdx.x - pt * D;
      double* L = sL[k][pt];
      if (c0 + pt < n) {
        const double x = (a.src[(s0 + c0 + pt) * D + k] - a.center[box * D + k]) * a.sc;
        double den = 0.0;
        int hit = -1;
        for (int i = 0; i < p; ++i) {
          const double dx = x - sx[i];
          if (dx == 0.0) hit = i;
          const double t = slam[i] / dx;
          L[i] = t;
          den += t;
        }
        const double inv = 1.0 / den;
        for (int i = 0; i < p; ++i) L[i] = hit < 0 ? L[i] * inv : (i == hit ? 1.0 : 0.0);
        if (k == 0) sq[pt] = a.q[s0 + c0 + pt];
      } else {
        for (int i = 0; i < p; ++i) L[i] = 0.0;
        if (k == 0) sq[pt] = 0.0;
      }
    }
    __syncthreads();
    const int row = mt * 8 + (lane >> 2);
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const int j = ks * 4 + (lane & 3);
      const double av = row < p ? sq[j] * sL[0][j][row] : 0.0;
#pragma unroll
      for (int t = 0; t < PROXY_NT; ++t) {
        const int nt = nt0 + t;
        if (nt < ntiles) {  // warp-uniform
          double bv;
          if (D == 1) {
            bv = (lane >> 2) == 0 ? 1.0 : 0.0;
          } else if (D == 2) {
            const int a1 = nt * 8 + (lane >> 2);
            bv = a1 < p ? sL[1][j][a1] : 0.0;
          } else {
            const int a1 = nt / P8, a2 = (nt - a1 * P8) * 8 + (lane >> 2);
            bv = a2 < p ? sL[1][j][a1] * sL[D - 1][j][a2] : 0.0;
          }
          dmma2(acc[t][0], acc[t][1], av, bv);
        }
      }
    }
    __syncthreads();
  }
  // C fragment: row a_0 = mt 8 + lane / 4, columns 2 (lane % 4) + {0, 1} of the n-tile
  const int row = mt * 8 + (lane >> 2);
  int64_t pd = 1;
  for (int k = 0; k < D; ++k) pd *= p;
  double* g = a.grid + bx * pd;
  if (row < p) {
#pragma unroll
    for (int t = 0; t < PROXY_NT; ++t) {
      const int nt = nt0 + t;
      if (nt >= ntiles) continue;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int cidx = 2 * (lane & 3) + e;
        if (D == 1) {
          if (cidx == 0) g[row] = acc[t][e];
        } else if (D == 2) {
          const int a1 = nt * 8 + cidx;
          if (a1 < p) g[row * p + a1] = acc[t][e];
        } else {
          const int a1 = nt / P8, a2 = (nt - a1 * P8) * 8 + cidx;
          if (a2 < p) g[((int64_t)row * p + a1) * p + a2] = acc[t][e];
        }
      }
    }
  }
}

void gauss_legendre(int n, std::vector<double>& x, std::vector<double>& wq) {
  x.resize(n);
  wq.resize(n);
  for (int i = 0; i < n; ++i) {
    double z = std::cos(M_PI * (i + 0.75) / (n + 0.5)), dp = 1.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = z;
      for (int k = 2; k <= n; ++k) {
        double p2 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      dp = n * (z * p1 - p0) / (z * z - 1.0);
      double dz = p1 / dp;
      z -= dz;
      if (std::fabs(dz) < 1e-16) break;
    }
    x[i] = z;
    wq[i] = 2.0 / ((1.0 - z * z) * dp * dp);
  }
}

}  // namespace

const NufftPlan& nufft_plan_cached(int n_f, double tol, double X, const double* w1d, cudaStream_t st) {
  // key: every input bit that shapes the plan, plus the device
  int dev = 0;
  FGT_CUDA(cudaGetDevice(&dev));
  std::string key(reinterpret_cast<const char*>(&dev), sizeof(dev));
  key.append(reinterpret_cast<const char*>(&n_f), sizeof(n_f));
  key.append(reinterpret_cast<const char*>(&tol), sizeof(tol));
  key.append(reinterpret_cast<const char*>(&X), sizeof(X));
  if (w1d) key.append(reinterpret_cast<const char*>(w1d), sizeof(double) * n_f);
  static std::mutex mu;
  static auto* cache = new std::map<std::string, NufftPlan*>();  // process lifetime
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache->find(key);
  if (it != cache->end()) return *it->second;
  auto* p = new NufftPlan();
  nufft_plan(*p, n_f, tol, X, w1d, st);
  FGT_CUDA(cudaStreamSynchronize(st));  // usable from any stream from now on
  (*cache)[key] = p;
  return *p;
}

// Piecewise-polynomial ES kernel (the Horner scheme FINUFFT uses for its spreader): a point
// whose first tap sits f in [0, 1) cells right of x - w/2 gives tap t the weight
// es((2 (f + t) - w) / w).  Per interior tap, Chebyshev interpolation in y = 2f - 1 at
// degree K, converted to monomials in long double; K grows until the worst interior-tap
// error on a fine grid is <= max(tol / 1000, 2e-14) (or the best K <= 24 is kept).  The
// edge taps t = 0, w-1 hold the kernel's square-root branch point (z = -+1) and are always
// evaluated exactly.  Output hc[p * 16 + t], p = 0..K.
static void es_fit(int w, double beta, double tol, std::vector<double>& hc, int& K_out) {
  const double target = std::max(1e-3 * tol, 2e-14);
  double best_err = 1e300;
  std::vector<double> best;
  int best_k = 0;
  for (int K = 8; K < HC_MAX; ++K) {
    std::vector<double> c((K + 1) * 16, 0.0);
    for (int t = 1; t + 1 < w; ++t) {
      std::vector<long double> a(K + 1, 0.0L);
      for (int k = 0; k <= K; ++k) {
        long double s = 0;
        for (int j = 0; j <= K; ++j) {
          const long double th = M_PIl * (j + 0.5L) / (K + 1);
          const double y = (double)cosl(th);
          s += (long double)es_kernel((2.0 * (0.5 * (y + 1.0) + t) - w) / w, beta) * cosl(k * th);
        }
        a[k] = 2.0L * s / (K + 1);
      }
      a[0] *= 0.5L;
      // sum_k a_k T_k(y) in monomials: T_{k+1} = 2 y T_k - T_{k-1}
      std::vector<long double> tm1(K + 1, 0.0L), tk(K + 1, 0.0L), mono(K + 1, 0.0L);
      tm1[0] = 1.0L;
      if (K >= 1) tk[1] = 1.0L;
      for (int p = 0; p <= K; ++p) mono[p] += a[0] * tm1[p];
      for (int k = 1; k <= K; ++k) {
        for (int p = 0; p <= K; ++p) mono[p] += a[k] * tk[p];
        std::vector<long double> nx(K + 1, 0.0L);
        for (int p = 0; p <= K; ++p) {
          if (p + 1 <= K) nx[p + 1] += 2.0L * tk[p];
          nx[p] -= tm1[p];
        }
        tm1.swap(tk);
        tk.swap(nx);
      }
      for (int p = 0; p <= K; ++p) c[p * 16 + t] = (double)mono[p];
    }
    double err = 0.0;
    for (int t = 1; t + 1 < w; ++t)
      for (int q = 0; q <= 2000; ++q) {
        const double f = q / 2000.0, y = 2.0 * f - 1.0;
        double v = c[K * 16 + t];
        for (int p = K - 1; p >= 0; --p) v = std::fma(v, y, c[p * 16 + t]);
        err = std::max(err, std::fabs(v - es_kernel((2.0 * (f + t) - w) / w, beta)));
      }
    if (err < best_err) { best_err = err; best = c; best_k = K; }
    if (err <= target) break;
  }
  hc = best;
  K_out = best_k;
}

void nufft_plan(NufftPlan& N, int n_f, double tol, double X, const double* w1d, cudaStream_t st) {
  N.n_f = n_f;
  N.tol = tol;
  N.X = X;
  if (w1d) N.w1d.assign(w1d, w1d + n_f);
  // w = ceil(log10(1/tol)) + 1 taps per axis; the 1e-9 guard keeps tol = 1e-10 at 11
  // taps instead of 12 when log10 lands a hair above an integer
  N.w = (int)std::ceil(std::log10(1.0 / tol) - 1e-9) + 1;
  N.w = std::max(2, std::min(N.w, MAXW));
  N.beta = 2.30 * N.w;
  N.Delta = M_PI / n_f;  // 2 pi / (sigma n_f), sigma = 2
  const double Xg = X / N.Delta;
  // exact tap range: a point at scaled offset t in [-Xg, Xg] has first tap
  // a0 = ceil(t - w/2) (spread_taps_kernel), so every tap lies in
  // [ceil(-Xg - w/2), ceil(Xg - w/2) + w - 1]; X carries a 1e-12 relative margin over the
  // half box side for the rounding of t.  (G = 29 instead of 33 at config 5's n_f = 30,
  // w = 8: 32 % fewer grid cells and DFT-stage work than a +-1-cell slack on each side.)
  N.gmin = (int)std::ceil(-Xg - 0.5 * N.w);
  const int gmax = (int)std::ceil(Xg - 0.5 * N.w) + N.w - 1;
  N.G = gmax - N.gmin + 1;
  std::vector<double> xs, ws;
  gauss_legendre(4 * N.w + 40, xs, ws);
  N.fh.assign(n_f, 0.0);
  for (int mi = 0; mi < n_f; ++mi) {
    const double m = mi - n_f / 2;
    double s = 0;
    for (size_t q = 0; q < xs.size(); ++q) {
      const double t = 0.5 * N.w * xs[q];
      s += 0.5 * N.w * ws[q] * es_kernel(xs[q], N.beta) * std::cos(m * N.Delta * t);
    }
    N.fh[mi] = s;
  }
  const int G = N.G;
  std::vector<double> Ef(2 * n_f * G), EfT(2 * n_f * G), Ee(2 * n_f * G), EeT(2 * n_f * G);
  for (int mi = 0; mi < n_f; ++mi) {
    const double m = mi - n_f / 2;
    for (int g = 0; g < G; ++g) {
      const double arg = m * (N.gmin + g) * N.Delta;
      const double c = std::cos(arg), sn = std::sin(arg);
      const double wf = (w1d ? w1d[mi] : 1.0) / N.fh[mi], we = 1.0 / N.fh[mi];
      Ef[2 * (mi * G + g)] = wf * c;
      Ef[2 * (mi * G + g) + 1] = -wf * sn;
      EfT[2 * (g * n_f + mi)] = wf * c;
      EfT[2 * (g * n_f + mi) + 1] = -wf * sn;
      Ee[2 * (g * n_f + mi)] = we * c;
      Ee[2 * (g * n_f + mi) + 1] = we * sn;
      EeT[2 * (mi * G + g)] = we * c;
      EeT[2 * (mi * G + g) + 1] = we * sn;
    }
  }
  N.Ef.alloc(Ef.size(), st);
  N.Ef.from_host(Ef.data(), Ef.size());
  N.EfT.alloc(EfT.size(), st);
  N.EfT.from_host(EfT.data(), EfT.size());
  N.Ee.alloc(Ee.size(), st);
  N.Ee.from_host(Ee.data(), Ee.size());
  N.EeT.alloc(EeT.size(), st);
  N.EeT.from_host(EeT.data(), EeT.size());
  // half-spectrum axis-0 matrices (d >= 2): rows / columns of the stored planes, the eval
  // side weighted by the Hermitian pair factor
  const int nh = n_f / 2 + 1;
  std::vector<double> EfH(2 * nh * G), EeH(2 * nh * G);
  for (int s = 0; s < nh; ++s) {
    const int mi = half_plane_mi(s, n_f, true);
    const double ws = half_plane_w(s, n_f, true);
    for (int g = 0; g < G; ++g) {
      EfH[2 * (s * G + g)] = Ef[2 * (mi * G + g)];
      EfH[2 * (s * G + g) + 1] = Ef[2 * (mi * G + g) + 1];
      EeH[2 * (g * nh + s)] = ws * Ee[2 * (g * n_f + mi)];
      EeH[2 * (g * nh + s) + 1] = ws * Ee[2 * (g * n_f + mi) + 1];
    }
  }
  N.EfH.alloc(EfH.size(), st);
  N.EfH.from_host(EfH.data(), EfH.size());
  N.EeH.alloc(EeH.size(), st);
  N.EeH.from_host(EeH.data(), EeH.size());
  std::vector<double> hc;
  es_fit(N.w, N.beta, tol, hc, N.hdeg);
  N.hc.alloc(hc.size(), st);
  N.hc.from_host(hc.data(), hc.size());
  // (pageable host -> device async copies are staged before they return: the host
  // vectors may go out of scope without a stream sync)
}

// ------------------------------------------------------------------ proxy-point plan

// worst weighted interpolation error of e^{-i m x} on [-X, X] from p Chebyshev nodes
static double proxy_error(int p, int n_f, double X, const double* w1d) {
  std::vector<double> xa(p), lam(p);
  for (int a = 0; a < p; ++a) {
    const double th = M_PI * (2 * a + 1) / (2.0 * p);
    xa[a] = X * std::cos(th);
    lam[a] = ((a & 1) ? -1.0 : 1.0) * std::sin(th);
  }
  double wmax = 0.0;
  for (int mi = 0; mi < n_f; ++mi) wmax = std::max(wmax, w1d ? std::fabs(w1d[mi]) : 1.0);
  const int ns = 3 * p + 1;
  double err = 0.0;
  std::vector<double> L(p);
  for (int q = 0; q < ns; ++q) {
    const double x = -X + 2.0 * X * (q + 0.37) / ns;
    double den = 0.0;
    for (int a = 0; a < p; ++a) {
      L[a] = lam[a] / (x - xa[a]);
      den += L[a];
    }
    for (int a = 0; a < p; ++a) L[a] /= den;
    for (int mi = 0; mi < n_f; ++mi) {
      const double m = mi - n_f / 2;
      double re = 0.0, im = 0.0;
      for (int a = 0; a < p; ++a) {
        re += L[a] * std::cos(m * xa[a]);
        im -= L[a] * std::sin(m * xa[a]);
      }
      const double dr = re - std::cos(m * x), di = im + std::sin(m * x);
      const double wgt = (w1d ? std::fabs(w1d[mi]) : 1.0) / wmax;
      err = std::max(err, wgt * std::sqrt(dr * dr + di * di));
    }
  }
  return err;
}

static void proxy_plan(NufftPlan& N, int n_f, double tol, double X, const double* w1d, cudaStream_t st) {
  N.n_f = n_f;
  N.tol = tol;
  N.X = X;
  N.w = 0;
  if (w1d) N.w1d.assign(w1d, w1d + n_f);
  int p = 4;
  while (p <= PROXY_PMAX && proxy_error(p, n_f, X, w1d) > tol) ++p;
  FGT_REQUIRE(p <= PROXY_PMAX, FGT_ERANGE, "proxy-point order beyond 48 nodes per axis");
  N.G = p;
  N.gmin = 0;
  std::vector<double> xa(p), lam(p);
  for (int a = 0; a < p; ++a) {
    const double th = M_PI * (2 * a + 1) / (2.0 * p);
    xa[a] = X * std::cos(th);
    lam[a] = ((a & 1) ? -1.0 : 1.0) * std::sin(th);
  }
  const int G = p, nh = n_f / 2 + 1;
  std::vector<double> Ef(2 * n_f * G), EfT(2 * n_f * G), EfH(2 * nh * G);
  for (int mi = 0; mi < n_f; ++mi) {
    const double m = mi - n_f / 2, wf = w1d ? w1d[mi] : 1.0;
    for (int g = 0; g < G; ++g) {
      const double c = wf * std::cos(m * xa[g]), sn = -wf * std::sin(m * xa[g]);
      Ef[2 * (mi * G + g)] = c;
      Ef[2 * (mi * G + g) + 1] = sn;
      EfT[2 * (g * n_f + mi)] = c;
      EfT[2 * (g * n_f + mi) + 1] = sn;
    }
  }
  for (int s = 0; s < nh; ++s) {
    const int mi = half_plane_mi(s, n_f, true);
    for (int g = 0; g < G; ++g) {
      EfH[2 * (s * G + g)] = Ef[2 * (mi * G + g)];
      EfH[2 * (s * G + g) + 1] = Ef[2 * (mi * G + g) + 1];
    }
  }
  N.Ef.alloc(Ef.size(), st);
  N.Ef.from_host(Ef.data(), Ef.size());
  N.EfT.alloc(EfT.size(), st);
  N.EfT.from_host(EfT.data(), EfT.size());
  N.EfH.alloc(EfH.size(), st);
  N.EfH.from_host(EfH.data(), EfH.size());
  N.cheb_x.alloc(p, st);
  N.cheb_x.from_host(xa.data(), p);
  N.cheb_lam.alloc(p, st);
  N.cheb_lam.from_host(lam.data(), p);
}

const NufftPlan& proxy_plan_cached(int n_f, double tol, double X, const double* w1d, cudaStream_t st) {
  int dev = 0;
  FGT_CUDA(cudaGetDevice(&dev));
  std::string key(reinterpret_cast<const char*>(&dev), sizeof(dev));
  key.append(reinterpret_cast<const char*>(&n_f), sizeof(n_f));
  key.append(reinterpret_cast<const char*>(&tol), sizeof(tol));
  key.append(reinterpret_cast<const char*>(&X), sizeof(X));
  if (w1d) key.append(reinterpret_cast<const char*>(w1d), sizeof(double) * n_f);
  static std::mutex mu;
  static auto* cache = new std::map<std::string, NufftPlan*>();  // process lifetime
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache->find(key);
  if (it != cache->end()) return *it->second;
  auto* p = new NufftPlan();
  proxy_plan(*p, n_f, tol, X, w1d, st);
  FGT_CUDA(cudaStreamSynchronize(st));
  (*cache)[key] = p;
  return *p;
}

namespace {
int64_t ipow(int64_t b, int e) {
  int64_t r = 1;
  while (e--) r *= b;
  return r;
}

// grid -> modes for a batch of spread grids (see nufft_form_impl)
// ---------------------------------------------------------------- fused d = 3 stages 2 + 3
// After the axis-0 stage (bgemm: X[s][g2 g3] = sum_g1 EfH[s][g1] grid[g1][g2 g3], the one
// stage that needs the whole grid of a box), the two remaining stages of a stored plane s
// run in ONE warp with the intermediate on chip:
//   stage 2  Y[m2][g3]      = sum_g2 Ef[m2][g2] X_s[g2][g3]     16 rows of m2 at a time
//   stage 3  phi[s][m2][m3] = sum_g3 Y[m2][g3] Ef[m3][g3]        Y through the warp's own
//            shared-memory rows; epilogue = the box's rephasing factor (fused translation)
// so Y (222 KB per box written and read back by the three-launch path) never reaches HBM.
// One CTA per box, 8 independent warps (no barrier after the prologue), warp w takes planes
// w, w + 8, ...: X_s (13 KB, contiguous) comes in by TMA bulk copies (one per row, into padded
// rows, completion on the warp's mbarrier), and the next plane's copy is issued as soon as
// stage 2 has consumed the current one, under stage 3.
// Complex x complex MACs as three real DMMAs (Gauss), like bgemm.  Row pitches make every
// fragment load bank-conflict free (16-byte lanes, quarter-warp phases).  Needs G <= 32 and
// n_f <= 32 (220 KB of shared memory at G = 29: config 5); larger grids keep three launches.
constexpr int DF_XP = 34;  // X row pitch in complex: 4 DF_XP = 8 (mod 32) words
constexpr int DF_EP = 36;  // Ef / Y row pitch: 4 DF_EP = 16 (mod 32) words
constexpr int DF_W = 8;    // warps per CTA

struct Dft3Args {
  const double2* x;     // (nbat, nh, G, G) complex: axis 0 already contracted
  const double2* Ef;    // (n_f, G)
  const int64_t* sl;    // expansion slot of each batch item
  double2* phi;         // (slot, nh n_f, n_f), slot stride NH
  int64_t NH;
  int G, n_f, nh;
  const double2* bp;    // optional box phases (slot, 3, n_f)
  int bp_half;
};

inline size_t dft3_smem(int G) {
  return sizeof(double2) * ((size_t)DF_W * (G * DF_XP + 16 * DF_EP) + (size_t)32 * DF_EP + 3 * 32);
}

__device__ __forceinline__ double2 df_cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

inline bool dft3_fused_ok(int G, int n_f) {
  const char* e = std::getenv("FGT_DFT_FUSED");
  return G <= 32 && n_f <= 32 && dft3_smem(G) <= 227 * 1024 && !(e && e[0] == '0');
}

__global__ void __launch_bounds__(DF_W * 32, 1) dft3_fused_kernel(Dft3Args a) {
  extern __shared__ double2 dsm[];
  const int G = a.G, n_f = a.n_f, nh = a.nh;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int lr = lane >> 2, lk = lane & 3;
  double2* Xs = dsm + (size_t)warp * (G * DF_XP + 16 * DF_EP);  // G x DF_XP
  double2* Yw = Xs + G * DF_XP;                                  // 16 x DF_EP
  double2* sE = dsm + (size_t)DF_W * (G * DF_XP + 16 * DF_EP);   // 32 x DF_EP (zero padded)
  double2* sQ = sE + 32 * DF_EP;                                 // 3 x 32 rephasing factors
  const int64_t b = blockIdx.x;
  const int plane = G * G;
  const double2 zero2 = make_double2(0.0, 0.0);
  const int64_t slot = a.sl ? a.sl[b] : b;
  // X_s of plane sp -> the warp's padded rows: one TMA bulk copy per row of G complex
  // (cp.async.bulk, SASS UBLKCP; lane g2 issues row g2), all completing on the warp's
  // mbarrier, whose phase flips once per plane
  __shared__ uint64_t s_bar[DF_W];
  const unsigned bar = (unsigned)__cvta_generic_to_shared(&s_bar[warp]);
  const unsigned row_bytes = (unsigned)(G * sizeof(double2));
  if (lane == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar));
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  __syncwarp();
  auto load_x = [&](int sp) {
    const double2* src = a.x + ((int64_t)b * nh + sp) * plane;
    // earlier generic-proxy reads of X_s are ordered before the async-proxy writes
    asm volatile("fence.proxy.async.shared::cta;\n" ::);
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(row_bytes * G));
    __syncwarp();
    for (int g2 = lane; g2 < G; g2 += 32) {
      const unsigned dst = (unsigned)__cvta_generic_to_shared(Xs + g2 * DF_XP);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
          "l"(src + (int64_t)g2 * G), "r"(row_bytes), "r"(bar)
          : "memory");
    }
  };
  auto wait_x = [&](unsigned parity) {
    unsigned done = 0;
    while (!done) {
      asm volatile(
          "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(done)
          : "r"(bar), "r"(parity)
          : "memory");
    }
  };
  if (warp < nh) load_x(warp);
  for (int e = threadIdx.x; e < 32 * DF_EP; e += blockDim.x) {
    const int m = e / DF_EP, g = e - m * DF_EP;
    sE[e] = (m < n_f && g < G) ? a.Ef[m * G + g] : zero2;
  }
  if (a.bp && threadIdx.x < 96) {
    const int ax = threadIdx.x >> 5, m = threadIdx.x & 31;
    sQ[threadIdx.x] = m < n_f ? a.bp[slot * 3 * n_f + ax * n_f + m] : zero2;
  }
  // pad columns of X (stage-2 B fragments read g3 up to 31; the copies never touch them)
  for (int e = lane; e < G * (DF_XP - G); e += 32) Xs[(e / (DF_XP - G)) * DF_XP + G + e % (DF_XP - G)] = zero2;
  __syncthreads();
  const bool q = a.bp != nullptr;
  const int nhalf = (n_f + 15) / 16;
  unsigned parity = 0;
  for (int sp = warp; sp < nh; sp += DF_W) {
    wait_x(parity);
    parity ^= 1u;
    double2* out = a.phi + slot * a.NH + (int64_t)sp * n_f * n_f;
    const double2 p0 = q ? sQ[a.bp_half ? (sp + n_f / 2) % n_f : sp] : make_double2(1.0, 0.0);
    for (int h = 0; h < nhalf; ++h) {
      double acc[2][4][4], gs[2][4][2];
      auto clear = [&]() {
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int nt = 0; nt < 4; ++nt) {
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[mt][nt][e] = 0.0;
            gs[mt][nt][0] = gs[mt][nt][1] = 0.0;
          }
      };
      auto mac = [&](const double2 (&av)[2], const double2 (&bw)[4]) {
        double bd[4], bs[4];
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
          bd[nt] = bw[nt].y - bw[nt].x;
          bs[nt] = bw[nt].x + bw[nt].y;
        }
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          const double as = av[mt].x + av[mt].y;
#pragma unroll
          for (int nt = 0; nt < 4; ++nt) {
            dmma2(acc[mt][nt][0], acc[mt][nt][1], as, bw[nt].x);
            dmma2(acc[mt][nt][2], acc[mt][nt][3], av[mt].x, bd[nt]);
            dmma2(gs[mt][nt][0], gs[mt][nt][1], av[mt].y, bs[nt]);
          }
        }
      };
      // stage 2: Y[16 h + ..][g3] = sum_g2 E[m2][g2] X_s[g2][g3]
      clear();
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int k = 4 * j + lk;
        double2 av[2], bw[4];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) av[mt] = sE[(16 * h + 8 * mt + lr) * DF_EP + k];
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) bw[nt] = k < G ? Xs[k * DF_XP + 8 * nt + lr] : zero2;
        mac(av, bw);
      }
      if (h == nhalf - 1 && sp + DF_W < nh) {
        __syncwarp();  // every lane has read X_s: the next plane may land
        load_x(sp + DF_W);
      }
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const double k1 = acc[mt][nt][i], k2 = acc[mt][nt][2 + i], k3 = gs[mt][nt][i];
            Yw[(8 * mt + lr) * DF_EP + 8 * nt + 2 * lk + i] = make_double2(k1 - k3, k1 + k2);
          }
      __syncwarp();
      // stage 3: phi[s][16 h + ..][m3] = sum_g3 Y[m2][g3] E[m3][g3]
      clear();
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int k = 4 * j + lk;
        double2 av[2], bw[4];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) av[mt] = Yw[(8 * mt + lr) * DF_EP + k];
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) bw[nt] = sE[(8 * nt + lr) * DF_EP + k];
        mac(av, bw);
      }
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        const int m2 = 16 * h + 8 * mt + lr;
        if (m2 >= n_f) continue;
        double2 p01 = p0;
        if (q) p01 = df_cmul(p0, sQ[32 + m2]);
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int m3 = 8 * nt + 2 * lk + i;
            if (m3 >= n_f) continue;
            const double k1 = acc[mt][nt][i], k2 = acc[mt][nt][2 + i], k3 = gs[mt][nt][i];
            double2 v = make_double2(k1 - k3, k1 + k2);
            if (q) v = df_cmul(df_cmul(p01, sQ[64 + m3]), v);
            out[(int64_t)m2 * n_f + m3] = v;
          }
      }
      __syncwarp();
    }
  }
}

template <int D>
void form_modes(const NufftPlan& N, PwDev& P, const double* grid, const int64_t* sl, int64_t nbat,
                GrowBuf<double>& g_t1, GrowBuf<double>& g_t2, cudaStream_t st) {
  const int G = N.G, n_f = N.n_f, nh = P.nh;
  const int64_t GD = ipow(G, D), plane = GD / G;
  // grid -> modes: separable GEMMs on the FP64 tensor cores, straight into phi[slot]
  // (d >= 2: only the nh stored axis-0 planes of the half spectrum, axis 0 contracted
  // first so the later stages run on nh planes)
  double* phi = P.phi.get();
  const int64_t NH = P.NH;
  if (D == 1) {
    bgemm<true, false, false>(gemm(N.Ef.get(), G, 0, grid, 1, G, phi, 1, NH, n_f, 1, G, (int)nbat, sl), st);
  } else if (D == 2) {
    auto t1 = g_t1.view(2 * nbat * G * n_f, st);
    // T1[g1][m2] = sum_g2 grid[g1][g2] EfT[g2][m2]
    bgemm<false, true, false>(gemm(grid, G, GD, N.EfT.get(), n_f, 0, t1.get(), n_f, (int64_t)G * n_f, G, n_f, G, (int)nbat), st);
    // phi[s][m2] = sum_g1 EfH[s][g1] T1[g1][m2]
    bgemm<true, true, false>(gemm(N.EfH.get(), G, 0, t1.get(), n_f, (int64_t)G * n_f, phi, n_f, NH, nh, n_f, G, (int)nbat, sl), st);
  } else if (dft3_fused_ok(G, n_f)) {
    auto x = g_t1.view(2 * nbat * nh * plane, st);
    // X[s][(g2 g3)] = sum_g1 EfH[s][g1] grid[g1][(g2 g3)]
    bgemm<true, false, false>(gemm(N.EfH.get(), G, 0, grid, plane, GD, x.get(), plane, nh * plane, nh, (int)plane, G, (int)nbat), st);
    Dft3Args da;
    da.x = reinterpret_cast<const double2*>(x.get());
    da.Ef = reinterpret_cast<const double2*>(N.Ef.get());
    da.sl = sl;
    da.phi = reinterpret_cast<double2*>(phi);
    da.NH = NH;
    da.G = G;
    da.n_f = n_f;
    da.nh = nh;
    da.bp = P.fused ? reinterpret_cast<const double2*>(P.bp.get()) : nullptr;
    da.bp_half = P.half;
    const size_t smem = dft3_smem(G);
    FGT_CUDA(cudaFuncSetAttribute(dft3_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    dft3_fused_kernel<<<(unsigned)nbat, DF_W * 32, smem, st>>>(da);
    FGT_LAUNCHED();
  } else {
    auto x = g_t1.view(2 * nbat * nh * plane, st);
    auto y = g_t2.view(2 * nbat * nh * n_f * G, st);
    // X[s][(g2 g3)] = sum_g1 EfH[s][g1] grid[g1][(g2 g3)]
    bgemm<true, false, false>(gemm(N.EfH.get(), G, 0, grid, plane, GD, x.get(), plane, nh * plane, nh, (int)plane, G, (int)nbat), st);
    // Y[s][m2][g3] = sum_g2 Ef[m2][g2] X[s][g2][g3]      (batch = box x s)
    bgemm<true, true, false>(gemm(N.Ef.get(), G, 0, x.get(), G, (int64_t)G * G, y.get(), G, (int64_t)n_f * G, n_f, G, G, nbat * nh), st);
    // phi[(s m2)][m3] = sum_g3 Y[(s m2)][g3] EfT[g3][m3], times the box's rephasing factor
    // e^{i k.(c_ref - c_S)} on the fused translation path (epilogue; no separate pass)
    GemmArgs g3 = gemm(y.get(), G, (int64_t)nh * n_f * G, N.EfT.get(), n_f, 0, phi, n_f, NH, nh * n_f, n_f, G, (int)nbat, sl);
    if (P.fused) {
      g3.bp = reinterpret_cast<const double2*>(P.bp.get());
      g3.bp_nf = n_f;
      g3.bp_half = P.half;
    }
    bgemm<true, true, false>(g3, st);
  }
}

template <int D>
void nufft_form_impl(const NufftPlan& N, PwDev& P, TreeDev& T, const std::vector<int64_t>& slots) {
  if (slots.empty()) return;
  cudaStream_t st = T.st;
  const int G = N.G, n_f = N.n_f, w = N.w;
  const int64_t GD = ipow(G, D);
  const int64_t plane = GD / G;
  // per-slot source counts (fetched once in pw_setup)
  const std::vector<int64_t>& scount = P.h_src;
  FGT_REQUIRE(G < 256 && G <= 64, FGT_ERANGE, "spreading grid too large (G > 64)");
  // batches bounded by ~6 GB of grid + stage buffers and 16M points (~350 B each)
  const int nh = P.nh;
  const int64_t per_box = GD * 8 + (D == 2 ? (int64_t)G * n_f * 16 : 0) +
                          (D == 3 ? (int64_t)nh * plane * 16 + (int64_t)nh * n_f * G * 16 : 0);
  const int64_t nb_max = std::max<int64_t>(1, std::min<int64_t>(1 << 20, ((int64_t)6 << 30) / per_box));
  const int CH = D == 2 ? 4096 : 2048;  // points per job
  // grid cells written by one job: a plane (d = 3), the whole grid (d = 2), a cell (d = 1)
  const int64_t job_cells = D == 3 ? plane : (D == 2 ? GD : 1);
  CubTmpBuf tmp;
  // per-batch work buffers, allocated once for the largest batch (GrowBuf)
  GrowBuf<int64_t> g_sl, g_boff, g_iota, g_perm, g_perm2;
  GrowBuf<double> g_wts, g_tt, g_qb, g_rw, g_rq, g_rw0, g_grid, g_scratch, g_t1, g_t2;
  GrowBuf<int> g_ai, g_ra, g_range;
  GrowBuf<uint64_t> g_key, g_skey;
  GrowBuf<int4> g_jobs, g_reds;
  GrowBuf<int> g_counter;
  size_t b0 = 0;
  while (b0 < slots.size()) {
    // grow the batch up to nb_max boxes and ~4M points
    int64_t nbat = 0, npts = 0;
    std::vector<int64_t> boff(1, 0);
    while (b0 + nbat < slots.size() && nbat < nb_max) {
      const int64_t n = scount[slots[b0 + nbat]];
      if (nbat > 0 && npts + n > (int64_t)16 << 20) break;
      npts += n;
      boff.push_back(npts);
      ++nbat;
    }
    auto sl_d = g_sl.view(nbat, st);
    auto boff_d = g_boff.view(nbat + 1, st);
    sl_d.from_host(slots.data() + b0, nbat);
    boff_d.from_host(boff.data(), nbat + 1);
    auto wts = g_wts.view(D == 1 ? npts * MAXW : 0, st);
    auto tt = g_tt.view(npts * D, st);
    auto qb = g_qb.view(npts, st);
    auto ai = g_ai.view(npts * D, st);
    auto key = g_key.view(npts, st);
    auto skey = g_skey.view(npts, st);
    auto iota = g_iota.view(npts, st);
    auto perm = g_perm.view(npts, st);
    WeightArgs wa;
    wa.src = T.src_sorted.get();
    wa.q = T.q_sorted.get();
    wa.center = T.center.get();
    wa.dense_ids = T.dense_ids.get();
    wa.src_start = T.src_start.get();
    wa.slots = sl_d.get();
    wa.boff = boff_d.get();
    wa.npts = npts;
    wa.nbat = nbat;
    wa.wts = wts.get();
    wa.tt = tt.get();
    wa.ai = ai.get();
    wa.qb = qb.get();
    wa.key = key.get();
    wa.sc = P.sc;
    wa.inv_delta = 1.0 / N.Delta;
    wa.beta = N.beta;
    wa.w = w;
    wa.gmin = N.gmin;
    wa.G = G;
    trace_mark(st, "form:alloc");
    spread_taps_kernel<D><<<grid_for(npts * D, 256), 256, 0, st>>>(wa);
    FGT_LAUNCHED();
    trace_mark(st, "form:taps");
    spread_keys_kernel<D><<<grid_for(npts, 256), 256, 0, st>>>(key.get(), ai.get(), npts, w);
    FGT_LAUNCHED();
    iota_i64(iota.get(), npts, st);
    const int tap_bits = D == 3 ? 16 : 8 * D;  // d = 3 key: 4 class + 6 + 6 tap bits
    int bits = tap_bits;
    while (((int64_t)1 << (bits - tap_bits)) < nbat) ++bits;
    sort_pairs_key(tmp, key.get(), skey.get(), iota.get(), perm.get(), npts, bits, st);
    // records first: the GPU builds them while the host waits for the job ranges
    BufView<double> rw{nullptr, 0, st}, rq{nullptr, 0, st}, rw0{nullptr, 0, st};
    BufView<int> ra{nullptr, 0, st};
    if (D >= 2) {
      rw = g_rw.view(npts * (D == 3 ? PEN_REC : 32), st);
      if (D != 3) rq = g_rq.view(npts, st);
      ra = g_ra.view(npts * 4, st);
      switch (w) {
#define FGT_REC(WV)                                                                                          \
  case WV:                                                                                                   \
    sort_records_kernel<D, WV><<<(unsigned)((npts + REC_PTS - 1) / REC_PTS), D * 32, 0, st>>>(              \
        perm.get(), npts, tt.get(), ai.get(), qb.get(), N.beta, N.hc.get(), N.hdeg, rw.get(), rq.get(), ra.get(), \
        rw0.get());                                                                                          \
    break;
        FGT_REC(2) FGT_REC(3) FGT_REC(4) FGT_REC(5) FGT_REC(6) FGT_REC(7) FGT_REC(8) FGT_REC(9)
        FGT_REC(10) FGT_REC(11) FGT_REC(12) FGT_REC(13) FGT_REC(14) FGT_REC(15) FGT_REC(16)
#undef FGT_REC
        default: throw Error(FGT_ERANGE, "kernel width out of range");
      }
      FGT_LAUNCHED();
    }
    const int NBP = (G + 7) / 8;  // d = 3: pencil row / column blocks
    const int64_t njob = D == 2 ? nbat : (D == 3 ? nbat * NBP : nbat * G);
    auto range = g_range.view(2 * njob, st);
    job_ranges_kernel<D><<<grid_for(njob, 256), 256, 0, st>>>(skey.get(), npts, nbat, G, w, range.get());
    FGT_LAUNCHED();
    trace_mark(st, "form:taps+sort");
    if constexpr (D == 3) {
      // pencil jobs: one per (box, b, chunk of <= PCH scanned points), x NB columns x parts,
      // built on the device (pencil_jobs_kernel) -- no host round trip.  Host-side bounds from
      // the per-box source counts: only boxes with > PCH points can split a row job.
      const int nparts = (G + PEN_PH - 1) / PEN_PH, PH = (G + nparts - 1) / nparts;
      const int per = NBP * nparts, PCH = 4096;
      int64_t extra = 0, red_bound = 0;
      for (int64_t b = 0; b < nbat; ++b) {
        const int64_t c = scount[slots[b0 + b]];
        if (c > PCH) {
          extra += NBP * ((c + PCH - 1) / PCH);
          red_bound += NBP;
        }
      }
      const int64_t job_bound = njob + extra;
      FGT_REQUIRE(job_bound < ((int64_t)1 << 30) / per, FGT_ERANGE, "too many pencil jobs");
      auto jobs_tmp = g_jobs.view(2 * job_bound, st);
      int4* jobs_sorted = jobs_tmp.get() + job_bound;
      auto reds_d = g_reds.view(std::max<int64_t>(1, red_bound), st);
      auto jkey = g_key.view(std::max<int64_t>(npts, 2 * job_bound), st);  // key/skey reused
      auto jval = g_iota.view(std::max<int64_t>(npts, job_bound), st);
      auto jperm = g_perm2.view(job_bound, st);
      auto counts = g_counter.view(3, st);
      pencil_jobs_kernel<<<1, 1024, 0, st>>>(range.get(), (int)njob, PCH, per, (int)job_bound, jobs_tmp.get(),
                                             jkey.get(), jval.get(), reds_d.get(), counts.get());
      FGT_LAUNCHED();
      sort_pairs_key(tmp, jkey.get(), jkey.get() + job_bound, jval.get(), jperm.get(), job_bound, 14, st);
      gather_jobs_kernel<<<grid_for(job_bound, 256), 256, 0, st>>>(jobs_tmp.get(), jperm.get(), counts.get(),
                                                                   jobs_sorted);
      FGT_LAUNCHED();
      auto grid = g_grid.view(nbat * GD, st);
      auto scratch = g_scratch.view(std::max<int64_t>(1, extra * per) * PEN_PH * 64, st);
      FGT_CUDA(cudaMemsetAsync(counts.get() + 2, 0, sizeof(int), st));
      PencilArgs pa;
      pa.jobs = jobs_sorted;
      pa.njobs = counts.get();
      pa.counter = counts.get() + 2;
      pa.rw = rw.get();
      pa.ra = ra.get();
      pa.grid = grid.get();
      pa.scratch = scratch.get();
      pa.w = w;
      pa.G = G;
      pa.NB = NBP;
      pa.nparts = nparts;
      pa.PH = PH;
      pa.per = per;
      // persistent CTAs: as many as fit on the device at once
      int dev_id = 0, nsm = 0;
      FGT_CUDA(cudaGetDevice(&dev_id));
      FGT_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev_id));
      // planes per dispatch: the w taps plus room for the group's a_0 spread
#define FGT_PEN(NPL)                                                                                         \
  {                                                                                                          \
    /* attribute + occupancy resolved once per device (0: unset), under a lock: the C ABI is */ \
    /* reentrant and a process may drive several GPUs from several threads */                 \
    static int per_sm_dev[64];                                                                               \
    static std::mutex per_sm_mu;                                                                             \
    int per_sm = 0;                                                                                          \
    {                                                                                                        \
      std::lock_guard<std::mutex> lock(per_sm_mu);                                                           \
      int& slot = per_sm_dev[dev_id & 63];                                                                   \
      if (slot <= 0) {                                                                                       \
        FGT_CUDA(cudaFuncSetAttribute(spread_pencil_kernel<NPL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PEN_SMEM)); \
        FGT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&slot, spread_pencil_kernel<NPL>, PEN_WARPS * 32, PEN_SMEM)); \
      }                                                                                                      \
      per_sm = slot;                                                                                         \
    }                                                                                                        \
    const unsigned nblk = (unsigned)std::max<int64_t>(1, std::min<int64_t>((int64_t)nsm * std::max(1, per_sm),       \
                                                        (job_bound * per + PEN_WARPS - 1) / PEN_WARPS));              \
    spread_pencil_kernel<NPL><<<nblk, PEN_WARPS * 32, PEN_SMEM, st>>>(pa);                                   \
  }
      {
        FGT_REQUIRE(w >= 2, FGT_ERANGE, "kernel width < 2");  // zero band >= NPL - w
        if (w <= 5) FGT_PEN(8)
        else if (w <= 9) FGT_PEN(12)
        else FGT_PEN(16)
        FGT_LAUNCHED();
      }
#undef FGT_PEN
      if (red_bound > 0) {
        pencil_reduce_kernel<<<dim3(1, (unsigned)red_bound, (unsigned)per), 256, 0, st>>>(
            scratch.get(), reds_d.get(), counts.get() + 1, NBP, nparts, PH, G, grid.get());
        FGT_LAUNCHED();
      }
      form_modes<D>(N, P, grid.get(), sl_d.get(), nbat, g_t1, g_t2, st);
      b0 += nbat;
      continue;
    }
    std::vector<int> hr(2 * njob);
    range.to_host(hr.data(), hr.size());
    FGT_CUDA(cudaStreamSynchronize(st));
    trace_mark(st, "form:ranges(sync)");
    std::vector<int4> jobs, reds;
    int nscr = 0;
    for (int64_t jid = 0; jid < njob; ++jid) {
      const int lo = hr[2 * jid], n = hr[2 * jid + 1] - lo;
      if (n <= CH) {
        jobs.push_back(make_int4((int)jid, lo, n, -1));
      } else {
        const int nc = (n + CH - 1) / CH;
        reds.push_back(make_int4((int)jid, nscr, nc, 0));
        for (int c = 0; c < nc; ++c) jobs.push_back(make_int4((int)jid, lo + c * CH, std::min(CH, n - c * CH), nscr++));
      }
    }
    auto jobs_d = g_jobs.view(jobs.size(), st);
    auto reds_d = g_reds.view(reds.size(), st);
    jobs_d.from_host(jobs.data(), jobs.size());
    if (!reds.empty()) reds_d.from_host(reds.data(), reds.size());
    auto grid = g_grid.view(nbat * GD, st);
    auto scratch = g_scratch.view((int64_t)nscr * job_cells, st);
    PlaneArgs pa;
    pa.rw = rw.get();
    pa.rq = rq.get();
    pa.ra = ra.get();
    pa.rw0 = rw0.get();
    pa.jobs = jobs_d.get();
    pa.njobs = (int)jobs.size();
    pa.perm = perm.get();
    pa.wts = wts.get();
    pa.ai = ai.get();
    pa.qb = qb.get();
    pa.grid = grid.get();
    pa.scratch = scratch.get();
    pa.w = w;
    pa.G = G;
    const unsigned nblk = (unsigned)((jobs.size() + 3) / 4);
    if constexpr (D == 1) {
      spread_line_kernel<<<nblk, 128, 0, st>>>(pa);
    } else {
      const int NB = (G + 7) / 8;
      switch (NB) {
#define FGT_TILE(NBV)                                                                          \
  case NBV:                                                                                    \
    FGT_CUDA(cudaFuncSetAttribute(spread_tile_kernel<D, NBV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TILE_SMEM)); \
    spread_tile_kernel<D, NBV><<<nblk, 128, TILE_SMEM, st>>>(pa);                              \
    break;
        FGT_TILE(1) FGT_TILE(2) FGT_TILE(3) FGT_TILE(4) FGT_TILE(5) FGT_TILE(6) FGT_TILE(7) FGT_TILE(8)
#undef FGT_TILE
        default: throw Error(FGT_ERANGE, "spreading grid too large");
      }
    }
    FGT_LAUNCHED();
    if (!reds.empty()) {
      plane_reduce_kernel<<<dim3(grid_for(job_cells, 256, 16), (unsigned)reds.size()), 256, 0, st>>>(
          scratch.get(), reds_d.get(), job_cells, 0, grid.get());
      FGT_LAUNCHED();
    }
    form_modes<D>(N, P, grid.get(), sl_d.get(), nbat, g_t1, g_t2, st);
    b0 += nbat;
  }
}

// proxy-point form of the listed P-box slots (see k_nufft.cuh)
template <int D>
void proxy_form_impl(const NufftPlan& N, PwDev& P, TreeDev& T, const std::vector<int64_t>& slots) {
  if (slots.empty()) return;
  cudaStream_t st = T.st;
  const int p = N.G, n_f = N.n_f, nh = P.nh;
  const int64_t GD = ipow(p, D), plane = GD / p;
  const std::vector<int64_t>& scount = P.h_src;
  const int64_t per_box = GD * 8 + (D == 2 ? (int64_t)p * n_f * 16 : 0) +
                          (D == 3 ? (int64_t)nh * plane * 16 + (int64_t)nh * n_f * p * 16 : 0);
  const int64_t nb_max = std::max<int64_t>(1, std::min<int64_t>(1 << 16, ((int64_t)4 << 30) / per_box));
  GrowBuf<int64_t> g_sl, g_boff;
  GrowBuf<double> g_grid, g_t1, g_t2;
  const int P8 = (p + 7) / 8;
  const int ntiles = D == 1 ? 1 : (D == 2 ? P8 : p * P8);
  const unsigned nz = (unsigned)((ntiles + 8 * PROXY_NT - 1) / (8 * PROXY_NT));
  for (size_t b0 = 0; b0 < slots.size();) {
    const int64_t nbat = std::min<int64_t>(nb_max, (int64_t)(slots.size() - b0));
    std::vector<int64_t> boff(nbat + 1, 0);
    for (int64_t b = 0; b < nbat; ++b) boff[b + 1] = boff[b] + scount[slots[b0 + b]];
    auto sl_d = g_sl.view(nbat, st);
    auto boff_d = g_boff.view(nbat + 1, st);
    sl_d.from_host(slots.data() + b0, nbat);
    boff_d.from_host(boff.data(), nbat + 1);
    auto grid = g_grid.view(nbat * GD, st);
    ProxyArgs pa;
    pa.src = T.src_sorted.get();
    pa.q = T.q_sorted.get();
    pa.center = T.center.get();
    pa.dense_ids = T.dense_ids.get();
    pa.src_start = T.src_start.get();
    pa.slots = sl_d.get();
    pa.boff = boff_d.get();
    pa.cheb_x = N.cheb_x.get();
    pa.cheb_lam = N.cheb_lam.get();
    pa.grid = grid.get();
    pa.sc = P.sc;
    pa.p = p;
    proxy_charges_kernel<D><<<dim3((unsigned)nbat, (unsigned)P8, nz), 256, 0, st>>>(pa);
    FGT_LAUNCHED();
    form_modes<D>(N, P, grid.get(), sl_d.get(), nbat, g_t1, g_t2, st);
    b0 += nbat;
  }
}

template <int D>
void nufft_eval_impl(const NufftPlan& N, PwDev& P, TreeDev& T, const std::vector<int64_t>& idx,
                     double* u_sorted) {
  if (idx.empty()) return;
  cudaStream_t st = T.st;
  const int G = N.G, n_f = N.n_f;
  const int64_t GD = ipow(G, D), plane = GD / G, NH = P.NH;
  const int nh = P.nh;
  const int64_t per_box = GD * 8 + (D == 2 ? (int64_t)G * n_f * 16 : 0) +
                          (D == 3 ? (int64_t)nh * n_f * G * 16 + (int64_t)nh * plane * 16 : 0);
  const int64_t nb_max = std::max<int64_t>(1, std::min<int64_t>(1 << 20, ((int64_t)6 << 30) / per_box));
  GrowBuf<int64_t> g_li;
  GrowBuf<double> g_grid, g_v1, g_v2;
  for (size_t b0 = 0; b0 < idx.size(); b0 += nb_max) {
    const int64_t nbat = std::min<int64_t>(nb_max, (int64_t)idx.size() - b0);
    auto li = g_li.view(nbat, st);
    li.from_host(idx.data() + b0, nbat);
    auto grid = g_grid.view(nbat * GD, st);
    const double* psi = P.psi_view();  // first stage reads psi[list[b]] through bidx
    if (D == 1) {
      // grid[g] = Re sum_m Ee[g][m] psi[m]
      bgemm<true, true, true>(gemm(N.Ee.get(), n_f, 0, psi, 1, NH, grid.get(), 1, GD, G, 1, n_f, (int)nbat, nullptr, li.get()), st);
    } else if (D == 2) {
      auto v1 = g_v1.view(2 * nbat * G * n_f, st);
      // V1[g1][m2] = sum_s EeH[g1][s] psi[s][m2]   (pair weights in EeH)
      bgemm<true, true, false>(gemm(N.EeH.get(), nh, 0, psi, n_f, NH, v1.get(), n_f, (int64_t)G * n_f, G, n_f, nh, (int)nbat, nullptr, li.get()), st);
      // grid[g1][g2] = Re sum_m2 V1[g1][m2] EeT[m2][g2]
      bgemm<true, true, true>(gemm(v1.get(), n_f, (int64_t)G * n_f, N.EeT.get(), G, 0, grid.get(), G, GD, G, G, n_f, (int)nbat), st);
    } else {
      auto v = g_v1.view(2 * nbat * nh * n_f * G, st);
      auto wv = g_v2.view(2 * nbat * nh * plane, st);
      // V[(s m2)][g3] = sum_m3 psi[(s m2)][m3] EeT[m3][g3]
      bgemm<true, true, false>(gemm(psi, n_f, NH, N.EeT.get(), G, 0, v.get(), G, (int64_t)nh * n_f * G, nh * n_f, G, n_f, (int)nbat, nullptr, nullptr, li.get()), st);
      // W[s][g2][g3] = sum_m2 Ee[g2][m2] V[s][m2][g3]      (batch = box x s)
      bgemm<true, true, false>(gemm(N.Ee.get(), n_f, 0, v.get(), G, (int64_t)n_f * G, wv.get(), G, (int64_t)G * G, G, G, n_f, nbat * nh), st);
      // grid[g1][(g2 g3)] = Re sum_s EeH[g1][s] W[s][(g2 g3)]   (pair weights in EeH)
      bgemm<true, true, true>(gemm(N.EeH.get(), nh, 0, wv.get(), plane, (int64_t)nh * plane, grid.get(), plane, GD, G, (int)plane, nh, (int)nbat), st);
    }
    InterpArgs ia;
    ia.tgt = T.tgt_sorted.get();
    ia.center = T.center.get();
    ia.psi_ids = T.psi_ids.get();
    ia.list = li.get();
    ia.tgt_start = T.tgt_start.get();
    ia.tgt_count = T.tgt_count.get();
    ia.grid = grid.get();
    ia.u = u_sorted;
    ia.sc = P.sc;
    ia.inv_delta = 1.0 / N.Delta;
    ia.beta = N.beta;
    ia.w = N.w;
    ia.gmin = N.gmin;
    ia.G = G;
    if (D == 2) {
      const size_t smem = (size_t)G * G * sizeof(double);
      switch (N.w) {
#define FGT_I2(WV)                                                                                  \
  case WV:                                                                                          \
    FGT_CUDA(cudaFuncSetAttribute(interp2_kernel<WV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    interp2_kernel<WV><<<(unsigned)nbat, 256, smem, st>>>(ia);                                      \
    break;
        FGT_I2(2) FGT_I2(3) FGT_I2(4) FGT_I2(5) FGT_I2(6) FGT_I2(7) FGT_I2(8) FGT_I2(9)
        FGT_I2(10) FGT_I2(11) FGT_I2(12) FGT_I2(13) FGT_I2(14) FGT_I2(15) FGT_I2(16)
#undef FGT_I2
        default: throw Error(FGT_ERANGE, "kernel width out of range");
      }
    } else {
      interp_kernel<D><<<(unsigned)nbat, 256, 0, st>>>(ia);
    }
    FGT_LAUNCHED();
  }
}
}  // namespace

void nufft_form(const NufftPlan& N, PwDev& P, TreeDev& T, const std::vector<int64_t>& slots) {
  if (nufft_mode() == 3) {
    const NufftPlan& X = proxy_plan_cached(N.n_f, N.tol, N.X, N.w1d.empty() ? nullptr : N.w1d.data(), T.st);
    if (T.d == 1) proxy_form_impl<1>(X, P, T, slots);
    else if (T.d == 2) proxy_form_impl<2>(X, P, T, slots);
    else proxy_form_impl<3>(X, P, T, slots);
    return;
  }
  if (T.d == 1) nufft_form_impl<1>(N, P, T, slots);
  else if (T.d == 2) nufft_form_impl<2>(N, P, T, slots);
  else nufft_form_impl<3>(N, P, T, slots);
}

void nufft_eval(const NufftPlan& N, PwDev& P, TreeDev& T, const std::vector<int64_t>& idx,
                double* u_sorted) {
  if (T.d == 1) nufft_eval_impl<1>(N, P, T, idx, u_sorted);
  else if (T.d == 2) nufft_eval_impl<2>(N, P, T, idx, u_sorted);
  else nufft_eval_impl<3>(N, P, T, idx, u_sorted);
}

}  // namespace fgt
