// GPU construction of the level-restricted point tree (Alg 1) and
// of the target-centric P/D interaction lists.
//
// Reference behaviour reproduced bit-exactly (tree.py line numbers):
//   * root: free space centre = midpoint of the bbox, side 2^l_c D0 sqrt(delta) with
//     the roundoff guard (:463-472); periodic root centre 0, side 1 (:458-461);
//   * a point's child is chosen by p_k >= centre_k of the box being split (:486-491),
//     centres from _Builder.center (:324-326) rounded op-by-op (no FMA);
//   * level-synchronous refinement of boxes with > n_s points up to l_c (:493-502);
//   * 2:1 balance (:378-403) and the dense-cutoff-leaf fix (:506-523).
// The balance / dense-fix closures are monotone, so their unique least fixpoint is
// reached by parallel rounds (every split made is forced in any closed superset);
// the box set, leaf relation and per-leaf ascending index lists therefore match the
// sequential LIFO build.  Boxes are numbered level-major, Morton within a level.
//
// Representation: each point carries its Morton code at level l_c (the path of child
// numbers it would take through every split).  A box (level l, code c) holds exactly
// the points whose code >> d(l_c-l) == c, so subtree counts are two binary searches
// in the sorted point codes.  Boxes live in one sorted array of keys (l<<58 | c).
#include <cub/cub.cuh>
#include "k_tree.cuh"

namespace fgt {

namespace {

struct CubTmp {
  DBuf<uint8_t> buf;
  void* get(size_t bytes, cudaStream_t st) {
    if (bytes > buf.size()) buf.alloc(bytes + 256, st);
    return buf.get();
  }
};

template <class T>
T read_scalar(const T* dptr, cudaStream_t st) {
  T h;
  FGT_CUDA(cudaMemcpyAsync(&h, dptr, sizeof(T), cudaMemcpyDeviceToHost, st));
  FGT_CUDA(cudaStreamSynchronize(st));
  return h;
}

struct Root {
  double low[3];
  double side;
};

// ------------------------------------------------------------------ bbox
template <int D>
__global__ void __launch_bounds__(256) bbox_partial_kernel(const double* __restrict__ a, int64_t n,
                                                           double* __restrict__ part) {
  double lo[D], hi[D];
#pragma unroll
  for (int k = 0; k < D; ++k) { lo[k] = INFINITY; hi[k] = -INFINITY; }
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int k = 0; k < D; ++k) {
      double v = a[i * D + k];
      lo[k] = fmin(lo[k], v);
      hi[k] = fmax(hi[k], v);
    }
  }
  __shared__ double s[2 * D][256];
#pragma unroll
  for (int k = 0; k < D; ++k) { s[k][threadIdx.x] = lo[k]; s[D + k][threadIdx.x] = hi[k]; }
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
#pragma unroll
      for (int k = 0; k < D; ++k) {
        s[k][threadIdx.x] = fmin(s[k][threadIdx.x], s[k][threadIdx.x + w]);
        s[D + k][threadIdx.x] = fmax(s[D + k][threadIdx.x], s[D + k][threadIdx.x + w]);
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < 2 * D; ++k) part[blockIdx.x * 2 * D + k] = s[k][0];
  }
}

void device_bbox(const double* src, int64_t ns, const double* tgt, int64_t nt, int d,
                 double* lo, double* hi, cudaStream_t st) {
  const int nblk = 296;
  DBuf<double> part(2 * nblk * 2 * d, st);
  for (int k = 0; k < d; ++k) { lo[k] = INFINITY; hi[k] = -INFINITY; }
  int used = 0;
  for (int which = 0; which < 2; ++which) {
    const double* a = which ? tgt : src;
    int64_t n = which ? nt : ns;
    if (n == 0) continue;
    double* p = part.get() + which * nblk * 2 * d;
    if (d == 1) bbox_partial_kernel<1><<<nblk, 256, 0, st>>>(a, n, p);
    else if (d == 2) bbox_partial_kernel<2><<<nblk, 256, 0, st>>>(a, n, p);
    else bbox_partial_kernel<3><<<nblk, 256, 0, st>>>(a, n, p);
    FGT_LAUNCHED();
    used |= 1 << which;
  }
  std::vector<double> h(2 * nblk * 2 * d);
  part.to_host(h.data(), h.size());
  FGT_CUDA(cudaStreamSynchronize(st));
  for (int which = 0; which < 2; ++which) {
    if (!(used >> which & 1)) continue;
    for (int b = 0; b < nblk; ++b) {
      const double* p = h.data() + (which * nblk + b) * 2 * d;
      for (int k = 0; k < d; ++k) {
        lo[k] = std::fmin(lo[k], p[k]);
        hi[k] = std::fmax(hi[k], p[d + k]);
      }
    }
  }
}

// ------------------------------------------------------------------ point codes
template <int D, class KT, class IT>
__global__ void __launch_bounds__(256) point_codes_kernel(
    const double* __restrict__ src, int64_t ns, const double* __restrict__ tgt, int64_t nt,
    int l_c, Root root, KT* __restrict__ code, IT* __restrict__ idx) {
  const int64_t ntot = ns + nt;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ntot;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double* p = (i < ns) ? src + i * D : tgt + (i - ns) * D;
    double x[D];
#pragma unroll
    for (int k = 0; k < D; ++k) x[k] = p[k];
    int64_t g[D];
#pragma unroll
    for (int k = 0; k < D; ++k) g[k] = 0;
    double s = root.side;  // side of the box being split at level l (exact halvings)
    for (int l = 0; l < l_c; ++l) {
#pragma unroll
      for (int k = 0; k < D; ++k) {
        double c = box_center_1d(root.low[k], g[k], s);
        g[k] = 2 * g[k] + (x[k] >= c ? 1 : 0);
      }
      s *= 0.5;
    }
    code[i] = (KT)morton_encode(g, D, l_c);
    idx[i] = (IT)i;
  }
}

// 32-bit sorted codes / indices -> the tree's 64-bit arrays
__global__ void widen_kernel(const uint32_t* __restrict__ k32, const int32_t* __restrict__ i32, int64_t n,
                             uint64_t* __restrict__ k64, int64_t* __restrict__ i64) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    k64[i] = k32[i];
    i64[i] = i32[i];
  }
}

// Sorted point codes with a coarse index: start[p] = first point whose code lies in the
// level-L0 cell p (codes >> sh0 == p), ncell + 1 entries.  A lower bound is then one table
// read when the value is a level-L0 cell boundary, else a binary search inside one cell
// (a few hundred points) instead of over all points.
struct PKeyIdx {
  const uint64_t* key;
  int64_t n;
  const int64_t* start;
  int sh0;
};

__device__ __forceinline__ int64_t pk_lower(const PKeyIdx& I, uint64_t v) {
  const uint64_t p = v >> I.sh0;
  int64_t lo = I.start[p];
  if ((v & ((uint64_t(1) << I.sh0) - 1)) == 0) return lo;
  int64_t hi = I.start[p + 1];
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (I.key[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__global__ void pkey_index_kernel(const uint64_t* __restrict__ key, int64_t n, int sh0, int64_t ncell,
                                  int64_t* __restrict__ start) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p <= ncell;
       p += (int64_t)gridDim.x * blockDim.x)
    start[p] = lower_bound_dev(key, n, (uint64_t)p << sh0);
}

// subtree point count of box (l, c): codes in [c << sh, (c+1) << sh)
__device__ __forceinline__ int64_t prefix_lo(const PKeyIdx& I, uint64_t c, int sh) { return pk_lower(I, c << sh); }
__device__ __forceinline__ int64_t prefix_hi(const PKeyIdx& I, uint64_t c, int sh) {
  return pk_lower(I, (c + 1) << sh);
}

// deepest existing box at level <= l containing cell `code` at level l (tree.py:107-115)
__device__ __forceinline__ int64_t find_covering_dev(const uint64_t* keys, int64_t nb, int d, int l,
                                                     uint64_t code) {
  for (int lv = l; lv >= 0; --lv) {
    int64_t i = find_dev(keys, nb, box_key(lv, code));
    if (i >= 0) return i;
    code >>= d;
  }
  return -1;
}

// neighbour cell of g at level l by offset o; returns false if outside (free space).
// Periodic: v = n div 2^l, n -= v 2^l (tree.py:186-188).
template <int D>
__device__ __forceinline__ bool neighbor_cell(const int64_t* g, const int* o, int l, bool periodic,
                                              int64_t* n, int* v) {
  const int64_t side = (int64_t)1 << l;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    int64_t c = g[k] + o[k];
    if (periodic) {
      int64_t vv = (c >= 0) ? c / side : -((-c + side - 1) / side);
      v[k] = (int)vv;
      c -= vv * side;
    } else {
      v[k] = 0;
      if (c < 0 || c >= side) return false;
    }
    n[k] = c;
  }
  return true;
}

// offsets in tree._offsets order (:419-426): axis 0 slowest, each in (-1, 0, 1)
template <int D>
__device__ __forceinline__ void offset_of(int t, int* o) {
#pragma unroll
  for (int k = D - 1; k >= 0; --k) {
    o[k] = t % 3 - 1;
    t /= 3;
  }
}

__global__ void make_children_kernel(const uint64_t* __restrict__ parents, int64_t np, int d,
                                     uint64_t* __restrict__ out) {
  const int nc = 1 << d;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < np * nc;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t p = parents[i / nc];
    out[i] = box_key(key_level(p) + 1, (key_code(p) << d) | (uint64_t)(i % nc));
  }
}

// Device-count variants for the level loop: the frontier size lives on the device, the
// launch covers a host-side capacity and entries past the count are flagged 0 / skipped.
__global__ void count_flag_dev_kernel(const uint64_t* __restrict__ keys, const int64_t* __restrict__ n_dev,
                                      int64_t cap, PKeyIdx pk, int d,
                                      int l_c, int64_t n_s, uint8_t* __restrict__ flag) {
  const int64_t n = n_dev ? (*n_dev << d) : 1;  // children of the boxes split one level up
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cap;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint8_t f = 0;
    if (i < n) {
      uint64_t k = keys[i];
      int sh = d * (l_c - key_level(k));
      uint64_t c = key_code(k);
      f = (prefix_hi(pk, c, sh) - prefix_lo(pk, c, sh)) > n_s ? 1 : 0;
    }
    flag[i] = f;
  }
}

__global__ void make_children_dev_kernel(const uint64_t* __restrict__ parents, const int64_t* __restrict__ k_dev,
                                         int64_t cap, int d, uint64_t* __restrict__ out) {
  const int nc = 1 << d;
  const int64_t n = *k_dev * nc;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n && i < cap * nc;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t p = parents[i / nc];
    out[i] = box_key(key_level(p) + 1, (key_code(p) << d) | (uint64_t)(i % nc));
  }
}

// merge of two sorted arrays with no common element: each element's rank in the other
__global__ void merge_unique_kernel(const uint64_t* __restrict__ a, int64_t na, const uint64_t* __restrict__ b,
                                    int64_t nb, uint64_t* __restrict__ out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < na + nb;
       t += (int64_t)gridDim.x * blockDim.x) {
    if (t < na) out[t + lower_bound_dev(b, nb, a[t])] = a[t];
    else out[t - na + lower_bound_dev(a, na, b[t - na])] = b[t - na];
  }
}

__global__ void leaf_flag_kernel(const uint64_t* __restrict__ keys, int64_t nb, int d,
                                 uint8_t* __restrict__ leaf) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nb;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k = keys[i];
    leaf[i] = find_dev(keys, nb, box_key(key_level(k) + 1, key_code(k) << d)) < 0 ? 1 : 0;
  }
}

// Incremental 2:1 balance round (tree.py:195-220): a leaf b at level l >= 2 forces the
// split of any leaf neighbour covering at level <= l-2.  Checked for a list of
// candidate boxes (by key), one thread per (candidate, offset); candidates that forced a
// split are marked active (their neighbourhood changed: re-checked next round).
template <int D>
__global__ void balance_cand_kernel(const uint64_t* __restrict__ keys, int64_t nb,
                                    const uint64_t* __restrict__ cand, int64_t ncand, int periodic,
                                    uint8_t* __restrict__ split, uint8_t* __restrict__ active) {
  constexpr int NOFF = D == 1 ? 3 : (D == 2 ? 9 : 27);
  for (int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; it < ncand * NOFF;
       it += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = it / NOFF;
    const int t = (int)(it - i * NOFF);
    const uint64_t key = cand[i];
    const int l = key_level(key);
    if (l < 2) continue;
    int o[D];
    offset_of<D>(t, o);
    bool self = true;
#pragma unroll
    for (int k = 0; k < D; ++k) self &= (o[k] == 0);
    if (self) continue;
    // only leaves force splits
    if (find_dev(keys, nb, box_key(l + 1, key_code(key) << D)) >= 0) continue;
    int64_t g[D];
    morton_decode(key_code(key), D, l, g);
    int64_t n[D];
    int v[D];
    if (!neighbor_cell<D>(g, o, l, periodic, n, v)) continue;
    const int64_t j = find_covering_dev(keys, nb, D, l, morton_encode(n, D, l));
    if (j < 0) continue;
    const uint64_t kj = keys[j];
    if (l - key_level(kj) >= 2 && find_dev(keys, nb, box_key(key_level(kj) + 1, key_code(kj) << D)) < 0) {
      split[j] = 1;
      active[i] = 1;
    }
  }
}

__global__ void concat_keys_kernel(const uint64_t* __restrict__ a, int64_t na, const uint64_t* __restrict__ b,
                                   int64_t nb, uint64_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < na + nb;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = i < na ? a[i] : b[i - na];
}

// dense-cutoff-leaf fix (tree.py:323-340): a level-l_c leaf with > n_s points forces
// the split of every leaf neighbour at level l_c-1.
template <int D>
__global__ void densefix_flag_kernel(const uint64_t* __restrict__ keys, int64_t nb, int64_t lo,
                                     int64_t hi, const uint8_t* __restrict__ leaf,
                                     PKeyIdx pk, int l_c,
                                     int64_t n_s, int periodic, uint8_t* __restrict__ split,
                                     int* __restrict__ any) {
  // one thread per (box, neighbour offset), as balance_cand_kernel
  constexpr int NOFF = D == 1 ? 3 : (D == 2 ? 9 : 27);
  for (int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; it < (hi - lo) * NOFF;
       it += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = lo + it / NOFF;
    const int t = (int)(it % NOFF);
    if (!leaf[i]) continue;
    uint64_t key = keys[i];
    if (key_level(key) != l_c) continue;
    int o[D];
    offset_of<D>(t, o);
    bool self = true;
#pragma unroll
    for (int k = 0; k < D; ++k) self &= (o[k] == 0);
    if (self) continue;
    uint64_t c = key_code(key);
    int64_t cnt = prefix_hi(pk, c, 0) - prefix_lo(pk, c, 0);
    if (cnt <= n_s) continue;
    int64_t g[D];
    morton_decode(c, D, l_c, g);
    int64_t n[D];
    int v[D];
    if (!neighbor_cell<D>(g, o, l_c, periodic, n, v)) continue;
    int64_t j = find_covering_dev(keys, nb, D, l_c, morton_encode(n, D, l_c));
    if (j >= 0 && leaf[j] && key_level(keys[j]) == l_c - 1) {
      split[j] = 1;
      *any = 1;
    }
  }
}

__global__ void level_offsets_kernel(const uint64_t* __restrict__ keys, int64_t nb, int nlev,
                                     int64_t* __restrict__ off) {
  int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l <= nlev) off[l] = lower_bound_dev(keys, nb, box_key(l, 0));
}

// Per-box finalisation: the Tree fields (tree.py:53-71) + subtree counts.
template <int D>
__global__ void finalize_boxes_kernel(const uint64_t* __restrict__ keys, int64_t nb,
                                      PKeyIdx pk,
                                      const int64_t* __restrict__ srcpre, int l_c, Root root,
                                      int32_t* __restrict__ level, int64_t* __restrict__ parent,
                                      int64_t* __restrict__ children, int64_t* __restrict__ coords,
                                      uint8_t* __restrict__ is_leaf, int64_t* __restrict__ npoints,
                                      int64_t* __restrict__ scount, int64_t* __restrict__ tcount,
                                      double* __restrict__ center) {
  constexpr int NC = 1 << D;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nb;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t key = keys[i];
    int l = key_level(key);
    uint64_t c = key_code(key);
    level[i] = l;
    int64_t g[D];
    morton_decode(c, D, l, g);
    double s = root.side;
    for (int t = 0; t < l; ++t) s *= 0.5;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      coords[i * D + k] = g[k];
      center[i * D + k] = box_center_1d(root.low[k], g[k], s);
    }
    parent[i] = l > 0 ? find_dev(keys, nb, box_key(l - 1, c >> D)) : -1;
    int64_t c0 = find_dev(keys, nb, box_key(l + 1, c << D));
#pragma unroll
    for (int t = 0; t < NC; ++t) children[i * NC + t] = c0 >= 0 ? c0 + t : -1;
    is_leaf[i] = c0 < 0;
    int sh = D * (l_c - l);
    int64_t lo = prefix_lo(pk, c, sh), hi = prefix_hi(pk, c, sh);
    npoints[i] = hi - lo;
    int64_t sc = srcpre[hi] - srcpre[lo];
    scount[i] = c0 < 0 ? sc : 0;
    tcount[i] = c0 < 0 ? (hi - lo - sc) : 0;
  }
}

__global__ void source_flag_kernel(const int64_t* __restrict__ pidx, int64_t npts, int64_t ns,
                                   int64_t* __restrict__ flag) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= npts;
       i += (int64_t)gridDim.x * blockDim.x)
    flag[i] = (i < npts && pidx[i] < ns) ? 1 : 0;
}

// leaf of every point (the deepest box containing its l_c cell), scattered to the
// original (combined) index, so a stable sort by leaf keeps ascending indices
// Leaves are contiguous ranges of the Morton-sorted points: each non-empty leaf marks its
// first point (two binary searches per leaf instead of one covering search per point);
// a fill-forward scan then gives every sorted point its leaf.
__global__ void iota_kernel(int64_t* a, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    a[i] = i;
}

// complete trees: stable partition of the code-sorted points into sources / targets with
// their leaf (the level-l_c box lc_off + code)
__global__ void partition_sorted_kernel(const uint64_t* __restrict__ pkey, const int64_t* __restrict__ pidx,
                                        int64_t np, int64_t ns, const int64_t* __restrict__ srcpre,
                                        int64_t lc_off, int64_t* __restrict__ src_perm,
                                        int64_t* __restrict__ leaf_src, int64_t* __restrict__ tgt_perm,
                                        int64_t* __restrict__ leaf_tgt) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < np;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = pidx[i], leaf = lc_off + (int64_t)pkey[i], k = srcpre[i];
    if (p < ns) {
      src_perm[k] = p;
      leaf_src[k] = leaf;
    } else {
      tgt_perm[i - k] = p - ns;
      leaf_tgt[i - k] = leaf;
    }
  }
}

// general trees: stable partition of the code-sorted points into sources / targets (the
// leaves' runs stay contiguous and in Morton order)
__global__ void partition_points_kernel(const int64_t* __restrict__ pidx, int64_t np, int64_t ns,
                                        const int64_t* __restrict__ srcpre, int64_t* __restrict__ seq_src,
                                        int64_t* __restrict__ seq_tgt) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < np;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = pidx[i], k = srcpre[i];
    if (p < ns) seq_src[k] = p;
    else seq_tgt[i - k] = p - ns;
  }
}

// per leaf: its sorted-point range [lo, hi) (a leaf covers a contiguous code range) mapped
// to the partitioned source / target sequences; empty ranges for the other boxes
__global__ void leaf_ranges_kernel(const uint64_t* __restrict__ keys, const uint8_t* __restrict__ is_leaf,
                                   int64_t nb, PKeyIdx pk, int d, int l_c, const int64_t* __restrict__ srcpre,
                                   int64_t* __restrict__ src_start, int64_t* __restrict__ src_end,
                                   int64_t* __restrict__ tgt_start, int64_t* __restrict__ tgt_end) {
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb;
       b += (int64_t)gridDim.x * blockDim.x) {
    int64_t s0 = 0, s1 = 0, t0 = 0, t1 = 0;
    bool fine = false;
    if (is_leaf[b]) {
      const uint64_t k = keys[b];
      fine = key_level(k) == l_c;
      const int sh = d * (l_c - key_level(k));
      const int64_t lo = prefix_lo(pk, key_code(k), sh), hi = prefix_hi(pk, key_code(k), sh);
      s0 = srcpre[lo];
      s1 = srcpre[hi];
      t0 = lo - s0;
      t1 = hi - s1;
    }
    src_start[b] = s0;
    tgt_start[b] = t0;
    // sort segments: only coarse leaves (< l_c: at most n_s points) span several codes; a
    // level-l_c leaf is one code, already in ascending index order
    src_end[b] = fine ? s0 : s1;
    tgt_end[b] = fine ? t0 : t1;
  }
}

__global__ void leaf_start_kernel(const int64_t* __restrict__ sorted_leaf, int64_t n,
                                  const uint8_t* __restrict__ is_leaf, int64_t nb,
                                  int64_t* __restrict__ start) {
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb;
       b += (int64_t)gridDim.x * blockDim.x)
    start[b] = is_leaf[b] ? lower_bound_dev(sorted_leaf, n, b) : 0;
}

__global__ void lc_target_stats_kernel(const int32_t* __restrict__ level, const uint8_t* __restrict__ leaf,
                                       const int64_t* __restrict__ tcount, int64_t nb, int l_c,
                                       int64_t* __restrict__ out) {
  unsigned long long nl = 0, nt = 0;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x)
    if (leaf[b] && level[b] == l_c && tcount[b] > 0) {
      ++nl;
      nt += (unsigned long long)tcount[b];
    }
  if (nl) {
    atomicAdd(reinterpret_cast<unsigned long long*>(out), nl);
    atomicAdd(reinterpret_cast<unsigned long long*>(out + 1), nt);
  }
}

__global__ void dense_flag_kernel(const int32_t* __restrict__ level, const uint8_t* __restrict__ leaf,
                                  const int64_t* __restrict__ npoints, int64_t nb, int l_c,
                                  int64_t n_s, uint8_t* __restrict__ flag) {
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb;
       b += (int64_t)gridDim.x * blockDim.x)
    flag[b] = (leaf[b] && level[b] == l_c && npoints[b] > n_s) ? 1 : 0;
}

__global__ void dense_slot_dev_kernel(const int64_t* __restrict__ ids, const int64_t* __restrict__ n_dev,
                                      int64_t cap, int64_t* __restrict__ slot) {
  const int64_t n = *n_dev;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n && i < cap;
       i += (int64_t)gridDim.x * blockDim.x)
    slot[ids[i]] = i;
}

__global__ void fill_i64_kernel(int64_t* a, int64_t n, int64_t v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    a[i] = v;
}



// Box-set state during construction.
struct BoxSet {
  DBuf<uint64_t> keys;
  int64_t n = 0;
};


// Split the boxes flagged in `flag` (aligned with keys[lo, lo+n)): append their 2^d
// children and re-sort.  Returns the number of boxes split.
// counts (optional): a 2-element device buffer whose slot 1 holds another count computed
// earlier on the stream; it is read back with the split count in the same round trip
// (*extra_out).
int64_t split_flagged(BoxSet& B, int64_t lo, int64_t n, const uint8_t* flag, int d, CubTmp& tmp,
                      cudaStream_t st, DBuf<uint64_t>* kids_out = nullptr, int64_t* counts = nullptr,
                      int64_t* extra_out = nullptr) {
  if (n == 0) return 0;
  DBuf<uint64_t> sel(n, st);
  DBuf<int64_t> nsel_own;
  if (!counts) nsel_own.alloc(1, st);
  int64_t* nsel = counts ? counts : nsel_own.get();
  size_t bytes = 0;
  FGT_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, B.keys.get() + lo, flag, sel.get(), nsel, (int)n, st));
  FGT_CUDA(cub::DeviceSelect::Flagged(tmp.get(bytes, st), bytes, B.keys.get() + lo, flag, sel.get(), nsel, (int)n, st));
  count_launch();
  int64_t k;
  if (counts) {
    int64_t h[2];
    FGT_CUDA(cudaMemcpyAsync(h, counts, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    FGT_CUDA(cudaStreamSynchronize(st));
    k = h[0];
    if (extra_out) *extra_out = h[1];
  } else {
    k = read_scalar(nsel, st);
  }
  if (k == 0) return 0;
  const int64_t nc = (int64_t)k << d;
  // the children of the (sorted, stably selected) flagged leaves are sorted and new: merge
  DBuf<uint64_t> kids(nc, st), grown(B.n + nc, st);
  make_children_kernel<<<grid_for(nc, 256), 256, 0, st>>>(sel.get(), k, d, kids.get());
  FGT_LAUNCHED();
  merge_unique_kernel<<<grid_for(B.n + nc, 256), 256, 0, st>>>(B.keys.get(), B.n, kids.get(), nc, grown.get());
  FGT_LAUNCHED();
  B.keys = std::move(grown);
  B.n += nc;
  if (kids_out) *kids_out = std::move(kids);
  return k;
}

// 2:1 balance to its fixpoint.  Round 1 checks every candidate; later rounds only the
// boxes whose neighbourhood changed: the children just created and the leaves that forced
// a split (a violation needs a fine leaf next to a coarse one, so any new one involves a
// new box or a leaf whose covering neighbour was just split).  One host round trip per
// round (the split count doubles as "changed").  cand == nullptr: all boxes.
template <int D>
void balance_rounds(BoxSet& B, int periodic, CubTmp& tmp, cudaStream_t st, const DBuf<uint64_t>* first = nullptr) {
  DBuf<uint64_t> cand;
  int64_t ncand;
  if (first) {
    ncand = first->size();
    cand.alloc(ncand, st);
    if (ncand) FGT_CUDA(cudaMemcpyAsync(cand.get(), first->get(), ncand * sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
  } else {
    ncand = B.n;
    cand.alloc(ncand, st);
    FGT_CUDA(cudaMemcpyAsync(cand.get(), B.keys.get(), ncand * sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
  }
  for (int round = 0; round < 4096; ++round) {
    if (ncand == 0) return;
    DBuf<uint8_t> split(B.n, st), active(ncand, st);
    split.zero();
    active.zero();
    balance_cand_kernel<D><<<grid_for(ncand * 27, 128), 128, 0, st>>>(B.keys.get(), B.n, cand.get(), ncand,
                                                                      periodic, split.get(), active.get());
    FGT_LAUNCHED();
    // active candidates, selected before the key array grows
    DBuf<uint64_t> act(ncand, st);
    DBuf<int64_t> counts(2, st);  // split count, active count: one read-back per round
    size_t bytes = 0;
    FGT_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, cand.get(), active.get(), act.get(), counts.get() + 1, (int)ncand, st));
    FGT_CUDA(cub::DeviceSelect::Flagged(tmp.get(bytes, st), bytes, cand.get(), active.get(), act.get(), counts.get() + 1, (int)ncand, st));
    count_launch();
    DBuf<uint64_t> kids;
    int64_t na = 0;
    const int64_t k = split_flagged(B, 0, B.n, split.get(), D, tmp, st, &kids, counts.get(), &na);
    if (k == 0) return;
    const int64_t nk = kids.size();
    DBuf<uint64_t> next(nk + na, st);
    concat_keys_kernel<<<grid_for(nk + na, 256), 256, 0, st>>>(kids.get(), nk, act.get(), na, next.get());
    FGT_LAUNCHED();
    cand = std::move(next);
    ncand = nk + na;
  }
  throw Error(FGT_ECUDA, "tree balance did not converge");
}

__global__ void dense_src_kernel(const int64_t* __restrict__ ids, const int64_t* __restrict__ n_dev,
                                 const int64_t* __restrict__ src_count, int64_t cap, int64_t* __restrict__ out) {
  const int64_t n = *n_dev;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n && i < cap;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = src_count[ids[i]];
}

// Per-leaf ascending lists of a general tree (see build_tree_impl): src_perm / tgt_perm = the
// leaf-partitioned indices, with the coarse leaves' runs sorted by original index (CUB
// segmented sort; level-l_c leaves are empty segments and keep the partitioned order).
// need_src / need_tgt ((nb) flags, multi-GPU shares): only the flagged leaves are sorted;
// the others keep the partitioned order (still a permutation, never read in leaf order).
__global__ void restrict_segments_kernel(const int64_t* __restrict__ start, int64_t* __restrict__ end,
                                         const uint8_t* __restrict__ need, int64_t nb) {
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x)
    if (!need[b]) end[b] = start[b];
}

}  // namespace

void order_leaf_points(TreeDev& T, const uint8_t* need_src, const uint8_t* need_tgt) {
  if (!T.order_pending) return;
  cudaStream_t st = T.st;
  CubTmp tmp;
  for (int which = 0; which < 2; ++which) {
    const int64_t n = which ? T.nt : T.ns;
    if (n == 0) continue;
    const int64_t* kin = which ? T.seq_tgt.get() : T.seq_src.get();
    int64_t* kout = which ? T.tgt_perm.get() : T.src_perm.get();
    const int64_t* beg = which ? T.tgt_start.get() : T.src_start.get();
    int64_t* end = which ? T.tgt_end.get() : T.src_end.get();
    const uint8_t* need = which ? need_tgt : need_src;
    if (need) {
      restrict_segments_kernel<<<grid_for(T.nb, 256), 256, 0, st>>>(beg, end, need, T.nb);
      FGT_LAUNCHED();
    }
    FGT_CUDA(cudaMemcpyAsync(kout, kin, n * sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
    size_t bytes = 0;
    FGT_CUDA(cub::DeviceSegmentedSort::SortKeys(nullptr, bytes, kin, kout, (int)n, (int)T.nb, beg, end, st));
    FGT_CUDA(cub::DeviceSegmentedSort::SortKeys(tmp.get(bytes, st), bytes, kin, kout, (int)n, (int)T.nb, beg, end, st));
    count_launch();
  }
  T.seq_src.release();
  T.seq_tgt.release();
  T.src_end.release();
  T.tgt_end.release();
  T.order_pending = false;
}

namespace {
template <int D>
void build_tree_impl(TreeDev& T, const double* src, int64_t ns, const double* tgt, int64_t nt,
                     const fgt_tree_params& tp, cudaStream_t st) {
  T.st = st;
  T.d = D;
  T.ns = ns;
  T.nt = nt;
  T.ntot = ns + nt;
  T.n_s = tp.n_s;
  T.periodic = tp.periodic;
  FGT_REQUIRE(T.ntot > 0, FGT_EINVAL, "need at least one source or target");
  FGT_REQUIRE(tp.n_s >= 1 || tp.periodic == 2, FGT_EINVAL, "n_s must be >= 1");
  FGT_REQUIRE(tp.periodic >= 0 && tp.periodic <= 2, FGT_EINVAL, "periodic must be 0, 1 or 2");
  FGT_REQUIRE(T.ntot < ((int64_t)1 << 31), FGT_ERANGE, "more than 2^31 points");

  // ---- root and cutoff level (tree.py:275-289, cutoff_level :24-50)
  if (tp.periodic == 2) {
    // root Fourier-series regime: the unit cell is the only box
    for (int k = 0; k < D; ++k) T.root_center[k] = 0.0;
    T.root_side = 1.0;
    T.l_c = 0;
    T.periodic = 0;  // the series carries every image: no image neighbours
  } else if (tp.periodic) {
    for (int k = 0; k < D; ++k) T.root_center[k] = 0.0;
    T.root_side = 1.0;
    T.l_c = tp.l_c_periodic;
  } else {
    double lo[3], hi[3];
    device_bbox(src, ns, tgt, nt, D, lo, hi, st);
    trace_mark(st, "tree:bbox(sync)");
    double spread = 0.0;
    for (int k = 0; k < D; ++k) {
      T.root_center[k] = 0.5 * (lo[k] + hi[k]);
      double e = hi[k] - lo[k];
      spread = (k == 0) ? e : std::fmax(spread, e);
    }
    const double cut = tp.D0 * std::sqrt(tp.delta);
    int l_c;
    if (spread <= cut) l_c = 0;
    else l_c = std::min((int)std::ceil(std::log2(spread / cut) - 1e-12), 30);
    double side = std::ldexp(tp.D0, l_c) * std::sqrt(tp.delta);
    if (side < spread) { l_c += 1; side *= 2.0; }
    T.l_c = l_c;
    T.root_side = side;
  }
  for (int k = 0; k < D; ++k) T.root_low[k] = T.root_center[k] - 0.5 * T.root_side;
  FGT_REQUIRE(D * T.l_c <= 57, FGT_ERANGE, "cutoff level too deep for 64-bit Morton keys");
  const int l_c = T.l_c;
  Root root;
  for (int k = 0; k < 3; ++k) root.low[k] = k < D ? T.root_low[k] : 0.0;
  root.side = T.root_side;

  // ---- point codes, stable radix sort
  const int64_t np = T.ntot;
  CubTmp tmp;
  if (D * l_c > 0 && D * l_c <= 32) {
    // codes fit 32 bits (and indices 31): sort 8-byte pairs instead of 16-byte ones
    DBuf<uint32_t> code(np, st), scode(np, st);
    DBuf<int32_t> idx(np, st), sidx(np, st);
    point_codes_kernel<D><<<grid_for(np, 256), 256, 0, st>>>(src, ns, tgt, nt, l_c, root, code.get(), idx.get());
    FGT_LAUNCHED();
    size_t bytes = 0;
    FGT_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, code.get(), scode.get(), idx.get(), sidx.get(), (int)np, 0, D * l_c, st));
    FGT_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(bytes, st), bytes, code.get(), scode.get(), idx.get(), sidx.get(), (int)np, 0, D * l_c, st));
    count_launch();
    T.pkey.alloc(np, st);
    T.pidx.alloc(np, st);
    widen_kernel<<<grid_for(np, 256), 256, 0, st>>>(scode.get(), sidx.get(), np, T.pkey.get(), T.pidx.get());
    FGT_LAUNCHED();
  } else {
    DBuf<uint64_t> code(np, st);
    DBuf<int64_t> idx(np, st);
    point_codes_kernel<D><<<grid_for(np, 256), 256, 0, st>>>(src, ns, tgt, nt, l_c, root, code.get(), idx.get());
    FGT_LAUNCHED();
    if (D * l_c > 0) {
      T.pkey.alloc(np, st);
      T.pidx.alloc(np, st);
      size_t bytes = 0;
      FGT_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, code.get(), T.pkey.get(), idx.get(), T.pidx.get(), (int)np, 0, D * l_c, st));
      FGT_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(bytes, st), bytes, code.get(), T.pkey.get(), idx.get(), T.pidx.get(), (int)np, 0, D * l_c, st));
      count_launch();
    } else {
      T.pkey = std::move(code);
      T.pidx = std::move(idx);
    }
  }
  // coarse index of the sorted codes (level L0 = min(l_c, 15 / D) cells)
  const int L0 = std::min(l_c, 15 / D);
  const int sh0 = D * (l_c - L0);
  const int64_t ncell = (int64_t)1 << (D * L0);
  T.pstart.alloc(ncell + 1, st);
  pkey_index_kernel<<<grid_for(ncell + 1, 256), 256, 0, st>>>(T.pkey.get(), np, sh0, ncell, T.pstart.get());
  FGT_LAUNCHED();
  const PKeyIdx pk{T.pkey.get(), np, T.pstart.get(), sh0};

  // ---- level-synchronous refinement (tree.py:310-319).  The frontier of level l is a
  // sorted key array; the children of its split boxes (consecutive codes) form the next
  // sorted frontier, so the level-major box array is their concatenation (no re-sort).
  // Frontier sizes stay on the device (capacities bound the launches: the boxes split at
  // one level are disjoint and hold > n_s points each), so the whole descent costs one
  // host round trip instead of one per level.
  BoxSet B;
  bool complete = false;
  {
    std::vector<DBuf<uint64_t>> levels;
    std::vector<int64_t> cap;
    levels.emplace_back(1, st);
    const uint64_t k0 = box_key(0, 0);
    levels.back().from_host(&k0, 1);
    cap.push_back(1);
    DBuf<int64_t> nsel(std::max(l_c, 1), st);  // boxes split at level l
    const int64_t split_cap = np / (T.n_s + 1);
    for (int l = 0; l < l_c; ++l) {
      const int64_t fn = cap.back();
      const int64_t kc = std::min<int64_t>(fn, split_cap);
      if (kc == 0) break;
      DBuf<uint8_t> flag(fn, st);
      count_flag_dev_kernel<<<grid_for(fn, 256), 256, 0, st>>>(levels.back().get(), l ? nsel.get() + (l - 1) : nullptr,
                                                               fn, pk, D, l_c, T.n_s, flag.get());
      FGT_LAUNCHED();
      DBuf<uint64_t> sel(fn, st);
      size_t bytes = 0;
      FGT_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, levels.back().get(), flag.get(), sel.get(), nsel.get() + l, (int)fn, st));
      FGT_CUDA(cub::DeviceSelect::Flagged(tmp.get(bytes, st), bytes, levels.back().get(), flag.get(), sel.get(), nsel.get() + l, (int)fn, st));
      count_launch();
      levels.emplace_back(kc << D, st);
      make_children_dev_kernel<<<grid_for(kc << D, 256), 256, 0, st>>>(sel.get(), nsel.get() + l, kc, D, levels.back().get());
      FGT_LAUNCHED();
      cap.push_back(kc << D);
    }
    std::vector<int64_t> hsel(cap.size() - 1);
    trace_mark(st, "tree:descent");
    if (!hsel.empty()) {
      nsel.to_host(hsel.data(), hsel.size());
      FGT_CUDA(cudaStreamSynchronize(st));
    }
    trace_mark(st, "tree:descent(sync)");
    std::vector<int64_t> lsize(1, 1);
    for (int64_t k : hsel) {
      if (k == 0) break;
      lsize.push_back(k << D);
    }
    // complete tree: every box of every level < l_c was split (e.g. uniform points), so all
    // leaves sit at l_c and no balance or dense-fix split can follow
    complete = (int)lsize.size() == l_c + 1;
    for (int l = 0; complete && l < l_c; ++l) complete = hsel[l] == lsize[l];
    int64_t tot = 0;
    for (int64_t v : lsize) tot += v;
    B.keys.alloc(tot, st);
    B.n = tot;
    int64_t off = 0;
    for (size_t l = 0; l < lsize.size(); ++l) {  // levels past the first empty one stay unused
      FGT_CUDA(cudaMemcpyAsync(B.keys.get() + off, levels[l].get(), lsize[l] * sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
      off += lsize[l];
    }
  }

  // ---- balance + dense-cutoff-leaf fix to the joint fixpoint (tree.py:321-340)
  balance_rounds<D>(B, tp.periodic, tmp, st);
  trace_mark(st, "tree:balance");
  if (l_c >= 1) {
    DBuf<int> any(1, st);
    for (int round = 0; round < 4096; ++round) {
      DBuf<uint8_t> leaf(B.n, st), split(B.n, st);
      split.zero();
      leaf_flag_kernel<<<grid_for(B.n, 256), 256, 0, st>>>(B.keys.get(), B.n, D, leaf.get());
      FGT_LAUNCHED();
      densefix_flag_kernel<D><<<grid_for(B.n * 27, 128), 128, 0, st>>>(
          B.keys.get(), B.n, 0, B.n, leaf.get(), pk, l_c, T.n_s, tp.periodic,
          split.get(), any.get());
      FGT_LAUNCHED();
      DBuf<uint64_t> kids;
      if (split_flagged(B, 0, B.n, split.get(), D, tmp, st, &kids) == 0) break;
      balance_rounds<D>(B, tp.periodic, tmp, st, &kids);
    }
  }

  // ---- finalise boxes
  trace_mark(st, "tree:densefix");
  const int64_t nb = B.n;
  T.nb = nb;
  // level offsets (l_c + 2), dense-box count, leaf count: one host round trip at the end
  DBuf<int64_t> fin(l_c + 6, st);  // + (level-l_c leaves with targets, their targets)
  level_offsets_kernel<<<1, 64, 0, st>>>(B.keys.get(), B.n, l_c + 1, fin.get());
  FGT_LAUNCHED();
  T.bkey = std::move(B.keys);

  DBuf<int64_t> srcpre(np + 1, st);
  {
    DBuf<int64_t> flag(np + 1, st);
    source_flag_kernel<<<grid_for(np + 1, 256), 256, 0, st>>>(T.pidx.get(), np, ns, flag.get());
    FGT_LAUNCHED();
    size_t bytes = 0;
    FGT_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, flag.get(), srcpre.get(), (int)(np + 1), st));
    FGT_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(bytes, st), bytes, flag.get(), srcpre.get(), (int)(np + 1), st));
    count_launch();
  }
  T.level.alloc(nb, st);
  T.parent.alloc(nb, st);
  T.children.alloc(nb << D, st);
  T.coords.alloc(nb * D, st);
  T.is_leaf.alloc(nb, st);
  T.n_points.alloc(nb, st);
  T.src_count.alloc(nb, st);
  T.tgt_count.alloc(nb, st);
  T.center.alloc(nb * D, st);
  finalize_boxes_kernel<D><<<grid_for(nb, 128), 128, 0, st>>>(
      T.bkey.get(), nb, pk, srcpre.get(), l_c, root, T.level.get(), T.parent.get(),
      T.children.get(), T.coords.get(), T.is_leaf.get(), T.n_points.get(), T.src_count.get(),
      T.tgt_count.get(), T.center.get());
  FGT_LAUNCHED();

  // ---- per-point leaves, stable sorts -> src_perm / tgt_perm (tree.py:350-381)
  if (complete && l_c > 0) {
    // Complete tree: the leaf of sorted point i is the level-l_c box level_off(l_c) + its
    // code, and the code sort (stable in the combined index) already lists every leaf's
    // sources and then its targets in ascending original index -- a stable partition of
    // the sorted points replaces the scatter and the two leaf sorts.
    int64_t lc_off = 0;
    for (int l = 0; l < l_c; ++l) lc_off += (int64_t)1 << (D * l);
    T.src_perm.alloc(ns, st);
    T.tgt_perm.alloc(nt, st);
    T.src_start.alloc(nb, st);
    T.tgt_start.alloc(nb, st);
    DBuf<int64_t> leaf_src(ns, st), leaf_tgt(nt, st);
    partition_sorted_kernel<<<grid_for(np, 256), 256, 0, st>>>(T.pkey.get(), T.pidx.get(), np, ns, srcpre.get(), lc_off,
                                                               T.src_perm.get(), leaf_src.get(), T.tgt_perm.get(),
                                                               leaf_tgt.get());
    FGT_LAUNCHED();
    leaf_start_kernel<<<grid_for(nb, 256), 256, 0, st>>>(leaf_src.get(), ns, T.is_leaf.get(), nb, T.src_start.get());
    FGT_LAUNCHED();
    leaf_start_kernel<<<grid_for(nb, 256), 256, 0, st>>>(leaf_tgt.get(), nt, T.is_leaf.get(), nb, T.tgt_start.get());
    FGT_LAUNCHED();
  } else {
    // General tree: every leaf covers a contiguous range of the code-sorted points, so a
    // stable source / target partition keeps each leaf's points contiguous (leaves in Morton
    // order); a segmented sort by original index then gives the reference's ascending
    // per-leaf lists (tree.py:350-381) without a scatter or a full re-sort.
    T.src_perm.alloc(ns, st);
    T.tgt_perm.alloc(nt, st);
    T.src_start.alloc(nb, st);
    T.tgt_start.alloc(nb, st);
    T.seq_src.alloc(ns, st);
    T.seq_tgt.alloc(nt, st);
    T.src_end.alloc(nb, st);
    T.tgt_end.alloc(nb, st);
    partition_points_kernel<<<grid_for(np, 256), 256, 0, st>>>(T.pidx.get(), np, ns, srcpre.get(), T.seq_src.get(),
                                                               T.seq_tgt.get());
    FGT_LAUNCHED();
    leaf_ranges_kernel<<<grid_for(nb, 256), 256, 0, st>>>(T.bkey.get(), T.is_leaf.get(), nb, pk, D, l_c,
                                                          srcpre.get(), T.src_start.get(), T.src_end.get(),
                                                          T.tgt_start.get(), T.tgt_end.get());
    FGT_LAUNCHED();
    // the ascending per-leaf order: now, or (multi-GPU shares) after the share is planned and
    // for the rank's own leaves only
    T.order_pending = true;
    if (!T.defer_order) order_leaf_points(T, nullptr, nullptr);
  }

  // ---- P-boxes: leaves at l_c with > n_s points
  {
    DBuf<uint8_t> flag(nb, st);
    dense_flag_kernel<<<grid_for(nb, 256), 256, 0, st>>>(T.level.get(), T.is_leaf.get(), T.n_points.get(), nb, l_c, T.n_s, flag.get());
    FGT_LAUNCHED();
    DBuf<int64_t> iota(nb, st), sel(nb, st);
    int64_t* nsel = fin.get() + l_c + 2;
    iota_kernel<<<grid_for(nb, 256), 256, 0, st>>>(iota.get(), nb);
    FGT_LAUNCHED();
    size_t bytes = 0;
    FGT_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, iota.get(), flag.get(), sel.get(), nsel, (int)nb, st));
    FGT_CUDA(cub::DeviceSelect::Flagged(tmp.get(bytes, st), bytes, iota.get(), flag.get(), sel.get(), nsel, (int)nb, st));
    count_launch();
    T.dense_slot.alloc(nb, st);
    fill_i64_kernel<<<grid_for(nb, 256), 256, 0, st>>>(T.dense_slot.get(), nb, -1);
    FGT_LAUNCHED();
    dense_slot_dev_kernel<<<grid_for(nb, 256), 256, 0, st>>>(sel.get(), nsel, nb, T.dense_slot.get());
    FGT_LAUNCHED();
    // source count of every P-box (the form's per-box path choice), read back with the
    // finalize round trip below (capacity nb; the first n_dense entries are used)
    DBuf<int64_t> dsrc(nb, st);
    dense_src_kernel<<<grid_for(nb, 256), 256, 0, st>>>(sel.get(), nsel, T.src_count.get(), nb, dsrc.get());
    FGT_LAUNCHED();
    T.dense_ids = std::move(sel);  // capacity nb, first n_dense entries used
    // leaf count
    size_t b2 = 0;
    FGT_CUDA(cub::DeviceReduce::Sum(nullptr, b2, T.is_leaf.get(), fin.get() + l_c + 3, (int)nb, st));
    FGT_CUDA(cub::DeviceReduce::Sum(tmp.get(b2, st), b2, T.is_leaf.get(), fin.get() + l_c + 3, (int)nb, st));
    count_launch();
    // level-l_c target leaves and their targets (the translation path choice)
    FGT_CUDA(cudaMemsetAsync(fin.get() + l_c + 4, 0, 2 * sizeof(int64_t), st));
    lc_target_stats_kernel<<<grid_for(nb, 256), 256, 0, st>>>(T.level.get(), T.is_leaf.get(), T.tgt_count.get(), nb,
                                                              l_c, fin.get() + l_c + 4);
    FGT_LAUNCHED();
    // one pinned block for both read-backs (per thread, grown as needed)
    static thread_local int64_t* hp = nullptr;
    static thread_local int64_t hp_cap = 0;
    const int64_t need = l_c + 6 + nb;
    if (need > hp_cap) {
      if (hp) FGT_CUDA(cudaFreeHost(hp));
      hp_cap = std::max<int64_t>(need, 2 * hp_cap);
      FGT_CUDA(cudaMallocHost((void**)&hp, hp_cap * sizeof(int64_t)));
    }
    trace_mark(st, "tree:finalize");
    FGT_CUDA(cudaMemcpyAsync(hp, fin.get(), (l_c + 6) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    FGT_CUDA(cudaMemcpyAsync(hp + l_c + 6, dsrc.get(), nb * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    FGT_CUDA(cudaStreamSynchronize(st));
    trace_mark(st, "tree:finalize(sync)");
    std::vector<int64_t> h(hp, hp + l_c + 6);
    T.h_dense_src.assign(hp + l_c + 6, hp + l_c + 6 + h[l_c + 2]);
    T.lc_tleaves = h[l_c + 4];
    T.lc_targets = h[l_c + 5];
    T.level_off.assign(h.begin(), h.begin() + l_c + 2);
    T.n_dense = h[l_c + 2];
    T.n_leaves = h[l_c + 3];
    T.n_levels = 0;
    for (int l = 0; l <= l_c; ++l)
      if (T.level_off[l + 1] > T.level_off[l]) T.n_levels = l + 1;
  }
}

}  // namespace

void build_tree(TreeDev& T, const double* src, int64_t ns, const double* tgt, int64_t nt,
                const fgt_tree_params& tp, cudaStream_t st) {
  FGT_REQUIRE(tp.dim >= 1 && tp.dim <= 3, FGT_EINVAL, "dim must be 1, 2, or 3");
  FGT_REQUIRE(tp.delta > 0, FGT_EINVAL, "delta must be positive");
  if (tp.dim == 1) build_tree_impl<1>(T, src, ns, tgt, nt, tp, st);
  else if (tp.dim == 2) build_tree_impl<2>(T, src, ns, tgt, nt, tp, st);
  else build_tree_impl<3>(T, src, ns, tgt, nt, tp, st);
}

// sources with their charges in one pass (one read of the permutation), UNR independent
// rows per thread so several random row reads are in flight
template <int D>
__global__ void __launch_bounds__(256) gather_src_q_kernel(const double* __restrict__ a, const double* __restrict__ q,
                                                           const int64_t* __restrict__ perm, int64_t n,
                                                           double* __restrict__ out, double* __restrict__ qout) {
  constexpr int UNR = 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += stride * UNR) {
    int64_t j[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) j[u] = i0 + u * stride < n ? perm[i0 + u * stride] : -1;
    double v[UNR][D + 1];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      if (j[u] < 0) continue;
#pragma unroll
      for (int k = 0; k < D; ++k) v[u][k] = a[j[u] * D + k];
      if (q) v[u][D] = q[j[u]];
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      if (j[u] < 0) continue;
      const int64_t i = i0 + u * stride;
#pragma unroll
      for (int k = 0; k < D; ++k) out[i * D + k] = v[u][k];
      if (q) qout[i] = v[u][D];
    }
  }
}

void gather_sorted_points(TreeDev& T, const double* src, const double* q, const double* tgt) {
  cudaStream_t st = T.st;
  const int d = T.d;
  T.src_sorted.alloc(T.ns * d, st);
  T.tgt_sorted.alloc(T.nt * d, st);
  if (q) T.q_sorted.alloc(T.ns, st);
  auto gather = [&](const double* a, const double* qq, const int64_t* perm, int64_t n, double* out, double* qo) {
    if (n == 0) return;
    unsigned g = grid_for(n, 256 * 4);
    if (d == 1) gather_src_q_kernel<1><<<g, 256, 0, st>>>(a, qq, perm, n, out, qo);
    else if (d == 2) gather_src_q_kernel<2><<<g, 256, 0, st>>>(a, qq, perm, n, out, qo);
    else gather_src_q_kernel<3><<<g, 256, 0, st>>>(a, qq, perm, n, out, qo);
    FGT_LAUNCHED();
  };
  gather(src, q, T.src_perm.get(), T.ns, T.src_sorted.get(), q ? T.q_sorted.get() : nullptr);
  gather(tgt, nullptr, T.tgt_perm.get(), T.nt, T.tgt_sorted.get(), nullptr);
}

// Multi-GPU shares: only the leaves a rank works on get their points gathered (warp per box:
// sources + charges of the boxes flagged in need_src, targets of those in need_tgt); the
// rest of src_sorted / tgt_sorted stays unwritten and is never read by that rank.
namespace {
// BIG = false: a warp per box of the tree, except P-boxes above GN_BIG points; BIG = true: a
// CTA per listed P-box above GN_BIG points (all 256 threads stride over its points) -- so a
// 50k-point leaf of a clustered input does not serialise on one warp.  Leaves that are not
// P-boxes hold <= n_s points.
constexpr int64_t GN_BIG = 1024;
template <int D, bool BIG>
__global__ void __launch_bounds__(256) gather_needed_kernel(
    const double* __restrict__ a, const double* __restrict__ q, const int64_t* __restrict__ perm,
    const int64_t* __restrict__ start, const int64_t* __restrict__ count, const uint8_t* __restrict__ is_leaf,
    const uint8_t* __restrict__ need, const int64_t* __restrict__ dense_slot, const int64_t* __restrict__ dense_ids,
    int64_t nb, double* __restrict__ out, double* __restrict__ qout) {
  const int lane = BIG ? threadIdx.x : (threadIdx.x & 31);
  const int width = BIG ? 256 : 32;
  const int64_t nunit = BIG ? (int64_t)gridDim.x : (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t unit = BIG ? (int64_t)blockIdx.x : (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  for (int64_t it = unit; it < nb; it += nunit) {
    const int64_t b = BIG ? dense_ids[it] : it;
    if (!need[b] || !is_leaf[b]) continue;
    const int64_t s0 = start[b], n = count[b];
    if (BIG ? n <= GN_BIG : (n > GN_BIG && dense_slot[b] >= 0)) continue;
    for (int64_t i = lane; i < n; i += width) {
      const int64_t j = perm[s0 + i];
#pragma unroll
      for (int k = 0; k < D; ++k) out[(s0 + i) * D + k] = a[j * D + k];
      if (q) qout[s0 + i] = q[j];
    }
  }
}
}  // namespace

void gather_needed_points(TreeDev& T, const double* src, const double* q, const double* tgt,
                          const uint8_t* need_src, const uint8_t* need_tgt) {
  cudaStream_t st = T.st;
  const int d = T.d;
  T.src_sorted.alloc(T.ns * d, st);
  T.tgt_sorted.alloc(T.nt * d, st);
  if (q) T.q_sorted.alloc(T.ns, st);
  const unsigned g = grid_for(T.nb, 8), gb = (unsigned)std::min<int64_t>(std::max<int64_t>(T.n_dense, 1), 148 * 8);
  auto run = [&](const double* a, const double* qq, const int64_t* perm, const int64_t* start, const int64_t* count,
                 const uint8_t* need, double* out, double* qo) {
    const uint8_t* lf = T.is_leaf.get();
    const int64_t* dsl = T.dense_slot.get();
    const int64_t* dids = T.dense_ids.get();
#define FGT_GN(DD)                                                                                           \
  gather_needed_kernel<DD, false><<<g, 256, 0, st>>>(a, qq, perm, start, count, lf, need, dsl, dids, T.nb, out, qo); \
  FGT_LAUNCHED();                                                                                            \
  if (T.n_dense > 0) {                                                                                       \
    gather_needed_kernel<DD, true><<<gb, 256, 0, st>>>(a, qq, perm, start, count, lf, need, dsl, dids, T.n_dense, out, qo); \
    FGT_LAUNCHED();                                                                                          \
  }
    if (d == 1) { FGT_GN(1) } else if (d == 2) { FGT_GN(2) } else { FGT_GN(3) }
#undef FGT_GN
  };
  if (T.ns > 0) run(src, q, T.src_perm.get(), T.src_start.get(), T.src_count.get(), need_src, T.src_sorted.get(),
                    q ? T.q_sorted.get() : nullptr);
  if (T.nt > 0) run(tgt, nullptr, T.tgt_perm.get(), T.tgt_start.get(), T.tgt_count.get(), need_tgt, T.tgt_sorted.get(),
                    nullptr);
}

// ====================================================================== lists
namespace {

// Enumerate the neighbour leaves of leaf T (tree recipe of SURVEY §8c, matching
// neighbor_cells tree.py:176-193 + find_covering :107-115): for each offset, the
// covering leaf (colleague or coarse) or, when the colleague is subdivided, its
// children touching T (fine neighbours; leaves by balance).  Deduplicated on (S, v).
template <int D>
constexpr int list_cap() { return D == 1 ? 4 : (D == 2 ? 16 : 64); }  // <= 4^d entries per leaf

// One enumeration per target leaf: P entries (dense slot) then D entries (box) into the
// leaf's fixed slots [i*CAP, (i+1)*CAP), plus their counts.
// Neighbour resolution, one thread per (target leaf, offset): the box covering the
// neighbour cell (-1 if none / outside) and the packed image shift.  The covering searches
// are latency chains, so they get 3^d x the threads of the per-leaf enumeration.
template <int D>
__global__ void __launch_bounds__(128) lists_resolve_kernel(
    const int64_t* __restrict__ tleaves, const int64_t* __restrict__ ntl_dev, const uint64_t* __restrict__ keys,
    int64_t nb, const int64_t* __restrict__ coords, int periodic, int32_t* __restrict__ cov_j,
    int32_t* __restrict__ cov_v) {
  constexpr int NOFF = D == 1 ? 3 : (D == 2 ? 9 : 27);
  const int64_t ntl = *ntl_dev;
  for (int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; it < ntl * NOFF;
       it += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = it / NOFF;
    const int t = (int)(it - i * NOFF);
    const int64_t T = tleaves[i];
    const int l = key_level(keys[T]);
    int64_t g[D], n[D];
    int o[D], v[D];
#pragma unroll
    for (int k = 0; k < D; ++k) g[k] = coords[T * D + k];
    offset_of<D>(t, o);
    int32_t j = -1, pv = 0;
    if (neighbor_cell<D>(g, o, l, periodic, n, v)) {
      j = (int32_t)find_covering_dev(keys, nb, D, l, morton_encode(n, D, l));
#pragma unroll
      for (int k = 0; k < D; ++k) pv |= (v[k] + 1) << (2 * k);
    }
    cov_j[it] = j;
    cov_v[it] = pv;
  }
}

// One enumeration per target leaf over its resolved neighbours (the reference order: offsets
// in order, a non-leaf neighbour's touching children in child order; a coarse leaf covering
// several neighbour cells once, at its first offset): P entries (dense slot) from the front
// of the leaf's fixed slots [i*CAP, (i+1)*CAP), D entries (box) from the back, plus counts.
template <int D>
__global__ void __launch_bounds__(128) lists_kernel(
    const int64_t* __restrict__ tleaves, const int64_t* __restrict__ ntl_dev,
    const uint8_t* __restrict__ leaf, const int64_t* __restrict__ coords,
    const int64_t* __restrict__ children, const int64_t* __restrict__ scount,
    const int64_t* __restrict__ dense_slot, const uint64_t* __restrict__ keys,
    const int32_t* __restrict__ cov_j, const int32_t* __restrict__ cov_v, int64_t* __restrict__ pcnt,
    int64_t* __restrict__ dcnt, int64_t* __restrict__ fix_id, int32_t* __restrict__ fix_v) {
  constexpr int CAP = list_cap<D>();
  constexpr int NOFF = D == 1 ? 3 : (D == 2 ? 9 : 27);
  constexpr int NC = 1 << D;
  const int64_t ntl = *ntl_dev;  // launch covers a capacity
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ntl;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t T = tleaves[i];
    const int l = key_level(keys[T]);
    const int64_t side = (int64_t)1 << l;
    int64_t g[D];
#pragma unroll
    for (int k = 0; k < D; ++k) g[k] = coords[T * D + k];
    const int32_t* cj = cov_j + i * NOFF;
    const int32_t* cv = cov_v + i * NOFF;
    int np_ = 0, nd_ = 0;
    auto emit = [&](int64_t S, int pv) {
      const int64_t slot = dense_slot[S];
      int at;
      if (slot >= 0) {
        at = np_++;
        fix_id[i * CAP + at] = slot;
      } else if (scount[S] > 0) {
        at = CAP - 1 - nd_++;
        fix_id[i * CAP + at] = S;
      } else {
        return;
      }
#pragma unroll
      for (int k = 0; k < D; ++k) fix_v[(i * CAP + at) * D + k] = ((pv >> (2 * k)) & 3) - 1;
    };
    for (int t = 0; t < NOFF; ++t) {
      const int32_t j = cj[t];
      if (j < 0) continue;
      const int pv = cv[t];
      if (leaf[j]) {
        // a coarse leaf covering several neighbour cells is listed once (first offset)
        bool seen = false;
        for (int u = 0; u < t; ++u) seen |= (cj[u] == j && cv[u] == pv);
        if (!seen) emit(j, pv);
      } else {
        for (int c = 0; c < NC; ++c) {
          const int64_t ch = children[(int64_t)j * NC + c];
          bool touch = true;
#pragma unroll
          for (int k = 0; k < D; ++k) {
            const int64_t gc = coords[ch * D + k] + 2 * (int64_t)(((pv >> (2 * k)) & 3) - 1) * side;
            touch &= (gc >= 2 * g[k] - 1) && (gc <= 2 * g[k] + 2);
          }
          if (touch) emit(ch, pv);
        }
      }
    }
    pcnt[i] = np_;
    dcnt[i] = nd_;
  }
}

template <int D>
__global__ void lists_compact_kernel(const int64_t* __restrict__ tleaves, int64_t ntl,
                                     const int64_t* __restrict__ pcnt, const int64_t* __restrict__ dcnt,
                                     const int64_t* __restrict__ poff, const int64_t* __restrict__ doff,
                                     const int64_t* __restrict__ fix_id, const int32_t* __restrict__ fix_v,
                                     const int64_t* __restrict__ scount, const int64_t* __restrict__ tcount,
                                     int64_t* __restrict__ p_src, int32_t* __restrict__ p_v,
                                     int64_t* __restrict__ p_tgt, int64_t* __restrict__ d_src,
                                     int32_t* __restrict__ d_v, int64_t* __restrict__ d_tgt,
                                     unsigned long long* __restrict__ pairs) {
  constexpr int CAP = list_cap<D>();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ntl;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t T = tleaves[i];
    for (int e = 0; e < pcnt[i]; ++e) {
      const int64_t o = poff[i] + e;
      p_src[o] = fix_id[i * CAP + e];
      p_tgt[o] = T;
#pragma unroll
      for (int k = 0; k < D; ++k) p_v[o * D + k] = fix_v[(i * CAP + e) * D + k];
    }
    unsigned long long pr = 0;
    for (int e = 0; e < dcnt[i]; ++e) {
      const int at = CAP - 1 - e;
      const int64_t o = doff[i] + e;
      const int64_t S = fix_id[i * CAP + at];
      d_src[o] = S;
      d_tgt[o] = T;
#pragma unroll
      for (int k = 0; k < D; ++k) d_v[o * D + k] = fix_v[(i * CAP + at) * D + k];
      pr += (unsigned long long)(scount[S] * tcount[T]);
    }
    if (pr) atomicAdd(pairs, pr);
  }
}

__global__ void target_leaf_flag_kernel(const uint8_t* __restrict__ leaf, const int64_t* __restrict__ tcount,
                                        int64_t nb, uint8_t* __restrict__ flag) {
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb;
       b += (int64_t)gridDim.x * blockDim.x)
    flag[b] = leaf[b] && tcount[b] > 0;
}

__global__ void nonzero_flag_kernel(const int64_t* __restrict__ a, int64_t n, uint8_t* __restrict__ flag) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    flag[i] = a[i] > 0;
}

}  // namespace

// intermediates kept between build_lists_begin and build_lists_end
struct ListsPending {
  CubTmp tmp;
  DBuf<int64_t> cnt, tl, pcnt, dcnt, poff, doff, sel, seloff;
  DBuf<int64_t> fix_id;
  DBuf<int32_t> fix_v;
  int64_t* h = nullptr;  // pinned (4): ntl, n_p, n_d, n_psi (per-thread block, kept)
  cudaEvent_t ev = nullptr;
  ~ListsPending() {
    if (ev) cudaEventDestroy(ev);
  }
};

static int64_t* lists_pinned() {
  static thread_local int64_t* h = nullptr;
  if (!h) FGT_CUDA(cudaMallocHost((void**)&h, 4 * sizeof(int64_t)));
  return h;
}

template <int D>
static void build_lists_begin_impl(TreeDev& T) {
  cudaStream_t st = T.st;
  auto L = std::make_shared<ListsPending>();
  T.lists_pending = L;
  CubTmp& tmp = L->tmp;
  const int64_t nb = T.nb;
  // Sizes stay on the device until one host read-back (target leaves, P/D entry totals,
  // psi boxes); launches before it cover the capacity n_leaves.
  const int64_t cap = T.n_leaves;
  L->cnt.alloc(4, st);
  DBuf<int64_t>& cnt = L->cnt;  // ntl, n_p, n_d, n_psi
  // target leaves (leaves with targets), canonical order
  DBuf<uint8_t> flag(nb, st);
  target_leaf_flag_kernel<<<grid_for(nb, 256), 256, 0, st>>>(T.is_leaf.get(), T.tgt_count.get(), nb, flag.get());
  FGT_LAUNCHED();
  L->tl.alloc(nb, st);
  DBuf<int64_t>& tl = L->tl;
  DBuf<int64_t> iota(nb, st);
  iota_kernel<<<grid_for(nb, 256), 256, 0, st>>>(iota.get(), nb);
  FGT_LAUNCHED();
  size_t bytes = 0;
  FGT_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, iota.get(), flag.get(), tl.get(), cnt.get(), (int)nb, st));
  FGT_CUDA(cub::DeviceSelect::Flagged(tmp.get(bytes, st), bytes, iota.get(), flag.get(), tl.get(), cnt.get(), (int)nb, st));
  count_launch();

  L->pcnt.alloc(cap + 1, st);
  L->dcnt.alloc(cap + 1, st);
  L->poff.alloc(cap + 1, st);
  L->doff.alloc(cap + 1, st);
  DBuf<int64_t>&pcnt = L->pcnt, &dcnt = L->dcnt, &poff = L->poff, &doff = L->doff;
  pcnt.zero();
  dcnt.zero();
  T.pairs_dev.alloc(1, st);
  T.pairs_dev.zero();
  constexpr int CAP = list_cap<D>();
  L->fix_id.alloc(cap * CAP, st);
  L->fix_v.alloc(cap * CAP * D, st);
  DBuf<int64_t>& fix_id = L->fix_id;
  DBuf<int32_t>& fix_v = L->fix_v;
  if (cap > 0) {
    constexpr int NOFF = D == 1 ? 3 : (D == 2 ? 9 : 27);
    DBuf<int32_t> cov_j(cap * NOFF, st), cov_v(cap * NOFF, st);
    lists_resolve_kernel<D><<<grid_for(cap * NOFF, 128), 128, 0, st>>>(
        tl.get(), cnt.get(), T.bkey.get(), nb, T.coords.get(), T.periodic, cov_j.get(), cov_v.get());
    FGT_LAUNCHED();
    lists_kernel<D><<<grid_for(cap, 128), 128, 0, st>>>(
        tl.get(), cnt.get(), T.is_leaf.get(), T.coords.get(), T.children.get(), T.src_count.get(),
        T.dense_slot.get(), T.bkey.get(), cov_j.get(), cov_v.get(), pcnt.get(), dcnt.get(), fix_id.get(),
        fix_v.get());
    FGT_LAUNCHED();
  }
  bytes = 0;
  FGT_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, pcnt.get(), poff.get(), (int)(cap + 1), st));
  FGT_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(bytes, st), bytes, pcnt.get(), poff.get(), (int)(cap + 1), st));
  FGT_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(bytes, st), bytes, dcnt.get(), doff.get(), (int)(cap + 1), st));
  count_launch(2);
  FGT_CUDA(cudaMemcpyAsync(cnt.get() + 1, poff.get() + cap, sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
  FGT_CUDA(cudaMemcpyAsync(cnt.get() + 2, doff.get() + cap, sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
  // psi boxes: target leaves with P entries -> compact CSR (entries past ntl have pcnt 0)
  DBuf<uint8_t> f2(cap + 1, st);
  nonzero_flag_kernel<<<grid_for(cap, 256), 256, 0, st>>>(pcnt.get(), cap, f2.get());
  FGT_LAUNCHED();
  L->sel.alloc(cap + 1, st);
  L->seloff.alloc(cap + 1, st);
  DBuf<int64_t>&sel = L->sel, &seloff = L->seloff;
  bytes = 0;
  FGT_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, tl.get(), f2.get(), sel.get(), cnt.get() + 3, (int)cap, st));
  FGT_CUDA(cub::DeviceSelect::Flagged(tmp.get(bytes, st), bytes, tl.get(), f2.get(), sel.get(), cnt.get() + 3, (int)cap, st));
  FGT_CUDA(cub::DeviceSelect::Flagged(tmp.get(bytes, st), bytes, poff.get(), f2.get(), seloff.get(), cnt.get() + 3, (int)cap, st));
  count_launch(2);
  L->h = lists_pinned();
  FGT_CUDA(cudaMemcpyAsync(L->h, cnt.get(), 4 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  FGT_CUDA(cudaEventCreateWithFlags(&L->ev, cudaEventDisableTiming));
  FGT_CUDA(cudaEventRecord(L->ev, st));
  trace_mark(st, "lists:enum");
}

template <int D>
static void build_lists_end_impl(TreeDev& T) {
  cudaStream_t st = T.st;
  auto L = std::static_pointer_cast<ListsPending>(T.lists_pending);
  FGT_CUDA(cudaEventSynchronize(L->ev));
  trace_mark(st, "lists:enum(sync)");
  const int64_t* h = L->h;
  DBuf<int64_t>&cnt = L->cnt, &tl = L->tl, &pcnt = L->pcnt, &dcnt = L->dcnt, &poff = L->poff, &doff = L->doff;
  DBuf<int64_t>&sel = L->sel, &seloff = L->seloff, &fix_id = L->fix_id;
  DBuf<int32_t>& fix_v = L->fix_v;
  const int64_t ntl = h[0];
  T.n_dtgt = ntl;
  T.n_p = h[1];
  T.n_d = h[2];
  T.n_psi = h[3];
  T.p_src.alloc(T.n_p, st);
  T.p_v.alloc(T.n_p * D, st);
  T.p_tgt.alloc(T.n_p, st);
  T.d_src.alloc(T.n_d, st);
  T.d_v.alloc(T.n_d * D, st);
  T.d_tgt.alloc(T.n_d, st);
  if (ntl > 0) {
    lists_compact_kernel<D><<<grid_for(ntl, 128), 128, 0, st>>>(
        tl.get(), ntl, pcnt.get(), dcnt.get(), poff.get(), doff.get(), fix_id.get(), fix_v.get(),
        T.src_count.get(), T.tgt_count.get(), T.p_src.get(), T.p_v.get(), T.p_tgt.get(),
        T.d_src.get(), T.d_v.get(), T.d_tgt.get(), reinterpret_cast<unsigned long long*>(T.pairs_dev.get()));
    FGT_LAUNCHED();
  }
  fix_id.release();
  fix_v.release();
  // direct CSR over all target leaves (d_off[ntl] = n_d: the counts past ntl are 0)
  T.d_tgt_ids = std::move(tl);
  T.d_off = std::move(doff);
  T.psi_ids = std::move(sel);
  T.p_off = std::move(seloff);
  FGT_CUDA(cudaMemcpyAsync(T.p_off.get() + T.n_psi, cnt.get() + 1, sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
  T.n_direct_pairs = -1;  // read lazily (direct_pairs)
  T.lists_built = true;
  T.lists_pending.reset();  // the remaining scratch is freed stream-ordered on its stream
}

int64_t direct_pairs(TreeDev& T) {
  if (T.n_direct_pairs < 0) {
    int64_t v = 0;
    if (T.pairs_dev.size()) {
      T.pairs_dev.to_host(&v, 1);
      FGT_CUDA(cudaStreamSynchronize(T.st));
    }
    T.n_direct_pairs = v;
  }
  return T.n_direct_pairs;
}

void build_lists_begin(TreeDev& T) {
  if (T.lists_built || T.lists_pending) return;
  if (T.d == 1) build_lists_begin_impl<1>(T);
  else if (T.d == 2) build_lists_begin_impl<2>(T);
  else build_lists_begin_impl<3>(T);
}

void build_lists_end(TreeDev& T) {
  if (T.lists_built) return;
  if (!T.lists_pending) build_lists_begin(T);
  if (T.d == 1) build_lists_end_impl<1>(T);
  else if (T.d == 2) build_lists_end_impl<2>(T);
  else build_lists_end_impl<3>(T);
}

void build_lists(TreeDev& T) {
  build_lists_begin(T);
  build_lists_end(T);
}

}  // namespace fgt
