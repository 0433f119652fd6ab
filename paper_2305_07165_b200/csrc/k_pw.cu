// Plane-wave phases of the discrete FGT (Alg 2) on sm_100a.
//
//   form    phi_l(S) = w_l sum_j q_j exp(-i k_l.(y_j - c_S))
//   gather  psi_l(T) = sum_{(S,v) in L_P(T)} exp(i k_l.(c_T - c_S - v)) phi_l(S)  (:825-828)
//   eval    u(x)    += Re sum_l exp(i k_l.(x - c_T)) psi_l(T)          (:833-835)
//   direct  u(x)    += sum_{(S,v) in L_D(T)} sum_{|x-y-v|^2 <= D0^2 delta} exp(-|x-y-v|^2/delta) q
//
// The reference evaluates form/eval with nufft_type1/2 (nufft.py:139-183), which at
// every BASELINE configuration dispatches to the exact tensor-factored sums of
// dft_oracle (nufft.py:65-103).  Here those sums are complex GEMMs on the FP64 tensor
// cores (mma.sync m8n8k4 .f64 -> SASS DMMA; tcgen05 has no f64 kind):
//   form: phi[r, c] = sum_j A[r, j] E_last[j, c],  A[r, j] = q_j prod_{k<d-1} E_k[j, r_k]
//   eval: T1[j, r]  = sum_c E'_last[j, c] psi[r, c];  u_j = Re sum_r T1[j, r] prod E'_k[j, r_k]
// with r the flattened leading d-1 mode indices (C order, axis 0 slowest, ModeGrid
// layout nufft.py:20-48) and c the last-axis mode.  Per-point 1-D phase tables are
// built in shared memory (sincos per 8-mode segment + rotation recurrence).
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "k_nufft.cuh"

namespace fgt {

int psi_mode() {
  const char* e = std::getenv("FGT_PSI");
  if (e && !std::strcmp(e, "materialise")) return 1;
  if (e && !std::strcmp(e, "fused")) return 2;
  return 0;
}

int nufft_mode() {
  const char* e = std::getenv("FGT_NUFFT_MODE");
  if (!e) return 0;
  if (!std::strcmp(e, "direct")) return 1;
  if (!std::strcmp(e, "spread")) return 2;
  if (!std::strcmp(e, "proxy")) return 3;  // form: proxy points (evaluation as "spread")
  return 0;
}

namespace {
// complex-MAC equivalents of the separable grid <-> mode transform of one box
// (half spectrum for d >= 2: nh = n_f/2 + 1 planes along axis 0)
double box_dft_cost(int D, int G, int n_f) {
  const double g = G, n = n_f, h = n_f / 2 + 1;
  if (D == 1) return n * g;
  if (D == 2) return 0.5 * g * g * n + h * n * g;
  return 0.5 * g * g * g * h + h * g * g * n + h * n * g * n;
}
// true if the box-local NUFFT beats the exact sums for a box with npts points
// tap_cost: relative cost of one kernel tap per point; fixed_mult: weight of the per-box
// grid <-> mode transform (the evaluation's batched transforms + interpolation measured ~2x
// the form's per box: with G = 39 at config 2 a factor 1 sent 145-164-target boxes to a
// slower NUFFT evaluation)
bool prefer_nufft(const NufftPlan* N, int D, int64_t NF, int64_t npts, double tap_cost, double fixed_mult = 1.0) {
  // NF: stored modes per expansion
  if (!N) return false;
  if (N->G > 64) return false;  // beyond the spreading kernels' grid (wide root series)
  const int mode = nufft_mode();
  if (mode == 1) return false;
  if (mode >= 2) return npts > 0;
  double taps = 1;
  for (int k = 0; k < D; ++k) taps *= N->w;
  const double direct = (double)npts * NF;
  const double spread = tap_cost * npts * taps + fixed_mult * (box_dft_cost(D, N->G, N->n_f) + 32.0 * NF);
  return direct > spread;
}
}  // namespace

namespace {

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  // not volatile: lets the scheduler interleave independent accumulators
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// etab[k][j][mi] = exp(sign * i * m * x_jk), m = mi - n_f/2, x_jk = (p_jk - ctr_k) * sc,
// zero for j >= cnt or mi >= n_f.  KC rows of NFP (multiple of 8) columns, row stride RS
// (>= NFP, padded so the fragment loads of consecutive rows hit distinct banks).
template <int D>
__device__ void build_etab(double2* __restrict__ etab, int KC, int NFP, int RS, const double* __restrict__ pts,
                           int64_t base, int cnt, const double* ctr, double sc, double sign, int n_f) {
  const int nseg = NFP >> 3;
  const int ntask = KC * D * nseg;
  for (int task = threadIdx.x; task < ntask; task += blockDim.x) {
    int seg = task % nseg;
    int rest = task / nseg;
    int k = rest % D;
    int j = rest / D;
    double2* out = etab + ((size_t)k * KC + j) * RS + seg * 8;
    if (j >= cnt) {
#pragma unroll
      for (int t = 0; t < 8; ++t) out[t] = make_double2(0.0, 0.0);
      continue;
    }
    double x = (pts[(base + j) * D + k] - ctr[k]) * sc;
    int m0 = seg * 8 - n_f / 2;
    double s0, c0, s1, c1;
    sincos(sign * (double)m0 * x, &s0, &c0);
    sincos(sign * x, &s1, &c1);
    double2 val = make_double2(c0, s0);
    const double2 step = make_double2(c1, s1);
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      out[t] = (seg * 8 + t < n_f) ? val : make_double2(0.0, 0.0);
      val = cmul(val, step);
    }
  }
}

// ------------------------------------------------------------------ form
struct FormArgs {
  const double* src;        // sorted sources (ns, d)
  const double* q;          // sorted charges
  const double* center;     // (nb, d)
  const int64_t* dense_ids; // slot -> box
  const int64_t* src_start;
  const int4* units;        // (slot, k0, kn, scratch index or -1)
  double2* phi;
  double2* scratch;
  const double* w1d;
  int n_f, R, MG, KS;  // R: stored rows (RH)
  int half;
  double sc;
};

constexpr int FORM_KC = 32;
constexpr int FORM_MT = 2;

template <int D, int NT>
__global__ void __launch_bounds__(256, 1) form_kernel(FormArgs a) {
  extern __shared__ double2 sm[];
  constexpr int KC = FORM_KC, MT = FORM_MT, NFP = NT * 8, RS = NFP + 2;
  double2* etab = sm;
  double* sq = reinterpret_cast<double*>(etab + D * KC * RS);
  const int4 u = a.units[blockIdx.y];
  const int slot = u.x, k0 = u.y, kn = u.z, oidx = u.w;
  const int64_t box = a.dense_ids[slot];
  const int64_t pbase = a.src_start[box] + k0;
  double ctr[D];
#pragma unroll
  for (int k = 0; k < D; ++k) ctr[k] = a.center[box * D + k];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mg = warp % a.MG, ks = warp / a.MG;
  const bool active = ks < a.KS;
  const int row0 = (blockIdx.x * a.MG + mg) * MT * 8;
  const int n_f = a.n_f;

  double acc[MT][NT][4];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[mt][nt][e] = 0.0;

  int ra[MT], rb[MT];
  bool rv[MT];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    int r = row0 + mt * 8 + (lane >> 2);
    rv[mt] = r < a.R;
    ra[mt] = half_plane_mi(D == 3 ? r / n_f : r, n_f, a.half);
    rb[mt] = D == 3 ? r % n_f : 0;
  }

  for (int c0 = 0; c0 < kn; c0 += KC) {
    const int cnt = min(KC, kn - c0);
    __syncthreads();
    build_etab<D>(etab, KC, NFP, RS, a.src, pbase + c0, cnt, ctr, a.sc, -1.0, n_f);
    for (int t = threadIdx.x; t < KC; t += blockDim.x) sq[t] = t < cnt ? a.q[pbase + c0 + t] : 0.0;
    __syncthreads();
    if (active) {
      for (int kk = ks; kk < KC / 4; kk += a.KS) {
        const int j = kk * 4 + (lane & 3);
        double2 b[NT];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) b[nt] = etab[((D - 1) * KC + j) * RS + nt * 8 + (lane >> 2)];
        const double qj = sq[j];
        double2 A[MT];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          A[mt] = make_double2(0.0, 0.0);
          if (rv[mt]) {
            if (D == 1) {
              A[mt] = make_double2(qj, 0.0);
            } else if (D == 2) {
              double2 e0 = etab[(0 * KC + j) * RS + ra[mt]];
              A[mt] = make_double2(qj * e0.x, qj * e0.y);
            } else {
              double2 e0 = etab[(0 * KC + j) * RS + ra[mt]];
              double2 e1 = etab[(1 * KC + j) * RS + rb[mt]];
              double2 p = cmul(e0, e1);
              A[mt] = make_double2(qj * p.x, qj * p.y);
            }
          }
        }
        // four passes so consecutive DMMAs never share an accumulator
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], A[mt].x, b[nt].x);
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) dmma(acc[mt][nt][2], acc[mt][nt][3], A[mt].x, b[nt].y);
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], -A[mt].y, b[nt].y);
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) dmma(acc[mt][nt][2], acc[mt][nt][3], A[mt].y, b[nt].x);
      }
    }
  }

  // reduce the K-split warps into the ks == 0 warp of each m-group
  if (a.KS > 1) {
    double* red = reinterpret_cast<double*>(sm);
    for (int s = 1; s < a.KS; ++s) {
      __syncthreads();
      if (ks == s) {
        double* dst = red + ((size_t)mg * 32 + lane) * MT * NT * 4;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) dst[(mt * NT + nt) * 4 + e] = acc[mt][nt][e];
      }
      __syncthreads();
      if (ks == 0) {
        const double* srcp = red + ((size_t)mg * 32 + lane) * MT * NT * 4;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[mt][nt][e] += srcp[(mt * NT + nt) * 4 + e];
      }
    }
  }
  if (ks != 0) return;
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    const int r = row0 + mt * 8 + (lane >> 2);
    if (r >= a.R) continue;
    double wr = 1.0;
    if (D == 2) wr = a.w1d[half_plane_mi(r, n_f, a.half)];
    if (D == 3) wr = a.w1d[half_plane_mi(r / n_f, n_f, a.half)] * a.w1d[r % n_f];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int c = nt * 8 + 2 * (lane & 3) + i;
        if (c >= n_f) continue;
        double re = acc[mt][nt][i], im = acc[mt][nt][2 + i];
        if (oidx < 0) {
          double w = wr * a.w1d[c];
          a.phi[((size_t)slot * a.R + r) * n_f + c] = make_double2(re * w, im * w);
        } else {
          a.scratch[((size_t)oidx * a.R + r) * n_f + c] = make_double2(re, im);
        }
      }
    }
  }
}

// sum the K-split partials of multi-unit boxes (fixed order: deterministic)
template <int D>
__global__ void form_reduce_kernel(const double2* __restrict__ scratch, const int4* __restrict__ red,
                                   int64_t NF, int n_f, int half, const double* __restrict__ w1d,
                                   double2* __restrict__ phi) {
  const int4 rj = red[blockIdx.y];  // (slot, first scratch, count, -)
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < NF;
       e += (int64_t)gridDim.x * blockDim.x) {
    double2 s = make_double2(0.0, 0.0);
    for (int t = 0; t < rj.z; ++t) {
      double2 v = scratch[(size_t)(rj.y + t) * NF + e];
      s.x += v.x;
      s.y += v.y;
    }
    int64_t rem = e;
    double w = 1.0;
#pragma unroll
    for (int k = D - 1; k >= 0; --k) {
      const int idx = k == 0 ? half_plane_mi((int)rem, n_f, half) : (int)(rem % n_f);
      w *= w1d[idx];
      rem /= n_f;
    }
    phi[(size_t)rj.x * NF + e] = make_double2(s.x * w, s.y * w);
  }
}

__global__ void psi_meta_kernel(const int64_t* __restrict__ ids, int64_t n,
                                const int64_t* __restrict__ cnt, const int64_t* __restrict__ parent,
                                int64_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    out[i] = cnt[ids[i]];
    out[n + i] = parent[ids[i]];
  }
}

__global__ void gather_counts_kernel(const int64_t* __restrict__ ids, int64_t n,
                                     const int64_t* __restrict__ cnt, int64_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = cnt[ids[i]];
}

// ------------------------------------------------------------------ gather
struct GatherArgs {
  const int64_t* psi_ids;
  const int64_t* p_off;
  const int64_t* p_src;   // dense slot
  const int32_t* p_v;
  const int64_t* dense_ids;
  const int64_t* coords;
  const double2* phase;   // (5, n_f): shifts o = -2..2, exp(i m sc o side_lc)
  const double2* phi;
  double2* psi;   // batch-local output
  const int64_t* goff;  // sibling groups: psi index ranges
  int64_t NF, i0; // NF: stored modes; i0: first psi index of the batch
  int n_f, l_c, half;
};

#ifndef FGT_GATHER_MPT
#define FGT_GATHER_MPT 4
#endif
#ifndef FGT_GATHER_MINB
#define FGT_GATHER_MINB 3
#endif
#ifndef FGT_GATHER_UNROLL
#define FGT_GATHER_UNROLL 1
#endif
constexpr int GATHER_THREADS = 256;
constexpr int GATHER_UNROLL = FGT_GATHER_UNROLL;
constexpr int GATHER_MPT = FGT_GATHER_MPT;  // modes per thread
constexpr int GATHER_CHUNK = GATHER_THREADS * GATHER_MPT;

// Diagonal translation is organised by sibling group: the <= 2^d psi boxes under one
// parent cell (contiguous in the psi list).  Every P entry of a member T (level l_c, child
// position c of parent p) is a source image S' = coords_S + v * 2^l_c with
// S' - 2p in [-1, 2]^d, so the sources of a group are indexed by that relative position
// (4^d slots): each distinct phi_S is loaded once per mode and applied to every member that
// uses it.  The shift of (T, S') along axis k is o_k = c_k - rel_k in {-1, 0, 1}, so the
// translation phase is a product of 1, P_k or conj(P_k), P_k = exp(i m_k sc side_lc).
//
// group_table_kernel: one CTA per group builds the compacted source table (slot, member
// mask | relative position) and the psi row of each child position.
template <int D>
__global__ void group_table_kernel(GatherArgs a, int64_t* __restrict__ gt_slot,
                                   unsigned* __restrict__ gt_code, int* __restrict__ gt_nu,
                                   int64_t* __restrict__ gt_out) {
  constexpr int NSIB = 1 << D;
  constexpr int NREL = 1 << (2 * D);
  __shared__ int64_t s_slot[NREL];
  __shared__ unsigned s_mask[NREL];
  const int64_t g = blockIdx.x;
  const int64_t g0 = a.goff[g], g1 = a.goff[g + 1];
  const int nmem = (int)(g1 - g0);
  const int64_t side = (int64_t)1 << a.l_c;
  for (int i = threadIdx.x; i < NREL; i += blockDim.x) s_mask[i] = 0;
  if (threadIdx.x < NSIB) gt_out[g * NSIB + threadIdx.x] = -1;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int m = warp; m < nmem; m += blockDim.x >> 5) {
    const int64_t i = g0 + m;
    const int64_t T = a.psi_ids[i];
    int c = 0;
    int64_t base[D];
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const int64_t ct = a.coords[T * D + k];
      c |= (int)(ct & 1) << k;
      base[k] = ct & ~(int64_t)1;
    }
    const int64_t e0 = a.p_off[i], e1 = a.p_off[i + 1];
    for (int64_t t = e0 + lane; t < e1; t += 32) {
      const int64_t slot = a.p_src[t];
      const int64_t S = a.dense_ids[slot];
      int idx = 0;
#pragma unroll
      for (int k = 0; k < D; ++k) {
        const int64_t rel = a.coords[S * D + k] + (int64_t)a.p_v[t * D + k] * side - base[k];
        idx |= (int)(rel + 1) << (2 * k);
      }
      s_slot[idx] = slot;
      atomicOr(&s_mask[idx], 1u << c);
    }
  }
  __syncthreads();
  // the psi row of each child position (written after the -1 fill above)
  for (int m = threadIdx.x; m < nmem; m += blockDim.x) {
    const int64_t T = a.psi_ids[g0 + m];
    int c = 0;
#pragma unroll
    for (int k = 0; k < D; ++k) c |= (int)(a.coords[T * D + k] & 1) << k;
    gt_out[g * NSIB + c] = g0 + m - a.i0;
  }
  if (threadIdx.x == 0) {
    int nu = 0;
    for (int idx = 0; idx < NREL; ++idx)
      if (s_mask[idx]) {
        gt_slot[g * NREL + nu] = s_slot[idx];
        gt_code[g * NREL + nu] = s_mask[idx] | ((unsigned)idx << 8);
        ++nu;
      }
    gt_nu[g] = nu;
  }
}

// One CTA per (group, chunk of GATHER_CHUNK modes), GATHER_MPT modes per thread; the
// group index runs fastest in the grid.
// The phase of (member c, source at relative position rel) factors per axis as
// P_k^(c_k - rel_k) = P_k^(-rel_k) P_k^(c_k): a per-source factor f0_u (rel_k in -1..2,
// read from the 5-row phase table in shared memory) and a per-member factor Q_c.  So
//   psi_c = Q_c * sum_{u serving c} (f0_u phi_u),
// one complex product per source and a complex add per (source, member) pair.
template <int D>
__global__ void __launch_bounds__(GATHER_THREADS, FGT_GATHER_MINB) gather_kernel(
    GatherArgs a, const int64_t* __restrict__ gt_slot, const unsigned* __restrict__ gt_code,
    const int* __restrict__ gt_nu, const int64_t* __restrict__ gt_out) {
  constexpr int NSIB = 1 << D;
  constexpr int NREL = 1 << (2 * D);
  constexpr int NFMAX = 64;  // pw_setup requires n_f <= 64
  __shared__ int64_t u_slot[NREL];
  __shared__ unsigned u_code[NREL];
  __shared__ double2 s_ph[5 * NFMAX];  // rows o = -2..2
  const int64_t g = blockIdx.x;  // group fastest: CTAs in flight share a mode chunk, so the
                                 // phi slices of neighbouring groups are reused from L2
  const int nu = gt_nu[g];
  for (int u = threadIdx.x; u < nu; u += blockDim.x) {
    u_slot[u] = gt_slot[g * NREL + u];
    u_code[u] = gt_code[g * NREL + u];
  }
  for (int i = threadIdx.x; i < 5 * a.n_f; i += blockDim.x) s_ph[(i / a.n_f) * NFMAX + i % a.n_f] = a.phase[i];
  int64_t outr[NSIB];
#pragma unroll
  for (int c = 0; c < NSIB; ++c) outr[c] = gt_out[g * NSIB + c];
  __syncthreads();
  const unsigned n_f = (unsigned)a.n_f;
  const unsigned NF = (unsigned)a.NF;
#pragma unroll 1
  for (int j = 0; j < GATHER_MPT; ++j) {
    const unsigned e = (unsigned)blockIdx.y * GATHER_CHUNK + j * GATHER_THREADS + threadIdx.x;
    if (e >= NF) return;
    int mk[D];
    {
      unsigned rem = e;
#pragma unroll
      for (int k = D - 1; k >= 0; --k) {
        mk[k] = k == 0 ? half_plane_mi((int)rem, (int)n_f, a.half) : (int)(rem % n_f);
        rem /= n_f;
      }
    }
    double2 S[NSIB];
#pragma unroll
    for (int c = 0; c < NSIB; ++c) S[c] = make_double2(0.0, 0.0);
#pragma unroll GATHER_UNROLL
    for (int u = 0; u < nu; ++u) {
      const unsigned code = u_code[u];
      const double2 f = a.phi[(size_t)u_slot[u] * NF + e];
      // f0 = prod_k P_k^(-rel_k): table row -rel_k + 2 = 3 - ((code >> (8 + 2k)) & 3)
      double2 f0 = s_ph[(3 - (int)((code >> 8) & 3)) * NFMAX + mk[0]];
#pragma unroll
      for (int k = 1; k < D; ++k) f0 = cmul(f0, s_ph[(3 - (int)((code >> (8 + 2 * k)) & 3)) * NFMAX + mk[k]]);
      const double2 gu = cmul(f0, f);
      // S_c += [member c served] gu as a multiply-add by 0 / 1 (branch- and select-free)
#pragma unroll
      for (int c = 0; c < NSIB; ++c) {
        const double bc = __hiloint2double((code >> c) & 1u ? 0x3ff00000 : 0, 0);
        S[c].x = fma(bc, gu.x, S[c].x);
        S[c].y = fma(bc, gu.y, S[c].y);
      }
    }
    // Q_c = prod_{k: c_k = 1} P_k (table row o = +1)
    double2 P1[D];
#pragma unroll
    for (int k = 0; k < D; ++k) P1[k] = s_ph[3 * NFMAX + mk[k]];
#pragma unroll
    for (int c = 0; c < NSIB; ++c) {
      if (outr[c] < 0) continue;
      double2 v = S[c];
#pragma unroll
      for (int k = 0; k < D; ++k)
        if ((c >> k) & 1) v = cmul(v, P1[k]);
      a.psi[(size_t)outr[c] * NF + e] = v;
    }
  }
}

// ------------------------------------------------------------------ fused gather + eval
// psi never reaches HBM: psi_T is consumed only by the evaluation at T's targets
// (PAPER.md:825-835), so translation and evaluation run in one kernel.
//
// Reference point.  The translation phase factors as
//   e^{i k.(c_T - c_S)} = e^{i k.(c_T - c_ref)} e^{i k.(c_ref - c_S)}
// for any point c_ref (here the root centre), so with phi'_S = e^{i k.(c_ref - c_S)} phi_S
// (phi_rephase_kernel, once per P-box) the translation is a plain sum and the target
// phases are taken from c_ref:
//   u(x) = Re sum_l e^{i k_l.(x - c_ref)} sum_{S in L_P(T)} phi'_{S,l}.
// The angles reach |k| |x - c_ref| ~ 1e4 rad, so every phase is formed in double-double
// (TwoSum / TwoProd) and reduced modulo a two-term 2 pi before the sincos (phase_dd): each
// factor is exact to ~1 ulp, like the local formulation.  Free space only (periodic image
// shifts keep the materialising path).
//
// One CTA per sibling group (see gather_eval_kernel).  Warp w owns the 8-row x 16-column
// mode tile (row tile w / CB, column block w % CB) of each chunk of RC = 8 RT stored rows;
// lane l holds the 4 modes of the DMMA B fragment, row (l >> 2), columns 4 kk + (l & 3).
// For every member c the lane accumulates S_c = sum_{u serving c} phi'_u in registers
// (members in halves of 4 for d = 3), each phi'_u read once per group and chunk, and
// contracts it at once with the member's targets: T1 = E S_c is a complex GEMM tile (3 real
// DMMAs per complex MAC, Gauss) whose epilogue reduces Re(T1 F) over the warp's 8 rows
// with F the per-row axis-0/axis-1 factor.  The phase tables come by recurrence from
// per-target e^{-i (n_f/2) x}, e^{i x}, e^{8 i x}.  Target sums are accumulated per warp in
// shared memory and combined in a fixed order (no atomics: deterministic).
constexpr double GE_TWO_PI_HI = 6.283185307179586;
constexpr int64_t PHI_PAD = 64 * 64 + 64;  // double2 past the expansions (>= RC n_f + 16)
constexpr double GE_TWO_PI_LO = 2.4492935982947064e-16;

// e^{i m sc (a - b)}, accurate to ~1 ulp for angles up to ~1e8 rad
__device__ __forceinline__ double2 phase_dd(int m, double sc, double a, double b) {
  // d = a - b exactly as d_hi + d_lo (TwoSum)
  const double d_hi = a - b;
  const double bb = d_hi - a;
  const double d_lo = (a - (d_hi - bb)) + (-b - bb);
  // k = m sc exactly as k_hi + k_lo (TwoProd)
  const double k_hi = (double)m * sc;
  const double k_lo = fma((double)m, sc, -k_hi);
  // A = k d in double-double
  const double p = k_hi * d_hi;
  const double p_lo = fma(k_hi, d_hi, -p) + (k_hi * d_lo + k_lo * d_hi);
  const double q = rint(p * (1.0 / GE_TWO_PI_HI));
  const double r = fma(-q, GE_TWO_PI_HI, p) + (p_lo - q * GE_TWO_PI_LO);
  double sn, cs;
  sincos(r, &sn, &cs);
  return make_double2(cs, sn);
}

// bp[slot][k][mi] = e^{i (mi - n_f/2) sc (c_ref_k - c_S,k)} for every P-box slot
template <int D>
__global__ void box_phase_kernel(const int64_t* __restrict__ dense_ids, int64_t nd,
                                 const double* __restrict__ center, double3 c_ref, double sc, int n_f,
                                 double2* __restrict__ bp) {
  const double cr[3] = {c_ref.x, c_ref.y, c_ref.z};
  const int64_t n = nd * D * n_f;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int mi = (int)(e % n_f);
    const int k = (int)((e / n_f) % D);
    const int64_t slot = e / ((int64_t)D * n_f);
    const int64_t S = dense_ids[slot];
    bp[e] = phase_dd(mi - n_f / 2, sc, cr[k], center[S * D + k]);
  }
}

// phi'_S = e^{i k.(c_ref - c_S)} phi_S in place (stored half spectrum): one CTA per P-box
// slot; the separable phase is a row factor (axes < d-1, from shared memory) times a
// column factor (last axis, one per thread), two complex products per mode.
template <int D>
__global__ void __launch_bounds__(256) phi_rephase_kernel(double2* __restrict__ phi, int64_t n,
                                                          const int64_t* __restrict__ slots, int64_t NH,
                                                          int n_f, int RH, int half,
                                                          const double2* __restrict__ bp) {
  extern __shared__ double2 s_row[];  // RH
  const int CW = n_f <= 32 ? 32 : 64;
  const int c = threadIdx.x % CW, r0 = threadIdx.x / CW, rstep = blockDim.x / CW;
  for (int64_t it = blockIdx.x; it < n; it += gridDim.x) {
    const int64_t slot = slots[it];
    const double2* b = bp + slot * D * n_f;
    __syncthreads();
    for (int r = threadIdx.x; r < RH; r += blockDim.x) {
      double2 v = make_double2(1.0, 0.0);
      if (D >= 2) v = b[half_plane_mi(D == 3 ? r / n_f : r, n_f, half)];
      if (D == 3) v = cmul(v, b[n_f + r % n_f]);
      s_row[r] = v;
    }
    __syncthreads();
    if (c >= n_f) continue;
    const double2 cf = b[(D - 1) * n_f + c];
    double2* p = phi + slot * NH + c;
    for (int r = r0; r < RH; r += rstep) p[(int64_t)r * n_f] = cmul(cmul(s_row[r], cf), p[(int64_t)r * n_f]);
  }
}

constexpr int64_t GE_AUTO_MAX_TPL = 16;  // fused path when targets per level-l_c target leaf <= this

struct GEArgs {
  const int64_t* psi_ids;
  const int64_t* tgt_start;
  const int64_t* tgt_count;
  const int64_t* pstart;   // (n_psi) first tph slot of the box's targets; -1: not fused
  const double2* tph;      // (n_ptgt, 3D): per target and axis e^{-i (n_f/2) x}, e^{i x}, e^{8 i x}
  const double2* phi;      // (n_dense, RH, n_f) rephased expansions phi' (+ PHI_PAD zeros)
  double* u;               // sorted potentials (accumulated)
  int64_t NH;
  int n_f, RH, nh, half, CB, RT, TR;
};

__host__ __device__ inline int ge_cb(int n_f) { return (n_f + 15) / 16; }
__host__ __device__ inline int ge_rt(int n_f) { return 8 / ge_cb(n_f) > 0 ? 8 / ge_cb(n_f) : 1; }
// targets whose phase tables are resident per round (member-aligned 8-target tiles)
inline int ge_tr(int n_f) { return n_f <= 32 ? 64 : 32; }
inline size_t ge_smem(int n_f, int D, int RH) {
  const int CB = ge_cb(n_f), TR = ge_tr(n_f), NREL = 1 << (2 * D);
  const int ES = CB * 16 + 4, nh = D >= 2 ? n_f / 2 + 1 : 1;
  return (size_t)TR * ES * sizeof(double2) * 2           // E (last axis), E1 (axis 1)
         + (size_t)TR * (nh + 1) * sizeof(double2)        // E0 (w x axis-0 factor per plane)
         + (size_t)8 * TR * sizeof(double)                // s_part: per warp, per target
         + (size_t)NREL * 8 * sizeof(double)              // u_bc: member masks as 0.0 / 1.0
         + (size_t)NREL * (sizeof(void*) + sizeof(unsigned) + sizeof(int))  // sources, lists
         + (size_t)(TR / 8) * 3 * sizeof(int)             // tile list
         + (size_t)(RH + 64) * sizeof(int);               // row info (padded to whole chunks)
}

__device__ __forceinline__ double2 cpow(double2 b, int e) {
  double2 r = make_double2(1.0, 0.0);
  while (e > 0) {
    if (e & 1) r = cmul(r, b);
    b = cmul(b, b);
    e >>= 1;
  }
  return r;
}

// per fused target and axis: e^{-i (n_f/2) x}, e^{i x}, e^{8 i x}, x = (t - c_ref) sc (phase_dd)
template <int D>
__global__ void ge_target_phase_kernel(const int64_t* __restrict__ psi_ids, const int64_t* __restrict__ tgt_start,
                                       const int64_t* __restrict__ tgt_count, const int64_t* __restrict__ pstart,
                                       int64_t n_psi, const double* __restrict__ tgt, double3 c_ref, double sc,
                                       int n_f, double2* __restrict__ tph) {
  const double cr[3] = {c_ref.x, c_ref.y, c_ref.z};
  for (int64_t i = blockIdx.x; i < n_psi; i += gridDim.x) {
    const int64_t p0 = pstart[i];
    if (p0 < 0) continue;
    const int64_t T = psi_ids[i];
    const int64_t t0 = tgt_start[T], n = tgt_count[T];
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
#pragma unroll
      for (int k = 0; k < D; ++k) {
        const double xk = tgt[(t0 + j) * D + k];
        double2* o = tph + (p0 + j) * 3 * D + 3 * k;
        o[0] = phase_dd(-(n_f / 2), sc, xk, cr[k]);
        o[1] = phase_dd(1, sc, xk, cr[k]);
        o[2] = phase_dd(8, sc, xk, cr[k]);
      }
    }
  }
}

// One CTA per sibling group.  Per round of <= TR targets (member-aligned 8-target tiles),
// the targets' phase tables are built once in shared memory (E: last axis; E1: axis 1;
// E0: pair-weighted axis-0 factor per stored plane), then the CTA sweeps the chunks of
// RC = 8 RT stored rows: per chunk and member half each warp accumulates S_c for its 8 x 16
// mode tile (a plain sum of phi' over the sources serving c) and immediately contracts it
// with the half's target tiles (3-DMMA complex GEMM + row-factor epilogue), adding the
// target partials into its own s_part row.  No synchronisation inside the sweep; the
// warps' rows are summed in a fixed order at the end of the round (deterministic).
template <int D>
__global__ void __launch_bounds__(256, 2) gather_eval_kernel(
    GEArgs a, const int64_t* __restrict__ gt_slot, const unsigned* __restrict__ gt_code,
    const int* __restrict__ gt_nu, const int64_t* __restrict__ gt_out) {
  constexpr int NSIB = 1 << D;
  constexpr int NREL = 1 << (2 * D);
  // Members are processed in halves of MH (d = 3: 4 + 4) so the per-member accumulators
  // S_c stay in registers at 2 CTAs per SM.
  constexpr int MH = NSIB < 4 ? NSIB : 4;
  constexpr int NHALF = NSIB / MH;
  extern __shared__ double2 sm[];
  const int CB = a.CB, RT = a.RT, RC = RT * 8, TR = a.TR, NTL = TR / 8;
  const int n_f = a.n_f, nh = a.nh;
  const int ES = CB * 16 + 4, FS = nh + 1;
  double2* sE = sm;                                      // TR x ES: last-axis phases
  double2* s_e1 = sE + TR * ES;                          // TR x ES: axis-1 phases (d = 3)
  double2* s_e0 = s_e1 + TR * ES;                        // TR x FS: w x axis-0 phase per plane
  double* s_part = reinterpret_cast<double*>(s_e0 + TR * FS);     // 8 warps x TR
  double* u_bc = s_part + 8 * TR;                                   // NREL x 8: member c served
  const double2** u_ptr = reinterpret_cast<const double2**>(u_bc + NREL * 8);  // NREL
  unsigned* u_code = reinterpret_cast<unsigned*>(u_ptr + NREL);    // NREL
  int* u_list = reinterpret_cast<int*>(u_code + NREL);              // NHALF lists, NREL total
  int* t_mem = u_list + NREL;                                       // NTL: tile member
  int* t_off = t_mem + NTL;                                         // tile first target
  int* t_n = t_off + NTL;                                           // tile size
  int* s_rinfo = t_n + NTL;                                         // n_chunks * RC rows
  __shared__ int64_t m_cnt[NSIB], m_p0[NSIB], m_t0[NSIB];
  __shared__ int s_nl[NHALF], s_ntile;
  const int64_t g = blockIdx.x;
  const int nu = gt_nu[g];
  const int n_chunks = (a.RH + RC - 1) / RC;
  for (int u = threadIdx.x; u < nu; u += blockDim.x) {
    const unsigned code = gt_code[g * NREL + u];
    u_ptr[u] = a.phi + gt_slot[g * NREL + u] * a.NH;
    u_code[u] = code;
#pragma unroll
    for (int c = 0; c < 8; ++c) u_bc[u * 8 + c] = (c < NSIB && ((code >> c) & 1u)) ? 1.0 : 0.0;
  }
  for (int r = threadIdx.x; r < n_chunks * RC; r += blockDim.x) {
    int info = -1;
    if (r < a.RH) {
      const int s = D == 3 ? r / n_f : r;
      const int i1 = D == 3 ? r % n_f : 0;
      info = (D >= 2 ? s : 0) | (i1 << 8);
    }
    s_rinfo[r] = info;
  }
  if (threadIdx.x < NSIB) {
    const int c = threadIdx.x;
    const int64_t i = gt_out[g * NSIB + c];
    const int64_t ps = i >= 0 ? a.pstart[i] : -1;
    m_cnt[c] = 0;
    if (ps >= 0) {
      const int64_t T = a.psi_ids[i];
      m_cnt[c] = a.tgt_count[T];
      m_t0[c] = a.tgt_start[T];
      m_p0[c] = ps;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // compact source list per member half (sources serving no member of a half skipped)
    int k = 0;
    for (int h = 0; h < NHALF; ++h) {
      const int k0 = k;
      for (int u = 0; u < nu; ++u)
        if ((u_code[u] >> (h * MH)) & ((1u << MH) - 1u)) u_list[k++] = u;
      s_nl[h] = k - k0;
    }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nunits = RT * CB;
  const bool wactive = warp < nunits;
  const int rt = wactive ? warp / CB : 0, cb = wactive ? warp % CB : 0;
  const int rloc = rt * 8 + (lane >> 2);
  const int col0 = cb * 16 + (lane & 3);
  int pc = 0;
  int64_t poff = 0;
  for (;;) {
    // ---- round: list <= NTL member-aligned tiles, build their phase tables once
    __syncthreads();  // the previous round is done with tables, tile list and s_part
    if (threadIdx.x == 0) {
      int nt = 0;
      while (nt < NTL && pc < NSIB) {
        if (poff >= m_cnt[pc]) { ++pc; poff = 0; continue; }
        t_mem[nt] = pc;
        t_off[nt] = (int)poff;
        t_n[nt] = (int)min((int64_t)8, m_cnt[pc] - poff);
        poff += 8;
        ++nt;
      }
      s_ntile = nt;
    }
    __syncthreads();
    const int ntile = s_ntile;
    if (ntile == 0) break;
    {
      const int nseg = 2 * CB;
      const int nE = TR * nseg, nE1 = D == 3 ? TR * nseg : 0, nE0 = D >= 2 ? TR : 0;
      for (int task = threadIdx.x; task < nE + nE1 + nE0; task += blockDim.x) {
        int tt = task, kind = 0;
        if (tt >= nE) { tt -= nE; kind = 1; if (tt >= nE1) { tt -= nE1; kind = 2; } }
        const int slot = kind == 2 ? tt : tt / nseg, seg = kind == 2 ? 0 : tt % nseg;
        const int j = slot >> 3, k = slot & 7;
        const bool have = j < ntile && k < t_n[j];
        const double2* tp = have ? a.tph + (m_p0[t_mem[j]] + t_off[j] + k) * 3 * D : nullptr;
        if (kind < 2) {
          double2* out = (kind == 0 ? sE : s_e1) + slot * ES + seg * 8;
          if (!have) {
#pragma unroll
            for (int q = 0; q < 8; ++q) out[q] = make_double2(0.0, 0.0);
            continue;
          }
          const int ax = kind == 0 ? D - 1 : 1;
          double2 v = tp[3 * ax];
          const double2 st = tp[3 * ax + 1], st8 = tp[3 * ax + 2];
          for (int q = 0; q < seg; ++q) v = cmul(v, st8);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            out[q] = seg * 8 + q < n_f ? v : make_double2(0.0, 0.0);
            v = cmul(v, st);
          }
        } else {
          // stored plane s: mode m_0 = s (s < n_f/2, weight 2 unless s = 0) or -n_f/2
          double2* out = s_e0 + slot * FS;
          if (!have) {
            for (int q = 0; q < nh; ++q) out[q] = make_double2(0.0, 0.0);
            continue;
          }
          double2 v = make_double2(1.0, 0.0);
          const double2 st = tp[1];
          for (int q = 0; q < nh; ++q) {
            const int mi = half_plane_mi(q, n_f, a.half);
            const double w = half_plane_w(q, n_f, a.half);
            const double2 e = mi - n_f / 2 == q ? v : cmul(tp[0], cpow(st, mi));
            out[q] = make_double2(w * e.x, w * e.y);
            v = cmul(v, st);
          }
        }
      }
      for (int i = threadIdx.x; i < 8 * TR; i += blockDim.x) s_part[i] = 0.0;
    }
    __syncthreads();
    // ---- sweep over the mode chunks (no block synchronisation inside)
    if (wactive) {
#pragma unroll 1
      for (int chunk = 0; chunk < n_chunks; ++chunk) {
        const int64_t r = (int64_t)chunk * RC + rloc;
        // columns >= n_f read the next row, rows >= RH the next expansion or the zeroed pad:
        // finite values that meet zero table entries / zero row factors below
        const int64_t lane_off = r * n_f + col0;
        int lbase = 0;
#pragma unroll 1
        for (int hf = 0; hf < NHALF; ++hf) {
          const int cbase = hf * MH;
          const int nl = s_nl[hf];
          const int* lst = u_list + lbase;
          lbase += nl;
          bool any = false;
          for (int j = 0; j < ntile; ++j) any |= (t_mem[j] >= cbase && t_mem[j] < cbase + MH);
          if (!any) continue;
          double2 S[MH][4];
#pragma unroll
          for (int c = 0; c < MH; ++c)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) S[c][kk] = make_double2(0.0, 0.0);
          // phi' fragments double-buffered one source ahead (ping-pong)
          auto load = [&](int q, double2 (&f)[4]) {
            const double2* p = u_ptr[lst[q < nl ? q : nl - 1]] + lane_off;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) f[kk] = p[4 * kk];
          };
          auto accumulate = [&](int q, const double2 (&f)[4]) {
            const double* bcu = u_bc + lst[q] * 8 + cbase;
#pragma unroll
            for (int c = 0; c < MH; ++c) {
              const double bc = bcu[c];
#pragma unroll
              for (int kk = 0; kk < 4; ++kk) {
                S[c][kk].x = fma(bc, f[kk].x, S[c][kk].x);
                S[c][kk].y = fma(bc, f[kk].y, S[c][kk].y);
              }
            }
          };
          if (nl > 0) {
            double2 fa[4], fb[4];
            load(0, fa);
#pragma unroll 1
            for (int q = 0; q < nl; q += 2) {
              load(q + 1, fb);
              accumulate(q, fa);
              if (q + 1 >= nl) break;
              load(q + 2, fa);
              accumulate(q + 1, fb);
            }
          }
          // contract with the half's target tiles
#pragma unroll 1
          for (int j = 0; j < ntile; ++j) {
            const int c = t_mem[j] - cbase;
            if (c < 0 || c >= MH) continue;
            double2 B[4];
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) B[kk] = S[0][kk];
#pragma unroll
            for (int cc = 1; cc < MH; ++cc)
              if (cc == c) {
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) B[kk] = S[cc][kk];
              }
            double acc[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
            const double2* arow = sE + (j * 8 + (lane >> 2)) * ES + col0;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const double2 A = arow[kk * 4];
              const double2 Bk = B[kk];
              dmma(acc[0][0], acc[0][1], A.x + A.y, Bk.x);
              dmma(acc[1][0], acc[1][1], A.x, Bk.y - Bk.x);
              dmma(acc[2][0], acc[2][1], A.y, Bk.x + Bk.y);
            }
            double part = 0.0;
            const int tslot = j * 8 + (lane >> 2);
#pragma unroll
            for (int i2 = 0; i2 < 2; ++i2) {
              const int inf = s_rinfo[chunk * RC + rt * 8 + 2 * (lane & 3) + i2];
              double2 F = make_double2(0.0, 0.0);  // rows past RH hold unrelated finite data
              if (inf >= 0) {
                F = D >= 2 ? s_e0[tslot * FS + (inf & 255)] : make_double2(1.0, 0.0);
                if (D == 3) F = cmul(F, s_e1[tslot * ES + (inf >> 8)]);
              }
              const double re = acc[0][i2] - acc[2][i2], im = acc[0][i2] + acc[1][i2];
              part += re * F.x - im * F.y;
            }
            part += __shfl_xor_sync(0xffffffffu, part, 1);
            part += __shfl_xor_sync(0xffffffffu, part, 2);
            if ((lane & 3) == 0) s_part[warp * TR + tslot] += part;
          }
        }
      }
    }
    __syncthreads();
    // ---- the round's targets: warps' partials summed in a fixed order
    for (int slot = threadIdx.x; slot < ntile * 8; slot += blockDim.x) {
      const int j = slot >> 3, k = slot & 7;
      if (k >= t_n[j]) continue;
      double sum = 0.0;
      for (int w = 0; w < nunits; ++w) sum += s_part[w * TR + slot];
      a.u[m_t0[t_mem[j]] + t_off[j] + k] += sum;
    }
  }
}

// ------------------------------------------------------------------ eval
struct EvalArgs {
  const double* tgt;      // sorted targets
  const double* center;
  const int64_t* psi_ids;
  const int64_t* tgt_start;
  const int64_t* tgt_count;
  const int64_t* list;    // blockIdx.x -> psi index
  const int* pstart;      // blockIdx.x -> first target of this 32-target pass
  const double2* psi;
  double* u;
  int n_f, R, ksteps, half;  // R: stored rows (RH)
  double sc;
};

constexpr int EVAL_TB = 32;
constexpr int EVAL_MT = 4;

// One pass over the box's modes for up to 8*MTP targets whose phase tables are in etab;
// per-warp partial sums go to s_u[warp][target].  MTP is the number of 8-target m-tiles
// actually used, fixed at compile time so the last (partial) pass issues no idle DMMAs.
template <int D, int NT, int MTP>
__device__ __forceinline__ void eval_pass(const double2* __restrict__ etab, const double2* __restrict__ psi,
                                          double* __restrict__ s_u, const int* __restrict__ rinfo, int R,
                                          int n_f, int ksteps) {
  constexpr int TB = EVAL_TB, NFP = NT * 8, RS = NFP + 4;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  const int ntiles = (R + 7) / 8;
  double part[MTP];
#pragma unroll
  for (int mt = 0; mt < MTP; ++mt) part[mt] = 0.0;
  for (int nt = warp; nt < ntiles; nt += nwarps) {
    // complex MAC in three real products (Gauss): k1 = (a_r + a_i) b_r, k2 = a_r (b_i - b_r),
    // k3 = a_i (b_r + b_i); re = k1 - k3, im = k1 + k2.  Three independent accumulators per
    // m-tile: 3 DMMAs per complex MAC instead of 4, none waiting on another
    double acc[MTP][3][2];
#pragma unroll
    for (int mt = 0; mt < MTP; ++mt)
#pragma unroll
      for (int e = 0; e < 3; ++e) acc[mt][e][0] = acc[mt][e][1] = 0.0;
    const int rb = nt * 8 + (lane >> 2);
    const bool rv = rb < R;
    const double2* prow = psi + (size_t)(rv ? rb : 0) * n_f;
    // psi fragments prefetched two k-steps ahead (L2 latency behind the DMMAs)
    auto ldB = [&](int kk) {
      const int c = kk * 4 + (lane & 3);
      return (rv && kk < ksteps && c < n_f) ? prow[c] : make_double2(0.0, 0.0);
    };
    double2 Bn0 = ldB(0), Bn1 = ldB(1);
    for (int kk = 0; kk < ksteps; ++kk) {
      const int c = kk * 4 + (lane & 3);
      const double2 B = Bn0;
      Bn0 = Bn1;
      Bn1 = ldB(kk + 2);
      double2 A[MTP];
#pragma unroll
      for (int mt = 0; mt < MTP; ++mt) A[mt] = etab[((D - 1) * TB + mt * 8 + (lane >> 2)) * RS + c];
      const double bd = B.y - B.x, bs = B.x + B.y;
#pragma unroll
      for (int mt = 0; mt < MTP; ++mt) {
        dmma(acc[mt][0][0], acc[mt][0][1], A[mt].x + A[mt].y, B.x);
        dmma(acc[mt][1][0], acc[mt][1][1], A[mt].x, bd);
        dmma(acc[mt][2][0], acc[mt][2][1], A[mt].y, bs);
      }
    }
    // epilogue: per output row its axis-0/1 mode indices and pair weight from rinfo
#pragma unroll
    for (int i2 = 0; i2 < 2; ++i2) {
      const int r = nt * 8 + 2 * (lane & 3) + i2;
      if (r >= R) continue;
      const int info = rinfo[r];
      const int i0 = info & 255, i1 = (info >> 8) & 255;
      const double wp = (info >> 16) ? 2.0 : 1.0;
#pragma unroll
      for (int mt = 0; mt < MTP; ++mt) {
        const int j = mt * 8 + (lane >> 2);
        double2 f = make_double2(1.0, 0.0);
        if (D == 2) f = etab[(0 * TB + j) * RS + i0];
        if (D == 3) f = cmul(etab[(0 * TB + j) * RS + i0], etab[(1 * TB + j) * RS + i1]);
        const double re = acc[mt][0][i2] - acc[mt][2][i2], im = acc[mt][0][i2] + acc[mt][1][i2];
        part[mt] += wp * (re * f.x - im * f.y);
      }
    }
  }
#pragma unroll
  for (int mt = 0; mt < MTP; ++mt) {
    double v = part[mt];
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    if ((lane & 3) == 0) s_u[warp * TB + mt * 8 + (lane >> 2)] = v;
  }
}

template <int D, int NT>
__global__ void __launch_bounds__(256, 2) eval_kernel(EvalArgs a) {
  extern __shared__ double2 sm[];
  constexpr int TB = EVAL_TB, NFP = NT * 8, RS = NFP + 4;
  static_assert(EVAL_MT == 4, "eval passes are dispatched for 1..4 m-tiles");
  double2* etab = sm;
  double* s_u = reinterpret_cast<double*>(etab + D * TB * RS);
  int* rinfo = reinterpret_cast<int*>(s_u + 8 * TB);
  // per stored row: axis-0 mode index (half spectrum), axis-1 index, pair-weight flag
  for (int r = threadIdx.x; r < a.R; r += blockDim.x) {
    const int s = D == 3 ? r / a.n_f : r;
    const int i1 = D == 3 ? r % a.n_f : 0;
    rinfo[r] = half_plane_mi(s, a.n_f, a.half) | (i1 << 8) | ((half_plane_w(s, a.n_f, a.half) > 1.5) << 16);
  }
  // one CTA per 32-target pass of a psi box (work items listed box by box, so the
  // passes of one box run together and share psi through L2)
  const int64_t i = a.list[blockIdx.x];
  const int64_t T = a.psi_ids[i];
  const int64_t t0 = a.tgt_start[T];
  const int ntg = (int)a.tgt_count[T];
  double ctr[D];
#pragma unroll
  for (int k = 0; k < D; ++k) ctr[k] = a.center[T * D + k];
  const int nwarps = blockDim.x >> 5;
  const int n_f = a.n_f, R = a.R;
  const double2* psi = a.psi + (size_t)i * R * n_f;
  {
    const int p0 = a.pstart[blockIdx.x];
    const int cnt = min(TB, ntg - p0);
    __syncthreads();
    build_etab<D>(etab, TB, NFP, RS, a.tgt, t0 + p0, cnt, ctr, a.sc, +1.0, n_f);
    __syncthreads();
    switch ((cnt + 7) >> 3) {
      case 1: eval_pass<D, NT, 1>(etab, psi, s_u, rinfo, R, n_f, a.ksteps); break;
      case 2: eval_pass<D, NT, 2>(etab, psi, s_u, rinfo, R, n_f, a.ksteps); break;
      case 3: eval_pass<D, NT, 3>(etab, psi, s_u, rinfo, R, n_f, a.ksteps); break;
      default: eval_pass<D, NT, 4>(etab, psi, s_u, rinfo, R, n_f, a.ksteps); break;
    }
    __syncthreads();
    // deterministic cross-warp sum in a fixed order
    for (int t = threadIdx.x; t < cnt; t += blockDim.x) {
      double s = 0.0;
      for (int w = 0; w < nwarps; ++w) s += s_u[w * TB + t];
      a.u[t0 + p0 + t] += s;
    }
  }
}

// ------------------------------------------------------------------ direct
struct DirectArgs {
  const int64_t* d_tgt_ids;
  const int64_t* d_beg;   // entries of leaf i: [d_beg[i], d_end[i])
  const int64_t* d_end;
  const int64_t* d_src;
  const int32_t* d_v;
  const int64_t* src_start;
  const int64_t* src_count;
  const int64_t* tgt_start;
  const int64_t* tgt_count;
  const double* src;   // sorted
  const double* q;     // sorted
  const double* tgt;   // sorted
  double* u;
  double inv_delta, r2_cut, root_side;
  int64_t n;
};

// CTA-per-target-leaf near field (128 lanes = targets): for leaves holding many targets.
template <int D>
__global__ void __launch_bounds__(128) direct_kernel(DirectArgs a) {
  constexpr int TILE = 128;
  __shared__ double s_y[TILE * D];
  __shared__ double s_q[TILE];
  for (int64_t i = blockIdx.x; i < a.n; i += gridDim.x) {
    const int64_t T = a.d_tgt_ids[i];
    const int64_t e0 = a.d_beg[i], e1 = a.d_end[i];
    if (e0 == e1) continue;
    const int64_t t0 = a.tgt_start[T];
    const int ntg = (int)a.tgt_count[T];
    for (int tb = 0; tb < ntg; tb += blockDim.x) {
      const int j = tb + threadIdx.x;
      const bool valid = j < ntg;
      double x[D];
#pragma unroll
      for (int k = 0; k < D; ++k) x[k] = valid ? a.tgt[(t0 + j) * D + k] : 0.0;
      double acc = 0.0;
      for (int64_t e = e0; e < e1; ++e) {
        const int64_t S = a.d_src[e];
        const int64_t s0 = a.src_start[S];
        const int nsrc = (int)a.src_count[S];
        double shift[D];
#pragma unroll
        for (int k = 0; k < D; ++k) shift[k] = (double)a.d_v[e * D + k] * a.root_side;
        for (int sb = 0; sb < nsrc; sb += TILE) {
          const int nj = min(TILE, nsrc - sb);
          __syncthreads();
          for (int t = threadIdx.x; t < nj; t += blockDim.x) {
#pragma unroll
            for (int k = 0; k < D; ++k) s_y[t * D + k] = a.src[(s0 + sb + t) * D + k] + shift[k];
            s_q[t] = a.q[s0 + sb + t];
          }
          __syncthreads();
          if (valid) {
            for (int t = 0; t < nj; ++t) {
              double r2 = 0.0;
#pragma unroll
              for (int k = 0; k < D; ++k) {
                double df = x[k] - s_y[t * D + k];
                r2 += df * df;
              }
              if (r2 <= a.r2_cut) acc += exp(-r2 * a.inv_delta) * s_q[t];
            }
          }
        }
      }
      if (valid) a.u[t0 + j] += acc;
    }
  }
}

// Warp-per-target-leaf near field: lane = target (chunks of 32 targets), sources of each
// D-list box staged 32 at a time in the warp's shared-memory slice (coalesced loads, image
// shift applied) and read back as broadcasts.  Leaves are taken from a global counter, so a
// leaf with 6 targets occupies one warp instead of a 128-thread CTA; every target is summed
// by one lane in list order (deterministic).
template <int D>
__global__ void __launch_bounds__(256) direct_warp_kernel(DirectArgs a, int* __restrict__ counter) {
  __shared__ double s_y[8][32 * D];
  __shared__ double s_q[8][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* sy = s_y[warp];
  double* sq = s_q[warp];
  for (;;) {
    int64_t i = 0;
    if (lane == 0) i = atomicAdd(counter, 1);
    i = __shfl_sync(0xffffffffu, i, 0);
    if (i >= a.n) break;
    const int64_t T = a.d_tgt_ids[i];
    const int64_t e0 = a.d_beg[i], e1 = a.d_end[i];
    if (e0 == e1) continue;
    const int64_t t0 = a.tgt_start[T];
    const int ntg = (int)a.tgt_count[T];
    // leaves with <= 16 targets: NS = 32 / TW lanes share a target, each summing every NS-th
    // staged source; the lanes' partials meet in a fixed shuffle tree (deterministic)
    int TW = 32;
    while (TW > 1 && TW / 2 >= ntg) TW >>= 1;
    const int NS = 32 / TW, split = lane / TW;
    for (int tb = 0; tb < ntg; tb += TW) {
      const int j = tb + lane % TW;
      const bool valid = j < ntg;
      double x[D];
#pragma unroll
      for (int k = 0; k < D; ++k) x[k] = valid ? a.tgt[(t0 + j) * D + k] : 0.0;
      double acc = 0.0;
      for (int64_t e = e0; e < e1; ++e) {
        const int64_t S = a.d_src[e];
        const int64_t s0 = a.src_start[S];
        const int nsrc = (int)a.src_count[S];
        double shift[D];
#pragma unroll
        for (int k = 0; k < D; ++k) shift[k] = (double)a.d_v[e * D + k] * a.root_side;
        for (int sb = 0; sb < nsrc; sb += 32) {
          const int nj = min(32, nsrc - sb);
          __syncwarp();
          if (lane < nj) {
#pragma unroll
            for (int k = 0; k < D; ++k) sy[lane * D + k] = a.src[(s0 + sb + lane) * D + k] + shift[k];
            sq[lane] = a.q[s0 + sb + lane];
          }
          __syncwarp();
          if (valid) {
            for (int t = split; t < nj; t += NS) {
              double r2 = 0.0;
#pragma unroll
              for (int k = 0; k < D; ++k) {
                const double df = x[k] - sy[t * D + k];
                r2 += df * df;
              }
              if (r2 <= a.r2_cut) acc += exp(-r2 * a.inv_delta) * sq[t];
            }
          }
        }
      }
      for (int o = TW; o < 32; o <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (valid && split == 0) a.u[t0 + j] += acc;
    }
  }
}

template <int D, int NT>
void launch_form(PwDev& P, TreeDev& T, const FormArgs& fa, int nrowblk, int nunits, size_t smem,
                 cudaStream_t st) {
  FGT_CUDA(cudaFuncSetAttribute(form_kernel<D, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid(nrowblk, nunits);
  form_kernel<D, NT><<<grid, 256, smem, st>>>(fa);
  FGT_LAUNCHED();
}

template <int D, int NT>
void launch_eval(const EvalArgs& ea, int64_t n_psi, cudaStream_t st) {
  size_t smem = (size_t)D * EVAL_TB * (NT * 8 + 4) * sizeof(double2) + 8 * EVAL_TB * sizeof(double) +
                (size_t)ea.R * sizeof(int);
  FGT_CUDA(cudaFuncSetAttribute(eval_kernel<D, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  eval_kernel<D, NT><<<(unsigned)n_psi, 256, smem, st>>>(ea);
  FGT_LAUNCHED();
}

}  // namespace

// ====================================================================== host side

void pw_setup(PwDev& P, const TreeDev& T, const fgt_pw_params& pw) {
  pw_setup_dense(P, T, pw);
  pw_setup_psi(P, T);
}

// parameters, phase tables and the source count of every P-box slot (the form's inputs;
// no list is needed)
void pw_setup_dense(PwDev& P, const TreeDev& T, const fgt_pw_params& pw) {
  FGT_REQUIRE(pw.dim == T.d, FGT_EINVAL, "plane-wave dim != tree dim");
  // n_f even: the quadrature's modes -n_f/2 .. n_f/2-1; odd: the periodic root series
  // -n_p .. n_p (n_f = 2 n_p + 1)
  FGT_REQUIRE(pw.n_f >= 2, FGT_EINVAL, "n_f must be >= 2");
  FGT_REQUIRE(pw.n_f <= 64, FGT_ERANGE, "n_f > 64 not supported by the plane-wave kernels");
  cudaStream_t st = T.st;
  P.d = T.d;
  P.n_f = pw.n_f;
  P.R = 1;
  for (int k = 0; k < P.d - 1; ++k) P.R *= P.n_f;
  P.NF = P.R * P.n_f;
  P.half = P.d >= 2;
  P.nh = P.half ? P.n_f / 2 + 1 : P.n_f;
  P.RH = P.half ? P.R / P.n_f * P.nh : P.R;
  P.NH = P.RH * P.n_f;
  P.sc = pw.h / std::sqrt(pw.delta);
  P.side_lc = T.root_side;
  for (int l = 0; l < T.l_c; ++l) P.side_lc *= 0.5;
  P.w1d.alloc(P.n_f, st);
  P.w1d.from_host(pw.weights_1d, P.n_f);
  // translation path: fused (psi on chip) unless the level-l_c target leaves hold more
  // than GE_AUTO_MAX_TPL targets on average (evaluation then amortises a stored psi);
  // periodic image shifts keep the materialised path
  {
    const int m = psi_mode();
    const bool few = T.lc_targets <= GE_AUTO_MAX_TPL * std::max<int64_t>(1, T.lc_tleaves);
    P.fused = !T.periodic && (m == 2 || (m == 0 && few));
  }
  std::vector<double> ph(5 * 2 * P.n_f);
  for (int o = 0; o < 5; ++o)
    for (int mi = 0; mi < P.n_f; ++mi) {
      double m = (double)(mi - P.n_f / 2);
      double arg = m * P.sc * (double)(o - 2) * P.side_lc;
      ph[(o * P.n_f + mi) * 2] = std::cos(arg);
      ph[(o * P.n_f + mi) * 2 + 1] = std::sin(arg);
    }
  P.phase.alloc(ph.size(), st);
  P.phase.from_host(ph.data(), ph.size());
  const int64_t nd = T.n_dense;
  if ((int64_t)T.h_dense_src.size() == nd) {  // read back with the tree's finalize
    P.h_src = T.h_dense_src;
    return;
  }
  P.h_src.assign(nd, 0);
  if (nd > 0) {
    DBuf<int64_t> m(nd, st);
    gather_counts_kernel<<<grid_for(nd, 256), 256, 0, st>>>(T.dense_ids.get(), nd, T.src_count.get(), m.get());
    FGT_LAUNCHED();
    trace_mark(st, "setup:dense");
    m.to_host(P.h_src.data(), nd);
    FGT_CUDA(cudaStreamSynchronize(st));
    trace_mark(st, "setup:dense(sync)");
  }
}

// targets per psi box and the sibling groups of the psi boxes (after the lists), fetched
// with one sync on T.st
void pw_setup_psi(PwDev& P, const TreeDev& T) {
  cudaStream_t st = T.st;
  const int64_t n = T.n_psi;
  P.h_cnt.assign(n, 0);
  P.h_goff.assign(1, 0);
  std::vector<int64_t> h(2 * n);
  if (n > 0) {
    DBuf<int64_t> m(2 * n, st);
    psi_meta_kernel<<<grid_for(n, 256), 256, 0, st>>>(T.psi_ids.get(), n, T.tgt_count.get(), T.parent.get(),
                                                      m.get());
    FGT_LAUNCHED();
    trace_mark(st, "setup:psi");
    m.to_host(h.data(), h.size());
    FGT_CUDA(cudaStreamSynchronize(st));
    trace_mark(st, "setup:psi(sync)");
    std::copy(h.begin(), h.begin() + n, P.h_cnt.begin());
    const int64_t nsib = (int64_t)1 << P.d;
    for (int64_t i = 1; i < n; ++i) {
      const int64_t p = h[n + i];
      if (p < 0 || p != h[n + i - 1] || i - P.h_goff.back() >= nsib) P.h_goff.push_back(i);
    }
    P.h_goff.push_back(n);
  }
}

template <int D>
static void pw_form_impl(PwDev& P, TreeDev& T, const NufftPlan* N) {
  cudaStream_t st = T.st;
  const int64_t nd = T.n_dense;
  // + PHI_PAD zeroed double2 past the last expansion: the fused translation kernel reads
  // whole 8 x 16 mode tiles without bounds checks (columns >= n_f, rows >= RH)
  P.phi.alloc((size_t)nd * P.NH * 2 + 2 * PHI_PAD, st);
  P.phi.zero();
  if (nd == 0) return;
  // per-box source counts -> work units of at most KU points (split-K for big boxes)
  const std::vector<int64_t>& cnt = P.h_src;
  const int KU = 2048;
  std::vector<int4> units, reds;
  std::vector<int64_t> spread_slots;
  int nscratch = 0;
  for (int64_t s = 0; s < nd; ++s) {
    int64_t n = cnt[s];
    if (n == 0) continue;
    if (!T.dense_need.empty() && !T.dense_need[s]) continue;
    if (prefer_nufft(N, D, P.NH, n, 3.0)) {
      spread_slots.push_back(s);
      P.n_src_spread += n;
      continue;
    }
    int nu = (int)((n + KU - 1) / KU);
    if (nu == 1) {
      units.push_back(make_int4((int)s, 0, (int)n, -1));
    } else {
      reds.push_back(make_int4((int)s, nscratch, nu, 0));
      for (int t = 0; t < nu; ++t) {
        int k0 = t * KU;
        units.push_back(make_int4((int)s, k0, (int)std::min<int64_t>(KU, n - k0), nscratch++));
      }
    }
  }
  P.n_src_dense = 0;
  for (int64_t s = 0; s < nd; ++s) P.n_src_dense += cnt[s];
  P.n_spread_boxes = (int64_t)spread_slots.size();
  P.k_form.begin(st);
  if (P.fused) {
    // box phases e^{i m sc (c_ref - c_S)} per slot and axis (phase_dd), used by the d = 3
    // NUFFT's fused last stages and by the rephasing of every other expansion below
    P.bp.alloc((size_t)nd * D * P.n_f * 2, st);
    const double3 cref = make_double3(T.root_center[0], T.root_center[1], T.root_center[2]);
    box_phase_kernel<D><<<grid_for(nd * D * P.n_f, 256), 256, 0, st>>>(T.dense_ids.get(), nd, T.center.get(), cref,
                                                                         P.sc, P.n_f,
                                                                         reinterpret_cast<double2*>(P.bp.get()));
    FGT_LAUNCHED();
  }
  if (!spread_slots.empty()) nufft_form(*N, P, T, spread_slots);
  trace_mark(st, "form:nufft");
  // rephase the expansions not rephased by the d = 3 NUFFT stages (exact-sum boxes; all
  // boxes for d <= 2) once they are complete
  auto rephase_rest = [&](const std::vector<int64_t>& slots) {
    if (!P.fused || slots.empty()) return;
    DBuf<int64_t> sd(slots.size(), st);
    sd.from_host(slots.data(), slots.size());
    phi_rephase_kernel<D><<<grid_for((int64_t)slots.size(), 1, (int64_t)148 * 16), 256, P.RH * sizeof(double2), st>>>(
        reinterpret_cast<double2*>(P.phi.get()), (int64_t)slots.size(), sd.get(), P.NH, P.n_f, (int)P.RH, P.half,
        reinterpret_cast<const double2*>(P.bp.get()));
    FGT_LAUNCHED();
  };
  if (D <= 2) rephase_rest(spread_slots);
  std::vector<int64_t> exact_slots;
  for (const int4& u : units)
    if (exact_slots.empty() || exact_slots.back() != u.x) exact_slots.push_back(u.x);
  if (units.empty()) {
    P.k_form.end(st);
    return;
  }
  DBuf<int4> units_d(units.size(), st);
  units_d.from_host(units.data(), units.size());
  DBuf<double> scratch((size_t)nscratch * P.NH * 2, st);

  const int n_f = P.n_f;
  const int NT = (n_f + 7) / 8;
  const int mtiles = (int)((P.RH + 7) / 8);
  const int groups = (mtiles + FORM_MT - 1) / FORM_MT;
  int MG, KS, nrowblk;
  if (groups >= 8) { MG = 8; KS = 1; nrowblk = (groups + 7) / 8; }
  else { MG = groups; KS = 8 / MG; nrowblk = 1; }
  FormArgs fa;
  fa.src = T.src_sorted.get();
  fa.q = T.q_sorted.get();
  fa.center = T.center.get();
  fa.dense_ids = T.dense_ids.get();
  fa.src_start = T.src_start.get();
  fa.units = units_d.get();
  fa.phi = reinterpret_cast<double2*>(P.phi.get());
  fa.scratch = reinterpret_cast<double2*>(scratch.get());
  fa.w1d = P.w1d.get();
  fa.n_f = n_f;
  fa.R = (int)P.RH;
  fa.half = P.half;
  fa.MG = MG;
  fa.KS = KS;
  fa.sc = P.sc;
  const size_t etab_bytes = (size_t)D * FORM_KC * (NT * 8 + 2) * sizeof(double2) + FORM_KC * sizeof(double);
  const size_t red_bytes = (size_t)MG * 32 * FORM_MT * NT * 4 * sizeof(double);
  const size_t smem = std::max(etab_bytes, red_bytes);
  const int nunits = (int)units.size();
  switch (NT) {
#define FGT_FORM_CASE(NTV) case NTV: launch_form<D, NTV>(P, T, fa, nrowblk, nunits, smem, st); break;
    FGT_FORM_CASE(1) FGT_FORM_CASE(2) FGT_FORM_CASE(3) FGT_FORM_CASE(4)
    FGT_FORM_CASE(5) FGT_FORM_CASE(6) FGT_FORM_CASE(7) FGT_FORM_CASE(8)
#undef FGT_FORM_CASE
    default: throw Error(FGT_ERANGE, "n_f too large");
  }
  P.k_form.end(st);
  if (!reds.empty()) {
    DBuf<int4> reds_d(reds.size(), st);
    reds_d.from_host(reds.data(), reds.size());
    dim3 grid(grid_for(P.NH, 256, 64), (unsigned)reds.size());
    form_reduce_kernel<D><<<grid, 256, 0, st>>>(reinterpret_cast<const double2*>(scratch.get()), reds_d.get(),
                                                P.NH, n_f, (int)P.half, P.w1d.get(), reinterpret_cast<double2*>(P.phi.get()));
    FGT_LAUNCHED();
  }
  rephase_rest(exact_slots);
}

void pw_form(PwDev& P, TreeDev& T, const NufftPlan* N) {
  if (T.d == 1) pw_form_impl<1>(P, T, N);
  else if (T.d == 2) pw_form_impl<2>(P, T, N);
  else pw_form_impl<3>(P, T, N);
}

void pw_gather(PwDev& P, TreeDev& T, int64_t lo, int64_t hi) {
  cudaStream_t st = T.st;
  if (P.psi.size() < (size_t)(hi - lo) * P.NH * 2) P.psi.alloc((size_t)(hi - lo) * P.NH * 2, st);
  P.psi_lo = lo;
  P.psi_hi = hi;
  if (hi == lo) return;
  GatherArgs ga;
  ga.psi_ids = T.psi_ids.get();
  ga.p_off = T.p_off.get();
  ga.p_src = T.p_src.get();
  ga.p_v = T.p_v.get();
  ga.dense_ids = T.dense_ids.get();
  ga.coords = T.coords.get();
  ga.phase = reinterpret_cast<const double2*>(P.phase.get());
  ga.phi = reinterpret_cast<const double2*>(P.phi.get());
  ga.psi = reinterpret_cast<double2*>(P.psi.get());
  ga.NF = P.NH;
  ga.half = P.half;
  ga.i0 = lo;
  ga.n_f = P.n_f;
  ga.l_c = T.l_c;
  FGT_REQUIRE(hi - lo <= 65535, FGT_ERANGE, "psi batch too large");
  // sibling groups of this batch (clamped to [lo, hi))
  std::vector<int64_t> goff;
  {
    const auto& G = P.h_goff;
    size_t g = std::upper_bound(G.begin(), G.end(), lo) - G.begin() - 1;
    goff.push_back(lo);
    for (++g; g < G.size() && G[g] < hi; ++g) goff.push_back(G[g]);
    goff.push_back(hi);
  }
  DBuf<int64_t> goff_d(goff.size(), st);
  goff_d.from_host(goff.data(), goff.size());
  ga.goff = goff_d.get();
  const int64_t n_groups = (int64_t)goff.size() - 1;
  FGT_REQUIRE(n_groups <= 65535, FGT_ERANGE, "too many sibling groups");
  const int nrel = 1 << (2 * T.d), nsib = 1 << T.d;
  DBuf<int64_t> gt_slot(n_groups * nrel, st), gt_out(n_groups * nsib, st);
  DBuf<unsigned> gt_code(n_groups * nrel, st);
  DBuf<int> gt_nu(n_groups, st);
  FGT_REQUIRE((P.NH + GATHER_CHUNK - 1) / GATHER_CHUNK <= 65535, FGT_ERANGE, "too many mode chunks");
  dim3 grid((unsigned)n_groups, (unsigned)((P.NH + GATHER_CHUNK - 1) / GATHER_CHUNK));
  P.k_gather.begin(st);
#define FGT_GATHER_D(DD)                                                                      \
  group_table_kernel<DD><<<(unsigned)n_groups, 64, 0, st>>>(ga, gt_slot.get(), gt_code.get(), \
                                                             gt_nu.get(), gt_out.get());      \
  FGT_LAUNCHED();                                                                             \
  gather_kernel<DD><<<grid, GATHER_THREADS, 0, st>>>(ga, gt_slot.get(), gt_code.get(),        \
                                                     gt_nu.get(), gt_out.get());
  if (T.d == 1) { FGT_GATHER_D(1) }
  else if (T.d == 2) { FGT_GATHER_D(2) }
  else { FGT_GATHER_D(3) }
#undef FGT_GATHER_D
  FGT_LAUNCHED();
  P.k_gather.end(st);
}

void pw_eval(PwDev& P, TreeDev& T, double* u_sorted, const NufftPlan* N, int64_t lo, int64_t hi,
             bool nufft_only) {
  if (hi == lo) return;
  cudaStream_t st = T.st;
  std::vector<int64_t> direct_list, spread_list;
  const int64_t* h_cnt_all = P.h_cnt.data() + lo;
  {
    const int64_t n = hi - lo;
    const int64_t* h = h_cnt_all;
    for (int64_t i = 0; i < n; ++i) {
      if (prefer_nufft(N, T.d, P.NH, h[i], 2.0, 2.0)) {
        spread_list.push_back(lo + i);
        P.n_tgt_spread += h[i];
        P.n_tgt_psi += h[i];
      } else if (!nufft_only) {
        direct_list.push_back(lo + i);
        P.n_tgt_psi += h[i];
      }
    }
  }
  P.n_spread_psi += (int64_t)spread_list.size();
  trace_mark(st, "gather");
  P.k_eval.begin(st);
  if (!spread_list.empty()) nufft_eval(*N, P, T, spread_list, u_sorted);
  if (direct_list.empty()) {
    P.k_eval.end(st);
    return;
  }
  // work items: (psi box, 32-target pass)
  std::vector<int64_t> work_box;
  std::vector<int> work_p0;
  for (int64_t ii : direct_list) {
    const int64_t n = h_cnt_all[ii - lo];
    for (int64_t p0 = 0; p0 < n; p0 += EVAL_TB) {
      work_box.push_back(ii);
      work_p0.push_back((int)p0);
    }
  }
  DBuf<int64_t> list_d(work_box.size(), st);
  list_d.from_host(work_box.data(), work_box.size());
  DBuf<int> p0_d(work_p0.size(), st);
  p0_d.from_host(work_p0.data(), work_p0.size());
  const int64_t n_direct = (int64_t)work_box.size();
  EvalArgs ea;
  ea.tgt = T.tgt_sorted.get();
  ea.center = T.center.get();
  ea.psi_ids = T.psi_ids.get();
  ea.tgt_start = T.tgt_start.get();
  ea.tgt_count = T.tgt_count.get();
  ea.list = list_d.get();
  ea.pstart = p0_d.get();
  ea.psi = reinterpret_cast<const double2*>(P.psi_view());
  ea.u = u_sorted;
  ea.n_f = P.n_f;
  ea.R = (int)P.RH;
  ea.half = P.half;
  ea.ksteps = (P.n_f + 3) / 4;
  ea.sc = P.sc;
  const int NT = (P.n_f + 7) / 8;
#define FGT_EVAL_D(DD)                                              \
  switch (NT) {                                                     \
    case 1: launch_eval<DD, 1>(ea, n_direct, st); break;            \
    case 2: launch_eval<DD, 2>(ea, n_direct, st); break;            \
    case 3: launch_eval<DD, 3>(ea, n_direct, st); break;            \
    case 4: launch_eval<DD, 4>(ea, n_direct, st); break;            \
    case 5: launch_eval<DD, 5>(ea, n_direct, st); break;            \
    case 6: launch_eval<DD, 6>(ea, n_direct, st); break;            \
    case 7: launch_eval<DD, 7>(ea, n_direct, st); break;            \
    case 8: launch_eval<DD, 8>(ea, n_direct, st); break;            \
    default: throw Error(FGT_ERANGE, "n_f too large");              \
  }
  if (T.d == 1) { FGT_EVAL_D(1) }
  else if (T.d == 2) { FGT_EVAL_D(2) }
  else { FGT_EVAL_D(3) }
  P.k_eval.end(st);
#undef FGT_EVAL_D
}

void pw_gather_eval(PwDev& P, TreeDev& T, double* u_sorted, const NufftPlan* N) {
  const int64_t n = T.n_psi;
  if (n == 0) return;
  cudaStream_t st = T.st;
  if (!P.fused) {
    // translate into psi (<= 1 GB batches), then evaluate (exact DMMA sums or NUFFT)
    const int64_t per = P.NH * 16;
    const int64_t batch = std::max<int64_t>(1, std::min<int64_t>(65535, ((int64_t)1 << 30) / per));
    for (int64_t lo = 0; lo < n; lo += batch) {
      const int64_t hi = std::min(n, lo + batch);
      pw_gather(P, T, lo, hi);
      pw_eval(P, T, u_sorted, N, lo, hi);
    }
    P.psi.release();
    return;
  }
  // fused: every psi box, exact evaluation (the expansions are stored rephased)
  (void)N;
  std::vector<int64_t> pstart(n, -1);
  int64_t np = 0;
  for (int64_t i = 0; i < n; ++i) {
    pstart[i] = np;
    np += P.h_cnt[i];
  }
  if (np == 0) return;
  P.n_tgt_psi += np;
  const int n_f = P.n_f;
  const int CB = ge_cb(n_f), RT = ge_rt(n_f), TR = ge_tr(n_f);
  const std::vector<int64_t>& goff = P.h_goff;
  const int64_t n_groups = (int64_t)goff.size() - 1;
  const int nrel = 1 << (2 * T.d), nsib = 1 << T.d;
  DBuf<int64_t> pstart_d(n, st), goff_d(goff.size(), st);
  pstart_d.from_host(pstart.data(), n);
  goff_d.from_host(goff.data(), goff.size());
  DBuf<int64_t> gt_slot(n_groups * nrel, st), gt_out(n_groups * nsib, st);
  DBuf<unsigned> gt_code(n_groups * nrel, st);
  DBuf<int> gt_nu(n_groups, st);
  GatherArgs ga;
  std::memset(&ga, 0, sizeof(ga));
  ga.psi_ids = T.psi_ids.get();
  ga.p_off = T.p_off.get();
  ga.p_src = T.p_src.get();
  ga.p_v = T.p_v.get();
  ga.dense_ids = T.dense_ids.get();
  ga.coords = T.coords.get();
  ga.goff = goff_d.get();
  ga.i0 = 0;
  ga.n_f = n_f;
  ga.l_c = T.l_c;
  DBuf<double> tph((size_t)np * 6 * T.d, st);
  GEArgs ea;
  ea.psi_ids = T.psi_ids.get();
  ea.tgt_start = T.tgt_start.get();
  ea.tgt_count = T.tgt_count.get();
  ea.pstart = pstart_d.get();
  ea.tph = reinterpret_cast<const double2*>(tph.get());
  ea.phi = reinterpret_cast<const double2*>(P.phi.get());
  ea.u = u_sorted;
  ea.NH = P.NH;
  ea.n_f = n_f;
  ea.RH = (int)P.RH;
  ea.nh = T.d >= 2 ? (int)P.nh : 1;
  ea.half = P.half;
  ea.CB = CB;
  ea.RT = RT;
  ea.TR = TR;
  const size_t smem = ge_smem(n_f, T.d, (int)P.RH);
  FGT_REQUIRE(smem <= 227 * 1024, FGT_ERANGE, "fused translation/evaluation tables exceed shared memory");
  const double3 cref = make_double3(T.root_center[0], T.root_center[1], T.root_center[2]);
  P.k_gather.begin(st);
#define FGT_GE_D(DD)                                                                                   \
  group_table_kernel<DD><<<(unsigned)n_groups, 64, 0, st>>>(ga, gt_slot.get(), gt_code.get(),          \
                                                             gt_nu.get(), gt_out.get());               \
  FGT_LAUNCHED();                                                                                      \
  P.k_gather.end(st);                                                                                  \
  P.k_eval.begin(st);                                                                                  \
  ge_target_phase_kernel<DD><<<grid_for(n, 1, (int64_t)148 * 32), 128, 0, st>>>(                       \
      T.psi_ids.get(), T.tgt_start.get(), T.tgt_count.get(), pstart_d.get(), n, T.tgt_sorted.get(),    \
      cref, P.sc, n_f, reinterpret_cast<double2*>(tph.get()));                                         \
  FGT_LAUNCHED();                                                                                      \
  FGT_CUDA(cudaFuncSetAttribute(gather_eval_kernel<DD>, cudaFuncAttributeMaxDynamicSharedMemorySize,    \
                                (int)smem));                                                           \
  gather_eval_kernel<DD><<<(unsigned)n_groups, 256, smem, st>>>(ea, gt_slot.get(), gt_code.get(),      \
                                                               gt_nu.get(), gt_out.get());
  if (T.d == 1) { FGT_GE_D(1) }
  else if (T.d == 2) { FGT_GE_D(2) }
  else { FGT_GE_D(3) }
#undef FGT_GE_D
  FGT_LAUNCHED();
  P.k_eval.end(st);
}

void direct_lists(TreeDev& T, double inv_delta, double r2_cut, double* u_sorted, KClock* clk) {
  if (T.n_d == 0 || T.n_dtgt == 0) return;
  cudaStream_t st = T.st;
  DirectArgs da;
  da.d_tgt_ids = T.d_tgt_ids.get();
  da.d_beg = T.d_off.get();
  da.d_end = T.d_end.size() ? T.d_end.get() : T.d_off.get() + 1;
  da.d_src = T.d_src.get();
  da.d_v = T.d_v.get();
  da.src_start = T.src_start.get();
  da.src_count = T.src_count.get();
  da.tgt_start = T.tgt_start.get();
  da.tgt_count = T.tgt_count.get();
  da.src = T.src_sorted.get();
  da.q = T.q_sorted.get();
  da.tgt = T.tgt_sorted.get();
  da.u = u_sorted;
  da.inv_delta = inv_delta;
  da.r2_cut = r2_cut;
  da.root_side = T.root_side;
  da.n = T.n_dtgt;
  int dev = 0, nsm = 0;
  FGT_CUDA(cudaGetDevice(&dev));
  FGT_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  // persistent warps (8 per CTA, up to 8 CTAs per SM) taking target leaves from a counter
  const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>((T.n_dtgt + 7) / 8, (int64_t)nsm * 8));
  DBuf<int> counter(1, st);
  counter.zero();
  if (clk) clk->begin(st);
  // leaves of a few dozen targets (config 5: ~40 per leaf): a warp each; leaves holding
  // hundreds (dense clusters): a 128-thread CTA each
  const bool small = T.n_leaves > 0 && T.nt <= 48 * T.n_leaves;
  if (small) {
    if (T.d == 1) direct_warp_kernel<1><<<g, 256, 0, st>>>(da, counter.get());
    else if (T.d == 2) direct_warp_kernel<2><<<g, 256, 0, st>>>(da, counter.get());
    else direct_warp_kernel<3><<<g, 256, 0, st>>>(da, counter.get());
  } else {
    const unsigned gc = (unsigned)std::min<int64_t>(T.n_dtgt, (int64_t)nsm * 16);
    if (T.d == 1) direct_kernel<1><<<gc, 128, 0, st>>>(da);
    else if (T.d == 2) direct_kernel<2><<<gc, 128, 0, st>>>(da);
    else direct_kernel<3><<<gc, 128, 0, st>>>(da);
  }
  FGT_LAUNCHED();
  if (clk) clk->end(st);
}

}  // namespace fgt
