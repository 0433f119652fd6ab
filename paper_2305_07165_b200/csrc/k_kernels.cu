// Kernel-level drop-ins for the reference backend slot fgt._kernels_cy.
//
//  gauss_direct / gauss_direct_periodic  <- _kernels_py.py:14-46
//  nufft_spread / nufft_interp           <- _kernels_py.py:49-100
//
// These are the generic all-pairs / all-taps forms with the reference's exact
// semantics (used by nufft.nufft_type1/2 and by the kernel-level parity tests).  The
// FGT pipeline itself uses the list-driven direct kernel (k_direct.cu) and the
// per-box plane-wave kernels (k_pw.cu).
#include <algorithm>

#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "fgt_common.cuh"
#include "k_kernels.cuh"

namespace fgt {

// ------------------------------------------------------------------ all-pairs direct
// One thread per target; sources stream through shared memory in tiles of TILE.
template <int D, bool PERIODIC>
__global__ void __launch_bounds__(256) gauss_direct_allpairs_kernel(
    const double* __restrict__ tgt, int64_t nt, const double* __restrict__ src, int64_t ns,
    const double* __restrict__ q, double inv_delta, double r2_cut, double* __restrict__ out) {
  constexpr int TILE = 256;
  __shared__ double s_src[TILE * D];
  __shared__ double s_q[TILE];
  const bool cut = r2_cut < INFINITY;
  for (int64_t t0 = (int64_t)blockIdx.x * blockDim.x; t0 < nt; t0 += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = t0 + threadIdx.x;
    double x[D];
    if (i < nt) {
#pragma unroll
      for (int k = 0; k < D; ++k) x[k] = tgt[i * D + k];
    }
    double acc = 0.0;
    for (int64_t j0 = 0; j0 < ns; j0 += TILE) {
      int nj = (int)((ns - j0) < TILE ? (ns - j0) : TILE);
      __syncthreads();
      for (int e = threadIdx.x; e < nj * D; e += blockDim.x) s_src[e] = src[j0 * D + e];
      for (int e = threadIdx.x; e < nj; e += blockDim.x) s_q[e] = q[j0 + e];
      __syncthreads();
      if (i < nt) {
        for (int j = 0; j < nj; ++j) {
          double r2 = 0.0;
#pragma unroll
          for (int k = 0; k < D; ++k) {
            double df = x[k] - s_src[j * D + k];
            if (PERIODIC) df -= rint(df);
            r2 += df * df;
          }
          double g = exp(-r2 * inv_delta);
          if (cut && r2 > r2_cut) g = 0.0;
          acc += g * s_q[j];
        }
      }
    }
    if (i < nt) out[i] += acc;
  }
}

void launch_gauss_direct_allpairs(const double* tgt, int64_t nt, const double* src, int64_t ns,
                                  const double* q, int d, double inv_delta, double r2_cut,
                                  bool periodic, double* out, cudaStream_t st) {
  if (nt == 0 || ns == 0) return;
  unsigned g = grid_for(nt, 256);
#define FGT_GD(DD, PP) gauss_direct_allpairs_kernel<DD, PP><<<g, 256, 0, st>>>(tgt, nt, src, ns, q, inv_delta, r2_cut, out)
  if (d == 1) { if (periodic) FGT_GD(1, true); else FGT_GD(1, false); }
  else if (d == 2) { if (periodic) FGT_GD(2, true); else FGT_GD(2, false); }
  else { if (periodic) FGT_GD(3, true); else FGT_GD(3, false); }
#undef FGT_GD
  FGT_LAUNCHED();
}

// ------------------------------------------------------------------ spreading
// Deterministic (no atomics): every (point, tap) contribution is keyed by its grid cell,
// the keys are stable-sorted with their (point, tap) position, and one thread per
// occupied cell adds the cell's contributions in that order -- ascending point index,
// then tap order, the accumulation order of the reference's np.add.at.  Per-axis weights
// as _kernels_py._spread_weights (:49-62):
//   i0 = rint(x / h_r); z_o = x - (i0 + o - m) h_r; w_o = exp(-z_o^2 / (4 tau)).
template <int D>
__global__ void spread_weights_kernel(const double* __restrict__ x, int64_t j0, int64_t nj, int n_r, int m_sp,
                                      double tau, double* __restrict__ w, int64_t* __restrict__ base) {
  const int nw = 2 * m_sp + 1;
  const double hr = 2.0 * M_PI / n_r;
  const double inv4tau = 1.0 / (4.0 * tau);
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nj * D;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = t / D;
    const int k = (int)(t % D);
    const double xk = x[(j0 + j) * D + k];
    const int64_t i0 = (int64_t)rint(xk / hr);
    for (int o = 0; o < nw; ++o) {
      const double z = xk - (double)(i0 + o - m_sp) * hr;
      w[(j * D + k) * nw + o] = exp(-z * z * inv4tau);
    }
    // first tap's cell, wrapped non-negative like Python's %
    base[j * D + k] = ((i0 - m_sp) % n_r + n_r) % n_r;
  }
}

template <int D>
__device__ __forceinline__ int64_t tap_cell(const int64_t* b, int64_t t, int nw, int n_r) {
  int64_t idx = 0;
  int64_t rem = t;
  int o[D];
#pragma unroll
  for (int k = D - 1; k >= 0; --k) {
    o[k] = (int)(rem % nw);
    rem /= nw;
  }
#pragma unroll
  for (int k = 0; k < D; ++k) idx = idx * n_r + (b[k] + o[k]) % n_r;
  return idx;
}

template <int D>
__global__ void spread_keys_kernel(const int64_t* __restrict__ base, int64_t nj, int nw, int n_r,
                                   uint64_t* __restrict__ key, int64_t* __restrict__ pos) {
  const int64_t T = [&] { int64_t v = 1; for (int k = 0; k < D; ++k) v *= nw; return v; }();
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nj * T;
       e += (int64_t)gridDim.x * blockDim.x) {
    key[e] = (uint64_t)tap_cell<D>(base + (e / T) * D, e % T, nw, n_r);
    pos[e] = e;
  }
}

__global__ void run_flag_kernel(const uint64_t* __restrict__ key, int64_t n, int* __restrict__ flag) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    flag[i] = (i == 0 || key[i] != key[i - 1]) ? 1 : 0;
}

template <int D>
__global__ void spread_runs_kernel(const uint64_t* __restrict__ key, const int64_t* __restrict__ pos, int64_t n,
                                   const int64_t* __restrict__ starts, const int* __restrict__ nruns,
                                   const double* __restrict__ w, const double* __restrict__ vals, int64_t j0,
                                   int nw, double* __restrict__ grid) {
  const int64_t T = [&] { int64_t v = 1; for (int k = 0; k < D; ++k) v *= nw; return v; }();
  const int64_t nr = *nruns;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nr; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = starts[r], b = r + 1 < nr ? starts[r + 1] : n;
    double sr = 0.0, si = 0.0;
    for (int64_t i = a; i < b; ++i) {
      const int64_t e = pos[i], j = e / T;
      int64_t rem = e % T;
      int o[D];
#pragma unroll
      for (int k = D - 1; k >= 0; --k) {
        o[k] = (int)(rem % nw);
        rem /= nw;
      }
      // weight product in axis order, as the reference's outer products (w0 w1) w2
      double wt = w[(j * D + 0) * nw + o[0]];
#pragma unroll
      for (int k = 1; k < D; ++k) wt *= w[(j * D + k) * nw + o[k]];
      sr += wt * vals[2 * (j0 + j)];
      si += wt * vals[2 * (j0 + j) + 1];
    }
    const int64_t c = (int64_t)key[a];
    grid[2 * c] += sr;
    grid[2 * c + 1] += si;
  }
}

template <int D>
__global__ void __launch_bounds__(128) nufft_interp_kernel(
    const double* __restrict__ x, int64_t M, const double* __restrict__ grid, int n_r, int m_sp,
    double tau, double* __restrict__ out) {
  const int nw = 2 * m_sp + 1;
  const double hr = 2.0 * M_PI / n_r;
  const double inv4tau = 1.0 / (4.0 * tau);
  extern __shared__ double s_w[];
  double* w = s_w + threadIdx.x * D * nw;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < M;
       j += (int64_t)gridDim.x * blockDim.x) {
    int64_t b[D];
#pragma unroll
    for (int k = 0; k < D; ++k) {
      double xk = x[j * D + k];
      int64_t i0 = (int64_t)rint(xk / hr);
      for (int o = 0; o < nw; ++o) {
        double z = xk - (double)(i0 + o - m_sp) * hr;
        w[k * nw + o] = exp(-z * z * inv4tau);
      }
      b[k] = ((i0 - m_sp) % n_r + n_r) % n_r;
    }
    double ar = 0.0, ai = 0.0;
    if (D == 1) {
      for (int o0 = 0; o0 < nw; ++o0) {
        int64_t idx = (b[0] + o0) % n_r;
        ar += w[o0] * grid[2 * idx];
        ai += w[o0] * grid[2 * idx + 1];
      }
    } else if (D == 2) {
      for (int o0 = 0; o0 < nw; ++o0) {
        int64_t r0 = ((b[0] + o0) % n_r) * n_r;
        double w0 = w[o0];
        for (int o1 = 0; o1 < nw; ++o1) {
          int64_t idx = r0 + (b[1] + o1) % n_r;
          double wt = w0 * w[nw + o1];
          ar += wt * grid[2 * idx];
          ai += wt * grid[2 * idx + 1];
        }
      }
    } else {
      for (int o0 = 0; o0 < nw; ++o0) {
        int64_t r0 = ((b[0] + o0) % n_r) * n_r;
        double w0 = w[o0];
        for (int o1 = 0; o1 < nw; ++o1) {
          int64_t r1 = (r0 + (b[1] + o1) % n_r) * n_r;
          double w01 = w0 * w[nw + o1];
          for (int o2 = 0; o2 < nw; ++o2) {
            int64_t idx = r1 + (b[2] + o2) % n_r;
            double wt = w01 * w[2 * nw + o2];
            ar += wt * grid[2 * idx];
            ai += wt * grid[2 * idx + 1];
          }
        }
      }
    }
    out[2 * j] = ar;
    out[2 * j + 1] = ai;
  }
}

void launch_nufft_spread(const double* x, int64_t M, int d, const double* vals, int64_t n_r,
                         int m_sp, double tau, double* grid, cudaStream_t st) {
  if (M == 0) return;
  const int nw = 2 * m_sp + 1;
  int64_t T = 1;
  for (int k = 0; k < d; ++k) T *= nw;
  FGT_REQUIRE(T <= ((int64_t)1 << 26), FGT_ERANGE, "spreading half-width too large");
  // points in batches of <= 2^25 contributions; batches add to the grid in order
  const int64_t per = std::max<int64_t>(1, ((int64_t)1 << 25) / T);
  const int64_t cap = std::min<int64_t>(M, per);
  DBuf<double> w(cap * d * nw, st);
  DBuf<int64_t> base(cap * d, st), pos(cap * T, st), spos(cap * T, st), starts(cap * T, st);
  DBuf<uint64_t> key(cap * T, st), skey(cap * T, st);
  DBuf<int> flag(cap * T, st), nruns(1, st);
  DBuf<uint8_t> tmp;
  int64_t iota_bits = 1;
  while (((int64_t)1 << iota_bits) <= n_r) ++iota_bits;
  const int kbits = (int)std::min<int64_t>(64, iota_bits * d);
  for (int64_t j0 = 0; j0 < M; j0 += cap) {
    const int64_t nj = std::min(cap, M - j0), ne = nj * T;
#define FGT_SP(DD)                                                                                        \
  spread_weights_kernel<DD><<<grid_for(nj * DD, 256), 256, 0, st>>>(x, j0, nj, (int)n_r, m_sp, tau, w.get(), \
                                                                   base.get());                          \
  FGT_LAUNCHED();                                                                                         \
  spread_keys_kernel<DD><<<grid_for(ne, 256), 256, 0, st>>>(base.get(), nj, nw, (int)n_r, key.get(), pos.get()); \
  FGT_LAUNCHED();
    if (d == 1) { FGT_SP(1) } else if (d == 2) { FGT_SP(2) } else { FGT_SP(3) }
#undef FGT_SP
    size_t bytes = 0;
    FGT_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, key.get(), skey.get(), pos.get(), spos.get(), (int)ne, 0, kbits, st));
    if (bytes > tmp.size()) tmp.alloc(bytes, st);
    FGT_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), bytes, key.get(), skey.get(), pos.get(), spos.get(), (int)ne, 0, kbits, st));
    count_launch();
    run_flag_kernel<<<grid_for(ne, 256), 256, 0, st>>>(skey.get(), ne, flag.get());
    FGT_LAUNCHED();
    bytes = 0;
    thrust::counting_iterator<int64_t> it(0);
    FGT_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, it, flag.get(), starts.get(), nruns.get(), (int)ne, st));
    if (bytes > tmp.size()) tmp.alloc(bytes, st);
    FGT_CUDA(cub::DeviceSelect::Flagged(tmp.get(), bytes, it, flag.get(), starts.get(), nruns.get(), (int)ne, st));
    count_launch();
#define FGT_SR(DD)                                                                                         \
  spread_runs_kernel<DD><<<grid_for(ne, 256), 256, 0, st>>>(skey.get(), spos.get(), ne, starts.get(), nruns.get(), \
                                                           w.get(), vals, j0, nw, grid);
    if (d == 1) { FGT_SR(1) } else if (d == 2) { FGT_SR(2) } else { FGT_SR(3) }
#undef FGT_SR
    FGT_LAUNCHED();
  }
}

void launch_nufft_interp(const double* x, int64_t M, int d, const double* grid, int64_t n_r,
                         int m_sp, double tau, double* out, cudaStream_t st) {
  if (M == 0) return;
  const int block = 128;
  size_t smem = (size_t)block * d * (2 * m_sp + 1) * sizeof(double);
  FGT_REQUIRE(smem <= 200 * 1024, FGT_ERANGE, "spreading half-width too large");
  unsigned g = grid_for(M, block);
  if (d == 1) {
    FGT_CUDA(cudaFuncSetAttribute(nufft_interp_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    nufft_interp_kernel<1><<<g, block, smem, st>>>(x, M, grid, (int)n_r, m_sp, tau, out);
  } else if (d == 2) {
    FGT_CUDA(cudaFuncSetAttribute(nufft_interp_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    nufft_interp_kernel<2><<<g, block, smem, st>>>(x, M, grid, (int)n_r, m_sp, tau, out);
  } else {
    FGT_CUDA(cudaFuncSetAttribute(nufft_interp_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    nufft_interp_kernel<3><<<g, block, smem, st>>>(x, M, grid, (int)n_r, m_sp, tau, out);
  }
  FGT_LAUNCHED();
}

}  // namespace fgt
