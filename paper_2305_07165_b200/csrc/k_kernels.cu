// Kernel-level drop-ins for the reference backend slot fgt._kernels_cy.
//
//  gauss_direct / gauss_direct_periodic  <- _kernels_py.py:14-46
//  nufft_spread / nufft_interp           <- _kernels_py.py:49-100
//
// These are the generic all-pairs / all-taps forms with the reference's exact
// semantics (used by nufft.nufft_type1/2 and by the kernel-level parity tests).  The
// FGT pipeline itself uses the list-driven direct kernel (k_direct.cu) and the
// per-box plane-wave kernels (k_pw.cu).
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
// Per-axis base index and Gaussian weights, _kernels_py._spread_weights (:49-62):
//   i0 = rint(x / h_r); z_o = x - (i0 + o) h_r; w_o = exp(-z_o^2 / (4 tau)).
template <int D>
__global__ void __launch_bounds__(128) nufft_spread_kernel(
    const double* __restrict__ x, int64_t M, const double* __restrict__ vals, int n_r, int m_sp,
    double tau, double* __restrict__ grid) {
  const int nw = 2 * m_sp + 1;
  const double hr = 2.0 * M_PI / n_r;
  const double inv4tau = 1.0 / (4.0 * tau);
  extern __shared__ double s_w[];  // per thread: D * nw weights
  double* w = s_w + threadIdx.x * D * nw;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < M;
       j += (int64_t)gridDim.x * blockDim.x) {
    int64_t i0[D];
#pragma unroll
    for (int k = 0; k < D; ++k) {
      double xk = x[j * D + k];
      i0[k] = (int64_t)rint(xk / hr);
      for (int o = 0; o < nw; ++o) {
        double z = xk - (double)(i0[k] + o - m_sp) * hr;
        w[k * nw + o] = exp(-z * z * inv4tau);
      }
    }
    const double vr = vals[2 * j], vi = vals[2 * j + 1];
    // wrap base indices once; (i0 + o - m) mod n_r, non-negative like Python's %
    int64_t b[D];
#pragma unroll
    for (int k = 0; k < D; ++k) b[k] = ((i0[k] - m_sp) % n_r + n_r) % n_r;
    if (D == 1) {
      for (int o0 = 0; o0 < nw; ++o0) {
        int64_t idx = (b[0] + o0) % n_r;
        double wt = w[o0];
        atomicAdd(&grid[2 * idx], wt * vr);
        atomicAdd(&grid[2 * idx + 1], wt * vi);
      }
    } else if (D == 2) {
      for (int o0 = 0; o0 < nw; ++o0) {
        int64_t r0 = ((b[0] + o0) % n_r) * n_r;
        double w0 = w[o0];
        for (int o1 = 0; o1 < nw; ++o1) {
          int64_t idx = r0 + (b[1] + o1) % n_r;
          double wt = w0 * w[nw + o1];
          atomicAdd(&grid[2 * idx], wt * vr);
          atomicAdd(&grid[2 * idx + 1], wt * vi);
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
            atomicAdd(&grid[2 * idx], wt * vr);
            atomicAdd(&grid[2 * idx + 1], wt * vi);
          }
        }
      }
    }
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
  const int block = 128;
  size_t smem = (size_t)block * d * (2 * m_sp + 1) * sizeof(double);
  FGT_REQUIRE(smem <= 200 * 1024, FGT_ERANGE, "spreading half-width too large");
  unsigned g = grid_for(M, block);
  if (d == 1) {
    FGT_CUDA(cudaFuncSetAttribute(nufft_spread_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    nufft_spread_kernel<1><<<g, block, smem, st>>>(x, M, vals, (int)n_r, m_sp, tau, grid);
  } else if (d == 2) {
    FGT_CUDA(cudaFuncSetAttribute(nufft_spread_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    nufft_spread_kernel<2><<<g, block, smem, st>>>(x, M, vals, (int)n_r, m_sp, tau, grid);
  } else {
    FGT_CUDA(cudaFuncSetAttribute(nufft_spread_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    nufft_spread_kernel<3><<<g, block, smem, st>>>(x, M, vals, (int)n_r, m_sp, tau, grid);
  }
  FGT_LAUNCHED();
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
