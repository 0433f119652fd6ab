#pragma once
#include "fgt_common.cuh"

namespace fgt {
void launch_gauss_direct_allpairs(const double* tgt, int64_t nt, const double* src, int64_t ns,
                                  const double* q, int d, double inv_delta, double r2_cut,
                                  bool periodic, double* out, cudaStream_t st);
void launch_nufft_spread(const double* x, int64_t M, int d, const double* vals, int64_t n_r,
                         int m_sp, double tau, double* grid, cudaStream_t st);
void launch_nufft_interp(const double* x, int64_t M, int d, const double* grid, int64_t n_r,
                         int m_sp, double tau, double* out, cudaStream_t st);
}  // namespace fgt
