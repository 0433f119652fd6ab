// Box-local NUFFT path for forming / evaluating plane-wave expansions of heavy boxes.
#pragma once
#include "k_pw.cuh"

namespace fgt {

// Exponential-of-semicircle spreading kernel psi(t) = exp(beta (sqrt(1 - (2t/w)^2) - 1)),
// |t| <= w/2 grid cells, on a NON-periodic grid g*Delta, g in [gmin, gmin+G), that
// covers the scaled coordinates of one cutoff box (|x_k| <= X) plus the kernel support.
// Delta = 2 pi / (sigma n_f), sigma = 2.  Then, for |m| <= n_f/2,
//   exp(-i m x) ~= (1/fh(m)) sum_g psi(g - x/Delta) exp(-i m g Delta),
//   fh(m) = int psi(s) cos(m Delta s) ds           (Gauss-Legendre on the host)
// with aliasing error ~ tol (no FFT, no wrap: the grid is only 2X/Delta + w wide).
struct NufftPlan {
  int n_f = 0, w = 0, gmin = 0, G = 0;
  double beta = 0, Delta = 0, X = 0, tol = 0;
  std::vector<double> fh;   // (n_f)
  DBuf<double> Ef, EfT;     // form: (n_f, G) and (G, n_f) complex  w1d[m]/fh[m] e^{-i m g Delta}
  DBuf<double> Ee, EeT;     // eval: (G, n_f) and (n_f, G) complex        e^{+i m g Delta}/fh[m]
  DBuf<double> EfH;         // (nh, G): rows of Ef for the stored axis-0 planes (half spectrum)
  DBuf<double> EeH;         // (G, nh): columns of Ee for the stored planes x pair weight
  // piecewise-polynomial kernel weights (interior taps): hc[p * 16 + t] is the degree-p
  // coefficient of tap t in y = 2f - 1, f in [0, 1) the first tap's offset (see es_fit)
  int hdeg = 0;
  DBuf<double> hc;
  std::vector<double> w1d;  // (n_f) plane-wave weights the form matrices carry
  // proxy-point plans only (proxy_plan_cached): G = p Chebyshev nodes per axis on [-X, X]
  // and their barycentric weights; Ef / EfT / EfH then hold w1d[m] e^{-i m x_a}
  DBuf<double> cheb_x, cheb_lam;
};

void nufft_plan(NufftPlan& N, int n_f, double tol, double X, const double* w1d_host, cudaStream_t st);
// Process-lifetime cache of plans keyed by (device, n_f, tol, X, weights): the host-side
// quadrature and the six small matrix uploads happen once per parameter set.
const NufftPlan& nufft_plan_cached(int n_f, double tol, double X, const double* w1d_host, cudaStream_t st);

// Proxy-point form: the sources of a box are replaced by equivalent
// charges on a tensor grid of p Chebyshev proxy points per axis (Lagrange anterpolation as
// one real DMMA GEMM per box), then the proxy grid goes to the plane-wave basis in tensor
// product form with the same batched DMMA stages as the NUFFT path -- no spreading kernel,
// no sort.  p is the smallest order whose interpolation error of e^{-i m x}, weighted by
// the plane-wave weight of mode m, is below tol on the box.  FGT_NUFFT_MODE=proxy.
const NufftPlan& proxy_plan_cached(int n_f, double tol, double X, const double* w1d_host, cudaStream_t st);

// phi[slot] for the listed P-box slots, by spreading + separable DFT (DMMA GEMMs)
// (or, with FGT_NUFFT_MODE=proxy, by proxy points + the same separable stages).
void nufft_form(const NufftPlan& N, PwDev& P, TreeDev& T, const std::vector<int64_t>& slots);
// u_sorted += Re(psi_i evaluated at the targets of psi box i) for the listed psi indices.
void nufft_eval(const NufftPlan& N, PwDev& P, TreeDev& T, const std::vector<int64_t>& psi_idx,
                double* u_sorted);

}  // namespace fgt
