#pragma once
#include "k_tree.cuh"

namespace fgt {

// Plane-wave data of one discrete FGT evaluation.
// Half spectrum.  The charges are real, so every expansion is Hermitian:
// phi[-m] = conj(phi[m]) (the weights are even in m) and the same holds for psi (the
// translation phases are conj-symmetric).  For d >= 2 only nh = n_f/2 + 1 planes along
// axis 0 are stored: plane s holds m_0 = s for s < n_f/2 and m_0 = -n_f/2 for s = n_f/2
// (the one plane without a partner); the potential Re sum_m psi_m e^{ik.x} then weighs
// plane s by 1 (m_0 = 0 or -n_f/2) or 2 (the pair +-m_0).  The pairing m <-> -m is exact
// for every mode whose other components lie in [-n_f/2+1, n_f/2-1]; a paired-plane mode
// with some m_k = -n_f/2 (k >= 1) stands in for its out-of-range partner m_k = +n_f/2.
// Those modes carry weight w_{n_f/2}/w_0 = exp(-n_f^2 h^2/16) <= 0.24 eps at every
// configuration, so the quadrature changes by O(eps/16) relative.
__host__ __device__ inline int half_plane_mi(int s, int n_f, bool half) {
  return half ? (s + n_f / 2) % n_f : s;
}
__host__ __device__ inline double half_plane_w(int s, int n_f, bool half) {
  // odd n_f (symmetric modes -n_f/2 .. n_f/2, the periodic root series): only m_0 = 0 is
  // unpaired
  return (!half || s == 0 || ((n_f & 1) == 0 && s == n_f / 2)) ? 1.0 : 2.0;
}

struct PwDev {
  int d = 0, n_f = 0;
  bool half = false;   // half-spectrum storage (d >= 2)
  int nh = 0;          // stored axis-0 planes
  int64_t R = 0;       // rows n_f^(d-1)
  int64_t NF = 0;      // n_f^d modes
  int64_t RH = 0;      // stored rows nh * n_f^(d-2) (d >= 2), else R
  int64_t NH = 0;      // stored modes per expansion: RH * n_f
  double sc = 0;       // coordinate scale h / sqrt(delta)
  double side_lc = 0;  // cutoff box side
  DBuf<double> w1d;    // (n_f) pre-multiplied 1-D weights (planewave.py:33-70)
  DBuf<double> phase;  // (3, n_f) complex: exp(+i m sc o side_lc), o = -1, 0, 1
  DBuf<double> phi;    // (n_dense, RH, n_f) complex outgoing expansions
  DBuf<double> psi;    // (psi_hi - psi_lo, RH, n_f) complex incoming expansions (one batch)
  int64_t psi_lo = 0, psi_hi = 0;
  // base pointer such that psi_view() + 2 * i * NH addresses psi box i of the batch
  double* psi_view() const { return psi.get() - 2 * psi_lo * NH; }
  // fused translation path (pw_gather_eval): chosen before the form from the tree's
  // level-l_c target statistics; the expansions are then stored rephased to the root
  // centre, phi' = e^{i k.(c_ref - c_S)} phi (bp: (n_dense, d, n_f) complex box phases)
  bool fused = false;
  DBuf<double> bp;
  KClock k_form, k_gather, k_eval, k_direct;
  int64_t n_src_dense = 0, n_tgt_psi = 0, n_spread_boxes = 0, n_spread_psi = 0;
  int64_t n_src_spread = 0, n_tgt_spread = 0;
  // host copies fetched once after the lists: targets per psi box and sibling groups
  // (runs of psi boxes with a common parent, offsets into psi_ids)
  std::vector<int64_t> h_cnt, h_goff;
  std::vector<int64_t> h_src;  // sources per P-box slot
};

struct NufftPlan;

// Per-box path selection between the exact tensor-factored sums (DMMA) and the box-local
// NUFFT (spread + separable DFT): FGT_NUFFT_MODE=direct|spread forces one (tests);
// proxy = 3: form by proxy points + separable stages, evaluation as spread.
int nufft_mode();
// FGT_PSI=materialise | fused forces the translation path (A/B checks); 0 = automatic
int psi_mode();

void pw_setup(PwDev& P, const TreeDev& T, const fgt_pw_params& pw);  // = dense + psi
void pw_setup_dense(PwDev& P, const TreeDev& T, const fgt_pw_params& pw);
void pw_setup_psi(PwDev& P, const TreeDev& T);
// Form outgoing expansions of all P-boxes: type-1 exponential sums.
void pw_form(PwDev& P, TreeDev& T, const NufftPlan* N);
// Diagonal translation phi -> psi over the P-lists.
void pw_gather(PwDev& P, TreeDev& T, int64_t lo, int64_t hi);
// Type-2 evaluation of psi at the targets of every psi box; u_sorted += Re(...).
void pw_eval(PwDev& P, TreeDev& T, double* u_sorted, const NufftPlan* N, int64_t lo, int64_t hi,
             bool nufft_only = false);
// Translation fused with evaluation (psi kept on chip) for every psi box evaluated by the
// exact sums; boxes routed to the NUFFT interpolation keep the gather + pw_eval path.
void pw_gather_eval(PwDev& P, TreeDev& T, double* u_sorted, const NufftPlan* N);
// Direct near field over the D-lists (ball cut PAPER.md:909-915).
void direct_lists(TreeDev& T, double inv_delta, double r2_cut, double* u_sorted, KClock* clk);
// Continuous (box) FGT executor (k_volume.cu).
// State kept between a transform and the Alg 5 refinement sweeps that follow it: the
// incoming expansions of every f = 1 box and the leaf grids of the density, on the
// state's own stream ("incoming expansions retained for f=1 boxes").
struct BoxState {
  cudaStream_t st = nullptr;  // owned
  DBuf<double> psi, values;
  int64_t n_pw = 0, NF = 0, KD = 0, n_values = 0;
  int dim = 0, k = 0, n_f = 0;
};
void box_fgt(const fgt_box_plan& pl, const double* values, double* u, cudaStream_t st,
             fgt_phase_times* times, BoxState* retain = nullptr, BoxState* resume = nullptr);
// Legendre tail estimate (Eq. funerr; poly1d.py:100-126) and weighted square sum of n leaf
// grids; children-touching 2:1 balance flags of a box set (k_volume.cu)
void box_tail(const double* values, int64_t n, int dim, int k, const double* val_to_pol,
              const double* weights, double* tail, double* wsq, cudaStream_t st);
void box_nodes(const int32_t* level, const int64_t* coords, int64_t n, int dim, int k,
               const double* nodes, const double* root_low, double root_side, double* pts,
               cudaStream_t st);
void box_balance_flags(const uint64_t* keys, const uint8_t* leaf, int64_t n, int dim, int periodic,
                       uint8_t* flags, cudaStream_t st);
// interp_at of a box-FGT output (k_volume.cu)
void box_interp(const fgt_interp_tree& t, const double* x, int64_t n, double* out, cudaStream_t st);

}  // namespace fgt
