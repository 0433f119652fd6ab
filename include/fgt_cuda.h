/*
 * fgt_cuda.h -- C ABI of libfgtcuda.so, the sm_100a (B200) hot path of the
 * plane-wave fast Gauss transform (Greengard, Jiang, Rachh, Wang; arXiv 2305.07165).
 *
 * Two layers:
 *
 *  1. Kernel-level drop-ins for the reference's compiled-backend slot
 *     `fgt._kernels_cy` (declared at /root/reference/pkg/setup.py:12-18, bound by
 *     /root/reference/pkg/src/fgt/backend.py:22-27).  Their contract is the numpy
 *     fallback /root/reference/pkg/src/fgt/_kernels_py.py:14-100.  All pointers are
 *     HOST pointers, caller-owned, C-contiguous float64 / complex128 (interleaved
 *     re,im).  Outputs are accumulated in place exactly as the numpy versions do.
 *
 *  2. Phase/pipeline entry points for the discrete transform (Alg 2,
 *     /root/reference/PAPER.md:840-872; contract SPEC.md:361-444): the GPU tree
 *     (Alg 1, reference tree.py:259-344), the P/D lists, and
 *     fgt_points.  `*_dev` variants take DEVICE pointers and a
 *     cudaStream_t (passed as void*), so a caller holding inputs already resident
 *     in HBM avoids the host round trip.
 *
 * Every function returns 0 on success.  Non-zero codes:
 *   FGT_EINVAL  (1)  bad argument        -> Python shim raises ValueError
 *   FGT_ECUDA   (2)  CUDA runtime error  -> RuntimeError (message via fgt_last_error)
 *   FGT_ERANGE  (3)  outside supported range (e.g. tree deeper than 19 levels in 3-D)
 *   FGT_ENOMEM  (4)  device allocation failed
 * Functions are reentrant.  Device scratch comes from two allocators: buffers under
 * 64 MB are stream-ordered (cudaMallocAsync pool); larger ones from a process-lifetime
 * cache of cudaMalloc blocks reused in stream order (cudaStreamWaitEvent on reuse) -- when
 * a new block does not fit, the cache frees its idle blocks after a cudaDeviceSynchronize
 * and retries once (FGT_ENOMEM if it still fails).
 */
#ifndef FGT_CUDA_H
#define FGT_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FGT_OK 0
#define FGT_EINVAL 1
#define FGT_ECUDA 2
#define FGT_ERANGE 3
#define FGT_ENOMEM 4

/* Thread-local text of the last error ("" if none). */
const char* fgt_last_error(void);
/* Library version string, e.g. "0.1.0+sm_100a". */
const char* fgt_version(void);
/* Number of kernel launches issued by this thread since the last reset. */
int64_t fgt_launch_count(void);
void fgt_reset_launch_count(void);

/* ---------------------------------------------------------------------------
 * Layer 1: kernel drop-ins (host pointers).
 * ------------------------------------------------------------------------- */

/* Replaces _kernels_py.gauss_direct (_kernels_py.py:14-30):
 *   out[i] += sum_j exp(-||tgt_i - src_j||^2 * inv_delta) * q_j, skipping pairs with
 *   r^2 > r2_cut (pass +inf to disable).  periodic != 0 replaces it with
 *   gauss_direct_periodic (_kernels_py.py:33-46): minimum image diff -= rint(diff). */
int fgt_gauss_direct(const double* tgt, int64_t nt, const double* src, int64_t ns,
                     const double* q, int d, double inv_delta, double r2_cut, int periodic,
                     double* out);

/* Replaces _kernels_py.nufft_spread (_kernels_py.py:65-81): Gaussian-kernel spreading
 *   grid[(i0+o) mod n_r] += exp(-z^2/(4 tau)) * val, z = x - (rint(x/h_r)+o) h_r,
 *   o in [-m_sp, m_sp] per axis, h_r = 2 pi / n_r.  x: (M,d) in [0,2pi); vals: (M,)
 *   complex128; grid: (n_r,)^d complex128 C-order, accumulated (caller zero-fills). */
int fgt_nufft_spread(const double* x, int64_t M, int d, const double* vals_c128,
                     int64_t n_r, int m_sp, double tau, double* grid_c128);

/* Replaces _kernels_py.nufft_interp (_kernels_py.py:84-100): out (M,) complex128 is
 *   overwritten with the adjoint gather of the same taps. */
int fgt_nufft_interp(const double* x, int64_t M, int d, const double* grid_c128,
                     int64_t n_r, int m_sp, double tau, double* out_c128);

/* Device-pointer variants of the three kernels (stream = cudaStream_t or NULL). */
int fgt_gauss_direct_dev(const double* tgt, int64_t nt, const double* src, int64_t ns,
                         const double* q, int d, double inv_delta, double r2_cut,
                         int periodic, double* out, void* stream);
int fgt_nufft_spread_dev(const double* x, int64_t M, int d, const double* vals_c128,
                         int64_t n_r, int m_sp, double tau, double* grid_c128, void* stream);
int fgt_nufft_interp_dev(const double* x, int64_t M, int d, const double* grid_c128,
                         int64_t n_r, int m_sp, double tau, double* out_c128, void* stream);

/* ---------------------------------------------------------------------------
 * Layer 2: discrete FGT pipeline.
 * ------------------------------------------------------------------------- */

/* Host-side plane-wave parameters.  The Python host computes them with the same
 * numpy expressions as planewave.pw_params (planewave.py:73-98) and
 * tree.cutoff_level (tree.py:24-50) so the tree is bit-identical; the library never
 * re-derives D0 from epsilon. */
typedef struct fgt_pw_params {
  int32_t dim;          /* 1, 2 or 3 */
  int32_t n_f;          /* modes per dimension (even) */
  double delta;         /* Gaussian variance */
  double D0;            /* sqrt(log(3/eps_clamped)) */
  double h;             /* mode spacing 2 pi / (R + D0) */
  const double* weights_1d; /* (n_f,) host array: h/(2 sqrt(pi)) exp(-m^2 h^2/4) */
} fgt_pw_params;

/* Tree construction controls (build_point_tree, tree.py:259-344). */
typedef struct fgt_tree_params {
  int32_t dim;
  int32_t periodic;     /* 0 free space, 1 unit cell [-1/2,1/2)^d with one image layer
                           (l_c >= 2), 2 root Fourier-series regime (l_c <= 1,
                           PAPER.md:1449-1453): the unit cell is the single box, n_s is
                           ignored, no image neighbours, no near field */
  int64_t n_s;          /* split boxes with more than n_s sources+targets */
  double D0;            /* cutoff factor (as above) */
  double delta;
  /* periodic trees only: l_c from cutoff_level(kind="density"), root side 1 */
  int32_t l_c_periodic;
  /* multi-GPU share: this process evaluates the targets of the part_rank-th of part_size
   * cost-balanced contiguous ranges of the target leaves in Morton order across levels
   * (key = Morton code at l_c of the leaf's first cell), so a share is a compact region
   * of space.  Two modes: fgt_points / fgt_points_dev form every P-box expansion the
   * range needs (the one-box halo is recomputed, no communication); fgt_points_begin ..
   * finish forms only the expansions the rank owns and the halo is exchanged between
   * begin and finish (fgt_points_pack / unpack + one all-to-all).  part_size <= 1 means
   * everything.  Targets outside the share get u = 0 (summing the shares gives u).
   * Every rank builds the same tree structure and lists from all the points; above 2^23
   * points the per-point tail of the build (per-leaf ascending order, leaf-ordered
   * coordinates) is done after the share is planned, for the rank's own leaves only. */
  int32_t part_rank;
  int32_t part_size;
} fgt_tree_params;

/* Split n items with non-negative costs into `parts` contiguous ranges of nearly
 * equal total cost: bounds[0..parts] (bounds[0] = 0, bounds[parts] = n).  Host-only. */
int fgt_partition_bounds(const double* cost, int64_t n, int32_t parts, int64_t* bounds);

/* Opaque GPU tree + partition, resident on the device. */
typedef struct fgt_tree fgt_tree;

/* Summary of a built tree. */
typedef struct fgt_tree_info {
  int32_t dim;
  int32_t l_c;
  int32_t n_levels;
  int32_t periodic;
  int64_t n_boxes;
  int64_t n_leaves;
  int64_t n_dense;      /* leaves at l_c holding > n_s points (the P-boxes) */
  int64_t n_sources;
  int64_t n_targets;
  double root_center[3];
  double root_side;
} fgt_tree_info;

/* Build the level-restricted tree of Alg 1 on the GPU from DEVICE arrays src (ns,d)
 * and tgt (nt,d).  Box order is canonical: level-major, Morton order within a level
 * (the reference numbers boxes by creation order; the box SET, parent/leaf relations,
 * per-leaf ascending index lists and subtree counts are bit-identical). */
int fgt_tree_build_dev(const double* src, int64_t ns, const double* tgt, int64_t nt,
                       const fgt_tree_params* prm, void* stream, fgt_tree** out);
int fgt_tree_get_info(const fgt_tree* t, fgt_tree_info* info);
/* Copy the tree to caller-owned HOST arrays (any pointer may be NULL to skip):
 * level (nb) i64, parent (nb) i64, children (nb, 2^d) i64, coords (nb, d) i64,
 * is_leaf (nb) u8, src_perm (ns) i64, tgt_perm (nt) i64, src_start/src_count/
 * tgt_start/tgt_count/n_points (nb) i64 -- the fields of tree.Tree (tree.py:53-115)
 * and tree.PointPartition (tree.py:246-256). */
int fgt_tree_copy_out(const fgt_tree* t, int64_t* level, int64_t* parent,
                      int64_t* children, int64_t* coords, uint8_t* is_leaf,
                      int64_t* src_perm, int64_t* tgt_perm, int64_t* src_start,
                      int64_t* src_count, int64_t* tgt_start, int64_t* tgt_count,
                      int64_t* n_points);
void fgt_tree_free(fgt_tree* t);

/* Interaction-list statistics for the built tree (target-centric P/D lists,
 * PAPER.md:769-788).  Counts are the entries (T,S,v) of each list. */
typedef struct fgt_list_info {
  int64_t n_p_entries;
  int64_t n_d_entries;
  int64_t n_psi_boxes;  /* target leaves with a non-empty P-list */
  int64_t n_direct_pairs; /* sum over D entries of n_tgt(T) * n_src(S) */
} fgt_list_info;
int fgt_tree_lists(fgt_tree* t, fgt_list_info* info);
/* Copy the lists out (host arrays sized from fgt_list_info); v is (n, d) int64. */
int fgt_tree_copy_lists(const fgt_tree* t, int64_t* p_tgt, int64_t* p_src, int64_t* p_v,
                        int64_t* d_tgt, int64_t* d_src, int64_t* d_v);

/* Per-phase device timings (ms, CUDA events) of the last fgt_points call. */
typedef struct fgt_phase_times {
  double tree_ms, lists_ms, form_ms, gather_ms, eval_ms, direct_ms, total_ms;
  double h2d_ms, d2h_ms;
  int64_t launches;
  /* device time of the hot kernels alone (CUDA events around each launch) */
  double k_form_ms, k_gather_ms, k_eval_ms, k_direct_ms;
  /* workload counters for algorithmic byte/flop accounting */
  int64_t n_boxes, n_dense, n_psi, n_src_dense, n_tgt_psi, n_p_entries, n_direct_pairs;
  int64_t n_modes; /* N_F = n_f^d */
  /* box-local NUFFT path: boxes / points routed to it and its kernel width and grid */
  int64_t n_spread_boxes, n_src_spread, n_spread_psi, n_tgt_spread;
  int32_t nufft_w, nufft_G;
} fgt_phase_times;

/* Discrete FGT, DEVICE pointers: u (nt) is OVERWRITTEN with
 *   u_i = sum_j exp(-||x_i - y_j||^2/delta) q_j   (relative l2 error <= ~eps)
 * following Alg 2 with the tree of fgt_tree_build_dev.  charges (ns) real. */
int fgt_points_dev(const double* src, int64_t ns, const double* charges,
                   const double* tgt, int64_t nt, const fgt_tree_params* tp,
                   const fgt_pw_params* pw, double* u, void* stream,
                   fgt_phase_times* times);
/* The same transform split at the multi-GPU exchange point (one process per GPU,
 * tp->part_rank / part_size set).  begin: tree, lists, this rank's cost-balanced share
 * of the target leaves, and the outgoing expansions of the P-boxes this rank OWNS (the
 * ones whose leaf lies in its range).  The one-box halo -- expansions owned by other
 * ranks that this rank's P-lists use -- is then exchanged: exchange_counts gives, per
 * peer, the slots to send and to receive (slot_doubles doubles each); pack writes this
 * rank's send slots, peer by peer, into a device buffer laid out for an all-to-all;
 * unpack scatters the received buffer (same peer order) into place.  finish: translation,
 * evaluation, near field; u (nt) gets this rank's targets (0 elsewhere).  All calls run on
 * the stream given to begin.  With part_size = 1 there is nothing to exchange. */
typedef struct fgt_points_run fgt_points_run;
int fgt_points_begin(const double* src, int64_t ns, const double* charges, const double* tgt,
                     int64_t nt, const fgt_tree_params* tp, const fgt_pw_params* pw, void* stream,
                     fgt_points_run** out);
int fgt_points_exchange_counts(const fgt_points_run* r, int64_t* send_slots, int64_t* recv_slots,
                               int64_t* slot_doubles);
int fgt_points_pack(fgt_points_run* r, double* send_buf);
int fgt_points_unpack(fgt_points_run* r, const double* recv_buf);
int fgt_points_finish(fgt_points_run* r, double* u, fgt_phase_times* times);
void fgt_points_run_free(fgt_points_run* r);

/* Same with HOST pointers; the H2D of inputs and D2H of u are inside the call. */
int fgt_points(const double* src, int64_t ns, const double* charges, const double* tgt,
               int64_t nt, const fgt_tree_params* tp, const fgt_pw_params* pw, double* u,
               fgt_phase_times* times);

/* ---------------------------------------------------------------------------
 * Layer 3: continuous (box) FGT, Alg 4.
 *
 * The density tree (Alg 3, tree.py:394-461) needs the user's sigma callable: the host
 * drives it (optionally with the per-grid tests on the device, fgt_box_tail_dev /
 * fgt_box_nodes_dev / fgt_box_balance_flags below); the host also builds the per-level 1-D
 * tables (J/I moments, poly1d.py:129-210) and the schedules below.  Everything else runs on
 * the GPU:
 * leaf->PW and PW->grid as d separable FP64-DMMA GEMMs per level, the diagonal
 * merge / gather / push shifts, and the direct near field as separable k x k
 * contractions.  All index arrays are HOST int64 arrays; complex = interleaved.
 * ------------------------------------------------------------------------- */
typedef struct fgt_box_plan {
  int32_t dim, k, n_f, n_levels, l_c;
  int64_t n_leaves;     /* leaf grids (values / u are (n_leaves, k^d)) */
  int64_t n_pw;         /* boxes with a plane-wave slot (f(B) = 1) */
  /* per-level 1-D matrices, complex (n_levels, n_f, k) and (n_levels, k, n_f) */
  const double* val2pw; /* (L/2) w_m conj(I[P_n](L m h / 2 sqrt(delta))) T_val->pol */
  const double* pw2val; /* exp(+i m h L xi_n / 2 sqrt(delta)) */
  /* phase rows, complex (n_rows, n_f); rows are referenced by the shift schedules */
  int64_t n_rows;
  const double* rows;
  /* direct tables, real (n_tables, k, k): (L/2) J_lam[P_n](2 o + r xi_i) T_val->pol */
  int64_t n_tables;
  const double* dtab;
  /* leaf -> PW: (leaf slot, pw slot, level) */
  int64_t n_form;
  const int64_t *form_leaf, *form_pw, *form_level;
  /* diagonal shifts, executed as stages in order; stage s covers destinations
   * [stage_off[s], stage_off[s+1]); kind 0 = merge (phi -> phi), 1 = gather
   * (phi -> psi), 2 = push (psi -> psi).  Per destination: pw slot, accumulate (1) or
   * overwrite (0), entries (src pw slot, d phase-row indices) summed in order. */
  int64_t n_stages, n_dst, n_entries;
  const int64_t *stage_off;  /* (n_stages+1) into dst list */
  const int64_t *stage_kind; /* (n_stages) */
  const int64_t *dst, *dst_acc, *dst_off; /* (n_dst), (n_dst), (n_dst+1) into entries */
  const int64_t *ent_src, *ent_rows;      /* (n_entries), (n_entries, d) */
  /* PW -> grid: (leaf slot, pw slot, level) */
  int64_t n_eval;
  const int64_t *eval_leaf, *eval_pw, *eval_level;
  /* direct pairs sorted by target leaf: (target leaf, source leaf, d table ids) */
  int64_t n_dpairs;
  const int64_t *d_tgt, *d_src, *d_tab;
} fgt_box_plan;

/* u (n_leaves, k^d) = box FGT of values (n_leaves, k^d); DEVICE pointers. */
int fgt_box_dev(const fgt_box_plan* plan, const double* values, double* u, void* stream,
                fgt_phase_times* times);
/* Same with HOST pointers (H2D / D2H inside). */
int fgt_box(const fgt_box_plan* plan, const double* values, double* u, fgt_phase_times* times);

/* Microbenchmarks used for the roofline denominators (FP64 pipes). */
/* interp_at (section 4.2 "simply use polynomial interpolation"):
 * evaluate the piecewise Legendre expansion of a box-FGT output at arbitrary points.
 * The tree is given by its leaves (host arrays); coeffs (n_leaves, k^dim) are the Legendre
 * coefficients of each leaf's k^dim grid values (LegendreBasis.val_to_pol per axis).  A
 * point is located by the deepest leaf containing it (periodic: wrapped into the cell). */
typedef struct fgt_interp_tree {
  int32_t dim, k, periodic, pad;
  int64_t n_leaves;
  const int32_t* level;   /* (n_leaves) */
  const int64_t* coords;  /* (n_leaves, dim), integer box coordinates at the box's level */
  const double* coeffs;   /* (n_leaves, k^dim) */
  double root_low[3];
  double root_side;
} fgt_interp_tree;
int fgt_box_interp(const fgt_interp_tree* t, const double* x, int64_t n, double* out);
int fgt_box_interp_dev(const fgt_interp_tree* t, const double* x, int64_t n, double* out,
                       void* stream);

/* ---------------------------------------------------------------------------
 * Alg 3 / 5 / 6 pieces on the device (the density tree and the output tree are decided
 * where the leaf grids live).
 *
 * fgt_box_tail: per leaf grid, the Legendre tail estimate of Eq. (funerr) -- values ->
 * coefficients axis by axis (poly1d.py:76-91), RMS of the coefficients with |alpha|_2 >= k
 * (tail_mask / tail_error, poly1d.py:100-126) -- and, if wsq is not NULL, the
 * quadrature-weighted sum of squares sum_i w_i v_i^2 (the caller scales by (side/2)^d).
 * val_to_pol (k, k) and weights (k) are HOST arrays (LegendreBasis, poly1d.py:50-73).
 * fgt_box_nodes_dev: the k^d tensor Gauss-Legendre nodes of n boxes (leaf_grid_points,
 * tree.py:384-391), pts (n, k^d, dim) on the device; level / coords / nodes are HOST arrays;
 * coordinates are rounded operation by operation like the reference's expressions.
 * fgt_box_balance_flags: one sweep of the level restriction (the condition of
 * _Builder.balance, tree.py:195-220): flags[j] = 1 for every leaf that covers a neighbour
 * cell of a leaf two or more levels deeper.  The caller splits the flagged leaves and calls
 * again until no flag is set; the result is the reference's box set (least fixpoint).
 * HOST arrays in any order. */
int fgt_box_tail_dev(const double* values, int64_t n, int dim, int k, const double* val_to_pol,
                     const double* weights, double* tail, double* wsq, void* stream);
int fgt_box_tail(const double* values, int64_t n, int dim, int k, const double* val_to_pol,
                 const double* weights, double* tail, double* wsq);
int fgt_box_nodes_dev(const int32_t* level, const int64_t* coords, int64_t n, int dim, int k,
                      const double* nodes, const double* root_low, double root_side, double* pts,
                      void* stream);
int fgt_box_balance_flags(const int32_t* level, const int64_t* coords, const uint8_t* is_leaf,
                          int64_t n, int dim, int periodic, uint8_t* flags);

/* Alg 5: output-tree refinement from RETAINED
 * incoming expansions.  fgt_box_retain = fgt_box that keeps psi of every f = 1 box and the
 * leaf grids of the density on the device (state).  fgt_box_refine evaluates new boxes
 * from that state: rplan is a box plan with n_form = 0 whose plane-wave slots [0, state
 * n_pw) are the retained ones and whose further slots are new children; its stages are
 * pushes only (kind 2: psi_child = T_p2c psi_parent), its eval list names the new leaves
 * (rows of u_new, (rplan->n_leaves, k^d), HOST) and its direct pairs take sources from the
 * retained leaf grids (d_src = leaf slot of the ORIGINAL transform) through the tables of
 * rplan (any centre offset / side ratio: the extended T_pol2pot tables of the Alg 5
 * Remark).  The state then also holds the new slots, so sweeps can be chained. */
typedef struct fgt_box_state fgt_box_state;
int fgt_box_retain(const fgt_box_plan* plan, const double* values, double* u, fgt_phase_times* times,
                   fgt_box_state** state);
int fgt_box_refine(fgt_box_state* state, const fgt_box_plan* rplan, double* u_new,
                   fgt_phase_times* times);
int fgt_box_state_free(fgt_box_state* state);

int fgt_bench_fp64_peak(int use_dmma, double* tflops);

#ifdef __cplusplus
}
#endif
#endif /* FGT_CUDA_H */
