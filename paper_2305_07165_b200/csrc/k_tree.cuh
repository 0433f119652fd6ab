// Device-resident point tree (Alg 1) and P/D interaction lists.
#pragma once
#include <memory>

#include "fgt_common.cuh"

namespace fgt {

struct TreeDev {
  cudaStream_t st = nullptr;
  int d = 0, l_c = 0, periodic = 0, n_levels = 0;
  int64_t n_s = 0;
  double root_center[3] = {0, 0, 0}, root_low[3] = {0, 0, 0}, root_side = 0;
  int64_t ns = 0, nt = 0, ntot = 0;

  // points, sorted by Morton code at l_c (stable: ties keep combined index order)
  DBuf<uint64_t> pkey;    // (ntot)
  DBuf<int64_t> pidx;     // (ntot) combined index: <ns source, else ns+target
  DBuf<int64_t> pstart;   // coarse index of pkey (k_tree.cu PKeyIdx)

  // boxes in canonical order: level-major, Morton within level
  int64_t nb = 0, n_leaves = 0, n_dense = 0;
  std::vector<int64_t> level_off;  // host, n_levels+1
  DBuf<uint64_t> bkey;     // (nb) sorted box keys
  DBuf<int32_t> level;     // (nb)
  DBuf<int64_t> parent;    // (nb)
  DBuf<int64_t> children;  // (nb * 2^d)
  DBuf<int64_t> coords;    // (nb * d)
  DBuf<uint8_t> is_leaf;   // (nb)
  DBuf<int64_t> n_points, src_start, src_count, tgt_start, tgt_count;  // (nb)
  DBuf<int64_t> src_perm, tgt_perm;  // original index of each sorted point
  // general trees: the per-leaf ascending order may be deferred (order_leaf_points)
  bool defer_order = false, order_pending = false;
  DBuf<int64_t> seq_src, seq_tgt, src_end, tgt_end;
  DBuf<double> center;     // (nb * d) box centres (exact builder arithmetic)
  DBuf<int64_t> dense_ids;   // (n_dense) box ids of P-boxes
  DBuf<int64_t> dense_slot;  // (nb) index into dense_ids or -1
  std::vector<int64_t> h_dense_src;  // host: source count of every P-box (n_dense)
  int64_t lc_tleaves = 0, lc_targets = 0;  // host: level-l_c leaves with targets, their targets

  // lists (target-centric), built by build_lists()
  bool lists_built = false;
  int64_t n_p = 0, n_d = 0, n_psi = 0, n_direct_pairs = 0;  // n_direct_pairs < 0: on device
  DBuf<int64_t> pairs_dev;  // direct pair statistic (unsigned long long counter)
  DBuf<int64_t> p_off;   // (n_psi+1) CSR over psi boxes
  DBuf<int64_t> psi_ids; // (n_psi) target box ids with P entries
  DBuf<int64_t> p_src;   // (n_p) dense slot of S
  DBuf<int32_t> p_v;     // (n_p * d) image shifts
  DBuf<int64_t> p_tgt;   // (n_p) target box id (for copy-out)
  DBuf<int64_t> d_off;   // (n_dtgt+1) CSR over direct target leaves (begin of leaf i)
  DBuf<int64_t> d_end;   // multi-GPU share: (n_dtgt) end of leaf i (else d_off[i + 1])
  DBuf<int64_t> d_tgt_ids; // (n_dtgt)
  int64_t n_dtgt = 0;
  DBuf<int64_t> d_src;   // (n_d) source box id
  DBuf<int32_t> d_v;     // (n_d * d)
  DBuf<int64_t> d_tgt;   // (n_d) target box id

  // build_lists_begin -> build_lists_end intermediates (k_tree.cu)
  std::shared_ptr<void> lists_pending;

  // multi-GPU share: P-boxes whose expansions this rank needs (empty = all)
  std::vector<uint8_t> dense_need;

  // sorted point data (leaf-contiguous)
  DBuf<double> src_sorted, q_sorted, tgt_sorted;
};

// Build the tree from device points; D0/delta/n_s/periodic from tp.
void build_tree(TreeDev& T, const double* src, int64_t ns, const double* tgt, int64_t nt,
                const fgt_tree_params& tp, cudaStream_t st);
// Gather sorted coordinates (and charges, if given) into T.*_sorted.
void gather_sorted_points(TreeDev& T, const double* src, const double* q, const double* tgt);
// deferred per-leaf order of a general tree (all leaves, or the flagged ones)
void order_leaf_points(TreeDev& T, const uint8_t* need_src, const uint8_t* need_tgt);
// same for the boxes flagged in need_src / need_tgt only ((nb) device flags; multi-GPU shares)
void gather_needed_points(TreeDev& T, const double* src, const double* q, const double* tgt,
                          const uint8_t* need_src, const uint8_t* need_tgt);
// Target-centric P/D lists.  build_lists = begin + end; begin enqueues
// the enumeration and the read-back of the list sizes on T.st without blocking, end waits
// for the sizes and enqueues the compaction.
void build_lists(TreeDev& T);
void build_lists_begin(TreeDev& T);
void build_lists_end(TreeDev& T);
// direct-pair statistic of the lists (one device read, cached)
int64_t direct_pairs(TreeDev& T);

}  // namespace fgt
