// Continuous (box) FGT, Alg 4 of arXiv 2305.07165, on sm_100a.
//
//   leaf->PW   phi = (val2pw_l)^{(x)d} values          d separable DMMA GEMMs per level
//   merge      phi_B = sum_C T_c2p(C) . phi_C            diagonal shifts (HBM streams)
//   gather     psi_T = sum_S T_out2in(T,S) . phi_S       (l_c, P-list of SURVEY §3(D))
//   push       psi_C = T_p2c(C) . psi_B
//   eval       u = Re (pw2val_l)^{(x)d} psi            d separable DMMA GEMMs per level
//   direct     u_T += (D1 (x) D2 (x) D3) values_S      real k x k tables, 11 per level
// The reference has no Alg 4 code (SPEC.md:446-542 specifies it); the per-axis
// contractions are its `_apply_per_axis` pattern (poly1d.py:76-81).
#include <algorithm>
#include <map>

#include "k_gemm.cuh"
#include "k_pw.cuh"

namespace fgt {

namespace {

int64_t ipw(int64_t b, int e) {
  int64_t r = 1;
  while (e--) r *= b;
  return r;
}

// ---------------------------------------------------------------- diagonal shifts
struct ShiftArgs {
  const int64_t* dst;
  const int64_t* dst_acc;
  const int64_t* dst_off;
  const int64_t* ent_src;
  const int64_t* ent_rows;
  const double2* rows;
  const double2* src;   // phi or psi
  double2* out;         // phi or psi
  int64_t NF, d0;       // first dst of this stage
  int n_f, D;
};

constexpr int SHIFT_MAXE = 64;

template <int D>
__global__ void __launch_bounds__(256) shift_kernel(ShiftArgs a) {
  __shared__ int64_t s_src[SHIFT_MAXE];
  __shared__ int s_row[SHIFT_MAXE][D];
  const int64_t t = a.d0 + blockIdx.y;
  const int64_t e0 = a.dst_off[t];
  const int64_t ne64 = a.dst_off[t + 1] - e0;
  const int ne = (int)(ne64 < SHIFT_MAXE ? ne64 : SHIFT_MAXE);
  for (int i = threadIdx.x; i < ne; i += blockDim.x) {
    s_src[i] = a.ent_src[e0 + i];
#pragma unroll
    for (int k = 0; k < D; ++k) s_row[i][k] = (int)a.ent_rows[(e0 + i) * D + k];
  }
  __syncthreads();
  const bool acc_in = a.dst_acc[t] != 0;
  double2* out = a.out + a.dst[t] * a.NF;
  const unsigned n_f = (unsigned)a.n_f, NF = (unsigned)a.NF;  // n_f^d < 2^32
  for (unsigned e = blockIdx.x * blockDim.x + threadIdx.x; e < NF; e += gridDim.x * blockDim.x) {
    int m[D];
    unsigned rem = e;
#pragma unroll
    for (int k = D - 1; k >= 0; --k) {
      m[k] = (int)(rem % n_f);
      rem /= n_f;
    }
    double2 acc = acc_in ? out[e] : make_double2(0.0, 0.0);
    // entries four at a time: the four expansion loads are issued before any phase product
    // (same summation order as one at a time)
    for (int i0 = 0; i0 < ne; i0 += 4) {
      double2 f[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (i0 + u < ne) f[u] = __ldg(a.src + s_src[i0 + u] * a.NF + e);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u;
        if (i >= ne) break;
        double2 p = __ldg(a.rows + (int64_t)s_row[i][0] * n_f + m[0]);
#pragma unroll
        for (int k = 1; k < D; ++k) {
          const double2 q = __ldg(a.rows + (int64_t)s_row[i][k] * n_f + m[k]);
          p = make_double2(p.x * q.x - p.y * q.y, p.x * q.y + p.y * q.x);
        }
        acc.x += p.x * f[u].x - p.y * f[u].y;
        acc.y += p.x * f[u].y + p.y * f[u].x;
      }
    }
    out[e] = acc;
  }
}

__global__ void repeat_kernel(const int64_t* __restrict__ in, int64_t n, int rep, int stride, int off,
                              int64_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n * rep;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[(i / rep) * stride + off];
}

__global__ void pair_reduce_kernel(const double* __restrict__ Y, const int64_t* __restrict__ toff,
                                   const int64_t* __restrict__ tleaf, int64_t kd, double* __restrict__ u) {
  const int64_t t = blockIdx.y;
  const int64_t p0 = toff[t], p1 = toff[t + 1];
  double* ut = u + tleaf[t] * kd;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < kd;
       e += (int64_t)gridDim.x * blockDim.x) {
    double s = ut[e];
    for (int64_t p = p0; p < p1; ++p) s += Y[p * kd + e];
    ut[e] = s;
  }
}

// Fused 3-D direct near field: one CTA per target leaf walks its (sorted) D-pairs; per
// pair the source leaf's k^3 values and the three k x k tables sit in shared memory and
// Y = (D0 (x) D1 (x) D2) V is formed by three DMMA contractions (V -> X1 -> X2 -> Y) with
// no global intermediates; Y accumulates in registers across the target's pairs (fixed
// pair order: deterministic) and is added to u once.  KP = k padded to a multiple of 8.
template <int KP, int NW>
__global__ void __launch_bounds__(32 * NW) direct3_kernel(const double* __restrict__ values, const double* __restrict__ dtab,
                                                      const int64_t* __restrict__ toff, const int64_t* __restrict__ tleaf,
                                                      const int64_t* __restrict__ src, const int64_t* __restrict__ tab,
                                                      int k, double* __restrict__ u) {
  // padded row stride: KP + 4 = 4 mod 16 doubles, so the 16 lanes of a half-warp fragment
  // load (4 rows x 4 columns, either orientation) hit 16 distinct double-bank pairs
  constexpr int RS = KP + 4;
  constexpr int NT1 = KP * KP / 8 * (KP / 8);  // C tiles per stage
  constexpr int TPW = NT1 / NW;         // tiles per warp
  extern __shared__ double dsm[];
  double* Vb = dsm;                     // (KP*KP) x RS : V, later X2
  double* X1 = Vb + KP * KP * RS;       // (KP*KP) x RS
  double* Tb = X1 + KP * KP * RS;       // 3 x KP x RS : D0, D1, D2
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t t = blockIdx.x;
  const int64_t p0 = toff[t], p1 = toff[t + 1];
  const int64_t kd = (int64_t)k * k * k;
  double acc[TPW][2];
#pragma unroll
  for (int i = 0; i < TPW; ++i) acc[i][0] = acc[i][1] = 0.0;
  const int r8 = lane >> 2, c4 = lane & 3;
  for (int64_t p = p0; p < p1; ++p) {
    __syncthreads();  // previous pair's buffers are free
    const double* vs = values + src[p] * kd;
    for (int i = threadIdx.x; i < KP * KP * KP; i += blockDim.x) {
      const int a = i / (KP * KP), b = (i / KP) % KP, c = i % KP;
      Vb[(a * KP + b) * RS + c] = (a < k && b < k && c < k) ? vs[((int64_t)a * k + b) * k + c] : 0.0;
    }
    for (int i = threadIdx.x; i < 3 * KP * KP; i += blockDim.x) {
      const int ax = i / (KP * KP), n = (i / KP) % KP, a = i % KP;
      const double* tb = dtab + tab[p * 3 + ax] * (int64_t)k * k;
      Tb[(ax * KP + n) * RS + a] = (n < k && a < k) ? tb[n * k + a] : 0.0;
    }
    __syncthreads();
    // stage 1: X1[(a b)][n3] = sum_c V[(a b)][c] D2[n3][c]
    for (int tt = warp; tt < NT1; tt += NW) {
      const int mt = tt / (KP / 8), nt = tt % (KP / 8);
      double c0 = 0.0, c1 = 0.0;
#pragma unroll
      for (int kk = 0; kk < KP; kk += 4) {
        const double A = Vb[(mt * 8 + r8) * RS + kk + c4];
        const double B = Tb[(2 * KP + nt * 8 + r8) * RS + kk + c4];
        dmma2(c0, c1, A, B);
      }
      X1[(mt * 8 + r8) * RS + nt * 8 + 2 * c4] = c0;
      X1[(mt * 8 + r8) * RS + nt * 8 + 2 * c4 + 1] = c1;
    }
    __syncthreads();
    // stage 2: X2[(a n2)][n3] = sum_b D1[n2][b] X1[(a b)][n3]   (into Vb)
    for (int tt = warp; tt < NT1; tt += NW) {
      const int a = tt / ((KP / 8) * (KP / 8)), rem = tt % ((KP / 8) * (KP / 8));
      const int mt = rem / (KP / 8), nt = rem % (KP / 8);
      double c0 = 0.0, c1 = 0.0;
#pragma unroll
      for (int kk = 0; kk < KP; kk += 4) {
        const double A = Tb[(KP + mt * 8 + r8) * RS + kk + c4];
        const double B = X1[(a * KP + kk + c4) * RS + nt * 8 + r8];
        dmma2(c0, c1, A, B);
      }
      Vb[(a * KP + mt * 8 + r8) * RS + nt * 8 + 2 * c4] = c0;
      Vb[(a * KP + mt * 8 + r8) * RS + nt * 8 + 2 * c4 + 1] = c1;
    }
    __syncthreads();
    // stage 3: Y[n1][(n2 n3)] += sum_a D0[n1][a] X2[(a n2)][n3]   (registers)
#pragma unroll
    for (int i = 0; i < TPW; ++i) {
      const int tt = warp + NW * i;
      const int mt = tt / (KP * KP / 8), nt = tt % (KP * KP / 8);
      const int col = nt * 8 + r8, n2 = col / KP, n3 = col % KP;
#pragma unroll
      for (int kk = 0; kk < KP; kk += 4) {
        const double A = Tb[(mt * 8 + r8) * RS + kk + c4];
        const double B = Vb[((kk + c4) * KP + n2) * RS + n3];
        dmma2(acc[i][0], acc[i][1], A, B);
      }
    }
  }
  // u[T] += Y  (fragment: row n1 = 8 mt + lane/4, cols 8 nt + 2 (lane%4) + {0, 1})
  double* ut = u + tleaf[t] * kd;
#pragma unroll
  for (int i = 0; i < TPW; ++i) {
    const int tt = warp + NW * i;
    const int mt = tt / (KP * KP / 8), nt = tt % (KP * KP / 8);
    const int n1 = mt * 8 + r8;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int col = nt * 8 + 2 * c4 + j, n2 = col / KP, n3 = col % KP;
      if (n1 < k && n2 < k && n3 < k) ut[((int64_t)n1 * k + n2) * k + n3] += acc[i][j];
    }
  }
}

template <class T>
DBuf<T> upload(const T* h, int64_t n, cudaStream_t st) {
  DBuf<T> d(n, st);
  if (n) d.from_host(h, n);
  return d;
}

struct LevelList {
  std::vector<int64_t> leaf, pw;
};

std::map<int, LevelList> group_by_level(int64_t n, const int64_t* leaf, const int64_t* pw,
                                        const int64_t* level) {
  std::map<int, LevelList> g;
  for (int64_t i = 0; i < n; ++i) {
    auto& L = g[(int)level[i]];
    L.leaf.push_back(leaf[i]);
    L.pw.push_back(pw[i]);
  }
  return g;
}

// complex transpose (rows x cols) -> (cols x rows), interleaved
std::vector<double> ctranspose(const double* a, int rows, int cols) {
  std::vector<double> t(2 * (size_t)rows * cols);
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < cols; ++c) {
      t[2 * ((size_t)c * rows + r)] = a[2 * ((size_t)r * cols + c)];
      t[2 * ((size_t)c * rows + r) + 1] = a[2 * ((size_t)r * cols + c) + 1];
    }
  return t;
}

// retain: the incoming expansions psi are handed to the state instead of being freed
// (Alg 5's "incoming expansions retained for f = 1 boxes").  resume: no
// leaf->PW / merge / gather; psi starts as the state's expansions (slots [0, state n_pw))
// plus zeroed new slots, the plan's stages may only push (kind 2), and the grown psi goes
// back into the state.
template <int D>
void box_impl(const fgt_box_plan& pl, const double* values, double* u, cudaStream_t st,
              fgt_phase_times* times, BoxState* retain, BoxState* resume) {
  const int k = pl.k, n_f = pl.n_f, L = pl.n_levels;
  const int64_t KD = ipw(k, D), NF = ipw(n_f, D);
  FGT_REQUIRE(pl.dim == D, FGT_EINVAL, "plan dim");
  FGT_REQUIRE(k >= 2 && k <= 32 && n_f >= 2 && n_f <= 128, FGT_ERANGE, "unsupported k / n_f");
  KClock c_form, c_shift, c_eval, c_direct;
  // ---- tables
  const size_t mat = 2 * (size_t)n_f * k;
  DBuf<double> v2p = upload(pl.val2pw, (int64_t)L * mat, st);      // (L, n_f, k)
  DBuf<double> p2v = upload(pl.pw2val, (int64_t)L * mat, st);      // (L, k, n_f)
  std::vector<double> v2pT_h, p2vT_h;
  for (int l = 0; l < L; ++l) {
    auto a = ctranspose(pl.val2pw + l * mat, n_f, k);  // (k, n_f)
    auto b = ctranspose(pl.pw2val + l * mat, k, n_f);  // (n_f, k)
    v2pT_h.insert(v2pT_h.end(), a.begin(), a.end());
    p2vT_h.insert(p2vT_h.end(), b.begin(), b.end());
  }
  DBuf<double> v2pT = upload(v2pT_h.data(), (int64_t)v2pT_h.size(), st);
  DBuf<double> p2vT = upload(p2vT_h.data(), (int64_t)p2vT_h.size(), st);
  DBuf<double> rows = upload(pl.rows, 2 * pl.n_rows * n_f, st);
  std::vector<double> dT_h((size_t)pl.n_tables * k * k);
  for (int64_t t = 0; t < pl.n_tables; ++t)
    for (int i = 0; i < k; ++i)
      for (int j = 0; j < k; ++j) dT_h[(t * k + j) * k + i] = pl.dtab[(t * k + i) * k + j];
  DBuf<double> dtab = upload(pl.dtab, pl.n_tables * k * k, st);
  DBuf<double> dtabT = upload(dT_h.data(), (int64_t)dT_h.size(), st);
  DBuf<double> phi(resume ? 0 : 2 * pl.n_pw * NF, st), psi(2 * pl.n_pw * NF, st);
  if (resume) {
    FGT_REQUIRE(resume->dim == D && resume->k == k && resume->n_f == n_f && resume->NF == NF,
                FGT_EINVAL, "refinement plan does not match the retained transform");
    FGT_REQUIRE(pl.n_pw >= resume->n_pw && pl.n_form == 0, FGT_EINVAL,
                "refinement plan must keep the retained plane-wave slots and form nothing");
    for (int64_t s = 0; s < pl.n_stages; ++s)
      FGT_REQUIRE(pl.stage_kind[s] == 2, FGT_EINVAL, "refinement stages must be pushes (psi -> psi)");
    if (resume->n_pw)
      FGT_CUDA(cudaMemcpyAsync(psi.get(), resume->psi.get(), sizeof(double) * 2 * resume->n_pw * NF,
                               cudaMemcpyDeviceToDevice, st));
    if (pl.n_pw > resume->n_pw)
      FGT_CUDA(cudaMemsetAsync(psi.get() + 2 * resume->n_pw * NF, 0,
                               sizeof(double) * 2 * (pl.n_pw - resume->n_pw) * NF, st));
  }

  // ---- leaf -> plane waves, level by level
  c_form.begin(st);
  auto forms = group_by_level(pl.n_form, pl.form_leaf, pl.form_pw, pl.form_level);
  for (auto& kv : forms) {
    const int l = kv.first;
    const int64_t nb = (int64_t)kv.second.leaf.size();
    DBuf<int64_t> lf = upload(kv.second.leaf.data(), nb, st), pw = upload(kv.second.pw.data(), nb, st);
    const double* A = v2p.get() + l * mat;
    const double* AT = v2pT.get() + l * mat;
    if (D == 1) {
      bgemm<true, false, false>(gemm(A, k, 0, values, 1, KD, phi.get(), 1, NF, n_f, 1, k, nb, pw.get(), lf.get()), st);
    } else if (D == 2) {
      DBuf<double> t1(2 * nb * k * n_f, st);
      bgemm<false, true, false>(gemm(values, k, KD, AT, n_f, 0, t1.get(), n_f, (int64_t)k * n_f, k, n_f, k, nb, nullptr, nullptr, lf.get()), st);
      bgemm<true, true, false>(gemm(A, k, 0, t1.get(), n_f, (int64_t)k * n_f, phi.get(), n_f, NF, n_f, n_f, k, nb, pw.get()), st);
    } else {
      DBuf<double> t1(2 * nb * k * k * n_f, st), t2(2 * nb * k * n_f * n_f, st);
      bgemm<false, true, false>(gemm(values, k, KD, AT, n_f, 0, t1.get(), n_f, (int64_t)k * k * n_f, k * k, n_f, k, nb, nullptr, nullptr, lf.get()), st);
      bgemm<true, true, false>(gemm(A, k, 0, t1.get(), n_f, (int64_t)k * n_f, t2.get(), n_f, (int64_t)n_f * n_f, n_f, n_f, k, nb * k), st);
      bgemm<true, true, false>(gemm(A, k, 0, t2.get(), (int64_t)n_f * n_f, (int64_t)k * n_f * n_f, phi.get(), (int64_t)n_f * n_f, NF, n_f, n_f * n_f, k, nb, pw.get()), st);
    }
  }
  c_form.end(st);

  // ---- merge / gather / push: diagonal shift stages in order
  c_shift.begin(st);
  {
    DBuf<int64_t> dst = upload(pl.dst, pl.n_dst, st), dacc = upload(pl.dst_acc, pl.n_dst, st);
    DBuf<int64_t> doff = upload(pl.dst_off, pl.n_dst + 1, st);
    DBuf<int64_t> esrc = upload(pl.ent_src, pl.n_entries, st), erow = upload(pl.ent_rows, pl.n_entries * D, st);
    for (int64_t s = 0; s < pl.n_stages; ++s) {
      const int64_t a0 = pl.stage_off[s], a1 = pl.stage_off[s + 1];
      if (a1 == a0) continue;
      const int64_t kind = pl.stage_kind[s];  // 0 merge, 1 gather, 2 push
      ShiftArgs sa;
      sa.dst = dst.get();
      sa.dst_acc = dacc.get();
      sa.dst_off = doff.get();
      sa.ent_src = esrc.get();
      sa.ent_rows = erow.get();
      sa.rows = reinterpret_cast<const double2*>(rows.get());
      sa.src = reinterpret_cast<const double2*>(kind == 2 ? psi.get() : phi.get());
      sa.out = reinterpret_cast<double2*>(kind == 0 ? phi.get() : psi.get());
      sa.NF = NF;
      sa.d0 = a0;
      sa.n_f = n_f;
      sa.D = D;
      FGT_REQUIRE(a1 - a0 <= 65535, FGT_ERANGE, "too many shift destinations in one stage");
      dim3 grid(grid_for(NF, 256, 64), (unsigned)(a1 - a0));
      shift_kernel<D><<<grid, 256, 0, st>>>(sa);
      FGT_LAUNCHED();
    }
  }
  c_shift.end(st);

  // ---- plane waves -> leaf grids (overwrites u of every evaluated leaf)
  FGT_CUDA(cudaMemsetAsync(u, 0, sizeof(double) * pl.n_leaves * KD, st));
  c_eval.begin(st);
  auto evals = group_by_level(pl.n_eval, pl.eval_leaf, pl.eval_pw, pl.eval_level);
  for (auto& kv : evals) {
    const int l = kv.first;
    const int64_t nb = (int64_t)kv.second.leaf.size();
    DBuf<int64_t> lf = upload(kv.second.leaf.data(), nb, st), pw = upload(kv.second.pw.data(), nb, st);
    const double* E = p2v.get() + l * mat;    // (k, n_f)
    const double* ET = p2vT.get() + l * mat;  // (n_f, k)
    if (D == 1) {
      bgemm<true, true, true>(gemm(E, n_f, 0, psi.get(), 1, NF, u, 1, KD, k, 1, n_f, nb, lf.get(), pw.get()), st);
    } else if (D == 2) {
      DBuf<double> v1(2 * nb * k * n_f, st);
      bgemm<true, true, false>(gemm(E, n_f, 0, psi.get(), n_f, NF, v1.get(), n_f, (int64_t)k * n_f, k, n_f, n_f, nb, nullptr, pw.get()), st);
      bgemm<true, true, true>(gemm(v1.get(), n_f, (int64_t)k * n_f, ET, k, 0, u, k, KD, k, k, n_f, nb, lf.get()), st);
    } else {
      DBuf<double> v1(2 * nb * k * n_f * n_f, st), v2(2 * nb * k * k * n_f, st);
      bgemm<true, true, false>(gemm(E, n_f, 0, psi.get(), (int64_t)n_f * n_f, NF, v1.get(), (int64_t)n_f * n_f, (int64_t)k * n_f * n_f, k, n_f * n_f, n_f, nb, nullptr, pw.get()), st);
      bgemm<true, true, false>(gemm(E, n_f, 0, v1.get(), n_f, (int64_t)n_f * n_f, v2.get(), n_f, (int64_t)k * n_f, k, n_f, n_f, nb * k), st);
      bgemm<true, true, true>(gemm(v2.get(), n_f, (int64_t)k * k * n_f, ET, k, 0, u, k, KD, k * k, k, n_f, nb, lf.get()), st);
    }
  }
  c_eval.end(st);
  phi.release();
  if (BoxState* keep = retain ? retain : resume) {
    keep->psi = std::move(psi);
    keep->n_pw = pl.n_pw;
    keep->NF = NF;
    keep->KD = KD;
    keep->dim = D;
    keep->k = k;
    keep->n_f = n_f;
  } else {
    psi.release();
  }

  // ---- direct near field: per pair separable contractions into Y, then a fixed-order
  // per-target sum (pairs arrive sorted by target)
  c_direct.begin(st);
  const int64_t np = pl.n_dpairs;
  if (np > 0) {
    std::vector<int64_t> toff(1, 0), tleaf;
    for (int64_t p = 0; p < np; ++p) {
      if (p == 0 || pl.d_tgt[p] != pl.d_tgt[p - 1]) {
        if (p) toff.push_back(p);
        tleaf.push_back(pl.d_tgt[p]);
      }
      FGT_REQUIRE(p == 0 || pl.d_tgt[p] >= pl.d_tgt[p - 1], FGT_EINVAL, "direct pairs not sorted by target");
    }
    toff.push_back(np);
    DBuf<int64_t> src = upload(pl.d_src, np, st), tab = upload(pl.d_tab, np * D, st);
    DBuf<int64_t> toff_d = upload(toff.data(), (int64_t)toff.size(), st), tleaf_d = upload(tleaf.data(), (int64_t)tleaf.size(), st);
    if (D == 3 && k <= 16) {
      // fused: tables and intermediates in shared memory, accumulation in registers
      const int KP = k <= 8 ? 8 : 16;
      const size_t smem = (size_t)(2 * KP * KP * (KP + 4) + 3 * KP * (KP + 4)) * sizeof(double);
      const unsigned nt = (unsigned)tleaf.size();
      if (KP == 8) {
        FGT_CUDA(cudaFuncSetAttribute(direct3_kernel<8, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        direct3_kernel<8, 4><<<nt, 128, smem, st>>>(values, dtab.get(), toff_d.get(), tleaf_d.get(), src.get(), tab.get(), k, u);
      } else {
        FGT_CUDA(cudaFuncSetAttribute(direct3_kernel<16, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        direct3_kernel<16, 8><<<nt, 256, smem, st>>>(values, dtab.get(), toff_d.get(), tleaf_d.get(), src.get(), tab.get(), k, u);
      }
      FGT_LAUNCHED();
    } else {
    const int64_t chunk = std::max<int64_t>(1, (int64_t)(512ll << 20) / (KD * 8 * 2));
    DBuf<double> Y(np * KD, st);
    for (int64_t p0 = 0; p0 < np; p0 += chunk) {
      const int64_t nb = std::min(chunk, np - p0);
      DBuf<int64_t> ta(nb * k, st), tb(nb, st), tc(nb, st);
      const int64_t* srcp = src.get() + p0;
      // table ids per axis: axis 0 -> tc (last stage), axis D-1 -> first stage
      repeat_kernel<<<grid_for(nb, 256), 256, 0, st>>>(tab.get() + p0 * D, nb, 1, D, D - 1, tb.get());
      FGT_LAUNCHED();
      repeat_kernel<<<grid_for(nb, 256), 256, 0, st>>>(tab.get() + p0 * D, nb, 1, D, 0, tc.get());
      FGT_LAUNCHED();
      double* Yp = Y.get() + p0 * KD;
      if (D == 1) {
        bgemm<false, false, true>(gemm(dtab.get(), k, k * k, values, 1, KD, Yp, 1, KD, k, 1, k, nb, nullptr, srcp, tc.get()), st);
      } else if (D == 2) {
        DBuf<double> x1(nb * KD, st);
        // X1[a][n2] = sum_b vals[a][b] D_axis1^T[b][n2]
        bgemm<false, false, true>(gemm(values, k, KD, dtabT.get(), k, k * k, x1.get(), k, KD, k, k, k, nb, nullptr, tb.get(), srcp), st);
        // Y[n1][n2] = sum_a D_axis0[n1][a] X1[a][n2]
        bgemm<false, false, true>(gemm(dtab.get(), k, k * k, x1.get(), k, KD, Yp, k, KD, k, k, k, nb, nullptr, nullptr, tc.get()), st);
      } else {
        DBuf<double> x1(nb * KD, st), x2(nb * KD, st);
        repeat_kernel<<<grid_for(nb * k, 256), 256, 0, st>>>(tab.get() + p0 * D, nb, k, D, 1, ta.get());
        FGT_LAUNCHED();
        // X1[(a b)][n3] = sum_c vals[(a b)][c] D_axis2^T[c][n3]
        bgemm<false, false, true>(gemm(values, k, KD, dtabT.get(), k, k * k, x1.get(), k, KD, k * k, k, k, nb, nullptr, tb.get(), srcp), st);
        // X2[a][n2][n3] = sum_b D_axis1[n2][b] X1[a][b][n3]      (batch = pair x a)
        bgemm<false, false, true>(gemm(dtab.get(), k, k * k, x1.get(), k, (int64_t)k * k, x2.get(), k, (int64_t)k * k, k, k, k, nb * k, nullptr, nullptr, ta.get()), st);
        // Y[n1][(n2 n3)] = sum_a D_axis0[n1][a] X2[a][(n2 n3)]
        bgemm<false, false, true>(gemm(dtab.get(), k, k * k, x2.get(), (int64_t)k * k, KD, Yp, (int64_t)k * k, KD, k, k * k, k, nb, nullptr, nullptr, tc.get()), st);
      }
    }
    const int64_t nt = (int64_t)tleaf.size();
    FGT_REQUIRE(nt <= 65535 * 64, FGT_ERANGE, "too many direct targets");
    for (int64_t t0 = 0; t0 < nt; t0 += 65535) {
      const int64_t n = std::min<int64_t>(65535, nt - t0);
      pair_reduce_kernel<<<dim3(grid_for(KD, 256, 16), (unsigned)n), 256, 0, st>>>(
          Y.get(), toff_d.get() + t0, tleaf_d.get() + t0, KD, u);
      FGT_LAUNCHED();
    }
    }
  }
  c_direct.end(st);
  if (times) {
    times->form_ms = times->k_form_ms = c_form.ms();
    times->gather_ms = times->k_gather_ms = c_shift.ms();
    times->eval_ms = times->k_eval_ms = c_eval.ms();
    times->direct_ms = times->k_direct_ms = c_direct.ms();
    times->total_ms = times->form_ms + times->gather_ms + times->eval_ms + times->direct_ms;
    times->n_modes = NF;
    times->n_boxes = pl.n_pw;
    times->n_src_dense = pl.n_form;
    times->n_tgt_psi = pl.n_eval;
    times->n_p_entries = pl.n_entries;
    times->n_direct_pairs = np;
  }
}

}  // namespace

void box_fgt(const fgt_box_plan& pl, const double* values, double* u, cudaStream_t st,
             fgt_phase_times* times, BoxState* retain, BoxState* resume) {
  FGT_REQUIRE(!(retain && resume), FGT_EINVAL, "retain and resume are exclusive");
  if (pl.dim == 1) box_impl<1>(pl, values, u, st, times, retain, resume);
  else if (pl.dim == 2) box_impl<2>(pl, values, u, st, times, retain, resume);
  else if (pl.dim == 3) box_impl<3>(pl, values, u, st, times, retain, resume);
  else throw Error(FGT_EINVAL, "dim must be 1, 2, or 3");
}


// ---------------------------------------------------------------- interp_at
namespace {
constexpr int IMAXK = 24;

struct InterpTreeDev {
  const uint64_t* keys;   // sorted leaf keys
  const int64_t* slots;   // coefficient row of each sorted key
  const double* coeffs;
  int64_t n_leaves;
  int dim, k, periodic, max_level;
  double low[3], side;
};

// deepest leaf containing x; its centre and half side
template <int D>
__device__ int64_t locate_leaf(const InterpTreeDev& t, double* x, double* ctr, double* half) {
  if (t.periodic)
#pragma unroll
    for (int c = 0; c < D; ++c) x[c] -= floor((x[c] - t.low[c]) / t.side) * t.side;
  for (int l = t.max_level; l >= 0; --l) {
    const int64_t n = (int64_t)1 << l;
    const double sl = t.side / (double)n;
    int64_t g[D];
#pragma unroll
    for (int c = 0; c < D; ++c) {
      int64_t v = (int64_t)floor((x[c] - t.low[c]) / sl);
      g[c] = v < 0 ? 0 : (v >= n ? n - 1 : v);
    }
    const uint64_t key = box_key(l, morton_encode(g, D, l));
    const int64_t i = find_dev(t.keys, t.n_leaves, key);
    if (i >= 0) {
#pragma unroll
      for (int c = 0; c < D; ++c) ctr[c] = t.low[c] + ((double)g[c] + 0.5) * sl;
      *half = 0.5 * sl;
      return t.slots[i];
    }
  }
  return -1;
}

__device__ __forceinline__ void legendre_row(double t, int k, double* P) {
  P[0] = 1.0;
  if (k > 1) P[1] = t;
  for (int n = 1; n + 1 < k; ++n) P[n + 1] = ((2 * n + 1) * t * P[n] - n * P[n - 1]) / (n + 1);
}

// d = 1, 2: one thread per point
template <int D>
__global__ void interp_at_kernel(InterpTreeDev t, const double* __restrict__ xs, int64_t n,
                                 double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double x[D], ctr[D], half;
#pragma unroll
    for (int c = 0; c < D; ++c) x[c] = xs[i * D + c];
    const int64_t s = locate_leaf<D>(t, x, ctr, &half);
    if (s < 0) {
      out[i] = NAN;
      continue;
    }
    const int k = t.k;
    double P0[IMAXK], P1[IMAXK];
    legendre_row((x[0] - ctr[0]) / half, k, P0);
    const double* C = t.coeffs + s * (D == 2 ? k * k : k);
    double acc = 0.0;
    if (D == 1) {
      for (int a = 0; a < k; ++a) acc += C[a] * P0[a];
    } else {
      legendre_row((x[1] - ctr[1]) / half, k, P1);
      for (int a = 0; a < k; ++a) {
        double r = 0.0;
        for (int b = 0; b < k; ++b) r += C[a * k + b] * P1[b];
        acc += P0[a] * r;
      }
    }
    out[i] = acc;
  }
}

// d = 3: one warp per point, lanes over the (b, c) pairs of each a-slice
__global__ void __launch_bounds__(256) interp_at3_kernel(InterpTreeDev t, const double* __restrict__ xs,
                                                         int64_t n, double* __restrict__ out) {
  __shared__ double s_P[8][3][IMAXK];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t i = (int64_t)blockIdx.x * 8 + warp; i < n; i += (int64_t)gridDim.x * 8) {
    double x[3], ctr[3], half;
#pragma unroll
    for (int c = 0; c < 3; ++c) x[c] = xs[i * 3 + c];
    const int64_t s = locate_leaf<3>(t, x, ctr, &half);
    const int k = t.k;
    if (s >= 0 && lane < 3) legendre_row((x[lane] - ctr[lane]) / half, k, s_P[warp][lane]);
    __syncwarp();
    double acc = 0.0;
    if (s >= 0) {
      const double* C = t.coeffs + s * (int64_t)k * k * k;
      for (int a = 0; a < k; ++a) {
        double r = 0.0;
        for (int bc = lane; bc < k * k; bc += 32) {
          const int b = bc / k, c = bc - b * k;
          r += C[(a * k + b) * k + c] * s_P[warp][1][b] * s_P[warp][2][c];
        }
        acc += s_P[warp][0][a] * r;
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == 0) out[i] = s >= 0 ? acc : NAN;
    __syncwarp();
  }
}
}  // namespace

void box_interp(const fgt_interp_tree& tr, const double* x, int64_t n, double* out, cudaStream_t st) {
  const int d = tr.dim, k = tr.k;
  FGT_REQUIRE(d >= 1 && d <= 3, FGT_EINVAL, "dim must be 1, 2, or 3");
  FGT_REQUIRE(k >= 2 && k <= IMAXK, FGT_ERANGE, "polynomial order outside [2, 24]");
  FGT_REQUIRE(tr.n_leaves >= 1 && tr.level && tr.coords && tr.coeffs, FGT_EINVAL, "empty tree");
  int64_t kd = 1;
  for (int c = 0; c < d; ++c) kd *= k;
  // leaf keys (level, Morton code) sorted on the host; coefficients stay in leaf order
  std::vector<std::pair<uint64_t, int64_t>> kv(tr.n_leaves);
  int max_level = 0;
  for (int64_t i = 0; i < tr.n_leaves; ++i) {
    const int l = tr.level[i];
    FGT_REQUIRE(l >= 0 && d * l <= 57, FGT_ERANGE, "leaf level out of range");
    max_level = std::max(max_level, l);
    kv[i] = {box_key(l, morton_encode(tr.coords + i * d, d, l)), i};
  }
  std::sort(kv.begin(), kv.end());
  std::vector<uint64_t> hk(tr.n_leaves);
  std::vector<int64_t> hs(tr.n_leaves);
  for (int64_t i = 0; i < tr.n_leaves; ++i) {
    hk[i] = kv[i].first;
    hs[i] = kv[i].second;
  }
  DBuf<uint64_t> keys(tr.n_leaves, st);
  DBuf<int64_t> slots(tr.n_leaves, st);
  DBuf<double> coeffs(tr.n_leaves * kd, st);
  keys.from_host(hk.data(), hk.size());
  slots.from_host(hs.data(), hs.size());
  coeffs.from_host(tr.coeffs, tr.n_leaves * kd);
  InterpTreeDev t;
  t.keys = keys.get();
  t.slots = slots.get();
  t.coeffs = coeffs.get();
  t.n_leaves = tr.n_leaves;
  t.dim = d;
  t.k = k;
  t.periodic = tr.periodic;
  t.max_level = max_level;
  for (int c = 0; c < 3; ++c) t.low[c] = tr.root_low[c];
  t.side = tr.root_side;
  if (n == 0) return;
  if (d == 1) interp_at_kernel<1><<<grid_for(n, 256), 256, 0, st>>>(t, x, n, out);
  else if (d == 2) interp_at_kernel<2><<<grid_for(n, 256), 256, 0, st>>>(t, x, n, out);
  else interp_at3_kernel<<<grid_for(n, 8, 148 * 64), 256, 0, st>>>(t, x, n, out);
  FGT_LAUNCHED();
  FGT_CUDA(cudaStreamSynchronize(st));  // host-side tables go out of scope
}
// ---------------------------------------------------------------- Alg 3 / 5 / 6 on the device
// tail test (Eq. funerr; reference poly1d.py:100-126), grid nodes of a set of boxes
// (tree.py:384-391) and the level-restriction sweep (tree.py:195-220) as kernels, so the
// density tree and the output tree are decided where the grids live.
namespace {
constexpr int TMAXK = 24;

// One CTA per leaf grid: values -> Legendre coefficients axis by axis in shared memory
// (the reference's _apply_per_axis, poly1d.py:76-81), then the RMS of the coefficients with
// |alpha|_2 >= k (d = 1: the last two) and the quadrature-weighted sum of squares.  Sums run
// in a fixed order (per-thread strided partials, then a shared-memory tree).
template <int D>
__global__ void __launch_bounds__(256) tail_kernel(const double* __restrict__ values, int k,
                                                   const double* __restrict__ v2p,
                                                   const double* __restrict__ wts,
                                                   double* __restrict__ tail, double* __restrict__ wsq) {
  extern __shared__ double sm[];
  int kd = 1;
  for (int c = 0; c < D; ++c) kd *= k;
  double* a = sm;            // kd
  double* b = sm + kd;       // kd
  double* M = b + kd;        // k * k
  double* w = M + k * k;     // k
  __shared__ double red[2][256];
  const double* v = values + (int64_t)blockIdx.x * kd;
  for (int i = threadIdx.x; i < kd; i += blockDim.x) a[i] = v[i];
  for (int i = threadIdx.x; i < k * k; i += blockDim.x) M[i] = v2p[i];
  for (int i = threadIdx.x; i < k; i += blockDim.x) w[i] = wts[i];
  __syncthreads();
  // weighted square sum of the values
  double s2 = 0.0;
  for (int i = threadIdx.x; i < kd; i += blockDim.x) {
    double ww = 1.0;
    int rem = i;
    for (int c = 0; c < D; ++c) {
      ww *= w[rem % k];
      rem /= k;
    }
    s2 += ww * a[i] * a[i];
  }
  // contract one axis per pass: out[.., n, ..] = sum_j M[n][j] in[.., j, ..]
  double* in = a;
  double* out = b;
  int stride = kd / k;  // axis 0 first (C order: axis 0 has the largest stride)
  for (int ax = 0; ax < D; ++ax) {
    for (int i = threadIdx.x; i < kd; i += blockDim.x) {
      const int n = (i / stride) % k;
      const int base = i - n * stride;
      double acc = 0.0;
      for (int j = 0; j < k; ++j) acc += M[n * k + j] * in[base + j * stride];
      out[i] = acc;
    }
    __syncthreads();
    double* t = in;
    in = out;
    out = t;
    stride /= k;
  }
  double ts = 0.0;
  int cnt = 0;
  for (int i = threadIdx.x; i < kd; i += blockDim.x) {
    int rem = i, r2 = 0;
    bool last2 = false;
    for (int c = 0; c < D; ++c) {
      const int q = rem % k;
      rem /= k;
      r2 += q * q;
      if (D == 1) last2 = q >= k - 2;
    }
    if (D == 1 ? last2 : r2 >= k * k) {
      ts += in[i] * in[i];
      ++cnt;
    }
  }
  red[0][threadIdx.x] = ts;
  red[1][threadIdx.x] = s2;
  __shared__ int cred[256];
  cred[threadIdx.x] = cnt;
  __syncthreads();
  for (int off = 128; off > 0; off >>= 1) {
    if ((int)threadIdx.x < off) {
      red[0][threadIdx.x] += red[0][threadIdx.x + off];
      red[1][threadIdx.x] += red[1][threadIdx.x + off];
      cred[threadIdx.x] += cred[threadIdx.x + off];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    tail[blockIdx.x] = cred[0] ? sqrt(red[0][0] / (double)cred[0]) : 0.0;
    if (wsq) wsq[blockIdx.x] = red[1][0];
  }
}

// pts[b][i_0..i_{d-1}][c] = centre_c + (0.5 side) node_{i_c}, every operation rounded as the
// host expression (rc - rs/2) + (g + 0.5) s, then + (0.5 s) node (no fused multiply-adds).
template <int D>
__global__ void nodes_kernel(const int32_t* __restrict__ level, const int64_t* __restrict__ coords,
                             int64_t n, int k, const double* __restrict__ nodes, double3 low,
                             double side, double* __restrict__ pts) {
  int64_t kd = 1;
  for (int c = 0; c < D; ++c) kd *= k;
  const double lowv[3] = {low.x, low.y, low.z};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n * kd;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t bx = i / kd;
    int64_t rem = i - bx * kd;
    const double s = side / (double)((int64_t)1 << level[bx]);
    const double hs = __dmul_rn(0.5, s);
    int idx[D];
#pragma unroll
    for (int c = D - 1; c >= 0; --c) {
      idx[c] = (int)(rem % k);
      rem /= k;
    }
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const double ctr = __dadd_rn(lowv[c], __dmul_rn((double)coords[bx * D + c] + 0.5, s));
      pts[i * D + c] = __dadd_rn(ctr, __dmul_rn(hs, nodes[idx[c]]));
    }
  }
}

// One thread per (box, neighbour offset): a leaf at level l >= 2 flags every leaf that
// covers one of its 3^d - 1 neighbour cells from two or more levels above (the condition the
// reference's LIFO sweep splits on, tree.py:205-214).  Rounds of flag + split reach the same
// least fixpoint as the sequential sweep.
template <int D>
__global__ void balance_flags_kernel(const uint64_t* __restrict__ keys, const uint8_t* __restrict__ leaf,
                                     int64_t n, int periodic, uint8_t* __restrict__ flags) {
  int n_off = 1;
  for (int c = 0; c < D; ++c) n_off *= 3;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n * n_off;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / n_off;
    int o = (int)(t - i * n_off);
    if (!leaf[i]) continue;
    const int l = key_level(keys[i]);
    if (l < 2) continue;
    int64_t g[D], nb[D];
    morton_decode(key_code(keys[i]), D, l, g);
    const int64_t side = (int64_t)1 << l;
    bool inside = true, self = true;
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const int oc = o % 3 - 1;
      o /= 3;
      self = self && oc == 0;
      int64_t v = g[c] + oc;
      if (periodic) v = (v % side + side) % side;
      else inside = inside && v >= 0 && v < side;
      nb[c] = v;
    }
    if (self || !inside) continue;
    for (int lv = l; lv >= 0; --lv) {
      const int64_t j = find_dev(keys, n, box_key(lv, morton_encode(nb, D, lv)));
      if (j >= 0) {
        if (leaf[j] && l - lv >= 2) flags[j] = 1;
        break;
      }
#pragma unroll
      for (int c = 0; c < D; ++c) nb[c] >>= 1;
    }
  }
}
}  // namespace

void box_tail(const double* values, int64_t n, int dim, int k, const double* val_to_pol,
              const double* weights, double* tail, double* wsq, cudaStream_t st) {
  FGT_REQUIRE(dim >= 1 && dim <= 3, FGT_EINVAL, "dim must be 1, 2, or 3");
  FGT_REQUIRE(k >= 2 && k <= TMAXK, FGT_ERANGE, "polynomial order outside [2, 24]");
  if (n == 0) return;
  const int64_t kd = ipw(k, dim);
  const size_t smem = sizeof(double) * (size_t)(2 * kd + k * k + k);
  FGT_REQUIRE(n <= 0x7fffffff, FGT_ERANGE, "too many leaf grids");
  auto launch = [&](auto kern) {
    FGT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<(unsigned)n, 256, smem, st>>>(values, k, val_to_pol, weights, tail, wsq);
    FGT_LAUNCHED();
  };
  if (dim == 1) launch(tail_kernel<1>);
  else if (dim == 2) launch(tail_kernel<2>);
  else launch(tail_kernel<3>);
}

void box_nodes(const int32_t* level, const int64_t* coords, int64_t n, int dim, int k,
               const double* nodes, const double* root_low, double root_side, double* pts,
               cudaStream_t st) {
  FGT_REQUIRE(dim >= 1 && dim <= 3, FGT_EINVAL, "dim must be 1, 2, or 3");
  if (n == 0) return;
  const double3 low = make_double3(root_low[0], dim > 1 ? root_low[1] : 0.0, dim > 2 ? root_low[2] : 0.0);
  const int64_t total = n * ipw(k, dim);
  const unsigned grid = grid_for(total, 256, 148 * 16);
  if (dim == 1) nodes_kernel<1><<<grid, 256, 0, st>>>(level, coords, n, k, nodes, low, root_side, pts);
  else if (dim == 2) nodes_kernel<2><<<grid, 256, 0, st>>>(level, coords, n, k, nodes, low, root_side, pts);
  else nodes_kernel<3><<<grid, 256, 0, st>>>(level, coords, n, k, nodes, low, root_side, pts);
  FGT_LAUNCHED();
}

void box_balance_flags(const uint64_t* keys, const uint8_t* leaf, int64_t n, int dim, int periodic,
                       uint8_t* flags, cudaStream_t st) {
  FGT_REQUIRE(dim >= 1 && dim <= 3, FGT_EINVAL, "dim must be 1, 2, or 3");
  if (n == 0) return;
  FGT_CUDA(cudaMemsetAsync(flags, 0, (size_t)n, st));
  const unsigned grid = grid_for(n * 27, 256, 148 * 16);
  if (dim == 1) balance_flags_kernel<1><<<grid, 256, 0, st>>>(keys, leaf, n, periodic, flags);
  else if (dim == 2) balance_flags_kernel<2><<<grid, 256, 0, st>>>(keys, leaf, n, periodic, flags);
  else balance_flags_kernel<3><<<grid, 256, 0, st>>>(keys, leaf, n, periodic, flags);
  FGT_LAUNCHED();
}
}  // namespace fgt
