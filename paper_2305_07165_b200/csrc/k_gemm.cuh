// Batched small GEMMs on the FP64 tensor cores (mma.sync m8n8k4 .f64 -> SASS DMMA).
// Shared by the NUFFT grid<->mode transforms and the volume FGT per-axis contractions
// (the separable `_apply_per_axis` pattern of poly1d.py:76-81).
#pragma once
#include "fgt_common.cuh"

namespace fgt {

__device__ __forceinline__ void dmma2(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

// C[b] = A[b] (M x K) * B[b] (K x N), row-major with leading dims, batch strides in
// elements; complex operands are interleaved (re, im).  CRE: store Re(C) only.
struct GemmArgs {
  const double* A;
  const double* B;
  double* C;
  int M, N, K;
  int64_t batch;
  int64_t lda, ldb, ldc, sA, sB, sC;
  const int64_t* cidx;  // optional C batch index
  const int64_t* bidx;  // optional B batch index
  const int64_t* aidx;  // optional A batch index
  int64_t boff;         // batch offset of this launch (grid.z limit)
  // optional epilogue rephasing of a d = 3 expansion stage (complex C, rows r = s n_f + m1
  // over the stored half-spectrum planes s, columns m2): C[r][c] *= bp[k][0][hmi(s)]
  // bp[k][1][m1] bp[k][2][c] with k = cidx[b] (box phases, (slot, 3, n_f) complex)
  const double2* bp;
  int bp_nf, bp_half;
};

// CTA tile 32 x 48 (2 x 2 warps of 16 x 24); FLAT: 16 x 96 (1 x 4 warps) for M <= 16, so
// a 16-row problem (e.g. the nh = 16 stored planes of config 5) wastes no DMMA rows
template <bool AC, bool BC, bool CRE, bool ACC, bool FLAT = false, bool TALL = false, int MID = 0>
__global__ void __launch_bounds__(128) bgemm_kernel(GemmArgs g) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // TALL (N <= 32): 64 x 32 (4 x 1 warps of 16 x 32, four 8-column tiles per warp)
  // MID = 4 / 5 (M <= 32, N <= 32 / 40, e.g. the n_f x G axis-1 stage per plane): 32 x 8 MID
  // (2 x 1 warps of 16 x 8 MID, MID 8-column tiles per warp; 64 threads)
  constexpr int NT = MID ? MID : (TALL ? 4 : 3);
  const int wm = FLAT ? 0 : ((TALL || MID) ? warp : warp >> 1), wn = FLAT ? warp : ((TALL || MID) ? 0 : warp & 1);
  const int64_t b = blockIdx.z + g.boff;
  const int m0 = blockIdx.y * (FLAT ? 16 : (TALL ? 64 : 32)) + wm * 16;
  const int n0 = blockIdx.x * (FLAT ? 96 : (TALL ? 32 : (MID ? 8 * MID : 48))) + wn * 24;
  const double* A = g.A + (g.aidx ? g.aidx[b] : b) * g.sA * (AC ? 2 : 1);
  const double* B = g.B + (g.bidx ? g.bidx[b] : b) * g.sB * (BC ? 2 : 1);
  const int64_t cb = g.cidx ? g.cidx[b] : b;
  double* C = g.C + cb * g.sC * (CRE ? 1 : 2);
  double acc[2][NT][4];
  double gauss[2][NT][2];  // k3 of the 3-product complex MAC (AC && BC && !CRE; not TALL: registers)
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) {
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[i][j][e] = 0.0;
      gauss[i][j][0] = gauss[i][j][1] = 0.0;
    }
  for (int k0 = 0; k0 < g.K; k0 += 4) {
    const int k = k0 + (lane & 3);
    double ar[2], ai[2], br[NT], bi[NT];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const int r = m0 + mt * 8 + (lane >> 2);
      ar[mt] = ai[mt] = 0.0;
      if (r < g.M && k < g.K) {
        if (AC) {
          double2 v = *reinterpret_cast<const double2*>(A + 2 * (r * g.lda + k));
          ar[mt] = v.x;
          ai[mt] = v.y;
        } else {
          ar[mt] = A[r * g.lda + k];
        }
      }
    }
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int c = n0 + nt * 8 + (lane >> 2);
      br[nt] = bi[nt] = 0.0;
      if (c < g.N && k < g.K) {
        if (BC) {
          double2 v = *reinterpret_cast<const double2*>(B + 2 * (k * g.ldb + c));
          br[nt] = v.x;
          bi[nt] = v.y;
        } else {
          br[nt] = B[k * g.ldb + c];
        }
      }
    }
    if constexpr (AC && BC && !CRE && !TALL) {
      // complex x complex in three real products (Gauss): k1 = (ar + ai) br,
      // k2 = ar (bi - br), k3 = ai (br + bi); re = k1 - k3, im = k1 + k2, accumulated as
      // acc[0..1] = k1, acc[2..3] = k2, gauss[..] = k3 and combined in the epilogue
      double bd[NT], bs[NT];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        bd[nt] = bi[nt] - br[nt];
        bs[nt] = br[nt] + bi[nt];
      }
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        const double as = ar[mt] + ai[mt];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          dmma2(acc[mt][nt][0], acc[mt][nt][1], as, br[nt]);
          dmma2(acc[mt][nt][2], acc[mt][nt][3], ar[mt], bd[nt]);
          dmma2(gauss[mt][nt][0], gauss[mt][nt][1], ai[mt], bs[nt]);
        }
      }
    } else {
      // re += ar br - ai bi ; im += ar bi + ai br   (terms with a real operand vanish)
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) dmma2(acc[mt][nt][0], acc[mt][nt][1], ar[mt], br[nt]);
      if (AC && BC) {
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) dmma2(acc[mt][nt][0], acc[mt][nt][1], -ai[mt], bi[nt]);
      }
      if (!CRE) {
        if (BC) {
#pragma unroll
          for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) dmma2(acc[mt][nt][2], acc[mt][nt][3], ar[mt], bi[nt]);
        }
        if (AC) {
#pragma unroll
          for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) dmma2(acc[mt][nt][2], acc[mt][nt][3], ai[mt], br[nt]);
        }
      }
    }
  }
  if (AC && BC && !CRE && !TALL) {
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const double k1 = acc[mt][nt][i], k2 = acc[mt][nt][2 + i], k3 = gauss[mt][nt][i];
          acc[mt][nt][i] = k1 - k3;
          acc[mt][nt][2 + i] = k1 + k2;
        }
  }
#pragma unroll
  for (int mt = 0; mt < 2; ++mt) {
    const int r = m0 + mt * 8 + (lane >> 2);
    if (r >= g.M) continue;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int c = n0 + nt * 8 + 2 * (lane & 3) + i;
        if (c >= g.N) continue;
        if (CRE) {
          double* cp = C + r * g.ldc + c;
          *cp = ACC ? *cp + acc[mt][nt][i] : acc[mt][nt][i];
        } else {
          double2* cp = reinterpret_cast<double2*>(C + 2 * (r * g.ldc + c));
          double2 v = make_double2(acc[mt][nt][i], acc[mt][nt][2 + i]);
          if (g.bp) {
            const int nf = g.bp_nf, s = r / nf, m1 = r - s * nf;
            const int i0 = g.bp_half ? (s + nf / 2) % nf : s;
            const double2* q = g.bp + cb * 3 * nf;
            const double2 p0 = q[i0], p1 = q[nf + m1], p2 = q[2 * nf + c];
            const double2 p01 = make_double2(p0.x * p1.x - p0.y * p1.y, p0.x * p1.y + p0.y * p1.x);
            const double2 ph = make_double2(p01.x * p2.x - p01.y * p2.y, p01.x * p2.y + p01.y * p2.x);
            v = make_double2(ph.x * v.x - ph.y * v.y, ph.x * v.y + ph.y * v.x);
          }
          if (ACC) { v.x += cp->x; v.y += cp->y; }
          *cp = v;
        }
      }
    }
  }
}

template <bool AC, bool BC, bool CRE, bool ACC = false>
void bgemm(const GemmArgs& g, cudaStream_t st) {
  if (g.batch == 0 || g.M == 0 || g.N == 0) return;
  for (int64_t b0 = 0; b0 < g.batch; b0 += 65535) {
    GemmArgs c = g;
    c.boff = b0;
    const unsigned nz = (unsigned)std::min<int64_t>(65535, g.batch - b0);
    if (g.M <= 16) {
      bgemm_kernel<AC, BC, CRE, ACC, true><<<dim3((g.N + 95) / 96, 1, nz), 128, 0, st>>>(c);
    } else if (g.M <= 32 && g.N <= 32) {
      // small square blocks (per-plane axis-1 stages): one 32 x 32 tile, 64 threads
      bgemm_kernel<AC, BC, CRE, ACC, false, false, 4><<<dim3(1, 1, nz), 64, 0, st>>>(c);
    } else if (g.M <= 32 && g.N <= 40) {
      bgemm_kernel<AC, BC, CRE, ACC, false, false, 5><<<dim3(1, 1, nz), 64, 0, st>>>(c);
    } else if (g.N <= 32) {
      bgemm_kernel<AC, BC, CRE, ACC, false, true><<<dim3(1, (g.M + 63) / 64, nz), 128, 0, st>>>(c);
    } else {
      bgemm_kernel<AC, BC, CRE, ACC><<<dim3((g.N + 47) / 48, (g.M + 31) / 32, nz), 128, 0, st>>>(c);
    }
    FGT_LAUNCHED();
  }
}

inline GemmArgs gemm(const double* A, int64_t lda, int64_t sA, const double* B, int64_t ldb, int64_t sB,
              double* C, int64_t ldc, int64_t sC, int M, int N, int K, int64_t batch,
              const int64_t* cidx = nullptr, const int64_t* bidx = nullptr,
              const int64_t* aidx = nullptr) {
  GemmArgs g;
  g.A = A; g.B = B; g.C = C;
  g.M = M; g.N = N; g.K = K; g.batch = batch;
  g.lda = lda; g.ldb = ldb; g.ldc = ldc; g.sA = sA; g.sB = sB; g.sC = sC;
  g.cidx = cidx;
  g.bidx = bidx;
  g.aidx = aidx;
  g.boff = 0;
  g.bp = nullptr;
  g.bp_nf = 0;
  g.bp_half = 0;
  return g;
}


}  // namespace fgt
