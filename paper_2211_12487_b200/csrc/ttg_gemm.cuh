// ttg_gemm.cuh — general FP64 GEMM on the DMMA tensor pipe (sm_100a has no
// f64 tcgen05 kind: mma.sync.m16n8k16.f64, SASS DMMA).
//
//   C (m x n) = alpha op(A) op(B) + beta C,  column-major, any strides,
//   op(X) = X or X^T (template TA / TB).
//
// Every plain GEMM of the sweep goes through it: the high-rank (r > 34)
// projections of tt_project / the companion sweep (op(A) = W^T, B = the
// streamed source), the explicit residual R = X - U (U^T X), small-side Grams
// R^T R, the append guard's [U_pad U_R]^T [U_pad U_R] and the a x a algebra of
// the raw-Gram projector.  It replaces cuBLAS DGEMM / DSYRK and the DFMA
// k_gemm of round 1.
//
// Tile BM x 64 x 16 (BM = 64 or 128), 2 x BM/32 warps of 32 x 32 (2 m16 x 4 n8
// DMMA blocks, 32 accumulators per lane).  Operands are staged global ->
// registers -> shared memory (double-buffered through registers, so both
// transposes use the same path) into k-major tiles As[k][m], Bs[k][n] with
// leading dimension = 4 (mod 16) doubles: the m16n8k16 fragment loads of a
// half-warp (g = 0..3, t = 0..3 -> offsets t*ld + g) then hit 16 distinct
// 8-byte banks.  Deterministic: every output is one fixed-order k chain; a
// split-K launch (grid z) writes per-chunk partials that k_dgemm_reduce sums
// in chunk order.
#pragma once
#include "ttg_kernels.cuh"

namespace ttg {

struct DgemmArgs {
  const double* A;
  long long lda;
  const double* B;
  long long ldb;
  double* C;
  long long ldc;
  long long m, n, k;
  double alpha, beta;
  long long kchunk;  // k range of one grid-z slice (multiple of 16)
  double* ws;        // split-K partials [gridDim.z][m][n] (compact), or null
};

constexpr int kGemmBN = 64, kGemmBK = 16;

template <int BM>
constexpr size_t dgemm_smem() {
  return sizeof(double) * 2 * kGemmBK * ((BM + 4) + (kGemmBN + 4));
}

template <bool TA, bool TB, int BM>
__global__ void __launch_bounds__(BM * 2) k_dgemm(DgemmArgs p) {
  griddep_wait();
  constexpr int BN = kGemmBN, BK = kGemmBK, NT = BM * 2, LDA = BM + 4, LDB = BN + 4;
  constexpr int NA = BM * BK / NT, NB = BK * BN / NT;  // elements per thread per tile (8 / 4)
  extern __shared__ __align__(16) double gsm[];
  double* As = gsm;                  // [2][BK][LDA]
  double* Bs = gsm + 2 * BK * LDA;   // [2][BK][LDB]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  constexpr int WM = BM / 32;
  const int wm = warp % WM, wn = warp / WM;
  const long long m0 = (long long)blockIdx.y * BM, n0 = (long long)blockIdx.x * BN;
  const long long kb = (long long)blockIdx.z * p.kchunk;
  const long long ke = min(p.k, kb + p.kchunk);

  double ra[NA], rb[NB];
  auto load = [&](long long k0) {
#pragma unroll
    for (int q = 0; q < NA; ++q) {
      const int e = tid + NT * q;
      int mm, kk;
      if (!TA) { mm = e % BM; kk = e / BM; } else { kk = e % BK; mm = e / BK; }
      const long long gm = m0 + mm, gk = k0 + kk;
      double v = 0.0;
      if (gm < p.m && gk < ke) v = TA ? p.A[gk + p.lda * gm] : p.A[gm + p.lda * gk];
      ra[q] = v;
    }
#pragma unroll
    for (int q = 0; q < NB; ++q) {
      const int e = tid + NT * q;
      int nn, kk;
      if (!TB) { kk = e % BK; nn = e / BK; } else { nn = e % BN; kk = e / BN; }
      const long long gn = n0 + nn, gk = k0 + kk;
      double v = 0.0;
      if (gn < p.n && gk < ke) v = TB ? p.B[gn + p.ldb * gk] : p.B[gk + p.ldb * gn];
      rb[q] = v;
    }
  };
  auto store = [&](int buf) {
    double* as = As + buf * BK * LDA;
    double* bs = Bs + buf * BK * LDB;
#pragma unroll
    for (int q = 0; q < NA; ++q) {
      const int e = tid + NT * q;
      int mm, kk;
      if (!TA) { mm = e % BM; kk = e / BM; } else { kk = e % BK; mm = e / BK; }
      as[kk * LDA + mm] = ra[q];
    }
#pragma unroll
    for (int q = 0; q < NB; ++q) {
      const int e = tid + NT * q;
      int nn, kk;
      if (!TB) { kk = e % BK; nn = e / BK; } else { nn = e % BN; kk = e / BN; }
      bs[kk * LDB + nn] = rb[q];
    }
  };

  double acc[2][4][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = acc[i][j][2] = acc[i][j][3] = 0.0;

  const int ntile = (int)((ke - kb + BK - 1) / BK);
  if (ntile > 0) {
    load(kb);
    store(0);
    __syncthreads();
    for (int it = 0; it < ntile; ++it) {
      const int buf = it & 1;
      if (it + 1 < ntile) load(kb + (long long)(it + 1) * BK);
      const double* as = As + buf * BK * LDA + wm * 32;
      const double* bs = Bs + buf * BK * LDB + wn * 32;
      double af[2][8], bf[4][4];
#pragma unroll
      for (int mb = 0; mb < 2; ++mb)
#pragma unroll
        for (int i = 0; i < 8; ++i) af[mb][i] = as[(t + 4 * (i >> 1)) * LDA + mb * 16 + g + 8 * (i & 1)];
#pragma unroll
      for (int nb = 0; nb < 4; ++nb)
#pragma unroll
        for (int i = 0; i < 4; ++i) bf[nb][i] = bs[(t + 4 * i) * LDB + nb * 8 + g];
#pragma unroll
      for (int mb = 0; mb < 2; ++mb)
#pragma unroll
        for (int nb = 0; nb < 4; ++nb) dmma16(acc[mb][nb], af[mb], bf[nb]);
      if (it + 1 < ntile) {
        store(buf ^ 1);
        __syncthreads();
      }
    }
  }
  // epilogue
#pragma unroll
  for (int mb = 0; mb < 2; ++mb)
#pragma unroll
    for (int nb = 0; nb < 4; ++nb)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const long long row = m0 + wm * 32 + mb * 16 + g + 8 * (i >> 1);
        const long long col = n0 + wn * 32 + nb * 8 + 2 * t + (i & 1);
        if (row >= p.m || col >= p.n) continue;
        const double v = acc[mb][nb][i];
        if (p.ws) {
          p.ws[(long long)blockIdx.z * p.m * p.n + row + p.m * col] = v;
        } else {
          double* cp = p.C + row + p.ldc * col;
          *cp = p.beta != 0.0 ? fma(p.alpha, v, p.beta * *cp) : p.alpha * v;
        }
      }
}

// C = alpha sum_z ws[z] + beta C, chunks summed in order (deterministic).
__global__ void k_dgemm_reduce(const double* __restrict__ ws, int nz, long long m, long long n, double* C,
                               long long ldc, double alpha, double beta) {
  griddep_wait();
  const long long tot = m * n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot;
       e += (long long)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int z = 0; z < nz; ++z) s += ws[(long long)z * tot + e];
    const long long row = e % m, col = e / m;
    double* cp = C + row + ldc * col;
    *cp = beta != 0.0 ? fma(alpha, s, beta * *cp) : alpha * s;
  }
}

}  // namespace ttg
