// ttg_io.cuh — device kernels of the metrics / checkpoint rows:
// relative reconstruction / prediction error without materialising the
// reconstruction, and the orthonormality measurement used when a TTC1
// checkpoint is loaded.
#pragma once
#include "ttg_pdl.cuh"
#include "ttg_kernels.cuh"
#include <cstdint>
#include <cuda_runtime.h>

namespace ttg {

// Partial sums over a slab of the data:  d = sum (x - Phi c)^2,  x2 = sum x^2.
// Phi: S x r (column-major, the spatial chain), C: r x m coefficients (ld ldc),
// X: S x m (ld ldx).  One thread per row s of Phi keeps that row in
// registers (r <= RMAX) and walks the m observations; the coefficients are
// staged in shared memory 64 observations at a time.  Per-block partials are
// written in fixed order (k_pair_sum reduces them deterministically).
constexpr int kRreObsChunk = 64;
template <int RMAX>
__global__ void __launch_bounds__(256) k_rre_partial(const double* __restrict__ Phi, long long S, int r,
                                                     const double* __restrict__ C, long long ldc, int m,
                                                     const double* __restrict__ X, long long ldx,
                                                     double* __restrict__ part) {
  griddep_wait();
  __shared__ __align__(16) double cs[kRreObsChunk * RMAX];
  __shared__ double red[2][8];
  double dsum = 0.0, xsum = 0.0;
  const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const bool live = s < S;
  double phi[RMAX];
#pragma unroll
  for (int k = 0; k < RMAX; ++k) phi[k] = (live && k < r) ? Phi[s + S * k] : 0.0;
  for (int o0 = 0; o0 < m; o0 += kRreObsChunk) {
    const int mo = min(kRreObsChunk, m - o0);
    __syncthreads();
    for (int e = threadIdx.x; e < mo * RMAX; e += blockDim.x) {
      const int o = e / RMAX, k = e - o * RMAX;
      cs[e] = k < r ? C[k + ldc * (o0 + o)] : 0.0;
    }
    __syncthreads();
    if (live) {
      // four observations per round: their X loads are issued together (one
      // 8-byte load in flight per thread kept the kernel at ~54 % of HBM: too
      // few bytes in flight per SM), and the coefficients come as broadcast
      // 16-byte shared loads, one LDS per two FMAs
      const double* xp = X + s + ldx * (long long)o0;
      int o = 0;
      for (; o + 4 <= mo; o += 4) {
        double x[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) x[q] = __ldcs(xp + ldx * (o + q));
        double d0[4], d1[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) d0[q] = d1[q] = 0.0;
#pragma unroll
        for (int k = 0; k < RMAX / 2; ++k) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const double2 cc = reinterpret_cast<const double2*>(cs + (o + q) * RMAX)[k];
            d0[q] = fma(phi[2 * k], cc.x, d0[q]);
            d1[q] = fma(phi[2 * k + 1], cc.y, d1[q]);
          }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double df = x[q] - (d0[q] + d1[q]);
          dsum = fma(df, df, dsum);
          xsum = fma(x[q], x[q], xsum);
        }
      }
      for (; o < mo; ++o) {
        const double2* co = reinterpret_cast<const double2*>(cs + o * RMAX);
        double dot0 = 0.0, dot1 = 0.0;
#pragma unroll
        for (int k = 0; k < RMAX / 2; ++k) {
          const double2 cc = co[k];
          dot0 = fma(phi[2 * k], cc.x, dot0);
          dot1 = fma(phi[2 * k + 1], cc.y, dot1);
        }
        const double x = __ldcs(xp + ldx * o);
        const double df = x - (dot0 + dot1);
        dsum = fma(df, df, dsum);
        xsum = fma(x, x, xsum);
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    dsum += __shfl_xor_sync(0xffffffffu, dsum, o);
    xsum += __shfl_xor_sync(0xffffffffu, xsum, o);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    red[0][warp] = dsum;
    red[1][warp] = xsum;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      a += red[0][w];
      b += red[1][w];
    }
    part[2 * blockIdx.x] = a;
    part[2 * blockIdx.x + 1] = b;
  }
}

// The same partial sums on the FP64 tensor pipe (r <= 32).  The DFMA kernel
// above issues one shared-memory load per two FMAs and its ncu capture shows
// it waiting on exactly those (short scoreboard 5.5, LSU pipe 44 % busy, 57 %
// of HBM).  Here a warp owns 32 rows (four m8n8k4 row blocks, its Phi
// fragments in registers for the whole chunk) and walks the observations
// eight at a time: 16 DMMAs per 4 coefficient loads, the eight X loads of a
// lane in flight together.  Coefficients sit in shared memory with a stride
// = 4 (mod 16), so a half-warp's fragment load hits 16 distinct banks.
template <int RMAX>
__global__ void __launch_bounds__(256) k_rre_dmma(const double* __restrict__ Phi, long long S, int r,
                                                  const double* __restrict__ C, long long ldc, int m,
                                                  const double* __restrict__ X, long long ldx,
                                                  double* __restrict__ part) {
  griddep_wait();
  constexpr int NJ = RMAX / 4, LDC_S = RMAX + 4;
  __shared__ __align__(16) double cs[kRreObsChunk * LDC_S];
  __shared__ double red[2][8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const long long s_base = blockIdx.x * (long long)blockDim.x + warp * 32;
  double a[4][NJ];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const long long s = s_base + 8 * q + g;
#pragma unroll
    for (int j = 0; j < NJ; ++j) a[q][j] = (s < S && 4 * j + t < r) ? Phi[s + S * (4 * j + t)] : 0.0;
  }
  double dsum = 0.0, xsum = 0.0;
  for (int o0 = 0; o0 < m; o0 += kRreObsChunk) {
    const int mo = min(kRreObsChunk, m - o0);
    __syncthreads();
    for (int e = threadIdx.x; e < kRreObsChunk * RMAX; e += blockDim.x) {
      const int o = e / RMAX, k = e - o * RMAX;
      cs[o * LDC_S + k] = (o < mo && k < r) ? C[k + ldc * (o0 + o)] : 0.0;
    }
    __syncthreads();
    for (int og = 0; og < mo; og += 8) {
      double x[4][2];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const long long s = s_base + 8 * q + g;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int o = og + 2 * t + h;
          x[q][h] = (s < S && o < mo) ? __ldcs(X + s + ldx * (long long)(o0 + o)) : 0.0;
        }
      }
      double b[NJ];
#pragma unroll
      for (int j = 0; j < NJ; ++j) b[j] = cs[(og + g) * LDC_S + 4 * j + t];
      double acc[4][2];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q][0] = acc[q][1] = 0.0;
#pragma unroll
      for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int q = 0; q < 4; ++q) dmma(acc[q][0], acc[q][1], a[q][j], b[j]);
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const double df = x[q][h] - acc[q][h];  // (masked entries: x = 0 and Phi row or coefficient column = 0)
          dsum = fma(df, df, dsum);
          xsum = fma(x[q][h], x[q][h], xsum);
        }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    dsum += __shfl_xor_sync(0xffffffffu, dsum, o);
    xsum += __shfl_xor_sync(0xffffffffu, xsum, o);
  }
  if (lane == 0) {
    red[0][warp] = dsum;
    red[1][warp] = xsum;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double u = 0.0, v = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      u += red[0][w];
      v += red[1][w];
    }
    part[2 * blockIdx.x] = u;
    part[2 * blockIdx.x + 1] = v;
  }
}

// Generic variant for r > 64: Phi row entries read through the cache.
__global__ void __launch_bounds__(256) k_rre_partial_any(const double* __restrict__ Phi, long long S, int r,
                                                         const double* __restrict__ C, long long ldc, int m,
                                                         const double* __restrict__ X, long long ldx,
                                                         double* __restrict__ part) {
  griddep_wait();
  __shared__ double red[2][8];
  double dsum = 0.0, xsum = 0.0;
  const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s < S) {
    for (int o = 0; o < m; ++o) {
      double dot = 0.0;
      for (int k = 0; k < r; ++k) dot = fma(Phi[s + S * k], C[k + ldc * o], dot);
      const double x = X[s + ldx * o];
      const double df = x - dot;
      dsum = fma(df, df, dsum);
      xsum = fma(x, x, xsum);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    dsum += __shfl_xor_sync(0xffffffffu, dsum, o);
    xsum += __shfl_xor_sync(0xffffffffu, xsum, o);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    red[0][warp] = dsum;
    red[1][warp] = xsum;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      a += red[0][w];
      b += red[1][w];
    }
    part[2 * blockIdx.x] = a;
    part[2 * blockIdx.x + 1] = b;
  }
}

// out[0..1] = fixed-order sums of the n pairs in part (one warp, strided
// per-lane partials then a butterfly: deterministic for a given n)
__global__ void k_pair_sum(const double* __restrict__ part, long long n, double* __restrict__ out) {
  griddep_wait();
  double a = 0.0, b = 0.0;
  for (long long i = threadIdx.x; i < n; i += 32) {
    a += part[2 * i];
    b += part[2 * i + 1];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  if (threadIdx.x == 0) {
    out[0] = a;
    out[1] = b;
  }
}

// dev = max |U^T U - I| of one left unfolding U (a x r, column-major),
// one block: entry (i, j) of the Gram per thread-strided loop.
__global__ void k_ortho_dev(const double* __restrict__ U, int a, int r, double* __restrict__ dev) {
  griddep_wait();
  __shared__ double red[32];
  double mx = 0.0;
  for (long long e = threadIdx.x; e < (long long)r * r; e += blockDim.x) {
    const int i = (int)(e % r), j = (int)(e / r);
    if (i > j) continue;
    double s = 0.0;
    for (int k = 0; k < a; ++k) s = fma(U[k + (long long)a * i], U[k + (long long)a * j], s);
    mx = fmax(mx, fabs(s - (i == j ? 1.0 : 0.0)));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, red[w]);
    *dev = m;
  }
}

}  // namespace ttg
