// ttg_eig.cuh — basis selection: one-sided Jacobi eigen-solve of the residual
// Gram, error-truncation rank rule, sign rule, and the 1e-10 Gram-guarded
// append (Householder re-orthogonalisation).
//
// Restates, on the Gram G = R R^T instead of R itself:
//   svd_trunc            truncated_svd.cpp:29-94 (rank loop :74-81 with the '>'
//                        test, sign rule :16-25 = largest-|.| entry, first index)
//   append_directions    update_common.hpp:19-36 (kGramGuard = 1e-10, Householder Q)
// sigma_j^2 of R are the eigenvalues of G; its left singular vectors are G's
// eigenvectors.  One-sided (Hestenes) Jacobi on W = G: columns converge to
// lambda_j v_j, so lambda_j = |w_j| and v_j = w_j / lambda_j — no V matrix is
// kept, which lets a <= 165 live entirely in shared memory.
#pragma once
#include "ttg_pdl.cuh"
#include <cstdint>
#include <cuda_runtime.h>

namespace ttg {

struct EigResult {
  int rank;
  int converged;
  int sweeps;
  int guard;      // append guard fired
  double tail_sq;
  double delta;
  double lam_max;
  double dev;     // append Gram deviation
  double lam_min_kept;  // smallest kept sigma^2
  long long t_phase[4];  // clock64 stamps of the solver phases (diagnostics)
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

constexpr int kEigThreads = 1024;

struct EigArgs {
  const double* G;    // a x a symmetric (global)
  int a;
  long long kmax;     // number of singular values of R = min(a, #columns)
  double* Wg;         // global scratch a x a (used when !in_smem)
  int in_smem;
  int factor;         // 1: G holds an upper-triangular factor T (T^T T = R R^T); solve on W = T^T,
                      //    column norms are sigma (not sigma^2)
  const double* delta_src;  // if non-null: delta = delta_mult * sqrt(*delta_src)
  double delta_mult;
  double tol;
  int max_sweeps;
  double* UR;         // out: a x rank (column-major, ld a)
  double* lam;        // out: a sorted eigenvalues (descending)
  EigResult* res;
};

__global__ void __launch_bounds__(kEigThreads) k_jacobi_eig(EigArgs p) {
  griddep_wait();
  extern __shared__ __align__(16) double esm[];
  const int a = p.a;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  double* W = p.in_smem ? esm : p.Wg;
  double* nrm = p.in_smem ? esm + (size_t)a * a : esm;  // a doubles
  int* perm = reinterpret_cast<int*>(nrm + a);            // a ints
  __shared__ int s_rot;
  __shared__ int s_sweeps;

  for (long long e = threadIdx.x; e < (long long)a * a; e += blockDim.x) {
    if (p.factor) {
      long long i = e % a, j = e / a;
      W[e] = p.G[j + (long long)a * i];  // W = T^T
    } else {
      W[e] = p.G[e];
    }
  }
  __syncthreads();

  const int n = a + (a & 1);
  int sweep = 0;
  for (; sweep < p.max_sweeps; ++sweep) {
    if (threadIdx.x == 0) s_rot = 0;
    __syncthreads();
    for (int rnd = 0; rnd < n - 1; ++rnd) {
      for (int k = warp; k < n / 2; k += nwarps) {
        int pp = (k == 0) ? 0 : ((k - 1 + rnd) % (n - 1)) + 1;
        int qq = ((n - 2 - k + rnd) % (n - 1)) + 1;
        if (pp >= a || qq >= a) continue;
        if (pp > qq) { int tmp = pp; pp = qq; qq = tmp; }
        double* wp = W + (size_t)pp * a;
        double* wq = W + (size_t)qq * a;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int i = lane; i < a; i += 32) {
          double x = wp[i], y = wq[i];
          al = fma(x, x, al);
          be = fma(y, y, be);
          ga = fma(x, y, ga);
        }
        al = warp_sum(al);
        be = warp_sum(be);
        ga = warp_sum(ga);
        if (ga != 0.0 && fabs(ga) > p.tol * sqrt(al) * sqrt(be)) {
          double zeta = (be - al) / (2.0 * ga);
          double tt = copysign(1.0, zeta) / (fabs(zeta) + hypot(1.0, zeta));
          double c = 1.0 / sqrt(1.0 + tt * tt);
          double s = c * tt;
          for (int i = lane; i < a; i += 32) {
            double x = wp[i], y = wq[i];
            wp[i] = c * x - s * y;
            wq[i] = s * x + c * y;
          }
          if (lane == 0) s_rot = 1;
        }
      }
      __syncthreads();
    }
    if (s_rot == 0) break;
    __syncthreads();
  }
  if (threadIdx.x == 0) s_sweeps = sweep;

  // eigenvalues = column norms
  for (int j = warp; j < a; j += nwarps) {
    double s = 0.0;
    for (int i = lane; i < a; i += 32) s = fma(W[(size_t)j * a + i], W[(size_t)j * a + i], s);
    s = warp_sum(s);
    if (lane == 0) nrm[j] = sqrt(s);  // lambda_j (Gram) or sigma_j (factor)
  }
  __syncthreads();
  // descending stable rank sort
  for (int j = threadIdx.x; j < a; j += blockDim.x) {
    double v = nrm[j];
    int pos = 0;
    for (int i = 0; i < a; ++i) {
      double u = nrm[i];
      pos += (u > v) || (u == v && i < j);
    }
    perm[pos] = j;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < a; j += blockDim.x) {
    double v = nrm[perm[j]];
    p.lam[j] = p.factor ? v * v : v;  // sigma_j^2, descending
  }
  __shared__ int s_rank;
  if (threadIdx.x == 0) {
    double delta = p.delta_src ? p.delta_mult * sqrt(*p.delta_src) : p.delta_mult;
    long long k = p.kmax < a ? p.kmax : a;
    double tail_sq = 0.0;
    long long rank = k;
    for (long long j = k - 1; j >= 0; --j) {  // truncated_svd.cpp:74-81
      double sj = nrm[perm[j]];
      double next = tail_sq + (p.factor ? sj * sj : sj);  // sigma_j^2
      if (sqrt(next) > delta) break;
      tail_sq = next;
      rank = j;
    }
    s_rank = (int)rank;
    p.res->rank = (int)rank;
    p.res->tail_sq = tail_sq;
    p.res->delta = delta;
    p.res->converged = (s_sweeps < p.max_sweeps);
    p.res->sweeps = s_sweeps;
    double l0 = a > 0 ? nrm[perm[0]] : 0.0;
    double lr = rank > 0 ? nrm[perm[rank - 1]] : 0.0;
    p.res->lam_max = p.factor ? l0 * l0 : l0;
    p.res->lam_min_kept = p.factor ? lr * lr : lr;
  }
  __syncthreads();
  const int rank = s_rank;
  // U_R columns: normalised, sign rule (truncated_svd.cpp:16-25)
  for (int j = warp; j < rank; j += nwarps) {
    const double* w = W + (size_t)perm[j] * a;
    double inv = 1.0 / nrm[perm[j]];
    double best = -1.0;
    int bi = a;
    for (int i = lane; i < a; i += 32) {
      double v = fabs(w[i] * inv);
      if (v > best) { best = v; bi = i; }  // first max within the lane's strided set
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      double ob = __shfl_xor_sync(0xffffffffu, best, o);
      int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    double sgn = (w[bi] * inv < 0.0) ? -1.0 : 1.0;
    for (int i = lane; i < a; i += 32) p.UR[(size_t)j * a + i] = sgn * (w[i] * inv);
  }
}

// ---------------------------------------------------------------------------
// append_directions (update_common.hpp:19-36): C = [U_pad U_R]; if
// max|C^T C - I| > 1e-10, U_R <- HouseholderQ(U_R - U_pad U_pad^T U_R).
// Single CTA; r_new is small.  Writes C (a x r_new, ld a) to `out`.
// ---------------------------------------------------------------------------
struct AppendArgs {
  const double* Upad;  // a x r_old
  const double* UR;    // a x r_R
  int a, r_old, r_R;
  double* out;         // a x (r_old + r_R)
  double* scratch;     // a x r_R + r_R
  EigResult* res;
  int* guard_count;    // incremented when the guard fires (read once per update: no host sync per mode)
  int precomputed;     // out already holds [U_pad U_R] and res->dev the Gram deviation (k_gram_dev)
};

// Gram deviation max |S_ij - delta_ij| over the lower triangle of S = C^T C
// (n x n, from cuBLAS DSYRK) -> res->dev as an atomic max on the bit pattern
// (non-negative doubles order like their bits); res->dev zeroed beforehand.
__global__ void k_gram_dev(const double* __restrict__ S, int n, EigResult* res) {
  griddep_wait();
  __shared__ double red[32];
  double m = 0.0;
  const long long tot = (long long)n * n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e % n), j = (int)(e / n);
    if (i >= j) m = fmax(m, fabs(S[e] - (i == j ? 1.0 : 0.0)));
  }
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) red[warp] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) b = fmax(b, red[w]);
    atomicMax(reinterpret_cast<unsigned long long*>(&res->dev), (unsigned long long)__double_as_longlong(b));
  }
}

__device__ void block_max_reduce(double& v, double* red) {
  v = fmax(v, __shfl_xor_sync(0xffffffffu, v, 16));
  v = fmax(v, __shfl_xor_sync(0xffffffffu, v, 8));
  v = fmax(v, __shfl_xor_sync(0xffffffffu, v, 4));
  v = fmax(v, __shfl_xor_sync(0xffffffffu, v, 2));
  v = fmax(v, __shfl_xor_sync(0xffffffffu, v, 1));
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = red[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, red[w]);
    red[32] = m;
  }
  __syncthreads();
  v = red[32];
  __syncthreads();
}

__device__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    red[32] = s;
  }
  __syncthreads();
  double r = red[32];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(1024) k_append(AppendArgs p) {
  griddep_wait();
  __shared__ double red[33];
  const int a = p.a, r0 = p.r_old, rr = p.r_R, rn = r0 + rr;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  double dev = 0.0;
  if (p.precomputed) {
    dev = p.res->dev;
  } else {
    for (long long e = threadIdx.x; e < (long long)a * rn; e += blockDim.x) {
      long long c = e / a;
      p.out[e] = (c < r0) ? p.Upad[e] : p.UR[e - (long long)r0 * a];
    }
    __syncthreads();
    // Gram deviation of the combined block
    for (int pr = warp; pr < rn * rn; pr += nwarps) {
      int ci = pr % rn, cj = pr / rn;
      if (cj < ci) continue;
      double s = 0.0;
      for (int i = lane; i < a; i += 32) s = fma(p.out[(size_t)ci * a + i], p.out[(size_t)cj * a + i], s);
      s = warp_sum(s);
      dev = fmax(dev, fabs(s - (ci == cj ? 1.0 : 0.0)));
    }
    block_max_reduce(dev, red);
  }
  if (threadIdx.x == 0) {
    p.res->dev = dev;
    p.res->guard = (dev > 1e-10) ? 1 : 0;
    if (dev > 1e-10 && p.guard_count) atomicAdd(p.guard_count, 1);
  }
  if (!(dev > 1e-10)) return;

  // corrected = U_R - U_pad (U_pad^T U_R)   -> scratch (a x rr)
  double* Cr = p.scratch;
  double* coef = p.scratch + (size_t)a * rr;  // r0 x rr
  for (int pr = warp; pr < r0 * rr; pr += nwarps) {
    int ci = pr % r0, cj = pr / r0;
    double s = 0.0;
    for (int i = lane; i < a; i += 32) s = fma(p.Upad[(size_t)ci * a + i], p.UR[(size_t)cj * a + i], s);
    s = warp_sum(s);
    if (lane == 0) coef[ci + (size_t)r0 * cj] = s;
  }
  __syncthreads();
  for (long long e = threadIdx.x; e < (long long)a * rr; e += blockDim.x) {
    long long c = e / a, i = e - c * a;
    double s = p.UR[e];
    for (int k = 0; k < r0; ++k) s -= p.Upad[(size_t)k * a + i] * coef[k + (size_t)r0 * c];
    Cr[e] = s;
  }
  __syncthreads();
  // Householder QR in place (Eigen makeHouseholderInPlace convention):
  // v_j = [1; x_{j+1:}/(x_j - beta)], tau_j = (beta - x_j)/beta, beta = -sign(x_j)|x|
  double* taus = coef;  // coef is no longer needed: reuse for the rr Householder taus
  for (int j = 0; j < rr; ++j) {
    double* x = Cr + (size_t)j * a;
    double tsq = 0.0;
    for (int i = j + 1 + threadIdx.x; i < a; i += blockDim.x) tsq = fma(x[i], x[i], tsq);
    tsq = block_sum(tsq, red);
    double c0 = x[j];
    double beta, tj;
    bool trivial = tsq <= 2.2250738585072014e-308;  // numeric_limits<double>::min()
    if (trivial) {
      tj = 0.0;
      beta = c0;
    } else {
      beta = sqrt(c0 * c0 + tsq);
      if (c0 >= 0.0) beta = -beta;
      tj = (beta - c0) / beta;
    }
    double scale = trivial ? 0.0 : 1.0 / (c0 - beta);
    __syncthreads();
    for (int i = j + 1 + threadIdx.x; i < a; i += blockDim.x) x[i] *= scale;
    if (threadIdx.x == 0) { x[j] = beta; taus[j] = tj; }
    __syncthreads();
    // apply H_j = I - tau v v^T to columns j+1..rr-1 (rows j..a-1)
    for (int c = j + 1; c < rr; ++c) {
      double* y = Cr + (size_t)c * a;
      double s = 0.0;
      for (int i = j + 1 + threadIdx.x; i < a; i += blockDim.x) s = fma(x[i], y[i], s);
      s = block_sum(s, red);
      s += y[j];
      double f = tj * s;
      __syncthreads();
      if (threadIdx.x == 0) y[j] -= f;
      for (int i = j + 1 + threadIdx.x; i < a; i += blockDim.x) y[i] -= f * x[i];
      __syncthreads();
    }
  }
  // Q = H_0 H_1 ... H_{rr-1} [I_rr; 0]  -> out[:, r0:]
  double* Q = p.out + (size_t)r0 * a;
  for (long long e = threadIdx.x; e < (long long)a * rr; e += blockDim.x) {
    long long c = e / a, i = e - c * a;
    Q[e] = (i == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int j = rr - 1; j >= 0; --j) {
    const double* v = Cr + (size_t)j * a;  // essential part below row j
    double tj = taus[j];
    for (int c = j; c < rr; ++c) {
      double* y = Q + (size_t)c * a;
      double s = 0.0;
      for (int i = j + 1 + threadIdx.x; i < a; i += blockDim.x) s = fma(v[i], y[i], s);
      s = block_sum(s, red);
      s += y[j];
      double f = tj * s;
      __syncthreads();
      if (threadIdx.x == 0) y[j] -= f;
      for (int i = j + 1 + threadIdx.x; i < a; i += blockDim.x) y[i] -= f * v[i];
      __syncthreads();
    }
  }
}

}  // namespace ttg
