// ttg_syev.cuh — fast symmetric eigen-solve of the residual Gram for the
// truncated-SVD rank rule (restates svd_trunc, truncated_svd.cpp:29-94, on
// G = R R^T).  One CTA:
//   1. Householder tridiagonalisation Q^T G Q = T (LAPACK dsytd2 'L' shape),
//      G in shared memory when it fits, else in an L2-resident scratch;
//   2. the top eigenvalues of T by Sturm-count multisection (one warp per
//      eigenvalue, 32 evaluation points per round), in batches of 32 until
//      trace(G) - sum_{j<r} lambda_j <= delta^2 decides the rank (the
//      reference's minimal-rank loop :74-81, '>' keeps the smaller rank);
//   3. eigenvectors of T for the kept eigenvalues by inverse iteration,
//      re-orthogonalised within clusters; back-transformed by the Householder
//      reflectors; sign rule (:16-25).
// Flops ~ 4/3 a^3 + O(a^2) instead of the O(sweeps * a^3) of Jacobi, with
// O(a) block barriers.  Accuracy: eigenvalues to eps |G| absolute,
// eigenvectors to eps |G| / gap — the same as a Jacobi solve of G.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "ttg_eig.cuh"

namespace ttg {

struct SyevArgs {
  const double* G;        // a x a symmetric (global)
  int a;
  long long kmax;         // rank cap = min(a, #columns)
  double* Ag;             // global scratch a x a when !in_smem
  int in_smem;
  const double* delta_src;  // delta = delta_mult * sqrt(*delta_src) if non-null
  double delta_mult;
  double* UR;             // out: a x rank
  double* lam;            // out: computed eigenvalues, descending (first n_lam)
  double* zbuf;           // scratch: 32 x 6a (inverse-iteration vectors + LU factors)
  EigResult* res;
};

constexpr int kSyevThreads = 1024;

// Block-wide sum, returned to every thread (fixed butterfly order: deterministic).
// `red` must not be reused until the caller has passed another barrier.
__device__ __forceinline__ double block_sum_all(double v, double* red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = (lane < nw) ? red[lane] : 0.0;
  return warp_sum(s);
}

// Number of eigenvalues of the tridiagonal (d, e2 = e^2) strictly below x:
// sign changes of the Sturm sequence p_k = (d_k - x) p_{k-1} - e2_{k-1} p_{k-2},
// kept in range by exact power-of-two rescaling (no divisions on the chain).
// A zero p_k takes the sign opposite to p_{k-1} (LAPACK's -pivmin convention).
__device__ __forceinline__ int sturm_count(const double* d, const double* e2, int n, double x) {
  const double kBig = 0x1p+600, kSmall = 0x1p-600;
  int cnt = 0;
  double p2 = 1.0;          // p_{k-1}
  double p1 = d[0] - x;     // p_k
  bool s_prev = false;      // sign bit of p_0 = +1
  bool s1 = (p1 < 0.0) || (p1 == 0.0 && !s_prev);
  cnt += (s1 != s_prev);
  for (int i = 1; i < n; ++i) {
    double pn = fma(d[i] - x, p1, -e2[i - 1] * p2);
    const bool sn = (pn < 0.0) || (pn == 0.0 && !s1);
    cnt += (sn != s1);
    p2 = p1;
    p1 = pn;
    s1 = sn;
    const double ap = fabs(p1);
    if (ap > kBig) {
      p1 *= kSmall;
      p2 *= kSmall;
    } else if (ap < kSmall && fabs(p2) < kSmall) {
      p1 *= kBig;
      p2 *= kBig;
    }
  }
  return cnt;
}

__global__ void __launch_bounds__(kSyevThreads) k_syev(SyevArgs p) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double red[33];
  __shared__ int s_rank, s_done;
  __shared__ double s_tail;
  const int a = p.a;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  double* A = p.in_smem ? sm : p.Ag;
  double* vec = p.in_smem ? sm + (size_t)a * a : sm;
  double* d = vec;            // a
  double* e = d + a;          // a (e[a-1] unused)
  double* e2 = e + a;         // a
  double* tau = e2 + a;       // a
  double* v = tau + a;        // a   current Householder vector
  double* w = v + a;          // a   p / w
  double* lam = w + a;        // a   top eigenvalues (descending)

  const long long t0 = clock64();
  for (long long i = tid; i < (long long)a * a; i += blockDim.x) A[i] = p.G[i];
  __syncthreads();
  double trace = 0.0;
  for (int i = 0; i < a; ++i) trace += A[i + (size_t)a * i];  // all threads, same order

  // ---- 1. tridiagonalisation --------------------------------------------
  double* red2 = red;  // alias; every use is separated by a barrier
  for (int k = 0; k + 2 < a; ++k) {
    const int m = a - k - 1;           // trailing size, rows k+1..a-1
    double* col = A + (size_t)a * k;   // column k
    double xs = 0.0;
    for (int i = k + 2 + tid; i < a; i += blockDim.x) xs = fma(col[i], col[i], xs);
    xs = block_sum_all(xs, red);
    const double alpha = col[k + 1];
    if (tid == 0) d[k] = col[k];
    if (xs == 0.0) {
      if (tid == 0) { e[k] = alpha; tau[k] = 0.0; }
      __syncthreads();
      continue;
    }
    double beta = sqrt(alpha * alpha + xs);
    if (alpha >= 0.0) beta = -beta;
    const double tk = (beta - alpha) / beta;
    const double sc = 1.0 / (alpha - beta);
    for (int i = tid; i < m; i += blockDim.x) v[i] = (i == 0) ? 1.0 : col[k + 1 + i] * sc;
    if (tid == 0) { e[k] = beta; tau[k] = tk; }
    __syncthreads();
    // lane-resident slices of v: rows/cols lane + 32*s for the first 256 (the rest from smem)
    double vr[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int i = lane + 32 * q;
      vr[q] = (i < m) ? v[i] : 0.0;
    }
    // w = tau * A22 v (A22 symmetric: row i = column i, contiguous); warp partial of w^T v
    double pvw = 0.0;
    for (int i = warp; i < m; i += nw) {
      const double* ci = A + (size_t)a * (k + 1 + i) + (k + 1);
      double s2 = 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int j = lane + 32 * q;
        if (j < m) s2 = fma(ci[j], vr[q], s2);
      }
      for (int j = lane + 256; j < m; j += 32) s2 = fma(ci[j], v[j], s2);  // a > 257 tail
      s2 = warp_sum(s2) * tk;
      if (lane == 0) w[i] = s2;
      pvw = fma(s2, v[i], pvw);
    }
    if (lane == 0) red2[warp] = pvw;
    __syncthreads();
    const double pv = warp_sum((lane < nw) ? red2[lane] : 0.0);
    const double al2 = -0.5 * tk * pv;
    double wr[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int i = lane + 32 * q;
      wr[q] = (i < m) ? fma(al2, vr[q], w[i]) : 0.0;
    }
    // A22 -= v w'^T + w' v^T with w' = w + al2 v  (2-D loop, v/w' in registers)
    for (int j = warp; j < m; j += nw) {
      const double vj = v[j], wj = fma(al2, vj, w[j]);
      double* cj = A + (size_t)a * (k + 1 + j) + (k + 1);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int i = lane + 32 * q;
        if (i < m) cj[i] -= vr[q] * wj + wr[q] * vj;
      }
      for (int i = lane + 256; i < m; i += 32) cj[i] -= v[i] * wj + fma(al2, v[i], w[i]) * vj;  // a > 257 tail
    }
    // keep v (essential part) in column k below the subdiagonal
    for (int i = 1 + tid; i < m; i += blockDim.x) col[k + 1 + i] = v[i];
    __syncthreads();
  }
  if (tid == 0) {
    if (a >= 2) {
      d[a - 2] = A[(a - 2) + (size_t)a * (a - 2)];
      e[a - 2] = A[(a - 1) + (size_t)a * (a - 2)];
      tau[a - 2] = 0.0;
    }
    d[a - 1] = A[(a - 1) + (size_t)a * (a - 1)];
    e[a - 1] = 0.0;
  }
  __syncthreads();
  double gl = 0.0, gu = 0.0, emax2 = 0.0;
  for (int i = 0; i < a; ++i) {  // Gershgorin bounds (all threads)
    double r = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < a ? fabs(e[i]) : 0.0);
    double lo = d[i] - r, hi = d[i] + r;
    if (i == 0 || lo < gl) gl = lo;
    if (i == 0 || hi > gu) gu = hi;
    if (i + 1 < a) emax2 = fmax(emax2, e[i] * e[i]);
  }
  for (int i = tid; i < a; i += blockDim.x) e2[i] = (i + 1 < a) ? e[i] * e[i] : 0.0;
  const double tnorm = fmax(fabs(gl), fabs(gu));
  const double pivmin = 2.2250738585072014e-308 * fmax(1.0, emax2);  // convergence floor
  gu += 2.2e-16 * tnorm * a + pivmin;
  gl -= 2.2e-16 * tnorm * a + pivmin;
  __syncthreads();

  const long long t1 = clock64();
  // ---- 2. top eigenvalues, batches of 32, until the rank rule decides ------
  const double delta = p.delta_src ? p.delta_mult * sqrt(*p.delta_src) : p.delta_mult;
  const long long kcap = p.kmax < a ? p.kmax : a;
  if (tid == 0) { s_done = 0; s_rank = (int)kcap; s_tail = 0.0; }
  __syncthreads();
  int n_lam = 0;
  int bsz = 4;  // the rank is usually tiny: start with 4 eigenvalues, then 32 per batch
  for (int base = 0; base < a && !s_done; base += bsz, bsz = nw) {
    const int j = base + warp;  // descending index
    if (warp < bsz && j < a) {
      const int t = a - 1 - j;  // ascending index
      double lo = gl, hi = gu;
      for (int it = 0; it < 40; ++it) {
        const double x = lo + (hi - lo) * (double)(lane + 1) / 33.0;
        const int cnt = sturm_count(d, e2, a, x);
        const unsigned above = __ballot_sync(0xffffffffu, cnt > t);  // x > lambda_t
        double nlo = lo, nhi = hi;
        if (above) {
          const int l = __ffs(above) - 1;
          nhi = lo + (hi - lo) * (double)(l + 1) / 33.0;
          nlo = (l == 0) ? lo : lo + (hi - lo) * (double)l / 33.0;
        } else {
          nlo = lo + (hi - lo) * 32.0 / 33.0;
        }
        lo = nlo;
        hi = nhi;
        if (hi - lo <= 2.2e-16 * fmax(fabs(lo), fabs(hi)) * 2.0 + pivmin) break;
      }
      if (lane == 0) lam[j] = 0.5 * (lo + hi);
    }
    __syncthreads();
    n_lam = min(a, base + bsz);
    if (tid == 0) {
      double pre = 0.0;
      int found = -1;
      for (int r = 0; r <= n_lam; ++r) {
        const double tail = trace - pre;  // sum of sigma^2 beyond the first r
        if (r <= kcap && !(sqrt(fmax(tail, 0.0)) > delta)) { found = r; break; }
        if (r < n_lam) pre += lam[r];
      }
      if (found >= 0 || n_lam >= a) {
        if (found < 0) found = (int)kcap;
        if (found > kcap) found = (int)kcap;
        double pre2 = 0.0;
        for (int r = 0; r < found; ++r) pre2 += lam[r];
        s_rank = found;
        s_tail = fmax(trace - pre2, 0.0);
        s_done = 1;
      }
    }
    __syncthreads();
  }
  const int rank = s_rank;
  const long long t2 = clock64();
  for (int j = tid; j < n_lam; j += blockDim.x) p.lam[j] = lam[j];
  if (tid == 0) {
    p.res->rank = rank;
    p.res->tail_sq = s_tail;
    p.res->delta = delta;
    p.res->converged = 1;
    p.res->sweeps = 0;
    p.res->lam_max = n_lam > 0 ? lam[0] : 0.0;
    p.res->lam_min_kept = rank > 0 ? lam[rank - 1] : 0.0;
  }

  // ---- 3. eigenvectors of the kept eigenvalues --------------------------------
  for (int base = 0; base < rank; base += nw) {
    const int j = base + warp;
    double* z = p.zbuf + (size_t)warp * 6 * a;  // row: z (a) + LU factors (4a) + swap flags
    if (j < rank && lane == 0) {
      // inverse iteration on (T - lambda I): pivoted LU (dgttrf shape) factored
      // once, then 3 division-free solves (pivot reciprocals stored)
      const double lj = lam[j];
      const double eps_piv = 2.2e-16 * fmax(tnorm, 1e-300);
      double* fac = z + a;
      double* fri = fac;            // 1 / pivot
      double* fdu = fac + a;        // upper 1
      double* fdu2 = fac + 2 * a;   // upper 2
      double* fml = fac + 3 * a;    // multiplier; sign bit of swap encoded in fsw
      unsigned char* fsw = reinterpret_cast<unsigned char*>(fac + 4 * a);
      double dd_prev = d[0] - lj, du_prev = (a > 1) ? e[0] : 0.0;
      for (int i = 0; i + 1 < a; ++i) {
        const double sub = e[i];
        const double dnext = d[i + 1] - lj;
        const double unext = (i + 2 < a) ? e[i + 1] : 0.0;
        if (fabs(dd_prev) >= fabs(sub)) {
          double piv = dd_prev;
          if (fabs(piv) < eps_piv) piv = eps_piv;
          const double rp = 1.0 / piv;
          const double mult = sub * rp;
          fri[i] = rp; fdu[i] = du_prev; fdu2[i] = 0.0; fml[i] = mult; fsw[i] = 0;
          dd_prev = dnext - mult * du_prev;
          du_prev = unext;
        } else {
          const double rp = 1.0 / sub;
          const double mult = dd_prev * rp;
          fri[i] = rp; fdu[i] = dnext; fdu2[i] = unext; fml[i] = mult; fsw[i] = 1;
          dd_prev = du_prev - mult * dnext;
          du_prev = -mult * unext;
        }
      }
      double pivl = dd_prev;
      if (fabs(pivl) < eps_piv) pivl = eps_piv;
      fri[a - 1] = 1.0 / pivl;
      unsigned long long hs = 0x9E3779B97F4A7C15ull * (unsigned long long)(j + 1);
      for (int i = 0; i < a; ++i) {
        hs ^= hs >> 33; hs *= 0xff51afd7ed558ccdull; hs ^= hs >> 33;
        z[i] = 0.5 + (double)(hs >> 11) * (1.0 / 9007199254740992.0);
      }
      for (int iter = 0; iter < 3; ++iter) {
        for (int i = 0; i + 1 < a; ++i) {  // apply L^{-1} P
          if (fsw[i]) {
            const double zi = z[i];
            z[i] = z[i + 1];
            z[i + 1] = zi - fml[i] * z[i];
          } else {
            z[i + 1] -= fml[i] * z[i];
          }
        }
        z[a - 1] *= fri[a - 1];
        if (a >= 2) z[a - 2] = (z[a - 2] - fdu[a - 2] * z[a - 1]) * fri[a - 2];
        for (int i = a - 3; i >= 0; --i) z[i] = (z[i] - fdu[i] * z[i + 1] - fdu2[i] * z[i + 2]) * fri[i];
        double nn = 0.0;
        for (int i = 0; i < a; ++i) nn = fma(z[i], z[i], nn);
        const double inv = 1.0 / sqrt(nn);
        for (int i = 0; i < a; ++i) z[i] *= inv;
      }
    }
    __syncwarp();
    __syncthreads();
    // re-orthogonalise against earlier vectors of the same cluster (sequential, warp 0)
    if (warp == 0) {
      for (int jj = base + 1; jj < min(rank, base + nw); ++jj) {
        double* zj = p.zbuf + (size_t)(jj - base) * 6 * a;
        for (int kk = base; kk < jj; ++kk) {
          if (fabs(lam[kk] - lam[jj]) > 1e-3 * fmax(fabs(lam[0]), 1e-300)) continue;
          const double* zk = p.zbuf + (size_t)(kk - base) * 6 * a;
          double s = 0.0;
          for (int i = lane; i < a; i += 32) s = fma(zk[i], zj[i], s);
          s = warp_sum(s);
          for (int i = lane; i < a; i += 32) zj[i] -= s * zk[i];
          double nn = 0.0;
          for (int i = lane; i < a; i += 32) nn = fma(zj[i], zj[i], nn);
          nn = warp_sum(nn);
          const double inv = 1.0 / sqrt(nn);
          for (int i = lane; i < a; i += 32) zj[i] *= inv;
        }
      }
    }
    __syncthreads();
    if (j < rank) {
      // back-transform: u = H_0 ... H_{a-3} z ; H_k acts on rows k+1.. with v_k = [1; A[k+2.., k]]
      for (int k = a - 3; k >= 0; --k) {
        const double tk = tau[k];
        if (tk == 0.0) continue;
        const double* vk = A + (size_t)a * k;
        double s = (lane == 0) ? z[k + 1] : 0.0;
        for (int i = k + 2 + lane; i < a; i += 32) s = fma(vk[i], z[i], s);
        s = warp_sum(s) * tk;
        if (lane == 0) z[k + 1] -= s;
        for (int i = k + 2 + lane; i < a; i += 32) z[i] -= s * vk[i];
        __syncwarp();
      }
      // sign rule: largest |.| entry (first index) positive
      double best = -1.0;
      int bi = a;
      for (int i = lane; i < a; i += 32) {
        const double vv = fabs(z[i]);
        if (vv > best) { best = vv; bi = i; }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      const double sgn = (z[bi] < 0.0) ? -1.0 : 1.0;
      for (int i = lane; i < a; i += 32) p.UR[(size_t)j * a + i] = sgn * z[i];
    }
    __syncthreads();
  }
  if (tid == 0) {
    p.res->t_phase[0] = t1 - t0;
    p.res->t_phase[1] = t2 - t1;
    p.res->t_phase[2] = clock64() - t2;
    p.res->t_phase[3] = n_lam;
  }
}

}  // namespace ttg
