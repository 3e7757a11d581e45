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
#include "ttg_pdl.cuh"
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
  const double* tri;      // non-null: Ag already holds Q^T G Q's reflectors (k_sytrd_grid) and tri = [d | e | tau]
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
  griddep_wait();
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
  double trace = 0.0;
  if (p.tri) {  // tridiagonalised by k_sytrd_grid (multi-CTA): reflectors in Ag, d / e / tau given
    for (int i = tid; i < a; i += blockDim.x) {
      d[i] = p.tri[i];
      e[i] = p.tri[a + i];
      tau[i] = p.tri[2 * a + i];
    }
    for (int i = 0; i < a; ++i) trace += p.G[i + (size_t)a * i];  // all threads, same order
    __syncthreads();
  } else {
  for (long long i = tid; i < (long long)a * a; i += blockDim.x) A[i] = p.G[i];
  __syncthreads();
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
  }  // phase 1
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
    if (j < rank && p.tri) {  // multi-CTA back-transform and sign rule follow (k_syev_bt)
      for (int i = lane; i < a; i += 32) p.UR[(size_t)j * a + i] = z[i];
    } else if (j < rank) {
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

namespace ttg {

// ---------------------------------------------------------------------------
// Fast path for the common case "few kept directions": block subspace
// iteration with Rayleigh–Ritz on G (a x a, shared memory when it fits),
// block size kSubK.  The rank rule uses trace(G) - sum_{j<r} theta_j (Ritz
// values are lower bounds of the eigenvalues, so an unconverged estimate can
// only over-state the rank; convergence is certified by the Ritz residuals
// |G u_j - theta_j u_j| <= 64 eps theta_0 for every kept j and the next one).
// If that does not happen within kSubIters, or r >= kSubK - 1, res->converged
// = 0 and the host falls back to the full tridiagonal solver (k_syev).
// ---------------------------------------------------------------------------
constexpr int kSubK = 8;
constexpr int kSubIters = 40;
constexpr int kSubThreads = 256;

// One warp: cyclic Jacobi on the symmetric k x k (k <= N, N = 4 or 8) H held
// in registers (lane (N/2) i + m owns H[i][2m..2m+1] and W[i][2m..2m+1]); the
// N/2 disjoint round-robin pairs of a round are rotated together (rows, then
// columns of H, then columns of W) with shuffles only.  A rotation is skipped
// when |h_pq| <= 1e-15 sqrt(|h_pp h_qq|) or |h_pq| <= 4 eps max_i |h_ii| (at
// that size a rotation only reshuffles rounding noise: eigenvalues move by
// O(h_pq^2 / gap)); stops after a sweep without rotations.  Output: eigenvalues descending in
// theta[0..k), eigenvectors as the matching columns of Wv (k x k, ld k);
// Wt is an 8 x 8 shared scratch.
template <int N>
__device__ int warp_sym_eig(const double* Hs, int k, double* theta, double* Wv, double* Wt) {
  constexpr int NH = N / 2, NR = N - 1;
  const int lane = threadIdx.x & 31, i = lane / NH, m = lane % NH;
  const bool valid = i < N;
  const int j0 = 2 * m, j1 = 2 * m + 1;
  auto hsym = [&](int r, int c) { return (r < k && c < k) ? 0.5 * (Hs[r + k * c] + Hs[c + k * r]) : 0.0; };
  double h0 = hsym(i, j0), h1 = hsym(i, j1);
  double w0 = (i == j0) ? 1.0 : 0.0, w1 = (i == j1) ? 1.0 : 0.0;
  int sweep = 0;
  for (; sweep < 30; ++sweep) {
    double dg = ((i >> 1) == m) ? ((i & 1) ? h1 : h0) : 0.0;
    double hmax = fabs(dg);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) hmax = fmax(hmax, __shfl_xor_sync(0xffffffffu, hmax, o));
    const double floor_abs = 8.881784197001252e-16 * hmax;
    bool rotated = false;
    for (int rnd = 0; rnd < NR; ++rnd) {
      // round-robin positions: index 0 fixed at position 0, 1..7 rotate;
      // pairs are positions (u, 7-u), slot = min(u, 7-u)
      auto idx_at = [&](int u) { return u == 0 ? 0 : ((u - 1 + rnd) % NR) + 1; };
      auto pos_of = [&](int x) { return x == 0 ? 0 : ((x - 1 - rnd + NR) % NR) + 1; };
      auto partner = [&](int x) { return idx_at(NR - pos_of(x)); };
      auto slot_of = [&](int x) { const int u = pos_of(x); return u < NR - u ? u : NR - u; };
      const int pi = partner(i);
      dg = ((i >> 1) == m) ? ((i & 1) ? h1 : h0) : 0.0;
      const double mypq = ((pi >> 1) == m) ? ((pi & 1) ? h1 : h0) : 0.0;
      // lane evaluates the rotation of slot (lane & 3); lanes 0..3 publish it
      double cme = 1.0, sme = 0.0;
      int ame = 0;
      {
        int p = idx_at(m), q = idx_at(NR - m);
        if (p > q) { const int t = p; p = q; q = t; }
        const double hpp = __shfl_sync(0xffffffffu, dg, p * NH + (p >> 1));
        const double hqq = __shfl_sync(0xffffffffu, dg, q * NH + (q >> 1));
        const double hpq = __shfl_sync(0xffffffffu, mypq, p * NH + (q >> 1));
        if (q < k && fabs(hpq) > floor_abs && fabs(hpq) > 1e-15 * sqrt(fabs(hpp * hqq))) {
          const double zeta = (hqq - hpp) / (2.0 * hpq);
          const double az = fabs(zeta);
          const double t = az > 1e150 ? 0.5 / zeta : copysign(1.0, zeta) / (az + sqrt(fma(zeta, zeta, 1.0)));
          cme = rsqrt(fma(t, t, 1.0));
          sme = cme * t;
          ame = 1;
        }
      }
      rotated |= __any_sync(0xffffffffu, ame != 0);
      // rows p, q of H
      {
        const int sl = slot_of(i);
        const double c = __shfl_sync(0xffffffffu, cme, sl), sn = __shfl_sync(0xffffffffu, sme, sl);
        const bool act = __shfl_sync(0xffffffffu, ame, sl) != 0;
        const double o0 = __shfl_sync(0xffffffffu, h0, pi * NH + m);
        const double o1 = __shfl_sync(0xffffffffu, h1, pi * NH + m);
        if (act) {
          const bool isp = i < pi;
          h0 = isp ? c * h0 - sn * o0 : sn * o0 + c * h0;
          h1 = isp ? c * h1 - sn * o1 : sn * o1 + c * h1;
        }
      }
      // columns p, q of H and W
      {
        const int pj0 = partner(j0), pj1 = partner(j1);
        const int s0 = slot_of(j0), s1 = slot_of(j1);
        const double c0s = __shfl_sync(0xffffffffu, cme, s0), s0s = __shfl_sync(0xffffffffu, sme, s0);
        const double c1s = __shfl_sync(0xffffffffu, cme, s1), s1s = __shfl_sync(0xffffffffu, sme, s1);
        const bool a0s = __shfl_sync(0xffffffffu, ame, s0) != 0, a1s = __shfl_sync(0xffffffffu, ame, s1) != 0;
        const double a0 = __shfl_sync(0xffffffffu, h0, i * NH + (pj0 >> 1));
        const double a1 = __shfl_sync(0xffffffffu, h1, i * NH + (pj0 >> 1));
        const double b0 = __shfl_sync(0xffffffffu, h0, i * NH + (pj1 >> 1));
        const double b1 = __shfl_sync(0xffffffffu, h1, i * NH + (pj1 >> 1));
        const double c0 = __shfl_sync(0xffffffffu, w0, i * NH + (pj0 >> 1));
        const double c1 = __shfl_sync(0xffffffffu, w1, i * NH + (pj0 >> 1));
        const double d0 = __shfl_sync(0xffffffffu, w0, i * NH + (pj1 >> 1));
        const double d1 = __shfl_sync(0xffffffffu, w1, i * NH + (pj1 >> 1));
        const double hx0 = (pj0 & 1) ? a1 : a0, hx1 = (pj1 & 1) ? b1 : b0;
        const double wx0 = (pj0 & 1) ? c1 : c0, wx1 = (pj1 & 1) ? d1 : d0;
        if (a0s) {
          const bool isp = j0 < pj0;
          h0 = isp ? c0s * h0 - s0s * hx0 : s0s * hx0 + c0s * h0;
          w0 = isp ? c0s * w0 - s0s * wx0 : s0s * wx0 + c0s * w0;
        }
        if (a1s) {
          const bool isp = j1 < pj1;
          h1 = isp ? c1s * h1 - s1s * hx1 : s1s * hx1 + c1s * h1;
          w1 = isp ? c1s * w1 - s1s * wx1 : s1s * wx1 + c1s * w1;
        }
      }
    }
    if (!__any_sync(0xffffffffu, rotated)) break;
  }
  // eigenvalues (diagonal) and W into scratch, then a stable descending sort
  if (valid) {
    Wt[i + 8 * j0] = w0;
    Wt[i + 8 * j1] = w1;
    if ((i >> 1) == m) Wt[64 + i] = (i & 1) ? h1 : h0;
  }
  __syncwarp();
  if (lane < k) {
    const double tx = Wt[64 + lane];
    int pos = 0;
    for (int y = 0; y < k; ++y) {
      const double ty = Wt[64 + y];
      pos += (ty > tx || (ty == tx && y < lane)) ? 1 : 0;
    }
    theta[pos] = tx;
    for (int r = 0; r < k; ++r) Wv[r + k * pos] = Wt[r + 8 * lane];
  }
  __syncwarp();
  return sweep;
}

// One thread: cyclic Jacobi on the symmetric k x k (k <= 4) Hs held in
// registers (same rotation formula and skip thresholds as warp_sym_eig; the
// k = 4 Rayleigh-Ritz problem is latency-bound, and one thread avoids the
// shuffle chains of the warp version).  Output as warp_sym_eig.
// Rotation (c, s) zeroing h_pq of the 2 x 2 block [[hpp, hpq], [hpq, hqq]]:
// t = sign(d) e / (|d| + sqrt(d^2 + e^2)) with d = hqq - hpp, e = 2 hpq (the
// tan of the smaller angle, one division and one square root), c = 1/sqrt(1+t^2).
// Same skip rule as warp_sym_eig (|h_pq| <= 1e-15 sqrt|h_pp h_qq| or <= the
// absolute floor), tested on squares.  Returns false (c = 1, s = 0) if skipped.
__device__ __forceinline__ bool jacobi_rot(double hpp, double hqq, double hpq, double floor_abs, bool active,
                                           double& c, double& sn) {
  c = 1.0;
  sn = 0.0;
  if (!active || !(fabs(hpq) > floor_abs) || !(hpq * hpq > 1e-30 * fabs(hpp * hqq))) return false;
  double dd = hqq - hpp, e = 2.0 * hpq;
  const double m = fmax(fabs(dd), fabs(e));
  if (m > 1e150) {  // exact power-of-two rescale keeps d^2 + e^2 finite
    dd *= 0x1p-600;
    e *= 0x1p-600;
  }
  const double t = copysign(1.0, dd) * e / (fabs(dd) + sqrt(fma(dd, dd, e * e)));
  c = rsqrt(fma(t, t, 1.0));
  sn = c * t;
  return true;
}

// One thread: Jacobi on the symmetric k x k (k <= 4) Hs held in registers,
// round-robin order: each round rotates two disjoint pairs, (0,1)(2,3),
// (0,2)(1,3), (0,3)(1,2), whose angles depend only on their own 2 x 2 blocks,
// so the two rotation chains run side by side (the k = 4 Rayleigh-Ritz problem
// is latency-bound).  Stops after a sweep without rotations.  Output as
// warp_sym_eig.
__device__ int thread_sym_eig4(const double* Hs, int k, double* theta, double* Wv) {
  double h[4][4], w[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      h[i][j] = (i < k && j < k) ? 0.5 * (Hs[i + k * j] + Hs[j + k * i]) : 0.0;
      w[i][j] = (i == j) ? 1.0 : 0.0;
    }
  int sweep = 0;
  for (; sweep < 30; ++sweep) {
    double hmax = 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i) hmax = fmax(hmax, fabs(h[i][i]));
    const double floor_abs = 8.881784197001252e-16 * hmax;
    bool rotated = false;
#pragma unroll
    for (int rd = 0; rd < 3; ++rd) {
      const int p1 = 0, q1 = rd + 1;                       // (0,1) (0,2) (0,3)
      const int p2 = rd == 0 ? 2 : 1, q2 = rd == 2 ? 2 : 3;  // (2,3) (1,3) (1,2)
      double c1, s1, c2, s2;
      const bool r1 = jacobi_rot(h[p1][p1], h[q1][q1], h[p1][q1], floor_abs, q1 < k, c1, s1);
      const bool r2 = jacobi_rot(h[p2][p2], h[q2][q2], h[p2][q2], floor_abs, q2 < k, c2, s2);
      if (!(r1 || r2)) continue;
      rotated = true;
#pragma unroll
      for (int j = 0; j < 4; ++j) {  // rows p, q of both pairs
        const double x1 = h[p1][j], y1 = h[q1][j], x2 = h[p2][j], y2 = h[q2][j];
        h[p1][j] = c1 * x1 - s1 * y1;
        h[q1][j] = s1 * x1 + c1 * y1;
        h[p2][j] = c2 * x2 - s2 * y2;
        h[q2][j] = s2 * x2 + c2 * y2;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {  // columns p, q of H and W
        const double x1 = h[i][p1], y1 = h[i][q1], x2 = h[i][p2], y2 = h[i][q2];
        h[i][p1] = c1 * x1 - s1 * y1;
        h[i][q1] = s1 * x1 + c1 * y1;
        h[i][p2] = c2 * x2 - s2 * y2;
        h[i][q2] = s2 * x2 + c2 * y2;
        const double u1 = w[i][p1], v1 = w[i][q1], u2 = w[i][p2], v2 = w[i][q2];
        w[i][p1] = c1 * u1 - s1 * v1;
        w[i][q1] = s1 * u1 + c1 * v1;
        w[i][p2] = c2 * u2 - s2 * v2;
        w[i][q2] = s2 * u2 + c2 * v2;
      }
    }
    if (!rotated) break;
  }
  // stable descending sort of the diagonal
  double d[4];
  int pos[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) d[i] = h[i][i];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int ps = 0;
#pragma unroll
    for (int y = 0; y < 4; ++y)
      if (y < k) ps += (d[y] > d[i] || (d[y] == d[i] && y < i)) ? 1 : 0;
    pos[i] = ps;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (i < k) {
      theta[pos[i]] = d[i];
#pragma unroll
      for (int r = 0; r < 4; ++r)
        if (r < k) Wv[r + k * pos[i]] = w[r][i];
    }
  return sweep;
}

// block_cholqr2 for k <= 4 with the k x k Cholesky in one thread's registers
// (fewer barriers / warp-serial steps; same column-scaled CholQR2 numerics)
__device__ void block_cholqr2_4(double* X, int a, int k, double* S, double* Ri) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  for (int pass = 0; pass < 2; ++pass) {
    for (int e = warp; e < 16; e += nw) {
      const int i = e & 3, j = e >> 2;
      if (i > j || j >= k) continue;
      double s0 = 0.0, s1 = 0.0;
      int r = lane;
      for (; r + 32 < a; r += 64) {
        s0 = fma(X[r + (size_t)a * i], X[r + (size_t)a * j], s0);
        s1 = fma(X[r + 32 + (size_t)a * i], X[r + 32 + (size_t)a * j], s1);
      }
      if (r < a) s0 = fma(X[r + (size_t)a * i], X[r + (size_t)a * j], s0);
      const double sacc = warp_sum(s0 + s1);
      if (lane == 0) S[i + 4 * j] = sacc;
    }
    __syncthreads();
    if (tid == 0) {
      double m[4][4], dsc[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) dsc[i] = (i < k && S[i + 4 * i] > 0.0) ? 1.0 / sqrt(S[i + 4 * i]) : 0.0;
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) m[i][j] = (i <= j && j < k) ? S[i + 4 * j] * dsc[i] * dsc[j] : 0.0;
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        if (jj < k) {
          const double piv = m[jj][jj];
          const double rjj = piv > 1e-28 ? sqrt(piv) : 0.0;
          const double inv = rjj > 0.0 ? 1.0 / rjj : 0.0;
          Ri[4 + jj] = inv;
#pragma unroll
          for (int l = 0; l < 4; ++l)
            if (l >= jj) m[jj][l] = (l == jj) ? rjj : m[jj][l] * inv;
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int l = 0; l < 4; ++l)
              if (i > jj && i <= l) m[i][l] -= m[jj][i] * m[jj][l];
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        Ri[i] = dsc[i];
#pragma unroll
        for (int j = 0; j < 4; ++j) S[i + 4 * j] = m[i][j];
      }
    }
    __syncthreads();
    for (int r = tid; r < a; r += blockDim.x) {
      double v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (j < k) {
          double t = X[r + (size_t)a * j] * Ri[j];
#pragma unroll
          for (int mm = 0; mm < 4; ++mm)
            if (mm < j) t -= v[mm] * S[mm + 4 * j];
          v[j] = t * Ri[4 + j];
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (j < k) X[r + (size_t)a * j] = v[j];
    }
    __syncthreads();
  }
}

// Orthonormalise the k (<= kSubK) columns of X (a x k, ld a) in place:
// column-scaled Cholesky QR, twice (X D R^-1 with D = diag(X^T X)^-1/2, so the
// Gram matrix factored is unit-diagonal and CholQR2 is stable up to
// cond ~ 1e8).  Exactly dependent / zero columns come out as zero columns.
// Y is an a x k scratch; S, Ri are k x k shared scratch.  Ends after a barrier.
template <int K>
__device__ void block_cholqr2(double* X, double* Y, int a, int k, double* S, double* Ri) {
  (void)Y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  for (int pass = 0; pass < 2; ++pass) {
    for (int e = warp; e < k * k; e += nw) {
      const int i = e % k, j = e / k;
      if (i > j) continue;
      double sacc = 0.0;
      for (int r = lane; r < a; r += 32) sacc = fma(X[r + (size_t)a * i], X[r + (size_t)a * j], sacc);
      sacc = warp_sum(sacc);
      if (lane == 0) S[i + k * j] = sacc;
    }
    __syncthreads();
    if (warp == 0) {
      // Ri[0..k) = D = diag(S)^-1/2; S <- D S D (upper); right-looking Cholesky
      // in place: R (upper) overwrites S.  Lane e owns upper entries e, e+32.
      if (lane < k) Ri[lane] = S[lane + k * lane] > 0.0 ? 1.0 / sqrt(S[lane + k * lane]) : 0.0;
      __syncwarp();
      for (int e = lane; e < k * k; e += 32) {
        const int i = e % k, j = e / k;
        if (i <= j) S[e] *= Ri[i] * Ri[j];
      }
      __syncwarp();
      for (int jj = 0; jj < k; ++jj) {
        const double piv = S[jj + k * jj];
        const double rjj = piv > 1e-28 ? sqrt(piv) : 0.0;
        const double inv = rjj > 0.0 ? 1.0 / rjj : 0.0;
        __syncwarp();
        if (lane == 0) Ri[K + jj] = inv;
        // row jj of R
        for (int l = jj + lane; l < k; l += 32) S[jj + k * l] = (l == jj) ? rjj : S[jj + k * l] * inv;
        __syncwarp();
        // trailing update S[i][l] -= R[jj][i] R[jj][l], jj < i <= l
        for (int e = lane; e < k * k; e += 32) {
          const int i = e % k, l = e / k;
          if (i > jj && i <= l) S[e] -= S[jj + k * i] * S[jj + k * l];
        }
        __syncwarp();
      }
    }
    __syncthreads();
    // X <- X D R^-1, row by row (forward substitution on the row vector)
    for (int r = tid; r < a; r += blockDim.x) {
      double v[K];
#pragma unroll
      for (int j = 0; j < K; ++j) {
        if (j < k) {
          double t = X[r + (size_t)a * j] * Ri[j];
#pragma unroll
          for (int m = 0; m < K; ++m)
            if (m < j) t -= v[m] * S[m + k * j];
          v[j] = t * Ri[K + j];
        }
      }
#pragma unroll
      for (int j = 0; j < K; ++j)
        if (j < k) X[r + (size_t)a * j] = v[j];
    }
    __syncthreads();
  }
}

template <int K>
__global__ void __launch_bounds__(kSubThreads, 1) k_syev_top(SyevArgs p) {
  griddep_wait();
  extern __shared__ __align__(16) double sm[];
  __shared__ double red[64];
  __shared__ double H[(K < 4 ? 4 : K) * (K < 4 ? 4 : K)], Wv[(K < 4 ? 4 : K) * (K < 4 ? 4 : K)], theta[K < 4 ? 4 : K],
      resn[K < 4 ? 4 : K];
  constexpr int KS = K < 4 ? 4 : K;  // block_cholqr2_4 / thread_sym_eig4 work on 4 x 4 scratch
  __shared__ double Sq[KS * KS], Rq[2 * KS], Wt[72];
  __shared__ int s_state, s_rank;
  __shared__ double s_tail;
  const long long t0 = clock64();
  const int a = p.a;
  const int k = a < K ? a : K;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  // in_smem: 1 = G in shared memory, 2 = its lower triangle packed in shared
  // memory (a <= ~220: the full square does not fit, the triangle does),
  // 0 = G read from L2
  const bool packed = p.in_smem == 2;
  const size_t gsz = packed ? (((size_t)a * (a + 1) / 2 + 1) & ~(size_t)1) : (size_t)a * a;
  double* G = p.in_smem ? sm : const_cast<double*>(p.G);
  double* X = p.in_smem ? sm + gsz : sm;
  double* Z = X + (size_t)a * K;
  auto gat = [&](int i, int j) -> double {  // G[i][j]
    if (packed) {
      const int hi = i > j ? i : j, lo = i > j ? j : i;
      return G[(size_t)hi * (hi + 1) / 2 + lo];
    }
    return G[i + (size_t)a * j];
  };
  if (packed) {
    for (long long e = tid; e < (long long)a * a; e += blockDim.x) {
      const int i = (int)(e % a), j = (int)(e / a);
      if (i >= j) G[(size_t)i * (i + 1) / 2 + j] = __ldg(p.G + e);
    }
  } else if (p.in_smem) {  // a*a is even or odd: copy pairs, then the odd tail
    const long long n = (long long)a * a, n2 = n >> 1;
    const double2* src = reinterpret_cast<const double2*>(p.G);
    double2* dst = reinterpret_cast<double2*>(G);
#pragma unroll 8
    for (long long i = tid; i < n2; i += blockDim.x) dst[i] = __ldg(src + i);
    if ((n & 1) && tid == 0) G[n - 1] = p.G[n - 1];
  }
  const long long ts1 = clock64();
  // deterministic pseudo-random orthonormal start block: k columns of the
  // Householder reflector I - 2 v v^T / v^T v (v pseudo-random), at pivots
  // spread over the rows -- orthonormal by construction, so no initial QR
  __syncthreads();  // G staged
  double vpart = 0.0, gpart = 0.0;
  for (int i = tid; i < a; i += blockDim.x) {
    unsigned long long h = 0x9E3779B97F4A7C15ull * (unsigned long long)(i + 1);
    h ^= h >> 31; h *= 0xbf58476d1ce4e5b9ull; h ^= h >> 27;
    const double vi = (double)(h >> 11) * (1.0 / 9007199254740992.0) - 0.5;
    Z[i] = vi;
    vpart = fma(vi, vi, vpart);
    gpart += gat(i, i);
  }
  const double vv = block_sum_all(vpart, red);
  __syncthreads();
  const double trace = block_sum_all(gpart, red);  // fixed order: identical on every thread
  for (int e = tid; e < a * k; e += blockDim.x) {
    const int i = e % a, c = e / a;
    const int piv = (int)(((long long)c * a) / k);
    X[e] = (i == piv ? 1.0 : 0.0) - 2.0 * Z[i] * (Z[piv] / vv);
  }
  __syncthreads();
  const double delta = p.delta_src ? p.delta_mult * sqrt(*p.delta_src) : p.delta_mult;
  const long long kcap = p.kmax < a ? p.kmax : a;
  if (tid == 0) { s_state = 0; s_rank = 0; s_tail = trace; }
  if (!(sqrt(fmax(trace, 0.0)) > delta) || kcap == 0) {  // everything fits under delta: rank 0
    if (tid == 0) {
      p.res->rank = 0; p.res->tail_sq = fmax(trace, 0.0); p.res->delta = delta; p.res->converged = 1;
      p.res->sweeps = 0; p.res->lam_max = 0.0; p.res->lam_min_kept = 0.0;
    }
    return;
  }
  const long long ts2 = clock64();
  const long long t1 = clock64();
  double prev_res = 1e300;
  long long ph[4] = {0, 0, 0, 0};
  int jac_sweeps = 0;
  int it = 0;
  for (; it < kSubIters; ++it) {
    long long tq0 = clock64();
    // Z = G X on DMMA m8n8k4: warp task = one 8-row block of Z (all K <= 8
    // columns at once, X padded to 8 columns by predicated zeros); two
    // accumulator chains over the even / odd k-steps.  G in shared memory or
    // L2 (a lane reads G[i0 + g][k0 + t]: 8 contiguous rows x 4 columns).
    {
      const int g = lane >> 2, t = lane & 3;
      const int nrb = (a + 7) >> 3;
      for (int rb = warp; rb < nrb; rb += nw) {
        const int i = rb * 8 + g;
        double c0 = 0.0, c1 = 0.0, e0 = 0.0, e1 = 0.0;
        int k0 = 0;
#pragma unroll 4
        for (; k0 + 8 <= a; k0 += 8) {
          const double ga = i < a ? gat(i, k0 + t) : 0.0;
          const double gb = i < a ? gat(i, k0 + 4 + t) : 0.0;
          const double xa = g < k ? X[(k0 + t) + (size_t)a * g] : 0.0;
          const double xb = g < k ? X[(k0 + 4 + t) + (size_t)a * g] : 0.0;
          dmma(c0, c1, ga, xa);
          dmma(e0, e1, gb, xb);
        }
        for (; k0 < a; k0 += 4) {
          const bool kv = k0 + t < a;
          const double ga = (i < a && kv) ? gat(i, k0 + t) : 0.0;
          const double xa = (g < k && kv) ? X[(k0 + t) + (size_t)a * g] : 0.0;
          dmma(c0, c1, ga, xa);
        }
        c0 += e0;
        c1 += e1;
        if (i < a) {
          if (2 * t < k) Z[i + (size_t)a * (2 * t)] = c0;
          if (2 * t + 1 < k) Z[i + (size_t)a * (2 * t + 1)] = c1;
        }
      }
    }
    __syncthreads();
    long long tq1 = clock64();
    // H = X^T Z (k x k), symmetrised
    for (int e = warp; e < k * k; e += nw) {
      const int i = e % k, j = e / k;
      double s = 0.0;
      for (int r = lane; r < a; r += 32) s = fma(X[r + (size_t)a * i], Z[r + (size_t)a * j], s);
      s = warp_sum(s);
      if (lane == 0) H[e] = s;
    }
    __syncthreads();
    long long tq2 = clock64();
    if constexpr (K <= 4) {
      if (tid == 0) jac_sweeps += thread_sym_eig4(H, k, theta, Wv);
    } else if (warp == 0) {
      const int nsw = warp_sym_eig<K>(H, k, theta, Wv, Wt);
      if (lane == 0) jac_sweeps += nsw;
    }
    __syncthreads();
    long long tq3 = clock64();
    // residuals |Z w_j - theta_j X w_j|
    for (int j = warp; j < k; j += nw) {
      double s = 0.0;
      for (int r = lane; r < a; r += 32) {
        double zw = 0.0, xw = 0.0;
        for (int c = 0; c < k; ++c) {
          zw = fma(Z[r + (size_t)a * c], Wv[c + k * j], zw);
          xw = fma(X[r + (size_t)a * c], Wv[c + k * j], xw);
        }
        const double d = zw - theta[j] * xw;
        s = fma(d, d, s);
      }
      s = warp_sum(s);
      if (lane == 0) resn[j] = sqrt(s);
    }
    __syncthreads();
    if (tid == 0) {
      // rank from the Ritz values (lower bounds => rank can only be over-stated)
      double pre = 0.0;
      int r = -1;
      for (int q = 0; q <= k; ++q) {
        if (q <= kcap && !(sqrt(fmax(trace - pre, 0.0)) > delta)) { r = q; break; }
        if (q < k) pre += fmax(theta[q], 0.0);
      }
      const double tol = 64.0 * 2.220446049250313e-16 * fmax(theta[0], 1e-300);
      double worst = 0.0;
      if (r >= 1 && r < k) {
        // only the kept Ritz pairs enter the tail and U_R: certify those
        for (int q = 0; q < r; ++q) worst = fmax(worst, resn[q]);
        if (worst <= tol || (worst <= 1e-12 * theta[0] && worst >= 0.9 * prev_res)) {
          double pre2 = 0.0;
          for (int q = 0; q < r; ++q) pre2 += theta[q];
          s_rank = r;
          s_tail = fmax(trace - pre2, 0.0);
          s_state = 1;  // converged
        }
      } else {
        worst = resn[0];
        if (it >= 3) s_state = 2;  // more kept directions than the block holds: larger block / full solver
      }
      prev_res = worst;
      red[63] = worst;
    }
    __syncthreads();
    if (tid == 0) {
      const long long tq4 = clock64();
      p.res->t_phase[2] += 0;  // keep
      ph[0] += tq1 - tq0; ph[1] += tq2 - tq1; ph[2] += tq3 - tq2; ph[3] += tq4 - tq3;
    }
    if (s_state) break;
    prev_res = red[63];
    // next block: X = orth(Z W)   (Ritz-rotated power step)
    for (int e = tid; e < a * k; e += blockDim.x) {
      const int i = e % a, j = e / a;
      double s = 0.0;
      for (int c = 0; c < k; ++c) s = fma(Z[i + (size_t)a * c], Wv[c + k * j], s);
      X[e] = s;
    }
    __syncthreads();
    if constexpr (K <= 4) block_cholqr2_4(X, a, k, Sq, Rq);
    else block_cholqr2<K>(X, Z, a, k, Sq, Rq);
  }
  const int rank = s_rank;
  if (tid == 0) {
    p.res->t_phase[0] = (ts1 - t0) | ((ts2 - ts1) << 20) | ((t1 - ts2) << 40);
    p.res->t_phase[1] = (clock64() - t1) | ((long long)jac_sweeps << 40);
    p.res->t_phase[2] = ph[0] | (ph[1] << 32);
    p.res->t_phase[3] = ph[2] | (ph[3] << 32);
    p.res->converged = (s_state == 1) ? 1 : 0;
    p.res->sweeps = it;
    p.res->rank = rank;
    p.res->tail_sq = s_tail;
    p.res->delta = delta;
    p.res->lam_max = theta[0];
    p.res->lam_min_kept = rank > 0 ? theta[rank - 1] : 0.0;
  }
  if (s_state != 1) return;
  for (int j = tid; j < k; j += blockDim.x) p.lam[j] = theta[j];
  // U_R = X W[:, :rank], normalised, sign rule
  for (int j = warp; j < rank; j += nw) {
    double* out = p.UR + (size_t)a * j;
    double nn = 0.0, best = -1.0;
    int bi = a;
    for (int r = lane; r < a; r += 32) {
      double u = 0.0;
      for (int c = 0; c < k; ++c) u = fma(X[r + (size_t)a * c], Wv[c + k * j], u);
      out[r] = u;
      nn = fma(u, u, nn);
    }
    nn = warp_sum(nn);
    const double inv = 1.0 / sqrt(nn);
    for (int r = lane; r < a; r += 32) {
      const double v = fabs(out[r]);
      if (v > best) { best = v; bi = r; }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    const double sgn = (out[bi] < 0.0) ? -inv : inv;
    __syncwarp();
    for (int r = lane; r < a; r += 32) out[r] *= sgn;
  }
}


}  // namespace ttg

namespace ttg {

// ---------------------------------------------------------------------------
// Multi-CTA Householder tridiagonalisation Q^T G Q = T for the large Grams
// (a > ~160) that do not fit one CTA's shared memory and keep too many
// directions for the block subspace path (replaces cuSOLVER syevd).  LAPACK
// dsytd2 'L' numerics with dlatrd's lazy panel update, on P co-resident CTAs
// (cooperative launch, one grid barrier per column).  Every CTA holds the
// whole current panel V, W (a x nb) in shared memory -- each computes every
// v and w itself, from identical inputs in the same order, so the copies are
// bitwise identical and no panel traffic crosses the grid:
//   A  step j (panel column jj): the updated column
//      a_j = A[:, j] - V W[j,:]^T - W V[j,:]^T (q < jj) and its reflector v;
//   B  this CTA's rows of p = (A - V W^T - W V^T) v (row i = column i of the
//      symmetric storage: contiguous reads), then the grid barrier;
//   C  w = tau p - tau/2 (tau p^T v) v from the gathered p, appended to W;
//   D  panel end: A_trailing -= V W^T + W V^T (both triangles), then a barrier.
// Output: d, e, tau (tri = [d | e | tau]) and the reflectors' essential parts
// in A's columns below the subdiagonal -- the layout of k_syev phases 2-3.
// ---------------------------------------------------------------------------
constexpr int kTrdThreads = 512;

struct TrdArgs {
  double* A;        // a x a (copy of G), overwritten
  int a;
  int nb;           // panel width (shared memory: (3 + 2 nb) a doubles)
  double* pbuf;     // a
  double* tri;      // 3a: d, e, tau
  unsigned* bar;    // [count, generation], zeroed by the host
};

__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* vgen = bar + 1;
    const unsigned gen = *vgen;
    __threadfence();
    if (atomicAdd(bar, 1u) == nblocks - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*vgen == gen) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kTrdThreads) k_sytrd_grid(TrdArgs p) {
  griddep_wait();  // launched cooperatively without PDL: a no-op, kept for the invariant
  extern __shared__ __align__(16) double tsm[];
  __shared__ double red[kTrdThreads / 32 + 1];
  __shared__ double vtw[2 * 64];
  const int a = p.a, nb = p.nb, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const unsigned P = gridDim.x;
  double* A = p.A;
  double* col = tsm;          // updated column j
  double* v = col + a;        // reflector of step j (zero above j + 1)
  double* pv = v + a;         // tau p of step j
  double* Vs = pv + a;        // panel V (a x nb)
  double* Ws = Vs + (size_t)a * nb;  // panel W (a x nb)
  const int rows_per = (a + (int)P - 1) / (int)P;
  const int r0 = (int)blockIdx.x * rows_per, r1 = min(a, r0 + rows_per);
  // A warp owns one row i_w of p when rows_per <= warps (the usual case): its
  // row (= column i_w, symmetric storage) is cached in registers for a whole
  // panel (the panel's updates are lazy; the column changes only at step D).
  constexpr int QC = 32;
  const int iw = r0 + warp;
  const bool own = rows_per <= nw && iw < r1;
  double creg[QC];
  constexpr int QA = 8;  // column j + 1 prefetched for step A (a <= 8 * kTrdThreads)
  double pre[QA];
  bool have_pre = false;
  for (int j0 = 0; j0 + 2 < a; j0 += nb) {
    const int jend = min(j0 + nb, a - 2);  // columns j0 .. jend-1 in this panel
    const bool cached = own && a - (j0 + 1) <= 32 * QC;
    if (cached) {
#pragma unroll
      for (int q = 0; q < QC; ++q) {
        const int k = j0 + 1 + lane + 32 * q;
        creg[q] = k < a ? A[k + (size_t)a * iw] : 0.0;
      }
    }
    for (int j = j0; j < jend; ++j) {
      const int jj = j - j0;
      // ---- A: updated column j and its reflector (every CTA) ----
#pragma unroll
      for (int q = 0; q < QA; ++q) {
        const int i = j + tid + q * (int)blockDim.x;
        if (i < a) {
          double x = have_pre ? pre[q] : A[i + (size_t)a * j];
          for (int qq = 0; qq < jj; ++qq)
            x -= Vs[i + (size_t)a * qq] * Ws[j + (size_t)a * qq] + Ws[i + (size_t)a * qq] * Vs[j + (size_t)a * qq];
          col[i] = x;
        }
      }
      __syncthreads();
      double xs = 0.0;
      for (int i = j + 2 + tid; i < a; i += blockDim.x) xs = fma(col[i], col[i], xs);
      xs = block_sum_all(xs, red);
      const double alpha = col[j + 1];
      double tk = 0.0, beta = alpha;
      if (xs != 0.0) {
        beta = sqrt(alpha * alpha + xs);
        if (alpha >= 0.0) beta = -beta;
        tk = (beta - alpha) / beta;
      }
      const double sc = xs != 0.0 ? 1.0 / (alpha - beta) : 0.0;
      for (int i = tid; i < a; i += blockDim.x) v[i] = (i <= j) ? 0.0 : (i == j + 1 ? 1.0 : col[i] * sc);
      if (blockIdx.x == 0 && tid == 0) {
        p.tri[j] = col[j];
        p.tri[a + j] = beta;
        p.tri[2 * a + j] = tk;
      }
      __syncthreads();
      // ---- B: W^T v, V^T v (q < jj), then this CTA's rows of p ----
      for (int q = warp; q < 2 * jj; q += nw) {
        const double* m = (q < jj ? Ws : Vs) + (size_t)a * (q % jj);
        double s = 0.0;
        for (int i = j + 1 + lane; i < a; i += 32) s = fma(m[i], v[i], s);
        s = warp_sum(s);
        if (lane == 0) vtw[q] = s;
      }
      __syncthreads();
      if (cached) {
        if (iw >= j + 1) {
          double s = 0.0;  // v is zero above row j + 1, so the cached rows <= j drop out
#pragma unroll
          for (int q = 0; q < QC; ++q) {
            const int k = j0 + 1 + lane + 32 * q;
            if (k < a) s = fma(creg[q], v[k], s);
          }
          s = warp_sum(s);
          if (lane == 0) {
            for (int q = 0; q < jj; ++q) s -= Vs[iw + (size_t)a * q] * vtw[q] + Ws[iw + (size_t)a * q] * vtw[jj + q];
            p.pbuf[iw] = s;
          }
        }
      } else {
        for (int i = max(r0, j + 1) + warp; i < r1; i += nw) {
          const double* ci = A + (size_t)a * i;
          double s = 0.0;
          for (int k = j + 1 + lane; k < a; k += 32) s = fma(ci[k], v[k], s);
          s = warp_sum(s);
          if (lane == 0) {
            for (int q = 0; q < jj; ++q) s -= Vs[i + (size_t)a * q] * vtw[q] + Ws[i + (size_t)a * q] * vtw[jj + q];
            p.pbuf[i] = s;
          }
        }
      }
      grid_barrier(p.bar, P);
      // prefetch column j + 1 for the next step A (unchanged until step D)
      have_pre = j + 1 < jend && a <= QA * (int)blockDim.x;
      if (have_pre) {
#pragma unroll
        for (int q = 0; q < QA; ++q) {
          const int i = j + 1 + tid + q * (int)blockDim.x;
          pre[q] = i < a ? A[i + (size_t)a * (j + 1)] : 0.0;
        }
      }
      // every CTA has read column j (step A): store the reflector in it
      if (blockIdx.x == 0)
        for (int i = j + 2 + tid; i < a; i += blockDim.x) A[i + (size_t)a * j] = v[i];
      // ---- C: w = tau p + alpha2 v (every CTA, full length) -> panel ----
      double pvs = 0.0;
      for (int i = j + 1 + tid; i < a; i += blockDim.x) {
        const double w0 = tk * __ldcg(p.pbuf + i);
        pv[i] = w0;
        pvs = fma(w0, v[i], pvs);
      }
      pvs = block_sum_all(pvs, red);
      const double al2 = -0.5 * tk * pvs;
      for (int i = tid; i < a; i += blockDim.x) {
        Ws[i + (size_t)a * jj] = (i <= j) ? 0.0 : fma(al2, v[i], pv[i]);
        Vs[i + (size_t)a * jj] = v[i];
      }
      __syncthreads();
    }
    // ---- D: trailing update of both triangles, rows / columns >= jend ----
    // (every CTA finished step B of the panel's last column at its barrier;
    // nothing reads A between there and here)
    const int np = jend - j0;
    const int m = a - jend;
    const long long tot = (long long)m * m;
    for (long long e = blockIdx.x * (long long)blockDim.x + tid; e < tot; e += (long long)P * blockDim.x) {
      const int i = jend + (int)(e % m), k = jend + (int)(e / m);
      double x = A[i + (size_t)a * k];
      for (int q = 0; q < np; ++q)
        x -= Vs[i + (size_t)a * q] * Ws[k + (size_t)a * q] + Ws[i + (size_t)a * q] * Vs[k + (size_t)a * q];
      A[i + (size_t)a * k] = x;
    }
    grid_barrier(p.bar, P);
    have_pre = false;
  }
  // last 2 x 2 block (k_syev's tail convention)
  if (blockIdx.x == 0 && tid == 0) {
    if (a >= 2) {
      p.tri[a - 2] = A[(a - 2) + (size_t)a * (a - 2)];
      p.tri[a + a - 2] = A[(a - 1) + (size_t)a * (a - 2)];
      p.tri[2 * a + a - 2] = 0.0;
    }
    p.tri[a - 1] = A[(a - 1) + (size_t)a * (a - 1)];
    p.tri[a + a - 1] = 0.0;
    p.tri[2 * a + a - 1] = 0.0;
  }
}

// Back-transform of the kept eigenvectors of T (k_syev in tri mode leaves the
// inverse-iteration vectors z in UR): u = H_0 ... H_{a-3} z with the reflectors
// of k_sytrd_grid (v_k = [1; A[k+2.., k]]), then the sign rule (largest-|.|
// entry, first index, positive: truncated_svd.cpp:16-25).  One CTA applies
// every reflector to VB vectors at once (each reflector read from L2 once per
// VB vectors, the next one prefetched into registers while the current dot
// products reduce); the rank is read from the eigen result.
constexpr int kBtThreads = 256;
template <int VB>
__global__ void __launch_bounds__(kBtThreads) k_syev_bt(const double* __restrict__ A, int a,
                                                         const double* __restrict__ tau, const EigResult* res,
                                                         double* __restrict__ UR) {
  griddep_wait();
  extern __shared__ __align__(16) double bsm[];
  __shared__ double red[VB][kBtThreads / 32];
  __shared__ double sv[VB];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = kBtThreads / 32;
  const int rank = res->rank;
  const int j0 = blockIdx.x * VB;
  if (j0 >= rank) return;
  const int nv = min(VB, rank - j0);
  double* z = bsm;  // VB x a
  for (int v = 0; v < nv; ++v)
    for (int i = tid; i < a; i += kBtThreads) z[(size_t)v * a + i] = UR[(size_t)(j0 + v) * a + i];
  __syncthreads();
  constexpr int PR = 16;  // prefetched reflector entries per thread (a <= 16 * 256 + 2)
  double cur[PR];
  auto fetch = [&](int k, double (&dst)[PR]) {
#pragma unroll
    for (int q = 0; q < PR; ++q) {
      const int i = k + 2 + tid + q * kBtThreads;
      dst[q] = (k >= 0 && i < a) ? A[(size_t)a * k + i] : 0.0;
    }
  };
  fetch(a - 3, cur);
  for (int k = a - 3; k >= 0; --k) {
    double nxt[PR];
    fetch(k - 1, nxt);  // next reflector in flight while this one reduces
    const double tk = tau[k];
    if (tk != 0.0) {
      double s[VB];
#pragma unroll
      for (int v = 0; v < VB; ++v) {
        s[v] = 0.0;
        if (v < nv) {
          const double* zv = z + (size_t)v * a;
#pragma unroll
          for (int q = 0; q < PR; ++q) {
            const int i = k + 2 + tid + q * kBtThreads;
            if (i < a) s[v] = fma(cur[q], zv[i], s[v]);
          }
          if (tid == 0) s[v] += zv[k + 1];
        }
        s[v] = warp_sum(s[v]);
      }
      if (lane == 0)
#pragma unroll
        for (int v = 0; v < VB; ++v) red[v][warp] = s[v];
      __syncthreads();
      if (tid < VB) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) t += red[tid][w];
        sv[tid] = t * tk;
      }
      __syncthreads();
#pragma unroll
      for (int v = 0; v < VB; ++v) {
        if (v < nv) {
          double* zv = z + (size_t)v * a;
          const double f = sv[v];
#pragma unroll
          for (int q = 0; q < PR; ++q) {
            const int i = k + 2 + tid + q * kBtThreads;
            if (i < a) zv[i] -= f * cur[q];
          }
          if (tid == 0) zv[k + 1] -= f;
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < PR; ++q) cur[q] = nxt[q];
  }
  // sign rule per vector, one warp each
  for (int v = warp; v < nv; v += NW) {
    const double* zv = z + (size_t)v * a;
    double best = -1.0;
    int bi = a;
    for (int i = lane; i < a; i += 32) {
      const double vv = fabs(zv[i]);
      if (vv > best) { best = vv; bi = i; }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    const double sgn = (zv[bi] < 0.0) ? -1.0 : 1.0;
    double* u = UR + (size_t)(j0 + v) * a;
    for (int i = lane; i < a; i += 32) u[i] = sgn * zv[i];
  }
}

}  // namespace ttg
