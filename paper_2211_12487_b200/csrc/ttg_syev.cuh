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

// one warp: parallel cyclic Jacobi on the symmetric k x k H (k <= 8, ld k),
// eigenvectors into W.  Round-robin pairs, one lane per pair; all row
// rotations of a round, then all column rotations (disjoint supports commute).
// A rotation is skipped when |h_pq| <= 1e-18 sqrt(|h_pp h_qq|); stops after a
// sweep without rotations.
__device__ void small_sym_eig(double* H, double* W, int k) {
  const int lane = threadIdx.x & 31;
  for (int i = lane; i < k * k; i += 32) W[i] = ((i % k) == (i / k)) ? 1.0 : 0.0;
  __syncwarp();
  const int n = k + (k & 1);
  for (int sweep = 0; sweep < 20; ++sweep) {
    int rotated = 0;
    for (int rnd = 0; rnd < n - 1; ++rnd) {
      int pp = -1, qq = -1;
      double c = 1.0, sn = 0.0;
      bool act = false;
      if (lane < n / 2) {
        pp = (lane == 0) ? 0 : ((lane - 1 + rnd) % (n - 1)) + 1;
        qq = ((n - 2 - lane + rnd) % (n - 1)) + 1;
        if (pp > qq) { const int tq = pp; pp = qq; qq = tq; }
        if (qq < k) {
          const double hpq = H[pp + k * qq], hpp = H[pp + k * pp], hqq = H[qq + k * qq];
          if (hpq != 0.0 && fabs(hpq) > 1e-18 * sqrt(fabs(hpp * hqq))) {
            const double zeta = (hqq - hpp) / (2.0 * hpq);
            const double t = copysign(1.0, zeta) / (fabs(zeta) + hypot(1.0, zeta));
            c = 1.0 / sqrt(1.0 + t * t);
            sn = c * t;
            act = true;
          }
        }
      }
      rotated |= __any_sync(0xffffffffu, act);
      __syncwarp();
      if (act)
        for (int r = 0; r < k; ++r) {  // rows p, q
          const double hp = H[pp + k * r], hq = H[qq + k * r];
          H[pp + k * r] = c * hp - sn * hq;
          H[qq + k * r] = sn * hp + c * hq;
        }
      __syncwarp();
      if (act) {
        for (int r = 0; r < k; ++r) {  // columns p, q
          const double hp = H[r + k * pp], hq = H[r + k * qq];
          H[r + k * pp] = c * hp - sn * hq;
          H[r + k * qq] = sn * hp + c * hq;
        }
        for (int r = 0; r < k; ++r) {
          const double wp = W[r + k * pp], wq = W[r + k * qq];
          W[r + k * pp] = c * wp - sn * wq;
          W[r + k * qq] = sn * wp + c * wq;
        }
      }
      __syncwarp();
    }
    if (!rotated) break;
  }
}

// block MGS (twice) of the k columns of X (a x k, ld a); warp-per-column dots,
// sequential over columns; all threads participate, returns after a barrier.
__device__ void block_mgs2(double* X, int a, int k, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int pass = 0; pass < 2; ++pass) {
    for (int j = 0; j < k; ++j) {
      double* xj = X + (size_t)a * j;
      // dots with earlier columns: warp i computes <x_i, x_j>
      for (int i = warp; i < j; i += nw) {
        const double* xi = X + (size_t)a * i;
        double s = 0.0;
        for (int r = lane; r < a; r += 32) s = fma(xi[r], xj[r], s);
        s = warp_sum(s);
        if (lane == 0) red[i] = s;
      }
      __syncthreads();
      for (int r = threadIdx.x; r < a; r += blockDim.x) {
        double v = xj[r];
        for (int i = 0; i < j; ++i) v -= red[i] * X[r + (size_t)a * i];
        xj[r] = v;
      }
      __syncthreads();
      double s = 0.0;
      for (int r = threadIdx.x; r < a; r += blockDim.x) s = fma(xj[r], xj[r], s);
      s = warp_sum(s);
      if (lane == 0) red[32 + warp] = s;
      __syncthreads();
      double nn = 0.0;
      for (int w = 0; w < nw; ++w) nn += red[32 + w];
      const double inv = nn > 0.0 ? 1.0 / sqrt(nn) : 0.0;
      for (int r = threadIdx.x; r < a; r += blockDim.x) xj[r] *= inv;
      __syncthreads();
    }
  }
}

__global__ void __launch_bounds__(kSubThreads) k_syev_top(SyevArgs p) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double red[64];
  __shared__ double H[kSubK * kSubK], Wv[kSubK * kSubK], theta[kSubK], resn[kSubK];
  __shared__ int s_state, s_rank;
  __shared__ double s_tail;
  const int a = p.a;
  const int k = a < kSubK ? a : kSubK;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  double* G = p.in_smem ? sm : const_cast<double*>(p.G);
  double* X = p.in_smem ? sm + (size_t)a * a : sm;
  double* Z = X + (size_t)a * kSubK;
  if (p.in_smem)
    for (long long i = tid; i < (long long)a * a; i += blockDim.x) G[i] = p.G[i];
  // deterministic pseudo-random start block
  for (int e = tid; e < a * k; e += blockDim.x) {
    unsigned long long h = 0x9E3779B97F4A7C15ull * (unsigned long long)(e + 1);
    h ^= h >> 31; h *= 0xbf58476d1ce4e5b9ull; h ^= h >> 27;
    X[e] = (double)(h >> 11) * (1.0 / 9007199254740992.0) - 0.5;
  }
  __syncthreads();
  double trace = 0.0;
  for (int i = 0; i < a; ++i) trace += G[i + (size_t)a * i];
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
  block_mgs2(X, a, k, red);
  double prev_res = 1e300;
  int it = 0;
  for (; it < kSubIters; ++it) {
    // Z = G X  (thread-consecutive rows i: G[i + a*j] is bank-conflict free)
    for (int e = tid; e < a * k; e += blockDim.x) {
      const int i = e % a, c = e / a;
      const double* xc = X + (size_t)a * c;
      double s0 = 0.0, s1 = 0.0;
      int j = 0;
      for (; j + 1 < a; j += 2) {
        s0 = fma(G[i + (size_t)a * j], xc[j], s0);
        s1 = fma(G[i + (size_t)a * (j + 1)], xc[j + 1], s1);
      }
      if (j < a) s0 = fma(G[i + (size_t)a * j], xc[j], s0);
      Z[e] = s0 + s1;
    }
    __syncthreads();
    // H = X^T Z (k x k), symmetrised
    for (int e = warp; e < k * k; e += nw) {
      const int i = e % k, j = e / k;
      double s = 0.0;
      for (int r = lane; r < a; r += 32) s = fma(X[r + (size_t)a * i], Z[r + (size_t)a * j], s);
      s = warp_sum(s);
      if (lane == 0) H[e] = s;
    }
    __syncthreads();
    if (warp == 0) {
      for (int e = lane; e < k * k; e += 32) {
        const int i = e % k, j = e / k;
        if (i < j) {
          const double m = 0.5 * (H[i + k * j] + H[j + k * i]);
          H[i + k * j] = m;
          H[j + k * i] = m;
        }
      }
      __syncwarp();
      small_sym_eig(H, Wv, k);
      if (lane == 0) {  // sort descending (selection sort on k <= 8), permute W
        for (int i = 0; i < k; ++i) theta[i] = H[i + k * i];
        for (int i = 0; i < k; ++i) {
          int m = i;
          for (int j = i + 1; j < k; ++j)
            if (theta[j] > theta[m]) m = j;
          if (m != i) {
            const double tv = theta[i]; theta[i] = theta[m]; theta[m] = tv;
            for (int r = 0; r < k; ++r) { const double w = Wv[r + k * i]; Wv[r + k * i] = Wv[r + k * m]; Wv[r + k * m] = w; }
          }
        }
      }
    }
    __syncthreads();
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
        if (it >= 5) s_state = 2;  // more kept directions than the block holds: full solver
      }
      prev_res = worst;
      red[63] = worst;
    }
    __syncthreads();
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
    block_mgs2(X, a, k, red);
  }
  const int rank = s_rank;
  if (tid == 0) {
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
