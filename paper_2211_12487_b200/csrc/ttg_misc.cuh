// ttg_misc.cuh — small kernels of the sweep: fragment swizzle, norms,
// core padding, TT-ICE* per-observation statistics and decisions, and the
// expansion used by reconstruct.
#pragma once
#include "ttg_pdl.cuh"
#include <cstdint>
#include <cuda_runtime.h>

#include "ttg_eig.cuh"
#include "ttg_kernels.cuh"

namespace ttg {

// U (a x r, ld) -> DMMA A-fragments of U^T ([r8/8][a8/4][32]) and of U
// ([a8/8][r8/4][32]); zero outside the matrix.
__global__ void k_make_frags(const double* __restrict__ U, int a, int r, int ld, int a8, int r8,
                             double* __restrict__ UTf, double* __restrict__ Uf) {
  griddep_wait();
  const int KA = a8 / 4, KR = r8 / 4;
  const long long n1 = (long long)(r8 / 8) * KA * 32;
  const long long n2 = (long long)(a8 / 8) * KR * 32;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n1 + n2;
       e += (long long)gridDim.x * blockDim.x) {
    if (e < n1) {
      if (!UTf) continue;
      int lane = (int)(e & 31);
      long long f = e >> 5;
      int kb = (int)(f % KA), mb = (int)(f / KA);
      int row = kb * 4 + (lane & 3), col = mb * 8 + (lane >> 2);  // A = U^T: A[m][k] = U[k][m]
      UTf[e] = (row < a && col < r) ? U[row + (long long)ld * col] : 0.0;
    } else {
      if (!Uf) continue;
      long long e2 = e - n1;
      int lane = (int)(e2 & 31);
      long long f = e2 >> 5;
      int sb = (int)(f % KR), ib = (int)(f / KR);
      int row = ib * 8 + (lane >> 2), col = sb * 4 + (lane & 3);
      Uf[e2] = (row < a && col < r) ? U[row + (long long)ld * col] : 0.0;
    }
  }
}

// Per-observation partial sums of squares: block (chunk, obs).
__global__ void k_sumsq_obs(const double* __restrict__ Y, long long S, int nchunk,
                            double* __restrict__ part) {
  griddep_wait();
  __shared__ double red[33];
  const int o = blockIdx.y, c = blockIdx.x;
  long long cs = (S + nchunk - 1) / nchunk;
  long long b = (long long)c * cs, e = b + cs;
  if (e > S) e = S;
  const double* y = Y + (long long)o * S;
  double s = 0.0;
  // 16-byte loads when aligned
  if ((((uintptr_t)(y + b)) & 15) == 0) {
    long long n2 = (e - b) / 2;
    const double2* y2 = reinterpret_cast<const double2*>(y + b);
    // four independent loads and accumulators per thread and round (fixed order)
    double s1 = 0.0, s2 = 0.0, s3 = 0.0;
    long long i = threadIdx.x;
    for (; i + 3 * (long long)blockDim.x < n2; i += 4 * (long long)blockDim.x) {
      const double2 v0 = y2[i], v1 = y2[i + blockDim.x], v2 = y2[i + 2 * blockDim.x], v3 = y2[i + 3 * blockDim.x];
      s = fma(v0.x, v0.x, s);
      s = fma(v0.y, v0.y, s);
      s1 = fma(v1.x, v1.x, s1);
      s1 = fma(v1.y, v1.y, s1);
      s2 = fma(v2.x, v2.x, s2);
      s2 = fma(v2.y, v2.y, s2);
      s3 = fma(v3.x, v3.x, s3);
      s3 = fma(v3.y, v3.y, s3);
    }
    for (; i < n2; i += blockDim.x) {
      double2 v = y2[i];
      s = fma(v.x, v.x, s);
      s = fma(v.y, v.y, s);
    }
    s = (s + s1) + (s2 + s3);
    for (long long i = b + 2 * n2 + threadIdx.x; i < e; i += blockDim.x) s = fma(y[i], y[i], s);
  } else {
    for (long long i = b + threadIdx.x; i < e; i += blockDim.x) s = fma(y[i], y[i], s);
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) part[(long long)o * nchunk + c] = s;
}

// on2[o] = sum of chunk partials (fixed order); out_total = sum_o on2[o].
__global__ void k_sumsq_finalize(const double* __restrict__ part, int nchunk, int nobs,
                                 double* __restrict__ on2, double* __restrict__ total) {
  griddep_wait();
  double s = 0.0;
  for (int o = threadIdx.x; o < nobs; o += blockDim.x) {
    double v = 0.0;
    for (int c = 0; c < nchunk; ++c) v += part[(long long)o * nchunk + c];
    on2[o] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int o = 0; o < nobs; ++o) s += on2[o];
    *total = s;
  }
}

// pad_core (tt_ice.cpp:43-58): core (r_old x n x r_right) -> (r_new x n x r_right)
__global__ void k_pad_core(const double* __restrict__ core, int r_old, int n, int r_right, int r_new,
                           double* __restrict__ out) {
  griddep_wait();
  long long tot = (long long)r_new * n * r_right;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot;
       e += (long long)gridDim.x * blockDim.x) {
    int p = (int)(e % r_new);
    long long rest = e / r_new;  // j + n*q
    out[e] = (p < r_old) ? core[p + (long long)r_old * rest] : 0.0;
  }
}


// The whole interface chain in one launch (one block, sequential over the
// modes, steps separated by block barriers; intermediates in global/L2):
// M_0 = [1], M_{i+1}[q, q'] = sum_{j, p, p'} core_i[p, j, q] M_i[p, p'] core_i[p', j, q'].
constexpr int kIfaceMaxModes = 64;
struct IfaceArgs {
  int d;
  const double* cores[kIfaceMaxModes];
  int rl[kIfaceMaxModes], n[kIfaceMaxModes], rr[kIfaceMaxModes];
  int rmax, nmax;
  double* out;  // rr_{d-1}^2 result
};
// shared memory: M ping-pong (2 rmax^2) + T + every core, prefetched up
// front (all loads in flight).  A core (rl x n x rr) and T are stored as rr
// columns of m = rl n entries with a padded stride m + 1, so the per-thread
// column walks of the second contraction hit distinct banks (m is often a
// multiple of 16).
__global__ void __launch_bounds__(1024) k_iface_all(IfaceArgs a) {
  griddep_wait();
  extern __shared__ double sm[];
  double* Mb[2] = {sm, sm + a.rmax * a.rmax};
  double* T = sm + 2 * a.rmax * a.rmax;
  double* Cs0 = T + (a.rmax * a.nmax + 1) * a.rmax;  // the current core (ld m + 1), staged per mode
  if (threadIdx.x == 0) Mb[0][0] = 1.0;
  int f = 0;
  const double* Cs = Cs0;
  for (int i = 0; i < a.d; ++i) {
    const int rl = a.rl[i], n = a.n[i], rr = a.rr[i];
    const int m = rl * n, t1 = m * rr, ms = m + 1;
    {
      const double* __restrict__ src = a.cores[i];
      for (int e = threadIdx.x; e < t1; e += blockDim.x) {
        const int q = e / m, x = e - q * m;
        Cs0[x + ms * q] = __ldg(src + e);
      }
    }
    __syncthreads();
    const double* M = Mb[f];
    // T[p', j, q] = sum_p M[p', p] core[p, j, q]
    for (int e = threadIdx.x; e < t1; e += blockDim.x) {
      const int q = e / m, x = e - q * m;  // x = p' + rl j
      const int pp = x % rl, jj = x / rl;
      const double* cc = Cs + ms * q + rl * jj;
      double s0 = 0.0, s1 = 0.0;
      int p = 0;
      for (; p + 1 < rl; p += 2) {
        s0 = fma(M[pp + rl * p], cc[p], s0);
        s1 = fma(M[pp + rl * (p + 1)], cc[p + 1], s1);
      }
      if (p < rl) s0 = fma(M[pp + rl * p], cc[p], s0);
      T[x + ms * q] = s0 + s1;
    }
    __syncthreads();
    // M'[q, q2] = sum_x core[x, q] T[x, q2]
    double* Mn = (i + 1 == a.d) ? a.out : Mb[f ^ 1];
    for (int e = threadIdx.x; e < rr * rr; e += blockDim.x) {
      const int q = e % rr, q2 = e / rr;
      const double* cq = Cs + ms * q;
      const double* tq = T + ms * q2;
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      int x = 0;
      for (; x + 3 < m; x += 4) {
        s0 = fma(cq[x], tq[x], s0);
        s1 = fma(cq[x + 1], tq[x + 1], s1);
        s2 = fma(cq[x + 2], tq[x + 2], s2);
        s3 = fma(cq[x + 3], tq[x + 3], s3);
      }
      for (; x < m; ++x) s0 = fma(cq[x], tq[x], s0);
      Mn[e] = (s0 + s1) + (s2 + s3);
    }
    __syncthreads();
    f ^= 1;
  }
}

// Q = K P  (rows x a): K = I_n (x) Psi (Psi: As x r, rows = As n, a = r n) or
// K = I_a (Psi null, As = r), P = I - U U^T (U: a x r_old, r_old >= 0).
// One thread per element; (K U)[i, k] is formed inline (r_old r FMA).
__global__ void k_build_q(const double* __restrict__ Psi, int As, int r, int n, const double* __restrict__ U,
                          int r_old, double* __restrict__ Q) {
  griddep_wait();
  const int rows = As * n, a = r * n;
  const long long tot = (long long)rows * a;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e % rows), j = (int)(e / rows);
    const int p = i % As, jn = i / As;
    const int q = j % r, jn2 = j / r;
    double kij = 0.0;
    if (jn == jn2) kij = Psi ? Psi[p + (long long)As * q] : (p == q ? 1.0 : 0.0);
    double s = 0.0;
    for (int k = 0; k < r_old; ++k) {
      double ku;
      if (Psi) {
        ku = 0.0;
        for (int qq = 0; qq < r; ++qq) ku = fma(Psi[p + (long long)As * qq], U[qq + r * jn + (long long)a * k], ku);
      } else {
        ku = U[i + (long long)a * k];
      }
      s = fma(ku, U[j + (long long)a * k], s);
    }
    Q[e] = kij - s;
  }
}

// cn2[o] = |c_o|^2, cmc[o] = c_o^T M c_o  (c: r x b, ld r).  One warp per
// observation: lane i forms (M c)_i for rows i, i + 32, ... (coalesced column
// reads of M, c broadcast), then two fixed-order warp sums.
__global__ void k_coef_stats(const double* __restrict__ C, int r, int b, const double* __restrict__ M,
                             double* __restrict__ cn2, double* __restrict__ cmc) {
  griddep_wait();
  const int lane = threadIdx.x & 31;
  const int nwarp = (gridDim.x * blockDim.x) >> 5;
  for (int o = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; o < b; o += nwarp) {
    const double* c = C + (long long)r * o;
    double s = 0.0, m = 0.0;
    for (int i = lane; i < r; i += 32) {
      const double ci = __ldg(c + i);
      double mi0 = 0.0, mi1 = 0.0;
      int k = 0;
      for (; k + 1 < r; k += 2) {
        mi0 = fma(__ldg(M + i + (long long)r * k), __ldg(c + k), mi0);
        mi1 = fma(__ldg(M + i + (long long)r * (k + 1)), __ldg(c + k + 1), mi1);
      }
      if (k < r) mi0 = fma(__ldg(M + i + (long long)r * k), __ldg(c + k), mi0);
      s = fma(ci, ci, s);
      m = fma(ci, mi0 + mi1, m);
    }
    s = warp_sum(s);
    m = warp_sum(m);
    if (lane == 0) {
      cn2[o] = s;
      cmc[o] = m;
    }
  }
}

// Large r: cn2 / cmc from T = M C computed by the DMMA GEMM (r^2 b flops on the
// tensor pipe instead of one warp's DFMA chain per observation).
__global__ void k_coef_dots(const double* __restrict__ C, const double* __restrict__ T, int r, int b,
                            double* __restrict__ cn2, double* __restrict__ cmc) {
  griddep_wait();
  const int lane = threadIdx.x & 31;
  const int nwarp = (gridDim.x * blockDim.x) >> 5;
  for (int o = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; o < b; o += nwarp) {
    const double* c = C + (long long)r * o;
    const double* t = T + (long long)r * o;
    double s = 0.0, m = 0.0;
    for (int i = lane; i < r; i += 32) {
      const double ci = __ldg(c + i);
      s = fma(ci, ci, s);
      m = fma(ci, __ldg(t + i), m);
    }
    s = warp_sum(s);
    m = warp_sum(m);
    if (lane == 0) {
      cn2[o] = s;
      cmc[o] = m;
    }
  }
}

// TT-ICE* per-observation errors and the partial sums the decision needs
// (tt_ice_star.cpp:22-65, 90-100, 121-158).  Single thread, observation order
// = the reference's loop order.  sums[] layout:
//  0 sum_err(on>0)  1 count(on>0)  2 sum_rn2  3 sum_on2  4 sum_rej_rn2(err<=eps)
//  5 sum_sel_on2(err>eps)  6 n_sel  7 n_rej  8 sum_rej_err
struct StarStats {
  double sums[9];
};
__global__ void __launch_bounds__(256) k_star_local(const double* __restrict__ on2, const double* __restrict__ cn2,
                                                    const double* __restrict__ cmc, int b, double eps,
                                                    double* __restrict__ errs, double* __restrict__ rn2_out,
                                                    StarStats* st) {
  griddep_wait();
  // Per observation (in parallel): err and the nine sum terms, each the value
  // the reference's loop adds or +0.0 when its condition is false (adding
  // +0.0 is exact).  Then lane t < 9 of warp 0 adds row t in observation order,
  // so every sum is bit-identical to one serial pass.  Terms: 0 err (on > 0),
  // 1 count (on > 0), 2 rn^2, 3 on^2 (on = sqrt(on2): the reference squares
  // the root), 4 (err on)^2 (err <= eps), 5 on2 (err > eps), 6 count
  // (err > eps), 7 count (err <= eps), 8 err (err <= eps).
  constexpr int kLd = 257;  // odd stride: the nine lanes read distinct banks
  __shared__ double s_term[9 * kLd];
  double acc = 0.0;
  const int t = threadIdx.x;
  for (int base = 0; base < b; base += 256) {
    const int o = base + t;
    if (o < b) {
      const double o2 = on2[o];
      const double on = sqrt(o2);
      // |y - Phi c|^2 = |y|^2 - 2|c|^2 + c^T (Phi^T Phi) c   (c = Phi^T y)
      double rsq = o2 - 2.0 * cn2[o] + cmc[o];
      if (rsq < 0.0) rsq = 0.0;
      const double rn = sqrt(rsq);
      const double err = (on == 0.0) ? 0.0 : rn / on;
      errs[o] = err;
      rn2_out[o] = rn * rn;
      const double rj = err * on;
      const bool pos = on > 0.0, sel = err > eps;
      s_term[0 * kLd + t] = pos ? err : 0.0;
      s_term[1 * kLd + t] = pos ? 1.0 : 0.0;
      s_term[2 * kLd + t] = rn * rn;
      s_term[3 * kLd + t] = on * on;
      s_term[4 * kLd + t] = sel ? 0.0 : rj * rj;
      s_term[5 * kLd + t] = sel ? o2 : 0.0;
      s_term[6 * kLd + t] = sel ? 1.0 : 0.0;
      s_term[7 * kLd + t] = sel ? 0.0 : 1.0;
      s_term[8 * kLd + t] = sel ? 0.0 : err;
    }
    __syncthreads();
    const int m = min(256, b - base);
    if (t < 9) {
      const double* row = s_term + t * kLd;
#pragma unroll 8
      for (int q = 0; q < m; ++q) acc += row[q];
    }
    __syncthreads();
  }
  if (t < 9) st->sums[t] = acc;
}

// W = I_n (x) Psi  ((As*n) x (r*n), block diagonal)
__global__ void k_kron_eye(const double* __restrict__ Psi, int As, int r, int n, double* __restrict__ W) {
  griddep_wait();
  const long long rows = (long long)As * n, tot = rows * r * n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot;
       e += (long long)gridDim.x * blockDim.x) {
    const long long row = e % rows, col = e / rows;
    const int j = (int)(row / As), k = (int)(row % As);
    const int j2 = (int)(col / r), p = (int)(col % r);
    W[e] = (j == j2) ? Psi[k + (long long)As * p] : 0.0;
  }
}

// out (rn x L) = [old (ro x L) ; add ((rn - ro) x L)] row-interleaved per column
__global__ void k_merge_rows(const double* __restrict__ old, int ro, const double* __restrict__ add, int rn,
                             long long L, double* __restrict__ out) {
  griddep_wait();
  const int ra = rn - ro;
  const long long tot = (long long)rn * L;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot;
       e += (long long)gridDim.x * blockDim.x) {
    const long long q = e / rn;
    const int p = (int)(e - q * rn);
    out[e] = (p < ro) ? old[p + (long long)ro * q] : add[(p - ro) + (long long)ra * q];
  }
}

// G <- (G + G^T) / 2 over a grid (one thread per strictly-lower element);
// block 0 also writes trace(Tsrc) -> *tr (Tsrc: nt x nt; G's diagonal is not
// modified, so Tsrc may be G; fixed warp-tree order, deterministic).
__global__ void k_symmetrize_trace(double* __restrict__ G, int a, const double* Tsrc, int nt, double* __restrict__ tr) {
  griddep_wait();
  const long long n = (long long)a * a;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e % a), j = (int)(e / a);
    if (i > j) {
      const double m = 0.5 * (G[i + (long long)a * j] + G[j + (long long)a * i]);
      G[i + (long long)a * j] = m;
      G[j + (long long)a * i] = m;
    }
  }
  if (blockIdx.x == 0 && tr && threadIdx.x < 32) {
    double s = 0.0;
    for (int i = threadIdx.x; i < nt; i += 32) s += Tsrc[i + (long long)nt * i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) *tr = s;
  }
}

// Residual Gram from the raw Gram in one CTA (no pre-projection, K = I):
//   G = P C P = C - (U Y^T + Y U^T),  W = C U,  M = sym(U^T W),  Y = W - M' ,
// with M' = U M / 2, so that U Y^T + Y U^T = U W^T + W U^T - U M U^T.
// Rank-r work (a^2 r) instead of the two dense a^3 GEMMs of the Q^T C Q form.
// W = C U, M = U^T W and the rank-2r update [U Y][Y U]^T run on DMMA
// (m8n8k4); only the lower 8 x 8 blocks of G are formed (the diagonal
// blocks' lower halves) and mirrored, so G is exactly symmetric; trace(C) goes
// to *tr for the raw-Gram accuracy guard.  C and G may alias.
// Shared memory, zero-padded to multiples of 8 with leading dimension
// ld = pcp_ld(a8) (== 4 mod 16 doubles: the fragment loads of a half-warp,
// rows g + 4 t, hit 16 distinct banks; with ld = a8 = 112 every column
// started in the same bank and the phases ran 4-13-way conflicted):
// C (ld x a8), U and W / Y (ld x r8 each), M (r8 x r8).  Needs a r <= 8 x
// threads and r <= 32.
constexpr int kPcpThreads = 512;
__host__ __device__ constexpr int pcp_ld(int a8) { return a8 + ((20 - a8 % 16) % 16); }
__host__ __device__ constexpr size_t pcp_smem_doubles(int a, int r) {
  return (size_t)pcp_ld((a + 7) & ~7) * (((a + 7) & ~7) + 2 * (((r > 1 ? r : 1) + 7) & ~7)) +
         (size_t)(((r > 1 ? r : 1) + 7) & ~7) * (((r > 1 ? r : 1) + 7) & ~7);
}
__global__ void __launch_bounds__(kPcpThreads) k_pcp(const double* C, int a, const double* __restrict__ U, int r,
                                                     double* G, double* __restrict__ tr) {
  griddep_wait();
  extern __shared__ double psm[];
  const int a8 = (a + 7) & ~7, r8 = (r + 7) & ~7, ld = pcp_ld(a8);
  double* Cs = psm;                       // ld x a8
  double* Us = Cs + (size_t)ld * a8;      // ld x r8
  double* Ws = Us + (size_t)ld * r8;      // ld x r8 (W, then Y)
  double* Ms = Ws + (size_t)ld * r8;      // r8 x r8
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarp = nt >> 5;
  const int g = lane >> 2, t = lane & 3;
  {  // staging: contiguous loads batched in registers (8 in flight per thread),
     // then scattered into the padded layout; padding rows / columns zeroed
    const int n = a * a, m = a * r;
    for (int base = tid; base < n + m; base += 8 * nt) {
      double v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int e = base + q * nt;
        v[q] = e < n ? __ldg(C + e) : (e < n + m ? __ldg(U + (e - n)) : 0.0);
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int e = base + q * nt;
        if (e < n) Cs[(e % a) + ld * (e / a)] = v[q];
        else if (e < n + m) Us[((e - n) % a) + ld * ((e - n) / a)] = v[q];
      }
    }
    for (int e = tid; e < a8 * a8; e += nt) {
      const int i = e % a8, j = e / a8;
      if (i >= a || j >= a) Cs[i + ld * j] = 0.0;
    }
    for (int e = tid; e < a8 * r8; e += nt) {
      const int i = e % a8, k = e / a8;
      if (i >= a || k >= r) Us[i + ld * k] = 0.0;
    }
  }
  __syncthreads();
  if (tid < 32) {
    double s = 0.0;
    for (int i = tid; i < a; i += 32) s += Cs[i + ld * i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (tid == 0) *tr = s;
  }
  // W = C U: task = 8-row block ib; accumulators for every 8-column block
  const int nbr = a8 / 8, nbc = r8 / 8;  // nbc <= 4 (r <= 32)
  for (int ib = warp; ib < nbr; ib += nwarp) {
    double acc[4][2];
#pragma unroll
    for (int jb = 0; jb < 4; ++jb) acc[jb][0] = acc[jb][1] = 0.0;
    const double* crow = Cs + ib * 8 + g;
#pragma unroll 2
    for (int k0 = 0; k0 < a8; k0 += 4) {
      const double av = crow[(size_t)ld * (k0 + t)];
#pragma unroll
      for (int jb = 0; jb < 4; ++jb)
        if (jb < nbc) dmma(acc[jb][0], acc[jb][1], av, Us[(k0 + t) + (size_t)ld * (jb * 8 + g)]);
    }
#pragma unroll
    for (int jb = 0; jb < 4; ++jb)
      if (jb < nbc) {
        Ws[ib * 8 + g + (size_t)ld * (jb * 8 + 2 * t)] = acc[jb][0];
        Ws[ib * 8 + g + (size_t)ld * (jb * 8 + 2 * t + 1)] = acc[jb][1];
      }
  }
  __syncthreads();
  // M = U^T W (r8 x r8, padded entries zero): one 8 x 8 block per warp task
  for (int blk = warp; blk < nbc * nbc; blk += nwarp) {
    const int kb = blk % nbc, lb = blk / nbc;
    double d0 = 0.0, d1 = 0.0;
#pragma unroll 2
    for (int k0 = 0; k0 < a8; k0 += 4)
      dmma(d0, d1, Us[(k0 + t) + (size_t)ld * (kb * 8 + g)], Ws[(k0 + t) + (size_t)ld * (lb * 8 + g)]);
    Ms[kb * 8 + g + r8 * (lb * 8 + 2 * t)] = d0;
    Ms[kb * 8 + g + r8 * (lb * 8 + 2 * t + 1)] = d1;
  }
  __syncthreads();
  // Y = W - U sym(M) / 2: work item (row i, column l); all reads of W precede
  // the barrier, writes go to the element's own slot after it
  double ynew[8];
  {
    int nmine = 0;
    for (int w = tid; w < a * r && nmine < 8; w += nt, ++nmine) {
      const int i = w % a, l = w / a;
      double s = 0.0;
      for (int k = 0; k < r; ++k) s = fma(Us[i + ld * k], 0.5 * (Ms[k + r8 * l] + Ms[l + r8 * k]), s);
      ynew[nmine] = Ws[i + ld * l] - 0.5 * s;
    }
  }
  __syncthreads();
  {
    int m = 0;
    for (int w = tid; w < a * r && m < 8; w += nt, ++m) Ws[(w % a) + ld * (w / a)] = ynew[m];
  }
  __syncthreads();
  // lower 8 x 8 blocks of G = C - [U Y][Y U]^T (k over 2 r8), mirrored
  const int nlow = nbr * (nbr + 1) / 2;
  for (int blk = warp; blk < nlow; blk += nwarp) {
    int ib = 0;
    while ((ib + 1) * (ib + 2) / 2 <= blk) ++ib;
    const int jb = blk - ib * (ib + 1) / 2;
    double d0 = 0.0, d1 = 0.0;
    const int i = ib * 8 + g, jrow = jb * 8 + g;
#pragma unroll 2
    for (int k0 = 0; k0 < r8; k0 += 4) {  // U_i . Y_j
      dmma(d0, d1, Us[i + (size_t)ld * (k0 + t)], Ws[jrow + (size_t)ld * (k0 + t)]);
    }
#pragma unroll 2
    for (int k0 = 0; k0 < r8; k0 += 4) {  // Y_i . U_j
      dmma(d0, d1, Ws[i + (size_t)ld * (k0 + t)], Us[jrow + (size_t)ld * (k0 + t)]);
    }
    const double dv[2] = {d0, d1};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = jb * 8 + 2 * t + h;
      if (i < a && j < a && (ib != jb || i >= j)) {
        const double gv = Cs[i + (size_t)ld * j] - dv[h];
        G[i + (long long)a * j] = gv;
        G[j + (long long)a * i] = gv;
      }
    }
  }
}

// k_pcp for Grams that do not fit shared memory (a8 <= 256, r <= 32): C stays
// in L2 (read as DMMA fragments for W = C U and once more for the output), U,
// W, Y = W - U sym(M)/2 and M = U^T W in shared memory.  G = P C P written in
// place of C (every read of C's upper triangle -- only in W = C U -- precedes
// the first write; the output phase reads only lower blocks and writes each
// element's mirror), trace(C) for the raw-Gram guard.  Replaces the 4-launch
// k_build_q + 2 GEMMs + k_symmetrize_trace path for the mode-3..7 Grams of
// configs[3] at bond ranks 17-32.
__host__ __device__ constexpr size_t pcp_l2_smem_doubles(int a, int r) {
  return (size_t)3 * pcp_ld((a + 7) & ~7) * (((r > 1 ? r : 1) + 7) & ~7) +
         (size_t)(((r > 1 ? r : 1) + 7) & ~7) * (((r > 1 ? r : 1) + 7) & ~7);
}
__global__ void __launch_bounds__(kPcpThreads) k_pcp_l2(double* C, int a, const double* __restrict__ U, int r,
                                                        double* __restrict__ tr) {
  griddep_wait();
  extern __shared__ double psm[];
  const int a8 = (a + 7) & ~7, r8 = (r + 7) & ~7, ld = pcp_ld(a8);
  double* Us = psm;                       // ld x r8
  double* Ws = Us + (size_t)ld * r8;      // ld x r8
  double* Ys = Ws + (size_t)ld * r8;      // ld x r8
  double* Ms = Ys + (size_t)ld * r8;      // r8 x r8
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarp = nt >> 5;
  const int g = lane >> 2, t = lane & 3;
  for (int e = tid; e < ld * r8; e += nt) {
    const int i = e % ld, k = e / ld;
    Us[e] = (i < a && k < r) ? __ldg(U + i + (size_t)a * k) : 0.0;
  }
  if (tid < 32) {
    double s = 0.0;
    for (int i = tid; i < a; i += 32) s += C[i + (size_t)a * i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (tid == 0) *tr = s;
  }
  __syncthreads();
  // W = C U: warp task = 8-row block; C fragments from L2
  const int nbr = a8 / 8, nbc = r8 / 8;  // nbc <= 4
  for (int ib = warp; ib < nbr; ib += nwarp) {
    double acc[4][2];
#pragma unroll
    for (int jb = 0; jb < 4; ++jb) acc[jb][0] = acc[jb][1] = 0.0;
    const int i = ib * 8 + g;
#pragma unroll 4
    for (int k0 = 0; k0 < a8; k0 += 4) {
      const int kk = k0 + t;
      const double av = (i < a && kk < a) ? C[i + (size_t)a * kk] : 0.0;
#pragma unroll
      for (int jb = 0; jb < 4; ++jb)
        if (jb < nbc) dmma(acc[jb][0], acc[jb][1], av, Us[kk + (size_t)ld * (jb * 8 + g)]);
    }
#pragma unroll
    for (int jb = 0; jb < 4; ++jb)
      if (jb < nbc) {
        Ws[i + (size_t)ld * (jb * 8 + 2 * t)] = acc[jb][0];
        Ws[i + (size_t)ld * (jb * 8 + 2 * t + 1)] = acc[jb][1];
      }
  }
  __syncthreads();
  // M = U^T W
  for (int blk = warp; blk < nbc * nbc; blk += nwarp) {
    const int kb = blk % nbc, lb = blk / nbc;
    double d0 = 0.0, d1 = 0.0;
#pragma unroll 2
    for (int k0 = 0; k0 < a8; k0 += 4)
      dmma(d0, d1, Us[(k0 + t) + (size_t)ld * (kb * 8 + g)], Ws[(k0 + t) + (size_t)ld * (lb * 8 + g)]);
    Ms[kb * 8 + g + r8 * (lb * 8 + 2 * t)] = d0;
    Ms[kb * 8 + g + r8 * (lb * 8 + 2 * t + 1)] = d1;
  }
  __syncthreads();
  // Y = W - U sym(M) / 2 (padded rows / columns zero)
  for (int w = tid; w < ld * r8; w += nt) {
    const int i = w % ld, l = w / ld;
    double y = 0.0;
    if (i < a && l < r) {
      double s = 0.0;
      for (int k = 0; k < r; ++k) s = fma(Us[i + ld * k], 0.5 * (Ms[k + r8 * l] + Ms[l + r8 * k]), s);
      y = Ws[i + ld * l] - 0.5 * s;
    }
    Ys[w] = y;
  }
  __syncthreads();
  // lower 8 x 8 blocks of G = C - [U Y][Y U]^T, mirrored
  const int nlow = nbr * (nbr + 1) / 2;
  for (int blk = warp; blk < nlow; blk += nwarp) {
    int ib = 0;
    while ((ib + 1) * (ib + 2) / 2 <= blk) ++ib;
    const int jb = blk - ib * (ib + 1) / 2;
    double d0 = 0.0, d1 = 0.0;
    const int i = ib * 8 + g, jrow = jb * 8 + g;
#pragma unroll 2
    for (int k0 = 0; k0 < r8; k0 += 4) dmma(d0, d1, Us[i + (size_t)ld * (k0 + t)], Ys[jrow + (size_t)ld * (k0 + t)]);
#pragma unroll 2
    for (int k0 = 0; k0 < r8; k0 += 4) dmma(d0, d1, Ys[i + (size_t)ld * (k0 + t)], Us[jrow + (size_t)ld * (k0 + t)]);
    const double dv[2] = {d0, d1};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = jb * 8 + 2 * t + h;
      if (i < a && j < a && (ib != jb || i >= j)) {
        const double gv = C[i + (size_t)a * j] - dv[h];
        C[i + (size_t)a * j] = gv;
        C[j + (size_t)a * i] = gv;
      }
    }
  }
}

// selection mask (err > eps, or all when subselect is off)
__global__ void k_star_mask(const double* __restrict__ errs, int b, double eps, int subselect,
                            uint8_t* __restrict__ sel) {
  griddep_wait();
  for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < b; o += gridDim.x * blockDim.x)
    sel[o] = subselect ? (errs[o] > eps ? 1 : 0) : 1;
}

// ---- tall unfoldings (a > 2 L): the small side ----------------------------
// The reference's own tall branch (truncated_svd.cpp:51-59) QR-reduces an
// a x L residual with a > 2 L before its SVD; here the eigen-problem is solved
// on the L x L side (R^T R, or the TSQR factor of R^T on the accurate path)
// and the left singular vectors are recovered as u_j = R v_j / |R v_j|.

// out (L x a) = X^T (X: a x L, column-major), 32 x 32 smem tiles
__global__ void k_transpose(const double* __restrict__ X, int a, long long L, double* __restrict__ out) {
  griddep_wait();
  __shared__ double tile[32][33];
  const long long c0 = (long long)blockIdx.x * 32;
  const int r0 = blockIdx.y * 32;
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int r = r0 + threadIdx.x;
    const long long c = c0 + j;
    tile[j][threadIdx.x] = (r < a && c < L) ? X[r + (long long)a * c] : 0.0;
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int r = r0 + j;
    const long long c = c0 + threadIdx.x;
    if (r < a && c < L) out[c + L * (long long)r] = tile[threadIdx.x][j];
  }
}

// U_R column j (one CTA per kept direction): u = R v_j (R: a x L, V: L x rank,
// ld L), normalised, sign rule (largest-|.| entry, first index, positive:
// truncated_svd.cpp:16-25).
__global__ void __launch_bounds__(256) k_tall_u(const double* __restrict__ R, int a, int L,
                                                const double* __restrict__ V, double* __restrict__ U) {
  griddep_wait();
  __shared__ double red[8];
  __shared__ int redi[8];
  __shared__ double s_inv;
  const int j = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double* v = V + (long long)L * j;
  double* u = U + (long long)a * j;
  double nn = 0.0, best = -1.0;
  int bi = a;
  for (int i = tid; i < a; i += blockDim.x) {
    double s = 0.0;
    for (int l = 0; l < L; ++l) s = fma(R[i + (long long)a * l], v[l], s);
    u[i] = s;
    nn = fma(s, s, nn);
    if (fabs(s) > best) { best = fabs(s); bi = i; }
  }
  for (int o = 16; o > 0; o >>= 1) {
    nn += __shfl_xor_sync(0xffffffffu, nn, o);
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
  }
  if (lane == 0) { red[warp] = nn; redi[warp] = bi; }
  __syncthreads();
  if (tid == 0) {
    double tot = 0.0, bb = -1.0;
    int bidx = a;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      const int ix = redi[w];
      const double vv = ix < a ? fabs(u[ix]) : -1.0;
      if (vv > bb || (vv == bb && ix < bidx)) { bb = vv; bidx = ix; }
    }
    const double inv = tot > 0.0 ? 1.0 / sqrt(tot) : 0.0;
    s_inv = (bidx < a && u[bidx] < 0.0) ? -inv : inv;
  }
  __syncthreads();
  const double f = s_inv;
  for (int i = tid; i < a; i += blockDim.x) u[i] *= f;
}

// ---------------------------------------------------------------------------
// The last modes of a projection chain (tt_project, tensor_train.cpp:195-226) in
// ONE launch.  Once an observation's unfolding fits shared memory (cfg3: from
// mode 5 on, 192 x 64 doubles), each remaining mode is a handful of
// microseconds of arithmetic behind a launch of its own; here one CTA owns one
// observation and walks the modes in place: stage t computes
// core_t^T (rows_t x cols_t block) -> rr_t x cols_t, which, read as
// (rr_t n_{t+1}) x (cols_t / n_{t+1}), is the next stage's input (the same flat
// buffer, first index fastest).  Intermediate unfoldings are also written to
// global memory when the caller keeps them (TT-ICE* reuses the statistics
// chain's intermediates in the sweep).  Plain DFMA, fixed summation order.
// ---------------------------------------------------------------------------
constexpr int kTailMaxModes = 6;
constexpr int kTailThreads = 512;
struct TailArgs {
  const double* X;  // rows[0] x (cols[0] * b), observation slowest
  int nm;
  const double* core[kTailMaxModes];  // (rows[t]) x rr[t], ld rows[t]
  int rows[kTailMaxModes], rr[kTailMaxModes], cols[kTailMaxModes];
  double* out[kTailMaxModes];  // rr[t] x (cols[t] * b) or null (the last one is the coefficient block)
  int obuf;                    // doubles of one ping-pong output buffer (max rr[t] cols[t])
};
__host__ __device__ inline int tail_ld(int rows) { return (rows + 3 + 15) / 16 * 16 + 4; }  // >= rows + 3, = 4 mod 16
__global__ void __launch_bounds__(kTailThreads) k_project_tail(TailArgs p) {
  griddep_wait();
  extern __shared__ __align__(16) double sm[];
  const long long o = blockIdx.x;
  const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);  // warp-uniform: no WARPSYNC per DMMA
  const int g = lane >> 2, tq = lane & 3;
  // shared memory: the observation's block and the current core with leading
  // dimensions = 4 (mod 16) (the m8n8k4 fragment loads of a half-warp then hit
  // 16 distinct banks) and zero rows up to a multiple of 4; two ping-pong
  // output buffers (flat: the next stage reads them with its own row count)
  const int rows0 = p.rows[0], cols0 = p.cols[0], ld0 = tail_ld(rows0);
  double* xin = sm;
  double* dstb[2] = {sm + (size_t)ld0 * cols0, nullptr};
  dstb[1] = dstb[0] + p.obuf;
  double* Us = dstb[1] + p.obuf;
  {
    const double* x = p.X + o * (long long)rows0 * cols0;
    // (cp.async: every copy of the block is in flight before the first wait)
    for (int c = warp; c < cols0; c += nw)
      for (int k = lane; k < ld0; k += 32)
        cp_async8(xin + k + (size_t)ld0 * c, x + (k < rows0 ? k : 0) + (size_t)rows0 * c, k < rows0);
  }
  const double* src = xin;
  int lds = ld0;
  for (int t = 0; t < p.nm; ++t) {
    const int rows = p.rows[t], rr = p.rr[t], cols = p.cols[t], ldu = tail_ld(rows);
    const double* __restrict__ U = p.core[t];
    for (int j = warp; j < rr; j += nw)
      for (int k = lane; k < ldu; k += 32)
        cp_async8(Us + k + (size_t)ldu * j, U + (k < rows ? k : 0) + (size_t)rows * j, k < rows);
    cp_async_commit();
    cp_async_wait_0();
    __syncthreads();
    double* dst = dstb[t & 1];
    double* gl = p.out[t] ? p.out[t] + o * (long long)rr * cols : nullptr;
    // out (rr x cols) = U^T src on DMMA: one 8 x 8 block per warp task
    const int nmb = (rr + 7) >> 3, nnb = (cols + 7) >> 3, nk = (rows + 3) >> 2;
    for (int task = warp; task < nmb * nnb; task += nw) {
      const int mb = task % nmb, nb = task / nmb;
      const int m = mb * 8 + g, n = nb * 8 + g;
      const double* ap = Us + (size_t)ldu * (m < rr ? m : rr - 1) + tq;       // A[m][k] = U[k][m]
      const double* bp = src + (size_t)lds * (n < cols ? n : cols - 1) + tq;  // B[k][n] = src[k][n]
      double c0 = 0.0, c1 = 0.0, e0 = 0.0, e1 = 0.0;
      int ks = 0;
      for (; ks + 1 < nk; ks += 2) {
        dmma(c0, c1, ap[4 * ks], bp[4 * ks]);
        dmma(e0, e1, ap[4 * ks + 4], 4 * ks + 4 + tq < rows ? bp[4 * ks + 4] : 0.0);
      }
      if (ks < nk) dmma(c0, c1, ap[4 * ks], 4 * ks + tq < rows ? bp[4 * ks] : 0.0);
      c0 += e0;
      c1 += e1;
      const int jo = mb * 8 + g, co = nb * 8 + 2 * tq;  // C[m = g][n = 2 tq, 2 tq + 1]
      if (jo < rr) {
        if (co < cols) { dst[jo + (size_t)rr * co] = c0; if (gl) gl[jo + (size_t)rr * co] = c0; }
        if (co + 1 < cols) { dst[jo + (size_t)rr * (co + 1)] = c1; if (gl) gl[jo + (size_t)rr * (co + 1)] = c1; }
      }
    }
    __syncthreads();
    src = dst;  // rr x cols, read by the next stage as (rr n) x (cols / n): the same flat buffer
    lds = t + 1 < p.nm ? p.rows[t + 1] : 1;
  }
}

}  // namespace ttg
