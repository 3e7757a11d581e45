// ttg_decide.cuh — one launch per mode for the common case of the update sweep:
// "old basis U (a x r), raw Gram C of the unfolding, a few new directions".
//
// Replaces, for a <= 320 and r <= 40, the chain
//   k_pcp | (k_build_q, 2 x k_dgemm, k_symmetrize_trace)  ->  k_syev_top  ->  k_append
// (svd_trunc truncated_svd.cpp:29-94 on the residual of tt_ice.cpp:34-41, then
// append_directions update_common.hpp:19-36) by ONE single-CTA kernel that never
// forms the residual Gram G = P C P (P = I - U U^T):
//   * block subspace iteration on the operator  X -> P (C X)  with X kept in
//     range(P).  Per iteration: one DMMA pass over C (read from L2, 8 rows x 4
//     columns per m8n8k4 A fragment, a whole k-range of loads in flight per
//     lane), T = U^T Y and [X | Z]^T Z as two small DMMA reductions, the K x K
//     algebra (Rayleigh-Ritz, Cholesky of the rotated Gram) in one lane, and
//     row-parallel updates in between: five block barriers per iteration;
//   * trace(G) = trace(C) - trace(U^T C U): C U rides on the first pass (the B
//     operand is [U | X0]; the U columns only feed the trace);
//   * rank rule (trace(G) - sum theta_j <= delta^2, Ritz values are lower
//     bounds), residual certificate and sign rule as k_syev_top;
//   * the appended core [U U_R] with the reference's 1e-10 Gram-deviation guard
//     is written here; when the guard fires (rare) res->guard = 2 and the host
//     runs k_append's Householder correction.
// Every reduction has a fixed order (bitwise reproducible).  When the solve
// cannot certify a rank below the block size, res->converged = 0 and the host
// falls back to the explicit chain; C is never modified.
//
// Speculative sweeps (ttg.cu, sweep()): `expect` is the rank the host assumed
// when it sized the following launches without waiting for this kernel; any
// disagreement (rank, convergence, guard, raw-Gram / accuracy fallbacks) sets
// *spec_flag and the host re-runs the sweep synchronously from the saved cores.
#pragma once

#include "ttg_eig.cuh"
#include "ttg_kernels.cuh"
#include "ttg_syev.cuh"

namespace ttg {

constexpr int kDecThreads = 512;
constexpr int kDecMaxA = 320;
constexpr int kDecMaxR = 40;
constexpr int kDecIters = 10;  // a spectrum without a gap below the kept directions belongs to the full solver
constexpr int kDecMaxSplit = 5;  // ceil(kDecMaxA / 64)

struct DecideArgs {
  const double* C;  // a x a raw Gram (symmetric, both triangles), global
  int a;
  const double* U;  // a x r orthonormal old basis (padded core), ld a; r >= 1
  int r;
  long long kmax;
  const double* delta_src;  // delta = delta_mult * sqrt(*delta_src) or delta_mult
  double delta_mult;
  double* UR;   // a x K: kept directions (sign rule applied)
  double* lam;  // K Ritz values
  double* out;  // appended core, capacity a x (r + K - 1); == U: extended in place
  EigResult* res;
  double* trC;  // trace(C) for the host's raw-Gram guard
  int* guard_count;
  int ldb;      // smem leading dimension: >= round_up(a, 4), = 4 mod 16
  int ksplit;   // k-range parts per 8-row block: ceil(a / 64) (dec_pass: 16 k-steps per task)
  int expect;   // speculative sweeps: assumed rank (-1: none)
  int* spec_flag;
  EigResult* log;  // per-mode copy of *res (read once per update), may be null
};

// (>= round_up(a, 64): the last k-range of a pass reads B rows up to there; rows >= a are zero)
__host__ __device__ inline int dec_ldb(int a) { return (a + 63) / 64 * 64 + 4; }
// The warp index as a warp-uniform value (lane 0's, broadcast): loops and
// branches on it are then compiled as uniform, and the mma.sync inside them are
// not each preceded by a WARPSYNC (which had serialised every DMMA of this kernel
// behind its operand load).
__device__ __forceinline__ int dec_warp() { return __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0); }
__host__ __device__ inline int dec_bcols(int r, int K) {
  const int nbt = (r + K + 7) / 8;
  return nbt * 8 > r + 8 ? nbt * 8 : r + 8;
}
inline size_t dec_smem_doubles(int a, int r, int K) {
  // [U | X | 0] (bcols), Yp (ksplit x K), Z, XW (K each), all ld ldb; gram partials (16 x 64)
  return (size_t)dec_ldb(a) * (dec_bcols(r, K) + (kDecMaxSplit + 2) * K) + 16 * 64;
}

// acc = C[rows of task] * B[:, col0 .. col0 + 8 nbt) over the task's k range.
// Columns < r_tr feed the task's trace partial sum_i U[i][n] (C U)[i][n];
// columns [xoff, xoff + K) are stored as the task's k-range partial of Y = C X
// (Yp[ks], summed in order by the consumers).  A task is one 8-row block x
// kDecTaskK k-steps (64 columns of C), always full length: the A-fragment loads
// of the last, partial range are clamped into the matrix and meet the zero
// rows of the padded B operand, so the body carries no bounds predicates --
// all loads of a task are in flight before its first DMMA.
constexpr int kDecTaskK = 16;
template <int NBMAX>
__device__ __noinline__ void dec_pass(const double* __restrict__ C, int a, const double* Bs, int ldb, int col0,
                                      int r_tr, int xoff, int K, int ksplit, double* Yp, double* trpart) {
  const int lane = threadIdx.x & 31, warp = dec_warp(), nw = blockDim.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int nrb = (a + 7) >> 3;
  const int ntask = nrb * ksplit;
#pragma unroll 1
  for (int task = warp; task < ntask; task += nw) {
    const int rb = task / ksplit, ks = task - rb * ksplit;
    const int i = rb * 8 + g;
    const bool iv = i < a;
    const double* crow = C + (size_t)a * (iv ? i : a - 1);  // C symmetric: row i read as column i
    const int k0 = ks * kDecTaskK * 4 + t;
    double av[kDecTaskK];
#pragma unroll
    for (int u = 0; u < kDecTaskK; ++u) {
      const int kk = k0 + 4 * u;
      av[u] = __ldg(crow + (kk < a ? kk : a - 1));
    }
    double acc[NBMAX][2];
#pragma unroll
    for (int nb = 0; nb < NBMAX; ++nb) acc[nb][0] = acc[nb][1] = 0.0;
    const double* bp = Bs + k0 + (size_t)ldb * (col0 + g);
#pragma unroll
    for (int u = 0; u < kDecTaskK; ++u) {
#pragma unroll
      for (int nb = 0; nb < NBMAX; ++nb)
        dmma(acc[nb][0], acc[nb][1], av[u], bp[4 * u + (size_t)ldb * 8 * nb]);
    }
    double trp = 0.0;
#pragma unroll
    for (int nb = 0; nb < NBMAX; ++nb) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int n = col0 + nb * 8 + 2 * t + h;
        const double v = acc[nb][h];
        if (iv) {
          if (n < r_tr) trp = fma(v, Bs[i + (size_t)ldb * n], trp);
          else if (n >= xoff && n < xoff + K) Yp[(size_t)ldb * (ks * K + (n - xoff)) + i] = v;
        }
      }
    }
    if (trpart) {
      trp = warp_sum(trp);
      if (lane == 0) trpart[task] = trp;
    }
  }
}

// One warp's share of a small DMMA reduction Q (nm x K) = A^T B over the a
// rows (A: nm columns of shared memory, B: a x K): the 8-column block of A
// and the k-step range are fixed per warp at kernel start (DecGramTask).
struct DecGramTask {
  int mb, k_lo, k_hi;  // k_hi <= k_lo: no task for this warp
};
__device__ __forceinline__ DecGramTask dec_gram_task(int nm, int a, int& kparts) {
  const int warp = dec_warp(), nw = blockDim.x >> 5;
  const int nmb = (nm + 7) >> 3, nk = (a + 3) >> 2;
  kparts = nw / nmb;
  kparts = kparts < 1 ? 1 : (kparts > 8 ? 8 : kparts);
  DecGramTask tk{0, 0, 0};
  if (warp < nmb * kparts) {
    tk.mb = warp / kparts;
    const int kp = warp - tk.mb * kparts;
    tk.k_lo = nk * kp / kparts;
    tk.k_hi = nk * (kp + 1) / kparts;
  }
  return tk;
}
// A column m of the block at shared offset aoff[m]; B summed over nsum buffers
// `bstride` apart (the k-range partials of Y).  Partial -> Qp[warp].
__device__ __noinline__ void dec_gram(const DecGramTask tk, const double* smbase, const int* aoff, int nm,
                                         const double* B, int ldb, int K, int nsum, int bstride, double* Qp) {
  if (tk.k_hi <= tk.k_lo) return;
  const int lane = threadIdx.x & 31, warp = dec_warp();
  const int g = lane >> 2, t = lane & 3;
  const int m = tk.mb * 8 + g;
  const bool mv = m < nm, bv = g < K;
  const double* ap = smbase + (mv ? aoff[m] : 0) + t;
  const double* bp = B + (size_t)ldb * (bv ? g : 0) + t;
  double c0 = 0.0, c1 = 0.0, e0 = 0.0, e1 = 0.0;
  int ks = tk.k_lo;
  for (; ks + 1 < tk.k_hi; ks += 2) {
    double b0 = bp[4 * ks], b1 = bp[4 * ks + 4];
    for (int q = 1; q < nsum; ++q) { b0 += bp[4 * ks + q * bstride]; b1 += bp[4 * ks + 4 + q * bstride]; }
    dmma(c0, c1, mv ? ap[4 * ks] : 0.0, bv ? b0 : 0.0);
    dmma(e0, e1, mv ? ap[4 * ks + 4] : 0.0, bv ? b1 : 0.0);
  }
  if (ks < tk.k_hi) {
    double b0 = bp[4 * ks];
    for (int q = 1; q < nsum; ++q) b0 += bp[4 * ks + q * bstride];
    dmma(c0, c1, mv ? ap[4 * ks] : 0.0, bv ? b0 : 0.0);
  }
  double* q = Qp + (size_t)warp * 64 + g * 8 + 2 * t;
  q[0] = c0 + e0;
  q[1] = c1 + e1;
}
// Q[m][c] (ld 8) = sum over the k-range partials, in order
__device__ __noinline__ void dec_gram_sum(const double* Qp, int nm, int K, int kparts, double* Q, int tid0, int nthr) {
  for (int e = tid0; e < nm * K; e += nthr) {
    const int m = e / K, c = e - m * K;
    const int mb = m >> 3, g = m & 7;
    double s = 0.0;
    for (int kp = 0; kp < kparts; ++kp) s += Qp[(size_t)(mb * kparts + kp) * 64 + g * 8 + c];
    Q[m * 8 + c] = s;
  }
}

// K x K (K <= 4), one lane: given S = Z^T Z (ld 4) and a rotation Wv (k x k,
// ld k), M = Wv D R^-1 with (Z M)^T (Z M) = I (column-scaled Cholesky of
// Wv^T S Wv).  Returns the smallest scaled pivot (conditioning of the pass).
template <int k>
__device__ __noinline__ double dec_chol_transform(const double* S, const double* Wv, double* M) {
  double g2[k][k], dsc[k], rinv[k][k], R[k][k];
#pragma unroll
  for (int i = 0; i < k; ++i)
#pragma unroll
    for (int j = 0; j < k; ++j) {
      double s = 0.0;
#pragma unroll
      for (int p = 0; p < k; ++p)
#pragma unroll
        for (int q = 0; q < k; ++q) s = fma(Wv[p + k * i] * 0.5 * (S[p * 4 + q] + S[q * 4 + p]), Wv[q + k * j], s);
      g2[i][j] = s;
    }
#pragma unroll
  for (int i = 0; i < k; ++i) dsc[i] = g2[i][i] > 0.0 ? 1.0 / sqrt(g2[i][i]) : 0.0;
#pragma unroll
  for (int i = 0; i < k; ++i)
#pragma unroll
    for (int j = 0; j < k; ++j) { g2[i][j] *= dsc[i] * dsc[j]; R[i][j] = 0.0; rinv[i][j] = 0.0; }
  double pivmin = 1.0;
#pragma unroll
  for (int j = 0; j < k; ++j) {
#pragma unroll
    for (int i = 0; i <= j; ++i) {
      double s = g2[i][j];
#pragma unroll
      for (int q = 0; q < i; ++q) s -= R[q][i] * R[q][j];
      if (i < j) R[i][j] = R[i][i] > 0.0 ? s / R[i][i] : 0.0;
      else {
        pivmin = fmin(pivmin, s);
        R[j][j] = s > 1e-28 ? sqrt(s) : 0.0;
      }
    }
  }
#pragma unroll
  for (int j = 0; j < k; ++j) {
    rinv[j][j] = R[j][j] > 0.0 ? 1.0 / R[j][j] : 0.0;
#pragma unroll
    for (int i = j - 1; i >= 0; --i) {
      double s = 0.0;
#pragma unroll
      for (int q = i + 1; q <= j; ++q) s -= R[i][q] * rinv[q][j];
      rinv[i][j] = R[i][i] > 0.0 ? s / R[i][i] : 0.0;
    }
  }
#pragma unroll
  for (int p = 0; p < k; ++p)
#pragma unroll
    for (int j = 0; j < k; ++j) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q <= j; ++q) s = fma(Wv[p + k * q] * dsc[q], rinv[q][j], s);
      M[p * 4 + j] = s;
    }
  return pivmin;
}

template <int K>
__global__ void __launch_bounds__(kDecThreads, 1) k_decide(DecideArgs p) {
  griddep_wait();
  // an earlier mode of this speculative sweep already disagreed: its operands are garbage
  if (p.expect >= 0 && *reinterpret_cast<volatile int*>(p.spec_flag) != 0) return;
  extern __shared__ __align__(16) double sm[];
  __shared__ double red[64], resp[16 * 4], trpart[(kDecMaxA / 8) * kDecMaxSplit];
  __shared__ double Qs[48 * 8], Ms[16], Wvs[16], Hs[16], Ss[16], thetas[4];
  __shared__ int aoff[64];
  __shared__ int s_rk, s_reorth;
  __shared__ double s_dev;
  const int a = p.a, r = p.r, ldb = p.ldb;
  const int tid = threadIdx.x, lane = tid & 31, warp = dec_warp(), nw = blockDim.x >> 5;
  const int bcols = dec_bcols(r, K);
  const int ksplit = p.ksplit;
  double* Bs = sm;                                     // [U | X | 0]
  double* X = Bs + (size_t)ldb * r;
  double* Yp = Bs + (size_t)ldb * bcols;               // k-range partials of Y = C X (ksplit x K columns)
  double* Zs = Yp + (size_t)ldb * kDecMaxSplit * K;    // Z = P Y
  double* XW = Zs + (size_t)ldb * K;                   // Ritz vectors X Wv
  double* Qp = XW + (size_t)ldb * K;                   // gram partials (one 8 x 8 block per warp)
  long long tph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long tq = clock64();
#define DEC_T(i) { const long long tn_ = clock64(); tph[i] += tn_ - tq; tq = tn_; }

  // per-warp tasks of the three reduction shapes
  int kpU, kpXZ, kpX;
  const DecGramTask tkU = dec_gram_task(r, a, kpU);        // U^T B
  const DecGramTask tkXZ = dec_gram_task(2 * K, a, kpXZ);  // [X | Z]^T B
  const DecGramTask tkX = dec_gram_task(K, a, kpX);        // X^T B (re-orthonormalisation, guard)

  // stage U (one column per warp pass); zero the padding, X, Yp, Z, XW
  const int ncol_all = bcols + (kDecMaxSplit + 2) * K;
  for (int j = warp; j < ncol_all; j += nw) {
    double* col = sm + (size_t)ldb * j;
    const double* src = p.U + (size_t)a * (j < r ? j : 0);
    for (int i = lane; i < ldb; i += 32) col[i] = (j < r && i < a) ? __ldg(src + i) : 0.0;
  }
  // (m < 48: the columns of U; 48 + m: [X | Z]; 56 + m: XW)
  for (int m = tid; m < 64; m += blockDim.x)
    aoff[m] = m < 48 ? ldb * (m < r ? m : 0)
            : m < 48 + K ? (int)(X - sm) + ldb * (m - 48)
            : m < 48 + 2 * K ? (int)(Zs - sm) + ldb * (m - 48 - K)
            : m >= 56 && m < 56 + K ? (int)(XW - sm) + ldb * (m - 56) : 0;
  double tpart = 0.0;
  for (int i = tid; i < a; i += blockDim.x) tpart += __ldg(p.C + i + (size_t)a * i);
  const double trC = block_sum_all(tpart, red);
  if (tid == 0) { s_rk = -1; s_reorth = 0; s_dev = 0.0; thetas[0] = thetas[1] = thetas[2] = thetas[3] = 0.0; }
  __syncthreads();
  // start block: K columns of a pseudo-random Householder reflector I - 2 v v^T / v^T v
  // (as k_syev_top) in Yp[0]; the "boot" round below projects it onto range(P)
  // and orthonormalises it.  Old-old part of the append guard, max |U^T U - I|,
  // on DMMA (one lower 8 x 8 block pair per warp).
  double vpart = 0.0, vi = 0.0;
  if (tid < a) {
    unsigned long long h = 0x9E3779B97F4A7C15ull * (unsigned long long)(tid + 1);
    h ^= h >> 31; h *= 0xbf58476d1ce4e5b9ull; h ^= h >> 27;
    vi = (double)(h >> 11) * (1.0 / 9007199254740992.0) - 0.5;
    Zs[tid] = vi;
    vpart = vi * vi;
  }
  const double vv = block_sum_all(vpart, red);
  __syncthreads();
  if (tid < a) {
#pragma unroll
    for (int c = 0; c < K; ++c) {
      const int piv = (int)(((long long)c * a) / K);
      Yp[tid + (size_t)ldb * c] = (tid == piv ? 1.0 : 0.0) - 2.0 * vi * (Zs[piv] / vv);
    }
  }
  double dev_old = 0.0;
  {
    const int nrb8 = (r + 7) >> 3, npair = nrb8 * (nrb8 + 1) / 2, nk = (a + 3) >> 2;
    const int g = lane >> 2, t = lane & 3;
    for (int pr = warp; pr < npair; pr += nw) {
      int mb = 0, rem = pr;
      while (rem > mb) { rem -= mb + 1; ++mb; }
      const int nb = rem;  // nb <= mb
      const double* ap = Bs + (size_t)ldb * (mb * 8 + g) + t;
      const double* bp = Bs + (size_t)ldb * (nb * 8 + g) + t;
      double c0 = 0.0, c1 = 0.0, e0 = 0.0, e1 = 0.0;
      int ks = 0;
      for (; ks + 1 < nk; ks += 2) {
        dmma(c0, c1, ap[4 * ks], bp[4 * ks]);
        dmma(e0, e1, ap[4 * ks + 4], bp[4 * ks + 4]);
      }
      if (ks < nk) dmma(c0, c1, ap[4 * ks], bp[4 * ks]);
      const int m = mb * 8 + g, n0 = nb * 8 + 2 * t;
      if (m < r && n0 < r) dev_old = fmax(dev_old, fabs(c0 + e0 - (m == n0 ? 1.0 : 0.0)));
      if (m < r && n0 + 1 < r) dev_old = fmax(dev_old, fabs(c1 + e1 - (m == n0 + 1 ? 1.0 : 0.0)));
    }
    for (int o = 16; o > 0; o >>= 1) dev_old = fmax(dev_old, __shfl_xor_sync(0xffffffffu, dev_old, o));
    if (lane == 0) red[32 + warp] = dev_old;
  }
  __syncthreads();
  if (tid < a) Zs[tid] = 0.0;
  dev_old = 0.0;
  for (int w = 0; w < nw; ++w) dev_old = fmax(dev_old, red[32 + w]);

  const double delta = p.delta_src ? p.delta_mult * sqrt(*p.delta_src) : p.delta_mult;
  const long long kcap = p.kmax < a ? p.kmax : a;
  int state = 0, rank = 0, it = -1;  // it = -1: boot round (Y = the start block, no Rayleigh-Ritz)
  double trace = 0.0, tail = 0.0, prev_res = 1e300;
  int nsum = 1;  // partial buffers of Y in use
  DEC_T(0)
  for (; state == 0 && it < kDecIters; ++it) {
    const bool boot = it < 0;
    // T = U^T Y on DMMA (explicitly from the computed Y: the operator stays
    // symmetric on range(P) to eps |Y|, which the residual certificate needs)
    dec_gram(tkU, sm, aoff, r, Yp, ldb, K, nsum, ldb * K, Qp);
    __syncthreads();
    dec_gram_sum(Qp, r, K, kpU, Qs, tid, blockDim.x);
    __syncthreads();
    DEC_T(2)
    // Z = Y - U T (row-parallel)
    if (tid < a) {
      double z[K];
#pragma unroll
      for (int c = 0; c < K; ++c) {
        double s = Yp[tid + (size_t)ldb * c];
        for (int q = 1; q < nsum; ++q) s += Yp[tid + (size_t)ldb * (q * K + c)];
        z[c] = s;
      }
      for (int j = 0; j < r; ++j) {
        const double u = Bs[tid + (size_t)ldb * j];
#pragma unroll
        for (int c = 0; c < K; ++c) z[c] = fma(-u, Qs[j * 8 + c], z[c]);
      }
#pragma unroll
      for (int c = 0; c < K; ++c) Zs[tid + (size_t)ldb * c] = z[c];
    }
    __syncthreads();
    DEC_T(3)
    // [X | Z]^T Z: H = X^T Z, S = Z^T Z in one DMMA reduction
    dec_gram(tkXZ, sm, aoff + 48, 2 * K, Zs, ldb, K, 1, 0, Qp);
    __syncthreads();
    if (warp == 0) {
      dec_gram_sum(Qp, 2 * K, K, kpXZ, Qs, lane, 32);
      __syncwarp();
      if (lane == 0) {
#pragma unroll
        for (int i = 0; i < K; ++i)
#pragma unroll
          for (int j = 0; j < K; ++j) {
            Hs[i + K * j] = Qs[i * 8 + j];
            Ss[i * 4 + j] = Qs[(K + i) * 8 + j];
          }
        if (boot) {
#pragma unroll
          for (int i = 0; i < K; ++i)
#pragma unroll
            for (int j = 0; j < K; ++j) Wvs[i + K * j] = i == j ? 1.0 : 0.0;
        } else {
          thread_sym_eig4(Hs, K, thetas, Wvs);
          // rank from the Ritz values (lower bounds => rank can only be over-stated)
          double pre = 0.0;
          int rk = -1;
          for (int q = 0; q <= K; ++q) {
            if (q <= kcap && !(sqrt(fmax(trace - pre, 0.0)) > delta)) { rk = q; break; }
            if (q < K) pre += fmax(thetas[q], 0.0);
          }
          s_rk = rk;
        }
        const double pivmin = dec_chol_transform<K>(Ss, Wvs, Ms);
        s_reorth = pivmin < 0.25 ? 1 : 0;
      }
    }
    __syncthreads();
    DEC_T(4)
    // row-parallel: Ritz vectors X Wv, residual columns Z Wv - theta X Wv, X <- Z M
    {
      double d2[K];
#pragma unroll
      for (int j = 0; j < K; ++j) d2[j] = 0.0;
      if (tid < a) {
        double x[K], z[K];
#pragma unroll
        for (int c = 0; c < K; ++c) { x[c] = X[tid + (size_t)ldb * c]; z[c] = Zs[tid + (size_t)ldb * c]; }
#pragma unroll
        for (int j = 0; j < K; ++j) {
          double xw = 0.0, zw = 0.0, xn = 0.0;
#pragma unroll
          for (int c = 0; c < K; ++c) {
            xw = fma(x[c], Wvs[c + K * j], xw);
            zw = fma(z[c], Wvs[c + K * j], zw);
            xn = fma(z[c], Ms[c * 4 + j], xn);
          }
          const double d = zw - thetas[j] * xw;
          d2[j] = d * d;
          XW[tid + (size_t)ldb * j] = xw;
          X[tid + (size_t)ldb * j] = xn;
        }
      }
      if (!boot) {
#pragma unroll
        for (int j = 0; j < K; ++j) {
          const double s = warp_sum(d2[j]);
          if (lane == 0) resp[warp * 4 + j] = s;
        }
      }
    }
    __syncthreads();
    // decision (every thread evaluates the same numbers)
    if (!boot) {
      double resn[K];
#pragma unroll
      for (int j = 0; j < K; ++j) {
        double s = 0.0;
        for (int w = 0; w < nw; ++w) s += resp[w * 4 + j];
        resn[j] = sqrt(s);
      }
      const int rk = s_rk;
      const double tol = 64.0 * 2.220446049250313e-16 * fmax(thetas[0], 1e-300);
      double worst = 0.0;
      if (rk >= 1 && rk < K) {
        for (int q = 0; q < rk; ++q) worst = fmax(worst, resn[q]);
        if (worst <= tol || (worst <= 1e-12 * thetas[0] && worst >= 0.9 * prev_res)) {
          double pre2 = 0.0;
          for (int q = 0; q < rk; ++q) pre2 += thetas[q];
          rank = rk;
          tail = fmax(trace - pre2, 0.0);
          state = 1;
        }
      } else {
        worst = resn[0];
        if (it >= 3) state = 2;  // more kept directions than the block holds
      }
      prev_res = worst;
    }
    DEC_T(5)
    if (state) { ++it; break; }
    if (s_reorth) {  // ill-conditioned single pass (boot / early rounds): CholQR again
      dec_gram(tkX, sm, aoff + 48, K, X, ldb, K, 1, 0, Qp);
      __syncthreads();
      if (warp == 0) {
        dec_gram_sum(Qp, K, K, kpX, Qs, lane, 32);
        __syncwarp();
        if (lane == 0) {
          double Id[K * K];
#pragma unroll
          for (int i = 0; i < K; ++i)
#pragma unroll
            for (int j = 0; j < K; ++j) { Ss[i * 4 + j] = Qs[i * 8 + j]; Id[i + K * j] = i == j ? 1.0 : 0.0; }
          dec_chol_transform<K>(Ss, Id, Ms);
        }
      }
      __syncthreads();
      if (tid < a) {
        double x[K];
#pragma unroll
        for (int c = 0; c < K; ++c) x[c] = X[tid + (size_t)ldb * c];
#pragma unroll
        for (int j = 0; j < K; ++j) {
          double s = 0.0;
#pragma unroll
          for (int c = 0; c < K; ++c) s = fma(x[c], Ms[c * 4 + j], s);
          X[tid + (size_t)ldb * j] = s;
        }
      }
      __syncthreads();
    }
    // Y = C X (k-range partials); the first pass also carries C U for the trace
    if (boot) {
      switch ((r + K + 7) >> 3) {  // (one instantiation runs; the others cost no instruction fetch)
        case 1: dec_pass<1>(p.C, a, Bs, ldb, 0, r, r, K, ksplit, Yp, trpart); break;
        case 2: dec_pass<2>(p.C, a, Bs, ldb, 0, r, r, K, ksplit, Yp, trpart); break;
        case 3: dec_pass<3>(p.C, a, Bs, ldb, 0, r, r, K, ksplit, Yp, trpart); break;
        case 4: dec_pass<4>(p.C, a, Bs, ldb, 0, r, r, K, ksplit, Yp, trpart); break;
        case 5: dec_pass<5>(p.C, a, Bs, ldb, 0, r, r, K, ksplit, Yp, trpart); break;
        default: dec_pass<6>(p.C, a, Bs, ldb, 0, r, r, K, ksplit, Yp, trpart); break;
      }
      __syncthreads();
      // trace(G) = trace(C) - trace(U^T C U), partials in task order
      const int ntask = ((a + 7) >> 3) * ksplit;
      double s = 0.0;
      for (int q = lane; q < ntask; q += 32) s += trpart[q];
      s = warp_sum(s);
      trace = fmax(trC - s, 0.0);
      tail = trace;
      if (!(sqrt(trace) > delta) || kcap == 0) state = 1;  // everything fits under delta: rank 0
      DEC_T(1)
    } else {
      dec_pass<1>(p.C, a, Bs, ldb, r, 0, r, K, ksplit, Yp, nullptr);
      __syncthreads();
      DEC_T(6)
    }
    nsum = ksplit;
  }
  const bool ok = state == 1;
  // U_R = (I - U U^T) X Wv[:, :rank], normalised, sign rule -> UR and the appended core
  if (ok) {
    if (p.out != p.U)
      for (int j = warp; j < r; j += nw)
        for (int i = lane; i < a; i += 32) p.out[i + (size_t)a * j] = Bs[i + (size_t)ldb * j];
    if (rank > 0) {
      dec_gram(tkU, sm, aoff, r, XW, ldb, K, 1, 0, Qp);
      __syncthreads();
      dec_gram_sum(Qp, r, K, kpU, Qs, tid, blockDim.x);
      __syncthreads();
      if (tid < a) {
        double z[K];
#pragma unroll
        for (int c = 0; c < K; ++c) z[c] = XW[tid + (size_t)ldb * c];
        for (int j = 0; j < r; ++j) {
          const double u = Bs[tid + (size_t)ldb * j];
#pragma unroll
          for (int c = 0; c < K; ++c) z[c] = fma(-u, Qs[j * 8 + c], z[c]);
        }
#pragma unroll
        for (int c = 0; c < K; ++c) XW[tid + (size_t)ldb * c] = z[c];
      }
      __syncthreads();
      for (int j = warp; j < rank; j += nw) {
        double* col = XW + (size_t)ldb * j;
        double nn = 0.0, best = -1.0;
        int bi = a;
        for (int q = lane; q < a; q += 32) {
          const double u = col[q];
          nn = fma(u, u, nn);
          const double v = fabs(u);
          if (v > best) { best = v; bi = q; }
        }
        nn = warp_sum(nn);
        const double inv = 1.0 / sqrt(nn);
        for (int o = 16; o > 0; o >>= 1) {
          const double ob = __shfl_xor_sync(0xffffffffu, best, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
        }
        const double sgn = (col[bi] < 0.0) ? -inv : inv;
        __syncwarp();
        for (int q = lane; q < a; q += 32) {
          const double v = col[q] * sgn;
          col[q] = v;
          p.UR[q + (size_t)a * j] = v;
          p.out[q + (size_t)a * (r + j)] = v;
        }
      }
      __syncthreads();
      // guard of append_directions: max |[U U_R]^T [U U_R] - I| over all pairs:
      // old-old from the start of the kernel, U^T U_R and U_R^T U_R here
      dec_gram(tkU, sm, aoff, r, XW, ldb, K, 1, 0, Qp);
      __syncthreads();
      dec_gram_sum(Qp, r, K, kpU, Qs, tid, blockDim.x);
      __syncthreads();
      dec_gram(tkX, sm, aoff + 56, K, XW, ldb, K, 1, 0, Qp);
      __syncthreads();
      if (tid == 0) {
        double dev = dev_old;
        for (int j = 0; j < r; ++j)
          for (int c = 0; c < rank; ++c) dev = fmax(dev, fabs(Qs[j * 8 + c]));
        for (int i = 0; i < rank; ++i)
          for (int c = 0; c < rank; ++c) {
            double s = 0.0;
            for (int kp = 0; kp < kpX; ++kp) s += Qp[(size_t)kp * 64 + i * 8 + c];
            dev = fmax(dev, fabs(s - (i == c ? 1.0 : 0.0)));
          }
        s_dev = dev;
      }
      __syncthreads();
    }
  }
  DEC_T(7)
  if (tid == 0) {
    EigResult e{};
    for (int q = 0; q < 4; ++q) e.t_phase[q] = (tph[2 * q] & 0xffffffffll) | (tph[2 * q + 1] << 32);
    e.converged = ok ? 1 : 0;
    e.sweeps = it;  // (kDecIters: no convergence -- the host does not retry with a larger block)
    e.rank = rank;
    e.tail_sq = tail;
    e.delta = delta;
    e.lam_max = (ok && rank == 0) ? 0.0 : thetas[0];
    e.lam_min_kept = rank > 0 ? thetas[rank - 1] : 0.0;
    e.dev = s_dev;
    e.guard = (ok && rank > 0 && s_dev > 1e-10) ? 2 : 0;  // 2: the host runs k_append's correction
    *p.res = e;
    *p.trC = trC;
    if (p.log) *p.log = e;
    if (p.expect >= 0) {
      bool bad = !ok || rank != p.expect || e.guard != 0;
      if (rank > 0 && e.lam_min_kept < 1e-3 * trC) bad = true;  // raw-Gram guard (sweep())
      if (e.lam_max > 0.0 && (delta * delta < 1e-9 * e.lam_max || (rank > 0 && e.lam_min_kept < 1e-6 * e.lam_max)))
        bad = true;  // needs_accurate()
      if (bad) atomicOr(p.spec_flag, 1);
    }
    for (int j = 0; j < K; ++j) p.lam[j] = thetas[j];
  }
#undef DEC_T
}

}  // namespace ttg
