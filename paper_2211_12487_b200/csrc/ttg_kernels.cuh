// ttg_kernels.cuh — sm_100a kernels of the TT-ICE / TT-ICE* per-increment sweep.
//
// Every matrix is column-major ("first-index-fastest"), so an
// unfolding  cur_i (a_i x L_i)  is the raw buffer: column q is a_i contiguous
// doubles and the observation index is the slowest (observation o owns the
// contiguous column range [o*cpo, (o+1)*cpo)).
//
// FP64 tensor-core math is DMMA (`mma.sync.aligned.m8n8k4 .f64`, SASS
// DMMA.8x8x4): tcgen05 has no f64 kind.  Measured on this pool's B200:
// DMMA 37.0 TF/s, DFMA 33.7 TF/s, cuBLAS DGEMM 35.5 TF/s (profiles/r01_box_probe.log).
//
// Fragment layouts of m8n8k4 (row.col), lane = 4*g + t:
//   A (8x4):  A[g][t]          B (4x8): B[t][g]          C (8x8): C[g][2t], C[g][2t+1]
#pragma once
#include "ttg_pdl.cuh"
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace ttg {

constexpr int kTC = 64;        // columns of cur per smem tile
constexpr int kConsumerWarps = 8;                        // warp-specialised kernels: 8 consumers
constexpr int kSyrkThreads = (kConsumerWarps + 1) * 32;  // + 1 TMA producer warp
constexpr int kThreads = 256;  // 8 warps; warp w owns tile columns [8w, 8w+8)

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// mma.m16n8k16 f64 (4096 FMA per instruction; layout verified by
// tools/probe/mma16_layout.cu):  lane = 4g + t,
//   A (16x16): a[i] = A[g + 8(i&1)][t + 4(i>>1)]    B (16x8): b[i] = B[t + 4i][g]
//   C (16x8):  c[i] = C[g + 8(i>>1)][2t + (i&1)]
__device__ __forceinline__ void dmma16(double (&c)[4], const double (&a)[8], const double (&b)[4]) {
  asm("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
      "{%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]), "d"(b[1]),
        "d"(b[2]), "d"(b[3]));
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int src_size = valid ? 8 : 0;  // 0 => zero-fill
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_size));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async16z(void* smem, const void* gmem, bool valid) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;\n" ::); }
__device__ __forceinline__ void cp_async_wait_0() { asm volatile("cp.async.wait_group 0;\n" ::); }
// wait until at most n (runtime, 0..4) cp.async groups of this thread are pending
__device__ __forceinline__ void cp_async_wait_n(int n) {
  switch (n) {
    case 0: asm volatile("cp.async.wait_group 0;\n" ::); break;
    case 1: asm volatile("cp.async.wait_group 1;\n" ::); break;
    case 2: asm volatile("cp.async.wait_group 2;\n" ::); break;
    case 3: asm volatile("cp.async.wait_group 3;\n" ::); break;
    default: asm volatile("cp.async.wait_group 4;\n" ::); break;
  }
}

// Leading dimension (in doubles) for an smem column-major tile with `rows`
// rows: >= rows and == 4 (mod 16), which makes both m8n8k4 fragment patterns
// (8 rows x 4 cols and 4 rows x 8 cols) hit every bank exactly twice.
__host__ __device__ inline int smem_ld(int rows) {
  int ld = rows;
  int m = ((4 - ld) % 16 + 16) % 16;
  return ld + m;
}

__host__ __device__ inline int round_up(int x, int m) { return (x + m - 1) / m * m; }

// ---------------------------------------------------------------------------
// Tile loader: TC columns of X (a x L) starting at column q0 into smem T with
// leading dimension ldt.  Rows a..a8 are pre-zeroed by the caller and never
// touched.  Columns past L and columns of unselected observations are
// zero-filled (cp.async src-size 0).
// ---------------------------------------------------------------------------
struct TileSrc {
  const double* X;
  int a;
  long long L;
  const uint8_t* sel;     // per-observation selection mask (nullable)
  long long cols_per_obs;
};

__device__ __forceinline__ void load_tile_async(const TileSrc& s, long long q0, double* T, int ldt) {
  const int n = s.a * kTC;
  // incremental (row, col) walk avoids a division per element
  int e = threadIdx.x;
  int col = e / s.a;
  int row = e - col * s.a;
  const int step_c = kThreads / s.a;
  const int step_r = kThreads - step_c * s.a;
  const double* base = s.X + (long long)s.a * q0;
  for (; e < n; e += kThreads) {
    long long qc = q0 + col;
    bool valid = qc < s.L;
    if (valid && s.sel) valid = s.sel[qc / s.cols_per_obs] != 0;
    cp_async8(&T[row + ldt * col], valid ? (const void*)(base + e) : (const void*)s.X, valid);
    row += step_r;
    col += step_c;
    if (row >= s.a) {
      row -= s.a;
      ++col;
    }
  }
}

// ---------------------------------------------------------------------------
// TMA tile pipeline (sm_100a cp.async.bulk + mbarrier).  A tile = kTC
// consecutive columns of X (a x L, column-major): each column is one
// contiguous a*8-byte run, copied by one bulk instruction into the padded smem
// tile (ld = ldt).  Warp 0 is the producer: it evaluates the 64 column flags
// (inside L, observation selected) once per tile, posts the expected bytes on
// the buffer's mbarrier, issues the bulk copies and zero-fills the invalid
// columns.  Requires a even (16-byte runs); odd a falls back to cp.async.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
// 1024-byte aligned start inside a dynamic shared array (128-byte swizzled
// TMA boxes need it).  Pointer arithmetic on the __shared__ array keeps the
// address space visible to the compiler (LDS, not generic LD): a round trip
// through uintptr_t would turn every tile access into a generic load.
__device__ __forceinline__ double* align1024(double* p) {
  return p + (((1024u - (smem_u32(p) & 1023u)) & 1023u) >> 3);
}
// Same alignment through a generic pointer (the compiler emits generic LD
// for the tile reads).  Kept for k_syrk_kx only: measured 5 % faster there
// than the LDS form (1.17 vs 1.23 ms at a = 64; the DMMA issue interleaves
// better with the longer-latency loads), although ncu counts 2x wavefronts.
__device__ __forceinline__ double* align1024_generic(double* p) {
  return reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
#ifdef TTG_MBAR_TEST
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
#else
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
#endif
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* tm) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(tm)) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }

// Issue the loads of tile [q0, q0+kTC) into T.  Uniform call by all threads.
// tma: bulk path (a even); else cp.async 8-byte path (caller commits/waits).
__device__ __forceinline__ void tile_issue(const TileSrc& s, long long q0, double* T, int ldt, uint64_t* bar,
                                           bool tma) {
  if (!tma) {
    load_tile_async(s, q0, T, ldt);
    return;
  }
  if ((threadIdx.x >> 5) != 0) return;
  const int lane = threadIdx.x & 31;
  bool v[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const long long q = q0 + lane + 32 * h;
    bool ok = q < s.L;
    if (ok && s.sel) ok = s.sel[q / s.cols_per_obs] != 0;
    v[h] = ok;
  }
  const unsigned m0 = __ballot_sync(0xffffffffu, v[0]), m1 = __ballot_sync(0xffffffffu, v[1]);
  const unsigned nvalid = __popc(m0) + __popc(m1);
  const unsigned colbytes = (unsigned)s.a * 8u;
  fence_proxy_async();  // earlier generic-proxy writes to this buffer precede the async copies
  if (lane == 0) mbar_expect_tx(bar, nvalid * colbytes);
  __syncwarp();
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int c = lane + 32 * h;
    if (v[h]) {
      bulk_g2s(T + (size_t)ldt * c, s.X + (size_t)s.a * (q0 + c), colbytes, bar);
    } else {
      for (int r = 0; r < s.a; ++r) T[r + (size_t)ldt * c] = 0.0;
    }
  }
}

// In-place residual of the warp's 8 tile columns: T_w -= U (U^T T_w), with U
// given as DMMA A-fragments (k_make_frags); Pw is the warp's r8 x 8 scratch.
__device__ __forceinline__ void tile_residual(double* T, int ldt, double* Pw, int ldp, const double* UTf,
                                              const double* Uf, int KA, int KR, int MR, int nb) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int c0 = warp * 8;
  // P = U^T T_w (r8 x 8): 4 m-blocks in flight (independent DMMA chains)
  for (int mb0 = 0; mb0 < MR; mb0 += 4) {
    double q[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
    for (int kb = 0; kb < KA; ++kb) {
      const double bv = T[(kb * 4 + t) + ldt * (c0 + g)];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (mb0 + u < MR) dmma(q[u][0], q[u][1], UTf[((long long)(mb0 + u) * KA + kb) * 32 + lane], bv);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (mb0 + u < MR) {
        Pw[((mb0 + u) * 8 + g) + ldp * (2 * t)] = q[u][0];
        Pw[((mb0 + u) * 8 + g) + ldp * (2 * t + 1)] = q[u][1];
      }
  }
  __syncwarp();
  // T_w -= U P: 4 row-blocks in flight
  for (int ib0 = 0; ib0 < nb; ib0 += 4) {
    double q[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
    for (int sb = 0; sb < KR; ++sb) {
      const double bv = Pw[(sb * 4 + t) + ldp * g];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (ib0 + u < nb) dmma(q[u][0], q[u][1], Uf[((long long)(ib0 + u) * KR + sb) * 32 + lane], bv);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (ib0 + u < nb) {
        T[((ib0 + u) * 8 + g) + ldt * (c0 + 2 * t)] -= q[u][0];
        T[((ib0 + u) * 8 + g) + ldt * (c0 + 2 * t + 1)] -= q[u][1];
      }
  }
  __syncwarp();
}

// ---------------------------------------------------------------------------
// Sum of squares of an smem tile (rows x kTC, ld) -> block total on thread 0.
// Fixed thread/element assignment and tree: deterministic.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double tile_sumsq(const double* T, int rows, int ld, double* red8) {
  double s = 0.0;
  for (int e = threadIdx.x; e < rows * kTC; e += kThreads) {
    const int c = e / rows, r = e - c * rows;
    const double v = T[r + ld * c];
    s = fma(v, v, s);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) red8[warp] = s;
  __syncthreads();
  double tot = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kThreads / 32; ++w) tot += red8[w];
  return tot;
}

// Pre-projection of the warp's 8 tile columns: the current unfolding's column
// is (I_nblk (x) Psi^T) applied to the source column (rows As*nblk):
//   Tc[p + rc*j][c] = sum_k Psi[k][p] * Ts[k + As*j][c]
__device__ __forceinline__ void tile_preproject(const double* Ts, int lds, double* Tc, int ldt, const double* PsiTf,
                                                int As, int nblk, int rc, int MRC, int KS) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int c0 = warp * 8;
  for (int mb = 0; mb < MRC; ++mb) {
    const int row = mb * 8 + g;
    for (int j0 = 0; j0 < nblk; j0 += 4) {
      double q[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
      for (int kb = 0; kb < KS; ++kb) {
        const double av = PsiTf[((long long)mb * KS + kb) * 32 + lane];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (j0 + u < nblk) dmma(q[u][0], q[u][1], av, Ts[(As * (j0 + u) + kb * 4 + t) + lds * (c0 + g)]);
      }
      if (row < rc) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (j0 + u < nblk) {
            Tc[(row + rc * (j0 + u)) + ldt * (c0 + 2 * t)] = q[u][0];
            Tc[(row + rc * (j0 + u)) + ldt * (c0 + 2 * t + 1)] = q[u][1];
          }
      }
    }
  }
  __syncwarp();
}

// ---------------------------------------------------------------------------
// Fused (pre-projection +) residual + Gram:  for every selected column x of
// the current unfolding cur_i (a x L):  r = x - U (U^T x);  G += r r^T.
// WBR x WBC 8x8 blocks per warp (warp grid 4 x 2) -> one 8*4*WBR super-tile
// (I, J), I >= J, per blockIdx.y; a grid-stride set of 64-column tiles per
// blockIdx.x; per-CTA partial written for a fixed-order reduction.
// PRE: the tile is loaded from the source S (rows As*nblk) and projected by
//      Psi (I_nblk (x) Psi^T) into the cur tile (mode i read straight from the
//      buffer of mode i-1 or earlier, no intermediate in HBM).
// DB : cp.async double-buffered source tiles (else single-buffered, for
//      a8 up to 256).
// U enters as pre-swizzled DMMA fragments read with coalesced 256-byte loads.
// ---------------------------------------------------------------------------
struct GramArgs {
  TileSrc src;        // tile source: rows src.a (= As*nblk when PRE, = a otherwise)
  int a, a8;          // rows of the current unfolding
  int ldt, lds, ldp;
  int As, nblk, rc, MRC, KS;  // pre-projection geometry (PRE)
  const double* PsiTf;        // A-fragments of Psi^T: [MRC][KS][32]
  const double* UTf;  // A-fragments of U^T: [r8/8][a8/4][32]
  const double* Uf;   // A-fragments of U:   [a8/8][r8/4][32]
  int r8;             // 0 => no residual (empty basis)
  double* partials;   // [gridDim.y][gridDim.x][SBD*SBD]
  double* tsumsq;     // per-tile sum of squares of the source tile (nullable)
  long long n_tiles;
  int frag_smem;      // stage UTf / Uf / PsiTf in shared memory
  int r_old;          // host-side accounting only
  double sel_frac;    // host-side accounting only
};

template <int WBR, int WBC, bool PRE, bool DB>
__global__ void __launch_bounds__(kThreads) k_gram_resid(GramArgs p) {
  griddep_wait();
  extern __shared__ __align__(16) double smem[];
  __shared__ double red8[kThreads / 32];
  __shared__ __align__(8) uint64_t bars[2];
  constexpr int SB = 4 * WBR;  // == 2*WBC blocks per super-tile side
  constexpr int SBD = 8 * SB;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int ldt = p.ldt, ldp = p.ldp;
  const int lds = PRE ? p.lds : ldt;
  const bool tma = (p.src.a & 1) == 0;
  // PRE: one source buffer (prefetched right after the pre-projection) + cur tile.
  // !PRE: DB ? two tiles : one tile (the residual is computed in place).
  const int nsrc = PRE ? 1 : (DB ? 2 : 1);
  double* S0 = smem;
  double* S1 = (!PRE && DB) ? S0 + (size_t)lds * kTC : S0;
  double* Tc = PRE ? S0 + (size_t)lds * kTC : nullptr;
  double* Pw0 = S0 + (size_t)nsrc * lds * kTC + (PRE ? (size_t)ldt * kTC : 0);
  double* Pw = Pw0 + warp * ldp * 8;
  double* fr = Pw0 + 8 * ldp * 8;  // fragment staging (when p.frag_smem)
  const int n_zero = (int)((nsrc * lds + (PRE ? ldt : 0)) * kTC);

  int I = 0, J = blockIdx.y;
  while (J > I) { J -= I + 1; ++I; }
  const int row_blk0 = I * SB + (warp >> 1) * WBR;  // in 8-row blocks
  const int col_blk0 = J * SB + (warp & 1) * WBC;
  const int nb = p.a8 >> 3;
  const int KA = p.a8 >> 2, KR = p.r8 >> 2, MR = p.r8 >> 3;

  const double* UTf = p.UTf;
  const double* Uf = p.Uf;
  const double* PsiTf = p.PsiTf;
  if (p.frag_smem) {  // stage the (small) fragment arrays once per CTA
    const int n1 = MR * KA * 32, n2 = nb * KR * 32, n3 = PRE ? p.MRC * p.KS * 32 : 0;
    for (int i = threadIdx.x; i < n1; i += kThreads) fr[i] = p.UTf[i];
    for (int i = threadIdx.x; i < n2; i += kThreads) fr[n1 + i] = p.Uf[i];
    for (int i = threadIdx.x; i < n3; i += kThreads) fr[n1 + n2 + i] = p.PsiTf[i];
    UTf = fr;
    Uf = fr + n1;
    PsiTf = fr + n1 + n2;
  }
  for (int i = threadIdx.x; i < n_zero; i += kThreads) smem[i] = 0.0;  // padded rows stay zero
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
  }
  __syncthreads();
  unsigned phase[2] = {0u, 0u};

  double acc[WBR][WBC][2];
#pragma unroll
  for (int i = 0; i < WBR; ++i)
#pragma unroll
    for (int j = 0; j < WBC; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // early-prefetch scheme (PRE, or DB): the first tile is issued before the loop
  const bool pre_issue = PRE ? tma : DB;
  long long tile = blockIdx.x;
  if (pre_issue) {
    if (tile < p.n_tiles) tile_issue(p.src, tile * kTC, S0, lds, &bars[0], tma);
    if (!tma) cp_async_commit();
  }
  int buf = 0;
  for (; tile < p.n_tiles; tile += gridDim.x) {
    const long long nxt = tile + gridDim.x;
    double* Ssrc = (!PRE && DB && buf) ? S1 : S0;
    const int cb = (!PRE && DB) ? buf : 0;
    if (!PRE && DB) {
      double* Sn = buf ? S0 : S1;
      if (nxt < p.n_tiles) tile_issue(p.src, nxt * kTC, Sn, lds, &bars[buf ^ 1], tma);
      if (!tma) {
        cp_async_commit();
        cp_async_wait_1();
      }
    } else if (!pre_issue) {
      tile_issue(p.src, tile * kTC, S0, lds, &bars[0], tma);
      if (!tma) {
        cp_async_commit();
        cp_async_wait_0();
      }
    }
    if (tma) {
      mbar_wait(&bars[cb], phase[cb]);
      phase[cb] ^= 1u;
    }
    __syncthreads();
    if (p.tsumsq) {
      const double ts = tile_sumsq(Ssrc, p.src.a, lds, red8);
      if (threadIdx.x < kConsumerWarps) p.tsumsq[tile * kConsumerWarps + threadIdx.x] = threadIdx.x == 0 ? ts : 0.0;
    }
    double* T = Ssrc;
    if (PRE) {
      tile_preproject(Ssrc, lds, Tc, ldt, PsiTf, p.As, p.nblk, p.rc, p.MRC, p.KS);
      T = Tc;
      __syncthreads();
      // the source buffer is free: fetch the next tile while residual + Gram run
      if (tma && nxt < p.n_tiles) tile_issue(p.src, nxt * kTC, S0, lds, &bars[0], tma);
    }
    if (p.r8 > 0) {
      tile_residual(T, ldt, Pw, ldp, UTf, Uf, KA, KR, MR, nb);
      __syncthreads();
    }
    // G(super-tile) += T T^T over the tile's 64 columns
#pragma unroll 4
    for (int k0 = 0; k0 < kTC; k0 += 4) {
      double af[WBR], bf[WBC];
#pragma unroll
      for (int i = 0; i < WBR; ++i) {
        const int rb = row_blk0 + i;
        af[i] = (rb < nb) ? T[(rb * 8 + g) + ldt * (k0 + t)] : 0.0;
      }
#pragma unroll
      for (int j = 0; j < WBC; ++j) {
        const int cb2 = col_blk0 + j;
        bf[j] = (cb2 < nb) ? T[(cb2 * 8 + g) + ldt * (k0 + t)] : 0.0;
      }
#pragma unroll
      for (int i = 0; i < WBR; ++i)
#pragma unroll
        for (int j = 0; j < WBC; ++j)
          if (col_blk0 + j <= row_blk0 + i)  // lower triangle only (the reduction reads row >= col)
            dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncthreads();
    buf ^= 1;
  }
  if (!tma) cp_async_wait_0();

  double* out = p.partials + ((long long)blockIdx.y * gridDim.x + blockIdx.x) * SBD * SBD;
#pragma unroll
  for (int i = 0; i < WBR; ++i)
#pragma unroll
    for (int j = 0; j < WBC; ++j) {
      const int r = ((warp >> 1) * WBR + i) * 8 + g;
      const int c = ((warp & 1) * WBC + j) * 8 + 2 * t;
      out[r + SBD * c] = acc[i][j][0];
      out[r + SBD * (c + 1)] = acc[i][j][1];
    }
}


// ---------------------------------------------------------------------------
// SYRK of the (selected) columns of X (a x L, column-major), any a:
//   C = sum_q x_q x_q^T      (the raw Gram; the residual projector is applied
//                             on the a x a side, see gram_raw_src in ttg.cu)
// blockIdx.y -> super-tile (I, J), I >= J, of SBD = 8*4*WBR rows; each CTA
// loads only the row slices I (and J) of every column with one TMA bulk copy
// per (column, slice) into an NST-deep ring of stages (mbarrier per stage),
// and accumulates the lower-triangle 8x8 blocks in registers (DMMA).
// ---------------------------------------------------------------------------
constexpr int kMaxStages = 4;

struct SyrkArgs {
  const double* X;
  int a, a8;
  long long L;
  const uint8_t* sel;
  long long cpo;
  int ldt;            // smem leading dimension of one slice tile
  int nst;            // ring stages (1..kMaxStages)
  double* partials;   // [gridDim.y][gridDim.x][SBD*SBD]
  double* tsumsq;     // per-tile sum of squares (only with a single full-height slice)
  long long n_tiles;
};

// warp 0: issue the (1 or 2) row slices of tile q0 into Ti (and Tj), one barrier
__device__ __forceinline__ void syrk_issue(const SyrkArgs& p, long long q0, int ri0, int nri, double* Ti, int rj0,
                                           int nrj, double* Tj, uint64_t* bar) {
  if ((threadIdx.x >> 5) != 0) return;
  const int lane = threadIdx.x & 31;
  bool v[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const long long q = q0 + lane + 32 * h;
    bool ok = q < p.L;
    if (ok && p.sel) ok = p.sel[q / p.cpo] != 0;
    v[h] = ok;
  }
  const unsigned nvalid = __popc(__ballot_sync(0xffffffffu, v[0])) + __popc(__ballot_sync(0xffffffffu, v[1]));
  const unsigned bytes = (unsigned)(nri + (Tj ? nrj : 0)) * 8u;
  fence_proxy_async();
  if (lane == 0) mbar_expect_tx(bar, nvalid * bytes);
  __syncwarp();
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int c = lane + 32 * h;
    const double* col = p.X + (size_t)p.a * (q0 + c);
    if (v[h]) {
      bulk_g2s(Ti + (size_t)p.ldt * c, col + ri0, (unsigned)nri * 8u, bar);
      if (Tj) bulk_g2s(Tj + (size_t)p.ldt * c, col + rj0, (unsigned)nrj * 8u, bar);
    } else {
      for (int r = 0; r < nri; ++r) Ti[r + (size_t)p.ldt * c] = 0.0;
      if (Tj)
        for (int r = 0; r < nrj; ++r) Tj[r + (size_t)p.ldt * c] = 0.0;
    }
  }
}

// Warp-specialised SYRK: warps 0..7 consume, warp 8 produces (TMA).  Each
// consumer warp owns up to MAXT 2x2 tiles of 8x8 blocks from the lower
// triangle of the super-tile (diagonal tiles also compute their upper block).
// full[s] / empty[s] mbarriers per ring stage; no block-wide barrier in the
// main loop.

template <int MAXT, int NCW = kConsumerWarps>
__global__ void __launch_bounds__((NCW + 1) * 32) k_syrk(SyrkArgs p) {
  griddep_wait();
  extern __shared__ __align__(16) double smem[];
  __shared__ __align__(8) uint64_t full[kMaxStages], empty[kMaxStages];
  __shared__ double red8[kConsumerWarps + 1];
  constexpr int SBD = 128;  // super-tile rows (16 blocks)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int ldt = p.ldt, nst = p.nst;
  int I = 0, J = blockIdx.y;
  while (J > I) { J -= I + 1; ++I; }
  const bool two = I != J;
  const int ri0 = I * SBD, nri = min(SBD, p.a - ri0);
  const int rj0 = J * SBD, nrj = min(SBD, p.a - rj0);
  const int per_stage = (two ? 2 : 1) * ldt * kTC;
  for (int i = threadIdx.x; i < nst * per_stage; i += blockDim.x) smem[i] = 0.0;  // padded rows stay zero
  if (threadIdx.x == 0)
    for (int s = 0; s < nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
  __syncthreads();
  auto Ti_of = [&](int s) { return smem + (size_t)s * per_stage; };
  auto Tj_of = [&](int s) { return two ? smem + (size_t)s * per_stage + (size_t)ldt * kTC : smem + (size_t)s * per_stage; };

  if (warp == NCW) {  // ---- producer ----
    int it = 0;
    for (long long tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x, ++it) {
      const int st = it % nst;
      if (it >= nst) mbar_wait(&empty[st], (unsigned)(((it / nst) - 1) & 1));
      // syrk_issue is written for warp 0: re-base the warp index
      const long long q0 = tile * kTC;
      bool v[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const long long q = q0 + lane + 32 * h;
        bool ok = q < p.L;
        if (ok && p.sel) ok = p.sel[q / p.cpo] != 0;
        v[h] = ok;
      }
      const unsigned nvalid = __popc(__ballot_sync(0xffffffffu, v[0])) + __popc(__ballot_sync(0xffffffffu, v[1]));
      const unsigned bytes = (unsigned)(nri + (two ? nrj : 0)) * 8u;
      double* Ti = Ti_of(st);
      double* Tj = two ? Tj_of(st) : nullptr;
      // zero-fill first: the arrive below releases these generic writes
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = lane + 32 * h;
        if (!v[h]) {
          for (int r = 0; r < nri; ++r) Ti[r + (size_t)ldt * c] = 0.0;
          if (Tj)
            for (int r = 0; r < nrj; ++r) Tj[r + (size_t)ldt * c] = 0.0;
        }
      }
      __syncwarp();
      fence_proxy_async();
      if (lane == 0) mbar_expect_tx(&full[st], nvalid * bytes);
      __syncwarp();
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = lane + 32 * h;
        const double* col = p.X + (size_t)p.a * (q0 + c);
        if (v[h]) {
          bulk_g2s(Ti + (size_t)ldt * c, col + ri0, (unsigned)nri * 8u, &full[st]);
          if (Tj) bulk_g2s(Tj + (size_t)ldt * c, col + rj0, (unsigned)nrj * 8u, &full[st]);
        }
      }
    }
    return;
  }

  // ---- consumers: 2x2 tiles of the lower triangle, assigned round-robin ----
  const int nbi = (nri + 7) >> 3, nbj = (nrj + 7) >> 3;
  const int tI = (nbi + 1) >> 1, tJ = (nbj + 1) >> 1;  // 2x2-block tiles per side
  const int ntiles = two ? tI * tJ : tI * (tI + 1) / 2;
  // tile idx = warp + 8u -> (ta, tb), lower-triangular row-major when !two.
  // Fully unrolled: the per-tile smem offsets stay in registers.
  int offA0[MAXT], offA1[MAXT], offB0[MAXT], offB1[MAXT];
  bool okA1[MAXT], okB1[MAXT], live[MAXT];
#pragma unroll
  for (int u = 0; u < MAXT; ++u) {
    const int idx = warp + NCW * u;
    live[u] = idx < ntiles;
    int ta = 0, tb = 0;
    if (two) {
      ta = idx / max(tJ, 1);
      tb = idx - ta * max(tJ, 1);
    } else {
      ta = (int)((sqrtf(8.0f * idx + 1.0f) - 1.0f) * 0.5f);
      while ((ta + 1) * (ta + 2) / 2 <= idx) ++ta;
      while (ta * (ta + 1) / 2 > idx) --ta;
      tb = idx - ta * (ta + 1) / 2;
    }
    const int bi = 2 * ta, bj = 2 * tb;
    offA0[u] = (bi * 8 + g) + ldt * t;
    offA1[u] = ((bi + 1) * 8 + g) + ldt * t;
    offB0[u] = (bj * 8 + g) + ldt * t;
    offB1[u] = ((bj + 1) * 8 + g) + ldt * t;
    okA1[u] = bi + 1 < nbi;
    okB1[u] = bj + 1 < nbj;
  }
  double acc[MAXT][2][2][2];
#pragma unroll
  for (int u = 0; u < MAXT; ++u)
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
      for (int y = 0; y < 2; ++y) acc[u][x][y][0] = acc[u][x][y][1] = 0.0;
  double tsq_acc = 0.0;
  int it = 0;
  for (long long tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x, ++it) {
    const int st = it % nst;
    mbar_wait(&full[st], (unsigned)((it / nst) & 1));
    const double* Ti = Ti_of(st);
    const double* Tj = Tj_of(st);
    if (p.tsumsq) {  // per-(tile, 8 virtual warps) sums of squares (single full-height slice only)
      for (int v = warp; v < kConsumerWarps; v += NCW) {
        double sq = 0.0;
        for (int e = lane + 32 * v; e < nri * kTC; e += 32 * kConsumerWarps) {
          const int c = e / nri, r = e - c * nri;
          const double vv = Ti[r + ldt * c];
          sq = fma(vv, vv, sq);
        }
        sq = warp_sum(sq);
        if (lane == 0) p.tsumsq[tile * kConsumerWarps + v] = sq;
      }
    }
#pragma unroll
    for (int u = 0; u < MAXT; ++u) {
      if (!live[u]) continue;  // warp-uniform
#pragma unroll 4
      for (int k0 = 0; k0 < kTC; k0 += 4) {
        const int ko = ldt * k0;
        const double a0 = Ti[offA0[u] + ko];
        const double a1 = okA1[u] ? Ti[offA1[u] + ko] : 0.0;
        const double b0 = Tj[offB0[u] + ko];
        const double b1 = okB1[u] ? Tj[offB1[u] + ko] : 0.0;
        dmma(acc[u][0][0][0], acc[u][0][0][1], a0, b0);
        dmma(acc[u][0][1][0], acc[u][0][1][1], a0, b1);
        dmma(acc[u][1][0][0], acc[u][1][0][1], a1, b0);
        dmma(acc[u][1][1][0], acc[u][1][1][1], a1, b1);
      }
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&empty[st])) : "memory");
  }
  double* out = p.partials + ((long long)blockIdx.y * gridDim.x + blockIdx.x) * SBD * SBD;
#pragma unroll
  for (int u = 0; u < MAXT; ++u) {
    if (!live[u]) continue;
    const int rI = offA0[u] - ldt * t - g, rJ = offB0[u] - ldt * t - g;  // first row of the tile
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
      for (int y = 0; y < 2; ++y) {
        const int r = rI + x * 8 + g;
        const int c = rJ + y * 8 + 2 * t;
        out[r + SBD * c] = acc[u][x][y][0];
        out[r + SBD * (c + 1)] = acc[u][x][y][1];
      }
  }
}

// K-split SYRK for a8 = 8 NBK <= 64 (one super-tile): every consumer warp
// accumulates ALL NBK(NBK+1)/2 lower 8x8 blocks (m8n8k4) over its own 8
// columns of each 64-column tile.  The m8n8k4 A and B fragments of row block
// b are the same value per lane (X[8b+g][k+t]), so a k-step is NBK
// shared-memory loads for NBK(NBK+1)/2 DMMAs, every warp does the same work
// (no triangle-tiling imbalance, no padded 16x16 tiles: 36 blocks for a = 64
// instead of 40), and the accumulators give the DMMA pipe ample independent
// work.  Tiles arrive by tensor-map TMA (16 x 64 boxes, 128-byte swizzle; one
// instruction per 8 KB box, rows >= a zero-filled); since a Gram is a sum
// over k, lane t of warp w reads column 8w + 2t + h at sub-step h (k permuted),
// which makes the fragment loads conflict-free under the swizzle.
// Unselected tiles (selection is tile-aligned) are skipped by producer and
// consumers alike.  One CTA per SM (registers).  The 8 warps' partial Grams
// are summed in shared memory in warp order (deterministic) and written as one
// SBD x SBD partial per CTA (gram_reduce layout 0).
template <int NBK>
__global__ void __launch_bounds__((kConsumerWarps + 1) * 32, 1) k_syrk_kx(const __grid_constant__ CUtensorMap tm,
                                                                          SyrkArgs p) {
  griddep_wait();
  constexpr int NBL = NBK * (NBK + 1) / 2;
  constexpr int NCW = kConsumerWarps;
  constexpr int SBD = 128;
  constexpr int NBOX = (NBK + 1) / 2;
  constexpr int BOX = 16 * kTC;
  constexpr int STAGE = NBOX * BOX;
  extern __shared__ __align__(1024) double smem_raw[];
  __shared__ __align__(8) uint64_t full[kMaxStages + 4], empty[kMaxStages + 4];
  double* smem = align1024_generic(smem_raw);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int nst = p.nst;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  auto selected = [&](long long tile) {
    return p.sel == nullptr || p.sel[(tile * kTC) / p.cpo] != 0;
  };

  if (warp == NCW) {  // ---- producer ----
    if (lane == 0) {
      tma_prefetch_desc(&tm);
      int it = 0, s = 0;
      for (long long tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x) {
        if (!selected(tile)) continue;
        if (it >= nst) mbar_wait(&empty[s], (unsigned)(((it / nst) - 1) & 1));
        mbar_expect_tx(&full[s], (unsigned)STAGE * 8u);
#pragma unroll
        for (int b = 0; b < NBOX; ++b) tma_load_2d(smem + s * STAGE + b * BOX, &tm, 16 * b, (int)(tile * kTC), &full[s]);
        ++it;
        if (++s == nst) s = 0;
      }
    }
    return;
  }

  // ---- consumers ----
  double acc[NBL][2];
#pragma unroll
  for (int u = 0; u < NBL; ++u) acc[u][0] = acc[u][1] = 0.0;
  int off[2][2];  // [h][b & 1]
  {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      // k column 2t + h of the warp's 8: each half-warp (g < 4 / g >= 4)
      // then covers 16 distinct 8-byte banks under the swizzle
      const int c = 8 * warp + 2 * t + h;
#pragma unroll
      for (int bp = 0; bp < 2; ++bp) off[h][bp] = c * 16 + ((((4 * bp + (g >> 1)) ^ (c & 7))) << 1) + (g & 1);
    }
  }
  int st = 0;
  unsigned ph = 0;
  for (long long tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x) {
    if (!selected(tile)) continue;
    mbar_wait(&full[st], ph);
    const double* Ti = smem + st * STAGE;
    if (p.tsumsq) {  // per-(tile, 8-column group) sums of squares: group = this warp's columns
      double sq = 0.0;
#pragma unroll
      for (int b = 0; b < NBOX; ++b)
#pragma unroll
        for (int e = lane; e < 128; e += 32) {
          const double vv = Ti[b * BOX + 128 * warp + e];
          sq = fma(vv, vv, sq);
        }
      sq = warp_sum(sq);
      if (lane == 0) p.tsumsq[tile * kConsumerWarps + warp] = sq;
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double f[NBK];
#pragma unroll
      for (int b = 0; b < NBK; ++b) f[b] = Ti[(b >> 1) * BOX + off[h][b & 1]];
      int u = 0;
#pragma unroll
      for (int bi = 0; bi < NBK; ++bi)
#pragma unroll
        for (int bj = 0; bj <= bi; ++bj, ++u) dmma(acc[u][0], acc[u][1], f[bi], f[bj]);
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&empty[st])) : "memory");
    if (++st == nst) {
      st = 0;
      ph ^= 1u;
    }
  }
  // ordered cross-warp sum in shared memory (the ring is idle: every stage was consumed)
  double* buf = smem;  // 8 NBK x 8 NBK, ld 8 NBK
  constexpr int LD = 8 * NBK;
  for (int w = 0; w < NCW; ++w) {
    asm volatile("bar.sync 1, %0;\n" ::"r"(NCW * 32) : "memory");
    if (warp == w) {
      int u = 0;
#pragma unroll
      for (int bi = 0; bi < NBK; ++bi)
#pragma unroll
        for (int bj = 0; bj <= bi; ++bj, ++u) {
          double* e = buf + (8 * bi + g) + LD * (8 * bj + 2 * t);
          if (w == 0) {
            e[0] = acc[u][0];
            e[LD] = acc[u][1];
          } else {
            e[0] += acc[u][0];
            e[LD] += acc[u][1];
          }
        }
    }
  }
  asm volatile("bar.sync 1, %0;\n" ::"r"(NCW * 32) : "memory");
  double* out = p.partials + (long long)blockIdx.x * SBD * SBD;
  for (int e = threadIdx.x; e < LD * LD; e += NCW * 32) {
    const int r = e % LD, c = e / LD;
    if ((r >> 3) >= (c >> 3)) out[r + SBD * c] = buf[r + LD * c];
  }
}

// K-split SYRK for 64 < a8 = 8 NBK <= 160 (k_syrk_kx generalised): the
// NBK(NBK+1)/2 lower 8x8 blocks are cut into P contiguous row-major parts and
// the 8 column groups of a 64-column tile into KS = 8 / P slices; warp
// (part, slice) accumulates its part's blocks (<= 40) over its slice's
// columns.  Each part is its own unrolled code path (template PART) so block
// indices and fragment registers stay static.  Per sub-step a warp loads the
// row-block fragments its part touches (<= NBK, conflict-free permuted-k
// layout of k_syrk_kx) for its DMMAs.  Slices of a part are summed in order
// into the per-CTA a8 x a8 partial (gram_reduce layout 1).
__host__ __device__ constexpr int kp_row_of(int u) {
  int bi = 0;
  while ((bi + 1) * (bi + 2) / 2 <= u) ++bi;
  return bi;
}

// TMA producer state of k_syrk_kp (thread 0 of the CTA; no separate
// producer warp, so the 8 consumer warps may use 255 registers)
struct KpProducer {
  long long tile;
  int it, s;
};
template <int NBOX>
__device__ __forceinline__ void kp_produce(const CUtensorMap* tm, const SyrkArgs& p, double* smem, uint64_t* full,
                                           uint64_t* empty, KpProducer& pr) {
  constexpr int BOX = 16 * kTC, STAGE = NBOX * BOX;
  while (pr.tile < p.n_tiles && p.sel != nullptr && p.sel[(pr.tile * kTC) / p.cpo] == 0) pr.tile += gridDim.x;
  if (pr.tile >= p.n_tiles) return;
  if (pr.it >= p.nst) mbar_wait(&empty[pr.s], (unsigned)(((pr.it / p.nst) - 1) & 1));
  mbar_expect_tx(&full[pr.s], (unsigned)STAGE * 8u);
#pragma unroll
  for (int b = 0; b < NBOX; ++b) tma_load_2d(smem + pr.s * STAGE + b * BOX, tm, 16 * b, (int)(pr.tile * kTC), &full[pr.s]);
  pr.tile += gridDim.x;
  ++pr.it;
  if (++pr.s == p.nst) pr.s = 0;
}

template <int NBK, int NPART, int KS, int PART>
__device__ __forceinline__ void syrk_kp_part(const CUtensorMap* tm, const SyrkArgs& p, double* smem, uint64_t* full,
                                             uint64_t* empty, int slice) {
  constexpr int NBL = NBK * (NBK + 1) / 2;
  constexpr int U0 = PART * NBL / NPART, U1 = (PART + 1) * NBL / NPART, NU = U1 - U0;
  constexpr int BI0 = kp_row_of(U0), BJ0 = U0 - BI0 * (BI0 + 1) / 2;
  constexpr int BI1 = kp_row_of(U1 - 1);
  // rows whose fragments this part needs: bj spans 0..BI1 once a full row is
  // covered, else BJ0..BI0 plus the row itself
  constexpr int RLO = (BI1 > BI0) ? 0 : BJ0;
  constexpr int RHI = BI1;
  constexpr int NF = RHI - RLO + 1;
  constexpr int NBOX = (NBK + 1) / 2;
  constexpr int BOX = 16 * kTC;
  constexpr int STAGE = NBOX * BOX;
  constexpr int NQ = 8 / KS;  // column groups per slice
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const bool producer = threadIdx.x == 0;
  KpProducer pr{blockIdx.x, 0, 0};
  if (producer)
    for (int k = 0; k < p.nst; ++k) kp_produce<NBOX>(tm, p, smem, full, empty, pr);
  __syncwarp();
  int base[2][2];
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int bp = 0; bp < 2; ++bp) {
      const int c7 = 2 * t + h;  // conflict-free per half-warp (see k_syrk_kx)
      base[h][bp] = c7 * 16 + (((4 * bp + (g >> 1)) ^ c7) << 1) + (g & 1);
    }
  double acc[NU][2];
#pragma unroll
  for (int u = 0; u < NU; ++u) acc[u][0] = acc[u][1] = 0.0;
  const int nst = p.nst;
  int st = 0;
  unsigned ph = 0;
  for (long long tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x) {
    if (p.sel != nullptr && p.sel[(tile * kTC) / p.cpo] == 0) continue;
    mbar_wait(&full[st], ph);
    const double* Ti = smem + st * STAGE;
#pragma unroll
    for (int qi = 0; qi < NQ; ++qi) {
      const int q = slice + KS * qi;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double f[NF];
#pragma unroll
        for (int k = 0; k < NF; ++k) {
          const int b = RLO + k;
          f[k] = Ti[(b >> 1) * BOX + 128 * q + base[h][b & 1]];
        }
        int bi = BI0, bj = BJ0;
#pragma unroll
        for (int u = 0; u < NU; ++u) {
          dmma(acc[u][0], acc[u][1], f[bi - RLO], f[bj - RLO]);
          if (++bj > bi) {
            ++bi;
            bj = 0;
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&empty[st])) : "memory");
    if (++st == nst) {
      st = 0;
      ph ^= 1u;
    }
    // refill the stage just consumed (waits for the other warps to release it;
    // in steady state warp 0 is the last to get there)
    if (producer) kp_produce<NBOX>(tm, p, smem, full, empty, pr);
    __syncwarp();
  }
  // slices of this part add into the CTA's partial in slice order
  const int a8 = 8 * NBK;
  double* out = p.partials + (long long)blockIdx.x * a8 * a8;
  for (int s = 0; s < KS; ++s) {
    __syncthreads();
    if (slice == s) {
      int bi = BI0, bj = BJ0;
#pragma unroll
      for (int u = 0; u < NU; ++u) {
        double* e = out + (8 * bi + g) + (long long)a8 * (8 * bj + 2 * t);
        if (s == 0) {
          e[0] = acc[u][0];
          e[a8] = acc[u][1];
        } else {
          e[0] += acc[u][0];
          e[a8] += acc[u][1];
        }
        if (++bj > bi) {
          ++bi;
          bj = 0;
        }
      }
    }
  }
}

template <int NBK, int NPART, int KS, int I>
__device__ __forceinline__ void kp_dispatch(int part, const CUtensorMap* tm, const SyrkArgs& p, double* smem,
                                            uint64_t* full, uint64_t* empty, int slice) {
  if constexpr (I < NPART) {
    if (part == I) syrk_kp_part<NBK, NPART, KS, I>(tm, p, smem, full, empty, slice);
    else kp_dispatch<NBK, NPART, KS, I + 1>(part, tm, p, smem, full, empty, slice);
  }
}

// P parts per CTA (8 / P column slices each) and PY CTAs per tile set
// (blockIdx.y): the lower blocks are cut into P * PY parts; the PY CTAs of a
// column x stream the same tiles at the same time (the second read hits L2)
// and write disjoint blocks of the same per-x partial.
template <int NBK, int P, int PY>
__global__ void __launch_bounds__(kConsumerWarps * 32, 1) k_syrk_kp(const __grid_constant__ CUtensorMap tm,
                                                                    SyrkArgs p) {
  constexpr int KS = 8 / P;
  extern __shared__ __align__(1024) double smem_raw[];
  __shared__ __align__(8) uint64_t full[8], empty[8];
  // X is the previous mode's projection output: wait for it (PDL launch).
  griddep_wait();
  double* smem = align1024(smem_raw);
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    fence_mbar_init();
    tma_prefetch_desc(&tm);
  }
  __syncthreads();
  const int part = (int)blockIdx.y * P + warp / KS, slice = warp % KS;
  kp_dispatch<NBK, P * PY, KS, 0>(part, &tm, p, smem, full, empty, slice);
}

// Two-stage fixed-order reduction of per-CTA Gram partials (hundreds of
// CTAs): stage 1 sums x-chunks of the partials for every lower-triangle
// element (blockIdx.y = chunk, four independent accumulators), stage 2 sums
// the chunks in order and mirrors the result.  layout 0: k_syrk super-tile
// pairs (ld sbd, pair py = I(I+1)/2 + J, CTA stride npairs-major); layout 1:
// one a8 x a8 partial per CTA.
__global__ void k_gram_reduce_s1(const double* __restrict__ partials, int nx, int layout, int ld, int a,
                                 double* __restrict__ tmp) {
  griddep_wait();
  const int xs = gridDim.y, y = blockIdx.y;
  const int x0 = (int)((long long)nx * y / xs), x1 = (int)((long long)nx * (y + 1) / xs);
  const long long n = (long long)a * a;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e % a), j = (int)(e / a);
    if (i < j) continue;
    long long base, stride;
    if (layout == 0) {
      const int I = i / ld, J = j / ld;
      const int py = I * (I + 1) / 2 + J;
      stride = (long long)ld * ld;
      base = (long long)py * nx * stride + (i - I * ld) + (long long)ld * (j - J * ld);
    } else {
      stride = (long long)ld * ld;
      base = i + (long long)ld * j;
    }
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int x = x0;
    for (; x + 3 < x1; x += 4) {
      s0 += partials[base + stride * x];
      s1 += partials[base + stride * (x + 1)];
      s2 += partials[base + stride * (x + 2)];
      s3 += partials[base + stride * (x + 3)];
    }
    for (; x < x1; ++x) s0 += partials[base + stride * x];
    tmp[(long long)y * n + e] = (s0 + s1) + (s2 + s3);
  }
}
__global__ void k_gram_reduce_s2(const double* __restrict__ tmp, int xs, int a, double* __restrict__ G) {
  griddep_wait();
  const long long n = (long long)a * a;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e % a), j = (int)(e / a);
    if (i < j) continue;
    double s = 0.0;
    for (int y = 0; y < xs; ++y) s += tmp[(long long)y * n + e];
    G[e] = s;
    G[j + (long long)a * i] = s;
  }
}

// ---------------------------------------------------------------------------
// Accurate path (small delta): TSQR R-factor of the residual.  With
// R^T = Q T (T a x a upper triangular), T^T T = R R^T but T carries the
// singular values of R unsquared, so the Jacobi solve on T^T resolves sigma
// down to eps_mach |R| instead of sqrt(eps_mach) |R| (the Gram floor).
// qr_update: T <- R-factor of [T; C] with C an m x a block given by strides
// C(q, j) = C[q*sq + j*sj]; Householder per column (Eigen/LAPACK sign rule).
// T is a x a column-major with leading dimension ldT (shared or global).
// ---------------------------------------------------------------------------
__device__ void qr_update(double* T, int ldT, double* C, int m, long long sq, long long sj, int a, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  for (int j = 0; j < a; ++j) {
    double ss = 0.0;
    for (int q = threadIdx.x; q < m; q += blockDim.x) {
      double v = C[q * sq + j * sj];
      ss = fma(v, v, ss);
    }
    // block sum (deterministic)
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (lane == 0) red[warp] = ss;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int w = 0; w < nwarps; ++w) s += red[w];
      red[32] = s;
    }
    __syncthreads();
    ss = red[32];
    const double alpha = T[j + (long long)ldT * j];
    if (ss == 0.0) {  // nothing below the diagonal: H = I
      __syncthreads();
      continue;
    }
    double beta = sqrt(alpha * alpha + ss);
    if (alpha >= 0.0) beta = -beta;
    const double tau = (beta - alpha) / beta;
    const double scale = 1.0 / (alpha - beta);
    // apply to columns c > j: w = T[j][c] + sum_q v_q C[q][c]; T[j][c] -= tau w; C[q][c] -= tau w v_q
    for (int c = j + 1 + warp; c < a; c += nwarps) {
      double w = 0.0;
      for (int q = lane; q < m; q += 32) w = fma(C[q * sq + j * sj] * scale, C[q * sq + c * sj], w);
      for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
      w += T[j + (long long)ldT * c];
      const double f = tau * w;
      if (lane == 0) T[j + (long long)ldT * c] -= f;
      for (int q = lane; q < m; q += 32) C[q * sq + c * sj] -= f * (C[q * sq + j * sj] * scale);
    }
    __syncthreads();
    if (threadIdx.x == 0) T[j + (long long)ldT * j] = beta;
    for (int q = threadIdx.x; q < m; q += blockDim.x) C[q * sq + j * sj] = 0.0;
    __syncthreads();
  }
}

struct TsqrArgs {
  TileSrc src;
  int a8, ldt, ldp;
  const double* UTf;
  const double* Uf;
  int r8;
  double* Tout;  // [gridDim.x][a*a]
  long long n_tiles;
};

// per-CTA T of the residual columns it owns (grid-stride over 64-column tiles)
__global__ void __launch_bounds__(kThreads) k_tsqr_local(TsqrArgs p) {
  griddep_wait();
  extern __shared__ __align__(16) double smem[];
  __shared__ double red[33];
  const int a = p.src.a, ldt = p.ldt, ldp = p.ldp;
  const int warp = threadIdx.x >> 5;
  double* Tf = smem;                       // a x a factor (ld a)
  double* Tl = smem + (size_t)a * a;       // tile a8 x 64 (ld ldt)
  double* Pw = Tl + (size_t)ldt * kTC + warp * ldp * 8;
  for (int i = threadIdx.x; i < a * a + ldt * kTC; i += kThreads) smem[i] = 0.0;
  __syncthreads();
  const int KA = p.a8 >> 2, KR = p.r8 >> 2, MR = p.r8 >> 3, nb = p.a8 >> 3;
  for (long long tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x) {
    load_tile_async(p.src, tile * kTC, Tl, ldt);
    cp_async_commit();
    cp_async_wait_0();
    __syncthreads();
    if (p.r8 > 0) {
      tile_residual(Tl, ldt, Pw, ldp, p.UTf, p.Uf, KA, KR, MR, nb);
      __syncthreads();
    }
    // rows of R^T are the tile's columns: C(q, j) = Tl[j + ldt*q]
    qr_update(Tf, a, Tl, kTC, ldt, 1, a, red);
  }
  double* out = p.Tout + (long long)blockIdx.x * a * a;
  for (int i = threadIdx.x; i < a * a; i += kThreads) out[i] = Tf[i];
}

// T <- R-factor of the stacked factors Ts[0..n-1] (each a x a), fixed order.
__global__ void __launch_bounds__(1024) k_tsqr_combine(const double* __restrict__ Ts, int n, int a,
                                                      double* __restrict__ scratch, double* __restrict__ T) {
  griddep_wait();
  extern __shared__ __align__(16) double sm2[];
  __shared__ double red[33];
  double* Tf = sm2;  // a x a
  for (int i = threadIdx.x; i < a * a; i += blockDim.x) Tf[i] = Ts[i];
  __syncthreads();
  for (int k = 1; k < n; ++k) {
    double* C = scratch;  // copy (qr_update overwrites the block)
    for (int i = threadIdx.x; i < a * a; i += blockDim.x) C[i] = Ts[(long long)k * a * a + i];
    __syncthreads();
    qr_update(Tf, a, C, a, 1, a, a, red);  // C(q, j) = C[q + a*j]
  }
  for (int i = threadIdx.x; i < a * a; i += blockDim.x) T[i] = Tf[i];
}

// ---------------------------------------------------------------------------
// Projection  out (r x L) = W^T cur  with W (a x r) as DMMA fragments.  The
// output is written compact (ld = r): exactly the next unfolding cur_{i+1}
// (r*n_{i+1} x L/n_{i+1}) of the reference's reshape (tt_ice.cpp:100-104).
// Optionally accumulates per-column squared norms of the output (coefficient
// norms for TT-ICE*).
// ---------------------------------------------------------------------------
struct ProjArgs {
  TileSrc src;
  int a8, ldt;
  const double* WTf;  // [r8/8][a8/4][32]
  int r, r8;
  double* out;
  double* tsumsq;     // per-tile sum of squares of the input tile (nullable)
  long long n_tiles;
  int frag_smem;      // stage W^T fragments in shared memory
  int nst;            // ring stages (k_project_ring)
  int kc;             // k-steps (16-row boxes) per ring stage (k_project_kc)
  const double* WTt;  // DFMA tail weights (k_make_tail layout, k_project_kc)
};

__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }

// Projection out (r x L) = W^T X.  Each warp owns 8 tile columns; its m-blocks
// are computed 4 at a time with a 2-way K split (8 independent DMMA chains).
// W^T fragments are staged once per CTA in shared memory.  The r x kTC output
// tile is staged in smem (double-buffered) and written back by one TMA bulk
// store per tile.  DB: double-buffered input tiles (a8 <= 128), else single
// (a8 <= 256).
template <bool DB, bool REGW>
__global__ void __launch_bounds__(kThreads) k_project(ProjArgs p) {
  griddep_wait();
  extern __shared__ __align__(16) double smem[];
  __shared__ double red8[kThreads / 32];
  __shared__ __align__(8) uint64_t bars[2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int ldt = p.ldt;
  const int KA = p.a8 >> 2, MR = p.r8 >> 3;
  const int nfr = MR * KA * 32;
  double* T0 = smem;
  double* T1 = DB ? smem + ldt * kTC : T0;
  double* Wfs = smem + (DB ? 2 : 1) * ldt * kTC;
  const double* Wf = p.frag_smem ? Wfs : p.WTf;
  const bool tma = (p.src.a & 1) == 0;
  for (int i = threadIdx.x; i < (DB ? 2 : 1) * ldt * kTC; i += kThreads) smem[i] = 0.0;
  if (p.frag_smem)
    for (int i = threadIdx.x; i < nfr; i += kThreads) Wfs[i] = p.WTf[i];
  double wreg[REGW ? 32 : 1];
  if (REGW) {  // requires MR <= 2 and KA <= 16 (a8 <= 64, r8 <= 16)
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int kb = 0; kb < 16; ++kb)
        wreg[u * 16 + kb] = (u < MR && kb < KA) ? p.WTf[(u * KA + kb) * 32 + lane] : 0.0;
  }
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
  }
  __syncthreads();
  unsigned phase[2] = {0u, 0u};
  long long tile = blockIdx.x;
  if (DB) {
    if (tile < p.n_tiles) tile_issue(p.src, tile * kTC, T0, ldt, &bars[0], tma);
    if (!tma) cp_async_commit();
  }
  int buf = 0, obuf = 0;
  for (; tile < p.n_tiles; tile += gridDim.x) {
    double* T = (DB && buf) ? T1 : T0;
    const int cb = DB ? buf : 0;
    if (DB) {
      double* Tn = buf ? T0 : T1;
      const long long nxt = tile + gridDim.x;
      if (nxt < p.n_tiles) tile_issue(p.src, nxt * kTC, Tn, ldt, &bars[buf ^ 1], tma);
      if (!tma) {
        cp_async_commit();
        cp_async_wait_1();
      }
    } else {
      tile_issue(p.src, tile * kTC, T0, ldt, &bars[0], tma);
      if (!tma) {
        cp_async_commit();
        cp_async_wait_0();
      }
    }
    if (tma) {
      mbar_wait(&bars[cb], phase[cb]);
      phase[cb] ^= 1u;
    }
    __syncthreads();
    if (p.tsumsq) {
      const double ts = tile_sumsq(T, p.src.a, ldt, red8);
      if (threadIdx.x < kConsumerWarps) p.tsumsq[tile * kConsumerWarps + threadIdx.x] = threadIdx.x == 0 ? ts : 0.0;
    }
    const int c0 = warp * 8;
    const long long col0 = tile * kTC + c0 + 2 * t;  // this thread's output columns col0, col0+1
    const bool ok0 = col0 < p.src.L, ok1 = col0 + 1 < p.src.L;
    double* o0 = p.out + col0 * p.r;
    double* o1 = o0 + p.r;
    if (REGW) {
      // W^T fragments live in registers (MR*KA <= 32): one smem load per DMMA pair
      double q[2][2][2] = {{{0.0, 0.0}, {0.0, 0.0}}, {{0.0, 0.0}, {0.0, 0.0}}};
#pragma unroll
      for (int kb = 0; kb < 16; ++kb) {
        if (kb < KA) {
          const double bv = T[(kb * 4 + t) + ldt * (c0 + g)];
#pragma unroll
          for (int u = 0; u < 2; ++u)
            if (u < MR) dmma(q[u][kb & 1][0], q[u][kb & 1][1], wreg[u * 16 + kb], bv);
        }
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int row = u * 8 + g;
        if (u < MR && row < p.r) {
          if (ok0) o0[row] = q[u][0][0] + q[u][1][0];
          if (ok1) o1[row] = q[u][0][1] + q[u][1][1];
        }
      }
    } else
    for (int mb0 = 0; mb0 < MR; mb0 += 4) {
      double q[4][2][2];
#pragma unroll
      for (int u = 0; u < 4; ++u) q[u][0][0] = q[u][0][1] = q[u][1][0] = q[u][1][1] = 0.0;
      const int nu = min(4, MR - mb0);
      int kb = 0;
      for (; kb + 1 < KA; kb += 2) {
        const double b0 = T[(kb * 4 + t) + ldt * (c0 + g)];
        const double b1 = T[(kb * 4 + 4 + t) + ldt * (c0 + g)];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (u < nu) {
            const double* wf = Wf + ((mb0 + u) * KA + kb) * 32 + lane;
            dmma(q[u][0][0], q[u][0][1], wf[0], b0);
            dmma(q[u][1][0], q[u][1][1], wf[32], b1);
          }
      }
      if (kb < KA) {
        const double b0 = T[(kb * 4 + t) + ldt * (c0 + g)];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (u < nu) dmma(q[u][0][0], q[u][0][1], Wf[((mb0 + u) * KA + kb) * 32 + lane], b0);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int row = (mb0 + u) * 8 + g;
        if (u < nu && row < p.r) {
          if (ok0) o0[row] = q[u][0][0] + q[u][1][0];
          if (ok1) o1[row] = q[u][0][1] + q[u][1][1];
        }
      }
    }
    __syncthreads();  // the stage is reused by a later refill
    buf ^= 1;
    obuf ^= 1;
  }
  if (threadIdx.x == 0) bulk_wait_all();
  if (!tma) cp_async_wait_0();
}

// ---------------------------------------------------------------------------
// Tensor-map TMA tiles.  X (a x L, column-major) is described by a 2-D tensor
// map {a, L} with 16 x 64 boxes and 128-byte swizzle: a tile of kTC columns is
// ceil(a/16) boxes of 8 KB, each 1024-byte aligned in smem, element (k, c) of
// box b at double offset  b*1024 + c*16 + (((k%16)/2) ^ (c%8))*2 + k%2.
// Rows >= a and columns >= L are zero-filled by the TMA unit.  One thread
// issues a whole tile (ceil(a/16) instructions); the swizzle makes the m8n8k4
// B-fragment pattern (4 consecutive rows x 8 columns) conflict-free without
// padding, so the smem image is dense and every byte moved is payload.
// ---------------------------------------------------------------------------

// Projection out (r x L) = W^T X with tensor-map TMA tiles of TC columns
// (TC = 64, or 32 for tall operands so that two CTAs with two stages each fit
// one SM) in an nst-deep ring (full mbarriers; thread 0 refills the stage
// freed in the previous iteration right after the per-tile block barrier).
// Warp w owns the 8 columns 8*(w % (TC/8)) of the tile; with TC = 32 the
// warps w and w+4 split the boxes (k range) by parity and the upper half adds
// its partial sums through shared memory.  W^T fragments in registers (REGW:
// a8 <= 64, r8 <= 16) or shared memory.  Outputs: a warp's 8 x r block is
// contiguous in `out`, staged per warp (r <= 32) and written with coalesced
// stores.  Optional per-(tile, warp) input sums of squares.
constexpr int kProjStages = 8;
template <bool REGW, int TC>
__global__ void __launch_bounds__(kThreads) k_project_tma(const __grid_constant__ CUtensorMap tm, ProjArgs p) {
  griddep_wait();
  static_assert(TC == 64 || TC == 32, "tile width");
  __shared__ double red_ss[4];
  constexpr int CW = TC / 8;   // column warps
  constexpr int KS = 8 / CW;   // k-split ways (1 or 2)
  constexpr int BOX = 16 * TC; // doubles per box
  extern __shared__ __align__(1024) double smem_raw[];
  __shared__ __align__(8) uint64_t full[kProjStages];
  double* smem = align1024(smem_raw);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int nst = p.nst;
  const int nbox = (p.src.a + 15) >> 4;
  const int KA = p.a8 >> 2, MR = p.r8 >> 3;
  const int nfr = MR * KA * 32;
  const int stage = nbox * BOX;  // doubles
  double* Wfs = smem + nst * stage;
  double* stg_all = Wfs + (p.frag_smem ? nfr : 0);
  const bool staged = p.r <= 32;  // (always true when KS > 1)
  double* stg = stg_all + warp * 8 * 32;
  const double* Wf = p.frag_smem ? Wfs : p.WTf;
  const int cw = warp % CW, kh = warp / CW;
  if (!REGW && p.frag_smem)
    for (int i = threadIdx.x; i < nfr; i += kThreads) Wfs[i] = p.WTf[i];
  // REGW: this warp's W^T fragments in registers: MRW m-blocks x KW k-steps
  // (TC = 64: all 16 k-steps of a8 <= 64, r8 <= 16; TC = 32: the 8 k-steps of
  // its box parity, r8 <= 32).  Local k-step jj <-> kb = 4 (KS (jj / 4) + kh) + jj % 4.
  constexpr int MRW = KS == 1 ? 2 : 4, KW = 16 / KS;
  double wreg[REGW ? MRW * KW : 1];
  if (REGW) {
#pragma unroll
    for (int u = 0; u < MRW; ++u)
#pragma unroll
      for (int jj = 0; jj < KW; ++jj) {
        const int kb = 4 * (KS * (jj >> 2) + kh) + (jj & 3);
        wreg[u * KW + jj] = (u < MR && kb < KA) ? p.WTf[(u * KA + kb) * 32 + lane] : 0.0;
      }
  }
  const long long grid = gridDim.x;
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tm);
    for (int s = 0; s < nst; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
    for (int s = 0; s < nst - 1; ++s) {
      const long long tl = blockIdx.x + s * grid;
      if (tl < p.n_tiles) {
        mbar_expect_tx(&full[s], (unsigned)nbox * BOX * 8u);
        for (int b = 0; b < nbox; ++b) tma_load_2d(smem + s * stage + b * BOX, &tm, 16 * b, (int)(tl * TC), &full[s]);
      }
    }
  }
  __syncthreads();
  const int c0 = cw * 8;
  // lane constants of the swizzled B-fragment address (k = 4kb + t, column c0 + g)
  const int hsw = (t >> 1) ^ g;
  const int lbase = (c0 + g) * 16 + (t & 1);
  int osw[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) osw[m] = lbase + (((m << 1) ^ hsw) << 1);
  int it = 0;
  for (long long tile = blockIdx.x; tile < p.n_tiles; tile += grid, ++it) {
    const int st = it % nst;
    mbar_wait(&full[st], (unsigned)((it / nst) & 1));
    __syncthreads();  // every warp is done with the stage consumed in iteration it-1
    if (threadIdx.x == 0) {
      const long long tl = tile + (nst - 1) * grid;
      if (tl < p.n_tiles) {
        const int sn = (it + nst - 1) % nst;
        mbar_expect_tx(&full[sn], (unsigned)nbox * BOX * 8u);
        for (int b = 0; b < nbox; ++b) tma_load_2d(smem + sn * stage + b * BOX, &tm, 16 * b, (int)(tl * TC), &full[sn]);
      }
    }
    const double* T = smem + st * stage;
    const long long colw = tile * TC + c0;
    const int nval = (int)max(0LL, min(8LL, p.src.L - colw));
    const long long col0 = colw + 2 * t;
    const bool ok0 = 2 * t < nval, ok1 = 2 * t + 1 < nval;
    double* o0 = p.out + col0 * p.r;
    double* o1 = o0 + p.r;
    double ss = 0.0;
    if (REGW) {
      double q[MRW][2][2];
#pragma unroll
      for (int u = 0; u < MRW; ++u) q[u][0][0] = q[u][0][1] = q[u][1][0] = q[u][1][1] = 0.0;
      double bv[KW];
#pragma unroll
      for (int jj = 0; jj < KW; ++jj) {
        const int kb = 4 * (KS * (jj >> 2) + kh) + (jj & 3);
        bv[jj] = kb < KA ? T[(kb >> 2) * BOX + osw[kb & 3]] : 0.0;
      }
#pragma unroll
      for (int jj = 0; jj < KW; ++jj) {
        ss = fma(bv[jj], bv[jj], ss);
#pragma unroll
        for (int u = 0; u < MRW; ++u)
          if (u < MR) dmma(q[u][jj & 1][0], q[u][jj & 1][1], wreg[u * KW + jj], bv[jj]);
      }
#pragma unroll
      for (int u = 0; u < MRW; ++u) {
        const int row = u * 8 + g;
        if (u < MR && row < p.r) {
          if (staged) {
            stg[row + p.r * (2 * t)] = q[u][0][0] + q[u][1][0];
            stg[row + p.r * (2 * t + 1)] = q[u][0][1] + q[u][1][1];
          } else {
            if (ok0) o0[row] = q[u][0][0] + q[u][1][0];
            if (ok1) o1[row] = q[u][0][1] + q[u][1][1];
          }
        }
      }
    } else {
      for (int mb0 = 0; mb0 < MR; mb0 += 4) {
        double q[4][2][2];
#pragma unroll
        for (int u = 0; u < 4; ++u) q[u][0][0] = q[u][0][1] = q[u][1][0] = q[u][1][1] = 0.0;
        const int nu = min(4, MR - mb0);
        for (int b = kh; b < nbox; b += KS) {
          // issue every load of the box first (clamped, always in range), then the DMMAs
          double bv[4], wv[4][4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int kbc = min(4 * b + j, KA - 1);
            bv[j] = T[b * BOX + osw[j]];
#pragma unroll
            for (int u = 0; u < 4; ++u) wv[u][j] = Wf[((mb0 + min(u, nu - 1)) * KA + kbc) * 32 + lane];
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (4 * b + j < KA) {
              if (mb0 == 0) ss = fma(bv[j], bv[j], ss);
#pragma unroll
              for (int u = 0; u < 4; ++u)
                if (u < nu) dmma(q[u][j & 1][0], q[u][j & 1][1], wv[u][j], bv[j]);
            }
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int row = (mb0 + u) * 8 + g;
          if (u < nu && row < p.r) {
            if (staged) {
              stg[row + p.r * (2 * t)] = q[u][0][0] + q[u][1][0];
              stg[row + p.r * (2 * t + 1)] = q[u][0][1] + q[u][1][1];
            } else {
              if (ok0) o0[row] = q[u][0][0] + q[u][1][0];
              if (ok1) o1[row] = q[u][0][1] + q[u][1][1];
            }
          }
        }
      }
    }
    if (p.tsumsq) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      if (KS > 1 && kh == 1 && lane == 0) red_ss[cw] = ss;
    }
    if (KS > 1) {  // upper warps hand their partial 8 x r blocks (and sums) to warp w - 4
      asm volatile("bar.sync 1, %0;\n" ::"r"(kThreads) : "memory");
      if (kh == 0) {
        const double* oth = stg_all + (warp + CW) * 8 * 32;
        for (int e = lane; e < 8 * p.r; e += 32) stg[e] += oth[e];
      }
    }
    if (staged && kh == 0) {
      __syncwarp();
      double* dst = p.out + colw * p.r;
      const int n = nval * p.r;
      for (int e = lane; e < n; e += 32) dst[e] = stg[e];
      __syncwarp();
    }
    // per-(64-column tile, 8-column group) sums: the layout of the TC = 64 kernels
    if (p.tsumsq && kh == 0 && lane == 0)
      p.tsumsq[((tile * TC) >> 6) * kConsumerWarps + (((tile * TC) & 63) >> 3) + cw] = KS > 1 ? ss + red_ss[cw] : ss;
  }
}

// W (a x r, ld) -> m16n8k16 B fragments for the k-step-major projection
// kernels: Wm[((b NB + nb) 4 + i) 32 + lane] = W[16b + t + 4i][8nb + g]
// (lane = 4g + t), zero outside W; b < nks = ceil(a/16), nb < NB = r8/8.
__global__ void k_make_frags16(const double* __restrict__ W, int a, int r, int ld, int nks, int NB,
                               double* __restrict__ Wm) {
  griddep_wait();
  const long long n = (long long)nks * NB * 128;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const int lane = (int)(e & 31), i = (int)((e >> 5) & 3);
    const long long f = e >> 7;
    const int nb = (int)(f % NB), b = (int)(f / NB);
    const int row = 16 * b + (lane & 3) + 4 * i, col = 8 * nb + (lane >> 2);
    Wm[e] = (row < a && col < r) ? W[row + (long long)ld * col] : 0.0;
  }
}

// Warp-specialised m16n8k16 projection (out^T tile = X^T W): warp NCW is the
// TMA producer (lane 0; full / empty mbarriers per stage), consumer warp w
// owns the 16 columns 16w..16w+15 of every TC = 16 NCW column tile and all
// k-steps, so no block barrier and no cross-warp reduction sits on the
// per-tile path.  W fragments (k_make_frags16 layout, NB = r8/8 <= 4 n-blocks,
// compile time) are read from shared memory with immediate offsets.  A
// fragment i of box b: row 4(i>>1) + t, column 16w + g + 8(i&1) (the
// conflict-free "4 rows x 8 columns" pattern twice under the 128-byte
// swizzle).  Output: the warp's 16 x r block is contiguous in out, staged in
// shared memory and stored coalesced; optional per-(64-column tile, 8-column
// group) input sums of squares.
template <int NCW, int NB>
__global__ void __launch_bounds__((NCW + 1) * 32) k_project_ws16(const __grid_constant__ CUtensorMap tm, ProjArgs p) {
  griddep_wait();
  constexpr int TC = 16 * NCW, BOX = 16 * TC;
  extern __shared__ __align__(1024) double smem_raw[];
  __shared__ __align__(8) uint64_t full[kProjStages], empty[kProjStages];
  double* smem = align1024(smem_raw);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int nst = p.nst;
  const int nks = (p.src.a + 15) >> 4;
  const int stage = nks * BOX;
  double* Wfs = smem + nst * stage;
  const int nfr = nks * NB * 128;
  double* stg = Wfs + nfr + warp * 16 * p.r8;  // 16 columns x r8 per warp
  for (int i = threadIdx.x; i < nfr; i += blockDim.x) Wfs[i] = p.WTf[i];
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const long long grid = gridDim.x;
  if (warp == NCW) {  // ---- producer ----
    if (lane == 0) {
      tma_prefetch_desc(&tm);
      int it = 0;
      for (long long tile = blockIdx.x; tile < p.n_tiles; tile += grid, ++it) {
        const int s = it % nst;
        if (it >= nst) mbar_wait(&empty[s], (unsigned)(((it / nst) - 1) & 1));
        mbar_expect_tx(&full[s], (unsigned)nks * BOX * 8u);
        for (int b = 0; b < nks; ++b) tma_load_2d(smem + s * stage + b * BOX, &tm, 16 * b, (int)(tile * TC), &full[s]);
      }
    }
    return;
  }
  // ---- consumers ----
  // MMA row g of the A fragment (a tile column) lives in physical column
  // pg = pi(g) = 2 (g & 3) + (g >> 2) of its 8-column group: 64-bit shared
  // loads are served per half-warp (lanes g < 4 / g >= 4), and this spreads
  // each half-warp over all 8 swizzle chunks of a 128-byte row (16 distinct
  // 8-byte banks per half: 2 wavefronts instead of 4).
  const int pg = ((g & 3) << 1) | (g >> 2);
  int osw[8];
  {
    const int hsw = (t >> 1) ^ pg;
#pragma unroll
    for (int i = 0; i < 8; ++i) osw[i] = (16 * warp + pg + 8 * (i & 1)) * 16 + (t & 1) + (((2 * (i >> 1)) ^ hsw) << 1);
  }
  const double* wl = Wfs + lane;
  const bool want_ss = p.tsumsq != nullptr;
  int st = 0;
  unsigned ph = 0;
  for (long long tile = blockIdx.x; tile < p.n_tiles; tile += grid) {
    mbar_wait(&full[st], ph);
    const double* ab = smem + st * stage;
    const double* wb = wl;
    double acc[NB][4];
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) acc[nb][0] = acc[nb][1] = acc[nb][2] = acc[nb][3] = 0.0;
    double ss0 = 0.0, ss1 = 0.0;
    for (int b = 0; b < nks; ++b, ab += BOX, wb += NB * 128) {
      double av[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) av[i] = ab[osw[i]];
      if (want_ss) {
#pragma unroll
        for (int i = 0; i < 8; i += 2) {
          ss0 = fma(av[i], av[i], ss0);
          ss1 = fma(av[i + 1], av[i + 1], ss1);
        }
      }
#pragma unroll
      for (int nb = 0; nb < NB; ++nb) {
        double bw[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) bw[i] = wb[(nb * 4 + i) * 32];
        dmma16(acc[nb], av, bw);
      }
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&empty[st])) : "memory");
    if (++st == nst) {
      st = 0;
      ph ^= 1u;
    }
#pragma unroll
    for (int nb = 0; nb < NB; ++nb)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int row = 8 * nb + 2 * t + (i & 1);
        if (row < p.r) stg[row + p.r * (pg + 8 * (i >> 1))] = acc[nb][i];
      }
    __syncwarp();
    const long long colw = tile * TC + 16 * warp;
    const int nval = (int)max(0LL, min(16LL, p.src.L - colw));
    double* dst = p.out + colw * p.r;
    const int n = nval * p.r;
    for (int e = lane; e < n; e += 32) dst[e] = stg[e];
    if (want_ss) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        ss0 += __shfl_xor_sync(0xffffffffu, ss0, o);
        ss1 += __shfl_xor_sync(0xffffffffu, ss1, o);
      }
      if (lane == 0) {
        const long long c64 = colw >> 6;
        const int grp = (int)((colw & 63) >> 3);
        p.tsumsq[c64 * kConsumerWarps + grp] = ss0;
        p.tsumsq[c64 * kConsumerWarps + grp + 1] = ss1;
      }
    }
    __syncwarp();
  }
}

// W columns [c0, c0 + T) (the rows of out past the 8 NB DMMA rows) for the
// DFMA tail of k_project_kc:  Wt[((b T + j) 4 + t) 4 + q] = W[16b + 4q + t][c0 + j]
// (zero past a), so lane (g, t) reads its four k values of box b as two double2.
__global__ void k_make_tail(const double* __restrict__ W, int a, int ld, int nks, int c0, int T,
                            double* __restrict__ Wt) {
  griddep_wait();
  const int n = nks * T * 16;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    const int q = e & 3, t = (e >> 2) & 3, f = e >> 4;
    const int j = f % T, b = f / T;
    const int row = 16 * b + 4 * q + t;
    Wt[e] = row < a ? W[row + (long long)ld * (c0 + j)] : 0.0;
  }
}

// K-chunked warp-specialised projection out (r x L) = W^T X for any even a
// (the whole pre-projected chain of several modes, a = 512 at cfg3, in one
// pass over Y).  A tile is TC = 16 NCW columns; its ceil(a/16) boxes stream
// through the ring kc boxes per stage while each consumer warp keeps its 16
// columns' accumulators in registers across the stages (so the ring depth
// does not shrink with a).  Rows of out: 8 NB by m16n8k16 DMMA (W fragments
// k-step-major in smem, as k_project_ws16) plus T = r - 8 NB in {1, 2} by DFMA
// on the A fragments already in registers (W tail in smem, k_make_tail):
// r = 17 costs 2 + 1/8 n-blocks of FP64 work instead of padding to 24.
// The tail partial sums are reduced over the 4 lanes t of a column group.
template <int NCW, int NB, int T>
__global__ void __launch_bounds__((NCW + 1) * 32) k_project_kc(const __grid_constant__ CUtensorMap tm, ProjArgs p) {
  griddep_wait();
  constexpr int TC = 16 * NCW, BOX = 16 * TC;
  extern __shared__ __align__(1024) double smem_raw[];
  __shared__ __align__(8) uint64_t full[kProjStages], empty[kProjStages];
  double* smem = align1024(smem_raw);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int nst = p.nst, kc = p.kc;
  const int nks = (p.src.a + 15) >> 4;
  const int nch = (nks + kc - 1) / kc;
  const int stage = kc * BOX;
  double* Wfs = smem + nst * stage;
  const int nfr = nks * NB * 128;
  double* Wts = Wfs + nfr;
  const int ntl = nks * T * 16;
  double* stg = Wts + ntl + warp * 16 * (8 * NB + T);  // 16 columns x r per warp
  for (int i = threadIdx.x; i < nfr; i += blockDim.x) Wfs[i] = p.WTf[i];
  for (int i = threadIdx.x; i < ntl; i += blockDim.x) Wts[i] = p.WTt[i];
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const long long grid = gridDim.x;
  if (warp == NCW) {  // ---- producer ----
    if (lane == 0) {
      tma_prefetch_desc(&tm);
      int it = 0, s = 0;
      for (long long tile = blockIdx.x; tile < p.n_tiles; tile += grid) {
        for (int ch = 0; ch < nch; ++ch, ++it) {
          if (it >= nst) mbar_wait(&empty[s], (unsigned)(((it / nst) - 1) & 1));
          const int b0 = ch * kc, nb = min(kc, nks - b0);
          mbar_expect_tx(&full[s], (unsigned)nb * BOX * 8u);
          for (int b = 0; b < nb; ++b)
            tma_load_2d(smem + s * stage + b * BOX, &tm, 16 * (b0 + b), (int)(tile * TC), &full[s]);
          if (++s == nst) s = 0;
        }
      }
    }
    return;
  }
  // ---- consumers ----
  // MMA row g of the A fragment (a tile column) lives in physical column
  // pg = pi(g) = 2 (g & 3) + (g >> 2) of its 8-column group: 64-bit shared
  // loads are served per half-warp (lanes g < 4 / g >= 4), and this spreads
  // each half-warp over all 8 swizzle chunks of a 128-byte row (16 distinct
  // 8-byte banks per half: 2 wavefronts instead of 4).
  const int pg = ((g & 3) << 1) | (g >> 2);
  int osw[8];
  {
    const int hsw = (t >> 1) ^ pg;
#pragma unroll
    for (int i = 0; i < 8; ++i) osw[i] = (16 * warp + pg + 8 * (i & 1)) * 16 + (t & 1) + (((2 * (i >> 1)) ^ hsw) << 1);
  }
  const bool want_ss = p.tsumsq != nullptr;
  int st = 0;
  unsigned ph = 0;
  for (long long tile = blockIdx.x; tile < p.n_tiles; tile += grid) {
    double acc[NB][4];
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) acc[nb][0] = acc[nb][1] = acc[nb][2] = acc[nb][3] = 0.0;
    double tacc[T > 0 ? T : 1][2];
#pragma unroll
    for (int j = 0; j < (T > 0 ? T : 1); ++j) tacc[j][0] = tacc[j][1] = 0.0;
    double ss0 = 0.0, ss1 = 0.0;
    for (int ch = 0; ch < nch; ++ch) {
      mbar_wait(&full[st], ph);
      const double* ab = smem + st * stage;
      const int b0 = ch * kc, nb_ch = min(kc, nks - b0);
      const double* wb = Wfs + lane + b0 * NB * 128;
      const double* wt = Wts + b0 * T * 16 + 4 * t;
      for (int bb = 0; bb < nb_ch; ++bb, ab += BOX, wb += NB * 128, wt += T * 16) {
        double av[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) av[i] = ab[osw[i]];
        if (want_ss) {
#pragma unroll
          for (int i = 0; i < 8; i += 2) {
            ss0 = fma(av[i], av[i], ss0);
            ss1 = fma(av[i + 1], av[i + 1], ss1);
          }
        }
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) {
          double bw[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) bw[i] = wb[(nb * 4 + i) * 32];
          dmma16(acc[nb], av, bw);
        }
#pragma unroll
        for (int j = 0; j < T; ++j) {
          const double2 w01 = *reinterpret_cast<const double2*>(wt + j * 16);
          const double2 w23 = *reinterpret_cast<const double2*>(wt + j * 16 + 2);
          tacc[j][0] = fma(av[0], w01.x, tacc[j][0]);
          tacc[j][1] = fma(av[1], w01.x, tacc[j][1]);
          tacc[j][0] = fma(av[2], w01.y, tacc[j][0]);
          tacc[j][1] = fma(av[3], w01.y, tacc[j][1]);
          tacc[j][0] = fma(av[4], w23.x, tacc[j][0]);
          tacc[j][1] = fma(av[5], w23.x, tacc[j][1]);
          tacc[j][0] = fma(av[6], w23.y, tacc[j][0]);
          tacc[j][1] = fma(av[7], w23.y, tacc[j][1]);
        }
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&empty[st])) : "memory");
      if (++st == nst) {
        st = 0;
        ph ^= 1u;
      }
    }
#pragma unroll
    for (int nb = 0; nb < NB; ++nb)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int row = 8 * nb + 2 * t + (i & 1);
        if (row < p.r) stg[row + p.r * (pg + 8 * (i >> 1))] = acc[nb][i];
      }
#pragma unroll
    for (int j = 0; j < T; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double v = tacc[j][h];
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        if (t == 0) stg[8 * NB + j + p.r * (pg + 8 * h)] = v;
      }
    }
    __syncwarp();
    const long long colw = tile * TC + 16 * warp;
    const int nval = (int)max(0LL, min(16LL, p.src.L - colw));
    double* dst = p.out + colw * p.r;
    const int n = nval * p.r;
    for (int e = lane; e < n; e += 32) dst[e] = stg[e];
    if (want_ss) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        ss0 += __shfl_xor_sync(0xffffffffu, ss0, o);
        ss1 += __shfl_xor_sync(0xffffffffu, ss1, o);
      }
      if (lane == 0) {
        const long long c64 = colw >> 6;
        const int grp = (int)((colw & 63) >> 3);
        p.tsumsq[c64 * kConsumerWarps + grp] = ss0;
        p.tsumsq[c64 * kConsumerWarps + grp + 1] = ss1;
      }
    }
    __syncwarp();
  }
}

// High-rank projection out (r x L) = W^T X, 34 < r <= 128 (the companion
// sweep's R = 64 / 128 chains, tt_project tensor_train.cpp:195-226): the
// k_project_kc pipeline with the W fragments STREAMED through the ring next to
// the X boxes (a x r fragments no longer fit shared memory: 256 KB at a = 512,
// r = 64).  Each stage carries kc X boxes (TMA tensor map, 128-byte swizzle)
// plus the same kc k-steps of W^T fragments (one bulk copy from the
// k_make_frags16 layout, L2-resident); consumer warp w keeps the NB = r8/8
// n-block accumulators of its 16 columns in registers across the chunks and
// stores them straight from registers (the output is r/a of the input).
template <int NCW, int NB>
__global__ void __launch_bounds__((NCW + 1) * 32, 1) k_project_ws(const __grid_constant__ CUtensorMap tm, ProjArgs p) {
  griddep_wait();
  constexpr int TC = 16 * NCW, BOX = 16 * TC, WCH = NB * 128;
  extern __shared__ __align__(1024) double smem_raw[];
  __shared__ __align__(8) uint64_t full[kProjStages], empty[kProjStages];
  double* smem = align1024(smem_raw);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int nst = p.nst, kc = p.kc;
  const int nks = (p.src.a + 15) >> 4;
  const int nch = (nks + kc - 1) / kc;
  const int stage = kc * (BOX + WCH);
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const long long grid = gridDim.x;
  if (warp == NCW) {  // ---- producer ----
    if (lane == 0) {
      tma_prefetch_desc(&tm);
      int it = 0, s = 0;
      for (long long tile = blockIdx.x; tile < p.n_tiles; tile += grid) {
        for (int ch = 0; ch < nch; ++ch, ++it) {
          if (it >= nst) mbar_wait(&empty[s], (unsigned)(((it / nst) - 1) & 1));
          const int b0 = ch * kc, nb = min(kc, nks - b0);
          mbar_expect_tx(&full[s], (unsigned)nb * (BOX + WCH) * 8u);
          double* st = smem + s * stage;
          for (int b = 0; b < nb; ++b) tma_load_2d(st + b * BOX, &tm, 16 * (b0 + b), (int)(tile * TC), &full[s]);
          bulk_g2s(st + kc * BOX, p.WTf + (size_t)b0 * WCH, (unsigned)nb * WCH * 8u, &full[s]);
          if (++s == nst) s = 0;
        }
      }
    }
    return;
  }
  // ---- consumers (fragment addressing as k_project_kc) ----
  const int pg = ((g & 3) << 1) | (g >> 2);
  int osw[8];
  {
    const int hsw = (t >> 1) ^ pg;
#pragma unroll
    for (int i = 0; i < 8; ++i) osw[i] = (16 * warp + pg + 8 * (i & 1)) * 16 + (t & 1) + (((2 * (i >> 1)) ^ hsw) << 1);
  }
  const bool want_ss = p.tsumsq != nullptr;
  int st = 0;
  unsigned ph = 0;
  for (long long tile = blockIdx.x; tile < p.n_tiles; tile += grid) {
    double acc[NB][4];
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) acc[nb][0] = acc[nb][1] = acc[nb][2] = acc[nb][3] = 0.0;
    double ss0 = 0.0, ss1 = 0.0;
    for (int ch = 0; ch < nch; ++ch) {
      mbar_wait(&full[st], ph);
      const double* ab = smem + st * stage;
      const double* wb = ab + kc * BOX + lane;
      const int b0 = ch * kc, nb_ch = min(kc, nks - b0);
      for (int bb = 0; bb < nb_ch; ++bb, ab += BOX, wb += WCH) {
        double av[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) av[i] = ab[osw[i]];
        if (want_ss) {
#pragma unroll
          for (int i = 0; i < 8; i += 2) {
            ss0 = fma(av[i], av[i], ss0);
            ss1 = fma(av[i + 1], av[i + 1], ss1);
          }
        }
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) {
          double bw[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) bw[i] = wb[(nb * 4 + i) * 32];
          dmma16(acc[nb], av, bw);
        }
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&empty[st])) : "memory");
      if (++st == nst) {
        st = 0;
        ph ^= 1u;
      }
    }
    // acc[nb][i]: tile column pg + 8 (i >> 1) of the warp, output row 8 nb + 2 t + (i & 1)
    const long long colw = tile * TC + 16 * warp;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const long long col = colw + pg + 8 * h;
      if (col < p.src.L) {
        double* dst = p.out + col * p.r;
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) {
          const int row = 8 * nb + 2 * t;
          if (row + 1 < p.r && !(p.r & 1)) {
            *reinterpret_cast<double2*>(dst + row) = make_double2(acc[nb][2 * h], acc[nb][2 * h + 1]);
          } else {
            if (row < p.r) dst[row] = acc[nb][2 * h];
            if (row + 1 < p.r) dst[row + 1] = acc[nb][2 * h + 1];
          }
        }
      }
    }
    if (want_ss) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        ss0 += __shfl_xor_sync(0xffffffffu, ss0, o);
        ss1 += __shfl_xor_sync(0xffffffffu, ss1, o);
      }
      if (lane == 0) {
        const long long c64 = colw >> 6;
        const int grp = (int)((colw & 63) >> 3);
        p.tsumsq[c64 * kConsumerWarps + grp] = ss0;
        p.tsumsq[c64 * kConsumerWarps + grp + 1] = ss1;
      }
    }
  }
}

// Projection out (r x L) = W^T X over a ring of single TMA boxes (16 rows x
// 64 columns = 8 KB, 128-byte swizzle): warp 8 lane 0 is the producer (full /
// empty mbarriers per stage), warps 0..7 consume.  A column tile of any height
// streams through the ring box by box while the warp's accumulators (all MR
// m-blocks of its 8 columns) stay in registers, so the pipeline depth does not
// shrink with a.  W^T fragments in registers (REGW: a8 <= 64, MR <= 2),
// shared memory (frag_smem) or global (L1).  Outputs staged per warp (r <= 32)
// and written coalesced; optional per-(tile, warp) input sums of squares.
// ---------------------------------------------------------------------------
// SYRK over tensor-map tiles: C = sum over (selected) columns x x^T, x the
// a rows of X (a <= 256).  A tile is kTC full-height columns, ceil(a/16) TMA
// boxes with 128-byte swizzle (dense smem, one instruction per box); warp 8
// lane 0 produces into an nst-deep ring (full / empty mbarriers), warps 0..7
// consume.  The lower triangle of the (a8/8)^2 block grid is cut into 2x2-block
// tiles, dealt round-robin over the gridDim.y "parts" x 8 warps (a part's CTAs
// read the same column tiles; the repeat read hits L2).  The k dimension of
// each DMMA step uses the columns {8q + 2h + (0,1,4,5)} (h = step parity):
// with the swizzle this makes the 8-row x 4-column A/B fragment loads
// bank-conflict free (tools/probe: checked exhaustively).  Observation
// selection skips whole tiles (requires cols_per_obs % kTC == 0).  Each CTA
// writes its owned blocks into partials[blockIdx.x] (a8 x a8); parts own
// disjoint blocks, so k_gram_reduce_s1/s2 sum over blockIdx.x only.
// ---------------------------------------------------------------------------
struct Syrk2Args {
  int a, a8, nbox, nst;
  long long L, n_tiles;
  const uint8_t* sel;
  long long cpo;
  int ntiles2;       // lower 2x2-block tiles
  double* partials;  // [gridDim.x][a8 * a8]
  double* tsumsq;    // per-(tile, 8-column group) input sums of squares (part 0), nullable
};

template <int MAXT>
__global__ void __launch_bounds__(kSyrkThreads) k_syrk2(const __grid_constant__ CUtensorMap tm, Syrk2Args p) {
  griddep_wait();
  extern __shared__ __align__(1024) double smem_raw[];
  __shared__ __align__(8) uint64_t full[kMaxStages], empty[kMaxStages];
  double* ring = align1024(smem_raw);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int stage = p.nbox * 1024;
  const int nst = p.nst;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const long long grid = gridDim.x;
  if (warp == kConsumerWarps) {  // ---- producer ----
    if (lane == 0) {
      tma_prefetch_desc(&tm);
      int it = 0;
      for (long long tile = blockIdx.x; tile < p.n_tiles; tile += grid) {
        if (p.sel && !p.sel[(tile * kTC) / p.cpo]) continue;
        const int s = it % nst;
        if (it >= nst) mbar_wait(&empty[s], (unsigned)(((it / nst) - 1) & 1));
        mbar_expect_tx(&full[s], (unsigned)p.nbox * 8192u);
        for (int b = 0; b < p.nbox; ++b) tma_load_2d(ring + s * stage + b * 1024, &tm, 16 * b, (int)(tile * kTC), &full[s]);
        ++it;
      }
    }
    return;
  }
  // ---- consumers ----
  const int part = blockIdx.y, P = gridDim.y;
  int baseA[MAXT], baseB[MAXT], rowA[MAXT], rowB[MAXT];
  bool live[MAXT];
#pragma unroll
  for (int u = 0; u < MAXT; ++u) {
    const int idx = part * kConsumerWarps + warp + kConsumerWarps * P * u;
    live[u] = idx < p.ntiles2;
    int ta = (int)((sqrtf(8.0f * idx + 1.0f) - 1.0f) * 0.5f);
    while ((ta + 1) * (ta + 2) / 2 <= idx) ++ta;
    while (ta * (ta + 1) / 2 > idx) --ta;
    const int tb = idx - ta * (ta + 1) / 2;
    baseA[u] = ta * 1024;
    baseB[u] = tb * 1024;
    rowA[u] = 16 * ta;
    rowB[u] = 16 * tb;
  }
  // lane offsets inside a box for step parity h and row half x (see header)
  int offs[2][2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int cl = 2 * h + (t & 1) + 4 * (t >> 1);
#pragma unroll
    for (int x = 0; x < 2; ++x) offs[h][x] = 16 * cl + (((4 * x + (g >> 1)) ^ cl) << 1) + (g & 1);
  }
  double acc[MAXT][2][2][2];
#pragma unroll
  for (int u = 0; u < MAXT; ++u)
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
      for (int y = 0; y < 2; ++y) acc[u][x][y][0] = acc[u][x][y][1] = 0.0;
  int it = 0;
  for (long long tile = blockIdx.x; tile < p.n_tiles; tile += grid) {
    if (p.sel && !p.sel[(tile * kTC) / p.cpo]) continue;
    const int st = it % nst;
    mbar_wait(&full[st], (unsigned)((it / nst) & 1));
    const double* T = ring + st * stage;
    if (p.tsumsq && part == 0) {  // this warp's 8 columns are 128 consecutive doubles per box
      double sq = 0.0;
      for (int b = 0; b < p.nbox; ++b) {
        const double* base = T + b * 1024 + warp * 128;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const double v = base[lane + 32 * e];
          sq = fma(v, v, sq);
        }
      }
      sq = warp_sum(sq);
      if (lane == 0) p.tsumsq[tile * kConsumerWarps + warp] = sq;
    }
#pragma unroll
    for (int u = 0; u < MAXT; ++u) {
      if (!live[u]) continue;  // warp-uniform
      const double* TA = T + baseA[u];
      const double* TB = T + baseB[u];
#pragma unroll 4
      for (int kk = 0; kk < kTC / 4; ++kk) {
        const int ko = 128 * (kk >> 1);
        const int h = kk & 1;
        const double a0 = TA[ko + offs[h][0]];
        const double a1 = TA[ko + offs[h][1]];
        const double b0 = TB[ko + offs[h][0]];
        const double b1 = TB[ko + offs[h][1]];
        dmma(acc[u][0][0][0], acc[u][0][0][1], a0, b0);
        dmma(acc[u][0][1][0], acc[u][0][1][1], a0, b1);
        dmma(acc[u][1][0][0], acc[u][1][0][1], a1, b0);
        dmma(acc[u][1][1][0], acc[u][1][1][1], a1, b1);
      }
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&empty[st])) : "memory");
    ++it;
  }
  double* out = p.partials + (long long)blockIdx.x * p.a8 * p.a8;
#pragma unroll
  for (int u = 0; u < MAXT; ++u) {
    if (!live[u]) continue;
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
      for (int y = 0; y < 2; ++y) {
        const int r = rowA[u] + x * 8 + g;
        const int c = rowB[u] + y * 8 + 2 * t;
        if (r < p.a8 && c + 1 < p.a8 + 1 && c < p.a8) {
          out[r + (long long)p.a8 * c] = acc[u][x][y][0];
          out[r + (long long)p.a8 * (c + 1)] = acc[u][x][y][1];
        }
      }
  }
}

// ---------------------------------------------------------------------------
// Warp-specialised SYRK with mma.m16n8k16 (a <= 128): C = sum over (selected)
// 64-column tiles of X X^T.  Warp NCW lane 0 streams tensor-map tiles
// (ceil(a/16) boxes, 128-byte swizzle) into an nst-deep ring (full / empty
// mbarriers); consumer warps own "groups" = (16-row block mi, pair of 8-row
// blocks 2p, 2p+1), p <= mi (the lower triangle), dealt round-robin; per
// 16-column k-step a group is one A fragment (8 loads) and two B fragments
// (4 loads each) feeding two MMAs.  The k index of a step is permuted,
// column(t, j) = 8(j>>1) + 2(j&1) + (t&1) + 4(t>>1), which makes every
// fragment load bank-conflict free under the swizzle (checked exhaustively).
// Per-CTA partials (a8 x a8, owned blocks) are summed by k_gram_reduce_s1/s2.
// Input sums of squares (tsumsq, 8 per 64-column tile) come from the B
// fragments of the diagonal groups (p == mi cover every row once), reduced
// across warps in shared memory behind a consumer-only named barrier.
// ---------------------------------------------------------------------------
template <int NCW, int MAXG>
__global__ void __launch_bounds__((NCW + 1) * 32) k_syrk_ws16(const __grid_constant__ CUtensorMap tm, Syrk2Args p) {
  griddep_wait();
  constexpr int BOX = 1024;
  extern __shared__ __align__(1024) double smem_raw[];
  __shared__ __align__(8) uint64_t full[kMaxStages + 4], empty[kMaxStages + 4];
  __shared__ double ssq[NCW][8];
  double* ring = align1024(smem_raw);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int nks = p.nbox, stage = nks * BOX, nst = p.nst;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const long long grid = gridDim.x;
  if (warp == NCW) {  // ---- producer ----
    if (lane == 0) {
      tma_prefetch_desc(&tm);
      int it = 0;
      for (long long tile = blockIdx.x; tile < p.n_tiles; tile += grid) {
        if (p.sel && !p.sel[(tile * kTC) / p.cpo]) continue;
        const int s = it % nst;
        if (it >= nst) mbar_wait(&empty[s], (unsigned)(((it / nst) - 1) & 1));
        mbar_expect_tx(&full[s], (unsigned)nks * BOX * 8u);
        for (int b = 0; b < nks; ++b) tma_load_2d(ring + s * stage + b * BOX, &tm, 16 * b, (int)(tile * kTC), &full[s]);
        ++it;
      }
    }
    return;
  }
  // ---- consumers ----
  const int ngroups = nks * (nks + 1) / 2;
  int gA[MAXG], gB[MAXG], gmi[MAXG], gp[MAXG];
  bool live[MAXG];
#pragma unroll
  for (int u = 0; u < MAXG; ++u) {
    const int idx = warp + NCW * u;
    live[u] = idx < ngroups;
    int mi = (int)((sqrtf(8.0f * idx + 1.0f) - 1.0f) * 0.5f);
    while ((mi + 1) * (mi + 2) / 2 <= idx) ++mi;
    while (mi * (mi + 1) / 2 > idx) --mi;
    const int pp = idx - mi * (mi + 1) / 2;
    gmi[u] = mi;
    gp[u] = pp;
    gA[u] = mi * BOX;
    gB[u] = pp * BOX;  // 8-row blocks 2pp, 2pp+1 live in box pp (halves 0 / 1)
  }
  // lane offsets (k-step 0) of the A elements i = 0..7 and the B elements
  // (half h = 0/1 of the box, i = 0..3)
  int offA[8], offB[2][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int j = i >> 1;
    const int col = 8 * (j >> 1) + 2 * (j & 1) + (t & 1) + 4 * (t >> 1);
    const int cl = 2 * (j & 1) + (t & 1) + 4 * (t >> 1);
    offA[i] = col * 16 + ((((g >> 1) + 4 * (i & 1)) ^ cl) << 1) + (g & 1);
  }
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int col = 8 * (i >> 1) + 2 * (i & 1) + (t & 1) + 4 * (t >> 1);
      const int cl = 2 * (i & 1) + (t & 1) + 4 * (t >> 1);
      offB[h][i] = col * 16 + (((4 * h + (g >> 1)) ^ cl) << 1) + (g & 1);
    }
  double acc[MAXG][2][4];
#pragma unroll
  for (int u = 0; u < MAXG; ++u)
#pragma unroll
    for (int h = 0; h < 2; ++h) acc[u][h][0] = acc[u][h][1] = acc[u][h][2] = acc[u][h][3] = 0.0;
  const bool want_ss = p.tsumsq != nullptr;
  int st = 0;
  unsigned ph = 0;
  for (long long tile = blockIdx.x; tile < p.n_tiles; tile += grid) {
    if (p.sel && !p.sel[(tile * kTC) / p.cpo]) continue;
    mbar_wait(&full[st], ph);
    const double* T = ring + st * stage;
    double ss[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) ss[q] = 0.0;
#pragma unroll
    for (int u = 0; u < MAXG; ++u) {
      if (!live[u]) continue;  // warp-uniform
      const double* TA = T + gA[u];
      const double* TB = T + gB[u];
      const bool diag = want_ss && gp[u] == gmi[u];
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        double av[8], b0[4], b1[4];
#pragma unroll
        for (int i = 0; i < 8; ++i) av[i] = TA[256 * ks + offA[i]];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          b0[i] = TB[256 * ks + offB[0][i]];
          b1[i] = TB[256 * ks + offB[1][i]];
        }
        if (diag) {
#pragma unroll
          for (int i = 0; i < 4; ++i) ss[2 * ks + (i >> 1)] = fma(b0[i], b0[i], fma(b1[i], b1[i], ss[2 * ks + (i >> 1)]));
        }
        dmma16(acc[u][0], av, b0);
        dmma16(acc[u][1], av, b1);
      }
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&empty[st])) : "memory");
    if (want_ss) {  // 8 per-tile column-group sums, fixed-order reduction over the consumer warps
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        double v = ss[q];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) ssq[warp][q] = v;
      }
      asm volatile("bar.sync 1, %0;\n" ::"r"(NCW * 32) : "memory");
      if (warp == 0 && lane < 8) {
        double tot = 0.0;
        for (int w = 0; w < NCW; ++w) tot += ssq[w][lane];
        p.tsumsq[tile * kConsumerWarps + lane] = tot;
      }
      asm volatile("bar.sync 1, %0;\n" ::"r"(NCW * 32) : "memory");
    }
    if (++st == nst) {
      st = 0;
      ph ^= 1u;
    }
  }
  // c[i] = C[16 mi + g + 8 (i >> 1)][8 nj + 2t + (i & 1)], nj = 2p + h
  double* out = p.partials + (long long)blockIdx.x * p.a8 * p.a8;
#pragma unroll
  for (int u = 0; u < MAXG; ++u) {
    if (!live[u]) continue;
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = 16 * gmi[u] + g + 8 * (i >> 1);
        const int c = 8 * (2 * gp[u] + h) + 2 * t + (i & 1);
        if (r < p.a8 && c < p.a8) out[r + (long long)p.a8 * c] = acc[u][h][i];
      }
  }
}

// per-observation sums from per-(tile, warp) partials (tiles never straddle
// observations): one block per observation, fixed assignment + fixed tree
__global__ void k_tiles_to_obs(const double* __restrict__ ts, long long tiles_per_obs, int nobs,
                               double* __restrict__ on2, double* __restrict__ unused) {
  griddep_wait();
  __shared__ double red[32];
  const long long per_obs = tiles_per_obs * kConsumerWarps;
  const int o = blockIdx.x;
  const double* src = ts + (long long)o * per_obs;
  double s = 0.0;
  for (long long k = threadIdx.x; k < per_obs; k += blockDim.x) s += src[k];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];
    on2[o] = tot;
  }
}

// total = sum_o v[o] in observation order (one thread: the reference's order)
__global__ void k_sum_vec(const double* __restrict__ v, int n, double* __restrict__ total) {
  griddep_wait();
  // the block stages chunks (coalesced, many loads in flight); thread 0 adds
  // them in index order, so the sum is bit-identical to a serial pass
  __shared__ double buf[1024];
  double s = 0.0;
  for (int base = 0; base < n; base += 1024) {
    const int m = min(1024, n - base);
#pragma unroll 4
    for (int i = threadIdx.x; i < m; i += blockDim.x) buf[i] = __ldg(v + base + i);
    __syncthreads();
    if (threadIdx.x == 0)
      for (int i = 0; i < m; ++i) s += buf[i];
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = s;
}


// zero the columns of observations that are not selected
__global__ void k_mask_cols(double* __restrict__ X, int a, long long L, const uint8_t* __restrict__ sel,
                            long long cpo) {
  griddep_wait();
  long long n = (long long)a * L;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    long long q = e / a;
    if (!sel[q / cpo]) X[e] = 0.0;
  }
}

}  // namespace ttg
