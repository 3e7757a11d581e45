// Isolated timing of the projection kernels (out = W^T X, a = 64) on a 4.29 GB
// operand: ring vs. double-buffered TMA, r = 1 / 16, with/without norms.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -I paper_2211_12487_b200/csrc tools/probe/proj_probe.cu
#include <cstdio>
#include <cstdlib>
#include "ttg_eig.cuh"
#include "ttg_kernels.cuh"

__global__ void fill(double* x, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    x[i] = (double)((i * 2654435761ull) % 1000) * 1e-3 - 0.5;
}

#include <cudaTypedefs.h>
CUtensorMap make_map(const double* X, int a, long long L, int bc = 64) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  }
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)a, (cuuint64_t)L};
  cuuint64_t strides[1] = {(cuuint64_t)a * 8};
  cuuint32_t box[2] = {16, (cuuint32_t)bc};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)X, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
  return m;
}
template <class K>
void timetma(const char* name, K kern, const CUtensorMap& tm, ttg::ProjArgs p, size_t smem, double bytes,
             int threads = ttg::kThreads);
void ws16_sweep(const double* X, int a, long long L, const double* W, double* out, int r) {
  ttg::ProjArgs p{};
  p.src = ttg::TileSrc{X, a, L, nullptr, 1};
  p.a8 = a; p.ldt = ttg::smem_ld(a); p.WTf = W; p.r = r; p.r8 = (r + 7) / 8 * 8; p.out = out; p.tsumsq = nullptr;
  const double bytes = 8.0 * (a + r) * L;
  const int nks = (a + 15) / 16, NB = p.r8 / 8;
  char nm[96];
  for (int ncw : {4, 8}) {
    const int tc = 16 * ncw;
    const CUtensorMap tm = make_map(X, a, L, tc);
    p.n_tiles = (L + tc - 1) / tc;
    for (int nst : {2, 3, 4, 6}) {
      p.nst = nst;
      const size_t smem = 1024 + (size_t)nst * nks * 16 * tc * 8 + nks * NB * 128 * 8 + ncw * 16 * 32 * 8;
      if (smem > 227 * 1024) continue;
      std::snprintf(nm, sizeof nm, "ws16 a=%d r=%d ncw=%d", a, r, ncw);
#define RUNWS(NC, N) timetma(nm, ttg::k_project_ws16<NC, N>, tm, p, smem, bytes, (NC + 1) * 32)
      if (ncw == 4) { if (NB == 1) RUNWS(4, 1); else if (NB == 2) RUNWS(4, 2); else if (NB == 3) RUNWS(4, 3); else RUNWS(4, 4); }
      else { if (NB == 1) RUNWS(8, 1); else if (NB == 2) RUNWS(8, 2); else if (NB == 3) RUNWS(8, 3); else RUNWS(8, 4); }
    }
  }
}
template <class K>
void timetma(const char* name, K kern, const CUtensorMap& tm, ttg::ProjArgs p, size_t smem, double bytes,
             int threads) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem);
  const int gx = 148 * (occ > 0 ? occ : 1);
  kern<<<gx, threads, smem>>>(tm, p);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) kern<<<gx, threads, smem>>>(tm, p);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  ms /= 5;
  printf("%-44s smem=%6zu occ=%d nst=%d  %.3f ms  %.0f GB/s  (%s)\n", name, smem, occ, p.nst, ms, bytes / (ms * 1e-3) / 1e9,
         cudaGetErrorString(cudaGetLastError()));
}
// correctness: out (r x L) vs a plain reference on the first columns
__global__ void ref_proj(const double* X, int a, const double* W, int r, double* out, long long n) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n * r) return;
  long long c = i / r;
  int j = (int)(i % r);
  double s = 0;
  for (int k = 0; k < a; ++k) s += W[k + (long long)a * j] * X[k + (long long)a * c];
  out[i] = s;
}
template <class K>
void timeit(const char* name, K kern, ttg::ProjArgs p, size_t smem, double bytes) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, ttg::kThreads, smem);
  const int gx = 148 * (occ > 0 ? occ : 1);
  kern<<<gx, ttg::kThreads, smem>>>(p);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) kern<<<gx, ttg::kThreads, smem>>>(p);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  ms /= 5;
  printf("%-44s smem=%6zu occ=%d nst=%d  %.3f ms  %.0f GB/s  (%s)\n", name, smem, occ, p.nst, ms, bytes / (ms * 1e-3) / 1e9,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const int a = 64;
  const long long L = 1ll << 23;
  double* X;
  cudaMalloc(&X, sizeof(double) * a * L);
  fill<<<4096, 256>>>(X, a * L);
  double *W, *out, *tsq;
  cudaMalloc(&W, sizeof(double) * 128 * 64);
  fill<<<16, 256>>>(W, 128 * 64);
  cudaMalloc(&out, sizeof(double) * 32 * L);
  cudaMalloc(&tsq, sizeof(double) * 8 * (L / 64));
  if (getenv("PROBE_WS16")) {
    ws16_sweep(X, 64, L, W, out, 17);
    ws16_sweep(X, 64, L, W, out, 16);
    ws16_sweep(X, 64, L, W, out, 1);
    ws16_sweep(X, 144, (1ll << 32) / (8 * 144), W, out, 18);
    ws16_sweep(X, 128, (1ll << 32) / (8 * 128), W, out, 16);
    return 0;
  }
  if (getenv("PROBE_R17")) {
    ttg::ProjArgs p{};
    p.src = ttg::TileSrc{X, a, L, nullptr, 1};
    p.a8 = 64; p.ldt = ttg::smem_ld(64); p.WTf = W; p.r = 17; p.r8 = 24; p.out = out; p.tsumsq = nullptr;
    const double bytes = 8.0 * (a + 17) * L;
    const size_t stg = sizeof(double) * 8 * 8 * 32;
    const CUtensorMap tm64 = make_map(X, a, L, 64), tm32 = make_map(X, a, L, 32);
    for (int nst : {2, 3, 4, 6, 8}) {
      p.nst = nst; p.n_tiles = L / 32; p.frag_smem = 0;
      timetma("r17 TC32 REGW", ttg::k_project_tma<true, 32>, tm32, p, 1024 + nst * 16384 + stg, bytes);
      p.n_tiles = L / 64;
      if (nst <= 4) timetma("r17 TC64 Wglobal", ttg::k_project_tma<false, 64>, tm64, p, 1024 + nst * 32768 + stg, bytes);
      if (nst <= 4) timetma("r17 W2", ttg::k_project_w2, tm64, p, 1024 + nst * 32768 + 8 * 16 * 32 * 8, bytes);
      if (nst <= 4) timetma("r17 M16", ttg::k_project_m16, tm64, p, 1024 + nst * 32768 + 8 * 16 * 32 * 8 + 3 * 16 * 32 * 8, bytes);
      p.frag_smem = 1;
      if (nst <= 4) timetma("r17 TC64 Wsmem", ttg::k_project_tma<false, 64>, tm64, p, 1024 + nst * 32768 + stg + 3 * 16 * 32 * 8, bytes);
    }
    p.r = 16; p.r8 = 16; p.frag_smem = 0;
    for (int nst : {2, 3, 4, 6}) {
      p.nst = nst; p.n_tiles = L / 32;
      timetma("r16 TC32 REGW", ttg::k_project_tma<true, 32>, tm32, p, 1024 + nst * 16384 + stg, 8.0 * (a + 16) * L);
      p.n_tiles = L / 64;
      if (nst <= 4) timetma("r16 TC64 REGW", ttg::k_project_tma<true, 64>, tm64, p, 1024 + nst * 32768 + stg, 8.0 * (a + 16) * L);
      if (nst <= 4) timetma("r16 M16", ttg::k_project_m16, tm64, p, 1024 + nst * 32768 + 8 * 16 * 32 * 8 + 2 * 16 * 32 * 8, 8.0 * (a + 16) * L);
    }
    return 0;
  }
  for (int r : {1, 16}) {
    for (int norms = 0; norms < 2; ++norms) {
      ttg::ProjArgs p{};
      p.src = ttg::TileSrc{X, a, L, nullptr, 1};
      p.a8 = 64;
      p.ldt = ttg::smem_ld(64);
      p.WTf = W;
      p.r = r;
      p.r8 = ttg::round_up(r, 8);
      p.out = out;
      p.tsumsq = norms ? tsq : nullptr;
      p.n_tiles = L / 64;
      const double bytes = 8.0 * (a + r) * L;
      const size_t stage = sizeof(double) * p.ldt * 64;
      const size_t stg = sizeof(double) * 8 * 8 * 32;
      char nm[128];
      const CUtensorMap tm = make_map(X, a, L);
      for (int nst : {2, 3, 4, 6}) {
        p.nst = nst;
        std::snprintf(nm, sizeof nm, "tmap r=%d norms=%d", r, norms);
        timetma(nm, ttg::k_project_tma<true, 64>, tm, p, 1024 + nst * 8192 * 4 + stg, bytes);
      }
      for (int nst : {6, 8, 11, 16}) {
        p.nst = nst;
        std::snprintf(nm, sizeof nm, "box r=%d norms=%d", r, norms);
        if (r <= 16)
          timetma(nm, ttg::k_project_box<2, true>, tm, p, 1024 + nst * 8192 + stg, bytes, ttg::kSyrkThreads);
        std::snprintf(nm, sizeof nm, "box-smemW r=%d norms=%d", r, norms);
        p.frag_smem = 1;
        timetma(nm, ttg::k_project_box<4, false>, tm, p, 1024 + nst * 8192 + stg + 8 * 4 * 16 * 32, bytes, ttg::kSyrkThreads);
        p.frag_smem = 0;
      }
      p.nst = 0;
      std::snprintf(nm, sizeof nm, "tma-db r=%d norms=%d", r, norms);
      timeit(nm, ttg::k_project<true, true>, p, 2 * stage, bytes);
    }
  }
  {  // a = 144 (cur_2-like), r = 18
    const int a2 = 144, r2 = 18;
    const long long L2 = (1ll << 32) / (8 * a2) / 64 * 64;
    ttg::ProjArgs p{};
    p.src = ttg::TileSrc{X, a2, L2, nullptr, 1};
    p.a8 = a2;
    p.ldt = ttg::smem_ld(a2);
    p.WTf = W;
    p.r = r2;
    p.r8 = 24;
    p.out = out;
    p.n_tiles = L2 / 64;
    const double bytes = 8.0 * (a2 + r2) * L2;
    const CUtensorMap tm = make_map(X, a2, L2);
    char nm[128];
    for (int nst : {6, 8, 11, 16}) {
      p.nst = nst;
      std::snprintf(nm, sizeof nm, "box a=144 r=18 (W global)");
      timetma(nm, ttg::k_project_box<4, false>, tm, p, 1024 + nst * 8192 + 8 * 8 * 32 * 8, bytes, ttg::kSyrkThreads);
    }
    {
      const CUtensorMap tm32 = make_map(X, a2, L2, 32);
      ttg::ProjArgs q = p;
      q.n_tiles = L2 / 32;
      for (int nst : {2, 3}) {
        q.nst = nst;
        timetma("tmap32 a=144 r=18 (W global)", ttg::k_project_tma<false, 32>, tm32, q, 1024 + nst * 9 * 4096 + 8 * 8 * 32 * 8, bytes);
      }
      const CUtensorMap tm32b = make_map(X, 128, (1ll << 32) / (8 * 128));
      q.src = ttg::TileSrc{X, 128, (1ll << 32) / (8 * 128), nullptr, 1};
      q.a8 = 128; q.r = 16; q.r8 = 16; q.n_tiles = q.src.L / 32;
      const CUtensorMap tm128 = make_map(X, 128, q.src.L, 32);
      for (int nst : {2, 3}) {
        q.nst = nst;
        timetma("tmap32 a=128 r=16 (W global)", ttg::k_project_tma<false, 32>, tm128, q, 1024 + nst * 8 * 4096 + 8 * 8 * 32 * 8, 8.0 * 144 * q.src.L);
      }
    }
    p.nst = 0;
    timeit("old single-buffer a=144 r=18", ttg::k_project<false, false>, p, sizeof(double) * p.ldt * 64, bytes);
  }
  return 0;
}
