// Pure streaming with tensor-map TMA (2-D boxes of 16 rows x TC columns, 128B
// swizzle) vs. 1-D bulk copies: bandwidth as a function of box width, ring
// depth and CTAs / SM, with no compute (thread 0 issues, all threads wait).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -I paper_2211_12487_b200/csrc tools/probe/tmap_probe.cu
#include <cstdio>
#include <cudaTypedefs.h>
#include "ttg_eig.cuh"
#include "ttg_kernels.cuh"

CUtensorMap make_map(const double* X, int a, long long L, int bc) {
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
  enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)X, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return m;
}

// MODE 0: tensor boxes; MODE 1: one 1-D bulk copy per tile
template <int MODE>
__global__ void __launch_bounds__(256) k_stream(const __grid_constant__ CUtensorMap tm, const double* X, int a, int tc,
                                                long long ntiles, int nst, double* out) {
  extern __shared__ __align__(1024) double raw[];
  __shared__ __align__(8) uint64_t full[16];
  double* sm = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  const int nbox = a / 16, stage = a * tc;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) ttg::mbar_init(&full[s], 1);
    ttg::fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](long long tile, int s) {
    ttg::mbar_expect_tx(&full[s], (unsigned)stage * 8u);
    if (MODE == 0)
      for (int b = 0; b < nbox; ++b) ttg::tma_load_2d(sm + s * stage + b * 16 * tc, &tm, 16 * b, (int)(tile * tc), &full[s]);
    else
      ttg::bulk_g2s(sm + s * stage, X + tile * stage, (unsigned)stage * 8u, &full[s]);
  };
  if (threadIdx.x == 0)
    for (int s = 0; s < nst - 1; ++s) {
      const long long t = blockIdx.x + (long long)s * gridDim.x;
      if (t < ntiles) issue(t, s);
    }
  double acc = 0.0;
  int it = 0;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int st = it % nst;
    ttg::mbar_wait(&full[st], (unsigned)((it / nst) & 1));
    __syncthreads();
    if (threadIdx.x == 0) {
      const long long t = tile + (long long)(nst - 1) * gridDim.x;
      if (t < ntiles) issue(t, (it + nst - 1) % nst);
    }
    acc += sm[st * stage + threadIdx.x];
  }
  if (acc == 123.456) out[0] = acc;
}

int main() {
  const long long bytes = 1ll << 32;
  double* X;
  cudaMalloc(&X, bytes);
  cudaMemset(X, 0, bytes);
  double* out;
  cudaMalloc(&out, 64);
  for (int a : {64, 128}) {
    for (int tc : {32, 64}) {
      const long long L = bytes / 8 / a;
      const CUtensorMap tm = make_map(X, a, L, tc);
      const long long ntiles = L / tc;
      const size_t stage = (size_t)a * tc * 8;
      for (int mode = 0; mode < 2; ++mode)
        for (int nst : {2, 3, 4, 6, 8}) {
          const size_t smem = nst * stage + 1024;
          if (smem > 220 * 1024) continue;
          auto k = mode == 0 ? k_stream<0> : k_stream<1>;
          cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
          int occ = 0;
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 256, smem);
          for (int o = 1; o <= occ; ++o) {
            k<<<148 * o, 256, smem>>>(tm, X, a, tc, ntiles, nst, out);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            for (int i = 0; i < 3; ++i) k<<<148 * o, 256, smem>>>(tm, X, a, tc, ntiles, nst, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("%s a=%3d tc=%2d nst=%d ctas/sm=%d  %.0f GB/s  (%s)\n", mode ? "bulk1d" : "tmap  ", a, tc, nst, o,
                   3.0 * bytes / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
          }
        }
    }
  }
  return 0;
}
