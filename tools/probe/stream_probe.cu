// Streaming-load probe for B200: how fast can a CTA ring pull 64 x 64-double
// column tiles from HBM with (A) one cp.async.bulk per 512-byte column,
// (B) one 32 KB cp.async.bulk per tile, (C) 16-byte cp.async by all threads.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(c)); }
__device__ __forceinline__ void expect_tx(uint64_t* b, unsigned n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void mwait(uint64_t* b, unsigned ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void* d, const void* s, unsigned n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(d)), "l"(s), "r"(n), "r"(su(b)) : "memory");
}

template <int MODE, int NST>
__global__ void __launch_bounds__(256) k_stream(const double* X, long long ntiles, double* out) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t full[NST];
  const int ld = (MODE == 1) ? 64 : 68;
  const int stage = ld * 64;
  if (threadIdx.x == 0) for (int s = 0; s < NST; ++s) mbar_init(&full[s], 1);
  __syncthreads();
  double acc = 0.0;
  auto issue = [&](long long tile, int s) {
    const double* src = X + tile * 4096;
    double* dst = sm + s * stage;
    if (MODE == 0) {
      if (threadIdx.x < 32) {
        if (threadIdx.x == 0) expect_tx(&full[s], 64 * 512);
        __syncwarp();
        bulk(dst + ld * threadIdx.x, src + 64 * threadIdx.x, 512, &full[s]);
        bulk(dst + ld * (threadIdx.x + 32), src + 64 * (threadIdx.x + 32), 512, &full[s]);
      }
    } else if (MODE == 1) {
      if (threadIdx.x == 0) { expect_tx(&full[s], 32768); bulk(dst, src, 32768, &full[s]); }
    } else {
      for (int e = threadIdx.x; e < 2048; e += 256) {
        const int c = (2 * e) / 64, r = (2 * e) % 64;
        unsigned d = su(dst + r + ld * c);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src + 2 * e));
      }
      asm volatile("cp.async.commit_group;");
    }
  };
  int it = 0;
  for (int s = 0; s < NST - 1; ++s) {
    long long t = blockIdx.x + (long long)s * gridDim.x;
    if (t < ntiles) issue(t, s);
    else if (MODE == 2) asm volatile("cp.async.commit_group;");
  }
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int st = it % NST;
    long long tn = tile + (long long)(NST - 1) * gridDim.x;
    if (tn < ntiles) issue(tn, (it + NST - 1) % NST);
    else if (MODE == 2) asm volatile("cp.async.commit_group;");
    if (MODE == 2) { asm volatile("cp.async.wait_group %0;" ::"n"(NST - 1)); }
    else mwait(&full[st], (it / NST) & 1);
    __syncthreads();
    const double* T = sm + st * stage;
    for (int e = threadIdx.x; e < 4096; e += 256) acc += T[(e & 63) + ld * (e >> 6)];
    __syncthreads();
  }
  if (acc == 123.456) out[0] = acc;
}

template <int MODE, int NST>
void run(const double* X, long long ntiles, double* out, int sms, const char* name) {
  const int ld = MODE == 1 ? 64 : 68;
  size_t smem = (size_t)NST * ld * 64 * 8;
  cudaFuncSetAttribute(k_stream<MODE, NST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_stream<MODE, NST>, 256, smem);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  k_stream<MODE, NST><<<sms * occ, 256, smem>>>(X, ntiles, out);
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) k_stream<MODE, NST><<<sms * occ, 256, smem>>>(X, ntiles, out);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("%-28s NST=%d occ=%d  %.1f GB/s  (%s)\n", name, NST, occ, 5.0 * ntiles * 32768 / (ms * 1e-3) / 1e9,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  long long ntiles = 131072;  // 4.29 GB
  double* X; cudaMalloc(&X, ntiles * 32768); cudaMemset(X, 0, ntiles * 32768);
  double* out; cudaMalloc(&out, 64);
  int sms = 148;
  run<0, 2>(X, ntiles, out, sms, "per-column bulk");
  run<0, 3>(X, ntiles, out, sms, "per-column bulk");
  run<0, 4>(X, ntiles, out, sms, "per-column bulk");
  run<0, 6>(X, ntiles, out, sms, "per-column bulk");
  run<1, 2>(X, ntiles, out, sms, "whole-tile bulk");
  run<1, 4>(X, ntiles, out, sms, "whole-tile bulk");
  run<1, 6>(X, ntiles, out, sms, "whole-tile bulk");
  run<2, 2>(X, ntiles, out, sms, "cp.async 16B");
  run<2, 4>(X, ntiles, out, sms, "cp.async 16B");
  return 0;
}
