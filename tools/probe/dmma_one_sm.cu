// Single-SM FP64 tensor throughput: one CTA of W warps, each issuing N
// mma.m8n8k4.f64 on C independent accumulator chains (operands in registers).
// Prints cycles per DMMA per SM.  (k_decide runs on one SM: is the DMMA rate
// per SM what the chip-wide 37 TF/s suggests, 1 per ~4 clocks?)
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int C>
__global__ void k(int n, double* out, long long* cyc) {
  double c[C][2];
  for (int i = 0; i < C; ++i) c[i][0] = c[i][1] = 0.0;
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < C; ++j) dmma(c[j][0], c[j][1], a, b);
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0.0;
  for (int i = 0; i < C; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int C>
void run(int warps, int blocks, int n) {
  double* out; long long* cyc;
  cudaMalloc(&out, sizeof(double) * 1024 * blocks); cudaMalloc(&cyc, sizeof(long long) * blocks);
  k<C><<<blocks, warps * 32>>>(n, out, cyc);
  k<C><<<blocks, warps * 32>>>(n, out, cyc);
  long long h = 0; cudaMemcpy(&h, cyc, sizeof h, cudaMemcpyDeviceToHost);
  const double total = (double)warps * n * C;
  printf("blocks %3d warps %2d chains %d: %lld cycles, %.2f cycles per DMMA per SM, %.1f flop/clk/SM\n", blocks, warps, C, h,
         h / total, total * 512.0 / h);
  cudaFree(out); cudaFree(cyc);
}
int main() {
  for (int blocks : {1, 148})
    for (int w : {1, 4, 8, 16, 32}) { run<1>(w, blocks, 2048); run<3>(w, blocks, 2048); }
  return 0;
}
