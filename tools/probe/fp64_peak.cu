// FP64 peak probe for B200 (sm_100a): DFMA chains vs DMMA (mma.sync f64) shapes.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma884_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 0.5;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma1688_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = 0.25, a2 = 0.125, a3 = 0.3, b0 = 0.5, b1 = 0.7;
  double c[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) s += c[i][j];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma16816_kernel(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 0.5 + i;
  double c[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) s += c[i][j];
  if (s == 12345.678) out[0] = s;
}

__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) b[i] = a[i];
}

template <typename F>
float time_it(F f) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  f(); cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  return best;
}

// half the warps run DMMA chains, the other half DFMA chains: do the FP64
// tensor and FP64 FMA pipes run concurrently?
__global__ void mix_kernel(double* out, int iters_mma, int iters_fma) {
  const int warp = threadIdx.x >> 5;
  double s = 0.0;
  if (warp & 1) {
    double x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters_fma; ++it) {
#pragma unroll
      for (int i = 0; i < 16; ++i) x[i] = fma(x[i], 0.999, 1e-3);
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) s += x[i];
  } else {
    double a = threadIdx.x * 1e-3, b = 0.5;
    double c[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
    for (int it = 0; it < iters_mma; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  }
  if (s == 12345.678) out[0] = s;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("device %s SMs %d smemPerBlockOptin %zu L2 %d clock %d kHz\n", p.name, p.multiProcessorCount,
         p.sharedMemPerBlockOptin, p.l2CacheSize, p.clockRate);
  double* out; cudaMalloc(&out, 64);
  int sms = p.multiProcessorCount;
  for (int bpsm : {1, 2, 4, 8}) {
    int threads = 256, iters = 4096;
    float ms = time_it([&] { dfma_kernel<<<sms * bpsm, threads>>>(out, iters, 0.999, 1e-3); });
    double fl = 2.0 * 16 * iters * (double)threads * sms * bpsm;
    printf("DFMA   blocks/SM %d: %.2f TFLOP/s\n", bpsm, fl / ms / 1e9);
  }
  for (int bpsm : {1, 2, 4, 8}) {
    int threads = 256, iters = 2048;
    float ms = time_it([&] { dmma884_kernel<<<sms * bpsm, threads>>>(out, iters); });
    double fl = 2.0 * 8 * 8 * 4 * 8 * iters * (threads / 32.0) * sms * bpsm;
    printf("DMMA m8n8k4  blocks/SM %d: %.2f TFLOP/s\n", bpsm, fl / ms / 1e9);
  }
  for (int bpsm : {1, 2, 4, 8}) {
    int threads = 256, iters = 1024;
    float ms = time_it([&] { dmma1688_kernel<<<sms * bpsm, threads>>>(out, iters); });
    double fl = 2.0 * 16 * 8 * 8 * 4 * iters * (threads / 32.0) * sms * bpsm;
    printf("DMMA m16n8k8 blocks/SM %d: %.2f TFLOP/s\n", bpsm, fl / ms / 1e9);
  }
  for (int bpsm : {1, 2, 4, 8}) {
    int threads = 256, iters = 512;
    float ms = time_it([&] { dmma16816_kernel<<<sms * bpsm, threads>>>(out, iters); });
    double fl = 2.0 * 16 * 8 * 16 * 4 * iters * (threads / 32.0) * sms * bpsm;
    printf("DMMA m16n8k16 blocks/SM %d: %.2f TFLOP/s\n", bpsm, fl / ms / 1e9);
  }
  for (int bpsm : {1, 2, 4}) {
    int threads = 512;
    // per DMMA warp: 8 x iters_mma m8n8k4 (512 flops each, per warp-instruction 32 lanes -> 8*8*4*2 flops)
    int im = 2048, iff = 4096;
    float ms = time_it([&] { mix_kernel<<<sms * bpsm, threads>>>(out, im, iff); });
    double fm = 2.0 * 8 * 8 * 4 * 8 * im * (threads / 64.0) * sms * bpsm;
    double ff = 2.0 * 16 * iff * (threads / 2.0) * sms * bpsm;
    printf("MIX blocks/SM %d: %.2f TFLOP/s total (DMMA part %.2f, DFMA part %.2f if concurrent)\n", bpsm,
           (fm + ff) / ms / 1e9, fm / ms / 1e9, ff / ms / 1e9);
  }
  size_t n = (size_t)1 << 28;  // 4 GiB of doubles as double2 pairs -> 2^28 double2 = 4 GiB
  double2 *a, *b; cudaMalloc(&a, n * 16); cudaMalloc(&b, n * 16);
  cudaMemset(a, 0, n * 16);
  float ms = time_it([&] { copy_kernel<<<sms * 8, 512>>>(a, b, n); });
  printf("copy: %.1f GB/s (read+write)\n", 2.0 * n * 16 / ms / 1e6);
  cudaError_t e = cudaGetLastError();
  printf("err: %s\n", cudaGetErrorString(e));
  return 0;
}
