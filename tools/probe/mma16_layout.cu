// Verifies the register fragment layout assumed for mma.m16n8k16.f64:
//   A (16x16, row): a[i] = A[g + 8*(i&1)][t + 4*(i>>1)]   i = 0..7
//   B (16x8, col):  b[i] = B[t + 4*i][g]                    i = 0..3
//   C (16x8):       c[i] = C[g + 8*(i>>1)][2t + (i&1)]      i = 0..3
// (lane = 4g + t).  Prints the max abs error against a host product.
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>

__global__ void k(const double* A, const double* B, double* C) {
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double a[8], b[4], c[4] = {0, 0, 0, 0};
  for (int i = 0; i < 8; ++i) a[i] = A[(g + 8 * (i & 1)) * 16 + t + 4 * (i >> 1)];
  for (int i = 0; i < 4; ++i) b[i] = B[(t + 4 * i) * 8 + g];
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
      "{%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]),
        "d"(b[1]), "d"(b[2]), "d"(b[3]));
  for (int i = 0; i < 4; ++i) C[(g + 8 * (i >> 1)) * 8 + 2 * t + (i & 1)] = c[i];
}

int main() {
  double hA[256], hB[128], hC[128], ref[128];
  for (int i = 0; i < 256; ++i) hA[i] = std::sin(1.0 + i);
  for (int i = 0; i < 128; ++i) hB[i] = std::cos(2.0 + 3 * i);
  for (int m = 0; m < 16; ++m)
    for (int n = 0; n < 8; ++n) {
      double s = 0;
      for (int kk = 0; kk < 16; ++kk) s += hA[m * 16 + kk] * hB[kk * 8 + n];
      ref[m * 8 + n] = s;
    }
  double *A, *B, *C;
  cudaMalloc(&A, sizeof hA); cudaMalloc(&B, sizeof hB); cudaMalloc(&C, sizeof hC);
  cudaMemcpy(A, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB, sizeof hB, cudaMemcpyHostToDevice);
  k<<<1, 32>>>(A, B, C);
  cudaMemcpy(hC, C, sizeof hC, cudaMemcpyDeviceToHost);
  double err = 0;
  for (int i = 0; i < 128; ++i) err = fmax(err, fabs(hC[i] - ref[i]));
  printf("m16n8k16 f64 layout max err %.3e (%s)\n", err, cudaGetErrorString(cudaGetLastError()));
  int main2();
  return main2();
}

// dependent-chain latency of m8n8k4 and m16n8k16 f64 (one warp, cycles / MMA)
__global__ void lat(double* out, long long* cyc, int n) {
  double a8[8], b4[4], c4[4] = {0, 0, 0, 0};
  for (int i = 0; i < 8; ++i) a8[i] = 1e-3 * (threadIdx.x + i);
  for (int i = 0; i < 4; ++i) b4[i] = 1e-3 * i;
  double c0 = 0, c1 = 0, a = 1e-3 * threadIdx.x, b = 0.5;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  long long t1 = clock64();
  for (int i = 0; i < n; ++i)
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
        "{%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
        : "+d"(c4[0]), "+d"(c4[1]), "+d"(c4[2]), "+d"(c4[3])
        : "d"(a8[0]), "d"(a8[1]), "d"(a8[2]), "d"(a8[3]), "d"(a8[4]), "d"(a8[5]), "d"(a8[6]), "d"(a8[7]), "d"(b4[0]),
          "d"(b4[1]), "d"(b4[2]), "d"(b4[3]));
  long long t2 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; }
  out[threadIdx.x] = c0 + c1 + c4[0] + c4[1] + c4[2] + c4[3];
}

int main2() {
  double* o; long long* c; cudaMalloc(&o, 256 * 8); cudaMalloc(&c, 16);
  lat<<<1, 32>>>(o, c, 1000);
  long long h[2]; cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
  printf("dependent chain: m8n8k4 %.1f cycles/MMA, m16n8k16 %.1f cycles/MMA\n", h[0] / 1000.0, h[1] / 1000.0);
  return 0;
}
