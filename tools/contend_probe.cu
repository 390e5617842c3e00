// Does a dependent DFMA chain slow down while another warp on the same SMSP issues DMMAs back to back?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, unsigned long long* t, int n, int mode) {
  const int warp = threadIdx.x >> 5;
  double x = 1.0 + threadIdx.x * 1e-9;
  if (warp == 0) {
    unsigned long long a = clock64();
    for (int i = 0; i < n; ++i) x = fma(x, 0.999999, 1e-7);
    t[0] = clock64() - a;
  } else if (mode == 1 && (warp % 4) == 0) {  // same SMSP as warp 0: DMMA stream
    double c[8][2] = {};
    for (int i = 0; i < 4 * n / 16; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(x), "d"(x));
    x += c[0][0] + c[7][1];
  } else if (mode == 2 && (warp % 4) == 0) {  // same SMSP: DFMA stream
    double y[8];
    for (int j = 0; j < 8; ++j) y[j] = x + j;
    for (int i = 0; i < 2 * n; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) y[j] = fma(y[j], 0.999, 1e-3);
    x += y[0] + y[7];
  }
  out[threadIdx.x] = x;
}
int main() {
  double* o; unsigned long long* t; cudaMalloc(&o, 8 * 256); cudaMallocManaged(&t, 64);
  const int n = 2000;
  for (int mode = 0; mode < 3; ++mode) {
    k<<<1, 256>>>(o, t, n, mode); cudaDeviceSynchronize();
    k<<<1, 256>>>(o, t, n, mode); cudaDeviceSynchronize();
    printf("mode %d (%s): DFMA chain %.1f clk/op\n", mode, mode == 0 ? "alone" : mode == 1 ? "with DMMA stream" : "with DFMA stream", double(t[0]) / n);
  }
  return 0;
}
