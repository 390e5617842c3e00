// Single-warp issue throughput of independent SHFL / DFMA / LDS streams.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, unsigned long long* t, int n) {
  __shared__ double sm[256];
  sm[threadIdx.x] = threadIdx.x; sm[threadIdx.x + 32] = 1.0;
  __syncwarp();
  double x[16];
  for (int j = 0; j < 16; ++j) x[j] = threadIdx.x + j;
  unsigned long long a = clock64();
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int j = 0; j < 16; ++j) x[j] = __shfl_sync(0xffffffffu, x[j], (threadIdx.x + j + 1) & 31);
  unsigned long long b = clock64(); t[0] = b - a; a = b;
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int j = 0; j < 16; ++j) x[j] = fma(x[j], 0.999, 1e-3);
  b = clock64(); t[1] = b - a; a = b;
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int j = 0; j < 16; ++j) x[j] += sm[(threadIdx.x + j * 3 + i) & 63];
  b = clock64(); t[2] = b - a; a = b;
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int j = 0; j < 16; ++j) { int v = __float_as_int(float(x[j])); x[j] = (double)__shfl_sync(0xffffffffu, v, (threadIdx.x + j + 1) & 31); }
  b = clock64(); t[3] = b - a;
  double s = 0; for (int j = 0; j < 16; ++j) s += x[j];
  out[threadIdx.x] = s;
}
int main() {
  double* o; unsigned long long* t; cudaMalloc(&o, 256); cudaMallocManaged(&t, 64);
  const int n = 200;
  k<<<1, 32>>>(o, t, n); cudaDeviceSynchronize(); k<<<1, 32>>>(o, t, n); cudaDeviceSynchronize();
  printf("SHFL.64 (2 SHFL): %.2f clk per double shuffle\nDFMA indep: %.2f clk/op\nLDS.64 indep: %.2f clk/op\nSHFL.32 (+cvt): %.2f clk/op\n",
         double(t[0]) / (16.0 * n), double(t[1]) / (16.0 * n), double(t[2]) / (16.0 * n), double(t[3]) / (16.0 * n));
  return 0;
}
