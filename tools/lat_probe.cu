// Latency probe (one warp, dependent chains): DFMA, DMUL, rcp.approx.f64, SHFL, redux.sync, LDS, FFMA.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, unsigned long long* t, double x0, int n) {
  __shared__ double sm[64];
  sm[threadIdx.x] = x0;
  __syncwarp();
  double x = x0 + threadIdx.x * 1e-9;
  unsigned long long a, b;
  a = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, 0.999999, 1e-7);
  b = clock64(); t[0] = b - a; a = b;
  for (int i = 0; i < n; ++i) x = x * 1.0000001;
  b = clock64(); t[1] = b - a; a = b;
  for (int i = 0; i < n; ++i) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r; }
  b = clock64(); t[2] = b - a; a = b;
  for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31);
  b = clock64(); t[3] = b - a; a = b;
  unsigned u = threadIdx.x;
  for (int i = 0; i < n; ++i) u = __reduce_max_sync(0xffffffffu, u) + threadIdx.x;
  b = clock64(); t[4] = b - a; a = b;
  int idx = threadIdx.x;
  for (int i = 0; i < n; ++i) { x += sm[idx & 63]; idx = (int)x & 31; }
  b = clock64(); t[5] = b - a; a = b;
  float f = x;
  for (int i = 0; i < n; ++i) f = fmaf(f, 0.999f, 1e-3f);
  b = clock64(); t[6] = b - a; a = b;
  for (int i = 0; i < n; ++i) x = 1.0 / x;
  b = clock64(); t[7] = b - a; a = b;
  for (int i = 0; i < n; ++i) x = fabs(x) + 1e-9;
  b = clock64(); t[8] = b - a;
  out[threadIdx.x] = x + f + u;
}
int main() {
  double* o; unsigned long long* t; cudaMalloc(&o, 256); cudaMallocManaged(&t, 16 * 8);
  const int n = 1000;
  k<<<1, 32>>>(o, t, 1.5, n); cudaDeviceSynchronize();
  k<<<1, 32>>>(o, t, 1.5, n); cudaDeviceSynchronize();
  const char* names[] = {"DFMA", "DMUL", "rcp.approx.f64", "SHFL", "REDUX", "LDS(+DADD+cvt)", "FFMA", "1.0/x (div)", "fabs+DADD"};
  for (int i = 0; i < 9; ++i) printf("%-18s %.1f clk/op\n", names[i], double(t[i]) / n);
  return 0;
}
