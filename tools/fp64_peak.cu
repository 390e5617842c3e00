// FP64 throughput probe for the roofline denominator (run on the B200 box).
// Measures: DMMA m8n8k4 / m16n8k4 / m16n8k8 / m16n8k16 issue-bound throughput and
// DFMA (FP64 FMA pipe) throughput, all with independent accumulator chains.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int ITERS>
__global__ void k_m8n8k4(double* out, double seed) {
  double a = seed + threadIdx.x * 1e-3, b = seed * 0.5;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int ITERS>
__global__ void k_m16n8k4(double* out, double seed) {
  double a0 = seed + threadIdx.x * 1e-3, a1 = seed * 0.25, b = seed * 0.5;
  double c[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int ITERS>
__global__ void k_m16n8k16(double* out, double seed) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed + i * 1e-3 + threadIdx.x * 1e-6;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = seed * 0.5 + i;
  double c[2][4];
#pragma unroll
  for (int i = 0; i < 2; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 2; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 2; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int ITERS>
__global__ void k_dfma(double* out, double seed) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = seed + i + threadIdx.x * 1e-6;
  const double m = 0.999999, ad = 1e-7;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], m, ad);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename K>
static float timeit(K kern, int grid, int block, double* out) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<grid, block>>>(out, 1.0);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    kern<<<grid, block>>>(out, 1.0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int sms = p.multiProcessorCount;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"smem_optin\": %zu, \"clock_khz\": %d}\n",
         p.name, sms, p.l2CacheSize, p.sharedMemPerBlockOptin, p.clockRate);
  double* out; CK(cudaMalloc(&out, sizeof(double) * sms * 64 * 1024));
  const int IT = 4096;
  for (int wpb : {4, 8, 16}) {
    int block = 32 * wpb, grid = sms * 2;
    double nw = double(grid) * wpb;
    float t;
    t = timeit(k_m8n8k4<IT>, grid, block, out);
    printf("{\"op\": \"dmma_m8n8k4\", \"warps_per_block\": %d, \"tflops\": %.3f}\n", wpb, nw * IT * 8 * 512.0 / (t * 1e-3) / 1e12);
    t = timeit(k_m16n8k4<IT>, grid, block, out);
    printf("{\"op\": \"dmma_m16n8k4\", \"warps_per_block\": %d, \"tflops\": %.3f}\n", wpb, nw * IT * 4 * 1024.0 / (t * 1e-3) / 1e12);
    t = timeit(k_m16n8k16<IT>, grid, block, out);
    printf("{\"op\": \"dmma_m16n8k16\", \"warps_per_block\": %d, \"tflops\": %.3f}\n", wpb, nw * IT * 2 * 4096.0 / (t * 1e-3) / 1e12);
    t = timeit(k_dfma<IT>, grid, block, out);
    printf("{\"op\": \"dfma\", \"warps_per_block\": %d, \"tflops\": %.3f}\n", wpb, nw * 32 * IT * 8 * 2.0 / (t * 1e-3) / 1e12);
  }
  CK(cudaGetLastError());
  return 0;
}
