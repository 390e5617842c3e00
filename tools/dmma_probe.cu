// DMMA.8x8x4 latency / single-warp throughput on this GPU (development probe).
#include <cstdio>
#include "rbns_common.cuh"
using namespace rbns;
template <int NACC>
__global__ void k(double* out, long long* t, int reps) {
  double acc[NACC][2];
  for (int i = 0; i < NACC; ++i) acc[i][0] = acc[i][1] = threadIdx.x * 1e-3;
  double a = 1.0 + threadIdx.x * 1e-6, b = 0.999;
  __syncwarp();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) dmma_8x8x4(acc[i][0], acc[i][1], a, b);
  }
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) t[blockIdx.x] = t1 - t0;
}
template <int NACC>
void run(int warps_per_sm_sub) {
  double* o; long long* t;
  cudaMallocManaged(&o, 1024 * 8); cudaMallocManaged(&t, 1024 * 8);
  const int reps = 2000;
  k<NACC><<<1, 32 * warps_per_sm_sub>>>(o, t, reps); cudaDeviceSynchronize();
  k<NACC><<<1, 32 * warps_per_sm_sub>>>(o, t, reps); cudaDeviceSynchronize();
  printf("NACC=%2d warps/CTA=%d: %.1f clk per DMMA per warp (%s)\n", NACC, warps_per_sm_sub,
         double(t[0]) / (reps * NACC), cudaGetErrorString(cudaGetLastError()));
}
int main() {
  run<1>(1); run<2>(1); run<4>(1); run<8>(1); run<16>(1);
  run<16>(4); run<16>(8);
  return 0;
}
