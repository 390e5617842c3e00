// Isolated timing + stall profile of the speculative panel factorization (one warp per CTA, many CTAs).
#include <cstdio>
#include "rbns_bgj.cuh"
using namespace rbns;
__global__ void k(unsigned long long* t, int N, int P, int reps) {
  extern __shared__ __align__(16) unsigned char smem[];
  auto& sh = *reinterpret_cast<BGJShared<13, 13, 8>*>(smem);
  __shared__ double saved[104 * 9];
  const int lane = threadIdx.x;
  for (int e = lane; e < 104 * 9; e += 32) saved[e] = (e % 9 == e / 9) ? 4.0 : 0.01 * ((e * 7) % 13);
  if (lane == 0) { sh.sing = 0; sh.fail = 0; sh.nc[0] = sh.nc[1] = sh.nc[2] = 0; }
  __syncwarp();
  unsigned long long acc = 0;
  for (int rep = 0; rep < reps; ++rep) {
    for (int e = lane; e < 104 * 9; e += 32) sh.panel[e] = saved[e];
    __syncwarp();
    unsigned long long a = clock64();
    bgj_factor_spec<13, 13, 8>(P, 1, N, sh);
    __syncwarp();
    acc += clock64() - a;
  }
  if (lane == 0 && blockIdx.x == 0) { t[0] = acc; t[1] = sh.fail; t[2] = sh.sing; }
}
int main() {
  unsigned long long* t; cudaMallocManaged(&t, 64);
  size_t sm = sizeof(BGJShared<13, 13, 8>);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  const int reps = 400;
  k<<<1, 32, sm>>>(t, 100, 0, reps); cudaDeviceSynchronize();
  k<<<1, 32, sm>>>(t, 100, 0, reps); cudaDeviceSynchronize();
  printf("factor_spec P=0: %.0f clk per panel (factor only) fail %llu sing %llu err=%s\n", double(t[0]) / reps, t[1], t[2],
         cudaGetErrorString(cudaGetLastError()));
  k<<<148, 32, sm>>>(t, 100, 0, reps); cudaDeviceSynchronize();
  return 0;
}
