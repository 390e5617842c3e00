// Isolated timing of the speculative panel factorization (one warp, nothing else on the SM).
#include <cstdio>
#include "rbns_bgj.cuh"
using namespace rbns;
__global__ void k(unsigned long long* t, int N, int P) {
  extern __shared__ __align__(16) unsigned char smem[];
  auto& sh = *reinterpret_cast<BGJShared<13, 13, 8>*>(smem);
  const int lane = threadIdx.x;
  for (int e = lane; e < 104 * 9; e += 32) sh.panel[e] = (e % 9 == e / 9) ? 4.0 : 0.01 * ((e * 7) % 13);
  if (lane == 0) { sh.sing = 0; sh.fail = 0; sh.nc[0] = sh.nc[1] = sh.nc[2] = 0; }
  __syncwarp();
  unsigned long long a = clock64();
  for (int rep = 0; rep < 200; ++rep) {
    for (int e = lane; e < 104 * 9; e += 32) sh.panel[e] = (e % 9 == e / 9) ? 4.0 : 0.01 * ((e * 7) % 13);
    __syncwarp();
    bgj_factor_spec<13, 13, 8>(P, 1, N, sh);
    __syncwarp();
  }
  unsigned long long b = clock64();
  if (lane == 0) { t[0] = b - a; t[1] = sh.fail; t[2] = sh.sing; }
}
int main() {
  unsigned long long* t; cudaMallocManaged(&t, 64);
  size_t sm = sizeof(BGJShared<13, 13, 8>);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  for (int r = 0; r < 3; ++r) { k<<<1, 32, sm>>>(t, 100, 0); cudaDeviceSynchronize(); }
  printf("factor_spec P=0 (x200 incl. reload): %llu clk (fail %llu sing %llu) err=%s\n", t[0], t[1], t[2], cudaGetErrorString(cudaGetLastError()));
  return 0;
}
