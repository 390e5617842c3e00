// Isolated timing of the Newton-update (Gauss–Jordan) kernels on a random batch, plus gj2 phase ablations
// (MODE bits: 1 no update, 2 no search, 4 no row publication).  Development tool, not part of the library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude -Ipaper_1807_11866_b200/csrc \
//        tools/lu_probe.cu -o tools/lu_probe
#include <cstdio>
#include <vector>

#include "rbns_bgj.cuh"
#include "rbns_newton.cuh"
#include "rbns_newton2.cuh"
#include "rbns_newton3.cuh"
#include "rbns_newton_spec.cuh"

using namespace rbns;

__global__ void fill(double* x, size_t n, unsigned seed) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    unsigned h = unsigned(i) * 2654435761u ^ seed;
    h ^= h >> 15; h *= 2246822519u; h ^= h >> 13; h *= 3266489917u; h ^= h >> 16;
    x[i] = (double(h) / 4294967296.0) * 2.0 - 1.0;
  }
}

using K = void (*)(const NewtonParams);
using NewtonKernel = K;

__global__ void add_diag(double* J, int64_t ldj, int N, int B, double d) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < int64_t(B) * N; i += int64_t(gridDim.x) * blockDim.x)
    J[(i / N) * ldj + (i % N) * (N + 1)] += d;
}

int main(int argc, char** argv) {
  const int N = argc > 1 ? atoi(argv[1]) : 100;
  const int B = argc > 2 ? atoi(argv[2]) : 8192;
  const int64_t ldj = int64_t(N) * N + N;
  double *J, *u, *mu, *f, *last;
  int32_t *act, *iters;
  int8_t* status;
  cudaMalloc(&J, sizeof(double) * ldj * B);
  cudaMalloc(&u, sizeof(double) * N * B);
  cudaMalloc(&mu, sizeof(double) * 2 * B);
  cudaMalloc(&f, sizeof(double) * N);
  cudaMalloc(&last, sizeof(double) * B);
  cudaMalloc(&act, sizeof(int32_t) * B);
  cudaMalloc(&iters, sizeof(int32_t) * B);
  cudaMalloc(&status, B);
  fill<<<1024, 256>>>(J, size_t(ldj) * B, 1u);
  fill<<<64, 256>>>(f, N, 2u);
  cudaMemset(u, 0, sizeof(double) * N * B);
  std::vector<int32_t> h(B);
  std::vector<double> hm(2 * B);
  for (int i = 0; i < B; ++i) { h[i] = i; hm[2 * i] = 0.3; hm[2 * i + 1] = 100.0; }
  cudaMemcpy(act, h.data(), sizeof(int32_t) * B, cudaMemcpyHostToDevice);
  cudaMemcpy(mu, hm.data(), sizeof(double) * 2 * B, cudaMemcpyHostToDevice);
  rbns_theta_term* thf;
  cudaMalloc(&thf, sizeof(rbns_theta_term));
  const rbns_theta_term one{RBNS_THETA_CONST, 0, 0, 0, 1.0};
  cudaMemcpy(thf, &one, sizeof(one), cudaMemcpyHostToDevice);
  NewtonParams p{};
  p.act = act; p.n = B; p.J = J; p.ldj = ldj; p.u = u; p.mu = mu; p.f = f; p.thf = thf;
  p.N = N; p.Qf = 1; p.G = 1; p.ge[0] = -1; p.n_stop = N; p.stop_abs = 0; p.iter = 1; p.max_iter = 100; p.tol = 1e-12;
  p.iters = iters; p.status = status; p.last = last;
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  struct V { const char* name; K k; int threads; };
  const V vs[] = {
      {"gj1", newton_gj_kernel<8, 16, 13, 7>, 128},
      {"gj2", newton_gj2_kernel<8, 16, 13, 7, 0>, 128},
      {"gj2 -update", newton_gj2_kernel<8, 16, 13, 7, 1>, 128},
      {"gj2 -search", newton_gj2_kernel<8, 16, 13, 7, 2>, 128},
      {"gj2 -publish", newton_gj2_kernel<8, 16, 13, 7, 4>, 128},
      {"gj2 -update-search", newton_gj2_kernel<8, 16, 13, 7, 3>, 128},
      {"gj2 -all", newton_gj2_kernel<8, 16, 13, 7, 7>, 128},
      {"gj3", newton_gj3_kernel<8, 16, 13, 7>, 128},
      {"gjs (random J: hint misses)", newton_gjs_kernel<8, 16, 13, 7>, 128},
  };
  const V vd[] = {
      {"gj2 (dominant J)", newton_gj2_kernel<8, 16, 13, 7, 0>, 128},
      {"gjs (dominant J: hint hits)", newton_gjs_kernel<8, 16, 13, 7>, 128},
      {"bgj 13x13x8 (dominant J)", newton_bgj_kernel<13, 13, 8>, 256},
      {"bgj 13x14x4 (dominant J)", newton_bgj_kernel<13, 14, 4>, 128},
      {"bgj 13x13x13 (dominant J)", newton_bgj_kernel<13, 13, 13>, 416},
      {"bgj 13x13x4 J0=1 (dominant J)", newton_bgj_kernel<13, 13, 4, 1>, 128},
      {"bgj 13x13x4 J0=1 1CTA/SM", newton_bgj_kernel<13, 13, 4, 1>, 129},
      {"gj2 wide 16x16 (dominant J)", newton_gj2_kernel<16, 16, 7, 7, 0>, 256},
      {"gjs wide 16x16 (dominant J)", newton_gjs_kernel<16, 16, 7, 7>, 256},
      {"gjs wide 16x16 2CTA/SM", newton_gjs_kernel<16, 16, 7, 7, 2>, 256},
      {"gj1 wide 16x16 (dominant J)", newton_gj_kernel<16, 16, 7, 7>, 256},
  };
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int32_t* miss;
  cudaMallocManaged(&miss, sizeof(int32_t));
  p.spec_miss = miss;
  int32_t *mlist, *mcount;
  cudaMalloc(&mlist, sizeof(int32_t) * B);
  cudaMallocManaged(&mcount, sizeof(int32_t));
  p.miss_list = mlist;
  p.miss_count = mcount;
  cudaFuncSetAttribute(newton_bgj_kernel<13, 13, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       int(sizeof(BGJShared<13, 13, 8>)));
  cudaFuncSetAttribute(newton_bgj_kernel<13, 14, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       int(sizeof(BGJShared<13, 14, 4>)));
  cudaFuncSetAttribute(newton_bgj_kernel<13, 13, 13>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       int(sizeof(BGJShared<13, 13, 13>)));
  cudaFuncSetAttribute(newton_bgj_kernel<12, 12, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       int(sizeof(BGJShared<12, 12, 4>)));
  cudaFuncSetAttribute(newton_bgj_kernel<13, 13, 4, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
  auto run = [&](const V& v) {
    const size_t dyn = v.threads == 129 ? size_t(120 * 1024)
                       : v.k == newton_bgj_kernel<13, 13, 8>   ? sizeof(BGJShared<13, 13, 8>)
                       : v.k == newton_bgj_kernel<13, 14, 4> ? sizeof(BGJShared<13, 14, 4>)
                       : v.k == newton_bgj_kernel<13, 13, 13> ? sizeof(BGJShared<13, 13, 13>)
                       : v.k == newton_bgj_kernel<12, 12, 4> ? sizeof(BGJShared<12, 12, 4>)
                       : v.k == newton_bgj_kernel<13, 13, 4, 1> ? sizeof(BGJShared<13, 13, 4>)
                                                            : 0;
    *miss = 0;
    *mcount = 0;
    const int nthr = v.threads == 129 ? 128 : v.threads;
    v.k<<<B, nthr, dyn>>>(p);
    cudaDeviceSynchronize();
    const int m0 = *miss;
    cudaEventRecord(e0);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) v.k<<<B, nthr, dyn>>>(p);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    // SM-clocks per (sample, elimination step): how long one SM spends per step of one sample
    const double clk = double(ms) * 1e-3 * clk_khz * 1e3 * sms / (double(B) * N);
    printf("%-30s %8.3f ms  %7.1f SM-clk per sample-step  (x2 CTAs/SM: %6.0f clk per CTA step) misses %d/%d  %s\n",
           v.name, ms, clk, 2 * clk, m0, B, cudaGetErrorString(cudaGetLastError()));
  };
  if (N <= 55) {  // small systems: one-warp rank-1 kernel vs blocked kernels
    cudaFuncSetAttribute(newton_bgj_kernel<7, 7, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(sizeof(BGJShared<7, 7, 4>)));
    cudaFuncSetAttribute(newton_bgj_kernel<7, 7, 3, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(sizeof(BGJShared<7, 7, 3>)));
    add_diag<<<256, 256>>>(J, ldj, N, B, 10.0);
    const V small[] = {
        {"gjs 4x8x13x7", newton_gjs_kernel<4, 8, 13, 7>, 32},
        {"gj2 4x8x13x7", newton_gj2_kernel<4, 8, 13, 7, 0>, 32},
    };
    for (const V& v : small) run(v);
    for (int w = 0; w < 2; ++w) {
      const NewtonKernel k = w == 0 ? newton_bgj_kernel<7, 7, 4> : newton_bgj_kernel<7, 7, 3, 1>;
      const size_t sm = w == 0 ? sizeof(BGJShared<7, 7, 4>) : sizeof(BGJShared<7, 7, 3>);
      const int thr = w == 0 ? 128 : 96;
      k<<<B, thr, sm>>>(p);
      cudaDeviceSynchronize();
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) k<<<B, thr, sm>>>(p);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= 5;
      printf("%-30s %8.3f ms  %7.1f SM-clk per sample-step  %s\n", w == 0 ? "bgj 7x7x4" : "bgj 7x7x3 J0=1", ms,
             double(ms) * 1e-3 * clk_khz * 1e3 * sms / (double(B) * N), cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
  }
  for (const V& v : vs) run(v);
  add_diag<<<256, 256>>>(J, ldj, N, B, 10.0);
  for (const V& v : vd) run(v);
  return 0;
}
