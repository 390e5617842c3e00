// rbns_project.cu — offline Galerkin projection of the convective tensor on the FP64 tensor cores
// (SPEC.md:449-457 build_reduced_model "contracts c-terms to tensors C^i_jkl").
//
//     C[j][k][l] = Σ_p w_p Σ_{c,d} vu[p][d][j] · g[p][c][d][k] · vw[p][c][l]
//
// the integral c(ψ_j, ψ_k, ψ_l) = ∫ (ψ_j·∇)ψ_k·ψ_l evaluated on the quadrature points p of the high-fidelity
// mesh (the reference assembles the same integral element by element and projects it with sparse products,
// /root/reference/pkg/src/rbflow/assemble.py:86-101 convection_matrices, N1[i,j] = c(U, φ_j, φ_i)).  As a GEMM
// over κ = (p, c), K = 2P:
//
//     Y[(j,k)][l] = Σ_κ T[κ][(j,k)] · Wv[κ][l],   T[κ][(j,k)] = Σ_d vu[p][d][j] g[p][c][d][k],   Wv[κ][l] = w_p vw[p][c][l]
//
// T is never materialised, not even in shared memory: each CTA stages the raw tabulations of a 32-point chunk
// (64 κ) with cp.async (double-buffered: chunk c+1 lands while chunk c is multiplied) and every warp forms its
// DMMA A fragments w_p·T in registers (2 FMAs + 1 multiply per element) right before the DMMA.8x8x4 GEMM
// (8 warps, warp tile 16 rows × 64 columns, CTA tile 128 rows (8 j × 16 k) × 64 columns l).  The point range is
// split over gridDim.z slices (split-K) whose partial tiles are summed in a fixed order by a second kernel, so
// the result is deterministic.
#include <algorithm>
#include <string>

#include "rbns_launch.h"

namespace rbns {
namespace {

constexpr int kPJ = 8;             // j per CTA tile
constexpr int kPK = 16;            // k per CTA tile
constexpr int kPR = kPJ * kPK;     // 128 rows (j, k)
constexpr int kPL = 64;            // columns l per CTA tile
constexpr int kPP = 32;            // quadrature points per chunk
constexpr int kPC = 2 * kPP;       // κ = (p, c) per chunk
constexpr int kGS = 2 * kPK + 4;   // g row stride (doubles) per κ: ≡ 4 (mod 16) → conflict-free fragment loads
constexpr int kVS = kPL + 4;       // vw row stride per κ
constexpr int kPThreads = 256;

struct ProjStage {
  alignas(16) double g[kPC][kGS];      // g[κ][d·16 + k] = ∂_d ψ_{k0+k, c}(p)
  alignas(16) double vw[kPC][kVS];     // vw[κ][l]       = ψ_{l0+l, c}(p)
  alignas(16) double vu[kPP][2][kPJ];  // vu[p][d][j]    = ψ_{j0+j, d}(p)
  double w[kPP];
};
struct ProjShared {
  ProjStage st[2];  // double-buffered raw tabulations (cp.async)
};

__device__ __forceinline__ void cp_async8(void* dst, const void* src, bool valid) {
  const int n = valid ? 8 : 0;  // zero-fill past the arrays
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(dst)), "l"(src), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// raw tabulations of points [p0, p0 + kPP) for this CTA's j, k, l ranges into stage S
__device__ __forceinline__ void proj_stage(ProjStage& S, const double* __restrict__ vu, const double* __restrict__ g,
                                           const double* __restrict__ vw, const double* __restrict__ w, int N,
                                           int64_t p0, int j0, int k0, int l0, int64_t p_end) {
  const int tid = threadIdx.x;
  for (int e = tid; e < kPP * 2 * kPJ; e += kPThreads) {
    const int p = e / (2 * kPJ), d = (e / kPJ) & 1, j = e % kPJ;
    const int64_t pp = p0 + p;
    const bool ok = pp < p_end && j0 + j < N;
    cp_async8(&S.vu[p][d][j], ok ? vu + (pp * 2 + d) * N + j0 + j : vu, ok);
  }
  for (int e = tid; e < kPC * 2 * kPK; e += kPThreads) {
    const int kap = e / (2 * kPK), d = (e / kPK) & 1, k = e % kPK;
    const int64_t pp = p0 + (kap >> 1);
    const bool ok = pp < p_end && k0 + k < N;
    cp_async8(&S.g[kap][d * kPK + k], ok ? g + ((pp * 2 + (kap & 1)) * 2 + d) * N + k0 + k : g, ok);
  }
  for (int e = tid; e < kPC * kPL; e += kPThreads) {
    const int kap = e / kPL, l = e % kPL;
    const int64_t pp = p0 + (kap >> 1);
    const bool ok = pp < p_end && l0 + l < N;
    cp_async8(&S.vw[kap][l], ok ? vw + (pp * 2 + (kap & 1)) * N + l0 + l : vw, ok);
  }
  if (tid < kPP) {
    const int64_t pp = p0 + tid;
    cp_async8(&S.w[tid], pp < p_end ? w + pp : w, pp < p_end);
  }
}

// Grid (j-k tiles, l tiles, split-K slices); 8 warps, warp tile 16 rows (2 j × 8 k... rows 16·warp ..) × 64 columns.
// Per k-step (4 κ) a warp forms its two A fragments in registers straight from the raw tabulations,
//     A[g][t] = T[κ+t][row] · w_p = w_p Σ_d vu[p][d][j] g[p][c][d][k]     (κ + t = 2p + c)
// and multiplies them into 8 B fragments B[t][g] = vw[κ+t][col]: 16 DMMA.8x8x4 per 2 fragment formations.
__global__ void __launch_bounds__(kPThreads, 2)
    project_convection_kernel(const double* __restrict__ vu, const double* __restrict__ g,
                              const double* __restrict__ vw, const double* __restrict__ w, int64_t P, int N,
                              int64_t pts_per_split, double* __restrict__ out, int64_t split_stride) {
  extern __shared__ __align__(16) unsigned char proj_smem[];
  ProjShared& sh = *reinterpret_cast<ProjShared*>(proj_smem);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, gq = lane >> 2, tq = lane & 3;
  const int nkb = (N + kPK - 1) / kPK;
  const int j0 = (blockIdx.x / nkb) * kPJ, k0 = (blockIdx.x % nkb) * kPK, l0 = blockIdx.y * kPL;
  const int64_t pb = int64_t(blockIdx.z) * pts_per_split;
  const int64_t pe = P < pb + pts_per_split ? P : pb + pts_per_split;
  // warp rows 16·warp + 8a + g, a ∈ {0, 1}: j = warp (row / 16), k = 8a + g
  const int jl = warp;
  double acc[2][8][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 8; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  int buf = 0;
  if (pb < pe) proj_stage(sh.st[0], vu, g, vw, w, N, pb, j0, k0, l0, pe);
  cp_async_commit();
#pragma unroll 1
  for (int64_t p0 = pb; p0 < pe; p0 += kPP) {
    cp_async_wait_all();
    __syncthreads();  // stage `buf` landed; every warp is done with the other stage
    if (p0 + kPP < pe) proj_stage(sh.st[buf ^ 1], vu, g, vw, w, N, p0 + kPP, j0, k0, l0, pe);
    cp_async_commit();
    const ProjStage& S = sh.st[buf];
#pragma unroll 4
    for (int ks = 0; ks < kPC; ks += 4) {
      const int kap = ks + tq, p = kap >> 1;
      const double wp = S.w[p];
      const double v0 = S.vu[p][0][jl] * wp, v1 = S.vu[p][1][jl] * wp;
      double af[2], bf[8];
#pragma unroll
      for (int a = 0; a < 2; ++a) af[a] = fma(v0, S.g[kap][8 * a + gq], v1 * S.g[kap][kPK + 8 * a + gq]);
#pragma unroll
      for (int b = 0; b < 8; ++b) bf[b] = S.vw[kap][8 * b + gq];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b) dmma_8x8x4(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
    buf ^= 1;
  }
  // D[g][2t+s] of fragment (a, b): j = j0 + warp, k = k0 + 8a + g, l = l0 + 8b + 2t + s
  double* o = out + int64_t(blockIdx.z) * split_stride;
  const int j = j0 + jl;
  if (j < N) {
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      const int k = k0 + 8 * a + gq;
      if (k >= N) continue;
#pragma unroll
      for (int b = 0; b < 8; ++b)
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          const int l = l0 + 8 * b + 2 * tq + s;
          if (l < N) o[(int64_t(j) * N + k) * N + l] = acc[a][b][s];
        }
    }
  }
}

// fixed-order sum of the split-K partial tensors
__global__ void project_reduce(const double* __restrict__ part, int splits, int64_t n, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int z = 0; z < splits; ++z) s += part[int64_t(z) * n + i];
    out[i] = s;
  }
}

}  // namespace
}  // namespace rbns

using namespace rbns;

extern "C" int rbns_project_convection(const double* val_u, const double* grad, const double* val_w, const double* w,
                                       int64_t points, int32_t n, double* C, int32_t splits, void* stream) {
  if (!val_u || !grad || !val_w || !w || !C) return set_last_error(RBNS_ERR_INVALID_ARGUMENT, "NULL buffer");
  if (points < 1 || n < 1 || n > 4096)
    return set_last_error(RBNS_ERR_INVALID_ARGUMENT, "need points >= 1 and 1 <= n <= 4096");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return set_last_error(RBNS_ERR_CUDA, "no CUDA device");
  const int nj = (n + kPJ - 1) / kPJ, nk = (n + kPK - 1) / kPK, nl = (n + kPL - 1) / kPL;
  const int64_t tiles = int64_t(nj) * nk * nl;
  // split-K: enough slices for ~4 waves of two CTAs per SM, each at least 16 chunks of points
  int z = splits > 0 ? splits : int(std::max<int64_t>(1, std::min<int64_t>((8 * sms + tiles - 1) / tiles,
                                                                          points / (16 * kPP))));
  z = std::max(1, std::min(z, 65535));
  const int64_t per = ((points + z - 1) / z + kPP - 1) / kPP * kPP;
  z = int((points + per - 1) / per);
  const int64_t nn = int64_t(n) * n * n;
  double* part = C;
  if (z > 1) {
    cudaError_t e = cudaMallocAsync(&part, size_t(z) * nn * sizeof(double), st);
    if (e != cudaSuccess) return set_last_error(RBNS_ERR_OUT_OF_MEMORY, "split-K workspace");
  }
  cudaError_t ea = cudaFuncSetAttribute(project_convection_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        int(sizeof(ProjShared)));
  if (ea != cudaSuccess) {
    if (z > 1) cudaFreeAsync(part, st);
    return set_last_error(RBNS_ERR_CUDA, std::string("projection kernel attribute: ") + cudaGetErrorString(ea));
  }
  project_convection_kernel<<<dim3(unsigned(nj * nk), unsigned(nl), unsigned(z)), kPThreads, sizeof(ProjShared), st>>>(
      val_u, grad, val_w, w, points, n, per, part, nn);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess && z > 1) {
    project_reduce<<<4 * sms, 256, 0, st>>>(part, z, nn, C);
    e = cudaGetLastError();
  }
  if (z > 1) cudaFreeAsync(part, st);
  if (e != cudaSuccess) return set_last_error(RBNS_ERR_CUDA, std::string("projection launch: ") + cudaGetErrorString(e));
  return RBNS_OK;
}
