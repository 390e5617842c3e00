// rbns_common.cuh — shared device helpers: θ evaluation, PTX wrappers (mbarrier, TMA, DMMA).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "rbns.h"

namespace rbns {

#ifdef RBNS_TRACE
__device__ unsigned long long g_trace[256];
#define RBNS_TR(slot)                                                               \
  do {                                                                              \
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0) g_trace[(slot) & 255] = clock64(); \
  } while (0)
#else
#define RBNS_TR(slot) \
  do {                \
  } while (0)
#endif

constexpr int kStatusActive = 127;  // internal: sample still iterating

// Checked build (-DRBNS_CHECKED, build/librbns_checked.so; compute-sanitizer is not available on this pool):
// bounds and protocol checks on the hot kernels' global and shared indexing.  A failed check records its
// source line (first one wins) and counts; rbns_debug_checks() reads the counters of every translation unit.
#ifdef RBNS_CHECKED
static __device__ int g_chk_line;
static __device__ unsigned long long g_chk_count;
#define RBNS_CHECK(cond)                              \
  do {                                                \
    if (!(cond)) {                                    \
      atomicCAS(&::rbns::g_chk_line, 0, __LINE__);    \
      atomicAdd(&::rbns::g_chk_count, 1ull);          \
    }                                                 \
  } while (0)
#else
#define RBNS_CHECK(cond) \
  do {                   \
  } while (0)
#endif

__device__ __forceinline__ double ipow(double x, int n) {
  double r = 1.0;
  for (int i = 0; i < n; ++i) r = r * x;
  return r;
}

// θ(μ) of one descriptor (the C-ABI rbns_theta_term, copied to device memory at model create) — same rule,
// term by term, as paper_1807_11866_b200/affine.py:evaluate_weights (SPEC.md:360-368 evaluate_weights;
// SPEC.md:335-338 CoefficientDescriptor "scale·φᵏ·u∞ᵐ").  μ = (mu0, mu1) = (α or φ, Re or u∞).
__device__ __forceinline__ double eval_theta(const rbns_theta_term& t, double mu0, double mu1) {
  double base;
  switch (t.kind) {
    case RBNS_THETA_CONST: base = 1.0; break;
    case RBNS_THETA_COS_K: base = cos(double(t.k) * mu0); break;
    case RBNS_THETA_SIN_K: base = sin(double(t.k) * mu0); break;
    case RBNS_THETA_COS_SIN_POW: base = ipow(cos(mu0), t.k) * ipow(sin(mu0), t.m); break;
    default: base = ipow(mu0, t.k) * ipow(mu1, t.m); break;
  }
  return t.scale * base;
}

// μ₁^e for the residual's h-group factors (e = −1: ν = 1/Re)
__device__ __forceinline__ double mu1_pow(double mu1, int e) { return e >= 0 ? ipow(mu1, e) : 1.0 / ipow(mu1, -e); }

// ---------------------------------------------------------------------------------------------------------
// PTX wrappers
// ---------------------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// mbar_wait with a sleep between failed probes (a producer lane that should leave issue slots to its SM
// sub-partition's consumer warps)
#ifndef RBNS_BACKOFF_NS
#define RBNS_BACKOFF_NS 64
#endif
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, uint32_t parity, uint32_t ns = RBNS_BACKOFF_NS) {
  uint32_t done = 0;
  while (true) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return;
    __nanosleep(ns);
  }
}

__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}

// 2-D TMA tile load global -> shared, completion signalled on an mbarrier (transaction bytes).
__device__ __forceinline__ void tma_load_2d(void* smem_dst, const void* tmap, uint64_t* bar, int c0, int c1,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;\n" ::"r"(smem_u32(smem_dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// Bulk prefetch of a global range into L2 (no destination, no completion); 16-byte aligned, size % 16 == 0.
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  for (uint32_t off = 0; off < bytes; off += 16384u) {
    const uint32_t n = bytes - off < 16384u ? bytes - off : 16384u;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(static_cast<const char*>(src) + off), "r"(n)
                 : "memory");
  }
}

__device__ __forceinline__ void prefetch_tmap(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(tmap) : "memory");
}

// Reciprocal for pivots: hardware approximation (MUFU.RCP64H) refined by two Newton–Raphson steps
// (~23 → ~46 → full 53 bits, within 1 ulp of 1/x).  Callers guarantee x is finite, nonzero and normal;
// it replaces the IEEE division sequence on the serial critical path of the Gauss–Jordan column steps.
__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// 1-D bulk copy global -> shared (TMA engine), completion signalled on an mbarrier (transaction bytes).
// 16-byte aligned addresses, size % 16 == 0.
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::
          "r"(smem_u32(smem_dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}

// orders this thread's earlier generic-proxy shared-memory accesses before later async-proxy (TMA) ones
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

// ---------------------------------------------------------------------------------------------------------
// Jacobian block layouts (the contraction writes J in the layout its Newton kernel reads; NewtonParams::jl)
//   0  row-major: J[l][m] at l·N + m
//   1  tile layout of the tiled Gauss–Jordan kernel (rbns_tgj.cuh): 8×8 tiles (row tile i = l/8, column
//      tile j = m/8) stored column-tile-major, row tiles in order inside a column tile, and inside a tile
//      column-major (g = m%8 outer, ts = l%8 inner) over the tile's real rows rr and columns cr only.  A full
//      tile is 64 contiguous doubles in which lane (g, t) of the DMMA fragment layout finds its pair
//      (rows 8i+2t, 8i+2t+1 of column 8j+g) at offset 2·lane: one 16-byte load per lane, no padding bytes.
//      The h rows (residual helpers) follow at N² + g·N + l in both layouts.
// ---------------------------------------------------------------------------------------------------------
__host__ __device__ inline int64_t jidx_tile(int l, int m, int N) {
  const int i = l >> 3, ts = l & 7, j = m >> 3, g = m & 7;
  const int rr = N - 8 * i < 8 ? N - 8 * i : 8;
  const int cr = N - 8 * j < 8 ? N - 8 * j : 8;
  return int64_t(8 * j) * N + int64_t(8 * i) * cr + g * rr + ts;
}

__host__ __device__ inline int64_t jidx(int l, int m, int N, int jl) {
  return jl ? jidx_tile(l, m, N) : int64_t(l) * N + m;
}

// inverse of jidx: position r < N² -> (l, m)
__host__ __device__ inline void jpos(int64_t r, int N, int jl, int& l, int& m) {
  if (!jl) {
    l = int(r / N);
    m = int(r - int64_t(l) * N);
    return;
  }
  const int j = int(r / (8 * int64_t(N)));
  const int rem = int(r - int64_t(8 * j) * N);
  const int cr = N - 8 * j < 8 ? N - 8 * j : 8;
  const int i = rem / (8 * cr);
  const int rem2 = rem - 8 * i * cr;
  const int rr = N - 8 * i < 8 ? N - 8 * i : 8;
  const int g = rem2 / rr;
  l = 8 * i + (rem2 - g * rr);
  m = 8 * j + g;
}

// Same contract with one cubic refinement, r·(1 + e + e²), e = 1 − x r: three dependent DFMAs instead of four
// (the error term e³ is far below double rounding).
__device__ __forceinline__ double rcp_cubic(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  return fma(r, fma(e, e, e), r);
}

// FP64 tensor-core MMA (lowers to DMMA.8x8x4 on sm_100a): D(8x8) += A(8x4) * B(4x8).
// Thread (g = lane>>2, t = lane&3) supplies A[g][t], B[t][g]; holds D[g][2t], D[g][2t+1].
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

}  // namespace rbns
