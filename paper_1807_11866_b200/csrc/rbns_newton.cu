// rbns_newton.cu — instantiation + dispatch of the register-resident Gauss–Jordan Newton-update kernel
// (rbns_newton.cuh); kept in its own translation unit so the instantiations compile in parallel with the rest
// of the library.  A few fixed shapes cover every N ≤ 127 (RS·TGR ≥ N rows, CS·TGC ≥ N+1 columns).
#include "rbns_launch.h"
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "rbns_bgj.cuh"
#include "rbns_newton.cuh"
#include "rbns_newton2.cuh"
#include "rbns_newton3.cuh"
#include "rbns_newton_spec.cuh"
#include "rbns_newton_cluster.cuh"
#include "rbns_tgj.cuh"

namespace rbns {

namespace {
using NewtonKernel = void (*)(const NewtonParams);

struct Shape {
  int tgr, tgc, rs, cs;
  NewtonKernel kern;
  NewtonKernel exact = nullptr;  // speculative kernels: the full-search kernel for the samples they hand back
};

#define RBNS_SPEC(R_, C_, RS_, CS_) {R_, C_, RS_, CS_, newton_gjs_kernel<R_, C_, RS_, CS_>, newton_gj2_kernel<R_, C_, RS_, CS_>}
const Shape kShapes[] = {
    RBNS_SPEC(4, 8, 4, 3),     // N ≤ 16   (1 warp)
    RBNS_SPEC(4, 8, 8, 5),     // N ≤ 32   (1 warp)
    RBNS_SPEC(4, 8, 13, 7),    // N ≤ 52   (1 warp)
    RBNS_SPEC(8, 16, 10, 6),   // N ≤ 80   (4 warps)
    RBNS_SPEC(8, 16, 13, 7),   // N ≤ 104  (4 warps)
    RBNS_SPEC(16, 16, 8, 8),   // N ≤ 127  (8 warps)
};
#undef RBNS_SPEC
// RBNS_NEWTON=gj2: full pivot search every step (rbns_newton2.cuh) — also the speculative kernel's fallback
const Shape kShapes2[] = {
    {4, 8, 4, 3, newton_gj2_kernel<4, 8, 4, 3>},
    {4, 8, 8, 5, newton_gj2_kernel<4, 8, 8, 5>},
    {4, 8, 13, 7, newton_gj2_kernel<4, 8, 13, 7>},
    {8, 16, 10, 6, newton_gj2_kernel<8, 16, 10, 6>},
    {8, 16, 13, 7, newton_gj2_kernel<8, 16, 13, 7>},
    {16, 16, 8, 8, newton_gj2_kernel<16, 16, 8, 8>},
};
// RBNS_NEWTON=gj1: the earlier owner-serial pivot search (rbns_newton.cuh), kept for comparison
const Shape kShapes1[] = {
    {4, 8, 4, 3, newton_gj_kernel<4, 8, 4, 3>},
    {4, 8, 8, 5, newton_gj_kernel<4, 8, 8, 5>},
    {4, 8, 13, 7, newton_gj_kernel<4, 8, 13, 7>},
    {8, 16, 10, 6, newton_gj_kernel<8, 16, 10, 6>},
    {8, 16, 13, 7, newton_gj_kernel<8, 16, 13, 7>},
    {16, 16, 8, 8, newton_gj_kernel<16, 16, 8, 8>},
};

// RBNS_NEWTON=gj3: one barrier per step, redundant per-warp search, pivot row by warp shuffles (rbns_newton3.cuh)
const Shape kShapes3[] = {
    {4, 8, 4, 3, newton_gj3_kernel<4, 8, 4, 3>},
    {4, 8, 8, 5, newton_gj3_kernel<4, 8, 8, 5>},
    {4, 8, 13, 7, newton_gj3_kernel<4, 8, 13, 7>},
    {8, 16, 10, 6, newton_gj3_kernel<8, 16, 10, 6>},
    {8, 16, 13, 7, newton_gj3_kernel<8, 16, 13, 7>},
    {16, 16, 8, 8, newton_gj3_kernel<16, 16, 8, 8>},
};

// RBNS_GJ_WIDE=1: 8 warps (16×16 grid, 49 register doubles per thread, two CTAs per SM) for 52 < N ≤ 112
const Shape kWide = {16, 16, 7, 7, newton_gj_kernel<16, 16, 7, 7>};

const Shape* plan(int N) {
  static const bool wide = [] {
    const char* v = std::getenv("RBNS_GJ_WIDE");
    return v && v[0] == '1';
  }();
  if (wide && N > 52 && N <= 111) return &kWide;
  static const int variant = [] {
    const char* v = std::getenv("RBNS_NEWTON");
    if (v && std::strcmp(v, "gj1") == 0) return 1;
    if (v && std::strcmp(v, "gj3") == 0) return 3;
    if (v && std::strcmp(v, "gj2") == 0) return 2;
    return 0;
  }();
  const Shape* table = variant == 1 ? kShapes1 : variant == 2 ? kShapes2 : variant == 3 ? kShapes3 : kShapes;
  for (int i = 0; i < int(sizeof(kShapes) / sizeof(kShapes[0])); ++i) {
    const Shape& s = table[i];
    if (N >= 1 && N <= s.tgr * s.rs && N + 1 <= s.tgc * s.cs) return &s;
  }
  return nullptr;
}

// blocked (DMMA) variant: RT×CT tiles of 8×8, NW warps
struct BShape {
  int rt, ct, nw;
  NewtonKernel kern;
  size_t smem;
};

#define RBNS_BS(R_, C_, W_) {R_, C_, W_, newton_bgj_kernel<R_, C_, W_>, sizeof(BGJShared<R_, C_, W_>)}
const BShape kBShapes[] = {
    RBNS_BS(2, 2, 2),     // N ≤ 15
    RBNS_BS(7, 7, 4),     // N ≤ 55
    RBNS_BS(12, 12, 4),   // N ≤ 95
    {13, 13, 4, newton_bgj_kernel<13, 13, 4, 1>, sizeof(BGJShared<13, 13, 4>)},  // N ≤ 103 (tile 0 never in
                                                                                  // registers: 4 warps, 2 CTAs/SM)
    RBNS_BS(16, 16, 8),   // N ≤ 127
};
#undef RBNS_BS

const BShape* bplan(int N) {
  for (const BShape& s : kBShapes)
    if (N >= 1 && N <= 8 * s.rt && N + 1 <= 8 * s.ct) return &s;
  return nullptr;
}

// Kernel choice: the blocked DMMA kernel (rbns_bgj.cuh) is the default where it measured faster (88 < N ≤ 103:
// cfg-2 Newton update 74 ms against 89 ms for the speculative rank-1 kernel); elsewhere the rank-1 register
// kernels (rbns_newton*.cuh) run.  RBNS_NEWTON=bgj forces the blocked kernel for every N it covers, any other
// RBNS_NEWTON value forces the rank-1 kernels (all are parity-tested).
bool use_blocked(int N) {
  static const int mode = [] {
    const char* v = std::getenv("RBNS_NEWTON");
    if (!v || !*v) return 0;
    return std::strcmp(v, "bgj") == 0 ? 1 : 2;
  }();
  return mode == 1 || (mode == 0 && N > 88 && N <= 103);
}

// tiled Gauss–Jordan kernel (rbns_tgj.cuh): RT = ⌈N/8⌉ row tiles, CT = ⌈(N+1)/8⌉ column tiles, NW warps
struct TShape {
  int rt, ct, nw;
  NewtonKernel kern;
  size_t base;  // shared memory before the J staging buffer
};
#define RBNS_TS(R_, C_, W_) {R_, C_, W_, newton_tgj_kernel<R_, C_, W_>, tgj_stage_offset<R_, W_>()}
const TShape kTShapes[] = {
    RBNS_TS(13, 13, 4),  // 96 < N ≤ 103 (config 2 / 4: N = 100)
};
#undef RBNS_TS

const TShape* tplan(int N) {
  static const bool off = [] {  // any RBNS_NEWTON value other than "tgj" selects the earlier kernels
    const char* v = std::getenv("RBNS_NEWTON");
    return v && *v && std::strcmp(v, "tgj") != 0;
  }();
  if (off || N <= 8) return nullptr;
  const int rt = (N + 7) / 8, ct = (N + 8) / 8;
  for (const TShape& s : kTShapes)
    if (s.rt == rt && s.ct == ct) return &s;
  return nullptr;
}
}  // namespace

// N > 127: the 2-CTA cluster kernel (rbns_newton_cluster.cuh), 16×(2×16) threads, N ≤ 207
constexpr int kClusterMaxN = 207;

bool newton_supported(int N) { return plan(N) != nullptr || bplan(N) != nullptr || (N >= 1 && N <= kClusterMaxN); }

int newton_layout(int N) { return tplan(N) != nullptr ? 1 : 0; }

cudaError_t newton_prepare(int N) {
  int dev = 0, max_smem = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  e = cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e != cudaSuccess) return e;
  // per-device function attributes (cudaFuncSetAttribute applies to the current device only)
  if (const TShape* t = tplan(N)) {
    e = cudaFuncSetAttribute(t->kern, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(t->kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
  }
  if (const BShape* b = bplan(N)) {
    e = cudaFuncSetAttribute(b->kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(b->smem));
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// the exact full-search kernel over the samples a speculative pass listed (device-side count)
static cudaError_t launch_exact(const Shape* s, const NewtonParams& p, cudaStream_t st) {
  NewtonParams q = p;
  q.sub = p.miss_list;
  q.n_sub = p.miss_count;
  s->exact<<<std::min(p.n, 2 * p.num_sms), s->tgr * s->tgc, 0, st>>>(q);
  return cudaGetLastError();
}

cudaError_t launch_newton_update(const NewtonParams& p, cudaStream_t st, int* launches) {
  *launches = 1;
  if (!p.prefer_rank1 && p.jl) {
    const TShape* t = tplan(p.N);
    const Shape* s = plan(p.N);
    if (t && s && s->exact) {
      cudaError_t e = cudaMemsetAsync(p.miss_count, 0, sizeof(int32_t), st);
      if (e != cudaSuccess) return e;
      const size_t smem = t->base + size_t(p.ldj) * sizeof(double);
      t->kern<<<std::min(p.n, 2 * p.num_sms), t->nw * 32, smem, st>>>(p);
      e = cudaGetLastError();
      if (e != cudaSuccess) return e;
      *launches = 2;
      return launch_exact(s, p, st);
    }
  }
  if (!p.prefer_rank1 && !p.jl && use_blocked(p.N)) {
    if (const BShape* b = bplan(p.N)) {
      b->kern<<<p.n, b->nw * 32, b->smem, st>>>(p);
      return cudaGetLastError();
    }
  }
  const Shape* s = plan(p.N);
  if (!s && p.N <= kClusterMaxN) {
    newton_gjc_kernel<16, 16, 13, 7><<<2 * p.n, 256, 0, st>>>(p);
    return cudaGetLastError();
  }
  if (!s) return cudaErrorInvalidValue;
  if (s->exact) {
    // speculative pass, then the exact kernel over the samples it handed back (device-side count)
    cudaError_t e = cudaMemsetAsync(p.miss_count, 0, sizeof(int32_t), st);
    if (e != cudaSuccess) return e;
    s->kern<<<p.n, s->tgr * s->tgc, 0, st>>>(p);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    *launches = 2;
    return launch_exact(s, p, st);
  }
  s->kern<<<p.n, s->tgr * s->tgc, 0, st>>>(p);
  return cudaGetLastError();
}

}  // namespace rbns

#ifdef RBNS_TRACE
extern "C" int rbns_debug_trace(unsigned long long* out, int n) {
  return cudaMemcpyFromSymbol(out, rbns::g_trace, sizeof(unsigned long long) * (n < 256 ? n : 256)) == cudaSuccess ? 0 : 2;
}
#endif
