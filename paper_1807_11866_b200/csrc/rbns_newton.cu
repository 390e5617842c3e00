// rbns_newton.cu — instantiation + dispatch of the Newton-update kernels; kept in its own translation unit so
// the instantiations compile in parallel with the rest of the library.
//   tiled Gauss–Jordan (rbns_tgj.cuh)      default for 32 < N ≤ 103 (shapes: rbns_tgj_shapes_*.cu)
//   speculative rank-1 (rbns_newton_spec)   N ≤ 32, hinted pivot order, misses → exact kernel
//   exact rank-1 (rbns_newton2.cuh)         full partial-pivot search: every miss of the speculative kernels
//   hybrid tiled Gauss–Jordan (rbns_tgh.cuh) 103 < N ≤ 200: one CTA per sample, registers + shared memory
//   2-CTA cluster (rbns_newton_cluster)     200 < N ≤ 207, and the exact path of the hybrid kernel
// RBNS_NEWTON=gjs forces the speculative rank-1 kernels, RBNS_NEWTON=gj2 the exact one (parity-tested).
#include "rbns_launch.h"
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <utility>

#include "rbns_newton.cuh"
#include "rbns_newton2.cuh"
#include "rbns_newton_spec.cuh"
#include "rbns_newton_cluster.cuh"
#include "rbns_tgj.cuh"
#include "rbns_tgh.cuh"
#include "rbns_tiled_plan.h"

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
const Shape* plan(int N) {
  static const bool full_search = [] {  // RBNS_NEWTON=gj2: the exact kernel for every sample
    const char* v = std::getenv("RBNS_NEWTON");
    return v && std::strcmp(v, "gj2") == 0;
  }();
  const Shape* table = full_search ? kShapes2 : kShapes;
  for (int i = 0; i < int(sizeof(kShapes) / sizeof(kShapes[0])); ++i) {
    const Shape& s = table[i];
    if (N >= 1 && N <= s.tgr * s.rs && N + 1 <= s.tgc * s.cs) return &s;
  }
  return nullptr;
}

const TShape* tplan(int N) {
  static const bool off = [] {  // any RBNS_NEWTON value other than "tgj" selects the earlier kernels
    const char* v = std::getenv("RBNS_NEWTON");
    return v && *v && std::strcmp(v, "tgj") != 0;
  }();
  if (off || N <= 8) return nullptr;
  const int rt = (N + 7) / 8, ct = (N + 8) / 8;
  for (int i = 0; i < kTShapesMain_n; ++i)
    if (kTShapesMain[i].rt == rt && kTShapesMain[i].ct == ct) return &kTShapesMain[i];
  for (int i = 0; i < kTShapesA_n; ++i)
    if (kTShapesA[i].rt == rt && kTShapesA[i].ct == ct) return &kTShapesA[i];
  for (int i = 0; i < kTShapesB_n; ++i)
    if (kTShapesB[i].rt == rt && kTShapesB[i].ct == ct) return &kTShapesB[i];
  return nullptr;
}

const HShape* hplan(int N) {
  static const int mode = [] {  // 0: default (config-3 shape), 1: off, 2: every instantiated shape
    const char* v = std::getenv("RBNS_NEWTON");
    if (!v || !*v || std::strcmp(v, "tgj") == 0) return 0;
    return std::strcmp(v, "tgh") == 0 ? 2 : 1;
  }();
  if (mode == 1 || N <= 8) return nullptr;
  const int rt = (N + 7) / 8, ct = (N + 8) / 8;
  for (const auto& [tab, cnt] : {std::pair{kHShapesMain, kHShapesMain_n}, std::pair{kHShapesA, kHShapesA_n},
                                  std::pair{kHShapesB, kHShapesB_n}, std::pair{kHShapesC, kHShapesC_n}})
    for (int i = 0; i < cnt; ++i)
      if (tab[i].rt == rt && tab[i].ct == ct && (mode == 2 || !tab[i].test_only)) return &tab[i];
  return nullptr;
}
}  // namespace

// N > 127: the 2-CTA cluster kernel (rbns_newton_cluster.cuh), 16×(2×16) threads, N ≤ 207
constexpr int kClusterMaxN = 207;

bool newton_supported(int N) { return plan(N) != nullptr || (N >= 1 && N <= kClusterMaxN); }

int newton_layout(int N) { return tplan(N) != nullptr || hplan(N) != nullptr ? 1 : 0; }

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
  if (const HShape* h = hplan(N)) {
    if (h->smem > size_t(max_smem)) return cudaErrorInvalidValue;
    e = cudaFuncSetAttribute(h->kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(h->smem));
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(h->kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
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
  if (!p.prefer_rank1 && p.jl && !hplan(p.N)) {
    const TShape* t = tplan(p.N);
    const Shape* s = plan(p.N);
    if (t && s && s->exact) {
      cudaError_t e = cudaMemsetAsync(p.miss_count, 0, sizeof(int32_t), st);
      if (e != cudaSuccess) return e;
      const size_t smem = t->base + size_t(p.ldj) * sizeof(double);
      t->kern<<<std::min(p.n, t->minb * p.num_sms), t->nw * 32, smem, st>>>(p);
      e = cudaGetLastError();
      if (e != cudaSuccess) return e;
      *launches = 2;
      return launch_exact(s, p, st);
    }
  }
  if (!p.prefer_rank1 && p.jl) {
    if (const HShape* h = hplan(p.N)) {
      cudaError_t e = cudaMemsetAsync(p.miss_count, 0, sizeof(int32_t), st);
      if (e != cudaSuccess) return e;
      h->kern<<<std::min(p.n, h->minb * p.num_sms), h->nw * 32, h->smem, st>>>(p);
      e = cudaGetLastError();
      if (e != cudaSuccess) return e;
      *launches = 2;
      // the samples it handed back: the exact kernel over the device-side list
      if (const Shape* s = plan(p.N); s && s->exact) return launch_exact(s, p, st);
      NewtonParams q = p;
      q.sub = p.miss_list;
      q.n_sub = p.miss_count;
      newton_gjc_kernel<16, 16, 13, 7><<<2 * std::min(p.n, std::max(1, p.num_sms / 2)), 256, 0, st>>>(q);
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

int rbns::newton_debug_checks(int* line, unsigned long long* count) {
#ifdef RBNS_CHECKED
  if (cudaMemcpyFromSymbol(line, rbns::g_chk_line, sizeof(int)) != cudaSuccess ||
      cudaMemcpyFromSymbol(count, rbns::g_chk_count, sizeof(unsigned long long)) != cudaSuccess)
    return 2;
#else
  *line = 0;
  *count = 0;
#endif
  return 0;
}

#ifdef RBNS_TGH_DUMP
extern "C" int rbns_debug_tgh(double* out) {
  return cudaMemcpyFromSymbol(out, rbns::g_tgh_dump, sizeof(double) * 4 * 256) == cudaSuccess ? 0 : 2;
}
#endif
#ifdef RBNS_TRACE
extern "C" int rbns_debug_trace(unsigned long long* out, int n) {
  return cudaMemcpyFromSymbol(out, rbns::g_trace, sizeof(unsigned long long) * (n < 256 ? n : 256)) == cudaSuccess ? 0 : 2;
}
#endif
