// rbns_newton.cu — instantiation + dispatch of the register-resident Gauss–Jordan Newton-update kernel
// (rbns_newton.cuh); kept in its own translation unit so the instantiations compile in parallel with the rest
// of the library.  A few fixed shapes cover every N ≤ 127 (RS·TGR ≥ N rows, CS·TGC ≥ N+1 columns).
#include "rbns_launch.h"
#include "rbns_newton.cuh"

namespace rbns {

namespace {
using NewtonKernel = void (*)(const NewtonParams);

struct Shape {
  int tgr, tgc, rs, cs;
  NewtonKernel kern;
};

const Shape kShapes[] = {
    {4, 8, 4, 3, newton_gj_kernel<4, 8, 4, 3>},       // N ≤ 16   (1 warp)
    {4, 8, 8, 5, newton_gj_kernel<4, 8, 8, 5>},       // N ≤ 32   (1 warp)
    {4, 8, 13, 7, newton_gj_kernel<4, 8, 13, 7>},     // N ≤ 52   (1 warp)
    {8, 16, 10, 6, newton_gj_kernel<8, 16, 10, 6>},   // N ≤ 80   (4 warps)
    {8, 16, 13, 7, newton_gj_kernel<8, 16, 13, 7>},   // N ≤ 104  (4 warps)
    {16, 16, 8, 8, newton_gj_kernel<16, 16, 8, 8>},   // N ≤ 127  (8 warps)
};

const Shape* plan(int N) {
  for (const Shape& s : kShapes)
    if (N >= 1 && N <= s.tgr * s.rs && N + 1 <= s.tgc * s.cs) return &s;
  return nullptr;
}
}  // namespace

bool newton_supported(int N) { return plan(N) != nullptr; }

cudaError_t launch_newton_update(const NewtonParams& p, cudaStream_t st) {
  const Shape* s = plan(p.N);
  if (!s) return cudaErrorInvalidValue;
  s->kern<<<p.n, s->tgr * s->tgc, 0, st>>>(p);
  return cudaGetLastError();
}

}  // namespace rbns
