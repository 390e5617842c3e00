// rbns_tiled_plan.h — the instantiated shapes of the tiled Gauss–Jordan Newton kernel (rbns_tgj.cuh).  The
// instantiations live in their own translation units (rbns_tgj_shapes_a.cu / _b.cu, compiled in parallel);
// rbns_newton.cu plans and launches through these tables.
#pragma once

#include <cstddef>

#include "rbns_newton.cuh"

namespace rbns {

struct TShape {
  int rt, ct, nw;                     // row tiles ⌈N/8⌉, column tiles ⌈(N+1)/8⌉, warps
  void (*kern)(const NewtonParams);   // newton_tgj_kernel<rt, ct, nw>
  size_t base;                        // shared memory before the J staging buffer
  int minb;                           // resident CTAs per SM (persistent grid = minb × SMs)
};

extern const TShape kTShapesA[];
extern const int kTShapesA_n;
extern const TShape kTShapesB[];
extern const int kTShapesB_n;

}  // namespace rbns

#define RBNS_TS(R_, C_, W_) \
  { R_, C_, W_, newton_tgj_kernel<R_, C_, W_>, tgj_stage_offset<R_, W_>(), tgj_min_blocks<R_>() }
