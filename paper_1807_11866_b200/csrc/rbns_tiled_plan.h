// rbns_tiled_plan.h — the instantiated shapes of the tiled Gauss–Jordan Newton kernels (register kernel
// rbns_tgj.cuh, hybrid register/shared-memory kernel rbns_tgh.cuh).  The instantiations live in their own
// translation units (rbns_tgj_shapes_{a,b}.cu, rbns_tgh_shapes_{a,b,c}.cu, compiled in parallel); rbns_newton.cu
// plans and launches through these tables.
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

// hybrid register/shared-memory tiled kernel (rbns_tgh.cuh) <rt, ct, nw, reg>
struct HShape {
  int rt, ct, nw;
  void (*kern)(const NewtonParams);
  size_t smem;
  int minb;        // resident CTAs per SM
  bool test_only;  // instantiated for the tests (RBNS_NEWTON=tgh), not the default for its N
};

extern const TShape kTShapesMain[];
extern const int kTShapesMain_n;
extern const HShape kHShapesMain[];
extern const int kHShapesMain_n;
extern const TShape kTShapesA[];
extern const int kTShapesA_n;
extern const TShape kTShapesB[];
extern const int kTShapesB_n;
extern const HShape kHShapesA[];
extern const int kHShapesA_n;
extern const HShape kHShapesB[];
extern const int kHShapesB_n;
extern const HShape kHShapesC[];
extern const int kHShapesC_n;

}  // namespace rbns

#define RBNS_TS(R_, C_, W_) \
  { R_, C_, W_, newton_tgj_kernel<R_, C_, W_>, tgj_stage_offset<R_, W_>(), tgj_min_blocks<R_>(W_) }
#define RBNS_HS(R_, C_, W_, G_, T_)                                                                           \
  { R_, C_, W_, newton_tgh_kernel<R_, C_, W_, G_>, tgh_smem_bytes<R_, C_, W_, G_>(), tgh_min_blocks<W_, G_>(), T_ }
