// rbns_tgj_shapes_b.cu — tiled Gauss–Jordan Newton kernel instantiations, 64 < N ≤ 103 (RT = 9 .. 13, two CTAs
// per SM).  N = 104 (RT 13, CT 14) would need four register column tiles per warp: the rank-1 kernels take it.
#include "rbns_tgj.cuh"
#include "rbns_tiled_plan.h"

namespace rbns {
const TShape kTShapesB[] = {
    RBNS_TS(9, 9, 4),   RBNS_TS(9, 10, 4),  RBNS_TS(10, 10, 4), RBNS_TS(10, 11, 4), RBNS_TS(11, 11, 4),
    RBNS_TS(11, 12, 4), RBNS_TS(12, 12, 4), RBNS_TS(12, 13, 4),
};
const int kTShapesB_n = int(sizeof(kTShapesB) / sizeof(kTShapesB[0]));
}  // namespace rbns
