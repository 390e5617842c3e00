// rbns_tgh_shapes_a.cu — hybrid tiled Newton kernel instantiations: 103 < N ≤ 127 (5 warps: two register slots
// + one shared slot per warp, two CTAs per SM) and the test-only shapes (RBNS_NEWTON=tgh).  N = 200 (config 3)
// is in rbns_tiled_main.cu.
#include "rbns_tgh.cuh"
#include "rbns_tiled_plan.h"

namespace rbns {
const HShape kHShapesA[] = {
    RBNS_HS(13, 14, 5, 6, false),   // N = 104
    RBNS_HS(14, 14, 5, 6, false),   // 104 < N < 112
    RBNS_HS(14, 15, 5, 6, false),   // N = 112
    RBNS_HS(15, 15, 5, 6, false),   // 112 < N < 120
    RBNS_HS(15, 16, 5, 6, false),   // N = 120
    RBNS_HS(16, 16, 5, 6, false),   // 120 < N < 128
    RBNS_HS(13, 13, 4, 6, true),    // 96 < N ≤ 103 (the register kernel is faster: tests only)
    RBNS_HS(7, 8, 3, 2, true),      // N = 56 (tests)
};
const int kHShapesA_n = int(sizeof(kHShapesA) / sizeof(kHShapesA[0]));
}  // namespace rbns
