// rbns_tgh_shapes_b.cu — hybrid tiled Newton kernel instantiations, 128 ≤ N ≤ 168 (12 warps: one shared slot
// and one register slot per warp, one CTA per SM; replaces the rank-1 2-CTA cluster kernel there).
#include "rbns_tgh.cuh"
#include "rbns_tiled_plan.h"

namespace rbns {
const HShape kHShapesB[] = {
    RBNS_HS(16, 17, 12, 2, false), RBNS_HS(17, 17, 12, 2, false), RBNS_HS(17, 18, 12, 2, false),
    RBNS_HS(18, 18, 12, 2, false), RBNS_HS(18, 19, 12, 2, false), RBNS_HS(19, 19, 12, 2, false),
    RBNS_HS(19, 20, 12, 2, false), RBNS_HS(20, 20, 12, 2, false), RBNS_HS(20, 21, 12, 2, false),
    RBNS_HS(21, 21, 12, 2, false), RBNS_HS(21, 22, 12, 2, false),
};
const int kHShapesB_n = int(sizeof(kHShapesB) / sizeof(kHShapesB[0]));
}  // namespace rbns
