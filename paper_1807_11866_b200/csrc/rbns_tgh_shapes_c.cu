// rbns_tgh_shapes_c.cu — hybrid tiled Newton kernel instantiations, 168 < N < 200 (12 warps, one CTA per SM).
#include "rbns_tgh.cuh"
#include "rbns_tiled_plan.h"

namespace rbns {
const HShape kHShapesC[] = {
    RBNS_HS(22, 22, 12, 2, false), RBNS_HS(22, 23, 12, 2, false), RBNS_HS(23, 23, 12, 2, false),
    RBNS_HS(23, 24, 12, 2, false), RBNS_HS(24, 24, 12, 2, false), RBNS_HS(24, 25, 12, 2, false),
    RBNS_HS(25, 25, 12, 2, false),
};
const int kHShapesC_n = int(sizeof(kHShapesC) / sizeof(kHShapesC[0]));
}  // namespace rbns
