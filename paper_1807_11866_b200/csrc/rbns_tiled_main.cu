// rbns_tiled_main.cu — the tiled Newton kernel shapes of the BASELINE configs, compiled with -lineinfo for the
// ncu source pages: the register kernel at N = 97..103 (configs 2 and 4) and N = 49..55 (config 1), the hybrid
// kernel at N = 200 (config 3).  The other shapes (rbns_*_shapes_*.cu) cover every N in (32, 200] and are
// compiled without line tables (they triple the object size).
#include "rbns_tgh.cuh"
#include "rbns_tiled_plan.h"

namespace rbns {
const TShape kTShapesMain[] = {RBNS_TS(13, 13, 4), RBNS_TS(7, 7, 3)};  // config 1: three warps (see shapes_a)
const int kTShapesMain_n = int(sizeof(kTShapesMain) / sizeof(kTShapesMain[0]));
const HShape kHShapesMain[] = {RBNS_HS(25, 26, 12, 2, false)};
const int kHShapesMain_n = int(sizeof(kHShapesMain) / sizeof(kHShapesMain[0]));
}  // namespace rbns
