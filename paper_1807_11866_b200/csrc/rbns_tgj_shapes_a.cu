// rbns_tgj_shapes_a.cu — tiled Gauss–Jordan Newton kernel instantiations, 32 < N ≤ 64 (RT = 5 .. 8, four CTAs
// per SM); an N that is not a multiple of 8 has CT = RT, a multiple of 8 has CT = RT + 1 (the right-hand side in
// its own tile).  Below N = 33 the one-warp rank-1 kernels are faster (tools/ntime.py: N = 10 18.5M vs 12.1M
// solves/s, N = 32 4.94M vs 4.77M; N = 40 2.51M vs 3.20M in favour of this kernel).
#include "rbns_tgj.cuh"
#include "rbns_tiled_plan.h"

namespace rbns {
// three warps (two register column tiles each, five CTAs per SM) where the column tiles number ≤ 6, four warps
// above (tools/ntime.py: N = 40 / 48 / 50 +2.4 / +1.8 / +2.5 % with three; N = 56 / 64 −9 / −21 %)
const TShape kTShapesA[] = {
    RBNS_TS(5, 5, 3), RBNS_TS(5, 6, 3), RBNS_TS(6, 6, 3), RBNS_TS(6, 7, 3),
    RBNS_TS(7, 8, 4), RBNS_TS(8, 8, 4), RBNS_TS(8, 9, 4),
};
const int kTShapesA_n = int(sizeof(kTShapesA) / sizeof(kTShapesA[0]));
}  // namespace rbns
