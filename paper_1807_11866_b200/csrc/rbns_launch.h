// rbns_launch.h — host-side launch entry points shared between the library's translation units.
#pragma once

#include <cuda_runtime.h>

#include "rbns_common.cuh"

namespace rbns {

struct NewtonParams;

bool newton_supported(int N);
// launches the Newton-update kernel(s) for p on st; *launches receives the number of kernels launched
cudaError_t launch_newton_update(const NewtonParams& p, cudaStream_t st, int* launches);

}  // namespace rbns
