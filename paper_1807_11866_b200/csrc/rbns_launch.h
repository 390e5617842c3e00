// rbns_launch.h — host-side launch entry points shared between the library's translation units.
#pragma once

#include <cuda_runtime.h>

#include "rbns_common.cuh"

namespace rbns {

struct NewtonParams;

bool newton_supported(int N);
cudaError_t launch_newton_update(const NewtonParams& p, cudaStream_t st);

}  // namespace rbns
