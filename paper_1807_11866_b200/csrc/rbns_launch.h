// rbns_launch.h — host-side launch entry points shared between the library's translation units.
#pragma once

#include <cuda_runtime.h>

#include <string>

#include "rbns_common.cuh"

namespace rbns {

struct NewtonParams;

bool newton_supported(int N);
// J block layout the Newton kernels for N read (jidx): 1 when the tiled Gauss–Jordan kernel handles N
int newton_layout(int N);
// per-device setup (function attributes) for the Newton kernels of size N; call with the model's device current
cudaError_t newton_prepare(int N);
// launches the Newton-update kernel(s) for p on st; *launches receives the number of kernels launched
cudaError_t launch_newton_update(const NewtonParams& p, cudaStream_t st, int* launches);

// checked builds (-DRBNS_CHECKED): this translation unit's failed-check counters (first source line, count)
int newton_debug_checks(int* line, unsigned long long* count);

// records msg as the calling thread's rbns_last_error_message() and returns code (entry points outside rbns.cu)
int set_last_error(int code, const std::string& msg);

}  // namespace rbns
