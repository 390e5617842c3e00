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

// INT8-sliced contraction on the tcgen05 tensor cores (rbns_oz.cuh / rbns_oz.cu)
namespace oz {
struct OperandI8 {
  uint8_t* A8 = nullptr;     // [row_tiles][kchunks][slices] shared-memory images of the sliced S
  double* sa = nullptr;      // [row_tiles·128] row scales
  int32_t* cexp = nullptr;   // [k32] column exponents
  double* aff = nullptr;     // [Ql][row_tiles·128] affine columns (added by the epilogue in binary64)
  int k32 = 0, kchunks = 0, Ql = 0;
  int64_t row_tiles = 0;
};
int slices();                              // digits per operand entry (compile-time RBNS_OZ_SLICES)
cudaError_t prepare();                     // function attributes, call with the model's device current
bool supported(int K, int Ql, int max_smem);  // K = θ ⊗ u columns, Ql = affine columns
// slices the leading K columns of S (rows × ldS) and gathers the Ql affine columns that follow them
cudaError_t build_operand(const double* S, int64_t rows, int K, int ldS, int Ql, OperandI8* op);
void free_operand(OperandI8* op);
int64_t operand_bytes(const OperandI8& op);
size_t scratch_b8_bytes(const OperandI8& op, int64_t cap);  // per-call buffers for `cap` samples per launch
size_t scratch_sb_bytes(int64_t cap);
// Y[i][r] = Σ_κ X[i][κ] S[r][κ] for the n samples act[0..n) (NULL = identity): slices X, runs the GEMM
cudaError_t launch(const OperandI8& op, const int32_t* act, int n, const double* u, const double* wts, int N, int Ne,
                   int Qb, int Ql, bool zero_u, uint8_t* B8, double* sb, double* out, int64_t ldo, int num_sms,
                   cudaStream_t st, int64_t B = 0);
// checked builds: this translation unit's failed-check counters
int debug_checks(int* line, unsigned long long* count);
}  // namespace oz

// checked builds (-DRBNS_CHECKED): this translation unit's failed-check counters (first source line, count)
int newton_debug_checks(int* line, unsigned long long* count);

// records msg as the calling thread's rbns_last_error_message() and returns code (entry points outside rbns.cu)
int set_last_error(int code, const std::string& msg);

}  // namespace rbns
