// rbns_oz.cu — host side of the INT8-sliced contraction (rbns_oz.cuh): operand slicing at model create and
// the per-launch pair (X slicing, tcgen05 GEMM).
#include "rbns_oz.cuh"

#include <algorithm>

#include "rbns_launch.h"

namespace rbns {
namespace oz {

int slices() { return kS; }

cudaError_t prepare() {
  return cudaFuncSetAttribute(oz_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmemBytes));
}

bool supported(int K, int Ql, int max_smem) {
  // int32 group sums: at most kS pairs of K products of two bytes
  return size_t(max_smem) >= kSmemBytes && Ql <= kMaxAff && K > 0 &&
         int64_t(kS) * ((K + 31) / 32 * 32) * 128 * 128 < (int64_t(1) << 31);
}

void free_operand(OperandI8* op) {
  for (void* p : {static_cast<void*>(op->A8), static_cast<void*>(op->sa), static_cast<void*>(op->cexp),
                  static_cast<void*>(op->aff)})
    if (p) cudaFree(p);
  *op = OperandI8{};
}

cudaError_t build_operand(const double* S, int64_t rows, int K, int ldS, int Ql, OperandI8* op) {
  *op = OperandI8{};
  op->Ql = Ql;
  op->k32 = (K + kKC - 1) / kKC * kKC;
  op->kchunks = op->k32 / kKC;
  op->row_tiles = (rows + kTM - 1) / kTM;
  const int64_t rows_pad = op->row_tiles * kTM;
  cudaError_t e;
  if ((e = cudaMalloc(&op->A8, size_t(op->row_tiles) * op->kchunks * kAStage)) != cudaSuccess ||
      (e = cudaMalloc(&op->sa, size_t(rows_pad) * sizeof(double))) != cudaSuccess ||
      (e = cudaMalloc(&op->cexp, size_t(op->k32) * sizeof(int32_t))) != cudaSuccess ||
      (e = cudaMalloc(&op->aff, size_t(std::max(Ql, 1)) * rows_pad * sizeof(double))) != cudaSuccess ||
      (e = cudaMemset(op->cexp, 0, size_t(op->k32) * sizeof(int32_t))) != cudaSuccess) {
    free_operand(op);
    return e;
  }
  oz_col_exponents<<<K, 256>>>(S, rows, K, ldS, op->cexp);
  oz_slice_S<<<unsigned((rows_pad + 7) / 8), 256>>>(S, rows, K, ldS, op->cexp, op->k32, op->A8, op->sa, rows_pad);
  if (Ql > 0)
    oz_gather_affine<<<unsigned((int64_t(Ql) * rows_pad + 255) / 256), 256>>>(S, rows, ldS, K, Ql, op->aff, rows_pad);
  if ((e = cudaGetLastError()) != cudaSuccess || (e = cudaDeviceSynchronize()) != cudaSuccess) free_operand(op);
  return e;
}

int64_t operand_bytes(const OperandI8& op) {
  return int64_t(op.row_tiles) * op.kchunks * kAStage + op.row_tiles * kTM * 8 * (1 + op.Ql) + int64_t(op.k32) * 4;
}

size_t scratch_b8_bytes(const OperandI8& op, int64_t cap) { return size_t((cap + kTN - 1) / kTN) * op.kchunks * kBStage; }
size_t scratch_sb_bytes(int64_t cap) { return size_t((cap + kTN - 1) / kTN) * kTN * sizeof(double); }

cudaError_t launch(const OperandI8& op, const int32_t* act, int n, const double* u, const double* wts, int N, int Ne,
                   int Qb, int Ql, bool zero_u, uint8_t* B8, double* sb, double* out, int64_t ldo, int num_sms,
                   cudaStream_t st, int64_t B) {
  if (n <= 0) return cudaSuccess;
  const int sample_tiles = (n + kTN - 1) / kTN;
  if (zero_u) {  // first Newton step: no convective part, the affine sums alone
    AffineParams ap{};
    ap.aff = op.aff;
    ap.aff_ld = op.row_tiles * kTM;
    ap.wts = wts;
    ap.act = act;
    ap.Qb = Qb;
    ap.Ql = Ql;
    ap.ldw = Qb + Ql;
    ap.n = n;
    ap.out = out;
    ap.ldo = ldo;
    ap.B = B;
    oz_affine_kernel<<<dim3(sample_tiles, unsigned(op.row_tiles)), kTM, 0, st>>>(ap);
    return cudaGetLastError();
  }
  {
    SliceXParams sp{};
    sp.act = act;
    sp.n = n;
    sp.u = u;
    sp.wts = wts;
    sp.cexp = op.cexp;
    sp.N = N;
    sp.Ne = Ne;
    sp.Qb = Qb;
    sp.Ql = Ql;
    sp.k32 = op.k32;
    sp.B8 = B8;
    sp.sb = sb;
    sp.B = B;
    oz_slice_X<<<sample_tiles * kTN / 8, 256, 0, st>>>(sp);
  }
  GemmParams gp{};
  gp.A8 = op.A8;
  gp.B8 = B8;
  gp.sa = op.sa;
  gp.sb = sb;
  gp.kchunks = op.kchunks;
  gp.kc_begin = 0;
  gp.row_tiles = int(op.row_tiles);
  gp.n = n;
  gp.out = out;
  gp.ldo = ldo;
  gp.aff = op.aff;
  gp.aff_ld = op.row_tiles * kTM;
  gp.wts = wts;
  gp.act = act;
  gp.Qb = Qb;
  gp.Ql = Ql;
  gp.ldw = Qb + Ql;
  gp.B = B;
  // CTAs per launch: every sample tile, split over row-tile groups until the grid covers a few waves
  const int64_t want = int64_t(4) * num_sms;
  int groups = int(std::max<int64_t>(1, (want + sample_tiles - 1) / sample_tiles));
  groups = int(std::min<int64_t>(groups, std::max<int64_t>(1, op.row_tiles / 2)));
  gp.tiles_per_group = int((op.row_tiles + groups - 1) / groups);
  groups = int((op.row_tiles + gp.tiles_per_group - 1) / gp.tiles_per_group);
  oz_gemm_kernel<<<dim3(sample_tiles, groups), kThreads, kSmemBytes, st>>>(gp);
  return cudaGetLastError();
}

int debug_checks(int* line, unsigned long long* count) {
#ifdef RBNS_CHECKED
  if (cudaMemcpyFromSymbol(line, rbns::g_chk_line, sizeof(int)) != cudaSuccess ||
      cudaMemcpyFromSymbol(count, rbns::g_chk_count, sizeof(unsigned long long)) != cudaSuccess)
    return 2;
#else
  *line = 0;
  *count = 0;
#endif
  return 0;
}

}  // namespace oz
}  // namespace rbns
