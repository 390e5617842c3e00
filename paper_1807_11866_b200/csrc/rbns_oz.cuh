// rbns_oz.cuh — K1+K2 on the 5th-generation tensor cores: the FP64 contraction GEMM
//
//   Y[b][r] = Σ_κ X[b][κ] · S[r][κ]                       (same operands and output as rbns_contract.cuh)
//
// evaluated as exact INT8 tcgen05 MMAs over error-free slices of both operands (the Ozaki splitting).
// tcgen05 has no f64 kind; the DMMA path of rbns_contract.cuh tops out at the 37 TF/s
// FP64 tensor peak, the INT8 path of the same SM runs 8192 MAC/clk.
//
// Splitting.  Columns are first equilibrated by powers of two (S[·][κ]·2^{-c_κ}, X[·][κ]·2^{c_κ}: exact), then
// every row v of either operand is scaled by a power of two to v' ∈ (−½, ½) and written in balanced
// radix-256 digits,
//     v' = d₀·2⁻⁷ + Σ_{i=1..s−1} d_i·2^{−7−8i} + ε,   d₀ ∈ [−64, 64],  d_i ∈ [−128, 127],  |ε| ≤ 2^{−8s},
// every step exact (scalings by powers of two, one rounding to an integer multiple of 2^{−8s+1}).  With s = 8
// the digits carry 63 bits: |ε| ≤ 2⁻⁶⁴ relative to the row's largest entry.  The product is
//     Σ_κ x'_κ s'_κ = Σ_g 2^{−14−8g} Σ_{i+j=g} Σ_κ dˣ_i[κ] dˢ_j[κ]   +  O(2⁻⁶²)·max|x'|·max|s'| per term,
// keeping the pairs with i + j < s (36 INT8 GEMMs).  Each group g accumulates exactly in int32
// (|Σ| ≤ 8·K·2¹⁴ < 2³¹ for K < 16 000) in its own TMEM columns; the epilogue converts the groups to binary64,
// sums them smallest first and applies the two row scales.  No atomics, no data-dependent order: results are
// bitwise reproducible and independent of the batch composition.
//
// The affine columns (X = [ν]θ_a, S = A_a[r]; a handful of columns whose magnitudes differ from the θ ⊗ u blocks by
// orders of magnitude) stay out of the sliced GEMM: the epilogue adds Σ_a w_a(b)·A_a[r] in binary64.  The u = 0
// launch of the first Newton step is that sum alone (oz_affine_kernel, bound by the J write).
//
// Kernel (one CTA per SM, 320 threads): output tile = 128 S-rows (MMA M) × 64 samples × s = 8 accumulator groups =
// all 512 TMEM columns.  Both operands are stored in global memory as ready-made shared-memory images (K-major,
// no swizzle: 8-row × 16-byte core matrices), so a stage (32 κ: 8 A images of 4 KB + 16 KB of X images) is two
// cp.async.bulk copies into a 4-stage mbarrier ring.  The X slices of a stage are stacked along N, so one MMA of
// N = 256 takes an A slice against four X slices: 12 MMAs per stage for the 36 products.  Warp 0 = TMA
// producer, warp 1 = MMA issuer (one elected lane, warp-uniform path) and TMEM owner, warps 2–9 = epilogue
// (tcgen05.ld, two warps per TMEM lane quadrant).  Measured per tile: 28.8k clocks of MMAs, at
// the shared-memory bandwidth of the 168 KB a stage moves, then 6.4k clocks of accumulator drain.
#pragma once

#include <cuda.h>

#include "rbns_common.cuh"

namespace rbns {
namespace oz {

#ifndef RBNS_OZ_SLICES
#define RBNS_OZ_SLICES 8
#endif
#ifndef RBNS_OZ_STAGES
#define RBNS_OZ_STAGES 4
#endif
constexpr int kS = RBNS_OZ_SLICES;            // digits per operand entry
constexpr int kTM = 128;                      // S rows per tile (MMA M, TMEM lanes)
#ifndef RBNS_OZ_TN
#define RBNS_OZ_TN 64
#endif
constexpr int kTN = RBNS_OZ_TN;               // samples per tile (MMA N, TMEM columns per group)
constexpr int kKC = 32;                       // κ per stage = K of one kind::i8 MMA
constexpr int kStages = RBNS_OZ_STAGES;
constexpr int kAImg = kTM * kKC;              // bytes of one A slice image
constexpr int kBImg = kTN * kKC;
constexpr int kAStage = kS * kAImg;
constexpr int kBStage = kS * kBImg;
constexpr int kStageBytes = kAStage + kBStage;
#ifndef RBNS_OZ_STREAM_J
#define RBNS_OZ_STREAM_J 0     // 1: J written with streaming (evict-first) stores
#endif
#ifndef RBNS_OZ_EPI_BACKOFF
#define RBNS_OZ_EPI_BACKOFF 0  // ns the epilogue warps sleep between probes of the accumulator barrier (0: spin)
#endif
#ifndef RBNS_OZ_EPI_WARPS
#define RBNS_OZ_EPI_WARPS 8
#endif
constexpr int kEpiWarps = RBNS_OZ_EPI_WARPS;  // 4 or 8: one or two warps per TMEM lane quadrant (the columns split)
constexpr int kThreads = (2 + kEpiWarps) * 32;
static_assert(kEpiWarps == 4 || kEpiWarps == 8, "epilogue warps");
constexpr uint32_t kTmemCols = 512;
static_assert(kS * kTN <= 512, "accumulator groups must fit the 512 TMEM columns");
static_assert(kS >= 2 && kS <= 8, "slices");

constexpr int kMaxAff = 16;                   // affine columns handled by the epilogue (more: DMMA path)
constexpr size_t kSmemBytes =
    size_t(kStages) * kStageBytes + (2 * kStages + 2) * sizeof(uint64_t) + 16 + size_t(kTN) * (kMaxAff + 1) * sizeof(double);

// byte offset of (row, kk) inside an image of ROWS rows × 32 κ: two 16-byte K chunks, row-contiguous inside
// a chunk (the canonical K-major no-swizzle layout: LBO = ROWS·16 between K chunks, SBO = 128 between 8-row groups)
__host__ __device__ inline int img_offset(int rows, int row, int kk) { return (kk >> 4) * (rows * 16) + row * 16 + (kk & 15); }

__device__ __forceinline__ double pow2(int e) { return __hiloint2double((1023 + e) << 20, 0); }  // |e| < 1022

// Digits of v' ∈ (−½, ½): F = rint(v'·2^{8s−1}) is exact for every binary64 whose low bits reach no further than
// 2^{−8s+1} (|ε| ≤ 2^{−8s} otherwise), and the balanced radix-256 digits of the integer F are the bytes of
// (F + C) xor C with C = 0x80 in every byte below the top one: adding 128 per position makes the unsigned bytes
// b_i of F + C the shifted digits d_i + 128 (the carries are the balancing), and x − 128 ≡ x xor 0x80 mod 256.
// d₀ ∈ [−64, 64] is the signed top byte.  One FP64 multiply, one conversion and two 64-bit integer operations
// per entry.  (The first form rounded to nearest digit by digit in binary64: 8 FP64 steps per entry, 0.75 ms
// per 65 536-sample launch of oz_slice_X against 0.3 ms.)
constexpr unsigned long long kBal = 0x0080808080808080ull >> (8 * (8 - kS));
__host__ __device__ __forceinline__ unsigned long long digits_packed(double vs) {
  const double f = vs * double(1ull << (8 * kS - 1));
#ifdef __CUDA_ARCH__
  const long long F = __double2ll_rn(f);
#else
  const long long F = llrint(f);
#endif
  return ((unsigned long long)F + kBal) ^ kBal;
}
__host__ __device__ __forceinline__ void digits(double vs, int (&d)[kS]) {
  const unsigned long long t = digits_packed(vs);
#pragma unroll
  for (int i = 0; i < kS; ++i) d[i] = int((signed char)((t >> (8 * (kS - 1 - i))) & 0xffu));
}

// Eight entries (one 8-κ item) -> the item's 8 bytes of every slice image: digit i of the entries in the two words
// of slice i (entry e in byte e).  A 4×4 byte transpose of the high and of the low words of four packed digit
// strings puts digit i of four entries into one word.
__device__ __forceinline__ void pack_item(const double (&v)[8], uint32_t (&w)[kS][2]) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    if constexpr (kS == 8) {
      uint32_t hi[4], lo[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const unsigned long long t = digits_packed(v[4 * h + e]);
        hi[e] = uint32_t(t >> 32);
        lo[e] = uint32_t(t);
      }
      const uint32_t h01a = __byte_perm(hi[0], hi[1], 0x5140), h23a = __byte_perm(hi[2], hi[3], 0x5140);
      const uint32_t h01b = __byte_perm(hi[0], hi[1], 0x7362), h23b = __byte_perm(hi[2], hi[3], 0x7362);
      const uint32_t l01a = __byte_perm(lo[0], lo[1], 0x5140), l23a = __byte_perm(lo[2], lo[3], 0x5140);
      const uint32_t l01b = __byte_perm(lo[0], lo[1], 0x7362), l23b = __byte_perm(lo[2], lo[3], 0x7362);
      w[0][h] = __byte_perm(h01b, h23b, 0x7632);  // byte 3 of the high words: d₀
      w[1][h] = __byte_perm(h01b, h23b, 0x5410);
      w[2][h] = __byte_perm(h01a, h23a, 0x7632);
      w[3][h] = __byte_perm(h01a, h23a, 0x5410);
      w[4][h] = __byte_perm(l01b, l23b, 0x7632);
      w[5][h] = __byte_perm(l01b, l23b, 0x5410);
      w[6][h] = __byte_perm(l01a, l23a, 0x7632);
      w[kS - 1][h] = __byte_perm(l01a, l23a, 0x5410);
    } else {
      uint32_t acc[kS];
#pragma unroll
      for (int i = 0; i < kS; ++i) acc[i] = 0u;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        int d[kS];
        digits(v[4 * h + e], d);
#pragma unroll
        for (int i = 0; i < kS; ++i) acc[i] |= uint32_t(d[i] & 0xff) << (8 * e);
      }
#pragma unroll
      for (int i = 0; i < kS; ++i) w[i][h] = acc[i];
    }
  }
}

// One warp slices one operand row.  val(κ) returns the (column-equilibrated) entry, 0 beyond the real columns.
// Writes the row's digits into the tile's images and returns the row's output scale 2^{E−6} (v = v'·2^{E+1},
// d₀ weighs 2⁻⁷): NaN for a non-finite row, 0 for a zero row.
// Layout of a stage (32 κ) of ROWS rows: digit i of (row, 16-byte K chunk c) sits at c·CSTRIDE + i·ISTRIDE + row·16.
// Work items are 8 κ wide (k32/8 per row, dealt round-robin to the lanes).  Up to kCacheItems items per lane (rows of
// up to 768 columns) keep their entries in registers between the row-maximum pass and the digit pass; wider rows
// evaluate val twice.
constexpr int kCacheItems = 3;
template <int ROWS, int CSTRIDE, int ISTRIDE, class F>
__device__ __forceinline__ double slice_row(F val, int k32, uint8_t* tile, int row, int lane) {
  const int items = k32 >> 3;
  const bool cached = items <= 32 * kCacheItems;  // warp-uniform
  double cache[kCacheItems][8];
  double m = 0.0;
  bool bad = false;
  if (cached) {
#pragma unroll
    for (int it = 0; it < kCacheItems; ++it) {
      const int item = lane + 32 * it;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const double v = item < items ? val(item * 8 + e) : 0.0;
        cache[it][e] = v;
        bad |= !(fabs(v) <= 1.7976931348623157e308);
        m = fmax(m, fabs(v));
      }
    }
  } else {
    for (int item = lane; item < items; item += 32) {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const double v = val(item * 8 + e);
        bad |= !(fabs(v) <= 1.7976931348623157e308);
        m = fmax(m, fabs(v));
      }
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    bad |= __shfl_xor_sync(0xffffffffu, int(bad), o) != 0;
  }
  int E = 0;
  double down = 0.0;  // 0 for a zero or non-finite row: every digit 0
  if (!bad && m > 0.0) {
    E = min(max(ilogb(m) + 1, -900), 900);  // 2^{E−1} ≤ m < 2^E
    down = pow2(-(E + 1));
  }
  auto store = [&](int item, const double (&v)[8]) {
    uint32_t w[kS][2];
    pack_item(v, w);
    const int kc = item >> 2, c = (item >> 1) & 1, half = item & 1;
    uint8_t* base = tile + size_t(kc) * kS * (ROWS * 32) + c * CSTRIDE + row * 16 + half * 8;
#pragma unroll
    for (int i = 0; i < kS; ++i) *reinterpret_cast<uint2*>(base + size_t(i) * ISTRIDE) = make_uint2(w[i][0], w[i][1]);
  };
  if (cached) {
#pragma unroll
    for (int it = 0; it < kCacheItems; ++it) {
      const int item = lane + 32 * it;
      if (item < items) {
        double v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] = down == 0.0 ? 0.0 : cache[it][e] * down;
        store(item, v);
      }
    }
  } else {
    for (int item = lane; item < items; item += 32) {
      double v[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) v[e] = down == 0.0 ? 0.0 : val(item * 8 + e) * down;
      store(item, v);
    }
  }
  if (bad) return __longlong_as_double(0x7ff8000000000000ll);
  if (m == 0.0) return 0.0;
  return pow2(E - 6);
}

// ---- S side (once per model) ---------------------------------------------------------------------------------
// column exponents c_κ: 2^{c_κ−1} ≤ max_r |S[r][κ]| < 2^{c_κ}  (0 for an empty column)
__global__ void oz_col_exponents(const double* __restrict__ S, int64_t rows, int K, int ldS, int32_t* __restrict__ cexp) {
  const int k = blockIdx.x;
  double m = 0.0;
  for (int64_t r = threadIdx.x; r < rows; r += blockDim.x) {
    const double v = fabs(S[r * ldS + k]);
    if (v <= 1.7976931348623157e308) m = fmax(m, v);
  }
  __shared__ double red[32];
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < int(blockDim.x >> 5); ++w) m = fmax(m, red[w]);
    cexp[k] = m > 0.0 ? min(max(ilogb(m) + 1, -400), 400) : 0;
  }
}

// A8[row_tile][kc][slice][image(128)], sa[row]: one warp per S row (rows beyond `rows` are zero)
__global__ void oz_slice_S(const double* __restrict__ S, int64_t rows, int K, int ldS, const int32_t* __restrict__ cexp,
                           int k32, uint8_t* __restrict__ A8, double* __restrict__ sa, int64_t rows_pad) {
  const int64_t r = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows_pad) return;
  const double* src = S + r * ldS;
  const bool live = r < rows;
  auto val = [&](int k) -> double { return (live && k < K) ? src[k] * pow2(-cexp[k]) : 0.0; };
  uint8_t* tile = A8 + size_t(r / kTM) * size_t(k32 / kKC) * kAStage;
  const double s = slice_row<kTM, kTM * 16, kAImg>(val, k32, tile, int(r % kTM), lane);
  if (lane == 0) sa[r] = s;
}

// aff[a][r] = S[r][kterms + a]: the affine columns, transposed for the epilogue's row-contiguous loads
__global__ void oz_gather_affine(const double* __restrict__ S, int64_t rows, int ldS, int kterms, int Ql,
                                 double* __restrict__ aff, int64_t rows_pad) {
  const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= int64_t(Ql) * rows_pad) return;
  const int a = int(idx / rows_pad);
  const int64_t r = idx - int64_t(a) * rows_pad;
  aff[idx] = r < rows ? S[r * ldS + kterms + a] : 0.0;
}

// ---- X side (every contraction launch) -----------------------------------------------------------------------
struct SliceXParams {
  const int32_t* act;   // sample ids of this chunk (NULL = identity)
  int32_t n;            // samples of the chunk
  const double* u;      // [B][N]
  const double* wts;    // [B][Qb + Ql] block and affine-column weights
  const int32_t* cexp;  // [k32] column exponents of S
  int32_t N, Ne, Qb, Ql, k32;  // κ = j·Ne + k over the Qb blocks (the Ql affine weights follow the block weights in wts)
  uint8_t* B8;          // [sample_tiles][kc][slice][image(64)]
  double* sb;           // [sample_tiles·64]
  int64_t B;            // samples of the call (sample ids < B; checked builds), 0 = n
};

__global__ void oz_slice_X(const SliceXParams p) {
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);  // position in the chunk (padded to tiles)
  const int lane = threadIdx.x & 31;
  const bool live = i < p.n;
  const int id = live ? (p.act ? p.act[i] : i) : 0;
  RBNS_CHECK(id >= 0 && id < (p.B > 0 ? p.B : p.n));
  RBNS_CHECK(i < ((p.n + kTN - 1) / kTN) * kTN);
  const double* u = p.u + int64_t(id) * p.N;
  const double* w = p.wts + int64_t(id) * (p.Qb + p.Ql);
  const int kterms = p.Qb * p.Ne;
  auto val = [&](int kap) -> double {
    if (!live || kap >= kterms) return 0.0;
    const int j = kap / p.Ne, k = kap - j * p.Ne;
    if (k >= p.N) return 0.0;
    return w[j] * u[k] * pow2(p.cexp[kap]);
  };
  uint8_t* tile = p.B8 + size_t(i / kTN) * size_t(p.k32 / kKC) * kBStage;
  const double s = slice_row<kTN, kS * kTN * 16, kTN * 16>(val, p.k32, tile, i % kTN, lane);
  if (lane == 0) p.sb[i] = s;
}

// ---- u = 0 launch (first Newton step): Y[i][r] = Σ_a w_a(i)·A_a[r], the affine columns alone -------------------------
struct AffineParams {
  const double* aff;   // [Ql][aff_ld]
  int64_t aff_ld;
  const double* wts;   // [B][ldw], the affine weights at column Qb
  const int32_t* act;  // sample ids (NULL = identity)
  int32_t Qb, Ql, ldw, n;
  double* out;         // [n][ldo]
  int64_t ldo;
  int64_t B;           // checked builds: sample ids < B (0 = n)
};

// One CTA = 128 rows (one thread per row, its Ql affine entries in registers) × 64 samples (their weights in shared
// memory); every sample's 128 outputs are one contiguous 1 KB store of the CTA.  Bound by the J write.
__global__ void __launch_bounds__(kTM) oz_affine_kernel(const AffineParams p) {
  __shared__ double wS[kMaxAff * kTN];
  const int64_t r = int64_t(blockIdx.y) * kTM + threadIdx.x;  // row tiles in y (few), sample tiles in x (many)
  const int i0 = blockIdx.x * kTN;
  for (int idx = threadIdx.x; idx < kTN * p.Ql; idx += kTM) {
    const int a = idx / kTN, c = idx % kTN;
    const int i = i0 + c;
    double v = 0.0;
    if (i < p.n) {
      const int id = p.act ? p.act[i] : i;
      RBNS_CHECK(id >= 0 && id < (p.B > 0 ? p.B : p.n));
      v = p.wts[int64_t(id) * p.ldw + p.Qb + a];
    }
    wS[a * kTN + c] = v;
  }
  double aff[kMaxAff];
#pragma unroll
  for (int a = 0; a < kMaxAff; ++a) aff[a] = a < p.Ql ? p.aff[int64_t(a) * p.aff_ld + r] : 0.0;
  __syncthreads();
  RBNS_CHECK(r < p.ldo && r < p.aff_ld);
#pragma unroll 1
  for (int c0 = 0; c0 < kTN; c0 += 8) {
    double y[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) y[e] = 0.0;
#pragma unroll
    for (int a = 0; a < kMaxAff; ++a) {
      if (a < p.Ql) {
        const double* wa = wS + a * kTN + c0;
#pragma unroll
        for (int e = 0; e < 8; ++e) y[e] = fma(wa[e], aff[a], y[e]);
      }
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int i = i0 + c0 + e;
      if (i < p.n) p.out[int64_t(i) * p.ldo + r] = y[e];
    }
  }
}

// ---- tcgen05 wrappers ----------------------------------------------------------------------------------------
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

__device__ __forceinline__ void tmem_alloc(uint32_t* slot) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(slot)), "n"(kTmemCols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t addr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(addr), "n"(kTmemCols) : "memory");
}

// D[tmem] (+)= A[smem] · B[smem]ᵀ, int8 × int8 → int32, M = 128, N = 64, K = 32
__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// arrives on the mbarrier once every tcgen05.mma issued so far by this thread has completed
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}

// 8 consecutive columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, int (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr)
               : "memory");
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile(
      "{\n"
      ".reg .b32 rx;\n"
      ".reg .pred px;\n"
      "elect.sync rx|px, 0xffffffff;\n"
      "selp.u32 %0, 1, 0, px;\n"
      "}\n"
      : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ uint64_t make_desc(uint32_t lo, uint32_t hi) { return (uint64_t(hi) << 32) | lo; }

// shared-memory matrix descriptor: K-major, no swizzle, version 1 (sm_100)
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  return uint64_t((saddr & 0x3ffffu) >> 4) | (uint64_t(lbo_bytes >> 4) << 16) | (uint64_t(sbo_bytes >> 4) << 32) |
         (uint64_t(1) << 46);
}

// instruction descriptor, kind::i8: D = s32, A = B = signed 8-bit, both K-major, M = 128, N = n
__host__ __device__ constexpr uint32_t idesc_n(int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(kTM >> 4) << 24);
}
#ifndef RBNS_OZ_WIDE
#define RBNS_OZ_WIDE 4
#endif
constexpr int kWide = RBNS_OZ_WIDE;  // X slices per MMA (N = 64·kWide ≤ 256)
static_assert(kWide >= 1 && kWide * kTN <= 256, "MMA N");

__host__ __device__ __forceinline__ double i32_to_f64(int x) {
#ifdef __CUDA_ARCH__
  // 2^52 + 2^31 + x as a bit pattern, minus the constant: exact, no I2F
  return __hiloint2double(0x43300000, x ^ int(0x80000000)) - 4503601774854144.0;
#else
  return double(x);
#endif
}

// Σ_g a_g·2^{−8g} for one output from its kS group sums: Horner in binary64, smallest group first.  (Measured and
// not kept: adjacent groups combined exactly in int64, one conversion per pair — the same drain time.)
__host__ __device__ __forceinline__ double combine_groups(const int (&a)[kS]) {
  double t = i32_to_f64(a[kS - 1]);
#pragma unroll
  for (int g = kS - 2; g >= 0; --g) t = fma(t, 0.00390625, i32_to_f64(a[g]));
  return t;
}

// Pipeline ablations and clock64 stamps exist only in the probe build (tools/oz_probe.cu defines RBNS_OZ_PROBE);
// in the library the conditions are compile-time false.
#ifdef RBNS_OZ_PROBE
#define OZ_DBG(p, bit) (((p).dbg & (bit)) != 0)
#define OZ_STAMP(p, cond, slot) \
  do {                          \
    if ((p).trace && (cond)) (p).trace[slot] = clock64(); \
  } while (0)
#else
#define OZ_DBG(p, bit) false
#define OZ_STAMP(p, cond, slot) \
  do {                          \
  } while (0)
#endif

struct GemmParams {
  const uint8_t* A8;  // [row_tiles][kchunks][kS][kAImg]
  const uint8_t* B8;  // [sample_tiles][kchunks][kS][kBImg]
  const double* sa;   // [row_tiles·128]
  const double* sb;   // [sample_tiles·64]
  int32_t kchunks, kc_begin;
  int32_t row_tiles, tiles_per_group;
  int32_t n;
  double* out;        // [n][ldo]
  int64_t ldo;
  const double* aff;  // [Ql][aff_ld] affine columns of S
  int64_t aff_ld;
  const double* wts;  // [B][ldw] weights, the affine ones at column Qb
  const int32_t* act; // sample ids (NULL = identity)
  int32_t Qb, Ql, ldw;
  int64_t B;          // samples of the call (sample ids < B; checked builds), 0 = n
#ifdef RBNS_OZ_PROBE
  long long* trace;   // clock64 stamps of CTA (0,0)
  int32_t dbg;        // 1 = no copies after the ring is primed, 2 = first A slice only, 4 = no stores, 8 = drain only
#endif
};

__global__ void __launch_bounds__(kThreads, 1) oz_gemm_kernel(const GemmParams p) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + size_t(kStages) * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 1);
  double* sbS = reinterpret_cast<double*>(tslot + 4);  // [kTN] X row scales of the tile's samples
  double* wS = sbS + kTN;                               // [Ql][kTN] affine weights of the tile's samples

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int st = blockIdx.x;
  const int rt_begin = blockIdx.y * p.tiles_per_group;
  const int rt_end = min(p.row_tiles, rt_begin + p.tiles_per_group);
  if (rt_begin >= rt_end) return;  // whole CTA, before any barrier or allocation

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, kEpiWarps * 32);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tslot);
  for (int idx = threadIdx.x; idx < kTN * (p.Ql + 1); idx += kThreads) {
    const int a = idx / kTN - 1, c = idx % kTN;
    const int i = st * kTN + c;
    double v = 0.0;
    if (i < p.n) {
      const int id = p.act ? p.act[i] : i;
      RBNS_CHECK(id >= 0 && id < (p.B > 0 ? p.B : p.n));
      if (a < 0)
        v = p.sb[i];
      else
        v = p.wts[int64_t(id) * p.ldw + p.Qb + a];
    }
    if (a < 0)
      sbS[c] = v;
    else
      wS[a * kTN + c] = v;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      const uint64_t pol = l2_policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int rt = rt_begin; rt < rt_end; ++rt) {
        RBNS_CHECK(rt >= 0 && rt < p.row_tiles && p.kc_begin >= 0 && p.kc_begin <= p.kchunks);
        const uint8_t* a = p.A8 + (size_t(rt) * p.kchunks + p.kc_begin) * kAStage;
        const uint8_t* b = p.B8 + (size_t(st) * p.kchunks + p.kc_begin) * kBStage;
        for (int kc = p.kc_begin; kc < p.kchunks; ++kc, a += kAStage, b += kBStage) {
          mbar_wait_backoff(&empty[stage], phase ^ 1u);
          if (OZ_DBG(p, 1) && (rt > rt_begin || kc >= p.kc_begin + kStages)) {
            mbar_arrive(&full[stage]);
          } else {
            mbar_arrive_expect_tx(&full[stage], kStageBytes);
            unsigned char* dst = smem + size_t(stage) * kStageBytes;
            bulk_g2s(dst, a, kAStage, &full[stage], pol);
            bulk_g2s(dst + kAStage, b, kBStage, &full[stage], pol);
          }
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    // The whole warp follows the barriers (a warp-uniform path keeps the tcgen05 issue free of per-instruction
    // election loops); one elected lane issues.  Descriptors: the high word is constant, the low word is the
    // stage's base plus a compile-time slice offset — one uniform add per operand per MMA.
    int stage = 0;
    uint32_t phase = 0, tphase = 0;
    const bool leader = elect_one();
    constexpr uint32_t kDescHi = (128u >> 4) | (1u << 14);  // SBO = 128 B (8-row groups), descriptor version 1
    for (int rt = rt_begin; rt < rt_end; ++rt) {
      mbar_wait(tempty, tphase ^ 1u);  // epilogue drained the previous tile's accumulators
      tphase ^= 1u;
      tc_fence_after();
      OZ_STAMP(p, leader && blockIdx.x == 0 && blockIdx.y == 0 && rt - rt_begin < 4, (rt - rt_begin) * 8 + 0);
      for (int kc = p.kc_begin; kc < p.kchunks; ++kc) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (leader) {
          const uint32_t sbase = smem_u32(smem + size_t(stage) * kStageBytes);
          const uint32_t alo = ((sbase & 0x3ffffu) >> 4) | (uint32_t(kTM * 16 >> 4) << 16);
          const uint32_t blo = (((sbase + kAStage) & 0x3ffffu) >> 4) | (uint32_t(kS * kTN * 16 >> 4) << 16);
          const uint32_t first = kc == p.kc_begin ? 0u : 1u;
          // A slice i meets the X slices j < kS − i.  The X slices of a stage are stacked along N (slice-major
          // rows inside each 16-byte K chunk), and the accumulator groups g = i + j are consecutive TMEM column
          // blocks, so up to four slices go into one MMA of N = 256: A is read once per four products and the
          // stage is bound by the MMA rate, not by shared-memory reads (12 MMAs per stage instead of 36).
#pragma unroll
          for (int i = 0; i < kS; ++i) {
            if (OZ_DBG(p, 2) && i > 0) break;
            const uint64_t ad = make_desc(alo + uint32_t(i) * (kAImg >> 4), kDescHi);
#pragma unroll
            for (int j = 0; j < kS - i; j += kWide) {
              const int w = (kS - i - j) < kWide ? (kS - i - j) : kWide;  // slices in this MMA
              const uint64_t bd = make_desc(blo + uint32_t(j) * (kTN * 16 >> 4), kDescHi);
              mma_i8(tmem + uint32_t(i + j) * kTN, ad, bd, idesc_n(w * kTN), i == 0 ? first : 1u);
            }
          }
          mma_commit(&empty[stage]);  // stage reusable once these MMAs have read it
        }
        __syncwarp();
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1u;
        }
      }
      if (leader) mma_commit(tfull);  // accumulators of this tile complete
      __syncwarp();
      OZ_STAMP(p, leader && blockIdx.x == 0 && blockIdx.y == 0 && rt - rt_begin < 4, (rt - rt_begin) * 8 + 1);
    }
  } else {
    // ---------------- epilogue: TMEM -> binary64 (+ affine columns) -> J buffer ----------------
    const int q = warp & 3;  // TMEM lane quadrant this warp may read
    constexpr int kCols = kTN / (kEpiWarps / 4);  // sample columns per warp
    const int cbeg = ((warp - 2) >> 2) * kCols;
    uint32_t tphase = 0;
    for (int rt = rt_begin; rt < rt_end; ++rt) {
      const int64_t r = int64_t(rt) * kTM + q * 32 + lane;
      RBNS_CHECK(r < p.ldo && r < p.aff_ld);
      // this row's scale and affine entries, fetched while the MMAs of the tile run
      const double sar = p.sa[r];
      double aff[kMaxAff];
#pragma unroll
      for (int a = 0; a < kMaxAff; ++a) aff[a] = a < p.Ql ? p.aff[int64_t(a) * p.aff_ld + r] : 0.0;
#if RBNS_OZ_EPI_BACKOFF
      mbar_wait_backoff(tfull, tphase, RBNS_OZ_EPI_BACKOFF);
#else
      mbar_wait(tfull, tphase);
#endif
      tphase ^= 1u;
      tc_fence_after();
      [[maybe_unused]] const bool tr = blockIdx.x == 0 && blockIdx.y == 0 && rt - rt_begin < 4 && warp == 2 && lane == 0;
      OZ_STAMP(p, tr, (rt - rt_begin) * 8 + 2);
#pragma unroll 1
      for (int c0 = cbeg; c0 < cbeg + kCols; c0 += 8) {
        int v[kS][8];
#pragma unroll
        for (int g = 0; g < kS; ++g) tmem_ld8(tmem + (uint32_t(q * 32) << 16) + uint32_t(g * kTN + c0), v[g]);
        tmem_ld_wait();
        if (c0 + 8 == cbeg + kCols) {
          tc_fence_before();
          mbar_arrive(tempty);
          OZ_STAMP(p, tr, (rt - rt_begin) * 8 + 3);
        }
        if (OZ_DBG(p, 8)) {  // probe: drain only
          if (v[0][0] == 0x7fffffff) p.out[0] = 0.0;
          continue;
        }
        double y[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          int a[kS];
#pragma unroll
          for (int g = 0; g < kS; ++g) a[g] = v[g][e];
          y[e] = combine_groups(a) * sar * sbS[c0 + e];
        }
#pragma unroll
        for (int a = 0; a < kMaxAff; ++a) {
          if (a < p.Ql) {
            const double* wa = wS + a * kTN + c0;
#pragma unroll
            for (int e = 0; e < 8; ++e) y[e] = fma(wa[e], aff[a], y[e]);
          }
        }
        if (!OZ_DBG(p, 4)) {
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int i = st * kTN + c0 + e;
#if RBNS_OZ_STREAM_J
            if (i < p.n) __stcs(p.out + int64_t(i) * p.ldo + r, y[e]);
#else
            if (i < p.n) p.out[int64_t(i) * p.ldo + r] = y[e];
#endif
          }
        }
      }
      OZ_STAMP(p, tr, (rt - rt_begin) * 8 + 4);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem);
}

}  // namespace oz
}  // namespace rbns
